// qfs_delta.cuh -- stage 2: Delta = Delta_1(f^(p-1)) mod p, dense, one CTA per surface.
//
// Replaces delta1(g) (polyring.py:335-401) and its inner power_mod_small (nttpower.py:447-507):
// instead of raising the N-term g to the p-th power (an NTT of length 2^21..2^27 over 3..6 helper
// primes in the reference) the carry is assembled from the pieces stage 1 produced,
//     Delta[p*s + rho] = [rho = 0] * A[s]  -  sum_{t >= 0, |t| = 4 - m}  E[rho + p*t] * h[s - t]      (mod p)
// for every residue class rho in [0,p)^4 with |rho| = m*p (m = 0..3) and every s of degree 4(p-1)-m
// (DESIGN.md section 3 derives it; tests/model_factorized.py restates it in numpy).
// That is C(4p+3,3) * C(4p-5,3) exact integer multiply-adds per surface (0.8 M at p=5, 8 M at p=7,
// 148 M at p=11) with no FFT and no floating point.
//
// Mapping.  h sits in shared memory as a zero-padded (dh+9)^3 box so that "s - t" is one subtraction
// of a compile-time offset and out-of-range reads are zeros.  The output is produced slab by slab
// (slab = all exponents with a fixed I1), staged in shared memory and written to HBM with 16-byte
// coalesced stores.  Inside a slab each warp takes one class (rho2, rho3) at a time: the <= 35 tap
// coefficients E[rho + p t] are then warp-uniform registers and the inner loop is
// one LDS.U8 + one IMAD per multiply-add.  Lanes enumerate the (s2, s3) triangle by diagonals
// through a small table, so all 32 lanes stay busy whatever the triangle size.
//
// Output layout: "lex43g" (qfs_shape.cuh) -- entry (I1,I2,I3,I4) at gbase(I1,I2) + I4, every run
// followed by G guard zeros, ZPAD leading zeros.  The slab staged in shared memory uses the same
// guard-banded layout (guards stay zero: the flush re-zeroes what it copied), so the guards and
// the zero pad are (re)written with every surface and need no separate memset.
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct DeltaCfg {
    using S = Shape<P>;
    static constexpr int NT = (P >= 11) ? 512 : 256;
    static constexpr int SB = S::dh + 9;  // box side: 4 zeros below, 4 above
    static constexpr int BOX = SB * SB * SB;
    static constexpr int RBDIM = S::dE + 1;
    static constexpr int NTRI = (S::d + 1) * (S::d + 2) / 2;
    static constexpr int SLAB = qc2(S::D + 2) + S::G * (S::D + 1) + 32;
    static constexpr bool A_IN_SMEM = (P < 11);  // p = 11: the slab needs the room, A is read from HBM
    static constexpr int OFF_E = 0;
    static constexpr int OFF_A = OFF_E + S::NE_pad;
    static constexpr int OFF_RB = OFF_A + (A_IN_SMEM ? S::pitch : 0);
    static constexpr int OFF_TRI = OFF_RB + qround16(2 * RBDIM * RBDIM);
    static constexpr int OFF_BOX = OFF_TRI + qround16(2 * NTRI);
    static constexpr int OFF_SLAB = OFF_BOX + qround16(BOX);
    static constexpr int SMEM = OFF_SLAB + qround16(SLAB);
};

// One class (rho; m = M) of one slab, executed by one warp.
template <int P, int M>
__device__ __forceinline__ void delta_class(const uint8_t* __restrict__ sE, const uint8_t* __restrict__ sA,
                                            const uint16_t* __restrict__ sRB, const uint16_t* __restrict__ sTri,
                                            const uint8_t* __restrict__ sBox, uint8_t* __restrict__ slab,
                                            int s1, int rho1, int rho2, int rho3, int rho4, int n, int lane)
{
    using S = Shape<P>;
    using C = DeltaCfg<P>;
    constexpr int K = 4 - M;                       // degree of the tap polynomial E_rho
    constexpr int CNT = (K + 1) * (K + 2) * (K + 3) / 6;
    constexpr int SB = C::SB;
    const int ns = (S::d - M) - s1;                // (s2,s3,s4) has degree ns
    if (ns < 0) return;

    uint32_t coef[CNT];
    {
        int j = 0;
#pragma unroll
        for (int t1 = 0; t1 <= K; ++t1)
#pragma unroll
            for (int t2 = 0; t2 <= K - t1; ++t2)
#pragma unroll
                for (int t3 = 0; t3 <= K - t1 - t2; ++t3)
                    coef[j++] = sE[sRB[(rho1 + P * t1) * C::RBDIM + rho2 + P * t2] + rho3 + P * t3];
    }
    const int ntri = (ns + 1) * (ns + 2) / 2;
    for (int q = lane; q < ntri; q += 32) {
        const uint32_t e = sTri[q];
        const int kk = e & 255, s2 = e >> 8, s3 = kk - s2;
        const uint8_t* hb = sBox + ((s1 + 4) * SB + (s2 + 4)) * SB + (s3 + 4);
        uint32_t acc = 0;
        int j = 0;
#pragma unroll
        for (int t1 = 0; t1 <= K; ++t1)
#pragma unroll
            for (int t2 = 0; t2 <= K - t1; ++t2)
#pragma unroll
                for (int t3 = 0; t3 <= K - t1 - t2; ++t3)
                    acc += coef[j++] * hb[-((t1 * SB + t2) * SB + t3)];
        uint32_t a = 0;
        if (M == 0) a = sA[qrowbase(S::d, s1, s2) + s3];  // sA: shared copy, or the surface's A in HBM (p = 11)
        const uint32_t r = (a + (uint32_t)P * 400u - acc) % (uint32_t)P;  // acc <= 35*(p-1)^2 < 400p
        const int I2 = P * s2 + rho2, I4 = P * (ns - kk) + rho4;
        slab[((I2 * (2 * n + 3 - I2)) >> 1) + S::G * I2 + I4] = (uint8_t)r;
    }
}

template <int P>
__global__ void __launch_bounds__(DeltaCfg<P>::NT)
k_delta(const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ A_all, const uint8_t* __restrict__ E_all,
        uint8_t* __restrict__ delta_all, int count)
{
    using S = Shape<P>;
    using C = DeltaCfg<P>;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* sE = smem + C::OFF_E;
    const uint8_t* sA = C::A_IN_SMEM ? smem + C::OFF_A : A_all + (size_t)blockIdx.x * S::pitch;
    uint16_t* sRB = reinterpret_cast<uint16_t*>(smem + C::OFF_RB);
    uint16_t* sTri = reinterpret_cast<uint16_t*>(smem + C::OFF_TRI);
    uint8_t* sBox = smem + C::OFF_BOX;
    uint8_t* sSlab = smem + C::OFF_SLAB;
    __shared__ int s_counter;

    const int slot = blockIdx.x;
    if (slot >= count) return;
    const int tid = threadIdx.x, lane = tid & 31;
    const uint8_t* gh = h_all + (size_t)slot * S::Nh_pad;
    uint8_t* gd = delta_all + (size_t)slot * S::Lg_pad;

    {   // stage E, A (16-byte vectors; strides are padded), zero the box, build tables
        const uint4* e4 = reinterpret_cast<const uint4*>(E_all + (size_t)slot * S::NE_pad);
        for (int i = tid; i < S::NE_pad / 16; i += C::NT) reinterpret_cast<uint4*>(sE)[i] = e4[i];
        if (C::A_IN_SMEM) {
            const uint4* a4 = reinterpret_cast<const uint4*>(A_all + (size_t)slot * S::pitch);
            for (int i = tid; i < S::pitch / 16; i += C::NT) reinterpret_cast<uint4*>(smem + C::OFF_A)[i] = a4[i];
        }
        for (int i = tid; i < qround16(C::SLAB) / 16; i += C::NT) reinterpret_cast<uint4*>(sSlab)[i] = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < S::ZPAD / 16; i += C::NT) reinterpret_cast<uint4*>(gd)[i] = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < qround16(C::BOX) / 16; i += C::NT) reinterpret_cast<uint4*>(sBox)[i] = make_uint4(0, 0, 0, 0);
        for (int e = tid; e < C::RBDIM * C::RBDIM; e += C::NT) {
            const int a1 = e / C::RBDIM, a2 = e - a1 * C::RBDIM;
            sRB[e] = (a1 + a2 <= S::dE) ? (uint16_t)qrowbase(S::dE, a1, a2) : (uint16_t)0;
        }
        for (int e = tid; e < (S::d + 1) * (S::d + 1); e += C::NT) {
            const int kk = e / (S::d + 1), s2 = e - kk * (S::d + 1);
            if (s2 <= kk) sTri[kk * (kk + 1) / 2 + s2] = (uint16_t)(kk | (s2 << 8));
        }
    }
    __syncthreads();
    for (int e = tid; e < (S::dh + 1) * (S::dh + 1); e += C::NT) {
        const int u1 = e / (S::dh + 1), u2 = e - u1 * (S::dh + 1);
        const int len = S::dh - u1 - u2;
        if (len < 0) continue;
        const uint8_t* src = gh + qrowbase(S::dh, u1, u2);
        uint8_t* dst = sBox + ((u1 + 4) * C::SB + (u2 + 4)) * C::SB + 4;
        for (int u3 = 0; u3 <= len; ++u3) dst[u3] = src[u3];
    }
    __syncthreads();

#pragma unroll 1
    for (int I1 = 0; I1 <= S::D; ++I1) {
        const int s1 = I1 / P, rho1 = I1 - s1 * P;
        const int n = S::D - I1;
        const int goff = S::gbase(I1, 0);
        const int bytes = qc2(n + 2) + S::G * (n + 1);  // the slab's runs with their guards
        uint8_t* slab = sSlab + (((size_t)(gd + goff)) & 15);
        if (tid == 0) s_counter = 0;
        __syncthreads();
        while (true) {
            int cls = 0;
            if (lane == 0) cls = atomicAdd(&s_counter, 1);
            cls = __shfl_sync(0xffffffffu, cls, 0);
            if (cls >= P * P) break;
            const int rho2 = cls / P, rho3 = cls - rho2 * P;
            const int rs = rho1 + rho2 + rho3;
            const int rho4 = (P - rs % P) % P;
            const int m = (rs + rho4) / P;
            switch (m) {
                case 0: delta_class<P, 0>(sE, sA, sRB, sTri, sBox, slab, s1, rho1, rho2, rho3, rho4, n, lane); break;
                case 1: delta_class<P, 1>(sE, sA, sRB, sTri, sBox, slab, s1, rho1, rho2, rho3, rho4, n, lane); break;
                case 2: delta_class<P, 2>(sE, sA, sRB, sTri, sBox, slab, s1, rho1, rho2, rho3, rho4, n, lane); break;
                default: delta_class<P, 3>(sE, sA, sRB, sTri, sBox, slab, s1, rho1, rho2, rho3, rho4, n, lane); break;
            }
        }
        __syncthreads();
        {   // flush: slab and destination share their alignment mod 16
            uint8_t* dst = gd + goff;
            int head = (16 - (int)(((size_t)dst) & 15)) & 15;
            if (head > bytes) head = bytes;
            if (tid < head) { dst[tid] = slab[tid]; slab[tid] = 0; }
            const int nvec = (bytes - head) >> 4;
            uint4* s4 = reinterpret_cast<uint4*>(slab + head);
            uint4* d4 = reinterpret_cast<uint4*>(dst + head);
            for (int i = tid; i < nvec; i += C::NT) { d4[i] = s4[i]; s4[i] = make_uint4(0, 0, 0, 0); }
            const int done = head + (nvec << 4);
            if (tid < bytes - done) { dst[done + tid] = slab[done + tid]; slab[done + tid] = 0; }
        }
        __syncthreads();
    }
}

// lex43g <-> lex.  TO_G = true: dense lex input -> guard-banded lex43g output (which must be zero-filled
// beforehand); TO_G = false: lex43g input -> dense lex output.  Used by the stage taps only.
template <int P, bool TO_G>
__global__ void k_delta_flip(const uint8_t* __restrict__ in, size_t in_stride, uint8_t* __restrict__ out,
                             size_t out_stride)
{
    using S = Shape<P>;
    const int I1 = blockIdx.x;
    const uint8_t* src = in + (size_t)blockIdx.y * in_stride;
    uint8_t* dst = out + (size_t)blockIdx.y * out_stride;
    const int n = S::D - I1;
    const int base = qc3(S::D + 3) - qc3(n + 3);
    const int total = qc2(n + 2);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        // locate the run: largest I2 with I2(2n+3-I2)/2 <= e
        int lo = 0, hi = n;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (((mid * (2 * n + 3 - mid)) >> 1) <= e) lo = mid; else hi = mid - 1;
        }
        const int rb = (lo * (2 * n + 3 - lo)) >> 1;
        const int I4 = (n - lo) - (e - rb);
        const int gi = S::gbase(I1, lo) + I4;
        if (TO_G) dst[gi] = src[base + e]; else dst[base + e] = src[gi];
    }
}
