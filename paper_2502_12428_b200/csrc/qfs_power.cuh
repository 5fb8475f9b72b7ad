// qfs_power.cuh -- stage 1: the power chain mod p^2, one CTA per surface.
//
// Replaces  power_mod_p(f, p-1)            polyring.py:253-272  (-> g, Fedder test polyring.py:316-332)
// and feeds the factorised Witt carry that replaces delta1 / power_mod_small
//                                           polyring.py:335-401, nttpower.py:447-507.
//
// With tau(a) = a^p mod p^2 (Teichmuller representative) and f_T = sum tau(a_J) x^J the chain
//     f_T^2, f_T^3, ..., f_T^p   (each step: dense product with the <= 35-term f_T, mod p^2)
// yields  H = f_T^(p-2), G = f_T^(p-1), Pw = f_T^p  and from them, exactly:
//     h = H mod p = f^(p-2),   g = G mod p = f^(p-1),
//     A[I] = ((G[I] - tau(g[I])) mod p^2)/p,     E[J] = ((Pw[J] - [p|J] tau(a_{J/p})) mod p^2)/p  (= Delta_1(f)).
// The divisions are exact; a violation raises QFS_ERRBIT_INVARIANT (the reference's
// InternalInvariantError, polyring.py:397-398).  All arithmetic is integer: residues < p^2 <= 121
// in uint8, products accumulated in uint32 (35 * 120^2 < 2^32), one reduction per output.
//
// FULL = false: chain only up to H, then the single coefficient G[cap] -> height 1 or "pending".
// FULL = true : whole chain; writes g, h, A, E for the surface into the chunk workspaces.
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct PowerCfg {
    using S = Shape<P>;
    static constexpr int NT = 128;
    static constexpr int BUF = S::NE_pad;                      // ping/pong polynomial buffers (uint8)
    static constexpr int RBDIM = S::dE + 1;                    // row-base table side
    static constexpr int SMEM = 2 * BUF + 2 * RBDIM * RBDIM;   // + uint16 table
};

template <int P, bool FULL>
__global__ void __launch_bounds__(PowerCfg<P>::NT)
k_power(const uint8_t* __restrict__ coeffs, const uint32_t* __restrict__ list, int count,
        int8_t* __restrict__ heights, uint8_t* __restrict__ fedder_out,
        uint8_t* __restrict__ g_out, uint8_t* __restrict__ h_out,
        uint8_t* __restrict__ A_out, uint8_t* __restrict__ E_out, int* __restrict__ err)
{
    using S = Shape<P>;
    using C = PowerCfg<P>;
    constexpr int PSQ = P * P;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* bufA = smem;
    uint8_t* bufB = smem + C::BUF;
    uint16_t* rbin = reinterpret_cast<uint16_t*>(smem + 2 * C::BUF);
    __shared__ uint32_t s_terms[35];  // j1 | j2<<4 | j3<<8 | j4<<12 | tau<<16
    __shared__ uint8_t s_tau35[35];
    __shared__ uint16_t s_mono[35];   // j1 | j2<<4 | j3<<8
    __shared__ int s_nf;

    const int slot = blockIdx.x;
    if (slot >= count) return;
    const uint32_t sid = list ? list[slot] : (uint32_t)slot;
    const uint8_t* cf = coeffs + (size_t)35 * sid;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = C::NT / 32;

    if (tid == 0) {
        int nf = 0, idx = 0, bad = 0, any = 0;
        for (int j1 = 0; j1 <= 4; ++j1)
            for (int j2 = 0; j1 + j2 <= 4; ++j2)
                for (int j3 = 0; j1 + j2 + j3 <= 4; ++j3, ++idx) {
                    uint32_t c = cf[idx];
                    if (c >= (uint32_t)P) { bad = 1; c = 0; }
                    uint32_t t = 1;
                    for (int i = 0; i < P; ++i) t = t * c % PSQ;  // tau(c) = c^p mod p^2
                    s_tau35[idx] = (uint8_t)t;
                    s_mono[idx] = (uint16_t)(j1 | (j2 << 4) | (j3 << 8));
                    if (c) {
                        any = 1;
                        s_terms[nf++] = (uint32_t)j1 | ((uint32_t)j2 << 4) | ((uint32_t)j3 << 8) |
                                        ((uint32_t)(4 - j1 - j2 - j3) << 12) | (t << 16);
                    }
                }
        s_nf = nf;
        if (bad || !any) atomicOr(err, QFS_ERRBIT_INPUT);
    }
    __syncthreads();
    const int nf = s_nf;
    if (tid < 35) bufA[tid] = s_tau35[tid];
    __syncthreads();

    uint8_t* cur = bufA;
    uint8_t* nxt = bufB;
    const size_t oN = (size_t)slot * S::pitch;

    if (FULL && P == 3) {  // H = f_T itself
        if (tid < 35) h_out[(size_t)slot * S::Nh_pad + tid] = (uint8_t)(cur[tid] % P);
    }

    constexpr int KMAX = FULL ? P : P - 2;
#pragma unroll 1
    for (int k = 2; k <= KMAX; ++k) {
        const int din = 4 * (k - 1), dout = 4 * k;
        for (int e = tid; e < (din + 1) * (din + 1); e += C::NT) {
            const int a1 = e / (din + 1), a2 = e - a1 * (din + 1);
            rbin[e] = (a1 + a2 <= din) ? (uint16_t)qrowbase(din, a1, a2) : (uint16_t)0;
        }
        __syncthreads();
        for (int rf = warp; rf < (dout + 1) * (dout + 1); rf += NW) {
            const int i1 = rf / (dout + 1), i2 = rf - i1 * (dout + 1);
            const int len = dout - i1 - i2;
            if (len < 0) continue;
            const int ob = qrowbase(dout, i1, i2);
            for (int i3 = lane; i3 <= len; i3 += 32) {
                uint32_t acc = 0;
                for (int t = 0; t < nf; ++t) {
                    const uint32_t tm = s_terms[t];
                    const int a1 = i1 - (int)(tm & 15), a2 = i2 - (int)((tm >> 4) & 15), a3 = i3 - (int)((tm >> 8) & 15);
                    if (a1 >= 0 && a2 >= 0 && a3 >= 0 && a1 + a2 + a3 <= din)
                        acc += (tm >> 16) * cur[rbin[a1 * (din + 1) + a2] + a3];
                }
                nxt[ob + i3] = (uint8_t)(acc % PSQ);
            }
        }
        __syncthreads();
        { uint8_t* t = cur; cur = nxt; nxt = t; }
        if (FULL) {
            if (k == P - 2) {
                for (int i = tid; i < S::Nh; i += C::NT) h_out[(size_t)slot * S::Nh_pad + i] = (uint8_t)(cur[i] % P);
            } else if (k == P - 1) {
                int bad = 0;
                for (int i = tid; i < S::pitch; i += C::NT) {
                    uint32_t gi = 0, ai = 0;
                    if (i < S::N) {
                        const uint32_t G = cur[i];
                        gi = G % P;
                        uint32_t t = 1;
                        for (int q = 0; q < P; ++q) t = t * gi % PSQ;
                        const uint32_t num = (G + PSQ - t) % PSQ;
                        if (num % P) bad = 1;
                        ai = num / P;
                    }
                    g_out[oN + i] = (uint8_t)gi;  // pad bytes are written as zero
                    A_out[oN + i] = (uint8_t)ai;
                }
                if (bad) atomicOr(err, QFS_ERRBIT_INVARIANT);
                if (fedder_out && tid == 0) fedder_out[slot] = (cur[S::cap] % P) != 0;
            } else if (k == P) {
                __syncthreads();
                if (tid < 35) {  // subtract tau(a_J) at exponent p*J
                    const int m = s_mono[tid];
                    const int idx = qrowbase(S::dE, P * (m & 15), P * ((m >> 4) & 15)) + P * ((m >> 8) & 15);
                    const uint32_t c = cf[tid] < P ? cf[tid] : 0;
                    cur[idx] = (uint8_t)((cur[idx] + PSQ - (c ? s_tau35[tid] : 0)) % PSQ);
                }
                __syncthreads();
                int bad = 0;
                for (int i = tid; i < S::NE; i += C::NT) {
                    const uint32_t v = cur[i];
                    if (v % P) bad = 1;
                    E_out[(size_t)slot * S::NE_pad + i] = (uint8_t)(v / P);
                }
                if (bad) atomicOr(err, QFS_ERRBIT_INVARIANT);
            }
        }
    }

    if (!FULL) {
        // Fedder coefficient G[cap] = sum_J f_T[J] * H[(p-1,..,p-1) - J]   (mod p)
        if (warp == 0) {
            uint32_t acc = 0;
            for (int t = lane; t < nf; t += 32) {
                const uint32_t tm = s_terms[t];
                const int a1 = P - 1 - (int)(tm & 15), a2 = P - 1 - (int)((tm >> 4) & 15);
                const int a3 = P - 1 - (int)((tm >> 8) & 15), a4 = P - 1 - (int)((tm >> 12) & 15);
                if (a1 >= 0 && a2 >= 0 && a3 >= 0 && a4 >= 0)
                    acc += (tm >> 16) * cur[qrowbase(S::dh, a1, a2) + a3];
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) heights[sid] = (acc % P) ? (int8_t)1 : (int8_t)-1;
        }
    }
}
