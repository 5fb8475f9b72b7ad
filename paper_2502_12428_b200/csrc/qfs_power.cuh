// qfs_power.cuh -- stage 1: powers of the quartic.
//
// Replaces  power_mod_p(f, p-1)            polyring.py:253-272  (-> g, Fedder test polyring.py:316-332)
// and feeds the factorised Witt carry that replaces delta1 / power_mod_small
//                                           polyring.py:335-401, nttpower.py:447-507.
//
// Two kernels:
//
// k_fedder (every surface, one WARP per surface, arithmetic mod p).
//   Height 1 <=> the coefficient of (x1x2x3x4)^(p-1) in f^(p-1) is nonzero.  Only that one
//   coefficient is needed, so the chain f^2, f^3, ... is computed in full only up to
//   j0 = (p-1)/2; above that only the cone of coefficients that can still reach the cap is kept:
//       R_j[K] = (f^j)[cap - K],  K in basis(4(p-1-j)),   R_j[K] = sum_J f[J] * R_{j-1}[K + J].
//   R_{p-1}[0] is the Fedder coefficient.  (p=5: 165 + 35 + 1 outputs instead of 165 + 455 + 969.)
//
// k_power_full (surfaces with height >= 2 only, one CTA per surface, arithmetic mod p^2).
//   With tau(a) = a^p mod p^2 (Teichmuller representative) and f_T = sum tau(a_J) x^J the chain
//       f_T^2, f_T^3, ..., f_T^p   (each step: dense product with the <= 35-term f_T, mod p^2)
//   yields  H = f_T^(p-2), G = f_T^(p-1), Pw = f_T^p  and from them, exactly:
//       h = H mod p = f^(p-2),   g = G mod p = f^(p-1),
//       A[I] = ((G[I] - tau(g[I])) mod p^2)/p,   E[J] = ((Pw[J] - [p|J] tau(a_{J/p})) mod p^2)/p  (= Delta_1(f)).
//   The divisions are exact; a violation raises QFS_ERRBIT_INVARIANT (the reference's
//   InternalInvariantError, polyring.py:397-398).
//
// All arithmetic is integer: residues < p^2 <= 121 in uint8, products accumulated in uint32
// (35 * 120^2 < 2^32), one reduction per output coefficient.  Lanes/threads own OUTPUT monomials
// (taken from a precomputed unrank table) and gather over the nonzero terms of f.
#pragma once
#include "qfs_shape.cuh"

// unrank table: for k = 1..p the monomials of degree 4k in lex order, packed a1 | a2<<8 | a3<<16;
// level k starts at unrank_offset(k).
QFS_HD constexpr int qunrank_offset(int k)
{
    int s = 0;
    for (int j = 1; j < k; ++j) s += qc3(4 * j + 3);
    return s;
}

QFS_HD constexpr int qrb_offset(int d)
{
    int s = 0;
    for (int e = 4; e < d; e += 4) s += (e + 1) * (e + 1);
    return s;
}

template <int P>
struct PowerCfg {
    using S = Shape<P>;
    static constexpr int J0 = (P - 1) / 2;              // last fully computed level of the Fedder chain
    static constexpr int FED_WPS = (P >= 11) ? 4 : 1;    // warps that share one surface (and one cube) in k_fedder
    static constexpr int FED_WARPS = (P >= 11) ? 4 : 8;  // warps per CTA in k_fedder: FED_WARPS / FED_WPS surfaces per CTA
    static constexpr int FED_BUF = qround16(qc3(4 * J0 + 3));
    static constexpr int RB_DEG = 4 * P;                // row-base tables up to this degree
#ifndef QFS_POWER_NT5
#define QFS_POWER_NT5 128
#endif
    static constexpr int FULL_NT = (P <= 5) ? QFS_POWER_NT5 : 256;   // F_5: 128 threads x 12 CTAs 0.59 ms, 256 x 8 0.64, 512 x 4 0.79; F_7: 256 is best
    // CTAs per SM k_power_full is compiled for: shared memory allows 7 (p = 5), 5 (p = 7), 1 (p >= 11); at p <= 5 the 35
    // multiplier coefficients otherwise sit in 55 registers and leave room for four CTAs only (F_5: 0.555 -> 0.49 ms)
#ifndef QFS_POWER_MINB5
#define QFS_POWER_MINB5 12
#endif
    static constexpr int FULL_MINB = (P <= 5) ? QFS_POWER_MINB5 : (P == 7 ? 5 : 1);
    static constexpr int FULL_BUF = S::NE_pad;
    // row-base tables rb_d for d = 4, 8, ..., RB_DEG; table d starts at rb_offset(d)
    static QFS_HD constexpr int rb_offset(int d) { return qrb_offset(d); }
    static constexpr int FED_RB = rb_offset(4 * J0 + 4);       // tables for degrees 4..4*J0
    static constexpr int FULL_RB = rb_offset(4 * P);           // tables for degrees 4..4(p-1)
    // cubes of the box-form products: side = largest OUTPUT coordinate (4*J0 resp. 4p) + 4 pad + 1, so that every
    // read in[o - e_t] stays inside the cube (inputs of lower degree leave the rest zero)
    static constexpr int FED_SB = 4 * J0 + 5;
    static constexpr int FED_BOX = (J0 > 1) ? qround16(FED_SB * FED_SB * FED_SB) : 0;
    static constexpr int FULL_SB = 4 * P + 5;
    static constexpr int FULL_BOX = qround16(FULL_SB * FULL_SB * FULL_SB);
    static constexpr int FED_SMEM = (FED_WARPS / FED_WPS) * (2 * FED_BUF + FED_BOX) + 2 * FED_RB;
    static constexpr int FULL_SMEM = FULL_BUF + FULL_BOX;
};

// term list of one quartic: packed j1 | j2<<4 | j3<<8 | j4<<12 | coef<<16, nonzero terms only
struct TermList {
    uint32_t t[35];
    int n;
};

template <int P>
__device__ __forceinline__ void fill_rb_tables(uint16_t* rb, int max_deg, int tid, int nt)
{
    for (int d = 4; d <= max_deg; d += 4) {
        uint16_t* t = rb + PowerCfg<P>::rb_offset(d);
        for (int e = tid; e < (d + 1) * (d + 1); e += nt) {
            const int a1 = e / (d + 1), a2 = e - a1 * (d + 1);
            t[e] = (a1 + a2 <= d) ? (uint16_t)qrowbase(d, a1, a2) : (uint16_t)0;
        }
    }
}

// out (degree dout = din+4, all C(dout+3,3) coefficients) = in * f  (mod MOD); threads idx0, idx0+stride, ...
template <int MOD>
__device__ __forceinline__ void mul_by_f_full(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int din,
                                              const uint16_t* __restrict__ rb_in, const uint32_t* __restrict__ unrank_out,
                                              const uint32_t* __restrict__ terms, int nf, int idx0, int stride)
{
    const int dout = din + 4;
    const int nout = qc3(dout + 3);
    for (int o = idx0; o < nout; o += stride) {
        const uint32_t m = unrank_out[o];
        const int i1 = m & 255, i2 = (m >> 8) & 255, i3 = m >> 16;
        uint32_t acc = 0;
        for (int t = 0; t < nf; ++t) {
            const uint32_t tm = terms[t];
            const int a1 = i1 - (int)(tm & 15), a2 = i2 - (int)((tm >> 4) & 15), a3 = i3 - (int)((tm >> 8) & 15);
            if ((a1 | a2 | a3) >= 0 && a1 + a2 + a3 <= din) acc += (tm >> 16) * in[rb_in[a1 * (din + 1) + a2] + a3];
        }
        out[o] = (uint8_t)(acc % (uint32_t)MOD);
    }
}

// Box form of the same product, used for the full levels.  The input lives in a zero-initialised cube
// box[(a1+4)*SB^2 + (a2+4)*SB + (a3+4)] (4 zeros below every axis, zeros outside the simplex), so that
// in[o - e_t] is one byte load at a COMPILE-TIME offset from the output's own cube index and needs no
// bounds check; the 35 coefficients of f sit in registers (zero where f has no term).  Two instructions
// per multiply-add instead of ~14.  out (lex order) = in * f mod MOD for outputs idx0, idx0+stride, ...
template <int MOD, int SB>
__device__ __forceinline__ void mul_by_f_box(const uint8_t* __restrict__ box, uint8_t* __restrict__ out, int dout,
                                             const uint32_t* __restrict__ unrank_out, const uint32_t (&c)[35],
                                             int idx0, int stride)
{
    const int nout = qc3(dout + 3);
    for (int o = idx0; o < nout; o += stride) {
        const uint32_t m = unrank_out[o];
        const uint8_t* b = box + (((int)(m & 255) + 4) * SB + (int)((m >> 8) & 255) + 4) * SB + (int)(m >> 16) + 4;
        uint32_t acc = 0;
        int t = 0;
#pragma unroll
        for (int j1 = 0; j1 <= 4; ++j1)
#pragma unroll
            for (int j2 = 0; j2 <= 4 - j1; ++j2)
#pragma unroll
                for (int j3 = 0; j3 <= 4 - j1 - j2; ++j3) {
                    acc += c[t] * b[-((j1 * SB + j2) * SB + j3)];
                    ++t;
                }
        // acc <= 35 (MOD-1)^2 < 2^32 / MOD: the magic-multiply quotient is exact
        out[o] = (uint8_t)(acc - __umulhi(acc, (uint32_t)(0xFFFFFFFFu / MOD + 1)) * (uint32_t)MOD);
    }
}

// lex -> box copy of a degree-deg form (the cube's zeros outside the simplex are never touched)
template <int SB>
__device__ __forceinline__ void lex_to_box(const uint8_t* __restrict__ lex, uint8_t* __restrict__ box, int deg,
                                           const uint32_t* __restrict__ unrank_deg, int idx0, int stride)
{
    const int n = qc3(deg + 3);
    for (int o = idx0; o < n; o += stride) {
        const uint32_t m = unrank_deg[o];
        box[(((int)(m & 255) + 4) * SB + (int)((m >> 8) & 255) + 4) * SB + (int)(m >> 16) + 4] = lex[o];
    }
}

// ---------------------------------------------------------------------------------------------
// Fedder test: height 1 iff the coefficient of (x1 x2 x3 x4)^(p-1) in f^(p-1) is nonzero (polyring.py:316-332).
// p - 1 = 2 J0, so that coefficient is a single dot product of F = f^J0 with its own reflection,
//     [f^(p-1)]_cap = sum_K F[K] * F[cap - K],     K in basis(4 J0) with every K_i <= p-1,
// and only the levels f^2 .. f^J0 are ever computed (box form: coefficients of f in registers, compile-time tap offsets).
// A group of WPS warps works on one surface: one warp for p <= 7 (FED_WARPS surfaces per CTA), the whole four-warp CTA for
// p >= 11, where the cube of the box form (15.6 / 24.4 KB) would otherwise leave room for 8 / 4 warps per SM.
template <int P>
__global__ void __launch_bounds__(PowerCfg<P>::FED_WARPS * 32)
k_fedder(const uint8_t* __restrict__ coeffs, int count, const uint32_t* __restrict__ unrank,
         int8_t* __restrict__ heights, int* __restrict__ err)
{
    using C = PowerCfg<P>;
    constexpr int WPS = C::FED_WPS, GT = 32 * WPS;     // warps / threads per surface
    constexpr int SPC = C::FED_WARPS / WPS;            // surfaces per CTA
    extern __shared__ __align__(16) uint8_t smem[];
    uint16_t* rb = reinterpret_cast<uint16_t*>(smem + SPC * (2 * C::FED_BUF + C::FED_BOX));
    __shared__ int s_dot[SPC];
    const int tid = threadIdx.x, lane = tid & 31;
    const int grp = tid / GT, gt = tid - grp * GT;     // surface of the CTA, thread inside its group
    auto gsync = [&]() { if (WPS == 1) __syncwarp(); else __syncthreads(); };   // WPS > 1: one surface per CTA
    static_assert(WPS == 1 || SPC == 1, "several warps per surface: one surface per CTA");
    fill_rb_tables<P>(rb, 4 * C::J0, tid, C::FED_WARPS * 32);
    if (tid < SPC) s_dot[tid] = 0;
    __syncthreads();

    const int sid = blockIdx.x * SPC + grp;
    if (sid >= count) return;                          // whole groups leave together (WPS > 1: the whole CTA)
    const uint8_t* cf = coeffs + (size_t)35 * sid;
    uint8_t* bufA = smem + (size_t)grp * (2 * C::FED_BUF + C::FED_BOX);
    uint8_t* bufB = bufA + C::FED_BUF;
    uint8_t* box = bufB + C::FED_BUF;  // cube of the box-form products
    if (C::J0 > 1)
        for (int i = gt; i < C::FED_BOX / 16; i += GT) reinterpret_cast<uint4*>(box)[i] = make_uint4(0, 0, 0, 0);

    // input checks (residues < p, not the zero form) by the group's first warp; every thread keeps the 35 coefficients
    if (gt < 32) {
        const uint32_t c0 = cf[lane];
        const uint32_t c1 = lane < 3 ? cf[32 + lane] : 0;
        const bool bad = (c0 >= (uint32_t)P) || (c1 >= (uint32_t)P);
        const unsigned badm = __ballot_sync(0xffffffffu, bad);
        const unsigned any = __ballot_sync(0xffffffffu, (c0 != 0 && c0 < (uint32_t)P) || (c1 != 0 && c1 < (uint32_t)P));
        if (lane == 0 && (badm || !any)) atomicOr(err, QFS_ERRBIT_INPUT);
        bufA[lane] = (uint8_t)(c0 < (uint32_t)P ? c0 : 0);
        if (lane < 3) bufA[32 + lane] = (uint8_t)(c1 < (uint32_t)P ? c1 : 0);
    }
    gsync();

    uint8_t* cur = bufA;
    uint8_t* nxt = bufB;
    // levels f^2 .. f^J0 in box form
    if (C::J0 > 1) {
        uint32_t c[35];
#pragma unroll
        for (int t = 0; t < 35; ++t) c[t] = cur[t];
#pragma unroll 1
        for (int j = 2; j <= C::J0; ++j) {
            lex_to_box<C::FED_SB>(cur, box, 4 * (j - 1), unrank + qunrank_offset(j - 1), gt, GT);
            gsync();
            mul_by_f_box<P, C::FED_SB>(box, nxt, 4 * j, unrank + qunrank_offset(j), c, gt, GT);
            gsync();
            uint8_t* t = cur; cur = nxt; nxt = t;
        }
    }
    // the dot product of F = f^J0 with its reflection about cap = (p-1, p-1, p-1, p-1)
    {
        constexpr int dF = 4 * C::J0, nF = qc3(dF + 3);
        const uint16_t* rbi = rb + C::rb_offset(dF);
        const uint32_t* un = unrank + qunrank_offset(C::J0);
        uint32_t acc = 0;
        for (int o = gt; o < nF; o += GT) {
            const uint32_t m = un[o];
            const int k1 = m & 255, k2 = (m >> 8) & 255, k3 = m >> 16, k4 = dF - k1 - k2 - k3;
            if (k1 < P && k2 < P && k3 < P && k4 < P)
                acc += (uint32_t)cur[o] * cur[rbi[(P - 1 - k1) * (dF + 1) + (P - 1 - k2)] + (P - 1 - k3)];
        }
        acc = __reduce_add_sync(0xffffffffu, acc % (uint32_t)P);
        if (WPS == 1) {
            if (lane == 0) heights[sid] = (acc % (uint32_t)P) ? (int8_t)1 : (int8_t)-1;
        } else {
            if (lane == 0) atomicAdd(&s_dot[grp], (int)(acc % (uint32_t)P));
            __syncthreads();
            if (gt == 0) heights[sid] = (s_dot[grp] % P) ? (int8_t)1 : (int8_t)-1;
        }
    }
}

// ---------------------------------------------------------------------------------------------
template <int P>
__global__ void __launch_bounds__(PowerCfg<P>::FULL_NT, PowerCfg<P>::FULL_MINB)
k_power_full(const uint8_t* __restrict__ coeffs, const uint32_t* __restrict__ list, int count,
             const uint32_t* __restrict__ unrank, uint8_t* __restrict__ fedder_out,
             uint8_t* __restrict__ g_out, uint8_t* __restrict__ h_out,
             uint8_t* __restrict__ A_out, uint8_t* __restrict__ E_out, int* __restrict__ err)
{
    using S = Shape<P>;
    using C = PowerCfg<P>;
    constexpr int PSQ = P * P;
    constexpr int NT = C::FULL_NT;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* cur = smem;                    // the current level, lex order
    uint8_t* box = smem + C::FULL_BUF;      // the same level as a zero-padded cube (input of the next product)
    __shared__ uint8_t s_tau35[36];

    const int slot = blockIdx.x;
    if (slot >= count) return;
    const uint32_t sid = list ? list[slot] : (uint32_t)slot;
    const uint8_t* cf = coeffs + (size_t)35 * sid;
    const int tid = threadIdx.x;
    const uint32_t* unrank4 = unrank + qunrank_offset(1);

    for (int i = tid; i < C::FULL_BOX / 16; i += NT) reinterpret_cast<uint4*>(box)[i] = make_uint4(0, 0, 0, 0);
    if (tid < 32) {  // warp 0: Teichmuller lift tau(c) = c^p mod p^2 of the 35 coefficients
        const int lane = tid;
        uint32_t c[2] = {cf[lane], lane < 3 ? (uint32_t)cf[32 + lane] : 0u};
        uint32_t tau[2];
        bool bad = false;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (c[q] >= (uint32_t)P) { bad = true; c[q] = 0; }
            uint32_t t = 1;
            for (int i = 0; i < P; ++i) t = t * c[q] % PSQ;
            tau[q] = t;
        }
        const unsigned badm = __ballot_sync(0xffffffffu, bad);
        const unsigned nz = __ballot_sync(0xffffffffu, (c[0] | c[1]) != 0);
        if (lane == 0 && (badm || !nz)) atomicOr(err, QFS_ERRBIT_INPUT);
        s_tau35[lane] = (uint8_t)tau[0];
        cur[lane] = (uint8_t)tau[0];
        if (lane < 3) { s_tau35[32 + lane] = (uint8_t)tau[1]; cur[32 + lane] = (uint8_t)tau[1]; }
    }
    __syncthreads();
    uint32_t c[35];  // f_T in registers: the multiplier of every level
#pragma unroll
    for (int t = 0; t < 35; ++t) c[t] = s_tau35[t];
    const size_t oN = (size_t)slot * S::pitch;

    if (P == 3) {  // H = f_T itself
        if (tid < 35) h_out[(size_t)slot * S::Nh_pad + tid] = (uint8_t)(cur[tid] % P);
    }
#pragma unroll 1
    for (int k = 2; k <= P; ++k) {
        lex_to_box<C::FULL_SB>(cur, box, 4 * (k - 1), unrank + qunrank_offset(k - 1), tid, NT);
        __syncthreads();
        mul_by_f_box<PSQ, C::FULL_SB>(box, cur, 4 * k, unrank + qunrank_offset(k), c, tid, NT);
        __syncthreads();
        if (k == P - 2) {
            for (int i = tid; i < S::Nh; i += NT) h_out[(size_t)slot * S::Nh_pad + i] = (uint8_t)(cur[i] % P);
        } else if (k == P - 1) {
            int bad = 0;
            for (int i = tid; i < S::pitch; i += NT) {
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
            if (tid < 35) {  // subtract tau(a_J) at exponent p*J
                const uint32_t mm = unrank4[tid];
                const int idx = qrowbase(S::dE, P * (mm & 255), P * ((mm >> 8) & 255)) + P * (mm >> 16);
                const uint32_t cc = cf[tid] < P ? cf[tid] : 0;
                cur[idx] = (uint8_t)((cur[idx] + PSQ - (cc ? s_tau35[tid] : 0)) % PSQ);
            }
            __syncthreads();
            int bad = 0;
            for (int i = tid; i < S::NE; i += NT) {
                const uint32_t v = cur[i];
                if (v % P) bad = 1;
                E_out[(size_t)slot * S::NE_pad + i] = (uint8_t)(v / P);
            }
            if (bad) atomicOr(err, QFS_ERRBIT_INVARIANT);
        }
    }
}
