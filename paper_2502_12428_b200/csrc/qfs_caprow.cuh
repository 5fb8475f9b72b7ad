// qfs_caprow.cuh -- the decisive row of the first operator application, before the operator matrix exists.
//
// height_matrix (height.py:135-144) stops at the first step k with (M^k g)[cap] != 0.  For the first step that is ONE row of M:
//     v1[cap] = sum_c M[cap, c] g[c],      M[r, c] = Delta[p r + (p-1) - c]        (mtsmatrix.py:249-281, column j = u(Delta m_j)),
// and with r = cap = (p-1, p-1, p-1, p-1) the exponent is I = (p^2 - 1) - c in every variable: always a real exponent of Delta
// (c_i <= 4p - 4 <= p^2 - 1).  A fraction 1 - 1/p of the surfaces that survive the Fedder test have v1[cap] != 0 (height 2): for them
// neither Delta nor M is ever needed.  k_caprow evaluates the N entries Delta[(p^2-1) - c] of that row from the factorised Witt carry
// (the identity of qfs_delta_direct.cuh / DESIGN.md section 3, entry by entry, no tensor cores: 35 taps each),
//     Delta[p s + rho] = [rho = 0] A[s] - sum_{t in T} E[rho + p t] h[s - t]   (mod p),      T = {t in N^3 : |t| <= 4},
// dots them with g and writes height 2 / iterations 1 where the result is nonzero (what k_chain writes for such a surface after
// the fused first step, qfs_chain.cuh); the others stay pending (-1) and take the full pipeline (Delta, M, chain).  This is the
// "lazy" mode of qfs_lib.cu (qfs_heights_lazy): same heights and iteration counts as qfs_heights, M built for ~1/p of the hard
// surfaces only.
//
// One CTA per surface: h and the negated E in shared memory, a thread per column c, rowbase tables for the two index maps.
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct CapRowCfg {
    using S = Shape<P>;
    static constexpr int NT = (P >= 11) ? 256 : 128;
    static constexpr int TE = S::dE + 1;    // rowbase table of E: [J1][J2]
    static constexpr int TH = S::dh + 1;    // rowbase table of h: [u1][u2]
    static constexpr int SMEM = S::Nh_pad + S::NE_pad + 4 * (TE * TE + TH * TH);
};

template <int P>
__global__ void __launch_bounds__(CapRowCfg<P>::NT)
k_caprow(const uint8_t* __restrict__ g_all, const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ A_all,
         const uint8_t* __restrict__ E_all, const uint32_t* __restrict__ unrank_d, const uint32_t* __restrict__ list, int count,
         int max_steps, int8_t* __restrict__ heights, int8_t* __restrict__ iters)
{
    using S = Shape<P>;
    using C = CapRowCfg<P>;
    extern __shared__ __align__(16) uint8_t cr_smem[];
    uint8_t* sh = cr_smem;
    uint8_t* sE = cr_smem + S::Nh_pad;
    int* tE = reinterpret_cast<int*>(cr_smem + S::Nh_pad + S::NE_pad);
    int* tH = tE + C::TE * C::TE;
    __shared__ uint32_t s_red[C::NT / 32];
    const int slot = blockIdx.x, tid = threadIdx.x;
    if (slot >= count) return;
    const uint8_t* gg = g_all + (size_t)slot * S::pitch;
    const uint8_t* gA = A_all + (size_t)slot * S::pitch;
    {
        const uint4* src = reinterpret_cast<const uint4*>(h_all + (size_t)slot * S::Nh_pad);
        for (int i = tid; i < S::Nh_pad / 16; i += C::NT) reinterpret_cast<uint4*>(sh)[i] = src[i];
        const uint8_t* gE = E_all + (size_t)slot * S::NE_pad;
        for (int i = tid; i < S::NE; i += C::NT) {
            const uint32_t e = gE[i];
            sE[i] = (uint8_t)(e ? P - e : 0u);   // -E mod p
        }
        for (int i = tid; i < C::TE * C::TE; i += C::NT) {
            const int a = i / C::TE, b = i - a * C::TE;
            tE[i] = (a + b <= S::dE) ? qrowbase(S::dE, a, b) : -1;
        }
        for (int i = tid; i < C::TH * C::TH; i += C::NT) {
            const int a = i / C::TH, b = i - a * C::TH;
            tH[i] = (a + b <= S::dh) ? qrowbase(S::dh, a, b) : -1;
        }
    }
    __syncthreads();

    uint32_t dot = 0;
    for (int c = tid; c < S::N; c += C::NT) {
        const uint32_t gv = gg[c];
        if (gv == 0) continue;
        const uint32_t m = unrank_d[c];   // column c = the monomial with first exponents (c1, c2, c3)
        const int I1 = P * P - 1 - (int)(m & 255), I2 = P * P - 1 - (int)((m >> 8) & 255), I3 = P * P - 1 - (int)(m >> 16);
        const int s1 = I1 / P, s2 = I2 / P, s3 = I3 / P;
        const int r1 = I1 - P * s1, r2 = I2 - P * s2, r3 = I3 - P * s3;
        uint32_t acc = (r1 | r2 | r3) ? 0u : (uint32_t)gA[qrowbase(S::d, s1, s2) + s3];
#pragma unroll
        for (int t1 = 0; t1 <= 4; ++t1) {
            const int u1 = s1 - t1, J1 = r1 + P * t1;
            if (u1 < 0) break;
#pragma unroll
            for (int t2 = 0; t2 <= 4 - t1; ++t2) {
                const int u2 = s2 - t2, J2 = r2 + P * t2;
                if (u2 < 0) break;
                const int bE = (J1 + J2 <= S::dE) ? tE[J1 * C::TE + J2] : -1;
                const int bH = (u1 + u2 <= S::dh) ? tH[u1 * C::TH + u2] : -1;
                if (bE < 0 || bH < 0) continue;
#pragma unroll
                for (int t3 = 0; t3 <= 4 - t1 - t2; ++t3) {
                    const int u3 = s3 - t3, J3 = r3 + P * t3;
                    if (u3 >= 0 && u1 + u2 + u3 <= S::dh && J1 + J2 + J3 <= S::dE) acc += (uint32_t)sE[bE + J3] * (uint32_t)sh[bH + u3];
                }
            }
        }
        dot += (acc % (uint32_t)P) * gv;   // < N (p-1)^2 < 2^31 in total
    }
    dot = __reduce_add_sync(0xffffffffu, dot);
    if ((tid & 31) == 0) s_red[tid >> 5] = dot;
    __syncthreads();
    if (tid == 0) {
        uint32_t tot = 0;
#pragma unroll
        for (int w = 0; w < C::NT / 32; ++w) tot += s_red[w];
        const bool decided = (tot % (uint32_t)P) != 0;
        if (decided || max_steps <= 1) {   // max_steps = bound - 1 operator applications allowed: after one, an undecided surface is infinity
            const uint32_t sid = list ? list[slot] : (uint32_t)slot;
            heights[sid] = (int8_t)(decided ? 2 : 0);
            iters[sid] = 1;
        }
    }
}
