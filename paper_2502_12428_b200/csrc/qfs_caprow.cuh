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
// One CTA per surface.  The row only meets the points s with s_i in [p-4, p-1] (I_i = p^2-1-c_i, 0 <= c_i <= 4p-4): at most 64.
// So the CTA first builds, in shared memory, the packed operands of qfs_delta_direct.cuh for exactly what the row needs -- per
// residue class rho the 35 negated coefficients -E[rho + p t] (a pass over E: every entry belongs to one (class, tap)), per point s the 35 neighbours
// h[s - t], both as 9 words of four bytes in the tap order of basis(4) -- and then a thread per column c turns its entry into
// nine LDS pairs + DP4A, one exact reduction mod p and one multiply-add with g[c].
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct CapRowCfg {
    using S = Shape<P>;
    static constexpr int NT = (P >= 11) ? 256 : 128;
    static constexpr int NWORD = 9;                   // 35 taps, four per word
    static constexpr int NCLS = P * P * P;
    static constexpr int S0 = (P > 4) ? P - 4 : 0;    // smallest s_i of the row
    static constexpr int NPT = 64;                    // points (s1, s2, s3), s_i = S0 .. S0 + 3
    static constexpr int SMEM = 4 * NWORD * (NCLS + NPT);
};

template <int P>
__global__ void __launch_bounds__(CapRowCfg<P>::NT)
k_caprow(const uint8_t* __restrict__ g_all, const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ A_all,
         const uint8_t* __restrict__ E_all, const uint32_t* __restrict__ unrank4, const uint32_t* __restrict__ unrank_E, const uint32_t* __restrict__ unrank_d,
         const uint32_t* __restrict__ list, int count, int max_steps, int8_t* __restrict__ heights, int8_t* __restrict__ iters,
         uint32_t* __restrict__ slotmap)
{
    using S = Shape<P>;
    using C = CapRowCfg<P>;
    extern __shared__ __align__(16) uint32_t cr_smem[];
    uint32_t* sEc = cr_smem;                      // [class][9]: byte j = -E[rho + p t_j] mod p
    uint32_t* sHp = cr_smem + C::NWORD * C::NCLS; // [point][9]: byte j = h[s - t_j]
    __shared__ uint32_t s_red[C::NT / 32];
    __shared__ uint8_t s_rb4[25];                              // rank of the tap t in basis(4): rowbase(4, t1, t2) (+ t3)
    __shared__ uint16_t s_rbh[(S::dh + 1) * (S::dh + 1)];      // rowbase(dh, u1, u2)
    const int slot = blockIdx.x, tid = threadIdx.x;
    if (slot >= count) return;
    const uint8_t* gg = g_all + (size_t)slot * S::pitch;
    const uint8_t* gA = A_all + (size_t)slot * S::pitch;
    const uint8_t* gh = h_all + (size_t)slot * S::Nh_pad;
    const uint8_t* gE = E_all + (size_t)slot * S::NE_pad;
    {
        // class table: every entry E[J] of the surface goes to exactly one (class, tap) = (J mod p, J div p); the rest stays zero
        for (int i = tid; i < C::NWORD * (C::NCLS + C::NPT); i += C::NT) cr_smem[i] = 0u;
        if (tid < 25) s_rb4[tid] = (uint8_t)((tid / 5 + tid % 5 <= 4) ? qrowbase(4, tid / 5, tid % 5) : 0);
        for (int i = tid; i < (S::dh + 1) * (S::dh + 1); i += C::NT) {
            const int a = i / (S::dh + 1), b = i - a * (S::dh + 1);
            s_rbh[i] = (uint16_t)((a + b <= S::dh) ? qrowbase(S::dh, a, b) : 0);
        }
        __syncthreads();
        uint8_t* bE = reinterpret_cast<uint8_t*>(sEc);
        for (int e = tid; e < S::NE; e += C::NT) {
            const uint32_t ev = gE[e];
            if (ev == 0) continue;
            const uint32_t m = unrank_E[e];
            const int J1 = m & 255, J2 = (m >> 8) & 255, J3 = m >> 16;
            const int t1 = J1 / P, t2 = J2 / P, t3 = J3 / P;
            const int cls = ((J1 - P * t1) * P + (J2 - P * t2)) * P + (J3 - P * t3);
            bE[cls * (4 * C::NWORD) + s_rb4[t1 * 5 + t2] + t3] = (uint8_t)(P - ev);   // |t| <= 4 because |J| <= 4p
        }
        // point table: h[s - t_j] for the 64 points the row can meet
        uint8_t* bH = reinterpret_cast<uint8_t*>(sHp);
        for (int e = tid; e < 35 * C::NPT; e += C::NT) {
            const int pt = e / 35, j = e - pt * 35;
            const uint32_t t = unrank4[j];
            const int u1 = C::S0 + (pt >> 4) - (int)(t & 255), u2 = C::S0 + ((pt >> 2) & 3) - (int)((t >> 8) & 255),
                      u3 = C::S0 + (pt & 3) - (int)(t >> 16);
            if (u1 >= 0 && u2 >= 0 && u3 >= 0 && u1 + u2 + u3 <= S::dh) bH[pt * (4 * C::NWORD) + j] = gh[s_rbh[u1 * (S::dh + 1) + u2] + u3];
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
        const int cls = ((I1 - P * s1) * P + (I2 - P * s2)) * P + (I3 - P * s3);
        const uint32_t* ec = sEc + cls * C::NWORD;
        const uint32_t* hp = sHp + (((s1 - C::S0) * 4 + (s2 - C::S0)) * 4 + (s3 - C::S0)) * C::NWORD;
        uint32_t acc = cls ? 0u : (uint32_t)gA[qrowbase(S::d, s1, s2) + s3];
#pragma unroll
        for (int w = 0; w < C::NWORD; ++w) acc = __dp4a(ec[w], hp[w], acc);
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
        const uint32_t sid = list ? list[slot] : (uint32_t)slot;
        if (decided || max_steps <= 1) {   // max_steps = bound - 1 operator applications allowed: after one, an undecided surface is infinity
            heights[sid] = (int8_t)(decided ? 2 : 0);
            iters[sid] = 1;
        } else if (slotmap) {
            slotmap[sid] = (uint32_t)slot;   // where the pending surface's g, h, A, E sit (k_gather_rows)
        }
    }
}

// The surfaces the cap row left pending keep the g, h, A, E that k_power_full computed for the cap-row pass: slot k of the
// compacted list takes the rows of the slot the surface had there (slotmap).  Rows are gathered into a scratch area (the rows
// move towards lower slots, so an in-place copy would race) and copied back by the caller.
struct GatherRows {
    const uint8_t* src[4];
    uint8_t* dst[4];
    uint32_t row16[4];   // row sizes in 16-byte units
};

__global__ void __launch_bounds__(128) k_gather_rows(GatherRows gr, const uint32_t* __restrict__ list, const uint32_t* __restrict__ slotmap, int count)
{
    const int k = blockIdx.x;
    if (k >= count) return;
    const uint32_t j = slotmap[list[k]];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint4* s = reinterpret_cast<const uint4*>(gr.src[a]) + (size_t)j * gr.row16[a];
        uint4* d = reinterpret_cast<uint4*>(gr.dst[a]) + (size_t)k * gr.row16[a];
        for (uint32_t i = threadIdx.x; i < gr.row16[a]; i += 128) d[i] = s[i];
    }
}
