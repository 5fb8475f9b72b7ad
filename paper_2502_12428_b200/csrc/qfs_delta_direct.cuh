// qfs_delta_direct.cuh -- stage 2 for primes whose slab does not fit shared memory (p = 13), and the in-repo
// cross-check of k_delta for the others.
//
// Same identity and the same packed-tap arithmetic as qfs_delta.cuh,
//     Delta[p*s + rho] = [rho = 0] * A[s]  -  sum_{t in T} E[rho + p*t] * h[s - t]     (mod p),
// but without the slab staging: a thread owns one point s (its 35 values h[s - t] packed in 9 registers),
// walks all residue classes rho -- uniform over the warp, so the class words are broadcast shared-memory
// loads -- and stores every entry straight into the quad-interleaved lex43g array (byte stores).  The
// guards and the zero pad of the array are NOT written here: the caller clears the array first.
// k_delta's slab of the first layer needs 218 KB at p = 13 (one layer is C(626,2) entries); this kernel
// needs the class table only (79 KB).  At p = 13 a surface is 434 MB of operator matrix, so the byte
// stores of the 41 MB Delta are not what bounds the pipeline.
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct DeltaDirectCfg {
    using S = Shape<P>;
    static constexpr int NT = 256;
    static constexpr int NWORD = 9;
    static constexpr int NCLS = P * P * P;
    static constexpr int SMEM = NCLS * NWORD * 4;
    static constexpr int NBLK = (S::N + NT - 1) / NT;  // CTAs per surface: one thread per point s of basis(d) (3 free exponents)
};

template <int P>
__global__ void __launch_bounds__(DeltaDirectCfg<P>::NT)
k_delta_direct(const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ A_all, const uint8_t* __restrict__ E_all,
               const uint32_t* __restrict__ unrank_d, uint8_t* __restrict__ delta_all, int count)
{
    using S = Shape<P>;
    using C = DeltaDirectCfg<P>;
    extern __shared__ __align__(16) uint32_t sEc[];  // [class][9]: byte b of word w = -E[rho + p*t_j] mod p, j = 4w+b
    const int slot = blockIdx.y;
    if (slot >= count) return;
    const int tid = threadIdx.x;
    const uint8_t* gh = h_all + (size_t)slot * S::Nh_pad;
    const uint8_t* gE = E_all + (size_t)slot * S::NE_pad;
    const uint8_t* gA = A_all + (size_t)slot * S::pitch;
    uint8_t* gq = delta_all + (size_t)(slot >> 2) * S::quad_stride + (slot & 3);

    for (int e = tid; e < C::NCLS * C::NWORD; e += C::NT) {
        const int c = e / C::NWORD, w = e - c * C::NWORD;
        const int rho1 = c / (P * P), rho2 = (c / P) % P, rho3 = c % P;
        uint32_t word = 0;
        int j = 0;
        for (int k = 0; k <= 4; ++k)
            for (int t1 = 0; t1 <= k; ++t1)
                for (int t2 = 0; t2 <= k - t1; ++t2) {
                    const int t3 = k - t1 - t2;
                    if ((j >> 2) == w) {
                        const int J1 = rho1 + P * t1, J2 = rho2 + P * t2, J3 = rho3 + P * t3;
                        if (J1 + J2 + J3 <= S::dE) {
                            const uint32_t ev = gE[qrowbase(S::dE, J1, J2) + J3];
                            word |= (ev ? (uint32_t)P - ev : 0u) << (8 * (j & 3));
                        }
                    }
                    ++j;
                }
        sEc[e] = word;
    }
    __syncthreads();

    const int pt = blockIdx.x * C::NT + tid;
    if (pt >= S::N) return;
    const uint32_t m = unrank_d[pt];  // point s = (s1,s2,s3), |s| <= d: the monomial of basis(d,4) with these first exponents
    const int s1 = m & 255, s2 = (m >> 8) & 255, s3 = m >> 16;
    uint32_t hp[C::NWORD];
    {
        int j = 0;
        uint32_t word = 0;
        for (int k = 0; k <= 4; ++k)
            for (int t1 = 0; t1 <= k; ++t1)
                for (int t2 = 0; t2 <= k - t1; ++t2) {
                    const int t3 = k - t1 - t2;
                    const int u1 = s1 - t1, u2 = s2 - t2, u3 = s3 - t3;
                    uint32_t hv = 0;
                    if (u1 >= 0 && u2 >= 0 && u3 >= 0 && u1 + u2 + u3 <= S::dh) hv = gh[qrowbase(S::dh, u1, u2) + u3];
                    word |= hv << (8 * (j & 3));
                    if ((j & 3) == 3) { hp[j >> 2] = word; word = 0; }
                    ++j;
                }
        hp[8] = word;  // taps 32..34
    }
    const uint32_t a = gA[pt];
    const int budget = S::D - P * (s1 + s2 + s3);  // |rho| <= budget are real exponents of Delta
    for (int rho1 = 0; rho1 < P; ++rho1)
        for (int rho2 = 0; rho2 < P; ++rho2) {
            if (rho1 + rho2 > budget) continue;
            const int I1 = P * s1 + rho1, I2 = P * s2 + rho2;
            const size_t base = 4 * (size_t)(S::gbase(I1, I2) + (S::D - I1 - I2 - P * s3));  // entry with rho3 = 0 (I4 largest)
            const uint32_t* ec = sEc + ((rho1 * P + rho2) * P) * C::NWORD;
            for (int rho3 = 0; rho3 < P && rho1 + rho2 + rho3 <= budget; ++rho3) {
                uint32_t acc = (rho1 | rho2 | rho3) ? 0u : a;
#pragma unroll
                for (int w = 0; w < C::NWORD; ++w) acc = __dp4a(ec[rho3 * C::NWORD + w], hp[w], acc);
                gq[base - 4 * (size_t)rho3] = (uint8_t)(acc % (uint32_t)P);
            }
        }
}
