// qfs_delta.cuh -- stage 2: Delta = Delta_1(f^(p-1)) mod p, dense, one CTA per surface.
//
// Replaces delta1(g) (polyring.py:335-401) and its inner power_mod_small (nttpower.py:447-507):
// instead of raising the N-term g to the p-th power (an NTT of length 2^21..2^27 over 3..6 helper
// primes in the reference) the carry is assembled from the pieces stage 1 produced,
//     Delta = phi(A) - phi(h) * E   (mod p),   phi: x_i -> x_i^p,
// (DESIGN.md section 3 derives it; tests/model_factorized.py restates it in numpy).  Dehomogenised
// (x4 = 1) this is a plain product of 3-variable polynomials: writing an exponent of Delta as
// I = p*s + rho with 0 <= rho_k < p (k = 1..3),
//     Delta[p*s + rho] = [rho = 0] * A[s]  -  sum_{t in T}  E[rho + p*t] * h[s - t],
// where T = {t in N^3 : t1+t2+t3 <= 4} has 35 elements and E, h are zero outside their supports.
// That is C(4p+3,3) * C(4p-5,3) useful integer multiply-adds per surface (0.8 M at p=5, 8 M at p=7,
// 148 M at p=11) with no FFT and no floating point.
//
// Mapping.  The 35 values h[s - t] depend on the point s only, the 35 coefficients E[rho + p*t] on
// the residue class rho only.  Both are packed four taps to a 32-bit word (taps ordered by
// t1+t2+t3, so a class whose rho leaves room for |t| <= k only needs a prefix of 1/3/5/9 words):
//   * sEc  [class][9 words]   -- built once per surface from E,
//   * sHp  [9 words][point]   -- built once per s1-layer from a zero-padded box copy of h,
// and one output is  (A - sum_w dp4a(sEc[class][w], sHp[w][point])) mod p : one broadcast LDS.32 and
// one DP4A per four multiply-adds.  The output is produced slab by slab (slab = all exponents with
// a fixed I1 = p*s1 + rho1), staged in shared memory in the final guard-banded layout and written
// to HBM with 16-byte coalesced stores.  KS consecutive slabs of one layer (they are contiguous in
// HBM) form a phase; its work items are (slab, rho2, pair of points (s2,s3)), dealt to threads with
// the class uniform per warp.  A thread handles two points at once so that every coefficient word
// it loads feeds two DP4As (the kernel is bound by shared-memory load issue otherwise).
//
// Output layout: "lex43g" (qfs_shape.cuh) -- entry (I1,I2,I3,I4) at gbase(I1,I2) + I4, every run
// followed by G guard zeros, ZPAD leading zeros.  The slab staged in shared memory uses the same
// guard-banded layout (guards stay zero: the flush re-zeroes what it copied), so the guards and
// the zero pad are (re)written with every surface and need no separate memset.
#pragma once
#include <cooperative_groups.h>

#include "qfs_shape.cuh"

// 4x4 byte transpose: in[s] holds bytes (x, x+1, x+2, x+3) of source s; out[j] = bytes (in[0].bj, in[1].bj, in[2].bj, in[3].bj)
__device__ __forceinline__ void transpose4x4(const uint32_t (&in)[4], uint32_t (&out)[4])
{
    const uint32_t t0 = __byte_perm(in[0], in[1], 0x5140), t1 = __byte_perm(in[2], in[3], 0x5140);
    const uint32_t t2 = __byte_perm(in[0], in[1], 0x7362), t3 = __byte_perm(in[2], in[3], 0x7362);
    out[0] = __byte_perm(t0, t1, 0x5410);
    out[1] = __byte_perm(t0, t1, 0x7632);
    out[2] = __byte_perm(t2, t3, 0x5410);
    out[3] = __byte_perm(t2, t3, 0x7632);
}

// predicated byte store to shared memory (one ISETP + one @P STS; a select between two generic pointers costs three)
__device__ __forceinline__ void st_shared_u8_le(uint32_t addr, uint32_t v, int a, int b)  // store if a <= b
{
    asm volatile("{\n.reg .pred q;\nsetp.le.s32 q, %2, %3;\n@q st.shared.u8 [%0], %1;\n}\n" ::"r"(addr), "r"(v), "r"(a), "r"(b) : "memory");
}

template <int P>
struct DeltaCfg {
    using S = Shape<P>;
#ifndef QFS_DELTA_NT11
#define QFS_DELTA_NT11 512
#endif
#ifndef QFS_DELTA_NT7
#define QFS_DELTA_NT7 256
#endif
#ifndef QFS_DELTA_NT5
#define QFS_DELTA_NT5 256
#endif
    static constexpr int NT = (P >= 11) ? QFS_DELTA_NT11 : (P >= 7 ? QFS_DELTA_NT7 : (P >= 5 ? QFS_DELTA_NT5 : 64));
    static constexpr bool USE_BOX = (P < 7);   // p >= 7: no box (h is read with bounds checks): at p = 7 its 24 KB buy a fourth slab per phase instead
    static constexpr bool A_IN_SMEM = (P < 11);
    static constexpr int SB = S::dh + 9;       // box side: 4 zeros below, 4 above
    static constexpr int BOX = USE_BOX ? SB * SB * SB : 0;
    static constexpr int NTAP = 35, NWORD = 9;
    static constexpr int NCLS = P * P * P;
    static constexpr int TMAX = (S::d + 1) * (S::d + 2) / 2;  // points (s2,s3) of the layer s1 = 0
    static constexpr int TPAD = (TMAX + 31) & ~31;
    static constexpr int RBH = (S::dh + 1) * (S::dh + 1);     // row bases of basis(dh) (bounds-checked path)
#ifndef QFS_DELTA_KS7
#define QFS_DELTA_KS7 1
#endif
    static constexpr int KS = (P >= 11) ? 1 : (P >= 7 ? QFS_DELTA_KS7 : P);  // slabs (consecutive rho1 of one layer) the phase buffer is sized for (layer 0); p = 7: one slab (48 KB of shared memory, four 256-thread CTAs per SM: 17.1 -> 16.0 ms against four slabs and two 512-thread CTAs)
    static QFS_HD constexpr int slab_bytes(int I1) { return qc2(S::D - I1 + 2) + S::G * (S::D - I1 + 1); }
    static QFS_HD constexpr int slabs_bytes(int n) { int t = 0; for (int k = 0; k < n; ++k) t += slab_bytes(k); return t; }
    static constexpr int SLAB = slabs_bytes(KS) + 32;
    static constexpr int OFF_EC = 0;                                   // uint32 [NCLS][9]
    static constexpr int OFF_HP = OFF_EC + qround16(NCLS * NWORD * 4);  // uint32 [9][TPAD]
    static constexpr int OFF_A = OFF_HP + NWORD * TPAD * 4;
    static constexpr int OFF_TRI = OFF_A + (A_IN_SMEM ? S::pitch : 0);  // uint16 [TMAX]
    static constexpr int OFF_H = OFF_TRI + qround16(2 * TMAX);          // box, or lex h + row-base table
    static constexpr int OFF_SLAB = OFF_H + (USE_BOX ? qround16(BOX) : qround16(S::Nh_pad + 2 * RBH));
    static constexpr int SMEM = OFF_SLAB + qround16(SLAB) + 16;  // + sink bytes
};

// acc[u][rho3] = sum over the first NW tap words of class (rho1,rho2,rho3) for the points 2jq+u, u = 0,1
// (hpq points at word 0 of the even point; the odd point is the next 32-bit word).
template <int P, int NW>
__device__ __forceinline__ void delta_classes(const uint32_t* __restrict__ ec, const uint32_t* __restrict__ hpq,
                                              uint32_t (&acc)[2][P])
{
    using C = DeltaCfg<P>;
    uint2 hp[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) hp[w] = *reinterpret_cast<const uint2*>(hpq + w * C::TPAD);
#pragma unroll
    for (int rho3 = 0; rho3 < P; ++rho3) {
        uint32_t a0 = 0, a1 = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const uint32_t cw = ec[rho3 * C::NWORD + w];
            a0 = __dp4a(cw, hp[w].x, a0);
            a1 = __dp4a(cw, hp[w].y, a1);
        }
        acc[0][rho3] = a0;
        acc[1][rho3] = a1;
    }
}

template <int P>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(DeltaCfg<P>::NT)
k_delta(const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ A_all, const uint8_t* __restrict__ E_all,
        uint8_t* __restrict__ delta_all, int count)
{
    using S = Shape<P>;
    using C = DeltaCfg<P>;
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t* sEc = reinterpret_cast<uint32_t*>(smem + C::OFF_EC);
    uint32_t* sHp = reinterpret_cast<uint32_t*>(smem + C::OFF_HP);
    uint16_t* sTri = reinterpret_cast<uint16_t*>(smem + C::OFF_TRI);
    uint8_t* sH = smem + C::OFF_H;
    uint8_t* sSlab = smem + C::OFF_SLAB;

    // One CTA per surface, four CTAs (one quad of surfaces) per cluster: the quad's Delta is written
    // byte-interleaved (qfs_shape.cuh), each CTA collecting its share of the four slabs over DSMEM.
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned crank = cluster.block_rank();
    const int slot = blockIdx.x;        // grid = 4 * quads; slots >= count are padding (their Delta is zero)
    const bool live = slot < count;
    const int tid = threadIdx.x;
    const uint8_t* gh = h_all + (size_t)slot * S::Nh_pad;
    const uint8_t* gE = E_all + (size_t)slot * S::NE_pad;
    const uint8_t* sA = C::A_IN_SMEM ? smem + C::OFF_A : A_all + (size_t)slot * S::pitch;
    uint8_t* gq = delta_all + (size_t)(slot >> 2) * S::quad_stride;  // the quad's interleaved Delta
    const uint8_t* peer[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) peer[r] = cluster.map_shared_rank(sSlab, r);

    // ---- per-surface setup -------------------------------------------------------------------
    if (C::A_IN_SMEM && live) {
        const uint4* a4 = reinterpret_cast<const uint4*>(A_all + (size_t)slot * S::pitch);
        for (int i = tid; i < S::pitch / 16; i += C::NT) reinterpret_cast<uint4*>(smem + C::OFF_A)[i] = a4[i];
    }
    for (int i = tid; i < qround16(C::SLAB) / 16; i += C::NT) reinterpret_cast<uint4*>(sSlab)[i] = make_uint4(0, 0, 0, 0);
    for (int i = crank * C::NT + tid; i < 4 * S::ZPAD / 16; i += 4 * C::NT) reinterpret_cast<uint4*>(gq)[i] = make_uint4(0, 0, 0, 0);
    for (int e = tid; e < (S::d + 1) * (S::d + 1); e += C::NT) {  // points of a layer by diagonals kk = s2+s3
        const int kk = e / (S::d + 1), s2 = e - kk * (S::d + 1);
        if (s2 <= kk) sTri[kk * (kk + 1) / 2 + s2] = (uint16_t)(kk | (s2 << 8));
    }
    if (C::USE_BOX) {
        for (int i = tid; i < qround16(C::BOX) / 16; i += C::NT) reinterpret_cast<uint4*>(sH)[i] = make_uint4(0, 0, 0, 0);
    } else if (live) {
        for (int i = tid; i < S::Nh_pad / 16; i += C::NT)
            reinterpret_cast<uint4*>(sH)[i] = reinterpret_cast<const uint4*>(gh)[i];
        uint16_t* rbh = reinterpret_cast<uint16_t*>(sH + S::Nh_pad);
        for (int e = tid; e < C::RBH; e += C::NT) {
            const int u1 = e / (S::dh + 1), u2 = e - u1 * (S::dh + 1);
            rbh[e] = (u1 + u2 <= S::dh) ? (uint16_t)qrowbase(S::dh, u1, u2) : (uint16_t)0;
        }
    }
    // class table: sEc[c][w] byte b = -E[rho + p*t_j] mod p, j = 4w+b, taps ordered by |t| then lex; 0 outside deg 4p.
    // One thread per class walks the 35 taps once (the loops are unrolled: tap offsets are immediates).
    for (int c = tid; c < (live ? C::NCLS : 0); c += C::NT) {
        const int rho1 = c / (P * P), rho2 = (c / P) % P, rho3 = c % P;
        uint32_t word = 0;
        int j = 0;
#pragma unroll
        for (int k = 0; k <= 4; ++k)
#pragma unroll
            for (int t1 = 0; t1 <= k; ++t1)
#pragma unroll
                for (int t2 = 0; t2 <= k - t1; ++t2) {
                    const int t3 = k - t1 - t2;
                    const int J1 = rho1 + P * t1, J2 = rho2 + P * t2, J3 = rho3 + P * t3;
                    if (J1 + J2 + J3 <= S::dE) {
                        const uint32_t ev = gE[qrowbase(S::dE, J1, J2) + J3];
                        word |= (ev ? (uint32_t)P - ev : 0u) << (8 * (j & 3));  // -E mod p: sums stay non-negative
                    }
                    if ((j & 3) == 3) { sEc[c * C::NWORD + (j >> 2)] = word; word = 0; }
                    ++j;
                }
        sEc[c * C::NWORD + 8] = word;  // taps 32..34
    }
    __syncthreads();
    if (C::USE_BOX && live) {
        for (int e = tid; e < (S::dh + 1) * (S::dh + 1); e += C::NT) {
            const int u1 = e / (S::dh + 1), u2 = e - u1 * (S::dh + 1);
            const int len = S::dh - u1 - u2;
            if (len < 0) continue;
            const uint8_t* src = gh + qrowbase(S::dh, u1, u2);
            uint8_t* dst = sH + ((u1 + 4) * C::SB + (u2 + 4)) * C::SB + 4;
            for (int u3 = 0; u3 <= len; ++u3) dst[u3] = src[u3];
        }
    }
    __syncthreads();

    // ---- slabs ---------------------------------------------------------------------------------
#pragma unroll 1
    for (int s1 = 0; s1 <= S::d; ++s1) {
        const int I1 = P * s1;  // first slab of the layer
        const int ns = S::d - s1;
        const int T = (ns + 1) * (ns + 2) / 2;
        {
            // packed h neighbourhoods of the layer's points: sHp[w][q] byte b = h[s - t_j], j = 4w+b
            for (int q = tid; q < (live ? T : 0); q += C::NT) {
                const uint32_t e = sTri[q];
                const int kk = e & 255, s2 = e >> 8, s3 = kk - s2;
                uint32_t word = 0;
                int j = 0;
#pragma unroll
                for (int k = 0; k <= 4; ++k)
#pragma unroll
                    for (int t1 = 0; t1 <= k; ++t1)
#pragma unroll
                        for (int t2 = 0; t2 <= k - t1; ++t2) {
                            const int t3 = k - t1 - t2;
                            uint32_t hv;
                            if (C::USE_BOX) {
                                hv = sH[((s1 + 4 - t1) * C::SB + (s2 + 4 - t2)) * C::SB + (s3 + 4 - t3)];
                            } else {
                                const int u1 = s1 - t1, u2 = s2 - t2, u3 = s3 - t3;
                                hv = 0;
                                if (u1 >= 0 && u2 >= 0 && u3 >= 0 && u1 + u2 + u3 <= S::dh)
                                    hv = sH[reinterpret_cast<const uint16_t*>(sH + S::Nh_pad)[u1 * (S::dh + 1) + u2] + u3];
                            }
                            word |= hv << (8 * (j & 3));
                            if ((j & 3) == 3) { sHp[(j >> 2) * C::TPAD + q] = word; word = 0; }
                            ++j;
                        }
                sHp[8 * C::TPAD + q] = word;  // taps 32..34
            }
            __syncthreads();
        }
        int ks_step = C::KS;
        for (int rho1_0 = 0; rho1_0 < P; rho1_0 += ks_step) {
        const int I1_0 = I1 + rho1_0;
        const int goff = S::gbase(I1_0, 0);
        // bytes of the phase's slabs with their guards; in the last layer (I1_0 = D) only the first slab exists.
        // slab_bytes(I) = (n+1)(n+2+2G)/2 with n = D-I, so the bytes of the first k slabs are a cubic in k.
        const int sl_a = S::D - I1_0 + 1, sl_b = S::D - I1_0 + 2 + 2 * S::G;
        const int sl_ab = sl_a * sl_b, sl_apb = sl_a + sl_b;
        auto slabs_before = [&](int k) { return (k * sl_ab - sl_apb * ((k * (k - 1)) >> 1) + ((k - 1) * k * (2 * k - 1)) / 6) >> 1; };
        // As many consecutive slabs as the phase buffer holds (it is sized for the KS largest ones, layer 0): the smaller slabs
        // of the later layers go through in fewer phases, i.e. fewer cluster barriers (p = 11: 441 -> 215 phases).
        int ks = min(C::KS, P - rho1_0);
        if constexpr (C::KS < P) {
            const int kmax = min(P - rho1_0, S::D - I1_0 + 1);  // slabs that exist
            while (ks < kmax && slabs_before(ks + 1) <= C::slabs_bytes(C::KS)) ++ks;
        }
        ks_step = ks;
        const int bytes = slabs_before(max(0, min(ks, S::D - I1_0 + 1)));
        if (bytes == 0) continue;  // uniform over the cluster: no slab, nothing to compute or flush
        uint8_t* slab0 = sSlab + (goff & 15);  // sSlab[0] <-> Delta offset goff & ~15
        const int TP2 = (T + 1) >> 1;
        const float invT = 1.0f / (float)TP2;
        for (int i = tid; i < (live ? ks * P * TP2 : 0); i += C::NT) {
            const int c = (int)(((float)i + 0.5f) * invT);  // = slab-in-phase * P + rho2
            const int jq = i - c * TP2;
            const int k = (c * ((65536 + P - 1) / P)) >> 16, rho2 = c - k * P;
            const int rho1 = rho1_0 + k;
            const int n = S::D - I1_0 - k;
            // bytes of the k slabs in front of this one, in closed form: no per-item loop over the slabs
            uint8_t* slab = slab0 + slabs_before(k);
            const uint32_t* ec = sEc + ((rho1 * P + rho2) * P) * C::NWORD;
            const uint32_t* hpq = sHp + 2 * jq;
            const int rs12 = rho1 + rho2;
            // |rho| = rs12 + rho3 leaves room for |t| <= 4 - ceil(|rho|/p): a prefix of 9/5/3/1 tap words.  The
            // prefix length is taken from rs12 alone (uniform over rho3; the extra words hold zeros).
            uint32_t acc[2][P];
            if (rs12 > 2 * P) delta_classes<P, 1>(ec, hpq, acc);
            else if (rs12 > P) delta_classes<P, 3>(ec, hpq, acc);
            else delta_classes<P, 5>(ec, hpq, acc);
            const int I2base = rho2;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int q = min(2 * jq + u, T - 1);
                const uint32_t e = sTri[q];
                const int kd = e & 255, s2 = e >> 8, s3 = kd - s2;
                const int I2 = P * s2 + I2base;
                const int n2 = n - I2;
                if (rs12 == 0) {  // class rho = 0: all 35 taps, plus the phi(A) term
                    uint32_t a = acc[u][0];
#pragma unroll
                    for (int w = 5; w < 9; ++w) a = __dp4a(ec[w], hpq[w * C::TPAD + u], a);
                    acc[u][0] = a + (uint32_t)sA[qrowbase(S::d, s1, s2) + s3];
                }
                // rho3 <= room are real exponents (I4 >= 0); the odd point of a last pair does not exist
                const int room = (2 * jq + u < T) ? n2 - P * s3 : -1;
                const uint32_t out32 = (uint32_t)__cvta_generic_to_shared(slab) + ((I2 * (2 * n + 3 - I2)) >> 1) + S::G * I2 + (n2 - P * s3);  // position of rho3 = 0
#pragma unroll
                for (int rho3 = 0; rho3 < P; ++rho3) {
                    // acc < 35 p (p-1) + p < 2^32 / p: the quotient by the magic multiply is exact
                    const uint32_t qq = __umulhi(acc[u][rho3], (uint32_t)(0xFFFFFFFFu / P + 1));
                    st_shared_u8_le(out32 - rho3, acc[u][rho3] - qq * (uint32_t)P, rho3, room);
                }
            }
        }
        cluster.sync();  // the four slabs of the quad are complete
        {   // flush: groups of four consecutive Delta offsets x..x+3, interleaved over the quad's four surfaces
            // into one 16-byte store.  The range is widened to whole groups: the bytes it adds in front are
            // guard zeros of the previous phase, the ones behind are rewritten by the next phase.
            const int x_lo = goff & ~3, x_hi = (goff + bytes + 3) & ~3;
            const int ng = (x_hi - x_lo) >> 2;
            const int per = (ng + 3) >> 2;  // each CTA of the cluster stores a contiguous quarter
            const int g_end = min(ng, (int)(crank + 1) * per);
            const int sbase = x_lo - (goff & ~15);
            for (int gi = crank * per + tid; gi < g_end; gi += C::NT) {
                uint32_t in[4], out[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) in[r] = *reinterpret_cast<const uint32_t*>(peer[r] + sbase + 4 * gi);
                transpose4x4(in, out);
                *reinterpret_cast<uint4*>(gq + 4 * (size_t)(x_lo + 4 * gi)) = make_uint4(out[0], out[1], out[2], out[3]);
            }
        }
        cluster.sync();  // everyone has read this CTA's slab: clear it for the next phase
        for (int i = tid; i < (bytes + 15 + 15) >> 4; i += C::NT) reinterpret_cast<uint4*>(sSlab)[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        }  // phases of the layer
    }
}

// lex43g (quad-interleaved) <-> lex.  TO_G = true: dense lex input [surface][L] -> interleaved lex43g output
// (which must be zero-filled beforehand); TO_G = false: the reverse.  Used by the stage taps only.
template <int P, bool TO_G>
__global__ void k_delta_flip(const uint8_t* __restrict__ dense, uint8_t* __restrict__ inter)
{
    using S = Shape<P>;
    const int I1 = blockIdx.x;
    const int slot = blockIdx.y;
    const uint8_t* src = dense + (size_t)slot * S::L;
    uint8_t* dst = const_cast<uint8_t*>(dense) + (size_t)slot * S::L;
    uint8_t* q = inter + (size_t)(slot >> 2) * S::quad_stride + (slot & 3);
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
        const size_t gi = 4 * (size_t)(S::gbase(I1, lo) + I4);
        if (TO_G) q[gi] = src[base + e]; else dst[base + e] = q[gi];
    }
}
