// qfs_delta_mma.cuh -- stage 2 on the tensor cores: Delta = Delta_1(f^(p-1)) mod p as a batch of small int8 GEMMs.
//
// Replaces delta1(g) (polyring.py:335-401) and its inner power_mod_small (nttpower.py:447-507).  Same identity as
// qfs_delta.cuh / DESIGN.md section 3,
//     Delta[p*s + rho] = [rho = 0] * A[s]  -  sum_{t in T}  E[rho + p*t] * h[s - t]     (mod p),   T = {t in N^3 : |t| <= 4},
// read as a matrix product: rows = points s of a layer s1, columns = residue classes rho, inner index = the taps t,
//     acc[s][rho] = sum_j Hp[s][j] * Ec[rho][j],     Hp[s][j] = h[s - t_j],   Ec[rho][j] = -E[rho + p*t_j] mod p,
// with u8 operands and exact s32 accumulators: mma.sync.m16n8k32.u8.u8.s32 (SASS IMMA.16832.U8.U8).  The taps are ordered by
// |t|; every class but rho = 0 only has the 20 taps with |t| <= 3 (|rho + p*t| <= 4p), so K = 32 covers the product and the
// three remaining taps of rho = 0 plus the phi(A) term are added by a scalar pass over that one class.
//
// One CTA works on a QUAD of surfaces (slots 4q..4q+3): the four accumulators a thread holds for the same (point, class) are
// reduced mod p and packed into one 32-bit word, which is exactly one word of the byte-interleaved Delta array the matrix
// builder reads (qfs_shape.cuh) -- no transposition between CTAs, no cluster.  The output goes through shared memory in the
// final guard-banded layout and leaves with bulk copies (cp.async.bulk shared -> global, SASS UBLKCP), double buffered.
//
// Work is cut into PHASES (host-built list, delta_plan): a phase = (layer s1, a group of consecutive rho1, a range of s2); its
// output is, per rho1 of the group, one contiguous piece of the slab I1 = p*s1 + rho1 (the runs I2 in [p*s2a, p*s2b)), so a
// phase ends with at most RG bulk stores.  Pieces are cut on 16-byte groups (4 entries x 4 surfaces); the <= 3 entries a piece
// leaves at its end are guard zeros of its last run and are written (as zeros) by the piece that follows it in memory.
// Inside a phase a warp takes (16 points) x (NCH x 8 classes) items: the A fragments (the points' packed h neighbourhoods, built
// once per phase from a zero-padded window of h in shared memory) stay in registers while it walks the class tiles.
//
// A quad's phases may be split over several CTAs (SPLIT parts of equal work) so that the few hundred surfaces of an F_11 / F_13
// chunk still fill 148 SMs.
#pragma once
#include <algorithm>
#include <vector>

#include "qfs_shape.cuh"

struct DeltaPhase {
    uint8_t s1, rho1a, nrho1, s2a, s2b, pad0;
    uint16_t q0;       // first point of the phase in the lex (s2,s3) order of the layer (unused by the kernel; for checks)
    uint16_t npts;     // points (s2,s3), s2a <= s2 < s2b
    uint16_t pad1;
    uint32_t piece0;   // first entry of the phase in the piece table (nrho1 entries)
    uint32_t nwords;   // words of the staging buffer the phase uses
};
struct DeltaPiece {
    uint32_t ga;       // first entry of the piece in the quad's Delta array (multiple of 4)
    uint32_t po;       // word offset of the piece in the staging buffer (multiple of 4)
    uint32_t nw;       // words (multiple of 4); 0: nothing to store
    int32_t cconst;    // po + gbase(I1, 0) - ga: the constant part of a word's index (see delta_word)
};

#ifndef QFS_DMMA_RG7
#define QFS_DMMA_RG7 1
#endif
#ifndef QFS_DMMA_RG5
#define QFS_DMMA_RG5 5
#endif
#ifndef QFS_DMMA_SBW5
#define QFS_DMMA_SBW5 6144
#endif
#ifndef QFS_DMMA_SBW7
#define QFS_DMMA_SBW7 6144
#endif
#ifndef QFS_DMMA_SBW11
#define QFS_DMMA_SBW11 12288
#endif
#ifndef QFS_DMMA_NT5
#define QFS_DMMA_NT5 256
#endif
#ifndef QFS_DMMA_NT7
#define QFS_DMMA_NT7 256
#endif
#ifndef QFS_DMMA_NT11
#define QFS_DMMA_NT11 512
#endif
#ifndef QFS_DMMA_NCH
#define QFS_DMMA_NCH 4
#endif
#ifndef QFS_DMMA_SPLIT11
#define QFS_DMMA_SPLIT11 16
#endif

template <int P>
struct DeltaMmaCfg {
    using S = Shape<P>;
    static constexpr int RG = (P >= 11) ? 1 : (P == 7 ? QFS_DMMA_RG7 : (P == 5 ? QFS_DMMA_RG5 : P));  // rho1 values per class group
    static constexpr int NCLS = RG * P * P;
    static constexpr int NCLS_PAD = (NCLS + 7) & ~7;
    static constexpr int NT = (P >= 11) ? QFS_DMMA_NT11 : (P == 7 ? QFS_DMMA_NT7 : (P == 5 ? QFS_DMMA_NT5 : 128));
    static constexpr int NCH = QFS_DMMA_NCH;                     // class tiles a warp walks with one set of A fragments
    static constexpr int SPLIT = (P >= 11) ? QFS_DMMA_SPLIT11 : 1;   // CTAs per quad
    static constexpr int MPTS = (P >= 7) ? 128 : 64;            // most points of a phase (multiple of 16)
    static constexpr int SBW = (P >= 11) ? QFS_DMMA_SBW11 : (P == 7 ? QFS_DMMA_SBW7 : (P == 5 ? QFS_DMMA_SBW5 : 2048));  // words per staging buffer
    static constexpr int SBX = S::d + 5;                        // window side: 4 zero cells below (taps reach t2, t3 <= 4), u = 0..d
    static constexpr int PLANE = SBX * SBX;
    static constexpr uint32_t MAGIC = 65536u / P + 1;           // x / p = (x * MAGIC) >> 16 for x * (MAGIC * p - 65536) < 65536
    static constexpr int EC_STRIDE = P * P * P * 32 + 16;       // bytes per surface of the class-major coefficient table
    // shared memory (bytes)
    static constexpr int OFF_EC = 0;                                   // [4][NCLS_PAD][32]
    static constexpr int OFF_HP = OFF_EC + 4 * NCLS_PAD * 32;          // [4][MPTS][32]
    static constexpr int OFF_ROW = OFF_HP + 4 * MPTS * 32;             // int4 [MPTS]
    static constexpr int OFF_COL = OFF_ROW + MPTS * 16;                // int4 [NCLS_PAD]
    static constexpr int OFF_WIN = OFF_COL + NCLS_PAD * 16;            // uint32 [4][PLANE]
    static constexpr int OFF_MISC = OFF_WIN + qround16(4 * PLANE * 4); // DeltaPiece [2][RG], uint32 ec8[4]
    static constexpr int OFF_STAGE = OFF_MISC + qround16(2 * RG * 16 + 16);
    static constexpr int SMEM = OFF_STAGE + 2 * SBW * 4;
    static_assert(MAGIC * P - 65536u < 65536u / (32u * (P - 1) * (P - 1) + 1), "magic quotient not exact");
};

// ---- index algebra shared by the host plan, the kernel and tools/check_delta_plan.cpp -------------------------------------
// Slab I1 (n = D - I1): runs I2 = 0..n, run I2 holds n-I2+1 entries (ordered by I4) and G guard zeros.
template <int P>
QFS_HD constexpr int delta_slab_start(int I1)   // first entry of slab I1; I1 = D+1: one past the last entry (Lg)
{
    using S = Shape<P>;
    return I1 > S::D ? S::Lg : S::gbase(I1, 0);
}
// entries [ga, gb) of the piece (slab I1, runs I2 in [p*s2a, p*s2b))
template <int P>
QFS_HD constexpr void delta_piece_range(int I1, int s2a, int s2b, int& ga, int& gb)
{
    using S = Shape<P>;
    const int n = S::D - I1;
    if (n < 0) { ga = gb = S::Lg; return; }
    ga = (P * s2a <= n) ? S::gbase(I1, P * s2a) : delta_slab_start<P>(I1 + 1);
    gb = (P * s2b <= n) ? S::gbase(I1, P * s2b) : delta_slab_start<P>(I1 + 1);
    if (I1 == 0 && s2a == 0) ga = 0;  // the leading zero pad goes out with the first piece
}
QFS_HD constexpr int delta_F(int x, int n) { return (x * (2 * n + 3 - x)) >> 1; }   // entries of the runs 0..x-1 of a slab, guards aside
// Word of entry (point (s2,s3), class (k,rho2,rho3)) in the staging buffer = R(row) + C(col) - a * m, a = p*s2, m = rho2 + k;
// it exists iff room(row) >= need(col).  n0 = D - p*s1 - rho1a.
template <int P>
QFS_HD constexpr void delta_row(int n0, int s2, int s3, int& R, int& a, int& room)
{
    using S = Shape<P>;
    a = P * s2;
    R = delta_F(a, n0) + (S::G - 1) * a + n0 - P * s3;
    room = n0 - a - P * s3;
}
template <int P>
QFS_HD constexpr void delta_col(int n0, int k, int rho2, int rho3, int cconst, int& C, int& m, int& need)
{
    using S = Shape<P>;
    C = cconst + delta_F(rho2, n0) + (S::G - 1) * rho2 - k - rho3 - k * rho2;
    m = rho2 + k;
    need = k + rho2 + rho3;
}

struct DeltaPlan {
    std::vector<DeltaPhase> phases;
    std::vector<DeltaPiece> pieces;
    std::vector<uint32_t> parts;   // SPLIT + 1 phase indices
};

template <int P>
inline bool delta_plan(DeltaPlan& plan)
{
    using S = Shape<P>;
    using C = DeltaMmaCfg<P>;
    plan.phases.clear();
    plan.pieces.clear();
    for (int s1 = 0; s1 <= S::d; ++s1) {
        const int ns = S::d - s1;
        for (int rho1a = 0; rho1a < P; rho1a += C::RG) {
            const int nrho1 = std::min(C::RG, P - rho1a);
            if (P * s1 + rho1a > S::D) continue;   // no slab in this group
            // Cut s2 = 0..ns into ranges whose pieces fit the staging buffer and whose points fit MPTS, minimising the
            // number of 16-point tiles (a phase pads its points to whole tiles) plus a small charge per phase.
            auto make = [&](int s2a, int s2b, std::vector<DeltaPiece>& pcs, uint32_t& words, int& npts) {
                npts = 0;
                for (int s2 = s2a; s2 < s2b; ++s2) npts += ns - s2 + 1;
                pcs.clear();
                uint32_t po = 0;
                for (int k = 0; k < nrho1; ++k) {
                    const int I1 = P * s1 + rho1a + k;
                    int ga, gb;
                    delta_piece_range<P>(I1, s2a, s2b, ga, gb);
                    DeltaPiece pc{};
                    if (ga < gb) {
                        const int ga_al = ga & ~3, gb_al = (gb == S::Lg) ? ((S::Lg + 3) & ~3) : (gb & ~3);
                        pc.ga = (uint32_t)ga_al;
                        pc.po = po;
                        pc.nw = (uint32_t)(gb_al - ga_al);
                        pc.cconst = (int32_t)po + delta_slab_start<P>(I1) - ga_al;
                        po += pc.nw;
                    }
                    pcs.push_back(pc);
                }
                words = po;
                return npts <= C::MPTS && po <= (uint32_t)C::SBW;
            };
            const int INF = 1 << 30;
            std::vector<int> cost(ns + 2, INF), from(ns + 2, -1);
            cost[0] = 0;
            std::vector<DeltaPiece> pcs;
            uint32_t words;
            int npts;
            for (int b = 1; b <= ns + 1; ++b)
                for (int a = b - 1; a >= 0; --a) {
                    if (!make(a, b, pcs, words, npts)) break;
                    if (cost[a] == INF) continue;
                    const int c = cost[a] + 4 * ((npts + 15) / 16) + 1;
                    if (c < cost[b]) { cost[b] = c; from[b] = a; }
                }
            if (cost[ns + 1] == INF) return false;   // one s2 does not fit: SBW / MPTS too small for this prime
            std::vector<int> cuts;
            for (int b = ns + 1; b > 0; b = from[b]) cuts.push_back(b);
            std::reverse(cuts.begin(), cuts.end());
            int s2a = 0;
            for (int s2b : cuts) {
                make(s2a, s2b, pcs, words, npts);
                int q0 = 0;
                for (int s2 = 0; s2 < s2a; ++s2) q0 += ns - s2 + 1;
                if (words > 0) {
                    DeltaPhase ph{};
                    ph.s1 = (uint8_t)s1; ph.rho1a = (uint8_t)rho1a; ph.nrho1 = (uint8_t)nrho1;
                    ph.s2a = (uint8_t)s2a; ph.s2b = (uint8_t)s2b;
                    ph.q0 = (uint16_t)q0; ph.npts = (uint16_t)npts;
                    ph.piece0 = (uint32_t)plan.pieces.size();
                    ph.nwords = words;
                    plan.phases.push_back(ph);
                    plan.pieces.insert(plan.pieces.end(), pcs.begin(), pcs.end());
                }
                s2a = s2b;
            }
        }
    }
    // parts of equal work (words), on phase boundaries
    plan.parts.assign(C::SPLIT + 1, 0);
    uint64_t total = 0;
    for (const auto& ph : plan.phases) total += ph.nwords;
    uint64_t run = 0;
    int part = 1;
    for (size_t i = 0; i < plan.phases.size() && part < C::SPLIT; ++i) {
        run += plan.phases[i].nwords;
        while (part < C::SPLIT && run * C::SPLIT >= total * part) plan.parts[part++] = (uint32_t)(i + 1);
    }
    for (; part <= C::SPLIT; ++part) plan.parts[part] = (uint32_t)plan.phases.size();
    return true;
}

#if defined(__CUDACC__)

// ---- class-major coefficient table -------------------------------------------------------------------------------------------
// ecm[slot][c][8 words], c = (rho1*p + rho2)*p + rho3: byte b of tap word w = -E[rho + p*t_j] mod p, j = 4w + b (taps ordered by
// |t|, then t1, then t2), stored in the order w = 0,4,1,5,2,6,3,7 (a thread of the MMA reads words tig and tig+4 as one uint2).
// Then 16 bytes: tap word 8 of the class rho = 0 (taps 32..34 and the coefficient 1 of the phi(A) term).
template <int P>
__global__ void __launch_bounds__(128) k_delta_prep(const uint8_t* __restrict__ E_all, uint8_t* __restrict__ ecm_all, int count)
{
    using S = Shape<P>;
    using C = DeltaMmaCfg<P>;
    const int slot = blockIdx.y;
    const int c = blockIdx.x * 128 + threadIdx.x;
    if (slot >= count || c >= P * P * P) return;
    const uint8_t* gE = E_all + (size_t)slot * S::NE_pad;
    uint32_t* out = reinterpret_cast<uint32_t*>(ecm_all + (size_t)slot * C::EC_STRIDE + (size_t)c * 32);
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
                    word |= (ev ? (uint32_t)P - ev : 0u) << (8 * (j & 3));
                }
                if ((j & 3) == 3) {
                    const int w = j >> 2;
                    out[2 * (w & 3) + (w >> 2)] = word;
                    word = 0;
                }
                ++j;
            }
    if (c == 0) {
        uint32_t* tail = reinterpret_cast<uint32_t*>(ecm_all + (size_t)slot * C::EC_STRIDE + (size_t)P * P * P * 32);
        tail[0] = word | (1u << 24);   // taps 32..34, then the phi(A) term
        tail[1] = tail[2] = tail[3] = 0;
    }
}

__device__ __forceinline__ void mma_u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1)
{
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};\n"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
}

// four accumulators (one per surface of the quad) -> their residues mod p, packed into one word (byte s = surface s)
template <int P>
__device__ __forceinline__ uint32_t reduce_pack4(int x0, int x1, int x2, int x3)
{
    constexpr uint32_t M = DeltaMmaCfg<P>::MAGIC;
    const uint32_t t0 = (uint32_t)x0 * M, t1 = (uint32_t)x1 * M, t2 = (uint32_t)x2 * M, t3 = (uint32_t)x3 * M;
    const uint32_t q02 = __byte_perm(t0, t2, 0x7632), q13 = __byte_perm(t1, t3, 0x7632);     // quotients in 16-bit lanes
    const uint32_t x02 = __byte_perm((uint32_t)x0, (uint32_t)x2, 0x5410), x13 = __byte_perm((uint32_t)x1, (uint32_t)x3, 0x5410);
    const uint32_t r02 = x02 - q02 * (uint32_t)P, r13 = x13 - q13 * (uint32_t)P;             // lane-wise: 0 <= r < p, no borrow
    return __byte_perm(r02, r13, 0x6240);
}

// 4 x 4 bytes (tap, surface) -> (surface, tap): in[t] = the four surfaces' h value of tap t; out[s] = surface s, taps 0..3
__device__ __forceinline__ void taps_to_surfaces(const uint32_t (&in)[4], uint32_t (&out)[4])
{
    const uint32_t t0 = __byte_perm(in[0], in[1], 0x5140), t1 = __byte_perm(in[2], in[3], 0x5140);
    const uint32_t t2 = __byte_perm(in[0], in[1], 0x7362), t3 = __byte_perm(in[2], in[3], 0x7362);
    out[0] = __byte_perm(t0, t1, 0x5410);
    out[1] = __byte_perm(t0, t1, 0x7632);
    out[2] = __byte_perm(t2, t3, 0x5410);
    out[3] = __byte_perm(t2, t3, 0x7632);
}

template <int P>
__global__ void __launch_bounds__(DeltaMmaCfg<P>::NT)
k_delta_mma(const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ A_all, const uint8_t* __restrict__ ecm_all,
            const DeltaPhase* __restrict__ phases, const DeltaPiece* __restrict__ pieces, const uint32_t* __restrict__ parts,
            uint8_t* __restrict__ delta_all, int count)
{
    using S = Shape<P>;
    using C = DeltaMmaCfg<P>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* sEc = smem + C::OFF_EC;
    uint8_t* sHp = smem + C::OFF_HP;
    int4* sRow = reinterpret_cast<int4*>(smem + C::OFF_ROW);
    int4* sCol = reinterpret_cast<int4*>(smem + C::OFF_COL);
    uint32_t* sWin = reinterpret_cast<uint32_t*>(smem + C::OFF_WIN);
    DeltaPiece* sPiece = reinterpret_cast<DeltaPiece*>(smem + C::OFF_MISC);
    uint32_t* sEc8 = reinterpret_cast<uint32_t*>(smem + C::OFF_MISC + 2 * C::RG * 16);
    uint32_t* sStage = reinterpret_cast<uint32_t*>(smem + C::OFF_STAGE);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tig = lane & 3;
    constexpr int NW = C::NT / 32;
    const int quad = blockIdx.x / C::SPLIT, part = blockIdx.x % C::SPLIT;
    const int nlive = min(4, count - 4 * quad);   // slots >= count are padding: their Delta is zero
    uint8_t* gq = delta_all + (size_t)quad * S::quad_stride;
    const uint8_t* gh = h_all + (size_t)(4 * quad) * S::Nh_pad;

    int cur_s1 = -100, cur_grp = -1;
    const uint32_t pa = parts[part], pb = parts[part + 1];
#pragma unroll 1
    for (uint32_t ph = pa; ph < pb; ++ph) {
        const DeltaPhase phd = phases[ph];
        const int s1 = phd.s1, rho1a = phd.rho1a, nrho1 = phd.nrho1, s2a = phd.s2a, npts = phd.npts;
        const int ns = S::d - s1;
        const int n0 = S::D - P * s1 - rho1a;
        const int buf = (int)((ph - pa) & 1);
        uint32_t* stage = sStage + buf * C::SBW;
        const int ncls = nrho1 * P * P;

        // ---- (1) tables that no copy in flight reads ----------------------------------------------------------------
        if (s1 != cur_s1) {
            // window of h: planes u1 = s1-3 .. s1 (slot u1 & 3), cell (u2+4, u3+4), the four surfaces' bytes in one word
            const int first = (s1 == cur_s1 + 1) ? s1 : s1 - 3;
            for (int u1 = first; u1 <= s1; ++u1) {
                uint32_t* plane = sWin + (u1 & 3) * C::PLANE;
                for (int e = tid; e < C::PLANE; e += C::NT) {
                    const int b2 = e / C::SBX, b3 = e - b2 * C::SBX;
                    const int u2 = b2 - 4, u3 = b3 - 4;
                    uint32_t w = 0;
                    if (u1 >= 0 && u2 >= 0 && u3 >= 0 && u1 + u2 + u3 <= S::dh) {
                        const uint8_t* src = gh + qrowbase(S::dh, u1, u2) + u3;
#pragma unroll
                        for (int s = 0; s < 4; ++s)
                            if (s < nlive) w |= (uint32_t)src[(size_t)s * S::Nh_pad] << (8 * s);
                    }
                    plane[e] = w;
                }
            }
            cur_s1 = s1;
        }
        if (rho1a != cur_grp) {
            // the group's class rows of the coefficient table: [surface][class][32 bytes], pad classes zero
            const int n16 = ncls * 2;   // 16-byte pieces per surface
            for (int e = tid; e < 4 * C::NCLS_PAD * 2; e += C::NT) {
                const int s = e / (C::NCLS_PAD * 2), i = e - s * (C::NCLS_PAD * 2);
                uint4 v = make_uint4(0, 0, 0, 0);
                if (s < nlive && i < n16)
                    v = reinterpret_cast<const uint4*>(ecm_all + (size_t)(4 * quad + s) * C::EC_STRIDE + (size_t)rho1a * P * P * 32)[i];
                reinterpret_cast<uint4*>(sEc)[e] = v;
            }
            if (tid < 4)
                sEc8[tid] = (tid < nlive) ? *reinterpret_cast<const uint32_t*>(ecm_all + (size_t)(4 * quad + tid) * C::EC_STRIDE + (size_t)P * P * P * 32) : 0u;
            cur_grp = rho1a;
        }
        if (tid < nrho1) sPiece[buf * C::RG + tid] = pieces[phd.piece0 + tid];
        for (int c = tid; c < C::NCLS_PAD; c += C::NT) {
            int4 ci = make_int4(0, 0, 0x7fff, 0);
            if (c < ncls) {
                const int k = c / (P * P), r = c - k * (P * P), rho2 = r / P, rho3 = r - rho2 * P;
                int Cc, m, need;
                delta_col<P>(n0, k, rho2, rho3, pieces[phd.piece0 + k].cconst, Cc, m, need);
                ci = make_int4(Cc, m, need, 0);
            }
            sCol[c] = ci;
        }
        __syncthreads();   // (S1) also: thread 0 has waited for the copies that read this staging buffer

        // ---- (2) clear the staging buffer; packed h neighbourhoods and row constants of the phase's points --------------
        for (int i = tid; i < (int)(phd.nwords >> 2); i += C::NT) reinterpret_cast<uint4*>(stage)[i] = make_uint4(0, 0, 0, 0);
        const int npad = (npts + 15) & ~15;
        for (int ql = tid; ql < npad; ql += C::NT) {
            int s2 = s2a, s3 = ql;
            while (s3 > ns - s2 && s2 < phd.s2b - 1) { s3 -= ns - s2 + 1; ++s2; }
            const bool real = ql < npts;
            int R, a, room;
            delta_row<P>(n0, s2, s3, R, a, room);
            sRow[ql] = make_int4(R, -a, real ? room : -1, 0);
            uint32_t hw[4][8];   // [surface][tap word]
            if (real) {
                const int cell = (s2 + 4) * C::SBX + (s3 + 4);
                int j = 0;
                uint32_t in[4];
#pragma unroll
                for (int k = 0; k <= 4; ++k)
#pragma unroll
                    for (int t1 = 0; t1 <= k; ++t1)
#pragma unroll
                        for (int t2 = 0; t2 <= k - t1; ++t2) {
                            const int t3 = k - t1 - t2;
                            if (j < 32) {
                                in[j & 3] = sWin[((s1 - t1) & 3) * C::PLANE + cell - t2 * C::SBX - t3];
                                if ((j & 3) == 3) {
                                    uint32_t o[4];
                                    taps_to_surfaces(in, o);
#pragma unroll
                                    for (int s = 0; s < 4; ++s) hw[s][j >> 2] = o[s];
                                }
                            }
                            ++j;
                        }
            } else {
#pragma unroll
                for (int s = 0; s < 4; ++s)
#pragma unroll
                    for (int w = 0; w < 8; ++w) hw[s][w] = 0;
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                uint4* dst = reinterpret_cast<uint4*>(sHp + ((size_t)s * C::MPTS + ql) * 32);
                dst[0] = make_uint4(hw[s][0], hw[s][4], hw[s][1], hw[s][5]);
                dst[1] = make_uint4(hw[s][2], hw[s][6], hw[s][3], hw[s][7]);
            }
        }
        __syncthreads();   // (S2)

        // ---- (3) items: (16 points) x (NCH class tiles) ------------------------------------------------------------------
        const int nmt = npad >> 4;
        const int ntile = (ncls + 7) >> 3;
        const int nch = (ntile + C::NCH - 1) / C::NCH;
#pragma unroll 1
        for (int it = warp; it < nmt * nch; it += NW) {
            const int ch = it / nmt, mt = it - ch * nmt;
            const int r0 = mt * 16 + g;
            uint32_t a[4][4];
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint2 x = *reinterpret_cast<const uint2*>(sHp + ((size_t)s * C::MPTS + r0) * 32 + tig * 8);
                const uint2 y = *reinterpret_cast<const uint2*>(sHp + ((size_t)s * C::MPTS + r0 + 8) * 32 + tig * 8);
                a[s][0] = x.x; a[s][1] = y.x; a[s][2] = x.y; a[s][3] = y.y;
            }
            const int4 row0 = sRow[r0], row1 = sRow[r0 + 8];   // (R, -a, room)
            const int nt_end = min(ntile, (ch + 1) * C::NCH);
#pragma unroll 2
            for (int nt = ch * C::NCH; nt < nt_end; ++nt) {
                int acc[4][4];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const uint2 b = *reinterpret_cast<const uint2*>(sEc + ((size_t)s * C::NCLS_PAD + nt * 8 + g) * 32 + tig * 8);
                    mma_u8(acc[s], a[s][0], a[s][1], a[s][2], a[s][3], b.x, b.y);
                }
                const int4 c0 = sCol[nt * 8 + 2 * tig], c1 = sCol[nt * 8 + 2 * tig + 1];   // (C, m, need)
                // accumulator i of the fragment: i = 0: (row g, col 2tig), 1: (g, 2tig+1), 2: (g+8, 2tig), 3: (g+8, 2tig+1)
                {
                    const uint32_t w = reduce_pack4<P>(acc[0][0], acc[1][0], acc[2][0], acc[3][0]);
                    if (row0.z >= c0.z) stage[row0.x + c0.x + row0.y * c0.y] = w;
                }
                {
                    const uint32_t w = reduce_pack4<P>(acc[0][1], acc[1][1], acc[2][1], acc[3][1]);
                    if (row0.z >= c1.z) stage[row0.x + c1.x + row0.y * c1.y] = w;
                }
                {
                    const uint32_t w = reduce_pack4<P>(acc[0][2], acc[1][2], acc[2][2], acc[3][2]);
                    if (row1.z >= c0.z) stage[row1.x + c0.x + row1.y * c0.y] = w;
                }
                {
                    const uint32_t w = reduce_pack4<P>(acc[0][3], acc[1][3], acc[2][3], acc[3][3]);
                    if (row1.z >= c1.z) stage[row1.x + c1.x + row1.y * c1.y] = w;
                }
            }
        }

        // ---- (4) class rho = 0: taps 32..34 and the phi(A) term ----------------------------------------------------------
        if (rho1a == 0) {
            __syncthreads();
            const int4 c0 = sCol[0];
            for (int ql = tid; ql < npts; ql += C::NT) {
                int s2 = s2a, s3 = ql;
                while (s3 > ns - s2) { s3 -= ns - s2 + 1; ++s2; }
                const int4 row = sRow[ql];
                const int cell = (s2 + 4) * C::SBX + (s3 + 4);
                // taps 32, 33, 34 = (3,0,1), (3,1,0), (4,0,0)
                const uint32_t h32 = sWin[((s1 - 3) & 3) * C::PLANE + cell - 1];
                const uint32_t h33 = sWin[((s1 - 3) & 3) * C::PLANE + cell - C::SBX];
                uint32_t h34 = 0, av = 0;
                const int u1 = s1 - 4;
                const bool in34 = u1 >= 0 && u1 + s2 + s3 <= S::dh;
                const int r34 = in34 ? qrowbase(S::dh, u1, s2) + s3 : 0;
                const int rA = qrowbase(S::d, s1, s2) + s3;
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    if (s < nlive) {
                        if (in34) h34 |= (uint32_t)gh[(size_t)s * S::Nh_pad + r34] << (8 * s);
                        av |= (uint32_t)A_all[(size_t)(4 * quad + s) * S::pitch + rA] << (8 * s);
                    }
                uint32_t* wp = stage + (row.x + c0.x);
                const uint32_t old = *wp;
                uint32_t nw = 0;
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const uint32_t e8 = sEc8[s];
                    const uint32_t x = ((old >> (8 * s)) & 255u) + (e8 & 255u) * ((h32 >> (8 * s)) & 255u) +
                                       ((e8 >> 8) & 255u) * ((h33 >> (8 * s)) & 255u) + ((e8 >> 16) & 255u) * ((h34 >> (8 * s)) & 255u) +
                                       (e8 >> 24) * ((av >> (8 * s)) & 255u);
                    nw |= (x % (uint32_t)P) << (8 * s);
                }
                *wp = nw;
            }
        }

        // ---- (5) the phase's pieces leave with bulk copies ----------------------------------------------------------------
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();   // (S3)
        if (tid == 0) {
            for (int k = 0; k < nrho1; ++k) {
                const DeltaPiece pc = sPiece[buf * C::RG + k];
                if (pc.nw) {
                    const uint32_t src = (uint32_t)__cvta_generic_to_shared(stage + pc.po);
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(gq + 4 * (size_t)pc.ga), "r"(src),
                                 "r"(pc.nw * 4u)
                                 : "memory");
                }
            }
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");   // the other staging buffer is free again
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

#endif  // __CUDACC__
