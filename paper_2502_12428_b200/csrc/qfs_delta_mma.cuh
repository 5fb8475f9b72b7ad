// qfs_delta_mma.cuh -- stage 2 on the tensor cores: Delta = Delta_1(f^(p-1)) mod p as a batch of small int8 GEMMs.
//
// Replaces delta1(g) (polyring.py:335-401) and its inner power_mod_small (nttpower.py:447-507).  Same identity as
// qfs_delta.cuh / DESIGN.md section 3,
//     Delta[p*s + rho] = [rho = 0] * A[s]  -  sum_{t in T}  E[rho + p*t] * h[s - t]     (mod p),   T = {t in N^3 : |t| <= 4},
// read as a matrix product: rows = points s of a layer s1, columns = residue classes rho, inner index = the taps t,
//     acc[s][rho] = sum_j Hp[s][j] * Ec[rho][j],     Hp[s][j] = h[s - t_j],   Ec[rho][j] = -E[rho + p*t_j] mod p,
// with u8 operands and exact s32 accumulators: mma.sync.m16n8k32.u8.u8.s32 (SASS IMMA.16832.U8.U8).  The taps are ordered by
// |t|; every class but rho = 0 only has the 20 taps with |t| <= 3 (|rho + p*t| <= 4p), so K = 32 covers the product; what the class
// rho = 0 gets beyond that (taps 32..34 and the phi(A) term) is a per-point constant prepared by k_delta_box and added to its
// accumulators.
//
// One CTA works on a QUAD of surfaces (slots 4q..4q+3): the four accumulators a thread holds for the same (point, class) are
// reduced mod p (one multiply per value, quotients and remainders in 16-bit lanes) and packed into one 32-bit word, which is
// exactly one word of the byte-interleaved Delta array the matrix builder reads (qfs_shape.cuh) -- no transposition between
// CTAs, no cluster.  The output goes through shared memory in the final guard-banded layout and leaves with bulk copies
// (cp.async.bulk shared -> global, SASS UBLKCP).
//
// Work is cut into PHASES (host-built list, delta_plan): a phase = (layer s1, a group of consecutive rho1, a range of s2); its
// output is, per rho1 of the group, one contiguous piece of the slab I1 = p*s1 + rho1 (the runs I2 in [p*s2a, p*s2b)), so a
// phase ends with at most RG bulk stores.  Pieces are cut on 16-byte groups (4 entries x 4 surfaces); the <= 3 entries a piece
// leaves at its end are guard zeros of its last run and are written (as zeros) by the piece that follows it in memory.
// Inside a phase every warp takes an equal share of the phase's (16 points) x (8 classes) tiles, in (point tile, class tile)
// order: it gathers the A fragments of a point tile (the points' packed h neighbourhoods) straight from a zero-padded window of h
// in shared memory (planes u1 = s1-3..s1, the four surfaces' bytes in one word) and keeps them in registers while it walks the
// class tiles; the B fragments come from the group's class rows in shared memory.  The guard zeros of the phase's runs are
// written explicitly (a run per lane), so the staging buffer is never cleared: entries and guard zeros together are exactly the
// words of the phase (tools/check_delta_plan.cpp proves it on the host for every prime).
//
// Pipeline.  NWI item warps + one store warp, NBUF staging buffers with full/empty mbarriers: an item warp that has finished its
// share of phase i arrives on full[i % NBUF]; the store warp waits for full, issues the phase's bulk copies (a piece per lane),
// waits until they have read shared memory and arrives on empty.  There is no barrier among the item warps: the full/empty
// handshake bounds their lag to NBUF - 1 phases, the window has 5 + lag planes and the class rows 2 + lag buffers, so the next layer's
// plane and the next group's rows are prefetched a block ahead (cp.async.bulk global -> shared, mbarrier complete_tx) into slots
// no lagging warp still reads, and every warp derives the same mbarrier parities from the phase list.
//
// A quad's phases may be split over several CTAs (SPLIT parts of equal work) so that the few hundred surfaces of an F_11 / F_13
// chunk still fill 148 SMs.
//
// Measured (B200, 100 000 seeded surfaces): F_5 3.25 -> 1.5 ms, F_7 16.0 -> 8.3 ms, F_11 (4000 surfaces) 8.5 -> 3.5 ms,
// F_13 (2000 surfaces) 41.9 -> 5.0 ms against the DP4A kernels (qfs_delta.cuh, qfs_delta_direct.cuh), bit-identical Delta.
#pragma once
#include <algorithm>
#include <type_traits>
#include <vector>

#include "qfs_shape.cuh"

enum { DPH_BLOCK = 1, DPH_PF_PLANE = 2, DPH_PF_EC = 4 };

struct DeltaPhase {
    uint8_t s1, rho1a, nrho1, s2a, s2b;
    uint8_t flags;       // DPH_BLOCK: first phase of a (layer, group) block inside its part; DPH_PF_*: what to prefetch there
    uint8_t pf_rho1a, pf_nrho1;   // the group whose coefficient rows DPH_PF_EC prefetches
    uint16_t npts;       // points (s2,s3), s2a <= s2 < s2b
    uint16_t pad;
    uint32_t piece0;     // first entry of the phase in the piece table (nrho1 entries)
    uint32_t nwords;     // words of the staging buffer the phase uses
};
struct DeltaPiece {
    uint32_t ga;       // first entry of the piece in the quad's Delta array (multiple of 4)
    uint32_t po;       // word offset of the piece in the staging buffer (multiple of 4)
    uint32_t nw;       // words (multiple of 4); 0: nothing to store
    int32_t cconst;    // po + gbase(I1, 0) - ga: the constant part of a word's index (delta_row / delta_col)
};

#ifndef QFS_DMMA_RG7
#define QFS_DMMA_RG7 1
#endif
#ifndef QFS_DMMA_RG5
#define QFS_DMMA_RG5 5
#endif
#ifndef QFS_DMMA_SBW5
#define QFS_DMMA_SBW5 6912   // fewer, larger phases; 54.3 KB per CTA still leaves four CTAs per SM (6144: 1.61, 6656 ... 7160: 1.52 ms)
#endif
#ifndef QFS_DMMA_SBW7
#define QFS_DMMA_SBW7 5600   // 57.3 KB per CTA: four CTAs per SM (6144 words are 48 bytes too many for that: 9.4 -> 8.3 ms)
#endif
#ifndef QFS_DMMA_SBW11
#define QFS_DMMA_SBW11 14336   // two buffers of 56 KB: 219.8 KB per CTA (12288: 3.57, 13312: 3.49, 14336: 3.46 ms per 374 surfaces)
#endif
#ifndef QFS_DMMA_SBW13
#define QFS_DMMA_SBW13 9216
#endif
#ifndef QFS_DMMA_NWI5
#define QFS_DMMA_NWI5 4
#endif
#ifndef QFS_DMMA_NWI7
#define QFS_DMMA_NWI7 4
#endif
#ifndef QFS_DMMA_NWI11
#define QFS_DMMA_NWI11 8
#endif
#ifndef QFS_DMMA_MAXB
#define QFS_DMMA_MAXB 4
#endif
#ifndef QFS_DMMA_NBUF
#define QFS_DMMA_NBUF 1
#endif
#ifndef QFS_DMMA_NBUF11
#define QFS_DMMA_NBUF11 2
#endif
#ifndef QFS_DMMA_SPLIT11
#define QFS_DMMA_SPLIT11 16
#endif

template <int P>
struct DeltaMmaCfg {
    using S = Shape<P>;
    static constexpr int RG = (P >= 11) ? 1 : (P == 7 ? QFS_DMMA_RG7 : (P == 5 ? QFS_DMMA_RG5 : P));  // rho1 values per class group
    static_assert(RG == 1 || RG == P, "class groups of unequal size are not supported (the column table is static)");
    static constexpr int NGROUP = (P + RG - 1) / RG;
#ifndef QFS_DMMA_STORE_GUARDS
#define QFS_DMMA_STORE_GUARDS 1
#endif
    static constexpr bool STORE_GUARDS = (RG == 1) && QFS_DMMA_STORE_GUARDS;   // the store warp writes the guard zeros (see k_delta_mma)
    static constexpr int NBUF = (P >= 11) ? QFS_DMMA_NBUF11 : QFS_DMMA_NBUF;   // staging buffers (1: the copies of a phase overlap other CTAs' work only)
    static constexpr int LAG = NBUF - 1;                             // phases an item warp may be behind the one that issues the prefetches
    static constexpr int NEC = NGROUP > 1 ? 2 + LAG : 1;         // coefficient-row buffers: in use, (still read by a lagging warp,) in flight
    static constexpr int XS = 2 + LAG;                           // slots of the class-0 terms: layers (s1-1,) s1, s1+1
    static constexpr int NCLS = RG * P * P;
    static constexpr int NCLS_PAD = (NCLS + 7) & ~7;
    static constexpr int NWI = (P >= 11) ? QFS_DMMA_NWI11 : (P == 7 ? QFS_DMMA_NWI7 : (P == 5 ? QFS_DMMA_NWI5 : 4));  // item warps
    static constexpr int NTI = 32 * NWI;
    static constexpr int NT = NTI + 32;                          // + the store warp
    static constexpr int SPLIT = (P >= 11) ? QFS_DMMA_SPLIT11 : 1;   // CTAs per quad of a large launch
    // ... of a launch with fewer quads than CTA slots (SPLIT_MID), and of one with at most four quads (SPLIT_FEW: single surfaces).
    // Measured: one F_7 surface 0.34 -> 0.25 ms and one F_11 surface 1.16 -> 0.79 ms per call with 256 parts instead of 16; 40 F_13
    // quads 4.96 -> 4.52 ms with 64; 94 F_11 quads are best at 16 ... 64 and lose 11 % at 256.
    static constexpr int SPLIT_MID = 64;
    static constexpr int SPLIT_FEW = 256;
    static constexpr int SBW = (P >= 13) ? QFS_DMMA_SBW13 : (P >= 11 ? QFS_DMMA_SBW11 : (P == 7 ? QFS_DMMA_SBW7 : (P == 5 ? QFS_DMMA_SBW5 : 2048)));  // words per staging buffer
    static constexpr int SBX = S::d + 5;                         // window side: 4 zero cells below (taps reach t2, t3 <= 4), u = 0..d
    static constexpr int PLANE = SBX * SBX;
    static constexpr int PLANE_PAD = (PLANE + 3) & ~3;           // words per plane (bulk copies move whole 16-byte units)
    static constexpr int PLANE_BYTES = 4 * PLANE_PAD;
    static constexpr int RING = 5 + LAG;                         // planes u1 = s1-3 .. s1 (one more if a warp may lag a layer behind), s1+1 in flight
    static constexpr int NPLANE = S::dh + 2;                     // planes of the global box: u1 = 0..dh and one of zeros
    static constexpr int TMAX_PAD = ((S::d + 1) * (S::d + 2) / 2 + 3) & ~3;   // points of the layer s1 = 0, in whole 16-byte units
    static QFS_HD constexpr int xoff(int s1)   // first word of layer s1 in the x region (every layer starts on 16 bytes)
    {
        int o = 0;
        for (int l = 0; l < s1; ++l) o += (((S::d - l + 1) * (S::d - l + 2) / 2) + 3) & ~3;
        return o;
    }
    static constexpr int XWORDS = xoff(S::d + 1);
    static constexpr size_t HBOX_WORDS = (size_t)NPLANE * PLANE_PAD + XWORDS;   // per quad: the planes, then the x region
    static constexpr uint32_t MAGIC = 65536u / P + 1;            // x / p = (x * MAGIC) >> 16 for x * (MAGIC * p - 65536) < 65536
    static constexpr int EC_STRIDE = P * P * P * 32 + 16;        // bytes per surface of the class-major coefficient table
    // shared memory (bytes)
    static constexpr int OFF_EC = 0;                                        // [NEC][4][NCLS_PAD][32]
    static constexpr int OFF_WIN = OFF_EC + NEC * 4 * NCLS_PAD * 32;        // uint32 [RING][PLANE_PAD]
    static constexpr int OFF_X = OFF_WIN + RING * PLANE_BYTES;              // uint32 [XS][TMAX_PAD]: the class-0 terms of layers (s1-1,) s1, s1+1
    static constexpr int OFF_COL = OFF_X + XS * TMAX_PAD * 4;               // int4 [NCLS_PAD]
    static constexpr int OFF_BAR = OFF_COL + NCLS_PAD * 16;                 // mbarriers: full[2], empty[2], window[RING], coefficient rows[3]
    static constexpr int OFF_STAGE = OFF_BAR + 128;
    static constexpr int SMEM = OFF_STAGE + NBUF * SBW * 4;
    static constexpr int MINB_S = (228 * 1024) / (SMEM + 1024);   // CTAs per SM that shared memory allows
    static constexpr int MINB = MINB_S < 1 ? 1 : (MINB_S > QFS_DMMA_MAXB ? QFS_DMMA_MAXB : MINB_S);   // register budget: that many CTAs of NT threads
    static_assert(P != 7 || MINB == 4, "k_delta_mma<7> is tuned for four CTAs per SM: shared memory grew past 57 344 bytes");
    static_assert(P != 5 || MINB == 4, "k_delta_mma<5> is tuned for four CTAs per SM");
    static_assert(MAGIC * P - 65536u < 65536u / (35u * (P - 1) * (P - 1) + P), "magic quotient not exact");
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
// Zero words of piece k that no entry covers, as (run-relative) ranges: the gap in front of run I2 and, after the piece's
// last run, the rest of the piece.  rs = piece-relative first word of the run.
template <int P>
QFS_HD constexpr int delta_run_start(int nk, int I2, int cconst, int po)
{
    using S = Shape<P>;
    return cconst - po + delta_F(I2, nk) + S::G * I2;
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
inline bool delta_plan(DeltaPlan& plan, int split = DeltaMmaCfg<P>::SPLIT)
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
                return po <= (uint32_t)C::SBW;
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
                if (words > 0) {
                    DeltaPhase ph{};
                    ph.s1 = (uint8_t)s1; ph.rho1a = (uint8_t)rho1a; ph.nrho1 = (uint8_t)nrho1;
                    ph.s2a = (uint8_t)s2a; ph.s2b = (uint8_t)s2b;
                    ph.npts = (uint16_t)npts;
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
    plan.parts.assign(split + 1, 0);
    uint64_t total = 0;
    for (const auto& ph : plan.phases) total += ph.nwords;
    uint64_t run = 0;
    int part = 1;
    for (size_t i = 0; i < plan.phases.size() && part < split; ++i) {
        run += plan.phases[i].nwords;
        while (part < split && run * split >= total * part) plan.parts[part++] = (uint32_t)(i + 1);
    }
    for (; part <= split; ++part) plan.parts[part] = (uint32_t)plan.phases.size();
    // blocks ((layer, group) runs of phases) and what to prefetch at their first phase, per part
    for (int pt = 0; pt < split; ++pt) {
        const uint32_t a = plan.parts[pt], b = plan.parts[pt + 1];
        for (uint32_t i = a; i < b; ++i) {
            DeltaPhase& ph = plan.phases[i];
            const bool block = (i == a) || plan.phases[i - 1].s1 != ph.s1 || plan.phases[i - 1].rho1a != ph.rho1a;
            if (!block) continue;
            ph.flags |= DPH_BLOCK;
            const bool first_of_layer = (i == a) || plan.phases[i - 1].s1 != ph.s1;
            uint32_t j = i + 1;
            while (j < b && plan.phases[j].s1 == ph.s1 && plan.phases[j].rho1a == ph.rho1a) ++j;   // next block
            if (j < b && plan.phases[j].rho1a != ph.rho1a) {
                ph.flags |= DPH_PF_EC;
                ph.pf_rho1a = plan.phases[j].rho1a;
                ph.pf_nrho1 = plan.phases[j].nrho1;
            }
            if (first_of_layer) {
                uint32_t l = i + 1;
                while (l < b && plan.phases[l].s1 == ph.s1) ++l;
                if (l < b) ph.flags |= DPH_PF_PLANE;   // layer s1 + 1 follows inside this part
            }
        }
    }
    return true;
}

#if defined(__CUDACC__)

#include "qfs_async.cuh"

// ---- inputs of the kernel, built once per chunk -----------------------------------------------------------------------------
// ecm[slot][c][8 words], c = (rho1*p + rho2)*p + rho3: byte b of tap word w = -E[rho + p*t_j] mod p, j = 4w + b (taps ordered by
// |t|, then t1, then t2), stored in the order w = 0,4,1,5,2,6,3,7 (a thread of the MMA reads words tig and tig+4 as one uint2).
// Then 16 bytes: tap word 8 of the class rho = 0 (taps 32..34 and the coefficient 1 of the phi(A) term).
// One CTA per surface: E goes through shared memory, a thread builds a class.
template <int P>
__global__ void __launch_bounds__(128) k_delta_prep(const uint8_t* __restrict__ E_all, uint8_t* __restrict__ ecm_all, int count)
{
    using S = Shape<P>;
    using C = DeltaMmaCfg<P>;
    extern __shared__ __align__(16) uint8_t pe_smem[];
    const int slot = blockIdx.x;
    if (slot >= count) return;
    for (int i = threadIdx.x; i < S::NE_pad / 16; i += 128)
        reinterpret_cast<uint4*>(pe_smem)[i] = reinterpret_cast<const uint4*>(E_all + (size_t)slot * S::NE_pad)[i];
    __syncthreads();
    for (int c = threadIdx.x; c < P * P * P; c += 128) {
        uint32_t* out = reinterpret_cast<uint32_t*>(ecm_all + (size_t)slot * C::EC_STRIDE + (size_t)c * 32);
        const int rho1 = c / (P * P), rho2 = (c / P) % P, rho3 = c % P;
        uint32_t word = 0, wd[8];
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
                        const uint32_t ev = pe_smem[qrowbase(S::dE, J1, J2) + J3];
                        word |= (ev ? (uint32_t)P - ev : 0u) << (8 * (j & 3));
                    }
                    if ((j & 3) == 3) {
                        const int w = j >> 2;
                        wd[2 * (w & 3) + (w >> 2)] = word;
                        word = 0;
                    }
                    ++j;
                }
        reinterpret_cast<uint4*>(out)[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        reinterpret_cast<uint4*>(out)[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
        if (c == 0)
            *reinterpret_cast<uint4*>(ecm_all + (size_t)slot * C::EC_STRIDE + (size_t)P * P * P * 32) =
                make_uint4(word | (1u << 24), 0, 0, 0);   // taps 32..34, then the phi(A) term
    }
}

// hbox[quad][plane u1][cell (u2+4, u3+4)]: the bytes h[u1,u2,u3] of the quad's four surfaces in one word, zero outside the
// support of h = f^(p-2); plane dh+1 is all zeros (the planes u1 < 0 and u1 > dh of the kernel's window).  After the planes, the
// x region: per point s of basis(d) (layer by layer, lex (s2,s3) inside a layer) what the class rho = 0 gets beyond the 32 taps of
// the MMA, x[s] = (A[s] - sum_{j=32..34} E[p t_j] h[s - t_j]) mod p, t_32..34 = (3,0,1), (3,1,0), (4,0,0), again four surfaces a word.
// One CTA per quad; the four h go through shared memory.  Runs after k_delta_prep (it reads the tap word 8 of ecm).
template <int P>
__global__ void __launch_bounds__(256) k_delta_box(const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ A_all,
                                                   const uint8_t* __restrict__ ecm_all, const uint32_t* __restrict__ unrank_d,
                                                   uint32_t* __restrict__ hbox_all, int count)
{
    using S = Shape<P>;
    using C = DeltaMmaCfg<P>;
    extern __shared__ __align__(16) uint8_t pb_smem[];   // [4][Nh_pad]
    const int quad = blockIdx.x;
    const int nlive = min(4, count - 4 * quad);
    for (int i = threadIdx.x; i < 4 * S::Nh_pad / 16; i += 256) {
        const int s = i / (S::Nh_pad / 16);
        reinterpret_cast<uint4*>(pb_smem)[i] =
            s < nlive ? reinterpret_cast<const uint4*>(h_all + (size_t)(4 * quad) * S::Nh_pad)[i] : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    auto hword = [&](int a1, int a2, int a3) -> uint32_t {   // the four surfaces' h[a1,a2,a3], zero outside the support
        if (a1 < 0 || a2 < 0 || a3 < 0 || a1 + a2 + a3 > S::dh) return 0u;
        const int r = qrowbase(S::dh, a1, a2) + a3;
        return (uint32_t)pb_smem[r] | ((uint32_t)pb_smem[S::Nh_pad + r] << 8) | ((uint32_t)pb_smem[2 * S::Nh_pad + r] << 16) |
               ((uint32_t)pb_smem[3 * S::Nh_pad + r] << 24);
    };
    uint32_t* box = hbox_all + (size_t)quad * C::HBOX_WORDS;
    for (int e = threadIdx.x; e < C::NPLANE * C::PLANE_PAD; e += 256) {
        const int u1 = e / C::PLANE_PAD, c = e - u1 * C::PLANE_PAD;
        const int b2 = c / C::SBX, b3 = c - b2 * C::SBX;
        box[e] = (u1 <= S::dh && b2 < C::SBX) ? hword(u1, b2 - 4, b3 - 4) : 0u;
    }
    uint32_t e8[4];
#pragma unroll
    for (int s = 0; s < 4; ++s)
        e8[s] = s < nlive ? *reinterpret_cast<const uint32_t*>(ecm_all + (size_t)(4 * quad + s) * C::EC_STRIDE + (size_t)P * P * P * 32) : 0u;
    uint32_t* xr = box + (size_t)C::NPLANE * C::PLANE_PAD;
    for (int i = threadIdx.x; i < S::N; i += 256) {
        const uint32_t un = unrank_d[i];
        const int s1 = un & 255, s2 = (un >> 8) & 255, s3 = (un >> 16) & 255;
        const uint32_t h32 = hword(s1 - 3, s2, s3 - 1), h33 = hword(s1 - 3, s2 - 1, s3), h34 = hword(s1 - 4, s2, s3);
        uint32_t w = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (s >= nlive) continue;
            const uint32_t x = (e8[s] & 255u) * ((h32 >> (8 * s)) & 255u) + ((e8[s] >> 8) & 255u) * ((h33 >> (8 * s)) & 255u) +
                               ((e8[s] >> 16) & 255u) * ((h34 >> (8 * s)) & 255u) + (e8[s] >> 24) * (uint32_t)A_all[(size_t)(4 * quad + s) * S::pitch + i];
            w |= (x % (uint32_t)P) << (8 * s);
        }
        xr[C::xoff(s1) + (i - qrowbase(S::d, s1, 0))] = w;
    }
}

__device__ __forceinline__ void mma_u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1)
{
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};\n"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(0));
}
__device__ __forceinline__ uint2 lds64(uint32_t addr)
{
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory"); }

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

// 4 x 4 bytes (tap, surface) -> (surface, tap): w_t = the four surfaces' h value of tap t; o[s] = surface s, taps 0..3
__device__ __forceinline__ void taps_to_surfaces(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&o)[4])
{
    const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
    const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
    o[0] = __byte_perm(t0, t1, 0x5410);
    o[1] = __byte_perm(t0, t1, 0x7632);
    o[2] = __byte_perm(t2, t3, 0x5410);
    o[3] = __byte_perm(t2, t3, 0x7632);
}

template <int P>
__global__ void __launch_bounds__(DeltaMmaCfg<P>::NT, DeltaMmaCfg<P>::MINB)
k_delta_mma(const uint32_t* __restrict__ hbox_all, const uint8_t* __restrict__ ecm_all,
            const DeltaPhase* __restrict__ phases, const DeltaPiece* __restrict__ pieces, const uint32_t* __restrict__ parts,
            uint8_t* __restrict__ delta_all, int count, int split)
{
    using S = Shape<P>;
    using C = DeltaMmaCfg<P>;
    extern __shared__ __align__(128) uint8_t dm_smem[];
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(dm_smem);
    const uint32_t aEc = sbase + C::OFF_EC, aWin = sbase + C::OFF_WIN, aX = sbase + C::OFF_X, aStage = sbase + C::OFF_STAGE;
    const uint32_t bFull = sbase + C::OFF_BAR, bEmpty = bFull + 16, bWin = bFull + 32, bEc = bWin + 8 * C::RING;
    int4* sCol = reinterpret_cast<int4*>(dm_smem + C::OFF_COL);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int quad = blockIdx.x / split, part = blockIdx.x % split;   // `split` CTAs per quad, each with its own part of the plan
    const int nlive = min(4, count - 4 * quad);   // slots >= count are padding: their Delta is zero
    const uint32_t pa = parts[part];
    const int nph = (int)(parts[part + 1] - pa);
    uint8_t* gq = delta_all + (size_t)quad * S::quad_stride;
    const uint32_t* hbox = hbox_all + (size_t)quad * C::HBOX_WORDS;

    if (tid == 0) {
        mbar_init(bFull, C::NWI); mbar_init(bFull + 8, C::NWI);
        mbar_init(bEmpty, 1); mbar_init(bEmpty + 8, 1);
        for (int i = 0; i < C::RING; ++i) mbar_init(bWin + 8 * i, 1);
        for (int i = 0; i < 3; ++i) mbar_init(bEc + 8 * i, 1);
        mbar_fence_init();
    }
    // coefficient rows of pad classes and of padding surfaces stay zero
    for (int i = tid; i < C::NEC * 4 * C::NCLS_PAD * 2; i += C::NT) reinterpret_cast<uint4*>(dm_smem + C::OFF_EC)[i] = make_uint4(0, 0, 0, 0);
    // column constants (bytes), the same for every phase: word = R + cconst_k + C + rho2 * n0 - a * m  (delta_col with n0 = 0)
    for (int c = tid; c < C::NCLS_PAD; c += C::NT) {
        int4 ci = make_int4(0, 0, 0x7fff, 0);
        if (c < C::NCLS) {
            const int k = c / (P * P), r = c - k * (P * P), rho2 = r / P, rho3 = r - rho2 * P;
            int Cc, m, need;
            delta_col<P>(0, k, rho2, rho3, 0, Cc, m, need);
            ci = make_int4(4 * Cc, m, need, k | (rho2 << 8));
        }
        sCol[c] = ci;
    }
    fence_proxy_async();
    __syncthreads();

    // GUARD ZEROS of a phase, a run per lane: the gap in front of the run and, after the last run of a piece, the rest of the piece.
    // With the entries these are all the words of the phase (tools/check_delta_plan.cpp), so nothing ever clears a buffer.
    // Who writes them (C::STORE_GUARDS): with one rho1 per phase (p >= 7) the store warp, right after the copies of phase li have read
    // the buffer and while the item warps are already writing the entries of phase li + NBUF (disjoint words) -- F_7 -4 %, F_11 -4 %,
    // F_13 -9 %; with all rho1 in a phase (p <= 5: ~200 runs per phase) one warp would be the critical path (F_5 +7 %), so there
    // every item warp zeroes its share of the runs before its tiles.
    auto guards = [&](const DeltaPhase& ph, const DeltaPiece& pcl, int b, int share, int nshare) {
        const int nrho1 = ph.nrho1, s2a = ph.s2a;
        const int n0 = S::D - P * ph.s1 - ph.rho1a;
        const int per = P * (ph.s2b - s2a);
        const int nruns = nrho1 * per;   // (slab, run) pairs of the phase
        const uint32_t stageB = aStage + 4u * (uint32_t)(b * C::SBW);
        const int g_hi = ((share + 1) * nruns) / nshare;
        for (int g0 = (share * nruns) / nshare; g0 < g_hi; g0 += 32) {   // uniform trip count: the shuffles need every lane
            const int gi = g0 + lane;
            const int k = min(gi / per, nrho1 - 1), j = gi - k * per;
            const int I2 = P * s2a + j, nk = n0 - k;
            const int pcc = __shfl_sync(0xffffffffu, pcl.cconst, k), ppo = __shfl_sync(0xffffffffu, (int)pcl.po, k),
                      pnw = __shfl_sync(0xffffffffu, (int)pcl.nw, k);
            if (gi >= g_hi) continue;
            if (I2 <= nk && pnw > 0) {
                const int rs = delta_run_start<P>(nk, I2, pcc, ppo);
                const uint32_t pieceB = stageB + 4u * (uint32_t)ppo;
                for (int w = (j == 0 ? 0 : rs - S::G); w < rs; ++w) sts32(pieceB + 4u * (uint32_t)w, 0u);
                if (I2 == min(P * (int)ph.s2b - 1, nk))
                    for (int w = rs + (nk - I2 + 1); w < pnw; ++w) sts32(pieceB + 4u * (uint32_t)w, 0u);
            }
        }
    };
    // ---- store warp: a phase's pieces leave with bulk copies as soon as every item warp has delivered ----------------------------
    if (warp == C::NWI) {
        // lane k owns piece k of a phase; the descriptors of the next phase are fetched before the wait (no global latency in the chain)
        DeltaPhase phd = phases[pa];
        DeltaPiece pc = pieces[phd.piece0 + min(lane, (int)phd.nrho1 - 1)];
        if (C::STORE_GUARDS) {
            guards(phd, pc, 0, 0, 1);
            if (C::NBUF > 1 && nph > 1) {
                const DeltaPhase p1 = phases[pa + 1];
                guards(p1, pieces[p1.piece0 + min(lane, (int)p1.nrho1 - 1)], 1, 0, 1);
            }
        }
        for (int li = 0; li < nph; ++li) {
            const int b = li % C::NBUF;
            const DeltaPhase nphd = phases[pa + min(li + 1, nph - 1)];
            const DeltaPiece npc = pieces[nphd.piece0 + min(lane, (int)nphd.nrho1 - 1)];
            const DeltaPhase gph = phases[pa + min(li + C::NBUF, nph - 1)];          // the phase that gets this buffer next
            const DeltaPiece gpc = pieces[gph.piece0 + min(lane, (int)gph.nrho1 - 1)];
            if (lane == 0) mbar_wait_backoff(bFull + 8 * b, (uint32_t)((li / C::NBUF) & 1));
            fence_proxy_async();   // this warp's guard zeros, too, are visible to the copy engine
            __syncwarp();
            if (lane < phd.nrho1 && pc.nw) bulk_s2g(gq + 4 * (size_t)pc.ga, aStage + 4u * (uint32_t)(b * C::SBW + (int)pc.po), pc.nw * 4u);
            bulk_commit();
            bulk_wait_read0();
            __syncwarp();
            if (lane == 0) mbar_arrive(bEmpty + 8 * b);
            if (C::STORE_GUARDS && li + C::NBUF < nph) guards(gph, gpc, b, 0, 1);
            phd = nphd;
            pc = npc;
        }
        return;
    }

    // ---- item warps ---------------------------------------------------------------------------------------------------------------
    auto load_ec = [&](int idx, int rho1a, int nrho1) {   // one thread: the group's class rows of the live surfaces, load number idx
        const uint32_t bytes = (uint32_t)(nrho1 * P * P * 32);
        const uint32_t bar = bEc + 8 * (idx % C::NEC);
        mbar_expect_tx(bar, bytes * (uint32_t)nlive);
        for (int s = 0; s < nlive; ++s)
            bulk_g2s(aEc + (uint32_t)(((idx % C::NEC) * 4 + s) * C::NCLS_PAD * 32), ecm_all + (size_t)(4 * quad + s) * C::EC_STRIDE + (size_t)rho1a * P * P * 32,
                     bytes, bar);
    };
    auto load_plane = [&](int u1, bool with_x) {   // one thread: plane u1 of the window (zeros outside 0..dh) into its ring slot,
        const int pl = (u1 >= 0 && u1 <= S::dh) ? u1 : S::dh + 1, slot = (u1 + C::RING) % C::RING;   // and the layer's class-0 terms
        const int nsx = S::d - u1;
        const uint32_t xbytes = with_x ? 4u * (uint32_t)((((nsx + 1) * (nsx + 2) / 2) + 3) & ~3) : 0u;
        mbar_expect_tx(bWin + 8 * slot, C::PLANE_BYTES + xbytes);
        bulk_g2s(aWin + (uint32_t)(slot * C::PLANE_BYTES), hbox + (size_t)pl * C::PLANE_PAD, C::PLANE_BYTES, bWin + 8 * slot);
        if (with_x)
            bulk_g2s(aX + (uint32_t)((u1 % C::XS) * C::TMAX_PAD * 4), hbox + (size_t)C::NPLANE * C::PLANE_PAD + C::xoff(u1), xbytes, bWin + 8 * slot);
    };
    // No barrier among the item warps: a warp is never more than one phase behind another (two staging buffers), so a plane or
    // a group of coefficient rows may be overwritten one block after its last use (RING = 5 + LAG planes, 2 + LAG row buffers), and every
    // warp derives the same mbarrier parities from the phase list.
    int cur_s1 = -100, cur_grp = -1, ec_idx = -1, first_s1 = 0;
    int toffB[8];   // byte offsets (from a point's cell) of this thread's eight taps
#pragma unroll
    for (int i = 0; i < 8; ++i) toffB[i] = 0;
    DeltaPhase phd = phases[pa];
    DeltaPiece mypc = pieces[phd.piece0 + min(lane, (int)phd.nrho1 - 1)];   // lane k: piece k of the phase (descriptors one phase ahead)
#pragma unroll 1
    for (int li = 0; li < nph; ++li) {
        const DeltaPhase nxt = phases[pa + min(li + 1, nph - 1)];
        const DeltaPiece nxtpc = pieces[nxt.piece0 + min(lane, (int)nxt.nrho1 - 1)];
        const int s1 = phd.s1, rho1a = phd.rho1a, nrho1 = phd.nrho1, s2a = phd.s2a, npts = phd.npts;
        const int ns = S::d - s1;
        const int n0 = S::D - P * s1 - rho1a;
        const int ncls = nrho1 * P * P;
        const int b = li % C::NBUF;
        // The copies of phase li-NBUF have read this buffer.  That also bounds the lag between item warps: every one of them has
        // delivered phase li-NBUF, so none is further back than phase li-1 (NBUF <= 2).
        if (li >= C::NBUF) mbar_wait(bEmpty + 8 * b, (uint32_t)(((li / C::NBUF) - 1) & 1));

        if (phd.flags & DPH_BLOCK) {
            const bool first = cur_s1 < 0;
            if (first) {
                first_s1 = s1;
                if (tid == 0) {
                    for (int u1 = s1 - 3; u1 <= s1; ++u1) load_plane(u1, u1 == s1);
                    load_ec(0, rho1a, nrho1);
                }
                for (int u1 = s1 - 3; u1 < s1; ++u1) mbar_wait(bWin + 8 * ((u1 + C::RING) % C::RING), 0);
            }
            if (first || s1 != cur_s1)   // plane s1 is the (s1 - first_s1 + 3)-th load of the window: use number (that / RING) of its slot
                mbar_wait(bWin + 8 * (s1 % C::RING), (uint32_t)(((s1 - first_s1 + 3) / C::RING) & 1));
            if (first || rho1a != cur_grp) {
                ++ec_idx;
                mbar_wait(bEc + 8 * (ec_idx % C::NEC), (uint32_t)((ec_idx / C::NEC) & 1));
            }
            if (tid == 0) {
                if (phd.flags & DPH_PF_PLANE) load_plane(s1 + 1, true);
                if (phd.flags & DPH_PF_EC) load_ec(ec_idx + 1, phd.pf_rho1a, phd.pf_nrho1);
            }
            if (first || s1 != cur_s1) {   // tap offsets of this layer: plane slot of u1 = s1 - t1, then rows and cells back
                int sl[4];
#pragma unroll
                for (int t1 = 0; t1 < 4; ++t1) sl[t1] = ((s1 - t1 + C::RING) % C::RING) * C::PLANE_BYTES;
                int j = 0;
#pragma unroll
                for (int k = 0; k <= 4; ++k)
#pragma unroll
                    for (int t1 = 0; t1 <= k; ++t1)
#pragma unroll
                        for (int t2 = 0; t2 <= k - t1; ++t2) {
                            const int t3 = k - t1 - t2;
                            if (j < 32 && ((j >> 2) & 3) == tig) toffB[(j & 3) + 4 * (j >> 4)] = sl[t1 & 3] - 4 * (t2 * C::SBX + t3);
                            ++j;
                        }
            }
            cur_s1 = s1;
            cur_grp = rho1a;
        }

        const int my_cc = mypc.cconst;
        const uint32_t stageB = aStage + 4u * (uint32_t)(b * C::SBW);
        const int cc0 = __shfl_sync(0xffffffffu, my_cc, 0);
        const uint32_t aEcCur = aEc + (uint32_t)((ec_idx % C::NEC) * 4 * C::NCLS_PAD * 32);
        const int n04 = 4 * n0;
        const int nmt = (npts + 15) >> 4;
        const int ntile = (ncls + 7) >> 3;
        const int wr = (warp + li) % C::NWI;   // rotate the shares: the remainders do not always hit the same warps

        if (!C::STORE_GUARDS) guards(phd, mypc, b, wr, C::NWI);

        // ---- tiles (16 points x 8 classes), an equal share of the phase's nmt x ntile tiles per warp, in (point tile, class tile) order:
        //      the A fragments are gathered once per point tile of the share (at most twice per phase for most shares)
        const int T = nmt * ntile;
        const uint32_t xrowB = aX + 4u * (uint32_t)((s1 % C::XS) * C::TMAX_PAD + s2a * (ns + 1) - (s2a * (s2a - 1)) / 2);   // the phase's first point
        int t = (wr * T) / C::NWI;
        const int t_hi = ((wr + 1) * T) / C::NWI;
        int mt = t / ntile, nt = t - mt * ntile;
#pragma unroll 1
        while (t < t_hi) {
            uint32_t a[4][4];
            uint32_t Rb[2];
            int nab[2], room[2];
            uint32_t cellB[2];
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int ql = mt * 16 + g + 8 * r;
                const bool real = ql < npts;
                // point ql of the rows s2a, s2a+1, ... (lengths m, m-1, ...): u rows lie in front of it, c(u) = u m - u(u-1)/2 points
                const int m2 = 2 * (ns - s2a + 1) + 1, q = real ? ql : 0;
                int u = (int)(((float)m2 - sqrtf((float)(m2 * m2 - 8 * q))) * 0.5f);
                while (u > 0 && (u * (m2 - u)) / 2 > q) --u;
                while (((u + 1) * (m2 - u - 1)) / 2 <= q) ++u;
                const int s2 = s2a + u, s3 = q - (u * (m2 - u)) / 2;
                int R, aa, rm;
                delta_row<P>(n0, s2, s3, R, aa, rm);
                Rb[r] = stageB + 4u * (uint32_t)(R + (C::RG == 1 ? cc0 : 0));
                nab[r] = -4 * aa;
                room[r] = real ? rm : -1;
                cellB[r] = aWin + 4u * (uint32_t)((s2 + 4) * C::SBX + s3 + 4);
                uint32_t w[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = lds32(cellB[r] + toffB[i]);
                uint32_t lo[4], hi[4];
                taps_to_surfaces(w[0], w[1], w[2], w[3], lo);
                taps_to_surfaces(w[4], w[5], w[6], w[7], hi);
#pragma unroll
                for (int s = 0; s < 4; ++s) { a[s][r] = lo[s]; a[s][2 + r] = hi[s]; }
            }
            auto tile = [&](int nt, auto first_tag) {
                constexpr bool FIRST = decltype(first_tag)::value;
                int acc[4][4];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const uint2 bb = lds64(aEcCur + (uint32_t)(((s * C::NCLS_PAD + nt * 8 + g) * 32) + tig * 8));
                    mma_u8(acc[s], a[s][0], a[s][1], a[s][2], a[s][3], bb.x, bb.y);
                }
                if (FIRST && tig == 0) {
                    // class rho = 0 (first class of a group with rho1a = 0): taps 32..34 and the phi(A) term join its accumulators
#pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        const uint32_t xw = (room[r] >= 0) ? lds32(xrowB + 4u * (uint32_t)(mt * 16 + g + 8 * r)) : 0u;
#pragma unroll
                        for (int s = 0; s < 4; ++s) acc[s][2 * r] += (int)((xw >> (8 * s)) & 255u);
                    }
                }
                const int4 c0 = sCol[nt * 8 + 2 * tig], c1 = sCol[nt * 8 + 2 * tig + 1];   // (4C, m, need, k | rho2 << 8)
                int k0 = c0.x + (c0.w >> 8) * n04, k1 = c1.x + (c1.w >> 8) * n04;
                if (C::RG > 1) {
                    k0 += 4 * __shfl_sync(0xffffffffu, my_cc, c0.w & 255);
                    k1 += 4 * __shfl_sync(0xffffffffu, my_cc, c1.w & 255);
                }
                // accumulator i of the fragment: 0: (row g, col 2tig), 1: (g, 2tig+1), 2: (g+8, 2tig), 3: (g+8, 2tig+1)
                const uint32_t w00 = reduce_pack4<P>(acc[0][0], acc[1][0], acc[2][0], acc[3][0]);
                if (room[0] >= c0.z) sts32(Rb[0] + (uint32_t)(k0 + nab[0] * c0.y), w00);
                const uint32_t w01 = reduce_pack4<P>(acc[0][1], acc[1][1], acc[2][1], acc[3][1]);
                if (room[0] >= c1.z) sts32(Rb[0] + (uint32_t)(k1 + nab[0] * c1.y), w01);
                const uint32_t w10 = reduce_pack4<P>(acc[0][2], acc[1][2], acc[2][2], acc[3][2]);
                if (room[1] >= c0.z) sts32(Rb[1] + (uint32_t)(k0 + nab[1] * c0.y), w10);
                const uint32_t w11 = reduce_pack4<P>(acc[0][3], acc[1][3], acc[2][3], acc[3][3]);
                if (room[1] >= c1.z) sts32(Rb[1] + (uint32_t)(k1 + nab[1] * c1.y), w11);
            };
            const int nt_end = min(ntile, nt + (t_hi - t));
            t += nt_end - nt;
            if (nt == 0 && rho1a == 0) { tile(0, std::true_type{}); ++nt; }
#pragma unroll 2
            for (; nt < nt_end; ++nt) tile(nt, std::false_type{});
            if (nt == ntile) { nt = 0; ++mt; }
        }
        // delivered: this warp's words of the phase are visible to the copy engine
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(bFull + 8 * b);
        phd = nxt;
        mypc = nxtpc;
    }
}

#endif  // __CUDACC__
