// qfs_matrix_staged.cuh -- stage 3, the operator-matrix builder (v6): the gather
//     M[r, c] = Delta[p*r + (p-1) - c]      (qfs_matrix.cuh has the derivation)
// with the Delta windows of a work item staged in shared memory by bulk asynchronous copies and
// the rows written with 8- or 16-byte stores.
//
// Why (measured, profiles/README.md).  The v4 builder gathers straight from global memory: a
// warp-wide LDG.32 touches ~10 cache lines (the 128 columns of a warp cross ~20 column runs that
// live in different Delta runs) and the L1 tag stage -- one line per cycle -- caps it at ~3.1 TB/s
// of matrix writes.  Shared memory has no tag stage, only banks.  And 4-byte stores (128 bytes
// per warp request) stall at ~4.8 TB/s on this part whatever feeds them (tools/micro/write_bw*.cu:
// STG.32 5.0-5.2 TB/s, STG.64 6.6, STG.128 7.0 TB/s), so a thread owns V consecutive words of a row.
//
// What is staged.  For a row group (r1,r2) the sources of the column block c1 (all c2, c3) are the
// Delta runs (I1, I2lo..I2hi), I1 = p r1+p-1-c1, I2 = p r2+p-1-c2: ONE contiguous piece of the
// guard-banded lex43g array (qfs_shape.cuh), because runs are ordered by (I1, I2).  A work item
// ("panel") = (r1, r2, word groups [glo, glo+ngrp) of the rows): a column range whose ends sit on
// 128-byte lines of the row (tools/micro/write_bw4.cu: segments that share no line with a neighbour
// panel write 1.2-1.8x faster).  It stages, for every column block c1 its columns touch, the piece
// restricted to the c2 it needs (first block: c2 >= c2lo, last block: c2 <= c2hi) and writes its word
// groups (V x 32 bits) of every row of the group.  The host cuts every row into panels that fit the
// shared-memory budget (p = 3, 5: one per row group).
//
// CTA = NT consumer threads + one producer warp.  Consumers: thread = (row team, word group); the
// V teams take the rows t = team, team+V, ...  Producer warp: issues the bulk copies of the next
// quad's pieces (cp.async.bulk -> mbarrier), prefetches the one after into L2, and finishes the
// fused first step v1 = M g of the previous quad (sums the per-warp partial dot products).
#pragma once
#include <limits.h>

#include "qfs_async.cuh"
#include "qfs_delta.cuh"  // transpose4x4
#include "qfs_shape.cuh"

struct PanelItem {
    uint8_t r1, r2, c1lo, c1hi;   // row group; first and last column block the panel's columns touch
    uint16_t glo, ngrp;           // owned word groups of a row: [glo, glo + ngrp), in units of V 32-bit words
    uint8_t c2lo, c2hi;           // c2 of the panel's first column (in block c1lo) and of its last column (in block c1hi)
    uint16_t pad;
};

template <int P>
struct StagedCfg {
    using S = Shape<P>;
#ifndef QFS_V5
#define QFS_V5 1
#endif
    static constexpr int V = (P >= 7) ? 2 : (P == 5 ? QFS_V5 : 1);                              // consecutive 32-bit words per thread (store width 4V bytes)
    static constexpr int TEAMS = V;                          // row teams
#ifndef QFS_NT7
#define QFS_NT7 128
#endif
#ifndef QFS_NT5
#define QFS_NT5 128
#endif
#ifndef QFS_BUDGET5
#define QFS_BUDGET5 6000
#endif
#ifndef QFS_SLICE5
#define QFS_SLICE5 24
#endif
#ifndef QFS_NT13
#define QFS_NT13 256
#endif
#ifndef QFS_BUDGET13
#define QFS_BUDGET13 24576
#endif
#ifndef QFS_NT11
#define QFS_NT11 256
#endif
#ifndef QFS_SLICE7
#define QFS_SLICE7 12
#endif
#ifndef QFS_SLICE11
#define QFS_SLICE11 8
#endif
#ifndef QFS_BUDGET7
#define QFS_BUDGET7 8400
#endif
#ifndef QFS_BUDGET11
#define QFS_BUDGET11 16384
#endif
    static constexpr int NT = (P >= 13) ? QFS_NT13 : (P == 11 ? QFS_NT11 : (P == 7 ? QFS_NT7 : (P >= 5 ? QFS_NT5 : 64)));  // consumer threads (p = 13: block c1 = 0 alone is 154 word groups; p = 7: 96-thread teams fit its ~91-group panels)
    static constexpr int TEAM = NT / TEAMS;                  // threads (= word groups) per team
    static constexpr int NTL = NT + 32;                      // launched: + the producer warp
    static constexpr int WORDS = S::pitch / 4;
    static constexpr int NGRP = WORDS / V;                   // word groups per row
    static constexpr int MAXG = TEAM;                        // most word groups a panel may own
    // Rows that start on 128-byte lines (QFS_PITCH_ALIGN = 128): the warps of a team start at the line in front of the
    // panel's first word group, so that every warp store covers whole lines (tools/micro/write_bw4.cu); the
    // glo % LINEG threads in front of the panel repeat its first word group.
    static constexpr int LINEG = (QFS_PITCH_ALIGN % 128 == 0) ? 128 / (4 * V) : 1;
    static constexpr int MAXROWS = S::d + 1;
#ifndef QFS_SLICE13
#define QFS_SLICE13 QFS_SLICE11
#endif
    static constexpr int SLICE = (P >= 13) ? QFS_SLICE13 : (P >= 11 ? QFS_SLICE11 : (P >= 7 ? QFS_SLICE7 : QFS_SLICE5));        // quads per CTA
    static constexpr int ZW = (P * S::d + 4 + 3) & ~3;       // zero region (entries) read by columns that never match
    static constexpr int MAXC = S::d + 2;                    // pieces per panel
    static constexpr int BUDGET = (P >= 13) ? QFS_BUDGET13 : (P >= 11 ? QFS_BUDGET11 : (P == 7 ? QFS_BUDGET7 : (P == 5 ? QFS_BUDGET5 : 12800)));  // default staged entries (x4 bytes) per panel
    static constexpr size_t MSTRIDE = (size_t)S::N * S::pitch;
    // launch order of the row groups: blocks of ORDER_T1 values of r1 x ORDER_T2 values of r2 (1 x 1: lexicographic); see build_tables
    static constexpr int ORDER_T1 = (P == 13) ? 2 : (P == 11 ? S::d + 1 : 1);
    static constexpr int ORDER_T2 = (P == 11) ? 4 : 1;
    static constexpr int VSEG = MAXG * 4 * V + 16;           // bytes of one surface's slice of v0 staged per buffer (16-byte aligned window)
    static constexpr int VWORDS = 4 * VSEG / 4;              // 32-bit words of the v0 area at the end of a buffer
    static_assert(WORDS % V == 0 && TEAM % 32 == 0 || P == 3, "teams are whole warps");
};

// The piece of Delta that column block c1 of row group (r1,r2) reads, restricted to c2min <= c2 <= c2max:
// entries [a, b) of the lex43g array (a rounded down, b rounded up to a multiple of 32 entries = 128 bytes
// of the quad-interleaved array).  Returns false when no column of the block can match.
template <int P>
QFS_HD bool staged_piece(int r1, int r2, int c1, int c2min, int c2max, int& a4, int& b4)
{
    using S = Shape<P>;
    const int I1 = P * r1 + P - 1 - c1;
    if (I1 < 0 || I1 > S::D) return false;
    int I2lo = P * r2 + P - 1 - c2max, I2hi = P * r2 + P - 1 - c2min;
    if (I2lo < 0) I2lo = 0;
    if (I2hi > S::D - I1) I2hi = S::D - I1;
    if (I2lo > I2hi) return false;
    a4 = (S::gbase(I1, I2lo) - S::G) & ~31;
    b4 = (S::gbase(I1, I2hi + 1) + 31) & ~31;
    return true;
}

template <int V> struct StoreVec;
template <> struct StoreVec<1> { using T = uint32_t; };
template <> struct StoreVec<2> { using T = uint2; };
template <> struct StoreVec<4> { using T = uint4; };

// One row (team row index u relative to the thread's current base) of the thread's word group, four surfaces.
// sp[k]: shared-memory byte address of the source word of column k of the group for the base row;
// dst[s]: the thread's word group in the base row of matrix s.
template <int P, bool FUSE, int U>
__device__ __forceinline__ void staged_row(const uint32_t (&sp)[4 * StagedCfg<P>::V], typename StoreVec<StagedCfg<P>::V>::T* const (&dst)[4],
                                           const uint32_t (&vw)[StagedCfg<P>::V][4], int* accp, int lane)
{
    using S = Shape<P>;
    using C = StagedCfg<P>;
    constexpr int STEP = C::TEAMS * U;  // rows between the base row and this one
    uint32_t o[C::V][4];
#pragma unroll
    for (int j = 0; j < C::V; ++j) {
        uint32_t in[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) in[k] = lds32(sp[4 * j + k] + 4 * P * STEP);
        transpose4x4(in, o[j]);  // o[j][s] = columns 4j..4j+3 of the group, surface s
    }
    uint32_t part[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        typename StoreVec<C::V>::T* a = dst[s] - STEP * (S::pitch / (4 * C::V));
        // streaming stores (st.global.cs): M is written once and not read back before the chain, and the lines it would
        // otherwise hold in L2 are the ones the staged Delta pieces want (F_11 / F_13: -1.3 %, F_5 / F_7: -0.5 %)
        if constexpr (C::V == 1) __stcs(a, o[0][s]);
        else if constexpr (C::V == 2) __stcs(a, make_uint2(o[0][s], o[1][s]));
        else __stcs(a, make_uint4(o[0][s], o[1][s], o[2][s], o[3][s]));
        if (FUSE) {
            part[s] = 0;
#pragma unroll
            for (int j = 0; j < C::V; ++j) part[s] = __dp4a(o[j][s], vw[j][s], part[s]);
        }
    }
    if (FUSE) {
        // two surfaces per 32-bit word (a warp sum stays < 2^16: 32 lanes x V x 4 x (p-1)^2), two REDUX,
        // lanes 0/1 store to the warp's own [row][pair] slot: no atomics, no branches
        const uint32_t t01 = __reduce_add_sync(0xffffffffu, part[0] + (part[1] << 16));
        const uint32_t t23 = __reduce_add_sync(0xffffffffu, part[2] + (part[3] << 16));
        if (lane < 2) accp[-2 * STEP] = (int)(lane ? t23 : t01);
    }
}

// items sorted by decreasing work.  vacc: [slot][pitch] int accumulators (used when a row group has
// several panels: flags & 1; zeroed by the caller).  Dynamic shared memory: nbuf buffers of `bufwords`
// 32-bit words (one word = one Delta entry of the 4 surfaces of a quad), each = [ZW zero words][pieces].
template <int P, bool FUSE>
__global__ void __launch_bounds__(StagedCfg<P>::NTL)
k_matrix_staged(const uint8_t* __restrict__ delta_all, const uint32_t* __restrict__ colinfo,
                const PanelItem* __restrict__ items, uint8_t* __restrict__ M_all, const uint8_t* __restrict__ v0_all,
                uint8_t* __restrict__ v1_all, int* __restrict__ vacc, int count, int bufwords, int nbuf, int flags)
{
    using S = Shape<P>;
    using C = StagedCfg<P>;
    using VT = typename StoreVec<C::V>::T;
    constexpr int WPT = C::TEAM / 32 > 0 ? C::TEAM / 32 : 1;  // warps per team
    constexpr int PART = WPT * C::MAXROWS * 2;                 // ints of one s_part parity: [warp in team][r3][surface pair]
    extern __shared__ __align__(128) uint32_t sm[];
    __shared__ __align__(8) uint64_t s_bar[4];
    __shared__ int s_part[FUSE ? 2 * PART : 1];
    __shared__ int s_rel[C::MAXC];
    __shared__ int s_cpa[C::MAXC], s_cpn[C::MAXC], s_cps[C::MAXC];
    __shared__ int s_ncp;

    const PanelItem it = items[blockIdx.x];
    const int r1 = it.r1, r2 = it.r2, c1lo = it.c1lo, c1hi = it.c1hi;
    const int R = S::d - r1 - r2;
    const int row0 = qrowbase(S::d, r1, r2);
    const int tid = threadIdx.x, lane = tid & 31;
    const int nquads = (count + 3) >> 2;
    const int q_begin = blockIdx.y * C::SLICE;
    const int q_end = min(nquads, q_begin + C::SLICE);
    const int cfirst = c1lo;
    const uint32_t sm_base = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(s_bar);
    const uint32_t bufbytes = 4u * (uint32_t)bufwords;

    if (tid == 0) {
        int so = C::ZW, n = 0;
        for (int c1 = cfirst; c1 <= c1hi; ++c1) {
            int a4, b4, rel = INT_MIN;
            const int c2min = (c1 == c1lo) ? it.c2lo : 0, c2max = (c1 == c1hi) ? it.c2hi : S::d - c1;
            if (staged_piece<P>(r1, r2, c1, c2min, c2max, a4, b4)) {
                rel = so - a4;
                s_cpa[n] = a4;
                s_cpn[n] = 4 * (b4 - a4);  // bytes
                s_cps[n] = 4 * so;         // byte offset inside a buffer
                ++n;
                so += b4 - a4;
            }
            s_rel[c1 - cfirst] = rel;
        }
        s_ncp = n;
        for (int b = 0; b < 4; ++b) mbar_init(bar0 + 8 * b, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int b = 0; b < nbuf; ++b)
        for (int i = tid; i < C::ZW; i += C::NTL) sm[b * bufwords + i] = 0u;
    __syncthreads();

    if (tid >= C::NT) {
        // ---- producer warp ----
        const int n = s_ncp;
        uint32_t total = 0;
        for (int ci = 0; ci < n; ++ci) total += (uint32_t)s_cpn[ci];
        // v0 window of this panel: bytes [vlo, vlo + vlen) of a surface's vector, 16-byte aligned
        const uint32_t vlo = (4u * C::V * it.glo) & ~15u;
        const uint32_t vlen = FUSE ? min((uint32_t)S::pitch, (4u * C::V * (it.glo + it.ngrp) + 15u) & ~15u) - vlo : 0u;
        auto issue = [&](int quad, int b) {
            if (n == 0 && !FUSE) return;
            const uint32_t bar = bar0 + 8u * b;
            const uint8_t* dq = delta_all + (size_t)quad * S::quad_stride;
            if (lane == 0) mbar_expect_tx(bar, total + 4u * vlen);
            __syncwarp();
            for (int ci = lane; ci < n; ci += 32)
                bulk_g2s(sm_base + b * bufbytes + (uint32_t)s_cps[ci], dq + 4 * (size_t)s_cpa[ci], (uint32_t)s_cpn[ci], bar);
            if (FUSE && lane >= 28)
                bulk_g2s(sm_base + (b + 1) * bufbytes - 4u * C::VWORDS + (lane - 28) * C::VSEG,
                         v0_all + (4 * (size_t)quad + (lane - 28)) * S::pitch + vlo, vlen, bar);
        };
        auto prefetch = [&](int quad) {  // pull the pieces of a later quad into L2 (first touch comes from HBM)
            const uint8_t* dq = delta_all + (size_t)quad * S::quad_stride;
            for (int ci = lane; ci < n; ci += 32) bulk_prefetch_l2(dq + 4 * (size_t)s_cpa[ci], (uint32_t)s_cpn[ci]);
        };
        auto epilogue = [&](int quad, int pb) {
            for (int e = lane; e < 4 * (R + 1); e += 32) {
                const int s = e / (R + 1), r3 = e - s * (R + 1);
                const int* pp = &s_part[pb * PART + r3 * 2 + (s >> 1)];
                uint32_t a = 0;
#pragma unroll
                for (int w = 0; w < WPT; ++w) a += ((uint32_t)pp[w * C::MAXROWS * 2] >> (16 * (s & 1))) & 0xffffu;
                const size_t o = (4 * (size_t)quad + s) * S::pitch + row0 + r3;
                if (flags & 1) atomicAdd(vacc + o, (int)a);
                else v1_all[o] = (uint8_t)(a % (uint32_t)P);
            }
        };
        for (int k = 0; k < nbuf - 1; ++k)
            if (q_begin + k < q_end) issue(q_begin + k, k);
        for (int quad = q_begin, i = 0; quad < q_end; ++quad, ++i) {
            // the consumers are past the rows of quad i-1 (barrier below): its buffer and s_part[(i-1)&1] are settled
            if (quad + nbuf - 1 < q_end) issue(quad + nbuf - 1, (i + nbuf - 1) % nbuf);
            if (quad + nbuf < q_end) prefetch(quad + nbuf);
            if (FUSE && i > 0) epilogue(quad - 1, (i - 1) & 1);
            asm volatile("bar.sync 1, %0;" ::"n"(C::NTL) : "memory");  // all consumers have arrived: quad i is written
        }
        if (FUSE && q_begin < q_end) epilogue(q_end - 1, (q_end - 1 - q_begin) & 1);
        return;
    }

    // ---- consumers ----
    const int team = tid / C::TEAM, tt = tid - team * C::TEAM;
    const int trel = tt - (int)(it.glo % C::LINEG);       // warps start on 128-byte lines of the row (LINEG > 1)
    const int grp = it.glo + max(0, min(trel, (int)it.ngrp - 1));   // threads outside the panel repeat its first / last word group
    const bool live = trel >= 0 && trel < (int)it.ngrp;
    uint32_t sp[4 * C::V];
#pragma unroll
    for (int k = 0; k < 4 * C::V; ++k) {
        int idx = 0;
        const uint32_t info = colinfo[4 * C::V * grp + k];
        if (info != 0xFFFFFFFFu) {
            const int c1 = info & 255, c2 = (info >> 8) & 255, c3 = info >> 16;
            const int I1 = P * r1 + P - 1 - c1, I2 = P * r2 + P - 1 - c2;
            if (I1 >= 0 && I2 >= 0 && I1 + I2 <= S::D)
                idx = s_rel[c1 - cfirst] + S::gbase(I1, I2) + (P - 1) - (S::d - c1 - c2) + c3;
        }
        sp[k] = sm_base + 4u * (uint32_t)(idx + P * team);  // row t = team
    }
    const bool staged = s_ncp > 0 || FUSE;
    // this thread's words of v0 inside the staged window (buffer 0, surface 0)
    const uint32_t vaddr = sm_base + bufbytes - 4u * C::VWORDS + (4u * C::V * grp - ((4u * C::V * it.glo) & ~15u));
    // team rows t = team, team + TEAMS, ...: r3 = R - t
    const int nmine = (R - team >= 0) ? (R - team) / C::TEAMS + 1 : 0;
    const int nblk = nmine / 2, nrem = nmine - 2 * nblk;
    const int acc0 = FUSE ? (((tid >> 5) % WPT) * C::MAXROWS + (R - team)) * 2 + (lane & 1) : 0;

    for (int quad = q_begin, i = 0; quad < q_end; ++quad, ++i) {
        const int b = i % nbuf, pb = i & 1;
        VT* dst[4];
        uint32_t vw[C::V][4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const size_t slot = 4 * (size_t)quad + s;
            dst[s] = reinterpret_cast<VT*>(M_all + slot * C::MSTRIDE + (size_t)(row0 + R - team) * S::pitch) + grp;
        }
        uint32_t spq[4 * C::V];
#pragma unroll
        for (int k = 0; k < 4 * C::V; ++k) spq[k] = sp[k] + b * bufbytes;
        int* accp = &s_part[FUSE ? pb * PART + acc0 : 0];
        if (staged) mbar_wait(bar0 + 8u * b, (uint32_t)(i / nbuf) & 1u);
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
            for (int j = 0; j < C::V; ++j)
                vw[j][s] = (FUSE && live) ? lds32(vaddr + b * bufbytes + s * C::VSEG + 4 * j) : 0u;

#pragma unroll 1
        for (int blk = 0; blk < nblk; ++blk) {
            staged_row<P, FUSE, 0>(spq, dst, vw, accp, lane);
            staged_row<P, FUSE, 1>(spq, dst, vw, accp, lane);
#pragma unroll
            for (int k = 0; k < 4 * C::V; ++k) spq[k] += 2 * C::TEAMS * 4 * P;
#pragma unroll
            for (int s = 0; s < 4; ++s) dst[s] -= 2 * C::TEAMS * (S::pitch / (4 * C::V));
            accp -= 2 * 2 * C::TEAMS;
        }
        if (nrem > 0) staged_row<P, FUSE, 0>(spq, dst, vw, accp, lane);
        // every read of buffer b is done and s_part[pb] is complete: tell the producer warp, do not wait for it
        asm volatile("bar.arrive 1, %0;" ::"n"(C::NTL) : "memory");
    }
}

// v1 = vacc mod p (row groups cut into several panels)
template <int P>
__global__ void k_vec_finish(const int* __restrict__ vacc, uint8_t* __restrict__ v1, size_t n)
{
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v1[i] = (uint8_t)((uint32_t)vacc[i] % (uint32_t)P);
}
