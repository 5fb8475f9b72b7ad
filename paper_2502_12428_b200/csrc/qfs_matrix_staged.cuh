// qfs_matrix_staged.cuh -- stage 3, builder v6: the same gather as qfs_matrix.cuh, but the Delta
// windows of a work item are first staged in shared memory with 16-byte asynchronous copies.
//
// Why.  The v4 builder gathers straight from global memory: a warp-wide LDG.32 touches ~10 cache
// lines (the 128 columns of a warp cross ~20 column runs that live in different Delta runs), and
// the L1 tag stage -- one line per cycle -- caps it at ~3.1 TB/s of matrix writes
// (profiles/r1_ncu_full_*).  Shared memory has no tag stage, only banks: the same access pattern
// costs ~3 wavefronts per request instead of ~10 tag cycles.
//
// What is staged.  For a row group (r1,r2) the sources of the column block c1 (all c2, c3) are the
// Delta runs (I1, I2lo..I2hi), I1 = p r1+p-1-c1, I2 = p r2+p-1-c2: ONE contiguous piece of the
// guard-banded lex43g array (qfs_shape.cuh), because runs are ordered by (I1, I2).  A work item
// ("panel") = (r1, r2, c1lo..c1hi): it stages the pieces of its column blocks (plus the last two
// runs of block c1lo-1, which the first owned word may straddle) and writes the 32-bit words of
// the rows of the group whose LAST column lies in its blocks.  The host cuts every row group into
// panels that fit the shared-memory budget (p = 3, 5: one panel per group).
//
// Fused first step as in v4; with several panels per row the partial dot products are added into
// a 32-bit accumulator array in global memory and k_vec_finish reduces it mod p.
#pragma once
#include <limits.h>

#include "qfs_delta.cuh"  // transpose4x4
#include "qfs_shape.cuh"

struct PanelItem {
    uint8_t r1, r2, c1lo, c1hi;
    uint16_t wlo, nwords;   // owned 32-bit words of a row: [wlo, wlo + nwords)
};

template <int P>
struct StagedCfg {
    using S = Shape<P>;
    static constexpr int WORDS = S::pitch / 4;
    static constexpr int NT = (P >= 5) ? 256 : 64;  // consumer threads (one 32-bit word of a row each)
    static constexpr int NTL = NT + 32;              // launched: + one producer warp (bulk copies, fused-step epilogue)
    static constexpr int WPT = 1;
    static constexpr int MAXW = NT * WPT;                  // most words a panel may own
    static constexpr int MAXROWS = S::d + 1;
    static constexpr int SLICE = (P >= 11) ? 2 : (P >= 7 ? 4 : 16);  // quads per CTA
    static constexpr int UNROLL = 4;
    static constexpr int ZW = (P * S::d + 4 + 3) & ~3;     // zero region (entries) read by columns that never match
    static constexpr int MAXC = S::d + 2;                  // pieces per panel
    static constexpr bool MULTI = (P >= 7);                // several panels per row group -> global accumulators
    static constexpr int BUDGET = (P >= 11) ? 20480 : 12800;  // staged entries (x4 bytes) per panel
    static constexpr size_t MSTRIDE = (size_t)S::N * S::pitch;
};

__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void* src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ uint32_t lds32(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// Fused first step, per warp and row: part[s] = this thread's share of (M g)[row] for surface s (< 2^11).
// Two surfaces are packed per 32-bit word (a warp sum stays < 2^16), two REDUX give the warp sums,
// and lanes 0/1 store them to the warp's own [row][pair] slot: no atomics, no branches.
template <int MAXROWS, int U>
__device__ __forceinline__ void fuse_store(const uint32_t (&part)[4], int* accp, int lane)
{
    const uint32_t t01 = __reduce_add_sync(0xffffffffu, part[0] + (part[1] << 16));
    const uint32_t t23 = __reduce_add_sync(0xffffffffu, part[2] + (part[3] << 16));
    if (lane < 2) accp[-2 * U] = (int)(lane ? t23 : t01);
}

// The piece of Delta that column block c1 of row group (r1,r2) reads, restricted to c2 >= c2min:
// entries [a, b) of the lex43g array (a rounded down, b rounded up to a multiple of 32 entries).  Returns false when no column of the block can match.
template <int P>
QFS_HD bool staged_piece(int r1, int r2, int c1, int c2min, int& a4, int& b4)
{
    using S = Shape<P>;
    const int I1 = P * r1 + P - 1 - c1;
    if (I1 < 0 || I1 > S::D) return false;
    int I2lo = P * r2 + P - 1 - (S::d - c1), I2hi = P * r2 + P - 1 - c2min;
    if (I2lo < 0) I2lo = 0;
    if (I2hi > S::D - I1) I2hi = S::D - I1;
    if (I2lo > I2hi) return false;
    a4 = (S::gbase(I1, I2lo) - S::G) & ~31;      // 32 entries = 128 bytes of the quad-interleaved array: the
    b4 = (S::gbase(I1, I2hi + 1) + 31) & ~31;    // unit of the staging loop (8 lanes x 16 bytes)
    return true;
}

template <int P, bool FUSE, int U>
__device__ __forceinline__ void staged_row(const uint32_t (&sp)[StagedCfg<P>::WPT][4], uint32_t* const (&dst)[StagedCfg<P>::WPT][4],
                                           const uint32_t (&vw)[StagedCfg<P>::WPT][4], int* accp, int lane)
{
    using S = Shape<P>;
    using C = StagedCfg<P>;
    uint32_t part[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < C::WPT; ++j) {
        uint32_t in[4], out[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) in[k] = lds32(sp[j][k] + 4 * P * U);
        transpose4x4(in, out);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            dst[j][s][-U * (S::pitch / 4)] = out[s];  // threads past the panel end repeat its last word
            if (FUSE) part[s] = __dp4a(out[s], vw[j][s], part[s]);
        }
    }
    if (FUSE) fuse_store<C::MAXROWS, U>(part, accp, lane);
}

// ---- bulk asynchronous copies (TMA engine) completing on an mbarrier ---------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src),
                 "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@p bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// items sorted by decreasing work.  vacc: [slot][pitch] int accumulators (MULTI only, zeroed by the caller).
// Dynamic shared memory: two buffers of `bufwords` 32-bit words (one word = one Delta entry of the 4 surfaces
// of a quad), each = [ZW zero words][staged pieces]; quad i of the slice uses buffer i & 1, and the pieces
// of quad i+1 are in flight (bulk copies issued by thread 0) while the rows of quad i are written.
template <int P, bool FUSE>
__global__ void __launch_bounds__(StagedCfg<P>::NTL)
k_matrix_staged(const uint8_t* __restrict__ delta_all, const uint32_t* __restrict__ colinfo,
                const PanelItem* __restrict__ items, uint8_t* __restrict__ M_all, const uint8_t* __restrict__ v0_all,
                uint8_t* __restrict__ v1_all, int* __restrict__ vacc, int count, int bufwords)
{
    using S = Shape<P>;
    using C = StagedCfg<P>;
    constexpr int NW = C::NT / 32;
    extern __shared__ __align__(128) uint32_t sm[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ int s_part[FUSE ? 2 * NW * C::MAXROWS * 2 : 1];  // [parity][warp][r3][surface pair]
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
    const int cfirst = c1lo > 0 ? c1lo - 1 : 0;
    const uint32_t sm_base = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(s_bar);
    const uint32_t bufbytes = 4u * (uint32_t)bufwords;

    if (tid == 0) {
        int so = C::ZW, n = 0;
        for (int c1 = cfirst; c1 <= c1hi; ++c1) {
            int a4, b4, rel = INT_MIN;
            const int c2min = (c1 < c1lo) ? max(0, S::d - c1 - 1) : 0;
            if (staged_piece<P>(r1, r2, c1, c2min, a4, b4)) {
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
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < C::ZW; i += C::NTL) sm[i] = sm[bufwords + i] = 0u;
    __syncthreads();

    if (tid >= C::NT) {
        // ---- producer warp: bulk copies one quad ahead, and the fused-step epilogue one quad behind ----
        const int n = s_ncp;
        uint32_t total = 0;
        for (int ci = 0; ci < n; ++ci) total += (uint32_t)s_cpn[ci];
        auto issue = [&](int quad, int b) {
            if (n == 0) return;
            const uint32_t bar = bar0 + 8u * b;
            const uint8_t* dq = delta_all + (size_t)quad * S::quad_stride;
            if (lane == 0) mbar_expect_tx(bar, total);
            __syncwarp();
            for (int ci = lane; ci < n; ci += 32)
                bulk_g2s(sm_base + b * bufbytes + (uint32_t)s_cps[ci], dq + 4 * (size_t)s_cpa[ci], (uint32_t)s_cpn[ci], bar);
        };
        auto epilogue = [&](int quad, int b) {
            for (int e = lane; e < 4 * (R + 1); e += 32) {
                const int s = e / (R + 1), r3 = e - s * (R + 1);
                const int* pp = &s_part[b * (NW * C::MAXROWS * 2) + r3 * 2 + (s >> 1)];
                uint32_t a = 0;
#pragma unroll
                for (int w = 0; w < NW; ++w) a += ((uint32_t)pp[w * C::MAXROWS * 2] >> (16 * (s & 1))) & 0xffffu;
                const size_t o = (4 * (size_t)quad + s) * S::pitch + row0 + r3;
                if (C::MULTI) atomicAdd(vacc + o, (int)a);
                else v1_all[o] = (uint8_t)(a % (uint32_t)P);
            }
        };
        if (q_begin < q_end) issue(q_begin, 0);
        for (int quad = q_begin, i = 0; quad < q_end; ++quad, ++i) {
            // the consumers are past the rows of quad i-1 (barrier below): buffer (i+1)&1 and s_part[(i-1)&1] are settled
            if (quad + 1 < q_end) issue(quad + 1, (i + 1) & 1);
            if (FUSE && i > 0) epilogue(quad - 1, (i - 1) & 1);
            __syncthreads();
        }
        if (FUSE && q_begin < q_end) epilogue(q_end - 1, (q_end - 1 - q_begin) & 1);
        return;
    }

    uint32_t sp[C::WPT][4];
    int wj[C::WPT];
#pragma unroll
    for (int j = 0; j < C::WPT; ++j) {
        const int w = it.wlo + min(tid + j * C::NT, (int)it.nwords - 1);
        wj[j] = w;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int idx = 0;
            const uint32_t info = colinfo[4 * w + k];
            if (info != 0xFFFFFFFFu) {
                const int c1 = info & 255, c2 = (info >> 8) & 255, c3 = info >> 16;
                const int I1 = P * r1 + P - 1 - c1, I2 = P * r2 + P - 1 - c2;
                if (I1 >= 0 && I2 >= 0 && I1 + I2 <= S::D)
                    idx = s_rel[c1 - cfirst] + S::gbase(I1, I2) + (P - 1) - (S::d - c1 - c2) + c3;
            }
            sp[j][k] = sm_base + 4u * (uint32_t)idx;
        }
    }
    const bool staged = s_ncp > 0;
    const int nblk = (R + 1) / C::UNROLL, nrem = (R + 1) - nblk * C::UNROLL;
    const int acc0 = FUSE ? ((tid >> 5) * C::MAXROWS + R) * 2 + (lane & 1) : 0;

    for (int quad = q_begin, i = 0; quad < q_end; ++quad, ++i) {
        const int b = i & 1;
        uint32_t* dst[C::WPT][4];
        uint32_t vw[C::WPT][4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const size_t slot = 4 * (size_t)quad + s;
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
                dst[j][s] = reinterpret_cast<uint32_t*>(M_all + slot * C::MSTRIDE + (size_t)(row0 + R) * S::pitch) + wj[j];
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
                vw[j][s] = (FUSE && tid + j * C::NT < (int)it.nwords) ? reinterpret_cast<const uint32_t*>(v0_all + slot * S::pitch)[wj[j]] : 0u;
        }
        uint32_t spq[C::WPT][4];
#pragma unroll
        for (int j = 0; j < C::WPT; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) spq[j][k] = sp[j][k] + b * bufbytes;
        int* accp = &s_part[FUSE ? b * (NW * C::MAXROWS * 2) + acc0 : 0];
        if (staged) mbar_wait(bar0 + 8u * b, (uint32_t)(i >> 1) & 1u);

#pragma unroll 1
        for (int blk = 0; blk < nblk; ++blk) {
            staged_row<P, FUSE, 0>(spq, dst, vw, accp, lane);
            staged_row<P, FUSE, 1>(spq, dst, vw, accp, lane);
            staged_row<P, FUSE, 2>(spq, dst, vw, accp, lane);
            staged_row<P, FUSE, 3>(spq, dst, vw, accp, lane);
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) spq[j][k] += C::UNROLL * 4 * P;
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                for (int s = 0; s < 4; ++s) dst[j][s] -= C::UNROLL * (S::pitch / 4);
            accp -= 2 * C::UNROLL;
        }
        if (nrem > 0) staged_row<P, FUSE, 0>(spq, dst, vw, accp, lane);
        if (nrem > 1) staged_row<P, FUSE, 1>(spq, dst, vw, accp, lane);
        if (nrem > 2) staged_row<P, FUSE, 2>(spq, dst, vw, accp, lane);
        __syncthreads();  // every read of buffer b is done and s_part[b] is complete: over to the producer warp
    }
}

// v1 = vacc mod p (MULTI builds only)
template <int P>
__global__ void k_vec_finish(const int* __restrict__ vacc, uint8_t* __restrict__ v1, size_t n)
{
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v1[i] = (uint8_t)((uint32_t)vacc[i] % (uint32_t)P);
}
