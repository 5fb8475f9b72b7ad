// qfs_chain.cuh -- stage 4: iterated mod-p matrix-vector chain with per-surface early exit.
//
// Replaces the loop of height_matrix (height.py:135-144) around matvec (modmatrix.py:109-131):
//     for h = 2..bound:  v <- M v (mod p);  iterations += 1;  if v[cap] != 0: height = h, stop.
// The reference accumulates uint64 products in column blocks of 2048 and reduces per block; any
// reduction cadence inside the overflow budget is bit-identical (modmatrix.py:35-49).  Here a row
// dot product is at most N (p-1)^2 <= 12341 * 100 < 2^31, so ONE reduction per row is exact:
// uint8 x uint8 products are summed four at a time with DP4A into a 32-bit accumulator.
//
// Mapping.  Persistent CTAs (1024 threads) pull surfaces from a global queue (early exit makes the work per
// surface vary from 1 to bound-1 passes over M).  The kernel is a latency-bound stream: what matters is the
// number of 16-byte loads in flight per SM (measured, F_5 / F_7 / F_11 stage ms: 512 threads x 4 rows x 2 CTAs
// 1.45 / 6.9 / 13.3; 1024 x 4 x 2 0.81 / 3.65 / 8.6; 1024 x 8 x 1 1.10 / 4.44 / 4.1).  The vector lives in shared memory (ping-pong);
// each warp owns UNROLL rows at a time, lanes stream 16-byte pieces of those rows from HBM with
// non-allocating loads, and a warp-shuffle tree finishes each dot product.
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct ChainCfg {
    using S = Shape<P>;
    static constexpr int NT = 1024;
    static constexpr int UNROLL = (P >= 11) ? 8 : 4;   // rows per warp pass: 16-byte loads in flight per lane
    static constexpr int CTAS_PER_SM = (P >= 11) ? 1 : 2;  // p <= 7: 64 warps per SM (32 registers); p >= 11: few, long surfaces -> more loads per CTA
    static constexpr int SMEM = 2 * S::pitch;
};

__device__ __forceinline__ uint4 ld_stream16(const uint4* p)
{
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// The loop only ever tests v[cap] (height.py:141-143), so the LAST operator application of a surface needs one row of M, not M:
// before streaming the matrix for a step the CTA computes the cap row's dot product with the current vector; if it is nonzero the
// height is decided and the other N - 1 rows of that step are never read.  A surface of height h reads M h - 3 times instead of
// h - 2 (height 3, a fraction 1 - 1/p of what reaches the chain: not at all).  Not taken when a trace of the vectors is asked for.
template <int P, int NT>
__device__ __forceinline__ bool cap_row_hit(const uint8_t* __restrict__ M, const uint8_t* v, uint32_t* s_red)
{
    using S = Shape<P>;
    constexpr int NCHR = (S::N + 15) / 16;
    const uint4* mrow = reinterpret_cast<const uint4*>(M + (size_t)S::cap * S::pitch);
    uint32_t acc = 0;
    for (int ch = threadIdx.x; ch < NCHR; ch += NT) {
        const uint4 m = ld_stream16(mrow + ch);
        const uint4 x = reinterpret_cast<const uint4*>(v)[ch];
        acc = __dp4a(m.x, x.x, acc);
        acc = __dp4a(m.y, x.y, acc);
        acc = __dp4a(m.z, x.z, acc);
        acc = __dp4a(m.w, x.w, acc);
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
    __syncthreads();
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) tot += s_red[w];   // <= N (p-1)^2 < 2^31
    __syncthreads();
    return tot % (uint32_t)P != 0;
}

template <int P>
__global__ void __launch_bounds__(ChainCfg<P>::NT, ChainCfg<P>::CTAS_PER_SM)
k_chain(const uint8_t* __restrict__ M_all, const uint8_t* __restrict__ v0_all, const uint32_t* __restrict__ list,
        int count, int start_it, int max_steps, uint8_t* __restrict__ trace, int8_t* __restrict__ heights,
        int8_t* __restrict__ iters, int* __restrict__ queue)
{
    using S = Shape<P>;
    using C = ChainCfg<P>;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int s_slot;
    __shared__ uint32_t s_red[C::NT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = C::NT / 32;
    constexpr int NCH = S::pitch / 16;
    constexpr int NCHR = (S::N + 15) / 16;   // 16-byte chunks of a row that hold a column: the pad chunks behind them are not read

    while (true) {
        if (tid == 0) s_slot = atomicAdd(queue, 1);
        __syncthreads();
        const int slot = s_slot;
        if (slot >= count) break;
        const uint8_t* M = M_all + (size_t)slot * ((size_t)S::N * S::pitch);
        uint8_t* va = smem;
        uint8_t* vb = smem + S::pitch;
        // start_it = 1: v0_all holds v1 = M g from the fused builder (qfs_matrix.cuh); most surfaces are
        // decided by v1[cap] alone and never touch M here.
        if (start_it > 0 && (v0_all[(size_t)slot * S::pitch + S::cap] != 0 || max_steps <= start_it)) {
            if (tid == 0) {
                const uint32_t sid = list ? list[slot] : (uint32_t)slot;
                heights[sid] = (int8_t)(v0_all[(size_t)slot * S::pitch + S::cap] != 0 ? start_it + 1 : 0);
                iters[sid] = (int8_t)start_it;
            }
            __syncthreads();
            continue;
        }
        {
            const uint4* src = reinterpret_cast<const uint4*>(v0_all + (size_t)slot * S::pitch);
            for (int i = tid; i < NCH; i += C::NT) {
                uint4 x = src[i];
                if (16 * i + 16 > S::N) {  // the pad bytes of v1 (and of M's rows) are never written by the builder: mask every chunk past N
                    uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int b = 0; b < 16; ++b)
                        if (16 * i + b >= S::N) w[b >> 2] &= ~(0xFFu << (8 * (b & 3)));
                    x = make_uint4(w[0], w[1], w[2], w[3]);
                }
                reinterpret_cast<uint4*>(va)[i] = x;
                reinterpret_cast<uint4*>(vb)[i] = make_uint4(0, 0, 0, 0);
            }
        }
        __syncthreads();
        int height = 0, it = start_it;
        for (int step = start_it + 1; step <= max_steps; ++step) {
            if (!trace) {
                const bool hit = cap_row_hit<P, C::NT>(M, va, s_red);
                if (hit || step == max_steps) {   // decided, or the last step allowed: the rest of v_step is never used
                    ++it;
                    if (hit) height = step + 1;
                    break;
                }
            }
            for (int row = warp * C::UNROLL; row < S::N; row += NW * C::UNROLL) {
                uint32_t acc[C::UNROLL];
#pragma unroll
                for (int u = 0; u < C::UNROLL; ++u) acc[u] = 0;
                for (int ch = lane; ch < NCHR; ch += 32) {
                    const uint4 v = reinterpret_cast<const uint4*>(va)[ch];
                    uint4 m[C::UNROLL];
#pragma unroll
                    for (int u = 0; u < C::UNROLL; ++u) {
                        const int rr = (row + u < S::N) ? row + u : S::N - 1;
                        m[u] = ld_stream16(reinterpret_cast<const uint4*>(M + (size_t)rr * S::pitch) + ch);
                    }
#pragma unroll
                    for (int u = 0; u < C::UNROLL; ++u) {
                        acc[u] = __dp4a(m[u].x, v.x, acc[u]);
                        acc[u] = __dp4a(m[u].y, v.y, acc[u]);
                        acc[u] = __dp4a(m[u].z, v.z, acc[u]);
                        acc[u] = __dp4a(m[u].w, v.w, acc[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < C::UNROLL; ++u) {
#pragma unroll
                    for (int o = 16; o; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
                }
                if (lane == 0) {
#pragma unroll
                    for (int u = 0; u < C::UNROLL; ++u)
                        if (row + u < S::N) vb[row + u] = (uint8_t)(acc[u] % (uint32_t)P);
                }
            }
            __syncthreads();
            ++it;
            if (trace) {
                uint8_t* tr = trace + ((size_t)slot * max_steps + (step - 1)) * S::N;
                for (int i = tid; i < S::N; i += C::NT) tr[i] = vb[i];
            }
            { uint8_t* t = va; va = vb; vb = t; }
            const bool hit = va[S::cap] != 0;
            __syncthreads();
            if (hit) { height = step + 1; break; }
        }
        if (tid == 0) {
            const uint32_t sid = list ? list[slot] : (uint32_t)slot;
            heights[sid] = (int8_t)height;
            iters[sid] = (int8_t)it;
        }
    }
}

// ---- the same chain with the WHOLE GRID on one surface at a time ---------------------------------------------
// k_chain gives a surface to one CTA; that is the right shape when thousands of surfaces are pending (p <= 7
// batches), and the wrong one when a chunk holds a few dozen long surfaces (p >= 11: <= 460 matrices of 152 MB
// per chunk, ~1/p of them undecided after the fused first step -- 40 busy CTAs of 148 streamed at 1.0-1.4 TB/s)
// or when the caller asks for one surface (height_matrix of a single quartic).  Here every warp of a cooperative
// grid owns the rows gw, gw + GW, ... of the current surface (GW = warps in the grid), streams each row with
// KCH 16-byte loads in flight per lane, and the new vector goes through a 2 x pitch global scratch (L2) and a
// grid barrier per step.  Same arithmetic, same results; the early exit is taken by all CTAs together.
#include <cooperative_groups.h>

template <int P>
struct ChainGridCfg {
    using S = Shape<P>;
    static constexpr int NT = 1024;
    static constexpr int KCH = 4;            // 16-byte loads in flight per lane
    static constexpr int MAXCOUNT = 4096;    // surfaces per launch (one flag byte each in shared memory)
    static constexpr int SMEM = S::pitch + MAXCOUNT;
};

template <int P>
__global__ void __launch_bounds__(ChainGridCfg<P>::NT, 1)
k_chain_grid(const uint8_t* __restrict__ M_all, const uint8_t* __restrict__ v0_all, const uint32_t* __restrict__ list,
             int count, int start_it, int max_steps, uint8_t* __restrict__ trace, int8_t* __restrict__ heights,
             int8_t* __restrict__ iters, uint8_t* __restrict__ scratch)
{
    namespace cg = cooperative_groups;
    using S = Shape<P>;
    using C = ChainGridCfg<P>;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* sv = smem;                 // the current vector, pad bytes zero
    uint8_t* sflag = smem + S::pitch;   // v0[slot][cap] of every slot of the launch
    __shared__ uint32_t s_red[C::NT / 32];
    const int tid = threadIdx.x, lane = tid & 31;
    // consecutive rows go to different CTAs: every SM streams the same number of rows (+-1)
    const int gw = (tid >> 5) * gridDim.x + blockIdx.x, GW = gridDim.x * (C::NT / 32);
    constexpr int NCH = S::pitch / 16;
    constexpr int NCHR = (S::N + 15) / 16;   // 16-byte chunks of a row that hold a column: the pad chunks behind them are not read

    for (int i = tid; i < count; i += C::NT) sflag[i] = start_it > 0 ? v0_all[(size_t)i * S::pitch + S::cap] : 0;
    __syncthreads();
    int par = 0;
    for (int slot = 0; slot < count; ++slot) {
        const uint32_t sid = list ? list[slot] : (uint32_t)slot;
        if (start_it > 0 && (sflag[slot] != 0 || max_steps <= start_it)) {  // decided by the fused first step
            if (blockIdx.x == 0 && tid == 0) {
                heights[sid] = (int8_t)(sflag[slot] != 0 ? start_it + 1 : 0);
                iters[sid] = (int8_t)start_it;
            }
            continue;
        }
        const uint8_t* M = M_all + (size_t)slot * ((size_t)S::N * S::pitch);
        __syncthreads();  // everyone is done with the previous surface's vector
        {
            const uint4* src = reinterpret_cast<const uint4*>(v0_all + (size_t)slot * S::pitch);
            for (int i = tid; i < NCH; i += C::NT) {
                uint4 x = src[i];
                if (16 * i + 16 > S::N) {  // pad bytes of a vector are never written by its producer: mask them
                    uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int b = 0; b < 16; ++b)
                        if (16 * i + b >= S::N) w[b >> 2] &= ~(0xFFu << (8 * (b & 3)));
                    x = make_uint4(w[0], w[1], w[2], w[3]);
                }
                reinterpret_cast<uint4*>(sv)[i] = x;
            }
        }
        __syncthreads();
        int height = 0, it = start_it;
        for (int step = start_it + 1; step <= max_steps; ++step) {
            if (!trace) {
                // every CTA holds the same vector and takes the same decision: no grid barrier for the test (and none is skipped
                // in a way that matters: a half of the scratch is rewritten only after a barrier that follows its last read)
                const bool hit = cap_row_hit<P, C::NT>(M, sv, s_red);
                if (hit || step == max_steps) {
                    ++it;
                    if (hit) height = step + 1;
                    break;
                }
            }
            uint8_t* nxt = scratch + (size_t)par * S::pitch;
            for (int row = gw; row < S::N; row += GW) {
                const uint4* mrow = reinterpret_cast<const uint4*>(M + (size_t)row * S::pitch);
                uint32_t acc = 0;
                int ch0 = 0;
                for (; ch0 + 32 * C::KCH <= NCHR; ch0 += 32 * C::KCH) {
                    uint4 m[C::KCH];
#pragma unroll
                    for (int k = 0; k < C::KCH; ++k) m[k] = ld_stream16(mrow + ch0 + 32 * k + lane);
#pragma unroll
                    for (int k = 0; k < C::KCH; ++k) {
                        const uint4 v = reinterpret_cast<const uint4*>(sv)[ch0 + 32 * k + lane];
                        acc = __dp4a(m[k].x, v.x, acc);
                        acc = __dp4a(m[k].y, v.y, acc);
                        acc = __dp4a(m[k].z, v.z, acc);
                        acc = __dp4a(m[k].w, v.w, acc);
                    }
                }
                for (int ch = ch0 + lane; ch < NCHR; ch += 32) {
                    const uint4 m = ld_stream16(mrow + ch);
                    const uint4 v = reinterpret_cast<const uint4*>(sv)[ch];
                    acc = __dp4a(m.x, v.x, acc);
                    acc = __dp4a(m.y, v.y, acc);
                    acc = __dp4a(m.z, v.z, acc);
                    acc = __dp4a(m.w, v.w, acc);
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) nxt[row] = (uint8_t)(acc % (uint32_t)P);
            }
            grid.sync();  // the new vector is complete (and everyone has finished reading the old one)
            for (int i = tid; i < NCH; i += C::NT) {
                uint4 x = __ldcg(reinterpret_cast<const uint4*>(nxt) + i);
                if (16 * i + 16 > S::N) {
                    uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int b = 0; b < 16; ++b)
                        if (16 * i + b >= S::N) w[b >> 2] &= ~(0xFFu << (8 * (b & 3)));
                    x = make_uint4(w[0], w[1], w[2], w[3]);
                }
                reinterpret_cast<uint4*>(sv)[i] = x;
            }
            par ^= 1;  // the next step writes the other half: nobody can still be reading it (one barrier ago)
            __syncthreads();
            ++it;
            if (trace && blockIdx.x == 0) {
                uint8_t* tr = trace + ((size_t)slot * max_steps + (step - 1)) * S::N;
                for (int i = tid; i < S::N; i += C::NT) tr[i] = sv[i];
            }
            if (sv[S::cap] != 0) { height = step + 1; break; }
        }
        if (blockIdx.x == 0 && tid == 0) {
            heights[sid] = (int8_t)height;
            iters[sid] = (int8_t)it;
        }
    }
}
