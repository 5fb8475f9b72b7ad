// qfs_lib.cu -- host side of libqfs.so: context, workspaces, the chunked pipeline and the C ABI
// declared in include/qfs.h.  One context drives one GPU; surfaces are independent, so multi-GPU
// runs are N contexts over disjoint blocks of the batch with no collective.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/qfs.h"
#include "qfs_caprow.cuh"
#include "qfs_chain.cuh"
#include "qfs_cubic.cuh"
#include "qfs_delta.cuh"
#include "qfs_delta_direct.cuh"
#include "qfs_delta_mma.cuh"
#include "qfs_form.cuh"
#include "qfs_literal.cuh"
#include "qfs_free.cuh"
#include "qfs_matrix.cuh"
#include "qfs_matrix_staged.cuh"
#include "qfs_power.cuh"
#include "qfs_sample.cuh"
#include "qfs_shape.cuh"

namespace {

thread_local std::string g_create_error;   // errors of the context-free entries (qfs_create, qfs_cubic_heights), per calling thread

struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    cudaError_t reserve(size_t bytes)
    {
        if (bytes <= cap) return cudaSuccess;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&ptr, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release()
    {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(ptr); }
};

enum { EV_COUNT = 8 };

// Every entry point runs on its context's device and leaves the caller's current device as it found it.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

struct qfs_ctx {
    int p = 0;
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[EV_COUNT] = {};
    cudaEvent_t ev_total[2] = {};
    std::vector<cudaEvent_t> chunk_ev;              // five per chunk of a call: stage boundaries, read after the call's last sync
    size_t workspace_limit = 0;
    size_t auto_limit = 0;                          // default workspace budget, fixed at first use
    size_t chunk_override = 0;
    int chain_grid_mode = -1;   // QFS_CHAIN_GRID: -1 automatic, 0 never, 1 always (k_chain_grid vs k_chain)
    int chain_grid_ctas = 0;
    int delta_wave = 0;         // CTAs of k_delta resident at a time (0: the direct kernel is used)
    std::string error;
    qfs_stats stats = {};
    // device state
    DevBuf flags;                                   // int err, int queue, int count (+ pad)
    DevBuf colinfo, groups, runs;                   // per-p index tables for the matrix builder
    DevBuf unrank;                                  // per-p unrank tables for the power chain
    DevBuf coeffs, heights, iters, list;            // batch-sized
    DevBuf compact_counts;                          // pending surfaces per tile of the batch (launch_compact)
    DevBuf slotmap;                                 // lazy mode: slot of a pending surface in the cap-row pass (k_gather_rows)
    DevBuf g, h, A, E, delta, M, v1;                // chunk-sized
    DevBuf chain_scratch;                           // 2 x pitch: the vector exchange of k_chain_grid
    DevBuf tapA, tapB;                              // staging for the stage taps
    DevBuf items, vacc;                             // staged matrix builder: panel work list, 32-bit v1 accumulators
    int n_items = 0;
    size_t staged_smem = 0;
    int staged_bufwords = 0;
    int staged_nbuf = 1;
    int occ[4] = {0, 0, 0, 0};   // resident CTAs per SM: k_power_full, k_delta_mma, k_matrix_staged (fused), k_chain
    int staged_multi = 0;
    int delta_direct = 0;                           // QFS_DELTA_DIRECT: use k_delta_direct for every prime (cross-check)
    int delta_version = 2;                          // QFS_DELTA_V: 2 = tensor-core kernel (k_delta_mma), 1 = DP4A slab kernel (k_delta)
    DevBuf ecm, hbox, dphases, dpieces, dparts;     // k_delta_mma: class-major coefficient tables and interleaved h boxes (chunk-sized), phase plan
    DevBuf dphases_few, dparts_few;                 // the same plan cut into SPLIT_FEW parts per quad (launches of at most four quads)
    DevBuf dphases_mid, dparts_mid;                 // ... and into SPLIT_MID parts (fewer quads than CTA slots)
    int matrix_version = 6;                         // 6 = shared-memory staged builder, 4 = direct gather (QFS_MATRIX_V)
    int* h_flags = nullptr;                         // pinned mirror of flags
};

namespace {

int fail(qfs_ctx* ctx, int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->error = buf; else g_create_error = buf;
    return code;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? QFS_ENOMEM : QFS_ECUDA, "%s: %s",  \
                        #call, cudaGetErrorString(e_));                                            \
    } while (0)

bool is_device_ptr(const void* p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Ordered stream compaction of {i : heights[i] < 0} in two launches over tiles of the batch: k_compact_count leaves the number of
// pending surfaces of every tile, k_compact_scatter sums the counts in front of its tile and writes the tile's indices in order
// (round 1 walked the batch with ONE 1024-thread CTA: ~40 us per 100 000 surfaces, twice per call in the lazy mode).
enum { COMPACT_NT = 1024, COMPACT_MAXTILES = 2048 };

__global__ void __launch_bounds__(COMPACT_NT) k_compact_count(const int8_t* __restrict__ heights, int B, int tile, int* __restrict__ counts)
{
    __shared__ int s_warp[32];
    const int tid = threadIdx.x;
    const long long start = (long long)blockIdx.x * tile;
    const int end = (int)min((long long)B, start + tile);
    int n = 0;
    for (int i = (int)start + tid; i < end; i += COMPACT_NT) n += heights[i] < 0;
    n = __reduce_add_sync(0xffffffffu, n);
    if ((tid & 31) == 0) s_warp[tid >> 5] = n;
    __syncthreads();
    if (tid < 32) {
        n = __reduce_add_sync(0xffffffffu, s_warp[tid]);
        if (tid == 0) counts[blockIdx.x] = n;
    }
}

__global__ void __launch_bounds__(COMPACT_NT) k_compact_scatter(const int8_t* __restrict__ heights, int B, int tile,
                                                                const int* __restrict__ counts, uint32_t* __restrict__ list,
                                                                int* __restrict__ count)
{
    __shared__ int s_warp[32];
    __shared__ int s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    {   // pending surfaces in front of this tile
        int part = 0;
        for (int j = tid; j < (int)blockIdx.x; j += COMPACT_NT) part += counts[j];
        part = __reduce_add_sync(0xffffffffu, part);
        if (lane == 0) s_warp[warp] = part;
        __syncthreads();
        if (warp == 0) {
            part = __reduce_add_sync(0xffffffffu, s_warp[lane]);
            if (lane == 0) s_base = part;
        }
        __syncthreads();
    }
    const long long start0 = (long long)blockIdx.x * tile;
    const int end = (int)min((long long)B, start0 + tile);
    for (int start = (int)start0; start < end; start += COMPACT_NT) {
        const int i = start + tid;
        const bool f = (i < end) && heights[i] < 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        const int pre = __popc(bal & ((1u << lane) - 1));
        if (lane == 0) s_warp[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
            int v = s_warp[lane];
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += t;
            }
            s_warp[lane] = v;  // inclusive
        }
        __syncthreads();
        const int wbase = warp ? s_warp[warp - 1] : 0;
        if (f) list[s_base + wbase + pre] = (uint32_t)i;
        __syncthreads();
        if (tid == 0) s_base += s_warp[31];
        __syncthreads();
    }
    if (tid == 0 && blockIdx.x == gridDim.x - 1) *count = s_base;
}

// M (uint8, row pitch `pitch`) -> the reference's entry block: uint16 little-endian, row-major n x n
// (mtsmatrix.py:350-365 matrix_to_bytes, MtsMatrix.entries is uint16, mtsmatrix.py:96)
__global__ void k_widen_u16(const uint8_t* __restrict__ M, int n, int pitch, uint16_t* __restrict__ out)
{
    const int r = blockIdx.x;
    const uint8_t* src = M + (size_t)blockIdx.y * n * pitch + (size_t)r * pitch;
    uint16_t* dst = out + ((size_t)blockIdx.y * n + r) * n;
    for (int c = threadIdx.x; c < n; c += blockDim.x) dst[c] = src[c];
}

// total number of operator applications of a call (stats.matvec_steps), also when the outputs stay on the device
__global__ void __launch_bounds__(1024) k_sum_iters(const int8_t* __restrict__ iters, size_t B, int* __restrict__ total)
{
    int s = 0;
    for (size_t i = (size_t)blockIdx.x * 1024 + threadIdx.x; i < B; i += (size_t)gridDim.x * 1024) s += iters[i];
    s = __reduce_add_sync(0xffffffffu, s);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(total, s);
}

// heights[i] == -1 (pending) -> 0 (infinity); used when bound < 2 (height.py:126-127)
__global__ void k_pending_to_inf(int8_t* heights, int B)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < B && heights[i] < 0) heights[i] = 0;
}

template <int P>
int build_tables(qfs_ctx* ctx)
{
    using S = Shape<P>;
    std::vector<uint32_t> col(S::pitch, 0xFFFFFFFFu);
    std::vector<uint16_t> grp(S::ngroups);
    int c = 0, gidx = 0;
    for (int c1 = 0; c1 <= S::d; ++c1)
        for (int c2 = 0; c1 + c2 <= S::d; ++c2) {
            grp[gidx++] = (uint16_t)(c1 | (c2 << 8));
            for (int c3 = 0; c1 + c2 + c3 <= S::d; ++c3) col[c++] = (uint32_t)c1 | ((uint32_t)c2 << 8) | ((uint32_t)c3 << 16);
        }
    if (c != S::N || gidx != S::ngroups) return fail(ctx, QFS_EINVAL, "internal: basis enumeration mismatch");
    const std::vector<uint16_t> runs_lex = grp;  // column runs (c1,c2) in lex order
    // longest row groups first: the builder's CTAs then finish together
    std::stable_sort(grp.begin(), grp.end(), [](uint16_t a, uint16_t b) { return (a & 255) + (a >> 8) < (b & 255) + (b >> 8); });
    CU(ctx->colinfo.reserve(col.size() * 4));
    CU(ctx->groups.reserve(grp.size() * 2));
    CU(ctx->runs.reserve(grp.size() * 2));
    CU(cudaMemcpy(ctx->runs.ptr, runs_lex.data(), runs_lex.size() * 2, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->colinfo.ptr, col.data(), col.size() * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->groups.ptr, grp.data(), grp.size() * 2, cudaMemcpyHostToDevice));
    {
        std::vector<uint32_t> un;
        for (int k = 1; k <= P; ++k) {
            const int deg = 4 * k;
            if ((int)un.size() != qunrank_offset(k)) return fail(ctx, QFS_EINVAL, "internal: unrank offset mismatch");
            for (int a1 = 0; a1 <= deg; ++a1)
                for (int a2 = 0; a1 + a2 <= deg; ++a2)
                    for (int a3 = 0; a1 + a2 + a3 <= deg; ++a3) un.push_back((uint32_t)a1 | ((uint32_t)a2 << 8) | ((uint32_t)a3 << 16));
        }
        CU(ctx->unrank.reserve(un.size() * 4));
        CU(cudaMemcpy(ctx->unrank.ptr, un.data(), un.size() * 4, cudaMemcpyHostToDevice));
    }
    {   // panels of the staged matrix builder (qfs_matrix_staged.cuh)
        using SC = StagedCfg<P>;
        int budget = SC::BUDGET;
        if (const char* e = getenv("QFS_STAGED_BUDGET")) budget = std::max(SC::BUDGET / 8, atoi(e));
        struct Tmp { PanelItem it; long work; int staged; };
        std::vector<Tmp> tmp;
        int max_staged = 0;
        // A panel = word groups [ga, gb) of the rows of one row group; ga and gb are multiples of LINEG (whole
        // 128-byte lines) except at the row end.  Its columns [first, last] run from (c1lo, c2lo, .) to (c1hi, c2hi, .).
        constexpr int CPG = 4 * SC::V;  // columns per word group
        for (int r1 = 0; r1 <= S::d; ++r1)
            for (int r2 = 0; r1 + r2 <= S::d; ++r2) {
                auto make = [&](int ga, int gb, PanelItem& it) {  // returns the staged entries of the panel, -1 if it has no column
                    const int first = CPG * ga, last = std::min(CPG * gb, S::N) - 1;
                    if (first > last) return -1;
                    const int c1lo = (int)(col[first] & 255), c2lo = (int)((col[first] >> 8) & 255);
                    const int c1hi = (int)(col[last] & 255), c2hi = (int)((col[last] >> 8) & 255);
                    int st = 0;
                    for (int c1 = c1lo; c1 <= c1hi; ++c1) {
                        int a4, b4;
                        if (staged_piece<P>(r1, r2, c1, c1 == c1lo ? c2lo : 0, c1 == c1hi ? c2hi : S::d - c1, a4, b4)) st += b4 - a4;
                    }
                    it = PanelItem{(uint8_t)r1, (uint8_t)r2, (uint8_t)c1lo, (uint8_t)c1hi, (uint16_t)ga, (uint16_t)(gb - ga),
                                   (uint8_t)c2lo, (uint8_t)c2hi, 0};
                    return st;
                };
                const int gend = (S::N + CPG - 1) / CPG;  // word groups that hold a column; the pad groups go with the last panel
                int ga = 0;
                while (ga < gend) {
                    PanelItem it{}, best{};
                    int best_st = -1, gb = ga;
                    // the rows are written up to the end of the 32-byte sector that holds the last column; the pad columns beyond it
                    // (pitch = N rounded up to 128) stay unwritten: nothing reads them (k_chain / k_chain_grid mask the vector's pad
                    // and stop at that sector, the taps and exports copy N columns)
                    constexpr int NGRPW = ((S::N + 31) / 32 * 32) / CPG;
                    while (gb < NGRPW) {
                        int nb = std::min(NGRPW, gb + SC::LINEG);
                        if (nb >= gend) nb = NGRPW;
                        if (nb - ga > SC::MAXG) break;
                        const int st = make(ga, nb, it);
                        if (st > budget && best_st >= 0) break;
                        if (st > budget) return fail(ctx, QFS_EINVAL, "internal: panel does not fit the shared-memory budget");
                        best = it; best_st = st; gb = nb;
                    }
                    if (best_st < 0) return fail(ctx, QFS_EINVAL, "internal: panel does not fit the shared-memory budget");
                    tmp.push_back({best, (long)best.ngrp * (S::d - r1 - r2 + 1), best_st});
                    max_staged = std::max(max_staged, best_st);
                    ga = gb;
                }
            }
        // Launch order = memory order of the rows (r1, r2 lexicographic, panels of a group adjacent): CTAs that
        // run at the same time write neighbouring rows, so their segments reach HBM together (measured: F_7
        // 38.1 -> 33.9 ms against a sort by decreasing work), and the grid ends with the short row groups.
        {
            // ... in T1 x T2 blocks of (r1, r2) where Delta does not fit L2 (p >= 11): a slab of Delta serves ~ (d+1)/p consecutive
            // values of r1 (and of r2), and in plain lexicographic order a whole sweep over r2 lies between two of them, so the staged
            // pieces are re-read from DRAM 3.5 x (F_11).  Measured (profiles/sweeps/r2_builder_experiments.txt): F_11 65.4 -> 62.4 ms
            // per 20 000 surfaces with blocks of four r2, F_13 17.5 -> 17.0 ms with blocks of two r1; F_5 / F_7 are best unblocked.
            int t1 = SC::ORDER_T1, t2 = SC::ORDER_T2;
            if (const char* e = getenv("QFS_PANEL_ORDER")) {
                if (sscanf(e, "%d,%d", &t1, &t2) != 2 || t1 < 1 || t2 < 1) { t1 = SC::ORDER_T1; t2 = SC::ORDER_T2; }
            }
            if (t1 > 1 || t2 > 1)
                std::stable_sort(tmp.begin(), tmp.end(), [&](const Tmp& a, const Tmp& b) {
                    const int ka[4] = {a.it.r1 / t1, a.it.r2 / t2, a.it.r1 % t1, a.it.r2 % t2};
                    const int kb[4] = {b.it.r1 / t1, b.it.r2 / t2, b.it.r1 % t1, b.it.r2 % t2};
                    return std::lexicographical_compare(ka, ka + 4, kb, kb + 4);
                });
        }
        std::vector<PanelItem> items(tmp.size());
        for (size_t i = 0; i < tmp.size(); ++i) items[i] = tmp[i].it;
        ctx->staged_multi = ((int)items.size() != S::ngroups);
        ctx->n_items = (int)items.size();
        ctx->staged_bufwords = SC::ZW + max_staged + SC::VWORDS;
        if (getenv("QFS_VERBOSE")) {
            long st = 0;
            for (auto& t : tmp) st += t.staged;
            fprintf(stderr, "qfs: p=%d builder panels %zu, staged entries per quad %ld (x4 bytes = %.2f x the 4 N^2 bytes written), largest %d\n", P,
                    tmp.size(), st, (double)st / ((double)S::N * S::N), max_staged);
        }
        // One staging buffer per CTA: with the arrive/sync split of k_matrix_staged a consumer must not be able to
        // run a quad ahead of the producer warp (more buffers would need one barrier per buffer).
        ctx->staged_smem = ctx->staged_nbuf * (size_t)ctx->staged_bufwords * 4;
        CU(ctx->items.reserve(items.size() * sizeof(PanelItem)));
        CU(cudaMemcpy(ctx->items.ptr, items.data(), items.size() * sizeof(PanelItem), cudaMemcpyHostToDevice));
        CU(cudaFuncSetAttribute(k_matrix_staged<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->staged_smem));
        CU(cudaFuncSetAttribute(k_matrix_staged<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ctx->staged_smem));
        if (const char* e = getenv("QFS_MATRIX_V")) ctx->matrix_version = atoi(e);
    }
    CU(cudaFuncSetAttribute(k_fedder<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, PowerCfg<P>::FED_SMEM));
    CU(cudaFuncSetAttribute(k_power_full<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, PowerCfg<P>::FULL_SMEM));
    if constexpr (DeltaCfg<P>::SMEM <= 227 * 1024)
        CU(cudaFuncSetAttribute(k_delta<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, DeltaCfg<P>::SMEM));
    CU(cudaFuncSetAttribute(k_delta_direct<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, DeltaDirectCfg<P>::SMEM));
    CU(cudaFuncSetAttribute(k_free<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, FreeCfg<P>::SMEM));
    CU(cudaFuncSetAttribute(k_caprow<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, CapRowCfg<P>::SMEM));
    ctx->delta_direct = getenv("QFS_DELTA_DIRECT") ? 1 : 0;
    if (const char* e = getenv("QFS_DELTA_V")) ctx->delta_version = atoi(e);
    {   // phase plan of the tensor-core Witt carry (qfs_delta_mma.cuh)
        static_assert(DeltaMmaCfg<P>::SMEM <= 227 * 1024, "k_delta_mma: shared memory");
        DeltaPlan plan;
        if (!delta_plan<P>(plan)) return fail(ctx, QFS_EINVAL, "internal: Witt-carry plan does not fit its buffers");
        CU(ctx->dphases.reserve(plan.phases.size() * sizeof(DeltaPhase)));
        CU(ctx->dpieces.reserve(plan.pieces.size() * sizeof(DeltaPiece)));
        CU(ctx->dparts.reserve(plan.parts.size() * sizeof(uint32_t)));
        CU(cudaMemcpy(ctx->dphases.ptr, plan.phases.data(), plan.phases.size() * sizeof(DeltaPhase), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->dpieces.ptr, plan.pieces.data(), plan.pieces.size() * sizeof(DeltaPiece), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->dparts.ptr, plan.parts.data(), plan.parts.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
        DeltaPlan few;   // same phases and pieces, more parts (the block / prefetch flags of a phase depend on its part)
        if (!delta_plan<P>(few, DeltaMmaCfg<P>::SPLIT_FEW)) return fail(ctx, QFS_EINVAL, "internal: Witt-carry plan does not fit its buffers");
        CU(ctx->dphases_few.reserve(few.phases.size() * sizeof(DeltaPhase)));
        CU(ctx->dparts_few.reserve(few.parts.size() * sizeof(uint32_t)));
        CU(cudaMemcpy(ctx->dphases_few.ptr, few.phases.data(), few.phases.size() * sizeof(DeltaPhase), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->dparts_few.ptr, few.parts.data(), few.parts.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
        DeltaPlan mid;
        if (!delta_plan<P>(mid, DeltaMmaCfg<P>::SPLIT_MID)) return fail(ctx, QFS_EINVAL, "internal: Witt-carry plan does not fit its buffers");
        CU(ctx->dphases_mid.reserve(mid.phases.size() * sizeof(DeltaPhase)));
        CU(ctx->dparts_mid.reserve(mid.parts.size() * sizeof(uint32_t)));
        CU(cudaMemcpy(ctx->dphases_mid.ptr, mid.phases.data(), mid.phases.size() * sizeof(DeltaPhase), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->dparts_mid.ptr, mid.parts.data(), mid.parts.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
        CU(cudaFuncSetAttribute(k_delta_mma<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, DeltaMmaCfg<P>::SMEM));
        CU(cudaFuncSetAttribute(k_delta_box<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * Shape<P>::Nh_pad));
    }
    if constexpr (DeltaCfg<P>::SMEM <= 227 * 1024) {
        // resident 4-CTA clusters (a GPC whose SM count is not a multiple of what a cluster needs leaves SMs idle)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(4 * 1024);
        cfg.blockDim = dim3(DeltaCfg<P>::NT);
        cfg.dynamicSmemBytes = DeltaCfg<P>::SMEM;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 4;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, k_delta<P>, &cfg) != cudaSuccess) { cudaGetLastError(); clusters = 0; }
        ctx->delta_wave = 4 * clusters;
        if (getenv("QFS_VERBOSE")) fprintf(stderr, "qfs: p=%d resident k_delta clusters %d (%d SMs)\n", P, clusters, ctx->sm_count);
    }
    if (const char* e = getenv("QFS_CHAIN_GRID")) ctx->chain_grid_mode = atoi(e);
    CU(cudaFuncSetAttribute(k_chain<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, ChainCfg<P>::SMEM));
    // resident CTAs per SM of the four stage kernels as built and configured (qfs_debug_occupancy): a few bytes of shared memory
    // or a few registers too many silently cost a CTA per SM (k_delta_mma<7> ran on three instead of four for half a round)
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->occ[0], k_power_full<P>, PowerCfg<P>::FULL_NT, PowerCfg<P>::FULL_SMEM));
    ctx->occ[1] = 0;
    if constexpr (P >= 3 && DeltaMmaCfg<P>::SMEM <= 227 * 1024)
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->occ[1], k_delta_mma<P>, DeltaMmaCfg<P>::NT, DeltaMmaCfg<P>::SMEM));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->occ[2], k_matrix_staged<P, true>, StagedCfg<P>::NTL, ctx->staged_smem));
    CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctx->occ[3], k_chain<P>, ChainCfg<P>::NT, ChainCfg<P>::SMEM));
    if (getenv("QFS_VERBOSE"))
        fprintf(stderr, "qfs: p=%d CTAs per SM: k_power_full %d, k_delta_mma %d, k_matrix_staged %d, k_chain %d\n", P, ctx->occ[0], ctx->occ[1],
                ctx->occ[2], ctx->occ[3]);
    return QFS_OK;
}

template <int P>
size_t per_surface_bytes()
{
    using S = Shape<P>;
    return (size_t)S::N * S::pitch + S::Lg_pad + 3 * (size_t)S::pitch + S::Nh_pad + S::NE_pad + DeltaMmaCfg<P>::EC_STRIDE + DeltaMmaCfg<P>::HBOX_WORDS;
}

template <int P>
int reserve_chunk(qfs_ctx* ctx, size_t cap)
{
    using S = Shape<P>;
    cap = (cap + 3) & ~(size_t)3;  // whole quads: the Witt carry and the matrix builder work on four surfaces at a time
    CU(ctx->g.reserve(cap * S::pitch));
    CU(ctx->A.reserve(cap * S::pitch));
    CU(ctx->h.reserve(cap * S::Nh_pad));
    CU(ctx->E.reserve(cap * S::NE_pad));
    CU(ctx->delta.reserve(cap * (size_t)S::Lg_pad));
    CU(ctx->ecm.reserve(cap * (size_t)DeltaMmaCfg<P>::EC_STRIDE));
    CU(ctx->hbox.reserve(cap * DeltaMmaCfg<P>::HBOX_WORDS));
    CU(ctx->M.reserve(cap * (size_t)S::N * S::pitch));
    CU(ctx->v1.reserve(cap * S::pitch));
    return QFS_OK;
}

template <int P>
int reserve_chunk_free(qfs_ctx* ctx, size_t cap)
{
    using S = Shape<P>;
    cap = (cap + 3) & ~(size_t)3;
    CU(ctx->g.reserve(cap * S::pitch));
    CU(ctx->A.reserve(cap * S::pitch));
    CU(ctx->h.reserve(cap * S::Nh_pad));
    CU(ctx->E.reserve(cap * S::NE_pad));
    return QFS_OK;
}

// ---- stage launchers (all on ctx->stream) ---------------------------------------------------
template <int P>
int launch_power_full(qfs_ctx* ctx, const uint8_t* d_coeffs, const uint32_t* d_list, int count, uint8_t* fedder)
{
    int* d_err = ctx->flags.as<int>();
    k_power_full<P><<<count, PowerCfg<P>::FULL_NT, PowerCfg<P>::FULL_SMEM, ctx->stream>>>(
        d_coeffs, d_list, count, ctx->unrank.as<uint32_t>(), fedder, ctx->g.as<uint8_t>(), ctx->h.as<uint8_t>(),
        ctx->A.as<uint8_t>(), ctx->E.as<uint8_t>(), d_err);
    ctx->stats.kernel_launches++;
    CU(cudaGetLastError());
    return QFS_OK;
}

template <int P>
int launch_delta(qfs_ctx* ctx, int count)
{
    using S = Shape<P>;
    if (ctx->delta_version == 2 && !ctx->delta_direct) {
        // tensor-core kernel: class-major coefficient tables, then one CTA per (quad, part of the phase plan)
        using DM = DeltaMmaCfg<P>;
        const unsigned quads = (unsigned)((count + 3) / 4);
        CU(ctx->ecm.reserve((size_t)count * DM::EC_STRIDE));
        CU(ctx->hbox.reserve((size_t)quads * DM::HBOX_WORDS * 4));
        k_delta_prep<P><<<(unsigned)count, 128, S::NE_pad, ctx->stream>>>(ctx->E.as<uint8_t>(), ctx->ecm.as<uint8_t>(), count);
        k_delta_box<P><<<quads, 256, 4 * S::Nh_pad, ctx->stream>>>(ctx->h.as<uint8_t>(), ctx->A.as<uint8_t>(), ctx->ecm.as<uint8_t>(),
                                                                  ctx->unrank.as<uint32_t>() + qunrank_offset(P - 1),
                                                                  ctx->hbox.as<uint32_t>(), count);
        ctx->stats.kernel_launches += 2;
        CU(cudaGetLastError());
        // few quads (single surfaces, small batches): more CTAs per quad, so that the launch still covers the SMs
        const int level = ((int)quads <= 4 && DM::SPLIT < DM::SPLIT_FEW) ? 2 : (((int)quads * DM::MINB < ctx->sm_count && DM::SPLIT < DM::SPLIT_MID) ? 1 : 0);
        const int split = level == 2 ? DM::SPLIT_FEW : (level == 1 ? DM::SPLIT_MID : DM::SPLIT);
        const DevBuf& ph = level == 2 ? ctx->dphases_few : (level == 1 ? ctx->dphases_mid : ctx->dphases);
        const DevBuf& pt = level == 2 ? ctx->dparts_few : (level == 1 ? ctx->dparts_mid : ctx->dparts);
        k_delta_mma<P><<<quads * split, DM::NT, DM::SMEM, ctx->stream>>>(ctx->hbox.as<uint32_t>(), ctx->ecm.as<uint8_t>(), ph.as<DeltaPhase>(),
                                                                         ctx->dpieces.as<DeltaPiece>(), pt.as<uint32_t>(), ctx->delta.as<uint8_t>(),
                                                                         count, split);
        ctx->stats.kernel_launches++;
        CU(cudaGetLastError());
        return QFS_OK;
    }
    if (DeltaCfg<P>::SMEM > 227 * 1024 || ctx->delta_direct) {
        // the slab of k_delta does not fit (p = 13), or QFS_DELTA_DIRECT asks for the cross-check kernel
        const size_t quads = ((size_t)count + 3) / 4;
        CU(cudaMemsetAsync(ctx->delta.ptr, 0, quads * S::quad_stride, ctx->stream));
        const dim3 grid(DeltaDirectCfg<P>::NBLK, (unsigned)count);
        k_delta_direct<P><<<grid, DeltaDirectCfg<P>::NT, DeltaDirectCfg<P>::SMEM, ctx->stream>>>(
            ctx->h.as<uint8_t>(), ctx->A.as<uint8_t>(), ctx->E.as<uint8_t>(), ctx->unrank.as<uint32_t>() + qunrank_offset(P - 1),
            ctx->delta.as<uint8_t>(), count);
        ctx->stats.kernel_launches++;
        CU(cudaGetLastError());
        return QFS_OK;
    }
    if constexpr (DeltaCfg<P>::SMEM <= 227 * 1024) {
        k_delta<P><<<4 * ((count + 3) / 4), DeltaCfg<P>::NT, DeltaCfg<P>::SMEM, ctx->stream>>>(ctx->h.as<uint8_t>(), ctx->A.as<uint8_t>(),
                                                                              ctx->E.as<uint8_t>(), ctx->delta.as<uint8_t>(), count);
        ctx->stats.kernel_launches++;
        CU(cudaGetLastError());
    }
    return QFS_OK;
}

template <int P>
int launch_matrix(qfs_ctx* ctx, int count, const uint8_t* v0, uint8_t* v1)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    const int nquads = (count + 3) / 4;
    if (ctx->matrix_version == 6) {
        using SC = StagedCfg<P>;
        const dim3 sgrid((unsigned)ctx->n_items, (unsigned)((nquads + SC::SLICE - 1) / SC::SLICE));
        if (v0) {
            const size_t nv = 4 * (size_t)nquads * S::pitch;
            if (ctx->staged_multi) {
                CU(ctx->vacc.reserve(nv * sizeof(int)));
                CU(cudaMemsetAsync(ctx->vacc.ptr, 0, nv * sizeof(int), ctx->stream));
            }
            k_matrix_staged<P, true><<<sgrid, SC::NTL, ctx->staged_smem, ctx->stream>>>(
                ctx->delta.as<uint8_t>(), ctx->colinfo.as<uint32_t>(), ctx->items.as<PanelItem>(), ctx->M.as<uint8_t>(), v0, v1,
                ctx->vacc.as<int>(), count, ctx->staged_bufwords, ctx->staged_nbuf, ctx->staged_multi);
            ctx->stats.kernel_launches++;
            CU(cudaGetLastError());
            if (ctx->staged_multi) {
                k_vec_finish<P><<<(unsigned)((nv + 255) / 256), 256, 0, ctx->stream>>>(ctx->vacc.as<int>(), v1, nv);
                ctx->stats.kernel_launches++;
                CU(cudaGetLastError());
            }
        } else {
            k_matrix_staged<P, false><<<sgrid, SC::NTL, ctx->staged_smem, ctx->stream>>>(
                ctx->delta.as<uint8_t>(), ctx->colinfo.as<uint32_t>(), ctx->items.as<PanelItem>(), ctx->M.as<uint8_t>(), nullptr,
                nullptr, nullptr, count, ctx->staged_bufwords, ctx->staged_nbuf, ctx->staged_multi);
            ctx->stats.kernel_launches++;
            CU(cudaGetLastError());
        }
        return QFS_OK;
    }
    const dim3 grid((unsigned)S::ngroups, (unsigned)((nquads + C::SLICE - 1) / C::SLICE));
    if (v0)
        k_matrix<P, true><<<grid, C::NT, 0, ctx->stream>>>(ctx->delta.as<uint8_t>(), ctx->colinfo.as<uint32_t>(),
                                                          ctx->groups.as<uint16_t>(), ctx->M.as<uint8_t>(), v0, v1, count);
    else
        k_matrix<P, false><<<grid, C::NT, 0, ctx->stream>>>(ctx->delta.as<uint8_t>(), ctx->colinfo.as<uint32_t>(),
                                                           ctx->groups.as<uint16_t>(), ctx->M.as<uint8_t>(), nullptr, nullptr, count);
    ctx->stats.kernel_launches++;
    CU(cudaGetLastError());
    return QFS_OK;
}

template <int P>
int launch_chain(qfs_ctx* ctx, const uint8_t* v0, const uint32_t* d_list, int count, int start_it, int max_steps,
                 uint8_t* trace, int8_t* heights, int8_t* iters)
{
    // Few, long surfaces (p >= 11 chunks, single-surface calls): the whole grid on one surface at a time
    // (k_chain_grid); otherwise one surface per persistent CTA (k_chain).  QFS_CHAIN_GRID=0/1 forces either.
    using G = ChainGridCfg<P>;
    // Cost model: the grid kernel pays a grid barrier (~3 us) plus N*pitch bytes at full bandwidth per step, a lone
    // CTA of k_chain streams ~50 GB/s; above half the CTA slots k_chain reaches full bandwidth by itself.
    const double expected = start_it > 0 ? (double)count / P : (double)count;  // surfaces the fused first step leaves undecided
    const double mbytes = (double)Shape<P>::N * Shape<P>::pitch;
    const double breakeven = (mbytes / 50e9) / (3e-6 + mbytes / 6e12);
    bool use_grid = count <= G::MAXCOUNT && expected < std::min(breakeven, 0.5 * ctx->sm_count * ChainCfg<P>::CTAS_PER_SM);
    if (ctx->chain_grid_mode >= 0) use_grid = ctx->chain_grid_mode > 0 && count <= G::MAXCOUNT;
    if (use_grid) {
        if (!ctx->chain_grid_ctas) {
            int per_sm = 0;
            CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chain_grid<P>, G::NT, G::SMEM));
            if (per_sm < 1) return fail(ctx, QFS_ECUDA, "k_chain_grid does not fit an SM");
            ctx->chain_grid_ctas = ctx->sm_count;  // one 1024-thread CTA per SM
        }
        CU(ctx->chain_scratch.reserve(2 * (size_t)Shape<P>::pitch));
        const uint8_t* M = ctx->M.as<uint8_t>();
        uint8_t* scratch = ctx->chain_scratch.as<uint8_t>();
        void* args[] = {(void*)&M, (void*)&v0, (void*)&d_list, (void*)&count, (void*)&start_it, (void*)&max_steps,
                        (void*)&trace, (void*)&heights, (void*)&iters, (void*)&scratch};
        const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_chain_grid<P>, dim3((unsigned)ctx->chain_grid_ctas),
                                                          dim3(G::NT), args, (size_t)G::SMEM, ctx->stream);
        if (e == cudaSuccess) {
            ctx->stats.kernel_launches++;
            return QFS_OK;
        }
        // a device partition that cannot hold one CTA per SM at once (MPS / green contexts): use the per-CTA kernel
        if (e != cudaErrorCooperativeLaunchTooLarge && e != cudaErrorNotSupported) CU(e);
        cudaGetLastError();
        ctx->chain_grid_mode = 0;
    }
    int* d_queue = ctx->flags.as<int>() + 1;
    CU(cudaMemsetAsync(d_queue, 0, sizeof(int), ctx->stream));
    const int grid = std::min(count, ctx->sm_count * ChainCfg<P>::CTAS_PER_SM);
    k_chain<P><<<grid, ChainCfg<P>::NT, ChainCfg<P>::SMEM, ctx->stream>>>(ctx->M.as<uint8_t>(), v0, d_list, count, start_it,
                                                                        max_steps, trace, heights, iters, d_queue);
    ctx->stats.kernel_launches++;
    CU(cudaGetLastError());
    return QFS_OK;
}

int check_device_flags(qfs_ctx* ctx)
{
    CU(cudaMemcpyAsync(ctx->h_flags, ctx->flags.ptr, 4 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->h_flags[0] & QFS_ERRBIT_INPUT)
        return fail(ctx, QFS_EINVAL, "input violates a precondition: a coefficient >= p or the zero form");
    if (ctx->h_flags[0] & QFS_ERRBIT_INVARIANT)
        return fail(ctx, QFS_EINVARIANT, "Witt-carry numerator not divisible by p");
    return QFS_OK;
}

float elapsed(cudaEvent_t a, cudaEvent_t b)
{
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int launch_compact(qfs_ctx* ctx, const int8_t* d_heights, size_t B, uint32_t* list, int* d_count)
{
    int tile = 4 * COMPACT_NT;
    if ((B + tile - 1) / tile > COMPACT_MAXTILES) tile = (int)(((B + COMPACT_MAXTILES - 1) / COMPACT_MAXTILES + COMPACT_NT - 1) / COMPACT_NT * COMPACT_NT);
    const unsigned tiles = (unsigned)((B + tile - 1) / tile);
    CU(ctx->compact_counts.reserve(COMPACT_MAXTILES * sizeof(int)));
    k_compact_count<<<tiles, COMPACT_NT, 0, ctx->stream>>>(d_heights, (int)B, tile, ctx->compact_counts.as<int>());
    k_compact_scatter<<<tiles, COMPACT_NT, 0, ctx->stream>>>(d_heights, (int)B, tile, ctx->compact_counts.as<int>(), list, d_count);
    ctx->stats.kernel_launches += 2;
    CU(cudaGetLastError());
    return QFS_OK;
}

// ---- the pipeline ----------------------------------------------------------------------------
template <int P>
int run_heights(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, int bound, int8_t* heights, int8_t* iters, void* user_stream, int mode)
{
    using S = Shape<P>;
    const bool matrix_free = mode == 1, lazy = mode == 2;   // 0: Delta and M for every hard surface (the reference's height_matrix)
    ctx->stats = qfs_stats{};
    ctx->stats.surfaces = (int64_t)B;
    if (B == 0) return QFS_OK;
    if (B > 0x7fffffffULL) return fail(ctx, QFS_EINVAL, "batch too large");
    DeviceGuard guard_(ctx->device);
    const bool in_dev = is_device_ptr(coeffs), hout_dev = is_device_ptr(heights), iout_dev = is_device_ptr(iters);
    if (user_stream || in_dev || hout_dev || iout_dev) {
        // Order the pipeline after whatever the caller has queued: on the stream it names, or -- no stream named -- on the
        // legacy default stream, which is where an unsuspecting producer of a device buffer runs (ctx->stream is non-blocking
        // and would not wait for it by itself).
        CU(cudaEventRecord(ctx->ev[0], user_stream ? (cudaStream_t)user_stream : cudaStreamLegacy));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev[0], 0));
    }
    const uint8_t* d_coeffs = coeffs;
    if (!in_dev) {
        CU(ctx->coeffs.reserve(B * 35));
        CU(cudaMemcpyAsync(ctx->coeffs.ptr, coeffs, B * 35, cudaMemcpyHostToDevice, ctx->stream));
        d_coeffs = ctx->coeffs.as<uint8_t>();
    }
    int8_t* d_heights = heights;
    int8_t* d_iters = iters;
    if (!hout_dev) { CU(ctx->heights.reserve(B)); d_heights = ctx->heights.as<int8_t>(); }
    if (!iout_dev) { CU(ctx->iters.reserve(B)); d_iters = ctx->iters.as<int8_t>(); }
    CU(ctx->list.reserve(B * sizeof(uint32_t)));
    int* d_flags = ctx->flags.as<int>();
    CU(cudaMemsetAsync(d_flags, 0, 4 * sizeof(int), ctx->stream));
    CU(cudaMemsetAsync(d_iters, 0, B, ctx->stream));
    CU(cudaEventRecord(ctx->ev_total[0], ctx->stream));

    // pass 1: Fedder test for every surface (height 1 or pending)
    CU(cudaEventRecord(ctx->ev[0], ctx->stream));
    constexpr int FED_SPC = PowerCfg<P>::FED_WARPS / PowerCfg<P>::FED_WPS;   // surfaces per CTA
    k_fedder<P><<<(unsigned)((B + FED_SPC - 1) / FED_SPC), PowerCfg<P>::FED_WARPS * 32,
                  PowerCfg<P>::FED_SMEM, ctx->stream>>>(d_coeffs, (int)B, ctx->unrank.as<uint32_t>(), d_heights, d_flags);
    ctx->stats.kernel_launches++;
    CU(cudaGetLastError());
    CU(cudaEventRecord(ctx->ev[1], ctx->stream));
    int hard = 0;
    if (bound < 2) {
        k_pending_to_inf<<<(unsigned)((B + 255) / 256), 256, 0, ctx->stream>>>(d_heights, (int)B);
        ctx->stats.kernel_launches++;
        int rc = check_device_flags(ctx);
        if (rc) return rc;
    } else {
        int rc = launch_compact(ctx, d_heights, B, ctx->list.as<uint32_t>(), d_flags + 2);
        if (rc) return rc;
        rc = check_device_flags(ctx);
        if (rc) return rc;
        hard = ctx->h_flags[2];
    }
    ctx->stats.ms_power += elapsed(ctx->ev[0], ctx->ev[1]);
    ctx->stats.hard = hard;
    ctx->stats.built = matrix_free ? 0 : hard;

    bool rows_kept = false;
    if (lazy && hard > 0) {
        // Lazy mode (qfs_caprow.cuh): the cap row of the first operator application decides 1 - 1/p of the hard surfaces
        // (height 2) from g, h, A, E alone; only the rest is compacted again and goes on to Delta, M and the chain.
        const size_t perf = (size_t)(3 * S::pitch + S::Nh_pad + S::NE_pad);
        const size_t budgetf = ctx->workspace_limit ? std::min<size_t>(ctx->workspace_limit, (size_t)1 << 30) : (size_t)1 << 30;
        const size_t capf = ctx->chunk_override ? std::min<size_t>((size_t)hard, ctx->chunk_override)
                                                : std::min<size_t>((size_t)hard, std::max<size_t>(1, budgetf / perf));
        int rc = reserve_chunk_free<P>(ctx, capf);
        if (rc) return rc;
        // one pass over all hard surfaces: the pending ones keep their g, h, A, E for the pipeline (k_gather_rows below)
        rows_kept = capf >= (size_t)hard && !getenv("QFS_LAZY_RECOMPUTE");
        if (rows_kept) CU(ctx->slotmap.reserve(B * sizeof(uint32_t)));
        CU(cudaEventRecord(ctx->ev[2], ctx->stream));
        for (size_t done = 0; done < (size_t)hard; done += capf) {
            const int cnt = (int)std::min<size_t>(capf, (size_t)hard - done);
            if ((rc = launch_power_full<P>(ctx, d_coeffs, ctx->list.as<uint32_t>() + done, cnt, nullptr))) return rc;
            k_caprow<P><<<cnt, CapRowCfg<P>::NT, CapRowCfg<P>::SMEM, ctx->stream>>>(
                ctx->g.as<uint8_t>(), ctx->h.as<uint8_t>(), ctx->A.as<uint8_t>(), ctx->E.as<uint8_t>(),
                ctx->unrank.as<uint32_t>() + qunrank_offset(1), ctx->unrank.as<uint32_t>() + qunrank_offset(P),
                ctx->unrank.as<uint32_t>() + qunrank_offset(P - 1),
                ctx->list.as<uint32_t>() + done, cnt, bound - 1, d_heights, d_iters, rows_kept ? ctx->slotmap.as<uint32_t>() : nullptr);
            ctx->stats.kernel_launches++;
            CU(cudaGetLastError());
        }
        CU(cudaEventRecord(ctx->ev[3], ctx->stream));
        if ((rc = launch_compact(ctx, d_heights, B, ctx->list.as<uint32_t>(), d_flags + 2))) return rc;
        rc = check_device_flags(ctx);
        if (rc) return rc;
        hard = ctx->h_flags[2];   // still pending: v1[cap] = 0 and bound > 2
        ctx->stats.ms_caprow = elapsed(ctx->ev[2], ctx->ev[3]);
        ctx->stats.built = hard;
        if (hard == 0) {   // every hard surface was decided by the cap row: the chunk loop below (and its sum of iterations) is skipped
            k_sum_iters<<<(unsigned)std::min<size_t>((B + 1023) / 1024, 1024), 1024, 0, ctx->stream>>>(d_iters, B, d_flags + 3);
            ctx->stats.kernel_launches++;
            if ((rc = check_device_flags(ctx))) return rc;
            ctx->stats.matvec_steps = ctx->h_flags[3];
        }
    }

    if (hard > 0) {
        // chunk capacity from the workspace budget
        size_t limit = ctx->workspace_limit;
        if (!limit) {
            if (!ctx->auto_limit) {  // asked once per context: cudaMemGetInfo costs milliseconds on a busy heap
                size_t fr = 0, tot = 0;
                CU(cudaMemGetInfo(&fr, &tot));
                size_t held = ctx->g.cap + ctx->A.cap + ctx->h.cap + ctx->E.cap + ctx->delta.cap + ctx->M.cap + ctx->v1.cap + ctx->ecm.cap + ctx->hbox.cap;
                ctx->auto_limit = (size_t)((double)(fr + held) * 0.75);
            }
            limit = ctx->auto_limit;
        }
        const size_t per = matrix_free ? (size_t)(3 * S::pitch + S::Nh_pad + S::NE_pad) : per_surface_bytes<P>();
        size_t cap = ctx->chunk_override ? ctx->chunk_override : std::max<size_t>(1, limit / per);
        cap = std::min<size_t>(cap, (size_t)hard);
        if (!matrix_free && !ctx->chunk_override && cap < (size_t)hard) {
            // Few, large surfaces per chunk (p >= 11): a chunk of whole Witt-carry waves (one CTA per surface, delta_wave
            // CTAs resident) avoids a partial last wave in every chunk (F_11: 460 -> 444 = 3 x 148; 80 -> 61 waves per 9016 surfaces)
            const size_t wave = (size_t)ctx->delta_wave;
            if (wave && cap >= wave && cap < 16 * wave) cap = cap / wave * wave;
        }
        const void* kept[4] = {ctx->g.ptr, ctx->h.ptr, ctx->A.ptr, ctx->E.ptr};
        while (true) {
            int rc = matrix_free ? reserve_chunk_free<P>(ctx, cap) : reserve_chunk<P>(ctx, cap);
            if (rc == QFS_OK) break;
            if (rc != QFS_ENOMEM || cap == 1) return rc;
            cudaGetLastError();
            cap = std::max<size_t>(1, cap / 2);
        }
        ctx->stats.chunk_capacity = (int64_t)cap;
        const uint32_t* d_list = ctx->list.as<uint32_t>();
        // Chunks are queued back to back: the stage boundaries of every chunk get their own events, read after the one
        // synchronisation at the end of the call (no host round trip between chunks).
        const size_t nchunks = ((size_t)hard + cap - 1) / cap;
        while (ctx->chunk_ev.size() < 5 * nchunks) {
            cudaEvent_t e = nullptr;
            CU(cudaEventCreate(&e));
            ctx->chunk_ev.push_back(e);
        }
        size_t ci = 0;
        for (size_t done = 0; done < (size_t)hard; done += cap, ++ci) {
            const int cnt = (int)std::min<size_t>(cap, (size_t)hard - done);
            cudaEvent_t* ev = &ctx->chunk_ev[5 * ci];
            int rc;
            CU(cudaEventRecord(ev[0], ctx->stream));
            if (rows_kept && nchunks == 1 && kept[0] == ctx->g.ptr && kept[1] == ctx->h.ptr && kept[2] == ctx->A.ptr && kept[3] == ctx->E.ptr) {
                // lazy mode, one chunk: g, h, A, E of the pending surfaces are still in the workspaces, at the slots of the cap-row
                // pass; gather them to the slots of the compacted list through the (still unused) matrix workspace
                GatherRows gr;
                const uint8_t* src[4] = {ctx->g.as<uint8_t>(), ctx->h.as<uint8_t>(), ctx->A.as<uint8_t>(), ctx->E.as<uint8_t>()};
                const size_t rowb[4] = {(size_t)S::pitch, (size_t)S::Nh_pad, (size_t)S::pitch, (size_t)S::NE_pad};
                uint8_t* scratch = ctx->M.as<uint8_t>();
                size_t off = 0;
                for (int a = 0; a < 4; ++a) {
                    gr.src[a] = src[a];
                    gr.dst[a] = scratch + off;
                    gr.row16[a] = (uint32_t)(rowb[a] / 16);
                    off += (size_t)cnt * rowb[a];
                }
                k_gather_rows<<<cnt, 128, 0, ctx->stream>>>(gr, d_list, ctx->slotmap.as<uint32_t>(), cnt);
                ctx->stats.kernel_launches++;
                CU(cudaGetLastError());
                for (int a = 0; a < 4; ++a)
                    CU(cudaMemcpyAsync(const_cast<uint8_t*>(src[a]), gr.dst[a], (size_t)cnt * rowb[a], cudaMemcpyDeviceToDevice, ctx->stream));
            } else if ((rc = launch_power_full<P>(ctx, d_coeffs, d_list + done, cnt, nullptr))) return rc;
            CU(cudaEventRecord(ev[1], ctx->stream));
            if (matrix_free) {
                // the operator iteration without Delta and without M (qfs_free.cuh): stage times delta = matrix = 0
                CU(cudaEventRecord(ev[2], ctx->stream));
                CU(cudaEventRecord(ev[3], ctx->stream));
                k_free<P><<<cnt, FreeCfg<P>::NT, FreeCfg<P>::SMEM, ctx->stream>>>(
                    ctx->g.as<uint8_t>(), ctx->h.as<uint8_t>(), ctx->E.as<uint8_t>(), ctx->unrank.as<uint32_t>() + qunrank_offset(P),
                    ctx->unrank.as<uint32_t>() + qunrank_offset(P - 1), d_list + done, bound - 1, d_heights, d_iters);
                ctx->stats.kernel_launches++;
                CU(cudaGetLastError());
            } else {
                if ((rc = launch_delta<P>(ctx, cnt))) return rc;
                CU(cudaEventRecord(ev[2], ctx->stream));
                if ((rc = launch_matrix<P>(ctx, cnt, ctx->g.as<uint8_t>(), ctx->v1.as<uint8_t>()))) return rc;
                CU(cudaEventRecord(ev[3], ctx->stream));
                if ((rc = launch_chain<P>(ctx, ctx->v1.as<uint8_t>(), d_list + done, cnt, 1, bound - 1, nullptr, d_heights, d_iters))) return rc;
            }
            CU(cudaEventRecord(ev[4], ctx->stream));
            ctx->stats.chunks++;
        }
        k_sum_iters<<<(unsigned)std::min<size_t>((B + 1023) / 1024, 1024), 1024, 0, ctx->stream>>>(d_iters, B, d_flags + 3);
        ctx->stats.kernel_launches++;
        int rc = check_device_flags(ctx);   // the call's one synchronisation after the chunk loop
        if (rc) return rc;
        ctx->stats.matvec_steps = ctx->h_flags[3];
        for (size_t c = 0; c < nchunks; ++c) {
            cudaEvent_t* ev = &ctx->chunk_ev[5 * c];
            ctx->stats.ms_power += elapsed(ev[0], ev[1]);
            ctx->stats.ms_delta += elapsed(ev[1], ev[2]);
            ctx->stats.ms_matrix += elapsed(ev[2], ev[3]);
            ctx->stats.ms_matvec += elapsed(ev[3], ev[4]);
        }
    }
    CU(cudaEventRecord(ctx->ev_total[1], ctx->stream));
    if (!hout_dev) CU(cudaMemcpyAsync(heights, d_heights, B, cudaMemcpyDeviceToHost, ctx->stream));
    if (!iout_dev) CU(cudaMemcpyAsync(iters, d_iters, B, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->stats.ms_total = elapsed(ctx->ev_total[0], ctx->ev_total[1]);
    return QFS_OK;
}

// copy a [B][n] dense host/device array into a padded device workspace and back
int to_padded(qfs_ctx* ctx, DevBuf& buf, const uint8_t* src, size_t rows, size_t n, size_t pitch)
{
    CU(buf.reserve(rows * pitch));
    CU(cudaMemsetAsync(buf.ptr, 0, rows * pitch, ctx->stream));
    CU(cudaMemcpy2DAsync(buf.ptr, pitch, src, n, n, rows, cudaMemcpyDefault, ctx->stream));
    return QFS_OK;
}
int from_padded(qfs_ctx* ctx, uint8_t* dst, const void* src, size_t rows, size_t n, size_t pitch)
{
    CU(cudaMemcpy2DAsync(dst, n, src, pitch, n, rows, cudaMemcpyDefault, ctx->stream));
    return QFS_OK;
}

// Taps process the batch in slices small enough for the workspaces.
template <int P>
size_t tap_slice(qfs_ctx* ctx, size_t B, size_t bytes_per_row)
{
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    size_t lim = ctx->workspace_limit ? ctx->workspace_limit : (size_t)(fr * 0.3);
    return std::max<size_t>(1, std::min<size_t>(std::min<size_t>(B, 32768), lim / std::max<size_t>(1, bytes_per_row)));
}

template <int P>
int run_stage_power(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, uint8_t* g, uint8_t* fedder)
{
    using S = Shape<P>;
    DeviceGuard guard_(ctx->device);
    CU(cudaMemsetAsync(ctx->flags.ptr, 0, 4 * sizeof(int), ctx->stream));
    const size_t slice = tap_slice<P>(ctx, B, per_surface_bytes<P>() - (size_t)S::N * S::pitch - S::Lg_pad + 64);
    CU(ctx->tapA.reserve(slice * 35));
    CU(ctx->tapB.reserve(slice));
    for (size_t done = 0; done < B; done += slice) {
        const int cnt = (int)std::min(slice, B - done);
        CU(ctx->g.reserve((size_t)cnt * S::pitch));
        CU(ctx->A.reserve((size_t)cnt * S::pitch));
        CU(ctx->h.reserve((size_t)cnt * S::Nh_pad));
        CU(ctx->E.reserve((size_t)cnt * S::NE_pad));
        CU(cudaMemcpyAsync(ctx->tapA.ptr, coeffs + done * 35, (size_t)cnt * 35, cudaMemcpyDefault, ctx->stream));
        int rc = launch_power_full<P>(ctx, ctx->tapA.as<uint8_t>(), nullptr, cnt, ctx->tapB.as<uint8_t>());
        if (rc) return rc;
        if (g && (rc = from_padded(ctx, g + done * S::N, ctx->g.ptr, cnt, S::N, S::pitch))) return rc;
        if (fedder) CU(cudaMemcpyAsync(fedder + done, ctx->tapB.ptr, cnt, cudaMemcpyDefault, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    return check_device_flags(ctx);
}

template <int P>
int run_stage_delta(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, uint8_t* delta)
{
    using S = Shape<P>;
    DeviceGuard guard_(ctx->device);
    CU(cudaMemsetAsync(ctx->flags.ptr, 0, 4 * sizeof(int), ctx->stream));
    const size_t slice = tap_slice<P>(ctx, B, per_surface_bytes<P>() - (size_t)S::N * S::pitch + S::L);
    CU(ctx->tapA.reserve(slice * 35));
    for (size_t done = 0; done < B; done += slice) {
        const int cnt = (int)std::min(slice, B - done);
        CU(ctx->g.reserve((size_t)cnt * S::pitch));
        CU(ctx->A.reserve((size_t)cnt * S::pitch));
        CU(ctx->h.reserve((size_t)cnt * S::Nh_pad));
        CU(ctx->E.reserve((size_t)cnt * S::NE_pad));
        const size_t cnt4 = ((size_t)cnt + 3) & ~(size_t)3;
        CU(ctx->delta.reserve(cnt4 * S::Lg_pad));
        CU(ctx->tapB.reserve((size_t)cnt * S::L));
        CU(cudaMemcpyAsync(ctx->tapA.ptr, coeffs + done * 35, (size_t)cnt * 35, cudaMemcpyDefault, ctx->stream));
        int rc = launch_power_full<P>(ctx, ctx->tapA.as<uint8_t>(), nullptr, cnt, nullptr);
        if (rc) return rc;
        if ((rc = launch_delta<P>(ctx, cnt))) return rc;
        dim3 grid(S::D + 1, cnt);
        k_delta_flip<P, false><<<grid, 256, 0, ctx->stream>>>(ctx->tapB.as<uint8_t>(), ctx->delta.as<uint8_t>());
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(delta + done * (size_t)S::L, ctx->tapB.ptr, (size_t)cnt * S::L, cudaMemcpyDefault, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    return check_device_flags(ctx);
}

template <int P>
int run_stage_matrix(qfs_ctx* ctx, const uint8_t* delta, size_t B, uint8_t* M)
{
    using S = Shape<P>;
    DeviceGuard guard_(ctx->device);
    const size_t slice = tap_slice<P>(ctx, B, (size_t)S::N * S::pitch + (size_t)S::Lg_pad + S::L);
    for (size_t done = 0; done < B; done += slice) {
        const int cnt = (int)std::min(slice, B - done);
        int rc;
        CU(ctx->tapB.reserve((size_t)cnt * S::L));
        CU(cudaMemcpyAsync(ctx->tapB.ptr, delta + done * (size_t)S::L, (size_t)cnt * S::L, cudaMemcpyDefault, ctx->stream));
        const size_t cnt4 = ((size_t)cnt + 3) & ~(size_t)3;
        CU(ctx->delta.reserve(cnt4 * S::Lg_pad));
        CU(cudaMemsetAsync(ctx->delta.ptr, 0, cnt4 * S::Lg_pad, ctx->stream));
        CU(ctx->M.reserve(cnt4 * S::N * S::pitch));
        dim3 grid(S::D + 1, cnt);
        k_delta_flip<P, true><<<grid, 256, 0, ctx->stream>>>(ctx->tapB.as<uint8_t>(), ctx->delta.as<uint8_t>());
        CU(cudaGetLastError());
        if ((rc = launch_matrix<P>(ctx, cnt, nullptr, nullptr))) return rc;
        if ((rc = from_padded(ctx, M + done * (size_t)S::N * S::N, ctx->M.ptr, (size_t)cnt * S::N, S::N, S::pitch))) return rc;
        CU(cudaStreamSynchronize(ctx->stream));
    }
    return QFS_OK;
}

// Operator matrices of B quartics in the reference's export layout (uint16 entries, no pitch), host or device output.
template <int P>
int run_export_matrix(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, uint16_t* M16)
{
    using S = Shape<P>;
    DeviceGuard guard_(ctx->device);
    CU(cudaMemsetAsync(ctx->flags.ptr, 0, 4 * sizeof(int), ctx->stream));
    const bool out_dev = is_device_ptr(M16);
    const size_t nn = (size_t)S::N * S::N;
    const size_t slice = tap_slice<P>(ctx, B, per_surface_bytes<P>() + 2 * nn);
    CU(ctx->tapA.reserve(slice * 35));
    for (size_t done = 0; done < B; done += slice) {
        const int cnt = (int)std::min(slice, B - done);
        int rc = reserve_chunk<P>(ctx, (size_t)cnt);
        if (rc) return rc;
        uint16_t* d_out = M16 + done * nn;
        if (!out_dev) { CU(ctx->tapB.reserve((size_t)cnt * nn * 2)); d_out = ctx->tapB.as<uint16_t>(); }
        CU(cudaMemcpyAsync(ctx->tapA.ptr, coeffs + done * 35, (size_t)cnt * 35, cudaMemcpyDefault, ctx->stream));
        if ((rc = launch_power_full<P>(ctx, ctx->tapA.as<uint8_t>(), nullptr, cnt, nullptr))) return rc;
        if ((rc = launch_delta<P>(ctx, cnt))) return rc;
        if ((rc = launch_matrix<P>(ctx, cnt, nullptr, nullptr))) return rc;
        k_widen_u16<<<dim3(S::N, cnt), 256, 0, ctx->stream>>>(ctx->M.as<uint8_t>(), S::N, S::pitch, d_out);
        CU(cudaGetLastError());
        if (!out_dev) CU(cudaMemcpyAsync(M16 + done * nn, d_out, (size_t)cnt * nn * 2, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    return check_device_flags(ctx);
}

template <int P>
int run_stage_chain(qfs_ctx* ctx, const uint8_t* M, const uint8_t* v0, size_t B, int max_steps, uint8_t* trace,
                    int8_t* heights, int8_t* iters)
{
    using S = Shape<P>;
    DeviceGuard guard_(ctx->device);
    if (max_steps < 0) return fail(ctx, QFS_EINVAL, "max_steps must be >= 0");
    const size_t slice = tap_slice<P>(ctx, B, (size_t)S::N * S::pitch + (size_t)(max_steps + 2) * S::pitch);
    CU(ctx->heights.reserve(B));
    CU(ctx->iters.reserve(B));
    CU(cudaMemsetAsync(ctx->heights.ptr, 0, B, ctx->stream));
    CU(cudaMemsetAsync(ctx->iters.ptr, 0, B, ctx->stream));
    for (size_t done = 0; done < B; done += slice) {
        const int cnt = (int)std::min(slice, B - done);
        int rc = to_padded(ctx, ctx->M, M + done * (size_t)S::N * S::N, (size_t)cnt * S::N, S::N, S::pitch);
        if (rc) return rc;
        if ((rc = to_padded(ctx, ctx->g, v0 + done * S::N, cnt, S::N, S::pitch))) return rc;
        uint8_t* d_trace = nullptr;
        if (trace && max_steps > 0) {
            CU(ctx->tapB.reserve((size_t)cnt * max_steps * S::N));
            CU(cudaMemsetAsync(ctx->tapB.ptr, 0, (size_t)cnt * max_steps * S::N, ctx->stream));
            d_trace = ctx->tapB.as<uint8_t>();
        }
        if ((rc = launch_chain<P>(ctx, ctx->g.as<uint8_t>(), nullptr, cnt, 0, max_steps, d_trace,
                                  ctx->heights.as<int8_t>() + done, ctx->iters.as<int8_t>() + done)))
            return rc;
        if (d_trace)
            CU(cudaMemcpyAsync(trace + done * (size_t)max_steps * S::N, d_trace, (size_t)cnt * max_steps * S::N,
                               cudaMemcpyDefault, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    CU(cudaMemcpyAsync(heights, ctx->heights.ptr, B, cudaMemcpyDefault, ctx->stream));
    CU(cudaMemcpyAsync(iters, ctx->iters.ptr, B, cudaMemcpyDefault, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return QFS_OK;
}

template <int P>
void fill_shape(qfs_shape* s)
{
    using S = Shape<P>;
    s->p = P; s->d = S::d; s->D = S::D; s->N = S::N; s->pitch = S::pitch; s->cap = S::cap; s->L = S::L;
}

#define QFS_FOR_PRIME(p, F, ...)                 \
    switch (p) {                                 \
        case 3: return F<3>(__VA_ARGS__);        \
        case 5: return F<5>(__VA_ARGS__);        \
        case 7: return F<7>(__VA_ARGS__);        \
        case 11: return F<11>(__VA_ARGS__);      \
        case 13: return F<13>(__VA_ARGS__);      \
        default: return QFS_EINVAL;              \
    }

}  // namespace

extern "C" {

int qfs_version(void) { return QFS_ABI_VERSION; }

int qfs_get_shape(int p, qfs_shape* out)
{
    qfs_shape tmp;
    qfs_shape* s = out ? out : &tmp;
    switch (p) {
        case 3: fill_shape<3>(s); return QFS_OK;
        case 5: fill_shape<5>(s); return QFS_OK;
        case 7: fill_shape<7>(s); return QFS_OK;
        case 11: fill_shape<11>(s); return QFS_OK;
        case 13: fill_shape<13>(s); return QFS_OK;
        default: return QFS_EINVAL;
    }
}

const char* qfs_last_error(const qfs_ctx* ctx) { return ctx ? ctx->error.c_str() : g_create_error.c_str(); }

void qfs_destroy(qfs_ctx* ctx)
{
    if (!ctx) return;
    DeviceGuard guard_(ctx->device);
    DevBuf* bufs[] = {&ctx->flags, &ctx->colinfo, &ctx->groups, &ctx->runs, &ctx->unrank, &ctx->coeffs, &ctx->heights, &ctx->iters, &ctx->list,
                      &ctx->g, &ctx->h, &ctx->A, &ctx->E, &ctx->delta, &ctx->M, &ctx->v1, &ctx->tapA, &ctx->tapB, &ctx->items, &ctx->vacc, &ctx->chain_scratch,
                      &ctx->ecm, &ctx->hbox, &ctx->dphases_few, &ctx->dparts_few, &ctx->dphases_mid, &ctx->dparts_mid, &ctx->dphases, &ctx->dpieces, &ctx->dparts};
    for (DevBuf* b : bufs) b->release();
    for (auto& e : ctx->ev) if (e) cudaEventDestroy(e);
    for (auto& e : ctx->ev_total) if (e) cudaEventDestroy(e);
    for (auto& e : ctx->chunk_ev) if (e) cudaEventDestroy(e);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
    delete ctx;
}

int qfs_create(int p, int device, size_t max_batch, qfs_ctx** out)
{
    (void)max_batch;
    if (!out) return fail(nullptr, QFS_EINVAL, "out is NULL");
    *out = nullptr;
    if (qfs_get_shape(p, nullptr) != QFS_OK)
        return fail(nullptr, QFS_EINVAL, "p=%d is not supported by this build (supported: 3, 5, 7, 11, 13)", p);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(nullptr, QFS_ECUDA, "no CUDA device available: %s", cudaGetErrorString(e));
    if (device < 0 || device >= ndev) return fail(nullptr, QFS_EINVAL, "device %d out of range (0..%d)", device, ndev - 1);
    qfs_ctx* ctx = new qfs_ctx;
    ctx->p = p;
    ctx->device = device;
    auto bail = [&](int rc) { g_create_error = ctx->error; qfs_destroy(ctx); return rc; };
#define CUC(call)                                                                                          \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess) { fail(ctx, QFS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); return bail(QFS_ECUDA); } \
    } while (0)
    CUC(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUC(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
        fail(ctx, QFS_ECUDA, "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device, prop.major, prop.minor);
        return bail(QFS_ECUDA);
    }
    ctx->sm_count = prop.multiProcessorCount;
    CUC(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    for (auto& ev : ctx->ev) CUC(cudaEventCreate(&ev));
    for (auto& ev : ctx->ev_total) CUC(cudaEventCreate(&ev));
    CUC(cudaMallocHost(&ctx->h_flags, 4 * sizeof(int)));
    CUC(ctx->flags.reserve(4 * sizeof(int)));
    CUC(cudaMemset(ctx->flags.ptr, 0, 4 * sizeof(int)));
#undef CUC
    int rc;
    switch (p) {
        case 3: rc = build_tables<3>(ctx); break;
        case 5: rc = build_tables<5>(ctx); break;
        case 7: rc = build_tables<7>(ctx); break;
        case 11: rc = build_tables<11>(ctx); break;
        default: rc = build_tables<13>(ctx); break;
    }
    if (rc) return bail(rc);
    *out = ctx;
    return QFS_OK;
}

int qfs_set_workspace_limit(qfs_ctx* ctx, size_t bytes)
{
    if (!ctx) return QFS_EINVAL;
    ctx->workspace_limit = bytes;
    return QFS_OK;
}

int qfs_set_chunk(qfs_ctx* ctx, size_t n)
{
    if (!ctx) return QFS_EINVAL;
    ctx->chunk_override = n;
    return QFS_OK;
}

int qfs_get_stats(const qfs_ctx* ctx, qfs_stats* out)
{
    if (!ctx || !out) return QFS_EINVAL;
    *out = ctx->stats;
    return QFS_OK;
}

int qfs_heights(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, int bound, int8_t* heights, int8_t* iters, void* stream)
{
    if (!ctx) return QFS_EINVAL;
    if (B && (!coeffs || !heights || !iters)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    if (bound < 1 || bound > 127) return fail(ctx, QFS_EINVAL, "bound must be in 1..127, got %d", bound);
    QFS_FOR_PRIME(ctx->p, run_heights, ctx, coeffs, B, bound, heights, iters, stream, 0)
}

int qfs_heights_free(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, int bound, int8_t* heights, int8_t* iters, void* stream)
{
    if (!ctx) return QFS_EINVAL;
    if (B && (!coeffs || !heights || !iters)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    if (bound < 1 || bound > 127) return fail(ctx, QFS_EINVAL, "bound must be in 1..127, got %d", bound);
    QFS_FOR_PRIME(ctx->p, run_heights, ctx, coeffs, B, bound, heights, iters, stream, 1)
}

int qfs_heights_lazy(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, int bound, int8_t* heights, int8_t* iters, void* stream)
{
    if (!ctx) return QFS_EINVAL;
    if (B && (!coeffs || !heights || !iters)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    if (bound < 1 || bound > 127) return fail(ctx, QFS_EINVAL, "bound must be in 1..127, got %d", bound);
    QFS_FOR_PRIME(ctx->p, run_heights, ctx, coeffs, B, bound, heights, iters, stream, 2)
}

int qfs_stage_power(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, uint8_t* g, uint8_t* fedder)
{
    if (!ctx) return QFS_EINVAL;
    if (B && !coeffs) return fail(ctx, QFS_EINVAL, "NULL buffer");
    QFS_FOR_PRIME(ctx->p, run_stage_power, ctx, coeffs, B, g, fedder)
}

int qfs_stage_delta(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, uint8_t* delta)
{
    if (!ctx) return QFS_EINVAL;
    if (B && (!coeffs || !delta)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    QFS_FOR_PRIME(ctx->p, run_stage_delta, ctx, coeffs, B, delta)
}

int qfs_stage_matrix(qfs_ctx* ctx, const uint8_t* delta, size_t B, uint8_t* M)
{
    if (!ctx) return QFS_EINVAL;
    if (B && (!delta || !M)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    QFS_FOR_PRIME(ctx->p, run_stage_matrix, ctx, delta, B, M)
}

int qfs_cubic_heights(int device, int p, const uint8_t* coeffs, size_t B, int bound, int8_t* heights, int8_t* iters)
{
    qfs_ctx* ctx = nullptr;  // errors of this context-free entry go where qfs_create's go: qfs_last_error(NULL)
    if (p < 3 || p > QFS_CUBIC_MAXP || p % 2 == 0) return fail(ctx, QFS_EINVAL, "cubic curves: p=%d is not an odd prime <= %d", p, QFS_CUBIC_MAXP);
    for (int q = 3; q * q <= p; q += 2)
        if (p % q == 0) return fail(ctx, QFS_EINVAL, "p=%d is not prime", p);
    if (bound < 1 || bound > 127) return fail(ctx, QFS_EINVAL, "bound must be in 1..127, got %d", bound);
    if (B == 0) return QFS_OK;
    if (!coeffs || !heights || !iters) return fail(ctx, QFS_EINVAL, "NULL buffer");
    if (B > 0x7fffffffULL) return fail(ctx, QFS_EINVAL, "batch too large");
    DeviceGuard guard_(device);
    const bool in_dev = is_device_ptr(coeffs), h_dev = is_device_ptr(heights), i_dev = is_device_ptr(iters);
    uint8_t* d_c = nullptr;
    int8_t *d_h = nullptr, *d_i = nullptr;
    int* d_err = nullptr;
    int rc = QFS_OK, h_err = 0;
    auto cleanup = [&]() {
        if (!in_dev && d_c) cudaFree(d_c);
        if (!h_dev && d_h) cudaFree(d_h);
        if (!i_dev && d_i) cudaFree(d_i);
        if (d_err) cudaFree(d_err);
    };
#define CUC(call)                                                                                          \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess) {                                                                           \
            rc = fail(ctx, e_ == cudaErrorMemoryAllocation ? QFS_ENOMEM : QFS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
            cleanup();                                                                                     \
            return rc;                                                                                     \
        }                                                                                                  \
    } while (0)
    if (in_dev) d_c = const_cast<uint8_t*>(coeffs);
    else { CUC(cudaMalloc(&d_c, B * 10)); CUC(cudaMemcpy(d_c, coeffs, B * 10, cudaMemcpyHostToDevice)); }
    if (h_dev) d_h = heights; else CUC(cudaMalloc(&d_h, B));
    if (i_dev) d_i = iters; else CUC(cudaMalloc(&d_i, B));
    CUC(cudaMalloc(&d_err, sizeof(int)));
    CUC(cudaMemset(d_err, 0, sizeof(int)));
    const size_t smem = qfs_cubic_smem(p);
    CUC(cudaFuncSetAttribute(k_cubic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_cubic<<<(unsigned)B, QFS_CUBIC_NT, smem>>>(d_c, (int)B, p, bound - 1, d_h, d_i, d_err);
    CUC(cudaGetLastError());
    CUC(cudaMemcpy(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (!h_dev) CUC(cudaMemcpy(heights, d_h, B, cudaMemcpyDeviceToHost));
    if (!i_dev) CUC(cudaMemcpy(iters, d_i, B, cudaMemcpyDeviceToHost));
    CUC(cudaDeviceSynchronize());
#undef CUC
    cleanup();
    if (h_err & QFS_ERRBIT_INPUT) return fail(ctx, QFS_EINVAL, "input violates a precondition: a coefficient >= p or the zero form");
    if (h_err & QFS_ERRBIT_INVARIANT) return fail(ctx, QFS_EINVARIANT, "Witt-carry numerator not divisible by p");
    return QFS_OK;
}

int qfs_form_heights(int device, int p, int n, const uint8_t* coeffs, size_t B, int bound, int8_t* heights, int8_t* iters)
{
    qfs_ctx* ctx = nullptr;  // errors of this context-free entry go where qfs_create's go: qfs_last_error(NULL)
    if (n < 2 || n > QFS_FORM_MAXN) return fail(ctx, QFS_EINVAL, "forms in n = 2..%d variables, got n=%d", QFS_FORM_MAXN, n);
    if (p < 3 || p > QFS_FORM_MAXP || p % 2 == 0) return fail(ctx, QFS_EINVAL, "p=%d is not an odd prime <= %d", p, QFS_FORM_MAXP);
    for (int q = 3; q * q <= p; q += 2)
        if (p % q == 0) return fail(ctx, QFS_EINVAL, "p=%d is not prime", p);
    {
        double box = 1;
        for (int i = 0; i < n - 1; ++i) box *= (double)(n * p + 1);
        if (box > (double)QFS_FORM_MAXBOX) return fail(ctx, QFS_EINVAL, "n=%d, p=%d: (n p + 1)^(n-1) exceeds 2^24 entries", n, p);
    }
    if (bound < 1 || bound > 127) return fail(ctx, QFS_EINVAL, "bound must be in 1..127, got %d", bound);
    if (B == 0) return QFS_OK;
    if (!coeffs || !heights || !iters) return fail(ctx, QFS_EINVAL, "NULL buffer");
    if (B > 0x7fffffffULL) return fail(ctx, QFS_EINVAL, "batch too large");
    // basis(n, n) in lex-ascending order, x1 most significant (monomials.py:182-196)
    std::vector<uint8_t> ex;
    {
        std::vector<int> e(n, 0);
        std::function<void(int, int)> rec = [&](int i, int left) {
            if (i == n - 1) { e[i] = left; for (int v : e) ex.push_back((uint8_t)v); return; }
            for (int a = 0; a <= left; ++a) { e[i] = a; rec(i + 1, left - a); }
        };
        rec(0, n);
    }
    const int nterms = (int)(ex.size() / n);
    DeviceGuard guard_(device);
    const bool in_dev = is_device_ptr(coeffs), h_dev = is_device_ptr(heights), i_dev = is_device_ptr(iters);
    uint8_t *d_c = nullptr, *d_ex = nullptr, *d_scratch = nullptr;
    int8_t *d_h = nullptr, *d_i = nullptr;
    int* d_err = nullptr;
    int rc = QFS_OK, h_err = 0;
    auto cleanup = [&]() {
        if (!in_dev && d_c) cudaFree(d_c);
        if (!h_dev && d_h) cudaFree(d_h);
        if (!i_dev && d_i) cudaFree(d_i);
        if (d_ex) cudaFree(d_ex);
        if (d_scratch) cudaFree(d_scratch);
        if (d_err) cudaFree(d_err);
    };
#define CUC(call)                                                                                          \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess) {                                                                           \
            rc = fail(ctx, e_ == cudaErrorMemoryAllocation ? QFS_ENOMEM : QFS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
            cleanup();                                                                                     \
            return rc;                                                                                     \
        }                                                                                                  \
    } while (0)
    const size_t row = (size_t)nterms;
    if (in_dev) d_c = const_cast<uint8_t*>(coeffs);
    else { CUC(cudaMalloc(&d_c, B * row)); CUC(cudaMemcpy(d_c, coeffs, B * row, cudaMemcpyHostToDevice)); }
    if (h_dev) d_h = heights; else CUC(cudaMalloc(&d_h, B));
    if (i_dev) d_i = iters; else CUC(cudaMalloc(&d_i, B));
    CUC(cudaMalloc(&d_ex, ex.size()));
    CUC(cudaMemcpy(d_ex, ex.data(), ex.size(), cudaMemcpyHostToDevice));
    CUC(cudaMalloc(&d_err, sizeof(int)));
    CUC(cudaMemset(d_err, 0, sizeof(int)));
    const size_t per = qfs_form_scratch(n, p);
    const size_t chunk = std::max<size_t>(1, std::min<size_t>(std::min<size_t>(B, 1184), ((size_t)1 << 30) / per));   // <= 8 CTAs per SM, <= 1 GB
    CUC(cudaMalloc(&d_scratch, chunk * per));
    for (size_t first = 0; first < B; first += chunk) {
        const unsigned cnt = (unsigned)std::min(chunk, B - first);
        k_form<<<cnt, QFS_FORM_NT>>>(d_c, d_ex, nterms, (int)B, (int)first, n, p, bound - 1, d_scratch, d_h, d_i, d_err);
        CUC(cudaGetLastError());
    }
    CUC(cudaMemcpy(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (!h_dev) CUC(cudaMemcpy(heights, d_h, B, cudaMemcpyDeviceToHost));
    if (!i_dev) CUC(cudaMemcpy(iters, d_i, B, cudaMemcpyDeviceToHost));
    CUC(cudaDeviceSynchronize());
#undef CUC
    cleanup();
    if (h_err & QFS_ERRBIT_INPUT) return fail(ctx, QFS_EINVAL, "input violates a precondition: a coefficient >= p or the zero form");
    if (h_err & QFS_ERRBIT_INVARIANT) return fail(ctx, QFS_EINVARIANT, "Witt-carry numerator not divisible by p");
    return QFS_OK;
}

int qfs_literal_heights(int device, int p, const uint8_t* coeffs, size_t B, int bound, int8_t* heights, int8_t* iters, uint8_t* g_out,
                        uint8_t* delta_out)
{
    qfs_ctx* ctx = nullptr;  // context-free: errors go where qfs_create's go, qfs_last_error(NULL)
    if (p != 3 && p != 5 && p != 7) return fail(ctx, QFS_EINVAL, "the literal route runs for p = 3, 5, 7 (got p=%d)", p);
    if (bound < 1 || bound > 127) return fail(ctx, QFS_EINVAL, "bound must be in 1..127, got %d", bound);
    if (B == 0) return QFS_OK;
    if (!coeffs || !heights || !iters) return fail(ctx, QFS_EINVAL, "NULL buffer");
    if (B > 0x7fffffffULL) return fail(ctx, QFS_EINVAL, "batch too large");
    const int d = 4 * (p - 1), D = p * d, W = D + 1;
    const size_t boxsize = ((size_t)W * W * W + 15) & ~(size_t)15;
    const size_t N = (size_t)qc3(d + 3), L = (size_t)qc3(D + 3);
    DeviceGuard guard_(device);
    const size_t chunk = std::max<size_t>(1, std::min<size_t>(std::min<size_t>(B, 8192), ((size_t)768 << 20) / (3 * boxsize)));
    uint8_t *d_c = nullptr, *X = nullptr, *Y = nullptr, *Gb = nullptr, *dense = nullptr;
    int8_t *d_h = nullptr, *d_i = nullptr;
    LitTerm* terms = nullptr;
    int *nterms = nullptr, *done = nullptr, *d_err = nullptr;
    int rc = QFS_OK, h_err = 0;
    auto cleanup = [&]() {
        for (void* q : {(void*)d_c, (void*)X, (void*)Y, (void*)Gb, (void*)dense, (void*)d_h, (void*)d_i, (void*)terms, (void*)nterms, (void*)done, (void*)d_err})
            if (q) cudaFree(q);
    };
#define CUC(call)                                                                                          \
    do {                                                                                                   \
        cudaError_t e_ = (call);                                                                           \
        if (e_ != cudaSuccess) {                                                                           \
            rc = fail(ctx, e_ == cudaErrorMemoryAllocation ? QFS_ENOMEM : QFS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
            cleanup();                                                                                     \
            return rc;                                                                                     \
        }                                                                                                  \
    } while (0)
    CUC(cudaMalloc(&d_c, B * 35));
    CUC(cudaMemcpy(d_c, coeffs, B * 35, cudaMemcpyDefault));
    CUC(cudaMalloc(&d_h, B));
    CUC(cudaMalloc(&d_i, B));
    CUC(cudaMalloc(&X, chunk * boxsize));
    CUC(cudaMalloc(&Y, chunk * boxsize));
    CUC(cudaMalloc(&Gb, chunk * boxsize));
    CUC(cudaMalloc(&terms, chunk * QFS_LIT_MAXTERMS * sizeof(LitTerm)));
    CUC(cudaMalloc(&nterms, chunk * sizeof(int)));
    CUC(cudaMalloc(&done, chunk * sizeof(int)));
    CUC(cudaMalloc(&d_err, sizeof(int)));
    CUC(cudaMemset(d_err, 0, sizeof(int)));
    if (g_out || delta_out) CUC(cudaMalloc(&dense, chunk * (delta_out ? L : N)));
    for (size_t first = 0; first < B; first += chunk) {
        const unsigned cnt = (unsigned)std::min(chunk, B - first);
        auto grid = [&](int deg) { return dim3((unsigned)((deg + 1) * (deg + 1)), cnt); };
        uint8_t *cur = X, *other = Y;
        // g = f^(p-1) mod p
        k_lit_load<<<cnt, 32>>>(d_c, (int)first, p, W, boxsize, cur, d_err);
        CUC(cudaMemsetAsync(nterms, 0, cnt * sizeof(int)));
        k_lit_terms<<<grid(4), 32>>>(cur, 4, W, boxsize, terms, nterms);
        for (int k = 2; k <= p - 1; ++k) {
            k_lit_mul<<<grid(4 * k), QFS_LIT_NT>>>(cur, 4 * (k - 1), terms, nterms, 4, W, boxsize, other, p, nullptr);
            std::swap(cur, other);
        }
        CUC(cudaMemcpyAsync(Gb, cur, cnt * boxsize, cudaMemcpyDeviceToDevice));
        if (g_out) {
            k_lit_dense<<<grid(d), 32>>>(Gb, d, W, boxsize, dense, N);
            CUC(cudaMemcpy(g_out + first * N, dense, cnt * N, cudaMemcpyDefault));
        }
        k_lit_check<<<(cnt + 127) / 128, 128>>>(Gb, p, W, boxsize, 0, bound, (int)first, (int)cnt, d_h, d_i, done);
        // Delta = ((lift g)^p - sum of the p-th powers of its terms) / p mod p; surfaces already decided are skipped unless Delta was asked for
        const int* skip = delta_out ? nullptr : done;
        CUC(cudaMemsetAsync(nterms, 0, cnt * sizeof(int)));
        k_lit_terms<<<grid(d), 32>>>(Gb, d, W, boxsize, terms, nterms);
        for (int k = 2; k <= p; ++k) {
            k_lit_mul<<<grid(d * k), QFS_LIT_NT>>>(cur, d * (k - 1), terms, nterms, d, W, boxsize, other, p * p, skip);
            std::swap(cur, other);
        }
        k_lit_carry<<<grid(D), 64>>>(cur, Gb, p, d, W, boxsize, d_err, skip);
        if (delta_out) {
            k_lit_dense<<<grid(D), 64>>>(cur, D, W, boxsize, dense, L);
            CUC(cudaMemcpy(delta_out + first * L, dense, cnt * L, cudaMemcpyDefault));
        }
        // g <- u(Delta g)
        uint8_t *ga = Gb, *gb = other;
        for (int step = 1; step <= bound - 1; ++step) {
            k_lit_step<<<grid(d), 32>>>(cur, ga, gb, done, p, d, W, boxsize);
            std::swap(ga, gb);
            k_lit_check<<<(cnt + 127) / 128, 128>>>(ga, p, W, boxsize, step, bound, (int)first, (int)cnt, d_h, d_i, done);
        }
        CUC(cudaGetLastError());
    }
    CUC(cudaMemcpy(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
    CUC(cudaMemcpy(heights, d_h, B, cudaMemcpyDefault));
    CUC(cudaMemcpy(iters, d_i, B, cudaMemcpyDefault));
    CUC(cudaDeviceSynchronize());
#undef CUC
    cleanup();
    if (h_err & QFS_ERRBIT_INPUT) return fail(ctx, QFS_EINVAL, "input violates a precondition: a coefficient >= p or the zero form");
    if (h_err & QFS_ERRBIT_INVARIANT) return fail(ctx, QFS_EINVARIANT, "Witt-carry numerator not divisible by p");
    return QFS_OK;
}

int qfs_debug_occupancy(const qfs_ctx* ctx, int ctas_per_sm[4])
{
    if (!ctx || !ctas_per_sm) return QFS_EINVAL;
    for (int i = 0; i < 4; ++i) ctas_per_sm[i] = ctx->occ[i];
    return QFS_OK;
}

int qfs_debug_fill_workspaces(qfs_ctx* ctx, int byte)
{
    if (!ctx) return QFS_EINVAL;
    DeviceGuard guard_(ctx->device);
    DevBuf* bufs[] = {&ctx->g, &ctx->h, &ctx->A, &ctx->E, &ctx->delta, &ctx->M, &ctx->v1, &ctx->vacc, &ctx->tapA, &ctx->tapB,
                      &ctx->coeffs, &ctx->heights, &ctx->iters, &ctx->list, &ctx->chain_scratch, &ctx->ecm, &ctx->hbox};
    for (DevBuf* b : bufs)
        if (b->ptr) CU(cudaMemsetAsync(b->ptr, byte, b->cap, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return QFS_OK;
}

int qfs_sample_quartics(qfs_ctx* ctx, const uint64_t state_inc[4], size_t count, uint8_t* coeffs, int* clean)
{
    if (!ctx) return QFS_EINVAL;
    if (!state_inc || !clean || (count && !coeffs)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    *clean = 1;
    if (count == 0) return QFS_OK;
    DeviceGuard guard_(ctx->device);
    const bool out_dev = is_device_ptr(coeffs);
    uint8_t* d_out = coeffs;
    if (!out_dev) { CU(ctx->coeffs.reserve(count * 35)); d_out = ctx->coeffs.as<uint8_t>(); }
    int* d_flags = ctx->flags.as<int>();
    CU(cudaMemsetAsync(d_flags, 0, 4 * sizeof(int), ctx->stream));
    k_sample_quartics<<<(unsigned)((count + 127) / 128), 128, 0, ctx->stream>>>(U128{state_inc[0], state_inc[1]}, U128{state_inc[2], state_inc[3]},
                                                                               (uint32_t)ctx->p, count, d_out, d_flags);
    CU(cudaGetLastError());
    if (!out_dev) CU(cudaMemcpyAsync(coeffs, d_out, count * 35, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(ctx->h_flags, d_flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *clean = ctx->h_flags[0] ? 0 : 1;
    return QFS_OK;
}

int qfs_export_matrix(qfs_ctx* ctx, const uint8_t* coeffs, size_t B, uint16_t* M16)
{
    if (!ctx) return QFS_EINVAL;
    if (B && (!coeffs || !M16)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    QFS_FOR_PRIME(ctx->p, run_export_matrix, ctx, coeffs, B, M16)
}

int qfs_stage_matvec_chain(qfs_ctx* ctx, const uint8_t* M, const uint8_t* v0, size_t B, int max_steps, uint8_t* trace,
                           int8_t* heights, int8_t* iters)
{
    if (!ctx) return QFS_EINVAL;
    if (B && (!M || !v0 || !heights || !iters)) return fail(ctx, QFS_EINVAL, "NULL buffer");
    QFS_FOR_PRIME(ctx->p, run_stage_chain, ctx, M, v0, B, max_steps, trace, heights, iters)
}

}  // extern "C"
