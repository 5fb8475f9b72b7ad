// qfs_matrix.cuh -- stage 3: the operator matrix of g -> u(Delta * g), written straight to HBM,
// with the first operator application v1 = M g fused into the producer.
//
// Replaces build_mts / mts_wics (mtsmatrix.py:287-295, 249-281; the TRIV and MERGE variants
// :173-246 produce the same entries) and the first pass of the loop in height.py:135-144.
// The reference scatters every Delta term into its matching (row, column) cells with np.add.at;
// here the map is inverted into a pure gather -- each cell has exactly one source (SURVEY.md
// section 7.1, verified in tests/model_factorized.py):
//     M[r, c] = Delta[p*r + (p-1) - c]      if every component is >= 0, else 0,
// for r, c in basis(d,4), d = 4(p-1).  No atomics, no hash table, no index search.
//
// Layout.  M is row-major with pitch = N rounded up to 16 bytes (pad columns are zero), one byte
// per entry (residues < p).  With Delta in "lex43g" order (qfs_shape.cuh) a column run (c1,c2,*)
// of row r = (r1,r2,r3,r4) is a forward copy:
//     M[r, (c1,c2,c3)] = Delta43g[ gbase(I1,I2) + I4 ],  I1 = p r1+p-1-c1, I2 = p r2+p-1-c2,
//     I4 = p r4 + p-1 - c4 = (p-1 - len_c) + c3 + p t,   len_c = d-c1-c2,  t = R - r3,  R = d-r1-r2.
// So for a whole ROW GROUP (r1,r2 fixed, t = 0..R) every column has a fixed source offset plus the
// row-uniform offset p*t, and the sources of one column run form a WINDOW of len_c + 1 + p*R
// consecutive bytes of one Delta run.  I3 < 0 or I4 < 0 (no match) reads a guard zero; I1 < 0,
// I2 < 0 or a pad column reads a zero region: no predicates in the inner loop.
//
// Mapping (v3).  One CTA per (row group, slice of surfaces).  Everything that depends on the group
// only -- the window of every column run, its slot in shared memory, the shared-memory address of
// every column -- is computed once per CTA.  Per surface the windows are staged into shared memory
// with 16-byte cp.async copies (double-buffered: the next surface's windows arrive while the
// current one is gathered), then every thread builds its words of each row from four LDS.U8 and
// stores them as aligned 32-bit words (128 bytes per warp).  A warp-wide byte gather touches ~20
// different column runs; from L1 that cost ~14 sectors per request (profiles/r1_matrix_v2.txt),
// from shared memory it is a 2-3-way bank conflict.  Groups with many rows are processed in passes
// of at most TB rows so that the windows fit.
//
// Fused first step.  When FUSE, each thread keeps its words of v0 = g in registers, adds
// dp4a(M word, v0 word) per row into a [row][lane] shared accumulator, and the CTA finishes the
// dot products of its rows:  v1[row] = (M g)[row] mod p.  About 80% of the surfaces that reach
// this stage are decided by v1[cap] != 0 (height 2), so their M is never read back.
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct MatrixCfg {
    using S = Shape<P>;
    static constexpr int WORDS = S::pitch / 4;
    static constexpr int NT = (P >= 11) ? 800 : (P >= 5 ? 256 : 64);
    static constexpr int WPT = (WORDS + NT - 1) / NT;  // words per thread: 1 (p=3,5), 3 (p=7), 4 (p=11)
    static constexpr int MAXROWS = S::d + 1;
    static constexpr int NR = S::ngroups;                                  // column runs (c1,c2)
    static constexpr int TB = (P >= 11) ? 8 : (P >= 7 ? 13 : S::d + 1);    // rows per pass
    static constexpr int NBUF = (P >= 11) ? 1 : 2;                         // window buffers
    static constexpr int SLICE = (P >= 11) ? 8 : (P >= 7 ? 16 : 64);       // surfaces per CTA
    static constexpr int ZRS = qround16(P * (TB - 1) + 1);                 // zero region of a buffer
    static constexpr int BUF = ZRS + qround16(S::N + NR * (P * (TB - 1) + 30));
    static constexpr int OFF_TAB = 0;                                      // int32 [4][NR]: src, dst, nch, col
    static constexpr int OFF_BUF = qround16(16 * NR);
    static constexpr int SMEM = OFF_BUF + NBUF * BUF;
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src)
{
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int IMM>
__device__ __forceinline__ uint32_t lds_u8(uint32_t saddr)
{
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(saddr), "n"(IMM));
    return v;
}

// One row of the group for every word this thread owns: gather, merge, store, (dot).
// ap[j][k]: shared-space address of the source byte of column 4*word_j + k for the block's first row.
template <int P, bool FUSE, int U>
__device__ __forceinline__ void matrix_row(const uint32_t (&ap)[MatrixCfg<P>::WPT][4], uint32_t* dst, uint32_t* dstL,
                                           const uint32_t (&vw)[MatrixCfg<P>::WPT], int* accp)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    uint32_t part = 0;
#pragma unroll
    for (int j = 0; j < C::WPT; ++j) {
        const uint32_t b0 = lds_u8<P * U>(ap[j][0]), b1 = lds_u8<P * U>(ap[j][1]);
        const uint32_t b2 = lds_u8<P * U>(ap[j][2]), b3 = lds_u8<P * U>(ap[j][3]);
        const uint32_t word = (b0 | (b1 << 8)) | ((b2 << 16) | (b3 << 24));
        if (j < C::WPT - 1) dst[-U * (S::pitch / 4) + j * C::NT] = word;
        else dstL[-U * (S::pitch / 4)] = word;  // the last word index is clamped for threads past the row end
        if (FUSE) part = __dp4a(word, vw[j], part);
    }
    if (FUSE) atomicAdd(accp - U * 32, (int)part);
}

// colinfo[c] = c1 | c2<<8 | c3<<16 for c < N, 0xFFFFFFFF for pad columns.
// groups[g] = r1 | r2<<8, sorted by decreasing group size (longest CTAs first).
// runs[rc] = c1 | c2<<8 of the rc-th column run in lex order, rc = c1(d+1) - c1(c1-1)/2 + c2.
// FUSE: also compute v1 = M v0 mod p (v0_all, v1_all with stride pitch per surface).
template <int P, bool FUSE>
__global__ void __launch_bounds__(MatrixCfg<P>::NT)
k_matrix(const uint8_t* __restrict__ delta_all, const uint32_t* __restrict__ colinfo,
         const uint16_t* __restrict__ groups, const uint16_t* __restrict__ runs, uint8_t* __restrict__ M_all,
         const uint8_t* __restrict__ v0_all, uint8_t* __restrict__ v1_all, int count)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ int s_acc[C::MAXROWS * 32];
    int* t_src = reinterpret_cast<int*>(smem + C::OFF_TAB);
    int* t_dst = t_src + C::NR;
    int* t_nch = t_dst + C::NR;
    int* t_col = t_nch + C::NR;
    uint8_t* bufs = smem + C::OFF_BUF;

    const int grp = groups[blockIdx.x];
    const int r1 = grp & 255, r2 = grp >> 8;
    const int R = S::d - r1 - r2;
    const int row0 = qrowbase(S::d, r1, r2);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s_begin = blockIdx.y * C::SLICE;
    const int s_end = min(count, s_begin + C::SLICE);

    int wj[C::WPT];
#pragma unroll
    for (int j = 0; j < C::WPT; ++j) wj[j] = min(tid + j * C::NT, C::WORDS - 1);
    if (FUSE)
        for (int i = tid; i < C::MAXROWS * 32; i += C::NT) s_acc[i] = 0;

#pragma unroll 1
    for (int t0 = 0; t0 <= R; t0 += C::TB) {
        const int nt = min(C::TB, R + 1 - t0);  // rows t0 .. t0+nt-1 of the walk (r3 = R - t)
        __syncthreads();
        // ---- per-pass tables (surface-independent) ------------------------------------------
        for (int i = tid; i < C::NBUF * C::BUF / 16; i += C::NT) reinterpret_cast<uint4*>(bufs)[i] = make_uint4(0, 0, 0, 0);
        for (int rc = tid; rc < C::NR; rc += C::NT) {
            const int cc = runs[rc];
            const int c1 = cc & 255, c2 = cc >> 8;
            const int lenc = S::d - c1 - c2;
            const int I1 = P * r1 + P - 1 - c1, I2 = P * r2 + P - 1 - c2;
            int size = 0, src = 0, nch = 0, col = 0xFFFF, dsto = 0;
            if (I1 >= 0 && I2 >= 0 && I1 + I2 <= S::D) {
                const int gb = S::gbase(I1, I2), n2 = S::D - I1 - I2;
                const int a_lo = gb + (P - 1) - lenc + P * t0;   // source of (c3 = 0, t = t0)
                const int a_hi = a_lo + lenc + P * (nt - 1);     // source of (c3 = len_c, t = t0+nt-1)
                const int c_lo = max(a_lo, gb), c_hi = min(a_hi, gb + n2);  // the part that is real data
                if (c_lo <= c_hi) {
                    const int w_lo = a_lo & ~15, w_hi = (a_hi + 16) & ~15;
                    const int k_lo = max(w_lo, c_lo & ~15), k_hi = min(w_hi, (c_hi + 16) & ~15);
                    size = w_hi - w_lo;
                    src = k_lo;
                    nch = (k_hi - k_lo) >> 4;
                    dsto = k_lo - w_lo;
                    col = a_lo - w_lo;  // < 16
                }
            }
            t_src[rc] = src;
            t_dst[rc] = size;   // slot size for now; turned into the slot offset by the scan below
            t_nch[rc] = nch;
            t_col[rc] = col | (dsto << 16);
        }
        __syncthreads();
        if (warp == 0) {  // exclusive scan of the slot sizes -> slot offsets (after the zero region)
            int carry = C::ZRS;
            for (int base = 0; base < C::NR; base += 32) {
                const int rc = base + lane;
                const int v = rc < C::NR ? t_dst[rc] : 0;
                int incl = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                if (rc < C::NR) {
                    const int off = carry + incl - v;
                    const int cd = t_col[rc];
                    t_dst[rc] = off + (cd >> 16);                                    // first copied chunk
                    t_col[rc] = (cd & 0xFFFF) == 0xFFFF ? 0 : off + (cd & 0xFFFF);  // byte of (c3 = 0, t = t0); 0 = zero region
                }
                carry += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        __syncthreads();
        // shared-memory offsets (inside a buffer) of this thread's columns at t = t0
        uint32_t sp[C::WPT][4];
#pragma unroll
        for (int j = 0; j < C::WPT; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t info = colinfo[4 * wj[j] + k];
                uint32_t a = 0;
                if (info != 0xFFFFFFFFu) {
                    const int c1 = info & 255, c2 = (info >> 8) & 255, c3 = info >> 16;
                    const int col = t_col[c1 * (S::d + 1) - ((c1 * (c1 - 1)) >> 1) + c2];
                    if (col) a = col + c3;
                }
                sp[j][k] = a;
            }

        // ---- surfaces of the slice ---------------------------------------------------------------
        auto stage = [&](int slot, uint8_t* buf) {
            const uint8_t* dl = delta_all + (size_t)slot * S::Lg_pad;
            for (int rc = tid; rc < C::NR; rc += C::NT) {
                const int n = t_nch[rc];
                const uint8_t* s = dl + t_src[rc];
                uint8_t* d = buf + t_dst[rc];
                for (int c = 0; c < n; ++c) cp_async16(d + 16 * c, s + 16 * c);
            }
            cp_async_commit();
        };
        if (C::NBUF == 2 && s_begin < s_end) stage(s_begin, bufs);
        const int nblk = nt / 4, nrem = nt - 4 * nblk;
        for (int slot = s_begin; slot < s_end; ++slot) {
            const uint8_t* win;
            if (C::NBUF == 2) {
                const int b = (slot - s_begin) & 1;
                if (slot + 1 < s_end) { stage(slot + 1, bufs + (b ^ 1) * C::BUF); cp_async_wait<1>(); }
                else cp_async_wait<0>();
                win = bufs + b * C::BUF;
            } else {
                stage(slot, bufs);
                cp_async_wait<0>();
                win = bufs;
            }
            __syncthreads();
            uint32_t ap[C::WPT][4];
            {
                const uint32_t wbase = (uint32_t)__cvta_generic_to_shared(win);
#pragma unroll
                for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                    for (int k = 0; k < 4; ++k) ap[j][k] = wbase + sp[j][k];
            }
            uint32_t* const rowT = reinterpret_cast<uint32_t*>(M_all + (size_t)slot * ((size_t)S::N * S::pitch) +
                                                               (size_t)(row0 + R - t0) * S::pitch);
            uint32_t* dst = rowT + tid;
            uint32_t* dstL = rowT + wj[C::WPT - 1];
            uint32_t vw[C::WPT];
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
                vw[j] = (FUSE && tid + j * C::NT < C::WORDS) ? reinterpret_cast<const uint32_t*>(v0_all + (size_t)slot * S::pitch)[wj[j]] : 0u;
            int* accp = &s_acc[(R - t0) * 32 + lane];
            // Rows are walked from t = t0 upwards (r3 = R - t downwards) four at a time, so that the source
            // offset p*t, the destination offset -t*pitch and the accumulator offset are immediates.
#pragma unroll 1
            for (int b = 0; b < nblk; ++b) {
                matrix_row<P, FUSE, 0>(ap, dst, dstL, vw, accp);
                matrix_row<P, FUSE, 1>(ap, dst, dstL, vw, accp);
                matrix_row<P, FUSE, 2>(ap, dst, dstL, vw, accp);
                matrix_row<P, FUSE, 3>(ap, dst, dstL, vw, accp);
#pragma unroll
                for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                    for (int k = 0; k < 4; ++k) ap[j][k] += 4 * P;
                dst -= 4 * (S::pitch / 4);
                dstL -= 4 * (S::pitch / 4);
                accp -= 4 * 32;
            }
#pragma unroll 1
            for (int b = 0; b < nrem; ++b) {
                matrix_row<P, FUSE, 0>(ap, dst, dstL, vw, accp);
#pragma unroll
                for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                    for (int k = 0; k < 4; ++k) ap[j][k] += P;
                dst -= S::pitch / 4;
                dstL -= S::pitch / 4;
                accp -= 32;
            }
            __syncthreads();  // all rows gathered: the buffer may be refilled, the accumulators are complete
            if (FUSE) {
                for (int t = t0 + warp; t < t0 + nt; t += C::NT / 32) {
                    const int r3 = R - t;
                    uint32_t a = (uint32_t)s_acc[r3 * 32 + lane];
                    s_acc[r3 * 32 + lane] = 0;
#pragma unroll
                    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                    if (lane == 0) v1_all[(size_t)slot * S::pitch + row0 + r3] = (uint8_t)(a % (uint32_t)P);
                }
            }
        }
    }
}
