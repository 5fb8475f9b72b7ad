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
// Layout.  M is row-major with pitch = N rounded up to 128 bytes (pad columns are zero), one byte
// per entry (residues < p).  With Delta in "lex43g" order (qfs_shape.cuh) a column run (c1,c2,*)
// of row r = (r1,r2,r3,r4) is a forward copy:
//     M[r, (c1,c2,c3)] = Delta43g[ gbase(I1,I2) + I4 ],  I1 = p r1+p-1-c1, I2 = p r2+p-1-c2,
//     I4 = p r4 + p-1 - c4 = (p-1 - len_c) + c3 + p t,   len_c = d-c1-c2,  t = R - r3,  R = d-r1-r2.
// So for a whole ROW GROUP (r1,r2 fixed, t = 0..R) every column has a fixed source offset plus the
// row-uniform offset p*t, and the sources of one column run form a WINDOW of len_c + 1 + p*R
// consecutive bytes of one Delta run.  I3 < 0 or I4 < 0 (no match) reads a guard zero; I1 < 0,
// I2 < 0 or a pad column reads a zero region: no predicates in the inner loop.
//
// Mapping (v4).  One CTA per (row group, slice of quads).  A quad = four surfaces whose Delta arrays
// are byte-interleaved (qfs_shape.cuh): one aligned 32-bit load at 4*(source offset) returns the
// entry of all four surfaces, so a thread that owns four consecutive columns issues four LDG.32,
// transposes the 4x4 bytes (8 PRMT) and stores one aligned word into each of the four matrices --
// a quarter of the load instructions and of the L1 wavefronts of a per-surface byte gather
// (profiles/: v2 gathered bytes through L1 at ~14 sectors per request, v3 through shared memory at
// ~3.2-way bank conflicts; both stalled at 1.7 TB/s of matrix writes).  The per-column source
// offsets depend on the group only: they are computed once per CTA into registers and reused for
// every quad of the slice and every row of the group.  Thread t owns the words t, t+NT, ... of a
// row (coalesced 128-byte stores per warp and matrix).
//
// Fused first step.  When FUSE, each thread keeps its words of v0 = g (of the four surfaces) in
// registers, accumulates dp4a(M word, v0 word) per row; warp-wide sums (REDUX) go to a [surface][row]
// shared accumulator and the CTA finishes the dot products of its rows:  v1[row] = (M g)[row] mod p.  About 80% of the
// surfaces that reach this stage are decided by v1[cap] != 0 (height 2), so their M is never read back.
#pragma once
#include "qfs_delta.cuh"  // transpose4x4
#include "qfs_shape.cuh"

template <int P>
struct MatrixCfg {
    using S = Shape<P>;
    static constexpr int WORDS = S::pitch / 4;
    static constexpr int NT = (P >= 11) ? 800 : (P >= 5 ? 256 : 64);
    static constexpr int WPT = (WORDS + NT - 1) / NT;  // words per thread: 1 (p=3,5), 3 (p=7), 4 (p=11)
    static constexpr int MAXROWS = S::d + 1;
    static constexpr int SLICE = (P >= 11) ? 2 : (P >= 7 ? 4 : 16);  // quads per CTA
    static constexpr int UNROLL = (P >= 11) ? 2 : 4;                 // rows per block of the row walk
    static constexpr size_t MSTRIDE = (size_t)S::N * S::pitch;       // bytes of one matrix
};

// One row of the group, for every word this thread owns and the four surfaces of the quad.
// sp[j][k]: address of the interleaved source word of column 4*word_j + k for the block's first row.
template <int P, bool FUSE, int U>
__device__ __forceinline__ void matrix_row(const uint8_t* const (&sp)[MatrixCfg<P>::WPT][4], uint32_t* const (&dst)[4],
                                           int lastw, const uint32_t (&vw)[MatrixCfg<P>::WPT][4], int* accp, int lane)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    uint32_t part[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < C::WPT; ++j) {
        uint32_t in[4], out[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) in[k] = *reinterpret_cast<const uint32_t*>(sp[j][k] + 4 * P * U);
        transpose4x4(in, out);  // out[s] = the four columns of surface s
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            // the last word index is clamped for threads past the row end (same value stored twice)
            if (j < C::WPT - 1) dst[s][-U * (S::pitch / 4) + j * C::NT] = out[s];
            else dst[s][-U * (S::pitch / 4) + lastw] = out[s];
            if (FUSE) part[s] = __dp4a(out[s], vw[j][s], part[s]);
        }
    }
    if (FUSE) {  // warp-wide sums in hardware (REDUX), one shared atomic per warp, surface and row
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int tot = (int)__reduce_add_sync(0xffffffffu, part[s]);
            if (lane == 0) atomicAdd(accp + s * C::MAXROWS - U, tot);
        }
    }
}

// colinfo[c] = c1 | c2<<8 | c3<<16 for c < N, 0xFFFFFFFF for pad columns.
// groups[g] = r1 | r2<<8, sorted by decreasing group size (longest CTAs first).
// count = number of surfaces; quads beyond it are padded (their Delta is zero, their M/v1 slots exist).
// FUSE: also compute v1 = M v0 mod p (v0_all, v1_all with stride pitch per surface).
template <int P, bool FUSE>
__global__ void __launch_bounds__(MatrixCfg<P>::NT)
k_matrix(const uint8_t* __restrict__ delta_all, const uint32_t* __restrict__ colinfo,
         const uint16_t* __restrict__ groups, uint8_t* __restrict__ M_all, const uint8_t* __restrict__ v0_all,
         uint8_t* __restrict__ v1_all, int count)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    __shared__ int s_acc[FUSE ? 4 * C::MAXROWS : 1];  // [surface][r3]

    const int grp = groups[blockIdx.x];
    const int r1 = grp & 255, r2 = grp >> 8;
    const int R = S::d - r1 - r2;
    const int row0 = qrowbase(S::d, r1, r2);
    const int tid = threadIdx.x, lane = tid & 31;
    const int nquads = (count + 3) >> 2;
    const int q_begin = blockIdx.y * C::SLICE;
    const int q_end = min(nquads, q_begin + C::SLICE);

    // Source pointers of this thread's columns for the first quad of the slice, row r3 = R (t = 0).
    // Threads past the last word duplicate the last word (same value stored twice, dot weight 0).
    const uint8_t* sp[C::WPT][4];
    int wj[C::WPT];
#pragma unroll
    for (int j = 0; j < C::WPT; ++j) {
        const int w = min(tid + j * C::NT, C::WORDS - 1);
        wj[j] = w;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            int a = 0;  // the leading zero pad
            const uint32_t info = colinfo[4 * w + k];
            if (info != 0xFFFFFFFFu) {
                const int c1 = info & 255, c2 = (info >> 8) & 255, c3 = info >> 16;
                const int I1 = P * r1 + P - 1 - c1, I2 = P * r2 + P - 1 - c2;
                if (I1 >= 0 && I2 >= 0 && I1 + I2 <= S::D) a = S::gbase(I1, I2) + (P - 1) - (S::d - c1 - c2) + c3;
            }
            sp[j][k] = delta_all + (size_t)q_begin * S::quad_stride + 4 * (size_t)a;
        }
    }
    const int lastw = wj[C::WPT - 1] - tid;
    if (FUSE) {
        if (tid < 4 * C::MAXROWS) s_acc[tid] = 0;
        __syncthreads();
    }
    // Rows are walked from r3 = R down to 0 (t = R - r3 = 0..R), UNROLL at a time, so that the source
    // offset 4*p*t, the destination offset -t*pitch and the accumulator offset are immediates.
    const int nblk = (R + 1) / C::UNROLL, nrem = (R + 1) - nblk * C::UNROLL;
    int* const accR = &s_acc[FUSE ? R : 0];

    for (int quad = q_begin; quad < q_end; ++quad) {
        uint32_t* dst[4];
        uint32_t vw[C::WPT][4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const size_t slot = 4 * (size_t)quad + s;
            dst[s] = reinterpret_cast<uint32_t*>(M_all + slot * C::MSTRIDE + (size_t)(row0 + R) * S::pitch) + tid;
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
                vw[j][s] = (FUSE && tid + j * C::NT < C::WORDS) ? reinterpret_cast<const uint32_t*>(v0_all + slot * S::pitch)[wj[j]] : 0u;
        }
        int* accp = accR;
#pragma unroll 1
        for (int b = 0; b < nblk; ++b) {
            matrix_row<P, FUSE, 0>(sp, dst, lastw, vw, accp, lane);
            matrix_row<P, FUSE, 1>(sp, dst, lastw, vw, accp, lane);
            if (C::UNROLL == 4) {
                matrix_row<P, FUSE, 2>(sp, dst, lastw, vw, accp, lane);
                matrix_row<P, FUSE, 3>(sp, dst, lastw, vw, accp, lane);
            }
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) sp[j][k] += C::UNROLL * 4 * P;
#pragma unroll
            for (int s = 0; s < 4; ++s) dst[s] -= C::UNROLL * (S::pitch / 4);
            accp -= C::UNROLL;
        }
        if (nrem > 0) matrix_row<P, FUSE, 0>(sp, dst, lastw, vw, accp, lane);
        if (C::UNROLL == 4) {
            if (nrem > 1) matrix_row<P, FUSE, 1>(sp, dst, lastw, vw, accp, lane);
            if (nrem > 2) matrix_row<P, FUSE, 2>(sp, dst, lastw, vw, accp, lane);
        }
        // next quad of the slice: undo the row walk, step one quad stride
#pragma unroll
        for (int j = 0; j < C::WPT; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) sp[j][k] += S::quad_stride - 4 * P * C::UNROLL * nblk;
        if (FUSE) {
            __syncthreads();
            if (tid < 4 * (R + 1)) {
                const int s = tid / (R + 1), r3 = tid - s * (R + 1);
                const uint32_t a = (uint32_t)s_acc[s * C::MAXROWS + r3];
                s_acc[s * C::MAXROWS + r3] = 0;
                v1_all[(4 * (size_t)quad + s) * S::pitch + row0 + r3] = (uint8_t)(a % (uint32_t)P);
            }
            __syncthreads();
        }
    }
}
