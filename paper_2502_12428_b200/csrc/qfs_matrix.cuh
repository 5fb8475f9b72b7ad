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
//     I4 = p r4 + p-1 - c4 = (p-1 - len_c) + c3 + p (R - r3),   len_c = d-c1-c2,  R = d-r1-r2.
// So for a whole ROW GROUP (r1,r2 fixed, r3 = 0..R) every column has a fixed source offset plus the
// row-uniform offset p(R-r3).  I3 < 0 or I4 < 0 (no match) reads a guard zero; I1 < 0, I2 < 0 or a
// pad column reads the leading zero pad.  The inner loop is therefore 4 byte loads, 3 merges and
// one aligned 32-bit store per four entries, with no predicate.
//
// Mapping (v2).  One CTA per (row group, slice of surfaces).  The per-column source offsets depend
// only on the group, so they are computed once per CTA into registers and reused for every
// surface of the slice and every row of the group.  Thread t owns the words t, t+NT, ... of a row
// (coalesced 128-byte stores per warp).
//
// Fused first step.  When v0 is given, each thread keeps its words of v0 = g in registers, adds
// dp4a(M word, v0 word) per row into a [row][lane] shared accumulator, and the CTA finishes the
// R+1 dot products of its rows:  v1[row] = (M g)[row] mod p.  About 80% of the surfaces that reach
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
    static constexpr int SLICE = (P >= 11) ? 4 : (P >= 7 ? 8 : 16);  // surfaces per CTA
    static constexpr int UNROLL = 4;                                 // rows per block of the row walk
};

// One row of the group for every word this thread owns: gather, merge, store, (dot).
template <int P, bool FUSE, int U>
__device__ __forceinline__ void matrix_row(const uint8_t* const (&sp)[MatrixCfg<P>::WPT][4], uint32_t* dst,
                                           uint32_t* dstL, const uint32_t (&vw)[MatrixCfg<P>::WPT], int* accp)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    uint32_t part = 0;
#pragma unroll
    for (int j = 0; j < C::WPT; ++j) {
        const uint32_t b0 = sp[j][0][P * U], b1 = sp[j][1][P * U];
        const uint32_t b2 = sp[j][2][P * U], b3 = sp[j][3][P * U];
        const uint32_t word = (b0 | (b1 << 8)) | ((b2 << 16) | (b3 << 24));
        if (j < C::WPT - 1) dst[-U * (S::pitch / 4) + j * C::NT] = word;
        else dstL[-U * (S::pitch / 4)] = word;  // the last word index is clamped for threads past the row end
        if (FUSE) part = __dp4a(word, vw[j], part);
    }
    if (FUSE) atomicAdd(accp - U * 32, (int)part);
}

// colinfo[c] = c1 | c2<<8 | c3<<16 for c < N, 0xFFFFFFFF for pad columns.
// groups[g] = r1 | r2<<8, sorted by decreasing group size (longest CTAs first).
// FUSE: also compute v1 = M v0 mod p (v0_all, v1_all with stride pitch per surface).
template <int P, bool FUSE>
__global__ void __launch_bounds__(MatrixCfg<P>::NT)
k_matrix(const uint8_t* __restrict__ delta_all, const uint32_t* __restrict__ colinfo,
         const uint16_t* __restrict__ groups, uint8_t* __restrict__ M_all, const uint8_t* __restrict__ v0_all,
         uint8_t* __restrict__ v1_all, int count)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    __shared__ int s_acc[C::MAXROWS * 32];

    const int grp = groups[blockIdx.x];
    const int r1 = grp & 255, r2 = grp >> 8;
    const int R = S::d - r1 - r2;
    const int row0 = qrowbase(S::d, r1, r2);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int s_begin = blockIdx.y * C::SLICE;
    const int s_end = min(count, s_begin + C::SLICE);

    // Source pointers of this thread's columns for the first surface of the slice, row r3 = R.
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
            sp[j][k] = delta_all + (size_t)s_begin * S::Lg_pad + a;
        }
    }
    if (FUSE) {
        for (int i = tid; i < C::MAXROWS * 32; i += C::NT) s_acc[i] = 0;
        __syncthreads();
    }
    // Rows are walked from r3 = R down to 0 (t = R - r3 = 0..R), UNROLL at a time, so that the source
    // offset p*t, the destination offset -t*pitch and the accumulator offset are immediates and the
    // per-row work is 4 loads + 3 merges + 1 store (+ dp4a and one shared atomic when fused).
    const int nblk = (R + 1) / C::UNROLL, nrem = (R + 1) - nblk * C::UNROLL;
    int* const accR = &s_acc[R * 32 + lane];

    for (int slot = s_begin; slot < s_end; ++slot) {
        uint32_t* const rowR = reinterpret_cast<uint32_t*>(M_all + (size_t)slot * ((size_t)S::N * S::pitch) +
                                                           (size_t)(row0 + R) * S::pitch);
        uint32_t* dst = rowR + tid;
        uint32_t* dstL = rowR + wj[C::WPT - 1];
        uint32_t vw[C::WPT];
#pragma unroll
        for (int j = 0; j < C::WPT; ++j)
            vw[j] = (FUSE && tid + j * C::NT < C::WORDS) ? reinterpret_cast<const uint32_t*>(v0_all + (size_t)slot * S::pitch)[wj[j]] : 0u;
        int* accp = accR;
#pragma unroll 1
        for (int b = 0; b < nblk; ++b) {
            matrix_row<P, FUSE, 0>(sp, dst, dstL, vw, accp);
            matrix_row<P, FUSE, 1>(sp, dst, dstL, vw, accp);
            matrix_row<P, FUSE, 2>(sp, dst, dstL, vw, accp);
            matrix_row<P, FUSE, 3>(sp, dst, dstL, vw, accp);
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) sp[j][k] += C::UNROLL * P;
            dst -= C::UNROLL * (S::pitch / 4);
            dstL -= C::UNROLL * (S::pitch / 4);
            accp -= C::UNROLL * 32;
        }
#pragma unroll 1
        for (int b = 0; b < nrem; ++b) {
            matrix_row<P, FUSE, 0>(sp, dst, dstL, vw, accp);
#pragma unroll
            for (int j = 0; j < C::WPT; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) sp[j][k] += P;
            dst -= S::pitch / 4;
            dstL -= S::pitch / 4;
            accp -= 32;
        }
        // next surface of the slice: undo the row walk, step one Delta stride
#pragma unroll
        for (int j = 0; j < C::WPT; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) sp[j][k] += S::Lg_pad - P * (R + 1);
        if (FUSE) {
            __syncthreads();
            for (int r3 = warp; r3 <= R; r3 += C::NT / 32) {
                uint32_t a = (uint32_t)s_acc[r3 * 32 + lane];
                s_acc[r3 * 32 + lane] = 0;
#pragma unroll
                for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (lane == 0) v1_all[(size_t)slot * S::pitch + row0 + r3] = (uint8_t)(a % (uint32_t)P);
            }
            __syncthreads();
        }
    }
}
