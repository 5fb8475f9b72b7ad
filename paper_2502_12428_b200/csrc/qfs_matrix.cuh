// qfs_matrix.cuh -- stage 3: the operator matrix of g -> u(Delta * g), written straight to HBM.
//
// Replaces build_mts / mts_wics (mtsmatrix.py:287-295, 249-281; the TRIV and MERGE variants
// :173-246 produce the same entries).  The reference scatters every Delta term into its matching
// (row, column) cells with np.add.at; here the map is inverted into a pure gather -- each cell has
// exactly one source (verified in tests/model_factorized.py):
//     M[r, c] = Delta[p*r + (p-1) - c]      if every component is >= 0, else 0,
// for r, c in basis(d,4), d = 4(p-1).  No atomics, no hash table, no index search.
//
// Layout.  M is row-major with pitch = N rounded up to 16 bytes (pad columns are zero), one byte
// per entry (residues < p).  With Delta in "lex43" order (qfs_shape.cuh) a column run (c1,c2,*) of
// row r = (r1,r2,r3,r4) is a forward copy:
//     M[r, (c1,c2,c3)] = Delta43[ rowbase(D,I1,I2) + I4 ],  I1 = p r1+p-1-c1, I2 = p r2+p-1-c2,
//     I4 = p r4 + p-1 - c4 = (p-1 - len_c) + c3 + p (R - r3),   len_c = d-c1-c2,  R = d-r1-r2,
// valid iff c_k <= p r_k + p-1 for k = 1..4.  So for a whole ROW GROUP (r1,r2 fixed, r3 = 0..R) every
// column has a fixed source address plus the row-uniform offset p(R-r3).
//
// Mapping (v1).  One CTA per (surface, row group).  A per-group table of run base addresses is
// built in shared memory; each thread then owns four consecutive columns (one aligned 32-bit
// store per row) and walks down the rows of the group with its four source addresses in registers.
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct MatrixCfg {
    using S = Shape<P>;
    static constexpr int NT = 256;
    static constexpr int RUNDIM = S::d + 1;
};

// colinfo[c] = (c1*(d+1)+c2) | c3<<16 for c < N, 0xFFFFFFFF for pad columns.
// groups[g] = r1 | r2<<8 for the g-th (r1,r2) pair in lex order.
template <int P>
__global__ void __launch_bounds__(MatrixCfg<P>::NT)
k_matrix(const uint8_t* __restrict__ delta_all, const uint32_t* __restrict__ colinfo,
         const uint16_t* __restrict__ groups, uint8_t* __restrict__ M_all, int count)
{
    using S = Shape<P>;
    using C = MatrixCfg<P>;
    __shared__ int s_runA0[C::RUNDIM * C::RUNDIM];
    constexpr int INVALID = INT32_MIN;

    const int slot = blockIdx.x / S::ngroups;
    if (slot >= count) return;
    const int grp = groups[blockIdx.x - slot * S::ngroups];
    const int r1 = grp & 255, r2 = grp >> 8;
    const int R = S::d - r1 - r2;
    const int row0 = qrowbase(S::d, r1, r2);
    const uint8_t* dl = delta_all + (size_t)slot * S::L_pad;
    uint8_t* Mrow = M_all + (size_t)slot * ((size_t)S::N * S::pitch) + (size_t)row0 * S::pitch;
    const int tid = threadIdx.x;

    for (int e = tid; e < C::RUNDIM * C::RUNDIM; e += C::NT) {
        const int c1 = e / C::RUNDIM, c2 = e - c1 * C::RUNDIM;
        const int I1 = P * r1 + P - 1 - c1, I2 = P * r2 + P - 1 - c2;
        const int lenc = S::d - c1 - c2;
        int a0 = INVALID;
        if (lenc >= 0 && I1 >= 0 && I2 >= 0 && I1 + I2 <= S::D) a0 = qrowbase(S::D, I1, I2) + (P - 1) - lenc;
        s_runA0[e] = a0;
    }
    __syncthreads();

    for (int w = tid; w < S::pitch / 4; w += C::NT) {
        int addr[4], c3v[4], c4v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t info = colinfo[4 * w + k];
            addr[k] = INVALID;
            c3v[k] = 0;
            c4v[k] = 0;
            if (info != 0xFFFFFFFFu) {
                const int run = info & 0xFFFF, c3 = info >> 16;
                const int a0 = s_runA0[run];
                const int c1 = run / C::RUNDIM, c2 = run - c1 * C::RUNDIM;
                c3v[k] = c3;
                c4v[k] = S::d - c1 - c2 - c3;
                if (a0 != INVALID) addr[k] = a0 + c3;
            }
        }
        uint8_t* dst = Mrow + 4 * w;
        for (int r3 = 0; r3 <= R; ++r3) {
            const int off = P * (R - r3);
            const int t3 = P * r3 + P - 1, t4 = off + P - 1;
            uint32_t word = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t b = 0;
                if (addr[k] != INVALID && c3v[k] <= t3 && c4v[k] <= t4) b = dl[addr[k] + off];
                word |= b << (8 * k);
            }
            *reinterpret_cast<uint32_t*>(dst + (size_t)r3 * S::pitch) = word;
        }
    }
}
