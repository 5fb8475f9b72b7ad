// qfs_free.cuh -- the operator iteration WITHOUT the operator matrix ("matrix-free" mode; the on-device
// counterpart of the reference's polynomial iteration height_naive, height.py:97-116).
//
// The contract path of this library builds M and streams it (qfs_matrix_staged.cuh, qfs_chain.cuh), as the
// reference's height_matrix does.  This kernel is the independent cross-check on the device, and an
// optional fast mode: with Delta = phi(A) - phi(h) E and u semilinear
// (u(phi(a) X) = a u(X)),
//     u(Delta g_k) = A * g_k[cap]  -  h * u(E g_k),
// and inside the loop g_k[cap] = 0 (otherwise the height has been decided), so
//     g_{k+1} = - h * q_k,     q_k = u(E g_k)  a quartic:  q_k[r] = sum_J E[J] g_k[p r + (p-1) 1 - J],  |r| = 4.
// One step costs 35 C(4p+3,3) + 35 C(4p-1,3) multiply-adds (96 k at p = 5, 260 k at p = 7) instead of a pass
// over the N x N matrix, and needs f^(p-2), f^(p-1) and E = Delta_1(f) only -- no Delta, no M.
// Same semantics as the loop of height.py:135-144 (iterations, bound, first k with g_k[cap] != 0).
#pragma once
#include "qfs_shape.cuh"

template <int P>
struct FreeCfg {
    using S = Shape<P>;
    static constexpr int NT = 256;
    static constexpr int RBD = (S::d + 1) * (S::d + 1);    // row bases of basis(d)
    static constexpr int RBH = (S::dh + 1) * (S::dh + 1);  // row bases of basis(dh)
    static constexpr int SMEM = 2 * S::pitch + S::Nh_pad + S::NE_pad + 4 * (RBD + RBH) + 64;
};

// unrank_E: monomials of degree 4p (level p of the unrank table), unrank_d: degree d = 4(p-1) (level p-1).
// list: original indices of the surfaces of this chunk (NULL: identity).
template <int P>
__global__ void __launch_bounds__(FreeCfg<P>::NT)
k_free(const uint8_t* __restrict__ g_all, const uint8_t* __restrict__ h_all, const uint8_t* __restrict__ E_all,
       const uint32_t* __restrict__ unrank_E, const uint32_t* __restrict__ unrank_d, const uint32_t* __restrict__ list,
       int max_steps, int8_t* __restrict__ heights, int8_t* __restrict__ iters)
{
    using S = Shape<P>;
    using C = FreeCfg<P>;
    extern __shared__ __align__(16) uint8_t smem[];
    uint8_t* sga = smem;
    uint8_t* sgb = smem + S::pitch;
    uint8_t* sh = sgb + S::pitch;
    uint8_t* sE = sh + S::Nh_pad;
    int* rbd = reinterpret_cast<int*>(sE + S::NE_pad);
    int* rbh = rbd + C::RBD;
    __shared__ int sq[35];
    const int slot = blockIdx.x, tid = threadIdx.x, lane = tid & 31;

    for (int i = tid; i < S::pitch / 16; i += C::NT)
        reinterpret_cast<uint4*>(sga)[i] = reinterpret_cast<const uint4*>(g_all + (size_t)slot * S::pitch)[i];
    for (int i = tid; i < S::Nh_pad / 16; i += C::NT)
        reinterpret_cast<uint4*>(sh)[i] = reinterpret_cast<const uint4*>(h_all + (size_t)slot * S::Nh_pad)[i];
    for (int i = tid; i < S::NE_pad / 16; i += C::NT)
        reinterpret_cast<uint4*>(sE)[i] = reinterpret_cast<const uint4*>(E_all + (size_t)slot * S::NE_pad)[i];
    for (int e = tid; e < C::RBD; e += C::NT) {
        const int a1 = e / (S::d + 1), a2 = e - a1 * (S::d + 1);
        rbd[e] = (a1 + a2 <= S::d) ? qrowbase(S::d, a1, a2) : 0;
    }
    for (int e = tid; e < C::RBH; e += C::NT) {
        const int a1 = e / (S::dh + 1), a2 = e - a1 * (S::dh + 1);
        rbh[e] = (a1 + a2 <= S::dh) ? qrowbase(S::dh, a1, a2) : 0;
    }
    __syncthreads();

    int height = 0, it = 0;
    for (int step = 1; step <= max_steps; ++step) {
        if (tid < 35) sq[tid] = 0;
        __syncthreads();
        // q[r] = sum_J E[J] g[p r + (p-1) - J]
        int acc[35];
#pragma unroll
        for (int r = 0; r < 35; ++r) acc[r] = 0;
        for (int J = tid; J < S::NE; J += C::NT) {
            const int e = sE[J];
            if (e == 0) continue;
            const uint32_t m = unrank_E[J];
            const int J1 = m & 255, J2 = (m >> 8) & 255, J3 = m >> 16, J4 = S::dE - J1 - J2 - J3;
            int r = 0;
#pragma unroll
            for (int r1 = 0; r1 <= 4; ++r1)
#pragma unroll
                for (int r2 = 0; r2 <= 4 - r1; ++r2)
#pragma unroll
                    for (int r3 = 0; r3 <= 4 - r1 - r2; ++r3) {
                        const int r4 = 4 - r1 - r2 - r3;
                        const int a1 = P * r1 + P - 1 - J1, a2 = P * r2 + P - 1 - J2, a3 = P * r3 + P - 1 - J3,
                                  a4 = P * r4 + P - 1 - J4;
                        if ((a1 | a2 | a3 | a4) >= 0) acc[r] += e * (int)sga[rbd[a1 * (S::d + 1) + a2] + a3];
                        ++r;
                    }
        }
#pragma unroll
        for (int r = 0; r < 35; ++r) {
            const int t = __reduce_add_sync(0xffffffffu, acc[r]);
            if (lane == 0 && t) atomicAdd(&sq[r], t);
        }
        __syncthreads();
        if (tid < 35) sq[tid] = sq[tid] % P;
        __syncthreads();
        // g_next[I] = - sum_r q[r] h[I - r]
        for (int I = tid; I < S::N; I += C::NT) {
            const uint32_t m = unrank_d[I];
            const int i1 = m & 255, i2 = (m >> 8) & 255, i3 = m >> 16, i4 = S::d - i1 - i2 - i3;
            int s = 0, r = 0;
#pragma unroll
            for (int r1 = 0; r1 <= 4; ++r1)
#pragma unroll
                for (int r2 = 0; r2 <= 4 - r1; ++r2)
#pragma unroll
                    for (int r3 = 0; r3 <= 4 - r1 - r2; ++r3) {
                        const int r4 = 4 - r1 - r2 - r3;
                        const int u1 = i1 - r1, u2 = i2 - r2, u3 = i3 - r3, u4 = i4 - r4;
                        if ((u1 | u2 | u3 | u4) >= 0) s += sq[r] * (int)sh[rbh[u1 * (S::dh + 1) + u2] + u3];
                        ++r;
                    }
            const int v = s % P;
            sgb[I] = (uint8_t)(v ? P - v : 0);
        }
        __syncthreads();
        { uint8_t* t = sga; sga = sgb; sgb = t; }
        ++it;
        if (sga[S::cap] != 0) { height = step + 1; break; }  // uniform: every thread reads the same byte
    }
    if (tid == 0) {
        const uint32_t sid = list ? list[slot] : (uint32_t)slot;
        heights[sid] = (int8_t)height;
        iters[sid] = (int8_t)it;
    }
}
