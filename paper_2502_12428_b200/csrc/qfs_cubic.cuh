// qfs_cubic.cuh -- heights of plane cubic curves (n = 3: a cubic form in x1..x3 over F_p, 10 coefficients),
// SURVEY.md section 8(f)4 "general n": the reference's drivers take any Calabi-Yau hypersurface
// (height.py:63-144; tests/test_height.py:131-140 exercises cubic curves), the quartic kernels of this library do not.
//
// One CTA per curve, any odd prime p <= 53 at run time, everything in shared memory; the operator matrices here are
// 91 x 91 (p = 5) ... 703 x 703 (p = 13), so there is nothing to stream: the kernel runs the matrix-free form of the
// iteration (qfs_free.cuh; the identities of DESIGN.md section 3 do not depend on the number of variables):
//     f_T = sum tau(a_J) x^J,  tau(a) = a^p mod p^2;   chain f_T^2 ... f_T^p mod p^2
//     h = f^(p-2), g = f^(p-1) (mod p),  E = Delta_1(f) = (f_T^p - phi(f_T)) / p mod p      (exact division, checked)
//     height 1 iff g[cap] != 0;  else  g <- -h * u(E g)  until g[cap] != 0  (height = steps + 1) or the bound.
// A degree-D form is a dense (D+1) x (D+1) triangle indexed by (a1, a2), a3 = D - a1 - a2, row stride W = 3p+1.
#pragma once
#include <stdint.h>

#include "qfs_shape.cuh"

#define QFS_CUBIC_MAXP 53
#define QFS_CUBIC_NT 128

// basis(3,3) in lex-ascending order, x1 most significant: index 0 = x3^3 ... 9 = x1^3 (monomials.py:182-196)
__constant__ uint8_t c_cubic_exp[10][3] = {{0, 0, 3}, {0, 1, 2}, {0, 2, 1}, {0, 3, 0}, {1, 0, 2},
                                            {1, 1, 1}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}, {3, 0, 0}};

__host__ __device__ inline size_t qfs_cubic_smem(int p) { const size_t W = 3 * (size_t)p + 1; return 8 * W * W + 64; }

__global__ void __launch_bounds__(QFS_CUBIC_NT)
k_cubic(const uint8_t* __restrict__ coeffs, int B, int p, int max_steps, int8_t* __restrict__ heights,
        int8_t* __restrict__ iters, int* __restrict__ err)
{
    extern __shared__ __align__(16) uint8_t smem[];
    const int W = 3 * p + 1, WW = W * W, psq = p * p;
    uint16_t* bufA = reinterpret_cast<uint16_t*>(smem);
    uint16_t* bufB = bufA + WW;
    uint8_t* sh = reinterpret_cast<uint8_t*>(bufB + WW);
    uint8_t* sga = sh + WW;
    uint8_t* sgb = sga + WW;
    uint8_t* sE = sgb + WW;
    __shared__ uint32_t fT[10];
    __shared__ int sq[10];
    __shared__ int s_bad;
    const int tid = threadIdx.x, lane = tid & 31, NT = QFS_CUBIC_NT;
    const int slot = blockIdx.x;
    if (slot >= B) return;

    if (tid == 0) s_bad = 0;
    if (tid < 10) {
        const uint32_t a = coeffs[(size_t)slot * 10 + tid];
        uint32_t t = 1;
        for (int k = 0; k < p; ++k) t = (t * a) % (uint32_t)psq;  // tau(a) = a^p mod p^2
        fT[tid] = (a < (uint32_t)p) ? t : 0u;
        if (a >= (uint32_t)p) atomicOr(err, QFS_ERRBIT_INPUT);
    }
    for (int i = tid; i < WW; i += NT) { bufA[i] = 0; bufB[i] = 0; }
    __syncthreads();
    {
        uint32_t any = 0;
        for (int t = 0; t < 10; ++t) any |= fT[t];
        if (any == 0) {  // the zero form (tau(a) = 0 iff a = 0)
            if (tid == 0) { atomicOr(err, QFS_ERRBIT_INPUT); heights[slot] = 0; iters[slot] = 0; }
            return;
        }
    }
    if (tid < 10) bufA[c_cubic_exp[tid][0] * W + c_cubic_exp[tid][1]] = (uint16_t)fT[tid];
    __syncthreads();

    // ---- chain cur = f_T^k mod p^2, k = 2..p ----
    uint16_t* cur = bufA;
    uint16_t* nxt = bufB;
    if (p == 3) {  // h = f^(p-2) = f
        for (int i = tid; i < WW; i += NT) sh[i] = (uint8_t)(cur[i] % (uint32_t)p);
    }
    for (int k = 2; k <= p; ++k) {
        const int din = 3 * (k - 1), dout = 3 * k;
        for (int o = tid; o < (dout + 1) * (dout + 1); o += NT) {
            const int i1 = o / (dout + 1), i2 = o - i1 * (dout + 1);
            if (i1 + i2 > dout) continue;
            uint32_t acc = 0;
#pragma unroll
            for (int t = 0; t < 10; ++t) {
                const int a1 = i1 - c_cubic_exp[t][0], a2 = i2 - c_cubic_exp[t][1];
                if (a1 >= 0 && a2 >= 0 && a1 + a2 <= din) acc += fT[t] * (uint32_t)cur[a1 * W + a2];
            }
            nxt[i1 * W + i2] = (uint16_t)(acc % (uint32_t)psq);
        }
        __syncthreads();
        { uint16_t* t = cur; cur = nxt; nxt = t; }
        if (k == p - 2)
            for (int i = tid; i < WW; i += NT) sh[i] = (uint8_t)(cur[i] % (uint32_t)p);
        if (k == p - 1)
            for (int i = tid; i < WW; i += NT) sga[i] = (uint8_t)(cur[i] % (uint32_t)p);
        if (k == p) {
            // E = (f_T^p - phi(f_T)) / p mod p
            for (int o = tid; o < WW; o += NT) {
                const int J1 = o / W, J2 = o - J1 * W, J3 = 3 * p - J1 - J2;
                uint32_t v = 0;
                if (J3 >= 0) {
                    v = cur[o];
                    if (J1 % p == 0 && J2 % p == 0) {  // then p | J3 too
                        const int r1 = J1 / p, r2 = J2 / p;
                        for (int t = 0; t < 10; ++t)
                            if (c_cubic_exp[t][0] == r1 && c_cubic_exp[t][1] == r2) v = (v + (uint32_t)psq - fT[t]) % (uint32_t)psq;
                    }
                    if (v % (uint32_t)p) s_bad = 1;
                    v = (v / (uint32_t)p) % (uint32_t)p;
                }
                sE[o] = (uint8_t)v;
            }
        }
        // the previous contents of nxt outside the new triangle are stale but never read (degree checks)
        __syncthreads();
    }
    if (s_bad) {
        if (tid == 0) atomicOr(err, QFS_ERRBIT_INVARIANT);
    }
    const int cap = (p - 1) * W + (p - 1);
    const int d = 3 * (p - 1), dh = 3 * (p - 2);
    int height = 0, it = 0;
    if (sga[cap] != 0) {
        height = 1;
    } else {
        for (int step = 1; step <= max_steps; ++step) {
            if (tid < 10) sq[tid] = 0;
            __syncthreads();
            int acc[10];
#pragma unroll
            for (int r = 0; r < 10; ++r) acc[r] = 0;
            for (int o = tid; o < WW; o += NT) {
                const int e = sE[o];
                if (e == 0) continue;
                const int J1 = o / W, J2 = o - J1 * W, J3 = 3 * p - J1 - J2;
                if (J3 < 0) continue;
#pragma unroll
                for (int r = 0; r < 10; ++r) {
                    const int a1 = p * c_cubic_exp[r][0] + p - 1 - J1, a2 = p * c_cubic_exp[r][1] + p - 1 - J2,
                              a3 = p * c_cubic_exp[r][2] + p - 1 - J3;
                    if ((a1 | a2 | a3) >= 0) acc[r] += e * (int)sga[a1 * W + a2];
                }
            }
#pragma unroll
            for (int r = 0; r < 10; ++r) {
                const int t = __reduce_add_sync(0xffffffffu, acc[r]);
                if (lane == 0 && t) atomicAdd(&sq[r], t);
            }
            __syncthreads();
            if (tid < 10) sq[tid] = sq[tid] % p;
            __syncthreads();
            for (int o = tid; o < (d + 1) * (d + 1); o += NT) {
                const int i1 = o / (d + 1), i2 = o - i1 * (d + 1);
                if (i1 + i2 > d) continue;
                int s = 0;
#pragma unroll
                for (int r = 0; r < 10; ++r) {
                    const int u1 = i1 - c_cubic_exp[r][0], u2 = i2 - c_cubic_exp[r][1];
                    if (u1 >= 0 && u2 >= 0 && u1 + u2 <= dh) s += sq[r] * (int)sh[u1 * W + u2];
                }
                const int v = s % p;
                sgb[i1 * W + i2] = (uint8_t)(v ? p - v : 0);
            }
            __syncthreads();
            { uint8_t* t = sga; sga = sgb; sgb = t; }
            ++it;
            if (sga[cap] != 0) { height = step + 1; break; }
        }
    }
    if (tid == 0) {
        heights[slot] = (int8_t)height;
        iters[slot] = (int8_t)it;
    }
}
