// qfs_literal.cuh -- the reference's definitions executed literally on the device: an independent route to g, Delta_1(g) and
// the heights that shares NOTHING with the engine's kernels (no Teichmueller lift, no f^(p-2), no Witt-carry factorisation,
// no operator matrix).  It is the on-device counterpart of height_naive (height.py:97-116):
//     g     = f^(p-1) mod p                     by p-2 dense multiplications by f                (power_mod_p, polyring.py:253-272)
//     Delta = ((lift g)^p - sum_J (g_J x^J)^p) / p mod p,  the power by p-1 dense multiplications by g mod p^2, the division
//             checked coefficient by coefficient                                                 (delta1, polyring.py:335-401)
//     g    <- u(Delta * g): the coefficients of Delta*g at the exponents p*m + (p-1)*1           (split_u, polyring.py:295-313)
//     until g[(p-1)*1] != 0 (height = steps + 1) or the bound is passed.
// A cross-check, not a fast path: p <= 7 (F_7: 6 G multiply-adds and 15 MB of scratch per surface).
//
// A form of degree `deg` in x1..x4 lives in a "box": cell (a1,a2,a3) at (a1*W + a2)*W + a3, W = p*d + 1 for every level, one
// byte per cell (values < p^2 <= 49); a4 = deg - a1 - a2 - a3 is implied.  The second factor of a product is a term list.
#pragma once
#include <stdint.h>

#include "qfs_shape.cuh"

#define QFS_LIT_MAXP 7
#define QFS_LIT_MAXTERMS 2925   // terms of g = f^(p-1) at p = 7
#define QFS_LIT_NT 128

struct LitTerm { uint32_t off, ec; };   // box offset of (e1,e2,e3); e1 | e2<<5 | e3<<10 | e4<<15 | coefficient<<20

// the quartic's coefficient vector (lex-ascending basis(4,4), index 0 = x4^4) into a box; validates the input
__global__ void k_lit_load(const uint8_t* __restrict__ coeffs, int first, int p, int W, size_t boxsize, uint8_t* __restrict__ box, int* __restrict__ err)
{
    const int s = blockIdx.x;
    const uint8_t* c = coeffs + (size_t)(first + s) * 35;
    uint8_t* b = box + (size_t)s * boxsize;
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        int i = 0;
        for (int a1 = 0; a1 <= 4; ++a1)
            for (int a2 = 0; a1 + a2 <= 4; ++a2)
                for (int a3 = 0; a1 + a2 + a3 <= 4; ++a3, ++i) {
                    const int v = c[i];
                    if (v >= p) atomicOr(err, QFS_ERRBIT_INPUT);
                    if (v) any = 1;
                    b[((size_t)a1 * W + a2) * W + a3] = (uint8_t)(v < p ? v : 0);
                }
        if (!any) atomicOr(err, QFS_ERRBIT_INPUT);
    }
}

// nonzero cells of a degree-`deg` box as a term list (order irrelevant: sums commute)
__global__ void k_lit_terms(const uint8_t* __restrict__ box, int deg, int W, size_t boxsize, LitTerm* __restrict__ terms, int* __restrict__ nterms)
{
    const int s = blockIdx.y;
    const int a1 = blockIdx.x / (deg + 1), a2 = blockIdx.x % (deg + 1);
    if (a1 + a2 > deg) return;
    const uint8_t* b = box + (size_t)s * boxsize;
    for (int a3 = threadIdx.x; a1 + a2 + a3 <= deg; a3 += blockDim.x) {
        const uint32_t off = (uint32_t)(((size_t)a1 * W + a2) * W + a3);
        const uint32_t v = b[off];
        if (v) {
            const int k = atomicAdd(&nterms[s], 1);
            if (k < QFS_LIT_MAXTERMS)
                terms[(size_t)s * QFS_LIT_MAXTERMS + k] = LitTerm{off, (uint32_t)a1 | ((uint32_t)a2 << 5) | ((uint32_t)a3 << 10) | ((uint32_t)(deg - a1 - a2 - a3) << 15) | (v << 20)};
        }
    }
}

// out = A * B mod m; A a box of degree degA, B a term list of degree degB.  One CTA per (a1,a2) of the product, a thread per a3.
__global__ void __launch_bounds__(QFS_LIT_NT)
k_lit_mul(const uint8_t* __restrict__ A, int degA, const LitTerm* __restrict__ terms, const int* __restrict__ nterms, int degB, int W, size_t boxsize,
          uint8_t* __restrict__ out, int m, const int* __restrict__ skip)
{
    __shared__ LitTerm sT[QFS_LIT_MAXTERMS];
    __shared__ int sN;
    const int degO = degA + degB;
    const int s = blockIdx.y;
    const int a1 = blockIdx.x / (degO + 1), a2 = blockIdx.x % (degO + 1);
    if (a1 + a2 > degO || (skip && skip[s])) return;
    if (threadIdx.x == 0) sN = 0;
    __syncthreads();
    const LitTerm* T = terms + (size_t)s * QFS_LIT_MAXTERMS;
    const int n = min(nterms[s], QFS_LIT_MAXTERMS);
    for (int t = threadIdx.x; t < n; t += QFS_LIT_NT) {
        const LitTerm x = T[t];
        if ((int)(x.ec & 31) <= a1 && (int)((x.ec >> 5) & 31) <= a2) sT[atomicAdd(&sN, 1)] = x;
    }
    __syncthreads();
    const uint8_t* a = A + (size_t)s * boxsize;
    uint8_t* o = out + (size_t)s * boxsize;
    const uint32_t base = (uint32_t)(((size_t)a1 * W + a2) * W);
    const int cnt = sN;
    for (int a3 = threadIdx.x; a1 + a2 + a3 <= degO; a3 += QFS_LIT_NT) {
        const int a4 = degO - a1 - a2 - a3;
        uint32_t acc = 0;
        for (int t = 0; t < cnt; ++t) {
            const LitTerm x = sT[t];
            if ((int)((x.ec >> 10) & 31) <= a3 && (int)((x.ec >> 15) & 31) <= a4) acc += (x.ec >> 20) * (uint32_t)a[base + a3 - x.off];
        }
        o[base + a3] = (uint8_t)(acc % (uint32_t)m);
    }
}

// pw = (lift g)^p mod p^2 (degree D = p d) -> Delta in place: subtract (g_J)^p at the exponents p*J, divide by p (checked), mod p
__global__ void k_lit_carry(uint8_t* __restrict__ pw, const uint8_t* __restrict__ g, int p, int d, int W, size_t boxsize, int* __restrict__ err,
                            const int* __restrict__ skip)
{
    const int D = p * d, psq = p * p;
    const int s = blockIdx.y;
    const int a1 = blockIdx.x / (D + 1), a2 = blockIdx.x % (D + 1);
    if (a1 + a2 > D || (skip && skip[s])) return;
    uint8_t* b = pw + (size_t)s * boxsize;
    const uint8_t* gb = g + (size_t)s * boxsize;
    for (int a3 = threadIdx.x; a1 + a2 + a3 <= D; a3 += blockDim.x) {
        const size_t off = ((size_t)a1 * W + a2) * W + a3;
        int v = b[off];
        if (a1 % p == 0 && a2 % p == 0 && a3 % p == 0) {   // then p divides a4 = D - a1 - a2 - a3 as well
            const int c = gb[((size_t)(a1 / p) * W + a2 / p) * W + a3 / p];
            int cp = 1;
            for (int k = 0; k < p; ++k) cp = cp * c % psq;
            v = (v + psq - (c ? cp : 0)) % psq;
        }
        if (v % p) atomicOr(err, QFS_ERRBIT_INVARIANT);
        b[off] = (uint8_t)((v / p) % p);
    }
}

// box of degree deg -> dense lex vector (qfs_shape.cuh)
__global__ void k_lit_dense(const uint8_t* __restrict__ box, int deg, int W, size_t boxsize, uint8_t* __restrict__ dense, size_t stride)
{
    const int s = blockIdx.y;
    const int a1 = blockIdx.x / (deg + 1), a2 = blockIdx.x % (deg + 1);
    if (a1 + a2 > deg) return;
    const uint8_t* b = box + (size_t)s * boxsize;
    uint8_t* o = dense + (size_t)s * stride + qrowbase(deg, a1, a2);
    for (int a3 = threadIdx.x; a1 + a2 + a3 <= deg; a3 += blockDim.x) o[a3] = b[((size_t)a1 * W + a2) * W + a3];
}

// gn[m] = sum_c g[c] * Delta[p m + (p-1) 1 - c] mod p over the monomials c of degree d (all four exponents of the index >= 0)
__global__ void k_lit_step(const uint8_t* __restrict__ delta, const uint8_t* __restrict__ g, uint8_t* __restrict__ gn, const int* __restrict__ done,
                           int p, int d, int W, size_t boxsize)
{
    const int s = blockIdx.y;
    if (done[s]) return;
    const int m1 = blockIdx.x / (d + 1), m2 = blockIdx.x % (d + 1);
    if (m1 + m2 > d) return;
    const uint8_t* dl = delta + (size_t)s * boxsize;
    const uint8_t* gb = g + (size_t)s * boxsize;
    for (int m3 = threadIdx.x; m1 + m2 + m3 <= d; m3 += blockDim.x) {
        const int m4 = d - m1 - m2 - m3;
        const int t1 = p * m1 + p - 1, t2 = p * m2 + p - 1, t3 = p * m3 + p - 1, t4 = p * m4 + p - 1;
        uint32_t acc = 0;
        for (int c1 = 0; c1 <= min(d, t1); ++c1)
            for (int c2 = 0; c2 <= min(d - c1, t2); ++c2) {
                const uint8_t* gr = gb + ((size_t)c1 * W + c2) * W;
                const uint8_t* dr = dl + ((size_t)(t1 - c1) * W + (t2 - c2)) * W + t3;
                const int rest = d - c1 - c2;
                for (int c3 = max(0, rest - t4); c3 <= min(rest, t3); ++c3) acc += (uint32_t)gr[c3] * dr[-c3];
            }
        gn[(size_t)s * boxsize + ((size_t)m1 * W + m2) * W + m3] = (uint8_t)(acc % (uint32_t)p);
    }
}

// step 0: the Fedder test on g = f^(p-1); step k >= 1: after the k-th application of the operator
__global__ void k_lit_check(const uint8_t* __restrict__ g, int p, int W, size_t boxsize, int step, int bound, int first, int count,
                            int8_t* __restrict__ heights, int8_t* __restrict__ iters, int* __restrict__ done)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= count) return;
    if (step == 0) {
        done[s] = 0;
        heights[first + s] = 0;
        iters[first + s] = 0;
    }
    if (done[s]) return;
    const int cap = g[(size_t)s * boxsize + ((size_t)(p - 1) * W + (p - 1)) * W + (p - 1)];
    iters[first + s] = (int8_t)step;
    if (cap != 0) {
        heights[first + s] = (int8_t)(step + 1);
        done[s] = 1;
    } else if (step + 2 > bound) {
        done[s] = 1;   // the next height to test would pass the bound: infinity (0) after `step` applications
    }
}
