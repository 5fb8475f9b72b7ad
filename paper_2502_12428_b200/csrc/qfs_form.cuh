// qfs_form.cuh -- heights of Calabi-Yau hypersurfaces in n variables for the n the quartic and cubic kernels do not cover
// (SURVEY.md section 8(f)4 "general n"): a form of degree n in x1..xn over F_p, n = 2 .. 6 and an odd prime p at run time with (n p + 1)^(n-1) <= 2^24
// (n = 2: p <= 53, n = 5: p <= 11, n = 6: p = 3).
// The reference's drivers take any such form (SurfaceProblem, height.py:63-94; height_matrix / height_naive, height.py:97-144).
//
// One CTA per form, toy sizes (n = 5: 126 coefficients, operator 1001 x 1001 at p = 3), nothing to stream: like qfs_cubic.cuh
// the kernel runs the matrix-free form of the iteration -- the identities of DESIGN.md section 3 do not depend on n:
//     f_T = sum tau(a_J) x^J,  tau(a) = a^p mod p^2;   chain f_T^2 ... f_T^p mod p^2
//     h = f^(p-2), g = f^(p-1) (mod p),  E = Delta_1(f) = (f_T^p - phi(f_T)) / p mod p      (exact division, checked)
//     height 1 iff g[cap] != 0;  else  g <- -h * u(E g)  until g[cap] != 0  (height = steps + 1) or the bound,
//     u(E g)[r] = sum_J E[J] g[p r + (p-1) 1 - J]   for the monomials r of degree n.
// A form of degree D is a dense box indexed by its first n-1 exponents (mixed radix, side W = n p + 1); the boxes live in a
// per-CTA slice of a global scratch buffer (8 W^(n-1) bytes: a few hundred KB, L2-resident), the term tables in shared memory.
#pragma once
#include <stdint.h>

#include "qfs_shape.cuh"

#define QFS_FORM_MAXN 6
#define QFS_FORM_MAXP 53
#define QFS_FORM_MAXBOX (1u << 24)   // entries of a box the kernel accepts: W^(n-1), W = n p + 1
#define QFS_FORM_MAXT 462   // C(2n-1, n-1) monomials of degree n in n variables, n = 6
#define QFS_FORM_NT 256

__host__ __device__ inline size_t qfs_form_box(int n, int p)
{
    size_t w = (size_t)n * p + 1, s = 1;
    for (int i = 0; i < n - 1; ++i) s *= w;
    return s;
}
__host__ __device__ inline size_t qfs_form_scratch(int n, int p) { return 8 * qfs_form_box(n, p) + 64; }   // bytes per CTA

// exps[t][i]: exponent of x_{i+1} in the t-th monomial of basis(n, n), lex-ascending with x1 most significant (monomials.py:182-196)
__global__ void __launch_bounds__(QFS_FORM_NT)
k_form(const uint8_t* __restrict__ coeffs, const uint8_t* __restrict__ exps, int nterms, int B, int first, int n, int p, int max_steps,
       uint8_t* __restrict__ scratch, int8_t* __restrict__ heights, int8_t* __restrict__ iters, int* __restrict__ err)
{
    __shared__ uint32_t fT[QFS_FORM_MAXT];
    __shared__ int sq[QFS_FORM_MAXT];
    __shared__ int soff[QFS_FORM_MAXT];              // linear offset of a term's first n-1 exponents
    __shared__ uint8_t sexp[QFS_FORM_MAXT][QFS_FORM_MAXN];
    __shared__ int s_bad, s_any;
    const int tid = threadIdx.x, NT = QFS_FORM_NT;
    const int slot = first + blockIdx.x;
    if (slot >= B) return;
    const int m = n - 1;                             // box dimensions
    const int W = n * p + 1, psq = p * p;
    size_t WN = 1;
    int stride[QFS_FORM_MAXN];                       // stride[i] of exponent i, x1 most significant
    for (int i = m - 1; i >= 0; --i) { stride[i] = (int)WN; WN *= (size_t)W; }
    uint8_t* base = scratch + (size_t)blockIdx.x * qfs_form_scratch(n, p);
    uint16_t* cur = reinterpret_cast<uint16_t*>(base);
    uint16_t* nxt = cur + WN;
    uint8_t* sh = reinterpret_cast<uint8_t*>(nxt + WN);
    uint8_t* sga = sh + WN;
    uint8_t* sgb = sga + WN;
    uint8_t* sE = sgb + WN;

    if (tid == 0) { s_bad = 0; s_any = 0; }
    __syncthreads();
    for (int t = tid; t < nterms; t += NT) {
        const uint32_t a = coeffs[(size_t)slot * nterms + t];
        uint32_t v = 1;
        for (int k = 0; k < p; ++k) v = (v * a) % (uint32_t)psq;   // tau(a) = a^p mod p^2
        fT[t] = (a < (uint32_t)p) ? v : 0u;
        if (a >= (uint32_t)p) atomicOr(err, QFS_ERRBIT_INPUT);
        if (fT[t]) s_any = 1;
        int off = 0;
        for (int i = 0; i < n; ++i) {
            sexp[t][i] = exps[t * n + i];
            if (i < m) off += (int)exps[t * n + i] * stride[i];
        }
        soff[t] = off;
    }
    for (size_t i = tid; i < WN; i += NT) { cur[i] = 0; nxt[i] = 0; sh[i] = 0; sga[i] = 0; sgb[i] = 0; sE[i] = 0; }
    __syncthreads();
    if (!s_any) {   // the zero form (tau(a) = 0 iff a = 0)
        if (tid == 0) { atomicOr(err, QFS_ERRBIT_INPUT); heights[slot] = 0; iters[slot] = 0; }
        return;
    }
    for (int t = tid; t < nterms; t += NT) cur[soff[t]] = (uint16_t)fT[t];
    __syncthreads();

    // decode position `o` of the box of side (deg+1) into exponents a[0..m-1]; returns the linear index, -1 outside the simplex
    auto locate = [&](size_t o, int deg, int* a) -> long {
        int sum = 0;
        long lin = 0;
        for (int i = m - 1; i >= 0; --i) {
            a[i] = (int)(o % (size_t)(deg + 1));
            o /= (size_t)(deg + 1);
            sum += a[i];
            lin += (long)a[i] * stride[i];
        }
        return sum <= deg ? lin : -1;
    };
    auto boxsize = [&](int deg) { size_t s = 1; for (int i = 0; i < m; ++i) s *= (size_t)(deg + 1); return s; };

    // ---- chain cur = f_T^k mod p^2, k = 2..p ----
    if (p == 3)   // h = f^(p-2) = f
        for (size_t i = tid; i < WN; i += NT) sh[i] = (uint8_t)(cur[i] % (uint32_t)p);
    for (int k = 2; k <= p; ++k) {
        const int din = n * (k - 1), dout = n * k;
        const size_t total = boxsize(dout);
        for (size_t o = tid; o < total; o += NT) {
            int a[QFS_FORM_MAXN];
            const long lin = locate(o, dout, a);
            if (lin < 0) continue;
            int asum = 0;
            for (int i = 0; i < m; ++i) asum += a[i];
            uint32_t acc = 0;
            for (int t = 0; t < nterms; ++t) {
                if (!fT[t]) continue;
                bool ok = asum - (n - (int)sexp[t][m]) <= din && (dout - asum) >= (int)sexp[t][m];
                for (int i = 0; i < m && ok; ++i) ok = a[i] >= (int)sexp[t][i];
                if (ok) acc += fT[t] * (uint32_t)cur[lin - soff[t]];
            }
            nxt[lin] = (uint16_t)(acc % (uint32_t)psq);
        }
        __syncthreads();
        { uint16_t* t = cur; cur = nxt; nxt = t; }
        for (size_t i = tid; i < WN; i += NT) nxt[i] = 0;   // the box the next level writes into starts clean
        if (k == p - 2)
            for (size_t i = tid; i < WN; i += NT) sh[i] = (uint8_t)(cur[i] % (uint32_t)p);
        if (k == p - 1)
            for (size_t i = tid; i < WN; i += NT) sga[i] = (uint8_t)(cur[i] % (uint32_t)p);
        if (k == p) {
            // E = (f_T^p - phi(f_T)) / p mod p
            const size_t tot = boxsize(n * p);
            for (size_t o = tid; o < tot; o += NT) {
                int a[QFS_FORM_MAXN];
                const long lin = locate(o, n * p, a);
                if (lin < 0) continue;
                uint32_t v = cur[lin];
                bool mult = true;
                for (int i = 0; i < m; ++i) mult = mult && (a[i] % p == 0);
                if (mult) {   // then p divides the last exponent too: J = p * (a term's exponents)?
                    for (int t = 0; t < nterms; ++t) {
                        bool same = true;
                        for (int i = 0; i < m; ++i) same = same && ((int)sexp[t][i] * p == a[i]);
                        if (same) v = (v + (uint32_t)psq - fT[t]) % (uint32_t)psq;
                    }
                }
                if (v % (uint32_t)p) s_bad = 1;
                sE[lin] = (uint8_t)((v / (uint32_t)p) % (uint32_t)p);
            }
        }
        __syncthreads();
    }
    if (s_bad && tid == 0) atomicOr(err, QFS_ERRBIT_INVARIANT);
    long cap = 0;
    for (int i = 0; i < m; ++i) cap += (long)(p - 1) * stride[i];
    const int d = n * (p - 1), dh = n * (p - 2);
    int height = 0, it = 0;
    if (sga[cap] != 0) {
        height = 1;
    } else {
        for (int step = 1; step <= max_steps; ++step) {
            for (int t = tid; t < nterms; t += NT) sq[t] = 0;
            __syncthreads();
            // q[r] = sum_J E[J] g[p r + (p-1) 1 - J]: a thread per exponent J of E, shared-memory adds per monomial r
            const size_t totE = boxsize(n * p);
            for (size_t o = tid; o < totE; o += NT) {
                int J[QFS_FORM_MAXN];
                const long lin = locate(o, n * p, J);
                if (lin < 0) continue;
                const int e = sE[lin];
                if (e == 0) continue;
                int Jsum = 0;
                for (int i = 0; i < m; ++i) Jsum += J[i];
                const int Jlast = n * p - Jsum;
                for (int r = 0; r < nterms; ++r) {
                    bool ok = p * (int)sexp[r][m] + p - 1 - Jlast >= 0;
                    long gi = 0;
                    for (int i = 0; i < m && ok; ++i) {
                        const int ai = p * (int)sexp[r][i] + p - 1 - J[i];
                        ok = ai >= 0;
                        gi += (long)ai * stride[i];
                    }
                    if (ok) {
                        const int gv = sga[gi];
                        if (gv) atomicAdd(&sq[r], e * gv);
                    }
                }
            }
            __syncthreads();
            for (int t = tid; t < nterms; t += NT) sq[t] = sq[t] % p;
            __syncthreads();
            const size_t totG = boxsize(d);
            for (size_t o = tid; o < totG; o += NT) {
                int a[QFS_FORM_MAXN];
                const long lin = locate(o, d, a);
                if (lin < 0) continue;
                int asum = 0;
                for (int i = 0; i < m; ++i) asum += a[i];
                int s = 0;
                for (int r = 0; r < nterms; ++r) {
                    if (!sq[r]) continue;
                    bool ok = asum - (n - (int)sexp[r][m]) <= dh && (d - asum) >= (int)sexp[r][m];
                    for (int i = 0; i < m && ok; ++i) ok = a[i] >= (int)sexp[r][i];
                    if (ok) s += sq[r] * (int)sh[lin - soff[r]];
                }
                const int v = s % p;
                sgb[lin] = (uint8_t)(v ? p - v : 0);
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
