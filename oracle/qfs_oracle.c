/*
 * qfs_oracle.c -- CPU ORACLE for the quartic-K3 quasi-F-split height path.
 *
 * THIS FILE IS TEST INFRASTRUCTURE, NOT PRODUCT.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product (paper_2502_12428_b200/) never links, imports or
 * falls back to anything here.
 *
 * It is a plain-C restatement of the reference package `qfsplit`
 * (/root/reference/pkg/src/qfsplit, pure Python + numpy + numba), following the
 * reference's *definitions* step by step -- NOT the algebraic shortcuts the
 * CUDA path uses (no Witt-carry factorisation, no gather formula for the
 * matrix).  Each function cites the reference lines it restates.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function below against
 * tests/golden/ (npz + json), which were produced by running the unmodified
 * reference in the authoring container (tests/golden/make_golden.py), and
 * against the reference's published fixture table (32 surfaces).
 *
 * Data conventions:
 *   - a form of degree d in x1..x4 is a dense uint8 vector over the
 *     lex-ASCENDING monomial basis with x1 most significant:
 *       rank(a1,a2,a3,a4; d) = C(d+3,3)-C(d-a1+3,3) + C(d2+2,2)-C(d2-a2+2,2) + a3,
 *       d2 = d-a1;  index 0 = x4^d, last = x1^d         (monomials.py:182-196,208-276)
 *   - the operator matrix is row-major N x N, N = C(4p-1,3), column j = image
 *     of basis monomial j (mtsmatrix.py:82-96); we hold residues in uint8
 *     (the reference holds the same residues in uint16).
 *   - heights: 1..bound, 0 encodes "infinity" (height.py:28, math.inf).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define QFO_OK 0
#define QFO_EINVAL (-1)
#define QFO_EINVARIANT (-3)
#define QFO_ENOMEM (-4)

static inline int64_t c2(int64_t n) { return n >= 2 ? n * (n - 1) / 2 : 0; }
static inline int64_t c3(int64_t n) { return n >= 3 ? n * (n - 1) * (n - 2) / 6 : 0; }

/* number of degree-d monomials in 4 variables (monomials.py:222) */
int64_t qfo_basis_size(int d) { return c3((int64_t)d + 3); }

/* index of the first monomial of the run (a1,a2,0,*) in basis(d,4) */
static inline int64_t rowbase(int d, int a1, int a2)
{
    int d2 = d - a1;
    return c3(d + 3) - c3(d - a1 + 3) + c2(d2 + 2) - c2(d2 - a2 + 2);
}

int64_t qfo_rank(int d, int a1, int a2, int a3) { return rowbase(d, a1, a2) + a3; }

static int is_prime_small(int p)
{
    if (p < 2) return 0;
    for (int q = 2; q * q <= p; ++q)
        if (p % q == 0) return 0;
    return 1;
}

/* ---------------------------------------------------------------------------
 * Dense product of two forms modulo m (m = p or p^2), schoolbook.
 * Restates polyring._mul_mod (polyring.py:192-225: all pair products, merge
 * equal exponents, reduce) on dense vectors; u32 accumulators are exact because
 * #pairs per output * (m-1)^2 <= 20825 * 168^2 < 2^32 for p <= 13.
 * ------------------------------------------------------------------------- */
#if defined(__x86_64__) && defined(__GNUC__)
__attribute__((target_clones("avx2", "default")))
#endif
static int poly_mul_mod(const uint8_t *a, int da, const uint8_t *b, int db, uint32_t m,
                        uint8_t *out, uint32_t *acc /* size basis(da+db) */)
{
    const int dout = da + db;
    const int64_t nout = qfo_basis_size(dout);
    memset(acc, 0, sizeof(uint32_t) * (size_t)nout);
    /* rows of b */
    int nbrows = (db + 1) * (db + 2) / 2;
    int32_t *brow = (int32_t *)malloc(sizeof(int32_t) * 4 * (size_t)nbrows);
    if (!brow) return QFO_ENOMEM;
    int nb = 0;
    for (int b1 = 0; b1 <= db; ++b1)
        for (int b2 = 0; b1 + b2 <= db; ++b2) {
            brow[4 * nb + 0] = b1;
            brow[4 * nb + 1] = b2;
            brow[4 * nb + 2] = (int32_t)rowbase(db, b1, b2);
            brow[4 * nb + 3] = db - b1 - b2 + 1;
            ++nb;
        }
    /* row bases of the output */
    int64_t *obase = (int64_t *)malloc(sizeof(int64_t) * (size_t)(dout + 1) * (size_t)(dout + 1));
    if (!obase) { free(brow); return QFO_ENOMEM; }
    for (int i1 = 0; i1 <= dout; ++i1)
        for (int i2 = 0; i1 + i2 <= dout; ++i2) obase[i1 * (dout + 1) + i2] = rowbase(dout, i1, i2);

    for (int a1 = 0; a1 <= da; ++a1)
        for (int a2 = 0; a1 + a2 <= da; ++a2) {
            const int64_t ab = rowbase(da, a1, a2);
            for (int a3 = 0; a1 + a2 + a3 <= da; ++a3) {
                const uint32_t ca = a[ab + a3];
                if (!ca) continue;
                for (int r = 0; r < nb; ++r) {
                    const uint8_t *bp = b + brow[4 * r + 2];
                    uint32_t *op = acc + obase[(a1 + brow[4 * r]) * (dout + 1) + a2 + brow[4 * r + 1]] + a3;
                    const int len = brow[4 * r + 3];
                    for (int k = 0; k < len; ++k) op[k] += ca * bp[k];
                }
            }
        }
    for (int64_t i = 0; i < nout; ++i) out[i] = (uint8_t)(acc[i] % m);
    free(brow);
    free(obase);
    return QFO_OK;
}

/* public wrapper: out = a*b mod m, all dense lex vectors */
int qfo_poly_mul_mod(const uint8_t *a, int da, const uint8_t *b, int db, int m, uint8_t *out)
{
    if (m < 2 || m > 255 || da < 0 || db < 0) return QFO_EINVAL;
    uint32_t *acc = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)qfo_basis_size(da + db));
    if (!acc) return QFO_ENOMEM;
    int rc = poly_mul_mod(a, da, b, db, (uint32_t)m, out, acc);
    free(acc);
    return rc;
}

/* ---------------------------------------------------------------------------
 * g = f^k mod p by square-and-multiply, restating polyring.power_mod_p
 * (polyring.py:253-272).  f is a dense form of degree df; out has degree k*df.
 * ------------------------------------------------------------------------- */
int qfo_power_mod_p(const uint8_t *f, int df, int k, int p, uint8_t *out)
{
    if (k < 1 || p < 2 || p > 15) return QFO_EINVAL;
    const int64_t nmax = qfo_basis_size(k * df);
    uint8_t *result = NULL, *square = (uint8_t *)malloc((size_t)nmax), *tmp = (uint8_t *)malloc((size_t)nmax);
    uint32_t *acc = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)nmax);
    uint8_t *resbuf = (uint8_t *)malloc((size_t)nmax);
    if (!square || !tmp || !acc || !resbuf) { free(square); free(tmp); free(acc); free(resbuf); return QFO_ENOMEM; }
    int dsq = df, dres = 0, rc = QFO_OK;
    memcpy(square, f, (size_t)qfo_basis_size(df));
    int e = k;
    while (e) {
        if (e & 1) {
            if (!result) {
                memcpy(resbuf, square, (size_t)qfo_basis_size(dsq));
                result = resbuf;
                dres = dsq;
            } else {
                rc = poly_mul_mod(result, dres, square, dsq, (uint32_t)p, tmp, acc);
                if (rc) break;
                dres += dsq;
                memcpy(resbuf, tmp, (size_t)qfo_basis_size(dres));
            }
        }
        e >>= 1;
        if (e) {
            rc = poly_mul_mod(square, dsq, square, dsq, (uint32_t)p, tmp, acc);
            if (rc) break;
            dsq *= 2;
            memcpy(square, tmp, (size_t)qfo_basis_size(dsq));
        }
    }
    if (!rc) memcpy(out, result, (size_t)qfo_basis_size(k * df));
    free(square); free(tmp); free(acc); free(resbuf);
    return rc;
}

/* Fedder test: coefficient of (x1 x2 x3 x4)^(p-1) in g (polyring.py:316-332) */
int qfo_fedder_survives(const uint8_t *g, int p)
{
    return g[qfo_rank(4 * (p - 1), p - 1, p - 1, p - 1)] != 0;
}

/* ---------------------------------------------------------------------------
 * delta1(g) = ((lift g)^p - sum_I c_I^p x^{pI}) / p  mod p   (polyring.py:335-401)
 * lift = representatives in [0,p) (polyring.py:275-281).  The reference gets
 * (lift g)^p mod p^2 from a multimodular NTT (nttpower.py:447-507); here the
 * same integer power is taken by p-1 exact schoolbook products reduced mod
 * p^2 (the reference's own "schoolbook" backend, polyring.py:357-361, with the
 * reduction mod p^2 commuting with the ring operations).  Divisibility by p is
 * checked coefficient by coefficient as polyring.py:397-398 does.
 * g has degree dg; out is dense over basis(p*dg, 4).
 * ------------------------------------------------------------------------- */
int qfo_delta1(const uint8_t *g, int dg, int p, uint8_t *out)
{
    if (!is_prime_small(p) || p > 13 || dg < 1) return QFO_EINVAL;
    const uint32_t psq = (uint32_t)(p * p);
    const int D = p * dg;
    const int64_t nD = qfo_basis_size(D);
    uint8_t *cur = (uint8_t *)malloc((size_t)nD), *nxt = (uint8_t *)malloc((size_t)nD);
    uint32_t *acc = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)nD);
    if (!cur || !nxt || !acc) { free(cur); free(nxt); free(acc); return QFO_ENOMEM; }
    int rc = QFO_OK, dcur = dg;
    memcpy(cur, g, (size_t)qfo_basis_size(dg));
    for (int step = 1; step < p && !rc; ++step) {
        rc = poly_mul_mod(cur, dcur, g, dg, psq, nxt, acc);
        dcur += dg;
        uint8_t *t = cur; cur = nxt; nxt = t;
    }
    if (!rc) {
        /* add (p^2 - c^p) at exponent p*I  (polyring.py:385-388) */
        for (int a1 = 0; a1 <= dg; ++a1)
            for (int a2 = 0; a1 + a2 <= dg; ++a2)
                for (int a3 = 0; a1 + a2 + a3 <= dg; ++a3) {
                    uint32_t c = g[qfo_rank(dg, a1, a2, a3)];
                    if (!c) continue;
                    uint32_t cp = 1;
                    for (int i = 0; i < p; ++i) cp = cp * c % psq;
                    int64_t idx = qfo_rank(D, p * a1, p * a2, p * a3);
                    cur[idx] = (uint8_t)((cur[idx] + psq - cp) % psq);
                }
        for (int64_t i = 0; i < nD; ++i) {
            uint32_t v = cur[i];
            if (v % (uint32_t)p) { rc = QFO_EINVARIANT; break; }
            out[i] = (uint8_t)((v / (uint32_t)p) % (uint32_t)p);
        }
    }
    free(cur); free(nxt); free(acc);
    return rc;
}

/* ---------------------------------------------------------------------------
 * Operator matrix of g -> u(delta*g), WICS construction (mtsmatrix.py:249-281):
 * for every nonzero delta term with exponent e: res = e mod p, quot = e div p,
 * comp = (p-1) - res, rem = d - |comp|; when rem >= 0 and p | rem, every weak
 * composition w of rem/p gives column comp + p*w and row quot + w, and the
 * coefficient is accumulated there; entries are reduced mod p at the end
 * (mtsmatrix.py:168-170).  target degree d' = (d + D - 4(p-1))/p
 * (mtsmatrix.py:42-52) equals d for the K3 shapes used here.
 * delta: dense over basis(D,4); M: row-major uint8 [N(dprime) x N(d)].
 * ------------------------------------------------------------------------- */
int qfo_build_mts(const uint8_t *delta, int D, int d, int p, uint8_t *M)
{
    const int num = d + D - 4 * (p - 1);
    if (num < 0 || num % p) return QFO_EINVAL; /* ZERO_MAP shapes are out of scope */
    const int dprime = num / p;
    const int64_t ncol = qfo_basis_size(d), nrow = qfo_basis_size(dprime);
    uint16_t *acc = (uint16_t *)calloc((size_t)(ncol * nrow), sizeof(uint16_t));
    if (!acc) return QFO_ENOMEM;
    for (int e1 = 0; e1 <= D; ++e1)
        for (int e2 = 0; e1 + e2 <= D; ++e2) {
            const int64_t base = rowbase(D, e1, e2);
            for (int e3 = 0; e1 + e2 + e3 <= D; ++e3) {
                const uint32_t c = delta[base + e3];
                if (!c) continue;
                const int e[4] = {e1, e2, e3, D - e1 - e2 - e3};
                int comp[4], quot[4], s = 0;
                for (int i = 0; i < 4; ++i) {
                    comp[i] = p - 1 - e[i] % p;
                    quot[i] = e[i] / p;
                    s += comp[i];
                }
                const int rem = d - s;
                if (rem < 0 || rem % p) continue;
                const int k = rem / p;
                for (int w1 = 0; w1 <= k; ++w1)
                    for (int w2 = 0; w1 + w2 <= k; ++w2)
                        for (int w3 = 0; w1 + w2 + w3 <= k; ++w3) {
                            int64_t col = qfo_rank(d, comp[0] + p * w1, comp[1] + p * w2, comp[2] + p * w3);
                            int64_t row = qfo_rank(dprime, quot[0] + w1, quot[1] + w2, quot[2] + w3);
                            acc[row * ncol + col] = (uint16_t)(acc[row * ncol + col] + c);
                        }
            }
        }
    for (int64_t i = 0; i < ncol * nrow; ++i) M[i] = (uint8_t)(acc[i] % (uint16_t)p);
    free(acc);
    return QFO_OK;
}

/* ---------------------------------------------------------------------------
 * M @ v over F_p with delayed reduction in column blocks of 2048 and uint64
 * accumulators (modmatrix.py:109-131, _COL_BLOCK at :19).
 * ------------------------------------------------------------------------- */
int qfo_matvec(const uint8_t *M, int64_t nrow, int64_t ncol, const uint8_t *v, int p, uint8_t *out)
{
    for (int64_t r = 0; r < nrow; ++r) {
        uint64_t acc = 0;
        const uint8_t *row = M + r * ncol;
        for (int64_t s = 0; s < ncol; s += 2048) {
            const int64_t e = s + 2048 < ncol ? s + 2048 : ncol;
            uint64_t part = 0;
            for (int64_t c = s; c < e; ++c) part += (uint64_t)row[c] * v[c];
            acc = (acc + part) % (uint64_t)p;
        }
        out[r] = (uint8_t)acc;
    }
    return QFO_OK;
}

/* ---------------------------------------------------------------------------
 * height_matrix (height.py:119-144) for a quartic given as its 35-vector.
 * Optional taps (may be NULL): g [N], delta [L], M [N*N], trace [(bound-1)*N].
 * ------------------------------------------------------------------------- */
int qfo_height_matrix(const uint8_t *coeffs35, int p, int bound, int8_t *height, int8_t *iters,
                      uint8_t *g_out, uint8_t *delta_out, uint8_t *M_out, uint8_t *trace_out)
{
    if (!is_prime_small(p) || p > 13 || bound < 1) return QFO_EINVAL;
    int any = 0;
    for (int i = 0; i < 35; ++i) {
        if (coeffs35[i] >= p) return QFO_EINVAL;
        any |= coeffs35[i];
    }
    if (!any) return QFO_EINVAL; /* height.py:85 */
    const int d = 4 * (p - 1), D = p * d;
    const int64_t N = qfo_basis_size(d), L = qfo_basis_size(D);
    int rc;
    uint8_t *g = (uint8_t *)malloc((size_t)N);
    if (!g) return QFO_ENOMEM;
    rc = qfo_power_mod_p(coeffs35, 4, p - 1, p, g);
    if (rc) { free(g); return rc; }
    if (g_out) memcpy(g_out, g, (size_t)N);
    *iters = 0;
    if (qfo_fedder_survives(g, p)) { *height = 1; free(g); return QFO_OK; }
    if (bound < 2) { *height = 0; free(g); return QFO_OK; }
    uint8_t *delta = (uint8_t *)malloc((size_t)L);
    uint8_t *M = (uint8_t *)malloc((size_t)(N * N));
    uint8_t *v = (uint8_t *)malloc((size_t)N), *w = (uint8_t *)malloc((size_t)N);
    if (!delta || !M || !v || !w) { rc = QFO_ENOMEM; goto done; }
    rc = qfo_delta1(g, d, p, delta);
    if (rc) goto done;
    if (delta_out) memcpy(delta_out, delta, (size_t)L);
    rc = qfo_build_mts(delta, D, d, p, M);
    if (rc) goto done;
    if (M_out) memcpy(M_out, M, (size_t)(N * N));
    memcpy(v, g, (size_t)N);
    const int64_t cap = qfo_rank(d, p - 1, p - 1, p - 1);
    *height = 0;
    for (int h = 2; h <= bound; ++h) {
        qfo_matvec(M, N, N, v, p, w);
        if (trace_out) memcpy(trace_out + (size_t)(*iters) * (size_t)N, w, (size_t)N);
        *iters += 1;
        uint8_t *t = v; v = w; w = t;
        if (v[cap]) { *height = (int8_t)h; break; }
    }
done:
    free(g); free(delta); free(M); free(v); free(w);
    return rc;
}

/* ---------------------------------------------------------------------------
 * height_naive (height.py:97-116): iterate g <- u(delta*g) on polynomials.
 * u = split_u (polyring.py:295-313): keep exponents = p-1 mod p, subtract p-1,
 * divide by p.  Independent of the matrix route; used to cross-check it.
 * ------------------------------------------------------------------------- */
int qfo_height_naive(const uint8_t *coeffs35, int p, int bound, int8_t *height, int8_t *iters)
{
    if (!is_prime_small(p) || p > 7 || bound < 1) return QFO_EINVAL;
    const int d = 4 * (p - 1), D = p * d;
    const int64_t N = qfo_basis_size(d), L = qfo_basis_size(D), LP = qfo_basis_size(D + d);
    uint8_t *g = (uint8_t *)malloc((size_t)N), *delta = (uint8_t *)malloc((size_t)L);
    uint8_t *prod = (uint8_t *)malloc((size_t)LP);
    uint32_t *acc = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)LP);
    int rc = QFO_ENOMEM;
    if (!g || !delta || !prod || !acc) goto done;
    rc = qfo_power_mod_p(coeffs35, 4, p - 1, p, g);
    if (rc) goto done;
    *iters = 0;
    if (qfo_fedder_survives(g, p)) { *height = 1; goto done; }
    *height = 0;
    if (bound < 2) goto done;
    rc = qfo_delta1(g, d, p, delta);
    if (rc) goto done;
    for (int h = 2; h <= bound; ++h) {
        rc = poly_mul_mod(delta, D, g, d, (uint32_t)p, prod, acc);
        if (rc) goto done;
        memset(g, 0, (size_t)N);
        for (int a1 = 0; a1 <= d; ++a1)
            for (int a2 = 0; a1 + a2 <= d; ++a2)
                for (int a3 = 0; a1 + a2 + a3 <= d; ++a3)
                    g[qfo_rank(d, a1, a2, a3)] =
                        prod[qfo_rank(D + d, p * a1 + p - 1, p * a2 + p - 1, p * a3 + p - 1)];
        *iters += 1;
        if (qfo_fedder_survives(g, p)) { *height = (int8_t)h; break; }
    }
done:
    free(g); free(delta); free(prod); free(acc);
    return rc;
}

/* batch driver: the loop body of search._worker_block (search.py:108-112) over
 * a block of coefficient vectors, fanned out over `threads` host threads. */
int qfo_heights_batch(const uint8_t *coeffs, int64_t B, int p, int bound, int8_t *heights, int8_t *iters,
                      int threads)
{
    int rc_all = QFO_OK;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t i = 0; i < B; ++i) {
        int rc = qfo_height_matrix(coeffs + 35 * i, p, bound, heights + i, iters + i, NULL, NULL, NULL, NULL);
        if (rc) {
#ifdef _OPENMP
#pragma omp critical
#endif
            rc_all = rc;
        }
    }
    return rc_all;
}

int qfo_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
