/*
 * qfs.h -- C ABI of libqfs.so: batched quasi-F-split (Artin-Mazur) heights of
 * quartic K3 surfaces over F_p on NVIDIA B200 (sm_100a).
 *
 * The reference package (`qfsplit`, pure Python) has no FFI boundary; its
 * boundary is its Python API.  Each entry point below names the reference
 * function whose work it replaces (paths relative to
 * /root/reference/pkg/src/qfsplit/).  The Python drop-in layer
 * (paper_2502_12428_b200/) binds these with ctypes; INTEGRATION.md shows the
 * stub a maintainer of the reference would add.
 *
 * Conventions
 *   - plain pointers and sizes only; no exceptions, no ownership transfer:
 *     the caller allocates every output.
 *   - every data pointer may be HOST or DEVICE memory (detected with
 *     cudaPointerGetAttributes); host pointers are staged through the
 *     context's own device buffers.
 *   - a quartic is its 35 coefficients (uint8, each < p) over the degree-4
 *     monomial basis in lex-ASCENDING order, x1 most significant: index 0 is
 *     x4^4, index 34 is x1^4  (monomials.py:182-196, search.py:92-98).
 *   - every dense vector over basis(deg,4) uses the same order:
 *       rank(a1,a2,a3,a4) = C(deg+3,3)-C(deg-a1+3,3) + C(e+2,2)-C(e-a2+2,2) + a3, e = deg-a1.
 *   - heights are int8: 1..bound, and 0 encodes "infinity" (math.inf in
 *     height.py:28); iterations counts operator applications (height.py:42-47).
 *   - return value 0 = success, negative = qfs_status; qfs_last_error() gives
 *     the message.  A context is single-threaded; use one per GPU.
 */
#ifndef QFS_H
#define QFS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QFS_ABI_VERSION 1

typedef enum qfs_status {
    QFS_OK = 0,
    QFS_EINVAL = -1,     /* bad argument / input violates a precondition (DomainError in errors.py:17) */
    QFS_ECUDA = -2,      /* CUDA runtime failure */
    QFS_EINVARIANT = -3, /* a Witt-carry numerator was not divisible by p (InternalInvariantError, polyring.py:397-398) */
    QFS_ENOMEM = -4      /* device memory exhausted even at the minimum chunk size */
} qfs_status;

typedef struct qfs_ctx qfs_ctx;

/* shape constants for a prime */
typedef struct qfs_shape {
    int32_t p;
    int32_t d;       /* deg f^(p-1) = 4(p-1)                       */
    int32_t D;       /* deg Delta_1(f^(p-1)) = 4p(p-1)             */
    int32_t N;       /* C(4p-1,3): operator dimension              */
    int32_t pitch;   /* internal row pitch of M in bytes (N rounded up to 128: rows start on 128-byte lines) */
    int32_t cap;     /* index of (x1x2x3x4)^(p-1) in basis(d,4)    */
    int64_t L;       /* C(D+3,3): dense length of Delta            */
} qfs_shape;

/* counters filled by the last qfs_heights call on the context */
typedef struct qfs_stats {
    int64_t surfaces;        /* B                                            */
    int64_t hard;            /* surfaces with height >= 2 (took the operator path) */
    int64_t matvec_steps;    /* sum over hard surfaces of operator applications */
    int64_t kernel_launches; /* CUDA kernels launched by the call            */
    int64_t chunks;          /* hard-surface chunks processed                */
    int64_t chunk_capacity;  /* hard surfaces per chunk                      */
    double  ms_power;        /* CUDA-event time of each stage, summed over chunks */
    double  ms_delta;
    double  ms_matrix;
    double  ms_matvec;
    double  ms_total;        /* first launch to last completion              */
    int64_t built;           /* surfaces whose Delta and M were built: = hard for qfs_heights, the ones the cap row left
                                undecided for qfs_heights_lazy, 0 for qfs_heights_free */
    double  ms_caprow;       /* qfs_heights_lazy: f^(p-1) and the cap row of the first step for every hard surface */
} qfs_stats;

int qfs_version(void);

/* 0 if p is supported by this build (3, 5, 7, 11, 13); fills *out when non-NULL. */
int qfs_get_shape(int p, qfs_shape *out);

/* Per-(p, device) context: index tables, workspaces, streams.
 * max_batch is a sizing hint (0 = default); larger batches still work.
 * Replaces nothing in the reference (it has no state); cf. the lru-cached
 * shape plan nttpower.py:197-250. */
int qfs_create(int p, int device, size_t max_batch, qfs_ctx **out);
void qfs_destroy(qfs_ctx *ctx);
const char *qfs_last_error(const qfs_ctx *ctx); /* ctx may be NULL: last create error */

/* Cap on device workspace the context may hold for operator matrices etc.
 * (bytes; 0 = default = 40% of the device's free memory at first use). */
int qfs_set_workspace_limit(qfs_ctx *ctx, size_t bytes);
/* Hard surfaces processed per chunk (0 = automatic). */
int qfs_set_chunk(qfs_ctx *ctx, size_t hard_surfaces_per_chunk);

/* ---- the hot path -------------------------------------------------------
 * Heights of B quartics.  Replaces the loop body of search._worker_block
 * (search.py:108-112) = SurfaceProblem checks (height.py:76-94) +
 * height_matrix (height.py:119-144) for every row of coeffs[B][35].
 * bound >= 1 (the reference default for quartics is 10, height.py:31-39).
 * heights[B], iters[B] are written on return (the call synchronises).
 * stream: a cudaStream_t cast to void* whose prior work the call must wait
 * for (NULL = none). */
int qfs_heights(qfs_ctx *ctx, const uint8_t *coeffs, size_t B, int bound,
                int8_t *heights, int8_t *iters, void *stream);
int qfs_get_stats(const qfs_ctx *ctx, qfs_stats *out);

/* The same heights and iteration counts by the polynomial iteration, without
 * Delta_1(f^(p-1)) and without the operator matrix: the on-device counterpart of
 * the reference's cross-check height_naive (height.py:97-116),
 *     g <- u(Delta * g),   computed as   g <- -f^(p-2) * u(Delta_1(f) * g)
 * (csrc/qfs_free.cuh; valid because g[cap] = 0 inside the loop).  Same
 * arguments and semantics as qfs_heights.  It is NOT the path the roofline of
 * this library is quoted on (that path builds and streams M, like the
 * reference's height_matrix); it exists to cross-check it and as a fast mode. */
int qfs_heights_free(qfs_ctx *ctx, const uint8_t *coeffs, size_t B, int bound,
                     int8_t *heights, int8_t *iters, void *stream);

/* The same heights and iteration counts on the operator-matrix path, with the
 * early exit of height.py:135-144 taken BEFORE the matrix is built where the first
 * step already decides: (M g)[cap] is one row of M, i.e. N entries of Delta
 * (M[cap, c] = Delta[(p^2-1) - c], mtsmatrix.py:249-281), which csrc/qfs_caprow.cuh
 * evaluates from the factorised Witt carry and dots with g.  A fraction 1 - 1/p of
 * the hard surfaces gets height 2 there; Delta and M are built, and the chain run,
 * only for the rest (qfs_stats.built).  Same arguments and semantics as qfs_heights.
 * Like qfs_heights_free it is NOT the path the roofline is quoted on: qfs_heights
 * builds M for every hard surface, as the reference does. */
int qfs_heights_lazy(qfs_ctx *ctx, const uint8_t *coeffs, size_t B, int bound,
                     int8_t *heights, int8_t *iters, void *stream);

/* ---- stage taps (parity against the reference's intermediates) ----------
 * All taps run the SAME kernels as qfs_heights on every input row (no
 * height-1 shortcut) and write the reference's layouts. */

/* g = f^(p-1) mod p, dense [B][N]; fedder[B] = 1 iff the (p-1,..,p-1)
 * coefficient is nonzero.  power_mod_p (polyring.py:253-272) +
 * fedder_survives (polyring.py:316-332) + to_dense (polyring.py:404-418). */
int qfs_stage_power(qfs_ctx *ctx, const uint8_t *coeffs, size_t B, uint8_t *g, uint8_t *fedder);

/* Delta = delta1(f^(p-1)) mod p, dense [B][L] over basis(D,4) (zero where the
 * reference's sparse result has no term).  delta1 (polyring.py:335-401) incl.
 * power_mod_small (nttpower.py:447-507). */
int qfs_stage_delta(qfs_ctx *ctx, const uint8_t *coeffs, size_t B, uint8_t *delta);

/* Operator matrix from a dense Delta: M[B][N][N] row-major uint8, column j =
 * u(Delta * m_j).  build_mts / mts_wics (mtsmatrix.py:287-295, 249-281);
 * MtsMatrix.entries holds the same residues as uint16 (mtsmatrix.py:96). */
int qfs_stage_matrix(qfs_ctx *ctx, const uint8_t *delta, size_t B, uint8_t *M);

/* Iterated matvec with early exit: v <- M v (mod p) up to max_steps times,
 * stopping at the first step k with v[cap] != 0 (height k+1).  matvec
 * (modmatrix.py:109-131) inside the loop of height.py:135-144.
 * M[B][N][N], v0[B][N]; trace (optional, may be NULL) [B][max_steps][N] gets
 * every v_k actually computed; heights/iters as in qfs_heights with
 * bound = max_steps+1. */
int qfs_stage_matvec_chain(qfs_ctx *ctx, const uint8_t *M, const uint8_t *v0, size_t B, int max_steps,
                           uint8_t *trace, int8_t *heights, int8_t *iters);

/* ---- plane cubic curves (n = 3) -------------------------------------------
 * Heights of B cubic forms in x1..x3 over F_p (elliptic curves: height 1 =
 * ordinary, 2 = supersingular), the other Calabi-Yau shape the reference's
 * drivers are exercised on (height.py:63-144, tests/test_height.py:131-140).
 * coeffs[B][10] over basis(3,3) in lex-ascending order, x1 most significant
 * (index 0 = x3^3 ... 9 = x1^3); p an odd prime <= 53; bound >= 1 must be
 * given (the reference has no default bound for n != 4, height.py:31-39).
 * Context-free (one kernel, everything in shared memory); errors are reported
 * through qfs_last_error(NULL).  Same output conventions as qfs_heights. */
int qfs_cubic_heights(int device, int p, const uint8_t *coeffs, size_t B, int bound,
                      int8_t *heights, int8_t *iters);

/* Heights of B forms of degree n in n variables, n = 2..6 (height.py:63-144 accept any n >= 2; the quartic context
 * and qfs_cubic_heights cover n = 4 and n = 3 at full speed, this is the general entry at toy sizes:
 * (n p + 1)^(n-1) <= 2^24).  coeffs[B][C(2n-1, n-1)]: the coefficients over MonomialBasis(n, n) of the reference,
 * lex-ascending with x1 most significant (monomials.py:182-196).  Matrix-free iteration; heights and iteration
 * counts are those of height_matrix and height_naive.  Context-free like qfs_cubic_heights. */
int qfs_form_heights(int device, int p, int n, const uint8_t *coeffs, size_t B, int bound,
                     int8_t *heights, int8_t *iters);

/* The reference's definitions executed literally on the device, for p = 3, 5, 7: g = f^(p-1) by dense multiplications
 * (power_mod_p, polyring.py:253-272), Delta_1(g) = ((lift g)^p - sum of the p-th powers of its terms) / p mod p with the
 * division checked (delta1, polyring.py:335-401), then g <- u(Delta g) until the Fedder coefficient survives (height_naive,
 * height.py:97-116; split_u, polyring.py:295-313).  Shares no kernel and no identity with qfs_heights / qfs_heights_free: the
 * on-device cross-check of both (a few ms per F_7 surface).  g_out [B][N] and delta_out [B][L] (dense, lex-ascending like the
 * stage taps) may be NULL; every buffer may live on the host or on the device.  Context-free like qfs_cubic_heights. */
int qfs_literal_heights(int device, int p, const uint8_t *coeffs, size_t B, int bound,
                        int8_t *heights, int8_t *iters, uint8_t *g_out, uint8_t *delta_out);

/* ---- export ---------------------------------------------------------------
 * Operator matrices of B quartics (given by their coefficient vectors) in the
 * reference's export layout: M16[B][N][N] row-major uint16 little-endian --
 * exactly the entry block of matrix_to_bytes (mtsmatrix.py:350-365) and the
 * values matrix_to_text prints (mtsmatrix.py:301-306); the caller adds the
 * "QFSMTX01" magic and the six-word header.  Replaces the body of cmd_matrix
 * (cli.py:108-122): power_mod_p + delta1 + build_mts.  M16 may be host or
 * device memory. */
int qfs_export_matrix(qfs_ctx *ctx, const uint8_t *coeffs, size_t B, uint16_t *M16);

/* ---- sampler ----------------------------------------------------------------
 * The `count` coefficient vectors a worker of the reference's search draws
 * (search.py:92-98, 103: numpy default_rng([seed, worker]).integers(0, p, 35),
 * zero draws redrawn), generated on the device: state_inc = {state_hi, state_lo,
 * inc_hi, inc_lo} of numpy's PCG64 bit generator right after seeding
 * (np.random.PCG64(np.random.SeedSequence([seed, worker])).state).  coeffs
 * [count][35] may be host or device memory.  *clean = 1 if the block is the
 * reference's stream bit for bit; 0 if a draw hit Lemire's rejection branch
 * (probability p / 2^32 per draw) or a row came out zero: the stream then
 * shifts from that point on and the caller draws this block on the host. */
int qfs_sample_quartics(qfs_ctx *ctx, const uint64_t state_inc[4], size_t count, uint8_t *coeffs,
                        int *clean);

/* ---- test hook -------------------------------------------------------------
 * Overwrites every device workspace the context currently holds with `byte`.
 * No kernel may depend on what a workspace held before the call that uses it
 * (recycled device memory is not zero); tests/test_gpu_api.py poisons the
 * workspaces between calls to prove it. */
int qfs_debug_fill_workspaces(qfs_ctx *ctx, int byte);

/* Resident CTAs per SM of the stage kernels as built and configured on this device (cudaOccupancyMaxActiveBlocksPerMultiprocessor):
 * [0] k_power_full, [1] k_delta_mma, [2] k_matrix_staged (with the fused first step), [3] k_chain.  The kernels are tuned for
 * specific counts; tests/test_gpu_api.py pins them so that a change that costs a CTA per SM is noticed. */
int qfs_debug_occupancy(const qfs_ctx *ctx, int ctas_per_sm[4]);

#ifdef __cplusplus
}
#endif
#endif /* QFS_H */
