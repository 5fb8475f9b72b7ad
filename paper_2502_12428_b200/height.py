"""Drop-in for the reference's height driver (qfsplit/height.py) backed by the B200 engine.

Same names, argument meaning, results and error behaviour as the reference for the hot path:

    SurfaceProblem(p, n, f, bound=None)            height.py:63-94   (validation, default bound 10 for n=4)
    HeightResult(height, bound_used, iterations)   height.py:42-60   (height int or math.inf)
    height_matrix(prob, algorithm="wics")          height.py:119-144
    default_bound(n), INFINITE                     height.py:28-39

plus the two batch entry points the reference only has as a loop body (search.py:108-112):

    height_of_coeffs(p, coeffs[35], bound=10)
    height_batch(p, coeffs[B,35], bound=10, devices=None) -> (heights int8[B], iterations int8[B])

All heights are computed by libqfs.so on the GPU (EngineUnavailableError without it; there is no
CPU fallback).  `height_naive` (the reference's cross-check driver) is the matrix-free GPU iteration of
csrc/qfs_free.cuh; the independent CPU check of this package is the oracle under oracle/, used by the tests only.
"""
from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np

from .errors import DomainError
from .quartic import NCOEFF, NVARS, coeff_vector

INFINITE = math.inf
SUPPORTED_PRIMES = (3, 5, 7, 11, 13)


def is_prime(n: int) -> bool:
    """Primality of a Python int (modarith.py:122-147 is a Miller-Rabin; trial division is enough for the
    primes the uint8 engine can hold, and still exact for anything else a caller passes)."""
    if not isinstance(n, (int, np.integer)) or n < 2:
        return False
    n = int(n)
    if n < 4:
        return True
    if n % 2 == 0:
        return False
    q = 3
    while q * q <= n:
        if n % q == 0:
            return False
        q += 2
    return True


def default_bound(n: int) -> int:
    """Proven ceiling of finite heights: 10 for quartic K3 surfaces, none known otherwise (height.py:31-39)."""
    if n == 4:
        return 10
    raise DomainError(f"no default height bound for n={n}; pass bound explicitly")


@dataclass(frozen=True)
class HeightResult:
    """height is a positive int or math.inf; iterations counts operator applications (height.py:42-60)."""

    height: object
    bound_used: int
    iterations: int

    def __post_init__(self):
        if self.is_finite:
            if not isinstance(self.height, int) or self.height < 1:
                raise DomainError(f"finite height must be a positive integer, got {self.height}")
            if self.height > self.bound_used:
                raise DomainError("finite height exceeds the bound used")

    @property
    def is_finite(self) -> bool:
        return not (isinstance(self.height, float) and math.isinf(self.height))


@dataclass(frozen=True)
class SurfaceProblem:
    """A degree-n hypersurface in n variables over F_p with a height bound (height.py:63-94).

    `f` is a Quartic or any object with the reference SparsePoly's attributes.  The checks and
    their order are the reference's; a valid problem that is not a quartic in 4 variables is
    rejected later, by height_matrix, because only that shape has a GPU path.
    """

    p: int
    n: int
    f: object
    bound: int | None = None

    def __post_init__(self):
        if not is_prime(self.p):
            raise DomainError(f"p={self.p} is not prime")
        if self.n < 2:
            raise DomainError(f"need at least 2 variables, got n={self.n}")
        if self.f.nvars != self.n:
            raise DomainError(f"f has {self.f.nvars} variables, expected {self.n}")
        if self.f.modulus != self.p:
            raise DomainError(f"f has modulus {self.f.modulus}, expected {self.p}")
        if self.f.is_zero:
            raise DomainError("f must be nonzero")
        if not self.f.is_homogeneous() or self.f.degree != self.n:
            raise DomainError(f"f must be homogeneous of degree {self.n} (Calabi-Yau condition)")
        if self.bound is None:
            object.__setattr__(self, "bound", default_bound(self.n))
        if not isinstance(self.bound, int) or self.bound < 1:
            raise DomainError(f"bound must be a positive integer, got {self.bound}")


def decode_height(h: int):
    """C-ABI height code -> reference value: 0 encodes infinity (include/qfs.h)."""
    return INFINITE if int(h) == 0 else int(h)


def _check_engine_shape(p: int, n: int = NVARS):
    if n != NVARS:
        raise DomainError(f"the quartic engine computes heights of quartics in 4 variables (cubics: cubic.py, other n: forms.py); got n={n}")
    if p not in SUPPORTED_PRIMES:
        raise DomainError(f"p={p} is not supported by the GPU engine (supported: {SUPPORTED_PRIMES})")


def _check_batch(p: int, coeffs, bound):
    if not is_prime(p):
        raise DomainError(f"p={p} is not prime")
    _check_engine_shape(p)
    if not isinstance(bound, (int, np.integer)) or bound < 1:
        raise DomainError(f"bound must be a positive integer, got {bound}")
    if bound > 127:
        raise DomainError("bound must be <= 127 (heights are int8 at the C ABI)")
    c = np.asarray(coeffs)
    if c.ndim != 2 or c.shape[1] != NCOEFF:
        raise DomainError(f"coeffs must have shape [B, {NCOEFF}], got {c.shape}")
    if c.dtype == np.uint8 and c.shape[0] > 4096:
        # large batches: residues >= p and zero forms are caught by the first kernel of the pipeline (k_fedder raises the input
        # flag, the library reports QFS_EINVAL, the binding raises DomainError): no host pass over the batch
        return np.ascontiguousarray(c)
    if c.size and ((c < 0).any() or (c >= p).any()):
        raise DomainError(f"coefficients must lie in [0, {p})")
    c = np.ascontiguousarray(c, dtype=np.uint8)
    if c.size and not c.any(axis=1).all():
        raise DomainError("f must be nonzero")
    return c


def split_blocks(total: int, parts: int):
    """Contiguous (start, count) blocks, the first `total % parts` one longer -- the reference's worker
    partition (search.py:128-135), used here with worker = GPU."""
    parts = max(1, min(int(parts), int(total))) if total > 0 else 1
    base, extra = divmod(int(total), parts)
    out, start = [], 0
    for w in range(parts):
        cnt = base + (1 if w < extra else 0)
        out.append((start, cnt))
        start += cnt
    return out


def height_batch(p: int, coeffs, bound: int = 10, devices=None, method: str = "matrix", out=None):
    """Heights of B quartics given as rows of `coeffs` (uint8 [B,35], reference basis order).

    Returns (heights int8[B], iterations int8[B]) with 0 encoding infinity.  `devices` is a list of
    CUDA device indices (default: [0]); the batch is cut into contiguous blocks, one per device,
    each driven from its own host thread through its own context, and the results are gathered on
    the host -- surfaces are independent, there is no collective.

    method: "matrix" (default; builds and streams the operator matrix like the reference's height_matrix) or
    "naive" (the polynomial iteration without the matrix, qfs_heights_free: the on-device counterpart of the
    reference's height_naive cross-check; same heights and iteration counts), or "literal" (p <= 7: the
    reference's definitions executed literally on the device, csrc/qfs_literal.cuh -- the independent cross-check),
    or "lazy" (the matrix path with the loop's early exit taken before the matrix is built: the cap row of the first
    step, N entries of Delta, decides 1 - 1/p of the hard surfaces; Delta and M are built for the rest only,
    qfs_heights_lazy; same heights and iteration counts).
    out: optional pair of int8[B] numpy arrays to receive the results (e.g. pinned host memory).
    """
    if method not in ("matrix", "naive", "literal", "lazy"):
        raise DomainError(f"unknown method {method!r}, expected 'matrix', 'naive', 'literal' or 'lazy'")
    free = method == "naive"
    lazy = method == "lazy"
    from .engine import get_engine
    c = _check_batch(p, coeffs, bound)
    B = c.shape[0]
    if method == "literal":   # the reference's definitions executed literally (literal.py): the cross-check route, p <= 7, one device
        from .literal import literal_heights
        hs, its = literal_heights(p, c, int(bound), 0 if devices is None else int(list(devices)[0]))
        if out is not None:
            out[0][:] = hs
            out[1][:] = its
            return out[0], out[1]
        return hs, its
    if out is not None:
        heights, iters = out
        for a in (heights, iters):
            if not isinstance(a, np.ndarray) or a.dtype != np.int8 or a.shape != (B,) or not a.flags.c_contiguous:
                raise DomainError(f"out must be a pair of contiguous int8 arrays of length {B}")
    else:
        heights = np.empty(B, dtype=np.int8)
        iters = np.empty(B, dtype=np.int8)
    devs = [0] if devices is None else [int(d) for d in devices]
    if not devs:
        raise DomainError("devices must name at least one GPU")
    if B == 0:
        return heights, iters
    blocks = split_blocks(B, len(devs))
    if len(blocks) == 1:
        get_engine(p, devs[0]).heights(c, int(bound), out=(heights, iters), matrix_free=free, lazy=lazy)
        return heights, iters
    errors = []

    def work(dev, start, cnt):
        try:
            get_engine(p, dev).heights(c[start:start + cnt], int(bound),
                                       out=(heights[start:start + cnt], iters[start:start + cnt]), matrix_free=free, lazy=lazy)
        except Exception as exc:  # re-raised on the caller's thread
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(dev, s, n)) for dev, (s, n) in zip(devs, blocks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    return heights, iters


def height_of_coeffs(p: int, coeffs, bound: int = 10, device: int = 0, method: str = "matrix") -> HeightResult:
    """HeightResult of one quartic given as its 35-entry coefficient vector."""
    c = np.asarray(coeffs)
    if c.shape != (NCOEFF,):
        raise DomainError(f"expected a {NCOEFF}-entry coefficient vector, got shape {c.shape}")
    hs, its = height_batch(p, c.reshape(1, NCOEFF), bound, devices=[device], method=method)
    return HeightResult(decode_height(hs[0]), int(bound), int(its[0]))


def height_matrix(prob, algorithm: str = "wics", device: int = 0) -> HeightResult:
    """Height by the operator-matrix method on the GPU (height.py:119-144).

    `algorithm` names the reference's matrix builder ("triv", "merge", "wics"); all three produce
    the same entries (mtsmatrix.py:173-281) and the GPU builder produces those entries too, so the
    argument is validated and otherwise ignored.
    """
    if algorithm not in ("triv", "merge", "wics"):
        raise DomainError(f"unknown matrix algorithm {algorithm!r}")
    if prob.n != NVARS:
        return _other_n_height(prob, device)
    _check_engine_shape(prob.p, prob.n)
    c = coeff_vector(prob.f, prob.p)
    return height_of_coeffs(prob.p, c, prob.bound, device)


def height_naive(prob, device: int = 0) -> HeightResult:
    """Height by the polynomial iteration g <- u(Delta g) without the operator matrix (height.py:97-116), on the GPU.

    The reference keeps this driver as the independent check of height_matrix (same height, bound_used and
    iterations: tests/test_acceptance.py:128-138); here it is the matrix-free kernel of csrc/qfs_free.cuh.
    """
    if prob.n != NVARS:
        return _other_n_height(prob, device)
    _check_engine_shape(prob.p, prob.n)
    c = coeff_vector(prob.f, prob.p)
    return height_of_coeffs(prob.p, c, prob.bound, device, method="naive")


def _other_n_height(prob, device: int = 0) -> HeightResult:
    """n = 3: csrc/qfs_cubic.cuh; n = 2, 5, 6: csrc/qfs_form.cuh.  The operators are small there, so both drivers run the
    matrix-free iteration; the results are the reference's (tests/golden/cubics.json, tests/golden/forms.json)."""
    if prob.n == 3:
        return _cubic_height(prob, device)
    from .forms import form_height_batch, form_vector
    hs, its = form_height_batch(prob.p, prob.n, form_vector(prob.f, prob.p, prob.n)[None, :], prob.bound, device)
    return HeightResult(decode_height(hs[0]), int(prob.bound), int(its[0]))


def _cubic_height(prob, device: int = 0) -> HeightResult:
    """n = 3 (plane cubic curves): one kernel, csrc/qfs_cubic.cuh.  The operator matrices are at most 703 x 703 here, so
    both drivers run the matrix-free iteration; the results are the reference's (tests/golden/cubics.json)."""
    from .cubic import cubic_height_batch, cubic_vector
    hs, its = cubic_height_batch(prob.p, cubic_vector(prob.f, prob.p)[None, :], prob.bound, device)
    return HeightResult(decode_height(hs[0]), int(prob.bound), int(its[0]))
