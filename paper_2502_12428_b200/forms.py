"""Calabi-Yau hypersurfaces in n != 3, 4 variables: a form of degree n in x1..xn over F_p (n = 2, 5, 6 at toy sizes).

The reference's drivers take any n >= 2 (SurfaceProblem, height.py:63-94; height_matrix / height_naive, height.py:97-144); the
quartic engine covers n = 4, csrc/qfs_cubic.cuh n = 3, and csrc/qfs_form.cuh (qfs_form_heights) everything else the box
(n p + 1)^(n-1) <= 2^24 admits -- n = 2 with p <= 53, n = 5 with p <= 11, n = 6 with p = 3.  Coefficient order:
`MonomialBasis(n, n)` of the reference, lex-ascending with x1 most significant (monomials.py:182-196).
"""
from __future__ import annotations

import functools

import numpy as np

from .errors import DomainError

MAX_N = 6
MAX_BOX = 1 << 24


@functools.lru_cache(maxsize=None)
def exponents(n: int):
    """basis(n, n) in lex-ascending order, x1 most significant: index 0 = xn^n, last = x1^n."""
    out = []

    def rec(prefix, left):
        if len(prefix) == n - 1:
            out.append(tuple(prefix) + (left,))
            return
        for a in range(left + 1):
            rec(prefix + [a], left - a)

    rec([], n)
    return tuple(out)


@functools.lru_cache(maxsize=None)
def index_of(n: int):
    return {e: i for i, e in enumerate(exponents(n))}


class Form:
    """A form of degree n in x1..xn over F_p as a read-only uint8 coefficient vector (quacks like the reference's SparsePoly)."""

    __slots__ = ("coeffs", "modulus", "nvars")

    def __init__(self, coeffs, modulus: int, nvars: int):
        if not 2 <= nvars <= MAX_N:
            raise DomainError(f"the GPU engine handles forms in 2..{MAX_N} variables, got n={nvars}")
        c = np.asarray(coeffs)
        if c.shape != (len(exponents(nvars)),):
            raise DomainError(f"a form of degree {nvars} in {nvars} variables has {len(exponents(nvars))} coefficients, got shape {c.shape}")
        if modulus < 2 or modulus > 255:
            raise DomainError(f"modulus {modulus} out of range for the uint8 engine")
        c = (np.asarray(c, dtype=np.int64) % modulus).astype(np.uint8)
        c.flags.writeable = False
        self.coeffs = c
        self.modulus = int(modulus)
        self.nvars = int(nvars)

    @classmethod
    def from_terms(cls, terms, modulus: int, nvars: int):
        idx = index_of(nvars)
        acc = np.zeros(len(idx), dtype=np.int64)
        for exps, c in terms:
            e = tuple(int(x) for x in exps)
            if len(e) != nvars or min(e) < 0:
                raise DomainError(f"bad exponent vector {exps}")
            if sum(e) != nvars:
                raise DomainError(f"term {e} is not of degree {nvars} (Calabi-Yau condition)")
            acc[idx[e]] += int(c) % modulus
        return cls(acc % modulus, modulus, nvars)

    @property
    def is_zero(self) -> bool:
        return not self.coeffs.any()

    @property
    def degree(self) -> int:
        return -1 if self.is_zero else self.nvars

    def is_homogeneous(self) -> bool:
        return True

    def terms(self):
        ex = exponents(self.nvars)
        for i in np.nonzero(self.coeffs)[0]:
            yield ex[int(i)], int(self.coeffs[i])

    def coefficient(self, exps) -> int:
        i = index_of(self.nvars).get(tuple(int(x) for x in exps))
        return int(self.coeffs[i]) if i is not None else 0

    def __len__(self):
        return int(np.count_nonzero(self.coeffs))

    def __eq__(self, other):
        return (isinstance(other, Form) and self.nvars == other.nvars and self.modulus == other.modulus
                and np.array_equal(self.coeffs, other.coeffs))

    def __hash__(self):
        return hash((self.nvars, self.modulus, self.coeffs.tobytes()))

    def __repr__(self):
        ex = exponents(self.nvars)
        parts = []
        for i in range(len(ex) - 1, -1, -1):
            if self.coeffs[i]:
                mono = "*".join(f"x{j + 1}" + (f"^{e}" if e > 1 else "") for j, e in enumerate(ex[i]) if e)
                parts.append(mono if self.coeffs[i] == 1 else f"{int(self.coeffs[i])}*{mono}")
        return f"Form(n={self.nvars}, p={self.modulus}, {' + '.join(parts) or '0'})"


def form_vector(f, p: int, n: int) -> np.ndarray:
    """uint8 coefficient vector of a Form, a reference SparsePoly in n variables (duck-typed), or a raw vector."""
    if isinstance(f, Form):
        if f.modulus != p or f.nvars != n:
            raise DomainError(f"f is a form in {f.nvars} variables over F_{f.modulus}, expected n={n}, p={p}")
        return f.coeffs
    if hasattr(f, "terms") and hasattr(f, "nvars"):
        if f.nvars != n:
            raise DomainError(f"f has {f.nvars} variables, expected {n}")
        return Form.from_terms(f.terms(), getattr(f, "modulus", None) or p, n).coeffs
    c = np.asarray(f)
    if c.shape != (len(exponents(n)),):
        raise DomainError(f"expected a {len(exponents(n))}-entry coefficient vector, got shape {c.shape}")
    if (c < 0).any() or (c >= p).any():
        raise DomainError(f"coefficients must lie in [0, {p})")
    return c.astype(np.uint8)


def form_height_batch(p: int, n: int, coeffs, bound: int, device: int = 0):
    """Heights of B forms of degree n in n variables given as rows of `coeffs`; returns (heights int8[B], iterations int8[B]),
    0 encoding infinity.  `bound` has no default: the reference knows none for n != 4 (height.py:31-39)."""
    from . import _native
    from .height import is_prime
    if not isinstance(n, (int, np.integer)) or not 2 <= n <= MAX_N:
        raise DomainError(f"the GPU engine handles forms in 2..{MAX_N} variables, got n={n}")
    if not is_prime(p):
        raise DomainError(f"p={p} is not prime")
    if p < 3 or (n * p + 1) ** (n - 1) > MAX_BOX:
        raise DomainError(f"n={n}, p={p} is outside the general-n kernel (odd p with (n p + 1)^(n-1) <= 2^24)")
    if not isinstance(bound, (int, np.integer)) or bound < 1:
        raise DomainError(f"bound must be a positive integer, got {bound}")
    if bound > 127:
        raise DomainError("bound must be <= 127 (heights are int8 at the C ABI)")
    nc = len(exponents(n))
    c = np.asarray(coeffs)
    if c.ndim != 2 or c.shape[1] != nc:
        raise DomainError(f"coeffs must have shape [B, {nc}], got {c.shape}")
    if c.size and ((c < 0).any() or (c >= p).any()):
        raise DomainError(f"coefficients must lie in [0, {p})")
    c = np.ascontiguousarray(c, dtype=np.uint8)
    if c.size and not c.any(axis=1).all():
        raise DomainError("f must be nonzero")
    hs = np.empty(c.shape[0], dtype=np.int8)
    its = np.empty(c.shape[0], dtype=np.int8)
    lib = _native.load()
    rc = lib.qfs_form_heights(int(device), int(p), int(n), c.ctypes.data, c.shape[0], int(bound), hs.ctypes.data, its.ctypes.data)
    _native.raise_for(rc, lib.qfs_last_error(None).decode())
    return hs, its
