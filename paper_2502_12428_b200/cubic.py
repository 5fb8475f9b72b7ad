"""Plane cubic curves (n = 3): the 10-coefficient counterpart of quartic.Quartic, and the batch entry point.

Coefficient order: `MonomialBasis(3, 3)` of the reference, lex-ascending with x1 most significant -- index 0 is
x3^3, index 9 is x1^3 (monomials.py:182-196).  Heights come from qfs_cubic_heights (csrc/qfs_cubic.cuh).
"""
from __future__ import annotations

import numpy as np

from .errors import DomainError

NVARS3 = 3
EXPONENTS3 = tuple((a1, a2, 3 - a1 - a2) for a1 in range(4) for a2 in range(4 - a1))
INDEX_OF3 = {e: i for i, e in enumerate(EXPONENTS3)}
NCOEFF3 = len(EXPONENTS3)  # 10
MAX_P3 = 53


class Cubic:
    """A cubic form in x1..x3 over F_p as a read-only uint8[10] coefficient vector (quacks like SparsePoly)."""

    __slots__ = ("coeffs", "modulus")
    nvars = NVARS3

    def __init__(self, coeffs, modulus: int):
        c = np.asarray(coeffs)
        if c.shape != (NCOEFF3,):
            raise DomainError(f"a cubic in 3 variables has {NCOEFF3} coefficients, got shape {c.shape}")
        if modulus < 2 or modulus > 255:
            raise DomainError(f"modulus {modulus} out of range for the uint8 engine")
        c = (np.asarray(c, dtype=np.int64) % modulus).astype(np.uint8)
        c.flags.writeable = False
        self.coeffs = c
        self.modulus = int(modulus)

    @classmethod
    def from_terms(cls, terms, modulus: int):
        acc = np.zeros(NCOEFF3, dtype=np.int64)
        for exps, c in terms:
            e = tuple(int(x) for x in exps)
            if len(e) != NVARS3 or min(e) < 0:
                raise DomainError(f"bad exponent vector {exps}")
            if sum(e) != 3:
                raise DomainError(f"term {e} is not of degree 3 (Calabi-Yau condition)")
            acc[INDEX_OF3[e]] += int(c) % modulus
        return cls(acc % modulus, modulus)

    @property
    def is_zero(self) -> bool:
        return not self.coeffs.any()

    @property
    def degree(self) -> int:
        return -1 if self.is_zero else 3

    def is_homogeneous(self) -> bool:
        return True

    def terms(self):
        for i in np.nonzero(self.coeffs)[0]:
            yield EXPONENTS3[int(i)], int(self.coeffs[i])

    def coefficient(self, exps) -> int:
        i = INDEX_OF3.get(tuple(int(x) for x in exps))
        return int(self.coeffs[i]) if i is not None else 0

    def __len__(self):
        return int(np.count_nonzero(self.coeffs))

    def __eq__(self, other):
        return isinstance(other, Cubic) and self.modulus == other.modulus and np.array_equal(self.coeffs, other.coeffs)

    def __hash__(self):
        return hash((self.modulus, self.coeffs.tobytes()))

    def __repr__(self):
        parts = []
        for i in range(NCOEFF3 - 1, -1, -1):
            if self.coeffs[i]:
                mono = "*".join(f"x{j + 1}" + (f"^{e}" if e > 1 else "") for j, e in enumerate(EXPONENTS3[i]) if e)
                parts.append(mono if self.coeffs[i] == 1 else f"{int(self.coeffs[i])}*{mono}")
        return f"Cubic(p={self.modulus}, {' + '.join(parts) or '0'})"


def cubic_vector(f, p: int) -> np.ndarray:
    """uint8[10] coefficient vector of a Cubic, a reference SparsePoly in 3 variables (duck-typed), or a raw vector."""
    if isinstance(f, Cubic):
        if f.modulus != p:
            raise DomainError(f"f has modulus {f.modulus}, expected {p}")
        return f.coeffs
    if hasattr(f, "terms") and hasattr(f, "nvars"):
        if f.nvars != NVARS3:
            raise DomainError(f"f has {f.nvars} variables, expected 3")
        return Cubic.from_terms(f.terms(), getattr(f, "modulus", None) or p).coeffs
    c = np.asarray(f)
    if c.shape != (NCOEFF3,):
        raise DomainError(f"expected a 10-entry coefficient vector, got shape {c.shape}")
    if (c < 0).any() or (c >= p).any():
        raise DomainError(f"coefficients must lie in [0, {p})")
    return c.astype(np.uint8)


def cubic_height_batch(p: int, coeffs, bound: int, device: int = 0):
    """Heights of B plane cubics given as rows of `coeffs` (uint8 [B,10]); returns (heights int8[B], iterations int8[B]),
    0 encoding infinity.  `bound` has no default: the reference knows none for n != 4 (height.py:31-39)."""
    from . import _native
    from .height import is_prime
    if not is_prime(p):
        raise DomainError(f"p={p} is not prime")
    if p < 3 or p > MAX_P3:
        raise DomainError(f"the cubic-curve kernel handles odd primes up to {MAX_P3}, got p={p}")
    if not isinstance(bound, (int, np.integer)) or bound < 1:
        raise DomainError(f"bound must be a positive integer, got {bound}")
    if bound > 127:
        raise DomainError("bound must be <= 127 (heights are int8 at the C ABI)")
    c = np.asarray(coeffs)
    if c.ndim != 2 or c.shape[1] != NCOEFF3:
        raise DomainError(f"coeffs must have shape [B, {NCOEFF3}], got {c.shape}")
    if c.size and ((c < 0).any() or (c >= p).any()):
        raise DomainError(f"coefficients must lie in [0, {p})")
    c = np.ascontiguousarray(c, dtype=np.uint8)
    if c.size and not c.any(axis=1).all():
        raise DomainError("f must be nonzero")
    hs = np.empty(c.shape[0], dtype=np.int8)
    its = np.empty(c.shape[0], dtype=np.int8)
    lib = _native.load()
    rc = lib.qfs_cubic_heights(int(device), int(p), c.ctypes.data, c.shape[0], int(bound), hs.ctypes.data, its.ctypes.data)
    _native.raise_for(rc, lib.qfs_last_error(None).decode())
    return hs, its
