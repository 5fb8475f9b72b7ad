"""The reference's definitions executed literally on the GPU (csrc/qfs_literal.cuh): the independent cross-check.

`height_naive` of the reference (height.py:97-116) iterates g <- u(Delta g) on polynomials, with g = f^(p-1) from
`power_mod_p` (polyring.py:253-272) and Delta = delta1(g) from the definition ((lift g)^p minus the p-th powers of the
terms, divided by p: polyring.py:335-401).  The engine's two modes (`method="matrix"`, `method="naive"`) both start
from the Witt-carry factorisation of DESIGN.md section 3; `literal_heights` does not: dense multiplications, the checked
division, the splitting operator.  Small primes only (p = 3, 5, 7; a few ms per F_7 surface), so it is what the tests
and tools/crosscheck.py hold the engine against beyond the sizes the goldens cover -- never a fallback of the engine.
"""
from __future__ import annotations

import math

import numpy as np

from . import _native
from .errors import DomainError
from .quartic import NCOEFF

LITERAL_PRIMES = (3, 5, 7)


def literal_heights(p: int, coeffs, bound: int = 10, device: int = 0, want_g: bool = False, want_delta: bool = False):
    """(heights int8[B], iterations int8[B][, g uint8[B,N]][, delta uint8[B,L]]) of B quartics over F_p, p in (3, 5, 7).

    Heights use 0 for infinity; g = f^(p-1) and delta = Delta_1(g) are dense vectors over the lex-ascending bases of
    degree 4(p-1) and 4p(p-1), as the stage taps return them.  With want_delta=True every surface gets its Delta
    (otherwise the surfaces of height 1 skip it, like the reference's driver)."""
    if p not in LITERAL_PRIMES:
        raise DomainError(f"the literal route runs for p in {LITERAL_PRIMES}, got p={p}")
    if not isinstance(bound, (int, np.integer)) or bound < 1:
        raise DomainError(f"bound must be a positive integer, got {bound}")
    c = np.ascontiguousarray(coeffs, dtype=np.uint8)
    if c.ndim != 2 or c.shape[1] != NCOEFF:
        raise DomainError(f"coeffs must have shape [B, {NCOEFF}], got {c.shape}")
    B = c.shape[0]
    d = 4 * (p - 1)
    hs = np.zeros(B, dtype=np.int8)
    its = np.zeros(B, dtype=np.int8)
    g = np.empty((B, math.comb(d + 3, 3)), dtype=np.uint8) if want_g else None
    dl = np.empty((B, math.comb(p * d + 3, 3)), dtype=np.uint8) if want_delta else None
    lib = _native.load()
    rc = lib.qfs_literal_heights(int(device), int(p), c.ctypes.data, B, int(bound), hs.ctypes.data, its.ctypes.data,
                                 g.ctypes.data if want_g else None, dl.ctypes.data if want_delta else None)
    if rc != 0:
        _native.raise_for(rc, lib.qfs_last_error(None).decode())
    out = (hs, its)
    if want_g:
        out += (g,)
    if want_delta:
        out += (dl,)
    return out
