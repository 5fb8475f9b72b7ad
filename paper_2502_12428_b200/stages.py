"""The reference's per-stage functions of the hot path, by their own names, on the GPU engine.

    g     = power_mod_p(f, p - 1)          polyring.py:253      k_power_full   (qfs_stage_power)
    one   = fedder_survives(g)             polyring.py:316
    delta = delta1(g)                      polyring.py:335      k_delta_mma    (qfs_stage_delta)
    m     = build_mts(delta, d, p, "wics") mtsmatrix.py:287     k_matrix_staged (qfs_stage_matrix)   [mtsmatrix.build_mts]
    gv    = to_dense(g)                    polyring.py:404
    gv    = matvec(m, gv)                  modmatrix.py:109     k_chain        (qfs_stage_matvec_chain)

so that `height_matrix` of the reference (height.py:119-144) reads the same against this package.  Polynomials of
degree > 4 live as DENSE vectors over the lex-ascending basis (x1 most significant, index 0 = x4^deg): `DenseForm`
quacks like the reference's SparsePoly where the hot path needs it (`degree`, `modulus`, `nvars`, `coefficient`,
`terms`, `is_zero`), `DenseVector` like its DenseVector (`values` as uint64).

One deviation, by construction of the Witt-carry kernel: `delta1`
is computed from the QUARTIC, through the factorisation Delta_1(f^(p-1)) = phi(A) - phi(f^(p-2)) Delta_1(f); it
accepts the g that `power_mod_p(f, p - 1)` returned (which remembers its f) and raises DomainError for any other
polynomial, instead of raising an arbitrary g to the p-th power as the reference does.
"""
from __future__ import annotations

import math

import numpy as np

from .errors import DomainError
from .quartic import NVARS, Quartic, coeff_vector


def _rank(e, deg):
    a1, a2, a3 = int(e[0]), int(e[1]), int(e[2])
    d2 = deg - a1
    return (math.comb(deg + 3, 3) - math.comb(deg - a1 + 3, 3) + math.comb(d2 + 2, 2) - math.comb(d2 - a2 + 2, 2) + a3)


class DenseForm:
    """A form of degree `degree` in x1..x4 over F_p as its dense coefficient vector (uint8, lex-ascending basis)."""

    nvars = NVARS

    def __init__(self, values, degree: int, modulus: int, origin=None):
        v = np.ascontiguousarray(values, dtype=np.uint8)
        if v.shape != (math.comb(degree + 3, 3),):
            raise DomainError(f"a form of degree {degree} in 4 variables has {math.comb(degree + 3, 3)} coefficients, got {v.shape}")
        v.flags.writeable = False
        self.values = v
        self._degree = int(degree)
        self.modulus = int(modulus)
        self._origin = origin          # the quartic f this is a power / carry of (None: unknown)

    @property
    def is_zero(self) -> bool:
        return not self.values.any()

    @property
    def degree(self) -> int:
        return -1 if self.is_zero else self._degree

    def is_homogeneous(self) -> bool:
        return True

    def coefficient(self, exps) -> int:
        e = tuple(int(x) for x in exps)
        if len(e) != NVARS or min(e) < 0 or sum(e) != self._degree:
            return 0
        return int(self.values[_rank(e, self._degree)])

    def terms(self):
        """(exponent tuple, coefficient) of the nonzero terms in basis order."""
        deg = self._degree
        nz = set(np.nonzero(self.values)[0].tolist())
        i = 0
        for a1 in range(deg + 1):
            for a2 in range(deg - a1 + 1):
                for a3 in range(deg - a1 - a2 + 1):
                    if i in nz:
                        yield (a1, a2, a3, deg - a1 - a2 - a3), int(self.values[i])
                    i += 1

    def __len__(self):
        return int(np.count_nonzero(self.values))

    def __repr__(self):
        return f"DenseForm(degree {self._degree} over F_{self.modulus}, {len(self)} terms)"


class DenseVector:
    """Coefficient vector over basis(degree, 4), `values` uint64 as in the reference (polyring.py:404-418)."""

    def __init__(self, values, degree: int, modulus: int):
        self.values = np.ascontiguousarray(values, dtype=np.uint64)
        self.degree = int(degree)
        self.modulus = int(modulus)

    def __len__(self):
        return int(self.values.shape[0])


def _engine(p, device):
    from .engine import get_engine
    from .height import _check_engine_shape
    _check_engine_shape(p)
    return get_engine(p, device)


def power_mod_p(f, k: int, device: int = 0) -> DenseForm:
    """f^k mod p for k = p - 1, the power the hot path takes (polyring.py:253-272, height.py:123)."""
    p = int(getattr(f, "modulus"))
    if int(k) != p - 1:
        raise DomainError(f"the GPU engine raises a quartic to the power p-1 = {p - 1} only, got k={k}")
    c = coeff_vector(f, p)
    g, _ = _engine(p, device).stage_power(c[None, :])
    return DenseForm(g[0], 4 * (p - 1), p, origin=np.array(c, dtype=np.uint8))


def fedder_survives(g) -> bool:
    """Coefficient of (x1 x2 x3 x4)^(p-1) in g is nonzero: height 1 (polyring.py:316-332)."""
    p = int(g.modulus)
    return g.coefficient((p - 1,) * NVARS) != 0


def delta1(g, device: int = 0) -> DenseForm:
    """Delta_1(g) = ((lift g)^p - sum of p-th powers of the terms) / p mod p (polyring.py:335-401) for g = f^(p-1)."""
    origin = getattr(g, "_origin", None)
    p = int(g.modulus)
    if origin is None or getattr(g, "_degree", None) != 4 * (p - 1):
        raise DomainError("delta1 on the GPU engine is defined for the g that power_mod_p(f, p-1) returned: the Witt carry is "
                          "assembled from the quartic f (Delta_1(f^(p-1)) = phi(A) - phi(f^(p-2)) Delta_1(f)); an arbitrary "
                          "polynomial is not supported")
    dl = _engine(p, device).stage_delta(origin[None, :])
    return DenseForm(dl[0], 4 * p * (p - 1), p, origin=origin)


def to_dense(g, basis=None) -> DenseVector:
    """Coefficient vector of g over basis(deg g, 4) (polyring.py:404-418); `basis` is accepted for signature parity."""
    if isinstance(g, Quartic):
        return DenseVector(g.coeffs, 4, g.modulus)
    if not isinstance(g, DenseForm):
        raise DomainError("to_dense expects a Quartic or a DenseForm")
    return DenseVector(g.values, g._degree, g.modulus)


def matvec(m, v, device: int = 0) -> DenseVector:
    """M v mod p on the device (modmatrix.py:109-131); any reduction cadence within the overflow budget gives these residues."""
    vals = np.asarray(v.values if hasattr(v, "values") else v)
    if vals.shape != (m.cols,):
        raise DomainError(f"vector of length {vals.shape} against a {m.rows}x{m.cols} matrix")
    if m.rows != m.cols:
        raise DomainError("the GPU engine multiplies by the square operator matrices of the height loop")
    if vals.size and int(vals.max()) >= m.p:
        raise DomainError("vector entries must be reduced mod p")
    eng = _engine(m.p, device)
    if m.rows != eng.shape.N:
        raise DomainError(f"matrix size {m.rows} is not the operator size {eng.shape.N} of quartics over F_{m.p}")
    _, _, tr = eng.stage_matvec_chain(np.asarray(m.entries, dtype=np.uint8), vals.astype(np.uint8), 1, trace=True)
    return DenseVector(tr[0][0], m.target_degree, m.p)
