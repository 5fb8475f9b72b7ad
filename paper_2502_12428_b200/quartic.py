"""Host-side representation of a quartic form in x1..x4 over F_p: its 35 coefficients.

This is the only polynomial type the GPU path needs (everything of higher degree lives on the
device).  The coefficient order is the reference's: `MonomialBasis(4, 4)` lex-ascending with x1
most significant -- index 0 is x4^4, index 34 is x1^4 (monomials.py:182-196, search.py:92-98).

`Quartic` quacks enough like the reference's `SparsePoly` (polyring.py:34-151: `nvars`, `modulus`,
`degree`, `is_zero`, `is_homogeneous()`, `terms()`, `coefficient()`) that `SurfaceProblem` and the
drivers accept either; `coeff_vector()` converts any such object to the 35-vector.  The text
grammar is the reference's human format `c*x1^a*x2^b + ...` (polyring.py:438-520) and its compact
format `c:a,b,c,d` (polyring.py:523-561), re-implemented here because the reference package is
not present on the GPU box.
"""
from __future__ import annotations

import numpy as np

from .errors import DomainError, ParseError

NVARS = 4
DEGREE = 4

# basis(4,4) in lex-ascending order, x1 most significant
EXPONENTS = tuple((a1, a2, a3, 4 - a1 - a2 - a3)
                  for a1 in range(5) for a2 in range(5 - a1) for a3 in range(5 - a1 - a2))
INDEX_OF = {e: i for i, e in enumerate(EXPONENTS)}
NCOEFF = len(EXPONENTS)  # 35


class Quartic:
    """A quartic form over F_p as a read-only uint8[35] coefficient vector."""

    __slots__ = ("coeffs", "modulus")
    nvars = NVARS

    def __init__(self, coeffs, modulus: int):
        c = np.asarray(coeffs)
        if c.shape != (NCOEFF,):
            raise DomainError(f"a quartic in 4 variables has {NCOEFF} coefficients, got shape {c.shape}")
        if modulus < 2 or modulus > 255:
            raise DomainError(f"modulus {modulus} out of range for the uint8 engine")
        c = np.asarray(c % modulus if c.dtype.kind in "iu" else c, dtype=np.int64) % modulus
        c = c.astype(np.uint8)
        c.flags.writeable = False
        self.coeffs = c
        self.modulus = int(modulus)

    # -- SparsePoly-compatible surface ------------------------------------------------------
    @classmethod
    def from_terms(cls, terms, modulus: int):
        """Build from (exponent 4-tuple, coefficient) pairs; repeated exponents add (polyring.py:62-101)."""
        acc = np.zeros(NCOEFF, dtype=np.int64)
        for exps, c in terms:
            e = tuple(int(x) for x in exps)
            if len(e) != NVARS or min(e) < 0:
                raise DomainError(f"bad exponent vector {exps}")
            if sum(e) != DEGREE:
                raise DomainError(f"term {e} is not of degree {DEGREE} (Calabi-Yau condition)")
            acc[INDEX_OF[e]] += int(c) % modulus
        return cls(acc % modulus, modulus)

    @property
    def is_zero(self) -> bool:
        return not self.coeffs.any()

    @property
    def degree(self) -> int:
        return -1 if self.is_zero else DEGREE

    def is_homogeneous(self) -> bool:
        return True

    def terms(self):
        """(exponent tuple, coefficient) of the nonzero terms in basis order."""
        for i in np.nonzero(self.coeffs)[0]:
            yield EXPONENTS[int(i)], int(self.coeffs[i])

    def coefficient(self, exps) -> int:
        i = INDEX_OF.get(tuple(int(x) for x in exps))
        return int(self.coeffs[i]) if i is not None else 0

    def __len__(self):
        return int(np.count_nonzero(self.coeffs))

    def __eq__(self, other):
        return isinstance(other, Quartic) and self.modulus == other.modulus and np.array_equal(self.coeffs, other.coeffs)

    def __hash__(self):
        return hash((self.modulus, self.coeffs.tobytes()))

    def __repr__(self):
        return f"Quartic(p={self.modulus}, {poly_to_text(self)})"


def coeff_vector(f, p: int | None = None) -> np.ndarray:
    """uint8[35] coefficient vector of a Quartic, a reference SparsePoly (duck-typed), or a raw vector."""
    if isinstance(f, Quartic):
        if p is not None and f.modulus != p:
            raise DomainError(f"f has modulus {f.modulus}, expected {p}")
        return f.coeffs
    if hasattr(f, "terms") and hasattr(f, "nvars"):
        if f.nvars != NVARS:
            raise DomainError(f"f has {f.nvars} variables; the GPU engine handles quartics in 4 variables")
        mod = getattr(f, "modulus", None) or p
        return Quartic.from_terms(f.terms(), mod).coeffs
    c = np.asarray(f)
    if c.shape != (NCOEFF,):
        raise DomainError(f"expected a 35-entry coefficient vector, got shape {c.shape}")
    if p is None:
        raise DomainError("a raw coefficient vector needs p")
    if (c < 0).any() or (c >= p).any():
        raise DomainError(f"coefficients must lie in [0, {p})")
    return c.astype(np.uint8)


# ---- text formats --------------------------------------------------------------------------------

def _parse_text_terms(text: str, nvars: int = NVARS):
    """[(exps, coeff)] from 'c*x1^a*x2^b + ...'; ParseError carries the offending position."""
    NVARS = max(nvars, 4)   # the scanner keeps at least four exponent slots (callers of the 3-variable grammar slice them)
    n = len(text)
    i = 0

    def skip(j):
        while j < n and text[j].isspace():
            j += 1
        return j

    def number(j):
        k = j
        while k < n and text[k].isdigit():
            k += 1
        return int(text[j:k]), k

    terms = []
    i = skip(i)
    if i >= n:
        raise ParseError("empty polynomial", 0)
    while True:
        coeff, exps = 1, [0] * NVARS
        while True:  # factors of one term
            i = skip(i)
            if i >= n:
                raise ParseError("term ended unexpectedly", n)
            ch = text[i]
            if ch.isdigit():
                v, i = number(i)
                coeff *= v
            elif ch == "x":
                j = i + 1
                if j >= n or not text[j].isdigit():
                    raise ParseError(f"unexpected character {ch!r}", i)
                idx, j = number(j)
                if idx < 1:
                    raise ParseError(f"bad variable x{idx}", i)
                if idx > NVARS:
                    raise ParseError(f"variable x{idx} exceeds nvars={NVARS}", 0)
                e = 1
                k = skip(j)
                if k < n and text[k] == "^":
                    k = skip(k + 1)
                    if k >= n or not text[k].isdigit():
                        raise ParseError("expected integer exponent after '^'", k)
                    e, k = number(k)
                    j = k
                exps[idx - 1] += e
                i = j
            elif ch in "*+^":
                raise ParseError(f"expected coefficient or variable, got {ch!r}", i)
            else:
                raise ParseError(f"unexpected character {ch!r}", i)
            i = skip(i)
            if i >= n:
                terms.append((tuple(exps), coeff))
                return terms
            if text[i] == "*":
                i += 1
                continue
            if text[i] == "+":
                plus = i
                i = skip(i + 1)
                if i >= n:
                    raise ParseError("trailing '+'", plus)
                break
            if text[i] in "^x" or text[i].isdigit():
                raise ParseError(f"expected '*' or '+', got {text[i]!r}", i)
            raise ParseError(f"unexpected character {text[i]!r}", i)
        terms.append((tuple(exps), coeff))


def _parse_compact_terms(text: str, nvars: int = NVARS):
    out = []
    pos = 0
    for chunk in text.splitlines():
        for piece in chunk.split(";"):
            line = piece.strip()
            start = pos
            pos += len(piece) + 1
            if not line or line.startswith("#"):
                continue
            if ":" not in line:
                raise ParseError(f"expected 'c:a,b,...', got {line!r}", start)
            cpart, epart = line.split(":", 1)
            try:
                coeff = int(cpart)
                exps = tuple(int(v) for v in epart.split(","))
            except ValueError:
                raise ParseError(f"malformed term {line!r}", start) from None
            if coeff < 0 or any(e < 0 for e in exps):
                raise ParseError(f"negative value in {line!r}", start)
            if len(exps) != nvars:
                raise ParseError(f"term has {len(exps)} exponents, expected {nvars}", start)
            out.append((exps, coeff))
    if not out:
        raise ParseError("no terms found", 0)
    return out


def parse_poly(text: str, nvars: int | None = NVARS, modulus: int | None = None) -> Quartic:
    """Parse either text format (auto-detected by ':') into a Quartic over F_modulus."""
    if nvars is not None and not 2 <= nvars <= 6:
        raise DomainError(f"the GPU engine handles forms of degree n in n = 2..6 variables, got nvars={nvars}")
    if modulus is None:
        raise DomainError("parse_poly needs the modulus p")
    if nvars is None and ":" not in text:
        # the reference infers the variable count from the highest variable that appears (polyring.py:438-520)
        used = max((max((j + 1 for j, e in enumerate(exps) if e), default=0) for exps, _ in _parse_text_terms(text, 6)), default=0)
        if used < 2:
            raise DomainError(f"f has {used} variables; f must be homogeneous of degree nvars in nvars >= 2 variables (Calabi-Yau condition)")
        if used != NVARS:
            nvars = used
    if nvars == 3:
        from .cubic import Cubic
        if ":" in text:
            terms = _parse_compact_terms(text, 3)
        else:
            terms = []
            for exps, c in _parse_text_terms(text):  # the term scanner works with four exponent slots
                if exps[3]:
                    raise ParseError("variable x4 exceeds nvars=3", 0)
                terms.append((tuple(exps[:3]), c))
        return Cubic.from_terms(terms, modulus)
    if nvars not in (None, NVARS):
        from .forms import Form
        if ":" in text:
            terms = _parse_compact_terms(text, nvars)
        else:
            terms = []
            for exps, c in _parse_text_terms(text, nvars):
                if any(exps[nvars:]):
                    raise ParseError(f"variable x{max(j + 1 for j, e in enumerate(exps) if e)} exceeds nvars={nvars}", 0)
                terms.append((tuple(exps[:nvars]), c))
        return Form.from_terms(terms, modulus, nvars)
    terms = _parse_compact_terms(text) if ":" in text else _parse_text_terms(text)
    return Quartic.from_terms(terms, modulus)


def poly_to_text(f) -> str:
    """Leading terms first, 'c*x1^a*x2^b' (the format of polyring.py:564-592 and of the fixture table)."""
    c = coeff_vector(f, getattr(f, "modulus", None))
    if not c.any():
        return "0"
    parts = []
    for i in range(NCOEFF - 1, -1, -1):
        if not c[i]:
            continue
        mono = "*".join(f"x{j + 1}" + (f"^{e}" if e > 1 else "") for j, e in enumerate(EXPONENTS[i]) if e)
        parts.append(mono if c[i] == 1 else f"{int(c[i])}*{mono}")
    return " + ".join(parts)
