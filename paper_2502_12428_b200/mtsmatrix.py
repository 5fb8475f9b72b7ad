"""Operator-matrix export in the reference's wire formats (mtsmatrix.py:82-130, 298-380).

`build_mts` here takes the quartic itself (the reference takes delta1(f^(p-1)): cli.py:108-113 always
builds it from f) and returns the same row-major uint16 entry block, produced on the GPU by
qfs_export_matrix (include/qfs.h).  The text form ("rows cols p" header + one row per line) and the
binary form ("QFSMTX01" magic + six little-endian uint32 header words rows, cols, p, n, d, d' + `<u2`
entries) are byte-identical to the reference's, so `qfsplit.matrix_from_bytes` / `matrix_from_text`
read them back.
"""
import math
import struct
from dataclasses import dataclass

import numpy as np

from .engine import get_engine
from .errors import DomainError
from .height import NVARS, SurfaceProblem, _check_batch, _check_engine_shape
from .quartic import coeff_vector

_MAGIC = b"QFSMTX01"


def target_degree(d: int, D: int, n: int, p: int):
    """Degree of u(delta * g) for deg g = d, deg delta = D, or None (mtsmatrix.py:42-52)."""
    num = d + D - n * (p - 1)
    if num < 0 or num % p != 0:
        return None
    return num // p


@dataclass(eq=False)
class MtsMatrix:
    """Dense matrix over F_p of g -> u(delta * g); column j = image of basis monomial j (mtsmatrix.py:82-130).

    The reference carries MonomialBasis objects; the bases are determined by (nvars, degree), which is what the
    wire formats store, so this mirror keeps the numbers.
    """
    entries: np.ndarray
    nvars: int
    source_degree: int
    target_degree: int
    p: int

    def __post_init__(self):
        self.entries = np.ascontiguousarray(self.entries, dtype=np.uint16)
        expected = (math.comb(self.target_degree + self.nvars - 1, self.nvars - 1),
                    math.comb(self.source_degree + self.nvars - 1, self.nvars - 1))
        if self.entries.shape != expected:
            raise DomainError(f"entry block shape {self.entries.shape} does not match bases {expected}")
        if self.p < 2:
            raise DomainError(f"modulus must be at least 2, got {self.p}")
        if self.entries.size and int(self.entries.max()) >= self.p:
            raise DomainError("matrix entries must be reduced mod p")
        self.entries.flags.writeable = False

    @property
    def rows(self) -> int:
        return self.entries.shape[0]

    @property
    def cols(self) -> int:
        return self.entries.shape[1]

    def __eq__(self, other):
        if not isinstance(other, MtsMatrix):
            return NotImplemented
        return (self.p == other.p and self.source_degree == other.source_degree
                and self.target_degree == other.target_degree and self.nvars == other.nvars
                and np.array_equal(self.entries, other.entries))

    def __repr__(self):
        return f"MtsMatrix({self.rows}x{self.cols} over F_{self.p})"


def build_mts(f, *args, algorithm: str = "wics", device: int = 0) -> MtsMatrix:
    """Operator matrix over F_p.  Two call forms:

    * `build_mts(delta, d, p, algorithm="wics")` -- the reference's own signature (mtsmatrix.py:287-295): `delta` is the dense
      Delta_1(g) that `stages.delta1` returned (or any DenseForm of degree p*d: the builder is a generic map Delta -> M);
    * `build_mts(f, p, algorithm="wics")` -- from the quartic: build_mts(delta1(f^(p-1)), 4(p-1), p) in one call.

    `algorithm` is validated like the reference's; TRIV, MERGE and WICS produce the same entries
    (tests/test_mtsmatrix.py in the reference), and the GPU builder is a fourth way to the same matrix.
    """
    from .stages import DenseForm
    if isinstance(f, DenseForm) and len(args) >= 2:
        d, p = int(args[0]), int(args[1])
        if len(args) >= 3:
            algorithm = args[2]
    else:
        if not args:
            raise DomainError("build_mts(f, p) needs the prime")
        d, p = None, int(args[0])
        if len(args) >= 2:
            algorithm = args[1]
        if len(args) >= 3:
            device = int(args[2])
    if algorithm not in ("triv", "merge", "wics"):
        raise DomainError(f"unknown algorithm {algorithm!r}, expected one of ['merge', 'triv', 'wics']")
    if d is not None:
        _check_engine_shape(p)
        if d != 4 * (p - 1) or f._degree != p * d or f.modulus != p:
            raise DomainError(f"the GPU engine builds the operator of quartic K3 surfaces: d = 4(p-1), deg delta = p d; got d={d}, deg delta={f._degree}")
        block = get_engine(p, device).stage_matrix(f.values[None, :])[0]
        return MtsMatrix(block, NVARS, d, target_degree(d, p * d, NVARS, p), p)
    if hasattr(f, "nvars"):
        SurfaceProblem(p, f.nvars, f)  # the reference's checks (cli.py:110), in its order
        _check_engine_shape(p, f.nvars)
        vec = coeff_vector(f, p)
    else:
        vec = _check_batch(p, np.asarray(f)[None, :], 10)[0]
    entries = get_engine(p, device).export_matrix(vec[None, :])[0]
    d = 4 * (p - 1)
    return MtsMatrix(entries, NVARS, d, target_degree(d, p * d, NVARS, p), p)


def build_mts_batch(p: int, coeffs, device: int = 0) -> np.ndarray:
    """Entry blocks [B][N][N] (uint16) of a batch of coefficient vectors."""
    return get_engine(p, device).export_matrix(_check_batch(p, coeffs, 10))


_HEADER = struct.Struct("<6I")  # rows, cols, p, n, d, d'


def matrix_to_text(m: MtsMatrix) -> str:
    """The text export: a "rows cols p" line, then the entries row by row, blank-separated (mtsmatrix.py:301-306)."""
    body = "\n".join(" ".join(row) for row in np.char.mod("%d", m.entries))
    return f"{m.rows} {m.cols} {m.p}\n{body}\n"


def _basis_degree(count: int, nvars: int, what: str) -> int:
    """The degree whose monomial basis in `nvars` variables has `count` elements (the text header does not store it)."""
    if nvars < 2:
        raise DomainError("degree inference needs at least 2 variables")
    degree, size = 0, 1
    while size < count:
        degree += 1
        size = size * (degree + nvars - 1) // degree      # C(degree+n-1, n-1) from C(degree+n-2, n-1)
    if size != count:
        raise DomainError(f"no degree-{nvars} basis has {count} {what}")
    return degree


def matrix_from_text(text: str, n: int, d=None, dprime=None) -> MtsMatrix:
    """Read the text export back (mtsmatrix.py:322-347).  `n` comes from the caller; degrees are inferred unless given."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise DomainError("empty matrix text")
    head = lines[0].split()
    if len(head) != 3:
        raise DomainError(f"matrix header needs 'rows cols p', got {lines[0]!r}")
    rows, cols, p = map(int, head)
    if len(lines) - 1 != rows:
        raise DomainError(f"expected {rows} entry rows, got {len(lines) - 1}")
    widths = [len(ln.split()) for ln in lines[1:]]
    for i, w in enumerate(widths):
        if w != cols:
            raise DomainError(f"row {i} has {w} entries, expected {cols}")
    entries = np.array(" ".join(lines[1:]).split(), dtype=np.int64).reshape(rows, cols)
    return MtsMatrix(entries, n,
                     _basis_degree(cols, n, "columns") if d is None else d,
                     _basis_degree(rows, n, "rows") if dprime is None else dprime, p)


def matrix_to_bytes(m: MtsMatrix) -> bytes:
    """The binary export: "QFSMTX01", six little-endian uint32 (rows, cols, p, n, d, d'), then the entries as
    little-endian uint16 in row-major order (mtsmatrix.py:350-365)."""
    return b"".join((_MAGIC, _HEADER.pack(m.rows, m.cols, m.p, m.nvars, m.source_degree, m.target_degree),
                     m.entries.astype("<u2", copy=False).tobytes()))


def matrix_from_bytes(data: bytes) -> MtsMatrix:
    """Read the binary export back (mtsmatrix.py:368-380)."""
    start = len(_MAGIC) + _HEADER.size
    if len(data) < start:
        raise DomainError("binary matrix data is truncated")
    if not data.startswith(_MAGIC):
        raise DomainError("bad magic; not a matrix export")
    rows, cols, p, n, d, dprime = _HEADER.unpack_from(data, len(_MAGIC))
    if len(data) - start != 2 * rows * cols:
        raise DomainError(f"entry block holds {len(data) - start} bytes, expected {2 * rows * cols}")
    return MtsMatrix(np.frombuffer(data, dtype="<u2", offset=start).reshape(rows, cols), n, d, dprime, p)
