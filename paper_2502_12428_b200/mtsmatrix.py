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


def build_mts(f, p: int, algorithm: str = "wics", device: int = 0) -> MtsMatrix:
    """Operator matrix of the quartic f over F_p (build_mts(delta1(f^(p-1)), 4(p-1), p), mtsmatrix.py:287-295).

    `algorithm` is validated like the reference's; TRIV, MERGE and WICS produce the same entries
    (tests/test_mtsmatrix.py in the reference), and the GPU builder is a fourth way to the same matrix.
    """
    if algorithm not in ("triv", "merge", "wics"):
        raise DomainError(f"unknown algorithm {algorithm!r}, expected one of ['merge', 'triv', 'wics']")
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


def matrix_to_text(m: MtsMatrix) -> str:
    """Header line "rows cols p", then one text row per matrix row (mtsmatrix.py:301-306)."""
    lines = [f"{m.rows} {m.cols} {m.p}"]
    digits = np.char.mod("%d", m.entries)
    lines.extend(" ".join(row) for row in digits)
    return "\n".join(lines) + "\n"


def _degree_for_size(size: int, n: int, what: str) -> int:
    if n < 2:
        raise DomainError("degree inference needs at least 2 variables")
    deg = 0
    while True:
        count = math.comb(deg + n - 1, n - 1)
        if count == size:
            return deg
        if count > size:
            raise DomainError(f"no degree-{n} basis has {size} {what}")
        deg += 1


def matrix_from_text(text: str, n: int, d=None, dprime=None) -> MtsMatrix:
    """Inverse of matrix_to_text (mtsmatrix.py:322-347); n comes from the caller, degrees are inferred unless given."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise DomainError("empty matrix text")
    head = lines[0].split()
    if len(head) != 3:
        raise DomainError(f"matrix header needs 'rows cols p', got {lines[0]!r}")
    rows, cols, p = (int(v) for v in head)
    if len(lines) - 1 != rows:
        raise DomainError(f"expected {rows} entry rows, got {len(lines) - 1}")
    if d is None:
        d = _degree_for_size(cols, n, "columns")
    if dprime is None:
        dprime = _degree_for_size(rows, n, "rows")
    entries = np.zeros((rows, cols), dtype=np.uint16)
    for i, line in enumerate(lines[1:]):
        vals = line.split()
        if len(vals) != cols:
            raise DomainError(f"row {i} has {len(vals)} entries, expected {cols}")
        entries[i] = [int(v) for v in vals]
    return MtsMatrix(entries, n, d, dprime, p)


def matrix_to_bytes(m: MtsMatrix) -> bytes:
    """Magic, six uint32 header words (rows, cols, p, n, d, d'), uint16 entries, little-endian (mtsmatrix.py:350-365)."""
    head = struct.pack("<6I", m.rows, m.cols, m.p, m.nvars, m.source_degree, m.target_degree)
    return _MAGIC + head + m.entries.astype("<u2").tobytes()


def matrix_from_bytes(data: bytes) -> MtsMatrix:
    """Inverse of matrix_to_bytes (mtsmatrix.py:368-380)."""
    if len(data) < len(_MAGIC) + 24:
        raise DomainError("binary matrix data is truncated")
    if data[: len(_MAGIC)] != _MAGIC:
        raise DomainError("bad magic; not a matrix export")
    rows, cols, p, n, d, dprime = struct.unpack_from("<6I", data, len(_MAGIC))
    body = data[len(_MAGIC) + 24:]
    if len(body) != 2 * rows * cols:
        raise DomainError(f"entry block holds {len(body)} bytes, expected {2 * rows * cols}")
    entries = np.frombuffer(body, dtype="<u2").astype(np.uint16).reshape(rows, cols)
    return MtsMatrix(entries, n, d, dprime, p)
