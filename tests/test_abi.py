"""The C-ABI library loads on a CPU-only box and exports every symbol include/qfs.h declares;
compute entry points fail loudly without a GPU (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    text = open(os.path.join(ROOT, "include", "qfs.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qfs_[a-z_]+)\s*\(", text)))


def test_header_declares_the_documented_entry_points():
    names = _declared()
    for must in ("qfs_version", "qfs_create", "qfs_destroy", "qfs_heights", "qfs_stage_power", "qfs_stage_delta",
                 "qfs_stage_matrix", "qfs_stage_matvec_chain", "qfs_last_error", "qfs_get_shape", "qfs_get_stats"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2502_12428_b200 import _native
    lib = _native.load()
    for name in _declared():
        assert hasattr(lib, name), f"libqfs.so does not export {name}"
    assert set(_declared()) == set(_native.EXPORTS)
    assert lib.qfs_version() == 1


@pytest.mark.parametrize("p,N,L,cap", [(3, 165, 2925, 96), (5, 969, 91881, 564), (7, 2925, 818805, 1700),
                                       (11, 12341, 14391741, 7160)])
def test_shape_constants(p, N, L, cap):
    """Operator dimensions and cap indices of SURVEY.md section 7/8 (tests/test_acceptance.py:165-174 in the reference)."""
    from paper_2502_12428_b200.engine import shape_of
    s = shape_of(p)
    assert (s.N, s.L, s.cap, s.d, s.D) == (N, L, cap, 4 * (p - 1), 4 * p * (p - 1))
    assert s.pitch % 16 == 0 and s.pitch >= N


def test_unsupported_prime_is_a_domain_error():
    from paper_2502_12428_b200.engine import shape_of
    from paper_2502_12428_b200.errors import DomainError
    with pytest.raises(DomainError):
        shape_of(17)
    s13 = shape_of(13)
    assert (s13.N, s13.d, s13.D, s13.L, s13.cap) == (20825, 48, 624, 40885625, 12076)


def test_no_cpu_fallback():
    """Without a CUDA device the engine refuses to exist; nothing silently computes on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA device present")
    import numpy as np
    from paper_2502_12428_b200 import EngineUnavailableError, height_batch
    with pytest.raises(EngineUnavailableError):
        height_batch(5, np.ones((2, 35), dtype=np.uint8))


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2502_12428_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, flags=re.M), f
                assert "qfs_oracle" not in src, f
