"""CPU tests of the export formats and of the command-line shell (no compute calls: no GPU here).

Wire formats follow the reference (mtsmatrix.py:298-380); the byte-level goldens in tests/golden/exports.json
were produced by the reference itself (tests/golden/make_golden_exports.py) and are compared on the GPU in
tests/test_gpu_export_cli.py.  Here: round trips, headers, error behaviour, parser flags and exit codes."""
import hashlib
import json
import os
import struct

import numpy as np
import pytest

import paper_2502_12428_b200 as q
from paper_2502_12428_b200.cli import _build_parser, main

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden_matrix(p, key="s1"):
    d = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
    return d[f"{key}_M"], d[f"{key}_coeffs"]


def test_binary_layout_matches_reference_spec():
    M, _ = _golden_matrix(3)
    m = q.MtsMatrix(M, 4, 8, 8, 3)
    b = q.matrix_to_bytes(m)
    assert b[:8] == b"QFSMTX01"
    assert struct.unpack_from("<6I", b, 8) == (165, 165, 3, 4, 8, 8)
    assert len(b) == 8 + 24 + 2 * 165 * 165
    assert np.array_equal(np.frombuffer(b[32:], dtype="<u2").reshape(165, 165), M)
    assert q.matrix_from_bytes(b) == m
    # the reference's own export of the same kind of matrix has this length (exports.json, F_3 rows)
    gold = json.load(open(os.path.join(GOLDEN, "exports.json")))
    assert gold["matrices"][0]["bytes_len"] == len(b)
    assert gold["matrices"][0]["bytes_head_hex"] == b[:32].hex()


def test_text_layout_and_round_trip():
    M, _ = _golden_matrix(3)
    m = q.MtsMatrix(M, 4, 8, 8, 3)
    t = q.matrix_to_text(m)
    lines = t.splitlines()
    assert lines[0] == "165 165 3" and len(lines) == 166 and t.endswith("\n")
    assert lines[1] == " ".join(str(int(v)) for v in M[0])
    assert q.matrix_from_text(t, 4) == m
    assert q.matrix_from_text(t, 4, d=8, dprime=8) == q.matrix_from_bytes(q.matrix_to_bytes(m))
    gold = json.load(open(os.path.join(GOLDEN, "exports.json")))
    assert gold["matrices"][0]["text_head"].startswith("165 165 3\n")


def test_golden_f5_matrix_exports_hash_like_the_reference_entries():
    """The F_5 staged golden matrix (reference MtsMatrix.entries) through OUR writers, re-read, and hashed."""
    d = np.load(os.path.join(GOLDEN, "stages_p5.npz"))
    key = [k[:-2] for k in d.files if k.endswith("_M")][0]
    M = d[key + "_M"]
    m = q.MtsMatrix(M, 4, 16, 16, 5)
    assert q.matrix_from_bytes(q.matrix_to_bytes(m)) == m
    assert hashlib.sha256(np.ascontiguousarray(M, dtype=np.uint8).tobytes()).digest() == bytes(d[key + "_Msha"]) \
        or hashlib.sha256(np.ascontiguousarray(M).tobytes()).digest() == bytes(d[key + "_Msha"])


def test_export_error_behaviour():
    M, _ = _golden_matrix(3)
    with pytest.raises(q.DomainError):
        q.MtsMatrix(M, 4, 8, 7, 3)              # shape does not match the bases
    with pytest.raises(q.DomainError):
        q.MtsMatrix(M, 4, 8, 8, 2)              # entries not reduced
    with pytest.raises(q.DomainError):
        q.matrix_from_bytes(b"QFSMTX01" + b"\0" * 8)
    with pytest.raises(q.DomainError):
        q.matrix_from_bytes(b"NOTMAGIC" + b"\0" * 24)
    good = q.matrix_to_bytes(q.MtsMatrix(M, 4, 8, 8, 3))
    with pytest.raises(q.DomainError):
        q.matrix_from_bytes(good[:-2])
    with pytest.raises(q.DomainError):
        q.matrix_from_text("", 4)
    with pytest.raises(q.DomainError):
        q.matrix_from_text("2 2\n0 1\n1 0\n", 4)
    with pytest.raises(q.DomainError):
        q.matrix_from_text("165 165 3\n0 1\n", 4)
    assert q.target_degree(16, 80, 4, 5) == 16 and q.target_degree(8, 24, 4, 3) == 8
    assert q.target_degree(3, 3, 4, 5) is None
    with pytest.raises(q.DomainError):
        q.build_mts(q.parse_poly("x1^4+x2^4+x3^4+x4^4", 4, 5), 5, algorithm="bogus")


def run(capsys, *argv):
    rc = main(list(argv))
    captured = capsys.readouterr()
    return rc, captured.out, captured.err


def test_cli_parser_matches_the_reference_flags(monkeypatch):
    """Same subcommands, flags and defaults as cli.py:193-247; QFSPLIT_JOBS as in cli.py:35-39 (tests/test_cli.py:102-108)."""
    ps = _build_parser()
    a = ps.parse_args(["height", "--p", "5", "--poly", "x1^4"])
    assert (a.method, a.mts, a.bound, a.nvars, a.json) == ("matrix", "wics", None, None, False)
    a = ps.parse_args(["search", "--p", "3"])
    assert (a.count, a.seed, a.bound, a.target_height, a.out, a.json) == (1000, 0, None, None, None, False)
    a = ps.parse_args(["matrix", "--p", "3", "--poly", "x", "--out", "o"])
    assert (a.mts, a.format) == ("wics", "text")
    a = ps.parse_args(["verify"])
    assert (a.fixtures, a.primes, a.method) == (None, None, "matrix")
    a = ps.parse_args(["bench"])
    assert (a.p, a.what, a.reps) == (5, "height", 3)
    monkeypatch.setenv("QFSPLIT_JOBS", "3")
    assert _build_parser().parse_args(["search", "--p", "3"]).jobs == 3
    monkeypatch.setenv("QFSPLIT_JOBS", "garbage")
    assert _build_parser().parse_args(["search", "--p", "3"]).jobs == 1
    with pytest.raises(SystemExit):
        ps.parse_args(["height", "--p", "5"])  # --poly is required


def test_cli_exit_codes_before_any_compute(capsys, tmp_path):
    """Parse / input / domain errors surface with the reference's exit codes (cli.py:250-265) without touching the GPU."""
    rc, _, err = run(capsys, "height", "--p", "5", "--poly", "x1^4 + $")
    assert rc == 2 and "position" in err
    rc, _, err = run(capsys, "height", "--p", "5", "--poly", "@" + str(tmp_path / "missing.txt"))
    assert rc == 2 and "input error" in err
    rc, _, err = run(capsys, "height", "--p", "6", "--poly", "x1^4+x2^4+x3^4+x4^4")
    assert rc == 3 and "not prime" in err
    rc, _, err = run(capsys, "height", "--p", "5", "--poly", "x1^4+x2^3")          # not homogeneous
    assert rc == 3
    rc, _, err = run(capsys, "height", "--p", "5", "--poly", "x1^4+x2^4", "--nvars", "4", "--bound", "0")
    assert rc == 3 and "bound" in err
    rc, _, err = run(capsys, "search", "--p", "5", "--count", "0")
    assert rc == 3
    rc, _, err = run(capsys, "matrix", "--p", "4", "--poly", "x1^4+x2^4+x3^4+x4^4", "--out", str(tmp_path / "m"))
    assert rc == 3
    with pytest.raises(SystemExit):
        run(capsys, "verify", "--method", "bogus")


def test_cli_reports_a_missing_engine_instead_of_falling_back(capsys):
    """No GPU in this container: compute commands must fail loudly (exit 5), never produce a height."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    rc, out, err = run(capsys, "height", "--p", "5", "--poly", "x1^4+x2^4+x3^4+x4^4")
    assert rc == 5 and "height" not in out and "engine unavailable" in err
