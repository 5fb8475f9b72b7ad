"""GPU tests: export formats and command-line shell against outputs of the reference itself
(tests/golden/exports.json, produced by tests/golden/make_golden_exports.py with the unmodified reference)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
GOLD = json.load(open(os.path.join(GOLDEN, "exports.json")))


def run(capsys, *argv):
    from paper_2502_12428_b200.cli import main
    rc = main(list(argv))
    captured = capsys.readouterr()
    return rc, captured.out, captured.err


@pytest.mark.parametrize("case", GOLD["matrices"], ids=lambda c: f"p{c['p']}-{c['nonzero']}")
def test_exports_are_byte_identical_to_the_reference(case):
    """matrix_to_bytes / matrix_to_text of the GPU-built matrix == the reference's files, byte for byte (sha256)."""
    import paper_2502_12428_b200 as q
    p = case["p"]
    m = q.build_mts(q.parse_poly(case["poly"], 4, p), p)
    assert (m.rows, m.cols) == (case["rows"], case["cols"])
    assert int((m.entries != 0).sum()) == case["nonzero"]
    b = q.matrix_to_bytes(m)
    assert len(b) == case["bytes_len"] and hashlib.sha256(b).hexdigest() == case["bytes_sha256"]
    if p <= 5:  # the F_7 text form is 17 MB of Python string work; the binary form pins the same entries
        t = q.matrix_to_text(m)
        assert len(t) == case["text_len"] and hashlib.sha256(t.encode()).hexdigest() == case["text_sha256"]


def test_export_batch_equals_stage_taps():
    """qfs_export_matrix (uint16, dense) == qfs_stage_matrix of qfs_stage_delta (uint8) on seeded surfaces, ragged batch."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    for p, B in ((3, 7), (5, 5)):
        c = q.sample_block(p, B, 11, 0)
        eng = get_engine(p, 0)
        M8 = eng.stage_matrix(eng.stage_delta(c))
        M16 = q.build_mts_batch(p, c)
        assert M16.dtype == np.dtype("<u2") and M16.shape == M8.shape
        assert np.array_equal(M16, M8)


@pytest.mark.parametrize("case", GOLD["cli"], ids=lambda c: " ".join(c["argv"][:4] + c["argv"][5:7]))
def test_cli_stdout_equals_the_reference(capsys, case):
    """`height --json` and `search --json` print exactly what the reference prints (tests/test_cli.py:24-30, 78-87)."""
    rc, out, _ = run(capsys, *case["argv"])
    assert rc == case["rc"]
    assert out == case["stdout"]


def test_cli_matrix_verify_bench(capsys, tmp_path):
    import paper_2502_12428_b200 as q
    fermat = "x1^4+x2^4+x3^4+x4^4"
    tpath, bpath = tmp_path / "m.txt", tmp_path / "m.bin"
    rc, out, _ = run(capsys, "matrix", "--p", "5", "--poly", fermat, "--out", str(tpath))
    assert rc == 0 and "969x969" in out
    m = q.matrix_from_text(tpath.read_text(), 4)
    assert m.rows == m.cols == 969 and m.p == 5
    run(capsys, "matrix", "--p", "3", "--poly", fermat, "--out", str(tpath))
    run(capsys, "matrix", "--p", "3", "--poly", fermat, "--out", str(bpath), "--format", "binary")
    assert q.matrix_from_text(tpath.read_text(), 4) == q.matrix_from_bytes(bpath.read_bytes())
    assert hashlib.sha256(bpath.read_bytes()).hexdigest() == GOLD["matrices"][0]["bytes_sha256"]
    # verify: the whole packaged table, F_5 ... F_13 (the reference's extended acceptance set)
    rc, out, _ = run(capsys, "verify")
    assert rc == 0 and "32 rows, 0 mismatches" in out
    fx = tmp_path / "fx.txt"
    fx.write_text("5 ; 2 ; " + fermat + "\n")            # wrong on purpose: Fermat over F_5 has height 1
    rc, out, _ = run(capsys, "verify", "--fixtures", str(fx))
    assert rc == 1 and "MISMATCH" in out
    fx.write_text("17 ; 1 ; " + fermat + "\n")            # a prime this build has no kernels for
    rc, out, _ = run(capsys, "verify", "--fixtures", str(fx))
    assert rc == 0 and "1 rows skipped" in out
    rc, out, err = run(capsys, "height", "--p", "17", "--poly", fermat)
    assert rc == 3 and "not supported" in err
    rc, out, _ = run(capsys, "height", "--p", "5", "--poly", fermat)
    assert rc == 0 and "height 1" in out and "iterations 0" in out
    # the two methods agree, as in the reference's tests/test_cli.py:32-40
    results = {}
    for method in ("naive", "matrix"):
        rc, out, _ = run(capsys, "height", "--p", "5", "--poly", fermat + "+x1*x2*x3*x4", "--method", method, "--json")
        assert rc == 0
        results[method] = json.loads(out)
    assert results["naive"]["height"] == results["matrix"]["height"] == "inf"
    assert results["naive"]["iterations"] == results["matrix"]["iterations"] == 9
    rc, out, _ = run(capsys, "verify", "--method", "naive", "--primes", "5,7")
    assert rc == 0 and "22 rows, 0 mismatches" in out
    for what in ("power", "mts", "matvec", "height"):
        rc, out, _ = run(capsys, "bench", "--p", "5", "--what", what, "--reps", "1")
        assert rc == 0 and "mean=" in out
