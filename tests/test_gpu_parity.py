"""GPU parity: every CUDA stage against the golden vectors produced by the reference and against
the C oracle on seeded inputs.  All calls go through the C ABI (ctypes -> libqfs.so)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _engine(p):
    from paper_2502_12428_b200.engine import get_engine
    return get_engine(p, 0)


def _stages(p):
    z = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
    return z, int(z["count"])


def _random_coeffs(p, B, seed):
    rng = np.random.default_rng([seed, p])
    c = rng.integers(0, p, size=(B, 35)).astype(np.uint8)
    c[(c == 0).all(axis=1), 0] = 1
    return c


@pytest.mark.parametrize("p", [3, 5, 7])
def test_stage_power_golden(p):
    z, n = _stages(p)
    coeffs = np.stack([z[f"s{i}_coeffs"] for i in range(n)])
    g, fed = _engine(p).stage_power(coeffs)
    for i in range(n):
        assert np.array_equal(g[i], z[f"s{i}_g"]), f"g mismatch surface {i}"
        assert bool(fed[i]) == (int(z[f"s{i}_height"]) == 1)


@pytest.mark.parametrize("p", [3, 5, 7])
def test_stage_delta_golden(p):
    z, n = _stages(p)
    idx = [i for i in range(n) if f"s{i}_delta" in z.files]
    coeffs = np.stack([z[f"s{i}_coeffs"] for i in idx])
    dl = _engine(p).stage_delta(coeffs)
    for k, i in enumerate(idx):
        want = z[f"s{i}_delta"]
        bad = np.nonzero(dl[k] != want)[0]
        assert bad.size == 0, f"delta mismatch surface {i}: {bad.size} entries, first {bad[:5]}"


@pytest.mark.parametrize("p", [3, 5, 7])
def test_stage_matrix_golden(p):
    z, n = _stages(p)
    idx = [i for i in range(n) if f"s{i}_delta" in z.files]
    dl = np.stack([z[f"s{i}_delta"] for i in idx])
    M = _engine(p).stage_matrix(dl)
    for k, i in enumerate(idx):
        sha = hashlib.sha256(np.ascontiguousarray(M[k]).tobytes()).digest()
        if f"s{i}_M" in z.files:
            bad = np.argwhere(M[k] != z[f"s{i}_M"])
            assert bad.shape[0] == 0, f"M mismatch surface {i}: {bad.shape[0]} cells, first {bad[:4].tolist()}"
        else:
            rows = z[f"s{i}_Mrows_idx"]
            assert np.array_equal(M[k][rows], z[f"s{i}_Mrows"])
        assert sha == bytes(z[f"s{i}_Msha"]), f"M sha256 mismatch surface {i}"


@pytest.mark.parametrize("p", [3, 5])
def test_stage_chain_golden(p):
    z, n = _stages(p)
    idx = [i for i in range(n) if f"s{i}_M" in z.files]
    M = np.stack([z[f"s{i}_M"] for i in idx])
    g = np.stack([z[f"s{i}_g"] for i in idx])
    hs, its, tr = _engine(p).stage_matvec_chain(M, g, 9, trace=True)
    for k, i in enumerate(idx):
        assert int(hs[k]) == int(z[f"s{i}_height"])
        assert int(its[k]) == int(z[f"s{i}_iters"])
        assert np.array_equal(tr[k][: its[k]], z[f"s{i}_trace"])


@pytest.mark.parametrize("p,name", [(3, "heights_p3_seed0_w0_3000"), (5, "heights_p5_seed0_w0_10000"),
                                    (7, "heights_p7_seed0_w0_10000")])
def test_heights_golden_sets(p, name):
    path = os.path.join(GOLDEN, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    z = np.load(path)
    hs, its = _engine(p).heights(z["coeffs"], 10)
    bad = np.nonzero((hs != z["heights"]) | (its != z["iters"]))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: got {hs[bad[:5]]} want {z['heights'][bad[:5]]}"


def test_fixture_table():
    rows = json.load(open(os.path.join(GOLDEN, "k3_fixture_vectors.json")))
    for p in (5, 7):
        sel = [r for r in rows if r["p"] == p]
        coeffs = np.array([r["coeffs"] for r in sel], dtype=np.uint8)
        hs, its = _engine(p).heights(coeffs, 10)
        assert [int(h) for h in hs] == [r["height"] for r in sel]
        for h, it in zip(hs, its):
            assert int(it) == (int(h) - 1 if h > 0 else 9)


@pytest.mark.parametrize("p,B", [(3, 64), (5, 24), (7, 6)])
def test_stages_vs_oracle_random(p, B):
    import oracle
    eng = _engine(p)
    coeffs = _random_coeffs(p, B, 77)
    g, fed = eng.stage_power(coeffs)
    dl = eng.stage_delta(coeffs)
    for i in range(B):
        h, it, t = oracle.height_matrix(coeffs[i], p, 10, taps=True)
        assert np.array_equal(g[i], t["g"])
        assert bool(fed[i]) == (h == 1)
        if h != 1:
            assert np.array_equal(dl[i], t["delta"]), f"delta mismatch {i}"
    hs, its = eng.heights(coeffs, 10)
    ohs, oits = oracle.heights_batch(coeffs, p, 10)
    assert np.array_equal(hs, ohs) and np.array_equal(its, oits)


@pytest.mark.parametrize("p", [3, 5])
def test_matrix_from_arbitrary_delta_vs_oracle(p):
    """The builder is a generic map Delta -> M: feed random dense Delta (not a Witt carry)."""
    import oracle
    eng = _engine(p)
    rng = np.random.default_rng(5)
    dl = rng.integers(0, p, size=(2, eng.shape.L)).astype(np.uint8)
    M = eng.stage_matrix(dl)
    for i in range(2):
        assert np.array_equal(M[i], oracle.build_mts(dl[i], p))


@pytest.mark.parametrize("bound", [1, 2, 3, 10])
def test_bound_semantics(bound):
    import oracle
    p = 5
    coeffs = _random_coeffs(p, 200, 3)
    hs, its = _engine(p).heights(coeffs, bound)
    ohs, oits = oracle.heights_batch(coeffs, p, bound)
    assert np.array_equal(hs, ohs) and np.array_equal(its, oits)


# ---- F_11, F_13: the reference's own intermediates (tests/golden/make_golden_p11.py; ~5 resp. ~25 CPU-minutes per surface) ----------
def _pbig(p):
    path = os.path.join(GOLDEN, f"stages_p{p}.npz")
    if not os.path.exists(path):
        pytest.skip(f"stages_p{p}.npz not generated")
    z = np.load(path)
    return z, int(z["count"])


@pytest.mark.parametrize("p", [11, 13])
def test_big_prime_stage_power_golden(p):
    z, n = _pbig(p)
    coeffs = np.stack([z[f"s{i}_coeffs"] for i in range(n)])
    g, fed = _engine(p).stage_power(coeffs)
    for i in range(n):
        assert np.array_equal(g[i], z[f"s{i}_g"]), f"g mismatch surface {i}"
        assert not fed[i]


@pytest.mark.parametrize("p", [11, 13])
def test_big_prime_delta_matrix_chain_golden(p):
    """Delta (sha256 of the dense vector -- 14 391 741 entries at p = 11, 40 885 625 at p = 13 -- and every 997th entry), M (sha256
    of the 12341^2 resp. 20825^2 operator and five rows) and the whole matvec trace, heights and iteration counts against what the
    reference computed (extended suite of the reference, tests/test_acceptance.py:84-89; tests/test_mtsmatrix.py:174-198)."""
    z, n = _pbig(p)
    eng = _engine(p)
    coeffs = np.stack([z[f"s{i}_coeffs"] for i in range(n)])
    step = 2 if p == 11 else 1        # surfaces at a time: 152 MB resp. 434 MB of M each on the host
    for lo in range(0, n, step):
        sel = list(range(lo, min(n, lo + step)))
        dl = eng.stage_delta(coeffs[sel])
        for k, i in enumerate(sel):
            assert np.array_equal(dl[k][::997], z[f"s{i}_delta_every"]), f"Delta sample mismatch surface {i}"
            assert int(np.count_nonzero(dl[k])) == int(z[f"s{i}_delta_nnz"])
            assert hashlib.sha256(dl[k].tobytes()).digest() == bytes(z[f"s{i}_delta_sha"]), f"Delta sha256 mismatch surface {i}"
        M = eng.stage_matrix(dl)
        g = np.stack([z[f"s{i}_g"] for i in sel])
        for k, i in enumerate(sel):
            assert np.array_equal(M[k][z[f"s{i}_M_rows_idx"]], z[f"s{i}_M_rows"]), f"M rows mismatch surface {i}"
            assert hashlib.sha256(np.ascontiguousarray(M[k]).tobytes()).digest() == bytes(z[f"s{i}_M_sha"]), f"M sha256 mismatch surface {i}"
        hs, its, tr = eng.stage_matvec_chain(M, g, 9, trace=True)
        for k, i in enumerate(sel):
            assert int(hs[k]) == int(z[f"s{i}_height"]) and int(its[k]) == int(z[f"s{i}_iters"])
            assert np.array_equal(tr[k][: its[k]], z[f"s{i}_trace"]), f"trace mismatch surface {i}"
        del M, dl
    hs, its = eng.heights(coeffs, 10)
    assert [int(h) for h in hs] == [int(z[f"s{i}_height"]) for i in range(n)]
    assert [int(t) for t in its] == [int(z[f"s{i}_iters"]) for i in range(n)]


def test_f7_chain_trace_golden():
    """F_7: build M on the GPU from the golden Delta, check its sha256, then every intermediate vector of the matvec chain
    against the reference's trace (the golden file holds only five rows of each 2925 x 2925 matrix)."""
    z, n = _stages(7)
    idx = [i for i in range(n) if f"s{i}_delta" in z.files]
    eng = _engine(7)
    M = eng.stage_matrix(np.stack([z[f"s{i}_delta"] for i in idx]))
    for k, i in enumerate(idx):
        assert hashlib.sha256(np.ascontiguousarray(M[k]).tobytes()).digest() == bytes(z[f"s{i}_Msha"])
    g = np.stack([z[f"s{i}_g"] for i in idx])
    hs, its, tr = eng.stage_matvec_chain(M, g, 9, trace=True)
    for k, i in enumerate(idx):
        assert int(hs[k]) == int(z[f"s{i}_height"]) and int(its[k]) == int(z[f"s{i}_iters"])
        assert np.array_equal(tr[k][: its[k]], z[f"s{i}_trace"]), f"trace mismatch surface {i}"
