"""The literal on-device route (csrc/qfs_literal.cuh: dense powers, checked division, splitting operator -- none of the
engine's identities) against the reference's goldens, and the engine against it beyond the sizes the goldens cover."""
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_literal_argument_checks_need_no_gpu():
    from paper_2502_12428_b200 import DomainError, literal_heights
    with pytest.raises(DomainError):
        literal_heights(11, np.zeros((1, 35), dtype=np.uint8))          # p = 3, 5, 7 only
    with pytest.raises(DomainError):
        literal_heights(5, np.zeros((1, 34), dtype=np.uint8))
    with pytest.raises(DomainError):
        literal_heights(5, np.ones((1, 35), dtype=np.uint8), bound=0)


@pytest.mark.gpu
@pytest.mark.parametrize("p", [3, 5, 7])
def test_literal_stages_match_the_reference(p):
    """g and Delta_1(g) of the golden surfaces (written by the unmodified reference, tests/golden/make_golden.py)."""
    from paper_2502_12428_b200 import literal_heights
    z = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
    n = int(z["count"])
    coeffs = np.stack([z[f"s{i}_coeffs"] for i in range(n)])
    hs, its, g, dl = literal_heights(p, coeffs, 10, want_g=True, want_delta=True)
    for i in range(n):
        assert np.array_equal(g[i], z[f"s{i}_g"]), f"g mismatch surface {i}"
        want_h = int(z[f"s{i}_height"])
        assert int(hs[i]) == (want_h if want_h <= 10 else 0) and int(its[i]) == int(z[f"s{i}_iters"]), (i, hs[i], its[i])
        if f"s{i}_delta" in z.files:
            bad = np.nonzero(dl[i] != z[f"s{i}_delta"])[0]
            assert bad.size == 0, f"delta mismatch surface {i}: {bad.size} entries, first {bad[:5]}"


@pytest.mark.gpu
@pytest.mark.parametrize("p,name,count", [(3, "heights_p3_seed0_w0_3000", 3000), (5, "heights_p5_seed0_w0_10000", 10000),
                                          (7, "heights_p7_seed0_w0_10000", 10000)])
def test_literal_heights_match_the_reference_stream(p, name, count):
    from paper_2502_12428_b200 import literal_heights
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    hs, its = literal_heights(p, z["coeffs"][:count], 10)
    bad = np.nonzero((hs != z["heights"][:count]) | (its != z["iters"][:count]))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: got {hs[bad[:5]]} want {z['heights'][bad[:5]]}"


@pytest.mark.gpu
@pytest.mark.parametrize("p,B,nd", [(3, 5000, 64), (5, 20000, 24), (7, 2000, 6)])
def test_engine_agrees_with_the_literal_route(p, B, nd):
    """Fresh seeded surfaces (not in any golden): heights and iteration counts of both engine modes, g of k_power_full and
    Delta of the tensor-core Witt carry against the literal computation."""
    from paper_2502_12428_b200 import height_batch, literal_heights
    from paper_2502_12428_b200.engine import get_engine
    rng = np.random.default_rng([2024, p])
    c = rng.integers(0, p, size=(B, 35)).astype(np.uint8)
    c[(c == 0).all(axis=1), 0] = 1
    lh, li = literal_heights(p, c, 10)
    hs, its = height_batch(p, c[:500], 10, method="literal")      # the same route through the batch entry
    assert np.array_equal(hs, lh[:500]) and np.array_equal(its, li[:500])
    for method in ("matrix", "naive"):
        hs, its = height_batch(p, c, 10, method=method)
        bad = np.nonzero((hs != lh) | (its != li))[0]
        assert bad.size == 0, f"{method}: {bad.size} mismatches, first {bad[:5]}: engine {hs[bad[:5]]} literal {lh[bad[:5]]}"
    hard = np.nonzero(lh != 1)[0][:nd]
    _, _, g, dl = literal_heights(p, c[hard], 10, want_g=True, want_delta=True)
    eng = get_engine(p, 0)
    g2, _ = eng.stage_power(c[hard])
    assert np.array_equal(g, g2)
    assert np.array_equal(dl, eng.stage_delta(c[hard]))


@pytest.mark.gpu
def test_literal_bound_and_errors():
    from paper_2502_12428_b200 import DomainError, literal_heights
    from paper_2502_12428_b200.engine import get_engine
    rng = np.random.default_rng([7, 7])
    c = rng.integers(0, 5, size=(4000, 35)).astype(np.uint8)
    c[(c == 0).all(axis=1), 0] = 1
    for bound in (1, 2, 3):
        lh, li = literal_heights(5, c, bound)
        hs, its = get_engine(5, 0).heights(c, bound)
        assert np.array_equal(lh, hs) and np.array_equal(li, its), bound
    bad = c[:8].copy()
    bad[3, 5] = 5
    with pytest.raises(DomainError):
        literal_heights(5, bad, 10)
    with pytest.raises(DomainError):
        literal_heights(5, np.zeros((2, 35), dtype=np.uint8), 10)


@pytest.mark.gpu
def test_published_rows_through_the_literal_route():
    """Every published row over F_3, F_5, F_7 (fixtures/k3_tables.txt, the paper's tables) by the literal computation."""
    import paper_2502_12428_b200 as q
    text = open(q.fixtures_path()).read()
    verdicts = q.verify_fixtures(text, primes=[3, 5, 7], method="literal")
    assert len(verdicts) == 22 and all(v.ok for v in verdicts), [(v.row.p, v.row.expected, v.got) for v in verdicts if not v.ok]
