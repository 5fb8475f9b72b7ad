"""Pins the CPU oracle (oracle/qfs_oracle.c) against output of the UNMODIFIED reference package.

The golden files under tests/golden/ were produced by tests/golden/make_golden.py, which imports the
reference (`qfsplit`) in the authoring container and dumps its own intermediates and heights on
seeded inputs; k3_fixture_vectors.json is the reference's published fixture table (heights 1..10 and
infinity over F_5 and F_7).  Everything here runs on CPU.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _stages(p):
    z = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
    return z, int(z["count"])


@pytest.mark.parametrize("p", [3, 5, 7])
def test_power_and_fedder(p):
    z, n = _stages(p)
    for i in range(n):
        g = oracle.power_mod_p(z[f"s{i}_coeffs"], 4, p - 1, p)
        assert np.array_equal(g, z[f"s{i}_g"])
        assert (g[oracle.cap_index(p)] != 0) == (int(z[f"s{i}_height"]) == 1)


@pytest.mark.parametrize("p", [3, 5])
def test_delta1_matrix_chain(p):
    z, n = _stages(p)
    for i in range(n):
        if f"s{i}_delta" not in z.files:
            continue
        d = 4 * (p - 1)
        dl = oracle.delta1(z[f"s{i}_g"], d, p)
        assert np.array_equal(dl, z[f"s{i}_delta"]), f"delta1 mismatch surface {i}"
        M = oracle.build_mts(dl, p)
        assert hashlib.sha256(M.tobytes()).digest() == bytes(z[f"s{i}_Msha"])
        if f"s{i}_M" in z.files:
            assert np.array_equal(M, z[f"s{i}_M"])
        v = z[f"s{i}_g"]
        for want in z[f"s{i}_trace"]:
            v = oracle.matvec(M, v, p)
            assert np.array_equal(v, want)


@pytest.mark.parametrize("p", [3, 5, 7])
def test_height_matrix_taps(p):
    z, n = _stages(p)
    for i in range(n if p < 7 else 2):
        h, it = oracle.height_matrix(z[f"s{i}_coeffs"], p, 10)
        assert (h, it) == (int(z[f"s{i}_height"]), int(z[f"s{i}_iters"]))
    if p < 7:
        for i in range(n):  # the independent polynomial-iteration driver agrees (height.py:97-116)
            assert oracle.height_naive(z[f"s{i}_coeffs"], p, 10) == (int(z[f"s{i}_height"]), int(z[f"s{i}_iters"]))


@pytest.mark.parametrize("p,name,count", [(3, "heights_p3_seed0_w0_3000", 3000), (5, "heights_p5_seed0_w0_10000", 400),
                                          (7, "heights_p7_seed0_w0_10000", 300)])
def test_seeded_streams(p, name, count):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    hs, its = oracle.heights_batch(z["coeffs"][:count], p, 10)
    assert np.array_equal(hs, z["heights"][:count]) and np.array_equal(its, z["iters"][:count])


def test_published_fixture_table_f5():
    rows = [r for r in json.load(open(os.path.join(GOLDEN, "k3_fixture_vectors.json"))) if r["p"] == 5]
    assert sorted(r["height"] for r in rows) == list(range(0, 11))
    coeffs = np.array([r["coeffs"] for r in rows], dtype=np.uint8)
    hs, its = oracle.heights_batch(coeffs, 5, 10)
    assert [int(h) for h in hs] == [r["height"] for r in rows]
    assert [int(i) for i in its] == [r["height"] - 1 if r["height"] else 9 for r in rows]


@pytest.mark.parametrize("bound", [1, 2, 5])
def test_bound_truncation(bound):
    """bound < 2 -> infinity with 0 iterations; otherwise at most bound-1 operator applications (height.py:126-144)."""
    z = np.load(os.path.join(GOLDEN, "heights_p3_seed0_w0_3000.npz"))
    c, full_h = z["coeffs"][:500], z["heights"][:500].astype(int)
    hs, its = oracle.heights_batch(c, 3, bound)
    want_h = np.where((full_h >= 1) & (full_h <= bound), full_h, 0)
    want_it = np.where(want_h > 0, want_h - 1, max(bound - 1, 0))
    assert np.array_equal(hs, want_h) and np.array_equal(its, want_it)


def test_factorised_identities_match_reference_intermediates():
    """The two identities the CUDA kernels rest on (tests/model_factorized.py), against the reference's Delta and M."""
    import model_factorized as mf
    p = 3
    z, n = _stages(3)
    z5, _ = _stages(5)
    done = 0
    for i in range(n):
        coeffs = z[f"s{i}_coeffs"]
        g, h, A, E = mf.carry_parts(coeffs, p)
        assert np.array_equal(g, z[f"s{i}_g"])
        if int(z[f"s{i}_height"]) == 1:
            continue
        dl = mf.delta_factorized(h, A, E, p)
        assert np.array_equal(dl, oracle.delta1(g, 4 * (p - 1), p))
        assert np.array_equal(mf.matrix_gather(dl, p), oracle.build_mts(dl, p))
        done += 1
        if done == 2:
            break
    assert done
    # gather form on a reference F_5 matrix (sampled rows: the pure-Python gather is slow)
    dl, M = z5["s0_delta"], z5["s0_M"]
    tb = mf.tuples(16)
    rng = np.random.default_rng(1)
    for r in rng.integers(0, len(tb), 12):
        for c in rng.integers(0, len(tb), 40):
            I = tuple(5 * a + 4 - b for a, b in zip(tb[r], tb[c]))
            want = int(dl[mf.rank(80, I)]) if min(I) >= 0 else 0
            assert int(M[r, c]) == want


@pytest.mark.parametrize("name", ["r1_spectrum_p5.txt", "r1_spectrum_p7.txt", "r1j_spectrum_p7.txt", "r1f_spectrum_p7_matrix_free.txt"])
def test_spectrum_witnesses(name):
    """The witnesses the GPU spectrum searches wrote (profiles/, fixture-table rows `p ; height ; poly`: one surface for
    every height 1..10 and infinity over F_5 and F_7) recomputed by the CPU oracle."""
    import paper_2502_12428_b200 as q
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rows = [ln for ln in open(os.path.join(root, "profiles", name)) if ln.strip() and not ln.startswith("#")]
    coeffs, want, p = [], [], None
    for ln in rows:
        p_s, h_s, poly = [t.strip() for t in ln.split(";", 2)]
        p = int(p_s)
        want.append(0 if h_s == "inf" else int(h_s))
        coeffs.append(q.parse_poly(poly, 4, p).coeffs)
    got, iters = oracle.heights_batch(np.stack(coeffs), p, 10)   # OpenMP over the surfaces
    assert [int(h) for h in got] == want
    assert [int(i) for i in iters] == [9 if h == 0 else h - 1 for h in want]
    assert set(want) == set(range(11))
