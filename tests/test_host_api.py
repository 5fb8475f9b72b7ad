"""Host-side drop-in layer on CPU: parsing, validation, sampling stream, block partition, search drivers.

The compute hook of the drivers is fed by the CPU oracle here (tests are the only place that may do
that); the GPU tests run the same drivers on the CUDA engine.  Expected values are reference outputs
(tests/golden/) or the reference's documented behaviour, cited per test.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import paper_2502_12428_b200 as q
from paper_2502_12428_b200 import search as qs
from paper_2502_12428_b200.height import split_blocks
from paper_2502_12428_b200.quartic import EXPONENTS

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROWS = json.load(open(os.path.join(GOLDEN, "k3_fixture_vectors.json")))


def cpu_compute(p, coeffs, bound, device):
    return oracle.heights_batch(coeffs, p, bound)


# ---- quartic / parser ---------------------------------------------------------------------------------------
def test_basis_order():
    """index 0 = x4^4, last = x1^4, lex ascending with x1 most significant (monomials.py:182-196)."""
    assert EXPONENTS[0] == (0, 0, 0, 4) and EXPONENTS[34] == (4, 0, 0, 0) and len(EXPONENTS) == 35
    assert list(EXPONENTS) == sorted(EXPONENTS)


def test_parser_matches_reference_on_the_fixture_table():
    for r in ROWS:
        f = q.parse_poly(r["text"], 4, r["p"])
        assert f.coeffs.tolist() == r["coeffs"], r["text"][:40]
        assert q.parse_poly(q.poly_to_text(f), 4, r["p"]) == f


def test_parser_formats_and_errors():
    f = q.parse_poly("x1^4 + 2*x2^2*x3*x4+x1*x2*x3*x4 + 3*x1*x2*x3*x4", 4, 5)
    assert f.coefficient((1, 1, 1, 1)) == 4 and f.coefficient((4, 0, 0, 0)) == 1 and len(f) == 3
    assert q.parse_poly("1:4,0,0,0;2:0,2,1,1\n4:1,1,1,1", 4, 5) == f
    assert q.poly_to_text(f) == "x1^4 + 4*x1*x2*x3*x4 + 2*x2^2*x3*x4"
    for bad, pos in (("", 0), ("x1^4 +", 5), ("x1^", 3), ("x1^4 & x2", 5), ("2**x1", 2)):
        with pytest.raises(q.ParseError) as e:
            q.parse_poly(bad, 4, 5)
        assert e.value.position == pos
    with pytest.raises(q.ParseError):
        q.parse_poly("x5^4", 4, 5)
    with pytest.raises(q.DomainError):
        q.parse_poly("x1^3", 4, 5)  # not a quartic


def test_surface_problem_validation():
    """Same checks as height.py:76-94."""
    f = q.parse_poly("x1^4+x2^4+x3^4+x4^4", 4, 5)
    prob = q.SurfaceProblem(5, 4, f)
    assert prob.bound == 10
    with pytest.raises(q.DomainError):
        q.SurfaceProblem(9, 4, q.Quartic(f.coeffs, 9))
    with pytest.raises(q.DomainError):
        q.SurfaceProblem(5, 3, f)
    with pytest.raises(q.DomainError):
        q.SurfaceProblem(7, 4, f)
    with pytest.raises(q.DomainError):
        q.SurfaceProblem(5, 4, q.Quartic(np.zeros(35, np.uint8), 5))
    with pytest.raises(q.DomainError):
        q.SurfaceProblem(5, 4, f, 0)
    with pytest.raises(q.DomainError):
        q.default_bound(3)
    assert q.HeightResult(math.inf, 10, 9).is_finite is False and q.HeightResult(3, 10, 2).is_finite
    with pytest.raises(q.DomainError):
        q.HeightResult(11, 10, 9)
    assert [q.is_prime(n) for n in (0, 1, 2, 3, 4, 5, 9, 11, 13, 91, 97)] == [False, False, True, True, False, True, False,
                                                                             True, True, False, True]


def test_batch_argument_checks_need_no_gpu():
    with pytest.raises(q.DomainError):
        q.height_batch(5, np.zeros((3, 34), np.uint8))
    with pytest.raises(q.DomainError):
        q.height_batch(5, np.full((3, 35), 5, np.uint8))
    with pytest.raises(q.DomainError):
        q.height_batch(5, np.zeros((3, 35), np.uint8))  # zero form
    with pytest.raises(q.DomainError):
        q.height_batch(4, np.ones((3, 35), np.uint8))
    with pytest.raises(q.DomainError):
        q.height_batch(17, np.ones((3, 35), np.uint8))
    with pytest.raises(q.DomainError):
        q.height_batch(5, np.ones((3, 35), np.uint8), bound=0)


# ---- partition / histogram -------------------------------------------------------------------------------------
def test_split_blocks_is_the_reference_partition():
    """base+1 for the first `extra` workers (search.py:128-135)."""
    assert split_blocks(10, 3) == [(0, 4), (4, 3), (7, 3)]
    assert split_blocks(2, 8) == [(0, 1), (1, 1)]
    assert split_blocks(100000, 8)[-1] == (87500, 12500)
    for total, parts in ((1, 1), (7, 7), (1000, 6)):
        b = split_blocks(total, parts)
        assert sum(n for _, n in b) == total and all(b[i][0] + b[i][1] == b[i + 1][0] for i in range(len(b) - 1))


def test_histogram():
    h = q.HeightHistogram(10)
    h.record_codes(np.array([1, 1, 2, 0, 3, 1], np.int8))
    h.record(math.inf)
    h.record(2)
    assert h.as_dict() == {"bound": 10, "counts": {"1": 3, "2": 2, "3": 1}, "inf": 2, "total": 8}
    assert h.fraction_at_least(2) == 5 / 8
    h.check()
    other = q.HeightHistogram(9)
    with pytest.raises(q.DomainError):
        h.merge(other)
    assert "inf" in q.histogram_text(h, 5)


# ---- sampling stream and drivers (CPU compute hook) ------------------------------------------------------------------
@pytest.mark.parametrize("p,name", [(3, "heights_p3_seed0_w0_3000"), (5, "heights_p5_seed0_w0_10000")])
def test_sampler_reproduces_the_reference_stream(p, name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    n = len(z["coeffs"])  # 3000 resp. 10000 rows dumped by the reference's own sampler
    assert np.array_equal(q.sample_block(p, n, int(z["seed"]), int(z["worker"])), z["coeffs"])
    # the vectorised sampler equals the reference's call-per-surface loop, also across a split
    rng_a, rng_b = np.random.default_rng([7, 3]), np.random.default_rng([7, 3])
    seq = np.stack([qs.sample_coeffs(rng_a, p) for _ in range(300)])
    assert np.array_equal(np.concatenate([qs.sample_rows(rng_b, p, 123), qs.sample_rows(rng_b, p, 177)]), seq)
    rng = np.random.default_rng([0, 0])
    assert np.array_equal(q.sample_surface(rng, p).coeffs, z["coeffs"][0])


def test_run_search_matches_reference_histogram():
    z = np.load(os.path.join(GOLDEN, "heights_p3_seed0_w0_3000.npz"))
    cfg = q.SearchConfig(p=3, sample_count=3000, rng_seed=0, parallelism=1)
    hist, found = q.run_search(cfg, compute=cpu_compute)
    want = np.bincount(z["heights"].astype(int), minlength=11)
    assert hist.total == 3000 and hist.infinite == want[0]
    assert all(hist.counts.get(h, 0) == want[h] for h in range(1, 11))
    # the found log is the sequence of strict new maxima of the finite heights (search.py:113-115)
    best, log = 0, []
    for i, h in enumerate(z["heights"].astype(int)):
        if h > best:
            best = h
            log.append((i, h))
    assert [(s.index, s.height) for s in found] == log
    assert np.array_equal(found[0].f.coeffs, z["coeffs"][found[0].index])


def test_run_search_parallelism_and_target():
    cfg2 = q.SearchConfig(p=3, sample_count=601, rng_seed=5, parallelism=2)
    h2, f2 = q.run_search(cfg2, compute=cpu_compute)
    # worker w draws from default_rng([seed, w]); blocks are 301 + 300 (search.py:103,128-135)
    c0, c1 = q.sample_block(3, 301, 5, 0), q.sample_block(3, 300, 5, 1)
    hs = np.concatenate([oracle.heights_batch(c0, 3, 10)[0], oracle.heights_batch(c1, 3, 10)[0]])
    assert h2.total == 601 and h2.counts == {int(h): int(c) for h, c in enumerate(np.bincount(hs)) if c and h}
    assert [s.index for s in f2] == sorted(s.index for s in f2)
    again = q.run_search(cfg2, compute=cpu_compute)
    assert again[0].as_dict() == h2.as_dict() and [(s.index, s.height) for s in again[1]] == [(s.index, s.height) for s in f2]
    # target_height: each worker stops right after its first hit (search.py:116-117)
    first = int(np.nonzero(oracle.heights_batch(c0, 3, 10)[0] == 3)[0][0])
    ht, _ = q.run_search(q.SearchConfig(p=3, sample_count=301, rng_seed=5, target_height=3), compute=cpu_compute)
    assert ht.total == first + 1 and ht.counts[3] == 1


def test_verify_fixtures_and_spectrum():
    text = open(q.fixtures_path()).read()
    rows = q.parse_fixtures(text)
    assert len(rows) == 32 and rows[10].expected == math.inf
    verdicts = q.verify_fixtures(text, primes=[5], compute=cpu_compute)
    assert len(verdicts) == 11 and all(v.ok for v in verdicts)
    with pytest.raises(q.ParseError):
        q.parse_fixtures("5 ; 2")
    with pytest.raises(q.DomainError):
        q.verify_fixtures(text, primes=[5], method="bogus")
    wit, hist, blocks = q.spectrum_search(3, block=400, rng_seed=0, bound=10, max_blocks=3, compute=cpu_compute, want=[1, 2, 3])
    assert {1, 2, 3} <= set(wit) and blocks == 1 and hist.total == 400
    for line, h in zip(q.spectrum_rows(wit).splitlines(), sorted(wit, key=lambda x: (x == 0, x))):
        p_s, h_s, poly = [t.strip() for t in line.split(";", 2)]
        assert int(p_s) == 3 and h_s == ("inf" if h == 0 else str(h))
        f = q.parse_poly(poly, 4, 3)
        assert oracle.height_matrix(f.coeffs, 3, 10)[0] == h


def test_sampler_stream_arithmetic_in_python_integers():
    """The arithmetic of csrc/qfs_sample.cuh, written in Python integers, against numpy's generator: PCG64 = 128-bit LCG stepped
    BEFORE the XSL-RR output, jump-ahead by the (multiplier, increment) doubling recurrence, two 32-bit draws per output (low half
    first), Lemire multiply-shift to [0, p).  (search.py:92-103 draws rng.integers(0, p, size=35) from default_rng([seed, w]).)"""
    A, M = 0x2360ED051FC65DA44385DF649FCCF645, (1 << 128) - 1

    def out(s):
        x, r = ((s >> 64) ^ s) & 0xFFFFFFFFFFFFFFFF, s >> 122
        return ((x >> r) | (x << (64 - r))) & 0xFFFFFFFFFFFFFFFF if r else x

    def advance(s, inc, delta):
        am, ap, cm, cp = 1, 0, A, inc
        while delta:
            if delta & 1:
                am, ap = (am * cm) & M, (ap * cm + cp) & M
            cp, cm, delta = ((cm + 1) * cp) & M, (cm * cm) & M, delta >> 1
        return (am * s + ap) & M

    for p, seed, w in ((5, 0, 0), (7, 3, 2), (11, 9, 1), (13, 0, 65)):
        st = np.random.PCG64(np.random.SeedSequence([seed, w])).state["state"]
        want = np.random.default_rng([seed, w]).integers(0, p, size=(40, 35))
        for r in (0, 1, 17, 39):
            s = advance(st["state"], st["inc"], (35 * r) >> 1)
            vals = []
            for _ in range(19):
                s = (s * A + st["inc"]) & M
                o = out(s)
                vals += [o & 0xFFFFFFFF, o >> 32]
            row = [(v * p) >> 32 for v in vals[(35 * r) & 1:][:35]]
            assert row == want[r].tolist()
