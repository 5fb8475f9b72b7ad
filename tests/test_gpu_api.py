"""GPU tests of the drop-in Python layer and of the pipeline's batching edge cases (all through the C ABI)."""
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ROWS = json.load(open(os.path.join(GOLDEN, "k3_fixture_vectors.json")))


def test_height_matrix_drop_in():
    """Fermat trio of the reference's acceptance suite (tests/test_acceptance.py:92-100) and API parity."""
    import paper_2502_12428_b200 as q
    fermat5 = q.SurfaceProblem(5, 4, q.parse_poly("x1^4+x2^4+x3^4+x4^4", 4, 5))
    assert q.height_matrix(fermat5) == q.HeightResult(1, 10, 0)
    dwork5 = q.SurfaceProblem(5, 4, q.parse_poly("x1^4+x2^4+x3^4+x4^4+x1*x2*x3*x4", 4, 5))
    assert q.height_matrix(dwork5) == q.HeightResult(math.inf, 10, 9)
    fermat3 = q.SurfaceProblem(3, 4, q.parse_poly("x1^4+x2^4+x3^4+x4^4", 4, 3))
    assert q.height_matrix(fermat3) == q.HeightResult(math.inf, 10, 9)
    assert q.height_matrix(q.SurfaceProblem(3, 4, fermat3.f, 4)) == q.HeightResult(math.inf, 4, 3)
    assert q.height_matrix(q.SurfaceProblem(5, 4, dwork5.f, 1)) == q.HeightResult(math.inf, 1, 0)
    with pytest.raises(q.DomainError):
        q.height_matrix(fermat5, algorithm="bogus")
    r = [x for x in ROWS if x["p"] == 7 and x["height"] == 6][0]
    assert q.height_of_coeffs(7, r["coeffs"]) == q.HeightResult(6, 10, 5)


def test_verify_fixtures_on_gpu():
    import paper_2502_12428_b200 as q
    verdicts = q.verify_fixtures(open(q.fixtures_path()).read(), primes=[5, 7])
    assert len(verdicts) == 22 and all(v.ok for v in verdicts)
    assert [v.got for v in verdicts[:11]] == list(range(1, 11)) + [math.inf]


def test_f11_published_rows():
    """The five F_11 rows of the published table (extended suite of the reference, tests/test_acceptance.py:84-89);
    12341 x 12341 operator, 152 MB per surface."""
    import paper_2502_12428_b200 as q
    rows = [r for r in ROWS if r["p"] == 11]
    hs, its = q.height_batch(11, np.array([r["coeffs"] for r in rows], dtype=np.uint8))
    assert [int(h) for h in hs] == [r["height"] for r in rows]
    assert [int(i) for i in its] == [r["height"] - 1 for r in rows]


def test_f13_published_rows():
    """The five F_13 rows of the published table (k3_tables.txt:30-34): 20825 x 20825 operator, 434 MB per surface,
    Delta from k_delta_mma (SPLIT CTAs per quad)."""
    import paper_2502_12428_b200 as q
    rows = [r for r in ROWS if r["p"] == 13]
    hs, its = q.height_batch(13, np.array([r["coeffs"] for r in rows], dtype=np.uint8))
    assert [int(h) for h in hs] == [r["height"] for r in rows]
    assert [int(i) for i in its] == [r["height"] - 1 for r in rows]
    # a seeded handful more: the distribution is ~1/13 hard, heights 1 and 2 only at this size
    c = q.sample_block(13, 40, 3, 0)
    hs, its = q.height_batch(13, c)
    assert set(int(h) for h in hs) <= {1, 2, 3} and (hs == 1).sum() >= 30


@pytest.mark.parametrize("p", [3, 5, 7, 11, 13])
def test_the_three_witt_carry_kernels_agree(p, monkeypatch):
    """k_delta_mma (tensor cores, the default) against the two DP4A kernels it replaced -- k_delta (slabs, 4-CTA clusters; does not
    fit shared memory at p = 13) and k_delta_direct -- on the same surfaces: identical dense Delta and, through the whole pipeline,
    identical heights (mirrors the reference pinning its three matrix builders on each other, tests/test_acceptance.py:110-125)."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import Engine, get_engine
    c = q.sample_block(p, 6 if p < 11 else 2, 21, 0)
    big = q.sample_block(p, 300 if p < 11 else 30, 22, 0)
    want = get_engine(p, 0).stage_delta(c)
    h0, i0 = get_engine(p, 0).heights(big, 10)
    for var, val in (("QFS_DELTA_DIRECT", "1"), ("QFS_DELTA_V", "1")):
        if p == 13 and var == "QFS_DELTA_V":
            continue
        monkeypatch.setenv(var, val)
        eng = Engine(p, 0)
        try:
            assert np.array_equal(eng.stage_delta(c), want), var
            h1, i1 = eng.heights(big, 10)
            assert np.array_equal(h1, h0) and np.array_equal(i1, i0), var
        finally:
            eng.close()
            monkeypatch.delenv(var)


@pytest.mark.parametrize("p", [3, 5, 7, 11])
def test_both_chain_kernels_agree(p, monkeypatch):
    """k_chain (a surface per persistent CTA) and k_chain_grid (the whole cooperative grid on one surface at a time,
    chosen automatically for few long surfaces) against each other and the golden traces: heights, iteration counts
    and every intermediate vector."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import Engine
    big = q.sample_block(p, {3: 4000, 5: 3000, 7: 1500, 11: 700}[p], 31, 0)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("QFS_CHAIN_GRID", mode)
        eng = Engine(p, 0)
        try:
            out[mode] = eng.heights(big, 10)
            if p <= 5:
                z = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
                idx = [i for i in range(int(z["count"])) if f"s{i}_M" in z.files]
                M = np.stack([z[f"s{i}_M"] for i in idx])
                g = np.stack([z[f"s{i}_g"] for i in idx])
                hs, its, tr = eng.stage_matvec_chain(M, g, 9, trace=True)
                for k, i in enumerate(idx):
                    assert int(hs[k]) == int(z[f"s{i}_height"]) and int(its[k]) == int(z[f"s{i}_iters"])
                    assert np.array_equal(tr[k][: its[k]], z[f"s{i}_trace"])
        finally:
            eng.close()
    assert np.array_equal(out["0"][0], out["1"][0]) and np.array_equal(out["0"][1], out["1"][1])
    assert (out["0"][0] > 2).sum() + (out["0"][0] == 0).sum() > 0  # the chain kernels did run


def test_run_search_on_gpu_matches_reference():
    import paper_2502_12428_b200 as q
    z = np.load(os.path.join(GOLDEN, "heights_p5_seed0_w0_10000.npz"))
    hist, found = q.run_search(q.SearchConfig(p=5, sample_count=10000, rng_seed=0, parallelism=1))
    want = np.bincount(z["heights"].astype(int), minlength=11)
    assert hist.infinite == want[0] and all(hist.counts.get(h, 0) == want[h] for h in range(1, 11))
    assert found[-1].height == int(z["heights"].max())
    h2, _ = q.run_search(q.SearchConfig(p=5, sample_count=2001, rng_seed=3, parallelism=2))
    a, b = q.sample_block(5, 1001, 3, 0), q.sample_block(5, 1000, 3, 1)
    hs, _ = q.height_batch(5, np.concatenate([a, b]))
    assert h2.counts == {int(h): int(c) for h, c in enumerate(np.bincount(hs)) if c and h}


@pytest.mark.parametrize("p,B", [(5, 0), (5, 1), (5, 3), (5, 5), (7, 6), (3, 9)])
def test_ragged_batches_and_chunking(p, B):
    """Batch sizes that are not whole quads, the empty batch, and hard-surface chunks smaller than the batch."""
    import oracle
    from paper_2502_12428_b200.engine import Engine
    rng = np.random.default_rng([11, p])
    coeffs = rng.integers(0, p, size=(B, 35)).astype(np.uint8)
    coeffs[(coeffs == 0).all(axis=1), 0] = 1
    # make sure the hard path is exercised: append known height>=2 rows of the golden stream
    z = np.load(os.path.join(GOLDEN, f"heights_p{p}_seed0_w0_{ {3: 3000, 5: 10000, 7: 10000}[p] }.npz"))
    hard = z["coeffs"][np.nonzero(z["heights"] != 1)[0][:B]]
    coeffs = np.concatenate([coeffs, hard]) if B else coeffs
    want = oracle.heights_batch(coeffs, p, 10) if len(coeffs) else (np.empty(0, np.int8),) * 2
    eng = Engine(p, 0)
    try:
        for chunk in (0, 1, 5):
            eng.set_chunk(chunk)
            hs, its = eng.heights(coeffs, 10)
            assert np.array_equal(hs, want[0]) and np.array_equal(its, want[1]), f"chunk={chunk}"
    finally:
        eng.close()


def test_device_buffers_and_errors():
    import torch
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    z = np.load(os.path.join(GOLDEN, "heights_p5_seed0_w0_10000.npz"))
    dev = torch.from_numpy(z["coeffs"][:2000]).cuda()
    hs, its = get_engine(5, 0).heights(dev, 10)
    assert hs.is_cuda and np.array_equal(hs.cpu().numpy(), z["heights"][:2000]) and np.array_equal(its.cpu().numpy(), z["iters"][:2000])
    bad = z["coeffs"][:8].copy()
    bad[3, 7] = 5  # not a residue mod 5: caught on the device, reported as the reference's DomainError
    with pytest.raises(q.DomainError):
        get_engine(5, 0).heights(torch.from_numpy(bad).cuda(), 10)
    zero = z["coeffs"][:8].copy()
    zero[2] = 0
    with pytest.raises(q.DomainError):
        get_engine(5, 0).heights(torch.from_numpy(zero).cuda(), 10)


def test_large_batch_properties():
    """Full-size batch (BASELINE.json configs[1]) through size-independent properties: heights are invariant under
    scaling f by a unit and under permuting the variables (tests/test_height.py in the reference), and the
    height-1 fraction is 1 - 1/p within 5 sigma (tests/test_acceptance.py:210-219)."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.quartic import EXPONENTS, INDEX_OF
    p, B = 5, 100000
    rng = np.random.default_rng(2024)
    c = rng.integers(0, p, size=(B, 35)).astype(np.uint8)
    c[(c == 0).all(axis=1), 0] = 1
    hs, its = q.height_batch(p, c)
    frac = float((hs == 1).mean())
    assert abs(frac - (1 - 1 / p)) < 5 * math.sqrt((1 / p) * (1 - 1 / p) / B)
    assert np.array_equal(its, np.where(hs > 0, hs - 1, 9))
    hs2, _ = q.height_batch(p, (c.astype(np.int64) * 3 % p).astype(np.uint8))
    assert np.array_equal(hs, hs2)
    perm = (2, 0, 3, 1)
    idx = np.array([INDEX_OF[tuple(e[perm[k]] for k in range(4))] for e in EXPONENTS])
    hs3, _ = q.height_batch(p, np.ascontiguousarray(c[:, idx]))
    assert np.array_equal(hs, hs3)


def test_full_size_f7_batch_matrix_path_equals_matrix_free_iteration():
    """BASELINE.json configs[2] at full size (100 000 seeded quartics over F_7, ~14 000 operator matrices of 8.6 MB, several
    HBM chunks): the matrix path (Delta, M in HBM, streamed chain) and the matrix-free polynomial iteration are independent
    routes to the same heights and iteration counts; the first 10 000 are the reference's own seeded golden set."""
    import paper_2502_12428_b200 as q
    c = q.sample_block(7, 100000, 0, 0)
    hs, its = q.height_batch(7, c)
    hf, itf = q.height_batch(7, c, method="naive")
    assert np.array_equal(hs, hf) and np.array_equal(its, itf)
    z = np.load(os.path.join(GOLDEN, "heights_p7_seed0_w0_10000.npz"))
    assert np.array_equal(c[:10000], z["coeffs"])
    assert np.array_equal(hs[:10000].astype(np.int64), z["heights"].astype(np.int64))
    assert np.array_equal(its[:10000].astype(np.int64), z["iters"].astype(np.int64))


@pytest.mark.parametrize("p", [3, 5, 7, 11])
def test_results_do_not_depend_on_what_the_workspaces_held(p):
    """Recycled device memory is not zero: poison every workspace between calls (qfs_debug_fill_workspaces)
    and demand identical heights, stage taps and exports.  Regression: the last slab of Delta (I1 = D) and its
    guard zeros were never written, which only showed once a context reused memory freed by another one."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    eng = get_engine(p, 0)
    rows = [r for r in ROWS if r["p"] == p] if p != 3 else []
    coeffs = np.array([r["coeffs"] for r in rows], dtype=np.uint8) if rows else q.sample_block(3, 40, 4, 0)
    coeffs = np.concatenate([coeffs, q.sample_block(p, 37, 9, 1)])
    want_h, want_i = eng.heights(coeffs, 10)
    if rows:
        assert [int(h) for h in want_h[:len(rows)]] == [int(r["height"]) for r in rows]   # 0 = infinity in both
    want_d = eng.stage_delta(coeffs[:3])
    want_m = eng.export_matrix(coeffs[:2])
    for byte in (0xFF, 0x01, 0xA7):
        eng.debug_fill_workspaces(byte)
        got_h, got_i = eng.heights(coeffs, 10)
        assert np.array_equal(got_h, want_h) and np.array_equal(got_i, want_i)
        eng.debug_fill_workspaces(byte)
        assert np.array_equal(eng.stage_delta(coeffs[:3]), want_d)
        eng.debug_fill_workspaces(byte)
        assert np.array_equal(eng.export_matrix(coeffs[:2]), want_m)


def test_matrix_free_iteration_equals_the_reference_heights():
    """qfs_heights_free (polynomial iteration, no Delta, no M) against the heights AND iteration counts the
    reference produced for its seeded streams (10000 F_5, 10000 F_7, 3000 F_3), and against the matrix path."""
    import paper_2502_12428_b200 as q
    for p, name in ((3, "heights_p3_seed0_w0_3000.npz"), (5, "heights_p5_seed0_w0_10000.npz"), (7, "heights_p7_seed0_w0_10000.npz")):
        z = np.load(os.path.join(GOLDEN, name))
        hs, its = q.height_batch(p, z["coeffs"], 10, method="naive")
        assert np.array_equal(hs.astype(np.int64), z["heights"].astype(np.int64))
        assert np.array_equal(its.astype(np.int64), z["iters"].astype(np.int64))
        hm, im = q.height_batch(p, z["coeffs"], 10)
        assert np.array_equal(hs, hm) and np.array_equal(its, im)


def test_matrix_free_bounds_fixtures_and_drivers():
    import paper_2502_12428_b200 as q
    verdicts = q.verify_fixtures(open(q.fixtures_path()).read(), method="naive")
    assert len(verdicts) == 32 and all(v.ok for v in verdicts)
    dwork5 = q.SurfaceProblem(5, 4, q.parse_poly("x1^4+x2^4+x3^4+x4^4+x1*x2*x3*x4", 4, 5))
    assert q.height_naive(dwork5) == q.height_matrix(dwork5) == q.HeightResult(math.inf, 10, 9)
    for bound in (1, 2, 3, 4, 7):
        prob = q.SurfaceProblem(5, 4, dwork5.f, bound)
        assert q.height_naive(prob) == q.height_matrix(prob) == q.HeightResult(math.inf, bound, bound - 1)
    c = q.sample_block(11, 300, 5, 0)
    h0, i0 = q.height_batch(11, c)
    h1, i1 = q.height_batch(11, c, method="naive")
    assert np.array_equal(h0, h1) and np.array_equal(i0, i1)


def test_reference_named_stage_functions():
    """power_mod_p / fedder_survives / delta1 / build_mts(delta, d, p) / to_dense / matvec under the reference's names and call
    forms (qfsplit/__init__.py:11-114; the loop is height_matrix's, height.py:119-144), against the reference's own
    intermediates (tests/golden/stages_p5.npz)."""
    import paper_2502_12428_b200 as q
    p = 5
    z = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
    i = [k for k in range(int(z["count"])) if f"s{k}_M" in z.files][0]
    f = q.Quartic(z[f"s{i}_coeffs"], p)
    g = q.power_mod_p(f, p - 1)
    assert np.array_equal(g.values, z[f"s{i}_g"]) and g.degree == 16 and g.modulus == p
    assert q.fedder_survives(g) == (int(z[f"s{i}_height"]) == 1)
    delta = q.delta1(g)
    assert np.array_equal(delta.values, z[f"s{i}_delta"]) and delta.degree == 80
    m = q.build_mts(delta, 16, p, "wics")
    assert np.array_equal(m.entries, z[f"s{i}_M"]) and m == q.build_mts(f, p)
    gv = q.to_dense(g)
    assert gv.values.dtype == np.uint64
    cap = 564
    h, iters = 2, 0
    while True:       # height.py:135-144
        gv = q.matvec(m, gv)
        assert np.array_equal(gv.values, z[f"s{i}_trace"][iters])
        iters += 1
        if int(gv.values[cap]) != 0 or h == 10:
            break
        h += 1
    assert iters == int(z[f"s{i}_iters"])
    with pytest.raises(q.DomainError):
        q.power_mod_p(f, 3)
    with pytest.raises(q.DomainError):     # an arbitrary polynomial is not a Witt-carry input here
        q.delta1(q.DenseForm(z[f"s{i}_g"], 16, p))
    with pytest.raises(q.DomainError):
        q.build_mts(delta, 16, p, "bogus")


@pytest.mark.parametrize("p", [3, 5, 7])
def test_direct_gather_builder_equals_the_staged_builder_and_the_reference(p, monkeypatch):
    """Two independent device builders -- k_matrix (QFS_MATRIX_V=4: every thread gathers its entries straight from global Delta)
    and k_matrix_staged (bulk-copied windows in shared memory) -- produce the reference's matrix (sha256 of the entry block),
    as the reference pins TRIV = MERGE = WICS on each other (tests/test_acceptance.py:110-125)."""
    import hashlib
    from paper_2502_12428_b200.engine import Engine, get_engine
    z = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
    idx = [i for i in range(int(z["count"])) if f"s{i}_delta" in z.files]
    dl = np.stack([z[f"s{i}_delta"] for i in idx])
    staged = get_engine(p, 0).stage_matrix(dl)
    monkeypatch.setenv("QFS_MATRIX_V", "4")
    eng = Engine(p, 0)
    try:
        direct = eng.stage_matrix(dl)
        c = np.stack([z[f"s{i}_coeffs"] for i in range(int(z["count"]))])
        h4 = eng.heights(c, 10)
    finally:
        eng.close()
    assert np.array_equal(direct, staged)
    for k, i in enumerate(idx):
        assert hashlib.sha256(np.ascontiguousarray(direct[k]).tobytes()).digest() == bytes(z[f"s{i}_Msha"])
    h6 = get_engine(p, 0).heights(c, 10)
    assert np.array_equal(h4[0], h6[0]) and np.array_equal(h4[1], h6[1])
    assert [int(h) for h in h6[0]] == [int(z[f"s{i}_height"]) for i in range(int(z["count"]))]


def test_stream_order_device_checks_and_shared_engine():
    """(1) a coefficient tensor written on the default stream right before the call is read after the write (the library orders
    its stream behind the caller's, the legacy default stream included); (2) large uint8 batches are validated on the device;
    (3) two threads on one Engine take turns (height_batch(devices=[0, 0])); (4) the caller's current device is left alone."""
    import torch
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    z = np.load(os.path.join(GOLDEN, "heights_p5_seed0_w0_10000.npz"))
    eng = get_engine(5, 0)
    src = torch.from_numpy(z["coeffs"]).cuda()
    for _ in range(5):
        dev = torch.ones_like(src)                     # stale content: the form x-everything, height known to differ
        big = torch.empty(64 << 20, device="cuda").normal_()   # keep the default stream busy in front of the copy
        dev.copy_(src, non_blocking=True)              # queued on the default stream, no synchronisation
        hs, its = eng.heights(dev, 10)
        assert np.array_equal(hs.cpu().numpy(), z["heights"]) and np.array_equal(its.cpu().numpy(), z["iters"])
        del big
    bad = z["coeffs"].copy()
    bad[7777, 3] = 9
    with pytest.raises(q.DomainError):
        q.height_batch(5, bad)
    zero = z["coeffs"].copy()
    zero[4242] = 0
    with pytest.raises(q.DomainError):
        q.height_batch(5, zero)
    hs, its = q.height_batch(5, z["coeffs"], devices=[0, 0])
    assert np.array_equal(hs, z["heights"]) and np.array_equal(its, z["iters"])
    out = (np.empty(10000, np.int8), np.empty(10000, np.int8))
    assert q.height_batch(5, z["coeffs"], out=out)[0] is out[0] and np.array_equal(out[0], z["heights"])
    assert torch.cuda.current_device() == 0
    assert eng.stats()["matvec_steps"] == int(z["iters"].astype(np.int64).sum())


def test_device_sampler_reproduces_the_reference_stream():
    """qfs_sample_quartics against the host sampler (which is pinned on the reference's own seeded dumps, tests/test_host_api.py):
    identical blocks for several primes / seeds / workers / sizes, into host and device memory; and the one thing the device
    only reports -- block (seed 0, worker 65) over F_13 holds a Lemire rejection at draw 541 684 -- is reported, and
    device_block falls back to the host stream for it."""
    import torch
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    from paper_2502_12428_b200.search import device_block
    for p, seed, w, n in ((5, 0, 0, 100000), (5, 0, 3, 777), (7, 12, 5, 50001), (11, 1, 0, 4000), (13, 0, 64, 20000), (3, 5, 1, 1)):
        got, clean = get_engine(p, 0).sample(seed, w, n)
        assert clean and np.array_equal(got, q.sample_block(p, n, seed, w)), (p, seed, w, n)
    dev = torch.empty((30000, 35), dtype=torch.uint8, device="cuda:0")
    _, clean = get_engine(7, 0).sample(2, 9, 30000, out=dev)
    assert clean and np.array_equal(dev.cpu().numpy(), q.sample_block(7, 30000, 2, 9))
    _, clean = get_engine(13, 0).sample(0, 65, 100000)
    assert not clean
    _, clean = get_engine(13, 0).sample(0, 65, 15000)      # the rejection sits behind row 15 000: this prefix is clean
    assert clean
    coeffs, codes, its = device_block(13, 100000, 0, 65)
    assert isinstance(coeffs, np.ndarray) and np.array_equal(coeffs, q.sample_block(13, 100000, 0, 65))
    hs, _ = q.height_batch(13, coeffs[:3000], method="naive")
    assert np.array_equal(codes[:3000], hs)


def test_spectrum_search_on_the_gpu_and_its_witnesses():
    """SURVEY 8(f)1 / BASELINE configs[3] at F_5: sample seeded blocks until every height 1..10 and infinity has a witness (blocks
    drawn and solved on the device), then re-verify every witness with the CPU oracle and regenerate it from (seed, block, index)."""
    import oracle
    import paper_2502_12428_b200 as q
    wit, hist, blocks = q.spectrum_search(5, block=100000, rng_seed=0, max_blocks=400)
    assert set(wit) == set(range(0, 11)) and hist.total == 100000 * blocks
    for code, (blk, i, f) in wit.items():
        oh, _ = oracle.heights_batch(f.coeffs[None, :], 5, 10)
        assert int(oh[0]) == code
        assert np.array_equal(q.sample_block(5, i + 1, 0, blk)[i], f.coeffs)
    rows = q.spectrum_rows(wit).splitlines()
    assert len(rows) == 11 and rows[-1].startswith("5 ; inf ;")
    verdicts = q.verify_fixtures(q.spectrum_rows(wit))
    assert all(v.ok for v in verdicts)
    # the matrix-free mode finds the same witnesses (same blocks, same heights)
    wit2, hist2, blocks2 = q.spectrum_search(5, block=100000, rng_seed=0, max_blocks=400, method="naive")
    assert blocks2 == blocks and {h: w[:2] for h, w in wit2.items()} == {h: w[:2] for h, w in wit.items()}


@pytest.mark.parametrize("p,want", [(5, (8, 4, 7, 2)), (7, (5, 4, 6, 2)), (11, (1, 1, 3, 1))])
def test_stage_kernels_keep_their_resident_cta_counts(p, want):
    """The stage kernels are tuned for specific CTA counts per SM; a few bytes of shared memory or a few
    registers too many cost one silently (k_delta_mma<7> ran on three CTAs instead of four for half of round 2)."""
    from paper_2502_12428_b200.engine import get_engine
    occ = get_engine(p, 0).occupancy()
    got = (occ["k_power_full"], occ["k_delta_mma"], occ["k_matrix_staged"], occ["k_chain"])
    for name, g, w in zip(("k_power_full", "k_delta_mma", "k_matrix_staged", "k_chain"), got, want):
        assert w is None or g >= w, f"{name}<{p}>: {g} resident CTAs per SM, tuned for {w}"


@pytest.mark.parametrize("p", [3, 5, 7])
def test_chain_cap_row_test_equals_the_traced_chain(p, monkeypatch):
    """Without a trace the chain kernels test the cap row of a step before they stream M for it (qfs_chain.cuh: cap_row_hit) and
    skip the last application's other rows; with a trace they compute every vector.  Same heights and iteration counts from the
    same matrices and start vectors, for both kernels, from v0 = g (start at step 1) and for every step budget."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import Engine
    c = q.sample_block(p, {3: 400, 5: 300, 7: 120}[p], 37, 0)
    for mode in ("0", "1"):
        monkeypatch.setenv("QFS_CHAIN_GRID", mode)
        eng = Engine(p, 0)
        try:
            g, fed = eng.stage_power(c)
            hard = np.flatnonzero(fed == 0)[: {3: 60, 5: 40, 7: 12}[p]]
            M = eng.export_matrix(c[hard]).astype(np.uint8)
            want_h, want_i = eng.heights(c[hard], 10)
            for steps in (1, 2, 3, 9):
                h1, i1, tr = eng.stage_matvec_chain(M, g[hard], steps, trace=True)
                h0, i0 = eng.stage_matvec_chain(M, g[hard], steps)
                assert np.array_equal(h0, h1) and np.array_equal(i0, i1), (p, mode, steps)
                for k in range(len(hard)):   # the traced vectors decide exactly as reported
                    hit = [s for s in range(int(i1[k])) if tr[k][s][eng.shape.cap] != 0]
                    assert (hit == [int(i1[k]) - 1] and int(h1[k]) == int(i1[k]) + 1) or (hit == [] and int(h1[k]) == 0 and int(i1[k]) == steps)
            assert np.array_equal(h0, want_h) and np.array_equal(i0, want_i)
        finally:
            eng.close()
