"""The lazy operator-matrix mode (qfs_heights_lazy, csrc/qfs_caprow.cuh): the cap row of the first step decides before
Delta and M are built.  It must return the heights AND iteration counts of the reference (height.py:119-144) and of the eager
matrix path on the same inputs, for every bound, and build M for about 1/p of the hard surfaces only."""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_lazy_mode_equals_the_reference_heights():
    import paper_2502_12428_b200 as q
    for p, name in ((3, "heights_p3_seed0_w0_3000.npz"), (5, "heights_p5_seed0_w0_10000.npz"), (7, "heights_p7_seed0_w0_10000.npz")):
        z = np.load(os.path.join(GOLDEN, name))
        hs, its = q.height_batch(p, z["coeffs"], 10, method="lazy")
        assert np.array_equal(hs.astype(np.int64), z["heights"].astype(np.int64))
        assert np.array_equal(its.astype(np.int64), z["iters"].astype(np.int64))


def test_lazy_mode_equals_the_matrix_path_and_builds_fewer_matrices():
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    for p, count in ((3, 5000), (5, 60000), (7, 20000), (11, 1500), (13, 400)):
        c = q.sample_block(p, count, 17, 3)
        eng = get_engine(p, 0)
        h0, i0 = eng.heights(c, 10)
        st0 = eng.stats()
        h1, i1 = eng.heights(c, 10, lazy=True)
        st1 = eng.stats()
        assert np.array_equal(h0, h1) and np.array_equal(i0, i1), p
        assert st0["hard"] == st1["hard"] == int((h0 != 1).sum())
        assert st0["built"] == st0["hard"]
        # M is built exactly for the surfaces the first step leaves undecided: every height but 1 and 2
        assert st1["built"] == int(((h0 != 1) & (h0 != 2)).sum()), p
        assert st1["matvec_steps"] == st0["matvec_steps"] == int(i0.astype(np.int64).sum())


def test_lazy_mode_bounds_and_fixtures():
    import paper_2502_12428_b200 as q
    verdicts = q.verify_fixtures(open(q.fixtures_path()).read(), method="lazy")
    assert len(verdicts) == 32 and all(v.ok for v in verdicts)
    c = q.sample_block(5, 4000, 3, 1)
    for bound in (1, 2, 3, 4, 10):
        h0, i0 = q.height_batch(5, c, bound)
        h1, i1 = q.height_batch(5, c, bound, method="lazy")
        assert np.array_equal(h0, h1) and np.array_equal(i0, i1), bound
    # a batch in which the cap row decides every hard surface (no chunk loop at all), and one with a single surface
    h0, _ = q.height_batch(5, c, 10)
    easy = c[(h0 == 1) | (h0 == 2)]
    h1, i1 = q.height_batch(5, easy, 10, method="lazy")
    assert set(np.unique(h1)) <= {1, 2} and np.array_equal(i1, (h1 == 2).astype(np.int8))
    dwork5 = q.parse_poly("x1^4+x2^4+x3^4+x4^4+x1*x2*x3*x4", 4, 5)
    hs, its = q.height_batch(5, np.asarray(dwork5.coeffs, dtype=np.uint8).reshape(1, 35), 10, method="lazy")
    assert int(hs[0]) == 0 and int(its[0]) == 9


def test_lazy_mode_through_the_search_driver():
    from paper_2502_12428_b200 import search
    a = search.device_block(7, 3000, 0, 2, 0, 10, "matrix")
    b = search.device_block(7, 3000, 0, 2, 0, 10, "lazy")
    assert np.array_equal(np.asarray(a[1]), np.asarray(b[1]))


def test_lazy_mode_with_chunked_filter_and_chunked_pipeline():
    """qfs_set_chunk cuts both the cap-row pass and the pipeline behind it into chunks of that many surfaces."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    for p, count, chunk in ((5, 30000, 257), (7, 8000, 61), (11, 1200, 5)):
        c = q.sample_block(p, count, 23, 1)
        eng = get_engine(p, 0)
        h0, i0 = eng.heights(c, 10)
        eng.set_chunk(chunk)
        try:
            h1, i1 = eng.heights(c, 10, lazy=True)
            st = eng.stats()
        finally:
            eng.set_chunk(0)
        assert np.array_equal(h0, h1) and np.array_equal(i0, i1), p
        assert st["chunks"] == -(-st["built"] // ((chunk + 3) // 4 * 4)) or st["chunks"] == -(-st["built"] // chunk), (p, st)


def test_lazy_mode_kept_rows_equal_recomputed_rows_and_survive_poisoned_workspaces():
    """One chunk: the pending surfaces keep the g, h, A, E of the cap-row pass (k_gather_rows); QFS_LAZY_RECOMPUTE=1 runs
    k_power_full on them again instead.  Both must agree with the eager path, also on workspaces filled with garbage."""
    import paper_2502_12428_b200 as q
    from paper_2502_12428_b200.engine import get_engine
    for p, count in ((3, 2001), (5, 20003), (7, 5002), (11, 801)):
        c = q.sample_block(p, count, 29, 2)
        eng = get_engine(p, 0)
        h0, i0 = eng.heights(c, 10)
        for byte in (0x00, 0xFF, 0x5A):
            eng.debug_fill_workspaces(byte)
            h1, i1 = eng.heights(c, 10, lazy=True)
            assert np.array_equal(h0, h1) and np.array_equal(i0, i1), (p, byte)
        os.environ["QFS_LAZY_RECOMPUTE"] = "1"
        try:
            eng.debug_fill_workspaces(0xA5)
            h2, i2 = eng.heights(c, 10, lazy=True)
        finally:
            del os.environ["QFS_LAZY_RECOMPUTE"]
        assert np.array_equal(h0, h2) and np.array_equal(i0, i2), p
