#!/usr/bin/env python3
"""Small run for compute-sanitizer: every kernel of the pipeline, the stage taps and the export, for a few primes.

    compute-sanitizer --tool memcheck  python tools/sanitize_run.py
    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_12428_b200 as q  # noqa: E402
from paper_2502_12428_b200.engine import get_engine  # noqa: E402

primes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [3, 5, 7]
for p in primes:
    eng = get_engine(p, 0)
    n = {3: 200, 5: 150, 7: 60}.get(p, 14)
    c = q.sample_block(p, n, 7, 0)
    hs, its = eng.heights(c, 10)
    d = eng.stage_delta(c[:3])
    m = eng.export_matrix(c[:2])
    hf, itf = eng.heights(c, 10, matrix_free=True)
    assert np.array_equal(hs, hf) and np.array_equal(its, itf)
    hl, itl = eng.heights(c, 10, lazy=True)   # k_caprow + the second compaction (qfs_caprow.cuh)
    assert np.array_equal(hs, hl) and np.array_equal(its, itl)
    if p <= 7:   # the literal route (qfs_literal.cuh)
        k = {3: 200, 5: 40, 7: 3}[p]
        lh, li, lg, ld = q.literal_heights(p, c[:k], 10, want_g=True, want_delta=True)
        assert np.array_equal(lh, hs[:k]) and np.array_equal(li, its[:k]) and np.array_equal(ld[:3], d)
    print(p, np.bincount(hs.astype(np.int64)).tolist(), d.shape, m.shape, flush=True)
rng = np.random.default_rng(5)
for p in (3, 5, 13):
    hs, its = q.cubic_height_batch(p, rng.integers(1, p, size=(40, 10)).astype(np.uint8), 5)
    print("cubic", p, np.bincount(hs.astype(np.int64)).tolist(), flush=True)
for n, p in ((2, 5), (5, 3), (6, 3)):
    from paper_2502_12428_b200.forms import exponents
    hs, its = q.form_height_batch(p, n, rng.integers(1, p, size=(6, len(exponents(n)))).astype(np.uint8), 3)
    print("form", n, p, np.bincount(hs.astype(np.int64)).tolist(), flush=True)
got, clean = get_engine(5, 0).sample(1, 2, 5000)
assert clean and np.array_equal(got, q.sample_block(5, 5000, 1, 2))
print("sampler ok", flush=True)
if os.environ.get("QFS_DELTA_DIRECT"):
    print("k_delta_direct was used for Delta")
