#!/usr/bin/env python3
"""Rate of the UNMODIFIED reference (qfsplit.height_matrix) on the authoring container's cores, on the benchmark's seeded stream.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tools/measure_reference.py

The reference is pure Python + numba and does not travel to the GPU box; its rate is measured here and committed
(profiles/reference_python_rate.json), bench.py quotes it beside the C port it times on the box."""
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def chunk(args):
    p, rows = args
    from qfsplit import DenseVector, MonomialBasis, SurfaceProblem, from_dense, height_matrix
    bas = MonomialBasis(4, 4)
    t0 = time.perf_counter()
    hs = []
    for c in rows:
        f = from_dense(DenseVector(bas, np.asarray(c, dtype=np.uint64)), p)
        r = height_matrix(SurfaceProblem(p, 4, f, 10))
        hs.append(r.height if r.is_finite else 0)
    return hs, time.perf_counter() - t0


def main():
    from paper_2502_12428_b200.search import sample_block
    cores = os.cpu_count()
    out = {"cores": cores, "what": "qfsplit.height_matrix (unmodified reference, numpy + numba), first n samples of default_rng([0, 0])"}
    for p, n in ((5, 240), (7, 48)):
        rows = sample_block(p, n, 0, 0)
        parts = [(p, rows[i::cores].tolist()) for i in range(cores)]
        with ProcessPoolExecutor(max_workers=cores) as pool:
            list(pool.map(chunk, [(p, rows[:2].tolist())] * cores))       # JIT warm-up in every worker
            t0 = time.perf_counter()
            res = list(pool.map(chunk, parts))
            wall = time.perf_counter() - t0
        hs = [h for r in res for h in r[0]]
        busy = sum(r[1] for r in res)
        out[f"F_{p}"] = {"samples": n, "hard": int(sum(1 for h in hs if h != 1)), "wall_s": wall, "surfaces_per_s": n / wall,
                         "surfaces_per_s_per_core": n / busy}
        print(p, out[f"F_{p}"], flush=True)
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "reference_python_rate.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
