#!/usr/bin/env python3
"""Developer helper: CUDA-event stage times of qfs_heights on the seeded benchmark batch (one line per prime)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_12428_b200.engine import get_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, nargs="+", default=[5, 7])
ap.add_argument("--batch", type=int, default=100000)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--free", action="store_true", help="matrix-free mode (qfs_heights_free)")
a = ap.parse_args()
for p in a.p:
    c = bench.cached_block(p, a.batch, 0, 0)
    eng = get_engine(p, 0)
    acc = {}
    for i in range(3 + a.reps):
        hs, its = eng.heights(c, 10, matrix_free=a.free)
        if i >= 3:
            for k, v in eng.stats().items():
                if k.startswith("ms_"):
                    acc[k] = acc.get(k, 0.0) + v / a.reps
    print(f"p={p} B={a.batch} hard={eng.stats()['hard']} " + " ".join(f"{k[3:]}={v:.3f}" for k, v in acc.items()),
          "hist", np.bincount(hs.astype(np.int64)).tolist(), flush=True)
