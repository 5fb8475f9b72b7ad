#!/usr/bin/env python3
"""Tiny driver for ncu: `calls` qfs_heights invocations on one seeded batch (no torch needed)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_12428_b200.engine import get_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=5)
ap.add_argument("--batch", type=int, default=20000)
ap.add_argument("--calls", type=int, default=2)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--lazy", action="store_true", help="qfs_heights_lazy (k_caprow before Delta and M)")
a = ap.parse_args()
c = bench.cached_block(a.p, 100000, 0, 0)[: a.batch]
eng = get_engine(a.p, 0)
if a.chunk:
    eng.set_chunk(a.chunk)
for _ in range(a.calls):
    hs, its = eng.heights(c, 10, lazy=a.lazy)
    print(eng.stats())
