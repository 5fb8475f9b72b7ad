#!/usr/bin/env python3
"""Developer helper: where the host time of a search block goes (search.device_block), and the driver rates."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_12428_b200 import search  # noqa: E402
from paper_2502_12428_b200.engine import get_engine  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 5
block = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
eng = get_engine(p, 0)
t_end = time.perf_counter() + 2.0          # warm up until the clocks have ramped
w = 1000
while time.perf_counter() < t_end:
    search.device_block(p, block, 0, w)
    w += 1
acc = {}
def lap(name, t0):
    t = time.perf_counter()
    acc[name] = acc.get(name, 0.0) + (t - t0)
    return t
nb = 20
for w in range(3, 3 + nb):
    t = time.perf_counter()
    dev = torch.empty((block, 35), dtype=torch.uint8, device="cuda:0")
    t = lap("alloc", t)
    _, clean = eng.sample(0, w, block, out=dev)
    t = lap("sample", t)
    hs, its = eng.heights(dev, 10)
    t = lap("heights", t)
    st = eng.stats()
    acc["gpu_ms_total"] = acc.get("gpu_ms_total", 0.0) + st["ms_total"] / 1e3
    t = time.perf_counter()
    codes = hs.cpu().numpy()
    it2 = its.cpu().numpy()
    t = lap("d2h", t)
    h = search.HeightHistogram(10)
    h.record_codes(codes)
    t = lap("hist", t)
    u = np.unique(codes)
    t = lap("unique", t)
print(f"p={p} block={block}: per block ms " + " ".join(f"{k}={1e3 * v / nb:.3f}" for k, v in acc.items()))
for method in ("matrix", "lazy", "naive"):
    t0 = time.perf_counter()
    wit, hist, nblk = search.spectrum_search(p, block=block, rng_seed=0, bound=10, max_blocks=30, want={99}, method=method)
    dt = time.perf_counter() - t0
    print(f"spectrum_search {method}: {nblk} blocks of {block} in {dt:.3f} s = {nblk * block / dt / 1e6:.2f} M samples/s")
