#!/usr/bin/env python3
"""Developer helper: latency of ONE surface (and of small batches) through Engine.heights with host buffers, per stage."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_12428_b200.engine import get_engine  # noqa: E402

for p in [int(x) for x in (sys.argv[1:] or ["5", "7", "11"])]:
    c = bench.cached_block(p, 20000 if p < 11 else 4000, 0, 0)
    eng = get_engine(p, 0)
    hs, its = eng.heights(c, 10)
    i = int(np.argmax(its))
    hard = np.nonzero(hs != 1)[0]
    for label, rows in (("1 surface", c[i:i + 1]), ("4 hard", c[hard[:4]]), ("64 hard", c[hard[:64]])):
        ts = []
        for k in range(43):
            t0 = time.perf_counter()
            eng.heights(np.ascontiguousarray(rows), 10)
            if k >= 3:
                ts.append(time.perf_counter() - t0)
        st = eng.stats()
        print(f"p={p} {label}: {1e3 * float(np.median(ts)):.3f} ms per call; stages " +
              " ".join(f"{k[3:]}={v:.3f}" for k, v in st.items() if k.startswith("ms_")), flush=True)
