#!/usr/bin/env python3
"""Developer helper: chain-stage time (CUDA events) of k_chain vs k_chain_grid vs the automatic choice, by prime and batch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2502_12428_b200.engine import Engine  # noqa: E402

for p, batches in ((5, (1, 30, 300, 3000, 30000)), (7, (1, 50, 500, 5000, 50000)), (11, (1, 100, 1000, 5000))):
    block = bench.cached_block(p, 100000, 0, 0)
    hard1 = block[np.nonzero(np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", f"heights_p{p}_seed0_w0_10000.npz"))["heights"] > 2)[0][:1]] if p < 11 else None
    for B in batches:
        c = block[:B] if (B > 1 or hard1 is None) else hard1
        row = []
        for mode in ("0", "1", None):
            if mode is None:
                os.environ.pop("QFS_CHAIN_GRID", None)
            else:
                os.environ["QFS_CHAIN_GRID"] = mode
            eng = Engine(p, 0)
            ts = []
            for i in range(6):
                hs, its = eng.heights(c, 10)
                if i >= 2:
                    ts.append(eng.stats()["ms_matvec"])
            row.append(float(np.median(ts)))
            eng.close()
        print(f"p={p} B={B} hard={int((hs != 1).sum())} beyond2={int(((hs > 2) | (hs == 0)).sum())}  k_chain {row[0]:.4f} ms  k_chain_grid {row[1]:.4f} ms  auto {row[2]:.4f} ms", flush=True)
