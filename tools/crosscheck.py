#!/usr/bin/env python3
"""Large-scale cross-check on the GPU: the matrix path (qfs_heights: Delta, operator matrix in HBM, streamed matvec chain)
against the matrix-free polynomial iteration (qfs_heights_free) on seeded random quartics -- two different algorithms that
must agree on every height and every iteration count.  With --literal N the first N surfaces of every block also go
through the literal route (qfs_literal_heights: dense powers, checked division, splitting operator; none of the engine's
identities), p <= 7.

    python tools/crosscheck.py --p 5 --count 10000000 [--block 1000000] [--seed 1] [--literal 100000] [--lazy]

--lazy replaces the matrix-free arm by the lazy operator-matrix mode (qfs_heights_lazy: the cap row of the first step decides
before Delta and M are built), again on every height and every iteration count.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_12428_b200 as q  # noqa: E402
from paper_2502_12428_b200.engine import get_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--p", type=int, default=5)
ap.add_argument("--count", type=int, default=10000000)
ap.add_argument("--block", type=int, default=1000000)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--literal", type=int, default=0, help="surfaces per block that also go through the literal route")
ap.add_argument("--lazy", action="store_true", help="second arm = qfs_heights_lazy instead of qfs_heights_free")
a = ap.parse_args()
eng = get_engine(a.p, 0)
hist = np.zeros(12, dtype=np.int64)
mism = 0
lit_done = lit_mism = 0
t_m = t_f = t_l = 0.0
done = 0
w = 0
while done < a.count:
    n = min(a.block, a.count - done)
    import torch
    c = torch.empty((n, 35), dtype=torch.uint8, device="cuda:0")
    _, clean = eng.sample(a.seed, w, n, out=c)          # the reference's seeded stream, drawn on the device
    if not clean:
        c = torch.from_numpy(q.sample_block(a.p, n, a.seed, w)).cuda()
    t0 = time.perf_counter(); hm, im = eng.heights(c, 10); torch.cuda.synchronize(); t1 = time.perf_counter()
    hf, jf = eng.heights(c, 10, matrix_free=not a.lazy, lazy=a.lazy); torch.cuda.synchronize(); t2 = time.perf_counter()
    t_m += t1 - t0; t_f += t2 - t1
    hm, im, hf, jf = (x.cpu().numpy() for x in (hm, im, hf, jf))
    mism += int((hm != hf).sum() + (im != jf).sum())
    if a.literal:
        k = min(a.literal, n)
        t3 = time.perf_counter()
        lh, li = q.literal_heights(a.p, c[:k].cpu().numpy(), 10)
        t_l += time.perf_counter() - t3
        lit_mism += int((lh != hm[:k]).sum() + (li != im[:k]).sum())
        lit_done += k
    hist += np.bincount(hm.astype(np.int64), minlength=12)[:12]
    done += n; w += 1
print(json.dumps({"p": a.p, "surfaces": done, "seed": a.seed, "mismatches": mism,
                  "histogram": {("inf" if h == 0 else str(h)): int(v) for h, v in enumerate(hist) if v},
                  "matrix_path_s": round(t_m, 2), ("lazy_matrix_s" if a.lazy else "matrix_free_s"): round(t_f, 2),
                  "literal": {"surfaces": lit_done, "mismatches": lit_mism, "s": round(t_l, 2)}}))
sys.exit(1 if mism or lit_mism else 0)
