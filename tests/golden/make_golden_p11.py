#!/usr/bin/env python3
"""F_11 (and, with GOLDEN_P=13, F_13) stage goldens from the UNMODIFIED reference package (qfsplit): minutes and GBs per surface.

Run in the authoring container only (the GPU box has no /root/reference):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_p11.py [jobs]

Surfaces: the five published F_11 rows (k3_tables.txt) and the first four height >= 2 samples of the
reference's seeded stream default_rng([0, 0]) (search.py:92-103).  Per surface, all from reference
functions (height.py:119-144): the coefficient vector, dense g = f^10, sha256 of the dense Delta_1(g)
(lex order of basis(440, 4), one byte per entry), every 997th entry of it, sha256 of M.entries as
bytes (12341 x 12341, row-major, one byte per entry), five rows of M, the whole matvec trace, height
and iteration count.  One process per surface (the NTT plan of delta1 holds a few GB).
"""
import hashlib
import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from make_golden import coeff_vector, dense_of  # noqa: E402

P = int(os.environ.get("GOLDEN_P", "11"))          # 11 (default) or 13: GOLDEN_P=13 python tests/golden/make_golden_p11.py 2
NN = math.comb(4 * (P - 1) + 3, 3)                # 12341 / 20825
ROWS = (0, 1, NN // 3, NN // 2, NN - 1)
STRIDE = 997
NSEED = 4 if P == 11 else 2                       # seeded hard surfaces beside the published rows


def _one(job):
    tag, coeffs = job
    from qfsplit import (DenseVector, MonomialBasis, SurfaceProblem, build_mts, delta1, from_dense,
                         height_matrix, matvec, power_mod_p, to_dense)
    t0 = time.time()
    f = from_dense(DenseVector(MonomialBasis(4, 4), np.asarray(coeffs, dtype=np.uint64)), P)
    d = 4 * (P - 1)
    g = power_mod_p(f, P - 1)
    rec = {"coeffs": np.asarray(coeffs, dtype=np.uint8), "g": dense_of(g, d)}
    dl = delta1(g)
    dd = dense_of(dl, P * d)
    rec["delta_sha"] = np.frombuffer(hashlib.sha256(dd.tobytes()).digest(), dtype=np.uint8)
    rec["delta_every"] = dd[::STRIDE].copy()
    rec["delta_nnz"] = np.int64(np.count_nonzero(dd))
    del dd
    m = build_mts(dl, d, P, "wics")
    del dl
    ent = np.asarray(m.entries)
    assert ent.max() < P
    m8 = ent.astype(np.uint8)
    rec["M_sha"] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(m8).tobytes()).digest(), dtype=np.uint8)
    rec["M_rows_idx"] = np.array(ROWS)
    rec["M_rows"] = m8[list(ROWS)].copy()
    del m8
    gv = to_dense(g, m.source_basis)
    cap = m.target_basis.index_of((P - 1,) * 4)
    trace, height, iters = [], 0, 0
    for h in range(2, 11):          # the loop of height.py:135-144
        gv = matvec(m, gv)
        iters += 1
        trace.append(gv.values.astype(np.uint8))
        if int(gv.values[cap]) != 0:
            height = h
            break
    rec["trace"] = np.stack(trace)
    rec["height"] = np.int64(height)
    rec["iters"] = np.int64(iters)
    rec["seconds"] = np.float64(time.time() - t0)
    np.savez_compressed(os.path.join(HERE, f"_p{P}_part_{tag}.npz"), **rec)
    print(tag, "height", height, "iters", iters, "%.0f s" % (time.time() - t0), flush=True)
    return tag


def main():
    jobs_n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    from qfsplit import fedder_survives, parse_fixtures, power_mod_p, sample_surface
    from qfsplit.search import fixtures_path
    jobs = []
    for i, r in enumerate(x for x in parse_fixtures(open(fixtures_path()).read()) if x.p == P):
        if r.expected == 1:
            continue        # decided by the Fedder test: no Delta, no M
        jobs.append((f"fix{i}_h{int(r.expected)}", coeff_vector(r.f).tolist()))
    rng = np.random.default_rng([0, 0])
    k = 0
    idx = 0
    while k < NSEED:
        f = sample_surface(rng, P)
        if not fedder_survives(power_mod_p(f, P - 1)):
            jobs.append((f"seed0_i{idx}", coeff_vector(f).tolist()))
            k += 1
        idx += 1
    todo = [j for j in jobs if not os.path.exists(os.path.join(HERE, f"_p{P}_part_{j[0]}.npz"))]
    print("jobs", [j[0] for j in jobs], "todo", len(todo), flush=True)
    with ProcessPoolExecutor(max_workers=jobs_n) as pool:
        list(pool.map(_one, todo))
    flat = {"p": np.int64(P), "count": np.int64(len(jobs)), "tags": np.array([j[0] for j in jobs])}
    for i, (tag, _) in enumerate(jobs):
        part = np.load(os.path.join(HERE, f"_p{P}_part_{tag}.npz"))
        for key in part.files:
            flat[f"s{i}_{key}"] = part[key]
    np.savez_compressed(os.path.join(HERE, f"stages_p{P}.npz"), **flat)
    print(f"stages_p{P}.npz", len(jobs), "surfaces")


if __name__ == "__main__":
    main()
