#!/usr/bin/env python3
"""Generate golden fixtures from the UNMODIFIED reference package (qfsplit).

Run in the authoring container only (the GPU box has no /root/reference):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [what ...]

`what` is any of: basis, fixtures, stages3, stages5, stages7, heights3,
heights5, heights7, fixtures11 (default: everything except fixtures11).

Everything written here is *output of the reference itself* on seeded inputs;
nothing is copied from its sources.  Dense layouts follow SURVEY.md section 8:
lex-ascending monomial order with x1 most significant, index 0 = x4^d.
Heights are stored as int8 with 0 meaning "infinity" (no finite height <= bound).
"""
import hashlib
import json
import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import qfsplit  # noqa: E402  (the reference)
from qfsplit import (  # noqa: E402
    MonomialBasis, SurfaceProblem, build_mts, delta1, height_matrix,
    parse_fixtures, power_mod_p, sample_surface, to_dense, matvec,
)
from qfsplit.search import fixtures_path  # noqa: E402


def comb3(n):
    return n * (n - 1) * (n - 2) // 6 if n >= 3 else 0


def comb2(n):
    return n * (n - 1) // 2 if n >= 2 else 0


def rank4(a, d):
    a1, a2, a3, _ = a
    d2 = d - a1
    return comb3(d + 3) - comb3(d - a1 + 3) + comb2(d2 + 2) - comb2(d2 - a2 + 2) + a3


def coeff_vector(f):
    """35-vector (uint8) of a reference SparsePoly quartic in lex-ascending basis order."""
    bas = MonomialBasis(4, 4)
    return to_dense(f, bas).values.astype(np.uint8)


def dense_of(poly, degree):
    """Dense uint8 vector of a reference SparsePoly over basis(degree, 4), lex ascending."""
    n = math.comb(degree + 3, 3)
    out = np.zeros(n, dtype=np.uint8)
    ex = poly.packing.unpack_rows(poly.words)
    for e, c in zip(ex.tolist(), poly.coeffs.tolist()):
        assert sum(e) == degree
        out[rank4(e, degree)] = c
    return out


def stage_dump(p, f, bound=10):
    """All intermediates of height_matrix for one surface, from reference functions."""
    g = power_mod_p(f, p - 1)
    d = 4 * (p - 1)
    rec = {"coeffs": coeff_vector(f), "g": dense_of(g, d)}
    res = height_matrix(SurfaceProblem(p, 4, f, bound))
    rec["height"] = 0 if not res.is_finite else res.height
    rec["iters"] = res.iterations
    if res.height == 1:
        return rec
    dl = delta1(g)
    rec["delta"] = dense_of(dl, p * d)
    m = build_mts(dl, d, p, "wics")
    rec["M"] = np.asarray(m.entries, dtype=np.uint8)
    gv = to_dense(g, m.source_basis)
    trace = []
    for _ in range(res.iterations):
        gv = matvec(m, gv)
        trace.append(gv.values.astype(np.uint8))
    rec["trace"] = np.stack(trace)
    return rec


def do_basis():
    out = {}
    for d in (4, 8, 12):
        b = MonomialBasis(d, 4)
        tup = [list(b.tuple_at(i)) for i in range(len(b))]
        for i, t in enumerate(tup):
            assert rank4(t, d) == i
        out[str(d)] = tup
    caps = {}
    for p in (3, 5, 7, 11, 13):
        d = 4 * (p - 1)
        caps[str(p)] = {"N": math.comb(d + 3, 3), "cap": rank4((p - 1,) * 4, d)}
    out["caps"] = caps
    with open(os.path.join(HERE, "basis.json"), "w") as fh:
        json.dump(out, fh)
    print("basis ok", caps)


def do_fixtures():
    rows = parse_fixtures(open(fixtures_path()).read())
    out = []
    for r in rows:
        out.append({
            "p": r.p,
            "height": 0 if (isinstance(r.expected, float)) else int(r.expected),
            "coeffs": coeff_vector(r.f).tolist(),
            "text": r.text,
        })
    with open(os.path.join(HERE, "k3_fixture_vectors.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print("fixtures", len(out))


def _stages(p, want_hard, seed, keep_matrix):
    rng = np.random.default_rng([seed, 0])
    recs = []
    hard = 0
    easy = 0
    while hard < want_hard:
        f = sample_surface(rng, p)
        rec = stage_dump(p, f)
        if rec["height"] == 1:
            if easy < 2:
                recs.append(rec)
                easy += 1
            continue
        hard += 1
        recs.append(rec)
    flat = {"p": np.int64(p), "count": np.int64(len(recs))}
    for i, rec in enumerate(recs):
        for k, v in rec.items():
            if k == "M":
                flat[f"s{i}_Msha"] = np.frombuffer(
                    hashlib.sha256(np.ascontiguousarray(v).tobytes()).digest(), dtype=np.uint8)
                if keep_matrix(i):
                    flat[f"s{i}_M"] = v
                else:
                    rows = np.array([0, 1, v.shape[0] // 3, v.shape[0] // 2, v.shape[0] - 1])
                    flat[f"s{i}_Mrows_idx"] = rows
                    flat[f"s{i}_Mrows"] = v[rows]
            else:
                flat[f"s{i}_{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, f"stages_p{p}.npz"), **flat)
    print("stages", p, len(recs), [r["height"] for r in recs])


def do_stages3():
    _stages(3, 6, 11, lambda i: True)


def do_stages5():
    _stages(5, 3, 0, lambda i: i < 4)


def do_stages7():
    _stages(7, 2, 0, lambda i: False)


def _height_chunk(args):
    p, coeffs = args
    bas = MonomialBasis(4, 4)
    from qfsplit import DenseVector, from_dense
    hs = np.zeros(len(coeffs), dtype=np.int8)
    its = np.zeros(len(coeffs), dtype=np.int8)
    for i, c in enumerate(coeffs):
        f = from_dense(DenseVector(bas, c.astype(np.uint64)), p)
        res = height_matrix(SurfaceProblem(p, 4, f, 10))
        hs[i] = res.height if res.is_finite else 0
        its[i] = res.iterations
    return hs, its


def _heights(p, count, seed=0, worker=0, chunk=25):
    rng = np.random.default_rng([seed, worker])
    coeffs = np.stack([coeff_vector(sample_surface(rng, p)) for _ in range(count)])
    t0 = time.time()
    jobs = [(p, coeffs[i:i + chunk]) for i in range(0, count, chunk)]
    with ProcessPoolExecutor(max_workers=int(os.environ.get("GOLDEN_JOBS", "6"))) as pool:
        parts = list(pool.map(_height_chunk, jobs))
    hs = np.concatenate([a for a, _ in parts])
    its = np.concatenate([b for _, b in parts])
    np.savez_compressed(os.path.join(HERE, f"heights_p{p}_seed{seed}_w{worker}_{count}.npz"),
                        p=np.int64(p), seed=np.int64(seed), worker=np.int64(worker),
                        coeffs=coeffs, heights=hs, iters=its)
    print("heights", p, count, "hist", np.bincount(hs.astype(np.int64)), "%.0fs" % (time.time() - t0))


def do_heights3():
    _heights(3, 3000)


def do_heights5():
    _heights(5, 10000)


def do_heights7():
    """The F_7 counterpart of the north star's 10k-surface seeded set (38 minutes on 7 cores: ~11 s per hard surface)."""
    _heights(7, 10000)


def do_fixtures11():
    """Recompute the F_11 published rows with the reference (slow, GBs of RAM)."""
    rows = [r for r in parse_fixtures(open(fixtures_path()).read()) if r.p == 11]
    out = []
    for r in rows:
        t0 = time.time()
        res = height_matrix(SurfaceProblem(11, 4, r.f, 10))
        out.append({"p": 11, "expected": int(r.expected),
                    "got": res.height if res.is_finite else 0,
                    "iters": res.iterations, "coeffs": coeff_vector(r.f).tolist(),
                    "seconds": time.time() - t0})
        print(out[-1]["expected"], out[-1]["got"], out[-1]["seconds"])
    with open(os.path.join(HERE, "ref_run_p11.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    what = sys.argv[1:] or ["basis", "fixtures", "stages3", "stages5", "stages7",
                            "heights3", "heights5", "heights7"]
    for w in what:
        globals()["do_" + w]()
