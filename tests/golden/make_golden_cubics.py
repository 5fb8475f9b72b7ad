#!/usr/bin/env python3
"""Golden heights of plane cubic curves (n = 3) from the UNMODIFIED reference:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_cubics.py

For p in 3, 5, 7, 11, 13 (and a few larger primes): seeded random cubics (coefficient vectors over
MonomialBasis(3,3), index 0 = x3^3 ... 9 = x1^3) with height and iterations from BOTH reference drivers
(height_matrix, height_naive; they must agree), at bound 5 and at bound 1/2; plus the Fermat cubics of
tests/test_height.py:131-140.  Writes tests/golden/cubics.json.
"""
import json
import math
import os

import numpy as np
from qfsplit import MonomialBasis, SparsePoly, SurfaceProblem, height_matrix, height_naive

HERE = os.path.dirname(os.path.abspath(__file__))
B3 = MonomialBasis(3, 3)
TUPLES = [tuple(B3.tuple_at(i).exponents) if hasattr(B3.tuple_at(i), "exponents") else tuple(B3.tuple_at(i)) for i in range(len(B3))]


def io(h):
    return 0 if (isinstance(h, float) and math.isinf(h)) else int(h)


def poly(vec, p):
    return SparsePoly.from_terms(3, {TUPLES[i]: int(c) for i, c in enumerate(vec) if c}, modulus=p)


out = {"tuples": TUPLES, "sets": []}
for p, count in ((3, 150), (5, 150), (7, 120), (11, 60), (13, 40), (17, 12), (23, 6)):
    rng = np.random.default_rng([33, p])
    rows = []
    for _ in range(count):
        vec = rng.integers(0, p, size=10)
        if not vec.any():
            continue
        f = poly(vec, p)
        res = {}
        for bound in (5, 2, 1):
            prob = SurfaceProblem(p, 3, f, bound=bound)
            a = height_matrix(prob)
            if p <= 7 or bound == 5:
                b = height_naive(prob)
                assert a == b, (p, vec, a, b)
            res[str(bound)] = [io(a.height), a.iterations]
        rows.append({"coeffs": [int(v) for v in vec], "results": res})
    out["sets"].append({"p": p, "rows": rows})
    print(p, len(rows), sorted({r["results"]["5"][0] for r in rows}))
fer = []
for p in (5, 7, 11, 13):
    vec = [0] * 10
    for i, t in enumerate(TUPLES):
        if sorted(t) == [0, 0, 3]:
            vec[i] = 1
    r = height_matrix(SurfaceProblem(p, 3, poly(vec, p), bound=5))
    fer.append({"p": p, "coeffs": vec, "height": io(r.height), "iterations": r.iterations})
out["fermat"] = fer
with open(os.path.join(HERE, "cubics.json"), "w") as fh:
    json.dump(out, fh)
print("fermat", [(f["p"], f["height"]) for f in fer])
