#!/usr/bin/env python3
"""Golden heights of Calabi-Yau hypersurfaces in n != 3, 4 variables (degree n forms) from the UNMODIFIED reference:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_forms.py

n = 2 (binary quadratics: two points on the line), n = 5 (quintic threefolds) and n = 6 at toy primes: seeded random forms
(coefficient vectors over MonomialBasis(n, n), lex-ascending, x1 most significant) with height and iteration count from the
reference's height_matrix (and height_naive where it is fast enough; they must agree: tests/test_acceptance.py:128-138), at a few
bounds; plus the Fermat forms.  Writes tests/golden/forms.json.   (height.py:63-144 accept any n >= 2.)
"""
import json
import math
import os
import time

import numpy as np
from qfsplit import MonomialBasis, SparsePoly, SurfaceProblem, height_matrix, height_naive

HERE = os.path.dirname(os.path.abspath(__file__))


def io(h):
    return 0 if (isinstance(h, float) and math.isinf(h)) else int(h)


def tuples(n):
    b = MonomialBasis(n, n)
    return [tuple(int(x) for x in b.tuple_at(i)) for i in range(len(b))]


out = {"sets": []}
PLAN = [(2, 3, 40, (6, 2, 1), True), (2, 5, 60, (6, 2, 1), True), (2, 7, 60, (6, 2, 1), True), (2, 11, 40, (6, 2, 1), True),
        (2, 13, 30, (6, 1), True), (5, 3, 24, (4, 2, 1), True), (6, 3, 4, (3, 1), False), (5, 5, 3, (3,), False)]
for n, p, count, bounds, naive in PLAN:
    T = tuples(n)
    rng = np.random.default_rng([44, n, p])
    rows = []
    t0 = time.time()
    for _ in range(count):
        vec = rng.integers(0, p, size=len(T))
        if not vec.any():
            continue
        f = SparsePoly.from_terms(n, {T[i]: int(c) for i, c in enumerate(vec) if c}, modulus=p)
        res = {}
        for bound in bounds:
            prob = SurfaceProblem(p, n, f, bound=bound)
            a = height_matrix(prob)
            if naive:
                b = height_naive(prob)
                assert a == b, (n, p, vec, a, b)
            res[str(bound)] = [io(a.height), a.iterations]
        rows.append({"coeffs": [int(v) for v in vec], "results": res})
    # the Fermat form x1^n + ... + xn^n
    vec = [1 if sorted(t) == [0] * (n - 1) + [n] else 0 for t in T]
    f = SparsePoly.from_terms(n, {T[i]: 1 for i, c in enumerate(vec) if c}, modulus=p)
    r = height_matrix(SurfaceProblem(p, n, f, bound=bounds[0]))
    rows.append({"coeffs": vec, "results": {str(bounds[0]): [io(r.height), r.iterations]}, "fermat": True})
    out["sets"].append({"n": n, "p": p, "tuples": T, "rows": rows})
    print(n, p, len(rows), sorted({r["results"][str(bounds[0])][0] for r in rows}), "%.0f s" % (time.time() - t0), flush=True)
    with open(os.path.join(HERE, "forms.json"), "w") as fh:
        json.dump(out, fh)
