"""Plane cubic curves (n = 3): host-side form class on CPU, kernel against the reference's own
results on GPU (tests/golden/cubics.json, produced by tests/golden/make_golden_cubics.py with the unmodified reference:
both of its drivers, three bounds, seven primes, including singular cubics of infinite height)."""
import json
import math
import os

import numpy as np
import pytest

import paper_2502_12428_b200 as q

GOLD = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cubics.json")))


def test_cubic_form_and_basis_order():
    from paper_2502_12428_b200.cubic import EXPONENTS3
    assert [list(t) for t in EXPONENTS3] == GOLD["tuples"]          # MonomialBasis(3,3) of the reference
    f = q.parse_poly("x1^3 + x2^3 + x3^3 + 2*x1*x2*x3", 3, 5)
    assert isinstance(f, q.Cubic) and f.nvars == 3 and f.degree == 3 and f.is_homogeneous() and not f.is_zero
    assert f.coeffs.tolist() == [1, 0, 0, 1, 0, 2, 0, 0, 0, 1]
    assert f.coefficient((1, 1, 1)) == 2 and len(f) == 4
    assert q.parse_poly("1:3,0,0; 2:1,1,1", 3, 7) == q.Cubic.from_terms([((3, 0, 0), 1), ((1, 1, 1), 2)], 7)
    with pytest.raises(q.DomainError):
        q.parse_poly("x1^4 + x2^3*x3", 3, 5)        # not of degree 3
    with pytest.raises(q.ParseError):
        q.parse_poly("x1^3 + x4^3", 3, 5)
    prob = q.SurfaceProblem(5, 3, f, bound=5)
    assert prob.bound == 5
    with pytest.raises(q.DomainError):
        q.SurfaceProblem(5, 3, f)                    # no default bound for n != 4 (height.py:31-39)
    with pytest.raises(q.DomainError):
        q.SurfaceProblem(5, 4, f)                    # variable count mismatch
    for bad in ((4, 5), (59, 5), (5, 0), (5, 200)):
        with pytest.raises(q.DomainError):
            q.cubic_height_batch(bad[0], np.ones((2, 10), np.uint8), bad[1])
    with pytest.raises(q.DomainError):
        q.cubic_height_batch(5, np.zeros((2, 10), np.uint8), 5)     # zero form
    with pytest.raises(q.DomainError):
        q.cubic_height_batch(5, np.full((2, 10), 5, np.uint8), 5)   # residue out of range


@pytest.mark.gpu
@pytest.mark.parametrize("gset", GOLD["sets"], ids=lambda s: f"p{s['p']}")
def test_cubic_heights_equal_the_reference(gset):
    p = gset["p"]
    coeffs = np.array([r["coeffs"] for r in gset["rows"]], dtype=np.uint8)
    for bound in (5, 2, 1):
        hs, its = q.cubic_height_batch(p, coeffs, bound)
        want = np.array([r["results"][str(bound)] for r in gset["rows"]])
        assert np.array_equal(hs.astype(np.int64), want[:, 0]), f"heights differ at p={p} bound={bound}"
        assert np.array_equal(its.astype(np.int64), want[:, 1]), f"iterations differ at p={p} bound={bound}"


@pytest.mark.gpu
def test_fermat_cubics_and_drivers():
    """tests/test_height.py:131-140 of the reference: x^3+y^3+z^3 is supersingular exactly when p = 2 mod 3."""
    for row in GOLD["fermat"]:
        p = row["p"]
        f = q.Cubic(row["coeffs"], p)
        assert f == q.parse_poly("x1^3+x2^3+x3^3", 3, p)
        prob = q.SurfaceProblem(p, 3, f, bound=5)
        want = q.HeightResult(math.inf if row["height"] == 0 else row["height"], 5, row["iterations"])
        assert q.height_matrix(prob) == want and q.height_naive(prob) == want
        assert want.height == (2 if p % 3 == 2 else 1)
    from paper_2502_12428_b200.cli import main
    assert main(["height", "--p", "5", "--poly", "x1^3+x2^3+x3^3", "--bound", "5"]) == 0
    assert main(["height", "--p", "5", "--poly", "x1^3+x2^3+x3^3"]) == 3      # no default bound for n = 3
