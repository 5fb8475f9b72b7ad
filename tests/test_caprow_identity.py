"""CPU check of the index identity the lazy mode rests on (csrc/qfs_caprow.cuh), on the REFERENCE'S OWN intermediates
(tests/golden/stages_p*.npz, produced by tests/golden/make_golden.py from qfsplit): the cap row of the operator matrix is
    M[cap, c] = Delta[(p^2 - 1) * (1,1,1,1) - c]          (M[r, c] = Delta[p r + (p-1) - c], mtsmatrix.py:249-281)
for every column c of basis(4(p-1)), and (M g)[cap] != 0 exactly for the surfaces of height 2 (height.py:135-144)."""
import os
from math import comb

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rank(deg, a1, a2, a3):
    """Index of x1^a1 x2^a2 x3^a3 x4^(deg-a1-a2-a3) in the lex-ascending dense layout (monomials.py:208-276; qfs_shape.cuh)."""
    rowbase = comb(deg + 3, 3) - comb(deg - a1 + 3, 3) + comb(deg - a1 + 2, 2) - comb(deg - a1 - a2 + 2, 2)
    return rowbase + a3


@pytest.mark.parametrize("p", [3, 5, 7])
def test_cap_row_is_a_slice_of_delta(p):
    z = np.load(os.path.join(GOLDEN, f"stages_p{p}.npz"))
    d, D = 4 * (p - 1), 4 * p * (p - 1)
    cols = [(a1, a2, a3) for a1 in range(d + 1) for a2 in range(d + 1 - a1) for a3 in range(d + 1 - a1 - a2)]
    cols.sort(key=lambda a: _rank(d, *a))
    assert [_rank(d, *a) for a in cols] == list(range(len(cols)))
    cap = _rank(d, p - 1, p - 1, p - 1)
    src = np.array([_rank(D, p * p - 1 - a1, p * p - 1 - a2, p * p - 1 - a3) for a1, a2, a3 in cols])
    seen = 0
    for i in range(int(z["count"])):
        if f"s{i}_delta" not in z.files:
            continue
        delta, g = z[f"s{i}_delta"].astype(np.int64), z[f"s{i}_g"].astype(np.int64)
        row = delta[src]
        if f"s{i}_M" in z.files:
            assert np.array_equal(row, z[f"s{i}_M"][cap].astype(np.int64)), (p, i)
        if f"s{i}_trace" in z.files and len(z[f"s{i}_trace"]):
            assert int(row @ g) % p == int(z[f"s{i}_trace"][0][cap]), (p, i)
        height = int(z[f"s{i}_height"])
        if height != 1:   # hard surface: decided by the first step iff its height is 2
            assert (int(row @ g) % p != 0) == (height == 2), (p, i, height)
            seen += 1
    assert seen >= 2
