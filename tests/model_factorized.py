"""numpy model of the algorithm the CUDA kernels implement (NOT the oracle, NOT product).

The CUDA path does not follow the reference step by step; it uses two algebraic
identities:

  (1) Witt-carry factorisation.  With tau(a) = a^p mod p^2, f_T = sum tau(a_J) x^J,
      H = f_T^(p-2), G = f_T^(p-1), Pw = f_T^p (all mod p^2), h = H mod p, g = G mod p,
         A[I] = ((G[I] - tau(g[I])) mod p^2) / p,       E[J] = ((Pw[J] - [p|J] tau(a_{J/p})) mod p^2) / p
      one has  Delta_1(f^(p-1)) = phi(A) - phi(h) * E  (mod p),  phi: x_i -> x_i^p.
  (2) Gather form of the operator matrix:  M[r, c] = Delta[p*r + (p-1) - c]  (0 if any component < 0).

This module restates them in slow, obviously-indexed numpy so CPU-only tests can pin the
identities against the oracle/golden vectors; the GPU tests then pin the kernels.
"""
from itertools import product
from math import comb

import numpy as np


def c2(n):
    return n * (n - 1) // 2 if n >= 2 else 0


def c3(n):
    return n * (n - 1) * (n - 2) // 6 if n >= 3 else 0


def rowbase(d, a1, a2):
    return c3(d + 3) - c3(d - a1 + 3) + c2(d - a1 + 2) - c2(d - a1 - a2 + 2)


def rank(d, a):
    return rowbase(d, a[0], a[1]) + a[2]


def tuples(d):
    """basis(d,4) in lex-ascending order, x1 most significant."""
    return [(a1, a2, a3, d - a1 - a2 - a3)
            for a1 in range(d + 1) for a2 in range(d + 1 - a1) for a3 in range(d + 1 - a1 - a2)]


def mul_mod(a, da, b, db, m):
    ta, tb = tuples(da), tuples(db)
    out = np.zeros(comb(da + db + 3, 3), dtype=np.int64)
    nzb = [(j, int(b[j])) for j in range(len(tb)) if b[j]]
    for i, ea in enumerate(ta):
        ca = int(a[i])
        if not ca:
            continue
        for j, cb in nzb:
            eb = tb[j]
            out[rank(da + db, (ea[0] + eb[0], ea[1] + eb[1], ea[2] + eb[2]))] += ca * cb
    return (out % m).astype(np.uint8)


def chain(coeffs, p, mul=mul_mod):
    """H, G, Pw mod p^2 from the 35-vector (multiply-by-f_T chain)."""
    psq = p * p
    fT = np.array([pow(int(c), p, psq) for c in coeffs], dtype=np.uint8)
    cur, k = fT, 1
    saved = {1: fT}
    while k < p:
        cur = mul(cur, 4 * k, fT, 4, psq)
        k += 1
        saved[k] = cur
    return fT, saved[p - 2] if p > 2 else None, saved[p - 1], saved[p]


def carry_parts(coeffs, p, mul=mul_mod):
    psq = p * p
    fT, H, G, Pw = chain(coeffs, p, mul)
    h = (H % p).astype(np.uint8)
    g = (G % p).astype(np.uint8)
    tau = np.array([pow(a, p, psq) for a in range(p)], dtype=np.int64)
    num = (G.astype(np.int64) - tau[g]) % psq
    assert not (num % p).any()
    A = ((num // p) % p).astype(np.uint8)
    corr = np.zeros(len(Pw), dtype=np.int64)
    for J, a in zip(tuples(4), coeffs):
        corr[rank(4 * p, (p * J[0], p * J[1], p * J[2]))] = tau[int(a)]
    num = (Pw.astype(np.int64) - corr) % psq
    assert not (num % p).any()
    E = ((num // p) % p).astype(np.uint8)
    return g, h, A, E


def delta_factorized(h, A, E, p):
    """Delta dense over basis(D,4), class by class: Delta[p s + rho] = [rho=0] A[s] - sum_t E[rho+p t] h[s-t]."""
    d, dh, dE = 4 * (p - 1), 4 * (p - 2), 4 * p
    D = p * d
    out = np.zeros(comb(D + 3, 3), dtype=np.uint8)
    hd = {e: int(h[i]) for i, e in enumerate(tuples(dh))}
    for rho in product(range(p), repeat=4):
        if sum(rho) % p:
            continue
        m = sum(rho) // p
        taps = []
        for t in tuples(4 - m):
            c = int(E[rank(dE, tuple(r + p * x for r, x in zip(rho, t)))])
            if c:
                taps.append((t, c))
        for s in tuples(d - m):
            acc = 0
            for t, c in taps:
                u = (s[0] - t[0], s[1] - t[1], s[2] - t[2], s[3] - t[3])
                if min(u) >= 0:
                    acc += c * hd[u]
            v = (int(A[rank(d, s)]) if m == 0 else 0) - acc
            out[rank(D, tuple(p * x + r for x, r in zip(s, rho)))] = v % p
    return out


def matrix_gather(delta, p):
    d = 4 * (p - 1)
    D = p * d
    tb = tuples(d)
    n = len(tb)
    M = np.zeros((n, n), dtype=np.uint8)
    for r, er in enumerate(tb):
        for c, ec in enumerate(tb):
            I = tuple(p * a + p - 1 - b for a, b in zip(er, ec))
            if min(I) >= 0:
                M[r, c] = delta[rank(D, I)]
    return M
