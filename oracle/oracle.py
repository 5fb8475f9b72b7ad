"""ctypes front end of the C oracle (qfs_oracle.c).  Test infrastructure only.

Every function mirrors one reference entry point on dense uint8 vectors
(lex-ascending basis, x1 most significant; heights use 0 for infinity):

    power_mod_p      <- qfsplit.polyring.power_mod_p        (polyring.py:253)
    delta1           <- qfsplit.polyring.delta1             (polyring.py:335)
    build_mts        <- qfsplit.mtsmatrix.build_mts         (mtsmatrix.py:287)
    matvec           <- qfsplit.modmatrix.matvec            (modmatrix.py:109)
    height_matrix    <- qfsplit.height.height_matrix        (height.py:119)
    height_naive     <- qfsplit.height.height_naive         (height.py:97)
    heights_batch    <- loop body of search._worker_block   (search.py:108)
"""
import ctypes
import os
import subprocess
from math import comb

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libqfs_oracle.so")
_lib = None

__all__ = ["build", "basis_size", "rank", "cap_index", "power_mod_p", "delta1", "build_mts", "matvec",
           "height_matrix", "height_naive", "heights_batch", "max_threads", "OracleError", "poly_mul_mod"]


class OracleError(RuntimeError):
    pass


def build(force=False):
    """Compile the C oracle with gcc (idempotent)."""
    src = os.path.join(_HERE, "qfs_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "-B", "all"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        lib = ctypes.CDLL(_SO)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        i8p = ctypes.POINTER(ctypes.c_int8)
        lib.qfo_basis_size.restype = ctypes.c_int64
        lib.qfo_basis_size.argtypes = [ctypes.c_int]
        lib.qfo_rank.restype = ctypes.c_int64
        lib.qfo_rank.argtypes = [ctypes.c_int] * 4
        lib.qfo_poly_mul_mod.argtypes = [u8p, ctypes.c_int, u8p, ctypes.c_int, ctypes.c_int, u8p]
        lib.qfo_power_mod_p.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p]
        lib.qfo_delta1.argtypes = [u8p, ctypes.c_int, ctypes.c_int, u8p]
        lib.qfo_build_mts.argtypes = [u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p]
        lib.qfo_matvec.argtypes = [u8p, ctypes.c_int64, ctypes.c_int64, u8p, ctypes.c_int, u8p]
        lib.qfo_height_matrix.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i8p, i8p, u8p, u8p, u8p, u8p]
        lib.qfo_height_naive.argtypes = [u8p, ctypes.c_int, ctypes.c_int, i8p, i8p]
        lib.qfo_heights_batch.argtypes = [u8p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, i8p, i8p, ctypes.c_int]
        lib.qfo_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _u8(a):
    a = np.ascontiguousarray(a, dtype=np.uint8)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _check(rc, what):
    if rc != 0:
        raise OracleError(f"{what} failed with code {rc}")


def basis_size(d):
    return comb(d + 3, 3)


def rank(d, a1, a2, a3):
    return int(_load().qfo_rank(d, a1, a2, a3))


def cap_index(p):
    return rank(4 * (p - 1), p - 1, p - 1, p - 1)


def max_threads():
    return int(_load().qfo_max_threads())


def poly_mul_mod(a, da, b, db, m):
    a, ap = _u8(a)
    b, bp = _u8(b)
    out = np.zeros(basis_size(da + db), dtype=np.uint8)
    _check(_load().qfo_poly_mul_mod(ap, da, bp, db, m, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))), "poly_mul_mod")
    return out


def power_mod_p(f, df, k, p):
    f, fp = _u8(f)
    assert f.size == basis_size(df)
    out = np.zeros(basis_size(df * k), dtype=np.uint8)
    _check(_load().qfo_power_mod_p(fp, df, k, p, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))), "power_mod_p")
    return out


def delta1(g, dg, p):
    g, gp = _u8(g)
    assert g.size == basis_size(dg)
    out = np.zeros(basis_size(dg * p), dtype=np.uint8)
    _check(_load().qfo_delta1(gp, dg, p, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))), "delta1")
    return out


def build_mts(delta, p):
    d = 4 * (p - 1)
    D = p * d
    delta, dp = _u8(delta)
    assert delta.size == basis_size(D)
    n = basis_size(d)
    out = np.zeros((n, n), dtype=np.uint8)
    _check(_load().qfo_build_mts(dp, D, d, p, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))), "build_mts")
    return out


def matvec(M, v, p):
    M, mp = _u8(M)
    v, vp = _u8(v)
    out = np.zeros(M.shape[0], dtype=np.uint8)
    _check(_load().qfo_matvec(mp, M.shape[0], M.shape[1], vp, p, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))), "matvec")
    return out


def height_matrix(coeffs, p, bound=10, taps=False):
    """(height, iterations[, taps dict]) for one 35-vector; height 0 = infinity."""
    c, cp = _u8(coeffs)
    assert c.size == 35
    h = ctypes.c_int8(0)
    it = ctypes.c_int8(0)
    u8p = ctypes.POINTER(ctypes.c_uint8)
    null = ctypes.cast(None, u8p)
    if not taps:
        _check(_load().qfo_height_matrix(cp, p, bound, ctypes.byref(h), ctypes.byref(it), null, null, null, null), "height_matrix")
        return int(h.value), int(it.value)
    d = 4 * (p - 1)
    n, L = basis_size(d), basis_size(p * d)
    g = np.zeros(n, np.uint8)
    dl = np.zeros(L, np.uint8)
    M = np.zeros((n, n), np.uint8)
    tr = np.zeros((max(bound - 1, 1), n), np.uint8)
    _check(_load().qfo_height_matrix(cp, p, bound, ctypes.byref(h), ctypes.byref(it),
                                     g.ctypes.data_as(u8p), dl.ctypes.data_as(u8p), M.ctypes.data_as(u8p),
                                     tr.ctypes.data_as(u8p)), "height_matrix")
    return int(h.value), int(it.value), {"g": g, "delta": dl, "M": M, "trace": tr[: it.value]}


def height_naive(coeffs, p, bound=10):
    c, cp = _u8(coeffs)
    h = ctypes.c_int8(0)
    it = ctypes.c_int8(0)
    _check(_load().qfo_height_naive(cp, p, bound, ctypes.byref(h), ctypes.byref(it)), "height_naive")
    return int(h.value), int(it.value)


def heights_batch(coeffs, p, bound=10, threads=0):
    c, cp = _u8(coeffs)
    assert c.ndim == 2 and c.shape[1] == 35
    B = c.shape[0]
    hs = np.zeros(B, np.int8)
    its = np.zeros(B, np.int8)
    i8p = ctypes.POINTER(ctypes.c_int8)
    _check(_load().qfo_heights_batch(cp, B, p, bound, hs.ctypes.data_as(i8p), its.ctypes.data_as(i8p), threads), "heights_batch")
    return hs, its
