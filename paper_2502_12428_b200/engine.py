"""Engine: one libqfs context per (prime, GPU), driven from Python.

Inputs and outputs may be numpy arrays (host memory; the library stages them itself) or torch
CUDA tensors (device memory; only their data_ptr() crosses the ABI).  PyTorch is optional here.
"""
import ctypes
import threading

import numpy as np

from . import _native
from .errors import DomainError

_lock = threading.Lock()
_engines = {}


def shape_of(p):
    """qfs_shape for a supported prime (DomainError otherwise)."""
    s = _native.QfsShape()
    if _native.load().qfs_get_shape(int(p), ctypes.byref(s)) != 0:
        raise DomainError(f"p={p} is not supported by the GPU engine (supported: 3, 5, 7, 11, 13)")
    return s


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _in_ptr(x, shape, what):
    """(pointer, keepalive) of a uint8 input with the given shape."""
    if _is_torch(x):
        if x.dtype.__str__() != "torch.uint8" or tuple(x.shape) != tuple(shape) or not x.is_contiguous():
            raise DomainError(f"{what}: expected contiguous uint8 tensor of shape {tuple(shape)}")
        return x.data_ptr(), x
    a = np.ascontiguousarray(x, dtype=np.uint8)
    if a.shape != tuple(shape):
        raise DomainError(f"{what}: expected shape {tuple(shape)}, got {a.shape}")
    return a.ctypes.data, a


class Engine:
    """Owns one qfs_ctx (single-threaded at the C ABI): every call into the library holds the engine's lock, so threads that
    share an Engine (get_engine caches one per prime and GPU) take turns instead of running on the same workspaces."""

    def __init__(self, p, device=0, max_batch=0):
        self.lib = _native.load()
        self.shape = shape_of(p)
        self.p = int(p)
        self.device = int(device)
        handle = ctypes.c_void_p()
        rc = self.lib.qfs_create(self.p, self.device, int(max_batch), ctypes.byref(handle))
        if rc != 0:
            _native.raise_for(rc, self.lib.qfs_last_error(None).decode())
        self._h = handle
        self._mutex = threading.RLock()

    def _call(self, fn, *args):
        with self._mutex:
            self._check(fn(self._h, *args))

    def close(self):
        if getattr(self, "_h", None):
            self.lib.qfs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            _native.raise_for(rc, self.lib.qfs_last_error(self._h).decode())

    # -- configuration -----------------------------------------------------------------------
    def set_workspace_limit(self, nbytes):
        self._call(self.lib.qfs_set_workspace_limit, int(nbytes))

    def set_chunk(self, n):
        self._call(self.lib.qfs_set_chunk, int(n))

    def occupancy(self):
        """Resident CTAs per SM of k_power_full, k_delta_mma, k_matrix_staged, k_chain as built (qfs_debug_occupancy)."""
        out = (ctypes.c_int * 4)()
        self._check(self.lib.qfs_debug_occupancy(self._h, out))
        return dict(zip(("k_power_full", "k_delta_mma", "k_matrix_staged", "k_chain"), (int(x) for x in out)))

    def stats(self):
        st = _native.QfsStats()
        self._check(self.lib.qfs_get_stats(self._h, ctypes.byref(st)))
        return st.as_dict()

    # -- hot path ----------------------------------------------------------------------------
    def heights(self, coeffs, bound=10, out=None, matrix_free=False, lazy=False):
        """(heights int8[B], iterations int8[B]); heights use 0 for infinity.

        coeffs: [B,35] uint8 numpy array or torch CUDA tensor.  With torch input the outputs are
        torch int8 tensors on the same device unless `out=(heights, iters)` is given.
        matrix_free: the polynomial iteration (qfs_heights_free).  lazy: the operator-matrix path with the cap row of the
        first step evaluated before Delta and M are built (qfs_heights_lazy); same results either way.
        """
        if matrix_free and lazy:
            raise DomainError("matrix_free and lazy are different modes: choose one")
        if not isinstance(bound, (int, np.integer)) or bound < 1:
            raise DomainError(f"bound must be a positive integer, got {bound}")
        B = int(coeffs.shape[0]) if hasattr(coeffs, "shape") and len(coeffs.shape) == 2 else -1
        if B < 0:
            raise DomainError("coeffs must have shape [B, 35]")
        cptr, keep = _in_ptr(coeffs, (B, 35), "coeffs")
        if out is not None:
            hs, its = out
        elif _is_torch(coeffs):
            import torch
            hs = torch.empty(B, dtype=torch.int8, device=coeffs.device)
            its = torch.empty(B, dtype=torch.int8, device=coeffs.device)
        else:
            hs = np.empty(B, dtype=np.int8)
            its = np.empty(B, dtype=np.int8)
        hp = hs.data_ptr() if _is_torch(hs) else hs.ctypes.data
        ip = its.data_ptr() if _is_torch(its) else its.ctypes.data
        stream = None
        for t in (coeffs, hs, its):
            if _is_torch(t) and t.is_cuda and t.device.index != self.device:
                raise DomainError(f"tensor on {t.device} handed to the engine of cuda:{self.device}")
        if _is_torch(coeffs) and coeffs.is_cuda:
            import torch
            # the library orders its own stream behind this one (a NULL handle -- the default stream -- included)
            stream = torch.cuda.current_stream(coeffs.device).cuda_stream
        fn = self.lib.qfs_heights_free if matrix_free else (self.lib.qfs_heights_lazy if lazy else self.lib.qfs_heights)
        self._call(fn, cptr, B, int(bound), hp, ip, stream)
        del keep
        return hs, its

    def sample(self, seed, worker, count, out=None):
        """The `count` coefficient vectors of worker `worker` of the reference's search (search.py:92-103), drawn on the device.

        Returns (coeffs, clean): coeffs is `out` (a uint8 [count,35] numpy array or torch CUDA tensor) or a new numpy array;
        clean is False when the block hit one of the stream-shifting events the device only reports (a Lemire rejection, a zero
        row) -- the caller must then draw the block on the host (search.sample_block)."""
        bg = np.random.PCG64(np.random.SeedSequence([int(seed), int(worker)]))
        st = bg.state["state"]
        mask = (1 << 64) - 1
        words = (ctypes.c_uint64 * 4)(st["state"] >> 64, st["state"] & mask, st["inc"] >> 64, st["inc"] & mask)
        if out is None:
            out = np.empty((int(count), 35), dtype=np.uint8)
        ptr, keep = _in_ptr(out, (int(count), 35), "out")
        if _is_torch(out) and out.is_cuda and out.device.index != self.device:
            raise DomainError(f"tensor on {out.device} handed to the engine of cuda:{self.device}")
        clean = ctypes.c_int(0)
        self._call(self.lib.qfs_sample_quartics, words, int(count), ptr, ctypes.byref(clean))
        del keep
        return out, bool(clean.value)

    # -- stage taps (host numpy in/out) ------------------------------------------------------
    def stage_power(self, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.uint8).reshape(-1, 35)
        B = c.shape[0]
        g = np.empty((B, self.shape.N), dtype=np.uint8)
        fed = np.empty(B, dtype=np.uint8)
        self._call(self.lib.qfs_stage_power, c.ctypes.data, B, g.ctypes.data, fed.ctypes.data)
        return g, fed

    def stage_delta(self, coeffs):
        c = np.ascontiguousarray(coeffs, dtype=np.uint8).reshape(-1, 35)
        B = c.shape[0]
        out = np.empty((B, self.shape.L), dtype=np.uint8)
        self._call(self.lib.qfs_stage_delta, c.ctypes.data, B, out.ctypes.data)
        return out

    def stage_matrix(self, delta):
        dl = np.ascontiguousarray(delta, dtype=np.uint8).reshape(-1, self.shape.L)
        B = dl.shape[0]
        n = self.shape.N
        out = np.empty((B, n, n), dtype=np.uint8)
        self._call(self.lib.qfs_stage_matrix, dl.ctypes.data, B, out.ctypes.data)
        return out

    def debug_fill_workspaces(self, byte):
        """Test hook: overwrite every device workspace with `byte` (include/qfs.h)."""
        self._call(self.lib.qfs_debug_fill_workspaces, int(byte))

    def export_matrix(self, coeffs):
        """Operator matrices [B][N][N] as uint16, the reference's MtsMatrix.entries (mtsmatrix.py:96)."""
        c = np.ascontiguousarray(coeffs, dtype=np.uint8).reshape(-1, 35)
        B = c.shape[0]
        n = self.shape.N
        out = np.empty((B, n, n), dtype="<u2")
        self._call(self.lib.qfs_export_matrix, c.ctypes.data, B, out.ctypes.data)
        return out

    def stage_matvec_chain(self, M, v0, max_steps, trace=False):
        n = self.shape.N
        M = np.ascontiguousarray(M, dtype=np.uint8).reshape(-1, n, n)
        v0 = np.ascontiguousarray(v0, dtype=np.uint8).reshape(-1, n)
        B = M.shape[0]
        if v0.shape[0] != B:
            raise DomainError("M and v0 disagree on the batch size")
        hs = np.empty(B, dtype=np.int8)
        its = np.empty(B, dtype=np.int8)
        tr = np.zeros((B, max_steps, n), dtype=np.uint8) if trace else None
        self._call(self.lib.qfs_stage_matvec_chain, M.ctypes.data, v0.ctypes.data, B, int(max_steps),
                   tr.ctypes.data if trace else None, hs.ctypes.data, its.ctypes.data)
        return (hs, its, tr) if trace else (hs, its)


def get_engine(p, device=0):
    """Process-wide cached Engine for (p, device)."""
    key = (int(p), int(device))
    with _lock:
        eng = _engines.get(key)
        if eng is None:
            eng = _engines[key] = Engine(p, device)
        return eng


def close_all():
    with _lock:
        for eng in _engines.values():
            eng.close()
        _engines.clear()
