"""ctypes binding of libqfs.so (C ABI in include/qfs.h).

The shared library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a) and must be
present: this package has no CPU fallback, and importing the engine without the library raises
EngineUnavailableError.
"""
import ctypes
import os
import subprocess

from .errors import DomainError, EngineUnavailableError, InternalInvariantError, QfsplitError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqfs.so")
CSRC = os.path.join(_HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

QFS_OK, QFS_EINVAL, QFS_ECUDA, QFS_EINVARIANT, QFS_ENOMEM = 0, -1, -2, -3, -4

EXPORTS = (
    "qfs_version", "qfs_get_shape", "qfs_create", "qfs_destroy", "qfs_last_error",
    "qfs_set_workspace_limit", "qfs_set_chunk", "qfs_heights", "qfs_heights_free", "qfs_heights_lazy", "qfs_get_stats",
    "qfs_stage_power", "qfs_stage_delta", "qfs_stage_matrix", "qfs_stage_matvec_chain",
    "qfs_export_matrix", "qfs_debug_fill_workspaces", "qfs_cubic_heights", "qfs_sample_quartics", "qfs_form_heights",
    "qfs_literal_heights", "qfs_debug_occupancy",
)


class QfsShape(ctypes.Structure):
    _fields_ = [("p", ctypes.c_int32), ("d", ctypes.c_int32), ("D", ctypes.c_int32), ("N", ctypes.c_int32),
                ("pitch", ctypes.c_int32), ("cap", ctypes.c_int32), ("L", ctypes.c_int64)]


class QfsStats(ctypes.Structure):
    _fields_ = [("surfaces", ctypes.c_int64), ("hard", ctypes.c_int64), ("matvec_steps", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("chunks", ctypes.c_int64), ("chunk_capacity", ctypes.c_int64),
                ("ms_power", ctypes.c_double), ("ms_delta", ctypes.c_double), ("ms_matrix", ctypes.c_double),
                ("ms_matvec", ctypes.c_double), ("ms_total", ctypes.c_double), ("built", ctypes.c_int64),
                ("ms_caprow", ctypes.c_double)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared"]


def build_library(force=False, verbose=False):
    """Compile csrc/qfs_lib.cu into libqfs.so with nvcc for sm_100a (cross-compiles without a GPU)."""
    srcs = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))] + [os.path.join(INCLUDE, "qfs.h")]
    if not force and os.path.exists(LIB_PATH) and all(os.path.getmtime(LIB_PATH) >= os.path.getmtime(s) for s in srcs):
        return LIB_PATH
    cmd = ["nvcc"] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + \
          ["-o", LIB_PATH, os.path.join(CSRC, "qfs_lib.cu")]
    subprocess.check_call(cmd)
    return LIB_PATH


_lib = None


def load():
    """The loaded library with argtypes set; raises EngineUnavailableError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise EngineUnavailableError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc, sm_100a).  This package has no CPU fallback.")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise EngineUnavailableError(f"cannot load {LIB_PATH}: {exc}") from None
    vp, sz, u8p, i8p = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p
    lib.qfs_version.restype = ctypes.c_int
    lib.qfs_get_shape.argtypes = [ctypes.c_int, ctypes.POINTER(QfsShape)]
    lib.qfs_create.argtypes = [ctypes.c_int, ctypes.c_int, sz, ctypes.POINTER(vp)]
    lib.qfs_destroy.argtypes = [vp]
    lib.qfs_destroy.restype = None
    lib.qfs_last_error.argtypes = [vp]
    lib.qfs_last_error.restype = ctypes.c_char_p
    lib.qfs_set_workspace_limit.argtypes = [vp, sz]
    lib.qfs_set_chunk.argtypes = [vp, sz]
    lib.qfs_heights.argtypes = [vp, u8p, sz, ctypes.c_int, i8p, i8p, vp]
    lib.qfs_heights_free.argtypes = [vp, u8p, sz, ctypes.c_int, i8p, i8p, vp]
    lib.qfs_heights_lazy.argtypes = [vp, u8p, sz, ctypes.c_int, i8p, i8p, vp]
    lib.qfs_get_stats.argtypes = [vp, ctypes.POINTER(QfsStats)]
    lib.qfs_stage_power.argtypes = [vp, u8p, sz, u8p, u8p]
    lib.qfs_stage_delta.argtypes = [vp, u8p, sz, u8p]
    lib.qfs_stage_matrix.argtypes = [vp, u8p, sz, u8p]
    lib.qfs_stage_matvec_chain.argtypes = [vp, u8p, u8p, sz, ctypes.c_int, u8p, i8p, i8p]
    lib.qfs_export_matrix.argtypes = [vp, u8p, sz, vp]
    lib.qfs_debug_fill_workspaces.argtypes = [vp, ctypes.c_int]
    lib.qfs_debug_occupancy.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
    lib.qfs_cubic_heights.argtypes = [ctypes.c_int, ctypes.c_int, u8p, sz, ctypes.c_int, i8p, i8p]
    lib.qfs_form_heights.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, u8p, sz, ctypes.c_int, i8p, i8p]
    lib.qfs_literal_heights.argtypes = [ctypes.c_int, ctypes.c_int, u8p, sz, ctypes.c_int, i8p, i8p, u8p, u8p]
    lib.qfs_sample_quartics.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64), sz, u8p, ctypes.POINTER(ctypes.c_int)]
    _lib = lib
    return lib


def raise_for(rc, message):
    """Map a qfs_status to the reference's exception types (height.py:76-94, polyring.py:397-398)."""
    if rc == QFS_OK:
        return
    if rc == QFS_EINVAL:
        raise DomainError(message)
    if rc == QFS_EINVARIANT:
        raise InternalInvariantError(message)
    if rc == QFS_ENOMEM:
        raise MemoryError(message)
    if "no CUDA device" in message or "sm_100a" in message:
        raise EngineUnavailableError(message + " (this package has no CPU fallback)")
    raise QfsplitError(f"CUDA failure: {message}")
