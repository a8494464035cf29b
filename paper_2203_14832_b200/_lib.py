"""ctypes binding of libh2b200.so (the C ABI declared in include/h2b.h).

The shared library is built in-tree by ``build()`` (nvcc, sm_100a).  There is
no fallback: if the library is missing or no CUDA device is present every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("H2B_LIB", os.path.join(HERE, "libh2b200.so"))  # H2B_LIB: dev override
CSRC = os.path.join(HERE, "csrc")

_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p
_lib = None


class H2BError(RuntimeError):
    """Error raised by the native engine."""


def build(force: bool = False) -> str:
    """Compile libh2b200.so for sm_100a in-tree (make -C csrc)."""
    if force:
        subprocess.run(["make", "-s", "-C", CSRC, "clean"], check=True)
    subprocess.run(["make", "-s", "-j8", "-C", CSRC], check=True)
    return LIB_PATH


def _declare(L):
    L.h2b_last_error.restype = ctypes.c_char_p
    L.h2b_version.restype = ctypes.c_int
    L.h2b_kernel_block.argtypes = [ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int64, _dp, ctypes.c_int64,
                                   ctypes.c_int, _dp]
    L.h2b_kernel_row.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _dp, ctypes.c_int64, ctypes.c_int, _dp]
    L.h2b_aca_kernel.argtypes = [ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int64, _dp, ctypes.c_int64,
                                 ctypes.c_int, ctypes.c_double, ctypes.c_int64, _dp, _dp, _i64p, _i64p,
                                 ctypes.POINTER(ctypes.c_int), _i64p, _i64p]
    L.h2b_tree_build.argtypes = [_vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int64, ctypes.c_double, ctypes.c_int, _vp, ctypes.POINTER(_vp)]
    L.h2b_tree_free.argtypes = [_vp]
    L.h2b_tree_free.restype = None
    L.h2b_tree_info.argtypes = [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _dp, _dp]
    L.h2b_tree_ncells.argtypes = [_vp, ctypes.c_int]
    L.h2b_tree_ncells.restype = ctypes.c_int64
    L.h2b_tree_get.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _i64p]
    L.h2b_tree_get.restype = ctypes.c_int64
    L.h2b_assemble.argtypes = [_vp, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int64,
                               _vp, ctypes.POINTER(_vp)]
    L.h2b_h2_free.argtypes = [_vp]
    L.h2b_h2_free.restype = None
    L.h2b_h2_get_i64.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _i64p]
    L.h2b_h2_get_i64.restype = ctypes.c_int64
    L.h2b_h2_get_interp.argtypes = [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int, _i64p, _dp]
    L.h2b_h2_get_interp.restype = ctypes.c_int64
    L.h2b_h2_stats.argtypes = [_vp, _i64p]
    L.h2b_h2_get_coeffs.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _dp]
    L.h2b_h2_get_coeffs.restype = ctypes.c_int64
    L.h2b_matvec.argtypes = [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp]
    L.h2b_matvec_launches.argtypes = [_vp, ctypes.c_int64]
    L.h2b_matvec_launches.restype = ctypes.c_int64
    L.h2b_set_profiling.argtypes = [ctypes.c_int]
    L.h2b_last_stage_ms.argtypes = [_dp]
    L.h2b_fp64_peak.argtypes = [_dp]
    L.h2b_dense_matvec.argtypes = [ctypes.c_int, ctypes.c_double, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                   ctypes.c_int, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp]
    L.h2b_dense_rows.argtypes = [ctypes.c_int, ctypes.c_double, _dp, ctypes.c_int64, _i64p, ctypes.c_int64, _dp,
                                 ctypes.c_int64, ctypes.c_int, _dp, _dp]
    L.h2b_host_alloc.argtypes = [ctypes.POINTER(_vp), ctypes.c_int64]
    L.h2b_host_free.argtypes = [_vp]
    L.h2b_host_free.restype = None
    L.h2b_release_workspace.argtypes = []
    return L


def lib():
    """Load libh2b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise H2BError(f"{LIB_PATH} is missing: run paper_2203_14832_b200._lib.build() (nvcc, sm_100a)")
        _lib = _declare(ctypes.CDLL(LIB_PATH))
    return _lib


# names exported by include/h2b.h (checked by the CPU test suite)
EXPORTS = (
    "h2b_last_error", "h2b_version", "h2b_kernel_block", "h2b_kernel_row", "h2b_aca_kernel", "h2b_tree_build",
    "h2b_tree_free", "h2b_tree_info", "h2b_tree_ncells", "h2b_tree_get", "h2b_assemble", "h2b_h2_free",
    "h2b_h2_get_i64", "h2b_h2_get_interp", "h2b_h2_stats", "h2b_matvec", "h2b_matvec_launches",
    "h2b_set_profiling", "h2b_last_stage_ms", "h2b_fp64_peak", "h2b_dense_matvec", "h2b_dense_rows",
    "h2b_host_alloc", "h2b_host_free", "h2b_release_workspace", "h2b_h2_get_coeffs",
)


def check(rc):
    if rc < 0:
        msg = lib().h2b_last_error().decode()
        if msg.startswith("ValueError: "):
            raise ValueError(msg[len("ValueError: "):])
        raise H2BError(msg)
    return rc


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def iptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)
