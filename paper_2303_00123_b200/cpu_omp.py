"""ctypes binding of libqc_omp.so (include/qc_omp.h): the paper's CPU OpenMP
program (Algs. 1-3, one ``#pragma omp parallel for`` per gate, P:8-11,
P:18-36).  A separate baseline, never a fallback of the GPU path: this module
and libqc.so do not load each other."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .qc import PRECISION, QCError, encode_ops

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqc_omp.so")
EXPORTS = ["qc_omp_run", "qc_omp_max_threads", "qc_omp_last_error"]
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2303_00123_b200.build`")
        L = ctypes.CDLL(LIB_PATH)
        L.qc_omp_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_int]
        L.qc_omp_run.restype = ctypes.c_int
        L.qc_omp_max_threads.restype = ctypes.c_int
        L.qc_omp_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def qc_omp_run(n: int, precision: str, state: np.ndarray, ops, nthreads: int = 0) -> None:
    """Apply ``ops`` in place to the host ``state`` (complex64 / complex128, 2^n)."""
    dt = np.complex128 if precision == "c128" else np.complex64
    if state.dtype != dt or not state.flags.c_contiguous or state.size != (1 << n):
        raise ValueError("state must be a contiguous 2^n array of the precision's dtype")
    arr = ops if isinstance(ops, np.ndarray) else encode_ops(ops)
    arr = np.ascontiguousarray(arr)
    rc = lib().qc_omp_run(n, PRECISION[precision], state.ctypes.data, arr.ctypes.data if len(arr) else None,
                          len(arr), int(nthreads))
    if rc != 0:
        raise QCError(rc, lib().qc_omp_last_error().decode())


def qc_omp_max_threads() -> int:
    return int(lib().qc_omp_max_threads())
