"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads ``oracle/liboracle.so`` (plain C99 + OpenMP, ``qc_oracle.c``) and runs
op lists from :mod:`qcgen` on complex128 numpy states.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / --impl reference)
may import this package; the product package never does.

See ``qc_oracle.c`` for what is computed and the PAPER.md passages it follows.
Every function here is pinned by tests/test_oracle.py (no "parity unpinned"
entries).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# The oracle's own op codes (must match the enum in qc_oracle.c).
KIND = {"H": 0, "X": 1, "Y": 2, "Z": 3, "P": 4, "RX": 5, "RY": 6, "RZ": 7,
        "CNOT": 8, "CZ": 9, "CP": 10, "SWAP": 11, "U1": 12, "CU1": 13, "U2": 14,
        "CCX": 15}

OP_DTYPE = np.dtype([("kind", "<i4"), ("nq", "<i4"), ("q", "<i4", (3,)),
                     ("ctrl_state", "<u4"), ("theta", "<f8"), ("m", "<f8", (32,))])
assert OP_DTYPE.itemsize == 288


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, no fast-math, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off", "-fPIC",
               "-shared", _SRC, "-o", _LIB, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_run.restype = ctypes.c_int64
        L.orc_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_int64, ctypes.c_int]
        L.orc_embed.restype = ctypes.c_int
        L.orc_embed.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_run_general.restype = ctypes.c_int64
        L.orc_run_general.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_int64, ctypes.c_int]
        _lib = L
    return _lib


def encode(ops: Sequence) -> np.ndarray:
    """qcgen.Op list -> array of the oracle's C struct."""
    arr = np.zeros(len(ops), dtype=OP_DTYPE)
    for i, op in enumerate(ops):
        arr[i]["kind"] = KIND[op.name]
        arr[i]["nq"] = len(op.qubits)
        q = list(op.qubits) + [0] * (3 - len(op.qubits))
        arr[i]["q"] = q
        arr[i]["ctrl_state"] = op.ctrl_state
        arr[i]["theta"] = 0.0 if op.theta is None else op.theta
        if op.matrix is not None:
            m = np.asarray(op.matrix, dtype=np.complex128).reshape(-1)
            flat = np.zeros(32)
            flat[0:2 * m.size:2] = m.real
            flat[1:2 * m.size:2] = m.imag
            arr[i]["m"] = flat
    return arr


GOP_DTYPE = np.dtype([("nq", "<i4"), ("nctrl", "<i4"), ("q", "<i4", (16,)), ("ctrl_state", "<u4"),
                      ("pad", "<i4"), ("m", "<u8")])
assert GOP_DTYPE.itemsize == 88


def _run_general(n: int, psi: np.ndarray, ops: Sequence, nthreads: int) -> None:
    """Generic (MCU) gates through orc_run_general, in order."""
    arr = np.zeros(len(ops), dtype=GOP_DTYPE)
    keep = []
    for i, op in enumerate(ops):
        arr[i]["nq"] = len(op.qubits)
        arr[i]["nctrl"] = op.nctrl
        arr[i]["q"] = list(op.qubits) + [0] * (16 - len(op.qubits))
        arr[i]["ctrl_state"] = op.ctrl_state
        m = np.ascontiguousarray(np.asarray(op.matrix, dtype=np.complex128)).view(np.float64).reshape(-1)
        keep.append(m)
        arr[i]["m"] = m.ctypes.data
    rc = lib().orc_run_general(n, psi.ctypes.data, arr.ctypes.data if len(arr) else None, len(arr),
                               int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle rejected generic op list (code {rc})")


def run(n: int, state: np.ndarray, ops: Sequence, nthreads: int = 0) -> np.ndarray:
    """Apply ``ops`` to a copy of ``state`` (any complex dtype, exact up-cast).
    Generic ``MCU`` ops go through orc_run_general, the rest through orc_run,
    in list order."""
    psi = np.ascontiguousarray(np.asarray(state).astype(np.complex128))
    if psi.size != (1 << n):
        raise ValueError("state size != 2^n")
    ops = list(ops)
    i = 0
    while i < len(ops) or i == 0:
        j = i
        gen = i < len(ops) and ops[i].name == "MCU"
        while j < len(ops) and (ops[j].name == "MCU") == gen:
            j += 1
        seg = ops[i:j]
        if gen:
            _run_general(n, psi, seg, nthreads)
        else:
            enc = encode(seg)
            rc = lib().orc_run(n, psi.ctypes.data, enc.ctypes.data if len(enc) else None,
                               len(enc), int(nthreads))
            if rc != 0:
                raise ValueError(f"oracle rejected op list (code {rc})")
        if j == i:
            break
        i = j
    return psi


def embed(op) -> np.ndarray:
    """The oracle's embedded 2^k x 2^k matrix of one op (listed qubit = MSB)."""
    enc = encode([op])
    U = np.zeros(64, dtype=np.complex128)
    k = lib().orc_embed(enc.ctypes.data, U.ctypes.data)
    if k < 0:
        raise ValueError("unknown op")
    d = 1 << k
    return U[: d * d].reshape(d, d).copy()


def max_threads() -> int:
    return int(lib().orc_max_threads())
