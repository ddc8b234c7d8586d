"""Thin ctypes binding of libqc.so (include/qc.h).  Argument marshalling only:
every step of the gate path runs in the library's CUDA kernels.  There is no
CPU fallback -- if the extension is missing this module raises on import of
the library.

Raw entry points keep the C names (``qc_state_create``, ``qc_apply_gate``,
``qc_run_circuit``, ``qc_state_read`` ...).  :class:`State` is a small
convenience wrapper used by the tests and ``bench.py``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QC_LIB", os.path.join(_HERE, "libqc.so"))

QC_OK, QC_ERR_INVALID_ARG, QC_ERR_OUT_OF_MEMORY, QC_ERR_CUDA, QC_ERR_NCCL, \
    QC_ERR_UNSUPPORTED, QC_ERR_STATE_FAILED = range(7)
QC_COMPLEX64, QC_COMPLEX128 = 0, 1
PRECISION = {"c64": QC_COMPLEX64, "c128": QC_COMPLEX128}
OPS = {"H": 0, "X": 1, "Y": 2, "Z": 3, "P": 4, "RX": 5, "RY": 6, "RZ": 7, "CNOT": 8,
       "CZ": 9, "CP": 10, "SWAP": 11, "U1": 12, "CU1": 13, "U2": 14, "CCX": 15}
ARITY = {"H": 1, "X": 1, "Y": 1, "Z": 1, "P": 1, "RX": 1, "RY": 1, "RZ": 1, "CNOT": 2,
         "CZ": 2, "CP": 2, "SWAP": 2, "U1": 1, "CU1": 2, "U2": 2, "CCX": 3}
QC_CTRL_ONES = 0xFFFFFFFF
OPTIONS = {"fusion": 0, "relabel_swap": 1, "use_graph": 2, "tile_bits": 3, "ctas": 4,
           "block_fusion": 5, "jit": 6, "row_bits": 7,
           "tma_mode": 8, "remap": 9, "exchange": 10}

GATE_DTYPE = np.dtype([("op", "<i4"), ("qubits", "<i4", (3,)), ("ctrl_state", "<u4"),
                       ("flags", "<u4"), ("theta", "<f8"), ("m", "<f8", (32,))])
assert GATE_DTYPE.itemsize == 288
QC_MGATE = 16
MGATE_DTYPE = np.dtype([("n_ctrl", "<i4"), ("n_targ", "<i4"), ("qubits", "<i4", (16,)),
                        ("ctrl_state", "<u4"), ("flags", "<u4"), ("matrix", "<u8")])
assert MGATE_DTYPE.itemsize == 88


class GateArray(np.ndarray):
    """qc_gate records plus the qc_mgate table their QC_MGATE ops refer to
    (``mtab``; ``keep`` holds the matrices the table points into)."""

    def __array_finalize__(self, obj):
        self.mtab = getattr(obj, "mtab", None)
        self.keep = getattr(obj, "keep", None)

EXPORTS = ["qc_state_create", "qc_state_create_ex", "qc_state_wrap", "qc_state_destroy",
           "qc_state_create_dist", "qc_state_create_loopback", "qc_nccl_unique_id",
           "qc_state_init_basis", "qc_state_init_random", "qc_apply_gate", "qc_run_circuit",
           "qc_run_circuit_ex", "qc_apply_mgate",
           "qc_state_read", "qc_state_write", "qc_state_readwrite", "qc_state_canonicalize", "qc_state_sync",
           "qc_state_norm2", "qc_set_option", "qc_get_info", "qc_qasm_parse", "qc_qasm_emit",
           "qc_last_error", "qc_version"]


class QCError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"qc status {status}: {msg}")
        self.status = status


class qc_info(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("device_ptr", ctypes.c_void_p), ("stream", ctypes.c_void_p),
                ("layout", ctypes.c_int32 * 64), ("layout_is_canonical", ctypes.c_int32),
                ("last_gates", ctypes.c_int64), ("last_passes", ctypes.c_int64),
                ("last_launches", ctypes.c_int64), ("last_relabels", ctypes.c_int64),
                ("last_graph", ctypes.c_int32), ("tile_bits", ctypes.c_int32),
                ("last_blocks", ctypes.c_int64), ("last_jit", ctypes.c_int32),
                ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("n_local", ctypes.c_int32),
                ("sharding", ctypes.c_int32), ("last_exchanges", ctypes.c_int64),
                ("last_flops_per_amp", ctypes.c_double), ("last_pair_segments", ctypes.c_int64)]


class qc_plan_stats(ctypes.Structure):
    _fields_ = [("gates", ctypes.c_int64), ("relabels", ctypes.c_int64), ("blocks", ctypes.c_int64),
                ("passes", ctypes.c_int64), ("substages", ctypes.c_int64),
                ("fused_ops", ctypes.c_int64), ("phase_runs", ctypes.c_int64),
                ("blob_bytes", ctypes.c_int64), ("tile_bits", ctypes.c_int32),
                ("jit_compiled", ctypes.c_int32), ("remap_swaps", ctypes.c_int64),
                ("restore_passes", ctypes.c_int64), ("flops_per_amp", ctypes.c_double),
                ("swz_substages", ctypes.c_int64)]


DEBUG_EXPORTS = ["qc_debug_plan", "qc_debug_exchange_runs", "qc_debug_dist_schedule", "qc_debug_dist_schedule_ex", "qc_debug_exchange",
                 "qc_debug_group_split",
                 "qc_debug_fma_peak", "qc_debug_box_layout"]

_lib = None


def lib() -> ctypes.CDLL:
    """Load libqc.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2303_00123_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, u64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_size_t
    L.qc_state_create.restype = vp
    L.qc_state_create.argtypes = [i32, i32]
    L.qc_state_create_ex.argtypes = [i32, i32, i32, vp, ctypes.POINTER(vp)]
    L.qc_state_wrap.argtypes = [i32, i32, vp, vp, ctypes.POINTER(vp)]
    L.qc_state_destroy.argtypes = [vp]
    L.qc_state_destroy.restype = None
    L.qc_state_init_basis.argtypes = [vp, u64]
    L.qc_state_init_random.argtypes = [vp, u64]
    L.qc_apply_gate.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
    L.qc_run_circuit.argtypes = [vp, vp, sz]
    L.qc_run_circuit_ex.argtypes = [vp, vp, sz, vp, sz]
    L.qc_apply_mgate.argtypes = [vp, vp]
    L.qc_state_read.argtypes = [vp, u64, u64, vp]
    L.qc_state_write.argtypes = [vp, u64, u64, vp]
    L.qc_state_readwrite.argtypes = [vp, u64, u64, vp, vp]
    L.qc_state_canonicalize.argtypes = [vp]
    L.qc_state_sync.argtypes = [vp]
    L.qc_state_norm2.argtypes = [vp, ctypes.POINTER(ctypes.c_double)]
    L.qc_set_option.argtypes = [vp, i32, ctypes.c_int64]
    L.qc_get_info.argtypes = [vp, ctypes.POINTER(qc_info)]
    L.qc_debug_plan.argtypes = [i32, i32, vp, sz, i32, i32, i32, i32, i32, ctypes.POINTER(qc_plan_stats),
                                ctypes.c_char_p, sz]
    L.qc_debug_plan.restype = ctypes.c_int
    L.qc_state_create_dist.argtypes = [i32, i32, i32, i32, vp, ctypes.POINTER(vp)]
    L.qc_state_create_loopback.argtypes = [i32, i32, i32, ctypes.POINTER(vp)]
    L.qc_nccl_unique_id.argtypes = [vp]
    L.qc_debug_exchange_runs.argtypes = [i32, i32, i32, i32, ctypes.POINTER(ctypes.c_int), vp, vp, i32,
                                         ctypes.POINTER(ctypes.c_int)]
    L.qc_debug_exchange_runs.restype = ctypes.c_int
    L.qc_debug_dist_schedule.argtypes = [i32, i32, i32, vp, sz, vp, i32, ctypes.POINTER(ctypes.c_int), vp]
    L.qc_debug_dist_schedule.restype = ctypes.c_int
    L.qc_debug_dist_schedule_ex.argtypes = [i32, i32, i32, i32, vp, sz, vp, i32, ctypes.POINTER(ctypes.c_int), vp]
    L.qc_debug_dist_schedule_ex.restype = ctypes.c_int
    L.qc_debug_group_split.argtypes = [i32, i32, u64, i32, ctypes.POINTER(ctypes.c_uint64),
                                       ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_int),
                                       ctypes.POINTER(ctypes.c_int)]
    L.qc_debug_group_split.restype = ctypes.c_int
    L.qc_debug_exchange.argtypes = [vp, i32, i32]
    L.qc_debug_exchange.restype = ctypes.c_int
    L.qc_debug_box_layout.argtypes = [u64, i32, i32, ctypes.POINTER(ctypes.c_int), vp, vp,
                                      ctypes.POINTER(ctypes.c_uint32)]
    L.qc_debug_box_layout.restype = ctypes.c_int
    L.qc_debug_fma_peak.argtypes = [i32, ctypes.POINTER(ctypes.c_double)]
    L.qc_debug_fma_peak.restype = ctypes.c_int
    L.qc_last_error.restype = ctypes.c_char_p
    L.qc_version.restype = ctypes.c_char_p
    L.qc_qasm_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), vp, sz, ctypes.POINTER(ctypes.c_size_t)]
    L.qc_qasm_parse.restype = ctypes.c_int
    L.qc_qasm_emit.argtypes = [i32, vp, sz, ctypes.c_char_p, sz, ctypes.POINTER(ctypes.c_size_t)]
    L.qc_qasm_emit.restype = ctypes.c_int
    for name in EXPORTS:
        f = getattr(L, name)
        if name not in ("qc_state_create", "qc_state_destroy", "qc_last_error", "qc_version"):
            f.restype = ctypes.c_int
    _lib = L
    return L


def _check(rc: int):
    if rc != QC_OK:
        raise QCError(rc, lib().qc_last_error().decode())


def encode_mgate(op, keep: list) -> np.ndarray:
    """A generic ("MCU") gate record -> one qc_mgate struct (matrix kept alive in ``keep``)."""
    g = np.zeros(1, dtype=MGATE_DTYPE)
    nc = int(op.nctrl)
    g[0]["n_ctrl"] = nc
    g[0]["n_targ"] = len(op.qubits) - nc
    g[0]["qubits"] = list(op.qubits) + [0] * (16 - len(op.qubits))
    g[0]["ctrl_state"] = op.ctrl_state
    m = np.ascontiguousarray(np.asarray(op.matrix, dtype=np.complex128)).view(np.float64).reshape(-1)
    keep.append(m)
    g[0]["matrix"] = m.ctypes.data
    return g


def encode_ops(ops: Iterable) -> np.ndarray:
    """Gate records (objects with name, qubits, theta, matrix, ctrl_state) ->
    contiguous array of ``qc_gate`` structs (a :class:`GateArray` carrying the
    qc_mgate table when the list holds generic "MCU" gates)."""
    ops = list(ops)
    arr = np.zeros(len(ops), dtype=GATE_DTYPE)
    mt, keep = [], []
    for i, op in enumerate(ops):
        name = op.name
        if name == "MCU":
            arr[i]["op"] = QC_MGATE
            arr[i]["qubits"] = [len(mt), 0, 0]
            mt.append(encode_mgate(op, keep))
            continue
        arr[i]["op"] = OPS[name]
        q = list(op.qubits) + [0] * (3 - len(op.qubits))
        arr[i]["qubits"] = q
        cs = getattr(op, "ctrl_state", None)
        arr[i]["ctrl_state"] = QC_CTRL_ONES if cs is None else cs
        th = getattr(op, "theta", None)
        arr[i]["theta"] = 0.0 if th is None else th
        m = getattr(op, "matrix", None)
        if m is not None:
            m = np.asarray(m, dtype=np.complex128).reshape(-1)
            flat = np.zeros(32)
            flat[0:2 * m.size:2] = m.real
            flat[1:2 * m.size:2] = m.imag
            arr[i]["m"] = flat
    if mt:
        arr = arr.view(GateArray)
        arr.mtab = np.concatenate(mt)
        arr.keep = keep
    return arr


def qasm_parse(text: str):
    """openQASM 2.0 text -> (n_qubits, qc_gate array) via qc_qasm_parse."""
    b = text.encode()
    n = ctypes.c_int(0)
    cnt = ctypes.c_size_t(0)
    _check(lib().qc_qasm_parse(b, ctypes.byref(n), None, 0, ctypes.byref(cnt)))
    arr = np.zeros(cnt.value, dtype=GATE_DTYPE)
    _check(lib().qc_qasm_parse(b, ctypes.byref(n), arr.ctypes.data if cnt.value else None, cnt.value,
                               ctypes.byref(cnt)))
    return n.value, arr


def qasm_emit(n: int, ops) -> str:
    """Gate list -> openQASM 2.0 text via qc_qasm_emit."""
    arr = ops if isinstance(ops, np.ndarray) else encode_ops(ops)
    arr = np.ascontiguousarray(arr)
    ln = ctypes.c_size_t(0)
    p = arr.ctypes.data if len(arr) else None
    _check(lib().qc_qasm_emit(n, p, len(arr), None, 0, ctypes.byref(ln)))
    buf = ctypes.create_string_buffer(ln.value + 1)
    _check(lib().qc_qasm_emit(n, p, len(arr), buf, ln.value + 1, ctypes.byref(ln)))
    return buf.value.decode()


class State:
    """Owning handle of one qc_state (device-resident 2^n amplitudes)."""

    def __init__(self, n: int, precision: str = "c128", device: int = 0,
                 stream: Optional[int] = None, _handle=None):
        self.n = n
        self.precision = precision
        self.dtype = np.complex128 if precision == "c128" else np.complex64
        if _handle is not None:
            self._h = _handle
            return
        h = ctypes.c_void_p()
        _check(lib().qc_state_create_ex(n, PRECISION[precision], device, stream, ctypes.byref(h)))
        self._h = h

    @classmethod
    def loopback(cls, n: int, precision: str, world: int) -> "State":
        """All `world` shards of a sharded state in this process / GPU (validation)."""
        h = ctypes.c_void_p()
        _check(lib().qc_state_create_loopback(n, PRECISION[precision], world, ctypes.byref(h)))
        return cls(n, precision, _handle=h)

    @classmethod
    def dist(cls, n: int, precision: str, rank: int, world: int, nccl_id: bytes) -> "State":
        """This rank's shard (one process per GPU, NCCL); collective."""
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().qc_state_create_dist(n, PRECISION[precision], rank, world, idbuf, ctypes.byref(h)))
        return cls(n, precision, _handle=h)

    @classmethod
    def wrap(cls, n: int, precision: str, dev_ptr: int, stream: Optional[int] = None) -> "State":
        h = ctypes.c_void_p()
        _check(lib().qc_state_wrap(n, PRECISION[precision], dev_ptr, stream, ctypes.byref(h)))
        return cls(n, precision, _handle=h)

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib().qc_state_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- init
    def init_random(self, seed: int):
        _check(lib().qc_state_init_random(self._h, seed))

    def init_basis(self, k: int):
        _check(lib().qc_state_init_basis(self._h, k))

    # -- the path
    def apply_gate(self, name: str, qubits: Sequence[int], matrix=None):
        q = (ctypes.c_int * 3)(*(list(qubits) + [0] * (3 - len(qubits))))
        mp = None
        if matrix is not None:
            m = np.asarray(matrix)
            if np.iscomplexobj(m):
                m = np.ascontiguousarray(np.stack([m.real, m.imag], -1).reshape(-1), dtype=np.float64)
            else:
                m = np.ascontiguousarray(m, dtype=np.float64).reshape(-1)
            self._keep = m
            mp = m.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        _check(lib().qc_apply_gate(self._h, OPS[name], q, mp))

    def run(self, ops) -> None:
        arr = ops if isinstance(ops, np.ndarray) else encode_ops(ops)
        mt = getattr(arr, "mtab", None)
        arr = np.ascontiguousarray(arr)
        if mt is None:
            _check(lib().qc_run_circuit(self._h, arr.ctypes.data if len(arr) else None, len(arr)))
        else:
            _check(lib().qc_run_circuit_ex(self._h, arr.ctypes.data if len(arr) else None, len(arr),
                                           mt.ctypes.data, len(mt)))

    def apply_mgate(self, qubits: Sequence[int], matrix, n_ctrl: int = 0, ctrl_state: Optional[int] = None):
        """One generic gate (controls first in ``qubits``) via qc_apply_mgate."""
        import types
        op = types.SimpleNamespace(qubits=tuple(qubits), nctrl=n_ctrl, matrix=matrix,
                                   ctrl_state=(1 << n_ctrl) - 1 if ctrl_state is None else ctrl_state)
        keep = []
        g = encode_mgate(op, keep)
        _check(lib().qc_apply_mgate(self._h, g.ctypes.data))

    # -- I/O
    def read(self, first: int = 0, count: Optional[int] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
        if count is None:
            count = (1 << self.n) - first
        if out is None:
            out = np.empty(count, dtype=self.dtype)
        _check(lib().qc_state_read(self._h, first, count, out.ctypes.data))
        return out

    def write(self, arr: np.ndarray, first: int = 0):
        a = np.ascontiguousarray(arr, dtype=self.dtype)
        _check(lib().qc_state_write(self._h, first, a.size, a.ctypes.data))

    def write_ptr(self, host_ptr: int, count: int, first: int = 0):
        _check(lib().qc_state_write(self._h, first, count, host_ptr))

    def read_ptr(self, host_ptr: int, count: int, first: int = 0):
        _check(lib().qc_state_read(self._h, first, count, host_ptr))

    def readwrite_ptr(self, dst_ptr: int, src_ptr: int, count: int, first: int = 0):
        """qc_state_readwrite: read [first, +count) into dst, upload src in its place."""
        _check(lib().qc_state_readwrite(self._h, first, count, dst_ptr, src_ptr))

    def exchange(self, g: int, l: int):
        """One qubit-swap exchange of physical rank bit g with local bit l (debug)."""
        _check(lib().qc_debug_exchange(self._h, g, l))

    def canonicalize(self):
        _check(lib().qc_state_canonicalize(self._h))

    def sync(self):
        _check(lib().qc_state_sync(self._h))

    def norm2(self) -> float:
        v = ctypes.c_double()
        _check(lib().qc_state_norm2(self._h, ctypes.byref(v)))
        return v.value

    def set_option(self, name: str, value: int):
        _check(lib().qc_set_option(self._h, OPTIONS[name], int(value)))

    def info(self) -> dict:
        i = qc_info()
        _check(lib().qc_get_info(self._h, ctypes.byref(i)))
        return {"n": i.n, "precision": i.precision, "device_ptr": i.device_ptr, "stream": i.stream,
                "layout": list(i.layout[: i.n]), "layout_is_canonical": bool(i.layout_is_canonical),
                "last_gates": i.last_gates, "last_passes": i.last_passes,
                "last_launches": i.last_launches, "last_relabels": i.last_relabels,
                "last_graph": bool(i.last_graph), "tile_bits": i.tile_bits,
                "last_blocks": i.last_blocks, "last_jit": bool(i.last_jit), "world": i.world,
                "rank": i.rank, "n_local": i.n_local, "sharding": i.sharding,
                "last_exchanges": i.last_exchanges, "last_flops_per_amp": i.last_flops_per_amp,
                "last_pair_segments": i.last_pair_segments}

    @property
    def stream(self) -> int:
        return self.info()["stream"] or 0


def debug_plan(n: int, ops, precision: str = "c128", tile_bits: int = 0, block_fusion: bool = True,
               compile_jit: bool = False, row_bits: int = 0, remap: bool = True) -> dict:
    """Plan an op list on the host (no GPU) and report its shape; optionally
    NVRTC-compile every pass's specialised kernel (qc_debug.h)."""
    arr = ops if isinstance(ops, np.ndarray) else encode_ops(ops)
    arr = np.ascontiguousarray(arr)
    st = qc_plan_stats()
    eb = ctypes.create_string_buffer(4096)
    rc = lib().qc_debug_plan(n, PRECISION[precision], arr.ctypes.data if len(arr) else None, len(arr),
                             tile_bits, row_bits, int(block_fusion), int(remap), int(compile_jit),
                             ctypes.byref(st),
                             eb, 4096)
    if rc != QC_OK:
        raise QCError(rc, eb.value.decode())
    return {f: getattr(st, f) for f, _ in qc_plan_stats._fields_}


def debug_box_layout(tile_set: int, nbits: int, dbl: bool = True):
    """(starts[0..dims], boxbits[0..dims), xmask) of a tile's TMA box layout, or None."""
    dims = ctypes.c_int(0)
    starts = np.zeros(8, dtype=np.int32)
    boxbits = np.zeros(8, dtype=np.int32)
    xm = ctypes.c_uint32(0)
    rc = lib().qc_debug_box_layout(tile_set, nbits, int(dbl), ctypes.byref(dims), starts.ctypes.data,
                                   boxbits.ctypes.data, ctypes.byref(xm))
    if rc == QC_ERR_UNSUPPORTED:
        return None
    _check(rc)
    return [int(x) for x in starts[:dims.value + 1]], [int(x) for x in boxbits[:dims.value]], int(xm.value)


def fma_peak(dbl: bool = True) -> float:
    """Measured FMA throughput of the current device, TFLOP/s (qc_debug.h)."""
    v = ctypes.c_double(0.0)
    rc = lib().qc_debug_fma_peak(int(dbl), ctypes.byref(v))
    if rc != QC_OK:
        raise QCError(rc, lib().qc_last_error().decode())
    return v.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().qc_nccl_unique_id(buf))
    return buf.raw


def debug_exchange_runs(n_loc: int, rank: int, g: int, l: int):
    """(partner, [(offset, count), ...]) of a qubit-swap exchange (host only)."""
    partner, nr = ctypes.c_int(), ctypes.c_int()
    cap = 1 << 16
    offs = np.zeros(cap, dtype=np.uint64)
    cnts = np.zeros(cap, dtype=np.uint64)
    _check(lib().qc_debug_exchange_runs(n_loc, rank, g, l, ctypes.byref(partner), offs.ctypes.data,
                                        cnts.ctypes.data, cap, ctypes.byref(nr)))
    return partner.value, [(int(offs[i]), int(cnts[i])) for i in range(min(nr.value, cap))]


def debug_dist_schedule(n: int, world: int, ops, relabel: bool = True, exchange: int = 0):
    """Host-only sharded schedule: ([(kind, g, l, gates)], final layout); kind 0
    local segment, 1 exchange, 2 pair segment (exchange mode 2)."""
    arr = ops if isinstance(ops, np.ndarray) else encode_ops(ops)
    arr = np.ascontiguousarray(arr)
    cap = 1 << 14
    steps = np.zeros(4 * cap, dtype=np.int32)
    lay = np.zeros(64, dtype=np.int32)
    ns = ctypes.c_int()
    _check(lib().qc_debug_dist_schedule_ex(n, world, int(relabel), int(exchange), arr.ctypes.data if len(arr) else None,
                                        len(arr), steps.ctypes.data, cap, ctypes.byref(ns), lay.ctypes.data))
    out = [tuple(int(x) for x in steps[4 * i:4 * i + 4]) for i in range(min(ns.value, cap))]
    return out, [int(x) for x in lay[:n]]


def debug_group_split(n: int, world: int, tile_bits_set: int, rank: int):
    """Group-plan tile split of one pass (host): (tile0, count, j, owners)."""
    t0, cnt, j = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int()
    own = (ctypes.c_int * 8)()
    _check(lib().qc_debug_group_split(n, world, tile_bits_set, rank, ctypes.byref(t0), ctypes.byref(cnt),
                                      ctypes.byref(j), own))
    return t0.value, cnt.value, j.value, [own[h] for h in range(1 << j.value)]


def version() -> str:
    return lib().qc_version().decode()
