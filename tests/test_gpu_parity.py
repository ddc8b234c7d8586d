"""GPU path vs the CPU oracle, through the C ABI (libqc.so).

Tolerances (north star / BASELINE.json): max |amplitude error| <= 1e-12 for
complex128, <= 1e-5 for complex64; permutation circuits (X/CNOT/SWAP/CCX)
bit-exact.  Inputs are seeded (qcgen); the oracle never sees device data.
"""
import json
import os

import numpy as np
import pytest

import oracle
import qcgen
from qcgen import Op

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def qcmod():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2303_00123_b200 as pkg
    pkg.lib()
    return pkg


def gpu_run(pkg, n, prec, ops, seed=qcgen.STATE_SEED, state=None, **opts):
    with pkg.State(n, prec) as s:
        for k, v in opts.items():
            s.set_option(k, v)
        if state is None:
            s.init_random(seed)
        else:
            s.write(state)
        s.run(ops)
        out = s.read()
        info = s.info()
    return out, info


def ref_run(n, prec, ops, seed=qcgen.STATE_SEED, state=None):
    st = qcgen.random_state(n, seed=seed, precision=prec) if state is None else state
    return oracle.run(n, st, ops)


def maxerr(a, b):
    return float(np.abs(a.astype(np.complex128) - b).max()) if a.size else 0.0


# -------------------------------------------------------------- generator
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("n", [1, 5, 10, 17])
def test_device_random_state_is_bit_identical(qcmod, prec, n):
    with qcmod.State(n, prec) as s:
        s.init_random(qcgen.STATE_SEED)
        got = s.read()
    ref = qcgen.random_state(n, precision=prec)
    assert got.dtype == ref.dtype and np.array_equal(got.view(np.uint8), ref.view(np.uint8))


# ---------------------------------------------------------- per-gate path
@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_every_gate_every_position_unfused(qcmod, prec):
    """qc_apply_gate: each kind on every qubit / ordered pair (all stride classes)."""
    n = 7
    rng = np.random.default_rng(1)
    phi = qcgen.random_state(n, seed=2, precision=prec)
    V = qcgen.random_unitary(2, rng)
    W = qcgen.random_unitary(4, rng)
    cases = []
    for q in range(n):
        for name in ("H", "X", "Y", "Z"):
            cases.append((name, (q,), None))
        for name in ("P", "RX", "RY", "RZ"):
            cases.append((name, (q,), float(rng.uniform(-7, 7))))
        cases.append(("U1", (q,), V))
    for a in range(n):
        for b in range(n):
            if a == b:
                continue
            cases += [("CNOT", (a, b), None), ("CZ", (a, b), None),
                      ("CP", (a, b), float(rng.uniform(-7, 7))), ("CU1", (a, b), V),
                      ("U2", (a, b), W)]
            if a < b:
                cases.append(("SWAP", (a, b), None))
    for c0, c1, t in ((0, 1, 2), (6, 0, 3), (2, 5, 1), (4, 3, 6)):
        cases.append(("CCX", (c0, c1, t), None))
    with qcmod.State(n, prec) as s:
        s.set_option("relabel_swap", 0)
        for name, qs, arg in cases:
            s.write(phi)
            if arg is None:
                s.apply_gate(name, qs)
                op = Op(name, qs)
            elif isinstance(arg, float):
                s.apply_gate(name, qs, np.array([arg]))
                op = Op(name, qs, theta=arg)
            else:
                s.apply_gate(name, qs, arg)
                op = Op(name, qs, matrix=arg)
            got = s.read()
            ref = oracle.run(n, phi, [op])
            if name in ("X", "CNOT", "SWAP", "CCX"):
                assert np.array_equal(got.astype(np.complex128), ref), (name, qs)
            else:
                assert maxerr(got, ref) <= TOL[prec], (name, qs, maxerr(got, ref))


@pytest.mark.parametrize("fusion", [0, 1])
def test_paper_index_tables_on_gpu(qcmod, fusion):
    """fig:1q / fig:ctrl-1q / fig:dctrl-1q
    through the device path, n=3 (fusion needs n>=4: n=3 runs unfused)."""
    with open(os.path.join(GOLD, "fig_index_tables.json")) as f:
        tab = json.load(f)
    n = 3

    def basis(k):
        v = np.zeros(8, complex)
        v[k] = 1
        return v

    for c in tab["fig_1q"]["cases"]:
        for a, b in zip(c["a"], c["b"]):
            out, _ = gpu_run(qcmod, n, "c128", [Op("X", (c["q"],))], state=basis(a), fusion=fusion)
            assert np.array_equal(out, basis(b))
    for c in tab["fig_ctrl_1q"]["cases"]:
        for a, b in zip(c["a"], c["b"]):
            out, _ = gpu_run(qcmod, n, "c128", [Op("CNOT", (c["qc"], c["qt"]), ctrl_state=c["ctrl"])],
                             state=basis(a), fusion=fusion)
            assert np.array_equal(out, basis(b))
    c = tab["fig_dctrl_1q"]["cases"][0]
    for x in range(8):
        out, _ = gpu_run(qcmod, n, "c128", [Op("CCX", tuple(c["qc"]) + (c["qt"],))],
                         state=basis(x), fusion=fusion)
        exp = {6: 7, 7: 6}.get(x, x)
        assert np.array_equal(out, basis(exp))


# ---------------------------------------------------------- random circuits
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("n,tile_bits", [(4, 0), (5, 4), (8, 0), (8, 5), (11, 6), (12, 0),
                                         (13, 7), (14, 0), (16, 9), (18, 0)])
def test_random_circuits_fused(qcmod, prec, n, tile_bits):
    ops = qcgen.random_circuit(n, 200, seed=100 + n)
    got, info = gpu_run(qcmod, n, prec, ops, tile_bits=tile_bits)
    ref = ref_run(n, prec, ops)
    assert maxerr(got, ref) <= TOL[prec], (maxerr(got, ref), info)


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("n", [2, 6, 13])
def test_random_circuits_unfused(qcmod, prec, n):
    ops = qcgen.random_circuit(n, 200, seed=300 + n)
    got, _ = gpu_run(qcmod, n, prec, ops, fusion=0)
    assert maxerr(got, ref_run(n, prec, ops)) <= TOL[prec]


@pytest.mark.parametrize("fusion", [0, 1])
@pytest.mark.parametrize("relabel", [0, 1])
@pytest.mark.parametrize("n,tile_bits", [(6, 0), (12, 0), (15, 8)])
def test_permutation_circuits_bit_exact(qcmod, fusion, relabel, n, tile_bits):
    ops = qcgen.random_circuit(n, 300, seed=7 + n, kinds=("X", "CNOT", "SWAP", "CCX"))
    for prec in ("c128", "c64"):
        got, _ = gpu_run(qcmod, n, prec, ops, fusion=fusion, relabel_swap=relabel, tile_bits=tile_bits)
        ref = ref_run(n, prec, ops)
        assert np.array_equal(got.astype(np.complex128), ref)


# ---------------------------------------------------------- paper workloads
@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_qft_c1_n10(qcmod, prec):
    """Config C1: QFT on 10 qubits, random initial state (both signs)."""
    n = 10
    for sign in (-1, +1):
        ops = qcgen.qft(n, sign=sign)
        got, info = gpu_run(qcmod, n, prec, ops)
        assert maxerr(got, ref_run(n, prec, ops)) <= TOL[prec]
        assert info["last_passes"] == 1  # whole circuit in one launch (n <= tile)


def test_tfxy_c2_n20_s10(qcmod):
    """Config C2: TFXY 1D Trotter circuit, 20 qubits, 10 steps, complex double."""
    n = 20
    ops = qcgen.tfxy(n, 10)
    got, info = gpu_run(qcmod, n, "c128", ops)
    assert maxerr(got, ref_run(n, "c128", ops)) <= 1e-12
    assert info["last_gates"] == 1178


@pytest.mark.parametrize("n", [14, 17])
def test_qft_multi_pass_with_relabel(qcmod, n):
    ops = qcgen.qft(n)
    got, info = gpu_run(qcmod, n, "c128", ops)
    assert info["last_relabels"] == n // 2 and not info["layout_is_canonical"]
    assert maxerr(got, ref_run(n, "c128", ops)) <= 1e-12


def test_tfxy_parity_sector_exact_zero_on_gpu(qcmod):
    n = 16
    st = qcgen.random_state_even_parity(n, seed=5)
    got, _ = gpu_run(qcmod, n, "c128", qcgen.tfxy(n, 3), state=st)
    w = np.array([bin(i).count("1") & 1 for i in range(1 << n)])
    assert np.all(got[w == 1] == 0)


# ---------------------------------------------------------- state plumbing
def test_graph_replay_matches(qcmod):
    n = 15
    ops = qcgen.random_circuit(n, 120, seed=42)
    inv = qcgen.inverse(ops)
    with qcmod.State(n, "c128") as s:
        s.init_random(1)
        ref0 = s.read()
        for _ in range(3):  # 1st run direct, 2nd+ graph replay
            s.run(ops)
            s.run(inv)
        assert s.info()["last_graph"]
        assert maxerr(s.read(), ref0) <= 1e-12


def test_read_write_ranges_and_canonicalize(qcmod):
    n = 12
    with qcmod.State(n, "c128") as s:
        s.init_random(9)
        s.run(qcgen.qft(n))
        full = s.read()
        assert not s.info()["layout_is_canonical"]
        part = s.read(100, 333)
        assert np.array_equal(part, full[100:433])
        x = (np.arange(50) + 1j).astype(np.complex128)
        s.write(x, first=1000)
        full[1000:1050] = x
        assert np.array_equal(s.read(), full)
        s.canonicalize()
        assert s.info()["layout_is_canonical"]
        assert np.array_equal(s.read(), full)
        ref_n2 = np.vdot(full, full).real
        assert abs(s.norm2() - ref_n2) <= 1e-14 * ref_n2


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_readwrite_overlapped_copies(qcmod, prec):
    """qc_state_readwrite == read then write (chunks of 256 MiB: n=25 c128 is
    2 chunks + a tail of 0; n=26 c64 has 2), distinct and identical host
    buffers, canonical and relabelled layouts."""
    dt = np.complex128 if prec == "c128" else np.complex64
    n = 25 if prec == "c128" else 26
    with qcmod.State(n, prec) as s:
        s.init_random(4)
        before = s.read()
        src = (np.arange(1 << n) * (1 + 0.5j)).astype(dt)
        dst = np.zeros(1 << n, dtype=dt)
        s.readwrite_ptr(dst.ctypes.data, src.ctypes.data, 1 << n)
        assert np.array_equal(dst, before) and np.array_equal(s.read(), src)
        # identical buffer: upload what was just read (a round trip), sub-range
        buf = np.zeros(3000, dtype=dt)
        s.readwrite_ptr(buf.ctypes.data, buf.ctypes.data, 3000, 777)
        assert np.array_equal(buf, src[777:3777]) and np.array_equal(s.read(), src)
    with qcmod.State(12, prec) as s:  # non-canonical layout (QFT relabels)
        s.init_random(9)
        s.run(qcgen.qft(12))
        full = s.read()
        x = np.full(50, 2 - 1j, dtype=dt)
        got = np.zeros(50, dtype=dt)
        s.readwrite_ptr(got.ctypes.data, x.ctypes.data, 50, 1000)
        full_new = full.copy()
        full_new[1000:1050] = x
        assert np.array_equal(got, full[1000:1050]) and np.array_equal(s.read(), full_new)


def test_invalid_ops_leave_state_unchanged(qcmod):
    from paper_2303_00123_b200 import QCError
    n = 6
    with qcmod.State(n, "c128") as s:
        s.init_random(3)
        before = s.read()
        bad = [Op("H", (0,)), Op("CNOT", (1, 2))]
        arr = qcmod.encode_ops(bad)
        arr[1]["qubits"][1] = 1  # repeated qubit
        with pytest.raises(QCError) as e:
            s.run(arr)
        assert e.value.status == 1
        arr = qcmod.encode_ops(bad)
        arr[1]["qubits"][0] = 6  # out of range
        with pytest.raises(QCError):
            s.run(arr)
        with pytest.raises(QCError):
            s.run([Op("RX", (0,), theta=float("inf"))])
        assert np.array_equal(s.read(), before)


def test_norm_preserved_and_inverse(qcmod):
    n = 20
    ops = qcgen.random_circuit(n, 150, seed=11)
    with qcmod.State(n, "c128") as s:
        s.init_random(2)
        n0 = s.norm2()
        s.run(ops)
        assert abs(s.norm2() - n0) < 1e-12
        s.run(qcgen.inverse(ops))
        s.canonicalize()
        ref = qcgen.random_state(n, seed=2)
        assert maxerr(s.read(), ref) <= 1e-12


# ---------------------------------------------------------- NVRTC-specialised passes
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("n,tile_bits", [(5, 4), (10, 0), (14, 7), (17, 9), (19, 0)])
def test_random_circuits_jit(qcmod, prec, n, tile_bits):
    ops = qcgen.random_circuit(n, 200, seed=500 + n)
    got, info = gpu_run(qcmod, n, prec, ops, tile_bits=tile_bits, jit=2)
    assert info["last_jit"], info
    assert maxerr(got, ref_run(n, prec, ops)) <= TOL[prec]


def test_permutation_circuit_jit_bit_exact(qcmod):
    n = 15
    ops = qcgen.random_circuit(n, 300, seed=77, kinds=("X", "CNOT", "SWAP", "CCX"))
    for prec in ("c128", "c64"):
        got, info = gpu_run(qcmod, n, prec, ops, tile_bits=8, jit=2, relabel_swap=0)
        assert info["last_jit"]
        assert np.array_equal(got.astype(np.complex128), ref_run(n, prec, ops))


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_paper_workloads_jit(qcmod, prec):
    for n, ops in ((10, qcgen.qft(10)), (16, qcgen.qft(16)), (20, qcgen.tfxy(20, 10))):
        got, info = gpu_run(qcmod, n, prec, ops, jit=2)
        assert info["last_jit"]
        assert maxerr(got, ref_run(n, prec, ops)) <= TOL[prec], (n, prec)


def test_jit_default_policy_second_run(qcmod):
    """Default policy: 1st run interprets, 2nd run specialises (then graphs)."""
    n = 16
    ops = qcgen.tfxy(n, 3)
    inv = qcgen.inverse(ops)
    with qcmod.State(n, "c128") as s:
        s.init_random(4)
        s.run(ops)
        assert not s.info()["last_jit"]
        s.run(inv)
        s.run(ops)
        assert s.info()["last_jit"]
        s.run(inv)
        got = s.read()
    assert maxerr(got, qcgen.random_state(n, seed=4)) <= 1e-12


# ---------------------------------------------------------- stress (pipeline races)
@pytest.mark.parametrize("n,prec,rb", [(26, "c128", 5), (26, "c128", 6), (26, "c64", 6), (25, "c128", 7)])
def test_repeated_runs_roundtrip(qcmod, n, prec, rb):
    """Many fused runs (JIT + graph replay) of QFT and its inverse: every
    pipeline launch must complete (device watchdog traps a deadlock) and the
    state must come back."""
    ops = qcgen.qft(n)
    with qcmod.State(n, prec) as s:
        s.set_option("row_bits", rb)
        s.init_random(3)
        n0 = s.norm2()
        arr, inv = qcmod.encode_ops(ops), qcmod.encode_ops(qcgen.inverse(ops))
        for _ in range(8):
            s.run(arr)
            s.run(inv)
        assert s.info()["last_jit"] and s.info()["last_graph"]
        s.canonicalize()
        got = s.read(0, 1 << 12)
        assert abs(s.norm2() - n0) <= (1e-9 if prec == "c128" else 1e-4) * n0
    ref = qcgen.random_state(n, seed=3, precision=prec)[: 1 << 12]
    assert maxerr(got, ref) <= TOL[prec] * 10


# ---------------------------------------------------------- remap (row-bit relabelling between passes)
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("n,tile_bits,circ", [(16, 0, "tfxy"), (18, 9, "tfxy"), (17, 8, "random"),
                                              (20, 0, "random"), (15, 7, "qft")])
def test_remap_matches_oracle_and_restores_layout(qcmod, prec, n, tile_bits, circ):
    """Passes that end by swapping row bits with tile bits (QC_OPT_REMAP) give
    the oracle's result, and the run leaves the layout it started with."""
    ops = {"tfxy": lambda: qcgen.tfxy(n, 4), "qft": lambda: qcgen.qft(n),
           "random": lambda: qcgen.random_circuit(n, 300, seed=900 + n)}[circ]()
    ref = ref_run(n, prec, ops)
    rb = 6 if prec == "c128" else 7  # fixed 1 KiB rows: the remap path is what is under test
    for jit in (0, 2):
        with qcmod.State(n, prec) as s:
            s.set_option("tile_bits", tile_bits)
            s.set_option("row_bits", rb)
            s.set_option("jit", jit)
            s.set_option("relabel_swap", 0)  # so the only relabelling is the remap
            s.init_random(qcgen.STATE_SEED)
            s.run(ops)
            info = s.info()
            got = s.read()
        assert info["layout_is_canonical"], info
        assert maxerr(got, ref) <= TOL[prec], (jit, maxerr(got, ref))
    st = qcmod.qc.debug_plan(n, ops, precision=prec, tile_bits=tile_bits, row_bits=rb)
    if circ != "qft":
        assert st["remap_swaps"] > 0, st


def test_remap_permutation_circuit_bit_exact(qcmod):
    n = 18
    ops = qcgen.random_circuit(n, 400, seed=78, kinds=("X", "CNOT", "SWAP", "CCX"))
    for prec in ("c128", "c64"):
        got, info = gpu_run(qcmod, n, prec, ops, tile_bits=8, jit=2)
        assert np.array_equal(got.astype(np.complex128), ref_run(n, prec, ops))


def test_fma_peak_measurement(qcmod):
    """The ALU roofline denominator bench.py reports (qc_debug_fma_peak)."""
    p64 = qcmod.qc.fma_peak(True)
    p32 = qcmod.qc.fma_peak(False)
    assert 10.0 < p64 < 200.0, p64
    assert p32 > p64, (p32, p64)


def test_qasm_program_on_gpu(qcmod):
    """A circuit read from openQASM 2.0 text (qc_qasm_parse) runs through the
    fused engine and matches the oracle on the same parsed list."""
    n = 14
    txt = qcmod.qc.qasm_emit(n, qcgen.qft(n) + qcgen.tfxy(n, 2))
    n2, arr = qcmod.qc.qasm_parse(txt)
    assert n2 == n
    names = {v: k for k, v in qcmod.qc.OPS.items()}
    ops = []
    for g in arr:
        name = names[int(g["op"])]
        k = qcgen.ARITY[name]
        ops.append(Op(name, tuple(int(q) for q in g["qubits"][:k]),
                      theta=float(g["theta"]) if name in qcgen.THETA_OPS else None))
    for prec in ("c128", "c64"):
        with qcmod.State(n, prec) as s:
            s.init_random(qcgen.STATE_SEED)
            s.run(arr)
            got = s.read()
        assert maxerr(got, ref_run(n, prec, ops)) <= TOL[prec]


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("tma,rb", [(0, 0), (0, 2), (0, 3), (0, 4), (2, 6), (1, 5)])
def test_tile_transports_match_oracle(qcmod, prec, tma, rb):
    """Every tile transport (0: one TMA box per tile -- several when a tile
    has > 5 bit runs, narrow rows; 2: gather4 rows; 1: one bulk copy per row)
    and row width gives the oracle's result on QFT, TFXY and random circuits,
    interpreting (1st run) and NVRTC (2nd) kernels."""
    for n, ops in ((19, qcgen.qft(19)), (20, qcgen.tfxy(20, 6)), (18, qcgen.random_circuit(18, 250, seed=21))):
        ref = ref_run(n, prec, ops)
        with qcmod.State(n, prec) as s:
            s.set_option("tma_mode", tma)
            s.set_option("row_bits", rb)
            for _ in range(2):
                s.init_random(qcgen.STATE_SEED)
                s.run(ops)
                assert maxerr(s.read(), ref) <= TOL[prec], (n, tma, rb)
