"""The paper's CPU OpenMP program (libqc_omp.so) vs the CPU
oracle: same gate semantics, so the same tolerances as the GPU path (1e-12
c128, 1e-5 c64; permutation circuits bit-exact).  Runs without a GPU."""
import json
import os

import numpy as np
import pytest

import oracle
import qcgen
from qcgen import Op
from paper_2303_00123_b200 import cpu_omp

TOL = {"c128": 1e-12, "c64": 1e-5}
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def run_omp(n, prec, ops, state, nthreads=0):
    x = np.ascontiguousarray(state.astype(np.complex128 if prec == "c128" else np.complex64))
    cpu_omp.qc_omp_run(n, prec, x, ops, nthreads)
    return x


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("n", [2, 3, 5, 9, 12])
def test_random_circuits_match_oracle(prec, n):
    ops = qcgen.random_circuit(n, 150, seed=40 + n)
    st = qcgen.random_state(n, seed=n, precision=prec)
    got = run_omp(n, prec, ops, st)
    exp = oracle.run(n, st, ops)
    assert np.abs(got.astype(np.complex128) - exp).max() < TOL[prec] * 10


@pytest.mark.parametrize("n", [4, 11])
def test_permutation_circuits_bit_exact(n):
    ops = qcgen.random_circuit(n, 200, seed=3, kinds=("X", "CNOT", "SWAP", "CCX"))
    st = qcgen.random_state(n, seed=1)
    assert np.array_equal(run_omp(n, "c128", ops, st), oracle.run(n, st, ops))


def test_paper_index_tables():
    """fig:1q / fig:ctrl-1q / fig:dctrl-1q:
    X moves |a_j> to |b_j>, CNOT and CCX swap exactly the printed pairs."""
    T = json.load(open(os.path.join(GOLD, "fig_index_tables.json")))
    e = lambda k: np.eye(8, dtype=complex)[k]
    for c in T["fig_1q"]["cases"]:
        for a, b in zip(c["a"], c["b"]):
            assert np.array_equal(run_omp(3, "c128", [Op("X", (c["q"],))], e(a)), e(b))
    for c in T["fig_ctrl_1q"]["cases"]:
        for a, b in zip(c["a"], c["b"]):
            got = run_omp(3, "c128", [Op("CNOT", (c["qc"], c["qt"]), ctrl_state=c["ctrl"])], e(a))
            assert np.array_equal(got, e(b))
    c = T["fig_dctrl_1q"]["cases"][0]
    for x in range(8):
        got = run_omp(3, "c128", [Op("CCX", tuple(c["qc"]) + (c["qt"],))], e(x))
        y = c["b"][0] if x in c["a"] else c["a"][0] if x in c["b"] else x
        assert np.array_equal(got, e(y))


@pytest.mark.parametrize("circ", ["qft", "tfxy"])
def test_paper_workloads(circ):
    n = 10
    ops = qcgen.qft(n) if circ == "qft" else qcgen.tfxy(n, 3)
    st = qcgen.random_state(n)
    assert np.abs(run_omp(n, "c128", ops, st) - oracle.run(n, st, ops)).max() < 1e-12


def test_thread_counts_agree():
    n = 12
    ops = qcgen.random_circuit(n, 60, seed=9)
    st = qcgen.random_state(n, seed=2)
    a = run_omp(n, "c128", ops, st, nthreads=1)
    b = run_omp(n, "c128", ops, st, nthreads=4)
    assert np.array_equal(a, b)  # each amplitude is written by one iteration: order-independent
    assert cpu_omp.qc_omp_max_threads() >= 1


def test_validation_and_generic_gates_rejected():
    from paper_2303_00123_b200.qc import QCError
    st = qcgen.random_state(4)
    x = st.copy()
    with pytest.raises(QCError):
        cpu_omp.qc_omp_run(4, "c128", x, [Op("H", (0,)), Op("CNOT", (1, 1))])
    assert np.array_equal(x, st)  # validated before any work
    with pytest.raises(QCError):
        cpu_omp.qc_omp_run(4, "c128", x, [Op("MCU", (0,), matrix=np.eye(2), nctrl=0)])
    with pytest.raises(ValueError):
        cpu_omp.qc_omp_run(4, "c64", x, [Op("H", (0,))])  # dtype mismatch


def test_library_is_separate_from_the_gpu_path():
    """The CPU program and libqc.so do not load each other (no CPU fallback)."""
    import subprocess
    here = os.path.dirname(cpu_omp.LIB_PATH)
    for so, other in (("libqc_omp.so", "libqc.so"), ("libqc.so", "libqc_omp.so")):
        out = subprocess.run(["readelf", "-d", os.path.join(here, so)], capture_output=True, text=True).stdout
        assert other not in out
