"""Generic gates (multi-controlled, k-target dense,
P:942-978) on the GPU vs the CPU oracle's orc_run_general, through the C ABI
(qc_run_circuit_ex / qc_apply_mgate).

Tolerances as tests/test_gpu_parity.py (1e-12 c128, 1e-5 c64); generic
permutation matrices under controls are pure moves, so circuits of them are
bit-exact."""
import numpy as np
import pytest

import oracle
import qcgen
from qcgen import Op

pytestmark = pytest.mark.gpu

TOL = {"c128": 1e-12, "c64": 1e-5}


@pytest.fixture(scope="module")
def pkg():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2303_00123_b200 as p
    p.lib()
    return p


def run_gpu(pkg, n, prec, ops, seed=qcgen.STATE_SEED, reps=1, **opts):
    with pkg.State(n, prec) as s:
        for k, v in opts.items():
            s.set_option(k, v)
        arr = pkg.encode_ops(ops)
        out = None
        for _ in range(reps):  # reps: 2nd use JIT-specialises, 3rd replays the graph
            s.init_random(seed)
            s.run(arr)
            out = s.read()
        return out, s.info()


def ref(n, prec, ops, seed=qcgen.STATE_SEED):
    return oracle.run(n, qcgen.random_state(n, seed=seed, precision=prec), ops)


def err(a, b):
    return float(np.abs(a.astype(np.complex128) - b).max())


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_apply_mgate_every_shape(pkg, prec):
    """qc_apply_mgate (per-gate kernels): 1..4 targets x 0..5 controls, random
    qubit order and control states, one gate at a time vs the oracle."""
    n = 9
    rng = np.random.default_rng(31)
    phi = qcgen.random_state(n, seed=4, precision=prec)
    with pkg.State(n, prec) as s:
        s.write(phi)
        cur = phi.astype(np.complex128)
        for k in (1, 2, 3, 4):
            for c in (0, 1, 2, 5):
                qs = tuple(int(q) for q in rng.choice(n, size=k + c, replace=False))
                U = qcgen.random_unitary(1 << k, rng)
                cs = int(rng.integers(1 << c))
                s.apply_mgate(qs, U, n_ctrl=c, ctrl_state=cs)
                cur = oracle.run(n, cur, [Op("MCU", qs, matrix=U, nctrl=c, ctrl_state=cs)])
                assert err(s.read(), cur) < TOL[prec] * 4, (k, c, qs, cs)


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("n,tile_bits,fusion", [(6, 0, 0), (6, 0, 1), (11, 0, 1), (13, 7, 1), (16, 0, 1),
                                                (20, 0, 1)])
def test_random_mcu_circuits(pkg, prec, n, tile_bits, fusion):
    """Mixed named + generic gates (0..4 controls, 1..4 targets) through the
    fused planner (AOT interpreter on the 1st run, NVRTC kernels on the 2nd,
    CUDA graph on the 3rd) and the per-gate path."""
    ops = qcgen.random_mcu_circuit(n, 120, seed=n + 17 * tile_bits, max_ctrl=4)
    exp = ref(n, prec, ops)
    for reps in (1, 2, 3):
        got, info = run_gpu(pkg, n, prec, ops, reps=reps, fusion=fusion, tile_bits=tile_bits)
        assert err(got, exp) < TOL[prec] * 10, (reps, info["last_passes"])


@pytest.mark.parametrize("n", [8, 14])
def test_mcu_permutations_bit_exact(pkg, n):
    """Multi-controlled permutation matrices (X under k controls, shuffles of 2-4
    targets) move amplitudes only: bit-exact on every path."""
    ops = qcgen.random_mcu_circuit(n, 80, seed=5, max_ctrl=5, perm_frac=1.0,
                                   mix=("X", "CNOT", "SWAP", "CCX"))
    exp = ref(n, "c128", ops)
    for fusion in (0, 1):
        for reps in (1, 2):
            got, _ = run_gpu(pkg, n, "c128", ops, reps=reps, fusion=fusion)
            assert np.array_equal(got, exp), (fusion, reps)


def test_fig_dctrl_1q_generic_u_on_gpu(pkg):
    """fig:dctrl-1q: a doubly controlled generic U on (0,1 | 2) at
    n=3 changes only amplitudes 6 and 7."""
    V = qcgen.random_unitary(2, np.random.default_rng(2))
    for fusion in (0, 1):
        for x in range(8):
            with pkg.State(3, "c128") as s:
                s.set_option("fusion", fusion)
                s.init_basis(x)
                s.run([Op("MCU", (0, 1, 2), matrix=V, nctrl=2)])
                got = s.read()
            exp = np.zeros(8, complex)
            if x in (6, 7):
                exp[6], exp[7] = V[0, x - 6], V[1, x - 6]
            else:
                exp[x] = 1
            assert err(got, exp) < 1e-15


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_mcu_sharded_loopback(pkg, prec):
    """Generic gates on a sharded state (loopback: 4 shards on one GPU):
    controls on rank bits are rank predicates, targets on rank bits trigger
    qubit-swap exchanges."""
    n = 14
    ops = qcgen.random_mcu_circuit(n, 60, seed=9, max_ctrl=3)
    exp = ref(n, prec, ops, seed=3)
    with pkg.State.loopback(n, prec, 4) as s:
        s.init_random(3)
        s.run(ops)
        got = s.read()
        assert s.info()["last_exchanges"] >= 0
    assert err(got, exp) < TOL[prec] * 10


def test_mcu_plan_cache_keyed_by_matrix_contents(pkg):
    """The plan cache keys generic gates by their contents: same op list and
    qubits with a different matrix must not replay the first plan."""
    n = 12
    rng = np.random.default_rng(3)
    A, B = qcgen.random_unitary(8, rng), qcgen.random_unitary(8, rng)
    with pkg.State(n, "c128") as s:
        for U in (A, A, B, B, A):
            ops = [Op("H", (q,)) for q in range(n)] + [Op("MCU", (1, 5, 9, 3), matrix=U, nctrl=1)]
            s.init_random(1)
            s.run(ops)
            got = s.read()
            assert err(got, ref(n, "c128", ops, seed=1)) < 1e-12


def test_mcu_validation(pkg):
    with pkg.State(5, "c128") as s:
        bad = [Op("MCU", (0, 1), matrix=np.eye(4), nctrl=0)]
        arr = pkg.encode_ops(bad)
        arr.mtab[0]["qubits"][1] = 0  # repeated qubit
        with pytest.raises(pkg.QCError):
            s.run(arr)
        arr = pkg.encode_ops(bad)
        arr.mtab[0]["qubits"][1] = 7  # out of range
        with pytest.raises(pkg.QCError):
            s.run(arr)
        arr = pkg.encode_ops(bad)
        arr.mtab[0]["n_targ"] = 5
        with pytest.raises(pkg.QCError):
            s.run(arr)
        a2 = pkg.encode_ops([Op("H", (0,))])
        a2[0]["op"] = 16  # QC_MGATE without a table
        with pytest.raises(pkg.QCError):
            s.run(a2)
