"""Sharded state on one GPU through the loopback backend: the
same schedule, per-rank fused segments (rank bits as predicates) and exchange
runs as the NCCL path, all shards in one buffer.  Compared with the oracle."""
import numpy as np
import pytest

import oracle
import qcgen
from qcgen import Op

pytestmark = pytest.mark.gpu
TOL = {"c128": 1e-12, "c64": 1e-5}


@pytest.fixture(scope="module")
def qcmod():
    import torch
    assert torch.cuda.is_available()
    import paper_2303_00123_b200 as pkg
    pkg.lib()
    return pkg


def run_lb(pkg, n, prec, world, ops, reps=1, **opts):
    with pkg.State.loopback(n, prec, world) as s:
        for k, v in opts.items():
            s.set_option(k, v)
        s.init_random(qcgen.STATE_SEED)
        for _ in range(reps):
            s.run(ops)
        info = s.info()
        out = s.read()
    return out, info


def ref(n, prec, ops, reps=1):
    st = qcgen.random_state(n, precision=prec)
    for _ in range(reps):
        st = oracle.run(n, st, ops)
    return st


def maxerr(a, b):
    return float(np.abs(a.astype(np.complex128) - b).max())


def test_loopback_init_matches_generator(qcmod):
    with qcmod.State.loopback(14, "c128", 4) as s:
        s.init_random(qcgen.STATE_SEED)
        assert np.array_equal(s.read(), qcgen.random_state(14))
        assert s.info()["world"] == 4 and s.info()["n_local"] == 12 and s.info()["sharding"] == 1


@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("world,n", [(2, 12), (4, 13), (8, 15)])
def test_loopback_random_circuits(qcmod, prec, world, n):
    ops = qcgen.random_circuit(n, 150, seed=40 + n + world)
    got, info = run_lb(qcmod, n, prec, world, ops)
    assert info["last_exchanges"] > 0
    assert maxerr(got, ref(n, prec, ops)) <= TOL[prec]


@pytest.mark.parametrize("world,n", [(2, 14), (4, 16), (8, 18)])
def test_loopback_qft_and_tfxy(qcmod, world, n):
    for ops in (qcgen.qft(n), qcgen.tfxy(n, 3)):
        got, info = run_lb(qcmod, n, "c128", world, ops)
        assert maxerr(got, ref(n, "c128", ops)) <= 1e-12


def test_loopback_repeated_runs_jit(qcmod):
    n, world = 16, 4
    ops = qcgen.qft(n)
    got, info = run_lb(qcmod, n, "c128", world, ops, reps=4)
    assert info["last_jit"]
    assert maxerr(got, ref(n, "c128", ops, reps=4)) <= 1e-12


def test_loopback_permutation_bit_exact(qcmod):
    n, world = 14, 4
    ops = qcgen.random_circuit(n, 200, seed=9, kinds=("X", "CNOT", "SWAP", "CCX"))
    for relabel in (0, 1):
        got, _ = run_lb(qcmod, n, "c128", world, ops, relabel_swap=relabel)
        assert np.array_equal(got, ref(n, "c128", ops))


def test_loopback_canonicalize_and_norm(qcmod):
    n, world = 15, 8
    ops = qcgen.qft(n) + qcgen.random_circuit(n, 50, seed=2)
    with qcmod.State.loopback(n, "c128", world) as s:
        s.init_random(5)
        s.run(ops)
        full = s.read()
        s.canonicalize()
        assert s.info()["layout_is_canonical"]
        assert np.array_equal(s.read(), full)
        assert abs(s.norm2() - np.vdot(full, full).real) < 1e-12
    assert maxerr(full, oracle.run(n, qcgen.random_state(n, seed=5), ops)) <= 1e-12


def test_loopback_global_controls_and_diagonals(qcmod):
    """Controls / diagonal gates on rank bits only (no exchange needed)."""
    n, world = 12, 4  # qubits 0, 1 are rank bits
    ops = [Op("CNOT", (0, 5)), Op("CP", (1, 7), theta=0.4), Op("RZ", (0,), theta=1.1),
           Op("CU1", (1, 3), matrix=qcgen.random_unitary(2, np.random.default_rng(1)), ctrl_state=0),
           Op("CCX", (0, 1, 9)), Op("Z", (1,)), Op("P", (0,), theta=-0.7)]
    got, info = run_lb(qcmod, n, "c128", world, ops)
    assert info["last_exchanges"] == 0
    assert maxerr(got, ref(n, "c128", ops)) <= 1e-12


# ---- collective-fused pair passes (QC_OPT_EXCHANGE 2): gates on one rank-bit
# qubit run in place over the pair's two shards (tile halves from both), no
# exchange.  Loopback: the two halves come from two shards of one buffer
# through the same PassDesc fields (tile0 / addr_strip / addr_bits1 / state1 /
# second tensor map) the NCCL path fills with the IPC-mapped partner buffer.
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("world,n", [(2, 13), (4, 14), (8, 16)])
def test_pair_passes_random_circuits(qcmod, prec, world, n):
    ops = qcgen.random_circuit(n, 150, seed=70 + n + world)
    got, info = run_lb(qcmod, n, prec, world, ops, exchange=2)
    assert info["last_pair_segments"] > 0
    assert maxerr(got, ref(n, prec, ops)) <= TOL[prec]


@pytest.mark.parametrize("world,n", [(2, 14), (4, 16), (8, 18)])
def test_pair_passes_qft_tfxy(qcmod, world, n):
    for ops in (qcgen.qft(n), qcgen.tfxy(n, 3)):
        got, info = run_lb(qcmod, n, "c128", world, ops, exchange=2)
        assert info["last_pair_segments"] > 0 and info["last_exchanges"] == 0
        assert maxerr(got, ref(n, "c128", ops)) <= 1e-12


@pytest.mark.parametrize("opts", [dict(), dict(tma_mode=2), dict(tma_mode=1), dict(row_bits=6),
                                  dict(remap=0), dict(jit=0)])
def test_pair_passes_transports(qcmod, opts):
    """Every tile transport (box halves, gather4 rows, per-row copies) and the
    AOT / JIT kernels on pair passes; the layout is unchanged afterwards."""
    n, world = 15, 4
    ops = qcgen.qft(n) + qcgen.random_circuit(n, 80, seed=12)
    got, info = run_lb(qcmod, n, "c128", world, ops, reps=2, exchange=2, **opts)
    assert info["last_pair_segments"] > 0
    assert maxerr(got, ref(n, "c128", ops, reps=2)) <= 1e-12


def test_pair_passes_permutation_bit_exact(qcmod):
    n, world = 14, 4
    ops = qcgen.random_circuit(n, 200, seed=19, kinds=("X", "CNOT", "SWAP", "CCX"))
    got, info = run_lb(qcmod, n, "c128", world, ops, exchange=2)
    assert info["last_pair_segments"] > 0
    assert np.array_equal(got, ref(n, "c128", ops))


# ---- group plans (QC_OPT_EXCHANGE 3): the whole circuit planned once over
# all n bits; a pass whose tile holds j rank bits moves its 2^j sub-tiles
# from / to 2^j shards (every shard its own buffer + tensor maps, as the
# IPC-mapped peers of the NCCL path); no exchanges, no layout drift.
@pytest.mark.parametrize("prec", ["c128", "c64"])
@pytest.mark.parametrize("world,n", [(2, 13), (4, 14), (8, 16)])
def test_group_plan_random_circuits(qcmod, prec, world, n):
    ops = qcgen.random_circuit(n, 150, seed=90 + n + world)
    got, info = run_lb(qcmod, n, prec, world, ops, exchange=3)
    assert info["last_exchanges"] == 0 and info["last_pair_segments"] > 0  # passes spanning shards
    assert maxerr(got, ref(n, prec, ops)) <= TOL[prec]


@pytest.mark.parametrize("world,n", [(2, 14), (4, 16), (8, 18)])
def test_group_plan_qft_tfxy(qcmod, world, n):
    for ops in (qcgen.qft(n), qcgen.tfxy(n, 3)):
        # 3 runs: QFT's relabels alternate two layouts (two plans), the 3rd
        # run is a plan's 2nd use -- NVRTC-specialised
        got, info = run_lb(qcmod, n, "c128", world, ops, reps=3, exchange=3)
        assert info["last_exchanges"] == 0 and info["last_jit"]
        assert maxerr(got, ref(n, "c128", ops, reps=3)) <= 1e-12


@pytest.mark.parametrize("opts", [dict(), dict(tma_mode=2), dict(tma_mode=1), dict(remap=0), dict(jit=0),
                                  dict(relabel_swap=0)])
def test_group_plan_transports(qcmod, opts):
    n, world = 15, 8
    ops = qcgen.qft(n) + qcgen.random_circuit(n, 80, seed=13) + qcgen.random_mcu_circuit(n, 10, seed=3)
    got, info = run_lb(qcmod, n, "c128", world, ops, reps=2, exchange=3, **opts)
    assert info["last_pair_segments"] > 0
    assert maxerr(got, ref(n, "c128", ops, reps=2)) <= 1e-12


def test_group_plan_permutation_bit_exact(qcmod):
    n, world = 14, 4
    ops = qcgen.random_circuit(n, 200, seed=29, kinds=("X", "CNOT", "SWAP", "CCX"))
    got, info = run_lb(qcmod, n, "c128", world, ops, exchange=3)
    assert np.array_equal(got, ref(n, "c128", ops))


@pytest.mark.parametrize("xmode", [0, 2, 3])
@pytest.mark.parametrize("world,n", [(2, 9), (2, 10), (4, 10), (4, 11), (8, 11), (8, 12)])
def test_smallest_sharded_states(qcmod, xmode, world, n):
    """The smallest shards allowed (8-10 local qubits: tiles smaller than the
    default, few tiles per pass, the group-plan tile split at its minimum)."""
    ops = qcgen.random_circuit(n, 60, seed=3 * n + world) + qcgen.qft(n)
    got, info = run_lb(qcmod, n, "c128", world, ops, reps=2, exchange=xmode)
    assert maxerr(got, ref(n, "c128", ops, reps=2)) <= 1e-12


def test_shards_below_8_local_qubits_rejected(qcmod):
    from paper_2303_00123_b200 import QCError
    with pytest.raises(QCError) as e:
        qcmod.State.loopback(9, "c128", 4)
    assert e.value.status == 1 and "8 local qubits" in str(e.value)
