"""NCCL-sharded states across >= 2 GPUs, one process per GPU:
every rank's canonical shard after QFT / TFXY / random (incl. generic) circuits
vs the CPU oracle, for every exchange backend (QC_OPT_EXCHANGE 0: NCCL
send/recv with ping-pong staging, 1: P2P swap kernel over CUDA IPC, 2: pair
passes reading / writing the partner's shard over the IPC mapping, 3: one
group plan whose tiles may span every shard), and
qc_state_init_basis on a shard.  Skipped on boxes with one GPU (the loopback
backend in test_gpu_dist.py covers the same schedule on one GPU)."""
import numpy as np
import pytest

import oracle
import qcgen

pytestmark = pytest.mark.gpu


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


need2 = pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs (NCCL across processes)")


def _circuit(kind, n):
    if kind == "qft":
        return qcgen.qft(n)
    if kind == "tfxy":
        return qcgen.tfxy(n, 4)
    return qcgen.random_mcu_circuit(n, 120, seed=n, max_ctrl=3, p_mcu=0.3)


def _worker(rank, world, uid, n, prec, kind, xmode, q):
    import torch
    torch.cuda.set_device(rank)
    import paper_2303_00123_b200 as pkg
    try:
        ops = _circuit(kind, n)
        nl = n - (world.bit_length() - 1)
        with pkg.State.dist(n, prec, rank, world, uid) as s:
            s.set_option("exchange", xmode)
            s.init_random(qcgen.STATE_SEED)
            s.run(ops)
            s.run(ops)  # second run: JIT kernels, cached sharded plan
            ex = s.info()["last_exchanges"] + s.info()["last_pair_segments"]
            s.canonicalize()
            got = s.read(rank << nl, 1 << nl)
            # init_basis on a shard: one unit amplitude, on the owning rank only
            k = (1 << nl) + 5 if world > 1 else 5
            s.init_basis(k)
            basis = s.read(rank << nl, 1 << nl)
        q.put((rank, got, ex, basis, None))
    except Exception as e:  # report, do not hang the parent
        q.put((rank, None, 0, None, repr(e)))


def _run(world, n, prec, kind, xmode):
    import torch.multiprocessing as mp
    from paper_2303_00123_b200 import qc
    uid = qc.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, uid, n, prec, kind, xmode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
    return res


@need2
@pytest.mark.parametrize("xmode", [0, 1, 2, 3])
@pytest.mark.parametrize("kind,prec", [("qft", "c128"), ("tfxy", "c128"), ("random", "c128"), ("qft", "c64")])
def test_nccl_shards_match_oracle(kind, prec, xmode):
    world = 2
    n = 18
    ops = _circuit(kind, n)
    st = qcgen.random_state(n, precision=prec)
    exp = oracle.run(n, oracle.run(n, st, ops), ops)
    nl = n - 1
    tol = 1e-12 if prec == "c128" else 1e-5
    for rank, got, ex, basis, err in _run(world, n, prec, kind, xmode):
        assert err is None, err
        assert ex > 0
        assert np.abs(got.astype(np.complex128) - exp[rank << nl:(rank + 1) << nl]).max() < tol * 10
        k = (1 << nl) + 5
        want = np.zeros(1 << nl)
        if rank == k >> nl:
            want[k & ((1 << nl) - 1)] = 1.0
        assert np.array_equal(basis.real, want) and not basis.imag.any()
