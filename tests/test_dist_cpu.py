"""Host-side logic of the sharded layer with real 2-process
communication over torch.distributed gloo (no GPU):
  * the qubit-swap exchange runs from libqc (qc_debug_exchange_runs), executed
    with gloo send/recv between two ranks, equal a swap of the two physical
    bits of the global vector;
  * the sharded schedule (qc_debug_dist_schedule) is identical on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import qcgen
from paper_2303_00123_b200 import qc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def swap_bits(vec, n, a, b):
    """Physical bit swap of a global vector (numpy reference)."""
    idx = np.arange(1 << n, dtype=np.int64)
    ba, bb = (idx >> a) & 1, (idx >> b) & 1
    src = idx ^ ((ba ^ bb) << a) ^ ((ba ^ bb) << b)
    return vec[src]


def _worker(rank, world, port, n, cases, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_loc = n - (world.bit_length() - 1)
        rng = np.random.default_rng(7)
        glob = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)).astype(np.complex128)
        ok = True
        for g, l in cases:
            shard = torch.from_numpy(glob[rank << n_loc:(rank + 1) << n_loc].copy())
            partner, runs = qc.debug_exchange_runs(n_loc, rank, g, l)
            for off, cnt in runs:
                send = shard[off:off + cnt].clone()
                recv = torch.empty_like(send)
                # deadlock-free pairwise exchange: lower rank sends first
                if rank < partner:
                    dist.send(torch.view_as_real(send).contiguous(), partner)
                    dist.recv(torch.view_as_real(recv), partner)
                else:
                    dist.recv(torch.view_as_real(recv), partner)
                    dist.send(torch.view_as_real(send).contiguous(), partner)
                shard[off:off + cnt] = recv
            ref = swap_bits(glob, n, g, l)[rank << n_loc:(rank + 1) << n_loc]
            ok = ok and np.array_equal(shard.numpy(), ref)
        # schedule determinism
        ops = qcgen.qft(n) + qcgen.tfxy(n, 2) + qcgen.random_circuit(n, 60, seed=3)
        steps, lay = qc.debug_dist_schedule(n, world, ops)
        t = torch.tensor([x for s in steps for x in s] + lay, dtype=torch.int64)
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([t.numel()]))
        gathered = [torch.zeros(int(sizes[0].item()), dtype=torch.int64) for _ in range(world)]
        same_size = all(int(x.item()) == t.numel() for x in sizes)
        if same_size:
            dist.all_gather(gathered, t)
            same = all(torch.equal(x, t) for x in gathered)
        else:
            same = False
        q.put((rank, ok, same, len(steps)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 9), (4, 11)])
def test_exchange_runs_and_schedule_over_gloo(world, n):
    port = _free_port()
    n_loc = n - (world.bit_length() - 1)
    cases = [(g, l) for g in range(n_loc, n) for l in (n_loc - 1, n_loc - 2, 3, 0)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, same, nsteps in res:
        assert ok, f"rank {rank}: exchange runs do not implement the bit swap"
        assert same, f"rank {rank}: schedule differs across ranks"
        assert nsteps > 1


def test_schedule_makes_every_target_local():
    """Replay the schedule's layout bookkeeping: at least p exchanges for the
    QFT (each global qubit needs its Hadamard) and the final layout is a
    permutation."""
    for world, n in ((2, 12), (4, 14), (8, 16)):
        p = world.bit_length() - 1
        steps, lay = qc.debug_dist_schedule(n, world, qcgen.qft(n))
        ex = [s for s in steps if s[0] == 1]
        assert len(ex) >= p
        assert sorted(lay) == list(range(n))
        for kind, g, l, _ in ex:
            assert g >= n - p and l == n - p - 1
        gates = sum(s[3] for s in steps if s[0] == 0)
        assert gates >= len(qcgen.qft(n)) - n // 2  # SWAPs are relabels


@pytest.mark.parametrize("n,world", [(33, 2), (34, 4), (36, 8), (36, 16), (40, 8)])
def test_schedule_64bit_qubit_masks(n, world):
    """Qubits >= 32 must not alias qubit q-32 (64-bit masks): gates whose
    non-diagonal targets are local need no exchange at any n; a single
    non-diagonal gate on a global qubit needs exactly one, on its rank bit."""
    p = world.bit_length() - 1
    local_ops = [qcgen.Op("H", (q,)) for q in range(p, n)] + \
                [qcgen.Op("CNOT", (q, q + 1)) for q in range(p, n - 1)] + \
                [qcgen.Op("RZ", (q,), theta=0.3) for q in range(n)]  # diagonal: never exchanged
    steps, lay = qc.debug_dist_schedule(n, world, local_ops)
    assert [s for s in steps if s[0] == 1] == []
    assert lay == [n - 1 - q for q in range(n)]
    for gq in range(p):
        steps, _ = qc.debug_dist_schedule(n, world, [qcgen.Op("H", (33 if n > 33 else n - 1,)),
                                                     qcgen.Op("H", (gq,))])
        ex = [s for s in steps if s[0] == 1 and s[3] == 0]
        assert len(ex) == 1 and ex[0][1] == n - 1 - gq and ex[0][2] == n - p - 1
        back = [s for s in steps if s[0] == 1 and s[3] == 1]  # the restore: the same exchange again
        assert back == [(1, n - 1 - gq, n - p - 1, 1)]


def test_schedule_exchange_counts_at_full_size():
    """Exchange counts of the north-star sharded workloads (C5, and TFXY at the
    sizes of the scaling grid) after the 64-bit-mask fix; the round-1 32-bit
    masks scheduled 6 / 62 / 42 (VERDICT r01 recomputation: 4 / 51 / 31)."""
    def count(n, world, ops):
        steps, lay = qc.debug_dist_schedule(n, world, ops)
        assert sorted(lay) == list(range(n))
        # restore exchanges at the end (the layout returns to the relabels-only
        # one, so a repeated circuit reuses its plan): at most 2 per rank bit
        p = world.bit_length() - 1
        assert sum(1 for s in steps if s[0] == 1 and s[3] == 1) <= 2 * p
        return sum(1 for s in steps if s[0] == 1 and s[3] == 0)
    assert count(36, 8, qcgen.qft(36)) == 4
    assert count(33, 8, qcgen.tfxy(33, 10)) == 51
    assert count(35, 4, qcgen.tfxy(35, 10)) == 31


def test_pair_segment_schedule():
    """QC_OPT_EXCHANGE 2: a run of gates whose only non-diagonal rank-bit
    qubit is g becomes one pair segment on g (no exchange, layout unchanged);
    a gate needing two rank bits at once falls back to exchanges."""
    def steps_of(n, world, ops):
        steps, lay = qc.debug_dist_schedule(n, world, ops, exchange=2)
        return steps, lay

    def relabelled(n, ops):  # canonical layout after the SWAP relabels only
        lay = [n - 1 - q for q in range(n)]
        for op in ops:
            if op.name == "SWAP":
                a, b = op.qubits
                lay[a], lay[b] = lay[b], lay[a]
        return lay
    n, world = 36, 8
    steps, lay = steps_of(n, world, qcgen.qft(n))
    assert [(k, g) for k, g, _, _ in steps] == [(2, 35), (2, 34), (2, 33)]
    assert lay == relabelled(n, qcgen.qft(n))
    assert sum(s[3] for s in steps) == sum(1 for op in qcgen.qft(n) if op.name != "SWAP")
    for n, world in ((33, 8), (35, 4), (16, 4)):
        ops = qcgen.tfxy(n, 4)
        steps, lay = steps_of(n, world, ops)
        assert all(k in (0, 2) for k, _, _, _ in steps) and any(k == 2 for k, _, _, _ in steps)
        assert lay == [n - 1 - q for q in range(n)]
        assert sum(s[3] for s in steps) == len(ops)
        p = world.bit_length() - 1
        assert all(n - p <= g < n for k, g, _, _ in steps if k == 2)
    # a dense 2-qubit gate on two rank-bit qubits: exchanges bring both local
    u = qcgen.random_unitary(4, np.random.default_rng(0))
    steps, lay = steps_of(14, 4, [qcgen.Op("U2", (0, 1), matrix=u)])
    assert [s[0] for s in steps if s[3] == 0].count(1) == 2 and sorted(lay) == list(range(14))
    assert lay == [13 - q for q in range(14)]  # restored
    # gates on local qubits only: one local segment
    steps, _ = steps_of(14, 4, [qcgen.Op("H", (q,)) for q in range(2, 14)])
    assert [s[0] for s in steps] == [0]


@pytest.mark.parametrize("n,world", [(16, 4), (18, 8), (36, 8)])
def test_schedule_restores_relabel_layout(n, world):
    """Exchange modes 0/1 end every sharded run in the layout the SWAP
    relabels alone give (so the plan of a repeated circuit is reused)."""
    for ops in (qcgen.qft(n), qcgen.tfxy(n, 3), qcgen.random_circuit(n, 80, seed=n)):
        lay = [n - 1 - q for q in range(n)]
        for op in ops:
            if op.name == "SWAP":
                a, b = op.qubits
                lay[a], lay[b] = lay[b], lay[a]
        steps, got = qc.debug_dist_schedule(n, world, ops)
        assert got == lay


def test_group_plan_schedule():
    """QC_OPT_EXCHANGE 3: the whole circuit is one step (a plan over all n
    bits), no exchanges; the layout changes by the SWAP relabels only."""
    for n, world, ops in ((36, 8, qcgen.qft(36)), (34, 2, qcgen.tfxy(34, 10)),
                          (16, 4, qcgen.random_circuit(16, 60, seed=5))):
        steps, lay = qc.debug_dist_schedule(n, world, ops, exchange=3)
        assert [s[0] for s in steps] == [3]
        assert steps[0][3] == sum(1 for op in ops if op.name != "SWAP")
        want = [n - 1 - q for q in range(n)]
        for op in ops:
            if op.name == "SWAP":
                a, b = op.qubits
                want[a], want[b] = want[b], want[a]
        assert lay == want


def _group_worker(rank, world, port, cases, q):
    """Emulate group-plan passes over gloo: every rank processes its tile
    range of each pass (qc_debug_group_split), fetching each tile's sub-tiles
    from their owner ranks and writing the result back to them; the pass
    applied here is the permutation x -> x XOR T of the global index (it
    touches every amplitude of every tile exactly once)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = True
        for n, T in cases:
            p = world.bit_length() - 1
            nl = n - p
            rng = np.random.default_rng(n * 131 + T % 9973)
            glob = (rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n))
            shard = torch.from_numpy(glob[rank << nl:(rank + 1) << nl].copy())
            # all shards visible (stands in for the IPC-mapped peer buffers)
            shards = [torch.zeros_like(shard) for _ in range(world)]
            dist.all_gather(shards, shard)
            t0, cnt, j, owners = qc.debug_group_split(n, world, T, rank)
            tpos = [b for b in range(n) if (T >> b) & 1]
            opos = [b for b in range(n) if not (T >> b) & 1]
            rank_t = [b for b in tpos if b >= nl]
            writes = []  # (owner, local index, value)
            for t in range(t0, t0 + cnt):
                base = sum(((t >> i) & 1) << b for i, b in enumerate(opos))
                for x in range(1 << len(tpos)):
                    g = base | sum(((x >> i) & 1) << b for i, b in enumerate(tpos))
                    h = sum(((g >> b) & 1) << i for i, b in enumerate(rank_t))
                    own = owners[h]
                    if own != (g >> nl):  # the owner of sub-tile h holds the amplitude
                        ok = False
                    src = g ^ T  # the pass: out[g] = in[g ^ T] (same tile: T bits flipped)
                    writes.append((own, g & ((1 << nl) - 1), shards[src >> nl][src & ((1 << nl) - 1)].item()))
            gathered = [None] * world
            dist.all_gather_object(gathered, writes)
            mine = np.full(1 << nl, np.nan + 0j)
            seen = np.zeros(1 << nl, dtype=np.int64)
            for w in gathered:
                for own, li, v in w:
                    if own == rank:
                        mine[li] = v
                        seen[li] += 1
            idx = np.arange(rank << nl, (rank + 1) << nl)
            ok = ok and bool(np.all(seen == 1)) and bool(np.allclose(mine, glob[idx ^ T]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_group_plan_tile_split_over_gloo(world):
    """Host logic of group plans (QC_OPT_EXCHANGE 3) with real multi-process
    communication: each rank's tile range and sub-tile owners, for passes
    whose tile holds 0, 1 or all rank bits, cover every amplitude exactly once
    and move it between the right shards."""
    n = 10
    p = world.bit_length() - 1
    nl = n - p
    low = (1 << 3) - 1  # row bits 0..2
    cases = [(n, low | (1 << 5)),                         # no rank bit: local tiles
             (n, low | (1 << (n - 1))),                   # the top rank bit
             (n, low | (1 << 6) | (((1 << p) - 1) << nl))]  # every rank bit
    if p > 1:
        cases.append((n, low | (1 << nl)))                # the lowest rank bit only
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_group_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, ok in res:
        assert ok, f"rank {rank}: group-plan tile split / owners wrong"
