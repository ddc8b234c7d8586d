"""Probe: do group plans (QC_OPT_EXCHANGE 3, TMA over IPC-mapped peer shards)
work on this multi-GPU node?  Launched by bench.py under torch.distributed.run
(one process per GPU) BEFORE the benchmark allocates its shards, in a process
of its own: a fault here (e.g. TMA refusing peer memory) cannot take the
benchmark down with it.

Every rank runs QFT, TFXY and a random circuit on a small sharded state with
exchange mode 3 and with mode 0 (NCCL qubit-swap exchanges, the reference
path), and compares its canonical shard of the two results.  Exit code 0 and
"PROBE OK" on rank 0 iff every rank matched to 1e-12.

  python -m torch.distributed.run --nproc-per-node N scripts/probe_sharded.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

import qcgen
import paper_2303_00123_b200 as qc


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = world.bit_length() - 1
    n = 15 + p
    nl = n - p
    uid = [qc.qc.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ok = True
    for ops in (qcgen.qft(n), qcgen.tfxy(n, 2), qcgen.random_circuit(n, 60, seed=11)):
        outs = []
        for xmode in (0, 3):
            with qc.State.dist(n, "c128", rank, world, uid[0]) as s:
                s.set_option("exchange", xmode)
                s.init_random(qcgen.STATE_SEED)
                s.run(ops)
                s.run(ops)
                s.canonicalize()
                outs.append(s.read(rank << nl, 1 << nl))
        ok = ok and bool(np.abs(outs[0] - outs[1]).max() <= 1e-12)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("PROBE OK" if int(flag.item()) == 1 else "PROBE MISMATCH", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) == 1 else 1)


if __name__ == "__main__":
    main()
