"""Loopback sharded circuit time, exchange modes side by side (one GPU):
QC_OPT_EXCHANGE 0 (qubit-swap exchanges as in-place swap kernels), 2 (pair
passes: tile halves from two shards) and 3 (group plan: one plan over all n
bits, tiles spanning up to all shards).  On one GPU every shard is local HBM,
so this checks the multi-buffer tile transport costs no more than a local
pass, and counts passes; NVLink rates need >= 2 GPUs.

  python scripts/time_pair.py qft:30:2 tfxy:28:2 ...   (family:n:world)
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import qcgen
import paper_2303_00123_b200 as qc

for w in sys.argv[1:]:
    fam, n, world = w.split(":")
    n, world = int(n), int(world)
    ops = qcgen.qft(n) if fam == "qft" else qcgen.tfxy(n, 10)
    arr = qc.encode_ops(ops)
    for xm in (0, 2, 3):
        with qc.State.loopback(n, "c128", world) as s:
            s.set_option("exchange", xm)
            s.init_random(1)
            st = torch.cuda.ExternalStream(s.stream)
            with torch.cuda.stream(st):
                for _ in range(6):  # 2 layouts (SWAP relabels) x (plan, JIT, warm)
                    s.run(arr)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                h0 = time.perf_counter()
                for _ in range(4):
                    s.run(arr)
                h1 = time.perf_counter()
                b.record(st)
                torch.cuda.synchronize()
            i = s.info()
            print(f"{w} exchange={xm}: {a.elapsed_time(b) / 4:.2f} ms, passes {i['last_passes']}, "
                  f"exchanges {i['last_exchanges']}, pair segments {i['last_pair_segments']}, "
                  f"host enqueue {(h1 - h0) / 4 * 1e3:.2f} ms/run, jit {i['last_jit']}", flush=True)
