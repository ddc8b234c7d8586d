"""Circuit time for a list of workloads x option sets (JIT passes, graph replay).

  python scripts/time_circ.py tfxy:28 qft:30:c64 ... [--opts remap=0,jit=2 remap=1]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import qcgen
import paper_2303_00123_b200 as qc

ap = argparse.ArgumentParser()
ap.add_argument("work", nargs="+")
ap.add_argument("--opts", nargs="*", default=[""])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()


def timeit(s, arr, reps, warm=4):
    st = torch.cuda.ExternalStream(s.stream)
    with torch.cuda.stream(st):
        for _ in range(warm):
            s.run(arr)
        torch.cuda.synchronize()
        x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x.record(st)
        for _ in range(reps):
            s.run(arr)
        y.record(st)
        torch.cuda.synchronize()
    return x.elapsed_time(y) / reps


res = {}
for w in a.work:
    parts = w.split(":")
    fam, n = parts[0], int(parts[1])
    prec = parts[2] if len(parts) > 2 else "c128"
    ops = qcgen.qft(n) if fam == "qft" else qcgen.tfxy(n, 10)
    arr = qc.encode_ops(ops)
    for oset in a.opts:
        s = qc.State(n, prec)
        s.init_random(1)
        for kv in filter(None, oset.split(",")):
            k, v = kv.split("=")
            s.set_option(k, int(v))
        t = timeit(s, arr, a.reps if n >= 26 else 20)
        inf = s.info()
        sb = (16 if prec == "c128" else 8) << n
        key = f"{w}|{oset}"
        res[key] = {"ms": round(t, 4), "passes": inf["last_passes"], "jit": inf["last_jit"],
                    "GBps_per_pass": round(2 * sb * inf["last_passes"] / (t / 1e3) / 1e9, 1)}
        print(key, res[key], flush=True)
        s.close()
        torch.cuda.empty_cache()
print(json.dumps(res))
