"""Circuit time vs tile configuration (JIT passes, graph replay)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import qcgen
import paper_2303_00123_b200 as qc

def timeit(s, arr, reps=5, warm=4):
    st = torch.cuda.ExternalStream(s.stream)
    with torch.cuda.stream(st):
        for _ in range(warm):
            s.run(arr)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            s.run(arr)
        b.record(st)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

cfgs = [(int(x.split(",")[0]), int(x.split(",")[1]), int(x.split(",")[2])) for x in sys.argv[2:]] or \
       [(12, 5, 0), (12, 6, 0), (12, 7, 0), (11, 6, 296), (11, 7, 296), (11, 5, 296)]
res = {}
for name, n, prec, ops in (("tfxy20", 20, "c128", qcgen.tfxy(20, 10)), ("qft30", 30, "c128", qcgen.qft(30)),
                           ("qft30c64", 30, "c64", qcgen.qft(30)), ("tfxy28", 28, "c128", qcgen.tfxy(28, 10))):
    if sys.argv[1] != "all" and name not in sys.argv[1].split("+"):
        continue
    s = qc.State(n, prec)
    s.init_random(1)
    arr = qc.encode_ops(ops)
    for k, rb, ctas in cfgs:
        s.set_option("tile_bits", k); s.set_option("row_bits", rb); s.set_option("ctas", ctas)
        t = timeit(s, arr)
        inf = s.info()
        res[f"{name}_k{k}_rb{rb}_c{ctas}"] = {"ms": round(t, 4), "passes": inf["last_passes"], "jit": inf["last_jit"],
            "GBps_per_pass": round(2 * ((16 if prec == "c128" else 8) << n) * inf["last_passes"] / (t / 1e3) / 1e9, 1)}
        print(name, k, rb, ctas, res[f"{name}_k{k}_rb{rb}_c{ctas}"], flush=True)
    s.close(); torch.cuda.empty_cache()
print(json.dumps(res))
