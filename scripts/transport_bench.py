"""Tile-transport ceiling of the fused pass: one cheap gate per pass (a single
Hadamard: the pass is pure HBM <-> smem traffic), n = 30 (c128) / 31 (c64),
for the TMA box transport (default) and gather4 rows, at row bits 3..7.
Reports GB/s of 2 * state bytes per pass and the fraction of MEASURED_PEAKS
hbm_gbs, i.e. the best any HBM-bound pass (QFT) can do with that row width.

  python scripts/transport_bench.py > profiles/round2_transport_ceiling.json
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import qcgen
import paper_2303_00123_b200 as qc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def timeit(s, arr, reps=6):
    st = torch.cuda.ExternalStream(s.stream)
    with torch.cuda.stream(st):
        for _ in range(3):
            s.run(arr)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            s.run(arr)
        b.record(st)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


res = {"peak_hbm_gbs": peak}
for prec in ("c128", "c64"):
    n = 30 if prec == "c128" else 31
    sb = (16 if prec == "c128" else 8) << n
    arr = qc.encode_ops([qcgen.Op("H", (n // 2,))])
    for tma, name in ((0, "box"), (2, "gather4")):
        for rb in (3, 4, 5, 6, 7):
            if prec == "c128" and rb == 7 and tma == 2:
                continue  # > 1 KiB gather4 rows are capped (row path)
            s = qc.State(n, prec)
            s.init_random(1)
            s.set_option("tma_mode", tma)
            s.set_option("row_bits", rb)
            s.set_option("jit", 2)
            t = timeit(s, arr)
            inf = s.info()
            gbs = 2 * sb * inf["last_passes"] / (t / 1e3) / 1e9
            key = f"{prec}_{name}_rb{rb}_row{(16 if prec == 'c128' else 8) << rb}B"
            res[key] = {"GBps": round(gbs, 1), "frac_of_hbm": round(gbs / peak, 3), "passes": inf["last_passes"]}
            print(key, res[key], file=sys.stderr, flush=True)
            s.close()
            torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
