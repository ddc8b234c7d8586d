"""Raw fused-pipeline bandwidth: one cheap op per pass, n=30 (HBM regime)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import qcgen
import paper_2303_00123_b200 as qc

def timeit(s, arr, reps=5):
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

res = {}
for prec in ("c128", "c64"):
    n = 30 if prec == "c128" else 31
    sb = (16 if prec == "c128" else 8) << n
    s = qc.State(n, prec)
    s.init_random(1)
    arr = qc.encode_ops([qcgen.Op("RX", (15,), theta=0.3)])
    for tile in (12, 13):
        for rb in (4, 5, 6, 7):
            for jit in (2,):
                for ctas in (0, 1):
                    if prec == "c128" and tile == 13: continue
                    s.set_option("tile_bits", tile); s.set_option("jit", jit); s.set_option("tma_mode", ctas)
                    s.set_option("row_bits", rb)
                    try:
                        t = timeit(s, arr)
                    except Exception as e:
                        res[f"{prec}_k{tile}_rb{rb}_tma{ctas}"] = str(e)[:80]; continue
                    res[f"{prec}_k{tile}_rb{rb}_tma{ctas}"] = round(2 * sb / (t / 1e3) / 1e9, 1)
    s.close(); torch.cuda.empty_cache()
print(json.dumps(res, indent=0))
