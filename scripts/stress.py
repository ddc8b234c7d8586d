"""Stress: repeated fused runs (JIT + graphs) at large n, checked by invariants."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import qcgen, paper_2303_00123_b200 as qc
cfgs = [c.split(":") for c in sys.argv[1:]] or [["qft30", "30", "c128", "6", "1"]]
for name, n, prec, rb, tma in cfgs:
    n, rb, tma = int(n), int(rb), int(tma)
    ops = qcgen.qft(n) if name.startswith("qft") else qcgen.tfxy(n, 4)
    s = qc.State(n, prec); s.set_option("row_bits", rb); s.set_option("tma_mode", tma)
    s.init_random(3)
    n0 = s.norm2()
    arr = qc.encode_ops(ops); inv = qc.encode_ops(qcgen.inverse(ops))
    t = time.time()
    for r in range(12):
        s.run(arr); s.run(inv)
    s.sync()
    s.canonicalize()
    got = s.read(0, 4096)
    ref = qcgen.random_state(n, seed=3, precision=prec)[:4096]
    err = float(np.abs(got.astype(np.complex128) - ref).max())
    print(name, "rb", rb, "tma", tma, "runs", 24, "jit", s.info()["last_jit"], "graph", s.info()["last_graph"],
          "roundtrip err", err, "norm drift", abs(s.norm2() - n0), "s", round(time.time() - t, 1), flush=True)
    s.close()
