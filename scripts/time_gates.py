"""Per-gate (unfused) kernel bandwidth at n=30, as in bench.py's sweep."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import qcgen
import paper_2303_00123_b200 as qc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import _time_runs, load_peaks

peak, _ = load_peaks()
for prec in ("c128", "c64"):
    n = 30
    sb = (16 if prec == "c128" else 8) << n
    s = qc.State(n, prec)
    s.init_random(1)
    s.set_option("fusion", 0)
    s.set_option("relabel_swap", 0)
    out = {}
    for name, qs, arg, nbytes in (("H", (0,), None, 2 * sb), ("H", (15,), None, 2 * sb), ("H", (29,), None, 2 * sb),
                                  ("RZ", (12,), 0.3, 2 * sb), ("P", (12,), 0.3, sb), ("X", (3,), None, 2 * sb),
                                  ("CNOT", (4, 20), None, sb), ("CP", (2, 27), 0.2, sb // 2),
                                  ("SWAP", (1, 28), None, sb), ("U2", (7, 22), "U", 2 * sb)):
        g = qcgen.Op(name, qs, theta=arg if isinstance(arg, float) else None,
                     matrix=qcgen.random_unitary(4, np.random.default_rng(0)) if arg == "U" else None)
        t = _time_runs(s, qc.encode_ops([g]), warm=1, reps=5)
        out[f"{name}{list(qs)}"] = round(nbytes / (t / 1e3) / 1e9 / peak, 3)
    print(prec, json.dumps(out), flush=True)
    s.close()
    torch.cuda.empty_cache()
