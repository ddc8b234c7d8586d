"""Oracle parity of a few circuits under given state options (experiments).

  python scripts/parity_opts.py tma_mode=2,row_bits=4 [...]
Runs QFT / TFXY / random circuits 3x (AOT, JIT, graph) per option set at
n = 14..24, c128 and c64, and prints max |err| vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import qcgen
import paper_2303_00123_b200 as qc

ok = True
for oset in sys.argv[1:] or [""]:
    opts = dict(kv.split("=") for kv in oset.split(",") if kv)
    for n, name, ops in ((14, "qft", qcgen.qft(14)), (18, "tfxy", qcgen.tfxy(18, 6)),
                         (16, "random", qcgen.random_circuit(16, 200, seed=5)),
                         (22, "tfxy", qcgen.tfxy(22, 4)), (24, "qft", qcgen.qft(24)),
                         (20, "mcu", qcgen.random_mcu_circuit(20, 80, seed=3))):
        for prec, tol in (("c128", 1e-12), ("c64", 1e-5)):
            ref = oracle.run(n, qcgen.random_state(n, precision=prec), ops)
            with qc.State(n, prec) as s:
                for k, v in opts.items():
                    s.set_option(k, int(v))
                errs = []
                for _ in range(3):
                    s.init_random(qcgen.STATE_SEED)
                    s.run(ops)
                    errs.append(float(np.abs(s.read().astype(np.complex128) - ref).max()))
            good = max(errs) <= tol * 10
            ok = ok and good
            print(f"{oset or 'default'} {name}{n} {prec}: max|err| {max(errs):.2e} {'ok' if good else 'FAIL'}", flush=True)
print("ALL OK" if ok else "FAILURES")
