"""Run one benchmark circuit a few times (for ncu / sanitizer passes)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import qcgen
import paper_2303_00123_b200 as qc

ap = argparse.ArgumentParser()
ap.add_argument("--circuit", default="tfxy")
ap.add_argument("--n", type=int, default=20)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--prec", default="c128")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fusion", type=int, default=1)
ap.add_argument("--jit", type=int, default=1)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--rb", type=int, default=0)
ap.add_argument("--gates", type=int, default=0)
ap.add_argument("--tma", type=int, default=0)
ap.add_argument("--reverse", type=int, default=0)
ap.add_argument("--first", type=int, default=0)
a = ap.parse_args()
ops = qcgen.qft(a.n) if a.circuit == "qft" else qcgen.tfxy(a.n, a.steps)
s = qc.State(a.n, a.prec)
s.set_option("fusion", a.fusion)
s.set_option("jit", a.jit)
s.set_option("tile_bits", a.tile)
s.set_option("row_bits", a.rb)
s.set_option("tma_mode", a.tma)
s.init_random(1)
ops = ops[a.first: a.gates] if a.gates else ops[a.first:]
if a.reverse:
    ops = [qcgen.Op(o.name, tuple(a.n - 1 - q for q in o.qubits), o.theta, o.matrix, o.ctrl_state) for o in ops]
arr = qc.encode_ops(ops)
for _ in range(a.reps):
    s.run(arr)
s.sync()
print(s.info())
