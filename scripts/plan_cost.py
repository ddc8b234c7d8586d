"""Host-only cost model of a fused plan (planner experiments without a GPU).

  python scripts/plan_cost.py [n] [steps]
Per pass: t = sqrt(H^2 + F^2) with H = the HBM time of one pass (2*Ns at
6.25 TB/s) and F = the pass's algorithmic flops / 26 TFLOP/s -- calibrated on
the round-2 ncu launch list of TFXY-33 (profiles/round2_launches_tfxy33_frames.csv:
model 1.96 s vs 1.96 s measured)."""
import os, re, subprocess, sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
code = (f"import qcgen\nfrom paper_2303_00123_b200 import qc\n"
        f"print(qc.debug_plan({n}, qcgen.tfxy({n},{steps})))")
env = dict(os.environ, QC_PLAN_DEBUG="1")
r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                   cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
fl = [float(m) for m in re.findall(r"flops/amp ([0-9.]+)", r.stderr)]
H = 2 * (16 << n) / 6.25e12 * 1e3
ts = [((H * H) + (f * (1 << n) / 26e12 * 1e3) ** 2) ** 0.5 for f in fl]
print(f"n={n}: {len(fl)} passes, model {sum(ts):.0f} ms;", " ".join(f"{t:.0f}" for t in ts))
