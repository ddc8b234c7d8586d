# GPU tests + bench (with sweep) on one B200
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
sw = d.pop("sweep", {})
print(json.dumps({k: d[k] for k in ("value", "ms_per_step", "roofline", "e2e")}))
print(json.dumps(sw.get("circuit_ms_vs_qubits")))
print(json.dumps(sw.get("north_star_n33_c128")))
PY
