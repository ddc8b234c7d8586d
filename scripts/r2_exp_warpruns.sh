# Warp-private sub-stage runs (group barrier -> __syncwarp, QC_JIT_WARP_RUNS=1 default) vs off: parity + timing
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py tests/test_gpu_mgate.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/warpruns_pytest.log 2>&1; tail -2 gpurun_out/warpruns_pytest.log
for R in 0 1; do
  echo "== QC_JIT_WARP_RUNS=$R"
  QC_JIT_WARP_RUNS=$R timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 tfxy:20 2>&1 | grep -v "^{"
  QC_JIT_WARP_RUNS=$R timeout 900 python scripts/time_circ.py tfxy:33 --reps 3 2>&1 | grep -v "^{"
done
