# Planner swaps deferred to a permuted final store (QC_JIT_PSTORE) A/B + parity
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py tests/test_gpu_mgate.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pstore_pytest.log 2>&1; tail -3 gpurun_out/pstore_pytest.log
for E in 1 0; do
  echo "== QC_JIT_PSTORE=$E"
  QC_JIT_PSTORE=$E timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 tfxy:28:c64 tfxy:20 2>&1 | grep -v "^{"
done
QC_JIT_PSTORE=1 timeout 600 python scripts/time_circ.py tfxy:33 --reps 2 2>&1 | grep -v "^{"
