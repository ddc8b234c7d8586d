# One compute group for passes below 100 flop/amp (default now) vs never (QC_JIT_MID=none)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py -m gpu -q -x > gpurun_out/light_pytest.log 2>&1; tail -2 gpurun_out/light_pytest.log
for M in none ""; do
  echo "== QC_JIT_MID=$M"
  QC_JIT_MID=$M timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:28 qft:30 qft:30:c64 2>&1 | grep -v "^{"
  QC_JIT_MID=$M timeout 900 python scripts/time_circ.py tfxy:33 qft:33 --reps 3 2>&1 | grep -v "^{"
done
