# Full register frames (pivot -> exactly 1; QC_JIT_FRAMES=2) vs unit-phase frames (=1): parity + timing A/B
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py tests/test_gpu_mgate.py tests/test_gpu_dist.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/frames2_pytest.log 2>&1; tail -3 gpurun_out/frames2_pytest.log
for F in 2 1; do
  echo "== QC_JIT_FRAMES=$F"
  QC_JIT_FRAMES=$F timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 tfxy:20 2>&1 | grep -v "^{"
done
for F in 2 1; do QC_JIT_FRAMES=$F timeout 600 python scripts/time_circ.py tfxy:33 --reps 2 2>&1 | grep -v "^{"; done
