# Global-store last sub-stage: parity + timing A/B (QC_JIT_GSTORE=1 vs 0)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_midsize.py -m gpu -x -q > gpurun_out/gst_pytest.log 2>&1; tail -3 gpurun_out/gst_pytest.log
for G in 1 0; do
  echo "== QC_JIT_GSTORE=$G"
  QC_JIT_GSTORE=$G timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 tfxy:20 2>&1 | grep -v "^{"
done
QC_JIT_GSTORE=1 timeout 600 python scripts/time_circ.py tfxy:33 --reps 2 2>&1 | grep -v "^{"
