# Mid-regime passes with one compute group of 8 warps (two ring buffers in flight): QC_JIT_MID=lo:hi
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
QC_JIT_MID=0:100000 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "random or qft or tfxy" > gpurun_out/mid_pytest.log 2>&1; tail -2 gpurun_out/mid_pytest.log
for M in "" 80:300 100:250 60:400 0:100000; do
  echo "== QC_JIT_MID=$M"
  QC_JIT_MID=$M timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 2>&1 | grep -v "^{"
done
for M in "" 80:300; do QC_JIT_MID=$M timeout 600 python scripts/time_circ.py tfxy:33 --reps 2 2>&1 | grep -v "^{"; done
