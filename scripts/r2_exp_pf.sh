# L2 prefetch distance of the fused-pass producer (QC_PF) A/B
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
QC_PF=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "jit or fused" > gpurun_out/pf_pytest.log 2>&1; tail -2 gpurun_out/pf_pytest.log
for P in 0 1 2 3 4; do
  echo "== QC_PF=$P"
  QC_PF=$P timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 2>&1 | grep -v "^{"
done
