# One vs two compute groups for 8-warp passes (QC_JIT_GROUPS8), all-8-warp passes
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
QC_JIT_GROUPS8=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "jit or fused" > gpurun_out/grp_pytest.log 2>&1; tail -2 gpurun_out/grp_pytest.log
for E in "QC_JIT_GROUPS8=2" "QC_JIT_GROUPS8=1" "QC_JIT_WARPS=8 QC_JIT_GROUPS8=1" "QC_JIT_WARPS=8 QC_JIT_GROUPS8=2"; do
  echo "== $E"
  env $E timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 2>&1 | grep -v "^{"
done
