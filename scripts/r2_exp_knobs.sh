# Knob sweep after register frames: swizzle threshold, warps per pass
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for E in "QC_SWZ_MIN=2" "QC_SWZ_MIN=1" "QC_JIT_WARPS=16" "QC_SWZ_MIN=1 QC_JIT_WARPS=16"; do
  echo "== $E"
  env $E timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 2>&1 | grep -v "^{"
done
