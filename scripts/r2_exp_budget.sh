# Planner FP64 budget / tile size experiment (TFXY-30, TFXY-33)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for B in 0 200 300 400 600; do
  echo "== QC_PASS_FLOPS=$B"
  QC_PASS_FLOPS=$B timeout 900 python scripts/time_circ.py tfxy:30 --opts "" tile_bits=11 2>&1 | tail -3
done
for B in 0 400; do
  echo "== n33 QC_PASS_FLOPS=$B"
  QC_PASS_FLOPS=$B timeout 900 python scripts/time_circ.py tfxy:33 --reps 2 2>&1 | tail -2
done
