# Planner tile-choice seeds (QC_PLAN_SEEDS 0: greedy + climb; 1: + climb from the best window; 2: climb every window)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
for S in 0 1 2; do
  echo "== QC_PLAN_SEEDS=$S"
  QC_PLAN_SEEDS=$S timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 tfxy:28:c64 --opts "" row_bits=4 2>&1 | grep -v "^{"
  QC_PLAN_SEEDS=$S timeout 900 python scripts/time_circ.py tfxy:33 --reps 2 --opts "" row_bits=4 2>&1 | grep -v "^{"
done
