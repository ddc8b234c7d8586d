# TMA box L2 promotion (QC_TMAP_PROMO 0 none / 1 64B / 2 128B / 3 256B default) on HBM-bound QFT passes
set -x
cd "${GRAFT_REPO_ROOT:-.}"
for P in 3 0 2; do
  echo "== QC_TMAP_PROMO=$P"
  QC_TMAP_PROMO=$P timeout 900 python scripts/time_circ.py qft:28 qft:30 qft:30:c64 tfxy:28 2>&1 | grep -v "^{"
  QC_TMAP_PROMO=$P timeout 900 python scripts/time_circ.py qft:33 --reps 3 2>&1 | grep -v "^{"
done
