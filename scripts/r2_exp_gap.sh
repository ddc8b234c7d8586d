# Inter-pass gaps: PDL on/off, graph on/off (TFXY-30, QFT-30)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
for E in "QC_PDL=1" "QC_PDL=0"; do
  echo "== $E"
  env $E timeout 900 python scripts/time_circ.py tfxy:30 qft:30 tfxy:28 --opts "" use_graph=0 2>&1 | grep -v "^{"
done
