# Select network from one bank-group slot bit on in light / mid passes (QC_SWZ1_FLOPS = flop/amp threshold)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
QC_SWZ1_FLOPS=300 timeout 600 python scripts/parity_opts.py "" 2>&1 | tail -1
for F in 0 150 300 500 0 300; do
  echo "== QC_SWZ1_FLOPS=$F"
  QC_SWZ1_FLOPS=$F timeout 600 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 qft:28 2>&1 | grep -v "^{"
done
for F in 0 300; do QC_SWZ1_FLOPS=$F timeout 600 python scripts/time_circ.py tfxy:33 qft:33 --reps 2 2>&1 | grep -v "^{"; done
