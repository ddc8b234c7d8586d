# Per-warp tag poll + empty-barrier arrive (QC_WARP_SYNC=1) vs per-thread: parity, racecheck/synccheck, timing
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
QC_WARP_SYNC=1 timeout 600 python scripts/parity_opts.py "" 2>&1 | tail -2
export QC_JIT_CACHE=/tmp/qcjit_ws
for tool in racecheck synccheck; do
  QC_WARP_SYNC=1 timeout 900 compute-sanitizer --tool $tool --print-limit 5 python scripts/run_circuit.py --circuit tfxy --n 16 --steps 3 --reps 2 --jit 2 > gpurun_out/ws_${tool}.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/ws_${tool}.txt | tail -1)"
done
unset QC_JIT_CACHE
for W in 0 1 0 1; do
  echo "== QC_WARP_SYNC=$W"
  QC_WARP_SYNC=$W timeout 600 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 2>&1 | grep -v "^{"
done
for W in 0 1; do QC_WARP_SYNC=$W timeout 600 python scripts/time_circ.py tfxy:33 --reps 2 2>&1 | grep -v "^{"; done
