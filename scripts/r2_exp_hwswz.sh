# TMA 128-byte swizzled tiles (QC_HW_SWZ=1, complex128): parity + timing A/B
set -x
cd "${GRAFT_REPO_ROOT:-.}"
QC_HW_SWZ=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mgate.py -m gpu -q -x > gpurun_out/hwswz_pytest.log 2>&1; tail -3 gpurun_out/hwswz_pytest.log
QC_HW_SWZ=1 timeout 600 python scripts/parity_opts.py "" row_bits=4 row_bits=3 2>&1 | grep -v " ok$" | tail -4
for E in 0 1; do
  echo "== QC_HW_SWZ=$E"
  QC_HW_SWZ=$E timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 2>&1 | grep -v "^{"
done
QC_HW_SWZ=1 timeout 900 python scripts/time_circ.py tfxy:33 --reps 2 2>&1 | grep -v "^{"
