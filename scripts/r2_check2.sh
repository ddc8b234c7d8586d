# Full -m gpu suite after pair passes + restore; TFXY(33) row-bits A/B (auto picks rb=4: 17 passes; rb=3: 15)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu_check2.log 2>&1; tail -14 gpurun_out/pytest_gpu_check2.log
timeout 900 python scripts/time_circ.py tfxy:33 --reps 2 --opts "" row_bits=3 2>&1 | grep -v "^{"
