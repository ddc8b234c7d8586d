set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
W=${W:-"tfxy:20 tfxy:24 tfxy:28 qft:28 qft:30 qft:30:c64 tfxy:28:c64 tfxy:33"}
timeout 1500 python scripts/time_circ.py $W --opts ${OPTS:-remap=0 remap=1} > gpurun_out/t_check.txt 2>&1; grep -v "^{" gpurun_out/t_check.txt
