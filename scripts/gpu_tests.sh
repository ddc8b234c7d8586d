#!/bin/bash
# Round-2 GPU check: full -m gpu suite + smoke, logs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; free -g >> gpurun_out/lscpu.txt
timeout 2400 python -m pytest tests -m gpu -x -q -s ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -3 gpurun_out/pytest_gpu.log
