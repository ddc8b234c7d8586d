set -x
mkdir -p gpurun_out
W="tfxy:20 tfxy:24 tfxy:28 tfxy:28:c64 qft:30 qft:30:c64"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random_circuits_jit" > gpurun_out/pytest_q.log 2>&1; tail -3 gpurun_out/pytest_q.log
timeout 900 python scripts/time_circ.py $W > gpurun_out/t_mx.txt 2>&1; grep -v "^{" gpurun_out/t_mx.txt | tail -8
