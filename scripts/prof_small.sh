set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 4 -c 2 -o gpurun_out/prof_qft16 python scripts/run_circuit.py --circuit qft --n 16 --reps 4 --jit 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 20 -c 3 -o gpurun_out/prof_tfxy20 python scripts/run_circuit.py --circuit tfxy --n 20 --steps 10 --reps 4 --jit 2 > /dev/null 2>&1
ls gpurun_out
