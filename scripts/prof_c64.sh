set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 5 -c 1 -o gpurun_out/prof_qft30c64 python scripts/run_circuit.py --circuit qft --n 30 --prec c64 --reps 3 --jit 2 > /dev/null 2>&1
ls gpurun_out
