python -m paper_2303_00123_b200.build
export QC_JIT_DUMP=gpurun_out/jd7
mkdir -p $QC_JIT_DUMP
ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 1 -c 1 -o gpurun_out/prof7_qft28c64 python scripts/run_circuit.py --circuit qft --n 28 --reps 1 --jit 2 --prec c64 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 1 -c 1 -o gpurun_out/prof7_qft28 python scripts/run_circuit.py --circuit qft --n 28 --reps 1 --jit 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 10 -c 2 -o gpurun_out/prof7_tfxy20 python scripts/run_circuit.py --circuit tfxy --n 20 --reps 2 --jit 2 > /dev/null 2>&1
ls gpurun_out
