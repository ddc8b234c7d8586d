python -m paper_2303_00123_b200.build
ncu --set full --clock-control none --import-source on -k regex:fused -s 30 -c 1 -o gpurun_out/prof_tfxy20 python scripts/run_circuit.py --circuit tfxy --n 20 --reps 2 > gpurun_out/prof_tfxy20.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused -s 4 -c 1 -o gpurun_out/prof_qft26 python scripts/run_circuit.py --circuit qft --n 26 --reps 2 > gpurun_out/prof_qft26.log 2>&1
ls -la gpurun_out
