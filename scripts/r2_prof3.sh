# ncu --set full with the round-2 default transport (box, auto row bits): TFXY-30 heaviest pass, QFT-30 pass, launch list
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_tfxy30_box.csv -k regex:qc_pass python scripts/run_circuit.py --circuit tfxy --n 30 --steps 10 --reps 2 --jit 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s ${HEAVY} -c 1 -o gpurun_out/prof3_tfxy30_heavy python scripts/run_circuit.py --circuit tfxy --n 30 --steps 10 --reps 2 --jit 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 4 -c 1 -o gpurun_out/prof3_qft30 python scripts/run_circuit.py --circuit qft --n 30 --reps 2 --jit 2 > /dev/null 2>&1
ls -la gpurun_out
