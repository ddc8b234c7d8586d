# ncu --set full of TFXY-28 passes after register frames: transitional (2, 5), heavy (7), light (13); QFT-30 c64 pass 1
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for P in 2 5 7; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s $((P+15)) -c 1 -o gpurun_out/prof2_tfxy28_p$P python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 5 -c 1 -o gpurun_out/prof2_qft30c64_p1 python scripts/run_circuit.py --circuit qft --n 30 --prec c64 --reps 3 --jit 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum,smsp__inst_executed_pipe_fp64.sum --clock-control none --csv --log-file gpurun_out/launches2_tfxy28.csv -k regex:qc_pass python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > /dev/null 2>&1
ls -la gpurun_out
