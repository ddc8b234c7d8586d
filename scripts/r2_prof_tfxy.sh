# ncu --set full of TFXY-28 fused passes: the heaviest (pass 7, 512 flop/amp), a mid one (pass 3) and a light one (13)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for P in 7 3 13; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s $P -c 1 -o gpurun_out/prof_tfxy28_p$P python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > gpurun_out/prof_p$P.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed.sum --clock-control none --csv --log-file gpurun_out/launches_tfxy28.csv -k regex:qc_pass python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > /dev/null 2>&1
ls -la gpurun_out
