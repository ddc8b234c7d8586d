set -x
mkdir -p gpurun_out
W="tfxy:20 tfxy:24 tfxy:28 qft:28 qft:30 qft:30:c64 tfxy:28:c64"
timeout 900 python scripts/time_circ.py $W --opts remap=0 remap=1 > gpurun_out/t_w8.txt 2>&1; cat gpurun_out/t_w8.txt | grep -v "^{"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 40 -c 1 -o gpurun_out/prof_tfxy28_remap python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > /dev/null 2>&1
QC_DEFS="-DQC_COMPUTE_WARPS=16" timeout 600 python -m paper_2303_00123_b200.build > gpurun_out/build16.log 2>&1; tail -2 gpurun_out/build16.log
timeout 900 python scripts/time_circ.py $W --opts remap=0 remap=1 > gpurun_out/t_w16.txt 2>&1; cat gpurun_out/t_w16.txt | grep -v "^{"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 40 -c 1 -o gpurun_out/prof_tfxy28_remap_w16 python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > /dev/null 2>&1
ls gpurun_out
