# Round 2 after full register frames: bench (C4 headline + sweep), reference arm, launch list with DRAM
# bytes of the bench workload, and ncu --set full of the heaviest TFXY-28 pass
set -x
cd "${GRAFT_REPO_ROOT:-.}"
bash scripts/r2_bench.sh
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 7 -c 1 -o gpurun_out/prof_frames_tfxy28_p7 python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > gpurun_out/prof_frames_p7.log 2>&1
ls -la gpurun_out
