# Round-2 final check on one B200: smoke, full -m gpu suite, bench (C4 headline + sweep + CPU baselines),
# reference arm, ncu launch list with DRAM bytes of the bench workload, ncu --set full of a heavy TFXY-28 pass
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -3 gpurun_out/final_smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/final_pytest_gpu.log 2>&1; tail -14 gpurun_out/final_pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -3 gpurun_out/final_bench.err
timeout 400 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu > gpurun_out/final_bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 7 -c 1 -o gpurun_out/final_prof_tfxy28_p7 python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > gpurun_out/final_prof.log 2>&1
ls -la gpurun_out/
