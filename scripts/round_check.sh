# Full round check on one B200: smoke, GPU tests, bench (+sweep, cpu baseline), reference arm,
# launch list and ncu --set full captures of the dominant kernel (bench workload, TFXY-28, QFT-30).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; tail -14 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 45 -c 2 -o gpurun_out/prof_bench_tfxy20 python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 20 -c 1 -o gpurun_out/prof_tfxy28 python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s 5 -c 1 -o gpurun_out/prof_qft30 python scripts/run_circuit.py --circuit qft --n 30 --reps 3 --jit 2 > /dev/null 2>&1
ls -la gpurun_out/
