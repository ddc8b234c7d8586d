# Round 2: smoke, default bench (C4 TFXY-33 headline), reference arm, launch list and a single-pass
# DRAM-traffic capture of the TFXY-33 fused pass (no replay needed for these metrics).
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
lscpu > gpurun_out/lscpu.txt 2>&1; free -g >> gpurun_out/lscpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -4 gpurun_out/smoke.log
timeout 1200 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-sweep --no-cpu > gpurun_out/bench_ncu.log 2>&1
ls -la gpurun_out/
