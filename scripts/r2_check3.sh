# After the sub-tile (group plan) pipeline generalisation: full -m gpu suite, smoke, bench headline
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c3_smoke.log 2>&1; tail -2 gpurun_out/c3_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/c3_pytest_gpu.log 2>&1; tail -4 gpurun_out/c3_pytest_gpu.log
timeout 1200 python bench.py --no-cpu > gpurun_out/c3_bench.json 2> gpurun_out/c3_bench.err; tail -2 gpurun_out/c3_bench.err
python -c "import json; d=json.loads(open('gpurun_out/c3_bench.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['clocks'])"
