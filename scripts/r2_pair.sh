# Collective-fused pair passes (QC_OPT_EXCHANGE 2) on one GPU: loopback parity (all transports, AOT/JIT),
# the rest of the sharded + parity suites, and loopback timing exchange 0 vs 2
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_nccl.py -m gpu -q -x > gpurun_out/pair_pytest.log 2>&1; tail -5 gpurun_out/pair_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_mgate.py -m gpu -q -x > gpurun_out/pair_pytest2.log 2>&1; tail -3 gpurun_out/pair_pytest2.log
timeout 600 python scripts/time_pair.py qft:30:2 qft:30:8 tfxy:28:2 2>&1 | tail -8
