set -x
mkdir -p gpurun_out
W="tfxy:20 tfxy:24 tfxy:28 tfxy:28:c64 qft:24 qft:30 qft:30:c64"
QC_DEFS="QC_COMPUTE_WARPS=16" timeout 600 python -m paper_2303_00123_b200.build > gpurun_out/build16.log 2>&1; tail -2 gpurun_out/build16.log
timeout 1500 python scripts/time_circ.py $W > gpurun_out/t_w16.txt 2>&1; grep -v "^{" gpurun_out/t_w16.txt
QC_DEFS="QC_COMPUTE_WARPS=12" timeout 600 python -m paper_2303_00123_b200.build > gpurun_out/build12.log 2>&1; tail -2 gpurun_out/build12.log
timeout 1500 python scripts/time_circ.py $W > gpurun_out/t_w12.txt 2>&1; grep -v "^{" gpurun_out/t_w12.txt
