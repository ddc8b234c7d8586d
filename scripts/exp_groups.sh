set -x
mkdir -p gpurun_out
W="tfxy:16 tfxy:20 tfxy:24 qft:20 qft:24"
timeout 900 python scripts/time_circ.py $W --opts "" tile_bits=11 tile_bits=10 > gpurun_out/t_g2.txt 2>&1; grep -v "^{" gpurun_out/t_g2.txt
QC_DEFS="QC_GROUPS=1" timeout 600 python -m paper_2303_00123_b200.build > gpurun_out/build_g1.log 2>&1; tail -1 gpurun_out/build_g1.log
timeout 900 python scripts/time_circ.py $W tfxy:28 qft:30 --opts "" tile_bits=11 tile_bits=10 > gpurun_out/t_g1.txt 2>&1; grep -v "^{" gpurun_out/t_g1.txt
