set -x
mkdir -p gpurun_out
W="tfxy:20 tfxy:24 tfxy:28 tfxy:28:c64 qft:30 qft:30:c64"
timeout 1500 python scripts/time_circ.py $W --opts "" tma_mode=1 tma_mode=1,row_bits=5 tma_mode=1,row_bits=7 > gpurun_out/t_tma.txt 2>&1; grep -v "^{" gpurun_out/t_tma.txt
