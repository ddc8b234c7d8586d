set -x
mkdir -p gpurun_out
timeout 900 python scripts/time_circ.py qft:30:c64 qft:28:c64 tfxy:28:c64 tfxy:20:c64 qft:30 --opts "" row_bits=7 row_bits=5 > gpurun_out/t_c64rb.txt 2>&1; grep -v "^{" gpurun_out/t_c64rb.txt
