# Box transport: row-bit sweep at the headline sizes and for c64
set -x
cd "${GRAFT_REPO_ROOT:-.}"
timeout 1200 python scripts/time_circ.py qft:30:c64 tfxy:28:c64 tfxy:30:c64 --opts tma_mode=2,row_bits=7 tma_mode=2,row_bits=6 tma_mode=2,row_bits=5 tma_mode=2,row_bits=4 2>&1 | grep -v "^{"
timeout 1200 python scripts/time_circ.py qft:33 --reps 2 --opts "" tma_mode=2 tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 2>&1 | grep -v "^{"
timeout 1500 python scripts/time_circ.py tfxy:33 --reps 2 --opts tma_mode=2 tma_mode=2,row_bits=5 tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 2>&1 | grep -v "^{"
