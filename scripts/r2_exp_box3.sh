# Box transport with several boxes per tile (> 5 bit runs): parity + headline sizes
set -x
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python scripts/parity_opts.py tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 tma_mode=2,row_bits=2 2>&1 | grep -v " ok$" | tail -8
timeout 1200 python scripts/time_circ.py tfxy:30 qft:30 qft:30:c64 tfxy:30:c64 --opts tma_mode=2,row_bits=5 tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 2>&1 | grep -v "^{"
timeout 1200 python scripts/time_circ.py qft:33 --reps 2 --opts tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 2>&1 | grep -v "^{"
timeout 1500 python scripts/time_circ.py tfxy:33 --reps 2 --opts tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 2>&1 | grep -v "^{"
