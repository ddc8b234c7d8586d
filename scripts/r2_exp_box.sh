# One 5-D TMA box per tile (QC_OPT_TMA_MODE 2): parity + timing, narrow rows
set -x
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python scripts/parity_opts.py tma_mode=2 tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 2>&1 | grep -v " ok$" | tail -8
timeout 1200 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 tfxy:28:c64 --opts "" tma_mode=2 tma_mode=2,row_bits=4 tma_mode=2,row_bits=3 tma_mode=2,row_bits=2 2>&1 | grep -v "^{"
