# Row transports: gather4 (default), SIMT cp.async (2), gather4 loads + SIMT stores (3); narrow rows
set -x
cd "${GRAFT_REPO_ROOT:-.}"
timeout 600 python scripts/parity_opts.py tma_mode=3 tma_mode=3,row_bits=4 2>&1 | tail -3
timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 qft:30 qft:30:c64 --opts "" tma_mode=3 tma_mode=3,row_bits=5 tma_mode=3,row_bits=4 tma_mode=3,row_bits=3 2>&1 | grep -v "^{"
