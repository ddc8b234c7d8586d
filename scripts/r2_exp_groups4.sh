# 4 compute groups of 4 warps on 32 KiB tiles (QC_JIT_GROUPS=4, tile_bits=11): 4 tiles under compute, 2 in flight
set -x
cd "${GRAFT_REPO_ROOT:-.}"
QC_JIT_GROUPS=4 timeout 600 python scripts/parity_opts.py tile_bits=11 "tile_bits=11,row_bits=4" 2>&1 | tail -6
timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 --opts "" tile_bits=11 2>&1 | grep -v "^{"
QC_JIT_GROUPS=4 timeout 900 python scripts/time_circ.py tfxy:28 tfxy:30 --opts tile_bits=11 2>&1 | grep -v "^{"
QC_JIT_GROUPS=4 timeout 900 python scripts/time_circ.py tfxy:33 --reps 2 --opts tile_bits=11 2>&1 | grep -v "^{"
