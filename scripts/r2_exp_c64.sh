# QFT-30 c64 / c128 tile and row geometry
set -x
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python scripts/time_circ.py qft:30:c64 --opts "" tile_bits=12 row_bits=6 row_bits=8 tile_bits=12,row_bits=6 2>&1 | grep -v "^{"
timeout 900 python scripts/time_circ.py qft:30 --opts "" tile_bits=11 row_bits=5 row_bits=7 2>&1 | grep -v "^{"
