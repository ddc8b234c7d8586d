# TFXY with narrower TMA rows (more free tile bits per pass, fewer passes)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python scripts/time_circ.py tfxy:30 --opts "" row_bits=5 row_bits=4 2>&1 | grep -v "^{"
timeout 900 python scripts/time_circ.py tfxy:33 --reps 2 --opts row_bits=4 row_bits=5 2>&1 | grep -v "^{"
