# quick A/B: parity tests + circuit sweep (usage: bash scripts/exp_sweep.sh "<circuits>")
C=${1:-tfxy20+qft30+tfxy28+qft30c64}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python scripts/circ_sweep.py $C 0,0,0 2>&1 | grep -v "^{"
