python -m paper_2303_00123_b200.build
for c in "qft --n 30" "qft --n 30 --prec c64" "tfxy --n 28 --steps 2"; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:qc_pass python scripts/run_circuit.py --circuit $c --reps 1 --jit 2 2>/dev/null | grep qc_pass | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"' | paste -sd' ' | sed "s/^/$c: /"
done
