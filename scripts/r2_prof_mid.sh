# ncu --set full of mid-regime TFXY-28 passes (1, 3) and the light pass 10: are they smem-bound?
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for P in 1 3 10; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qc_pass -s $P -c 1 -o gpurun_out/prof_mid_tfxy28_p$P python scripts/run_circuit.py --circuit tfxy --n 28 --steps 10 --reps 3 --jit 2 > gpurun_out/prof_mid_p$P.log 2>&1
done
ls -la gpurun_out
