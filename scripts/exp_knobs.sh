set -x
mkdir -p gpurun_out
W="tfxy:20 tfxy:28 qft:28 qft:30:c64 tfxy:28:c64"
for e in "QC_SWZ_MIN=1" "QC_SWZ_MIN=2" "QC_JIT_WARPS=16" "QC_JIT_WARPS=16 QC_SWZ_MIN=1" "QC_JIT_WARPS=8"; do
  env $e timeout 900 python scripts/time_circ.py $W > gpurun_out/t_knob.txt 2>&1; echo "== $e"; grep -v "^{" gpurun_out/t_knob.txt
done
