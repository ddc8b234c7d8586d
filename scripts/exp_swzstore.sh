set -x
W="tfxy:20 tfxy:24 tfxy:28 tfxy:28:c64 qft:30 qft:30:c64"
for e in "QC_SWZ_STORE=1" "QC_SWZ_STORE=0" "QC_SWZ_STORE=0 QC_SWZ_MIN=1"; do
  env $e timeout 900 python scripts/time_circ.py $W > gpurun_out/t_knob.txt 2>&1; echo "== $e"; grep -v "^{" gpurun_out/t_knob.txt
done
