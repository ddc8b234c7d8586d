set -x
mkdir -p gpurun_out
W="tfxy:20 tfxy:28 qft:30 qft:30:c64 tfxy:28:c64"
for m in 1 2 3 4; do
  QC_SWZ_MIN=$m timeout 900 python scripts/time_circ.py $W --opts remap=0 remap=1 > gpurun_out/t_swz$m.txt 2>&1; grep -v "^{" gpurun_out/t_swz$m.txt
done
QC_DEFS="QC_COMPUTE_WARPS=12 QC_GROUPS=3" timeout 600 python -m paper_2303_00123_b200.build > gpurun_out/build12.log 2>&1; tail -2 gpurun_out/build12.log
for m in 1 4; do
  QC_SWZ_MIN=$m timeout 600 python scripts/time_circ.py $W --opts remap=1 > gpurun_out/t_g3_swz$m.txt 2>&1; grep -v "^{" gpurun_out/t_g3_swz$m.txt
done
