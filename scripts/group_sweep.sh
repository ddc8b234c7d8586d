for lib in g1 g2; do
  QC_LIB=$PWD/paper_2303_00123_b200/libqc_$lib.so timeout 900 python scripts/circ_sweep.py qft30+tfxy28+tfxy20 12,5,0 11,5,0 12,6,0 2>&1 | grep -v "^{" | sed "s/^/$lib /"
  QC_LIB=$PWD/paper_2303_00123_b200/libqc_$lib.so timeout 900 python scripts/circ_sweep.py qft30c64 13,6,0 12,6,0 12,5,0 2>&1 | grep -v "^{" | sed "s/^/$lib /"
done
