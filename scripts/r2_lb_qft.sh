# Why is loopback QFT(30) slow?  launch list of one warm run (both exchange modes)
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/lb_qft_launches.csv python scripts/time_pair.py qft:30:2 > gpurun_out/lb_qft.log 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/lb_qft_launches.csv')) if len(r)>10]
h=rows[0]; ki,mi,vi=(h.index(x) for x in ("Kernel Name","Metric Name","Metric Value"))
per=defaultdict(dict); nm={}
for r in rows[1:]:
    per[int(r[0])][r[mi]]=float(r[vi].replace(',','')); nm[int(r[0])]=r[ki]
for i in sorted(per)[-60:]:
    print(i, nm[i][:40], round(per[i]['gpu__time_duration.sum']/1e6,3), 'ms', round((per[i]['dram__bytes_read.sum']+per[i]['dram__bytes_write.sum'])/1e9,2), 'GB')
PY
