"""Per-launch DRAM traffic of qc_pass from an ncu --csv launch list
(metrics gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum).

  python scripts/ncu_traffic_csv.py LAUNCHES.csv CONFIG N_LAST [out.json]
Averages the last N_LAST qc_pass launches (one circuit) and merges
{CONFIG: {...}} into profiles/ncu_traffic.json (read by bench.py)."""
import csv, json, os, sys
from collections import defaultdict

src, cfg, nlast = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "profiles", "ncu_traffic.json")
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
per, name = defaultdict(dict), {}
for r in rows[1:]:
    per[int(r[0])][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    name[int(r[0])] = r[ki]
ids = sorted(i for i in per if name[i] == "qc_pass")[-nlast:]
rd = sum(per[i]["dram__bytes_read.sum"] for i in ids) / len(ids)
wr = sum(per[i]["dram__bytes_write.sum"] for i in ids) / len(ids)
du = sum(per[i]["gpu__time_duration.sum"] for i in ids) / len(ids)
res = json.load(open(out)) if os.path.exists(out) else {}
res[cfg] = {"bytes_per_launch": rd + wr, "read_per_launch": rd, "write_per_launch": wr, "launches": len(ids),
            "duration_per_launch": du * 1e3, "duration_unit": "ms",
            "source": os.path.basename(src) + " (ncu launch list, dram__bytes_read.sum + dram__bytes_write.sum, "
                      f"mean over the last {len(ids)} qc_pass launches = one circuit)"}
json.dump(res, open(out, "w"), indent=1)
print(cfg, res[cfg])
