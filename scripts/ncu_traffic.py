"""Per-launch DRAM traffic of qc_pass from an ncu --set full capture.

  python scripts/ncu_traffic.py REPORT.ncu-rep CONFIG [out.json]
Merges {CONFIG: {bytes_per_launch, duration_us, launches, source}} into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic)."""
import csv, io, json, os, subprocess, sys

rep, cfg = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                         "profiles", "ncu_traffic.json")
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
data = [r for r in rows[2:] if len(r) == len(h) and "qc_pass" in r[h.index("Kernel Name")]]


def col(name, r):
    return float(r[h.index(name)].replace(",", ""))


def scale(name):
    u = rows[1][h.index(name)]
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


rd = [col("dram__bytes_read.sum", r) * scale("dram__bytes_read.sum") for r in data]
wr = [col("dram__bytes_write.sum", r) * scale("dram__bytes_write.sum") for r in data]
du = [col("gpu__time_duration.sum", r) for r in data]
res = json.load(open(out)) if os.path.exists(out) else {}
res[cfg] = {"bytes_per_launch": (sum(rd) + sum(wr)) / len(data), "read_per_launch": sum(rd) / len(data),
            "write_per_launch": sum(wr) / len(data), "launches": len(data),
            "duration_per_launch": sum(du) / len(data), "duration_unit": rows[1][h.index("gpu__time_duration.sum")],
            "source": os.path.basename(rep) + " (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum)"}
json.dump(res, open(out, "w"), indent=1)
print(cfg, res[cfg])
