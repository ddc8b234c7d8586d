"""Key metrics of every qc_pass launch in one or more .ncu-rep captures (text)."""
import csv, io, subprocess, sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_sol_%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_sol_%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pipe_%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
        ("launch__registers_per_thread", "regs"), ("smsp__inst_executed.sum", "warp_insts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_%"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts")]
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    print(f"== {rep}")
    for r in rows[2:]:
        if len(r) != len(h) or "qc_pass" not in r[h.index("Kernel Name")]:
            continue
        parts = []
        for k, name in KEYS:
            if k in h:
                parts.append(f"{name}={r[h.index(k)]}{'' if u[h.index(k)] in ('', '%') else ' ' + u[h.index(k)]}")
        st = sorted(((float(r[i]), h[i]) for i in range(len(h)) if "average_warps_issue_stalled" in h[i]
                     and "per_issue_active" in h[i] and r[i] not in ("", "n/a")), reverse=True)[:4]
        parts.append("top stalls: " + ", ".join(f"{n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {x:.2f}" for x, n in st))
        print("  qc_pass: " + ", ".join(parts))
