"""bench.py -- QFT / TFXY circuit time on B200 through libqc (the C ABI).

Default workload = BASELINE.json configs[1]: TFXY 1D Trotter circuit, 20
qubits, 10 Trotter steps, complex double, random initial state, 1 B200.
A "step" is one qc_run_circuit of the whole circuit on the resident state.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config tfxy20|qft10|qft30|qft30c64|tfxy33] [--no-sweep]

Under torchrun (N > 1) every rank runs its own replica of the workload
("replicas only": the default workload does not shard), timing
is max over ranks, value = N*K circuits / max time ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QFT & TFXY circuit time vs qubits at 1-8 B200; per-gate HBM GB/s vs peak"

CONFIGS = {
    # name: (family, n, steps, precision, description)
    "qft10": ("qft", 10, 0, "c128", "QFT on 10 qubits, complex double, random initial state"),
    "tfxy20": ("tfxy", 20, 10, "c128", "TFXY 1D Trotter circuit, 20 qubits, 10 time steps, complex double, 1 B200"),
    "qft30": ("qft", 30, 0, "c128", "QFT on 30 qubits, complex double, 1 B200"),
    "qft30c64": ("qft", 30, 0, "c64", "QFT on 30 qubits, complex single, 1 B200"),
    "tfxy33": ("tfxy", 33, 10, "c128", "TFXY Trotter circuit, 33 qubits complex double, 1 B200"),
    # sharded (one process per GPU, NCCL qubit-swap exchanges): n = local + log2(N)
    "qft_shard": ("qft", None, 0, "c128",
                  "QFT complex double sharded over N B200 by the top log2(N) qubits (weak scaling)"),
}


def build_ops(cfg, n=None):
    import qcgen
    fam, n0, steps, prec, _ = CONFIGS[cfg]
    n = n0 if n is None else n
    return qcgen.qft(n) if fam == "qft" else qcgen.tfxy(n, steps)


# Algorithmic flops per amplitude of each unfused gate: dense
# 1q 14, dense 2q 30, a diagonal factor 6 per touched amplitude, 0 for
# permutations (X, CNOT, SWAP, CCX; Y and CZ are sign / i-multiples).
FLOPS_PER_AMP = {"H": 14, "RX": 14, "RY": 14, "U1": 14, "RZ": 6, "P": 3, "CP": 1.5, "Z": 0, "CZ": 0,
                 "Y": 0, "X": 0, "CNOT": 0, "SWAP": 0, "CCX": 0, "CU1": 7, "U2": 30}


def circuit_flops(ops, n):
    return float(sum(FLOPS_PER_AMP[o.name] for o in ops)) * float(1 << n)


def load_traffic(cfg):
    """dram read+write bytes per launch of qc_pass from the committed ncu
    --set full capture of this workload (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f).get(cfg)
        return (d["bytes_per_launch"], d["source"]) if d else (None, None)
    except Exception:
        return None, None


def derived_fma_peak(prec, device=0):
    """ALU roofline denominator derived from unit counts and clocks (DESIGN
    section 6): SMs x FMA lanes per SM per clock (FP64 64, FP32 128 on
    sm_100) x 2 flops x the max SM clock (MEASURED_PEAKS.json sm_max_mhz).
    qc_debug_fma_peak measures 92 % of it (bench sweep, fma_peak_TFLOPs)."""
    import torch
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f)["sm_max_mhz"])
    except Exception:
        mhz = 1965.0
    lanes = 64 if prec == "c128" else 128
    tf = sms * lanes * 2 * mhz * 1e6 / 1e12
    return tf, (f"derived: {sms} SMs x {lanes} {'FP64' if prec == 'c128' else 'FP32'} FMA/clk/SM x 2 flops x "
                f"{mhz:.0f} MHz (sm_max_mhz)")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------- CPU oracle
def cpu_oracle_rate(cfg: str, budget_s: float = 15.0, n_override=None):
    """Time the oracle (as it stands) on the host cores on a bounded prefix of
    the same circuit; returns circuits/s extrapolated from the prefix."""
    import oracle
    import qcgen
    fam, n, steps, prec, _ = CONFIGS[cfg]
    n = n if n_override is None else n_override
    ops = build_ops(cfg, n)
    n_s = min(n, 24)  # largest size the host holds comfortably for a bounded sample
    st = qcgen.random_state(n_s, precision=prec)
    sample_ops = ops if n_s == n else [o for o in ops if max(o.qubits) < n_s]
    done, t0 = 0, time.perf_counter()
    psi = st
    chunk = 8
    while done < len(sample_ops) and time.perf_counter() - t0 < budget_s:
        psi = oracle.run(n_s, psi, sample_ops[done:done + chunk])
        done += min(chunk, len(sample_ops) - done)
    el = time.perf_counter() - t0
    per_gate = el / max(done, 1) * (2.0 ** (n - n_s))
    rate = 1.0 / (per_gate * len(ops))
    sample = (f"first {done} of {len(ops)} gates of the {cfg} circuit at n={n_s}"
              + ("" if n_s == n else f", per-gate time scaled x2 per qubit to n={n} (P:112 law)")
              + f", {el:.1f} s")
    return rate, oracle.max_threads(), sample


# ----------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2303_00123_b200 as qc

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    fam, n, steps_c, prec, desc = CONFIGS[args.config]
    ops = build_ops(args.config)
    arr = qc.encode_ops(ops)
    s = qc.State(n, prec, device=local_rank)
    stream = torch.cuda.ExternalStream(s.stream, device=dev)
    s.init_random(12345)
    state_bytes = (16 if prec == "c128" else 8) << n
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        s.run(arr)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        info = s.info()
        launches_per_step = info["last_launches"]
        passes = info["last_passes"]
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        clk = ClockSampler(local_rank)
        clk.start()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (not inside the events)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        clocks = clk.stop()
    per = [a.elapsed_time(b) for a, b in ev]  # ms
    t_total = sum(per)
    if world > 1:
        t = torch.tensor([t_total], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_total = float(t.item())
    ms_per_step = t_total / args.steps
    value = world * args.steps / (t_total / 1e3)

    # ---- e2e: pinned host state in, circuit, full state out, every step
    # (states above 8 GiB share one pinned buffer for input and output: the
    # read-back of step i is the upload of step i+1 -- same bytes moved)
    h_in = torch.empty(state_bytes, dtype=torch.uint8, pin_memory=True)
    h_out = h_in if state_bytes > (8 << 30) else torch.empty(state_bytes, dtype=torch.uint8, pin_memory=True)
    s.read_ptr(h_in.data_ptr(), 1 << n)  # a valid state to start from
    e2e_steps = max(1, min(args.steps, 5 if state_bytes <= (8 << 30) else 2))
    torch.cuda.synchronize()
    e_ev = []
    for i in range(e2e_steps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        s.write_ptr(h_in.data_ptr(), 1 << n)
        s.run(arr)
        s.read_ptr(h_out.data_ptr(), 1 << n)
        b.record(stream)
        if i > 0:
            e_ev.append((a, b))
    torch.cuda.synchronize()
    e_ms = sum(a.elapsed_time(b) for a, b in e_ev) / len(e_ev)
    if world > 1:
        t = torch.tensor([e_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e_ms = float(t.item())

    peak, peak_kind = load_peaks()
    # dominant kernel = the fused pass (every launch of the step is one).
    # HBM view: algorithmic bytes per launch = read + write of the state (2*Ns).
    # ALU view: algorithmic flops of the fused plan's ops per launch, against
    # the FP64 (c128) / FP32 (c64) FMA peak derived from unit counts and
    # clocks.  TFXY is bound by the FP64 pipe (block-fused pair blocks, ~8 FP64
    # instructions per amplitude each), QFT by HBM.
    avg_launch_ms = ms_per_step / max(launches_per_step, 1)
    achieved = 2 * state_bytes / (avg_launch_ms / 1e3) / 1e9
    fma_peak, fma_src = derived_fma_peak(prec, local_rank)
    flops = info["last_flops_per_amp"] * float(1 << n)
    alu_achieved = flops / max(launches_per_step, 1) / (avg_launch_ms / 1e3) / 1e12
    traffic, traffic_src = load_traffic(args.config)
    hbm_view = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)", "bytes_per_launch": 2 * state_bytes}
    alu_view = {"bound": "alu", "achieved": alu_achieved, "peak": fma_peak, "unit": "TFLOP/s",
                "frac": alu_achieved / fma_peak,
                "peak_source": fma_src,
                "flops_per_launch": flops / max(launches_per_step, 1),
                "flops_note": "algorithmic flops of the fused plan's ops (qc_info.last_flops_per_amp: complex "
                              "arithmetic, general cmul 6 / cmac 8 flops, unit coefficients free, x fraction of "
                              "amplitudes touched) x 2^n, / fused launches per step",
                "unfused_gate_flops_per_step": circuit_flops(ops, n)}
    main_view = alu_view if fam == "tfxy" else hbm_view
    out = {
        "metric": METRIC, "value": value, "unit": "circuit/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if prec == "c128" else "f32", "data": "synthetic",
        "config": {"workload": desc, "circuit": fam, "qubits": n, "trotter_steps": steps_c or None,
                   "gates": len(ops), "precision": prec, "state_bytes": state_bytes,
                   "initial_state": "splitmix64 seed 12345 (DESIGN input recipe)",
                   "l2": "flushed (512 MiB write) between timed iterations",
                   "parallelism": f"replicas x{world}", "fused_passes_per_step": passes,
                   "tile_bits": info["tile_bits"], "cuda_graph": info["last_graph"],
                   "jit_specialised": info["last_jit"], "ops_after_block_fusion": info["last_blocks"]},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {**main_view, "kernel": "qc_pass (NVRTC-specialised fused tile pass)",
                     "traffic": traffic, "traffic_source": traffic_src,
                     "avg_launch_ms": avg_launch_ms, "hbm_view": hbm_view, "alu_view": alu_view,
                     "note": "avg launch = timed step time / fused launches per step (every launch of "
                             "the step is a fused pass, timed by CUDA events on the state's stream)"},
        "e2e": {"value": world / (e_ms / 1e3), "unit": "circuit/s", "h2d_bytes_per_step": state_bytes,
                "d2h_bytes_per_step": state_bytes, "ms_per_step": e_ms},
        "clocks": clocks,
    }
    s.close()
    return out


def _time_runs(s, arr, warm=4, reps=3):
    import torch
    stream = torch.cuda.ExternalStream(s.stream)
    with torch.cuda.stream(stream):
        for _ in range(warm):  # >= 4: JIT on the 2nd use, graphs after; QFT relabels alternate 2 plans
            s.run(arr)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            s.run(arr)
        b.record(stream)
        torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_sharded(args, rank, world, local_rank):
    """QFT on a state sharded over `world` GPUs (qc_state_create_dist, NCCL
    send/recv exchanges); weak scaling: 2^local_qubits amplitudes per GPU."""
    import torch
    import paper_2303_00123_b200 as qc
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p = world.bit_length() - 1
    n = args.local_qubits + p
    prec = "c128"
    ops = build_ops(args.config, n)
    arr = qc.encode_ops(ops)
    if world > 1:
        uid = [qc.qc.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(uid, src=0)
        s = qc.State.dist(n, prec, rank, world, uid[0])
    else:
        s = qc.State(n, prec, device=local_rank)
    stream = torch.cuda.ExternalStream(s.stream, device=dev)
    s.init_random(12345)
    ab = 16
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            s.run(arr)
        torch.cuda.synchronize()
        info = s.info()
        if world > 1:
            torch.distributed.barrier()
        clk = ClockSampler(local_rank)
        clk.start()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            s.run(arr)
        b.record(stream)
        torch.cuda.synchronize()
        clocks = clk.stop()
        t = a.elapsed_time(b)
        ex = None
        if world > 1:  # NVLink: one exchange of the top rank bit with the top local bit, timed alone
            torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 4
            e0.record(stream)
            for _ in range(reps):
                s.exchange(n - 1, n - p - 1)
            e1.record(stream)
            torch.cuda.synchronize()
            te = e0.elapsed_time(e1) / reps
            bytes_dir = (ab << (n - p)) // 2
            ex = {"ms": te, "bytes_per_direction": bytes_dir, "GBps_per_direction": bytes_dir / (te / 1e3) / 1e9}
    tt = torch.tensor([t], device=dev)
    if world > 1:
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        if ex is not None:
            te_t = torch.tensor([ex["ms"]], device=dev)
            torch.distributed.all_reduce(te_t, op=torch.distributed.ReduceOp.MAX)
            ex["ms"] = float(te_t.item())
            ex["GBps_per_direction"] = ex["bytes_per_direction"] / (ex["ms"] / 1e3) / 1e9
    t = float(tt.item())
    ms = t / args.steps
    peak, kind = load_peaks()
    sb_loc = ab << (n - p)
    out = {
        "metric": METRIC, "value": 1e3 / ms, "unit": "circuit/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config][4], "circuit": "qft", "qubits": n,
                   "local_qubits": n - p, "precision": prec, "parallelism": f"sharded x{world} (NCCL)",
                   "exchanges_per_step": info.get("last_exchanges", 0),
                   "fused_passes_per_step": info["last_passes"], "jit_specialised": info["last_jit"],
                   "l2": f"state {sb_loc >> 20} MiB per GPU >> 126 MB L2"},
        "gpu_launches": int(info["last_launches"] * args.steps),
        "roofline": {"bound": "hbm", "kernel": "qc_pass (fused tile pass, per shard)",
                     "achieved": 2 * sb_loc * info["last_passes"] / (ms / 1e3) / 1e9, "peak": peak,
                     "unit": "GB/s", "traffic": None,
                     "note": "lower bound: step time includes exchanges"},
        "nvlink_exchange": ex, "clocks": clocks,
    }
    out["roofline"]["frac"] = out["roofline"]["achieved"] / peak
    if ex is not None:
        out["nvlink_exchange"]["frac_of_900"] = ex["GBps_per_direction"] / 900.0
    s.close()
    return out


def sweep(args, local_rank):
    """Single-GPU measurements beside the main line (BASELINE metric: circuit
    time vs qubits; per-gate HBM GB/s vs peak; fused-pass GB/s)."""
    import torch
    import paper_2303_00123_b200 as qc
    import qcgen
    res = {"circuit_ms_vs_qubits": {}, "fused_pass": {}, "per_gate_n30": {}}
    peak, _ = load_peaks()
    plan = [("qft", "c128", (16, 20, 24, 28, 30)), ("qft", "c64", (20, 26, 30)),
            ("tfxy", "c128", (16, 20, 24, 28, 30)), ("tfxy", "c64", (20, 28))]
    fma = {"c128": derived_fma_peak("c128", local_rank)[0], "c64": derived_fma_peak("c64", local_rank)[0]}
    res["fma_peak_TFLOPs"] = {"fp64_derived": fma["c128"], "fp32_derived": fma["c64"],
                              "fp64_measured": qc.qc.fma_peak(True), "fp32_measured": qc.qc.fma_peak(False)}
    for fam, prec, ns in plan:
        key = f"{fam}_{prec}" + ("_S10" if fam == "tfxy" else "")
        res["circuit_ms_vs_qubits"][key] = {}
        for n in ns:
            ops = qcgen.qft(n) if fam == "qft" else qcgen.tfxy(n, 10)
            s = qc.State(n, prec, device=local_rank)
            s.init_random(1)
            t = _time_runs(s, qc.encode_ops(ops))
            inf = s.info()
            sb = (16 if prec == "c128" else 8) << n
            entry = {"ms": round(t, 4), "gates": len(ops), "passes": inf["last_passes"],
                     "jit": inf["last_jit"]}
            alg = inf["last_flops_per_amp"] * float(1 << n) / (t / 1e3) / 1e12
            entry["fused_alg_TFLOPs"] = round(alg, 2)
            entry["fused_alg_flops_frac_of_fma_peak"] = round(alg / fma[prec], 4)
            if n >= 28:
                gbps = 2 * sb * inf["last_passes"] / (t / 1e3) / 1e9
                entry["fused_pass_GBps"] = round(gbps, 1)
                entry["fused_pass_frac_of_measured_hbm"] = round(gbps / peak, 4)
                res["fused_pass"][f"{fam}{n}_{prec}"] = entry["fused_pass_GBps"]
            res["circuit_ms_vs_qubits"][key][str(n)] = entry
            s.close()
            torch.cuda.empty_cache()
    # north-star capacity: configs C4 (TFXY n=33, 10 steps) and QFT n=33, complex128, 137 GB
    res["north_star_n33_c128"] = {}
    free, _ = torch.cuda.mem_get_info()
    if free > (16 << 33) * 1.05:
        for fam in ("tfxy", "qft"):
            ops = qcgen.qft(33) if fam == "qft" else qcgen.tfxy(33, 10)
            s = qc.State(33, "c128", device=local_rank)
            s.init_random(1)
            t = _time_runs(s, qc.encode_ops(ops), warm=4 if fam == "qft" else 2, reps=2)
            inf = s.info()
            gbps = 2 * (16 << 33) * inf["last_passes"] / (t / 1e3) / 1e9
            alg = inf["last_flops_per_amp"] * float(1 << 33) / (t / 1e3) / 1e12
            res["north_star_n33_c128"][f"{fam}33" + ("_S10" if fam == "tfxy" else "")] = {
                "ms": round(t, 2), "gates": len(ops), "passes": inf["last_passes"], "jit": inf["last_jit"],
                "fused_alg_TFLOPs": round(alg, 2), "fused_alg_flops_frac_of_fp64_peak": round(alg / fma["c128"], 4),
                "fused_pass_GBps": round(gbps, 1), "fused_pass_frac_of_measured_hbm": round(gbps / peak, 4)}
            s.close()
            torch.cuda.empty_cache()
    for prec in ("c128", "c64"):
        n = 30
        sb = (16 if prec == "c128" else 8) << n
        s = qc.State(n, prec, device=local_rank)
        s.init_random(1)
        s.set_option("fusion", 0)
        s.set_option("relabel_swap", 0)
        pg = {}
        for name, qs, arg, nbytes in (("H", (0,), None, 2 * sb), ("H", (15,), None, 2 * sb),
                                      ("H", (29,), None, 2 * sb), ("RZ", (12,), 0.3, 2 * sb),
                                      ("P", (12,), 0.3, sb), ("X", (3,), None, 2 * sb),
                                      ("CNOT", (4, 20), None, sb), ("CP", (2, 27), 0.2, sb // 2),
                                      ("SWAP", (1, 28), None, sb), ("U2", (7, 22), "U", 2 * sb)):
            g = qcgen.Op(name, qs, theta=arg if isinstance(arg, float) else None,
                         matrix=qcgen.random_unitary(4, np.random.default_rng(0)) if arg == "U" else None)
            tg = _time_runs(s, qc.encode_ops([g]), warm=1, reps=5)
            gb = nbytes / (tg / 1e3) / 1e9
            pg[f"{name}{list(qs)}"] = {"ms": round(tg, 4), "GBps": round(gb, 1),
                                       "frac_of_measured_hbm": round(gb / peak, 4)}
        res["per_gate_n30"][prec] = pg
        s.close()
        torch.cuda.empty_cache()
    return res


def run_reference(args, rank, world):
    """--impl reference: the oracle (deliberately slow CPU program) as it stands."""
    if rank != 0:
        return None
    fam, n, steps_c, prec, desc = CONFIGS[args.config]
    if n is None:  # sharded config: the whole state, n = local + log2(N)
        n = args.local_qubits + (world.bit_length() - 1)
    rate, cores, sample = cpu_oracle_rate(args.config, budget_s=max(5.0, 4.0 * args.steps), n_override=n)
    return {"impl": "reference", "metric": METRIC, "value": rate, "unit": "circuit/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / rate, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "circuit": fam, "qubits": n, "precision": prec},
            "cpu_baseline": {"value": rate, "unit": "circuit/s", "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": rate, "unit": "circuit/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="tfxy20", choices=sorted(CONFIGS))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--local-qubits", type=int, default=30, help="qft_shard: qubits per GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 5)  # JIT on 2nd use + graph capture; QFT relabels alternate plans
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch
    if world > 1:
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.config == "qft_shard":
        out = run_sharded(args, rank, world, local_rank)
        if rank == 0:
            print(json.dumps(out), flush=True)
        if world > 1:
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()
        return
    out = run_ours(args, rank, world, local_rank)
    if rank == 0 and world == 1:
        if not args.no_sweep:
            out["sweep"] = sweep(args, local_rank)
        if not args.no_cpu:
            rate, cores, sample = cpu_oracle_rate(args.config)
            out["cpu_baseline"] = {"value": rate, "unit": "circuit/s", "cores": cores,
                                   "kind": "oracle", "sample": sample}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
