"""bench.py -- QFT / TFXY state-vector circuit time on B200 through libqc (the C ABI).

Default workload at N = 1: BASELINE.json configs[3] (C4), the largest
single-GPU configuration -- TFXY 1D Trotter circuit (DESIGN R8),
33 qubits, 10 Trotter steps, complex double, a 137 GB state resident in HBM,
seeded random initial state.  A "step" is one qc_run_circuit of the whole
circuit on the resident state (all SURVEY 8(a) rows: fused tile passes with
SWAP relabels and row-bit remaps).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config tfxy33|tfxy20|qft10|qft30|qft30c64|tfxy_shard|qft_shard]
                  [--no-sweep] [--no-cpu]

N > 1: one process per GPU (torchrun; `--gpus N` without WORLD_SIZE re-execs
itself under torch.distributed.run).  The default N > 1 workload is the
sharded weak-scaling grid of SURVEY 8(d): TFXY S=10 at n = 33 + log2 N
(128 GiB per GPU), sharded by the top log2 N qubits with NCCL qubit-swap
exchanges (`--config qft_shard`: BASELINE configs[4], QFT n = 33 + log2 N,
= C5 at N = 8).

value = whole-job throughput in amplitude-gate updates per second: gates of
the circuit x 2^n amplitudes / circuit time (units all ranks processed / max
time over ranks), reported in 1e9 ("Gamp-gate/s"); circuits/s and ms per
circuit are in the line too.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QFT & TFXY circuit time vs qubits at 1-8 B200; per-gate HBM GB/s vs peak"
UNIT = "Gamp-gate/s"

CONFIGS = {
    # name: (family, n (None: 33 + log2 N), trotter steps, precision, description)
    "qft10": ("qft", 10, 0, "c128", "C1: QFT on 10 qubits, complex double, random initial state"),
    "tfxy20": ("tfxy", 20, 10, "c128", "C2: TFXY 1D Trotter circuit, 20 qubits, 10 time steps, complex double, "
                                       "1 B200 (16 MiB state, L2-resident)"),
    "qft30": ("qft", 30, 0, "c128", "C3: QFT on 30 qubits, complex double, 1 B200"),
    "qft30c64": ("qft", 30, 0, "c64", "C3: QFT on 30 qubits, complex single, 1 B200"),
    "tfxy33": ("tfxy", 33, 10, "c128", "C4: TFXY Trotter circuit, 33 qubits, 10 time steps, complex double "
                                       "(137 GB state), 1 B200"),
    # sharded (one process per GPU, qubit-swap exchanges): n = local + log2(N)
    "tfxy_shard": ("tfxy", None, 10, "c128", "TFXY Trotter circuit S=10, complex double, n = 33 + log2(N) "
                                             "sharded over N B200 by the top log2(N) qubits (weak scaling)"),
    "qft_shard": ("qft", None, 0, "c128", "C5: QFT complex double, n = 33 + log2(N) sharded over N B200 by the "
                                          "top log2(N) qubits (weak scaling; n=36 at N=8)"),
}


def default_config(world):
    return "tfxy33" if world == 1 else "tfxy_shard"


def build_ops(cfg, n):
    import qcgen
    fam, _, steps, _, _ = CONFIGS[cfg]
    return qcgen.qft(n) if fam == "qft" else qcgen.tfxy(n, steps)


def gamp(ops, n, seconds):
    """amplitude-gate updates per second, in 1e9."""
    return len(ops) * float(1 << n) / seconds / 1e9


# Algorithmic flops per amplitude of each unfused gate: dense
# 1q 14, dense 2q 30, a diagonal factor 6 per touched amplitude, 0 for
# permutations (X, CNOT, SWAP, CCX; Y and CZ are sign / i-multiples).
FLOPS_PER_AMP = {"H": 14, "RX": 14, "RY": 14, "U1": 14, "RZ": 6, "P": 3, "CP": 1.5, "Z": 0, "CZ": 0,
                 "Y": 0, "X": 0, "CNOT": 0, "SWAP": 0, "CCX": 0, "CU1": 7, "U2": 30}


def circuit_flops(ops, n):
    return float(sum(FLOPS_PER_AMP[o.name] for o in ops)) * float(1 << n)


def load_traffic(cfg):
    """dram read+write bytes per launch of qc_pass from the committed ncu
    capture of this workload (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f).get(cfg)
        return (d["bytes_per_launch"], d["source"]) if d else (None, None)
    except Exception:
        return None, None


def derived_fma_peak(prec, device=0):
    """ALU roofline denominator derived from unit counts and clocks (DESIGN
    section 6): SMs x FMA lanes per SM per clock (FP64 64, FP32 128 on
    sm_100) x 2 flops x the max SM clock (MEASURED_PEAKS.json sm_max_mhz)."""
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


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


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
class OracleSampler:
    """The oracle (as it stands) on a BOUNDED sample of the workload: the
    first gates of the circuit whose qubits lie below n_s, applied to the
    seeded random state of n_s qubits.  Per-gate time is extrapolated to the
    workload's n by x2 per qubit (the paper's scaling law) and to the
    whole circuit by its gate count -- labelled "extrapolated" when n_s < n."""

    def __init__(self, cfg, n, n_sample=26, step_s=2.0):
        os.environ.setdefault("OMP_PROC_BIND", "close")  # before libgomp initialises
        import oracle
        import qcgen
        self.oracle = oracle
        self.cfg, self.n = cfg, n
        self.ops = build_ops(cfg, n)
        self.n_s = min(n, n_sample)
        self.sample_ops = [o for o in self.ops if max(o.qubits) < self.n_s]
        prec = CONFIGS[cfg][3]
        self.psi = qcgen.random_state(self.n_s, precision=prec)
        self.pos = 0
        self.per_gate = []
        # calibrate: gates per step so one step takes ~step_s
        self._apply(1)  # first call loads the library
        t = self._apply(1)
        self.g_step = max(1, min(len(self.sample_ops), int(step_s / max(t, 1e-6))))

    def _apply(self, g):
        ops = [self.sample_ops[(self.pos + i) % len(self.sample_ops)] for i in range(g)]
        self.pos = (self.pos + g) % len(self.sample_ops)
        t0 = time.perf_counter()
        self.psi = self.oracle.run(self.n_s, self.psi, ops)
        dt = time.perf_counter() - t0
        self.per_gate.append(dt / g)
        return dt / g

    def step(self):
        t0 = time.perf_counter()
        self._apply(self.g_step)
        return time.perf_counter() - t0

    def circuit_seconds(self, last=None):
        pg = self.per_gate[-last:] if last else self.per_gate
        return statistics.median(pg) * (2.0 ** (self.n - self.n_s)) * len(self.ops)

    def describe(self, steps, secs):
        ext = self.n_s < self.n
        return (f"{steps} steps x {self.g_step} gates of the {self.cfg} circuit (its gates on qubits < {self.n_s}) "
                f"at n={self.n_s}, {secs:.1f} s of oracle time; median per-gate time"
                + (f" x2 per qubit to n={self.n} (P:112 law; extrapolated)" if ext else "")
                + f" x {len(self.ops)} gates; {self.oracle.max_threads()} OpenMP threads, "
                f"OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')}, host CPU: {cpu_model()}")


def cpu_baseline(cfg, n, budget_s=15.0):
    smp = OracleSampler(cfg, n)
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < budget_s:
        smp.step()
        k += 1
    secs = time.perf_counter() - t0
    csec = smp.circuit_seconds()
    ops = smp.ops
    return {"value": gamp(ops, n, csec), "unit": UNIT, "cores": smp.oracle.max_threads(), "kind": "oracle",
            "extrapolated": smp.n_s < n, "circuit_s": csec, "sample": smp.describe(k, secs)}


# ----------------------------------------------------------------- our arm
def _max_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def make_state(args, n, prec, rank, world, local_rank):
    import torch
    import paper_2303_00123_b200 as qc
    if world == 1:
        return qc.State(n, prec, device=local_rank)
    uid = [qc.qc.nccl_unique_id() if rank == 0 else None]
    torch.distributed.broadcast_object_list(uid, src=0)
    return qc.State.dist(n, prec, rank, world, uid[0])


def choose_exchange_mode(rank, world):
    """Sharded runs: group plans (QC_OPT_EXCHANGE 3: one plan over all n bits,
    tiles spanning shards through TMA on IPC-mapped peer buffers) if a probe
    job -- its own processes, launched before any shard is allocated, so a
    fault cannot take this run down -- reproduces the NCCL-exchange results on
    this node; else qubit-swap exchanges over NCCL (mode 0).
    QC_BENCH_EXCHANGE=<mode> skips the probe."""
    import torch
    forced = os.environ.get("QC_BENCH_EXCHANGE")
    if forced is not None:
        return int(forced), {"mode": int(forced), "probe": "skipped (QC_BENCH_EXCHANGE)"}
    res = [None]
    if rank == 0:
        env = {k: v for k, v in os.environ.items()
               if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "GROUP_RANK", "ROLE_RANK",
                            "MASTER_ADDR", "MASTER_PORT") and not k.startswith("TORCHELASTIC")}
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
               os.path.join(ROOT, "scripts", "probe_sharded.py")]
        t0 = time.time()
        try:
            r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=420)
            ok = r.returncode == 0 and "PROBE OK" in r.stdout
            why = "PROBE OK" if ok else f"rc={r.returncode}: {(r.stdout + r.stderr).strip().splitlines()[-1:]}"
        except Exception as e:  # timeout / launch failure: stay on the NCCL exchanges
            ok, why = False, repr(e)[:200]
        res = [{"ok": ok, "why": why, "seconds": round(time.time() - t0, 1)}]
    torch.distributed.broadcast_object_list(res, src=0)
    r = res[0]
    mode = 3 if r["ok"] else 0
    return mode, {"mode": mode, "probe": r}


def run_ours(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    fam, n0, steps_c, prec, desc = CONFIGS[args.config]
    p = world.bit_length() - 1
    n = n0 if n0 is not None else args.local_qubits + p
    if n0 is not None and world > 1:
        raise SystemExit(f"--config {args.config} is a single-GPU workload; use tfxy_shard / qft_shard for N > 1")
    ops = build_ops(args.config, n)
    import paper_2303_00123_b200 as qc
    arr = qc.encode_ops(ops)
    xmode, xinfo = choose_exchange_mode(rank, world) if world > 1 else (0, None)
    s = make_state(args, n, prec, rank, world, local_rank)
    if world > 1:
        s.set_option("exchange", xmode)
    stream = torch.cuda.ExternalStream(s.stream, device=dev)
    s.init_random(12345)
    ab = 16 if prec == "c128" else 8
    n_loc = n - p
    shard_bytes = ab << n_loc
    small = shard_bytes < (1 << 30)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if small else None

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            s.run(arr)
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
            if flush is not None:
                flush.zero_()  # L2 flush between timed iterations (outside the events)
            ev[i][0].record(stream)
            s.run(arr)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        clocks = clk.stop()
    per = [a.elapsed_time(b) for a, b in ev]  # ms
    t_total = _max_over_ranks(sum(per), world, dev)
    ms_per_step = t_total / args.steps
    value = gamp(ops, n, ms_per_step / 1e3)

    # NVLink: one exchange of the top rank bit with the top local bit, timed
    # alone, for both backends (QC_OPT_EXCHANGE 0: NCCL send/recv + ping-pong
    # staging copies; 1: P2P swap kernel over CUDA IPC mappings)
    ex = None
    if world > 1:
        ex = {}
        bytes_dir = shard_bytes // 2
        for xm_t, name in ((0, "nccl_sendrecv_pingpong"), (1, "p2p_swap_kernel")):
            s.set_option("exchange", xm_t)
            torch.distributed.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                s.exchange(n - 1, n_loc - 1)  # warm-up (P2P: IPC mapping)
                e0.record(stream)
                for _ in range(4):
                    s.exchange(n - 1, n_loc - 1)
                e1.record(stream)
            torch.cuda.synchronize()
            te = _max_over_ranks(e0.elapsed_time(e1) / 4, world, dev)
            ex[name] = {"ms": te, "bytes_per_direction": bytes_dir,
                        "GBps_per_direction": bytes_dir / (te / 1e3) / 1e9,
                        "frac_of_900": bytes_dir / (te / 1e3) / 1e9 / 900.0}
        s.set_option("exchange", 0)
    if world > 1:
        # the same circuit in the other sharded modes (exchanges over NCCL;
        # pair passes and group plans only if the probe cleared peer-memory
        # TMA), timed like the headline over a few steps
        ex["headline_exchange_mode"] = xinfo
        alts = [m for m in (0, 2, 3) if m != xmode and (m == 0 or xmode == 3)]
        for m in alts:
            s.set_option("exchange", m)
            with torch.cuda.stream(stream):
                s.run(arr)
                s.run(arr)
                torch.cuda.synchronize()
                torch.distributed.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                k_alt = max(1, min(args.steps, 3))
                e0.record(stream)
                for _ in range(k_alt):
                    s.run(arr)
                e1.record(stream)
                torch.cuda.synchronize()
            tp = _max_over_ranks(e0.elapsed_time(e1) / k_alt, world, dev)
            pi = s.info()
            ex[f"circuit_exchange_mode_{m}"] = {
                "ms_per_step": tp, "value": gamp(ops, n, tp / 1e3), "unit": UNIT, "passes": pi["last_passes"],
                "exchanges": pi["last_exchanges"], "pair_segments_or_spanning_passes": pi["last_pair_segments"]}
        s.set_option("exchange", xmode)
        s.run(arr)  # back to the headline mode's plan (warm) before e2e

    # ---- e2e: pinned host state in, circuit, full state out, every step
    # (states above 8 GiB share one pinned buffer for input and output: the
    # read-back of step i is the upload of step i+1 -- same bytes moved; a
    # shard larger than this rank's share of host RAM moves in chunks through
    # a smaller pinned buffer, every byte of the shard still crossing the link
    # both ways each step)
    try:
        import psutil
        host_cap = int(psutil.virtual_memory().available * 0.6) // int(os.environ.get("LOCAL_WORLD_SIZE", world))
    except Exception:
        host_cap = shard_bytes
    hb = min(shard_bytes, max(host_cap, 1 << 30))
    hb -= hb % ab
    h_in = torch.empty(hb, dtype=torch.uint8, pin_memory=True)
    h_out = h_in if hb < shard_bytes or hb > (8 << 30) else torch.empty(hb, dtype=torch.uint8, pin_memory=True)
    first = rank << n_loc
    chunk = hb // ab
    spans = [(first + o, min(chunk, (1 << n_loc) - o)) for o in range(0, 1 << n_loc, chunk)]
    if world > 1:
        s.canonicalize()
    s.read_ptr(h_in.data_ptr(), spans[0][1], spans[0][0])  # a valid state (first chunk) to start from
    e2e_steps = max(1, min(args.steps, 5 if small else 3))
    torch.cuda.synchronize()
    e_ev = []
    with torch.cuda.stream(stream):
        for i in range(e2e_steps + 1):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for f0, cnt in spans:
                s.write_ptr(h_in.data_ptr(), cnt, f0)
            s.run(arr)
            if world > 1:
                s.canonicalize()
            for f0, cnt in spans:
                s.read_ptr(h_out.data_ptr(), cnt, f0)
            b.record(stream)
            if i > 0:
                e_ev.append((a, b))
        torch.cuda.synchronize()
    e_seq_ms = _max_over_ranks(sum(a.elapsed_time(b) for a, b in e_ev) / len(e_ev), world, dev)
    # pipelined: step i's result read-back and step i+1's input upload in one
    # qc_state_readwrite (D2H of chunk c+1 overlaps H2D of chunk c; the link
    # is full duplex).  Every step still uploads its input and reads back its
    # result: write(in_0); for each step: run, then readwrite(out_i, in_i+1)
    # (the last step: read(out)).  One untimed round first.
    def e2e_pipelined(steps):
        for f0, cnt in spans:
            s.write_ptr(h_in.data_ptr(), cnt, f0)
        for i in range(steps):
            s.run(arr)
            if world > 1:
                s.canonicalize()
            for f0, cnt in spans:
                if i == steps - 1:
                    s.read_ptr(h_out.data_ptr(), cnt, f0)
                else:
                    s.readwrite_ptr(h_out.data_ptr(), h_in.data_ptr(), cnt, f0)
    with torch.cuda.stream(stream):
        e2e_pipelined(1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_pipelined(e2e_steps)
        b.record(stream)
        torch.cuda.synchronize()
    e_ms = _max_over_ranks(a.elapsed_time(b) / e2e_steps, world, dev)
    del h_in, h_out

    peak, peak_kind = load_peaks()
    # dominant kernel = the fused pass (every launch of the step is one).
    # HBM view: algorithmic bytes per launch = read + write of the shard (2*Ns).
    # ALU view: algorithmic flops of the fused plan's ops per launch, against
    # the FP64 (c128) / FP32 (c64) FMA peak derived from unit counts and clocks.
    avg_launch_ms = ms_per_step / max(launches_per_step, 1)
    achieved = 2 * shard_bytes / (avg_launch_ms / 1e3) / 1e9
    fma_peak, fma_src = derived_fma_peak(prec, local_rank)
    # last_flops_per_amp sums every pass of the plan: per launch = that / passes
    flops = info["last_flops_per_amp"] * float(1 << n_loc) / max(passes, 1)
    alu_achieved = flops / (avg_launch_ms / 1e3) / 1e12
    traffic, traffic_src = load_traffic(args.config if world == 1 else f"{fam}{n_loc}")
    hbm_view = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)", "bytes_per_launch": 2 * shard_bytes}
    alu_view = {"bound": "alu", "achieved": alu_achieved, "peak": fma_peak, "unit": "TFLOP/s",
                "frac": alu_achieved / fma_peak, "peak_source": fma_src, "flops_per_launch": flops,
                "flops_note": "algorithmic flops of the fused plan's ops (qc_info.last_flops_per_amp: complex "
                              "arithmetic, general cmul 6 / cmac 8 flops, unit coefficients free, x fraction of "
                              "amplitudes touched, summed over the plan's passes) x 2^n_local / passes "
                              "(the mean launch)",
                "unfused_gate_flops_per_step": circuit_flops(ops, n)}
    # binding roof: the larger fraction (ALU for block-fused TFXY, HBM for QFT)
    main_view = alu_view if alu_view["frac"] > hbm_view["frac"] else hbm_view
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if prec == "c128" else "f32", "data": "synthetic",
        "circuits_per_s": 1e3 / ms_per_step,
        "config": {"workload": desc, "circuit": fam, "qubits": n, "local_qubits": n_loc,
                   "trotter_steps": steps_c or None, "gates": len(ops), "precision": prec,
                   "state_bytes": ab << n, "shard_bytes": shard_bytes,
                   "initial_state": "splitmix64 seed 12345 (DESIGN input recipe)",
                   "l2": ("flushed (512 MiB write) between timed iterations" if small else
                          f"inputs larger than L2: {shard_bytes / 1e9:.1f} GB per GPU >> 126 MB"),
                   "parallelism": "single GPU" if world == 1 else
                   f"sharded x{world} by the top {p} qubits, exchange mode {xmode} "
                   f"({'group plan: tiles spanning shards over NVLink' if xmode == 3 else 'NCCL qubit-swap exchanges'})",
                   "fused_passes_per_step": passes, "exchanges_per_step": info.get("last_exchanges", 0),
                   "tile_bits": info["tile_bits"], "cuda_graph": info["last_graph"],
                   "jit_specialised": info["last_jit"], "ops_after_block_fusion": info["last_blocks"],
                   "value_definition": "gates x 2^n / circuit time (max over ranks), 1e9 units"},
        "gpu_launches": int(launches_per_step * args.steps),
        "roofline": {**main_view, "kernel": "qc_pass (NVRTC-specialised fused tile pass)",
                     "traffic": traffic, "traffic_source": traffic_src,
                     "avg_launch_ms": avg_launch_ms, "hbm_view": hbm_view, "alu_view": alu_view,
                     "note": "avg launch = timed step time / fused launches per step (every launch of "
                             "the step is a fused pass, timed by CUDA events on the state's stream)"
                             + ("; the step also holds the exchanges" if world > 1 else "")},
        "e2e": {"value": gamp(ops, n, e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": shard_bytes,
                "d2h_bytes_per_step": shard_bytes, "ms_per_step": e_ms, "pinned_host_buffer_bytes": hb,
                "steps": e2e_steps,
                "path": "per rank, through the C ABI with pinned host buffers: qc_state_write (step 0's input), "
                        "then per step qc_run_circuit + qc_state_readwrite (this step's result read back while "
                        "the next step's input is uploaded, D2H / H2D chunks overlapped; the last step "
                        "qc_state_read); every step moves its input in and its result out",
                "sequential_ms_per_step": e_seq_ms,
                "sequential_path": "qc_state_write + qc_run_circuit + qc_state_read per step (no overlap)"},
        "clocks": clocks,
    }
    if ex is not None:
        out["nvlink_exchange"] = ex
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
                     "jit": inf["last_jit"], "Gamp_gate_per_s": round(gamp(ops, n, t / 1e3), 1)}
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
    # north-star capacity: QFT n=33 complex128, 137 GB (TFXY-33 is the headline)
    res["north_star_n33_c128"] = {}
    free, _ = torch.cuda.mem_get_info()
    if free > (16 << 33) * 1.05:
        ops = qcgen.qft(33)
        s = qc.State(33, "c128", device=local_rank)
        s.init_random(1)
        t = _time_runs(s, qc.encode_ops(ops), warm=4, reps=2)
        inf = s.info()
        gbps = 2 * (16 << 33) * inf["last_passes"] / (t / 1e3) / 1e9
        res["north_star_n33_c128"]["qft33"] = {
            "ms": round(t, 2), "gates": len(ops), "passes": inf["last_passes"], "jit": inf["last_jit"],
            "fused_pass_GBps": round(gbps, 1), "fused_pass_frac_of_measured_hbm": round(gbps / peak, 4)}
        s.close()
        torch.cuda.empty_cache()
    # qubit-swap exchange on one GPU (loopback backend: both shards of a
    # world-2 state in one buffer, the swap kernel the P2P backend runs over
    # NVLink, here HBM-local): bytes per direction / time
    n = 32
    s = qc.State.loopback(n, "c128", 2)
    s.init_random(1)
    st = torch.cuda.ExternalStream(s.stream)
    with torch.cuda.stream(st):
        s.exchange(n - 1, n - 2)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(4):
            s.exchange(n - 1, n - 2)
        b.record(st)
        torch.cuda.synchronize()
    te = a.elapsed_time(b) / 4
    bytes_dir = (16 << (n - 1)) // 2  # per rank per direction
    res["exchange_loopback_n32_w2_c128"] = {
        "ms": round(te, 3), "bytes_per_direction_per_rank": bytes_dir,
        "swap_kernel_GBps_hbm": round(2 * 2 * bytes_dir / (te / 1e3) / 1e9, 1),
        "note": "both ranks' halves swapped in place by one kernel: 2 x (read + write) of the exchanged bytes"}
    s.close()
    torch.cuda.empty_cache()
    # generic dense k-target gates: fused passes of random
    # dense 2^k x 2^k blocks (FP64 work 8 * 2^k flop/amp per gate) -- the
    # "is a dense block a real contraction" evaluation -- and the per-gate
    # DENSEK kernel's HBM rate
    res["dense_k_blocks_n28_c128"] = {}
    n = 28
    rng = np.random.default_rng(5)
    for k in (2, 3, 4):
        ops = []
        for _ in range(40):
            qs = tuple(int(q) for q in rng.choice(n, size=k, replace=False))
            ops.append(qcgen.Op("MCU", qs, matrix=qcgen.random_unitary(1 << k, rng), nctrl=0))
        s = qc.State(n, "c128", device=local_rank)
        s.init_random(1)
        t = _time_runs(s, qc.encode_ops(ops), warm=4, reps=3)
        inf = s.info()
        alg = inf["last_flops_per_amp"] * float(1 << n) / (t / 1e3) / 1e12
        s.set_option("fusion", 0)
        tg = _time_runs(s, qc.encode_ops(ops[:1]), warm=1, reps=5)
        res["dense_k_blocks_n28_c128"][f"k{k}"] = {
            "gates": len(ops), "ms": round(t, 3), "passes": inf["last_passes"],
            "fused_alg_TFLOPs": round(alg, 2), "fused_alg_flops_frac_of_fp64_peak": round(alg / fma["c128"], 4),
            "per_gate_ms": round(tg, 4), "per_gate_GBps": round(2 * (16 << n) / (tg / 1e3) / 1e9, 1)}
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


def cpu_omp_curve(budget_s=40.0):
    """The paper's CPU program (libqc_omp.so: Algs. 1-3, one OpenMP parallel
    loop per gate) -- circuit time vs qubits on this host's cores, the
    CPU side of the paper's CPU-vs-GPU experiments.  Bounded: sizes
    are skipped once the budget is spent."""
    os.environ.setdefault("OMP_PROC_BIND", "close")
    import qcgen
    from paper_2303_00123_b200 import cpu_omp
    res = {"threads": cpu_omp.qc_omp_max_threads(), "cpu": cpu_model(),
           "omp_proc_bind": os.environ.get("OMP_PROC_BIND"), "ms": {}}
    cpu_omp.qc_omp_run(12, "c128", qcgen.random_state(12), qcgen.qft(12))  # thread-pool start-up
    t_start = time.perf_counter()
    for fam, prec, ns in (("qft", "c128", (16, 20, 22, 24)), ("qft", "c64", (20, 24)),
                          ("tfxy", "c128", (16, 20, 22))):
        key = f"{fam}_{prec}" + ("_S10" if fam == "tfxy" else "")
        res["ms"][key] = {}
        for n in ns:
            if time.perf_counter() - t_start > budget_s:
                break
            ops = qcgen.qft(n) if fam == "qft" else qcgen.tfxy(n, 10)
            x = qcgen.random_state(n, precision=prec)
            t0 = time.perf_counter()
            cpu_omp.qc_omp_run(n, prec, x, ops)
            res["ms"][key][str(n)] = round((time.perf_counter() - t0) * 1e3, 2)
    return res


def run_reference(args, rank, world):
    """--impl reference: the oracle (deliberately slow CPU program) as it
    stands, on this arm's workload, metric and unit: W untimed + K timed steps,
    each step a bounded sample of the workload (OracleSampler)."""
    if rank != 0:
        return None
    fam, n0, steps_c, prec, desc = CONFIGS[args.config]
    n = n0 if n0 is not None else args.local_qubits + (world.bit_length() - 1)
    smp = OracleSampler(args.config, n, step_s=2.0)
    for _ in range(args.warmup):
        smp.step()
    smp.per_gate.clear()
    times = [smp.step() for _ in range(args.steps)]
    secs = sum(times)
    csec = smp.circuit_seconds()
    value = gamp(smp.ops, n, csec)
    sample = smp.describe(args.steps, secs)
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "circuits_per_s": 1.0 / csec,
            "config": {"workload": desc, "circuit": fam, "qubits": n, "precision": prec,
                       "step": "one bounded oracle sample (ms_per_step = its wall time); value = the "
                               "workload's amplitude-gate rate from the median per-gate time"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": smp.oracle.max_threads(), "kind": "oracle",
                             "extrapolated": smp.n_s < n, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--local-qubits", type=int, default=33, help="sharded configs: qubits per GPU")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-exec under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__),
               *sys.argv[1:]]
        os.execv(sys.executable, cmd)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.config is None:
        args.config = default_config(world)
    if args.impl == "ours":
        args.warmup = max(args.warmup, 4)  # JIT on the 2nd use + graph capture; QFT relabels alternate 2 plans

    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return

    import torch
    if world > 1:
        # NCCL's init log (ranks, NVLink / NVLS topology) on stderr, so the
        # communicator size can be checked without touching the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_ours(args, rank, world, local_rank)
    if rank == 0 and world == 1:
        if not args.no_sweep:
            out["sweep"] = sweep(args, local_rank)
        if not args.no_cpu:
            n = out["config"]["qubits"]
            out["cpu_baseline"] = cpu_baseline(args.config, n)
            out["cpu_omp_paper_program"] = cpu_omp_curve()
            # the paper's CPU-vs-GPU comparison (E1/E2) on this box:
            # the paper's CPU program vs the fused GPU path, same circuits
            sw = out.get("sweep", {}).get("circuit_ms_vs_qubits", {})
            cmp = {}
            for key, ms in out["cpu_omp_paper_program"]["ms"].items():
                for nq, cpu_ms in ms.items():
                    g = sw.get(key, {}).get(nq)
                    if g:
                        cmp[f"{key}_n{nq}"] = {"cpu_ms": cpu_ms, "gpu_ms": g["ms"], "speedup": round(cpu_ms / g["ms"], 1)}
            out["cpu_vs_gpu_paper_E1E2"] = cmp
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
