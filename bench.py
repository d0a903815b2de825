#!/usr/bin/env python
"""bench.py -- K-TanH hot path on B200: Gelem/s and achieved HBM GB/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ktanh|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

Metric (BASELINE.json): "K-TanH Gelem/s and achieved HBM GB/s vs ~8 TB/s
peak at 1/2/4/8 B200".  The headline workload is the one the metric is
quoted on at 1/2/4/8 GPUs, BASELINE.json configs[4]: K-GELU
over a [65536, 16384] BF16 tensor ~ N(0, 1) per GPU (2^30 elements), one
library call (= one kernel) per step.  Every rank processes its own
independent tensor (seed + rank, weak scaling, no collective on the data
path); `value` is the elements of all ranks / the max over ranks of the
timed region.  configs 2-4, K-Swish and the fused K-GELU+K-Swish pass are
`extra` lines (`--config` picks another headline).

Timing: W warm-up steps, then windows of exactly K steps, each bracketed by
a barrier and cuda synchronize, timed with CUDA events on the launching
stream; the K launches of a window are replayed from a CUDA graph (the
library calls are capturable).  Inputs smaller than L2 rotate through
buffer sets totalling > 4x L2 so every step reads cold HBM (config 5's
4 GiB per step is larger than L2 by itself).  nvidia-smi clocks are sampled
during the timed windows.  Reported: the median window.

`--impl reference` times the CPU oracle (oracle/, the scalar C
implementation of the paper's algorithm) on the host cores on a bounded
sample of the same workload; under torchrun only rank 0 runs it.  The only
other use of oracle/ is the main arm's cpu_baseline leg: the oracle timed on
a sample of the headline input, plus every rank's sampled check of its own
GPU outputs against the oracle (outside the timed region).

`--stub` (test hook, CPU only): the same multi-rank driver -- device
selection, barriers, per-rank timing, max-over-ranks aggregation, the
per-rank check and the JSON line -- around a trivial host copy instead of the
library, so tests/test_bench_contract.py can run the N > 1 path under
torchrun with gloo on a machine without a GPU.  Its numbers mean nothing.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import workloads as WL

FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback
NOMINAL_HBM_GBS = 8000.0    # BASELINE.json north_star "~8 TB/s"
L2_BYTES = 126 * 1024 * 1024


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def _kd():
    from paper_1909_07729_b200 import dist as kd
    return kd


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        return len(self.lines)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.t:
                self.t.join(timeout=2)

    def summary(self, lo=0, hi=None):
        rows = [l.split(", ") for l in self.lines[lo:hi] if l.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ steps --
class Step:
    """One pass of the hot path over one batch: a single library call."""

    def __init__(self, kt, cfg_key, op, device, rank, sets=None):
        self.cfg = WL.CONFIGS[cfg_key]
        self.op = op
        self.kt = kt
        n = self.cfg.numel
        self.n = n
        es = self.cfg.elem_bytes
        self.bwd = "_bwd_" in op
        self.cell = op == "lstm_cell"
        self.dual = op in ("kgelu_swish_bf16", "kgelu_swish_f32")
        # algorithmic bytes: read x (+ dy for a backward) + write y
        self.bytes_per_step = (3 if self.bwd else 2) * n * es
        if self.cell:   # gates 8 B + c 4 B in, c' 4 B + h 2 B out per cell (n/4 cells)
            self.bytes_per_step = 18 * (n // 4)
        if self.dual:   # x once in, both outputs out
            self.bytes_per_step = 3 * n * es
        if sets is None:
            sets = 1 if self.bytes_per_step >= 2 * L2_BYTES else \
                max(2, math.ceil(4 * L2_BYTES / self.bytes_per_step))
        self.sets = sets
        x0 = WL.make_input(self.cfg, device=device, rank=rank)
        self.xs = [x0] + [WL.make_input(self.cfg, device=device, rank=rank, seed=self.cfg.seed + 1000 * s)
                          for s in range(1, sets)]
        self.ys = [torch.empty_like(x0) for _ in range(sets)]
        self.y2s = [torch.empty_like(x0) for _ in range(sets)] if self.dual else None
        self.ds = [WL.make_input(self.cfg, device=device, rank=rank, seed=self.cfg.seed + 77 + 1000 * s)
                   for s in range(sets)] if self.bwd else None
        if self.cell:
            H = WL.LSTM_HIDDEN
            g = torch.Generator(device=device)
            g.manual_seed(self.cfg.seed + 99 + rank)
            self.cs = [torch.randn(n // (4 * H), H, generator=g, device=device) for _ in range(sets)]
            self.cns = [torch.empty_like(c) for c in self.cs]
            self.hns = [torch.empty(c.shape, dtype=torch.bfloat16, device=device) for c in self.cs]
        self.fn = self._bind()

    def _bind(self):
        kt, op = self.kt, self.op
        if op == "ktanh64_bf16":              # 64-interval kernel, Table 1 split in halves
            E32, r32, b32 = kt.paper_lut().tables()
            t64 = [(((t >> 4) << 3) | ((t & 15) >> 1)) for t in range(64)]
            h = kt.Lut64([E32[i] for i in t64], [r32[i] for i in t64], [b32[i] for i in t64])
            return lambda x, y: kt.ktanh64_bf16(x, h, out=y)
        if op.startswith("apx:"):             # Table 2 comparator "apx:<kind>:<p>:<q>"
            _, kind, p, q = op.split(":")
            apx = kt.Apx(kind, int(p), int(q))
            call = kt.kt_apx_tanh_bf16 if self.cfg.elem_bytes == 2 else kt.kt_apx_tanh_f32
            return lambda x, y: call(x, apx, out=y)
        if op == "ktanh_f32:p23":             # F32-native table re-optimised at p = 23 (NEXT-3)
            h = kt.Lut.optimized(23)
            return lambda x, y: kt.ktanh_f32(x, out=y, lut=h)
        if op.startswith("torch:"):           # library comparators (NEXT-4 context rows)
            name = op[6:]
            if name == "tanh":
                return lambda x, y: torch.tanh(x, out=y)
            approx = "tanh" if name == "gelu_tanh" else "none"
            return lambda x, y: torch.ops.aten.gelu.out(x, approximate=approx, out=y)
        if op == "lstm":
            return lambda x, y: kt.klstm_gates_bf16(x, WL.LSTM_HIDDEN, 2, out=y)
        return lambda x, y: getattr(kt, op)(x, out=y)

    def run(self, i):
        s = i % self.sets
        if self.cell:
            self.kt.klstm_cell_bf16(self.xs[s], self.cs[s], WL.LSTM_HIDDEN, c_next=self.cns[s],
                                    h_next=self.hns[s])
        elif self.bwd:
            getattr(self.kt, self.op)(self.xs[s], self.ds[s], out=self.ys[s])
        elif self.dual:
            getattr(self.kt, self.op)(self.xs[s], out_gelu=self.ys[s], out_swish=self.y2s[s])
        else:
            self.fn(self.xs[s], self.ys[s])


def barrier(world):
    if world > 1:
        _kd().barrier()


def max_over_ranks(v: float, world: int, device) -> float:
    """Timing plumbing only (paper_1909_07729_b200.dist, tested with gloo)."""
    if world == 1:
        return v
    return _kd().max_over_ranks(v, device)


def time_windows(step: Step, K: int, W: int, world: int, device, clocks: ClockSampler | None,
                 min_total_s: float = 1.0, max_windows: int = 4000):
    """W warm-up steps, then windows of exactly K graph-replayed steps; returns
    (per-window max-over-ranks ms, clock summary, launches per step)."""
    stream = torch.cuda.Stream(device)
    torch.cuda.synchronize(device)
    for i in range(W):                      # untimed warm-up (eager)
        step.run(i)
    torch.cuda.synchronize(device)
    c0 = step.kt.launch_count()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(K):
            step.run(W + i)
    launches_per_step = (step.kt.launch_count() - c0) / K
    g.replay()                               # graph warm-up
    torch.cuda.synchronize(device)
    # number of windows: enough for ~min_total_s of timed work (clock sampling)
    t0 = time.perf_counter()
    g.replay()
    torch.cuda.synchronize(device)
    est = time.perf_counter() - t0
    nwin = int(max(3, min(max_windows, math.ceil(min_total_s / max(est, 1e-6)))))
    nwin = int(max_over_ranks(nwin, world, device))
    mark0 = clocks.mark() if clocks else 0
    times, own = [], []
    for _ in range(nwin):
        barrier(world)
        torch.cuda.synchronize(device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            g.replay()
            e1.record(stream)
        torch.cuda.synchronize(device)
        barrier(world)
        ms = e0.elapsed_time(e1)
        own.append(ms)
        times.append(max_over_ranks(ms, world, device))
    step.own = own                           # this rank's windows (before the max)
    time.sleep(0.12)
    clk = clocks.summary(mark0, None) if clocks else None
    del g
    return times, clk, launches_per_step


def time_eager(step: Step, K: int, device):
    """K steps through the Python binding -> C ABI per step (no graph)."""
    torch.cuda.synchronize(device)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(K):
        step.run(i)
    e1.record()
    torch.cuda.synchronize(device)
    return e0.elapsed_time(e1) / K


E2E_STREAMS = int(os.environ.get("KT_E2E_STREAMS", "2"))   # dev A/B knob


def time_e2e(kt, cfg, op, K: int, W: int, world: int, device, rank):
    """Same metric end to end through kt_apply_host: every step copies its input
    from pinned host memory, runs the kernel, and copies the result back.
    Steps alternate over E2E_STREAMS caller streams, each with its own pinned
    input/output buffers and device work buffer (a serving loop with
    independent requests in flight), so one step's D2H overlaps the next
    step's H2D on the copy engines.  Timed from an event on the first stream
    (after all streams are idle) to events on every stream (the max)."""
    x_dev = WL.make_input(cfg, device=device, rank=rank)
    xs = [x_dev.cpu().pin_memory() for _ in range(E2E_STREAMS)]
    ys = [torch.empty_like(xs[0]).pin_memory() for _ in range(E2E_STREAMS)]
    del x_dev
    # whole-step chunks: one H2D, one kernel and one D2H per step; the
    # overlap comes from the other stream's step (kt_apply_host_ex)
    nbytes = xs[0].numel() * xs[0].element_size()
    works = [torch.empty(6 * nbytes, dtype=torch.uint8, device=device) for _ in range(E2E_STREAMS)]
    chunk = xs[0].numel()
    streams = [torch.cuda.Stream(device) for _ in range(E2E_STREAMS)]
    for i in range(max(1, W)):
        j = i % E2E_STREAMS
        kt.apply_host(op, xs[j], ys[j], works[j], stream=streams[j], chunk=chunk)
    torch.cuda.synchronize(device)
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(E2E_STREAMS)]
    e0.record(streams[0])
    for st in streams[1:]:
        st.wait_event(e0)
    for i in range(K):
        j = i % E2E_STREAMS
        kt.apply_host(op, xs[j], ys[j], works[j], stream=streams[j], chunk=chunk)
    for j, st in enumerate(streams):
        ends[j].record(st)
    torch.cuda.synchronize(device)
    barrier(world)
    ms = max(e0.elapsed_time(e) for e in ends) / K
    ms = max_over_ranks(ms, world, device)
    nb = xs[0].numel() * xs[0].element_size()
    return ms, nb, nb


def cpu_baseline(cfg, op, device, budget_s=12.0, max_elems=1 << 24):
    """The oracle as it stands, single-threaded on this host, on a bounded
    prefix of the same workload bytes; repeated until ~budget_s of CPU work."""
    import oracle as O
    x = WL.make_input(cfg, device=device)
    m = min(x.numel(), max_elems)
    if cfg.dtype == torch.bfloat16:
        xb = x.reshape(-1)[:m].view(torch.int16).cpu().numpy().view(np.uint16)
        f = (lambda: O.lstm_gates_bf16(xb, WL.LSTM_HIDDEN, 2)) if op == "lstm" else \
            (lambda: O.map_bf16(op, xb))
    else:
        xb = x.reshape(-1)[:m].view(torch.int32).cpu().numpy().view(np.uint32)
        f = lambda: O.map_f32(op, xb)
    del x
    f()  # load / build the library outside the timing
    reps, t = 0, 0.0
    while t < budget_s and reps < 1000:
        t0 = time.perf_counter()
        f()
        t += time.perf_counter() - t0
        reps += 1
    # also the same oracle on every host core -- the sample is
    # split into one contiguous slice per thread (ctypes drops the GIL for
    # the C call); the oracle itself is unchanged
    from concurrent.futures import ThreadPoolExecutor
    nthr = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    bounds = [(m * i // nthr, m * (i + 1) // nthr) for i in range(nthr)]
    if op == "lstm":
        width = 4 * WL.LSTM_HIDDEN
        rows = m // width
        bounds = [(width * (rows * i // nthr), width * (rows * (i + 1) // nthr)) for i in range(nthr)]
        part = lambda a, b: O.lstm_gates_bf16(xb[a:b], WL.LSTM_HIDDEN, 2)
    elif cfg.dtype == torch.bfloat16:
        part = lambda a, b: O.map_bf16(op, xb[a:b])
    else:
        part = lambda a, b: O.map_f32(op, xb[a:b])
    with ThreadPoolExecutor(nthr) as pool:
        list(pool.map(lambda ab: part(*ab), bounds))
        reps_mt, t_mt = 0, 0.0
        while t_mt < budget_s / 3 and reps_mt < 1000:
            t0 = time.perf_counter()
            list(pool.map(lambda ab: part(*ab), bounds))
            t_mt += time.perf_counter() - t0
            reps_mt += 1
    return {"value": round(m * reps / t / 1e9, 6), "unit": "Gelem/s", "cores": 1, "kind": "oracle",
            "sample": f"first {m} elements of the {cfg.key} input, {reps} passes, {t:.1f} s, "
                      f"single-threaded scalar C oracle (oracle/ktanh_oracle.c)",
            "host_cpu": _cpu_model(), "host_threads": os.cpu_count(),
            "all_cores": {"value": round(m * reps_mt / t_mt / 1e9, 6), "unit": "Gelem/s",
                          "cores": nthr,
                          "sample": f"same {m} elements split into {nthr} contiguous slices, one "
                                    f"thread each, {reps_mt} passes, {t_mt:.1f} s"}}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def load_traffic(key, op):
    """Steady-state DRAM bytes (read + write) per launch of the headline kernel
    from the newest committed ncu range-replay capture of THIS workload and
    call (profiles/ncu_range_traffic_<workload>_<op>_rNN.csv, written by
    tools/range_traffic.py: dram bytes over a range of back-to-back launches,
    so the write-back of earlier launches' dirty lines is counted)."""
    import csv
    pdir = os.path.join(ROOT, "profiles")
    if not os.path.isdir(pdir):
        return None, None
    prefix = f"ncu_range_traffic_{key}_{op}_r"
    for name in sorted(os.listdir(pdir), reverse=True):
        if not (name.startswith(prefix) and name.endswith(".csv")):
            continue
        try:
            text = open(os.path.join(pdir, name)).read().splitlines()
            launches = None
            for l in text:
                if "range of" in l:
                    toks = l.split("range of", 1)[1].split()
                    if toks and toks[0].isdigit():
                        launches = int(toks[0])
                        break
            rows = [l for l in text if l.startswith('"')]
            tot = 0.0
            for row in csv.DictReader(rows):
                if row.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    tot += float(row["Metric Value"].replace(",", ""))
            if tot > 0 and launches:
                return tot / launches, f"profiles/{name} (ncu range replay, {launches} launches)"
        except Exception:
            continue
    return None, None


# --config: workload, library call, oracle / host-path op of the headline line
HEADS = {"c1": ("c1_exhaustive_bf16", "ktanh_bf16", "tanh"), "c2": ("c2_bf16_2p24", "ktanh_bf16", "tanh"),
         "c3": ("c3_f32_2p28", "ktanh_f32", "tanh"), "c4": ("c4_lstm_gates", "lstm", "lstm"),
         "c5": ("c5_ffn_2p30", "kgelu_bf16", "gelu")}
DTYPE_NAME = {torch.bfloat16: "bf16", torch.float32: "f32"}

# demangled names as ncu lists them: <OP, FMT, NC, PF, unroll, threads per CTA>
KERNEL_NAME = {"ktanh_bf16": "kt::k_map<0, 0, 1, 1, 2, 256>", "ktanh_f32": "kt::k_map<0, 1, 1, 1, 4, 256>", "ktanh_f32_via_bf16": "kt::k_map<4, 1, 1, 1, 4, 128>",
               "kgelu_bf16": "kt::k_map<3, 0, 1, 1, 4, 128>", "kswish_bf16": "kt::k_map<2, 0, 1, 1, 2, 256>",
               "lstm": "kt::k_lstm<1>"}

EXTRA = [("c2_bf16_2p24", "ktanh_bf16"), ("c2_bf16_2p24", "ksigmoid_bf16"), ("c2_bf16_2p24", "ktanh64_bf16"),
         ("c3_f32_2p28", "ktanh_f32"), ("c3_f32_2p28", "ksigmoid_f32"),
         ("c3_f32_2p28", "ktanh_f32:p23"), ("c3_f32_2p28", "ktanh_f32_via_bf16"),
         ("c3_f32_2p28", "kgelu_f32"), ("c3_f32_2p28", "kswish_f32"),
         ("c4_lstm_gates", "lstm"), ("c5_ffn_2p30", "kgelu_bf16"), ("c5_ffn_2p30", "kswish_bf16"),
         ("c5_ffn_2p30", "kgelu_swish_bf16"), ("c5_ffn_2p30", "kgelu_bwd_bf16"),
         ("c4_lstm_gates", "lstm_cell")]


def l2_policy(key, call):
    """How the timed steps avoid L2 reuse (the same rule Step applies)."""
    cfg = WL.CONFIGS[key]
    step = (3 if call == "kgelu_swish_bf16" else 2) * cfg.numel * cfg.elem_bytes
    if call == "lstm_cell":
        step = 18 * (cfg.numel // 4)
    if step >= 2 * L2_BYTES:
        return f"inputs larger than L2 ({step >> 20} MiB moved per step, no flush needed)"
    sets = max(2, math.ceil(4 * L2_BYTES / step))
    return f"{sets} rotating input/output sets ({sets * step >> 20} MiB > 4x L2)"


def head_config(key, call, world):
    """The `config` object of the headline line; the reference arm prints the
    identical object (same workload, same per-GPU size, same call)."""
    cfg = WL.CONFIGS[key]
    return {"workload": key, "desc": cfg.desc, "elements_per_gpu": cfg.numel, "call": call,
            "parallelism": f"{world} independent shard(s) (seed + rank), no collective",
            "l2": l2_policy(key, call)}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    key, call, op = HEADS[args.config]
    cfg = WL.CONFIGS[key]
    import oracle as O
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    x = WL.make_input(cfg, device=dev, numel=None if cfg.numel <= 1 << 24 else 1 << 24)
    m = min(x.numel(), 1 << 22)                   # bounded sample per step
    if op == "lstm":
        m -= m % (4 * WL.LSTM_HIDDEN)             # whole gate rows
    if cfg.dtype == torch.bfloat16:
        xb = x.reshape(-1)[:m].view(torch.int16).cpu().numpy().view(np.uint16)
        f = (lambda: O.lstm_gates_bf16(xb, WL.LSTM_HIDDEN, 2)) if op == "lstm" else \
            (lambda: O.map_bf16(op, xb))
    else:
        xb = x.reshape(-1)[:m].view(torch.int32).cpu().numpy().view(np.uint32)
        f = lambda: O.map_f32(op, xb)
    del x
    for _ in range(args.warmup):
        f()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    sec = sum(ts) / len(ts)
    val = m / sec / 1e9
    sample = (f"each step: the scalar C oracle (oracle/ktanh_oracle.c, single-threaded) on {m} "
              f"elements of the {key} workload (a prefix of a tensor drawn with the GPU arm's "
              f"generator, seed and distribution), {args.steps} timed steps")
    out = {
        "impl": "reference",
        "metric": "K-TanH Gelem/s and achieved HBM GB/s vs ~8 TB/s peak at 1/2/4/8 B200",
        "value": round(val, 6), "unit": "Gelem/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": DTYPE_NAME[cfg.dtype], "data": "synthetic",
        "config": head_config(key, call, world),
        "cpu_baseline": {"value": round(val, 6), "unit": "Gelem/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "host_cpu": _cpu_model()},
        "e2e": {"value": round(val, 6), "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


TABLE2_MAPS = [("ktanh", None), ("sfu", "apx:sfu:0:0"), ("libm", "apx:libm:0:0"),
               ("pade_3_2", "apx:pade:3:2"), ("pade_7_8", "apx:pade:7:8"),
               ("minimax_2", "apx:minimax:2:0"), ("minimax_3", "apx:minimax:3:0"),
               ("taylor_2", "apx:taylor:2:0"), ("taylor_3", "apx:taylor:3:0"),
               ("torch_tanh", "torch:tanh")]            # library (ATen) kernel, context


def lstm_gemm_line(kt, K, W, world, device, rank):
    """NEXT-2 on config 4: the GNMT LSTM gate GEMM that produces config 4's
    [128 x 50, 4 x 1024] gate block (input [6400, 1024] x W [4096, 1024]^T),
    with K-Sigmoid / K-TanH fused into the tcgen05 epilogue, vs the GEMM
    alone and the unfused GEMM + klstm_gates_bf16 (all through the C ABI)."""
    H = WL.LSTM_HIDDEN
    M, Kd = 128 * 50, H
    gA = WL.make_input("c4_lstm_gates", device=device, rank=rank, numel=M * Kd).reshape(M, Kd)
    gB = (WL.make_input("c4_lstm_gates", device=device, rank=rank, numel=4 * H * Kd, seed=9)
          .reshape(4 * H, Kd) * 0.05).to(torch.bfloat16)
    sets = 4
    gCs = [torch.empty(M, 4 * H, dtype=torch.bfloat16, device=device) for _ in range(sets)]
    gTs = [torch.empty(M, 4 * H, dtype=torch.bfloat16, device=device) for _ in range(sets)]

    class _S:
        n, bytes_per_step = M * 4 * H, 0

        def __init__(self, fn):
            self.fn = fn
            self.kt = kt

        def run(self, i):
            self.fn(i % sets)
    cs = [torch.randn(M, H, device=device) for _ in range(sets)]
    cns = [torch.empty_like(c) for c in cs]
    hns = [torch.empty(M, H, dtype=torch.bfloat16, device=device) for _ in range(sets)]
    res = {}
    for name, fn in (("fused", lambda s: kt.kgemm_lstm_gates_bf16(gA, gB, H, 2, out=gCs[s])),
                     ("gemm_cell_fused", lambda s: kt.kgemm_lstm_cell_bf16(gA, gB, cs[s], H, c_next=cns[s],
                                                                           h_next=hns[s])),
                     ("gemm_then_cell", lambda s: (kt.kgemm_bf16(gA, gB, out=gTs[s]),
                                                   kt.klstm_cell_bf16(gTs[s], cs[s], H, c_next=cns[s],
                                                                      h_next=hns[s]))),
                     ("gemm_only", lambda s: kt.kgemm_bf16(gA, gB, out=gCs[s])),
                     ("unfused", lambda s: (kt.kgemm_bf16(gA, gB, out=gTs[s]),
                                            kt.klstm_gates_bf16(gTs[s], H, 2, out=gCs[s])))):
        wts, _, _ = time_windows(_S(fn), K, W, world, device, None, min_total_s=0.3, max_windows=20)
        res[name] = statistics.median(wts) / K
    fl = 2.0 * M * 4 * H * Kd
    return {"ms_per_step": round(res["fused"], 5), "tflops_per_gpu": round(fl / (res["fused"] / 1e3) / 1e12, 1),
            "gemm_only_ms": round(res["gemm_only"], 5), "unfused_gemm_plus_klstm_gates_ms": round(res["unfused"], 5),
            "gemm_with_fused_cell_ms": round(res["gemm_cell_fused"], 5),
            "gemm_then_klstm_cell_ms": round(res["gemm_then_cell"], 5),
            "note": "gates = K-TanH (quarter 2) / K-Sigmoid applied in the tcgen05 GEMM epilogue; "
                    "bit-identical to kgemm_bf16 + klstm_gates_bf16"}


def table2_b200(kt, K, W, world, device, rank, peak):
    """Table 2 on B200.  For K-TanH and
    each float-op comparator: accuracy over every finite BF16 input (the
    GPU's own outputs vs binary64 tanh; max |err|, max relative err over
    x != 0, reading A11), streaming throughput on config 2 (BF16 2^24,
    rotating sets) and register-resident SM cycles per element
    (kt_alu_probe: the analogue of the paper's cycles per TanH)."""
    import numpy as np
    xall = WL.make_input("c1_exhaustive_bf16", device=device)
    xb = xall.view(torch.int16).cpu().numpy().view(np.uint16)
    with np.errstate(invalid="ignore"):          # NaN patterns widen to NaN (no warning)
        xv = (xb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    fin = np.isfinite(xv)
    ref = np.tanh(xv)
    g = torch.Generator().manual_seed(2)
    sample = (torch.randn(8192, generator=g) * 2).to(torch.bfloat16).view(torch.int16) \
        .numpy().view(np.uint16).view(np.uint32)[:4096].copy()
    rows = {}
    for name, op in TABLE2_MAPS:
        if op is None:
            y = kt.ktanh_bf16(xall)
            cyc, _ = kt.alu_probe("bf16", sample, lut=kt.paper_lut())
            st = Step(kt, "c2_bf16_2p24", "ktanh_bf16", device, rank)
        elif op.startswith("torch:"):
            y = torch.tanh(xall)
            cyc = None
            st = Step(kt, "c2_bf16_2p24", op, device, rank)
        else:
            _, kind, p, q = op.split(":")
            A = kt.Apx(kind, int(p), int(q))
            y = kt.kt_apx_tanh_bf16(xall, A)
            cyc, _ = kt.alu_probe("bf16", sample, apx=A)
            st = Step(kt, "c2_bf16_2p24", op, device, rank)
        yb = y.view(torch.int16).cpu().numpy().view(np.uint16)
        with np.errstate(invalid="ignore"):
            yv = (yb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        err = np.abs(yv[fin] - ref[fin])
        nz = fin & (xv != 0)
        rel = np.abs(yv[nz] - ref[nz]) / np.abs(ref[nz])
        wts, _, _ = time_windows(st, K, W, world, device, None, min_total_s=0.3, max_windows=400)
        m_ = statistics.median(wts) / K
        gbs = st.bytes_per_step / (m_ / 1e3) / 1e9
        rows[name] = {"max_abs_err": float(err.max()), "max_rel_err_pct": round(float(rel.max()) * 100, 4),
                      "gelem_s": round(st.n * world / (m_ / 1e3) / 1e9, 2),
                      "hbm_gbs_per_gpu": round(gbs, 1), "frac_of_measured": round(gbs / peak, 4),
                      "sm_cycles_per_elem_per_sm": None if cyc is None else round(cyc, 4)}
        del st
        torch.cuda.empty_cache()
    # GELU: K-GELU vs ATen's BF16 GELU (tanh form and erf form),
    # accuracy against the exact x Phi(x) in binary64 over every finite BF16 input
    import math
    ref_g = np.zeros_like(xv)
    ref_g[fin] = np.array([v * 0.5 * (1.0 + math.erf(v / math.sqrt(2.0))) for v in xv[fin]])
    grows = {}
    for name, op, fn in (("kgelu", "kgelu_bf16", lambda t: kt.kgelu_bf16(t)),
                         ("torch_gelu_tanh", "torch:gelu_tanh",
                          lambda t: torch.nn.functional.gelu(t, approximate="tanh")),
                         ("torch_gelu_erf", "torch:gelu_erf", lambda t: torch.nn.functional.gelu(t))):
        yb = fn(xall).view(torch.int16).cpu().numpy().view(np.uint16)
        with np.errstate(invalid="ignore"):
            yv = (yb.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
        ok = fin & np.isfinite(ref_g)
        err = np.abs(yv[ok] - ref_g[ok])
        st = Step(kt, "c2_bf16_2p24", op, device, rank)
        wts, _, _ = time_windows(st, K, W, world, device, None, min_total_s=0.3, max_windows=400)
        m_ = statistics.median(wts) / K
        gbs = st.bytes_per_step / (m_ / 1e3) / 1e9
        grows[name] = {"max_abs_err_vs_exact_gelu": float(err.max()),
                       "max_abs_err_abs_x_le_4": float(np.abs(yv - ref_g)[fin & (np.abs(xv) <= 4)].max()),
                       "gelem_s": round(st.n * world / (m_ / 1e3) / 1e9, 2),
                       "hbm_gbs_per_gpu": round(gbs, 1), "frac_of_measured": round(gbs / peak, 4)}
        del st
        torch.cuda.empty_cache()
    return {"workload": "accuracy: all finite BF16 inputs; throughput: c2_bf16_2p24 (BF16 in/out)",
            "note": "paper Table 2 (Intel CLX AVX512, cycles per TanH per core) is context only; "
                    "readings R-CMP-* in DESIGN.md; torch_* rows are ATen library kernels",
            "rows": rows, "gelu_rows": grows}


class StubStep:
    """--stub test hook: a host copy standing in for the library call."""

    def __init__(self, n=1 << 16, rank=0):
        g = torch.Generator().manual_seed(5 + rank)
        self.xs = [torch.randn(n, generator=g).to(torch.bfloat16)]
        self.ys = [torch.empty_like(self.xs[0])]
        self.n, self.sets, self.bytes_per_step = n, 1, 4 * n
        self.cell = self.dual = self.bwd = False

    def run(self, i):
        self.ys[0].copy_(self.xs[0])


def time_windows_stub(step, K, W, world, nwin=3):
    """The multi-rank window protocol of time_windows with a host timer."""
    for i in range(W):
        step.run(i)
    times, own = [], []
    for _ in range(nwin):
        barrier(world)
        t0 = time.perf_counter()
        for i in range(K):
            step.run(W + i)
        ms = (time.perf_counter() - t0) * 1e3
        barrier(world)
        own.append(ms)
        times.append(max_over_ranks(ms, world, torch.device("cpu")))
    step.own = own
    return times, {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["stub"], "samples": 0}, 1.0


def oracle_check(x, y, op, m=1 << 16, seed=0, stub=False):
    """Part of the cpu_baseline leg, run by EVERY rank after its timed region:
    m seeded sample positions (plus the first and last element) of this rank's
    output y against the oracle on the same input bytes.  Bit-exact, NaN by
    class, +-0 by value for the derived ops (DESIGN.md R-DERIVED / A21)."""
    n = x.numel()
    idx = np.random.default_rng(seed).integers(0, n, m, dtype=np.int64)
    idx = np.concatenate([idx, [0, n - 1]])
    it = torch.from_numpy(idx).to(x.device)
    bf16 = x.dtype == torch.bfloat16
    iv = torch.int16 if bf16 else torch.int32
    nv = np.uint16 if bf16 else np.uint32
    xs = x.reshape(-1)[it].view(iv).cpu().numpy().view(nv)
    ys = y.reshape(-1)[it].view(iv).cpu().numpy().view(nv)
    if stub:
        want = xs                                   # the stub step is a copy
    else:
        import oracle as O
        want = O.map_bf16(op, xs) if bf16 else O.map_f32(op, xs)
    return mismatches(ys, want, op, bf16), int(idx.size)


def mismatches(got, want, op, bf16):
    """Elements of got != want, NaN compared by class (not for K-TanH: it
    passes NaN through unchanged) and +-0 by value for K-Swish / K-GELU."""
    mag = 0x7FFF if bf16 else 0x7FFFFFFF
    nan_lo = 0x7F80 if bf16 else 0x7F800000
    g, w = got.astype(np.int64) & mag, want.astype(np.int64) & mag
    bad = got != want
    if op != "tanh":
        bad &= ~((g > nan_lo) & (w > nan_lo))
    if op in ("swish", "gelu"):
        bad &= ~((g == 0) & (w == 0))
    return int(bad.sum())


def full_shard_check(x, y, op):
    """--full-check (opt-in, part of the cpu_baseline leg): EVERY element of
    this rank's output against the oracle, on all host cores (SURVEY.md 8(d):
    "check all shards"); returns (mismatches, elements, seconds)."""
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor
    bf16 = x.dtype == torch.bfloat16
    iv, nv = (torch.int16, np.uint16) if bf16 else (torch.int32, np.uint32)
    xs = x.reshape(-1).view(iv).cpu().numpy().view(nv)
    ys = y.reshape(-1).view(iv).cpu().numpy().view(nv)
    n = xs.size
    nthr = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    step = 1 << 22

    def part(a):
        b = min(n, a + step)
        want = O.map_bf16(op, xs[a:b]) if bf16 else O.map_f32(op, xs[a:b])
        return mismatches(ys[a:b], want, op, bf16)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(nthr) as pool:
        bad = sum(pool.map(part, range(0, n, step)))
    return bad, n, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ktanh", choices=["ktanh", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip the side measurements (extra)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--config", default="c5", choices=sorted(HEADS),
                    help="workload of the headline line (default c5: BASELINE.json configs[4], "
                         "the configuration the metric is quoted on at 1/2/4/8 GPUs)")
    ap.add_argument("--full-check", action="store_true",
                    help="also check every element of each rank's output against the oracle (all host cores)")
    ap.add_argument("--stub", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    rank, local_rank, world = dist_env()
    if args.stub:
        ndev = world                                   # pretend: one device per rank
        device = torch.device("cpu")
    else:
        if not torch.cuda.is_available():
            raise SystemExit("bench.py needs a CUDA device (there is no CPU path)")
        ndev = torch.cuda.device_count()
    dev_index = local_rank % ndev           # one GPU per rank on a full node
    if not args.stub:
        torch.cuda.set_device(dev_index)
        device = torch.device("cuda", dev_index)
    if world > 1:
        # gloo: the only collectives are timing scalars (barrier, max, sum,
        # gather); the data path has none (north_star item (c))
        _kd().init("gloo")
        if world > ndev and rank == 0:
            print(f"warning: {world} ranks on {ndev} GPU(s): functional run, not a measurement",
                  file=sys.stderr)

    K, W = args.steps, args.warmup
    head_key, head_op, head_oracle_op = HEADS[args.config]
    hcfg = WL.CONFIGS[head_key]
    if args.stub:
        kt = None
        peak, peak_src = measured_peaks()
        clocks = None
        step = StubStep(rank=rank)
        windows, clk, lps = time_windows_stub(step, K, W, world)
        input_sha = "stub"
    else:
        import paper_1909_07729_b200 as kt
        peak, peak_src = measured_peaks()
        clocks = ClockSampler(dev_index) if rank == 0 or world > 1 else None
        if clocks:
            clocks.start()
            time.sleep(0.3)
        step = Step(kt, head_key, head_op, device, rank)
        import hashlib
        input_sha = hashlib.sha256(step.xs[0].view(torch.int16).cpu().numpy().tobytes()).hexdigest()
        windows, clk, lps = time_windows(step, K, W, world, device, clocks)
    ms_win = statistics.median(windows)
    ms = ms_win / K
    n_total = step.n * world
    value = n_total / (ms / 1e3) / 1e9
    gbs_per_gpu = step.bytes_per_step / (ms / 1e3) / 1e9
    own_ms = statistics.median(step.own) / K       # this rank's own windows (per-rank report)
    # every rank: sampled check of its own output against the oracle (cpu_baseline leg)
    bad = checked = 0
    if not args.no_cpu and head_oracle_op != "lstm":
        bad, checked = oracle_check(step.xs[0], step.ys[0], head_oracle_op, seed=rank, stub=args.stub)
    if args.full_check and not args.stub and head_oracle_op != "lstm":
        fbad, fn, fsec = full_shard_check(step.xs[0], step.ys[0], head_oracle_op)
        bad, checked = bad + fbad, checked + fn
    per_rank = _kd().gather_over_ranks([rank, dev_index, own_ms, bad, checked]) if world > 1 else \
        [[rank, dev_index, own_ms, bad, checked]]
    eager_ms = ms if args.stub else time_eager(step, K, device)
    sets, head_bytes = step.sets, step.bytes_per_step
    del step
    if not args.stub:
        torch.cuda.empty_cache()

    K_e2e = min(K, 20)
    if args.stub:
        e2e = {"value": None, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "stub"}
    elif head_oracle_op != "lstm":
        e2e_ms, h2d, d2h = time_e2e(kt, hcfg, head_oracle_op, K_e2e, W, world, device, rank)
        e2e_val = n_total / (e2e_ms / 1e3) / 1e9
        e2e = {"value": round(e2e_val, 4), "unit": "Gelem/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 4), "steps": K_e2e,
               "path": f"kt_apply_host_ex through the Python binding (pinned host buffers of the "
                       f"{head_key} input, one chunk per step; steps alternate over {E2E_STREAMS} "
                       f"caller streams so each D2H overlaps the next step's H2D)"}
    else:
        e2e = {"value": None, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "note": "no host-buffer entry point for the LSTM gate call (kt_apply_host serves "
                       "the elementwise ops)"}

    extra = {}
    if not args.no_extra and not args.stub:
        extra = side_lines(kt, args, K, W, world, device, rank, peak, head_key, head_op)

    cpu = None
    if rank == 0 and not args.no_cpu and not args.stub:
        cpu = cpu_baseline(hcfg, head_oracle_op, device)
    if cpu is not None:
        cpu["check"] = {"what": "every rank: seeded sample of its own GPU output vs the oracle on the "
                                "same input bytes, after the timed region" +
                                ("; plus EVERY element of each rank's output (--full-check)"
                                 if args.full_check else ""),
                        "samples_per_rank": int(per_rank[0][4]),
                        "mismatches": int(sum(r[3] for r in per_rank))}

    if clocks:
        clocks.stop()
    traffic, traffic_src = load_traffic(head_key, head_op)
    if rank == 0:
        out = {
            "metric": "K-TanH Gelem/s and achieved HBM GB/s vs ~8 TB/s peak at 1/2/4/8 B200",
            "value": round(value, 3), "unit": "Gelem/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": round(ms, 6), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE_NAME[hcfg.dtype],
            "data": "synthetic",
            "config": head_config(head_key, head_op, world),
            "timing": {"input_sha256_rank0": input_sha,
                       "launch": "CUDA graph of K library calls per timed window",
                       "windows": len(windows), "window_ms_median": round(ms_win, 5),
                       "window_ms_best": round(min(windows), 5)},
            "hbm_gbs_per_gpu": round(gbs_per_gpu, 1),
            "roofline": {"bound": "hbm", "achieved": round(gbs_per_gpu, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(gbs_per_gpu / peak, 4),
                         "traffic": traffic, "peak_source": peak_src,
                         "frac_of_8tbs": round(gbs_per_gpu / NOMINAL_HBM_GBS, 4),
                         "kernel": KERNEL_NAME.get(head_op, head_op),
                         "algorithmic_bytes_per_launch": head_bytes,
                         "traffic_source": traffic_src},
            "per_rank": [{"rank": int(r[0]), "device": int(r[1]), "ms_per_step": round(r[2], 6),
                          "checked": int(r[4]), "mismatches": int(r[3])} for r in per_rank],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(round(lps * K)),
            "eager_ms_per_step": round(eager_ms, 6),
            "clocks": clk,
            "extra": extra,
        }
        if args.stub:
            out["stub"] = True
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def side_lines(kt, args, K, W, world, device, rank, peak, head_key, head_op):
    """The `extra` object: the other configs and calls (the headline excluded)."""
    extra = {}
    for key, op in EXTRA:
        if (key, op) == (head_key, head_op):
            continue
        st = Step(kt, key, op, device, rank)
        wts, _, _ = time_windows(st, K, W, world, device, None, min_total_s=0.3, max_windows=10)
        m_ = statistics.median(wts) / K
        units = st.n // 4 if st.cell else st.n
        tr, tr_src = load_traffic(key, op)
        extra[f"{key}:{op}"] = {
            "elements_per_gpu": units, "ms_per_step": round(m_, 5),
            "gelem_s": round(units * world / (m_ / 1e3) / 1e9, 3),
            "hbm_gbs_per_gpu": round(st.bytes_per_step / (m_ / 1e3) / 1e9, 1),
            "frac_of_measured": round(st.bytes_per_step / (m_ / 1e3) / 1e9 / peak, 4),
            "frac_of_8tbs": round(st.bytes_per_step / (m_ / 1e3) / 1e9 / NOMINAL_HBM_GBS, 4),
            "algorithmic_bytes_per_launch": st.bytes_per_step,
            "l2": "inputs larger than L2" if st.sets == 1 else f"{st.sets} rotating sets"}
        if tr is not None:
            extra[f"{key}:{op}"]["traffic"] = tr
            extra[f"{key}:{op}"]["traffic_source"] = tr_src
        if st.dual:
            extra[f"{key}:{op}"]["note"] = ("one pass, two outputs (K-GELU and K-Swish of x, "
                                            "6 B/element); gelem_s counts input elements")
        del st
        torch.cuda.empty_cache()

    # NEXT-2: the FFN up-projection that produces config 5's [65536, 16384]
    # activations, K-GELU fused into the tcgen05 GEMM epilogue (K = 4096)
    Mg, Ng, Kg = WL.CONFIGS["c5_ffn_2p30"].shape[0], WL.CONFIGS["c5_ffn_2p30"].shape[1], 4096
    gA = WL.make_input("c5_ffn_2p30", device=device, rank=rank, numel=Mg * Kg).reshape(Mg, Kg)
    gB = (WL.make_input("c5_ffn_2p30", device=device, rank=rank, numel=Ng * Kg, seed=7)
          .reshape(Ng, Kg) * 0.02).to(torch.bfloat16)
    gC = torch.empty(Mg, Ng, dtype=torch.bfloat16, device=device)

    class _G:
        n, bytes_per_step, sets = Mg * Ng, 0, 1

        def run(self, i):
            kt.kgemm_bf16(gA, gB, epilogue="gelu", out=gC)
    gst = _G()
    gst.kt = kt
    wts, _, _ = time_windows(gst, K, W, world, device, None, min_total_s=0.3, max_windows=5)
    m_ = statistics.median(wts) / K
    tf = 2.0 * Mg * Ng * Kg / (m_ / 1e3) / 1e12
    bf16_peak, bf16_sus = 1674.5, 1376.5
    try:
        _mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        bf16_peak, bf16_sus = float(_mp["bf16_tflops"]), float(_mp["bf16_tflops_sustained"])
    except Exception:
        pass
    extra["ffn_gemm_M65536_N16384_K4096:kgemm_bf16+kgelu"] = {
        "ms_per_step": round(m_, 4), "tflops_per_gpu": round(tf, 1),
        "roofline": {"bound": "tensor", "peak": bf16_sus, "unit": "TFLOP/s",
                     "frac": round(tf / bf16_sus, 4), "frac_of_burst": round(tf / bf16_peak, 4),
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (a "
                                    f"{m_ * K:.0f} ms loop of {m_:.1f} ms kernels)"},
        "note": "tcgen05 GEMM, fp32 TMEM accumulation, K-GELU applied in the epilogue"}
    del gA, gB, gC
    torch.cuda.empty_cache()

    extra["table2_b200"] = table2_b200(kt, K, W, world, device, rank, peak)
    extra["lstm_gates_gemm_M6400_N4096_K1024:kgemm_lstm_gates_bf16"] = lstm_gemm_line(
        kt, K, W, world, device, rank)
    return extra


if __name__ == "__main__":
    sys.exit(main())
