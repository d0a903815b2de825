"""Summarise ncu --set full reports into profiles/ (JSON + markdown).  Dev tool.

    python tools/ncu_summary.py ROUND report1.ncu-rep [report2 ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "gpu_dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "dram__cycles_elapsed.avg.per_second": "dram_clock",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed":
        "tensor_pipe_pct",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
        "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "Hz": 1, "Khz": 1e3,
        "Mhz": 1e6, "Ghz": 1e9}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarise(rep):
    hdr, units, rows = raw(rep)
    res = []
    for r in rows:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * UNIT.get(units[i], 1)
        stalls = {}
        for i, h in enumerate(hdr):
            pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
            if h.startswith(pre) and h.endswith(suf):
                try:
                    stalls[h[len(pre):-len(suf)]] = round(float(r[i]), 3)
                except ValueError:
                    pass
        d["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        if "dram_read" in d and "duration" in d:
            d["dram_bytes_per_launch"] = d["dram_read"] + d.get("dram_write", 0)
            d["dram_gbs"] = d["dram_bytes_per_launch"] / d["duration"] / 1e9
        res.append(d)
    return res


def attach_algorithmic(allk, alg_bytes):
    for tag, ks in allk.items():
        for d in ks:
            if alg_bytes.get(tag) and "duration" in d:
                d["algorithmic_bytes_per_launch"] = alg_bytes[tag]
                d["algorithmic_gbs"] = alg_bytes[tag] / d["duration"] / 1e9


if __name__ == "__main__":
    rnd = sys.argv[1]
    allk = {}
    for rep in sys.argv[2:]:
        tag = os.path.basename(rep).replace(".ncu-rep", "")
        allk[tag] = summarise(rep)
    alg = {}
    for tag in allk:
        if "tanh_bf16" in tag or "sigmoid" in tag:
            alg[tag] = 4 << 24
        elif "tanh_f32" in tag:
            alg[tag] = 8 << 28
        elif "gemm" in tag:
            alg[tag] = 0
        elif "gelu" in tag or "swish" in tag:
            alg[tag] = 4 << 30
        elif "lstm_cell" in tag or "cell" in tag:
            alg[tag] = 18 * 128 * 50 * 1024
        elif "gelu_bwd" in tag:
            alg[tag] = 6 << 30
        elif "lstm" in tag:
            alg[tag] = 4 * 128 * 50 * 4096
    attach_algorithmic(allk, alg)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_full_{rnd}.json"), "w") as f:
        json.dump(allk, f, indent=1)
    for tag, ks in allk.items():
        for d in ks:
            print(f"{tag}: {d['kernel'][:60]}")
            for k in ("duration", "dram_read", "dram_write", "dram_gbs", "algorithmic_gbs", "tensor_pipe_pct", "dram_pct_peak", "alu_pipe_pct",
                      "fma_pipe_pct", "issue_active_pct", "warps_active_pct", "regs", "grid", "sm_clock"):
                if k in d:
                    print(f"   {k:18s} {d[k]:.4g}")
            print("   stalls", d["top_stalls"])
