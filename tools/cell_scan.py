"""LSTM cell throughput vs batch rows (dev tool): is the standalone cell
limited by its wave tail?  Config 4 is [6400, 1024] = 2.70 resident waves of
256-thread CTAs at 4 CTAs/SM; B = 7104 is exactly 3.

    python tools/cell_scan.py [B ...]    (KT_LIB selects the library build)
"""
import json
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1909_07729_b200 as kt

H = 1024
rows = [int(a) for a in sys.argv[1:]] or [2368, 4736, 5920, 6400, 7104, 9472, 14208]
peak, _ = bench.measured_peaks()
dev = torch.device("cuda", 0)
L2 = 126 << 20
out = {"lib": os.environ.get("KT_LIB", "in-tree")}


class _Cell:
    def __init__(self, B):
        step_bytes = 18 * B * H
        self.sets = max(2, math.ceil(4 * L2 / step_bytes))
        g = torch.Generator(device=dev).manual_seed(B)
        self.xs = [(torch.randn(B, 4 * H, device=dev, generator=g) * 2).to(torch.bfloat16)
                   for _ in range(self.sets)]
        self.cs = [torch.randn(B, H, device=dev, generator=g) for _ in range(self.sets)]
        self.cns = [torch.empty_like(c) for c in self.cs]
        self.hs = [torch.empty(B, H, dtype=torch.bfloat16, device=dev) for _ in range(self.sets)]
        self.bytes_per_step = step_bytes
        self.kt = kt

    def run(self, i):
        s = i % self.sets
        kt.klstm_cell_bf16(self.xs[s], self.cs[s], H, c_next=self.cns[s], h_next=self.hs[s])


for B in rows:
    st = _Cell(B)
    wts, clk, _ = bench.time_windows(st, 200, 5, 1, dev, None, min_total_s=1.0, max_windows=40)
    ms = statistics.median(wts) / 200
    gbs = st.bytes_per_step / (ms / 1e3) / 1e9
    out[B] = {"waves": round(B * H / 16 / (148 * 4 * 256), 2), "us": round(ms * 1e3, 3),
              "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    del st
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
