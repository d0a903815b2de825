"""A/B of library builds on the streaming lines (dev tool).

    python tools/ab_stream.py [key:op ...]     (library from KT_LIB, default in-tree)

Times each line like bench.py's headline (graph-replayed windows of K = 200
library calls, median window) and prints one JSON object.  Run it once per
build, interleaved (e.g. default, variant, default, variant) so clock drift
under the power cap shows up as spread rather than as a difference.
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import bench
import paper_1909_07729_b200 as kt

lines = sys.argv[1:] or ["c5_ffn_2p30:kgelu_bf16", "c5_ffn_2p30:kswish_bf16",
                         "c5_ffn_2p30:kgelu_swish_bf16", "c4_lstm_gates:lstm_cell"]
peak, _ = bench.measured_peaks()
dev = torch.device("cuda", 0)
out = {"lib": os.environ.get("KT_LIB", "in-tree")}
for line in lines:
    key, op = line.split(":", 1)
    st = bench.Step(kt, key, op, dev, 0)
    wts, clk, _ = bench.time_windows(st, 200, 5, 1, dev, None, min_total_s=1.0, max_windows=40)
    ms = statistics.median(wts) / 200
    gbs = st.bytes_per_step / (ms / 1e3) / 1e9
    out[line] = {"us": round(ms * 1e3, 3), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    del st
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
