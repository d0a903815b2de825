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
def gemm_line(epi, K=200):
    """FFN GEMM 65536 x 16384 x 4096 with a K-op epilogue (bench.py's line)."""
    M, N, Kd = 65536, 16384, 4096
    import workloads as WL
    A = WL.make_input("c5_ffn_2p30", device=dev, numel=M * Kd).reshape(M, Kd)
    B = (WL.make_input("c5_ffn_2p30", device=dev, numel=N * Kd, seed=7).reshape(N, Kd) * 0.02).to(torch.bfloat16)
    C = torch.empty(M, N, dtype=torch.bfloat16, device=dev)

    class _G:
        n, bytes_per_step, sets = M * N, 0, 1

        def run(self, i):
            kt.kgemm_bf16(A, B, epilogue=epi, out=C)
    g = _G()
    g.kt = kt
    wts, _, _ = bench.time_windows(g, 20, 3, 1, dev, None, min_total_s=1.0, max_windows=10)
    ms = statistics.median(wts) / 20
    return {"ms": round(ms, 4), "tflops": round(2.0 * M * N * Kd / (ms / 1e3) / 1e12, 1)}


for line in lines:
    if line.startswith("gemm:"):
        out[line] = gemm_line(line[5:] or None)
        torch.cuda.empty_cache()
        continue
    key, op = line.split(":", 1)
    st = bench.Step(kt, key, op, dev, 0)
    wts, clk, _ = bench.time_windows(st, 200, 5, 1, dev, None, min_total_s=1.0, max_windows=40)
    ms = statistics.median(wts) / 200
    gbs = st.bytes_per_step / (ms / 1e3) / 1e9
    out[line] = {"us": round(ms * 1e3, 3), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    del st
    torch.cuda.empty_cache()
print(json.dumps(out), flush=True)
