"""GEMM + fused LSTM cell vs GEMM alone over the reduction size K (is the
cell epilogue hidden behind the mainloop?).  Graph-replayed windows as in
bench.py.  python tools/cell_gemm_scan.py"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_07729_b200 as kt  # noqa: E402


class S:
    def __init__(self, fn):
        self.fn, self.kt, self.n, self.bytes_per_step = fn, kt, 1, 0

    def run(self, i):
        self.fn(i % 4)


dev = torch.device("cuda", 0)
H, M = 1024, 6400
out = []
for Kd in (256, 512, 1024, 2048, 4096):
    g = torch.Generator(device=dev).manual_seed(1)
    A = torch.randn(M, Kd, device=dev, generator=g).to(torch.bfloat16)
    B = (torch.randn(4 * H, Kd, device=dev, generator=g) * 0.05).to(torch.bfloat16)
    cs = [torch.randn(M, H, device=dev, generator=g) for _ in range(4)]
    cns = [torch.empty_like(c) for c in cs]
    hns = [torch.empty(M, H, dtype=torch.bfloat16, device=dev) for _ in range(4)]
    Cs = [torch.empty(M, 4 * H, dtype=torch.bfloat16, device=dev) for _ in range(4)]
    row = {"K": Kd}
    for name, fn in (("gemm", lambda s: kt.kgemm_bf16(A, B, out=Cs[s])),
                     ("gemm_cell", lambda s: kt.kgemm_lstm_cell_bf16(A, B, cs[s], H, c_next=cns[s], h_next=hns[s]))):
        w, _, _ = bench.time_windows(S(fn), 100, 5, 1, dev, None, min_total_s=0.2, max_windows=20)
        row[name + "_us"] = round(statistics.median(w) / 100 * 1e3, 2)
    row["extra_us"] = round(row["gemm_cell_us"] - row["gemm_us"], 2)
    out.append(row)
    print(json.dumps(row), flush=True)
