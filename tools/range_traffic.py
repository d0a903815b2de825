"""Steady-state DRAM traffic per step of one bench workload, measured over a
RANGE of back-to-back launches (ncu --replay-mode range between
cudaProfilerStart / Stop), so the write-back of earlier launches' dirty
output lines is counted (a single-kernel capture misses it for inputs that
fit in L2).  bench.py reads the result from
profiles/ncu_range_traffic_<workload>_<op>_rNN.csv as roofline.traffic.

  ncu --replay-mode range --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      python tools/range_traffic.py <workload> <op> [launches]

  e.g. c5_ffn_2p30 kgelu_bf16 8   |   c2_bf16_2p24 ktanh_bf16 64   |   c3_f32_2p28 ktanh_f32 16
       c4_lstm_gates lstm 64         |   c5_ffn_2p30 kgelu_swish_bf16 4 (op names as in bench.py)
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1909_07729_b200 as kt
import workloads as WL

L2_BYTES = 126 * 1024 * 1024

key = sys.argv[1] if len(sys.argv) > 1 else "c2_bf16_2p24"
op = sys.argv[2] if len(sys.argv) > 2 else "ktanh_bf16"
n_launch = int(sys.argv[3]) if len(sys.argv) > 3 else 64
cfg = WL.CONFIGS[key]
step_bytes = (3 if op == "kgelu_swish_bf16" else 2) * cfg.numel * cfg.elem_bytes
sets = 1 if step_bytes >= 2 * L2_BYTES else max(2, math.ceil(4 * L2_BYTES / step_bytes))
xs = [WL.make_input(cfg, device="cuda", seed=cfg.seed + 1000 * k) for k in range(sets)]
ys = [torch.empty_like(xs[0]) for _ in range(sets)]
if op == "lstm":
    fn = lambda x, y: kt.klstm_gates_bf16(x, WL.LSTM_HIDDEN, 2, out=y)
elif op == "kgelu_swish_bf16":
    y2s = {id(y): torch.empty_like(y) for y in ys}
    fn = lambda x, y: kt.kgelu_swish_bf16(x, out_gelu=y, out_swish=y2s[id(y)])
else:
    fn = lambda x, y, f=getattr(kt, op): f(x, out=y)
for i in range(3 * sets):
    fn(xs[i % sets], ys[i % sets])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(n_launch):
    fn(xs[i % sets], ys[i % sets])
torch.cuda.cudart().cudaProfilerStop()
torch.cuda.synchronize()
print(f"range of {n_launch} launches x {step_bytes} algorithmic bytes ({key} {op}, {sets} sets)",
      flush=True)
