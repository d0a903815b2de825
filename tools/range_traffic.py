"""Steady-state DRAM traffic per config-2 step, measured over a RANGE of
back-to-back launches (ncu --replay-mode range between cudaProfilerStart /
Stop), so the write-back of earlier launches' dirty output lines is counted
(a single-kernel capture misses it).  Dev tool:

  ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      python tools/range_traffic.py [launches=64]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt
import workloads as WL

n_launch = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sets = 8
xs = [WL.make_input("c2_bf16_2p24", device="cuda", seed=2 + 1000 * k) for k in range(sets)]
ys = [torch.empty_like(xs[0]) for _ in range(sets)]
for i in range(3 * sets):
    kt.ktanh_bf16(xs[i % sets], out=ys[i % sets])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(n_launch):
    kt.ktanh_bf16(xs[i % sets], out=ys[i % sets])
torch.cuda.cudart().cudaProfilerStop()
torch.cuda.synchronize()
print(f"range of {n_launch} launches x {4 * xs[0].numel()} algorithmic bytes", flush=True)
