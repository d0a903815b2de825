"""Time klstm_cell_bf16 on config 4 ([6400, 1024] cells) per launch variant
(KT_CELL_PERSIST is read once per process: run once per value)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt
import workloads as WL
H = WL.LSTM_HIDDEN
sets = 5
xs = [WL.make_input("c4_lstm_gates", device="cuda", seed=4 + 1000 * k) for k in range(sets)]
cs = [torch.randn(x.numel() // (4 * H), H, device="cuda") for x in xs]
cn = [torch.empty_like(c) for c in cs]
hn = [torch.empty(c.shape, dtype=torch.bfloat16, device="cuda") for c in cs]
for i in range(10):
    kt.klstm_cell_bf16(xs[i % sets], cs[i % sets], H, c_next=cn[i % sets], h_next=hn[i % sets])
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(20):
        kt.klstm_cell_bf16(xs[i % sets], cs[i % sets], H, c_next=cn[i % sets], h_next=hn[i % sets])
ts = []
for _ in range(50):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); g.replay(); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b) / 20)
m = statistics.median(ts)
cells = xs[0].numel() // 4
print(f"KT_LIB={os.environ.get('KT_LIB') or 'default'}: {m*1e3:.2f} us/launch, "
      f"{cells / m / 1e6:.1f} Gcell/s, {18 * cells / m / 1e6:.1f} GB/s")
