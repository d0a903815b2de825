"""e2e host-path sweep (dev tool): pinned H2D/D2H bandwidth and kt_apply_host
per-step time for several scratch sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt

n = 1 << 24
x = (torch.randn(n) * 2).to(torch.bfloat16).pin_memory()
y = torch.empty_like(x).pin_memory()
d = torch.empty_like(x, device="cuda")
s = torch.cuda.current_stream()

def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

b = n * 2
print(f"H2D pinned 32MiB: {b / t(lambda: d.copy_(x, non_blocking=True)) / 1e6:.1f} GB/s")
print(f"D2H pinned 32MiB: {b / t(lambda: y.copy_(d, non_blocking=True)) / 1e6:.1f} GB/s")
for mb in (8, 16, 32, 64, 128, 256):
    work = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    ms = t(lambda: kt.apply_host("tanh", x, y, work))
    print(f"apply_host work={mb:4d} MiB: {ms:.4f} ms/step  {n / ms / 1e6:.2f} Gelem/s")

# bidirectional: H2D on one stream, D2H on another, concurrently
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty_like(d)
def bidir():
    with torch.cuda.stream(s1):
        d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(d2, non_blocking=True)
    s.wait_stream(s1); s.wait_stream(s2)
ms = t(bidir)
print(f"bidirectional 32MiB each way: {ms:.4f} ms  ({2 * b / ms / 1e6:.1f} GB/s total)")
for nch in (1, 2, 4, 8, 16):
    c = n // nch
    def chunked():
        for k in range(nch):
            with torch.cuda.stream(s1):
                d[k*c:(k+1)*c].copy_(x[k*c:(k+1)*c], non_blocking=True)
    print(f"H2D in {nch} chunks: {b / t(chunked) / 1e6:.1f} GB/s")
