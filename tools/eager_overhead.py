"""Host overhead per eager library call (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt
x = torch.randn(1 << 16, device="cuda").to(torch.bfloat16)
y = torch.empty_like(x)
for _ in range(100): kt.ktanh_bf16(x, out=y)
torch.cuda.synchronize()
N = 20000
t0 = time.perf_counter()
for _ in range(N): kt.ktanh_bf16(x, out=y)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"python binding: {(t1 - t0) / N * 1e6:.2f} us/call (host)")
lut = kt.paper_lut().handle
s = torch.cuda.current_stream().cuda_stream
xp, yp = x.data_ptr(), y.data_ptr()
t0 = time.perf_counter()
for _ in range(N): kt._lib.ktanh_bf16(xp, yp, x.numel(), lut, s)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"raw ctypes C-ABI: {(t1 - t0) / N * 1e6:.2f} us/call (host)")
