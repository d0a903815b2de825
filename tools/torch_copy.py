"""Reference copy rate with torch on this box (dev tool): b.copy_(a) over 1 Gi bf16."""
import torch
a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda").normal_()
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(f"torch copy_ 1Gi bf16: {2 * a.numel() * 2 / (best / 1e3) / 1e9:.1f} GB/s (best of 10)")
