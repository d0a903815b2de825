"""Dev tool: kt_apply_host per-step time on pinned host buffers for several
sizes, zero-copy kernel vs the copy-engine pipeline (run with
KT_HOST_ZEROCOPY=0 / 1).  Prints ms/step, Gelem/s and PCIe GB/s (in + out)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt

mode = os.environ.get("KT_HOST_ZEROCOPY", "1")
work = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for dt, logs in ((torch.bfloat16, (20, 22, 24, 26)), (torch.float32, (24, 26))):
    for lg in logs:
        n = 1 << lg
        x = (torch.randn(n) * 2).to(dt).pin_memory()
        y = torch.empty_like(x).pin_memory()
        for _ in range(3):
            kt.apply_host("tanh", x, y, work)
        torch.cuda.synchronize()
        reps = max(3, min(50, (1 << 27) // n))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            kt.apply_host("tanh", x, y, work)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        gb = 2 * n * x.element_size() / ms / 1e6
        print(f"zc={mode} {str(dt):15s} n=2^{lg}: {ms:.4f} ms/step {n / ms / 1e6:8.2f} Gelem/s  PCIe {gb:6.1f} GB/s", flush=True)
