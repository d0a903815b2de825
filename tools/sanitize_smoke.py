"""Small calls of every library entry point, for compute-sanitizer (dev tool):
ragged sizes, unaligned heads/tails, mismatched alignment, in place, LSTM
gates and cell (vector and element paths; KT_CELL_KERNEL=1 for the staged
ring), backward, GEMM + epilogue, host pipeline, and inputs with x/2 ties
(the K-Swish / K-GELU tie screen and its out-of-line fix-up).

  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_smoke.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt

dev = "cuda"
for n in (1, 17, 1000, 4099):
    for off in (0, 1, 3):
        for dt, sfx in ((torch.bfloat16, "bf16"), (torch.float32, "f32")):
            base = (torch.randn(n + 8, device=dev) * 3).to(dt)
            x = base[off:off + n]
            out = torch.empty(n + 8, device=dev, dtype=dt)
            for op in ("tanh", "sigmoid", "swish", "gelu"):
                getattr(kt, f"k{op}_{sfx}")(x, out=out[off:off + n])        # same offset
                getattr(kt, f"k{op}_{sfx}")(x, out=out[(off + 1) % 4:(off + 1) % 4 + n])  # mismatched
                getattr(kt, f"k{op}_bwd_{sfx}")(x, x.clone(), out=out[off:off + n])
            z = x.clone()
            kt.ktanh_bf16(z, out=z) if sfx == "bf16" else kt.ktanh_f32(z, out=z)
ties = torch.tensor([w | s for w in range(1, 0x100, 2) for s in (0, 0x8000)], dtype=torch.int32)
for n in (4096, 70000):
    xb = (torch.randn(n, device=dev) * 2).to(torch.bfloat16)
    xi = xb.view(torch.int16)
    xi[torch.arange(0, n, 61, device=dev)[:ties.numel()]] = ties[: len(range(0, n, 61))].to(torch.int16).to(dev)
    for op in ("swish", "gelu"):
        getattr(kt, f"k{op}_bf16")(xb)
    kt.kgelu_swish_bf16(xb)
for rows, H in ((3, 16), (5, 10), (2, 1024), (7, 256), (40, 1024)):
    g = (torch.randn(rows, 4 * H, device=dev) * 1.5).to(torch.bfloat16)
    kt.klstm_gates_bf16(g, H, 2)
    c = torch.randn(rows, H, device=dev)
    kt.klstm_cell_bf16(g, c, H)
A = torch.randn(128, 128, device=dev).to(torch.bfloat16)
B = torch.randn(256, 128, device=dev).to(torch.bfloat16)
for epi in (None, "tanh", "gelu"):
    kt.kgemm_bf16(A, B, epilogue=epi)
xh = (torch.randn(100003) * 2).to(torch.bfloat16).pin_memory()
yh = torch.empty_like(xh).pin_memory()
work = torch.empty(1 << 22, dtype=torch.uint8, device=dev)
kt.apply_host("gelu", xh, yh, work)
torch.cuda.synchronize()
print("sanitize smoke ok, launches:", kt.launch_count())
