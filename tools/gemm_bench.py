"""tcgen05 GEMM (+K-GELU epilogue) vs torch.matmul (cuBLAS) and the unfused
pair (dev tool).  FFN-like shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt

def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for (M, N, K) in [(8192, 8192, 4096), (16384, 16384, 4096), (8192, 16384, 2048), (65536, 4096, 1024)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    ms_ours = t(lambda: kt.kgemm_bf16(A, B, out=C))
    ms_fused = t(lambda: kt.kgemm_bf16(A, B, epilogue="gelu", out=C))
    ms_cublas = t(lambda: torch.matmul(A, B.t(), out=C))
    ms_unfused = t(lambda: (torch.matmul(A, B.t(), out=C), kt.kgelu_bf16(C, out=C)))
    print(f"M={M} N={N} K={K}: tcgen05 {fl/ms_ours/1e9:.0f} TF/s ({ms_ours:.3f} ms) | +K-GELU fused "
          f"{ms_fused:.3f} ms | cuBLAS {fl/ms_cublas/1e9:.0f} TF/s ({ms_cublas:.3f} ms) | cuBLAS + kgelu "
          f"{ms_unfused:.3f} ms", flush=True)
