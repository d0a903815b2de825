"""One GEMM shape, a few launches (for ncu -k regex:k_gemm -s 2 -c 1).
python tools/gemm_one.py M N K [epilogue]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt
M, N, K = (int(v) for v in sys.argv[1:4])
epi = sys.argv[4] if len(sys.argv) > 4 and sys.argv[4] != "none" else None
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    kt.kgemm_bf16(A, B, epilogue=epi, out=C)
torch.cuda.synchronize()
print("ok", flush=True)
