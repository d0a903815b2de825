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
if epi == "cell":            # N = 4 * hidden: GEMM + fused LSTM cell
    c = torch.randn(M, N // 4, device="cuda")
    for _ in range(4):
        kt.kgemm_lstm_cell_bf16(A, B, c, N // 4)
else:
  for _ in range(4):
    kt.kgemm_bf16(A, B, epilogue=epi, out=C)
torch.cuda.synchronize()
print("ok", flush=True)
