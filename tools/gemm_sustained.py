"""Sustained FFN-shape GEMM (+K-GELU) timing: M=65536 N=16384 K=4096, `reps`
back-to-back launches per measurement (power-capped steady state).  Dev tool.
python tools/gemm_sustained.py [reps=40] [epi=gelu]"""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1909_07729_b200 as kt
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
epi = sys.argv[2] if len(sys.argv) > 2 else "gelu"
epi = None if epi == "none" else epi
M, N, K = 65536, 16384, 4096
A = (torch.randn(M, K, device="cuda") ).to(torch.bfloat16)
B = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    kt.kgemm_bf16(A, B, epilogue=epi, out=C)
torch.cuda.synchronize()
for trial in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        kt.kgemm_bf16(A, B, epilogue=epi, out=C)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    print(f"KT_GEMM_2CTA={os.environ.get('KT_GEMM_2CTA', 'default')} epi={epi}: {ms:.3f} ms "
          f"{2 * M * N * K / ms / 1e9:.0f} TF/s  (after: {clk})", flush=True)
