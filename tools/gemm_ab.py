"""A/B timing of the tcgen05 GEMM family for whichever libktanh.so KT_LIB
names (dev tool: run it once per library, alternating, on the same box).
Prints one JSON line {case: ms}.

python tools/gemm_ab.py [reps=30]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1909_07729_b200 as kt  # noqa: E402


def t(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 5)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    torch.manual_seed(0)
    res = {"lib": os.environ.get("KT_LIB", "in-tree"), "pair": os.environ.get("KT_GEMM_2CTA", "auto")}
    for (M, N, K, epi) in [(16384, 16384, 4096, None), (65536, 4096, 1024, None),
                           (8192, 8192, 4096, "gelu"), (65536, 16384, 4096, "gelu")]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        r = reps if M * N * K < 2 ** 40 else max(4, reps // 4)
        res[f"{M}x{N}x{K}:{epi}"] = t(lambda: kt.kgemm_bf16(A, B, epilogue=epi, out=C), r)
        del A, B, C
    H, M = 1024, 6400
    A = (torch.randn(M, H, device="cuda")).to(torch.bfloat16)
    B = (torch.randn(4 * H, H, device="cuda") * 0.05).to(torch.bfloat16)
    G = torch.empty(M, 4 * H, device="cuda", dtype=torch.bfloat16)
    c = torch.randn(M, H, device="cuda")
    cn = torch.empty_like(c)
    hn = torch.empty(M, H, device="cuda", dtype=torch.bfloat16)
    res["lstm_gates"] = t(lambda: kt.kgemm_lstm_gates_bf16(A, B, H, 2, out=G), reps * 10)
    res["lstm_cell"] = t(lambda: kt.kgemm_lstm_cell_bf16(A, B, c, H, c_next=cn, h_next=hn), reps * 10)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
