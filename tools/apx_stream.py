"""Streaming throughput of K-TanH vs the Table 2 comparators on one B200.

python tools/apx_stream.py [log2_n=28] [fmt=bf16]

Each launch reads n elements and writes n (inputs > L2), CUDA events on the
current stream, best and median of 20 after 3 warm-ups.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1909_07729_b200 as kt  # noqa: E402

CMP = [("ktanh", 0, 0), ("sfu", 0, 0), ("libm", 0, 0), ("pade", 3, 2), ("pade", 7, 8),
       ("minimax", 2, 0), ("minimax", 3, 0), ("taylor", 2, 0), ("taylor", 3, 0)]


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    fmt = sys.argv[2] if len(sys.argv) > 2 else "bf16"
    n = 1 << lg
    dt = torch.bfloat16 if fmt == "bf16" else torch.float32
    es = 2 if fmt == "bf16" else 4
    x = (torch.randn(n, device="cuda") * 2).to(dt)
    y = torch.empty_like(x)
    for name, p, q in CMP:
        if name == "ktanh":
            f = (lambda: kt.ktanh_bf16(x, out=y)) if fmt == "bf16" else (lambda: kt.ktanh_f32(x, out=y))
        else:
            A = kt.Apx(name, p, q)
            call = kt.kt_apx_tanh_bf16 if fmt == "bf16" else kt.kt_apx_tanh_f32
            f = (lambda A=A, call=call: call(x, A, out=y))
        for _ in range(3):
            f()
        ts = []
        for _ in range(20):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e-3)
        ts.sort()
        best, med = ts[0], ts[len(ts) // 2]
        print(f"{name:8s} {p}/{q} {fmt}: best {best*1e6:8.1f} us  {n/best/1e9:8.1f} Gelem/s  "
              f"{2*es*n/best/1e9:7.1f} GB/s   median {2*es*n/med/1e9:7.1f} GB/s")


if __name__ == "__main__":
    main()
