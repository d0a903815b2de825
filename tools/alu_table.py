"""Table 2 analogue on B200: SM cycles per element, register-resident.

python tools/alu_table.py [iters=256]

For K-TanH and every comparator, kt_alu_probe runs one wave of CTAs that
apply the map to register-held inputs (the config-2 distribution, N(0, 2^2)
rounded to BF16; F32 uses the same values widened) with no memory traffic.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1909_07729_b200 as kt  # noqa: E402

CMP = [("ktanh", 0, 0), ("sfu", 0, 0), ("libm", 0, 0), ("pade", 3, 2), ("pade", 7, 8),
       ("minimax", 2, 0), ("minimax", 3, 0), ("taylor", 2, 0), ("taylor", 3, 0)]


def sample(fmt, seed=2):
    g = torch.Generator().manual_seed(seed)
    v = (torch.randn(8192, generator=g) * 2).to(torch.bfloat16)
    if fmt == "bf16":
        return v.view(torch.int16).numpy().view(np.uint16).view(np.uint32)[:4096].copy()
    return v[:4096].float().numpy().view(np.uint32).copy()


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    out = []
    for fmt in ("bf16", "f32"):
        s = sample(fmt)
        for name, p, q in CMP:
            if name == "ktanh":
                net, gross = kt.alu_probe(fmt, s, lut=kt.paper_lut(), iters=iters)
            else:
                net, gross = kt.alu_probe(fmt, s, apx=kt.Apx(name, p, q), iters=iters)
            row = {"map": name if name in ("ktanh", "sfu", "libm") else f"{name}_{p}_{q}",
                   "fmt": fmt, "cycles_per_elem_per_sm_net": round(net, 4),
                   "cycles_per_elem_per_sm_gross": round(gross, 4),
                   "elems_per_clk_per_sm_net": round(1 / net, 3) if net > 0 else None}
            out.append(row)
            print(f"{row['map']:14s} {fmt:5s} net {net:7.4f}  gross {gross:7.4f} cyc/elem/SM"
                  f"   ({1/net if net > 0 else float('inf'):6.2f} elem/clk/SM)")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
