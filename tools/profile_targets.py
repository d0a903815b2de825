"""Run each library call on its BASELINE.json config a few times (for ncu -k/-s
selection of one warm launch per kernel).  Dev/profiling tool.

    python tools/profile_targets.py [op ...]     ops: tanh_bf16 tanh_f32 gelu swish sigmoid lstm
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1909_07729_b200 as kt
import workloads as WL

TARGETS = {
    "tanh_bf16": ("c2_bf16_2p24", lambda x, y: kt.ktanh_bf16(x, out=y)),
    "tanh_f32": ("c3_f32_2p28", lambda x, y: kt.ktanh_f32(x, out=y)),
    "gelu": ("c5_ffn_2p30", lambda x, y: kt.kgelu_bf16(x, out=y)),
    "swish": ("c5_ffn_2p30", lambda x, y: kt.kswish_bf16(x, out=y)),
    "sigmoid": ("c2_bf16_2p24", lambda x, y: kt.ksigmoid_bf16(x, out=y)),
    "lstm": ("c4_lstm_gates", lambda x, y: kt.klstm_gates_bf16(x, WL.LSTM_HIDDEN, 2, out=y)),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(TARGETS)
    for name in names:
        key, fn = TARGETS[name]
        x = WL.make_input(key, device="cuda")
        y = torch.empty_like(x)
        for _ in range(4):          # 3 warm launches, then the one ncu captures (-s 3 -c 1)
            fn(x, y)
        torch.cuda.synchronize()
        print(name, "ok", flush=True)
        del x, y
        torch.cuda.empty_cache()
