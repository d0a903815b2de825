"""A/B of library builds on bench.py's LSTM GEMM line (dev tool): the gate
GEMM [6400,1024] x [4096,1024]^T with fused gates, with the fused cell, and
unfused.  KT_LIB selects the build.

    python tools/lstm_gemm_ab.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_1909_07729_b200 as kt

dev = torch.device("cuda", 0)
r = bench.lstm_gemm_line(kt, 20, 3, 1, dev, 0)
r.pop("note", None)
r["lib"] = os.environ.get("KT_LIB", "in-tree")
print(json.dumps(r), flush=True)
