"""bench.py's LSTM GEMM line alone (graph-replayed windows), for A/B of
libktanh.so builds via KT_LIB.  python tools/lstm_gemm_ab.py [K=200]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1909_07729_b200 as kt  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 200
r = bench.lstm_gemm_line(kt, K, 5, 1, torch.device("cuda", 0), 0)
print(json.dumps({"lib": os.environ.get("KT_LIB", "in-tree"), "pair": os.environ.get("KT_GEMM_2CTA", "auto"),
                  **{k: v for k, v in r.items() if k != "note"}}))
