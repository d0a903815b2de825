"""K-Swish / K-GELU on every one of the 2^32 F32 bit patterns against the
oracle (run on every host core), bit-exact with NaN by class and +-0 by value
(reading R-DERIVED / A21).  ~6 min per op on a 16-core GPU box, so it is a
tool run once per kernel change rather than part of `pytest -m gpu` (which
runs the stratified 2^28 subset, tests/test_gpu_exhaustive_f32.py).

    python tools/f32_derived_sweep.py [swish gelu]   -> one line per op; exit 1 on a mismatch
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch

from test_gpu_exhaustive_f32 import CHUNK, _derived_sweep

import paper_1909_07729_b200 as kt

bad = 0
for op in sys.argv[1:] or ["swish", "gelu"]:
    try:
        n = _derived_sweep(kt, op, (np.arange(c * CHUNK, (c + 1) * CHUNK, dtype=np.uint64).astype(np.uint32)
                                    for c in range(1 << 32 >> 28)))
        print(f"k{op}_f32: all {n} F32 patterns bit-exact vs the oracle (NaN by class, +-0 by value)",
              flush=True)
    except AssertionError as e:
        bad += 1
        print(f"k{op}_f32: MISMATCH {str(e)[:500]}", flush=True)
sys.exit(1 if bad else 0)
