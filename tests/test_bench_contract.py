"""bench.py output contract (the driver parses these JSON lines): the
reference arm runs here on CPU; the main arm needs the GPU."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"], 600)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["unit"] == "Gelem/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["warmup"] >= 3 and d["config"]["workload"] == "c5_ffn_2p30" and d["dtype"] == "bf16"
    assert d["config"]["elements_per_gpu"] == 1 << 30 and d["config"]["call"] == "kgelu_bf16"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "Gelem/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_main_arm_contract():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--steps", "20", "--warmup", "3", "--no-extra", "--no-cpu"], 900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["data"] == "synthetic" and d["dtype"] == "bf16" and d["vs_baseline"] is None
    assert d["config"]["workload"] == "c5_ffn_2p30" and "larger than L2" in d["config"]["l2"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-3 and rf["traffic"] > 0
    assert rf["algorithmic_bytes_per_launch"] == 4 << 30
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 2 << 30
    assert d["gpu_launches"] == 20
    c = d["clocks"]
    assert c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    assert d["per_rank"] == [{"rank": 0, "device": 0, "ms_per_step": d["per_rank"][0]["ms_per_step"],
                              "checked": 65538, "mismatches": 0}] or d["cpu_baseline"] is None


def test_reference_arm_same_config_as_main_arm():
    """Both arms print the identical `config` object (the driver compares them)."""
    sys.path.insert(0, ROOT)
    import bench
    ref = _run(["--impl", "reference", "--steps", "1", "--warmup", "3"], 600)
    assert ref["config"] == bench.head_config("c5_ffn_2p30", "kgelu_bf16", 1)


def test_multirank_path_under_torchrun_stub():
    """bench.py's N > 1 path end to end on CPU (gloo, world size 2, --stub):
    device selection (local_rank % devices), barriers, per-rank windows, the
    max over ranks, the per-rank check and one JSON line from rank 0 only."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "5", "--warmup", "3", "--stub"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["stub"] is True and d["n_gpus"] == 2 and d["steps"] == 5 and d["warmup"] == 3
    pr = d["per_rank"]
    assert [p["rank"] for p in pr] == [0, 1] and [p["device"] for p in pr] == [0, 1]
    assert all(p["mismatches"] == 0 and p["checked"] == (1 << 16) + 2 for p in pr)
    # value = all ranks' elements / the slowest rank's (median) window
    assert max(p["ms_per_step"] for p in pr) <= d["ms_per_step"] * 1.5 + 1e-3
    assert abs(d["value"] - 2 * (1 << 16) / (d["ms_per_step"] / 1e3) / 1e9) <= 1e-3 * d["value"] + 1e-3


def test_traffic_is_read_per_workload_from_committed_captures():
    """roofline.traffic comes from the committed range-replay capture of the
    bench line's OWN workload and call (the c2 capture must not
    stand in for another config); every capture is within 2% of the
    algorithmic bytes per launch."""
    sys.path.insert(0, ROOT)
    import bench
    alg = {("c5_ffn_2p30", "kgelu_bf16"): 4 << 30, ("c5_ffn_2p30", "kswish_bf16"): 4 << 30,
           ("c5_ffn_2p30", "kgelu_swish_bf16"): 6 << 30, ("c3_f32_2p28", "ktanh_f32"): 8 << 28,
           ("c2_bf16_2p24", "ktanh_bf16"): 4 << 24, ("c4_lstm_gates", "lstm"): 4 * 128 * 50 * 4096}
    for (key, op), a in alg.items():
        t, src = bench.load_traffic(key, op)
        assert t is not None and f"_{key}_{op}_r" in src, (key, op, src)
        assert 0.98 * a <= t <= 1.02 * a, (key, op, t, a)
    assert bench.load_traffic("c5_ffn_2p30", "no_such_call") == (None, None)


def test_bench_mismatch_rule():
    """bench.py's per-rank oracle check compares bit-exactly, NaN by class
    except for K-TanH (which passes NaN bits through), +-0 by value for the
    derived ops only."""
    import numpy as np
    sys.path.insert(0, ROOT)
    import bench
    w = np.array([0x7FC0, 0x8000, 0x3F80], np.uint16)
    g = np.array([0x7FC1, 0x0000, 0x3F80], np.uint16)
    assert bench.mismatches(g, w, "gelu", True) == 0
    assert bench.mismatches(g, w, "sigmoid", True) == 1        # -0 vs +0 counts outside swish/gelu
    assert bench.mismatches(g, w, "tanh", True) == 2           # NaN payload and zero sign both count
    wf = np.array([0x7FC00000, 0x80000000], np.uint32)
    gf = np.array([0xFFC00000, 0x00000000], np.uint32)
    assert bench.mismatches(gf, wf, "swish", False) == 0
    assert bench.mismatches(gf + np.uint32(1), wf, "swish", False) == 1   # 0x00000001 is not zero
