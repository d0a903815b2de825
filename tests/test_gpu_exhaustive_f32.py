"""Exhaustive FP32 parity ("all 2^32 patterns streamed in 2^28
chunks through ktanh_f32 and ksigmoid_f32, bytewise vs oracle") and the
branch-freedom throughput check (§4: identical throughput on all-bypass,
all-saturate, all-table and N(0, sigma) inputs).

The oracle runs on every host core (ctypes releases the GIL), one slice per
thread; the GPU side streams each 2^28 chunk through the C ABI.
"""
import os
import statistics
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle as O
from _cmp import assert_bitexact

pytestmark = pytest.mark.gpu

CHUNK = 1 << 28


@pytest.fixture(scope="module")
def kt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_07729_b200 as kt
    return kt


def _oracle_parallel(op, bits, pool, nthreads, lut=None):
    out = np.empty_like(bits)
    step = (bits.size + nthreads - 1) // nthreads

    def work(k):
        s = k * step
        out[s:s + step] = O.map_f32(op, bits[s:s + step], lut)
    list(pool.map(work, range(nthreads)))
    return out


@pytest.mark.slow
@pytest.mark.parametrize("op,call,nan_by_class", [
    ("tanh", "ktanh_f32", False),
    ("sigmoid", "ksigmoid_f32", True),
    ("tanh_via_bf16", "ktanh_f32_via_bf16", True),
    ("tanh", "ktanh_f32:p23", False)])
def test_exhaustive_f32(kt, op, call, nan_by_class):
    """Every one of the 2^32 F32 bit patterns, bit-exact (NaN by class where
    the GPU's arithmetic canonicalises the payload).  ":p23": with the F32
    table re-optimised at p = 23 (kt_lut_create_f32, NEXT-3)."""
    lut = hlut = None
    if call.endswith(":p23"):
        call = call[:-4]
        lut = O.build_lut_sp(3, 23)[0]
        hlut = kt.Lut.from_tables_f32(lut.E, lut.r, lut.b)
    fn = getattr(kt, call)
    nthreads = max(1, os.cpu_count() or 1)
    x = torch.empty(CHUNK, dtype=torch.float32, device="cuda")
    y = torch.empty_like(x)
    with ThreadPoolExecutor(nthreads) as pool:
        for c in range(1 << 32 >> 28):
            bits = np.arange(c * CHUNK, (c + 1) * CHUNK, dtype=np.uint64).astype(np.uint32)
            x.copy_(torch.from_numpy(bits.view(np.int32)).view(torch.float32))
            fn(x, out=y, lut=hlut)
            got = y.view(torch.int32).cpu().numpy().view(np.uint32)
            want = _oracle_parallel(op, bits, pool, nthreads, lut)
            assert_bitexact(got, want, 32, nan_by_class=nan_by_class, ctx=f"{op} chunk {c}")


def _stratified_f32(c, nchunks, rng):
    """Chunk c of the stratified F32 set (~2^28 patterns in total): every
    pattern with biased exponent 0 or 1 (subnormals and the smallest normals,
    where x/2 can be an F32 tie, reading R-DERIVED), and for each of the 2^20
    (sign, exponent, top-11-mantissa-bit) classes the low 12 bits 0x000, 0xFFF
    and 222 seeded random values."""
    cls = np.arange(c * (1 << 20) // nchunks, (c + 1) * (1 << 20) // nchunks, dtype=np.uint64)
    low = rng.integers(0, 1 << 12, (cls.size, 224), dtype=np.uint64)
    low[:, 0], low[:, 1] = 0, 0xFFF
    bits = ((cls[:, None] << 12) | low).reshape(-1)
    tiny = np.arange(c * (1 << 24) // nchunks, (c + 1) * (1 << 24) // nchunks, dtype=np.uint64)
    tiny = np.concatenate([tiny, tiny | (1 << 31)])      # |x| < 2^-125, both signs
    return np.concatenate([bits, tiny]).astype(np.uint32)


def _derived_sweep(kt, op, chunks):
    from _cmp import assert_bitexact
    fn = getattr(kt, f"k{op}_f32")
    nthreads = max(1, os.cpu_count() or 1)
    total = 0
    with ThreadPoolExecutor(nthreads) as pool:
        for bits in chunks:
            x = torch.from_numpy(bits.view(np.int32)).cuda().view(torch.float32)
            got = fn(x).view(torch.int32).cpu().numpy().view(np.uint32)
            want = _oracle_parallel(op, bits, pool, nthreads)
            assert_bitexact(got, want, 32, nan_by_class=True, zero_by_value=True, ctx=f"{op} f32")
            total += bits.size
    return total


@pytest.mark.parametrize("op", ["swish", "gelu"])
def test_f32_derived_stratified(kt, op):
    """K-Swish / K-GELU on F32 (R-DERIVED): bit-exact against
    the oracle (NaN by class, +-0 by value; the north_star allows 2 ulp) on a
    stratified 2^28-pattern set covering every (sign, exponent, top-11-bit)
    class plus ALL inputs below 2^-125.  Part of -m gpu (~1 min per op); the
    full 2^32 sweep is tools/f32_derived_sweep.py (profiles/f32_derived_sweep_r02.txt)."""
    rng = np.random.default_rng(1234)
    n = _derived_sweep(kt, op, (_stratified_f32(c, 16, rng) for c in range(16)))
    print(f"k{op}_f32: {n} stratified F32 patterns bit-exact")


def _time(fn, reps=30):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def test_branch_free_throughput(kt):
    """Alg. 1's three regions cost the same: the kernel is branch-free, so
    throughput on all-bypass, all-saturate, all-table and N(0, 2^2) inputs
    agrees within 5% (HBM-bound, 2^27 BF16 elements > L2)."""
    n = 1 << 27
    g = torch.Generator(device="cuda").manual_seed(9)
    u = torch.rand(n, device="cuda", generator=g)
    inputs = {
        "bypass": (u * 0.49 - 0.245).to(torch.bfloat16),          # |x| < 0.25
        "saturate": (u * 100 + 3.8).to(torch.bfloat16),           # x > 3.75
        "table": (u * 3.4 + 0.3).to(torch.bfloat16),              # 0.3 .. 3.7
        "normal": (torch.randn(n, device="cuda", generator=g) * 2).to(torch.bfloat16),
    }
    y = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    ms = {k: _time(lambda v=v: kt.ktanh_bf16(v, out=y)) for k, v in inputs.items()}
    lo, hi = min(ms.values()), max(ms.values())
    print("ms per 2^27 launch by region mix:", {k: round(v, 4) for k, v in ms.items()})
    assert hi / lo <= 1.05, ms
