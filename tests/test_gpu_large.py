"""Maximum-size edge cases: element counts past 2^31 and 2^32 (every 32-bit
index overflows there), misaligned starts, ragged tails, outputs past 2^32
elements for the GEMM.  Outputs are checked on samples the oracle computes one
by one: the first and last elements, +-64 around 2^31 and 2^32, and 2^16
random positions.  Memory: at most ~72 GiB at a time (B200: 180 GB)."""
import gc

import numpy as np
import pytest
import torch

import oracle as O
from _cmp import assert_bitexact, assert_ulp
from test_gpu_bwd import check_bwd

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def kt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_07729_b200 as kt
    return kt


@pytest.fixture(autouse=True)
def _free():
    yield
    gc.collect()
    torch.cuda.empty_cache()


def sample_idx(n, seed=0):
    edges = [np.arange(0, 64), np.arange(n - 64, n)]
    for b in (1 << 31, 1 << 32):
        if b + 64 < n:
            edges.append(np.arange(b - 64, b + 64))
    rnd = np.random.default_rng(seed).integers(0, n, 1 << 16)
    return np.unique(np.concatenate(edges + [rnd])).astype(np.int64)


def take(t, idx):
    return t.reshape(-1)[torch.from_numpy(idx).to(t.device)]


def bits16(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def bits32(t):
    return t.contiguous().view(torch.int32).cpu().numpy().view(np.uint32)


def rand_bf16(n, seed, scale=2.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(n, device="cuda", dtype=torch.bfloat16, generator=g).mul_(scale)


def test_ktanh_bf16_past_2p32_misaligned(kt):
    n = (1 << 32) + (1 << 20) + 7
    base = rand_bf16(n + 1, 1)
    x = base[1:]                                   # 2-byte offset: scalar head + vector body + tail
    y = kt.ktanh_bf16(x)
    idx = sample_idx(n)
    assert_bitexact(bits16(take(y, idx)), O.map_bf16("tanh", bits16(take(x, idx))), 16,
                    ctx="ktanh_bf16 n > 2^32")


def test_kgelu_bf16_past_2p32_misaligned(kt):
    """K-GELU BF16 takes its own launch shape (4 vectors per lane, 128-thread
    CTAs) and the tie screen: past 2^32 elements, from an odd element offset."""
    n = (1 << 32) + (1 << 20) + 5
    base = rand_bf16(n + 3, 11)
    x = base[3:]
    y = kt.kgelu_bf16(x)
    idx = sample_idx(n, seed=11)
    assert_bitexact(bits16(take(y, idx)), O.map_bf16("gelu", bits16(take(x, idx))), 16,
                    nan_by_class=True, zero_by_value=True, ctx="kgelu_bf16 n > 2^32")


def test_ktanh_f32_via_bf16_past_2p31(kt):
    """The F32-through-BF16 map (128-thread CTAs, 4 vectors per lane) past 2^31."""
    n = (1 << 31) + 13
    g = torch.Generator(device="cuda").manual_seed(12)
    x = torch.randn(n, device="cuda", generator=g).mul_(3)
    y = kt.ktanh_f32_via_bf16(x)
    idx = sample_idx(n, seed=12)
    assert_bitexact(bits32(take(y, idx)), O.map_f32("tanh_via_bf16", bits32(take(x, idx))), 32,
                    nan_by_class=True, ctx="ktanh_f32_via_bf16 n > 2^31")


def test_ksigmoid_f32_past_2p31(kt):
    n = (1 << 31) + 9
    g = torch.Generator(device="cuda").manual_seed(2)
    x = torch.randn(n, device="cuda", generator=g).mul_(3)
    y = kt.ksigmoid_f32(x)
    idx = sample_idx(n)
    assert_bitexact(bits32(take(y, idx)), O.map_f32("sigmoid", bits32(take(x, idx))), 32,
                    nan_by_class=True, ctx="ksigmoid_f32 n > 2^31")


def test_kgelu_swish_bf16_past_2p32(kt):
    n = (1 << 32) + 5
    x = rand_bf16(n, 3)
    g, s = kt.kgelu_swish_bf16(x)
    idx = sample_idx(n)
    xb = bits16(take(x, idx))
    assert_bitexact(bits16(take(g, idx)), O.map_bf16("gelu", xb), 16, nan_by_class=True,
                    zero_by_value=True, ctx="dual gelu n > 2^32")
    assert_bitexact(bits16(take(s, idx)), O.map_bf16("swish", xb), 16, nan_by_class=True,
                    zero_by_value=True, ctx="dual swish n > 2^32")


def test_kgelu_bwd_bf16_past_2p32(kt):
    n = (1 << 32) + 3
    a, dy = rand_bf16(n, 4), rand_bf16(n, 5, 1.0)
    dx = kt.kgelu_bwd_bf16(a, dy)
    idx = sample_idx(n)
    ab, db = bits16(take(a, idx)), bits16(take(dy, idx))
    check_bwd("gelu", 16, ab, db, bits16(take(dx, idx)), O.bwd_bf16("gelu", ab, db))


def test_klstm_gates_past_2p32(kt):
    H = 1024
    rows = (1 << 20) + 3                           # rows * 4H = 2^32 + 12288 elements
    x = rand_bf16(rows * 4 * H, 6).view(rows, 4 * H)
    y = kt.klstm_gates_bf16(x, H, 2)
    n = rows * 4 * H
    idx = sample_idx(n)
    xb, yb = bits16(take(x, idx)), bits16(take(y, idx))
    q = (idx % (4 * H)) // H
    for quarter, op in ((2, "tanh"), (0, "sigmoid")):
        m = q == quarter if quarter == 2 else q != 2
        assert_bitexact(yb[m], O.map_bf16(op, xb[m]), 16, nan_by_class=True, ctx=f"lstm {op} n > 2^32")


def test_klstm_cell_past_2p32_cells(kt):
    H = 1024
    rows = (1 << 22) + 1                           # rows * H = 2^32 + 1024 cells
    gates = rand_bf16(rows * 4 * H, 7).view(rows, 4 * H)
    g = torch.Generator(device="cuda").manual_seed(8)
    c = torch.randn(rows, H, device="cuda", generator=g)
    cn, hn = kt.klstm_cell_bf16(gates, c, H)
    cells = rows * H
    idx = sample_idx(cells)
    r, j = idx // H, idx % H
    gi = np.stack([bits16(take(gates, r * 4 * H + q * H + j)) for q in range(4)])   # [4, m]
    want_c, want_h = O.lstm_cell_bf16(np.ascontiguousarray(gi.T), bits32(take(c, idx)), 1)
    assert_bitexact(bits32(take(cn, idx)), want_c, 32, ctx="lstm cell c' past 2^32 cells")
    assert_bitexact(bits16(take(hn, idx)), want_h, 16, ctx="lstm cell h' past 2^32 cells")


def test_kgemm_output_past_2p32(kt):
    """C = A B^T with M N = 2^32 + 2^24 outputs (CTA-pair kernel): sampled
    entries against the float64 dot product (bound of test_gemm_vs_float64)."""
    M, N, K = 65536 + 256, 65536, 64
    g = torch.Generator(device="cuda").manual_seed(9)
    A = torch.randn(M, K, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda", generator=g).mul_(0.5).to(torch.bfloat16)
    C = kt.kgemm_bf16(A, B)
    idx = sample_idx(M * N)
    r, cidx = idx // N, idx % N
    a = O.bf16_to_f64(bits16(A)).reshape(M, K)[r]
    b = O.bf16_to_f64(bits16(B)).reshape(N, K)[cidx]
    exact = (a * b).sum(axis=1)
    got = O.bf16_to_f64(bits16(take(C, idx)))
    bound = np.abs(exact) * 2.0 ** -8 + K * 2.0 ** -23 * (np.abs(a) * np.abs(b)).sum(axis=1) + 1e-30
    assert np.all(np.abs(got - exact) <= bound)
