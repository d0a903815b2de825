"""GPU parity of the backward kernels (reading R-BWD) against the oracle.

Tolerance, derived from the kernels' fp32 evaluation (kt_device.cuh
bwd_f32 / bwd_factor2) against the oracle's one rounding of the exact
binary64 value, u = 2^-24:

    |dx - oracle| <= ulp_fmt(oracle) + c u |dy| S

  tanh     g = fma(-y, y, 1)              one rounding of g, one of dy g: c = 3, S = 1
  sigmoid  g = fma(-s, s, s)              the same:                           c = 3, S = 1
  swish    g = fma(x/4, RN(1 - t^2), RN((1 + t)/2))                           c = 4, S = 1 + |x|/4
  gelu     g = fma(RN(x/2 RN(1 - t^2)), RN(C3 RN(x^2) + C0), RN((1 + t)/2))   c = 8,
           S = 1 + 0.8 |x| (1 + 0.134 x^2)  (>= |(1+t)/2| + |x/2 (1 - t^2) u'(x)|)

(relative errors: 1 - t^2 and (1+t)/2 one rounding each, x/2 (1 - t^2) two,
u' = C3 x^2 + C0 three (C0, C3 themselves RN32 of their binary64 values), the
final fma one, dy g one: |g_hat - g| <= (c - 1) u S and |dy g_hat rounded -
dy g| <= c u |dy| S; the last rounding to the format costs the ulp term).
The c u |dy| S term only matters where g cancels ((1+t)/2 against the
negative x-term); elsewhere the bound is ~1 ulp.  Each check also returns
the largest measured fraction of the c u |dy| S allowance actually used,
printed by the tests.  NaN compared by class."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as WL
from _cmp import _isnan

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_07729_b200 as kt
    return kt


def u16(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def u32(t):
    return t.contiguous().view(torch.int32).cpu().numpy().view(np.uint32)


def _vals(bits, nbits):
    if nbits == 16:
        return O.bf16_to_f64(bits)
    return np.asarray(bits, np.uint32).view(np.float32).astype(np.float64)


BWD_C = {"tanh": 3, "sigmoid": 3, "swish": 4, "gelu": 8}


def _spacing(v, nbits):
    """ulp of the format at |v| (the upward spacing; min subnormal spacing at 0)."""
    a = np.abs(v).astype(np.float32)
    sp = np.spacing(a).astype(np.float64)
    if nbits == 16:
        sp = np.maximum(sp * 65536.0, 2.0 ** -133)
    return sp


def check_bwd(op, nbits, a, dy, got, want):
    """Assert the derived bound of the module docstring; return the largest
    fraction of the c u |dy| S allowance used (0 when within the ulp term)."""
    x = _vals(a, nbits)
    g = _vals(dy, nbits)
    with np.errstate(invalid="ignore", over="ignore"):
        if op in ("tanh", "sigmoid"):
            S = np.ones_like(x)
        elif op == "swish":
            S = 1 + np.abs(x) / 4
        else:
            S = 1 + np.abs(x) * 0.8 * (1 + 0.134 * x * x)
        gv, wv = _vals(got, nbits), _vals(want, nbits)
        allow = BWD_C[op] * 2.0 ** -24 * np.abs(g) * S
        excess = np.abs(gv - wv) - _spacing(wv, nbits)
        finite = np.isfinite(wv) & np.isfinite(gv)
        ok = np.where(finite, excess <= allow, got == want)
    nan = _isnan(got, nbits) & _isnan(want, nbits)
    bad = ~(ok | nan)
    assert not bad.any(), (op, nbits, int(bad.sum()), [hex(int(v)) for v in a[bad][:4]],
                           [hex(int(v)) for v in got[bad][:4]], [hex(int(v)) for v in want[bad][:4]])
    m = finite & ~nan & (allow > 0)
    with np.errstate(invalid="ignore", divide="ignore"):
        frac = np.where(m & (excess > 0), excess / np.where(m, allow, 1.0), 0.0)
    return float(frac.max()) if frac.size else 0.0


def _domain(op, a_vals):
    """tanh/sigmoid backward take the SAVED forward output: |y| <= 1, 0 <= s <= 1."""
    with np.errstate(invalid="ignore"):
        if op == "tanh":
            return np.abs(a_vals) <= 1
        if op == "sigmoid":
            return (a_vals >= 0) & (a_vals <= 1)
    return np.ones(a_vals.shape, bool)


@pytest.mark.parametrize("op", ["tanh", "sigmoid", "swish", "gelu"])
def test_bwd_bf16_all_patterns(kt, op):
    a = WL.make_input("c1_exhaustive_bf16", device="cuda")
    keep = torch.from_numpy(_domain(op, O.bf16_to_f64(u16(a)))).cuda()
    a = a[keep].contiguous()
    g = torch.Generator(device="cuda").manual_seed(17)
    dy = torch.randn(a.numel(), device="cuda", generator=g).to(torch.bfloat16)
    dx = getattr(kt, f"k{op}_bwd_bf16")(a, dy)
    want = O.bwd_bf16(op, u16(a), u16(dy))
    used = check_bwd(op, 16, u16(a), u16(dy), u16(dx), want)
    print(f"{op} bwd bf16: largest fraction of the derived c u |dy| S allowance used: {used:.3g}")


@pytest.mark.parametrize("op", ["tanh", "sigmoid", "swish", "gelu"])
def test_bwd_f32_patterns(kt, op):
    rng = np.random.default_rng(5)
    a_bits = np.concatenate([
        (np.arange(1 << 18, dtype=np.uint64) << 14).astype(np.uint32),
        (rng.standard_normal(1 << 18).astype(np.float32) * 3).view(np.uint32),
        np.array(WL.special_values_f32(), np.uint32)])
    a_bits = a_bits[_domain(op, a_bits.view(np.float32).astype(np.float64))]
    dy_bits = (rng.standard_normal(a_bits.size).astype(np.float32)).view(np.uint32)
    a = torch.from_numpy(a_bits.view(np.int32)).cuda().view(torch.float32)
    dy = torch.from_numpy(dy_bits.view(np.int32)).cuda().view(torch.float32)
    dx = getattr(kt, f"k{op}_bwd_f32")(a, dy)
    want = O.bwd_f32(op, a_bits, dy_bits)
    used = check_bwd(op, 32, a_bits, dy_bits, u32(dx), want)
    print(f"{op} bwd f32: largest fraction of the derived c u |dy| S allowance used: {used:.3g}")


@pytest.mark.parametrize("n,off", [(1, 0), (17, 1), (1000, 3), (65537, 0), (100003, 5)])
def test_bwd_sizes_offsets_inplace(kt, n, off):
    base = (torch.randn(n + 8, device="cuda") * 2).to(torch.bfloat16)
    dyb = torch.randn(n + 8, device="cuda").to(torch.bfloat16)
    a, dy = base[off:off + n], dyb[off:off + n]
    want = O.bwd_bf16("gelu", u16(a), u16(dy))
    out = kt.kgelu_bwd_bf16(a, dy)
    check_bwd("gelu", 16, u16(a), u16(dy), u16(out), want)
    z = dy.clone()
    kt.kgelu_bwd_bf16(a, z, out=z)                       # in place over dy
    check_bwd("gelu", 16, u16(a), u16(dy), u16(z), want)


def test_bwd_config5_sampled(kt):
    """Config 5 size (2^30 BF16) for the GELU backward, sampled outputs."""
    x = WL.make_input("c5_ffn_2p30", device="cuda")
    dy = WL.make_input("c5_ffn_2p30", device="cuda", seed=55)
    dx = kt.kgelu_bwd_bf16(x, dy)
    idx = torch.from_numpy(np.random.default_rng(9).integers(0, x.numel(), 1 << 16)).cuda()
    a_s, d_s, g_s = (u16(t.view(-1)[idx]) for t in (x, dy, dx))
    check_bwd("gelu", 16, a_s, d_s, g_s, O.bwd_bf16("gelu", a_s, d_s))
    del x, dy, dx
    torch.cuda.empty_cache()


def test_bwd_errors(kt):
    a = torch.zeros(64, device="cuda", dtype=torch.bfloat16)
    assert kt._lib.kgelu_bwd_bf16(a.data_ptr(), a.data_ptr(), a.data_ptr(), 64, None, None) == kt.KT_ERR_ARG
    b = torch.zeros(64, device="cuda", dtype=torch.bfloat16)
    assert kt._lib.ktanh_bwd_bf16(a.data_ptr(), b.data_ptr(), b.data_ptr(), 64, None) == kt.KT_OK  # dx == dy
    assert kt._lib.ktanh_bwd_bf16(a.data_ptr(), b.data_ptr(), a.data_ptr(), 64, None) == kt.KT_OK  # dx == a
    # dx partially overlapping an input is rejected
    assert kt._lib.ktanh_bwd_bf16(a.data_ptr(), b.data_ptr(), a.data_ptr() + 2, 32, None) == kt.KT_ERR_ARG
    torch.cuda.synchronize()
