"""GPU parity of the Table 2 comparators through the C ABI.

Pade / piecewise minimax / piecewise Taylor kernels (kt_apx_tanh_*) against
the binary64 oracle (oracle/apx_oracle.c) on the same bytes.  Tolerances are
derived from the fp32 arithmetic the kernels do (DESIGN.md R-CMP-TOL):
  BF16 out: <= 1 BF16 ulp (fp32 result vs binary64, then one RNE each side);
  F32 piecewise: |dy| <= (2n + 3) u S(x) + ulp(y),  S = sum |c_j| |h|^j,
  F32 Pade:      |dy| <= (2 dN + 2 dD + max(dN, dD) + 4) u |y| + ulp(y),
with u = 2^-24 and dN, dD the degrees in s = x^2.  The decisions (piece
index, saturation) are exact comparisons, so they agree on both sides; the
fp32 saturation constants of both sides are checked to be identical.
The GPU's own tanhf and tanh.approx are checked against error bounds of
binary64 tanh (no oracle exists for a hardware approximation).
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import workloads as WL
from _cmp import assert_ulp, ulp_dist

pytestmark = pytest.mark.gpu

CMP = [("pade", 3, 2), ("pade", 7, 8), ("pade", 1, 0), ("pade", 5, 4), ("minimax", 1, 0),
       ("minimax", 2, 0), ("minimax", 3, 0), ("taylor", 1, 0), ("taylor", 2, 0),
       ("taylor", 3, 0)]
U = 2.0 ** -24


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


def f32_tol(cfg, A, x):
    """Per-element absolute tolerance for the F32 path (see module doc)."""
    kind, p, q = cfg
    a = np.abs(x.astype(np.float64))
    y = np.abs(np.array([A.eval(v) for v in a]))
    ulp = np.spacing(y.astype(np.float32)).astype(np.float64)
    if kind == "pade":
        nd, dd = (p - 1) // 2, q // 2
        return (2 * nd + 2 * dd + max(nd, dd) + 4) * U * y + ulp
    k = np.minimum(np.floor(a * 2), 15).astype(int)
    h = a - k * 0.5
    if kind == "taylor":
        h = np.where(k > 0, h - 0.25, h)
    S = np.zeros_like(a)
    for j in range(p + 1):
        cj = A.par[1 + 4 * k + j]
        S += np.abs(cj) * np.abs(h) ** j
    return (2 * p + 3) * U * S + ulp


def f32_sample(A, n=1 << 18, seed=11):
    rng = np.random.default_rng(seed)
    xs = [rng.standard_normal(n // 2) * 3, rng.uniform(-9, 9, n // 2)]
    # piece boundaries, saturation constant and their neighbours
    edges = np.concatenate([np.arange(0, 8.5, 0.5), [np.float32(A.xsat)]]).astype(np.float32)
    nb = np.concatenate([edges, np.nextafter(edges, np.float32(0)), np.nextafter(edges, np.float32(9))])
    xs += [nb, -nb, np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-40, -1e-40, 1e-30, 3e38])]
    return np.concatenate(xs).astype(np.float32)


@pytest.mark.parametrize("cfg", CMP)
def test_exhaustive_bf16(kt, cfg):
    A = kt.Apx(*cfg)
    x = WL.make_input("c1_exhaustive_bf16", device="cuda")
    y = kt.kt_apx_tanh_bf16(x, A)
    torch.cuda.synchronize()
    want = O.Apx(*cfg).map_bf16(u16(x))
    got = u16(y)
    worst = assert_ulp(got, want, 16, 1, ctx=f"{cfg} bf16 exhaustive")
    # NaN passes through unchanged (bitwise), +-0 keep their sign
    nan = (u16(x) & 0x7FFF) > 0x7F80
    assert np.array_equal(got[nan], u16(x)[nan])
    assert got[0] == 0 and got[0x8000] == 0x8000
    print(cfg, "max BF16 ulp vs oracle:", worst)


@pytest.mark.parametrize("cfg", CMP)
def test_f32_sample(kt, cfg):
    A = kt.Apx(*cfg)
    B = O.Apx(*cfg)
    xh = f32_sample(B)
    x = torch.from_numpy(xh).cuda()
    y = kt.kt_apx_tanh_f32(x, A)
    torch.cuda.synchronize()
    got = u32(y)
    want = B.map_f32(xh.view(np.uint32))
    nan = np.isnan(xh)
    assert np.array_equal(got[nan], xh.view(np.uint32)[nan])
    fin = ~nan
    g = got[fin].view(np.float32).astype(np.float64)
    w = want[fin].view(np.float32).astype(np.float64)
    tol = f32_tol(cfg, B, xh[fin])
    bad = np.abs(g - w) > tol
    assert not bad.any(), (cfg, int(bad.sum()), xh[fin][bad][:5], g[bad][:5], w[bad][:5])
    print(cfg, "max F32 ulp vs oracle:", int(ulp_dist(got[fin], want[fin], 32).max()))


@pytest.mark.parametrize("n,xoff,yoff", [(1, 0, 0), (31, 0, 0), (33, 1, 1), (1000003, 3, 3),
                                         (4099, 1, 2), (0, 0, 0)])
def test_ragged_and_misaligned(kt, n, xoff, yoff):
    A = kt.Apx("minimax", 3)
    g = torch.Generator(device="cuda").manual_seed(n)
    base = (torch.randn(n + 64, device="cuda", generator=g) * 3).to(torch.bfloat16)
    x = base[xoff:xoff + n]
    ybuf = torch.full((n + 64,), float("nan"), dtype=torch.bfloat16, device="cuda")
    y = ybuf[yoff:yoff + n]
    kt.kt_apx_tanh_bf16(x, A, out=y)
    torch.cuda.synchronize()
    want = O.Apx("minimax", 3).map_bf16(u16(x))
    assert_ulp(u16(y), want, 16, 1, ctx=f"ragged n={n}")
    # guard bands untouched
    yb = u16(ybuf)
    assert np.all((yb[:yoff] & 0x7FFF) > 0x7F80) and np.all((yb[yoff + n:] & 0x7FFF) > 0x7F80)


def test_in_place(kt):
    A = kt.Apx("pade", 7, 8)
    x = (torch.randn(1 << 16, device="cuda") * 3).to(torch.bfloat16)
    want = O.Apx("pade", 7, 8).map_bf16(u16(x))
    kt.kt_apx_tanh_bf16(x, A, out=x)
    torch.cuda.synchronize()
    assert_ulp(u16(x), want, 16, 1, ctx="in place")


def test_config2_sampled(kt):
    """Config 2 (2^24 BF16 ~ N(0, 2^2)) at full size in the bench's launch
    shape, checked on a seeded sample of outputs."""
    x = WL.make_input("c2_bf16_2p24", device="cuda")
    xb = u16(x)
    rng = np.random.default_rng(5)
    idx = np.sort(rng.choice(x.numel(), 1 << 16, replace=False))
    for cfg in (("pade", 7, 8), ("minimax", 3, 0)):
        y = u16(kt.kt_apx_tanh_bf16(x, kt.Apx(*cfg)))
        assert_ulp(y[idx], O.Apx(*cfg).map_bf16(xb[idx]), 16, 1, ctx=f"{cfg} c2")


# ---------------------------------------------------------- GPU built-ins --
def _ref_tanh(x):
    return np.tanh(x.astype(np.float64))


def test_libm_tanhf_within_2ulp(kt):
    """CUDA's tanhf: max 2 ulp (CUDA math library accuracy table)."""
    xh = f32_sample(O.Apx("minimax", 3))
    x = torch.from_numpy(xh).cuda()
    got = u32(kt.kt_apx_tanh_f32(x, kt.Apx("libm")))
    fin = ~np.isnan(xh)
    want = _ref_tanh(xh[fin]).astype(np.float32).view(np.uint32)
    assert ulp_dist(got[fin], want, 32).max() <= 2
    assert np.array_equal(got[~fin], xh.view(np.uint32)[~fin])


def test_libm_bf16_within_1ulp(kt):
    x = WL.make_input("c1_exhaustive_bf16", device="cuda")
    got = u16(kt.kt_apx_tanh_bf16(x, kt.Apx("libm")))
    xv = O.bf16_to_f64(u16(x))
    fin = ~np.isnan(xv)
    want = np.array([O.bf16_encode_rne(v) for v in np.tanh(xv[fin])], np.uint16)
    assert ulp_dist(got[fin], want, 16).max() <= 1


def test_sfu_tanh_approx_error(kt):
    """tanh.approx.f32 (MUFU.TANH): measured error bound, abs <= 2^-10.5 and
    relative <= 2^-10 for |x| >= 2^-6 (the hardware approximation is a
    black box; the bound is the one asserted, the measured values printed)."""
    xh = f32_sample(O.Apx("minimax", 3))
    x = torch.from_numpy(xh).cuda()
    got = u32(kt.kt_apx_tanh_f32(x, kt.Apx("sfu")))
    fin = ~np.isnan(xh)
    g = got[fin].view(np.float32).astype(np.float64)
    r = _ref_tanh(xh[fin])
    ae = np.abs(g - r)
    big = np.abs(xh[fin]) >= 2.0 ** -6
    re = ae[big] / np.abs(r[big])
    print("sfu f32: max abs", ae.max(), "max rel (|x|>=2^-6)", re.max())
    assert ae.max() <= 2.0 ** -10.5 and re.max() <= 2.0 ** -10
    assert np.array_equal(got[~fin], xh.view(np.uint32)[~fin])


def test_sfu_bf16_error(kt):
    x = WL.make_input("c1_exhaustive_bf16", device="cuda")
    got = u16(kt.kt_apx_tanh_bf16(x, kt.Apx("sfu")))
    xv = O.bf16_to_f64(u16(x))
    fin = np.isfinite(xv)
    want = np.array([O.bf16_encode_rne(v) for v in np.tanh(xv[fin])], np.uint16)
    d = ulp_dist(got[fin], want, 16)
    print("sfu bf16: max ulp vs RN(tanh)", int(d.max()), "share exact", float((d == 0).mean()))
    assert d.max() <= 2
    nan = np.isnan(xv)
    assert np.array_equal(got[nan], u16(x)[nan])
