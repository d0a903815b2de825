"""GPU parity for F32-native tables re-optimised at p = 23 (SURVEY.md NEXT-3,
kt_lut_create_f32): the same F32 kernels with b in 2^-23 units, against the
oracle's kto_map_f32_p / kto_bwd_map_f32_p with the oracle-built table
(tests/test_oracle_f32_tables.py pins that table)."""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as WL
from _cmp import assert_bitexact, assert_ulp
from test_gpu_bwd import check_bwd      # the backward tolerance of reading R-BWD

pytestmark = pytest.mark.gpu

TOL = {"tanh": 0, "sigmoid": 0, "swish": 0, "gelu": 0}   # derived ops: exact (R-DERIVED)
T1_BITS = int(np.float32(0.25).view(np.uint32))
T2_BITS = int(np.float32(3.75).view(np.uint32))


@pytest.fixture(scope="module")
def kt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_07729_b200 as kt
    return kt


@pytest.fixture(scope="module")
def tables(kt):
    L, _ = O.build_lut_sp(3, 23)
    return L, kt.Lut.from_tables_f32(L.E, L.r, L.b)


def u32(t):
    return t.contiguous().view(torch.int32).cpu().numpy().view(np.uint32)


def dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int32)).cuda().view(torch.float32)


def check(op, got, want, ctx):
    if TOL[op] == 0:
        assert_bitexact(got, want, 32, nan_by_class=(op != "tanh"),
                        zero_by_value=op in ("swish", "gelu"), ctx=ctx)
    else:
        assert_ulp(got, want, 32, TOL[op], ctx=ctx)


def patterns():
    rng = np.random.default_rng(23)
    return np.concatenate([
        (np.arange(1 << 20, dtype=np.uint64) << 12).astype(np.uint32),
        ((np.arange(1 << 20, dtype=np.uint64) << 12) | 0xFFF).astype(np.uint32),
        rng.integers(0, 2**32, 1 << 20, dtype=np.uint64).astype(np.uint32),
        (rng.standard_normal(1 << 20) * 2).astype(np.float32).view(np.uint32),
        np.array(WL.special_values_f32(), np.uint32)])


def test_table_region_every_input(kt, tables):
    """K-TanH on every F32 input of the table path (T1 <= |x| <= T2, both signs)
    and its neighbours: bit-exact."""
    L, h = tables
    pos = np.arange(T1_BITS - 4096, T2_BITS + 4097, dtype=np.uint32)
    for bits in (pos, pos | np.uint32(0x80000000)):
        y = kt.ktanh_f32(dev(bits), lut=h)
        assert_bitexact(u32(y), O.map_f32("tanh", bits, L), 32, ctx="p23 tanh region")


@pytest.mark.parametrize("op", ["tanh", "sigmoid", "swish", "gelu"])
def test_ops_patterns(kt, tables, op):
    L, h = tables
    bits = patterns()
    y = getattr(kt, f"k{op}_f32")(dev(bits), lut=h)
    check(op, u32(y), O.map_f32(op, bits, L), f"p23 {op}")


@pytest.mark.parametrize("op", ["swish", "gelu"])
def test_bwd(kt, tables, op):
    L, h = tables
    rng = np.random.default_rng(5)
    a = np.concatenate([(rng.standard_normal(1 << 20) * 3).astype(np.float32).view(np.uint32),
                        np.array(WL.special_values_f32(), np.uint32)])
    dy = rng.standard_normal(a.size).astype(np.float32).view(np.uint32)
    dx = getattr(kt, f"k{op}_bwd_f32")(dev(a), dev(dy), lut=h)
    check_bwd(op, 32, a, dy, u32(dx), O.bwd_f32(op, a, dy, L))


def test_fused_gelu_swish(kt, tables):
    L, h = tables
    bits = patterns()
    g, s = kt.kgelu_swish_f32(dev(bits), lut=h)
    check("gelu", u32(g), O.map_f32("gelu", bits, L), "p23 dual gelu")
    check("swish", u32(s), O.map_f32("swish", bits, L), "p23 dual swish")


def test_config3_sampled(kt, tables):
    """Config 3 at full size (2^28 F32) in the bench's launch: sampled outputs."""
    L, h = tables
    x = WL.make_input("c3_f32_2p28", device="cuda")
    y = kt.ktanh_f32(x, lut=h)
    idx = torch.randint(0, x.numel(), (1 << 20,), generator=torch.Generator().manual_seed(3))
    xb = u32(x.view(-1)[idx.cuda()])
    assert_bitexact(u32(y.view(-1)[idx.cuda()]), O.map_f32("tanh", xb, L), 32, ctx="p23 c3")


def test_apply_host(kt, tables):
    L, h = tables
    bits = patterns()[: 3 << 20]
    x = torch.from_numpy(bits.view(np.int32)).view(torch.float32).pin_memory()
    y = torch.empty_like(x).pin_memory()
    work = torch.empty(1 << 22, dtype=torch.uint8, device="cuda")
    kt.apply_host("tanh", x, y, work, lut=h)
    torch.cuda.synchronize()
    assert_bitexact(y.view(torch.int32).numpy().view(np.uint32), O.map_f32("tanh", bits, L), 32,
                    ctx="p23 apply_host")


def test_bf16_calls_reject(kt, tables):
    _, h = tables
    x = torch.zeros(64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(kt.KTanhError) as ei:
        kt.ktanh_bf16(x, lut=h)
    assert ei.value.status == kt.KT_ERR_LUT
    with pytest.raises(kt.KTanhError):
        kt.ktanh_f32_via_bf16(x.float(), lut=h)


def test_more_accurate_than_table1(kt, tables):
    """The point of re-optimising: lower squared error against tanh over the
    table region than Table 1 on F32 (reading A8), same kernel throughput."""
    _, h = tables
    bits = np.arange(T1_BITS, T2_BITS + 1, dtype=np.uint32)
    x = dev(bits)
    ref = np.tanh(bits.view(np.float32).astype(np.float64))
    e23 = u32(kt.ktanh_f32(x, lut=h)).view(np.float32).astype(np.float64) - ref
    e7 = u32(kt.ktanh_f32(x)).view(np.float32).astype(np.float64) - ref
    assert (e23 ** 2).sum() < 0.85 * (e7 ** 2).sum()
