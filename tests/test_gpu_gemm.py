"""tcgen05 GEMM + K-activation epilogue (NEXT-2): numerics vs a float64 matmul
(the definition of the contraction) and bitwise equality of the fused epilogue
with the elementwise K-op applied to the plain GEMM output."""
import numpy as np
import pytest
import torch

import oracle as O
from _cmp import assert_bitexact, ulp_dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_07729_b200 as kt
    return kt


def u16(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def rand_bf16(shape, seed, scale=1.0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(shape, device="cuda", generator=g) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (128, 256, 128), (256, 512, 256),
                                   (384, 768, 1024)])
def test_gemm_vs_float64(kt, M, N, K):
    A, B = rand_bf16((M, K), 1, 0.5), rand_bf16((N, K), 2, 0.5)
    C = kt.kgemm_bf16(A, B)
    torch.cuda.synchronize()
    a = O.bf16_to_f64(u16(A)).reshape(M, K)
    b = O.bf16_to_f64(u16(B)).reshape(N, K)
    exact = a @ b.T                                        # float64 reference
    got = O.bf16_to_f64(u16(C)).reshape(M, N)
    # one BF16 rounding of the fp32 accumulator + fp32 accumulation error
    bound = np.abs(exact) * 2.0 ** -8 + K * 2.0 ** -23 * (np.abs(a) @ np.abs(b).T) + 1e-30
    err = np.abs(got - exact)
    assert np.all(err <= bound), (float(err.max()), float((err / bound).max()))


@pytest.mark.parametrize("epi", ["tanh", "sigmoid", "swish", "gelu"])
def test_gemm_epilogue_bitwise(kt, epi):
    M, N, K = 256, 512, 512
    A, B = rand_bf16((M, K), 3, 0.3), rand_bf16((N, K), 4, 0.3)
    plain = kt.kgemm_bf16(A, B)
    fused = kt.kgemm_bf16(A, B, epilogue=epi)
    ref = getattr(kt, f"k{epi}_bf16")(plain)
    torch.cuda.synchronize()
    assert_bitexact(u16(fused), u16(ref), 16, nan_by_class=True, ctx=f"gemm+{epi}")
    # and the epilogue itself is the oracle's K-op on the BF16 GEMM output (0 ulp;
    # the sign of a zero result is not compared, reading A21)
    want = O.map_bf16(epi, u16(plain))
    assert int(ulp_dist(u16(fused), want, 16).max()) == 0, f"gemm+{epi} vs oracle"


def test_gemm_bad_shapes(kt):
    A = rand_bf16((100, 64), 5)
    B = rand_bf16((256, 64), 6)
    with pytest.raises(kt.KTanhError):
        kt.kgemm_bf16(A, B)


_PAIR_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1909_07729_b200 as kt
out = {}
for (M, N, K) in [(256, 256, 64), (512, 768, 320), (768, 512, 1024), (1024, 2048, 256)]:
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = (torch.randn(M, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    for epi in (None, "gelu", "tanh"):
        C = kt.kgemm_bf16(A, B, epilogue=epi)
        out[f"{M}_{N}_{K}_{epi}"] = C.view(torch.int16).cpu().numpy()
np.savez(sys.argv[2], **out)
"""


def test_gemm_cta_pair_equals_single_cta(kt, tmp_path):
    """The CTA-pair kernel (tcgen05.mma.cta_group::2, M = 256) and the 1-CTA
    kernel give bit-identical C, plain and with epilogues (KT_GEMM_2CTA
    forces either; read once per process, hence the subprocesses)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "pair.py"
    script.write_text(_PAIR_SCRIPT)
    res = {}
    for mode in ("0", "1"):
        f = tmp_path / f"out{mode}.npz"
        env = dict(os.environ, KT_GEMM_2CTA=mode)
        subprocess.run([sys.executable, str(script), root, str(f)], check=True, env=env, timeout=300)
        res[mode] = np.load(f)
    for k in res["0"].files:
        assert np.array_equal(res["0"][k], res["1"][k]), k


@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (512, 768, 320), (1024, 2048, 1024)])
def test_gemm_pair_shapes_vs_float64(kt, M, N, K):
    """Shapes with M % 256 == 0 take the CTA-pair kernel (plain GEMM)."""
    A, B = rand_bf16((M, K), 7, 0.5), rand_bf16((N, K), 8, 0.5)
    C = kt.kgemm_bf16(A, B)
    torch.cuda.synchronize()
    a = O.bf16_to_f64(u16(A)).reshape(M, K)
    b = O.bf16_to_f64(u16(B)).reshape(N, K)
    exact = a @ b.T
    got = O.bf16_to_f64(u16(C)).reshape(M, N)
    bound = np.abs(exact) * 2.0 ** -8 + K * 2.0 ** -23 * (np.abs(a) @ np.abs(b).T) + 1e-30
    assert np.all(np.abs(got - exact) <= bound)


@pytest.mark.parametrize("M,H,K,tq", [(128, 256, 64, 2), (256, 512, 320, 0), (6400, 1024, 1024, 2),
                                      (384, 256, 128, 3)])
def test_gemm_lstm_gates_fused(kt, M, H, K, tq):
    """kgemm_lstm_gates_bf16 == kgemm_bf16 then klstm_gates_bf16 (bitwise, NaN
    by class), and the gate map is the oracle's on the BF16 GEMM output."""
    A, B = rand_bf16((M, K), 11, 0.4), rand_bf16((4 * H, K), 12, 0.4)
    fused = kt.kgemm_lstm_gates_bf16(A, B, H, tq)
    plain = kt.kgemm_bf16(A, B)
    ref = kt.klstm_gates_bf16(plain, H, tq)
    torch.cuda.synchronize()
    assert_bitexact(u16(fused), u16(ref), 16, nan_by_class=True, ctx=f"gemm+lstm {M}x{H}x{K}")
    want = O.lstm_gates_bf16(u16(plain), H, tq)
    assert_bitexact(u16(fused), want.reshape(-1), 16, nan_by_class=True, ctx="gemm+lstm vs oracle")


def test_gemm_lstm_gates_bad_args(kt):
    A, B = rand_bf16((128, 64), 13), rand_bf16((4 * 128, 64), 14)
    with pytest.raises(kt.KTanhError):
        kt.kgemm_lstm_gates_bf16(A, B, 128, 2)          # hidden % 256 != 0
    A, B = rand_bf16((128, 64), 13), rand_bf16((4 * 256, 64), 14)
    with pytest.raises(kt.KTanhError):
        kt.kgemm_lstm_gates_bf16(A, B, 256, 4)          # bad quarter


@pytest.mark.parametrize("M,H,K", [(128, 64, 64), (256, 192, 320), (6400, 1024, 1024), (384, 128, 128)])
def test_gemm_lstm_cell_fused(kt, M, H, K):
    """kgemm_lstm_cell_bf16 == kgemm_bf16 then klstm_cell_bf16 (bitwise), and
    the oracle's cell on the BF16 gate block; c_next in place over c_prev."""
    A, B = rand_bf16((M, K), 21, 0.4), rand_bf16((4 * H, K), 22, 0.4)
    g = torch.Generator(device="cuda").manual_seed(23)
    c = torch.randn(M, H, device="cuda", generator=g) * 2
    cn, hn = kt.kgemm_lstm_cell_bf16(A, B, c, H)
    gates = kt.kgemm_bf16(A, B)
    cn_ref, hn_ref = kt.klstm_cell_bf16(gates, c, H)
    torch.cuda.synchronize()
    assert torch.equal(cn.view(torch.int32), cn_ref.view(torch.int32)), "c_next"
    assert torch.equal(hn.view(torch.int16), hn_ref.view(torch.int16)), "h_next"
    if M * H <= 1 << 17:
        wc, wh = O.lstm_cell_bf16(u16(gates), c.view(torch.int32).cpu().numpy().view(np.uint32), H)
        assert np.array_equal(cn.view(torch.int32).cpu().numpy().view(np.uint32).reshape(-1), wc)
        assert np.array_equal(u16(hn).reshape(-1), wh)
    c2 = c.clone()
    cn2, hn2 = kt.kgemm_lstm_cell_bf16(A, B, c2, H, c_next=c2)        # in place
    torch.cuda.synchronize()
    assert torch.equal(cn2.view(torch.int32), cn_ref.view(torch.int32))
    assert torch.equal(hn2.view(torch.int16), hn_ref.view(torch.int16))


def test_gemm_lstm_cell_bad_args(kt):
    A, B = rand_bf16((128, 64), 24), rand_bf16((4 * 96, 64), 25)
    c = torch.zeros(128, 96, device="cuda")
    with pytest.raises(kt.KTanhError):
        kt.kgemm_lstm_cell_bf16(A, B, c, 96)                             # hidden % 64 != 0


def test_ffn_gemm_full_size(kt):
    """bench.py's FFN line at full size (65536 x 16384 x 4096, inputs from
    workloads/, the 1-CTA fused kernel the bench times): the fused K-GELU
    output equals kgelu_bf16 of the plain GEMM output on every element, and
    sampled plain outputs are within the bound of test_gemm_vs_float64 of the
    float64 dot products."""
    import workloads as WL
    M, N, K = 65536, 16384, 4096
    A = WL.make_input("c5_ffn_2p30", device="cuda", numel=M * K).reshape(M, K)
    B = (WL.make_input("c5_ffn_2p30", device="cuda", numel=N * K, seed=7).reshape(N, K) * 0.02
         ).to(torch.bfloat16)
    fused = kt.kgemm_bf16(A, B, epilogue="gelu")
    plain = kt.kgemm_bf16(A, B)
    ref = kt.kgelu_bf16(plain)
    assert torch.equal(fused.view(torch.int16), ref.view(torch.int16))
    del fused, ref
    rng = np.random.default_rng(12)
    r, c = rng.integers(0, M, 4096), rng.integers(0, N, 4096)
    a = O.bf16_to_f64(u16(A[torch.from_numpy(r).cuda()]))
    b = O.bf16_to_f64(u16(B[torch.from_numpy(c).cuda()]))
    exact = (a * b).sum(axis=1)
    got = O.bf16_to_f64(u16(plain[torch.from_numpy(r).cuda(), torch.from_numpy(c).cuda()]))
    bound = np.abs(exact) * 2.0 ** -8 + K * 2.0 ** -23 * (np.abs(a) * np.abs(b)).sum(axis=1) + 1e-30
    assert np.all(np.abs(got - exact) <= bound)


@pytest.mark.parametrize("epi", ["swish", "gelu"])
@pytest.mark.parametrize("M", [128, 256])
def test_gemm_epilogue_tiny_preactivations(kt, epi, M):
    """Pre-activations below 2^-125 (the x/2 ties of R-DERIVED) in some rows
    and ordinary values in others: the epilogue's screen must send those
    chunks through the exact outer step.  A[i, 0] = m_i 2^-70 with odd m_i,
    B[j, 0] = 2^-63, so A B^T holds m_i 2^-133 exactly (a BF16 subnormal tie
    candidate) unless the MMA flushes it; either way the fused output equals
    the oracle applied to the plain GEMM output, bit for bit."""
    N, K = 256, 64
    a = np.zeros((M, K), np.float32)
    b = np.zeros((N, K), np.float32)
    rng = np.random.default_rng(M)
    tiny_rows = np.arange(0, M, 2)
    a[tiny_rows, 0] = (2 * rng.integers(0, 128, tiny_rows.size) + 1).astype(np.float32) * 2.0 ** -70
    a[tiny_rows, 0] *= np.where(rng.random(tiny_rows.size) < 0.5, -1.0, 1.0).astype(np.float32)
    b[:, 0] = 2.0 ** -63
    a[1::2, 1:] = rng.standard_normal((M // 2, K - 1)).astype(np.float32) * 0.5
    b[:, 1:] = rng.standard_normal((N, K - 1)).astype(np.float32) * 0.5
    A = torch.from_numpy(a).cuda().to(torch.bfloat16)
    B = torch.from_numpy(b).cuda().to(torch.bfloat16)
    plain = u16(kt.kgemm_bf16(A, B))
    fused = u16(kt.kgemm_bf16(A, B, epilogue=epi))
    assert_bitexact(fused, O.map_bf16(epi, plain), 16, nan_by_class=True, zero_by_value=True,
                    ctx=f"gemm {epi} tiny pre-activations")
    ties = int(np.count_nonzero(((plain & 0x7FFF) < 0x100) & ((plain & 1) == 1)))
    print(f"gemm {epi} M={M}: {ties} x/2-tie pre-activations in the output")
