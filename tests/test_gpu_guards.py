"""Out-of-bounds write checks (compute-sanitizer is closed on this pool):
every output buffer is embedded in a sentinel-filled guard band, which must
be untouched after the call, for ragged sizes / offsets on every kernel."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
G = 64                          # guard elements on each side


@pytest.fixture(scope="module")
def kt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1909_07729_b200 as kt
    return kt


def guarded(n, dtype, off=0, sentinel=-7.0):
    buf = torch.full((n + 2 * G + off,), sentinel, dtype=dtype, device="cuda")
    return buf, buf[G + off:G + off + n]


def intact(buf, n, off=0, sentinel=-7.0):
    torch.cuda.synchronize()
    b = buf.float().cpu().numpy()
    return np.all(b[:G + off] == sentinel) and np.all(b[G + off + n:] == sentinel)


@pytest.mark.parametrize("n", [1, 15, 16, 17, 999, 4097, 65537])
@pytest.mark.parametrize("off", [0, 1, 5])
def test_forward_and_backward_guards(kt, n, off):
    for dt, sfx in ((torch.bfloat16, "bf16"), (torch.float32, "f32")):
        x = (torch.randn(n, device="cuda") * 3).to(dt)
        dy = torch.randn(n, device="cuda").to(dt)
        for op in ("tanh", "gelu"):
            buf, y = guarded(n, dt, off)
            getattr(kt, f"k{op}_{sfx}")(x, out=y)
            assert intact(buf, n, off), (op, sfx, n, off)
            buf, y = guarded(n, dt, off)
            getattr(kt, f"k{op}_bwd_{sfx}")(x, dy, out=y)
            assert intact(buf, n, off), (op, "bwd", sfx, n, off)


@pytest.mark.parametrize("rows,H", [(3, 16), (5, 10), (7, 1024)])
def test_lstm_guards(kt, rows, H):
    g = (torch.randn(rows, 4 * H, device="cuda") * 1.5).to(torch.bfloat16)
    buf, y = guarded(rows * 4 * H, torch.bfloat16)
    kt.klstm_gates_bf16(g, H, 2, out=y.view(rows, 4 * H))
    assert intact(buf, rows * 4 * H)
    c = torch.randn(rows, H, device="cuda")
    cbuf, cn = guarded(rows * H, torch.float32)
    hbuf, hn = guarded(rows * H, torch.bfloat16)
    kt.klstm_cell_bf16(g, c, H, c_next=cn.view(rows, H), h_next=hn.view(rows, H))
    assert intact(cbuf, rows * H) and intact(hbuf, rows * H)


def test_gemm_guards(kt):
    M, N, K = 256, 512, 192
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    buf = torch.full((M * N + 2 * 4096,), -7.0, dtype=torch.bfloat16, device="cuda")
    C = buf[4096:4096 + M * N].view(M, N)                 # 32-byte aligned interior
    kt.kgemm_bf16(A, B, epilogue="gelu", out=C)
    torch.cuda.synchronize()
    b = buf.float().cpu().numpy()
    assert np.all(b[:4096] == -7.0) and np.all(b[4096 + M * N:] == -7.0)


@pytest.mark.parametrize("epi", [None, "gelu"])
def test_gemm_pair_guards(kt, epi):
    """CTA-pair kernel (M % 256 == 0) writes nothing outside C."""
    M, N, K = 512, 768, 128
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    buf = torch.full((M * N + 2 * 4096,), -7.0, dtype=torch.bfloat16, device="cuda")
    C = buf[4096:4096 + M * N].view(M, N)
    kt.kgemm_bf16(A, B, epilogue=epi, out=C)
    torch.cuda.synchronize()
    b = buf.float().cpu().numpy()
    assert np.all(b[:4096] == -7.0) and np.all(b[4096 + M * N:] == -7.0)


def test_gemm_lstm_guards(kt):
    """Fused gate GEMM and GEMM + cell write only their outputs."""
    M, H, K = 256, 256, 128
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(4 * H, K, device="cuda").to(torch.bfloat16)
    gbuf = torch.full((M * 4 * H + 2 * 4096,), -7.0, dtype=torch.bfloat16, device="cuda")
    kt.kgemm_lstm_gates_bf16(A, B, H, 2, out=gbuf[4096:4096 + M * 4 * H].view(M, 4 * H))
    cbuf = torch.full((M * H + 2 * 4096,), -7.0, dtype=torch.float32, device="cuda")
    hbuf = torch.full((M * H + 2 * 4096,), -7.0, dtype=torch.bfloat16, device="cuda")
    c = torch.randn(M, H, device="cuda")
    kt.kgemm_lstm_cell_bf16(A, B, c, H, c_next=cbuf[4096:4096 + M * H].view(M, H),
                            h_next=hbuf[4096:4096 + M * H].view(M, H))
    torch.cuda.synchronize()
    for buf, n in ((gbuf, M * 4 * H), (cbuf, M * H), (hbuf, M * H)):
        b = buf.float().cpu().numpy()
        assert np.all(b[:4096] == -7.0) and np.all(b[4096 + n:] == -7.0)


@pytest.mark.parametrize("n", [1, 17, 4097, 65537])
@pytest.mark.parametrize("off", [0, 3])
def test_other_streaming_guards(kt, n, off):
    """Fused GELU+Swish, 64-interval K-TanH, via-BF16 and the Table 2
    comparators (flat and pipelined launches) write only their outputs."""
    x = (torch.randn(n, device="cuda") * 3).to(torch.bfloat16)
    gb, g = guarded(n, torch.bfloat16, off)
    sb, s = guarded(n, torch.bfloat16, off + 1)
    kt.kgelu_swish_bf16(x, out_gelu=g, out_swish=s)
    assert intact(gb, n, off) and intact(sb, n, off + 1)
    E, r, b = kt.paper_lut().tables()
    t64 = [(((t >> 4) << 3) | ((t & 15) >> 1)) for t in range(64)]
    L64 = kt.Lut64([E[i] for i in t64], [r[i] for i in t64], [b[i] for i in t64])
    buf, y = guarded(n, torch.bfloat16, off)
    kt.ktanh64_bf16(x, L64, out=y)
    assert intact(buf, n, off)
    xf = x.float()
    buf, y = guarded(n, torch.float32, off)
    kt.ktanh_f32_via_bf16(xf, out=y)
    assert intact(buf, n, off)
    for kind, p, q in (("pade", 7, 8), ("minimax", 3, 0), ("taylor", 2, 0)):
        A = kt.Apx(kind, p, q)
        buf, y = guarded(n, torch.bfloat16, off)
        kt.kt_apx_tanh_bf16(x, A, out=y)
        assert intact(buf, n, off), kind
        buf, y = guarded(n, torch.float32, off)
        kt.kt_apx_tanh_f32(xf, A, out=y)
        assert intact(buf, n, off), kind


@pytest.mark.parametrize("n", [1, 1000, 3 * 65536 + 7])
def test_apply_host_guards(kt, n):
    """The host-buffer pipeline writes only the n output elements of the
    (pinned) host buffer."""
    x = (torch.randn(n) * 3).to(torch.bfloat16).pin_memory()
    buf = torch.full((n + 2 * G,), -7.0, dtype=torch.bfloat16).pin_memory()
    work = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    kt.apply_host("tanh", x, buf[G:G + n], work, chunk=4096)
    torch.cuda.synchronize()
    b = buf.float().numpy()
    assert np.all(b[:G] == -7.0) and np.all(b[G + n:] == -7.0)
