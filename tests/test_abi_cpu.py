"""C-ABI library checks that need no GPU: the library loads, exports every
symbol include/ktanh.h declares, validates parameter tables, rejects bad
arguments before touching the device, and computes shard ranges."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import oracle as O

HEADER = os.path.join(ROOT, "include", "ktanh.h")


@pytest.fixture(scope="module")
def kt():
    import __graft_entry__
    __graft_entry__._build_module().build()
    import paper_1909_07729_b200 as kt
    return kt


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"KT_API\s+[\w\s\*]+?\b(\w+)\s*\(", txt)))


def test_header_declares_the_north_star_calls():
    names = declared_symbols()
    for n in ("ktanh_bf16", "ktanh_f32", "ksigmoid_bf16", "ksigmoid_f32", "kswish_bf16",
              "kswish_f32", "kgelu_bf16", "kgelu_f32", "kt_lut_create", "kt_lut_destroy",
              "klstm_gates_bf16", "kt_apply_host", "kt_shard_range"):
        assert n in names


def test_library_exports_every_declared_symbol(kt):
    lib = ctypes.CDLL(kt.LIB_PATH)
    for n in declared_symbols():
        assert hasattr(lib, n), n
    assert set(declared_symbols()) == set(kt.EXPORTS)
    assert kt.abi_version() == 1


def test_paper_lut_roundtrip(kt):
    E, r, b = kt.Lut.paper().tables()
    T = O.table1()
    assert (E, r, b) == (list(T.E), list(T.r), list(T.b))


def test_lut_validation_accepts_optimizer_tables(kt):
    for bz in (False, True):
        L, _ = O.build_lut(bz)
        h = kt.Lut.from_tables(L.E, L.r, L.b)
        assert h.tables() == (list(L.E), list(L.r), list(L.b))


def test_lut_validation_bounds(kt):
    """Every b within the Sec. 2.4 bounds is accepted; b_max + 1
    and r outside [0, 7] are rejected with KT_ERR_LUT."""
    T = O.table1()
    rng = np.random.default_rng(0)
    for _ in range(200):
        E, r, b = T.E.copy(), T.r.copy(), T.b.copy()
        t = int(rng.integers(0, 32))
        if t == 7:
            continue
        r[t] = int(rng.integers(0, 8))
        lo, hi = O.bounds(int(r[t]), t & 7)
        b[t] = int(rng.integers(lo, hi + 1))
        kt.Lut.from_tables(E, r, b)
        b[t] = hi + 1
        with pytest.raises(kt.KTanhError) as ei:
            kt.Lut.from_tables(E, r, b)
        assert ei.value.status == kt.KT_ERR_LUT
    E, r, b = T.E.copy(), T.r.copy(), T.b.copy()
    r[3] = 8
    with pytest.raises(kt.KTanhError):
        kt.Lut.from_tables(E, r, b)
    E[3], r[3] = 128, 4
    with pytest.raises(kt.KTanhError):
        kt.Lut.from_tables(E, r, b)


def test_bad_arguments_rejected_before_device(kt):
    lut = kt.Lut.paper()
    lib = kt._lib
    for name in kt.MAP_CALLS:
        f = getattr(lib, name)
        assert f(None, None, 0, lut.handle, None) == kt.KT_OK          # n == 0: no launch
        assert f(None, None, 16, lut.handle, None) == kt.KT_ERR_ARG    # NULL with n > 0
        assert f(None, None, 16, None, None) == kt.KT_ERR_ARG          # NULL lut
    # misaligned element pointers and partial overlap are argument errors
    assert lib.ktanh_f32(ctypes.c_void_p(0x1002), ctypes.c_void_p(0x10002), 4, lut.handle, None) == kt.KT_ERR_ARG
    assert lib.ktanh_bf16(ctypes.c_void_p(0x1000), ctypes.c_void_p(0x1002), 64, lut.handle, None) == kt.KT_ERR_ARG
    assert lib.klstm_gates_bf16(None, None, 1, 0, 2, lut.handle, None) == kt.KT_ERR_ARG
    assert lib.klstm_gates_bf16(None, None, 1, 16, 4, lut.handle, None) == kt.KT_ERR_ARG
    assert lib.kt_apply(7, 0, None, None, 16, lut.handle, None) == kt.KT_ERR_ARG
    assert "overlap" in lib.kt_last_error().decode() or lib.kt_last_error()


@pytest.mark.parametrize("n", [0, 1, 15, 16, 17, 1000, 65537, 1 << 30, (1 << 33) + 5])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_partition(kt, n, world):
    """Shards tile [0, n) exactly, in rank order, each starting on a multiple of 16."""
    pos = 0
    for rank in range(world):
        b, c = kt.shard_range(n, world, rank, 16)
        assert b == pos and b % 16 == 0 or c == 0
        pos = b + c
    assert pos == n
    sizes = [kt.shard_range(n, world, r, 16)[1] for r in range(world)]
    assert max(sizes) - min(sizes) <= max(16, -(-n // world) + 16)


def test_shard_range_errors(kt):
    with pytest.raises(kt.KTanhError):
        kt.shard_range(10, 0, 0)
    with pytest.raises(kt.KTanhError):
        kt.shard_range(10, 2, 2)
    with pytest.raises(kt.KTanhError):
        kt.shard_range(10, 2, 0, 0)


def test_product_and_oracle_do_not_import_each_other():
    """The CUDA path and the oracle share no code and never import each other."""
    imp = re.compile(r"^\s*(import|from)\s+(\S+)|#include\s+[<\"]([^>\"]+)", re.M)
    pkg = os.path.join(ROOT, "paper_1909_07729_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                for m in imp.finditer(open(os.path.join(dp, f)).read()):
                    assert "oracle" not in "".join(g or "" for g in m.groups()), (f, m.group(0))
    for f in ("ktanh_oracle.c", "apx_oracle.c", "__init__.py"):
        for m in imp.finditer(open(os.path.join(ROOT, "oracle", f)).read()):
            tgt = "".join(g or "" for g in m.groups())
            assert "paper_1909_07729_b200" not in tgt and "ktanh.h" not in tgt and "kt_" not in tgt


# --------------------------------------------------------------------------
# Table 2 comparators: host-side coefficient generation
# --------------------------------------------------------------------------
APX_CMP = [("pade", 3, 2), ("pade", 7, 8), ("pade", 1, 0), ("pade", 1, 2), ("pade", 5, 4),
           ("pade", 5, 6), ("pade", 7, 6), ("minimax", 1, 0), ("minimax", 2, 0),
           ("minimax", 3, 0), ("taylor", 1, 0), ("taylor", 2, 0), ("taylor", 3, 0)]


@pytest.mark.parametrize("cfg", APX_CMP)
def test_apx_coefficients_match_oracle(kt, cfg):
    """The product derives its coefficients one way (Lambert convergents in
    integers, its own Remez with Newton-refined extrema, derivative
    polynomials in tanh(m)), the oracle another (the Pade linear system,
    Remez with golden-section extrema, the addition formula): they agree,
    and the fp32 saturation constants the kernels compare against are
    identical."""
    A = kt.Apx(*cfg)
    B = O.Apx(*cfg)
    c = np.array(A.coeffs())
    assert np.float32(c[0]) == np.float32(B.par[0])
    n = 1 + (cfg[1] + cfg[2] + 2 if cfg[0] == "pade" else 4 * O.APX_PIECES)
    np.testing.assert_allclose(c[1:n], B.par[1:n], rtol=1e-6, atol=1e-12)
    a32 = c[1:n].astype(np.float32).view(np.int32).astype(np.int64)
    b32 = B.par[1:n].astype(np.float32).view(np.int32).astype(np.int64)
    assert np.abs(a32 - b32).max() <= 1      # same sign: at most 1 fp32 ulp apart


@pytest.mark.parametrize("bad", [("pade", 2, 2), ("pade", 3, 3), ("pade", 3, 6), ("pade", 11, 12),
                                 ("minimax", 0, 0), ("minimax", 4, 0), ("taylor", 7, 0)])
def test_apx_rejects_unsupported(kt, bad):
    with pytest.raises(kt.KTanhError):
        kt.Apx(*bad)


def test_apx_calls_reject_host_pointers(kt):
    import torch
    A = kt.Apx("minimax", 3)
    x = torch.zeros(64, dtype=torch.bfloat16)
    with pytest.raises(TypeError):
        kt.kt_apx_tanh_bf16(x, A)
    buf = (ctypes.c_uint16 * 64)()
    # a host pointer never reaches a launch (KT_ERR_ARG on a GPU box, KT_ERR_CUDA without a device)
    st = kt._lib.kt_apx_tanh_bf16(ctypes.addressof(buf), ctypes.addressof(buf), 64, A.handle, None)
    assert st in (kt.KT_ERR_ARG, kt.KT_ERR_CUDA)
    lib = kt._lib
    for f in (lib.kt_apx_tanh_bf16, lib.kt_apx_tanh_f32):
        assert f(None, None, 0, A.handle, None) == kt.KT_OK               # n == 0: no launch
        assert f(None, None, 16, A.handle, None) == kt.KT_ERR_ARG         # NULL with n > 0
        assert f(ctypes.addressof(buf), ctypes.addressof(buf), 16, None, None) == kt.KT_ERR_ARG
    assert lib.kt_apx_tanh_f32(ctypes.c_void_p(0x1002), ctypes.c_void_p(0x10002), 4, A.handle,
                               None) == kt.KT_ERR_ARG                     # misaligned


def test_gelu_swish_fused_argument_errors(kt):
    lut = kt.Lut.paper()
    lib = kt._lib
    for f in (lib.kgelu_swish_bf16, lib.kgelu_swish_f32):
        assert f(None, None, None, 0, lut.handle, None) == kt.KT_OK
        assert f(None, None, None, 16, lut.handle, None) == kt.KT_ERR_ARG
    x, a, b = ctypes.c_void_p(0x10000), ctypes.c_void_p(0x20000), ctypes.c_void_p(0x20010)
    assert lib.kgelu_swish_bf16(x, a, a, 64, lut.handle, None) == kt.KT_ERR_ARG   # same output
    assert lib.kgelu_swish_bf16(x, a, b, 64, lut.handle, None) == kt.KT_ERR_ARG   # outputs overlap
    assert lib.kgelu_swish_bf16(x, ctypes.c_void_p(0x10010), b, 64, lut.handle, None) == kt.KT_ERR_ARG
    assert lib.kgelu_swish_bf16(x, a, ctypes.c_void_p(0x30000), 64, None, None) == kt.KT_ERR_ARG


def test_lut64_roundtrip_and_validation(kt):
    """64-interval tables: the Sec. 2.4 optimizer's s = 4 table
    is accepted and round-trips; out-of-bounds entries are KT_ERR_LUT."""
    L4, _ = O.build_lut_s(4)
    h = kt.Lut64(L4.E, L4.r, L4.b)
    E, r, b = h.tables()
    assert E == list(L4.E) and r == list(L4.r) and b == list(L4.b)
    bad_b = list(L4.b)
    t = 20                                      # v = 4: m in [32, 39]
    bad_b[t] = 127 - (32 >> L4.r[t]) + 1        # M_o = 128 for m = 32
    with pytest.raises(kt.KTanhError) as e:
        kt.Lut64(L4.E, L4.r, bad_b)
    assert e.value.status == kt.KT_ERR_LUT
    with pytest.raises(kt.KTanhError):
        kt.Lut64(L4.E, [8] * 64, L4.b)          # r > 7
    with pytest.raises(ValueError):
        kt.Lut64(L4.E[:32], L4.r[:32], L4.b[:32])
    assert kt._lib.ktanh64_bf16(None, None, 0, h.handle, None) == kt.KT_OK
    assert kt._lib.ktanh64_bf16(None, None, 16, h.handle, None) == kt.KT_ERR_ARG



# --------------------------------------------------------------------------
# Property-based checks of the host logic (hypothesis)
# --------------------------------------------------------------------------
from hypothesis import given, settings, strategies as st


@settings(max_examples=300, deadline=None)
@given(n=st.integers(0, 1 << 40), world=st.integers(1, 64), align=st.integers(1, 4096))
def test_shard_range_properties(kt, n, world, align):
    """kt_shard_range: the shards tile [0, n) in rank order, every non-empty
    shard starts on a multiple of `align`, and no shard exceeds
    ceil(n / world) rounded up to `align`."""
    cap = -(-(-(-n // world)) // align) * align
    pos = 0
    for rank in range(world):
        b, c = kt.shard_range(n, world, rank, align)
        assert b == pos or c == 0
        assert c == 0 or b % align == 0
        assert c <= cap
        pos = b + c if c else pos
    assert pos == n


def _lut_ok(E, r, b):
    """include/ktanh.h's validation rule, restated from the header: r in
    0..7, E in 1..127; for every mantissa the table path can reach in entry t
    (16v..16v+15, v = t & 7; only m = 112 when E & 3 == 0 i.e. E = 128),
    0 <= (m >> r) + b <= 127 (BF16) and the F32 M_o stays in [0, 2^23);
    E = 127 only if every reachable M_o is 0 (BF16 and F32)."""
    for t in range(32):
        if not (0 <= r[t] <= 7 and 1 <= E[t] <= 127):
            return False
        v = t & 7
        ms = [112] if (t >> 3) == 0 and v == 7 else list(range(16 * v, 16 * v + 16))
        for m in ms:
            mo = (m >> r[t]) + b[t]
            if not 0 <= mo <= 127 or (E[t] == 127 and mo != 0):
                return False
        lo23 = ms[0] << 16
        hi23 = lo23 if len(ms) == 1 else (ms[-1] << 16) | 0xFFFF
        if (lo23 >> r[t]) + b[t] * 65536 < 0 or (hi23 >> r[t]) + b[t] * 65536 > 0x7FFFFF:
            return False
        if E[t] == 127 and (hi23 >> r[t]) + b[t] * 65536 != 0:
            return False
    return True


@settings(max_examples=200, deadline=None)
@given(data=st.data())
def test_lut_validation_matches_the_rule(kt, data):
    """Random tables near Table 1: kt_lut_create accepts exactly those the
    documented rule accepts (KT_ERR_LUT otherwise)."""
    T = O.table1()
    E, r, b = list(T.E), list(T.r), list(T.b)
    for _ in range(data.draw(st.integers(1, 4))):
        t = data.draw(st.integers(0, 31))
        which = data.draw(st.sampled_from(["E", "r", "b"]))
        if which == "E":
            E[t] = data.draw(st.sampled_from([0, 1, 100, 125, 126, 127, 128]))
        elif which == "r":
            r[t] = data.draw(st.integers(-1, 8))
        else:
            b[t] = data.draw(st.integers(-130, 130))
    ok = _lut_ok(E, r, b)
    try:
        kt.Lut.from_tables(E, r, b)
        accepted = True
    except kt.KTanhError as e:
        assert e.status == kt.KT_ERR_LUT
        accepted = False
    assert accepted == ok, (E, r, b)


# ---- F32-native tables re-optimised at p = 23 -----------

def test_lut_f32_accepts_p23_optimizer_table(kt):
    L, _ = O.build_lut_sp(3, 23)
    h = kt.Lut.from_tables_f32(L.E, L.r, L.b)
    assert h.p == 23 and kt.Lut.paper().p == 7
    assert h.tables() == (list(L.E), list(L.r), list(L.b))
    T = O.table1()                           # Table 1 lifted to 2^-23 units is valid too
    kt.Lut.from_tables_f32(T.E, T.r, [int(v) * 65536 for v in T.b])


def test_lut_f32_validation_bounds(kt):
    """b within the p = 23 bounds (PAPER.md:210-219 with p = 23) accepted, b_max + 1
    and b_min - 1 rejected; r outside [0, 23] rejected."""
    L, _ = O.build_lut_sp(3, 23)
    rng = np.random.default_rng(1)
    for _ in range(100):
        E, r, b = L.E.copy(), L.r.copy(), L.b.copy()
        t = int(rng.integers(0, 32))
        if t == 7:
            continue
        r[t] = int(rng.integers(0, 24))
        lo, hi = O.bounds_sp(int(r[t]), t & 7, 3, 23)
        b[t] = int(rng.integers(lo, hi + 1))
        kt.Lut.from_tables_f32(E, r, b)
        # b_min = -v floor(2^(p-s-r)) is tight only for r <= p - s = 20
        for bad in ((hi + 1, lo - 1) if r[t] <= 20 else (hi + 1,)):
            b[t] = bad
            with pytest.raises(kt.KTanhError) as ei:
                kt.Lut.from_tables_f32(E, r, b)
            assert ei.value.status == kt.KT_ERR_LUT
    E, r, b = L.E.copy(), L.r.copy(), L.b.copy()
    r[3] = 24
    with pytest.raises(kt.KTanhError):
        kt.Lut.from_tables_f32(E, r, b)
    r[3], E[3] = L.r[3], 127                  # E = 127 needs M_o == 0
    with pytest.raises(kt.KTanhError):
        kt.Lut.from_tables_f32(E, r, b)


def test_lut_f32_rejected_by_bf16_calls(kt):
    """A p = 23 handle has no BF16 words: every BF16 call returns KT_ERR_LUT
    before touching the device; F32 calls accept it (n == 0: no launch)."""
    L, _ = O.build_lut_sp(3, 23)
    F = kt.Lut.from_tables_f32(L.E, L.r, L.b)       # keep the object: it owns the handle
    h = F.handle
    lib = kt._lib
    for name in kt.MAP_CALLS:
        want = kt.KT_ERR_LUT if ("bf16" in name) else kt.KT_OK
        assert getattr(lib, name)(None, None, 0, h, None) == want, name
    assert lib.kt_apply(0, 0, None, None, 0, h, None) == kt.KT_ERR_LUT
    assert lib.kt_apply(0, 1, None, None, 0, h, None) == kt.KT_OK
    assert lib.kswish_bwd_bf16(None, None, None, 0, h, None) == kt.KT_ERR_LUT
    assert lib.kswish_bwd_f32(None, None, None, 0, h, None) == kt.KT_OK
    assert lib.kgelu_swish_bf16(None, None, None, 0, h, None) == kt.KT_ERR_LUT
    assert lib.kgelu_swish_f32(None, None, None, 0, h, None) == kt.KT_OK
    assert lib.klstm_gates_bf16(None, None, 0, 16, 2, h, None) == kt.KT_ERR_LUT
    assert lib.klstm_cell_bf16(None, None, None, None, 0, 16, h, None) == kt.KT_ERR_LUT
    assert lib.kgemm_bf16(None, None, None, 0, 0, 0, 3, h, None) == kt.KT_ERR_LUT
    assert lib.kgemm_bf16(None, None, None, 0, 0, 0, -1, h, None) == kt.KT_OK
    assert lib.kgemm_lstm_cell_bf16(None, None, None, None, None, 0, 0, 0, h, None) == kt.KT_ERR_LUT
    assert "kt_lut_create_f32" in lib.kt_last_error().decode()


def test_library_optimizer_matches_oracle(kt):
    """kt_lut_create_optimized (product, kt_tables.cu) and the oracle's
    kto_build_lut_sp are separate implementations of Sec. 2.4: identical tables
    for p = 7 (both b_min readings), p = 23, and the 64-interval p = 7 table."""
    for bz in (False, True):
        L, _ = O.build_lut_sp(3, 7, bz)
        h = kt.Lut.optimized(7, bz)
        assert h.p == 7 and h.tables() == (list(L.E), list(L.r), list(L.b))
        L64, _ = O.build_lut_sp(4, 7, bz)
        assert kt.Lut64.optimized(bz).tables() == (list(L64.E), list(L64.r), list(L64.b))
    L, _ = O.build_lut_sp(3, 23)
    h = kt.Lut.optimized(23)
    assert h.p == 23 and h.tables() == (list(L.E), list(L.r), list(L.b))
    with pytest.raises(kt.KTanhError):
        kt.Lut.optimized(10)


def test_table_json_roundtrip(kt):
    """JSON table format (fields of SPEC.md:183): round trip for
    BF16, F32 (p = 23) and 64-interval tables; byte-identical text for equal
    tables; the text dump row 11000 of Table 1 reads (126, 0, 65)."""
    import json
    P = kt.Lut.paper()
    j = P.to_json("Table 1, PAPER.md:225-252")
    d = json.loads(j)
    assert d["format"] == "bfloat16" and d["man_msb_bits"] == 3 and d["t1_bits"] == "0x3E80"
    assert kt.lut_from_json(j).tables() == P.tables()
    assert kt.lut_from_json(j).to_json("Table 1, PAPER.md:225-252") == j
    row = [ln for ln in P.dump().splitlines() if ln.startswith("11000 ")][0].split()
    assert row[1:] == ["126", "0", "65"]
    F = kt.Lut.optimized(23)
    jf = F.to_json()
    assert json.loads(jf)["format"] == "float32" and json.loads(jf)["b_unit_bits"] == 23
    G = kt.lut_from_json(jf)
    assert G.p == 23 and G.tables() == F.tables()
    L64 = kt.Lut64.optimized()
    j64 = L64.to_json()
    assert kt.lut_from_json(j64).tables() == L64.tables() and len(L64.dump().splitlines()) == 64
    bad = json.loads(j)
    bad["r"][3] = 9
    with pytest.raises(kt.KTanhError):
        kt.lut_from_json(json.dumps(bad))
    bad = json.loads(j)
    bad["man_msb_bits"] = 5
    with pytest.raises(ValueError):
        kt.lut_from_json(json.dumps(bad))


def _build_c_demo(kt, tmp_path):
    import subprocess
    exe = str(tmp_path / "c_api_demo")
    libdir = os.path.dirname(kt.LIB_PATH)
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_api_demo.c"),
           "-L", libdir, "-lktanh", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{libdir}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_demo_builds_and_runs_host_part(kt, tmp_path):
    """The C ABI from plain C (gcc, no torch): table handles, the optimizer and
    validation errors (examples/c_api_demo.c, --no-gpu)."""
    import subprocess
    exe = _build_c_demo(kt, tmp_path)
    out = subprocess.run([exe, "--no-gpu"], check=True, capture_output=True, text=True).stdout
    assert "Table 1, row 11000: E=126 r=0 b=65" in out
    assert "p = 23 table" in out and "KT_ERR_LUT" in out


def test_lstm_cell_overlap_rule_exact(kt):
    """klstm_cell_bf16 / kgemm_lstm_cell_bf16 reject exactly the overlapping
    layouts: buffers of different sizes placed right next to each other (any
    order) are accepted by the overlap check (found when an allocator put
    h_next just below the gate block); real overlaps are rejected."""
    lib = kt._lib
    P = kt.Lut.paper()                               # keep the object: it owns the handle
    lut = P.handle
    rows, H = 4, 16
    n = rows * H
    base = 1 << 40                                   # fake, never dereferenced: no GPU here
    g, cp, cn = base, base + 8 * n, base + 12 * n     # gates | c_prev | c_next
    def cell(h, c_next=cn):
        st = lib.klstm_cell_bf16(ctypes.c_void_p(g), ctypes.c_void_p(cp), ctypes.c_void_p(c_next),
                                 ctypes.c_void_p(h), rows, H, lut, None)
        return st, lib.kt_last_error().decode()
    for h in (g - 2 * n, cn + 4 * n, g - 2 * n - 64):  # adjacent below gates, after c_next, gap
        st, err = cell(h)
        assert "overlap" not in err, (hex(h), err)
    for h in (g - 2 * n + 2, g + 8 * n - 2, cp + 2, cn + 4 * n - 2):
        st, err = cell(h)
        assert st == kt.KT_ERR_ARG and "overlap" in err, hex(h)
    st, err = cell(cn + 4 * n, c_next=cp)            # in place c_next == c_prev is allowed
    assert "overlap" not in err


def _ov(p, pb, q, qb):
    return pb > 0 and qb > 0 and p < q + qb and q < p + pb


def _layout(rng, sizes, align):
    """Random placement of buffers of the given byte sizes inside a small
    window (so that overlaps, adjacency and aliasing are all frequent)."""
    span = sum(sizes) * 2
    base = 1 << 40
    return [base + int(rng.integers(0, span // align)) * align for _ in sizes]


@pytest.mark.parametrize("fn", ["cell", "gemm_cell", "dual", "bwd", "gemm"])
def test_overlap_rules_random_layouts(kt, fn):
    """Every multi-buffer entry point flags an overlap exactly when its rule
    says so, over 3000 random layouts each (fake device addresses: the overlap
    check runs before any device access, so this needs no GPU)."""
    P = kt.Lut.paper()                               # keep the object: it owns the handle
    lib, lut = kt._lib, P.handle
    rng = np.random.default_rng(hash(fn) % 2**32)
    vp = ctypes.c_void_p
    for _ in range(3000):
        if fn == "cell":
            rows, H = 2, 16
            n = rows * H
            g, cp, cn, h = _layout(rng, [8 * n, 4 * n, 4 * n, 2 * n], 32)
            if rng.random() < 0.2:
                cn = cp
            want = ((cn != cp and _ov(cn, 4 * n, cp, 4 * n)) or _ov(cn, 4 * n, g, 8 * n) or
                    _ov(h, 2 * n, g, 8 * n) or _ov(h, 2 * n, cp, 4 * n) or _ov(h, 2 * n, cn, 4 * n))
            lib.klstm_cell_bf16(vp(g), vp(cp), vp(cn), vp(h), rows, H, lut, None)
        elif fn == "gemm_cell":
            M, H, K = 128, 64, 64
            a, b, cp, cn, h = _layout(rng, [M * K * 2, 4 * H * K * 2, M * H * 4, M * H * 4, M * H * 2], 32)
            if rng.random() < 0.2:
                cn = cp
            cb, hb = M * H * 4, M * H * 2
            want = ((cn != cp and _ov(cn, cb, cp, cb)) or _ov(h, hb, cn, cb) or
                    any(_ov(h, hb, p, s) for p, s in ((a, M * K * 2), (b, 4 * H * K * 2), (cp, cb))) or
                    any(_ov(cn, cb, p, s) for p, s in ((a, M * K * 2), (b, 4 * H * K * 2))))
            lib.kgemm_lstm_cell_bf16(vp(a), vp(b), vp(cp), vp(cn), vp(h), M, H, K, lut, None)
        elif fn == "dual":
            n = 64
            x, yg, ys = _layout(rng, [2 * n] * 3, 2)
            if rng.random() < 0.2:
                yg = x
            want = (yg == ys or _ov(yg, 2 * n, ys, 2 * n) or (yg != x and _ov(x, 2 * n, yg, 2 * n)) or
                    (ys != x and _ov(x, 2 * n, ys, 2 * n)))
            lib.kgelu_swish_bf16(vp(x), vp(yg), vp(ys), n, lut, None)
        elif fn == "bwd":
            n = 64
            a, dy, dx = _layout(rng, [2 * n] * 3, 2)
            if rng.random() < 0.2:
                dx = a if rng.random() < 0.5 else dy
            want = (dx != a and _ov(dx, 2 * n, a, 2 * n)) or (dx != dy and _ov(dx, 2 * n, dy, 2 * n))
            lib.kgelu_bwd_bf16(vp(a), vp(dy), vp(dx), n, lut, None)
        else:
            M, N, K = 128, 256, 64
            a, b, c = _layout(rng, [M * K * 2, N * K * 2, M * N * 2], 32)
            want = _ov(c, M * N * 2, a, M * K * 2) or _ov(c, M * N * 2, b, N * K * 2)
            lib.kgemm_bf16(vp(a), vp(b), vp(c), M, N, K, -1, None, None)
        got = "overlap" in lib.kt_last_error().decode()
        assert got == want, (fn, _)


def _lut_f32_ok(E, r, b):
    """The kt_lut_create_f32 rule written out (include/ktanh.h): r in [0, 23],
    E in [1, 127], every reachable M_o = (M23 >> r) + b in [0, 2^23), and
    E == 127 only with M_o == 0.  Reachable M23 of interval t: [2^20 v,
    2^20 (v + 1)), except t = 7 (E = 128), where only x = 3.75 (M23 = 7 2^20)
    is <= T2."""
    for t in range(32):
        if not (0 <= r[t] <= 23 and 1 <= E[t] <= 127):
            return False
        v = t & 7
        lo = v << 20
        hi = lo if t == 7 else ((v + 1) << 20) - 1
        mlo, mhi = (lo >> r[t]) + b[t], (hi >> r[t]) + b[t]
        if mlo < 0 or mhi > (1 << 23) - 1 or (E[t] == 127 and mhi != 0):
            return False
    return True


@settings(max_examples=300, deadline=None)
@given(data=st.data())
def test_lut_f32_validation_matches_the_rule(kt, data):
    """Random tables near the p = 23 optimizer table: kt_lut_create_f32 accepts
    exactly those the documented rule accepts."""
    L, _ = O.build_lut_sp(3, 23)
    E, r, b = [int(v) for v in L.E], [int(v) for v in L.r], [int(v) for v in L.b]
    for _ in range(data.draw(st.integers(1, 4))):
        t = data.draw(st.integers(0, 31))
        which = data.draw(st.sampled_from(["E", "r", "b"]))
        if which == "E":
            E[t] = data.draw(st.sampled_from([0, 1, 100, 125, 126, 127, 128]))
        elif which == "r":
            r[t] = data.draw(st.integers(-1, 24))
        else:
            rr = min(max(r[t], 0), 23)
            lo, hi = O.bounds_sp(rr, t & 7, 3, 23)
            b[t] = data.draw(st.sampled_from([lo - 1, lo, hi, hi + 1, (lo + hi) // 2, b[t] + 1, b[t] - 1]))
    ok = _lut_f32_ok(E, r, b)
    try:
        kt.Lut.from_tables_f32(E, r, b)
        accepted = True
    except kt.KTanhError as e:
        assert e.status == kt.KT_ERR_LUT
        accepted = False
    assert accepted == ok, (E, r, b)


def test_binding_rejects_unsupported_dtypes_and_strided_host_buffers(kt):
    """the generic entry points accept only bfloat16 and
    float32 (a float16 / int16 tensor used to go down the F32 path and read or
    write numel*4 bytes of a 2-byte buffer), and apply_host needs contiguous
    host tensors (the C ABI sees one pointer and an element count)."""
    import torch
    for dt in (torch.float16, torch.int16, torch.float64, torch.int32):
        x = torch.zeros(64, dtype=dt)
        with pytest.raises(TypeError, match="unsupported dtype"):
            kt.apply("tanh", x)
        with pytest.raises(TypeError, match="unsupported dtype"):
            kt.apply_host("tanh", x, torch.zeros_like(x), x)
    xs = torch.zeros(128, dtype=torch.bfloat16)[::2]
    with pytest.raises(ValueError, match="contiguous"):
        kt.apply_host("tanh", xs, torch.zeros(64, dtype=torch.bfloat16), xs)
    with pytest.raises(ValueError, match="must match"):
        kt.apply_host("tanh", torch.zeros(64, dtype=torch.bfloat16), torch.zeros(64), xs)


def test_binding_output_checks_cpu_side(kt):
    """caller-supplied outputs are validated before any
    pointer reaches the C ABI (_check_out): wrong dtype, size, device or layout."""
    import torch
    t = torch.zeros(16, dtype=torch.float32)
    with pytest.raises(TypeError, match="CUDA tensor"):
        kt._check_out(t, "c_next", torch.float32, 16, torch.device("cuda", 0))
