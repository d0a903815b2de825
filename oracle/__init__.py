"""oracle -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

ctypes front end of ``oracle/ktanh_oracle.c``: a plain, slow, scalar CPU
implementation of K-TanH (arXiv 1909.07729) written from PAPER.md.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  It never imports the
product package ``paper_1909_07729_b200`` and shares no code with it.

numpy is used for array plumbing only; all of the method's arithmetic is
in the C file (each function there cites its PAPER.md passage).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ktanh_oracle.c")
_SRC_APX = os.path.join(_HERE, "apx_oracle.c")     # Table 2 comparators
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OPS = {"tanh": 0, "sigmoid": 1, "swish": 2, "gelu": 3,
       "tanh_via_bf16": 4}     # F32 only: K-TanH of RN_bf16(x), widened (NEXT-3)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (binary64, no FP contraction)."""
    stale = not os.path.exists(_LIB) or any(
        os.path.getmtime(_LIB) < os.path.getmtime(f) for f in (_SRC, _SRC_APX))
    if force or stale:
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
             "-fPIC", "-shared", "-o", tmp, _SRC, _SRC_APX, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            ip = ctypes.POINTER(ctypes.c_int)
            u16p = ctypes.POINTER(ctypes.c_uint16)
            u32p = ctypes.POINTER(ctypes.c_uint32)
            L.kto_bf16_decode.argtypes = [ctypes.c_uint16]
            L.kto_bf16_decode.restype = ctypes.c_double
            L.kto_bf16_encode_rne.argtypes = [ctypes.c_double]
            L.kto_bf16_encode_rne.restype = ctypes.c_uint16
            L.kto_table1.argtypes = [ip, ip, ip]
            L.kto_table1.restype = None
            L.kto_ktanh_bf16.argtypes = [ctypes.c_uint16, ip, ip, ip]
            L.kto_ktanh_bf16.restype = ctypes.c_uint16
            L.kto_ktanh_f32.argtypes = [ctypes.c_uint32, ip, ip, ip]
            L.kto_ktanh_f32.restype = ctypes.c_uint32
            L.kto_map_bf16.argtypes = [ctypes.c_int, u16p, u16p, ctypes.c_size_t, ip, ip, ip]
            L.kto_map_bf16.restype = None
            L.kto_map_f32.argtypes = [ctypes.c_int, u32p, u32p, ctypes.c_size_t, ip, ip, ip]
            L.kto_map_f32.restype = None
            L.kto_map_bf16_at.argtypes = [ctypes.c_int, u16p, ctypes.POINTER(ctypes.c_uint64),
                                          u16p, ctypes.c_size_t, ip, ip, ip]
            L.kto_map_bf16_at.restype = None
            L.kto_lstm_gates_bf16.argtypes = [u16p, u16p, ctypes.c_size_t, ctypes.c_size_t,
                                              ctypes.c_int, ip, ip, ip]
            L.kto_lstm_gates_bf16.restype = None
            L.kto_bounds.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip]
            L.kto_bounds.restype = None
            L.kto_build_lut.argtypes = [ctypes.c_int, ip, ip, ip, ctypes.POINTER(ctypes.c_double)]
            L.kto_build_lut.restype = None
            L.kto_interval_sse.argtypes = [ctypes.c_int, ip, ip, ip]
            L.kto_interval_sse.restype = ctypes.c_double
            L.kto_overflow_flag.argtypes = []
            L.kto_overflow_flag.restype = ctypes.c_int
            L.kto_bwd_map_bf16.argtypes = [ctypes.c_int, u16p, u16p, u16p, ctypes.c_size_t, ip, ip, ip]
            L.kto_bwd_map_bf16.restype = None
            L.kto_bwd_map_f32.argtypes = [ctypes.c_int, u32p, u32p, u32p, ctypes.c_size_t, ip, ip, ip]
            L.kto_bwd_map_f32.restype = None
            L.kto_lstm_cell_bf16.argtypes = [u16p, u32p, u32p, u16p, ctypes.c_size_t,
                                             ctypes.c_size_t, ip, ip, ip]
            L.kto_lstm_cell_bf16.restype = None
            L.kto_build_lut_s.argtypes = [ctypes.c_int, ctypes.c_int, ip, ip, ip,
                                          ctypes.POINTER(ctypes.c_double)]
            L.kto_build_lut_s.restype = None
            L.kto_map_bf16_s.argtypes = [u16p, u16p, ctypes.c_size_t, ctypes.c_int, ip, ip, ip]
            L.kto_map_bf16_s.restype = None
            L.kto_bounds_s.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip]
            L.kto_bounds_s.restype = None
            L.kto_bounds_sp.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip]
            L.kto_bounds_sp.restype = None
            L.kto_build_lut_sp.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ip, ip, ip,
                                           ctypes.POINTER(ctypes.c_double)]
            L.kto_build_lut_sp.restype = ctypes.c_int
            L.kto_map_f32_p.argtypes = [ctypes.c_int, u32p, u32p, ctypes.c_size_t, ip, ip, ip,
                                        ctypes.c_int]
            L.kto_map_f32_p.restype = None
            L.kto_bwd_map_f32_p.argtypes = [ctypes.c_int, u32p, u32p, u32p, ctypes.c_size_t, ip, ip,
                                            ip, ctypes.c_int]
            L.kto_bwd_map_f32_p.restype = None
            L.kto_rn32_exact_sum.argtypes = [ctypes.c_double, ctypes.c_double]
            L.kto_rn32_exact_sum.restype = ctypes.c_float
            L.kto_ktanh_f32_p23.argtypes = [ctypes.c_uint32, ip, ip, ip]
            L.kto_ktanh_f32_p23.restype = ctypes.c_uint32
            L.kto_gelu_consts.argtypes = [ctypes.c_int]
            L.kto_gelu_consts.restype = ctypes.c_uint32
            dp = ctypes.POINTER(ctypes.c_double)
            L.kto_tanh_maclaurin.argtypes = [ctypes.c_int, dp]
            L.kto_tanh_maclaurin.restype = None
            L.kto_pade.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp]
            L.kto_pade.restype = ctypes.c_int
            L.kto_pade_sat.argtypes = [ctypes.c_int, ctypes.c_int]
            L.kto_pade_sat.restype = ctypes.c_double
            L.kto_minimax_piece.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp]
            L.kto_minimax_piece.restype = ctypes.c_int
            L.kto_taylor_piece.argtypes = [ctypes.c_int, ctypes.c_int, dp]
            L.kto_taylor_piece.restype = ctypes.c_int
            L.kto_apx_params.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
            L.kto_apx_params.restype = ctypes.c_int
            L.kto_apx_eval.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, ctypes.c_double]
            L.kto_apx_eval.restype = ctypes.c_double
            L.kto_apx_map_bf16.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, u16p, u16p,
                                           ctypes.c_size_t]
            L.kto_apx_map_bf16.restype = None
            L.kto_apx_map_f32.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, u32p, u32p,
                                          ctypes.c_size_t]
            L.kto_apx_map_f32.restype = None
            _lib = L
    return _lib


class Lut:
    """Three integer tables (T_E, T_r, T_b), Alg. 1 line 1: 32 entries (3 mantissa
    index bits, Table 1 layout) or 64 entries (4 bits).  p = the
    mantissa width b is expressed in: 7 (BF16 tables such as Table 1; on F32
    data b is scaled by 2^16, reading A8) or 23 (F32-only tables re-optimised
    at p = 23)."""

    def __init__(self, E, r, b, p: int = 7):
        self.E = np.ascontiguousarray(E, dtype=np.int32)
        self.r = np.ascontiguousarray(r, dtype=np.int32)
        self.b = np.ascontiguousarray(b, dtype=np.int32)
        self.p = int(p)
        assert self.E.shape == self.r.shape == self.b.shape and self.E.shape[0] in (32, 64)
        assert self.p in (7, 23)

    @property
    def s_bits(self):
        return 3 if self.E.shape[0] == 32 else 4

    def ptrs(self):
        ip = ctypes.POINTER(ctypes.c_int)
        return (self.E.ctypes.data_as(ip), self.r.ctypes.data_as(ip), self.b.ctypes.data_as(ip))

    def rows(self):
        return [(int(self.E[t]), int(self.r[t]), int(self.b[t])) for t in range(32)]


def table1() -> Lut:
    """The oracle's own transcription of Table 1."""
    E = np.zeros(32, np.int32); r = np.zeros(32, np.int32); b = np.zeros(32, np.int32)
    ip = ctypes.POINTER(ctypes.c_int)
    lib().kto_table1(E.ctypes.data_as(ip), r.ctypes.data_as(ip), b.ctypes.data_as(ip))
    return Lut(E, r, b)


def build_lut(bmin_zero: bool = False):
    """Sec. 2.4 optimizer (reading R*); returns (Lut, per-interval integer score)."""
    E = np.zeros(32, np.int32); r = np.zeros(32, np.int32); b = np.zeros(32, np.int32)
    sse = np.zeros(32, np.float64)
    ip = ctypes.POINTER(ctypes.c_int)
    lib().kto_build_lut(int(bmin_zero), E.ctypes.data_as(ip), r.ctypes.data_as(ip),
                        b.ctypes.data_as(ip), sse.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return Lut(E, r, b), sse


def build_lut_s(s_bits: int, bmin_zero: bool = False):
    """Sec. 2.4 optimizer with s mantissa index bits (s=4: the 64-interval table)."""
    n = 4 << s_bits
    E = np.zeros(n, np.int32); r = np.zeros(n, np.int32); b = np.zeros(n, np.int32)
    sse = np.zeros(n, np.float64)
    ip = ctypes.POINTER(ctypes.c_int)
    lib().kto_build_lut_s(s_bits, int(bmin_zero), E.ctypes.data_as(ip), r.ctypes.data_as(ip),
                          b.ctypes.data_as(ip), sse.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return Lut(E, r, b), sse


def build_lut_sp(s_bits: int, p: int, bmin_zero: bool = False):
    """Sec. 2.4 optimizer with s index bits and p mantissa bits (p = 23: the
    F32-native table); returns (Lut(p=p), per-interval score)."""
    key = (s_bits, p, bool(bmin_zero))
    if key not in _SP_CACHE:
        n = 4 << s_bits
        E = np.zeros(n, np.int32); r = np.zeros(n, np.int32); b = np.zeros(n, np.int32)
        sse = np.zeros(n, np.float64)
        ip = ctypes.POINTER(ctypes.c_int)
        rc = lib().kto_build_lut_sp(s_bits, p, int(bmin_zero), E.ctypes.data_as(ip),
                                    r.ctypes.data_as(ip), b.ctypes.data_as(ip),
                                    sse.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        if rc != 0:
            raise ValueError(f"unsupported (s, p) = ({s_bits}, {p})")
        _SP_CACHE[key] = (E, r, b, sse)
    E, r, b, sse = _SP_CACHE[key]
    return Lut(E.copy(), r.copy(), b.copy(), p=p), sse.copy()


_SP_CACHE: dict = {}


def bounds_sp(r: int, v: int, s_bits: int, p: int):
    lo = ctypes.c_int(); hi = ctypes.c_int()
    lib().kto_bounds_sp(r, v, s_bits, p, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def bounds_s(r: int, v: int, s_bits: int):
    lo = ctypes.c_int(); hi = ctypes.c_int()
    lib().kto_bounds_s(r, v, s_bits, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def bounds(r: int, v: int):
    lo = ctypes.c_int(); hi = ctypes.c_int()
    lib().kto_bounds(r, v, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def interval_sse(t: int, lut: Lut) -> float:
    return lib().kto_interval_sse(t, *lut.ptrs())


def overflow_flag() -> bool:
    return bool(lib().kto_overflow_flag())


def rn32_exact_sum(a: float, b: float) -> float:
    return float(lib().kto_rn32_exact_sum(float(a), float(b)))


def gelu_consts():
    return lib().kto_gelu_consts(0), lib().kto_gelu_consts(1)


def bf16_decode(w: int) -> float:
    return lib().kto_bf16_decode(int(w))


def bf16_encode_rne(x: float) -> int:
    return int(lib().kto_bf16_encode_rne(float(x)))


def _lut(lut):
    return table1() if lut is None else lut


def map_bf16(op: str, x_u16: np.ndarray, lut: Lut | None = None) -> np.ndarray:
    """y = op(x) for a uint16 array of BF16 bit patterns (any shape)."""
    lut = _lut(lut)
    assert lut.p == 7, "p = 23 tables are F32-only"
    x = np.ascontiguousarray(x_u16, dtype=np.uint16)
    y = np.empty_like(x)
    u16p = ctypes.POINTER(ctypes.c_uint16)
    if lut.s_bits != 3:
        assert op == "tanh", "64-entry tables: K-TanH only in the oracle"
        lib().kto_map_bf16_s(x.ctypes.data_as(u16p), y.ctypes.data_as(u16p), x.size, lut.s_bits,
                             *lut.ptrs())
        return y
    lib().kto_map_bf16(OPS[op], x.ctypes.data_as(u16p), y.ctypes.data_as(u16p), x.size, *lut.ptrs())
    return y


def map_f32(op: str, x_u32: np.ndarray, lut: Lut | None = None) -> np.ndarray:
    """y = op(x) for a uint32 array of FP32 bit patterns (any shape)."""
    lut = _lut(lut)
    x = np.ascontiguousarray(x_u32, dtype=np.uint32)
    y = np.empty_like(x)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    assert lut.s_bits == 3
    assert not (op == "tanh_via_bf16" and lut.p != 7), "via-BF16 needs a BF16 table"
    lib().kto_map_f32_p(OPS[op], x.ctypes.data_as(u32p), y.ctypes.data_as(u32p), x.size,
                        *lut.ptrs(), lut.p)
    return y


def bwd_bf16(op: str, a_u16: np.ndarray, dy_u16: np.ndarray, lut: Lut | None = None) -> np.ndarray:
    """Backward pass (reading R-BWD): a = saved output (tanh, sigmoid) or input x (swish, gelu)."""
    lut = _lut(lut)
    a = np.ascontiguousarray(a_u16, dtype=np.uint16)
    d = np.ascontiguousarray(dy_u16, dtype=np.uint16)
    assert a.shape == d.shape
    y = np.empty_like(a)
    u16p = ctypes.POINTER(ctypes.c_uint16)
    lib().kto_bwd_map_bf16(OPS[op], a.ctypes.data_as(u16p), d.ctypes.data_as(u16p),
                           y.ctypes.data_as(u16p), a.size, *lut.ptrs())
    return y


def bwd_f32(op: str, a_u32: np.ndarray, dy_u32: np.ndarray, lut: Lut | None = None) -> np.ndarray:
    lut = _lut(lut)
    a = np.ascontiguousarray(a_u32, dtype=np.uint32)
    d = np.ascontiguousarray(dy_u32, dtype=np.uint32)
    assert a.shape == d.shape
    y = np.empty_like(a)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    lib().kto_bwd_map_f32_p(OPS[op], a.ctypes.data_as(u32p), d.ctypes.data_as(u32p),
                            y.ctypes.data_as(u32p), a.size, *lut.ptrs(), lut.p)
    return y


def map_bf16_at(op: str, x_u16: np.ndarray, idx: np.ndarray, lut: Lut | None = None) -> np.ndarray:
    """Sampled evaluation: y[j] = op(x[idx[j]])."""
    lut = _lut(lut)
    x = np.ascontiguousarray(x_u16.reshape(-1), dtype=np.uint16)
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    y = np.empty(idx.shape, np.uint16)
    u16p = ctypes.POINTER(ctypes.c_uint16)
    lib().kto_map_bf16_at(OPS[op], x.ctypes.data_as(u16p),
                          idx.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                          y.ctypes.data_as(u16p), idx.size, *lut.ptrs())
    return y


def lstm_gates_bf16(x_u16: np.ndarray, hidden: int, tanh_quarter: int = 2,
                    lut: Lut | None = None) -> np.ndarray:
    """[rows, 4*hidden] BF16 gate block: K-TanH on quarter `tanh_quarter`, K-Sigmoid elsewhere."""
    lut = _lut(lut)
    x = np.ascontiguousarray(x_u16, dtype=np.uint16)
    assert x.size % (4 * hidden) == 0
    rows = x.size // (4 * hidden)
    y = np.empty_like(x)
    u16p = ctypes.POINTER(ctypes.c_uint16)
    lib().kto_lstm_gates_bf16(x.ctypes.data_as(u16p), y.ctypes.data_as(u16p), rows, hidden,
                              tanh_quarter, *lut.ptrs())
    return y


def lstm_cell_bf16(gates_u16: np.ndarray, c_prev_u32: np.ndarray, hidden: int,
                   lut: Lut | None = None):
    """Fused LSTM cell (reading R-LSTM-CELL): returns (c_next bits u32, h_next bits u16)."""
    lut = _lut(lut)
    g = np.ascontiguousarray(gates_u16, dtype=np.uint16)
    c = np.ascontiguousarray(c_prev_u32, dtype=np.uint32)
    rows = g.size // (4 * hidden)
    assert g.size == rows * 4 * hidden and c.size == rows * hidden
    cn = np.empty(rows * hidden, np.uint32)
    hn = np.empty(rows * hidden, np.uint16)
    u16p = ctypes.POINTER(ctypes.c_uint16)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    lib().kto_lstm_cell_bf16(g.ctypes.data_as(u16p), c.ctypes.data_as(u32p), cn.ctypes.data_as(u32p),
                             hn.ctypes.data_as(u16p), rows, hidden, *lut.ptrs())
    return cn, hn


def all_bf16() -> np.ndarray:
    return np.arange(65536, dtype=np.uint32).astype(np.uint16)


def bf16_to_f64(w: np.ndarray) -> np.ndarray:
    """Exact decode of BF16 bit patterns (via the F32 embedding)."""
    with np.errstate(invalid="ignore"):
        return (np.asarray(w, dtype=np.uint32) << 16).view(np.float32).astype(np.float64)


def error_sweep(lut: Lut | None = None):
    """Table 2 accuracy columns: max |K-TanH(x) - tanh(x)| and max
    relative error over every finite BF16 x (relative error over x != 0)."""
    w = all_bf16()
    xv = bf16_to_f64(w)
    finite = np.isfinite(xv)
    y = bf16_to_f64(map_bf16("tanh", w, lut))
    ref = np.tanh(xv)
    err = np.abs(y - ref)
    err[~finite] = 0.0
    nz = finite & (xv != 0)
    rel = np.zeros_like(err)
    rel[nz] = err[nz] / np.abs(ref[nz])
    i = int(np.argmax(err)); j = int(np.argmax(rel))
    return {"max_abs": float(err[i]), "argmax_abs": int(w[i]),
            "max_rel": float(rel[j]), "argmax_rel": int(w[j])}


# ---------------------------------------------------------------------------
# Table 2 comparators: Pade,
# piecewise minimax and piecewise Taylor forms of TanH, apx_oracle.c.
# ---------------------------------------------------------------------------
APX_KINDS = {"pade": 0, "minimax": 1, "taylor": 2}
APX_PIECES = 16        # reading R-CMP-LAYOUT: 16 pieces of width 1/2 on [0, 8)
APX_WIDTH = 0.5
APX_XSAT = 8.0


def tanh_maclaurin(n: int) -> np.ndarray:
    t = np.zeros(n + 1)
    lib().kto_tanh_maclaurin(n, t.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return t


def pade(p: int, q: int):
    """(a[0..p], b[0..q]) with b[0] = 1, or None if (p, q) is unsupported."""
    a = np.zeros(p + 1); b = np.zeros(q + 1)
    dp = ctypes.POINTER(ctypes.c_double)
    if lib().kto_pade(p, q, a.ctypes.data_as(dp), b.ctypes.data_as(dp)) != 0:
        return None
    return a, b


def pade_sat(p: int, q: int) -> float:
    return float(lib().kto_pade_sat(p, q))


def minimax_piece(deg: int, k: int):
    """(c[0..3] in h = x - k/2, levelled error E, Remez iterations)."""
    c = np.zeros(4); E = np.zeros(1)
    dp = ctypes.POINTER(ctypes.c_double)
    it = lib().kto_minimax_piece(deg, k, c.ctypes.data_as(dp), E.ctypes.data_as(dp))
    return c, float(E[0]), int(it)


def taylor_piece(deg: int, k: int) -> np.ndarray:
    c = np.zeros(4)
    rc = lib().kto_taylor_piece(deg, k, c.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert rc == 0
    return c


class Apx:
    """One comparator: kind in APX_KINDS; (p, q) = Pade orders, or (degree, 0)."""

    def __init__(self, kind: str, p: int, q: int = 0):
        self.kind, self.p, self.q = kind, p, q
        self.par = np.zeros(1 + 4 * APX_PIECES)
        rc = lib().kto_apx_params(APX_KINDS[kind], p, q, self._dp())
        if rc != 0:
            raise ValueError(f"unsupported comparator {kind} {p}/{q}")

    def _dp(self):
        return self.par.ctypes.data_as(ctypes.POINTER(ctypes.c_double))

    def _args(self):
        return (APX_KINDS[self.kind], self.p, self.q, self._dp())

    @property
    def xsat(self) -> float:
        return float(self.par[0])

    def piece(self, k: int) -> np.ndarray:
        return self.par[1 + 4 * k: 5 + 4 * k].copy()

    def pade_coeffs(self):
        return self.par[1:self.p + 2].copy(), self.par[self.p + 2:self.p + self.q + 3].copy()

    def eval(self, x: float) -> float:
        return float(lib().kto_apx_eval(*self._args(), float(x)))

    def map_bf16(self, x_u16: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x_u16, dtype=np.uint16)
        y = np.empty_like(x)
        u16p = ctypes.POINTER(ctypes.c_uint16)
        lib().kto_apx_map_bf16(*self._args(), x.ctypes.data_as(u16p), y.ctypes.data_as(u16p), x.size)
        return y

    def map_f32(self, x_u32: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x_u32, dtype=np.uint32)
        y = np.empty_like(x)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        lib().kto_apx_map_f32(*self._args(), x.ctypes.data_as(u32p), y.ctypes.data_as(u32p), x.size)
        return y
