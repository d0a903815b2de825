"""paper_1909_07729_b200 -- K-TanH (arXiv 1909.07729) on B200 (sm_100a).

Thin ctypes binding over ``libktanh.so`` (C ABI in ``include/ktanh.h``).
This module only marshals arguments: every step of the K-TanH path runs in
the library's CUDA kernels.  PyTorch is used for device memory and streams
only.  There is no CPU fallback: if the library is missing, importing this
package raises ImportError (build it with ``python
paper_1909_07729_b200/build.py`` or ``__graft_entry__.build()``).

Names follow the C ABI: ktanh_bf16, ktanh_f32, ksigmoid_bf16, ksigmoid_f32,
kswish_bf16, kswish_f32, kgelu_bf16, kgelu_f32, klstm_gates_bf16,
apply_host (kt_apply_host) and shard_range (kt_shard_range).
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KT_LIB") or os.path.join(_PKG, "libktanh.so")   # KT_LIB: dev A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: the K-TanH CUDA library is not built "
        "(python paper_1909_07729_b200/build.py). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

_c_i32p = ctypes.POINTER(ctypes.c_int32)
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t

KT_OK, KT_ERR_ARG, KT_ERR_LUT, KT_ERR_CUDA = 0, 1, 2, 3
OPS = {"tanh": 0, "sigmoid": 1, "swish": 2, "gelu": 3}
DTYPES = {"bf16": 0, "f32": 1}

MAP_CALLS = ("ktanh_bf16", "ktanh_f32", "ksigmoid_bf16", "ksigmoid_f32",
             "kswish_bf16", "kswish_f32", "kgelu_bf16", "kgelu_f32", "ktanh_f32_via_bf16")
BWD_CALLS = ("ktanh_bwd_bf16", "ktanh_bwd_f32", "ksigmoid_bwd_bf16", "ksigmoid_bwd_f32")
BWD_LUT_CALLS = ("kswish_bwd_bf16", "kswish_bwd_f32", "kgelu_bwd_bf16", "kgelu_bwd_f32")
EXPORTS = MAP_CALLS + BWD_CALLS + BWD_LUT_CALLS + ("kt_apply_bwd", "kt_lut_create", "kt_lut_create_paper", "kt_lut_get", "kt_lut_destroy",
                       "kt_lut_create_f32", "kt_lut_mantissa_bits", "kt_lut_create_optimized",
                       "kt_lut64_create_optimized",
                       "klstm_gates_bf16", "klstm_cell_bf16", "kgemm_bf16", "kt_apply", "kt_apply_host", "kt_shard_range",
                       "kt_status_string", "kt_last_error", "kt_abi_version", "kt_launch_count",
                       "kt_apx_create", "kt_apx_coeffs", "kt_apx_destroy", "kt_apx_tanh_bf16",
                       "kt_apx_tanh_f32", "kt_alu_probe", "kgelu_swish_bf16", "kgelu_swish_f32",
                       "kgemm_lstm_gates_bf16", "kgemm_lstm_cell_bf16", "kt_lut64_create",
                       "kt_lut64_get", "kt_lut64_destroy", "ktanh64_bf16", "kt_apply_host_ex")

for _name in MAP_CALLS:
    _f = getattr(_lib, _name)
    _f.argtypes = [_vp, _vp, _sz, _vp, _vp]
    _f.restype = ctypes.c_int
for _name in BWD_CALLS:
    _f = getattr(_lib, _name)
    _f.argtypes = [_vp, _vp, _vp, _sz, _vp]
    _f.restype = ctypes.c_int
for _name in BWD_LUT_CALLS:
    _f = getattr(_lib, _name)
    _f.argtypes = [_vp, _vp, _vp, _sz, _vp, _vp]
    _f.restype = ctypes.c_int
_lib.kt_apply_bwd.argtypes = [ctypes.c_int, ctypes.c_int, _vp, _vp, _vp, _sz, _vp, _vp]
_lib.kt_apply_bwd.restype = ctypes.c_int
_lib.kt_lut_create.argtypes = [_c_i32p, _c_i32p, _c_i32p, ctypes.POINTER(_vp)]
_lib.kt_lut_create.restype = ctypes.c_int
_lib.kt_lut_create_f32.argtypes = [_c_i32p, _c_i32p, _c_i32p, ctypes.POINTER(_vp)]
_lib.kt_lut_create_f32.restype = ctypes.c_int
_lib.kt_lut_mantissa_bits.argtypes = [_vp, ctypes.POINTER(ctypes.c_int32)]
_lib.kt_lut_mantissa_bits.restype = ctypes.c_int
_lib.kt_lut_create_optimized.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_vp)]
_lib.kt_lut_create_optimized.restype = ctypes.c_int
_lib.kt_lut64_create_optimized.argtypes = [ctypes.c_int32, ctypes.POINTER(_vp)]
_lib.kt_lut64_create_optimized.restype = ctypes.c_int
_lib.kt_lut_create_paper.argtypes = [ctypes.POINTER(_vp)]
_lib.kt_lut_create_paper.restype = ctypes.c_int
_lib.kt_lut_get.argtypes = [_vp, _c_i32p, _c_i32p, _c_i32p]
_lib.kt_lut_get.restype = ctypes.c_int
_lib.kt_lut_destroy.argtypes = [_vp]
_lib.kt_lut_destroy.restype = None
_lib.klstm_gates_bf16.argtypes = [_vp, _vp, _sz, _sz, ctypes.c_int, _vp, _vp]
_lib.klstm_gates_bf16.restype = ctypes.c_int
_lib.klstm_cell_bf16.argtypes = [_vp, _vp, _vp, _vp, _sz, _sz, _vp, _vp]
_lib.klstm_cell_bf16.restype = ctypes.c_int
_lib.kgemm_bf16.argtypes = [_vp, _vp, _vp, _sz, _sz, _sz, ctypes.c_int, _vp, _vp]
_lib.kgemm_bf16.restype = ctypes.c_int
_lib.kt_apply.argtypes = [ctypes.c_int, ctypes.c_int, _vp, _vp, _sz, _vp, _vp]
_lib.kt_apply.restype = ctypes.c_int
_lib.kt_apply_host.argtypes = [ctypes.c_int, ctypes.c_int, _vp, _vp, _sz, _vp, _vp, _sz, _vp]
_lib.kt_apply_host.restype = ctypes.c_int
_lib.kt_apply_host_ex.argtypes = [ctypes.c_int, ctypes.c_int, _vp, _vp, _sz, _vp, _vp, _sz, _sz, _vp]
_lib.kt_apply_host_ex.restype = ctypes.c_int
_lib.kt_shard_range.argtypes = [_sz, ctypes.c_int, ctypes.c_int, _sz, ctypes.POINTER(_sz),
                                ctypes.POINTER(_sz)]
_lib.kt_shard_range.restype = ctypes.c_int
_lib.kt_status_string.argtypes = [ctypes.c_int]
_lib.kt_status_string.restype = ctypes.c_char_p
_lib.kt_last_error.argtypes = []
_lib.kt_last_error.restype = ctypes.c_char_p
_lib.kt_abi_version.argtypes = []
_lib.kt_abi_version.restype = ctypes.c_int
_lib.kt_launch_count.argtypes = []
_lib.kt_launch_count.restype = ctypes.c_uint64
_lib.kt_apx_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]
_lib.kt_apx_create.restype = ctypes.c_int
_lib.kt_apx_coeffs.argtypes = [_vp, ctypes.POINTER(ctypes.c_double)]
_lib.kt_apx_coeffs.restype = ctypes.c_int
_lib.kt_apx_destroy.argtypes = [_vp]
_lib.kt_apx_destroy.restype = None
for _name in ("kt_apx_tanh_bf16", "kt_apx_tanh_f32"):
    _f = getattr(_lib, _name)
    _f.argtypes = [_vp, _vp, _sz, _vp, _vp]
    _f.restype = ctypes.c_int

for _name in ("kgelu_swish_bf16", "kgelu_swish_f32"):
    _f = getattr(_lib, _name)
    _f.argtypes = [_vp, _vp, _vp, _sz, _vp, _vp]
    _f.restype = ctypes.c_int
_lib.kt_lut64_create.argtypes = [_c_i32p, _c_i32p, _c_i32p, ctypes.POINTER(_vp)]
_lib.kt_lut64_create.restype = ctypes.c_int
_lib.kt_lut64_get.argtypes = [_vp, _c_i32p, _c_i32p, _c_i32p]
_lib.kt_lut64_get.restype = ctypes.c_int
_lib.kt_lut64_destroy.argtypes = [_vp]
_lib.kt_lut64_destroy.restype = None
_lib.ktanh64_bf16.argtypes = [_vp, _vp, _sz, _vp, _vp]
_lib.ktanh64_bf16.restype = ctypes.c_int
_lib.kgemm_lstm_gates_bf16.argtypes = [_vp, _vp, _vp, _sz, _sz, _sz, ctypes.c_int, _vp, _vp]
_lib.kgemm_lstm_gates_bf16.restype = ctypes.c_int
_lib.kgemm_lstm_cell_bf16.argtypes = [_vp, _vp, _vp, _vp, _vp, _sz, _sz, _sz, _vp, _vp]
_lib.kgemm_lstm_cell_bf16.restype = ctypes.c_int
_lib.kt_alu_probe.argtypes = [ctypes.c_int, _vp, _vp, _vp, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
_lib.kt_alu_probe.restype = ctypes.c_int

APX_KINDS = {"pade": 0, "minimax": 1, "taylor": 2, "libm": 3, "sfu": 4}
APX_NCOEF = 65


class KTanhError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.kt_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_lib.kt_status_string(status).decode()}: {msg}")


def _check(status: int, where: str):
    if status != KT_OK:
        raise KTanhError(status, where)


def abi_version() -> int:
    return _lib.kt_abi_version()


def launch_count() -> int:
    """Kernel launches issued by the library in this process."""
    return int(_lib.kt_launch_count())


# ---- parameter-table serialization (SURVEY.md §8(b) "a JSON table format") --
# {format, exp_lsb_bits, man_msb_bits, b_unit_bits, t1_bits, t2_bits, E, r, b,
#  provenance}; fixed key order and formatting, so equal tables give
# byte-identical text.  Host-side marshalling only: the handle is created
# (and validated) by the C ABI.

def _table_json(fmt, s_bits, b_unit, E, r, b, provenance):
    import json
    t1, t2 = ("0x3E80", "0x4070") if fmt == "bfloat16" else ("0x3E800000", "0x40700000")
    doc = {"format": fmt, "exp_lsb_bits": 2, "man_msb_bits": s_bits, "b_unit_bits": b_unit,
           "t1_bits": t1, "t2_bits": t2, "E": [int(v) for v in E], "r": [int(v) for v in r],
           "b": [int(v) for v in b], "provenance": str(provenance)}
    return json.dumps(doc, indent=None, separators=(", ", ": ")) + "\n"


def _table_dump(s_bits, E, r, b):
    """Table 1's layout: index bit string, E_t, r_t, b_t."""
    nb = 2 + s_bits
    return "".join(f"{t:0{nb}b} {E[t]:4d} {r[t]:3d} {b[t]:9d}\n" for t in range(len(E)))


def lut_from_json(text: str):
    """Lut (32 entries; format bfloat16 with b_unit_bits 7, or float32 with
    b_unit_bits 23) or Lut64 (man_msb_bits 4) from the JSON table format."""
    import json
    d = json.loads(text)
    fmt, s_bits, unit = d["format"], int(d["man_msb_bits"]), int(d.get("b_unit_bits", 7))
    if int(d.get("exp_lsb_bits", 2)) != 2:
        raise ValueError("exp_lsb_bits must be 2 (Alg. 1 line 6)")
    E, r, b = d["E"], d["r"], d["b"]
    if fmt == "bfloat16" and unit == 7 and s_bits == 3:
        return Lut.from_tables(E, r, b)
    if fmt == "bfloat16" and unit == 7 and s_bits == 4:
        return Lut64(E, r, b)
    if fmt == "float32" and unit == 23 and s_bits == 3:
        return Lut.from_tables_f32(E, r, b)
    raise ValueError(f"unsupported table: format={fmt} man_msb_bits={s_bits} b_unit_bits={unit}")


class Lut:
    """Immutable parameter-table handle (T_E, T_r, T_b), Alg. 1 line 1."""

    def __init__(self, handle: int):
        self._h = _vp(handle)

    @classmethod
    def paper(cls) -> "Lut":
        """Table 1 of the paper."""
        h = _vp()
        _check(_lib.kt_lut_create_paper(ctypes.byref(h)), "kt_lut_create_paper")
        return cls(h.value)

    @classmethod
    def from_tables(cls, E, r, b) -> "Lut":
        arr = [(ctypes.c_int32 * 32)(*[int(v) for v in a]) for a in (E, r, b)]
        if any(len(a) != 32 for a in (E, r, b)):
            raise ValueError("tables must have 32 entries")
        h = _vp()
        _check(_lib.kt_lut_create(arr[0], arr[1], arr[2], ctypes.byref(h)), "kt_lut_create")
        return cls(h.value)

    @classmethod
    def optimized(cls, p: int = 7, bmin_zero: bool = False) -> "Lut":
        """Sec. 2.4 optimizer in the library: p = 7 (BF16) or 23 (F32-native)."""
        h = _vp()
        _check(_lib.kt_lut_create_optimized(int(p), int(bmin_zero), ctypes.byref(h)),
               "kt_lut_create_optimized")
        return cls(h.value)

    @classmethod
    def from_tables_f32(cls, E, r, b) -> "Lut":
        """F32-only table with b in 2^-23 units (re-optimised at p = 23, NEXT-3)."""
        if any(len(a) != 32 for a in (E, r, b)):
            raise ValueError("tables must have 32 entries")
        arr = [(ctypes.c_int32 * 32)(*[int(v) for v in a]) for a in (E, r, b)]
        h = _vp()
        _check(_lib.kt_lut_create_f32(arr[0], arr[1], arr[2], ctypes.byref(h)), "kt_lut_create_f32")
        return cls(h.value)

    def tables(self):
        E, r, b = ((ctypes.c_int32 * 32)() for _ in range(3))
        _check(_lib.kt_lut_get(self._h, E, r, b), "kt_lut_get")
        return list(E), list(r), list(b)

    def to_json(self, provenance: str = "") -> str:
        fmt = "bfloat16" if self.p == 7 else "float32"
        return _table_json(fmt, 3, self.p, *self.tables(), provenance)

    def dump(self) -> str:
        return _table_dump(3, *self.tables())

    @property
    def p(self) -> int:
        """Unit of b: 7 (BF16 tables) or 23 (F32-only tables)."""
        v = ctypes.c_int32()
        _check(_lib.kt_lut_mantissa_bits(self._h, ctypes.byref(v)), "kt_lut_mantissa_bits")
        return v.value

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = globals().get("_lib")
        if h is not None and h.value and lib is not None:
            lib.kt_lut_destroy(h)
            self._h = _vp()


_default_lut = None


def paper_lut() -> Lut:
    global _default_lut
    if _default_lut is None:
        _default_lut = Lut.paper()
    return _default_lut


def _stream_ptr(stream, device_index=None):
    import torch
    if stream is None:
        if device_index is None:
            device_index = torch.cuda.current_device()
        return torch._C._cuda_getCurrentRawStream(device_index)
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class _on_device:
    """Make x's device current for the call only if it is not already."""
    __slots__ = ("idx", "prev")

    def __init__(self, idx):
        self.idx = idx
        self.prev = None

    def __enter__(self):
        import torch
        cur = torch.cuda.current_device()
        if cur != self.idx:
            self.prev = cur
            torch.cuda.set_device(self.idx)
        return self

    def __exit__(self, *a):
        if self.prev is not None:
            import torch
            torch.cuda.set_device(self.prev)


def _prep(x, out, dtype):
    import torch
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError("x must be a CUDA tensor (no CPU path)")
    if x.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {x.dtype}")
    if not x.is_contiguous():
        raise ValueError("x must be contiguous")
    if out is None:
        out = torch.empty_like(x)
    elif (out.dtype != dtype or not out.is_cuda or not out.is_contiguous()
          or out.numel() != x.numel() or out.device != x.device):
        raise ValueError("out must be a contiguous CUDA tensor like x")
    return out


def _check_out(t, name, dtype, numel, device):
    """Validate a caller-supplied output tensor: the C ABI only sees a raw
    pointer and cannot bound-check it."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.device != device:
        raise TypeError(f"{name} must be a CUDA tensor on {device}")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous() or t.numel() != numel:
        raise ValueError(f"{name} must be contiguous with {numel} elements")
    return t


def _fmt_of(dtype):
    """'bf16' / 'f32' for the two formats the library has; TypeError otherwise."""
    import torch
    if dtype == torch.bfloat16:
        return "bf16"
    if dtype == torch.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {dtype}: the library has BF16 and FP32 paths only")


def _make_call(name, dtype_name):
    fn = getattr(_lib, name)

    def call(x, out=None, lut: Lut | None = None, stream=None):
        import torch
        dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
        out = _prep(x, out, dt)
        lut = lut or paper_lut()
        idx = x.device.index
        with _on_device(idx):
            _check(fn(x.data_ptr(), out.data_ptr(), x.numel(), lut.handle, _stream_ptr(stream, idx)),
                   name)
        return out

    call.__name__ = name
    call.__doc__ = f"{name}(x, out=None, lut=None, stream=None) -> out   (C ABI: include/ktanh.h)"
    return call


ktanh_bf16 = _make_call("ktanh_bf16", "bf16")
ktanh_f32 = _make_call("ktanh_f32", "f32")
ksigmoid_bf16 = _make_call("ksigmoid_bf16", "bf16")
ksigmoid_f32 = _make_call("ksigmoid_f32", "f32")
kswish_bf16 = _make_call("kswish_bf16", "bf16")
kswish_f32 = _make_call("kswish_f32", "f32")
kgelu_bf16 = _make_call("kgelu_bf16", "bf16")
kgelu_f32 = _make_call("kgelu_f32", "f32")
ktanh_f32_via_bf16 = _make_call("ktanh_f32_via_bf16", "f32")


def _make_bwd(name, dtype_name, needs_lut):
    fn = getattr(_lib, name)

    def call(a, dy, out=None, lut: Lut | None = None, stream=None):
        """dx = dy * g(a); a = saved output (tanh, sigmoid) or input x (swish, gelu)."""
        import torch
        dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
        out = _prep(a, out, dt)
        _prep(dy, out, dt)
        if dy.numel() != a.numel():
            raise ValueError("a and dy must have the same number of elements")
        idx = a.device.index
        with _on_device(idx):
            if needs_lut:
                lut = lut or paper_lut()
                st = fn(a.data_ptr(), dy.data_ptr(), out.data_ptr(), a.numel(), lut.handle,
                        _stream_ptr(stream, idx))
            else:
                st = fn(a.data_ptr(), dy.data_ptr(), out.data_ptr(), a.numel(),
                        _stream_ptr(stream, idx))
            _check(st, name)
        return out

    call.__name__ = name
    return call


ktanh_bwd_bf16 = _make_bwd("ktanh_bwd_bf16", "bf16", False)
ktanh_bwd_f32 = _make_bwd("ktanh_bwd_f32", "f32", False)
ksigmoid_bwd_bf16 = _make_bwd("ksigmoid_bwd_bf16", "bf16", False)
ksigmoid_bwd_f32 = _make_bwd("ksigmoid_bwd_f32", "f32", False)
kswish_bwd_bf16 = _make_bwd("kswish_bwd_bf16", "bf16", True)
kswish_bwd_f32 = _make_bwd("kswish_bwd_f32", "f32", True)
kgelu_bwd_bf16 = _make_bwd("kgelu_bwd_bf16", "bf16", True)
kgelu_bwd_f32 = _make_bwd("kgelu_bwd_f32", "f32", True)


def klstm_gates_bf16(x, hidden: int, tanh_quarter: int = 2, out=None, lut: Lut | None = None,
                     stream=None):
    """[..., 4*hidden] BF16 gate block: K-TanH on quarter `tanh_quarter`, K-Sigmoid elsewhere."""
    import torch
    out = _prep(x, out, torch.bfloat16)
    if x.numel() % (4 * hidden):
        raise ValueError("numel must be a multiple of 4*hidden")
    lut = lut or paper_lut()
    with torch.cuda.device(x.device):
        _check(_lib.klstm_gates_bf16(x.data_ptr(), out.data_ptr(), x.numel() // (4 * hidden),
                                     hidden, tanh_quarter, lut.handle, _stream_ptr(stream)),
               "klstm_gates_bf16")
    return out


def klstm_cell_bf16(gates, c_prev, hidden: int, c_next=None, h_next=None,
                    lut: Lut | None = None, stream=None):
    """Fused LSTM cell: gates [..., 4*hidden] BF16, c_prev [..., hidden] F32 ->
    (c_next F32, h_next BF16).  c_next may be c_prev (in place)."""
    import torch
    if not (gates.is_cuda and c_prev.is_cuda) or gates.dtype != torch.bfloat16 \
            or c_prev.dtype != torch.float32:
        raise TypeError("gates: CUDA bfloat16, c_prev: CUDA float32")
    if not (gates.is_contiguous() and c_prev.is_contiguous()):
        raise ValueError("inputs must be contiguous")
    rows = c_prev.numel() // hidden
    if c_prev.numel() != rows * hidden or gates.numel() != rows * 4 * hidden:
        raise ValueError("shapes: gates [rows, 4*hidden], c_prev [rows, hidden]")
    if gates.device != c_prev.device:
        raise ValueError("gates and c_prev must be on the same device")
    if c_next is None:
        c_next = torch.empty_like(c_prev)
    _check_out(c_next, "c_next", torch.float32, rows * hidden, c_prev.device)
    if h_next is None:
        h_next = torch.empty(c_prev.shape, dtype=torch.bfloat16, device=c_prev.device)
    _check_out(h_next, "h_next", torch.bfloat16, rows * hidden, c_prev.device)
    lut = lut or paper_lut()
    idx = gates.device.index
    with _on_device(idx):
        _check(_lib.klstm_cell_bf16(gates.data_ptr(), c_prev.data_ptr(), c_next.data_ptr(),
                                    h_next.data_ptr(), rows, hidden, lut.handle,
                                    _stream_ptr(stream, idx)), "klstm_cell_bf16")
    return c_next, h_next


def kgemm_bf16(A, B, epilogue: str | None = None, out=None, lut: Lut | None = None, stream=None):
    """C = act(A @ B.T) on tcgen05 tensor cores; A [M, K], B [N, K] BF16 CUDA
    tensors, act in {None, "tanh", "sigmoid", "swish", "gelu"}."""
    import torch
    if not (A.is_cuda and B.is_cuda) or A.dtype != torch.bfloat16 or B.dtype != torch.bfloat16:
        raise TypeError("A, B must be CUDA bfloat16 tensors")
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[1]:
        raise ValueError("A [M, K], B [N, K]")
    if not (A.is_contiguous() and B.is_contiguous()):
        raise ValueError("A, B must be contiguous")
    if A.device != B.device:
        raise ValueError("A and B must be on the same device")
    M, K = A.shape
    N = B.shape[0]
    if out is None:
        out = torch.empty(M, N, dtype=torch.bfloat16, device=A.device)
    _check_out(out, "out", torch.bfloat16, M * N, A.device)
    epi = -1 if epilogue is None else OPS[epilogue]
    lut = lut or paper_lut()
    idx = A.device.index
    with _on_device(idx):
        _check(_lib.kgemm_bf16(A.data_ptr(), B.data_ptr(), out.data_ptr(), M, N, K, epi, lut.handle,
                               _stream_ptr(stream, idx)), "kgemm_bf16")
    return out


def apply(op: str, x, out=None, lut: Lut | None = None, stream=None):
    """Generic kt_apply dispatch by op name and the tensor's dtype."""
    import torch
    dname = _fmt_of(x.dtype)
    out = _prep(x, out, x.dtype)
    lut = lut or paper_lut()
    with torch.cuda.device(x.device):
        _check(_lib.kt_apply(OPS[op], DTYPES[dname], x.data_ptr(), out.data_ptr(), x.numel(),
                             lut.handle, _stream_ptr(stream)), "kt_apply")
    return out


def apply_host(op: str, x_host, y_host, work, lut: Lut | None = None, stream=None,
               chunk: int = 0):
    """kt_apply_host(_ex): x_host/y_host are (pinned) CPU tensors, `work` a CUDA
    uint8 scratch tensor on the current device, `chunk` elements per pipeline
    chunk (0 = default).  Asynchronous on `stream`."""
    import torch
    dname = _fmt_of(x_host.dtype)
    if x_host.dtype != y_host.dtype or x_host.numel() != y_host.numel():
        raise ValueError("x_host and y_host must match")
    if not (x_host.is_contiguous() and y_host.is_contiguous()):
        raise ValueError("x_host and y_host must be contiguous")
    if x_host.is_cuda or y_host.is_cuda or not work.is_cuda:
        raise TypeError("x_host / y_host must be CPU tensors, work a CUDA tensor")
    if not work.is_contiguous():
        raise ValueError("work must be contiguous")
    if stream is None and work.device.index != torch.cuda.current_device():
        raise ValueError("work must be on the current CUDA device (or pass its stream)")
    lut = lut or paper_lut()
    with torch.cuda.device(work.device):
        _check(_lib.kt_apply_host_ex(OPS[op], DTYPES[dname], x_host.data_ptr(), y_host.data_ptr(),
                                     x_host.numel(), lut.handle, work.data_ptr(),
                                     work.numel() * work.element_size(), int(chunk),
                                     _stream_ptr(stream)),
               "kt_apply_host_ex")
    return y_host


def shard_range(n: int, world: int, rank: int, align: int = 16):
    """kt_shard_range: (begin, count) of rank's contiguous shard."""
    b, c = _sz(), _sz()
    _check(_lib.kt_shard_range(n, world, rank, align, ctypes.byref(b), ctypes.byref(c)),
           "kt_shard_range")
    return b.value, c.value


# ---------------------------------------------------------------------------
# Table 2 comparators (include/ktanh.h "Table 2 comparators")
# ---------------------------------------------------------------------------
class Apx:
    """Immutable float-op TanH approximation handle (kt_apx_create):
    kind in APX_KINDS; (p, q) = Pade orders, or (degree, 0) for minimax/taylor."""

    def __init__(self, kind: str, p: int = 0, q: int = 0):
        if kind not in APX_KINDS:
            raise ValueError(f"kind must be one of {sorted(APX_KINDS)}")
        self.kind, self.p, self.q = kind, p, q
        h = _vp()
        _check(_lib.kt_apx_create(APX_KINDS[kind], p, q, ctypes.byref(h)), "kt_apx_create")
        self._h = h

    def coeffs(self):
        """Binary64 coefficient block (layout: KT_APX_NCOEF in include/ktanh.h)."""
        c = (ctypes.c_double * APX_NCOEF)()
        _check(_lib.kt_apx_coeffs(self._h, c), "kt_apx_coeffs")
        return list(c)

    @property
    def handle(self):
        return self._h

    def __repr__(self):
        return f"Apx({self.kind!r}, {self.p}, {self.q})"

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = globals().get("_lib")
        if h is not None and h.value and lib is not None:
            lib.kt_apx_destroy(h)
            self._h = _vp()


def _make_apx_call(name, dtype_name):
    fn = getattr(_lib, name)

    def call(x, apx: Apx, out=None, stream=None):
        import torch
        dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
        out = _prep(x, out, dt)
        idx = x.device.index
        with _on_device(idx):
            _check(fn(x.data_ptr(), out.data_ptr(), x.numel(), apx.handle, _stream_ptr(stream, idx)),
                   name)
        return out

    call.__name__ = name
    call.__doc__ = f"{name}(x, apx, out=None, stream=None) -> out   (C ABI: include/ktanh.h)"
    return call


kt_apx_tanh_bf16 = _make_apx_call("kt_apx_tanh_bf16", "bf16")
kt_apx_tanh_f32 = _make_apx_call("kt_apx_tanh_f32", "f32")


def alu_probe(dtype: str, sample, lut: Lut | None = None, apx: Apx | None = None,
              iters: int = 256):
    """kt_alu_probe: (net, gross) SM cycles per element per SM of K-TanH (lut)
    or a comparator (apx), register-resident.  `sample`: 4096 uint32 words
    (numpy) -- BF16 pairs or F32 bit patterns.  Synchronous."""
    import numpy as np
    words = np.ascontiguousarray(sample, dtype=np.uint32)
    if words.size != 4096:
        raise ValueError("sample must hold 4096 words")
    if (lut is None) == (apx is None):
        raise ValueError("pass exactly one of lut, apx")
    net, gross = ctypes.c_double(), ctypes.c_double()
    _check(_lib.kt_alu_probe(DTYPES[dtype], lut.handle if lut else None,
                             apx.handle if apx else None, words.ctypes.data, iters,
                             ctypes.byref(net), ctypes.byref(gross)), "kt_alu_probe")
    return net.value, gross.value


def _make_dual(name, dtype_name):
    fn = getattr(_lib, name)

    def call(x, out_gelu=None, out_swish=None, lut: Lut | None = None, stream=None):
        """(K-GELU(x), K-Swish(x)) in one pass over x (config 5, reading A20)."""
        import torch
        dt = torch.bfloat16 if dtype_name == "bf16" else torch.float32
        out_gelu = _prep(x, out_gelu, dt)
        out_swish = _prep(x, out_swish, dt)
        lut = lut or paper_lut()
        idx = x.device.index
        with _on_device(idx):
            _check(fn(x.data_ptr(), out_gelu.data_ptr(), out_swish.data_ptr(), x.numel(), lut.handle,
                      _stream_ptr(stream, idx)), name)
        return out_gelu, out_swish

    call.__name__ = name
    return call


kgelu_swish_bf16 = _make_dual("kgelu_swish_bf16", "bf16")
kgelu_swish_f32 = _make_dual("kgelu_swish_f32", "f32")


def kgemm_lstm_gates_bf16(A, B, hidden: int, tanh_quarter: int = 2, out=None, lut: Lut | None = None,
                          stream=None):
    """LSTM gate GEMM with fused gate activations: A [M, K], B [4*hidden, K]
    (BF16 CUDA) -> K-Sigmoid / K-TanH(RN_bf16(A @ B.T)) per quarter."""
    import torch
    if not (A.is_cuda and B.is_cuda) or A.dtype != torch.bfloat16 or B.dtype != torch.bfloat16:
        raise TypeError("A, B must be CUDA bfloat16 tensors")
    if A.dim() != 2 or B.dim() != 2 or A.shape[1] != B.shape[1] or B.shape[0] != 4 * hidden:
        raise ValueError("A [M, K], B [4*hidden, K]")
    if not (A.is_contiguous() and B.is_contiguous()):
        raise ValueError("A, B must be contiguous")
    if A.device != B.device:
        raise ValueError("A and B must be on the same device")
    M, K = A.shape
    if out is None:
        out = torch.empty(M, 4 * hidden, dtype=torch.bfloat16, device=A.device)
    _check_out(out, "out", torch.bfloat16, M * 4 * hidden, A.device)
    lut = lut or paper_lut()
    idx = A.device.index
    with _on_device(idx):
        _check(_lib.kgemm_lstm_gates_bf16(A.data_ptr(), B.data_ptr(), out.data_ptr(), M, hidden, K,
                                          tanh_quarter, lut.handle, _stream_ptr(stream, idx)),
               "kgemm_lstm_gates_bf16")
    return out


def kgemm_lstm_cell_bf16(A, B, c_prev, hidden: int, c_next=None, h_next=None, lut: Lut | None = None,
                         stream=None):
    """Gate GEMM + fused LSTM cell: A [M, K], B [4*hidden, K] (i,f,g,o row
    blocks) BF16, c_prev [M, hidden] F32 -> (c_next F32, h_next BF16)."""
    import torch
    if not (A.is_cuda and B.is_cuda and c_prev.is_cuda) or A.dtype != torch.bfloat16 \
            or B.dtype != torch.bfloat16 or c_prev.dtype != torch.float32:
        raise TypeError("A, B: CUDA bfloat16; c_prev: CUDA float32")
    M, K = A.shape
    if B.shape != (4 * hidden, K) or c_prev.numel() != M * hidden:
        raise ValueError("A [M, K], B [4*hidden, K], c_prev [M, hidden]")
    if not (A.is_contiguous() and B.is_contiguous() and c_prev.is_contiguous()):
        raise ValueError("inputs must be contiguous")
    if not (A.device == B.device == c_prev.device):
        raise ValueError("A, B and c_prev must be on the same device")
    if c_next is None:
        c_next = torch.empty_like(c_prev)
    _check_out(c_next, "c_next", torch.float32, M * hidden, A.device)
    if h_next is None:
        h_next = torch.empty(c_prev.shape, dtype=torch.bfloat16, device=c_prev.device)
    _check_out(h_next, "h_next", torch.bfloat16, M * hidden, A.device)
    lut = lut or paper_lut()
    idx = A.device.index
    with _on_device(idx):
        _check(_lib.kgemm_lstm_cell_bf16(A.data_ptr(), B.data_ptr(), c_prev.data_ptr(),
                                         c_next.data_ptr(), h_next.data_ptr(), M, hidden, K,
                                         lut.handle, _stream_ptr(stream, idx)), "kgemm_lstm_cell_bf16")
    return c_next, h_next


class Lut64:
    """64-interval parameter table, for ktanh64_bf16."""

    def __init__(self, E, r, b):
        if any(len(a) != 64 for a in (E, r, b)):
            raise ValueError("tables must have 64 entries")
        arr = [(ctypes.c_int32 * 64)(*[int(v) for v in a]) for a in (E, r, b)]
        h = _vp()
        _check(_lib.kt_lut64_create(arr[0], arr[1], arr[2], ctypes.byref(h)), "kt_lut64_create")
        self._h = h

    @classmethod
    def optimized(cls, bmin_zero: bool = False) -> "Lut64":
        """Sec. 2.4 optimizer with 4 mantissa index bits (64 intervals)."""
        self = cls.__new__(cls)
        h = _vp()
        _check(_lib.kt_lut64_create_optimized(int(bmin_zero), ctypes.byref(h)),
               "kt_lut64_create_optimized")
        self._h = h
        return self

    def tables(self):
        E, r, b = ((ctypes.c_int32 * 64)() for _ in range(3))
        _check(_lib.kt_lut64_get(self._h, E, r, b), "kt_lut64_get")
        return list(E), list(r), list(b)

    def to_json(self, provenance: str = "") -> str:
        return _table_json("bfloat16", 4, 7, *self.tables(), provenance)

    def dump(self) -> str:
        return _table_dump(4, *self.tables())

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        lib = globals().get("_lib")
        if h is not None and h.value and lib is not None:
            lib.kt_lut64_destroy(h)
            self._h = _vp()


def ktanh64_bf16(x, lut64: Lut64, out=None, stream=None):
    """K-TanH on BF16 with a 64-interval table (C ABI ktanh64_bf16)."""
    import torch
    out = _prep(x, out, torch.bfloat16)
    idx = x.device.index
    with _on_device(idx):
        _check(_lib.ktanh64_bf16(x.data_ptr(), out.data_ptr(), x.numel(), lut64.handle,
                                 _stream_ptr(stream, idx)), "ktanh64_bf16")
    return out
