"""Comparison helpers for parity tests (test infrastructure)."""
import numpy as np


def _ordered(w, bits):
    w = np.asarray(w).astype(np.int64)
    sign = 1 << (bits - 1)
    mag = w & (sign - 1)
    return np.where(w & sign, -mag, mag)


def _isnan(w, bits):
    w = np.asarray(w).astype(np.int64)
    if bits == 16:
        return (w & 0x7FFF) > 0x7F80
    return (w & 0x7FFFFFFF) > 0x7F800000


def ulp_dist(a, b, bits):
    """Distance in units in the last place between bit patterns of the same
    format (+0 and -0 are the same point); NaN pairs -> 0, NaN vs number -> huge."""
    na, nb = _isnan(a, bits), _isnan(b, bits)
    d = np.abs(_ordered(a, bits) - _ordered(b, bits))
    d = np.where(na & nb, 0, d)
    d = np.where(na ^ nb, 1 << 40, d)
    return d


def _iszero(w, bits):
    w = np.asarray(w).astype(np.int64)
    return (w & ((1 << (bits - 1)) - 1)) == 0


def assert_bitexact(got, want, bits, nan_by_class=False, zero_by_value=False, ctx=""):
    """Bit-for-bit equality; nan_by_class: any NaN matches any NaN (GPU
    arithmetic canonicalises payloads); zero_by_value: +0 matches -0 (reading
    A21: the sign of a zero result of the derived ops is not specified)."""
    got = np.asarray(got).reshape(-1)
    want = np.asarray(want).reshape(-1)
    assert got.shape == want.shape
    bad = got != want
    if nan_by_class:
        bad &= ~(_isnan(got, bits) & _isnan(want, bits))
    if zero_by_value:
        bad &= ~(_iszero(got, bits) & _iszero(want, bits))
    if bad.any():
        i = np.flatnonzero(bad)[:8]
        raise AssertionError(f"{ctx}: {bad.sum()} mismatches, first at {i.tolist()}: "
                             f"got {[hex(int(v)) for v in got[i]]} want {[hex(int(v)) for v in want[i]]}")


def assert_ulp(got, want, bits, max_ulp, ctx=""):
    d = ulp_dist(np.asarray(got).reshape(-1), np.asarray(want).reshape(-1), bits)
    if (d > max_ulp).any():
        i = np.flatnonzero(d > max_ulp)[:8]
        raise AssertionError(f"{ctx}: {(d > max_ulp).sum()} elements beyond {max_ulp} ulp, "
                             f"first at {i.tolist()}: got {[hex(int(v)) for v in np.asarray(got).reshape(-1)[i]]} "
                             f"want {[hex(int(v)) for v in np.asarray(want).reshape(-1)[i]]}")
    return int(d.max()) if d.size else 0
