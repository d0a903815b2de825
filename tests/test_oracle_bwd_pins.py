"""Pins of the oracle's backward passes (reading R-BWD).

The paper never states the gradient it trained GNMT with;
R-BWD takes the derivative of the approximated function through the K-TanH
value.  The pins below check the oracle against closed forms and against the
TRUE derivatives of tanh / sigmoid / swish / tanh-GELU within bounds derived
from Table 2's error bound eps = 1.67e-2, plus invariants.
"""
import math

import numpy as np

import oracle as O
from conftest import read_golden

W = O.all_bf16()
XV = O.bf16_to_f64(W)
FIN = np.isfinite(XV)
ONE = np.full(W.shape, 0x3F80, np.uint16)          # dy = 1
EPS = 0.0167


def f(w):
    return O.bf16_to_f64(w)


def test_tanh_bwd_closed_forms_and_bound():
    y = O.map_bf16("tanh", W)
    g = f(O.bwd_bf16("tanh", y, ONE))
    sat = FIN & (np.abs(XV) > 3.75)
    assert np.all(g[sat] == 0.0)                    # y = +-1  ->  1 - y^2 = 0
    assert g[0] == 1.0                              # tanh'(0) = 1
    true = 1 - np.tanh(XV[FIN]) ** 2
    # |(1-y^2) - (1-tanh^2)| = |tanh - y| |tanh + y| <= 2 eps, plus output rounding
    assert np.max(np.abs(g[FIN] - true)) <= 2 * EPS + 2 ** -8
    # even in y, odd in dy
    nn = ~np.isnan(XV)
    assert np.array_equal(O.bwd_bf16("tanh", y ^ 0x8000, ONE)[nn], O.bwd_bf16("tanh", y, ONE)[nn])
    assert np.array_equal(O.bwd_bf16("tanh", y, ONE ^ 0x8000)[nn],
                          (O.bwd_bf16("tanh", y, ONE) ^ 0x8000)[nn])


def test_sigmoid_bwd_bound():
    s = O.map_bf16("sigmoid", W)
    g = f(O.bwd_bf16("sigmoid", s, ONE))
    assert g[0] == 0.25                             # sigma'(0) = 1/4 (s = 1/2 exactly)
    sig = 1 / (1 + np.exp(-XV[FIN]))
    true = sig * (1 - sig)
    # |s(1-s) - sig(1-sig)| <= |s - sig| (|1 - s - sig|) <= eps/2 + rounding
    assert np.max(np.abs(g[FIN] - true)) <= EPS / 2 + 2 ** -9 + 2 ** -9


def test_swish_bwd_bound():
    g = f(O.bwd_bf16("swish", W, ONE))
    assert g[0] == 0.5                              # swish'(0) = 1/2
    m = FIN & (np.abs(XV) <= 32)
    x = XV[m]
    sig = 1 / (1 + np.exp(-x))
    true = sig + x * sig * (1 - sig)
    h = np.array([O.bf16_decode(O.bf16_encode_rne(v / 2)) for v in x])
    # t differs from tanh(x/2) by <= eps + |h - x/2|; the swish derivative in t is
    # 1/2 + (x/4)(-2t): |dg| <= (1/2 + |x|/2)(eps + |h - x/2|) + output rounding
    bound = (0.5 + np.abs(x) / 2) * (EPS + np.abs(h - x / 2)) + np.abs(true) * 2 ** -8 + 1e-12
    assert np.all(np.abs(g[m] - true) <= bound)


def test_gelu_bwd_closed_forms_and_bound():
    a = float(read_golden("gelu_a.txt")[0][1])
    g = f(O.bwd_bf16("gelu", W, ONE))
    assert g[0] == 0.5                              # GELU'(0) = 1/2
    assert np.all(g[FIN & (XV > 4)] == 1.0)         # t = 1: (1+1)/2 + 0
    assert np.all(g[FIN & (XV < -4)] == 0.0)        # t = -1: 0 + x/2 * 0
    m = FIN & (np.abs(XV) <= 8)
    x = XV[m]
    c = math.sqrt(2 / math.pi)
    u = c * (x + a * x ** 3)
    th = np.tanh(u)
    up = c * (1 + 3 * a * x ** 2)
    true = 0.5 * (1 + th) + 0.5 * x * (1 - th ** 2) * up
    ub = np.array([O.bf16_decode(O.bf16_encode_rne(v)) for v in u])
    dt = EPS + np.abs(ub - u) + 1e-6 * np.abs(u)
    bound = (0.5 + np.abs(x) * up) * dt + np.abs(true) * 2 ** -8 + 1e-12
    assert np.all(np.abs(g[m] - true) <= bound + 2 ** -8)


def test_bwd_scales_with_dy():
    """dx is linear in dy up to one output rounding: check dy = 2^k exactly scales."""
    rng = np.random.default_rng(0)
    x = W[FIN & (np.abs(XV) < 6) & (np.abs(XV) > 1e-3)]
    x = rng.choice(x, 4000)
    for op, a in (("tanh", O.map_bf16("tanh", x)), ("sigmoid", O.map_bf16("sigmoid", x)),
                  ("swish", x), ("gelu", x)):
        g1 = f(O.bwd_bf16(op, a, np.full(x.shape, 0x3F80, np.uint16)))
        g4 = f(O.bwd_bf16(op, a, np.full(x.shape, 0x4080, np.uint16)))    # dy = 4
        ok = np.abs(g1) > 2.0 ** -120
        assert np.array_equal(g4[ok], 4 * g1[ok]), op


def test_f32_bwd_consistent_with_bf16_on_bf16_inputs():
    """On BF16-exact inputs the F32 backward factor differs from the BF16 one only
    through the F32 K-TanH value (A8 closed form) and the output rounding."""
    x = W[FIN & (np.abs(XV) < 8)]
    x32 = x.astype(np.uint32) << 16
    one32 = np.full(x.shape, 0x3F800000, np.uint32)
    for op in ("swish", "gelu"):
        g16 = f(O.bwd_bf16(op, x, np.full(x.shape, 0x3F80, np.uint16)))
        g32 = O.bwd_f32(op, x32, one32).view(np.float32).astype(np.float64)
        xv = f(x)
        # K-TanH f32 vs bf16 differ by < 2^-8 relative (A8 relation); derivative
        # sensitivity to t is <= 1/2 + |x| u'(x)
        sens = 0.5 + np.abs(xv) * (1 + 0.14 * xv ** 2)
        assert np.all(np.abs(g16 - g32) <= sens * 2 ** -7 + np.abs(g32) * 2 ** -8 + 1e-9), op


def test_gelu_bwd_f32_bypass_transcription():
    """Transcription check of R-BWD for GELU on F32 where K-TanH is the identity
    (|u| < T1, Alg. 1 line 3), so t = u with no table involved:
    g = (1 + u)/2 + (x/2)(1 - u^2) sqrt(2/pi)(1 + 3 a x^2), u from the golden a."""
    a = float(read_golden("gelu_a.txt")[0][1])
    c = math.sqrt(2 / math.pi)
    x = np.linspace(-0.3, 0.3, 4001).astype(np.float32)
    x = x[np.abs(c * (x + a * x.astype(np.float64) ** 3)) < 0.249]
    g = O.bwd_f32("gelu", x.view(np.uint32), np.ones(x.size, np.float32).view(np.uint32))
    g = g.view(np.float32).astype(np.float64)
    xd = x.astype(np.float64)
    u = c * (xd + a * xd ** 3)
    want = 0.5 * (1 + u) + 0.5 * xd * (1 - u * u) * c * (1 + 3 * a * xd ** 2)
    assert np.max(np.abs(g - want)) < 1e-6
