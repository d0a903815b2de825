"""Pins of the Table 2 comparator oracle (oracle/apx_oracle.c).

The paper compares K-TanH with Pade, piecewise minimax and Taylor forms of
TanH (Sec. 2.1-2.2, Table 2).  Nothing here
re-types the oracle's formulas: the Maclaurin coefficients are checked
against textbook values, the Pade forms against Lambert's continued fraction
(a different construction) and the contact-order definition, the minimax
pieces against the Chebyshev alternation theorem (a certificate of
optimality) and competing polynomials, the Taylor pieces against finite
differences of tanh, and the evaluation against invariants and error bounds.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from conftest import read_golden

W = O.all_bf16()
XV = O.bf16_to_f64(W)
FIN = np.isfinite(XV)
NANM = np.isnan(XV)

COMPARATORS = [("pade", 3, 2), ("pade", 7, 8), ("minimax", 2, 0), ("minimax", 3, 0),
               ("taylor", 2, 0), ("taylor", 3, 0)]
# Pade orders in the order of Lambert's convergents (j = 1, 2, ...)
PADE_ORDERS = [(1, 0), (1, 2), (3, 2), (3, 4), (5, 4), (5, 6), (7, 6), (7, 8)]


def maclaurin_golden():
    return {int(k): Fraction(int(n), int(d)) for k, n, d in read_golden("tanh_maclaurin.txt")}


def polyval(c, x):
    s = 0.0
    for v in reversed(list(c)):
        s = s * x + v
    return s


# --------------------------------------------------------------------------
# Maclaurin coefficients (the derivatives at zero of PAPER.md:127)
# --------------------------------------------------------------------------
def test_maclaurin_matches_textbook():
    t = O.tanh_maclaurin(15)
    g = maclaurin_golden()
    for k in range(16):
        want = float(g.get(k, 0))
        assert t[k] == pytest.approx(want, rel=1e-13, abs=1e-300), k


def test_maclaurin_series_sums_to_tanh():
    t = O.tanh_maclaurin(15)
    for x in (0.01, 0.05, 0.1):
        assert polyval(t, x) == pytest.approx(math.tanh(x), rel=1e-15)


# --------------------------------------------------------------------------
# Pade [p/q] (Sec. 2.2)
# --------------------------------------------------------------------------
def lambert_cf(j, x):
    """j-th convergent of Lambert's continued fraction
    tanh x = x / (1 + x^2 / (3 + x^2 / (5 + ...)))."""
    v = 2.0 * j - 1.0
    for i in range(j - 1, 0, -1):
        v = (2.0 * i - 1.0) + x * x / v
    return x / v


def test_pade_3_2_closed_form():
    """Pade[3/2] of tanh = x (15 + x^2) / (15 + 6 x^2)."""
    a, b = O.pade(3, 2)
    np.testing.assert_allclose(a, [0, 1, 0, 1 / 15], rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(b, [1, 0, 6 / 15], rtol=1e-14, atol=1e-16)


@pytest.mark.parametrize("j,pq", list(enumerate(PADE_ORDERS, 1)))
def test_pade_equals_lambert_convergent(j, pq):
    """The Pade approximants of tanh on the staircase [2m-1/2m-2], [2m-1/2m]
    are the convergents of Lambert's continued fraction."""
    a, b = O.pade(*pq)
    for x in (0.1, 0.7, 1.9, 3.3, 6.0, 11.0):
        assert polyval(a, x) / polyval(b, x) == pytest.approx(lambert_cf(j, x), rel=1e-13)


@pytest.mark.parametrize("pq", PADE_ORDERS)
def test_pade_contact_order(pq):
    """Definition: value and first p+q derivatives at 0 equal
    tanh's, i.e. the series of N - T D vanishes through x^(p+q); checked with
    the textbook coefficients, and the next odd coefficient is nonzero."""
    p, q = pq
    a, b = O.pade(p, q)
    g = maclaurin_golden()
    t = [float(g.get(k, 0)) for k in range(16)]
    for k in range(min(p + q + 3, 16)):
        ak = a[k] if k <= p else 0.0
        conv = sum(b[j] * t[k - j] for j in range(0, min(k, q) + 1))
        resid = ak - conv
        if k <= p + q:
            assert abs(resid) < 1e-13, (pq, k, resid)
        elif k % 2 == 1:
            assert abs(resid) > 1e-12, (pq, k, resid)


def test_pade_rejects_even_odd_orders():
    assert O.pade(2, 2) is None and O.pade(3, 3) is None and O.pade(9, 8) is None


@pytest.mark.parametrize("pq", PADE_ORDERS)
def test_pade_saturation_point(pq):
    """Reading R-CMP-SAT: X_p = first x > 0 where R reaches 1 or stops rising."""
    p, q = pq
    a, b = O.pade(p, q)
    X = O.pade_sat(p, q)
    R = lambda x: polyval(a, x) / polyval(b, x)
    xs = np.linspace(1e-3, X * (1 - 1e-9), 20001)
    r = np.array([R(v) for v in xs])
    assert np.all(np.diff(r) > 0) and np.all(r < 1.0)
    hit_one = abs(R(X) - 1.0) < 1e-12
    d = (R(X + 1e-6) - R(X - 1e-6)) / 2e-6
    at_max = abs(d) < 1e-5
    assert hit_one or at_max, (pq, X, R(X), d)


def test_pade_saturation_closed_forms():
    # [1/0] = x reaches 1 at x = 1; [3/2] reaches 1 at the real root of
    # x^3 - 6x^2 + 15x - 15 (x(15 + x^2) = 15 + 6x^2); [1/2] = 3x/(3 + x^2)
    # peaks at sqrt(3).
    assert O.pade_sat(1, 0) == pytest.approx(1.0, abs=1e-12)
    roots = np.roots([1, -6, 15, -15])
    real = float(roots[np.argmin(np.abs(roots.imag))].real)
    assert O.pade_sat(3, 2) == pytest.approx(real, abs=1e-12)
    assert O.pade_sat(1, 2) == pytest.approx(math.sqrt(3), abs=1e-9)


# --------------------------------------------------------------------------
# Piecewise minimax (Sec. 2.1), layout R-CMP-LAYOUT
# --------------------------------------------------------------------------
def piece_error(c, k, x):
    h = x - k * O.APX_WIDTH
    return np.tanh(x) - np.polyval(np.asarray(c)[::-1], h)


def alternation_count(e, E, tol):
    """Number of alternating-sign clusters with |e| within tol of E."""
    near = np.abs(e) >= E - tol
    signs = []
    for i in np.flatnonzero(near) if near.any() else []:
        s = e[i] > 0
        if not signs or (s != signs[-1]):
            signs.append(s)
    return len(signs)


@pytest.mark.parametrize("deg", [1, 2, 3])
def test_minimax_equioscillation(deg):
    """Chebyshev alternation theorem: P is the best max-norm approximation of
    degree n iff the error attains its max with alternating signs at
    (number of free coefficients + 1) points."""
    for k in range(O.APX_PIECES):
        c, E, it = O.minimax_piece(deg, k)
        assert it > 0
        lo = k * O.APX_WIDTH
        x = np.linspace(lo, lo + O.APX_WIDTH, 400001)
        e = piece_error(c, k, x)
        Emax = np.abs(e).max()
        assert Emax == pytest.approx(E, rel=2e-5, abs=1e-15), (deg, k)
        free = deg + 1 - (1 if k == 0 else 0)
        n_alt = alternation_count(e, Emax, 1e-5 * Emax + 4e-16)
        assert n_alt >= free + 1, (deg, k, n_alt)
        if k == 0:
            assert c[0] == 0.0


@pytest.mark.parametrize("deg", [1, 2, 3])
def test_minimax_beats_competitors(deg):
    """No other polynomial of the same form does better in max norm: least
    squares, the Taylor piece, and random perturbations all lose."""
    rng = np.random.default_rng(deg)
    for k in (0, 1, 3, 7, 12):
        c, E, _ = O.minimax_piece(deg, k)
        lo = k * O.APX_WIDTH
        x = np.linspace(lo, lo + O.APX_WIDTH, 20001)
        h = x - lo
        emm = np.abs(piece_error(c, k, x)).max()
        j0 = 1 if k == 0 else 0
        V = np.stack([h ** j for j in range(j0, deg + 1)], 1)
        ls = np.linalg.lstsq(V, np.tanh(x), rcond=None)[0]
        cls = np.zeros(4); cls[j0:deg + 1] = ls
        assert emm <= np.abs(piece_error(cls, k, x)).max() * (1 + 1e-9)
        for _ in range(20):
            d = np.zeros(4)
            d[j0:deg + 1] = rng.standard_normal(deg + 1 - j0) * E * 0.05
            assert np.abs(piece_error(c + d, k, x)).max() >= emm * (1 - 1e-7)


# --------------------------------------------------------------------------
# Piecewise Taylor (Table 2 rows "Taylor approx degree n"), reading R-CMP-TAYLOR
# --------------------------------------------------------------------------
def test_taylor_piece0_is_maclaurin():
    g = maclaurin_golden()
    for deg in (1, 2, 3):
        c = O.taylor_piece(deg, 0)
        want = [float(g.get(j, 0)) if j <= deg else 0.0 for j in range(4)]
        np.testing.assert_allclose(c, want, rtol=1e-15, atol=1e-300)


def test_taylor_coefficients_are_derivatives():
    """c_j = f^(j)(m)/j! about the midpoint m = k/2 + 1/4: finite differences of tanh."""
    f = math.tanh
    for k in range(1, O.APX_PIECES):
        m = k * 0.5 + 0.25
        c = O.taylor_piece(3, k)
        assert c[0] == pytest.approx(f(m), abs=1e-15)
        d = 1e-5
        assert c[1] == pytest.approx((f(m + d) - f(m - d)) / (2 * d), abs=1e-9)
        d = 1e-4
        assert c[2] == pytest.approx((f(m + d) - 2 * f(m) + f(m - d)) / (2 * d * d), abs=1e-6)
        d = 1e-3
        d3 = (f(m + 2 * d) - 2 * f(m + d) + 2 * f(m - d) - f(m - 2 * d)) / (2 * d ** 3)
        assert c[3] == pytest.approx(d3 / 6, abs=1e-5)
        for deg in (1, 2):   # lower degrees are truncations
            np.testing.assert_array_equal(O.taylor_piece(deg, k)[:deg + 1], c[:deg + 1])


@pytest.mark.parametrize("deg", [1, 2, 3])
def test_taylor_error_order(deg):
    """Remainder ~ f^(n+1)(m) h^(n+1)/(n+1)!: halving h divides the error by ~2^(n+1)."""
    for k in (2, 5, 9):
        m = k * 0.5 + 0.25
        c = O.taylor_piece(deg, k)
        err = lambda h: abs(polyval(c[:deg + 1], h) - math.tanh(m + h))
        ratio = err(0.02) / err(0.01)
        assert ratio == pytest.approx(2.0 ** (deg + 1), rel=0.15), (k, ratio)


# --------------------------------------------------------------------------
# Evaluation over every BF16 pattern and a F32 sample
# --------------------------------------------------------------------------
@pytest.fixture(scope="module")
def apx_maps():
    out = {}
    for kind, p, q in COMPARATORS:
        A = O.Apx(kind, p, q)
        out[(kind, p, q)] = (A, A.map_bf16(W))
    return out


@pytest.mark.parametrize("cfg", COMPARATORS)
def test_eval_invariants_bf16(apx_maps, cfg):
    A, y = apx_maps[cfg]
    y = y.astype(np.int64)
    w = W.astype(np.int64)
    nn = ~NANM
    # NaN passes through (as K-TanH, reading A6)
    assert np.array_equal(y[NANM], w[NANM])
    # odd symmetry, bitwise
    assert np.array_equal(y[w[nn] ^ 0x8000], y[nn] ^ 0x8000)
    # range [-1, 1] and saturation at |x| >= RN32(X_sat)
    yv = O.bf16_to_f64(y.astype(np.uint16))
    assert np.all(np.abs(yv[nn]) <= 1.0)
    sat = nn & (np.abs(XV) >= np.float32(A.xsat))
    assert np.all(y[sat] == ((w[sat] & 0x8000) | 0x3F80))
    # signed zeros
    assert y[0x0000] == 0x0000 and y[0x8000] == 0x8000


@pytest.mark.parametrize("cfg", COMPARATORS)
def test_eval_is_rne_of_binary64_value(apx_maps, cfg):
    """The BF16 output is the nearest-even BF16 of the binary64 value."""
    A, y = apx_maps[cfg]
    sel = np.flatnonzero(FIN)[::97]
    for i in sel:
        v = A.eval(XV[i])
        assert y[i] == O.bf16_encode_rne(v)


@pytest.mark.parametrize("cfg", COMPARATORS)
def test_eval_invariants_f32(cfg):
    A = O.Apx(*cfg)
    rng = np.random.default_rng(7)
    x = np.concatenate([(rng.standard_normal(1 << 15) * 3).astype(np.float32),
                        rng.uniform(-9, 9, 1 << 15).astype(np.float32),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-40, -1e-40,
                                  A.xsat, -A.xsat, 8.0, 7.9999995], np.float32)])
    u = x.view(np.uint32)
    y = A.map_f32(u)
    yn = A.map_f32(u ^ np.uint32(0x80000000))
    nn = ~np.isnan(x)
    assert np.array_equal(yn[nn], y[nn] ^ np.uint32(0x80000000))
    assert np.array_equal(y[~nn], u[~nn])
    yv = y.view(np.float32)
    assert np.all(np.abs(yv[nn]) <= 1.0)
    sat = nn & (np.abs(x) >= np.float32(A.xsat))
    assert np.all(np.abs(yv[sat]) == 1.0)


def _max_errs(A):
    xs = XV[FIN]
    v = np.array([A.eval(x) for x in xs])
    e = np.abs(v - np.tanh(xs))
    return e.max()


def test_error_bounds_and_ordering():
    """Minimax error equals its levelled E; the mathematics orders the forms
    (SPEC.md:348); Table 2 puts Pade 7/8 below K-TanH."""
    err = {cfg: _max_errs(O.Apx(*cfg)) for cfg in COMPARATORS + [("minimax", 1, 0)]}
    for deg in (1, 2, 3):
        Es = max(O.minimax_piece(deg, k)[1] for k in range(O.APX_PIECES))
        assert err[("minimax", deg, 0)] <= Es * (1 + 1e-6) + 1e-15
    assert err[("minimax", 3, 0)] < err[("minimax", 2, 0)] < err[("minimax", 1, 0)]
    assert err[("taylor", 3, 0)] < err[("taylor", 2, 0)]
    assert err[("minimax", 2, 0)] <= err[("taylor", 2, 0)]
    assert err[("minimax", 3, 0)] <= err[("taylor", 3, 0)]
    assert err[("pade", 7, 8)] <= err[("pade", 3, 2)] / 10
    ktanh = O.error_sweep()["max_abs"]
    assert err[("pade", 7, 8)] < ktanh
    paper = {r[0]: r for r in read_golden("table2_comparators.txt")}
    assert float(paper["pade_7_8"][1]) < float(paper["ktanh_bf16"][1])


@pytest.mark.parametrize("deg", [2, 3])
def test_piecewise_layout_last_piece_and_saturation(deg):
    """Reading R-CMP-LAYOUT: 16 pieces of width 1/2 cover [0, 8) and |x| >= 8
    saturates.  On the last piece [7.5, 8) the minimax map is within its own
    levelled error of tanh (binary64) -- not the constant 1 -- and from 8 on
    it is exactly 1."""
    A = O.Apx("minimax", deg)
    _, E15, _ = O.minimax_piece(deg, 15)
    xs = np.linspace(7.5, 8.0, 257)[:-1]
    err = max(abs(A.eval(x) - math.tanh(x)) for x in xs)
    assert err <= E15 * (1 + 1e-6) + 1e-15
    assert all(A.eval(x) == 1.0 for x in (8.0, 8.5, 100.0))
    T = O.Apx("taylor", deg)
    assert max(abs(T.eval(x) - math.tanh(x)) for x in xs) < 1e-7 < 1.0 - math.tanh(7.5)


@pytest.mark.parametrize("j,pq", [(3, (3, 2)), (8, (7, 8))])
def test_pade_eval_is_the_lambert_convergent(j, pq):
    """The comparator's evaluated map (not only its coefficients) is the Lambert
    convergent below its saturation point, and exactly 1 from X_p on."""
    A = O.Apx("pade", *pq)
    X = A.xsat
    for x in np.linspace(0.01, X * 0.999, 97):
        assert A.eval(x) == pytest.approx(min(lambert_cf(j, x), 1.0), rel=1e-13, abs=1e-15)
    assert A.eval(X * 1.001) == 1.0 and A.eval(50.0) == 1.0


@pytest.mark.parametrize("deg", [2, 3])
def test_taylor_pieces_interpolate_at_their_centres(deg):
    """A Taylor polynomial equals the function at its expansion point: piece k
    (k >= 1) is expanded about k/2 + 1/4 (reading R-CMP-LAYOUT), piece 0 about 0."""
    T = O.Apx("taylor", deg)
    for k in range(1, 16):
        c = k / 2 + 0.25
        assert T.eval(c) == pytest.approx(math.tanh(c), rel=1e-15, abs=1e-16), k
    assert T.eval(0.0) == 0.0
