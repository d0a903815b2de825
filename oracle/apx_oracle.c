/*
 * oracle/apx_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain, slow, scalar CPU implementations of the float-op TanH
 * approximations that Table 2 of the K-TanH paper compares against
 * (Kundu et al., arXiv 1909.07729), written from the
 * paper's Sec. 2.1-2.2 and the readings R-CMP-* in
 * DESIGN.md.  SURVEY.md NEXT-4.  Same rules as ktanh_oracle.c: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu legs may use it; it shares no
 * code with paper_1909_07729_b200/ and never imports it.
 *
 * Precision: binary64 throughout; results are rounded once to the output
 * format.  The only decisions taken in floating point (which piece, whether
 * to saturate) are exact comparisons of the input value against constants
 * that are powers of two (piecewise forms) or against RN32(X_p) (Pade), the
 * kernel's fp32 constant (reading R-CMP-SAT).
 *
 * Parity status:
 *   kto_tanh_maclaurin ...... pinned (known coefficients 1, -1/3, 2/15, -17/315,
 *                             62/2835; series sum vs tanh at small x)
 *   kto_pade ................ pinned (SPEC closed form [3/2]; Lambert continued
 *                             fraction convergents for every (p,q) tested;
 *                             contact order p+q+1 at 0)
 *   kto_pade_sat ............ pinned (R(X_p) = 1 or R'(X_p) = 0, R < 1 and
 *                             increasing on (0, X_p))
 *   kto_minimax_piece ....... pinned (Chebyshev equioscillation on a dense
 *                             grid; beats least squares and Taylor in max norm)
 *   kto_taylor_piece ........ pinned (value and derivatives vs finite
 *                             differences of tanh; error order h^(n+1))
 *   kto_apx_* evaluation .... pinned (odd symmetry, saturation, NaN, error
 *                             ordering, error bounds vs tanh)
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

uint16_t kto_bf16_encode_rne(double x);   /* ktanh_oracle.c */
double kto_bf16_decode(uint16_t w);       /* ktanh_oracle.c */

/* Piecewise layout (reading R-CMP-LAYOUT): the paper divides "the input
 * range into intervals" without giving them; here 16 uniform
 * pieces of width 1/2 on [0, 8), odd extension, |x| >= 8 -> +-1. */
#define APX_PIECES 16
#define APX_WIDTH 0.5
#define APX_XSAT 8.0
#define APX_MAXDEG 3

enum { APX_PADE = 0, APX_MINIMAX = 1, APX_TAYLOR = 2 };

/* ------------------------------------------------------------------ */
/* Maclaurin coefficients of TanH ("the first p+q derivatives of f at   */
/* zero").  From TanH' = 1 - TanH^2 (differentiate the     */
/* definition): with T(x) = sum t_k x^k,                     */
/*   (k+1) t_{k+1} = [k == 0] - sum_{i=0..k} t_i t_{k-i},  t_0 = 0.       */
/* ------------------------------------------------------------------ */
static void maclaurin_ld(int n, long double *t)
{
    t[0] = 0.0L;
    for (int k = 0; k < n; ++k) {
        long double conv = 0.0L;
        for (int i = 0; i <= k; ++i) conv += t[i] * t[k - i];
        t[k + 1] = ((k == 0 ? 1.0L : 0.0L) - conv) / (long double)(k + 1);
    }
}

void kto_tanh_maclaurin(int n, double *t)
{
    long double tl[64];
    if (n > 62) n = 62;
    maclaurin_ld(n, tl);
    for (int k = 0; k <= n; ++k) t[k] = (double)tl[k];
}

/* Gaussian elimination with partial pivoting, n <= 16, A row-major n x n,
 * in x87 extended precision (the Pade system is ill-conditioned). */
static int solve(int n, long double *A, long double *rhs, long double *sol)
{
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabsl(A[r * n + c]) > fabsl(A[piv * n + c])) piv = r;
        if (A[piv * n + c] == 0.0L) return -1;
        if (piv != c) {
            for (int k = 0; k < n; ++k) {
                long double tmp = A[c * n + k]; A[c * n + k] = A[piv * n + k]; A[piv * n + k] = tmp;
            }
            long double tmp = rhs[c]; rhs[c] = rhs[piv]; rhs[piv] = tmp;
        }
        for (int r = c + 1; r < n; ++r) {
            long double f = A[r * n + c] / A[c * n + c];
            for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
            rhs[r] -= f * rhs[c];
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        long double s = rhs[r];
        for (int k = r + 1; k < n; ++k) s -= A[r * n + k] * sol[k];
        sol[r] = s / A[r * n + r];
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Pade [p/q] of TanH, Sec. 2.2: the ratio           */
/* sum a_i x^i / sum b_i x^i whose value and first p+q derivatives at 0   */
/* equal TanH's.  Equivalently N(x) - T(x) D(x) = O(x^(p+q+1)), b_0 = 1:  */
/*   a_k - sum_{j=1..min(k,q)} b_j t_{k-j} = t_k,   k = 0..p+q            */
/* (a_k = 0 for k > p).  TanH is odd, so for p odd and q even the system  */
/* is solved in its reduced form (reading R-CMP-PADE): a_k = 0 for even   */
/* k and b_j = 0 for odd j, leaving unknowns a_1, a_3, .., a_p and        */
/* b_2, b_4, .., b_q and the equations of odd k.                          */
/* a has p+1 entries, b has q+1 (b[0] = 1).  Returns 0, or -1 if (p, q)   */
/* is not (odd, even) with p+q <= 15 or the system is singular.           */
/* ------------------------------------------------------------------ */
int kto_pade(int p, int q, double *a, double *b)
{
    if (p < 1 || (p & 1) == 0 || q < 0 || (q & 1) || p + q > 15) return -1;
    long double t[17];
    maclaurin_ld(16, t);
    const int na = (p + 1) / 2, nb = q / 2, n = na + nb;
    long double A[16 * 16], rhs[16], sol[16];
    /* unknown u: u < na -> a_{2u+1}; u >= na -> b_{2(u-na+1)} */
    for (int e = 0; e < n; ++e) {          /* equation for odd k = 2e+1 */
        const int k = 2 * e + 1;
        for (int u = 0; u < n; ++u) {
            long double v = 0.0L;
            if (u < na) {
                v = (2 * u + 1 == k) ? 1.0L : 0.0L;
            } else {
                const int j = 2 * (u - na + 1);
                v = (j <= k) ? -t[k - j] : 0.0L;
            }
            A[e * n + u] = v;
        }
        rhs[e] = t[k];
    }
    if (solve(n, A, rhs, sol) != 0) return -1;
    for (int i = 0; i <= p; ++i) a[i] = 0.0;
    for (int i = 0; i <= q; ++i) b[i] = 0.0;
    b[0] = 1.0;
    for (int u = 0; u < na; ++u) a[2 * u + 1] = (double)sol[u];
    for (int u = na; u < n; ++u) b[2 * (u - na + 1)] = (double)sol[u];
    return 0;
}

static double poly(const double *c, int deg, double x)
{
    double s = c[deg];
    for (int i = deg - 1; i >= 0; --i) s = s * x + c[i];
    return s;
}

static double dpoly(const double *c, int deg, double x)
{
    double s = 0.0;
    for (int i = deg; i >= 1; --i) s = s * x + (double)i * c[i];
    return s;
}

/* Sign of R'(x) numerator: N'D - ND'. */
static double pade_dnum(int p, int q, const double *a, const double *b, double x)
{
    return dpoly(a, p, x) * poly(b, q, x) - poly(a, p, x) * dpoly(b, q, x);
}

/* Saturation point X_p of the Pade form (reading R-CMP-SAT): the first
 * x > 0 at which R(x) reaches 1 or stops increasing; for |x| >= X_p the
 * approximation returns +-1 (like Alg. 1 line 4).  Bracketed by a scan with
 * step 1/1024 on (0, 64], refined by bisection; 64 if neither happens. */
double kto_pade_sat(int p, int q)
{
    double a[16], b[16];
    if (kto_pade(p, q, a, b) != 0) return NAN;
    double prev = 0.0;
    for (int i = 1; i <= 64 * 1024; ++i) {
        const double x = i / 1024.0;
        const double r = poly(a, p, x) / poly(b, q, x);
        const double d = pade_dnum(p, q, a, b, x);
        if (r >= 1.0 || d <= 0.0) {
            double lo = prev, hi = x;
            for (int it = 0; it < 200; ++it) {
                const double m = 0.5 * (lo + hi);
                if (m <= lo || m >= hi) break;
                const double rm = poly(a, p, m) / poly(b, q, m);
                if (rm >= 1.0 || pade_dnum(p, q, a, b, m) <= 0.0) hi = m; else lo = m;
            }
            return hi;
        }
        prev = x;
    }
    return 64.0;
}

/* ------------------------------------------------------------------ */
/* Minimax polynomial, Sec. 2.1: on each piece        */
/* [lo, lo + w] the degree-n polynomial P minimising                      */
/* max |TanH(x) - P(x)|, written in h = x - lo.  Piece 0 is constrained   */
/* to P(0) = 0 (reading R-CMP-LAYOUT: keeps the odd extension continuous  */
/* and the relative error finite near 0).  Remez exchange: solve          */
/* P(x_i) + (-1)^i E = TanH(x_i) on m+1 reference points, move the        */
/* reference to the alternating extrema of the error, repeat until the    */
/* extrema are level.                                                     */
/* ------------------------------------------------------------------ */
static double mm_err(const double *c, int j0, int deg, double lo, double x)
{
    const double h = x - lo;
    double s = 0.0;
    for (int j = deg; j >= j0; --j) s = s * h + c[j];
    for (int j = 0; j < j0; ++j) s *= h;
    return tanh(x) - s;
}

/* golden-section maximisation of |e| on [l, r] */
static double mm_refine(const double *c, int j0, int deg, double lo, double l, double r)
{
    const double g = 0.6180339887498949;
    double x1 = r - g * (r - l), x2 = l + g * (r - l);
    double f1 = fabs(mm_err(c, j0, deg, lo, x1)), f2 = fabs(mm_err(c, j0, deg, lo, x2));
    for (int it = 0; it < 80; ++it) {
        if (f1 < f2) { l = x1; x1 = x2; f1 = f2; x2 = l + g * (r - l); f2 = fabs(mm_err(c, j0, deg, lo, x2)); }
        else         { r = x2; x2 = x1; f2 = f1; x1 = r - g * (r - l); f1 = fabs(mm_err(c, j0, deg, lo, x1)); }
    }
    return 0.5 * (l + r);
}

/* c[0..deg] in powers of h = x - lo (c[0] = 0 for piece 0); *E = levelled
 * error; returns the number of exchange iterations (or -1). */
int kto_minimax_piece(int deg, int k, double *c, double *E)
{
    if (deg < 1 || deg > APX_MAXDEG || k < 0 || k >= APX_PIECES) return -1;
    const double lo = k * APX_WIDTH, hi = lo + APX_WIDTH;
    const int j0 = (k == 0) ? 1 : 0;
    const int m = deg + 1 - j0, npts = m + 1;
    double ref[8];
    for (int i = 0; i < npts; ++i)
        ref[i] = lo + (hi - lo) * 0.5 * (1.0 - cos(M_PI * (double)(i + j0) / (double)(npts - 1 + j0)));
    for (int j = 0; j <= APX_MAXDEG; ++j) c[j] = 0.0;
    int it;
    for (it = 1; it <= 100; ++it) {
        long double A[64], rhs[8], sol[8];
        for (int i = 0; i < npts; ++i) {
            const double h = ref[i] - lo;
            for (int u = 0; u < m; ++u) A[i * npts + u] = powl(h, (long double)(u + j0));
            A[i * npts + m] = (i & 1) ? -1.0L : 1.0L;
            rhs[i] = tanh(ref[i]);
        }
        if (solve(npts, A, rhs, sol) != 0) return -1;
        for (int u = 0; u < m; ++u) c[u + j0] = (double)sol[u];
        *E = fabs((double)sol[m]);
        /* local extrema of e on a dense grid, then refined */
        enum { G = 4096 };
        double ex[G + 1], ev[G + 1];
        int ne = 0;
        double prev = mm_err(c, j0, deg, lo, lo), cur = mm_err(c, j0, deg, lo, lo + (hi - lo) / G);
        if (j0 == 0) { ex[ne] = lo; ev[ne] = prev; ++ne; }
        for (int g = 1; g < G; ++g) {
            const double nx = lo + (hi - lo) * (g + 1) / G;
            const double next = mm_err(c, j0, deg, lo, nx);
            if (fabs(cur) >= fabs(prev) && fabs(cur) >= fabs(next) && cur != 0.0) {
                const double xr = mm_refine(c, j0, deg, lo, lo + (hi - lo) * (g - 1) / G, nx);
                ex[ne] = xr; ev[ne] = mm_err(c, j0, deg, lo, xr); ++ne;
            }
            prev = cur; cur = next;
        }
        ex[ne] = hi; ev[ne] = mm_err(c, j0, deg, lo, hi); ++ne;
        /* merge same-sign neighbours, keeping the larger |e| */
        int na = 0;
        for (int i = 0; i < ne; ++i) {
            if (na > 0 && (ev[i] > 0) == (ev[na - 1] > 0)) {
                if (fabs(ev[i]) > fabs(ev[na - 1])) { ex[na - 1] = ex[i]; ev[na - 1] = ev[i]; }
            } else {
                ex[na] = ex[i]; ev[na] = ev[i]; ++na;
            }
        }
        if (na < npts) return -1;
        int first = 0, last = na - 1;
        while (last - first + 1 > npts) {
            if (fabs(ev[first]) < fabs(ev[last])) ++first; else --last;
        }
        double emax = 0.0, emin = INFINITY;
        for (int i = 0; i < npts; ++i) {
            ref[i] = ex[first + i];
            emax = fmax(emax, fabs(ev[first + i]));
            emin = fmin(emin, fabs(ev[first + i]));
        }
        if (emax - emin <= 1e-10 * emax + 4e-16) break;   /* level to rounding noise */
    }
    return it;
}

/* ------------------------------------------------------------------ */
/* Taylor polynomial of degree n (Table 2 rows "Taylor approx degree n",  */
/* PAPER.md:268-269), piecewise on the same layout (reading R-CMP-TAYLOR): */
/* piece 0 is the Maclaurin polynomial (about 0), piece k >= 1 is         */
/* expanded about its midpoint m_k = k/2 + 1/4, in h = x - m_k.            */
/* Coefficients from the addition formula                                 */
/*   TanH(m + h) = (T + TanH h) / (1 + T TanH h),  T = TanH(m),            */
/* as a power-series quotient in h using the Maclaurin series of TanH h.  */
/* ------------------------------------------------------------------ */
int kto_taylor_piece(int deg, int k, double *c)
{
    if (deg < 1 || deg > APX_MAXDEG || k < 0 || k >= APX_PIECES) return -1;
    double t[APX_MAXDEG + 2];
    kto_tanh_maclaurin(APX_MAXDEG + 1, t);
    for (int j = 0; j <= APX_MAXDEG; ++j) c[j] = 0.0;
    if (k == 0) {
        for (int j = 0; j <= deg; ++j) c[j] = t[j];
        return 0;
    }
    const double T = tanh(k * APX_WIDTH + 0.25);
    double num[APX_MAXDEG + 1], den[APX_MAXDEG + 1];
    for (int j = 0; j <= deg; ++j) {
        num[j] = (j == 0 ? T : 0.0) + t[j];
        den[j] = (j == 0 ? 1.0 : 0.0) + T * t[j];
    }
    for (int j = 0; j <= deg; ++j) {
        double s = num[j];
        for (int i = 1; i <= j; ++i) s -= den[i] * c[j - i];
        c[j] = s / den[0];
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Parameter block for evaluation: par[0] = saturation point (Pade: X_p;  */
/* piecewise: 8), Pade: par[1..p+1] = a, par[p+2..p+q+2] = b; piecewise:  */
/* par[1 + 4k + j] = c_j of piece k.  Returns 0 or -1.                    */
/* ------------------------------------------------------------------ */
int kto_apx_params(int kind, int p, int q, double *par)
{
    memset(par, 0, sizeof(double) * (1 + 4 * APX_PIECES));
    if (kind == APX_PADE) {
        if (kto_pade(p, q, par + 1, par + 2 + p) != 0) return -1;
        par[0] = kto_pade_sat(p, q);
        return 0;
    }
    par[0] = APX_XSAT;
    for (int k = 0; k < APX_PIECES; ++k) {
        double E;
        const int rc = (kind == APX_MINIMAX) ? (kto_minimax_piece(p, k, par + 1 + 4 * k, &E) < 0 ? -1 : 0)
                                             : kto_taylor_piece(p, k, par + 1 + 4 * k);
        if (rc != 0) return -1;
    }
    return 0;
}

/* Magnitude map a >= 0 (finite or +inf) -> approximation of TanH(a),
 * clamped to [0, 1] (reading R-CMP-SAT). */
static double apx_mag(int kind, int p, int q, const double *par, double a)
{
    if (kind == APX_PADE) {
        if (a >= (double)(float)par[0]) return 1.0;    /* saturate at RN32(X_p) */
        const double y = poly(par + 1, p, a) / poly(par + 2 + p, q, a);
        return y > 1.0 ? 1.0 : y;
    }
    if (a >= APX_XSAT) return 1.0;
    const int k = (int)floor(a / APX_WIDTH);
    const double h = (kind == APX_TAYLOR && k > 0) ? a - (k * APX_WIDTH + 0.25) : a - k * APX_WIDTH;
    const double y = poly(par + 1 + 4 * k, p, h);
    return y > 1.0 ? 1.0 : (y < 0.0 ? 0.0 : y);
}

/* Double-precision value before output rounding (for the tests). */
double kto_apx_eval(int kind, int p, int q, const double *par, double x)
{
    if (isnan(x)) return x;
    const double y = apx_mag(kind, p, q, par, fabs(x));
    return signbit(x) ? -y : y;
}

/* BF16 in -> BF16 out: decode, evaluate in binary64, one RNE to BF16.
 * NaN passes through unchanged (as K-TanH, reading A6). */
uint16_t kto_apx_bf16(int kind, int p, int q, const double *par, uint16_t w)
{
    if ((w & 0x7FFF) > 0x7F80) return w;
    return kto_bf16_encode_rne(kto_apx_eval(kind, p, q, par, kto_bf16_decode(w)));
}

/* F32 in -> F32 out: one RN to binary32 (C's double -> float conversion in
 * the default rounding mode). */
uint32_t kto_apx_f32(int kind, int p, int q, const double *par, uint32_t u)
{
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) return u;
    float xf;
    memcpy(&xf, &u, 4);
    const float y = (float)kto_apx_eval(kind, p, q, par, (double)xf);
    uint32_t r;
    memcpy(&r, &y, 4);
    return r;
}

void kto_apx_map_bf16(int kind, int p, int q, const double *par, const uint16_t *x, uint16_t *y,
                      size_t n)
{
    for (size_t i = 0; i < n; ++i) y[i] = kto_apx_bf16(kind, p, q, par, x[i]);
}

void kto_apx_map_f32(int kind, int p, int q, const double *par, const uint32_t *x, uint32_t *y,
                     size_t n)
{
    for (size_t i = 0; i < n; ++i) y[i] = kto_apx_f32(kind, p, q, par, x[i]);
}
