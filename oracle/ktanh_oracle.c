/*
 * oracle/ktanh_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, scalar CPU implementation of K-TanH (Kundu et al.,
 * "K-TanH: Efficient TanH for Deep Learning", arXiv 1909.07729), written
 * from /root/reference/PAPER.md.  Every function cites the passage it
 * follows ("PAPER.md:L (section / Alg. / Eq. / Table)").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load, call or execute anything in oracle/.
 * It shares no code, header, table or constant generator with the CUDA
 * path in paper_1909_07729_b200/ and it never imports it.
 *
 * Precision: the K-TanH core is integer-only (as the paper defines it);
 * every floating-point step that is not a "decision" is done in IEEE
 * binary64, and where binary64 is not exact (x/2 (1+t) in both formats --
 * for a subnormal BF16 x the two terms are 2^133 apart -- and the LSTM cell's
 * f c + i g) the exact sum of two exact binary64 products is rounded once
 * (rn32_exact_sum, rnbf16_exact_sum).  The one decision made in floating point -- the argument
 * u = sqrt(2/pi)(x + a x^3) of the K-GELU, whose rounding picks the LUT
 * entry -- is taken in binary32 with the op order written in
 * gelu_arg_f32() below (reading R-GELU-ARG), because the CUDA
 * path takes that decision in binary32.
 *
 * Compile: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared -lm
 * (-ffp-contract=off: no silent a*b+c contraction anywhere).
 *
 * Parity status of each function:
 *   kto_bf16_decode / kto_bf16_encode_rne ..... pinned (round trip, nearest)
 *   kto_ktanh_bf16 ............................ pinned (Table 2 error bound,
 *                                               invariants, value-domain check)
 *   kto_ktanh_f32 ............................. pinned (BF16 closed-form relation,
 *                                               error bound, invariants)
 *   kto_ksigmoid_* ............................ pinned (exact rational (1+t)/2)
 *   kto_kswish_* / kto_kgelu_* ................ pinned (BF16: exact rational single
 *                                               rounding over all 65,536 patterns;
 *                                               special cases + error bound)
 *   kto_bwd_* (reading R-BWD) ................. pinned (closed forms at 0, in the
 *                                               bypass/saturation regions, and
 *                                               error bounds vs the true derivative)
 *   kto_build_lut (Sec. 2.4 optimizer) ........ pinned (Table 1 match counts,
 *                                               SSE dominance, Table 2 ablation)
 *   kto_build_lut_sp at p = 23 (NEXT-3) ....... pinned (tests/test_oracle_f32_tables.py:
 *                                               brute-force Step 3 optimality with
 *                                               numpy's RNE, validity, dominance)
 *   kto_map_f32_p / kto_bwd_map_f32_p (pb=23) . pinned (lifted Table 1 == A8)
 *   kto_bounds ................................ pinned (exhaustive no-overflow)
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------ */
/* Number format, PAPER.md:80-81 (Sec. 1): x = (-1)^s 2^E (1 + M/2^p),   */
/* BFloat16 (s,E,M) = (1,8,7), Float32 (1,8,23), E bias-added.          */
/* ------------------------------------------------------------------ */

/* Exact real value of a BF16 bit pattern (E=0 subnormal, E=255 inf/NaN). */
double kto_bf16_decode(uint16_t w)
{
    int s = (w >> 15) & 1;
    int E = (w >> 7) & 0xFF;
    int M = w & 0x7F;
    double v;
    if (E == 0xFF) {
        v = (M == 0) ? INFINITY : NAN;
    } else if (E == 0) {
        v = ldexp((double)M / 128.0, -126);          /* subnormal */
    } else {
        v = ldexp(1.0 + (double)M / 128.0, E - 127);  /* normal */
    }
    return s ? -v : v;
}

/* Round a binary64 value to the nearest BF16, ties to even.            */
/* NaN -> 0x7FC0 (canonical quiet NaN), overflow -> +-inf.              */
uint16_t kto_bf16_encode_rne(double x)
{
    if (isnan(x)) return 0x7FC0;
    uint16_t s = signbit(x) ? 0x8000 : 0;
    double a = fabs(x);
    if (isinf(a)) return s | 0x7F80;
    if (a == 0.0) return s;
    int k;
    frexp(a, &k);             /* a = f 2^k, f in [0.5,1) => a in [2^(k-1), 2^k) */
    int e = k - 1;            /* unbiased exponent of a                           */
    double quantum;           /* spacing of BF16 numbers around a                 */
    if (e < -126) quantum = ldexp(1.0, -133);       /* subnormal spacing 2^-126/2^7 */
    else          quantum = ldexp(1.0, e - 7);
    double q = a / quantum;   /* exact: division by a power of two                */
    double nq = nearbyint(q); /* default rounding mode: nearest, ties to even     */
    long n = (long)nq;
    long bits;
    if (e < -126) {
        bits = n;                                   /* E=0, M=n; n=128 -> 0x0080 */
    } else {
        bits = ((long)(e + 127) << 7) + (n - 128);  /* n=256 carries into E      */
    }
    if (bits >= 0x7F80) bits = 0x7F80;              /* overflow -> inf           */
    return (uint16_t)(s | (uint16_t)bits);
}

static float f32_from_bits(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t bits_from_f32(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* ------------------------------------------------------------------ */
/* Parameter tables T_E, T_r, T_b (Alg. 1 line 1).         */
/* Table 1, transcribed here independently of the     */
/* CUDA path, index t = 5-bit string "e1 e0 m6 m5 m4".                   */
/* ------------------------------------------------------------------ */
typedef struct { int E[32]; int r[32]; int b[32]; } kto_lut;

/* rows in the order printed in Table 1: left column then right column */
static const struct { int t; int E, r, b; } TABLE1_ROWS[32] = {
    /* left column */
    {0x07, 126, 6, 126}, {0x06, 126, 6, 126}, {0x05, 126, 6, 126}, {0x04, 126, 6, 126},
    {0x03, 126, 4, 123}, {0x02, 126, 4, 123}, {0x01, 126, 4, 122}, {0x00, 126, 2, 119},
    {0x1F, 126, 4, 110}, {0x1E, 126, 2,  89}, {0x1D, 126, 2,  89}, {0x1C, 126, 2,  88},
    {0x1B, 126, 1,  73}, {0x1A, 126, 1,  73}, {0x19, 126, 1,  72}, {0x18, 126, 0,  65},
    /* right column */
    {0x17, 126, 1,   4}, {0x16, 126, 1,   4}, {0x15, 126, 1,   4}, {0x14, 126, 1,   3},
    {0x13, 126, 1,   2}, {0x12, 126, 1,  -1}, {0x11, 126, 1,  -4}, {0x10, 125, 0, 112},
    {0x0F, 125, 0, -18}, {0x0E, 125, 0, -15}, {0x0D, 125, 0, -12}, {0x0C, 125, 0, -10},
    {0x0B, 125, 0,  -7}, {0x0A, 125, 0,  -6}, {0x09, 125, 0,  -4}, {0x08, 125, 1,   1},
};

void kto_table1(int *E, int *r, int *b)
{
    for (int i = 0; i < 32; ++i) {
        int t = TABLE1_ROWS[i].t;
        E[t] = TABLE1_ROWS[i].E;
        r[t] = TABLE1_ROWS[i].r;
        b[t] = TABLE1_ROWS[i].b;
    }
}

/* Thresholds, PAPER.md:144 (Sec. 2.3): T1 = 0.25, T2 = 3.75. */
static const double T1 = 0.25;
static const double T2 = 3.75;

/* Index t (Alg. 1 line 6; Sec. 2.4):      */
/* "2 LSBs of exponent and 3 MSBs of mantissa"; the exponent bits are the  */
/* high bits of t (layout fixed by Table 1, reading A1).         */
static int index_t(int E, int M_top3) { return ((E & 3) << 3) | M_top3; }

/* Set when a table entry pushes M_o outside [0, 2^q - 1] (an invalid LUT). */
static int g_overflow = 0;
int kto_overflow_flag(void) { int f = g_overflow; g_overflow = 0; return f; }

/* ------------------------------------------------------------------ */
/* Algorithm 1, K-TanH, BFloat16.                      */
/* ------------------------------------------------------------------ */
uint16_t kto_ktanh_bf16(uint16_t x, const int *TE, const int *Tr, const int *Tb)
{
    /* line 1: x_i = (s_i, E_i, M_i) */
    int s = (x >> 15) & 1;
    int E = (x >> 7) & 0xFF;
    int M = x & 0x7F;
    double ax = fabs(kto_bf16_decode(x));
    /* NaN: Alg. 1 is silent; reading A6 passes the input through. */
    if (isnan(ax)) return x;
    /* line 3: |x_i| < T1  ->  y_o = x_i */
    if (ax < T1) return x;
    /* line 4: |x_i| > T2  ->  (s_i, E_bias, 0), i.e. +-1 (incl. +-inf, reading A5) */
    if (ax > T2) return (uint16_t)((s << 15) | (127 << 7) | 0);
    /* line 6: bit string t from lower bits of E_i and higher bits of M_i */
    int t = index_t(E, M >> 4);
    /* line 7: theta_t = (E_t, r_t, b_t) */
    int Et = TE[t], rt = Tr[t], bt = Tb[t];
    /* line 8: s_o = s_i, E_o = E_t, M_o = (M_i >> r_t) + b_t */
    int Mo = (M >> rt) + bt;
    if (Mo < 0 || Mo > 127) g_overflow = 1;
    /* line 9 */
    return (uint16_t)((s << 15) | ((Et & 0xFF) << 7) | (Mo & 0x7F));
}

/* ------------------------------------------------------------------ */
/* 64-interval variant ("Our parameter values are 8-bit only, */
/* so we can create 64 intervals to achieve more accurate approximation"):  */
/* s index bits of the mantissa (s = 3: Table 1 layout, 32 entries; s = 4:  */
/* 64 entries), t = ((E & 3) << s) | (M >> (7 - s)).  Everything else is   */
/* Algorithm 1 as above.                                                     */
/* ------------------------------------------------------------------ */
uint16_t kto_ktanh_bf16_s(uint16_t x, int s_bits, const int *TE, const int *Tr, const int *Tb)
{
    int s = (x >> 15) & 1;
    int E = (x >> 7) & 0xFF;
    int M = x & 0x7F;
    double ax = fabs(kto_bf16_decode(x));
    if (isnan(ax)) return x;
    if (ax < T1) return x;
    if (ax > T2) return (uint16_t)((s << 15) | (127 << 7));
    int t = ((E & 3) << s_bits) | (M >> (7 - s_bits));
    int Mo = (M >> Tr[t]) + Tb[t];
    if (Mo < 0 || Mo > 127) g_overflow = 1;
    return (uint16_t)((s << 15) | ((TE[t] & 0xFF) << 7) | (Mo & 0x7F));
}

void kto_map_bf16_s(const uint16_t *x, uint16_t *y, size_t n, int s_bits,
                    const int *TE, const int *Tr, const int *Tb)
{
    for (size_t i = 0; i < n; ++i) y[i] = kto_ktanh_bf16_s(x[i], s_bits, TE, Tr, Tb);
}

/* ------------------------------------------------------------------ */
/* Algorithm 1 on Float32, native reading A8 ("compatible    */
/* with multiple such data formats"): same T1/T2 and 5-bit index from    */
/* (E & 3, top 3 of the 23-bit mantissa); line 8 with p = 23:            */
/* M_o = (M_i >> r_t) + b_t * 2^(23-7)  (b_t is in units of 2^-7).        */
/* ------------------------------------------------------------------ */
/* pb = the mantissa width b_t is expressed in: 7 (reading A8, Table 1's    */
/* BF16-unit b, scaled by 2^16) or 23 (an F32 table re-optimised at p = 23, */
/* M_o = (M_i >> r_t) + b_t).                             */
static uint32_t ktanh_f32_pb(uint32_t x, const int *TE, const int *Tr, const int *Tb, int pb)
{
    uint32_t s = x >> 31;
    int E = (int)((x >> 23) & 0xFF);
    int32_t M = (int32_t)(x & 0x7FFFFF);
    double ax = fabs((double)f32_from_bits(x));
    if (isnan(ax)) return x;                              /* A6 */
    if (ax < T1) return x;                                /* line 3 */
    if (ax > T2) return (s << 31) | (127u << 23);         /* line 4 */
    int t = index_t(E, (int)(M >> 20));                   /* line 6 */
    int Et = TE[t], rt = Tr[t], bt = Tb[t];               /* line 7 */
    int32_t Mo = (M >> rt) + bt * (1 << (23 - pb));       /* line 8, p = 23 */
    if (Mo < 0 || Mo > 0x7FFFFF) g_overflow = 1;
    return (s << 31) | ((uint32_t)(Et & 0xFF) << 23) | ((uint32_t)Mo & 0x7FFFFF);
}

uint32_t kto_ktanh_f32(uint32_t x, const int *TE, const int *Tr, const int *Tb)
{
    return ktanh_f32_pb(x, TE, Tr, Tb, 7);
}

uint32_t kto_ktanh_f32_p23(uint32_t x, const int *TE, const int *Tr, const int *Tb)
{
    return ktanh_f32_pb(x, TE, Tr, Tb, 23);
}

/* ------------------------------------------------------------------ */
/* K-TanH of a Float32 value through BFloat16 (the     */
/* alternative to reading A8): "We assume BFloat16 input    */
/* for K-TanH (Float32 to BFloat16 conversion cost is not considered)".  */
/* Round the F32 value to the nearest BF16 (ties to even), apply Alg. 1, */
/* and return the BF16 result as an F32 (exact widening: append 16 zero  */
/* bits).  NaN -> the BF16 canonical NaN widened.                        */
/* ------------------------------------------------------------------ */
uint32_t kto_ktanh_f32_via_bf16(uint32_t x, const int *TE, const int *Tr, const int *Tb)
{
    const uint16_t b = kto_bf16_encode_rne((double)f32_from_bits(x));
    return (uint32_t)kto_ktanh_bf16(b, TE, Tr, Tb) << 16;
}

/* ------------------------------------------------------------------ */
/* Derived activations, PAPER.md:60-71 (Sec. 1).                          */
/*   Sigmoid(x) = (1 + TanH(x/2))/2   (parentheses garbled in the paper,  */
/*                                     reading A7)                        */
/*   Swish(x)   = x * Sigmoid(x)                                          */
/*   GELU(x)   ~= x/2 (1 + TanH(sqrt(2/pi)(x + a x^3))),  a = 0.044715    */
/* The TanH is K-TanH on the format's own bits: its argument is rounded   */
/* (RNE) to the format first; the outer affine step is exact and rounded  */
/* once to the format (R-DERIVED).                                        */
/* ------------------------------------------------------------------ */

/* GELU argument, decision precision binary32 (reading R-GELU-ARG):       */
/*   C0 = f32(sqrt(2/pi)), C1 = f32(sqrt(2/pi) * a)                        */
/*   u  = x * fma(C1, x*x, C0)        == sqrt(2/pi)(x + a x^3) in exact math */
static const double GELU_A = 0.044715;

/* RN32 of the EXACT sum a + b of two doubles.  Reading R-DERIVED (and
 * R-LSTM-CELL) round the exact value of the outer step ONCE to binary32; for
 * F32 data that value can need more than binary64's 53 bits (x/2 (1 + t) with
 * a 24-bit t spans up to 65 bits), so evaluating it in binary64 and then
 * converting would round twice.  s = RN64(a + b) with its exact error e
 * (Knuth's TwoSum); RN32(s) equals RN32(a + b) unless s lies exactly halfway
 * between two floats and e != 0, in which case e decides the side. */
static float rn32_exact_sum(double a, double b)
{
    double s = a + b;
    if (!isfinite(s) || !isfinite(a) || !isfinite(b)) return (float)s;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    float f = (float)s;
    if (e == 0.0 || (double)f == s || isinf(f)) return f;
    float g = (s > (double)f) ? nextafterf(f, INFINITY) : nextafterf(f, -INFINITY);
    double mid = ((double)f + (double)g) / 2.0;      /* exact in binary64 */
    if (s != mid) return f;
    return ((e > 0.0) == ((double)g > (double)f)) ? g : f;
}

float kto_rn32_exact_sum(double a, double b) { return rn32_exact_sum(a, b); }   /* for the pins */

/* RN_bf16 of the EXACT sum a + b of two doubles (reading R-DERIVED for the
 * BF16 K-Swish / K-GELU outer step x/2 + (x/2) t).  For a subnormal x the two
 * terms are ~2^133 apart, so RN64(a + b) drops b; when a itself is a BF16
 * tie (x/2 with x odd in the last subnormal place) b decides the side.  Same
 * TwoSum construction as rn32_exact_sum: RN_bf16(s) is the answer unless s is
 * exactly a BF16 midpoint and the error e of s is non-zero. */
static uint16_t rnbf16_exact_sum(double a, double b)
{
    double s = a + b;
    uint16_t f = kto_bf16_encode_rne(s);
    if (!isfinite(s) || !isfinite(a) || !isfinite(b)) return f;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    double fv = kto_bf16_decode(f);
    if (e == 0.0 || fv == s || isinf(fv)) return f;
    uint16_t sg = f & 0x8000, mag = f & 0x7FFF;
    uint16_t g = sg | (uint16_t)(fabs(s) > fabs(fv) ? mag + 1 : mag - 1);   /* neighbour on s's side */
    double gv = kto_bf16_decode(g);
    if (s != (fv + gv) / 2.0) return f;                   /* not a midpoint: s rounds as the sum */
    return ((e > 0.0) == (gv > fv)) ? g : f;              /* midpoint: the exact sum lies on e's side */
}

static float gelu_arg_f32(float x)
{
    const float C0 = (float)sqrt(2.0 / M_PI);
    const float C1 = (float)(sqrt(2.0 / M_PI) * GELU_A);
    float x2 = x * x;
    float p = fmaf(C1, x2, C0);
    float u = x * p;
    return u;
}

uint32_t kto_gelu_consts(int which)   /* for the pin tests: bit patterns of C0, C1 */
{
    float C0 = (float)sqrt(2.0 / M_PI);
    float C1 = (float)(sqrt(2.0 / M_PI) * GELU_A);
    return which == 0 ? bits_from_f32(C0) : bits_from_f32(C1);
}

uint16_t kto_ksigmoid_bf16(uint16_t x, const int *TE, const int *Tr, const int *Tb)
{
    double xv = kto_bf16_decode(x);
    uint16_t h = kto_bf16_encode_rne(xv / 2.0);          /* x/2 in BF16 */
    uint16_t t = kto_ktanh_bf16(h, TE, Tr, Tb);          /* K-TanH(x/2) */
    double tv = kto_bf16_decode(t);
    return kto_bf16_encode_rne((1.0 + tv) / 2.0);
}

static uint32_t ksigmoid_f32_pb(uint32_t x, const int *TE, const int *Tr, const int *Tb, int pb)
{
    double xv = (double)f32_from_bits(x);
    float h = (float)(xv / 2.0);                          /* x/2 in F32 (RNE) */
    uint32_t t = ktanh_f32_pb(bits_from_f32(h), TE, Tr, Tb, pb);
    double tv = (double)f32_from_bits(t);
    return bits_from_f32((float)((1.0 + tv) / 2.0));
}

uint32_t kto_ksigmoid_f32(uint32_t x, const int *TE, const int *Tr, const int *Tb)
{
    return ksigmoid_f32_pb(x, TE, Tr, Tb, 7);
}

uint16_t kto_kswish_bf16(uint16_t x, const int *TE, const int *Tr, const int *Tb)
{
    double xv = kto_bf16_decode(x);
    uint16_t h = kto_bf16_encode_rne(xv / 2.0);
    uint16_t t = kto_ktanh_bf16(h, TE, Tr, Tb);
    double tv = kto_bf16_decode(t);
    const double hx = xv / 2.0;                           /* exact */
    return rnbf16_exact_sum(hx, hx * tv);                 /* RN_bf16(x (1+t)/2), product exact */
}

static uint32_t kswish_f32_pb(uint32_t x, const int *TE, const int *Tr, const int *Tb, int pb)
{
    double xv = (double)f32_from_bits(x);
    float h = (float)(xv / 2.0);
    uint32_t t = ktanh_f32_pb(bits_from_f32(h), TE, Tr, Tb, pb);
    double tv = (double)f32_from_bits(t);
    const double hx = xv / 2.0;                           /* exact */
    return bits_from_f32(rn32_exact_sum(hx, hx * tv));    /* RN32(x (1+t)/2), products exact */
}

uint32_t kto_kswish_f32(uint32_t x, const int *TE, const int *Tr, const int *Tb)
{
    return kswish_f32_pb(x, TE, Tr, Tb, 7);
}

uint16_t kto_kgelu_bf16(uint16_t x, const int *TE, const int *Tr, const int *Tb)
{
    double xv = kto_bf16_decode(x);
    float u = gelu_arg_f32((float)xv);                   /* exact widening of x */
    uint16_t ub = kto_bf16_encode_rne((double)u);        /* argument in BF16 */
    uint16_t t = kto_ktanh_bf16(ub, TE, Tr, Tb);
    double tv = kto_bf16_decode(t);
    const double hx = xv / 2.0;                           /* exact */
    return rnbf16_exact_sum(hx, hx * tv);                 /* RN_bf16(x/2 (1+t)), product exact */
}

static uint32_t kgelu_f32_pb(uint32_t x, const int *TE, const int *Tr, const int *Tb, int pb)
{
    float xf = f32_from_bits(x);
    float u = gelu_arg_f32(xf);
    uint32_t t = ktanh_f32_pb(bits_from_f32(u), TE, Tr, Tb, pb);
    double tv = (double)f32_from_bits(t);
    const double hx = (double)xf / 2.0;                   /* exact */
    return bits_from_f32(rn32_exact_sum(hx, hx * tv));    /* RN32(x/2 (1+t)) */
}

uint32_t kto_kgelu_f32(uint32_t x, const int *TE, const int *Tr, const int *Tb)
{
    return kgelu_f32_pb(x, TE, Tr, Tb, 7);
}

/* ------------------------------------------------------------------ */
/* Backward passes.  The paper trains GNMT with K-TanH */
/* but never states the gradient; reading R-BWD: the  */
/* derivative of the function K-TanH approximates, evaluated through the  */
/* K-TanH value, in binary64, rounded once to the format:                 */
/*   tanh:    dx = dy (1 - y^2),          y = saved K-TanH output         */
/*   sigmoid: dx = dy s (1 - s),          s = saved K-Sigmoid output      */
/*   swish:   dx = dy ((1+t)/2 + x (1-t^2)/4),  t = K-TanH(RN(x/2))       */
/*   gelu:    dx = dy ((1+t)/2 + x/2 (1-t^2) sqrt(2/pi)(1 + 3 a x^2)),   */
/*            t = K-TanH(u) with u as in the forward (R-GELU-ARG)         */
/* op: 0 tanh, 1 sigmoid, 2 swish, 3 gelu; a = saved output (0, 1) or the  */
/* input x (2, 3).                                                         */
/* ------------------------------------------------------------------ */
static double bwd_factor(int op, double a, double tv)
{
    const double c = sqrt(2.0 / M_PI), ga = GELU_A;
    switch (op) {
    case 0: return 1.0 - a * a;
    case 1: return a * (1.0 - a);
    case 2: return (1.0 + tv) / 2.0 + a * (1.0 - tv * tv) / 4.0;
    default: return (1.0 + tv) / 2.0 + a / 2.0 * (1.0 - tv * tv) * c * (1.0 + 3.0 * ga * a * a);
    }
}

uint16_t kto_bwd_bf16(int op, uint16_t a, uint16_t dy, const int *TE, const int *Tr, const int *Tb)
{
    double av = kto_bf16_decode(a), dv = kto_bf16_decode(dy), tv = 0.0;
    if (op == 2) {
        tv = kto_bf16_decode(kto_ktanh_bf16(kto_bf16_encode_rne(av / 2.0), TE, Tr, Tb));
    } else if (op == 3) {
        float u = gelu_arg_f32((float)av);
        tv = kto_bf16_decode(kto_ktanh_bf16(kto_bf16_encode_rne((double)u), TE, Tr, Tb));
    }
    return kto_bf16_encode_rne(dv * bwd_factor(op, av, tv));
}

static uint32_t bwd_f32_pb(int op, uint32_t a, uint32_t dy, const int *TE, const int *Tr,
                           const int *Tb, int pb)
{
    double av = (double)f32_from_bits(a), dv = (double)f32_from_bits(dy), tv = 0.0;
    if (op == 2) {
        float h = (float)(av / 2.0);
        tv = (double)f32_from_bits(ktanh_f32_pb(bits_from_f32(h), TE, Tr, Tb, pb));
    } else if (op == 3) {
        float u = gelu_arg_f32((float)av);
        tv = (double)f32_from_bits(ktanh_f32_pb(bits_from_f32(u), TE, Tr, Tb, pb));
    }
    return bits_from_f32((float)(dv * bwd_factor(op, av, tv)));
}

uint32_t kto_bwd_f32(int op, uint32_t a, uint32_t dy, const int *TE, const int *Tr, const int *Tb)
{
    return bwd_f32_pb(op, a, dy, TE, Tr, Tb, 7);
}

void kto_bwd_map_bf16(int op, const uint16_t *a, const uint16_t *dy, uint16_t *dx, size_t n,
                      const int *TE, const int *Tr, const int *Tb)
{
    for (size_t i = 0; i < n; ++i) dx[i] = kto_bwd_bf16(op, a[i], dy[i], TE, Tr, Tb);
}

void kto_bwd_map_f32_p(int op, const uint32_t *a, const uint32_t *dy, uint32_t *dx, size_t n,
                       const int *TE, const int *Tr, const int *Tb, int pb)
{
    for (size_t i = 0; i < n; ++i) dx[i] = bwd_f32_pb(op, a[i], dy[i], TE, Tr, Tb, pb);
}

void kto_bwd_map_f32(int op, const uint32_t *a, const uint32_t *dy, uint32_t *dx, size_t n,
                     const int *TE, const int *Tr, const int *Tb)
{
    kto_bwd_map_f32_p(op, a, dy, dx, n, TE, Tr, Tb, 7);
}

/* ------------------------------------------------------------------ */
/* Array entry points (loops over the scalar functions above).            */
/* op: 0 tanh, 1 sigmoid, 2 swish, 3 gelu (4: F32 only, tanh via BF16)   */
/* ------------------------------------------------------------------ */
void kto_map_bf16(int op, const uint16_t *x, uint16_t *y, size_t n,
                  const int *TE, const int *Tr, const int *Tb)
{
    for (size_t i = 0; i < n; ++i) {
        switch (op) {
        case 0: y[i] = kto_ktanh_bf16(x[i], TE, Tr, Tb); break;
        case 1: y[i] = kto_ksigmoid_bf16(x[i], TE, Tr, Tb); break;
        case 2: y[i] = kto_kswish_bf16(x[i], TE, Tr, Tb); break;
        default: y[i] = kto_kgelu_bf16(x[i], TE, Tr, Tb); break;
        }
    }
}

/* pb: unit of b_t, 7 (Table 1's tables, reading A8) or 23 (re-optimised   */
/* F32 tables); op 4 (via BF16) needs a BF16 table (pb = 7).               */
void kto_map_f32_p(int op, const uint32_t *x, uint32_t *y, size_t n,
                   const int *TE, const int *Tr, const int *Tb, int pb)
{
    for (size_t i = 0; i < n; ++i) {
        switch (op) {
        case 0: y[i] = ktanh_f32_pb(x[i], TE, Tr, Tb, pb); break;
        case 1: y[i] = ksigmoid_f32_pb(x[i], TE, Tr, Tb, pb); break;
        case 2: y[i] = kswish_f32_pb(x[i], TE, Tr, Tb, pb); break;
        case 4: y[i] = kto_ktanh_f32_via_bf16(x[i], TE, Tr, Tb); break;
        default: y[i] = kgelu_f32_pb(x[i], TE, Tr, Tb, pb); break;
        }
    }
}

void kto_map_f32(int op, const uint32_t *x, uint32_t *y, size_t n,
                 const int *TE, const int *Tr, const int *Tb)
{
    kto_map_f32_p(op, x, y, n, TE, Tr, Tb, 7);
}

/* Strided gather variant for sampled full-size checks: y[j] = f(x[idx[j]]). */
void kto_map_bf16_at(int op, const uint16_t *x, const uint64_t *idx, uint16_t *y, size_t m,
                     const int *TE, const int *Tr, const int *Tb)
{
    for (size_t j = 0; j < m; ++j) kto_map_bf16(op, &x[idx[j]], &y[j], 1, TE, Tr, Tb);
}

/* LSTM gate block (BASELINE.json config 4; GNMT LSTM):      */
/* x is [rows, 4*hidden]; quarter q of each row is K-TanH if q ==          */
/* tanh_quarter (the cell candidate g) else K-Sigmoid (gates i, f, o).     */
void kto_lstm_gates_bf16(const uint16_t *x, uint16_t *y, size_t rows, size_t hidden,
                         int tanh_quarter, const int *TE, const int *Tr, const int *Tb)
{
    size_t width = 4 * hidden;
    for (size_t row = 0; row < rows; ++row) {
        for (size_t col = 0; col < width; ++col) {
            size_t i = row * width + col;
            int q = (int)(col / hidden);
            y[i] = (q == tanh_quarter) ? kto_ktanh_bf16(x[i], TE, Tr, Tb)
                                       : kto_ksigmoid_bf16(x[i], TE, Tr, Tb);
        }
    }
}

/* Fused LSTM cell (GNMT LSTM), reading   */
/* R-LSTM-CELL: gates [rows, 4H] BF16 in i, f, g, o order; c_prev, c_next  */
/* [rows, H] F32; h_next [rows, H] BF16.                                   */
/*   i, f, o = K-Sigmoid_bf16(gate), g = K-TanH_bf16(gate)  (as above)     */
/*   c'  = RN32(f c + i g)             (exact sum, one rounding)           */
/*   h'  = RN_bf16(o K-TanH_f32(c'))   (F32 native reading A8, one rounding)*/
void kto_lstm_cell_bf16(const uint16_t *gates, const uint32_t *c_prev, uint32_t *c_next,
                        uint16_t *h_next, size_t rows, size_t hidden,
                        const int *TE, const int *Tr, const int *Tb)
{
    for (size_t r = 0; r < rows; ++r) {
        for (size_t j = 0; j < hidden; ++j) {
            const uint16_t *gr = gates + r * 4 * hidden;
            double i = kto_bf16_decode(kto_ksigmoid_bf16(gr[j], TE, Tr, Tb));
            double f = kto_bf16_decode(kto_ksigmoid_bf16(gr[hidden + j], TE, Tr, Tb));
            double g = kto_bf16_decode(kto_ktanh_bf16(gr[2 * hidden + j], TE, Tr, Tb));
            double o = kto_bf16_decode(kto_ksigmoid_bf16(gr[3 * hidden + j], TE, Tr, Tb));
            double c = (double)f32_from_bits(c_prev[r * hidden + j]);
            float cn = rn32_exact_sum(f * c, i * g);   /* products exact, one rounding */
            double t = (double)f32_from_bits(kto_ktanh_f32(bits_from_f32(cn), TE, Tr, Tb));
            c_next[r * hidden + j] = bits_from_f32(cn);
            h_next[r * hidden + j] = kto_bf16_encode_rne(o * t);
        }
    }
}

/* ------------------------------------------------------------------ */
/* Sec. 2.4 bounds, with p = 7 mantissa bits and       */
/* s = 3 index bits of the mantissa, v = mantissa_idx_val:                 */
/*   b_max = 2^p - 1 - floor(((v+1) 2^(p-s) - 1) / 2^r)                    */
/*   b_min = -v * floor(2^(p-s-r))          (Eq. 3; reading A16)           */
/* ------------------------------------------------------------------ */
void kto_bounds(int r, int v, int *bmin, int *bmax)
{
    const int p = 7, s = 3;
    *bmax = (1 << p) - 1 - (int)floor((double)((v + 1) * (1 << (p - s)) - 1) / ldexp(1.0, r));
    *bmin = -v * (int)floor(ldexp(1.0, p - s - r));
}

/* Eq. 3 / b_max with s index bits and p mantissa bits: */
/*   b_max = 2^p - 1 - floor(((v+1) 2^(p-s) - 1) / 2^r)                     */
/*   b_min = -v floor(2^(p-s-r))            (0 when r > p - s)              */
void kto_bounds_sp(int r, int v, int s_bits, int p, int *bmin, int *bmax)
{
    *bmax = (1 << p) - 1 - (int)((((int64_t)(v + 1) << (p - s_bits)) - 1) >> r);
    *bmin = r <= p - s_bits ? -v * (1 << (p - s_bits - r)) : 0;
}

void kto_bounds_s(int r, int v, int s_bits, int *bmin, int *bmax)
{
    kto_bounds_sp(r, v, s_bits, 7, bmin, bmax);
}

/* RNE of y > 0 to the p-bit format (p = 7: BFloat16, p = 23: Float32),    */
/* returned as biased exponent and mantissa fields.                        */
static void rne_fields(double y, int p, int *E, int *M)
{
    uint32_t u;
    if (p == 7) u = (uint32_t)kto_bf16_encode_rne(y) << 16;
    else u = bits_from_f32((float)y);                       /* C cast: RNE */
    *E = (int)((u >> 23) & 0xFF);
    *M = (int)((u & 0x7FFFFF) >> (23 - p));
}

/* floor(a / b) for b > 0 */
static __int128 floor_div(__int128 a, __int128 b)
{
    __int128 q = a / b;
    if ((a % b != 0) && (a < 0)) q -= 1;
    return q;
}

/* ------------------------------------------------------------------ */
/* Sec. 2.4 optimizer, Steps 1-3, reading R*, for s     */
/* mantissa index bits and inputs / outputs with p mantissa bits (p = 7:   */
/* BFloat16, the paper's case; p = 23: Float32 tables re-optimised for the */
/* native F32 path, SURVEY.md NEXT-3 -- the paper's text is written for a  */
/* general p: "p = 7 in case of BFloat16"):              */
/*  inputs: every positive x = 2^(E-127)(1 + M/2^p), T1 <= x <= T2, whose  */
/*     index ((E & 3) << s) | (M >> (p - s)) is t.                          */
/*  Step 1: y_i = tanh(x_i) in binary64, (E_i, M_i) =   */
/*     fields of RNE_p(y_i) (reading A12).                                 */
/*  Step 2: for each candidate E in {min(E_i, 126)}     */
/*     (reading A15), M^_j = M_j if E = E_j, 0 if E > E_j, 2^q - 1 if      */
/*     E < E_j (q = p); pick the E minimising sum (y_i - y^_i)^2 against   */
/*     the unrounded y_i; ties -> smaller E.                               */
/*  Step 3 (Eq. 2): for r = 0..r_max (= p):               */
/*     b* = mean(M^_i - m_i / 2^r) (real division as printed, A13),        */
/*     b = floor(b* + 1/2) (A14), clamped to [b_min, b_max]; score         */
/*     sum (M^_i - ((m_i >> r) + b))^2; keep the minimum, ties -> smaller r */
/*     (A17).  bmin_zero != 0 is the Sec. 3.1 ablation.      */
/* b* and the scores are computed exactly in 128-bit integers.  Returns    */
/* the per-interval minimum score in sse_out (may be NULL); returns 0, or  */
/* -1 for an unsupported (s, p).                                           */
/* ------------------------------------------------------------------ */
int kto_build_lut_sp(int s_bits, int p, int bmin_zero, int *TE, int *Tr, int *Tb, double *sse_out)
{
    if ((p != 7 && p != 23) || s_bits < 1 || s_bits > 5) return -1;
    const int q = p;
    const int nent = 4 << s_bits, per = 1 << (p - s_bits);
    double *xs = malloc(sizeof(double) * per), *ys = malloc(sizeof(double) * per);
    int *ms = malloc(sizeof(int) * per), *Ei = malloc(sizeof(int) * per);
    int *Mi = malloc(sizeof(int) * per), *Mhat = malloc(sizeof(int) * per);
    int *Mhat_best = malloc(sizeof(int) * per);
    for (int t = 0; t < nent; ++t) {
        int cnt = 0;
        for (int E = 125; E <= 128; ++E) {          /* T1 = 2^-2 <= x <= T2 < 2^2 */
            if ((E & 3) != (t >> s_bits)) continue;
            for (int j = 0; j < per; ++j) {
                int M = ((t & ((1 << s_bits) - 1)) << (p - s_bits)) | j;
                double xv = ldexp(1.0 + ldexp((double)M, -p), E - 127);
                if (xv < T1 || xv > T2) continue;
                xs[cnt] = xv;
                ms[cnt] = M;
                cnt++;
            }
        }
        if (cnt == 0) { TE[t] = 126; Tr[t] = 0; Tb[t] = 0; if (sse_out) sse_out[t] = 0; continue; }
        /* Step 1 */
        for (int i = 0; i < cnt; ++i) {
            ys[i] = tanh(xs[i]);
            rne_fields(ys[i], p, &Ei[i], &Mi[i]);
        }
        /* Step 2 (each distinct candidate once; a repeat scores the same) */
        int bestE = -1, tried[4] = {-1, -1, -1, -1}, ntried = 0;
        double bestSSE = INFINITY;
        for (int c = 0; c < cnt; ++c) {
            int E = Ei[c] < 126 ? Ei[c] : 126;
            int seen = 0;
            for (int k = 0; k < ntried; ++k) seen |= tried[k] == E;
            if (seen) continue;
            if (ntried < 4) tried[ntried++] = E;
            double sse = 0.0;
            for (int j = 0; j < cnt; ++j) {
                if (E == Ei[j]) Mhat[j] = Mi[j];
                else if (E > Ei[j]) Mhat[j] = 0;
                else Mhat[j] = (1 << q) - 1;
                double yhat = ldexp(1.0 + ldexp((double)Mhat[j], -q), E - 127);
                sse += (ys[j] - yhat) * (ys[j] - yhat);
            }
            if (sse < bestSSE || (sse == bestSSE && E < bestE)) {
                bestSSE = sse;
                bestE = E;
                memcpy(Mhat_best, Mhat, sizeof(int) * cnt);
            }
        }
        /* Step 3 */
        int v = t & ((1 << s_bits) - 1);
        int bestR = -1, bestB = 0;
        __int128 bestScore = -1;
        for (int r = 0; r <= p; ++r) {
            __int128 S = 0;                          /* cnt 2^r b* = sum(M^ 2^r - m) */
            for (int j = 0; j < cnt; ++j) S += ((__int128)Mhat_best[j] << r) - ms[j];
            int b = (int)floor_div(2 * S + ((__int128)cnt << r), (__int128)cnt << (r + 1));
            int bmin, bmax;
            kto_bounds_sp(r, v, s_bits, p, &bmin, &bmax);
            if (bmin_zero) bmin = 0;
            if (b < bmin) b = bmin;
            if (b > bmax) b = bmax;
            __int128 score = 0;
            for (int j = 0; j < cnt; ++j) {
                int64_t d = (int64_t)Mhat_best[j] - ((ms[j] >> r) + b);
                score += (__int128)(d * d);
            }
            if (bestScore < 0 || score < bestScore) {
                bestScore = score;
                bestR = r;
                bestB = b;
            }
        }
        TE[t] = bestE;
        Tr[t] = bestR;
        Tb[t] = bestB;
        if (sse_out) sse_out[t] = (double)bestScore;
    }
    free(xs); free(ys); free(ms); free(Ei); free(Mi); free(Mhat); free(Mhat_best);
    return 0;
}

void kto_build_lut_s(int s_bits, int bmin_zero, int *TE, int *Tr, int *Tb, double *sse_out)
{
    kto_build_lut_sp(s_bits, 7, bmin_zero, TE, Tr, Tb, sse_out);
}

void kto_build_lut(int bmin_zero, int *TE, int *Tr, int *Tb, double *sse_out)
{
    kto_build_lut_s(3, bmin_zero, TE, Tr, Tb, sse_out);
}

/* End-to-end squared error of one interval of a LUT against binary64 tanh */
/* (used by the dominance pin: the optimizer's rows vs the printed rows).  */
double kto_interval_sse(int t, const int *TE, const int *Tr, const int *Tb)
{
    double sse = 0.0;
    for (int w = 0; w < 0x7F80; ++w) {
        double xv = kto_bf16_decode((uint16_t)w);
        if (xv < T1 || xv > T2) continue;
        int E = (w >> 7) & 0xFF, M = w & 0x7F;
        if (index_t(E, M >> 4) != t) continue;
        double yv = kto_bf16_decode(kto_ktanh_bf16((uint16_t)w, TE, Tr, Tb));
        double d = yv - tanh(xv);
        sse += d * d;
    }
    return sse;
}
