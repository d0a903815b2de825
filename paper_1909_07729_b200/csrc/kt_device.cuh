// kt_device.cuh -- sm_100a device code for the K-TanH element maps.
//
// Everything here works on the input's BITS (Sec. 2.3):
// the BF16 core handles two elements packed in one 32-bit register, the F32
// core one element.  All selects are branch-free; the only memory touched
// per element is the streaming load/store in kt_kernels.cu, the parameter
// table lives in one register per lane and is read with a warp shuffle.
#pragma once

#include <cstdint>

#include "kt_internal.h"

namespace kt {

// ---------------------------------------------------------------- helpers --

// theta_t fetch (Alg. 1 line 7): lane t of the warp holds entry t.  The
// shuffle lane index is taken from bits [4:0] of `src_lane` (c = 0x1f, no
// segment mask), so callers pass `x >> 4` / `x >> 20` without masking.
__device__ __forceinline__ uint32_t shfl_lut(uint32_t lane_word, uint32_t src_lane) {
  uint32_t d;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;"
               : "=r"(d) : "r"(lane_word), "r"(src_lane));
  return d;
}

// a >> (n mod 32)   (one SHF.R.W; the LUT word keeps r_t in its low bits)
__device__ __forceinline__ uint32_t shr_wrap(uint32_t a, uint32_t n) {
  uint32_t d;
  asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(0u), "r"(n));
  return d;
}

// Per-half BF16 compares producing 0xFFFF / 0x0000 masks (HSET2.BF16_V2).
// ltu: less-than OR unordered -> NaN lands in the bypass mask (reading A6).
__device__ __forceinline__ uint32_t hset2_ltu(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("set.ltu.u32.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hset2_gt(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("set.gt.u32.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hset2_ne(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("set.ne.u32.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// hi32(a*b) and hi32(a*b) + c (IMAD.HI, FMA pipe)
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t madhi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// packed fp32x2 arithmetic (FMUL2 / FFMA2), round-to-nearest-even, no FTZ
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

// m ? a : b, bitwise (one LOP3)
__device__ __forceinline__ uint32_t bsel(uint32_t m, uint32_t a, uint32_t b) {
  return (m & a) | (~m & b);
}

// two fp32 -> packed bf16x2, round-to-nearest-even (F2FP.BF16.F32.PACK_AB)
__device__ __forceinline__ uint32_t pack_bf16x2(float hi, float lo) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
__device__ __forceinline__ float lo_f32(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float hi_f32(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
// the two BF16 of w widened exactly to fp32: .x = low half, .y = high half
__device__ __forceinline__ float2 widen2(uint32_t w) { return make_float2(lo_f32(w), hi_f32(w)); }
__device__ __forceinline__ uint32_t pack2(float2 v) { return pack_bf16x2(v.y, v.x); }
__device__ __forceinline__ float2 splat2(float a) { return make_float2(a, a); }

// Thresholds: T1 = 0.25 = 0x3E80, T2 = 3.75 = 0x4070 (BF16);
// 0x3E800000 / 0x40700000 (F32).  +-1 = (s, E_bias = 127, 0).
constexpr uint32_t kT1x2 = 0x3E803E80u;
constexpr uint32_t kT2x2 = 0x40704070u;
constexpr uint32_t kOnex2 = 0x3F803F80u;
constexpr uint32_t kSignx2 = 0x80008000u;
constexpr uint32_t kMagx2 = 0x7FFF7FFFu;
constexpr uint32_t kT1f = 0x3E800000u;
constexpr uint32_t kT2f = 0x40700000u;
constexpr uint32_t kInff = 0x7F800000u;

// GELU argument constants (a = 0.044715):
// C0 = RN32(sqrt(2/pi)), C1 = RN32(sqrt(2/pi) * a)
constexpr uint32_t kGeluC0Bits = 0x3F4C422Au;
constexpr uint32_t kGeluC1Bits = 0x3D122279u;

// ------------------------------------------------------------- K-TanH core --

// Algorithm 1 on two BF16 values packed in x.
//
// Line 8, M_o = (M >> r_t) + b_t with E_o = E_t, is computed by ONE fp32 add in
// round-toward-zero per element.  For a table-path input of exponent E_in the
// LUT word L_t = bits((2^(E_in + 16 + r_t - 127)) (1 + D_t / 2^23)), with
// D_t = ((E_t << 7) + b_t - 2^(7 - r_t)) mod 2^16, has ulp(L_t) = 2^r_t input
// mantissa ulps, so RZ(|x| + L_t) = L_t + floor(|x| / ulp) ulp and
//   low16(bits(RZ(|x| + L_t))) = D_t + 2^(7-r_t) + (M >> r_t) = (E_t << 7) + M_o.
// Bits of |x| below the BF16 mantissa add < 1 to the floored numerator
// (128 + M), so the high element can use the packed word as its fp32 operand
// directly.  The FADD runs on the FMA pipe; the ALU pipe only carries the two
// lane shifts, the pack and the masks/selects.  Exhaustively checked against
// the oracle (tests/test_gpu_parity.py).
//   lw = this lane's word LutWords::bf16[lane] = L_lane.
__device__ __forceinline__ uint32_t ktanh_bf16x2(uint32_t x, uint32_t lw, uint32_t &mag) {
  // line 6: t = bits [8:4] of each half = (E & 3) : (M >> 4)
  // line 7: theta_t by shuffle from lane t
  const uint32_t Ll = shfl_lut(lw, x >> 4);
  const uint32_t Lh = shfl_lut(lw, x >> 20);
  // line 8: (E_t, (M >> r_t) + b_t) in the low 16 bits of the RZ sums
  const float ql = __fadd_rz(fabsf(__uint_as_float(x << 16)), __uint_as_float(Ll));
  const float qh = __fadd_rz(fabsf(__uint_as_float(x)), __uint_as_float(Lh));
  const uint32_t ymag = __byte_perm(__float_as_uint(ql), __float_as_uint(qh), 0x5410);
  // lines 3-4: region masks per half.  |x| by abs.bf16x2, which ptxas
  // emits as HFMA2 (-0 * 0 + |x|) on the FMA pipe: one ALU op fewer per
  // pair than x & 0x7FFF7FFF (NaN stays NaN, subnormals compare as bypass
  // either way).  |x| is handed back to the caller (K-Swish/K-GELU reuse it).
  asm("abs.bf16x2 %0, %1;" : "=r"(mag) : "r"(x));
  const uint32_t byp = hset2_ltu(mag, kT1x2);      // |x| < T1, or NaN
  const uint32_t sat = hset2_gt(mag, kT2x2);       // |x| > T2, incl. inf
  const uint32_t m = bsel(sat, kOnex2, ymag);      // line 4: (s, E_bias, 0)
  const uint32_t o = bsel(byp, x, m);              // line 3: y = x
  return o | (x & kSignx2);                        // s_o = s_i
}
__device__ __forceinline__ uint32_t ktanh_bf16x2(uint32_t x, uint32_t lw) {
  uint32_t mag;
  return ktanh_bf16x2(x, lw, mag);
}

// Algorithm 1 with the 64-interval table of PAPER.md:223 (4 mantissa index
// bits): t = (E & 3) : (M >> 3) = bits [8:3] of each half.
// Lane i holds entries i (w0) and 32 + i (w1); both are shuffled from lane
// t & 31 and bit 5 of t (bit 8 of the half) picks one.  The words have the
// same form as the 32-entry ones (the RZ-add identity does not depend on the
// number of index bits).
__device__ __forceinline__ uint32_t ktanh64_bf16x2(uint32_t x, uint32_t w0, uint32_t w1) {
  const uint32_t il = x >> 3, ih = x >> 19;
  const uint32_t l0 = shfl_lut(w0, il), l1 = shfl_lut(w1, il);
  const uint32_t h0 = shfl_lut(w0, ih), h1 = shfl_lut(w1, ih);
  const uint32_t Ll = (x & 0x100u) ? l1 : l0;
  const uint32_t Lh = (x & 0x1000000u) ? h1 : h0;
  const float ql = __fadd_rz(fabsf(__uint_as_float(x << 16)), __uint_as_float(Ll));
  const float qh = __fadd_rz(fabsf(__uint_as_float(x)), __uint_as_float(Lh));
  const uint32_t ymag = __byte_perm(__float_as_uint(ql), __float_as_uint(qh), 0x5410);
  uint32_t mag;
  asm("abs.bf16x2 %0, %1;" : "=r"(mag) : "r"(x));
  const uint32_t byp = hset2_ltu(mag, kT1x2);
  const uint32_t sat = hset2_gt(mag, kT2x2);
  const uint32_t m = bsel(sat, kOnex2, ymag);
  const uint32_t o = bsel(byp, x, m);
  return o | (x & kSignx2);
}

// Algorithm 1 on one F32 (native reading A8).  lk = f32K[lane], lc = f32C[lane].
// The region tests compare u << 1 (|x| shifted up, sign dropped -- it is the
// umulhi operand anyway, computed on the FMA pipe) instead of masking |x|:
// bypass (|x| < T1 or NaN) is ONE unsigned range test
// (u2 - 2 T1) > (2 inf - 2 T1); the sign is ORed in once after the
// saturation select.  6 ALU-pipe ops instead of 10.
__device__ __forceinline__ uint32_t ktanh_f32(uint32_t u, uint32_t lk, uint32_t lc, uint32_t &u2out) {
  const uint32_t K = shfl_lut(lk, u >> 20);        // line 6-7, t = bits [24:20]
  const uint32_t C = shfl_lut(lc, u >> 20);
  const uint32_t u2 = u << 1;
  u2out = u2;                                      // |x| << 1 (the tie screen's key)
  const uint32_t ym = __umulhi(u2, K) + C;         // line 8: C_t + (|x| >> r_t)
  uint32_t y = (u2 > (kT2f << 1)) ? 0x3F800000u : ym;                  // line 4
  y |= u & 0x80000000u;                                                // s_o = s_i
  const bool byp = (u2 - (kT1f << 1)) > ((kInff << 1) - (kT1f << 1));  // line 3, or NaN (A6)
  return byp ? u : y;
}
__device__ __forceinline__ uint32_t ktanh_f32(uint32_t u, uint32_t lk, uint32_t lc) {
  uint32_t u2;
  return ktanh_f32(u, lk, lc, u2);
}

// ------------------------------------------------------- derived (Sec. 1) --
// PAPER.md:60-71.  Sigmoid(x) = (1 + TanH(x/2))/2, Swish = x Sigmoid(x),
// GELU ~= x/2 (1 + TanH(sqrt(2/pi)(x + a x^3))).  fp32 scaffolding with
// explicit _rn intrinsics (no contraction), one rounding to the format.

// Packed BF16 arithmetic (HMUL2/HFMA2.BF16, FMA pipe): the exact result
// rounded once to BF16 (RNE), subnormals kept.
__device__ __forceinline__ uint32_t hmul2_bf16(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hfma2_bf16(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
constexpr uint32_t kHalfx2 = 0x3F003F00u;   // (0.5, 0.5) in BF16

// K-Sigmoid: h = RN_bf16(x/2) and RN_bf16((1 + t)/2) each in ONE packed BF16
// instruction (exact product / fma rounded once) instead of widen + fp32 op +
// pack: 2 FMA-pipe ops per pair instead of 2 FMA + 6 ALU.  Same values as the
// fp32 route (x/2 is exact in fp32; 0.5 t + 0.5 is exact in fp32 whenever
// the BF16 rounding could be affected), checked over all 65,536 patterns.
__device__ __forceinline__ uint32_t ksigmoid_bf16x2(uint32_t x, uint32_t lw) {
  const uint32_t h = hmul2_bf16(x, kHalfx2);                              // RN_bf16(x/2)
  const uint32_t t = ktanh_bf16x2(h, lw);
  return hfma2_bf16(t, kHalfx2, kHalfx2);                                 // RN((1+t)/2)
}

// K-Swish / K-GELU outer step y = RN_bf16(x/2 (1 + t)), the exact value
// rounded once (reading R-DERIVED).  With h = RN_bf16(x/2) (one packed mul),
// one packed fma RN_bf16(h + h t) IS that value whenever x/2 is a BF16, i.e.
// for every x except |x| < 2^-125 with an odd last bit, where x/2 is a BF16
// tie.  There t is tiny with the sign of x, so the exact term (x/2) t > 0
// breaks the tie toward +inf (when t != 0): r = x - 2h (exact, +-1 subnormal
// ulp) is > 0 exactly when h was rounded down, and the addend becomes h + r.
//   outer_exact:  3 FMA-pipe + 3 ALU ops more than the plain fma, exact for
//                 every x (the element-wise paths and the GEMM epilogue).
//   streaming kernels: the plain fma, plus ONE packed-u16 min per pair over the
//                 |argument| the K-TanH core computes anyway (|x/2| or
//                 |RN_bf16(u)|); a warp whose minimum is < 0x100 in some half
//                 (an argument below 2^-125, or a zero) re-reads x and patches
//                 the pairs with |x| < 2^-125 from the closed form tie_patch
//                 (never taken on the bench's N(0,1) data).
constexpr uint32_t kNegTwox2 = 0xC000C000u;   // (-2, -2) in BF16

__device__ __forceinline__ uint32_t outer_exact(uint32_t x, uint32_t h, uint32_t t) {
  const uint32_t r = hfma2_bf16(h, kNegTwox2, x);                     // x - 2h, exact
  const uint32_t up = hset2_gt(r, 0u) & hset2_ne(t, 0u) & kOnex2;     // 1.0 where the t-term rounds up
  return hfma2_bf16(h, t, hfma2_bf16(r, up, h));                      // RN(h t + (h + [up] r))
}

__device__ __forceinline__ uint32_t umin16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// some half of the running minimum of |argument| is < 0x100 (2^-125)
__device__ __forceinline__ bool tie_possible(uint32_t kmin) {
  return (kmin & 0xFF00u) == 0 || (kmin & 0xFF000000u) == 0;
}

// Closed form of the exact outer step for |x| < 2^-125 (magnitude bits
// m < 0x100 are then linear in 2^-133 units, x/2 = m/2 units, t is tiny with
// the sign s of x): y = s | ((m + 1 - s) >> 1), except K-Swish at m = 1 where
// t = K-TanH(RN(x/2)) = 0 and the tie goes to even (0).  y (the plain-fma
// result) is kept for every half with |x| >= 2^-125.
template <int OP>
__device__ __forceinline__ uint32_t tie_patch(uint32_t x, uint32_t y) {
  uint32_t out = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t xv = (x >> (16 * k)) & 0xFFFFu, m = xv & 0x7FFFu, s = xv & 0x8000u;
    uint32_t yv = (y >> (16 * k)) & 0xFFFFu;
    if (m < 0x100u) {
      const uint32_t inc = (s == 0 && (OP == OP_GELU || m >= 2)) ? 1u : 0u;
      yv = s | ((m + inc) >> 1);
    }
    out |= yv << (16 * k);
  }
  return out;
}

// plain-fma forms (exact unless tie_patch applies); mag = |argument| of the
// K-TanH core (the caller folds it into the tie screen's running minimum)
__device__ __forceinline__ uint32_t kswish_bf16x2_fast(uint32_t x, uint32_t lw, uint32_t &mag) {
  const uint32_t h = hmul2_bf16(x, kHalfx2);                              // RN_bf16(x/2)
  const uint32_t t = ktanh_bf16x2(h, lw, mag);
  return hfma2_bf16(h, t, h);                                             // RN(h (1+t))
}

__device__ __forceinline__ uint32_t kswish_bf16x2(uint32_t x, uint32_t lw) {
  const uint32_t h = hmul2_bf16(x, kHalfx2);
  const uint32_t t = ktanh_bf16x2(h, lw);
  return outer_exact(x, h, t);
}

__device__ __forceinline__ float gelu_arg(float x) {
  const float x2 = __fmul_rn(x, x);
  const float p = __fmaf_rn(__uint_as_float(kGeluC1Bits), x2, __uint_as_float(kGeluC0Bits));
  return __fmul_rn(x, p);
}

// t = K-TanH(RN_bf16(u)) of the GELU argument (R-GELU-ARG, fp32x2), |RN_bf16(u)| in mag
__device__ __forceinline__ uint32_t kgelu_t_bf16x2(uint32_t x, uint32_t lw, uint32_t &mag) {
  const float2 xv = widen2(x);
  const float2 x2 = mul2(xv, xv);
  const float2 p = fma2(splat2(__uint_as_float(kGeluC1Bits)), x2, splat2(__uint_as_float(kGeluC0Bits)));
  return ktanh_bf16x2(pack2(mul2(xv, p)), lw, mag);                       // RN_bf16(u)
}

__device__ __forceinline__ uint32_t kgelu_bf16x2_fast(uint32_t x, uint32_t lw, uint32_t &mag) {
  const uint32_t t = kgelu_t_bf16x2(x, lw, mag);   // |x| < 2^-125 => |RN(u)| < 0xCD ulps
  const uint32_t h = hmul2_bf16(x, kHalfx2);                              // RN_bf16(x/2)
  return hfma2_bf16(h, t, h);                                             // RN(h (1+t))
}

__device__ __forceinline__ uint32_t kgelu_bf16x2(uint32_t x, uint32_t lw) {
  uint32_t mag;
  const uint32_t t = kgelu_t_bf16x2(x, lw, mag);
  return outer_exact(x, hmul2_bf16(x, kHalfx2), t);
}

__device__ __forceinline__ uint32_t ksigmoid_f32(uint32_t u, uint32_t lk, uint32_t lc) {
  const float h = __fmul_rn(__uint_as_float(u), 0.5f);
  const float t = __uint_as_float(ktanh_f32(__float_as_uint(h), lk, lc));
  return __float_as_uint(__fmaf_rn(0.5f, t, 0.5f));
}

// F32 outer step y = RN32(x/2 (1 + t)), exact (R-DERIVED): hx = RN32(x/2) is
// x/2 except for |x| < 2^-125 with an odd last bit (an F32 tie); as for BF16
// the exact t-term (sign of x, t != 0) then breaks the tie toward +inf.
// r = x - 2 hx is exact (0 or +-1 subnormal ulp).  4 more ops per element
// than fma(hx, t, hx); the F32 derived ops are not on the headline path.
__device__ __forceinline__ float outer_exact_f32(float x, float hx, float t) {
  const float r = __fmaf_rn(hx, -2.0f, x);
  const float c = (r > 0.0f && t != 0.0f) ? __fadd_rn(hx, r) : hx;
  return __fmaf_rn(hx, t, c);
}

__device__ __forceinline__ uint32_t kswish_f32(uint32_t u, uint32_t lk, uint32_t lc) {
  const float x = __uint_as_float(u);
  const float hx = __fmul_rn(x, 0.5f);
  const float t = __uint_as_float(ktanh_f32(__float_as_uint(hx), lk, lc));
  return __float_as_uint(outer_exact_f32(x, hx, t));
}

__device__ __forceinline__ uint32_t kgelu_f32(uint32_t u, uint32_t lk, uint32_t lc) {
  const float x = __uint_as_float(u);
  const float t = __uint_as_float(ktanh_f32(__float_as_uint(gelu_arg(x)), lk, lc));
  const float hx = __fmul_rn(x, 0.5f);
  return __float_as_uint(outer_exact_f32(x, hx, t));
}

// F32 streaming forms with the tie screen (as for BF16): the plain fma, and
// key = |argument| << 1 from the core; a key below 2^-125 << 1 (or a zero)
// sends the warp's chunk through tie_patch_f32.
constexpr uint32_t kTieKeyF32 = 0x01000000u << 1;   // (2^-125 bits) << 1
__device__ __forceinline__ uint32_t kswish_f32_fast(uint32_t u, uint32_t lk, uint32_t lc, uint32_t &key) {
  const float hx = __fmul_rn(__uint_as_float(u), 0.5f);
  const float t = __uint_as_float(ktanh_f32(__float_as_uint(hx), lk, lc, key));
  return __float_as_uint(__fmaf_rn(hx, t, hx));
}
__device__ __forceinline__ uint32_t kgelu_f32_fast(uint32_t u, uint32_t lk, uint32_t lc, uint32_t &key) {
  const float x = __uint_as_float(u);
  const float t = __uint_as_float(ktanh_f32(__float_as_uint(gelu_arg(x)), lk, lc, key));
  const float hx = __fmul_rn(x, 0.5f);
  return __float_as_uint(__fmaf_rn(hx, t, hx));
}
// closed form for |x| < 2^-125 (bits m < 0x01000000 linear in 2^-149 units),
// as tie_patch for BF16
template <int OP>
__device__ __forceinline__ uint32_t tie_patch_f32(uint32_t x, uint32_t y) {
  const uint32_t m = x & 0x7FFFFFFFu, s = x & 0x80000000u;
  if (m >= 0x01000000u) return y;
  const uint32_t inc = (s == 0 && (OP == OP_GELU || m >= 2)) ? 1u : 0u;
  return s | ((m + inc) >> 1);
}

// ------------------------------------------------------- backward (NEXT-1) --
// Reading R-BWD: derivative of the approximated function, taken
// through the K-TanH value; fp32 with a fixed op order, one rounding to the
// format.  a = saved output y (tanh, sigmoid) or the input x (swish, gelu).
//   tanh:    dx = dy * fma(-y, y, 1)
//   sigmoid: dx = dy * fma(-s, s, s)
//   swish:   t = K(RN(x/2)),  g = fma(x/4, fma(-t, t, 1), fma(t, 1/2, 1/2))
//   gelu:    t = K(RN(u)),    g = fma((x/2) fma(-t, t, 1), fma(C3, x^2, C0), fma(t, 1/2, 1/2))
//            with C0 = RN32(sqrt(2/pi)), C3 = RN32(3 sqrt(2/pi) 0.044715)
constexpr uint32_t kGeluC3Bits = 0x3DDB33B6u;

__device__ __forceinline__ float2 neg2(float2 v) { return make_float2(-v.x, -v.y); }

template <int OP>
__device__ __forceinline__ float2 bwd_factor2(float2 av, uint32_t a, uint32_t lw) {
  if (OP == OP_TANH) return fma2(neg2(av), av, splat2(1.0f));
  if (OP == OP_SIGMOID) return fma2(neg2(av), av, av);
  const float2 half = splat2(0.5f);
  if (OP == OP_SWISH) {
    const float2 hx = mul2(av, half);
    const float2 t = widen2(ktanh_bf16x2(pack2(hx), lw));
    return fma2(mul2(hx, half), fma2(neg2(t), t, splat2(1.0f)), fma2(t, half, half));
  }
  // GELU
  const float2 x2 = mul2(av, av);
  const float2 p = fma2(splat2(__uint_as_float(kGeluC1Bits)), x2, splat2(__uint_as_float(kGeluC0Bits)));
  const float2 t = widen2(ktanh_bf16x2(pack2(mul2(av, p)), lw));
  // x^2 clamped to FLT_MAX for u' only: where it overflows, t = +-1 and the
  // term (x/2)(1 - t^2) u' must be exactly 0 (not 0 * inf)
  const float2 x2c = make_float2(fminf(x2.x, 3.4028235e38f), fminf(x2.y, 3.4028235e38f));
  const float2 up = fma2(splat2(__uint_as_float(kGeluC3Bits)), x2c, splat2(__uint_as_float(kGeluC0Bits)));
  const float2 hx = mul2(av, half);
  return fma2(mul2(hx, fma2(neg2(t), t, splat2(1.0f))), up, fma2(t, half, half));
}

template <int OP>
__device__ __forceinline__ uint32_t bwd_bf16x2(uint32_t a, uint32_t dy, uint32_t lw) {
  const float2 g = bwd_factor2<OP>(widen2(a), a, lw);
  return pack2(mul2(widen2(dy), g));
}

template <int OP>
__device__ __forceinline__ uint32_t bwd_f32(uint32_t a, uint32_t dy, const uint32_t lk, const uint32_t lc) {
  const float av = __uint_as_float(a);
  float g;
  if (OP == OP_TANH) {
    g = __fmaf_rn(-av, av, 1.0f);
  } else if (OP == OP_SIGMOID) {
    g = __fmaf_rn(-av, av, av);
  } else if (OP == OP_SWISH) {
    const float hx = __fmul_rn(av, 0.5f);
    const float t = __uint_as_float(ktanh_f32(__float_as_uint(hx), lk, lc));
    g = __fmaf_rn(__fmul_rn(hx, 0.5f), __fmaf_rn(-t, t, 1.0f), __fmaf_rn(t, 0.5f, 0.5f));
  } else {
    const float x2 = __fmul_rn(av, av);
    const float t = __uint_as_float(ktanh_f32(__float_as_uint(gelu_arg(av)), lk, lc));
    const float up = __fmaf_rn(__uint_as_float(kGeluC3Bits), fminf(x2, 3.4028235e38f),
                               __uint_as_float(kGeluC0Bits));
    const float hx = __fmul_rn(av, 0.5f);
    g = __fmaf_rn(__fmul_rn(hx, __fmaf_rn(-t, t, 1.0f)), up, __fmaf_rn(t, 0.5f, 0.5f));
  }
  return __float_as_uint(__fmul_rn(__uint_as_float(dy), g));
}

// ------------------------------------------------------------- dispatch ----

struct LaneLut {
  uint32_t w16, k32, c32;
};

template <int OP>
__device__ __forceinline__ uint32_t apply_bf16x2(uint32_t x, const LaneLut &L) {
  if (OP == OP_TANH) return ktanh_bf16x2(x, L.w16);
  if (OP == OP_SIGMOID) return ksigmoid_bf16x2(x, L.w16);
  if (OP == OP_SWISH) return kswish_bf16x2(x, L.w16);
  return kgelu_bf16x2(x, L.w16);
}

// Streaming form: K-Swish / K-GELU BF16 take the plain-fma outer step and
// return |argument| in mag (the kernel folds it into the screen's minimum and
// patches a flagged warp's chunk with tie_patch); every other op is
// apply_word itself (mag = all ones).
// KT_TIE_MODE (dev A/B builds only): 0 = tie screen (default), 1 = the exact
// outer step on every pair, 2 = the plain fma with no screen (NOT exact on
// the x/2 ties; measures the screen's cost).
#ifndef KT_TIE_MODE
#define KT_TIE_MODE 0
#endif
template <int OP>
__device__ __forceinline__ uint32_t apply_bf16x2_fast(uint32_t x, const LaneLut &L, uint32_t &mag) {
  mag = 0xFFFFFFFFu;
#if KT_TIE_MODE == 1
  return apply_bf16x2<OP>(x, L);
#else
  uint32_t m = 0xFFFFFFFFu;
  uint32_t r;
  if (OP == OP_SWISH) r = kswish_bf16x2_fast(x, L.w16, m);
  else if (OP == OP_GELU) r = kgelu_bf16x2_fast(x, L.w16, m);
  else r = apply_bf16x2<OP>(x, L);
  if (KT_TIE_MODE == 0) mag = m;
  return r;
#endif
}

// K-TanH of an F32 value through BF16 (the A8 alternative;
// PAPER.md:256 "We assume BFloat16 input ... conversion cost is not
// considered"): RNE to BF16 (F2FP), Alg. 1 on the BF16 bits, widen exactly.
__device__ __forceinline__ uint32_t ktanh_f32_via_bf16(uint32_t u, uint32_t lw) {
  const uint32_t b = pack_bf16x2(0.0f, __uint_as_float(u));     // low half = RN_bf16(x)
  return ktanh_bf16x2(b, lw) << 16;
}

template <int OP>
__device__ __forceinline__ uint32_t apply_f32(uint32_t u, const LaneLut &L) {
  if (OP == OP_TANH_VIA_BF16) return ktanh_f32_via_bf16(u, L.w16);
  if (OP == OP_TANH) return ktanh_f32(u, L.k32, L.c32);
  if (OP == OP_SIGMOID) return ksigmoid_f32(u, L.k32, L.c32);
  if (OP == OP_SWISH) return kswish_f32(u, L.k32, L.c32);
  return kgelu_f32(u, L.k32, L.c32);
}

// One 32-bit word: two BF16 or one F32.
template <int OP, int FMT>
__device__ __forceinline__ uint32_t apply_word(uint32_t w, const LaneLut &L) {
  if (FMT == FMT_BF16) return apply_bf16x2<OP>(w, L);
  return apply_f32<OP>(w, L);
}

template <int OP, int FMT>
__device__ __forceinline__ uint32_t apply_word_fast(uint32_t w, const LaneLut &L, uint32_t &mag) {
  mag = 0xFFFFFFFFu;
  if (FMT == FMT_BF16) return apply_bf16x2_fast<OP>(w, L, mag);
#if KT_TIE_MODE != 1
  uint32_t k = 0xFFFFFFFFu, r;
  if (OP == OP_SWISH) r = kswish_f32_fast(w, L.k32, L.c32, k);
  else if (OP == OP_GELU) r = kgelu_f32_fast(w, L.k32, L.c32, k);
  else r = apply_f32<OP>(w, L);
  if (KT_TIE_MODE == 0) mag = k;
  return r;
#else
  return apply_f32<OP>(w, L);
#endif
}
// the tie screen's running minimum and test, per format: BF16 keys are two
// packed u16 magnitudes, F32 keys one |argument| << 1
template <int FMT>
__device__ __forceinline__ uint32_t key_min(uint32_t a, uint32_t b) {
  return FMT == FMT_BF16 ? umin16x2(a, b) : (a < b ? a : b);
}
template <int FMT>
__device__ __forceinline__ bool tie_possible_fmt(uint32_t kmin) {
  return FMT == FMT_BF16 ? tie_possible(kmin) : kmin < kTieKeyF32;
}
// closed-form patch of one word (x in, plain-fma y in) for the format
template <int OP, int FMT>
__device__ __forceinline__ uint32_t tie_patch_word(uint32_t x, uint32_t y) {
  return FMT == FMT_BF16 ? tie_patch<OP>(x, y) : tie_patch_f32<OP>(x, y);
}
template <int FMT>
__device__ __forceinline__ bool tie_word_candidate(uint32_t w) {   // some |x| < 2^-125 in the word
  return FMT == FMT_BF16 ? ((w & 0x7F00u) == 0 || (w & 0x7F000000u) == 0) : (w & 0x7F000000u) == 0;
}
// does apply_word_fast need the tie screen for this op/format?
template <int OP, int FMT>
__host__ __device__ constexpr bool needs_tie_screen() {
  return OP == OP_SWISH || OP == OP_GELU;
}

template <int OP, int FMT>
__device__ __forceinline__ uint32_t apply_bwd_word(uint32_t a, uint32_t dy, const LaneLut &L) {
  if (FMT == FMT_BF16) return bwd_bf16x2<OP>(a, dy, L.w16);
  return bwd_f32<OP>(a, dy, L.k32, L.c32);
}

// ------------------------------------------------- fused LSTM cell (NEXT-2) --
// Reading R-LSTM-CELL: i, f, o = K-Sigmoid, g = K-TanH on the BF16
// gates; c' = RN32(f c + i g) (i g is exact in fp32, one fma); h' =
// RN_bf16(o K-TanH_f32(c')) computed exactly: the fp32 product is taken
// round-toward-zero and made round-to-odd with the fma residual, so the one
// rounding to BF16 is correct (24 >= 8 + 2 bits).
__device__ __forceinline__ float mul_rodd(float a, float b) {
  const float p = __fmul_rz(a, b);
  const float r = __fmaf_rn(a, b, -p);                  // exact residual
  uint32_t pb = __float_as_uint(p);
  // sticky bit as a predicated OR (FSETP + @P LOP3, no SEL: the cell kernel
  // 20.33 -> 20.00 us, profiles/cell_variants_r01.txt)
  asm("{\n\t.reg .pred q;\n\tsetp.ne.f32 q, %1, 0f00000000;\n\t@q or.b32 %0, %0, 1;\n\t}"
      : "+r"(pb) : "f"(r));
  return __uint_as_float(pb);
}

// 2 cells: gate words gi, gf, gg, go (BF16 pairs), c (2 floats) -> c', h (BF16 pair)
__device__ __forceinline__ uint32_t lstm_cell2(uint32_t gi, uint32_t gf, uint32_t gg, uint32_t go,
                                               float2 c, float2 &cn, const LaneLut &L) {
  const float2 iv = widen2(ksigmoid_bf16x2(gi, L.w16));
  const float2 fv = widen2(ksigmoid_bf16x2(gf, L.w16));
  const float2 gv = widen2(ktanh_bf16x2(gg, L.w16));
  const float2 ov = widen2(ksigmoid_bf16x2(go, L.w16));
  cn = fma2(fv, c, mul2(iv, gv));
  const float tl = __uint_as_float(ktanh_f32(__float_as_uint(cn.x), L.k32, L.c32));
  const float th = __uint_as_float(ktanh_f32(__float_as_uint(cn.y), L.k32, L.c32));
  return pack_bf16x2(mul_rodd(ov.y, th), mul_rodd(ov.x, tl));
}

// LSTM gate pair: K-TanH (is_tanh) or K-Sigmoid, same core, per-lane choice.
__device__ __forceinline__ uint32_t lstm_bf16x2(uint32_t x, uint32_t lw, bool is_tanh) {
  const uint32_t h = is_tanh ? x : hmul2_bf16(x, kHalfx2);
  const uint32_t t = ktanh_bf16x2(h, lw);
  return is_tanh ? t : hfma2_bf16(t, kHalfx2, kHalfx2);
}

// ------------------------------------------------------ streaming memory --

// L2 eviction-priority qualifiers for the streaming loads / stores (default
// policy; dev A/B builds: -DKT_LD_EF=1 / -DKT_ST_EF=1 evict_first,
// -DKT_ST_EL=1 evict_last).
#if defined(KT_LD_EF) && KT_LD_EF
#define KT_LD_L2 ".L2::evict_first"
#else
#define KT_LD_L2 ""
#endif
#if defined(KT_ST_EF) && KT_ST_EF
#define KT_ST_L2 ".L2::evict_first"
#elif defined(KT_ST_EL) && KT_ST_EL
#define KT_ST_L2 ".L2::evict_last"
#else
#define KT_ST_L2 ""
#endif

// 32-byte (256-bit) predicated global load / store (LDG.E.256 / STG.E.256).
// NC: read-only non-coherent path, used only when y does not alias x.
template <bool NC>
__device__ __forceinline__ void ld256(const void *p, uint32_t (&r)[8], bool pred) {
  if (NC) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
        "@p ld.global.nc.L1::no_allocate" KT_LD_L2 ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p), "r"((int)pred));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
        "@p ld.global.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p), "r"((int)pred)
        : "memory");
  }
}

__device__ __forceinline__ void st256(void *p, const uint32_t (&r)[8], bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %9, 0;\n\t"
      "@p st.global.L1::no_allocate" KT_ST_L2 ".v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n\t}" ::"l"(p),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"((int)pred)
      : "memory");
}

}  // namespace kt
