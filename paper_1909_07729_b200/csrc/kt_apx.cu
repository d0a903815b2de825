// kt_apx.cu -- the float-op TanH approximations that Table 2 of the paper
// compares K-TanH with (Sec. 2.1-2.2, PAPER.md:115-137;
// SURVEY.md NEXT-4), as sm_100a streaming kernels, plus the host code that
// derives their coefficients.  Readings R-CMP-* in DESIGN.md.
//
//   Pade [p/q]        y = x N(x^2) / D(x^2), IEEE division, saturating to +-1
//                     at |x| >= X_p (first point where R reaches 1 or peaks).
//                     Coefficients: convergents of Lambert's continued fraction
//                     tanh x = x/(1 + x^2/(3 + x^2/(5 + ...))), in integers.
//   minimax deg n     16 pieces of width 1/2 on [0, 8), Remez exchange per
//                     piece (piece 0 with P(0) = 0); |x| >= 8 -> +-1.
//   Taylor deg n      same layout; piece 0 = Maclaurin, piece k >= 1 about its
//                     midpoint k/2 + 1/4; coefficients from the derivative
//                     polynomials of tanh in T = tanh(m).
//   libm              tanhf() of the CUDA math library (the "SVML high
//                     precision" row's GPU analogue).
//   sfu               tanh.approx (MUFU.TANH; bf16x2 for BF16): the hardware
//                     approximation (the "SVML low precision" analogue).
//
// Everything is odd-extended (sign of x restored by a bit OR) and NaN passes
// through unchanged, as for K-TanH (reading A6).  BF16 inputs are widened
// exactly to fp32, evaluated in fp32, and rounded once (RNE) to BF16.
//
// Streaming shape = the K-TanH kernels' (kt_kernels.cu): one warp per 2 KiB
// chunk, 256-bit loads/stores, flat grid, PDL, L2 prefetch in the first wave;
// piecewise coefficients are held one piece per lane and fetched with warp
// shuffles (4 per element), Pade coefficients are uniform kernel parameters.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>

#include "kt_device.cuh"
#include "kt_internal.h"

namespace kt {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 2;
constexpr int kVecBytes = 32;
constexpr int kChunkVecs = 32 * kUnroll;

// ---------------------------------------------------------------- device --

__device__ __forceinline__ uint32_t shfl_f(float v, uint32_t lane) {
  return __shfl_sync(0xffffffffu, __float_as_uint(v), (int)lane);
}

// This lane's coefficient j (piece = lane).  The empty volatile asm makes the
// register value opaque: otherwise the compiler may rematerialise it inside
// loops as a lane-indexed (divergent, serialised) constant-bank load -- seen
// in SASS as LDC c[0x0][Rlane + ...] per round, 3x slower.
__device__ __forceinline__ float lane_coef(const ApxWords &w, int j, uint32_t lane) {
  float v = w.pc[j][lane];
  asm volatile("" : "+f"(v));
  return v;
}

// Magnitude maps a >= 0 (not NaN) -> approximation of tanh(a) in [0, 1].

// Piecewise polynomial: k = floor(2a) via one round-toward-zero FMA
// (2a + 2^23 keeps floor(2a) in the low mantissa bits for 2a < 2^23), h exact.
template <int KIND, int DEG>
__device__ __forceinline__ float pw_mag(float a, const float (&c)[4]) {
  const float kf = __fmaf_rz(a, 2.0f, 8388608.0f);
  const uint32_t k = __float_as_uint(kf) & 15u;
  const float fk = __fsub_rn(kf, 8388608.0f);          // floor(2a), exact
  float h = __fmaf_rn(fk, -0.5f, a);                   // a - k/2, exact
  if (KIND == APX_TAYLOR) h = __fsub_rn(h, k != 0 ? 0.25f : 0.0f);   // about the midpoint, exact
  float y = __uint_as_float(shfl_f(c[DEG], k));
#pragma unroll
  for (int j = DEG - 1; j >= 0; --j) y = __fmaf_rn(y, h, __uint_as_float(shfl_f(c[j], k)));
  y = fminf(fmaxf(y, 0.0f), 1.0f);
  return a >= 8.0f ? 1.0f : y;
}

// Pade: y = a N(s) / D(s), s = a^2 (ND/DD = degrees in s).
template <int ND, int DD>
__device__ __forceinline__ float pade_mag(float a, const ApxWords &w) {
  const float s = __fmul_rn(a, a);
  float N = w.num[ND], D = w.den[DD];
#pragma unroll
  for (int j = ND - 1; j >= 0; --j) N = __fmaf_rn(N, s, w.num[j]);
#pragma unroll
  for (int j = DD - 1; j >= 0; --j) D = __fmaf_rn(D, s, w.den[j]);
  const float y = fminf(__fdiv_rn(__fmul_rn(a, N), D), 1.0f);
  return a >= w.xsat ? 1.0f : y;
}

__device__ __forceinline__ float sfu_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// KIND x (Pade degrees or polynomial degree) selector
template <int KIND, int A, int B>
__device__ __forceinline__ float apx_mag(float a, const float (&c)[4], const ApxWords &w) {
  if (KIND == APX_PADE) return pade_mag<A, B>(a, w);
  if (KIND == APX_LIBM) return tanhf(a);
  return pw_mag<KIND, A>(a, c);
}

// one F32 word
template <int KIND, int A, int B>
__device__ __forceinline__ uint32_t apx_f32(uint32_t u, const float (&c)[4], const ApxWords &w) {
  const uint32_t mag = u & 0x7FFFFFFFu;
  float y;
  if (KIND == APX_SFU) {
    y = sfu_tanh(__uint_as_float(u));
    return mag > kInff ? u : __float_as_uint(y);
  }
  y = apx_mag<KIND, A, B>(__uint_as_float(mag), c, w);
  return mag > kInff ? u : (__float_as_uint(y) | (u & 0x80000000u));
}

// two BF16 in one word
template <int KIND, int A, int B>
__device__ __forceinline__ uint32_t apx_bf16x2(uint32_t x, const float (&c)[4], const ApxWords &w) {
  uint32_t nan;   // 0xFFFF per NaN half
  asm("set.nan.u32.bf16x2 %0, %1, %1;" : "=r"(nan) : "r"(x));
  if (KIND == APX_SFU) {
    uint32_t y;
    asm("tanh.approx.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
    return bsel(nan, x, y);
  }
  const uint32_t mag = x & kMagx2;
  const float lo = apx_mag<KIND, A, B>(lo_f32(mag), c, w);
  const float hi = apx_mag<KIND, A, B>(hi_f32(mag), c, w);
  const uint32_t y = pack_bf16x2(hi, lo) | (x & kSignx2);
  return bsel(nan, x, y);
}

template <int KIND, int A, int B, int FMT>
__device__ __forceinline__ uint32_t apx_word(uint32_t w32, const float (&c)[4], const ApxWords &w) {
  if (FMT == FMT_BF16) return apx_bf16x2<KIND, A, B>(w32, c, w);
  return apx_f32<KIND, A, B>(w32, c, w);
}

__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// An empty volatile asm that "modifies" every loaded register: it stays after
// the (volatile) loads, and all arithmetic depends on its outputs.
__device__ __forceinline__ void after_loads(uint32_t (&v)[2][8]) {
  asm volatile(""
               : "+r"(v[0][0]), "+r"(v[0][1]), "+r"(v[0][2]), "+r"(v[0][3]), "+r"(v[0][4]),
                 "+r"(v[0][5]), "+r"(v[0][6]), "+r"(v[0][7]), "+r"(v[1][0]), "+r"(v[1][1]),
                 "+r"(v[1][2]), "+r"(v[1][3]), "+r"(v[1][4]), "+r"(v[1][5]), "+r"(v[1][6]),
                 "+r"(v[1][7]));
}

__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <int KIND, int A, int B, int FMT>
__device__ __forceinline__ void apx_span(const uint8_t *xp, uint8_t *yp, uint32_t cnt,
                                         const float (&c)[4], const ApxWords &w) {
  const uint32_t lane = threadIdx.x & 31;
  const bool on = lane < cnt;
  uint32_t v = 0;
  if (FMT == FMT_BF16) {
    if (on) v = reinterpret_cast<const uint16_t *>(xp)[lane];
  } else if (on) {
    v = reinterpret_cast<const uint32_t *>(xp)[lane];
  }
  const uint32_t r = apx_word<KIND, A, B, FMT>(v, c, w);
  if (on) {
    if (FMT == FMT_BF16) reinterpret_cast<uint16_t *>(yp)[lane] = (uint16_t)r;
    else reinterpret_cast<uint32_t *>(yp)[lane] = r;
  }
}

// Flat streaming kernel (see k_map in kt_kernels.cu for the shape).
template <int KIND, int A, int B, int FMT, bool NC>
__global__ void __launch_bounds__(kThreads)
k_apx(const uint8_t *x, uint8_t *y, uint32_t head, uint64_t nvec, uint32_t tail,
      uint32_t pf_blocks, const __grid_constant__ ApxWords w) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const uint32_t lane = threadIdx.x & 31;
  float c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = lane_coef(w, j, lane);
  const uint8_t *xb = x + (size_t)head * es;
  uint8_t *yb = y + (size_t)head * es;
  const uint64_t ch = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (NC && blockIdx.x < pf_blocks && lane == 0 && ch * kChunkVecs < nvec) {
    const uint64_t left = nvec - ch * kChunkVecs;
    prefetch_l2(xb + ch * kChunkVecs * kVecBytes,
                (uint32_t)((left < kChunkVecs ? left : kChunkVecs) * kVecBytes));
  }
  pdl_enter();
  const uint64_t base = ch * kChunkVecs + lane;
  uint32_t v[kUnroll][8];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    ld256<NC>(xb + i * kVecBytes, v[u], i < nvec);
  }
  // Keep both loads in flight before any compute: the last-loaded vector is
  // processed first (ptxas otherwise schedules the first vector's arithmetic
  // between the two loads, serialising them; measured minimax-3 BF16 3.4 TB/s).
  after_loads(v);
#pragma unroll
  for (int u = kUnroll - 1; u >= 0; --u) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[u][j] = apx_word<KIND, A, B, FMT>(v[u][j], c, w);
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    st256(yb + i * kVecBytes, v[u], i < nvec);
  }
  if ((head | tail) != 0 && blockIdx.x == 0 && threadIdx.x < 32) {
    apx_span<KIND, A, B, FMT>(x, y, head, c, w);
    const size_t toff = ((size_t)head + (size_t)nvec * (kVecBytes / es)) * es;
    apx_span<KIND, A, B, FMT>(x + toff, y + toff, tail, c, w);
  }
}

// Persistent, software-pipelined variant for the compute-heavy maps: each
// warp walks chunks c, c + stride, ... and loads chunk c + stride while it
// computes and stores chunk c, so memory traffic overlaps the arithmetic
// within the warp (the flat one-chunk-per-warp shape leaves a compute-bound
// map at ~55% of both ALU and HBM rate).
#ifndef KT_APX_PIPE_MINB
#define KT_APX_PIPE_MINB 3   // <= 80 regs, 3 CTAs/SM: minimax-3 BF16 1140 -> 1214 Gelem/s (apx_stream_r01.txt)
#endif
template <int KIND, int A, int B, int FMT, bool NC>
__global__ void __launch_bounds__(kThreads, KT_APX_PIPE_MINB)
k_apx_pipe(const uint8_t *x, uint8_t *y, uint32_t head, uint64_t nvec, uint32_t tail,
           const __grid_constant__ ApxWords w) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const uint32_t lane = threadIdx.x & 31;
  float c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = lane_coef(w, j, lane);
  const uint8_t *xb = x + (size_t)head * es;
  uint8_t *yb = y + (size_t)head * es;
  const uint64_t nch = (nvec + kChunkVecs - 1) / kChunkVecs;
  const uint64_t stride = (uint64_t)gridDim.x * kWarps;
  uint64_t ch = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  pdl_enter();
  uint32_t a[kUnroll][8], b[kUnroll][8];
  auto load = [&](uint64_t cc, uint32_t (&v)[kUnroll][8]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t i = cc * kChunkVecs + lane + (uint64_t)u * 32;
      ld256<NC>(xb + i * kVecBytes, v[u], cc < nch && i < nvec);
    }
  };
  auto work = [&](uint64_t cc, uint32_t (&v)[kUnroll][8]) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[u][j] = apx_word<KIND, A, B, FMT>(v[u][j], c, w);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t i = cc * kChunkVecs + lane + (uint64_t)u * 32;
      st256(yb + i * kVecBytes, v[u], i < nvec);
    }
  };
  load(ch, a);
  while (ch < nch) {
    load(ch + stride, b);
    work(ch, a);
    ch += stride;
    if (ch >= nch) break;
    load(ch + stride, a);
    work(ch, b);
    ch += stride;
  }
  if ((head | tail) != 0 && blockIdx.x == 0 && threadIdx.x < 32) {
    apx_span<KIND, A, B, FMT>(x, y, head, c, w);
    const size_t toff = ((size_t)head + (size_t)nvec * (kVecBytes / es)) * es;
    apx_span<KIND, A, B, FMT>(x + toff, y + toff, tail, c, w);
  }
}

// x and y with different offsets mod 32 B: element-wise, grid-stride.
template <int KIND, int A, int B, int FMT>
__global__ void __launch_bounds__(kThreads)
k_apx_elem(const uint8_t *x, uint8_t *y, uint64_t n, const __grid_constant__ ApxWords w) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const uint32_t lane = threadIdx.x & 31;
  float c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = lane_coef(w, j, lane);
  pdl_enter();
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t ch = warp0; ch < (n + 31) / 32; ch += nwarps) {
    const uint64_t off = ch * 32, rem = n - off;
    apx_span<KIND, A, B, FMT>(x + off * es, y + off * es, (uint32_t)(rem < 32 ? rem : 32), c, w);
  }
}

// ------------------------------------------------------------------ host --

// Launch shape per map (KT_APX_PIPE=0/1 forces flat/pipelined): the
// pipelined persistent kernel for the maps whose arithmetic per element is
// comparable to its memory time, flat otherwise (profiles/apx_*_r01.txt).
bool apx_pipelined(int kind, int fmt) {
  static const int force = [] {
    const char *e = getenv("KT_APX_PIPE");
    return e ? atoi(e) : -1;
  }();
  if (force >= 0) return force != 0;
  (void)fmt;
  return kind == APX_MINIMAX || kind == APX_TAYLOR;   // 4 shuffles + Horner per element
}

template <class K>
int occupancy(K kernel) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, kThreads, 0) != cudaSuccess || b < 1)
    b = 1;
  return b;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), unsigned grid, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
  count_launch();
  return e;
}

template <int KIND, int A, int B, int FMT>
cudaError_t launch_apx_t(const void *x, void *y, size_t n, const ApxWords &w, cudaStream_t s,
                         const LaunchInfo &li) {
  constexpr size_t es = (FMT == FMT_BF16) ? 2 : 4;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
  const uint8_t *xp = static_cast<const uint8_t *>(x);
  uint8_t *yp = static_cast<uint8_t *>(y);
  if ((xa % kVecBytes) != (ya % kVecBytes)) {
    const uint64_t chunks = (n + 31) / 32;
    const uint64_t maxw = (uint64_t)li.sm_count * 8 * kWarps * 4;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, (std::min(chunks, maxw) + kWarps - 1) / kWarps);
    return launch_k(k_apx_elem<KIND, A, B, FMT>, grid, s, xp, yp, (uint64_t)n, w);
  }
  const size_t mis = xa % kVecBytes;
  size_t head = mis ? (kVecBytes - mis) / es : 0;
  if (head > n) head = n;
  const size_t body = n - head;
  const uint64_t nvec = body / (kVecBytes / es);
  const uint32_t tail = (uint32_t)(body - nvec * (kVecBytes / es));
  const uint64_t nchunks = (nvec + kChunkVecs - 1) / kChunkVecs;
  if (nchunks / kWarps >= 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, (nchunks + kWarps - 1) / kWarps);
  if (apx_pipelined(w.kind, FMT)) {
    if (x != y) {
      static const int bps = occupancy(k_apx_pipe<KIND, A, B, FMT, true>);   // thread-safe init
      const unsigned pgrid = std::min<unsigned>(grid, (unsigned)(li.sm_count * bps));
      return launch_k(k_apx_pipe<KIND, A, B, FMT, true>, pgrid, s, xp, yp, (uint32_t)head, nvec,
                      tail, w);
    }
    static const int bps = occupancy(k_apx_pipe<KIND, A, B, FMT, false>);
    const unsigned pgrid = std::min<unsigned>(grid, (unsigned)(li.sm_count * bps));
    return launch_k(k_apx_pipe<KIND, A, B, FMT, false>, pgrid, s, xp, yp, (uint32_t)head, nvec, tail,
                    w);
  }
  if (x != y) {
    const uint32_t pf = prefetch_enabled() ? (uint32_t)li.sm_count * 8u : 0u;   // 8 CTAs/SM resident
    return launch_k(k_apx<KIND, A, B, FMT, true>, grid, s, xp, yp, (uint32_t)head, nvec, tail, pf, w);
  }
  return launch_k(k_apx<KIND, A, B, FMT, false>, grid, s, xp, yp, (uint32_t)head, nvec, tail, 0u, w);
}

template <int FMT>
cudaError_t launch_apx_fmt(const void *x, void *y, size_t n, const ApxWords &w, cudaStream_t s,
                           const LaunchInfo &li) {
  switch (w.kind) {
  case APX_PADE: {
    // degrees in s = x^2: N has (p-1)/2, D has q/2
    const int nd = (w.p - 1) / 2, dd = w.q / 2;
#define KT_PADE(NDv, DDv) \
  if (nd == NDv && dd == DDv) return launch_apx_t<APX_PADE, NDv, DDv, FMT>(x, y, n, w, s, li);
    KT_PADE(0, 0) KT_PADE(0, 1) KT_PADE(1, 1) KT_PADE(1, 2) KT_PADE(2, 2) KT_PADE(2, 3)
    KT_PADE(3, 3) KT_PADE(3, 4) KT_PADE(4, 4) KT_PADE(4, 5)
#undef KT_PADE
    return cudaErrorInvalidValue;
  }
  case APX_MINIMAX:
    if (w.p == 1) return launch_apx_t<APX_MINIMAX, 1, 0, FMT>(x, y, n, w, s, li);
    if (w.p == 2) return launch_apx_t<APX_MINIMAX, 2, 0, FMT>(x, y, n, w, s, li);
    if (w.p == 3) return launch_apx_t<APX_MINIMAX, 3, 0, FMT>(x, y, n, w, s, li);
    return cudaErrorInvalidValue;
  case APX_TAYLOR:
    if (w.p == 1) return launch_apx_t<APX_TAYLOR, 1, 0, FMT>(x, y, n, w, s, li);
    if (w.p == 2) return launch_apx_t<APX_TAYLOR, 2, 0, FMT>(x, y, n, w, s, li);
    if (w.p == 3) return launch_apx_t<APX_TAYLOR, 3, 0, FMT>(x, y, n, w, s, li);
    return cudaErrorInvalidValue;
  case APX_LIBM:
    return launch_apx_t<APX_LIBM, 0, 0, FMT>(x, y, n, w, s, li);
  case APX_SFU:
    return launch_apx_t<APX_SFU, 0, 0, FMT>(x, y, n, w, s, li);
  default:
    return cudaErrorInvalidValue;
  }
}

// ---- coefficient generation (host, long double) ---------------------------

typedef long double ld;

ld poly_ld(const ld *c, int deg, ld x) {
  ld s = c[deg];
  for (int i = deg - 1; i >= 0; --i) s = s * x + c[i];
  return s;
}

// Lambert convergent j: tanh x ~ x N_j(s) / D_j(s), s = x^2, with
// N_j = (2j-1) N_{j-1} + s N_{j-2}, D_j likewise; N_0 = 0, N_1 = 1, D_0 = D_1 = 1.
// Integer coefficients (exact for j <= 10).  Returns degrees in s.
void lambert(int j, int64_t *N, int *nd, int64_t *D, int *dd) {
  int64_t Nm2[8] = {0}, Nm1[8] = {1}, Dm2[8] = {1}, Dm1[8] = {1};
  for (int i = 2; i <= j; ++i) {
    int64_t Nn[8] = {0}, Dn[8] = {0};
    for (int k = 0; k < 8; ++k) {
      Nn[k] = (2 * i - 1) * Nm1[k] + (k > 0 ? Nm2[k - 1] : 0);
      Dn[k] = (2 * i - 1) * Dm1[k] + (k > 0 ? Dm2[k - 1] : 0);
    }
    memcpy(Nm2, Nm1, sizeof(Nm1)); memcpy(Nm1, Nn, sizeof(Nn));
    memcpy(Dm2, Dm1, sizeof(Dm1)); memcpy(Dm1, Dn, sizeof(Dn));
  }
  if (j <= 0) { Nm1[0] = 0; }
  memcpy(N, Nm1, sizeof(Nm1));
  memcpy(D, Dm1, sizeof(Dm1));
  *nd = 0; *dd = 0;
  for (int k = 0; k < 8; ++k) {
    if (N[k]) *nd = k;
    if (D[k]) *dd = k;
  }
}

// First x > 0 with R(x) >= 1 or R'(x) <= 0 (reading R-CMP-SAT), R = x N(x^2)/D(x^2).
ld pade_xsat(const ld *N, int nd, const ld *D, int dd) {
  auto R = [&](ld x) { return x * poly_ld(N, nd, x * x) / poly_ld(D, dd, x * x); };
  auto stop = [&](ld x) {
    const ld h = x * 1e-7L;
    return R(x) >= 1.0L || R(x + h) <= R(x);
  };
  ld prev = 0.0L;
  for (int i = 1; i <= 64 * 256; ++i) {
    const ld x = i / 256.0L;
    if (stop(x)) {
      ld lo = prev, hi = x;
      // refine: R >= 1 crossing by bisection; a maximum by bisection on the
      // sign of R' (analytic: (xN)' D - xN D')
      auto dR = [&](ld t) {
        const ld s = t * t;
        ld Nv = poly_ld(N, nd, s), Dv = poly_ld(D, dd, s), dN = 0, dD = 0;
        for (int k = nd; k >= 1; --k) dN = dN * s + k * N[k];
        for (int k = dd; k >= 1; --k) dD = dD * s + k * D[k];
        // d/dt [t N(t^2)] = N + 2 t^2 N'(s);  d/dt D(t^2) = 2 t D'(s)
        return (Nv + 2 * s * dN) * Dv - t * Nv * 2 * t * dD;
      };
      for (int it = 0; it < 200; ++it) {
        const ld m = 0.5L * (lo + hi);
        if (m <= lo || m >= hi) break;
        if (R(m) >= 1.0L || dR(m) <= 0.0L) hi = m; else lo = m;
      }
      return hi;
    }
    prev = x;
  }
  return 64.0L;
}

// Gaussian elimination with partial pivoting (n <= 8).
bool gauss(int n, ld (*A)[9], ld *b, ld *x) {
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r) if (fabsl(A[r][c]) > fabsl(A[p][c])) p = r;
    if (A[p][c] == 0) return false;
    if (p != c) { for (int k = 0; k < n; ++k) std::swap(A[p][k], A[c][k]); std::swap(b[p], b[c]); }
    for (int r = c + 1; r < n; ++r) {
      const ld f = A[r][c] / A[c][c];
      for (int k = c; k < n; ++k) A[r][k] -= f * A[c][k];
      b[r] -= f * b[c];
    }
  }
  for (int r = n - 1; r >= 0; --r) {
    ld s = b[r];
    for (int k = r + 1; k < n; ++k) s -= A[r][k] * x[k];
    x[r] = s / A[r][r];
  }
  return true;
}

// Remez exchange for one piece [lo, lo + w]: c[j] (powers of h = x - lo),
// j0 = 1 fixes c[0] = 0.  Extrema of the error are located as zeros of e'
// (Newton, safeguarded by bisection) between sign changes on a grid.
bool remez_piece(int deg, ld lo, ld w, int j0, ld *c, ld *Eout) {
  const int m = deg + 1 - j0, np = m + 1;
  ld ref[8];
  for (int i = 0; i < np; ++i) {
    const ld t = (j0 == 0) ? (ld)i / (np - 1) : (ld)(i + 1) / np;
    ref[i] = lo + w * 0.5L * (1.0L - cosl(3.14159265358979323846264338L * t));
  }
  for (int j = 0; j < 4; ++j) c[j] = 0;
  auto P = [&](ld h) { ld s = 0; for (int j = deg; j >= 0; --j) s = s * h + c[j]; return s; };
  auto dP = [&](ld h) { ld s = 0; for (int j = deg; j >= 1; --j) s = s * h + j * c[j]; return s; };
  auto d2P = [&](ld h) { ld s = 0; for (int j = deg; j >= 2; --j) s = s * h + j * (j - 1) * c[j]; return s; };
  auto e = [&](ld x) { return tanhl(x) - P(x - lo); };
  auto de = [&](ld x) { const ld t = tanhl(x); return (1 - t * t) - dP(x - lo); };
  auto d2e = [&](ld x) { const ld t = tanhl(x); return -2 * t * (1 - t * t) - d2P(x - lo); };
  for (int it = 0; it < 60; ++it) {
    ld A[8][9], b[8], sol[8];
    for (int i = 0; i < np; ++i) {
      const ld h = ref[i] - lo;
      ld pw = 1;
      for (int j = 0; j < j0; ++j) pw *= h;
      for (int u = 0; u < m; ++u) { A[i][u] = pw; pw *= h; }
      A[i][m] = (i & 1) ? -1.0L : 1.0L;
      b[i] = tanhl(ref[i]);
    }
    if (!gauss(np, A, b, sol)) return false;
    for (int u = 0; u < m; ++u) c[u + j0] = sol[u];
    *Eout = fabsl(sol[m]);
    // candidate extrema: interior zeros of e', plus the endpoints
    ld ex[80];
    int ne = 0;
    if (j0 == 0) ex[ne++] = lo;
    const int G = 64;
    ld xa = lo, da = de(lo);
    for (int g = 1; g <= G && ne < 78; ++g) {
      const ld xb = lo + w * g / G, db = de(xb);
      if ((da > 0) != (db > 0) && da != 0) {
        ld l = xa, r = xb, x = 0.5L * (l + r);
        for (int k = 0; k < 100; ++k) {
          const ld f = de(x), f2 = d2e(x);
          if ((f > 0) == (da > 0)) l = x; else r = x;
          ld xn = (f2 != 0) ? x - f / f2 : 0.5L * (l + r);
          if (!(xn > l && xn < r)) xn = 0.5L * (l + r);
          if (fabsl(xn - x) <= 1e-18L * fabsl(x) + 1e-30L) { x = xn; break; }
          x = xn;
        }
        ex[ne++] = x;
      }
      xa = xb; da = db;
    }
    ex[ne++] = lo + w;
    // alternation: merge same-sign neighbours, keep the larger |e|
    ld ev[80];
    int na = 0;
    for (int i = 0; i < ne; ++i) {
      const ld v = e(ex[i]);
      if (na > 0 && (v > 0) == (ev[na - 1] > 0)) {
        if (fabsl(v) > fabsl(ev[na - 1])) { ex[na - 1] = ex[i]; ev[na - 1] = v; }
      } else {
        ex[na] = ex[i]; ev[na] = v; ++na;
      }
    }
    if (na < np) return false;
    int f = 0, l = na - 1;
    while (l - f + 1 > np) { if (fabsl(ev[f]) < fabsl(ev[l])) ++f; else --l; }
    ld emax = 0, emin = 1e300L;
    for (int i = 0; i < np; ++i) {
      ref[i] = ex[f + i];
      emax = std::max(emax, fabsl(ev[f + i]));
      emin = std::min(emin, fabsl(ev[f + i]));
    }
    if (emax - emin <= 1e-12L * emax + 1e-19L) break;
  }
  return true;
}

// Taylor coefficients of tanh about m: d^j tanh / dx^j = D_j(T), T = tanh(m),
// D_0 = T, D_{j+1} = D_j'(T) (1 - T^2); c_j = D_j(T) / j!.
void taylor_coeffs(ld m, int deg, ld *c) {
  ld Dp[8] = {0, 1};          // polynomial in T, D_0 = T
  const ld T = tanhl(m);
  ld fact = 1;
  for (int j = 0; j <= deg; ++j) {
    if (j > 0) fact *= j;
    c[j] = poly_ld(Dp, 7, T) / fact;
    ld d[8] = {0}, nx[8] = {0};
    for (int k = 1; k < 8; ++k) d[k - 1] = k * Dp[k];
    for (int k = 0; k < 8; ++k) {      // nx = d * (1 - T^2)
      nx[k] += d[k];
      if (k + 2 < 8) nx[k + 2] -= d[k];
    }
    memcpy(Dp, nx, sizeof(nx));
  }
  for (int j = deg + 1; j < 4; ++j) c[j] = 0;
}


// ---- in-register throughput probe (kt_alu_probe) --------------------------
// Every thread holds 16 words in registers and applies the map to each, for
// `iters` rounds, XOR-accumulating the results (no memory traffic in the
// loop).  Round it perturbs the low mantissa bits (w + (it & 3) per value) so
// the compiler cannot hoist the map out of the loop while the region mix of
// the input stays that of the data.  One wave (grid = SMs x resident CTAs);
// each CTA records its clock64 span.  WHICH: 0 identity (loop overhead),
// 1 K-TanH (Alg. 1), 2 a comparator.
template <int WHICH, int KIND, int A, int B, int FMT>
__global__ void __launch_bounds__(kThreads)
k_alu(const uint32_t *in, uint32_t *out, long long *cyc, int iters,
      const __grid_constant__ LutWords lw, const __grid_constant__ ApxWords w) {
  const uint32_t lane = threadIdx.x & 31;
  LaneLut L{lw.bf16[lane], lw.f32K[lane], lw.f32C[lane]};
  asm volatile("" : "+r"(L.w16), "+r"(L.k32), "+r"(L.c32));   // see lane_coef
  float c[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = lane_coef(w, j, lane);
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = in[(t * 16 + j) & 4095];
  uint32_t acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0;
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const uint32_t off = (FMT == FMT_BF16) ? (uint32_t)(it & 3) * 0x00010001u : (uint32_t)(it & 3);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t x = v[j] + off;
      uint32_t r;
      if (WHICH == 0) r = x;
      else if (WHICH == 1) r = apply_word<OP_TANH, FMT>(x, L);
      else r = apx_word<KIND, A, B, FMT>(x, c, w);
      acc[j] ^= r;           // 16 independent chains
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t a = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) a ^= acc[j];
  out[t] = a;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int WHICH, int KIND, int A, int B, int FMT>
cudaError_t alu_run(const uint32_t *in, uint32_t *out, long long *cyc, int iters, const LutWords &lw,
                    const ApxWords &w, int sms, int *grid_out, int *bps_out) {
  auto k = k_alu<WHICH, KIND, A, B, FMT>;
  int bps = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, kThreads, 0);
  if (e != cudaSuccess) return e;
  if (bps < 1) bps = 1;
  *grid_out = sms * bps;
  *bps_out = bps;
  k<<<sms * bps, kThreads>>>(in, out, cyc, iters, lw, w);
  count_launch();
  return cudaGetLastError();
}

template <int WHICH, int FMT>
cudaError_t alu_dispatch(const uint32_t *in, uint32_t *out, long long *cyc, int iters,
                         const LutWords &lw, const ApxWords &w, int sms, int *g, int *b) {
  if (WHICH != 2) return alu_run<WHICH, 0, 0, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
  switch (w.kind) {
  case APX_PADE: {
    const int nd = (w.p - 1) / 2, dd = w.q / 2;
#define KT_PADE(NDv, DDv) \
  if (nd == NDv && dd == DDv) return alu_run<2, APX_PADE, NDv, DDv, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
    KT_PADE(0, 0) KT_PADE(0, 1) KT_PADE(1, 1) KT_PADE(1, 2) KT_PADE(2, 2) KT_PADE(2, 3)
    KT_PADE(3, 3) KT_PADE(3, 4) KT_PADE(4, 4) KT_PADE(4, 5)
#undef KT_PADE
    return cudaErrorInvalidValue;
  }
  case APX_MINIMAX:
    if (w.p == 1) return alu_run<2, APX_MINIMAX, 1, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
    if (w.p == 2) return alu_run<2, APX_MINIMAX, 2, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
    return alu_run<2, APX_MINIMAX, 3, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
  case APX_TAYLOR:
    if (w.p == 1) return alu_run<2, APX_TAYLOR, 1, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
    if (w.p == 2) return alu_run<2, APX_TAYLOR, 2, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
    return alu_run<2, APX_TAYLOR, 3, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
  case APX_LIBM:
    return alu_run<2, APX_LIBM, 0, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
  case APX_SFU:
    return alu_run<2, APX_SFU, 0, 0, FMT>(in, out, cyc, iters, lw, w, sms, g, b);
  default:
    return cudaErrorInvalidValue;
  }
}

}  // namespace

// Synchronous: allocates a small scratch, runs the identity loop and the map
// in one wave each on the current device, returns SM cycles per element per
// SM for the map, net of the loop overhead (and gross).
cudaError_t alu_probe(int which, int fmt, const LutWords &lw, const ApxWords &w, int iters,
                      const uint32_t *host_in4096, double *cyc_net, double *cyc_gross, int sms) {
  uint32_t *in = nullptr, *out = nullptr;
  long long *cyc = nullptr;
  cudaError_t e;
  const int maxgrid = sms * 16;
  if ((e = cudaMalloc(&in, 4096 * 4)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&out, (size_t)maxgrid * kThreads * 4)) != cudaSuccess) { cudaFree(in); return e; }
  if ((e = cudaMalloc(&cyc, (size_t)maxgrid * 8)) != cudaSuccess) { cudaFree(in); cudaFree(out); return e; }
  double res[2] = {0, 0};
  e = cudaMemcpy(in, host_in4096, 4096 * 4, cudaMemcpyHostToDevice);
  for (int pass = 0; pass < 2 && e == cudaSuccess; ++pass) {
    const int wh = pass == 0 ? 0 : which;
    double best = 1e300;
    for (int rep = 0; rep < 3 && e == cudaSuccess; ++rep) {
      int grid = 0, bps = 0;
      if (fmt == FMT_BF16)
        e = wh == 0 ? alu_dispatch<0, FMT_BF16>(in, out, cyc, iters, lw, w, sms, &grid, &bps)
          : wh == 1 ? alu_dispatch<1, FMT_BF16>(in, out, cyc, iters, lw, w, sms, &grid, &bps)
                    : alu_dispatch<2, FMT_BF16>(in, out, cyc, iters, lw, w, sms, &grid, &bps);
      else
        e = wh == 0 ? alu_dispatch<0, FMT_F32>(in, out, cyc, iters, lw, w, sms, &grid, &bps)
          : wh == 1 ? alu_dispatch<1, FMT_F32>(in, out, cyc, iters, lw, w, sms, &grid, &bps)
                    : alu_dispatch<2, FMT_F32>(in, out, cyc, iters, lw, w, sms, &grid, &bps);
      if (e != cudaSuccess) break;
      if (grid > maxgrid) { e = cudaErrorInvalidConfiguration; break; }
      long long hc[16 * 1024];
      if ((e = cudaMemcpy(hc, cyc, (size_t)grid * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) break;
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = std::max(mx, hc[i]);
      const double elems_per_sm = (double)bps * kThreads * 16 * (fmt == FMT_BF16 ? 2 : 1) * iters;
      best = std::min(best, (double)mx / elems_per_sm);
    }
    res[pass] = best;
  }
  cudaFree(in);
  cudaFree(out);
  cudaFree(cyc);
  if (e != cudaSuccess) return e;
  *cyc_gross = res[1];
  *cyc_net = res[1] - res[0];
  return cudaSuccess;
}


bool apx_build(int kind, int p, int q, ApxWords *w, double *coef, char *err, size_t errlen) {
  memset(w, 0, sizeof(*w));
  w->kind = kind;
  w->p = p;
  w->q = q;
  for (int i = 0; i < kApxCoef; ++i) coef[i] = 0.0;
  if (kind == APX_PADE) {
    int j = -1;
    if (p >= 1 && (p & 1) && q >= 0 && !(q & 1)) {
      if (q == p + 1) j = q;
      else if (q == p - 1) j = p;
    }
    if (j < 1 || j > 10) {
      snprintf(err, errlen, "Pade [%d/%d] unsupported: need p odd, q = p +- 1 even, p + q <= 19", p,
               q);
      return false;
    }
    int64_t N[8], D[8];
    int nd, dd;
    lambert(j, N, &nd, D, &dd);
    if (nd != (p - 1) / 2 || dd != q / 2) {
      snprintf(err, errlen, "internal: convergent %d has degrees %d/%d", j, nd, dd);
      return false;
    }
    ld Nl[8], Dl[8];
    for (int k = 0; k < 8; ++k) {      // normalise D(0) = 1
      Nl[k] = (ld)N[k] / (ld)D[0];
      Dl[k] = (ld)D[k] / (ld)D[0];
    }
    const ld xs = pade_xsat(Nl, nd, Dl, dd);
    w->xsat = (float)xs;
    coef[0] = (double)xs;
    for (int k = 0; k <= nd; ++k) {
      w->num[k] = (float)Nl[k];
      coef[1 + 2 * k + 1] = (double)Nl[k];     // a_{2k+1}
    }
    for (int k = 0; k <= dd; ++k) {
      w->den[k] = (float)Dl[k];
      coef[1 + p + 1 + 2 * k] = (double)Dl[k];  // b_{2k}
    }
    return true;
  }
  if (kind == APX_MINIMAX || kind == APX_TAYLOR) {
    if (p < 1 || p > 3) {
      snprintf(err, errlen, "polynomial degree %d unsupported (1..3)", p);
      return false;
    }
    w->q = 0;
    w->xsat = (float)kApxXsat;
    coef[0] = kApxXsat;
    for (int k = 0; k < kApxPieces; ++k) {
      ld c[4];
      if (kind == APX_MINIMAX) {
        ld E;
        if (!remez_piece(p, (ld)k * kApxWidth, (ld)kApxWidth, k == 0 ? 1 : 0, c, &E)) {
          snprintf(err, errlen, "Remez failed on piece %d", k);
          return false;
        }
        if (k == 0) c[0] = 0;
      } else {
        taylor_coeffs(k == 0 ? 0.0L : (ld)k * kApxWidth + 0.25L, p, c);
      }
      for (int j = 0; j < 4; ++j) {
        coef[1 + 4 * k + j] = (double)c[j];
        w->pc[j][k] = (float)c[j];
        w->pc[j][k + 16] = (float)c[j];   // lanes 16..31 mirror (never selected)
      }
    }
    return true;
  }
  if (kind == APX_LIBM || kind == APX_SFU) {
    w->p = w->q = 0;
    return true;
  }
  snprintf(err, errlen, "unknown approximation kind %d", kind);
  return false;
}

cudaError_t launch_apx(int fmt, const void *x, void *y, size_t n, const ApxWords &w,
                       cudaStream_t s, const LaunchInfo &li) {
  if (fmt == FMT_BF16) return launch_apx_fmt<FMT_BF16>(x, y, n, w, s, li);
  return launch_apx_fmt<FMT_F32>(x, y, n, w, s, li);
}

}  // namespace kt
