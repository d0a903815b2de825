// kt_kernels.cu -- sm_100a streaming kernels for the K-TanH element maps and
// their launchers.
//
// Layout: x, y are flat contiguous arrays in HBM.  The body of the array
// (from the first 32-byte boundary) is processed as 32-byte vectors
// (16 BF16 or 8 F32) with 256-bit LDG/STG.  Each warp owns ONE "chunk" of
// 32 lanes x kUnroll vectors (2 KiB) and the grid has one warp per chunk
// ("flat" launch): the hardware block scheduler streams CTAs over the array
// in address order.  Measured on B200 (profiles/),
// this beats persistent grid-stride loops for a read-once/write-once stream:
// a plain copy reaches 6.93 TB/s flat vs 6.05-6.70 TB/s persistent (torch
// copy_: 6.56).  All lanes of a warp execute the shuffle-held LUT path
// (loads/stores are predicated, never branched around), so the shuffles
// never see a diverged warp.  The unaligned head (< 32 B before the first
// boundary) and the tail (< 32 B) are done element-wise by warp 0 of block 0
// inside the same launch.
//
// Launches use programmatic dependent launch (PDL): the kernel starts with
// griddepcontrol.wait (it does not touch memory before the preceding grid in
// the stream has completed and flushed), then immediately allows the next
// PDL launch to be scheduled, so back-to-back calls overlap launch latency
// and ramp-up with the previous call's tail.  Set KT_PDL=0 to disable.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "kt_async.cuh"
#include "kt_device.cuh"
#include "kt_internal.h"

namespace kt {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef KT_UNROLL
#define KT_UNROLL 2
#endif
constexpr int kUnroll = KT_UNROLL;            // 32-B vectors per lane per chunk (flat: 1 chunk/warp)
constexpr int kVecBytes = 32;
constexpr int kChunkVecs = 32 * kUnroll;      // vectors per warp-chunk

// Vectors per lane per chunk, per kernel (measured on B200 under the power
// cap, profiles/unroll_r02.txt): the ALU-heavier maps keep more loads in
// flight per warp -- K-GELU BF16 and every F32 map 4 (+6% / +11% over 2);
// K-TanH / K-Sigmoid / K-Swish BF16 and the LSTM gates 2; the fused
// K-GELU + K-Swish pass 2 at 48 registers (5 CTAs/SM; +7% over one vector
// at 40 registers / 6 CTAs per SM, which itself beat two vectors at 40).
#ifndef KT_UNROLL_GELU
#define KT_UNROLL_GELU 4
#endif
#ifndef KT_UNROLL_F32
#define KT_UNROLL_F32 4
#endif
#ifndef KT_UNROLL_DUAL
#define KT_UNROLL_DUAL 2
#endif
#ifndef KT_UNROLL_F32D
#define KT_UNROLL_F32D 4
#endif
template <int OP, int FMT>
__host__ __device__ constexpr int map_unroll() {
  return FMT == FMT_F32 ? ((OP == OP_SWISH || OP == OP_GELU) ? KT_UNROLL_F32D : KT_UNROLL_F32)
                        : (OP == OP_GELU ? KT_UNROLL_GELU : kUnroll);
}
template <int FMT>
__host__ __device__ constexpr int dual_unroll() {
  return FMT == FMT_BF16 ? KT_UNROLL_DUAL : kUnroll;
}
// Threads per CTA of k_map: K-GELU BF16 and F32-through-BF16 (50-54
// registers at U = 4) fit 9 CTAs of 128 threads per SM (36 warps) but only 4
// of 256 (32 warps); for the other maps both sizes give the same warps per SM.
#ifndef KT_MAP_TPB_GELU
#define KT_MAP_TPB_GELU 128
#endif
template <int OP, int FMT>
__host__ __device__ constexpr int map_threads() {
  return ((FMT == FMT_BF16 && OP == OP_GELU) || OP == OP_TANH_VIA_BF16) ? KT_MAP_TPB_GELU : kThreads;
}
#ifndef KT_UNROLL_BWD
#define KT_UNROLL_BWD 2
#endif
#ifndef KT_UNROLL_64
#define KT_UNROLL_64 2
#endif

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

// L2 prefetch of [p, p + bytes) by one thread (TMA bulk prefetch, no data
// returned to the SM).  A prefetch has no architectural effect on the values
// later loads observe (L2 is the point of coherence for global memory), so it
// is issued BEFORE griddepcontrol.wait: under PDL this warms L2 with the
// chunk while the preceding grid drains.
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// PDL: wait for the preceding grid (no-op without a programmatic dependency),
// then let the next grid in the stream begin launching.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ LaneLut load_lane_lut(const LutWords &lut) {
  const uint32_t lane = threadIdx.x & 31;
  return LaneLut{lut.bf16[lane], lut.f32K[lane], lut.f32C[lane]};
}

// For the grid-stride (looping) kernels: the empty volatile asm makes the
// lane's words opaque, so the compiler cannot rematerialise them inside the
// loop as lane-indexed (divergent, serialised) constant-bank loads.
__device__ __forceinline__ LaneLut load_lane_lut_reg(const LutWords &lut) {
  LaneLut L = load_lane_lut(lut);
  asm volatile("" : "+r"(L.w16), "+r"(L.k32), "+r"(L.c32));
  return L;
}

// Element-wise head/tail helper: lane i handles element i (i < cnt) of the
// range starting at p.  All 32 lanes execute apply_word (shuffle-safe).
template <int OP, int FMT>
__device__ __forceinline__ void scalar_span(const uint8_t *xp, uint8_t *yp, uint32_t cnt,
                                            const LaneLut &L) {
  const uint32_t lane = threadIdx.x & 31;
  const bool on = lane < cnt;
  uint32_t w = 0;
  if (FMT == FMT_BF16) {
    if (on) w = reinterpret_cast<const uint16_t *>(xp)[lane];
  } else {
    if (on) w = reinterpret_cast<const uint32_t *>(xp)[lane];
  }
  const uint32_t r = apply_word<OP, FMT>(w, L);
  if (FMT == FMT_BF16) {
    if (on) reinterpret_cast<uint16_t *>(yp)[lane] = (uint16_t)r;
  } else {
    if (on) reinterpret_cast<uint32_t *>(yp)[lane] = r;
  }
}

// Tie-screen fix-up (K-Swish / K-GELU BF16, kt_device.cuh tie_patch): after
// the chunk's stores, this lane re-reads its x and y words and rewrites the
// BF16 pairs with |x| < 2^-125 from the closed form.  Out of line and word by
// word so that it costs the streaming kernels no registers; plain (coherent)
// loads see the lane's own preceding stores.  Out-of-place calls only.
template <int OP, int FMT, int U>
__device__ __noinline__ void tie_fixup(const uint8_t *xb, uint8_t *yb, uint64_t base, uint64_t nvec) {
#pragma unroll 1
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    if (i >= nvec) continue;
    const uint32_t *xs = reinterpret_cast<const uint32_t *>(xb + i * kVecBytes);
    uint32_t *ys = reinterpret_cast<uint32_t *>(yb + i * kVecBytes);
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
      const uint32_t w = xs[j];
      if (tie_word_candidate<FMT>(w)) ys[j] = tie_patch_word<OP, FMT>(w, ys[j]);
    }
  }
}

template <int FMT, int U>
__device__ __noinline__ void tie_fixup_dual(const uint8_t *xb, uint8_t *gb, uint8_t *sb, uint64_t base,
                                            uint64_t nvec) {
#pragma unroll 1
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    if (i >= nvec) continue;
    const uint32_t *xs = reinterpret_cast<const uint32_t *>(xb + i * kVecBytes);
    uint32_t *gs = reinterpret_cast<uint32_t *>(gb + i * kVecBytes);
    uint32_t *ss = reinterpret_cast<uint32_t *>(sb + i * kVecBytes);
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
      const uint32_t w = xs[j];
      if (tie_word_candidate<FMT>(w)) {
        gs[j] = tie_patch_word<OP_GELU, FMT>(w, gs[j]);
        ss[j] = tie_patch_word<OP_SWISH, FMT>(w, ss[j]);
      }
    }
  }
}

// Main streaming kernel.  x/y: original (element-aligned) pointers; `head`
// elements precede the first 32-B boundary of x (and of y: same offset mod
// 32, checked on the host); nvec vectors follow; then `tail` elements.
#ifdef KT_MAP_MINB
template <int OP, int FMT, bool NC, bool PF, int U, int TPB>
__global__ void __launch_bounds__(TPB, KT_MAP_MINB)
#else
template <int OP, int FMT, bool NC, bool PF, int U, int TPB>
__global__ void __launch_bounds__(TPB)
#endif
k_map(const uint8_t *x, uint8_t *y, uint32_t head, uint64_t nvec, uint32_t tail,
      uint32_t pf_blocks, uint32_t pf_depth, const __grid_constant__ LutWords lut) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const LaneLut L = load_lane_lut(lut);
  const uint32_t lane = threadIdx.x & 31;
  const uint8_t *xb = x + (size_t)head * es;
  uint8_t *yb = y + (size_t)head * es;
  constexpr int kW = TPB / 32;                                             // warps per CTA
  const uint64_t c = (uint64_t)blockIdx.x * kW + (threadIdx.x >> 5);       // this warp's chunk
  // only the first resident wave can be waiting behind a predecessor's tail
  if (PF && blockIdx.x < pf_blocks && lane < pf_depth) {
    // lane d prefetches the chunk of the warp d resident waves later
    const uint64_t cc = c + (uint64_t)lane * pf_blocks * kW;
    if (cc * (32 * U) < nvec) {
      const uint64_t left = nvec - cc * (32 * U);
      prefetch_l2(xb + cc * (32 * U) * kVecBytes,
                  (uint32_t)((left < (32 * U) ? left : (32 * U)) * kVecBytes));
    }
  }
  pdl_enter();
  const uint64_t base = c * (32 * U) + lane;
  uint32_t v[U][8];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    ld256<NC>(xb + i * kVecBytes, v[u], i < nvec);
  }
  // K-Swish / K-GELU BF16 out of place: plain-fma outer step + tie screen
  // (kt_device.cuh); in place (x == y, no copy of x survives the stores) the
  // exact outer step on every pair
  constexpr bool kScreen = needs_tie_screen<OP, FMT>() && NC;
  uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      if (kScreen) {
        uint32_t m0, m1;
        v[u][j] = apply_word_fast<OP, FMT>(v[u][j], L, m0);
        v[u][j + 1] = apply_word_fast<OP, FMT>(v[u][j + 1], L, m1);
        kmin = key_min<FMT>(kmin, key_min<FMT>(m0, m1));  // one 3-input min per two words
      } else {
        v[u][j] = apply_word<OP, FMT>(v[u][j], L);
        v[u][j + 1] = apply_word<OP, FMT>(v[u][j + 1], L);
      }
    }
  }
  // all U loads were issued before any arithmetic and all stores follow it
  // (the ld/st asm statements are volatile, so storing a vector early would
  // also delay the next vector's load: fewer bytes in flight)
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    st256(yb + i * kVecBytes, v[u], i < nvec);
  }
  if (kScreen && __any_sync(0xffffffffu, tie_possible_fmt<FMT>(kmin)))
    tie_fixup<OP, FMT, U>(xb, yb, base, nvec);   // rare: an |argument| < 2^-125 (or a zero) in the chunk
  if ((head | tail) != 0 && blockIdx.x == 0 && threadIdx.x < 32) {
    scalar_span<OP, FMT>(x, y, head, L);
    const size_t toff = ((size_t)head + (size_t)nvec * (kVecBytes / es)) * es;
    scalar_span<OP, FMT>(x + toff, y + toff, tail, L);
  }
}

// ---- K-TanH BF16 with the 64-interval table (NEXT-3) -------------------------
// Same streaming shape as k_map (flat, 256-bit, PDL, first-wave L2 prefetch).
__device__ __forceinline__ void span64(const uint8_t *xp, uint8_t *yp, uint32_t cnt, uint32_t w0,
                                       uint32_t w1) {
  const uint32_t lane = threadIdx.x & 31;
  const bool on = lane < cnt;
  const uint32_t v = on ? reinterpret_cast<const uint16_t *>(xp)[lane] : 0u;
  const uint32_t r = ktanh64_bf16x2(v, w0, w1);
  if (on) reinterpret_cast<uint16_t *>(yp)[lane] = (uint16_t)r;
}

template <bool NC, int U>
__global__ void __launch_bounds__(kThreads)
k_map64(const uint8_t *x, uint8_t *y, uint32_t head, uint64_t nvec, uint32_t tail, uint32_t pf_blocks,
        const __grid_constant__ LutWords64 lut) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t w0 = lut.w[lane], w1 = lut.w[32 + lane];
  const uint8_t *xb = x + (size_t)head * 2;
  uint8_t *yb = y + (size_t)head * 2;
  const uint64_t c = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (NC && blockIdx.x < pf_blocks && lane == 0 && c * (32 * U) < nvec) {
    const uint64_t left = nvec - c * (32 * U);
    prefetch_l2(xb + c * (32 * U) * kVecBytes,
                (uint32_t)((left < (32 * U) ? left : (32 * U)) * kVecBytes));
  }
  pdl_enter();
  const uint64_t base = c * (32 * U) + lane;
  uint32_t v[U][8];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    ld256<NC>(xb + i * kVecBytes, v[u], i < nvec);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[u][j] = ktanh64_bf16x2(v[u][j], w0, w1);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    st256(yb + i * kVecBytes, v[u], i < nvec);
  }
  if ((head | tail) != 0 && blockIdx.x == 0 && threadIdx.x < 32) {
    span64(x, y, head, w0, w1);
    const size_t toff = ((size_t)head + (size_t)nvec * 16) * 2;
    span64(x + toff, y + toff, tail, w0, w1);
  }
}

__global__ void __launch_bounds__(kThreads)
k_map64_elem(const uint8_t *x, uint8_t *y, uint64_t n, const __grid_constant__ LutWords64 lut) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t w0 = lut.w[lane], w1 = lut.w[32 + lane];
  asm volatile("" : "+r"(w0), "+r"(w1));
  pdl_enter();
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t c = warp0; c < (n + 31) / 32; c += nwarps) {
    const uint64_t off = c * 32, rem = n - off;
    span64(x + off * 2, y + off * 2, (uint32_t)(rem < 32 ? rem : 32), w0, w1);
  }
}

// ---- fused K-GELU + K-Swish over one input (config 5, reading A20) -----------
// Config 5 applies both derived activations to the same FFN tensor; one pass
// that reads x once and writes both outputs moves 6 B per BF16 element
// instead of 2 x 4 B.  Each output is bit-identical to its single-op call.
template <int FMT>
__device__ __forceinline__ void dual_span(const uint8_t *xp, uint8_t *gp, uint8_t *sp, uint32_t cnt,
                                          const LaneLut &L) {
  const uint32_t lane = threadIdx.x & 31;
  const bool on = lane < cnt;
  uint32_t w = 0;
  if (FMT == FMT_BF16) {
    if (on) w = reinterpret_cast<const uint16_t *>(xp)[lane];
  } else if (on) {
    w = reinterpret_cast<const uint32_t *>(xp)[lane];
  }
  const uint32_t g = apply_word<OP_GELU, FMT>(w, L), sw = apply_word<OP_SWISH, FMT>(w, L);
  if (on) {
    if (FMT == FMT_BF16) {
      reinterpret_cast<uint16_t *>(gp)[lane] = (uint16_t)g;
      reinterpret_cast<uint16_t *>(sp)[lane] = (uint16_t)sw;
    } else {
      reinterpret_cast<uint32_t *>(gp)[lane] = g;
      reinterpret_cast<uint32_t *>(sp)[lane] = sw;
    }
  }
}

#ifndef KT_DUAL_MINB
#define KT_DUAL_MINB 5   // 48 regs: 5 CTAs/SM with two vectors per lane (profiles/unroll_r02.txt)
#endif
#ifndef KT_BWD_MINB
#define KT_BWD_MINB 5    // 48 regs: 5 CTAs/SM (+17% on config 5 backward)
#endif
template <int FMT, bool NC, int U>
__global__ void __launch_bounds__(kThreads, KT_DUAL_MINB)
k_dual(const uint8_t *x, uint8_t *yg, uint8_t *ys, uint32_t head, uint64_t nvec, uint32_t tail,
       uint32_t pf_blocks, const __grid_constant__ LutWords lut) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const LaneLut L = load_lane_lut(lut);
  const uint32_t lane = threadIdx.x & 31;
  const size_t hb = (size_t)head * es;
  const uint64_t c = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (NC && blockIdx.x < pf_blocks && lane == 0 && c * (32 * U) < nvec) {
    const uint64_t left = nvec - c * (32 * U);
    prefetch_l2(x + hb + c * (32 * U) * kVecBytes,
                (uint32_t)((left < (32 * U) ? left : (32 * U)) * kVecBytes));
  }
  pdl_enter();
  const uint64_t base = c * (32 * U) + lane;
  uint32_t v[U][8];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    ld256<NC>(x + hb + i * kVecBytes, v[u], i < nvec);
  }
  constexpr bool kScreen = needs_tie_screen<OP_GELU, FMT>() && NC;   // as in k_map
  uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    uint32_t g[8], sw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (kScreen) {
        // |RN_bf16(u)| < 2^-125 for every |x| < 2^-125: the K-GELU key covers both outputs
        uint32_t m, munused;
        g[j] = apply_word_fast<OP_GELU, FMT>(v[u][j], L, m);
        sw[j] = apply_word_fast<OP_SWISH, FMT>(v[u][j], L, munused);
        kmin = key_min<FMT>(kmin, m);
      } else {
        g[j] = apply_word<OP_GELU, FMT>(v[u][j], L);
        sw[j] = apply_word<OP_SWISH, FMT>(v[u][j], L);
      }
    }
    const uint64_t i = base + (uint64_t)u * 32;
    st256(yg + hb + i * kVecBytes, g, i < nvec);
    st256(ys + hb + i * kVecBytes, sw, i < nvec);
  }
  if (kScreen && __any_sync(0xffffffffu, tie_possible_fmt<FMT>(kmin)))
    tie_fixup_dual<FMT, U>(x + hb, yg + hb, ys + hb, base, nvec);   // rare
  if ((head | tail) != 0 && blockIdx.x == 0 && threadIdx.x < 32) {
    dual_span<FMT>(x, yg, ys, head, L);
    const size_t toff = ((size_t)head + (size_t)nvec * (kVecBytes / es)) * es;
    dual_span<FMT>(x + toff, yg + toff, ys + toff, tail, L);
  }
}

template <int FMT>
__global__ void __launch_bounds__(kThreads)
k_dual_elem(const uint8_t *x, uint8_t *yg, uint8_t *ys, uint64_t n, const __grid_constant__ LutWords lut) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const LaneLut L = load_lane_lut_reg(lut);
  pdl_enter();
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t c = warp0; c < (n + 31) / 32; c += nwarps) {
    const uint64_t off = c * 32, rem = n - off;
    dual_span<FMT>(x + off * es, yg + off * es, ys + off * es, (uint32_t)(rem < 32 ? rem : 32), L);
  }
}

// ---- backward (NEXT-1): dx = dy * g(a), two input streams -----------------
template <int OP, int FMT>
__device__ __forceinline__ void scalar_span_bwd(const uint8_t *ap, const uint8_t *dp, uint8_t *xp,
                                                uint32_t cnt, const LaneLut &L) {
  const uint32_t lane = threadIdx.x & 31;
  const bool on = lane < cnt;
  uint32_t a = 0, d = 0;
  if (FMT == FMT_BF16) {
    if (on) {
      a = reinterpret_cast<const uint16_t *>(ap)[lane];
      d = reinterpret_cast<const uint16_t *>(dp)[lane];
    }
  } else if (on) {
    a = reinterpret_cast<const uint32_t *>(ap)[lane];
    d = reinterpret_cast<const uint32_t *>(dp)[lane];
  }
  const uint32_t r = apply_bwd_word<OP, FMT>(a, d, L);
  if (on) {
    if (FMT == FMT_BF16) reinterpret_cast<uint16_t *>(xp)[lane] = (uint16_t)r;
    else reinterpret_cast<uint32_t *>(xp)[lane] = r;
  }
}

template <int OP, int FMT, bool NC, int U>
__global__ void __launch_bounds__(kThreads, KT_BWD_MINB)
k_bwd(const uint8_t *a, const uint8_t *dy, uint8_t *dx, uint32_t head, uint64_t nvec, uint32_t tail,
      const __grid_constant__ LutWords lut) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const LaneLut L = load_lane_lut(lut);
  pdl_enter();
  const uint32_t lane = threadIdx.x & 31;
  const size_t hb = (size_t)head * es;
  const uint64_t c = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t base = c * (32 * U) + lane;
  uint32_t va[U][8], vd[U][8];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    ld256<NC>(a + hb + i * kVecBytes, va[u], i < nvec);
    ld256<NC>(dy + hb + i * kVecBytes, vd[u], i < nvec);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
#pragma unroll
    for (int j = 0; j < 8; ++j) va[u][j] = apply_bwd_word<OP, FMT>(va[u][j], vd[u][j], L);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = base + (uint64_t)u * 32;
    st256(dx + hb + i * kVecBytes, va[u], i < nvec);
  }
  if ((head | tail) != 0 && blockIdx.x == 0 && threadIdx.x < 32) {
    scalar_span_bwd<OP, FMT>(a, dy, dx, head, L);
    const size_t toff = ((size_t)head + (size_t)nvec * (kVecBytes / es)) * es;
    scalar_span_bwd<OP, FMT>(a + toff, dy + toff, dx + toff, tail, L);
  }
}

template <int OP, int FMT>
__global__ void __launch_bounds__(kThreads)
k_bwd_elem(const uint8_t *a, const uint8_t *dy, uint8_t *dx, uint64_t n,
           const __grid_constant__ LutWords lut) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const LaneLut L = load_lane_lut_reg(lut);
  pdl_enter();
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t c = warp0; c < (n + 31) / 32; c += nwarps) {
    const uint64_t off = c * 32, rem = n - off;
    scalar_span_bwd<OP, FMT>(a + off * es, dy + off * es, dx + off * es,
                             (uint32_t)(rem < 32 ? rem : 32), L);
  }
}

// Fallback when x and y have different offsets mod 32 B: one element per
// lane per step, warp-uniform loop.
template <int OP, int FMT>
__global__ void __launch_bounds__(kThreads)
k_map_elem(const uint8_t *__restrict__ x, uint8_t *__restrict__ y, uint64_t n,
           const __grid_constant__ LutWords lut) {
  constexpr uint32_t es = (FMT == FMT_BF16) ? 2 : 4;
  const LaneLut L = load_lane_lut_reg(lut);
  pdl_enter();
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  const uint64_t nch = (n + 31) / 32;
  for (uint64_t c = warp0; c < nch; c += nwarps) {
    const uint64_t off = c * 32;
    const uint64_t rem = n - off;
    scalar_span<OP, FMT>(x + off * es, y + off * es, (uint32_t)(rem < 32 ? rem : 32), L);
  }
}

// LSTM gates, vector path: x, y 32-B aligned, hidden % 16 == 0, so each
// 16-element vector lies in one quarter of its row.  vpr = vectors per row
// (= hidden / 4), vpq = vectors per quarter (= hidden / 16).
template <bool NC>
__global__ void __launch_bounds__(kThreads)
k_lstm(const uint8_t *x, uint8_t *y, uint32_t nvec, uint32_t vpr, uint32_t vpq, int tanh_quarter,
       uint32_t pf_blocks, const __grid_constant__ LutWords lut) {
  const LaneLut L = load_lane_lut(lut);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (NC && blockIdx.x < pf_blocks && lane == 0 && c * kChunkVecs < nvec) {
    const uint32_t left = nvec - c * kChunkVecs;
    prefetch_l2(x + (size_t)c * kChunkVecs * kVecBytes,
                (left < (uint32_t)kChunkVecs ? left : (uint32_t)kChunkVecs) * kVecBytes);
  }
  pdl_enter();
  const uint32_t base = c * kChunkVecs + lane;
  uint32_t v[kUnroll][8];
  bool tq[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint32_t i = base + u * 32;
    ld256<NC>(x + (size_t)i * kVecBytes, v[u], i < nvec);
    tq[u] = ((i % vpr) / vpq) == (uint32_t)tanh_quarter;
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[u][j] = lstm_bf16x2(v[u][j], L.w16, tq[u]);
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint32_t i = base + u * 32;
    st256(y + (size_t)i * kVecBytes, v[u], i < nvec);
  }
}

// Fused LSTM cell, vector path: 16 consecutive cells of one row per lane
// (hidden % 16 == 0, all pointers 32-B aligned).  Per 16 cells: 4 x 32 B of
// gates + 64 B of c in, 64 B of c' + 32 B of h out (18 B per cell).
// NCC: c_prev read on the non-coherent path; the launcher picks the coherent
// instantiation when c_next == c_prev (in place), as launch_op does for x == y.
#ifndef KT_CELL_TPB
#define KT_CELL_TPB 256
#endif
constexpr int kCellTPB = KT_CELL_TPB, kCellW = KT_CELL_TPB / 32;
#ifdef KT_CELL_MINB
template <bool NCC>
__global__ void __launch_bounds__(kCellTPB, KT_CELL_MINB)
#else
template <bool NCC>
__global__ void __launch_bounds__(kCellTPB)   // (kThreads, 1) lets ptxas take > 64 regs: slower
#endif
k_lstm_cell(const uint8_t *gates, const uint8_t *c_prev, uint8_t *c_next, uint8_t *h_next,
            uint32_t nvec, uint32_t vpr, uint32_t hidden, uint32_t pf_blocks,
            const __grid_constant__ LutWords lut) {
  const LaneLut L = load_lane_lut(lut);
  // First resident wave (blockIdx.x < pf_blocks): lanes 0-4 prefetch this
  // warp's own 4 gate segments and c segment into L2 BEFORE
  // griddepcontrol.wait, so under PDL the DRAM reads start while the previous
  // launch drains (k_map does the same).  A prefetch has no architectural
  // effect on the values later loads see.  (Round 1 tried prefetching the NEXT
  // wave's data instead: slower, 26.3 vs 20.8 us.)
  if (blockIdx.x < pf_blocks && (threadIdx.x & 31) < 5) {
    const uint32_t v2 = (blockIdx.x * kCellW + (threadIdx.x >> 5)) * 32;
    if (v2 < nvec) {
      const uint32_t row2 = v2 / vpr, j2 = v2 - row2 * vpr;
      const uint32_t cnt = min(min(32u, nvec - v2), vpr - j2);
      const uint32_t q = threadIdx.x & 31;
      if (q < 4)
        prefetch_l2(gates + ((size_t)row2 * 4 * hidden + (size_t)j2 * 16) * 2 + (size_t)q * hidden * 2,
                    cnt * 32);
      else
        prefetch_l2(c_prev + ((size_t)row2 * hidden + (size_t)j2 * 16) * 4, cnt * 64);
    }
  }
  pdl_enter();
  const uint32_t v = (blockIdx.x * kCellW + (threadIdx.x >> 5)) * 32 + (threadIdx.x & 31);
  const bool on = v < nvec;
  const uint32_t row = on ? v / vpr : 0, j16 = on ? v - row * vpr : 0;
  const uint8_t *gr = gates + ((size_t)row * 4 * hidden + (size_t)j16 * 16) * 2;
  const size_t qb = (size_t)hidden * 2;
  const size_t cidx = (size_t)row * hidden + (size_t)j16 * 16;
  uint32_t gi[8], gf[8], gg[8], go[8], c0[8], c1[8];
  ld256<true>(gr, gi, on);
  ld256<true>(gr + qb, gf, on);
  ld256<true>(gr + 2 * qb, gg, on);
  ld256<true>(gr + 3 * qb, go, on);
  ld256<NCC>(c_prev + cidx * 4, c0, on);
  ld256<NCC>(c_prev + cidx * 4 + 32, c1, on);
  uint32_t cn0[8], cn1[8], h[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t *cs = k < 4 ? c0 : c1;
    const int kk = (k & 3) * 2;
    float2 cn;
    h[k] = lstm_cell2(gi[k], gf[k], gg[k], go[k],
                      make_float2(__uint_as_float(cs[kk]), __uint_as_float(cs[kk + 1])), cn, L);
    uint32_t *cd = k < 4 ? cn0 : cn1;
    cd[kk] = __float_as_uint(cn.x);
    cd[kk + 1] = __float_as_uint(cn.y);
  }
  st256(c_next + cidx * 4, cn0, on);
  st256(c_next + cidx * 4 + 32, cn1, on);
  st256(h_next + cidx * 2, h, on);
}

// ---- fused LSTM cell, staged through shared memory (bulk async copies) -------
// The register-staged k_lstm_cell holds six 256-bit loads per lane across the
// whole cell computation, so its bytes in flight are bounded by the register
// file (64 regs, ~41% warps active, long-scoreboard bound: 0.91 of the copy
// bandwidth).  Here the loads are decoupled from the registers:
//   * persistent CTAs, each owning a contiguous, balanced range of cells,
//     cut into tiles of kCellTile cells;
//   * one producer warp per CTA streams each tile's 4 gate segments (per row
//     the tile touches) and its c segment into a kCellStages-deep ring of
//     shared-memory stages with cp.async.bulk (TMA engine), completion counted
//     in bytes on the stage's "full" mbarrier;
//   * kCellConsumerWarps consumer warps: thread i takes kCellGroups groups of
//     4 cells (group g: cells g T/G + 4i .. +3 of the tile, so every shared
//     load is conflict-free: LDS.64 per gate row, LDS.128 for c), releases the
//     stage ("empty" mbarrier, one arrive per warp), computes the cells
//     (lstm_cell2, the same device code as the register kernel) and stores c'
//     (128-bit) and h (64-bit) straight from registers.
// c_next may alias c_prev: a tile's c is in shared memory before any c' of
// that tile is written, and other tiles' c ranges are disjoint.
#ifndef KT_CELL_WARPS
#define KT_CELL_WARPS 16
#endif
#ifndef KT_CELL_GROUPS
#define KT_CELL_GROUPS 1
#endif
#ifndef KT_CELL_STAGES
#define KT_CELL_STAGES 4
#endif
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
constexpr int kCellConsumerWarps = KT_CELL_WARPS;
constexpr int kCellGroups = KT_CELL_GROUPS;
constexpr int kCellThreads = (kCellConsumerWarps + 1) * 32;             // + producer warp
constexpr uint32_t kCellGroupCells = kCellConsumerWarps * 32 * 4;       // cells per group
constexpr uint32_t kCellTile = kCellGroupCells * kCellGroups;           // cells per tile
constexpr int kCellStages = KT_CELL_STAGES;
constexpr uint32_t kCellStageBytes = kCellTile * (4 * 2 + 4);           // gates BF16 + c F32
constexpr uint32_t kCellSmem = kCellStages * kCellStageBytes + 2 * kCellStages * 8;
constexpr uint32_t kCellMinHidden = 256;   // tiles touch few rows: few, large copies
#ifndef KT_CELL_DEFAULT
#define KT_CELL_DEFAULT 0
#endif

__global__ void __launch_bounds__(kCellThreads)
k_lstm_cell_tma(const uint8_t *gates, const uint8_t *c_prev, uint8_t *c_next, uint8_t *h_next,
                uint64_t n, uint32_t hidden, const __grid_constant__ LutWords lut) {
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + kCellStages * kCellStageBytes;      // kCellStages x 8 B
  const uint32_t bar_empty = bar_full + kCellStages * 8;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const LaneLut L = load_lane_lut(lut);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kCellStages; ++s) {
      mbar_init(bar_full + 8 * s, 1);
      mbar_init(bar_empty + 8 * s, kCellConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this CTA's contiguous range [v_beg, v_end), 16-cell granules balanced over the grid
  const uint64_t gran = n / 16, gq = gran / gridDim.x, gr = gran % gridDim.x;
  const uint64_t v_beg = (gq * blockIdx.x + umin64(blockIdx.x, gr)) * 16;
  const uint64_t v_end = v_beg + (gq + (blockIdx.x < gr ? 1 : 0)) * 16;
  const uint32_t ntiles = (uint32_t)((v_end - v_beg + kCellTile - 1) / kCellTile);

  if (warp == kCellConsumerWarps) {
    // ---------------- producer warp ----------------
    asm volatile("griddepcontrol.wait;" ::: "memory");   // the preceding grid's writes are visible
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t s = t % kCellStages, ph = (t / kCellStages) & 1;
      const uint64_t v0 = v_beg + (uint64_t)t * kCellTile;
      const uint32_t len = (uint32_t)umin64(kCellTile, v_end - v0);
      mbar_wait(bar_empty + 8 * s, ph ^ 1);               // every consumer warp released it
      if (lane == 0) mbar_expect_tx(bar_full + 8 * s, len * 12u);
      __syncwarp();
      const uint32_t st = sbase + s * kCellStageBytes;
      const uint64_t row0 = v0 / hidden;
      const uint32_t nseg = (uint32_t)((v0 + len - 1) / hidden - row0 + 1);
      // copy k < 4 nseg: gate q = k & 3 of row segment k >> 2; copy 4 nseg: c
      for (uint32_t k = lane; k <= 4 * nseg; k += 32) {
        if (k == 4 * nseg) {
          bulk_g2s(st + kCellTile * 8, c_prev + v0 * 4, len * 4, bar_full + 8 * s);
          continue;
        }
        const uint32_t q = k & 3;
        const uint64_t row = row0 + (k >> 2);
        const uint64_t sb = row * hidden > v0 ? row * hidden : v0;           // segment [sb, se)
        const uint64_t se = umin64((row + 1) * hidden, v0 + len);
        const uint8_t *src = gates + (row * 4 * hidden + (uint64_t)q * hidden + (sb - row * hidden)) * 2;
        bulk_g2s(st + q * kCellTile * 2 + (uint32_t)(sb - v0) * 2, src, (uint32_t)(se - sb) * 2,
                 bar_full + 8 * s);
      }
    }
    return;
  }
  // ---------------- consumer warps ----------------
  for (uint32_t t = 0; t < ntiles; ++t) {
    const uint32_t s = t % kCellStages, ph = (t / kCellStages) & 1;
    const uint64_t v0 = v_beg + (uint64_t)t * kCellTile;
    const uint32_t len = (uint32_t)umin64(kCellTile, v_end - v0);
    mbar_wait(bar_full + 8 * s, ph);
    const uint8_t *st = smem + s * kCellStageBytes;
    uint2 gi[kCellGroups], gf[kCellGroups], gg[kCellGroups], go[kCellGroups];
    float4 c[kCellGroups];
#pragma unroll
    for (int g = 0; g < kCellGroups; ++g) {
      const uint32_t i4 = g * kCellGroupCells + threadIdx.x * 4;         // first cell of the group
      gi[g] = *reinterpret_cast<const uint2 *>(st + 0 * kCellTile * 2 + i4 * 2);
      gf[g] = *reinterpret_cast<const uint2 *>(st + 1 * kCellTile * 2 + i4 * 2);
      gg[g] = *reinterpret_cast<const uint2 *>(st + 2 * kCellTile * 2 + i4 * 2);
      go[g] = *reinterpret_cast<const uint2 *>(st + 3 * kCellTile * 2 + i4 * 2);
      c[g] = *reinterpret_cast<const float4 *>(st + kCellTile * 8 + i4 * 4);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_empty + 8 * s);       // stage s may be refilled
#pragma unroll
    for (int g = 0; g < kCellGroups; ++g) {
      const uint32_t i4 = g * kCellGroupCells + threadIdx.x * 4;
      float2 cn0, cn1;
      const uint32_t h0 = lstm_cell2(gi[g].x, gf[g].x, gg[g].x, go[g].x, make_float2(c[g].x, c[g].y), cn0, L);
      const uint32_t h1 = lstm_cell2(gi[g].y, gf[g].y, gg[g].y, go[g].y, make_float2(c[g].z, c[g].w), cn1, L);
      if (i4 < len) {
        const uint64_t v = v0 + i4;
        asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(c_next + v * 4),
                     "f"(cn0.x), "f"(cn0.y), "f"(cn1.x), "f"(cn1.y) : "memory");
        asm volatile("st.global.L1::no_allocate.v2.b32 [%0], {%1, %2};" ::"l"(h_next + v * 2), "r"(h0),
                     "r"(h1) : "memory");
      }
    }
  }
}

// Fused LSTM cell, element fallback.
__global__ void __launch_bounds__(kThreads)
k_lstm_cell_elem(const uint16_t *gates, const float *c_prev, float *c_next, uint16_t *h_next,
                 uint64_t n, uint64_t hidden, const __grid_constant__ LutWords lut) {
  const LaneLut L = load_lane_lut_reg(lut);
  pdl_enter();
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t c = warp0; c * 32 < n; c += nwarps) {
    const uint64_t i = c * 32 + (threadIdx.x & 31);
    const bool on = i < n;
    const uint64_t row = on ? i / hidden : 0, j = on ? i - row * hidden : 0;
    const uint16_t *gr = gates + row * 4 * hidden + j;
    const uint32_t gi = on ? gr[0] : 0u, gf = on ? gr[hidden] : 0u, gg = on ? gr[2 * hidden] : 0u,
                   go = on ? gr[3 * hidden] : 0u;
    const float cp = on ? c_prev[i] : 0.0f;
    float2 cn;
    const uint32_t h = lstm_cell2(gi, gf, gg, go, make_float2(cp, 0.0f), cn, L);
    if (on) {
      c_next[i] = cn.x;
      h_next[i] = (uint16_t)h;
    }
  }
}

// LSTM gates, element fallback (any alignment / hidden).
__global__ void __launch_bounds__(kThreads)
k_lstm_elem(const uint16_t *__restrict__ x, uint16_t *__restrict__ y, uint64_t n, uint64_t width,
            uint64_t hidden, int tanh_quarter, const __grid_constant__ LutWords lut) {
  const LaneLut L = load_lane_lut_reg(lut);
  pdl_enter();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t c = warp0; c * 32 < n; c += nwarps) {
    const uint64_t i = c * 32 + lane;
    const bool on = i < n;
    const uint32_t w = on ? x[i] : 0u;
    const bool is_tanh = on && ((i % width) / hidden) == (uint64_t)tanh_quarter;
    const uint32_t r = lstm_bf16x2(w, L.w16, is_tanh);
    if (on) y[i] = (uint16_t)r;
  }
}

// ---------------------------------------------------------------- host ----

bool pdl_enabled() {
  static const bool on = [] {
    const char *e = getenv("KT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// cudaLaunchKernelEx with the programmatic-stream-serialization attribute.
// Early L2 prefetch of each warp's input chunk (before the PDL wait);
// KT_PREFETCH=0 disables.
bool prefetch_enabled() {
  static const bool on = [] {
    const char *e = getenv("KT_PREFETCH");
    return !(e && e[0] == '0');
  }();
  return on && pdl_enabled();
}

// Chunks prefetched per first-wave warp (KT_PF_DEPTH, default 1).
static uint32_t prefetch_depth() {
  static const uint32_t d = [] {
    const char *e = getenv("KT_PF_DEPTH");
    const int v = e ? atoi(e) : 1;
    return (uint32_t)(v < 1 ? 1 : v > 8 ? 8 : v);
  }();
  return d;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_tpb(void (*kernel)(KArgs...), unsigned grid, unsigned tpb, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tpb);
  cfg.dynamicSmemBytes = 0;
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

template <typename... KArgs, typename... Args>
static cudaError_t launch(void (*kernel)(KArgs...), unsigned grid, cudaStream_t s, Args... args) {
  return launch_tpb(kernel, grid, kThreads, s, args...);
}

template <class K>
static int resident_blocks(K kernel, int tpb = kThreads) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, tpb, 0) != cudaSuccess || b < 1)
    b = 1;
  return b;
}

// Grid for the grid-stride fallback kernels: about 4 waves' worth of warps.
static unsigned grid_for(uint64_t nchunks, int sm_count, int blocks_per_sm) {
  const uint64_t max_warps = (uint64_t)sm_count * blocks_per_sm * kWarps * 4;
  const uint64_t warps = nchunks < max_warps ? nchunks : max_warps;
  return (unsigned)std::max<uint64_t>(1, (warps + kWarps - 1) / kWarps);
}

// Flat grid: one warp per chunk (at least one block for head/tail work).
static unsigned flat_grid(uint64_t nchunks) {
  return (unsigned)std::max<uint64_t>(1, (nchunks + kWarps - 1) / kWarps);
}

template <int OP, int FMT>
static cudaError_t launch_op(const void *x, void *y, size_t n, const LutWords &lut, cudaStream_t s,
                             const LaunchInfo &li, bool sysmem) {
  constexpr size_t es = (FMT == FMT_BF16) ? 2 : 4;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
  const uint8_t *xp = static_cast<const uint8_t *>(x);
  uint8_t *yp = static_cast<uint8_t *>(y);
  if ((xa % kVecBytes) != (ya % kVecBytes)) {
    static const int bps = resident_blocks(k_map_elem<OP, FMT>);
    const unsigned grid = grid_for((n + 31) / 32, li.sm_count, bps);
    return launch(k_map_elem<OP, FMT>, grid, s, xp, yp, (uint64_t)n, lut);
  }
  const size_t mis = xa % kVecBytes;
  size_t head = mis ? (kVecBytes - mis) / es : 0;
  if (head > n) head = n;
  const size_t body = n - head;
  const uint64_t nvec = body / (kVecBytes / es);
  const uint32_t tail = (uint32_t)(body - nvec * (kVecBytes / es));
  constexpr int U = map_unroll<OP, FMT>();
  constexpr int TPB = map_threads<OP, FMT>(), kW = TPB / 32;
  const uint64_t nchunks = (nvec + 32 * U - 1) / (32 * U);
  if (nchunks / kW >= 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, (nchunks + kW - 1) / kW);
  if (x != y) {
    if (prefetch_enabled() && !sysmem) {   // L2 prefetch is for HBM inputs only
      static const int bps = resident_blocks(k_map<OP, FMT, true, true, U, TPB>, TPB);
      const uint32_t pf_blocks = (uint32_t)(li.sm_count * bps);
      return launch_tpb(k_map<OP, FMT, true, true, U, TPB>, grid, TPB, s, xp, yp, (uint32_t)head, nvec, tail,
                    pf_blocks, prefetch_depth(), lut);
    }
    return launch_tpb(k_map<OP, FMT, true, false, U, TPB>, grid, TPB, s, xp, yp, (uint32_t)head, nvec, tail, 0u, 0u,
                  lut);
  }
  return launch_tpb(k_map<OP, FMT, false, false, U, TPB>, grid, TPB, s, xp, yp, (uint32_t)head, nvec, tail, 0u, 0u,
                lut);
}

cudaError_t launch_map(int op, int fmt, const void *x, void *y, size_t n, const LutWords &lut,
                       cudaStream_t s, const LaunchInfo &li, bool sysmem) {
#define KT_CASE(O, F) \
  if (op == O && fmt == F) return launch_op<O, F>(x, y, n, lut, s, li, sysmem);
  KT_CASE(OP_TANH, FMT_BF16)
  KT_CASE(OP_SIGMOID, FMT_BF16)
  KT_CASE(OP_SWISH, FMT_BF16)
  KT_CASE(OP_GELU, FMT_BF16)
  KT_CASE(OP_TANH, FMT_F32)
  KT_CASE(OP_SIGMOID, FMT_F32)
  KT_CASE(OP_SWISH, FMT_F32)
  KT_CASE(OP_GELU, FMT_F32)
  KT_CASE(OP_TANH_VIA_BF16, FMT_F32)
#undef KT_CASE
  return cudaErrorInvalidValue;
}

template <int OP, int FMT>
static cudaError_t launch_bwd_op(const void *a, const void *dy, void *dx, size_t n,
                                 const LutWords &lut, cudaStream_t s, const LaunchInfo &li) {
  constexpr size_t es = (FMT == FMT_BF16) ? 2 : 4;
  const uintptr_t aa = reinterpret_cast<uintptr_t>(a), da = reinterpret_cast<uintptr_t>(dy),
                  xa = reinterpret_cast<uintptr_t>(dx);
  const uint8_t *ap = static_cast<const uint8_t *>(a), *dp = static_cast<const uint8_t *>(dy);
  uint8_t *xp = static_cast<uint8_t *>(dx);
  if (aa % kVecBytes != xa % kVecBytes || da % kVecBytes != xa % kVecBytes) {
    static const int bps = resident_blocks(k_bwd_elem<OP, FMT>);
    const unsigned grid = grid_for((n + 31) / 32, li.sm_count, bps);
    return launch(k_bwd_elem<OP, FMT>, grid, s, ap, dp, xp, (uint64_t)n, lut);
  }
  const size_t mis = xa % kVecBytes;
  size_t head = mis ? (kVecBytes - mis) / es : 0;
  if (head > n) head = n;
  const size_t body = n - head;
  const uint64_t nvec = body / (kVecBytes / es);
  const uint32_t tail = (uint32_t)(body - nvec * (kVecBytes / es));
  constexpr int U = KT_UNROLL_BWD;
  const uint64_t nchunks = (nvec + 32 * U - 1) / (32 * U);
  if (nchunks / kWarps >= 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const unsigned grid = flat_grid(nchunks);
  if (dx != a && dx != dy)
    return launch(k_bwd<OP, FMT, true, U>, grid, s, ap, dp, xp, (uint32_t)head, nvec, tail, lut);
  return launch(k_bwd<OP, FMT, false, U>, grid, s, ap, dp, xp, (uint32_t)head, nvec, tail, lut);
}

cudaError_t launch_bwd(int op, int fmt, const void *a, const void *dy, void *dx, size_t n,
                       const LutWords &lut, cudaStream_t s, const LaunchInfo &li) {
#define KT_CASE(O, F) \
  if (op == O && fmt == F) return launch_bwd_op<O, F>(a, dy, dx, n, lut, s, li);
  KT_CASE(OP_TANH, FMT_BF16)
  KT_CASE(OP_SIGMOID, FMT_BF16)
  KT_CASE(OP_SWISH, FMT_BF16)
  KT_CASE(OP_GELU, FMT_BF16)
  KT_CASE(OP_TANH, FMT_F32)
  KT_CASE(OP_SIGMOID, FMT_F32)
  KT_CASE(OP_SWISH, FMT_F32)
  KT_CASE(OP_GELU, FMT_F32)
#undef KT_CASE
  return cudaErrorInvalidValue;
}

cudaError_t launch_map64(const void *x, void *y, size_t n, const LutWords64 &lut, cudaStream_t s,
                         const LaunchInfo &li) {
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
  const uint8_t *xp = static_cast<const uint8_t *>(x);
  uint8_t *yp = static_cast<uint8_t *>(y);
  if ((xa % kVecBytes) != (ya % kVecBytes)) {
    static const int bps = resident_blocks(k_map64_elem);
    const unsigned grid = grid_for((n + 31) / 32, li.sm_count, bps);
    return launch(k_map64_elem, grid, s, xp, yp, (uint64_t)n, lut);
  }
  const size_t mis = xa % kVecBytes;
  size_t head = mis ? (kVecBytes - mis) / 2 : 0;
  if (head > n) head = n;
  const size_t body = n - head;
  const uint64_t nvec = body / 16;
  const uint32_t tail = (uint32_t)(body - nvec * 16);
  constexpr int U = KT_UNROLL_64;
  const uint64_t nchunks = (nvec + 32 * U - 1) / (32 * U);
  if (nchunks / kWarps >= 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const unsigned grid = flat_grid(nchunks);
  if (x != y) {
    static const int bps = resident_blocks(k_map64<true, U>);
    const uint32_t pf = prefetch_enabled() ? (uint32_t)(li.sm_count * bps) : 0u;
    return launch(k_map64<true, U>, grid, s, xp, yp, (uint32_t)head, nvec, tail, pf, lut);
  }
  return launch(k_map64<false, U>, grid, s, xp, yp, (uint32_t)head, nvec, tail, 0u, lut);
}

template <int FMT>
static cudaError_t launch_dual_t(const void *x, void *yg, void *ys, size_t n, const LutWords &lut,
                                 cudaStream_t s, const LaunchInfo &li) {
  constexpr size_t es = (FMT == FMT_BF16) ? 2 : 4;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ga = reinterpret_cast<uintptr_t>(yg),
                  sa = reinterpret_cast<uintptr_t>(ys);
  const uint8_t *xp = static_cast<const uint8_t *>(x);
  uint8_t *gp = static_cast<uint8_t *>(yg), *sp = static_cast<uint8_t *>(ys);
  if (xa % kVecBytes != ga % kVecBytes || xa % kVecBytes != sa % kVecBytes) {
    static const int bps = resident_blocks(k_dual_elem<FMT>);
    const unsigned grid = grid_for((n + 31) / 32, li.sm_count, bps);
    return launch(k_dual_elem<FMT>, grid, s, xp, gp, sp, (uint64_t)n, lut);
  }
  const size_t mis = xa % kVecBytes;
  size_t head = mis ? (kVecBytes - mis) / es : 0;
  if (head > n) head = n;
  const size_t body = n - head;
  const uint64_t nvec = body / (kVecBytes / es);
  const uint32_t tail = (uint32_t)(body - nvec * (kVecBytes / es));
  constexpr int U = dual_unroll<FMT>();
  const uint64_t nchunks = (nvec + 32 * U - 1) / (32 * U);
  if (nchunks / kWarps >= 0x7FFFFFFFull) return cudaErrorInvalidValue;
  const unsigned grid = flat_grid(nchunks);
  if (x != yg && x != ys) {
    static const int bps = resident_blocks(k_dual<FMT, true, U>);
    const uint32_t pf = prefetch_enabled() ? (uint32_t)(li.sm_count * bps) : 0u;
    return launch(k_dual<FMT, true, U>, grid, s, xp, gp, sp, (uint32_t)head, nvec, tail, pf, lut);
  }
  return launch(k_dual<FMT, false, U>, grid, s, xp, gp, sp, (uint32_t)head, nvec, tail, 0u, lut);
}

cudaError_t launch_dual(int fmt, const void *x, void *yg, void *ys, size_t n, const LutWords &lut,
                        cudaStream_t s, const LaunchInfo &li) {
  if (fmt == FMT_BF16) return launch_dual_t<FMT_BF16>(x, yg, ys, n, lut, s, li);
  return launch_dual_t<FMT_F32>(x, yg, ys, n, lut, s, li);
}

cudaError_t launch_lstm(const uint16_t *x, uint16_t *y, size_t rows, size_t hidden,
                        int tanh_quarter, const LutWords &lut, cudaStream_t s,
                        const LaunchInfo &li) {
  const size_t n = rows * 4 * hidden;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(y);
  const uint64_t nvec = n / 16;
  const bool vec_ok = (xa % kVecBytes) == 0 && (ya % kVecBytes) == 0 && hidden % 16 == 0 &&
                      nvec < (1ull << 31);
  if (vec_ok) {
    const uint64_t nchunks = (nvec + kChunkVecs - 1) / kChunkVecs;
    const unsigned grid = flat_grid(nchunks);
    const uint8_t *xp = reinterpret_cast<const uint8_t *>(x);
    uint8_t *yp = reinterpret_cast<uint8_t *>(y);
    const uint32_t vpr = (uint32_t)(hidden / 4), vpq = (uint32_t)(hidden / 16);
    if (static_cast<const void *>(x) != static_cast<const void *>(y)) {
      static const int bps = resident_blocks(k_lstm<true>);
      const uint32_t pf_blocks = prefetch_enabled() ? (uint32_t)(li.sm_count * bps) : 0u;
      return launch(k_lstm<true>, grid, s, xp, yp, (uint32_t)nvec, vpr, vpq, tanh_quarter,
                    pf_blocks, lut);
    }
    return launch(k_lstm<false>, grid, s, xp, yp, (uint32_t)nvec, vpr, vpq, tanh_quarter, 0u, lut);
  }
  static const int bps = resident_blocks(k_lstm_elem);
  const unsigned grid = grid_for((n + 31) / 32, li.sm_count, bps);
  return launch(k_lstm_elem, grid, s, x, y, (uint64_t)n, (uint64_t)(4 * hidden), (uint64_t)hidden,
                tanh_quarter, lut);
}

cudaError_t launch_lstm_cell(const uint16_t *gates, const float *c_prev, float *c_next,
                             uint16_t *h_next, size_t rows, size_t hidden, const LutWords &lut,
                             cudaStream_t s, const LaunchInfo &li) {
  const size_t n = rows * hidden;
  const bool aligned = ((reinterpret_cast<uintptr_t>(gates) | reinterpret_cast<uintptr_t>(c_prev) |
                         reinterpret_cast<uintptr_t>(c_next) | reinterpret_cast<uintptr_t>(h_next)) %
                        kVecBytes) == 0;
  const uint64_t nvec = n / 16;
  static const int which = [] {
    // dev A/B: 0 = register-staged (default, measured fastest), 1 = persistent
    // shared-memory ring (profiles/cell_variants_r02.txt)
    const char *e = getenv("KT_CELL_KERNEL");
    return e ? atoi(e) : KT_CELL_DEFAULT;
  }();
  if (which == 1 && aligned && hidden % 16 == 0 && hidden >= kCellMinHidden && n > 0) {
    static int attr_done[64];   // per device: the limit is a per-context function attribute
    if (li.device < 0 || li.device >= 64) return cudaErrorInvalidDevice;
    if (!__atomic_load_n(&attr_done[li.device], __ATOMIC_ACQUIRE)) {
      const cudaError_t ea = cudaFuncSetAttribute(k_lstm_cell_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)kCellSmem);
      if (ea != cudaSuccess) return ea;
      __atomic_store_n(&attr_done[li.device], 1, __ATOMIC_RELEASE);
    }
    static const int bps = [] {
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_lstm_cell_tma, kCellThreads, kCellSmem) !=
              cudaSuccess || b < 1)
        b = 1;
      return b;
    }();
    const uint64_t tiles = (n + kCellTile - 1) / kCellTile;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)li.sm_count * bps));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kCellThreads);
    cfg.dynamicSmemBytes = kCellSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_lstm_cell_tma, reinterpret_cast<const uint8_t *>(gates),
                                             reinterpret_cast<const uint8_t *>(c_prev),
                                             reinterpret_cast<uint8_t *>(c_next), reinterpret_cast<uint8_t *>(h_next),
                                             (uint64_t)n, (uint32_t)hidden, lut);
    count_launch();
    return e;
  }
  if (aligned && hidden % 16 == 0 && nvec < (1ull << 31)) {
    const uint64_t nwarps = (nvec + 31) / 32;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, (nwarps + kCellW - 1) / kCellW);
    static const int bps = resident_blocks(k_lstm_cell<true>, kCellTPB);
    static const int pf_on = [] {
      const char *e = getenv("KT_CELL_PF");     // dev A/B: 0 = no first-wave L2 prefetch
      return e ? atoi(e) : 1;
    }();
    const uint32_t pf_blocks = (pf_on && prefetch_enabled()) ? (uint32_t)(li.sm_count * bps) : 0u;
    auto kern = (static_cast<const void *>(c_next) == static_cast<const void *>(c_prev)) ? k_lstm_cell<false>
                                                                                         : k_lstm_cell<true>;
    return launch_tpb(kern, grid, kCellTPB, s, reinterpret_cast<const uint8_t *>(gates),
                      reinterpret_cast<const uint8_t *>(c_prev), reinterpret_cast<uint8_t *>(c_next),
                      reinterpret_cast<uint8_t *>(h_next), (uint32_t)nvec, (uint32_t)(hidden / 16),
                      (uint32_t)hidden, pf_blocks, lut);
  }
  static const int bps = resident_blocks(k_lstm_cell_elem);
  const unsigned grid = grid_for((n + 31) / 32, li.sm_count, bps);
  return launch(k_lstm_cell_elem, grid, s, gates, c_prev, c_next, h_next, (uint64_t)n,
                (uint64_t)hidden, lut);
}

}  // namespace kt
