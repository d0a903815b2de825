// kt_gemm.cu -- tcgen05 GEMM with a K-TanH-family epilogue (SURVEY.md NEXT-2:
// "a K-GELU epilogue on the FFN GEMM output ... removes a full HBM round
// trip"; the paper's motivation: activations matter more as
// GEMMs accelerate).
//
//   C[M, N] = act( RN_bf16( A[M, K] . B[N, K]^T ) ),  A, B, C BF16 row-major,
//   fp32 accumulation in TMEM, act in {none, K-TanH, K-Sigmoid, K-Swish,
//   K-GELU} applied to the BF16-rounded accumulator exactly as the
//   elementwise kernels apply it to a BF16 tensor -- so the fused output is
//   bit-identical to "GEMM with BF16 output, then k<op>_bf16".
//
// Structure (one 128 x 256 output tile per CTA, 192 threads):
//   warp 0      TMEM allocation (whole warp), then lane 0 = TMA producer:
//               A/B tiles (128 x 64 and 256 x 64 BF16, 128-byte swizzle) into
//               a 4-stage shared-memory ring, mbarrier expect_tx completion.
//   warp 1      lane 0 = MMA issuer: tcgen05.mma.cta_group::1.kind::f16,
//               M=128 N=256 K=16, four per 64-wide K block, accumulating in
//               256 TMEM columns; tcgen05.commit frees each smem stage and,
//               after the last K block, signals the epilogue.
//   warps 2-5   epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes
//               32*(w%4)..+31 = tile rows), pack to BF16 (RNE), apply the
//               K-op with the warp-shuffle LUT, 256-bit stores.
// Every mbarrier wait is bounded (a trap instead of a hang).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kt_device.cuh"
#include "kt_internal.h"

namespace kt {

constexpr int kBM = 128, kBN = 256, kBK = 64, kStages = 4;
constexpr uint32_t kABytes = kBM * kBK * 2;          // 16 KiB
constexpr uint32_t kBBytes = kBN * kBK * 2;          // 32 KiB
constexpr uint32_t kStageBytes = kABytes + kBBytes;  // 48 KiB
constexpr uint32_t kTmemCols = 256;
constexpr size_t kGemmSmem = (size_t)kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
static_assert(8 * 4 * 4 + 64 <= 256, "barrier area");

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t phase) {
  uint32_t ok = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(a), "r"(phase) : "memory");
    if (ok) return;
    if (spin > (1u << 26)) __trap();   // never hang the GPU on a protocol bug
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms of
// 1024 B (SBO), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;          // SBO = 1024 B
  d |= (uint64_t)1 << 46;                    // version
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

// Instruction descriptor: A/B BF16, D F32, K-major both, N = 256, M = 128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);

// 32 consecutive TMEM columns of this warp's 32 lanes -> r[0..31] (async;
// complete with tcgen05.wait::ld).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t *r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// Epilogue id for the LSTM gate block (config 4): K-TanH on the tanh
// quarter's columns, K-Sigmoid elsewhere; the quarter is uniform per tile
// (hidden % 256 == 0), so each tile resolves to OP_TANH or OP_SIGMOID.
constexpr int kEpiLstm = 8;

template <int EPI>
__device__ __forceinline__ uint32_t epi_word(uint32_t w, uint32_t lw) {
  if (EPI == OP_TANH) return ktanh_bf16x2(w, lw);
  if (EPI == OP_SIGMOID) return ksigmoid_bf16x2(w, lw);
  if (EPI == OP_SWISH) return kswish_bf16x2(w, lw);
  if (EPI == OP_GELU) return kgelu_bf16x2(w, lw);
  return w;
}

// 32 fp32 accumulators (TMEM columns c..c+31 of one row) -> RN_bf16 -> op ->
// two 16-element output vectors.
template <int EPI>
__device__ __forceinline__ void epi_chunk32(const uint32_t *r, uint32_t (&o0)[8], uint32_t (&o1)[8],
                                            uint32_t lw) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    o0[j] = epi_word<EPI>(pack_bf16x2(__uint_as_float(r[2 * j + 1]), __uint_as_float(r[2 * j])), lw);
    o1[j] = epi_word<EPI>(pack_bf16x2(__uint_as_float(r[2 * j + 17]), __uint_as_float(r[2 * j + 16])),
                          lw);
  }
}

template <int EPI>
__device__ __forceinline__ void epi_tile_chunk(const uint32_t *r, uint32_t (&o0)[8], uint32_t (&o1)[8],
                                               uint32_t lw, bool tanh_tile) {
  if (EPI == kEpiLstm) {
    if (tanh_tile) epi_chunk32<OP_TANH>(r, o0, o1, lw);          // warp-uniform per tile
    else epi_chunk32<OP_SIGMOID>(r, o0, o1, lw);
  } else {
    epi_chunk32<EPI>(r, o0, o1, lw);
  }
}

// Persistent variant: grid = min(tiles, SMs); each CTA walks tiles
// blockIdx.x, += gridDim.x (n fastest within a group of kGroupM row blocks, so
// concurrently running CTAs share B panels in L2).  Two TMEM accumulator
// stages (2 x 256 columns = all 512): the epilogue of tile i (8 warps: lane
// quarter = warp % 4, column half = (warp - 2) / 4) overlaps the mainloop of
// tile i + 1.  Barriers: smem ring full/empty (continuous across tiles),
// tmem_full[2] (MMA -> epilogue), tmem_empty[2] (epilogue -> MMA, 8 arrivals).
constexpr int kEpiWarps = 8;
constexpr int kGemmPThreads = 64 + 32 * kEpiWarps;
constexpr int kGroupM = 16;

__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t mt, uint32_t ntiles_n, uint32_t &mb,
                                            uint32_t &nb) {
  const uint32_t per_group = kGroupM * ntiles_n;
  const uint32_t g = t / per_group, r = t - g * per_group;
  const uint32_t rows = min((uint32_t)kGroupM, mt - g * kGroupM);
  mb = g * kGroupM + r % rows;
  nb = r / rows;
}

template <int EPI>
__global__ void __launch_bounds__(kGemmPThreads, 1)
k_gemm(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
       uint16_t *C, uint32_t M, uint32_t N, uint32_t K, uint32_t epi_hidden, uint32_t epi_tq, const __grid_constant__ LutWords lut) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar = base + kStages * kStageBytes;
  const uint32_t full_bar = bar, empty_bar = bar + 8 * kStages;
  const uint32_t tfull_bar = bar + 16 * kStages, tempty_bar = tfull_bar + 16;
  const uint32_t tmem_slot = tempty_bar + 16;
  uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem_raw + (tmem_slot - raw));

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t mt = M / kBM, ntn = N / kBN, ntiles = mt * ntn;
  const uint32_t nk = K / kBK;
  const uint32_t lw = lut.bf16[lane];

  if (threadIdx.x == 32) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar + 8 * a, 1);
      mbar_init(tempty_bar + 8 * a, kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "n"(2 * kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % kStages;
        if (it >= (uint32_t)kStages) mbar_wait(empty_bar + 8 * s, ((it / kStages) + 1) & 1);
        const uint32_t sa = base + s * kStageBytes, sb = sa + kABytes;
        mbar_expect_tx(full_bar + 8 * s, kStageBytes);
        tma_load_2d(sa, &map_a, (int)(kb * kBK), (int)(mb * kBM), full_bar + 8 * s);
        tma_load_2d(sb, &map_b, (int)(kb * kBK), (int)(nb * kBN), full_bar + 8 * s);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    uint32_t it = 0, i = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const uint32_t a = i & 1;
      if (i >= 2) mbar_wait(tempty_bar + 8 * a, ((i / 2) + 1) & 1);   // epilogue drained stage a
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + a * kTmemCols;
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % kStages;
        mbar_wait(full_bar + 8 * s, (it / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_sdesc(base + s * kStageBytes);
        const uint64_t db = umma_sdesc(base + s * kStageBytes + kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint32_t acc = (kb | k) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(kIdesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         empty_bar + 8 * s)
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       tfull_bar + 8 * a)
                   : "memory");
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (8 warps) ----------------
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    uint32_t i = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      const uint32_t a = i & 1;
      mbar_wait(tfull_bar + 8 * a, (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t row = mb * kBM + 32 * q + lane;
      uint16_t *crow = C + (size_t)row * N + nb * kBN + half * 128;
      const bool tanh_tile = EPI == kEpiLstm && (nb * kBN) / epi_hidden == epi_tq;
#pragma unroll 1
      for (uint32_t c = 0; c < 128; c += 32) {
        uint32_t r[32];
        const uint32_t taddr = tmem + ((32 * q) << 16) + a * kTmemCols + half * 128 + c;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
            "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c == 96) {
          // all of this warp's TMEM reads for tile i are done: release stage a
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_bar + 8 * a) : "memory");
        }
        uint32_t o0[8], o1[8];
        epi_tile_chunk<EPI>(r, o0, o1, lw, tanh_tile);
        st256(crow + c, o0, true);
        st256(crow + c + 16, o1, true);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * kTmemCols));
  }
}

// ------------------------------------- GEMM + fused LSTM cell (NEXT-2) ----
// gates = RN_bf16(A[M, K] . B[4H, K]^T) with B in PyTorch's row-block order
// (i, f, g, o), then the cell of klstm_cell_bf16 -- without writing the gate
// block: c_next = RN32(f c_prev + i g), h_next = RN_bf16(o K-TanH_f32(c_next)),
// i, f, o = K-Sigmoid, g = K-TanH of the BF16 gates (reading R-LSTM-CELL).
// A tile covers 128 rows x 64 hidden units: its B operand is the four
// 64-row boxes B[q*H + 64 nb .. +64) (q = i, f, g, o) stacked in shared
// memory -- the same 256-row, 128-byte-swizzled layout as one 256-row box --
// so TMEM column q*64 + u holds gate q of unit u.  Epilogue warp (lane
// quarter, unit half) loads gates i, f, g, o of its 32 units (4 x 32 columns)
// and c_prev of its row, and writes c_next (F32) and h_next (BF16).  The MMA
// side is k_gemm's.  10 bytes of cell traffic per element instead of 8 (gate
// write) + 18 (cell kernel).
__global__ void __launch_bounds__(kGemmPThreads, 1)
k_gemm_cell(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b64,
            const float *c_prev, float *c_next, uint16_t *h_next, uint32_t M, uint32_t H, uint32_t K,
            const __grid_constant__ LutWords lut) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar = base + kStages * kStageBytes;
  const uint32_t full_bar = bar, empty_bar = bar + 8 * kStages;
  const uint32_t tfull_bar = bar + 16 * kStages, tempty_bar = tfull_bar + 16;
  const uint32_t tmem_slot = tempty_bar + 16;
  uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem_raw + (tmem_slot - raw));

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t mt = M / kBM, ntn = H / 64, ntiles = mt * ntn;
  const uint32_t nk = K / kBK;

  if (threadIdx.x == 32) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar + 8 * a, 1);
      mbar_init(tempty_bar + 8 * a, kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "n"(2 * kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer: A box + four 64-row B boxes ----------------
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % kStages;
        if (it >= (uint32_t)kStages) mbar_wait(empty_bar + 8 * s, ((it / kStages) + 1) & 1);
        const uint32_t sa = base + s * kStageBytes, sb = sa + kABytes;
        mbar_expect_tx(full_bar + 8 * s, kStageBytes);
        tma_load_2d(sa, &map_a, (int)(kb * kBK), (int)(mb * kBM), full_bar + 8 * s);
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          tma_load_2d(sb + q * (64 * kBK * 2), &map_b64, (int)(kb * kBK), (int)(q * H + nb * 64),
                      full_bar + 8 * s);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (as k_gemm) ----------------
    uint32_t it = 0, i = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      const uint32_t a = i & 1;
      if (i >= 2) mbar_wait(tempty_bar + 8 * a, ((i / 2) + 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + a * kTmemCols;
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % kStages;
        mbar_wait(full_bar + 8 * s, (it / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_sdesc(base + s * kStageBytes);
        const uint64_t db = umma_sdesc(base + s * kStageBytes + kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint32_t acc = (kb | k) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(kIdesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         empty_bar + 8 * s)
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       tfull_bar + 8 * a)
                   : "memory");
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: LSTM cell of 32 units of one row ----------------
    const LaneLut L{lut.bf16[lane], lut.f32K[lane], lut.f32C[lane]};
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    uint32_t i = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      const uint32_t a = i & 1;
      const uint32_t row = mb * kBM + 32 * q + lane;
      const size_t cbase = (size_t)row * H + nb * 64 + half * 32;     // first unit of this thread
      uint32_t cp[4][8];                                              // c_prev, 32 floats
#pragma unroll
      for (int v = 0; v < 4; ++v) ld256<true>(c_prev + cbase + 8 * v, cp[v], true);
      mbar_wait(tfull_bar + 8 * a, (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[128];                                                // i, f, g, o x 32 units
      const uint32_t tbase = tmem + ((32 * q) << 16) + a * kTmemCols + half * 32;
#pragma unroll
      for (int g = 0; g < 4; ++g) tmem_ld32(tbase + 64 * g, r + 32 * g);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_bar + 8 * a) : "memory");
      uint32_t cn[4][8], h[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {                                  // units 2k, 2k + 1
        const uint32_t gi = pack_bf16x2(__uint_as_float(r[2 * k + 1]), __uint_as_float(r[2 * k]));
        const uint32_t gf = pack_bf16x2(__uint_as_float(r[32 + 2 * k + 1]), __uint_as_float(r[32 + 2 * k]));
        const uint32_t gg = pack_bf16x2(__uint_as_float(r[64 + 2 * k + 1]), __uint_as_float(r[64 + 2 * k]));
        const uint32_t go = pack_bf16x2(__uint_as_float(r[96 + 2 * k + 1]), __uint_as_float(r[96 + 2 * k]));
        float2 cnv;
        h[k] = lstm_cell2(gi, gf, gg, go,
                          make_float2(__uint_as_float(cp[k >> 2][(2 * k) & 7]),
                                      __uint_as_float(cp[k >> 2][(2 * k + 1) & 7])),
                          cnv, L);
        cn[k >> 2][(2 * k) & 7] = __float_as_uint(cnv.x);
        cn[k >> 2][(2 * k + 1) & 7] = __float_as_uint(cnv.y);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) st256(c_next + cbase + 8 * v, cn[v], true);
      uint32_t h0[8], h1[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        h0[j] = h[j];
        h1[j] = h[8 + j];
      }
      st256(h_next + cbase, h0, true);
      st256(h_next + cbase + 16, h1, true);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * kTmemCols));
  }
}

// ------------------------------------------------ CTA-pair (cta_group::2) ----
// Two CTAs of a cluster (two SMs of one TPC) compute one 256 x 256 output
// tile: CTA r loads rows [r*128, +128) of the A block and rows [r*128, +128)
// of the B panel (its half of N); the leader (rank 0) issues
// tcgen05.mma.cta_group::2 M=256 N=256 K=16, which reads both CTAs' shared
// memory and accumulates rows r*128.. into CTA r's TMEM.  Per CTA and K block
// that is 32 KiB of operands instead of 48 KiB for the same 128 x 256 output,
// so 6 pipeline stages fit.  Barrier protocol:
//   full[s]   leader only: 1 arrival (leader's expect_tx of both CTAs' bytes);
//             both CTAs' TMA loads complete_tx on it (.cta_group::2 TMA)
//   empty[s]  both CTAs: the leader's tcgen05.commit multicasts to both
//   tfull[a]  both CTAs: commit multicast after the last K block of a tile
//   tempty[a] leader only: 2 x 8 epilogue-warp arrivals (the peer's remote)
constexpr int k2Stages = 6;
constexpr uint32_t k2HalfBytes = 128 * kBK * 2;                // 16 KiB
constexpr uint32_t k2StageBytes = 2 * k2HalfBytes;             // A half + B half
constexpr size_t k2Smem = (size_t)k2Stages * k2StageBytes + 1024 + 256;
constexpr uint32_t kIdesc2 = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) |
                             ((256u >> 4) << 24);
static_assert(8 * 2 * k2Stages + 8 * 4 + 8 <= 256, "barrier area");

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_rank0(uint32_t a) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(d) : "r"(a));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                                 uint32_t mbar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(map), "r"(c0), "r"(c1), "r"(mbar_cluster)
      : "memory");
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmPThreads, 1)
k_gemm2(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
        uint16_t *C, uint32_t M, uint32_t N, uint32_t K, uint32_t epi_hidden, uint32_t epi_tq, const __grid_constant__ LutWords lut) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar = base + k2Stages * k2StageBytes;
  const uint32_t full_bar = bar, empty_bar = bar + 8 * k2Stages;
  const uint32_t tfull_bar = bar + 16 * k2Stages, tempty_bar = tfull_bar + 16;
  const uint32_t tmem_slot = tempty_bar + 16;
  uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem_raw + (tmem_slot - raw));

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const uint32_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t mt = M / 256, ntn = N / 256, ntiles = mt * ntn;
  const uint32_t nk = K / kBK;
  const uint32_t lw = lut.bf16[lane];

  if (threadIdx.x == 32) {
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar + 8 * a, 1);
      mbar_init(tempty_bar + 8 * a, 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "n"(2 * kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();   // barriers of both CTAs initialised before any remote use
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    uint32_t it = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % k2Stages;
        if (it >= (uint32_t)k2Stages) mbar_wait(empty_bar + 8 * s, ((it / k2Stages) + 1) & 1);
        const uint32_t sa = base + s * k2StageBytes, sb = sa + k2HalfBytes;
        const uint32_t fb = map_to_rank0(full_bar + 8 * s);
        if (leader) mbar_expect_tx(full_bar + 8 * s, 2 * k2StageBytes);
        tma_load_2d_pair(sa, &map_a, (int)(kb * kBK), (int)(mb * 256 + rank * 128), fb);
        tma_load_2d_pair(sb, &map_b, (int)(kb * kBK), (int)(nb * 256 + rank * 128), fb);
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (leader only) ----------------
    uint32_t it = 0, i = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl, ++i) {
      const uint32_t a = i & 1;
      if (i >= 2) mbar_wait(tempty_bar + 8 * a, ((i / 2) + 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + a * kTmemCols;
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % k2Stages;
        mbar_wait(full_bar + 8 * s, (it / k2Stages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_sdesc(base + s * k2StageBytes);
        const uint64_t db = umma_sdesc(base + s * k2StageBytes + k2HalfBytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint32_t acc = (kb | k) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(kIdesc2), "r"(acc));
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;" ::"r"(empty_bar + 8 * s), "h"((uint16_t)3)
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
          " [%0], %1;" ::"r"(tfull_bar + 8 * a), "h"((uint16_t)3)
          : "memory");
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (8 warps, both CTAs) ----------------
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    const uint32_t tempty_leader = map_to_rank0(tempty_bar);
    uint32_t i = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl, ++i) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      const uint32_t a = i & 1;
      mbar_wait(tfull_bar + 8 * a, (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t row = mb * 256 + rank * 128 + 32 * q + lane;
      uint16_t *crow = C + (size_t)row * N + nb * 256 + half * 128;
      const bool tanh_tile = EPI == kEpiLstm && (nb * 256) / epi_hidden == epi_tq;
      // All 128 of this warp's columns in flight at once, one wait, then the
      // TMEM stage is released before any epilogue arithmetic (the MMA of the
      // tile after next can start while the activation runs).
      uint32_t r[128];
      const uint32_t tbase = tmem + ((32 * q) << 16) + a * kTmemCols + half * 128;
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) tmem_ld32(tbase + 32 * c4, r + 32 * c4);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      // Relaxed: the TMEM reads are complete (wait::ld) and fenced by
      // tcgen05.fence::before_thread_sync; a .release.cluster arrive would
      // add a GPU-scope MEMBAR that waits for this warp's outstanding C
      // stores.
      if (lane == 0) {
        if (leader)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_bar + 8 * a) : "memory");
        else
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           tempty_leader + 8 * a)
                       : "memory");
      }
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        uint32_t o0[8], o1[8];
        epi_tile_chunk<EPI>(r + 32 * c4, o0, o1, lw, tanh_tile);
        st256(crow + 32 * c4, o0, true);
        st256(crow + 32 * c4 + 16, o1, true);
      }
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();   // both CTAs done with TMEM and with each other's barriers
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * kTmemCols));
  }
}

// CTA-pair version of k_gemm_cell: a cluster computes 256 rows x 64 units;
// CTA r loads gates 2r, 2r + 1 (its half of the 256 B rows).
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmPThreads, 1)
k_gemm2_cell(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b64,
             const float *c_prev, float *c_next, uint16_t *h_next, uint32_t M, uint32_t H, uint32_t K,
             const __grid_constant__ LutWords lut) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar = base + k2Stages * k2StageBytes;
  const uint32_t full_bar = bar, empty_bar = bar + 8 * k2Stages;
  const uint32_t tfull_bar = bar + 16 * k2Stages, tempty_bar = tfull_bar + 16;
  const uint32_t tmem_slot = tempty_bar + 16;
  uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem_raw + (tmem_slot - raw));

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const uint32_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const uint32_t mt = M / 256, ntn = H / 64, ntiles = mt * ntn;
  const uint32_t nk = K / kBK;

  if (threadIdx.x == 32) {
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar + 8 * a, 1);
      mbar_init(tempty_bar + 8 * a, 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                 "n"(2 * kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();   // barriers of both CTAs initialised before any remote use
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    uint32_t it = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % k2Stages;
        if (it >= (uint32_t)k2Stages) mbar_wait(empty_bar + 8 * s, ((it / k2Stages) + 1) & 1);
        const uint32_t sa = base + s * k2StageBytes, sb = sa + k2HalfBytes;
        const uint32_t fb = map_to_rank0(full_bar + 8 * s);
        if (leader) mbar_expect_tx(full_bar + 8 * s, 2 * k2StageBytes);
        tma_load_2d_pair(sa, &map_a, (int)(kb * kBK), (int)(mb * 256 + rank * 128), fb);
        // this CTA's half of N = gates 2r, 2r + 1 (64 rows each) of units [64 nb, +64)
        tma_load_2d_pair(sb, &map_b64, (int)(kb * kBK), (int)((2 * rank) * H + nb * 64), fb);
        tma_load_2d_pair(sb + 64 * kBK * 2, &map_b64, (int)(kb * kBK), (int)((2 * rank + 1) * H + nb * 64),
                         fb);
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (leader only) ----------------
    uint32_t it = 0, i = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl, ++i) {
      const uint32_t a = i & 1;
      if (i >= 2) mbar_wait(tempty_bar + 8 * a, ((i / 2) + 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + a * kTmemCols;
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % k2Stages;
        mbar_wait(full_bar + 8 * s, (it / k2Stages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_sdesc(base + s * k2StageBytes);
        const uint64_t db = umma_sdesc(base + s * k2StageBytes + k2HalfBytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint32_t acc = (kb | k) != 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
              "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(kIdesc2), "r"(acc));
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
            " [%0], %1;" ::"r"(empty_bar + 8 * s), "h"((uint16_t)3)
            : "memory");
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
          " [%0], %1;" ::"r"(tfull_bar + 8 * a), "h"((uint16_t)3)
          : "memory");
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: LSTM cell, both CTAs (as k_gemm_cell) ----------------
    const LaneLut L{lut.bf16[lane], lut.f32K[lane], lut.f32C[lane]};
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    const uint32_t tempty_leader = map_to_rank0(tempty_bar);
    uint32_t i = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl, ++i) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      const uint32_t a = i & 1;
      const uint32_t row = mb * 256 + rank * 128 + 32 * q + lane;
      const size_t cbase = (size_t)row * H + nb * 64 + half * 32;
      uint32_t cp[4][8];
#pragma unroll
      for (int v = 0; v < 4; ++v) ld256<true>(c_prev + cbase + 8 * v, cp[v], true);
      mbar_wait(tfull_bar + 8 * a, (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t r[128];
      const uint32_t tbase = tmem + ((32 * q) << 16) + a * kTmemCols + half * 32;
#pragma unroll
      for (int g = 0; g < 4; ++g) tmem_ld32(tbase + 64 * g, r + 32 * g);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (leader)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_bar + 8 * a) : "memory");
        else
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           tempty_leader + 8 * a)
                       : "memory");
      }
      uint32_t cn[4][8], h[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint32_t gi = pack_bf16x2(__uint_as_float(r[2 * k + 1]), __uint_as_float(r[2 * k]));
        const uint32_t gf = pack_bf16x2(__uint_as_float(r[32 + 2 * k + 1]), __uint_as_float(r[32 + 2 * k]));
        const uint32_t gg = pack_bf16x2(__uint_as_float(r[64 + 2 * k + 1]), __uint_as_float(r[64 + 2 * k]));
        const uint32_t go = pack_bf16x2(__uint_as_float(r[96 + 2 * k + 1]), __uint_as_float(r[96 + 2 * k]));
        float2 cnv;
        h[k] = lstm_cell2(gi, gf, gg, go,
                          make_float2(__uint_as_float(cp[k >> 2][(2 * k) & 7]),
                                      __uint_as_float(cp[k >> 2][(2 * k + 1) & 7])),
                          cnv, L);
        cn[k >> 2][(2 * k) & 7] = __float_as_uint(cnv.x);
        cn[k >> 2][(2 * k + 1) & 7] = __float_as_uint(cnv.y);
      }
#pragma unroll
      for (int v = 0; v < 4; ++v) st256(c_next + cbase + 8 * v, cn[v], true);
      uint32_t h0[8], h1[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        h0[j] = h[j];
        h1[j] = h[8 + j];
      }
      st256(h_next + cbase, h0, true);
      st256(h_next + cbase + 16, h1, true);
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();   // both CTAs done with TMEM and with each other's barriers
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(2 * kTmemCols));
  }
}

// ---------------------------------------------------------------- host ----

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// rows x K BF16 row-major, box (64 K-elements x box_rows rows), 128-byte swizzle
static bool make_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint64_t K, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {K, rows};
  cuuint64_t strides[1] = {K * 2};
  cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int EPI>
static cudaError_t launch_gemm_t(const CUtensorMap &ma, const CUtensorMap &mb, uint16_t *C, size_t M,
                                 size_t N, size_t K, const LutWords &lut, cudaStream_t s, int sms,
                                 uint32_t eh, uint32_t etq) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_gemm<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kGemmSmem);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const size_t tiles = (M / kBM) * (N / kBN);
  const unsigned grid = (unsigned)(tiles < (size_t)sms ? tiles : (size_t)sms);
  k_gemm<EPI><<<grid, kGemmPThreads, kGemmSmem, s>>>(ma, mb, C, (uint32_t)M, (uint32_t)N,
                                                     (uint32_t)K, eh, etq, lut);
  count_launch();
  return cudaGetLastError();
}

template <int EPI>
static cudaError_t launch_gemm2_t(const CUtensorMap &ma, const CUtensorMap &mb, uint16_t *C, size_t M,
                                  size_t N, size_t K, const LutWords &lut, cudaStream_t s, int sms,
                                  uint32_t eh, uint32_t etq) {
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_gemm2<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)k2Smem);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const size_t tiles = (M / 256) * (N / 256);
  const size_t pairs = (size_t)(sms / 2);
  const unsigned grid = (unsigned)(2 * (tiles < pairs ? tiles : pairs));
  k_gemm2<EPI><<<grid, kGemmPThreads, k2Smem, s>>>(ma, mb, C, (uint32_t)M, (uint32_t)N, (uint32_t)K,
                                                   eh, etq, lut);
  count_launch();
  return cudaGetLastError();
}

// Kernel choice (profiles/gemm_2cta_r01.txt): the CTA pair is faster for the
// plain GEMM (1.44 vs 1.51 ms at 16384^2 x 4096; 0.40 vs 0.47 ms at
// 65536 x 4096 x 1024) and for fused epilogues up to ~2^38 MACs; on the
// sustained, power-capped FFN GEMM with K-GELU the 1-CTA kernel is 1-3%
// ahead.  KT_GEMM_2CTA=0/1 forces either for M % 256 == 0.
static bool use_pair(size_t M, size_t N, size_t K, int epi) {
  static const int force = [] {
    const char *e = getenv("KT_GEMM_2CTA");
    return e ? atoi(e) : -1;
  }();
  if (M % 256 != 0) return false;
  if (force >= 0) return force != 0;
  // fused epilogues on very large, power-capped GEMMs (the FFN line:
  // 2^42 MACs) run 1-3% faster on the 1-CTA kernel; smaller fused GEMMs (the
  // LSTM gate GEMM, 2^34.7 MACs: 51.3 vs 53.1 us) on the pair
  return epi < 0 || (double)M * (double)N * (double)K < 274877906944.0;   // 2^38
}

cudaError_t launch_gemm(int epi, const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M,
                        size_t N, size_t K, const LutWords &lut, cudaStream_t s, int sms,
                        uint32_t lstm_hidden, uint32_t lstm_tq) {
  CUtensorMap ma, mb;
  const uint32_t eh = lstm_hidden ? lstm_hidden : 1u, etq = lstm_tq;
#define KT_EPIS(L)                                                       \
  switch (epi) {                                                         \
    case -1: return L<-1>(ma, mb, C, M, N, K, lut, s, sms, eh, etq);      \
    case OP_TANH: return L<OP_TANH>(ma, mb, C, M, N, K, lut, s, sms, eh, etq);       \
    case OP_SIGMOID: return L<OP_SIGMOID>(ma, mb, C, M, N, K, lut, s, sms, eh, etq); \
    case OP_SWISH: return L<OP_SWISH>(ma, mb, C, M, N, K, lut, s, sms, eh, etq);     \
    case OP_GELU: return L<OP_GELU>(ma, mb, C, M, N, K, lut, s, sms, eh, etq);       \
    case kEpiLstm: return L<kEpiLstm>(ma, mb, C, M, N, K, lut, s, sms, eh, etq);     \
  }                                                                      \
  return cudaErrorInvalidValue;
  if (use_pair(M, N, K, epi) && sms >= 2) {
    if (!make_map(&ma, A, M, K, 128) || !make_map(&mb, B, N, K, 128)) return cudaErrorInvalidValue;
    KT_EPIS(launch_gemm2_t)
  }
  if (!make_map(&ma, A, M, K, kBM) || !make_map(&mb, B, N, K, kBN)) return cudaErrorInvalidValue;
  KT_EPIS(launch_gemm_t)
#undef KT_EPIS
}

cudaError_t launch_gemm_cell(const uint16_t *A, const uint16_t *B, const float *c_prev, float *c_next,
                             uint16_t *h_next, size_t M, size_t H, size_t K, const LutWords &lut,
                             cudaStream_t s, int sms) {
  CUtensorMap ma, mb;
  if (use_pair(M, 4 * H, K, OP_TANH) && sms >= 2) {
    if (!make_map(&ma, A, M, K, 128) || !make_map(&mb, B, 4 * H, K, 64)) return cudaErrorInvalidValue;
    static std::once_flag once2;
    static cudaError_t attr_err2 = cudaSuccess;
    std::call_once(once2, [] {
      attr_err2 = cudaFuncSetAttribute(k_gemm2_cell, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)k2Smem);
    });
    if (attr_err2 != cudaSuccess) return attr_err2;
    const size_t tiles = (M / 256) * (H / 64), pairs = (size_t)(sms / 2);
    const unsigned grid = (unsigned)(2 * (tiles < pairs ? tiles : pairs));
    k_gemm2_cell<<<grid, kGemmPThreads, k2Smem, s>>>(ma, mb, c_prev, c_next, h_next, (uint32_t)M,
                                                     (uint32_t)H, (uint32_t)K, lut);
    count_launch();
    return cudaGetLastError();
  }
  if (!make_map(&ma, A, M, K, kBM) || !make_map(&mb, B, 4 * H, K, 64)) return cudaErrorInvalidValue;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(k_gemm_cell, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kGemmSmem);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const size_t tiles = (M / kBM) * (H / 64);
  const unsigned grid = (unsigned)(tiles < (size_t)sms ? tiles : (size_t)sms);
  k_gemm_cell<<<grid, kGemmPThreads, kGemmSmem, s>>>(ma, mb, c_prev, c_next, h_next, (uint32_t)M,
                                                     (uint32_t)H, (uint32_t)K, lut);
  count_launch();
  return cudaGetLastError();
}

}  // namespace kt
