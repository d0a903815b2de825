// kt_gemm.cu -- tcgen05 GEMMs with K-TanH-family epilogues (SURVEY.md NEXT-2:
// "a K-GELU epilogue on the FFN GEMM output ... removes a full HBM round
// trip"; the paper's motivation: activations matter more as
// GEMMs accelerate; GNMT's LSTM).
//
//   C[M, N] = act( RN_bf16( A[M, K] . B[N, K]^T ) ),  A, B, C BF16 row-major,
//   fp32 accumulation in TMEM, act in {none, K-TanH, K-Sigmoid, K-Swish,
//   K-GELU, LSTM gates} applied to the BF16-rounded accumulator exactly as
//   the elementwise kernels apply it to a BF16 tensor -- so the fused output
//   is bit-identical to "GEMM with BF16 output, then k<op>_bf16"; or, for the
//   LSTM cell epilogue, no C at all: c_next / h_next of klstm_cell_bf16.
//
// One kernel template k_gemm_t<EPI, CTAS>, persistent (one CTA per SM):
//   warp 0      TMEM allocation (whole warp), then lane 0 = TMA producer:
//               A/B tiles (128-byte swizzle) into a shared-memory ring,
//               mbarrier expect_tx completion.
//   warp 1      lane 0 = MMA issuer: tcgen05.mma.cta_group::CTAS.kind::f16,
//               M = 128 * CTAS, N = 256, K = 16, four per 64-wide K block,
//               into one of two 256-column TMEM accumulator stages;
//               tcgen05.commit frees each smem stage and, after the last K
//               block, signals the epilogue.
//   warps 2-9   epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes
//               32*(w%4)..+31 = tile rows, column half (w-2)/4), RNE to BF16,
//               the K-op with the warp-shuffle LUT, 256-bit stores.  The
//               epilogue of tile i overlaps the mainloop of tile i + 1.
// CTAS = 1: a CTA computes 128 x 256 (4-stage ring of 16 + 32 KiB).
// CTAS = 2: a 2-CTA cluster (two SMs of a TPC) computes 256 x 256; CTA r
//   loads its 128 rows of A and its 128-row half of the B panel (6-stage
//   ring of 16 + 16 KiB); the leader issues tcgen05.mma.cta_group::2 over
//   both CTAs' shared memory; both CTAs' TMA loads complete_tx on the
//   leader's full barrier (.cta_group::2 TMA); commits multicast to both
//   CTAs' empty / tfull barriers; the peer's epilogue releases TMEM stages
//   with a relaxed remote arrive (a .release.cluster arrive compiles to a
//   GPU-scope MEMBAR that waits for the warp's outstanding C stores).
// LSTM cell epilogue (EPI = kEpiCell): a tile is 64 hidden units; its B
//   operand is the four (CTAS = 1) or two (CTAS = 2, CTA r: gates 2r, 2r+1)
//   64-row boxes B[q*H + 64 nb, +64) stacked into the same swizzled layout,
//   so TMEM column q*64 + u holds gate q of unit u.
// Every mbarrier wait is bounded (a trap instead of a hang).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kt_async.cuh"
#include "kt_device.cuh"
#include "kt_internal.h"

namespace kt {

constexpr int kBK = 64;                               // K block (one 128-byte swizzle row)
constexpr uint32_t kABytes = 128 * kBK * 2;          // A tile per CTA and stage: 16 KiB
constexpr uint32_t kTmemCols = 256;                  // one accumulator stage
static_assert(16 * 6 + 64 <= 256, "barrier area");

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

// 8 consecutive TMEM columns of this warp's 32 lanes -> r[0..7] (async)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t *r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
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
// K-Swish / K-GELU: the plain-fma outer step, exact unless the chunk holds an
// x/2 tie (R-DERIVED, kt_device.cuh).  The 16 packed pre-activations are
// screened first (|x| via abs.bf16x2 and a packed-u16 min: a warp-uniform
// branch on "some |x| below 2^-125, or a zero"), then the whole chunk takes
// the plain fma or the exact outer step -- 1.5 ops per pair instead of the
// exact step's 6.  KT_GEMM_EXACT_EPI=1 (dev A/B): the exact step always.
#ifndef KT_GEMM_EXACT_EPI
#define KT_GEMM_EXACT_EPI 0
#endif
template <int EPI>
__device__ __forceinline__ void epi_chunk32(const uint32_t *r, uint32_t (&o0)[8], uint32_t (&o1)[8],
                                            uint32_t lw) {
  uint32_t w0[8], w1[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    w0[j] = pack_bf16x2(__uint_as_float(r[2 * j + 1]), __uint_as_float(r[2 * j]));
    w1[j] = pack_bf16x2(__uint_as_float(r[2 * j + 17]), __uint_as_float(r[2 * j + 16]));
  }
  if ((EPI == OP_SWISH || EPI == OP_GELU) && !KT_GEMM_EXACT_EPI) {
    uint32_t kmin = 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t a0, a1;
      asm("abs.bf16x2 %0, %1;" : "=r"(a0) : "r"(w0[j]));
      asm("abs.bf16x2 %0, %1;" : "=r"(a1) : "r"(w1[j]));
      kmin = umin16x2(kmin, umin16x2(a0, a1));
    }
    if (!__any_sync(0xffffffffu, tie_possible(kmin))) {
      uint32_t m;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        o0[j] = EPI == OP_GELU ? kgelu_bf16x2_fast(w0[j], lw, m) : kswish_bf16x2_fast(w0[j], lw, m);
        o1[j] = EPI == OP_GELU ? kgelu_bf16x2_fast(w1[j], lw, m) : kswish_bf16x2_fast(w1[j], lw, m);
      }
      return;
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    o0[j] = epi_word<EPI>(w0[j], lw);
    o1[j] = epi_word<EPI>(w1[j], lw);
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
// LSTM cell epilogue warps: each warp of a TMEM lane quarter takes 64 / (W/4)
// hidden units of the tile in rounds of 8 (4 x 8 TMEM columns, 123 registers
// at W = 8, no spills; profiles/gemm_cell_epi_r02.txt).  W = 16 (88
// registers) was 4% slower on the fused step (dev A/B: -DKT_GEMM_CELL_WARPS=16).
#ifndef KT_GEMM_CELL_WARPS
#define KT_GEMM_CELL_WARPS 8
#endif
static_assert(KT_GEMM_CELL_WARPS == 8 || KT_GEMM_CELL_WARPS == 16, "cell epilogue: 8 or 16 warps");
constexpr int kGroupM = 16;

__device__ __forceinline__ void tile_coords(uint32_t t, uint32_t mt, uint32_t ntiles_n, uint32_t &mb,
                                            uint32_t &nb) {
  const uint32_t per_group = kGroupM * ntiles_n;
  const uint32_t g = t / per_group, r = t - g * per_group;
  const uint32_t rows = min((uint32_t)kGroupM, mt - g * kGroupM);
  mb = g * kGroupM + r % rows;
  nb = r / rows;
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

constexpr int kEpiCell = 9;   // the LSTM cell epilogue (see kgemm_lstm_cell_bf16)
template <int EPI>
__host__ __device__ constexpr int epi_warps() { return EPI == kEpiCell ? KT_GEMM_CELL_WARPS : kEpiWarps; }
template <int EPI>
__host__ __device__ constexpr int gemm_threads() { return 64 + 32 * epi_warps<EPI>(); }

struct GemmArgs {
  uint16_t *C;                 // output of the activation epilogues (unused for the cell)
  const float *c_prev;         // cell epilogue: c_prev, c_next [M, H] F32, h_next [M, H] BF16
  float *c_next;
  uint16_t *h_next;
  uint32_t M, N, K;            // N = 4 H for the LSTM epilogues
  uint32_t H, tq;              // LSTM: hidden size, tanh quarter (gates epilogue)
};

template <int CTAS>
struct GemmShape {
  static constexpr uint32_t kBRows = 256 / CTAS;                    // B rows per CTA and stage
  static constexpr uint32_t kStageBytes = kABytes + kBRows * kBK * 2;
  static constexpr int kStages = CTAS == 1 ? 4 : 6;
  static constexpr size_t kSmem = (size_t)kStages * kStageBytes + 1024 + 256;
  // instruction descriptor: A/B BF16, D F32, K-major both, N = 256, M = 128 * CTAS
  static constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) |
                                     ((uint32_t)((128 * CTAS) >> 4) << 24);
};

template <int CTAS>
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                         uint32_t mbar) {
  if (CTAS == 1) tma_load_2d(dst, map, c0, c1, mbar);
  else tma_load_2d_pair(dst, map, c0, c1, mbar);
}

template <int CTAS>
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  if (CTAS == 1)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
  else
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar), "h"((uint16_t)3)
        : "memory");
}

// LSTM cell of this thread's row for 8 hidden units: r = gates i, f, g, o (8
// TMEM columns each), cp = c_prev (8 floats) -> c_next, h_next.
__device__ __forceinline__ void cell_epilogue8(const uint32_t *r, const uint32_t (&cp)[8], float *c_next,
                                               uint16_t *h_next, size_t cbase, const LaneLut &L) {
  uint32_t cn[8], h[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {                                     // units 2k, 2k + 1
    const uint32_t gi = pack_bf16x2(__uint_as_float(r[2 * k + 1]), __uint_as_float(r[2 * k]));
    const uint32_t gf = pack_bf16x2(__uint_as_float(r[8 + 2 * k + 1]), __uint_as_float(r[8 + 2 * k]));
    const uint32_t gg = pack_bf16x2(__uint_as_float(r[16 + 2 * k + 1]), __uint_as_float(r[16 + 2 * k]));
    const uint32_t go = pack_bf16x2(__uint_as_float(r[24 + 2 * k + 1]), __uint_as_float(r[24 + 2 * k]));
    float2 cnv;
    h[k] = lstm_cell2(gi, gf, gg, go, make_float2(__uint_as_float(cp[2 * k]), __uint_as_float(cp[2 * k + 1])),
                      cnv, L);
    cn[2 * k] = __float_as_uint(cnv.x);
    cn[2 * k + 1] = __float_as_uint(cnv.y);
  }
  st256(c_next + cbase, cn, true);
  asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(h_next + cbase), "r"(h[0]),
               "r"(h[1]), "r"(h[2]), "r"(h[3])
               : "memory");
}

template <int EPI, int CTAS>
__global__ void __launch_bounds__(gemm_threads<EPI>(), 1)
k_gemm_t(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
         const GemmArgs g, const __grid_constant__ LutWords lut) {
  using Sh = GemmShape<CTAS>;
  constexpr bool kCell = EPI == kEpiCell;
  constexpr int S = Sh::kStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bar = base + S * Sh::kStageBytes;
  const uint32_t full_bar = bar, empty_bar = bar + 8 * S;
  const uint32_t tfull_bar = bar + 16 * S, tempty_bar = tfull_bar + 16;
  const uint32_t tmem_slot = tempty_bar + 16;
  uint32_t *tmem_slot_ptr = reinterpret_cast<uint32_t *>(smem_raw + (tmem_slot - raw));

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CTAS == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const uint32_t cid = blockIdx.x / CTAS, ncl = gridDim.x / CTAS;
  const uint32_t mt = g.M / (128 * CTAS), ntn = kCell ? g.H / 64 : g.N / 256, ntiles = mt * ntn;
  const uint32_t nk = g.K / kBK;

  if (threadIdx.x == 32) {
    for (int s = 0; s < S; ++s) {
      mbar_init(full_bar + 8 * s, 1);
      mbar_init(empty_bar + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar + 8 * a, 1);
      mbar_init(tempty_bar + 8 * a, CTAS * epi_warps<EPI>());
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    if (CTAS == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                   "n"(2 * kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                   "n"(2 * kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CTAS == 2) cluster_sync_all();   // both CTAs' barriers initialised before any remote use
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (every CTA) ----------------
    uint32_t it = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % S;
        if (it >= (uint32_t)S) mbar_wait(empty_bar + 8 * s, ((it / S) + 1) & 1);
        const uint32_t sa = base + s * Sh::kStageBytes, sb = sa + kABytes;
        const uint32_t fb = CTAS == 1 ? full_bar + 8 * s : map_to_rank0(full_bar + 8 * s);
        if (leader) mbar_expect_tx(full_bar + 8 * s, CTAS * Sh::kStageBytes);
        const int kc = (int)(kb * kBK);
        tma_load<CTAS>(sa, &map_a, kc, (int)(mb * 128 * CTAS + rank * 128), fb);
        if (kCell) {
#pragma unroll
          for (uint32_t j = 0; j < 4 / CTAS; ++j)                   // gates of this CTA
            tma_load<CTAS>(sb + j * (64 * kBK * 2), &map_b, kc,
                           (int)((rank * (4 / CTAS) + j) * g.H + nb * 64), fb);
        } else {
          tma_load<CTAS>(sb, &map_b, kc, (int)(nb * 256 + rank * Sh::kBRows), fb);
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (the leader) ----------------
    uint32_t it = 0, i = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl, ++i) {
      const uint32_t a = i & 1;
      if (i >= 2) mbar_wait(tempty_bar + 8 * a, ((i / 2) + 1) & 1);   // epilogue drained stage a
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + a * kTmemCols;
      for (uint32_t kb = 0; kb < nk; ++kb, ++it) {
        const uint32_t s = it % S;
        mbar_wait(full_bar + 8 * s, (it / S) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint64_t da = umma_sdesc(base + s * Sh::kStageBytes);
        const uint64_t db = umma_sdesc(base + s * Sh::kStageBytes + kABytes);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          const uint32_t acc = (kb | k) != 0;
          if (CTAS == 1)
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(Sh::kIdesc), "r"(acc));
          else
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(da + (uint64_t)(2 * k)), "l"(db + (uint64_t)(2 * k)), "r"(Sh::kIdesc), "r"(acc));
        }
        umma_commit<CTAS>(empty_bar + 8 * s);
      }
      umma_commit<CTAS>(tfull_bar + 8 * a);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (8 warps, every CTA) ----------------
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    const uint32_t tempty_leader = CTAS == 1 ? tempty_bar : map_to_rank0(tempty_bar);
    const uint32_t lw = lut.bf16[lane];
    const LaneLut L{lut.bf16[lane], lut.f32K[lane], lut.f32C[lane]};
    auto release = [&](uint32_t a) {   // this warp's TMEM reads of stage a are complete
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (leader)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_bar + 8 * a) : "memory");
        else   // relaxed: see the header comment
          asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           tempty_leader + 8 * a)
                       : "memory");
      }
    };
    uint32_t i = 0;
    for (uint32_t t = cid; t < ntiles; t += ncl, ++i) {
      uint32_t mb, nb;
      tile_coords(t, mt, ntn, mb, nb);
      const uint32_t a = i & 1;
      const uint32_t row = mb * 128 * CTAS + rank * 128 + 32 * q + lane;
      if (kCell) {
        constexpr int kParts = epi_warps<EPI>() / 4, kUnits = 64 / kParts, kRounds = kUnits / 8;
        const uint32_t part = (warp - 2) >> 2;                      // kUnits hidden units of the tile
        const size_t cbase = (size_t)row * g.H + nb * 64 + part * kUnits;
        // c_prev, before the wait.  Non-coherent loads are safe even when
        // c_next == c_prev: the only write to these elements is this
        // thread's own c' store, issued after this read; other threads may
        // write other elements of the same lines, which this read never uses.
        uint32_t cp[kRounds][8];
#pragma unroll
        for (int v = 0; v < kRounds; ++v) ld256<true>(g.c_prev + cbase + 8 * v, cp[v], true);
        mbar_wait(tfull_bar + 8 * a, (i / 2) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tbase = tmem + ((32 * q) << 16) + a * kTmemCols + part * kUnits;
#pragma unroll
        for (int rd = 0; rd < kRounds; ++rd) {
          uint32_t r[32];                                           // i, f, g, o x 8 units
#pragma unroll
          for (int gq = 0; gq < 4; ++gq) tmem_ld8(tbase + 64 * gq + 8 * rd, r + 8 * gq);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (rd == kRounds - 1) release(a);
          cell_epilogue8(r, cp[rd], g.c_next, g.h_next, cbase + 8 * rd, L);
        }
        continue;
      }
      mbar_wait(tfull_bar + 8 * a, (i / 2) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint16_t *crow = g.C + (size_t)row * g.N + nb * 256 + half * 128;
      const bool tanh_tile = EPI == kEpiLstm && (nb * 256) / g.H == g.tq;
      const uint32_t tbase = tmem + ((32 * q) << 16) + a * kTmemCols + half * 128;
      if (CTAS == 2) {
        // all 128 columns in flight at once, stage released before the activation
        uint32_t r[128];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) tmem_ld32(tbase + 32 * c4, r + 32 * c4);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        release(a);
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          uint32_t o0[8], o1[8];
          epi_tile_chunk<EPI>(r + 32 * c4, o0, o1, lw, tanh_tile);
          st256(crow + 32 * c4, o0, true);
          st256(crow + 32 * c4 + 16, o1, true);
        }
      } else {
        // 32 columns at a time (measured faster for the 1-CTA kernel)
#pragma unroll 1
        for (uint32_t c = 0; c < 128; c += 32) {
          uint32_t r[32];
          tmem_ld32(tbase + c, r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c == 96) release(a);
          uint32_t o0[8], o1[8];
          epi_tile_chunk<EPI>(r, o0, o1, lw, tanh_tile);
          st256(crow + c, o0, true);
          st256(crow + c + 16, o1, true);
        }
      }
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CTAS == 2) cluster_sync_all();   // both CTAs done with TMEM and each other's barriers
  else __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CTAS == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "n"(2 * kTmemCols));
    else
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

template <int EPI, int CTAS>
static cudaError_t launch_t(const CUtensorMap &ma, const CUtensorMap &mb, const GemmArgs &g,
                            const LutWords &lut, cudaStream_t s, int sms) {
  using Sh = GemmShape<CTAS>;
  // The dynamic-smem limit is a per-device (per-context) function attribute:
  // set it once per device, not once per process, so the first call on a
  // second GPU does not launch with the 48 KB default.  Two threads racing on
  // a fresh device both set the same value (idempotent).
  constexpr int kMaxDevGemm = 64;
  static int attr_done[kMaxDevGemm];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevGemm) return cudaErrorInvalidDevice;
  if (!__atomic_load_n(&attr_done[dev], __ATOMIC_ACQUIRE)) {
    e = cudaFuncSetAttribute(k_gemm_t<EPI, CTAS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Sh::kSmem);
    if (e != cudaSuccess) return e;
    __atomic_store_n(&attr_done[dev], 1, __ATOMIC_RELEASE);
  }
  const size_t tiles = (g.M / (128 * CTAS)) * (EPI == kEpiCell ? g.H / 64 : g.N / 256);
  const size_t units = (size_t)(sms / CTAS);
  const unsigned grid = (unsigned)(CTAS * (tiles < units ? tiles : units));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(gemm_threads<EPI>());
  cfg.dynamicSmemBytes = Sh::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CTAS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CTAS == 2 ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, k_gemm_t<EPI, CTAS>, ma, mb, g, lut);
  count_launch();
  return e;
}

template <int CTAS>
static cudaError_t dispatch(int epi, const CUtensorMap &ma, const CUtensorMap &mb, const GemmArgs &g,
                            const LutWords &lut, cudaStream_t s, int sms) {
  switch (epi) {
    case -1: return launch_t<-1, CTAS>(ma, mb, g, lut, s, sms);
    case OP_TANH: return launch_t<OP_TANH, CTAS>(ma, mb, g, lut, s, sms);
    case OP_SIGMOID: return launch_t<OP_SIGMOID, CTAS>(ma, mb, g, lut, s, sms);
    case OP_SWISH: return launch_t<OP_SWISH, CTAS>(ma, mb, g, lut, s, sms);
    case OP_GELU: return launch_t<OP_GELU, CTAS>(ma, mb, g, lut, s, sms);
    case kEpiLstm: return launch_t<kEpiLstm, CTAS>(ma, mb, g, lut, s, sms);
    case kEpiCell: return launch_t<kEpiCell, CTAS>(ma, mb, g, lut, s, sms);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t run(int epi, const uint16_t *A, const uint16_t *B, const GemmArgs &g,
                       const LutWords &lut, cudaStream_t s, int sms) {
  const bool cell = epi == kEpiCell;
  const bool pair = use_pair(g.M, g.N, g.K, epi) && sms >= 2;
  CUtensorMap ma, mb;
  const uint32_t b_rows = cell ? 64 : (pair ? 128 : 256);
  if (!make_map(&ma, A, g.M, g.K, 128) || !make_map(&mb, B, g.N, g.K, b_rows))
    return cudaErrorInvalidValue;
  return pair ? dispatch<2>(epi, ma, mb, g, lut, s, sms) : dispatch<1>(epi, ma, mb, g, lut, s, sms);
}

cudaError_t launch_gemm(int epi, const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M,
                        size_t N, size_t K, const LutWords &lut, cudaStream_t s, int sms,
                        uint32_t lstm_hidden, uint32_t lstm_tq) {
  GemmArgs g = {};
  g.C = C;
  g.M = (uint32_t)M;
  g.N = (uint32_t)N;
  g.K = (uint32_t)K;
  g.H = lstm_hidden ? lstm_hidden : 1u;
  g.tq = lstm_tq;
  return run(epi, A, B, g, lut, s, sms);
}

cudaError_t launch_gemm_cell(const uint16_t *A, const uint16_t *B, const float *c_prev, float *c_next,
                             uint16_t *h_next, size_t M, size_t H, size_t K, const LutWords &lut,
                             cudaStream_t s, int sms) {
  GemmArgs g = {};
  g.c_prev = c_prev;
  g.c_next = c_next;
  g.h_next = h_next;
  g.M = (uint32_t)M;
  g.N = (uint32_t)(4 * H);
  g.K = (uint32_t)K;
  g.H = (uint32_t)H;
  return run(kEpiCell, A, B, g, lut, s, sms);
}

}  // namespace kt
