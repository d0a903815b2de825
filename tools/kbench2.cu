// tools/kbench2.cu -- second variant sweep (dev tool, not part of the library).
// Register-streaming kernels (LDG/STG.256) with v1/v2 cores, CTA size,
// min-blocks and software prefetch, and a TMA-bulk (cp.async.bulk + mbarrier)
// smem-staged variant.  Big case: 2^30 BF16 (4 GiB of traffic); small case:
// 2^24 BF16 over 8 rotating sets, 64 launches replayed from a CUDA graph.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kt_device.cuh"

using namespace kt;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

// ---- v1 core (round-1 first version), kept here for comparison ------------
__device__ __forceinline__ uint32_t shr_wrap_(uint32_t a, uint32_t n) {
  uint32_t d;
  asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(0u), "r"(n));
  return d;
}
__device__ __forceinline__ uint32_t core_v1(uint32_t x, uint32_t lw) {
  const uint32_t mag = x & kMagx2;
  const uint32_t Ll = shfl_lut(lw, x >> 4);
  const uint32_t Lh = shfl_lut(lw, x >> 20);
  const uint32_t Kl = shr_wrap_(0x10000u, Ll);
  const uint32_t Kh = shr_wrap_(0x10000u, Lh);
  const uint32_t dl = (mag & 0xffffu) * Kl + Ll;
  const uint32_t dh = (mag >> 16) * Kh + Lh;
  const uint32_t ymag = __byte_perm(dl, dh, 0x7632);
  const uint32_t byp = hset2_ltu(mag, kT1x2);
  const uint32_t sat = hset2_gt(mag, kT2x2);
  const uint32_t m2 = bsel(sat, kOnex2, ymag);
  const uint32_t m3 = bsel(byp, mag, m2);
  return (x & kSignx2) | m3;
}

// v3: v1 with K from a second shuffled table (no SHF.R.W), LUT word for the
// addend as in v1: Ll = (C << 16) | r; lk = 2^(16 - r)
__device__ __forceinline__ uint32_t core_v3(uint32_t x, uint32_t lw, uint32_t lk) {
  const uint32_t mag = x & kMagx2;
  const uint32_t il = x >> 4, ih = x >> 20;
  const uint32_t Ll = shfl_lut(lw, il), Lh = shfl_lut(lw, ih);
  const uint32_t Kl = shfl_lut(lk, il), Kh = shfl_lut(lk, ih);
  const uint32_t dl = (mag & 0xffffu) * Kl + Ll;
  const uint32_t dh = (mag >> 16) * Kh + Lh;
  const uint32_t ymag = __byte_perm(dl, dh, 0x7632);
  const uint32_t byp = hset2_ltu(mag, kT1x2);
  const uint32_t sat = hset2_gt(mag, kT2x2);
  const uint32_t m = bsel(sat, kOnex2, ymag);
  const uint32_t o = bsel(byp, x, m);
  return o | (x & kSignx2);
}
// v4: v1 with the 3-select tail of v2 and mag_hi via IMAD.HI-free SHF
__device__ __forceinline__ uint32_t core_v4(uint32_t x, uint32_t lw) {
  const uint32_t mag = x & kMagx2;
  const uint32_t Ll = shfl_lut(lw, x >> 4);
  const uint32_t Lh = shfl_lut(lw, x >> 20);
  const uint32_t Kl = shr_wrap_(0x10000u, Ll);
  const uint32_t Kh = shr_wrap_(0x10000u, Lh);
  const uint32_t dl = (mag & 0xffffu) * Kl + Ll;
  const uint32_t dh = (mag >> 16) * Kh + Lh;
  const uint32_t ymag = __byte_perm(dl, dh, 0x7632);
  const uint32_t byp = hset2_ltu(mag, kT1x2);
  const uint32_t sat = hset2_gt(mag, kT2x2);
  const uint32_t m = bsel(sat, kOnex2, ymag);
  const uint32_t o = bsel(byp, x, m);
  return o | (x & kSignx2);
}
// v5: v4 with lane extraction for the hi element via IMAD.HI (FMA pipe)
__device__ __forceinline__ uint32_t core_v5(uint32_t x, uint32_t lw) {
  const uint32_t mag = x & kMagx2;
  const uint32_t Ll = shfl_lut(lw, x >> 4);
  const uint32_t Lh = shfl_lut(lw, mulhi(x, 1u << 12));
  const uint32_t Kl = shr_wrap_(0x10000u, Ll);
  const uint32_t Kh = shr_wrap_(0x10000u, Lh);
  const uint32_t dl = (mag & 0xffffu) * Kl + Ll;
  const uint32_t dh = (mag >> 16) * Kh + Lh;
  const uint32_t ymag = __byte_perm(dl, dh, 0x7632);
  const uint32_t byp = hset2_ltu(mag, kT1x2);
  const uint32_t sat = hset2_gt(mag, kT2x2);
  const uint32_t m = bsel(sat, kOnex2, ymag);
  const uint32_t o = bsel(byp, x, m);
  return o | (x & kSignx2);
}

template <int OP>
__device__ __forceinline__ uint32_t opw(uint32_t w, uint32_t lw) {
  if (OP == 0) return ktanh_bf16x2(w, lw);
  if (OP == 1) return ksigmoid_bf16x2(w, lw);
  if (OP == 2) return kswish_bf16x2(w, lw);
  if (OP == 3) return kgelu_bf16x2(w, lw);
  if (OP == 10) return core_v1(w, lw);
  if (OP == 11) return core_v3(w, lw, lw >> 3);
  if (OP == 12) return core_v4(w, lw);
  if (OP == 13) return core_v5(w, lw);
  return w;  // copy
}

// ---- register streaming kernel --------------------------------------------
template <int OP, int U, int T, int MINB, int PF>
__global__ void __launch_bounds__(T, MINB)
kreg(const uint8_t *x, uint8_t *y, uint64_t nvec, uint64_t nchunks, const __grid_constant__ LutWords lut) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lw = lut.bf16[lane];
  const uint64_t warp0 = (uint64_t)blockIdx.x * (T / 32) + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * (T / 32);
  if (PF == 0) {
    for (uint64_t c = warp0; c < nchunks; c += nwarps) {
      const uint64_t base = c * (32 * U) + lane;
      uint32_t v[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = base + (uint64_t)u * 32;
        ld256<true>(x + i * 32, v[u], i < nvec);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[u][j] = opw<OP>(v[u][j], lw);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = base + (uint64_t)u * 32;
        st256(y + i * 32, v[u], i < nvec);
      }
    }
  } else {
    uint32_t nx[U][8];
    uint64_t c = warp0;
    if (c < nchunks) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = c * (32 * U) + lane + (uint64_t)u * 32;
        ld256<true>(x + i * 32, nx[u], i < nvec);
      }
    }
    for (; c < nchunks; c += nwarps) {
      uint32_t v[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[u][j] = nx[u][j];
      const uint64_t cn = c + nwarps;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = cn * (32 * U) + lane + (uint64_t)u * 32;
        ld256<true>(x + i * 32, nx[u], cn < nchunks && i < nvec);
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[u][j] = opw<OP>(v[u][j], lw);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = c * (32 * U) + lane + (uint64_t)u * 32;
        st256(y + i * 32, v[u], i < nvec);
      }
    }
  }
}

// ---- flat (non-persistent) kernel: each warp does CPW consecutive chunks ----
template <int OP, int U, int T, int CPW>
__global__ void __launch_bounds__(T)
kflat(const uint8_t *x, uint8_t *y, uint64_t nvec, uint64_t nchunks, const __grid_constant__ LutWords lut) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lw = lut.bf16[lane];
  const uint64_t w = (uint64_t)blockIdx.x * (T / 32) + (threadIdx.x >> 5);
#pragma unroll 1
  for (int k = 0; k < CPW; ++k) {
    const uint64_t c = w * CPW + k;
    if (c >= nchunks) break;
    const uint64_t base = c * (32 * U) + lane;
    uint32_t v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * 32;
      ld256<true>(x + i * 32, v[u], i < nvec);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int j = 0; j < 8; ++j) v[u][j] = opw<OP>(v[u][j], lw);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * 32;
      st256(y + i * 32, v[u], i < nvec);
    }
  }
}

// ---- TMA bulk kernel ------------------------------------------------------
__device__ __forceinline__ uint32_t saddr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t ph) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(a), "r"(ph) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int OP, int TILE, int ST, int T, int MINB>
__global__ void __launch_bounds__(T, MINB)
ktma(const uint8_t *x, uint8_t *y, uint64_t ntiles, const __grid_constant__ LutWords lut) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[ST];
  const uint32_t lw = lut.bf16[threadIdx.x & 31];
  const uint32_t sbase = saddr(sm);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(saddr(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t G = gridDim.x;
  const uint64_t t0 = blockIdx.x;
  // prologue: fill all stages
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      const uint64_t tile = t0 + (uint64_t)s * G;
      if (tile < ntiles) {
        mbar_expect_tx(saddr(&full[s]), TILE);
        bulk_load(sbase + s * TILE, x + tile * TILE, TILE, saddr(&full[s]));
      }
    }
  }
  uint32_t k = 0;
  for (uint64_t tile = t0; tile < ntiles; tile += G, ++k) {
    const uint32_t s = k % ST;
    const uint32_t ph = (k / ST) & 1;
    while (!mbar_try(saddr(&full[s]), ph)) {
    }
    uint4 *p = reinterpret_cast<uint4 *>(sm + s * TILE);
#pragma unroll
    for (int j = 0; j < TILE / 16 / T; ++j) {
      uint4 v = p[j * T + threadIdx.x];
      v.x = opw<OP>(v.x, lw);
      v.y = opw<OP>(v.y, lw);
      v.z = opw<OP>(v.z, lw);
      v.w = opw<OP>(v.w, lw);
      p[j * T + threadIdx.x] = v;
    }
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(const_cast<uint8_t *>(y) + tile * TILE, sbase + s * TILE, TILE);
      bulk_commit();
      // refill the stage used by the previous tile once its store has read smem
      if (k >= 1) {
        bulk_wait_read<1>();
        const uint32_t sp = (k - 1) % ST;
        const uint64_t nt = tile - G + (uint64_t)ST * G;
        if (nt < ntiles) {
          mbar_expect_tx(saddr(&full[sp]), TILE);
          bulk_load(sbase + sp * TILE, x + nt * TILE, TILE, saddr(&full[sp]));
        }
      }
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

struct Variant {
  const char *name;
  const void *fn;
  int threads, unroll, tma, tile, smem, cpw;
};

#define VR(OP, U, T, MINB, PF) \
  Variant{"reg op" #OP " U" #U " T" #T " minb" #MINB " pf" #PF, (const void *)kreg<OP, U, T, MINB, PF>, T, U, 0, 0, 0, 0}
#define VT(OP, TILE, ST, T, MINB)                                                                   \
  Variant{"tma op" #OP " tile" #TILE " st" #ST " T" #T " minb" #MINB, (const void *)ktma<OP, TILE, ST, T, MINB>, \
          T, 0, 1, TILE, TILE * ST, 0}
#define VF(OP, U, T, CPW) \
  Variant{"flat op" #OP " U" #U " T" #T " cpw" #CPW, (const void *)kflat<OP, U, T, CPW>, T, U, 0, 0, 0, CPW}

static Variant variants[] = {
    VF(-1, 1, 256, 1), VF(-1, 2, 256, 1), VF(-1, 1, 128, 1), VF(-1, 1, 256, 4),
    VR(0, 2, 64, 1, 0),
    VF(0, 1, 256, 1), VF(0, 2, 256, 1), VF(0, 1, 128, 1), VF(0, 2, 128, 1), VF(0, 1, 64, 1),
    VF(0, 1, 512, 1), VF(0, 1, 256, 2), VF(0, 1, 256, 4), VF(0, 2, 128, 2), VF(0, 4, 128, 1),
    VF(10, 1, 256, 1), VF(10, 2, 128, 1),
    VF(3, 1, 256, 1), VF(3, 1, 128, 1), VF(3, 2, 128, 1), VF(3, 1, 256, 2),
    VF(2, 1, 256, 1), VF(2, 1, 128, 1), VF(1, 1, 256, 1), VF(1, 1, 128, 1),
};

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t big = (size_t)1 << 30, small = (size_t)1 << 24;
  const int sets = 8;
  uint8_t *xb, *yb;
  CK(cudaMalloc(&xb, big * 2));
  CK(cudaMalloc(&yb, big * 2));
  {
    std::vector<uint16_t> h(1 << 20);
    uint32_t s = 12345;
    for (auto &w : h) {
      s = s * 1664525u + 1013904223u;
      w = (uint16_t)(0x3C00 + (s >> 16) % 0x0500) | (uint16_t)((s & 1) << 15);
    }
    for (size_t off = 0; off < big * 2; off += h.size() * 2)
      CK(cudaMemcpy(xb + off, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  }
  LutWords lut;
  memset(&lut, 0, sizeof(lut));
  for (int t = 0; t < 32; ++t) lut.bf16[t] = (1u << (15 - (t & 7))) << 16 | (uint32_t)(t * 37);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  printf("%-44s %10s %10s %10s %6s %6s %6s\n", "variant", "big GB/s", "small GB/s", "L2res GB/s", "regs", "blk/SM", "grid");
  for (const Variant &v : variants) {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, v.fn));
    if (v.smem > 48 * 1024) CK(cudaFuncSetAttribute(v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, v.smem));
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, v.fn, v.threads, v.smem));
    if (bps == 0) {
      printf("%-44s (does not fit)\n", v.name);
      continue;
    }
    double gbs[3];
    unsigned grid_big = 0;
    for (int which = 0; which < 3; ++which) {
      const size_t n = which == 0 ? big : small;
      const int nsets = which == 1 ? sets : 1;
      unsigned grid;
      uint64_t a1, a2;
      if (v.tma) {
        a1 = n * 2 / v.tile;
        a2 = 0;
        grid = (unsigned)std::min<uint64_t>((uint64_t)sms * bps, a1);
      } else if (v.cpw) {
        uint64_t nvec = n / 16;
        uint64_t nchunks = (nvec + 32 * v.unroll - 1) / (32 * v.unroll);
        uint64_t warps = (nchunks + v.cpw - 1) / v.cpw;
        grid = (unsigned)((warps + v.threads / 32 - 1) / (v.threads / 32));
        a1 = nvec;
        a2 = nchunks;
      } else {
        uint64_t nvec = n / 16;
        uint64_t nchunks = (nvec + 32 * v.unroll - 1) / (32 * v.unroll);
        uint64_t maxw = (uint64_t)sms * bps * (v.threads / 32);
        uint64_t iters = (nchunks + maxw - 1) / maxw;
        uint64_t warps = (nchunks + iters - 1) / iters;
        grid = (unsigned)((warps + v.threads / 32 - 1) / (v.threads / 32));
        a1 = nvec;
        a2 = nchunks;
      }
      if (which == 0) grid_big = grid;
      const int reps = which == 0 ? 10 : 64;
      cudaGraph_t g;
      cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
      for (int r = 0; r < reps; ++r) {
        const size_t off = (size_t)(r % nsets) * n * 2;
        const uint8_t *xp = xb + off;
        uint8_t *yp = yb + off;
        if (v.tma) {
          void *args[] = {(void *)&xp, (void *)&yp, (void *)&a1, (void *)&lut};
          CK(cudaLaunchKernel(v.fn, dim3(grid), dim3(v.threads), args, v.smem, st));
        } else {
          void *args[] = {(void *)&xp, (void *)&yp, (void *)&a1, (void *)&a2, (void *)&lut};
          CK(cudaLaunchKernel(v.fn, dim3(grid), dim3(v.threads), args, 0, st));
        }
      }
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, st));
      CK(cudaStreamSynchronize(st));
      float best = 1e30f;
      for (int trial = 0; trial < 5; ++trial) {
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      CK(cudaGraphExecDestroy(ge));
      CK(cudaGraphDestroy(g));
      gbs[which] = (double)n * 4 * reps / (best / 1e3) / 1e9;
    }
    printf("%-44s %10.1f %10.1f %10.1f %6d %6d %6u\n", v.name, gbs[0], gbs[1], gbs[2], fa.numRegs, bps, grid_big);
    fflush(stdout);
  }
  return 0;
}
