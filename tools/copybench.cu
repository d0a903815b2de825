// tools/copybench.cu -- DRAM access-pattern sweep with plain copies (dev tool).
// Which grid / bytes-in-flight / ordering gets the most out of HBM for a
// read-once write-once stream?  Reference: cudaMemcpyAsync D2D.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

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

// grid-stride over warp chunks (lockstep sweep)
template <int U, int T>
__global__ void __launch_bounds__(T) c_stride(const uint8_t *x, uint8_t *y, uint64_t nvec) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nch = (nvec + 32 * U - 1) / (32 * U);
  for (uint64_t c = (uint64_t)blockIdx.x * (T / 32) + (threadIdx.x >> 5); c < nch;
       c += (uint64_t)gridDim.x * (T / 32)) {
    uint32_t v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = c * 32 * U + u * 32 + lane;
      ld256<true>(x + i * 32, v[u], i < nvec);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = c * 32 * U + u * 32 + lane;
      st256(y + i * 32, v[u], i < nvec);
    }
  }
}

// each warp owns a contiguous range of chunks
template <int U, int T>
__global__ void __launch_bounds__(T) c_range(const uint8_t *x, uint8_t *y, uint64_t nvec) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nch = (nvec + 32 * U - 1) / (32 * U);
  const uint64_t nw = (uint64_t)gridDim.x * (T / 32);
  const uint64_t w = (uint64_t)blockIdx.x * (T / 32) + (threadIdx.x >> 5);
  const uint64_t per = (nch + nw - 1) / nw;
  const uint64_t c0 = w * per, c1 = c0 + per < nch ? c0 + per : nch;
  for (uint64_t c = c0; c < c1; ++c) {
    uint32_t v[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = c * 32 * U + u * 32 + lane;
      ld256<true>(x + i * 32, v[u], i < nvec);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = c * 32 * U + u * 32 + lane;
      st256(y + i * 32, v[u], i < nvec);
    }
  }
}

// one chunk per warp, big grid (hardware block scheduler balances)
template <int U, int T>
__global__ void __launch_bounds__(T) c_flat(const uint8_t *x, uint8_t *y, uint64_t nvec) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t c = (uint64_t)blockIdx.x * (T / 32) + (threadIdx.x >> 5);
  uint32_t v[U][8];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = c * 32 * U + u * 32 + lane;
    ld256<true>(x + i * 32, v[u], i < nvec);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t i = c * 32 * U + u * 32 + lane;
    st256(y + i * 32, v[u], i < nvec);
  }
}

// 16-byte accesses, grid-stride, U vectors per lane
template <int U, int T>
__global__ void __launch_bounds__(T) c_stride16(const uint4 *x, uint4 *y, uint64_t n16) {
  const uint64_t tid = (uint64_t)blockIdx.x * T + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * T;
  for (uint64_t b = tid; b < n16; b += nt * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + u * nt;
      if (i < n16) v[u] = __ldcs(x + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = b + u * nt;
      if (i < n16) __stcs(y + i, v[u]);
    }
  }
}

typedef void (*KFn)(const uint8_t *, uint8_t *, uint64_t);

int main() {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = (size_t)2 << 30;  // 2 GiB in + 2 GiB out
  uint8_t *x, *y;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMalloc(&y, bytes));
  CK(cudaMemset(x, 1, bytes));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto timeit = [&](auto launch, const char *name) {
    launch();
    CK(cudaStreamSynchronize(st));
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
      CK(cudaEventRecord(e0, st));
      for (int r = 0; r < 5; ++r) launch();
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (ms < best) best = ms;
    }
    printf("%-40s %9.1f GB/s\n", name, 2.0 * bytes * 5 / (best / 1e3) / 1e9);
    fflush(stdout);
  };
  timeit([&] { CK(cudaMemcpyAsync(y, x, bytes, cudaMemcpyDeviceToDevice, st)); }, "cudaMemcpyAsync D2D");
  const uint64_t nvec = bytes / 32;
  struct V {
    const char *name;
    KFn f;
    int T, U, kind;
  } vs[] = {
      {"stride U1 T256", c_stride<1, 256>, 256, 1, 0}, {"stride U2 T256", c_stride<2, 256>, 256, 2, 0},
      {"stride U4 T256", c_stride<4, 256>, 256, 4, 0}, {"stride U2 T128", c_stride<2, 128>, 128, 2, 0},
      {"stride U2 T512", c_stride<2, 512>, 512, 2, 0}, {"range U1 T256", c_range<1, 256>, 256, 1, 0},
      {"range U2 T256", c_range<2, 256>, 256, 2, 0},   {"range U4 T128", c_range<4, 128>, 128, 4, 0},
      {"flat U1 T256", c_flat<1, 256>, 256, 1, 1},     {"flat U2 T256", c_flat<2, 256>, 256, 2, 1},
      {"flat U4 T256", c_flat<4, 256>, 256, 4, 1},     {"flat U1 T128", c_flat<1, 128>, 128, 1, 1},
      {"flat U2 T512", c_flat<2, 512>, 512, 2, 1},
  };
  for (auto &v : vs) {
    int bps;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, (const void *)v.f, v.T, 0));
    const uint64_t nch = (nvec + 32 * v.U - 1) / (32 * v.U);
    if (v.kind == 1) {
      const unsigned grid = (unsigned)((nch + v.T / 32 - 1) / (v.T / 32));
      timeit([&] { v.f<<<grid, v.T, 0, st>>>(x, y, nvec); }, v.name);
    } else {
      for (int k : {1, 2, 4, bps}) {
        if (k > bps) continue;
        char nm[96];
        snprintf(nm, sizeof nm, "%s x%d/SM", v.name, k);
        const unsigned grid = sms * k;
        timeit([&] { v.f<<<grid, v.T, 0, st>>>(x, y, nvec); }, nm);
      }
    }
  }
  const uint64_t n16 = bytes / 16;
  for (int k : {2, 4, 8}) {
    char nm[96];
    snprintf(nm, sizeof nm, "stride16 cs U4 T256 x%d/SM", k);
    const unsigned grid = sms * k;
    timeit([&] { c_stride16<4, 256><<<grid, 256, 0, st>>>((const uint4 *)x, (uint4 *)y, n16); }, nm);
    snprintf(nm, sizeof nm, "stride16 cs U1 T256 x%d/SM", k);
    timeit([&] { c_stride16<1, 256><<<grid, 256, 0, st>>>((const uint4 *)x, (uint4 *)y, n16); }, nm);
  }
  return 0;
}
