// zcbench.cu -- dev tool: SM-initiated PCIe streaming (zero-copy) on mapped
// pinned host memory.  Copy kernel host->host through the SMs (read x over
// PCIe, write y over PCIe), persistent grid-stride, for several grid sizes
// and vector widths; plus read-only and write-only variants and the
// copy-engine reference (cudaMemcpyAsync H2D || D2H on two streams).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/zcbench tools/zcbench.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>  // 0 copy, 1 read only, 2 write only
__global__ void k_stream(const uint4 *__restrict__ x, uint4 *__restrict__ y, size_t nv, int per) {
  // each warp owns runs of `per` consecutive 512-B warp-vectors
  const size_t lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  uint32_t acc = 0;
  for (size_t base = warp * per * 32; base < nv; base += nw * per * 32) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u < per) {
        const size_t i = base + u * 32 + lane;
        if (MODE != 2 && i < nv) v[u] = x[i];
        else v[u] = make_uint4(u, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u < per) {
        const size_t i = base + u * 32 + lane;
        if (MODE == 1) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
        else if (i < nv) y[i] = v[u];
      }
    }
  }
  if (MODE == 1 && acc == 0x12345678u) y[0] = make_uint4(acc, 0, 0, 0);
}

int main() {
  const size_t bytes = 64ull << 20;
  void *hx, *hy;
  CK(cudaHostAlloc(&hx, bytes, cudaHostAllocMapped));
  CK(cudaHostAlloc(&hy, bytes, cudaHostAllocMapped));
  memset(hx, 1, bytes);
  memset(hy, 0, bytes);
  void *dx, *dy;
  CK(cudaHostGetDevicePointer(&dx, hx, 0));
  CK(cudaHostGetDevicePointer(&dy, hy, 0));
  void *gx, *gy;
  CK(cudaMalloc(&gx, bytes));
  CK(cudaMalloc(&gy, bytes));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const size_t nv = bytes / 16;
  const int reps = 10;
  for (int mode = 0; mode < 3; ++mode) {
    for (int per : {1, 4, 8}) {
      for (int bps : {1, 2, 4, 8}) {
        for (int thr : {128, 512}) {
          const int grid = sms * bps;
          auto run = [&]() {
            if (mode == 0) k_stream<0><<<grid, thr>>>((const uint4 *)dx, (uint4 *)dy, nv, per);
            if (mode == 1) k_stream<1><<<grid, thr>>>((const uint4 *)dx, (uint4 *)dy, nv, per);
            if (mode == 2) k_stream<2><<<grid, thr>>>((const uint4 *)dx, (uint4 *)dy, nv, per);
          };
          run();
          CK(cudaDeviceSynchronize());
          cudaEventRecord(a);
          for (int r = 0; r < reps; ++r) run();
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          ms /= reps;
          const double moved = (mode == 0 ? 2.0 : 1.0) * bytes;
          printf("mode=%s per=%d grid=%4d thr=%3d inflight/warp=%5d B: %.3f ms  %.1f GB/s\n",
                 mode == 0 ? "copy " : mode == 1 ? "read " : "write", per, grid, thr, per * 512, ms,
                 moved / ms / 1e6);
        }
      }
    }
  }
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) {
    cudaMemcpyAsync(gx, hx, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(hy, gy, bytes, cudaMemcpyDeviceToHost, s2);
  }
  cudaStreamSynchronize(s1);
  cudaStreamSynchronize(s2);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  printf("copy engines H2D || D2H: %.3f ms  %.1f GB/s\n", ms, 2.0 * bytes / ms / 1e6);
  return 0;
}
