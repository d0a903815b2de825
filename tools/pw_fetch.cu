// pw_fetch.cu -- how should a piecewise-polynomial comparator fetch its
// per-piece coefficients on sm_100a?  Register-resident throughput of a
// degree-3, 16-piece Horner evaluation (the minimax-3 comparator's shape)
// with the 4 coefficients fetched by (a) 4 warp shuffles, (b) one 128-bit
// shared-memory load, (c) four 32-bit shared loads, (d) a uniform
// (warp-constant) piece -- the no-gather lower bound.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pw_fetch tools/pw_fetch.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int V>
__device__ __forceinline__ float eval(float a, const float (&c)[4], const float4 *tab) {
  const float kf = __fmaf_rz(a, 2.0f, 8388608.0f);
  const uint32_t k = __float_as_uint(kf) & 15u;
  const float h = __fmaf_rn(__fsub_rn(kf, 8388608.0f), -0.5f, a);
  float c0, c1, c2, c3;
  if (V == 0) {
    c3 = __shfl_sync(~0u, c[3], k); c2 = __shfl_sync(~0u, c[2], k);
    c1 = __shfl_sync(~0u, c[1], k); c0 = __shfl_sync(~0u, c[0], k);
  } else if (V == 1) {
    const float4 t = tab[k];
    c0 = t.x; c1 = t.y; c2 = t.z; c3 = t.w;
  } else if (V == 2) {
    const float *tf = reinterpret_cast<const float *>(tab);
    c0 = tf[k]; c1 = tf[16 + k]; c2 = tf[32 + k]; c3 = tf[48 + k];
  } else {
    c0 = c[0]; c1 = c[1]; c2 = c[2]; c3 = c[3];
  }
  float y = __fmaf_rn(__fmaf_rn(__fmaf_rn(c3, h, c2), h, c1), h, c0);
  y = fminf(fmaxf(y, 0.0f), 1.0f);
  return a >= 8.0f ? 1.0f : y;
}

template <int V>
__global__ void __launch_bounds__(256) k(const float *in, uint32_t *out, long long *cyc, int iters) {
  __shared__ float4 tab4[16];
  __shared__ float tabs[64];
  const uint32_t lane = threadIdx.x & 31;
  float c[4];
  for (int j = 0; j < 4; ++j) c[j] = 0.1f * (j + 1) + 0.01f * (lane & 15);
  if (threadIdx.x < 16) tab4[threadIdx.x] = make_float4(c[0], c[1], c[2], c[3]);
  if (threadIdx.x < 64) tabs[threadIdx.x] = 0.1f * ((threadIdx.x >> 4) + 1) + 0.01f * (threadIdx.x & 15);
  __syncthreads();
  const float4 *tab = (V == 2) ? reinterpret_cast<const float4 *>(tabs) : tab4;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float v[16];
  for (int j = 0; j < 16; ++j) v[j] = fabsf(in[(t * 16 + j) & 4095]);
  uint32_t acc[16] = {0};
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
    const float off = (float)(it & 3) * 1e-6f;
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] ^= __float_as_uint(eval<V>(v[j] + off, c, tab));
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t a = 0;
  for (int j = 0; j < 16; ++j) a ^= acc[j];
  out[t] = a;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
int run(const char *name, const float *in, uint32_t *out, long long *cyc, int sms) {
  int bps = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k<V>, 256, 0));
  const int iters = 1024;
  double best = 1e300;
  for (int r = 0; r < 3; ++r) {
    k<V><<<sms * bps, 256>>>(in, out, cyc, iters);
    CK(cudaDeviceSynchronize());
    std::vector<long long> h(sms * bps);
    CK(cudaMemcpy(h.data(), cyc, h.size() * 8, cudaMemcpyDeviceToHost));
    const long long mx = *std::max_element(h.begin(), h.end());
    best = std::min(best, (double)mx / ((double)bps * 256 * 16 * iters));
  }
  printf("%-28s bps %d  %.4f cycles/elem/SM  (%.2f elem/clk/SM)\n", name, bps, best, 1 / best);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<float> h(4096);
  uint32_t s = 12345;
  for (auto &x : h) {   // ~N(0, 2^2)-ish: sum of uniforms
    float a = 0;
    for (int i = 0; i < 4; ++i) { s = s * 1664525u + 1013904223u; a += (s >> 8) * (1.0f / 16777216.0f) - 0.5f; }
    x = a * 3.46f;
  }
  float *in; uint32_t *out; long long *cyc;
  CK(cudaMalloc(&in, 4096 * 4));
  CK(cudaMalloc(&out, sms * 16 * 256 * 4));
  CK(cudaMalloc(&cyc, sms * 16 * 8));
  CK(cudaMemcpy(in, h.data(), 4096 * 4, cudaMemcpyHostToDevice));
  run<0>("(a) 4x SHFL.IDX", in, out, cyc, sms);
  run<1>("(b) 1x LDS.128", in, out, cyc, sms);
  run<2>("(c) 4x LDS.32", in, out, cyc, sms);
  run<3>("(d) uniform coefficients", in, out, cyc, sms);
  return 0;
}
