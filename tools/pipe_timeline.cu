// pipe_timeline.cu -- dev tool: the kt_apply_host copy-engine pipeline
// (H2D -> kernel -> D2H on three streams, rotating device buffers) rebuilt
// with a plain copy kernel and CUDA events around every op, for a chosen
// chunk plan, to see where a 2^24-element BF16 step loses time against the
// ~96 GB/s bidirectional PCIe ceiling.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pipe_timeline tools/pipe_timeline.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_copy(const uint4 *x, uint4 *y, size_t nv) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv; i += (size_t)gridDim.x * blockDim.x)
    y[i] = x[i];
}

struct Pipe {
  cudaStream_t st[3], st2[3];
  cudaEvent_t ev_in[6], ev_comp[6], ev_out[6];
};

// lanes: 1 = one stream per engine; 2 = chunks alternate between two
// independent 3-stream pipelines (two DMA ops in flight per direction).
// fuse: the kernel runs on the H2D stream (no H2D -> kernel event hop).
static int g_lanes = 1, g_fuse = 0, g_nbuf = 3;

static void step(Pipe &p, const std::vector<size_t> &plan, char *hx, char *hy, char *work, size_t cmax,
                 std::vector<cudaEvent_t> *tl) {
  size_t off = 0;
  int k = 0;
  for (size_t c : plan) {
    const int lane = k % g_lanes;
    cudaStream_t *st = lane ? p.st2 : p.st;
    const int b = k % g_nbuf;
    char *dx = work + (size_t)b * 2 * cmax, *dy = dx + cmax;
    cudaStream_t sk = g_fuse ? st[0] : st[1];
    if (k >= g_nbuf) CK(cudaStreamWaitEvent(st[0], p.ev_comp[b], 0));
    if (k >= g_nbuf) CK(cudaStreamWaitEvent(st[0], p.ev_out[b], 0));
    if (tl) CK(cudaEventRecord((*tl)[6 * k + 0], st[0]));
    CK(cudaMemcpyAsync(dx, hx + off, c, cudaMemcpyHostToDevice, st[0]));
    if (tl) CK(cudaEventRecord((*tl)[6 * k + 1], st[0]));
    if (!g_fuse) {
      CK(cudaEventRecord(p.ev_in[b], st[0]));
      CK(cudaStreamWaitEvent(sk, p.ev_in[b], 0));
    }
    if (tl) CK(cudaEventRecord((*tl)[6 * k + 2], sk));
    k_copy<<<148 * 8, 256, 0, sk>>>((const uint4 *)dx, (uint4 *)dy, c / 16);
    if (tl) CK(cudaEventRecord((*tl)[6 * k + 3], sk));
    CK(cudaEventRecord(p.ev_comp[b], sk));
    CK(cudaStreamWaitEvent(st[2], p.ev_comp[b], 0));
    if (tl) CK(cudaEventRecord((*tl)[6 * k + 4], st[2]));
    CK(cudaMemcpyAsync(hy + off, dy, c, cudaMemcpyDeviceToHost, st[2]));
    if (tl) CK(cudaEventRecord((*tl)[6 * k + 5], st[2]));
    CK(cudaEventRecord(p.ev_out[b], st[2]));
    off += c;
    ++k;
  }
  for (int i = 0; i < 3; ++i) CK(cudaStreamSynchronize(p.st[i]));
  for (int i = 0; i < 3; ++i) CK(cudaStreamSynchronize(p.st2[i]));
}

int main() {
  const size_t bytes = 32ull << 20;  // 2^24 BF16
  char *hx, *hy, *work;
  CK(cudaHostAlloc(&hx, bytes, 0));
  CK(cudaHostAlloc(&hy, bytes, 0));
  memset(hx, 1, bytes);
  const size_t cmax = 16ull << 20;
  CK(cudaMalloc(&work, 12 * cmax));
  Pipe p;
  for (int i = 0; i < 6; ++i) {
    CK(cudaEventCreateWithFlags(&p.ev_in[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p.ev_comp[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p.ev_out[i], cudaEventDisableTiming));
  }
  for (int i = 0; i < 3; ++i) {
    CK(cudaStreamCreateWithFlags(&p.st2[i], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p.st[i], cudaStreamNonBlocking));
  }
  struct Plan { const char *name; std::vector<size_t> c; };
  std::vector<Plan> plans;
  for (int nch : {2, 4, 8, 16, 32}) {
    Plan pl{nullptr, {}};
    static char names[8][32];
    static int ni = 0;
    snprintf(names[ni], 32, "uniform %d", nch);
    pl.name = names[ni++];
    for (int i = 0; i < nch; ++i) pl.c.push_back(bytes / nch);
    plans.push_back(pl);
  }
  {  // geometric ramp up and down around 4 MiB chunks
    Plan pl{"ramp 0.5-4-0.5 MiB", {}};
    const size_t M = 1 << 20;
    size_t sz[] = {M / 2, M, 2 * M, 4 * M, 4 * M, 4 * M, 4 * M, 4 * M, 4 * M, 2 * M, M, M / 2, M};
    size_t tot = 0;
    for (size_t s : sz) tot += s;
    for (size_t s : sz) pl.c.push_back(s);
    pl.c.back() += bytes - tot;
    plans.push_back(pl);
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int cfg = 0; cfg < 6; ++cfg) {
    g_lanes = 1 + (cfg & 1);
    g_fuse = (cfg >> 1) & 1;
    g_nbuf = cfg >= 4 ? 6 : 3 * g_lanes;
    if (cfg >= 4) g_lanes = 2, g_fuse = cfg == 5;
    for (auto &pl : plans) {
      for (int w = 0; w < 3; ++w) step(p, pl.c, hx, hy, work, cmax, nullptr);
      float best = 1e9;
      for (int r = 0; r < 10; ++r) {
        CK(cudaEventRecord(a, p.st[0]));
        CK(cudaStreamWaitEvent(p.st[1], a, 0));
        CK(cudaStreamWaitEvent(p.st[2], a, 0));
        for (int i = 0; i < 3; ++i) CK(cudaStreamWaitEvent(p.st2[i], a, 0));
        step(p, pl.c, hx, hy, work, cmax, nullptr);
        CK(cudaEventRecord(b, p.st[2]));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
      }
      printf("lanes=%d fuse=%d nbuf=%d %-22s ops=%2zu: best %.4f ms  (%.1f GB/s bidirectional)\n",
             g_lanes, g_fuse, g_nbuf, pl.name, pl.c.size(), best, 2.0 * bytes / best / 1e6);
    }
  }
  g_lanes = 1, g_fuse = 0, g_nbuf = 3;
  // timeline of uniform 8 and the ramp
  for (int which : {2, 5}) {
    auto &pl = plans[which];
    std::vector<cudaEvent_t> tl(6 * pl.c.size());
    for (auto &ev : tl) CK(cudaEventCreate(&ev));
    CK(cudaEventRecord(a, p.st[0]));
    CK(cudaStreamWaitEvent(p.st[1], a, 0));
    CK(cudaStreamWaitEvent(p.st[2], a, 0));
    step(p, pl.c, hx, hy, work, cmax, &tl);
    printf("timeline %s (us): H2D [s e] GB/s | K [s e] | D2H [s e] GB/s\n", pl.name);
    for (size_t k = 0; k < pl.c.size(); ++k) {
      float t[6];
      for (int j = 0; j < 6; ++j) CK(cudaEventElapsedTime(&t[j], a, tl[6 * k + j]));
      printf("  %2zu %5.2f MiB: H2D %7.1f %7.1f %5.1f | K %7.1f %7.1f | D2H %7.1f %7.1f %5.1f\n", k,
             pl.c[k] / 1048576.0, t[0] * 1e3, t[1] * 1e3, pl.c[k] / ((t[1] - t[0]) * 1e6), t[2] * 1e3,
             t[3] * 1e3, t[4] * 1e3, t[5] * 1e3, pl.c[k] / ((t[5] - t[4]) * 1e6));
    }
  }
  // single-op costs
  for (size_t c : {256ull << 10, 1ull << 20, 4ull << 20, 16ull << 20}) {
    float h, d;
    CK(cudaEventRecord(a, p.st[0]));
    for (int r = 0; r < 20; ++r) CK(cudaMemcpyAsync(work, hx, c, cudaMemcpyHostToDevice, p.st[0]));
    CK(cudaEventRecord(b, p.st[0]));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&h, a, b));
    CK(cudaEventRecord(a, p.st[0]));
    for (int r = 0; r < 20; ++r) CK(cudaMemcpyAsync(hy, work, c, cudaMemcpyDeviceToHost, p.st[0]));
    CK(cudaEventRecord(b, p.st[0]));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&d, a, b));
    printf("single-direction back-to-back %6zu KiB: H2D %.1f us (%.1f GB/s)  D2H %.1f us (%.1f GB/s)\n",
           c >> 10, h * 1e3 / 20, c * 20 / (h * 1e6), d * 1e3 / 20, c * 20 / (d * 1e6));
  }
  return 0;
}
