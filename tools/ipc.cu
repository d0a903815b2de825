// tools/ipc.cu -- per-instruction throughput on this GPU (dev tool).
// Each thread runs 8 independent dependency chains of one instruction kind;
// reports warp-level instructions per SM per clock (max 4 = one per SMSP).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                  \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int ITERS = 4096;

#define CHAIN8(STMT) \
  STMT(a0) STMT(a1) STMT(a2) STMT(a3) STMT(a4) STMT(a5) STMT(a6) STMT(a7)

#define KERNEL(NAME, STMT)                                                            \
  __global__ void NAME(uint32_t *out, uint32_t s) {                                   \
    uint32_t a0 = threadIdx.x ^ s, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, \
             a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;                                  \
    const uint32_t k = s | 0x10001;                                                   \
    _Pragma("unroll 16") for (int i = 0; i < ITERS; ++i) {                           \
      CHAIN8(STMT)                                                                    \
    }                                                                                 \
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7; \
  }

#define S_LOP3(a) asm volatile("lop3.b32 %0, %0, %1, 0x7fff7fff, 0xc8;" : "+r"(a) : "r"(k));
#define S_SHF(a) asm volatile("shr.b32 %0, %0, 3;" : "+r"(a));
#define S_SHFW(a) asm volatile("shf.r.wrap.b32 %0, %0, %1, %0;" : "+r"(a) : "r"(k));
#define S_IADD(a) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(k));
#define S_IMAD(a) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(a) : "r"(k));
#define S_IMADHI(a) asm volatile("mad.hi.u32 %0, %0, %1, %1;" : "+r"(a) : "r"(k));
#define S_MULHI(a) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a) : "r"(k));
#define S_PRMT(a) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a) : "r"(k));
#define S_SHFL(a) asm volatile("shfl.sync.idx.b32 %0, %0, %0, 0x1f, 0xffffffff;" : "+r"(a));
#define S_HSET2(a) asm volatile("set.gt.u32.bf16x2 %0, %0, %1;" : "+r"(a) : "r"(k));
#define S_F2FP(a) asm volatile("{.reg .f32 f; mov.b32 f, %0; cvt.rn.bf16x2.f32 %0, f, f;}" : "+r"(a));
#define S_FFMA(a) asm volatile("{.reg .f32 f; mov.b32 f, %0; fma.rn.f32 f, f, f, f; mov.b32 %0, f;}" : "+r"(a));
#define S_SHL(a) asm volatile("shl.b32 %0, %0, 3;" : "+r"(a));

KERNEL(k_lop3, S_LOP3)
KERNEL(k_shf, S_SHF)
KERNEL(k_shfw, S_SHFW)
KERNEL(k_iadd, S_IADD)
KERNEL(k_imad, S_IMAD)
KERNEL(k_imadhi, S_IMADHI)
KERNEL(k_mulhi, S_MULHI)
KERNEL(k_prmt, S_PRMT)
KERNEL(k_shfl, S_SHFL)
KERNEL(k_hset2, S_HSET2)
KERNEL(k_f2fp, S_F2FP)
KERNEL(k_ffma, S_FFMA)
KERNEL(k_shl, S_SHL)

__global__ void k_ffma2(uint32_t *out, uint32_t s) {
  uint64_t a[8];
  for (int j = 0; j < 8; ++j) a[j] = ((uint64_t)(threadIdx.x + j) << 32) | (s + j);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(a[j]));
  }
  uint64_t r = 0;
  for (int j = 0; j < 8; ++j) r ^= a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)r;
}

// mixes to see pipe overlap: LOP3 + IMAD interleaved
#define S_MIX(a) asm volatile("lop3.b32 %0, %0, %1, 0x7fff7fff, 0xc8;\n\tmad.lo.u32 %0, %0, %1, %1;" : "+r"(a) : "r"(k));
KERNEL(k_mix_lop_imad, S_MIX)
#define S_MIX2(a) asm volatile("shr.b32 %0, %0, 3;\n\tshfl.sync.idx.b32 %0, %0, %0, 0x1f, 0xffffffff;" : "+r"(a));
KERNEL(k_mix_shf_shfl, S_MIX2)
#define S_MIX3(a) asm volatile("lop3.b32 %0, %0, %1, 0x7fff7fff, 0xc8;\n\tset.gt.u32.bf16x2 %0, %0, %1;" : "+r"(a) : "r"(k));
KERNEL(k_mix_lop_hset, S_MIX3)
#define S_MIX4(a) asm volatile("mad.lo.u32 %0, %0, %1, %1;\n\tset.gt.u32.bf16x2 %0, %0, %1;" : "+r"(a) : "r"(k));
KERNEL(k_mix_imad_hset, S_MIX4)
#define S_MIX5(a) asm volatile("lop3.b32 %0, %0, %1, 0x7fff7fff, 0xc8;\n\tprmt.b32 %0, %0, %1, 0x5410;" : "+r"(a) : "r"(k));
KERNEL(k_mix_lop_prmt, S_MIX5)
#define S_MIX6(a) asm volatile("{.reg .f32 f; mov.b32 f, %0; cvt.rn.bf16x2.f32 %0, f, f;}\n\tmad.lo.u32 %0, %0, %1, %1;" : "+r"(a) : "r"(k));
KERNEL(k_mix_f2fp_imad, S_MIX6)
#define S_MIX7(a) asm volatile("{.reg .f32 f; mov.b32 f, %0; cvt.rn.bf16x2.f32 %0, f, f;}\n\tlop3.b32 %0, %0, %1, 0x7fff7fff, 0xc8;" : "+r"(a) : "r"(k));
KERNEL(k_mix_f2fp_lop, S_MIX7)
#define S_MIX8(a) asm volatile("lop3.b32 %0, %0, %1, 0x7fff7fff, 0xc8;\n\tshfl.sync.idx.b32 %0, %0, %0, 0x1f, 0xffffffff;" : "+r"(a) : "r"(k));
KERNEL(k_mix_lop_shfl, S_MIX8)
#define S_MIX9(a) asm volatile("lop3.b32 %0, %0, %1, 0x7fff7fff, 0xc8;\n\tadd.u32 %0, %0, %1;" : "+r"(a) : "r"(k));
KERNEL(k_mix_lop_iadd, S_MIX9)
#define S_MIX10(a) asm volatile("mad.lo.u32 %0, %0, %1, %1;\n\tadd.u32 %0, %0, %1;" : "+r"(a) : "r"(k));
KERNEL(k_mix_imad_iadd, S_MIX10)

int main() {
  int sms, clk;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  uint32_t *out;
  CK(cudaMalloc(&out, 1 << 26));
  struct K {
    const char *n;
    void (*f)(uint32_t *, uint32_t);
    int per;
  } ks[] = {{"LOP3", k_lop3, 1},   {"SHF(const)", k_shf, 1}, {"SHF.R.W(var)", k_shfw, 1},
            {"IADD", k_iadd, 1},   {"IMAD", k_imad, 1},      {"IMAD.HI(mad.hi)", k_imadhi, 1},
            {"mul.hi", k_mulhi, 1}, {"PRMT", k_prmt, 1},     {"SHFL.IDX", k_shfl, 1},
            {"HSET2.BF16", k_hset2, 1}, {"F2FP.BF16", k_f2fp, 1}, {"FFMA", k_ffma, 1},
            {"SHL(const)", k_shl, 1}, {"FFMA2", k_ffma2, 1}, {"LOP3+IMAD", k_mix_lop_imad, 2},
            {"SHF+SHFL", k_mix_shf_shfl, 2}, {"LOP3+HSET2", k_mix_lop_hset, 2},
            {"IMAD+HSET2", k_mix_imad_hset, 2}, {"LOP3+PRMT", k_mix_lop_prmt, 2},
            {"F2FP+IMAD", k_mix_f2fp_imad, 2}, {"F2FP+LOP3", k_mix_f2fp_lop, 2},
            {"LOP3+SHFL", k_mix_lop_shfl, 2}, {"LOP3+IADD", k_mix_lop_iadd, 2},
            {"IMAD+IADD", k_mix_imad_iadd, 2}};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int threads = 512, blocks = sms * 4;
  printf("clock %d MHz, %d SMs, %d threads/SM\n", clk / 1000, sms, threads * 4);
  for (auto &k : ks) {
    k.f<<<blocks, threads>>>(out, 1);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    k.f<<<blocks, threads>>>(out, 3);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double warp_instr = (double)blocks * threads / 32 * ITERS * 8 * k.per;
    // use the observed SM clock from a clock64 calibration is overkill; report per ns
    double per_sm_per_ns = warp_instr / sms / (ms * 1e6);
    printf("%-18s %8.3f ms  %6.3f warp-instr/SM/ns  (= %5.2f /clk at 1.965 GHz)\n", k.n, ms,
           per_sm_per_ns, per_sm_per_ns / 1.965);
  }
  return 0;
}
