// kt_internal.h -- host-side types shared by the C-ABI layer (kt_api.cu) and
// the kernel launchers (kt_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace kt {

// Per-format packed LUT words, passed to every kernel BY VALUE (a
// __grid_constant__ parameter); lane i of every warp loads entry i into a
// register once and the per-element fetch of theta_t (Alg. 1 line 7,
// PAPER.md:165) is a warp shuffle from lane t.
//
// Let E_in(t) be the input exponent of interval t on the table path
// (t >> 3 = E & 3 with E in {125,126,127,128}) and
// |x| = (E_in << p) | M its magnitude bits, p = 7 (BF16) or 23 (F32).
// Because E_in << p is a multiple of 2^r, |x| >> r = (E_in << (p - r)) + (M >> r),
// so Alg. 1 line 8, (E_t, (M >> r_t) + b_t), equals
//     (|x| >> r_t) + C_t,   C_t = (E_t << p) + b_t 2^(p-7) - (E_in << (p - r_t)).
//
//   bf16[t] = fp32 bits: exponent E_in + 16 + r_t, mantissa
//             ((E_t << 7) + b_t - 2^(7 - r_t)) mod 2^16
//             kernel: low16(bits(RZ(|x| + bf16[t]))) = (E_t << 7) + M_o
//             (see ktanh_bf16x2 in kt_device.cuh)
//   f32K[t] = 2^(31 - r_t),  f32C[t] = C_t (mod 2^32)
//             kernel: umulhi(|x| << 1, f32K[t]) + f32C[t] = (|x| >> r_t) + C_t
struct LutWords {
  uint32_t bf16[32];
  uint32_t f32K[32];
  uint32_t f32C[32];
};

enum Op { OP_TANH = 0, OP_SIGMOID = 1, OP_SWISH = 2, OP_GELU = 3 };
enum Fmt { FMT_BF16 = 0, FMT_F32 = 1 };

struct LaunchInfo {
  int device;
  int sm_count;
};

// Enqueue op over n elements (x, y device-accessible pointers on the current
// device).  sysmem: x / y are mapped pinned HOST memory read and written by
// the kernel over PCIe (kt_apply_host's zero-copy path): no L2 prefetch.
cudaError_t launch_map(int op, int fmt, const void *x, void *y, size_t n, const LutWords &lut,
                       cudaStream_t s, const LaunchInfo &li, bool sysmem = false);

// Backward: dx = dy * g(a) (a = saved output for tanh/sigmoid, input x for
// swish/gelu); reading R-BWD.
cudaError_t launch_bwd(int op, int fmt, const void *a, const void *dy, void *dx, size_t n,
                       const LutWords &lut, cudaStream_t s, const LaunchInfo &li);

cudaError_t launch_lstm(const uint16_t *x, uint16_t *y, size_t rows, size_t hidden,
                        int tanh_quarter, const LutWords &lut, cudaStream_t s,
                        const LaunchInfo &li);

// Fused LSTM cell (DESIGN.md R-LSTM-CELL).
cudaError_t launch_lstm_cell(const uint16_t *gates, const float *c_prev, float *c_next,
                             uint16_t *h_next, size_t rows, size_t hidden, const LutWords &lut,
                             cudaStream_t s, const LaunchInfo &li);

// tcgen05 GEMM C = act(RN_bf16(A . B^T)); epi = -1 (none) or an Op.
// Requires M % 128 == 0, N % 256 == 0, K % 64 == 0 (checked by the caller).
cudaError_t launch_gemm(int epi, const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M,
                        size_t N, size_t K, const LutWords &lut, cudaStream_t s, int sms);

void count_launch();

}  // namespace kt
