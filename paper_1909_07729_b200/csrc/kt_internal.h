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

// 64-interval table: per-entry words of the same form as
// LutWords::bf16, entry t in w[t] (lane i loads w[i] and w[32 + i]).
struct LutWords64 {
  uint32_t w[64];
};

enum Op { OP_TANH = 0, OP_SIGMOID = 1, OP_SWISH = 2, OP_GELU = 3,
          OP_TANH_VIA_BF16 = 4 /* F32 only: RNE to BF16, Alg. 1, widen (NEXT-3) */ };
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

// K-TanH BF16 with a 64-entry table (x, y as for launch_map).
cudaError_t launch_map64(const void *x, void *y, size_t n, const LutWords64 &lut, cudaStream_t s,
                         const LaunchInfo &li);

// Backward: dx = dy * g(a) (a = saved output for tanh/sigmoid, input x for
// swish/gelu); reading R-BWD.
cudaError_t launch_bwd(int op, int fmt, const void *a, const void *dy, void *dx, size_t n,
                       const LutWords &lut, cudaStream_t s, const LaunchInfo &li);

// Fused K-GELU + K-Swish over one input (config 5, reading A20).
cudaError_t launch_dual(int fmt, const void *x, void *yg, void *ys, size_t n, const LutWords &lut,
                        cudaStream_t s, const LaunchInfo &li);

cudaError_t launch_lstm(const uint16_t *x, uint16_t *y, size_t rows, size_t hidden,
                        int tanh_quarter, const LutWords &lut, cudaStream_t s,
                        const LaunchInfo &li);

// Fused LSTM cell (DESIGN.md R-LSTM-CELL).
cudaError_t launch_lstm_cell(const uint16_t *gates, const float *c_prev, float *c_next,
                             uint16_t *h_next, size_t rows, size_t hidden, const LutWords &lut,
                             cudaStream_t s, const LaunchInfo &li);

// tcgen05 GEMM C = act(RN_bf16(A . B^T)); epi = -1 (none) or an Op.
// Requires M % 128 == 0, N % 256 == 0, K % 64 == 0 (checked by the caller).
// epi = 8: LSTM gate block (K-TanH on columns of quarter lstm_tq of each
// 4*lstm_hidden row, K-Sigmoid elsewhere; lstm_hidden % 256 == 0).
cudaError_t launch_gemm(int epi, const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M,
                        size_t N, size_t K, const LutWords &lut, cudaStream_t s, int sms,
                        uint32_t lstm_hidden = 0, uint32_t lstm_tq = 0);

// tcgen05 GEMM with the LSTM cell fused into its epilogue (B in i,f,g,o
// row blocks of H rows; H % 64 == 0, M % 128 == 0, K % 64 == 0).
cudaError_t launch_gemm_cell(const uint16_t *A, const uint16_t *B, const float *c_prev, float *c_next,
                             uint16_t *h_next, size_t M, size_t H, size_t K, const LutWords &lut,
                             cudaStream_t s, int sms);

// Sec. 2.4 optimizer (kt_tables.cu): 4 << s entries for s mantissa index bits,
// p = 7 (BF16) or 23 (F32-native); false for unsupported (s, p).
bool optimize_table(int s, int p, bool bmin_zero, int32_t *E, int32_t *r, int32_t *b);

void count_launch();
bool pdl_enabled();        // KT_PDL != 0
bool prefetch_enabled();   // KT_PREFETCH != 0 (and PDL on)

// ---- Table 2 comparators (kt_apx.cu) --------------------
enum ApxKind { APX_PADE = 0, APX_MINIMAX = 1, APX_TAYLOR = 2, APX_LIBM = 3, APX_SFU = 4 };
// Piecewise layout, reading R-CMP-LAYOUT: 16 pieces of width 1/2 on [0, 8).
constexpr int kApxPieces = 16;
constexpr double kApxWidth = 0.5;
constexpr double kApxXsat = 8.0;
constexpr int kApxCoef = 1 + 4 * kApxPieces;   // == KT_APX_NCOEF

// Kernel parameter block (by value, __grid_constant__).  Pade: y = x N(s)/D(s)
// with s = x^2, num/den in powers of s (D(0) = 1), xsat = RN32(X_p).
// Piecewise: pc[j][k] = coefficient j of piece k (lanes 16..31 mirror 0..15).
struct ApxWords {
  int32_t kind, p, q, pad;
  float xsat;
  float num[6];
  float den[6];
  float pc[4][32];
};

// Derive the coefficients (host); coef[kApxCoef] receives them in binary64
// in the layout of KT_APX_NCOEF (include/ktanh.h).  false + message if the
// (kind, p, q) is unsupported.
bool apx_build(int kind, int p, int q, ApxWords *w, double *coef, char *err, size_t errlen);
// In-register throughput probe (kt_alu_probe): which = 1 K-TanH, 2 comparator.
cudaError_t alu_probe(int which, int fmt, const LutWords &lw, const ApxWords &w, int iters,
                      const uint32_t *host_in4096, double *cyc_net, double *cyc_gross, int sms);
cudaError_t launch_apx(int fmt, const void *x, void *y, size_t n, const ApxWords &w,
                       cudaStream_t s, const LaunchInfo &li);

}  // namespace kt
