/*
 * ktanh.h -- C ABI of libktanh.so, the B200 (sm_100a) hot path of K-TanH
 * (Kundu et al., "K-TanH: Efficient TanH for Deep Learning", arXiv 1909.07729).
 *
 * Problem statement (Sec. 2.3): replace TanH with a parametric
 * integer map f(x; theta) ~= TanH(x), theta_t = (E_t, r_t, b_t) fetched from
 * small parameter tables by a 5-bit index t.  Algorithm 1:
 *   |x| <  T1 = 0.25 -> y = x                       (line 3, bypass)
 *   |x| >  T2 = 3.75 -> y = (s, E_bias, 0) = +-1    (line 4, saturate)
 *   else   t = (2 LSBs of E) : (3 MSBs of M)        (line 6)
 *          y = (s, E_t, (M >> r_t) + b_t)           (lines 7-8)
 * Derived activations (Sec. 1):
 *   Sigmoid(x) = (1 + TanH(x/2))/2,  Swish(x) = x Sigmoid(x),
 *   GELU(x) ~= x/2 (1 + TanH(sqrt(2/pi)(x + 0.044715 x^3))).
 *
 * Plain C: no C++ or torch types cross this boundary.  Every entry point
 * returns a kt_status; values never cause errors (the maps are total over
 * all bit patterns, NaN/inf/subnormal behaviour in DESIGN.md readings A2-A6,
 * A21).  A failing call leaves a human-readable reason in kt_last_error()
 * (thread-local).
 *
 * CONVENTIONS FOR ALL DEVICE ENTRY POINTS
 *   x, y     device pointers (cudaMalloc / torch CUDA storage), caller-owned,
 *            contiguous, element-aligned (2 B for BF16, 4 B for F32).  32-byte
 *            alignment is NOT required (unaligned heads/tails are handled;
 *            if x and y differ in their offset mod 32 a slower element-wise
 *            kernel runs).  Both must live on the CURRENT CUDA device.
 *   aliasing y == x (in place) is allowed; any other overlap -> KT_ERR_ARG.
 *   n        element count; n == 0 -> KT_OK without a launch.
 *   NULL     x or y NULL with n > 0 -> KT_ERR_ARG; lut NULL -> KT_ERR_ARG.
 *   stream   a cudaStream_t passed as void* (NULL = legacy default stream).
 *            Calls are asynchronous with respect to the host: they enqueue
 *            one kernel and return.  The library allocates nothing and never
 *            synchronises on these paths, so calls are CUDA-graph capturable.
 *   BF16     data are passed as their uint16_t bit patterns.
 *   errors   KT_ERR_CUDA if the launch fails (cudaGetLastError after launch).
 *   threads  the LUT handle is immutable: concurrent calls from any host
 *            thread, on any stream or device, are safe.
 */
#ifndef KTANH_H
#define KTANH_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define KT_API __attribute__((visibility("default")))
#else
#define KT_API
#endif

#define KT_ABI_VERSION 1

typedef enum {
    KT_OK = 0,
    KT_ERR_ARG = 1,   /* bad pointer, size, overlap, device or enum value  */
    KT_ERR_LUT = 2,   /* parameter table fails validation (kt_lut_create)   */
    KT_ERR_CUDA = 3   /* CUDA runtime error (launch, copy, stream, event)   */
} kt_status;

typedef enum { KT_OP_TANH = 0, KT_OP_SIGMOID = 1, KT_OP_SWISH = 2, KT_OP_GELU = 3 } kt_op;
typedef enum { KT_BF16 = 0, KT_F32 = 1 } kt_dtype;

/* Opaque, immutable parameter-table handle (host memory).  It holds the
 * validated (E_t, r_t, b_t) and the per-format packed words that kernels
 * receive BY VALUE as a kernel parameter, so one handle serves every GPU. */
typedef struct kt_lut_s *kt_lut;

/* ---------------------------------------------------------------------- */
/* Parameter tables T_E, T_r, T_b (Alg. 1 line 1; Sec. 2.4). */
/* ---------------------------------------------------------------------- */

/* Create a handle from three 32-entry host arrays indexed by t (t as in
 * Alg. 1 line 6: t = ((E & 3) << 3) | (M >> 4) for BF16).  Validation
 * (KT_ERR_LUT on failure, *out untouched):
 *   0 <= r_t <= 7 (r_max <= p, Eq. 2), 1 <= E_t <= 127;
 *   no mantissa overflow/underflow for every input the table path can reach
 *   (the purpose of b_min/b_max): 0 <= (m >> r_t) + b_t <= 127
 *   for BF16, 0 <= (M23 >> r_t) + b_t 2^16 < 2^23 for F32;
 *   E_t == 127 only if every reachable M_o is 0 (keeps |y| <= 1).
 * The caller keeps ownership of E, r, b; *out must be released with
 * kt_lut_destroy. */
KT_API kt_status kt_lut_create(const int32_t E[32], const int32_t r[32], const int32_t b[32],
                               kt_lut *out);

/* Handle for the paper's Table 1. */
KT_API kt_status kt_lut_create_paper(kt_lut *out);

/* F32-native table re-optimised at p = 23 (the Sec. 2.4
 * optimizer run with p = 23, "p = 7 in case of BFloat16").
 * Same index t (= ((E & 3) << 3) | (M23 >> 20)), thresholds and Alg. 1, but
 * b_t is in units of 2^-23: line 8 is M_o = (M23 >> r_t) + b_t.  Validation
 * (KT_ERR_LUT): 0 <= r_t <= 23, 1 <= E_t <= 127, 0 <= M_o < 2^23 for every
 * reachable M23, E_t == 127 only with M_o == 0.  The handle serves the F32
 * calls only (ktanh/ksigmoid/kswish/kgelu_f32, their backward passes,
 * kgelu_swish_f32, kt_apply / kt_apply_host with KT_F32); every call that
 * reads BF16 data (incl. ktanh_f32_via_bf16, the LSTM and GEMM calls) returns
 * KT_ERR_LUT for it.  Ownership as kt_lut_create. */
KT_API kt_status kt_lut_create_f32(const int32_t E[32], const int32_t r[32], const int32_t b[32],
                                   kt_lut *out);

/* Build a table with the Sec. 2.4 optimizer (Steps 1-3,
 * Eq. 2-3) from tanh itself, readings A12-A17 of DESIGN.md §3: p = 7 gives a
 * BF16 table (the paper's "R*" table: it differs from the printed Table 1 in
 * 6 of 32 rows) as kt_lut_create would; p = 23 gives the
 * F32-native table as kt_lut_create_f32 would.  bmin_zero != 0 is the Sec.
 * 3.1 ablation (b_min = 0).  Host-only, deterministic; p = 23
 * takes well under a second on a multi-core host (intervals run on host
 * threads).  KT_ERR_ARG for another p. */
KT_API kt_status kt_lut_create_optimized(int32_t p, int32_t bmin_zero, kt_lut *out);

/* Unit of the handle's b: *p = 7 (kt_lut_create / _paper) or 23 (kt_lut_create_f32). */
KT_API kt_status kt_lut_mantissa_bits(kt_lut lut, int32_t *p);

/* Copy the handle's tables back out (host arrays of 32; b in the
 * handle's unit, see kt_lut_mantissa_bits). */
KT_API kt_status kt_lut_get(kt_lut lut, int32_t E[32], int32_t r[32], int32_t b[32]);

/* Release a handle; NULL is a no-op. */
KT_API void kt_lut_destroy(kt_lut lut);

/* 64-interval tables ("we can use 64 entries by choosing 4
 * bits of mantissa").  Index t = ((E & 3) << 4) | (M >> 3)
 * (2 exponent LSBs, 4 mantissa MSBs); validation as kt_lut_create with the
 * 8-mantissa intervals m in [8v, 8v + 7], v = t & 15.  A separate handle
 * type: only ktanh64_bf16 takes it. */
typedef struct kt_lut64_s *kt_lut64;
KT_API kt_status kt_lut64_create(const int32_t E[64], const int32_t r[64], const int32_t b[64],
                                 kt_lut64 *out);
KT_API kt_status kt_lut64_get(kt_lut64 lut, int32_t E[64], int32_t r[64], int32_t b[64]);

/* 64-interval table from the Sec. 2.4 optimizer with 4 mantissa index bits
 * (as kt_lut_create_optimized with p = 7). */
KT_API kt_status kt_lut64_create_optimized(int32_t bmin_zero, kt_lut64 *out);
KT_API void kt_lut64_destroy(kt_lut64 lut);   /* NULL-safe */

/* ---------------------------------------------------------------------- */
/* Elementwise maps over device memory (conventions above).               */
/* ---------------------------------------------------------------------- */

/* K-TanH, Algorithm 1 on BF16 bit patterns.  Bit-exact
 * with the paper's algorithm; NaN passes through unchanged (A6). */
KT_API kt_status ktanh_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream);

/* K-TanH (Algorithm 1) on BF16 with a 64-interval table: lane i holds
 * entries i and 32 + i, both shuffled, one selected by bit 5 of t. */
KT_API kt_status ktanh64_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut64 lut, void *stream);

/* K-TanH on F32, native reading A8 ("compatible with multiple
 * such data formats"): same thresholds and 5-bit index (E & 3, top 3
 * mantissa bits), M_o = (M23 >> r_t) + b_t 2^16. */
KT_API kt_status ktanh_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream);

/* K-TanH of F32 data through BF16 (the alternative to
 * reading A8; "We assume BFloat16 input for K-TanH (Float32 to
 * BFloat16 conversion cost is not considered)"): y = widen(ktanh_bf16(
 * RNE_bf16(x))), so every output is a BF16 value stored as F32.  NaN -> NaN
 * (canonical quiet NaN); |x| > max BF16 rounds to inf and saturates to +-1. */
KT_API kt_status ktanh_f32_via_bf16(const float *x, float *y, size_t n, kt_lut lut, void *stream);

/* K-Sigmoid = (1 + K-TanH(x/2))/2 (reading A7).  x/2 is
 * rounded to the format, the affine step is one fp32 fma rounded once to
 * the format. */
KT_API kt_status ksigmoid_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream);
KT_API kt_status ksigmoid_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream);

/* K-Swish = x K-Sigmoid(x) = hx (1 + K-TanH(RN(hx))), hx = x/2.
 * The outer step is the exact value hx (1 + t) rounded ONCE to the format
 * (reading R-DERIVED), also where x/2 itself is not representable (|x| <
 * 2^-125 with an odd last bit): there the exact t-term decides the tie.
 * The sign of a zero result is not specified (reading A21). */
KT_API kt_status kswish_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream);
KT_API kt_status kswish_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream);

/* K-GELU = x/2 (1 + K-TanH(u)), u = x fma(C1, x^2, C0) in fp32 with
 * C0 = f32(sqrt(2/pi)), C1 = f32(sqrt(2/pi) 0.044715) (PAPER.md:69-71,
 * reading R-GELU-ARG); for BF16, u is rounded to BF16 before K-TanH.  The
 * outer step x/2 (1 + t) is rounded once from its exact value, as for
 * kswish_* (reading R-DERIVED). */
KT_API kt_status kgelu_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream);
KT_API kt_status kgelu_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream);

/* K-GELU and K-Swish of the same input in ONE pass (BASELINE.json config 5
 * applies both to the FFN tensor; reading A20): reads x once, writes both
 * outputs -- 6 B of HBM traffic per BF16 element instead of 2 x 4 B.  Each
 * output is bit-identical to kgelu_* / kswish_* on the same x.  y_gelu and
 * y_swish must not overlap each other; either may equal x (in place), any
 * other overlap -> KT_ERR_ARG. */
KT_API kt_status kgelu_swish_bf16(const uint16_t *x, uint16_t *y_gelu, uint16_t *y_swish, size_t n,
                                  kt_lut lut, void *stream);
KT_API kt_status kgelu_swish_f32(const float *x, float *y_gelu, float *y_swish, size_t n, kt_lut lut,
                                 void *stream);

/* LSTM gate block (BASELINE.json config 4; GNMT LSTM):
 * x, y are row-major [rows, 4*hidden] BF16; quarter q of every row gets
 * K-TanH if q == tanh_quarter (the cell candidate g; 2 in PyTorch's
 * i,f,g,o order) and K-Sigmoid otherwise, in one pass.
 * KT_ERR_ARG if hidden == 0 or tanh_quarter is not in 0..3. */
KT_API kt_status klstm_gates_bf16(const uint16_t *x, uint16_t *y, size_t rows, size_t hidden,
                                  int tanh_quarter, kt_lut lut, void *stream);

/* Fused LSTM cell (GNMT LSTM), one pass:
 *   gates  [rows, 4*hidden] BF16, quarters in PyTorch order i, f, g, o;
 *   c_prev [rows, hidden] F32 -> c_next [rows, hidden] F32,
 *   h_next [rows, hidden] BF16:
 *   i, f, o = K-Sigmoid(gate), g = K-TanH(gate) (BF16, as klstm_gates_bf16)
 *   c_next  = RN32(f * c_prev + i * g)
 *   h_next  = RN_bf16(o * K-TanH_f32(c_next))   (reading R-LSTM-CELL)
 * 18 bytes of HBM traffic per cell element.  c_next may equal c_prev (in
 * place); any other overlap between outputs and inputs -> KT_ERR_ARG.
 * hidden % 16 == 0 and 32-B aligned pointers take the vector path. */
KT_API kt_status klstm_cell_bf16(const uint16_t *gates, const float *c_prev, float *c_next,
                                 uint16_t *h_next, size_t rows, size_t hidden, kt_lut lut,
                                 void *stream);

/* GEMM with a K-activation epilogue (fuse K-GELU into the
 * FFN GEMM).  C[M, N] = act(RN_bf16(A[M, K] . B[N, K]^T))
 * with A, B, C BF16 row-major (B is [N, K], like nn.Linear's weight), fp32
 * accumulation (tcgen05 tensor cores, TMEM accumulator, TMA operand loads),
 * epilogue = -1 (plain BF16 output) or a kt_op applied exactly as the
 * elementwise k<op>_bf16 applies it to a BF16 tensor: the fused output is
 * bit-identical to "epilogue -1, then k<op>_bf16".
 * Requires M % 128 == 0, N % 256 == 0, K % 64 == 0, A and B 16-byte and C
 * 32-byte aligned, C disjoint from A and B (KT_ERR_ARG otherwise); lut may
 * be NULL only for epilogue -1. */
KT_API kt_status kgemm_bf16(const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M, size_t N,
                            size_t K, int epilogue, kt_lut lut, void *stream);

/* The LSTM gate GEMM with the gate activations fused (
 * BASELINE.json config 4; GNMT LSTM): C[M, 4*hidden] =
 * gates(RN_bf16(A[M, K] . B[4*hidden, K]^T)) where columns of quarter
 * tanh_quarter (the cell candidate g; 2 in PyTorch's i,f,g,o order) get
 * K-TanH and the other quarters K-Sigmoid -- bit-identical to kgemm_bf16
 * (epilogue -1) followed by klstm_gates_bf16.  Requires hidden % 256 == 0
 * (each 256-column tile lies in one quarter) and the kgemm_bf16 shape and
 * alignment rules (M % 128 == 0, K % 64 == 0); KT_ERR_ARG otherwise. */
KT_API kt_status kgemm_lstm_gates_bf16(const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M,
                                       size_t hidden, size_t K, int tanh_quarter, kt_lut lut,
                                       void *stream);

/* The LSTM step core with the cell fused into the gate GEMM's epilogue
 * (GNMT LSTM): gates = RN_bf16(A[M, K] .
 * B[4*hidden, K]^T) with B's rows in PyTorch's i, f, g, o blocks, then
 * exactly klstm_cell_bf16's cell (c_next = RN32(f c_prev + i g), h_next =
 * RN_bf16(o K-TanH_f32(c_next)), i, f, o = K-Sigmoid, g = K-TanH) -- the gate
 * block is never written.  Bit-identical to kgemm_bf16 then klstm_cell_bf16.
 * c_prev, c_next [M, hidden] F32, h_next [M, hidden] BF16, row-major;
 * c_next may equal c_prev.  Requires M % 128 == 0, hidden % 64 == 0,
 * K % 64 == 0, A, B 16-byte and c/h 32-byte aligned; KT_ERR_ARG otherwise. */
KT_API kt_status kgemm_lstm_cell_bf16(const uint16_t *A, const uint16_t *B, const float *c_prev,
                                      float *c_next, uint16_t *h_next, size_t M, size_t hidden,
                                      size_t K, kt_lut lut, void *stream);

/* Generic dispatcher over (op, dtype); same contract as the calls above. */
KT_API kt_status kt_apply(kt_op op, kt_dtype dtype, const void *x, void *y, size_t n,
                          kt_lut lut, void *stream);

/* ---------------------------------------------------------------------- */
/* Backward passes (the paper trains GNMT with K-TanH,   */
/* PAPER.md:308, but never states the gradient).  Reading R-BWD            */
/* (DESIGN.md): the derivative of the approximated function taken through  */
/* the K-TanH value, dx = dy * g, fp32 arithmetic with a fixed op order and */
/* one rounding to the format:                                              */
/*   tanh:    g = 1 - y^2        (y = saved K-TanH output)                  */
/*   sigmoid: g = s (1 - s)      (s = saved K-Sigmoid output)               */
/*   swish:   g = (1+t)/2 + x (1-t^2)/4,  t = K-TanH(RN(x/2))               */
/*   gelu:    g = (1+t)/2 + x/2 (1-t^2) sqrt(2/pi)(1 + 3*0.044715 x^2),     */
/*            t = K-TanH(u), u as in kgelu_*                                */
/* Same conventions as the forward maps; dx may equal dy or the first       */
/* input (in place), any other overlap -> KT_ERR_ARG.  tanh/sigmoid need no */
/* table; swish/gelu recompute K-TanH and need lut (NULL -> KT_ERR_ARG).    */
/* 6 bytes of HBM traffic per BF16 element (12 per F32).                    */
/* ---------------------------------------------------------------------- */
KT_API kt_status ktanh_bwd_bf16(const uint16_t *y, const uint16_t *dy, uint16_t *dx, size_t n,
                                void *stream);
KT_API kt_status ktanh_bwd_f32(const float *y, const float *dy, float *dx, size_t n, void *stream);
KT_API kt_status ksigmoid_bwd_bf16(const uint16_t *s, const uint16_t *dy, uint16_t *dx, size_t n,
                                   void *stream);
KT_API kt_status ksigmoid_bwd_f32(const float *s, const float *dy, float *dx, size_t n,
                                  void *stream);
KT_API kt_status kswish_bwd_bf16(const uint16_t *x, const uint16_t *dy, uint16_t *dx, size_t n,
                                 kt_lut lut, void *stream);
KT_API kt_status kswish_bwd_f32(const float *x, const float *dy, float *dx, size_t n, kt_lut lut,
                                void *stream);
KT_API kt_status kgelu_bwd_bf16(const uint16_t *x, const uint16_t *dy, uint16_t *dx, size_t n,
                                kt_lut lut, void *stream);
KT_API kt_status kgelu_bwd_f32(const float *x, const float *dy, float *dx, size_t n, kt_lut lut,
                               void *stream);
/* Generic dispatcher; a = y (tanh), s (sigmoid) or x (swish, gelu). */
KT_API kt_status kt_apply_bwd(kt_op op, kt_dtype dtype, const void *a, const void *dy, void *dx,
                              size_t n, kt_lut lut, void *stream);

/* ---------------------------------------------------------------------- */
/* Table 2 comparators: the float-op TanH approximations */
/* the paper measures K-TanH against, Sec. 2.1 minimax   */
/* and Sec. 2.2 Pade, plus the GPU's own tanh routines.  */
/* Readings R-CMP-* (DESIGN.md):                                            */
/*   KT_APX_PADE     [p/q], p odd, q = p +- 1 even, p + q <= 19:            */
/*                   y = x N(x^2) / D(x^2) (the Pade approximant, built as  */
/*                   a convergent of Lambert's continued fraction),         */
/*                   fp32 Horner + IEEE division, min(y, 1), and +-1 for    */
/*                   |x| >= RN32(X_p), X_p = first x > 0 where the rational */
/*                   reaches 1 or stops increasing.                         */
/*   KT_APX_MINIMAX  degree p in 1..3 (q ignored): 16 pieces of width 1/2   */
/*                   on [0, 8), per-piece minimax polynomial (Remez; piece  */
/*                   0 constrained to P(0) = 0) in h = |x| - k/2;           */
/*                   |x| >= 8 -> +-1.                                       */
/*   KT_APX_TAYLOR   degree p in 1..3: same layout, piece 0 = Maclaurin     */
/*                   polynomial, piece k >= 1 = Taylor polynomial about     */
/*                   k/2 + 1/4.                                             */
/*   KT_APX_LIBM     tanhf() of the CUDA math library (p, q ignored).       */
/*   KT_APX_SFU      tanh.approx.f32 / tanh.approx.bf16x2 (MUFU.TANH).      */
/* All are odd-extended (sign restored from x), NaN passes through          */
/* unchanged; BF16 inputs are widened exactly, evaluated in fp32 with a     */
/* fixed operation order and rounded once (RNE) to BF16.                    */
/* kt_apx_create: KT_ERR_ARG for an unsupported (kind, p, q).  Handles are  */
/* immutable host objects (thread-safe), passed to kernels by value.        */
/* kt_apx_tanh_*: same conventions as ktanh_bf16 / ktanh_f32.               */
/* ---------------------------------------------------------------------- */
typedef enum {
  KT_APX_PADE = 0, KT_APX_MINIMAX = 1, KT_APX_TAYLOR = 2, KT_APX_LIBM = 3, KT_APX_SFU = 4
} kt_apx_kind;
typedef struct kt_apx_s *kt_apx;

/* Coefficient block returned by kt_apx_coeffs, binary64 (the kernels use
 * these rounded to fp32):  coef[0] = saturation point (X_p, or 8);
 * Pade: coef[1 + i] = a_i (i = 0..p), coef[2 + p + i] = b_i (i = 0..q),
 *       b_0 = 1, R(x) = sum a_i x^i / sum b_i x^i;
 * piecewise: coef[1 + 4k + j] = c_j of piece k (powers of h, see above). */
#define KT_APX_NCOEF 65

KT_API kt_status kt_apx_create(kt_apx_kind kind, int p, int q, kt_apx *out);
KT_API kt_status kt_apx_coeffs(kt_apx a, double coef[KT_APX_NCOEF]);
KT_API void kt_apx_destroy(kt_apx a);   /* NULL-safe */
KT_API kt_status kt_apx_tanh_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_apx a,
                                  void *stream);
KT_API kt_status kt_apx_tanh_f32(const float *x, float *y, size_t n, kt_apx a, void *stream);

/* ---------------------------------------------------------------------- */
/* Host-buffer path (the end-to-end call a user with host data makes).    */
/* ---------------------------------------------------------------------- */

/* y_host = op(x_host) for n elements resident in HOST memory.  The call
 * splits the data into chunks and pipelines them over three internal
 * streams, one per engine (host->device copies, kernels, device->host
 * copies), with three rotating device buffers, so that both copy directions
 * and the kernel overlap; the internal streams
 * are forked from and joined back into `stream`, so the whole operation is
 * ordered on `stream` and the call returns without waiting: synchronise
 * `stream` before reading y_host.  x_host / y_host should be pinned
 * (cudaHostAlloc / torch pin_memory) for asynchronous, full-bandwidth
 * copies; pageable memory works but the copies become synchronous.
 * d_work: caller-owned device scratch of work_bytes; at least
 * 3 * 2 * 4096 * elem_size bytes (KT_ERR_ARG otherwise).  The chunk is
 * about n/3 elements (at least 1 MiB, at most work_bytes / (6 * elem_size)),
 * a multiple of 256 elements.
 * Strategy knob (environment, read per call): KT_HOST_ZEROCOPY=1 runs ONE
 * kernel that reads x_host and writes y_host in place over PCIe when both
 * are pinned and mapped (UVA); =2 keeps the H2D copies but lets the kernel
 * store straight into a mapped y_host; unset/0 (default) is the copy-engine
 * pipeline, the fastest measured on B200 (profiles/host_path_r01.txt).
 * Pageable buffers always take the pipeline.  x_host and y_host may be
 * equal (in place); any other overlap is KT_ERR_ARG.  Calls on DIFFERENT
 * caller streams with different d_work buffers overlap on the copy engines
 * (one call's D2H with the next one's H2D); calls that reuse the same
 * d_work are ordered on it internally, so sharing d_work is always safe.  d_work may be NULL
 * only on the mode-1 zero-copy path. */
KT_API kt_status kt_apply_host(kt_op op, kt_dtype dtype, const void *x_host, void *y_host,
                               size_t n, kt_lut lut, void *d_work, size_t work_bytes,
                               void *stream);

/* kt_apply_host with the chunk size chosen by the caller: chunk_elems = 0
 * is kt_apply_host's default (~n/3); otherwise chunks of chunk_elems
 * elements (>= 4096, rounded down to a multiple of 256; still capped by
 * work_bytes / (6 * elem_size)).  Fewer, larger chunks suit callers that
 * overlap calls on several streams (each call's D2H under the next call's
 * H2D: config 2 end to end 24.0 Gelem/s with whole-call chunks on two
 * streams vs 22.6 with 3 chunks); more chunks suit a lone call. */
KT_API kt_status kt_apply_host_ex(kt_op op, kt_dtype dtype, const void *x_host, void *y_host,
                                  size_t n, kt_lut lut, void *d_work, size_t work_bytes,
                                  size_t chunk_elems, void *stream);

/* ---------------------------------------------------------------------- */
/* Multi-GPU sharding (host logic; BASELINE.json north_star item (c)).     */
/* ---------------------------------------------------------------------- */

/* Contiguous flat shard of rank `rank` out of `world`: shard size is
 * ceil(n / world) rounded up to a multiple of `align` elements (align >= 1;
 * 16 keeps BF16 shards on 32-byte boundaries); the last shards take the
 * remainder and may be empty.  No data moves: every rank owns its range
 * and the path has no reduction, so there is no collective.
 * KT_ERR_ARG if world < 1, rank outside [0, world), align == 0 or an
 * output pointer is NULL. */
KT_API kt_status kt_shard_range(size_t n, int world, int rank, size_t align,
                                size_t *begin, size_t *count);

/* ---------------------------------------------------------------------- */
/* Diagnostics                                                            */
/* ---------------------------------------------------------------------- */
KT_API const char *kt_status_string(kt_status s);
KT_API const char *kt_last_error(void);      /* thread-local; "" if none */
KT_API int kt_abi_version(void);             /* == KT_ABI_VERSION */

/* In-register throughput of one map on the current GPU: the B200 analogue of
 * Table 2's "cycles per TanH".  Pass exactly one of lut
 * (K-TanH, Alg. 1) or apx (a comparator).  sample_host: 4096 host words of
 * input (BF16 pairs or F32) that every thread cycles through.  One full wave
 * of CTAs holds 16 words per thread in registers and applies the map `iters`
 * rounds with no memory traffic; *cycles_gross = SM clock cycles per element
 * per SM (max CTA clock64 span / elements per SM), *cycles_net = the same
 * minus an identity map's loop cost.  SYNCHRONOUS (allocates and frees
 * 64 KiB-scale scratch, synchronises the device): a diagnostic, not a hot-
 * path call. */
KT_API kt_status kt_alu_probe(kt_dtype dtype, kt_lut lut, kt_apx apx, const void *sample_host,
                              int iters, double *cycles_net, double *cycles_gross);

/* Number of kernel launches this process has issued through the library
 * (all devices, all threads); used by bench.py's gpu_launches count. */
KT_API uint64_t kt_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* KTANH_H */
