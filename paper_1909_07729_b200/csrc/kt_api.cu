// kt_api.cu -- the C ABI of libktanh.so (declared in include/ktanh.h):
// parameter-table handles, argument validation, dispatch to the kernel
// launchers, the pipelined host-buffer path and the shard helper.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <new>
#include <string>

#include "ktanh.h"
#include "kt_internal.h"

namespace kt {
uint64_t launch_count();
}

struct kt_lut_s {
  int32_t E[32], r[32], b[32];
  int32_t p = 7;            // unit of b: 2^-7 (BF16 tables) or 2^-23 (kt_lut_create_f32)
  kt::LutWords words;
};

struct kt_lut64_s {
  int32_t E[64], r[64], b[64];
  kt::LutWords64 words;
};

struct kt_apx_s {
  double coef[kt::kApxCoef];
  kt::ApxWords words;
};

namespace {

thread_local std::string g_err;

kt_status fail(kt_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
kt_status fail(kt_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

kt_status cuda_fail(cudaError_t e, const char *what) {
  return fail(KT_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// Table 1 of the paper, indexed by t = (E&3):(M>>4).
// This is the product's own transcription (the test oracle keeps another).
constexpr int32_t kPaperE[32] = {126, 126, 126, 126, 126, 126, 126, 126,   // 00000-00111
                                 125, 125, 125, 125, 125, 125, 125, 125,   // 01000-01111
                                 125, 126, 126, 126, 126, 126, 126, 126,   // 10000-10111
                                 126, 126, 126, 126, 126, 126, 126, 126};  // 11000-11111
constexpr int32_t kPaperR[32] = {2, 4, 4, 4, 6, 6, 6, 6,
                                 1, 0, 0, 0, 0, 0, 0, 0,
                                 0, 1, 1, 1, 1, 1, 1, 1,
                                 0, 1, 1, 1, 2, 2, 2, 4};
constexpr int32_t kPaperB[32] = {119, 122, 123, 123, 126, 126, 126, 126,
                                 1,   -4,  -6,  -7,  -10, -12, -15, -18,
                                 112, -4,  -1,  2,   3,   4,   4,   4,
                                 65,  72,  73,  73,  88,  89,  89,  110};

// Input exponent of interval t on the table path: t >> 3 = E & 3 with
// E in {125, 126, 127, 128} (T1 = 2^-2 .. T2 = 3.75 < 2^2).
inline int e_in(int t) { return 125 + (((t >> 3) + 3) & 3); }

// Mantissa range [lo, hi] (p = 7) that the table path can reach in interval t:
// all 16 values of the 3 index bits' sub-range, except t = 00111 (E = 128),
// where only M = 0x70 (x = 3.75 = T2) is <= T2.
inline void reach(int t, int *lo, int *hi) {
  const int v = t & 7;
  *lo = 16 * v;
  *hi = 16 * v + 15;
  if (e_in(t) == 128 && v == 7) *hi = *lo;
}

kt_status validate_and_pack(const int32_t *E, const int32_t *r, const int32_t *b, kt_lut_s *L) {
  for (int t = 0; t < 32; ++t) {
    if (r[t] < 0 || r[t] > 7) return fail(KT_ERR_LUT, "r[%d] = %d outside [0, 7]", t, r[t]);
    if (E[t] < 1 || E[t] > 127) return fail(KT_ERR_LUT, "E[%d] = %d outside [1, 127]", t, E[t]);
    int lo, hi;
    reach(t, &lo, &hi);
    for (int m = lo; m <= hi; ++m) {
      const int mo = (m >> r[t]) + b[t];
      if (mo < 0 || mo > 127)
        return fail(KT_ERR_LUT, "entry %d: (m=%d >> r=%d) + b=%d = %d leaves [0, 127]", t, m,
                    r[t], b[t], mo);
      if (E[t] == 127 && mo != 0)
        return fail(KT_ERR_LUT, "entry %d: E=127 with M_o=%d != 0 gives |y| > 1", t, mo);
    }
    // F32 (p = 23): endpoints of the reachable M23 range (the map is monotone in M23).
    const int64_t lo23 = (int64_t)lo << 16;
    const int64_t hi23 = (t == 7) ? lo23 : (((int64_t)hi << 16) | 0xFFFF);
    const int64_t mlo = (lo23 >> r[t]) + (int64_t)b[t] * 65536;
    const int64_t mhi = (hi23 >> r[t]) + (int64_t)b[t] * 65536;
    if (mlo < 0 || mhi > 0x7FFFFF)
      return fail(KT_ERR_LUT, "entry %d overflows the F32 mantissa", t);
    if (E[t] == 127 && mhi != 0)
      return fail(KT_ERR_LUT, "entry %d: E=127 gives |y| > 1 on F32", t);
  }
  for (int t = 0; t < 32; ++t) {
    L->E[t] = E[t];
    L->r[t] = r[t];
    L->b[t] = b[t];
    const int ei = e_in(t);
    const int32_t c16 = (E[t] << 7) + b[t] - (ei << (7 - r[t]));
    // fp32 word with exponent E_in + 16 + r and mantissa D = C + E_in 2^(7-r) - 2^(7-r)
    // (mod 2^16): see ktanh_bf16x2 in kt_device.cuh
    const int32_t d16 = (E[t] << 7) + b[t] - (1 << (7 - r[t]));
    L->words.bf16[t] = ((uint32_t)(ei + 16 + r[t]) << 23) | ((uint32_t)d16 & 0xFFFFu);
    (void)c16;
    L->words.f32K[t] = 1u << (31 - r[t]);
    const int64_t c32 = ((int64_t)E[t] << 23) + (int64_t)b[t] * 65536 - ((int64_t)ei << (23 - r[t]));
    L->words.f32C[t] = (uint32_t)(c32 & 0xFFFFFFFFll);
  }
  return KT_OK;
}

// F32-native table re-optimised at p = 23: b in units of
// 2^-23, r in [0, 23]; Alg. 1 line 8 on F32 is M_o = (M23 >> r) + b.  Only
// the F32 words exist (C_t of kt_internal.h with b_t 2^(p-7) -> b_t).
kt_status validate_and_pack_f32(const int32_t *E, const int32_t *r, const int32_t *b, kt_lut_s *L) {
  for (int t = 0; t < 32; ++t) {
    if (r[t] < 0 || r[t] > 23) return fail(KT_ERR_LUT, "r[%d] = %d outside [0, 23]", t, r[t]);
    if (E[t] < 1 || E[t] > 127) return fail(KT_ERR_LUT, "E[%d] = %d outside [1, 127]", t, E[t]);
    int lo, hi;
    reach(t, &lo, &hi);
    const int64_t lo23 = (int64_t)lo << 16;
    const int64_t hi23 = (t == 7) ? lo23 : (((int64_t)hi << 16) | 0xFFFF);
    const int64_t mlo = (lo23 >> r[t]) + b[t], mhi = (hi23 >> r[t]) + b[t];   // monotone in M23
    if (mlo < 0 || mhi > 0x7FFFFF)
      return fail(KT_ERR_LUT, "entry %d: M_o in [%lld, %lld] leaves [0, 2^23 - 1]", t, (long long)mlo,
                  (long long)mhi);
    if (E[t] == 127 && mhi != 0)
      return fail(KT_ERR_LUT, "entry %d: E=127 with M_o != 0 gives |y| > 1", t);
  }
  L->p = 23;
  L->words = kt::LutWords{};
  for (int t = 0; t < 32; ++t) {
    L->E[t] = E[t];
    L->r[t] = r[t];
    L->b[t] = b[t];
    L->words.f32K[t] = 1u << (31 - r[t]);
    const int64_t c32 = ((int64_t)E[t] << 23) + (int64_t)b[t] - ((int64_t)e_in(t) << (23 - r[t]));
    L->words.f32C[t] = (uint32_t)(c32 & 0xFFFFFFFFll);
  }
  return KT_OK;
}

// The host optimizer allocates and starts threads: no C++ exception may
// cross the C ABI.
kt_status run_optimizer(int s, int p, int32_t bmin_zero, int32_t *E, int32_t *r, int32_t *b) {
  try {
    if (!kt::optimize_table(s, p, bmin_zero != 0, E, r, b)) return fail(KT_ERR_ARG, "optimizer failed");
  } catch (const std::exception &ex) {
    return fail(KT_ERR_ARG, "optimizer: %s", ex.what());
  }
  return KT_OK;
}

// Calls that touch BF16 data need the BF16 words: a p = 23 table has none.
kt_status need_bf16(kt_lut lut) {
  if (lut && lut->p != 7)
    return fail(KT_ERR_LUT, "table from kt_lut_create_f32 (b in 2^-23 units) serves F32 calls only");
  return KT_OK;
}

// ---- device info ----------------------------------------------------------
constexpr int kMaxDev = 64;
int g_sm_count[kMaxDev];  // 0 = unknown
std::mutex g_dev_mu;

kt_status launch_info(kt::LaunchInfo *li) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= kMaxDev) return fail(KT_ERR_ARG, "device %d out of range", dev);
  int sm = __atomic_load_n(&g_sm_count[dev], __ATOMIC_ACQUIRE);
  if (sm == 0) {
    e = cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    __atomic_store_n(&g_sm_count[dev], sm, __ATOMIC_RELEASE);
  }
  li->device = dev;
  li->sm_count = sm;
  return KT_OK;
}

// x, y must be device (or managed) memory of the current device.
kt_status check_device_ptr(const void *p, int dev, const char *name) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(KT_ERR_ARG, "%s: not a CUDA pointer (%s)", name, cudaGetErrorName(e));
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    return fail(KT_ERR_ARG, "%s: not device memory", name);
  if (a.type == cudaMemoryTypeDevice && a.device != dev)
    return fail(KT_ERR_ARG, "%s lives on device %d, current device is %d", name, a.device, dev);
  return KT_OK;
}

kt_status check_buffers(const void *x, const void *y, size_t n, size_t es, kt::LaunchInfo *li) {
  if (!x || !y) return fail(KT_ERR_ARG, "NULL pointer with n = %zu", n);
  const uintptr_t xa = (uintptr_t)x, ya = (uintptr_t)y;
  if (xa % es || ya % es) return fail(KT_ERR_ARG, "pointers must be %zu-byte aligned", es);
  if (n > (SIZE_MAX / es)) return fail(KT_ERR_ARG, "n too large");
  const size_t bytes = n * es;
  if (x != y && xa < ya + bytes && ya < xa + bytes)
    return fail(KT_ERR_ARG, "x and y overlap without being equal");
  kt_status s = launch_info(li);
  if (s != KT_OK) return s;
  if ((s = check_device_ptr(x, li->device, "x")) != KT_OK) return s;
  if ((s = check_device_ptr(y, li->device, "y")) != KT_OK) return s;
  return KT_OK;
}

kt_status run_map(int op, int fmt, const void *x, void *y, size_t n, kt_lut lut, void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (op < 0 || op > 4 || fmt < 0 || fmt > 1 || (op == 4 && fmt != kt::FMT_F32))
    return fail(KT_ERR_ARG, "bad op/dtype");
  if (fmt == kt::FMT_BF16 || op == 4) {
    kt_status s = need_bf16(lut);
    if (s != KT_OK) return s;
  }
  if (n == 0) return KT_OK;
  const size_t es = fmt == kt::FMT_BF16 ? 2 : 4;
  kt::LaunchInfo li;
  kt_status s = check_buffers(x, y, n, es, &li);
  if (s != KT_OK) return s;
  cudaError_t e = kt::launch_map(op, fmt, x, y, n, lut->words, (cudaStream_t)stream, li);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KT_OK;
}

bool overlaps(const void *p, const void *q, size_t bytes) {
  const uintptr_t a = (uintptr_t)p, b = (uintptr_t)q;
  return p != q && a < b + bytes && b < a + bytes;
}

// [p, p + pb) and [q, q + qb) share a byte (ranges of different sizes).
bool spans_overlap(const void *p, size_t pb, const void *q, size_t qb) {
  const uintptr_t a = (uintptr_t)p, b = (uintptr_t)q;
  return pb != 0 && qb != 0 && a < b + qb && b < a + pb;
}

kt_status run_bwd(int op, int fmt, const void *a, const void *dy, void *dx, size_t n, kt_lut lut,
                  void *stream) {
  if (op < 0 || op > 3 || fmt < 0 || fmt > 1) return fail(KT_ERR_ARG, "bad op/dtype");
  if ((op == kt::OP_SWISH || op == kt::OP_GELU) && !lut)
    return fail(KT_ERR_ARG, "lut is NULL (needed to recompute K-TanH)");
  if (fmt == kt::FMT_BF16) {
    kt_status s = need_bf16(lut);
    if (s != KT_OK) return s;
  }
  if (n == 0) return KT_OK;
  const size_t es = fmt == kt::FMT_BF16 ? 2 : 4;
  if (!a || !dy || !dx) return fail(KT_ERR_ARG, "NULL pointer with n = %zu", n);
  if ((uintptr_t)a % es || (uintptr_t)dy % es || (uintptr_t)dx % es)
    return fail(KT_ERR_ARG, "pointers must be %zu-byte aligned", es);
  if (n > SIZE_MAX / es) return fail(KT_ERR_ARG, "n too large");
  const size_t bytes = n * es;
  if (overlaps(dx, a, bytes) || overlaps(dx, dy, bytes))
    return fail(KT_ERR_ARG, "dx overlaps an input without being equal to it");
  kt::LaunchInfo li;
  kt_status s = launch_info(&li);
  if (s != KT_OK) return s;
  if ((s = check_device_ptr(a, li.device, "a")) != KT_OK) return s;
  if ((s = check_device_ptr(dy, li.device, "dy")) != KT_OK) return s;
  if ((s = check_device_ptr(dx, li.device, "dx")) != KT_OK) return s;
  static const kt::LutWords kNoLut = {};
  cudaError_t e = kt::launch_bwd(op, fmt, a, dy, dx, n, lut ? lut->words : kNoLut,
                                 (cudaStream_t)stream, li);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KT_OK;
}

// ---- host-buffer path -------------------------------------------------------
// Role streams: [0] host->device copies, [1] kernels, [2] device->host copies,
// so each copy engine streams chunks back to back.  kBufs buffer pairs
// (dx, dy) rotate; per buffer b: ev_in (H2D done), ev_comp (kernel done, dx
// free), ev_out (D2H done, dy free).
constexpr int kStages = 3;
constexpr int kBufs = 3;
struct HostPipe {
  bool init = false;
  cudaStream_t st[kStages];
  cudaEvent_t fork, join[kStages];
  cudaEvent_t ev_in[kBufs], ev_comp[kBufs], ev_out[kBufs];
  // Device byte range each buffer slot last used, and whether its last
  // event is the D2H (ev_out) or, for the mapped-y mode, the kernel
  // (ev_comp).  Cross-call reuse guard: a call on another caller stream may
  // start while an earlier call still uses its slots; it waits for those
  // slots only if its own work region overlaps theirs.
  uintptr_t slot_lo[kBufs] = {}, slot_hi[kBufs] = {};
  bool slot_mapped[kBufs] = {};
  std::mutex mu;
};
HostPipe g_pipe[kMaxDev];

kt_status pipe_for(int dev, HostPipe **out) {
  HostPipe &p = g_pipe[dev];
  std::lock_guard<std::mutex> g(g_dev_mu);
  if (!p.init) {
    cudaError_t e;
    for (int i = 0; i < kStages; ++i)
      if ((e = cudaStreamCreateWithFlags(&p.st[i], cudaStreamNonBlocking)) != cudaSuccess)
        return cuda_fail(e, "cudaStreamCreate");
    cudaEvent_t *evs[] = {&p.fork, &p.join[0], &p.join[1], &p.join[2]};
    for (cudaEvent_t *ev : evs)
      if ((e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "cudaEventCreate");
    for (int i = 0; i < kBufs; ++i) {
      if ((e = cudaEventCreateWithFlags(&p.ev_in[i], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&p.ev_comp[i], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&p.ev_out[i], cudaEventDisableTiming)) != cudaSuccess)
        return cuda_fail(e, "cudaEventCreate");
    }
    p.init = true;
  }
  *out = &p;
  return KT_OK;
}

}  // namespace

extern "C" {

KT_API kt_status kt_lut_create(const int32_t E[32], const int32_t r[32], const int32_t b[32],
                               kt_lut *out) {
  if (!E || !r || !b || !out) return fail(KT_ERR_ARG, "NULL argument");
  kt_lut_s tmp;
  kt_status s = validate_and_pack(E, r, b, &tmp);
  if (s != KT_OK) return s;
  kt_lut_s *L = new (std::nothrow) kt_lut_s(tmp);
  if (!L) return fail(KT_ERR_ARG, "out of host memory");
  *out = L;
  return KT_OK;
}

KT_API kt_status kt_lut_create_f32(const int32_t E[32], const int32_t r[32], const int32_t b[32],
                                   kt_lut *out) {
  if (!E || !r || !b || !out) return fail(KT_ERR_ARG, "NULL argument");
  kt_lut_s tmp;
  kt_status s = validate_and_pack_f32(E, r, b, &tmp);
  if (s != KT_OK) return s;
  kt_lut_s *L = new (std::nothrow) kt_lut_s(tmp);
  if (!L) return fail(KT_ERR_ARG, "out of host memory");
  *out = L;
  return KT_OK;
}

KT_API kt_status kt_lut_create_optimized(int32_t p, int32_t bmin_zero, kt_lut *out) {
  if (!out) return fail(KT_ERR_ARG, "NULL argument");
  if (p != 7 && p != 23) return fail(KT_ERR_ARG, "p = %d: only 7 (BF16) and 23 (F32) tables", p);
  int32_t E[32], r[32], b[32];
  if (kt_status so = run_optimizer(3, p, bmin_zero, E, r, b)) return so;
  return p == 7 ? kt_lut_create(E, r, b, out) : kt_lut_create_f32(E, r, b, out);
}

KT_API kt_status kt_lut_mantissa_bits(kt_lut lut, int32_t *p) {
  if (!lut || !p) return fail(KT_ERR_ARG, "NULL argument");
  *p = lut->p;
  return KT_OK;
}

KT_API kt_status kt_lut_create_paper(kt_lut *out) {
  return kt_lut_create(kPaperE, kPaperR, kPaperB, out);
}

KT_API kt_status kt_lut_get(kt_lut lut, int32_t E[32], int32_t r[32], int32_t b[32]) {
  if (!lut || !E || !r || !b) return fail(KT_ERR_ARG, "NULL argument");
  memcpy(E, lut->E, sizeof(lut->E));
  memcpy(r, lut->r, sizeof(lut->r));
  memcpy(b, lut->b, sizeof(lut->b));
  return KT_OK;
}

KT_API void kt_lut_destroy(kt_lut lut) { delete lut; }

// ---- 64-interval tables -------------------
// Index t = ((E & 3) << 4) | (M >> 3): entry t covers the 8 mantissas
// m in [8v, 8v + 7], v = t & 15, of input exponent E_in(t) = 125 + (((t >> 4)
// + 3) & 3); for E_in = 128 only m <= 0x70 (|x| <= T2) is reachable.
KT_API kt_status kt_lut64_create(const int32_t E[64], const int32_t r[64], const int32_t b[64],
                                 kt_lut64 *out) {
  if (!E || !r || !b || !out) return fail(KT_ERR_ARG, "NULL argument");
  kt_lut64_s tmp;
  for (int t = 0; t < 64; ++t) {
    if (r[t] < 0 || r[t] > 7) return fail(KT_ERR_LUT, "r[%d] = %d outside [0, 7]", t, r[t]);
    if (E[t] < 1 || E[t] > 127) return fail(KT_ERR_LUT, "E[%d] = %d outside [1, 127]", t, E[t]);
    const int ei = 125 + (((t >> 4) + 3) & 3);
    const int v = t & 15;
    int lo = 8 * v, hi = 8 * v + 7;
    if (ei == 128) hi = hi < 0x70 ? hi : 0x70;   // only |x| <= 3.75 reaches the table
    for (int m = lo; m <= hi; ++m) {
      const int mo = (m >> r[t]) + b[t];
      if (mo < 0 || mo > 127)
        return fail(KT_ERR_LUT, "entry %d: (m=%d >> r=%d) + b=%d = %d leaves [0, 127]", t, m, r[t],
                    b[t], mo);
      if (E[t] == 127 && mo != 0)
        return fail(KT_ERR_LUT, "entry %d: E=127 with M_o=%d != 0 gives |y| > 1", t, mo);
    }
    tmp.E[t] = E[t];
    tmp.r[t] = r[t];
    tmp.b[t] = b[t];
    const int32_t d16 = (E[t] << 7) + b[t] - (1 << (7 - r[t]));
    tmp.words.w[t] = ((uint32_t)(ei + 16 + r[t]) << 23) | ((uint32_t)d16 & 0xFFFFu);
  }
  kt_lut64_s *L = new (std::nothrow) kt_lut64_s(tmp);
  if (!L) return fail(KT_ERR_ARG, "out of host memory");
  *out = L;
  return KT_OK;
}

KT_API kt_status kt_lut64_create_optimized(int32_t bmin_zero, kt_lut64 *out) {
  if (!out) return fail(KT_ERR_ARG, "NULL argument");
  int32_t E[64], r[64], b[64];
  if (kt_status so = run_optimizer(4, 7, bmin_zero, E, r, b)) return so;
  return kt_lut64_create(E, r, b, out);
}

KT_API kt_status kt_lut64_get(kt_lut64 lut, int32_t E[64], int32_t r[64], int32_t b[64]) {
  if (!lut || !E || !r || !b) return fail(KT_ERR_ARG, "NULL argument");
  memcpy(E, lut->E, sizeof(lut->E));
  memcpy(r, lut->r, sizeof(lut->r));
  memcpy(b, lut->b, sizeof(lut->b));
  return KT_OK;
}

KT_API void kt_lut64_destroy(kt_lut64 lut) { delete lut; }

KT_API kt_status ktanh64_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut64 lut, void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (n == 0) return KT_OK;
  kt::LaunchInfo li;
  kt_status s = check_buffers(x, y, n, 2, &li);
  if (s != KT_OK) return s;
  cudaError_t e = kt::launch_map64(x, y, n, lut->words, (cudaStream_t)stream, li);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KT_OK;
}

KT_API kt_status ktanh_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_TANH, kt::FMT_BF16, x, y, n, lut, stream);
}
KT_API kt_status ktanh_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_TANH, kt::FMT_F32, x, y, n, lut, stream);
}
KT_API kt_status ktanh_f32_via_bf16(const float *x, float *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_TANH_VIA_BF16, kt::FMT_F32, x, y, n, lut, stream);
}
KT_API kt_status ksigmoid_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_SIGMOID, kt::FMT_BF16, x, y, n, lut, stream);
}
KT_API kt_status ksigmoid_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_SIGMOID, kt::FMT_F32, x, y, n, lut, stream);
}
KT_API kt_status kswish_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_SWISH, kt::FMT_BF16, x, y, n, lut, stream);
}
KT_API kt_status kswish_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_SWISH, kt::FMT_F32, x, y, n, lut, stream);
}
KT_API kt_status kgelu_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_GELU, kt::FMT_BF16, x, y, n, lut, stream);
}
KT_API kt_status kgelu_f32(const float *x, float *y, size_t n, kt_lut lut, void *stream) {
  return run_map(kt::OP_GELU, kt::FMT_F32, x, y, n, lut, stream);
}

KT_API kt_status kt_apply(kt_op op, kt_dtype dtype, const void *x, void *y, size_t n, kt_lut lut,
                          void *stream) {
  if ((int)op < 0 || (int)op > 3) return fail(KT_ERR_ARG, "bad op %d", (int)op);
  return run_map((int)op, (int)dtype, x, y, n, lut, stream);
}

// ---- fused K-GELU + K-Swish (config 5, reading A20) -------------------------
static kt_status run_dual(int fmt, const void *x, void *yg, void *ys, size_t n, kt_lut lut,
                          void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (fmt == kt::FMT_BF16) {
    kt_status s = need_bf16(lut);
    if (s != KT_OK) return s;
  }
  if (n == 0) return KT_OK;
  const size_t es = fmt == kt::FMT_BF16 ? 2 : 4;
  if (!x || !yg || !ys) return fail(KT_ERR_ARG, "NULL pointer with n = %zu", n);
  if ((uintptr_t)x % es || (uintptr_t)yg % es || (uintptr_t)ys % es)
    return fail(KT_ERR_ARG, "pointers must be %zu-byte aligned", es);
  if (n > SIZE_MAX / es) return fail(KT_ERR_ARG, "n too large");
  const size_t bytes = n * es;
  if (yg == ys || overlaps(yg, ys, bytes)) return fail(KT_ERR_ARG, "y_gelu and y_swish overlap");
  if (overlaps(x, yg, bytes) || overlaps(x, ys, bytes))
    return fail(KT_ERR_ARG, "an output overlaps x without being equal to it");
  kt::LaunchInfo li;
  kt_status s = launch_info(&li);
  if (s != KT_OK) return s;
  if ((s = check_device_ptr(x, li.device, "x")) != KT_OK) return s;
  if ((s = check_device_ptr(yg, li.device, "y_gelu")) != KT_OK) return s;
  if ((s = check_device_ptr(ys, li.device, "y_swish")) != KT_OK) return s;
  cudaError_t e = kt::launch_dual(fmt, x, yg, ys, n, lut->words, (cudaStream_t)stream, li);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KT_OK;
}

KT_API kt_status kgelu_swish_bf16(const uint16_t *x, uint16_t *y_gelu, uint16_t *y_swish, size_t n,
                                  kt_lut lut, void *stream) {
  return run_dual(kt::FMT_BF16, x, y_gelu, y_swish, n, lut, stream);
}
KT_API kt_status kgelu_swish_f32(const float *x, float *y_gelu, float *y_swish, size_t n, kt_lut lut,
                                 void *stream) {
  return run_dual(kt::FMT_F32, x, y_gelu, y_swish, n, lut, stream);
}

// ---- Table 2 comparators --------------------------------
KT_API kt_status kt_apx_create(kt_apx_kind kind, int p, int q, kt_apx *out) {
  if (!out) return fail(KT_ERR_ARG, "NULL argument");
  if ((int)kind < 0 || (int)kind > 4) return fail(KT_ERR_ARG, "bad approximation kind %d", (int)kind);
  kt_apx_s tmp;
  char err[256];
  if (!kt::apx_build((int)kind, p, q, &tmp.words, tmp.coef, err, sizeof(err)))
    return fail(KT_ERR_ARG, "%s", err);
  kt_apx_s *A = new (std::nothrow) kt_apx_s(tmp);
  if (!A) return fail(KT_ERR_ARG, "out of host memory");
  *out = A;
  return KT_OK;
}

KT_API kt_status kt_apx_coeffs(kt_apx a, double coef[KT_APX_NCOEF]) {
  if (!a || !coef) return fail(KT_ERR_ARG, "NULL argument");
  memcpy(coef, a->coef, sizeof(a->coef));
  return KT_OK;
}

KT_API void kt_apx_destroy(kt_apx a) { delete a; }

static kt_status run_apx(int fmt, const void *x, void *y, size_t n, kt_apx a, void *stream) {
  if (!a) return fail(KT_ERR_ARG, "approximation handle is NULL");
  if (n == 0) return KT_OK;
  const size_t es = fmt == kt::FMT_BF16 ? 2 : 4;
  kt::LaunchInfo li;
  kt_status s = check_buffers(x, y, n, es, &li);
  if (s != KT_OK) return s;
  cudaError_t e = kt::launch_apx(fmt, x, y, n, a->words, (cudaStream_t)stream, li);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KT_OK;
}

KT_API kt_status kt_apx_tanh_bf16(const uint16_t *x, uint16_t *y, size_t n, kt_apx a, void *stream) {
  return run_apx(kt::FMT_BF16, x, y, n, a, stream);
}
KT_API kt_status kt_apx_tanh_f32(const float *x, float *y, size_t n, kt_apx a, void *stream) {
  return run_apx(kt::FMT_F32, x, y, n, a, stream);
}

KT_API kt_status kt_alu_probe(kt_dtype dtype, kt_lut lut, kt_apx apx, const void *sample_host,
                              int iters, double *cycles_net, double *cycles_gross) {
  if ((!lut) == (!apx)) return fail(KT_ERR_ARG, "pass exactly one of lut, apx");
  if ((int)dtype < 0 || (int)dtype > 1) return fail(KT_ERR_ARG, "bad dtype");
  if (dtype == KT_BF16)
    if (kt_status sb = need_bf16(lut)) return sb;
  if (!sample_host || !cycles_net || !cycles_gross || iters < 1)
    return fail(KT_ERR_ARG, "NULL argument or iters < 1");
  kt::LaunchInfo li;
  kt_status s = launch_info(&li);
  if (s != KT_OK) return s;
  static const kt::LutWords zero_lut = {};
  static const kt::ApxWords zero_apx = {};
  cudaError_t e = kt::alu_probe(lut ? 1 : 2, (int)dtype, lut ? lut->words : zero_lut,
                                apx ? apx->words : zero_apx, iters,
                                static_cast<const uint32_t *>(sample_host), cycles_net,
                                cycles_gross, li.sm_count);
  if (e != cudaSuccess) return cuda_fail(e, "kt_alu_probe");
  return KT_OK;
}

KT_API kt_status ktanh_bwd_bf16(const uint16_t *y, const uint16_t *dy, uint16_t *dx, size_t n,
                                void *stream) {
  return run_bwd(kt::OP_TANH, kt::FMT_BF16, y, dy, dx, n, nullptr, stream);
}
KT_API kt_status ktanh_bwd_f32(const float *y, const float *dy, float *dx, size_t n, void *stream) {
  return run_bwd(kt::OP_TANH, kt::FMT_F32, y, dy, dx, n, nullptr, stream);
}
KT_API kt_status ksigmoid_bwd_bf16(const uint16_t *s, const uint16_t *dy, uint16_t *dx, size_t n,
                                   void *stream) {
  return run_bwd(kt::OP_SIGMOID, kt::FMT_BF16, s, dy, dx, n, nullptr, stream);
}
KT_API kt_status ksigmoid_bwd_f32(const float *s, const float *dy, float *dx, size_t n, void *stream) {
  return run_bwd(kt::OP_SIGMOID, kt::FMT_F32, s, dy, dx, n, nullptr, stream);
}
KT_API kt_status kswish_bwd_bf16(const uint16_t *x, const uint16_t *dy, uint16_t *dx, size_t n,
                                 kt_lut lut, void *stream) {
  return run_bwd(kt::OP_SWISH, kt::FMT_BF16, x, dy, dx, n, lut, stream);
}
KT_API kt_status kswish_bwd_f32(const float *x, const float *dy, float *dx, size_t n, kt_lut lut,
                                void *stream) {
  return run_bwd(kt::OP_SWISH, kt::FMT_F32, x, dy, dx, n, lut, stream);
}
KT_API kt_status kgelu_bwd_bf16(const uint16_t *x, const uint16_t *dy, uint16_t *dx, size_t n,
                                kt_lut lut, void *stream) {
  return run_bwd(kt::OP_GELU, kt::FMT_BF16, x, dy, dx, n, lut, stream);
}
KT_API kt_status kgelu_bwd_f32(const float *x, const float *dy, float *dx, size_t n, kt_lut lut,
                               void *stream) {
  return run_bwd(kt::OP_GELU, kt::FMT_F32, x, dy, dx, n, lut, stream);
}
KT_API kt_status kt_apply_bwd(kt_op op, kt_dtype dtype, const void *a, const void *dy, void *dx,
                              size_t n, kt_lut lut, void *stream) {
  return run_bwd((int)op, (int)dtype, a, dy, dx, n, lut, stream);
}

KT_API kt_status klstm_gates_bf16(const uint16_t *x, uint16_t *y, size_t rows, size_t hidden,
                                  int tanh_quarter, kt_lut lut, void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (kt_status sb = need_bf16(lut)) return sb;
  if (hidden == 0) return fail(KT_ERR_ARG, "hidden == 0");
  if (tanh_quarter < 0 || tanh_quarter > 3) return fail(KT_ERR_ARG, "tanh_quarter not in 0..3");
  if (rows > SIZE_MAX / 4 / hidden) return fail(KT_ERR_ARG, "size overflow");
  const size_t n = rows * 4 * hidden;
  if (n == 0) return KT_OK;
  kt::LaunchInfo li;
  kt_status s = check_buffers(x, y, n, 2, &li);
  if (s != KT_OK) return s;
  cudaError_t e =
      kt::launch_lstm(x, y, rows, hidden, tanh_quarter, lut->words, (cudaStream_t)stream, li);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KT_OK;
}

KT_API kt_status klstm_cell_bf16(const uint16_t *gates, const float *c_prev, float *c_next,
                                 uint16_t *h_next, size_t rows, size_t hidden, kt_lut lut,
                                 void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (kt_status sb = need_bf16(lut)) return sb;
  if (hidden == 0) return fail(KT_ERR_ARG, "hidden == 0");
  if (rows > SIZE_MAX / 4 / hidden) return fail(KT_ERR_ARG, "size overflow");
  const size_t n = rows * hidden;
  if (n == 0) return KT_OK;
  if (!gates || !c_prev || !c_next || !h_next) return fail(KT_ERR_ARG, "NULL pointer");
  if ((uintptr_t)gates % 2 || (uintptr_t)h_next % 2 || (uintptr_t)c_prev % 4 || (uintptr_t)c_next % 4)
    return fail(KT_ERR_ARG, "misaligned pointer");
  // gates n*8 B, c_prev / c_next n*4 B, h_next n*2 B; only c_next == c_prev may alias
  if (overlaps(c_next, c_prev, n * 4) || spans_overlap(c_next, n * 4, gates, n * 8) ||
      spans_overlap(h_next, n * 2, gates, n * 8) || spans_overlap(h_next, n * 2, c_prev, n * 4) ||
      spans_overlap(h_next, n * 2, c_next, n * 4))
    return fail(KT_ERR_ARG, "outputs overlap inputs (only c_next == c_prev is allowed)");
  kt::LaunchInfo li;
  kt_status s = launch_info(&li);
  if (s != KT_OK) return s;
  if ((s = check_device_ptr(gates, li.device, "gates")) != KT_OK) return s;
  if ((s = check_device_ptr(c_prev, li.device, "c_prev")) != KT_OK) return s;
  if ((s = check_device_ptr(c_next, li.device, "c_next")) != KT_OK) return s;
  if ((s = check_device_ptr(h_next, li.device, "h_next")) != KT_OK) return s;
  cudaError_t e = kt::launch_lstm_cell(gates, c_prev, c_next, h_next, rows, hidden, lut->words,
                                       (cudaStream_t)stream, li);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KT_OK;
}

static kt_status run_gemm(int epilogue, const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M,
                          size_t N, size_t K, kt_lut lut, void *stream, uint32_t lstm_hidden,
                          uint32_t lstm_tq) {
  if (epilogue >= 0 && !lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (epilogue >= 0)
    if (kt_status sb = need_bf16(lut)) return sb;
  if (M == 0 || N == 0) return KT_OK;
  if (M % 128 || N % 256 || K % 64 || K == 0)
    return fail(KT_ERR_ARG, "kgemm needs M %% 128 == 0, N %% 256 == 0, K %% 64 == 0 (K > 0)");
  if (M > (1u << 31) || N > (1u << 31) || K > (1u << 31)) return fail(KT_ERR_ARG, "size too large");
  if (!A || !B || !C) return fail(KT_ERR_ARG, "NULL pointer");
  if ((uintptr_t)A % 16 || (uintptr_t)B % 16 || (uintptr_t)C % 32)
    return fail(KT_ERR_ARG, "A, B must be 16-byte and C 32-byte aligned");
  if (((uintptr_t)C < (uintptr_t)A + M * K * 2 && (uintptr_t)A < (uintptr_t)C + M * N * 2) ||
      ((uintptr_t)C < (uintptr_t)B + N * K * 2 && (uintptr_t)B < (uintptr_t)C + M * N * 2))
    return fail(KT_ERR_ARG, "C overlaps A or B");
  kt::LaunchInfo li;
  kt_status s = launch_info(&li);
  if (s != KT_OK) return s;
  if ((s = check_device_ptr(A, li.device, "A")) != KT_OK) return s;
  if ((s = check_device_ptr(B, li.device, "B")) != KT_OK) return s;
  if ((s = check_device_ptr(C, li.device, "C")) != KT_OK) return s;
  static const kt::LutWords kNoLut = {};
  cudaError_t e = kt::launch_gemm(epilogue, A, B, C, M, N, K, lut ? lut->words : kNoLut,
                                  (cudaStream_t)stream, li.sm_count, lstm_hidden, lstm_tq);
  if (e != cudaSuccess) return cuda_fail(e, "kgemm launch");
  return KT_OK;
}

KT_API kt_status kgemm_bf16(const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M, size_t N,
                            size_t K, int epilogue, kt_lut lut, void *stream) {
  if (epilogue < -1 || epilogue > 3) return fail(KT_ERR_ARG, "epilogue must be -1 or a kt_op");
  return run_gemm(epilogue, A, B, C, M, N, K, lut, stream, 0, 0);
}

KT_API kt_status kgemm_lstm_gates_bf16(const uint16_t *A, const uint16_t *B, uint16_t *C, size_t M,
                                       size_t hidden, size_t K, int tanh_quarter, kt_lut lut,
                                       void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (hidden == 0 || hidden % 256 || hidden > (1u << 29))
    return fail(KT_ERR_ARG, "hidden must be a positive multiple of 256");
  if (tanh_quarter < 0 || tanh_quarter > 3) return fail(KT_ERR_ARG, "tanh_quarter must be 0..3");
  return run_gemm(8, A, B, C, M, 4 * hidden, K, lut, stream, (uint32_t)hidden, (uint32_t)tanh_quarter);
}

KT_API kt_status kgemm_lstm_cell_bf16(const uint16_t *A, const uint16_t *B, const float *c_prev,
                                      float *c_next, uint16_t *h_next, size_t M, size_t hidden,
                                      size_t K, kt_lut lut, void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if (kt_status sb = need_bf16(lut)) return sb;
  if (M == 0 || hidden == 0) return KT_OK;
  if (M % 128 || hidden % 64 || K % 64 || K == 0)
    return fail(KT_ERR_ARG, "needs M %% 128 == 0, hidden %% 64 == 0, K %% 64 == 0 (K > 0)");
  if (M > (1u << 31) || 4 * hidden > (1u << 31) || K > (1u << 31)) return fail(KT_ERR_ARG, "too large");
  if (!A || !B || !c_prev || !c_next || !h_next) return fail(KT_ERR_ARG, "NULL pointer");
  if ((uintptr_t)A % 16 || (uintptr_t)B % 16 || (uintptr_t)c_prev % 32 || (uintptr_t)c_next % 32 ||
      (uintptr_t)h_next % 32)
    return fail(KT_ERR_ARG, "A, B must be 16-byte and c_prev, c_next, h_next 32-byte aligned");
  const size_t cb = M * hidden * 4, hb = M * hidden * 2;
  if (overlaps(c_next, c_prev, cb)) return fail(KT_ERR_ARG, "c_next overlaps c_prev without being equal");
  if (spans_overlap(h_next, hb, c_next, cb)) return fail(KT_ERR_ARG, "h_next overlaps c_next");
  const void *ins[3] = {A, B, c_prev};
  const size_t inb[3] = {M * K * 2, 4 * hidden * K * 2, cb};
  for (int j = 0; j < 3; ++j) {
    const uintptr_t p0 = (uintptr_t)ins[j], p1 = p0 + inb[j];
    const uintptr_t h0 = (uintptr_t)h_next, h1 = h0 + hb;
    if (h0 < p1 && p0 < h1) return fail(KT_ERR_ARG, "h_next overlaps an input");
    if (j < 2) {
      const uintptr_t c0 = (uintptr_t)c_next, c1 = c0 + cb;
      if (c0 < p1 && p0 < c1) return fail(KT_ERR_ARG, "c_next overlaps A or B");
    }
  }
  kt::LaunchInfo li;
  kt_status s = launch_info(&li);
  if (s != KT_OK) return s;
  const void *dev_ptrs[5] = {A, B, c_prev, c_next, h_next};
  const char *names[5] = {"A", "B", "c_prev", "c_next", "h_next"};
  for (int j = 0; j < 5; ++j)
    if ((s = check_device_ptr(dev_ptrs[j], li.device, names[j])) != KT_OK) return s;
  cudaError_t e = kt::launch_gemm_cell(A, B, c_prev, c_next, h_next, M, hidden, K, lut->words,
                                       (cudaStream_t)stream, li.sm_count);
  if (e != cudaSuccess) return cuda_fail(e, "kgemm_lstm_cell launch");
  return KT_OK;
}

// Host-buffer strategy (KT_HOST_ZEROCOPY): 0 = copy-engine pipeline,
// 1 = one zero-copy kernel, 2 = hybrid (copy-engine H2D, the kernel stores
// its output straight into the mapped host buffer).  Default: see
// kt_apply_host.
static int host_mode() {
  const char *e = getenv("KT_HOST_ZEROCOPY");   // read per call (tests switch it)
  const int m = e ? atoi(e) : 0;
  return (m == 1 || m == 2) ? m : 0;
}

// Device address of a pinned, mapped host buffer; NULL for pageable memory
// or a host allocation that is not mapped into the current device.
static const void *mapped_device_ptr(const void *h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer) return nullptr;
  return a.devicePointer;
}

KT_API kt_status kt_apply_host_ex(kt_op op, kt_dtype dtype, const void *x_host, void *y_host,
                                  size_t n, kt_lut lut, void *d_work, size_t work_bytes,
                                  size_t chunk_elems, void *stream);

KT_API kt_status kt_apply_host(kt_op op, kt_dtype dtype, const void *x_host, void *y_host, size_t n,
                               kt_lut lut, void *d_work, size_t work_bytes, void *stream) {
  return kt_apply_host_ex(op, dtype, x_host, y_host, n, lut, d_work, work_bytes, 0, stream);
}

KT_API kt_status kt_apply_host_ex(kt_op op, kt_dtype dtype, const void *x_host, void *y_host,
                                  size_t n, kt_lut lut, void *d_work, size_t work_bytes,
                                  size_t chunk_elems, void *stream) {
  if (!lut) return fail(KT_ERR_ARG, "lut is NULL");
  if ((int)op < 0 || (int)op > 3 || (int)dtype < 0 || (int)dtype > 1)
    return fail(KT_ERR_ARG, "bad op/dtype");
  if (dtype == KT_BF16)
    if (kt_status sb = need_bf16(lut)) return sb;

  if (n == 0) return KT_OK;
  if (!x_host || !y_host) return fail(KT_ERR_ARG, "NULL pointer");
  const size_t es = dtype == KT_BF16 ? 2 : 4;
  if (n > SIZE_MAX / es) return fail(KT_ERR_ARG, "n too large");
  {
    const uintptr_t xa = (uintptr_t)x_host, ya = (uintptr_t)y_host;
    if (xa % es || ya % es) return fail(KT_ERR_ARG, "pointers must be %zu-byte aligned", es);
    if (x_host != y_host && xa < ya + n * es && ya < xa + n * es)
      return fail(KT_ERR_ARG, "x_host and y_host overlap without being equal");
  }
  // Zero-copy path (KT_HOST_ZEROCOPY=1): when both host buffers are pinned
  // and mapped into the device address space (cudaHostAlloc / torch
  // pin_memory under UVA), ONE kernel reads x over PCIe, applies the op and
  // writes y back over PCIe.  Measured on B200 (profiles/host_path_r01.txt):
  // SM-initiated traffic tops out at ~80 GB/s read+write vs ~96 GB/s for the
  // two copy engines, and the hybrid (mode 2) is within noise of the
  // pipeline, so the copy-engine pipeline is the default.
  const int mode = host_mode();
  void *y_mapped = mode ? const_cast<void *>(mapped_device_ptr(y_host)) : nullptr;
  if (mode == 1) {
    const void *xd = mapped_device_ptr(x_host);
    if (xd && y_mapped) {
      kt::LaunchInfo li;
      kt_status s = launch_info(&li);
      if (s != KT_OK) return s;
      cudaError_t e = kt::launch_map((int)op, (int)dtype, xd, y_mapped, n, lut->words,
                                     (cudaStream_t)stream, li, /*sysmem=*/true);
      if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
      return KT_OK;
    }
  }
  if (!d_work) return fail(KT_ERR_ARG, "NULL pointer");
  size_t chunk = work_bytes / (2 * kBufs * es);
  chunk -= chunk % 256;
  if (chunk < 4096)
    return fail(KT_ERR_ARG, "work_bytes too small (need >= %zu)", 2 * kBufs * es * 4096);
  // ~3 chunks per call (one per buffer slot, at least 1 MiB each): within a
  // call the copy directions and the kernel overlap chunk by chunk, and calls
  // on different caller streams overlap each other's fill/drain, where fewer,
  // larger copies run closer to the PCIe rate (config 2 end to end: 8 chunks
  // 19.9, 4 chunks 22.0, 3 chunks 22.6 Gelem/s; profiles/host_path_r01.txt).
  size_t want = ((n + kBufs - 1) / kBufs + 255) / 256 * 256;
  const size_t min_chunk = ((size_t)1 << 20) / es;
  if (want < min_chunk) want = min_chunk;
  if (chunk_elems) {                                // caller's choice (elements)
    if (chunk_elems < 4096) return fail(KT_ERR_ARG, "chunk_elems must be 0 or >= 4096");
    want = chunk_elems - chunk_elems % 256;
  } else if (const char *ev = getenv("KT_HOST_CHUNK")) {   // tuning override (elements)
    const size_t c = (size_t)strtoull(ev, nullptr, 10);
    if (c >= 4096) want = c - c % 256;
  }
  if (want < chunk) chunk = want;
  kt::LaunchInfo li;
  kt_status s = launch_info(&li);
  if (s != KT_OK) return s;
  if ((s = check_device_ptr(d_work, li.device, "d_work")) != KT_OK) return s;
  HostPipe *p;
  if ((s = pipe_for(li.device, &p)) != KT_OK) return s;
  std::lock_guard<std::mutex> g(p->mu);
  cudaStream_t caller = (cudaStream_t)stream;
  cudaStream_t h2d = p->st[0], comp = p->st[1], d2h = p->st[2];
  cudaError_t e;
#define KT_CK(call, what) \
  if ((e = (call)) != cudaSuccess) return cuda_fail(e, what);
  KT_CK(cudaEventRecord(p->fork, caller), "cudaEventRecord");
  for (int i = 0; i < kStages; ++i) KT_CK(cudaStreamWaitEvent(p->st[i], p->fork, 0), "cudaStreamWaitEvent");
  const char *xh = static_cast<const char *>(x_host);
  char *yh = static_cast<char *>(y_host);
  char *work = static_cast<char *>(d_work);
  {
    // earlier calls (possibly on other caller streams) whose slots overlap
    // this call's work region must be done with them before our first H2D;
    // later H2Ds, kernels and D2Hs of this call follow it in stream order
    const uintptr_t lo = (uintptr_t)work, hi = lo + (uintptr_t)kBufs * 2 * chunk * es;
    for (int j = 0; j < kBufs; ++j) {
      if (p->slot_hi[j] > lo && p->slot_lo[j] < hi)
        KT_CK(cudaStreamWaitEvent(h2d, p->slot_mapped[j] ? p->ev_comp[j] : p->ev_out[j], 0), "wait");
    }
  }
  size_t k = 0;
  for (size_t off = 0; off < n; off += chunk, ++k) {
    const size_t cnt = (n - off < chunk) ? n - off : chunk;
    const int b = (int)(k % kBufs);
    char *dx = work + (size_t)b * 2 * chunk * es;
    // hybrid (mode 2): the kernel stores straight into the mapped y_host
    char *dy = y_mapped ? static_cast<char *>(y_mapped) + off * es : dx + chunk * es;
    if (k >= (size_t)kBufs) KT_CK(cudaStreamWaitEvent(h2d, p->ev_comp[b], 0), "wait");  // dx free
    KT_CK(cudaMemcpyAsync(dx, xh + off * es, cnt * es, cudaMemcpyHostToDevice, h2d), "H2D");
    KT_CK(cudaEventRecord(p->ev_in[b], h2d), "record");
    KT_CK(cudaStreamWaitEvent(comp, p->ev_in[b], 0), "wait");
    if (k >= (size_t)kBufs && !y_mapped)
      KT_CK(cudaStreamWaitEvent(comp, p->ev_out[b], 0), "wait");  // dy free
    KT_CK(kt::launch_map((int)op, (int)dtype, dx, dy, cnt, lut->words, comp, li), "kernel launch");
    KT_CK(cudaEventRecord(p->ev_comp[b], comp), "record");
    p->slot_lo[b] = (uintptr_t)dx;
    p->slot_hi[b] = (uintptr_t)dx + 2 * chunk * es;
    p->slot_mapped[b] = y_mapped != nullptr;
    if (y_mapped) continue;
    KT_CK(cudaStreamWaitEvent(d2h, p->ev_comp[b], 0), "wait");
    KT_CK(cudaMemcpyAsync(yh + off * es, dy, cnt * es, cudaMemcpyDeviceToHost, d2h), "D2H");
    KT_CK(cudaEventRecord(p->ev_out[b], d2h), "record");
  }
  for (int i = 0; i < kStages; ++i) {
    KT_CK(cudaEventRecord(p->join[i], p->st[i]), "record");
    KT_CK(cudaStreamWaitEvent(caller, p->join[i], 0), "wait");
  }
#undef KT_CK
  return KT_OK;
}

KT_API kt_status kt_shard_range(size_t n, int world, int rank, size_t align, size_t *begin,
                                size_t *count) {
  if (world < 1 || rank < 0 || rank >= world || align == 0 || !begin || !count)
    return fail(KT_ERR_ARG, "bad shard arguments");
  size_t per = n / (size_t)world + (n % (size_t)world != 0);
  per = (per + align - 1) / align * align;
  size_t b = per * (size_t)rank;
  if (b > n) b = n;
  size_t c = n - b;
  if (c > per) c = per;
  *begin = b;
  *count = c;
  return KT_OK;
}

KT_API const char *kt_status_string(kt_status s) {
  switch (s) {
    case KT_OK: return "KT_OK";
    case KT_ERR_ARG: return "KT_ERR_ARG";
    case KT_ERR_LUT: return "KT_ERR_LUT";
    case KT_ERR_CUDA: return "KT_ERR_CUDA";
  }
  return "KT_UNKNOWN";
}

KT_API const char *kt_last_error(void) { return g_err.c_str(); }
KT_API int kt_abi_version(void) { return KT_ABI_VERSION; }
KT_API uint64_t kt_launch_count(void) { return kt::launch_count(); }

}  // extern "C"
