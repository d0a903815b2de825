// kt_tables.cu -- host-side Sec. 2.4 table optimizer for
// kt_lut_create_optimized: the parameter tables (T_E, T_r, T_b) of Alg. 1
// line 1 computed from tanh itself, for p = 7 (BFloat16, the paper's case)
// or p = 23 (an F32-native table).  Readings A12-A17 of
// DESIGN.md §3 fix the steps the text leaves open; the test oracle has its
// own implementation (oracle/ktanh_oracle.c kto_build_lut_sp) and
// tests/test_abi_cpu.py checks the two produce identical tables.
//
// Per interval t (index bits: 2 exponent LSBs, s mantissa MSBs):
//   inputs  x = 2^(E_in - 127) (1 + m / 2^p), T1 <= x <= T2, m in the
//           interval's mantissa range (one input exponent E_in per t);
//   Step 1  y = tanh(x) (binary64), (E_y, M_y) = fields of RNE_p(y)   [A12]
//   Step 2  E_t = argmin over the distinct min(E_y, 126) of
//           sum (y - yhat)^2, yhat = 2^(E_t-127)(1 + Mhat/2^p) with Mhat =
//           M_y (same exponent), 0 (E_t above), 2^p - 1 (E_t below);
//           ties -> smaller E_t                                     [A15]
//   Step 3  for r = 0..p: b = floor(mean(Mhat - m / 2^r) + 1/2)  [A13, A14]
//           clamped to [b_min, b_max] (Eq. 3), score sum (Mhat - (m >> r)
//           - b)^2; keep the smallest score, ties -> smaller r      [A17]
// All of Step 3 is exact integer arithmetic (128-bit accumulators).
// Intervals are independent and run on host threads.
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "kt_internal.h"

namespace kt {

namespace {

struct Row {
  int E, r, b;
};

// RNE of y in (0, 1) to p mantissa bits: biased exponent and mantissa.
void round_fields(double y, int p, int *E, int64_t *M) {
  int k;
  const double f = std::frexp(y, &k);                    // y = f 2^k, f in [0.5, 1)
  int e = k - 1 + 127;
  double mr = std::nearbyint(std::ldexp(2.0 * f - 1.0, p));   // default mode: ties to even
  int64_t m = (int64_t)mr;
  if (m == ((int64_t)1 << p)) {
    m = 0;
    e += 1;
  }
  *E = e;
  *M = m;
}

__int128 floor_div128(__int128 a, __int128 d) {   // d > 0
  __int128 q = a / d;
  if (a % d != 0 && a < 0) --q;
  return q;
}

Row optimize_interval(int t, int s, int p, bool bmin_zero) {
  const int e_in = 125 + (((t >> s) + 3) & 3);           // E & 3 = t >> s, T1 <= x <= T2
  const int v = t & ((1 << s) - 1);
  const int64_t span = (int64_t)1 << (p - s);
  const int64_t m0 = (int64_t)v * span;
  std::vector<double> y;
  std::vector<int> ey;
  std::vector<int64_t> my;
  y.reserve(span);
  ey.reserve(span);
  my.reserve(span);
  for (int64_t j = 0; j < span; ++j) {
    const double x = std::ldexp(1.0 + std::ldexp((double)(m0 + j), -p), e_in - 127);
    if (x < 0.25 || x > 3.75) continue;                 // T1, T2
    const double yt = std::tanh(x);
    int E;
    int64_t M;
    round_fields(yt, p, &E, &M);
    y.push_back(yt);
    ey.push_back(E);
    my.push_back(M);
  }
  const size_t cnt = y.size();
  if (cnt == 0) return Row{126, 0, 0};
  const int64_t mfull = ((int64_t)1 << p) - 1;

  // Step 2
  int bestE = -1;
  double bestSSE = INFINITY;
  int cands[4], nc = 0;
  for (size_t c = 0; c < cnt; ++c) {
    const int E = ey[c] < 126 ? ey[c] : 126;
    bool seen = false;
    for (int k = 0; k < nc; ++k) seen = seen || cands[k] == E;
    if (seen || nc == 4) continue;
    cands[nc++] = E;
    double sse = 0.0;
    for (size_t j = 0; j < cnt; ++j) {
      const int64_t mh = E == ey[j] ? my[j] : (E > ey[j] ? 0 : mfull);
      const double yh = std::ldexp(1.0 + std::ldexp((double)mh, -p), E - 127);
      sse += (y[j] - yh) * (y[j] - yh);
    }
    if (sse < bestSSE || (sse == bestSSE && E < bestE)) {
      bestSSE = sse;
      bestE = E;
    }
  }
  std::vector<int64_t> mhat(cnt);
  for (size_t j = 0; j < cnt; ++j) mhat[j] = bestE == ey[j] ? my[j] : (bestE > ey[j] ? 0 : mfull);

  // Step 3
  Row best{bestE, -1, 0};
  __int128 bestScore = -1;
  for (int r = 0; r <= p; ++r) {
    __int128 sum_scaled = 0, sd = 0, sdd = 0;   // sum(mhat 2^r - m), sum d, sum d^2
    for (size_t j = 0; j < cnt; ++j) {
      const int64_t m = m0 + (int64_t)j;
      sum_scaled += ((__int128)mhat[j] << r) - m;
      const int64_t d = mhat[j] - (m >> r);
      sd += d;
      sdd += (__int128)d * d;
    }
    int64_t b = (int64_t)floor_div128(2 * sum_scaled + ((__int128)cnt << r), (__int128)cnt << (r + 1));
    // Eq. 3 bounds with p mantissa and s index bits
    const int64_t bmax = mfull - ((((int64_t)(v + 1)) << (p - s)) - 1 >> r);
    const int64_t bmin = bmin_zero ? 0 : (r <= p - s ? -(int64_t)v * ((int64_t)1 << (p - s - r)) : 0);
    if (b < bmin) b = bmin;
    if (b > bmax) b = bmax;
    const __int128 score = sdd - 2 * (__int128)b * sd + (__int128)cnt * b * b;
    if (bestScore < 0 || score < bestScore) {
      bestScore = score;
      best.r = r;
      best.b = (int)b;
    }
  }
  return best;
}

}  // namespace

bool optimize_table(int s, int p, bool bmin_zero, int32_t *E, int32_t *r, int32_t *b) {
  if ((p != 7 && p != 23) || s < 1 || s > 5) return false;
  const int n = 4 << s;
  std::vector<Row> rows(n);
  unsigned nt = std::thread::hardware_concurrency();
  nt = nt == 0 ? 1 : (nt > (unsigned)n ? (unsigned)n : nt);
  if (p == 7) nt = 1;                                    // 16 points per interval
  std::vector<std::thread> pool;
  for (unsigned k = 0; k < nt; ++k)
    pool.emplace_back([&, k] {
      for (int t = (int)k; t < n; t += (int)nt) rows[t] = optimize_interval(t, s, p, bmin_zero);
    });
  for (auto &th : pool) th.join();
  for (int t = 0; t < n; ++t) {
    E[t] = rows[t].E;
    r[t] = rows[t].r;
    b[t] = rows[t].b;
  }
  return true;
}

}  // namespace kt
