// Host scheduler: minimal-recomputation reversal schedules, bit-exact with
// the reference scheduler (pkg/src/asyncckpt/schedule.py).
//
// Cost model (schedule.py:17-27):
//   c[s][0] = 0, c[s][1] = 1, c[s][n] = n for n <= s+1,
//   c[0][n] = INF for n >= 2,
//   c[s][n] = min_{0<k<n} k + c[s-1][n-k] + c[s][k] otherwise.
//
// The reference builds that table with one numpy pass per cell, O(s n^2)
// (schedule.py:139-155).  Here the table is int32 with saturation at CAP and
// rows are built by a team of threads in a software pipeline: row s only
// needs row s-1 up to column n-1 to produce column n, so thread t owns rows
// t+1, t+1+T, ... and spins on its predecessor's progress counter.  The inner
// min over k runs over two forward-contiguous int32 arrays and vectorises.
//
// Saturation is exact for every value below CAP: a candidate whose true sum is
// below CAP has all of its terms below CAP, so it is stored exactly, and every
// candidate holding a saturated term sums to >= CAP.  Minima and first
// argmins (_best_split, schedule.py:177-181) are therefore unchanged.  Row 1 is
// the only row that exceeds CAP inside the supported range, and its exact
// value is closed-form: c[1][n] = n(n+1)/2 - 1 (schedule.py:26-27).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <queue>
#include <thread>
#include <vector>

#include "common.h"

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace ackpt {
namespace {

constexpr int64_t kInf = int64_t(1) << 40;  // schedule.py:45
constexpr int32_t kCap = int32_t(1) << 29;   // int32 saturation point

std::atomic<int> g_threads{0};

struct CostTable {
  int64_t n_max = 0, s_max = 0;
  // c[s*(n_max+1) + n], saturated at kCap.  Row 0 holds kCap for n >= 2.
  std::vector<int32_t> c;
  // ra[s*(n_max+1) + (n_max - k)] = min(k + c[s][k], kCap + n_max): the
  // "k + cost(k, s)" term stored reversed so the inner loop walks forward.
  std::vector<int32_t> ra;
  bool overflow = false;  // some row >= 2 saturated: exact values unavailable

  int32_t at(int64_t s, int64_t n) const { return c[size_t(s) * size_t(n_max + 1) + size_t(n)]; }

  int64_t exact(int64_t s, int64_t n) const {
    if (n == 0) return 0;
    if (n == 1) return 1;
    if (n <= s + 1) return n;
    if (s == 0) return kInf;
    if (s == 1) return n * (n + 1) / 2 - 1;
    int32_t v = at(s, n);
    if (v >= kCap) fail(ACKPT_VALUE_ERROR, "cost table exceeds the int32 range for this (n, s)");
    return v;
  }
};

inline int32_t min_row(const int32_t* __restrict a, const int32_t* __restrict b, int64_t len) {
  // min over m in [0, len) of a[m] + b[m]; both arrays ascend in memory.
  int64_t m = 0;
  int32_t best = INT32_MAX;
#if defined(__AVX2__)
  __m256i vb = _mm256_set1_epi32(INT32_MAX);
  for (; m + 32 <= len; m += 32) {
    __m256i s0 = _mm256_add_epi32(_mm256_loadu_si256((const __m256i*)(a + m)),
                                  _mm256_loadu_si256((const __m256i*)(b + m)));
    __m256i s1 = _mm256_add_epi32(_mm256_loadu_si256((const __m256i*)(a + m + 8)),
                                  _mm256_loadu_si256((const __m256i*)(b + m + 8)));
    __m256i s2 = _mm256_add_epi32(_mm256_loadu_si256((const __m256i*)(a + m + 16)),
                                  _mm256_loadu_si256((const __m256i*)(b + m + 16)));
    __m256i s3 = _mm256_add_epi32(_mm256_loadu_si256((const __m256i*)(a + m + 24)),
                                  _mm256_loadu_si256((const __m256i*)(b + m + 24)));
    vb = _mm256_min_epi32(vb, _mm256_min_epi32(_mm256_min_epi32(s0, s1), _mm256_min_epi32(s2, s3)));
  }
  for (; m + 8 <= len; m += 8) {
    __m256i s0 = _mm256_add_epi32(_mm256_loadu_si256((const __m256i*)(a + m)),
                                  _mm256_loadu_si256((const __m256i*)(b + m)));
    vb = _mm256_min_epi32(vb, s0);
  }
  alignas(32) int32_t lanes[8];
  _mm256_store_si256((__m256i*)lanes, vb);
  for (int i = 0; i < 8; ++i) best = std::min(best, lanes[i]);
#endif
  for (; m < len; ++m) best = std::min(best, a[m] + b[m]);
  return best;
}

std::unique_ptr<CostTable> build_table(int64_t n_max, int64_t s_max) {
  auto t = std::make_unique<CostTable>();
  t->n_max = n_max;
  t->s_max = s_max;
  const size_t W = size_t(n_max + 1);
  t->c.assign(size_t(s_max + 1) * W, kCap);
  t->ra.assign(size_t(s_max + 1) * W, kCap);
  // Trivial part of every row (schedule.py:141-147).
  for (int64_t s = 0; s <= s_max; ++s) {
    int32_t* row = &t->c[size_t(s) * W];
    row[0] = 0;
    if (n_max >= 1) row[1] = 1;
    int64_t top = std::min(s + 1, n_max);
    for (int64_t n = 2; n <= top; ++n) row[n] = int32_t(std::min<int64_t>(n, kCap));
  }
  auto set_ra = [&](int64_t s, int64_t k) {
    int64_t v = k + int64_t(t->c[size_t(s) * W + size_t(k)]);
    t->ra[size_t(s) * W + size_t(n_max - k)] = int32_t(std::min<int64_t>(v, int64_t(kCap) + n_max));
  };
  for (int64_t k = 1; k <= std::min<int64_t>(n_max, 1); ++k) set_ra(0, k);

  // Rows needing the DP: s in [1, s_max] with s + 2 <= n_max.
  const int64_t dp_rows = std::min(s_max, n_max - 2);
  if (dp_rows >= 1) {
    int nthreads = g_threads.load();
    if (nthreads <= 0) nthreads = int(std::max(1u, std::thread::hardware_concurrency()));
    // Small tables are faster on one thread.
    if (double(dp_rows) * double(n_max) * double(n_max) < 4e6) nthreads = 1;
    nthreads = int(std::min<int64_t>(nthreads, dp_rows));
    std::vector<std::atomic<int64_t>> progress(size_t(s_max + 1));
    for (auto& p : progress) p.store(n_max + 1, std::memory_order_relaxed);
    // Row 0 is complete; DP rows start "done up to s+1".
    for (int64_t s = 1; s <= dp_rows; ++s) progress[size_t(s)].store(s + 1, std::memory_order_relaxed);
    std::atomic<bool> saturated{false};

    auto worker = [&](int tid) {
      for (int64_t s = 1 + tid; s <= dp_rows; s += nthreads) {
        int32_t* row = &t->c[size_t(s) * W];
        const int32_t* prev = &t->c[size_t(s - 1) * W];
        const int32_t* ra_s = &t->ra[size_t(s) * W];
        // ra for the trivial prefix of row s: k in [1, s+1].
        for (int64_t k = 1; k <= std::min(s + 1, n_max); ++k) set_ra(s, k);
        const std::atomic<int64_t>& prev_done = progress[size_t(s - 1)];
        for (int64_t n = s + 2; n <= n_max; ++n) {
          // Column n needs prev[1 .. n-1] (prev row is complete when s == 1).
          if (s > 1) {
            while (prev_done.load(std::memory_order_acquire) < n - 1) {
#if defined(__x86_64__)
              _mm_pause();
#endif
            }
          }
          // min_{k=1}^{n-1} (k + c[s][k]) + c[s-1][n-k]; with m = n - k:
          // (k + c[s][k]) = ra_s[n_max - n + m], c[s-1][m] = prev[m], m = 1..n-1.
          int32_t v = min_row(ra_s + (n_max - n + 1), prev + 1, n - 1);
          if (v >= kCap) {
            v = kCap;
            if (s >= 2) saturated.store(true, std::memory_order_relaxed);
          }
          row[n] = v;
          set_ra(s, n);
          progress[size_t(s)].store(n, std::memory_order_release);
        }
        progress[size_t(s)].store(n_max + 1, std::memory_order_release);
      }
    };
    if (nthreads == 1) {
      worker(0);
    } else {
      std::vector<std::thread> team;
      for (int i = 1; i < nthreads; ++i) team.emplace_back(worker, i);
      worker(0);
      for (auto& th : team) th.join();
    }
    t->overflow = saturated.load();
  }
  return t;
}

// Grow-on-demand cache (schedule.py:121-136).  Values do not depend on the
// table's extent, so a covering table answers any smaller query; a handful
// of recent tables are kept so alternating small/large queries do not force
// rebuilds of the largest one.
struct TableCache {
  std::mutex mu;
  std::vector<std::shared_ptr<CostTable>> tables;

  std::shared_ptr<CostTable> ensure(int64_t n, int64_t s) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& t : tables)
      if (t->n_max >= n && t->s_max >= s) return t;
    // Build the union extent of the largest table and the query only when
    // that stays cheap; otherwise build exactly what is asked.
    std::shared_ptr<CostTable> t(build_table(n, s).release());
    tables.push_back(t);
    if (tables.size() > 4) tables.erase(tables.begin());
    return t;
  }
};

TableCache& cache() {
  static TableCache c;
  return c;
}

void check_params(int64_t n, int64_t s) {
  // ScheduleParams.__post_init__ (schedule.py:59-66)
  if (n < 1) fail(ACKPT_VALUE_ERROR, "n must be >= 1, got " + std::to_string(n));
  if (s < 0) fail(ACKPT_VALUE_ERROR, "s must be >= 0, got " + std::to_string(s));
  if (n > 1 && s == 0)
    fail(ACKPT_INFEASIBLE_SCHEDULE,
         "cannot reverse " + std::to_string(n) + " steps with zero checkpoint slots");
}

// Clamp the table's slot extent: rows with s >= n - 1 are trivial (c = n),
// so a query (n, s) never needs more than min(s, n) rows.
int64_t table_s(int64_t n, int64_t s) { return std::max<int64_t>(0, std::min(s, n)); }

int64_t best_split(const CostTable& t, int64_t length, int64_t slots) {
  // Smallest k in [1, length) minimising k + c[slots-1][length-k] + c[slots][k].
  if (slots == 1) return length - 1;  // only finite candidate (row 0 is INF for m >= 2)
  const size_t W = size_t(t.n_max + 1);
  const int32_t* prev = &t.c[size_t(slots - 1) * W];
  const int32_t* row = &t.c[size_t(slots) * W];
  int64_t best_k = 1;
  int64_t best = INT64_MAX;
  for (int64_t k = 1; k < length; ++k) {
    int64_t v = k + int64_t(prev[length - k]) + int64_t(row[k]);
    if (v < best) {
      best = v;
      best_k = k;
    }
  }
  if (best >= kCap) fail(ACKPT_VALUE_ERROR, "cost table exceeds the int32 range for this (n, s)");
  return best_k;
}

}  // namespace

int64_t forward_cost_exact(int64_t n, int64_t s) {
  check_params(n, s);
  if (n <= s + 1) return n;
  if (s == 1) return n * (n + 1) / 2 - 1;
  auto t = cache().ensure(n, table_s(n, s));
  int64_t v = t->exact(s, n);
  if (v >= kInf) fail(ACKPT_INFEASIBLE_SCHEDULE, "no schedule for n=" + std::to_string(n));
  return v;
}

void taped_actions(int64_t length, std::vector<Action>& out) {
  // schedule.py:279-285
  out.push_back({ACKPT_TAPE, 0, length});
  for (int64_t step = length - 1; step >= 0; --step) out.push_back({ACKPT_REVERSE, step, 0});
  out.push_back({ACKPT_DONE, 0, 0});
}

void revolve_actions(int64_t n, int64_t s, std::vector<Action>& out) {
  // revolve_schedule / _emit_segment (schedule.py:188-235), with the right-part
  // recursion unrolled onto an explicit stack (frame = one _emit_segment call).
  check_params(n, s);
  std::shared_ptr<CostTable> t;
  if (n > s + 1 && s >= 2) t = cache().ensure(n, table_s(n, s));
  std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> free_slots;
  for (int64_t i = 0; i < s; ++i) free_slots.push(i);
  struct Frame {
    int64_t lo, hi, slots, slot, k;
    bool waiting;
  };
  std::vector<Frame> stack;
  stack.push_back({0, n, s, -1, 0, false});
  while (!stack.empty()) {
    size_t fi = stack.size() - 1;
    if (stack[fi].waiting) {
      // right part done: LoadCheckpoint(slot), heappush, hi = lo + k
      out.push_back({ACKPT_LOAD, stack[fi].slot, 0});
      free_slots.push(stack[fi].slot);
      stack[fi].hi = stack[fi].lo + stack[fi].k;
      stack[fi].waiting = false;
    }
    Frame f = stack[fi];
    int64_t length = f.hi - f.lo;
    if (length == 0) {
      stack.pop_back();
      continue;
    }
    if (length <= f.slots + 1) {
      out.push_back({ACKPT_TAPE, f.lo, f.hi});
      for (int64_t step = f.hi - 1; step >= f.lo; --step) out.push_back({ACKPT_REVERSE, step, 0});
      stack.pop_back();
      continue;
    }
    if (f.slots == 0)
      fail(ACKPT_INFEASIBLE_SCHEDULE, "segment [" + std::to_string(f.lo) + ", " +
                                          std::to_string(f.hi) +
                                          ") cannot be reversed without slots");
    int64_t k = (f.slots == 1) ? length - 1 : best_split(*t, length, f.slots);
    int64_t slot = free_slots.top();
    free_slots.pop();
    out.push_back({ACKPT_SAVE, f.lo, slot});
    out.push_back({ACKPT_ADVANCE, f.lo, f.lo + k});
    stack[fi].slot = slot;
    stack[fi].k = k;
    stack[fi].waiting = true;
    stack.push_back({f.lo + k, f.hi, f.slots - 1, -1, 0, false});
  }
  out.push_back({ACKPT_DONE, 0, 0});
}

void slot_read_liveness(const std::vector<Action>& actions, std::vector<int64_t>& last_read) {
  last_read.assign(actions.size(), -1);
  std::vector<int64_t> open_write;  // slot -> action index of its latest Save
  for (size_t idx = 0; idx < actions.size(); ++idx) {
    const Action& a = actions[idx];
    if (a.op == ACKPT_SAVE) {
      if (size_t(a.b) >= open_write.size()) open_write.resize(size_t(a.b) + 1, -1);
      open_write[size_t(a.b)] = int64_t(idx);
      last_read[idx] = -1;
    } else if (a.op == ACKPT_LOAD && a.a >= 0 && size_t(a.a) < open_write.size() &&
               open_write[size_t(a.a)] >= 0) {
      last_read[size_t(open_write[size_t(a.a)])] = int64_t(idx);
    }
  }
}

namespace {
// Decompose a finite positive double into m * 2^e with integer m < 2^53.
void decompose(double x, int64_t& m, int& e) {
  int ex = 0;
  double fr = std::frexp(x, &ex);  // x = fr * 2^ex, fr in [0.5, 1)
  m = int64_t(std::ldexp(fr, 53));
  e = ex - 53;
  while (m != 0 && (m & 1) == 0) {
    m >>= 1;
    ++e;
  }
}
}  // namespace

int64_t interval_length_exact(double t_t, double t_a) {
  // max(1, ceil(Fraction(t_t) / Fraction(t_a)))  (perfmodel.py:56-64)
  if (!(t_t > 0) || !(t_a > 0) || std::isinf(t_t) || std::isinf(t_a))
    fail(ACKPT_VALUE_ERROR, "t_t and t_a must be positive");
  int64_t m1, m2;
  int e1, e2;
  decompose(t_t, m1, e1);
  decompose(t_a, m2, e2);
  int e = e1 - e2;  // ratio = m1 / m2 * 2^e
  using u128 = unsigned __int128;
  const u128 kMax = u128(INT64_MAX);
  u128 q;
  if (e < 0) {
    if (-e > 74) return 1;  // m1 < 2^53 <= m2 * 2^-e / 2^21: ratio < 1
    u128 num = u128(m1), den = u128(m2) << (-e);
    q = num / den + (num % den != 0 ? 1 : 0);
  } else if (e <= 74) {
    u128 num = u128(m1) << e, den = u128(m2);
    q = num / den + (num % den != 0 ? 1 : 0);
  } else {
    // m1 2^e / m2 = (qq + r/m2) 2^(e-74) with qq, r from m1 2^74 / m2.
    if (e - 53 >= 63) return INT64_MAX;  // ratio >= 2^(e-53) >= 2^63
    u128 num = u128(m1) << 74, den = u128(m2);
    u128 qq = num / den, r = num % den;
    int sh = e - 74;  // <= 42
    if (qq > (kMax >> sh)) return INT64_MAX;
    u128 rs = r << sh;  // r < 2^53: fits
    q = (qq << sh) + rs / den + (rs % den != 0 ? 1 : 0);
  }
  if (q > kMax) return INT64_MAX;
  return std::max<int64_t>(1, int64_t(q));
}

}  // namespace ackpt

// ---------------------------------------------------------------------------
// C ABI

namespace {
thread_local std::vector<ackpt::Action> tl_actions;
thread_local int64_t tl_n = -1, tl_s = -1, tl_kind = -1;

int copy_out(ackpt_action* out, int64_t cap, int64_t* len) {
  if (len) *len = int64_t(tl_actions.size());
  if (out && cap > 0) {
    int64_t m = std::min<int64_t>(cap, int64_t(tl_actions.size()));
    for (int64_t i = 0; i < m; ++i) {
      out[i].op = tl_actions[size_t(i)].op;
      out[i].reserved = 0;
      out[i].a = tl_actions[size_t(i)].a;
      out[i].b = tl_actions[size_t(i)].b;
    }
  }
  return ACKPT_OK;
}
}  // namespace

extern "C" {

ACKPT_API int ackpt_forward_cost(int64_t n, int64_t s, int64_t* out) {
  return ackpt::guard([&] { *out = ackpt::forward_cost_exact(n, s); });
}

ACKPT_API int ackpt_best_split(int64_t length, int64_t slots, int64_t* out) {
  return ackpt::guard([&] {
    ackpt::check_params(length, slots);
    if (length <= slots + 1 || length < 2)
      ackpt::fail(ACKPT_VALUE_ERROR, "segment fits the tape: no split");
    if (slots == 1) {
      *out = length - 1;
      return;
    }
    auto t = ackpt::cache().ensure(length, ackpt::table_s(length, slots));
    *out = ackpt::best_split(*t, length, slots);
  });
}

ACKPT_API int ackpt_revolve_schedule(int64_t n, int64_t s, ackpt_action* out, int64_t cap,
                                     int64_t* len) {
  return ackpt::guard([&] {
    if (!(tl_kind == 0 && tl_n == n && tl_s == s)) {
      tl_kind = -1;
      tl_actions.clear();
      ackpt::revolve_actions(n, s, tl_actions);
      tl_kind = 0;
      tl_n = n;
      tl_s = s;
    }
    copy_out(out, cap, len);
  });
}

ACKPT_API int ackpt_taped_schedule(int64_t length, ackpt_action* out, int64_t cap, int64_t* len) {
  return ackpt::guard([&] {
    if (length < 1) ackpt::fail(ACKPT_VALUE_ERROR, "length must be >= 1");
    if (!(tl_kind == 1 && tl_n == length)) {
      tl_kind = -1;
      tl_actions.clear();
      ackpt::taped_actions(length, tl_actions);
      tl_kind = 1;
      tl_n = length;
      tl_s = -1;
    }
    copy_out(out, cap, len);
  });
}

ACKPT_API int ackpt_interval_length(double t_t, double t_a, int64_t* out) {
  return ackpt::guard([&] { *out = ackpt::interval_length_exact(t_t, t_a); });
}

ACKPT_API int ackpt_set_schedule_threads(int32_t threads) {
  ackpt::g_threads.store(threads);
  return ACKPT_OK;
}

}  // extern "C"
