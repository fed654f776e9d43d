/* TEST INFRASTRUCTURE ONLY: plain C restatement of the reference cost table
 * (pkg/src/asyncckpt/schedule.py:139-155) for sizes the Python oracle cannot
 * reach.  O(s n^2), no tricks: every cell is min_k k + c[s-1][n-k] + c[s][k]
 * over int64 with INF = 2^40 exactly as the reference.  Used by tests to
 * cross-check the product's saturated, threaded table at large (n, s).
 * Build: make -C oracle (output in oracle/_build/, git-ignored). */
#include <stdint.h>
#include <stdlib.h>

#define INF (((int64_t)1) << 40)

/* Fills out[s * (n_max + 1) + n] for s <= s_max, n <= n_max.  Returns 0. */
int oracle_cost_table(int64_t n_max, int64_t s_max, int64_t *out) {
  const int64_t W = n_max + 1;
  for (int64_t s = 0; s <= s_max; ++s) {
    int64_t *row = out + s * W;
    for (int64_t n = 0; n <= n_max; ++n) row[n] = INF;
    row[0] = 0;
    if (n_max >= 1) row[1] = 1;
    int64_t top = s + 1 < n_max ? s + 1 : n_max;
    for (int64_t n = 2; n <= top; ++n) row[n] = n;
    if (s == 0) continue;
    const int64_t *prev = out + (s - 1) * W;
    for (int64_t n = s + 2; n <= n_max; ++n) {
      int64_t best = INT64_MAX;
      for (int64_t k = 1; k < n; ++k) {
        int64_t v = k + prev[n - k] + row[k];
        if (v < best) best = v;
      }
      row[n] = best;
    }
  }
  return 0;
}

/* Smallest k minimising k + c[slots-1][length-k] + c[slots][k]
 * (schedule.py:177-181), given a table built by oracle_cost_table. */
int64_t oracle_best_split(const int64_t *table, int64_t n_max, int64_t length, int64_t slots) {
  const int64_t W = n_max + 1;
  int64_t best = INT64_MAX, best_k = 1;
  for (int64_t k = 1; k < length; ++k) {
    int64_t v = k + table[(slots - 1) * W + length - k] + table[slots * W + k];
    if (v < best) {
      best = v;
      best_k = k;
    }
  }
  return best_k;
}
