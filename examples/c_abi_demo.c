/* A reverse pass through the C ABI only (include/ackpt.h + libackpt.so),
 * the way a non-Python host would drive it:
 * build an LSTM cell, take its operator, run FullStorage, Revolve and
 * Multistage (pinned-host tier, calibrated interval) on one fp32 batch and
 * check that the three adjoints are bit-identical and the counters are the
 * schedule's.  Prints one JSON line; exit 0 on success.
 *
 *   gcc -O2 -Iinclude -I/usr/local/cuda/include examples/c_abi_demo.c \
 *       -Lpaper_1806_01117_b200 -lackpt -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1806_01117_b200 -o build/c_abi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ackpt.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    int rc_ = (call);                                                            \
    if (rc_ != ACKPT_OK) {                                                       \
      fprintf(stderr, "%s failed: %d %s\n", #call, rc_, ackpt_last_error());     \
      return 1;                                                                  \
    }                                                                            \
  } while (0)

static double urand(unsigned long long* s) { /* deterministic U(-0.1, 0.1) */
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return ((double)(*s >> 11) / 9007199254740992.0 - 0.5) * 0.2;
}

int main(void) {
  const int d = 8;
  const int64_t n = 40, B = 4096;
  unsigned long long seed = 7;
  double* w[4];
  double* b[4];
  for (int g = 0; g < 4; ++g) {
    w[g] = (double*)malloc(sizeof(double) * d * 2 * d); /* [d x 2d], W_h | W_x */
    b[g] = (double*)malloc(sizeof(double) * d);
    for (int i = 0; i < d * 2 * d; ++i) w[g][i] = urand(&seed);
    for (int i = 0; i < d; ++i) b[g][i] = urand(&seed);
  }
  double* xs = (double*)malloc(sizeof(double) * n * d);
  double* target = (double*)malloc(sizeof(double) * d);
  for (int i = 0; i < n * d; ++i) xs[i] = urand(&seed);
  for (int i = 0; i < d; ++i) target[i] = urand(&seed);

  ackpt_lstm* cell;
  CHECK(ackpt_lstm_create(d, n, B, ACKPT_F32, w[0], w[1], w[2], w[3], b[0], b[1], b[2], b[3], xs, target, &cell));
  ackpt_operator op;
  CHECK(ackpt_lstm_operator(cell, &op));
  const size_t S = (size_t)op.state_bytes;

  float* h_state = (float*)malloc(S);
  for (size_t i = 0; i < S / 4; ++i) h_state[i] = (float)urand(&seed);
  void *d_state, *d_adj[3];
  if (cudaMalloc(&d_state, S) != cudaSuccess) return 1;
  for (int i = 0; i < 3; ++i)
    if (cudaMalloc(&d_adj[i], S) != cudaSuccess) return 1;
  cudaMemcpy(d_state, h_state, S, cudaMemcpyHostToDevice);

  ackpt_engine* eng;
  ackpt_tier* tier;
  CHECK(ackpt_engine_create(&op, &eng));
  CHECK(ackpt_tier_create(0, (int64_t)S, &tier));
  CHECK(ackpt_engine_set_fusion(eng, 1));

  ackpt_stats st[3];
  CHECK(ackpt_engine_prepare(eng, ACKPT_FULL_STORAGE, 0, 0, tier));
  CHECK(ackpt_engine_run(eng, d_state, NULL, d_adj[0], &st[0], NULL));
  CHECK(ackpt_engine_prepare(eng, ACKPT_REVOLVE, 5, 0, tier));
  CHECK(ackpt_engine_run(eng, d_state, NULL, d_adj[1], &st[1], NULL));
  double t_a, t_b, t_t;
  int64_t interval;
  CHECK(ackpt_engine_calibrate(eng, tier, 5, d_state, &t_a, &t_b, &t_t));
  CHECK(ackpt_interval_length(t_t, t_a, &interval));
  if (interval >= n) interval = 8; /* keep a two-level plan at this small n */
  CHECK(ackpt_engine_prepare(eng, ACKPT_MULTISTAGE, interval, interval, tier));
  CHECK(ackpt_engine_run(eng, d_state, NULL, d_adj[2], &st[2], NULL));

  float* h_adj[3];
  int finite = 1;
  for (int i = 0; i < 3; ++i) {
    h_adj[i] = (float*)malloc(S);
    cudaMemcpy(h_adj[i], d_adj[i], S, cudaMemcpyDeviceToHost);
  }
  for (size_t i = 0; i < S / 4; ++i) finite &= isfinite(h_adj[0][i]) != 0;
  const int same = memcmp(h_adj[0], h_adj[1], S) == 0 && memcmp(h_adj[0], h_adj[2], S) == 0;
  int64_t cost;
  CHECK(ackpt_forward_cost(n, 5, &cost));
  const int counters = st[0].forward_evals == n && st[1].forward_evals == cost && st[2].forward_evals == 2 * n &&
                       st[2].stores_issued == (n + interval - 1) / interval && st[0].backward_evals == n;
  printf("{\"version\": \"%s\", \"state_bytes\": %lld, \"interval\": %lld, \"forward_evals\": [%lld, %lld, %lld], "
         "\"stores\": %lld, \"bit_identical\": %s, \"finite\": %s, \"counters_ok\": %s}\n",
         ackpt_version(), (long long)S, (long long)interval, (long long)st[0].forward_evals,
         (long long)st[1].forward_evals, (long long)st[2].forward_evals, (long long)st[2].stores_issued,
         same ? "true" : "false", finite ? "true" : "false", counters ? "true" : "false");

  CHECK(ackpt_engine_destroy(eng));
  CHECK(ackpt_tier_destroy(tier));
  CHECK(ackpt_lstm_destroy(cell));
  return (same && finite && counters) ? 0 : 2;
}
