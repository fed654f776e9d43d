// Launchers of the tensor-core fused LSTM kernels (lstm_f32_tc.cuh).
#include "lstm_f32_tc.cuh"

#include <cstdint>
#include <cstdlib>

namespace ackpt {

namespace {

tc::Weights tc_weights(const ackpt_lstm* c) {
  f32m::ScaledParams<8> sp;
  f32m::fill_scaled<8>(c, -1, sp);
  tc::Weights w;
  std::memcpy(w.ws, sp.ws, sizeof(w.ws));
  for (int g = 0; g < 4; ++g)
    for (int j = 0; j < 8; ++j)
      for (int k = 0; k < 8; ++k) w.wu[g][j][k] = float(c->wh64[(size_t(g) * 8 + j) * 8 + k]);
  return w;
}

unsigned tc_grid(int64_t B) { return unsigned((B + tc::kTile - 1) / tc::kTile); }

}  // namespace

thread_local int g_chain_hint = 0;
thread_local int g_chain_native = 0;

void tc_advance(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, cudaStream_t s) {
  tc::OutPtrs none{};
  bool pdl = false;
  const tc::Chain ch = chain::next(c, s, tc_grid(c->B), pdl);
  chain::launch(tc::fwd_tc<false>, tc_grid(c->B), tc::kThreads, 0, pdl, s, in, out, c->B, static_cast<const float*>(c->d_xbs),
            int64_t(from), count, tc_weights(c), none, ch);
}

void tc_forward_many(const ackpt_lstm* c, int64_t from, int count, const float* in, float* const* outs,
                     cudaStream_t s) {
  tc::OutPtrs o{};
  for (int i = 0; i < count; ++i) o.p[i] = outs[i];
  bool pdl = false;
  const tc::Chain ch = chain::next(c, s, tc_grid(c->B), pdl);
  chain::launch(tc::fwd_tc<true>, tc_grid(c->B), tc::kThreads, 0, pdl, s, in, static_cast<float*>(nullptr), c->B,
            static_cast<const float*>(c->d_xbs), int64_t(from), count, tc_weights(c), o, ch);
}

// Reverse run: rev_tc<true> streams each step's taped state into shared
// memory one step ahead with cp.async.bulk (B % 4 == 0, 16-byte aligned
// states); rev_tc<false> loads it at the top of each step.
void tc_backward_many(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* adj_in,
                      float* adj_out, cudaStream_t s) {
  tc::StatePtrs sp{};
  for (int i = 0; i < count; ++i) sp.p[i] = states[i];
  bool pf = c->B % 4 == 0;
  for (int i = 0; i < count; ++i) pf = pf && !(reinterpret_cast<uintptr_t>(states[i]) & 15u);
  bool pdl = false;
  const tc::Chain ch = chain::next(c, s, tc_grid(c->B), pdl);
  if (pf)
    chain::launch(tc::rev_tc<true>, tc_grid(c->B), tc::kThreads, 0, pdl, s, adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs),
              int64_t(from), count, tc_weights(c), sp, ch);
  else
    chain::launch(tc::rev_tc<false>, tc_grid(c->B), tc::kThreads, 0, pdl, s, adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs),
              int64_t(from), count, tc_weights(c), sp, ch);
}

}  // namespace ackpt
