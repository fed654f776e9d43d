// Launchers of the tensor-core fused LSTM kernels (lstm_f32_tc.cuh).
#include "lstm_f32_tc.cuh"
#include "lstm_f32_tcp.cuh"
#include "lstm_f32_tcr.cuh"
#include "lstm_f32_tcq.cuh"

#include <cstdint>
#include <cstdlib>
#include <string>

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

// ACKPT_TC_FWD=pp: ping-pong forward (lstm_f32_tcp.cuh: one tile's MMA behind
// the other tile's activations).  Correct but measured slower than fwd_tc at
// the C2 shape (advance 15.5-15.8 vs 14.8 us/step, tape 19.6-20.6 vs 18.1 at
// 6-8 CTAs/SM: the second barrier per step and spills outweigh the hidden
// MMA latency), so fwd_tc is the default.
bool tc_pingpong() {
  static const bool pp = [] {
    const char* e = std::getenv("ACKPT_TC_FWD");
    return e && std::string(e) == "pp";
  }();
  return pp;
}

tcp::Weights tcp_weights(const ackpt_lstm* c) {
  f32m::ScaledParams<8> sp;
  f32m::fill_scaled<8>(c, -1, sp);
  tcp::Weights w;
  std::memcpy(w.ws, sp.ws, sizeof(w.ws));
  return w;
}

// ACKPT_TC_P=2: two float2 pairs per thread in the forward (lstm_f32_tcq.cuh).
int tc_pairs() {
  static const int p = [] {
    const char* e = std::getenv("ACKPT_TC_P");
    return (e && std::string(e) == "2") ? 2 : 1;
  }();
  return p;
}

void tc_advance(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, cudaStream_t s) {
  if (tc_pairs() == 2) {
    tc::OutPtrs none{};
    tcq::fwd_tcq<2><<<unsigned((c->B + 511) / 512), tcq::kThreads, 0, s>>>(
        in, out, c->B, static_cast<const float*>(c->d_xbs), from, count, false, tc_weights(c), none);
    return;
  }
  if (tc_pingpong()) {
    tcp::OutPtrs none{};
    tcp::fwd_tcp<false, true><<<tc_grid(c->B), tcp::kThreads, 0, s>>>(
        in, out, c->B, static_cast<const float*>(c->d_xbs), from, count, tcp_weights(c), none);
    return;
  }
  tc::OutPtrs none{};
  tc::fwd_tc<false><<<tc_grid(c->B), tc::kThreads, 0, s>>>(in, out, c->B, static_cast<const float*>(c->d_xbs),
                                                            from, count, tc_weights(c), none);
}

void tc_forward_many(const ackpt_lstm* c, int64_t from, int count, const float* in, float* const* outs,
                     cudaStream_t s) {
  if (tc_pairs() == 2) {
    tc::OutPtrs o{};
    for (int i = 0; i < count; ++i) o.p[i] = outs[i];
    tcq::fwd_tcq<2><<<unsigned((c->B + 511) / 512), tcq::kThreads, 0, s>>>(
        in, nullptr, c->B, static_cast<const float*>(c->d_xbs), from, count, true, tc_weights(c), o);
    return;
  }
  if (tc_pingpong()) {
    tcp::OutPtrs o{};
    for (int i = 0; i < count; ++i) o.p[i] = outs[i];
    tcp::fwd_tcp<true, true><<<tc_grid(c->B), tcp::kThreads, 0, s>>>(
        in, nullptr, c->B, static_cast<const float*>(c->d_xbs), from, count, tcp_weights(c), o);
    return;
  }
  tc::OutPtrs o{};
  for (int i = 0; i < count; ++i) o.p[i] = outs[i];
  tc::fwd_tc<true><<<tc_grid(c->B), tc::kThreads, 0, s>>>(in, nullptr, c->B, static_cast<const float*>(c->d_xbs),
                                                           from, count, tc_weights(c), o);
}

void tc_backward_many(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* adj_in,
                      float* adj_out, cudaStream_t s) {
  tc::StatePtrs sp{};
  for (int i = 0; i < count; ++i) sp.p[i] = states[i];
  bool pf = c->B % 4 == 0 && std::getenv("ACKPT_TC_NO_PF") == nullptr;
  for (int i = 0; i < count; ++i) pf = pf && !(reinterpret_cast<uintptr_t>(states[i]) & 15u);
  // ACKPT_TC_REV: default / "1" gates on the tensor cores (rev_tc, fastest
  // measured, 28.4 us/step); "2" both matvecs on the tensor cores (rev_tc2,
  // 34.2: its second MMA round trip per step costs more than the FMA work it
  // removes at 4 CTAs/SM), "2nr" the same with Newton rcp,
  // "3" the same with the two tiles in ping-pong (rev_tcr, 34.9: a third
  // barrier per step), "sp" rev_tc software-pipelined across steps (rev_tcs,
  // 29.7: its double-buffered accumulator allows 4 CTAs/SM instead of 5).
  // All pass the parity suite (tests/test_gpu_variants.py).
  static const int rev = [] {
    const char* e = std::getenv("ACKPT_TC_REV");
    if (!e) return 1;
    const std::string v(e);
    return v == "2" ? 2 : v == "2nr" ? 3 : v == "3" ? 4 : v == "sp" ? 5 : 1;
  }();
  if (pf && rev == 5) {
    tc::rev_tcs<<<tc_grid(c->B), tc::kThreads, 0, s>>>(adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs),
                                                       from, count, tc_weights(c), sp);
    return;
  }
  if (pf && rev == 4) {  // both products on tensor cores, tiles in ping-pong (lstm_f32_tcr.cuh)
    tcr::StatePtrs rp{};
    for (int i = 0; i < count; ++i) rp.p[i] = states[i];
    tcr::Weights w;
    f32m::ScaledParams<8> sp8;
    f32m::fill_scaled<8>(c, -1, sp8);
    std::memcpy(w.ws, sp8.ws, sizeof(w.ws));
    tcr::rev_tcr<<<tc_grid(c->B), tcr::kThreads, 0, s>>>(adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs),
                                                         from, count, w, rp);
    return;
  }
  if (pf && rev == 2)
    tc::rev_tc2<false><<<tc_grid(c->B), tc::kThreads, 0, s>>>(
        adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs), from, count, tc_weights(c), sp);
  else if (pf && rev == 3)
    tc::rev_tc2<true><<<tc_grid(c->B), tc::kThreads, 0, s>>>(
        adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs), from, count, tc_weights(c), sp);
  else if (pf)
    tc::rev_tc<true><<<tc_grid(c->B), tc::kThreads, 0, s>>>(
        adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs), from, count, tc_weights(c), sp);
  else
    tc::rev_tc<false><<<tc_grid(c->B), tc::kThreads, 0, s>>>(
        adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs), from, count, tc_weights(c), sp);
}

}  // namespace ackpt
