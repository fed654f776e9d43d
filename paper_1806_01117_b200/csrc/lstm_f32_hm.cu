// Launchers of the register-fragment tensor-core kernels (lstm_f32_hm.cuh)
// and their per-cell tables.
#include "lstm_f32_hm.cuh"

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace ackpt {

namespace {

unsigned hm_grid(int64_t B) {
  const int64_t per_cta = int64_t(hm::kRows) * hm::kWarps;
  return unsigned((B + per_cta - 1) / per_cta);
}

// ACKPT_HM_NR: "0" MUFU reciprocals everywhere, "1" Newton reciprocals
// everywhere, default "f": Newton in the forward (MUFU-bound), MUFU in the
// reverse (FMA-bound).
struct NrChoice {
  bool fwd = true, rev = false;
  NrChoice() {
    const char* e = std::getenv("ACKPT_HM_NR");
    if (!e) return;
    const std::string v(e);
    if (v == "0") fwd = rev = false;
    if (v == "1") fwd = rev = true;
  }
};
const NrChoice& nr() {
  static NrChoice c;
  return c;
}

}  // namespace

void hm_tables(ackpt_lstm* c) {
  constexpr int D = 8;
  const double scale[4] = {-1.4426950408889634, -1.4426950408889634, -1.4426950408889634, 2.0 * 1.4426950408889634};
  float ws[4][D][D];
  for (int g = 0; g < 4; ++g)
    for (int j = 0; j < D; ++j)
      for (int k = 0; k < D; ++k) ws[g][j][k] = float(c->wh64[(size_t(g) * D + j) * D + k] * scale[g]);
  auto hi = [](float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u &= 0xFFFFE000u;
    float y;
    std::memcpy(&y, &u, 4);
    return y;
  };
  auto unit = [](int n) { return n / 2 + 4 * (n % 2); };
  std::vector<float> frag(32 * 32);
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    float* w = &frag[size_t(lane) * 32];
    for (int gi = 0; gi < 4; ++gi)
      for (int e = 0; e < 2; ++e) {
        const float x = ws[gi][unit(g)][t + 4 * e];  // gates: B[k][n] = W[u(n)][k]
        w[2 * gi + e] = hi(x);
        w[8 + 2 * gi + e] = x - hi(x);
        const float y = ws[gi][t + 4 * e][unit(g)];  // transposed: B2[8 gate + k][n] = W[k][u(n)]
        w[16 + 2 * gi + e] = hi(y);
        w[24 + 2 * gi + e] = y - hi(y);
      }
  }
  std::vector<float> xbs(size_t(c->n) * 32);
  for (int64_t k = 0; k < c->n; ++k)
    for (int t = 0; t < 4; ++t)
      for (int gi = 0; gi < 4; ++gi)
        for (int e = 0; e < 2; ++e)
          xbs[(size_t(k) * 4 + t) * 8 + 2 * gi + e] =
              float(c->xb64[(size_t(k) * 4 + gi) * D + (t + 4 * e)] * scale[gi]);
  ACKPT_CUDA_CHECK(cudaMalloc(&c->d_frag_hm, frag.size() * sizeof(float)));
  ACKPT_CUDA_CHECK(cudaMemcpy(c->d_frag_hm, frag.data(), frag.size() * sizeof(float), cudaMemcpyHostToDevice));
  ACKPT_CUDA_CHECK(cudaMalloc(&c->d_xbs_hm, xbs.size() * sizeof(float)));
  ACKPT_CUDA_CHECK(cudaMemcpy(c->d_xbs_hm, xbs.data(), xbs.size() * sizeof(float), cudaMemcpyHostToDevice));
}

void hm_advance(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, cudaStream_t s) {
  hm::OutPtrs none{};
  const auto xb = static_cast<const float*>(c->d_xbs_hm);
  const auto fr = static_cast<const float*>(c->d_frag_hm);
  if (nr().fwd)
    hm::fwd_hm<false, true><<<hm_grid(c->B), hm::kThreads, 0, s>>>(in, out, c->B, xb, fr, from, count, none);
  else
    hm::fwd_hm<false, false><<<hm_grid(c->B), hm::kThreads, 0, s>>>(in, out, c->B, xb, fr, from, count, none);
}

void hm_forward_many(const ackpt_lstm* c, int64_t from, int count, const float* in, float* const* outs,
                     cudaStream_t s) {
  hm::OutPtrs o{};
  for (int i = 0; i < count; ++i) o.p[i] = outs[i];
  const auto xb = static_cast<const float*>(c->d_xbs_hm);
  const auto fr = static_cast<const float*>(c->d_frag_hm);
  if (nr().fwd)
    hm::fwd_hm<true, true><<<hm_grid(c->B), hm::kThreads, 0, s>>>(in, nullptr, c->B, xb, fr, from, count, o);
  else
    hm::fwd_hm<true, false><<<hm_grid(c->B), hm::kThreads, 0, s>>>(in, nullptr, c->B, xb, fr, from, count, o);
}

void hm_backward_many(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* adj_in,
                      float* adj_out, cudaStream_t s) {
  hm::StatePtrs sp{};
  for (int i = 0; i < count; ++i) sp.p[i] = states[i];
  const auto xb = static_cast<const float*>(c->d_xbs_hm);
  const auto fr = static_cast<const float*>(c->d_frag_hm);
  if (nr().rev)
    hm::rev_hm<true><<<hm_grid(c->B), hm::kThreads, 0, s>>>(adj_in, adj_out, c->B, xb, fr, from, count, sp);
  else
    hm::rev_hm<false><<<hm_grid(c->B), hm::kThreads, 0, s>>>(adj_in, adj_out, c->B, xb, fr, from, count, sp);
}

}  // namespace ackpt
