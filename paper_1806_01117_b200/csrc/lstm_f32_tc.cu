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

// Launch chain (lstm_f32_tc.cuh Chain): ACKPT_TC_CHAIN=0 off, =force chains
// every back-to-back fused launch of a cell on one stream (probes that
// enqueue nothing else in between), default: chain when the executor says
// the previous compute-stream operation was this operator's fused launch.
int chain_mode() {
  static const int m = [] {
    const char* e = std::getenv("ACKPT_TC_CHAIN");
    if (!e) return 1;
    const std::string v(e);
    return v == "0" ? 0 : v == "force" ? 2 : 1;
  }();
  return m;
}

tc::Chain chain_for(const ackpt_lstm* c, cudaStream_t s, bool& pdl) {
  auto* cell = const_cast<ackpt_lstm*>(c);
  pdl = false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  ACKPT_CUDA_CHECK(cudaStreamIsCapturing(s, &cs));
  const int mode = chain_mode();
  if (mode == 0 || cs != cudaStreamCaptureStatusNone) return tc::Chain{nullptr, 0u, 0u};  // chain stays closed
  const int64_t tiles = int64_t(tc_grid(c->B));
  if (!cell->d_chain || cell->chain_tiles < tiles) {
    if (cell->d_chain) {
      ACKPT_CUDA_CHECK(cudaStreamSynchronize(s));
      cudaFree(cell->d_chain);
      cell->d_chain = nullptr;
    }
    ACKPT_CUDA_CHECK(cudaMalloc(&cell->d_chain, size_t(tiles) * sizeof(uint32_t)));
    ACKPT_CUDA_CHECK(cudaMemset(cell->d_chain, 0, size_t(tiles) * sizeof(uint32_t)));
    cell->chain_tiles = tiles;
    cell->chain_epoch = 0;
    cell->chain_prev = false;
  }
  const bool chained = (mode == 2 || g_chain_hint) && cell->chain_prev && cell->chain_stream == s;
  tc::Chain ch{cell->d_chain, chained ? cell->chain_epoch : 0u, cell->chain_epoch + 1};
  if (++cell->chain_epoch == 0) cell->chain_epoch = 1;  // (flags compare by signed distance)
  cell->chain_open = true;
  cell->chain_stream = s;
  pdl = chained;
  return ch;
}

template <class K, class... A>
void tc_launch(K kernel, unsigned grid, bool pdl, cudaStream_t s, A... args) {
  if (!pdl) {
    kernel<<<grid, tc::kThreads, 0, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tc::kThreads);
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ACKPT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, args...));
}

}  // namespace

thread_local int g_chain_hint = 0;

void tc_advance(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, cudaStream_t s) {
  tc::OutPtrs none{};
  bool pdl = false;
  const tc::Chain ch = chain_for(c, s, pdl);
  tc_launch(tc::fwd_tc<false>, tc_grid(c->B), pdl, s, in, out, c->B, static_cast<const float*>(c->d_xbs),
            int64_t(from), count, tc_weights(c), none, ch);
}

void tc_forward_many(const ackpt_lstm* c, int64_t from, int count, const float* in, float* const* outs,
                     cudaStream_t s) {
  tc::OutPtrs o{};
  for (int i = 0; i < count; ++i) o.p[i] = outs[i];
  bool pdl = false;
  const tc::Chain ch = chain_for(c, s, pdl);
  tc_launch(tc::fwd_tc<true>, tc_grid(c->B), pdl, s, in, static_cast<float*>(nullptr), c->B,
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
  const tc::Chain ch = chain_for(c, s, pdl);
  if (pf)
    tc_launch(tc::rev_tc<true>, tc_grid(c->B), pdl, s, adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs),
              int64_t(from), count, tc_weights(c), sp, ch);
  else
    tc_launch(tc::rev_tc<false>, tc_grid(c->B), pdl, s, adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs),
              int64_t(from), count, tc_weights(c), sp, ch);
}

}  // namespace ackpt
