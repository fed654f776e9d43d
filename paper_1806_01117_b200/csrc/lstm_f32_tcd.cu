// Launchers of the larger-d tensor-core kernels (lstm_f32_tcd.cuh).  The
// per-step operators are the count = 1 case of the fused launches.
#include "lstm_f32_tcd.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

namespace ackpt {

namespace {

unsigned tcd_tiles(int64_t B) { return unsigned((B + tcd::kThreads - 1) / tcd::kThreads); }

// The cell's shared-memory weight image (tcd::w_image, tcd_build_images).
template <int D>
const float* tcd_wimg(const ackpt_lstm* c, cudaStream_t) {
  return static_cast<const float*>(c->d_wimg);
}

// Grid: one CTA per tile for fused launches (long-running); per-step
// launches run persistent CTAs, as many per SM as fit, each looping over
// tiles so the weight setup is paid once per CTA.
template <class K>
unsigned tcd_grid(int64_t B, int count, K kernel, size_t smem, bool persistent, int tmem_cols) {
  const unsigned tiles = tcd_tiles(B);
  if (count > 1 || !persistent) return tiles;
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  // resident CTAs per SM from the three real limits (the occupancy API does
  // not know TMEM and reported 1 here): 512 TMEM columns, shared memory
  // (1 KB reserved per CTA), registers
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kernel);
  int smem_sm = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const int by_tmem = 512 / std::max(32, tmem_cols);
  const int by_smem = int(size_t(smem_sm) / (smem + fa.sharedSizeBytes + 1024));
  const int by_regs = 65536 / std::max(1, fa.numRegs * tcd::kThreads);
  const int per_sm = std::min({by_tmem, by_smem, by_regs});
  if (std::getenv("ACKPT_TCD_TRACE"))
    std::fprintf(stderr, "tcd grid: %d CTAs/SM (tmem %d smem %d regs %d)\n", per_sm, by_tmem, by_smem, by_regs);
  const unsigned cap = unsigned(std::max(1, per_sm) * sms);
  return std::min(tiles, cap);
}

template <class K>
void tcd_attrs(K k, size_t smem) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);  // max shared memory
}

template <int D>
void fwd_launch(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, float* const* outs,
                cudaStream_t s) {
  using L = tcd::Layout<D>;
  static bool attr = [] {
    tcd_attrs(tcd::fwd_tcd<D, false>, L::fwd_bytes);
    tcd_attrs(tcd::fwd_tcd<D, true>, L::fwd_bytes);
    return true;
  }();
  (void)attr;
  tcd::OutPtrs o{};
  const auto xb = static_cast<const float*>(c->d_xbs);
  const auto ws = tcd_wimg<D>(c, s);
  const int cols = tcd::tmem_cols(4 * D);
  bool pdl = false;
  const chain::Chain ch = chain::next(c, s, tcd_tiles(c->B), pdl);
  if (outs) {
    for (int i = 0; i < count; ++i) o.p[i] = outs[i];
    auto k = tcd::fwd_tcd<D, true>;
    chain::launch(k, tcd_grid(c->B, count, k, L::fwd_bytes, true, cols), tcd::kThreads, L::fwd_bytes, pdl, s, in,
                  static_cast<float*>(nullptr), c->B, xb, ws, from, count, o, ch);
  } else {
    auto k = tcd::fwd_tcd<D, false>;
    chain::launch(k, tcd_grid(c->B, count, k, L::fwd_bytes, true, cols), tcd::kThreads, L::fwd_bytes, pdl, s, in,
                  out, c->B, xb, ws, from, count, o, ch);
  }
}

template <int D>
void rev_launch(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* ai, float* ao,
                cudaStream_t s) {
  using L = tcd::Layout<D>;
  static bool attr = [] {
    tcd_attrs(tcd::rev_tcd<D>, L::rev_bytes);
    return true;
  }();
  (void)attr;
  tcd::StatePtrs sp{};
  for (int i = 0; i < count; ++i) sp.p[i] = states[i];
  auto k = tcd::rev_tcd<D>;
  bool pdl = false;
  const chain::Chain ch = chain::next(c, s, tcd_tiles(c->B), pdl);
  chain::launch(k, tcd_grid(c->B, count, k, L::rev_bytes, true, tcd::tmem_cols(7 * D)), tcd::kThreads, L::rev_bytes,
                pdl, s, ai, ao, c->B, static_cast<const float*>(c->d_xbs), tcd_wimg<D>(c, s), from, count, sp, ch);
}

// d = 64 reverse: one kernel per launch (rev_tcd64: Wᵀ streamed through a
// shared-memory ring from a chunk image built once per cell and cached in
// cell->d_scratch).
void rev64_launch(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* ai,
                  float* ao, cudaStream_t s) {
  static bool attr = [] {
    cudaFuncSetAttribute(tcd::rev_tcd64, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tcd::kRev64Smem));
    cudaFuncSetAttribute(tcd::rev_tcd64, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    return true;
  }();
  (void)attr;
  static int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  tcd::StatePtrs sp{};
  for (int i = 0; i < count; ++i) sp.p[i] = states[i];
  const unsigned tiles = tcd_tiles(c->B);
  const unsigned grid = count > 1 ? tiles : std::min<unsigned>(tiles, unsigned(sms));  // one CTA per SM
  bool pdl = false;
  const chain::Chain ch = chain::next(c, s, tiles, pdl);
  chain::launch(tcd::rev_tcd64, grid, tcd::kThreads64, tcd::kRev64Smem, pdl, s, ai, ao, c->B,
                static_cast<const float*>(c->d_xbs), tcd_wimg<64>(c, s), static_cast<const float*>(c->d_scratch), from,
                count, sp, ch);
}

}  // namespace

void tcd_build_images(ackpt_lstm* c) {
  const auto ws = static_cast<const float*>(c->d_ws);
  const size_t img = size_t(16) * c->d * c->d * sizeof(float);
  ACKPT_CUDA_CHECK(cudaMalloc(&c->d_wimg, img));
  if (c->d == 16) tcd::w_image<16><<<64, 256>>>(ws, static_cast<float*>(c->d_wimg));
  else if (c->d == 32) tcd::w_image<32><<<64, 256>>>(ws, static_cast<float*>(c->d_wimg));
  else tcd::w_image<64><<<64, 256>>>(ws, static_cast<float*>(c->d_wimg));
  if (c->d == 64) {
    const size_t chunks = size_t(tcd::kChunks64) * 2 * tcd::kChunkFloats64 * sizeof(float);
    ACKPT_CUDA_CHECK(cudaMalloc(&c->d_scratch, chunks));
    c->scratch_bytes = chunks;
    tcd::w2_image64<<<64, 256>>>(ws, static_cast<float*>(c->d_scratch));
  }
  ACKPT_CUDA_CHECK(cudaGetLastError());
  ACKPT_CUDA_CHECK(cudaDeviceSynchronize());
}

namespace {
bool tcd_common(const ackpt_lstm* c, std::initializer_list<const void*> ptrs) {
  static const bool on = [] {
    const char* e = std::getenv("ACKPT_TCD");
    return !(e && std::string(e) == "0");
  }();
  if (!on || c->dtype != ACKPT_F32 || !c->d_ws || !c->d_xbs) return false;
  for (const void* p : ptrs)
    if (reinterpret_cast<uintptr_t>(p) & 3u) return false;
  return true;
}
}  // namespace

// Forward kernels: d in {16, 32, 64} (d = 64: A + W hi/lo + bias = 212 KB of
// shared memory, 256 TMEM columns, one CTA per SM).
bool tcd_ok(const ackpt_lstm* c, std::initializer_list<const void*> ptrs) {
  return (c->d == 16 || c->d == 32 || c->d == 64) && tcd_common(c, ptrs);
}
// Reverse kernels: d in {16, 32} (rev_tcd), d = 64 (rev_tcd64, Wᵀ streamed).
bool tcd_rev_ok(const ackpt_lstm* c, std::initializer_list<const void*> ptrs) {
  return (c->d == 16 || c->d == 32 || c->d == 64) && tcd_common(c, ptrs);
}

void tcd_forward(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, float* const* outs,
                 cudaStream_t s) {
  if (c->d == 16) fwd_launch<16>(c, from, count, in, out, outs, s);
  else if (c->d == 32) fwd_launch<32>(c, from, count, in, out, outs, s);
  else fwd_launch<64>(c, from, count, in, out, outs, s);
}

void tcd_reverse(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* adj_in,
                 float* adj_out, cudaStream_t s) {
  if (c->d == 16) rev_launch<16>(c, from, count, states, adj_in, adj_out, s);
  else if (c->d == 32) rev_launch<32>(c, from, count, states, adj_in, adj_out, s);
  else rev64_launch(c, from, count, states, adj_in, adj_out, s);
}

}  // namespace ackpt
