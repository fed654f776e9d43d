// Device-resident LSTM cell (lstm.py:39-69 LstmCell, batched) and the kernel
// launch entry points shared by the kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <initializer_list>
#include <mutex>
#include <vector>

#include "common.h"

struct ackpt_lstm {
  int d = 0;
  int64_t n = 0, B = 0;
  int dtype = ACKPT_F32;
  size_t esize = 4;
  std::vector<double> wh64, xb64, target64;         // float64 master copies
  std::vector<unsigned char> wh_t, xb_t, target_t;  // rounded to the cell dtype
  void* d_wh = nullptr;                             // 4 x d x d, dtype
  void* d_wht = nullptr;                            // d x 4d (W_h transposed), dtype
  void* d_xb = nullptr;                             // n x 4 x d, dtype
  void* d_xbs = nullptr;  // n x 4 x d fp32, pre-scaled per gate (fp32 fast path, d <= 16)
  void* d_ws = nullptr;       // fp32 d in {16, 32, 64}: 4 x d x d pre-scaled W (lstm_f32_tcd.cu)
  void* d_scratch = nullptr;  // fp32 d = 64 reverse: chunk image of the scaled W^T (tcd_build_images)
  void* d_wimg = nullptr;     // fp32 d in {16, 32, 64}: shared-memory image of W / W^T hi|lo (tcd_build_images)
  size_t scratch_bytes = 0;
  // launch chain of the tensor-core kernels (chain.cuh): per-tile completion
  // epochs, one flag array per stream the cell launches on (launches on
  // different streams never share flags)
  struct ChainSlot {
    void* stream = nullptr;
    uint32_t* flags = nullptr;
    int64_t tiles = 0;
    int64_t last_tiles = 0;  // tile count of the last launch (chains only between equal tilings)
    uint32_t epoch = 0;      // the last epoch handed out on this stream
  };
  ChainSlot chain_slots[4];
  int chain_victim = 0;
  bool chain_prev = false;            // the process's last cell launch was a chain-publishing
  void* chain_prev_stream = nullptr;  // launch of this cell, on this stream (chain_touch;
                                      // 0 is a valid stream handle: the legacy default stream)
};

namespace ackpt {

// Parameter block of the fast step kernels (lives in the constant bank).
template <typename T, int D>
struct StepParams {
  T wh[4][D][D];  // gate g (f, i, o, c), row j, column i over h
  T xb[4][D];     // W_x x_k + b of this step
};

template <typename T>
struct TargetParams {
  T target[128];
};

constexpr int kMaxD = 128;
constexpr int64_t kSmallBatch = (int64_t(1) << 31) - 1;  // CTA-per-sequence kernels (lstm_small.cu): grid-x limit
constexpr int64_t kSbFirstBatch = 2048;   // ... preferred over the batch-tiled fp32 kernels up to this one

// fp32 fast path, d in {4, 8}: float2-paired kernels (lstm_f32_d*.cu).
template <int D>
void f32_forward(const ackpt_lstm* c, int64_t step, const float* in, float* out, cudaStream_t s);
template <int D>
void f32_backward(const ackpt_lstm* c, int64_t step, const float* st, const float* ai, float* ao,
                  cudaStream_t s);
template <int D>
void f32_advance(const ackpt_lstm* c, int64_t from, int64_t to, const float* in, float* out,
                 cudaStream_t s);
// Temporal fusion: a TapeForward run / a Reverse run in one launch (count <= 64).
template <int D>
void f32_forward_many(const ackpt_lstm* c, int64_t from, int count, const float* in,
                      float* const* outs, cudaStream_t s);
template <int D>
void f32_backward_many(const ackpt_lstm* c, int64_t from, int count, const float* const* states,
                       const float* adj_in, float* adj_out, cudaStream_t s);
// Launch chain bookkeeping.  The process-wide token names the (cell, stream)
// of the last cell launch if it was a tensor-core launch that publishes tile
// flags; every cell API entry point calls chain_touch first, which hands the
// token to the cell if it is its own and clears it -- so a launch can only be
// chained to the immediately preceding launch of ANY cell, on the same
// stream (another cell's or a non-chain kernel in between breaks the chain).
struct ChainToken {
  std::mutex mu;
  const ackpt_lstm* cell = nullptr;
  void* stream = nullptr;
};
inline ChainToken& chain_token() {
  static ChainToken t;
  return t;
}
inline void chain_touch(const ackpt_lstm* c) {
  auto& t = chain_token();
  std::lock_guard<std::mutex> lk(t.mu);
  auto* m = const_cast<ackpt_lstm*>(c);
  m->chain_prev = t.cell == c;
  m->chain_prev_stream = t.stream;
  t.cell = nullptr;
  t.stream = nullptr;
}
// Frees the cell's flag arrays (after a device synchronization).
void chain_release(ackpt_lstm* c);

// The chain bookkeeping of one launch, host only (chain.cuh's next() runs it
// with a CUDA allocator, ackpt_chain_selftest with a fake one).  Caller holds
// chain_token().mu and called chain_touch(cell) at the API entry.  Picks the
// stream's flag slot -- (re)allocating it through alloc(old_flags, tiles) when
// missing or too small, evicting round-robin when all four are taken -- and
// decides: chained iff the slot is not fresh, the previous launch on it had
// the same tile count, the launch is marked (executor mark or =force), and the
// process's last cell launch was this cell's on this stream.
struct ChainStep {
  uint32_t* flags;
  uint32_t wait, set;
  bool chained;
};
template <class Alloc>
ChainStep chain_step(ackpt_lstm* cell, void* s, int64_t tiles, bool marked, Alloc&& alloc) {
  ackpt_lstm::ChainSlot* slot = nullptr;
  for (auto& sl : cell->chain_slots)
    if (sl.flags && sl.stream == s) slot = &sl;
  bool fresh = false;
  if (!slot || slot->tiles < tiles) {
    if (!slot) {
      for (auto& sl : cell->chain_slots)
        if (!sl.flags && !slot) slot = &sl;
      if (!slot) slot = &cell->chain_slots[cell->chain_victim++ % 4];
    }
    uint32_t* old = slot->flags;
    slot->flags = nullptr;  // (stays empty if the allocation throws)
    slot->flags = alloc(old, tiles);
    slot->stream = s;
    slot->tiles = tiles;
    slot->last_tiles = 0;
    slot->epoch = 0;
    fresh = true;
  }
  // (tile t must cover the same sequences in both launches: equal tile counts)
  const bool chained = !fresh && slot->last_tiles == tiles && marked && cell->chain_prev &&
                       cell->chain_prev_stream == s;
  slot->last_tiles = tiles;
  ChainStep r{slot->flags, chained ? slot->epoch : 0u, slot->epoch + 1, chained};
  if (++slot->epoch == 0) slot->epoch = 1;  // (flags compare by signed distance)
  chain_token().cell = cell;  // this launch is now the last cell launch
  chain_token().stream = s;
  return r;
}
// Tensor-core (tcgen05, 3xTF32) fused kernels, d = 8 (lstm_f32_tc.cu).
void tc_advance(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, cudaStream_t s);
void tc_forward_many(const ackpt_lstm* c, int64_t from, int count, const float* in, float* const* outs,
                     cudaStream_t s);
void tc_backward_many(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* adj_in,
                      float* adj_out, cudaStream_t s);
// Small-batch kernels (B <= kSmallBatch, any d, f32 / f64): one CTA per
// sequence, one thread per gate row (lstm_small.cu); per-step = count 1.
bool sb_ok(const ackpt_lstm* c);
bool sb_first(const ackpt_lstm* c);
template <typename T>
void sb_forward(const ackpt_lstm* c, int64_t from, int count, const void* in, void* out, void* const* outs,
                cudaStream_t s);
template <typename T>
void sb_reverse(const ackpt_lstm* c, int64_t from, int count, const void* const* states, const void* adj_in,
                void* adj_out, cudaStream_t s);
// Tensor-core kernels for d in {16, 32} (lstm_f32_tcd.cu); per-step = count 1.
bool tcd_ok(const ackpt_lstm* c, std::initializer_list<const void*> ptrs);      // forward kernels
bool tcd_rev_ok(const ackpt_lstm* c, std::initializer_list<const void*> ptrs);  // reverse kernels
void tcd_forward(const ackpt_lstm* c, int64_t from, int count, const float* in, float* out, float* const* outs,
                 cudaStream_t s);
void tcd_reverse(const ackpt_lstm* c, int64_t from, int count, const float* const* states, const float* adj_in,
                 float* adj_out, cudaStream_t s);
// At cell creation (d in {16, 32, 64}): the split-weight images the kernels
// copy into shared memory (d_wimg; d = 64 also the streamed W^T chunks,
// d_scratch); synchronous.
void tcd_build_images(ackpt_lstm* c);
// Generic path, any d <= 128, f32 or f64 (lstm_generic.cu).
template <typename T>
void generic_forward(const ackpt_lstm* c, int64_t step, const T* in, T* out, cudaStream_t s);
template <typename T>
void generic_backward(const ackpt_lstm* c, int64_t step, const T* st, const T* ai, T* ao,
                      cudaStream_t s);
template <typename T>
void generic_advance(const ackpt_lstm* c, int64_t from, int64_t to, const T* in, T* out,
                     cudaStream_t s);
template <typename T>
void launch_seed(const ackpt_lstm* c, const T* st, T* adj, cudaStream_t s);
template <typename T>
void launch_loss(const ackpt_lstm* c, const T* st, T* loss, cudaStream_t s);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline unsigned blocks_for(int64_t items, int threads) {
  return unsigned((items + threads - 1) / threads);
}

}  // namespace ackpt
