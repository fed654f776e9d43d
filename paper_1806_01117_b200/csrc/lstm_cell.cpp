// Device LSTM cell object and the ackpt_lstm_* C ABI (lstm.py:39-173).
#include "lstm_cell.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

namespace ackpt {
namespace {

template <typename T>
void round_into(const std::vector<double>& src, std::vector<unsigned char>& dst) {
  dst.resize(src.size() * sizeof(T));
  T* p = reinterpret_cast<T*>(dst.data());
  for (size_t i = 0; i < src.size(); ++i) p[i] = T(src[i]);
}

void check_step(const ackpt_lstm* c, int64_t step) {
  if (step < 0 || step >= c->n)
    fail(ACKPT_VALUE_ERROR,
         "step " + std::to_string(step) + " outside [0, " + std::to_string(c->n) + ")");
}

void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) fail(ACKPT_CUDA_ERROR, std::string("kernel launch: ") + cudaGetErrorString(e));
}

// fp32 pair kernels need an even batch and 8-byte aligned rows.
bool f32_fast(const ackpt_lstm* c, std::initializer_list<const void*> ptrs) {
  if (c->dtype != ACKPT_F32 || (c->d != 4 && c->d != 8) || (c->B & 1)) return false;
  for (const void* p : ptrs)
    if (reinterpret_cast<uintptr_t>(p) & 7u) return false;
  return true;
}

// Fused launches (advance / forward_many / backward_many) for d=8 pick a
// kernel family: 1 tcgen05 (default: the fastest measured at the C2 shape,
// DESIGN.md §3) or 0 packed FFMA2 (the documented fallback, also the family
// of the per-step kernels).  Env ACKPT_TC=0 selects FFMA2.  The families round
// differently (each within the fp32 tolerance); within one family the
// strategies stay bit-identical.
std::atomic<int> g_family{-1};  // -1: not yet read from the environment
int family() {
  int f = g_family.load(std::memory_order_relaxed);
  if (f < 0) {
    const char* e = std::getenv("ACKPT_TC");
    f = (e && std::string(e) == "0") ? 0 : 1;
    g_family.store(f, std::memory_order_relaxed);
  }
  return f;
}
bool tc_on() { return family() == 1; }

}  // namespace

// The executor's chain mark applies to the cell calls made here (and only
// here): see g_chain_native in common.h.
struct NativeCall {
  NativeCall() { g_chain_native = g_chain_hint; }
  ~NativeCall() { g_chain_native = 0; }
};

int lstm_op_forward(void* ctx, int64_t step, const void* in, void* out, void* stream) {
  NativeCall nc;
  return ackpt_lstm_forward(static_cast<ackpt_lstm*>(ctx), step, in, out, stream);
}
int lstm_op_backward(void* ctx, int64_t step, const void* st, const void* ai, void* ao,
                     void* stream) {
  NativeCall nc;
  return ackpt_lstm_backward(static_cast<ackpt_lstm*>(ctx), step, st, ai, ao, stream);
}
int lstm_op_seed(void* ctx, const void* fin, void* adj, void* stream) {
  return ackpt_lstm_seed(static_cast<ackpt_lstm*>(ctx), fin, adj, stream);
}
int lstm_op_advance(void* ctx, int64_t from, int64_t to, const void* in, void* out, void* stream) {
  NativeCall nc;
  return ackpt_lstm_advance(static_cast<ackpt_lstm*>(ctx), from, to, in, out, stream);
}
int lstm_op_forward_many(void* ctx, int64_t from, int64_t count, const void* in, void* const* outs,
                         void* stream) {
  NativeCall nc;
  return ackpt_lstm_forward_many(static_cast<ackpt_lstm*>(ctx), from, count, in, outs, stream);
}
int lstm_op_backward_many(void* ctx, int64_t from, int64_t count, const void* const* states,
                          const void* ai, void* ao, void* stream) {
  NativeCall nc;
  return ackpt_lstm_backward_many(static_cast<ackpt_lstm*>(ctx), from, count, states, ai, ao, stream);
}

}  // namespace ackpt

namespace ackpt {
void chain_release(ackpt_lstm* c) {
  bool any = false;
  for (auto& sl : c->chain_slots) any = any || sl.flags;
  if (any) cudaDeviceSynchronize();  // no kernel may still publish into the flags
  for (auto& sl : c->chain_slots) {
    if (sl.flags) cudaFree(sl.flags);
    sl = ackpt_lstm::ChainSlot{};
  }
  auto& t = chain_token();
  std::lock_guard<std::mutex> lk(t.mu);
  if (t.cell == c) t.cell = nullptr, t.stream = nullptr;
}
}  // namespace ackpt

extern "C" {

ACKPT_API int ackpt_lstm_create(int32_t d, int64_t n_steps, int64_t batch, int32_t dtype,
                                const double* w_f, const double* w_i, const double* w_o,
                                const double* w_c, const double* b_f, const double* b_i,
                                const double* b_o, const double* b_c, const double* xs,
                                const double* target, ackpt_lstm** out) {
  return ackpt::guard([&] {
    using ackpt::fail;
    if (d < 1 || d > ackpt::kMaxD) fail(ACKPT_VALUE_ERROR, "hidden size must be in [1, 128]");
    if (n_steps < 1) fail(ACKPT_VALUE_ERROR, "n_steps must be >= 1");
    if (batch < 1) fail(ACKPT_VALUE_ERROR, "batch must be >= 1");
    if (dtype != ACKPT_F32 && dtype != ACKPT_F64) fail(ACKPT_VALUE_ERROR, "dtype must be f32 or f64");
    std::unique_ptr<ackpt_lstm> c(new ackpt_lstm());
    c->d = d;
    c->n = n_steps;
    c->B = batch;
    c->dtype = dtype;
    c->esize = dtype == ACKPT_F32 ? 4 : 8;
    const double* W[4] = {w_f, w_i, w_o, w_c};
    const double* Bv[4] = {b_f, b_i, b_o, b_c};
    const size_t D = size_t(d);
    // W_h: the first d columns of each d x 2d gate matrix (z = [h; x], lstm.py:115)
    c->wh64.resize(4 * D * D);
    for (size_t g = 0; g < 4; ++g)
      for (size_t j = 0; j < D; ++j)
        for (size_t i = 0; i < D; ++i) c->wh64[(g * D + j) * D + i] = W[g][j * 2 * D + i];
    // xb[k][g][j] = sum_i W_g[j][d + i] x_k[i] + b_g[j], in float64
    c->xb64.resize(size_t(n_steps) * 4 * D);
    for (int64_t k = 0; k < n_steps; ++k)
      for (size_t g = 0; g < 4; ++g)
        for (size_t j = 0; j < D; ++j) {
          double acc = 0.0;
          for (size_t i = 0; i < D; ++i) acc += W[g][j * 2 * D + D + i] * xs[size_t(k) * D + i];
          c->xb64[(size_t(k) * 4 + g) * D + j] = acc + Bv[g][j];
        }
    c->target64.assign(target, target + D);
    if (dtype == ACKPT_F32) {
      ackpt::round_into<float>(c->wh64, c->wh_t);
      ackpt::round_into<float>(c->xb64, c->xb_t);
      ackpt::round_into<float>(c->target64, c->target_t);
    } else {
      ackpt::round_into<double>(c->wh64, c->wh_t);
      ackpt::round_into<double>(c->xb64, c->xb_t);
      ackpt::round_into<double>(c->target64, c->target_t);
    }
    ACKPT_CUDA_CHECK(cudaMalloc(&c->d_wh, c->wh_t.size()));
    ACKPT_CUDA_CHECK(cudaMalloc(&c->d_xb, c->xb_t.size()));
    ACKPT_CUDA_CHECK(cudaMemcpy(c->d_wh, c->wh_t.data(), c->wh_t.size(), cudaMemcpyHostToDevice));
    ACKPT_CUDA_CHECK(cudaMemcpy(c->d_xb, c->xb_t.data(), c->xb_t.size(), cudaMemcpyHostToDevice));
    {  // W_h transposed ([k][n] = W_h[n][k]): coalesced gate rows when W is read from global memory
      const size_t es = size_t(c->esize), R = 4 * D;
      std::vector<unsigned char> wt(c->wh_t.size());
      for (size_t r = 0; r < R; ++r)
        for (size_t k = 0; k < D; ++k) std::memcpy(&wt[(k * R + r) * es], &c->wh_t[(r * D + k) * es], es);
      ACKPT_CUDA_CHECK(cudaMalloc(&c->d_wht, wt.size()));
      ACKPT_CUDA_CHECK(cudaMemcpy(c->d_wht, wt.data(), wt.size(), cudaMemcpyHostToDevice));
    }
    if (dtype == ACKPT_F32 && (d <= 32 || d == 64)) {
      // per-gate pre-scaled projections for the fused fp32 advance (lstm_f32_math.cuh)
      const float scale[4] = {-1.4426950408889634f, -1.4426950408889634f, -1.4426950408889634f,
                              2.0f * 1.4426950408889634f};
      std::vector<float> xbs(c->xb64.size());
      for (int64_t k = 0; k < n_steps; ++k)
        for (size_t g = 0; g < 4; ++g)
          for (size_t j = 0; j < D; ++j) {
            const size_t at = (size_t(k) * 4 + g) * D + j;
            xbs[at] = float(c->xb64[at] * double(scale[g]));
          }
      ACKPT_CUDA_CHECK(cudaMalloc(&c->d_xbs, xbs.size() * sizeof(float)));
      ACKPT_CUDA_CHECK(cudaMemcpy(c->d_xbs, xbs.data(), xbs.size() * sizeof(float), cudaMemcpyHostToDevice));
      if (d == 16 || d == 32 || d == 64) {  // pre-scaled W for the tensor-core kernels
        std::vector<float> ws(size_t(4) * D * D);
        for (size_t g = 0; g < 4; ++g)
          for (size_t j = 0; j < D; ++j)
            for (size_t k = 0; k < D; ++k)
              ws[(g * D + j) * D + k] = float(c->wh64[(g * D + j) * D + k] * double(scale[g]));
        ACKPT_CUDA_CHECK(cudaMalloc(&c->d_ws, ws.size() * sizeof(float)));
        ACKPT_CUDA_CHECK(cudaMemcpy(c->d_ws, ws.data(), ws.size() * sizeof(float), cudaMemcpyHostToDevice));
        ackpt::tcd_build_images(c.get());  // shared-memory weight images, complete before any launch
      }
    }
    // pageable-host uploads may still be in flight on the legacy stream when
    // cudaMemcpy returns; the step kernels run on other (non-blocking) streams
    ACKPT_CUDA_CHECK(cudaDeviceSynchronize());
    *out = c.release();
  });
}

ACKPT_API int ackpt_lstm_destroy(ackpt_lstm* cell) {
  return ackpt::guard([&] {
    if (!cell) return;
    if (cell->d_wh) cudaFree(cell->d_wh);
    if (cell->d_wht) cudaFree(cell->d_wht);
    if (cell->d_xb) cudaFree(cell->d_xb);
    if (cell->d_xbs) cudaFree(cell->d_xbs);
    if (cell->d_ws) cudaFree(cell->d_ws);
    if (cell->d_scratch) cudaFree(cell->d_scratch);
    if (cell->d_wimg) cudaFree(cell->d_wimg);
    ackpt::chain_release(cell);
    delete cell;
  });
}

ACKPT_API int64_t ackpt_lstm_state_bytes(const ackpt_lstm* cell) {
  return cell ? 2 * int64_t(cell->d) * cell->B * int64_t(cell->esize) : -1;
}

ACKPT_API int ackpt_lstm_forward(const ackpt_lstm* cell, int64_t step, const void* state_in,
                                 void* state_out, void* stream) {
  return ackpt::guard([&] {
    ackpt::chain_touch(cell);
    ackpt::check_step(cell, step);
    auto s = static_cast<cudaStream_t>(stream);
    if (ackpt::sb_first(cell)) {
      if (cell->dtype == ACKPT_F32) ackpt::sb_forward<float>(cell, step, 1, state_in, state_out, nullptr, s);
      else ackpt::sb_forward<double>(cell, step, 1, state_in, state_out, nullptr, s);
    } else if (ackpt::tcd_ok(cell, {state_in, state_out})) {
      ackpt::tcd_forward(cell, step, 1, static_cast<const float*>(state_in), static_cast<float*>(state_out), nullptr,
                         s);
    } else if (ackpt::f32_fast(cell, {state_in, state_out})) {
      auto i = static_cast<const float*>(state_in);
      auto o = static_cast<float*>(state_out);
      if (cell->d == 8) ackpt::f32_forward<8>(cell, step, i, o, s);
      else ackpt::f32_forward<4>(cell, step, i, o, s);
    } else if (ackpt::sb_ok(cell)) {
      if (cell->dtype == ACKPT_F32) ackpt::sb_forward<float>(cell, step, 1, state_in, state_out, nullptr, s);
      else ackpt::sb_forward<double>(cell, step, 1, state_in, state_out, nullptr, s);
    } else if (cell->dtype == ACKPT_F32) {
      ackpt::generic_forward<float>(cell, step, static_cast<const float*>(state_in),
                                    static_cast<float*>(state_out), s);
    } else {
      ackpt::generic_forward<double>(cell, step, static_cast<const double*>(state_in),
                                     static_cast<double*>(state_out), s);
    }
    ackpt::check_launch();
  });
}

ACKPT_API int ackpt_lstm_advance(const ackpt_lstm* cell, int64_t from_step, int64_t to_step,
                                 const void* state_in, void* state_out, void* stream) {
  return ackpt::guard([&] {
    ackpt::chain_touch(cell);
    if (from_step < 0 || to_step > cell->n || from_step >= to_step)
      ackpt::fail(ACKPT_VALUE_ERROR, "advance range out of bounds");
    auto s = static_cast<cudaStream_t>(stream);
    if (ackpt::sb_first(cell)) {
      const int cnt = int(to_step - from_step);
      if (cell->dtype == ACKPT_F32) ackpt::sb_forward<float>(cell, from_step, cnt, state_in, state_out, nullptr, s);
      else ackpt::sb_forward<double>(cell, from_step, cnt, state_in, state_out, nullptr, s);
    } else if (ackpt::f32_fast(cell, {state_in, state_out})) {
      auto i = static_cast<const float*>(state_in);
      auto o = static_cast<float*>(state_out);
      if (cell->d == 8 && ackpt::tc_on()) ackpt::tc_advance(cell, from_step, int(to_step - from_step), i, o, s);
      else if (cell->d == 8) ackpt::f32_advance<8>(cell, from_step, to_step, i, o, s);
      else ackpt::f32_advance<4>(cell, from_step, to_step, i, o, s);
    } else if (ackpt::tcd_ok(cell, {state_in, state_out})) {
      ackpt::tcd_forward(cell, from_step, int(to_step - from_step), static_cast<const float*>(state_in),
                         static_cast<float*>(state_out), nullptr, s);
    } else if (ackpt::sb_ok(cell)) {
      const int cnt = int(to_step - from_step);
      if (cell->dtype == ACKPT_F32) ackpt::sb_forward<float>(cell, from_step, cnt, state_in, state_out, nullptr, s);
      else ackpt::sb_forward<double>(cell, from_step, cnt, state_in, state_out, nullptr, s);
    } else if (cell->dtype == ACKPT_F32) {
      ackpt::generic_advance<float>(cell, from_step, to_step, static_cast<const float*>(state_in),
                                    static_cast<float*>(state_out), s);
    } else {
      ackpt::generic_advance<double>(cell, from_step, to_step,
                                     static_cast<const double*>(state_in),
                                     static_cast<double*>(state_out), s);
    }
    ackpt::check_launch();
  });
}

ACKPT_API int ackpt_lstm_backward(const ackpt_lstm* cell, int64_t step, const void* state,
                                  const void* adjoint_in, void* adjoint_out, void* stream) {
  return ackpt::guard([&] {
    ackpt::chain_touch(cell);
    ackpt::check_step(cell, step);
    auto s = static_cast<cudaStream_t>(stream);
    if (ackpt::sb_first(cell)) {
      if (cell->dtype == ACKPT_F32) ackpt::sb_reverse<float>(cell, step, 1, &state, adjoint_in, adjoint_out, s);
      else ackpt::sb_reverse<double>(cell, step, 1, &state, adjoint_in, adjoint_out, s);
    } else if (ackpt::tcd_rev_ok(cell, {state, adjoint_in, adjoint_out})) {
      const float* st = static_cast<const float*>(state);
      ackpt::tcd_reverse(cell, step, 1, &st, static_cast<const float*>(adjoint_in), static_cast<float*>(adjoint_out),
                         s);
    } else if (ackpt::f32_fast(cell, {state, adjoint_in, adjoint_out})) {
      auto x = static_cast<const float*>(state);
      auto a = static_cast<const float*>(adjoint_in);
      auto o = static_cast<float*>(adjoint_out);
      if (cell->d == 8) ackpt::f32_backward<8>(cell, step, x, a, o, s);
      else ackpt::f32_backward<4>(cell, step, x, a, o, s);
    } else if (ackpt::sb_ok(cell)) {
      if (cell->dtype == ACKPT_F32) ackpt::sb_reverse<float>(cell, step, 1, &state, adjoint_in, adjoint_out, s);
      else ackpt::sb_reverse<double>(cell, step, 1, &state, adjoint_in, adjoint_out, s);
    } else if (cell->dtype == ACKPT_F32) {
      ackpt::generic_backward<float>(cell, step, static_cast<const float*>(state),
                                     static_cast<const float*>(adjoint_in),
                                     static_cast<float*>(adjoint_out), s);
    } else {
      ackpt::generic_backward<double>(cell, step, static_cast<const double*>(state),
                                      static_cast<const double*>(adjoint_in),
                                      static_cast<double*>(adjoint_out), s);
    }
    ackpt::check_launch();
  });
}

ACKPT_API int ackpt_lstm_forward_many(const ackpt_lstm* cell, int64_t from_step, int64_t count,
                                      const void* state_in, void* const* states_out, void* stream) {
  return ackpt::guard([&] {
    ackpt::chain_touch(cell);
    if (count < 1 || count > ACKPT_MAX_FUSED) ackpt::fail(ACKPT_VALUE_ERROR, "count must be in [1, 64]");
    if (from_step < 0 || from_step + count > cell->n) ackpt::fail(ACKPT_VALUE_ERROR, "steps out of range");
    auto s = static_cast<cudaStream_t>(stream);
    std::vector<const void*> all{state_in};
    for (int64_t i = 0; i < count; ++i) all.push_back(states_out[i]);
    bool fast = !ackpt::sb_first(cell) && ackpt::f32_fast(cell, {});
    for (const void* p : all) fast = fast && !(reinterpret_cast<uintptr_t>(p) & 7u);
    if (fast) {
      auto in = static_cast<const float*>(state_in);
      auto outs = reinterpret_cast<float* const*>(states_out);
      if (cell->d == 8 && ackpt::tc_on()) ackpt::tc_forward_many(cell, from_step, int(count), in, outs, s);
      else if (cell->d == 8) ackpt::f32_forward_many<8>(cell, from_step, int(count), in, outs, s);
      else ackpt::f32_forward_many<4>(cell, from_step, int(count), in, outs, s);
      ackpt::check_launch();
      return;
    }
    bool tcd = !ackpt::sb_first(cell) && ackpt::tcd_ok(cell, {});
    for (const void* q : all) tcd = tcd && !(reinterpret_cast<uintptr_t>(q) & 3u);
    if (tcd) {
      ackpt::tcd_forward(cell, from_step, int(count), static_cast<const float*>(state_in), nullptr,
                         reinterpret_cast<float* const*>(states_out), s);
      ackpt::check_launch();
      return;
    }
    if (ackpt::sb_ok(cell)) {
      if (cell->dtype == ACKPT_F32) ackpt::sb_forward<float>(cell, from_step, int(count), state_in, nullptr, states_out, s);
      else ackpt::sb_forward<double>(cell, from_step, int(count), state_in, nullptr, states_out, s);
      ackpt::check_launch();
      return;
    }
    const void* cur = state_in;  // per-step launches
    for (int64_t i = 0; i < count; ++i) {
      int rc = ackpt_lstm_forward(cell, from_step + i, cur, states_out[i], stream);
      if (rc != ACKPT_OK) ackpt::fail(rc, ackpt_last_error());
      cur = states_out[i];
    }
  });
}

ACKPT_API int ackpt_lstm_backward_many(const ackpt_lstm* cell, int64_t from_step, int64_t count,
                                       const void* const* states, const void* adjoint_in,
                                       void* adjoint_out, void* stream) {
  return ackpt::guard([&] {
    ackpt::chain_touch(cell);
    if (count < 1 || count > ACKPT_MAX_FUSED) ackpt::fail(ACKPT_VALUE_ERROR, "count must be in [1, 64]");
    if (from_step < 0 || from_step + count > cell->n) ackpt::fail(ACKPT_VALUE_ERROR, "steps out of range");
    auto s = static_cast<cudaStream_t>(stream);
    const bool sbf = ackpt::sb_first(cell);
    bool tcd = !sbf && ackpt::tcd_rev_ok(cell, {adjoint_in, adjoint_out});
    for (int64_t i = 0; i < count; ++i) tcd = tcd && !(reinterpret_cast<uintptr_t>(states[i]) & 3u);
    if (tcd) {
      ackpt::tcd_reverse(cell, from_step, int(count), reinterpret_cast<const float* const*>(states),
                         static_cast<const float*>(adjoint_in), static_cast<float*>(adjoint_out), s);
      ackpt::check_launch();
      return;
    }
    bool fast = !sbf && ackpt::f32_fast(cell, {adjoint_in, adjoint_out});
    for (int64_t i = 0; i < count; ++i) fast = fast && !(reinterpret_cast<uintptr_t>(states[i]) & 7u);
    if (!fast && ackpt::sb_ok(cell)) {
      if (cell->dtype == ACKPT_F32) ackpt::sb_reverse<float>(cell, from_step, int(count), states, adjoint_in, adjoint_out, s);
      else ackpt::sb_reverse<double>(cell, from_step, int(count), states, adjoint_in, adjoint_out, s);
      ackpt::check_launch();
      return;
    }
    if (!fast)
      ackpt::fail(ACKPT_VALUE_ERROR, "fused backward needs a fused kernel (fp32 d in {4, 8, 16, 32} or the CTA-per-sequence kernels)");
    auto sp = reinterpret_cast<const float* const*>(states);
    auto ai = static_cast<const float*>(adjoint_in);
    auto ao = static_cast<float*>(adjoint_out);
    if (cell->d == 8 && ackpt::tc_on()) ackpt::tc_backward_many(cell, from_step, int(count), sp, ai, ao, s);
    else if (cell->d == 8) ackpt::f32_backward_many<8>(cell, from_step, int(count), sp, ai, ao, s);
    else ackpt::f32_backward_many<4>(cell, from_step, int(count), sp, ai, ao, s);
    ackpt::check_launch();
  });
}

ACKPT_API int ackpt_lstm_seed(const ackpt_lstm* cell, const void* final_state, void* adjoint_out,
                              void* stream) {
  return ackpt::guard([&] {
    ackpt::chain_touch(cell);
    auto s = static_cast<cudaStream_t>(stream);
    if (cell->dtype == ACKPT_F32)
      ackpt::launch_seed<float>(cell, static_cast<const float*>(final_state),
                                static_cast<float*>(adjoint_out), s);
    else
      ackpt::launch_seed<double>(cell, static_cast<const double*>(final_state),
                                 static_cast<double*>(adjoint_out), s);
    ackpt::check_launch();
  });
}

ACKPT_API int ackpt_lstm_loss(const ackpt_lstm* cell, const void* final_state, void* loss_out,
                              void* stream) {
  return ackpt::guard([&] {
    ackpt::chain_touch(cell);
    auto s = static_cast<cudaStream_t>(stream);
    if (cell->dtype == ACKPT_F32)
      ackpt::launch_loss<float>(cell, static_cast<const float*>(final_state),
                                static_cast<float*>(loss_out), s);
    else
      ackpt::launch_loss<double>(cell, static_cast<const double*>(final_state),
                                 static_cast<double*>(loss_out), s);
    ackpt::check_launch();
  });
}

ACKPT_API int ackpt_set_fused_family(int32_t family) {
  return ackpt::guard([&] {
    if (family < 0 || family > 1) ackpt::fail(ACKPT_VALUE_ERROR, "family must be 0 (ffma2) or 1 (tcgen05)");
    ackpt::g_family.store(family);
  });
}

ACKPT_API int32_t ackpt_get_fused_family(void) { return ackpt::family(); }

ACKPT_API int ackpt_chain_selftest(void) {
  // The launch-chain bookkeeping (chain_touch / chain_step, lstm_cell.h) on
  // host-only cells with a fake flag allocator: no CUDA call is made.
  return ackpt::guard([&] {
    using namespace ackpt;
    static uint32_t fake[4][64];
    int allocs = 0, frees = 0;
    auto alloc = [&](uint32_t* old, int64_t) {
      if (old) ++frees;
      return fake[allocs++ % 4];
    };
    ackpt_lstm A, Bc;
    void* s1 = reinterpret_cast<void*>(0x10);
    void* s2 = reinterpret_cast<void*>(0x20);
    void* s0 = nullptr;  // the legacy default stream is a valid handle
    auto launch = [&](ackpt_lstm& c, void* s, int64_t tiles, bool marked) {
      chain_touch(&c);  // every cell API entry
      std::lock_guard<std::mutex> lk(chain_token().mu);
      return chain_step(&c, s, tiles, marked, alloc);
    };
    auto expect = [&](bool ok, const char* what) {
      if (!ok) fail(ACKPT_EXECUTION_ERROR, std::string("chain self-test: ") + what);
    };
    ChainStep a = launch(A, s1, 16, true);
    expect(!a.chained && a.wait == 0 && a.set == 1, "first launch on a fresh slot is unchained");
    ChainStep b = launch(A, s1, 16, true);
    expect(b.chained && b.wait == a.set && b.set == a.set + 1 && b.flags == a.flags, "back-to-back launch chains");
    expect(!launch(A, s1, 16, false).chained, "an unmarked launch never chains");
    launch(A, s1, 16, true);
    launch(Bc, s1, 16, true);  // another cell in between
    expect(!launch(A, s1, 16, true).chained, "no chaining across another cell's launch");
    expect(launch(A, s1, 16, true).chained, "chains again once adjacent");
    expect(!launch(A, s2, 16, true).chained, "a new stream starts unchained (own slot)");
    expect(!launch(A, s1, 16, true).chained, "no chaining across a launch on another stream");
    expect(!launch(A, s1, 32, true).chained, "a larger tiling reallocates: unchained");
    expect(!launch(A, s1, 16, true).chained, "different tile counts never chain");
    expect(launch(A, s1, 16, true).chained, "equal tile counts chain again");
    launch(A, s0, 16, true);
    expect(launch(A, s0, 16, true).chained, "stream 0 chains with itself");
    chain_touch(&Bc);  // e.g. a seed kernel of another cell
    expect(!launch(A, s0, 16, true).chained, "any cell API call in between breaks the chain");
    void* s3 = reinterpret_cast<void*>(0x30);
    void* s4 = reinterpret_cast<void*>(0x40);
    const int frees0 = frees;
    launch(A, s3, 16, true);
    launch(A, s4, 16, true);  // fifth stream: evicts a slot
    expect(frees == frees0 + 1, "the fifth stream evicts one slot");
    int live = 0;
    for (auto& sl : A.chain_slots) live += sl.flags != nullptr;
    expect(live == 4, "four slots at most");
    {
      std::lock_guard<std::mutex> lk(chain_token().mu);
      chain_token().cell = nullptr;  // leave no host-only cell in the token
      chain_token().stream = nullptr;
    }
  });
}

ACKPT_API int ackpt_lstm_operator(ackpt_lstm* cell, ackpt_operator* out) {
  return ackpt::guard([&] {
    out->ctx = cell;
    out->forward = ackpt::lstm_op_forward;
    out->backward = ackpt::lstm_op_backward;
    out->seed = ackpt::lstm_op_seed;
    out->advance = ackpt::lstm_op_advance;
    out->state_bytes = ackpt_lstm_state_bytes(cell);
    out->n_steps = cell->n;
    const bool fused = (cell->dtype == ACKPT_F32 && (cell->d == 4 || cell->d == 8) && !(cell->B & 1)) ||
                       ackpt::tcd_ok(cell, {}) || ackpt::sb_ok(cell);
    out->forward_many = fused ? ackpt::lstm_op_forward_many : nullptr;
    out->backward_many = fused ? ackpt::lstm_op_backward_many : nullptr;
  });
}

}  // extern "C"
