// Generic LSTM step kernels (any d <= 128, f32 or f64), K3 seed and K4 loss.
//
// This is the path for hidden sizes without a specialised kernel and for the
// float64 build that reproduces the reference's arithmetic type
// (lstm.py:36, "<f8").  One thread per batch element; feature rows are
// batch-contiguous so every global access is coalesced across the warp.
// Weights and the step's input projection are read through the read-only
// path (uniform addresses -> L1 broadcast).  Per-element scratch (h, dh)
// lives in local memory for large d; this path is for parity, not speed.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "lstm_cell.h"

namespace ackpt {
namespace gk {

__device__ __forceinline__ float sigmoid(float z) { return 1.0f / (1.0f + expf(-z)); }
__device__ __forceinline__ double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }
__device__ __forceinline__ float tanh_(float z) { return tanhf(z); }
__device__ __forceinline__ double tanh_(double z) { return tanh(z); }

template <typename T>
__device__ __forceinline__ void gate_preacts(const T* __restrict__ wh, const T* __restrict__ xb,
                                             const T* h, int d, int j, T (&a)[4]) {
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    T acc = __ldg(xb + g * d + j);
    const T* w = wh + (int64_t(g) * d + j) * d;
#pragma unroll 1
    for (int i = 0; i < d; ++i) acc = fma(__ldg(w + i), h[i], acc);
    a[g] = acc;
  }
}

template <typename T>
__global__ void __launch_bounds__(128) fwd(const T* __restrict__ in, T* __restrict__ out,
                                           int64_t B, int d, const T* __restrict__ wh,
                                           const T* __restrict__ xb) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  T h[kMaxD];
#pragma unroll 1
  for (int i = 0; i < d; ++i) h[i] = in[int64_t(i) * B + b];
#pragma unroll 1
  for (int j = 0; j < d; ++j) {
    T a[4];
    gate_preacts(wh, xb, h, d, j, a);
    const T f = sigmoid(a[0]), ig = sigmoid(a[1]), o = sigmoid(a[2]), g = tanh_(a[3]);
    const T cn = f * in[int64_t(d + j) * B + b] + ig * g;  // lstm.py:127
    out[int64_t(d + j) * B + b] = cn;
    out[int64_t(j) * B + b] = o * tanh_(cn);               // lstm.py:128
  }
}

template <typename T>
__global__ void __launch_bounds__(128) adv(const T* __restrict__ in, T* __restrict__ out,
                                           int64_t B, int d, const T* __restrict__ wh,
                                           const T* __restrict__ xb_all, int64_t from,
                                           int64_t to) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  T h[kMaxD], c[kMaxD], hn[kMaxD];
#pragma unroll 1
  for (int i = 0; i < d; ++i) {
    h[i] = in[int64_t(i) * B + b];
    c[i] = in[int64_t(d + i) * B + b];
  }
#pragma unroll 1
  for (int64_t k = from; k < to; ++k) {
    const T* xb = xb_all + k * 4 * d;
#pragma unroll 1
    for (int j = 0; j < d; ++j) {
      T a[4];
      gate_preacts(wh, xb, h, d, j, a);
      const T f = sigmoid(a[0]), ig = sigmoid(a[1]), o = sigmoid(a[2]), g = tanh_(a[3]);
      c[j] = f * c[j] + ig * g;
      hn[j] = o * tanh_(c[j]);
    }
#pragma unroll 1
    for (int j = 0; j < d; ++j) h[j] = hn[j];
  }
#pragma unroll 1
  for (int i = 0; i < d; ++i) {
    out[int64_t(i) * B + b] = h[i];
    out[int64_t(d + i) * B + b] = c[i];
  }
}

template <typename T>
__global__ void __launch_bounds__(128) bwd(const T* __restrict__ st, const T* __restrict__ adj_in,
                                           T* __restrict__ adj_out, int64_t B, int d,
                                           const T* __restrict__ wh, const T* __restrict__ xb) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  T h[kMaxD], dh[kMaxD];
#pragma unroll 1
  for (int i = 0; i < d; ++i) {
    h[i] = st[int64_t(i) * B + b];
    dh[i] = T(0);
  }
#pragma unroll 1
  for (int j = 0; j < d; ++j) {
    T a[4];
    gate_preacts(wh, xb, h, d, j, a);
    const T f = sigmoid(a[0]), ig = sigmoid(a[1]), o = sigmoid(a[2]), g = tanh_(a[3]);
    const T c = st[int64_t(d + j) * B + b];
    const T cn = f * c + ig * g;
    const T t = tanh_(cn);
    const T dhn = adj_in[int64_t(j) * B + b];
    const T dco = adj_in[int64_t(d + j) * B + b] + dhn * o * (T(1) - t * t);  // lstm.py:143
    const T da[4] = {dco * c * f * (T(1) - f),                                 // lstm.py:144
                     dco * g * ig * (T(1) - ig),                               // lstm.py:145
                     dhn * t * o * (T(1) - o),                                 // lstm.py:142,146
                     dco * ig * (T(1) - g * g)};                               // lstm.py:147
#pragma unroll
    for (int g4 = 0; g4 < 4; ++g4) {
      const T* w = wh + (int64_t(g4) * d + j) * d;
#pragma unroll 1
      for (int m = 0; m < d; ++m) dh[m] = fma(__ldg(w + m), da[g4], dh[m]);  // lstm.py:149
    }
    adj_out[int64_t(d + j) * B + b] = dco * f;  // lstm.py:151
  }
#pragma unroll 1
  for (int m = 0; m < d; ++m) adj_out[int64_t(m) * B + b] = dh[m];  // lstm.py:150
}

template <typename T>
__global__ void seed(const T* __restrict__ st, T* __restrict__ adj, int64_t B, int d,
                     const __grid_constant__ TargetParams<T> tp) {
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = int64_t(d) * B;
  if (idx >= total) return;
  const int j = int(idx / B);
  adj[idx] = T(2) * (st[idx] - tp.target[j]);  // lstm.py:163
  adj[total + idx] = T(0);
}

template <typename T>
__global__ void loss(const T* __restrict__ st, T* __restrict__ out, int64_t B, int d,
                     const __grid_constant__ TargetParams<T> tp) {
  const int64_t b = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= B) return;
  T acc = T(0);
  for (int j = 0; j < d; ++j) {
    const T diff = st[int64_t(j) * B + b] - tp.target[j];
    acc = fma(diff, diff, acc);  // lstm.py:157-158
  }
  out[b] = acc;
}

template <typename T>
TargetParams<T> target_params(const ackpt_lstm* c) {
  TargetParams<T> tp;
  std::memset(&tp, 0, sizeof(tp));
  std::memcpy(tp.target, c->target_t.data(), size_t(c->d) * sizeof(T));
  return tp;
}

}  // namespace gk

template <typename T>
void generic_forward(const ackpt_lstm* c, int64_t step, const T* in, T* out, cudaStream_t s) {
  gk::fwd<T><<<blocks_for(c->B, 128), 128, 0, s>>>(
      in, out, c->B, c->d, static_cast<const T*>(c->d_wh),
      static_cast<const T*>(c->d_xb) + size_t(step) * 4 * size_t(c->d));
}

template <typename T>
void generic_backward(const ackpt_lstm* c, int64_t step, const T* st, const T* ai, T* ao,
                      cudaStream_t s) {
  gk::bwd<T><<<blocks_for(c->B, 128), 128, 0, s>>>(
      st, ai, ao, c->B, c->d, static_cast<const T*>(c->d_wh),
      static_cast<const T*>(c->d_xb) + size_t(step) * 4 * size_t(c->d));
}

template <typename T>
void generic_advance(const ackpt_lstm* c, int64_t from, int64_t to, const T* in, T* out,
                     cudaStream_t s) {
  gk::adv<T><<<blocks_for(c->B, 128), 128, 0, s>>>(in, out, c->B, c->d,
                                                   static_cast<const T*>(c->d_wh),
                                                   static_cast<const T*>(c->d_xb), from, to);
}

template <typename T>
void launch_seed(const ackpt_lstm* c, const T* st, T* adj, cudaStream_t s) {
  gk::seed<T><<<blocks_for(int64_t(c->d) * c->B, 256), 256, 0, s>>>(st, adj, c->B, c->d,
                                                                     gk::target_params<T>(c));
}

template <typename T>
void launch_loss(const ackpt_lstm* c, const T* st, T* out, cudaStream_t s) {
  gk::loss<T><<<blocks_for(c->B, 256), 256, 0, s>>>(st, out, c->B, c->d, gk::target_params<T>(c));
}

#define ACKPT_INST(T)                                                                         \
  template void generic_forward<T>(const ackpt_lstm*, int64_t, const T*, T*, cudaStream_t);   \
  template void generic_backward<T>(const ackpt_lstm*, int64_t, const T*, const T*, T*,       \
                                    cudaStream_t);                                            \
  template void generic_advance<T>(const ackpt_lstm*, int64_t, int64_t, const T*, T*,         \
                                   cudaStream_t);                                             \
  template void launch_seed<T>(const ackpt_lstm*, const T*, T*, cudaStream_t);                \
  template void launch_loss<T>(const ackpt_lstm*, const T*, T*, cudaStream_t);
ACKPT_INST(float)
ACKPT_INST(double)
#undef ACKPT_INST

}  // namespace ackpt
