// fp32 LSTM step kernels for sm_100a, hidden size D in {4, 8}: K1 forward,
// K2 adjoint, K1f fused advance.  Register-staged variant: every thread loads
// its rows straight into registers (all loads issued before any math, so each
// warp keeps 2D (or 4D) 8-byte requests in flight), computes, stores.
// Included by lstm_f32_d<D>.cu, which instantiate one D each.
//
// Reference operator: lstm.py:110-152 (gates, forward step, exact adjoint).
//
//  * Each thread owns 2 consecutive batch elements (one float2 pair).
//    Feature row j of h (or c, dh, dc) for them is one 8-byte load; a warp
//    covers a contiguous 256 B span of that row: fully coalesced 32 B sectors.
//    Callers require even B and 8-byte aligned pointers.
//  * Packed fp32: fma.rn.f32x2 (FFMA2) with the weight as a uniform-register
//    scalar broadcast (ptxas loads the __grid_constant__ parameter block with
//    LDCU), so the 4d x d recurrent matvec costs 2 d^2 FFMA2 per element.
//  * Activation math: lstm_f32_math.cuh (pre-scaled weights, one shared MUFU
//    reciprocal per hidden unit).
#pragma once

#include <cuda_runtime.h>

#include <cstring>

#include "lstm_f32_math.cuh"

namespace ackpt {
namespace f32k {

using namespace f32m;

__device__ __forceinline__ float2 ld2(const float* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void st2(float* p, float2 v) {
  asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB)
    fwd_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t B,
               const __grid_constant__ ScaledParams<D> p) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
  if (b0 >= B) return;
  const float* src = in + b0;
  float* dst = out + b0;
  float2 h[D], c[D], hn[D];
#pragma unroll
  for (int j = 0; j < D; ++j) h[j] = ld2(src + int64_t(j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = ld2(src + int64_t(D + j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    float2 af, ai, ao, ag;
    preacts<D>(p.ws, p.xbs, h, j, af, ai, ao, ag);
    hn[j] = fwd_unit(af, ai, ao, ag, c[j]);
  }
#pragma unroll
  for (int j = 0; j < D; ++j) st2(dst + int64_t(j) * B, hn[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) st2(dst + int64_t(D + j) * B, c[j]);
}

template <int D, int MINB>
__global__ void __launch_bounds__(256, MINB)
    bwd_kernel(const float* __restrict__ st, const float* __restrict__ adj_in,
               float* __restrict__ adj_out, int64_t B, const __grid_constant__ ScaledParams<D> p) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
  if (b0 >= B) return;
  const float* xs = st + b0;
  const float* as = adj_in + b0;
  float* dst = adj_out + b0;
  float2 h[D], c[D], dh[D], dc[D];
#pragma unroll
  for (int j = 0; j < D; ++j) h[j] = ld2(xs + int64_t(j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = ld2(xs + int64_t(D + j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) dh[j] = ld2(as + int64_t(j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) dc[j] = ld2(as + int64_t(D + j) * B);
  float2 acc[D];
#pragma unroll
  for (int m = 0; m < D; ++m) acc[m] = bc(0.0f);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    float2 af, ai, ao, ag, daf, dai, dao, dag;
    preacts<D>(p.ws, p.xbs, h, j, af, ai, ao, ag);
    bwd_unit(af, ai, ao, ag, c[j], dh[j], dc[j], daf, dai, dao, dag, dc[j]);
    // dh += sum_g (scale_g W_g[j, :d])^T (da_g / scale_g)   (lstm.py:149-150)
#pragma unroll
    for (int m = 0; m < D; ++m) {
      acc[m] = fma2(bc(p.ws[0][j][m]), daf, acc[m]);
      acc[m] = fma2(bc(p.ws[1][j][m]), dai, acc[m]);
      acc[m] = fma2(bc(p.ws[2][j][m]), dao, acc[m]);
      acc[m] = fma2(bc(p.ws[3][j][m]), dag, acc[m]);
    }
  }
#pragma unroll
  for (int j = 0; j < D; ++j) st2(dst + int64_t(j) * B, acc[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) st2(dst + int64_t(D + j) * B, dc[j]);
}

// Fused forward over [from, to): state in registers; per step only the
// (scaled) input projection of that step is read (uniform broadcast loads).
// Same arithmetic as fwd_kernel, so results are bit-identical to a chain of
// per-step launches.  One launch moves 2S bytes for any number of steps.
template <int D>
struct AdvParams {
  float ws[4][D][D];
};

template <int D>
__global__ void __launch_bounds__(256, 2)
    adv_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t B,
               const float* __restrict__ xbs_all, int64_t from, int64_t to,
               const __grid_constant__ AdvParams<D> p) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
  if (b0 >= B) return;
  float2 h[D], c[D], hn[D];
#pragma unroll
  for (int j = 0; j < D; ++j) h[j] = ld2(in + b0 + int64_t(j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = ld2(in + b0 + int64_t(D + j) * B);
  for (int64_t k = from; k < to; ++k) {
    float xbs[4][D];
    const float4* src = reinterpret_cast<const float4*>(xbs_all + k * 4 * D);
#pragma unroll
    for (int v = 0; v < D; ++v) {
      const float4 x = __ldg(src + v);
      xbs[(4 * v) / D][(4 * v) % D] = x.x;
      xbs[(4 * v + 1) / D][(4 * v + 1) % D] = x.y;
      xbs[(4 * v + 2) / D][(4 * v + 2) % D] = x.z;
      xbs[(4 * v + 3) / D][(4 * v + 3) % D] = x.w;
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float2 af, ai, ao, ag;
      preacts<D>(p.ws, xbs, h, j, af, ai, ao, ag);
      hn[j] = fwd_unit(af, ai, ao, ag, c[j]);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) h[j] = hn[j];
  }
#pragma unroll
  for (int j = 0; j < D; ++j) st2(out + b0 + int64_t(j) * B, h[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) st2(out + b0 + int64_t(D + j) * B, c[j]);
}

// Scaled input projections of step k from the device table (uniform loads).
template <int D>
__device__ __forceinline__ void load_xbs(const float* __restrict__ xbs_all, int64_t k, float (&xbs)[4][D]) {
  const float4* src = reinterpret_cast<const float4*>(xbs_all + k * 4 * D);
#pragma unroll
  for (int v = 0; v < D; ++v) {
    const float4 x = __ldg(src + v);
    xbs[(4 * v) / D][(4 * v) % D] = x.x;
    xbs[(4 * v + 1) / D][(4 * v + 1) % D] = x.y;
    xbs[(4 * v + 2) / D][(4 * v + 2) % D] = x.z;
    xbs[(4 * v + 3) / D][(4 * v + 3) % D] = x.w;
  }
}

struct StatePtrs {
  const float* p[ACKPT_MAX_FUSED];
};
struct OutPtrs {
  float* p[ACKPT_MAX_FUSED];
};

// Fused TapeForward: steps [from, from+count), the state after each step
// stored to outs.p[i]; the state itself never leaves registers, so a step
// costs S of HBM writes instead of 2S.  Bit-identical to per-step launches.
template <int D>
__global__ void __launch_bounds__(256, 2)
    tape_kernel(const float* __restrict__ in, int64_t B, const float* __restrict__ xbs_all,
                int64_t from, int count, const __grid_constant__ AdvParams<D> p,
                const __grid_constant__ OutPtrs outs) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
  if (b0 >= B) return;
  float2 h[D], c[D], hn[D];
#pragma unroll
  for (int j = 0; j < D; ++j) h[j] = ld2(in + b0 + int64_t(j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = ld2(in + b0 + int64_t(D + j) * B);
  for (int i = 0; i < count; ++i) {
    float xbs[4][D];
    load_xbs<D>(xbs_all, from + i, xbs);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float2 af, ai, ao, ag;
      preacts<D>(p.ws, xbs, h, j, af, ai, ao, ag);
      hn[j] = fwd_unit(af, ai, ao, ag, c[j]);
    }
    float* dst = outs.p[i] + b0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      h[j] = hn[j];
      st2(dst + int64_t(j) * B, hn[j]);
    }
#pragma unroll
    for (int j = 0; j < D; ++j) st2(dst + int64_t(D + j) * B, c[j]);
  }
}

// Fused run of Reverse actions: steps from+count-1 down to from; the adjoint
// stays in registers, each step reads only its taped state (S instead of 3S
// of HBM traffic).  Bit-identical to per-step launches.
template <int D>
__global__ void __launch_bounds__(256, 2)
    rev_kernel(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B,
               const float* __restrict__ xbs_all, int64_t from, int count,
               const __grid_constant__ AdvParams<D> p, const __grid_constant__ StatePtrs states) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 2;
  if (b0 >= B) return;
  float2 dh[D], dc[D];
#pragma unroll
  for (int j = 0; j < D; ++j) dh[j] = ld2(adj_in + b0 + int64_t(j) * B);
#pragma unroll
  for (int j = 0; j < D; ++j) dc[j] = ld2(adj_in + b0 + int64_t(D + j) * B);
  for (int i = count - 1; i >= 0; --i) {
    const float* xs = states.p[i] + b0;
    float2 h[D], c[D];
#pragma unroll
    for (int j = 0; j < D; ++j) h[j] = ld2(xs + int64_t(j) * B);
#pragma unroll
    for (int j = 0; j < D; ++j) c[j] = ld2(xs + int64_t(D + j) * B);
    float xbs[4][D];
    load_xbs<D>(xbs_all, from + i, xbs);
    float2 acc[D];
#pragma unroll
    for (int m = 0; m < D; ++m) acc[m] = bc(0.0f);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float2 af, ai, ao, ag, daf, dai, dao, dag;
      preacts<D>(p.ws, xbs, h, j, af, ai, ao, ag);
      bwd_unit(af, ai, ao, ag, c[j], dh[j], dc[j], daf, dai, dao, dag, dc[j]);
#pragma unroll
      for (int m = 0; m < D; ++m) {
        acc[m] = fma2(bc(p.ws[0][j][m]), daf, acc[m]);
        acc[m] = fma2(bc(p.ws[1][j][m]), dai, acc[m]);
        acc[m] = fma2(bc(p.ws[2][j][m]), dao, acc[m]);
        acc[m] = fma2(bc(p.ws[3][j][m]), dag, acc[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < D; ++m) dh[m] = acc[m];
  }
#pragma unroll
  for (int j = 0; j < D; ++j) st2(adj_out + b0 + int64_t(j) * B, dh[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) st2(adj_out + b0 + int64_t(D + j) * B, dc[j]);
}

}  // namespace f32k

template <int D>
f32k::AdvParams<D> adv_params(const ackpt_lstm* c) {
  f32k::AdvParams<D> p;
  f32m::ScaledParams<D> sp;
  f32m::fill_scaled<D>(c, -1, sp);
  std::memcpy(p.ws, sp.ws, sizeof(p.ws));
  return p;
}

template <int D>
void f32_forward_many(const ackpt_lstm* c, int64_t from, int count, const float* in,
                      float* const* outs, cudaStream_t s) {
  f32k::OutPtrs o;
  for (int i = 0; i < count; ++i) o.p[i] = outs[i];
  f32k::tape_kernel<D><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(
      in, c->B, static_cast<const float*>(c->d_xbs), from, count, adv_params<D>(c), o);
}

template <int D>
void f32_backward_many(const ackpt_lstm* c, int64_t from, int count, const float* const* states,
                       const float* adj_in, float* adj_out, cudaStream_t s) {
  f32k::StatePtrs sp;
  for (int i = 0; i < count; ++i) sp.p[i] = states[i];
  f32k::rev_kernel<D><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(
      adj_in, adj_out, c->B, static_cast<const float*>(c->d_xbs), from, count, adv_params<D>(c), sp);
}

template <int D, int MINB>
void f32_forward_v(const ackpt_lstm* c, int64_t step, const float* in, float* out, cudaStream_t s) {
  f32m::ScaledParams<D> p;
  f32m::fill_scaled<D>(c, step, p);
  f32k::fwd_kernel<D, MINB><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(in, out, c->B, p);
}

template <int D, int MINB>
void f32_backward_v(const ackpt_lstm* c, int64_t step, const float* st, const float* ai, float* ao,
                    cudaStream_t s) {
  f32m::ScaledParams<D> p;
  f32m::fill_scaled<D>(c, step, p);
  f32k::bwd_kernel<D, MINB><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(st, ai, ao, c->B, p);
}

template <int D>
void f32_forward(const ackpt_lstm* c, int64_t step, const float* in, float* out, cudaStream_t s) {
  f32_forward_v<D, 2>(c, step, in, out, s);
}
template <int D>
void f32_backward(const ackpt_lstm* c, int64_t step, const float* st, const float* ai, float* ao,
                  cudaStream_t s) {
  f32_backward_v<D, 2>(c, step, st, ai, ao, s);
}

template <int D>
void f32_advance(const ackpt_lstm* c, int64_t from, int64_t to, const float* in, float* out,
                 cudaStream_t s) {
  f32k::AdvParams<D> p;
  f32m::ScaledParams<D> sp;
  f32m::fill_scaled<D>(c, -1, sp);
  std::memcpy(p.ws, sp.ws, sizeof(p.ws));
  f32k::adv_kernel<D><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(
      in, out, c->B, static_cast<const float*>(c->d_xbs), from, to, p);
}

}  // namespace ackpt

#define ACKPT_INSTANTIATE_F32(D)                                                              \
  namespace ackpt {                                                                           \
  template void f32_forward<D>(const ackpt_lstm*, int64_t, const float*, float*, cudaStream_t); \
  template void f32_backward<D>(const ackpt_lstm*, int64_t, const float*, const float*, float*, \
                                cudaStream_t);                                                \
  template void f32_advance<D>(const ackpt_lstm*, int64_t, int64_t, const float*, float*,      \
                               cudaStream_t);                                                 \
  template void f32_forward_many<D>(const ackpt_lstm*, int64_t, int, const float*,            \
                                    float* const*, cudaStream_t);                             \
  template void f32_backward_many<D>(const ackpt_lstm*, int64_t, int, const float* const*,    \
                                     const float*, float*, cudaStream_t);                     \
  }
