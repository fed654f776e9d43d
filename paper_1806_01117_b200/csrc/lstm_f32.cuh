// fp32 LSTM step kernels for sm_100a, hidden size D in {4, 8} (K1 forward,
// K2 adjoint, K1f fused advance).  Included by lstm_f32_d<D>.cu, which
// instantiate one D each so the translation units compile in parallel.
//
// Reference operator: lstm.py:110-152 (gates, forward step, exact adjoint).
//
// Mapping to the hardware:
//  * Each thread owns 2 consecutive batch elements (one float2 pair; the
//    kernels are templated on P pairs, P=1 is used: P=2 spills under the
//    2-blocks/SM register cap).  Feature row j of h (or c, dh, dc) for them is
//    one 8-byte load; a warp covers a contiguous 256 B span of that row ->
//    fully coalesced 32 B sectors, no smem staging needed.  Callers require
//    even B and 8-byte aligned pointers (odd B takes the generic kernel).
//  * Elements are processed as float2 pairs with the Blackwell packed-fp32
//    pipe: fma.rn.f32x2 (FFMA2) takes the weight as a uniform-register scalar
//    broadcast (ptxas loads W_h / xb from the __grid_constant__ parameter
//    bank with LDCU.128), so the 4d x d recurrent matvec costs d*d*2 FFMA2 per
//    element instead of 4 d^2 FFMA.
//  * The MUFU pipe (16/clk/SM) is the scarce unit: the four gate activations
//    of one hidden unit share ONE reciprocal: with y_g = 1 + e^{t_g},
//    1/y_f = (y_i y_o y_c) / (y_f y_i y_o y_c), etc.  Exponent arguments are
//    clamped at 30 (|sigmoid error| < 1e-9 there) so the product stays finite.
//    Per element and unit: 5 EX2 + 2 RCP instead of 5 EX2 + 5 RCP.
#pragma once

#include <cuda_runtime.h>

#include <cstring>

#include "lstm_cell.h"

namespace ackpt {
namespace f32k {

union P2 {
  float2 f;
  unsigned long long u;
};

__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  P2 x{a}, y{b}, z{c}, r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.u) : "l"(x.u), "l"(y.u), "l"(z.u));
  return r.f;
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
  P2 x{a}, y{b}, r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(x.u), "l"(y.u));
  return r.f;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  P2 x{a}, y{b}, r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(x.u), "l"(y.u));
  return r.f;
}
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 ex2c(float2 t) {  // e^(ln2 t), t clamped at 30
  return make_float2(ex2(fminf(t.x, 30.0f)), ex2(fminf(t.y, 30.0f)));
}
__device__ __forceinline__ float2 rcp2(float2 y) { return make_float2(rcp(y.x), rcp(y.y)); }

constexpr float kL2e = 1.4426950408889634f;

// f, i, o = sigmoid(af, ai, ao); g = tanh(ag)   (lstm.py:116-119)
__device__ __forceinline__ void activate(float2 af, float2 ai, float2 ao, float2 ag, float2& f,
                                         float2& i, float2& o, float2& g) {
  const float2 yf = add2(ex2c(mul2(af, bc(-kL2e))), bc(1.0f));
  const float2 yi = add2(ex2c(mul2(ai, bc(-kL2e))), bc(1.0f));
  const float2 yo = add2(ex2c(mul2(ao, bc(-kL2e))), bc(1.0f));
  const float2 yg = add2(ex2c(mul2(ag, bc(2.0f * kL2e))), bc(1.0f));
  const float2 p12 = mul2(yf, yi), p34 = mul2(yo, yg);
  const float2 r = rcp2(mul2(p12, p34));
  const float2 q34 = mul2(r, p34), q12 = mul2(r, p12);
  f = mul2(q34, yi);
  i = mul2(q34, yf);
  o = mul2(q12, yg);
  g = fma2(mul2(q12, yo), bc(-2.0f), bc(1.0f));  // tanh = 1 - 2/(1 + e^2a)
}

// tanh(x) = 1 - 2 / (1 + e^2x); saturates correctly without a clamp.
__device__ __forceinline__ float2 tanh2(float2 x) {
  const float2 t = mul2(x, bc(2.0f * kL2e));
  const float2 y = add2(make_float2(ex2(t.x), ex2(t.y)), bc(1.0f));
  return fma2(rcp2(y), bc(-2.0f), bc(1.0f));
}

template <int P>
struct Row {  // 2P consecutive batch elements of one feature row
  float2 p[P];
};

template <int P>
__device__ __forceinline__ Row<P> ld_row(const float* ptr) {
  Row<P> r;
  if constexpr (P == 2) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(ptr));
    r.p[0] = make_float2(v.x, v.y);
    r.p[1] = make_float2(v.z, v.w);
  } else {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];"
                 : "=f"(v.x), "=f"(v.y)
                 : "l"(ptr));
    r.p[0] = v;
  }
  return r;
}

template <int P>
__device__ __forceinline__ void st_row(float* ptr, const Row<P>& r) {
  if constexpr (P == 2) {
    asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(ptr), "f"(r.p[0].x),
                 "f"(r.p[0].y), "f"(r.p[1].x), "f"(r.p[1].y)
                 : "memory");
  } else {
    asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(ptr), "f"(r.p[0].x), "f"(r.p[0].y)
                 : "memory");
  }
}

// One forward step for one pair; h/c in, hn/c out.
template <int D>
__device__ __forceinline__ void fwd_pair(const float (&wh)[4][D][D], const float (&xb)[4][D],
                                         const float2 (&h)[D], float2 (&c)[D], float2 (&hn)[D]) {
#pragma unroll
  for (int j = 0; j < D; ++j) {
    float2 af = bc(xb[0][j]), ai = bc(xb[1][j]), ao = bc(xb[2][j]), ag = bc(xb[3][j]);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      af = fma2(bc(wh[0][j][i]), h[i], af);
      ai = fma2(bc(wh[1][j][i]), h[i], ai);
      ao = fma2(bc(wh[2][j][i]), h[i], ao);
      ag = fma2(bc(wh[3][j][i]), h[i], ag);
    }
    float2 f, ig, o, g;
    activate(af, ai, ao, ag, f, ig, o, g);
    const float2 cn = fma2(f, c[j], mul2(ig, g));  // c' = f c + i g   (lstm.py:127)
    c[j] = cn;
    hn[j] = mul2(o, tanh2(cn));                   // h' = o tanh(c')  (lstm.py:128)
  }
}

template <int D, int P>
__global__ void __launch_bounds__(256, 2)
    fwd_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t B,
               const __grid_constant__ StepParams<float, D> p) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * (2 * P);
  if (b0 >= B) return;
  Row<P> h[D], c[D];
#pragma unroll
  for (int j = 0; j < D; ++j) h[j] = ld_row<P>(in + int64_t(j) * B + b0);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = ld_row<P>(in + int64_t(D + j) * B + b0);
  Row<P> hn[D];
#pragma unroll
  for (int q = 0; q < P; ++q) {
    float2 hq[D], cq[D], hnq[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      hq[j] = h[j].p[q];
      cq[j] = c[j].p[q];
    }
    fwd_pair<D>(p.wh, p.xb, hq, cq, hnq);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      c[j].p[q] = cq[j];
      hn[j].p[q] = hnq[j];
    }
  }
#pragma unroll
  for (int j = 0; j < D; ++j) st_row<P>(out + int64_t(j) * B + b0, hn[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) st_row<P>(out + int64_t(D + j) * B + b0, c[j]);
}

template <int D, int P>
__global__ void __launch_bounds__(256, 2)
    bwd_kernel(const float* __restrict__ st, const float* __restrict__ adj_in,
               float* __restrict__ adj_out, int64_t B,
               const __grid_constant__ StepParams<float, D> p) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * (2 * P);
  if (b0 >= B) return;
  Row<P> h[D], c[D], dh[D], dc[D];
#pragma unroll
  for (int j = 0; j < D; ++j) h[j] = ld_row<P>(st + int64_t(j) * B + b0);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = ld_row<P>(st + int64_t(D + j) * B + b0);
#pragma unroll
  for (int j = 0; j < D; ++j) dh[j] = ld_row<P>(adj_in + int64_t(j) * B + b0);
#pragma unroll
  for (int j = 0; j < D; ++j) dc[j] = ld_row<P>(adj_in + int64_t(D + j) * B + b0);
  Row<P> dho[D];
#pragma unroll
  for (int q = 0; q < P; ++q) {
    float2 acc[D];
#pragma unroll
    for (int m = 0; m < D; ++m) acc[m] = bc(0.0f);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      float2 af = bc(p.xb[0][j]), ai = bc(p.xb[1][j]), ao = bc(p.xb[2][j]), ag = bc(p.xb[3][j]);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        const float2 hi = h[i].p[q];
        af = fma2(bc(p.wh[0][j][i]), hi, af);
        ai = fma2(bc(p.wh[1][j][i]), hi, ai);
        ao = fma2(bc(p.wh[2][j][i]), hi, ao);
        ag = fma2(bc(p.wh[3][j][i]), hi, ag);
      }
      float2 f, ig, o, g;
      activate(af, ai, ao, ag, f, ig, o, g);
      const float2 cj = c[j].p[q];
      const float2 cn = fma2(f, cj, mul2(ig, g));
      const float2 t = tanh2(cn);
      const float2 dhn = dh[j].p[q];
      const float2 omt2 = fma2(t, make_float2(-t.x, -t.y), bc(1.0f));  // 1 - t^2
      const float2 dco = fma2(mul2(dhn, o), omt2, dc[j].p[q]);         // lstm.py:143
      const float2 dob = mul2(dhn, t);                                 // lstm.py:142
      const float2 daf = mul2(mul2(dco, cj), fma2(f, make_float2(-f.x, -f.y), f));     // :144
      const float2 dai = mul2(mul2(dco, g), fma2(ig, make_float2(-ig.x, -ig.y), ig));  // :145
      const float2 dao = mul2(dob, fma2(o, make_float2(-o.x, -o.y), o));               // :146
      const float2 dag = mul2(mul2(dco, ig), fma2(g, make_float2(-g.x, -g.y), bc(1.0f)));  // :147
      dc[j].p[q] = mul2(dco, f);                                                        // :151
      // dh += W_f[j,:d]^T da_f + W_i^T da_i + W_o^T da_o + W_c^T da_g   (lstm.py:149-150)
#pragma unroll
      for (int m = 0; m < D; ++m) {
        acc[m] = fma2(bc(p.wh[0][j][m]), daf, acc[m]);
        acc[m] = fma2(bc(p.wh[1][j][m]), dai, acc[m]);
        acc[m] = fma2(bc(p.wh[2][j][m]), dao, acc[m]);
        acc[m] = fma2(bc(p.wh[3][j][m]), dag, acc[m]);
      }
    }
#pragma unroll
    for (int m = 0; m < D; ++m) dho[m].p[q] = acc[m];
  }
#pragma unroll
  for (int j = 0; j < D; ++j) st_row<P>(adj_out + int64_t(j) * B + b0, dho[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) st_row<P>(adj_out + int64_t(D + j) * B + b0, dc[j]);
}

// Fused forward over [from, to): state in registers, xb of each step read with
// uniform (broadcast) loads.  One launch moves 2S bytes for any step count.
template <int D>
struct AdvParams {
  float wh[4][D][D];
};

template <int D, int P>
__global__ void __launch_bounds__(256, 2)
    adv_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t B,
               const float* __restrict__ xb_all, int64_t from, int64_t to,
               const __grid_constant__ AdvParams<D> p) {
  const int64_t b0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * (2 * P);
  if (b0 >= B) return;
  Row<P> h[D], c[D];
#pragma unroll
  for (int j = 0; j < D; ++j) h[j] = ld_row<P>(in + int64_t(j) * B + b0);
#pragma unroll
  for (int j = 0; j < D; ++j) c[j] = ld_row<P>(in + int64_t(D + j) * B + b0);
  for (int64_t k = from; k < to; ++k) {
    float xb[4][D];
    const float4* src = reinterpret_cast<const float4*>(xb_all + k * 4 * D);
#pragma unroll
    for (int v = 0; v < D; ++v) {
      const float4 x = __ldg(src + v);
      xb[(4 * v) / D][(4 * v) % D] = x.x;
      xb[(4 * v + 1) / D][(4 * v + 1) % D] = x.y;
      xb[(4 * v + 2) / D][(4 * v + 2) % D] = x.z;
      xb[(4 * v + 3) / D][(4 * v + 3) % D] = x.w;
    }
#pragma unroll
    for (int q = 0; q < P; ++q) {
      float2 hq[D], cq[D], hnq[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        hq[j] = h[j].p[q];
        cq[j] = c[j].p[q];
      }
      fwd_pair<D>(p.wh, xb, hq, cq, hnq);
#pragma unroll
      for (int j = 0; j < D; ++j) {
        c[j].p[q] = cq[j];
        h[j].p[q] = hnq[j];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < D; ++j) st_row<P>(out + int64_t(j) * B + b0, h[j]);
#pragma unroll
  for (int j = 0; j < D; ++j) st_row<P>(out + int64_t(D + j) * B + b0, c[j]);
}

template <int D>
StepParams<float, D> step_params(const ackpt_lstm* cell, int64_t step) {
  StepParams<float, D> p;
  std::memcpy(p.wh, cell->wh_t.data(), sizeof(p.wh));
  std::memcpy(p.xb, cell->xb_t.data() + size_t(step) * sizeof(p.xb), sizeof(p.xb));
  return p;
}

}  // namespace f32k

template <int D>
void f32_forward(const ackpt_lstm* c, int64_t step, const float* in, float* out, cudaStream_t s) {
  const auto p = f32k::step_params<D>(c, step);
  f32k::fwd_kernel<D, 1><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(in, out, c->B, p);
}

template <int D>
void f32_backward(const ackpt_lstm* c, int64_t step, const float* st, const float* ai, float* ao,
                  cudaStream_t s) {
  const auto p = f32k::step_params<D>(c, step);
  f32k::bwd_kernel<D, 1><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(st, ai, ao, c->B, p);
}

template <int D>
void f32_advance(const ackpt_lstm* c, int64_t from, int64_t to, const float* in, float* out,
                 cudaStream_t s) {
  f32k::AdvParams<D> p;
  std::memcpy(p.wh, c->wh_t.data(), sizeof(p.wh));
  const float* xb = static_cast<const float*>(c->d_xb);
  f32k::adv_kernel<D, 1><<<blocks_for(c->B / 2, 256), 256, 0, s>>>(in, out, c->B, xb, from, to, p);
}

}  // namespace ackpt

#define ACKPT_INSTANTIATE_F32(D)                                                              \
  namespace ackpt {                                                                           \
  template void f32_forward<D>(const ackpt_lstm*, int64_t, const float*, float*, cudaStream_t); \
  template void f32_backward<D>(const ackpt_lstm*, int64_t, const float*, const float*, float*, \
                                cudaStream_t);                                                \
  template void f32_advance<D>(const ackpt_lstm*, int64_t, int64_t, const float*, float*,      \
                               cudaStream_t);                                                 \
  }
