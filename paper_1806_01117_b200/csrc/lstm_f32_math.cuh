// Packed-fp32 (f32x2) math shared by the fp32 LSTM step kernels.
//
// The gate activations are computed from PRE-SCALED accumulators: the
// weights and input projections are multiplied on the host by
// -log2(e) (gates f, i, o) or +2 log2(e) (gate g), so an accumulator is
// directly the argument of ex2:
//   sigmoid(a) = 1 / (1 + 2^(-log2e a)),   tanh(a) = 1 - 2 / (1 + 2^(2 log2e a)).
// The four activations of a hidden unit share ONE reciprocal on the MUFU
// pipe: 1/y_f = (y_i y_o y_g) / (y_f y_i y_o y_g).  If the product is large
// (P > kShareMax: pre-activations summing past ~60) a branch computes separate
// reciprocals, which is exact there because rcp(inf) = 0.  The bound keeps
// 1/P a normal float: above 2^126 rcp.approx.ftz flushes 1/P to 0 (so f = i =
// o = 0 where e.g. f = 1/y_f = 1), and the Newton seed 0x7EF311C3 - bits(P)
// leaves the normal range -- both seen with pre-activations of +-100
// (tests/test_gpu_saturation.py).
constexpr float kShareMax = 1.0e37f;
#pragma once

#include <cuda_runtime.h>

#include <cstring>

#include "lstm_cell.h"

namespace ackpt {
namespace f32m {

constexpr float kL2e = 1.4426950408889634f;
constexpr float kLn2 = 0.69314718055994531f;
// per-gate exponent scales (f, i, o, c) and their inverses
constexpr float kScale[4] = {-kL2e, -kL2e, -kL2e, 2.0f * kL2e};

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
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  P2 x{a}, y{b}, r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.u) : "l"(x.u), "l"(y.u));
  return r.f;
}
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 neg(float2 a) { return make_float2(-a.x, -a.y); }
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
__device__ __forceinline__ float2 ex2_2(float2 t) { return make_float2(ex2(t.x), ex2(t.y)); }
__device__ __forceinline__ float2 rcp2(float2 y) { return make_float2(rcp(y.x), rcp(y.y)); }

__device__ __forceinline__ void activate(float2 tf, float2 ti, float2 to, float2 tg, float2& f,
                                         float2& i, float2& o, float2& g) {
  const float2 one = bc(1.0f);
  const float2 yf = add2(ex2_2(tf), one), yi = add2(ex2_2(ti), one);
  const float2 yo = add2(ex2_2(to), one), yg = add2(ex2_2(tg), one);
  const float2 p12 = mul2(yf, yi), p34 = mul2(yo, yg);
  const float2 P = mul2(p12, p34);
  if (__builtin_expect(P.x <= kShareMax && P.y <= kShareMax, 1)) {
    const float2 r = rcp2(P);
    const float2 q34 = mul2(r, p34), q12 = mul2(r, p12);
    f = mul2(q34, yi);
    i = mul2(q34, yf);
    o = mul2(q12, yg);
    g = fma2(mul2(q12, yo), bc(-2.0f), one);
  } else {
    f = rcp2(yf);
    i = rcp2(yi);
    o = rcp2(yo);
    g = fma2(rcp2(yg), bc(-2.0f), one);
  }
}

__device__ __forceinline__ float2 tanh2(float2 x) {
  const float2 y = add2(ex2_2(mul2(x, bc(2.0f * kL2e))), bc(1.0f));
  return fma2(rcp2(y), bc(-2.0f), bc(1.0f));
}

// ---- Newton-Raphson variants (tensor-core family) ------------------------
// With the matvec on the tensor cores the FMA pipe idles while MUFU (16/clk/SM)
// saturates, so reciprocals move to the FMA pipe: a bit-trick seed (<= 12 %
// error) and Newton steps for any normal y >= 1 (the only arguments here).
// Newton converges from below (r (1 - e) -> r (1 - e^2)), so the iterate
// carries a one-signed error e^2: after three steps up to 4e-8 (0.7 ulp),
// the same sign in every reciprocal of every step.  That bias reached the
// forget gate and, compounded over a 10^4-step long-memory chain, put the
// adjoint at 6e-4 rel-L2 from float64 against 1e-4 for MUFU reciprocals
// (tools/long_chain_mix.py).  A fourth step in the form r + r (1 - y r)
// leaves ~1e-15 of bias plus one rounding.
__device__ __forceinline__ float2 rcp2_nr(float2 y) {
  float2 r = make_float2(__int_as_float(0x7EF311C3 - __float_as_int(y.x)),
                         __int_as_float(0x7EF311C3 - __float_as_int(y.y)));
#pragma unroll
  for (int it = 0; it < 3; ++it) r = mul2(r, fma2(neg(y), r, bc(2.0f)));
  return fma2(r, fma2(neg(y), r, bc(1.0f)), r);
}

__device__ __forceinline__ void activate_nr(float2 tf, float2 ti, float2 to, float2 tg, float2& f, float2& i,
                                            float2& o, float2& g) {
  const float2 one = bc(1.0f);
  const float2 yf = add2(ex2_2(tf), one), yi = add2(ex2_2(ti), one);
  const float2 yo = add2(ex2_2(to), one), yg = add2(ex2_2(tg), one);
  const float2 p12 = mul2(yf, yi), p34 = mul2(yo, yg);
  const float2 P = mul2(p12, p34);
  if (__builtin_expect(P.x <= kShareMax && P.y <= kShareMax, 1)) {
    const float2 r = rcp2_nr(P);
    const float2 q34 = mul2(r, p34), q12 = mul2(r, p12);
    f = mul2(q34, yi);
    i = mul2(q34, yf);
    o = mul2(q12, yg);
    g = fma2(mul2(q12, yo), bc(-2.0f), one);
  } else {
    f = rcp2(yf);
    i = rcp2(yi);
    o = rcp2(yo);
    g = fma2(rcp2(yg), bc(-2.0f), one);
  }
}

// tanh of two float2s sharing one Newton reciprocal: 1/y_a = y_b / (y_a y_b).
// The exponent argument is clamped at 31, so the product stays below 2^63
// and the Newton seed in the normal range; tanh = 1 - 2/(1 + 2^31) already
// rounds to 1.0f, so the clamp changes no result.
__device__ __forceinline__ void tanh2x2_nr(float2 xa, float2 xb, float2& ta, float2& tb) {
  const float2 sa = mul2(xa, bc(2.0f * kL2e)), sb = mul2(xb, bc(2.0f * kL2e));
  const float2 ya = add2(make_float2(ex2(fminf(sa.x, 31.0f)), ex2(fminf(sa.y, 31.0f))), bc(1.0f));
  const float2 yb = add2(make_float2(ex2(fminf(sb.x, 31.0f)), ex2(fminf(sb.y, 31.0f))), bc(1.0f));
  const float2 r = rcp2_nr(mul2(ya, yb));
  ta = fma2(mul2(r, yb), bc(-2.0f), bc(1.0f));
  tb = fma2(mul2(r, ya), bc(-2.0f), bc(1.0f));
}

// Forward of two hidden units (or two unit pairs) at once (lstm.py:123-129):
// c' = f c + i g, h' = o tanh(c'), the two tanh(c') sharing one reciprocal
// (tanh2x2_nr).
// The forward needs only c' and o, not f and i: with the shared reciprocal
// r = 1/P, c' = f c + i g = r y_o y_g (y_i c + y_f g)  (lstm.py:127).
__device__ __forceinline__ void fwd_cell_nr(float2 tf, float2 ti, float2 to, float2 tg, float2& c, float2& o) {
  const float2 one = bc(1.0f);
  const float2 yf = add2(ex2_2(tf), one), yi = add2(ex2_2(ti), one);
  const float2 yo = add2(ex2_2(to), one), yg = add2(ex2_2(tg), one);
  const float2 p12 = mul2(yf, yi), p34 = mul2(yo, yg);
  const float2 P = mul2(p12, p34);
  if (__builtin_expect(P.x <= kShareMax && P.y <= kShareMax, 1)) {
    const float2 r = rcp2_nr(P);
    const float2 q34 = mul2(r, p34), q12 = mul2(r, p12);
    const float2 g = fma2(mul2(q12, yo), bc(-2.0f), one);
    c = mul2(q34, fma2(yi, c, mul2(yf, g)));
    o = mul2(q12, yg);
  } else {
    const float2 g = fma2(rcp2(yg), bc(-2.0f), one);
    c = fma2(rcp2(yf), c, mul2(rcp2(yi), g));
    o = rcp2(yo);
  }
}

__device__ __forceinline__ void fwd_units2_nr(const float2 (&pa)[4], const float2 (&pb)[4], float2& ca, float2& cb,
                                              float2& ha, float2& hb) {
  float2 oa, ob;
  fwd_cell_nr(pa[0], pa[1], pa[2], pa[3], ca, oa);
  fwd_cell_nr(pb[0], pb[1], pb[2], pb[3], cb, ob);
  float2 ta, tb;
  tanh2x2_nr(ca, cb, ta, tb);
  ha = mul2(oa, ta);
  hb = mul2(ob, tb);
}


// Weights pre-scaled per gate (see file comment).
template <int D>
struct ScaledParams {
  float ws[4][D][D];
  float xbs[4][D];
};

template <int D>
inline void fill_scaled(const ackpt_lstm* c, int64_t step, ScaledParams<D>& p) {
  for (int g = 0; g < 4; ++g)
    for (int j = 0; j < D; ++j) {
      for (int k = 0; k < D; ++k)
        p.ws[g][j][k] = float(c->wh64[(size_t(g) * D + j) * D + k] * double(kScale[g]));
      p.xbs[g][j] = step >= 0 ? float(c->xb64[(size_t(step) * 4 + g) * D + j] * double(kScale[g])) : 0.0f;
    }
}

// Pre-activations of unit j (scaled) for one pair, from h and scaled xb.
template <int D>
__device__ __forceinline__ void preacts(const float (&ws)[4][D][D], const float (&xbs)[4][D],
                                        const float2 (&h)[D], int j, float2& af, float2& ai,
                                        float2& ao, float2& ag) {
  af = bc(xbs[0][j]);
  ai = bc(xbs[1][j]);
  ao = bc(xbs[2][j]);
  ag = bc(xbs[3][j]);
#pragma unroll
  for (int k = 0; k < D; ++k) {
    af = fma2(bc(ws[0][j][k]), h[k], af);
    ai = fma2(bc(ws[1][j][k]), h[k], ai);
    ao = fma2(bc(ws[2][j][k]), h[k], ao);
    ag = fma2(bc(ws[3][j][k]), h[k], ag);
  }
}

// Forward of unit j: c <- f c + i g, returns h' = o tanh(c')   (lstm.py:127-128)
__device__ __forceinline__ float2 fwd_unit(float2 af, float2 ai, float2 ao, float2 ag, float2& c) {
  float2 f, ig, o, g;
  activate(af, ai, ao, ag, f, ig, o, g);
  c = fma2(f, c, mul2(ig, g));
  return mul2(o, tanh2(c));
}

// Adjoint of unit j (lstm.py:141-151).  Returns the four scaled gate
// adjoints da_g / scale_g (so that sum_g (scale_g W_g)^T (da_g / scale_g) =
// W^T da) and dc_k in dco_f.
__device__ __forceinline__ void bwd_unit(float2 af, float2 ai, float2 ao, float2 ag, float2 c,
                                         float2 dhn, float2 dcn, float2& daf, float2& dai,
                                         float2& dao, float2& dag, float2& dck) {
  float2 f, ig, o, g;
  activate(af, ai, ao, ag, f, ig, o, g);
  const float2 cn = fma2(f, c, mul2(ig, g));
  const float2 t = tanh2(cn);
  // shared products as in bwd_unit_u, with the scales folded in
  const float2 A = mul2(dhn, o);
  const float2 dco = fma2(A, fma2(neg(t), t, bc(1.0f)), dcn);  // :143
  const float2 dcs = mul2(dco, bc(-kLn2));
  const float2 X = mul2(dcs, ig), Y = mul2(X, g);
  const float2 Z = mul2(mul2(dcs, c), f);
  const float2 Bs = mul2(mul2(A, t), bc(-kLn2));
  daf = fma2(neg(Z), f, Z);                          // -ln2 dc c f (1 - f)      :144
  dai = fma2(neg(Y), ig, Y);                         // -ln2 dc g i (1 - i)      :145
  dao = fma2(neg(Bs), o, Bs);                        // -ln2 dh' t o (1 - o)     :142, :146
  dag = mul2(fma2(neg(Y), g, X), bc(-0.5f));         // ln2/2 dc i (1 - g^2)     :147
  dck = mul2(dco, f);                                //                          :151
}

// As bwd_unit, but the gate adjoints are the true ones (dL/da, not divided
// by the exponent scales): the transposed matvec then uses the unscaled
// weights and three constant multiplies per unit disappear.
__device__ __forceinline__ void bwd_unit_u(float2 af, float2 ai, float2 ao, float2 ag, float2 c, float2 dhn,
                                           float2 dcn, float2& daf, float2& dai, float2& dao, float2& dag,
                                           float2& dck) {
  float2 f, ig, o, g;
  activate(af, ai, ao, ag, f, ig, o, g);
  const float2 cn = fma2(f, c, mul2(ig, g));
  const float2 t = tanh2(cn);
  // Shared products (3 FMA-pipe instructions per unit fewer than the
  // formulas written out): A = dh' o, Bt = dh' o t, X = dc i, Y = dc i g.
  const float2 A = mul2(dhn, o);
  const float2 dco = fma2(A, fma2(neg(t), t, bc(1.0f)), dcn);  // lstm.py:143
  const float2 Bt = mul2(A, t);
  const float2 X = mul2(dco, ig), Y = mul2(X, g);
  const float2 Z = mul2(mul2(dco, c), f);
  daf = fma2(neg(Z), f, Z);   // dc c f (1 - f)          :144
  dai = fma2(neg(Y), ig, Y);  // dc g i (1 - i)          :145
  dao = fma2(neg(Bt), o, Bt); // dh' t o (1 - o)         :142, :146
  dag = fma2(neg(Y), g, X);   // dc i (1 - g^2)          :147
  dck = mul2(dco, f);         //                         :151
}

}  // namespace f32m
}  // namespace ackpt
