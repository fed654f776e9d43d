// fp32 LSTM step kernels, TMA-pipelined persistent variant (K1 forward, K2
// adjoint) for sm_100a.  Same arithmetic contract as lstm.py:110-152.
//
// Data movement.  A tile is TILE = 2*THREADS consecutive batch elements.  Its
// input rows (h, c [, dh, dc]) are TILE*4-byte contiguous segments of the
// batch-fastest state layout, moved by one thread with cp.async.bulk
// (UBLKCP, the TMA bulk-copy path) into a STAGES-deep shared-memory ring whose
// slots complete on an mbarrier (expect_tx).  Each thread reads its float2
// pair with LDS.64 (conflict-free), computes, writes its results back into
// the same smem slots, and the tile leaves with bulk stores (smem -> global).
// Memory requests therefore do not depend on registers or occupancy: the ring
// keeps STAGES-1 tiles in flight per CTA while the warps compute.
//
// Arithmetic per element (d=8): the recurrent matvec is d*d*2 FFMA2 with
// weights broadcast from uniform registers; the exponent scales of the gate
// activations are pre-folded into the weights (-log2e for f, i, o; +2 log2e
// for g), so each accumulator is directly the ex2 argument; the four
// activations of a hidden unit share one MUFU reciprocal (1/y_f = y_i y_o y_g
// / (y_f y_i y_o y_g)), with a branch to separate reciprocals only when that
// product overflows (pre-activations beyond ~22).
#pragma once

#include <cuda_runtime.h>

#include <cstring>

#include "lstm_cell.h"

namespace ackpt {
namespace tma {

constexpr float kL2e = 1.4426950408889634f;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------------ packed fp32 math
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

// Activations of one hidden unit from pre-scaled accumulators:
// tf = -log2e a_f, ti = -log2e a_i, to = -log2e a_o, tg = 2 log2e a_g.
__device__ __forceinline__ void activate(float2 tf, float2 ti, float2 to, float2 tg, float2& f,
                                         float2& i, float2& o, float2& g) {
  const float2 one = bc(1.0f);
  const float2 yf = add2(ex2_2(tf), one), yi = add2(ex2_2(ti), one);
  const float2 yo = add2(ex2_2(to), one), yg = add2(ex2_2(tg), one);
  const float2 p12 = mul2(yf, yi), p34 = mul2(yo, yg);
  const float2 P = mul2(p12, p34);
  if (__builtin_expect(P.x <= 3.0e38f && P.y <= 3.0e38f, 1)) {
    const float2 r = rcp2(P);
    const float2 q34 = mul2(r, p34), q12 = mul2(r, p12);
    f = mul2(q34, yi);
    i = mul2(q34, yf);
    o = mul2(q12, yg);
    g = fma2(mul2(q12, yo), bc(-2.0f), one);
  } else {  // a product overflowed: separate reciprocals (1/inf = 0 is exact here)
    f = rcp2(yf);
    i = rcp2(yi);
    o = rcp2(yo);
    g = fma2(rcp2(yg), bc(-2.0f), one);
  }
}
// tanh(x) = 1 - 2 / (1 + e^{2x})
__device__ __forceinline__ float2 tanh2(float2 x) {
  const float2 y = add2(ex2_2(mul2(x, bc(2.0f * kL2e))), bc(1.0f));
  return fma2(rcp2(y), bc(-2.0f), bc(1.0f));
}

// Pre-scaled weights: ws[g][j][i] = scale_g W_g[j][i], xbs[g][j] = scale_g xb[g][j].
template <int D>
struct ScaledParams {
  float ws[4][D][D];
  float xbs[4][D];
};

constexpr float kScale[4] = {-kL2e, -kL2e, -kL2e, 2.0f * kL2e};

// ------------------------------------------------------------------- kernels
enum Mode { kFwd = 0, kBwd = 1 };

template <int D, int MODE, int THREADS>
struct Geometry {
  static constexpr int kTile = 2 * THREADS;                       // elements per tile
  static constexpr int kRows = MODE == kFwd ? 2 * D : 4 * D;      // input rows
  static constexpr int kRowBytes = kTile * 4;
  static constexpr int kStageFloats = kRows * kTile;
  static constexpr int kStageBytes = kStageFloats * 4;
};

// grid: persistent; tile t = blockIdx.x + k * gridDim.x.
// x: state (2D rows of B), a: adjoint in (2D rows, bwd only), y: output (2D rows).
// Pipeline per CTA: the prologue loads tiles 0..STAGES-2; iteration i waits
// for tile i, computes it in place, bulk-stores it, then refills the stage of
// tile i-1 (whose store has been reading smem for one iteration) with tile
// i+STAGES-1.
template <int D, int MODE, int THREADS, int STAGES>
__global__ void __launch_bounds__(THREADS, MODE == kFwd ? 2 : 1)
    step_kernel(const float* __restrict__ x, const float* __restrict__ a, float* __restrict__ y,
                int64_t B, int64_t ntiles, const __grid_constant__ ScaledParams<D> p) {
  using G = Geometry<D, MODE, THREADS>;
  constexpr int kHalf = G::kTile / 2;  // float2 slots per row
  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t full[STAGES];
  const int tid = threadIdx.x;
  const int64_t first = blockIdx.x, stride = gridDim.x;

  auto tile_bytes = [&](int64_t t) -> uint32_t {
    const int64_t left = B - t * G::kTile;
    return uint32_t(left < G::kTile ? left : G::kTile) * 4u;
  };
  auto issue = [&](int s, int64_t t) {  // thread 0 only
    const uint32_t bytes = tile_bytes(t);
    float* st = smem + s * G::kStageFloats;
    mbar_expect_tx(&full[s], bytes * G::kRows);
    const int64_t base = t * G::kTile;
#pragma unroll
    for (int r = 0; r < 2 * D; ++r) bulk_load(st + r * G::kTile, x + int64_t(r) * B + base, bytes, &full[s]);
    if constexpr (MODE == kBwd) {
#pragma unroll
      for (int r = 0; r < 2 * D; ++r)
        bulk_load(st + (2 * D + r) * G::kTile, a + int64_t(r) * B + base, bytes, &full[s]);
    }
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES - 1; ++s) {
      const int64_t t = first + s * stride;
      if (t < ntiles) issue(s, t);
    }
  }

  int64_t i = 0;
  for (int64_t t = first; t < ntiles; t += stride, ++i) {
    const int s = int(i % STAGES);
    float2* st2 = reinterpret_cast<float2*>(smem + s * G::kStageFloats);
    mbar_wait(&full[s], uint32_t((i / STAGES) & 1));

    float2 h[D];
#pragma unroll
    for (int j = 0; j < D; ++j) h[j] = st2[j * kHalf + tid];

    if constexpr (MODE == kFwd) {
      float2 hn[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        float2 af = bc(p.xbs[0][j]), ai = bc(p.xbs[1][j]), ao = bc(p.xbs[2][j]), ag = bc(p.xbs[3][j]);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          af = fma2(bc(p.ws[0][j][k]), h[k], af);
          ai = fma2(bc(p.ws[1][j][k]), h[k], ai);
          ao = fma2(bc(p.ws[2][j][k]), h[k], ao);
          ag = fma2(bc(p.ws[3][j][k]), h[k], ag);
        }
        float2 f, ig, o, g;
        activate(af, ai, ao, ag, f, ig, o, g);
        float2* cslot = st2 + (D + j) * kHalf + tid;
        const float2 cn = fma2(f, *cslot, mul2(ig, g));  // c' = f c + i g   (lstm.py:127)
        *cslot = cn;
        hn[j] = mul2(o, tanh2(cn));                      // h' = o tanh(c')  (lstm.py:128)
      }
#pragma unroll
      for (int j = 0; j < D; ++j) st2[j * kHalf + tid] = hn[j];
    } else {
      constexpr float kLn2 = 0.69314718055994531f;
      float2 acc[D];
#pragma unroll
      for (int m = 0; m < D; ++m) acc[m] = bc(0.0f);
#pragma unroll
      for (int j = 0; j < D; ++j) {
        float2 af = bc(p.xbs[0][j]), ai = bc(p.xbs[1][j]), ao = bc(p.xbs[2][j]), ag = bc(p.xbs[3][j]);
#pragma unroll
        for (int k = 0; k < D; ++k) {
          af = fma2(bc(p.ws[0][j][k]), h[k], af);
          ai = fma2(bc(p.ws[1][j][k]), h[k], ai);
          ao = fma2(bc(p.ws[2][j][k]), h[k], ao);
          ag = fma2(bc(p.ws[3][j][k]), h[k], ag);
        }
        float2 f, ig, o, g;
        activate(af, ai, ao, ag, f, ig, o, g);
        float2* cslot = st2 + (D + j) * kHalf + tid;
        const float2 c = *cslot;
        const float2 dhn = st2[(2 * D + j) * kHalf + tid];
        const float2 dcn = st2[(3 * D + j) * kHalf + tid];
        const float2 cn = fma2(f, c, mul2(ig, g));
        const float2 t = tanh2(cn);
        const float2 dco = fma2(mul2(dhn, o), fma2(neg(t), t, bc(1.0f)), dcn);  // lstm.py:143
        // da_g / scale_g, so that sum_g (scale_g W_g)^T (da_g / scale_g) = W^T da
        const float2 dcs = mul2(dco, bc(-kLn2));
        const float2 daf = mul2(mul2(dcs, c), fma2(neg(f), f, f));                      // :144
        const float2 dai = mul2(mul2(dcs, g), fma2(neg(ig), ig, ig));                   // :145
        const float2 dao = mul2(mul2(dhn, mul2(t, bc(-kLn2))), fma2(neg(o), o, o));    // :142,146
        const float2 dag = mul2(mul2(dco, mul2(ig, bc(0.5f * kLn2))), fma2(neg(g), g, bc(1.0f)));  // :147
        *cslot = mul2(dco, f);                                                          // :151
#pragma unroll
        for (int m = 0; m < D; ++m) {                                                   // :149-150
          acc[m] = fma2(bc(p.ws[0][j][m]), daf, acc[m]);
          acc[m] = fma2(bc(p.ws[1][j][m]), dai, acc[m]);
          acc[m] = fma2(bc(p.ws[2][j][m]), dao, acc[m]);
          acc[m] = fma2(bc(p.ws[3][j][m]), dag, acc[m]);
        }
      }
#pragma unroll
      for (int m = 0; m < D; ++m) st2[m * kHalf + tid] = acc[m];
    }

    fence_async_smem();  // generic smem writes -> visible to the bulk-copy (async) proxy
    __syncthreads();
    if (tid == 0) {
      const uint32_t bytes = tile_bytes(t);
      const float* st = smem + s * G::kStageFloats;
      const int64_t base = t * G::kTile;
#pragma unroll
      for (int r = 0; r < 2 * D; ++r) bulk_store(y + int64_t(r) * B + base, st + r * G::kTile, bytes);
      bulk_commit();
      // refill the stage of tile i-1 with tile i+STAGES-1 once its store has read smem
      const int64_t tn = t + int64_t(STAGES - 1) * stride;
      if (tn < ntiles) {
        bulk_wait_read<1>();
        issue(int((i + STAGES - 1) % STAGES), tn);
      }
    }
  }
  if (tid == 0) bulk_wait_all();
}

template <int D>
ScaledParams<D> scaled_params(const ackpt_lstm* c, int64_t step) {
  ScaledParams<D> p;
  for (int g = 0; g < 4; ++g) {
    for (int j = 0; j < D; ++j) {
      for (int k = 0; k < D; ++k) p.ws[g][j][k] = float(c->wh64[(size_t(g) * D + j) * D + k] * double(kScale[g]));
      p.xbs[g][j] = float(c->xb64[(size_t(step) * 4 + g) * D + j] * double(kScale[g]));
    }
  }
  return p;
}

}  // namespace tma

// Launch: persistent grid sized to the resident-CTA capacity of the device.
template <int D, int MODE, int THREADS, int STAGES>
void tma_launch(const ackpt_lstm* c, int64_t step, const float* x, const float* a, float* y,
                cudaStream_t s) {
  using G = tma::Geometry<D, MODE, THREADS>;
  auto kern = tma::step_kernel<D, MODE, THREADS, STAGES>;
  constexpr int kSmem = STAGES * G::kStageBytes;
  static int grid_cap = [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, kSmem);
    return sms * (per_sm > 0 ? per_sm : 1);
  }();
  const int64_t ntiles = (c->B + G::kTile - 1) / G::kTile;
  const int grid = int(ntiles < grid_cap ? ntiles : grid_cap);
  kern<<<grid, THREADS, kSmem, s>>>(x, a, y, c->B, ntiles, tma::scaled_params<D>(c, step));
}

}  // namespace ackpt

#define ACKPT_INSTANTIATE_TMA(D, MODE, THREADS, STAGES)                                         \
  namespace ackpt {                                                                            \
  template void tma_launch<D, MODE, THREADS, STAGES>(const ackpt_lstm*, int64_t, const float*, \
                                                     const float*, float*, cudaStream_t);      \
  }
