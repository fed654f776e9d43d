// Ping-pong tensor-core forward for d = 8 (fused Advance / TapeForward):
// the same 3xTF32 gate products as fwd_tc (lstm_f32_tc.cuh), restructured so
// the tensor core works on one tile while the threads finish the other.
//
// CTA = 128 threads, 256 sequences: tile 0 = b0 + r, tile 1 = b0 + 128 + r
// (thread r owns row r of both; TMEM lanes = rows, tile t at columns 32t).
// Per step i the CTA runs
//     wait MMA0(i); epilogue tile 0; stage tile 0 (i+1); barrier; issue MMA0(i+1)
//     wait MMA1(i); epilogue tile 1; stage tile 1 (i+1); barrier; issue MMA1(i+1)
// so each tile's MMA round trip hides behind the other tile's activations.
// Arithmetic is packed over unit pairs: gate rows are ordered
// n = 8p + 2 gate + e (unit 2p + e), so one tcgen05.ld.x8 at column 8p yields
// (f, i, o, g) of units 2p, 2p+1 as float2s.  The step bias is a two-slot
// ring (the other tile's MMA may still read the previous slot).
#pragma once

#include <cuda_runtime.h>

#include "lstm_f32_math.cuh"

namespace ackpt {
namespace tcp {

using namespace f32m;

constexpr int kThreads = 128;
constexpr int kTile = 256;
constexpr int kD = 8;
constexpr int kN = 32;
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(kN >> 3) << 17) | (uint32_t(128 >> 4) << 24);

struct Weights {
  float ws[4][kD][kD];
};
struct OutPtrs {
  float* p[ACKPT_MAX_FUSED];
};

// K = 8 operands: 8-row groups of two 16-byte core matrices (LBO 128 B, SBO 256 B)
__device__ __forceinline__ int kofs(int r, int k) { return (r >> 3) * 64 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3); }
__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ float hi_part(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

struct Smem {
  float a[2][2][128 * kD];  // [tile][hi, lo]
  float one[128 * kD];      // rows [1, 0, ..., 0]
  float w[2][kN * kD];      // [hi, lo]
  float bias[2][2][kN * kD];  // [slot][hi, lo], column 0
  uint64_t mbar[2];
  uint32_t tmem;
};

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(bar)), "r"(phase)
        : "memory");
  } while (!done);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Row r of tile t: h (4 unit pairs) split hi / lo into the A operand.
__device__ __forceinline__ void stage_a(Smem& sm, int t, const float2 (&h)[4]) {
  const int r = threadIdx.x;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const float4 x = make_float4(h[2 * c].x, h[2 * c].y, h[2 * c + 1].x, h[2 * c + 1].y);
    const float4 hx = make_float4(hi_part(x.x), hi_part(x.y), hi_part(x.z), hi_part(x.w));
    const float2 l01 = sub2(make_float2(x.x, x.y), make_float2(hx.x, hx.y));
    const float2 l23 = sub2(make_float2(x.z, x.w), make_float2(hx.z, hx.w));
    *reinterpret_cast<float4*>(&sm.a[t][0][kofs(r, 4 * c)]) = hx;
    *reinterpret_cast<float4*>(&sm.a[t][1][kofs(r, 4 * c)]) = make_float4(l01.x, l01.y, l23.x, l23.y);
  }
}
// Bias column of step k into slot s (threads < 32: row n = 8p + 2 gate + e).
__device__ __forceinline__ void stage_bias(Smem& sm, int s, float x) {
  const int n = threadIdx.x;
  if (n < kN) {
    sm.bias[s][0][kofs(n, 0)] = hi_part(x);
    sm.bias[s][1][kofs(n, 0)] = x - hi_part(x);
  }
}
__device__ __forceinline__ float load_bias(const float* __restrict__ xbs_all, int64_t k) {
  const int n = threadIdx.x;
  if (n >= kN) return 0.f;
  const int gi = (n & 7) >> 1, j = 2 * (n >> 3) + (n & 1);
  return __ldg(xbs_all + k * kN + gi * kD + j);  // table is gate-major
}

// Barrier, then thread 0 issues tile t's 5 MMAs (bias slot s) and commits.
__device__ __forceinline__ void issue(Smem& sm, int t, int s) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t d = sm.tmem + uint32_t(t * kN);
    const uint64_t ah = desc(su32(sm.a[t][0])), al = desc(su32(sm.a[t][1]));
    const uint64_t wh = desc(su32(sm.w[0])), wl = desc(su32(sm.w[1])), one = desc(su32(sm.one));
    mma(d, al, wh, 0u);
    mma(d, ah, wl, 1u);
    mma(d, ah, wh, 1u);
    mma(d, one, desc(su32(sm.bias[s][1])), 1u);
    mma(d, one, desc(su32(sm.bias[s][0])), 1u);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(&sm.mbar[t]))
                 : "memory");
  }
}

// Tile t epilogue: gates from TMEM -> new (h, c) of this row.
template <bool NR>
__device__ __forceinline__ void epilogue(const Smem& sm, int t, float2 (&h)[4], float2 (&c)[4]) {
  const uint32_t base = sm.tmem + (uint32_t((threadIdx.x >> 5) * 32) << 16) + uint32_t(t * kN);
  uint32_t g[4][8];
#pragma unroll
  for (int p = 0; p < 4; ++p)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(g[p][0]), "=r"(g[p][1]), "=r"(g[p][2]), "=r"(g[p][3]), "=r"(g[p][4]), "=r"(g[p][5]),
                   "=r"(g[p][6]), "=r"(g[p][7])
                 : "r"(base + uint32_t(8 * p)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const float2 f = make_float2(__uint_as_float(g[p][0]), __uint_as_float(g[p][1]));
    const float2 ig = make_float2(__uint_as_float(g[p][2]), __uint_as_float(g[p][3]));
    const float2 o = make_float2(__uint_as_float(g[p][4]), __uint_as_float(g[p][5]));
    const float2 gg = make_float2(__uint_as_float(g[p][6]), __uint_as_float(g[p][7]));
    h[p] = NR ? fwd_unit_nr(f, ig, o, gg, c[p]) : fwd_unit(f, ig, o, gg, c[p]);
  }
}

__device__ __forceinline__ void load_row(const float* __restrict__ x, int64_t B, int64_t b, int base, float2 (&v)[4]) {
#pragma unroll
  for (int p = 0; p < 4; ++p)
    v[p] = make_float2(__ldg(x + int64_t(base + 2 * p) * B + b), __ldg(x + int64_t(base + 2 * p + 1) * B + b));
}
__device__ __forceinline__ void store_row(float* __restrict__ x, int64_t B, int64_t b, int base, const float2 (&v)[4]) {
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    x[int64_t(base + 2 * p) * B + b] = v[p].x;
    x[int64_t(base + 2 * p + 1) * B + b] = v[p].y;
  }
}

template <bool TAPE, bool NR>
__global__ void __launch_bounds__(kThreads, 7)
    fwd_tcp(const float* __restrict__ in, float* __restrict__ out, int64_t B, const float* __restrict__ xbs_all,
            int64_t from, int count, const __grid_constant__ Weights w, const __grid_constant__ OutPtrs outs) {
  __shared__ __align__(128) Smem sm;
  const int r = threadIdx.x;
  const int64_t b[2] = {int64_t(blockIdx.x) * kTile + r, int64_t(blockIdx.x) * kTile + 128 + r};
  const bool live[2] = {b[0] < B, b[1] < B};
  if (r < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&sm.tmem)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (r == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  *reinterpret_cast<float4*>(&sm.one[kofs(r, 0)]) = make_float4(1.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(&sm.one[kofs(r, 4)]) = make_float4(0.f, 0.f, 0.f, 0.f);
  if (r < kN) {
    const int gi = (r & 7) >> 1, j = 2 * (r >> 3) + (r & 1);
#pragma unroll
    for (int k = 0; k < kD; ++k) {
      const float x = w.ws[gi][j][k];
      sm.w[0][kofs(r, k)] = hi_part(x);
      sm.w[1][kofs(r, k)] = x - hi_part(x);
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        sm.bias[s][0][kofs(r, k)] = 0.f;
        sm.bias[s][1][kofs(r, k)] = 0.f;
      }
    }
  }
  float2 h[2][4], c[2][4];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (live[t]) {
      load_row(in, B, b[t], 0, h[t]);
      load_row(in, B, b[t], kD, c[t]);
    } else {
#pragma unroll
      for (int p = 0; p < 4; ++p) h[t][p] = c[t][p] = make_float2(0.f, 0.f);
    }
  }
  // prologue: both tiles' step-0 products
  stage_bias(sm, 0, load_bias(xbs_all, from));
  stage_a(sm, 0, h[0]);
  stage_a(sm, 1, h[1]);
  issue(sm, 0, 0);
  if (r == 0) {
    const uint32_t d = sm.tmem + uint32_t(kN);  // tile 1, same bias slot (no barrier needed in between)
    const uint64_t ah = desc(su32(sm.a[1][0])), al = desc(su32(sm.a[1][1]));
    const uint64_t wh = desc(su32(sm.w[0])), wl = desc(su32(sm.w[1])), one = desc(su32(sm.one));
    mma(d, al, wh, 0u);
    mma(d, ah, wl, 1u);
    mma(d, ah, wh, 1u);
    mma(d, one, desc(su32(sm.bias[0][1])), 1u);
    mma(d, one, desc(su32(sm.bias[0][0])), 1u);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     su32(&sm.mbar[1]))
                 : "memory");
  }
  float xb = count > 1 ? load_bias(xbs_all, from + 1) : 0.f;
  for (int i = 0; i < count; ++i) {
    const bool more = i + 1 < count;
    const int slot = (i + 1) & 1;
    // tile 0
    wait_bar(&sm.mbar[0], uint32_t(i & 1));
    epilogue<NR>(sm, 0, h[0], c[0]);
    if (TAPE && live[0]) {
      store_row(outs.p[i], B, b[0], 0, h[0]);
      store_row(outs.p[i], B, b[0], kD, c[0]);
    }
    if (more) {
      stage_bias(sm, slot, xb);
      stage_a(sm, 0, h[0]);
      issue(sm, 0, slot);
      if (i + 2 < count) xb = load_bias(xbs_all, from + i + 2);
    }
    // tile 1
    wait_bar(&sm.mbar[1], uint32_t(i & 1));
    epilogue<NR>(sm, 1, h[1], c[1]);
    if (TAPE && live[1]) {
      store_row(outs.p[i], B, b[1], 0, h[1]);
      store_row(outs.p[i], B, b[1], kD, c[1]);
    }
    if (more) {
      stage_a(sm, 1, h[1]);
      issue(sm, 1, slot);
    }
  }
  if (!TAPE) {
#pragma unroll
    for (int t = 0; t < 2; ++t)
      if (live[t]) {
        store_row(out, B, b[t], 0, h[t]);
        store_row(out, B, b[t], kD, c[t]);
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (r < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem), "r"(64));
}

}  // namespace tcp
}  // namespace ackpt
