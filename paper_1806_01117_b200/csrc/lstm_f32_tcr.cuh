// Tensor-core reverse run for d = 8 with both products on tcgen05 and the
// two tiles in ping-pong (opt-in, ACKPT_TC_REV=3):
//   per step:  gates MMA (both tiles) -> epilogue tile 0 -> dh MMA tile 0
//              -> epilogue tile 1 (hides tile 0's MMA) -> dh MMA tile 1
// CTA = 128 threads, 256 sequences: tile 0 = b0 + r, tile 1 = b0 + 128 + r
// (thread r = row r of both, arithmetic packed over unit pairs).  Gate rows
// n = 8p + 2 gate + e (unit 2p + e); da back into TMEM as the A operand of
// dh = da . B2^T (tf32 head in place over G, bf16 residual, as rev_tc2).
// TMEM (128 columns): G_t [32t, 32t+32), lo_t [64 + 16t, +16), dh_t [96 + 16t, +16).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "lstm_f32_math.cuh"

namespace ackpt {
namespace tcr {

using namespace f32m;

constexpr int kThreads = 128;
constexpr int kTile = 256;
constexpr int kD = 8;
constexpr int kN = 32;
constexpr uint32_t kIdesc1 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(kN >> 3) << 17) | (uint32_t(128 >> 4) << 24);
constexpr uint32_t kIdescT = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(16 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
constexpr uint32_t kIdescB = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(16 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
constexpr uint32_t kLo = 64, kDh = 96;

struct Weights {
  float ws[4][kD][kD];
};
struct StatePtrs {
  const float* p[ACKPT_MAX_FUSED];
};

// K = 8 operand (gates): 8-row groups of two core matrices (LBO 128, SBO 256)
__device__ __forceinline__ int kofs8(int r, int k) { return (r >> 3) * 64 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3); }
// K = 32 operand (B2, 16 rows): K chunks of 2 row groups (LBO 256, SBO 128)
__device__ __forceinline__ int kofs32(int m, int k) { return (k >> 2) * 64 + (m >> 3) * 32 + (m & 7) * 4 + (k & 3); }
__device__ __forceinline__ int kofs32b(int m, int k) { return (k >> 3) * 128 + (m >> 3) * 64 + (m & 7) * 8 + (k & 7); }
__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ float hi_part(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

struct Smem {
  float a[2][2][128 * kD];        // [tile][hi, lo] h rows
  float one[128 * kD];
  float w[2][kN * kD];            // gate rows n, hi / lo
  float bias[2][kN * kD];         // hi / lo, column 0
  float b2[2][16 * kN];           // B2 tf32 hi / lo
  __nv_bfloat16 b2b[16 * kN];     // B2 bf16
  float st[2 * kD][kTile];        // prefetched taped state of the next step
  uint64_t mbar_g, mbar2[2], mbar_st;
  uint32_t tmem;
};

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc, bool f16) {
  if (f16)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
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
__device__ __forceinline__ void publish() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
}
__device__ __forceinline__ uint32_t bf16x2(float even, float odd) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(odd), "f"(even));
  return r;
}
__device__ __forceinline__ void stage_state(Smem& sm, const float* state, int64_t B, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&sm.mbar_st)),
               "r"(bytes * uint32_t(2 * kD))
               : "memory");
  const float* src = state + int64_t(blockIdx.x) * kTile;
#pragma unroll 1
  for (int j = 0; j < 2 * kD; ++j)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm.st[j])),
                 "l"(src + int64_t(j) * B), "r"(bytes), "r"(su32(&sm.mbar_st))
                 : "memory");
}
__device__ __forceinline__ float load_bias(const float* __restrict__ xbs_all, int64_t k) {
  const int n = threadIdx.x;
  if (n >= kN) return 0.f;
  const int gi = (n & 7) >> 1, j = 2 * (n >> 3) + (n & 1);
  return __ldg(xbs_all + k * kN + gi * kD + j);  // table is gate-major
}

// Tile t: gates -> gate adjoints (dc updated) -> da into TMEM (hi in place, lo bf16).
__device__ __forceinline__ void epilogue(uint32_t tmem, uint32_t lane, int t, const float2 (&c)[4],
                                         const float2 (&dh)[4], float2 (&dc)[4]) {
  const uint32_t g0 = tmem + lane + uint32_t(t * kN);
  uint32_t g[4][8];
#pragma unroll
  for (int p = 0; p < 4; ++p)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(g[p][0]), "=r"(g[p][1]), "=r"(g[p][2]), "=r"(g[p][3]), "=r"(g[p][4]), "=r"(g[p][5]),
                   "=r"(g[p][6]), "=r"(g[p][7])
                 : "r"(g0 + uint32_t(8 * p)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    float2 da[4];
    bwd_unit(make_float2(__uint_as_float(g[p][0]), __uint_as_float(g[p][1])),
             make_float2(__uint_as_float(g[p][2]), __uint_as_float(g[p][3])),
             make_float2(__uint_as_float(g[p][4]), __uint_as_float(g[p][5])),
             make_float2(__uint_as_float(g[p][6]), __uint_as_float(g[p][7])), c[p], dh[p], dc[p], da[0], da[1],
             da[2], da[3], dc[p]);
    uint32_t hv[8], lv[4];
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
      const float2 hi = make_float2(hi_part(da[gi].x), hi_part(da[gi].y));
      const float2 lo = sub2(da[gi], hi);
      hv[2 * gi] = __float_as_uint(hi.x);
      hv[2 * gi + 1] = __float_as_uint(hi.y);
      lv[gi] = bf16x2(lo.x, lo.y);
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(g0 + uint32_t(8 * p)),
                 "r"(hv[0]), "r"(hv[1]), "r"(hv[2]), "r"(hv[3]), "r"(hv[4]), "r"(hv[5]), "r"(hv[6]), "r"(hv[7])
                 : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(
                     tmem + lane + kLo + uint32_t(16 * t + 4 * p)),
                 "r"(lv[0]), "r"(lv[1]), "r"(lv[2]), "r"(lv[3])
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Thread 0: dh_t = da_t . B2^T (tf32 head x B2 hi/lo over 4 K-steps, bf16 residual x B2 over 2).
__device__ __forceinline__ void issue_dh(Smem& sm, uint32_t tmem, int t) {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t d = tmem + kDh + uint32_t(16 * t), a = tmem + uint32_t(t * kN);
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    const uint32_t off = uint32_t(ks) * 512u;
    mma_ts(d, a + uint32_t(8 * ks), desc(su32(sm.b2[1]) + off, 256, 128), kIdescT, ks ? 1u : 0u, false);
    mma_ts(d, a + uint32_t(8 * ks), desc(su32(sm.b2[0]) + off, 256, 128), kIdescT, 1u, false);
  }
#pragma unroll
  for (int ks = 0; ks < 2; ++ks)
    mma_ts(d, tmem + kLo + uint32_t(16 * t + 8 * ks), desc(su32(sm.b2b) + uint32_t(ks) * 512u, 256, 128), kIdescB, 1u,
           true);
  commit(&sm.mbar2[t]);
}

__global__ void __launch_bounds__(kThreads, 4)
    rev_tcr(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B, const float* __restrict__ xbs_all,
            int64_t from, int count, const __grid_constant__ Weights w, const __grid_constant__ StatePtrs states) {
  __shared__ __align__(128) Smem sm;
  const int r = threadIdx.x;
  const int64_t base = int64_t(blockIdx.x) * kTile;
  const int64_t b[2] = {base + r, base + 128 + r};
  const bool live[2] = {b[0] < B, b[1] < B};
  const int64_t rem = B - base;
  const uint32_t seg = uint32_t(rem < kTile ? rem : kTile) * 4u;
  if (r < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&sm.tmem)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // constant operands
  *reinterpret_cast<float4*>(&sm.one[kofs8(r, 0)]) = make_float4(1.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(&sm.one[kofs8(r, 4)]) = make_float4(0.f, 0.f, 0.f, 0.f);
  if (r < kN) {
    const int gi = (r & 7) >> 1, j = 2 * (r >> 3) + (r & 1);
#pragma unroll
    for (int k = 0; k < kD; ++k) {
      const float x = w.ws[gi][j][k];
      sm.w[0][kofs8(r, k)] = hi_part(x);
      sm.w[1][kofs8(r, k)] = x - hi_part(x);
      sm.bias[0][kofs8(r, k)] = 0.f;
      sm.bias[1][kofs8(r, k)] = 0.f;
    }
  }
  for (int idx = r; idx < 16 * kN; idx += kThreads) {  // B2[m][n] = s_g W_g[j(n)][m]
    const int m = idx / kN, n = idx % kN, gi = (n & 7) >> 1, j = 2 * (n >> 3) + (n & 1);
    const float x = m < kD ? w.ws[gi][j][m] : 0.f;
    sm.b2[0][kofs32(m, n)] = hi_part(x);
    sm.b2[1][kofs32(m, n)] = x - hi_part(x);
    sm.b2b[kofs32b(m, n)] = __float2bfloat16_rn(x);
  }
  if (r == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar_g)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar2[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar2[1])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar_st)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stage_state(sm, states.p[count - 1], B, seg);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(&sm.tmem);
  const uint32_t lane = uint32_t((r >> 5) * 32) << 16;
  float2 dh[2][4], dc[2][4];
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      dh[t][p] = live[t] ? make_float2(__ldg(adj_in + int64_t(2 * p) * B + b[t]), __ldg(adj_in + int64_t(2 * p + 1) * B + b[t]))
                         : make_float2(0.f, 0.f);
      dc[t][p] = live[t] ? make_float2(__ldg(adj_in + int64_t(kD + 2 * p) * B + b[t]),
                                       __ldg(adj_in + int64_t(kD + 2 * p + 1) * B + b[t]))
                         : make_float2(0.f, 0.f);
    }
  float xb = load_bias(xbs_all, from + count - 1);
  uint32_t ph = 0;
  for (int i = count - 1; i >= 0; --i, ph ^= 1u) {
    // taped state (both tiles) from shared memory, staged as the gates' A operand
    wait_bar(&sm.mbar_st, ph);
    float2 c[2][4];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      float2 h[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        h[p] = make_float2(sm.st[2 * p][128 * t + r], sm.st[2 * p + 1][128 * t + r]);
        c[t][p] = make_float2(sm.st[kD + 2 * p][128 * t + r], sm.st[kD + 2 * p + 1][128 * t + r]);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float4 x = make_float4(h[2 * q].x, h[2 * q].y, h[2 * q + 1].x, h[2 * q + 1].y);
        const float4 hx = make_float4(hi_part(x.x), hi_part(x.y), hi_part(x.z), hi_part(x.w));
        const float2 l01 = sub2(make_float2(x.x, x.y), make_float2(hx.x, hx.y));
        const float2 l23 = sub2(make_float2(x.z, x.w), make_float2(hx.z, hx.w));
        *reinterpret_cast<float4*>(&sm.a[t][0][kofs8(r, 4 * q)]) = hx;
        *reinterpret_cast<float4*>(&sm.a[t][1][kofs8(r, 4 * q)]) = make_float4(l01.x, l01.y, l23.x, l23.y);
      }
    }
    if (r < kN) {
      sm.bias[0][kofs8(r, 0)] = hi_part(xb);
      sm.bias[1][kofs8(r, 0)] = xb - hi_part(xb);
    }
    if (i > 0) xb = load_bias(xbs_all, from + i - 1);
    publish();  // every thread has read sm.st and written its A rows
    if (r == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t wh = desc(su32(sm.w[0]), 128, 256), wl = desc(su32(sm.w[1]), 128, 256);
      const uint64_t one = desc(su32(sm.one), 128, 256);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint32_t d = tmem + uint32_t(t * kN);
        const uint64_t ah = desc(su32(sm.a[t][0]), 128, 256), al = desc(su32(sm.a[t][1]), 128, 256);
        mma_ss(d, al, wh, kIdesc1, 0u);
        mma_ss(d, ah, wl, kIdesc1, 1u);
        mma_ss(d, ah, wh, kIdesc1, 1u);
        mma_ss(d, one, desc(su32(sm.bias[1]), 128, 256), kIdesc1, 1u);
        mma_ss(d, one, desc(su32(sm.bias[0]), 128, 256), kIdesc1, 1u);
      }
      commit(&sm.mbar_g);
      if (i > 0) stage_state(sm, states.p[i - 1], B, seg);
    }
    wait_bar(&sm.mbar_g, ph);
    // tile 0 adjoints -> its dh MMA, overlapped with tile 1's adjoints
    epilogue(tmem, lane, 0, c[0], dh[0], dc[0]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (r == 0) issue_dh(sm, tmem, 0);
    epilogue(tmem, lane, 1, c[1], dh[1], dc[1]);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (r == 0) issue_dh(sm, tmem, 1);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      wait_bar(&sm.mbar2[t], ph);
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                   : "r"(tmem + lane + kDh + uint32_t(16 * t)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int p = 0; p < 4; ++p) dh[t][p] = make_float2(__uint_as_float(v[2 * p]), __uint_as_float(v[2 * p + 1]));
    }
  }
#pragma unroll
  for (int t = 0; t < 2; ++t)
    if (live[t]) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        adj_out[int64_t(2 * p) * B + b[t]] = dh[t][p].x;
        adj_out[int64_t(2 * p + 1) * B + b[t]] = dh[t][p].y;
        adj_out[int64_t(kD + 2 * p) * B + b[t]] = dc[t][p].x;
        adj_out[int64_t(kD + 2 * p + 1) * B + b[t]] = dc[t][p].y;
      }
    }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (r < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

}  // namespace tcr
}  // namespace ackpt
