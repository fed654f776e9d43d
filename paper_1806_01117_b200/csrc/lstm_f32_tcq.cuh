// tcgen05 forward for d = 8 with P float2 pairs of sequences per thread
// (fused Advance / TapeForward).  Same arithmetic as fwd_tc (P = 1): the
// per-step fixed work of a CTA (operand staging, barrier, MMA issue, the
// mbarrier wait, bias load, address arithmetic) is shared by P pairs, and
// each thread carries P independent dependency chains.
// CTA = 128 threads, 256 P sequences; pair q of thread r is (base + 256 q +
// 2r, +1), tiles 2q (x lanes) and 2q+1 (y lanes), TMEM columns 32 t.
#pragma once

#include "lstm_f32_tc.cuh"

namespace ackpt {
namespace tcq {

using namespace f32m;
using tc::desc;
using tc::hi_part;
using tc::kD;
using tc::kN;
using tc::kofs;
using tc::ld8;
using tc::ldg2;
using tc::load_bias;
using tc::mbar_wait;
using tc::mma;
using tc::OutPtrs;
using tc::stg2;
using tc::su32;
using tc::Weights;

constexpr int kThreads = 128;

template <int P>
struct Smem {
  float a[2 * P][2][128 * kD];  // [tile][hi, lo]
  float a1[128 * kD];
  float bw[2][kN * kD];
  float bb[2][kN * kD];
  uint64_t mbar;
  uint32_t tmem;
};

template <int P>
__global__ void __launch_bounds__(kThreads, (P == 1 ? 8 : 4))
    fwd_tcq(const float* __restrict__ in, float* __restrict__ out, int64_t B, const float* __restrict__ xbs_all,
            int64_t from, int count, bool tape, const __grid_constant__ Weights w, const __grid_constant__ OutPtrs outs) {
  __shared__ __align__(128) Smem<P> sm;
  const int tid = threadIdx.x;
  const int64_t base = int64_t(blockIdx.x) * 256 * P;
  int64_t b0[P];
  bool live[P];
#pragma unroll
  for (int q = 0; q < P; ++q) {
    b0[q] = base + 256 * q + 2 * tid;
    live[q] = b0[q] < B;
  }
  constexpr uint32_t kCols = 64 * P;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&sm.tmem)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  *reinterpret_cast<float4*>(&sm.a1[kofs(tid, 0)]) = make_float4(1.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(&sm.a1[kofs(tid, 4)]) = make_float4(0.f, 0.f, 0.f, 0.f);
  if (tid < kN) {
    const int j = tid >> 2, g = tid & 3;
#pragma unroll
    for (int k = 0; k < kD; ++k) {
      const float x = w.ws[g][j][k];
      sm.bw[0][kofs(tid, k)] = hi_part(x);
      sm.bw[1][kofs(tid, k)] = x - hi_part(x);
      sm.bb[0][kofs(tid, k)] = 0.f;
      sm.bb[1][kofs(tid, k)] = 0.f;
    }
  }
  float2 h[P][kD], c[P][kD];
#pragma unroll
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int j = 0; j < kD; ++j) {
      h[q][j] = live[q] ? ldg2(in + b0[q] + int64_t(j) * B) : make_float2(0.f, 0.f);
      c[q][j] = live[q] ? ldg2(in + b0[q] + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
    }
  const uint32_t lane = uint32_t((tid >> 5) * 32) << 16;
  float xb = load_bias(xbs_all, from);
  for (int i = 0; i < count; ++i) {
    // stage A (h hi / lo of every tile) and the bias column
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const float4 a = make_float4(h[q][4 * cc].x, h[q][4 * cc + 1].x, h[q][4 * cc + 2].x, h[q][4 * cc + 3].x);
        const float4 b = make_float4(h[q][4 * cc].y, h[q][4 * cc + 1].y, h[q][4 * cc + 2].y, h[q][4 * cc + 3].y);
        const float4 ah = make_float4(hi_part(a.x), hi_part(a.y), hi_part(a.z), hi_part(a.w));
        const float4 bh = make_float4(hi_part(b.x), hi_part(b.y), hi_part(b.z), hi_part(b.w));
        const float2 a01 = sub2(make_float2(a.x, a.y), make_float2(ah.x, ah.y));
        const float2 a23 = sub2(make_float2(a.z, a.w), make_float2(ah.z, ah.w));
        const float2 b01 = sub2(make_float2(b.x, b.y), make_float2(bh.x, bh.y));
        const float2 b23 = sub2(make_float2(b.z, b.w), make_float2(bh.z, bh.w));
        *reinterpret_cast<float4*>(&sm.a[2 * q][0][kofs(tid, 4 * cc)]) = ah;
        *reinterpret_cast<float4*>(&sm.a[2 * q][1][kofs(tid, 4 * cc)]) = make_float4(a01.x, a01.y, a23.x, a23.y);
        *reinterpret_cast<float4*>(&sm.a[2 * q + 1][0][kofs(tid, 4 * cc)]) = bh;
        *reinterpret_cast<float4*>(&sm.a[2 * q + 1][1][kofs(tid, 4 * cc)]) = make_float4(b01.x, b01.y, b23.x, b23.y);
      }
    if (tid < kN) {
      sm.bb[0][kofs(tid, 0)] = hi_part(xb);
      sm.bb[1][kofs(tid, 0)] = xb - hi_part(xb);
    }
    if (i + 1 < count) xb = load_bias(xbs_all, from + i + 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint64_t wh = desc(su32(sm.bw[0])), wl = desc(su32(sm.bw[1]));
      const uint64_t xh = desc(su32(sm.bb[0])), xl = desc(su32(sm.bb[1])), one = desc(su32(sm.a1));
#pragma unroll
      for (int t = 0; t < 2 * P; ++t) {
        const uint32_t d = sm.tmem + uint32_t(t * kN);
        const uint64_t ah = desc(su32(sm.a[t][0])), al = desc(su32(sm.a[t][1]));
        mma(d, ah, wh, 0u);
        mma(d, al, wh, 1u);
        mma(d, ah, wl, 1u);
        mma(d, one, xh, 1u);
        mma(d, one, xl, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32(&sm.mbar))
                   : "memory");
    }
    mbar_wait(&sm.mbar, uint32_t(i & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = sm.tmem + lane;
#pragma unroll
    for (int u = 0; u < kD; u += 2) {
      float v[2 * P][8];
#pragma unroll
      for (int t = 0; t < 2 * P; ++t) ld8(tm + uint32_t(t * kN + 4 * u), v[t]);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < P; ++q)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float* x = v[2 * q];
          const float* y = v[2 * q + 1];
          h[q][u + e] = fwd_unit_nr(make_float2(x[4 * e], y[4 * e]), make_float2(x[4 * e + 1], y[4 * e + 1]),
                                    make_float2(x[4 * e + 2], y[4 * e + 2]), make_float2(x[4 * e + 3], y[4 * e + 3]),
                                    c[q][u + e]);
        }
    }
    if (tape) {
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (live[q]) {
          float* dst = outs.p[i] + b0[q];
#pragma unroll
          for (int j = 0; j < kD; ++j) {
            stg2(dst + int64_t(j) * B, h[q][j]);
            stg2(dst + int64_t(kD + j) * B, c[q][j]);
          }
        }
    }
  }
  if (!tape) {
#pragma unroll
    for (int q = 0; q < P; ++q)
      if (live[q]) {
#pragma unroll
        for (int j = 0; j < kD; ++j) {
          stg2(out + b0[q] + int64_t(j) * B, h[q][j]);
          stg2(out + b0[q] + int64_t(kD + j) * B, c[q][j]);
        }
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem), "r"(kCols));
}

}  // namespace tcq
}  // namespace ackpt
