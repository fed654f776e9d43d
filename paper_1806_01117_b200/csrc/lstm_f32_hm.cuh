// Register-fragment tensor-core LSTM kernels (warp-level mma.sync, tf32
// m16n8k8, 3xTF32 split), hidden size 8: fused Advance, TapeForward and
// Reverse runs.  No TMEM, shared memory, barriers or mbarriers: each warp
// steps its own 16 sequences with every operand in registers.
//
// Fragment bookkeeping (m16n8k8, lane = 4 g + t):
//   A (16 x 8):  a0 = A[g][t], a1 = A[g+8][t], a2 = A[g][t+4], a3 = A[g+8][t+4]
//   B (8 x 8):   b0 = B[t][g], b1 = B[t+4][g]
//   C (16 x 8):  c0 = C[g][2t], c1 = C[g][2t+1], c2 = C[g+8][2t], c3 = C[g+8][2t+1]
// Rows g and g+8 of a warp's tile are sequences e0 = base + 2g and e0 + 1
// (adjacent: float2 loads / stores of the batch-fastest state), and thread
// (g, t) owns hidden units t and t+4 of both.  With the column maps below
// every product lands where the next one needs it, so no shuffles:
//   gates:  G[r][n] = sum_k h[r][k] W_gate[u(n)][k], one n-tile per gate,
//           u(n) = n/2 + 4 (n%2): c0/c1 = units t, t+4 of row g (a float2
//           for the packed activation math), c2/c3 of row g+8; the step's
//           bias initialises C; the new h is next step's A fragment.
//   reverse: dh[r][m(n)] = sum_k da[r][k] B2[k][n], k = 8 gate + unit, so the
//           thread's own gate adjoints are the A fragment and c0/c1 are
//           dh of units t, t+4: next step's adjoint layout.
// All weights are the pre-scaled s_g W_g of lstm_f32_math.cuh (accumulators
// are ex2 arguments; the reverse uses the scaled adjoints of bwd_unit).
// Accuracy: x.y ~ x_lo.y_hi + x_hi.y_lo + x_hi.y_hi (hi = tf32 bits), the
// same split as the tcgen05 family.
#pragma once

#include <cuda_runtime.h>

#include "lstm_f32_math.cuh"

namespace ackpt {
namespace hm {

using namespace f32m;

constexpr int kD = 8;
constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kRows = 16;  // sequences per warp

struct OutPtrs {
  float* p[ACKPT_MAX_FUSED];
};
struct StatePtrs {
  const float* p[ACKPT_MAX_FUSED];
};

__device__ __forceinline__ uint32_t hi_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }
__device__ __forceinline__ float f(uint32_t x) { return __uint_as_float(x); }

__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                    uint32_t b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// A fragment of rows (g, g+8) from their float2 (units t, t+4), split hi / lo.
struct Split {
  uint32_t h[4], l[4];
  __device__ __forceinline__ Split(float2 x0, float2 x1) {
    h[0] = hi_bits(x0.x);
    h[1] = hi_bits(x1.x);
    h[2] = hi_bits(x0.y);
    h[3] = hi_bits(x1.y);
    const float2 l0 = sub2(x0, make_float2(f(h[0]), f(h[2])));
    const float2 l1 = sub2(x1, make_float2(f(h[1]), f(h[3])));
    l[0] = __float_as_uint(l0.x);
    l[1] = __float_as_uint(l1.x);
    l[2] = __float_as_uint(l0.y);
    l[3] = __float_as_uint(l1.y);
  }
};

// c += A . B with 3xTF32 (small terms first).
__device__ __forceinline__ void mma3(float (&c)[4], const Split& a, uint32_t bh0, uint32_t bh1, uint32_t bl0,
                                     uint32_t bl1) {
  mma(c, a.l[0], a.l[1], a.l[2], a.l[3], bh0, bh1);
  mma(c, a.h[0], a.h[1], a.h[2], a.h[3], bl0, bl1);
  mma(c, a.h[0], a.h[1], a.h[2], a.h[3], bh0, bh1);
}

// Per-lane constant B fragments: [0, 8) gates hi, [8, 16) gates lo,
// [16, 24) transposed hi, [24, 32) transposed lo; entry 2 gate + (0: b0, 1: b1).
struct Frags {
  uint32_t w[32];
  __device__ __forceinline__ void load(const float* __restrict__ table, int lane, bool reverse) {
    const float4* p = reinterpret_cast<const float4*>(table + lane * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 v = __ldg(p + q);
      w[4 * q] = __float_as_uint(v.x);
      w[4 * q + 1] = __float_as_uint(v.y);
      w[4 * q + 2] = __float_as_uint(v.z);
      w[4 * q + 3] = __float_as_uint(v.w);
    }
    if (reverse) {
#pragma unroll
      for (int q = 4; q < 8; ++q) {
        const float4 v = __ldg(p + q);
        w[4 * q] = __float_as_uint(v.x);
        w[4 * q + 1] = __float_as_uint(v.y);
        w[4 * q + 2] = __float_as_uint(v.z);
        w[4 * q + 3] = __float_as_uint(v.w);
      }
    }
  }
};

// Scaled step bias of this thread: [2 gate + e] = xb_gate[t + 4 e] (table [k][t][8]).
struct Bias {
  float4 a, b;
  __device__ __forceinline__ void load(const float* __restrict__ xbs_hm, int64_t k, int t) {
    const float4* p = reinterpret_cast<const float4*>(xbs_hm + (k * 4 + t) * 8);
    a = __ldg(p);
    b = __ldg(p + 1);
  }
  __device__ __forceinline__ float2 gate(int gidx) const {
    return gidx == 0 ? make_float2(a.x, a.y) : gidx == 1 ? make_float2(a.z, a.w)
         : gidx == 2 ? make_float2(b.x, b.y) : make_float2(b.z, b.w);
  }
};

// Scaled gate pre-activations of rows g (x0) and g+8 (x1) for units (t, t+4).
struct Gates {
  float2 r0[4], r1[4];  // [gate]
};

__device__ __forceinline__ void gates(const Frags& fr, const Bias& bias, float2 h0, float2 h1, Gates& out) {
  const Split a(h0, h1);
#pragma unroll
  for (int gi = 0; gi < 4; ++gi) {
    const float2 b = bias.gate(gi);
    float c[4] = {b.x, b.y, b.x, b.y};
    mma3(c, a, fr.w[2 * gi], fr.w[2 * gi + 1], fr.w[8 + 2 * gi], fr.w[8 + 2 * gi + 1]);
    out.r0[gi] = make_float2(c[0], c[1]);
    out.r1[gi] = make_float2(c[2], c[3]);
  }
}

// Rows (e0, e0+1) x units (t, t+4) of feature block `base` (0: h, D: c):
// two float2 loads of adjacent sequences, regrouped per row.
__device__ __forceinline__ void load_pair(const float* __restrict__ x, int64_t B, int64_t e0, int t, int base,
                                          float2& r0, float2& r1) {
  const float2 u = *reinterpret_cast<const float2*>(x + int64_t(base + t) * B + e0);
  const float2 v = *reinterpret_cast<const float2*>(x + int64_t(base + t + 4) * B + e0);
  r0 = make_float2(u.x, v.x);
  r1 = make_float2(u.y, v.y);
}
__device__ __forceinline__ void store_pair(float* __restrict__ x, int64_t B, int64_t e0, int t, int base, float2 r0,
                                           float2 r1) {
  *reinterpret_cast<float2*>(x + int64_t(base + t) * B + e0) = make_float2(r0.x, r1.x);
  *reinterpret_cast<float2*>(x + int64_t(base + t + 4) * B + e0) = make_float2(r0.y, r1.y);
}

// Fused forward over `count` steps from `from`: TAPE stores every step's
// output state to outs.p[i], otherwise only the final state to `out`.
template <bool TAPE, bool NR>
__global__ void __launch_bounds__(kThreads)
    fwd_hm(const float* __restrict__ in, float* __restrict__ out, int64_t B, const float* __restrict__ xbs_hm,
           const float* __restrict__ frag, int64_t from, int count, const __grid_constant__ OutPtrs outs) {
  const int lane = threadIdx.x & 31, t = lane & 3;
  const int64_t e0 = (int64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5)) * kRows + 2 * (lane >> 2);
  const bool live = e0 < B;  // B even: e0 + 1 < B as well
  Frags fr;
  fr.load(frag, lane, false);
  float2 h0 = make_float2(0.f, 0.f), h1 = h0, c0 = h0, c1 = h0;
  if (live) {
    load_pair(in, B, e0, t, 0, h0, h1);
    load_pair(in, B, e0, t, kD, c0, c1);
  }
  Bias bias, next;
  bias.load(xbs_hm, from, t);
  for (int i = 0; i < count; ++i) {
    if (i + 1 < count) next.load(xbs_hm, from + i + 1, t);
    Gates gt;
    gates(fr, bias, h0, h1, gt);
    if (NR) {
      h0 = fwd_unit_nr(gt.r0[0], gt.r0[1], gt.r0[2], gt.r0[3], c0);
      h1 = fwd_unit_nr(gt.r1[0], gt.r1[1], gt.r1[2], gt.r1[3], c1);
    } else {
      h0 = fwd_unit(gt.r0[0], gt.r0[1], gt.r0[2], gt.r0[3], c0);
      h1 = fwd_unit(gt.r1[0], gt.r1[1], gt.r1[2], gt.r1[3], c1);
    }
    if (TAPE && live) {
      store_pair(outs.p[i], B, e0, t, 0, h0, h1);
      store_pair(outs.p[i], B, e0, t, kD, c0, c1);
    }
    bias = next;
  }
  if (!TAPE && live) {
    store_pair(out, B, e0, t, 0, h0, h1);
    store_pair(out, B, e0, t, kD, c0, c1);
  }
}

// Fused run of Reverse actions, steps from+count-1 .. from: gates and the
// transposed matvec on the tensor cores, the taped state of the next step
// loaded one step ahead.
template <bool NR>
__global__ void __launch_bounds__(kThreads)
    rev_hm(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B, const float* __restrict__ xbs_hm,
           const float* __restrict__ frag, int64_t from, int count, const __grid_constant__ StatePtrs states) {
  const int lane = threadIdx.x & 31, t = lane & 3;
  const int64_t e0 = (int64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5)) * kRows + 2 * (lane >> 2);
  const bool live = e0 < B;
  Frags fr;
  fr.load(frag, lane, true);
  float2 dh0 = make_float2(0.f, 0.f), dh1 = dh0, dc0 = dh0, dc1 = dh0;
  if (live) {
    load_pair(adj_in, B, e0, t, 0, dh0, dh1);
    load_pair(adj_in, B, e0, t, kD, dc0, dc1);
  }
  // taped states two steps ahead (DRAM latency exceeds one short iteration)
  float2 h0n = make_float2(0.f, 0.f), h1n = h0n, c0n = h0n, c1n = h0n;
  float2 h0m = h0n, h1m = h0n, c0m = h0n, c1m = h0n;
  if (live) {
    load_pair(states.p[count - 1], B, e0, t, 0, h0n, h1n);
    load_pair(states.p[count - 1], B, e0, t, kD, c0n, c1n);
    if (count > 1) {
      load_pair(states.p[count - 2], B, e0, t, 0, h0m, h1m);
      load_pair(states.p[count - 2], B, e0, t, kD, c0m, c1m);
    }
  }
  Bias bias, next;
  bias.load(xbs_hm, from + count - 1, t);
  for (int i = count - 1; i >= 0; --i) {
    const float2 h0 = h0n, h1 = h1n, c0 = c0n, c1 = c1n;
    h0n = h0m;
    h1n = h1m;
    c0n = c0m;
    c1n = c1m;
    if (i > 0) next.load(xbs_hm, from + i - 1, t);
    if (i > 1 && live) {
      load_pair(states.p[i - 2], B, e0, t, 0, h0m, h1m);
      load_pair(states.p[i - 2], B, e0, t, kD, c0m, c1m);
    }
    Gates gt;
    gates(fr, bias, h0, h1, gt);
    float2 da0[4], da1[4];
    if (NR) {
      bwd_unit_nr(gt.r0[0], gt.r0[1], gt.r0[2], gt.r0[3], c0, dh0, dc0, da0[0], da0[1], da0[2], da0[3], dc0);
      bwd_unit_nr(gt.r1[0], gt.r1[1], gt.r1[2], gt.r1[3], c1, dh1, dc1, da1[0], da1[1], da1[2], da1[3], dc1);
    } else {
      bwd_unit(gt.r0[0], gt.r0[1], gt.r0[2], gt.r0[3], c0, dh0, dc0, da0[0], da0[1], da0[2], da0[3], dc0);
      bwd_unit(gt.r1[0], gt.r1[1], gt.r1[2], gt.r1[3], c1, dh1, dc1, da1[0], da1[1], da1[2], da1[3], dc1);
    }
    // dh = da . B2 over K = 32 (chunk = gate), two accumulators to halve the chain
    float ea[4] = {0.f, 0.f, 0.f, 0.f}, eb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
      const Split a(da0[gi], da1[gi]);
      mma3(gi & 1 ? eb : ea, a, fr.w[16 + 2 * gi], fr.w[16 + 2 * gi + 1], fr.w[24 + 2 * gi], fr.w[24 + 2 * gi + 1]);
    }
    dh0 = add2(make_float2(ea[0], ea[1]), make_float2(eb[0], eb[1]));
    dh1 = add2(make_float2(ea[2], ea[3]), make_float2(eb[2], eb[3]));
    bias = next;
  }
  if (live) {
    store_pair(adj_out, B, e0, t, 0, dh0, dh1);
    store_pair(adj_out, B, e0, t, kD, dc0, dc1);
  }
}

}  // namespace hm
}  // namespace ackpt
