// Tensor-core (tcgen05) fused LSTM kernels for sm_100a, hidden size 8:
// fused Advance, fused TapeForward and fused Reverse runs.  Same results
// contract as lstm_f32.cuh (fp32 state, rel-L2 <= 1e-5 vs float64), different
// arithmetic for the gate matvec, so NOT bit-identical to the FFMA2 kernels:
// an execution uses one family for every step.
//
// Gate pre-activations of a step, for the 256 batch elements of a CTA, are one
// MMA problem per M-tile: D[128 x 32] = A[128 x 16] . B[32 x 16]^T with
//   A row r = [h_0..h_7, 1, 1, 1, 0 x 5]                         (element of the tile)
//   B row n = [s_g W_g[j][0..7], split3(s_g xb_k[g][j]), 0 x 5]  n = 4 j + g (unit-major)
// (s_g: the exponent scale folded into the weights, lstm_f32_math.cuh), so the
// bias / input projection of step k rides in the MMA and D holds the ex2
// arguments directly.  fp32 accuracy from TF32 tensor cores with the 3xTF32
// split x = hi + lo (hi = x rounded to tf32, lo = x - hi exact):
// A.B ~ Ahi.Bhi + Alo.Bhi + Ahi.Blo (rel. error <= ~2^-22), and the bias
// split exactly into three tf32 parts (one MMA, no split error).
// Operands are K-major, no swizzle, in shared memory; D (fp32) is in TMEM,
// one column per gate, one lane per tile row, read back with tcgen05.ld.
//
// CTA = 128 threads = the 128 TMEM lanes.  Tile 0 row r is element base+2r,
// tile 1 row r is element base+2r+1, so thread r owns the float2 pair at
// base+2r in global memory and processes it with the packed-fp32 math.
#pragma once

#include <cuda_runtime.h>

#include "chain.cuh"
#include "lstm_f32_math.cuh"

namespace ackpt {
namespace tc {

using namespace f32m;

constexpr int kThreads = 128;
constexpr int kTile = 256;     // elements per CTA
constexpr int kD = 8;          // hidden size
constexpr int kN = 4 * kD;     // gate columns
constexpr int kK = 8;          // one MMA K step
constexpr uint32_t kLBO = 128; // bytes between the two 16-byte K chunks (8 rows x 16 B core matrices)
constexpr uint32_t kSBO = 256; // bytes between 8-row groups
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(kN >> 3) << 17) | (uint32_t(128 >> 4) << 24);

// ~23 KB: h operands per tile (hi, lo), one constant bias operand
// A1 = [1, 1, 1, 0 x 5] shared by both tiles, the weights (hi, lo) and the
// step's bias split exactly into three tf32 parts (columns 0..2): the bias
// term enters the accumulator with no split error.  It is the same for every
// element of a step and dominates the forget-gate pre-activation of
// long-memory cells, so a split error there is systematic: over a 10^4-step
// chain it accumulated to ~1e-3 rel-L2 in the adjoint (2-way truncated split,
// tools/long_chain_err.py) against 1e-4 for exact fp32 FMAs.
// A1 is one 8-row group read with stride-byte-offset 0: all 16 row groups of
// the M = 128 operand alias it (256 B instead of 4 KB of shared memory).
struct Smem {
  float a[2][2][128 * kK];  // [tile][hi, lo]
  float a1[8 * kK];         // rows [1, 1, 1, 0, ..., 0], broadcast over the 16 row groups
  float bw[2][kN * kK];     // [hi, lo] scaled W rows n = 4 j + g
  float bb[kN * kK];        // row n: [hi, mid, lo] of scaled xb_k, rest 0
  uint64_t mbar;
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t sbo = kSBO) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((kLBO >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
// float offset of (row, k) in a K-major no-swizzle 16-wide operand
__device__ __forceinline__ int kofs(int r, int k) { return (r >> 3) * (kSBO / 4) + (k >> 2) * (kLBO / 4) + (r & 7) * 4 + (k & 3); }
// tf32 head of x rounded to nearest (ties away from zero, = cvt.rna.tf32.f32):
// x - hi_part(x) is exact in fp32 and at most half a tf32 ulp of x, so the
// MMA's truncation of that residual to tf32 costs <= 2^-23 |x|.
__device__ __forceinline__ float hi_part(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

// Unit pair (2 hidden units = 8 columns) of one tile row, from TMEM.
__device__ __forceinline__ void ld8(uint32_t addr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

struct Weights {
  float ws[4][kD][kD];  // pre-scaled (lstm_f32_math.cuh ScaledParams layout): gate products
  float wu[4][kD][kD];  // unscaled W_h: rev_tc's transposed matvec of true adjoints
};

// One-time CTA setup: TMEM, mbarrier, constant operand parts.
__device__ __forceinline__ void setup(Smem& sm, const Weights& w, uint32_t tmem_cols = 64) {
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&sm.tmem)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sm.mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // bias operand row of this thread: [1, 1, 1, 0, ..., 0]
  if (tid < 8) {
    *reinterpret_cast<float4*>(&sm.a1[kofs(tid, 0)]) = make_float4(1.f, 1.f, 1.f, 0.f);
    *reinterpret_cast<float4*>(&sm.a1[kofs(tid, 4)]) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  // weight rows n = 4 j + g (scaled, split), bias rows zero but for columns 0..2 (per step)
  if (tid < kN) {
    const int j = tid >> 2, g = tid & 3;
#pragma unroll
    for (int k = 0; k < kD; ++k) {
      const float x = w.ws[g][j][k];
      sm.bw[0][kofs(tid, k)] = hi_part(x);
      sm.bw[1][kofs(tid, k)] = x - hi_part(x);
      sm.bb[kofs(tid, k)] = 0.f;
    }
  }
}

// x = hi + mid + lo exactly, each part a tf32 value (11 + 11 + <= 2 bits).
__device__ __forceinline__ float4 split3(float x) {
  const float hi = hi_part(x), r = x - hi, mid = hi_part(r);
  return make_float4(hi, mid, r - mid, 0.f);
}

// Scaled bias of step k for B row n = tid (threads < kN), loaded one step ahead.
__device__ __forceinline__ float load_bias(const float* __restrict__ xbs_all, int64_t k) {
  const int tid = threadIdx.x;
  if (tid >= kN) return 0.f;
  return __ldg(xbs_all + k * kN + (tid & 3) * kD + (tid >> 2));  // table is gate-major
}

// Writes A (h hi/lo for both tiles) and, in warp 0, B's bias column (x from load_bias).
__device__ __forceinline__ void stage_operands(Smem& sm, const float2 (&h)[kD], float x) {
  const int tid = threadIdx.x;
  float4 hx[2], hy[2];
  hx[0] = make_float4(h[0].x, h[1].x, h[2].x, h[3].x);
  hx[1] = make_float4(h[4].x, h[5].x, h[6].x, h[7].x);
  hy[0] = make_float4(h[0].y, h[1].y, h[2].y, h[3].y);
  hy[1] = make_float4(h[4].y, h[5].y, h[6].y, h[7].y);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const float4 a = hx[c], b = hy[c];
    const float4 ah = make_float4(hi_part(a.x), hi_part(a.y), hi_part(a.z), hi_part(a.w));
    const float4 bh = make_float4(hi_part(b.x), hi_part(b.y), hi_part(b.z), hi_part(b.w));
    // lo = x - hi, packed two at a time (every FMA-pipe instruction costs 2 cycles)
    const float2 a01 = sub2(make_float2(a.x, a.y), make_float2(ah.x, ah.y));
    const float2 a23 = sub2(make_float2(a.z, a.w), make_float2(ah.z, ah.w));
    const float2 b01 = sub2(make_float2(b.x, b.y), make_float2(bh.x, bh.y));
    const float2 b23 = sub2(make_float2(b.z, b.w), make_float2(bh.z, bh.w));
    *reinterpret_cast<float4*>(&sm.a[0][0][kofs(tid, 4 * c)]) = ah;
    *reinterpret_cast<float4*>(&sm.a[0][1][kofs(tid, 4 * c)]) = make_float4(a01.x, a01.y, a23.x, a23.y);
    *reinterpret_cast<float4*>(&sm.a[1][0][kofs(tid, 4 * c)]) = bh;
    *reinterpret_cast<float4*>(&sm.a[1][1][kofs(tid, 4 * c)]) = make_float4(b01.x, b01.y, b23.x, b23.y);
  }
  if (tid < kN) *reinterpret_cast<float4*>(&sm.bb[kofs(tid, 0)]) = split3(x);
}

__device__ __forceinline__ void mbar_wait(const uint64_t* bar, uint32_t phase) {
  // the retry loop in one asm block: no register re-materialisation per spin
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(su32(bar)),
      "r"(phase)
      : "memory");
}

// Barrier, then thread 0 issues the 8 MMAs of a step and commits them to
// sm.mbar.  Every thread's shared-memory reads and writes of the step so far
// are complete (and visible to the async proxy) when this returns.
__device__ __forceinline__ void gates_issue(Smem& sm) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint64_t wh = desc(su32(sm.bw[0])), wl = desc(su32(sm.bw[1]));
    const uint64_t xb = desc(su32(sm.bb)), one = desc(su32(sm.a1), 0u);
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t d = sm.tmem + uint32_t(t * kN);
      const uint64_t ah = desc(su32(sm.a[t][0])), al = desc(su32(sm.a[t][1]));
      mma(d, one, xb, 0u);  // 1 . (xb_hi + xb_mid + xb_lo), exact
      mma(d, ah, wh, 1u);   // h_hi . W_hi
      mma(d, al, wh, 1u);   // h_lo . W_hi
      mma(d, ah, wl, 1u);   // h_hi . W_lo
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&sm.mbar))
                 : "memory");
  }
}

__device__ __forceinline__ void gates_wait(Smem& sm, uint32_t phase) {
  mbar_wait(&sm.mbar, phase);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Barrier, issue the 10 MMAs of a step (thread 0), wait for them.
__device__ __forceinline__ void gates_mma(Smem& sm, uint32_t phase) {
  gates_issue(sm);
  gates_wait(sm, phase);
}

// Scaled pre-activations (f, i, o, g) of units u, u+1 for the thread's pair.
__device__ __forceinline__ void read_units(const Smem& sm, int u, float2 (&pre)[2][4]) {
  const uint32_t lane = uint32_t((threadIdx.x >> 5) * 32) << 16;
  float a[8], b[8];
  ld8(sm.tmem + lane + uint32_t(4 * u), a);
  ld8(sm.tmem + lane + uint32_t(kN + 4 * u), b);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int g = 0; g < 4; ++g) pre[q][g] = make_float2(a[4 * q + g], b[4 * q + g]);
}

__device__ __forceinline__ void teardown(Smem& sm, uint32_t tmem_cols = 64) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(sm.tmem), "r"(tmem_cols));
}

__device__ __forceinline__ float2 ldg2(const float* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg2(float* p, float2 v) {
  asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

struct OutPtrs {
  float* p[ACKPT_MAX_FUSED];
};
struct StatePtrs {
  const float* p[ACKPT_MAX_FUSED];
};

// Launch chain (chain.cuh): one tile per CTA, so CTA b waits for and
// publishes tile b.
using Chain = chain::Chain;
using chain::ldcg2;
__device__ __forceinline__ void chain_begin(const Chain& ch) {
  if (!ch.flags) return;
  __syncthreads();  // TMEM allocated (setup): dependents may be scheduled now
  chain::allow_dependents(ch);
  chain::wait_tile(ch, blockIdx.x, 0);
}
__device__ __forceinline__ void chain_end(const Chain& ch) { chain::set_tile(ch, blockIdx.x, 0); }

// Fused forward over `count` steps from `from`; TAPE stores every step's
// output to outs.p[i], otherwise only the final state goes to `out`.
template <bool TAPE>
__global__ void __launch_bounds__(kThreads, 8)
    fwd_tc(const float* __restrict__ in, float* __restrict__ out, int64_t B, const float* __restrict__ xbs_all,
           int64_t from, int count, const __grid_constant__ Weights w, const __grid_constant__ OutPtrs outs,
           Chain chain) {
  __shared__ __align__(128) Smem sm;
  const int64_t b0 = int64_t(blockIdx.x) * kTile + 2 * threadIdx.x;
  const bool live = b0 < B;  // every thread takes part in the MMA protocol
  setup(sm, w);
  chain_begin(chain);
  float2 h[kD], c[kD];
#pragma unroll
  for (int j = 0; j < kD; ++j) {
    h[j] = live ? ldcg2(in + b0 + int64_t(j) * B) : make_float2(0.f, 0.f);
    c[j] = live ? ldcg2(in + b0 + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
  }
  float xb = load_bias(xbs_all, from);
  for (int i = 0; i < count; ++i) {
    stage_operands(sm, h, xb);
    if (i + 1 < count) xb = load_bias(xbs_all, from + i + 1);
    gates_mma(sm, uint32_t(i & 1));
#pragma unroll
    for (int u = 0; u < kD; u += 2) {
      float2 pre[2][4];
      read_units(sm, u, pre);
      fwd_units2_nr(pre[0], pre[1], c[u], c[u + 1], h[u], h[u + 1]);
    }
    if (TAPE && live) {
      float* dst = outs.p[i] + b0;
#pragma unroll
      for (int j = 0; j < kD; ++j) {
        stg2(dst + int64_t(j) * B, h[j]);
        stg2(dst + int64_t(kD + j) * B, c[j]);
      }
    }
  }
  if (!TAPE && live) {
#pragma unroll
    for (int j = 0; j < kD; ++j) {
      stg2(out + b0 + int64_t(j) * B, h[j]);
      stg2(out + b0 + int64_t(kD + j) * B, c[j]);
    }
  }
  chain_end(chain);
  teardown(sm);
}

// Reverse-run shared memory: the gate operands plus one staging buffer for
// the taped state of the next step (16 rows of the CTA's 256 elements).
struct RevSmem {
  Smem g;
  float st[2 * kD][kTile];
  uint64_t mbar_st;
};

// Thread 0: the CTA's 16 row segments of `state` into sm.st with
// cp.async.bulk, completing on sm.mbar_st.
template <class RS>
__device__ __forceinline__ void stage_state(RS& sm, const float* state, int64_t B, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&sm.mbar_st)),
               "r"(bytes * uint32_t(2 * kD))
               : "memory");
  const float* src = state + int64_t(blockIdx.x) * kTile;
#pragma unroll
  for (int j = 0; j < 2 * kD; ++j)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm.st[j])),
                 "l"(src + int64_t(j) * B), "r"(bytes), "r"(su32(&sm.mbar_st))
                 : "memory");
}

// Lane 0 of every warp: 4 of the 16 row segments (warp w: rows 4w .. 4w+3),
// thread 0 also the barrier's expected bytes -- the copies of a step are
// issued by four threads at once instead of one (a complete_tx that lands
// before the expect_tx only drives the transaction count negative; the
// phase cannot complete before thread 0's arrival).
template <class RS>
__device__ __forceinline__ void stage_state_split(RS& sm, const float* state, int64_t B, uint32_t bytes) {
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&sm.mbar_st)),
                 "r"(bytes * uint32_t(2 * kD))
                 : "memory");
  const int w = threadIdx.x >> 5;
  const float* src = state + int64_t(blockIdx.x) * kTile;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int j = 4 * w + q;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm.st[j])),
                 "l"(src + int64_t(j) * B), "r"(bytes), "r"(su32(&sm.mbar_st))
                 : "memory");
  }
}

// Fused run of Reverse actions, steps from+count-1 .. from.  Gates on the
// tensor cores; the transpose matvec dh = sum_g (s_g W_g)^T (da_g / s_g) on
// the packed-fp32 pipe with uniform-register weights.  PF (B % 4 == 0, 16-byte
// aligned states): the taped state of step i-1 streams into shared memory by
// cp.async.bulk while step i computes, instead of a dependent load at the top
// of every step.
//
// 6 CTAs/SM (80 registers, ~36 KB of shared memory with the broadcast bias
// operand): 27.5 us/step at the C2 shape vs 27.9 at 5 CTAs (96 registers)
// and 29.6 at 7 (72 registers, 148 B of spills).  Deferring the last units'
// transposed-product FMAs past the next step's MMA issue (to cover the MMA
// round trip) measured 28.1 / 30.3 us (2 / 4 units): the per-step wait is
// the CTA barrier's warp skew, not the MMA latency (ncu source page:
// barrier 17 %, mbarrier long-scoreboard 5 % of warp samples).
#ifndef ACKPT_REV_MINB
#define ACKPT_REV_MINB 6
#endif

__device__ __forceinline__ void tmatvec_unit(const Weights& w, int j, const float2 (&da)[4], float2 (&acc)[kD]) {
#pragma unroll
  for (int m = 0; m < kD; ++m) {
    acc[m] = fma2(bc(w.wu[0][j][m]), da[0], acc[m]);
    acc[m] = fma2(bc(w.wu[1][j][m]), da[1], acc[m]);
    acc[m] = fma2(bc(w.wu[2][j][m]), da[2], acc[m]);
    acc[m] = fma2(bc(w.wu[3][j][m]), da[3], acc[m]);
  }
}

template <bool PF>
__global__ void __launch_bounds__(kThreads, ACKPT_REV_MINB)
    rev_tc(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B, const float* __restrict__ xbs_all,
           int64_t from, int count, const __grid_constant__ Weights w, const __grid_constant__ StatePtrs states,
           Chain chain) {
  __shared__ __align__(128) RevSmem rs;
  Smem& sm = rs.g;
  const int64_t b0 = int64_t(blockIdx.x) * kTile + 2 * threadIdx.x;
  const bool live = b0 < B;
  const int64_t rem = B - int64_t(blockIdx.x) * kTile;
  const uint32_t seg = uint32_t(rem < kTile ? rem : kTile) * 4u;
  setup(sm, w);
  chain_begin(chain);
  if (PF) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rs.mbar_st)));
      asm volatile("fence.mbarrier_init.release.cluster;");
      stage_state(rs, states.p[count - 1], B, seg);
    }
    __syncthreads();
  }
  float2 dh[kD], dc[kD];
#pragma unroll
  for (int j = 0; j < kD; ++j) {
    dh[j] = live ? ldcg2(adj_in + b0 + int64_t(j) * B) : make_float2(0.f, 0.f);
    dc[j] = live ? ldcg2(adj_in + b0 + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
  }
  int phase = 0;
  float xb = load_bias(xbs_all, from + count - 1);
  for (int i = count - 1; i >= 0; --i, ++phase) {
    float2 h[kD], c[kD];
    if (PF) {
      mbar_wait(&rs.mbar_st, uint32_t(phase & 1));
#pragma unroll
      for (int j = 0; j < kD; ++j) {
        h[j] = *reinterpret_cast<const float2*>(&rs.st[j][2 * threadIdx.x]);
        c[j] = *reinterpret_cast<const float2*>(&rs.st[kD + j][2 * threadIdx.x]);
      }
    } else {
      const float* xs = states.p[i] + b0;
#pragma unroll
      for (int j = 0; j < kD; ++j) {
        h[j] = live ? ldcg2(xs + int64_t(j) * B) : make_float2(0.f, 0.f);
        c[j] = live ? ldcg2(xs + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
      }
    }
    stage_operands(sm, h, xb);
    if (i > 0) xb = load_bias(xbs_all, from + i - 1);
    gates_issue(sm);  // after its barrier every thread has read rs.st
    if (PF && i > 0 && (threadIdx.x & 31) == 0) stage_state_split(rs, states.p[i - 1], B, seg);
    gates_wait(sm, uint32_t(phase & 1));
    float2 acc[kD];
#pragma unroll
    for (int m = 0; m < kD; ++m) acc[m] = bc(0.0f);
#pragma unroll
    for (int u = 0; u < kD; u += 2) {
      float2 pre[2][4];
      read_units(sm, u, pre);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int j = u + q;
        float2 da[4];
        bwd_unit_u(pre[q][0], pre[q][1], pre[q][2], pre[q][3], c[j], dh[j], dc[j], da[0], da[1], da[2], da[3], dc[j]);
        tmatvec_unit(w, j, da, acc);
      }
    }
#pragma unroll
    for (int m = 0; m < kD; ++m) dh[m] = acc[m];
  }
  if (live) {
#pragma unroll
    for (int j = 0; j < kD; ++j) {
      stg2(adj_out + b0 + int64_t(j) * B, dh[j]);
      stg2(adj_out + b0 + int64_t(kD + j) * B, dc[j]);
    }
  }
  chain_end(chain);
  teardown(sm);
}

}  // namespace tc
}  // namespace ackpt
