// Tensor-core (tcgen05) fused LSTM kernels for sm_100a, hidden size 8:
// fused Advance, fused TapeForward and fused Reverse runs.  Same results
// contract as lstm_f32.cuh (fp32 state, rel-L2 <= 1e-5 vs float64), different
// arithmetic for the gate matvec, so NOT bit-identical to the FFMA2 kernels:
// an execution uses one family for every step.
//
// Gate pre-activations of a step, for the 256 batch elements of a CTA, are one
// MMA problem per M-tile: D[128 x 32] = A[128 x 16] . B[32 x 16]^T with
//   A row r = [h_0..h_7, 1, 0 x 7]                    (element of the tile)
//   B row n = [s_g W_g[j][0..7], s_g xb_k[g][j], 0 x 7]  n = 4 j + g (unit-major)
// (s_g: the exponent scale folded into the weights, lstm_f32_math.cuh), so the
// bias / input projection of step k rides in the MMA and D holds the ex2
// arguments directly.  fp32 accuracy from TF32 tensor cores with the 3xTF32
// split x = hi + lo (hi = x with the low 13 mantissa bits cleared):
// A.B ~ Ahi.Bhi + Alo.Bhi + Ahi.Blo (rel. error ~5e-7, tools/umma_probe.cu).
// Operands are K-major, no swizzle, in shared memory; D (fp32) is in TMEM,
// one column per gate, one lane per tile row, read back with tcgen05.ld.
//
// CTA = 128 threads = the 128 TMEM lanes.  Tile 0 row r is element base+2r,
// tile 1 row r is element base+2r+1, so thread r owns the float2 pair at
// base+2r in global memory and processes it with the packed-fp32 math.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

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

// 24 KB: h operands per tile (hi, lo), one constant bias operand A1 = [1, 0 x 7]
// shared by both tiles, the weights (hi, lo) and the step's bias column (hi, lo).
struct Smem {
  float a[2][2][128 * kK];  // [tile][hi, lo]
  float a1[128 * kK];       // rows [1, 0, ..., 0]
  float bw[2][kN * kK];     // [hi, lo] scaled W rows n = 4 j + g
  float bb[2][kN * kK];     // [hi, lo] column 0 = scaled xb_k, rest 0
  uint64_t mbar;
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((kLBO >> 4) & 0x3FFF) << 16) |
         (uint64_t((kSBO >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
// float offset of (row, k) in a K-major no-swizzle 16-wide operand
__device__ __forceinline__ int kofs(int r, int k) { return (r >> 3) * (kSBO / 4) + (k >> 2) * (kLBO / 4) + (r & 7) * 4 + (k & 3); }
__device__ __forceinline__ float hi_part(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

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
  // bias operand row of this thread: [1, 0, ..., 0]
  *reinterpret_cast<float4*>(&sm.a1[kofs(tid, 0)]) = make_float4(1.f, 0.f, 0.f, 0.f);
  *reinterpret_cast<float4*>(&sm.a1[kofs(tid, 4)]) = make_float4(0.f, 0.f, 0.f, 0.f);
  // weight rows n = 4 j + g (scaled, split), bias rows zero but for column 0 (per step)
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
  if (tid < kN) {
    sm.bb[0][kofs(tid, 0)] = hi_part(x);
    sm.bb[1][kofs(tid, 0)] = x - hi_part(x);
  }
}

__device__ __forceinline__ void mbar_wait(const uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

// Barrier, then thread 0 issues the 10 MMAs of a step and commits them to
// sm.mbar.  Every thread's shared-memory reads and writes of the step so far
// are complete (and visible to the async proxy) when this returns.
__device__ __forceinline__ void gates_issue(Smem& sm) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint64_t wh = desc(su32(sm.bw[0])), wl = desc(su32(sm.bw[1]));
    const uint64_t xh = desc(su32(sm.bb[0])), xl = desc(su32(sm.bb[1])), one = desc(su32(sm.a1));
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t d = sm.tmem + uint32_t(t * kN);
      const uint64_t ah = desc(su32(sm.a[t][0])), al = desc(su32(sm.a[t][1]));
      mma(d, ah, wh, 0u);   // h_hi . W_hi
      mma(d, al, wh, 1u);   // h_lo . W_hi
      mma(d, ah, wl, 1u);   // h_hi . W_lo
      mma(d, one, xh, 1u);  // 1 . xb_hi
      mma(d, one, xl, 1u);  // 1 . xb_lo
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

// Fused forward over `count` steps from `from`; TAPE stores every step's
// output to outs.p[i], otherwise only the final state goes to `out`.
template <bool TAPE>
__global__ void __launch_bounds__(kThreads, 8)
    fwd_tc(const float* __restrict__ in, float* __restrict__ out, int64_t B, const float* __restrict__ xbs_all,
           int64_t from, int count, const __grid_constant__ Weights w, const __grid_constant__ OutPtrs outs) {
  __shared__ __align__(128) Smem sm;
  const int64_t b0 = int64_t(blockIdx.x) * kTile + 2 * threadIdx.x;
  const bool live = b0 < B;  // every thread takes part in the MMA protocol
  setup(sm, w);
  float2 h[kD], c[kD];
#pragma unroll
  for (int j = 0; j < kD; ++j) {
    h[j] = live ? ldg2(in + b0 + int64_t(j) * B) : make_float2(0.f, 0.f);
    c[j] = live ? ldg2(in + b0 + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
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
#pragma unroll
      for (int q = 0; q < 2; ++q) h[u + q] = fwd_unit_nr(pre[q][0], pre[q][1], pre[q][2], pre[q][3], c[u + q]);
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
#pragma unroll 1
  for (int j = 0; j < 2 * kD; ++j)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm.st[j])),
                 "l"(src + int64_t(j) * B), "r"(bytes), "r"(su32(&sm.mbar_st))
                 : "memory");
}

// Fused run of Reverse actions, steps from+count-1 .. from.  Gates on the
// tensor cores; the transpose matvec dh = sum_g (s_g W_g)^T (da_g / s_g) on
// the packed-fp32 pipe with uniform-register weights.  PF (B % 4 == 0, 16-byte
// aligned states): the taped state of step i-1 streams into shared memory by
// cp.async.bulk while step i computes, instead of a dependent load at the top
// of every step.
template <bool PF>
__global__ void __launch_bounds__(kThreads, 5)  // 96 registers, 5 CTAs/SM: 28.3 vs 30.2 us/step at 4
    rev_tc(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B, const float* __restrict__ xbs_all,
           int64_t from, int count, const __grid_constant__ Weights w, const __grid_constant__ StatePtrs states) {
  __shared__ __align__(128) RevSmem rs;
  Smem& sm = rs.g;
  const int64_t b0 = int64_t(blockIdx.x) * kTile + 2 * threadIdx.x;
  const bool live = b0 < B;
  const int64_t rem = B - int64_t(blockIdx.x) * kTile;
  const uint32_t seg = uint32_t(rem < kTile ? rem : kTile) * 4u;
  setup(sm, w);
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
    dh[j] = live ? ldg2(adj_in + b0 + int64_t(j) * B) : make_float2(0.f, 0.f);
    dc[j] = live ? ldg2(adj_in + b0 + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
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
        h[j] = live ? ldg2(xs + int64_t(j) * B) : make_float2(0.f, 0.f);
        c[j] = live ? ldg2(xs + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
      }
    }
    stage_operands(sm, h, xb);
    if (i > 0) xb = load_bias(xbs_all, from + i - 1);
    gates_issue(sm);  // after its barrier every thread has read rs.st
    if (PF && i > 0 && threadIdx.x == 0) stage_state(rs, states.p[i - 1], B, seg);
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
        float2 daf, dai, dao, dag;
        bwd_unit_u(pre[q][0], pre[q][1], pre[q][2], pre[q][3], c[j], dh[j], dc[j], daf, dai, dao, dag, dc[j]);
#pragma unroll
        for (int m = 0; m < kD; ++m) {
          acc[m] = fma2(bc(w.wu[0][j][m]), daf, acc[m]);
          acc[m] = fma2(bc(w.wu[1][j][m]), dai, acc[m]);
          acc[m] = fma2(bc(w.wu[2][j][m]), dao, acc[m]);
          acc[m] = fma2(bc(w.wu[3][j][m]), dag, acc[m]);
        }
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
  teardown(sm);
}

// ---- software-pipelined reverse (ACKPT_TC_REV=sp) ----------------------------
// The gates of step i-1 depend only on the taped state, not on the adjoint,
// so their MMAs are issued before the epilogue of step i and run underneath
// it: the accumulator is double-buffered in TMEM (columns [0, 64) and
// [64, 128)), one barrier per step, the MMA round trip off the critical path.
__device__ __forceinline__ void read_units_at(const Smem& sm, uint32_t col0, int u, float2 (&pre)[2][4]) {
  const uint32_t lane = uint32_t((threadIdx.x >> 5) * 32) << 16;
  float a[8], b[8];
  ld8(sm.tmem + lane + col0 + uint32_t(4 * u), a);
  ld8(sm.tmem + lane + col0 + uint32_t(kN + 4 * u), b);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int g = 0; g < 4; ++g) pre[q][g] = make_float2(a[4 * q + g], b[4 * q + g]);
}

// Barrier (A and bias staged by every thread), then thread 0 issues the gate
// MMAs into columns col0 and commits them to sm.mbar.
__device__ __forceinline__ void gates_issue_at(Smem& sm, uint32_t col0) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint64_t wh = desc(su32(sm.bw[0])), wl = desc(su32(sm.bw[1]));
    const uint64_t xh = desc(su32(sm.bb[0])), xl = desc(su32(sm.bb[1])), one = desc(su32(sm.a1));
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const uint32_t d = sm.tmem + col0 + uint32_t(t * kN);
      const uint64_t ah = desc(su32(sm.a[t][0])), al = desc(su32(sm.a[t][1]));
      mma(d, ah, wh, 0u);
      mma(d, al, wh, 1u);
      mma(d, ah, wl, 1u);
      mma(d, one, xh, 1u);
      mma(d, one, xl, 1u);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&sm.mbar))
                 : "memory");
  }
}

__global__ void __launch_bounds__(kThreads, 4)
    rev_tcs(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B, const float* __restrict__ xbs_all,
            int64_t from, int count, const __grid_constant__ Weights w, const __grid_constant__ StatePtrs states) {
  __shared__ __align__(128) RevSmem rs;
  Smem& sm = rs.g;
  const int64_t b0 = int64_t(blockIdx.x) * kTile + 2 * threadIdx.x;
  const bool live = b0 < B;
  const int64_t rem = B - int64_t(blockIdx.x) * kTile;
  const uint32_t seg = uint32_t(rem < kTile ? rem : kTile) * 4u;
  setup(sm, w, 128);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rs.mbar_st)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stage_state(rs, states.p[count - 1], B, seg);
  }
  __syncthreads();
  float2 dh[kD], dc[kD], c[kD];
#pragma unroll
  for (int j = 0; j < kD; ++j) {
    dh[j] = live ? ldg2(adj_in + b0 + int64_t(j) * B) : make_float2(0.f, 0.f);
    dc[j] = live ? ldg2(adj_in + b0 + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
  }
  // prologue: gates of the last step
  uint32_t st_phase = 0;
  {
    mbar_wait(&rs.mbar_st, st_phase);
    st_phase ^= 1u;
    float2 h[kD];
#pragma unroll
    for (int j = 0; j < kD; ++j) {
      h[j] = *reinterpret_cast<const float2*>(&rs.st[j][2 * threadIdx.x]);
      c[j] = *reinterpret_cast<const float2*>(&rs.st[kD + j][2 * threadIdx.x]);
    }
    stage_operands(sm, h, load_bias(xbs_all, from + count - 1));
    gates_issue_at(sm, 0);  // every thread has read rs.st
    if (count > 1 && threadIdx.x == 0) stage_state(rs, states.p[count - 2], B, seg);
  }
  uint32_t g_phase = 0;
  float xb = count > 1 ? load_bias(xbs_all, from + count - 2) : 0.f;
  for (int i = count - 1; i >= 0; --i) {
    const uint32_t cur = uint32_t((count - 1 - i) & 1) * 64u;
    mbar_wait(&sm.mbar, g_phase);  // gates of step i are in TMEM
    g_phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float2 cn[kD];
    if (i > 0) {  // stage step i-1 and start its gate MMAs under this step's epilogue
      mbar_wait(&rs.mbar_st, st_phase);
      st_phase ^= 1u;
      float2 h[kD];
#pragma unroll
      for (int j = 0; j < kD; ++j) {
        h[j] = *reinterpret_cast<const float2*>(&rs.st[j][2 * threadIdx.x]);
        cn[j] = *reinterpret_cast<const float2*>(&rs.st[kD + j][2 * threadIdx.x]);
      }
      stage_operands(sm, h, xb);
      if (i > 1) xb = load_bias(xbs_all, from + i - 2);
      gates_issue_at(sm, 64u - cur);
      if (i > 1 && threadIdx.x == 0) stage_state(rs, states.p[i - 2], B, seg);
    }
    float2 acc[kD];
#pragma unroll
    for (int m = 0; m < kD; ++m) acc[m] = bc(0.0f);
#pragma unroll
    for (int u = 0; u < kD; u += 2) {
      float2 pre[2][4];
      read_units_at(sm, cur, u, pre);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int j = u + q;
        float2 daf, dai, dao, dag;
        bwd_unit_u(pre[q][0], pre[q][1], pre[q][2], pre[q][3], c[j], dh[j], dc[j], daf, dai, dao, dag, dc[j]);
#pragma unroll
        for (int m = 0; m < kD; ++m) {
          acc[m] = fma2(bc(w.wu[0][j][m]), daf, acc[m]);
          acc[m] = fma2(bc(w.wu[1][j][m]), dai, acc[m]);
          acc[m] = fma2(bc(w.wu[2][j][m]), dao, acc[m]);
          acc[m] = fma2(bc(w.wu[3][j][m]), dag, acc[m]);
        }
      }
    }
#pragma unroll
    for (int m = 0; m < kD; ++m) {
      dh[m] = acc[m];
      c[m] = cn[m];
    }
  }
  if (live) {
#pragma unroll
    for (int j = 0; j < kD; ++j) {
      stg2(adj_out + b0 + int64_t(j) * B, dh[j]);
      stg2(adj_out + b0 + int64_t(kD + j) * B, dc[j]);
    }
  }
  teardown(sm, 128);
}

// ---- reverse run with both matvecs on the tensor cores ---------------------
// Step i: gates G = [h 1] . [W xb]^T as in rev_tc (MMA1, 3xTF32, TMEM cols
// [0, 64)); each thread turns its rows' pre-activations into the scaled gate
// adjoints da (bwd_unit) and writes them back into TMEM as the A operand of
// the transposed matvec dh = da . B2^T, B2[m][4 j + g] = s_g W_g[j][m]:
//   da_hi (tf32 bits) over G in place, da_lo = da - da_hi as packed bf16
//   (even k in the low half) in cols [64, 96);
//   MMA2: da_hi x B2_hi + da_hi x B2_lo (kind::tf32, 4 K-steps) + da_lo x B2
//   (kind::f16, bf16, 2 K-steps) -> D2 (fp32) in cols [96, 128), 16 per tile.
// da_lo carries <= 2^-11 |da| and its bf16 rounding adds <= 2^-20 |da|, the
// order of the 3xTF32 split's own dropped term (tools/umma_ts_probe.cu:
// rel. error 9.4e-7 vs 6.5e-7 for 3xTF32).  128 TMEM columns per CTA.
constexpr uint32_t kN2 = 16;                   // MMA2 N (m = 0..7 real, 8..15 zero)
constexpr uint32_t kLBO2 = 256, kSBO2 = 128;   // B2: K chunks of 16 B, 2 row groups each
constexpr uint32_t kIdescT2 = (1u << 4) | (2u << 7) | (2u << 10) | ((kN2 >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescB2 = (1u << 4) | (1u << 7) | (1u << 10) | ((kN2 >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kColLo = 64, kColD2 = 96, kCols2 = 128;

struct Rev2Smem {
  Smem g;
  float st[2 * kD][kTile];                  // prefetched taped state
  unsigned char b2h[kN2 * kN * 4];          // tf32 hi, K-major, (k/4)*LBO + (r/8)*SBO + (r%8)*16 + (k%4)*4
  unsigned char b2l[kN2 * kN * 4];          // tf32 lo
  unsigned char b2b[kN2 * kN * 2];          // bf16, (k/8)*LBO + (r/8)*SBO + (r%8)*16 + (k%8)*2
  uint64_t mbar_st, mbar2;
};

__device__ __forceinline__ uint64_t desc2(uint32_t addr) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((kLBO2 >> 4) & 0x3FFF) << 16) |
         (uint64_t((kSBO2 >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc,
                                       bool f16) {
  if (f16)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ uint32_t bf16x2(float even, float odd) {  // even k -> low half
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(odd), "f"(even));
  return r;
}
__device__ __forceinline__ void st8(uint32_t addr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void st4(uint32_t addr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}

// B2 (constant): rows m < 8 = scaled W columns, rows 8..15 zero.
__device__ __forceinline__ void setup_b2(Rev2Smem& rs, const Weights& w) {
  for (int i = threadIdx.x; i < int(kN2) * kN; i += kThreads) {
    const int m = i / kN, k = i % kN, j = k >> 2, g = k & 3;
    const float x = m < kD ? w.ws[g][j][m] : 0.f;
    const int o32 = (k / 4) * kLBO2 + (m / 8) * kSBO2 + (m % 8) * 16 + (k % 4) * 4;
    const int o16 = (k / 8) * kLBO2 + (m / 8) * kSBO2 + (m % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<float*>(rs.b2h + o32) = hi_part(x);
    *reinterpret_cast<float*>(rs.b2l + o32) = x - hi_part(x);
    *reinterpret_cast<__nv_bfloat16*>(rs.b2b + o16) = __float2bfloat16_rn(x);
  }
}

// Gate adjoints of unit pair (u, u+1) -> TMEM A operand of both tiles.
__device__ __forceinline__ void store_da(uint32_t tmem_lane, int u, const float2 (&v)[8]) {
  float2 hi[8], lo[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    hi[q] = make_float2(hi_part(v[q].x), hi_part(v[q].y));
    lo[q] = sub2(v[q], hi[q]);
  }
  uint32_t h0[8], h1[8], l0[4], l1[4];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    h0[q] = __float_as_uint(hi[q].x);
    h1[q] = __float_as_uint(hi[q].y);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    l0[q] = bf16x2(lo[2 * q].x, lo[2 * q + 1].x);
    l1[q] = bf16x2(lo[2 * q].y, lo[2 * q + 1].y);
  }
  st8(tmem_lane + uint32_t(4 * u), h0);
  st8(tmem_lane + uint32_t(kN + 4 * u), h1);
  st4(tmem_lane + kColLo + uint32_t(2 * u), l0);
  st4(tmem_lane + kColLo + kN2 + uint32_t(2 * u), l1);
}

// Fused run of Reverse actions, both matvecs on the tensor cores (PF: taped
// state streamed into shared memory one step ahead, as in rev_tc<true>).
template <bool NR>
__global__ void __launch_bounds__(kThreads, 4)
    rev_tc2(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B,
            const float* __restrict__ xbs_all, int64_t from, int count, const __grid_constant__ Weights w,
            const __grid_constant__ StatePtrs states) {
  __shared__ __align__(128) Rev2Smem rs;
  Smem& sm = rs.g;
  const int64_t b0 = int64_t(blockIdx.x) * kTile + 2 * threadIdx.x;
  const bool live = b0 < B;
  const int64_t rem = B - int64_t(blockIdx.x) * kTile;
  const uint32_t seg = uint32_t(rem < kTile ? rem : kTile) * 4u;
  setup(sm, w, kCols2);
  setup_b2(rs, w);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rs.mbar_st)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&rs.mbar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stage_state(rs, states.p[count - 1], B, seg);
  }
  __syncthreads();
  const uint32_t lane = uint32_t((threadIdx.x >> 5) * 32) << 16;
  float2 dh[kD], dc[kD];
#pragma unroll
  for (int j = 0; j < kD; ++j) {
    dh[j] = live ? ldg2(adj_in + b0 + int64_t(j) * B) : make_float2(0.f, 0.f);
    dc[j] = live ? ldg2(adj_in + b0 + int64_t(kD + j) * B) : make_float2(0.f, 0.f);
  }
  int phase = 0;
  float xb = load_bias(xbs_all, from + count - 1);
  for (int i = count - 1; i >= 0; --i, ++phase) {
    float2 h[kD], c[kD];
    mbar_wait(&rs.mbar_st, uint32_t(phase & 1));
#pragma unroll
    for (int j = 0; j < kD; ++j) {
      h[j] = *reinterpret_cast<const float2*>(&rs.st[j][2 * threadIdx.x]);
      c[j] = *reinterpret_cast<const float2*>(&rs.st[kD + j][2 * threadIdx.x]);
    }
    stage_operands(sm, h, xb);
    if (i > 0) xb = load_bias(xbs_all, from + i - 1);
    gates_issue(sm);  // after its barrier every thread has read rs.st
    if (i > 0 && threadIdx.x == 0) stage_state(rs, states.p[i - 1], B, seg);
    gates_wait(sm, uint32_t(phase & 1));
#pragma unroll
    for (int u = 0; u < kD; u += 2) {
      float2 pre[2][4];
      read_units(sm, u, pre);
      float2 da[8];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int j = u + q;
        if (NR)
          bwd_unit_nr(pre[q][0], pre[q][1], pre[q][2], pre[q][3], c[j], dh[j], dc[j], da[4 * q], da[4 * q + 1],
                      da[4 * q + 2], da[4 * q + 3], dc[j]);
        else
          bwd_unit(pre[q][0], pre[q][1], pre[q][2], pre[q][3], c[j], dh[j], dc[j], da[4 * q], da[4 * q + 1],
                   da[4 * q + 2], da[4 * q + 3], dc[j]);
      }
      store_da(sm.tmem + lane, u, da);
    }
    // MMA2: dh = da . B2^T per tile
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const uint32_t d2 = sm.tmem + kColD2 + uint32_t(t) * kN2;
        const uint32_t ahi = sm.tmem + uint32_t(t * kN), alo = sm.tmem + kColLo + uint32_t(t) * kN2;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // tf32: K = 8 per MMA
          mma_ts(d2, ahi + 8 * ks, desc2(su32(rs.b2h) + ks * 2 * kLBO2), kIdescT2, ks ? 1u : 0u, false);
          mma_ts(d2, ahi + 8 * ks, desc2(su32(rs.b2l) + ks * 2 * kLBO2), kIdescT2, 1u, false);
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)  // bf16: K = 16 per MMA (8 packed columns)
          mma_ts(d2, alo + 8 * ks, desc2(su32(rs.b2b) + ks * 2 * kLBO2), kIdescB2, 1u, true);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32(&rs.mbar2))
                   : "memory");
    }
    mbar_wait(&rs.mbar2, uint32_t(phase & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    {
      float a[8], b[8];
      ld8(sm.tmem + lane + kColD2, a);
      ld8(sm.tmem + lane + kColD2 + kN2, b);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int m = 0; m < kD; ++m) dh[m] = make_float2(a[m], b[m]);
    }
  }
  if (live) {
#pragma unroll
    for (int j = 0; j < kD; ++j) {
      stg2(adj_out + b0 + int64_t(j) * B, dh[j]);
      stg2(adj_out + b0 + int64_t(kD + j) * B, dc[j]);
    }
  }
  teardown(sm, kCols2);
}

}  // namespace tc
}  // namespace ackpt
