// Tensor-core (tcgen05) LSTM kernels for larger hidden sizes, D in {16, 32},
// fp32 state: forward (one step, a fused Advance, or a TapeForward run) and
// reverse (one step or a fused Reverse run).  Same results contract as the
// other fp32 kernels (rel-L2 <= 1e-5 vs float64, lstm.py:114-152).
//
// CTA = 128 threads = one M=128 tile of sequences (thread r owns sequence
// b0 + r, the TMEM lane r); arithmetic is packed over unit pairs (j, j+1).
//   gates   G[128 x 4D] = h[128 x D] . W[4D x D]^T + 1 . xb^T, 3xTF32
//           (h_hi W_hi + h_lo W_hi + h_hi W_lo, bias as two K=8 MMAs against
//           a constant ones column), in TMEM.  Gate rows are permuted,
//           n = 8 p + 2 gate + e for unit j = 2 p + e, so one tcgen05.ld.x8
//           at column 8p returns (f, i, o, g) of units 2p, 2p+1 as float2s.
//   reverse da (the scaled gate adjoints of bwd_unit) go back into TMEM as
//           the A operand of dh[128 x D] = da[128 x 4D] . B2[D x 4D]^T with
//           B2[m][n] = s_gate W_gate[j(n)][m], 3xTF32 as well: da_hi over G in
//           place, da_lo of one K half at a time in [4D, 6D), dh in [6D, 7D)
//           (TMEM-A form validated in tools/umma_ts_probe.cu).  (A bf16 residual would save 2D columns
//           but costs ~2^-19 per product: 1.2e-5 rel-L2 after 100 steps at d=32.)
// Operands are K-major, no swizzle, 8-row groups of 16-byte core matrices
// (LBO 128 B between K chunks, SBO = 32 K bytes between row groups).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "chain.cuh"
#include "lstm_f32_math.cuh"

namespace ackpt {
namespace tcd {

using namespace f32m;

constexpr int kThreads = 128;

struct OutPtrs {
  float* p[ACKPT_MAX_FUSED];
};
struct StatePtrs {
  const float* p[ACKPT_MAX_FUSED];
};

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
         (uint64_t(1) << 46);
}
// tf32 head of x rounded to nearest, ties away from zero (|x - hi| <= 2^-11
// |x|; the tensor core truncates the residual to tf32, so each split product
// carries ~2^-22).  The same bits as cvt.rna.tf32.f32 for finite x, in two
// integer instructions (cvt.rna.tf32 compiles to four: it also handles NaN).
__device__ __forceinline__ float hi_part(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// float index of (row, k) in a tf32 operand with K-extent K; bf16 index likewise
template <int K>
__device__ __forceinline__ int kofs(int r, int k) {
  return (r >> 3) * (8 * K) + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}
template <int K>
__device__ __forceinline__ int kofs16(int r, int k) {
  return (r >> 3) * (8 * K) + (k >> 3) * 64 + (r & 7) * 8 + (k & 7);
}
template <int N>
__host__ __device__ constexpr uint32_t idesc(bool bf16) {
  return (1u << 4) | ((bf16 ? 1u : 2u) << 7) | ((bf16 ? 1u : 2u) << 10) | (uint32_t(N >> 3) << 17) |
         (uint32_t(128 >> 4) << 24);
}
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
  asm volatile(  // the retry loop in one asm block: no register re-materialisation per spin
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(su32(bar)),
      "r"(phase)
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// Barrier that publishes this step's shared-memory / TMEM writes to the
// tensor core (issued by thread 0 afterwards).
__device__ __forceinline__ void publish() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
}
__device__ __forceinline__ void ld8(uint32_t addr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
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
__device__ __forceinline__ uint32_t bf16x2(float even, float odd) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(odd), "f"(even));
  return r;
}
__host__ __device__ constexpr int tmem_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

// Shared-memory carve-up (dynamic).  Forward: A (h hi/lo), ones, W hi/lo,
// bias hi/lo.  Reverse adds B2 hi/lo (tf32).
template <int D>
struct Layout {
  // ones: one 8-row group [1, 1, 1, 0 x 5] read with stride-byte-offset 0
  // (broadcast to all 16 row groups); bias: row n = split3(scaled xb) exactly
  static constexpr int kA = 128 * D, kOne = 8 * 8, kW = 4 * D * D, kBias = 4 * D * 8, kW2 = 4 * D * D;
  static constexpr int a_hi = 0, a_lo = a_hi + kA, one = a_lo + kA, w_hi = one + kOne, w_lo = w_hi + kW,
                       b_hi = w_lo + kW, fwd_end = b_hi + kBias;
  static constexpr int w2_hi = fwd_end, w2_lo = w2_hi + kW2, rev_end = w2_lo + kW2;
  static constexpr size_t fwd_bytes = size_t(fwd_end) * 4 + 64, rev_bytes = size_t(rev_end) * 4 + 64;
};

// TMEM base address written by tcgen05.alloc: visible to every thread only
// after before_thread_sync / barrier / after_thread_sync.
__device__ __forceinline__ uint32_t tmem_base(const uint32_t* slot) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  return *reinterpret_cast<const volatile uint32_t*>(slot);
}

// gate row n -> (gate, unit)
__device__ __forceinline__ void gate_of(int n, int& gi, int& j) {
  gi = (n & 7) >> 1;
  j = 2 * (n >> 3) + (n & 1);
}

// Shared-memory image of the split weights, built once per cell
// (w_image<D>): [W hi | W lo] in the gate operand's layout (rows n = gate
// rows, K-major, kofs<D>), then [B2 hi | B2 lo] (B2[m][n] = s_gate W_gate[j(n)][m],
// the reverse's transposed-product operand, kofs<4D>).  The kernels copy it
// in with cp.async.bulk instead of gathering and splitting W per CTA (the
// per-step launches spent ~20 % of their stall samples there).
template <int D>
__global__ void w_image(const float* __restrict__ ws, float* __restrict__ img) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 4 * D * D; idx += gridDim.x * blockDim.x) {
    {
      const int n = idx / D, k = idx % D;  // gate operand row n, column k
      int gi, j;
      gate_of(n, gi, j);
      const float x = ws[(gi * D + j) * D + k];
      img[kofs<D>(n, k)] = hi_part(x);
      img[4 * D * D + kofs<D>(n, k)] = x - hi_part(x);
    }
    {
      const int m = idx / (4 * D), n = idx % (4 * D);  // B2 row m, column n
      int gi, j;
      gate_of(n, gi, j);
      const float x = ws[(gi * D + j) * D + m];
      img[8 * D * D + kofs<4 * D>(m, n)] = hi_part(x);
      img[12 * D * D + kofs<4 * D>(m, n)] = x - hi_part(x);
    }
  }
}

// Thread 0: `floats` floats of the image into shared memory by
// cp.async.bulk (pieces of <= 32 KB), completing on `bar`, whose expected
// transaction bytes were set beforehand (expect_bytes, once per phase).
__device__ __forceinline__ void expect_bytes(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_in(float* dst, const float* src, int floats, uint64_t* bar) {
  for (int off = 0; off < floats; off += 8192) {
    const uint32_t bytes = uint32_t(min(8192, floats - off)) * 4u;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst + off)),
                 "l"(src + off), "r"(bytes), "r"(su32(bar))
                 : "memory");
  }
}

// One-time setup shared by both kernels: TMEM, barriers, ones, zero bias
// rows, and the weight image (W, plus B2 for the reverse) in flight on
// bars[nbars] -- thread 0 waits for it before its first MMA (weights_ready).
template <int D>
__device__ __forceinline__ void setup(float* sm, uint64_t* bars, uint32_t* tslot, const float* __restrict__ wimg,
                                      int cols, int nbars, bool rev) {
  using L = Layout<D>;
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i <= nbars; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    expect_bytes(bars + nbars, uint32_t((rev ? 16 : 8) * D * D * 4));
    bulk_in(sm + L::w_hi, wimg, 8 * D * D, bars + nbars);
    if (rev) bulk_in(sm + L::w2_hi, wimg + 8 * D * D, 8 * D * D, bars + nbars);
  }
  if (tid < 8) {
    *reinterpret_cast<float4*>(sm + L::one + kofs<8>(tid, 0)) = make_float4(1.f, 1.f, 1.f, 0.f);
    *reinterpret_cast<float4*>(sm + L::one + kofs<8>(tid, 4)) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int idx = tid; idx < 4 * D * 8; idx += kThreads) {
    const int n = idx / 8, k = idx % 8;
    sm[L::b_hi + kofs<8>(n, k)] = 0.f;
  }
}

// Thread 0, before its first MMA: the weight image has landed.
__device__ __forceinline__ void weights_ready(uint64_t* wbar, bool& ready) {
  if (!ready) {
    wait_bar(wbar, 0);
    ready = true;
  }
}

// Stage A (this thread's row = its h, hi/lo) and the step's bias column.
template <int D>
__device__ __forceinline__ void stage(float* sm, const float2 (&h)[D / 2], const float* __restrict__ xbs_k) {
  using L = Layout<D>;
  const int tid = threadIdx.x;
#pragma unroll
  for (int c = 0; c < D / 4; ++c) {
    const float4 x = make_float4(h[2 * c].x, h[2 * c].y, h[2 * c + 1].x, h[2 * c + 1].y);
    const float4 hx = make_float4(hi_part(x.x), hi_part(x.y), hi_part(x.z), hi_part(x.w));
    const float2 l01 = sub2(make_float2(x.x, x.y), make_float2(hx.x, hx.y));
    const float2 l23 = sub2(make_float2(x.z, x.w), make_float2(hx.z, hx.w));
    *reinterpret_cast<float4*>(sm + L::a_hi + kofs<D>(tid, 4 * c)) = hx;
    *reinterpret_cast<float4*>(sm + L::a_lo + kofs<D>(tid, 4 * c)) = make_float4(l01.x, l01.y, l23.x, l23.y);
  }
  for (int n = tid; n < 4 * D; n += kThreads) {
    int gi, j;
    gate_of(n, gi, j);
    const float x = __ldg(xbs_k + gi * D + j);  // table is gate-major
    const float hi = hi_part(x), r = x - hi, mid = hi_part(r);  // x = hi + mid + lo exactly (tf32 parts)
    *reinterpret_cast<float4*>(sm + L::b_hi + kofs<8>(n, 0)) = make_float4(hi, mid, r - mid, 0.f);
  }
}

// Thread 0: the gate MMAs of a step into TMEM columns [0, 4D).
template <int D>
__device__ __forceinline__ void issue_gates(float* sm, uint32_t tmem, uint64_t* bar) {
  using L = Layout<D>;
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  constexpr uint32_t id = idesc<4 * D>(false), sbo = 32 * D;
#pragma unroll
  for (int ks = 0; ks < D / 8; ++ks) {
    const uint32_t off = uint32_t(ks) * 256u;
    const uint64_t ah = desc(su32(sm + L::a_hi) + off, sbo), al = desc(su32(sm + L::a_lo) + off, sbo);
    const uint64_t wh = desc(su32(sm + L::w_hi) + off, sbo), wl = desc(su32(sm + L::w_lo) + off, sbo);
    mma_ss(tmem, al, wh, id, ks ? 1u : 0u);
    mma_ss(tmem, ah, wl, id, 1u);
    mma_ss(tmem, ah, wh, id, 1u);
  }
  const uint64_t one = desc(su32(sm + L::one), 0);  // broadcast row group
  mma_ss(tmem, one, desc(su32(sm + L::b_hi), 256), id, 1u);  // exact bias (lstm_f32_tc.cuh)
  commit(bar);
}

// Unit pairs of this thread's sequence, block `base` (0: h, D: c) of a state.
// Through L2 (ld.global.cg): a chained predecessor may have written the rows
// while this kernel was resident (chain.cuh).
template <int D>
__device__ __forceinline__ void load_rows(const float* __restrict__ x, int64_t B, int64_t b, int base,
                                          float2 (&v)[D / 2]) {
#pragma unroll
  for (int p = 0; p < D / 2; ++p)
    v[p] = make_float2(chain::ldcg(x + int64_t(base + 2 * p) * B + b),
                       chain::ldcg(x + int64_t(base + 2 * p + 1) * B + b));
}
template <int D>
__device__ __forceinline__ void store_rows(float* __restrict__ x, int64_t B, int64_t b, int base,
                                           const float2 (&v)[D / 2]) {
#pragma unroll
  for (int p = 0; p < D / 2; ++p) {
    x[int64_t(base + 2 * p) * B + b] = v[p].x;
    x[int64_t(base + 2 * p + 1) * B + b] = v[p].y;
  }
}

// Forward over `count` steps from `from` (count = 1: the per-step operator).
// TAPE stores every step's output state to outs.p[i]; otherwise the final
// state goes to `out`.
template <int D, bool TAPE>
__global__ void __launch_bounds__(kThreads, D == 16 ? 6 : D == 32 ? 4 : 1)  // register caps: d = 16 85, d = 32 128
    fwd_tcd(const float* __restrict__ in, float* __restrict__ out, int64_t B, const float* __restrict__ xbs_all,
            const float* __restrict__ ws, int64_t from, int count, const __grid_constant__ OutPtrs outs,
            chain::Chain ch) {
  using L = Layout<D>;
  extern __shared__ __align__(128) float sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::fwd_end);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  setup<D>(sm, bars, tslot, ws, tmem_cols(4 * D), 1, false);
  const uint32_t tmem = tmem_base(tslot);
  chain::allow_dependents(ch);
  const uint32_t lane = uint32_t((threadIdx.x >> 5) * 32) << 16;
  uint32_t ph = 0;
  bool wready = false;
  // persistent over 128-sequence tiles (the weight setup is paid once per CTA)
  for (int64_t tile = blockIdx.x; tile * kThreads < B; tile += gridDim.x) {
  chain::wait_tile(ch, tile, 0);
  const int64_t b = tile * kThreads + threadIdx.x;
  const bool live = b < B;
  // d = 64 (one CTA per SM, latency-bound): c is loaded after the first gate
  // MMAs are issued, overlapping them (36.1 vs 37.4 us per step); at d = 16 /
  // 32 the later loads cost more than they hide (measured, not kept)
  constexpr bool kLateC = D == 64;
  float2 h[D / 2], c[D / 2];
  if (live) {
    load_rows<D>(in, B, b, 0, h);
    if (!kLateC) load_rows<D>(in, B, b, D, c);
  } else {
#pragma unroll
    for (int p = 0; p < D / 2; ++p) h[p] = c[p] = make_float2(0.f, 0.f);
  }
  for (int i = 0; i < count; ++i, ++ph) {
    stage<D>(sm, h, xbs_all + (from + i) * 4 * D);
    publish();
    if (threadIdx.x == 0) {
      weights_ready(bars + 1, wready);
      issue_gates<D>(sm, tmem, bars);
    }
    if (kLateC && i == 0 && live) load_rows<D>(in, B, b, D, c);
    wait_bar(bars, ph & 1u);
#pragma unroll
    for (int p0 = 0; p0 < D / 2; p0 += 4) {  // 4 unit pairs per TMEM round trip
      float g[4][8];
#pragma unroll
      for (int q = 0; q < 4; ++q) ld8(tmem + lane + uint32_t(8 * (p0 + q)), g[q]);
      ld_wait();
#pragma unroll
      for (int q = 0; q < 4; q += 2) {  // two unit pairs share the tanh reciprocal
        const float2 pa[4] = {make_float2(g[q][0], g[q][1]), make_float2(g[q][2], g[q][3]),
                              make_float2(g[q][4], g[q][5]), make_float2(g[q][6], g[q][7])};
        const float2 pb[4] = {make_float2(g[q + 1][0], g[q + 1][1]), make_float2(g[q + 1][2], g[q + 1][3]),
                              make_float2(g[q + 1][4], g[q + 1][5]), make_float2(g[q + 1][6], g[q + 1][7])};
        fwd_units2_nr(pa, pb, c[p0 + q], c[p0 + q + 1], h[p0 + q], h[p0 + q + 1]);
      }
    }
    if (TAPE && live) {
      store_rows<D>(outs.p[i], B, b, 0, h);
      store_rows<D>(outs.p[i], B, b, D, c);
    }
  }
  if (!TAPE && live) {
    store_rows<D>(out, B, b, 0, h);
    store_rows<D>(out, B, b, D, c);
  }
  chain::set_tile(ch, tile, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols(4 * D)));
}

// Reverse over steps from+count-1 .. from (count = 1: the per-step adjoint).
// The transposed product runs in two K halves (unit pairs p < D/4, then the
// rest) that share one 2D-column residual region: the first half's MMAs run
// while the threads compute the second half's gate adjoints, and TMEM drops
// from 9D to 7D columns (d=32: 512 -> 256, so 2 CTAs/SM instead of 1).
template <int D>
__global__ void __launch_bounds__(kThreads)
    rev_tcd(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B, const float* __restrict__ xbs_all,
            const float* __restrict__ ws, int64_t from, int count, const __grid_constant__ StatePtrs states,
            chain::Chain ch) {
  using L = Layout<D>;
  extern __shared__ __align__(128) float sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L::rev_end);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3);
  constexpr int kCols = tmem_cols(7 * D);
  constexpr uint32_t kLo = 4 * D, kDh = 6 * D;
  constexpr int kHalf = D / 4;  // unit pairs per K half
  setup<D>(sm, bars, tslot, ws, kCols, 2, true);
  const uint32_t tmem = tmem_base(tslot);
  chain::allow_dependents(ch);
  bool wready = false;
  const uint32_t lane = uint32_t((threadIdx.x >> 5) * 32) << 16;
  // Thread 0: dh (+)= da . B2^T over unit pairs [p0, p0 + kHalf) (residual at kLo).
  auto issue_half = [&](int p0, bool first) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    constexpr uint32_t it = idesc<D>(false), sbo32 = 32 * 4 * D;
#pragma unroll
    for (int q = 0; q < kHalf; ++q) {  // K = 8 per MMA = one unit pair, small terms first
      const int ks = p0 + q;
      const uint32_t off = uint32_t(ks) * 256u;
      const uint64_t bh = desc(su32(sm + L::w2_hi) + off, sbo32), bl = desc(su32(sm + L::w2_lo) + off, sbo32);
      mma_ts(tmem + kDh, tmem + kLo + uint32_t(8 * q), bh, it, (first && q == 0) ? 0u : 1u, false);
      mma_ts(tmem + kDh, tmem + uint32_t(8 * ks), bl, it, 1u, false);
      mma_ts(tmem + kDh, tmem + uint32_t(8 * ks), bh, it, 1u, false);
    }
    commit(bars + 1);
  };
  uint32_t phase = 0, phase2 = 0;
  // persistent over 128-sequence tiles (the weight setup is paid once per CTA)
  for (int64_t tile = blockIdx.x; tile * kThreads < B; tile += gridDim.x) {
  chain::wait_tile(ch, tile, 0);
  const int64_t b = tile * kThreads + threadIdx.x;
  const bool live = b < B;
  float2 dh[D / 2], dc[D / 2];
  if (live) {
    load_rows<D>(adj_in, B, b, 0, dh);
    load_rows<D>(adj_in, B, b, D, dc);
  } else {
#pragma unroll
    for (int p = 0; p < D / 2; ++p) dh[p] = dc[p] = make_float2(0.f, 0.f);
  }
  // d = 32 (two CTAs per SM, set by TMEM, so registers are free): the taped
  // state of the next step is loaded into registers while this step computes
  constexpr bool kAhead = D == 32;
  float2 hn[D / 2], cn[D / 2];
  if (kAhead) {
    if (live) {
      load_rows<D>(states.p[count - 1], B, b, 0, hn);
      load_rows<D>(states.p[count - 1], B, b, D, cn);
    } else {
#pragma unroll
      for (int p = 0; p < D / 2; ++p) hn[p] = cn[p] = make_float2(0.f, 0.f);
    }
  }
  for (int i = count - 1; i >= 0; --i, ++phase) {
    float2 h[D / 2], c[D / 2];
    if (kAhead) {
#pragma unroll
      for (int p = 0; p < D / 2; ++p) h[p] = hn[p], c[p] = cn[p];
    } else if (live) {
      load_rows<D>(states.p[i], B, b, 0, h);
      load_rows<D>(states.p[i], B, b, D, c);
    } else {
#pragma unroll
      for (int p = 0; p < D / 2; ++p) h[p] = c[p] = make_float2(0.f, 0.f);
    }
    stage<D>(sm, h, xbs_all + (from + i) * 4 * D);
    publish();
    if (threadIdx.x == 0) {
      weights_ready(bars + 2, wready);
      issue_gates<D>(sm, tmem, bars);
    }
    if (kAhead && live && i > 0) {
      load_rows<D>(states.p[i - 1], B, b, 0, hn);
      load_rows<D>(states.p[i - 1], B, b, D, cn);
    }
    wait_bar(bars, phase & 1u);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
#pragma unroll
      for (int p0 = half * kHalf; p0 < (half + 1) * kHalf; p0 += 4) {
        float g[4][8];
#pragma unroll
        for (int q = 0; q < 4; ++q) ld8(tmem + lane + uint32_t(8 * (p0 + q)), g[q]);
        ld_wait();
        if (half == 1 && p0 == kHalf) {  // the residual region is free once the first half's MMAs are done
          wait_bar(bars + 1, phase2 & 1u);
          ++phase2;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int p = p0 + q;
          float2 da[4];
          bwd_unit(make_float2(g[q][0], g[q][1]), make_float2(g[q][2], g[q][3]), make_float2(g[q][4], g[q][5]),
                   make_float2(g[q][6], g[q][7]), c[p], dh[p], dc[p], da[0], da[1], da[2], da[3], dc[p]);
          uint32_t hv[8], lv[8];
#pragma unroll
          for (int gi = 0; gi < 4; ++gi) {
            const float2 hi = make_float2(hi_part(da[gi].x), hi_part(da[gi].y));
            const float2 lo = sub2(da[gi], hi);
            hv[2 * gi] = __float_as_uint(hi.x);
            hv[2 * gi + 1] = __float_as_uint(hi.y);
            lv[2 * gi] = __float_as_uint(lo.x);
            lv[2 * gi + 1] = __float_as_uint(lo.y);
          }
          st8(tmem + lane + uint32_t(8 * p), hv);
          st8(tmem + lane + kLo + uint32_t(8 * (p - half * kHalf)), lv);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      publish();
      if (threadIdx.x == 0) issue_half(half * kHalf, half == 0);
    }
    wait_bar(bars + 1, phase2 & 1u);
    ++phase2;
#pragma unroll
    for (int m0 = 0; m0 < D; m0 += 8) {
      float v[8];
      ld8(tmem + lane + kDh + uint32_t(m0), v);
      ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) dh[m0 / 2 + q] = make_float2(v[2 * q], v[2 * q + 1]);
    }
  }
  if (live) {
    store_rows<D>(adj_out, B, b, 0, dh);
    store_rows<D>(adj_out, B, b, D, dc);
  }
  chain::set_tile(ch, tile, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

// ---- d = 64 reverse: one kernel, Wᵀ streamed ------------------------------
// At d = 64 the gate operands (A = h hi/lo 64 KB, W hi/lo 128 KB, bias 8 KB)
// fill the shared memory, so the B operand of the transposed product
// dh = da · B2ᵀ (B2 = Wᵀ, another 128 KB as hi/lo, and kind::tf32 operands
// cannot be read transposed: tools/umma_layout_probe.cu) streams every step
// from a pre-split chunk image in global memory (128 KB per cell, L2
// resident) through a ring of kRing64 shared-memory stages, one K = 8 chunk
// (N = 64 rows x K = 8, hi and lo, 4 KB) per stage.  Warp roles: warps 0-3
// compute (sequence = thread = TMEM lane, as rev_tcd), warp 4 issues every
// MMA (one thread), warp 5 produces the ring (one thread, cp.async.bulk,
// full / empty mbarriers; an empty barrier is released by tcgen05.commit when
// the MMAs reading the stage complete).  The compute warps and the issuer
// meet at named barrier 1 (160 threads); the producer runs ahead on the
// mbarriers only.  Arithmetic as rev_tcd: 3xTF32 gates and transposed
// product, da in TMEM as the A operand, two K halves sharing the residual.
constexpr int kChunks64 = 4 * 64 / 8;    // K = 8 chunks of the transposed product per step
constexpr int kChunkFloats64 = 64 * 8;   // one part (hi or lo) of a chunk: 2 KB
#ifndef ACKPT_RING64
#define ACKPT_RING64 6
#endif
constexpr int kRing64 = ACKPT_RING64;
constexpr int kThreads64 = 192;
constexpr size_t kRev64Smem = size_t(Layout<64>::fwd_end) * 4 + size_t(kRing64) * 2 * kChunkFloats64 * 4 + 256;

// Chunk image of B2 = scaled Wᵀ for the d = 64 reverse: chunk c (gate rows
// n in [8c, 8c + 8), the K index of the transposed product) is [hi | lo],
// each N = 64 (m) x K = 8, K-major core matrices (LBO 128 B, SBO 256 B).
__global__ void w2_image64(const float* __restrict__ ws, float* __restrict__ img) {
  constexpr int D = 64;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < kChunks64 * 2 * kChunkFloats64;
       idx += gridDim.x * blockDim.x) {
    const int c = idx / (2 * kChunkFloats64), part = (idx / kChunkFloats64) & 1, e = idx % kChunkFloats64;
    const int m = (e / 64) * 8 + ((e % 32) / 4), k = ((e % 64) / 32) * 4 + (e % 4);
    int gi, j;
    gate_of(8 * c + k, gi, j);
    const float x = ws[(gi * D + j) * D + m];
    img[idx] = part ? x - hi_part(x) : hi_part(x);
  }
}

__device__ __forceinline__ void bar_compute_issue() { asm volatile("bar.sync 1, 160;" ::: "memory"); }

__global__ void __launch_bounds__(kThreads64, 1)
    rev_tcd64(const float* __restrict__ adj_in, float* __restrict__ adj_out, int64_t B,
              const float* __restrict__ xbs_all, const float* __restrict__ wimg, const float* __restrict__ w2img,
              int64_t from, int count, const __grid_constant__ StatePtrs states, chain::Chain ch) {
  constexpr int D = 64;
  using L = Layout<D>;
  extern __shared__ __align__(128) float sm[];
  float* ring = sm + L::fwd_end;
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + kRing64 * 2 * kChunkFloats64);
  uint64_t* bar_g = bars;               // gate MMAs done
  uint64_t* bar_t = bars + 1;           // transposed-product half done (completes twice per step)
  uint64_t* full = bars + 2;            // [kRing64] chunk landed
  uint64_t* empty = bars + 2 + kRing64; // [kRing64] chunk consumed by the MMAs
  uint64_t* wbar = bars + 2 + 2 * kRing64;  // weight image landed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3 + 2 * kRing64);
  constexpr int kCols = 512;
  constexpr uint32_t kLo = 4 * D, kDh = 6 * D;
  constexpr int kHalf = D / 4;  // unit pairs (= K chunks) per K half
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t tiles = (B + kThreads - 1) / kThreads;
  const int my_tiles = blockIdx.x < tiles ? int((tiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;

  // setup: TMEM (warp 0), barriers, ones, W, zero bias rows (compute threads)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 3 + 2 * kRing64; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    expect_bytes(wbar, uint32_t(8 * D * D * 4));
    bulk_in(sm + L::w_hi, wimg, 8 * D * D, wbar);  // W hi | lo (the issuer waits before its first MMA)
  }
  if (tid < kThreads) {
    if (tid < 8) {
      *reinterpret_cast<float4*>(sm + L::one + kofs<8>(tid, 0)) = make_float4(1.f, 1.f, 1.f, 0.f);
      *reinterpret_cast<float4*>(sm + L::one + kofs<8>(tid, 4)) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int idx = tid; idx < 4 * D * 8; idx += kThreads) sm[L::b_hi + kofs<8>(idx / 8, idx % 8)] = 0.f;
  }
  const uint32_t tmem = tmem_base(tslot);  // (all 192 threads: a full barrier)
  chain::allow_dependents(ch);

  if (warp == 5) {  // ---- producer: the chunk sequence, step after step
    if (tid == 5 * 32) {
      const int64_t total = int64_t(my_tiles) * count * kChunks64;
      for (int64_t it = 0; it < total; ++it) {
        const int st = int(it % kRing64);
        if (it >= kRing64) wait_bar(empty + st, uint32_t((it / kRing64 - 1) & 1));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + st)),
                     "r"(uint32_t(2 * kChunkFloats64 * 4))
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(ring + st * 2 * kChunkFloats64)),
                     "l"(w2img + (it % kChunks64) * 2 * kChunkFloats64), "r"(uint32_t(2 * kChunkFloats64 * 4)),
                     "r"(su32(full + st))
                     : "memory");
      }
    }
  } else if (warp == 4) {  // ---- MMA issuer
    int64_t it = 0;
    bool wready = false;
    for (int t = 0; t < my_tiles; ++t)
      for (int i = 0; i < count; ++i) {
        bar_compute_issue();  // A operand and bias staged
        if (tid == 4 * 32) {
          weights_ready(wbar, wready);
          issue_gates<D>(sm, tmem, bar_g);
        }
        __syncwarp();
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          bar_compute_issue();  // this half's da in TMEM
          if (tid == 4 * 32) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            constexpr uint32_t id = idesc<D>(false);
#pragma unroll 1
            for (int q = 0; q < kHalf; ++q, ++it) {
              const int ks = half * kHalf + q, st = int(it % kRing64);
              wait_bar(full + st, uint32_t((it / kRing64) & 1));
              const uint32_t base = su32(ring + st * 2 * kChunkFloats64);
              const uint64_t bh = desc(base, 256), bl = desc(base + kChunkFloats64 * 4, 256);
              mma_ts(tmem + kDh, tmem + kLo + uint32_t(8 * q), bh, id, (half == 0 && q == 0) ? 0u : 1u, false);
              mma_ts(tmem + kDh, tmem + uint32_t(8 * ks), bl, id, 1u, false);
              mma_ts(tmem + kDh, tmem + uint32_t(8 * ks), bh, id, 1u, false);
              commit(empty + st);
            }
            commit(bar_t);
          }
          __syncwarp();
        }
      }
  } else {  // ---- compute warps
    const uint32_t lane = uint32_t(warp * 32) << 16;
    uint32_t phase = 0, phase_t = 0;
    for (int t = 0; t < my_tiles; ++t) {
      const int64_t tile = blockIdx.x + int64_t(t) * gridDim.x;
      chain::wait_tile(ch, tile, 0, 2, kThreads);  // the compute warps (named barrier 2)
      const int64_t b = tile * kThreads + tid;
      const bool live = b < B;
      float2 dh[D / 2], dc[D / 2];
      if (live) {
        load_rows<D>(adj_in, B, b, 0, dh);
        load_rows<D>(adj_in, B, b, D, dc);
      } else {
#pragma unroll
        for (int p = 0; p < D / 2; ++p) dh[p] = dc[p] = make_float2(0.f, 0.f);
      }
      for (int i = count - 1; i >= 0; --i, ++phase) {
        {
          float2 h[D / 2];
          if (live) load_rows<D>(states.p[i], B, b, 0, h);
          else
#pragma unroll
            for (int p = 0; p < D / 2; ++p) h[p] = make_float2(0.f, 0.f);
          stage<D>(sm, h, xbs_all + (from + i) * 4 * D);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        bar_compute_issue();
        const float* xs = states.p[i];
        // c of a group of 4 unit pairs is loaded one group ahead (the first
        // group while the gate MMAs run)
        float2 cq[4];
        auto load_c = [&](int p0) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            cq[q] = live ? make_float2(chain::ldcg(xs + int64_t(D + 2 * (p0 + q)) * B + b),
                                       chain::ldcg(xs + int64_t(D + 2 * (p0 + q) + 1) * B + b))
                         : make_float2(0.f, 0.f);
        };
        load_c(0);
        wait_bar(bar_g, phase & 1u);
#pragma unroll
        for (int grp = 0; grp < D / 8; ++grp) {
          const int p0 = 4 * grp, half = grp / (kHalf / 4);
          float g[4][8];
#pragma unroll
          for (int q = 0; q < 4; ++q) ld8(tmem + lane + uint32_t(8 * (p0 + q)), g[q]);
          float2 c[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = cq[q];
          if (grp + 1 < D / 8) load_c(p0 + 4);
          ld_wait();
          if (p0 == kHalf) {  // the residual region is free once half 0's MMAs are done
            wait_bar(bar_t, phase_t & 1u);
            ++phase_t;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int p = p0 + q;
            float2 da[4];
            bwd_unit(make_float2(g[q][0], g[q][1]), make_float2(g[q][2], g[q][3]), make_float2(g[q][4], g[q][5]),
                     make_float2(g[q][6], g[q][7]), c[q], dh[p], dc[p], da[0], da[1], da[2], da[3], dc[p]);
            uint32_t hv[8], lv[8];
#pragma unroll
            for (int gi = 0; gi < 4; ++gi) {
              const float2 hi = make_float2(hi_part(da[gi].x), hi_part(da[gi].y));
              const float2 lo = sub2(da[gi], hi);
              hv[2 * gi] = __float_as_uint(hi.x);
              hv[2 * gi + 1] = __float_as_uint(hi.y);
              lv[2 * gi] = __float_as_uint(lo.x);
              lv[2 * gi + 1] = __float_as_uint(lo.y);
            }
            st8(tmem + lane + uint32_t(8 * p), hv);
            st8(tmem + lane + kLo + uint32_t(8 * (p - half * kHalf)), lv);
          }
          if (p0 + 4 == (half + 1) * kHalf) {  // this half's da is in TMEM: the issuer may go
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            bar_compute_issue();
          }
        }
        wait_bar(bar_t, phase_t & 1u);
        ++phase_t;
#pragma unroll
        for (int m0 = 0; m0 < D; m0 += 8) {
          float v[8];
          ld8(tmem + lane + kDh + uint32_t(m0), v);
          ld_wait();
#pragma unroll
          for (int q = 0; q < 4; ++q) dh[m0 / 2 + q] = make_float2(v[2 * q], v[2 * q + 1]);
        }
      }
      if (live) {
        store_rows<D>(adj_out, B, b, 0, dh);
        store_rows<D>(adj_out, B, b, D, dc);
      }
      chain::set_tile(ch, tile, 0, 2, kThreads);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
}

}  // namespace tcd
}  // namespace ackpt
