// fp32 LSTM step kernels, TMA-pipelined persistent variant (K1 forward, K2
// adjoint) for sm_100a.  Same arithmetic as lstm_f32.cuh (shared helpers in
// lstm_f32_math.cuh), so both variants give bit-identical results.
//
// Data movement.  A tile is TILE = 2*THREADS consecutive batch elements.  Its
// input rows (h, c [, dh, dc]) are TILE*4-byte contiguous segments of the
// batch-fastest state layout, moved by one thread with cp.async.bulk
// (UBLKCP, the TMA bulk-copy path) into a STAGES-deep shared-memory ring whose
// slots complete on an mbarrier (expect_tx).  Each thread reads its float2
// pair with LDS.64 (conflict-free), computes, writes its results back into
// the same smem slots, and the tile leaves with bulk stores (smem -> global).
// Memory requests do not depend on registers or occupancy: the ring keeps
// STAGES-1 tiles in flight per CTA while the warps compute.
#pragma once

#include <cuda_runtime.h>

#include "lstm_f32_math.cuh"

namespace ackpt {
namespace tma {

using namespace f32m;

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

enum Mode { kFwd = 0, kBwd = 1 };

template <int D, int MODE, int THREADS>
struct Geometry {
  static constexpr int kTile = 2 * THREADS;                   // elements per tile
  static constexpr int kRows = MODE == kFwd ? 2 * D : 4 * D;  // input rows
  static constexpr int kStageFloats = kRows * kTile;
  static constexpr int kStageBytes = kStageFloats * 4;
};

// grid: persistent; tile t = blockIdx.x + k * gridDim.x.
// x: state (2D rows of B), a: adjoint in (2D rows, bwd only), y: output (2D rows).
// Per CTA: the prologue loads tiles 0..STAGES-2; iteration i waits for tile
// i, computes it in place, bulk-stores it, then refills the stage of tile i-1
// (whose store has been reading smem for one iteration) with tile i+STAGES-1.
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
        float2 af, ai, ao, ag;
        preacts<D>(p.ws, p.xbs, h, j, af, ai, ao, ag);
        float2* cslot = st2 + (D + j) * kHalf + tid;
        float2 c = *cslot;
        hn[j] = fwd_unit(af, ai, ao, ag, c);
        *cslot = c;
      }
#pragma unroll
      for (int j = 0; j < D; ++j) st2[j * kHalf + tid] = hn[j];
    } else {
      float2 acc[D];
#pragma unroll
      for (int m = 0; m < D; ++m) acc[m] = bc(0.0f);
#pragma unroll
      for (int j = 0; j < D; ++j) {
        float2 af, ai, ao, ag, daf, dai, dao, dag, dck;
        preacts<D>(p.ws, p.xbs, h, j, af, ai, ao, ag);
        float2* cslot = st2 + (D + j) * kHalf + tid;
        bwd_unit(af, ai, ao, ag, *cslot, st2[(2 * D + j) * kHalf + tid], st2[(3 * D + j) * kHalf + tid],
                 daf, dai, dao, dag, dck);
        *cslot = dck;
#pragma unroll
        for (int m = 0; m < D; ++m) {  // lstm.py:149-150
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
      const int64_t tn = t + int64_t(STAGES - 1) * stride;
      if (tn < ntiles) {
        bulk_wait_read<1>();
        issue(int((i + STAGES - 1) % STAGES), tn);
      }
    }
  }
  if (tid == 0) bulk_wait_all();
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
  f32m::ScaledParams<D> p;
  f32m::fill_scaled<D>(c, step, p);
  kern<<<grid, THREADS, kSmem, s>>>(x, a, y, c->B, ntiles, p);
}

}  // namespace ackpt

#define ACKPT_INSTANTIATE_TMA(D, MODE, THREADS, STAGES)                                         \
  namespace ackpt {                                                                            \
  template void tma_launch<D, MODE, THREADS, STAGES>(const ackpt_lstm*, int64_t, const float*, \
                                                     const float*, float*, cudaStream_t);      \
  }
