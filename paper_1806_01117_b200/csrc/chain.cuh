// Per-tile launch chain of the tensor-core LSTM kernels (lstm_f32_tc.cuh,
// lstm_f32_tcd.cuh).
//
// Consecutive launches of one cell on one stream touch the batch tile by tile:
// tile t of a launch reads and writes only tile t of its states / adjoints
// (every sequence is independent), so tile t of the next launch depends on
// tile t of this one and nothing else.  A chained launch is a programmatic
// dependent launch: its CTAs are scheduled while the previous launch drains,
// and each waits only for its own tile's completion flag
// (flags[t] = the previous launch's epoch, release / acquire at gpu scope)
// instead of the whole grid.  The last wave of one launch then overlaps the
// first wave (and the TMEM / barrier / weight-image setup) of the next.
//
// Deadlock freedom: a launch allows dependents (griddepcontrol.launch_dependents)
// only after each CTA holds its TMEM, so the next launch is scheduled once every
// CTA of this one is resident or done; a waiting CTA then waits on a resident
// producer.  With wait = 0 the kernel is a plain launch (it still publishes).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <string>

#include "lstm_cell.h"

namespace ackpt {
namespace chain {

struct Chain {
  uint32_t* flags;  // one epoch per tile; nullptr: chaining off
  uint32_t wait;    // 0: not chained; else wait until flags[t] reaches it
  uint32_t set;     // this launch's epoch
};

// All threads of the CTA (after the TMEM allocation): dependents may start.
__device__ __forceinline__ void allow_dependents(const Chain& ch) {
  if (ch.flags) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// One thread: spin until tile t of the previous launch is published.
__device__ __forceinline__ void spin_tile(const Chain& ch, int64_t t) {
  uint32_t v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ch.flags + t) : "memory");
    if (int32_t(v - ch.wait) >= 0) break;
    __nanosleep(128);
  }
}

// CTA-wide wait for tile t (bar: __syncthreads when nthreads = 0, else the
// named barrier `id` over nthreads threads -- the threads that touch the tile).
__device__ __forceinline__ void sync_group(int id, int nthreads) {
  if (nthreads == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void wait_tile(const Chain& ch, int64_t t, int leader, int id = 0, int nthreads = 0) {
  if (!ch.flags || !ch.wait) return;
  if (int(threadIdx.x) == leader) spin_tile(ch, t);
  sync_group(id, nthreads);
  // the producer's generic-proxy stores, now acquired, before this CTA's
  // bulk-copy (async-proxy) reads of the same data
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// CTA-wide publish of tile t (after this launch's last access of it): the
// barrier orders every thread's accesses before the leader's gpu-scope
// release fence (cumulative), so only the leader fences -- a per-thread
// __threadfence() made every warp wait for its stores to drain, once per
// tile of a persistent kernel.
__device__ __forceinline__ void set_tile(const Chain& ch, int64_t t, int leader, int id = 0, int nthreads = 0) {
  if (!ch.flags) return;
  sync_group(id, nthreads);
  if (int(threadIdx.x) == leader)
    asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u32 [%0], %1;" ::"l"(ch.flags + t), "r"(ch.set)
                 : "memory");
}

// Loads of inputs a chained predecessor may have written while this kernel
// was already resident: plain (weak) global loads, never the non-coherent
// path -- ordered after the producer's stores by the leader's acquire and the
// CTA barrier (wait_tile), and not allocated in L1 (stream-once data).
// Measured against ld.global.cg: per-step d = 16 backward 25.0 -> 24.1 us.
__device__ __forceinline__ float ldcg(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ldcg2(const float* p) {
  float2 v;
  asm volatile("ld.global.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// ---- host side -------------------------------------------------------------

// ACKPT_TC_CHAIN=0 off, =force chains every back-to-back launch of a cell on
// one stream (probes that enqueue nothing else in between); default: chain
// when the executor marks the launch of its native operator (g_chain_hint /
// g_chain_native, common.h).
inline int mode() {
  static const int m = [] {
    const char* e = std::getenv("ACKPT_TC_CHAIN");
    if (!e) return 1;
    const std::string v(e);
    return v == "0" ? 0 : v == "force" ? 2 : 1;
  }();
  return m;
}

// The chain parameters of the next launch of cell c on stream s over `tiles`
// tiles; pdl = launch it as a programmatic dependent launch.  Chained only
// when marked (the executor's hint through the native operator, or =force), when the process's last cell launch
// was a chain-publishing launch of this cell on this stream (chain_touch),
// and never under stream capture (the graph keeps full dependencies).
inline Chain next(const ackpt_lstm* c, cudaStream_t s, int64_t tiles, bool& pdl) {
  auto* cell = const_cast<ackpt_lstm*>(c);
  pdl = false;
  std::lock_guard<std::mutex> lk(chain_token().mu);  // the cell's slots and the token
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  ACKPT_CUDA_CHECK(cudaStreamIsCapturing(s, &cs));
  const int m = mode();
  if (m == 0 || cs != cudaStreamCaptureStatusNone) return Chain{nullptr, 0u, 0u};  // the chain stays closed
  const ChainStep st = chain_step(cell, s, tiles, m == 2 || g_chain_native, [&](uint32_t* old, int64_t n) {
    if (old) {  // evicted or too small: no kernel may still use it
      ACKPT_CUDA_CHECK(cudaDeviceSynchronize());
      cudaFree(old);
    }
    uint32_t* p = nullptr;
    ACKPT_CUDA_CHECK(cudaMalloc(&p, size_t(n) * sizeof(uint32_t)));
    // on the launch stream: a legacy-stream memset is not ordered before work
    // on a non-blocking stream and could land after the first flag publish
    ACKPT_CUDA_CHECK(cudaMemsetAsync(p, 0, size_t(n) * sizeof(uint32_t), s));
    return p;
  });
  pdl = st.chained;
  return Chain{st.flags, st.wait, st.set};
}

// kernel<<<grid, block, smem, s>>>(args...), as a programmatic dependent
// launch when pdl.
template <class... P, class... A>
void launch(void (*kernel)(P...), unsigned grid, unsigned block, size_t smem, bool pdl, cudaStream_t s,
            A&&... args) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  ACKPT_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, P(args)...));
}

}  // namespace chain
}  // namespace ackpt
