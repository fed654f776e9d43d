// Latency injection for the operator plugin interface: wraps an operator so
// every forward / backward call also holds the compute stream for a fixed
// time.  This is the device-side counterpart of the reference tests'
// pad_operators (pkg/tests/test_runtime.py:33-52, time.sleep per step): the
// stall / overlap / calibration tests need steps of known duration running
// concurrently with the copy engines, which a host sleep cannot give on a
// GPU stream.
#include <cuda_runtime.h>

#include <memory>

#include "common.h"

namespace ackpt {
namespace {

__global__ void spin_ns(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

struct Pad {
  ackpt_operator base;
  unsigned long long fwd_ns, bwd_ns;
};

int hold(unsigned long long ns, void* stream) {
  if (ns == 0) return ACKPT_OK;
  spin_ns<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(ns);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error(std::string("delay kernel: ") + cudaGetErrorString(e));
    return ACKPT_CUDA_ERROR;
  }
  return ACKPT_OK;
}

int pad_forward(void* ctx, int64_t step, const void* in, void* out, void* stream) {
  auto* p = static_cast<Pad*>(ctx);
  int rc = hold(p->fwd_ns, stream);
  return rc != ACKPT_OK ? rc : p->base.forward(p->base.ctx, step, in, out, stream);
}
int pad_backward(void* ctx, int64_t step, const void* st, const void* ai, void* ao, void* stream) {
  auto* p = static_cast<Pad*>(ctx);
  int rc = hold(p->bwd_ns, stream);
  return rc != ACKPT_OK ? rc : p->base.backward(p->base.ctx, step, st, ai, ao, stream);
}
int pad_seed(void* ctx, const void* fin, void* adj, void* stream) {
  auto* p = static_cast<Pad*>(ctx);
  return p->base.seed(p->base.ctx, fin, adj, stream);
}

}  // namespace
}  // namespace ackpt

extern "C" {

ACKPT_API int ackpt_pad_operator_create(const ackpt_operator* base, double forward_seconds,
                                        double backward_seconds, ackpt_operator* out) {
  return ackpt::guard([&] {
    if (!base || !base->forward || !base->backward)
      ackpt::fail(ACKPT_VALUE_ERROR, "base operator needs forward and backward");
    if (forward_seconds < 0 || backward_seconds < 0)
      ackpt::fail(ACKPT_VALUE_ERROR, "delays must be >= 0");
    auto* p = new ackpt::Pad{*base, (unsigned long long)(forward_seconds * 1e9),
                             (unsigned long long)(backward_seconds * 1e9)};
    *out = *base;
    out->ctx = p;
    out->forward = ackpt::pad_forward;
    out->backward = ackpt::pad_backward;
    out->seed = base->seed ? ackpt::pad_seed : nullptr;
    out->advance = nullptr;  // padding is per step
    out->forward_many = nullptr;
    out->backward_many = nullptr;
  });
}

ACKPT_API int ackpt_pad_operator_destroy(ackpt_operator* op) {
  return ackpt::guard([&] {
    if (op && op->ctx) delete static_cast<ackpt::Pad*>(op->ctx);
    if (op) op->ctx = nullptr;
  });
}

}  // extern "C"
