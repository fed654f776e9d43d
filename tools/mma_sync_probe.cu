// Throughput of warp-level mma.sync (the legacy HMMA path) on sm_100a:
// tf32 m16n8k8 and bf16 m16n8k16 with fp32 accumulators, 8 independent
// accumulator chains per warp, 16 warps per SM, one CTA per SM x 8.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_sync_probe tools/mma_sync_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int kChains = 8, kIters = 4096;

__global__ void tf32_loop(float* out, float seed) {
  float c[kChains][4] = {};
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(seed + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(seed - threadIdx.x * 1e-3f + i);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void bf16_loop(float* out, float seed) {
  float c[kChains][4] = {};
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x + i;
  for (int i = 0; i < 2; ++i) b[i] = 0x3f803f80u + threadIdx.x + 2 * i;
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int q = 0; q < kChains; ++q)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = seed;
  for (int q = 0; q < kChains; ++q) s += c[q][0] + c[q][1] + c[q][2] + c[q][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, size_t(sms) * 8 * 512 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int threads = 32 * (warps < 16 ? warps : 16), blocks = sms * (warps < 16 ? 1 : warps / 16);
    for (int kind = 0; kind < 2; ++kind) {
      auto launch = [&] {
        if (kind == 0) tf32_loop<<<blocks, threads>>>(out, 1.0f);
        else bf16_loop<<<blocks, threads>>>(out, 1.0f);
      };
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double mmas = double(blocks) * (threads / 32) * kChains * kIters;
      const double flops = mmas * (kind == 0 ? 16 * 8 * 8 * 2 : 16 * 8 * 16 * 2);
      printf("%s warps/SM=%2d: %.3f ms, %.1f TFLOP/s, %.2f mma/clk/SM (at 1.965 GHz)\n", kind ? "bf16 m16n8k16" : "tf32 m16n8k8 ",
             warps, ms, flops / (ms * 1e-3) / 1e12, mmas / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
