// Probe of the A-from-TMEM ("TS") tcgen05 forms used by the tensor-core
// reverse run: D[128 x 16] = A[128 x 32] * B[16 x 32]^T with
//   mode 0: A tf32 in TMEM (columns = k), B tf32 K-major smem, plain TF32
//   mode 1: A = hi + lo: hi tf32 in TMEM (x W_hi and x W_lo, kind::tf32),
//           lo as packed bf16 in TMEM (x W as bf16, kind::f16), all into
//           one fp32 accumulator
//   mode 2: as mode 1 with the bf16 pair packing swapped (layout check)
// against float64.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_ts_probe tools/umma_ts_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int K = 32, N = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc(int a_fmt, int b_fmt, int M, int Nn) {
  return (1u << 4) | (uint32_t(a_fmt) << 7) | (uint32_t(b_fmt) << 10) | (uint32_t(Nn >> 3) << 17) |
         (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// K-major no swizzle, 16-byte core-matrix rows; LBO between K chunks, SBO between 8-row groups
constexpr uint32_t kLBO = 256, kSBO = 128;  // N = 16: two row groups per K chunk
__device__ __forceinline__ int off32(int r, int k) { return (k / 4) * kLBO + (r / 8) * kSBO + (r % 8) * 16 + (k % 4) * 4; }
__device__ __forceinline__ int off16(int r, int k) { return (k / 8) * kLBO + (r / 8) * kSBO + (r % 8) * 16 + (k % 8) * 2; }

__device__ __forceinline__ void mma_ts_tf32(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts_f16(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(id), "r"(acc));
}

__device__ __forceinline__ void st8(uint32_t addr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}

__global__ void probe(const float* a, const float* b, float* d, int mode) {
  __shared__ __align__(128) unsigned char Bh[N * K * 4], Bl[N * K * 4], Bb[N * K * 2];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    const float x = b[i];
    *reinterpret_cast<float*>(Bh + off32(r, k)) = tf32_hi(x);
    *reinterpret_cast<float*>(Bl + off32(r, k)) = x - tf32_hi(x);
    *reinterpret_cast<__nv_bfloat16*>(Bb + off16(r, k)) = __float2bfloat16_rn(x);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;  // D: cols [0,16); A hi: [32, 64); A lo (tf32 or bf16): [64, 96)
  const uint32_t lane = uint32_t(warp * 32) << 16;
  {
    const int r = tid;
    for (int c0 = 0; c0 < K; c0 += 8) {
      uint32_t hv[8], lv[8];
      for (int q = 0; q < 8; ++q) {
        const float x = a[r * K + c0 + q];
        hv[q] = __float_as_uint(mode == 0 ? x : tf32_hi(x));
      }
      st8(tmem + lane + 32 + c0, hv);
      if (mode != 0 && c0 < K / 2) {  // bf16 pairs: 2 k per column -> 16 columns
        for (int q = 0; q < 8; ++q) {
          const int k0 = 2 * (c0 + q), k1 = k0 + 1;
          const float x0 = a[r * K + k0] - tf32_hi(a[r * K + k0]), x1 = a[r * K + k1] - tf32_hi(a[r * K + k1]);
          const uint32_t lo16 = __bfloat16_as_ushort(__float2bfloat16_rn(mode == 1 ? x0 : x1));
          const uint32_t hi16 = __bfloat16_as_ushort(__float2bfloat16_rn(mode == 1 ? x1 : x0));
          lv[q] = lo16 | (hi16 << 16);
        }
        st8(tmem + lane + 64 + c0, lv);
      }
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t it = idesc(2, 2, 128, N), ib = idesc(1, 1, 128, N);
    for (int ks = 0; ks < K / 8; ++ks) {  // tf32: K = 8 per MMA = 2 chunks
      const uint64_t bh = smem_desc(smem_u32(Bh) + ks * 2 * kLBO, kLBO, kSBO);
      const uint64_t bl = smem_desc(smem_u32(Bl) + ks * 2 * kLBO, kLBO, kSBO);
      mma_ts_tf32(tmem, tmem + 32 + ks * 8, bh, it, ks ? 1u : 0u);
      if (mode != 0) mma_ts_tf32(tmem, tmem + 32 + ks * 8, bl, it, 1u);
    }
    if (mode != 0)
      for (int ks = 0; ks < K / 16; ++ks) {  // bf16: K = 16 per MMA = 2 chunks = 8 columns
        const uint64_t bb = smem_desc(smem_u32(Bb) + ks * 2 * kLBO, kLBO, kSBO);
        mma_ts_f16(tmem, tmem + 64 + ks * 8, bb, ib, 1u);
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(smem_u32(&mbar))
                 : "memory");
  } while (!done);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(tmem + lane));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < N; ++j) d[tid * N + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
}

int main() {
  std::vector<float> a(128 * K), b(N * K), d(128 * N);
  srand(3);
  for (auto& x : a) x = 2.0f * (float(rand()) / RAND_MAX - 0.5f);
  for (auto& x : b) x = 0.4f * (float(rand()) / RAND_MAX - 0.5f);
  float *da, *db, *dd;
  cudaMalloc(&da, a.size() * 4);
  cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&dd, d.size() * 4);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  int bad = 0;
  for (int mode = 0; mode < 3; ++mode) {
    probe<<<1, 128>>>(da, db, dd, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode=%d CUDA error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += double(a[r * K + k]) * double(b[n * K + k]);
        num += (d[r * N + n] - ref) * (d[r * N + n] - ref);
        den += ref * ref;
      }
    printf("mode=%d rel_l2=%.3e\n", mode, sqrt(num / den));
  }
  return bad;
}
