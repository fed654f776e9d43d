// Probe of the tcgen05 (UMMA) encodings used by the tensor-core LSTM kernels:
// D[128 x N] = A[128 x K] * B[N x K]^T with kind::tf32, A/B K-major in smem
// (no swizzle), D in TMEM, read back with tcgen05.ld.32x32b.  Checks plain
// TF32 and the 3xTF32 split (hi*hi + lo*hi + hi*lo) against float64, and the
// A-from-TMEM (TS) form used for the adjoint matvec.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe tools/umma_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major, no swizzle: element (r, k) at (r/8)*SBO + (k/4)*LBO + (r%8)*16 + (k%4)*4 bytes
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // sm100 descriptor version
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

template <int K>
__device__ __forceinline__ int kmaj(int r, int k) {  // float index
  constexpr int LBOf = 32, SBOf = 32 * (K / 4);
  return (r / 8) * SBOf + (k / 4) * LBOf + (r % 8) * 4 + (k % 4);
}

__device__ __forceinline__ void mma_ss(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

// mode 0: plain tf32 SS; mode 1: 3xTF32 SS; mode 2: 3xTF32 with A from TMEM (TS)
template <int K, int N>
__global__ void probe(const float* a, const float* b, float* d, int mode) {
  __shared__ __align__(128) float As[2][128 * K];
  __shared__ __align__(128) float Bs[2][N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < 128 * K; i += 128) {
    const int r = i / K, k = i % K;
    const float x = a[i];
    As[0][kmaj<K>(r, k)] = tf32_hi(x);
    As[1][kmaj<K>(r, k)] = x - tf32_hi(x);
  }
  for (int i = tid; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    const float x = b[i];
    Bs[0][kmaj<K>(r, k)] = tf32_hi(x);
    Bs[1][kmaj<K>(r, k)] = x - tf32_hi(x);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;  // columns [0, N): D; [128, 128 + 2K): A hi/lo for TS
  if (mode == 2) {
    // A hi / lo into TMEM: lane = row, column = k (thread = row of its warp's lane quadrant)
    uint32_t hi[K], lo[K];
    const int r = tid;
    for (int k = 0; k < K; ++k) {
      const float x = a[r * K + k];
      hi[k] = __float_as_uint(tf32_hi(x));
      lo[k] = __float_as_uint(x - tf32_hi(x));
    }
    const uint32_t lane_addr = tmem + (uint32_t(warp * 32) << 16);
    static_assert(K == 8 || K == 32, "probe K");
    if constexpr (K == 8) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lane_addr + 128),
                   "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7]));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lane_addr + 128 + K),
                   "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (tid == 0) {
    constexpr uint32_t LBO = 128, SBO = 128 * (K / 4);
    const uint32_t id = idesc_tf32(128, N);
    int first = 1;
    for (int kk = 0; kk < K / 8; ++kk) {
      const uint32_t off = kk * 2 * LBO;  // two 16-byte K chunks per K=8 step
      const uint64_t ah = smem_desc(smem_u32(As[0]) + off, LBO, SBO), al = smem_desc(smem_u32(As[1]) + off, LBO, SBO);
      const uint64_t bh = smem_desc(smem_u32(Bs[0]) + off, LBO, SBO), bl = smem_desc(smem_u32(Bs[1]) + off, LBO, SBO);
      if (mode == 0) {
        mma_ss(tmem, ah, bh, id, first ? 0u : 1u);
      } else if (mode == 1) {
        mma_ss(tmem, ah, bh, id, first ? 0u : 1u);
        mma_ss(tmem, al, bh, id, 1u);
        mma_ss(tmem, ah, bl, id, 1u);
      } else {
        const uint32_t at = tmem + 128 + kk * 8, atl = tmem + 128 + K + kk * 8;
        mma_ts(tmem, at, bh, id, first ? 0u : 1u);
        mma_ts(tmem, atl, bh, id, 1u);
        mma_ts(tmem, at, bl, id, 1u);
      }
      first = 0;
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  {
    uint32_t done = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done)
                   : "r"(smem_u32(&mbar))
                   : "memory");
    } while (!done);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[N];
  const uint32_t lane_addr = tmem + (uint32_t(warp * 32) << 16);
  if constexpr (N == 32) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
        "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(lane_addr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(lane_addr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < N; ++j) d[tid * N + j] = __uint_as_float(v[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int K, int N>
int run(int mode) {
  std::vector<float> a(128 * K), b(N * K), d(128 * N);
  srand(1);
  for (auto& x : a) x = float(rand()) / RAND_MAX - 0.5f;
  for (auto& x : b) x = 0.2f * (float(rand()) / RAND_MAX - 0.5f);
  float *da, *db, *dd;
  cudaMalloc(&da, a.size() * 4);
  cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&dd, d.size() * 4);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  probe<K, N><<<1, 128>>>(da, db, dd, mode);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("K=%d N=%d mode=%d CUDA error %s\n", K, N, mode, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
  double num = 0, den = 0, maxrel = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += double(a[r * K + k]) * double(b[n * K + k]);
      const double err = d[r * N + n] - ref;
      num += err * err;
      den += ref * ref;
      maxrel = fmax(maxrel, fabs(err) / (fabs(ref) + 1e-12));
    }
  printf("K=%d N=%d mode=%d rel_l2=%.3e d[0]=%.6f\n", K, N, mode, sqrt(num / den), d[0]);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dd);
  return 0;
}

int main() {
  int bad = 0;
  bad |= run<8, 32>(0);
  bad |= run<8, 32>(1);
  bad |= run<8, 32>(2);
  bad |= run<32, 16>(0);
  bad |= run<32, 16>(1);
  return bad;
}
