// Probe of tcgen05 operand layouts the kernels do not use yet: MN-major
// (transposed) tf32 operands in shared memory, no swizzle, and where the rows
// of an M = 64 accumulator land in TMEM.  The host builds each operand's
// shared-memory image from a layout hypothesis, the kernel copies the images
// in and issues kind::tf32 MMAs with the given descriptors, and the host
// compares D (all 128 lanes read back) with the exact product (operands are
// small multiples of 1/8, exact in tf32, so any layout error is visible).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_layout_probe tools/umma_layout_probe.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

struct Cfg {
  int M, N, K;             // MMA shape (K = 8 per instruction; K / 8 instructions)
  int a_major, b_major;    // 0 = K-major, 1 = MN-major
  uint32_t a_lbo, a_sbo;   // descriptor fields (bytes)
  uint32_t b_lbo, b_sbo;
  uint32_t a_step, b_step; // start-address advance per K = 8 instruction (bytes)
  uint32_t a_lt = 0, b_lt = 0;  // descriptor layout type (bits 61-63): 0 none, 2 128B, 4 64B, 6 32B swizzle
};

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t lt = 0) {
  return uint64_t((addr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(lt) << 61);
}

constexpr int kImg = 4096;  // floats per operand image (16 KB)

__global__ void probe(const float* a_img, const float* b_img, float* d, Cfg c) {
  __shared__ __align__(1024) float As[kImg];
  __shared__ __align__(1024) float Bs[kImg];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < kImg; i += 128) {
    As[i] = a_img[i];
    Bs[i] = b_img[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  // zero the accumulator region first (M = 64 leaves lanes untouched)
  {
    const uint32_t lane = tmem + (uint32_t(warp * 32) << 16);
    for (int col = 0; col < 256; col += 8)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(lane + col),
                   "r"(0x7FC00000u));  // NaN marks "not written"
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if (tid == 0) {
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(c.a_major) << 15) |
                        (uint32_t(c.b_major) << 16) | (uint32_t(c.N >> 3) << 17) | (uint32_t(c.M >> 4) << 24);
    for (int ks = 0; ks < c.K / 8; ++ks) {
      const uint64_t a = desc(su32(As) + ks * c.a_step, c.a_lbo, c.a_sbo, c.a_lt);
      const uint64_t b = desc(su32(Bs) + ks * c.b_step, c.b_lbo, c.b_sbo, c.b_lt);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                   "l"(a), "l"(b), "r"(id), "r"(ks ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar))
                 : "memory");
  }
  uint32_t done = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(su32(&mbar))
                 : "memory");
  } while (!done);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t lane = tmem + (uint32_t(warp * 32) << 16);
  for (int col = 0; col < c.N; col += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(lane + col));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) d[tid * 256 + col + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// float index of element (mn, k) of an operand
static int kmajor(int mn, int k, uint32_t lbo, uint32_t sbo) {  // the layout the kernels use
  return int(((mn / 8) * sbo + (k / 4) * lbo) / 4) + (mn % 8) * 4 + (k % 4);
}
// MN-major no-swizzle hypotheses: 4 consecutive mn (16 B) x 8 k rows (stride 16 B) per core matrix
static int mnmajor(int mn, int k, uint32_t mn_stride, uint32_t k_stride) {
  return int(((mn / 4) * mn_stride + (k / 8) * k_stride) / 4) + (k % 8) * 4 + (mn % 4);
}

static float* dev(const std::vector<float>& v) {
  float* p;
  cudaMalloc(&p, v.size() * 4);
  cudaMemcpy(p, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
  return p;
}

// returns max |err| over rows found, and reports the lane map for M = 64
static double run(const char* name, Cfg c, int a_layout, int b_layout, uint32_t a_mn_stride, uint32_t a_k_stride,
                  uint32_t b_mn_stride, uint32_t b_k_stride) {
  std::vector<float> A(c.M * c.K), B(c.N * c.K);
  srand(7);
  for (auto& x : A) x = float(rand() % 17 - 8) / 8.0f;
  for (auto& x : B) x = float(rand() % 17 - 8) / 8.0f;
  std::vector<float> ai(kImg, 0.f), bi(kImg, 0.f);
  for (int m = 0; m < c.M; ++m)
    for (int k = 0; k < c.K; ++k)
      ai[a_layout ? mnmajor(m, k, a_mn_stride, a_k_stride) : kmajor(m, k, c.a_lbo, c.a_sbo)] = A[m * c.K + k];
  for (int n = 0; n < c.N; ++n)
    for (int k = 0; k < c.K; ++k)
      bi[b_layout ? mnmajor(n, k, b_mn_stride, b_k_stride) : kmajor(n, k, c.b_lbo, c.b_sbo)] = B[n * c.K + k];
  float *da = dev(ai), *db = dev(bi), *dd;
  cudaMalloc(&dd, 128 * 256 * 4);
  probe<<<1, 128>>>(da, db, dd, c);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("%-44s CUDA error %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  std::vector<float> D(128 * 256);
  cudaMemcpy(D.data(), dd, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dd);
  // match each logical row m to the TMEM lane holding it
  double worst = 0;
  int lane_of[128];
  for (int m = 0; m < c.M; ++m) {
    lane_of[m] = -1;
    double best = 1e30;
    for (int l = 0; l < 128; ++l) {
      double err = 0;
      for (int n = 0; n < c.N; ++n) {
        double ref = 0;
        for (int k = 0; k < c.K; ++k) ref += double(A[m * c.K + k]) * double(B[n * c.K + k]);
        const double v = D[l * 256 + n];
        err = fmax(err, std::isnan(v) ? 1e9 : fabs(v - ref));
      }
      if (err < best) {
        best = err;
        lane_of[m] = l;
      }
    }
    worst = fmax(worst, best);
  }
  printf("%-44s max|err| %.3g", name, worst);
  if (c.M == 64) {
    printf("  lanes:");
    for (int m = 0; m < 64; m += 8) printf(" %d->%d", m, lane_of[m]);
  } else {
    int identity = 1;
    for (int m = 0; m < c.M; ++m) identity &= lane_of[m] == m;
    printf("  rows on lanes %s", identity ? "0..127 in order" : "PERMUTED");
  }
  printf("\n");
  return worst;
}


// Discovery: one-hot operand images.  For each float position p of the
// MN-major operand image, set that float to 1 (the other operand holds k + 1
// in every row), run the MMA and read which (mn, k) the hardware took it for.
static void discover(const char* name, int which, uint32_t lbo, uint32_t sbo, int positions, uint32_t lt = 0) {
  Cfg c{128, 32, 8, which == 0, which == 1, 128, 256, 128, 256, 0, 0};
  const bool ctl = which == 2;
  if (ctl) which = 1;
  if (which == 0) { c.a_lbo = lbo; c.a_sbo = sbo; c.a_lt = lt; } else { c.b_lbo = lbo; c.b_sbo = sbo; c.b_lt = lt; }
  std::vector<float> other(kImg, 0.f), hot(kImg, 0.f);
  const int other_rows = which == 0 ? c.N : c.M;
  for (int r = 0; r < other_rows; ++r)
    for (int k = 0; k < 8; ++k) other[kmajor(r, k, 128, 256)] = float(k + 1);
  float *dothr = dev(other), *dhot, *dd;
  cudaMalloc(&dhot, kImg * 4);
  cudaMalloc(&dd, 128 * 256 * 4);
  std::vector<float> D(128 * 256);
  printf("%s (LBO %u, SBO %u, layout %u):", name, lbo, sbo, lt);
  int shown = 0;
  for (int p = 0; p < positions; ++p) {
    std::fill(hot.begin(), hot.end(), 0.f);
    hot[p] = 1.f;
    cudaMemcpy(dhot, hot.data(), kImg * 4, cudaMemcpyHostToDevice);
    if (which == 0) probe<<<1, 128>>>(dhot, dothr, dd, c);
    else probe<<<1, 128>>>(dothr, dhot, dd, c);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf(" error\n"); exit(1); }
    cudaMemcpy(D.data(), dd, D.size() * 4, cudaMemcpyDeviceToHost);
    int hits = 0, mn = -1, k = -1;
    for (int l = 0; l < 128; ++l)
      for (int n = 0; n < c.N; ++n) {
        const float v = D[l * 256 + n];
        if (v != 0.f && !std::isnan(v)) { ++hits; mn = which == 0 ? l : n; k = int(v) - 1; }
      }
    if (hits != 0 && shown++ < 64) printf(" %d:(%d,%d)%s", p, mn, k, (which == 0 ? hits != c.N : hits != 128) ? "?" : "");
  }
  printf("\n");
  cudaFree(dothr); cudaFree(dhot); cudaFree(dd);
}

int main() {
  // reference: both K-major (as the kernels), M = 128, N = 32, K = 16
  Cfg c{128, 32, 16, 0, 0, 128, 128 * 4, 128, 128 * 4, 256, 256};
  run("K-major A, K-major B (kernels' layout)", c, 0, 0, 0, 0, 0, 0);
  // MN-major B (N = 32, K = 16): mn groups of 4 at stride X, k groups of 8 at stride Y
  // hypothesis 1: SBO field = mn-group stride, LBO field = k-group stride
  {
    const uint32_t mn_stride = 128, k_stride = 128 * (32 / 4);  // mn groups contiguous, then next 8 k
    Cfg h = c;
    h.b_major = 1;
    h.b_sbo = mn_stride;
    h.b_lbo = k_stride;
    h.b_step = k_stride;
    run("MN-major B, SBO=mn stride, LBO=k stride", h, 0, 1, 0, 0, mn_stride, k_stride);
    h.b_sbo = k_stride;
    h.b_lbo = mn_stride;
    run("MN-major B, LBO=mn stride, SBO=k stride", h, 0, 1, 0, 0, mn_stride, k_stride);
    // k groups contiguous, then next mn group
    const uint32_t mn2 = 128 * (16 / 8), k2 = 128;
    h.b_sbo = mn2;
    h.b_lbo = k2;
    h.b_step = k2;
    run("MN-major B (k-fast), SBO=mn stride, LBO=k", h, 0, 1, 0, 0, mn2, k2);
    h.b_sbo = k2;
    h.b_lbo = mn2;
    run("MN-major B (k-fast), LBO=mn stride, SBO=k", h, 0, 1, 0, 0, mn2, k2);
  }
  // MN-major A (M = 128, K = 16)
  {
    const uint32_t mn_stride = 128, k_stride = 128 * (128 / 4);
    Cfg h = c;
    h.a_major = 1;
    h.a_sbo = mn_stride;
    h.a_lbo = k_stride;
    h.a_step = k_stride;
    run("MN-major A, SBO=mn stride, LBO=k stride", h, 1, 0, mn_stride, k_stride, 0, 0);
    h.a_sbo = k_stride;
    h.a_lbo = mn_stride;
    run("MN-major A, LBO=mn stride, SBO=k stride", h, 1, 0, mn_stride, k_stride, 0, 0);
  }
  // M = 64 accumulator lane map (K-major operands)
  {
    Cfg h{64, 32, 16, 0, 0, 128, 128 * 4, 128, 128 * 4, 256, 256};
    run("M=64 K-major", h, 0, 0, 0, 0, 0, 0);
  }
  discover("B K-major (control)", 2, 128, 256, 512);
  for (uint32_t lt : {0u, 6u, 4u, 2u}) {
    discover("B MN-major", 1, 128, 1024, 4096, lt);
    discover("B MN-major", 1, 1024, 128, 4096, lt);
  }
  discover("A MN-major", 0, 128, 1024, 4096, 0);
  discover("A MN-major", 0, 4096, 128, 4096, 0);
  return 0;
}
