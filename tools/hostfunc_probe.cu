// Latency of the two ways a copy stream can wait for host-side file I/O:
// (1) cudaLaunchHostFunc (the host function runs the I/O in stream order),
// (2) a host thread doing the I/O and releasing the stream through a
//     stream memory operation (cuStreamWaitValue32 on pinned host memory).
// Prints median microseconds between events bracketing the wait.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>

static void CUDART_CB nop(void*) {}

__global__ void spin(int64_t cycles) {
  const int64_t t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

int main() {
  cudaSetDevice(0);
  cudaStream_t s, c;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 50;
  std::vector<float> v;
  // (1) host function latency with the stream idle before it
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(e0, s);
    cudaLaunchHostFunc(s, nop, nullptr);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    v.push_back(ms * 1e3f);
  }
  std::sort(v.begin(), v.end());
  std::printf("hostfunc idle: median %.1f us, min %.1f, max %.1f\n", v[v.size() / 2], v[0], v.back());
  // (1b) host function behind a kernel on another busy stream, host thread enqueuing meanwhile
  v.clear();
  for (int i = 0; i < reps; ++i) {
    spin<<<1, 32, 0, c>>>(200000);
    spin<<<1, 32, 0, s>>>(20000);
    cudaEventRecord(e0, s);
    cudaLaunchHostFunc(s, nop, nullptr);
    cudaEventRecord(e1, s);
    for (int k = 0; k < 50; ++k) spin<<<1, 32, 0, c>>>(2000);
    cudaEventSynchronize(e1);
    cudaStreamSynchronize(c);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    v.push_back(ms * 1e3f);
  }
  std::sort(v.begin(), v.end());
  std::printf("hostfunc busy: median %.1f us, min %.1f, max %.1f\n", v[v.size() / 2], v[0], v.back());
  // (2) stream memory op released by a host thread
  cuInit(0);
  int ok = 0;
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  cuDeviceGetAttribute(&ok, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, &dev == nullptr ? 0 : dev);
  int memops = 0;
  cuDeviceGetAttribute(&memops, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, dev);
  std::printf("stream mem ops: wait_value_nor=%d 64bit=%d\n", ok, memops);
  uint32_t* flag = nullptr;
  cudaHostAlloc(reinterpret_cast<void**>(&flag), 64, cudaHostAllocMapped);
  CUdeviceptr dflag;
  cuMemHostGetDevicePointer(&dflag, flag, 0);
  v.clear();
  std::vector<float> hv;
  for (int i = 1; i <= reps; ++i) {
    std::atomic<bool> go{false};
    std::chrono::steady_clock::time_point tw;
    std::thread th([&] {
      while (!go.load()) {
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
      tw = std::chrono::steady_clock::now();
      __atomic_store_n(flag, uint32_t(i), __ATOMIC_RELEASE);
    });
    cudaEventRecord(e0, s);
    CUresult r = cuStreamWaitValue32(reinterpret_cast<CUstream>(s), dflag, uint32_t(i), CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) {
      std::printf("cuStreamWaitValue32 failed: %d\n", int(r));
      go = true;
      th.join();
      return 1;
    }
    cudaEventRecord(e1, s);
    go = true;
    cudaEventSynchronize(e1);
    const auto tdone = std::chrono::steady_clock::now();
    th.join();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    v.push_back(ms * 1e3f);
    hv.push_back(std::chrono::duration<float, std::micro>(tdone - tw).count());
  }
  std::sort(v.begin(), v.end());
  std::sort(hv.begin(), hv.end());
  std::printf("wait_value (50 us host work): stream wait median %.1f us; flag->host-observed done median %.1f us\n",
              v[v.size() / 2], hv[hv.size() / 2]);
  return 0;
}
