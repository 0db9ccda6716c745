// Design probe 6: which CUDA calls of a proxy thread block while the user
// thread sits in a synchronous pageable cudaMemcpy behind a stream parked on
// a stream-memory wait (the deadlock found by test_pair_sendrecv_bytes), and
// copy-engine pull vs push bandwidth over NVLink.  Not part of the product.
#include <cuda.h>
#include <cuda_runtime.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
#define CKD(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  fprintf(stderr, "CU %s at %s:%d: %s\n", #x, __FILE__, __LINE__, s_); exit(1);} } while (0)

static double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

__global__ void noop_kernel(int* p) { if (p) p[0] = 1; }

int main() {
  CKD(cuInit(0));
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaSetDevice(0));
  volatile uint32_t* hf;
  CK(cudaHostAlloc((void**)&hf, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  memset((void*)hf, 0, 4096);
  char *d0, *d0b, *d1;
  const size_t big = 64 << 20;
  CK(cudaMalloc(&d0, big));
  CK(cudaMalloc(&d0b, big));
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&d1, big));
  CK(cudaSetDevice(0));
  std::vector<char> pageable(3 << 20, 1);
  cudaStream_t user, proxy;
  CK(cudaStreamCreateWithFlags(&user, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&proxy, cudaStreamNonBlocking));
  noop_kernel<<<1, 1, 0, proxy>>>(nullptr);
  CK(cudaDeviceSynchronize());
  printf("# 1. proxy call latency while the user thread is in a pageable 3 MiB H2D behind a parked stream\n");
  const char* names[] = {"cuMemcpyDtoDAsync peer", "cuMemcpyDtoDAsync local", "kernel launch", "cuStreamWaitValue32",
                         "cudaEventRecord", "cudaMemcpyAsync H2D pinned"};
  for (int which = 0; which < 6; which++) {
    hf[0] = 0;
    CKD(cuStreamWaitValue32((CUstream)user, (CUdeviceptr)hf, 1, CU_STREAM_WAIT_VALUE_GEQ));
    std::atomic<int> in_memcpy{0};
    std::thread t([&] {
      cudaSetDevice(0);
      in_memcpy = 1;
      cudaMemcpyAsync(d0, pageable.data(), pageable.size(), cudaMemcpyHostToDevice, user);  // pageable: synchronous
      in_memcpy = 2;
    });
    while (in_memcpy.load() == 0) std::this_thread::yield();
    std::this_thread::sleep_for(std::chrono::milliseconds(50));
    std::atomic<int> done{0};
    double t0 = now_s(), t1 = 0;
    std::thread p([&] {
      cudaSetDevice(0);
      cudaEvent_t ev;
      cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      switch (which) {
        case 0: cuMemcpyDtoDAsync((CUdeviceptr)d1, (CUdeviceptr)d0b, 1 << 20, (CUstream)proxy); break;
        case 1: cuMemcpyDtoDAsync((CUdeviceptr)d0, (CUdeviceptr)d0b, 1 << 20, (CUstream)proxy); break;
        case 2: noop_kernel<<<1, 1, 0, proxy>>>(nullptr); break;
        case 3: cuStreamWaitValue32((CUstream)proxy, (CUdeviceptr)(hf + 16), 0, CU_STREAM_WAIT_VALUE_GEQ); break;
        case 4: cudaEventRecord(ev, proxy); break;
        case 5: cudaMemcpyAsync(d0b, (const void*)(hf + 64), 64, cudaMemcpyHostToDevice, proxy); break;
      }
      t1 = now_s();
      done = 1;
    });
    // release the parked stream after 1 s if the proxy call is stuck
    double deadline = now_s() + 1.0;
    while (!done.load() && now_s() < deadline) std::this_thread::yield();
    bool blocked = !done.load();
    hf[0] = 1;
    p.join();
    t.join();
    CK(cudaDeviceSynchronize());
    printf("  %-28s %s (%.1f us)\n", names[which], blocked ? "BLOCKED until the user memcpy finished" : "returned",
           (t1 - t0) * 1e6);
    fflush(stdout);
  }
  printf("# 2. copy-engine push (stream on GPU0 writes GPU1) vs pull (stream on GPU1 reads GPU0), 64 MiB x 8\n");
  for (int dir = 0; dir < 2; dir++) {
    cudaStream_t s;
    int dev = dir == 0 ? 0 : 1;
    CK(cudaSetDevice(dev));
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e9;
    for (int rep = 0; rep < 5; rep++) {
      CK(cudaEventRecord(a, s));
      for (int k = 0; k < 8; k++) CK(cudaMemcpyAsync(d1, d0, big, cudaMemcpyDefault, s));
      CK(cudaEventRecord(b, s));
      CK(cudaEventSynchronize(b));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    printf("  %s: %.1f GB/s\n", dir == 0 ? "push" : "pull", 8.0 * big / (best * 1e-3) / 1e9);
    fflush(stdout);
  }
  return 0;
}
