// Design probe 5: flag placement for the memop chain: separates CPU enqueue cost from GPU
// copy-engine cost by pre-enqueueing work behind a host-flag gate, measures
// CE concurrency across streams, SM pull vs push, and the latency chains.
// Single process, 2 GPUs with peer access. Not part of the product.
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <unistd.h>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
#define CKD(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  fprintf(stderr, "CU %s at %s:%d: %s\n", #x, __FILE__, __LINE__, s_); exit(1);} } while (0)

static const size_t MiB = 1ull << 20;
static double now_s() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
static double T0;
#define SECTION(name) printf("\n# [%.1fs] %s\n", now_s() - T0, name); fflush(stdout)

template <int U>
__global__ void copy_ldst(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = tid;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++)
      asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; u++) dst[i + u * stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

// block-contiguous variant: each CTA copies one contiguous slab
template <int U>
__global__ void copy_slab(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t per = (n16 + gridDim.x - 1) / gridDim.x;
  size_t b = blockIdx.x * per, e = min(n16, b + per);
  for (size_t i = b + threadIdx.x; i < e; i += (size_t)U * blockDim.x) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < e) asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                              : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + j));
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      size_t j = i + (size_t)u * blockDim.x;
      if (j < e) dst[j] = v[u];
    }
  }
}

__global__ void pingpong_kernel(volatile uint32_t* my_flag, volatile uint32_t* peer_flag, int iters, int initiator,
                                unsigned long long* out_ns) {
  uint64_t t0, t1, tl;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; i++) {
    if (initiator) asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(peer_flag), "r"(i) : "memory");
    uint32_t v = 0;
    do { asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flag) : "memory");
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl));
      if (tl - t0 > 2000000000ull) return; } while ((int)(v - i) < 0);
    if (!initiator) asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(peer_flag), "r"(i) : "memory");
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (initiator) *out_ns = t1 - t0;
}

static float ev_ms(cudaEvent_t a, cudaEvent_t b) { float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }




__global__ void stamp_kernel(unsigned long long* p) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); *p = t; }

// probe 5: flag placement for the stream-memop synchronisation chain
int main(int argc, char** argv) {
  T0 = now_s();
  CKD(cuInit(0));
  int ndev; CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));
  cudaStream_t s0, s1; cudaEvent_t a, b;
  CK(cudaSetDevice(0)); CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking)); CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  CK(cudaSetDevice(1)); CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  uint32_t* hf; CK(cudaHostAlloc(&hf, 1 << 16, cudaHostAllocMapped | cudaHostAllocPortable)); memset(hf, 0, 1 << 16);
  uint32_t *d0, *d1;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&d0, 4096)); CK(cudaMemset(d0, 0, 4096));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&d1, 4096)); CK(cudaMemset(d1, 0, 4096));
  CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
  // fA: GPU0 -> GPU1 signal, fB: GPU1 -> GPU0 signal
  struct Cfg { const char* name; CUdeviceptr fA, fB; };
  Cfg cfgs[] = {{"host flags", (CUdeviceptr)(hf + 64), (CUdeviceptr)(hf + 128)},
                {"device flags, peer write + local wait", (CUdeviceptr)(d1 + 0), (CUdeviceptr)(d0 + 0)},
                {"device flags, local write + remote wait", (CUdeviceptr)(d0 + 64), (CUdeviceptr)(d1 + 64)}};
  SECTION("1. memop ping-pong one-way (us)");
  for (auto& cf : cfgs) {
    CK(cudaSetDevice(0)); CK(cudaMemset(d0, 0, 4096)); CK(cudaSetDevice(1)); CK(cudaMemset(d1, 0, 4096));
    memset(hf, 0, 4096); CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    const int N = 300;
    CK(cudaEventRecord(a, s0));
    for (int i = 1; i <= N; i++) {
      CK(cudaSetDevice(0));
      CKD(cuStreamWriteValue32((CUstream)s0, cf.fA, i, 0));
      CKD(cuStreamWaitValue32((CUstream)s0, cf.fB, i, CU_STREAM_WAIT_VALUE_GEQ));
      if (i == N) CK(cudaEventRecord(b, s0));
      CK(cudaSetDevice(1));
      CKD(cuStreamWaitValue32((CUstream)s1, cf.fA, i, CU_STREAM_WAIT_VALUE_GEQ));
      CKD(cuStreamWriteValue32((CUstream)s1, cf.fB, i, 0));
    }
    CK(cudaSetDevice(0)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    printf("  %s: %.2f us\n", cf.name, ms * 1e3 / N / 2); fflush(stdout);
  }
  SECTION("2. same ping-pong with a 1-thread kernel after each wait (kernel launch latency behind a memop)");
  unsigned long long* ts0; unsigned long long* ts1;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&ts0, 64)); CK(cudaSetDevice(1)); CK(cudaMalloc(&ts1, 64));
  stamp_kernel<<<1, 1, 0, s1>>>(ts1); CK(cudaSetDevice(0)); stamp_kernel<<<1, 1, 0, s0>>>(ts0); CK(cudaDeviceSynchronize());
  for (auto& cf : cfgs) {
    CK(cudaSetDevice(0)); CK(cudaMemset(d0, 0, 4096)); CK(cudaSetDevice(1)); CK(cudaMemset(d1, 0, 4096));
    memset(hf, 0, 4096); CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    const int N = 300;
    CK(cudaEventRecord(a, s0));
    for (int i = 1; i <= N; i++) {
      CK(cudaSetDevice(0));
      CKD(cuStreamWriteValue32((CUstream)s0, cf.fA, i, 0));
      CKD(cuStreamWaitValue32((CUstream)s0, cf.fB, i, CU_STREAM_WAIT_VALUE_GEQ));
      stamp_kernel<<<1, 1, 0, s0>>>(ts0);
      if (i == N) CK(cudaEventRecord(b, s0));
      CK(cudaSetDevice(1));
      CKD(cuStreamWaitValue32((CUstream)s1, cf.fA, i, CU_STREAM_WAIT_VALUE_GEQ));
      stamp_kernel<<<1, 1, 0, s1>>>(ts1);
      CKD(cuStreamWriteValue32((CUstream)s1, cf.fB, i, 0));
    }
    CK(cudaSetDevice(0)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    printf("  %s: %.2f us\n", cf.name, ms * 1e3 / N / 2); fflush(stdout);
  }
  SECTION("3. one CE 64 MiB copy between stream ops: bare / +event / +stamp kernels (us)");
  char *x0, *x1; CK(cudaSetDevice(0)); CK(cudaMalloc(&x0, 64 << 20)); CK(cudaSetDevice(1)); CK(cudaMalloc(&x1, 64 << 20)); CK(cudaSetDevice(0));
  for (int mode = 0; mode < 3; mode++) {
    std::vector<double> v;
    for (int rep = 0; rep < 12; rep++) {
      CK(cudaEventRecord(a, s0));
      for (int k = 0; k < 4; k++) {
        if (mode == 2) stamp_kernel<<<1, 1, 0, s0>>>(ts0);
        CK(cudaMemcpyAsync(x1, x0, 64 << 20, cudaMemcpyDefault, s0));
        if (mode == 1) CK(cudaEventRecord(b, s0));
        if (mode == 2) stamp_kernel<<<1, 1, 0, s0>>>(ts0 + 1);
      }
      CK(cudaEventRecord(b, s0)); CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (rep > 1) v.push_back(ms * 1e3 / 4);
    }
    std::sort(v.begin(), v.end());
    printf("  mode %d: %.1f us per 64 MiB copy (%.1f GB/s)\n", mode, v[v.size() / 2], (64 << 20) / v[v.size() / 2] / 1e3); fflush(stdout);
  }
  SECTION("4. full op chain one-way (us): user WriteValue(ready) x2 -> copy stream waits both, CE copy, WriteValue(done) x2 -> user waits done");
  {
    cudaStream_t c0, c1;
    CK(cudaSetDevice(0)); CK(cudaStreamCreateWithFlags(&c0, cudaStreamNonBlocking));
    CK(cudaSetDevice(1)); CK(cudaStreamCreateWithFlags(&c1, cudaStreamNonBlocking));
    char *b0, *b1; CK(cudaSetDevice(0)); CK(cudaMalloc(&b0, 1 << 20)); CK(cudaSetDevice(1)); CK(cudaMalloc(&b1, 1 << 20));
    // flags: r0 r1 (ready of rank0/1 for the current op), e0 e1 (done)
    struct Pl { const char* name; CUdeviceptr r0, r1, e0, e1; };
    Pl pls[] = {{"host flags", (CUdeviceptr)(hf + 256), (CUdeviceptr)(hf + 320), (CUdeviceptr)(hf + 384), (CUdeviceptr)(hf + 448)},
                {"device flags (owner-local)", (CUdeviceptr)(d0 + 256), (CUdeviceptr)(d1 + 256), (CUdeviceptr)(d0 + 320), (CUdeviceptr)(d1 + 320)}};
    for (size_t sz : {(size_t)8, (size_t)65536, (size_t)1 << 20}) {
      for (auto& pl : pls) {
        CK(cudaSetDevice(0)); CK(cudaMemset(d0, 0, 4096)); CK(cudaSetDevice(1)); CK(cudaMemset(d1, 0, 4096));
        memset(hf, 0, 4096); CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
        const int N = 200;
        CK(cudaEventRecord(a, s0));
        uint32_t g = 0;
        for (int i = 1; i <= N; i++) {
          for (int dir = 0; dir < 2; dir++) {  // 0: 0->1 copy by c0, 1: 1->0 copy by c1
            g++;
            CK(cudaSetDevice(0)); CKD(cuStreamWriteValue32((CUstream)s0, pl.r0, g, 0));
            CK(cudaSetDevice(1)); CKD(cuStreamWriteValue32((CUstream)s1, pl.r1, g, 0));
            int d = dir == 0 ? 0 : 1;
            cudaStream_t cs = d == 0 ? c0 : c1;
            CK(cudaSetDevice(d));
            CKD(cuStreamWaitValue32((CUstream)cs, pl.r0, g, CU_STREAM_WAIT_VALUE_GEQ));
            CKD(cuStreamWaitValue32((CUstream)cs, pl.r1, g, CU_STREAM_WAIT_VALUE_GEQ));
            CK(cudaMemcpyAsync(d == 0 ? b1 : b0, d == 0 ? b0 : b1, sz, cudaMemcpyDefault, cs));
            CKD(cuStreamWriteValue32((CUstream)cs, pl.e1, g, 0));
            CKD(cuStreamWriteValue32((CUstream)cs, pl.e0, g, 0));
            CK(cudaSetDevice(0)); CKD(cuStreamWaitValue32((CUstream)s0, pl.e0, g, CU_STREAM_WAIT_VALUE_GEQ));
            CK(cudaSetDevice(1)); CKD(cuStreamWaitValue32((CUstream)s1, pl.e1, g, CU_STREAM_WAIT_VALUE_GEQ));
          }
          if (i == N) { CK(cudaSetDevice(0)); CK(cudaEventRecord(b, s0)); }
        }
        CK(cudaSetDevice(0)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        printf("  %zu B %s: %.2f us per op\n", sz, pl.name, ms * 1e3 / N / 2); fflush(stdout);
      }
    }
  }
  SECTION("5. 16 x 8 MiB peer copies on one stream: bare / untimed event / timed event between copies (us per copy)");
  {
    char *y0, *y1; CK(cudaSetDevice(0)); CK(cudaMalloc(&y0, 128 << 20)); CK(cudaSetDevice(1)); CK(cudaMalloc(&y1, 128 << 20)); CK(cudaSetDevice(0));
    cudaEvent_t ut[16], tt[16];
    for (int i = 0; i < 16; i++) { CK(cudaEventCreateWithFlags(&ut[i], cudaEventDisableTiming)); CK(cudaEventCreate(&tt[i])); }
    for (int mode = 0; mode < 3; mode++) {
      std::vector<double> v;
      for (int rep = 0; rep < 10; rep++) {
        CK(cudaEventRecord(a, s0));
        for (int k = 0; k < 16; k++) {
          CK(cudaMemcpyAsync(y1 + ((size_t)k << 23), y0 + ((size_t)k << 23), 8 << 20, cudaMemcpyDefault, s0));
          if (mode == 1) CK(cudaEventRecord(ut[k], s0));
          if (mode == 2) CK(cudaEventRecord(tt[k], s0));
        }
        CK(cudaEventRecord(b, s0)); CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (rep > 1) v.push_back(ms * 1e3 / 16);
      }
      std::sort(v.begin(), v.end());
      printf("  mode %d: %.2f us per 8 MiB copy (%.1f GB/s)\n", mode, v[v.size() / 2], (8 << 20) / v[v.size() / 2] / 1e3); fflush(stdout);
    }
  }
  SECTION("done");
  return 0;
}
