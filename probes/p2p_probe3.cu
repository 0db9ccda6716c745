// Design probe 3 (see p2p_probe.cu, p2p_probe2.cu): separates CPU enqueue cost from GPU
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


// time from the first stream's post-gate event to the joined end
int main() {
  T0 = now_s();
  CKD(cuInit(0));
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));
  const size_t MAXB = 1024 * MiB;
  char *b0, *b1, *c0, *c1;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&b0, MAXB)); CK(cudaMalloc(&c0, MAXB)); CK(cudaMemset(b0, 1, MAXB));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&b1, MAXB)); CK(cudaMalloc(&c1, MAXB)); CK(cudaMemset(b1, 2, MAXB));
  const int NS = 8;
  cudaStream_t s0[NS], s1[NS];
  cudaEvent_t es[NS], ee[NS], e1a, e1b;
  CK(cudaSetDevice(0)); for (int i = 0; i < NS; i++) { CK(cudaStreamCreateWithFlags(&s0[i], cudaStreamNonBlocking)); CK(cudaEventCreate(&es[i])); CK(cudaEventCreate(&ee[i])); }
  CK(cudaSetDevice(1)); for (int i = 0; i < NS; i++) CK(cudaStreamCreateWithFlags(&s1[i], cudaStreamNonBlocking));
  CK(cudaEventCreate(&e1a)); CK(cudaEventCreate(&e1b));
  uint32_t* hf; CK(cudaHostAlloc(&hf, 1 << 16, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(hf, 0, 1 << 16);
  CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
  uint32_t gate_val = 0;
  // every stream records es[k] after the gate and ee[k] at its end; time = max(ee) - min(es)
  auto gated = [&](int S, auto enqueue) {
    gate_val++;
    CK(cudaSetDevice(0));
    for (int k = 0; k < S; k++) { CKD(cuStreamWaitValue32((CUstream)s0[k], (CUdeviceptr)(hf), gate_val, CU_STREAM_WAIT_VALUE_GEQ)); CK(cudaEventRecord(es[k], s0[k])); }
    enqueue();
    for (int k = 0; k < S; k++) CK(cudaEventRecord(ee[k], s0[k]));
    usleep(200);
    __atomic_store_n(hf, gate_val, __ATOMIC_SEQ_CST);
    for (int k = 0; k < S; k++) CK(cudaEventSynchronize(ee[k]));
    float lo = 1e30f, hi = -1e30f;
    for (int k = 0; k < S; k++) { float a, b; CK(cudaEventElapsedTime(&a, es[0], es[k])); CK(cudaEventElapsedTime(&b, es[0], ee[k])); lo = std::min(lo, a); hi = std::max(hi, b); }
    return (double)(hi - lo) * 1e3;
  };
  SECTION("B. GPU-only chunked CE push: total chunkMiB S wv us GB/s");
  for (size_t tot : {64 * MiB, 256 * MiB}) {
    for (size_t ch : {2 * MiB, 4 * MiB, 8 * MiB, 16 * MiB, 32 * MiB, 64 * MiB}) {
      if (ch > tot) continue;
      for (int S : {1, 2, 4}) {
        for (int wv = 0; wv < 2; wv++) {
          auto enq = [&]() {
            size_t nch = tot / ch;
            for (size_t c = 0; c < nch; c++) {
              CK(cudaMemcpyAsync(b1 + c * ch, b0 + c * ch, ch, cudaMemcpyDefault, s0[c % S]));
              if (wv) CKD(cuStreamWriteValue32((CUstream)s0[c % S], (CUdeviceptr)(hf + 64 + 16 * (c % S)), (uint32_t)c, 0));
            }
          };
          gated(S, enq);
          std::vector<double> v; for (int r = 0; r < 5; r++) v.push_back(gated(S, enq));
          std::sort(v.begin(), v.end());
          printf("%zu %zu %d %d %.1f %.1f\n", tot / MiB, ch / MiB, S, wv, v[2], tot / v[2] / 1e3);
        }
      }
    }
  }
  SECTION("C. one copy split across S streams: total S us GB/s");
  for (size_t tot : {16 * MiB, 64 * MiB, 256 * MiB, 1024 * MiB}) {
    for (int S : {1, 2, 3, 4}) {
      auto enq = [&]() { size_t part = tot / S; for (int k = 0; k < S; k++) CK(cudaMemcpyAsync(b1 + k * part, b0 + k * part, part, cudaMemcpyDefault, s0[k])); };
      gated(S, enq);
      std::vector<double> v; for (int r = 0; r < 5; r++) v.push_back(gated(S, enq));
      std::sort(v.begin(), v.end());
      printf("%zu %d %.1f %.1f\n", tot / MiB, S, v[2], tot / v[2] / 1e3);
    }
  }
  SECTION("C3. CE + SM pull-free push split: total frac_sm ctas us GB/s");
  for (size_t tot : {64 * MiB, 256 * MiB}) {
    for (double f : {0.0, 0.1, 0.2, 0.3, 0.5}) {
      for (int ctas : {16, 32}) {
        size_t nsm = ((size_t)(tot * f)) & ~(size_t)4095;
        auto enq = [&]() {
          if (tot - nsm) CK(cudaMemcpyAsync(b1, b0, tot - nsm, cudaMemcpyDefault, s0[0]));
          if (nsm) copy_ldst<4><<<ctas, 512, 0, s0[1]>>>((const int4*)(b0 + tot - nsm), (int4*)(b1 + tot - nsm), nsm / 16);
        };
        gated(2, enq);
        std::vector<double> v; for (int r = 0; r < 5; r++) v.push_back(gated(2, enq));
        std::sort(v.begin(), v.end());
        printf("%zu %.1f %d %.1f %.1f\n", tot / MiB, f, ctas, v[2], tot / v[2] / 1e3);
      }
    }
  }
  SECTION("E0. memop wait reaction vs idle time: idle_us reaction_us (host write -> GPU write seen by host)");
  for (int idle : {0, 10, 100, 1000, 10000, 50000}) {
    std::vector<double> v;
    for (int rep = 0; rep < 9; rep++) {
      hf[2000] = 0; hf[2016] = 0;
      CK(cudaSetDevice(0));
      CKD(cuStreamWaitValue32((CUstream)s0[0], (CUdeviceptr)(hf + 2000), 1, CU_STREAM_WAIT_VALUE_GEQ));
      CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)(hf + 2016), 1, 0));
      double t = now_s();
      while (now_s() - t < idle * 1e-6) {}
      t = now_s();
      __atomic_store_n(hf + 2000, 1u, __ATOMIC_SEQ_CST);
      while (__atomic_load_n(hf + 2016, __ATOMIC_ACQUIRE) != 1) {}
      v.push_back((now_s() - t) * 1e6);
      CK(cudaStreamSynchronize(s0[0]));
    }
    std::sort(v.begin(), v.end());
    printf("%d %.2f (min %.2f max %.2f)\n", idle, v[4], v[0], v[8]);
  }
  SECTION("E1. host->GPU->host round trip through a copy: bytes us");
  for (size_t sz : {8ul, 4096ul, 65536ul}) {
    std::vector<double> v;
    for (int rep = 0; rep < 21; rep++) {
      hf[2000] = 0; hf[2016] = 0;
      CKD(cuStreamWaitValue32((CUstream)s0[0], (CUdeviceptr)(hf + 2000), 1, CU_STREAM_WAIT_VALUE_GEQ));
      CK(cudaMemcpyAsync(b1, b0, sz, cudaMemcpyDefault, s0[0]));
      CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)(hf + 2016), 1, 0));
      usleep(100);
      double t = now_s();
      __atomic_store_n(hf + 2000, 1u, __ATOMIC_SEQ_CST);
      while (__atomic_load_n(hf + 2016, __ATOMIC_ACQUIRE) != 1) {}
      v.push_back((now_s() - t) * 1e6);
      CK(cudaStreamSynchronize(s0[0]));
    }
    std::sort(v.begin(), v.end());
    printf("CE %zu B: %.2f us (min %.2f)\n", sz, v[10], v[0]);
    v.clear();
    for (int rep = 0; rep < 21; rep++) {
      hf[2000] = 0; hf[2016] = 0;
      CKD(cuStreamWaitValue32((CUstream)s0[0], (CUdeviceptr)(hf + 2000), 1, CU_STREAM_WAIT_VALUE_GEQ));
      copy_ldst<4><<<1, 512, 0, s0[0]>>>((const int4*)b0, (int4*)b1, sz / 16);
      CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)(hf + 2016), 1, 0));
      usleep(100);
      double t = now_s();
      __atomic_store_n(hf + 2000, 1u, __ATOMIC_SEQ_CST);
      while (__atomic_load_n(hf + 2016, __ATOMIC_ACQUIRE) != 1) {}
      v.push_back((now_s() - t) * 1e6);
      CK(cudaStreamSynchronize(s0[0]));
    }
    std::sort(v.begin(), v.end());
    printf("SM %zu B: %.2f us (min %.2f)\n", sz, v[10], v[0]);
  }
  SECTION("E2. interleaved ping-pongs (one-way us)");
  CUdeviceptr fA = (CUdeviceptr)(hf + 1024), fB = (CUdeviceptr)(hf + 1040);
  for (int mode = 0; mode < 3; mode++) {
    for (size_t sz : {8ul, 65536ul}) {
      if (mode == 0 && sz > 8) continue;
      hf[1024] = 0; hf[1040] = 0;
      const int N = 500;
      CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0)); CK(cudaEventRecord(es[0], s0[0]));
      for (int i = 1; i <= N; i++) {
        CK(cudaSetDevice(0));
        if (mode == 1) CK(cudaMemcpyAsync(c1, b0, sz, cudaMemcpyDefault, s0[0]));
        if (mode == 2) copy_ldst<4><<<1, 512, 0, s0[0]>>>((const int4*)b0, (int4*)c1, sz / 16);
        CKD(cuStreamWriteValue32((CUstream)s0[0], fA, i, 0));
        CKD(cuStreamWaitValue32((CUstream)s0[0], fB, i, CU_STREAM_WAIT_VALUE_GEQ));
        if (i == N) CK(cudaEventRecord(ee[0], s0[0]));
        CK(cudaSetDevice(1));
        CKD(cuStreamWaitValue32((CUstream)s1[0], fA, i, CU_STREAM_WAIT_VALUE_GEQ));
        if (mode == 1) CK(cudaMemcpyAsync(c0, b1, sz, cudaMemcpyDefault, s1[0]));
        if (mode == 2) copy_ldst<4><<<1, 512, 0, s1[0]>>>((const int4*)b1, (int4*)c0, sz / 16);
        CKD(cuStreamWriteValue32((CUstream)s1[0], fB, i, 0));
      }
      CK(cudaSetDevice(0)); CK(cudaEventSynchronize(ee[0]));
      float ms; CK(cudaEventElapsedTime(&ms, es[0], ee[0]));
      printf("%s %zu B: one-way %.2f us\n", mode == 0 ? "memop-only" : (mode == 1 ? "CE+memop" : "SM1cta+memop"), sz, ms * 1e3 / N / 2);
    }
  }
  {
    uint32_t *d0f, *d1f;
    CK(cudaSetDevice(0)); CK(cudaMalloc(&d0f, 256)); CK(cudaMemset(d0f, 0, 256));
    CK(cudaSetDevice(1)); CK(cudaMalloc(&d1f, 256)); CK(cudaMemset(d1f, 0, 256));
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    unsigned long long* ons; CK(cudaHostAlloc(&ons, 8, cudaHostAllocMapped)); *ons = 0;
    pingpong_kernel<<<1, 1, 0, s0[0]>>>(d0f, d1f, 10000, 1, ons);
    CK(cudaSetDevice(1));
    pingpong_kernel<<<1, 1, 0, s1[0]>>>(d1f, d0f, 10000, 0, ons);
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    printf("persistent kernel ping-pong one-way %.3f us\n", *ons / 1e3 / 10000 / 2);
  }
  SECTION("done");
  return 0;
}
