// Design probe 4 (see p2p_probe.cu .. p2p_probe3.cu): separates CPU enqueue cost from GPU
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



// probe 4: each test selected by argv[1] so a hang in one cannot hide the others
int main(int argc, char** argv) {
  T0 = now_s();
  int test = argc > 1 ? atoi(argv[1]) : 0;
  CKD(cuInit(0));
  int ndev; CK(cudaGetDeviceCount(&ndev));
  CK(cudaSetDevice(0)); if (ndev > 1) CK(cudaDeviceEnablePeerAccess(1, 0));
  if (ndev > 1) { CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0)); }
  const size_t MAXB = 256 * MiB;
  char *b0, *b1 = nullptr, *c0, *c1 = nullptr;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&b0, MAXB)); CK(cudaMalloc(&c0, MAXB)); CK(cudaMemset(b0, 1, MAXB));
  if (ndev > 1) { CK(cudaSetDevice(1)); CK(cudaMalloc(&b1, MAXB)); CK(cudaMalloc(&c1, MAXB)); CK(cudaMemset(b1, 2, MAXB)); }
  if (ndev < 2) { b1 = c0; c1 = c0; }
  const int NS = 4;
  cudaStream_t s0[NS], s1[NS];
  cudaEvent_t es[NS], ee[NS];
  CK(cudaSetDevice(0)); for (int i = 0; i < NS; i++) { CK(cudaStreamCreateWithFlags(&s0[i], cudaStreamNonBlocking)); CK(cudaEventCreate(&es[i])); CK(cudaEventCreate(&ee[i])); }
  if (ndev > 1) { CK(cudaSetDevice(1)); for (int i = 0; i < NS; i++) CK(cudaStreamCreateWithFlags(&s1[i], cudaStreamNonBlocking)); }
  uint32_t* hf; CK(cudaHostAlloc(&hf, 1 << 16, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(hf, 0, 1 << 16);
  CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
  volatile uint32_t* H = hf;
  auto wait_host = [&](int idx, uint32_t v, double tmo) {
    double t = now_s();
    while (H[idx] != v) { if (now_s() - t > tmo) { printf("  TIMEOUT waiting host word %d for %u (have %u)\n", idx, v, H[idx]); fflush(stdout); return false; } }
    return true;
  };
  if (test == 1) {
    SECTION("1. WaitValue(host) -> kernel -> WriteValue(host)");
    for (int rep = 0; rep < 5; rep++) {
      hf[100] = 0; hf[116] = 0;
      CKD(cuStreamWaitValue32((CUstream)s0[0], (CUdeviceptr)(hf + 100), 1, CU_STREAM_WAIT_VALUE_GEQ));
      copy_ldst<4><<<16, 512, 0, s0[0]>>>((const int4*)b0, (int4*)c0, MiB / 16);
      CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)(hf + 116), 1, 0));
      usleep(1000);
      printf("  before release: done=%u\n", H[116]);
      double t = now_s();
      __atomic_store_n(hf + 100, 1u, __ATOMIC_SEQ_CST);
      bool ok = wait_host(116, 1, 2.0);
      printf("  rep %d ok=%d %.2f us\n", rep, ok, (now_s() - t) * 1e6); fflush(stdout);
      if (!ok) return 3;
      CK(cudaStreamSynchronize(s0[0]));
    }
  }
  if (test == 2) {
    SECTION("2. E0 memop wait reaction vs idle (host write -> GPU WriteValue seen by host)");
    for (int idle : {0, 10, 100, 1000, 10000, 100000}) {
      std::vector<double> v;
      for (int rep = 0; rep < 9; rep++) {
        hf[200] = 0; hf[216] = 0;
        CKD(cuStreamWaitValue32((CUstream)s0[0], (CUdeviceptr)(hf + 200), 1, CU_STREAM_WAIT_VALUE_GEQ));
        CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)(hf + 216), 1, 0));
        double t = now_s();
        while (now_s() - t < idle * 1e-6) {}
        t = now_s();
        __atomic_store_n(hf + 200, 1u, __ATOMIC_SEQ_CST);
        if (!wait_host(216, 1, 2.0)) return 3;
        v.push_back((now_s() - t) * 1e6);
        CK(cudaStreamSynchronize(s0[0]));
      }
      std::sort(v.begin(), v.end());
      printf("  idle %d us: reaction %.2f us (min %.2f max %.2f)\n", idle, v[4], v[0], v[8]); fflush(stdout);
    }
  }
  if (test == 3) {
    SECTION("3. host-released single op round trip: CE copy vs SM kernel (1 CTA) vs memop only");
    for (int kind = 0; kind < 3; kind++) {
      for (size_t sz : {8ul, 4096ul, 65536ul, 1ul << 20}) {
        if (kind == 2 && sz > 8) continue;
        std::vector<double> v;
        for (int rep = 0; rep < 21; rep++) {
          hf[300] = 0; hf[316] = 0;
          CKD(cuStreamWaitValue32((CUstream)s0[0], (CUdeviceptr)(hf + 300), 1, CU_STREAM_WAIT_VALUE_GEQ));
          if (kind == 0) CK(cudaMemcpyAsync(b1, b0, sz, cudaMemcpyDefault, s0[0]));
          if (kind == 1) copy_ldst<4><<<1, 512, 0, s0[0]>>>((const int4*)b0, (int4*)b1, (sz + 15) / 16);
          CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)(hf + 316), 1, 0));
          usleep(200);
          double t = now_s();
          __atomic_store_n(hf + 300, 1u, __ATOMIC_SEQ_CST);
          if (!wait_host(316, 1, 2.0)) return 3;
          v.push_back((now_s() - t) * 1e6);
          CK(cudaStreamSynchronize(s0[0]));
        }
        std::sort(v.begin(), v.end());
        printf("  %s %zu B: p50 %.2f us (min %.2f)\n", kind == 0 ? "CE" : (kind == 1 ? "SM" : "memop"), sz, v[10], v[0]); fflush(stdout);
      }
    }
  }
  if (test == 4 && ndev > 1) {
    SECTION("4. interleaved ping-pong between GPUs (one-way us)");
    CUdeviceptr fA = (CUdeviceptr)(hf + 1024), fB = (CUdeviceptr)(hf + 1040);
    for (int mode = 0; mode < 3; mode++) {
      for (size_t sz : {8ul, 65536ul}) {
        if (mode == 0 && sz > 8) continue;
        hf[1024] = 0; hf[1040] = 0;
        const int N = 300;
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
        CK(cudaSetDevice(0));
        if (!wait_host(1040, N, 10.0)) return 3;
        CK(cudaEventSynchronize(ee[0]));
        float ms; CK(cudaEventElapsedTime(&ms, es[0], ee[0]));
        printf("  %s %zu B: one-way %.2f us\n", mode == 0 ? "memop-only" : (mode == 1 ? "CE+memop" : "SM1cta+memop"), sz, ms * 1e3 / N / 2); fflush(stdout);
      }
    }
  }
  if (test == 5 && ndev > 1) {
    SECTION("5. CE + SM concurrently into the peer: total frac_sm ctas us GB/s");
    for (size_t tot : {64 * MiB, 256 * MiB}) {
      for (double f : {0.0, 0.1, 0.2, 0.3, 0.5}) {
        for (int ctas : {16, 32}) {
          size_t nsm = ((size_t)(tot * f)) & ~(size_t)4095;
          std::vector<double> v;
          for (int rep = 0; rep < 6; rep++) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(es[0], s0[0]));
            CK(cudaStreamWaitEvent(s0[1], es[0], 0));
            if (tot - nsm) CK(cudaMemcpyAsync(b1, b0, tot - nsm, cudaMemcpyDefault, s0[0]));
            if (nsm) copy_ldst<4><<<ctas, 512, 0, s0[1]>>>((const int4*)(b0 + tot - nsm), (int4*)(b1 + tot - nsm), nsm / 16);
            CK(cudaEventRecord(ee[1], s0[1])); CK(cudaStreamWaitEvent(s0[0], ee[1], 0));
            CK(cudaEventRecord(ee[0], s0[0])); CK(cudaEventSynchronize(ee[0]));
            float ms; CK(cudaEventElapsedTime(&ms, es[0], ee[0]));
            if (rep) v.push_back(ms * 1e3);
          }
          std::sort(v.begin(), v.end());
          printf("  %zu %.1f %d %.1f %.1f\n", tot / MiB, f, ctas, v[2], tot / v[2] / 1e3); fflush(stdout);
        }
      }
    }
  }
  if (test == 6 && ndev > 1) {
    SECTION("6. chunked CE with EventRecord between chunks (GPU time): chunkMiB us GB/s");
    for (size_t ch : {4 * MiB, 16 * MiB, 64 * MiB}) {
      std::vector<double> v;
      cudaEvent_t evs[64]; for (int i = 0; i < 64; i++) CK(cudaEventCreate(&evs[i]));
      for (int rep = 0; rep < 6; rep++) {
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(es[0], s0[0]));
        size_t n = 256 * MiB / ch;
        for (size_t c = 0; c < n; c++) { CK(cudaMemcpyAsync(b1 + c * ch, b0 + c * ch, ch, cudaMemcpyDefault, s0[0])); CK(cudaEventRecord(evs[c % 64], s0[0])); }
        CK(cudaEventRecord(ee[0], s0[0])); CK(cudaEventSynchronize(ee[0]));
        float ms; CK(cudaEventElapsedTime(&ms, es[0], ee[0]));
        if (rep) v.push_back(ms * 1e3);
      }
      std::sort(v.begin(), v.end());
      printf("  %zu %.1f %.1f\n", ch / MiB, v[2], 256 * MiB / v[2] / 1e3); fflush(stdout);
    }
    SECTION("6b. one 256 MiB copy vs 2D-free memcpy of pitch? (skipped)");
  }
  if (test == 7) {
    SECTION("7. local HBM: CE D2D and SM copy (payload GB/s)");
    for (size_t sz : {64 * MiB, 256 * MiB}) {
      std::vector<double> v;
      for (int rep = 0; rep < 6; rep++) {
        CK(cudaEventRecord(es[0], s0[0]));
        CK(cudaMemcpyAsync(c0, b0, sz, cudaMemcpyDefault, s0[0]));
        CK(cudaEventRecord(ee[0], s0[0])); CK(cudaEventSynchronize(ee[0]));
        float ms; CK(cudaEventElapsedTime(&ms, es[0], ee[0])); if (rep) v.push_back(ms * 1e3);
      }
      std::sort(v.begin(), v.end());
      printf("  CE %zu MiB %.1f us %.1f GB/s\n", sz / MiB, v[2], sz / v[2] / 1e3);
      for (int ctas : {148, 296, 592}) {
        v.clear();
        for (int rep = 0; rep < 6; rep++) {
          CK(cudaEventRecord(es[0], s0[0]));
          copy_ldst<4><<<ctas, 512, 0, s0[0]>>>((const int4*)b0, (int4*)c0, sz / 16);
          CK(cudaEventRecord(ee[0], s0[0])); CK(cudaEventSynchronize(ee[0]));
          float ms; CK(cudaEventElapsedTime(&ms, es[0], ee[0])); if (rep) v.push_back(ms * 1e3);
        }
        std::sort(v.begin(), v.end());
        printf("  SM%d %zu MiB %.1f us %.1f GB/s\n", ctas, sz / MiB, v[2], sz / v[2] / 1e3);
      }
    }
  }
  SECTION("done");
  return 0;
}
