// Design probe 2 (see p2p_probe.cu): separates CPU enqueue cost from GPU
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
  cudaEvent_t e0a, e0b, e1a, e1b, j0[NS];
  CK(cudaSetDevice(0)); for (int i = 0; i < NS; i++) CK(cudaStreamCreateWithFlags(&s0[i], cudaStreamNonBlocking));
  CK(cudaEventCreate(&e0a)); CK(cudaEventCreate(&e0b));
  for (int i = 0; i < NS; i++) CK(cudaEventCreateWithFlags(&j0[i], cudaEventDisableTiming));
  CK(cudaSetDevice(1)); for (int i = 0; i < NS; i++) CK(cudaStreamCreateWithFlags(&s1[i], cudaStreamNonBlocking));
  CK(cudaEventCreate(&e1a)); CK(cudaEventCreate(&e1b));
  uint32_t* hf; CK(cudaHostAlloc(&hf, 1 << 16, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(hf, 0, 1 << 16);
  CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());

  SECTION("A. CPU cost of cudaMemcpyAsync (peer, 4 MiB) and memops per call");
  {
    const int N = 2000;
    double t = now_s();
    for (int i = 0; i < N; i++) CK(cudaMemcpyAsync(b1 + (i % 64) * 4 * MiB, b0, 4 * MiB, cudaMemcpyDefault, s0[0]));
    double dt = now_s() - t;
    CK(cudaStreamSynchronize(s0[0]));
    printf("memcpyAsync peer: %.2f us/call (host)\n", dt / N * 1e6);
    t = now_s();
    for (int i = 0; i < N; i++) CK(cudaMemcpyAsync(c0 + (i % 64) * 4 * MiB, b0, 4 * MiB, cudaMemcpyDefault, s0[0]));
    dt = now_s() - t; CK(cudaStreamSynchronize(s0[0]));
    printf("memcpyAsync local: %.2f us/call (host)\n", dt / N * 1e6);
    t = now_s();
    for (int i = 0; i < N; i++) CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)(hf + 100), i, 0));
    dt = now_s() - t; CK(cudaStreamSynchronize(s0[0]));
    printf("WriteValue32: %.2f us/call (host)\n", dt / N * 1e6);
    t = now_s();
    for (int i = 0; i < N; i++) CK(cudaEventRecord(j0[0], s0[0]));
    dt = now_s() - t; CK(cudaStreamSynchronize(s0[0]));
    printf("EventRecord: %.2f us/call (host)\n", dt / N * 1e6);
    t = now_s();
    for (int i = 0; i < N; i++) { volatile cudaError_t q = cudaEventQuery(j0[0]); (void)q; }
    dt = now_s() - t;
    printf("EventQuery: %.2f us/call (host)\n", dt / N * 1e6);
  }

  SECTION("B. GPU-only chunked CE push (pre-enqueued behind a gate): total chunkMiB S wv us GB/s");
  uint32_t gate_val = 0;
  auto gated = [&](int S, auto enqueue) {
    gate_val++;
    CK(cudaSetDevice(0));
    for (int k = 0; k < S; k++) CKD(cuStreamWaitValue32((CUstream)s0[k], (CUdeviceptr)(hf), gate_val, CU_STREAM_WAIT_VALUE_GEQ));
    CK(cudaEventRecord(e0a, s0[0]));
    enqueue();
    for (int k = 1; k < S; k++) { CK(cudaEventRecord(j0[k], s0[k])); CK(cudaStreamWaitEvent(s0[0], j0[k], 0)); }
    CK(cudaEventRecord(e0b, s0[0]));
    __atomic_store_n(hf, gate_val, __ATOMIC_SEQ_CST);
    CK(cudaEventSynchronize(e0b));
    return ev_ms(e0a, e0b) * 1e3;
  };
  for (size_t tot : {64 * MiB, 256 * MiB}) {
    for (size_t ch : {1 * MiB, 2 * MiB, 4 * MiB, 8 * MiB, 16 * MiB, 32 * MiB, 64 * MiB}) {
      if (ch > tot) continue;
      for (int S : {1, 2, 4}) {
        for (int wv = 0; wv < 2; wv++) {
          auto enq = [&]() {
            size_t nch = tot / ch;
            for (size_t c = 0; c < nch; c++) {
              CK(cudaMemcpyAsync(b1 + c * ch, b0 + c * ch, ch, cudaMemcpyDefault, s0[c % S]));
              if (wv) CKD(cuStreamWriteValue32((CUstream)s0[c % S], (CUdeviceptr)(hf + 64 + (c % S)), (uint32_t)c, 0));
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
  SECTION("C. one large copy split across S streams concurrently (gated): total S us GB/s");
  for (size_t tot : {16 * MiB, 64 * MiB, 256 * MiB, 1024 * MiB}) {
    for (int S : {1, 2, 4, 8}) {
      auto enq = [&]() { size_t part = tot / S; for (int k = 0; k < S; k++) CK(cudaMemcpyAsync(b1 + k * part, b0 + k * part, part, cudaMemcpyDefault, s0[k])); };
      gated(S, enq);
      std::vector<double> v; for (int r = 0; r < 5; r++) v.push_back(gated(S, enq));
      std::sort(v.begin(), v.end());
      printf("%zu %d %.1f %.1f\n", tot / MiB, S, v[2], tot / v[2] / 1e3);
    }
  }
  SECTION("C2. single copy size sweep, gated (GPU-only latency+bw): bytes us GB/s");
  for (size_t sz = 8; sz <= 1024 * MiB; sz *= 2) {
    auto enq = [&]() { CK(cudaMemcpyAsync(b1, b0, sz, cudaMemcpyDefault, s0[0])); };
    gated(1, enq);
    std::vector<double> v; for (int r = 0; r < 7; r++) v.push_back(gated(1, enq));
    std::sort(v.begin(), v.end());
    printf("%zu %.2f %.1f\n", sz, v[3], sz / v[3] / 1e3);
  }
  SECTION("D. SM kernels: kind ctas threads bytes us GB/s");
  for (int dir = 0; dir < 2; dir++) {
    // dir 0: push (dev0 kernel writes b1); dir 1: pull (dev1 kernel reads b0 into c1)
    CK(cudaSetDevice(dir));
    cudaStream_t st = dir ? s1[0] : s0[0];
    cudaEvent_t ea = dir ? e1a : e0a, eb = dir ? e1b : e0b;
    const int4* src = (const int4*)b0;
    int4* dst = dir ? (int4*)c1 : (int4*)b1;
    for (size_t sz : {64 * MiB, 256 * MiB}) {
      for (int ctas : {8, 16, 20, 32, 64, 148}) {
        for (int kind = 0; kind < 3; kind++) {
          int thr = kind == 2 ? 1024 : 512;
          auto launch = [&]() {
            if (kind == 0) copy_ldst<4><<<ctas, thr, 0, st>>>(src, dst, sz / 16);
            else if (kind == 1) copy_slab<8><<<ctas, thr, 0, st>>>(src, dst, sz / 16);
            else copy_slab<4><<<ctas, thr, 0, st>>>(src, dst, sz / 16);
          };
          launch(); CK(cudaGetLastError());
          CK(cudaEventRecord(ea, st));
          for (int i = 0; i < 5; i++) launch();
          CK(cudaEventRecord(eb, st)); CK(cudaEventSynchronize(eb));
          double us = ev_ms(ea, eb) * 1e3 / 5;
          printf("%s %s %d %d %zu %.1f %.1f\n", dir ? "pull" : "push", kind == 0 ? "grid-stride-u4" : (kind == 1 ? "slab-u8" : "slab-u4"),
                 ctas, thr, sz, us, sz / us / 1e3);
        }
      }
    }
  }
  SECTION("E. latency chains");
  CK(cudaSetDevice(0));
  CUdeviceptr fA = (CUdeviceptr)(hf + 1024), fB = (CUdeviceptr)(hf + 1040);
  {
    const int N = 2000;
    CK(cudaEventRecord(e0a, s0[0]));
    for (int i = 1; i <= N; i++) {
      CKD(cuStreamWriteValue32((CUstream)s0[0], fA, i, 0));
      CKD(cuStreamWaitValue32((CUstream)s0[0], fB, i, CU_STREAM_WAIT_VALUE_GEQ));
    }
    CK(cudaEventRecord(e0b, s0[0]));
    CK(cudaSetDevice(1));
    for (int i = 1; i <= N; i++) {
      CKD(cuStreamWaitValue32((CUstream)s1[0], fA, i, CU_STREAM_WAIT_VALUE_GEQ));
      CKD(cuStreamWriteValue32((CUstream)s1[0], fB, i, 0));
    }
    CK(cudaSetDevice(0)); CK(cudaEventSynchronize(e0b));
    printf("host-flag memop ping-pong one-way %.2f us\n", ev_ms(e0a, e0b) * 1e3 / N / 2);
  }
  {
    uint32_t *d0f, *d1f;
    CK(cudaSetDevice(0)); CK(cudaMalloc(&d0f, 256)); CK(cudaMemset(d0f, 0, 256));
    CK(cudaSetDevice(1)); CK(cudaMalloc(&d1f, 256)); CK(cudaMemset(d1f, 0, 256));
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    const int N = 2000;
    CK(cudaEventRecord(e0a, s0[0]));
    for (int i = 1; i <= N; i++) {
      CKD(cuStreamWriteValue32((CUstream)s0[0], (CUdeviceptr)d1f, i, 0));
      CKD(cuStreamWaitValue32((CUstream)s0[0], (CUdeviceptr)d0f, i, CU_STREAM_WAIT_VALUE_GEQ));
    }
    CK(cudaEventRecord(e0b, s0[0]));
    CK(cudaSetDevice(1));
    for (int i = 1; i <= N; i++) {
      CKD(cuStreamWaitValue32((CUstream)s1[0], (CUdeviceptr)d1f, i, CU_STREAM_WAIT_VALUE_GEQ));
      CKD(cuStreamWriteValue32((CUstream)s1[0], (CUdeviceptr)d0f, i, 0));
    }
    CK(cudaSetDevice(0)); CK(cudaEventSynchronize(e0b));
    printf("device-flag memop ping-pong one-way %.2f us\n", ev_ms(e0a, e0b) * 1e3 / N / 2);
    CK(cudaMemset(d0f, 0, 256)); CK(cudaSetDevice(1)); CK(cudaMemset(d1f, 0, 256)); CK(cudaDeviceSynchronize());
    unsigned long long* ons; CK(cudaSetDevice(0)); CK(cudaHostAlloc(&ons, 8, cudaHostAllocMapped)); *ons = 0;
    pingpong_kernel<<<1, 1, 0, s0[0]>>>(d0f, d1f, 10000, 1, ons);
    CK(cudaSetDevice(1));
    pingpong_kernel<<<1, 1, 0, s1[0]>>>(d1f, d0f, 10000, 0, ons);
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    printf("kernel ping-pong one-way %.3f us\n", *ons / 1e3 / 10000 / 2);
  }
  for (size_t sz : {8ul, 4096ul, 65536ul, 1ul << 20}) {
    for (int i = 1024; i < 1100; i++) hf[i] = 0;
    const int N = 1000;
    CK(cudaSetDevice(0)); CK(cudaEventRecord(e0a, s0[0]));
    for (int i = 1; i <= N; i++) {
      CK(cudaMemcpyAsync(c1, b0, sz, cudaMemcpyDefault, s0[0]));
      CKD(cuStreamWriteValue32((CUstream)s0[0], fA, i, 0));
      CKD(cuStreamWaitValue32((CUstream)s0[0], fB, i, CU_STREAM_WAIT_VALUE_GEQ));
    }
    CK(cudaEventRecord(e0b, s0[0]));
    CK(cudaSetDevice(1));
    for (int i = 1; i <= N; i++) {
      CKD(cuStreamWaitValue32((CUstream)s1[0], fA, i, CU_STREAM_WAIT_VALUE_GEQ));
      CK(cudaMemcpyAsync(c0, b1, sz, cudaMemcpyDefault, s1[0]));
      CKD(cuStreamWriteValue32((CUstream)s1[0], fB, i, 0));
    }
    CK(cudaSetDevice(0)); CK(cudaEventSynchronize(e0b));
    printf("CE ping-pong %zu B: one-way %.2f us\n", sz, ev_ms(e0a, e0b) * 1e3 / N / 2);
  }
  SECTION("done");
  return 0;
}
