// Design probe: measures the B200 primitives the ICCL hot path is built from,
// before committing to a design (SURVEY.md §7 hard parts H1, H2, H5, H8).
//   - copy-engine (CE) peer copy bandwidth: one stream vs chunk striping over
//     S streams, push (writer-side issue) vs pull (reader-side issue), bidir
//   - SM copy kernels (LDG/STG.128 and TMA bulk) into a peer, vs CTA count
//   - stream memop latency: WriteValue/WaitValue ping-pong through host-mapped
//     memory and through peer device memory
//   - CE small-copy latency chain and %globaltimer resolution
// Single process, 2 GPUs with peer access. Not part of the product.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)
#define CKD(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  fprintf(stderr, "CU %s at %s:%d: %s\n", #x, __FILE__, __LINE__, s_); exit(1);} } while (0)

static const size_t MiB = 1ull << 20;

__global__ void copy_ldst(const int4* __restrict__ src, int4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  const int U = 4;
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

// TMA bulk: one thread per CTA drives S smem stages of B bytes: global->smem
// (cp.async.bulk + mbarrier), smem->global (cp.async.bulk bulk_group).
template <int S>
__global__ void copy_tma(const char* __restrict__ src, char* __restrict__ dst, size_t n, int tile) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t mbar[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; s++) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(a));
  }
  asm volatile("fence.mbarrier_init.release.cluster;");
  size_t ntiles = (n + tile - 1) / tile;
  // tiles assigned round-robin over CTAs
  size_t first = blockIdx.x;
  size_t mine = first < ntiles ? (ntiles - first + gridDim.x - 1) / gridDim.x : 0;
  auto load = [&](size_t j) {
    size_t t = first + j * gridDim.x;
    size_t off = t * (size_t)tile;
    uint32_t bytes = (uint32_t)min((size_t)tile, n - off);
    int s = j % S;
    uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + (size_t)s * tile);
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(sm), "l"(src + off), "r"(bytes), "r"(mb) : "memory");
  };
  for (size_t j = 0; j < mine && j < S; j++) load(j);
  for (size_t j = 0; j < mine; j++) {
    int s = j % S;
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar[s]);
    uint32_t par = (j / S) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                   : "=r"(done) : "r"(mb), "r"(par) : "memory");
    size_t t = first + j * gridDim.x;
    size_t off = t * (size_t)tile;
    uint32_t bytes = (uint32_t)min((size_t)tile, n - off);
    uint32_t sm = (uint32_t)__cvta_generic_to_shared(smem + (size_t)s * tile);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + off), "r"(sm), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (j + S < mine) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(j + S);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void gtimer_res(uint64_t* out, int n) {
  uint64_t prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int k = 0;
  while (k < n) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { out[k++] = t - prev; prev = t; }
  }
}

// persistent ping-pong through peer device memory flags (pure NVLink RTT)
__global__ void pingpong_kernel(volatile uint32_t* my_flag, volatile uint32_t* peer_flag, int iters, int initiator,
                                unsigned long long* out_ns) {
  uint64_t t0, t1, tl;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; i++) {
    if (initiator) {
      asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(peer_flag), "r"(i) : "memory");
      uint32_t v = 0;
      do { asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flag) : "memory");
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl));
        if (tl - t0 > 2000000000ull) return; } while ((int)(v - i) < 0);
    } else {
      uint32_t v = 0;
      do { asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(my_flag) : "memory");
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl));
        if (tl - t0 > 2000000000ull) return; } while ((int)(v - i) < 0);
      asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(peer_flag), "r"(i) : "memory");
    }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (initiator) *out_ns = t1 - t0;
}

static float ev_ms(cudaEvent_t a, cudaEvent_t b) { float ms; CK(cudaEventElapsedTime(&ms, a, b)); return ms; }

int main(int argc, char** argv) {
  CKD(cuInit(0));
  int ndev = 0; CK(cudaGetDeviceCount(&ndev));
  printf("devices %d\n", ndev);
  for (int d = 0; d < ndev && d < 2; d++) {
    CUdevice cd; CKD(cuDeviceGet(&cd, d));
    int ae, mo, m64, nor, flush, sms;
    cuDeviceGetAttribute(&ae, CU_DEVICE_ATTRIBUTE_ASYNC_ENGINE_COUNT, cd);
    cuDeviceGetAttribute(&mo, (CUdevice_attribute)92, cd);
    cuDeviceGetAttribute(&m64, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, cd);
    cuDeviceGetAttribute(&nor, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, cd);
    cuDeviceGetAttribute(&flush, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, cd);
    cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, cd);
    printf("dev%d async_engines=%d memops_v1=%d memops64=%d wait_nor=%d flush_remote=%d sms=%d\n", d, ae, mo, m64, nor, flush, sms);
  }
  if (ndev < 2) { printf("need 2 GPUs\n"); return 0; }
  int can01, can10; CK(cudaDeviceCanAccessPeer(&can01, 0, 1)); CK(cudaDeviceCanAccessPeer(&can10, 1, 0));
  printf("peer 0->1 %d 1->0 %d\n", can01, can10);
  CK(cudaSetDevice(0)); CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaSetDevice(1)); CK(cudaDeviceEnablePeerAccess(0, 0));

  const size_t MAXB = 1024 * MiB;
  char *b0, *b1, *c0, *c1;
  CK(cudaSetDevice(0)); CK(cudaMalloc(&b0, MAXB)); CK(cudaMalloc(&c0, MAXB)); CK(cudaMemset(b0, 1, MAXB));
  CK(cudaSetDevice(1)); CK(cudaMalloc(&b1, MAXB)); CK(cudaMalloc(&c1, MAXB)); CK(cudaMemset(b1, 2, MAXB));
  const int NS = 8;
  cudaStream_t s0[NS], s1[NS];
  cudaEvent_t e0a, e0b, e1a, e1b;
  CK(cudaSetDevice(0)); for (int i = 0; i < NS; i++) CK(cudaStreamCreateWithFlags(&s0[i], cudaStreamNonBlocking));
  CK(cudaEventCreate(&e0a)); CK(cudaEventCreate(&e0b));
  CK(cudaSetDevice(1)); for (int i = 0; i < NS; i++) CK(cudaStreamCreateWithFlags(&s1[i], cudaStreamNonBlocking));
  CK(cudaEventCreate(&e1a)); CK(cudaEventCreate(&e1b));
  cudaEvent_t join0[NS]; CK(cudaSetDevice(0)); for (int i = 0; i < NS; i++) CK(cudaEventCreateWithFlags(&join0[i], cudaEventDisableTiming));
  cudaEvent_t join1[NS]; CK(cudaSetDevice(1)); for (int i = 0; i < NS; i++) CK(cudaEventCreateWithFlags(&join1[i], cudaEventDisableTiming));

  // ---- 1. CE push, single stream, size sweep ------------------------------------
  printf("\n# CE push single stream (dev0 stream copies b0 -> b1)\n# bytes us GB/s\n");
  CK(cudaSetDevice(0));
  for (size_t sz = 8; sz <= MAXB; sz *= 4) {
    int iters = sz >= 256 * MiB ? 10 : (sz >= 4 * MiB ? 50 : 200);
    for (int w = 0; w < 3; w++) CK(cudaMemcpyAsync(b1, b0, sz, cudaMemcpyDefault, s0[0]));
    CK(cudaEventRecord(e0a, s0[0]));
    for (int i = 0; i < iters; i++) CK(cudaMemcpyAsync(b1, b0, sz, cudaMemcpyDefault, s0[0]));
    CK(cudaEventRecord(e0b, s0[0])); CK(cudaEventSynchronize(e0b));
    double us = ev_ms(e0a, e0b) * 1e3 / iters;
    printf("%zu %.2f %.1f\n", sz, us, sz / us / 1e3);
  }
  // ---- 2. CE push striped over S streams, chunk C -------------------------------
  printf("\n# CE push striped: total chunkMiB streams us GB/s\n");
  for (size_t tot : {64 * MiB, 256 * MiB, 1024 * MiB}) {
    for (size_t ch : {1 * MiB, 2 * MiB, 4 * MiB, 8 * MiB, 16 * MiB, 64 * MiB}) {
      if (ch > tot) continue;
      for (int S : {1, 2, 4, 8}) {
        auto run = [&]() {
          CK(cudaEventRecord(e0a, s0[0]));
          for (int k = 1; k < S; k++) CK(cudaStreamWaitEvent(s0[k], e0a, 0));
          size_t nch = tot / ch;
          for (size_t c = 0; c < nch; c++) CK(cudaMemcpyAsync(b1 + c * ch, b0 + c * ch, ch, cudaMemcpyDefault, s0[c % S]));
          for (int k = 1; k < S; k++) { CK(cudaEventRecord(join0[k], s0[k])); CK(cudaStreamWaitEvent(s0[0], join0[k], 0)); }
          CK(cudaEventRecord(e0b, s0[0])); CK(cudaEventSynchronize(e0b));
          return ev_ms(e0a, e0b) * 1e3;
        };
        run(); run();
        std::vector<double> v; for (int r = 0; r < 7; r++) v.push_back(run());
        std::sort(v.begin(), v.end());
        printf("%zu %zu %d %.1f %.1f\n", tot / MiB, ch / MiB, S, v[3], tot / v[3] / 1e3);
      }
    }
  }
  // ---- 3. CE pull (dev1 stream reads b0 into c1) --------------------------------
  printf("\n# CE pull single stream (dev1 stream copies b0 -> c1)\n");
  CK(cudaSetDevice(1));
  for (size_t sz : {64 * MiB, 256 * MiB, 1024 * MiB}) {
    for (int w = 0; w < 2; w++) CK(cudaMemcpyAsync(c1, b0, sz, cudaMemcpyDefault, s1[0]));
    CK(cudaEventRecord(e1a, s1[0]));
    for (int i = 0; i < 5; i++) CK(cudaMemcpyAsync(c1, b0, sz, cudaMemcpyDefault, s1[0]));
    CK(cudaEventRecord(e1b, s1[0])); CK(cudaEventSynchronize(e1b));
    double us = ev_ms(e1a, e1b) * 1e3 / 5;
    printf("%zu %.1f %.1f\n", sz, us, sz / us / 1e3);
  }
  // ---- 4. CE bidirectional push --------------------------------------------------
  printf("\n# CE bidir push 256MiB each way, 4MiB chunks over S streams each side\n");
  for (int S : {1, 2, 4}) {
    size_t tot = 256 * MiB, ch = 4 * MiB;
    double best = 1e30;
    for (int r = 0; r < 5; r++) {
      CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize()); CK(cudaSetDevice(1)); CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0)); CK(cudaEventRecord(e0a, s0[0]));
      for (int k = 1; k < S; k++) CK(cudaStreamWaitEvent(s0[k], e0a, 0));
      CK(cudaSetDevice(1)); CK(cudaEventRecord(e1a, s1[0]));
      for (int k = 1; k < S; k++) CK(cudaStreamWaitEvent(s1[k], e1a, 0));
      for (size_t c = 0; c < tot / ch; c++) {
        CK(cudaSetDevice(0)); CK(cudaMemcpyAsync(b1 + c * ch, b0 + c * ch, ch, cudaMemcpyDefault, s0[c % S]));
        CK(cudaSetDevice(1)); CK(cudaMemcpyAsync(b0 + MAXB / 2 + c * ch, b1 + MAXB / 2 + c * ch, ch, cudaMemcpyDefault, s1[c % S]));
      }
      CK(cudaSetDevice(0));
      for (int k = 1; k < S; k++) { CK(cudaEventRecord(join0[k], s0[k])); CK(cudaStreamWaitEvent(s0[0], join0[k], 0)); }
      CK(cudaEventRecord(e0b, s0[0]));
      CK(cudaSetDevice(1));
      for (int k = 1; k < S; k++) { CK(cudaEventRecord(join1[k], s1[k])); CK(cudaStreamWaitEvent(s1[0], join1[k], 0)); }
      CK(cudaEventRecord(e1b, s1[0]));
      CK(cudaEventSynchronize(e1b)); CK(cudaSetDevice(0)); CK(cudaEventSynchronize(e0b));
      double t = std::max(ev_ms(e0a, e0b), ev_ms(e1a, e1b)) * 1e3;
      best = std::min(best, t);
    }
    printf("S=%d %.1f us, per-direction %.1f GB/s\n", S, best, tot / best / 1e3);
  }
  // ---- 5. SM copy kernels into peer vs CTA count ---------------------------------
  printf("\n# SM copy push (dev0 kernel writes b1): kind ctas threads bytes us GB/s\n");
  CK(cudaSetDevice(0));
  CK(cudaFuncSetAttribute(copy_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(copy_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (size_t sz : {64 * MiB, 256 * MiB}) {
    for (int ctas : {1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 148, 296}) {
      for (int kind = 0; kind < 3; kind++) {
        auto launch = [&]() {
          if (kind == 0) copy_ldst<<<ctas, 512, 0, s0[0]>>>((const int4*)b0, (int4*)b1, sz / 16);
          else if (kind == 1) copy_tma<4><<<ctas, 32, 4 * 32768, s0[0]>>>(b0, b1, sz, 32768);
          else copy_tma<8><<<ctas, 32, 8 * 16384, s0[0]>>>(b0, b1, sz, 16384);
        };
        if (kind > 0 && ctas > 148) continue;
        launch(); launch();
        CK(cudaGetLastError());
        CK(cudaEventRecord(e0a, s0[0]));
        for (int i = 0; i < 5; i++) launch();
        CK(cudaEventRecord(e0b, s0[0])); CK(cudaEventSynchronize(e0b));
        double us = ev_ms(e0a, e0b) * 1e3 / 5;
        printf("%s %d %zu %.1f %.1f\n", kind == 0 ? "ldst" : (kind == 1 ? "tma4x32K" : "tma8x16K"), ctas, sz, us, sz / us / 1e3);
      }
    }
  }
  // verify tma copy bytes
  {
    CK(cudaMemset(b1, 0, 64 * MiB));
    copy_tma<4><<<16, 32, 4 * 32768, s0[0]>>>(b0, b1, 64 * MiB - 48, 32768);
    CK(cudaStreamSynchronize(s0[0]));
    std::vector<char> h(64 * MiB);
    CK(cudaMemcpy(h.data(), b1, 64 * MiB, cudaMemcpyDefault));
    size_t bad = 0; for (size_t i = 0; i < 64 * MiB - 48; i++) bad += h[i] != 1;
    for (size_t i = 64 * MiB - 48; i < 64 * MiB; i++) bad += h[i] != 0;
    printf("tma verify bad=%zu\n", bad);
  }
  // ---- 6. SM pull kernel (dev1 kernel reads b0) ------------------------------------
  printf("\n# SM copy pull (dev1 kernel reads b0 into c1): ctas us GB/s\n");
  CK(cudaSetDevice(1));
  for (int ctas : {8, 16, 32, 64, 148, 296}) {
    size_t sz = 256 * MiB;
    copy_ldst<<<ctas, 512, 0, s1[0]>>>((const int4*)b0, (int4*)c1, sz / 16);
    CK(cudaEventRecord(e1a, s1[0]));
    for (int i = 0; i < 5; i++) copy_ldst<<<ctas, 512, 0, s1[0]>>>((const int4*)b0, (int4*)c1, sz / 16);
    CK(cudaEventRecord(e1b, s1[0])); CK(cudaEventSynchronize(e1b));
    double us = ev_ms(e1a, e1b) * 1e3 / 5;
    printf("%d %.1f %.1f\n", ctas, us, sz / us / 1e3);
  }
  // ---- 7. stream memop ping-pong via host-mapped flags -----------------------------
  printf("\n# memop ping-pong\n");
  uint32_t* hflags; CK(cudaHostAlloc(&hflags, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(hflags, 0, 4096);
  CUdeviceptr fA = (CUdeviceptr)(hflags), fB = (CUdeviceptr)(hflags + 16);
  {
    const int N = 2000;
    CK(cudaSetDevice(0)); CK(cudaEventRecord(e0a, s0[0]));
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
    printf("host-flag memop RTT %.2f us\n", ev_ms(e0a, e0b) * 1e3 / N);
  }
  // device-memory flags (each GPU waits on its own memory, peer writes via P2P mapping)
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
    printf("device-flag (peer write, local wait) memop RTT %.2f us\n", ev_ms(e0a, e0b) * 1e3 / N);
    // persistent kernel ping-pong through peer memory
    CK(cudaMemset(d0f, 0, 256)); CK(cudaSetDevice(1)); CK(cudaMemset(d1f, 0, 256)); CK(cudaDeviceSynchronize());
    unsigned long long* ons; CK(cudaSetDevice(0)); CK(cudaMallocManaged(&ons, 8)); *ons = 0; CK(cudaDeviceSynchronize());
    pingpong_kernel<<<1, 1, 0, s0[0]>>>(d0f, d1f, 10000, 1, ons);
    CK(cudaSetDevice(1));
    pingpong_kernel<<<1, 1, 0, s1[0]>>>(d1f, d0f, 10000, 0, ons);
    CK(cudaDeviceSynchronize()); CK(cudaSetDevice(0)); CK(cudaDeviceSynchronize());
    printf("kernel ping-pong RTT %.3f us\n", *ons / 1e3 / 10000);
  }
  // ---- 8. CE small-copy chain latency: copy 8B -> flag -> peer waits -> copy back --
  for (size_t sz : {8ul, 4096ul, 65536ul, 1ul << 20}) {
    memset(hflags, 0, 4096);
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
  // back-to-back small copies throughput (per-copy cost on one stream)
  for (size_t sz : {8ul, 4096ul, 65536ul}) {
    const int N = 2000;
    CK(cudaSetDevice(0)); CK(cudaEventRecord(e0a, s0[0]));
    for (int i = 0; i < N; i++) CK(cudaMemcpyAsync(b1, b0, sz, cudaMemcpyDefault, s0[0]));
    CK(cudaEventRecord(e0b, s0[0])); CK(cudaEventSynchronize(e0b));
    printf("CE back-to-back %zu B: %.2f us/copy\n", sz, ev_ms(e0a, e0b) * 1e3 / N);
  }
  // ---- 9. %globaltimer resolution --------------------------------------------------
  {
    uint64_t* d; CK(cudaSetDevice(0)); CK(cudaMallocManaged(&d, 64 * 8));
    gtimer_res<<<1, 1>>>(d, 64); CK(cudaDeviceSynchronize());
    std::vector<uint64_t> v(d, d + 64); std::sort(v.begin(), v.end());
    printf("globaltimer tick: min %lu median %lu ns\n", v[0], v[32]);
  }
  // ---- 10. local HBM copy via CE and via kernel (self-send path) ------------------
  {
    CK(cudaSetDevice(0));
    size_t sz = 256 * MiB;
    CK(cudaEventRecord(e0a, s0[0]));
    for (int i = 0; i < 10; i++) CK(cudaMemcpyAsync(c0, b0, sz, cudaMemcpyDefault, s0[0]));
    CK(cudaEventRecord(e0b, s0[0])); CK(cudaEventSynchronize(e0b));
    double us = ev_ms(e0a, e0b) * 1e3 / 10;
    printf("local CE D2D 256MiB %.1f us %.1f GB/s (payload)\n", us, sz / us / 1e3);
    CK(cudaEventRecord(e0a, s0[0]));
    for (int i = 0; i < 10; i++) copy_ldst<<<148 * 4, 512, 0, s0[0]>>>((const int4*)b0, (int4*)c0, sz / 16);
    CK(cudaEventRecord(e0b, s0[0])); CK(cudaEventSynchronize(e0b));
    us = ev_ms(e0a, e0b) * 1e3 / 10;
    printf("local kernel D2D 256MiB %.1f us %.1f GB/s (payload)\n", us, sz / us / 1e3);
  }
  printf("done\n");
  return 0;
}
