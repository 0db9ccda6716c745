// Design probe 7: can one GPU's copy engines run a push (local -> peer) and a
// pull (peer -> local) concurrently at full NVLink rate, compared with each
// GPU pushing its own direction?  Single process, 2 GPUs with peer access.
// Not part of the product.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d: %s\n", #x, __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

int main() {
  const size_t n = 256ull << 20;
  char *a0, *b0, *a1, *b1;
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&a0, n));
  CK(cudaMalloc(&b0, n));
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&a1, n));
  CK(cudaMalloc(&b1, n));
  cudaStream_t s0a, s0b, s1a;
  cudaEvent_t e0, e1, f0, f1;
  CK(cudaSetDevice(1));
  CK(cudaStreamCreateWithFlags(&s1a, cudaStreamNonBlocking));
  CK(cudaEventCreate(&f1));
  CK(cudaSetDevice(0));
  CK(cudaEventCreate(&f0));
  CK(cudaStreamCreateWithFlags(&s0a, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s0b, cudaStreamNonBlocking));
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const char* names[] = {"push 0->1 alone (GPU0 CE)", "pull 1->0 alone (GPU0 CE)",
                         "push 0->1 + pull 1->0 both on GPU0 CEs", "push 0->1 on GPU0 + push 1->0 on GPU1",
                         "push 0->1 + push 0->1 on 2 GPU0 streams"};
  for (int mode = 0; mode < 5; mode++) {
    float best = 1e9;
    for (int rep = 0; rep < 6; rep++) {
      CK(cudaSetDevice(0));
      CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(1));
      CK(cudaDeviceSynchronize());
      CK(cudaSetDevice(0));
      CK(cudaEventRecord(e0, s0a));
      CK(cudaStreamWaitEvent(s0b, e0, 0));
      if (mode == 0) CK(cudaMemcpyAsync(a1, a0, n, cudaMemcpyDefault, s0a));
      if (mode == 1) CK(cudaMemcpyAsync(b0, b1, n, cudaMemcpyDefault, s0a));
      if (mode == 2) {
        CK(cudaMemcpyAsync(a1, a0, n, cudaMemcpyDefault, s0a));
        CK(cudaMemcpyAsync(b0, b1, n, cudaMemcpyDefault, s0b));
      }
      if (mode == 3) {
        CK(cudaMemcpyAsync(a1, a0, n, cudaMemcpyDefault, s0a));
        CK(cudaSetDevice(1));
        CK(cudaStreamWaitEvent(s1a, e0, 0));
        CK(cudaMemcpyAsync(b0, b1, n, cudaMemcpyDefault, s1a));
        CK(cudaEventRecord(f1, s1a));
        CK(cudaSetDevice(0));
        CK(cudaStreamWaitEvent(s0a, f1, 0));
      }
      if (mode == 4) {
        CK(cudaMemcpyAsync(a1, a0, n / 2, cudaMemcpyDefault, s0a));
        CK(cudaMemcpyAsync(a1 + n / 2, a0 + n / 2, n / 2, cudaMemcpyDefault, s0b));
      }
      CK(cudaEventRecord(f0, s0b));
      CK(cudaStreamWaitEvent(s0a, f0, 0));
      CK(cudaEventRecord(e1, s0a));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (rep > 0 && ms < best) best = ms;
    }
    const double bytes = (mode == 2 || mode == 3) ? 2.0 * n : (double)n;
    printf("  %-44s %8.1f us  %7.1f GB/s total\n", names[mode], best * 1e3, bytes / (best * 1e-3) / 1e9);
    fflush(stdout);
  }
  return 0;
}
