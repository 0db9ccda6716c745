// Does ncu's kernel serialisation span processes?  Parent launches a kernel
// that spins on a host-mapped shared word (5 s self-timeout); a forked child
// launches, 0.5 s later, a kernel that sets the word.  Prints how long the
// spin took: ~0.5 s = the child's kernel ran while the parent's was being
// profiled; ~5 s (timeout) = ncu serialised the two processes.
#include <cuda_runtime.h>
#include <stdio.h>
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>
#include <time.h>

__global__ void spin(volatile unsigned* f, unsigned long long* out) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (*f == 0 && t - t0 < 5000000000ull);
  *out = t - t0;
}
__global__ void setf(volatile unsigned* f) { *f = 1; __threadfence_system(); }

int main() {
  unsigned* shm = (unsigned*)mmap(nullptr, 4096, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
  shm[0] = 0;
  pid_t pid = fork();
  if (pid == 0) {
    usleep(500000);
    cudaHostRegister(shm, 4096, cudaHostRegisterMapped);
    setf<<<1, 1>>>(shm);
    cudaError_t e = cudaDeviceSynchronize();
    printf("child: set kernel done (%s)\n", cudaGetErrorString(e));
    return 0;
  }
  cudaHostRegister(shm, 4096, cudaHostRegisterMapped);
  unsigned long long* out;
  cudaHostAlloc(&out, 8, cudaHostAllocMapped);
  *out = 0;
  spin<<<1, 1>>>(shm, out);
  cudaError_t e = cudaDeviceSynchronize();
  int st;
  waitpid(pid, &st, 0);
  printf("parent: spin took %.3f s (%s) -> %s\n", *out * 1e-9, cudaGetErrorString(e),
         *out > 4000000000ull ? "SERIALISED across processes" : "concurrent across processes");
  return 0;
}
