// Round-trip cost of a device scalar read-back, three ways:
//  A: cudaMemcpyAsync D2H into pinned memory + cudaStreamSynchronize
//  B: the producing kernel's value copied by a 1-thread kernel into mapped
//     pinned memory with a sequence flag; the host spins on the flag
//  C: as B, then cudaStreamSynchronize instead of spinning
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/readback_probe.cu -o /tmp/rb && /tmp/rb
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <immintrin.h>
#include <cuda_runtime.h>

__global__ void k_work(int* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(x, 1);
}
__global__ void k_publish(const int* x, volatile int* val, volatile unsigned* seq, unsigned s) {
  *val = *x;
  __threadfence_system();
  *seq = s;
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  int* d;
  cudaMalloc(&d, 4);
  cudaMemset(d, 0, 4);
  int* hp;
  cudaHostAlloc(&hp, 64, cudaHostAllocMapped);
  volatile int* hval = hp;
  volatile unsigned* hseq = (volatile unsigned*)(hp + 8);
  *hseq = 0;
  const int iters = 2000;
  for (int mode = 0; mode < 3; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      auto t0 = std::chrono::steady_clock::now();
      long sum = 0;
      for (int it = 1; it <= iters; it++) {
        k_work<<<4, 128, 0, st>>>(d, 512);
        k_work<<<4, 128, 0, st>>>(d, 512);
        if (mode == 0) {
          cudaMemcpyAsync(hp, d, 4, cudaMemcpyDeviceToHost, st);
          cudaStreamSynchronize(st);
          sum += hp[0];
        } else {
          unsigned s = (unsigned)(mode * 100000 + rep * 10000 + it);
          k_publish<<<1, 1, 0, st>>>(d, (int*)hval, (unsigned*)hseq, s);
          if (mode == 1) {
            while (*hseq != s) _mm_pause();
          } else {
            cudaStreamSynchronize(st);
          }
          sum += *hval;
        }
      }
      double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters;
      printf("mode %c rep %d: %.2f us per (2 kernels + read-back)  [%ld]\n", "ABC"[mode], rep, us, sum);
    }
  }
  // baseline: the two kernels alone, one sync at the end
  auto t0 = std::chrono::steady_clock::now();
  for (int it = 0; it < iters; it++) {
    k_work<<<4, 128, 0, st>>>(d, 512);
    k_work<<<4, 128, 0, st>>>(d, 512);
  }
  cudaStreamSynchronize(st);
  printf("no read-back: %.2f us per 2 kernels\n",
         std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / iters);
  return 0;
}
