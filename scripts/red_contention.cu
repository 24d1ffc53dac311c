// Same-address RED throughput on B200: W warps, lane 0 of each issues M
// red.add.u64 into one of A words (word = warp % A, 256 B apart), optionally
// with P polling warps reading the same words (8 lanes each, like a bundled
// consumer).  Timed on the device (%globaltimer, first RED to last RED).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_contention red_contention.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k_red(unsigned long long* w, int A, int M, int pollers, int* done, unsigned long long* tt, int nred) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  if (warp >= nw - pollers) {
    unsigned long long s = 0;
    while (*(volatile int*)done < nred) {
      if (lane < 8) {
        unsigned long long x;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(w + (size_t)((warp + lane) % A) * 32));
        s += x;
      }
    }
    if (s == 42) w[0] = s;
    return;
  }
  if (lane != 0) return;
  unsigned long long* p = w + (size_t)(warp % A) * 32;
  const unsigned long long t0 = gt();
  for (int i = 0; i < M; ++i) asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" :: "l"(p) : "memory");
  __threadfence();
  const unsigned long long t1 = gt();
  atomicMin(&tt[0], t0);
  atomicMax(&tt[1], t1);
  atomicAdd(done, 1);
}
int main() {
  unsigned long long *w, *tt; int* done;
  cudaMalloc(&w, 1 << 24); cudaMalloc(&done, 4); cudaMalloc(&tt, 16);
  const int M = 256;
  for (int pollers : {0, 1024, 3072}) {
    for (int A : {1, 8, 64, 128, 512, 4096}) {
      for (int W : {1024, 4096}) {
        cudaMemset(w, 0, 1 << 24); cudaMemset(done, 0, 4);
        unsigned long long init[2] = {~0ull, 0};
        cudaMemcpy(tt, init, 16, cudaMemcpyHostToDevice);
        k_red<<<(W + pollers) / 4, 128>>>(w, A, M, pollers, done, tt, W);
        cudaDeviceSynchronize();
        unsigned long long h[2]; cudaMemcpy(h, tt, 16, cudaMemcpyDeviceToHost);
        const double ns = (double)(h[1] - h[0]);
        printf("pollers %4d  words %5d  warps %5d  REDs %8d  %9.1f us  %.3e REDs/s  %6.2f ns per RED on one word\n", pollers,
               A, W, W * M, ns / 1e3, W * (double)M / (ns * 1e-9), ns / ((double)W * M / A));
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
