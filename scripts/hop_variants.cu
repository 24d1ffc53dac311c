// Why two ping-pong harnesses disagree (150 vs 250-480 ns one-way): the same
// kernel under launch / rounds / pair-count / word-layout variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hop_variants hop_variants.cu
#include <cstdio>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long w; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory"); return w;
}
__global__ void k_pp(unsigned long long* buf, const long long* wa, const long long* wb, int rounds, unsigned long long* out_ns) {
  if (threadIdx.x) return;
  const int pair = blockIdx.x >> 1, me = blockIdx.x & 1;
  unsigned long long* mine = buf + (me ? wb[pair] : wa[pair]);
  unsigned long long* other = buf + (me ? wa[pair] : wb[pair]);
  unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < rounds; ++r) {
    if (me == 0) {
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(other) : "memory");
      while (ld_relaxed(mine) < (unsigned long long)(r + 1)) {}
    } else {
      while (ld_relaxed(mine) < (unsigned long long)(r + 1)) {}
      asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(other) : "memory");
    }
  }
  unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (me == 0) out_ns[pair] = t1 - t0;
}
int main() {
  const size_t bytes = 64ull << 20;
  unsigned long long* buf; cudaMalloc(&buf, bytes);
  long long *d_wa, *d_wb; unsigned long long* d_out;
  cudaMalloc(&d_wa, 8 * 128); cudaMalloc(&d_wb, 8 * 128); cudaMalloc(&d_out, 8 * 128);
  for (int layout = 0; layout < 3; ++layout)
    for (int pairs : {16, 74})
      for (int coop = 0; coop < 2; ++coop)
        for (int rounds : {5000, 20000}) {
          std::vector<long long> wa(pairs), wb(pairs);
          for (int p = 0; p < pairs; ++p) {
            if (layout == 0) { wa[p] = (2LL * p) * 32; wb[p] = (2LL * p + 1) * 32; }                 // 256 B apart
            else if (layout == 1) { wa[p] = (2LL * p) * 512; wb[p] = (2LL * p + 1) * 512; }          // 4 KB apart
            else { wa[p] = ((2LL * p * 131 + 7) % 32768) * 256; wb[p] = (((2LL * p + 1) * 131 + 7) % 32768) * 256; }  // scattered 2 KB chunks
          }
          cudaMemset(buf, 0, bytes);
          cudaMemcpy(d_wa, wa.data(), 8 * pairs, cudaMemcpyHostToDevice);
          cudaMemcpy(d_wb, wb.data(), 8 * pairs, cudaMemcpyHostToDevice);
          void* args[] = {&buf, &d_wa, &d_wb, &rounds, &d_out};
          if (coop) cudaLaunchCooperativeKernel((void*)k_pp, dim3(2 * pairs), dim3(32), args, 0, 0);
          else k_pp<<<2 * pairs, 32>>>(buf, d_wa, d_wb, rounds, d_out);
          cudaDeviceSynchronize();
          std::vector<unsigned long long> o(pairs); cudaMemcpy(o.data(), d_out, 8 * pairs, cudaMemcpyDeviceToHost);
          std::vector<double> v(pairs); for (int p = 0; p < pairs; ++p) v[p] = o[p] / (2.0 * rounds);
          std::sort(v.begin(), v.end());
          printf("layout %s pairs %2d %s rounds %5d: min %.0f median %.0f max %.0f ns\n",
                 layout == 0 ? "256B " : layout == 1 ? "4KB  " : "rand2K", pairs, coop ? "coop " : "plain", rounds,
                 v[0], v[pairs / 2], v[pairs - 1]);
        }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
