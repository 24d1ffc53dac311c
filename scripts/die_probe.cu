// L2 die topology probe (diagnostic): which SMs and which 2 KB address chunks
// are on which die, and what the executor's message hop (producer red.add.u64
// -> consumer ld.relaxed poll) costs for each (producer die, consumer die,
// word die) combination.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o die_probe die_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long w; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory"); return w;
}
// one block per SM slot: latency (clock64 cycles per dependent load) of block's SM to chunk c
__global__ void k_lat(const unsigned long long* buf, const int* chunks, int nchunks, int reps, float* out, int* sm_of) {
  if (threadIdx.x) return;
  sm_of[blockIdx.x] = (int)smid();
  for (int i = 0; i < nchunks; ++i) {
    const unsigned long long* p = buf + (size_t)chunks[i] * 256;  // 2 KB chunk = 256 words
    unsigned long long x = 0;
    ld_relaxed(p);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) x += ld_relaxed(p + (x & 1));  // dependent chain
    const long long t1 = clock64();
    out[blockIdx.x * nchunks + i] = (float)(t1 - t0) / reps + (x == 12345 ? 1.f : 0.f);
  }
}
// ping-pong pairs: block 2p (producer side A) and 2p+1; words at given chunks
__global__ void k_pp(unsigned long long* buf, const int* wa, const int* wb, int rounds, unsigned long long* out_ns, int* sm_of) {
  if (threadIdx.x) return;
  const int pair = blockIdx.x >> 1, me = blockIdx.x & 1;
  sm_of[blockIdx.x] = (int)smid();
  unsigned long long* mine = buf + (size_t)(me ? wb[pair] : wa[pair]) * 256;
  unsigned long long* other = buf + (size_t)(me ? wa[pair] : wb[pair]) * 256;
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
  int nsm = 0; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 64ull << 20, nchunk_all = bytes / 2048;
  unsigned long long* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 0, bytes);
  // 1) every SM against 64 chunks
  const int NC = 64;
  std::vector<int> ch(NC); for (int i = 0; i < NC; ++i) ch[i] = i * 97 % (int)nchunk_all;
  int *d_ch, *d_sm; float* d_lat;
  cudaMalloc(&d_ch, 4 * 4096); cudaMalloc(&d_sm, 4 * 1024); cudaMalloc(&d_lat, 4 * 1024 * 4096);
  cudaMemcpy(d_ch, ch.data(), 4 * NC, cudaMemcpyHostToDevice);
  k_lat<<<nsm, 32>>>(buf, d_ch, NC, 200, d_lat, d_sm);
  cudaDeviceSynchronize();
  std::vector<float> lat(nsm * NC); std::vector<int> sm(nsm);
  cudaMemcpy(lat.data(), d_lat, 4 * nsm * NC, cudaMemcpyDeviceToHost);
  cudaMemcpy(sm.data(), d_sm, 4 * nsm, cudaMemcpyDeviceToHost);
  // classify chunks by block 0's latency (bimodal), SMs by agreement with block 0
  std::vector<float> l0(lat.begin(), lat.begin() + NC);
  std::vector<float> s = l0; std::sort(s.begin(), s.end());
  const float thr = (s.front() + s.back()) / 2;
  printf("block0 (sm %d) latency to %d chunks: min %.0f max %.0f cycles (threshold %.0f)\n", sm[0], NC, s.front(), s.back(), thr);
  std::vector<int> chunk_near(NC); for (int i = 0; i < NC; ++i) chunk_near[i] = l0[i] < thr;
  std::vector<int> sm_die(1024, -1);
  int same = 0;
  for (int b = 0; b < nsm; ++b) {
    int agree = 0;
    for (int i = 0; i < NC; ++i) agree += ((lat[b * NC + i] < thr) == chunk_near[i]);
    sm_die[sm[b]] = agree > NC / 2 ? 0 : 1;  // 0: same die as block 0
    same += sm_die[sm[b]] == 0;
  }
  printf("SMs on block 0's die: %d of %d\n", same, nsm);
  float near_avg = 0, far_avg = 0; int nn = 0, nf = 0;
  for (int i = 0; i < NC; ++i) (chunk_near[i] ? (near_avg += l0[i], ++nn) : (far_avg += l0[i], ++nf));
  printf("block 0 load latency: near chunks %.0f cycles (%d), far chunks %.0f (%d)\n", near_avg / std::max(nn, 1), nn, far_avg / std::max(nf, 1), nf);
  // 2) classify more chunks by block 0 (for pairing)
  const int NC2 = 512;
  std::vector<int> ch2(NC2); for (int i = 0; i < NC2; ++i) ch2[i] = (i * 131 + 7) % (int)nchunk_all;
  cudaMemcpy(d_ch, ch2.data(), 4 * NC2, cudaMemcpyHostToDevice);
  k_lat<<<1, 32>>>(buf, d_ch, NC2, 100, d_lat, d_sm);
  cudaDeviceSynchronize();
  std::vector<float> l2(NC2); cudaMemcpy(l2.data(), d_lat, 4 * NC2, cudaMemcpyDeviceToHost);
  std::vector<int> near_chunks, far_chunks;
  for (int i = 0; i < NC2; ++i) (l2[i] < thr ? near_chunks : far_chunks).push_back(ch2[i]);
  // 3) ping-pong: 74 pairs (148 blocks, one per SM), words chosen near/far to block 0's die
  const int P = nsm / 2;
  int *d_wa, *d_wb; unsigned long long* d_out;
  cudaMalloc(&d_wa, 4 * P); cudaMalloc(&d_wb, 4 * P); cudaMalloc(&d_out, 8 * P);
  for (int mode = 0; mode < 4; ++mode) {  // word A / word B die: 00 near-near, 01, 10, 11 (relative to block 0's die)
    std::vector<int> wa(P), wb(P);
    for (int p = 0; p < P; ++p) {
      // (distinct chunks for every pair: pairs sharing a word would count each
      // other's messages, which made an early version read ~150 ns)
      const auto& A = (mode & 1) ? far_chunks : near_chunks;
      const auto& B = (mode & 2) ? far_chunks : near_chunks;
      wa[p] = A[(2 * p) % A.size()];
      wb[p] = B[(2 * p + 1) % B.size()];
    }
    cudaMemset(buf, 0, bytes);
    cudaMemcpy(d_wa, wa.data(), 4 * P, cudaMemcpyHostToDevice);
    cudaMemcpy(d_wb, wb.data(), 4 * P, cudaMemcpyHostToDevice);
    const int rounds = 5000;
    k_pp<<<2 * P, 32>>>(buf, d_wa, d_wb, rounds, d_out, d_sm);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> o(P); cudaMemcpy(o.data(), d_out, 8 * P, cudaMemcpyDeviceToHost);
    std::vector<int> smp(2 * P); cudaMemcpy(smp.data(), d_sm, 4 * 2 * P, cudaMemcpyDeviceToHost);
    // group by (die of A's SM, die of B's SM): the word mine of A is wa (A polls wa, B reds into wa)
    double acc[2][2] = {{0, 0}, {0, 0}}; int cnt[2][2] = {{0, 0}, {0, 0}};
    for (int p = 0; p < P; ++p) {
      const int da = sm_die[smp[2 * p]], db = sm_die[smp[2 * p + 1]];
      if (da < 0 || db < 0) continue;
      acc[da][db] += (double)o[p] / (2.0 * rounds); cnt[da][db]++;
    }
    printf("words A:%s B:%s (rel. die 0) | one-way hop ns by (SM A die, SM B die): ", (mode & 1) ? "far" : "near", (mode & 2) ? "far" : "near");
    for (int a = 0; a < 2; ++a) for (int b = 0; b < 2; ++b) printf(" [%d%d] %.0f (n=%d)", a, b, cnt[a][b] ? acc[a][b] / cnt[a][b] : 0.0, cnt[a][b]);
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
