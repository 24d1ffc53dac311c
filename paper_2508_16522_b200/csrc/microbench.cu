// microbench.cu — K3 roofline microbenchmarks for the executor (SURVEY.md §7
// step 1, §8(d)): the denominators of R_roof = min(A_L2/atomics_task,
// BW/bytes_task, W_active/L_level).
//   td_mb_atomic_rate   : L2 atomic throughput (red / atom, distinct or shared)
//   td_mb_flag_latency  : one-way dependent-chain latency between two SMs via
//                         an L2 flag (the executor's signal hop)
//   td_mb_launch_latency: empty-kernel launch cost, stream and CUDA-graph
//   td_mb_p2p_latency   : one-way flag latency GPU->GPU over NVLink
//   td_mb_compute_peak  : chip peak of the compute_bound body (u64 LCG lane-updates/s)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

extern "C" {

static char mb_err[256];
const char* td_mb_last_error(void) { return mb_err; }
#define MB_TRY(x)                                                                     \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      snprintf(mb_err, sizeof mb_err, "%s: %s", #x, cudaGetErrorString(e_));          \
      return -1.0;                                                                    \
    }                                                                                 \
  } while (0)
}

__global__ void k_red(uint32_t* base, int mode, int iters) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  // mode 0: distinct addresses (one 128B line per warp lane group); 1: one address
  uint32_t* p = mode == 0 ? base + (size_t)tid * 32 : base;
  for (int i = 0; i < iters; ++i) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__global__ void k_atom(uint32_t* base, int mode, int iters, uint32_t* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t* p = mode == 0 ? base + (size_t)tid * 32 : base;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) acc += atomicAdd(p, 1u);
  if (acc == 0xFFFFFFFFu) *sink = acc;
}

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acq_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Ping-pong between block 0 and block 1 (different SMs): the executor's hop.
// mode 0: fence.acq_rel + red.relaxed      mode 1: red.release
// mode 2: token store + fence + red        mode 3: token store + red.release
// mode 4: token store + st.release flag (no counter)
__device__ __forceinline__ void hop_signal(uint32_t* other, unsigned long long* tok, int mode, int r) {
  if (mode >= 2) tok[0] = (unsigned long long)r * 0x9E3779B97F4A7C15ull;
  if (mode == 0 || mode == 2) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(other) : "memory");
  } else if (mode == 1 || mode == 3) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(other) : "memory");
  } else {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(other), "r"((uint32_t)(r + 1)) : "memory");
  }
}

__global__ void k_pingpong(uint32_t* flags, int rounds, int mode, unsigned long long* toks, unsigned long long* out_ns) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;
  uint32_t* mine = flags + me * 32;
  uint32_t* other = flags + (1 - me) * 32;
  unsigned long long* mytok = toks + me * 16;
  unsigned long long* othertok = toks + (1 - me) * 16;
  unsigned long long sink = 0;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < rounds; ++r) {
    if (me == 0) {
      hop_signal(other, mytok, mode, r);
      while (ld_acq(mine) < (uint32_t)(r + 1)) {}
      if (mode >= 2) sink += __ldcg(othertok);
    } else {
      while (ld_acq(mine) < (uint32_t)(r + 1)) {}
      if (mode >= 2) sink += __ldcg(othertok);
      hop_signal(other, mytok, mode, r);
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (me == 0) *out_ns = t1 - t0;
  if (sink == 1) out_ns[1] = sink;
}

__global__ void k_pingpong_p2p(uint32_t* mine, uint32_t* other, int me, int rounds, unsigned long long* out_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < rounds; ++r) {
    if (me == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(other) : "memory");
      while (ld_acq_sys(mine) < (uint32_t)(r + 1)) {}
    } else {
      while (ld_acq_sys(mine) < (uint32_t)(r + 1)) {}
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" ::"l"(other) : "memory");
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  *out_ns = t1 - t0;
}

// The executor's actual message hop: producer red.add.u64 into the consumer's
// mailbox word, consumer polls it with ld.relaxed.gpu.u64 (no fence, no token
// load).  Pairs (2p, 2p+1) ping-pong independently so SM / die placement is
// sampled; out_ns[p] = one-way hop of pair p.
template <bool SYS>
__device__ __forceinline__ void mb_red(unsigned long long* p) {
  if (SYS) asm volatile("red.relaxed.sys.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
  else asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(p) : "memory");
}
template <bool SYS>
__device__ __forceinline__ unsigned long long mb_ld(const unsigned long long* p) {
  unsigned long long w;
  if (SYS) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  else asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

template <bool SYS>
__global__ void k_pingpong_mbox(unsigned long long* words, int rounds, unsigned long long* out_ns, int stride) {
  if (threadIdx.x != 0) return;
  const int pair = blockIdx.x >> 1, me = blockIdx.x & 1;
  unsigned long long* mine = words + (size_t)(2 * pair + me) * stride;
  unsigned long long* other = words + (size_t)(2 * pair + (1 - me)) * stride;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < rounds; ++r) {
    if (me == 0) {
      mb_red<SYS>(other);
      while (mb_ld<SYS>(mine) < (unsigned long long)(r + 1)) {}
    } else {
      while (mb_ld<SYS>(mine) < (unsigned long long)(r + 1)) {}
      mb_red<SYS>(other);
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (me == 0) out_ns[pair] = t1 - t0;
}

// GPU<->GPU mailbox hop: red.relaxed.sys into the peer's word, poll own word.
__global__ void k_pingpong_mbox_p2p(unsigned long long* mine, unsigned long long* other, int me, int rounds,
                                    unsigned long long* out_ns) {
  if (threadIdx.x != 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < rounds; ++r) {
    if (me == 0) {
      mb_red<true>(other);
      while (mb_ld<true>(mine) < (unsigned long long)(r + 1)) {}
    } else {
      while (mb_ld<true>(mine) < (unsigned long long)(r + 1)) {}
      mb_red<true>(other);
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  *out_ns = t1 - t0;
}

// Cluster / CTA mailbox hop: the message is a red.add.u64 into the peer's
// SHARED-memory word (distributed shared memory across the CTAs of a cluster,
// or plain shared memory between two warps of one CTA); the receiver polls
// its own shared word.  mode 0: CTA ranks 0 and 1 of a 2-CTA cluster; mode 1:
// warps 0 and 1 of one CTA.
__global__ void k_pingpong_dsmem(int rounds, int mode, unsigned long long* out_ns) {
  __shared__ unsigned long long box[2];
  if (threadIdx.x < 2) box[threadIdx.x] = 0;
  asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int me = mode == 0 ? (int)crank : warp;
  if (lane != 0 || (mode == 1 && warp > 1) || (mode == 0 && warp != 0)) {
    if (mode == 0)  // the peer's shared word must outlive its sender
      asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
    return;
  }
  const uint32_t mine = (uint32_t)__cvta_generic_to_shared(&box[mode == 0 ? 0 : me]);
  uint32_t other = (uint32_t)__cvta_generic_to_shared(&box[mode == 0 ? 0 : 1 - me]);
  if (mode == 0) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(other) : "r"(other), "r"(1u - crank));
  unsigned long long t0, t1, w;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int r = 0; r < rounds; ++r) {
    if (me == 1) {
      do { asm volatile("ld.relaxed.cluster.shared.u64 %0, [%1];" : "=l"(w) : "r"(mine) : "memory"); }
      while (w < (unsigned long long)(r + 1));
    }
    if (mode == 0) asm volatile("red.relaxed.cluster.shared::cluster.add.u64 [%0], 1;" ::"r"(other) : "memory");
    else asm volatile("red.relaxed.cta.shared.add.u64 [%0], 1;" ::"r"(other) : "memory");
    if (me == 0) {
      do { asm volatile("ld.relaxed.cluster.shared.u64 %0, [%1];" : "=l"(w) : "r"(mine) : "memory"); }
      while (w < (unsigned long long)(r + 1));
    }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  const unsigned cl = mode == 0 ? blockIdx.x / 2 : blockIdx.x;
  if (me == 0) out_ns[cl] = t1 - t0;
  if (mode == 0)
    asm volatile("barrier.cluster.arrive.release; barrier.cluster.wait.acquire;" ::: "memory");
}

// Floor of one node's dependent arithmetic (the executor's token rule with a
// compute_bound(1) body, fed through a shared-memory ring as for a same-worker
// chain): no descriptors, no mailboxes, no bookkeeping.  One warp per CTA
// runs T nodes; out_cycles = clock64 cycles for the T nodes.
__device__ __forceinline__ uint64_t fl_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void k_chain_floor(int T, uint64_t seed, unsigned long long* out_cycles, unsigned long long* sink) {
  __shared__ uint64_t ring[64];
  const int lane = threadIdx.x & 31;
  if (lane == 0) ring[0] = 0;
  __syncwarp();
  const uint64_t G1 = 0x9E3779B97F4A7C15ull, G2 = 0xD1B54A32D192ED03ull, G3 = 0x8CB92BA72F3D8DD7ull;
  const uint64_t A = 6364136223846793005ull, C = 1442695040888963407ull;
  uint64_t acc = 0;
  const long long t0 = clock64();
  for (int t = 0; t < T; ++t) {
    const uint64_t v = (uint64_t)blockIdx.x * T + t;
    const uint64_t h0 = fl_mix64(seed ^ fl_mix64(v + G1));   // (the executor precomputes the inner hash)
    const uint64_t sum = ring[t & 63];
    const uint64_t h = fl_mix64(h0 ^ sum);
    uint64_t x0 = fl_mix64(h ^ ((uint64_t)(lane + 1) * G2)), x1 = fl_mix64(h ^ ((uint64_t)(lane + 33) * G2));
    x0 = A * x0 + C;
    x1 = A * x1 + C;
    const uint64_t y = x0 ^ x1;
    const uint32_t lo = __reduce_xor_sync(0xffffffffu, (uint32_t)y), hi = __reduce_xor_sync(0xffffffffu, (uint32_t)(y >> 32));
    const uint64_t tok = h ^ (((uint64_t)hi << 32) | lo);
    const uint64_t term = fl_mix64(tok ^ fl_mix64(v + G3)) >> 32;
    if (lane == 0) ring[(t + 1) & 63] = sum * 0 + term;
    __syncwarp();
    acc ^= tok;
  }
  const long long t1 = clock64();
  if (lane == 0) {
    out_cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    sink[blockIdx.x] = acc;
  }
}


// Chip peak of the compute_bound body's unit of work (one
// "lane-update" = x <- A*x + C in u64): every resident thread runs CHAINS
// independent LCG chains, the loop unrolled by 8.  This is the fixed
// denominator of METG efficiency (PAPER.md:951-965 normalises to the machine's
// peak), independent of how any executor configuration performs.
template <int CHAINS>
__global__ void __launch_bounds__(128) k_lcg_peak(int iters, unsigned long long* sink) {
  const uint64_t A = 6364136223846793005ull, C = 1442695040888963407ull;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t x[CHAINS];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) x[k] = fl_mix64(tid * CHAINS + k);
  for (int i = 0; i < iters; i += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int k = 0; k < CHAINS; ++k) {
        x[k] = A * x[k] + C;
        asm volatile("" : "+l"(x[k]));  // opaque: no folding of 8 affine steps into one
      }
  }
  uint64_t r = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) r ^= x[k];
  if (r == 0x5EED5EED5EED5EEDull) sink[0] = r;
}

__global__ void k_empty() {}

extern "C" {

// Returns atomic ops per second.
double td_mb_atomic_rate(int device, int use_atom, int shared_addr, int blocks, int threads, int iters) {
  MB_TRY(cudaSetDevice(device));
  uint32_t *buf, *sink;
  const size_t n = (size_t)blocks * threads * 32 + 32;
  MB_TRY(cudaMalloc(&buf, n * sizeof(uint32_t)));
  MB_TRY(cudaMalloc(&sink, 4));
  MB_TRY(cudaMemset(buf, 0, n * sizeof(uint32_t)));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    if (use_atom) k_atom<<<blocks, threads>>>(buf, shared_addr, iters, sink);
    else k_red<<<blocks, threads>>>(buf, shared_addr, iters);
    cudaEventRecord(b);
    MB_TRY(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0 && ms < best) best = ms;
  }
  MB_TRY(cudaGetLastError());
  cudaFree(buf);
  cudaFree(sink);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return (double)blocks * threads * iters / (best * 1e-3);
}

// Returns one-way latency in ns of a signal hop between SMs (mode: see k_pingpong).
double td_mb_flag_latency(int device, int rounds, int mode) {
  MB_TRY(cudaSetDevice(device));
  uint32_t* flags;
  unsigned long long *out, *toks;
  MB_TRY(cudaMalloc(&flags, 64 * sizeof(uint32_t)));
  MB_TRY(cudaMalloc(&out, 16));
  MB_TRY(cudaMalloc(&toks, 64 * sizeof(unsigned long long)));
  double best = 1e30;
  for (int rep = 0; rep < 3; ++rep) {
    MB_TRY(cudaMemset(flags, 0, 64 * sizeof(uint32_t)));
    void* args[] = {&flags, &rounds, &mode, &toks, &out};
    MB_TRY(cudaLaunchCooperativeKernel((const void*)k_pingpong, dim3(2), dim3(32), args, 0, 0));
    MB_TRY(cudaDeviceSynchronize());
    unsigned long long ns;
    MB_TRY(cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost));
    const double one_way = (double)ns / (2.0 * rounds);
    if (one_way < best) best = one_way;
  }
  cudaFree(flags);
  cudaFree(out);
  cudaFree(toks);
  return best;
}

// Median / min one-way mailbox hop over `pairs` concurrent CTA pairs (ns),
// the words `stride` u64 apart.  The hop depends on where the two words and
// SMs sit: over 16 / 74 pairs the minimum is 232-246 ns on every box and
// layout measured, the median 272-480 ns depending on the layout
// (scripts/hop_variants.cu, profiles/r02_hop_variants.log).
double td_mb_mailbox_hop_strided(int device, int pairs, int rounds, double* min_out, int sys_scope, int stride) {
  MB_TRY(cudaSetDevice(device));
  unsigned long long *words, *out;
  MB_TRY(cudaMalloc(&words, (size_t)pairs * 2 * stride * 8));
  MB_TRY(cudaMalloc(&out, (size_t)pairs * 8));
  MB_TRY(cudaMemset(words, 0, (size_t)pairs * 2 * stride * 8));
  void* args[] = {&words, &rounds, &out, &stride};
  const void* fn = sys_scope ? (const void*)k_pingpong_mbox<true> : (const void*)k_pingpong_mbox<false>;
  MB_TRY(cudaLaunchCooperativeKernel(fn, dim3(2 * pairs), dim3(32), args, 0, 0));
  MB_TRY(cudaDeviceSynchronize());
  unsigned long long* h = new unsigned long long[pairs];
  MB_TRY(cudaMemcpy(h, out, (size_t)pairs * 8, cudaMemcpyDeviceToHost));
  double* v = new double[pairs];
  for (int i = 0; i < pairs; ++i) v[i] = (double)h[i] / (2.0 * rounds);
  for (int i = 1; i < pairs; ++i)  // insertion sort (tiny)
    for (int j = i; j > 0 && v[j] < v[j - 1]; --j) { double t = v[j]; v[j] = v[j - 1]; v[j - 1] = t; }
  const double med = v[pairs / 2];
  if (min_out) *min_out = v[0];
  delete[] h;
  delete[] v;
  cudaFree(words);
  cudaFree(out);
  return med;
}
double td_mb_mailbox_hop(int device, int pairs, int rounds, double* min_out, int sys_scope) {
  return td_mb_mailbox_hop_strided(device, pairs, rounds, min_out, sys_scope, 32);
}

// Median one-way shared-memory mailbox hop (ns) over `pairs` concurrent
// pairs: mode 0 = two CTAs of a cluster (DSMEM), mode 1 = two warps of a CTA.
double td_mb_dsmem_hop(int device, int pairs, int rounds, int mode, double* min_out) {
  MB_TRY(cudaSetDevice(device));
  unsigned long long* out;
  MB_TRY(cudaMalloc(&out, (size_t)pairs * 8));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(mode == 0 ? 2 * pairs : pairs);
  cfg.blockDim = dim3(mode == 0 ? 32 : 64);
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = mode == 0 ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  MB_TRY(cudaLaunchKernelEx(&cfg, k_pingpong_dsmem, rounds, mode, out));
  MB_TRY(cudaDeviceSynchronize());
  unsigned long long* h = new unsigned long long[pairs];
  MB_TRY(cudaMemcpy(h, out, (size_t)pairs * 8, cudaMemcpyDeviceToHost));
  double* v = new double[pairs];
  for (int i = 0; i < pairs; ++i) v[i] = (double)h[i] / (2.0 * rounds);
  for (int i = 1; i < pairs; ++i)
    for (int j = i; j > 0 && v[j] < v[j - 1]; --j) { double t = v[j]; v[j] = v[j - 1]; v[j - 1] = t; }
  const double med = v[pairs / 2];
  if (min_out) *min_out = v[0];
  delete[] h;
  delete[] v;
  cudaFree(out);
  return med;
}

// Lane-updates per second of k_lcg_peak<chains> over `blocks` CTAs of
// `threads` threads (148 x 8 x 128 = the executor's lean geometry, 32 warps
// per SM; 148 x 32 = one warp per SM); best of `reps`.
double td_mb_compute_peak(int device, int chains, int blocks, int threads, int iters, int reps) {
  MB_TRY(cudaSetDevice(device));
  unsigned long long* sink;
  MB_TRY(cudaMalloc(&sink, 8));
  cudaEvent_t a, b;
  MB_TRY(cudaEventCreate(&a));
  MB_TRY(cudaEventCreate(&b));
  if (threads < 32 || threads > 128 || threads % 32) {
    snprintf(mb_err, sizeof mb_err, "threads must be 32..128, a multiple of 32");
    return -1.0;
  }
  iters = (iters + 7) / 8 * 8;
  double best = 0;
  for (int r = 0; r <= reps; ++r) {  // r == 0: warm-up
    MB_TRY(cudaEventRecord(a));
    if (chains == 2) k_lcg_peak<2><<<blocks, threads>>>(iters, sink);
    else if (chains == 4) k_lcg_peak<4><<<blocks, threads>>>(iters, sink);
    else if (chains == 8) k_lcg_peak<8><<<blocks, threads>>>(iters, sink);
    else { snprintf(mb_err, sizeof mb_err, "chains must be 2, 4 or 8"); return -1.0; }
    MB_TRY(cudaEventRecord(b));
    MB_TRY(cudaEventSynchronize(b));
    float ms = 0;
    MB_TRY(cudaEventElapsedTime(&ms, a, b));
    const double rate = (double)blocks * threads * chains * iters / (ms * 1e-3);
    if (r > 0 && rate > best) best = rate;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return best;
}

// The same kernel run back to back for `seconds`: the median rate of the
// launches in the second half (the sustained rate, after clocks settle under
// the load's power draw), for comparison with long METG sweep points.
double td_mb_compute_peak_sustained(int device, int chains, int blocks, int threads, int iters, double seconds) {
  MB_TRY(cudaSetDevice(device));
  if (chains != 2 && chains != 4 && chains != 8) { snprintf(mb_err, sizeof mb_err, "chains must be 2, 4 or 8"); return -1.0; }
  unsigned long long* sink;
  MB_TRY(cudaMalloc(&sink, 8));
  cudaEvent_t a, b;
  MB_TRY(cudaEventCreate(&a));
  MB_TRY(cudaEventCreate(&b));
  iters = (iters + 7) / 8 * 8;
  double* rates = new double[100000];
  int nr = 0;
  double elapsed = 0;
  while (elapsed < seconds * 1e3 && nr < 100000) {
    MB_TRY(cudaEventRecord(a));
    if (chains == 2) k_lcg_peak<2><<<blocks, threads>>>(iters, sink);
    else if (chains == 4) k_lcg_peak<4><<<blocks, threads>>>(iters, sink);
    else k_lcg_peak<8><<<blocks, threads>>>(iters, sink);
    MB_TRY(cudaEventRecord(b));
    MB_TRY(cudaEventSynchronize(b));
    float ms = 0;
    MB_TRY(cudaEventElapsedTime(&ms, a, b));
    elapsed += ms;
    rates[nr++] = (double)blocks * threads * chains * iters / (ms * 1e-3);
  }
  const int lo = nr / 2;
  for (int i = lo + 1; i < nr; ++i)  // insertion sort of the second half
    for (int j = i; j > lo && rates[j] < rates[j - 1]; --j) { const double t = rates[j]; rates[j] = rates[j - 1]; rates[j - 1] = t; }
  const double med = nr > 0 ? rates[lo + (nr - lo) / 2] : 0.0;
  delete[] rates;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return med;
}

// Cycles per node of k_chain_floor (median over `warps` single-warp CTAs).
double td_mb_chain_floor(int device, int warps, int T) {
  MB_TRY(cudaSetDevice(device));
  unsigned long long *out, *sink;
  MB_TRY(cudaMalloc(&out, (size_t)warps * 8));
  MB_TRY(cudaMalloc(&sink, (size_t)warps * 8));
  k_chain_floor<<<warps, 32>>>(T, 1ull, out, sink);
  MB_TRY(cudaGetLastError());
  MB_TRY(cudaDeviceSynchronize());
  unsigned long long* h = new unsigned long long[warps];
  MB_TRY(cudaMemcpy(h, out, (size_t)warps * 8, cudaMemcpyDeviceToHost));
  for (int i = 1; i < warps; ++i)
    for (int j = i; j > 0 && h[j] < h[j - 1]; --j) { unsigned long long t = h[j]; h[j] = h[j - 1]; h[j - 1] = t; }
  const double med = (double)h[warps / 2] / T;
  delete[] h;
  cudaFree(out);
  cudaFree(sink);
  return med;
}

// GPU<->GPU mailbox hop (ns) between dev0 and dev1 (peer access enabled).
double td_mb_p2p_mailbox_hop(int dev0, int dev1, int rounds) {
  unsigned long long *f0, *f1, *o0, *o1;
  MB_TRY(cudaSetDevice(dev0));
  cudaError_t pe = cudaDeviceEnablePeerAccess(dev1, 0);
  if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) MB_TRY(pe);
  cudaGetLastError();
  MB_TRY(cudaMalloc(&f0, 256));
  MB_TRY(cudaMemset(f0, 0, 256));
  MB_TRY(cudaMalloc(&o0, 8));
  MB_TRY(cudaSetDevice(dev1));
  pe = cudaDeviceEnablePeerAccess(dev0, 0);
  if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) MB_TRY(pe);
  cudaGetLastError();
  MB_TRY(cudaMalloc(&f1, 256));
  MB_TRY(cudaMemset(f1, 0, 256));
  MB_TRY(cudaMalloc(&o1, 8));
  MB_TRY(cudaDeviceSynchronize());
  k_pingpong_mbox_p2p<<<1, 32>>>(f1, f0, 1, rounds, o1);
  MB_TRY(cudaSetDevice(dev0));
  k_pingpong_mbox_p2p<<<1, 32>>>(f0, f1, 0, rounds, o0);
  MB_TRY(cudaDeviceSynchronize());
  MB_TRY(cudaSetDevice(dev1));
  MB_TRY(cudaDeviceSynchronize());
  unsigned long long ns;
  MB_TRY(cudaSetDevice(dev0));
  MB_TRY(cudaMemcpy(&ns, o0, 8, cudaMemcpyDeviceToHost));
  cudaFree(f0);
  cudaFree(o0);
  MB_TRY(cudaSetDevice(dev1));
  cudaFree(f1);
  cudaFree(o1);
  return (double)ns / (2.0 * rounds);
}

// mode 0: back-to-back <<<>>> launches (us per launch, device-timed);
// mode 1: CUDA graph of `count` empty kernel nodes (us per node).
double td_mb_launch_latency(int device, int mode, int count) {
  MB_TRY(cudaSetDevice(device));
  cudaStream_t s;
  MB_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0;
  if (mode == 0) {
    for (int i = 0; i < 100; ++i) k_empty<<<1, 32, 0, s>>>();
    cudaEventRecord(a, s);
    for (int i = 0; i < count; ++i) k_empty<<<1, 32, 0, s>>>();
    cudaEventRecord(b, s);
  } else {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    MB_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < count; ++i) k_empty<<<1, 32, 0, s>>>();
    MB_TRY(cudaStreamEndCapture(s, &g));
    MB_TRY(cudaGraphInstantiate(&ge, g, 0));
    MB_TRY(cudaGraphLaunch(ge, s));
    MB_TRY(cudaStreamSynchronize(s));
    cudaEventRecord(a, s);
    MB_TRY(cudaGraphLaunch(ge, s));
    cudaEventRecord(b, s);
    MB_TRY(cudaStreamSynchronize(s));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  MB_TRY(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaStreamDestroy(s);
  return ms * 1e3 / count;
}

// One-way GPU->GPU flag latency (ns) between dev0 and dev1 in ONE process
// (peer access enabled); both kernels are resident on their own GPU.
double td_mb_p2p_latency(int dev0, int dev1, int rounds) {
  uint32_t *f0, *f1;
  unsigned long long *o0, *o1;
  MB_TRY(cudaSetDevice(dev0));
  cudaError_t pe = cudaDeviceEnablePeerAccess(dev1, 0);
  if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) MB_TRY(pe);
  cudaGetLastError();
  MB_TRY(cudaMalloc(&f0, 128));
  MB_TRY(cudaMemset(f0, 0, 128));
  MB_TRY(cudaMalloc(&o0, 8));
  MB_TRY(cudaSetDevice(dev1));
  pe = cudaDeviceEnablePeerAccess(dev0, 0);
  if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) MB_TRY(pe);
  cudaGetLastError();
  MB_TRY(cudaMalloc(&f1, 128));
  MB_TRY(cudaMemset(f1, 0, 128));
  MB_TRY(cudaMalloc(&o1, 8));
  MB_TRY(cudaDeviceSynchronize());
  MB_TRY(cudaSetDevice(dev1));
  k_pingpong_p2p<<<1, 32>>>(f1, f0, 1, rounds, o1);
  MB_TRY(cudaSetDevice(dev0));
  k_pingpong_p2p<<<1, 32>>>(f0, f1, 0, rounds, o0);
  MB_TRY(cudaDeviceSynchronize());
  MB_TRY(cudaSetDevice(dev1));
  MB_TRY(cudaDeviceSynchronize());
  unsigned long long ns;
  MB_TRY(cudaSetDevice(dev0));
  MB_TRY(cudaMemcpy(&ns, o0, 8, cudaMemcpyDeviceToHost));
  cudaFree(f0);
  cudaFree(o0);
  MB_TRY(cudaSetDevice(dev1));
  cudaFree(f1);
  cudaFree(o1);
  return (double)ns / (2.0 * rounds);
}

}  // extern "C"
