// tdexec.cu — B200 (sm_100a) persistent executor for traced task graphs.
//
// Replaces the reference's Alg. 1 interpreter (SPEC.md
// compiler 351-425): INIT / COMPLETED_EDGE / EXECUTE_OP messages between
// per-resource Worker actors become, inside ONE persistent kernel per GPU,
//   * a worker  = one resident warp owning a static, topologically ordered
//                 list of nodes (Alg. 1 V_w),
//   * a message = a release-ordered atomic increment of the successor's
//                 dependence counter in L2 (or in a peer GPU's memory over
//                 NVLink for cross-shard edges),
//   * dispatch  = the owner warp observing (acquire) that the counter reached
//                 indeg*(epoch+1).  Epoch-scaled targets replace Alg. 1's
//                 "E <- reset(E)" / SPEC.md:412's re-arm, so no counter is ever
//                 reset between replays and nothing returns to the host
//                 between tasks.
// See DESIGN.md for the memory layout and the roofline of each phase.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <stdio.h>
#include <stdarg.h>
#include <time.h>

#include <vector>

#include "../../include/tdexec.h"

#define TD_MAX_RANKS 8

namespace {

constexpr uint64_t G1 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t G2 = 0xD1B54A32D192ED03ull;
constexpr uint64_t LCG_A = 6364136223846793005ull;
constexpr uint64_t LCG_C = 1442695040888963407ull;

thread_local char g_err[512] = "";

td_status set_err(td_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

#define CUDA_TRY(expr)                                                          \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess)                                                      \
      return set_err(TD_E_CUDA, "%s failed: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const volatile uint32_t* p) { return *p; }
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
// release-only fences (no L1 invalidation): order the token stores before the
// counter increments that publish them
__device__ __forceinline__ void fence_rel_gpu() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_rel_sys() { asm volatile("fence.release.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_gpu() { asm volatile("fence.acquire.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_sys() { asm volatile("fence.acquire.sys;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_relaxed_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ uint64_t warp_xor_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
// One node's slot in its worker's program (Alg. 1 (V_w, E_w) flattened):
// everything the owner warp needs, contiguous in worker order so that a
// 1-D TMA bulk copy stages the next CHUNK descriptors into shared memory
// while the current ones execute.  Up to 3 predecessor and 3 successor
// intervals are inline; more spill to a per-graph interval pool
// (npiv/nsiv == TD_OVF, piv[0] = (pool offset, count)).
// Multi-GPU: successor intervals never straddle shards and carry the owning
// shard in bits 28..30 of .x (graphs are limited to 2^28 nodes when sharded).
struct __align__(16) Desc {
  int32_t v;
  uint32_t indeg;
  uint32_t arg;
  uint8_t kind, npiv, nsiv, rmask;
  int2 piv[3];
  int2 siv[3];
};
static_assert(sizeof(Desc) == 64, "descriptor must be 64 bytes");
constexpr uint8_t TD_OVF = 0xFF;
constexpr int RANK_SHIFT = 28;
constexpr int32_t ID_MASK = (1 << RANK_SHIFT) - 1;

constexpr int WARPS_PER_CTA = 4;   // 128 threads
constexpr int CHUNK = 16;          // descriptors per stage (1 KiB)
constexpr int STAGES = 2;

struct Params {
  const Desc* desc;          // [positions] worker-major programs
  const int64_t* work_ptr;   // [n_workers+1]
  const int2* pred_pool;     // overflow intervals
  const int2* succ_pool;
  const int32_t* worker_of;  // stats only
  int32_t n_workers;
  const int32_t* col;
  unsigned long long* colsum;
  uint32_t* ctr;
  unsigned long long* token;
  uint32_t* tally;
  unsigned long long* stats;          // [0]=executed [1]=cross [2]=local [3]=init [4]=cross_rank
  const volatile uint32_t* ext_pre;   // host-mapped
  uint32_t* ext_post;                 // host-mapped
  volatile uint32_t* abort_flag;      // host-mapped: host asks the kernel to stop
  uint32_t* poison;                   // device: set when a worker gave up
  uint64_t seed;
  uint32_t epoch;     // counter epoch (targets are indeg*(epoch+1))
  uint32_t exec_no;   // monotonically increasing execution number (flags)
  uint32_t flags;
  uint64_t spin_limit;
  // sharding
  int32_t my_rank, n_ranks;
  uint32_t* started;                  // [TD_MAX_RANKS] local: exec_no once peer r started
  unsigned long long* peer_token[TD_MAX_RANKS];
  uint32_t* peer_ctr[TD_MAX_RANKS];
  uint32_t* peer_started[TD_MAX_RANKS];
};

// --- shared-memory staging (mbarrier + cp.async.bulk, i.e. 1-D TMA) ---------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

// --- input gather -------------------------------------------------------------
// position j of a row of up to 3 inline intervals -> node id
__device__ __forceinline__ int inline_id(const int2* iv, int n, int j) {
  const int l0 = iv[0].y - iv[0].x + 1;
  if (j < l0 || n == 1) return iv[0].x + j;
  j -= l0;
  const int l1 = iv[1].y - iv[1].x + 1;
  if (j < l1 || n == 2) return iv[1].x + j;
  return iv[2].x + (j - l1);
}

__device__ __forceinline__ uint64_t fold_range(const unsigned long long* tok, int lo, int len, uint32_t base, int lane) {
  uint64_t acc = 0;
  int o = lane;
  for (; o + 96 < len; o += 128) {  // 4 loads in flight per lane
    const uint64_t t0 = __ldcg(&tok[lo + o]);
    const uint64_t t1 = __ldcg(&tok[lo + o + 32]);
    const uint64_t t2 = __ldcg(&tok[lo + o + 64]);
    const uint64_t t3 = __ldcg(&tok[lo + o + 96]);
    acc += mix64(t0 + (uint64_t)(base + o + 1) * G1) + mix64(t1 + (uint64_t)(base + o + 33) * G1) +
           mix64(t2 + (uint64_t)(base + o + 65) * G1) + mix64(t3 + (uint64_t)(base + o + 97) * G1);
  }
  for (; o < len; o += 32) acc += mix64(__ldcg(&tok[lo + o]) + (uint64_t)(base + o + 1) * G1);
  return acc;
}

constexpr int SMALL_DEG = 6;

// Small inline rows (the common Task Bench case, d_in <= 6): every lane folds
// all inputs redundantly -- the loads are broadcast and issued back to back,
// and no warp reduction sits on the critical path.
__device__ __forceinline__ uint64_t gather_small(const Params& P, const Desc& d) {
  const int n = (int)d.indeg;
  const int2 a = d.piv[0], b = d.piv[1], c = d.piv[2];
  const int l0 = a.y - a.x + 1, l1 = d.npiv > 1 ? b.y - b.x + 1 : 0;
  uint64_t t[SMALL_DEG];
#pragma unroll
  for (int j = 0; j < SMALL_DEG; ++j) {
    if (j < n) {
      const int id = j < l0 ? a.x + j : (j < l0 + l1 ? b.x + (j - l0) : c.x + (j - l0 - l1));
      t[j] = __ldcg(&P.token[id]);
    }
  }
  uint64_t acc = 0;
#pragma unroll
  for (int j = 0; j < SMALL_DEG; ++j)
    if (j < n) acc += mix64(t[j] + (uint64_t)(j + 1) * G1);
  return acc;
}

__device__ __forceinline__ uint64_t gather_inputs(const Params& P, const Desc& d, int lane) {
  uint64_t acc = 0;
  if (d.npiv == 0) return 0;
  if (d.npiv != TD_OVF && d.indeg <= SMALL_DEG) return gather_small(P, d);
  if (d.npiv != TD_OVF) {
    const int total = (int)d.indeg - 0;  // inline rows: indeg == total members
    if (d.npiv == 1) {
      acc = fold_range(P.token, d.piv[0].x, total, 0, lane);
    } else {
      for (int j = lane; j < total; j += 32)
        acc += mix64(__ldcg(&P.token[inline_id(d.piv, d.npiv, j)]) + (uint64_t)(j + 1) * G1);
    }
  } else {
    const int2* pool = P.pred_pool + d.piv[0].x;
    const int cnt = d.piv[0].y;
    uint32_t base = 0;
    for (int k = 0; k < cnt; ++k) {
      const int2 iv = pool[k];
      const int len = iv.y - iv.x + 1;
      acc += fold_range(P.token, iv.x, len, base, lane);
      base += len;
    }
  }
  return warp_sum_u64(acc);
}

__device__ __forceinline__ uint64_t run_body(int kind, uint32_t arg, uint64_t h, int lane) {
  if (kind == TD_BODY_COMPUTE) {
    uint64_t x0 = mix64(h ^ ((uint64_t)(lane + 1) * G2));
    uint64_t x1 = mix64(h ^ ((uint64_t)(lane + 33) * G2));
    for (uint32_t i = 0; i < arg; ++i) {
      x0 = LCG_A * x0 + LCG_C;
      x1 = LCG_A * x1 + LCG_C;
    }
    return warp_xor_u64(x0 ^ x1);
  }
  if (kind == TD_BODY_BUSY_WAIT) {
    const uint64_t t0 = globaltimer();
    while (globaltimer() - t0 < (uint64_t)arg) {
    }
  }
  return 0;
}

// --- successor signalling: one counter increment per edge -----
template <bool MULTI>
__device__ __forceinline__ void signal_range(const Params& P, int2 iv, int w, int lane, bool stats,
                                             unsigned long long& n_cross, unsigned long long& n_local,
                                             unsigned long long& n_xrank) {
  int lo = iv.x, hi = iv.y;
  int r = 0;
  if (MULTI) {
    r = (lo >> RANK_SHIFT) & 7;
    lo &= ID_MASK;
  }
  const int len = hi - lo + 1;
  uint32_t* ctr = (MULTI && r != P.my_rank) ? P.peer_ctr[r] : P.ctr;
  for (int o = lane; o < len; o += 32) {
    if (MULTI) red_add_sys(&ctr[lo + o], 1u);
    else red_add_gpu(&ctr[lo + o], 1u);
    if (stats) {
      if (__ldg(&P.worker_of[lo + o]) != w) ++n_cross;
      else ++n_local;
      if (MULTI && r != P.my_rank) ++n_xrank;
    }
  }
}

template <bool MULTI>
__device__ __forceinline__ void signal_succs(const Params& P, const Desc& d, int w, int lane,
                                             unsigned long long& n_cross, unsigned long long& n_local,
                                             unsigned long long& n_xrank) {
  const bool stats = P.flags & TD_F_STATS;
  if (d.nsiv != TD_OVF) {
    // flattened: lane l signals successor position l (one RED per lane)
    const int2 a = d.siv[0], b = d.siv[1], c = d.siv[2];
    const int ns = d.nsiv;
    const int lo0 = MULTI ? (a.x & ID_MASK) : a.x, lo1 = MULTI ? (b.x & ID_MASK) : b.x,
              lo2 = MULTI ? (c.x & ID_MASK) : c.x;
    const int l0 = ns > 0 ? a.y - lo0 + 1 : 0, l1 = ns > 1 ? b.y - lo1 + 1 : 0, l2 = ns > 2 ? c.y - lo2 + 1 : 0;
    const int total = l0 + l1 + l2;
    if (total <= 32) {
      if (lane < total) {
        int s, rx;
        if (lane < l0) { s = lo0 + lane; rx = a.x; }
        else if (lane < l0 + l1) { s = lo1 + (lane - l0); rx = b.x; }
        else { s = lo2 + (lane - l0 - l1); rx = c.x; }
        if (MULTI) {
          const int r = (rx >> RANK_SHIFT) & 7;
          red_add_sys(&((r != P.my_rank) ? P.peer_ctr[r] : P.ctr)[s], 1u);
          if (stats && r != P.my_rank) ++n_xrank;
        } else {
          red_add_gpu(&P.ctr[s], 1u);
        }
        if (stats) {
          if (__ldg(&P.worker_of[s]) != w) ++n_cross;
          else ++n_local;
        }
      }
      return;
    }
    for (int k = 0; k < d.nsiv; ++k) signal_range<MULTI>(P, d.siv[k], w, lane, stats, n_cross, n_local, n_xrank);
  } else {
    const int2* pool = P.succ_pool + d.siv[0].x;
    const int cnt = d.siv[0].y;
    for (int k = 0; k < cnt; ++k) signal_range<MULTI>(P, pool[k], w, lane, stats, n_cross, n_local, n_xrank);
  }
}

template <bool MULTI>
__device__ bool wait_counter(const Params& P, int v, uint32_t need) {
  const uint32_t target = need * (P.epoch + 1u);
  uint64_t spins = 0;
  for (;;) {
    // relaxed polling, one acquire fence once the target is observed
    // (acquire pattern: strong read + fence.acquire; no L1 invalidation per poll)
    const uint32_t c = MULTI ? ld_relaxed_sys(&P.ctr[v]) : ld_relaxed_gpu(&P.ctr[v]);
    if ((int32_t)(c - target) >= 0) {
      if (MULTI) fence_acq_sys();
      else fence_acq_gpu();
      return true;
    }
    if ((++spins & 4095u) == 0) {
      if (ld_relaxed_gpu(P.poison) || *P.abort_flag) return false;
      if (P.spin_limit && spins > P.spin_limit) {
        atomicExch(P.poison, 1u);
        return false;
      }
    }
  }
}

__device__ bool wait_peers_started(const Params& P) {
  uint64_t spins = 0;
  for (int r = 0; r < P.n_ranks; ++r) {
    if (r == P.my_rank) continue;
    while ((int32_t)(ld_acquire_sys(&P.started[r]) - P.exec_no) < 0) {
      if ((++spins & 4095u) == 0 && (ld_relaxed_gpu(P.poison) || *P.abort_flag)) return false;
    }
  }
  return true;
}

// Execute one node on its owner warp.  Returns false if the execution was
// aborted/poisoned.
template <bool MULTI>
__device__ __forceinline__ bool execute_node(const Params& P, const Desc& d, int w, int lane, bool& peers_ok,
                                             unsigned long long& n_cross, unsigned long long& n_local,
                                             unsigned long long& n_xrank) {
  const int v = d.v;
  const uint64_t h0 = mix64(P.seed ^ mix64((uint64_t)v + G1));
  if (d.indeg && !wait_counter<MULTI>(P, v, d.indeg)) return false;
  if (d.kind == TD_BODY_EXT_PRE) {
    uint64_t spins = 0;
    while ((int32_t)(ld_volatile_u32(&P.ext_pre[d.arg]) - P.exec_no) < 0) {
      if ((++spins & 4095u) == 0 && (ld_relaxed_gpu(P.poison) || *P.abort_flag)) return false;
    }
    fence_sys();
  }
  const uint64_t acc = gather_inputs(P, d, lane);
  const uint64_t h = mix64(h0 ^ acc);
  const uint64_t tok = h ^ run_body(d.kind, d.arg, h, lane);

  if (lane == 0) P.token[v] = tok;
  if (MULTI && d.rmask) {
    if (!peers_ok) {
      if (!wait_peers_started(P)) return false;
      peers_ok = true;
    }
    if (lane < P.n_ranks && ((d.rmask >> lane) & 1u)) P.peer_token[lane][v] = tok;
  }
  __syncwarp();
  if (MULTI) fence_rel_sys();
  else fence_rel_gpu();
  if (d.kind == TD_BODY_EXT_POST && lane == 0) st_release_sys(&P.ext_post[d.arg], P.exec_no);
  signal_succs<MULTI>(P, d, w, lane, n_cross, n_local, n_xrank);
  // accounting off the critical path (after the successors were signalled)
  if (lane == 0) {
    if (P.flags & TD_F_CHECKSUM) {
      const int c = __ldg(&P.col[v]);
      if (c >= 0) atomicXor(&P.colsum[c], (unsigned long long)tok);
    }
    if (P.flags & TD_F_TALLY) atomicAdd(&P.tally[v], 1u);
  }
  return true;
}

template <bool MULTI>
__global__ void __launch_bounds__(128, 8) td_exec_kernel(const Params P) {
  __shared__ __align__(128) Desc ring[WARPS_PER_CTA][STAGES][CHUNK];
  __shared__ __align__(8) uint64_t bar[WARPS_PER_CTA][STAGES];
  const int lane = threadIdx.x & 31;
  const int wc = threadIdx.x >> 5;
  const int w = (int)(blockIdx.x * WARPS_PER_CTA + wc);

  if (MULTI && blockIdx.x == 0 && threadIdx.x < P.n_ranks && (int)threadIdx.x != P.my_rank) {
    // publish "this shard started execution exec_no" to every peer (our
    // counter reset, if any, is stream-ordered before this kernel)
    fence_sys();
    st_release_sys(&P.peer_started[threadIdx.x][P.my_rank], P.exec_no);
  }
  if (w >= P.n_workers) return;
  const int64_t beg = P.work_ptr[w];
  const int npos = (int)(P.work_ptr[w + 1] - beg);
  const int nchunks = (npos + CHUNK - 1) / CHUNK;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[wc][s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  if (lane == 0)
    for (int c = 0; c < STAGES && c < nchunks; ++c) {
      const int cnt = min(CHUNK, npos - c * CHUNK);
      bulk_load(&ring[wc][c][0], P.desc + beg + (int64_t)c * CHUNK, cnt * (uint32_t)sizeof(Desc), &bar[wc][c]);
    }

  unsigned long long n_exec = 0, n_cross = 0, n_local = 0, n_xrank = 0;
  bool peers_ok = !MULTI;
  int issued = min(STAGES, nchunks);
  int c = 0;
  for (; c < nchunks; ++c) {
    const int s = c % STAGES;
    mbar_wait(&bar[wc][s], (uint32_t)((c / STAGES) & 1));
    const int cnt = min(CHUNK, npos - c * CHUNK);
    bool ok = true;
    for (int j = 0; j < cnt; ++j) {
      const Desc& d = ring[wc][s][j];
      if (!execute_node<MULTI>(P, d, w, lane, peers_ok, n_cross, n_local, n_xrank)) { ok = false; break; }
      ++n_exec;
    }
    __syncwarp();
    if (!ok) break;
    if (lane == 0 && issued < nchunks) {
      const int cc = min(CHUNK, npos - issued * CHUNK);
      bulk_load(&ring[wc][s][0], P.desc + beg + (int64_t)issued * CHUNK, cc * (uint32_t)sizeof(Desc), &bar[wc][s]);
    }
    issued = min(issued + 1, nchunks);
  }
  // aborted: drain bulk copies still in flight into this warp's ring
  for (int k = c + 1; k < issued; ++k) mbar_wait(&bar[wc][k % STAGES], (uint32_t)((k / STAGES) & 1));
  if (P.flags & TD_F_STATS) {
    n_cross = warp_sum_u64(n_cross);
    n_local = warp_sum_u64(n_local);
    n_xrank = warp_sum_u64(n_xrank);
    if (lane == 0) {
      atomicAdd(&P.stats[0], n_exec);
      atomicAdd(&P.stats[1], n_cross);
      atomicAdd(&P.stats[2], n_local);
      atomicAdd(&P.stats[3], (unsigned long long)(npos > 0));
      atomicAdd(&P.stats[4], n_xrank);
    }
  }
}

template <typename T>
cudaError_t upload(T** dst, const T* src, size_t count) {
  *dst = nullptr;
  if (count == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc((void**)dst, count * sizeof(T));
  if (e != cudaSuccess) return e;
  return src ? cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice) : cudaMemset(*dst, 0, count * sizeof(T));
}

}  // namespace

struct td_graph {
  int device;
  int64_t n;
  int32_t n_workers, n_cols, n_ranks, my_rank, n_ext_pre, n_ext_post;
  uint32_t max_indeg;
  int64_t n_positions, n_pred_pool, n_succ_pool;
  // device arrays
  Desc* desc;
  int64_t* work_ptr;
  int2 *pred_pool, *succ_pool;
  int32_t *worker_of, *col;
  unsigned long long *colsum, *token, *stats;
  uint32_t *ctr, *tally, *poison, *started;
  // host-mapped flags
  uint32_t *h_ext_pre, *h_ext_post, *h_abort;
  uint32_t *d_ext_pre, *d_ext_post, *d_abort;
  // peers
  unsigned long long* peer_token[TD_MAX_RANKS];
  uint32_t* peer_ctr[TD_MAX_RANKS];
  uint32_t* peer_started[TD_MAX_RANKS];
  bool peer_opened[TD_MAX_RANKS];
  // execution state
  uint32_t epoch;          // counter epoch of the next launch (reset with the counters)
  uint32_t launches;       // executions launched (never reset; flag values)
  uint64_t completed;
  bool outstanding;
  uint32_t last_flags;
  int32_t blocks, tpb;
  cudaEvent_t ev_start, ev_stop;
  void* last_stream;
};

extern "C" {

const char* td_last_error(void) { return g_err; }

static int occupancy_blocks(uint32_t tpb, int* per_sm) {
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, td_exec_kernel<false>, (int)tpb, 0);
}

td_status td_device_info_get(int32_t device, uint32_t tpb, td_device_info* out) {
  if (!out) return set_err(TD_E_CONTRACT, "null out");
  if (tpb == 0) tpb = 32 * WARPS_PER_CTA;
  int count = 0;
  CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return set_err(TD_E_RESOURCE, "unknown device %d", device);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  int per_sm = 0;
  CUDA_TRY((cudaError_t)occupancy_blocks(tpb, &per_sm));
  memset(out, 0, sizeof *out);
  out->sm_count = prop.multiProcessorCount;
  out->l2_bytes = prop.l2CacheSize;
  out->max_workers = per_sm * prop.multiProcessorCount * (int)(tpb / 32);
  out->cc_major = prop.major;
  out->cc_minor = prop.minor;
  strncpy(out->name, prop.name, sizeof out->name - 1);
  return TD_OK;
}

td_status td_graph_destroy(td_graph* g) {
  if (!g) return TD_OK;
  cudaSetDevice(g->device);
  if (g->outstanding) cudaEventSynchronize(g->ev_stop);
  void* bufs[] = {g->desc, g->work_ptr, g->pred_pool, g->succ_pool, g->worker_of, g->col,
                  g->colsum, g->token, g->stats, g->ctr, g->tally, g->poison, g->started};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (int r = 0; r < TD_MAX_RANKS; ++r) {
    if (g->peer_opened[r]) {
      cudaIpcCloseMemHandle(g->peer_token[r]);
      cudaIpcCloseMemHandle(g->peer_ctr[r]);
      cudaIpcCloseMemHandle(g->peer_started[r]);
    }
  }
  if (g->h_ext_pre) cudaFreeHost(g->h_ext_pre);
  if (g->h_ext_post) cudaFreeHost(g->h_ext_post);
  if (g->h_abort) cudaFreeHost(g->h_abort);
  if (g->ev_start) cudaEventDestroy(g->ev_start);
  if (g->ev_stop) cudaEventDestroy(g->ev_stop);
  delete g;
  return TD_OK;
}

namespace {
// Intervals of a neighbour row, split at shard boundaries when sharded, with
// the owning shard encoded in bits 28..30 of lo (RANK_SHIFT).
void row_intervals(const int64_t* ptr, const int32_t* iv, int64_t v, const uint8_t* node_rank, bool tag,
                   std::vector<int2>& out) {
  out.clear();
  for (int64_t k = ptr[v]; k < ptr[v + 1]; ++k) {
    int32_t lo = iv[2 * k], hi = iv[2 * k + 1];
    if (!tag) {
      out.push_back(make_int2(lo, hi));
      continue;
    }
    int32_t a = lo;
    while (a <= hi) {
      const uint8_t r = node_rank[a];
      int32_t b = a;
      while (b < hi && node_rank[b + 1] == r) ++b;
      out.push_back(make_int2(a | ((int32_t)r << RANK_SHIFT), b));
      a = b + 1;
    }
  }
}
}  // namespace

td_status td_graph_upload(const td_csr* c, int32_t device, td_graph** out) {
  if (!c || !out) return set_err(TD_E_CONTRACT, "null argument");
  *out = nullptr;
  const int64_t n = c->n_nodes;
  const int nr = c->n_ranks < 1 ? 1 : c->n_ranks;
  if (n < 0 || n >= (int64_t)INT32_MAX) return set_err(TD_E_GRAPH, "node count %lld out of range", (long long)n);
  if (nr > 1 && n >= (1ll << RANK_SHIFT)) return set_err(TD_E_GRAPH, "sharded graphs are limited to 2^28 nodes");
  if (c->n_workers < 1 && n > 0 && nr == 1) return set_err(TD_E_COMPILE, "graph has nodes but no workers");
  if (nr > TD_MAX_RANKS) return set_err(TD_E_RESOURCE, "at most %d shards", TD_MAX_RANKS);
  if (c->my_rank < 0 || c->my_rank >= nr) return set_err(TD_E_RESOURCE, "bad shard rank %d", c->my_rank);
  if (nr > 1 && !c->node_rank) return set_err(TD_E_CONTRACT, "sharded graph needs node_rank");
  int count = 0;
  CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return set_err(TD_E_RESOURCE, "unknown device %d", device);
  CUDA_TRY(cudaSetDevice(device));

  // ---- host-side validation ------------------------------------------------
  uint32_t max_indeg = 1;
  for (int64_t v = 0; v < n; ++v) {
    int64_t d = 0;
    int32_t prev_hi = -2;
    for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k) {
      const int32_t lo = c->pred_iv[2 * k], hi = c->pred_iv[2 * k + 1];
      if (lo < 0 || hi >= n || hi < lo || lo <= prev_hi)
        return set_err(TD_E_GRAPH, "dangling/unsorted predecessor interval of node %lld", (long long)v);
      prev_hi = hi;
      d += hi - lo + 1;
    }
    if (d >= (1ll << 30)) return set_err(TD_E_GRAPH, "in-degree too large");
    if ((uint32_t)d > max_indeg) max_indeg = (uint32_t)d;
    if (c->kind[v] > TD_BODY_EXT_POST)
      return set_err(TD_E_COMPILE, "node %lld has unknown body kind %d", (long long)v, c->kind[v]);
    if (c->kind[v] == TD_BODY_EXT_PRE && (int32_t)c->arg[v] >= c->n_ext_pre)
      return set_err(TD_E_GRAPH, "ext precondition index out of range");
    if (c->kind[v] == TD_BODY_EXT_POST && (int32_t)c->arg[v] >= c->n_ext_post)
      return set_err(TD_E_GRAPH, "ext postcondition index out of range");
    for (int64_t k = c->succ_ptr[v]; k < c->succ_ptr[v + 1]; ++k) {
      const int32_t lo = c->succ_iv[2 * k], hi = c->succ_iv[2 * k + 1];
      if (lo < 0 || hi >= n || hi < lo)
        return set_err(TD_E_GRAPH, "dangling successor interval of node %lld", (long long)v);
    }
  }
  std::vector<int32_t> worker_of((size_t)(n > 0 ? n : 1), -1);
  const int64_t npos = c->n_workers > 0 ? c->work_ptr[c->n_workers] : 0;
  for (int32_t w = 0; w < c->n_workers; ++w) {
    for (int64_t i = c->work_ptr[w]; i < c->work_ptr[w + 1]; ++i) {
      const int32_t v = c->work[i];
      if (v < 0 || v >= n) return set_err(TD_E_COMPILE, "worker list references unknown node");
      if (worker_of[v] != -1) return set_err(TD_E_COMPILE, "node %d assigned to two workers", v);
      if (nr > 1 && c->node_rank[v] != c->my_rank) return set_err(TD_E_COMPILE, "worker list holds a node of another shard");
      worker_of[v] = w;
    }
  }
  if (nr == 1 && npos != n) return set_err(TD_E_COMPILE, "worker lists do not cover the graph");

  // ---- worker programs (descriptors) ----------------------------------------
  std::vector<Desc> desc((size_t)(npos > 0 ? npos : 1));
  std::vector<int2> ppool, spool, tmp;
  for (int64_t i = 0; i < npos; ++i) {
    const int32_t v = c->work[i];
    Desc& d = desc[i];
    memset(&d, 0, sizeof d);
    d.v = v;
    d.kind = c->kind[v];
    d.arg = c->arg[v];
    row_intervals(c->pred_ptr, c->pred_iv, v, nullptr, false, tmp);
    uint32_t indeg = 0;
    for (auto& iv : tmp) indeg += (uint32_t)(iv.y - iv.x + 1);
    d.indeg = indeg;
    if (tmp.size() <= 3) {
      d.npiv = (uint8_t)tmp.size();
      for (size_t k = 0; k < tmp.size(); ++k) d.piv[k] = tmp[k];
    } else {
      d.npiv = TD_OVF;
      d.piv[0] = make_int2((int32_t)ppool.size(), (int32_t)tmp.size());
      ppool.insert(ppool.end(), tmp.begin(), tmp.end());
    }
    row_intervals(c->succ_ptr, c->succ_iv, v, c->node_rank, nr > 1, tmp);
    uint32_t rmask = 0;
    if (nr > 1)
      for (auto& iv : tmp) {
        const int r = (iv.x >> RANK_SHIFT) & 7;
        if (r != c->my_rank) rmask |= 1u << r;
      }
    d.rmask = (uint8_t)rmask;
    if (tmp.size() <= 3) {
      d.nsiv = (uint8_t)tmp.size();
      for (size_t k = 0; k < tmp.size(); ++k) d.siv[k] = tmp[k];
    } else {
      d.nsiv = TD_OVF;
      d.siv[0] = make_int2((int32_t)spool.size(), (int32_t)tmp.size());
      spool.insert(spool.end(), tmp.begin(), tmp.end());
    }
  }

  td_graph* g = new td_graph();
  memset(g, 0, sizeof *g);
  g->device = device;
  g->n = n;
  g->n_workers = c->n_workers;
  g->n_cols = c->n_cols;
  g->n_ranks = nr;
  g->my_rank = c->my_rank;
  g->n_ext_pre = c->n_ext_pre;
  g->n_ext_post = c->n_ext_post;
  g->max_indeg = max_indeg;
  g->n_positions = npos;
  g->n_pred_pool = (int64_t)ppool.size();
  g->n_succ_pool = (int64_t)spool.size();
  cudaError_t e = cudaSuccess;
#define UP(field, src, cnt) if (e == cudaSuccess) e = upload(&g->field, src, (size_t)(cnt))
  UP(desc, desc.data(), npos > 0 ? npos : 1);
  UP(work_ptr, c->work_ptr, c->n_workers + 1);
  UP(pred_pool, ppool.data(), ppool.size());
  UP(succ_pool, spool.data(), spool.size());
  UP(worker_of, worker_of.data(), n > 0 ? n : 1);
  UP(col, c->col, c->col ? n : 0);
  UP(colsum, (const unsigned long long*)nullptr, c->n_cols > 0 ? c->n_cols : 1);
  UP(token, (const unsigned long long*)nullptr, n > 0 ? n : 1);
  UP(ctr, (const uint32_t*)nullptr, n > 0 ? n : 1);
  UP(tally, (const uint32_t*)nullptr, n > 0 ? n : 1);
  UP(stats, (const unsigned long long*)nullptr, 8);
  UP(poison, (const uint32_t*)nullptr, 1);
  UP(started, (const uint32_t*)nullptr, TD_MAX_RANKS);
#undef UP
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&g->h_ext_pre, sizeof(uint32_t) * (g->n_ext_pre + 1), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&g->h_ext_post, sizeof(uint32_t) * (g->n_ext_post + 1), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&g->h_abort, sizeof(uint32_t), cudaHostAllocMapped);
  if (e == cudaSuccess) {
    memset(g->h_ext_pre, 0, sizeof(uint32_t) * (g->n_ext_pre + 1));
    memset(g->h_ext_post, 0, sizeof(uint32_t) * (g->n_ext_post + 1));
    *g->h_abort = 0;
    e = cudaHostGetDevicePointer((void**)&g->d_ext_pre, g->h_ext_pre, 0);
  }
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&g->d_ext_post, g->h_ext_post, 0);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer((void**)&g->d_abort, g->h_abort, 0);
  if (e == cudaSuccess) e = cudaEventCreate(&g->ev_start);
  if (e == cudaSuccess) e = cudaEventCreate(&g->ev_stop);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    td_status s = set_err(e == cudaErrorMemoryAllocation ? TD_E_ALLOCATION : TD_E_CUDA,
                          "upload failed: %s", cudaGetErrorString(e));
    td_graph_destroy(g);
    return s;
  }
  *out = g;
  return TD_OK;
}

td_status td_graph_launch(td_graph* g, const td_launch_params* p, void* stream) {
  if (!g || !p) return set_err(TD_E_CONTRACT, "null argument");
  CUDA_TRY(cudaSetDevice(g->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (g->outstanding && !(p->flags & TD_F_QUEUE)) {
    cudaError_t q = cudaEventQuery(g->ev_stop);
    if (q == cudaErrorNotReady)
      return set_err(TD_E_EXEC_STATE, "an execution of this graph is still outstanding");
    if (q != cudaSuccess) return set_err(TD_E_CUDA, "event query: %s", cudaGetErrorString(q));
  }
  const uint32_t tpb = 32 * WARPS_PER_CTA;
  if (p->threads_per_block && p->threads_per_block != tpb)
    return set_err(TD_E_RESOURCE, "threads_per_block is fixed at %u", tpb);
  const bool multi = g->n_ranks > 1;
  int per_sm = 0, sms = 0;
  if (multi) CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, td_exec_kernel<true>, (int)tpb, 0));
  else CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, td_exec_kernel<false>, (int)tpb, 0));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
  int64_t blocks = (g->n_workers + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
  if (multi && blocks == 0) blocks = 1;  // the start handshake still runs
  if (blocks > (int64_t)per_sm * sms)
    return set_err(TD_E_RESOURCE, "%d workers exceed the %lld co-resident warps of this GPU",
                   g->n_workers, (long long)per_sm * sms * WARPS_PER_CTA);
  if (multi)
    for (int r = 0; r < g->n_ranks; ++r)
      if (r != g->my_rank && !g->peer_opened[r]) return set_err(TD_E_RESOURCE, "peer shard %d not attached", r);
  // epoch-scaled counter targets: reset counters before they could wrap
  if ((uint64_t)(g->epoch + 2) * g->max_indeg >= (1ull << 31)) {
    CUDA_TRY(cudaMemsetAsync(g->ctr, 0, sizeof(uint32_t) * (g->n > 0 ? g->n : 1), s));
    g->epoch = 0;
  }
  if (p->flags & TD_F_CHECKSUM)
    CUDA_TRY(cudaMemsetAsync(g->colsum, 0, sizeof(unsigned long long) * (g->n_cols > 0 ? g->n_cols : 1), s));
  if (p->flags & TD_F_STATS) CUDA_TRY(cudaMemsetAsync(g->stats, 0, sizeof(unsigned long long) * 8, s));
  if (p->flags & TD_F_TALLY) CUDA_TRY(cudaMemsetAsync(g->tally, 0, sizeof(uint32_t) * (g->n > 0 ? g->n : 1), s));
  CUDA_TRY(cudaMemsetAsync(g->poison, 0, sizeof(uint32_t), s));
  *g->h_abort = 0;
  for (int j = 0; j < g->n_ext_post; ++j) g->h_ext_post[j] = 0;

  Params P;
  memset(&P, 0, sizeof P);
  P.desc = g->desc;
  P.work_ptr = g->work_ptr;
  P.pred_pool = g->pred_pool;
  P.succ_pool = g->succ_pool;
  P.worker_of = g->worker_of;
  P.n_workers = g->n_workers;
  P.col = g->col;
  P.colsum = g->colsum;
  P.ctr = g->ctr;
  P.token = g->token;
  P.tally = g->tally;
  P.stats = g->stats;
  P.ext_pre = g->d_ext_pre;
  P.ext_post = g->d_ext_post;
  P.abort_flag = g->d_abort;
  P.poison = g->poison;
  P.seed = p->seed;
  P.epoch = g->epoch;
  P.exec_no = g->launches + 1u;
  P.flags = p->flags;
  P.spin_limit = p->spin_limit;
  P.my_rank = g->my_rank;
  P.n_ranks = g->n_ranks;
  P.started = g->started;
  for (int r = 0; r < TD_MAX_RANKS; ++r) {
    P.peer_token[r] = g->peer_token[r];
    P.peer_ctr[r] = g->peer_ctr[r];
    P.peer_started[r] = g->peer_started[r];
  }

  CUDA_TRY(cudaEventRecord(g->ev_start, s));
  if (blocks > 0) {
    void* args[] = {&P};
    const void* fn = multi ? (const void*)td_exec_kernel<true> : (const void*)td_exec_kernel<false>;
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3((unsigned)blocks), dim3(tpb), args, 0, s));
  }
  CUDA_TRY(cudaEventRecord(g->ev_stop, s));
  g->outstanding = true;
  g->last_flags = p->flags;
  g->blocks = (int32_t)blocks;
  g->tpb = (int32_t)tpb;
  g->last_stream = stream;
  g->epoch += 1;
  g->launches += 1;
  return TD_OK;
}

static td_status finish_wait(td_graph* g) {
  g->outstanding = false;
  g->completed += 1;
  uint32_t poison = 0;
  CUDA_TRY(cudaMemcpy(&poison, g->poison, sizeof poison, cudaMemcpyDeviceToHost));
  if (poison) return set_err(TD_E_POISONED, "execution poisoned (spin limit exceeded)");
  return TD_OK;
}

td_status td_graph_query(td_graph* g, int32_t* done) {
  if (!g || !done) return set_err(TD_E_CONTRACT, "null argument");
  CUDA_TRY(cudaSetDevice(g->device));
  if (!g->outstanding) { *done = 1; return TD_OK; }
  cudaError_t q = cudaEventQuery(g->ev_stop);
  if (q == cudaErrorNotReady) { *done = 0; return TD_OK; }
  if (q != cudaSuccess) return set_err(TD_E_CUDA, "event query: %s", cudaGetErrorString(q));
  *done = 1;
  return TD_OK;
}

td_status td_graph_wait(td_graph* g, double timeout_s) {
  if (!g) return set_err(TD_E_CONTRACT, "null argument");
  CUDA_TRY(cudaSetDevice(g->device));
  if (!g->outstanding) return TD_OK;
  if (timeout_s < 0) {
    CUDA_TRY(cudaEventSynchronize(g->ev_stop));
    return finish_wait(g);
  }
  struct timespec t0, t1;
  clock_gettime(CLOCK_MONOTONIC, &t0);
  for (;;) {
    cudaError_t q = cudaEventQuery(g->ev_stop);
    if (q == cudaSuccess) return finish_wait(g);
    if (q != cudaErrorNotReady) return set_err(TD_E_CUDA, "event query: %s", cudaGetErrorString(q));
    clock_gettime(CLOCK_MONOTONIC, &t1);
    const double el = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
    if (el > timeout_s) {
      // ask the kernel to stop (workers poll the mapped abort flag), then drain
      *(volatile uint32_t*)g->h_abort = 1;
      cudaEventSynchronize(g->ev_stop);
      g->outstanding = false;
      return set_err(TD_E_WAIT_TIMEOUT, "execution did not finish within %.3f s", timeout_s);
    }
    struct timespec ts = {0, 20000};
    nanosleep(&ts, nullptr);
  }
}

td_status td_graph_trigger_pre(td_graph* g, int32_t index) {
  if (!g) return set_err(TD_E_CONTRACT, "null argument");
  if (index < 0 || index >= g->n_ext_pre) return set_err(TD_E_RESOURCE, "precondition %d out of range", index);
  // the current (or next) execution uses epoch value g->epoch-1 if launched
  const uint32_t e = g->outstanding ? g->launches : g->launches + 1;
  __atomic_store_n(&g->h_ext_pre[index], e, __ATOMIC_RELEASE);
  return TD_OK;
}

td_status td_graph_post_fired(td_graph* g, int32_t index, int32_t* fired) {
  if (!g || !fired) return set_err(TD_E_CONTRACT, "null argument");
  if (index < 0 || index >= g->n_ext_post) return set_err(TD_E_RESOURCE, "postcondition %d out of range", index);
  *fired = __atomic_load_n(&g->h_ext_post[index], __ATOMIC_ACQUIRE) == g->launches;
  return TD_OK;
}

td_status td_graph_tokens(td_graph* g, uint64_t* host, int64_t n) {
  if (!g || (!host && n)) return set_err(TD_E_CONTRACT, "null argument");
  if (n != g->n) return set_err(TD_E_CONTRACT, "token buffer has %lld entries, graph %lld", (long long)n, (long long)g->n);
  CUDA_TRY(cudaSetDevice(g->device));
  if (n) CUDA_TRY(cudaMemcpy(host, g->token, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return TD_OK;
}

td_status td_graph_checksums(td_graph* g, uint64_t* host, int32_t n_cols) {
  if (!g || (!host && n_cols)) return set_err(TD_E_CONTRACT, "null argument");
  if (n_cols != g->n_cols) return set_err(TD_E_CONTRACT, "column count mismatch");
  CUDA_TRY(cudaSetDevice(g->device));
  if (n_cols) CUDA_TRY(cudaMemcpy(host, g->colsum, sizeof(uint64_t) * n_cols, cudaMemcpyDeviceToHost));
  return TD_OK;
}

td_status td_graph_tally(td_graph* g, uint32_t* host, int64_t n) {
  if (!g || (!host && n)) return set_err(TD_E_CONTRACT, "null argument");
  if (n != g->n) return set_err(TD_E_CONTRACT, "tally buffer size mismatch");
  CUDA_TRY(cudaSetDevice(g->device));
  if (n) CUDA_TRY(cudaMemcpy(host, g->tally, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
  return TD_OK;
}

td_status td_graph_stats(td_graph* g, td_stats* out) {
  if (!g || !out) return set_err(TD_E_CONTRACT, "null argument");
  CUDA_TRY(cudaSetDevice(g->device));
  unsigned long long s[8];
  CUDA_TRY(cudaMemcpy(s, g->stats, sizeof s, cudaMemcpyDeviceToHost));
  uint32_t poison = 0;
  CUDA_TRY(cudaMemcpy(&poison, g->poison, sizeof poison, cudaMemcpyDeviceToHost));
  memset(out, 0, sizeof *out);
  out->executed = s[0];
  out->cross_worker_edges = s[1];
  out->local_decrements = s[2];
  out->init_messages = s[3];
  out->cross_rank_edges = s[4];
  out->epoch = g->completed;
  out->poisoned = (int32_t)poison;
  out->workers = g->n_workers;
  out->blocks = g->blocks;
  out->threads_per_block = g->tpb;
  return TD_OK;
}

td_status td_graph_last_ms(td_graph* g, float* ms) {
  if (!g || !ms) return set_err(TD_E_CONTRACT, "null argument");
  CUDA_TRY(cudaSetDevice(g->device));
  CUDA_TRY(cudaEventElapsedTime(ms, g->ev_start, g->ev_stop));
  return TD_OK;
}

td_status td_graph_ipc_export(td_graph* g, void* out, size_t cap, size_t* len) {
  if (!g || !out || !len) return set_err(TD_E_CONTRACT, "null argument");
  const size_t need = 3 * sizeof(cudaIpcMemHandle_t);
  *len = need;
  if (cap < need) return set_err(TD_E_CONTRACT, "handle buffer too small (%zu < %zu)", cap, need);
  CUDA_TRY(cudaSetDevice(g->device));
  cudaIpcMemHandle_t* h = (cudaIpcMemHandle_t*)out;
  CUDA_TRY(cudaIpcGetMemHandle(&h[0], g->token));
  CUDA_TRY(cudaIpcGetMemHandle(&h[1], g->ctr));
  CUDA_TRY(cudaIpcGetMemHandle(&h[2], g->started));
  return TD_OK;
}

td_status td_graph_ipc_attach(td_graph* g, int32_t rank, const void* handle, size_t len) {
  if (!g || !handle) return set_err(TD_E_CONTRACT, "null argument");
  if (rank < 0 || rank >= g->n_ranks || rank == g->my_rank) return set_err(TD_E_RESOURCE, "bad peer rank %d", rank);
  if (len < 3 * sizeof(cudaIpcMemHandle_t)) return set_err(TD_E_CONTRACT, "short handle");
  CUDA_TRY(cudaSetDevice(g->device));
  const cudaIpcMemHandle_t* h = (const cudaIpcMemHandle_t*)handle;
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h[0], cudaIpcMemLazyEnablePeerAccess));
  g->peer_token[rank] = (unsigned long long*)p;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h[1], cudaIpcMemLazyEnablePeerAccess));
  g->peer_ctr[rank] = (uint32_t*)p;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h[2], cudaIpcMemLazyEnablePeerAccess));
  g->peer_started[rank] = (uint32_t*)p;
  g->peer_opened[rank] = true;
  return TD_OK;
}


}  // extern "C"

// ---------------------------------------------------------------------------
// Per-task launch runtime (generic path; one warp-sized kernel per task)
// ---------------------------------------------------------------------------
namespace {
struct RtTask {
  uint64_t seed, key;
  int64_t slot;
  uint32_t arg;
  int32_t n_pred;
  uint32_t kind;
  int64_t pred[TD_RT_MAX_PREDS];
};

__global__ void __launch_bounds__(32) td_rt_task_kernel(const __grid_constant__ RtTask A, unsigned long long* tok) {
  const int lane = threadIdx.x;
  uint64_t acc = 0;
  for (int j = lane; j < A.n_pred; j += 32) acc += mix64(tok[A.pred[j]] + (uint64_t)(j + 1) * G1);
  acc = warp_sum_u64(acc);
  const uint64_t h = mix64(mix64(A.seed ^ mix64(A.key + G1)) ^ acc);
  const uint64_t t = h ^ run_body((int)A.kind, A.arg, h, lane);
  if (lane == 0) tok[A.slot] = t;
}
}  // namespace

struct td_rt {
  int device;
  int64_t capacity;
  unsigned long long* tok;
  cudaStream_t stream;
};

extern "C" {

td_status td_rt_create(int32_t device, int64_t capacity, td_rt** out) {
  if (!out || capacity < 1) return set_err(TD_E_CONTRACT, "bad argument");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  td_rt* rt = new td_rt();
  rt->device = device;
  rt->capacity = capacity;
  cudaError_t e = cudaMalloc(&rt->tok, sizeof(unsigned long long) * capacity);
  if (e == cudaSuccess) e = cudaMemset(rt->tok, 0, sizeof(unsigned long long) * capacity);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    if (rt->tok) cudaFree(rt->tok);
    delete rt;
    return set_err(e == cudaErrorMemoryAllocation ? TD_E_ALLOCATION : TD_E_CUDA, "td_rt_create: %s", cudaGetErrorString(e));
  }
  *out = rt;
  return TD_OK;
}

td_status td_rt_launch_task(td_rt* rt, int64_t slot, uint64_t key, uint8_t kind, uint32_t arg, uint64_t seed,
                            const int64_t* pred_slots, int32_t n_pred) {
  if (!rt || (n_pred && !pred_slots)) return set_err(TD_E_CONTRACT, "null argument");
  if (slot < 0 || slot >= rt->capacity) return set_err(TD_E_RESOURCE, "slot %lld out of range", (long long)slot);
  if (n_pred < 0 || n_pred > TD_RT_MAX_PREDS) return set_err(TD_E_RESOURCE, "at most %d predecessors per task", TD_RT_MAX_PREDS);
  if (kind > TD_BODY_BUSY_WAIT + 1) return set_err(TD_E_COMPILE, "body kind %d not supported by task launch", kind);
  RtTask A;
  A.seed = seed; A.key = key; A.slot = slot; A.arg = arg; A.n_pred = n_pred; A.kind = kind;
  for (int j = 0; j < n_pred; ++j) {
    if (pred_slots[j] < 0 || pred_slots[j] >= rt->capacity) return set_err(TD_E_RESOURCE, "predecessor slot out of range");
    A.pred[j] = pred_slots[j];
  }
  CUDA_TRY(cudaSetDevice(rt->device));
  td_rt_task_kernel<<<1, 32, 0, rt->stream>>>(A, rt->tok);
  CUDA_TRY(cudaGetLastError());
  return TD_OK;
}

td_status td_rt_sync(td_rt* rt) {
  if (!rt) return set_err(TD_E_CONTRACT, "null argument");
  CUDA_TRY(cudaSetDevice(rt->device));
  CUDA_TRY(cudaStreamSynchronize(rt->stream));
  return TD_OK;
}

td_status td_rt_tokens(td_rt* rt, int64_t first, int64_t n, uint64_t* host) {
  if (!rt || (n && !host)) return set_err(TD_E_CONTRACT, "null argument");
  if (first < 0 || n < 0 || first + n > rt->capacity) return set_err(TD_E_RESOURCE, "range out of bounds");
  CUDA_TRY(cudaSetDevice(rt->device));
  CUDA_TRY(cudaStreamSynchronize(rt->stream));
  if (n) CUDA_TRY(cudaMemcpy(host, rt->tok + first, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return TD_OK;
}

td_status td_rt_destroy(td_rt* rt) {
  if (!rt) return TD_OK;
  cudaSetDevice(rt->device);
  cudaStreamSynchronize(rt->stream);
  cudaStreamDestroy(rt->stream);
  cudaFree(rt->tok);
  delete rt;
  return TD_OK;
}

}  // extern "C"

