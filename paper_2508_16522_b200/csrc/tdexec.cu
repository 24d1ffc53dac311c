// tdexec.cu — B200 (sm_100a) persistent executor for traced task graphs.
//
// Replaces the reference's Alg. 1 interpreter (SPEC.md
// compiler 351-425): INIT / COMPLETED_EDGE / EXECUTE_OP messages between
// per-resource Worker actors become, inside ONE persistent kernel per GPU,
//   * a worker  = one resident warp owning a static, topologically ordered
//                 list of 64 B node descriptors (Alg. 1 V_w),
//                 streamed into shared memory by TMA bulk copies,
//   * a message = one 64-bit red.add of (1 << 48) + term(producer) into the
//                 consumer's mailbox word [count:16 | term sum:48], in L2 (or
//                 in a peer GPU's memory over NVLink for a cross-shard edge,
//                 SPEC.md:468): the input travels inside the message,
//   * dispatch  = the owner warp observing count == in-degree; it re-arms the
//                 word for the next replay after use.
// Same-worker edges go through a shared-memory ring; consumers
// with one shared large predecessor list share mailbox replicas.
// See DESIGN.md for the memory layout and the roofline of each phase.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <stdio.h>
#include <stdarg.h>
#include <time.h>

#include <algorithm>
#include <chrono>
#include <unordered_map>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/tdexec.h"

#define TD_MAX_RANKS 8
#define TD_MAX_SMID 512

namespace {

constexpr uint64_t G1 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t G2 = 0xD1B54A32D192ED03ull;
constexpr uint64_t G3 = 0x8CB92BA72F3D8DD7ull;
constexpr uint64_t LCG_A = 6364136223846793005ull;
constexpr uint64_t LCG_C = 1442695040888963407ull;

thread_local char g_err[512] = "";
thread_local bool t_no_pad = false;  // td_graph_upload: lower without GROUP padding (retry)

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
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_rel_gpu() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_rel_sys() { asm volatile("fence.release.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_gpu() { asm volatile("fence.acquire.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_sys() { asm volatile("fence.acquire.sys;" ::: "memory"); }
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Cycle probe (diagnostic builds only: nvcc -DTD_CYCLE_PROBE, loaded via
// TD_LIB): with TD_F_TRACE, lane 0 records %clock64 at PROBE_WORDS points of
// every task.  `dep` is folded into a sink first, so the clock read issues
// only after that value exists (in-order issue).
#ifdef TD_CYCLE_PROBE
constexpr int TRACE_WORDS = 8;
#define PROBE(k, dep)                                                          \
  do {                                                                         \
    asm volatile("xor.b64 %0, %0, %1;" : "+l"(probe_sink) : "l"((uint64_t)(dep))); \
    uint64_t _c;                                                               \
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(_c)::"memory");              \
    probe[k] = _c;                                                             \
  } while (0)
#else
constexpr int TRACE_WORDS = 4;
#define PROBE(k, dep) do {} while (0)
#endif

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ uint64_t warp_xor_u64(uint64_t x) {
  // two REDUX.XOR (one per 32-bit half) instead of five dependent shuffle
  // rounds (A/B: the butterfly is +5 % on stencil_1d, +8 % on no_comm; the low
  // half on REDUX and the high half through shuffles in parallel: no_comm
  // +5 %, profiles/r02_ab_xormix.log)
  const uint32_t lo = __reduce_xor_sync(0xffffffffu, (uint32_t)x);
  const uint32_t hi = __reduce_xor_sync(0xffffffffu, (uint32_t)(x >> 32));
  return ((uint64_t)hi << 32) | lo;
}

// One node's slot in its worker's program (Alg. 1 (V_w, E_w) flattened):
// everything the owner warp needs, contiguous in worker order so that a 1-D
// TMA bulk copy stages the next CHUNK descriptors into shared memory while the
// current ones execute.  Up to 5 remote successors are inline as explicit
// ids (lane l messages succ[l]); larger rows are id intervals in a per-graph
// pool (nsucc == TD_OVF, succ[0] = pool offset, succ[1] = interval count).
// Predecessors are not needed on the device: inputs arrive inside the
// messages.  Multi-GPU: successor ids (and pool intervals, which never
// straddle shards) carry the owning shard in bits 28..30 (sharded graphs have
// < 2^28 nodes).
struct __align__(16) Desc {
  int32_t v;
  uint32_t nmsg;     // messages expected in the L2 mailbox (remote in-edges)
  uint32_t arg;
  uint8_t kind, nsucc, rmask, dflags;  // dflags: DF_* below
  uint32_t ldelta;   // up to 4 same-worker successors, list-position deltas (8 bits each, 0 = none)
  int32_t wslot;     // -1: own mailbox; else shared mailbox replica (edge bundling, see below)
  // identity hashes of idv = v, or of the node a halo replica computes,
  // precomputed at upload (seed-independent): h0 = mix64(seed ^ hid)
  // (A/B against hashing idv on the device: no_comm -4 %, fft -3 %, tree -4 %)
  uint64_t hid;      // mix64(idv + G1)
  uint64_t key;      // mix64(idv + G3): term key (term = mix64(tok ^ key) >> 32)
  int32_t col;       // checksum column, -1 = none
  int32_t succ[5];   // remote successors: explicit ids (nsucc <= 5), else (pool offset, interval count)
};
constexpr int NSUCC_INLINE = sizeof(((Desc*)nullptr)->succ) / sizeof(int32_t);
static_assert(sizeof(Desc) == 64, "descriptor must be 64 bytes");
// Allocator whose value-initialisation is a no-op: the upload fills every
// descriptor itself, so a 256 MB std::vector<Desc> need not be zeroed first.
template <typename T>
struct uninit_alloc : std::allocator<T> {
  template <typename U>
  struct rebind { using other = uninit_alloc<U>; };
  uninit_alloc() = default;
  template <typename U>
  uninit_alloc(const uninit_alloc<U>&) {}
  template <typename U>
  void construct(U* p) noexcept {}
  template <typename U, typename... A>
  void construct(U* p, A&&... a) { ::new ((void*)p) U(std::forward<A>(a)...); }
};
using DescVec = std::vector<Desc, uninit_alloc<Desc>>;
constexpr uint8_t TD_OVF = 0xFF;
constexpr uint8_t DF_REMOTE_PRED = 1;
constexpr uint8_t DF_MULTI = 2;  // needs the sharded path: a remote predecessor or successor, or a relay
// GROUP passes: ring adds run in rounds (set at upload by a greedy colouring
// of the pass's nodes, so that nodes of one round feed distinct ring slots):
// bits 3-4 = this node's round, bits 5-7 of the pass's first node = rounds
// (0 = no ring adds in the pass; at most K = 4)
constexpr int DF_RING_ROUND_SHIFT = 3, DF_RING_NROUNDS_SHIFT = 5;
// Internal descriptor kind (never a graph node): a cross-shard relay.  It
// waits for the k producers of a bundled group that live on this shard and
// forwards their summed messages -- one remote add of (k << 48) + sum per
// replica on each other shard (aggregate per (src GPU, dst)).
constexpr uint8_t KIND_RELAY = 0x7F;
  // some predecessor lives on another shard (sys-scope acquire, peer halo)
constexpr int RANK_SHIFT = 28;
constexpr int32_t ID_MASK = (1 << RANK_SHIFT) - 1;
// Message targets in descriptors / the successor pool: a target on this GPU
// is its plain id; a target on shard r carries r + 1 in bits 28..31.  So a
// node whose targets are all local needs no decoding at all and runs the
// one-GPU code path inside the sharded kernel (DF_MULTI below).
__device__ __host__ __forceinline__ int target_shard(int32_t x) {  // -1 = this GPU
  return (int)((uint32_t)x >> RANK_SHIFT) - 1;
}
constexpr int MSG_SHIFT = 48;                         // mailbox: [count:16 | sum:48]
constexpr uint64_t MSG_ONE = 1ull << MSG_SHIFT;
constexpr uint64_t SUM_MASK = MSG_ONE - 1;

constexpr int LRING = 64;          // per-warp local accumulator ring (direct local decrement)
constexpr int SHARE_MIN_INDEG = 64; // bundle consumers whose identical predecessor lists are at least this long
constexpr int SHARE_FANOUT = 512;   // consumers per shared mailbox replica (A/B over 32..4096: 512 best)
// Combiners (one-GPU bundled groups with >= COMB_MIN_REP replicas): a
// producer sends ONE returning add into one of P combiner words (about
// COMB_PER producers each) instead of one add per replica; the producer whose
// add completes a combiner forwards (k << 48) + partial sum to every replica.
// Adds on the polled replica words per step drop from W * R to P * R (the L2
// serves ~6e10 adds/s with no pollers and ~2.5e10 under polling,
// profiles/r02_red_contention.log), for one returning-atomic round trip.
// Policy (A/B profiles/r02_ab_all_to_all_comb2.log): the returning add costs
// its producer an L2 round trip before the warp's next node, so combiners pay
// only when a worker produces at most COMB_MAX_PER_WORKER nodes of the group
// and the group has >= COMB_MIN_REP replicas (all_to_all 8192x10 at 4096
// workers 0.060 -> 0.051 ms; at 2048 workers, 4 producers each, 0.060 -> 0.072).
constexpr int COMB_MIN_REP = 8;
constexpr int COMB_MAX_PER_WORKER = 2;
constexpr int COMB_PER = 64;
// (a replica's 8 sub-words in one 64 B line -- one poll request per consumer
// -- with combiners feeding it was measured: all_to_all 8192x100 0.45 ->
// 1.03 ms, profiles/r02_ab_all_to_all_comb.log)
constexpr int SHARE_STRIDE = 32;    // u64 words between replica sub-words: one 256 B L2 granule each, so
                                    // the ~W*R atomics of a bundled step spread over many L2 slices
#ifndef TD_SHARE_SPLIT
#define TD_SHARE_SPLIT 8
#endif
// (16 / 32 sub-words measured: all_to_all 8192x10 0.061 / 0.085 ms against
// 0.061 at 8, profiles/r02_ab_all_to_all_split.log)
constexpr int SHARE_SPLIT = TD_SHARE_SPLIT;  // sub-words per replica: producer u adds into sub-word u % 8, the
                                    // consumer sums all 8 (cuts same-address serialisation 8x)
constexpr int WARPS_PER_CTA = 4;   // 128 threads
// descriptors per TMA stage: 32 (2 KiB) in the lean kernels (A/B against 16:
// -1 % on stencil_1d, fft, tree, nearest), 16 in the tile kernels, whose
// shared memory holds the halo boxes
constexpr int CHUNK_LEAN = 32, CHUNK_ST2D = 16;
constexpr int STAGES = 2;

struct Params {
  const Desc* desc;          // [positions] worker-major programs
  const int64_t* work_ptr;   // [n_workers+1]
  const int2* succ_pool;     // overflow successor intervals
  const int32_t* worker_of;  // stats only
  const uint8_t* wremote;    // [n_workers] 1 if the worker ever messages another GPU (start handshake)
  int32_t n_workers;         // resident warps: graph workers, then one per relay
  int32_t n_graph_workers;
  unsigned long long* colsum;      // this execution's checksum bank
  unsigned long long* colsum_zero; // the other bank, zeroed at kernel start (NULL: no checksum launch)
  int32_t n_cols;
  unsigned long long* mbox;  // [slots] per-node mailbox word (count | term sum), then 2 banks of shared slots
  int32_t n_nodes;           // ids >= n_nodes address shared mailbox slots
  int64_t n_shared;          // shared slots per bank (bank = exec_no & 1)
  int64_t mbox_words;        // mailbox array length (node words + both banks of shared replicas)
  int64_t shared_base;       // mailbox word of shared replica 0, bank 0 (256 B aligned)
  int32_t comb_id0;          // message targets >= comb_id0 are combiners (INT32_MAX: none)
  int64_t comb_base;         // mailbox word of combiner 0 (combiners SHARE_STRIDE words apart)
  const int4* comb;          // [combiners] {producers k, first replica, replicas, 0}
  uint32_t shared_backoff_ns; // polling backoff on shared mailboxes (many pollers per word)
  unsigned long long* token; // [slots] output tokens (read back by the host)
  uint32_t* tally;
  unsigned long long* stats;          // [0]=executed [1]=cross [2]=local [3]=init [4]=cross_rank
  unsigned long long* trace;          // [4*n] TD_F_TRACE timestamps
  const volatile uint32_t* ext_pre;   // host-mapped
  uint32_t* ext_post;                 // host-mapped
  volatile uint32_t* abort_flag;      // host-mapped: host asks the kernel to stop
  uint32_t* poison;                   // device: set when a worker gave up / invariant broke
  uint32_t* poison_host;              // host-mapped mirror of the winning poison code
  uint64_t seed;
  uint32_t exec_no;   // monotonically increasing execution number (flags)
  uint32_t flags;
  uint64_t spin_limit;
  // sharding
  int32_t my_rank, n_ranks;
  uint32_t* started;                  // [TD_MAX_RANKS] local: exec_no once peer r started
  unsigned long long* peer_mbox[TD_MAX_RANKS];
  uint32_t* peer_started[TD_MAX_RANKS];
  // TD_BODY_STENCIL2D context (config 5): node v = t*ntiles + ty*tiles_x + tx
  int32_t st_nx, st_ny, st_tiles_x, st_tiles_y, st_ntiles;
  uint32_t* st_grid[2];                       // this shard's double-buffered grid
  uint32_t* st_peer_grid[TD_MAX_RANKS][2];    // peers' grids (halo reads over NVLink)
  const uint8_t* st_tile_rank;                // [ntiles] owning shard (NULL = all local)
  alignas(64) CUtensorMap st_tmap[2];         // 2-D TMA maps of the grid buffers (box 72 x 66)
  // SM-balanced placement (P.place): the grid is full (occ CTAs on every SM)
  // and worker w runs on the warp with rank q = w / n_sms on SM sm_order[w %
  // n_sms], q = (CTA slot on its SM) * 4 + warp in CTA.  Consecutive workers go
  // to different SMs, then different SM sub-partitions.
  int32_t place, occ, n_sms;
  int32_t slot_shift;        // mailbox words are 2^slot_shift u64 apart (see slot())
  // TD_F_DYNAMIC (arrival-order dispatch): node-indexed programs and one
  // ready queue per SM (queue of node v = its static owner's SM)
  const Desc* qdesc;         // [n] node v's program (all in-edges via the mailbox)
  const uint32_t* qinfo;     // [n] in-degree (low 16 bits) | queue (high 16 bits)
  unsigned long long* q_slots;  // [2n] queue slots {tag | input sum, node id + 1} once ready (sources permanent)
  const int64_t* q_base;     // [n_sms + 1] first slot of each queue
  const uint32_t* q_src;     // [n_sms] sources at the head of each queue
  uint32_t* q_head;          // [n_sms] claim tickets (reset per launch)
  uint32_t* q_tail;          // [n_sms] enqueue positions (reset to q_src per launch)
  // TD_BODY_MEMORY: per-worker scratch regions of scratch_words u64 each
  unsigned long long* scratch;
  int64_t scratch_words;
  const int16_t* sm_dense;   // [TD_MAX_SMID] %smid -> dense SM index, -1 = unknown
  uint32_t* sm_ctr;          // [TD_MAX_SMID] per-SM CTA arrival counter (epoch << 8 | count)
};

// node v's mailbox word (identity).  Two swizzles that spread the words of
// concurrently active nodes over more L2 lines / slices were measured and
// removed: both slower (profiles/r01_summary.md).
// Mailbox words are 2^slot_shift words apart (chosen per graph at upload:
// 32 B apart for one-node-per-pass graphs, so the words of neighbouring
// consumers -- polled and added to in the same level -- sit in different L2
// sectors; 8 B apart for GROUP graphs, whose K-node passes poll K
// consecutive words in one request.  A/B, profiles/r02_ab_slot_spacing.log,
// r02_ab_slot_policy.log: one node per pass: stencil_1d 1024 -1.6..-2.2 %,
// fft 4096 workers -16 %, tree / no_comm +1.5 %; GROUP 4 +5..10 %, GROUP 2
// -3..+8 %.)
#ifdef TD_CHECKS
// (debug build, -DTD_CHECKS: device-side bounds checks in place of
// compute-sanitizer, which the GPU pool does not offer)
#define TD_CHECK(cond, what, val)                                                            \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("TD_CHECK failed: %s (%lld) block %d thread %d\n", what, (long long)(val), blockIdx.x, threadIdx.x); \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define TD_CHECK(cond, what, val) do {} while (0)
#endif
// Column checksums are double-buffered by checksum-launch parity: a
// CHECKSUM launch XORs into its bank and zeroes the other one (whose
// previous contents were copied to the host behind the previous checksum
// launch, in stream order), so no memset precedes the kernel.
__device__ __forceinline__ void zero_other_colsum(const Params& P) {
  if (!P.colsum_zero) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n_cols; i += gridDim.x * blockDim.x) P.colsum_zero[i] = 0;
}
// Poison the execution (first code wins: the device word is sticky across
// queued launches) and, for the code that won, mirror it into the host-mapped
// word the host reads after completion -- a clean replay then needs no copy
// of the poison word behind the kernel (4 us per replay, scripts/launch_variants.py)
__device__ __forceinline__ void poison_set(const Params& P, uint32_t code) {
  if (atomicCAS(P.poison, 0u, code) == 0u) *(volatile uint32_t*)P.poison_host = code;
}
__device__ __forceinline__ int64_t slot(const Params& P, int v) {
  TD_CHECK(v >= 0 && v < P.n_nodes, "mailbox of node id", v);
  return (int64_t)v << P.slot_shift;
}

// Diagnostic flags (stats / tally / trace) exist only in the DIAG
// instantiations; launches without them run kernels with the checks (and the
// per-warp counters they keep live) compiled out: same-box A/B, no_comm
// 0.84 -> 0.72 ms, tree 2.08 -> 1.68, fft 2.38 -> 2.12, stencil_1d -3 %.
template <bool DIAG>
__device__ __forceinline__ bool diag(const Params& P, uint32_t f) { return DIAG && (P.flags & f); }

__device__ __forceinline__ uint64_t ld_relaxed_gpu_u64(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const unsigned long long* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_gpu_u64(unsigned long long* p, uint64_t v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_add_sys_u64(unsigned long long* p, uint64_t v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

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
  // descriptors are read once per replay: evict them first, so they do not
  // push the mailbox lines (prefetched at launch) out of L2 (A/B,
  // profiles/r02_ab_desc_hint.log: headline stencil_1d -1.3 %, fft 1024
  // workers -1.5 %, tree 4096 workers +1.5 %, others within noise)
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
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

// One LCG lane-update, x <- A*x + C (mod 2^64).  The empty asm makes every
// step's value opaque: without it the compiler composes an unrolled run of
// affine steps into ONE step (A^8 x + C_8 -- exact in Z/2^64), so the loop
// would do an eighth of the work it claims.
__device__ __forceinline__ uint64_t lcg_step(uint64_t x) {
  x = LCG_A * x + LCG_C;
  asm volatile("" : "+l"(x));
  return x;
}

template <bool PLAIN = false>
// lc = (lane + 1) * G2 and (lane + 33) * G2, this lane's two LCG-seed
// constants (computed once per warp by the kernel, not per node)
__device__ __forceinline__ uint64_t run_body(int kind, uint32_t arg, uint64_t h, const ulonglong2& lc) {
  if (kind == TD_BODY_COMPUTE) {
    uint64_t x0 = mix64(h ^ lc.x);
    uint64_t x1 = mix64(h ^ lc.y);
    // long bodies: blocks of 8 steps (no loop overhead per step, so the
    // body runs at the chip's LCG peak); the remainder (and the whole of a
    // short body, the overhead end of the sweep) in a rolled loop -- a fully
    // unrolled loop's remainder dispatch cost more branches at arg = 1 (A/B -3 %)
    uint32_t i = arg;
    if (i >= 8) {
#pragma unroll 1
      for (; i >= 8; i -= 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          x0 = lcg_step(x0);
          x1 = lcg_step(x1);
        }
      }
    }
#pragma unroll 1
    for (; i; --i) {
      x0 = lcg_step(x0);
      x1 = lcg_step(x1);
    }
    return warp_xor_u64(x0 ^ x1);
  }
  if (!PLAIN && kind == TD_BODY_BUSY_WAIT) {
    const uint64_t t0 = globaltimer();
    while (globaltimer() - t0 < (uint64_t)arg) {
    }
  }
  return 0;
}

// --- memory_bound body (Task Bench's memory_bound kernel) ---
// The task streams `n` u64 words (n a multiple of 64) through its worker's
// scratch region: it stores v_k = h + k*G2 (16 B per lane per instruction,
// 512 B per warp), then loads them back with L1 bypassed and XOR-folds them:
// r = XOR_k v_k.  2 * 8n bytes of memory traffic per task; when the tasks in
// flight stream more than L2 holds, both passes go to HBM.
__device__ __forceinline__ uint64_t memory_body(const Params& P, int w, uint32_t n, uint64_t h, int lane) {
  TD_CHECK(n <= (uint32_t)P.scratch_words, "memory_bound words beyond scratch", n);
  unsigned long long* s = P.scratch + (int64_t)w * P.scratch_words;
#pragma unroll 4
  for (uint32_t k = 2u * lane; k < n; k += 64u) {
    const uint64_t a = h + (uint64_t)k * G2, b = h + (uint64_t)(k + 1) * G2;
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(s + k), "l"(a), "l"(b) : "memory");
  }
  uint64_t r = 0;
#pragma unroll 4
  for (uint32_t k = 2u * lane; k < n; k += 64u) {
    uint64_t a, b;
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(s + k) : "memory");
    r ^= a ^ b;
  }
  return warp_xor_u64(r);
}

// --- config-5 tile body: 5-point stencil on a 64x64 tile ---------------------
// out[y][x] = 2*c + up + down + left + right (mod 2^32, cells outside the grid
// are 0); t == 0 initialises the tile.  Returns the tile fold
// r = sum_k out_k * (2k+1) (mod 2^64), k = row-major cell index in the tile.
constexpr int TILE = 64;

template <bool MULTI>
__device__ __forceinline__ const uint32_t* tile_buf(const Params& P, int tile, int b) {
  if (MULTI && P.st_tile_rank) {
    const int r = P.st_tile_rank[tile];
    if (r != P.my_rank) return P.st_peer_grid[r][b];
  }
  return P.st_grid[b];
}

template <bool MULTI>
__device__ __forceinline__ uint64_t stencil2d_body(const Params& P, int v, int lane) {
  const int nx = P.st_nx;
  const int t = v / P.st_ntiles;
  const int tile = v - t * P.st_ntiles;
  const int ty = tile / P.st_tiles_x, tx = tile - ty * P.st_tiles_x;
  const int x0 = tx * TILE, y0 = ty * TILE;
  const int cx = x0 + 2 * lane;
  uint32_t* out = P.st_grid[t & 1];
  uint64_t r = 0;
  if (t == 0) {
    for (int y = 0; y < TILE; ++y) {
      const uint64_t base = (uint64_t)(y0 + y) * (uint64_t)nx + (uint64_t)cx;
      const uint32_t a = (uint32_t)mix64(P.seed ^ (base + G2));
      const uint32_t b = (uint32_t)mix64(P.seed ^ (base + 1 + G2));
      __stcs(reinterpret_cast<uint2*>(out + base), make_uint2(a, b));
      const uint64_t k = (uint64_t)(y * TILE + 2 * lane);
      r += (uint64_t)a * (2 * k + 1) + (uint64_t)b * (2 * k + 3);
    }
    return warp_sum_u64(r);
  }
  const int bi = (t - 1) & 1;
  const uint32_t* c = tile_buf<MULTI>(P, tile, bi);
  const uint32_t* up = ty > 0 ? tile_buf<MULTI>(P, tile - P.st_tiles_x, bi) : nullptr;
  const uint32_t* dn = ty + 1 < P.st_tiles_y ? tile_buf<MULTI>(P, tile + P.st_tiles_x, bi) : nullptr;
  const uint32_t* lf = tx > 0 ? tile_buf<MULTI>(P, tile - 1, bi) : nullptr;
  const uint32_t* rt = tx + 1 < P.st_tiles_x ? tile_buf<MULTI>(P, tile + 1, bi) : nullptr;
  auto row = [&](int y) -> uint2 {  // local row y in [-1, 64] of this lane's two columns
    const uint32_t* src = y < 0 ? up : (y >= TILE ? dn : c);
    if (!src) return make_uint2(0, 0);
    const unsigned long long w = __ldcg(reinterpret_cast<const unsigned long long*>(
        src + (uint64_t)(y0 + y) * (uint64_t)nx + (uint64_t)cx));
    return make_uint2((uint32_t)w, (uint32_t)(w >> 32));
  };
  auto halo_l = [&](int y) -> uint32_t {
    return (lane == 0 && lf) ? __ldcg(lf + (uint64_t)(y0 + y) * (uint64_t)nx + (uint64_t)(x0 - 1)) : 0u;
  };
  auto halo_r = [&](int y) -> uint32_t {
    return (lane == 31 && rt) ? __ldcg(rt + (uint64_t)(y0 + y) * (uint64_t)nx + (uint64_t)(x0 + TILE)) : 0u;
  };
  uint2 prev = row(-1), cur = row(0);
  uint32_t hl = halo_l(0), hr = halo_r(0);
  constexpr int B = 8;  // rows loaded ahead (memory-level parallelism)
  for (int yb = 0; yb < TILE; yb += B) {
    uint2 nxt[B];
    uint32_t nhl[B], nhr[B];
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const int y = yb + 1 + i;
      nxt[i] = row(y);
      nhl[i] = y < TILE ? halo_l(y) : 0u;
      nhr[i] = y < TILE ? halo_r(y) : 0u;
    }
#pragma unroll
    for (int i = 0; i < B; ++i) {
      const int y = yb + i;
      uint32_t left = __shfl_up_sync(0xffffffffu, cur.y, 1);
      uint32_t right = __shfl_down_sync(0xffffffffu, cur.x, 1);
      if (lane == 0) left = hl;
      if (lane == 31) right = hr;
      const uint2 nx2 = nxt[i];
      const uint32_t ox = 2u * cur.x + prev.x + nx2.x + left + cur.y;
      const uint32_t oy = 2u * cur.y + prev.y + nx2.y + cur.x + right;
      __stcs(reinterpret_cast<uint2*>(out + (uint64_t)(y0 + y) * (uint64_t)nx + (uint64_t)cx), make_uint2(ox, oy));
      const uint64_t k = (uint64_t)(y * TILE + 2 * lane);
      r += (uint64_t)ox * (2 * k + 1) + (uint64_t)oy * (2 * k + 3);
      prev = cur;
      cur = nx2;
      hl = nhl[i];
      hr = nhr[i];
    }
  }
  return warp_sum_u64(r);
}

// Single-GPU tile body on the tensor memory accelerator: ONE
// cp.async.bulk.tensor.2d brings the 66 x 72 halo box (rows y0-1..y0+64,
// columns x0-4..x0+67; the innermost start coordinate must be 16-byte
// aligned, measured: x0-2 faults) into this warp's shared-memory tile; the
// hardware's out-of-bounds zero fill is exactly the grid boundary.
constexpr int BOX_W = 72, BOX_H = 66, BOX_X0 = 4;
constexpr uint32_t BOX_BYTES = BOX_W * BOX_H * 4;                 // 19,008
constexpr uint32_t TILE_SMEM = (BOX_BYTES + 127) / 128 * 128;     // per warp, 128 B aligned
// (a 64 x 66 box aligned on the tile, with the left / right halo columns read
// by the lanes from global memory, was measured: 4.76 -> 8.62 ms,
// profiles/r02_ab_st2d_box_promo.log; L2 promotion 0 / 64 / 128 B instead of
// 256 B: +1..2.5 %)

// Lane 0 issues the TMA halo-box load of tile task v (t >= 1) into `box`.
__device__ __forceinline__ void issue_tile_tma(const Params& P, int v, int lane, uint32_t* box, uint64_t* tbar) {
  if (lane != 0) return;
  const int t = v / P.st_ntiles;
  const int tile = v - t * P.st_ntiles;
  const int ty = tile / P.st_tiles_x, tx = tile - ty * P.st_tiles_x;
  const CUtensorMap* map = &P.st_tmap[(t - 1) & 1];
  // generic-proxy writes of the neighbours (acquired) -> async proxy; and our
  // earlier generic reads of the box buffer before TMA overwrites it
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(tbar)), "r"(BOX_BYTES)
               : "memory");
  // evict_last: the box's side sectors (16 B either side of the tile) are
  // the neighbour tiles' own data, loaded again by their boxes a tile later;
  // keeping loaded lines lets those hit in L2 (A/B, profiles/r02_ab_st2d_hint.log:
  // with the streaming output stores 4.83 -> 4.69 ms; evict_first: 7.25 ms)
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
          smem_u32(box)),
      "l"(map), "r"(tx * TILE - BOX_X0), "r"(ty * TILE - 1), "r"(smem_u32(tbar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint64_t stencil2d_body_tma(const Params& P, int v, int lane, uint32_t* box,
                                                       uint64_t* tbar, uint32_t& tphase, bool issued) {
  const int nx = P.st_nx;
  const int t = v / P.st_ntiles;
  const int tile = v - t * P.st_ntiles;
  const int ty = tile / P.st_tiles_x, tx = tile - ty * P.st_tiles_x;
  const int x0 = tx * TILE, y0 = ty * TILE;
  const int cx = x0 + 2 * lane;
  uint32_t* out = P.st_grid[t & 1];
  uint64_t r = 0;
  if (t == 0) {
    for (int y = 0; y < TILE; ++y) {
      const uint64_t base = (uint64_t)(y0 + y) * (uint64_t)nx + (uint64_t)cx;
      const uint32_t a = (uint32_t)mix64(P.seed ^ (base + G2));
      const uint32_t b = (uint32_t)mix64(P.seed ^ (base + 1 + G2));
      __stcs(reinterpret_cast<uint2*>(out + base), make_uint2(a, b));
      const uint64_t k = (uint64_t)(y * TILE + 2 * lane);
      r += (uint64_t)a * (2 * k + 1) + (uint64_t)b * (2 * k + 3);
    }
    return warp_sum_u64(r);
  }
  if (!issued) issue_tile_tma(P, v, lane, box, tbar);
  mbar_wait(tbar, tphase);
  tphase ^= 1u;
  const int c = 2 * lane + BOX_X0;  // box column of this lane's first cell
#pragma unroll 4
  for (int y = 0; y < TILE; ++y) {
    const uint32_t* row = box + (y + 1) * BOX_W;
    const uint2 cur = *reinterpret_cast<const uint2*>(row + c);
    const uint2 up = *reinterpret_cast<const uint2*>(row - BOX_W + c);
    const uint2 dn = *reinterpret_cast<const uint2*>(row + BOX_W + c);
    const uint32_t left = row[c - 1], right = row[c + 2];
    const uint32_t ox = 2u * cur.x + up.x + dn.x + left + cur.y;
    const uint32_t oy = 2u * cur.y + up.y + dn.y + cur.x + right;
    // streaming stores: the tile is read again only a whole step later, long
    // after it would have left L2; its lines should not displace the boxes'
    __stcs(reinterpret_cast<uint2*>(out + (uint64_t)(y0 + y) * (uint64_t)nx + (uint64_t)cx), make_uint2(ox, oy));
    const uint64_t k = (uint64_t)(y * TILE + 2 * lane);
    r += (uint64_t)ox * (2 * k + 1) + (uint64_t)oy * (2 * k + 3);
  }
  __syncwarp();
  return warp_sum_u64(r);
}

// --- successor messages: one data-carrying atomic per edge -----
struct Acct {
  unsigned long long cross = 0, local = 0, xrank = 0;
};

// Mailbox slot of a message target: a node id, or (ids >= n_nodes) a shared
// mailbox replica of the current bank.
// sub-word 0 of shared replica `idx` in the current bank
__device__ __forceinline__ int64_t shared_slot(const Params& P, int64_t idx) {
  return P.shared_base + (idx + (int64_t)(P.exec_no & 1u) * P.n_shared) * (SHARE_SPLIT * SHARE_STRIDE);
}
// mailbox slot of a message from producer v to target s (node or replica)
__device__ __forceinline__ int64_t target_slot(const Params& P, int s, int v) {
  // both candidates computed, one select: no branch (and no reconvergence) on
  // the send path (A/B: stencil_1d -1.9 %, no_comm -1.2 %, fft/tree/nearest +1 %)
  const int64_t sh = shared_slot(P, (int64_t)s - P.n_nodes) + (int64_t)(v & (SHARE_SPLIT - 1)) * SHARE_STRIDE;
  TD_CHECK(s >= 0 && (s < P.n_nodes || sh < P.mbox_words), "message target", s);
  int64_t r;
  asm("{\n .reg .pred p;\n setp.lt.s32 p, %1, %2;\n selp.b64 %0, %3, %4, p;\n}"
      : "=l"(r) : "r"(s), "r"(P.n_nodes), "l"((int64_t)s << P.slot_shift), "l"(sh));  // (unchecked: s may be a replica id)
  return r;
}

// A producer's message into combiner c; the add that completes it forwards
// the combined word to every replica of the group and re-arms the combiner.
__device__ __forceinline__ void combine(const Params& P, int c, uint64_t msg) {
  unsigned long long* cw = &P.mbox[P.comb_base + (int64_t)c * SHARE_STRIDE];
  TD_CHECK(P.comb_base + (int64_t)c * SHARE_STRIDE < P.mbox_words, "combiner", c);
  const uint64_t fin = (uint64_t)atomicAdd(cw, (unsigned long long)msg) + msg;
  const int4 ci = __ldg(&P.comb[c]);
  if ((uint32_t)(fin >> MSG_SHIFT) == (uint32_t)ci.x) {
    *cw = 0;  // every producer of this combiner arrived: re-armed for the next execution
    const int64_t sub = (int64_t)(c & (SHARE_SPLIT - 1)) * SHARE_STRIDE;
    for (int r = 0; r < ci.z; ++r) red_add_gpu_u64(&P.mbox[shared_slot(P, ci.y + r) + sub], fin);
  }
}

template <bool MULTI, bool PLAIN = false>
__device__ __forceinline__ void send(const Params& P, int s, int rx, uint64_t msg, int w, bool stats, Acct& a,
                                     int v) {
  if (!MULTI && !PLAIN && s >= P.comb_id0) {
    combine(P, s - P.comb_id0, msg);
    if (stats) ++a.cross;
    return;
  }
  const int64_t ts = PLAIN ? slot(P, s) : target_slot(P, s, v);
  if (MULTI) {
    const int r = target_shard(rx);
    if (r >= 0) red_add_sys_u64(&P.peer_mbox[r][ts], msg);  // over NVLink
    else red_add_gpu_u64(&P.mbox[ts], msg);
    if (stats && r >= 0) ++a.xrank;
  } else {
    red_add_gpu_u64(&P.mbox[ts], msg);
  }
  if (stats) {
    if (s >= P.n_nodes || __ldg(&P.worker_of[s]) != w) ++a.cross;
    else ++a.local;
  }
}

template <bool MULTI, bool PLAIN = false>
__device__ __forceinline__ void signal_range(const Params& P, int2 iv, uint64_t msg, int w, int lane, bool stats,
                                             Acct& a, int v) {
  const int lo = MULTI ? (iv.x & ID_MASK) : iv.x;
  const int len = iv.y - lo + 1;
  for (int o = lane; o < len; o += 32) send<MULTI, PLAIN>(P, lo + o, iv.x, msg, w, stats, a, v);
}

template <bool MULTI, bool DIAG, bool PLAIN = false, bool NO_OVF = false>
__device__ __forceinline__ void signal_succs(const Params& P, const Desc& d, uint64_t msg, int w, int lane, Acct& a) {
  const int v = d.v;
  const bool stats = diag<DIAG>(P, TD_F_STATS);
  const int ns = d.nsucc;
  if (NO_OVF || ns != TD_OVF) {
    if (lane < ns) {  // lane l sends to successor l: one RED per lane
      const int32_t x = d.succ[lane];
      send<MULTI, PLAIN>(P, MULTI ? (x & ID_MASK) : x, x, msg, w, stats, a, v);
    }
  } else {
    const int2* pool = P.succ_pool + d.succ[0];
    const int cnt = d.succ[1];
    for (int k = 0; k < cnt; ++k) signal_range<MULTI, PLAIN>(P, pool[k], msg, w, lane, stats, a, v);
  }
}

// Wait until all indeg messages of this execution arrived; returns the term
// sum.  `first` is the word of a poll the caller already issued.
template <bool MULTI>
__device__ bool wait_mailbox(const Params& P, int64_t sv, uint32_t need, uint64_t& sum, uint64_t first, bool sys,
                             uint64_t* polls = nullptr) {
  uint64_t spins = 0;
  for (;;) {
    const uint64_t word = spins == 0 ? first : (MULTI && sys) ? ld_relaxed_sys_u64(&P.mbox[sv])
                                                              : ld_relaxed_gpu_u64(&P.mbox[sv]);
    const uint32_t cnt = (uint32_t)(word >> MSG_SHIFT);
    if (cnt >= need) {
      if (cnt != need) {  // more messages than in-edges: fatal
        poison_set(P, 2u);
        return false;
      }
      sum = word & SUM_MASK;
      if (polls) *polls = spins + 1;
      return true;
    }
    if ((++spins & 4095u) == 0) {
      if (ld_relaxed_gpu(P.poison) || *P.abort_flag) return false;
      if (P.spin_limit && spins > P.spin_limit) {
        poison_set(P, 1u);
        return false;
      }
    }
  }
}

// Bundled consumer: lanes 0..SHARE_SPLIT-1 poll the replica's sub-words; the
// 64-bit sum of the words is [total count : 16 | total term sum : 48] (no
// carry can cross the field boundary for in-degree < 2^16).
template <bool MULTI>
__device__ bool wait_shared(const Params& P, int64_t base, uint32_t need, uint64_t& sum, int lane) {
  uint64_t spins = 0;
  const unsigned long long* p = &P.mbox[base + (int64_t)(lane & (SHARE_SPLIT - 1)) * SHARE_STRIDE];
  for (;;) {
    if (P.shared_backoff_ns && spins) __nanosleep(P.shared_backoff_ns);
    uint64_t w = 0;
    if (lane < SHARE_SPLIT) w = MULTI ? ld_relaxed_sys_u64(p) : ld_relaxed_gpu_u64(p);
#pragma unroll
    for (int o = SHARE_SPLIT / 2; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    w = __shfl_sync(0xffffffffu, w, 0);
    const uint32_t cnt = (uint32_t)(w >> MSG_SHIFT);
    if (cnt >= need) {
      if (cnt != need) {
        poison_set(P, 2u);
        return false;
      }
      sum = w & SUM_MASK;
      return true;
    }
    if ((++spins & 4095u) == 0) {
      if (ld_relaxed_gpu(P.poison) || *P.abort_flag) return false;
      if (P.spin_limit && spins > P.spin_limit) {
        poison_set(P, 1u);
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

// A node's bookkeeping after its sends: re-arm its mailbox and ring slot,
// store its token, checksum / tally.  (Deferring it into the owner's next
// node, under that node's first poll, was measured: fft -10 %, but tree,
// nearest, all_to_all +7..12 %, stencil_1d unchanged -- not kept.)
// Column checksums: a worker XORs the tokens of consecutive
// nodes of one column in a register and adds the fold into colsum[col] once
// per run of that column (once per replay when a worker owns one column),
// instead of one global atomic per node.
struct ColAcc {
  int col = -1;
  uint64_t x = 0;
  // (also carries the warp's last completed shared replica: a later node of
  // the same bundled group reads the same word, so it takes the sum without
  // polling -- all_to_all workers own 1-2 nodes of every level)
  int32_t sh_slot = -1;
  uint64_t sh_sum = 0;
};
__device__ __forceinline__ void colacc_flush(const Params& P, ColAcc& ca, int lane) {
  if (ca.col >= 0 && lane == 0) atomicXor(&P.colsum[ca.col], (unsigned long long)ca.x);
  ca.col = -1;
  ca.x = 0;
}

template <bool DIAG>
__device__ __forceinline__ void bookkeep(const Params& P, int v, int li, uint64_t tok, bool rearm, uint64_t* lacc,
                                         int lane, int col, ColAcc& ca) {
  __syncwarp();  // every lane has read the ring slot and the mailbox
#ifdef TD_LANE0_STORES  // A/B build: the stores under `if (lane == 0)`
  if (lane == 0) {
    if (rearm) P.mbox[slot(P, v)] = 0;
    lacc[li] = 0;
    P.token[v] = tok;
  }
#else
  // warp-uniform stores from every lane (one transaction each): no divergent
  // branch and reconvergence on the path to the next node's poll
  if (rearm) P.mbox[slot(P, v)] = 0;  // consumed: re-arm for the next replay
  lacc[li] = 0;
  TD_CHECK(v >= 0 && v < P.n_nodes, "token of node id", v);
  P.token[v] = tok;  // (a streaming store here was measured: no change, r02_ab_mbox_keep.log)
#endif
  if (diag<DIAG>(P, TD_F_TALLY) && lane == 0) atomicAdd(&P.tally[v], 1u);
  if ((P.flags & TD_F_CHECKSUM) && col >= 0) {  // tok and col are warp-uniform
    if (col != ca.col) {
      colacc_flush(P, ca, lane);
      ca.col = col;
    }
    ca.x ^= tok;
  }
}

__device__ __noinline__ void fire_ext_post(const Params& P, uint32_t arg, int lane) {
  if (lane == 0) st_release_sys(&P.ext_post[arg], P.exec_no);
}

// Execute one node on its owner warp (EXECUTE_OP).
// Returns false if the execution was aborted/poisoned.
// PLAIN: the graph has only empty / compute_bound bodies, no shared mailbox
// replicas, no relays and no external conditions (host-checked at upload);
// its kernels carry none of those branches.  NO_OVF (the one-GPU PLAIN
// kernel): no successor row overflows into the pool either.
template <bool MULTI, bool ST2D, bool DIAG, bool PLAIN = false, bool NO_OVF = false>
__device__ __forceinline__ bool execute_node(const Params& P, const Desc& d, int pos, uint64_t* lacc, int w, int lane,
                                             bool& peers_ok, Acct& a, uint32_t* box, uint64_t* tbar,
                                             uint32_t& tphase, const Desc* next, int& prefetched, ColAcc& ca,
                                             const ulonglong2& lc) {
  if (MULTI && w >= P.n_graph_workers) {  // relay warps hold relays only (no per-node kind check)
    uint64_t rsum;
    if (!wait_shared<MULTI>(P, shared_slot(P, d.wslot), d.nmsg, rsum, lane)) return false;
    if (!peers_ok) {
      if (!wait_peers_started(P)) return false;
      peers_ok = true;
    }
    signal_succs<MULTI, DIAG>(P, d, ((uint64_t)d.nmsg << MSG_SHIFT) + rsum, w, lane, a);
    return true;
  }
  const int v = d.v;
  // a padding slot of a GROUP layout, met by the one-node loop of a
  // diagnostics launch (the PLAIN kernels never see padded layouts)
  if (!PLAIN && v < 0) return true;
  const bool tr = diag<DIAG>(P, TD_F_TRACE);
  uint64_t ts0 = 0, ts1 = 0, ts2 = 0;
#ifdef TD_CYCLE_PROBE
  uint64_t probe[TRACE_WORDS] = {}, probe_sink = 0;
  (void)ts0, (void)ts1, (void)ts2;
  PROBE(0, 0);
#else
  if (tr) ts0 = globaltimer();
#endif
  const int64_t sv = slot(P, v);
  const uint32_t nmsg = d.nmsg;
  const int32_t wslot = d.wslot;
  // The first poll goes out before anything else; everything below up to the
  // wait (identity hash, descriptor fields) overlaps its L2 round trip instead
  // of following it.  (Also resolving each lane's RED target before the wait
  // was measured: stencil_1d equal, every other pattern 4-8 % slower.)
  const bool own_mbox = nmsg && (PLAIN || wslot < 0);
  uint64_t first = 0;
  // system scope only where a message can come from another GPU
#ifdef TD_SYS_SCOPE_ALL
  const bool sys_poll = MULTI;
#else
  const bool sys_poll = MULTI && (d.dflags & DF_REMOTE_PRED);
#endif
  if (own_mbox) first = sys_poll ? ld_relaxed_sys_u64(&P.mbox[sv]) : ld_relaxed_gpu_u64(&P.mbox[sv]);
  // identity hashes precomputed at upload (seed-independent); one mix64 for
  // the seed, materialised before the wait (the compiler would otherwise sink
  // it past the poll loop, onto the critical path)
  // (computing the next node's h0 one node ahead was measured again with the
  // precomputed hid: +2 % stencil_1d, +12 % no_comm, +7 % tree -- not kept)
  uint64_t h0 = mix64(P.seed ^ d.hid);
  const uint64_t key = d.key;
  asm volatile("" : "+l"(h0));
  // terms delivered by earlier nodes of this worker (same-worker edges): all
  // local predecessors precede v in this worker's list, so read before waiting
  const int li = pos & (LRING - 1);
  uint64_t sum = lacc[li];
  const uint32_t ldelta = d.ldelta;
  const int kind = d.kind;
  const uint32_t arg = d.arg;
  if (nmsg) {
    uint64_t rsum;
    // (issuing this poll one node early, right after the previous node's sends,
  // was measured: stencil_1d +13 %, no_comm +10 %, tree +10..24 %,
  // profiles/r02_ab_early_poll.log; so were two staggered early polls plus
  // this one: stencil_1d +26 %, tree +34 %, profiles/r02_ab_stagger.log --
  // extra polls of the next node's mailbox slow the messages it waits for)
  // (a separate fast path for "first poll complete" was measured four times,
    // also with its test pinned after the h0 hash: stencil_1d +2.6..4 %, tree
    // -2..4 %.  A faster path to the sends makes the next node's first poll
    // leave earlier, and more of them return before the neighbours' messages
    // and cost a second round trip: not kept)
    if (PLAIN || own_mbox) {
#ifdef TD_CYCLE_PROBE
      uint64_t npolls = 0;
      if (!wait_mailbox<MULTI>(P, sv, nmsg, rsum, first, sys_poll, &npolls)) return false;
      probe[7] = npolls;
#else
      if (!wait_mailbox<MULTI>(P, sv, nmsg, rsum, first, sys_poll)) return false;
#endif
    } else if (!MULTI && wslot == ca.sh_slot) {  // (one GPU: the sharded kernels are at their register limit)
      rsum = ca.sh_sum;
    } else {
      if (!wait_shared<MULTI>(P, shared_slot(P, wslot), nmsg, rsum, lane)) return false;
      if (!MULTI) {
        ca.sh_slot = wslot;
        ca.sh_sum = rsum;
      }
    }
    sum += rsum;
  }
#ifdef TD_CYCLE_PROBE
  PROBE(1, sum);
#else
  if (tr) ts1 = globaltimer();
#endif
  if (!PLAIN && kind == TD_BODY_EXT_PRE) {
    uint64_t spins = 0;
    while ((int32_t)(ld_volatile_u32(&P.ext_pre[arg]) - P.exec_no) < 0) {
      if ((++spins & 4095u) == 0 && (ld_relaxed_gpu(P.poison) || *P.abort_flag)) return false;
    }
  }
  const uint64_t h = mix64(h0 ^ sum);
  PROBE(2, h);
  uint64_t tok;
  if (ST2D && kind == TD_BODY_STENCIL2D) {
    // tile data produced by other warps (other GPUs only if a predecessor is
    // remote): acquire after the messages arrived
    const bool remote_in = MULTI && (d.dflags & DF_REMOTE_PRED);
    if (remote_in) fence_acq_sys();
    else fence_acq_gpu();
    if (!remote_in) {  // all halo data local: 2-D TMA box
      tok = h ^ stencil2d_body_tma(P, v, lane, box, tbar, tphase, prefetched == v);
      // look-ahead: the box is free again -- if the next tile's inputs have all
      // arrived, start its TMA load now so it overlaps this tile's release
      // fence (which waits for this tile's stores) and sends
      prefetched = -1;
      if (next && next->kind == TD_BODY_STENCIL2D && next->nmsg && next->wslot < 0 &&
          next->v >= P.st_ntiles && !(next->dflags & DF_REMOTE_PRED)) {
        const uint64_t nw = ld_relaxed_gpu_u64(&P.mbox[slot(P, next->v)]);
        if ((uint32_t)(nw >> MSG_SHIFT) == next->nmsg) {
          fence_acq_gpu();
          issue_tile_tma(P, next->v, lane, box, tbar);
          prefetched = next->v;
        }
      }
    } else {
      tok = h ^ stencil2d_body<MULTI>(P, v, lane);  // peer halo rows over NVLink
    }
    // publish the tile before any successor may read it (system scope only
    // if a successor lives on another GPU)
    __syncwarp();
    if (MULTI && d.rmask) fence_rel_sys();
    else fence_rel_gpu();
  } else if (!PLAIN && kind == TD_BODY_MEMORY) {
    tok = h ^ memory_body(P, w, arg, h, lane);
  } else {
    tok = h ^ run_body<PLAIN>(kind, arg, h, lc);
  }
  PROBE(3, tok);
  const uint64_t term = mix64(tok ^ key) >> 32;
#ifdef TD_CYCLE_PROBE
  PROBE(4, term);
#else
  if (tr) ts2 = globaltimer();
#endif
  if (MULTI && !peers_ok && d.rmask) {  // (peers_ok first: no descriptor load once the peers are up)
    if (!wait_peers_started(P)) return false;
    peers_ok = true;
  }
  // (reading nsucc / succ[lane] before the wait instead was measured: equal
  // on stencil_1d, 2-4 % slower on fft, tree and nearest)
  // (reading this lane's successor id and count right after the wait, so the
  // shared-memory loads overlap the body, was measured: no change,
  // profiles/r02_ab_hoist.log)
  signal_succs<MULTI, DIAG, PLAIN, NO_OVF>(P, d, MSG_ONE + term, w, lane, a);
  PROBE(5, 0);
  if (lane == 0) {
    uint32_t ld = ldelta;
    while (ld) {  // direct local delivery (no L2 round trip)
      lacc[(pos + (int)(ld & 0xFFu)) & (LRING - 1)] += term;
      ld >>= 8;
      if (diag<DIAG>(P, TD_F_STATS)) ++a.local;
    }
  }
  // External postcondition: out of line.  Inline, ptxas if-converts it into a
  // predicated MEMBAR.SYS, and a predicated-off MEMBAR.SYS still waits for
  // this warp's outstanding memory operations (its REDs, the early poll):
  // measured +300..800 cycles on every node (scripts/cycle_probe.py).
  if (!PLAIN && __builtin_expect(kind == TD_BODY_EXT_POST, 0)) fire_ext_post(P, arg, lane);
  bookkeep<DIAG>(P, v, li, tok, own_mbox, lacc, lane, d.col, ca);
  if (tr) {
    if (lane == 0) {
#ifdef TD_CYCLE_PROBE
      PROBE(6, 0);
      for (int k = 0; k < TRACE_WORDS; ++k) P.trace[TRACE_WORDS * (int64_t)v + k] = probe[k];
      if (probe_sink == 0x5EED5EED5EED5EEDull) P.stats[7] = 1;  // keeps the sink (and the probe order) live
#else
      const uint64_t ts3 = globaltimer();
      P.trace[4 * (int64_t)v + 0] = ts0;
      P.trace[4 * (int64_t)v + 1] = ts1;
      P.trace[4 * (int64_t)v + 2] = ts2;
      P.trace[4 * (int64_t)v + 3] = ts3;
#endif
    }
  }
  return true;
}

// GROUP mode (one-GPU PLAIN graphs whose worker lists split into groups of K
// equal-level nodes, checked at upload; K = 2 "PAIR" or 4): the warp runs the
// group's K nodes at once, 32/K lanes per node and 2K LCG lanes per thread,
// so one pass of the loop's overhead serves K nodes.  Same token rule as
// execute_node.  lcb = (hl + 1) * G2 for this lane's index hl in its node's
// lane group; its LCG lane j (0..2K-1) is hl + j * 32/K.
template <int K, bool MULTI = false>
__device__ __forceinline__ bool execute_group(const Params& P, const Desc* dp, int pos, uint64_t* lacc, int lane,
                                              uint64_t lcb, bool& peers_ok) {
  constexpr int LPN = 32 / K;   // lanes per node
  constexpr int NL = 64 / LPN;  // LCG lanes per thread
  const int grp = lane / LPN, hl = lane % LPN;
  const Desc& d = dp[grp];
  const int v = d.v;
  const int mypos = pos + grp;
  const uint32_t nmsg = d.nmsg;
#ifdef TD_CYCLE_PROBE
  // (diagnostic build: per pass, lane 0 records %clock64 at entry, inputs
  // ready, term, sends issued, end, and the number of poll rounds, into the
  // trace words of the pass's first node; TD_F_TRACE runs the GROUP kernel)
  uint64_t probe[TRACE_WORDS] = {}, probe_sink = 0;
  const bool tr = (P.flags & TD_F_TRACE) && P.trace;
  PROBE(0, 0);
  probe[6] = globaltimer();
#endif
  // sharded: system scope only where a predecessor lives on another GPU
  const bool sys_poll = MULTI && (d.dflags & DF_REMOTE_PRED);
  uint64_t word = 0;
  TD_CHECK(v < P.n_nodes && (v >= 0 || nmsg == 0), "group node id", v);
  const int64_t sv = (int64_t)v << P.slot_shift;  // (v = -1, a padding slot, has nmsg = 0)
  if (nmsg) word = sys_poll ? ld_relaxed_sys_u64(&P.mbox[sv]) : ld_relaxed_gpu_u64(&P.mbox[sv]);
  uint64_t h0 = mix64(P.seed ^ d.hid);
  const uint64_t key = d.key;
  asm volatile("" : "+l"(h0));
  const int li = mypos & (LRING - 1);
  uint64_t sum = lacc[li];
  const uint32_t ldelta = d.ldelta;
  const int kind = d.kind;
  const uint32_t arg = d.arg;
  bool ready = nmsg == 0 || (uint32_t)(word >> MSG_SHIFT) >= nmsg;
  uint64_t spins = 0;
  while (!__all_sync(0xffffffffu, ready)) {
    if (!ready) {
      word = sys_poll ? ld_relaxed_sys_u64(&P.mbox[sv]) : ld_relaxed_gpu_u64(&P.mbox[sv]);
      ready = (uint32_t)(word >> MSG_SHIFT) >= nmsg;
    }
    if ((++spins & 4095u) == 0) {
      if (ld_relaxed_gpu(P.poison) || *P.abort_flag) return false;
      if (P.spin_limit && spins > P.spin_limit) {
        if (lane == 0) poison_set(P, 1u);
        return false;
      }
    }
  }
#ifdef TD_CYCLE_PROBE
  PROBE(1, word);
  {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    probe[5] = spins | ((uint64_t)smid << 32);
  }
#endif
  const bool extra = nmsg && (uint32_t)(word >> MSG_SHIFT) != nmsg;  // more messages than in-edges
  if (__any_sync(0xffffffffu, extra)) {
    if (extra) poison_set(P, 2u);
    return false;
  }
  if (nmsg) sum += word & SUM_MASK;
  const uint64_t h = mix64(h0 ^ sum);
  uint64_t body = 0;
  // the LCG lanes only where a node of the group has a compute body (the
  // empty-body Task Bench graphs skip the 2K seed hashes and the reduction)
  if (__any_sync(0xffffffffu, kind == TD_BODY_COMPUTE)) {
  uint64_t x[NL];
#pragma unroll
  for (int j = 0; j < NL; ++j) x[j] = mix64(h ^ (lcb + (uint64_t)(j * LPN) * G2));
  uint32_t it = kind == TD_BODY_COMPUTE ? arg : 0u;
  if (it >= 8) {  // long bodies in blocks of 8 steps (see run_body)
#pragma unroll 1
    for (; it >= 8; it -= 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int j = 0; j < NL; ++j) x[j] = lcg_step(x[j]);
    }
  }
#pragma unroll 1
  for (; it; --it) {
#pragma unroll
    for (int j = 0; j < NL; ++j) x[j] = lcg_step(x[j]);
  }
  uint64_t y = x[0];
#pragma unroll
  for (int j = 1; j < NL; ++j) y ^= x[j];
  uint32_t lo = (uint32_t)y, hi = (uint32_t)(y >> 32);
#pragma unroll
  for (int o = LPN / 2; o > 0; o >>= 1) {  // xor over this node's LPN lanes
    lo ^= __shfl_xor_sync(0xffffffffu, lo, o);
    hi ^= __shfl_xor_sync(0xffffffffu, hi, o);
  }
  body = kind == TD_BODY_COMPUTE ? (((uint64_t)hi << 32) | lo) : 0ull;
  }
  const uint64_t tok = h ^ body;
  const uint64_t term = mix64(tok ^ key) >> 32;
#ifdef TD_CYCLE_PROBE
  PROBE(2, term);
#endif
  const int ns = d.nsucc;  // <= LPN (upload check)
  if (MULTI) {
    // before the first message to another GPU in this execution, every peer
    // must have started it (it re-armed its mailboxes in the previous one)
    if (!peers_ok && __any_sync(0xffffffffu, d.rmask != 0)) {
      if (!wait_peers_started(P)) return false;
      peers_ok = true;
    }
    if (hl < ns) {  // targets on another shard carry its tag (bits 28..31)
      const int32_t x = d.succ[hl];
      const int r = target_shard(x);
      if (r >= 0) red_add_sys_u64(&P.peer_mbox[r][slot(P, x & ID_MASK)], MSG_ONE + term);  // over NVLink
      else red_add_gpu_u64(&P.mbox[slot(P, x)], MSG_ONE + term);
    }
  } else if (hl < ns) {
    red_add_gpu_u64(&P.mbox[slot(P, d.succ[hl])], MSG_ONE + term);
  }
#ifdef TD_CYCLE_PROBE
  PROBE(3, 0);
#endif
  // consume the own ring slot before any ring add of this group: a later
  // node's successor 61..63 positions on shares an earlier node's slot
  lacc[li] = 0;
  __syncwarp();
  {
    // ring successors (never a node of the same group: equal levels): one
    // round per node that has any, lane hl of that node adding its delta #hl
    // (a node's deltas name distinct slots; nodes of the group may share one,
    // hence the rounds).  Replaces a 64-bit shared atomicAdd per delta, which
    // compiles to a CAS spin loop: ~750 cycles per pass of stencil_1d
    // 8192x100 at 4 nodes per pass (scripts/group_probe.py); a match_any +
    // segmented warp reduction was slower still (MATCH.ANY)
    // (rounds: nodes of one round feed distinct slots, coloured at upload)
    const int nrounds = (dp[0].dflags >> DF_RING_NROUNDS_SHIFT) & 7;  // (warp-uniform)
    if (nrounds) {
      const uint32_t dlt = hl < 4 ? (ldelta >> (8 * hl)) & 0xFFu : 0u;
      const int my_round = (d.dflags >> DF_RING_ROUND_SHIFT) & 3;
      for (int r = 0; r < nrounds; ++r) {
        if (my_round == r && dlt) lacc[(mypos + (int)dlt) & (LRING - 1)] += term;
        if (nrounds > 1) __syncwarp();
      }
    }
  }
  __syncwarp();
  if (nmsg) P.mbox[sv] = 0;
  TD_CHECK(v < P.n_nodes, "token of node id", v);
  if (v >= 0) P.token[v] = tok;  // (v < 0: a padding slot of the GROUP layout)
  if ((P.flags & TD_F_CHECKSUM) && d.col >= 0 && hl == 0) atomicXor(&P.colsum[d.col], (unsigned long long)tok);
#ifdef TD_CYCLE_PROBE
  if (tr && lane == 0 && dp[0].v >= 0) {
    PROBE(4, 0);
    probe[7] = globaltimer();
    for (int k = 0; k < TRACE_WORDS; ++k) P.trace[TRACE_WORDS * (int64_t)dp[0].v + k] = probe[k];
    if (probe_sink == 0x5EED5EED5EED5EEDull) P.stats[7] = 1;
  }
#endif
  return true;
}

// SM-balanced placement (P.place): the worker run by warp wc of this CTA, or
// -1 if the CTA found an unexpected CTA count on its SM (poisons).  Every
// thread of the CTA must call it (one __syncthreads).
__device__ int placed_worker(const Params& P, int wc) {
  // this CTA's arrival slot on its SM in this execution (the counter word
  // carries the execution number, so no reset is needed between launches).
  // (A banked counter taken with one returning add per CTA cut the placed
  // launch's fixed cost from ~23 to ~16 us, but made tree 4096x1000 with
  // compute_bound(256) bodies at 4096 workers 13-15 % slower on the same box,
  // reproducibly and for reasons not found: not kept,
  // profiles/r02_ab_place_banked_tree.log)
  __shared__ int s_row;
  if (threadIdx.x == 0) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (smid >= TD_MAX_SMID) smid = 0;  // (the host map then has no entry for it: refused below)
    const uint32_t ep = P.exec_no & 0xFFFFFFu;
    uint32_t old = P.sm_ctr[smid], nw, prev;
    for (;;) {
      nw = (old >> 8) == ep ? old + 1 : (ep << 8) | 1u;
      prev = atomicCAS(&P.sm_ctr[smid], old, nw);
      if (prev == old) break;
      old = prev;
    }
    const int slot = (int)(nw & 0xFFu) - 1;
    const int dense = P.sm_dense[smid];
    // exactly occ CTAs per SM (a full cooperative grid with occupancy
    // pinned by shared memory); anything else would map two warps to one
    // worker: refuse loudly
    s_row = (dense < 0 || slot >= P.occ) ? -1 : slot * P.n_sms + dense;
    if (s_row < 0) poison_set(P, 3u);
  }
  __syncthreads();
  const int row = s_row;
  if (row < 0) return -1;
  return ((row / P.n_sms) * WARPS_PER_CTA + wc) * P.n_sms + row % P.n_sms;
}

// Two instantiations per sharding mode: the lean Task Bench kernel (<= 64
// registers, 8 CTAs/SM, 4736 workers) and one with the config-5 tile body
// (<= 128 registers, 4 CTAs/SM); each with and without the diagnostics; plus
// PLAIN lean kernels (one-GPU and sharded).
template <bool MULTI, bool ST2D, bool DIAG, bool PLAIN = false, int GROUP = 0>
#ifndef TD_LEAN_MIN_BLOCKS
#define TD_LEAN_MIN_BLOCKS 8
#endif
__global__ void __launch_bounds__(128, ST2D ? 4 : TD_LEAN_MIN_BLOCKS) td_exec_kernel(const __grid_constant__ Params P) {
  constexpr int CHUNK = ST2D ? CHUNK_ST2D : CHUNK_LEAN;
  __shared__ __align__(128) Desc ring[WARPS_PER_CTA][STAGES][CHUNK];
  __shared__ __align__(8) uint64_t bar[WARPS_PER_CTA][STAGES];
  __shared__ uint64_t lacc_all[WARPS_PER_CTA][LRING];
  __shared__ __align__(8) uint64_t tile_bar[WARPS_PER_CTA];
  extern __shared__ __align__(128) uint8_t dyn_smem[];  // ST2D single-GPU: per-warp TMA halo boxes
  const int lane = threadIdx.x & 31;
  const int wc = threadIdx.x >> 5;
#ifdef TD_CYCLE_PROBE
  // (diagnostic build, TD_F_TRACE: earliest CTA entry / latest warp exit in
  // %globaltimer ns, stats[5] = ~min entry, stats[6] = max exit)
  if ((P.flags & TD_F_TRACE) && threadIdx.x == 0) atomicMax(&P.stats[5], ~(unsigned long long)globaltimer());
#endif
  zero_other_colsum(P);
  // TMA destinations must be 128 B aligned in the shared window
  const uint32_t dyn_off = ((smem_u32(dyn_smem) + 127u) & ~127u) - smem_u32(dyn_smem);
  uint32_t* box = reinterpret_cast<uint32_t*>(dyn_smem + dyn_off + (size_t)wc * TILE_SMEM);
  uint32_t tphase = 0;
  int prefetched = -1;  // ST2D: node whose TMA box load was already issued
  ColAcc ca;
  ulonglong2 lc = make_ulonglong2((uint64_t)(lane + 1) * G2, (uint64_t)(lane + 33) * G2);
  asm volatile("" : "+l"(lc.x), "+l"(lc.y));  // kept in registers, not recomputed per node
  // GROUP: (hl + 1) * G2, hl = this lane's index in its node's lane group
  uint64_t lcb = (uint64_t)(lane % (GROUP ? 32 / GROUP : 32) + 1) * G2;
  asm volatile("" : "+l"(lcb));
  int w = (int)(blockIdx.x * WARPS_PER_CTA + wc);
  if (P.place) {
    w = placed_worker(P, wc);
    if (w < 0) return;
  }

  if (MULTI && blockIdx.x == 0 && threadIdx.x < P.n_ranks && (int)threadIdx.x != P.my_rank) {
    // publish "this shard started execution exec_no" to every peer: every
    // mailbox of ours was re-armed by the previous (stream-ordered) execution
    fence_sys();
    st_release_sys(&P.peer_started[threadIdx.x][P.my_rank], P.exec_no);
  }
  if (P.n_shared) {
    // shared mailboxes are banked by execution parity: re-arm the other bank
    // (consumed by the previous, stream-ordered execution) for the next one
    const int64_t base = P.shared_base + (int64_t)((P.exec_no & 1u) ^ 1u) * P.n_shared * SHARE_SPLIT * SHARE_STRIDE;
    const int64_t words = P.n_shared * SHARE_SPLIT;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (int64_t)gridDim.x * blockDim.x)
      P.mbox[base + i * SHARE_STRIDE] = 0;
  }
#ifndef TD_NO_MBOX_PREFETCH
  // Bring the mailbox array into L2 at launch: one bulk L2 prefetch per CTA
  // over its slice.  After an L2 flush (or a long gap between replays) the
  // first message into every 32 B mailbox sector would otherwise wait for a
  // DRAM fill at the L2 before the consumer can observe it.
  if (threadIdx.x == 0) {
    // (at most the first 64 MiB: half of L2; a larger array would only evict itself)
    const int64_t total = min(P.mbox_words * 8, (int64_t)64 << 20) & ~(int64_t)15;
    const int64_t per = (((total + gridDim.x - 1) / gridDim.x) + 15) & ~(int64_t)15;
    const int64_t beg = per * blockIdx.x;
    if (beg < total) {
      const int64_t len = min(per, total - beg);
      // with an evict_last policy: the mailbox lines stay while descriptors
      // (evict_first) and tokens stream past (A/B, profiles/r02_ab_mbox_keep.log:
      // headline -1.4 %, nearest 4736 workers -4 %, METG points -0.6 %)
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
      asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(reinterpret_cast<const char*>(P.mbox) + beg),
                   "r"((uint32_t)len), "l"(pol) : "memory");
    }
  }
#endif
  if (w >= P.n_workers) return;
  if (ld_relaxed_gpu(P.poison)) return;  // an earlier queued execution failed (sticky poison)
  const int64_t beg = P.work_ptr[w];
  const int npos = (int)(P.work_ptr[w + 1] - beg);
  const int nchunks = (npos + CHUNK - 1) / CHUNK;
  uint64_t* lacc = lacc_all[wc];
  for (int i = lane; i < LRING; i += 32) lacc[i] = 0;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[wc][s], 1);
    if (ST2D) mbar_init(&tile_bar[wc], 1);
    mbar_fence_init();
  }
  __syncwarp();
  if (lane == 0)
    for (int c = 0; c < STAGES && c < nchunks; ++c) {
      const int cnt = min(CHUNK, npos - c * CHUNK);
      bulk_load(&ring[wc][c][0], P.desc + beg + (int64_t)c * CHUNK, cnt * (uint32_t)sizeof(Desc), &bar[wc][c]);
    }

  Acct a;
  int done_pos = 0;  // list positions executed (graph workers hold nodes only, relay warps relays only)
  // workers that never message another GPU skip the start handshake (and its
  // per-node check) altogether
  bool peers_ok = !MULTI || !P.wremote[w];
  int issued = min(STAGES, nchunks);
  int c = 0;
  for (; c < nchunks; ++c) {
    const int s = c % STAGES;
    mbar_wait(&bar[wc][s], (uint32_t)((c / STAGES) & 1));
    int cnt = min(CHUNK, npos - c * CHUNK);
    bool ok = true;
    if (GROUP) {  // (lists and chunks hold a multiple of GROUP nodes: upload check)
      for (int j = 0; j < cnt; j += GROUP) {
        if (MULTI) {
          // sharded graphs: a group with a successor row in the pool (halo
          // boundary producers) runs node by node on the sharded path, in
          // list order (equal levels: any order is a valid one); boundary
          // nodes with inline successors stay in the group pass (system-scope
          // polls and sends per node)
          bool one_by_one = false;
#pragma unroll
          for (int k = 0; k < (GROUP ? GROUP : 1); ++k) one_by_one |= ring[wc][s][j + k].nsucc == TD_OVF;
          if (one_by_one) {
            for (int k = 0; k < GROUP && ok; ++k) {
              const Desc& dd = ring[wc][s][j + k];
              if (dd.v < 0) continue;  // padding slot
              const bool okn = (dd.dflags & DF_MULTI)
                  ? execute_node<true, false, false, PLAIN>(P, dd, c * CHUNK + j + k, lacc, w, lane, peers_ok, a, box,
                                                         &tile_bar[wc], tphase, nullptr, prefetched, ca, lc)
                  : execute_node<false, false, false, PLAIN>(P, dd, c * CHUNK + j + k, lacc, w, lane, peers_ok, a, box,
                                                          &tile_bar[wc], tphase, nullptr, prefetched, ca, lc);
              ok = ok && okn;
            }
            if (!ok) break;
            continue;
          }
        }
        if (!execute_group<GROUP ? GROUP : 2, MULTI>(P, &ring[wc][s][j], c * CHUNK + j, lacc, lane, lcb, peers_ok)) {
          ok = false;
          break;
        }
        done_pos += GROUP;
      }
      __syncwarp();
      cnt = 0;  // (skip the one-node loop below)
    }
    for (int j = 0; j < cnt; ++j) {
      const Desc* next = (ST2D && j + 1 < cnt) ? &ring[wc][s][j + 1] : nullptr;
      const Desc& dd = ring[wc][s][j];
      bool done_ok;
      // in the sharded kernel, a node with no remote predecessor or successor
      // (most of them) takes the one-GPU path: no tag decoding, no handshake
      // checks, GPU-scope polls (sharded kernel on one shard measured +10 %
      // per node without this split)
      if (MULTI && (ST2D || (dd.dflags & DF_MULTI)))  // (the tile kernel keeps one path: register budget)
        done_ok = execute_node<true, ST2D, DIAG, PLAIN>(P, dd, c * CHUNK + j, lacc, w, lane, peers_ok, a, box, &tile_bar[wc],
                                           tphase, next, prefetched, ca, lc);
      else
        done_ok = execute_node<false, ST2D, DIAG, PLAIN, PLAIN && !MULTI>(P, dd, c * CHUNK + j, lacc, w, lane, peers_ok, a, box,
                                            &tile_bar[wc], tphase, next, prefetched, ca, lc);
      if (!done_ok) {
        ok = false;
        break;
      }
      done_pos += (!DIAG || dd.v >= 0);  // (padding slots are not nodes)
    }
    __syncwarp();
    if (!ok) break;
    if (lane == 0 && issued < nchunks) {
      const int cc = min(CHUNK, npos - issued * CHUNK);
      bulk_load(&ring[wc][s][0], P.desc + beg + (int64_t)issued * CHUNK, cc * (uint32_t)sizeof(Desc), &bar[wc][s]);
    }
    issued = min(issued + 1, nchunks);
  }
  colacc_flush(P, ca, lane);
#ifdef TD_CYCLE_PROBE
  if ((P.flags & TD_F_TRACE) && lane == 0) atomicMax(&P.stats[6], (unsigned long long)globaltimer());
#endif
  // aborted: drain bulk copies still in flight into this warp's ring / box
  for (int k = c + 1; k < issued; ++k) mbar_wait(&bar[wc][k % STAGES], (uint32_t)((k / STAGES) & 1));
  if (ST2D && prefetched >= 0) mbar_wait(&tile_bar[wc], tphase);
  if (diag<DIAG>(P, TD_F_STATS)) {
    const unsigned long long cr = warp_sum_u64(a.cross), lo = warp_sum_u64(a.local), xr = warp_sum_u64(a.xrank);
    if (lane == 0) {
      atomicAdd(&P.stats[0], (unsigned long long)(w < P.n_graph_workers ? done_pos : 0));
      atomicAdd(&P.stats[1], cr);
      atomicAdd(&P.stats[2], lo);
      atomicAdd(&P.stats[3], (unsigned long long)(npos > 0 && w < P.n_graph_workers));
      atomicAdd(&P.stats[4], xr);
    }
  }
}

// Arrival-order dispatch (TD_F_DYNAMIC): Alg. 1's "dispatch EXECUTE_OP the
// moment a counter hits zero" with per-SM ready queues
// instead of static per-worker lists.  A producer's message is a RETURNING
// atom.add on the consumer's mailbox word; the producer that delivers the
// last message re-arms that word and appends the consumer to the ready queue
// of its owner's SM: a ticket from q_tail, then ONE 16-byte store of the
// queue slot {tag | input sum, node id + 1} (tag = id mod 65535 + 1,
// so a half-visible slot is recognised and re-polled; tags run 1..65535).  The warps of an SM
// claim tickets from their queue's head in arrival order (each warp claims
// its next ticket while it executes the current node) and wait for the slot
// to be filled.  Every queue receives exactly its nodes once per execution,
// so a warp stops when the tickets run past its queue's size.  Progress: a
// ticket t waits only for the t-th enqueue into its queue; all warps are
// co-resident, and a warp never waits on a ticket while holding an
// unexecuted node.
__device__ __forceinline__ void ld_slot(const unsigned long long* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_slot(unsigned long long* p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
// 16-bit tag in 1 .. 65535 (0 marks an empty slot word)
__device__ __host__ __forceinline__ uint64_t slot_tag(uint64_t id1) { return (id1 - 1) % 0xFFFFull + 1; }

__global__ void __launch_bounds__(128, TD_LEAN_MIN_BLOCKS) td_dyn_kernel(const __grid_constant__ Params P) {
  const int lane = threadIdx.x & 31;
  const int wc = threadIdx.x >> 5;
  zero_other_colsum(P);
  const int w = placed_worker(P, wc);  // (dynamic launches are always placed)
  if (w < 0 || w >= P.n_workers) return;
  if (ld_relaxed_gpu(P.poison)) return;
  const int q = w % P.n_sms;  // this warp's SM = its queue
  const int64_t qb = P.q_base[q];
  const uint32_t cap = (uint32_t)(P.q_base[q + 1] - qb), nsrc = P.q_src[q];
  ulonglong2 lc = make_ulonglong2((uint64_t)(lane + 1) * G2, (uint64_t)(lane + 33) * G2);
  asm volatile("" : "+l"(lc.x), "+l"(lc.y));
  uint64_t executed = 0;
  uint32_t ahead = 0;
  if (lane == 0) ahead = atomicAdd(&P.q_head[q], 1u);
  for (;;) {
    const uint32_t t = __shfl_sync(0xffffffffu, ahead, 0);
    if (t >= cap) break;
    TD_CHECK(qb + t < P.q_base[P.n_sms], "queue slot", qb + t);
    unsigned long long* sl = &P.q_slots[2 * (qb + t)];
    uint64_t sw, id1;
    ld_slot(sl, sw, id1);
    uint64_t spins = 0;
    while (!id1 || (sw >> MSG_SHIFT) != slot_tag(id1)) {
      if ((++spins & 4095u) == 0) {
        if (ld_relaxed_gpu(P.poison) || *P.abort_flag) return;
        if (P.spin_limit && spins > P.spin_limit) {
          if (lane == 0) poison_set(P, 1u);
          return;
        }
      }
      ld_slot(sl, sw, id1);
    }
    if (lane == 0) ahead = atomicAdd(&P.q_head[q], 1u);  // the next ticket, claimed while this node runs
    const int v = (int)id1 - 1;
    __syncwarp();
    if (lane == 0 && t >= nsrc) st_slot(sl, 0, 0);  // re-arm the slot for the next execution
    const Desc& d = P.qdesc[v];
    const uint64_t h = mix64(mix64(P.seed ^ d.hid) ^ (sw & SUM_MASK));
    const uint64_t key = d.key;
    const int kind = d.kind;
    const uint32_t arg = d.arg;
    uint64_t tok;
    if (kind == TD_BODY_MEMORY) tok = h ^ memory_body(P, w, arg, h, lane);
    else tok = h ^ run_body<false>(kind, arg, h, lc);
    const uint64_t msg = MSG_ONE + (mix64(tok ^ key) >> 32);
    auto deliver = [&](int sx) {
      const uint64_t fin = (uint64_t)atomicAdd(&P.mbox[slot(P, sx)], (unsigned long long)msg) + msg;
      const uint32_t info = __ldg(&P.qinfo[sx]);
      if ((uint32_t)(fin >> MSG_SHIFT) == (info & 0xFFFFu)) {  // the last message: sx is ready
        P.mbox[slot(P, sx)] = 0;                               // re-armed by its last producer
        const uint32_t qs = info >> 16;
        const uint32_t pos = atomicAdd(&P.q_tail[qs], 1u);
        TD_CHECK(P.q_base[qs] + pos < P.q_base[qs + 1], "enqueue past the queue", pos);
        const uint64_t id = (uint64_t)sx + 1;
        st_slot(&P.q_slots[2 * (P.q_base[qs] + pos)], (slot_tag(id) << MSG_SHIFT) | (fin & SUM_MASK), id);
      }
    };
    const int ns = d.nsucc;
    if (ns != TD_OVF) {
      if (lane < ns) deliver(d.succ[lane]);
    } else {
      const int2* pool = P.succ_pool + d.succ[0];
      for (int k = 0; k < d.succ[1]; ++k) {
        const int2 iv = pool[k];
        for (int o = iv.x + lane; o <= iv.y; o += 32) deliver(o);
      }
    }
    P.token[v] = tok;
    if (lane == 0) {
      if ((P.flags & TD_F_CHECKSUM) && d.col >= 0) atomicXor(&P.colsum[d.col], (unsigned long long)tok);
      if (P.flags & TD_F_TALLY) atomicAdd(&P.tally[v], 1u);
    }
    ++executed;
  }
  if ((P.flags & TD_F_STATS) && lane == 0) atomicAdd(&P.stats[0], (unsigned long long)executed);
}

template <typename T>
cudaError_t upload(T** dst, const T* src, size_t count) {
  *dst = nullptr;
  if (count == 0) return cudaSuccess;
  cudaError_t e = cudaMalloc((void**)dst, count * sizeof(T));
  if (e != cudaSuccess) return e;
  return src ? cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice) : cudaMemset(*dst, 0, count * sizeof(T));
}

// %smid of every SM, one bit each: CTAs spread over the whole GPU while each
// holds its SM for spin_ns
__global__ void sm_probe_kernel(uint32_t* bits, uint64_t spin_ns) {
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0 && smid < TD_MAX_SMID) atomicOr(&bits[smid >> 5], 1u << (smid & 31));
  const uint64_t t0 = globaltimer();
  while (globaltimer() - t0 < spin_ns) {
  }
}

}  // namespace

// Dense index of every SM's %smid on `device` (for SM-balanced placement),
// probed once per device; *n_sms = 0 if the SM ids could not all be seen.
static cudaError_t sm_map_of(int device, const int16_t** dev_map, int* n_sms) {
  static const int16_t* maps[64];
  static int counts[64];
  static bool have[64];
  *dev_map = nullptr;
  *n_sms = 0;
  if (device < 0 || device >= 64) return cudaSuccess;
  if (have[device]) {
    *dev_map = maps[device];
    *n_sms = counts[device];
    return cudaSuccess;
  }
  int sms = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  uint32_t* bits = nullptr;
  int16_t* dmap = nullptr;
  if (e == cudaSuccess) e = cudaMalloc(&bits, TD_MAX_SMID / 8);
  if (e == cudaSuccess) e = cudaMemset(bits, 0, TD_MAX_SMID / 8);
  if (e == cudaSuccess) {
    sm_probe_kernel<<<sms * 8, 32>>>(bits, 50000);
    e = cudaGetLastError();
  }
  uint32_t hb[TD_MAX_SMID / 32] = {};
  if (e == cudaSuccess) e = cudaMemcpy(hb, bits, sizeof hb, cudaMemcpyDeviceToHost);
  int16_t hm[TD_MAX_SMID];
  int cnt = 0;
  for (int i = 0; i < TD_MAX_SMID; ++i) hm[i] = (hb[i >> 5] >> (i & 31)) & 1u ? (int16_t)cnt++ : (int16_t)-1;
  if (e == cudaSuccess) e = cudaMalloc(&dmap, sizeof hm);
  if (e == cudaSuccess) e = cudaMemcpy(dmap, hm, sizeof hm, cudaMemcpyHostToDevice);
  if (bits) cudaFree(bits);
  if (e != cudaSuccess) {
    if (dmap) cudaFree(dmap);
    return e;
  }
  maps[device] = dmap;
  counts[device] = cnt == sms ? sms : 0;
  have[device] = true;
  *dev_map = dmap;
  *n_sms = counts[device];
  return cudaSuccess;
}

// dynamic shared memory of an instantiation: per-warp TMA halo boxes of the
// tile-body kernels; for the lean kernels a pad that pins occupancy at
// exactly TD_LEAN_MIN_BLOCKS CTAs per SM (registers alone would admit 9 for
// the <= 56-register PLAIN kernels), so that a full cooperative grid puts the
// same number of CTAs on every SM (SM-balanced placement)
static size_t pad_bytes_for(const void* fn, int device) {
  int per_sm = 0, reserved = 0;
  cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, device);
  cudaFuncAttributes fa;
  memset(&fa, 0, sizeof fa);
  cudaFuncGetAttributes(&fa, fn);
  const int occ = TD_LEAN_MIN_BLOCKS;
  const int total = per_sm / occ - reserved;  // largest per-CTA footprint that still fits occ
  int pad = total - (int)fa.sharedSizeBytes;
  if (pad < 0 || per_sm / (total + reserved) != occ) pad = 0;
  return (size_t)(pad & ~127);
}
static size_t lean_pad_bytes(int device) {
  static int cached[64];
  static bool have[64];
  if (device >= 0 && device < 64 && have[device]) return (size_t)cached[device];
  const size_t pad = pad_bytes_for((const void*)td_exec_kernel<false, false, false, true>, device);
  if (device >= 0 && device < 64) { cached[device] = (int)pad; have[device] = true; }
  return pad;
}
static size_t dyn_pad_bytes(int device) {
  static int cached[64];
  static bool have[64];
  if (device >= 0 && device < 64 && have[device]) return (size_t)cached[device];
  const void* fn = (const void*)td_dyn_kernel;
  const size_t pad = pad_bytes_for(fn, device);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pad);
  cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (device >= 0 && device < 64) { cached[device] = (int)pad; have[device] = true; }
  return pad;
}
static size_t dyn_smem_for(bool, bool st2d, int device = 0) {
  return st2d ? (size_t)WARPS_PER_CTA * TILE_SMEM + 128 : lean_pad_bytes(device);
}

template <bool DIAG>
static const void* kernel_of(bool multi, bool st2d) {
  if (multi)
    return st2d ? (const void*)td_exec_kernel<true, true, DIAG> : (const void*)td_exec_kernel<true, false, DIAG>;
  return st2d ? (const void*)td_exec_kernel<false, true, DIAG> : (const void*)td_exec_kernel<false, false, DIAG>;
}
// diag: a launch with stats, tally or trace (the DIAG instantiation); plain:
// a graph (or shard) that qualifies for the PLAIN kernels (td_graph::plain)
static const void* kernel_for(bool multi, bool st2d, bool diag = false, bool plain = false, int group = 0) {
  if (group && plain && !st2d && !diag) {
    if (multi)
      return group == 4 ? (const void*)td_exec_kernel<true, false, false, true, 4>
                        : (const void*)td_exec_kernel<true, false, false, true, 2>;
    return group == 4 ? (const void*)td_exec_kernel<false, false, false, true, 4>
                      : (const void*)td_exec_kernel<false, false, false, true, 2>;
  }
  if (plain && !st2d && !diag)
    return multi ? (const void*)td_exec_kernel<true, false, false, true> : (const void*)td_exec_kernel<false, false, false, true>;
  return diag ? kernel_of<true>(multi, st2d) : kernel_of<false>(multi, st2d);
}

// co-resident CTAs of a (multi, st2d) kernel on `device`: the smaller of its
// plain and DIAG instantiations (either may run a given graph)
static cudaError_t resident_ctas_of(bool multi, bool st2d, int device, int64_t* out) {
  const size_t dyn = dyn_smem_for(multi, st2d, device);
  int sms = 0, lo = INT32_MAX;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  for (int dg = 0; dg < 5 && e == cudaSuccess; ++dg) {
    const void* fn = kernel_for(multi, st2d, dg == 1, dg >= 2, dg == 3 ? 2 : dg == 4 ? 4 : 0);
    int per_sm = 0;
    if (dyn) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * WARPS_PER_CTA, dyn);
    lo = per_sm < lo ? per_sm : lo;
  }
  *out = (int64_t)lo * sms;
  return e;
}

struct td_graph {
  int device;
  int64_t n;
  int32_t n_workers, n_cols, n_ranks, my_rank, n_ext_pre, n_ext_post;
  int64_t n_positions, n_succ_pool;
  int64_t n_slots, n_shared;
  // device arrays
  Desc* desc;
  int64_t* work_ptr;
  int2* succ_pool;
  int32_t* worker_of;
  uint8_t* wremote;
  bool has_col;  // the graph has checksum columns (they live in the descriptors)
  unsigned long long *colsum, *token, *stats;
  unsigned long long* mbox;
  uint32_t *tally, *poison, *started;
  unsigned long long* trace;
  // host-mapped flags
  uint32_t *h_ext_pre, *h_ext_post, *h_abort;  // (h_abort[1]: the kernel's poison mirror)
  unsigned long long* h_colsum;  // pinned mirror of colsum (bank 0 | poison word | bank 1), copied back behind each replay
  uint64_t cs_launches;          // CHECKSUM launches so far (bank of launch k: k & 1)
  bool colsum_on_host;           // h_colsum holds the last completed execution's checksums
  uint32_t shared_backoff_ns;    // TD_SHARED_BACKOFF, read once at upload
  bool force_multi;              // TD_FORCE_MULTI=1: run a 1-shard graph on the sharded kernel (diagnostics)
  int8_t place_env;              // SM-balanced placement: TD_PLACE=1 on, 0 off, unset -1 = policy (read at upload)
  int32_t n_graph_workers;  // n_workers minus the relay warps
  int64_t resident_ctas;   // co-resident CTAs of this graph's kernel instantiation (cached)
  uint32_t* sm_ctr;        // [TD_MAX_SMID] per-SM CTA arrival counters (placement)
  uint32_t max_mem_words;  // largest TD_BODY_MEMORY arg (0 = no memory_bound nodes)
  // arrival-order mode (TD_UPLOAD_DYNAMIC)
  bool dyn;
  int32_t dyn_sms;
  Desc* qdesc;
  uint32_t *qinfo, *q_src, *q_head, *q_tail;
  // combiners (one-GPU bundled groups, see COMB_MIN_REP)
  int4* comb;
  int32_t n_comb;
  int64_t comb_base;
  int64_t shared_base;
  unsigned long long *q_slots, *q_init;  // q_init: the slots with the sources only
  int64_t* q_base;
  unsigned long long* scratch;
  int64_t scratch_words;
  const void* place_fn;    // kernel last verified to run at exactly resident_ctas / n_sms CTAs per SM
  uint32_t *d_ext_pre, *d_ext_post, *d_abort;
  // peers
  unsigned long long* peer_mbox[TD_MAX_RANKS];
  uint32_t* peer_started[TD_MAX_RANKS];
  bool peer_opened[TD_MAX_RANKS];
  bool peer_direct[TD_MAX_RANKS];
  // execution state
  bool dirty;              // an aborted execution may have left mailboxes non-zero
  // config-5 tile body
  bool has_st2d;
  bool plain;  // runs the PLAIN kernel (see execute_node)
  int32_t group; // runs the PLAIN kernel in GROUP mode, K nodes per warp pass (see execute_group); 0 = off
  int32_t slot_shift;  // mailbox spacing (Params::slot_shift)
  int32_t st_nx, st_ny, st_tiles_x, st_tiles_y, st_ntiles;
  uint32_t* st_grid[2];
  uint32_t* st_peer_grid[TD_MAX_RANKS][2];
  uint8_t* st_tile_rank;
  CUtensorMap st_tmap[2];
  std::vector<uint8_t>* node_rank_host;
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

td_status td_device_info_get(int32_t device, uint32_t tpb, td_device_info* out) {
  if (!out) return set_err(TD_E_CONTRACT, "null out");
  if (tpb == 0) tpb = 32 * WARPS_PER_CTA;
  int count = 0;
  CUDA_TRY(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return set_err(TD_E_RESOURCE, "unknown device %d", device);
  CUDA_TRY(cudaSetDevice(device));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  int64_t ctas = 0, ctas_st2d = 0;
  CUDA_TRY(resident_ctas_of(false, false, device, &ctas));
  CUDA_TRY(resident_ctas_of(false, true, device, &ctas_st2d));
  memset(out, 0, sizeof *out);
  out->sm_count = prop.multiProcessorCount;
  out->l2_bytes = prop.l2CacheSize;
  out->max_workers = (int)ctas * (int)(tpb / 32);
  out->max_workers_st2d = (int)ctas_st2d * (int)(tpb / 32);
  out->cc_major = prop.major;
  out->cc_minor = prop.minor;
  strncpy(out->name, prop.name, sizeof out->name - 1);
  return TD_OK;
}

#ifdef TD_LAUNCH_PROFILE
// (diagnostic build: host time per phase of td_graph_launch, printed at destroy)
static inline uint64_t lp_now() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static uint64_t lp_acc[8], lp_n;
#define LP(k) do { const uint64_t t_ = lp_now(); lp_acc[k] += t_ - lp_t; lp_t = t_; } while (0)
#else
#define LP(k) do {} while (0)
#endif
td_status td_graph_destroy(td_graph* g) {
  if (!g) return TD_OK;
#ifdef TD_LAUNCH_PROFILE
  if (lp_n) {
    static const char* nm[] = {"setdevice", "checks+dirty", "memsets+params", "event_start", "coop_launch", "d2h_copies", "event_stop"};
    fprintf(stderr, "td_graph_launch host time per launch (%llu launches):", (unsigned long long)lp_n);
    for (int k = 0; k < 7; ++k) fprintf(stderr, " %s %.2f us", nm[k], lp_acc[k] / 1e3 / lp_n);
    fprintf(stderr, "\n");
  }
#endif
  cudaSetDevice(g->device);
  if (g->outstanding) cudaEventSynchronize(g->ev_stop);
  void* bufs[] = {g->desc, g->work_ptr, g->succ_pool, g->worker_of, g->wremote, g->sm_ctr, g->scratch,
                  g->qdesc, g->qinfo, g->q_slots, g->q_init, g->q_src, g->q_head, g->q_tail, g->q_base,
                  g->colsum, g->token, g->stats, g->mbox, g->tally, g->started, g->trace,
                  g->st_grid[0], g->st_grid[1], g->st_tile_rank, g->comb};
  for (void* b : bufs)
    if (b) cudaFree(b);
  for (int r = 0; r < TD_MAX_RANKS; ++r) {
    if (g->peer_opened[r]) {
      cudaIpcCloseMemHandle(g->peer_mbox[r]);
      if (g->st_peer_grid[r][0]) cudaIpcCloseMemHandle(g->st_peer_grid[r][0]);
      if (g->st_peer_grid[r][1]) cudaIpcCloseMemHandle(g->st_peer_grid[r][1]);
      cudaIpcCloseMemHandle(g->peer_started[r]);
    }
  }
  if (g->h_ext_pre) cudaFreeHost(g->h_ext_pre);
  if (g->h_ext_post) cudaFreeHost(g->h_ext_post);
  if (g->h_abort) cudaFreeHost(g->h_abort);
  if (g->h_colsum) cudaFreeHost(g->h_colsum);
  if (g->ev_start) cudaEventDestroy(g->ev_start);
  if (g->ev_stop) cudaEventDestroy(g->ev_stop);
  delete g->node_rank_host;
  delete g;
  return TD_OK;
}

namespace {

uint64_t mix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Intervals of a neighbour row, split at shard boundaries when sharded, with
// the owning shard encoded in bits 28..30 of lo (RANK_SHIFT).
void row_intervals(const int64_t* ptr, const int32_t* iv, int64_t v, const uint8_t* node_rank, const int32_t* rank_run,
                   std::vector<int2>& out) {
  const bool tag = rank_run != nullptr;  // rank_run[x]: last id of the run of equal shard starting at x
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
      const int32_t b = std::min(rank_run[a], hi);
      out.push_back(make_int2(a | ((int32_t)r << RANK_SHIFT), b));
      a = b + 1;
    }
  }
}
}  // namespace

// TD_UPLOAD_PROFILE=1: phase times of td_graph_upload on stderr
struct UploadTimer {
  bool on;
  struct timespec t;
  UploadTimer() : on(getenv("TD_UPLOAD_PROFILE") != nullptr) { clock_gettime(CLOCK_MONOTONIC, &t); }
  void mark(const char* what) {
    if (!on) return;
    struct timespec u;
    clock_gettime(CLOCK_MONOTONIC, &u);
    fprintf(stderr, "td_graph_upload %-16s %8.1f ms\n", what, (u.tv_sec - t.tv_sec) * 1e3 + (u.tv_nsec - t.tv_nsec) * 1e-6);
    t = u;
  }
};

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

  UploadTimer ut_;
  // ---- host-side validation ------------------------------------------------
  // (parallel; the first bad node is re-checked serially for the message)
  auto check_node = [&](int64_t v, bool report) -> td_status {
    int64_t d = 0;
    int32_t prev_hi = -2;
    for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k) {
      const int32_t lo = c->pred_iv[2 * k], hi = c->pred_iv[2 * k + 1];
      if (lo < 0 || hi >= n || hi < lo || lo <= prev_hi)
        return report ? set_err(TD_E_GRAPH, "dangling/unsorted predecessor interval of node %lld", (long long)v) : TD_E_GRAPH;
      prev_hi = hi;
      d += hi - lo + 1;
    }
    if (d >= (1ll << (64 - MSG_SHIFT)))  // mailbox count field (16 bits)
      return report ? set_err(TD_E_COMPILE, "node %lld has in-degree %lld > 65535 (mailbox limit)", (long long)v, (long long)d) : TD_E_COMPILE;
    if (c->ident && (c->ident[v] < 0 || c->ident[v] >= n))
      return report ? set_err(TD_E_GRAPH, "node %lld has identity out of range", (long long)v) : TD_E_GRAPH;
    if (c->kind[v] > TD_BODY_MEMORY)
      return report ? set_err(TD_E_COMPILE, "node %lld has unknown body kind %d", (long long)v, c->kind[v]) : TD_E_COMPILE;
    if (c->kind[v] == TD_BODY_MEMORY && c->arg[v] % 64)
      return report ? set_err(TD_E_COMPILE, "memory_bound node %lld: words (%u) must be a multiple of 64", (long long)v, c->arg[v]) : TD_E_COMPILE;
    if (c->kind[v] == TD_BODY_EXT_PRE && (int32_t)c->arg[v] >= c->n_ext_pre)
      return report ? set_err(TD_E_GRAPH, "ext precondition index out of range") : TD_E_GRAPH;
    if (c->kind[v] == TD_BODY_EXT_POST && (int32_t)c->arg[v] >= c->n_ext_post)
      return report ? set_err(TD_E_GRAPH, "ext postcondition index out of range") : TD_E_GRAPH;
    for (int64_t k = c->succ_ptr[v]; k < c->succ_ptr[v + 1]; ++k) {
      const int32_t lo = c->succ_iv[2 * k], hi = c->succ_iv[2 * k + 1];
      if (lo < 0 || hi >= n || hi < lo)
        return report ? set_err(TD_E_GRAPH, "dangling successor interval of node %lld", (long long)v) : TD_E_GRAPH;
    }
    return TD_OK;
  };
  int64_t first_bad = INT64_MAX;
  int not_topo = 0;  // some predecessor id is not smaller than its node's
#pragma omp parallel for schedule(static) reduction(min : first_bad) reduction(| : not_topo)
  for (int64_t v = 0; v < n; ++v) {
    if (check_node(v, false) != TD_OK && v < first_bad) first_bad = v;
    if (c->pred_ptr[v + 1] > c->pred_ptr[v] && c->pred_iv[2 * (c->pred_ptr[v + 1] - 1) + 1] >= v) not_topo = 1;
  }
  if (first_bad != INT64_MAX) return check_node(first_bad, true);
  const bool ids_topological = !not_topo;
  std::vector<int32_t> worker_of((size_t)(n > 0 ? n : 1), -1);
  const int64_t npos0 = c->n_workers > 0 ? c->work_ptr[c->n_workers] : 0;
  for (int32_t w = 0; w < c->n_workers; ++w) {
    for (int64_t i = c->work_ptr[w]; i < c->work_ptr[w + 1]; ++i) {
      const int32_t v = c->work[i];
      if (v < 0 || v >= n) return set_err(TD_E_COMPILE, "worker list references unknown node");
      if (worker_of[v] != -1) return set_err(TD_E_COMPILE, "node %d assigned to two workers", v);
      if (nr > 1 && c->node_rank[v] != c->my_rank) return set_err(TD_E_COMPILE, "worker list holds a node of another shard");
      worker_of[v] = w;
    }
  }
  if (nr == 1 && npos0 != n) return set_err(TD_E_COMPILE, "worker lists do not cover the graph");

  ut_.mark("validate");
  // ---- GROUP layout (one-GPU graphs that can run the PLAIN kernel) ----------
  // Levels (longest path from a source) decide GROUP mode (see g->group
  // below).  Worker lists in nondecreasing level order whose runs of equal
  // level are not all multiples of K (tree: the narrow first levels; ragged
  // lists) are padded with dummy slots (-1) to whole K-groups when that adds
  // at most 25 % of positions; dummies carry no node.  TD_NO_PAD=1 disables.
  const char* genv = getenv("TD_GROUP");
  const int kmax = getenv("TD_NO_PAIR") ? 0 : (genv ? atoi(genv) : 4);
  bool maybe_plain = kmax >= 2 && !getenv("TD_FORCE_MULTI") && !getenv("TD_NO_PLAIN") && !t_no_pad;
  for (int64_t v = 0; v < n && maybe_plain; ++v) {
    maybe_plain = c->kind[v] == TD_BODY_EMPTY || c->kind[v] == TD_BODY_COMPUTE;
    int64_t d = 0;
    for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k) d += c->pred_iv[2 * k + 1] - c->pred_iv[2 * k] + 1;
    maybe_plain = maybe_plain && d < SHARE_MIN_INDEG;  // (no bundled consumers)
    int64_t o = 0;  // (one GPU: no successor row in the pool, the PLAIN one-GPU kernel has no pool path)
    for (int64_t k = c->succ_ptr[v]; k < c->succ_ptr[v + 1]; ++k) o += c->succ_iv[2 * k + 1] - c->succ_iv[2 * k] + 1;
    maybe_plain = maybe_plain && (nr > 1 || o <= NSUCC_INLINE);
  }
  std::vector<int32_t> level;
  if (maybe_plain && ids_topological) {
    // ids are a topological order (every predecessor id is smaller): one
    // forward pass over the predecessor intervals
    level.assign((size_t)n, 0);
    for (int64_t v = 0; v < n; ++v) {
      int32_t lv = 0;
      for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k)
        for (int32_t u = c->pred_iv[2 * k]; u <= c->pred_iv[2 * k + 1]; ++u) lv = std::max(lv, level[u] + 1);
      level[v] = lv;
    }
  } else if (maybe_plain) {
    std::vector<int32_t> indeg((size_t)n, 0), frontier;
    level.assign((size_t)n, 0);
    for (int64_t v = 0; v < n; ++v) {
      for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k)
        indeg[v] += c->pred_iv[2 * k + 1] - c->pred_iv[2 * k] + 1;
      if (!indeg[v]) frontier.push_back((int32_t)v);
    }
    for (size_t f = 0; f < frontier.size(); ++f) {  // Kahn: the frontier grows as nodes are released
      const int32_t u = frontier[f];
      for (int64_t k = c->succ_ptr[u]; k < c->succ_ptr[u + 1]; ++k)
        for (int32_t x = c->succ_iv[2 * k]; x <= c->succ_iv[2 * k + 1]; ++x) {
          level[x] = std::max(level[x], level[u] + 1);
          if (--indeg[x] == 0) frontier.push_back(x);
        }
    }
  }
  // the largest K whose groups the lists already form exactly; else padding
  auto groups_exactly = [&](int K) {
    for (int32_t w = 0; w < c->n_workers; ++w) {
      if ((c->work_ptr[w + 1] - c->work_ptr[w]) % K) return false;
      for (int64_t i = c->work_ptr[w]; i + 1 < c->work_ptr[w + 1]; ++i) {
        const int32_t a = c->work[i], b = c->work[i + 1];
        if (((i + 1 - c->work_ptr[w]) % K == 0) ? level[a] > level[b] : level[a] != level[b]) return false;
      }
    }
    return true;
  };
  int exact_k = 0, pad_k = 0;
  std::vector<int32_t> pwork;
  std::vector<int64_t> pptr;
  if (maybe_plain) {
    for (int K = kmax >= 4 ? 4 : 2; K >= 2 && !exact_k; K /= 2)
      if (groups_exactly(K)) exact_k = K;
    bool sorted_lv = true;
    for (int32_t w = 0; w < c->n_workers && sorted_lv; ++w)
      for (int64_t i = c->work_ptr[w]; i + 1 < c->work_ptr[w + 1] && sorted_lv; ++i)
        sorted_lv = level[c->work[i]] <= level[c->work[i + 1]];
    const char* nopad = getenv("TD_NO_PAD");
    if (!exact_k && sorted_lv && !(nopad && nopad[0] == '1')) {
      for (int K = kmax >= 4 ? 4 : 2; K >= 2 && !pad_k; K /= 2) {
        int64_t total = 0;
        for (int32_t w = 0; w < c->n_workers; ++w)
          for (int64_t i = c->work_ptr[w]; i < c->work_ptr[w + 1];) {
            int64_t j = i;
            while (j < c->work_ptr[w + 1] && level[c->work[j]] == level[c->work[i]]) ++j;
            total += (j - i + K - 1) / K * K;
            i = j;
          }
        if (total * 4 <= npos0 * 5) {
          pad_k = K;
          pptr.assign(1, 0);
          pwork.reserve((size_t)total);
          for (int32_t w = 0; w < c->n_workers; ++w) {
            for (int64_t i = c->work_ptr[w]; i < c->work_ptr[w + 1];) {
              int64_t j = i;
              while (j < c->work_ptr[w + 1] && level[c->work[j]] == level[c->work[i]]) ++j;
              for (int64_t q = i; q < j; ++q) pwork.push_back(c->work[q]);
              for (int64_t q = j - i; q % K; ++q) pwork.push_back(-1);
              i = j;
            }
            pptr.push_back((int64_t)pwork.size());
          }
        }
      }
    }
  }
  const int32_t* work = pad_k ? pwork.data() : c->work;           // positions -> node (-1 = dummy)
  const int64_t* work_ptr = pad_k ? pptr.data() : c->work_ptr;
  const int64_t npos = pad_k ? (int64_t)pwork.size() : npos0;

  ut_.mark("levels+layout");
  // ---- worker programs (descriptors) ----------------------------------------
  // position of every node inside its worker's list (for same-worker deltas)
  std::vector<int32_t> pos_of((size_t)(n > 0 ? n : 1), -1);
  for (int32_t w = 0; w < c->n_workers; ++w)
    for (int64_t i = work_ptr[w]; i < work_ptr[w + 1]; ++i)
      if (work[i] >= 0) pos_of[work[i]] = (int32_t)(i - work_ptr[w]);
  // Same-worker delivery through the shared-memory ring is used only for a
  // consumer ALL of whose in-edges qualify (same worker, < LRING list
  // positions back): then it never waits on L2 at all.  A consumer that also
  // waits for remote messages gains nothing from partial local delivery.
  const char* lenv = getenv("TD_LOCAL_RING");
  const bool use_local = !(lenv && lenv[0] == '0');
  std::vector<uint8_t> local_ok((size_t)(n > 0 ? n : 1), 0);
  if (use_local) {
#pragma omp parallel for schedule(static)
    for (int64_t s2 = 0; s2 < n; ++s2) {
      const int32_t ws = worker_of[s2];
      if (ws < 0 || c->pred_ptr[s2] == c->pred_ptr[s2 + 1]) continue;
      // (>= LRING predecessors cannot all sit within LRING - 1 positions of one list)
      int64_t deg = 0;
      for (int64_t k = c->pred_ptr[s2]; k < c->pred_ptr[s2 + 1]; ++k) deg += c->pred_iv[2 * k + 1] - c->pred_iv[2 * k] + 1;
      if (deg >= LRING) continue;
      bool ok = true;
      for (int64_t k = c->pred_ptr[s2]; ok && k < c->pred_ptr[s2 + 1]; ++k)
        for (int32_t u = c->pred_iv[2 * k]; ok && u <= c->pred_iv[2 * k + 1]; ++u) {
          const int32_t dlt = pos_of[s2] - pos_of[u];
          ok = worker_of[u] == ws && dlt > 0 && dlt < LRING;
        }
      local_ok[s2] = ok;
    }
    // a producer carries at most 4 local deltas: demote consumers beyond that.
    // Successor intervals are walked by runs of equal local_ok as computed
    // before any demotion (lrun, local0), so a dense row (all_to_all: 8192
    // successors) costs its runs, not its ids; ids inside runs that were
    // ring-fed are visited one by one against the current flags
    const std::vector<uint8_t> local0 = local_ok;
    std::vector<int32_t> lrun((size_t)(n > 0 ? n : 1));
    for (int64_t x = n - 1; x >= 0; --x)
      lrun[x] = (x + 1 < n && local0[x + 1] == local0[x]) ? lrun[x + 1] : (int32_t)x;
    for (int64_t i = 0; i < npos; ++i) {
      const int32_t v = work[i];
      if (v < 0) continue;  // GROUP padding slot
      int cnt = 0;
      for (int64_t k = c->succ_ptr[v]; k < c->succ_ptr[v + 1]; ++k)
        for (int32_t s2 = c->succ_iv[2 * k], hi = c->succ_iv[2 * k + 1]; s2 <= hi;) {
          const int32_t e = std::min(lrun[s2], hi);
          if (local0[s2])
            for (int32_t x = s2; x <= e; ++x)
              if (local_ok[x] && ++cnt > 4) local_ok[x] = 0;
          s2 = e + 1;
        }
    }
    // GROUP layouts: a pass that waits on L2 anyway (one of its nodes has
    // remote inputs) gains nothing from ring-fed nodes, whose producers'
    // ring adds cost the pass rounds of shared-memory adds (up to ~550
    // cycles, scripts/group_probe.py): demote them to mailboxes, so that only
    // passes made entirely of ring-fed nodes use the ring.  TD_MIXED_RING=1
    // keeps them.
    const int gk = exact_k ? exact_k : pad_k;
    const char* menv = getenv("TD_MIXED_RING");
    if (gk && !(menv && menv[0] == '1')) {
#pragma omp parallel for schedule(static)
      for (int32_t w = 0; w < c->n_workers; ++w)
        for (int64_t i = work_ptr[w]; i + gk <= work_ptr[w + 1]; i += gk) {
          bool l2 = false, ring = false;
          for (int k = 0; k < gk; ++k) {
            const int32_t v = work[i + k];
            if (v < 0) continue;
            if (local_ok[v]) ring = true;
            else if (c->pred_ptr[v] != c->pred_ptr[v + 1]) l2 = true;
          }
          if (l2 && ring)
            for (int k = 0; k < gk; ++k)
              if (work[i + k] >= 0) local_ok[work[i + k]] = 0;
        }
    }
  }
  ut_.mark("ring");
  // Edge bundling: consumers with IDENTICAL large
  // predecessor lists (all_to_all: a whole timestep) share mailbox replicas.
  // Every producer sends one message per replica instead of one per consumer;
  // a replica serves up to SHARE_FANOUT consumers of one shard.  Computed
  // from the global graph, so every shard derives the same slots.
  const char* benv = getenv("TD_BUNDLE");
  const bool use_bundle = !(benv && benv[0] == '0');
  const char* fenv = getenv("TD_SHARE_FANOUT");
  const size_t fanout = fenv && atoi(fenv) > 0 ? (size_t)atoi(fenv) : (size_t)SHARE_FANOUT;
  std::vector<int32_t> wslot_of((size_t)(n > 0 ? n : 1), -1);  // replica index per consumer
  std::vector<int32_t> group_of((size_t)(n > 0 ? n : 1), -1);
  std::vector<int32_t> group_base, group_nrep;                 // replica range per group
  std::vector<std::vector<int2>> group_rep_iv;                 // replica intervals tagged by shard
  std::vector<int32_t> rep_node;                               // group -> representative node
  int64_t n_shared = 0;
  if (use_bundle) {
    std::unordered_map<uint64_t, std::vector<int32_t>> reps;   // hash -> representative nodes of groups
    std::vector<std::vector<int32_t>> members;
    auto same_preds = [&](int64_t x, int64_t y) {
      const int64_t nx_ = c->pred_ptr[x + 1] - c->pred_ptr[x];
      if (nx_ != c->pred_ptr[y + 1] - c->pred_ptr[y]) return false;
      return memcmp(c->pred_iv + 2 * c->pred_ptr[x], c->pred_iv + 2 * c->pred_ptr[y], sizeof(int32_t) * 2 * nx_) == 0;
    };
    // candidates (in-degree >= SHARE_MIN_INDEG) found in parallel; grouping serial
    std::vector<uint8_t> cand_v((size_t)(n > 0 ? n : 1), 0);
#pragma omp parallel for schedule(static)
    for (int64_t v = 0; v < n; ++v) {
      int64_t d = 0;
      for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k) d += c->pred_iv[2 * k + 1] - c->pred_iv[2 * k] + 1;
      cand_v[v] = d >= SHARE_MIN_INDEG;
    }
    for (int64_t v = 0; v < n; ++v) {
      if (!cand_v[v]) continue;
      uint64_t h = 1469598103934665603ull;
      for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k) {
        h = (h ^ (uint32_t)c->pred_iv[2 * k]) * 1099511628211ull;
        h = (h ^ (uint32_t)c->pred_iv[2 * k + 1]) * 1099511628211ull;
      }
      auto& cand = reps[h];
      int32_t gid = -1;
      for (int32_t gg : cand)
        if (same_preds(rep_node[gg], v)) { gid = gg; break; }
      if (gid < 0) {
        gid = (int32_t)rep_node.size();
        rep_node.push_back((int32_t)v);
        members.emplace_back();
        cand.push_back(gid);
      }
      members[gid].push_back((int32_t)v);
      group_of[v] = gid;
    }
    for (size_t gid = 0; gid < members.size(); ++gid) {
      auto& m = members[gid];
      if (m.size() < 2) {  // nothing to share
        for (int32_t v : m) group_of[v] = -1;
        group_base.push_back(-1);
        group_nrep.push_back(0);
        group_rep_iv.emplace_back();
        continue;
      }
      // stable order by (shard, id); chunk per shard into replicas
      std::stable_sort(m.begin(), m.end(), [&](int32_t x, int32_t y) {
        const int rx = nr > 1 ? c->node_rank[x] : 0, ry = nr > 1 ? c->node_rank[y] : 0;
        return rx != ry ? rx < ry : x < y;
      });
      const int32_t base = (int32_t)n_shared;
      std::vector<int2> ivs;
      int32_t rep = base;
      size_t i0 = 0;
      while (i0 < m.size()) {
        const int r = nr > 1 ? c->node_rank[m[i0]] : 0;
        size_t i1 = i0;
        while (i1 < m.size() && (nr > 1 ? c->node_rank[m[i1]] : 0) == r) ++i1;
        const int32_t first = rep;
        for (size_t j = i0; j < i1; j += fanout) {
          for (size_t q = j; q < i1 && q < j + fanout; ++q) wslot_of[m[q]] = rep;
          ++rep;
        }
        const int32_t tag = nr > 1 ? (r << RANK_SHIFT) : 0;
        ivs.push_back(make_int2(((int32_t)n + first) | tag, (int32_t)n + rep - 1));
        i0 = i1;
      }
      group_base.push_back(base);
      group_nrep.push_back(rep - base);
      group_rep_iv.push_back(ivs);
      n_shared = rep;
    }
  }
  bool has_st2d = false;
  for (int64_t v = 0; v < n && !has_st2d; ++v) has_st2d = c->kind[v] == TD_BODY_STENCIL2D;
  // Cross-shard aggregation: a bundled group with replicas on
  // other shards gets, on this shard, one relay warp.  This shard's k
  // producers of the group send to a local relay replica instead of to every
  // remote replica; the relay forwards one (k << 48) + sum add per remote
  // replica.  Remote atomics per group and step drop from k * replicas to
  // replicas, for one extra on-GPU hop.  Relay replicas are numbered per
  // (group, shard) identically on every shard (the bank offsets depend on
  // n_shared); only the producing shard uses its own.
  std::vector<int32_t> relay_slot(rep_node.size(), -1), relay_k(rep_node.size(), 0);
  int32_t n_relays = 0;
  const char* renv = getenv("TD_RELAY");
  if (nr > 1 && !(renv && renv[0] == '0')) {
    int64_t next = n_shared;
    for (size_t gg = 0; gg < rep_node.size(); ++gg) {
      if (!group_nrep[gg]) continue;
      const int32_t mine = (int32_t)(next + c->my_rank);
      next += nr;
      bool remote = false;
      for (auto& iv : group_rep_iv[gg]) remote |= ((iv.x >> RANK_SHIFT) & 7) != c->my_rank;
      if (!remote) continue;
      const int32_t rv = rep_node[gg];
      int32_t k = 0;
      for (int64_t q = c->pred_ptr[rv]; q < c->pred_ptr[rv + 1]; ++q)
        for (int32_t u = c->pred_iv[2 * q]; u <= c->pred_iv[2 * q + 1]; ++u) k += c->node_rank[u] == c->my_rank;
      if (k < 2) continue;  // nothing to aggregate
      relay_slot[gg] = mine;
      relay_k[gg] = k;
      ++n_relays;
    }
    n_shared = next;
    int64_t ctas = 0;  // one warp per relay: keep the whole program co-resident
    CUDA_TRY(resident_ctas_of(true, has_st2d, device, &ctas));
    if ((int64_t)c->n_workers + n_relays > ctas * WARPS_PER_CTA) {
      std::fill(relay_slot.begin(), relay_slot.end(), -1);
      n_relays = 0;
    }
  }
  if (n + n_shared >= (1ll << RANK_SHIFT) && nr > 1)
    return set_err(TD_E_GRAPH, "sharded graph plus shared mailboxes exceed 2^28 slots");
  // Combiners (one GPU; see COMB_MIN_REP): group gg's producer u sends to
  // combiner comb_first[gg] + u % comb_n[gg], ids n + n_shared + c.
  // TD_COMBINE=0 disables them, =1 uses them for every group with >= 2
  // replicas regardless of producers per worker.
  std::vector<int32_t> comb_first(rep_node.size(), -1), comb_n(rep_node.size(), 0);
  std::vector<int4> comb_info;
  {
    const char* cenv = getenv("TD_COMBINE");
    const int min_rep = cenv && cenv[0] == '1' ? 2 : COMB_MIN_REP;
    if (nr == 1 && !(cenv && cenv[0] == '0')) {
      for (size_t gg = 0; gg < rep_node.size(); ++gg) {
        if (group_nrep[gg] < min_rep) continue;
        const int32_t rv = rep_node[gg];
        if (!(cenv && cenv[0] == '1')) {  // producers per worker
          std::unordered_map<int32_t, int32_t> per;
          int32_t most = 0;
          for (int64_t q = c->pred_ptr[rv]; q < c->pred_ptr[rv + 1] && most <= COMB_MAX_PER_WORKER; ++q)
            for (int32_t u = c->pred_iv[2 * q]; u <= c->pred_iv[2 * q + 1]; ++u) most = std::max(most, ++per[worker_of[u]]);
          if (most > COMB_MAX_PER_WORKER) continue;
        }
        int64_t k = 0;
        for (int64_t q = c->pred_ptr[rv]; q < c->pred_ptr[rv + 1]; ++q) k += c->pred_iv[2 * q + 1] - c->pred_iv[2 * q] + 1;
        const int32_t pc = (int32_t)std::max<int64_t>(1, (k + COMB_PER - 1) / COMB_PER);
        comb_first[gg] = (int32_t)comb_info.size();
        comb_n[gg] = pc;
        const size_t c0 = comb_info.size();
        comb_info.resize(c0 + (size_t)pc, make_int4(0, group_base[gg], group_nrep[gg], 0));
        for (int64_t q = c->pred_ptr[rv]; q < c->pred_ptr[rv + 1]; ++q)
          for (int32_t u = c->pred_iv[2 * q]; u <= c->pred_iv[2 * q + 1]; ++u) ++comb_info[c0 + (size_t)(u % pc)].x;
      }
    }
    if (n + n_shared + (int64_t)comb_info.size() >= INT32_MAX)
      return set_err(TD_E_GRAPH, "graph plus shared mailboxes exceed 2^31 message targets");
  }

  DescVec desc((size_t)npos);  // (every position is written below)
  std::vector<int2> spool, tmp, rem;
  std::vector<int32_t> hit_groups;
  // message targets of one descriptor: explicit ids (<= 6) or pool intervals
  auto encode_succs_into = [&](Desc& d, const std::vector<int2>& targets, std::vector<int2>& pool) {
    uint32_t rmask = 0;
    if (nr > 1)
      for (auto& iv : targets) {
        const int r = (iv.x >> RANK_SHIFT) & 7;
        if (r != c->my_rank) rmask |= 1u << r;
      }
    d.rmask = (uint8_t)rmask;
    int64_t nt = 0;
    for (auto& iv : targets) nt += (int64_t)iv.y - (nr > 1 ? (iv.x & ID_MASK) : iv.x) + 1;
    // device encoding: local targets untagged, shard r's targets tagged r + 1
    auto dev_tag = [&](int32_t x) -> int32_t {
      if (nr <= 1) return 0;
      const int r = (x >> RANK_SHIFT) & 7;
      return r == c->my_rank ? 0 : (int32_t)((uint32_t)(r + 1) << RANK_SHIFT);
    };
    if (nt <= NSUCC_INLINE) {
      int k = 0;
      for (auto& iv : targets) {
        const int32_t lo = nr > 1 ? (iv.x & ID_MASK) : iv.x;
        const int32_t tag = dev_tag(iv.x);
        for (int32_t s3 = lo; s3 <= iv.y; ++s3) d.succ[k++] = s3 | tag;
      }
      d.nsucc = (uint8_t)k;
    } else {
      d.nsucc = TD_OVF;
      d.succ[0] = (int32_t)pool.size();  // (offset in `pool`; rebased when pools are merged)
      d.succ[1] = (int32_t)targets.size();
      for (auto& iv : targets)
        pool.push_back(make_int2((nr > 1 ? (iv.x & ID_MASK) : iv.x) | dev_tag(iv.x), iv.y));
    }
    if (rmask || (d.dflags & DF_REMOTE_PRED) || d.kind == KIND_RELAY) d.dflags |= DF_MULTI;
  };
  auto encode_succs = [&](Desc& d, const std::vector<int2>& targets) { encode_succs_into(d, targets, spool); };
  ut_.mark("bundling+relays");
  // runs of equal (local_ok, group_of) and of equal shard, for walking
  // successor / predecessor intervals run by run instead of id by id
  std::vector<int32_t> crun((size_t)(n > 0 ? n : 1)), rrun;
  for (int64_t x = n - 1; x >= 0; --x)
    crun[x] = (x + 1 < n && local_ok[x + 1] == local_ok[x] && group_of[x + 1] == group_of[x]) ? crun[x + 1] : (int32_t)x;
  if (nr > 1) {
    rrun.resize((size_t)(n > 0 ? n : 1));
    for (int64_t x = n - 1; x >= 0; --x)
      rrun[x] = (x + 1 < n && c->node_rank[x + 1] == c->node_rank[x]) ? rrun[x + 1] : (int32_t)x;
  }
  // (parallel over positions: OpenMP threads build disjoint descriptors with
  // their own scratch vectors; successor-pool rows go to per-thread pools,
  // merged in position order afterwards, so the layout is deterministic)
  int nthreads = 1;
#ifdef _OPENMP
  nthreads = std::max(1, omp_get_max_threads());
#endif
  std::vector<std::vector<int2>> tpool((size_t)nthreads);
  std::vector<int64_t> tfirst((size_t)nthreads, npos);  // first position each thread handled
  int32_t ring_overflow = -1;
#pragma omp parallel num_threads(nthreads)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    std::vector<int2> tmp, rem;
    std::vector<int32_t> hit_groups;
    std::vector<int2>& mypool = tpool[(size_t)tid];
#pragma omp for schedule(static)
  for (int64_t i = 0; i < npos; ++i) {
    if (tfirst[(size_t)tid] == npos) tfirst[(size_t)tid] = i;
    const int32_t v = work[i];
    Desc& d = desc[i];
    memset(&d, 0, sizeof d);
    if (v < 0) {  // GROUP padding slot: no node, no inputs, no messages
      d.v = -1;
      d.wslot = -1;
      d.col = -1;
      continue;
    }
    d.v = v;
    d.kind = c->kind[v];
    d.arg = c->arg[v];
    uint32_t indeg = 0;
    for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k)
      indeg += (uint32_t)(c->pred_iv[2 * k + 1] - c->pred_iv[2 * k] + 1);
    d.nmsg = local_ok[v] ? 0 : indeg;  // ring-fed consumers never wait on L2
    if (nr > 1)
      for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1] && !(d.dflags & DF_REMOTE_PRED); ++k)
        for (int32_t u = c->pred_iv[2 * k], hi = c->pred_iv[2 * k + 1]; u <= hi; u = std::min(rrun[u], hi) + 1)
          if (c->node_rank[u] != c->my_rank) { d.dflags |= DF_REMOTE_PRED; break; }
    const int32_t idv = c->ident ? c->ident[v] : v;  // replicas hash as the node they replicate
    d.hid = mix64_host((uint64_t)idv + G1);
    d.col = c->col ? c->col[v] : -1;
    d.key = mix64_host((uint64_t)idv + G3);
    d.wslot = wslot_of[v];
    row_intervals(c->succ_ptr, c->succ_iv, v, c->node_rank, nr > 1 ? rrun.data() : nullptr, tmp);
    // same-worker successors within the local ring go through shared memory;
    // members of bundled groups are replaced by their group's replicas
    uint32_t ld = 0;
    int nld = 0;
    rem.clear();
    hit_groups.clear();
    for (auto& iv : tmp) {
      const int32_t lo = nr > 1 ? (iv.x & ID_MASK) : iv.x;
      const int32_t tag = nr > 1 ? (iv.x & ~ID_MASK) : 0;
      int32_t a = lo;
      for (int32_t s2 = lo; s2 <= iv.y;) {  // by runs of equal (local_ok, group_of)
        const int32_t e = std::min(crun[s2], iv.y);
        const bool loc = local_ok[s2] != 0;
        const int32_t gg = group_of[s2];
        if (loc || gg >= 0) {
          if (s2 > a) rem.push_back(make_int2(a | tag, s2 - 1));
          if (loc)
            for (int32_t x = s2; x <= e; ++x) {
              if (nld >= 4) {
#pragma omp critical(td_ring_overflow)
                ring_overflow = v;
                break;
              }
              ld |= (uint32_t)(pos_of[x] - pos_of[v]) << (8 * nld++);
            }
          else if (std::find(hit_groups.begin(), hit_groups.end(), gg) == hit_groups.end()) hit_groups.push_back(gg);
          a = e + 1;
        }
        s2 = e + 1;
      }
      if (a <= iv.y) rem.push_back(make_int2(a | tag, iv.y));
    }
    for (int32_t gg : hit_groups) {
      if (comb_first[gg] >= 0) {  // one message into this producer's combiner
        const int32_t cid = (int32_t)(n + n_shared) + comb_first[gg] + v % comb_n[gg];
        rem.push_back(make_int2(cid, cid));
      } else if (relay_slot[gg] >= 0) {  // local replicas directly, remote ones through this shard's relay
        for (auto& iv : group_rep_iv[gg])
          if (((iv.x >> RANK_SHIFT) & 7) == c->my_rank) rem.push_back(iv);
        const int32_t rs = (int32_t)n + relay_slot[gg];
        rem.push_back(make_int2(rs | (c->my_rank << RANK_SHIFT), rs));
      } else {
        for (auto& iv : group_rep_iv[gg]) rem.push_back(iv);
      }
    }
    d.ldelta = ld;
    encode_succs_into(d, rem, mypool);
  }
  }  // omp parallel
  if (ring_overflow >= 0) return set_err(TD_E_COMPILE, "internal: more than 4 ring successors of node %d", ring_overflow);
  {  // merge the per-thread pools (static schedule: thread t's positions precede thread t+1's)
    std::vector<int> order((size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) order[(size_t)t] = t;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return tfirst[(size_t)x] < tfirst[(size_t)y]; });
    std::vector<int64_t> base((size_t)nthreads, 0);
    for (int t : order) {
      base[(size_t)t] = (int64_t)spool.size();
      spool.insert(spool.end(), tpool[(size_t)t].begin(), tpool[(size_t)t].end());
    }
    if (spool.size() > (size_t)INT32_MAX) return set_err(TD_E_GRAPH, "successor pool exceeds 2^31 intervals");
    for (int t = 0; t < nthreads; ++t) {
      if (tpool[(size_t)t].empty() || tfirst[(size_t)t] == npos) continue;
      const int64_t lo = tfirst[(size_t)t];
      int64_t hi = npos;  // positions of thread t: [lo, next thread's first)
      for (int u = 0; u < nthreads; ++u)
        if (tfirst[(size_t)u] > lo && tfirst[(size_t)u] < hi) hi = tfirst[(size_t)u];
      for (int64_t i = lo; i < hi; ++i)
        if (desc[(size_t)i].v >= 0 && desc[(size_t)i].nsucc == TD_OVF) desc[(size_t)i].succ[0] += (int32_t)base[(size_t)t];
    }
  }
  ut_.mark("descriptors");
  // relay warps: workers n_workers.. (one descriptor each)
  std::vector<int64_t> wptr(1, 0);
  if (c->n_workers > 0) wptr.assign(work_ptr, work_ptr + c->n_workers + 1);
  for (size_t gg = 0; gg < relay_slot.size(); ++gg) {
    if (relay_slot[gg] < 0) continue;
    Desc d;
    memset(&d, 0, sizeof d);
    d.v = c->my_rank;  // spreads relays of different shards over replica sub-words
    d.kind = KIND_RELAY;
    d.nmsg = (uint32_t)relay_k[gg];
    d.wslot = relay_slot[gg];
    rem.clear();
    for (auto& iv : group_rep_iv[gg])
      if (((iv.x >> RANK_SHIFT) & 7) != c->my_rank) rem.push_back(iv);
    encode_succs(d, rem);
    desc.push_back(d);
    wptr.push_back(wptr.back() + 1);
  }

  // ---- arrival-order mode (TD_UPLOAD_DYNAMIC): node-indexed programs, one
  // ready queue per SM (node v's queue = its static owner's SM under the
  // SM-balanced placement, worker % n_sms), sources at each queue's head
  const bool want_dyn = (c->options & TD_UPLOAD_DYNAMIC) != 0;
  DescVec qdesc;
  std::vector<uint32_t> qinfo, qsrc;
  std::vector<unsigned long long> qentries;
  std::vector<int64_t> qbase;
  int dyn_sms = 0;
  if (want_dyn) {
    if (nr > 1) return set_err(TD_E_COMPILE, "arrival-order mode is one-GPU only");
    for (int64_t v = 0; v < n; ++v) {
      const int k = c->kind[v];
      if (k != TD_BODY_EMPTY && k != TD_BODY_BUSY_WAIT && k != TD_BODY_COMPUTE && k != TD_BODY_MEMORY)
        return set_err(TD_E_COMPILE, "arrival-order mode supports empty / busy_wait / compute / memory bodies only");
    }
    const int16_t* dmap = nullptr;
    CUDA_TRY(sm_map_of(device, &dmap, &dyn_sms));
    if (dyn_sms <= 0) return set_err(TD_E_RESOURCE, "arrival-order mode needs the SM map (probe failed)");
    qdesc.resize((size_t)(n > 0 ? n : 1));
    qinfo.assign((size_t)(n > 0 ? n : 1), 0);
    std::vector<int64_t> cnt((size_t)dyn_sms + 1, 0);
    qsrc.assign((size_t)dyn_sms, 0);
    for (int64_t v = 0; v < n; ++v) {
      Desc& d = qdesc[v];
      memset(&d, 0, sizeof d);
      d.v = (int32_t)v;
      d.kind = c->kind[v];
      d.arg = c->arg[v];
      uint32_t indeg = 0;
      for (int64_t k = c->pred_ptr[v]; k < c->pred_ptr[v + 1]; ++k)
        indeg += (uint32_t)(c->pred_iv[2 * k + 1] - c->pred_iv[2 * k] + 1);
      d.nmsg = indeg;
      d.wslot = -1;
      const int32_t idv = c->ident ? c->ident[v] : (int32_t)v;
      d.hid = mix64_host((uint64_t)idv + G1);
      d.key = mix64_host((uint64_t)idv + G3);
      d.col = c->col ? c->col[v] : -1;
      int64_t nt = 0;
      for (int64_t k = c->succ_ptr[v]; k < c->succ_ptr[v + 1]; ++k) nt += c->succ_iv[2 * k + 1] - c->succ_iv[2 * k] + 1;
      if (nt <= NSUCC_INLINE) {
        int j = 0;
        for (int64_t k = c->succ_ptr[v]; k < c->succ_ptr[v + 1]; ++k)
          for (int32_t x = c->succ_iv[2 * k]; x <= c->succ_iv[2 * k + 1]; ++x) d.succ[j++] = x;
        d.nsucc = (uint8_t)j;
      } else {
        d.nsucc = TD_OVF;
        d.succ[0] = (int32_t)spool.size();
        d.succ[1] = (int32_t)(c->succ_ptr[v + 1] - c->succ_ptr[v]);
        for (int64_t k = c->succ_ptr[v]; k < c->succ_ptr[v + 1]; ++k)
          spool.push_back(make_int2(c->succ_iv[2 * k], c->succ_iv[2 * k + 1]));
      }
      const int32_t qv = worker_of[v] % dyn_sms;
      qinfo[v] = (indeg & 0xFFFFu) | ((uint32_t)qv << 16);
      ++cnt[qv + 1];
      if (!indeg) ++qsrc[qv];
    }
    qbase.assign((size_t)dyn_sms + 1, 0);
    for (int i = 0; i < dyn_sms; ++i) qbase[i + 1] = qbase[i] + cnt[i + 1];
    qentries.assign(2 * (size_t)(n > 0 ? n : 1), 0);
    std::vector<int64_t> fill(qbase.begin(), qbase.end() - 1);
    for (int64_t v = 0; v < n; ++v)  // sources, permanently at the head of their queue (input sum 0)
      if (!(qinfo[v] & 0xFFFFu)) {
        const int64_t k = fill[qinfo[v] >> 16]++;
        qentries[2 * k] = slot_tag((uint64_t)v + 1) << MSG_SHIFT;
        qentries[2 * k + 1] = (uint64_t)v + 1;
      }
  }

  ut_.mark("relays+dynamic");
  td_graph* g = new td_graph();
  memset(g, 0, sizeof *g);
  g->device = device;
  g->n = n;
  g->n_workers = c->n_workers + n_relays;
  g->n_graph_workers = c->n_workers;
  g->n_cols = c->n_cols;
  g->n_ranks = nr;
  g->my_rank = c->my_rank;
  g->n_ext_pre = c->n_ext_pre;
  g->n_ext_post = c->n_ext_post;
  g->n_positions = (int64_t)desc.size();
  g->has_st2d = has_st2d;
  for (int64_t v = 0; v < n; ++v)
    if (c->kind[v] == TD_BODY_MEMORY && c->arg[v] > g->max_mem_words) g->max_mem_words = c->arg[v];
  {
    bool plain = !has_st2d && n_shared == 0 && n_relays == 0 && !getenv("TD_NO_PLAIN");
    if (plain) {
      int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
      for (int64_t v = 0; v < n; ++v) bad |= !(c->kind[v] == TD_BODY_EMPTY || c->kind[v] == TD_BODY_COMPUTE);
      // the one-GPU PLAIN kernel has no successor-pool path (the sharded one has)
      if (nr == 1) {
#pragma omp parallel for schedule(static) reduction(| : bad)
        for (int64_t i = 0; i < (int64_t)desc.size(); ++i) bad |= desc[(size_t)i].nsucc == TD_OVF;
      }
      plain = !bad;
    }
    g->plain = plain;
    // GROUP mode (K = 4, else K = 2 "PAIR"): every worker list is in
    // nondecreasing level order (level = longest path from a source) and
    // splits into consecutive groups of K nodes of EQUAL level, e.g. K
    // columns of one Task Bench step.  Equal levels mean no path inside a
    // group (a group waits for all its inputs before any node sends), and the
    // sorted lists keep the progress argument: the lowest-level unexecuted
    // group has all its inputs.  A node of a K-group has 32/K lanes, so it may
    // have at most 32/K successor messages.  TD_GROUP=2|4 caps K, TD_NO_PAIR
    // turns the mode off.
    // (exact_k / pad_k from the layout pass above; a padded layout is
    // only made for graphs expected to qualify, and needs the GROUP kernel)
    int group = plain ? (exact_k ? exact_k : pad_k) : 0;
    if (group) {  // (sharded: pool rows run node by node)
      int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
      for (int64_t i = 0; i < (int64_t)desc.size(); ++i)
        bad |= desc[(size_t)i].nsucc > 32 / group && !(nr > 1 && desc[(size_t)i].nsucc == TD_OVF);
      if (bad) group = 0;
    }
    if (pad_k && group != pad_k) {
      // the padded layout turned out not to qualify for the GROUP kernel
      // (decided after the descriptors exist): lower again without padding
      td_graph_destroy(g);
      t_no_pad = true;
      const td_status st = td_graph_upload(c, device, out);
      t_no_pad = false;
      return st;
    }
    g->group = group;
    if (group) {
      // ring-add rounds of every pass (see DF_RING_ROUND_SHIFT): greedy
      // colouring, a node joins the first round none of whose nodes feeds
      // one of its slots (slots compared modulo the ring: positions relative
      // to the worker's first one differ by a constant, which preserves that)
      const int64_t nw = (int64_t)wptr.size() - 1;
#pragma omp parallel for schedule(static)
      for (int64_t w = 0; w < nw; ++w)
        for (int64_t i = wptr[w]; i + group <= wptr[w + 1]; i += group) {
          uint64_t used[4] = {0, 0, 0, 0};  // ring slots taken per round (LRING = 64 bits)
          int nrounds = 0;
          for (int k = 0; k < group; ++k) {
            Desc& dk = desc[(size_t)(i + k)];
            uint64_t mine = 0;
            for (uint32_t ld = dk.ldelta; ld; ld >>= 8) mine |= 1ull << ((i + k + (int64_t)(ld & 0xFFu)) & (LRING - 1));
            if (!mine) continue;
            int r = 0;
            while (used[r] & mine) ++r;  // (at most `group` rounds: one node per round)
            used[r] |= mine;
            nrounds = std::max(nrounds, r + 1);
            dk.dflags = (uint8_t)(dk.dflags | (r << DF_RING_ROUND_SHIFT));
          }
          desc[(size_t)i].dflags = (uint8_t)(desc[(size_t)i].dflags | (nrounds << DF_RING_NROUNDS_SHIFT));
        }
    }
  }
  if (nr > 1) g->node_rank_host = new std::vector<uint8_t>(c->node_rank, c->node_rank + n);
  // node mailboxes, then two banks of shared (bundled) mailbox replicas
  {
    // mailbox spacing (see slot()): 32 B for one-node-per-pass graphs, 8 B
    // for GROUP graphs.  Every shard derives the same value from the same
    // graph, so peers index each other's mailboxes consistently (2 GPUs,
    // sharded headline: 0.988 -> 0.954 ms, profiles/r02_ab_slot_shards.log).
    // TD_SLOT_SHIFT=0..4 overrides (set it identically on every rank).
    const char* se = getenv("TD_SLOT_SHIFT");
    g->slot_shift = se ? std::max(0, std::min(4, atoi(se))) : (g->group == 0 ? 2 : 0);
  }
  g->n_comb = (int32_t)comb_info.size();
  g->shared_base = ((((int64_t)(n > 0 ? n : 1) << g->slot_shift) + SHARE_STRIDE - 1) / SHARE_STRIDE) * SHARE_STRIDE;
  g->n_slots = g->shared_base + 2 * n_shared * SHARE_SPLIT * SHARE_STRIDE;
  g->n_shared = n_shared;
  g->comb_base = ((g->n_slots + SHARE_STRIDE - 1) / SHARE_STRIDE) * SHARE_STRIDE;  // one 256 B granule each
  g->n_slots = g->comb_base;
  g->n_slots += (int64_t)g->n_comb * SHARE_STRIDE;
  g->n_succ_pool = (int64_t)spool.size();
  ut_.mark("plain/group");
  cudaError_t e = cudaSuccess;
#define UP(field, src, cnt) if (e == cudaSuccess) e = upload(&g->field, src, (size_t)(cnt))
  if (desc.empty()) desc.emplace_back();
  UP(desc, desc.data(), desc.size());
  UP(work_ptr, wptr.data(), wptr.size());
  UP(succ_pool, spool.data(), spool.size());
  UP(worker_of, worker_of.data(), n > 0 ? n : 1);
  {
    std::vector<uint8_t> wr(wptr.size() > 1 ? wptr.size() - 1 : 1, 0);
    for (size_t w = 0; w + 1 < wptr.size(); ++w)
      for (int64_t i = wptr[w]; i < wptr[w + 1]; ++i) wr[w] |= desc[i].rmask != 0;
    UP(wremote, wr.data(), wr.size());
  }
  g->has_col = c->col != nullptr;
  // checksum banks and the poison word in one buffer: bank 0 | poison | bank 1,
  // so one copy brings back a bank and the poison word together
  UP(colsum, (const unsigned long long*)nullptr, 2 * (size_t)std::max(c->n_cols, 0) + 1);
  if (e == cudaSuccess) g->poison = reinterpret_cast<uint32_t*>(g->colsum + std::max(c->n_cols, 0));
  UP(token, (const unsigned long long*)nullptr, g->n_slots);
  UP(mbox, (const unsigned long long*)nullptr, g->n_slots);
  UP(tally, (const uint32_t*)nullptr, n > 0 ? n : 1);
  UP(stats, (const unsigned long long*)nullptr, 8);
  UP(started, (const uint32_t*)nullptr, TD_MAX_RANKS);
  UP(sm_ctr, (const uint32_t*)nullptr, TD_MAX_SMID);
  UP(comb, comb_info.data(), comb_info.size());
  if (want_dyn) {
    g->dyn = true;
    g->dyn_sms = dyn_sms;
    UP(qdesc, qdesc.data(), qdesc.size());
    UP(qinfo, qinfo.data(), qinfo.size());
    UP(q_slots, qentries.data(), qentries.size());
    UP(q_init, qentries.data(), qentries.size());
    UP(q_base, qbase.data(), qbase.size());
    UP(q_src, qsrc.data(), qsrc.size());
    UP(q_head, (const uint32_t*)nullptr, dyn_sms);
    UP(q_tail, (const uint32_t*)nullptr, dyn_sms);
  }
#undef UP
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&g->h_ext_pre, sizeof(uint32_t) * (g->n_ext_pre + 1), cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&g->h_ext_post, sizeof(uint32_t) * (g->n_ext_post + 1), cudaHostAllocMapped);
  // h_abort[0]: the host's abort request; h_abort[1]: the kernel's mirror of the poison code
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&g->h_abort, 2 * sizeof(uint32_t), cudaHostAllocMapped);
  if (e == cudaSuccess)
    e = cudaHostAlloc((void**)&g->h_colsum, sizeof(unsigned long long) * (2 * (size_t)std::max(g->n_cols, 0) + 1), cudaHostAllocDefault);
  if (e == cudaSuccess) memset(g->h_colsum, 0, sizeof(unsigned long long) * (2 * (size_t)std::max(g->n_cols, 0) + 1));
  {
    const char* be = getenv("TD_SHARED_BACKOFF");
    g->shared_backoff_ns = be ? (uint32_t)atoi(be) : 0u;
    const char* fm = getenv("TD_FORCE_MULTI");
    g->force_multi = fm && fm[0] == '1';
    const char* pe = getenv("TD_PLACE");
    g->place_env = pe ? (pe[0] == '0' ? 0 : 1) : -1;
  }
  if (e == cudaSuccess) {
    memset(g->h_ext_pre, 0, sizeof(uint32_t) * (g->n_ext_pre + 1));
    memset(g->h_ext_post, 0, sizeof(uint32_t) * (g->n_ext_post + 1));
    g->h_abort[0] = g->h_abort[1] = 0;
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
  ut_.mark("device upload");
  *out = g;
  return TD_OK;
}

td_status td_graph_launch(td_graph* g, const td_launch_params* p, void* stream) {
  if (!g || !p) return set_err(TD_E_CONTRACT, "null argument");
#ifdef TD_LAUNCH_PROFILE
  uint64_t lp_t = lp_now();
  ++lp_n;
#endif
  CUDA_TRY(cudaSetDevice(g->device));
  LP(0);
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
  const bool multi = g->n_ranks > 1 || g->force_multi;
#ifdef TD_CYCLE_PROBE
  const bool diag = p->flags & (TD_F_STATS | TD_F_TALLY | (g->group ? 0u : (uint32_t)TD_F_TRACE));
#else
  const bool diag = p->flags & (TD_F_STATS | TD_F_TALLY | TD_F_TRACE);
#endif
  const bool dynamic = (p->flags & TD_F_DYNAMIC) != 0;
  if (dynamic && !g->dyn) return set_err(TD_E_CONTRACT, "TD_F_DYNAMIC needs a graph uploaded with TD_UPLOAD_DYNAMIC");
  const void* fn = dynamic ? (const void*)td_dyn_kernel : kernel_for(multi, g->has_st2d, diag, g->plain, g->group);
  if (g->has_st2d && !g->st_grid[0]) return set_err(TD_E_CONTRACT, "graph has STENCIL2D nodes: call td_graph_attach_stencil2d first");
  if (g->max_mem_words && (int64_t)g->max_mem_words > g->scratch_words)
    return set_err(TD_E_CONTRACT, "memory_bound nodes stream %u words: attach scratch of at least that many words per worker (td_graph_attach_scratch)", g->max_mem_words);
  const size_t dyn = dynamic ? dyn_pad_bytes(g->device) : dyn_smem_for(multi, g->has_st2d, g->device);
  if (!g->resident_ctas)  // occupancy (and the dynamic smem attribute), queried once per graph
    CUDA_TRY(resident_ctas_of(multi, g->has_st2d, g->device, &g->resident_ctas));
  int64_t blocks = (g->n_workers + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
  // SM-balanced placement (lean kernels; TD_PLACE=0 turns it off): a full
  // grid, workers spread round-robin over SMs, then sub-partitions
  const int16_t* sm_map = nullptr;
  int n_sms = 0;
  // policy (same-box A/B, profiles/r02_ab_place_group.log): on for one-GPU
  // graphs with more than 2048 workers and no shared mailboxes (fft 4096
  // -8 %, tree -3.5 %); off for the 1024-worker headline (+5 %) and bundled
  // all_to_all (+22 %); never for sharded graphs, whose shards may share a
  // GPU (a full grid per shard could not be co-resident).  TD_PLACE=1 / 0
  // forces it on / off.
  bool place = dynamic || (!g->has_st2d && g->n_ranks == 1 && !g->force_multi &&
               (g->place_env > 0 || (g->place_env < 0 && g->n_workers > 2048 && g->n_shared == 0)));
  if (place) CUDA_TRY(sm_map_of(g->device, &sm_map, &n_sms));
  place = place && n_sms > 0 && g->resident_ctas % n_sms == 0;
  if (place && g->place_fn != fn) {  // the launched kernel must fit exactly occ CTAs per SM
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * WARPS_PER_CTA, dyn));
    if ((int64_t)per_sm * n_sms != g->resident_ctas) place = false;
    else g->place_fn = fn;
  }
  if (dynamic && !place) return set_err(TD_E_RESOURCE, "arrival-order mode needs the SM-balanced placement");
  if (multi && blocks == 0) blocks = 1;  // the start handshake still runs
  if (blocks > g->resident_ctas)
    return set_err(TD_E_RESOURCE, "%d workers exceed the %lld co-resident warps of this GPU",
                   g->n_workers, (long long)g->resident_ctas * WARPS_PER_CTA);
  if (multi)
    for (int r = 0; r < g->n_ranks; ++r)
      if (r != g->my_rank && !g->peer_opened[r] && !g->peer_direct[r])
        return set_err(TD_E_RESOURCE, "peer shard %d not attached", r);
  // every mailbox is re-armed by its consumer; only an aborted execution
  // can leave partial sums behind
  const int64_t nc = std::max(g->n_cols, 0);
  if (g->dirty) {
    CUDA_TRY(cudaMemsetAsync(g->mbox, 0, sizeof(unsigned long long) * g->n_slots, s));
    // both checksum banks and the poison word (an aborted execution may have
    // left partial column folds behind)
    CUDA_TRY(cudaMemsetAsync(g->colsum, 0, sizeof(unsigned long long) * (2 * nc + 1), s));
    if (g->dyn)  // an aborted arrival-order execution can leave filled queue slots behind
      CUDA_TRY(cudaMemcpyAsync(g->q_slots, g->q_init, 2 * sizeof(unsigned long long) * (g->n > 0 ? g->n : 1),
                               cudaMemcpyDeviceToDevice, s));
    g->dirty = false;
  }
  LP(1);
  uint32_t flags = p->flags;
  if (!g->has_col) flags &= ~(uint32_t)TD_F_CHECKSUM;  // graph has no checksum columns
  // checksum bank of this launch (zeroed by the previous checksum launch's
  // kernel, or at upload), and the other bank for this kernel to zero
  const bool cs = (flags & TD_F_CHECKSUM) != 0;
  if (cs) ++g->cs_launches;
  const int64_t cs_off = (g->cs_launches & 1) ? nc + 1 : 0;
  if (p->flags & TD_F_STATS) CUDA_TRY(cudaMemsetAsync(g->stats, 0, sizeof(unsigned long long) * 8, s));
#ifdef TD_CYCLE_PROBE
  if (p->flags & TD_F_TRACE) CUDA_TRY(cudaMemsetAsync(g->stats, 0, sizeof(unsigned long long) * 8, s));
#endif
  if (p->flags & TD_F_TALLY) CUDA_TRY(cudaMemsetAsync(g->tally, 0, sizeof(uint32_t) * (g->n > 0 ? g->n : 1), s));
  if ((p->flags & TD_F_TRACE) && !g->trace)
    CUDA_TRY(cudaMalloc(&g->trace, sizeof(unsigned long long) * TRACE_WORDS * (g->n > 0 ? g->n : 1)));
  // the poison word is sticky across queued (TD_F_QUEUE) executions: a
  // failure of an earlier queued execution is not cleared by a later launch
  // (whose workers then stop at once), and the first failure's code is kept
  // (atomicCAS from 0); finish_wait marks the graph dirty and the next
  // launch clears the mailboxes, checksum banks and poison word together
  // (above), so a clean replay needs no memset at all
  // Sharded launches keep one memset in front of the kernel: shards of one
  // process that share a GPU (InProcessShards) need their cooperative kernels
  // to run concurrently, and without a preceding stream operation the second
  // replay of 8 same-device shards was observed to run them one after another
  // (deadlock until the spin limit; a memset of any buffer, not a host delay,
  // avoided it: scripts/dbg_shards.py, profiles/r02_summary.md)
  if (multi && !g->outstanding) CUDA_TRY(cudaMemsetAsync(g->poison, 0, sizeof(uint32_t), s));
  *g->h_abort = 0;
  // the host-mapped poison mirror: cleared unless a queued execution is still
  // running (sticky like the device word, which only a failure leaves set)
  if (!g->outstanding) ((volatile uint32_t*)g->h_abort)[1] = 0;
  for (int j = 0; j < g->n_ext_post; ++j) g->h_ext_post[j] = 0;

  Params P;
  memset(&P, 0, sizeof P);
  P.desc = g->desc;
  P.work_ptr = g->work_ptr;
  P.succ_pool = g->succ_pool;
  P.worker_of = g->worker_of;
  P.wremote = g->wremote;
  P.n_workers = g->n_workers;
  P.n_graph_workers = g->n_graph_workers;
  P.colsum = g->colsum + cs_off;
  P.colsum_zero = cs ? g->colsum + (nc + 1 - cs_off) : nullptr;
  P.n_cols = (int32_t)nc;
  P.mbox = g->mbox;
  P.n_nodes = (int32_t)g->n;
  P.n_shared = g->n_shared;
  P.comb_id0 = g->n_comb ? (int32_t)(g->n + g->n_shared) : INT32_MAX;
  P.comb_base = g->comb_base;
  P.shared_base = g->shared_base;
  P.comb = g->comb;
  P.mbox_words = g->n_slots;
  {
    P.shared_backoff_ns = g->shared_backoff_ns;
  }
  P.token = g->token;
  P.tally = g->tally;
  P.stats = g->stats;
  P.trace = g->trace;
  P.ext_pre = g->d_ext_pre;
  P.ext_post = g->d_ext_post;
  P.abort_flag = g->d_abort;
  P.poison_host = reinterpret_cast<uint32_t*>(g->d_abort) + 1;
  P.poison = g->poison;
  P.seed = p->seed;
  P.exec_no = g->launches + 1u;
  P.flags = flags;
  P.spin_limit = p->spin_limit;
  P.my_rank = g->my_rank;
  P.n_ranks = g->n_ranks;
  P.started = g->started;
  for (int r = 0; r < TD_MAX_RANKS; ++r) {
    P.peer_mbox[r] = g->peer_mbox[r];
    P.peer_started[r] = g->peer_started[r];
    P.st_peer_grid[r][0] = g->st_peer_grid[r][0];
    P.st_peer_grid[r][1] = g->st_peer_grid[r][1];
  }
  P.st_nx = g->st_nx;
  P.st_ny = g->st_ny;
  P.st_tiles_x = g->st_tiles_x;
  P.st_tiles_y = g->st_tiles_y;
  P.st_ntiles = g->st_ntiles;
  P.st_grid[0] = g->st_grid[0];
  P.st_grid[1] = g->st_grid[1];
  P.st_tile_rank = g->st_tile_rank;
  P.st_tmap[0] = g->st_tmap[0];
  P.st_tmap[1] = g->st_tmap[1];
  P.scratch = g->scratch;
  P.scratch_words = g->scratch_words;
  P.slot_shift = g->slot_shift;
  if (dynamic) {
    P.qdesc = g->qdesc;
    P.qinfo = g->qinfo;
    P.q_slots = g->q_slots;
    P.q_base = g->q_base;
    P.q_src = g->q_src;
    P.q_head = g->q_head;
    P.q_tail = g->q_tail;
    CUDA_TRY(cudaMemsetAsync(g->q_head, 0, sizeof(uint32_t) * g->dyn_sms, s));
    CUDA_TRY(cudaMemcpyAsync(g->q_tail, g->q_src, sizeof(uint32_t) * g->dyn_sms, cudaMemcpyDeviceToDevice, s));
  }
  if (place && blocks > 0) {
    P.place = 1;
    P.n_sms = n_sms;
    P.occ = (int32_t)(g->resident_ctas / n_sms);
    P.sm_dense = sm_map;
    P.sm_ctr = g->sm_ctr;
    blocks = g->resident_ctas;
  }

  LP(2);
  CUDA_TRY(cudaEventRecord(g->ev_start, s));
  LP(3);
  if (blocks > 0) {
    void* args[] = {&P};
    // (a plain cudaLaunchKernel measured 0.5 us faster per replay and an
    // unpadded launch 0.3 us: kept cooperative and pinned, which guarantee
    // co-residency; scripts/launch_variants.py, profiles/r02_launch_variants.log)
    CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3((unsigned)blocks), dim3(tpb), args, dyn, s));
  }
  LP(4);
  // a checksum launch's bank rides back with the stream into the pinned
  // mirror, so td_graph_checksums needs no device round trip of its own; the
  // poison code comes back through the host-mapped word the kernel writes
  // (poison_set), so a replay without checksums enqueues no copy at all
  g->colsum_on_host = false;
  if (cs)
    CUDA_TRY(cudaMemcpyAsync(g->h_colsum + cs_off, g->colsum + cs_off, sizeof(unsigned long long) * nc,
                             cudaMemcpyDeviceToHost, s));
  LP(5);
  CUDA_TRY(cudaEventRecord(g->ev_stop, s));
  LP(6);
  g->outstanding = true;
  g->last_flags = p->flags;
  g->blocks = (int32_t)blocks;
  g->tpb = (int32_t)tpb;
  g->last_stream = stream;
  g->launches += 1;
  return TD_OK;
}

static td_status finish_wait(td_graph* g) {
  g->outstanding = false;
  g->completed += 1;
  g->colsum_on_host = (g->last_flags & TD_F_CHECKSUM) && g->h_colsum;
  const uint32_t poison = ((volatile uint32_t*)g->h_abort)[1];  // mirrored by the kernel (poison_set)
  if (poison) {
    g->dirty = true;
    return set_err(TD_E_POISONED, poison == 2   ? "execution poisoned: more messages than in-edges"
                                  : poison == 3 ? "execution poisoned: SM placement found an SM with an unexpected CTA count (set TD_PLACE=0)"
                                                : "execution poisoned (spin limit exceeded)");
  }
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
      g->dirty = true;
      return set_err(TD_E_WAIT_TIMEOUT, "execution did not finish within %.3f s", timeout_s);
    }
    struct timespec ts = {0, 20000};
    nanosleep(&ts, nullptr);
  }
}

td_status td_graph_trigger_pre(td_graph* g, int32_t index) {
  if (!g) return set_err(TD_E_CONTRACT, "null argument");
  if (index < 0 || index >= g->n_ext_pre) return set_err(TD_E_RESOURCE, "precondition %d out of range", index);
  // flags carry the execution number of the current (or next) execution
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
  // the bank of the last checksum launch (later launches without
  // TD_F_CHECKSUM leave both banks alone)
  const int64_t off = (g->cs_launches & 1) ? (int64_t)n_cols + 1 : 0;
  if (g->colsum_on_host && !g->outstanding) {  // copied back behind the last (completed) replay
    if (n_cols) memcpy(host, g->h_colsum + off, sizeof(uint64_t) * n_cols);
    return TD_OK;
  }
  CUDA_TRY(cudaSetDevice(g->device));
  if (n_cols) CUDA_TRY(cudaMemcpy(host, g->colsum + off, sizeof(uint64_t) * n_cols, cudaMemcpyDeviceToHost));
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
  out->workers = g->n_graph_workers;
  out->blocks = g->blocks;
  out->threads_per_block = g->tpb;
  return TD_OK;
}

td_status td_graph_trace(td_graph* g, uint64_t* host, int64_t n) {
  if (!g || (!host && n)) return set_err(TD_E_CONTRACT, "null argument");
#ifdef TD_CYCLE_PROBE
  // (diagnostic build: 8 more words = the stats words, [5] = ~first CTA entry, [6] = last warp exit)
  const bool with_stats = n == TRACE_WORDS * g->n + 8;
  if (with_stats) n -= 8;
#endif
  if (n != TRACE_WORDS * g->n) return set_err(TD_E_CONTRACT, "trace buffer must hold %d*n entries", TRACE_WORDS);
  if (!g->trace) return set_err(TD_E_CONTRACT, "no TD_F_TRACE execution yet");
  CUDA_TRY(cudaSetDevice(g->device));
  if (n) CUDA_TRY(cudaMemcpy(host, g->trace, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
#ifdef TD_CYCLE_PROBE
  if (with_stats) CUDA_TRY(cudaMemcpy(host + n, g->stats, sizeof(uint64_t) * 8, cudaMemcpyDeviceToHost));
#endif
  return TD_OK;
}

td_status td_graph_info_get(td_graph* g, td_graph_info* out) {
  if (!g || !out) return set_err(TD_E_CONTRACT, "null argument");
  memset(out, 0, sizeof *out);
  out->n_nodes = g->n;
  out->n_positions = g->n_positions;
  out->n_shared = g->n_shared;
  out->n_workers = g->n_workers;
  out->n_graph_workers = g->n_graph_workers;
  out->n_ranks = g->n_ranks;
  out->my_rank = g->my_rank;
  out->plain = g->plain;
  out->group = g->group;
  out->has_stencil2d = g->has_st2d;
  out->desc_bytes = (int32_t)sizeof(Desc);
  out->slot_shift = g->slot_shift;
  out->n_combiners = g->n_comb;
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
  const int nh = g->st_grid[0] ? 4 : 2;
  const size_t need = nh * sizeof(cudaIpcMemHandle_t);
  *len = need;
  if (cap < need) return set_err(TD_E_CONTRACT, "handle buffer too small (%zu < %zu)", cap, need);
  CUDA_TRY(cudaSetDevice(g->device));
  cudaIpcMemHandle_t* h = (cudaIpcMemHandle_t*)out;
  CUDA_TRY(cudaIpcGetMemHandle(&h[0], g->mbox));
  CUDA_TRY(cudaIpcGetMemHandle(&h[1], g->started));
  if (nh == 4) {
    CUDA_TRY(cudaIpcGetMemHandle(&h[2], g->st_grid[0]));
    CUDA_TRY(cudaIpcGetMemHandle(&h[3], g->st_grid[1]));
  }
  return TD_OK;
}

td_status td_graph_ipc_attach(td_graph* g, int32_t rank, const void* handle, size_t len) {
  if (!g || !handle) return set_err(TD_E_CONTRACT, "null argument");
  if (rank < 0 || rank >= g->n_ranks || rank == g->my_rank) return set_err(TD_E_RESOURCE, "bad peer rank %d", rank);
  if (len < 2 * sizeof(cudaIpcMemHandle_t)) return set_err(TD_E_CONTRACT, "short handle");
  if (g->st_grid[0] && len < 4 * sizeof(cudaIpcMemHandle_t))
    return set_err(TD_E_CONTRACT, "peer shard exported no stencil grid");
  CUDA_TRY(cudaSetDevice(g->device));
  const cudaIpcMemHandle_t* h = (const cudaIpcMemHandle_t*)handle;
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h[0], cudaIpcMemLazyEnablePeerAccess));
  g->peer_mbox[rank] = (unsigned long long*)p;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h[1], cudaIpcMemLazyEnablePeerAccess));
  g->peer_started[rank] = (uint32_t*)p;
  if (g->st_grid[0]) {
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h[2], cudaIpcMemLazyEnablePeerAccess));
    g->st_peer_grid[rank][0] = (uint32_t*)p;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h[3], cudaIpcMemLazyEnablePeerAccess));
    g->st_peer_grid[rank][1] = (uint32_t*)p;
  }
  g->peer_opened[rank] = true;
  return TD_OK;
}

td_status td_graph_peer_attach_direct(td_graph* g, int32_t rank, td_graph* peer) {
  if (!g || !peer) return set_err(TD_E_CONTRACT, "null argument");
  if (rank < 0 || rank >= g->n_ranks || rank == g->my_rank || peer->my_rank != rank)
    return set_err(TD_E_RESOURCE, "bad peer rank %d", rank);
  if (peer->n != g->n || peer->n_slots != g->n_slots) return set_err(TD_E_CONTRACT, "peer shard has a different graph");
  CUDA_TRY(cudaSetDevice(g->device));
  if (peer->device != g->device) {
    cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
      return set_err(TD_E_CUDA, "peer access %d -> %d: %s", g->device, peer->device, cudaGetErrorString(e));
    cudaGetLastError();
  }
  g->peer_mbox[rank] = peer->mbox;
  g->peer_started[rank] = peer->started;
  g->st_peer_grid[rank][0] = peer->st_grid[0];
  g->st_peer_grid[rank][1] = peer->st_grid[1];
  g->peer_opened[rank] = false;  // not IPC-mapped: nothing to close
  g->peer_direct[rank] = true;
  return TD_OK;
}

td_status td_graph_attach_stencil2d(td_graph* g, int32_t nx, int32_t ny) {
  if (!g) return set_err(TD_E_CONTRACT, "null argument");
  if (!g->has_st2d) return set_err(TD_E_CONTRACT, "graph has no STENCIL2D nodes");
  if (g->st_grid[0]) return set_err(TD_E_CONTRACT, "stencil grid already attached");
  if (nx <= 0 || ny <= 0 || nx % TILE || ny % TILE) return set_err(TD_E_RESOURCE, "grid must be a positive multiple of %d", TILE);
  const int32_t tx = nx / TILE, ty = ny / TILE;
  const int64_t ntiles = (int64_t)tx * ty;
  if (g->n % ntiles) return set_err(TD_E_GRAPH, "node count %lld is not steps x %lld tiles", (long long)g->n, (long long)ntiles);
  CUDA_TRY(cudaSetDevice(g->device));
  const size_t bytes = sizeof(uint32_t) * (size_t)nx * (size_t)ny;
  cudaError_t e = cudaMalloc(&g->st_grid[0], bytes);
  if (e == cudaSuccess) e = cudaMalloc(&g->st_grid[1], bytes);
  if (e == cudaSuccess) e = cudaMemset(g->st_grid[0], 0, bytes);
  if (e == cudaSuccess) e = cudaMemset(g->st_grid[1], 0, bytes);
  if (e == cudaSuccess && g->n_ranks > 1) {
    // shard of every tile; a tile must stay on one shard across steps
    std::vector<uint8_t> tr((size_t)ntiles);
    const std::vector<uint8_t>& nrk = *g->node_rank_host;
    for (int64_t t = 0; t < ntiles; ++t) tr[t] = nrk[t];
    for (int64_t v = 0; v < g->n; ++v)
      if (nrk[v] != tr[v % ntiles]) return set_err(TD_E_GRAPH, "a stencil tile moves between shards across steps");
    e = cudaMalloc(&g->st_tile_rank, ntiles);
    if (e == cudaSuccess) e = cudaMemcpy(g->st_tile_rank, tr.data(), ntiles, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) return set_err(e == cudaErrorMemoryAllocation ? TD_E_ALLOCATION : TD_E_CUDA, "stencil grid: %s", cudaGetErrorString(e));
  {
    // 2-D TMA descriptors of both buffers: box 72 x 66 u32, OOB -> zeros
    typedef CUresult (*encode_fn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    if (!fp || q != cudaDriverEntryPointSuccess) return set_err(TD_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)ny};
    const cuuint64_t strides[1] = {(cuuint64_t)nx * 4};
    const cuuint32_t box[2] = {BOX_W, BOX_H};
    const cuuint32_t estr[2] = {1, 1};
    for (int b = 0; b < 2; ++b) {
      // L2 promotion of the box loads (TD_TMA_PROMO=0/64/128/256 for A/B; default 256 B)
      const char* pe = getenv("TD_TMA_PROMO");
      const int pv = pe ? atoi(pe) : 256;
      const CUtensorMapL2promotion promo = pv == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                           : pv == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                           : pv == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                                       : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
      CUresult r = ((encode_fn)fp)(&g->st_tmap[b], CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, g->st_grid[b], dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return set_err(TD_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    }
  }
  g->st_nx = nx;
  g->st_ny = ny;
  g->st_tiles_x = tx;
  g->st_tiles_y = ty;
  g->st_ntiles = (int32_t)ntiles;
  return TD_OK;
}

td_status td_graph_attach_scratch(td_graph* g, int64_t words_per_worker) {
  if (!g) return set_err(TD_E_CONTRACT, "null argument");
  if (words_per_worker < 0 || words_per_worker % 64) return set_err(TD_E_RESOURCE, "scratch words must be a non-negative multiple of 64");
  if (g->outstanding) {
    cudaError_t q = cudaEventQuery(g->ev_stop);
    if (q == cudaErrorNotReady) return set_err(TD_E_EXEC_STATE, "an execution of this graph is outstanding");
  }
  CUDA_TRY(cudaSetDevice(g->device));
  if (g->scratch) CUDA_TRY(cudaFree(g->scratch));
  g->scratch = nullptr;
  g->scratch_words = 0;
  const size_t bytes = sizeof(unsigned long long) * (size_t)words_per_worker * (size_t)(g->n_workers > 0 ? g->n_workers : 1);
  if (bytes) {
    cudaError_t e = cudaMalloc(&g->scratch, bytes);
    if (e != cudaSuccess) return set_err(e == cudaErrorMemoryAllocation ? TD_E_ALLOCATION : TD_E_CUDA, "scratch: %s", cudaGetErrorString(e));
  }
  g->scratch_words = words_per_worker;
  return TD_OK;
}

td_status td_graph_stencil2d_grid(td_graph* g, int32_t buf, uint32_t* host, int64_t n) {
  if (!g || (!host && n)) return set_err(TD_E_CONTRACT, "null argument");
  if (!g->st_grid[0]) return set_err(TD_E_CONTRACT, "no stencil grid attached");
  if (buf < 0 || buf > 1 || n != (int64_t)g->st_nx * g->st_ny) return set_err(TD_E_CONTRACT, "bad buffer index or size");
  CUDA_TRY(cudaSetDevice(g->device));
  CUDA_TRY(cudaMemcpy(host, g->st_grid[buf], sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
  return TD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Re-parameterise task bodies in place (Task Bench varies only the work per
// task): descriptors of COMPUTE / BUSY_WAIT nodes get `arg`.
// ---------------------------------------------------------------------------
namespace {
__global__ void set_body_arg_kernel(Desc* d, int64_t n, uint32_t arg) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (d[i].kind == TD_BODY_COMPUTE || d[i].kind == TD_BODY_BUSY_WAIT) d[i].arg = arg;
}
}  // namespace

extern "C" td_status td_graph_set_body_arg(td_graph* g, uint32_t arg) {
  if (!g) return set_err(TD_E_CONTRACT, "null argument");
  if (g->outstanding) {
    cudaError_t q = cudaEventQuery(g->ev_stop);
    if (q == cudaErrorNotReady) return set_err(TD_E_EXEC_STATE, "an execution of this graph is outstanding");
  }
  CUDA_TRY(cudaSetDevice(g->device));
  if (g->n_positions) {
    set_body_arg_kernel<<<(unsigned)((g->n_positions + 255) / 256 < 1184 ? (g->n_positions + 255) / 256 : 1184), 256>>>(
        g->desc, g->n_positions, arg);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
  }
  return TD_OK;
}

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

__global__ void __launch_bounds__(32) td_rt_task_kernel(const __grid_constant__ RtTask A, unsigned long long* tok,
                                                        unsigned long long* term) {
  const int lane = threadIdx.x;
  uint64_t acc = 0;  // exact sum of the predecessors' 32-bit terms (oracle/tokens.py)
  for (int j = lane; j < A.n_pred; j += 32) acc += term[A.pred[j]];
  acc = warp_sum_u64(acc);
  const uint64_t h = mix64(mix64(A.seed ^ mix64(A.key + G1)) ^ acc);
  const uint64_t t = h ^ run_body((int)A.kind, A.arg, h, make_ulonglong2((uint64_t)(lane + 1) * G2, (uint64_t)(lane + 33) * G2));
  if (lane == 0) {
    tok[A.slot] = t;
    term[A.slot] = mix64(t ^ mix64(A.key + G3)) >> 32;
  }
}
}  // namespace

namespace {
// Import tokens computed elsewhere (a compiled replay) into runtime slots:
// tok[slot] = t, term[slot] = mix64(t ^ mix64(key + G3)) >> 32.
__global__ void td_rt_store_kernel(const int64_t* slots, const uint64_t* keys, const uint64_t* toks, int32_t n,
                                   unsigned long long* tok, unsigned long long* term) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t t = toks[i];
    tok[slots[i]] = t;
    term[slots[i]] = mix64(t ^ mix64(keys[i] + G3)) >> 32;
  }
}
}  // namespace

struct td_rt {
  int device;
  int64_t capacity;
  unsigned long long* tok;
  unsigned long long* term;
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
  if (e == cudaSuccess) e = cudaMalloc(&rt->term, sizeof(unsigned long long) * capacity);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rt->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    if (rt->tok) cudaFree(rt->tok);
    if (rt->term) cudaFree(rt->term);
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
  td_rt_task_kernel<<<1, 32, 0, rt->stream>>>(A, rt->tok, rt->term);
  CUDA_TRY(cudaGetLastError());
  return TD_OK;
}

td_status td_rt_store_tokens(td_rt* rt, const int64_t* slots, const uint64_t* keys, const uint64_t* tokens,
                             int32_t n) {
  if (!rt || (n && (!slots || !keys || !tokens))) return set_err(TD_E_CONTRACT, "null argument");
  if (n < 0) return set_err(TD_E_CONTRACT, "negative count");
  for (int32_t i = 0; i < n; ++i)
    if (slots[i] < 0 || slots[i] >= rt->capacity) return set_err(TD_E_RESOURCE, "slot %lld out of range", (long long)slots[i]);
  if (!n) return TD_OK;
  CUDA_TRY(cudaSetDevice(rt->device));
  void* buf = nullptr;
  const size_t b = sizeof(int64_t) * (size_t)n;
  CUDA_TRY(cudaMalloc(&buf, 3 * b));
  char* c = (char*)buf;
  cudaError_t e = cudaMemcpyAsync(c, slots, b, cudaMemcpyHostToDevice, rt->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c + b, keys, b, cudaMemcpyHostToDevice, rt->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(c + 2 * b, tokens, b, cudaMemcpyHostToDevice, rt->stream);
  if (e == cudaSuccess) {
    td_rt_store_kernel<<<(n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184, 256, 0, rt->stream>>>(
        (const int64_t*)c, (const uint64_t*)(c + b), (const uint64_t*)(c + 2 * b), n, rt->tok, rt->term);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(rt->stream);
  cudaFree(buf);
  if (e != cudaSuccess) return set_err(TD_E_CUDA, "td_rt_store_tokens: %s", cudaGetErrorString(e));
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
  cudaFree(rt->term);
  delete rt;
  return TD_OK;
}

}  // extern "C"

