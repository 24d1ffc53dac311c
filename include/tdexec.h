/*
 * tdexec.h — C ABI of the B200 persistent task-graph executor (libtdexec.so).
 *
 * This is the drop-in boundary for the paper's hot path: replaying a
 * pre-analysed (traced) task graph with actor-style, counter-based triggering
 * (Alg. 1, 632-693; SPEC.md compiler 351-425, implicit.replay
 * 465-473).  The reference is Python and has no FFI; each entry point below
 * names the reference operation it replaces.  Plain pointers and sizes only —
 * no torch or CUDA types cross this boundary (streams are passed as void*).
 *
 * Status codes map 1:1 onto the reference's exception classes
 * (reference pkg/src/taskdual/errors.py:4-53); see td_status below.
 *
 * Threading: all calls for one td_graph come from
 * one host thread.  Executions of one graph never overlap:
 * launches are stream-ordered and td_graph_launch refuses a second
 * un-awaited launch unless TD_F_QUEUE is set.
 */
#ifndef TDEXEC_H
#define TDEXEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t td_status;
enum {
  TD_OK = 0,
  TD_E_RESOURCE = 1,      /* ResourceError      errors.py:8   */
  TD_E_ALLOCATION = 2,    /* AllocationError    errors.py:12  */
  TD_E_REGISTRATION = 3,  /* RegistrationError  errors.py:16  */
  TD_E_CONTRACT = 4,      /* ContractViolation  errors.py:20  */
  TD_E_QUIESCENCE = 5,    /* QuiescenceTimeout  errors.py:24  */
  TD_E_WAIT_TIMEOUT = 6,  /* WaitTimeout        errors.py:28  */
  TD_E_GRAPH = 7,         /* GraphError         errors.py:32  */
  TD_E_GRAPH_PARSE = 8,   /* GraphParseError    errors.py:36  */
  TD_E_COMPILE = 9,       /* CompileError       errors.py:40  */
  TD_E_EXEC_STATE = 10,   /* ExecutionStateError errors.py:44 */
  TD_E_POISONED = 11,     /* ExecutionPoisoned  errors.py:48  */
  TD_E_TRACE = 12,        /* TraceError         errors.py:52  */
  TD_E_CUDA = 13          /* CUDA runtime failure (no reference analogue) */
};

/* Device task bodies (SPEC.md:161-164 TaskFn, narrowed to a device table). */
enum {
  TD_BODY_EMPTY = 0,      /* r = 0                                          */
  TD_BODY_BUSY_WAIT = 1,  /* spin arg ns on %globaltimer, r = 0             */
  TD_BODY_COMPUTE = 2,    /* 64-lane u64 LCG, arg iterations                */
  TD_BODY_STENCIL2D = 3,  /* 2D tile update (config 5), see td_stencil2d    */
  TD_BODY_EXT_PRE = 4,    /* wait ext precondition flag arg   */
  TD_BODY_EXT_POST = 5,   /* raise ext postcondition flag arg */
  TD_BODY_MEMORY = 6      /* memory_bound: stream arg u64 words (a multiple of 64) through the
                             worker's scratch (store, load back, XOR fold); td_graph_attach_scratch */
};

/* Launch flags. */
enum {
  TD_F_CHECKSUM = 1u << 0,  /* fold tokens into per-column checksums       */
  TD_F_STATS = 1u << 1,     /* per-execution message accounting            */
  TD_F_TALLY = 1u << 2,     /* per-node execution tally (exactly-once)     */
  TD_F_QUEUE = 1u << 3,     /* allow stream-queued launches before a wait  */
  TD_F_TRACE = 1u << 4,    /* per-node %globaltimer trace (td_graph_trace) */
  TD_F_DYNAMIC = 1u << 5   /* arrival-order dispatch: per-SM ready queues (needs TD_UPLOAD_DYNAMIC) */
};

/* Upload options (td_csr.options). */
enum {
  TD_UPLOAD_DYNAMIC = 1u << 0  /* also build the node-indexed programs and per-SM ready queues of the
                                  arrival-order mode (dispatch when a counter hits 0) */
};

/*
 * Flattened graph (replaces Alg. 1's per-worker (V_w, E_w), PAPER.md:650-658,
 * SPEC.md WorkerProgram 356-359).  Node ids are dense.
 * Neighbour lists are sorted, disjoint, inclusive id intervals stored as
 * (lo, hi) int32 pairs; interval k of node v is iv[2k], iv[2k+1] for
 * ptr[v] <= k < ptr[v+1].  All arrays are borrowed for the upload call only.
 */
typedef struct td_csr {
  int64_t n_nodes;
  const int64_t* pred_ptr;  /* [n_nodes+1] */
  const int32_t* pred_iv;   /* [2*pred_ptr[n]] ascending predecessor ids  */
  const int64_t* succ_ptr;  /* [n_nodes+1] */
  const int32_t* succ_iv;   /* [2*succ_ptr[n]]                            */
  const uint8_t* kind;      /* [n_nodes] TD_BODY_*                        */
  const uint32_t* arg;      /* [n_nodes]                                  */
  int32_t n_workers;        /* static owners (Alg. 1 resources)           */
  const int64_t* work_ptr;  /* [n_workers+1]                              */
  const int32_t* work;      /* [n_nodes] per-worker lists, topological    */
  int32_t n_cols;           /* checksum columns (0 = none)                */
  const int32_t* col;       /* [n_nodes] column of node, -1 = none        */
  /* sharding: NULL / n_ranks=1 for one GPU */
  int32_t n_ranks;
  int32_t my_rank;
  const uint8_t* node_rank; /* [n_nodes] shard owning each node            */
  int32_t n_ext_pre;        /* external precondition flags                */
  int32_t n_ext_post;       /* external postcondition flags               */
  /* [n_nodes] identity of each node (NULL = its own id).  A node whose
   * identity is another node u is a replica of u: it computes u's token from
   * the same inputs (halo replication of a sharded lowering, shard.py). */
  const int32_t* ident;
  uint32_t options;         /* TD_UPLOAD_* */
} td_csr;

typedef struct td_launch_params {
  uint64_t seed;
  uint32_t flags;           /* TD_F_* */
  uint32_t threads_per_block; /* 0 = default (128) */
  uint64_t spin_limit;      /* 0 = unbounded; else poisoned after this many polls */
} td_launch_params;

typedef struct td_stats {
  uint64_t executed;            /* nodes executed in the last execution   */
  uint64_t cross_worker_edges;  /* COMPLETED_EDGE messages  */
  uint64_t local_decrements;    /* same-worker decrements  */
  uint64_t init_messages;       /* workers started  */
  uint64_t cross_rank_edges;    /* of cross_worker_edges, over NVLink     */
  uint64_t epoch;               /* executions completed on this graph     */
  int32_t poisoned;             /* nonzero if the last execution failed   */
  int32_t workers;              /* resident workers (warps) launched      */
  int32_t blocks;               /* CTAs launched                          */
  int32_t threads_per_block;
} td_stats;

typedef struct td_device_info {
  int32_t sm_count;
  int32_t l2_bytes;
  int32_t max_workers;       /* co-resident warps for the executor kernel */
  int32_t max_workers_st2d;  /* ... for the config-5 tile-body kernel      */
  int32_t cc_major, cc_minor;
  char name[96];
} td_device_info;

typedef struct td_graph td_graph;

/* How an uploaded graph was lowered (introspection; no reference analogue). */
typedef struct td_graph_info {
  int64_t n_nodes;
  int64_t n_positions;      /* descriptors (nodes of this shard + relays)   */
  int64_t n_shared;         /* shared mailbox replicas per bank (bundling)  */
  int32_t n_workers;        /* resident warps launched (graph + relays)     */
  int32_t n_graph_workers;
  int32_t n_ranks, my_rank;
  int32_t plain;            /* 1: the PLAIN kernel (no ext/bundle/pool paths) */
  int32_t group;            /* K nodes per warp pass (2 or 4), 0 = one node */
  int32_t has_stencil2d;
  int32_t desc_bytes;       /* bytes per node descriptor                    */
  int32_t slot_shift;       /* mailbox words are 2^slot_shift u64 apart     */
  int32_t n_combiners;      /* combiner words of bundled groups (one GPU)   */
} td_graph_info;

/* Last error message of this thread (static storage). */
const char* td_last_error(void);

/* Device and kernel limits; replaces MachineSpec validation (machine.py:75-84). */
td_status td_device_info_get(int32_t device, uint32_t threads_per_block, td_device_info* out);

/* compile(g) -> CompiledGraph: copy the
 * flattened graph to device, allocate counters/tokens, validate owners. */
td_status td_graph_upload(const td_csr* csr, int32_t device, td_graph** out);

/* execute(cg, pre): ONE persistent
 * kernel per replay on `stream` (cudaStream_t as void*, NULL = legacy). */
td_status td_graph_launch(td_graph* g, const td_launch_params* p, void* stream);

/* wait(done): returns TD_E_WAIT_TIMEOUT after timeout_s
 * (< 0 = forever), TD_E_POISONED if the execution failed. */
td_status td_graph_wait(td_graph* g, double timeout_s);

/* Non-blocking completion query: *done = 1 when the last execution finished. */
td_status td_graph_query(td_graph* g, int32_t* done);

/* Host-side external precondition trigger: flag i := epoch+1. */
td_status td_graph_trigger_pre(td_graph* g, int32_t index);

/* Postcondition j of the current execution has fired. */
td_status td_graph_post_fired(td_graph* g, int32_t index, int32_t* fired);

/* memory_image (machine.py:395-397) analogue: D2H copy of all node tokens. */
td_status td_graph_tokens(td_graph* g, uint64_t* host_tokens, int64_t n);

/* Per-column checksum fold of the last execution. */
td_status td_graph_checksums(td_graph* g, uint64_t* host_cols, int32_t n_cols);

/* Per-node execution tally (exactly-once invariant). */
td_status td_graph_tally(td_graph* g, uint32_t* host_tally, int64_t n);

/* message_stats(cg) plus launch geometry. */
td_status td_graph_stats(td_graph* g, td_stats* out);

/* Per-node timestamps of the last TD_F_TRACE execution: 4 x u64 per node
 * (wait start, dependences observed, inputs gathered, successors signalled),
 * %globaltimer ns.  The profiling hook of SURVEY.md §5 "Tracing". */
td_status td_graph_trace(td_graph* g, uint64_t* host, int64_t n);

/* Re-parameterise every COMPUTE / BUSY_WAIT body of the resident graph to
 * `arg` (Task Bench varies only the work per task). */
td_status td_graph_set_body_arg(td_graph* g, uint32_t arg);

/* Lowering summary of an uploaded graph (kernel variant, group size). */
td_status td_graph_info_get(td_graph* g, td_graph_info* out);

/* Device time of the last execution in ms (CUDA events around the kernel). */
td_status td_graph_last_ms(td_graph* g, float* ms);

/* Multi-GPU (sharded lowering): export this
 * shard's counter/token/flag buffers as CUDA IPC handles (opaque bytes) and
 * map a peer shard's.  Cross-shard edges then become direct P2P token stores
 * plus release-ordered counter increments into the peer's memory. */
td_status td_graph_ipc_export(td_graph* g, void* out, size_t cap, size_t* len);
td_status td_graph_ipc_attach(td_graph* g, int32_t rank, const void* handle, size_t len);
/* Same wiring for shards of ONE process on different devices (SPEC.md:483:
 * shards as processor groups of one process): peer access + direct pointers. */
td_status td_graph_peer_attach_direct(td_graph* g, int32_t rank, td_graph* peer);

/* Config-5 mini-app (BASELINE configs[4]): attach the double-buffered nx x ny
 * u32 grid that TD_BODY_STENCIL2D nodes update in 64x64 tiles.  Node v is
 * (t, tile) with v = t*ntiles + ty*(nx/64) + tx; t=0 initialises the grid,
 * step t reads buffer (t-1)&1 and writes buffer t&1.  Call before
 * td_graph_ipc_export when sharded (halo rows of a peer's tiles are read from
 * the peer's grid over NVLink). */
td_status td_graph_attach_stencil2d(td_graph* g, int32_t nx, int32_t ny);
td_status td_graph_stencil2d_grid(td_graph* g, int32_t buf, uint32_t* host, int64_t n);

/* Per-worker scratch for TD_BODY_MEMORY nodes (Task Bench memory_bound):
 * words_per_worker u64 (a multiple of 64) for every worker; required before
 * launching a graph with memory_bound nodes (their arg must not exceed it). */
td_status td_graph_attach_scratch(td_graph* g, int64_t words_per_worker);

/* Free device resources; safe on NULL. */
td_status td_graph_destroy(td_graph* g);

/*
 * Per-task launch runtime: the generic path that compiled replay replaces
 * (task_rt.launch; Fig. 6, 298-331).  One kernel
 * launch per task, ordered by one CUDA stream; used for untraced / memoized
 * issue in the implicit frontend and as the "one
 * kernel per task" comparator of PAPER.md:954-955.  Tokens live in a device
 * slot array of fixed capacity; a task reads its predecessors' slots.
 */
#define TD_RT_MAX_PREDS 480
typedef struct td_rt td_rt;
td_status td_rt_create(int32_t device, int64_t capacity, td_rt** out);
td_status td_rt_launch_task(td_rt* rt, int64_t slot, uint64_t key, uint8_t kind, uint32_t arg,
                            uint64_t seed, const int64_t* pred_slots, int32_t n_pred);
/* Import n tokens computed elsewhere (a compiled replay of a trace) into
 * runtime slots, so untraced tasks issued afterwards can consume them; keys
 * are the producing ops' token keys (trace-local index). */
td_status td_rt_store_tokens(td_rt* rt, const int64_t* slots, const uint64_t* keys, const uint64_t* tokens,
                             int32_t n);
td_status td_rt_sync(td_rt* rt);
td_status td_rt_tokens(td_rt* rt, int64_t first, int64_t n, uint64_t* host);
td_status td_rt_destroy(td_rt* rt);

#ifdef __cplusplus
}
#endif
#endif /* TDEXEC_H */
