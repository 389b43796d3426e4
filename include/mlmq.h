/*
 * mlmq.h — C ABI of libmlmq.so, the B200 (sm_100a) Multi-Level-Multi-Queue SSSP engine.
 *
 * The reference (arxiv/paper_2602_10080, package `mlq_sssp`) has no FFI boundary: its
 * operator API is the Python function
 *     mlq_sssp.engine.sssp_solve(graph, source, config, engine, *, features,
 *                                unit_weights, watchdog_s) -> SsspResult
 * (pkg/src/mlq_sssp/engine.py:245-297).  Every entry point below replaces one piece of
 * that function's body; the Python host package (paper_2602_10080_b200, re-exported as
 * `mlq_sssp`) binds them through ctypes exactly as INTEGRATION.md shows.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / CUDA types in signatures;
 *   - all device memory is owned by the library, all host buffers by the caller;
 *   - every function returns an mlmq_status (0 = OK); mlmq_last_error() returns a
 *     thread-local message for the last failing call on this thread;
 *   - one solve in flight per mlmq_graph (internal mutex); distinct graphs may solve
 *     concurrently.
 */
#ifndef MLMQ_H
#define MLMQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MLMQ_ABI_VERSION 1

/* Status codes; the Python shim maps them onto the reference's exception types. */
typedef enum {
  MLMQ_OK = 0,
  MLMQ_EINVAL = 1,     /* ValueError         (core.py:107-136, core.py:199-200)            */
  MLMQ_EOVERFLOW = 2,  /* QueueOverflowError (l2.py:116-135)                               */
  MLMQ_EENGINE = 3,    /* EngineError: watchdog / audit (engine.py:229-242, 267-279)       */
  MLMQ_ECUDA = 4,      /* EngineError: CUDA runtime failure / no device                    */
  MLMQ_ENOMEM = 5,     /* EngineError: device allocation failed                            */
  MLMQ_EFORMAT = 6,    /* GraphFormatError (loaders, core.py:49-51)                         */
  MLMQ_ENEGATIVE = 7,  /* NegativeWeightError (loaders, core.py:53-54)                      */
  MLMQ_EIO = 8,        /* the file cannot be opened or read (OSError)                       */
  MLMQ_EFALLBACK = 9   /* input the native loader does not restate exactly (e.g. Python's
                          "1_000" integer syntax, weights >= 2^32): use the Python reader */
} mlmq_status;

/* Weight storage kinds accepted by mlmq_graph_create. */
typedef enum {
  MLMQ_W_U32 = 0,  /* integer weights (graph.py:18-36 `weights`, all >= 0, < 2^32) */
  MLMQ_W_F32 = 1,  /* float32 weights >= 0 (extension: config 5, no reference analogue) */
  MLMQ_W_UNIT = 2  /* every weight is 1 (engine.py:125 unit_weights / bfs_solve) */
} mlmq_weight_kind;

/* Queue type codes, in the order of core.py:20-21 (L1_TYPES, L2_TYPES). */
enum { MLMQ_L1_VECTOR = 0, MLMQ_L1_NEAR_FAR = 1, MLMQ_L1_FILTER = 2, MLMQ_L1_SLF = 3 };
enum { MLMQ_L2_FIFO = 0, MLMQ_L2_BUCKET = 1, MLMQ_L2_PRIORITY = 2, MLMQ_L2_MULTI = 3 };

/* Device distance width selection. */
enum { MLMQ_DIST_AUTO = 0, MLMQ_DIST_U32 = 1, MLMQ_DIST_U64 = 2 };

/*
 * Resolved configuration: MlmqConfig + L1Params + L2Params + EngineConfig after
 * resolve_config (engine.py:57-103).  Integer-semantics fields (delta_nf, filter_f,
 * delta) are doubles so the f32 path can carry unrounded values.
 */
typedef struct {
  int32_t l1_type, l2_type;         /* MLMQ_L1_*, MLMQ_L2_*                           */
  int32_t l0_capacity;              /* core.py:24  (GPU: 1..16)                       */
  int32_t l1_capacity;              /* core.py:25                                     */
  int32_t wb;                       /* core.py:26  0 disables the periodic flush      */
  double delta_nf;                  /* L1 near/far Δ (l1.py:139-189)                  */
  double filter_f;                  /* L1 filter bound F (l1.py:192-242)              */
  double delta;                     /* L2 bucket width Δ (l2.py:181-301)              */
  int32_t block_size;               /* core.py:28                                     */
  int64_t block_num;                /* core.py:29  treated as a LOWER bound on GPU    */
  int32_t bmax, bnum;               /* core.py:30-31                                  */
  int32_t node_batch;               /* core.py:32                                     */
  int32_t pnum;                     /* l2.py:416-451 (already clamped by the caller)  */
  int32_t num_groups;               /* one warp per group; <= 0 means "auto"          */
  int32_t lanes_per_group;          /* 1..32                                          */
  int32_t th_v;                     /* engine.py:195 cooperative-expansion threshold  */
  int32_t dup_elim;                 /* EngineConfig.duplicate_elimination             */
  int32_t unit_weights;             /* engine.py:125                                  */
  int32_t dist_mode;                /* MLMQ_DIST_*                                    */
  double watchdog_s;                /* engine.py:267-279; <= 0 disables               */
  double spin_timeout_s;            /* ring-slot wait before QueueOverflowError (l2.py:94) */
  int32_t hub_chunk;                /* edges per hub chunk (0 = library default 2048) */
  int32_t share;                    /* 1: eager L1/L0 write-back while groups are idle */
  int32_t fifo_park;                /* 1: FIFO readers take unconditional tickets      */
  int32_t bucket_window;            /* bucket L2: winners >= this many buckets above the
                                       floor bypass L0/L1 (0 = reference cascade)       */
  int32_t read_batch;               /* elements per L1 read (0 = lanes_per_group, the
                                       reference's `want`); up to max(block_size, 32)   */
  int32_t hub_threshold;            /* lists longer than this become hub descriptors
                                       (0 = 4 x hub_chunk)                              */
  int32_t test_capacity;            /* > 0: every queue store (ring slots, hub descriptors,
                                       heap nodes) gets exactly this many entries -- a
                                       test hook that forces the overflow paths (l2.py:116-135) */
  int32_t flags;                    /* MLMQ_F_* engine extensions (0 = none)             */
  int32_t heavy_delta;              /* FIFO L2, integer weights: edges with w < heavy_delta
                                       are relaxed when a vertex is expanded, the rest
                                       later from a deferred "heavy token" (0 = off)      */
  float heavy_delta_f;              /* the same threshold for f32 weights (0 = off)       */
} mlmq_config_t;

/* mlmq_config_t.flags */
enum { MLMQ_F_PREFETCH_TARGETS = 1 /* prefetch row offsets of improved targets into L2 */ };
/* bits 8..23 of flags: light/heavy split -- defer the heavy edges of a row only when it has
 * at least this many of them (smaller rows relax all edges at once) */
#define MLMQ_F_HEAVY_MIN_SHIFT 8

/*
 * Aggregate counters; the first 11 fields follow core.py:142-154 (METRIC_FIELDS),
 * wall_time_us is core.py:176.  The rest are GPU-side extras kept outside the schema.
 */
typedef struct {
  uint64_t relaxations, distance_updates, l0_enqueues, l0_dequeues, l1_enqueues,
      l1_dequeues, l2_enqueues, l2_dequeues, l2_atomic_ops, flushes, settled_reads;
  uint64_t wall_time_us;
  double kernel_ms;        /* cudaEvent: init kernel start -> audit kernel end     */
  uint64_t num_groups;     /* groups (warps) actually launched                     */
  uint64_t hub_items;      /* hub edge-range work items pushed                     */
  uint32_t dist_bits;      /* 32 or 64: device distance width that produced result */
  uint32_t reruns;         /* 1 if an optimistic u32 run overflowed and re-ran u64 */
} mlmq_metrics_t;

#define MLMQ_GROUP_METRIC_FIELDS 11

typedef struct mlmq_graph mlmq_graph;

/* Library / device info. */
int mlmq_abi_version(void);
const char* mlmq_last_error(void);
int mlmq_device_count(int* out);
int mlmq_device_info(int device, int* sm_count, size_t* free_bytes, size_t* total_bytes);

/*
 * Graph upload (replaces handing the CsrGraph lists to _Run, engine.py:109-125).
 * Copies row_offsets[n+1], col[m] and (unless UNIT) w[m] to device memory of `device`.
 */
int mlmq_graph_create(const uint64_t* row_offsets, const uint32_t* col, const void* w,
                      int weight_kind, uint64_t n, uint64_t m, int device,
                      mlmq_graph** out);
void mlmq_graph_destroy(mlmq_graph* g);
int mlmq_graph_device_bytes(const mlmq_graph* g, uint64_t* out);

/*
 * Number of groups "auto" resolves to for this config on this graph's device:
 * SM count x resident warps per SM, given the config's shared-memory footprint.
 */
int mlmq_auto_groups(const mlmq_graph* g, const mlmq_config_t* cfg, int32_t* out);

/*
 * One SSSP solve (engine.py:245-297).  dist_out: caller-allocated n entries, INF =
 * UINT64_MAX.  group_metrics (optional, may be NULL): caller-allocated
 * num_groups x MLMQ_GROUP_METRIC_FIELDS u64, in METRIC_FIELDS order.
 * Raises (returns) EINVAL for a bad source (core.py:199-200).
 */
int mlmq_sssp(mlmq_graph* g, uint64_t source, const mlmq_config_t* cfg,
              uint64_t* dist_out, mlmq_metrics_t* metrics_out, uint64_t* group_metrics,
              uint64_t group_metrics_cap);

/* Float-weight solve (graph created with MLMQ_W_F32); INF = +inf. */
int mlmq_sssp_f32(mlmq_graph* g, uint64_t source, const mlmq_config_t* cfg,
                  float* dist_out, mlmq_metrics_t* metrics_out, uint64_t* group_metrics,
                  uint64_t group_metrics_cap);

/*
 * Device-resident variant for benchmarking: runs the solve but leaves distances on
 * the device (no D2H); returns kernel time in metrics_out->kernel_ms.
 */
int mlmq_sssp_device(mlmq_graph* g, uint64_t source, const mlmq_config_t* cfg,
                     mlmq_metrics_t* metrics_out);

/* Page-locked host memory for result buffers: D2H into it runs at full PCIe/C2C speed
 * (the Python shim recycles these buffers across solves). */
int mlmq_host_alloc(uint64_t bytes, void** out);
void mlmq_host_free(void* p);

/* Copy the last solve's device distances (as stored: u32/u64 words) to the host. */
int mlmq_last_dist(mlmq_graph* g, uint64_t* dist_out);

/*
 * Reachability summary of the last solve: V_reach = #{dist < INF},
 * E_reach = sum of out-degrees over reached vertices.
 */
int mlmq_reach(mlmq_graph* g, uint64_t* v_reach, uint64_t* e_reach);

/*
 * Sharded solve (the reference has none -- PAPER.md:797 names a multi-GPU
 * "L3 queue" as future work).  1D vertex partition: shard `rank` of `nparts` (a power of
 * two <= 64) owns global vertices v with v mod nparts == rank, stored at local id
 * v / nparts.  row_offsets/w are the owned rows in local order; col holds GLOBAL ids.
 * A solve is a sequence of supersteps driven by the host (one process per GPU,
 * exchanging the send buffers with an all-to-all):
 *   mlmq_shard_begin(g)                        dist = ghost = INF
 *   mlmq_shard_step(g, cfg, inbox, n_in, ...)  apply the inbox (device pairs of (global v,
 *       d) owned by this shard, e.g. (source, 0) on its owner for the first step), run K1 to
 *       local quiescence, then write the remote improvements grouped by owner into the
 *       caller's DEVICE buffer d_send (send_cap pairs) and their per-owner counts into
 *       send_counts[nparts] (host).  The solve is done when no shard sends anything.
 * Distances: mlmq_last_dist (local order), mlmq_reach (this shard's V/E_reach).
 */
int mlmq_shard_create(const uint64_t* row_offsets, const uint32_t* col, const void* w, int weight_kind,
                      uint64_t n_local, uint64_t m_local, uint64_t n_global, uint32_t rank,
                      uint32_t nparts, int device, mlmq_graph** out);
int mlmq_shard_begin(mlmq_graph* g);
/* The cudaStream_t the library runs g's kernels on (as void*), so a caller can order its
 * own stream (NCCL's) against it with events instead of host synchronisation. */
int mlmq_graph_stream(mlmq_graph* g, void** out);
int mlmq_shard_step(mlmq_graph* g, const mlmq_config_t* cfg, const uint32_t* d_inbox, uint64_t n_in,
                    uint32_t* d_send, uint64_t send_cap, uint64_t* send_counts,
                    mlmq_metrics_t* metrics_out);

/*
 * K4: the 8 selector features (graph.py:428-460) as exact integer sums:
 * out[0]=n out[1]=m out[2]=sum deg out[3]=sum deg^2 (lo) out[4]=sum deg^2 (hi)
 * out[5]=max deg out[6]=sum w out[7]=sum w^2 (lo) out[8]=sum w^2 (hi) out[9]=max w.
 * (float weights: out[6..9] are the bit patterns of double sums / max.)
 */
int mlmq_feature_sums(mlmq_graph* g, uint64_t out[10]);

/*
 * Seeded generators bit-compatible with the reference's CPython-random generators
 * (graph.py:306-420) followed by build_csr (graph.py:89-124).  key/keylen are the
 * 32-bit little-endian limbs of |seed| (CPython random_seed; seed 0 -> {0}).
 * mlmq_gen_size reports (n, m) so the caller can allocate; mlmq_gen_graph fills them.
 * kind: 0 grid2d, 1 path, 2 uniform, 3 rmat.
 */
typedef struct {
  int64_t rows, cols;        /* grid2d                      */
  int64_t n, m;              /* path (n) / uniform (n, m)   */
  int64_t scale, edge_factor;/* rmat                        */
  double a, b, c, d;         /* rmat quadrant probabilities */
  int64_t wmin, wmax;
} mlmq_gen_params_t;

enum { MLMQ_GEN_GRID2D = 0, MLMQ_GEN_PATH = 1, MLMQ_GEN_UNIFORM = 2, MLMQ_GEN_RMAT = 3 };

int mlmq_gen_size(int kind, const mlmq_gen_params_t* p, uint64_t* n_out, uint64_t* m_out);
int mlmq_gen_graph(int kind, const mlmq_gen_params_t* p, const uint32_t* key, uint64_t keylen,
                   uint64_t* row_offsets, uint32_t* col, uint32_t* w);

/* One shard of a generated graph (sharded.py shard_csr layout): rows u with
 * u % nparts == rank at local id u / nparts, global column ids, from the same RNG stream
 * (each rank generates only its own slice: no rank holds the whole graph).  Call twice:
 * first with col == NULL (fills row_offsets[n_local + 1] and *m_out), then with col / w
 * of *m_out entries. */
int mlmq_gen_shard(int kind, const mlmq_gen_params_t* p, const uint32_t* key, uint64_t keylen,
                   uint32_t nparts, uint32_t rank, uint64_t* row_offsets, uint32_t* col, uint32_t* w,
                   uint64_t* m_out);

/* Stable CSR build from an edge list (graph.py:89-124 ordering; zero-weight self loops
 * dropped).  Returns m_kept via *m_out; caller allocates row_offsets[n+1], col[m], w[m]. */
int mlmq_build_csr(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                   const uint32_t* w, uint64_t* row_offsets, uint32_t* col, uint32_t* w_out,
                   uint64_t* m_out);

/*
 * Float weights for config 5: U[0,1) f32 from a seeded counter-based stream
 * (splitmix64 of seed ^ edge index; no reference analogue).
 */
int mlmq_gen_f32_weights(uint64_t m, uint64_t seed, float* w_out);

/*
 * Native graph readers (graph.py:132-175 load_dimacs, graph.py:185-257 load_matrix_market):
 * same acceptance rules, messages and edge order, then the build_csr counting sort.
 *   mlmq_load_*  -> an owned host CSR; mlmq_csr_size / mlmq_csr_copy read it out
 *   (row_offsets[n+1], col[m], w[m]); mlmq_csr_free releases it.
 */
typedef struct mlmq_csr mlmq_csr;
int mlmq_load_dimacs(const char* path, mlmq_csr** out);
int mlmq_load_matrix_market(const char* path, int64_t weight_scale, mlmq_csr** out);
int mlmq_csr_size(const mlmq_csr* c, uint64_t* n, uint64_t* m);
int mlmq_csr_copy(const mlmq_csr* c, uint64_t* row_offsets, uint32_t* col, uint32_t* w);
void mlmq_csr_free(mlmq_csr* c);

/*
 * Device queue harness: one L2 queue (l2.py:73-451) in device memory, driven by the same
 * device code the solve kernel runs.  Replaces the reference's Python queue objects
 * L2BlockFifo / L2Bucket / L2PriorityQueue / L2MultiQueue (l2.py:73, 181, 304, 416) for
 * its queue tests (pkg/tests/test_l2_queues.py, test_acceptance.py:282).
 *   write: one write(batch, group) of n (v, d) pairs (l2.py:96-114, 224-233, 322-344, 430-438)
 *   read : one try_read(group) -> up to one block / 32 heap elements (l2.py:161-166, 235-292,
 *          362-389, 440-442)
 *   stats: out[0] resident elements, [1] claimed-but-unconsumed tickets, [2] structurally
 *          empty, [3] bucket epoch (floor = epoch * delta), [4] heap property holds,
 *          [5] write tickets, [6] read tickets, [7..7+min(pnum,32)) elements per heap
 *   stress: `writers` warps write ids [w*stride+begin, w*stride+end) with d = f(id) while
 *          `readers` warps read until `stop_at` elements were consumed; every element read
 *          is appended to pairs_out (v, d) (cap pairs); bucket readers log the epoch of each
 *          read (epochs_out[reader * log_cap + k], counts in log_n[reader]).
 */
typedef struct mlmq_queue mlmq_queue;
typedef struct {
  int32_t l2_type;        /* MLMQ_L2_*                                          */
  int32_t block_size;     /* elements per ring block                            */
  int64_t block_num;      /* ring slots (rounded up to a power of two)          */
  double delta;           /* bucket width                                       */
  int32_t bmax, bnum;     /* bucket ring count / read window                    */
  int32_t node_batch;     /* heap node size (<= 32)                             */
  int32_t pnum;           /* heaps of the multi queue                           */
  int32_t num_groups;     /* group ids that may call (multi write cursors)      */
  int32_t reserved0;
  int64_t heap_nodes;     /* node pool per heap (0 = 65536)                     */
  double spin_timeout_s;  /* slot wait before QueueOverflowError                */
} mlmq_queue_params_t;

int mlmq_queue_create(int device, const mlmq_queue_params_t* params, mlmq_queue** out);
void mlmq_queue_destroy(mlmq_queue* q);
int mlmq_queue_write(mlmq_queue* q, const uint32_t* pairs, uint64_t n, int32_t group);
int mlmq_queue_read(mlmq_queue* q, int32_t group, uint32_t* pairs_out, uint64_t cap, uint64_t* n_out);
int mlmq_queue_stats(mlmq_queue* q, uint64_t out[40]);
int mlmq_queue_stress(mlmq_queue* q, int32_t writers, int32_t readers, uint64_t stride, uint64_t begin,
                      uint64_t end, uint64_t stop_at, uint32_t* pairs_out, uint64_t cap, uint64_t* n_out,
                      uint64_t* epochs_out, uint64_t log_cap, uint64_t* log_n, double* ms_out);

#ifdef __cplusplus
}
#endif

#endif /* MLMQ_H */
