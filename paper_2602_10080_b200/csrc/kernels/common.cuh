// common.cuh — shared device vocabulary of the MLMQ engine (sm_100a).
//
// Distance kinds, queue elements, memory-ordering helpers and the kernel parameter
// block.  Reference vocabulary: core.py:14-32 (Element, INF, defaults).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mlmq {

constexpr unsigned FULL = 0xFFFFFFFFu;

// Persistent-kernel launch shape: MLMQ_WPB warps per CTA, MLMQ_MINB CTAs per SM
// (the register budget follows: 65536 / (32 * WPB * MINB) rounded to the allocator).
#ifndef MLMQ_WPB
#define MLMQ_WPB 9
#endif
#ifndef MLMQ_MINB
#define MLMQ_MINB 2
#endif
constexpr int kWarpsPerBlockMax = MLMQ_WPB;
#ifndef MLMQ_F32_WPB
#define MLMQ_F32_WPB MLMQ_WPB
#endif
// The f32-distance kernels are compiled with MLMQ_WPB = MLMQ_F32_WPB (Makefile): C5 measured
// 6.59 -> 6.20 ms with 10-warp CTAs (20 warps/SM), while the u32 kernels lose with them
// (C2 1.39 -> 1.80 ms, C4 19.1 -> 31.5 ms), so only dk = f32 uses it.
constexpr int kF32WarpsPerBlock = MLMQ_F32_WPB;

// MLMQ_ASYNC=1: the flattened expansion stages the next step's adjacency into shared
// memory with cp.async (LDGSTS) while the current step runs, so two steps of DRAM loads
// are in flight per lane without holding them in registers.  Per-warp staging: two
// buffers of 32 x MLMQ_U (col, w) pairs.
#ifndef MLMQ_ASYNC
#define MLMQ_ASYNC 0
#endif
#ifndef MLMQ_U
#define MLMQ_U 4
#endif
constexpr int kAdjStageBytes = MLMQ_ASYNC ? 2 * 32 * MLMQ_U * 8 + 16 : 0;

// Debug hooks (phase profile, wait states, uniformity checks) exist only in the debug
// library (make debug -> libmlmq_debug.so, loaded when MLMQ_DEBUG=1).
#ifdef MLMQ_DEBUG_HOOKS
constexpr bool kDebug = true;
#else
constexpr bool kDebug = false;
#endif

// Device distance kinds.  The API domain is u64 with INF = 2^64-1 (core.py:17-18);
// the engine runs u32 when the result provably (or, optimistically, actually) fits,
// and f32 for float-weight graphs.
enum { DK_U32 = 0, DK_U64 = 1, DK_F32 = 2 };
// L2 kernel families: FIFO ring, bucket (Δ window over rings), batch heap
// (priority = one heap, multi = pnum heaps).
enum { L2K_FIFO = 0, L2K_BUCKET = 1, L2K_HEAP = 2 };
enum { L1K_VECTOR = 0, L1K_NEAR_FAR = 1, L1K_FILTER = 2, L1K_SLF = 3 };

enum {
  ERR_NONE = 0,
  ERR_OVERFLOW = 1,      // ring slot stayed busy (l2.py:116-135)
  ERR_ABORT = 2,         // host watchdog abort (engine.py:267-272)
  ERR_HEAP_OVERFLOW = 3, // batch-heap node pool exhausted
  ERR_HUB_OVERFLOW = 4,  // hub work ring slot stayed busy
  ERR_CORRUPT = 5,       // a queue element named a vertex >= n (internal error)
  ERR_OBOX = 6           // sharded solve: remote-update outbox full
};

// Control block: u64 words, every hot word on its own 128-byte line.
enum : int {
  C_DONE = 0,             // global_done (l2.py:33-70), in queue units
  C_STOP = 16,            // work flag cleared by the manager (engine.py:152-169)
  C_GEN = 17,             // work generation (same 16-byte pair as C_STOP: one idle poll)
  C_ERR = 32,             // ERR_* code
  C_EPOCH = 48,           // bucket floor index (l2.py:181-301)
  C_HUB_WP = 64,          // hub descriptor tickets issued
  C_HUB_RP = 80,          // oldest hub descriptor that may still have chunks
  C_DIST_OVF = 96,        // optimistic u32 distance overflowed
  C_LOCAL_NONEMPTY = 112, // audit: sum of L0+L1 sizes at exit (engine.py:233-237)
  C_DIAG = 128,           // overflow diagnostics: ring, slot, write_ptr, read_ptr
  C_HUB_ITEMS = 144,      // hub items pushed
  C_IDLE = 160,           // number of groups currently idle (demand signal for eager spill)
  C_HUB_RES = 176,        // hub chunks reserved (termination units)
  C_WORDS = 192
};

// Per-group metric slots, in METRIC_FIELDS order (core.py:142-154).
enum {
  M_RELAX = 0, M_UPD, M_L0E, M_L0D, M_L1E, M_L1D, M_L2E, M_L2D, M_L2A, M_FLUSH, M_SETTLED,
  M_COUNT
};
// Debug-only phase profile slots (per warp, clock64 cycles / counts), MLMQ_DEBUG=1.
enum {
  P_L0L1 = 0, P_HUB, P_L2R, P_RELAX, P_L2W, P_IDLE, P_NBATCH, P_BATCHSUM, P_NL2R, P_NL2W,
  P_SPINS, P_CASFAIL, P_L2WELEMS, P_TOTAL, P_HEAD, P_STEPS, P_COUNT
};
constexpr int kMetSlots = 32;  // M_COUNT metric slots + P_COUNT profile slots (smem, per warp)
constexpr int kProfBase = 16;
// Debug wait-state codes written to wstate[gid] >> 56
enum { W_NONE = 0, W_RING_WRITE = 1, W_RING_READ = 2, W_HUB_READ = 3, W_HUB_WRITE = 4, W_HEAP = 5 };

template <int K> struct DT;

template <> struct DT<DK_U32> {
  using S = uint32_t;
  static constexpr uint32_t INF = 0xFFFFFFFFu;
  __device__ __forceinline__ static S add(S a, uint32_t w, bool& ovf) {
    uint64_t s = (uint64_t)a + w;
    if (s >= 0xFFFFFFFFull) { ovf = true; return INF; }
    return (S)s;
  }
  // saturating add for thresholds (NF / F rebases); never produces INF
  __device__ __forceinline__ static S add_thr(S a, S b) {
    uint64_t s = (uint64_t)a + b;
    return s >= 0xFFFFFFFFull ? (S)0xFFFFFFFEu : (S)s;
  }
};

template <> struct DT<DK_U64> {
  using S = unsigned long long;
  static constexpr unsigned long long INF = ~0ull;
  __device__ __forceinline__ static S add(S a, uint32_t w, bool& ovf) {
    S s = a + w;
    if (s < a || s == INF) { ovf = true; return INF; }
    return s;
  }
  __device__ __forceinline__ static S add_thr(S a, S b) {
    S s = a + b;
    return (s < a || s == INF) ? INF - 1 : s;
  }
};

// f32 distances live as their IEEE bit patterns; for non-negative floats the unsigned
// order of the bits is the numeric order, so atomicMin on u32 is a float min.
template <> struct DT<DK_F32> {
  using S = uint32_t;
  static constexpr uint32_t INF = 0x7f800000u;  // +inf
  __device__ __forceinline__ static S add(S a, uint32_t w, bool&) {
    return __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(w)));
  }
  __device__ __forceinline__ static S add_thr(S a, S b) {
    return __float_as_uint(__fadd_rn(__uint_as_float(a), __uint_as_float(b)));
  }
};

// Queue element (core.py:14): (vertex id, tentative distance at enqueue time).
template <class S> struct Elem;
template <> struct __align__(8) Elem<uint32_t> {
  uint32_t v, d;
};
template <> struct __align__(16) Elem<unsigned long long> {
  uint32_t v, pad;
  unsigned long long d;
};

// Hub work item: an edge range of one high-degree vertex (new tier).
struct __align__(16) HubItem {
  unsigned long long lo, hi;
  unsigned long long du;  // distance snapshot (S bits)
  uint32_t u, pad;
};

// ---------------------------------------------------------------------------------
// memory-ordering helpers (PTX memory model, gpu scope unless noted)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// host-mapped pinned word written by the host watchdog
__device__ __forceinline__ uint32_t ld_sys_u32(const volatile uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// L2-coherent (L1-bypassing) element loads for queue storage that is reused.
__device__ __forceinline__ Elem<uint32_t> ld_cg_elem(const Elem<uint32_t>* p) {
  uint2 r = __ldcg(reinterpret_cast<const uint2*>(p));
  Elem<uint32_t> e;
  e.v = r.x;
  e.d = r.y;
  return e;
}
__device__ __forceinline__ Elem<unsigned long long> ld_cg_elem(const Elem<unsigned long long>* p) {
  uint4 r = __ldcg(reinterpret_cast<const uint4*>(p));
  Elem<unsigned long long> e;
  e.v = r.x;
  e.pad = 0;
  e.d = ((unsigned long long)r.w << 32) | r.z;
  return e;
}
// Adjacency (col, w) load.  MLMQ_ADJ_HINT: 0 read-only path (__ldg), 1 cache-streaming
// (__ldcs), 2 (default) L1 no-allocate + L2 evict-first policy, so the streamed adjacency
// does not push the distance array and row offsets out of L2 (B200: C2 1.42 -> 1.41 ms,
// C4 20.8 -> 20.3 ms, C5 7.01 -> 6.85 ms; profiles/r2_experiments.md).
#ifndef MLMQ_ADJ_HINT
#define MLMQ_ADJ_HINT 2
#endif
__device__ __forceinline__ uint2 ld_adj(const uint2* p) {
#if MLMQ_ADJ_HINT == 1
  return __ldcs(p);
#elif MLMQ_ADJ_HINT == 2
  uint2 r;
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
      : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  return r;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ uint32_t ldcg_dist(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ldcg_dist(const unsigned long long* p) { return __ldcg(p); }

__device__ __forceinline__ void red_add(unsigned long long* a, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
// 16-byte relaxed load of two adjacent control words
__device__ __forceinline__ void ld_relaxed_v2(const unsigned long long* p, unsigned long long& a,
                                              unsigned long long& b) {
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* a) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}
// atomic min without a return value (RED.MIN at L2)
__device__ __forceinline__ void red_min(uint32_t* a, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void red_min(unsigned long long* a, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// ---------------------------------------------------------------------------------
// kernel parameter block
// ---------------------------------------------------------------------------------
struct KParams {
  // graph (device CSR; adjacency interleaved as (col, weight bits))
  const unsigned long long* off;
  const uint2* adj;
  unsigned long long n;
  void* dist;  // S[n]
  unsigned long long source;

  // resolved config (engine.py:57-103)
  int L;            // lanes_per_group
  int l0cap;        // l0_capacity
  int l1type;       // L1K_*
  int l1cap;        // l1 capacity
  int wb;           // flush period
  int th_v;         // cooperative threshold
  int dup;          // duplicate elimination
  int unit;         // unit weights
  int bs;           // block_size
  int bmax, bnum;   // bucket window
  int nb;           // heap node batch (<= 32)
  int pnum;         // number of heaps (multi)
  int G;            // worker groups (warps); warp G is the manager
  unsigned long long delta_nf_s;  // thresholds in distance encoding (S bits)
  unsigned long long filter_f_s;
  unsigned long long delta_i;     // bucket Δ, integer kinds
  double delta_f;                 // bucket Δ, f32 kind

  // L2 rings: nrings rings of bn slots; slot = bs elements
  unsigned long long* seq;   // [nrings * bn]
  uint32_t* cnt;             // [nrings * bn]
  void* data;                // [nrings * bn * bs] elements
  unsigned long long* ptrs;  // per ring: wp at [r*32], rp at [r*32+16]
  unsigned long long bn_mask;
  int nrings;

  // batch heaps
  uint32_t* hlock;              // [pnum * 32]
  unsigned long long* hsize;    // [pnum * 16]
  unsigned long long* hwc;      // [pnum * 16] element write counter (termination units)
  void* hnodes;                 // [pnum * hcap * 32] elements
  uint32_t* hcnt;               // [pnum * hcap]
  unsigned long long hcap;      // nodes per heap

  // hub work ring
  unsigned long long* hub_seq;
  HubItem* hub_data;              // descriptors: lo, hi, du, u, pad = nch
  unsigned long long* hub_next;   // claim words: ticket << 24 | chunks claimed
  uint32_t* hub_fin;              // chunks completed
  unsigned long long hub_mask;
  unsigned long long hub_chunk;
  unsigned long long hub_thresh;

  // control
  unsigned long long* ctl;
  const volatile uint32_t* host_abort;
  unsigned long long* metrics;  // [G * M_COUNT]
  unsigned long long* prof;     // debug: [G * P_COUNT] or null
  unsigned long long* wstate;   // debug: [G] current wait (code << 56 | ticket) or null
  unsigned long long spin_timeout_ns;
  int smem_per_warp;            // bytes
  int share;                    // eager spill to L2 when groups are idle (B200 extension)
  int fifo_park;                // FIFO readers take unconditional tickets
  int bscratch;                 // bucket writes use the per-warp histogram scratch (bmax <= 256)
  int bwin;                     // bucket window: winners >= bwin buckets above the floor skip L0/L1 (0 = off)
  int batch_cap, out_cap, spill_cap;  // elements
  int far_cap;                  // far staging elements (bucket window), 0 when unused
  // light/heavy split (FIFO L2, unsharded): rows are partitioned light-first; an expanded
  // vertex relaxes its light edges at once and defers the heavy ones to a token in ring 1
  int heavy;                    // 1: split on
  const uint32_t* nlight;       // [n] light edges at the head of each row
  int hvy_cap;                  // heavy-token staging elements per group (smem)
  int heavy_min;                // defer only rows with at least this many heavy edges
  int l1_want;                  // elements per L1 read (reference: lanes_per_group)
  int adj_prefetch;             // prefetch adjacency list heads into L2 at batch start
  long long ring_margin;        // bucket rings: pending blocks kept free for racing writers

  // 1D-partitioned shard; nparts == 1 for an unpartitioned graph
  int nparts;                   // P (power of two)
  int part_shift;               // log2 P
  uint32_t rank;                // this shard
  void* ghost;                  // S[n_global]: ghost distances of remote vertices
  uint2* obox;                  // outbox of remote improvements (global v, d)
  unsigned long long* obox_n;   // outbox fill
  unsigned long long obox_cap;
};

// Queue harness launch arguments (queue_harness.cu; mlmq_queue_* in include/mlmq.h).
struct HarnessArgs {
  int mode;                          // 0 write op, 1 read op, 2 stress
  int group;                         // op mode: the calling group (multi: queue group % pnum)
  const uint2* in;                   // op write: (v, d) pairs
  unsigned long long n_in;
  uint2* out;                        // read pairs
  unsigned long long* out_n;         // fill of `out`
  unsigned long long out_cap;
  int* cursors;                      // multi: persistent per-group write cursor (l2.py:424)
  int writers, readers;              // stress: warp gid < readers reads, the rest write
  unsigned long long w_stride, w_begin, w_end;  // writer w writes ids [w*stride+begin, w*stride+end)
  unsigned long long stop_at;        // readers stop once out_n >= stop_at
  unsigned long long* epoch_log;     // bucket: [reader * log_cap + k] floor seen at read k
  unsigned long long log_cap;
  unsigned long long* log_n;         // per reader
};

}  // namespace mlmq
