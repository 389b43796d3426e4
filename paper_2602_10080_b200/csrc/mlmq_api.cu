// mlmq_api.cu — the C ABI of include/mlmq.h: graph upload, workspace management,
// solve orchestration (K3 init -> K1/K2 persistent kernel -> K5 audit), the host
// watchdog, error mapping, features and reachability.
//
// Replaces the body of sssp_solve (pkg/src/mlq_sssp/engine.py:245-297): _Run
// construction (:109-125), bootstrap (compose.py:92-101), worker/manager threads
// (:260-265), watchdog (:267-279), audit (:229-242) and metric merge (:285-297).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/mlmq.h"
#include "kernels/aux_kernels.cuh"
#include "kernels/common.cuh"

namespace mlmq {

const void* kernel_dk0_l0_c4_q0();
const void* kernel_dk0_l0_c4_q1();
const void* kernel_dk0_l0_c4_q2();
const void* kernel_dk0_l0_c4_q3();
const void* kernel_dk0_l0_c16_q0();
const void* kernel_dk0_l0_c16_q1();
const void* kernel_dk0_l0_c16_q2();
const void* kernel_dk0_l0_c16_q3();
const void* kernel_dk0_l1_c4_q0();
const void* kernel_dk0_l1_c4_q1();
const void* kernel_dk0_l1_c4_q2();
const void* kernel_dk0_l1_c4_q3();
const void* kernel_dk0_l1_c16_q0();
const void* kernel_dk0_l1_c16_q1();
const void* kernel_dk0_l1_c16_q2();
const void* kernel_dk0_l1_c16_q3();
const void* kernel_dk0_l2_c4_q0();
const void* kernel_dk0_l2_c4_q1();
const void* kernel_dk0_l2_c4_q2();
const void* kernel_dk0_l2_c4_q3();
const void* kernel_dk0_l2_c16_q0();
const void* kernel_dk0_l2_c16_q1();
const void* kernel_dk0_l2_c16_q2();
const void* kernel_dk0_l2_c16_q3();
const void* kernel_dk1_l0_c4_q0();
const void* kernel_dk1_l0_c4_q1();
const void* kernel_dk1_l0_c4_q2();
const void* kernel_dk1_l0_c4_q3();
const void* kernel_dk1_l0_c16_q0();
const void* kernel_dk1_l0_c16_q1();
const void* kernel_dk1_l0_c16_q2();
const void* kernel_dk1_l0_c16_q3();
const void* kernel_dk1_l1_c4_q0();
const void* kernel_dk1_l1_c4_q1();
const void* kernel_dk1_l1_c4_q2();
const void* kernel_dk1_l1_c4_q3();
const void* kernel_dk1_l1_c16_q0();
const void* kernel_dk1_l1_c16_q1();
const void* kernel_dk1_l1_c16_q2();
const void* kernel_dk1_l1_c16_q3();
const void* kernel_dk1_l2_c4_q0();
const void* kernel_dk1_l2_c4_q1();
const void* kernel_dk1_l2_c4_q2();
const void* kernel_dk1_l2_c4_q3();
const void* kernel_dk1_l2_c16_q0();
const void* kernel_dk1_l2_c16_q1();
const void* kernel_dk1_l2_c16_q2();
const void* kernel_dk1_l2_c16_q3();
const void* kernel_dk2_l0_c4_q0();
const void* kernel_dk2_l0_c4_q1();
const void* kernel_dk2_l0_c4_q2();
const void* kernel_dk2_l0_c4_q3();
const void* kernel_dk2_l0_c16_q0();
const void* kernel_dk2_l0_c16_q1();
const void* kernel_dk2_l0_c16_q2();
const void* kernel_dk2_l0_c16_q3();
const void* kernel_dk2_l1_c4_q0();
const void* kernel_dk2_l1_c4_q1();
const void* kernel_dk2_l1_c4_q2();
const void* kernel_dk2_l1_c4_q3();
const void* kernel_dk2_l1_c16_q0();
const void* kernel_dk2_l1_c16_q1();
const void* kernel_dk2_l1_c16_q2();
const void* kernel_dk2_l1_c16_q3();
const void* kernel_dk2_l2_c4_q0();
const void* kernel_dk2_l2_c4_q1();
const void* kernel_dk2_l2_c4_q2();
const void* kernel_dk2_l2_c4_q3();
const void* kernel_dk2_l2_c16_q0();
const void* kernel_dk2_l2_c16_q1();
const void* kernel_dk2_l2_c16_q2();
const void* kernel_dk2_l2_c16_q3();

static thread_local char g_err[1024] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

}  // namespace mlmq

using namespace mlmq;

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t _e = (call);                                                         \
    if (_e != cudaSuccess) {                                                         \
      set_last_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, \
                     __LINE__, cudaGetErrorString(_e));                              \
      return MLMQ_ECUDA;                                                             \
    }                                                                                \
  } while (0)

namespace {

constexpr int kOutCap = 32 * 8 + 32;  // L - 1 carried + 32 lanes x U (<= 8) winners
constexpr int kAuditWords = 14;

struct Workspace {
  int es = 0, bs = 0, nrings = 0, nheaps = 0;
  unsigned long long bn = 0, hcap = 0, hub_cap = 0;
  bool exact = false;  // sized by the test_capacity hook
  unsigned long long* seq = nullptr;
  uint32_t* cnt = nullptr;
  void* data = nullptr;
  unsigned long long* ptrs = nullptr;
  uint32_t* hlock = nullptr;
  unsigned long long* hsize = nullptr;
  unsigned long long* hwc = nullptr;
  void* hnodes = nullptr;
  uint32_t* hcnt = nullptr;
  unsigned long long* hub_seq = nullptr;
  HubItem* hub_data = nullptr;
  unsigned long long* hub_next = nullptr;
  uint32_t* hub_fin = nullptr;
  bool dirty = true;
  size_t bytes = 0;
};

void ws_free(Workspace& w) {
  cudaFree(w.seq);
  cudaFree(w.cnt);
  cudaFree(w.data);
  cudaFree(w.ptrs);
  cudaFree(w.hlock);
  cudaFree(w.hsize);
  cudaFree(w.hwc);
  cudaFree(w.hnodes);
  cudaFree(w.hcnt);
  cudaFree(w.hub_seq);
  cudaFree(w.hub_data);
  cudaFree(w.hub_next);
  cudaFree(w.hub_fin);
  w = Workspace();
}

unsigned long long next_pow2(unsigned long long x) {
  unsigned long long p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace

struct mlmq_graph {
  int device = 0;
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  unsigned long long n = 0, m = 0;
  int wkind = MLMQ_W_U32;
  unsigned long long* d_off = nullptr;
  uint2* d_adj = nullptr;
  void* d_dist = nullptr;               // n x 8 bytes
  unsigned long long* d_dist64 = nullptr;  // widen buffer
  unsigned long long* d_ctl = nullptr;
  unsigned long long* d_audit = nullptr;
  unsigned long long* d_metrics = nullptr;
  unsigned long long metrics_cap = 0;
  unsigned long long* d_scratch = nullptr;  // 16 words for features / reach
  unsigned long long* d_prof = nullptr;     // MLMQ_DEBUG: per-warp phase profile
  unsigned long long* d_wstate = nullptr;   // MLMQ_DEBUG: per-warp wait state
  unsigned long long prof_cap = 0;
  uint32_t* h_abort = nullptr;
  uint32_t* d_abort = nullptr;
  Workspace ws;
  int last_dk = -1;
  bool poisoned = false;  // a kernel did not stop after an abort: the handle is unusable
  uint32_t* d_nlight = nullptr;  // light/heavy split: light edges at the head of each row
  uint32_t part_bits = 0;        // threshold (weight bits) the rows are partitioned by
  bool part_valid = false;
  bool l2win_set = false, l2win_failed = false;  // apply_l2_window state
  // vertex relabeling (ensure_relabel): device id = perm[caller id]; state 0 undecided,
  // 1 relabeled, 2 kept in caller order
  uint32_t* d_perm = nullptr;
  std::vector<uint32_t> h_perm;
  int relabel_state = 0;
  unsigned long long hot_n = 0;  // relabeled: the prefix of vertices that takes 95 % of the edge targets
  void* d_gather = nullptr;  // caller-order copy of the distances (n x 8 bytes)
  // per-vertex arrays packed into one buffer [off | nlight | dist] so one persisting L2
  // window covers every random per-vertex load of K1 (pack_vertex_arrays)
  void* d_vtx = nullptr;
  size_t vtx_bytes = 0;
  uint32_t* h_stage = nullptr;           // pinned staging of u32 results (copy_dist_u64)
  unsigned long long stage_cap = 0;
  cudaEvent_t chunk_ev[8] = {};
  std::mutex mu;
  // sharded solve: 1D partition, v -> shard v mod P, local id v / P
  uint32_t nparts = 1, rank = 0;
  int shift = 0;
  unsigned long long n_global = 0;
  void* d_ghost = nullptr;                // S[n_global]
  uint2* d_obox = nullptr;                // remote-update outbox
  unsigned long long obox_cap = 0;
  uint2* d_seeds = nullptr;               // improved inbox entries (<= inbox size)
  unsigned long long seeds_cap = 0;
  unsigned long long* d_sscratch = nullptr;  // [0] outbox fill [1] seed count [8..] counts [72..] cursors
};

// Inputs/outputs of one superstep of a sharded solve.
struct ShardIo {
  const uint2* inbox = nullptr;
  unsigned long long n_in = 0;
  uint2* send = nullptr;
  unsigned long long send_cap = 0;
  uint64_t* send_counts = nullptr;  // host [nparts]
};

namespace mlmq {
int harness_launch(int l2k, const KParams& p, const HarnessArgs& h, int warps, int wpb, size_t smem_per_warp,
                   cudaStream_t stream);
}

namespace {

const void* kernel_for(int dk, int l2k, int cm, int l1) {
  using Fn = const void* (*)();
  static const Fn table[3][3][2][4] = {
    {{{kernel_dk0_l0_c4_q0, kernel_dk0_l0_c4_q1, kernel_dk0_l0_c4_q2, kernel_dk0_l0_c4_q3}, {kernel_dk0_l0_c16_q0, kernel_dk0_l0_c16_q1, kernel_dk0_l0_c16_q2, kernel_dk0_l0_c16_q3}}, {{kernel_dk0_l1_c4_q0, kernel_dk0_l1_c4_q1, kernel_dk0_l1_c4_q2, kernel_dk0_l1_c4_q3}, {kernel_dk0_l1_c16_q0, kernel_dk0_l1_c16_q1, kernel_dk0_l1_c16_q2, kernel_dk0_l1_c16_q3}}, {{kernel_dk0_l2_c4_q0, kernel_dk0_l2_c4_q1, kernel_dk0_l2_c4_q2, kernel_dk0_l2_c4_q3}, {kernel_dk0_l2_c16_q0, kernel_dk0_l2_c16_q1, kernel_dk0_l2_c16_q2, kernel_dk0_l2_c16_q3}}},
    {{{kernel_dk1_l0_c4_q0, kernel_dk1_l0_c4_q1, kernel_dk1_l0_c4_q2, kernel_dk1_l0_c4_q3}, {kernel_dk1_l0_c16_q0, kernel_dk1_l0_c16_q1, kernel_dk1_l0_c16_q2, kernel_dk1_l0_c16_q3}}, {{kernel_dk1_l1_c4_q0, kernel_dk1_l1_c4_q1, kernel_dk1_l1_c4_q2, kernel_dk1_l1_c4_q3}, {kernel_dk1_l1_c16_q0, kernel_dk1_l1_c16_q1, kernel_dk1_l1_c16_q2, kernel_dk1_l1_c16_q3}}, {{kernel_dk1_l2_c4_q0, kernel_dk1_l2_c4_q1, kernel_dk1_l2_c4_q2, kernel_dk1_l2_c4_q3}, {kernel_dk1_l2_c16_q0, kernel_dk1_l2_c16_q1, kernel_dk1_l2_c16_q2, kernel_dk1_l2_c16_q3}}},
    {{{kernel_dk2_l0_c4_q0, kernel_dk2_l0_c4_q1, kernel_dk2_l0_c4_q2, kernel_dk2_l0_c4_q3}, {kernel_dk2_l0_c16_q0, kernel_dk2_l0_c16_q1, kernel_dk2_l0_c16_q2, kernel_dk2_l0_c16_q3}}, {{kernel_dk2_l1_c4_q0, kernel_dk2_l1_c4_q1, kernel_dk2_l1_c4_q2, kernel_dk2_l1_c4_q3}, {kernel_dk2_l1_c16_q0, kernel_dk2_l1_c16_q1, kernel_dk2_l1_c16_q2, kernel_dk2_l1_c16_q3}}, {{kernel_dk2_l2_c4_q0, kernel_dk2_l2_c4_q1, kernel_dk2_l2_c4_q2, kernel_dk2_l2_c4_q3}, {kernel_dk2_l2_c16_q0, kernel_dk2_l2_c16_q1, kernel_dk2_l2_c16_q2, kernel_dk2_l2_c16_q3}}}};
  return table[dk][l2k][cm <= 4 ? 0 : 1][l1]();
}

int l2_kind(int l2_type) {
  switch (l2_type) {
    case MLMQ_L2_FIFO: return L2K_FIFO;
    case MLMQ_L2_BUCKET: return L2K_BUCKET;
    default: return L2K_HEAP;
  }
}

int validate(const mlmq_config_t* c) {
  if (c->l1_type < 0 || c->l1_type > 3) { set_last_error("unknown l1_type code %d", c->l1_type); return MLMQ_EINVAL; }
  if (c->l2_type < 0 || c->l2_type > 3) { set_last_error("unknown l2_type code %d", c->l2_type); return MLMQ_EINVAL; }
  if (c->l0_capacity < 1 || c->l0_capacity > 16) { set_last_error("l0_capacity must be in [1, 16] on the GPU engine (got %d)", c->l0_capacity); return MLMQ_EINVAL; }
  if (c->l1_capacity < 1) { set_last_error("l1 capacity must be >= 1"); return MLMQ_EINVAL; }
  if (c->wb < 0) { set_last_error("wb must be >= 0 (0 disables periodic flushing)"); return MLMQ_EINVAL; }
  if (c->lanes_per_group < 1 || c->lanes_per_group > 32) { set_last_error("lanes_per_group must be in [1, 32] on the GPU engine (got %d)", c->lanes_per_group); return MLMQ_EINVAL; }
  if (c->th_v < 0) { set_last_error("th_v must be >= 0"); return MLMQ_EINVAL; }
  if (c->block_size < 1 || c->block_size > 4096 || c->block_num < 1) { set_last_error("block_size must be in [1, 4096] and block_num >= 1"); return MLMQ_EINVAL; }
  if (c->bmax < 1 || c->bnum < 1 || c->bmax > 4096) { set_last_error("bmax and bnum must be >= 1 (bmax <= 4096)"); return MLMQ_EINVAL; }
  if (c->bnum > c->bmax) { set_last_error("bnum must not exceed bmax"); return MLMQ_EINVAL; }
  if (c->node_batch < 1) { set_last_error("node_batch must be >= 1"); return MLMQ_EINVAL; }
  if (c->l2_type == MLMQ_L2_BUCKET && !(c->delta > 0)) { set_last_error("bucket delta must be > 0"); return MLMQ_EINVAL; }
  if (c->l2_type == MLMQ_L2_MULTI && c->pnum < 1) { set_last_error("pnum must be >= 1"); return MLMQ_EINVAL; }
  return MLMQ_OK;
}

struct LaunchShape {
  const void* fn = nullptr;
  int dk = 0, l2k = 0, cm = 4;
  int smem_per_warp = 0, wpb = 0;
  int batch_cap = 0, spill_cap = 0, far_cap = 0, hvy_cap = 0;
  int max_groups = 0;
  int bscratch = 0;
};

// The light/heavy split applies to the FIFO L2 (whole graphs and shards); returns the
// threshold as weight bits (0 = off).
uint32_t heavy_bits(const mlmq_graph* g, const mlmq_config_t* c) {
  if (c->l2_type != MLMQ_L2_FIFO || c->unit_weights || g->wkind == MLMQ_W_UNIT) return 0;
  if (g->wkind == MLMQ_W_F32) {
    if (!(c->heavy_delta_f > 0.f)) return 0;
    uint32_t b;
    std::memcpy(&b, &c->heavy_delta_f, 4);
    return b;
  }
  return c->heavy_delta > 0 ? (uint32_t)c->heavy_delta : 0u;
}

// Partition every row light-first for threshold bits h (once per threshold; the edge order
// within a row never changes a distance).
int ensure_partition(mlmq_graph* g, uint32_t h) {
  if (g->part_valid && g->part_bits == h) return MLMQ_OK;
  if (g->n >= 0x80000000ull) { set_last_error("the light/heavy split needs fewer than 2^31 vertices"); return MLMQ_EINVAL; }
  if (!g->d_nlight) CK(cudaMalloc(&g->d_nlight, std::max<size_t>(4, g->n * 4)));
  if (g->m) {
    uint2* tmp = nullptr;
    cudaError_t e = cudaMalloc(&tmp, g->m * 8);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_last_error("light/heavy partition: %s", cudaGetErrorString(e));
      return MLMQ_ENOMEM;
    }
    partition_rows_kernel<<<8 * g->sm_count, 256, 0, g->stream>>>(g->d_off, g->d_adj, tmp, g->d_nlight, g->n, h);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(g->stream));
    cudaFree(g->d_adj);
    g->d_adj = tmp;
  } else {
    CK(cudaMemsetAsync(g->d_nlight, 0, g->n * 4, g->stream));
  }
  g->part_bits = h;
  g->part_valid = true;
  return MLMQ_OK;
}

// Vertex order in HBM (B200 layout, not an algorithm change).  On a power-law graph most
// edges target a few hubs scattered over the id space (RMAT/Kronecker ids carry the skew
// in every bit), so K1's random dist[v] prefilter loads and RED mins pull a 32-byte sector
// for one 4-byte word and miss L2 once dist outgrows it (C4: 268 MB, 5x B_alg of DRAM
// reads).  Renumbering the vertices by in-degree class (hottest first; stable, so ties keep
// the caller's order; never-targeted vertices last) packs the hot words into a dense,
// L2-resident prefix.  Done once per graph on the device at the first unpartitioned solve:
// in-degrees (warp-aggregated atomics), an 8-bit class key, a stable radix sort (CUB) of
// the vertex ids by key, the new row offsets (scan) and the rows copied with their targets
// renamed.  Sources map through perm, results gather back to caller order, so the ABI is
// unchanged.  Auto policy: only when the graph is skewed (max in-degree >= 32 x mean) and
// its distance words fill half of L2 (n x 4 B >= 64 MiB: C4 20.3 -> 19.0 ms, 18.1 ms with
// the hot-prefix L2 window; C5 6.58 -> 6.51 ms; C2, whose 16.8 MB of distances stay
// L2-resident anyway, measured 1.40 -> 1.57 ms relabeled, so it keeps the caller order);
// MLMQ_RELABEL=0/1 forces it off/on.
int ensure_relabel(mlmq_graph* g) {
  if (g->relabel_state) return MLMQ_OK;
  const char* env = getenv("MLMQ_RELABEL");
  const int force = env ? atoi(env) : -1;
  if (force == 0 || g->nparts > 1 || g->n < 2 || g->m == 0 || g->n >= 0xFFFFFFFFull ||
      (force < 0 && g->n * 4ull < (64ull << 20))) {
    g->relabel_state = 2;
    return MLMQ_OK;
  }
  const unsigned long long n = g->n, m = g->m;
  uint32_t *indeg = nullptr, *val = nullptr, *iperm = nullptr, *perm = nullptr;
  uint8_t *key = nullptr, *key2 = nullptr;
  unsigned long long *noff = nullptr;
  uint2* nadj = nullptr;
  void* tmp = nullptr;
  size_t tb1 = 0, tb2 = 0;
  int st = MLMQ_OK;
  unsigned int mx = 0;
  auto fail = [&](cudaError_t e, const char* what) {
    cudaGetLastError();
    set_last_error("vertex relabel (%s): %s", what, cudaGetErrorString(e));
    st = e == cudaErrorMemoryAllocation ? MLMQ_ENOMEM : MLMQ_EENGINE;
  };
#define RL(x, what)                          \
  do {                                       \
    cudaError_t e_ = (x);                    \
    if (e_ != cudaSuccess) { fail(e_, what); goto done; } \
  } while (0)
  {
    const int blocks = (int)std::min<unsigned long long>(16ull * g->sm_count, (std::max(n, m) + 255) / 256 + 1);
    RL(cudaMalloc(&indeg, n * 4), "alloc");
    RL(cudaMemsetAsync(indeg, 0, n * 4, g->stream), "memset");
    RL(cudaMemsetAsync(g->d_scratch, 0, 8, g->stream), "memset");
    indeg_kernel<<<blocks, 256, 0, g->stream>>>(g->d_adj, m, indeg);
    RL(cudaMalloc(&key, n), "alloc");
    RL(cudaMalloc(&val, n * 4), "alloc");
    relabel_keys_kernel<<<blocks, 256, 0, g->stream>>>(indeg, n, key, val, (unsigned int*)g->d_scratch);
    RL(cudaGetLastError(), "launch");
    RL(cudaMemcpyAsync(&mx, g->d_scratch, 4, cudaMemcpyDeviceToHost, g->stream), "copy");
    {  // the hot prefix: classes in key order until 95 % of the in-edges are covered
      unsigned long long* cm = nullptr;
      RL(cudaMalloc(&cm, 512 * 8), "alloc");
      cudaMemsetAsync(cm, 0, 512 * 8, g->stream);
      class_mass_kernel<<<blocks, 256, 0, g->stream>>>(indeg, key, n, cm, cm + 256);
      std::vector<unsigned long long> hm(512);
      cudaError_t e = cudaMemcpyAsync(hm.data(), cm, 512 * 8, cudaMemcpyDeviceToHost, g->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
      cudaFree(cm);
      RL(e, "class mass");
      unsigned long long acc = 0, cnt = 0;
      for (int k = 0; k < 256 && (double)acc < 0.95 * (double)m; ++k) {
        acc += hm[k];
        cnt += hm[256 + k];
      }
      g->hot_n = cnt;
    }
    RL(cudaStreamSynchronize(g->stream), "in-degrees");
    cudaFree(indeg);
    indeg = nullptr;
    if (force < 0 && (double)mx < 32.0 * (double)m / (double)n) {  // not skewed: keep caller order
      g->relabel_state = 2;
      goto done;
    }
    RL(cudaMalloc(&key2, n), "alloc");
    RL(cudaMalloc(&iperm, n * 4), "alloc");
    RL(cub::DeviceRadixSort::SortPairs(nullptr, tb1, key, key2, val, iperm, (int)n, 0, 8, g->stream), "sort size");
    RL(cudaMalloc(&noff, (n + 1) * 8), "alloc");
    RL(cub::DeviceScan::ExclusiveSum(nullptr, tb2, noff, noff, (int)(n + 1), g->stream), "scan size");
    RL(cudaMalloc(&tmp, std::max(tb1, tb2)), "alloc");
    RL(cub::DeviceRadixSort::SortPairs(tmp, tb1, key, key2, val, iperm, (int)n, 0, 8, g->stream), "sort");
    cudaFree(key); key = nullptr;
    cudaFree(key2); key2 = nullptr;
    cudaFree(val); val = nullptr;
    RL(cudaMalloc(&perm, n * 4), "alloc");
    relabel_perm_kernel<<<blocks, 256, 0, g->stream>>>(iperm, g->d_off, n, perm, noff);
    RL(cudaGetLastError(), "launch");
    RL(cub::DeviceScan::ExclusiveSum(tmp, tb2, noff, noff, (int)(n + 1), g->stream), "scan");
    RL(cudaMalloc(&nadj, m * 8), "alloc");
    relabel_rows_kernel<<<8 * g->sm_count, 256, 0, g->stream>>>(g->d_off, g->d_adj, iperm, perm, noff, nadj, n);
    RL(cudaGetLastError(), "launch");
    g->h_perm.resize(n);
    RL(cudaMemcpyAsync(g->h_perm.data(), perm, n * 4, cudaMemcpyDeviceToHost, g->stream), "copy");
    RL(cudaStreamSynchronize(g->stream), "rows");
    cudaFree(g->d_off);
    cudaFree(g->d_adj);
    g->d_off = noff;
    g->d_adj = nadj;
    g->d_perm = perm;
    noff = nullptr;
    nadj = nullptr;
    perm = nullptr;
    g->part_valid = false;  // the light/heavy split is per device row
    g->relabel_state = 1;
  }
done:
#undef RL
  cudaFree(indeg);
  cudaFree(key);
  cudaFree(key2);
  cudaFree(val);
  cudaFree(iperm);
  cudaFree(perm);
  cudaFree(noff);
  cudaFree(nadj);
  cudaFree(tmp);
  if (st != MLMQ_OK) g->relabel_state = 2;  // solve in caller order rather than fail
  return st;
}

// The distances in caller vertex order: d_dist itself, or (relabeled graph) a gathered copy.
const void* dist_caller_order(mlmq_graph* g, int bytes) {
  if (g->relabel_state != 1) return g->d_dist;
  if (!g->d_gather && cudaMalloc(&g->d_gather, std::max<size_t>(8, g->n * 8)) != cudaSuccess) return nullptr;
  const int blocks = (int)std::min<unsigned long long>(8ull * g->sm_count, (g->n + 255) / 256 + 1);
  if (bytes == 8)
    gather_kernel<unsigned long long><<<blocks, 256, 0, g->stream>>>((const unsigned long long*)g->d_dist,
                                                                     (unsigned long long*)g->d_gather, g->n, g->d_perm);
  else
    gather_kernel<uint32_t><<<blocks, 256, 0, g->stream>>>((const uint32_t*)g->d_dist, (uint32_t*)g->d_gather,
                                                           g->n, g->d_perm);
  return g->d_gather;
}

int launch_shape(mlmq_graph* g, const mlmq_config_t* c, int dk, LaunchShape* s) {
  s->dk = dk;
  s->l2k = l2_kind(c->l2_type);
  s->cm = c->l0_capacity <= 4 ? 4 : 16;
  s->fn = kernel_for(dk, s->l2k, s->cm, c->l1_type);
  if (!s->fn) {  // experiment libraries (make KSET=...) carry a subset of the variants
    set_last_error("kernel variant dk=%d l2=%d l0cap=%d l1=%d is not built into this library", dk, s->l2k, s->cm, c->l1_type);
    return MLMQ_EENGINE;
  }
  const int es = dk == DK_U64 ? 16 : 8;
  const int L = c->lanes_per_group;
  s->batch_cap = std::max(c->block_size, 32);
  s->spill_cap = L * c->l0_capacity + L;
  const int l1n = (c->l1_type == MLMQ_L1_NEAR_FAR ? 2 : 1) * c->l1_capacity;
  s->bscratch = (s->l2k == L2K_BUCKET && c->bmax <= 256) ? 1 : 0;
  s->far_cap = (s->l2k == L2K_BUCKET && c->bucket_window > 0 && c->bmax >= 3) ? kOutCap : 0;
  s->hvy_cap = heavy_bits(g, c) ? 256 : 0;
  long long bytes = (long long)es * (s->batch_cap + kOutCap + s->spill_cap + l1n + s->far_cap + s->hvy_cap) + kMetSlots * 8 +
                    (s->bscratch ? 20LL * c->bmax : 0LL) + 32LL * 4 + kAdjStageBytes;
  bytes = (bytes + 15) / 16 * 16;
  int max_smem_block = 0;
  CK(cudaDeviceGetAttribute(&max_smem_block, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device));
  if (bytes > max_smem_block) {
    set_last_error("queue configuration needs %lld bytes of shared memory per group; the device allows %d (reduce l1 capacity or block_size)", bytes, max_smem_block);
    return MLMQ_EINVAL;
  }
  // the kernel's static shared memory (the per-CTA idle-poll cache) comes off the top
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, s->fn));
  const int dyn_max = max_smem_block - (int)fa.sharedSizeBytes;
  if (bytes > dyn_max) {
    set_last_error("queue configuration needs %lld bytes of shared memory per group; the device allows %d (reduce l1 capacity or block_size)", bytes, dyn_max);
    return MLMQ_EINVAL;
  }
  s->smem_per_warp = (int)bytes;
  s->wpb = (int)std::min<long long>(dk == DK_F32 ? kF32WarpsPerBlock : kWarpsPerBlockMax, dyn_max / bytes);
  static std::mutex attr_mu;
  static std::unordered_set<const void*> attr_done;
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    if (!attr_done.count(s->fn)) {
      CK(cudaFuncSetAttribute(s->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
      attr_done.insert(s->fn);
    }
  }
  int bps = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, s->fn, s->wpb * 32, (size_t)s->wpb * bytes));
  if (bps < 1) { set_last_error("persistent kernel cannot be made resident for this configuration"); return MLMQ_EINVAL; }
  s->max_groups = bps * g->sm_count * s->wpb - 1;
  return MLMQ_OK;
}

int ensure_workspace(mlmq_graph* g, const mlmq_config_t* c, const LaunchShape& sh, unsigned long long hub_chunk,
                     int groups) {
  Workspace need;
  need.es = sh.dk == DK_U64 ? 16 : 8;
  need.bs = c->block_size;
  const unsigned long long n = g->n;
  if (sh.l2k == L2K_HEAP) {
    need.nrings = 0;
    need.bn = 1;
    need.nheaps = c->l2_type == MLMQ_L2_MULTI ? c->pnum : 1;
    // nodes hold <= node_batch elements: small batches need proportionally more nodes;
    // writers rotate over the heaps, so each heap gets twice its even share
    const unsigned long long nb = (unsigned long long)std::max(1, std::min(c->node_batch, 32));
    const unsigned long long total =
        std::max<unsigned long long>(65536ull, (4ull * n + 4096ull) * std::min<unsigned long long>(8ull, (32ull + nb - 1) / nb));
    need.hcap = std::max<unsigned long long>(1024ull, 2ull * total / (unsigned long long)need.nheaps);
  } else {
    need.nrings = sh.l2k == L2K_BUCKET ? c->bmax : (sh.hvy_cap ? 2 : 1);  // ring 1: heavy tokens
    const unsigned long long slots = 8ull * n / (unsigned long long)c->block_size + 16384ull;
    // bucket rings: a quarter of the FIFO ring each (the whole of it with one bucket), and
    // room for every group to race a few blocks into a ring past the occupancy check
    unsigned long long per = sh.l2k == L2K_BUCKET
                                 ? std::max<unsigned long long>(slots / (unsigned long long)std::min(4, std::max(1, c->bmax)) + 1024,
                                                                16ull * (unsigned long long)groups + 1024ull)
                                 : slots;
    need.bn = next_pow2(std::max<unsigned long long>((unsigned long long)c->block_num, per));
    need.nheaps = 0;
    need.hcap = 0;
  }
  need.hub_cap = next_pow2(2ull * g->m / hub_chunk + 4096ull);
  const bool exact = c->test_capacity > 0;  // test hook: force small stores (overflow paths)
  if (exact) {
    const unsigned long long tc = next_pow2((unsigned long long)c->test_capacity);
    if (need.nrings) need.bn = tc;
    if (need.nheaps) need.hcap = (unsigned long long)c->test_capacity;
    need.hub_cap = tc;
  }

  Workspace& w = g->ws;
  const bool fits = w.es == need.es && w.bs == need.bs && w.nrings == need.nrings &&
                    w.nheaps == need.nheaps && w.bn >= need.bn && w.hcap >= need.hcap &&
                    w.hub_cap >= need.hub_cap && w.ptrs != nullptr &&
                    (!exact ? !w.exact : (w.bn == need.bn && w.hcap == need.hcap && w.hub_cap == need.hub_cap));
  if (!fits) {
    ws_free(w);
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const double budget = 0.7 * (double)free_b;
    auto ring_bytes = [&](unsigned long long bn) {
      return (double)need.nrings * (double)bn * ((double)need.bs * need.es + 12.0);
    };
    while (need.nrings && ring_bytes(need.bn) > budget && need.bn > (unsigned long long)c->block_num && need.bn > 1024) need.bn >>= 1;
    if (need.nrings && ring_bytes(need.bn) > budget) {
      set_last_error("L2 queue rings need %.1f GB; only %.1f GB of device memory is free", ring_bytes(need.bn) / 1e9, free_b / 1e9);
      return MLMQ_ENOMEM;
    }
    const double heap_bytes = (double)need.nheaps * (double)need.hcap * (32.0 * need.es + 4.0);
    if (heap_bytes > budget) {
      need.hcap = std::max<unsigned long long>(64ull, (unsigned long long)(budget / ((double)need.nheaps * (32.0 * need.es + 4.0))));
    }
    const size_t nslots = (size_t)std::max(need.nrings, 1) * need.bn;
    cudaError_t e = cudaSuccess;
    auto alloc = [&](void** p, size_t b) {
      if (e == cudaSuccess) e = cudaMalloc(p, std::max<size_t>(b, 256));
      w.bytes += b;
    };
    w = need;
    w.exact = exact;
    w.bytes = 0;
    w.seq = nullptr;
    alloc((void**)&w.seq, nslots * 8);
    alloc((void**)&w.cnt, nslots * 4);
    alloc(&w.data, need.nrings ? nslots * (size_t)need.bs * need.es : 256);
    alloc((void**)&w.ptrs, (size_t)std::max(need.nrings, 1) * 32 * 8);
    const size_t nh = (size_t)std::max(need.nheaps, 1);
    alloc((void**)&w.hlock, nh * 32 * 4);
    alloc((void**)&w.hsize, nh * 16 * 8);
    alloc((void**)&w.hwc, nh * 16 * 8);
    alloc(&w.hnodes, need.nheaps ? nh * need.hcap * 32 * need.es : 256);
    alloc((void**)&w.hcnt, need.nheaps ? nh * need.hcap * 4 : 256);
    alloc((void**)&w.hub_seq, need.hub_cap * 8);
    alloc((void**)&w.hub_data, need.hub_cap * sizeof(HubItem));
    alloc((void**)&w.hub_next, need.hub_cap * 8);
    alloc((void**)&w.hub_fin, need.hub_cap * 4);
    if (e != cudaSuccess) {
      cudaGetLastError();
      ws_free(w);
      set_last_error("device allocation of the queue workspace failed: %s", cudaGetErrorString(e));
      return MLMQ_ENOMEM;
    }
    w.dirty = true;
  }
  if (w.dirty) {
    const size_t nslots = (size_t)std::max(w.nrings, 1) * w.bn;
    reset_queues_kernel<<<1024, 256, 0, g->stream>>>(w.seq, nslots, w.bn - 1, w.ptrs, std::max(w.nrings, 1),
                                                      w.hub_seq, w.hub_next, w.hub_fin, w.hub_cap, g->d_ctl, w.hlock, w.hsize, w.hwc,
                                                      std::max(w.nheaps, 1));
    CK(cudaGetLastError());
    w.dirty = false;
  }
  return MLMQ_OK;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

bool debug_enabled() {
  if (!kDebug) return false;
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("MLMQ_DEBUG");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// The distance array as a persisting L2 access-policy window on the library stream: the
// K1 prefilter loads of dist[v] are random and compete for L2 with the streamed adjacency.
// Default: only when the whole array fits the persisting carve-out (B200: 79 MB; C5's
// 67 MB: 6.85 -> 6.65 ms, C2 neutral; a partial window on C4's 268 MB costs 16 %).
// MLMQ_L2PERSIST=<fraction> forces a window of that fraction, 0 turns it off.
// Pack off, nlight and dist into one buffer (after the relabel and the light/heavy
// partition, which replace off/nlight) so a single persisting window can hold all three
// when they fit the carve-out together (C2: 33.5 + 16.8 + 16.8 MB).  MLMQ_VTXPACK=1.
void pack_vertex_arrays(mlmq_graph* g) {
  static const int on = [] {
    const char* e = getenv("MLMQ_VTXPACK");
    return e ? atoi(e) : 0;
  }();
  if (!on || g->d_vtx || !g->d_nlight || g->nparts > 1) return;
  const size_t ob = (g->n + 1) * 8, nb = g->n * 4, db = std::max<size_t>(8, g->n * 8);
  const size_t nb_al = (nb + 255) / 256 * 256, ob_al = (ob + 255) / 256 * 256;
  unsigned char* buf = nullptr;
  if (cudaMalloc(&buf, ob_al + nb_al + db) != cudaSuccess) { cudaGetLastError(); return; }
  if (cudaMemcpyAsync(buf, g->d_off, ob, cudaMemcpyDeviceToDevice, g->stream) != cudaSuccess ||
      cudaMemcpyAsync(buf + ob_al, g->d_nlight, nb, cudaMemcpyDeviceToDevice, g->stream) != cudaSuccess ||
      cudaStreamSynchronize(g->stream) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(buf);
    return;
  }
  cudaFree(g->d_off);
  cudaFree(g->d_nlight);
  cudaFree(g->d_dist);
  g->d_off = (unsigned long long*)buf;
  g->d_nlight = (uint32_t*)(buf + ob_al);
  g->d_dist = buf + ob_al + nb_al;
  g->d_vtx = buf;
  g->vtx_bytes = ob_al + nb_al;  // + the distance words in use
  g->l2win_set = false;
}

void apply_l2_window(mlmq_graph* g, int dk) {
  static const float frac = [] {
    const char* e = getenv("MLMQ_L2PERSIST");
    return e ? (float)atof(e) : -1.f;
  }();
  if (frac == 0.f || g->l2win_failed) return;
  int maxp = 0, maxw = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, g->device);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, g->device);
  cudaGetLastError();
  // A relabeled graph whose distances outgrow the carve-out persists only its hot prefix
  // (95 % of the edge targets): C4 19.05 -> 18.12 ms.  A whole array that fits keeps the
  // whole-array window (C5 relabeled: hot prefix only 6.62 ms vs 6.51).
  const size_t esz = dk == DK_U64 ? 8 : 4;
  size_t bytes = (size_t)g->n * esz;
  if (g->relabel_state == 1 && g->hot_n && maxp > 0 && bytes > (size_t)maxp) bytes = (size_t)g->hot_n * esz;
  void* base = g->d_dist;
  if (g->d_vtx && maxp > 0 && g->vtx_bytes + (size_t)g->n * esz <= (size_t)maxp) {  // packed [off|nlight|dist]
    base = g->d_vtx;
    bytes = g->vtx_bytes + (size_t)g->n * esz;
  }
  if (maxp <= 0 || maxw <= 0 || (frac < 0.f && (bytes > (size_t)maxp || bytes > (size_t)maxw))) {
    if (g->l2win_set) {  // a different distance kind no longer fits: drop the window
      cudaStreamAttrValue a = {};
      cudaStreamSetAttribute(g->stream, cudaStreamAttributeAccessPolicyWindow, &a);
      g->l2win_set = false;
    }
    cudaGetLastError();
    return;
  }
  const double f = frac < 0.f ? 1.0 : (double)frac;
  const size_t win = std::min(bytes, (size_t)maxw);
  const size_t lim = std::min((size_t)maxp, (size_t)(win * f));
  size_t cur = 0;
  if (cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize) != cudaSuccess || cur < lim)
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, lim);
  cudaStreamAttrValue a = {};
  a.accessPolicyWindow.base_ptr = base;
  a.accessPolicyWindow.num_bytes = win;
  a.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)lim / (double)win);
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(g->stream, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess)
    g->l2win_failed = true;  // best effort: never fail a solve over a cache hint
  else
    g->l2win_set = true;
  cudaGetLastError();
}

// MLMQ_DEBUG=1: per-phase cycle breakdown and the wait states of stuck warps.
void debug_dump(mlmq_graph* g, int G, const char* tag) {
  std::vector<unsigned long long> pr((size_t)G * P_COUNT), ws((size_t)2 * G + 8 + (size_t)G * 32 + 8192);
  std::vector<unsigned long long> ctl(C_WORDS), ptr(64);
  if (cudaMemcpy(pr.data(), g->d_prof, pr.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(ws.data(), g->d_wstate, ws.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(ctl.data(), g->d_ctl, C_WORDS * 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(ptr.data(), g->ws.ptrs, 32 * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    fprintf(stderr, "[mlmq debug] copy failed\n");
    return;
  }
  unsigned long long tot[P_COUNT] = {0};
  for (int i = 0; i < G; ++i)
    for (int f = 0; f < P_COUNT; ++f) tot[f] += pr[(size_t)i * P_COUNT + f];
  const double T = tot[P_TOTAL] ? (double)tot[P_TOTAL] : 1.0;
  fprintf(stderr,
          "[mlmq debug] %s G=%d cycles/warp=%.3g  L0L1 %.1f%%  hub %.1f%%  L2read %.1f%%  relax %.1f%% "
          "(of which L2write %.1f%%)  idle %.1f%% | batches %llu avg %.1f  L2 reads %llu  L2 writes %llu "
          "(%.1f elems avg)  search %.1f%%  endflush %.1f%% | relax: head %.1f%% steps %.1f%%\n",
          tag, G, T / G, 100 * tot[P_L0L1] / T, 100 * tot[P_HUB] / T, 100 * tot[P_L2R] / T,
          100 * tot[P_RELAX] / T, 100 * tot[P_L2W] / T, 100 * tot[P_IDLE] / T, tot[P_NBATCH],
          tot[P_NBATCH] ? (double)tot[P_BATCHSUM] / tot[P_NBATCH] : 0.0, tot[P_NL2R], tot[P_NL2W],
          tot[P_NL2W] ? (double)tot[P_L2WELEMS] / tot[P_NL2W] : 0.0, 100 * tot[P_SPINS] / T, 100 * tot[P_CASFAIL] / T,
          100 * tot[P_HEAD] / T, 100 * tot[P_STEPS] / T);
  int hist[8] = {0};
  int shown = 0;
  for (int i = 0; i < G; ++i) {
    const int code = (int)(ws[i] >> 56);
    hist[code & 7]++;
    if (code && shown < 16) {
      fprintf(stderr, "[mlmq debug]   warp %d waits code %d ticket %llu\n", i, code,
              ws[i] & ((1ull << 56) - 1));
      ++shown;
    }
  }
  fprintf(stderr, "[mlmq debug]   wait states: none %d ringW %d ringR %d hubR %d hubW %d heap %d\n",
          hist[0], hist[1], hist[2], hist[3], hist[4], hist[5]);
  int lh[128] = {0};
  shown = 0;
  for (int i = 0; i < G; ++i) {
    const unsigned long long x = ws[(size_t)G + i];
    const int ph = (int)(x >> 56);
    lh[ph & 127]++;
    if (ph != 99 && ph != 10 && shown < 24) {
      fprintf(stderr, "[mlmq debug]   warp %d phase %d l0size %llu n1 %llu n2 %llu outn %llu\n", i, ph,
              (x >> 40) & 0xFFFF, (x >> 24) & 0xFFFF, (x >> 12) & 0xFFF, x & 0xFFF);
      ++shown;
    }
  }
  fprintf(stderr, "[mlmq debug]   manager iters %llu d %llu r %llu state %llu audit %llu | ctl done %llu stop %llu err %llu epoch %llu hubwp %llu hubrp %llu idle %llu | ring0 wp %llu rp %llu | diag %llu %llu %llu %llu\n",
          ws[2 * (size_t)G], ws[2 * (size_t)G + 2], ws[2 * (size_t)G + 3], ws[2 * (size_t)G + 4], ws[2 * (size_t)G + 5],
          ctl[C_DONE], ctl[C_STOP], ctl[C_ERR], ctl[C_EPOCH], ctl[C_HUB_WP], ctl[C_HUB_RP], ctl[C_IDLE], ptr[0], ptr[16], ctl[C_DIAG], ctl[C_DIAG + 1], ctl[C_DIAG + 2], ctl[C_DIAG + 3]);
  {
    int shown2 = 0;
    for (int i = 0; i < G && shown2 < 8; ++i) {
      const unsigned long long* L = &ws[(size_t)2 * G + 8 + (size_t)i * 32];
      bool same = true;
      for (int l = 1; l < 32; ++l) same &= L[l] == L[0];
      const bool stuck = ((ws[(size_t)G + i] >> 56) != 99);
      if (!same || stuck) {
        fprintf(stderr, "[mlmq debug]   warp %d lanes:", i);
        for (int l = 0; l < 32; ++l) fprintf(stderr, " %llu", L[l]);
        fprintf(stderr, "\n");
        ++shown2;
      }
    }
  }
  {  // managed-floor epoch log: [0] count, then (timestamp << 16 | busy groups) per advance;
     // without a managed floor: the timeline ((t >> 6) << 40 | busy << 24 | outstanding)
    const unsigned long long* E = &ws[(size_t)2 * G + 8 + (size_t)G * 32];
    const unsigned long long ne = std::min<unsigned long long>(E[0], 8191);
    if (ne > 1 && ctl[C_EPOCH] == 0) {
      const double t0 = (double)(E[1] >> 40) * 64.0, t1 = (double)(E[ne] >> 40) * 64.0;
      const int NB = 24;
      double sb[NB] = {0}, so[NB] = {0};
      int cnt[NB] = {0};
      for (unsigned long long i = 1; i <= ne; ++i) {
        const double t = (double)(E[i] >> 40) * 64.0;
        int b = t1 > t0 ? (int)((t - t0) / (t1 - t0) * NB) : 0;
        b = std::min(NB - 1, std::max(0, b));
        sb[b] += (double)((E[i] >> 24) & 0xFFFF);
        so[b] += (double)(E[i] & 0xFFFFFF);
        cnt[b]++;
      }
      fprintf(stderr, "[mlmq debug]   timeline %.1f us, %llu samples (bin: busy groups / outstanding units):", (t1 - t0) / 1e3, ne);
      for (int b = 0; b < NB; ++b)
        if (cnt[b]) fprintf(stderr, " %.0f/%.0f", sb[b] / cnt[b], so[b] / cnt[b]);
        else fprintf(stderr, " -");
      fprintf(stderr, "\n");
    } else if (ne > 1) {
      std::vector<double> d;
      double busy = 0;
      for (unsigned long long i = 2; i <= ne; ++i) {
        d.push_back(((E[i] >> 16) - (E[i - 1] >> 16)) / 1e3);
        busy += (double)(E[i] & 0xFFFF);
      }
      std::sort(d.begin(), d.end());
      double s = 0;
      for (double x : d) s += x;
      fprintf(stderr, "[mlmq debug]   epochs %llu: gap us mean %.2f median %.2f p90 %.2f max %.2f; busy groups at advance %.1f\n",
              ne, s / d.size(), d[d.size() / 2], d[d.size() * 9 / 10], d.back(), busy / (ne - 1));
    }
  }
  fprintf(stderr, "[mlmq debug]   phases:");
  for (int i = 0; i < 128; ++i)
    if (lh[i]) fprintf(stderr, " %d:%d", i, lh[i]);
  fprintf(stderr, "\n");
}

// The kernel parameter block of one launch (shared by the solve and the queue harness).
KParams make_params(mlmq_graph* g, const mlmq_config_t* c, int dk, const LaunchShape& sh, int G,
                    unsigned long long hub_chunk, unsigned long long source, bool dbg) {
  KParams p;
  std::memset(&p, 0, sizeof(p));
  Workspace& w = g->ws;
  p.off = g->d_off;
  p.adj = g->d_adj;
  p.n = g->n;
  p.dist = g->d_dist;
  p.source = source;
  p.L = c->lanes_per_group;
  p.l0cap = c->l0_capacity;
  p.l1type = c->l1_type;
  p.l1cap = c->l1_capacity;
  p.wb = c->wb;
  p.th_v = c->th_v;
  p.dup = c->dup_elim;
  p.unit = c->unit_weights || g->wkind == MLMQ_W_UNIT;
  p.bs = c->block_size;
  p.bmax = c->bmax;
  p.bnum = c->bnum;
  p.nb = std::min(c->node_batch, 32);
  p.G = G;
  if (dk == DK_F32) {
    // a zero NF step would leave far elements stranded in L1: clamp to the smallest step
    float nf = c->delta_nf > 0 ? (float)c->delta_nf : 1e-30f, ff = (float)c->filter_f;
    uint32_t bnf, bff;
    std::memcpy(&bnf, &nf, 4);
    std::memcpy(&bff, &ff, 4);
    p.delta_nf_s = bnf;
    p.filter_f_s = bff;
    p.delta_f = c->delta > 0 ? c->delta : 1.0;
    p.delta_i = 1;
  } else {
    const double cap = dk == DK_U32 ? 4294967294.0 : 1.8e19;
    p.delta_nf_s = (unsigned long long)std::min(std::max(c->delta_nf, 1.0), cap);
    p.filter_f_s = (unsigned long long)std::min(std::max(c->filter_f, 0.0), cap);
    p.delta_i = (unsigned long long)std::max(1.0, c->delta);
    p.delta_f = (double)p.delta_i;
  }
  p.seq = w.seq;
  p.cnt = w.cnt;
  p.data = w.data;
  p.ptrs = w.ptrs;
  p.bn_mask = w.bn - 1;
  p.nrings = w.nrings;
  p.hlock = w.hlock;
  p.hsize = w.hsize;
  p.hwc = w.hwc;
  p.hnodes = w.hnodes;
  p.hcnt = w.hcnt;
  p.hcap = w.hcap;
  p.pnum = sh.l2k == L2K_HEAP ? w.nheaps : 0;
  p.hub_seq = w.hub_seq;
  p.hub_data = w.hub_data;
  p.hub_next = w.hub_next;
  p.hub_fin = w.hub_fin;
  p.hub_mask = w.hub_cap - 1;
  p.hub_chunk = hub_chunk;
  // lists above the threshold become hub descriptors; measured on C2 (chunk 2048):
  // threshold 4096 2.93 ms, 6144 1.53, 8192 1.51, 12288 1.55, 16384 1.63
  // (clamped so a warp's flattened expansion of 32 lists stays within int range)
  p.hub_thresh = c->hub_threshold > 0
                     ? std::min<unsigned long long>(std::max<unsigned long long>((unsigned long long)c->hub_threshold, hub_chunk),
                                                    1ull << 24)
                     : 4 * hub_chunk;
  p.ctl = g->d_ctl;
  p.host_abort = g->d_abort;
  p.metrics = g->d_metrics;
  p.prof = dbg ? g->d_prof : nullptr;
  p.wstate = dbg ? g->d_wstate : nullptr;
  const double spin = c->spin_timeout_s > 0 ? c->spin_timeout_s : 15.0;
  p.spin_timeout_ns = (unsigned long long)(spin * 1e9);
  p.smem_per_warp = sh.smem_per_warp;
  p.batch_cap = sh.batch_cap;
  p.out_cap = kOutCap;
  p.spill_cap = sh.spill_cap;
  p.far_cap = sh.far_cap;
  p.heavy = sh.hvy_cap ? 1 : 0;
  p.hvy_cap = sh.hvy_cap;
  p.heavy_min = (c->flags >> 8) & 0xFFFF;
  p.nlight = g->d_nlight;
  p.l1_want = std::max(1, std::min(c->read_batch > 0 ? c->read_batch : c->lanes_per_group, sh.batch_cap));
  p.adj_prefetch = 1 + ((c->flags & MLMQ_F_PREFETCH_TARGETS) ? 1 : 0);
  p.ring_margin = std::min<long long>((long long)w.bn / 2, 4LL * G + 64);
  p.share = c->share ? 1 : 0;
  p.fifo_park = (sh.l2k == L2K_FIFO && c->fifo_park) ? 1 : 0;
  p.bscratch = sh.bscratch;
  // a single group gains nothing from a managed floor and keeps the reference's
  // deterministic one-group schedule (test_engine.py:141-148, test_cli.py:171-179)
  p.bwin = (sh.l2k == L2K_BUCKET && c->bmax >= 3 && G > 1) ? std::max(0, c->bucket_window) : 0;
  p.nparts = (int)g->nparts;
  p.part_shift = g->shift;
  p.rank = g->rank;
  p.ghost = g->d_ghost;
  p.obox = g->d_obox;
  p.obox_n = g->d_sscratch;
  p.obox_cap = g->obox_cap;
  return p;
}

// One attempt at a given distance kind.  Returns MLMQ_OK, an error, or 100 when the
// optimistic u32 distances overflowed (caller re-runs in u64).
int run_once(mlmq_graph* g, unsigned long long source, const mlmq_config_t* c, int dk,
             mlmq_metrics_t* mo, uint64_t* gm, uint64_t gm_cap, const ShardIo* io = nullptr) {
  LaunchShape sh;
  int st = launch_shape(g, c, dk, &sh);
  if (st) return st;
  int G = c->num_groups > 0 ? c->num_groups : sh.max_groups;
  if (G > sh.max_groups) {
    set_last_error("num_groups=%d exceeds the %d groups the device keeps resident for this configuration", G, sh.max_groups);
    return MLMQ_EINVAL;
  }
  const unsigned long long hub_chunk = c->hub_chunk > 0 ? std::min<unsigned long long>((unsigned long long)c->hub_chunk, 1ull << 20) : 2048ull;
  if (!io && (st = ensure_relabel(g))) return st;
  if (g->relabel_state == 1) source = g->h_perm[source];
  if (sh.hvy_cap && (st = ensure_partition(g, heavy_bits(g, c)))) return st;
  if (sh.hvy_cap) pack_vertex_arrays(g);
  if ((st = ensure_workspace(g, c, sh, hub_chunk, G))) return st;
  if (g->metrics_cap < (unsigned long long)G) {
    cudaFree(g->d_metrics);
    g->d_metrics = nullptr;
    g->metrics_cap = 0;
    CK(cudaMalloc(&g->d_metrics, (size_t)G * M_COUNT * 8));
    g->metrics_cap = G;
  }
  Workspace& w = g->ws;
  const bool dbg = debug_enabled();
  if (dbg && g->prof_cap < (unsigned long long)G) {
    cudaFree(g->d_prof);
    cudaFree(g->d_wstate);
    CK(cudaMalloc(&g->d_prof, (size_t)G * P_COUNT * 8));
    CK(cudaMalloc(&g->d_wstate, (size_t)G * 16 + 64 + (size_t)G * 256 + 8 * 8192));
    g->prof_cap = G;
  }
  if (dbg) {
    CK(cudaMemset(g->d_prof, 0, (size_t)G * P_COUNT * 8));
    CK(cudaMemset(g->d_wstate, 0, (size_t)G * 16 + 64 + (size_t)G * 256 + 8 * 8192));
  }
  KParams p = make_params(g, c, dk, sh, G, hub_chunk, source, dbg);
  const double spin = c->spin_timeout_s > 0 ? c->spin_timeout_s : 15.0;

  if (g->poisoned) {
    set_last_error("device graph is unusable: an earlier solve did not stop after its abort");
    return MLMQ_EENGINE;
  }
  *g->h_abort = 0;
  const int blocks = (G + 1 + sh.wpb - 1) / sh.wpb;
  const int init_blocks = (int)std::min<unsigned long long>(4ull * g->sm_count, (g->n + 255) / 256 + 1);
  CK(cudaEventRecord(g->ev0, g->stream));
  const int step = io ? 1 : 0;
  if (dk == DK_U64)
    init_kernel<unsigned long long><<<init_blocks, 256, 0, g->stream>>>((unsigned long long*)g->d_dist, g->n, source, ~0ull, p, sh.l2k, step);
  else
    init_kernel<uint32_t><<<init_blocks, 256, 0, g->stream>>>((uint32_t*)g->d_dist, g->n, source,
                                                              dk == DK_F32 ? 0x7f800000u : 0xFFFFFFFFu, p, sh.l2k, step);
  CK(cudaGetLastError());
  if (io) {  // superstep: apply the inbox, seed ring 0 with the improved vertices
    CK(cudaMemsetAsync(g->d_sscratch, 0, 256 * 8, g->stream));
    if (io->n_in) {
      const int sb = (int)std::min<unsigned long long>(8ull * g->sm_count, (io->n_in + 255) / 256 + 1);
      seed_apply_kernel<uint32_t><<<sb, 256, 0, g->stream>>>(io->inbox, io->n_in, (uint32_t*)g->d_dist, g->shift, g->n,
                                                            g->d_seeds, g->d_sscratch + 1, g->d_ctl + C_ERR);
      seed_ring_kernel<uint32_t><<<2 * g->sm_count, 256, 0, g->stream>>>(g->d_seeds, g->d_sscratch + 1, p);
      seed_commit_kernel<<<1, 1, 0, g->stream>>>(g->d_sscratch + 1, p);
      CK(cudaGetLastError());
    }
  }
  apply_l2_window(g, dk);
  void* args[] = {(void*)&p};
  CK(cudaLaunchCooperativeKernel(sh.fn, dim3(blocks), dim3(sh.wpb * 32), args,
                                 (size_t)sh.wpb * sh.smem_per_warp, g->stream));
  audit_kernel<<<1, 256, 0, g->stream>>>(p, g->d_audit, p.fifo_park);
  CK(cudaGetLastError());
  if (io) {  // group the outbox by owner shard into the caller's send buffer
    const uint32_t pmask = g->nparts - 1;
    const int ob = 2 * g->sm_count;
    obox_hist_kernel<<<ob, 256, 0, g->stream>>>(g->d_obox, g->d_sscratch, g->obox_cap, g->d_sscratch + 8, pmask);
    obox_scan_kernel<<<1, 1, 0, g->stream>>>(g->d_sscratch + 8, g->d_sscratch + 72, (int)g->nparts);
    obox_scatter_kernel<<<ob, 256, 0, g->stream>>>(g->d_obox, g->d_sscratch, g->obox_cap, g->d_sscratch + 72, io->send, pmask);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(g->ev1, g->stream));

  // host watchdog (engine.py:267-279)
  const double wd = c->watchdog_s;
  if (wd > 0) {
    const double t0 = now_s();
    bool aborted = false;
    double abort_t = 0;
    for (;;) {
      cudaError_t q = cudaEventQuery(g->ev1);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) CK(q);
      const double t = now_s();
      if (!aborted && t - t0 > wd) {
        *(volatile uint32_t*)g->h_abort = 1u;
        aborted = true;
        abort_t = t;
      }
      if (aborted && t - abort_t > 5.0) {
        if (dbg) debug_dump(g, G, "stuck-after-abort");
        w.dirty = true;
        // the persistent kernel may still be resident: clearing the abort word for a new
        // solve would un-abort it, and destroy must not wait on its stream
        g->poisoned = true;
        set_last_error("worker failed to stop after abort; the device graph is no longer usable "
                       "(create a new one, or restart the process if the device stays busy)");
        return MLMQ_EENGINE;
      }
      // spin for the first 2 ms (short solves return without a sleep quantum of host
      // latency), then poll every 20 us
      if (t - t0 > 2e-3) std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  } else {
    CK(cudaEventSynchronize(g->ev1));
  }
  unsigned long long au[kAuditWords];
  CK(cudaMemcpy(au, g->d_audit, sizeof(au), cudaMemcpyDeviceToHost));
  if (dbg) {
    char tag[160];
    snprintf(tag, sizeof(tag), "l1=%d l2=%d dk=%d err=%llu done=%llu reserve=%llu epoch=%llu", c->l1_type,
             c->l2_type, dk, au[6], au[0], au[1], au[13]);
    debug_dump(g, G, tag);
  }
  const unsigned long long err = au[6];
  if (err == ERR_ABORT) {
    w.dirty = true;
    set_last_error("watchdog expired after %gs", wd);
    return MLMQ_EENGINE;
  }
  if (err == ERR_OVERFLOW) {
    w.dirty = true;
    if (au[8] >= 1000000ull)
      set_last_error("batch heap %llu lock stayed busy for %gs; the heap is likely too contended for this workload",
                     au[8] - 1000000ull, spin);
    else
      set_last_error("ring slot %llu stayed busy for %gs (block_num=%llu, write_ptr=%llu, read_ptr=%llu); block_num is likely too small for this workload",
                     au[9], spin, (unsigned long long)w.bn, au[10], au[11]);
    return MLMQ_EOVERFLOW;
  }
  if (err == ERR_HEAP_OVERFLOW) {
    w.dirty = true;
    set_last_error("batch heap %llu is full (%llu of %llu nodes); raise node_batch or reduce pnum", au[8], au[9], au[10]);
    return MLMQ_EOVERFLOW;
  }
  if (err == ERR_HUB_OVERFLOW) {
    w.dirty = true;
    set_last_error("hub work ring slot %llu stayed busy for %gs (capacity %llu)", au[9], spin, au[11]);
    return MLMQ_EOVERFLOW;
  }
  if (err == ERR_OBOX) {
    w.dirty = true;
    set_last_error("sharded solve: remote-update outbox full (%llu of %llu pairs); raise the send capacity",
                   au[8], au[9]);
    return MLMQ_EOVERFLOW;
  }
  if (err == ERR_CORRUPT) {
    w.dirty = true;
    set_last_error("internal error: corrupt queue state code=%llu value=%llu (n=%llu) group=%llu extra=%llu",
                   au[8], au[9], g->n, au[10], au[11]);
    return MLMQ_EENGINE;
  }
  if (err == 99) {
    w.dirty = true;
    set_last_error("queue ring state inconsistent at solve start");
    return 101;  // caller resets and retries
  }
  if (au[7] && dk == DK_U32) return 100;
  if (au[0] != au[1]) {
    w.dirty = true;
    set_last_error("termination audit failed: reserve=%llu done=%llu", au[1], au[0]);
    return MLMQ_EENGINE;
  }
  if (au[5] != 0) {
    w.dirty = true;
    set_last_error("termination audit failed: groups hold %llu undelivered elements", au[5]);
    return MLMQ_EENGINE;
  }
  if (au[2] || au[3] || au[4]) {
    w.dirty = true;
    set_last_error("termination audit failed: global queue not empty");
    return MLMQ_EENGINE;
  }
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
  std::vector<unsigned long long> hm((size_t)G * M_COUNT);
  CK(cudaMemcpy(hm.data(), g->d_metrics, hm.size() * 8, cudaMemcpyDeviceToHost));
  // the bootstrap write_through is charged to group 0 (compose.py:79-86, 92-101)
  hm[M_L2E] += 1;
  hm[M_L2A] += 1;
  unsigned long long tot[M_COUNT] = {0};
  for (int gi = 0; gi < G; ++gi)
    for (int f = 0; f < M_COUNT; ++f) tot[f] += hm[(size_t)gi * M_COUNT + f];
  if (mo) {
    mo->relaxations = tot[M_RELAX];
    mo->distance_updates = tot[M_UPD];
    mo->l0_enqueues = tot[M_L0E];
    mo->l0_dequeues = tot[M_L0D];
    mo->l1_enqueues = tot[M_L1E];
    mo->l1_dequeues = tot[M_L1D];
    mo->l2_enqueues = tot[M_L2E];
    mo->l2_dequeues = tot[M_L2D];
    mo->l2_atomic_ops = tot[M_L2A];
    mo->flushes = tot[M_FLUSH];
    mo->settled_reads = tot[M_SETTLED];
    mo->kernel_ms = ms;
    mo->num_groups = (uint64_t)G;
    mo->hub_items = au[12];
    mo->dist_bits = dk == DK_U64 ? 64 : 32;
  }
  if (gm) {
    const size_t cnt = std::min<size_t>((size_t)gm_cap, (size_t)G) * M_COUNT;
    std::memcpy(gm, hm.data(), cnt * 8);
  }
  if (io && io->send_counts) {
    CK(cudaMemcpy(io->send_counts, g->d_sscratch + 8, (size_t)g->nparts * 8, cudaMemcpyDeviceToHost));
    io->send_counts[g->rank] = 0;  // never produced (own vertices relax locally)
  }
  g->last_dk = dk;
  return MLMQ_OK;
}

// Host side of the result copy for 32-bit distances: the u32 array crosses PCIe in
// kChunks pieces (half the bytes of a u64 copy) and a small persistent pool of host
// threads widens piece k to u64 (0xFFFFFFFF -> 2^64-1, core.py:17-18) while piece k+1 is
// still in flight, so the caller's u64 array is ready shortly after the last byte lands.
constexpr int kChunks = 8;
struct WidenPool {
  std::vector<std::thread> th;
  std::mutex mu;
  std::condition_variable go, fin;
  const uint32_t* src = nullptr;
  uint64_t* dst = nullptr;
  unsigned long long n = 0, chunk = 0;
  cudaEvent_t* ev = nullptr;
  int device = 0, gen = 0, busy = 0;
  explicit WidenPool(int nt) {
    for (int t = 0; t < nt; ++t) th.emplace_back([this, t, nt] { loop(t, nt); });
  }
  void loop(int t, int nt) {
    int seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      go.wait(lk, [&] { return gen != seen; });
      seen = gen;
      const uint32_t* s = src;
      uint64_t* d = dst;
      const unsigned long long nn = n, ch = chunk;
      cudaEvent_t* e = ev;
      const int dev = device;
      lk.unlock();
      cudaSetDevice(dev);
      for (int k = 0; k < kChunks; ++k) {
        const unsigned long long lo = k * ch, hi = std::min(nn, lo + ch);
        if (lo >= hi) break;
        cudaEventSynchronize(e[k]);
        const unsigned long long part = (hi - lo + nt - 1) / nt;
        const unsigned long long a = lo + t * part, b = std::min(hi, a + part);
        for (unsigned long long i = a; i < b; ++i) {
          const uint32_t x = s[i];
          d[i] = x == 0xFFFFFFFFu ? ~0ull : (uint64_t)x;
        }
      }
      lk.lock();
      if (--busy == 0) fin.notify_all();
    }
  }
  std::mutex job_mu;  // one job at a time (graphs may be solved from several host threads)
  void run(const uint32_t* s, uint64_t* d, unsigned long long nn, unsigned long long ch, cudaEvent_t* e, int dev) {
    std::lock_guard<std::mutex> job(job_mu);
    std::unique_lock<std::mutex> lk(mu);
    src = s, dst = d, n = nn, chunk = ch, ev = e, device = dev;
    busy = (int)th.size();
    ++gen;
    go.notify_all();
    fin.wait(lk, [&] { return busy == 0; });
  }
};

WidenPool& widen_pool() {
  // detached workers live for the process (never joined: no shutdown-order hazards)
  static WidenPool* pool = [] {
    const unsigned hc = std::thread::hardware_concurrency();
    auto* p = new WidenPool((int)std::max(1u, std::min(8u, hc ? hc : 4u)));
    for (auto& t : p->th) t.detach();
    return p;
  }();
  return *pool;
}

int copy_dist_u64(mlmq_graph* g, uint64_t* out) {
  if (g->last_dk < 0) { set_last_error("no solve has run on this graph"); return MLMQ_EINVAL; }
  if (g->last_dk == DK_U64) {
    const void* src = dist_caller_order(g, 8);
    if (!src) { set_last_error("out of device memory for the result gather"); return MLMQ_ENOMEM; }
    CK(cudaMemcpyAsync(out, src, g->n * 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    return MLMQ_OK;
  }
  // Default: widen on the device and DMA the u64 array (measured on B200, C2: 0.76 ms of
  // library overhead vs 0.85 ms for the u32 copy + host-thread widening into the caller's
  // pinned buffer); MLMQ_D2H=host selects the latter.
  static const bool host_widen = [] {
    const char* e = getenv("MLMQ_D2H");
    return e && std::strcmp(e, "host") == 0;
  }();
  if (g->n < (1ull << 16) || !host_widen) {  // device widen + one copy
    if (!g->d_dist64) CK(cudaMalloc(&g->d_dist64, std::max<size_t>(8, g->n * 8)));
    const int blocks = (int)std::min<unsigned long long>(8ull * g->sm_count, (g->n + 255) / 256 + 1);
    widen_kernel<<<blocks, 256, 0, g->stream>>>((const uint32_t*)g->d_dist, g->d_dist64, g->n,
                                                g->relabel_state == 1 ? g->d_perm : nullptr);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, g->d_dist64, g->n * 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    return MLMQ_OK;
  }
  if (g->stage_cap < g->n) {
    if (g->h_stage) cudaFreeHost(g->h_stage);
    g->h_stage = nullptr;
    g->stage_cap = 0;
    CK(cudaHostAlloc((void**)&g->h_stage, g->n * 4, cudaHostAllocDefault));
    g->stage_cap = g->n;
  }
  if (!g->chunk_ev[0])
    for (int k = 0; k < kChunks; ++k) CK(cudaEventCreateWithFlags(&g->chunk_ev[k], cudaEventDisableTiming));
  const unsigned long long ch = (g->n + kChunks - 1) / kChunks;
  const uint32_t* d32 = (const uint32_t*)dist_caller_order(g, 4);
  if (!d32) { set_last_error("out of device memory for the result gather"); return MLMQ_ENOMEM; }
  for (int k = 0; k < kChunks; ++k) {
    const unsigned long long lo = k * ch, hi = std::min(g->n, lo + ch);
    if (lo < hi)
      CK(cudaMemcpyAsync(g->h_stage + lo, d32 + lo, (hi - lo) * 4, cudaMemcpyDeviceToHost,
                         g->stream));
    CK(cudaEventRecord(g->chunk_ev[k], g->stream));
  }
  widen_pool().run(g->h_stage, out, g->n, ch, g->chunk_ev, g->device);
  return MLMQ_OK;
}

int solve(mlmq_graph* g, uint64_t source, const mlmq_config_t* c, void* dist_out, bool f32,
          mlmq_metrics_t* mo, uint64_t* gm, uint64_t gm_cap) {
  if (!g || !c) { set_last_error("null argument"); return MLMQ_EINVAL; }
  const double t0 = now_s();
  std::lock_guard<std::mutex> lk(g->mu);
  CK(cudaSetDevice(g->device));
  if (g->nparts > 1) {
    set_last_error("this graph is a shard of a partitioned graph: use mlmq_shard_step");
    return MLMQ_EINVAL;
  }
  if (source >= g->n) {
    set_last_error("source %llu out of range for %llu vertices", (unsigned long long)source, g->n);
    return MLMQ_EINVAL;
  }
  int st = validate(c);
  if (st) return st;
  const bool graph_f32 = g->wkind == MLMQ_W_F32;
  if (f32 != graph_f32 && dist_out) {
    set_last_error(graph_f32 ? "float-weight graph: use mlmq_sssp_f32" : "integer-weight graph: use mlmq_sssp");
    return MLMQ_EINVAL;
  }
  int dk = graph_f32 ? DK_F32 : (c->dist_mode == MLMQ_DIST_U64 ? DK_U64 : DK_U32);
  uint32_t reruns = 0;
  for (int attempt = 0; attempt < 4; ++attempt) {
    st = run_once(g, source, c, dk, mo, gm, gm_cap);
    if (st == 100) { dk = DK_U64; reruns = 1; continue; }
    if (st == 101) continue;
    break;
  }
  if (st) return st;
  if (dist_out) {
    if (f32) {
      const void* src = dist_caller_order(g, 4);
      if (!src) { set_last_error("out of device memory for the result gather"); return MLMQ_ENOMEM; }
      CK(cudaMemcpyAsync(dist_out, src, g->n * 4, cudaMemcpyDeviceToHost, g->stream));
      CK(cudaStreamSynchronize(g->stream));
    } else if ((st = copy_dist_u64(g, (uint64_t*)dist_out))) {
      return st;
    }
  }
  if (mo) {
    mo->reruns = reruns;
    mo->wall_time_us = (uint64_t)((now_s() - t0) * 1e6);
  }
  return MLMQ_OK;
}

// Interleave (col, weight) and count columns outside [0, col_bound) into *bad: a column
// >= n would make the kernel read and atomically write past dist; the
// reference raises IndexError on such a graph, the ABI returns MLMQ_EINVAL.
__global__ void interleave_kernel(const uint32_t* col, const uint32_t* w, uint2* adj, unsigned long long m, int unit,
                                  unsigned long long col_bound, unsigned long long* bad) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned nbad = 0;
  for (unsigned long long k = tid; k < m; k += stride) {
    const uint32_t c = col[k];
    nbad += (unsigned long long)c >= col_bound;
    adj[k] = make_uint2(c, unit ? 1u : w[k]);
  }
  if (nbad) atomicAdd(bad, (unsigned long long)nbad);
}

// Row offsets must be non-decreasing (a decreasing pair makes a huge unsigned degree).
__global__ void offsets_check_kernel(const unsigned long long* off, unsigned long long n, unsigned long long* bad) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned nbad = 0;
  for (unsigned long long i = tid; i < n; i += stride) nbad += off[i] > off[i + 1];
  if (nbad) atomicAdd(bad, (unsigned long long)nbad);
}

}  // namespace


// ------------------------------------------------------------------ queue harness
struct mlmq_queue {
  mlmq_graph* g = nullptr;   // carrier: device, stream, control words, queue workspace
  mlmq_config_t c{};
  LaunchShape sh;
  KParams p{};
  int l2k = 0, G = 0;
  uint2* d_io = nullptr;
  unsigned long long io_cap = 0;
  unsigned long long* d_n = nullptr;
  int* d_cursors = nullptr;
  std::mutex mu;
};

static int queue_check_error(mlmq_queue* q) {
  unsigned long long ctl[C_WORDS];
  CK(cudaMemcpy(ctl, q->g->d_ctl, sizeof(ctl), cudaMemcpyDeviceToHost));
  const unsigned long long err = ctl[C_ERR];
  if (!err) return MLMQ_OK;
  const double spin = q->c.spin_timeout_s > 0 ? q->c.spin_timeout_s : 15.0;
  // the queue is wedged: later calls report the same error (like an aborted solve)
  if (err == ERR_OVERFLOW) {
    set_last_error("ring slot %llu stayed busy for %gs (block_num=%llu, write_ptr=%llu, read_ptr=%llu); block_num is likely too small for this workload",
                   ctl[C_DIAG + 1], spin, (unsigned long long)q->g->ws.bn, ctl[C_DIAG + 2], ctl[C_DIAG + 3]);
    return MLMQ_EOVERFLOW;
  }
  if (err == ERR_HEAP_OVERFLOW) {
    set_last_error("batch heap %llu is full (%llu of %llu nodes)", ctl[C_DIAG], ctl[C_DIAG + 1], ctl[C_DIAG + 2]);
    return MLMQ_EOVERFLOW;
  }
  set_last_error("queue harness error %llu (%llu %llu %llu %llu)", err, ctl[C_DIAG], ctl[C_DIAG + 1],
                 ctl[C_DIAG + 2], ctl[C_DIAG + 3]);
  return MLMQ_EENGINE;
}

static int queue_io(mlmq_queue* q, unsigned long long n) {
  if (n <= q->io_cap) return MLMQ_OK;
  cudaFree(q->d_io);
  q->d_io = nullptr;
  q->io_cap = 0;
  CK(cudaMalloc(&q->d_io, std::max<unsigned long long>(n, 1024) * 8));
  q->io_cap = std::max<unsigned long long>(n, 1024);
  return MLMQ_OK;
}

extern "C" {

int mlmq_abi_version(void) { return MLMQ_ABI_VERSION; }

const char* mlmq_last_error(void) { return g_err; }

int mlmq_device_count(int* out) {
  if (!out) return MLMQ_EINVAL;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *out = 0;
    set_last_error("no CUDA device: %s", cudaGetErrorString(e));
    return MLMQ_ECUDA;
  }
  *out = n;
  return MLMQ_OK;
}

int mlmq_device_info(int device, int* sm_count, size_t* free_bytes, size_t* total_bytes) {
  CK(cudaSetDevice(device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  if (sm_count) *sm_count = sms;
  size_t f = 0, t = 0;
  CK(cudaMemGetInfo(&f, &t));
  if (free_bytes) *free_bytes = f;
  if (total_bytes) *total_bytes = t;
  return MLMQ_OK;
}

static int graph_create_impl(const uint64_t* row_offsets, const uint32_t* col, const void* w, int weight_kind,
                             uint64_t n, uint64_t m, int device, uint64_t col_bound, mlmq_graph** out);

int mlmq_graph_create(const uint64_t* row_offsets, const uint32_t* col, const void* w, int weight_kind,
                      uint64_t n, uint64_t m, int device, mlmq_graph** out) {
  return graph_create_impl(row_offsets, col, w, weight_kind, n, m, device, n, out);
}

static int graph_create_impl(const uint64_t* row_offsets, const uint32_t* col, const void* w, int weight_kind,
                             uint64_t n, uint64_t m, int device, uint64_t col_bound, mlmq_graph** out) {
  if (!out || !row_offsets || (m && !col) || (m && weight_kind != MLMQ_W_UNIT && !w)) {
    set_last_error("null argument");
    return MLMQ_EINVAL;
  }
  if (n == 0 || n > 0xFFFFFFFFull) { set_last_error("vertex count must be in [1, 2^32-1]"); return MLMQ_EINVAL; }
  if (row_offsets[n] != m) { set_last_error("row_offsets[n]=%llu does not match m=%llu", (unsigned long long)row_offsets[n], (unsigned long long)m); return MLMQ_EINVAL; }
  *out = nullptr;
  mlmq_graph* g = new mlmq_graph();
  g->device = device;
  g->n = n;
  g->m = m;
  g->wkind = weight_kind;
  auto fail = [&](int code) {
    mlmq_graph_destroy(g);
    return code;
  };
#define CKG(call)                                                                          \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess) {                                                               \
      set_last_error("CUDA error %s during graph upload: %s", cudaGetErrorName(_e),        \
                     cudaGetErrorString(_e));                                              \
      return fail(_e == cudaErrorMemoryAllocation ? MLMQ_ENOMEM : MLMQ_ECUDA);             \
    }                                                                                      \
  } while (0)
  CKG(cudaSetDevice(device));
  CKG(cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, device));
  int coop = 0;
  CKG(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  if (!coop) { set_last_error("device %d does not support cooperative launch", device); return fail(MLMQ_ECUDA); }
  CKG(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
  CKG(cudaEventCreate(&g->ev0));
  CKG(cudaEventCreate(&g->ev1));
  CKG(cudaMalloc(&g->d_off, (n + 1) * 8));
  CKG(cudaMalloc(&g->d_adj, std::max<size_t>(8, m * 8)));
  CKG(cudaMalloc(&g->d_dist, std::max<size_t>(8, n * 8)));
  CKG(cudaMalloc(&g->d_ctl, C_WORDS * 8));
  CKG(cudaMemset(g->d_ctl, 0, C_WORDS * 8));
  CKG(cudaMalloc(&g->d_audit, kAuditWords * 8));
  CKG(cudaMalloc(&g->d_scratch, 16 * 8));
  CKG(cudaHostAlloc(&g->h_abort, 64, cudaHostAllocMapped));
  *g->h_abort = 0;
  CKG(cudaHostGetDevicePointer((void**)&g->d_abort, g->h_abort, 0));
  CKG(cudaMemcpy(g->d_off, row_offsets, (n + 1) * 8, cudaMemcpyHostToDevice));
  CKG(cudaMemsetAsync(g->d_scratch, 0, 16 * 8, g->stream));
  offsets_check_kernel<<<512, 256, 0, g->stream>>>(g->d_off, n, g->d_scratch);
  CKG(cudaGetLastError());
  if (m) {
    // interleave (col, weight) on the device in chunks: one 8-byte load per edge
    const unsigned long long chunk = std::min<unsigned long long>(m, 1ull << 25);
    uint32_t *dc = nullptr, *dw = nullptr;
    CKG(cudaMalloc(&dc, chunk * 4));
    cudaError_t e2 = cudaMalloc(&dw, chunk * 4);
    if (e2 != cudaSuccess) { cudaFree(dc); CKG(e2); }
    for (unsigned long long k0 = 0; k0 < m; k0 += chunk) {
      const unsigned long long c = std::min(chunk, m - k0);
      cudaError_t e = cudaMemcpyAsync(dc, col + k0, c * 4, cudaMemcpyHostToDevice, g->stream);
      if (e == cudaSuccess && weight_kind != MLMQ_W_UNIT)
        e = cudaMemcpyAsync(dw, (const uint32_t*)w + k0, c * 4, cudaMemcpyHostToDevice, g->stream);
      if (e == cudaSuccess) {
        interleave_kernel<<<1024, 256, 0, g->stream>>>(dc, dw, g->d_adj + k0, c, weight_kind == MLMQ_W_UNIT,
                                                       col_bound, g->d_scratch + 1);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess) e = cudaStreamSynchronize(g->stream);
      if (e != cudaSuccess) { cudaFree(dc); cudaFree(dw); CKG(e); }
    }
    cudaFree(dc);
    cudaFree(dw);
  }
  CKG(cudaStreamSynchronize(g->stream));
  unsigned long long bad[2] = {0, 0};
  CKG(cudaMemcpy(bad, g->d_scratch, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad[0] || bad[1]) {
    if (bad[0]) set_last_error("row_offsets must be non-decreasing (%llu decreasing pairs)", bad[0]);
    else set_last_error("%llu column indices lie outside [0, %llu)", bad[1], (unsigned long long)col_bound);
    return fail(MLMQ_EINVAL);
  }
#undef CKG
  *out = g;
  return MLMQ_OK;
}

void mlmq_graph_destroy(mlmq_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->poisoned) {  // a kernel may still run on this stream: leak rather than hang or free under it
    delete g;
    return;
  }
  if (g->stream) cudaStreamSynchronize(g->stream);
  ws_free(g->ws);
  if (g->d_vtx) {  // off / nlight / dist live inside the packed buffer
    cudaFree(g->d_vtx);
    g->d_off = nullptr;
    g->d_nlight = nullptr;
    g->d_dist = nullptr;
  }
  cudaFree(g->d_off);
  cudaFree(g->d_adj);
  cudaFree(g->d_dist);
  cudaFree(g->d_dist64);
  cudaFree(g->d_ctl);
  cudaFree(g->d_audit);
  cudaFree(g->d_metrics);
  cudaFree(g->d_scratch);
  cudaFree(g->d_prof);
  cudaFree(g->d_wstate);
  cudaFree(g->d_ghost);
  cudaFree(g->d_obox);
  cudaFree(g->d_seeds);
  cudaFree(g->d_sscratch);
  cudaFree(g->d_nlight);
  cudaFree(g->d_perm);
  cudaFree(g->d_gather);
  if (g->h_abort) cudaFreeHost(g->h_abort);
  if (g->h_stage) cudaFreeHost(g->h_stage);
  for (cudaEvent_t e : g->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (g->ev0) cudaEventDestroy(g->ev0);
  if (g->ev1) cudaEventDestroy(g->ev1);
  if (g->stream) cudaStreamDestroy(g->stream);
  cudaGetLastError();
  delete g;
}

int mlmq_graph_device_bytes(const mlmq_graph* g, uint64_t* out) {
  if (!g || !out) return MLMQ_EINVAL;
  *out = (g->n + 1) * 8 + g->m * 8 + g->n * 8 + g->ws.bytes;
  return MLMQ_OK;
}

int mlmq_auto_groups(const mlmq_graph* gc, const mlmq_config_t* c, int32_t* out) {
  if (!gc || !c || !out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  mlmq_graph* g = const_cast<mlmq_graph*>(gc);
  CK(cudaSetDevice(g->device));
  int st = validate(c);
  if (st) return st;
  LaunchShape sh;
  const int dk = g->wkind == MLMQ_W_F32 ? DK_F32 : (c->dist_mode == MLMQ_DIST_U64 ? DK_U64 : DK_U32);
  if ((st = launch_shape(g, c, dk, &sh))) return st;
  *out = sh.max_groups;
  return MLMQ_OK;
}

int mlmq_sssp(mlmq_graph* g, uint64_t source, const mlmq_config_t* cfg, uint64_t* dist_out,
              mlmq_metrics_t* metrics_out, uint64_t* group_metrics, uint64_t group_metrics_cap) {
  if (!dist_out) { set_last_error("null dist_out"); return MLMQ_EINVAL; }
  return solve(g, source, cfg, dist_out, false, metrics_out, group_metrics, group_metrics_cap);
}

int mlmq_sssp_f32(mlmq_graph* g, uint64_t source, const mlmq_config_t* cfg, float* dist_out,
                  mlmq_metrics_t* metrics_out, uint64_t* group_metrics, uint64_t group_metrics_cap) {
  if (!dist_out) { set_last_error("null dist_out"); return MLMQ_EINVAL; }
  return solve(g, source, cfg, dist_out, true, metrics_out, group_metrics, group_metrics_cap);
}

int mlmq_sssp_device(mlmq_graph* g, uint64_t source, const mlmq_config_t* cfg, mlmq_metrics_t* metrics_out) {
  return solve(g, source, cfg, nullptr, g && g->wkind == MLMQ_W_F32, metrics_out, nullptr, 0);
}

int mlmq_last_dist(mlmq_graph* g, uint64_t* dist_out) {
  if (!g || !dist_out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  std::lock_guard<std::mutex> lk(g->mu);
  CK(cudaSetDevice(g->device));
  if (g->last_dk == DK_F32) {
    const void* src = dist_caller_order(g, 4);
    if (!src) { set_last_error("out of device memory for the result gather"); return MLMQ_ENOMEM; }
    CK(cudaMemcpyAsync(dist_out, src, g->n * 4, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    return MLMQ_OK;
  }
  return copy_dist_u64(g, dist_out);
}

int mlmq_reach(mlmq_graph* g, uint64_t* v_reach, uint64_t* e_reach) {
  if (!g || !v_reach || !e_reach) { set_last_error("null argument"); return MLMQ_EINVAL; }
  std::lock_guard<std::mutex> lk(g->mu);
  CK(cudaSetDevice(g->device));
  if (g->last_dk < 0) { set_last_error("no solve has run on this graph"); return MLMQ_EINVAL; }
  CK(cudaMemsetAsync(g->d_scratch, 0, 16, g->stream));
  const int blocks = (int)std::min<unsigned long long>(8ull * g->sm_count, (g->n + 255) / 256 + 1);
  if (g->last_dk == DK_U64)
    reach_kernel<unsigned long long><<<blocks, 256, 0, g->stream>>>((const unsigned long long*)g->d_dist, ~0ull, g->d_off, g->n, g->d_scratch);
  else
    reach_kernel<uint32_t><<<blocks, 256, 0, g->stream>>>((const uint32_t*)g->d_dist,
                                                          g->last_dk == DK_F32 ? 0x7f800000u : 0xFFFFFFFFu,
                                                          g->d_off, g->n, g->d_scratch);
  CK(cudaGetLastError());
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, g->d_scratch, 16, cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  *v_reach = h[0];
  *e_reach = h[1];
  return MLMQ_OK;
}

int mlmq_host_alloc(uint64_t bytes, void** out) {
  if (!out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  *out = nullptr;
  CK(cudaHostAlloc(out, std::max<uint64_t>(bytes, 64), cudaHostAllocPortable));
  return MLMQ_OK;
}

void mlmq_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int mlmq_graph_stream(mlmq_graph* g, void** out) {
  if (!g || !out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  *out = (void*)g->stream;
  return MLMQ_OK;
}

int mlmq_shard_create(const uint64_t* row_offsets, const uint32_t* col, const void* w, int weight_kind,
                      uint64_t n_local, uint64_t m_local, uint64_t n_global, uint32_t rank, uint32_t nparts,
                      int device, mlmq_graph** out) {
  if (!out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  if (nparts < 1 || nparts > 64 || (nparts & (nparts - 1)) || rank >= nparts) {
    set_last_error("nparts must be a power of two in [1, 64] and rank < nparts (got %u, %u)", nparts, rank);
    return MLMQ_EINVAL;
  }
  if (n_global == 0 || n_global > 0xFFFFFFFFull || n_local != (n_global - rank + nparts - 1) / nparts) {
    set_last_error("shard %u of %u must own ceil((n - rank) / nparts) = %llu vertices (got %llu)", rank, nparts,
                   (unsigned long long)((n_global - rank + nparts - 1) / nparts), (unsigned long long)n_local);
    return MLMQ_EINVAL;
  }
  int st = graph_create_impl(row_offsets, col, w, weight_kind, n_local, m_local, device, n_global, out);
  if (st) return st;
  mlmq_graph* g = *out;
  g->nparts = nparts;
  g->rank = rank;
  while ((1u << g->shift) < nparts) ++g->shift;
  g->n_global = n_global;
  cudaError_t e = cudaMalloc(&g->d_ghost, n_global * 4);
  if (e == cudaSuccess) e = cudaMalloc(&g->d_sscratch, 256 * 8);
  if (e != cudaSuccess) {
    cudaGetLastError();
    mlmq_graph_destroy(g);
    *out = nullptr;
    set_last_error("shard allocation failed: %s", cudaGetErrorString(e));
    return MLMQ_ENOMEM;
  }
  return MLMQ_OK;
}

int mlmq_shard_begin(mlmq_graph* g) {
  if (!g || g->nparts < 1 || !g->d_ghost) { set_last_error("not a shard"); return MLMQ_EINVAL; }
  std::lock_guard<std::mutex> lk(g->mu);
  CK(cudaSetDevice(g->device));
  const uint32_t inf = g->wkind == MLMQ_W_F32 ? 0x7f800000u : 0xFFFFFFFFu;
  const int b = 4 * g->sm_count;
  fill_kernel<uint32_t><<<b, 256, 0, g->stream>>>((uint32_t*)g->d_dist, g->n, inf);
  fill_kernel<uint32_t><<<b, 256, 0, g->stream>>>((uint32_t*)g->d_ghost, g->n_global, inf);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(g->stream));
  g->last_dk = g->wkind == MLMQ_W_F32 ? DK_F32 : DK_U32;
  return MLMQ_OK;
}

int mlmq_shard_step(mlmq_graph* g, const mlmq_config_t* c, const uint32_t* d_inbox, uint64_t n_in,
                    uint32_t* d_send, uint64_t send_cap, uint64_t* send_counts, mlmq_metrics_t* metrics_out) {
  if (!g || !c || !send_counts || (n_in && !d_inbox) || !d_send) { set_last_error("null argument"); return MLMQ_EINVAL; }
  if (!g->d_ghost) { set_last_error("not a shard: create it with mlmq_shard_create"); return MLMQ_EINVAL; }
  if (c->l2_type != MLMQ_L2_FIFO) { set_last_error("sharded solves run the FIFO L2 (got l2_type code %d)", c->l2_type); return MLMQ_EINVAL; }
  if (c->dist_mode == MLMQ_DIST_U64) { set_last_error("sharded solves keep u32 / f32 distances"); return MLMQ_EINVAL; }
  const double t0 = now_s();
  std::lock_guard<std::mutex> lk(g->mu);
  CK(cudaSetDevice(g->device));
  int st = validate(c);
  if (st) return st;
  if (g->obox_cap < send_cap) {
    cudaFree(g->d_obox);
    g->d_obox = nullptr;
    g->obox_cap = 0;
    CK(cudaMalloc(&g->d_obox, std::max<size_t>(8, send_cap * 8)));
    g->obox_cap = send_cap;
  }
  if (g->seeds_cap < n_in) {  // an inbox may improve one vertex several times
    cudaFree(g->d_seeds);
    g->d_seeds = nullptr;
    g->seeds_cap = 0;
    CK(cudaMalloc(&g->d_seeds, std::max<size_t>(8, n_in * 8)));
    g->seeds_cap = n_in;
  }
  ShardIo io;
  io.inbox = reinterpret_cast<const uint2*>(d_inbox);
  io.n_in = n_in;
  io.send = reinterpret_cast<uint2*>(d_send);
  io.send_cap = send_cap;
  io.send_counts = send_counts;
  const int dk = g->wkind == MLMQ_W_F32 ? DK_F32 : DK_U32;
  for (int attempt = 0; attempt < 3; ++attempt) {
    st = run_once(g, 0, c, dk, metrics_out, nullptr, 0, &io);
    if (st == 101) continue;
    break;
  }
  if (st == 100) {
    set_last_error("sharded solve: a distance overflowed u32 (use an unpartitioned u64 solve)");
    return MLMQ_EOVERFLOW;
  }
  if (st) return st;
  if (metrics_out) metrics_out->wall_time_us = (uint64_t)((now_s() - t0) * 1e6);
  return MLMQ_OK;
}

int mlmq_feature_sums(mlmq_graph* g, uint64_t out[10]) {
  if (!g || !out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  std::lock_guard<std::mutex> lk(g->mu);
  CK(cudaSetDevice(g->device));
  CK(cudaMemsetAsync(g->d_scratch, 0, 16 * 8, g->stream));
  const int blocks = 4 * g->sm_count;
  feature_sums_kernel<<<blocks, 256, 0, g->stream>>>(g->d_off, g->d_adj, g->n, g->m,
                                                     g->wkind == MLMQ_W_UNIT, g->d_scratch);
  CK(cudaGetLastError());
  if (g->wkind == MLMQ_W_F32) {
    feature_sums_f32_kernel<<<blocks, 256, 0, g->stream>>>(g->d_adj, g->m, (double*)(g->d_scratch + 8),
                                                           (unsigned int*)(g->d_scratch + 10));
    CK(cudaGetLastError());
  }
  unsigned long long h[16];
  CK(cudaMemcpyAsync(h, g->d_scratch, sizeof(h), cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  out[0] = g->n;
  out[1] = g->m;
  out[2] = h[0];
  out[3] = h[1];
  out[4] = h[2];
  out[5] = h[3];
  if (g->wkind == MLMQ_W_F32) {
    out[6] = h[8];   // double bits of sum w
    out[7] = h[9];   // double bits of sum w^2
    out[8] = 0;
    out[9] = h[10] & 0xFFFFFFFFull;  // float bits of max w
  } else {
    out[6] = h[4];
    out[7] = h[5];
    out[8] = h[6];
    out[9] = h[7];
  }
  return MLMQ_OK;
}


int mlmq_queue_create(int device, const mlmq_queue_params_t* qp, mlmq_queue** out) {
  if (!qp || !out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  *out = nullptr;
  if (qp->l2_type < 0 || qp->l2_type > 3) { set_last_error("unknown l2_type code %d", qp->l2_type); return MLMQ_EINVAL; }
  if (qp->block_size < 1 || qp->block_size > 4096 || qp->block_num < 1) {
    set_last_error("block_size must be in [1, 4096] and block_num >= 1");
    return MLMQ_EINVAL;
  }
  const uint64_t off[2] = {0, 0};
  mlmq_graph* g = nullptr;
  int st = graph_create_impl(off, nullptr, nullptr, MLMQ_W_UNIT, 1, 0, device, 1, &g);
  if (st) return st;
  mlmq_queue* q = new mlmq_queue();
  q->g = g;
  mlmq_config_t& c = q->c;
  c.l1_type = MLMQ_L1_VECTOR;
  c.l2_type = qp->l2_type;
  c.l0_capacity = 4;
  c.l1_capacity = 64;
  c.wb = 0;
  c.delta = qp->delta > 0 ? qp->delta : 1.0;
  c.block_size = qp->block_size;
  c.block_num = qp->block_num;
  c.bmax = std::max(1, qp->bmax);
  c.bnum = std::max(1, std::min(qp->bnum, c.bmax));
  c.node_batch = std::max(1, std::min(qp->node_batch, 32));
  c.pnum = qp->l2_type == MLMQ_L2_MULTI ? std::max(1, qp->pnum) : 1;
  c.num_groups = std::max(1, qp->num_groups);
  c.lanes_per_group = 32;
  c.dup_elim = 1;
  c.spin_timeout_s = qp->spin_timeout_s > 0 ? qp->spin_timeout_s : 15.0;
  c.read_batch = 32;
  const bool heap = c.l2_type == MLMQ_L2_PRIORITY || c.l2_type == MLMQ_L2_MULTI;
  c.test_capacity = (int32_t)std::min<long long>(heap ? (qp->heap_nodes > 0 ? qp->heap_nodes : 65536) : qp->block_num,
                                                 1LL << 30);
  auto fail = [&](int code) {
    mlmq_queue_destroy(q);
    return code;
  };
  if ((st = validate(&c))) return fail(st);
  if ((st = launch_shape(g, &c, DK_U32, &q->sh))) return fail(st);
  q->l2k = q->sh.l2k;
  q->G = std::min(q->sh.max_groups, 1024);
  if ((st = ensure_workspace(g, &c, q->sh, 2048ull, q->G))) return fail(st);
  const size_t nslots = (size_t)std::max(g->ws.nrings, 1) * g->ws.bn;
  reset_queues_kernel<<<1024, 256, 0, g->stream>>>(g->ws.seq, nslots, g->ws.bn - 1, g->ws.ptrs, std::max(g->ws.nrings, 1),
                                                    g->ws.hub_seq, g->ws.hub_next, g->ws.hub_fin, g->ws.hub_cap, g->d_ctl,
                                                    g->ws.hlock, g->ws.hsize, g->ws.hwc, std::max(g->ws.nheaps, 1));
  g->ws.dirty = false;
  if (cudaMemsetAsync(g->d_ctl, 0, C_WORDS * 8, g->stream) != cudaSuccess ||
      cudaMalloc(&q->d_n, 64) != cudaSuccess ||
      cudaMalloc(&q->d_cursors, sizeof(int) * (size_t)c.num_groups) != cudaSuccess) {
    cudaGetLastError();
    set_last_error("queue harness allocation failed");
    return fail(MLMQ_ENOMEM);
  }
  std::vector<int> cur((size_t)c.num_groups);
  for (int i = 0; i < c.num_groups; ++i) cur[(size_t)i] = i % c.pnum;
  if (cudaMemcpy(q->d_cursors, cur.data(), cur.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaStreamSynchronize(g->stream) != cudaSuccess) {
    cudaGetLastError();
    set_last_error("queue harness initialisation failed");
    return fail(MLMQ_ECUDA);
  }
  q->p = make_params(g, &c, DK_U32, q->sh, q->G, 2048ull, 0, false);
  q->p.fifo_park = 0;  // conditional readers: no claim outlives a call (l2.py:141-148)
  q->p.bwin = 0;       // the reference's floor rule (l2.py:282-287)
  q->p.share = 0;
  *out = q;
  return MLMQ_OK;
}

void mlmq_queue_destroy(mlmq_queue* q) {
  if (!q) return;
  cudaFree(q->d_io);
  cudaFree(q->d_n);
  cudaFree(q->d_cursors);
  mlmq_graph_destroy(q->g);
  delete q;
}

int mlmq_queue_write(mlmq_queue* q, const uint32_t* pairs, uint64_t n, int32_t group) {
  if (!q || (n && !pairs)) { set_last_error("null argument"); return MLMQ_EINVAL; }
  if (group < 0 || group >= q->c.num_groups) { set_last_error("group %d out of range", group); return MLMQ_EINVAL; }
  if (n == 0) return MLMQ_OK;
  std::lock_guard<std::mutex> lk(q->mu);
  int st = queue_io(q, n);
  if (st) return st;
  CK(cudaMemcpyAsync(q->d_io, pairs, n * 8, cudaMemcpyHostToDevice, q->g->stream));
  HarnessArgs h{};
  h.mode = 0;
  h.group = group;
  h.in = q->d_io;
  h.n_in = n;
  h.cursors = q->l2k == L2K_HEAP ? q->d_cursors : nullptr;
  if (harness_launch(q->l2k, q->p, h, 1, 1, (size_t)q->sh.smem_per_warp, q->g->stream) != 0) {
    set_last_error("queue harness launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return MLMQ_ECUDA;
  }
  CK(cudaStreamSynchronize(q->g->stream));
  return queue_check_error(q);
}

int mlmq_queue_read(mlmq_queue* q, int32_t group, uint32_t* pairs_out, uint64_t cap, uint64_t* n_out) {
  if (!q || !n_out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  if (group < 0 || group >= q->c.num_groups) { set_last_error("group %d out of range", group); return MLMQ_EINVAL; }
  std::lock_guard<std::mutex> lk(q->mu);
  int st = queue_io(q, (unsigned long long)std::max(q->c.block_size, 32));
  if (st) return st;
  HarnessArgs h{};
  h.mode = 1;
  h.group = group;
  h.out = q->d_io;
  h.out_n = q->d_n;
  h.out_cap = q->io_cap;
  if (harness_launch(q->l2k, q->p, h, 1, 1, (size_t)q->sh.smem_per_warp, q->g->stream) != 0) {
    set_last_error("queue harness launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return MLMQ_ECUDA;
  }
  unsigned long long c = 0;
  CK(cudaMemcpyAsync(&c, q->d_n, 8, cudaMemcpyDeviceToHost, q->g->stream));
  CK(cudaStreamSynchronize(q->g->stream));
  if ((st = queue_check_error(q))) return st;
  if (c > cap) { set_last_error("read returned %llu elements; buffer holds %llu", c, (unsigned long long)cap); return MLMQ_EINVAL; }
  if (c) CK(cudaMemcpy(pairs_out, q->d_io, c * 8, cudaMemcpyDeviceToHost));
  *n_out = c;
  return MLMQ_OK;
}

int mlmq_queue_stats(mlmq_queue* q, uint64_t out[40]) {
  if (!q || !out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  std::lock_guard<std::mutex> lk(q->mu);
  std::memset(out, 0, 40 * sizeof(uint64_t));
  const Workspace& w = q->g->ws;
  unsigned long long ctl[C_WORDS];
  CK(cudaMemcpy(ctl, q->g->d_ctl, sizeof(ctl), cudaMemcpyDeviceToHost));
  out[3] = ctl[C_EPOCH];
  bool empty = true, heap_ok = true;
  if (q->l2k != L2K_HEAP) {
    std::vector<unsigned long long> ptrs((size_t)w.nrings * 32), seq((size_t)w.nrings * w.bn);
    std::vector<uint32_t> cnt((size_t)w.nrings * w.bn);
    CK(cudaMemcpy(ptrs.data(), w.ptrs, ptrs.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(seq.data(), w.seq, seq.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cnt.data(), w.cnt, cnt.size() * 4, cudaMemcpyDeviceToHost));
    for (int r = 0; r < w.nrings; ++r) {
      const unsigned long long wp = ptrs[(size_t)r * 32], rp = ptrs[(size_t)r * 32 + 16];
      out[5] += wp;
      out[6] += rp;
      if (wp != rp) empty = false;
      for (unsigned long long t = rp; t < wp; ++t) {  // written, unclaimed
        const size_t i = (size_t)r * w.bn + (t & (w.bn - 1));
        if (seq[i] == t + 1) out[0] += cnt[i];
      }
      const unsigned long long lo = rp > w.bn ? rp - w.bn : 0;
      for (unsigned long long t = lo; t < rp; ++t) {  // claimed: consumed iff freed to t + bn
        const size_t i = (size_t)r * w.bn + (t & (w.bn - 1));
        if (seq[i] == t + 1) ++out[1];
      }
    }
  } else {
    std::vector<unsigned long long> hs((size_t)w.nheaps * 16), hw((size_t)w.nheaps * 16);
    CK(cudaMemcpy(hs.data(), w.hsize, hs.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hw.data(), w.hwc, hw.size() * 8, cudaMemcpyDeviceToHost));
    for (int h = 0; h < w.nheaps; ++h) {
      const unsigned long long size = hs[(size_t)h * 16];
      out[5] += hw[(size_t)h * 16];
      if (size) empty = false;
      std::vector<uint32_t> hc(size);
      std::vector<uint2> nodes(size * 32);
      if (size) {
        CK(cudaMemcpy(hc.data(), w.hcnt + (size_t)h * w.hcap, size * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(nodes.data(), (uint2*)w.hnodes + (size_t)h * w.hcap * 32, size * 32 * 8, cudaMemcpyDeviceToHost));
      }
      unsigned long long elems = 0;
      for (unsigned long long i = 0; i < size; ++i) {  // l2.py:391-402: sorted nodes, parent min <= child min
        elems += hc[i];
        if (hc[i] == 0 || hc[i] > 32) heap_ok = false;
        for (uint32_t k = 1; k < hc[i] && k < 32; ++k)
          if (nodes[i * 32 + k].y < nodes[i * 32 + k - 1].y) heap_ok = false;
        if (i > 0 && nodes[i * 32].y < nodes[((i - 1) / 2) * 32].y) heap_ok = false;
      }
      out[0] += elems;
      if (h < 32) out[7 + h] = elems;
    }
  }
  out[2] = empty ? 1 : 0;
  out[4] = heap_ok ? 1 : 0;
  return MLMQ_OK;
}

int mlmq_queue_stress(mlmq_queue* q, int32_t writers, int32_t readers, uint64_t stride, uint64_t begin, uint64_t end,
                      uint64_t stop_at, uint32_t* pairs_out, uint64_t cap, uint64_t* n_out, uint64_t* epochs_out,
                      uint64_t log_cap, uint64_t* log_n, double* ms_out) {
  if (!q || !pairs_out || !n_out) { set_last_error("null argument"); return MLMQ_EINVAL; }
  if (writers < 0 || readers < 1 || writers + readers > q->G || writers + readers > q->c.num_groups) {
    set_last_error("need 1 <= readers and writers + readers <= %d", std::min(q->G, q->c.num_groups));
    return MLMQ_EINVAL;
  }
  std::lock_guard<std::mutex> lk(q->mu);
  mlmq_graph* g = q->g;
  uint2* d_out = nullptr;
  unsigned long long* d_log = nullptr;
  unsigned long long* d_logn = nullptr;
  const bool logs = epochs_out && log_n && log_cap;
  cudaError_t e = cudaMalloc(&d_out, std::max<uint64_t>(cap, 1) * 8);
  if (e == cudaSuccess && logs) e = cudaMalloc(&d_log, (size_t)readers * log_cap * 8);
  if (e == cudaSuccess && logs) e = cudaMalloc(&d_logn, (size_t)readers * 8);
  auto cleanup = [&]() { cudaFree(d_out); cudaFree(d_log); cudaFree(d_logn); };
  if (e != cudaSuccess) { cudaGetLastError(); cleanup(); set_last_error("stress buffers: %s", cudaGetErrorString(e)); return MLMQ_ENOMEM; }
  HarnessArgs h{};
  h.mode = 2;
  h.out = d_out;
  h.out_n = q->d_n;
  h.out_cap = cap;
  h.writers = writers;
  h.readers = readers;
  h.w_stride = stride;
  h.w_begin = begin;
  h.w_end = end;
  h.stop_at = stop_at;
  h.epoch_log = d_log;
  h.log_cap = logs ? log_cap : 0;
  h.log_n = d_logn;
  KParams p = q->p;
  p.G = writers + readers;
  if (cudaMemsetAsync(q->d_n, 0, 8, g->stream) != cudaSuccess) { cleanup(); CK(cudaGetLastError()); }
  CK(cudaEventRecord(g->ev0, g->stream));
  const int wpb = std::max(1, std::min(q->sh.wpb, 9));  // queue_harness_kernel: __launch_bounds__(288)
  if (harness_launch(q->l2k, p, h, writers + readers, wpb, (size_t)q->sh.smem_per_warp, g->stream) != 0) {
    cleanup();
    set_last_error("queue stress launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return MLMQ_ECUDA;
  }
  CK(cudaEventRecord(g->ev1, g->stream));
  e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) { cleanup(); CK(e); }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, g->ev0, g->ev1);
  if (ms_out) *ms_out = ms;
  unsigned long long n = 0;
  e = cudaMemcpy(&n, q->d_n, 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && n) e = cudaMemcpy(pairs_out, d_out, std::min<unsigned long long>(n, cap) * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && logs) e = cudaMemcpy(epochs_out, d_log, (size_t)readers * log_cap * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && logs) e = cudaMemcpy(log_n, d_logn, (size_t)readers * 8, cudaMemcpyDeviceToHost);
  cleanup();
  CK(e);
  *n_out = n;
  return queue_check_error(q);
}

}  // extern "C"
