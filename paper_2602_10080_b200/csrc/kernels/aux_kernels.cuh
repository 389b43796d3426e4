// aux_kernels.cuh — K3 init/bootstrap, ring reset, K5 audit, K4 features, reach, widen.
#pragma once
#include "common.cuh"

namespace mlmq {

// Full reset of every queue structure (first use of a workspace, or after an aborted
// solve left tickets dangling).  Vyukov slots start with seq[s] = s.
__global__ void reset_queues_kernel(unsigned long long* seq, unsigned long long nslots_total,
                                    unsigned long long bn_mask, unsigned long long* ptrs,
                                    int nrings, unsigned long long* hub_seq,
                                    unsigned long long* hub_next, uint32_t* hub_fin,
                                    unsigned long long hub_cap, unsigned long long* ctl,
                                    uint32_t* hlock, unsigned long long* hsize,
                                    unsigned long long* hwc, int nheaps) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < nslots_total; i += stride) seq[i] = i & bn_mask;
  for (unsigned long long i = tid; i < hub_cap; i += stride) {
    hub_seq[i] = i;
    hub_next[i] = 0;
    hub_fin[i] = 0;
  }
  for (unsigned long long i = tid; i < (unsigned long long)nrings * 32; i += stride) ptrs[i] = 0;
  for (unsigned long long i = tid; i < (unsigned long long)nheaps; i += stride) {
    hlock[i * 32] = 0;
    hsize[i * 16] = 0;
    hwc[i * 16] = 0;
  }
  if (tid == 0) {
    ctl[C_HUB_WP] = 0;
    ctl[C_HUB_RP] = 0;
    ctl[C_HUB_RES] = 0;
  }
}

// K3 (DistanceTable.__init__ core.py:198-203 + mlmq_bootstrap compose.py:92-101):
// dist = INF except dist[s] = 0; control words reset; done := current reserve total;
// (s, 0) written straight through to the L2 queue.
// step = 1: a superstep of a sharded solve -- distances persist, no bootstrap (the
// seeds arrive through seed_* below).
template <class S>
__global__ void init_kernel(S* dist, unsigned long long n, unsigned long long source, S inf,
                            KParams p, int l2k, int step = 0) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  if (!step)
    for (unsigned long long i = tid; i < n; i += stride) dist[i] = (i == source) ? (S)0 : inf;
  if (tid != 0) return;
  unsigned long long* ctl = p.ctl;
  ctl[C_STOP] = 0;
  ctl[C_GEN] = 0;
  ctl[C_ERR] = 0;
  ctl[C_EPOCH] = 0;
  ctl[C_DIST_OVF] = 0;
  ctl[C_LOCAL_NONEMPTY] = 0;
  ctl[C_HUB_ITEMS] = 0;
  ctl[C_IDLE] = 0;
  for (int i = 0; i < 4; ++i) ctl[C_DIAG + i] = 0;
  ctl[C_HUB_RP] = ctl[C_HUB_WP];  // every descriptor of the last solve completed
  unsigned long long reserve = ctl[C_HUB_RES];
  for (int r = 0; r < p.nrings; ++r) reserve += p.ptrs[(size_t)r * 32];
  for (int h = 0; h < p.pnum; ++h) reserve += p.hwc[(size_t)h * 16];
  ctl[C_DONE] = reserve;
  if (step) {
    __threadfence();
    return;
  }
  if (l2k == L2K_HEAP) {
    Elem<S> e;
    e.v = (uint32_t)source;
    e.d = 0;
    reinterpret_cast<Elem<S>*>(p.hnodes)[0] = e;
    p.hcnt[0] = 1;
    p.hsize[0] = 1;
    p.hwc[0] += 1;
  } else {
    const unsigned long long t = p.ptrs[0];
    const unsigned long long slot = t & p.bn_mask;
    if (p.seq[slot] != t) ctl[C_ERR] = 99;  // inconsistent ring: host resets and retries
    Elem<S> e;
    e.v = (uint32_t)source;
    e.d = 0;
    reinterpret_cast<Elem<S>*>(p.data)[slot * p.bs] = e;
    p.cnt[slot] = 1;
    p.seq[slot] = t + 1;
    p.ptrs[0] = t + 1;
  }
  __threadfence();
}

// K5 (_Run.audit engine.py:229-242): reserve == done, rings drained, heaps empty,
// no group holding elements.
// With parked FIFO readers (fifo_fix), tickets still pending at termination are
// retired here: their slots are marked consumed and the write pointer catches up.
__global__ void audit_kernel(KParams p, unsigned long long* out, int fifo_fix) {
  __shared__ unsigned long long s_res[256], s_bad[256], s_hs[256];
  const int t = threadIdx.x;
  unsigned long long res = 0, bad = 0, hs = 0;
  for (int r = t; r < p.nrings; r += blockDim.x) {
    const unsigned long long w = p.ptrs[(size_t)r * 32], rd = p.ptrs[(size_t)r * 32 + 16];
    res += w;
    bad += fifo_fix ? (rd < w) : (w != rd);
  }
  for (int h = t; h < p.pnum; h += blockDim.x) {
    res += p.hwc[(size_t)h * 16];
    hs += p.hsize[(size_t)h * 16];
  }
  s_res[t] = res;
  s_bad[t] = bad;
  s_hs[t] = hs;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (t < o) {
      s_res[t] += s_res[t + o];
      s_bad[t] += s_bad[t + o];
      s_hs[t] += s_hs[t + o];
    }
    __syncthreads();
  }
  if (t == 0) {
    const unsigned long long* ctl = p.ctl;
    if (kDebug && p.wstate) p.wstate[2 * (size_t)p.G + 5] = 1;
    out[0] = ctl[C_DONE];
    out[1] = s_res[0] + ctl[C_HUB_RES];
    out[2] = s_bad[0];
    out[3] = 0;  // hub descriptors: covered by reserve == done (C_HUB_RES)
    out[4] = s_hs[0];
    out[5] = ctl[C_LOCAL_NONEMPTY];
    out[6] = ctl[C_ERR];
    out[7] = ctl[C_DIST_OVF];
    for (int i = 0; i < 4; ++i) out[8 + i] = ctl[C_DIAG + i];
    out[12] = ctl[C_HUB_ITEMS];
    out[13] = ctl[C_EPOCH];
    if (kDebug && p.wstate) p.wstate[2 * (size_t)p.G + 5] = 2;
  }
  if (fifo_fix) {  // retire the parked FIFO tickets, all threads in parallel
    __syncthreads();
    const unsigned long long w = p.ptrs[0], rd = p.ptrs[16];
    for (unsigned long long tk = w + t; tk < rd; tk += blockDim.x) p.seq[tk & p.bn_mask] = tk + p.bn_mask + 1;
    __syncthreads();
    if (t == 0 && rd > w) p.ptrs[0] = rd;
    __threadfence();
  }
}

// ---------------------------------------------------------------------------------
// Sharded solve: superstep plumbing around K1
// ---------------------------------------------------------------------------------
template <class S>
__global__ void fill_kernel(S* a, unsigned long long n, S v) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < n; i += stride) a[i] = v;
}

// Apply the inbox (global v, d) to this shard's distances; improved vertices become
// seeds (local id, d).  scratch[0] = seed count.
template <class S>
__global__ void seed_apply_kernel(const uint2* inbox, unsigned long long n_in, S* dist, int shift,
                                  unsigned long long n_local, uint2* seeds, unsigned long long* scratch,
                                  unsigned long long* err) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  // whole warps iterate together so the seed append is one fetch-add per warp
  const unsigned long long n_up = (n_in + 31) & ~31ull;
  for (unsigned long long i = tid; i < n_up; i += stride) {
    bool up = false;
    uint2 m = make_uint2(0u, 0u);
    unsigned long long lv = 0;
    if (i < n_in) {
      m = inbox[i];
      lv = (unsigned long long)(m.x >> shift);
      if (lv >= n_local) atomicCAS(err, 0ull, (unsigned long long)ERR_CORRUPT);
      else up = (S)m.y < atomicMin(dist + lv, (S)m.y);
    }
    const unsigned bal = __ballot_sync(FULL, up);
    if (!bal) continue;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(scratch, (unsigned long long)__popc(bal));
    base = __shfl_sync(FULL, base, 0);
    if (up) seeds[base + __popc(bal & lanemask_lt())] = make_uint2((uint32_t)lv, m.y);
  }
}

// Write the seeds into L2 ring 0 as full blocks (write_through, compose.py:79-86): the
// write tickets are the reservation (the init kernel already set done = reserve).
template <class S>
__global__ void seed_ring_kernel(const uint2* seeds, const unsigned long long* scratch, KParams p) {
  __shared__ unsigned long long t0;
  const unsigned long long ns = scratch[0];
  const unsigned long long nblk = (ns + p.bs - 1) / p.bs;
  if (threadIdx.x == 0) t0 = p.ptrs[0];
  __syncthreads();
  for (unsigned long long b = blockIdx.x; b < nblk; b += gridDim.x) {
    const unsigned long long tk = t0 + b, slot = tk & p.bn_mask;
    const unsigned long long lo = b * p.bs, c = min((unsigned long long)p.bs, ns - lo);
    Elem<S>* dst = reinterpret_cast<Elem<S>*>(p.data) + slot * p.bs;
    for (unsigned long long i = threadIdx.x; i < c; i += blockDim.x) {
      Elem<S> e;
      e.v = seeds[lo + i].x;
      e.d = (S)seeds[lo + i].y;
      dst[i] = e;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (p.seq[slot] != tk) atomicCAS(p.ctl + C_ERR, 0ull, (unsigned long long)ERR_CORRUPT);
      p.cnt[slot] = (uint32_t)c;
      __threadfence();
      p.seq[slot] = tk + 1;
    }
    __syncthreads();
  }
}
__global__ void seed_commit_kernel(const unsigned long long* scratch, KParams p) {
  const unsigned long long nblk = (scratch[0] + p.bs - 1) / p.bs;
  p.ptrs[0] += nblk;
  __threadfence();
}

// Group the outbox by owner shard (counting sort): send[] = concatenation per rank,
// counts[r] = pairs for rank r.  scratch layout: [0] outbox fill, [8..8+P) counts,
// [72..72+P) cursors.
__global__ void obox_hist_kernel(const uint2* obox, const unsigned long long* scratch_n, unsigned long long cap,
                                 unsigned long long* counts, uint32_t pmask) {
  __shared__ unsigned int h[64];
  if (threadIdx.x < 64) h[threadIdx.x] = 0;
  __syncthreads();
  const unsigned long long n = min(*scratch_n, cap);  // an overflowing step is an error anyway
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < n; i += stride) {
    const uint32_t v = obox[i].x;
    if (v != 0xFFFFFFFFu) atomicAdd(h + (v & pmask), 1u);  // ~0: an unfilled reserved slot
  }
  __syncthreads();
  if (threadIdx.x <= pmask && h[threadIdx.x]) atomicAdd(counts + threadIdx.x, (unsigned long long)h[threadIdx.x]);
}
__global__ void obox_scan_kernel(const unsigned long long* counts, unsigned long long* cursors, int P) {
  unsigned long long s = 0;
  for (int r = 0; r < P; ++r) {
    cursors[r] = s;
    s += counts[r];
  }
}
// Group the outbox by owner into the send buffer.  Per tile of blockDim x 8 entries a
// block counts its entries per owner in shared memory, reserves one range per owner with
// a single global fetch-add, and scatters through shared cursors: 2P global atomics per
// tile instead of one per entry on P hot cursor words.
__global__ void obox_scatter_kernel(const uint2* obox, const unsigned long long* scratch_n,
                                    unsigned long long cap, unsigned long long* cursors, uint2* send,
                                    uint32_t pmask) {
  __shared__ unsigned int cnt[64];
  __shared__ unsigned long long base[64];
  const unsigned long long n = min(*scratch_n, cap);
  constexpr int kPer = 8;
  const unsigned long long tile = (unsigned long long)blockDim.x * kPer;
  for (unsigned long long t0 = (unsigned long long)blockIdx.x * tile; t0 < n; t0 += (unsigned long long)gridDim.x * tile) {
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();
    uint2 m[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const unsigned long long i = t0 + (unsigned long long)k * blockDim.x + threadIdx.x;
      m[k] = i < n ? obox[i] : make_uint2(0xFFFFFFFFu, 0u);
      if (m[k].x != 0xFFFFFFFFu) atomicAdd(cnt + (m[k].x & pmask), 1u);
    }
    __syncthreads();
    if (threadIdx.x <= pmask) {
      const unsigned c = cnt[threadIdx.x];
      base[threadIdx.x] = c ? atomicAdd(cursors + threadIdx.x, (unsigned long long)c) : 0ull;
      cnt[threadIdx.x] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k)
      if (m[k].x != 0xFFFFFFFFu) {
        const uint32_t o = m[k].x & pmask;
        send[base[o] + atomicAdd(cnt + o, 1u)] = m[k];
      }
    __syncthreads();
  }
}

// Light/heavy row partition for the split relaxation: each row's (col, w) pairs are
// written to `out` light-first (w < h, compared as u32 bits: valid for integer and for
// non-negative f32 weights), both classes in their original order, and nlight[u] records
// the light count.  One warp per row; rows are independent.
__global__ void partition_rows_kernel(const unsigned long long* off, const uint2* adj, uint2* out,
                                      uint32_t* nlight, unsigned long long n, uint32_t h) {
  const int lane = threadIdx.x & 31;
  const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nw = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  for (unsigned long long u = w0; u < n; u += nw) {
    const unsigned long long lo = off[u], hi = off[u + 1];
    unsigned nl = 0;
    for (unsigned long long k0 = lo; k0 < hi; k0 += 32) {
      const unsigned long long k = k0 + lane;
      nl += __popc(__ballot_sync(FULL, k < hi && adj[k].y < h));
    }
    unsigned ls = 0, hs = 0;
    for (unsigned long long k0 = lo; k0 < hi; k0 += 32) {
      const unsigned long long k = k0 + lane;
      const bool has = k < hi;
      const uint2 x = has ? adj[k] : make_uint2(0u, 0u);
      const bool light = has && x.y < h;
      const unsigned lm = __ballot_sync(FULL, light), hm = __ballot_sync(FULL, has && !light);
      if (light) out[lo + ls + __popc(lm & lanemask_lt())] = x;
      else if (has) out[lo + nl + hs + __popc(hm & lanemask_lt())] = x;
      ls += __popc(lm);
      hs += __popc(hm);
    }
    if (lane == 0) nlight[u] = nl;
  }
}

// u32 device distances -> u64 API distances (INF -> 2^64-1), in caller vertex order
// (perm = caller id -> device id of a relabeled graph, or null).
__global__ void widen_kernel(const uint32_t* in, unsigned long long* out, unsigned long long n,
                             const uint32_t* perm) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < n; i += stride) {
    const uint32_t v = in[perm ? __ldg(perm + i) : i];
    out[i] = v == 0xFFFFFFFFu ? ~0ull : (unsigned long long)v;
  }
}

// out[i] = in[perm[i]]: device-order distances back to caller order (4- or 8-byte words).
template <class T>
__global__ void gather_kernel(const T* in, T* out, unsigned long long n, const uint32_t* perm) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < n; i += stride) out[i] = in[__ldg(perm + i)];
}

// ---- vertex relabeling by in-degree class (B200 layout; see ensure_relabel) ----
// indeg[v] += 1 per edge targeting v; warp-aggregated when a warp's lanes share a target
// (the hubs of a power-law graph take most of the edges).
__global__ void indeg_kernel(const uint2* adj, unsigned long long m, uint32_t* indeg) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (unsigned long long k0 = tid - lane; k0 < m; k0 += stride) {
    const unsigned long long k = k0 + lane;
    const bool has = k < m;
    const uint32_t v = has ? adj[k].x : 0xFFFFFFFFu;
    const unsigned peers = __match_any_sync(FULL, v);
    if (has && (__ffs(peers) - 1) == lane) atomicAdd(indeg + v, (uint32_t)__popc(peers));
  }
}

// key[v] = in-degree class, hottest first: 4 classes per octave of in-degree, vertices that
// no edge reaches last; val[v] = v.  Also max in-degree into *mx.
__global__ void relabel_keys_kernel(const uint32_t* indeg, unsigned long long n, uint8_t* key, uint32_t* val,
                                    unsigned int* mx) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned int m = 0;
  for (unsigned long long i = tid; i < n; i += stride) {
    const uint32_t d = indeg[i];
    m = d > m ? d : m;
    int k = 255;
    if (d > 0) {
      const int lg = 31 - __clz(d);                                   // octave
      const int sub = lg >= 2 ? (int)((d >> (lg - 2)) & 3u) : (int)(d & ((1u << lg) - 1u)) << (2 - lg);
      k = 254 - (lg * 4 + sub);                                       // 2^31 -> 130, 1 -> 254
    }
    key[i] = (uint8_t)k;
    val[i] = (uint32_t)i;
  }
  m = __reduce_max_sync(FULL, m);
  if ((threadIdx.x & 31) == 0) atomicMax(mx, m);
}

// Per class key: number of vertices and in-edges (mass[256] and cnt[256], zeroed by the
// caller) -- the host picks the hot prefix that takes 95 % of the edge targets.
__global__ void class_mass_kernel(const uint32_t* indeg, const uint8_t* key, unsigned long long n,
                                  unsigned long long* mass, unsigned long long* cnt) {
  __shared__ unsigned long long sm[256], sc[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = sc[i] = 0;
  __syncthreads();
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < n; i += stride) {
    atomicAdd(&sm[key[i]], (unsigned long long)indeg[i]);
    atomicAdd(&sc[key[i]], 1ull);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (sc[i]) {
      atomicAdd(mass + i, sm[i]);
      atomicAdd(cnt + i, sc[i]);
    }
}

// perm[iperm[i]] = i; ndeg[i] = degree of the vertex that becomes row i.
__global__ void relabel_perm_kernel(const uint32_t* iperm, const unsigned long long* off, unsigned long long n,
                                    uint32_t* perm, unsigned long long* ndeg) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < n; i += stride) {
    const uint32_t u = iperm[i];
    perm[u] = (uint32_t)i;
    ndeg[i] = off[u + 1] - off[u];
  }
  if (tid == 0) ndeg[n] = 0;
}

// Row i of the relabeled CSR = row iperm[i] of the old one, targets renamed through perm,
// edge order kept.  One warp per row.
__global__ void relabel_rows_kernel(const unsigned long long* off, const uint2* adj, const uint32_t* iperm,
                                    const uint32_t* perm, const unsigned long long* noff, uint2* nadj,
                                    unsigned long long n) {
  const int lane = threadIdx.x & 31;
  const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nw = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
  for (unsigned long long i = w0; i < n; i += nw) {
    const uint32_t u = iperm[i];
    const unsigned long long lo = off[u], hi = off[u + 1], o = noff[i];
    for (unsigned long long k = lo + lane; k < hi; k += 32) {
      uint2 x = adj[k];
      x.x = __ldg(perm + x.x);
      nadj[o + (k - lo)] = x;
    }
  }
}

// V_reach / E_reach of the device distances.
template <class S>
__global__ void reach_kernel(const S* dist, S inf, const unsigned long long* off,
                             unsigned long long n, unsigned long long* out) {
  unsigned long long v = 0, e = 0;
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long i = tid; i < n; i += stride)
    if (dist[i] != inf) {
      ++v;
      e += off[i + 1] - off[i];
    }
  v = warp_sum_u64(v);
  e = warp_sum_u64(e);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, v);
    atomicAdd(out + 1, e);
  }
}

// 128-bit accumulate (lo, hi) for exact sums of squares
__device__ __forceinline__ void add128(unsigned long long* lo_hi, unsigned long long x) {
  const unsigned long long old = atomicAdd(lo_hi, x);
  if (old + x < old) atomicAdd(lo_hi + 1, 1ull);
}

// K4 (extract_features graph.py:428-460) as exact integer sums:
// out: [0] sum deg, [1..2] sum deg^2 (lo, hi), [3] max deg,
//      [4] sum w, [5..6] sum w^2 (lo, hi), [7] max w     (integer weights)
__global__ void feature_sums_kernel(const unsigned long long* off, const uint2* adj,
                                    unsigned long long n, unsigned long long m, int unit,
                                    unsigned long long* out) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long sd = 0, sd2 = 0, sd2_hi = 0, md = 0, sw = 0, sw2 = 0, sw2_hi = 0, mw = 0;
  for (unsigned long long i = tid; i < n; i += stride) {
    const unsigned long long d = off[i + 1] - off[i];
    sd += d;
    const unsigned long long before = sd2;
    sd2 += d * d;
    sd2_hi += sd2 < before;
    md = d > md ? d : md;
  }
  for (unsigned long long k = tid; k < m; k += stride) {
    const unsigned long long w = unit ? 1ull : (unsigned long long)adj[k].y;
    sw += w;
    const unsigned long long before = sw2;
    sw2 += w * w;
    sw2_hi += sw2 < before;
    mw = w > mw ? w : mw;
  }
  atomicAdd(out + 0, sd);
  add128(out + 1, sd2);
  if (sd2_hi) atomicAdd(out + 2, sd2_hi);
  atomicMax(out + 3, md);
  atomicAdd(out + 4, sw);
  add128(out + 5, sw2);
  if (sw2_hi) atomicAdd(out + 6, sw2_hi);
  atomicMax(out + 7, mw);
}

// float-weight features: out[0] = sum w, out[1] = sum w^2 (double), maxbits = max w bits
__global__ void feature_sums_f32_kernel(const uint2* adj, unsigned long long m, double* out,
                                        unsigned int* maxbits) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  double sw = 0, sw2 = 0;
  unsigned int mw = 0;
  for (unsigned long long k = tid; k < m; k += stride) {
    const unsigned int b = adj[k].y;
    const double w = (double)__uint_as_float(b);
    sw += w;
    sw2 += w * w;
    mw = b > mw ? b : mw;
  }
  atomicAdd(out + 0, sw);
  atomicAdd(out + 1, sw2);
  atomicMax(maxbits, mw);
}

}  // namespace mlmq
