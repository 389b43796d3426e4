// mlmq_kernel.cuh — K1 persistent MLMQ relax kernel + K2 manager warp (sm_100a).
//
// One warp = one worker group, one lane = one lane.  Per warp:
//   L0  per-lane FIFOs of l0_capacity elements held in REGISTERS (l1.py:21-96)
//   L1  a warp-private shared-memory ring: vector / near_far / filter / slf (l1.py:99-280)
//   L2  shared HBM queue: ticketed block ring FIFO, Δ-bucket window over rings, or
//       lock-protected batch heaps (l2.py:73-451)
// behind the unified Read/Write cascade of compose.py:30-86 (PAPER Listing 1):
//   Read : L0 -> L1 -> hub items -> L2, served entirely from the first non-empty level;
//          a full miss flushes local_done into global done (l2.py:56-62).
//   Write: L0 -> (full transfer) L1 -> (write-back) L2.
// Relaxation (engine.py:171-227) is warp-cooperative: dup-elim, degree split at th_v,
// flattened load-balanced expansion of small lists, warp-strided walks of big lists,
// hub lists split into edge-range work items shared by all warps, atomicMin on dist.
// Termination is the delayed-count protocol of PAPER.md:589 / l2.py:33-70, counted in
// queue units (blocks written/read), checked by a manager warp that needs three
// consecutive equal observations (engine.py:32-33, 152-169).
#pragma once
#include "common.cuh"

namespace mlmq {

#ifndef MLMQ_COLD_RING
#define MLMQ_COLD_RING 0  // measured slower (caller-side spills in the hot loop), see r2_experiments.md
#endif

// The L2 block-ring writer (l2.py:96-114) as an out-of-line FREE function.  It runs a few
// thousand times per solve but, inlined at every cascade-write and flush site, it was
// ~8 K of the K1 variant's 23 K SASS instructions and pushed the hot read/relax loop out of
// the instruction cache (ncu: 17 % of C2 stall samples "no instruction").  A member
// function would take `this` and force the Worker into local memory (measured +50 % in
// round 2), so everything it needs is passed by value.  Per-slot Vyukov sequence numbers:
// one fetch-add claims ceil(n/bs) tickets; slot waits, element stores and publications
// proceed lane-parallel.  Returns false after raising an overflow error (spin timeout) or
// when the solve is stopping.
template <class E, int L2K>
__device__ __noinline__ bool ring_write_cold(const KParams* pp, int rid, const E* base, int start, int n, int cap,
                                             int lane) {
  const KParams& p = *pp;
  const int bs = p.bs;
  const int nseg = (n + bs - 1) / bs;
  unsigned long long t = 0;
  unsigned long long* wpr = p.ptrs + (size_t)rid * 32;
  if (lane == 0) t = atomicAdd(wpr, (unsigned long long)nseg);
  t = __shfl_sync(FULL, t, 0);
  bool ok = true;
  for (int sg = lane; sg < nseg; sg += 32) {  // wait until the claimed slots are free
    const unsigned long long tk = t + sg, slot = tk & p.bn_mask;
    const unsigned long long* sp = p.seq + (size_t)rid * (p.bn_mask + 1) + slot;
    unsigned long long t0 = 0;
    int spins = 0, ns = 32;
    while (ok && ld_acquire(sp) != tk) {
      if (++spins % 64 == 0) {
        if (ld_relaxed(p.ctl + C_STOP) != 0) { ok = false; break; }
        const unsigned long long now = globaltimer_ns();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > p.spin_timeout_ns) {
          if (atomicCAS(p.ctl + C_ERR, 0ull, (unsigned long long)ERR_OVERFLOW) == 0ull) {
            p.ctl[C_DIAG + 0] = (unsigned long long)rid;
            p.ctl[C_DIAG + 1] = slot;
            p.ctl[C_DIAG + 2] = ld_relaxed(wpr);
            p.ctl[C_DIAG + 3] = ld_relaxed(wpr + 16);
          }
          __threadfence();
          st_release(p.ctl + C_STOP, 1ull);
          ok = false;
          break;
        }
      }
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
    }
  }
  if (!__all_sync(FULL, ok)) return false;
  for (int i = lane; i < n; i += 32) {
    const int sg = i / bs;
    reinterpret_cast<E*>(p.data)[((size_t)rid * (p.bn_mask + 1) + ((t + sg) & p.bn_mask)) * bs + (i - sg * bs)] =
        base[(unsigned)(start + i) % (unsigned)cap];
  }
  __threadfence();
  __syncwarp();
  for (int sg = lane; sg < nseg; sg += 32) {
    const unsigned long long tk = t + sg, slot = tk & p.bn_mask;
    const size_t i = (size_t)rid * (p.bn_mask + 1) + slot;
    p.cnt[i] = (uint32_t)min(bs, n - sg * bs);
    st_release(p.seq + i, tk + 1);
  }
  __syncwarp();
  bool bump = true;
  if (L2K == L2K_BUCKET && p.bwin > 0) {  // managed floor: only near-window rings wake readers
    unsigned long long e = 0;
    if (lane == 0) e = ld_relaxed(p.ctl + C_EPOCH);
    const int emod = (int)(__shfl_sync(FULL, e, 0) % (unsigned long long)p.bmax);
    const int rel = rid >= emod ? rid - emod : rid + p.bmax - emod;
    bump = rel == 0 || rel == p.bmax - 1;
  }
  if (bump && lane == 0) red_add(p.ctl + C_GEN, 1ull);
  return true;
}

// Raise a queue error (QueueOverflowError analogue) and stop every warp: cold, out of line.
static __device__ __noinline__ void raise_error_cold(unsigned long long* ctl, int code, unsigned long long a,
                                              unsigned long long b, unsigned long long c, unsigned long long d) {
  if (atomicCAS(ctl + C_ERR, 0ull, (unsigned long long)code) == 0ull) {
    ctl[C_DIAG + 0] = a;
    ctl[C_DIAG + 1] = b;
    ctl[C_DIAG + 2] = c;
    ctl[C_DIAG + 3] = d;
  }
  __threadfence();
  st_release(ctl + C_STOP, 1ull);
}

template <int K, int L2K, int CM, int L1T>
struct Worker {
  using Tr = DT<K>;
  using S = typename Tr::S;
  using E = Elem<S>;
// MLMQ_U (common.cuh, default 4) measured on B200 (C2): U=2 2.26 ms, 3 1.69, 4 1.64, 5 1.78,
// 6 1.88, 8 1.98, 12 2.82
  static constexpr int U = MLMQ_U;  // edge slots per lane per step (U independent loads in flight)
#ifndef MLMQ_PIPE
#define MLMQ_PIPE 0  // 1: issue step k+1's adjacency loads before step k's checks (2U loads in flight)
#endif
#ifndef MLMQ_SHARE_MIN
#define MLMQ_SHARE_MIN (2 * L)  // eager sharing: local elements a group keeps before giving work away
#endif
#ifndef MLMQ_TPF
#define MLMQ_TPF 0  // 1: split relax step (adjacency issue / loaded check) with the target-offset prefetch
#endif
#ifndef MLMQ_DIRECT_TOKEN
#define MLMQ_DIRECT_TOKEN 0  // 1: improved targets without light edges become heavy tokens at once
#endif
#ifndef MLMQ_SMALLDEG
#define MLMQ_SMALLDEG 0  // 1: lane-per-row relaxation when every row of a sub-batch has <= U edges
#endif
#ifndef MLMQ_HUB_LAST
#define MLMQ_HUB_LAST 0  // 1: the read cascade tries the L2 queue before hub chunks
#endif
#ifndef MLMQ_SEARCH
#define MLMQ_SEARCH 0  // 1: owner lookup by REDUX over compacted row starts (expand_step_c)
#endif

  const KParams& p;
  S* dist;
  E* batch;
  E* outs;
  E* spill;
  E* l1a;
  E* l1b;
  E* fars;
  unsigned long long* met;
  unsigned long long* btick;  // bucket write scratch (smem): ticket base per bucket
  uint32_t* bhist;            // elements per bucket
  uint32_t* bcur;             // scatter cursor per bucket
  uint32_t* bremap;           // bucket -> ring actually written (occupancy-aware)
  uint32_t* bremap_row;       // expansion: start position -> owner lane (32 entries)
  int lane, gid, L;

  // L0: per-lane register FIFO (shift register, pop at index 0)
  uint32_t l0v[CM];
  S l0d[CM];
  int l0n;
  int wc, rc, l0size;

  // L1 (ring a: vector/filter/slf/near; ring b: far)
  int h1, n1, h2, n2;
  S thr, rej_min;
  bool has_rej;
  int wcount;

  unsigned long long local_done;
  unsigned n_relax, n_upd;  // relaxations (per lane) / distance updates (warp), folded at exit
  int mcursor;
  int outn;
  int nfar;  // far elements staged (bucket window)
  int nhvy;  // heavy tokens staged (light/heavy split), at fars + far_cap
  bool dist_ovf;
  bool idle;
  int last_src;  // level that served the current batch (1 L0, 2 L1, 3 L2) for diagnostics
  // sharded solve: this group's private slice of the outbox (reserved kOboxChunk slots at
  // a time with one fetch-add, so 2663 groups do not serialise on one counter)
  unsigned long long ob_next;
  unsigned ob_left;
  // bucket floor as last read by this group's bucket_read.  While the group holds work its
  // unflushed done count keeps the floor from moving, so far_split can bin against it
  // without another round trip (a stale, lower floor only sends more elements "far",
  // where bucket_write re-bins them against the current floor).
  unsigned long long ep_seen;

  __device__ Worker(const KParams& prm, unsigned char* sm, int g, int ln) : p(prm), lane(ln), gid(g) {
    L = p.L;
    dist = reinterpret_cast<S*>(p.dist);
    E* base = reinterpret_cast<E*>(sm);
    batch = base;
    outs = batch + p.batch_cap;
    spill = outs + p.out_cap;
    l1a = spill + p.spill_cap;
    l1b = l1a + p.l1cap;
    const int l1n = (L1T == L1K_NEAR_FAR ? 2 : 1) * p.l1cap;
    fars = l1a + l1n;  // far staging (bucket window), p.far_cap elements
    met = reinterpret_cast<unsigned long long*>(fars + p.far_cap + p.hvy_cap);  // heavy-token stage before it
    met[lane] = 0;  // metric + profile slots (kMetSlots == 32)
    btick = met + kMetSlots;
    bhist = reinterpret_cast<uint32_t*>(btick + (p.bscratch ? p.bmax : 0));
    bcur = bhist + (p.bscratch ? p.bmax : 0);
    bremap = bcur + (p.bscratch ? p.bmax : 0);
    bremap_row = bremap + (p.bscratch ? p.bmax : 0);  // 32 u32: row owner map (expansion)
    l0n = 0;
    wc = rc = l0size = 0;
    h1 = n1 = h2 = n2 = 0;
    thr = (S)(L1T == L1K_NEAR_FAR ? p.delta_nf_s : p.filter_f_s);
    rej_min = (S)Tr::INF;
    has_rej = false;
    wcount = 0;
    local_done = 0;
    n_relax = n_upd = 0;
    mcursor = p.pnum > 0 ? gid % p.pnum : 0;
    outn = 0;
    nfar = 0;
    nhvy = 0;
    dist_ovf = false;
    pend = ~0ull;
    idle = false;
    ob_next = 0;
    ob_left = 0;
    ep_seen = 0;
    __syncwarp();
  }

  __device__ __forceinline__ void count(int f, unsigned long long v) {
    if (lane == 0) met[f] += v;
  }
  // debug profile (MLMQ_DEBUG=1): cycles per phase, counts
  __device__ __forceinline__ unsigned long long pclk() const { return (kDebug && p.prof) ? clock64() : 0ull; }
  __device__ __forceinline__ void pacc(int slot, unsigned long long t0) {
    if ((kDebug && p.prof) && lane == 0) met[kProfBase + slot] += clock64() - t0;
  }
  __device__ __forceinline__ void pcnt(int slot, unsigned long long v) {
    if ((kDebug && p.prof) && lane == 0) met[kProfBase + slot] += v;
  }
// Per-lane source-line trace (build with -DMLMQ_TRACE, run with MLMQ_DEBUG=1): the stuck
// dump prints every lane's last line, which exposes lanes that left warp-uniform flow.
#ifdef MLMQ_TRACE
#define LOC() trace(__LINE__)
#else
#define LOC() ((void)0)
#endif
#define CHKU() check_uniform(__LINE__)
  // debug: every "warp-uniform" scalar of the worker must agree with lane 0
  __device__ void check_uniform(int line) {
    if (!(kDebug && p.wstate)) return;
    unsigned long long h = (unsigned long long)l0size ^ ((unsigned long long)n1 << 13) ^
                           ((unsigned long long)n2 << 26) ^ ((unsigned long long)outn << 39) ^
                           ((unsigned long long)h1 << 45) ^ ((unsigned long long)h2 << 51) ^
                           ((unsigned long long)wc << 57) ^ ((unsigned long long)rc << 3) ^
                           ((unsigned long long)thr * 0x9E3779B97F4A7C15ull) ^ (local_done * 0x100000001B3ull) ^
                           ((unsigned long long)wcount << 20) ^ ((unsigned long long)idle << 62) ^
                           ((unsigned long long)has_rej << 61) ^ ((unsigned long long)rej_min * 31ull);
    const unsigned long long h0 = __shfl_sync(FULL, h, 0);
    const unsigned bad = __ballot_sync(FULL, h != h0);
    if (bad && lane == 0) raise_error(ERR_CORRUPT, 7000000ull + line, bad, (unsigned long long)gid, h0);
  }
  __device__ __forceinline__ void trace(int line) {
    if (kDebug && p.wstate) p.wstate[2 * (size_t)p.G + 8 + (size_t)gid * 32 + lane] = (unsigned long long)line;
  }
  // debug: where the warp is and its local queue sizes (wstate[G + gid])
  __device__ __forceinline__ void loc(int ph) {
    if ((kDebug && p.wstate) && lane == 0)
      p.wstate[p.G + gid] = ((unsigned long long)ph << 56) | ((unsigned long long)(l0size & 0xFFFF) << 40) |
                            ((unsigned long long)(n1 & 0xFFFF) << 24) | ((unsigned long long)(n2 & 0xFFF) << 12) |
                            (unsigned long long)(outn & 0xFFF);
  }
  __device__ __forceinline__ void wstate(int code, unsigned long long tk) {
    if (kDebug && p.wstate) p.wstate[gid] = ((unsigned long long)code << 56) | (tk & ((1ull << 56) - 1));
  }
  // per-lane check, only for spins that a single lane runs
  __device__ __forceinline__ bool stopped() const {
    return ld_relaxed(p.ctl + C_STOP) != 0;
  }
  // warp-uniform check (lane 0 loads, everyone agrees) for warp control flow
  __device__ __forceinline__ bool stopped_warp() const {
    int s = 0;
    if (lane == 0) s = ld_relaxed(p.ctl + C_STOP) != 0;
    return __shfl_sync(FULL, s, 0) != 0;
  }
  // A global word read by lane 0 and broadcast: concurrent writers can make a warp-wide
  // load of one address return different values to different lanes, so every global
  // value that steers warp control flow is read this way.
  __device__ __forceinline__ unsigned long long warp_ld(const unsigned long long* a) const {
    unsigned long long v = 0;
    if (lane == 0) v = ld_relaxed(a);
    return __shfl_sync(FULL, v, 0);
  }
  // Work generation (B200 extension): bumped after every publication of new shared work
  // (ring block, hub descriptor, heap node, floor advance).  An idle group polls this
  // one word (with the stop flag beside it) instead of re-walking the whole cascade.
  // managed floor: is ring rid the head or the ring behind it (claimable by readers)?
  __device__ __forceinline__ bool near_ring(int rid, int emod) const {
    const int rel = rid >= emod ? rid - emod : rid + p.bmax - emod;
    return rel == 0 || rel == p.bmax - 1;
  }
  __device__ __forceinline__ void bump_gen() const {
    if (lane == 0) red_add(p.ctl + C_GEN, 1ull);
  }
  __device__ __forceinline__ unsigned long long* wp(int r) const { return p.ptrs + (size_t)r * 32; }
  __device__ __forceinline__ unsigned long long* rp(int r) const { return p.ptrs + (size_t)r * 32 + 16; }

  // Raise a queue error (QueueOverflowError analogue) and stop every warp.
  __device__ void raise_error(int code, unsigned long long a, unsigned long long b,
                              unsigned long long c, unsigned long long d) {
#if MLMQ_COLD_RING >= 2
    if (!kDebug) {
      raise_error_cold(p.ctl, code, a, b, c, d);
      return;
    }
#endif
    if (atomicCAS(p.ctl + C_ERR, 0ull, (unsigned long long)code) == 0ull) {
      p.ctl[C_DIAG + 0] = a;
      p.ctl[C_DIAG + 1] = b;
      p.ctl[C_DIAG + 2] = c;
      p.ctl[C_DIAG + 3] = d;
    }
    __threadfence();
    st_release(p.ctl + C_STOP, 1ull);
  }

  // ============================================================ L0 (registers)
  __device__ __forceinline__ void l0_push(uint32_t v, S d) {
#pragma unroll
    for (int j = 0; j < CM; ++j)
      if (j == l0n) { l0v[j] = v; l0d[j] = d; }
    ++l0n;
  }
  __device__ __forceinline__ void l0_pop(uint32_t& v, S& d) {
    v = l0v[0];
    d = l0d[0];
#pragma unroll
    for (int j = 0; j + 1 < CM; ++j) { l0v[j] = l0v[j + 1]; l0d[j] = l0d[j + 1]; }
    --l0n;
  }

  // Drain every lane, lanes in round-robin order from the read cursor, each lane FIFO
  // (l1.py:87-96).  Returns the number of elements written to dst.
  __device__ int l0_drain(E* dst) {
    LOC();
    const int q = lane;
    const int srcl = (rc + q) % L;
    int c = __shfl_sync(FULL, l0n, srcl);
    if (q >= L) c = 0;
    int incl = warp_incl_scan(c, lane);
    const int total = __shfl_sync(FULL, incl, 31);
    const int excl_q = incl - c;
    const int r = (lane - rc + L) % L;
    const int ex = __shfl_sync(FULL, excl_q, r & 31);
    if (lane < L) {
#pragma unroll
      for (int j = 0; j < CM; ++j)
        if (j < l0n) {
          E e;
          e.v = l0v[j];
          e.d = l0d[j];
          dst[ex + j] = e;
        }
      l0n = 0;
    }
    __syncwarp();
    return total;
  }

  // Pop up to `want`, one per non-empty lane per round from the read cursor
  // (l1.py:66-85); the cursor ends after the lane that gave the last element.
  __device__ int l0_read(E* dst, int want) {
    LOC();
    loc(11);
    const int T = min(want, l0size);
    int taken = 0, last = 0;
    const unsigned lmask = (L == 32) ? FULL : ((1u << L) - 1u);
    const int r = (lane - rc + L) % L;
    while (taken < T) {
      LOC();
      const bool ne = lane < L && l0n > 0;
      const unsigned m = __ballot_sync(FULL, ne);
      const unsigned rot = rc == 0 ? m : (((m >> rc) | (m << (L - rc))) & lmask);
      const int rank = __popc(rot & ((1u << r) - 1u));
      const int a = __popc(m);
      const int t = min(a, T - taken);
      const bool take = ne && rank < t;
      if (take) {
        uint32_t v;
        S d;
        l0_pop(v, d);
        E e;
        e.v = v;
        e.d = d;
        dst[taken + rank] = e;
      }
      const unsigned tm = __ballot_sync(FULL, take && rank == t - 1);
      last = __ffs(tm) - 1;
      taken += t;
    }
    rc = (last + 1) % L;
    l0size -= T;
    __syncwarp();
    CHKU();
    return T;
  }

  // ============================================================ L2: block rings
  // Per-slot sequence numbers (Vyukov): slot s is free for ticket t when seq == t,
  // holds ticket t's block when seq == t + 1, and is freed by the reader to t + bn.
  // Unlike the reference's bare tags (l2.py:110-114) this is ABA-safe on wrap-around.
  __device__ __forceinline__ unsigned long long* seq_ptr(int rid, unsigned long long slot) const {
    return p.seq + (size_t)rid * (p.bn_mask + 1) + slot;
  }
  __device__ __forceinline__ E* slot_data(int rid, unsigned long long slot) const {
    return reinterpret_cast<E*>(p.data) + ((size_t)rid * (p.bn_mask + 1) + slot) * p.bs;
  }

  // Per-lane bounded spin until *s == want; false on stop or timeout (overflow error).
  __device__ bool lane_spin(const unsigned long long* s, unsigned long long want, int rid,
                            unsigned long long slot) {
    unsigned long long t0 = 0;
    int spins = 0, ns = 32;
    while (ld_acquire(s) != want) {
      LOC();
      if (++spins % 64 == 0) {
        if (stopped()) return false;
        const unsigned long long now = globaltimer_ns();
        if (t0 == 0) t0 = now;
        else if (now - t0 > p.spin_timeout_ns) {
          raise_error(ERR_OVERFLOW, (unsigned long long)rid, slot, ld_relaxed(wp(rid)), ld_relaxed(rp(rid)));
          return false;
        }
      }
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
    }
    return true;
  }

  // Wait (lanes in parallel) until the nseg slots of tickets t..t+nseg-1 are free.
  __device__ bool wait_free(int rid, unsigned long long t, int nseg) {
    LOC();
    bool ok = true;
    if (lane == 0) wstate(W_RING_WRITE, t);
    for (int sg = lane; sg < nseg; sg += 32) {
      LOC();
      const unsigned long long tk = t + sg, slot = tk & p.bn_mask;
      if (ok && !lane_spin(seq_ptr(rid, slot), tk, rid, slot)) ok = false;
    }
    ok = __all_sync(FULL, ok);
    if (lane == 0) wstate(W_NONE, 0);
    return ok;
  }

  // Publish (lanes in parallel) the nseg blocks of tickets t.. holding `n` elements.
  __device__ void publish_all(int rid, unsigned long long t, int nseg, int n) {
    LOC();
    __threadfence();
    __syncwarp();
    for (int sg = lane; sg < nseg; sg += 32) {
      LOC();
      const unsigned long long tk = t + sg, slot = tk & p.bn_mask;
      const size_t i = (size_t)rid * (p.bn_mask + 1) + slot;
      p.cnt[i] = (uint32_t)min(p.bs, n - sg * p.bs);
      st_release(p.seq + i, tk + 1);
    }
    __syncwarp();
    if (L2K == L2K_BUCKET && p.bwin > 0) {  // warp-uniform here
      const int emod = (int)(warp_ld(p.ctl + C_EPOCH) % (unsigned long long)p.bmax);
      if (near_ring(rid, emod)) bump_gen();
    } else {
      bump_gen();
    }
  }

  // Writer (l2.py:96-114): one fetch-add claims ceil(n/bs) tickets; all slot waits,
  // element stores and publications of the write proceed warp-parallel.
  __device__ void ring_write(int rid, const E* base, int start, int n, int cap) {
    LOC();
    if (n <= 0) return;
#if MLMQ_COLD_RING
    if (!kDebug) {  // the debug builds keep the inlined form with its wait-state hooks
      count(M_L2A, 1);
      ring_write_cold<E, L2K>(&p, rid, base, start, n, cap, lane);
      return;
    }
#endif
    const int bs = p.bs;
    const int nseg = (n + bs - 1) / bs;
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(wp(rid), (unsigned long long)nseg);
    t = __shfl_sync(FULL, t, 0);
    count(M_L2A, 1);
    if (!wait_free(rid, t, nseg)) return;
    for (int i = lane; i < n; i += 32) {
      LOC();
      const int sg = i / bs;
      slot_data(rid, (t + sg) & p.bn_mask)[i - sg * bs] = base[(unsigned)(start + i) % (unsigned)cap];
    }
    publish_all(rid, t, nseg, n);
  }

  // Same, with the elements held one per lane (grp = writing lanes, rank within grp).
  __device__ void ring_write_lanes(int rid, unsigned grp, int rank, const E& x, bool mine) {
    LOC();
    const int c = __popc(grp);
    const int bs = p.bs;
    const int nseg = (c + bs - 1) / bs;
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(wp(rid), (unsigned long long)nseg);
    t = __shfl_sync(FULL, t, 0);
    count(M_L2A, 1);
    if (!wait_free(rid, t, nseg)) return;
    if (mine) {
      const int sg = rank / bs;
      slot_data(rid, (t + sg) & p.bn_mask)[rank - sg * bs] = x;
    }
    publish_all(rid, t, nseg, c);
  }

  // Copy ticket r's published block out and free the slot.
  __device__ int take_block(int rid, unsigned long long r, E* dst) {
    LOC();
    const unsigned long long slot = r & p.bn_mask;
    const size_t i = (size_t)rid * (p.bn_mask + 1) + slot;
    int c = 0;
    if (lane == 0) c = (int)__ldcg(p.cnt + i);
    c = __shfl_sync(FULL, c, 0);
    if (c < 0 || c > p.bs) {
      if (lane == 0) raise_error(ERR_CORRUPT, 10ull + rid, (unsigned long long)c, (unsigned long long)gid, r);
      return 0;
    }
    const E* d = slot_data(rid, slot);
    for (int k = lane; k < c; k += 32) dst[k] = ld_cg_elem(d + k);
    __syncwarp();
    if (lane == 0) st_release(p.seq + i, r + p.bn_mask + 1);
    local_done += 1;  // every consumed ticket is one termination unit (l2.py:56-62)
    pcnt(P_NL2R, 1);
    return c;
  }

  // Conditional reader (l2.py:137-162): claim a ticket only when a written block
  // exists, then wait for the in-flight writer; never leaves a dangling claim.
  __device__ int ring_read(int rid, E* dst) {
    LOC();
    unsigned long long r = 0, elo = 0;
    int got = 0;
    bool ok = true, empty = false;
    if (lane == 0) {
      unsigned long long* rpp = rp(rid);
      unsigned long long* wpp = wp(rid);
      r = ld_relaxed(rpp);
      unsigned long long w = ld_relaxed(wpp);
      if (r < w) {
        // One fetch-add claims a ticket (no CAS retry storm).  A racing reader can
        // over-claim past the write pointer; it then either waits for the writer that
        // already owns its ticket, or takes every ticket from the write pointer up to
        // its own as a writer (ONE CAS) and publishes them as EMPTY blocks: each is
        // consumed by the over-claimer that holds it (reserve and done both count it),
        // so no claim is ever left dangling (the audit's "no pending tickets",
        // engine.py:241-242), and a burst of k over-claims resolves in one round trip
        // instead of a k-long chain of CAS hand-offs.
        r = atomicAdd(rpp, 1ull);
        got = 1;
        unsigned long long t0 = 0;
        int spins = 0;
        while ((w = ld_relaxed(wpp)) <= r) {
          if (atomicCAS(wpp, w, r + 1) == w) { empty = true; elo = w; break; }
          if (++spins % 64 == 0) {
            if (stopped()) { ok = false; break; }
            const unsigned long long now = globaltimer_ns();
            if (t0 == 0) t0 = now;
            else if (now - t0 > p.spin_timeout_ns) {
              raise_error(ERR_OVERFLOW, (unsigned long long)rid, r & p.bn_mask, w, r);
              ok = false;
              break;
            }
          }
          __nanosleep(32);
        }
      }
    }
    got = __shfl_sync(FULL, got, 0);
    if (!got) return 0;
    r = __shfl_sync(FULL, r, 0);
    count(M_L2A, 1);
    if (__shfl_sync(FULL, (int)empty, 0)) {  // publish the empty blocks elo..r, lanes in parallel
      elo = __shfl_sync(FULL, elo, 0);
      for (unsigned long long t = elo + (unsigned long long)lane; t <= r; t += 32) {
        const unsigned long long slot = t & p.bn_mask;
        if (ok && lane_spin(seq_ptr(rid, slot), t, rid, slot)) {  // slot free for ticket t
          p.cnt[(size_t)rid * (p.bn_mask + 1) + slot] = 0u;
          st_release(seq_ptr(rid, slot), t + 1);
        } else {
          ok = false;
        }
      }
      ok = __all_sync(FULL, ok);
    }
    if (lane == 0 && ok) {
      const unsigned long long slot = r & p.bn_mask;
      wstate(W_RING_READ, r + 1);
      ok = lane_spin(seq_ptr(rid, slot), r + 1, rid, slot);
      wstate(W_NONE, 0);
    }
    if (!__shfl_sync(FULL, (int)ok, 0)) return 0;
    __syncwarp();
    return take_block(rid, r, dst);
  }

  // Parked FIFO reader: one unconditional fetch-add takes the next
  // ticket; the ticket persists in a register ("pending", l2.py:151-154) and the warp
  // polls only its own slot, so idle warps do not contend on the read pointer.
  // Tickets still pending at termination are retired by the audit kernel.
  unsigned long long pend;
  __device__ int fifo_read(E* dst) {
    LOC();
    if (pend == ~0ull) {
      unsigned long long r = 0;
      if (lane == 0) r = atomicAdd(rp(0), 1ull);
      pend = __shfl_sync(FULL, r, 0);
      count(M_L2A, 1);
    }
    int ready = 0;
    if (lane == 0) ready = ld_acquire(seq_ptr(0, pend & p.bn_mask)) == pend + 1;
    if (!__shfl_sync(FULL, ready, 0)) return 0;
    __syncwarp();
    const int c = take_block(0, pend, dst);
    pend = ~0ull;
    return c;
  }

  // ============================================================ L2: bucket window
  // ring of bucket rel relative to epoch e (emod = e % bmax)
  __device__ __forceinline__ int bring(int emod, int rel) const {
    const int x = emod + rel;
    return x >= p.bmax ? x - p.bmax : x;
  }
  // l2.py:209-222 clamps far elements to bmax-1; with managed epochs that ring is the one
  // just behind the floor (read first), so far elements clamp one ring earlier
  __device__ __forceinline__ int rel_clamp() const { return p.bwin > 0 ? p.bmax - 2 : p.bmax - 1; }
  __device__ __forceinline__ int bucket_rel(S d, unsigned long long e) const {
    if (K == DK_F32) {
      const double base = (double)e * p.delta_f;
      const double dv = (double)__uint_as_float((uint32_t)d);
      if (dv < base) return 0;
      const double q = floor((dv - base) / p.delta_f);
      return q >= (double)rel_clamp() ? rel_clamp() : (int)q;
    } else {
      const unsigned long long base = e * p.delta_i;
      const unsigned long long dd = (unsigned long long)d;
      if (dd < base) return 0;
      const unsigned long long diff = dd - base;
      unsigned long long q;
      if ((diff >> 32) == 0 && (p.delta_i >> 32) == 0)
        q = (unsigned)diff / (unsigned)p.delta_i;  // 32-bit divide on the common path
      else
        q = diff / p.delta_i;
      return q >= (unsigned long long)rel_clamp() ? rel_clamp() : (int)q;
    }
  }

  // Group the lanes' elements by target bucket ring and write each group as blocks.
  __device__ void bucket_scatter_lanes(bool has, const E& x, int f) {
    LOC();
    unsigned act = __ballot_sync(FULL, has);
    while (act) {
      LOC();
      const int leader = __ffs(act) - 1;
      const int fl = __shfl_sync(FULL, f, leader);
      const bool mine = has && f == fl;
      const unsigned grp = __ballot_sync(FULL, mine);
      const int rank = __popc(grp & lanemask_lt());
      ring_write_lanes(fl, grp, rank, x, mine);
      act &= ~grp;
    }
  }

  // l2.py:209-233: rel = 0 below the floor, (d-base)//Δ above, clamped to bmax-1.
  // Warp-parallel: (1) per-bucket histogram in shared memory, (2) one ticket fetch-add
  // per non-empty bucket, (3) parallel slot waits, (4) scatter, (5) parallel publish.
  __device__ void bucket_write(const E* base, int start, int n, int cap) {
    LOC();
    const unsigned long long e = warp_ld(p.ctl + C_EPOCH);
    const int emod = (int)(e % (unsigned long long)p.bmax);
    if (!p.bscratch) {  // very wide windows: per-round grouping
      for (int o = 0; o < n; o += 32) {
        LOC();
        const bool has = o + lane < n;
        E x = E();
        int f = 0;
        if (has) {
          x = base[(unsigned)(start + o + lane) % (unsigned)cap];
          f = bring(emod, bucket_rel(x.d, e));
        }
        bucket_scatter_lanes(has, x, f);
      }
      return;
    }
    const int bs = p.bs;
    // Occupancy-aware placement: a bucket ring that is nearly full (pending blocks within
    // `ring_margin` of capacity) passes its elements on to the next ring.  Any ring is a
    // correct home (the reader rebins or processes them), so a burst of far work can no
    // longer wedge a writer on a full ring while the floor waits for near work.
    const long long room = (long long)(p.bn_mask + 1) - p.ring_margin;
    for (int b = lane; b < p.bmax; b += 32) {
      bhist[b] = 0;
      bcur[b] = 0;
      bremap[b] = b;
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      LOC();
      const E x = base[(unsigned)(start + i) % (unsigned)cap];
      atomicAdd(bhist + bring(emod, bucket_rel(x.d, e)), 1u);
    }
    __syncwarp();
    bool anyfull = false;  // occupancy of the rings this write uses (one load pair each)
    for (int b = lane; b < p.bmax; b += 32)
      if (bhist[b]) anyfull |= (long long)(ld_relaxed(wp(b)) - ld_relaxed(rp(b))) > room;
    if (__any_sync(FULL, anyfull)) {
      for (int b = lane; b < p.bmax; b += 32)
        bcur[b] = (long long)(ld_relaxed(wp(b)) - ld_relaxed(rp(b))) > room ? 1u : 0u;
      __syncwarp();
      for (int b = lane; b < p.bmax; b += 32) {
        // move only farther from the floor and never past the clamp ring: an element is
        // never placed where it would be rebinned straight back (no livelock)
        int t = b;
        int rel = b >= emod ? b - emod : b + p.bmax - emod;
        while (bcur[t] && rel > 0 && rel < rel_clamp()) {
          t = t + 1 == p.bmax ? 0 : t + 1;
          ++rel;
        }
        bremap[b] = bcur[t] ? b : t;  // no room anywhere farther: keep the home ring (bounded wait)
      }
      __syncwarp();
      for (int b = lane; b < p.bmax; b += 32) {
        bcur[b] = 0;
        bhist[b] = 0;
      }
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        const E x = base[(unsigned)(start + i) % (unsigned)cap];
        atomicAdd(bhist + bremap[bring(emod, bucket_rel(x.d, e))], 1u);
      }
      __syncwarp();
    }
    int used = 0;
    for (int b = lane; b < p.bmax; b += 32) {
      LOC();
      const int c = (int)bhist[b];
      if (c) {
        btick[b] = atomicAdd(wp(b), (unsigned long long)((c + bs - 1) / bs));
        ++used;
      }
    }
    count(M_L2A, (unsigned long long)__reduce_add_sync(FULL, used));
    __syncwarp();
    bool ok = true;
    if (lane == 0) wstate(W_RING_WRITE, e);
    for (int b = lane; b < p.bmax; b += 32) {
      LOC();
      const int c = (int)bhist[b];
      const int nseg = (c + bs - 1) / bs;
      for (int sg = 0; ok && sg < nseg; ++sg) {
        LOC();
        const unsigned long long tk = btick[b] + sg, slot = tk & p.bn_mask;
        ok = lane_spin(seq_ptr(b, slot), tk, b, slot);
      }
    }
    if (lane == 0) wstate(W_NONE, 0);
    if (!__all_sync(FULL, ok)) return;
    for (int i = lane; i < n; i += 32) {
      LOC();
      const E x = base[(unsigned)(start + i) % (unsigned)cap];
      const int f = bremap[bring(emod, bucket_rel(x.d, e))];
      const int r = (int)atomicAdd(bcur + f, 1u);
      const int sg = r / bs;
      slot_data(f, (btick[f] + sg) & p.bn_mask)[r - sg * bs] = x;
    }
    __threadfence();
    __syncwarp();
    for (int b = lane; b < p.bmax; b += 32) {
      LOC();
      const int c = (int)bhist[b];
      const int nseg = (c + bs - 1) / bs;
      for (int sg = 0; sg < nseg; ++sg) {
        LOC();
        const unsigned long long tk = btick[b] + sg, slot = tk & p.bn_mask;
        const size_t i = (size_t)b * (p.bn_mask + 1) + slot;
        p.cnt[i] = (uint32_t)min(bs, c - sg * bs);
        st_release(p.seq + i, tk + 1);
      }
    }
    __syncwarp();
    // managed floor: only blocks in the head / behind rings are claimable now, so only
    // they wake idle groups (far rings wait for the manager's floor advance, which bumps)
    bool wake = !(p.bwin > 0);
    for (int b = lane; b < p.bmax; b += 32) wake |= bhist[b] && near_ring(b, emod);
    if (__any_sync(FULL, wake)) bump_gen();
  }

  // l2.py:235-295: scan bnum buckets from the floor; rebin stale-slot elements; advance
  // the floor by one when the head is seen empty while elements remain elsewhere.
  __device__ int bucket_read(E* dst) {
    LOC();
    loc(16);
    const unsigned long long e0 = warp_ld(p.ctl + C_EPOCH);
    ep_seen = e0;
    const int e0mod = (int)(e0 % (unsigned long long)p.bmax);
    bool head_empty = false;
    // managed epochs (bwin > 0): the ring just behind the floor is read first -- it holds
    // elements binned against a floor that has since advanced
    const int j0 = (p.bwin > 0 && p.bmax > 1) ? -1 : 0;
    for (int j = j0; j < p.bnum; ++j) {
      LOC();
      const int f = j < 0 ? bring(e0mod, p.bmax - 1) : bring(e0mod, j);
      for (;;) {
        LOC();
        const int c = ring_read(f, dst);
        if (c == 0) {
          if (j == 0) head_empty = true;
          break;
        }
        const unsigned long long en = warp_ld(p.ctl + C_EPOCH);
        ep_seen = en;
        const int enmod = (int)(en % (unsigned long long)p.bmax);
        const int rel_slot = f >= enmod ? f - enmod : f + p.bmax - enmod;
        int kept = 0;
        for (int o = 0; o < c; o += 32) {
          LOC();
          const bool has = o + lane < c;
          E x = E();
          int rel = 0;
          if (has) {
            x = dst[o + lane];
            rel = bucket_rel(x.d, en);
          }
          __syncwarp();
          const bool rb = has && rel > rel_slot;
          const bool keep = has && !rb;
          const unsigned km = __ballot_sync(FULL, keep);
          if (keep) dst[kept + __popc(km & lanemask_lt())] = x;
          kept += __popc(km);
          if (__any_sync(FULL, rb))
            bucket_scatter_lanes(rb, x, bring(enmod, rel));
          __syncwarp();
        }
        if (kept > 0) return kept;
        if (stopped_warp()) return 0;
      }
    }
    if (head_empty && p.bwin == 0) {  // managed epochs: only the manager advances the floor
      bool ne = false;
      for (int k = lane; k < p.bmax; k += 32)
        if (k != e0mod) ne |= ld_relaxed(wp(k)) > ld_relaxed(rp(k));
      if (__any_sync(FULL, ne)) {
        if (lane == 0 && atomicCAS(p.ctl + C_EPOCH, e0, e0 + 1) == e0) {
          met[M_L2A] += 1;
          red_add(p.ctl + C_GEN, 1ull);
        }
        __syncwarp();
      }
    }
    return 0;
  }

  // ============================================================ L2: batch heaps
  __device__ __forceinline__ E* node_elems(int h, unsigned long long i) const {
    return reinterpret_cast<E*>(p.hnodes) + ((size_t)h * p.hcap + i) * 32;
  }
  __device__ __forceinline__ uint32_t* node_cnt(int h, unsigned long long i) const {
    return p.hcnt + (size_t)h * p.hcap + i;
  }
  __device__ __forceinline__ S node_min(int h, unsigned long long i) const {
    S v = 0;
    if (lane == 0) v = ld_cg_elem(node_elems(h, i)).d;
    return __shfl_sync(FULL, v, 0);
  }
  __device__ void node_swap(int h, unsigned long long a, unsigned long long b) {
    LOC();
    E* A = node_elems(h, a);
    E* B = node_elems(h, b);
    E xa = ld_cg_elem(A + lane), xb = ld_cg_elem(B + lane);
    uint32_t ca = 0, cb = 0;
    if (lane == 0) { ca = __ldcg(node_cnt(h, a)); cb = __ldcg(node_cnt(h, b)); }
    __syncwarp();
    A[lane] = xb;
    B[lane] = xa;
    if (lane == 0) { *node_cnt(h, a) = cb; *node_cnt(h, b) = ca; }
    __threadfence();
    __syncwarp();
  }
  __device__ bool heap_lock(int h) {
    LOC();
    int ok = 1;
    if (lane == 0) {
      uint32_t* lk = p.hlock + (size_t)h * 32;
      wstate(W_HEAP, (unsigned long long)h);
      unsigned long long t0 = 0;
      int spins = 0, ns = 32;
      while (atomicCAS(lk, 0u, 1u) != 0u) {
        LOC();
        if (++spins % 64 == 0) {
          if (stopped()) { ok = 0; break; }
          unsigned long long now = globaltimer_ns();
          if (t0 == 0) t0 = now;
          else if (now - t0 > p.spin_timeout_ns) {
            raise_error(ERR_OVERFLOW, 1000000ull + h, 0, 0, 0);
            ok = 0;
            break;
          }
        }
        __nanosleep(ns);
        if (ns < 512) ns <<= 1;
      }
      wstate(W_NONE, 0);
      __threadfence();
    }
    ok = __shfl_sync(FULL, ok, 0);
    __syncwarp();
    return ok != 0;
  }
  __device__ void heap_unlock(int h) {
    LOC();
    __threadfence();
    __syncwarp();
    if (lane == 0) atomicExch(p.hlock + (size_t)h * 32, 0u);
  }
  __device__ void sift_up(int h, unsigned long long i) {
    LOC();
    while (i > 0) {
      LOC();
      const unsigned long long par = (i - 1) >> 1;
      if (node_min(h, i) < node_min(h, par)) {
        node_swap(h, i, par);
        i = par;
      } else
        break;
    }
  }
  __device__ void sift_down(int h, unsigned long long i, unsigned long long size) {
    LOC();
    for (;;) {
      LOC();
      unsigned long long c = 2 * i + 1;
      if (c >= size) return;
      if (c + 1 < size && node_min(h, c + 1) < node_min(h, c)) ++c;
      if (node_min(h, c) < node_min(h, i)) {
        node_swap(h, i, c);
        i = c;
      } else
        return;
    }
  }
  __device__ __forceinline__ static bool elem_less(S da, uint32_t va, S db, uint32_t vb) {
    return da < db || (da == db && va < vb);
  }
  // bitonic sort of one element per lane (invalid lanes sort last)
  __device__ void warp_sort(E& x, bool has) {
    LOC();
    S d = has ? x.d : (S)Tr::INF;
    uint32_t v = has ? x.v : 0xFFFFFFFFu;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
      LOC();
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        LOC();
        const S pd = __shfl_xor_sync(FULL, d, j);
        const uint32_t pv = __shfl_xor_sync(FULL, v, j);
        const bool up = (lane & k) == 0;
        const bool lower = (lane & j) == 0;
        const bool take_min = (lower == up);
        const bool pless = elem_less(pd, pv, d, v);
        if (pless == take_min) { d = pd; v = pv; }
      }
    }
    x.d = d;
    x.v = v;
  }
  // l2.py:322-344: sorted batch -> nodes of <= node_batch, appended as leaves + sift-up.
  __device__ void heap_write(int h, const E* base, int start, int n, int cap) {
    LOC();
    for (int o = 0; o < n; o += 32) {
      LOC();
      const int c = min(32, n - o);
      const bool has = lane < c;
      E x = E();
      if (has) x = base[(unsigned)(start + o + lane) % (unsigned)cap];
      warp_sort(x, has);
      const int nb = p.nb;
      const int nn = (c + nb - 1) / nb;
      if (!heap_lock(h)) return;
      unsigned long long size = 0;
      if (lane == 0) size = __ldcg(p.hsize + (size_t)h * 16);
      size = __shfl_sync(FULL, size, 0);
      if (size + (unsigned long long)nn > p.hcap) {
        if (lane == 0) raise_error(ERR_HEAP_OVERFLOW, (unsigned long long)h, size, p.hcap, 0);
        heap_unlock(h);
        return;
      }
      for (int q = 0; q < nn; ++q) {
        LOC();
        const unsigned long long i = size + (unsigned long long)q;
        if (has && lane / nb == q) node_elems(h, i)[lane % nb] = x;
        if (lane == 0) *node_cnt(h, i) = (uint32_t)min(nb, c - q * nb);
        // realign so the node's elements start at slot 0 (lanes q*nb .. q*nb+nb-1)
        __threadfence();
        __syncwarp();
        sift_up(h, i);
      }
      if (lane == 0) {
        p.hsize[(size_t)h * 16] = size + (unsigned long long)nn;
        p.hwc[(size_t)h * 16] += (unsigned long long)c;  // reserve units, before unlock
      }
      count(M_L2A, 1);
      heap_unlock(h);
      bump_gen();
    }
  }
  // l2.py:362-389: pop runs off the root while root.min <= min(child mins).
  __device__ int heap_read(int h, E* dst, int want) {
    LOC();
    if (lane == 0 && ld_relaxed(p.hsize + (size_t)h * 16) == 0) want = -1;
    if (__shfl_sync(FULL, want, 0) < 0) return 0;
    if (!heap_lock(h)) return 0;
    unsigned long long size = 0;
    if (lane == 0) size = __ldcg(p.hsize + (size_t)h * 16);
    size = __shfl_sync(FULL, size, 0);
    int n = 0;
    while (size > 0 && n < want) {
      LOC();
      int c0 = 0;
      if (lane == 0) c0 = (int)__ldcg(node_cnt(h, 0));
      c0 = __shfl_sync(FULL, c0, 0);
      E e = ld_cg_elem(node_elems(h, 0) + lane);
      const bool has_child = size > 1;
      S cm = (S)Tr::INF;
      if (has_child) {
        cm = node_min(h, 1);
        if (size > 2) {
          const S c2 = node_min(h, 2);
          if (c2 < cm) cm = c2;
        }
      }
      const bool take = lane < c0 && (!has_child || e.d <= cm);
      const int t = min(__popc(__ballot_sync(FULL, take)), want - n);
      if (lane < t) dst[n + lane] = e;
      n += t;
      const int rem = c0 - t;
      E sh = E();
      sh.v = __shfl_sync(FULL, e.v, (lane + t) & 31);
      sh.d = __shfl_sync(FULL, e.d, (lane + t) & 31);
      __syncwarp();
      if (lane < rem) node_elems(h, 0)[lane] = sh;
      if (lane == 0) *node_cnt(h, 0) = (uint32_t)rem;
      __threadfence();
      __syncwarp();
      const S newmin = __shfl_sync(FULL, sh.d, 0);
      if (rem == 0) {
        --size;
        if (size > 0) {
          E* R = node_elems(h, 0);
          E lx = ld_cg_elem(node_elems(h, size) + lane);
          uint32_t lc = 0;
          if (lane == 0) lc = __ldcg(node_cnt(h, size));
          __syncwarp();
          R[lane] = lx;
          if (lane == 0) *node_cnt(h, 0) = lc;
          __threadfence();
          __syncwarp();
          sift_down(h, 0, size);
        }
      } else if (has_child && newmin > cm) {
        sift_down(h, 0, size);
      } else {
        break;
      }
    }
    if (lane == 0) p.hsize[(size_t)h * 16] = size;
    if (n > 0) count(M_L2A, 1);
    heap_unlock(h);
    local_done += (unsigned long long)n;
    return n;
  }

  // ============================================================ L2 dispatch
  // write_through (compose.py:79-86): the termination reservation is the ring ticket
  // (or heap write counter) itself, claimed before the block is published.
  __device__ void write_back(const E* base, int start, int n, int cap) {
    LOC();
    if (n <= 0) return;
    const unsigned long long t0 = pclk();
    count(M_L2E, (unsigned long long)n);
    pcnt(P_NL2W, 1);
    pcnt(P_L2WELEMS, (unsigned long long)n);
    if (L2K == L2K_FIFO) {
      ring_write(0, base, start, n, cap);
    } else if (L2K == L2K_BUCKET) {
      bucket_write(base, start, n, cap);
    } else {
      heap_write(mcursor, base, start, n, cap);
      if (p.pnum > 1) mcursor = (mcursor + 1) % p.pnum;
    }
    pacc(P_L2W, t0);
  }

  __device__ int l2_read(E* dst) {
    LOC();
    int c;
    if (L2K == L2K_FIFO) {
      c = p.fifo_park ? fifo_read(dst) : ring_read(0, dst);
    } else if (L2K == L2K_BUCKET) {
      c = bucket_read(dst);
    } else {
      c = heap_read(p.pnum > 1 ? gid % p.pnum : 0, dst, L);
    }
    if (c > 0) count(M_L2D, (unsigned long long)c);
    return c;
  }

  // ============================================================ L1 (shared memory)
  __device__ __forceinline__ static int ridx(int h, int i, int cap) { return (int)((unsigned)(h + i) % (unsigned)cap); }
  __device__ __forceinline__ static int ridx_neg(int h, long long i, int cap) {
    int x = h + (int)(i % (long long)cap);
    if (x < 0) x += cap;
    return x >= cap ? x - cap : x;
  }
  static constexpr int LINEAR = 0x7fffffff;

  // pop min(want, size) from the front of a ring
  __device__ int ring_pop_front(E* ring, int& h, int& n, E* dst, int want) {
    LOC();
    const int c = min(want, n);
    const int cap = p.l1cap;
    for (int i = lane; i < c; i += 32) dst[i] = ring[ridx(h, i, cap)];
    h = ridx(h, c, cap);
    n -= c;
    __syncwarp();
    return c;
  }

  // append spill[from..to) (predicate-filtered, stable) to the ring tail; returns count
  __device__ void ring_append(E* ring, int h, int& n, const E* src, int i0, int cnt) {
    LOC();
    const int cap = p.l1cap;
    for (int i = lane; i < cnt; i += 32) ring[ridx(h, n + i, cap)] = src[i0 + i];
    n += cnt;
    __syncwarp();
  }

  // L1 Vector write (l1.py:116-129): append, evict the front over capacity, flush all
  // after every wb write invocations.
  __device__ void l1_vector_write(int ns) {
    LOC();
    const int cap = p.l1cap;
    const int total = n1 + ns;
    const int evict = max(0, total - cap);
    const int er = min(evict, n1), es = evict - er;
    if (er) { write_back(l1a, h1, er, cap); h1 = ridx(h1, er, cap); n1 -= er; }
    if (es) write_back(spill, 0, es, LINEAR);
    ring_append(l1a, h1, n1, spill, es, ns - es);
    count(M_L1E, (unsigned long long)ns);
    count(M_L1D, (unsigned long long)evict);
    if (p.wb > 0 && ++wcount >= p.wb) {
      count(M_L1D, (unsigned long long)n1);
      write_back(l1a, h1, n1, cap);
      h1 = 0;
      n1 = 0;
      wcount = 0;
      count(M_FLUSH, 1);
    }
  }

  // stable in-place compaction of flagged spill elements to spill[0..); returns count
  // (the caller computed `flag(i)` per element; write index never passes read index)
  // L1 Filter write (l1.py:213-230): admit d <= F, reject to L2 tracking reject_min,
  // evict the front over capacity.
  __device__ void l1_filter_write(int ns) {
    LOC();
    const int cap = p.l1cap;
    int A = 0;
    S rmin = rej_min;
    for (int o = 0; o < ns; o += 32) {
      LOC();
      const bool has = o + lane < ns;
      S d = has ? spill[o + lane].d : (S)0;
      const bool adm = has && d <= thr;
      A += __popc(__ballot_sync(FULL, adm));
      S rd = (has && !adm) ? d : (S)Tr::INF;
#pragma unroll
      for (int k = 16; k > 0; k >>= 1) {
        LOC();
        S t = __shfl_xor_sync(FULL, rd, k);
        rd = t < rd ? t : rd;
      }
      if (__any_sync(FULL, has && !adm)) {
        has_rej = true;
        if (rd < rmin) rmin = rd;
      }
    }
    rej_min = rmin;
    const int total = n1 + A;
    const int evict = max(0, total - cap);
    const int er = min(evict, n1), en = evict - er;
    if (er) { write_back(l1a, h1, er, cap); h1 = ridx(h1, er, cap); n1 -= er; }
    // second pass: admitted beyond the first `en` go to the ring; rejects and the
    // first `en` admitted are compacted to the spill front and written back
    int adm_seen = 0, back = 0;
    for (int o = 0; o < ns; o += 32) {
      LOC();
      const bool has = o + lane < ns;
      E x = E();
      if (has) x = spill[o + lane];
      __syncwarp();
      const bool adm = has && x.d <= thr;
      const unsigned am = __ballot_sync(FULL, adm);
      const int arank = adm_seen + __popc(am & lanemask_lt());
      const bool to_ring = adm && arank >= en;
      const bool to_back = has && !to_ring;
      const unsigned rm = __ballot_sync(FULL, to_ring);
      const unsigned bm = __ballot_sync(FULL, to_back);
      if (to_ring) l1a[ridx(h1, n1 + __popc(rm & lanemask_lt()), cap)] = x;
      if (to_back) spill[back + __popc(bm & lanemask_lt())] = x;
      n1 += __popc(rm);
      back += __popc(bm);
      adm_seen += __popc(am);
      __syncwarp();
    }
    write_back(spill, 0, back, LINEAR);
    count(M_L1E, (unsigned long long)A);
    count(M_L1D, (unsigned long long)evict);
  }

  // L1 NearFar write (l1.py:157-177): partition by d < NF; over capacity evict
  // far-front first, then near-front.
  __device__ void l1_nearfar_write(int ns) {
    LOC();
    const int cap = p.l1cap;
    int Nn = 0;
    for (int o = 0; o < ns; o += 32) {
      LOC();
      const bool has = o + lane < ns;
      const bool nr = has && spill[o + lane].d < thr;
      Nn += __popc(__ballot_sync(FULL, nr));
    }
    const int Nf = ns - Nn;
    const int total = n1 + n2 + ns;
    const int over = max(0, total - cap);
    const int ef = min(over, n2 + Nf);
    const int efr = min(ef, n2), efn = ef - efr;
    const int en = over - ef;
    const int enr = min(en, n1), enn = en - enr;
    if (efr) { write_back(l1b, h2, efr, cap); h2 = ridx(h2, efr, cap); n2 -= efr; }
    if (enr) { write_back(l1a, h1, enr, cap); h1 = ridx(h1, enr, cap); n1 -= enr; }
    int ns_seen = 0, fs_seen = 0, back = 0;
    for (int o = 0; o < ns; o += 32) {
      LOC();
      const bool has = o + lane < ns;
      E x = E();
      if (has) x = spill[o + lane];
      __syncwarp();
      const bool nr = has && x.d < thr;
      const bool fr = has && !nr;
      const unsigned nm = __ballot_sync(FULL, nr), fm = __ballot_sync(FULL, fr);
      const int nrk = ns_seen + __popc(nm & lanemask_lt());
      const int frk = fs_seen + __popc(fm & lanemask_lt());
      const bool to_near = nr && nrk >= enn;
      const bool to_far = fr && frk >= efn;
      const bool to_back = has && !to_near && !to_far;
      const unsigned tn = __ballot_sync(FULL, to_near), tf = __ballot_sync(FULL, to_far),
                     tb = __ballot_sync(FULL, to_back);
      if (to_near) l1a[ridx(h1, n1 + __popc(tn & lanemask_lt()), cap)] = x;
      if (to_far) l1b[ridx(h2, n2 + __popc(tf & lanemask_lt()), cap)] = x;
      if (to_back) spill[back + __popc(tb & lanemask_lt())] = x;
      n1 += __popc(tn);
      n2 += __popc(tf);
      back += __popc(tb);
      ns_seen += __popc(nm);
      fs_seen += __popc(fm);
      __syncwarp();
    }
    write_back(spill, 0, back, LINEAR);
    count(M_L1E, (unsigned long long)ns);
    count(M_L1D, (unsigned long long)over);
  }

  // L1 SLF write (l1.py:263-274): head distance snapshot; shorter -> push front
  // (reversing arrival order), else push back; over capacity pop from the tail.
  __device__ void l1_slf_write(int ns) {
    LOC();
    const int cap = p.l1cap;
    S hd = (S)Tr::INF;
    if (n1 > 0) hd = l1a[h1].d;
    int pf = 0;
    for (int o = 0; o < ns; o += 32) {
      LOC();
      const bool has = o + lane < ns;
      pf += __popc(__ballot_sync(FULL, has && spill[o + lane].d < hd));
    }
    const int total = pf + n1 + ns - pf;
    const int over = max(0, total - cap);
    // old content with deque index pf + j >= cap is evicted (ring tail); copy it out
    // before front pushers reuse those slots
    const int keep_old = max(0, min(n1, cap - pf));
    const int eo = n1 - keep_old;
    if (eo) write_back(l1a, ridx(h1, keep_old, cap), eo, cap);
    const int sb = max(0, cap - pf - n1);  // surviving back pushers
    int f_seen = 0, b_seen = 0, back = 0;
    for (int o = 0; o < ns; o += 32) {
      LOC();
      const bool has = o + lane < ns;
      E x = E();
      if (has) x = spill[o + lane];
      __syncwarp();
      const bool fr = has && x.d < hd;
      const bool bk = has && !fr;
      const unsigned fm = __ballot_sync(FULL, fr), bm = __ballot_sync(FULL, bk);
      const int frk = f_seen + __popc(fm & lanemask_lt());
      const int brk = b_seen + __popc(bm & lanemask_lt());
      const bool f_keep = fr && (pf - 1 - frk) < cap;
      const bool b_keep = bk && brk < sb;
      const bool to_back = has && !f_keep && !b_keep;
      const unsigned tb = __ballot_sync(FULL, to_back);
      if (f_keep) l1a[ridx_neg(h1, -1 - (long long)frk, cap)] = x;
      if (b_keep) l1a[ridx(h1, n1 + brk, cap)] = x;
      if (to_back) spill[back + __popc(tb & lanemask_lt())] = x;
      back += __popc(tb);
      f_seen += __popc(fm);
      b_seen += __popc(bm);
      __syncwarp();
    }
    h1 = ridx_neg(h1, -(long long)min(pf, cap), cap);
    n1 = min(total, cap);
    write_back(spill, 0, back, LINEAR);
    count(M_L1E, (unsigned long long)ns);
    count(M_L1D, (unsigned long long)over);
  }

  __device__ void l1_write(int ns) {
    LOC();
    switch (L1T) {
      case L1K_VECTOR: l1_vector_write(ns); break;
      case L1K_NEAR_FAR: l1_nearfar_write(ns); break;
      case L1K_FILTER: l1_filter_write(ns); break;
      default: l1_slf_write(ns); break;
    }
  }

  // L1 reads (l1.py:131-136, 179-189, 232-242, 276-280)
  __device__ int l1_read(E* dst, int want) {
    LOC();
    loc(12);
    const int cap = p.l1cap;
    if (L1T == L1K_NEAR_FAR) {
      if (n1 == 0 && n2 > 0) {
        S mn = (S)Tr::INF;
        for (int i = lane; i < n2; i += 32) {
          LOC();
          const S d = l1b[ridx(h2, i, cap)].d;
          mn = d < mn ? d : mn;
        }
#pragma unroll
        for (int k = 16; k > 0; k >>= 1) {
          LOC();
          S t = __shfl_xor_sync(FULL, mn, k);
          mn = t < mn ? t : mn;
        }
        thr = Tr::add_thr(mn, (S)p.delta_nf_s);
        // stable repartition of far (near is empty: restart it at slot 0)
        h1 = 0;
        int kf = 0;
        for (int o = 0; o < n2; o += 32) {
          LOC();
          const bool has = o + lane < n2;
          E x = E();
          if (has) x = l1b[ridx(h2, o + lane, cap)];
          __syncwarp();
          const bool nr = has && x.d < thr;
          const bool fr = has && !nr;
          const unsigned nm = __ballot_sync(FULL, nr), fm = __ballot_sync(FULL, fr);
          if (nr) l1a[n1 + __popc(nm & lanemask_lt())] = x;
          if (fr) l1b[ridx(h2, kf + __popc(fm & lanemask_lt()), cap)] = x;
          n1 += __popc(nm);
          kf += __popc(fm);
          __syncwarp();
        }
        n2 = kf;
      }
      return ring_pop_front(l1a, h1, n1, dst, want);
    }
    if (L1T == L1K_FILTER && n1 == 0) {
      if (has_rej) {
        thr = Tr::add_thr(rej_min, (S)p.filter_f_s);
        rej_min = (S)Tr::INF;
        has_rej = false;
      }
      return 0;
    }
    return ring_pop_front(l1a, h1, n1, dst, want);
  }

  // ============================================================ cascade write
  // compose.py:56-77: L0.write; a full target lane triggers a full transfer of L0 plus
  // the unplaced remainder into L1; L1's write-back goes through to L2.
  __device__ __forceinline__ void cascade_write(const E* src, int k) {
    LOC();
    loc(14);
    const bool has = lane < k;
    E b = E();
    if (has) b = src[lane];
    const bool isfull = lane < L && l0n >= p.l0cap;
    const unsigned fullmask = __ballot_sync(FULL, isfull);
    const int t = (wc + lane) % L;
    const bool fi = has && ((fullmask >> t) & 1u);
    const unsigned fm = __ballot_sync(FULL, fi);
    const int f = fm ? __ffs(fm) - 1 : k;
    const int si = (lane - wc + L) % L;
    const uint32_t gv = __shfl_sync(FULL, b.v, si & 31);
    const S gd = __shfl_sync(FULL, b.d, si & 31);
    if (lane < L && si < f) l0_push(gv, gd);
    count(M_L0E, (unsigned long long)f);
    if (f == k) {
      wc = (wc + k) % L;
      l0size += k;
      CHKU();
      return;
    }
    const int before = l0size;
    if (k > L || l0size > L * p.l0cap) {
      if (lane == 0) raise_error(ERR_CORRUPT, 30, (unsigned long long)k, (unsigned long long)gid, (unsigned long long)l0size);
      return;
    }
    int ns = l0_drain(spill);
    if (has && lane >= f) spill[ns + lane - f] = b;
    ns += k - f;
    wc = (wc + f) % L;
    l0size = 0;
    count(M_L0D, (unsigned long long)(before + f));
    __syncwarp();
    CHKU();
    l1_write(ns);
    CHKU();
  }

  // B200 extension for the bucket L2 (Delta-stepping order): winners whose bucket lies
  // bwin or more buckets above the current floor bypass the group-private L0/L1 and go
  // straight to their L2 bucket, so the private levels only ever hold near-floor work
  // and thousands of groups cannot run far ahead of the floor (work inflation).
  __device__ void far_flush() {
    if (nfar > 0) write_back(fars, 0, nfar, LINEAR);
    nfar = 0;
  }
  // Light/heavy split: staged heavy tokens (u | kHeavyBit, d) go to the heavy ring (ring 1),
  // which the read cascade consults only after every other level came up empty.
  static constexpr uint32_t kHeavyBit = 0x80000000u;
  __device__ void hvy_flush() {
    if (nhvy > 0) {
      count(M_L2E, (unsigned long long)nhvy);
      ring_write(1, fars + p.far_cap, 0, nhvy, LINEAR);
    }
    nhvy = 0;
  }
  __device__ void far_split() {
    // The floor cannot move while this group holds work (its unflushed done count keeps
    // the near window busy), so far elements are staged across flushes and written as
    // full, bucket-grouped blocks when the stage fills or the group runs out of work.
    const unsigned long long e = ep_seen;
    int kept = 0;
    for (int o = 0; o < outn; o += 32) {
      if (nfar + 32 > p.far_cap) far_flush();
      const bool has = o + lane < outn;
      E x = E();
      int rel = 0;
      if (has) {
        x = outs[o + lane];
        rel = bucket_rel(x.d, e);
      }
      __syncwarp();
      const bool far = has && rel >= p.bwin;
      const bool near = has && !far;
      const unsigned nm = __ballot_sync(FULL, near);
      if (near) outs[kept + __popc(nm & lanemask_lt())] = x;
      kept += __popc(nm);
      const unsigned fm = __ballot_sync(FULL, far);
      if (far) fars[nfar + __popc(fm & lanemask_lt())] = x;
      nfar += __popc(fm);
      __syncwarp();
    }
    outn = kept;
  }

  __device__ __forceinline__ void flush_out(bool all) {
    if (L2K == L2K_BUCKET && p.bwin > 0 && outn > 0) far_split();
    LOC();
    int d = 0;
    while (outn - d >= L) {
      LOC();
      cascade_write(outs + d, L);
      d += L;
    }
    if (all && outn - d > 0) {
      cascade_write(outs + d, outn - d);
      d = outn;
    }
    const int rem = outn - d;
    if (d > 0 && rem > 0) {
      E tmp;
      if (lane < rem) tmp = outs[d + lane];
      __syncwarp();
      if (lane < rem) outs[lane] = tmp;
    }
    outn = rem;
    __syncwarp();
  }

  // ============================================================ relaxation
  // engine.py:201-220 per edge: nd = dist[u] + w; if nd < dist[v] and atomic-min
  // improves (core.py:205-213): emit (v, nd).
  // Split in two so the expansion loops can software-pipeline: the U adjacency loads of
  // step k+1 are issued (adj_issue) before step k's dependent distance checks run
  // (relax_loaded), so a warp keeps 2U independent DRAM loads in flight per lane.
  __device__ __forceinline__ void adj_issue(const bool (&act)[U], const unsigned long long (&kk)[U], uint2 (&a)[U]) const {
#pragma unroll
    for (int j = 0; j < U; ++j) a[j] = act[j] ? ld_adj(p.adj + kk[j]) : make_uint2(0u, 0u);
  }
  __device__ void relax_loaded(bool (&act)[U], const uint2 (&a)[U], const S (&du)[U]) {
    LOC();
    uint32_t v[U];
    S nd[U];
    int c = 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      v[j] = 0;
      nd[j] = 0;
      if (act[j]) {
        v[j] = a[j].x;
        nd[j] = Tr::add(du[j], p.unit ? 1u : a[j].y, dist_ovf);
        ++c;
        if (nd[j] == (S)Tr::INF) act[j] = false;
      }
    }
    if (p.nparts > 1) relax_remote(act, v, nd);  // 1D-partitioned shard
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (act[j]) act[j] = nd[j] < ldcg_dist(dist + v[j]);
    // Fire-and-forget atomic min (RED, no round trip): an edge whose prefilter saw an
    // improvement enqueues (v, nd) whether or not its RED ends up the minimum.  The
    // writer of the final dist[v] always passed its prefilter, so v is expanded with
    // its final distance; a concurrently beaten element is a stale duplicate that the
    // dequeue-side check (engine.py:190-191) drops.
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (act[j]) {
        red_min(dist + v[j], nd[j]);
        // v will be expanded soon: warm L2 with its row offsets so the expansion's head
        // load is an L2 hit (high-diameter graphs pay one such round trip per hop)
        if (p.adj_prefetch > 1) prefetch_l2(p.off + v[j]);
      }
    int upd = 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const unsigned m = __ballot_sync(FULL, act[j]);
      if (act[j]) {
        E e;
        e.v = v[j];
        e.d = nd[j];
        outs[outn + __popc(m & lanemask_lt())] = e;
      }
      outn += __popc(m);
      upd += __popc(m);
    }
    n_relax += (unsigned)c;  // per lane; folded at exit
    n_upd += (unsigned)upd;  // warp total, lane-replicated
    __syncwarp();
    if (outn >= L) flush_out(false);
  }
#if MLMQ_TPF
  __device__ void relax_slots(bool (&act)[U], const unsigned long long (&kk)[U], const S (&du)[U]) {
    uint2 a[U];
    adj_issue(act, kk, a);
    relax_loaded(act, a, du);
  }
#else
  // the fused form (loads, checks, RED and compaction in one pass): the lowest register
  // footprint, used by the default (non-pipelined) expansion
  __device__ void relax_slots(bool (&act)[U], const unsigned long long (&kk)[U], const S (&du)[U]) {
    LOC();
    uint32_t v[U];
    S nd[U];
    int c = 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      v[j] = 0;
      nd[j] = 0;
      if (act[j]) {
        const uint2 a = ld_adj(p.adj + kk[j]);
        v[j] = a.x;
        nd[j] = Tr::add(du[j], p.unit ? 1u : a.y, dist_ovf);
        ++c;
        if (nd[j] == (S)Tr::INF) act[j] = false;
      }
    }
    if (p.nparts > 1) relax_remote(act, v, nd);  // 1D-partitioned shard
#if MLMQ_DIRECT_TOKEN
    // light/heavy split: the light-edge count of each target is loaded beside the
    // prefilter; an improved target without light edges needs no light pass, so it goes
    // straight to the heavy ring as a token (one queue hop and one expansion fewer)
    unsigned nz = 0;  // bit j: target j has no light edges
    if (p.heavy) {
#pragma unroll
      for (int j = 0; j < U; ++j)
        if (act[j] && __ldg(p.nlight + v[j]) == 0u) nz |= 1u << j;
    }
#endif
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (act[j]) act[j] = nd[j] < ldcg_dist(dist + v[j]);
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (act[j]) red_min(dist + v[j], nd[j]);
    int upd = 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
#if MLMQ_DIRECT_TOKEN
      const bool tok = act[j] && ((nz >> j) & 1u);
      const bool nrm = act[j] && !tok;
      const unsigned tm = __ballot_sync(FULL, tok);
      if (tm) {
        if (nhvy + 32 > p.hvy_cap) hvy_flush();
        if (tok) {
          E t;
          t.v = v[j] | kHeavyBit;
          t.d = nd[j];
          (fars + p.far_cap)[nhvy + __popc(tm & lanemask_lt())] = t;
        }
        nhvy += __popc(tm);
        upd += __popc(tm);
      }
#else
      const bool nrm = act[j];
#endif
      const unsigned m = __ballot_sync(FULL, nrm);
      if (nrm) {
        E e;
        e.v = v[j];
        e.d = nd[j];
        outs[outn + __popc(m & lanemask_lt())] = e;
      }
      outn += __popc(m);
      upd += __popc(m);
    }
    n_relax += (unsigned)c;  // per lane; folded at exit
    n_upd += (unsigned)upd;  // warp total, lane-replicated
    __syncwarp();
    if (outn >= L) flush_out(false);
  }
#endif

  // Sharded solve: this group's shard owns global vertices v with
  // v mod P == rank (local id v / P).  Local targets are remapped to local ids and relax
  // as usual; a remote target is pruned against the shard's ghost copy of remote
  // distances (a ghost is never below the true distance, so nd >= ghost[v] is safely
  // dropped), and an improving remote relaxation is appended to the outbox as
  // (global v, nd) -- one fetch-add per warp and step -- for the owner to apply after
  // the superstep's exchange.
  static constexpr unsigned kOboxChunk = 512;
  // Outbox slots this group reserved but did not fill are marked (v = ~0) so the grouping
  // kernels skip them.
  __device__ void obox_close() {
    for (unsigned k = lane; k < ob_left; k += 32) p.obox[ob_next + k] = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    ob_next += ob_left;
    ob_left = 0;
    __syncwarp();
  }
  __device__ void relax_remote(bool (&act)[U], uint32_t (&v)[U], const S (&nd)[U]) {
    const uint32_t pmask = (uint32_t)p.nparts - 1u;
    S* ghost = reinterpret_cast<S*>(p.ghost);
    bool em[U];
    int tot = 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      em[j] = false;
      if (act[j]) {
        if ((v[j] & pmask) == p.rank) {
          v[j] >>= p.part_shift;
        } else {
          act[j] = false;
          em[j] = nd[j] < ldcg_dist(ghost + v[j]);
        }
      }
    }
    // the ghost takes a fire-and-forget min (as dist does): an edge that passed the
    // prefilter is sent even if a racing edge lowers the ghost further; the owner's
    // inbox apply is a min, so such a duplicate is harmless
#pragma unroll
    for (int j = 0; j < U; ++j)
      if (em[j]) red_min(ghost + v[j], nd[j]);
#pragma unroll
    for (int j = 0; j < U; ++j) tot += __popc(__ballot_sync(FULL, em[j]));
    if (tot == 0) return;
    if ((unsigned)tot > ob_left) {
      obox_close();
      unsigned long long base = 0;
      const unsigned want = max((unsigned)tot, kOboxChunk);
      if (lane == 0) base = atomicAdd(p.obox_n, (unsigned long long)want);
      ob_next = __shfl_sync(FULL, base, 0);
      ob_left = want;
      if (ob_next + want > p.obox_cap) {
        if (lane == 0) raise_error(ERR_OBOX, ob_next + want, p.obox_cap, 0, 0);
        ob_left = 0;
        return;
      }
    }
    int off = 0;
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const unsigned m = __ballot_sync(FULL, em[j]);
      if (em[j]) p.obox[ob_next + off + __popc(m & lanemask_lt())] = make_uint2(v[j], (uint32_t)nd[j]);
      off += __popc(m);
    }
    ob_next += (unsigned long long)tot;
    ob_left -= (unsigned)tot;
  }

  // the whole warp strides one edge list (engine.py:212-220 "big" tier, hub chunks)
  __device__ void relax_range(unsigned long long lo, unsigned long long hi, S du) {
    LOC();
    S dus[U];
#pragma unroll
    for (int j = 0; j < U; ++j) dus[j] = du;
    bool act[U];
    unsigned long long kk[U];
    uint2 a[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      kk[j] = lo + (unsigned long long)(j * 32 + lane);
      act[j] = kk[j] < hi;
    }
#if MLMQ_PIPE
    adj_issue(act, kk, a);
    for (unsigned long long k0 = lo; k0 < hi; k0 += 32 * U) {
      LOC();
      bool act2[U];
      uint2 a2[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {  // next step's loads go out before this step's checks
        kk[j] += 32 * U;
        act2[j] = kk[j] < hi;
      }
      adj_issue(act2, kk, a2);
      relax_loaded(act, a, dus);
#pragma unroll
      for (int j = 0; j < U; ++j) {
        act[j] = act2[j];
        a[j] = a2[j];
      }
    }
#else
    (void)a;
    for (unsigned long long k0 = lo; k0 < hi; k0 += 32 * U) {
      LOC();
#pragma unroll
      for (int j = 0; j < U; ++j) {
        kk[j] = k0 + (unsigned long long)(j * 32 + lane);
        act[j] = kk[j] < hi;
      }
      relax_slots(act, kk, dus);
    }
#endif
  }

  // Hub descriptors (new tier): one descriptor per hub list, split into
  // nch chunks of hub_chunk edges that any warp claims with ONE fetch-add on the
  // descriptor's claim word (ticket << 24 | count) -- no CAS retry storms.  The slot is
  // freed only when all nch chunks have completed, so a valid claim always reads a stable
  // descriptor.  Termination: C_HUB_RES += nch before publication; each valid claim adds
  // one to local_done.
  static constexpr unsigned long long kClaimBits = 24, kClaimMask = (1ull << kClaimBits) - 1;
  __device__ void push_hub(uint32_t u, S du, unsigned long long lo, unsigned long long hi) {
    LOC();
    const unsigned long long ch = p.hub_chunk;
    const unsigned long long nch = (hi - lo + ch - 1) / ch;
    if (lane == 0) {
      atomicAdd(p.ctl + C_HUB_RES, nch);  // reserve before publication (compose.py:82-85)
      atomicAdd(p.ctl + C_HUB_ITEMS, nch);
      const unsigned long long t = atomicAdd(p.ctl + C_HUB_WP, 1ull);
      const unsigned long long slot = t & p.hub_mask;
      unsigned long long t0 = 0;
      int spins = 0;
      bool ok = true;
      wstate(W_HUB_WRITE, t);
      while (ld_acquire(p.hub_seq + slot) != t) {
        if (++spins % 64 == 0) {
          if (stopped()) { ok = false; break; }
          const unsigned long long now = globaltimer_ns();
          if (t0 == 0) t0 = now;
          else if (now - t0 > p.spin_timeout_ns) {
            raise_error(ERR_HUB_OVERFLOW, 0, slot, t, p.hub_mask + 1);
            ok = false;
            break;
          }
        }
        __nanosleep(64);
      }
      wstate(W_NONE, 0);
      if (ok) {
        HubItem it;
        it.lo = lo;
        it.hi = hi;
        it.du = (unsigned long long)du;
        it.u = u;
        it.pad = (uint32_t)nch;
        p.hub_data[slot] = it;
        p.hub_fin[slot] = 0u;
        atomicExch(p.hub_next + slot, t << kClaimBits);
        __threadfence();
        st_release(p.hub_seq + slot, t + 1);
        red_add(p.ctl + C_GEN, 1ull);
      }
    }
    __syncwarp();
  }

  // Claim one hub chunk if any; returns true (and relaxes it) when a chunk was claimed.
  __device__ bool hub_try() {
    LOC();
    int got = 0;
    unsigned long long tk = 0, c = 0;
    HubItem it = HubItem();
    // The window of 8 descriptors from the head is inspected by 8 lanes at once (one
    // round trip instead of up to 24 dependent ones when many hub lists are live).
    unsigned long long h = 0, w = 0;
    if (lane == 0) {
      h = ld_relaxed(p.ctl + C_HUB_RP);
      w = ld_relaxed(p.ctl + C_HUB_WP);
    }
    h = __shfl_sync(FULL, h, 0);
    w = __shfl_sync(FULL, w, 0);
    if (h >= w) return false;
    bool cand = false, finished = false;
    if (lane < 8 && h + lane < w) {
      const unsigned long long d = h + lane, slot = d & p.hub_mask;
      const unsigned long long s = ld_acquire(p.hub_seq + slot);
      const unsigned long long x0 = ld_relaxed(p.hub_next + slot);
      const uint32_t nch0 = __ldcg(&p.hub_data[slot].pad);
      if (s > d + 1) {
        finished = true;  // freed
      } else if (s == d + 1) {
        const bool exhausted = (x0 >> kClaimBits) == d && (x0 & kClaimMask) >= nch0;
        finished = exhausted;
        cand = !exhausted;
      }
    }
    const unsigned cm = __ballot_sync(FULL, cand);
    const unsigned fm = __ballot_sync(FULL, finished);
    const int adv = __ffs(~fm) - 1;  // leading run of finished descriptors from the head
    if (lane == 0 && adv > 0) atomicCAS(p.ctl + C_HUB_RP, h, h + (unsigned long long)adv);  // best effort
    if (cm == 0) return false;
    if (lane == 0) {
      unsigned rem = cm;
      while (rem && !got) {
        const int l = __ffs(rem) - 1;
        rem &= rem - 1;
        const unsigned long long d = h + (unsigned long long)l, slot = d & p.hub_mask;
        const unsigned long long x = atomicAdd(p.hub_next + slot, 1ull);
        tk = x >> kClaimBits;
        c = x & kClaimMask;
        // the descriptor our claim belongs to (the slot may have been recycled to tk)
        for (;;) {
          const unsigned long long s1 = ld_acquire(p.hub_seq + slot);
          if (s1 > tk + 1 || s1 < tk) break;  // tk already freed (claim invalid) or stale
          if (s1 == tk + 1) {
            const uint4* src = reinterpret_cast<const uint4*>(p.hub_data + slot);
            const uint4 a = __ldcg(src), b = __ldcg(src + 1);
            if (ld_acquire(p.hub_seq + slot) != tk + 1) continue;  // seqlock re-check
            it.lo = ((unsigned long long)a.y << 32) | a.x;
            it.hi = ((unsigned long long)a.w << 32) | a.z;
            it.du = ((unsigned long long)b.y << 32) | b.x;
            it.u = b.z;
            it.pad = b.w;
            if (c < it.pad) got = 1;
            break;
          }
          if (stopped()) break;
          __nanosleep(32);
        }
      }
    }
    if (!__shfl_sync(FULL, got, 0)) return false;
    tk = __shfl_sync(FULL, tk, 0);
    c = __shfl_sync(FULL, c, 0);
    it.lo = __shfl_sync(FULL, it.lo, 0);
    it.hi = __shfl_sync(FULL, it.hi, 0);
    it.du = __shfl_sync(FULL, it.du, 0);
    it.u = __shfl_sync(FULL, it.u, 0);
    it.pad = __shfl_sync(FULL, it.pad, 0);
    local_done += 1;
    const unsigned long long clo = it.lo + c * p.hub_chunk;
    const unsigned long long chi = min(it.hi, clo + p.hub_chunk);
    S du = (S)it.du;
    S cur = 0;
    if (lane == 0) cur = ldcg_dist(dist + it.u);
    cur = __shfl_sync(FULL, cur, 0);
    if (!(p.dup && du > cur)) {  // stale hub descriptor (engine.py:190 analogue)
      if (cur < du) du = cur;
      relax_range(clo, chi, du);
    }
    // completion: the last finished chunk frees the slot
    __syncwarp();
    if (lane == 0) {
      const unsigned long long slot = tk & p.hub_mask;
      __threadfence();
      if (atomicAdd(p.hub_fin + slot, 1u) + 1u == it.pad) st_release(p.hub_seq + slot, tk + p.hub_mask + 1);
    }
    return true;
  }


  // One step of the flattened expansion: edge slot idx = e0 + j*32 + lane finds its
  // owner row by a 5-step shuffle search over the warp's inclusive degree scan (all U
  // searches unconditional so they interleave), then its adjacency load is issued.
  __device__ __forceinline__ void expand_step(int e0, int total, int incl, unsigned long long base_e, S du,
                                              bool (&act)[U], S (&dus)[U], uint2 (&a)[U]) {
    if (e0 >= total) {  // warp-uniform: past the last step
#pragma unroll
      for (int j = 0; j < U; ++j) {
        act[j] = false;
        dus[j] = 0;
        a[j] = make_uint2(0u, 0u);
      }
      return;
    }
    const unsigned long long tq0 = pclk();
    unsigned long long kk[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int idx = e0 + j * 32 + lane;
      int o = 0;
#pragma unroll
      for (int s = 16; s >= 1; s >>= 1) {
        const int probe = __shfl_sync(FULL, incl, o + s - 1);
        if (probe <= idx) o += s;
      }
      const unsigned long long ob = __shfl_sync(FULL, base_e, o);
      dus[j] = __shfl_sync(FULL, du, o);
      act[j] = idx < total;
      kk[j] = ob + (unsigned long long)idx;
    }
    pacc(P_SPINS, tq0);
    adj_issue(act, kk, a);
  }

  // Owner lookup without the dependent search (MLMQ_SEARCH=1).  The non-empty rows of
  // the sub-batch are compacted once (lane k holds the k-th non-empty row's start cs, edge
  // base cb and distance cd); their starts are strictly increasing, so for a window of 32
  // edge slots one REDUX.OR collects the starts that fall inside it and one REDUX.ADD
  // counts the rows that began before it: owner(slot) = before + popc(starts <= slot) - 1.
  // Two warp-wide steps instead of a 5-deep shuffle chain per slot.
  __device__ __forceinline__ void expand_step_c(int e0, int total, int nne, int cs, unsigned long long cb, S cd,
                                                bool (&act)[U], S (&dus)[U], uint2 (&a)[U]) {
    if (e0 >= total) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        act[j] = false;
        dus[j] = 0;
        a[j] = make_uint2(0u, 0u);
      }
      return;
    }
    const unsigned lmle = lanemask_lt() | (1u << lane);
    unsigned long long kk[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int B = e0 + j * 32;
      const int t = cs - B;
      const bool mine = lane < nne;
      const unsigned W = __reduce_or_sync(FULL, (mine && t >= 0 && t < 32) ? (1u << (t & 31)) : 0u);
      const unsigned before = __reduce_add_sync(FULL, (mine && t < 0) ? 1u : 0u);
      const int own = (int)(before + __popc(W & lmle)) - 1;
      const int idx = B + lane;
      const unsigned long long ob = __shfl_sync(FULL, cb, own & 31);
      dus[j] = __shfl_sync(FULL, cd, own & 31);
      act[j] = idx < total;
      kk[j] = ob + (unsigned long long)idx;
    }
    adj_issue(act, kk, a);
  }

  // MLMQ_ASYNC: owner search for step e0, then its adjacency copied into `buf` (this lane's
  // slots j*32+lane) with cp.async; one commit group per step (empty past the end).
  __device__ __forceinline__ void stage_step(int e0, int total, int incl, unsigned long long base_e, S du,
                                             bool (&act)[U], S (&dus)[U], uint2* buf) {
    if (e0 < total) {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int idx = e0 + j * 32 + lane;
        int o = 0;
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
          const int probe = __shfl_sync(FULL, incl, o + s - 1);
          if (probe <= idx) o += s;
        }
        const unsigned long long ob = __shfl_sync(FULL, base_e, o);
        dus[j] = __shfl_sync(FULL, du, o);
        act[j] = idx < total;
        if (act[j]) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(buf + j * 32 + lane);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(p.adj + ob + (unsigned long long)idx)
                       : "memory");
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < U; ++j) {
        act[j] = false;
        dus[j] = 0;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }

  // engine.py:171-227 for one batch in shared memory
  __device__ void relax_batch(int nb) {
    LOC();
    loc(13);
    if (nb > p.batch_cap) {
      if (lane == 0) raise_error(ERR_CORRUPT, 40, (unsigned long long)nb, (unsigned long long)gid, 0);
      return;
    }
    for (int base = 0; base < nb; base += 32) {
      unsigned long long th0 = pclk();
      LOC();
      const int i = base + lane;
      bool valid = i < nb;
      E e = E();
      S du = (S)Tr::INF;
      unsigned long long lo = 0, hi = 0;
      bool htok = false;  // a deferred heavy-edge token (light/heavy split)
      if (valid) {
        e = batch[i];
        if (p.heavy) {
          htok = (e.v & kHeavyBit) != 0;
          e.v &= ~kHeavyBit;
        }
        if (e.v >= p.n) {  // never expected: report instead of faulting
          raise_error(ERR_CORRUPT, (unsigned long long)last_src, (unsigned long long)e.v,
                      (unsigned long long)gid, (unsigned long long)i | ((unsigned long long)nb << 32));
          valid = false;
        }
      }
      S cur = (S)Tr::INF;
      uint32_t nl = 0;
      if (valid) {  // dist[u] and the row offsets are independent loads: issue together
        cur = ldcg_dist(dist + e.v);
        lo = __ldg(p.off + e.v);
        hi = __ldg(p.off + e.v + 1);
        if (p.heavy) nl = __ldg(p.nlight + e.v);
      }
      if (valid) {
        if (p.dup && e.d > cur) valid = false;  // stale duplicate (engine.py:190-191)
        du = e.d < cur ? e.d : cur;
      }
      if (!valid) lo = hi = 0;
      if (p.heavy) {
        // a vertex relaxes its light edges now and leaves a token for the heavy ones; the
        // token is relaxed later only if no better copy of the vertex appeared meanwhile
        // (Delta-stepping's light/heavy classification, without bucket synchronisation)
        // rows with fewer than heavy_min heavy edges relax everything at once: deferring
        // them would cost a second expansion (head loads, a queue round trip) for little
        const bool emit = valid && !htok && hi - lo - nl >= (unsigned long long)p.heavy_min && hi > lo + nl;
        if (valid) {  // (an invalid lane keeps the empty range lo = hi = 0)
          if (htok) lo += nl;
          else if (emit) hi = lo + nl;
        }
        const unsigned hm = __ballot_sync(FULL, emit);
        if (hm) {
          if (nhvy + 32 > p.hvy_cap) hvy_flush();
          if (emit) {
            E t;
            t.v = e.v | kHeavyBit;
            t.d = du;
            (fars + p.far_cap)[nhvy + __popc(hm & lanemask_lt())] = t;
          }
          nhvy += __popc(hm);
          __syncwarp();
        }
      }
      // warm L2 with the head of each adjacency list while the warp does the scan and
      // the first step's address math (the step's loads then hit L2 instead of DRAM)
      if (valid && p.adj_prefetch) {
        const uint2* a0 = p.adj + lo;
        prefetch_l2(a0);
        if (hi - lo > 16) prefetch_l2(a0 + 16);
        if (hi - lo > 32) prefetch_l2(a0 + 32);
      }
      const unsigned vm = __ballot_sync(FULL, valid);
      pacc(P_HEAD, th0);
      count(M_SETTLED, (unsigned long long)__popc(vm));
      // hub tier: split huge lists into shared edge-range items
      unsigned hm = __ballot_sync(FULL, valid && (hi - lo) > p.hub_thresh);
      while (hm) {
        LOC();
        const int l = __ffs(hm) - 1;
        const uint32_t hu = __shfl_sync(FULL, e.v, l);
        const S hdu = __shfl_sync(FULL, du, l);
        const unsigned long long hlo = __shfl_sync(FULL, lo, l);
        const unsigned long long hhi = __shfl_sync(FULL, hi, l);
        push_hub(hu, hdu, hlo + p.hub_chunk, hhi);
        if (lane == l) hi = lo + p.hub_chunk;
        hm &= hm - 1;
      }
      // Every list up to the hub threshold is flattened across the warp (warp scan +
      // shuffle search), so lists of any length keep all 32 x U edge slots busy.  The
      // reference's th_v split (engine.py:195-220) only orders the same edge set; the
      // relaxed edges and the metrics are identical, and on the GPU one load-balanced
      // pass beats a warp-wide walk per list above th_v.
      const int ds = (int)(hi - lo);
#if MLMQ_SMALLDEG
      // Short lists (every row of the sub-batch has <= U edges, e.g. road grids): each lane
      // relaxes its own row directly -- no degree scan, no owner search.  On high-diameter
      // graphs a group's iteration is a serial chain of warp instructions on the critical
      // path, so a shorter code path per hop is a shorter solve.
      if (__reduce_max_sync(FULL, (unsigned)ds) <= (unsigned)U) {
        bool act[U];
        unsigned long long kk[U];
        S dus[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
          act[j] = j < ds;
          kk[j] = lo + (unsigned long long)j;
          dus[j] = du;
        }
        relax_slots(act, kk, dus);
        continue;
      }
#endif
      const int incl = warp_incl_scan(ds, lane);
      const int total = __shfl_sync(FULL, incl, 31);
      const int excl = incl - ds;
      const unsigned long long base_e = lo - (unsigned long long)excl;  // edge = base[owner] + slot
#if MLMQ_SEARCH
      // compact the non-empty rows once per sub-batch (see expand_step_c)
      const unsigned nem = __ballot_sync(FULL, ds > 0);
      const int nne = __popc(nem);
      const int rk = lane < nne ? (int)__fns(nem, 0, lane + 1) : 0;
      const int cs = __shfl_sync(FULL, excl, rk);
      const unsigned long long cb = __shfl_sync(FULL, base_e, rk);
      const S cd = __shfl_sync(FULL, du, rk);
#define MLMQ_EXPAND(E0, ACT, DUS, A) expand_step_c(E0, total, nne, cs, cb, cd, ACT, DUS, A)
#else
#define MLMQ_EXPAND(E0, ACT, DUS, A) expand_step(E0, total, incl, base_e, du, ACT, DUS, A)
#endif
#if MLMQ_PIPE
      // step e0's owner search + adjacency loads are issued one step ahead
      bool act[U];
      S dus[U];
      uint2 a[U];
      MLMQ_EXPAND(0, act, dus, a);
      for (int e0 = 0; e0 < total; e0 += 32 * U) {
        LOC();
        const unsigned long long ts0 = pclk();
        bool act2[U];
        S dus2[U];
        uint2 a2[U];
        MLMQ_EXPAND(e0 + 32 * U, act2, dus2, a2);
        relax_loaded(act, a, dus);
#pragma unroll
        for (int j = 0; j < U; ++j) {
          act[j] = act2[j];
          dus[j] = dus2[j];
          a[j] = a2[j];
        }
        pacc(P_STEPS, ts0);
      }
#elif MLMQ_ASYNC
      // adjacency of step k+1 is copied to shared memory (cp.async) while step k runs
      {
        uint2* stage = reinterpret_cast<uint2*>((reinterpret_cast<uintptr_t>(bremap_row + 32) + 15) & ~uintptr_t(15));
        bool act[U];
        S dus[U];
        stage_step(0, total, incl, base_e, du, act, dus, stage);
        int k = 0;
        for (int e0 = 0; e0 < total; e0 += 32 * U, ++k) {
          LOC();
          const unsigned long long ts0 = pclk();
          bool act2[U];
          S dus2[U];
          stage_step(e0 + 32 * U, total, incl, base_e, du, act2, dus2, stage + ((k + 1) & 1) * (32 * U));
          asm volatile("cp.async.wait_group 1;" ::: "memory");
          uint2 a[U];
          const uint2* cur = stage + (k & 1) * (32 * U);
#pragma unroll
          for (int j = 0; j < U; ++j) a[j] = act[j] ? cur[j * 32 + lane] : make_uint2(0u, 0u);
          relax_loaded(act, a, dus);
#pragma unroll
          for (int j = 0; j < U; ++j) {
            act[j] = act2[j];
            dus[j] = dus2[j];
          }
          pacc(P_STEPS, ts0);
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
#elif MLMQ_SEARCH
      for (int e0 = 0; e0 < total; e0 += 32 * U) {
        LOC();
        const unsigned long long ts0 = pclk();
        bool act[U];
        S dus[U];
        uint2 a[U];
        MLMQ_EXPAND(e0, act, dus, a);
        relax_loaded(act, a, dus);
        pacc(P_STEPS, ts0);
      }
#else
      // default: the 5-step shuffle search then the step (loads issued inside the step,
      // which keeps the register allocation spill-free at 96 registers)
      for (int e0 = 0; e0 < total; e0 += 32 * U) {
        LOC();
        const unsigned long long tq0 = pclk();
        bool act[U];
        unsigned long long kk[U];
        S dus[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const int idx = e0 + j * 32 + lane;
          int o = 0;
#pragma unroll
          for (int s = 16; s >= 1; s >>= 1) {
            const int probe = __shfl_sync(FULL, incl, o + s - 1);
            if (probe <= idx) o += s;
          }
          const unsigned long long ob = __shfl_sync(FULL, base_e, o);
          dus[j] = __shfl_sync(FULL, du, o);
          act[j] = idx < total;
          kk[j] = ob + (unsigned long long)idx;
        }
        pacc(P_SPINS, tq0);
        const unsigned long long ts0 = pclk();
        relax_slots(act, kk, dus);
        pacc(P_STEPS, ts0);
      }
#endif
#undef MLMQ_EXPAND
    }
    const unsigned long long tf0 = pclk();
    flush_out(true);
    pacc(P_CASFAIL, tf0);
  }

  // ============================================================ eager sharing
  // B200 extension of the cache-like collaboration: thousands of warps
  // starve if a few hoard work in private L0/L1, so while any group is idle a group
  // holding more than two batches of local work writes its L1 (or, with L1 empty, its
  // L0) back to L2 where the idle groups can read it.
  __device__ void maybe_share() {
    LOC();
    if (!p.share) return;
    loc(15);
    const int local = l0size + n1 + n2;
    if (local <= MLMQ_SHARE_MIN) return;
    unsigned long long idle_now = 0;
    if (lane == 0) idle_now = ld_relaxed(p.ctl + C_IDLE);
    if (__shfl_sync(FULL, idle_now, 0) == 0) return;
    const int cap = p.l1cap;
    if (n1 + n2 > 0) {
      count(M_L1D, (unsigned long long)(n1 + n2));
      count(M_FLUSH, 1);
      write_back(l1a, h1, n1, cap);
      if (n2) write_back(l1b, h2, n2, cap);
      h1 = n1 = h2 = n2 = 0;
      wcount = 0;
    } else {
      const int ns = l0_drain(spill);
      count(M_L0D, (unsigned long long)ns);
      l0size = 0;
      write_back(spill, 0, ns, LINEAR);
    }
  }

  // ============================================================ read cascade
  // compose.py:30-54. Returns >0 batch size, -1 when a hub item was processed, 0 on a
  // full miss.
  __device__ int read_cascade() {
    LOC();
    unsigned long long t0 = pclk();
    if (l0size > 0) {
      last_src = 1;
      const int c = l0_read(batch, L);
      count(M_L0D, (unsigned long long)c);
      pacc(P_L0L1, t0);
      return c;
    }
    last_src = 2;
    const int c1 = l1_read(batch, p.l1_want);
    pacc(P_L0L1, t0);
    if (c1 > 0) {
      count(M_L1D, (unsigned long long)c1);
      return c1;
    }
#if MLMQ_HUB_LAST
    // hub chunks after the L2 queue: a chunk claimed later re-reads dist[u] and is
    // skipped when a better copy of u exists, so late hub work is less often wasted
    t0 = pclk();
    last_src = 3;
    const int c2 = l2_read(batch);
    pacc(P_L2R, t0);
    if (c2 > 0) return c2;
    t0 = pclk();
    const bool h = hub_try();
    pacc(P_HUB, t0);
    return h ? -1 : 0;
#else
    t0 = pclk();
    if (hub_try()) {
      pacc(P_HUB, t0);
      return -1;
    }
    pacc(P_HUB, t0);
    t0 = pclk();
    last_src = 3;
    int c2 = l2_read(batch);
    if (L2K == L2K_FIFO && c2 == 0 && p.heavy) {
      last_src = 4;
      c2 = ring_read(1, batch);  // deferred heavy-edge tokens, lowest priority
      if (c2 > 0) count(M_L2D, (unsigned long long)c2);
    }
    pacc(P_L2R, t0);
    return c2;
#endif
  }

  __device__ void run() {
    LOC();
    int backoff = 0;
    const unsigned long long tstart = pclk();
    int since_check = 0;
    unsigned long long seen = ~0ull;
    for (;;) {
      LOC();
      if (idle) {
        // idle: one 16-byte load of (generation, stop); re-walk the cascade only when
        // new work was published since this group's last full miss
        unsigned long long gen = 0, st = 0;
        if (lane == 0) ld_relaxed_v2(p.ctl + C_STOP, st, gen);
        st = __shfl_sync(FULL, st, 0);
        gen = __shfl_sync(FULL, gen, 0);
        if (st) break;
        if (gen == seen) {
          __nanosleep(32u << min(backoff, 5));
          ++backoff;
          continue;
        }
        seen = gen;
      } else if (++since_check >= 16) {  // a busy group polls stop every 16 iterations
        since_check = 0;
        if (stopped_warp()) break;
      }
      CHKU();
      loc(10);
      const int c = read_cascade();
      if (c != 0 && idle) {
        idle = false;
        if (lane == 0) atomicAdd(p.ctl + C_IDLE, ~0ull);  // -1
      }
      if (c > 0) {
        const unsigned long long t0 = pclk();
        pcnt(P_NBATCH, 1);
        pcnt(P_BATCHSUM, (unsigned long long)c);
        CHKU();
        relax_batch(c);
        CHKU();
        pacc(P_RELAX, t0);
        maybe_share();
        CHKU();
        backoff = 0;
        continue;
      }
      if (c < 0) {
        CHKU();
        flush_out(true);
        maybe_share();
        backoff = 0;
        continue;
      }
      if (L2K == L2K_FIFO && nhvy > 0) {  // staged heavy tokens leave before idling
        hvy_flush();
        continue;
      }
      if (L2K == L2K_BUCKET && nfar > 0) {  // staged far work leaves before idling, and the
        far_flush();                        // cascade runs once more: with bnum > 1 some of
        continue;                           // it may be readable by this very group
      }
      if (!idle) {
        idle = true;
        seen = ~0ull;  // the first miss re-checks once against a generation read before it
        if (lane == 0) atomicAdd(p.ctl + C_IDLE, 1ull);
      }
      // full miss: flush local_done (l2.py:56-62)
      if (local_done) {
        if (lane == 0) {
          __threadfence();
          atomicAdd(p.ctl + C_DONE, local_done);
          met[M_L2A] += 1;
        }
        local_done = 0;
        __syncwarp();
      }
      const unsigned long long t0 = pclk();
      __nanosleep(32u << min(backoff, 5));
      ++backoff;
      pacc(P_IDLE, t0);
    }
    pacc(P_TOTAL, tstart);
    if (p.nparts > 1) obox_close();
    loc(99);
    // exit: metric shard + audit evidence
    if (__any_sync(FULL, dist_ovf) && lane == 0) atomicOr(p.ctl + C_DIST_OVF, 1ull);
    const int l1size = n1 + n2;
    {
      const unsigned long long rl = warp_sum_u64((unsigned long long)n_relax);
      if (lane == 0) {
        met[M_RELAX] += rl;
        met[M_UPD] += (unsigned long long)n_upd;
      }
      __syncwarp();
    }
    if (lane == 0) {
      for (int f = 0; f < M_COUNT; ++f) p.metrics[(size_t)gid * M_COUNT + f] = met[f];
      if (kDebug && p.prof)
        for (int f = 0; f < P_COUNT; ++f) p.prof[(size_t)gid * P_COUNT + f] = met[kProfBase + f];
      if (l0size + l1size + outn + nfar + nhvy)
        atomicAdd(p.ctl + C_LOCAL_NONEMPTY, (unsigned long long)(l0size + l1size + outn + nfar + nhvy));
    }
  }
};

// K2: manager warp (engine.py:152-169): reserve == done on three consecutive polls.
static __device__ __noinline__ void manager_loop(const KParams& p, int lane) {
  int k = 0, kq = 0;
  if ((kDebug && p.wstate) && lane == 0) p.wstate[2 * (size_t)p.G + 4] = 1;
  for (int it = 0;; ++it) {
    // the abort word lives in host memory (a PCIe round trip): poll it every 32 iterations
    if (p.host_abort && lane == 0 && (it & 31) == 0 && ld_sys_u32(p.host_abort) != 0u) {
      atomicCAS(p.ctl + C_ERR, 0ull, (unsigned long long)ERR_ABORT);
      __threadfence();
      st_release(p.ctl + C_STOP, 1ull);
    }
    __syncwarp();
    int st = 0;
    unsigned long long d = 0;
    if (lane == 0) {
      st = ld_relaxed(p.ctl + C_STOP) != 0ull;
      d = ld_acquire(p.ctl + C_DONE);
    }
    if (__shfl_sync(FULL, st, 0)) break;
    d = __shfl_sync(FULL, d, 0);
    unsigned long long r = 0;
    for (int i = lane; i < p.nrings; i += 32) r += ld_relaxed(p.ptrs + (size_t)i * 32);
    for (int i = lane; i < p.pnum; i += 32) r += ld_relaxed(p.hwc + (size_t)i * 16);
    if (lane == 0) r += ld_relaxed(p.ctl + C_HUB_RES);
    r = warp_sum_u64(r);
    k = (d == r) ? k + 1 : 0;
    if (p.bwin > 0 && p.bmax > 2 && d != r) {
      // Managed bucket floor (Delta-stepping order, B200 extension): all units not done
      // are unclaimed blocks of rings other than the head and the ring behind it
      // <=> the near window is quiescent (counters monotone, done read first).  Then
      // the floor jumps to the first non-empty far bucket.
      unsigned long long e = 0;
      if (lane == 0) e = ld_relaxed(p.ctl + C_EPOCH);
      e = __shfl_sync(FULL, e, 0);
      const int emod = (int)(e % (unsigned long long)p.bmax);
      unsigned long long far = 0;
      int first = p.bmax;
      for (int i = lane; i < p.nrings; i += 32) {
        const int rel = i >= emod ? i - emod : i + p.bmax - emod;
        if (rel == 0 || rel == p.bmax - 1) continue;
        const unsigned long long w = ld_relaxed(p.ptrs + (size_t)i * 32);
        const unsigned long long rd = ld_relaxed(p.ptrs + (size_t)i * 32 + 16);
        if (w > rd) {
          far += w - rd;
          first = min(first, rel);
        }
      }
      far = warp_sum_u64(far);
      first = __reduce_min_sync(FULL, first);
      kq = (far > 0 && d == r - far) ? kq + 1 : 0;
      // one observation suffices: the counters are monotone and done was read first, and
      // an early advance would only cost work efficiency, never correctness
      if (kq >= 1 && first < p.bmax) {
        if (lane == 0) {
          st_release(p.ctl + C_EPOCH, e + (unsigned long long)first);
          red_add(p.ctl + C_GEN, 1ull);
          if (kDebug && p.wstate) {  // epoch log for the debug dump
            unsigned long long* E = p.wstate + 2 * (size_t)p.G + 8 + (size_t)p.G * 32;
            const unsigned long long i = ++E[0];
            const unsigned long long busy = (unsigned long long)p.G - ld_relaxed(p.ctl + C_IDLE);
            if (i < 8192) E[i] = (globaltimer_ns() << 16) | (busy & 0xFFFF);
          }
        }
        kq = 0;
      }
    } else {
      kq = 0;
      if ((kDebug && p.wstate) && lane == 0 && p.bwin == 0 && (it & 3) == 0) {
        // timeline (debug/profile builds): (time, busy groups, outstanding units) every
        // 4th poll, so the parallelism profile of a FIFO solve can be read back
        unsigned long long* E = p.wstate + 2 * (size_t)p.G + 8 + (size_t)p.G * 32;
        const unsigned long long i = ++E[0];
        const unsigned long long busy = (unsigned long long)p.G - ld_relaxed(p.ctl + C_IDLE);
        const unsigned long long out = r > d ? r - d : 0ull;
        if (i < 8192)
          E[i] = ((globaltimer_ns() >> 6) << 40) | ((busy & 0xFFFF) << 24) | (out > 0xFFFFFFull ? 0xFFFFFFull : out);
      }
    }
    if ((kDebug && p.wstate) && lane == 0) {
      p.wstate[2 * (size_t)p.G] += 1;
      p.wstate[2 * (size_t)p.G + 2] = d;
      p.wstate[2 * (size_t)p.G + 3] = r;
    }
    if (k >= 3) {
      if (lane == 0) st_release(p.ctl + C_STOP, 1ull);
      break;
    }
    __nanosleep(p.bwin > 0 ? 64 : 256);  // a managed floor is latency-critical
  }
}

template <int K, int L2K, int CM, int L1T>
#ifdef MLMQ_MAXNREG  // experiment: an explicit register cap instead of the min-blocks bound
__global__ void __maxnreg__(MLMQ_MAXNREG) mlmq_persistent_kernel(const __grid_constant__ KParams p) {
#else
__global__ void __launch_bounds__(32 * MLMQ_WPB, MLMQ_MINB) mlmq_persistent_kernel(const __grid_constant__ KParams p) {
#endif
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = blockIdx.x * (blockDim.x >> 5) + warp;
  if (gid > p.G) return;
  if (gid == p.G) {
    manager_loop(p, lane);
    if ((kDebug && p.wstate) && lane == 0) p.wstate[2 * (size_t)p.G + 4] = 2;
    return;
  }
  Worker<K, L2K, CM, L1T> w(p, smem + (size_t)warp * p.smem_per_warp, gid, lane);
  w.run();
}

}  // namespace mlmq
