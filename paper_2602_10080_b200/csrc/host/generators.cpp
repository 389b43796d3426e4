// generators.cpp — fast, reference-bit-compatible graph generators and CSR builder.
//
// Each generator consumes a PyRandom stream in exactly the order of the reference
// generator it mirrors, so the CSR arrays it produces are byte-identical to
// build_csr(generate_*(...)) from pkg/src/mlq_sssp/graph.py:
//   grid2d  graph.py:310-329   (one randint per right edge, then per down edge)
//   path    graph.py:332-342
//   uniform graph.py:345-359   (randrange(n), randrange(n), weight; w=0 self loop -> 1)
//   rmat    graph.py:362-404   (scale x random() quadrant walk, then weight)
// Weight draws are skipped when wmin == wmax (graph.py:306-307).
// The CSR build is a stable counting sort by source that drops zero-weight self
// loops (graph.py:89-124).  SURVEY §8(f) row f1.
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <stdexcept>

#include "../../../include/mlmq.h"
#include "pyrandom.hpp"

namespace mlmq {
void set_last_error(const char* fmt, ...);
}

using mlmq::PyRandom;

namespace {

inline uint32_t draw_weight(PyRandom& rng, int64_t wmin, int64_t wmax) {
  return wmin == wmax ? (uint32_t)wmin : (uint32_t)rng.randint(wmin, wmax);
}

// Edge list of one shard: with nparts > 1 only edges whose source u satisfies
// u % nparts == rank are kept, at local row u / nparts (columns stay global), so the
// CSR built from it is exactly rank's slice of the full CSR (sharded.py shard_csr).
// Zero-weight self loops are dropped here, on global ids (graph.py:89-124).
struct EdgeList {
  std::vector<uint32_t> src, dst, w;
  uint32_t nparts = 1, rank = 0, shift = 0;
  void reserve(size_t m) { src.reserve(m); dst.reserve(m); w.reserve(m); }
  void push(uint32_t u, uint32_t v, uint32_t wt) {
    if ((u & (nparts - 1)) != rank || (u == v && wt == 0)) return;
    src.push_back(u >> shift);
    dst.push_back(v);
    w.push_back(wt);
  }
};

int check_weights(const mlmq_gen_params_t* p) {
  if (p->wmin < 0 || p->wmax < p->wmin || p->wmax > 0xFFFFFFFFLL ||
      (p->wmax - p->wmin) >= 0xFFFFFFFFLL) {
    mlmq::set_last_error("weights must satisfy 0 <= wmin <= wmax < 2^32 for the native generator");
    return MLMQ_EINVAL;
  }
  return MLMQ_OK;
}

int sizes(int kind, const mlmq_gen_params_t* p, uint64_t* n, uint64_t* m) {
  switch (kind) {
    case MLMQ_GEN_GRID2D: {
      if (p->rows < 1 || p->cols < 1) { mlmq::set_last_error("grid dimensions must be >= 1"); return MLMQ_EINVAL; }
      uint64_t r = (uint64_t)p->rows, c = (uint64_t)p->cols;
      *n = r * c;
      *m = 2 * (r * (c - 1) + (r - 1) * c);
      break;
    }
    case MLMQ_GEN_PATH:
      if (p->n < 1) { mlmq::set_last_error("path length must be >= 1"); return MLMQ_EINVAL; }
      *n = (uint64_t)p->n;
      *m = 2 * ((uint64_t)p->n - 1);
      break;
    case MLMQ_GEN_UNIFORM:
      if (p->n < 1 || p->m < 0) { mlmq::set_last_error("need n >= 1 and m >= 0"); return MLMQ_EINVAL; }
      *n = (uint64_t)p->n;
      *m = (uint64_t)p->m;
      break;
    case MLMQ_GEN_RMAT:
      if (p->scale < 1 || p->scale > 31) { mlmq::set_last_error("scale must be in [1, 31]"); return MLMQ_EINVAL; }
      if (p->edge_factor < 1) { mlmq::set_last_error("edge_factor must be >= 1"); return MLMQ_EINVAL; }
      *n = 1ULL << p->scale;
      *m = (uint64_t)p->edge_factor * *n;
      break;
    default:
      mlmq::set_last_error("unknown generator kind %d", kind);
      return MLMQ_EINVAL;
  }
  if (*n > 0xFFFFFFFFULL) { mlmq::set_last_error("vertex count exceeds 2^32-1"); return MLMQ_EINVAL; }
  return MLMQ_OK;
}

// Stable counting sort by source; drops (u == v && w == 0).
uint64_t csr_from_edges(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                        const uint32_t* w, uint64_t* off, uint32_t* col, uint32_t* wout, bool drop = true) {
  std::memset(off, 0, sizeof(uint64_t) * (n + 1));
  for (uint64_t e = 0; e < m; ++e)
    if (!(drop && src[e] == dst[e] && w[e] == 0)) off[src[e] + 1]++;
  for (uint64_t i = 0; i < n; ++i) off[i + 1] += off[i];
  std::vector<uint64_t> cursor(off, off + n);
  for (uint64_t e = 0; e < m; ++e) {
    uint32_t u = src[e];
    if (drop && u == dst[e] && w[e] == 0) continue;
    uint64_t k = cursor[u]++;
    col[k] = dst[e];
    wout[k] = w[e];
  }
  return off[n];
}

}  // namespace

extern "C" int mlmq_gen_size(int kind, const mlmq_gen_params_t* p, uint64_t* n_out, uint64_t* m_out) {
  if (!p || !n_out || !m_out) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  return sizes(kind, p, n_out, m_out);
}

static int gen_impl(int kind, const mlmq_gen_params_t* p, const uint32_t* key, uint64_t keylen, uint32_t nparts,
                    uint32_t rank, uint64_t* off, std::vector<uint32_t>* colv, std::vector<uint32_t>* wv,
                    uint32_t* col, uint32_t* wout, uint64_t* m_out);

extern "C" int mlmq_gen_graph(int kind, const mlmq_gen_params_t* p, const uint32_t* key,
                              uint64_t keylen, uint64_t* off, uint32_t* col, uint32_t* wout) {
  uint64_t kept = 0;
  return gen_impl(kind, p, key, keylen, 1, 0, off, nullptr, nullptr, col, wout, &kept);
}

// One shard of a generated graph (rows u with u % nparts == rank at local id u / nparts,
// global columns): the same RNG stream, only the shard's edges are stored.  Two calls:
// the first (col == NULL) fills off[n_local + 1] and *m_out; the second fills col / w.
extern "C" int mlmq_gen_shard(int kind, const mlmq_gen_params_t* p, const uint32_t* key, uint64_t keylen,
                              uint32_t nparts, uint32_t rank, uint64_t* off, uint32_t* col, uint32_t* wout,
                              uint64_t* m_out) {
  if (nparts < 1 || (nparts & (nparts - 1)) || rank >= nparts) {
    mlmq::set_last_error("nparts must be a power of two and rank < nparts");
    return MLMQ_EINVAL;
  }
  if (!m_out) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  // generate once, keep the shard's arrays between the sizing and the filling call
  static thread_local std::vector<uint32_t> s_col, s_w;
  static thread_local std::vector<uint64_t> s_off;
  if (!col) {
    uint64_t n = 0, m = 0;
    int st = sizes(kind, p, &n, &m);
    if (st) return st;
    s_off.assign((n - rank + nparts - 1) / nparts + 1, 0);
    st = gen_impl(kind, p, key, keylen, nparts, rank, s_off.data(), &s_col, &s_w, nullptr, nullptr, m_out);
    if (st) return st;
    if (off) std::memcpy(off, s_off.data(), s_off.size() * sizeof(uint64_t));
    return MLMQ_OK;
  }
  if (*m_out != s_col.size()) { mlmq::set_last_error("mlmq_gen_shard: call it first with col == NULL"); return MLMQ_EINVAL; }
  std::memcpy(col, s_col.data(), s_col.size() * 4);
  if (wout) std::memcpy(wout, s_w.data(), s_w.size() * 4);
  if (off) std::memcpy(off, s_off.data(), s_off.size() * sizeof(uint64_t));
  std::vector<uint32_t>().swap(s_col);
  std::vector<uint32_t>().swap(s_w);
  std::vector<uint64_t>().swap(s_off);
  return MLMQ_OK;
}

static int gen_impl(int kind, const mlmq_gen_params_t* p, const uint32_t* key, uint64_t keylen, uint32_t nparts,
                    uint32_t rank, uint64_t* off, std::vector<uint32_t>* colv, std::vector<uint32_t>* wv,
                    uint32_t* col, uint32_t* wout, uint64_t* m_out) {
  if (!p || !key || keylen == 0 || !off) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  uint64_t n = 0, m = 0;
  int st = sizes(kind, p, &n, &m);
  if (st) return st;
  if ((st = check_weights(p))) return st;
  try {
    PyRandom rng(key, (size_t)keylen);
    const int64_t wmin = p->wmin, wmax = p->wmax;
    EdgeList E;
    E.nparts = nparts;
    E.rank = rank;
    while ((1u << E.shift) < nparts) ++E.shift;
    E.reserve(nparts > 1 ? m / nparts + m / (4 * nparts) + 1024 : m);
    switch (kind) {
      case MLMQ_GEN_GRID2D: {
        const uint64_t rows = p->rows, cols = p->cols;
        for (uint64_t r = 0; r < rows; ++r)
          for (uint64_t c = 0; c < cols; ++c) {
            uint32_t u = (uint32_t)(r * cols + c);
            if (c + 1 < cols) {
              uint32_t wt = draw_weight(rng, wmin, wmax);
              E.push(u, u + 1, wt);
              E.push(u + 1, u, wt);
            }
            if (r + 1 < rows) {
              uint32_t wt = draw_weight(rng, wmin, wmax);
              E.push(u, (uint32_t)(u + cols), wt);
              E.push((uint32_t)(u + cols), u, wt);
            }
          }
        break;
      }
      case MLMQ_GEN_PATH:
        for (uint64_t u = 0; u + 1 < n; ++u) {
          uint32_t wt = draw_weight(rng, wmin, wmax);
          E.push((uint32_t)u, (uint32_t)(u + 1), wt);
          E.push((uint32_t)(u + 1), (uint32_t)u, wt);
        }
        break;
      case MLMQ_GEN_UNIFORM:
        for (uint64_t e = 0; e < m; ++e) {
          uint32_t u = (uint32_t)rng.randbelow(n);
          uint32_t v = (uint32_t)rng.randbelow(n);
          uint32_t wt = draw_weight(rng, wmin, wmax);
          if (u == v && wt == 0) wt = 1;
          E.push(u, v, wt);
        }
        break;
      case MLMQ_GEN_RMAT: {
        // graph.py:384-399 compares random() against a, a+b, a+b+c (double sums); the
        // comparisons run on random()'s exact 53-bit numerator against ceil(t * 2^53)
        const uint64_t a = PyRandom::ceil53(p->a), ab = PyRandom::ceil53(p->a + p->b),
                       abc = PyRandom::ceil53(p->a + p->b + p->c);
        const int scale = (int)p->scale;
        for (uint64_t e = 0; e < m; ++e) {
          uint32_t u = 0, v = 0;
          for (int lv = 0; lv < scale; ++lv) {
            // quadrant a: (0,0)  b: (0,1)  c: (1,0)  d: (1,1) — branchless
            const uint64_t r = rng.random53();
            const uint32_t ub = r >= ab;
            const uint32_t vb = (uint32_t)(r >= a) ^ (uint32_t)(r >= ab) ^ (uint32_t)(r >= abc);
            u = (u << 1) | ub;
            v = (v << 1) | vb;
          }
          uint32_t wt = draw_weight(rng, wmin, wmax);
          if (u == v && wt == 0) wt = 1;
          E.push(u, v, wt);
        }
        break;
      }
    }
    const uint64_t n_rows = nparts > 1 ? (n - rank + nparts - 1) / nparts : n;
    const uint64_t mk = E.src.size();
    if (colv) {  // shard: caller-owned vectors
      colv->resize(mk);
      wv->resize(mk);
      col = colv->data();
      wout = wv->data();
    }
    uint64_t kept = csr_from_edges(n_rows, mk, E.src.data(), E.dst.data(), E.w.data(), off, col, wout, false);
    if (nparts == 1 && kept != m) { mlmq::set_last_error("internal: kept %llu of %llu edges", (unsigned long long)kept, (unsigned long long)m); return MLMQ_EINVAL; }
    *m_out = kept;
  } catch (const std::bad_alloc&) {
    mlmq::set_last_error("host allocation failed while generating %llu edges", (unsigned long long)m);
    return MLMQ_ENOMEM;
  }
  return MLMQ_OK;
}

extern "C" int mlmq_build_csr(uint64_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                              const uint32_t* w, uint64_t* off, uint32_t* col, uint32_t* wout,
                              uint64_t* m_out) {
  if (!off || (m && (!src || !dst || !w || !col || !wout))) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  for (uint64_t e = 0; e < m; ++e)
    if (src[e] >= n || dst[e] >= n) {
      mlmq::set_last_error("edge %u->%u references a vertex outside [0, %llu)", src[e], dst[e], (unsigned long long)n);
      return MLMQ_EINVAL;
    }
  try {
    uint64_t kept = csr_from_edges(n, m, src, dst, w, off, col, wout);
    if (m_out) *m_out = kept;
  } catch (const std::bad_alloc&) {
    mlmq::set_last_error("host allocation failed");
    return MLMQ_ENOMEM;
  }
  return MLMQ_OK;
}

// splitmix64 finaliser: a counter-based stream, so weight e is independent of order.
static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

extern "C" int mlmq_gen_f32_weights(uint64_t m, uint64_t seed, float* w_out) {
  if (m && !w_out) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  const uint64_t s = splitmix64(seed ^ 0x6A09E667F3BCC909ULL);
  for (uint64_t e = 0; e < m; ++e) {
    uint64_t r = splitmix64(s + e);
    w_out[e] = (float)(r >> 40) * (1.0f / 16777216.0f);  // 24 random bits -> [0, 1)
  }
  return MLMQ_OK;
}
