// loaders.cpp — native DIMACS .gr and Matrix Market coordinate readers.
//
// Restates the reference readers (pkg/src/mlq_sssp/graph.py:132-175 load_dimacs,
// graph.py:185-257 load_matrix_market) with the same acceptance rules, the same error
// classes and messages, and the same edge order, then builds the CSR with the stable
// counting sort of build_csr (graph.py:89-124).  The whole file is read at once and
// tokenised in place, so a road network of ~60 M arcs loads in seconds instead of the
// minutes the Python line loop takes.
//
// Status codes: MLMQ_EFORMAT (GraphFormatError), MLMQ_ENEGATIVE (NegativeWeightError),
// MLMQ_EIO (the file cannot be opened: OSError / FileNotFoundError), MLMQ_EFALLBACK (a
// token this reader does not restate exactly -- e.g. Python's "1_000" integer syntax or a
// weight >= 2^32 -- the caller falls back to the Python reader, which accepts it).
#include <cerrno>
#include <cfenv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../../include/mlmq.h"

namespace mlmq {
void set_last_error(const char* fmt, ...);
}

namespace {

uint64_t csr_build(uint64_t n, const std::vector<uint32_t>& src, const std::vector<uint32_t>& dst,
                   const std::vector<uint32_t>& w, std::vector<uint64_t>& off, std::vector<uint32_t>& col,
                   std::vector<uint32_t>& wo) {
  // stable counting sort by source; zero-weight self loops dropped (graph.py:89-124)
  const uint64_t m = src.size();
  off.assign(n + 1, 0);
  for (uint64_t e = 0; e < m; ++e)
    if (!(src[e] == dst[e] && w[e] == 0)) off[src[e] + 1]++;
  for (uint64_t i = 0; i < n; ++i) off[i + 1] += off[i];
  col.resize(off[n]);
  wo.resize(off[n]);
  std::vector<uint64_t> cur(off.begin(), off.end() - 1);
  for (uint64_t e = 0; e < m; ++e) {
    const uint32_t u = src[e];
    if (u == dst[e] && w[e] == 0) continue;
    const uint64_t k = cur[u]++;
    col[k] = dst[e];
    wo[k] = w[e];
  }
  return off[n];
}

// A line split into whitespace-separated tokens (pointers into the file buffer).
struct Line {
  std::vector<std::pair<const char*, size_t>> tok;
  std::string text() const {  // the stripped line, for messages
    if (tok.empty()) return "";
    const char* a = tok.front().first;
    const char* b = tok.back().first + tok.back().second;
    return std::string(a, b);
  }
  bool is(size_t i, const char* s) const {
    return i < tok.size() && tok[i].second == std::strlen(s) && std::memcmp(tok[i].first, s, tok[i].second) == 0;
  }
};

inline bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f'; }

// Python int(): optional sign, decimal digits.  0 ok, 1 not an integer, 2 an integer
// form this reader does not restate (underscores) -> fall back.
int parse_int(const std::pair<const char*, size_t>& t, long long* out) {
  const char* p = t.first;
  const char* e = t.first + t.second;
  bool neg = false;
  if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
  if (p == e) return 1;
  unsigned long long v = 0;
  for (const char* q = p; q < e; ++q) {
    if (*q == '_') return 2;
    if (*q < '0' || *q > '9') return 1;
    if (v > (0x7FFFFFFFFFFFFFFFull - 9) / 10) return 2;  // beyond int64: Python's bigint path
    v = v * 10 + (unsigned long long)(*q - '0');
  }
  *out = neg ? -(long long)v : (long long)v;
  return 0;
}

struct Reader {
  std::vector<char> buf;
  size_t pos = 0;
  long long lineno = 0;
  bool next(Line& L) {  // false at EOF
    if (pos >= buf.size()) return false;
    ++lineno;
    L.tok.clear();
    size_t i = pos;
    while (i < buf.size() && buf[i] != '\n') {
      while (i < buf.size() && buf[i] != '\n' && is_space(buf[i])) ++i;
      const size_t s = i;
      while (i < buf.size() && buf[i] != '\n' && !is_space(buf[i])) ++i;
      if (i > s) L.tok.emplace_back(&buf[s], i - s);
    }
    pos = i + 1;
    return true;
  }
};

int read_file(const char* path, std::vector<char>& buf) {
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    mlmq::set_last_error("[Errno %d] %s: '%s'", errno, std::strerror(errno), path);
    return MLMQ_EIO;
  }
  std::fseek(f, 0, SEEK_END);
  const long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  if (sz > 0 && std::fread(buf.data(), 1, (size_t)sz, f) != (size_t)sz) {
    std::fclose(f);
    mlmq::set_last_error("%s: read failed", path);
    return MLMQ_EIO;
  }
  std::fclose(f);
  return MLMQ_OK;
}

}  // namespace

struct mlmq_csr {
  uint64_t n = 0;
  std::vector<uint64_t> off;
  std::vector<uint32_t> col, w;
};

extern "C" {

int mlmq_load_dimacs(const char* path, mlmq_csr** out) {
  if (!path || !out) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  *out = nullptr;
  Reader R;
  int st = read_file(path, R.buf);
  if (st) return st;
  long long n = -1, declared = -1;
  std::vector<uint32_t> src, dst, w;
  Line L;
  while (R.next(L)) {
    if (L.tok.empty() || L.tok[0].first[0] == 'c') continue;  // graph.py:141 (startswith "c")
    const long long ln = R.lineno;
    if (L.is(0, "p")) {
      if (L.tok.size() != 4 || !L.is(1, "sp")) {
        mlmq::set_last_error("%s:%lld: malformed problem line '%s'", path, ln, L.text().c_str());
        return MLMQ_EFORMAT;
      }
      if (n >= 0) { mlmq::set_last_error("%s:%lld: duplicate problem line", path, ln); return MLMQ_EFORMAT; }
      long long a = 0, b = 0;
      const int ra = parse_int(L.tok[2], &a), rb = parse_int(L.tok[3], &b);
      if (ra || rb) return MLMQ_EFALLBACK;  // Python would raise ValueError / accept bigints
      if (a < 0 || a > 0xFFFFFFFFll) return MLMQ_EFALLBACK;
      n = a;
      declared = b;
      src.reserve((size_t)std::max(0LL, std::min(b, 1LL << 33)));
      dst.reserve(src.capacity());
      w.reserve(src.capacity());
    } else if (L.is(0, "a")) {
      if (n < 0) { mlmq::set_last_error("%s:%lld: arc before problem line", path, ln); return MLMQ_EFORMAT; }
      if (L.tok.size() != 4) {
        mlmq::set_last_error("%s:%lld: malformed arc line '%s'", path, ln, L.text().c_str());
        return MLMQ_EFORMAT;
      }
      long long u = 0, v = 0, wt = 0;
      const int r1 = parse_int(L.tok[1], &u), r2 = parse_int(L.tok[2], &v), r3 = parse_int(L.tok[3], &wt);
      if (r1 == 2 || r2 == 2 || r3 == 2) return MLMQ_EFALLBACK;
      if (r1 || r2 || r3) { mlmq::set_last_error("%s:%lld: non-integer arc field", path, ln); return MLMQ_EFORMAT; }
      if (wt < 0) { mlmq::set_last_error("%s:%lld: negative weight %lld", path, ln, wt); return MLMQ_ENEGATIVE; }
      if (!(1 <= u && u <= n) || !(1 <= v && v <= n)) {
        mlmq::set_last_error("%s:%lld: vertex id out of range", path, ln);
        return MLMQ_EFORMAT;
      }
      if (wt > 0xFFFFFFFFll) return MLMQ_EFALLBACK;
      src.push_back((uint32_t)(u - 1));
      dst.push_back((uint32_t)(v - 1));
      w.push_back((uint32_t)wt);
    } else {
      mlmq::set_last_error("%s:%lld: unknown line type '%.*s'", path, ln, (int)L.tok[0].second, L.tok[0].first);
      return MLMQ_EFORMAT;
    }
  }
  if (n < 0) { mlmq::set_last_error("%s: missing problem line", path); return MLMQ_EFORMAT; }
  if (declared != (long long)src.size()) {
    mlmq::set_last_error("%s: header declares %lld arcs but file has %zu", path, declared, src.size());
    return MLMQ_EFORMAT;
  }
  mlmq_csr* c = new mlmq_csr();
  c->n = (uint64_t)n;
  csr_build(c->n, src, dst, w, c->off, c->col, c->w);
  *out = c;
  return MLMQ_OK;
}

int mlmq_load_matrix_market(const char* path, int64_t weight_scale, mlmq_csr** out) {
  if (!path || !out) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  *out = nullptr;
  Reader R;
  int st = read_file(path, R.buf);
  if (st) return st;
  Line L;
  // header: the first physical line, as read (graph.py:191-202)
  size_t eol = 0;
  while (eol < R.buf.size() && R.buf[eol] != '\n') ++eol;
  const std::string head(R.buf.data(), eol);
  if (head.compare(0, 14, "%%MatrixMarket") != 0) {
    mlmq::set_last_error("%s: missing MatrixMarket header", path);
    return MLMQ_EFORMAT;
  }
  R.next(L);
  if (L.tok.size() < 5 || !L.is(1, "matrix") || !L.is(2, "coordinate")) {
    mlmq::set_last_error("%s: unsupported header '%s'", path, L.text().c_str());
    return MLMQ_EFORMAT;
  }
  const std::string vt(L.tok[3].first, L.tok[3].second), sym(L.tok[4].first, L.tok[4].second);
  if (vt != "real" && vt != "integer" && vt != "pattern") {
    mlmq::set_last_error("%s: unsupported value type '%s'", path, vt.c_str());
    return MLMQ_EFORMAT;
  }
  if (sym != "general" && sym != "symmetric") {
    mlmq::set_last_error("%s: unsupported symmetry '%s'", path, sym.c_str());
    return MLMQ_EFORMAT;
  }
  bool have_size = false;
  while (R.next(L)) {
    if (L.tok.empty() || L.tok[0].first[0] == '%') continue;
    have_size = true;
    break;
  }
  if (!have_size) { mlmq::set_last_error("%s: missing size line", path); return MLMQ_EFORMAT; }
  if (L.tok.size() != 3) {
    mlmq::set_last_error("%s: malformed size line '%s'", path, L.text().c_str());
    return MLMQ_EFORMAT;
  }
  long long rows = 0, cols = 0, nnz = 0;
  if (parse_int(L.tok[0], &rows) || parse_int(L.tok[1], &cols) || parse_int(L.tok[2], &nnz)) return MLMQ_EFALLBACK;
  if (rows != cols) {
    mlmq::set_last_error("%s: matrix is %lldx%lld, expected square", path, rows, cols);
    return MLMQ_EFORMAT;
  }
  if (rows < 0 || rows > 0xFFFFFFFFll) return MLMQ_EFALLBACK;
  const bool pattern = vt == "pattern", integer = vt == "integer", symmetric = sym == "symmetric";
  std::vector<uint32_t> src, dst, w;
  const size_t cap = (size_t)std::max(0LL, std::min(nnz, 1LL << 33)) * (symmetric ? 2 : 1);
  src.reserve(cap);
  dst.reserve(cap);
  w.reserve(cap);
  long long seen = 0;
  const int old_round = std::fegetround();
  std::fesetround(FE_TONEAREST);  // Python round(): nearest, ties to even
  auto done = [&](int code) {
    std::fesetround(old_round);
    return code;
  };
  while (R.next(L)) {
    if (L.tok.empty() || L.tok[0].first[0] == '%') continue;
    long long i = 0, j = 0;
    const int ri = L.tok.size() > 0 ? parse_int(L.tok[0], &i) : 1;
    const int rj = L.tok.size() > 1 ? parse_int(L.tok[1], &j) : 1;
    if (ri == 2 || rj == 2) return done(MLMQ_EFALLBACK);
    if (ri || rj) { mlmq::set_last_error("%s: malformed entry '%s'", path, L.text().c_str()); return done(MLMQ_EFORMAT); }
    long long wt = 1;
    if (pattern) {
      if (L.tok.size() != 2) {
        mlmq::set_last_error("%s: pattern entry with a value: '%s'", path, L.text().c_str());
        return done(MLMQ_EFORMAT);
      }
    } else {
      if (L.tok.size() != 3) {
        mlmq::set_last_error("%s: entry missing value: '%s'", path, L.text().c_str());
        return done(MLMQ_EFORMAT);
      }
      if (integer) {
        if (parse_int(L.tok[2], &wt)) return done(MLMQ_EFALLBACK);  // Python: ValueError / bigint
      } else {
        const std::string t(L.tok[2].first, L.tok[2].second);
        char* endp = nullptr;
        const double x = std::strtod(t.c_str(), &endp);
        if (!endp || *endp || !std::isfinite(x)) return done(MLMQ_EFALLBACK);
        if (x < 0) {
          mlmq::set_last_error("%s: negative weight %s", path, t.c_str());
          return done(MLMQ_ENEGATIVE);
        }
        const double r = std::nearbyint(x * (double)weight_scale);
        if (!(r < 4294967296.0)) return done(MLMQ_EFALLBACK);
        wt = (long long)r;
      }
    }
    if (wt < 0) { mlmq::set_last_error("%s: negative weight %lld", path, wt); return done(MLMQ_ENEGATIVE); }
    if (!(1 <= i && i <= rows) || !(1 <= j && j <= cols)) {
      mlmq::set_last_error("%s: entry (%lld,%lld) out of range", path, i, j);
      return done(MLMQ_EFORMAT);
    }
    if (wt > 0xFFFFFFFFll) return done(MLMQ_EFALLBACK);
    ++seen;
    src.push_back((uint32_t)(i - 1));
    dst.push_back((uint32_t)(j - 1));
    w.push_back((uint32_t)wt);
    if (symmetric && i != j) {
      src.push_back((uint32_t)(j - 1));
      dst.push_back((uint32_t)(i - 1));
      w.push_back((uint32_t)wt);
    }
  }
  std::fesetround(old_round);
  if (seen != nnz) {
    mlmq::set_last_error("%s: size line declares %lld entries, found %lld", path, nnz, seen);
    return MLMQ_EFORMAT;
  }
  mlmq_csr* c = new mlmq_csr();
  c->n = (uint64_t)rows;
  csr_build(c->n, src, dst, w, c->off, c->col, c->w);
  *out = c;
  return MLMQ_OK;
}

int mlmq_csr_size(const mlmq_csr* c, uint64_t* n, uint64_t* m) {
  if (!c || !n || !m) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  *n = c->n;
  *m = c->col.size();
  return MLMQ_OK;
}

int mlmq_csr_copy(const mlmq_csr* c, uint64_t* row_offsets, uint32_t* col, uint32_t* w) {
  if (!c || !row_offsets || (!c->col.empty() && (!col || !w))) { mlmq::set_last_error("null argument"); return MLMQ_EINVAL; }
  std::memcpy(row_offsets, c->off.data(), c->off.size() * 8);
  if (!c->col.empty()) {
    std::memcpy(col, c->col.data(), c->col.size() * 4);
    std::memcpy(w, c->w.data(), c->w.size() * 4);
  }
  return MLMQ_OK;
}

void mlmq_csr_free(mlmq_csr* c) { delete c; }

}  // extern "C"
