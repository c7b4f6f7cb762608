// CSR-native MatrixMarket reader (host code).
//
// The reference reads a coordinate MatrixMarket file with scipy and densifies
// it (io.py:104-109: mmread -> coo_matrix -> todense), i.e. n x m float64 in
// host memory -- 5.2 GB at 1.3M x 500.  This reader goes straight to the CSR
// the device path uploads (int64 row pointers, int32 columns and counts):
//   * `coordinate` files with `integer`, `real` (integral values) or `pattern`
//     fields, `general` or `symmetric` symmetry (symmetric entries mirrored,
//     as scipy does);
//   * 1-based indices checked against the size line; duplicate coordinates
//     summed (coo -> dense semantics); explicit zeros dropped;
//   * rows sorted by column (the tile index of gmf_create relies on it).
// Two calls: gmf_mm_header (sizes, so the caller can allocate) and
// gmf_mm_read_csr (caller-owned buffers).  Errors: GMF_ERR_CONFIG for a
// malformed file, GMF_ERR_DOMAIN for a negative / non-integral / > 2^31-1
// value, GMF_ERR_UNSUPPORTED for `array` or complex/hermitian files.
#include <algorithm>
#include <chrono>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gmf_common.cuh"

namespace {

struct MMHeader {
  int64_t n = 0, m = 0, entries = 0;
  int pattern = 0, symmetric = 0;
  long data_offset = 0;
  int64_t line = 0;
};

std::string lower(std::string s) {
  for (auto& c : s) c = (char)tolower((unsigned char)c);
  return s;
}

int read_header(FILE* f, const char* path, MMHeader* h) {
  char buf[4096];
  if (!fgets(buf, sizeof buf, f)) { gmf::set_error("%s: empty file", path); return GMF_ERR_CONFIG; }
  h->line = 1;
  char b0[64] = {0}, b1[64] = {0}, b2[64] = {0}, b3[64] = {0}, b4[64] = {0};
  if (sscanf(buf, "%63s %63s %63s %63s %63s", b0, b1, b2, b3, b4) != 5 ||
      lower(b0) != "%%matrixmarket" || lower(b1) != "matrix") {
    gmf::set_error("%s: missing '%%%%MatrixMarket matrix ...' banner", path);
    return GMF_ERR_CONFIG;
  }
  const std::string fmt = lower(b2), field = lower(b3), sym = lower(b4);
  if (fmt != "coordinate") {
    gmf::set_error("%s: only coordinate MatrixMarket files are read as CSR (got %s)", path, b2);
    return GMF_ERR_UNSUPPORTED;
  }
  if (field != "integer" && field != "real" && field != "pattern") {
    gmf::set_error("%s: unsupported field '%s'", path, b3);
    return GMF_ERR_UNSUPPORTED;
  }
  if (sym != "general" && sym != "symmetric") {
    gmf::set_error("%s: unsupported symmetry '%s'", path, b4);
    return GMF_ERR_UNSUPPORTED;
  }
  h->pattern = field == "pattern";
  h->symmetric = sym == "symmetric";
  while (fgets(buf, sizeof buf, f)) {
    ++h->line;
    const char* p = buf;
    while (*p == ' ' || *p == '\t') ++p;
    if (*p == '%' || *p == '\n' || *p == '\r' || *p == 0) continue;
    long long n, m, e;
    if (sscanf(p, "%lld %lld %lld", &n, &m, &e) != 3 || n < 0 || m < 0 || e < 0) {
      gmf::set_error("%s: line %lld: malformed size line", path, (long long)h->line);
      return GMF_ERR_CONFIG;
    }
    h->n = n; h->m = m; h->entries = e;
    h->data_offset = ftell(f);
    return GMF_OK;
  }
  gmf::set_error("%s: no size line", path);
  return GMF_ERR_CONFIG;
}

}  // namespace

extern "C" {

int gmf_mm_header(const char* path, int64_t* n, int64_t* m, int64_t* max_nnz) {
  if (!path || !n || !m || !max_nnz) { gmf::set_error("mm_header: null argument"); return GMF_ERR_CONFIG; }
  FILE* f = fopen(path, "rb");
  if (!f) { gmf::set_error("%s: %s", path, strerror(errno)); return GMF_ERR_CONFIG; }
  MMHeader h;
  const int rc = read_header(f, path, &h);
  fclose(f);
  if (rc) return rc;
  *n = h.n;
  *m = h.m;
  *max_nnz = h.symmetric ? 2 * h.entries : h.entries;
  return GMF_OK;
}

}  // extern "C"

namespace {

struct Chunk {
  std::vector<int32_t> r, c;
  std::vector<int64_t> v;
  int err = 0;           // GMF_ERR_* of the first bad line
  const char* bad = nullptr;
  int64_t parsed = 0;    // coordinate lines seen
};

inline bool is_sp(char ch) { return ch == ' ' || ch == '\t' || ch == '\r'; }

// parse one unsigned decimal integer; false if no digits
inline bool parse_u(const char*& p, const char* e, long long& out) {
  while (p < e && is_sp(*p)) ++p;
  const char* s0 = p;
  long long v = 0;
  while (p < e && *p >= '0' && *p <= '9' && v < (1LL << 60)) v = v * 10 + (*p++ - '0');
  out = v;
  return p > s0;
}

// entries of [b, e) (whole lines); value: integer fast path, strtod otherwise
void parse_chunk(const char* b, const char* e, const MMHeader& h, Chunk* c) {
  const char* p = b;
  const size_t guess = (size_t)(e - b) / 8 + 16;   // ~8+ bytes per coordinate line
  c->r.reserve(guess); c->c.reserve(guess); c->v.reserve(guess);
  while (p < e) {
    const char* line = p;
    const char* nl = (const char*)memchr(p, '\n', (size_t)(e - p));
    const char* le = nl ? nl : e;
    p = nl ? nl + 1 : e;
    const char* q = line;
    while (q < le && is_sp(*q)) ++q;
    if (q == le || *q == '%') continue;
    long long i, j, v = 1;
    if (!parse_u(q, le, i) || !parse_u(q, le, j)) { c->err = GMF_ERR_CONFIG; c->bad = line; return; }
    if (!h.pattern) {
      while (q < le && is_sp(*q)) ++q;
      const char* t = q;
      bool neg = false;
      if (q < le && (*q == '-' || *q == '+')) neg = *q++ == '-';
      long long iv = 0;
      const char* d0 = q;
      while (q < le && *q >= '0' && *q <= '9' && iv < (1LL << 60)) iv = iv * 10 + (*q++ - '0');
      if (q < le && !is_sp(*q)) {       // '.', exponent, ... : full float parse
        char tmp[64];
        const size_t len = std::min((size_t)(le - t), sizeof tmp - 1);
        memcpy(tmp, t, len);
        tmp[len] = 0;
        char* endp;
        const double dv = strtod(tmp, &endp);
        if (endp == tmp) { c->err = GMF_ERR_CONFIG; c->bad = line; return; }
        if (!(dv >= 0.0) || dv != std::floor(dv) || dv > 2147483647.0) {
          c->err = GMF_ERR_DOMAIN; c->bad = line; return;
        }
        v = (long long)dv;
      } else {
        if (q == d0) { c->err = GMF_ERR_CONFIG; c->bad = line; return; }
        if (neg && iv != 0) { c->err = GMF_ERR_DOMAIN; c->bad = line; return; }
        if (iv > 2147483647LL) { c->err = GMF_ERR_DOMAIN; c->bad = line; return; }
        v = iv;
      }
    }
    if (i < 1 || i > h.n || j < 1 || j > h.m) { c->err = GMF_ERR_CONFIG - 100; c->bad = line; return; }
    ++c->parsed;
    c->r.push_back((int32_t)(i - 1)); c->c.push_back((int32_t)(j - 1)); c->v.push_back(v);
    if (h.symmetric && i != j) {
      c->r.push_back((int32_t)(j - 1)); c->c.push_back((int32_t)(i - 1)); c->v.push_back(v);
    }
  }
}

}  // namespace

extern "C" {

int gmf_mm_read_csr(const char* path, int64_t cap, int64_t* indptr, int32_t* indices,
                    int32_t* counts, int64_t* nnz_out) {
  if (!path || !indptr || !nnz_out || (cap > 0 && (!indices || !counts))) {
    gmf::set_error("mm_read_csr: null argument");
    return GMF_ERR_CONFIG;
  }
  FILE* f = fopen(path, "rb");
  if (!f) { gmf::set_error("%s: %s", path, strerror(errno)); return GMF_ERR_CONFIG; }
  MMHeader h;
  int rc = read_header(f, path, &h);
  if (rc) { fclose(f); return rc; }
  if (h.n > INT32_MAX || h.m > INT32_MAX) {
    fclose(f);
    gmf::set_error("%s: dimensions exceed int32 indices", path);
    return GMF_ERR_UNSUPPORTED;
  }
  const int64_t need = h.symmetric ? 2 * h.entries : h.entries;
  if (cap < need) {
    fclose(f);
    gmf::set_error("%s: buffers hold %lld entries, the file needs %lld", path, (long long)cap,
                   (long long)need);
    return GMF_ERR_CONFIG;
  }
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  const bool verbose = getenv("GMF_VERBOSE") != nullptr;
  auto lap = [&](const char* what) {
    if (verbose)
      fprintf(stderr, "[gmf] mm_read_csr %s: %.1f ms\n", what,
              std::chrono::duration<double, std::milli>(clk::now() - t_start).count());
  };
  // the data section in memory, split at line boundaries across threads
  fseek(f, 0, SEEK_END);
  const long fend = ftell(f);
  fseek(f, h.data_offset, SEEK_SET);
  std::string buf((size_t)(fend - h.data_offset), '\0');
  const size_t got_bytes = buf.empty() ? 0 : fread(&buf[0], 1, buf.size(), f);
  fclose(f);
  buf.resize(got_bytes);
  lap("read");
  const char* b = buf.data();
  const char* e = b + buf.size();
  unsigned T = std::thread::hardware_concurrency();
  T = T < 1 ? 1 : (T > 32 ? 32 : T);
  if (buf.size() < ((size_t)1 << 20)) T = 1;
  std::vector<const char*> cut(T + 1, e);
  cut[0] = b;
  for (unsigned t = 1; t < T; ++t) {
    const char* x = b + buf.size() * t / T;
    if (x < cut[t - 1]) x = cut[t - 1];
    const char* nl = (const char*)memchr(x, '\n', (size_t)(e - x));
    cut[t] = nl ? nl + 1 : e;
  }
  std::vector<Chunk> ch(T);
  {
    std::vector<std::thread> th;
    for (unsigned t = 1; t < T; ++t) th.emplace_back(parse_chunk, cut[t], cut[t + 1], std::cref(h), &ch[t]);
    parse_chunk(cut[0], cut[1], h, &ch[0]);
    for (auto& x : th) x.join();
  }
  lap("parse");
  int64_t lines = 0;
  for (unsigned t = 0; t < T; ++t) {
    if (ch[t].err) {
      const int64_t ln = h.line + 1 + std::count(b, ch[t].bad, '\n');
      if (ch[t].err == GMF_ERR_CONFIG - 100) {
        gmf::set_error("%s: line %lld: index out of range", path, (long long)ln);
        return GMF_ERR_CONFIG;
      }
      if (ch[t].err == GMF_ERR_DOMAIN) {
        gmf::set_error("%s: line %lld: value is not a count (nonnegative integer < 2^31)", path,
                       (long long)ln);
        return GMF_ERR_DOMAIN;
      }
      gmf::set_error("%s: line %lld: expected 'row col%s'", path, (long long)ln,
                     h.pattern ? "" : " value");
      return GMF_ERR_CONFIG;
    }
    lines += ch[t].parsed;
  }
  if (lines != h.entries) {
    gmf::set_error("%s: %lld entries declared, %lld found", path, (long long)h.entries,
                   (long long)lines);
    return GMF_ERR_CONFIG;
  }
  // CSR by two stable counting sorts -- by column, then by row -- so every
  // row comes out column-sorted with duplicates adjacent (file order among
  // equal coordinates); duplicates are summed (scipy coo -> dense adds them)
  // and zeros dropped.  O(nnz + n + m), no per-row sorting.
  // Fast path: files written row by row (scipy's mmwrite of a dense or CSR
  // matrix, most count-matrix exports) are already grouped by row; then only
  // rows whose columns are out of order are sorted, locally.
  bool row_sorted = true;
  {
    int32_t prev = 0;
    for (auto& c : ch) {
      for (int32_t r : c.r) {
        if (r < prev) { row_sorted = false; break; }
        prev = r;
      }
      if (!row_sorted) break;
    }
  }
  if (row_sorted && !h.symmetric) {
    std::vector<int32_t> cc;
    std::vector<int64_t> vv, rowp(h.n + 1, 0);
    for (auto& c : ch)
      for (int32_t r : c.r) ++rowp[r + 1];
    for (int64_t r = 0; r < h.n; ++r) rowp[r + 1] += rowp[r];
    cc.reserve(rowp[h.n]);
    vv.reserve(rowp[h.n]);
    for (auto& c : ch) {
      cc.insert(cc.end(), c.c.begin(), c.c.end());
      vv.insert(vv.end(), c.v.begin(), c.v.end());
    }
    lap("scatter");
    std::vector<std::pair<int32_t, int64_t>> row;
    int64_t w = 0;
    indptr[0] = 0;
    for (int64_t r = 0; r < h.n; ++r) {
      const int64_t lo = rowp[r], hi = rowp[r + 1];
      bool sorted = true;
      for (int64_t k = lo + 1; k < hi && sorted; ++k) sorted = cc[k] > cc[k - 1];
      if (!sorted) {
        row.clear();
        for (int64_t k = lo; k < hi; ++k) row.emplace_back(cc[k], vv[k]);
        std::stable_sort(row.begin(), row.end(),
                         [](const std::pair<int32_t, int64_t>& a,
                            const std::pair<int32_t, int64_t>& x) { return a.first < x.first; });
        for (int64_t k = lo; k < hi; ++k) { cc[k] = row[k - lo].first; vv[k] = row[k - lo].second; }
      }
      for (int64_t k = lo; k < hi;) {
        int64_t e2 = k, sum = 0;
        while (e2 < hi && cc[e2] == cc[k]) sum += vv[e2++];
        if (sum > 2147483647LL) {
          gmf::set_error("%s: summed duplicate entry exceeds int32", path);
          return GMF_ERR_DOMAIN;
        }
        if (sum != 0) {
          indices[w] = cc[k];
          counts[w] = (int32_t)sum;
          ++w;
        }
        k = e2;
      }
      indptr[r + 1] = w;
    }
    *nnz_out = w;
    lap("rows (row-sorted input)");
    return GMF_OK;
  }
  std::vector<int64_t> cstart(h.m + 1, 0);
  for (auto& c : ch)
    for (int32_t j : c.c) ++cstart[j + 1];
  for (int64_t j = 0; j < h.m; ++j) cstart[j + 1] += cstart[j];
  const int64_t t_all = cstart[h.m];
  std::vector<int32_t> r1(t_all), c1(t_all);
  std::vector<int64_t> v1(t_all);
  for (auto& c : ch) {
    for (size_t k = 0; k < c.c.size(); ++k) {
      const int64_t at = cstart[c.c[k]]++;
      r1[at] = c.r[k];
      c1[at] = c.c[k];
      v1[at] = c.v[k];
    }
    std::vector<int32_t>().swap(c.r);
    std::vector<int32_t>().swap(c.c);
    std::vector<int64_t>().swap(c.v);
  }
  std::vector<int64_t> start(h.n + 1, 0);
  for (int64_t k = 0; k < t_all; ++k) ++start[r1[k] + 1];
  for (int64_t r = 0; r < h.n; ++r) start[r + 1] += start[r];
  std::vector<int32_t> cc(t_all);
  std::vector<int64_t> vv(t_all);
  {
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t k = 0; k < t_all; ++k) {
      const int64_t at = fill[r1[k]]++;
      cc[at] = c1[k];
      vv[at] = v1[k];
    }
  }
  lap("scatter");
  int64_t w = 0;
  indptr[0] = 0;
  for (int64_t r = 0; r < h.n; ++r) {
    const int64_t lo = start[r], hi = start[r + 1];
    for (int64_t k = lo; k < hi;) {
      int64_t e2 = k, sum = 0;
      while (e2 < hi && cc[e2] == cc[k]) sum += vv[e2++];
      if (sum > 2147483647LL) {
        gmf::set_error("%s: summed duplicate entry exceeds int32", path);
        return GMF_ERR_DOMAIN;
      }
      if (sum != 0) {
        indices[w] = cc[k];
        counts[w] = (int32_t)sum;
        ++w;
      }
      k = e2;
    }
    indptr[r + 1] = w;
  }
  *nnz_out = w;
  lap("rows");
  return GMF_OK;
}

}  // extern "C"
