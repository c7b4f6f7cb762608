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
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
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
    gmf::set_error("%s: dimensions exceed int32 column indices", path);
    return GMF_ERR_UNSUPPORTED;
  }
  const int64_t need = h.symmetric ? 2 * h.entries : h.entries;
  if (cap < need) {
    fclose(f);
    gmf::set_error("%s: buffers hold %lld entries, the file needs %lld", path, (long long)cap,
                   (long long)need);
    return GMF_ERR_CONFIG;
  }
  // pass 1: coordinates into (row, col, value) triplets
  std::vector<int32_t> ri, ci;
  std::vector<double> vv;
  ri.reserve(need); ci.reserve(need); vv.reserve(need);
  char buf[4096];
  int64_t got = 0;
  while (got < h.entries && fgets(buf, sizeof buf, f)) {
    ++h.line;
    char* p = buf;
    while (*p == ' ' || *p == '\t') ++p;
    if (*p == '%' || *p == '\n' || *p == '\r' || *p == 0) continue;
    char* end;
    errno = 0;
    const long long i = strtoll(p, &end, 10);
    if (end == p) goto malformed;
    p = end;
    {
      const long long j = strtoll(p, &end, 10);
      if (end == p) goto malformed;
      p = end;
      double v = 1.0;
      if (!h.pattern) {
        v = strtod(p, &end);
        if (end == p) goto malformed;
      }
      if (i < 1 || i > h.n || j < 1 || j > h.m) {
        fclose(f);
        gmf::set_error("%s: line %lld: index (%lld, %lld) out of range", path, (long long)h.line, i, j);
        return GMF_ERR_CONFIG;
      }
      if (!(v >= 0.0) || v != std::floor(v) || v > 2147483647.0) {
        fclose(f);
        gmf::set_error("%s: line %lld: value %g is not a count (nonnegative integer < 2^31)", path,
                       (long long)h.line, v);
        return GMF_ERR_DOMAIN;
      }
      ri.push_back((int32_t)(i - 1)); ci.push_back((int32_t)(j - 1)); vv.push_back(v);
      if (h.symmetric && i != j) {
        ri.push_back((int32_t)(j - 1)); ci.push_back((int32_t)(i - 1)); vv.push_back(v);
      }
      ++got;
      continue;
    }
  malformed:
    fclose(f);
    gmf::set_error("%s: line %lld: expected 'row col%s'", path, (long long)h.line,
                   h.pattern ? "" : " value");
    return GMF_ERR_CONFIG;
  }
  fclose(f);
  if (got < h.entries) {
    gmf::set_error("%s: %lld entries declared, %lld found", path, (long long)h.entries,
                   (long long)got);
    return GMF_ERR_CONFIG;
  }
  // pass 2: counting sort by row, then each row sorted by column with
  // duplicates summed (scipy coo -> dense adds them) and zeros dropped
  const int64_t t = (int64_t)ri.size();
  std::vector<int64_t> start(h.n + 1, 0);
  for (int64_t k = 0; k < t; ++k) ++start[ri[k] + 1];
  for (int64_t r = 0; r < h.n; ++r) start[r + 1] += start[r];
  std::vector<int64_t> fill(start.begin(), start.end() - 1), order(t);
  for (int64_t k = 0; k < t; ++k) order[fill[ri[k]]++] = k;
  int64_t w = 0;
  indptr[0] = 0;
  std::vector<std::pair<int32_t, double>> row;
  for (int64_t r = 0; r < h.n; ++r) {
    row.clear();
    for (int64_t k = start[r]; k < start[r + 1]; ++k) row.emplace_back(ci[order[k]], vv[order[k]]);
    std::stable_sort(row.begin(), row.end(),
                     [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
                       return a.first < b.first;
                     });
    for (size_t k = 0; k < row.size();) {
      size_t e = k;
      double sum = 0.0;
      while (e < row.size() && row[e].first == row[k].first) sum += row[e++].second;
      if (sum > 2147483647.0) {
        gmf::set_error("%s: summed duplicate entry exceeds int32", path);
        return GMF_ERR_DOMAIN;
      }
      if (sum != 0.0) {
        indices[w] = row[k].first;
        counts[w] = (int32_t)sum;
        ++w;
      }
      k = e;
    }
    indptr[r + 1] = w;
  }
  *nnz_out = w;
  return GMF_OK;
}

}  // extern "C"
