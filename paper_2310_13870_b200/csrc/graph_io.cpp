// Graph files on either side of the hot path.
//
//  * Text edge list, byte-compatible with the reference
//    (proj/src/graph.cpp:234-276): header "n m\n", then one "u v w\n" line
//    per edge with w printed as "%.17g" (round-trip exact). The reference's
//    CLI and tools (--graph-out, eigengap, cluster) read these files.
//  * Binary CSR: the upper-triangular CSR of include/fsgg.h's fsgg_graph,
//    written as raw little-endian arrays (no text conversion).
//
// Host code: formatting and parsing are split over threads in fixed chunks,
// and each chunk's output is identical to the sequential loop's, so files do
// not depend on the thread count.
#include <algorithm>
#include <atomic>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fsgg.h"
#include "common.cuh"

namespace fsgg {
namespace {

struct IoError : Error {
  explicit IoError(const std::string& m) : Error(m, 3) {}
};

struct File {
  std::FILE* f = nullptr;
  File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

uint32_t resolve_threads(uint32_t threads, uint64_t work, uint64_t per_thread_min) {
  uint32_t t = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
  const uint64_t useful = std::max<uint64_t>(1, work / std::max<uint64_t>(1, per_thread_min));
  return static_cast<uint32_t>(std::min<uint64_t>(t, useful));
}

template <class F>
void parallel_for(uint32_t threads, uint64_t count, F&& f) {
  if (threads <= 1 || count <= 1) {
    for (uint64_t i = 0; i < count; ++i) f(i);
    return;
  }
  std::atomic<uint64_t> next{0};
  std::vector<std::thread> pool;
  std::exception_ptr err;
  std::atomic<bool> failed{false};
  for (uint32_t t = 0; t < threads; ++t) {
    pool.emplace_back([&] {
      try {
        for (uint64_t i = next++; i < count && !failed; i = next++) f(i);
      } catch (...) {
        if (!failed.exchange(true)) err = std::current_exception();
      }
    });
  }
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

template <class T>
T* host_array(uint64_t count) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<uint64_t>(count, 1)));
  if (!p) throw std::bad_alloc();
  return p;
}

inline char* put_u64(char* p, uint64_t x) { return std::to_chars(p, p + 24, x).ptr; }

// One "u v w\n" line; w exactly as printf("%.17g") (std::to_chars with a
// precision is specified "as if by printf in the C locale").
inline char* put_edge(char* p, uint32_t u, uint32_t v, double w) {
  p = put_u64(p, u);
  *p++ = ' ';
  p = put_u64(p, v);
  *p++ = ' ';
  p = std::to_chars(p, p + 40, w, std::chars_format::general, 17).ptr;
  *p++ = '\n';
  return p;
}

constexpr uint64_t kLineMax = 10 + 1 + 10 + 1 + 32 + 1;  // u32, u32, %.17g
constexpr uint64_t kChunkEdges = 1u << 18;

// Degrees and total weight in the reference's order
// (WeightedGraph::WeightedGraph, proj/src/graph.cpp:14-21).
void finish_host_graph(fsgg_graph* g) {
  const uint32_t n = g->n;
  const uint64_t m = g->num_edges;
  g->degrees = host_array<double>(n);
  g->row_ptr = host_array<uint64_t>(uint64_t(n) + 1);
  std::fill(g->degrees, g->degrees + n, 0.0);
  double total = 0.0;
  for (uint64_t i = 0; i < m; ++i) {
    g->degrees[g->u[i]] += g->w[i];
    g->degrees[g->v[i]] += g->w[i];
    total += g->w[i];
  }
  g->total_weight = total;
  uint64_t e = 0;
  for (uint32_t r = 0; r <= n; ++r) {
    while (e < m && g->u[e] < r) ++e;
    g->row_ptr[r] = e;
  }
}

inline bool is_space(char c) {
  return c == ' ' || c == '\n' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}

}  // namespace

void graph_save_text(const char* path, uint32_t n, uint64_t m, const uint32_t* u,
                     const uint32_t* v, const double* w, uint32_t threads) {
  if (!path) throw ConfigError("path is null");
  if (m && (!u || !v || !w)) throw ConfigError("edge arrays are null");
  File out(path, "wb");
  if (!out.f) throw IoError(std::string("cannot write ") + path);  // graph.cpp:265-268
  char head[64];
  char* p = put_u64(head, n);
  *p++ = ' ';
  p = put_u64(p, m);
  *p++ = '\n';
  if (std::fwrite(head, 1, p - head, out.f) != size_t(p - head))
    throw IoError(std::string("failed writing ") + path);
  const uint64_t chunks = (m + kChunkEdges - 1) / kChunkEdges;
  const uint32_t t = resolve_threads(threads, chunks, 1);
  // format `t` chunks in parallel, then append them in order
  std::vector<std::vector<char>> buf(t);
  std::vector<uint64_t> len(t);
  for (uint64_t c0 = 0; c0 < chunks; c0 += t) {
    const uint64_t batch = std::min<uint64_t>(t, chunks - c0);
    parallel_for(t, batch, [&](uint64_t b) {
      const uint64_t e0 = (c0 + b) * kChunkEdges, e1 = std::min(m, e0 + kChunkEdges);
      buf[b].resize((e1 - e0) * kLineMax);
      char* q = buf[b].data();
      for (uint64_t e = e0; e < e1; ++e) q = put_edge(q, u[e], v[e], w[e]);
      len[b] = q - buf[b].data();
    });
    for (uint64_t b = 0; b < batch; ++b)
      if (std::fwrite(buf[b].data(), 1, len[b], out.f) != len[b])
        throw IoError(std::string("failed writing ") + path);
  }
  if (std::fflush(out.f) != 0) throw IoError(std::string("failed writing ") + path);
}

// fsg::read_edge_list (graph.cpp:243-263): whitespace-separated tokens
// "n m" then m triples "u v w"; u > v is swapped, unsorted input is sorted by
// (u, v); trailing tokens are ignored. Indices >= n are rejected here (the
// reference would index out of bounds).
void graph_load_text(const char* path, uint32_t threads, fsgg_graph* g) {
  if (!path || !g) throw ConfigError("null argument");
  std::memset(g, 0, sizeof(*g));
  File in(path, "rb");
  if (!in.f) throw IoError(std::string("cannot open ") + path);  // graph.cpp:273-274
  std::fseek(in.f, 0, SEEK_END);
  const long size = std::ftell(in.f);
  std::fseek(in.f, 0, SEEK_SET);
  if (size < 0) throw IoError(std::string("cannot read ") + path);
  std::vector<char> text(size_t(size) + 1);
  if (std::fread(text.data(), 1, size_t(size), in.f) != size_t(size))
    throw IoError(std::string("cannot read ") + path);
  text[size] = '\n';
  const char* s = text.data();
  const char* end = s + size;

  auto next_token = [&](const char*& p, const char*& tb, const char*& te) {
    while (p < end && is_space(*p)) ++p;
    tb = p;
    while (p < end && !is_space(*p)) ++p;
    te = p;
    return tb < te;
  };
  const char* p = s;
  const char *tb, *te;
  uint64_t hv[2];
  for (int k = 0; k < 2; ++k) {
    if (!next_token(p, tb, te) || std::from_chars(tb, te, hv[k]).ptr != te ||
        (k == 0 && hv[0] > UINT32_MAX))
      throw IoError("edge list: malformed header");
  }
  const uint32_t n = static_cast<uint32_t>(hv[0]);
  const uint64_t m = hv[1];
  if (m > uint64_t(size)) throw IoError("edge list: malformed edge");  // >= 6 bytes per edge

  // Split the body at whitespace into chunks, count tokens per chunk, then
  // parse each chunk knowing the global index of its first token.
  const char* body = p;
  const uint64_t body_len = end - body;
  const uint64_t target = 1u << 22;
  std::vector<const char*> cut{body};
  while (cut.back() < end) {
    const char* c = cut.back() + std::min<uint64_t>(target, end - cut.back());
    while (c < end && !is_space(*c)) ++c;
    cut.push_back(c);
  }
  const uint64_t nch = cut.size() - 1;
  const uint32_t t = resolve_threads(threads, body_len, 1u << 20);
  std::vector<uint64_t> ntok(nch + 1, 0);
  parallel_for(t, nch, [&](uint64_t c) {
    const char* q = cut[c];
    const char *b, *e;
    uint64_t k = 0;
    while (q < cut[c + 1]) {
      while (q < cut[c + 1] && is_space(*q)) ++q;
      if (q >= cut[c + 1]) break;
      b = q;
      while (q < cut[c + 1] && !is_space(*q)) ++q;
      e = q;
      k += b < e;
    }
    ntok[c + 1] = k;
  });
  for (uint64_t c = 0; c < nch; ++c) ntok[c + 1] += ntok[c];
  if (ntok[nch] < 3 * m) throw IoError("edge list: malformed edge");

  g->n = n;
  g->num_edges = m;
  g->u = host_array<uint32_t>(m);
  g->v = host_array<uint32_t>(m);
  g->w = host_array<double>(m);
  std::atomic<bool> bad{false}, range{false};
  parallel_for(t, nch, [&](uint64_t c) {
    uint64_t k = ntok[c];
    if (k >= 3 * m) return;
    const char* q = cut[c];
    while (q < cut[c + 1] && k < 3 * m) {
      while (q < cut[c + 1] && is_space(*q)) ++q;
      if (q >= cut[c + 1]) break;
      const char* b = q;
      while (q < cut[c + 1] && !is_space(*q)) ++q;
      const uint64_t e = k / 3;
      bool ok;
      if (k % 3 == 2) {
        double x;
        const auto r = std::from_chars(b, q, x);
        ok = r.ec == std::errc() && r.ptr == q;
        g->w[e] = x;
      } else {
        uint32_t x;
        const auto r = std::from_chars(b, q, x);
        ok = r.ec == std::errc() && r.ptr == q;
        if (ok && x >= n) range = true;
        (k % 3 == 0 ? g->u : g->v)[e] = x;
      }
      if (!ok) bad = true;
      ++k;
    }
  });
  auto fail = [&](const char* msg) {
    fsgg_graph_free(g);
    throw IoError(msg);
  };
  if (bad) fail("edge list: malformed edge");
  if (range) fail("edge list: vertex index out of range");
  bool sorted = true;
  for (uint64_t e = 0; e < m; ++e) {
    if (g->u[e] > g->v[e]) std::swap(g->u[e], g->v[e]);
    if (e && (g->u[e - 1] > g->u[e] || (g->u[e - 1] == g->u[e] && g->v[e - 1] > g->v[e])))
      sorted = false;
  }
  if (!sorted) {
    std::vector<uint64_t> idx(m);
    for (uint64_t e = 0; e < m; ++e) idx[e] = e;
    std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
      return g->u[a] != g->u[b] ? g->u[a] < g->u[b] : g->v[a] < g->v[b];
    });
    std::vector<uint32_t> uu(m), vv(m);
    std::vector<double> ww(m);
    for (uint64_t e = 0; e < m; ++e) {
      uu[e] = g->u[idx[e]];
      vv[e] = g->v[idx[e]];
      ww[e] = g->w[idx[e]];
    }
    std::copy(uu.begin(), uu.end(), g->u);
    std::copy(vv.begin(), vv.end(), g->v);
    std::copy(ww.begin(), ww.end(), g->w);
  }
  finish_host_graph(g);
}

// Binary CSR: "FSGGCSR1", u32 n, u32 0, u64 m, f64 total_weight,
// row_ptr[n+1] u64, v[m] u32, w[m] f64, degrees[n] f64 (little-endian).
namespace {
constexpr char kCsrMagic[8] = {'F', 'S', 'G', 'G', 'C', 'S', 'R', '1'};
}

void graph_save_csr(const char* path, const fsgg_graph* g) {
  if (!path || !g) throw ConfigError("null argument");
  if (g->num_edges && (!g->v || !g->w)) throw ConfigError("edge arrays are null");
  if (!g->row_ptr || !g->degrees) throw ConfigError("graph has no row_ptr/degrees");
  File out(path, "wb");
  if (!out.f) throw IoError(std::string("cannot write ") + path);
  const uint32_t hdr32[2] = {g->n, 0u};
  const uint64_t m = g->num_edges;
  bool ok = std::fwrite(kCsrMagic, 1, 8, out.f) == 8 &&
            std::fwrite(hdr32, 4, 2, out.f) == 2 && std::fwrite(&m, 8, 1, out.f) == 1 &&
            std::fwrite(&g->total_weight, 8, 1, out.f) == 1 &&
            std::fwrite(g->row_ptr, 8, uint64_t(g->n) + 1, out.f) == uint64_t(g->n) + 1 &&
            std::fwrite(g->v, 4, m, out.f) == m && std::fwrite(g->w, 8, m, out.f) == m &&
            std::fwrite(g->degrees, 8, g->n, out.f) == g->n && std::fflush(out.f) == 0;
  if (!ok) throw IoError(std::string("failed writing ") + path);
}

void graph_load_csr(const char* path, fsgg_graph* g) {
  if (!path || !g) throw ConfigError("null argument");
  std::memset(g, 0, sizeof(*g));
  File in(path, "rb");
  if (!in.f) throw IoError(std::string("cannot open ") + path);
  char magic[8];
  uint32_t hdr32[2];
  uint64_t m = 0;
  double tw = 0.0;
  if (std::fread(magic, 1, 8, in.f) != 8 || std::memcmp(magic, kCsrMagic, 8) != 0 ||
      std::fread(hdr32, 4, 2, in.f) != 2 || std::fread(&m, 8, 1, in.f) != 1 ||
      std::fread(&tw, 8, 1, in.f) != 1)
    throw IoError(std::string("not an fsgg CSR file: ") + path);
  const uint32_t n = hdr32[0];
  std::fseek(in.f, 0, SEEK_END);
  const uint64_t size = uint64_t(std::ftell(in.f));
  const uint64_t expect = 32 + 8 * (uint64_t(n) + 1) + 12 * m + 8 * uint64_t(n);
  if (size != expect) throw IoError(std::string("truncated or corrupt CSR file: ") + path);
  std::fseek(in.f, 32, SEEK_SET);
  g->n = n;
  g->num_edges = m;
  g->total_weight = tw;
  g->row_ptr = host_array<uint64_t>(uint64_t(n) + 1);
  g->u = host_array<uint32_t>(m);
  g->v = host_array<uint32_t>(m);
  g->w = host_array<double>(m);
  g->degrees = host_array<double>(n);
  bool ok = std::fread(g->row_ptr, 8, uint64_t(n) + 1, in.f) == uint64_t(n) + 1 &&
            std::fread(g->v, 4, m, in.f) == m && std::fread(g->w, 8, m, in.f) == m &&
            std::fread(g->degrees, 8, n, in.f) == n;
  ok = ok && g->row_ptr[0] == 0 && g->row_ptr[n] == m;
  for (uint32_t r = 0; ok && r < n; ++r) {
    if (g->row_ptr[r] > g->row_ptr[r + 1]) {
      ok = false;
      break;
    }
    for (uint64_t e = g->row_ptr[r]; e < g->row_ptr[r + 1]; ++e) {
      g->u[e] = r;
      if (g->v[e] <= r || g->v[e] >= n) ok = false;
    }
  }
  if (!ok) {
    fsgg_graph_free(g);
    throw IoError(std::string("corrupt CSR file: ") + path);
  }
}

// ---- point files (proj/src/dataset.cpp:54-130) ------------------------------
// load_csv: lines split at '\n' (empty lines skipped), fields at ',', '\r'
// dropped; a first row whose first field is not a number is a header, and
// a trailing "label" header column marks integer labels. Values parse as
// std::from_chars doubles with surrounding whitespace allowed; any other
// field, a wrong field count, a negative label or no data rows is an I/O
// error (code 3), a non-finite value a config error (the Dataset
// constructor's check, code 2). Rows are parsed in parallel chunks; the
// error reported is the first one in file order, as sequentially.
namespace {

bool csv_double(const char* b, const char* e, double& out) {
  while (b < e && std::isspace(static_cast<unsigned char>(*b))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(e[-1]))) --e;
  if (b == e) return false;
  const auto r = std::from_chars(b, e, out);
  return r.ec == std::errc() && r.ptr == e;
}

// fields of [b, e) (one line) with '\r' removed, as split_fields does
void csv_fields(const char* b, const char* e, std::vector<std::string>& out) {
  out.clear();
  std::string cur;
  for (const char* p = b; p < e; ++p) {
    if (*p == ',') {
      out.push_back(cur);
      cur.clear();
    } else if (*p != '\r') {
      cur += *p;
    }
  }
  out.push_back(cur);
}

struct CsvChunk {
  std::vector<double> values;
  std::vector<uint32_t> labels;
  std::string error;  // first error in this chunk ("" = none)
};

}  // namespace

void csv_load(const char* path, uint32_t threads, double** points, uint32_t* n_out,
              uint32_t* d_out, uint32_t** labels_out) {
  if (!path || !points || !n_out || !d_out) throw ConfigError("null argument");
  *points = nullptr;
  if (labels_out) *labels_out = nullptr;
  File in(path, "rb");
  if (!in.f) throw IoError(std::string("cannot open ") + path);
  std::fseek(in.f, 0, SEEK_END);
  const long size = std::ftell(in.f);
  std::fseek(in.f, 0, SEEK_SET);
  if (size < 0) throw IoError(std::string("cannot read ") + path);
  std::vector<char> text(size_t(size) + 1);
  if (size && std::fread(text.data(), 1, size_t(size), in.f) != size_t(size))
    throw IoError(std::string("cannot read ") + path);
  const char* s = text.data();
  const char* end = s + size;
  auto line_end = [&](const char* p) {
    const void* q = std::memchr(p, '\n', size_t(end - p));
    return q ? static_cast<const char*>(q) : end;
  };
  // first non-empty line: header or the first data row
  const char* p = s;
  std::vector<std::string> f;
  bool has_labels = false, header = false;
  uint32_t d = 0;
  while (p < end) {
    const char* le = line_end(p);
    if (le > p) {
      csv_fields(p, le, f);
      double probe;
      if (!csv_double(f[0].data(), f[0].data() + f[0].size(), probe)) {
        has_labels = !f.empty() && f.back() == "label";
        d = static_cast<uint32_t>(f.size() - (has_labels ? 1 : 0));
        header = true;
        p = le < end ? le + 1 : end;
      } else {
        d = static_cast<uint32_t>(f.size());
      }
      break;
    }
    p = le < end ? le + 1 : end;
  }
  (void)header;
  const uint32_t expect = d + (has_labels ? 1u : 0u);
  // line-aligned chunks of the body, parsed in parallel
  const uint64_t target = 1u << 22;
  std::vector<const char*> cut{p};
  while (cut.back() < end) {
    const char* c = cut.back() + std::min<uint64_t>(target, uint64_t(end - cut.back()));
    c = c < end ? line_end(c) : end;
    cut.push_back(c < end ? c + 1 : end);
  }
  const uint64_t nch = cut.size() - 1;
  std::vector<CsvChunk> chunks(nch);
  const uint32_t t = resolve_threads(threads, uint64_t(end - p), 1u << 20);
  parallel_for(t, nch, [&](uint64_t c) {
    CsvChunk& ch = chunks[c];
    std::vector<std::string> fl;
    for (const char* q = cut[c]; q < cut[c + 1];) {
      const char* le = line_end(q);
      if (le > q) {
        csv_fields(q, le, fl);
        if (fl.size() != expect) {
          ch.error = std::string(path) + ": row with " + std::to_string(fl.size()) +
                     " fields, expected " + std::to_string(expect);
          return;
        }
        for (uint32_t k = 0; k < d; ++k) {
          double v;
          if (!csv_double(fl[k].data(), fl[k].data() + fl[k].size(), v)) {
            ch.error = std::string(path) + ": cannot parse value '" + fl[k] + "'";
            return;
          }
          ch.values.push_back(v);
        }
        if (has_labels) {
          double v;
          if (!csv_double(fl[d].data(), fl[d].data() + fl[d].size(), v) || v < 0) {
            ch.error = std::string(path) + ": cannot parse label '" + fl[d] + "'";
            return;
          }
          ch.labels.push_back(static_cast<uint32_t>(v));
        }
      }
      q = le < end ? le + 1 : end;
    }
  });
  uint64_t nv = 0;
  for (const CsvChunk& ch : chunks) {
    if (!ch.error.empty()) throw IoError(ch.error);
    nv += ch.values.size();
  }
  if (nv == 0) throw IoError(std::string(path) + ": no data rows");
  if (d < 1) throw ConfigError("dataset needs n >= 1 and d >= 1");
  const uint64_t n = nv / d;
  if (n > UINT32_MAX) throw ConfigError("too many points");
  double* pts = host_array<double>(nv);
  uint32_t* lab = has_labels && labels_out ? host_array<uint32_t>(n) : nullptr;
  uint64_t at = 0, la = 0;
  for (const CsvChunk& ch : chunks) {
    std::copy(ch.values.begin(), ch.values.end(), pts + at);
    at += ch.values.size();
    if (lab) {
      std::copy(ch.labels.begin(), ch.labels.end(), lab + la);
      la += ch.labels.size();
    }
  }
  for (uint64_t i = 0; i < nv; ++i)
    if (!std::isfinite(pts[i])) {  // Dataset::Dataset (dataset.cpp:19-22)
      std::free(pts);
      std::free(lab);
      throw ConfigError("dataset coordinates must be finite");
    }
  *points = pts;
  *n_out = static_cast<uint32_t>(n);
  *d_out = d;
  if (labels_out) *labels_out = lab;
}

// save_csv: header "x0,...,x{d-1}[,label]", values "%.17g" (std::to_chars
// with precision 17), rows formatted in parallel chunks, written in order.
void csv_save(const char* path, const double* pts, uint32_t n, uint32_t d,
              const uint32_t* labels, uint32_t threads) {
  if (!path || (n && !pts)) throw ConfigError("null argument");
  if (d < 1 || n < 1) throw ConfigError("dataset needs n >= 1 and d >= 1");
  File out(path, "wb");
  if (!out.f) throw IoError(std::string("cannot write ") + path);
  std::string head;
  for (uint32_t c = 0; c < d; ++c) {
    if (c) head += ',';
    head += 'x';
    head += std::to_string(c);
  }
  if (labels) head += ",label";
  head += '\n';
  bool ok = std::fwrite(head.data(), 1, head.size(), out.f) == head.size();
  const uint64_t rows_per = std::max<uint64_t>(1, (1u << 18) / d);
  const uint64_t chunks = (uint64_t(n) + rows_per - 1) / rows_per;
  const uint32_t t = resolve_threads(threads, chunks, 1);
  std::vector<std::vector<char>> buf(t);
  std::vector<uint64_t> len(t);
  for (uint64_t c0 = 0; ok && c0 < chunks; c0 += t) {
    const uint64_t batch = std::min<uint64_t>(t, chunks - c0);
    parallel_for(t, batch, [&](uint64_t b) {
      const uint64_t r0 = (c0 + b) * rows_per, r1 = std::min<uint64_t>(n, r0 + rows_per);
      buf[b].resize((r1 - r0) * (uint64_t(d) * 33 + 12));
      char* q = buf[b].data();
      for (uint64_t r = r0; r < r1; ++r) {
        for (uint32_t c = 0; c < d; ++c) {
          if (c) *q++ = ',';
          q = std::to_chars(q, q + 32, pts[r * d + c], std::chars_format::general, 17).ptr;
        }
        if (labels) {
          *q++ = ',';
          q = put_u64(q, labels[r]);
        }
        *q++ = '\n';
      }
      len[b] = q - buf[b].data();
    });
    for (uint64_t b = 0; ok && b < batch; ++b)
      ok = std::fwrite(buf[b].data(), 1, len[b], out.f) == len[b];
  }
  if (!ok || std::fflush(out.f) != 0) throw IoError(std::string("failed writing ") + path);
}

}  // namespace fsgg
