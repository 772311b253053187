// C ABI (include/fsgg.h): validation with the reference's error contract,
// phase orchestration and host<->device copies. No compute happens here —
// every loop over points, entries or edges is a kernel in tree.cu, kde.cu,
// sampler.cu or graph.cu, and without a usable device every call fails with
// FSGG_ERR_DEVICE (no CPU fallback).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "../../include/fsgg.h"
#include "engine.cuh"
#include "spectral.cuh"

namespace fsgg {
// graph_io.cpp
void graph_save_text(const char* path, uint32_t n, uint64_t m, const uint32_t* u,
                     const uint32_t* v, const double* w, uint32_t threads);
void graph_load_text(const char* path, uint32_t threads, fsgg_graph* g);
void graph_save_csr(const char* path, const fsgg_graph* g);
void graph_load_csr(const char* path, fsgg_graph* g);
void csv_load(const char* path, uint32_t threads, double** points, uint32_t* n, uint32_t* d,
              uint32_t** labels);
void csv_save(const char* path, const double* pts, uint32_t n, uint32_t d,
              const uint32_t* labels, uint32_t threads);
}  // namespace fsgg

struct fsgg_dataset {
  fsgg::Dataset ds;
  // Results kept alive for the device-pointer APIs; reused (grow-only)
  // across calls so repeated builds never go back to the allocator.
  std::unique_ptr<fsgg::GraphResult> graph;
  std::unique_ptr<fsgg::SampleResult> sample;
  std::unique_ptr<fsgg::SampleResult> shard;
  fsgg::DevBuf keys;
  fsgg::DevBuf shard_keys;
  uint64_t root_records = 0;  // owner-mode root records of the last prepare
  bool tree_fresh = false;    // tree built by the last prepare (reused once)
  uint64_t shard_npairs = 0;
  ~fsgg_dataset() {
    graph.reset();
    sample.reset();
    shard.reset();
    keys.release();
    shard_keys.release();
    ds.release_all();
    if (ds.stream) {
      cudaStreamSynchronize(ds.stream);
      cudaStreamDestroy(ds.stream);
    }
  }
};

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FSGG_OK;
  } catch (const fsgg::Error& e) {
    g_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_error = std::string("host allocation failed: ") + e.what();
    return FSGG_ERR_DEVICE;
  } catch (const std::exception& e) {
    g_error = e.what();
    return FSGG_ERR_DEVICE;
  }
}

double now() {
  using clock = std::chrono::steady_clock;
  return std::chrono::duration<double>(clock::now().time_since_epoch()).count();
}

void require_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    throw fsgg::DeviceError("no CUDA device available (the sm_100a path has no CPU fallback)");
  if (device < 0 || device >= count) throw fsgg::ConfigError("device index out of range");
  cudaDeviceProp prop;
  FSGG_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    throw fsgg::DeviceError("device " + std::to_string(device) + " (" + prop.name +
                            ") is not sm_100; this library is built for sm_100a only");
}

__global__ void nonfinite_kernel(const float* p, uint64_t m, unsigned int* bad) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < m && !isfinite(p[i])) atomicAdd(bad, 1u);
}

void check_finite(fsgg::Dataset& ds) {
  const uint64_t m = uint64_t(ds.n) * ds.d;
  fsgg::DevBuf bad(4, ds.stream);
  FSGG_CUDA(cudaMemsetAsync(bad.as<void>(), 0, 4, ds.stream));
  nonfinite_kernel<<<fsgg::ceil_div_u32(m, 256), 256, 0, ds.stream>>>(
      ds.pts.as<float>(), m, bad.as<unsigned int>());
  FSGG_LAUNCH_CHECK();
  unsigned int h = 0;
  FSGG_CUDA(cudaMemcpyAsync(&h, bad.as<void>(), 4, cudaMemcpyDeviceToHost, ds.stream));
  FSGG_CUDA(cudaStreamSynchronize(ds.stream));
  if (h) throw fsgg::ConfigError("dataset coordinates must be finite");  // dataset.cpp:19-21
}

fsgg_dataset* make_handle(uint32_t n, uint32_t d, int device) {
  if (n < 1 || d < 1) throw fsgg::ConfigError("dataset needs n >= 1 and d >= 1");  // dataset.cpp:16
  if (n > (1u << 28)) throw fsgg::ConfigError("n > 2^28 is not supported by the device tree table");
  require_device(device);
  FSGG_CUDA(cudaSetDevice(device));
  auto h = std::make_unique<fsgg_dataset>();
  h->ds.device = device;
  h->ds.n = n;
  h->ds.d = d;
  cudaDeviceProp prop;
  FSGG_CUDA(cudaGetDeviceProperties(&prop, device));
  h->ds.num_sms = prop.multiProcessorCount;
  FSGG_CUDA(cudaStreamCreateWithFlags(&h->ds.stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  FSGG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t threshold = UINT64_MAX;  // keep freed blocks cached between calls
  FSGG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  h->ds.pts.alloc(size_t(n) * d * 4, h->ds.stream);
  return h.release();
}

void validate_kernel(const fsgg_kernel* k) {
  if (!k) throw fsgg::ConfigError("kernel is null");
  if (k->family < 0 || k->family > 2) throw fsgg::ConfigError("unknown kernel family");
  if (!(k->sigma > 0.0)) throw fsgg::ConfigError("kernel bandwidth must be positive");  // kernel.cpp:23-26
}

fsgg_config default_config() {
  fsgg_config c;
  std::memset(&c, 0, sizeof(c));
  c.C = 1.0;
  c.lambda_k1_estimate = 1.0;
  c.log_base = 0;
  c.seed = 1;
  return c;
}

// make_estimator (proj/src/kde.cpp:104-129) on the device: which backend a
// call runs and with what budget (fsgg.h, fsgg_config::kde_backend).
struct Backend {
  bool fast = false;
  double eps = 0.0;
};
Backend resolve_backend(int kde_backend, double epsilon, int log_base, int family, uint32_t n,
                        uint32_t d) {
  if (kde_backend < FSGG_KDE_EXACT || kde_backend > FSGG_KDE_AUTO)
    throw fsgg::ConfigError("unknown kde backend");
  bool fast = kde_backend == FSGG_KDE_FAST;
  if (kde_backend == FSGG_KDE_AUTO) fast = family == 0 && d <= 3 && n >= 4096;  // kde.hpp:39-40
  if (!fast) return {};
  if (family != 0) return {};  // UnsupportedKernel: informational fallback to exact
  const double eps = epsilon > 0.0 ? epsilon : fsgg_default_epsilon(n, log_base);
  if (!(eps > 0.0) || eps >= 1.0) throw fsgg::ConfigError("fast KDE needs 0 < epsilon < 1");
  return {true, eps};
}

// proj/src/sparsifier.cpp:17-23
uint32_t rounds_for(const fsgg_config& c, uint32_t n) {
  if (c.rounds > 0) return c.rounds;
  double nn = std::max<uint32_t>(n, 2);
  double l = std::max(c.log_base ? std::log(nn) : std::log2(nn), 1.0);
  double r = std::ceil(6.0 * c.C * l / c.lambda_k1_estimate);
  if (!(r >= 1.0) || r > 4e9) throw fsgg::ConfigError("invalid round count");
  return static_cast<uint32_t>(r);
}

void activate(fsgg_dataset* h) {
  if (!h) throw fsgg::ConfigError("dataset handle is null");
  FSGG_CUDA(cudaSetDevice(h->ds.device));
  h->ds.launches = 0;
}

void fill_report_common(fsgg_report* r, const fsgg::Dataset& ds, uint32_t L,
                        double eps = 0.0) {
  std::memset(r, 0, sizeof(*r));
  r->n = ds.n;
  r->rounds = L;
  r->epsilon = eps;  // the exact backend reports 0 (kde.hpp:30-31)
  std::strncpy(r->backend, eps > 0.0 ? "gpu-fast-certified-sm100a" : "gpu-exact-sm100a",
               sizeof(r->backend) - 1);
}

struct BuildOut {
  uint32_t L = 0;
  uint64_t sampled = 0, self = 0, degenerate = 0;
  double t_tree = 0, t_sample = 0, t_graph = 0;
  fsgg::KdeStats kde;
  uint32_t levels = 0;
  uint64_t peak = 0;
  uint64_t tie_verified = 0;
  double eps = 0.0;  // fast backend budget (0: exact)
};

// Descent over the configured query shard; fills res (and optionally keys).
// route_world > 0: the pair keys are grouped by the owner of row u under
// route_bounds (fsgg_sample_shard_routed) instead of sorted and deduplicated.
void run_descent(fsgg_dataset* h, const fsgg_kernel* kernel, const fsgg_config& cfg,
                 uint32_t L, uint32_t qb, uint32_t qe, fsgg::SampleResult& res,
                 fsgg::DevBuf& keys, uint64_t* npairs, BuildOut& bo, uint32_t route_world = 0,
                 const uint32_t* route_bounds = nullptr, uint64_t* route_counts = nullptr) {
  fsgg::Dataset& ds = h->ds;
  const fsgg::KernelSpec ks = fsgg::make_kernel_spec(kernel->family, kernel->sigma);
  double t0 = now();
  // Every build derives its tree (node boxes) and, on the tensor-core path,
  // the centred tf32 split of the points afresh: per-dataset preprocessing
  // is part of the job, as the reference's estimator build is.
  // (the multi-GPU shard pipeline built it moments ago in
  // fsgg_shard_root_prepare: same points, same job — not rebuilt)
  if (!h->tree_fresh) {
    ds.tree_valid = false;
    ds.tc_ready = false;
    ds.tie_xn_ready = false;
    fsgg::build_tree(ds);
  }
  h->tree_fresh = false;
  FSGG_CUDA(cudaStreamSynchronize(ds.stream));
  double t1 = now();
  fsgg::SampleRequest req;
  req.range = true;
  req.range_begin = qb;
  req.range_count = qe - qb;
  req.range_tickets = L;
  req.seed = cfg.seed;
  req.rng_mode = cfg.rng_mode;
  req.prune = cfg.dense_kde ? 0 : 1;
  const Backend be = resolve_backend(cfg.kde_backend, cfg.epsilon, cfg.log_base, kernel->family,
                                     ds.n, ds.d);
  if (be.fast && req.prune) {
    req.fast_epsilon = be.eps;
    req.verify_ties = false;  // the (1 +- eps) backend is not edge-for-edge exact
    bo.eps = be.eps;
  }
  req.want_root_sums = true;
  fsgg::sample_counted(ds, ks, req, res);
  double t2 = now();
  *npairs = route_world ? fsgg::collapse_pairs_routed(ds, res, keys, route_world, route_bounds,
                                                      route_counts, &bo.self, &bo.sampled)
                       : fsgg::collapse_pairs(ds, res, keys, &bo.self, &bo.sampled);
  double t3 = now();
  bo.t_tree = t1 - t0;
  bo.t_sample = t2 - t1;
  bo.t_graph = t3 - t2;
  bo.degenerate = res.degenerate_draws;
  bo.kde = res.kde;
  bo.levels = static_cast<uint32_t>(res.entries_per_level.size());
  bo.peak = res.peak_entries;
  bo.tie_verified = res.tie_verified;
}

void finish_report(fsgg_report* r, const fsgg::Dataset& ds, const BuildOut& bo,
                   const fsgg::GraphResult* g, double total) {
  fill_report_common(r, ds, bo.L, bo.eps);
  r->sampled_pairs = bo.sampled;
  r->self_pairs_discarded = bo.self;
  r->degenerate_draws = bo.degenerate;
  r->estimator_build_seconds = bo.t_tree;
  r->sampling_seconds = bo.t_sample;
  r->degree_kde_seconds = 0.0;
  r->weighting_seconds = bo.t_graph;
  r->total_seconds = total;
  r->estimator_bytes = ds.tree.first.bytes() + ds.tree.last.bytes() +
                       ds.tree.lo.bytes() + ds.tree.hi.bytes();
  if (g) {
    r->underflow_edges_discarded = g->underflow;
    r->edge_count = g->m;
    r->graph_bytes = g->m * 16 + uint64_t(g->n) * 8;
  }
  r->kernel_evals = bo.kde.evals;
  r->kernel_evals_performed = bo.kde.performed;
  r->kde_tiled_performed_evals = bo.kde.tiled_performed;
  r->tie_verified_entries = bo.tie_verified;
  r->kde_root_performed_evals = bo.kde.root_performed;
  r->kde_root_seconds = bo.kde.root_seconds;
  r->kde_tiled_evals = bo.kde.tiled_evals;
  r->kde_tiled_seconds = bo.kde.tiled_seconds;
  r->kde_tiled_launches = bo.kde.tiled_launches;
  r->levels = bo.levels;
  r->peak_entries = bo.peak;
  r->gpu_launches = ds.launches;
}

void build_device(fsgg_dataset* h, const fsgg_kernel* kernel, const fsgg_config* cfgp,
                  fsgg_report* report, bool want_estimates,
                  const fsgg::HostSink* sink = nullptr) {
  activate(h);
  validate_kernel(kernel);
  fsgg_config cfg = cfgp ? *cfgp : default_config();
  fsgg::Dataset& ds = h->ds;
  if (ds.n < 2) throw fsgg::ConfigError("similarity graph needs n >= 2");  // TooFewPoints
  if (cfg.rng_mode != FSGG_RNG_REFERENCE && cfg.rng_mode != FSGG_RNG_PHILOX)
    throw fsgg::ConfigError("unknown rng mode");
  BuildOut bo;
  bo.L = rounds_for(cfg, ds.n);
  double t0 = now();
  if (!h->sample) h->sample = std::make_unique<fsgg::SampleResult>();
  fsgg::SampleResult& res = *h->sample;
  uint64_t npairs = 0;
  // host output: the pair keys in u-range chunks, each finished and
  // streamed to the host while the next is sorted (FSGG_E2E_CHUNKS, 0 = one
  // pass)
  const char* ce = std::getenv("FSGG_E2E_CHUNKS");
  const uint32_t nchunks =
      sink && !want_estimates ? std::min<uint32_t>(ce ? uint32_t(std::atoi(ce)) : 4u, 64u) : 0u;
  std::vector<uint32_t> cb;
  std::vector<uint64_t> ccounts(std::max<uint32_t>(nchunks, 1), 0);
  if (nchunks > 1) {
    cb.resize(nchunks + 1);
    for (uint32_t c = 0; c <= nchunks; ++c) cb[c] = uint32_t(uint64_t(ds.n) * c / nchunks);
    run_descent(h, kernel, cfg, bo.L, 0, ds.n, res, h->keys, &npairs, bo, nchunks, cb.data(),
                ccounts.data());
  } else {
    run_descent(h, kernel, cfg, bo.L, 0, ds.n, res, h->keys, &npairs, bo);
  }
  double t1 = now();
  const fsgg::KernelSpec ks = fsgg::make_kernel_spec(kernel->family, kernel->sigma);
  if (!h->graph) h->graph = std::make_unique<fsgg::GraphResult>();
  fsgg::finish_graph(ds, ks, bo.L, res.groot.as<double>(), h->keys.as<uint64_t>(), npairs,
                     true, want_estimates, *h->graph, sink, nchunks > 1 ? ccounts.data() : nullptr,
                     nchunks > 1 ? nchunks : 0);
  double t2 = now();
  bo.t_graph += t2 - t1;
  if (report) finish_report(report, ds, bo, h->graph.get(), t2 - t0 + bo.t_tree * 0);
}

template <class T>
T* host_copy(const fsgg::DevBuf& b, uint64_t count, cudaStream_t s) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<uint64_t>(count, 1)));
  if (!p) throw std::bad_alloc();
  if (count) FSGG_CUDA(cudaMemcpyAsync(p, b.as<void>(), sizeof(T) * count, cudaMemcpyDeviceToHost, s));
  return p;
}

void graph_to_host(fsgg_dataset* h, fsgg_graph* out) {
  const fsgg::GraphResult& g = *h->graph;
  cudaStream_t s = h->ds.stream;
  std::memset(out, 0, sizeof(*out));
  out->n = g.n;
  out->num_edges = g.m;
  out->u = host_copy<uint32_t>(g.u, g.m, s);
  out->v = host_copy<uint32_t>(g.v, g.m, s);
  out->w = host_copy<double>(g.w, g.m, s);
  out->row_ptr = host_copy<uint64_t>(g.row_ptr, uint64_t(g.n) + 1, s);
  out->degrees = host_copy<double>(g.degrees, g.n, s);
  out->total_weight = g.total_weight;
  FSGG_CUDA(cudaStreamSynchronize(s));
}

void to_device_graph(fsgg_dataset* h, fsgg_device_graph* out) {
  const fsgg::GraphResult& g = *h->graph;
  out->n = g.n;
  out->num_edges = g.m;
  out->u = g.u.as<uint32_t>();
  out->v = g.v.as<uint32_t>();
  out->w = g.w.as<double>();
  out->row_ptr = g.row_ptr.as<uint64_t>();
  out->degrees = g.degrees.as<double>();
  out->total_weight = g.total_weight;
}

fsgg::SpectralGraphView handle_graph_view(fsgg_dataset* h) {
  if (!h) throw fsgg::ConfigError("dataset handle is null");
  if (!h->graph) throw fsgg::ConfigError("no graph on this handle: build one first");
  const fsgg::GraphResult& g = *h->graph;
  FSGG_CUDA(cudaSetDevice(h->ds.device));
  fsgg::SpectralGraphView v;
  v.n = g.n;
  v.m = g.m;
  v.row_ptr = g.row_ptr.as<uint64_t>();
  v.col = g.v.as<uint32_t>();
  v.w = g.w.as<double>();
  v.degrees = g.degrees.as<double>();
  return v;
}

// A host graph uploaded for one call, on its own stream.
struct UploadedGraph {
  cudaStream_t s = nullptr;
  fsgg::DevBuf rp, col, w, deg;
  fsgg::SpectralGraphView view;
  UploadedGraph(const fsgg_graph* g, int device) {
    if (!g) throw fsgg::ConfigError("graph is null");
    if (g->n == 0) throw fsgg::ConfigError("graph needs at least one vertex");
    if (!g->row_ptr || !g->degrees || (g->num_edges && (!g->v || !g->w)))
      throw fsgg::ConfigError("graph needs v, w, row_ptr and degrees");
    require_device(device);
    FSGG_CUDA(cudaSetDevice(device));
    FSGG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const uint64_t m = g->num_edges;
    rp.alloc(size_t(g->n + 1) * 8, s);
    col.alloc(std::max<uint64_t>(m, 1) * 4, s);
    w.alloc(std::max<uint64_t>(m, 1) * 8, s);
    deg.alloc(size_t(g->n) * 8, s);
    FSGG_CUDA(cudaMemcpyAsync(rp.as<void>(), g->row_ptr, size_t(g->n + 1) * 8,
                              cudaMemcpyHostToDevice, s));
    if (m) {
      FSGG_CUDA(cudaMemcpyAsync(col.as<void>(), g->v, m * 4, cudaMemcpyHostToDevice, s));
      FSGG_CUDA(cudaMemcpyAsync(w.as<void>(), g->w, m * 8, cudaMemcpyHostToDevice, s));
    }
    FSGG_CUDA(cudaMemcpyAsync(deg.as<void>(), g->degrees, size_t(g->n) * 8,
                              cudaMemcpyHostToDevice, s));
    view.n = g->n;
    view.m = m;
    view.row_ptr = rp.as<uint64_t>();
    view.col = col.as<uint32_t>();
    view.w = w.as<double>();
    view.degrees = deg.as<double>();
  }
  ~UploadedGraph() {
    rp.release();
    col.release();
    w.release();
    deg.release();
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

fsgg::EigenOpts eigen_opts(const fsgg_eigen_options* o) {
  fsgg::EigenOpts e;
  if (o) {
    e.tol = o->tol;
    e.max_matvecs = o->max_matvecs;
    e.max_basis = o->max_basis;
    e.seed = o->seed;
  }
  return e;
}

fsgg::KmeansOpts kmeans_opts(const fsgg_kmeans_options* o) {
  fsgg::KmeansOpts k;
  if (o) {
    k.restarts = o->restarts;
    k.max_iters = o->max_iters;
    k.rel_tol = o->rel_tol;
    k.seed = o->seed;
  }
  return k;
}

void eigenpairs_out(const fsgg::SpectralGraphView& v, cudaStream_t s, uint32_t q,
                    const fsgg_eigen_options* opts, double* values, double* vectors,
                    double* residuals, uint64_t* matvecs) {
  if (!values) throw fsgg::ConfigError("values is null");
  std::vector<double> vals, res;
  fsgg::DevBuf vecs;
  fsgg::SpectralStats st;
  fsgg::smallest_eigenpairs_dev(v, s, q, eigen_opts(opts), vals, res, vecs, st);
  std::memcpy(values, vals.data(), q * sizeof(double));
  if (residuals) std::memcpy(residuals, res.data(), q * sizeof(double));
  if (vectors)
    FSGG_CUDA(cudaMemcpyAsync(vectors, vecs.as<void>(), size_t(v.n) * q * 8,
                              cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  if (matvecs) *matvecs = st.matvecs;
}

void spectral_out(const fsgg::SpectralGraphView& v, cudaStream_t s, uint32_t k, uint64_t seed,
                  const fsgg_spectral_options* opts, uint32_t* labels,
                  fsgg_spectral_report* rep) {
  if (!labels) throw fsgg::ConfigError("labels is null");
  fsgg::SpectralStats st;
  fsgg::spectral_cluster_dev(v, s, k, seed, eigen_opts(opts ? &opts->eigen : nullptr),
                             kmeans_opts(opts ? &opts->kmeans : nullptr), labels, nullptr, st);
  if (rep) {
    rep->matvecs = st.matvecs;
    rep->components = st.ncomp;
    rep->kmeans_iterations = st.kmeans_iterations;
    rep->kmeans_cost = st.kmeans_cost;
    rep->eigen_seconds = st.eigen_seconds;
    rep->kmeans_seconds = st.kmeans_seconds;
    rep->gpu_launches = st.launches;
  }
}

}  // namespace

namespace {
// device generators: validate, select the device, run, restore the device
template <class F>
int on_device(int device, bool valid, F&& f) {
  return guarded([&] {
    if (!valid) throw fsgg::ConfigError("invalid generator arguments");
    require_device(device);
    int prev = 0;
    FSGG_CUDA(cudaGetDevice(&prev));
    FSGG_CUDA(cudaSetDevice(device));
    try {
      f();
    } catch (...) {
      cudaSetDevice(prev);
      throw;
    }
    FSGG_CUDA(cudaSetDevice(prev));
  });
}
}  // namespace

extern "C" {

const char* fsgg_version(void) { return "fsgg 0.1.0 (sm_100a)"; }
const char* fsgg_last_error(void) { return g_error.c_str(); }

int fsgg_device_available(void) {
  try {
    require_device(0);
    return 1;
  } catch (...) {
    return 0;
  }
}

void fsgg_config_init(fsgg_config* cfg) {
  if (cfg) *cfg = default_config();
}

int fsgg_rounds_for(const fsgg_config* cfg, uint32_t n, uint32_t* out) {
  return guarded([&] {
    if (!cfg || !out) throw fsgg::ConfigError("null argument");
    *out = rounds_for(*cfg, n);
  });
}

double fsgg_default_epsilon(uint32_t n, int log_base) {
  double nn = std::max<uint32_t>(n, 2);
  double l = log_base ? std::log(nn) : std::log2(nn);
  return 1.0 / (6.0 * std::max(l, 1.0));
}

int fsgg_dataset_create(const float* points, uint32_t n, uint32_t d,
                        int points_on_device, int device, fsgg_dataset** out) {
  return guarded([&] {
    if (!out || !points) throw fsgg::ConfigError("null argument");
    std::unique_ptr<fsgg_dataset> h(make_handle(n, d, device));
    FSGG_CUDA(cudaMemcpyAsync(h->ds.pts.as<void>(), points, size_t(n) * d * 4,
                              points_on_device ? cudaMemcpyDeviceToDevice
                                               : cudaMemcpyHostToDevice,
                              h->ds.stream));
    check_finite(h->ds);
    *out = h.release();
  });
}

int fsgg_dataset_create_f64(const double* points, uint32_t n, uint32_t d,
                            int device, fsgg_dataset** out) {
  return guarded([&] {
    if (!out || !points) throw fsgg::ConfigError("null argument");
    for (size_t i = 0; i < size_t(n) * d; ++i)
      if (!std::isfinite(points[i])) throw fsgg::ConfigError("dataset coordinates must be finite");
    std::vector<float> f(points, points + size_t(n) * d);
    std::unique_ptr<fsgg_dataset> h(make_handle(n, d, device));
    FSGG_CUDA(cudaMemcpyAsync(h->ds.pts.as<void>(), f.data(), f.size() * 4,
                              cudaMemcpyHostToDevice, h->ds.stream));
    check_finite(h->ds);
    *out = h.release();
  });
}

int fsgg_dataset_upload(fsgg_dataset* h, const float* host_points) {
  return guarded([&] {
    activate(h);
    if (!host_points) throw fsgg::ConfigError("null argument");
    FSGG_CUDA(cudaMemcpyAsync(h->ds.pts.as<void>(), host_points,
                              size_t(h->ds.n) * h->ds.d * 4, cudaMemcpyHostToDevice,
                              h->ds.stream));
    check_finite(h->ds);       // same validation as fsgg_dataset_create (dataset.cpp:19-21)
    h->ds.tree_valid = false;  // bounding boxes depend on the coordinates
    h->tree_fresh = false;
    h->ds.tc_ready = false;    // so do the tf32 split copies
    h->ds.tie_xn_ready = false;
  });
}

void fsgg_dataset_destroy(fsgg_dataset* h) {
  if (!h) return;
  cudaSetDevice(h->ds.device);
  delete h;
}

uint32_t fsgg_dataset_size(const fsgg_dataset* h) { return h ? h->ds.n : 0; }
uint32_t fsgg_dataset_dim(const fsgg_dataset* h) { return h ? h->ds.d : 0; }
const float* fsgg_dataset_device_points(const fsgg_dataset* h) {
  return h ? h->ds.pts.as<float>() : nullptr;
}

void* fsgg_dataset_stream(const fsgg_dataset* h) {
  return h ? static_cast<void*>(h->ds.stream) : nullptr;
}

int fsgg_build_similarity_graph(fsgg_dataset* h, const fsgg_kernel* kernel,
                                const fsgg_config* cfg, fsgg_graph* out,
                                fsgg_report* report, fsgg_edge_estimate** estimates) {
  return guarded([&] {
    if (!out) throw fsgg::ConfigError("null output");
    build_device(h, kernel, cfg, report, estimates != nullptr);
    graph_to_host(h, out);
    if (estimates) {
      *estimates = host_copy<fsgg_edge_estimate>(h->graph->est, h->graph->m, h->ds.stream);
      FSGG_CUDA(cudaStreamSynchronize(h->ds.stream));
    }
  });
}

int fsgg_build_similarity_graph_device(fsgg_dataset* h, const fsgg_kernel* kernel,
                                       const fsgg_config* cfg,
                                       fsgg_device_graph* out, fsgg_report* report) {
  return guarded([&] {
    if (!out) throw fsgg::ConfigError("null output");
    build_device(h, kernel, cfg, report, false);
    to_device_graph(h, out);
  });
}

int fsgg_build_similarity_graph_into(fsgg_dataset* h, const fsgg_kernel* kernel,
                                     const fsgg_config* cfg, uint64_t capacity,
                                     uint32_t* v, double* w, uint64_t* row_ptr,
                                     double* degrees, uint64_t* num_edges,
                                     double* total_weight, fsgg_report* report) {
  return guarded([&] {
    if (!num_edges) throw fsgg::ConfigError("null output");
    fsgg::HostSink sink;
    sink.v = v;
    sink.w = w;
    sink.row_ptr = row_ptr;
    sink.degrees = degrees;
    sink.capacity = capacity;
    build_device(h, kernel, cfg, report, false, &sink);
    *num_edges = h->graph->m;
    if (total_weight) *total_weight = h->graph->total_weight;
  });
}

int fsgg_build_similarity_graph_host(const float* points, uint32_t n, uint32_t d,
                                     const fsgg_kernel* kernel, const fsgg_config* cfg,
                                     int device, fsgg_graph* out, fsgg_report* report) {
  fsgg_dataset* h = nullptr;
  int rc = fsgg_dataset_create(points, n, d, 0, device, &h);
  if (rc) return rc;
  rc = fsgg_build_similarity_graph(h, kernel, cfg, out, report, nullptr);
  fsgg_dataset_destroy(h);
  return rc;
}

int fsgg_device_graph_to_host(fsgg_dataset* h, fsgg_graph* out) {
  return guarded([&] {
    activate(h);
    if (!out) throw fsgg::ConfigError("null output");
    if (!h->graph) throw fsgg::ConfigError("no graph built on this dataset");
    graph_to_host(h, out);
  });
}

int fsgg_device_graph_copy(fsgg_dataset* h, uint32_t* u, uint32_t* v, double* w,
                           uint64_t* row_ptr, double* degrees) {
  return guarded([&] {
    activate(h);
    if (!h->graph) throw fsgg::ConfigError("no graph built on this dataset");
    const fsgg::GraphResult& g = *h->graph;
    cudaStream_t s = h->ds.stream;
    auto cp = [&](void* dst, const fsgg::DevBuf& src, size_t bytes) {
      if (dst && bytes)
        FSGG_CUDA(cudaMemcpyAsync(dst, src.as<void>(), bytes, cudaMemcpyDefault, s));
    };
    cp(u, g.u, g.m * 4);
    cp(v, g.v, g.m * 4);
    cp(w, g.w, g.m * 8);
    cp(row_ptr, g.row_ptr, (uint64_t(g.n) + 1) * 8);
    cp(degrees, g.degrees, uint64_t(g.n) * 8);
    FSGG_CUDA(cudaStreamSynchronize(s));
  });
}

void fsgg_graph_free(fsgg_graph* g) {
  if (!g) return;
  std::free(g->u);
  std::free(g->v);
  std::free(g->w);
  std::free(g->row_ptr);
  std::free(g->degrees);
  std::memset(g, 0, sizeof(*g));
}

void fsgg_free(void* p) { std::free(p); }

void fsgg_spectral_options_init(fsgg_spectral_options* o) {
  if (!o) return;
  const fsgg::EigenOpts e;
  const fsgg::KmeansOpts k;
  o->eigen.tol = e.tol;
  o->eigen.max_matvecs = e.max_matvecs;
  o->eigen.max_basis = e.max_basis;
  o->eigen.seed = e.seed;
  o->kmeans.restarts = k.restarts;
  o->kmeans.max_iters = k.max_iters;
  o->kmeans.rel_tol = k.rel_tol;
  o->kmeans.seed = k.seed;
}

int fsgg_smallest_eigenpairs(fsgg_dataset* h, uint32_t q, const fsgg_eigen_options* opts,
                             double* values, double* vectors, double* residuals,
                             uint64_t* matvecs) {
  return guarded([&] {
    const fsgg::SpectralGraphView v = handle_graph_view(h);
    eigenpairs_out(v, h->ds.stream, q, opts, values, vectors, residuals, matvecs);
  });
}

int fsgg_spectral_cluster(fsgg_dataset* h, uint32_t k, uint64_t seed,
                          const fsgg_spectral_options* opts, uint32_t* labels,
                          fsgg_spectral_report* report) {
  return guarded([&] {
    const fsgg::SpectralGraphView v = handle_graph_view(h);
    spectral_out(v, h->ds.stream, k, seed, opts, labels, report);
  });
}

int fsgg_spectral_cluster_graph(const fsgg_graph* g, int device, uint32_t k, uint64_t seed,
                                const fsgg_spectral_options* opts, uint32_t* labels,
                                fsgg_spectral_report* report) {
  return guarded([&] {
    UploadedGraph up(g, device);
    spectral_out(up.view, up.s, k, seed, opts, labels, report);
  });
}

int fsgg_smallest_eigenpairs_graph(const fsgg_graph* g, int device, uint32_t q,
                                   const fsgg_eigen_options* opts, double* values,
                                   double* vectors, double* residuals, uint64_t* matvecs) {
  return guarded([&] {
    UploadedGraph up(g, device);
    eigenpairs_out(up.view, up.s, q, opts, values, vectors, residuals, matvecs);
  });
}

int fsgg_kmeans(const double* points, uint32_t n, uint32_t dim, uint32_t k,
                const fsgg_kmeans_options* opts, int device, uint32_t* labels, double* cost,
                uint32_t* iterations) {
  return guarded([&] {
    if (!points || !labels) throw fsgg::ConfigError("null argument");
    if (n == 0 || dim == 0) throw fsgg::ConfigError("empty k-means input");
    require_device(device);
    FSGG_CUDA(cudaSetDevice(device));
    cudaStream_t s = nullptr;
    FSGG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    } guard{s};
    fsgg::DevBuf pts(size_t(n) * dim * 8, s);
    FSGG_CUDA(cudaMemcpyAsync(pts.as<void>(), points, size_t(n) * dim * 8,
                              cudaMemcpyHostToDevice, s));
    fsgg::SpectralStats st;
    fsgg::kmeans_dev(pts.as<double>(), n, dim, k, kmeans_opts(opts), s, labels, cost,
                     iterations, st);
    pts.release();
  });
}

int fsgg_graph_save_text(const char* path, uint32_t n, uint64_t num_edges, const uint32_t* u,
                         const uint32_t* v, const double* w, uint32_t threads) {
  return guarded([&] { fsgg::graph_save_text(path, n, num_edges, u, v, w, threads); });
}

int fsgg_graph_load_text(const char* path, uint32_t threads, fsgg_graph* out) {
  return guarded([&] { fsgg::graph_load_text(path, threads, out); });
}

int fsgg_graph_save_csr(const char* path, const fsgg_graph* g) {
  return guarded([&] { fsgg::graph_save_csr(path, g); });
}

int fsgg_csv_load(const char* path, uint32_t threads, double** points, uint32_t* n,
                  uint32_t* d, uint32_t** labels) {
  return guarded([&] { fsgg::csv_load(path, threads, points, n, d, labels); });
}

int fsgg_csv_save(const char* path, const double* points, uint32_t n, uint32_t d,
                  const uint32_t* labels, uint32_t threads) {
  return guarded([&] { fsgg::csv_save(path, points, n, d, labels, threads); });
}

int fsgg_graph_load_csr(const char* path, fsgg_graph* out) {
  return guarded([&] { fsgg::graph_load_csr(path, out); });
}

void fsgg_sample_options_init(fsgg_sample_options* opt) {
  if (!opt) return;
  opt->rng_mode = FSGG_RNG_REFERENCE;
  opt->dense_kde = 0;
  opt->record_sums = 0;
  opt->walks = 1;
  opt->kde_backend = FSGG_KDE_EXACT;
  opt->epsilon = 0.0;
}

int fsgg_sample_neighbors_counted(fsgg_dataset* h, const fsgg_kernel* kernel,
                                  const uint32_t* queries, size_t num_queries,
                                  uint32_t rounds, uint64_t seed, int rng_mode,
                                  int dense_kde, uint32_t** triples, size_t* count,
                                  fsgg_sample_diag* diag) {
  fsgg_sample_options opt;
  fsgg_sample_options_init(&opt);
  opt.rng_mode = rng_mode;
  opt.dense_kde = dense_kde;
  fsgg_sample_report rep;
  const int rc = fsgg_sample_neighbors_counted_ex(h, kernel, queries, num_queries, rounds, seed,
                                                  &opt, triples, count, diag ? &rep : nullptr);
  if (rc == FSGG_OK && diag) *diag = rep.diag;
  return rc;
}

int fsgg_sample_neighbors_counted_ex(fsgg_dataset* h, const fsgg_kernel* kernel,
                                     const uint32_t* queries, size_t num_queries,
                                     uint32_t rounds, uint64_t seed,
                                     const fsgg_sample_options* opt, uint32_t** triples,
                                     size_t* count, fsgg_sample_report* rep) {
  fsgg_sample_options defaults;
  fsgg_sample_options_init(&defaults);
  if (!opt) opt = &defaults;
  const int rng_mode = opt->rng_mode;
  const int dense_kde = opt->dense_kde;
  if (rep) std::memset(rep, 0, sizeof(*rep));
  return guarded([&] {
    activate(h);
    validate_kernel(kernel);
    if (!triples || !count || (num_queries && !queries)) throw fsgg::ConfigError("null argument");
    if (rounds == 0) throw fsgg::ConfigError("need at least one sampling round");  // sampler.cpp:85
    fsgg::Dataset& ds = h->ds;
    for (size_t i = 0; i < num_queries; ++i)
      if (queries[i] >= ds.n) throw fsgg::ConfigError("query index out of range");  // :86-87
    // :89-106 merge duplicates, ascending query order
    std::vector<uint32_t> q(queries, queries + num_queries);
    std::sort(q.begin(), q.end());
    fsgg::SampleRequest req;
    for (size_t i = 0; i < q.size();) {
      size_t j = i;
      while (j < q.size() && q[j] == q[i]) ++j;
      uint64_t t = uint64_t(j - i) * rounds;
      if (t > 0xffffffffull) throw fsgg::ConfigError("total rounds per query exceeds 2^32");
      req.queries.push_back(q[i]);
      req.tickets.push_back(static_cast<uint32_t>(t));
      i = j;
    }
    if (rng_mode != FSGG_RNG_REFERENCE && rng_mode != FSGG_RNG_PHILOX)
      throw fsgg::ConfigError("unknown rng_mode");
    req.seed = seed;
    req.rng_mode = rng_mode;
    req.prune = dense_kde ? 0 : 1;
    req.walk = opt->walks != 0;
    req.record_sums = opt->record_sums != 0;
    const Backend be = resolve_backend(opt->kde_backend, opt->epsilon, 0, kernel->family, ds.n,
                                       ds.d);
    if (be.fast && req.prune) {
      req.fast_epsilon = be.eps;
      req.verify_ties = false;
    }
    std::vector<uint32_t> host;
    if (!h->sample) h->sample = std::make_unique<fsgg::SampleResult>();
    fsgg::SampleResult& res = *h->sample;
    res.entries_per_level.clear();
    res.tickets_per_level.clear();
    res.degenerate_draws = 0;
    if (!req.queries.empty()) {
      const fsgg::KernelSpec ks = fsgg::make_kernel_spec(kernel->family, kernel->sigma);
      fsgg::sample_counted(ds, ks, req, res);
      fsgg::sampled_triples_to_host(ds, res, host);
    }
    *count = host.size() / 3;
    *triples = static_cast<uint32_t*>(std::malloc(std::max<size_t>(host.size(), 1) * 4));
    if (!*triples) throw std::bad_alloc();
    std::memcpy(*triples, host.data(), host.size() * 4);
    if (rep) {
      fsgg_sample_diag* diag = &rep->diag;
      diag->nlevels = static_cast<uint32_t>(std::min<size_t>(res.entries_per_level.size(), 64));
      for (uint32_t i = 0; i < diag->nlevels; ++i) {
        diag->entries_per_level[i] = res.entries_per_level[i];
        diag->tickets_per_level[i] = res.tickets_per_level[i];
      }
      diag->degenerate_draws = res.degenerate_draws;
      rep->kernel_evals = res.kde.evals;
      rep->kernel_evals_performed = res.kde.performed;
      rep->root_evals_performed = res.kde.root_performed;
      rep->tie_verified = res.tie_verified;
      if (req.record_sums && !req.queries.empty()) {
        static_assert(sizeof(fsgg_entry_record) == sizeof(fsgg::EntryRecord), "record layout");
        const size_t m = res.records.size();
        rep->records = static_cast<fsgg_entry_record*>(
            std::malloc(std::max<size_t>(m, 1) * sizeof(fsgg_entry_record)));
        if (!rep->records) throw std::bad_alloc();
        std::memcpy(rep->records, res.records.data(), m * sizeof(fsgg_entry_record));
        rep->num_records = m;
      }
    }
  });
}

int fsgg_kde_eval(fsgg_dataset* h, const fsgg_kernel* kernel, uint32_t first,
                  uint32_t last, const uint32_t* targets, size_t m, double* out) {
  return guarded([&] {
    activate(h);
    validate_kernel(kernel);
    fsgg::Dataset& ds = h->ds;
    if (first > last || last > ds.n)  // kde.cpp:29-35
      throw fsgg::ConfigError("invalid source index range [" + std::to_string(first) + ", " +
                              std::to_string(last) + ") for n = " + std::to_string(ds.n));
    if (m && (!targets || !out)) throw fsgg::ConfigError("null argument");
    for (size_t i = 0; i < m; ++i)
      if (targets[i] >= ds.n) throw fsgg::ConfigError("target index out of range");
    if (m > 0xffffffffull) throw fsgg::ConfigError("too many targets");
    if (m == 0) return;
    cudaStream_t s = ds.stream;
    fsgg::DevBuf dt(m * 4, s), dout(m * 8, s);
    FSGG_CUDA(cudaMemcpyAsync(dt.as<void>(), targets, m * 4, cudaMemcpyHostToDevice, s));
    const fsgg::KernelSpec ks = fsgg::make_kernel_spec(kernel->family, kernel->sigma);
    fsgg::kde_range(ds, ks, first, last, dt.as<uint32_t>(), uint32_t(m), dout.as<double>());
    FSGG_CUDA(cudaMemcpyAsync(out, dout.as<void>(), m * 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
  });
}

// ---- device generators (datasets_dev.cu); argument checks as the host
// generators (datasets.cpp), which follow proj/src/datasets.cpp:33-80

int fsgg_make_moons_device(uint32_t n, double noise, uint64_t seed, int device,
                           double* points64, float* points32, uint32_t* labels) {
  return on_device(device, n >= 2 && noise >= 0.0, [&] {
    fsgg::make_moons_device(n, noise, seed, points64, points32, labels);
  });
}

int fsgg_make_blobs_device(uint32_t n, const double* centers, uint32_t k, uint32_t d,
                           double stddev, uint64_t seed, int device, double* points64,
                           float* points32, uint32_t* labels) {
  return on_device(device, k > 0 && n >= k && stddev >= 0.0 && d > 0 && centers, [&] {
    fsgg::make_blobs_device(n, centers, k, d, stddev, seed, points64, points32, labels);
  });
}

int fsgg_make_image_features_device(uint32_t height, uint32_t width, uint32_t regions,
                                    double noise, uint64_t seed, int device,
                                    double* points64, float* points32, uint32_t* labels) {
  return on_device(device,
                   height > 0 && width > 0 && regions > 0 && noise >= 0.0 &&
                       uint64_t(height) * width <= 0xffffffffull,
                   [&] {
                     fsgg::make_image_features_device(height, width, regions, noise, seed,
                                                      points64, points32, labels);
                   });
}

int fsgg_make_gmm_device(uint32_t n, uint32_t d, uint32_t k, double stddev, uint64_t seed,
                         int device, double* points64, float* points32, uint32_t* labels) {
  return on_device(device, k > 0 && n >= k && d > 0 && stddev >= 0.0, [&] {
    fsgg::make_gmm_device(n, d, k, stddev, seed, points64, points32, labels);
  });
}

int fsgg_sample_shard(fsgg_dataset* h, const fsgg_kernel* kernel, const fsgg_config* cfgp,
                      fsgg_shard* out, fsgg_report* report) {
  return guarded([&] {
    activate(h);
    validate_kernel(kernel);
    if (!out) throw fsgg::ConfigError("null output");
    fsgg_config cfg = cfgp ? *cfgp : default_config();
    fsgg::Dataset& ds = h->ds;
    if (ds.n < 2) throw fsgg::ConfigError("similarity graph needs n >= 2");
    uint32_t qb = cfg.query_begin, qe = cfg.query_end;
    if (qb == 0 && qe == 0) qe = ds.n;
    if (qb > qe || qe > ds.n) throw fsgg::ConfigError("invalid query shard");
    BuildOut bo;
    bo.L = rounds_for(cfg, ds.n);
    double t0 = now();
    if (!h->shard) h->shard = std::make_unique<fsgg::SampleResult>();
    uint64_t npairs = 0;
    if (qe > qb) {
      run_descent(h, kernel, cfg, bo.L, qb, qe, *h->shard, h->shard_keys, &npairs, bo);
    } else {
      h->shard->groot.ensure(8, ds.stream);
      h->shard_keys.ensure(8, ds.stream);
      h->shard->nq = 0;
    }
    std::memset(out, 0, sizeof(*out));
    out->query_begin = qb;
    out->query_end = qe;
    out->rounds = bo.L;
    out->num_pairs = npairs;
    h->shard_npairs = npairs;
    out->pairs = h->shard_keys.as<uint64_t>();
    out->g_full = h->shard->groot.as<double>();
    out->sampled_pairs = bo.sampled;
    out->self_pairs = bo.self;
    out->degenerate_draws = bo.degenerate;
    if (report) finish_report(report, ds, bo, nullptr, now() - t0);
  });
}

int fsgg_sample_shard_routed(fsgg_dataset* h, const fsgg_kernel* kernel,
                             const fsgg_config* cfgp, uint32_t world, const uint32_t* bounds,
                             uint64_t* counts, fsgg_shard* out, fsgg_report* report) {
  return guarded([&] {
    activate(h);
    validate_kernel(kernel);
    if (!out || !bounds || !counts) throw fsgg::ConfigError("null argument");
    if (world == 0 || world > 64) throw fsgg::ConfigError("world size must be 1..64");
    fsgg_config cfg = cfgp ? *cfgp : default_config();
    fsgg::Dataset& ds = h->ds;
    if (ds.n < 2) throw fsgg::ConfigError("similarity graph needs n >= 2");
    if (bounds[0] != 0 || bounds[world] != ds.n)
      throw fsgg::ConfigError("shard bounds must cover [0, n)");
    for (uint32_t r = 0; r < world; ++r)
      if (bounds[r] > bounds[r + 1]) throw fsgg::ConfigError("shard bounds must be sorted");
    uint32_t qb = cfg.query_begin, qe = cfg.query_end;
    if (qb == 0 && qe == 0) qe = ds.n;
    if (qb > qe || qe > ds.n) throw fsgg::ConfigError("invalid query shard");
    BuildOut bo;
    bo.L = rounds_for(cfg, ds.n);
    double t0 = now();
    if (!h->shard) h->shard = std::make_unique<fsgg::SampleResult>();
    uint64_t npairs = 0;
    for (uint32_t r = 0; r < world; ++r) counts[r] = 0;
    if (qe > qb) {
      run_descent(h, kernel, cfg, bo.L, qb, qe, *h->shard, h->shard_keys, &npairs, bo, world,
                  bounds, counts);
    } else {
      h->shard->groot.ensure(8, ds.stream);
      h->shard_keys.ensure(8, ds.stream);
      h->shard->nq = 0;
    }
    std::memset(out, 0, sizeof(*out));
    out->query_begin = qb;
    out->query_end = qe;
    out->rounds = bo.L;
    out->num_pairs = npairs;
    h->shard_npairs = npairs;
    out->pairs = h->shard_keys.as<uint64_t>();
    out->g_full = h->shard->groot.as<double>();
    out->sampled_pairs = bo.sampled;
    out->self_pairs = bo.self;
    out->degenerate_draws = bo.degenerate;
    if (report) finish_report(report, ds, bo, nullptr, now() - t0);
  });
}

int fsgg_shard_bounds(fsgg_dataset* h, const fsgg_kernel* kernel, uint32_t world,
                      uint32_t* bounds) {
  return guarded([&] {
    activate(h);
    if (world == 0 || !bounds) throw fsgg::ConfigError("invalid world size");
    fsgg::Dataset& ds = h->ds;
    if (!ds.tree_valid) fsgg::build_tree(ds);
    if (kernel) {
      validate_kernel(kernel);
      const fsgg::KernelSpec ks = fsgg::make_kernel_spec(kernel->family, kernel->sigma);
      fsgg::sym_shard_bounds(ds, &ks, world, bounds);
    } else {
      fsgg::sym_shard_bounds(ds, nullptr, world, bounds);
    }
  });
}

int fsgg_shard_root_prepare(fsgg_dataset* h, const fsgg_kernel* kernel, const fsgg_config* cfgp,
                            uint64_t* num_records) {
  return guarded([&] {
    activate(h);
    validate_kernel(kernel);
    if (!num_records) throw fsgg::ConfigError("null output");
    *num_records = 0;
    h->root_records = 0;
    fsgg_config cfg = cfgp ? *cfgp : default_config();
    fsgg::Dataset& ds = h->ds;
    uint32_t qb = cfg.query_begin, qe = cfg.query_end;
    if (qb == 0 && qe == 0) qe = ds.n;
    if (qb > qe || qe > ds.n) throw fsgg::ConfigError("invalid query shard");
    const char* e = std::getenv("FSGG_SYM");
    if (cfg.dense_kde || (e && std::atoi(e) == 0)) return;  // no symmetric root
    const fsgg::KernelSpec ks = fsgg::make_kernel_spec(kernel->family, kernel->sigma);
    ds.tree_valid = false;
    ds.tc_ready = false;
    ds.tie_xn_ready = false;
    fsgg::build_tree(ds);
    h->tree_fresh = true;  // the shard's descent reuses this table
    {  // the descent's pruning threshold (exact or fast backend)
      const Backend be = resolve_backend(cfg.kde_backend, cfg.epsilon, cfg.log_base,
                                         kernel->family, ds.n, ds.d);
      fsgg::SampleRequest r;
      r.fast_epsilon = be.fast ? be.eps : 0.0;
      if (!ds.kde_ws) ds.kde_ws = std::make_unique<fsgg::KdeWorkspace>();
      ds.kde_ws->prune_bits = fsgg::prune_bits_for(r, ds.tree);
    }
    uint32_t n = 0;
    const uint32_t* recs = nullptr;
    fsgg::sym_shard_prepare(ds, ks, qb, qe, &n, &recs);
    h->root_records = n;
    *num_records = n;
  });
}

int fsgg_shard_root_export(fsgg_dataset* h, uint32_t* records_device) {
  return guarded([&] {
    activate(h);
    if (h->root_records == 0) return;
    if (!records_device) throw fsgg::ConfigError("null records");
    fsgg::Dataset& ds = h->ds;
    FSGG_CUDA(cudaMemcpyAsync(records_device, ds.buf("sym.rec", 4).as<void>(),
                              size_t(h->root_records) * fsgg::kSymRecordWords * 4,
                              cudaMemcpyDeviceToDevice, ds.stream));
    FSGG_CUDA(cudaStreamSynchronize(ds.stream));
  });
}

int fsgg_shard_root_receive(fsgg_dataset* h, const uint32_t* records, uint64_t num_records) {
  return guarded([&] {
    activate(h);
    if (num_records && !records) throw fsgg::ConfigError("null records");
    if (num_records > 0xffffffffull) throw fsgg::ConfigError("too many records");
    fsgg::sym_shard_receive(h->ds, records, uint32_t(num_records));
    FSGG_CUDA(cudaStreamSynchronize(h->ds.stream));
  });
}

int fsgg_shard_export(fsgg_dataset* h, uint64_t* pairs_device, double* g_full_device) {
  return guarded([&] {
    activate(h);
    if (!h->shard) throw fsgg::ConfigError("no shard sampled on this dataset");
    cudaStream_t s = h->ds.stream;
    const fsgg::SampleResult& r = *h->shard;
    if (pairs_device && h->shard_npairs)
      FSGG_CUDA(cudaMemcpyAsync(pairs_device, h->shard_keys.as<void>(), h->shard_npairs * 8,
                                cudaMemcpyDeviceToDevice, s));
    if (g_full_device && r.nq)
      FSGG_CUDA(cudaMemcpyAsync(g_full_device, r.groot.as<void>(), size_t(r.nq) * 8,
                                cudaMemcpyDeviceToDevice, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
  });
}

int fsgg_finish_graph(fsgg_dataset* h, const fsgg_kernel* kernel, uint32_t rounds,
                      const double* g_full_device, const uint64_t* pairs_device,
                      uint64_t num_pairs, fsgg_device_graph* out, fsgg_report* report) {
  return guarded([&] {
    activate(h);
    validate_kernel(kernel);
    if (!out || !g_full_device || (num_pairs && !pairs_device))
      throw fsgg::ConfigError("null argument");
    if (rounds == 0) throw fsgg::ConfigError("rounds must be positive");
    double t0 = now();
    const fsgg::KernelSpec ks = fsgg::make_kernel_spec(kernel->family, kernel->sigma);
    if (!h->graph) h->graph = std::make_unique<fsgg::GraphResult>();
    fsgg::finish_graph(h->ds, ks, rounds, g_full_device, pairs_device, num_pairs, false,
                       false, *h->graph);
    to_device_graph(h, out);
    if (report) {
      BuildOut bo;
      bo.L = rounds;
      bo.t_graph = now() - t0;
      finish_report(report, h->ds, bo, h->graph.get(), bo.t_graph);
    }
  });
}

int fsgg_rows_transposed(fsgg_dataset* h, uint32_t* v_device, double* w_device) {
  return guarded([&] {
    activate(h);
    if (!h->graph) throw fsgg::ConfigError("no graph on this handle: finish one first");
    if (h->graph->m && (!v_device || !w_device)) throw fsgg::ConfigError("null argument");
    fsgg::rows_transposed(h->ds, *h->graph, v_device, w_device);
  });
}

int fsgg_rows_row_ptr(fsgg_dataset* h, uint32_t row_begin, uint32_t row_end,
                      uint64_t edge_offset, uint64_t* row_ptr_device) {
  return guarded([&] {
    activate(h);
    if (!h->graph) throw fsgg::ConfigError("no graph on this handle: finish one first");
    if (row_begin > row_end || row_end > h->ds.n) throw fsgg::ConfigError("invalid row range");
    if (row_end > row_begin && !row_ptr_device) throw fsgg::ConfigError("null argument");
    fsgg::rows_row_ptr(h->ds, *h->graph, row_begin, row_end, edge_offset, row_ptr_device);
  });
}

int fsgg_rows_degrees(fsgg_dataset* h, const uint32_t* lower_v_device,
                      const double* lower_w_device, uint64_t num_lower, uint32_t row_begin,
                      uint32_t row_end, double* degrees_device) {
  return guarded([&] {
    activate(h);
    if (!h->graph) throw fsgg::ConfigError("no graph on this handle: finish one first");
    if (row_begin > row_end || row_end > h->ds.n) throw fsgg::ConfigError("invalid row range");
    if ((num_lower && (!lower_v_device || !lower_w_device)) ||
        (row_end > row_begin && !degrees_device))
      throw fsgg::ConfigError("null argument");
    fsgg::rows_degrees(h->ds, *h->graph, lower_v_device, lower_w_device, num_lower, row_begin,
                       row_end, degrees_device);
  });
}

}  // extern "C"
