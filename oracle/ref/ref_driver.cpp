// TEST INFRASTRUCTURE ONLY — not product code.
//
// A thin extern "C" harness around the UNMODIFIED reference hot-path sources
// (compiled in place from /root/reference/proj by oracle/Makefile into
// oracle/_ref/libfsgref.so). It lets the pytest suite, the golden-fixture
// generator and bench.py's CPU-baseline leg call the reference's own
// implementation through ctypes:
//   * fsg::build_similarity_graph   proj/src/sparsifier.cpp:51-142
//   * fsg::sample_neighbors_counted proj/src/sampler.cpp:77-247
//   * fsg::KdeEstimator::eval       proj/include/fsg/kde.hpp:54-58
//   * fsg::make_moons / make_blobs  proj/src/datasets.cpp:32-124
// plus a recording KdeEstimator (the plugin seam, proj/include/fsg/kde.hpp:49)
// that captures every (range, query) -> child sum the sampler asks for.
//
// Nothing here re-implements the algorithm; every number comes from the
// reference's code. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs load this library.

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "fsg/common.hpp"
#include "fsg/dataset.hpp"
#include "fsg/graph.hpp"
#include "fsg/datasets.hpp"
#include "fsg/kde.hpp"
#include "fsg/kernel.hpp"
#include "fsg/sampler.hpp"
#include "fsg/sparsifier.hpp"
#include "fsg/spectral.hpp"

// proj/src/spectral.cpp is compiled in place against oracle/ref/eigen_shim
// (a stand-in for the absent Eigen headers), so the spectral pipeline below
// is the reference's own code.

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const fsg::Error& e) {
    g_error = e.what();
    return e.exit_code();
  } catch (const std::exception& e) {
    g_error = e.what();
    return 1;
  }
}

template <class T>
T* dup_vector(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * (v.size() ? v.size() : 1)));
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

fsg::KernelFamily family_of(int f) {
  switch (f) {
    case 0: return fsg::KernelFamily::gaussian;
    case 1: return fsg::KernelFamily::exponential;
    case 2: return fsg::KernelFamily::laplacian;
  }
  throw fsg::InvalidConfig("unknown kernel family id");
}

fsg::KdeBackend backend_of(int b) {
  switch (b) {
    case 0: return fsg::KdeBackend::exact;
    case 1: return fsg::KdeBackend::fast;
    case 2: return fsg::KdeBackend::autoselect;
  }
  throw fsg::InvalidConfig("unknown backend id");
}

// Records every call the sampler makes through the plugin seam.
class RecordingEstimator final : public fsg::KdeEstimator {
public:
  RecordingEstimator(const fsg::KdeEstimator& inner)
      : fsg::KdeEstimator(inner.data(), inner.kernel(), "recording",
                          inner.sum_floor(), false),
        inner_(inner) {}
  void eval(fsg::IndexRange range, std::span<const uint32_t> targets,
            std::span<double> out) const override {
    inner_.eval(range, targets, out);
    std::lock_guard<std::mutex> lock(mu_);
    for (size_t t = 0; t < targets.size(); ++t) {
      first_.push_back(range.first);
      last_.push_back(range.last);
      query_.push_back(targets[t]);
      sum_.push_back(out[t]);
    }
  }
  void eval_points(fsg::IndexRange range, const double* points, uint32_t m,
                   std::span<double> out) const override {
    inner_.eval_points(range, points, m, out);
  }
  double epsilon() const override { return inner_.epsilon(); }
  size_t memory_bytes() const override { return inner_.memory_bytes(); }

  const fsg::KdeEstimator& inner_;
  mutable std::mutex mu_;
  mutable std::vector<uint32_t> first_, last_, query_;
  mutable std::vector<double> sum_;
};

struct EstimatorHandle {
  std::unique_ptr<fsg::Dataset> ds;
  std::unique_ptr<fsg::Kernel> kernel;
  std::unique_ptr<fsg::KdeEstimator> est;
};

}  // namespace

extern "C" {

const char* fsgref_last_error(void) { return g_error.c_str(); }
void fsgref_free(void* p) { std::free(p); }
void fsgref_set_threads(unsigned n) { fsg::set_worker_count(n); }
unsigned fsgref_worker_count(void) { return fsg::worker_count(); }

// fsg::load_csv / save_csv (proj/src/dataset.cpp:54-130), called as is.
int fsgref_load_csv(const char* path, double** pts, uint32_t* n, uint32_t* d,
                    uint32_t** labels) {
  *pts = nullptr;
  *labels = nullptr;
  return guarded([&] {
    auto cd = fsg::load_csv(path);
    *n = cd.data.size();
    *d = cd.data.dim();
    *pts = dup_vector(cd.data.raw());
    if (cd.labels) *labels = dup_vector(*cd.labels);
  });
}

int fsgref_save_csv(const char* path, const double* pts, uint32_t n, uint32_t d,
                    const uint32_t* labels) {
  return guarded([&] {
    fsg::Dataset ds(std::vector<double>(pts, pts + size_t(n) * d), n, d);
    std::vector<uint32_t> lab;
    if (labels) lab.assign(labels, labels + n);
    fsg::save_csv(path, ds, labels ? &lab : nullptr);
  });
}

int fsgref_make_moons(uint32_t n, double noise, uint64_t seed, double* pts,
                      uint32_t* labels) {
  return guarded([&] {
    auto ld = fsg::make_moons(n, noise, seed);
    std::memcpy(pts, ld.data.raw().data(), sizeof(double) * ld.data.raw().size());
    if (labels)
      std::memcpy(labels, ld.labels.labels.data(), sizeof(uint32_t) * n);
  });
}

int fsgref_make_blobs(uint32_t n, const double* centers, uint32_t k,
                      uint32_t d, double stddev, uint64_t seed, double* pts,
                      uint32_t* labels) {
  return guarded([&] {
    std::vector<std::vector<double>> c(k, std::vector<double>(d));
    for (uint32_t i = 0; i < k; ++i)
      for (uint32_t a = 0; a < d; ++a) c[i][a] = centers[size_t(i) * d + a];
    auto ld = fsg::make_blobs(n, c, stddev, seed);
    std::memcpy(pts, ld.data.raw().data(), sizeof(double) * ld.data.raw().size());
    if (labels)
      std::memcpy(labels, ld.labels.labels.data(), sizeof(uint32_t) * n);
  });
}

double fsgref_default_epsilon(uint32_t n, int log_base) {
  return fsg::default_epsilon(n, log_base ? fsg::LogBase::natural
                                          : fsg::LogBase::two);
}

int fsgref_rounds_for(uint32_t n, double C, double lambda, uint32_t rounds,
                      int log_base, uint32_t* out) {
  return guarded([&] {
    fsg::SparsifierConfig cfg;
    cfg.C = C;
    cfg.lambda_k1_estimate = lambda;
    cfg.rounds = rounds;
    cfg.log_base = log_base ? fsg::LogBase::natural : fsg::LogBase::two;
    *out = cfg.rounds_for(n);
  });
}

int fsgref_kernel_eval(int family, double sigma, const double* x,
                       const double* y, uint32_t d, double* out) {
  return guarded([&] {
    fsg::Kernel k(family_of(family), sigma);
    *out = k(x, y, d);
  });
}

void* fsgref_estimator_create(const double* pts, uint32_t n, uint32_t d,
                              int family, double sigma, int backend,
                              double epsilon) {
  EstimatorHandle* h = nullptr;
  int rc = guarded([&] {
    auto hh = std::make_unique<EstimatorHandle>();
    hh->ds = std::make_unique<fsg::Dataset>(
        std::vector<double>(pts, pts + size_t(n) * d), n, d);
    hh->kernel = std::make_unique<fsg::Kernel>(family_of(family), sigma);
    fsg::KdeConfig cfg;
    cfg.backend = backend_of(backend);
    cfg.epsilon = epsilon;
    hh->est = fsg::make_estimator(*hh->ds, *hh->kernel, cfg);
    h = hh.release();
  });
  return rc == 0 ? h : nullptr;
}

void fsgref_estimator_destroy(void* h) {
  delete static_cast<EstimatorHandle*>(h);
}

const char* fsgref_estimator_backend(void* h) {
  return static_cast<EstimatorHandle*>(h)->est->backend_name();
}

double fsgref_estimator_epsilon(void* h) {
  return static_cast<EstimatorHandle*>(h)->est->epsilon();
}

int fsgref_kde_eval(void* h, uint32_t first, uint32_t last,
                    const uint32_t* targets, size_t m, double* out) {
  return guarded([&] {
    auto* hh = static_cast<EstimatorHandle*>(h);
    hh->est->eval({first, last}, std::span<const uint32_t>(targets, m),
                  std::span<double>(out, m));
  });
}

// sample_neighbors_counted through the handle's estimator. When `record` is
// non-zero the estimator is wrapped in RecordingEstimator and the captured
// per-node sums are returned (rec_* arrays, rec_count rows).
int fsgref_sample_counted(void* h, const uint32_t* queries, size_t nq,
                          uint32_t rounds, uint64_t seed,
                          uint32_t inline_range, int record,
                          uint32_t** triples, size_t* count,
                          uint64_t* entries_per_level,
                          uint64_t* tickets_per_level, uint32_t* nlevels,
                          uint64_t* degenerate, uint32_t** rec_first,
                          uint32_t** rec_last, uint32_t** rec_query,
                          double** rec_sum, size_t* rec_count) {
  return guarded([&] {
    auto* hh = static_cast<EstimatorHandle*>(h);
    fsg::SampleDiagnostics diag;
    fsg::SamplerOptions opts;
    opts.inline_range = inline_range;
    std::unique_ptr<RecordingEstimator> rec;
    const fsg::KdeEstimator* est = hh->est.get();
    if (record) {
      rec = std::make_unique<RecordingEstimator>(*hh->est);
      est = rec.get();
    }
    auto out = fsg::sample_neighbors_counted(
        std::span<const uint32_t>(queries, nq), *est, rounds, seed, &diag,
        opts);
    std::vector<uint32_t> flat(out.size() * 3);
    for (size_t i = 0; i < out.size(); ++i) {
      flat[3 * i] = out[i].query;
      flat[3 * i + 1] = out[i].source;
      flat[3 * i + 2] = out[i].count;
    }
    *triples = dup_vector(flat);
    *count = out.size();
    uint32_t L = static_cast<uint32_t>(diag.entries_per_level.size());
    if (L > 64) L = 64;
    for (uint32_t i = 0; i < L; ++i) {
      if (entries_per_level) entries_per_level[i] = diag.entries_per_level[i];
      if (tickets_per_level) tickets_per_level[i] = diag.tickets_per_level[i];
    }
    if (nlevels) *nlevels = L;
    if (degenerate) *degenerate = diag.degenerate_draws;
    if (record) {
      *rec_first = dup_vector(rec->first_);
      *rec_last = dup_vector(rec->last_);
      *rec_query = dup_vector(rec->query_);
      *rec_sum = dup_vector(rec->sum_);
      *rec_count = rec->sum_.size();
    } else if (rec_count) {
      *rec_count = 0;
    }
  });
}

// fsg::build_similarity_graph with the reference's own SparsifierConfig.
// report[] receives, in order: n, rounds, epsilon, sampled_pairs,
// self_pairs_discarded, underflow_edges_discarded, edge_count,
// degenerate_draws, estimator_build_seconds, sampling_seconds,
// degree_kde_seconds, weighting_seconds, total_seconds, total_weight.
// estimates (8 doubles per edge): i, j, k_ij, g_i, g_j, p_i, p_j, p_hat.
int fsgref_build_graph(const double* pts, uint32_t n, uint32_t d, int family,
                       double sigma, uint32_t rounds, uint64_t seed,
                       int backend, double C, double lambda, double epsilon,
                       int log_base, size_t* m, uint32_t** u, uint32_t** v,
                       double** w, double** degrees, double** estimates,
                       double* report, char* backend_name, size_t name_cap) {
  return guarded([&] {
    fsg::Dataset ds(std::vector<double>(pts, pts + size_t(n) * d), n, d);
    fsg::Kernel kernel(family_of(family), sigma);
    fsg::SparsifierConfig cfg;
    cfg.C = C;
    cfg.lambda_k1_estimate = lambda;
    cfg.rounds = rounds;
    cfg.epsilon = epsilon;
    cfg.log_base = log_base ? fsg::LogBase::natural : fsg::LogBase::two;
    cfg.seed = seed;
    cfg.kde.backend = backend_of(backend);
    fsg::BuildReport rep;
    std::vector<fsg::EdgeEstimate> est;
    fsg::WeightedGraph g = fsg::build_similarity_graph(
        ds, kernel, cfg, &rep, estimates ? &est : nullptr);
    const auto& e = g.edges();
    std::vector<uint32_t> uu(e.size()), vv(e.size());
    std::vector<double> ww(e.size());
    for (size_t i = 0; i < e.size(); ++i) {
      uu[i] = e[i].u;
      vv[i] = e[i].v;
      ww[i] = e[i].w;
    }
    *m = e.size();
    *u = dup_vector(uu);
    *v = dup_vector(vv);
    *w = dup_vector(ww);
    if (degrees) *degrees = dup_vector(g.degrees());
    if (estimates) {
      std::vector<double> flat(est.size() * 8);
      for (size_t i = 0; i < est.size(); ++i) {
        const auto& x = est[i];
        double row[8] = {double(x.i), double(x.j), x.k_ij, x.g_i,
                         x.g_j,       x.p_hat_i_j, x.p_hat_j_i, x.p_hat};
        std::memcpy(&flat[8 * i], row, sizeof(row));
      }
      *estimates = dup_vector(flat);
    }
    if (report) {
      double r[14] = {double(rep.n),
                      double(rep.rounds),
                      rep.epsilon,
                      double(rep.sampled_pairs),
                      double(rep.self_pairs_discarded),
                      double(rep.underflow_edges_discarded),
                      double(rep.edge_count),
                      double(rep.degenerate_draws),
                      rep.estimator_build_seconds,
                      rep.sampling_seconds,
                      rep.degree_kde_seconds,
                      rep.weighting_seconds,
                      rep.total_seconds,
                      g.total_weight()};
      std::memcpy(report, r, sizeof(r));
    }
    if (backend_name && name_cap) {
      std::strncpy(backend_name, rep.backend.c_str(), name_cap - 1);
      backend_name[name_cap - 1] = 0;
    }
  });
}

// fsg::save_edge_list on a graph adopted from sorted unique arrays
// (GraphBuilder::adopt_sorted_unique, proj/src/graph.cpp:40-54).
int fsgref_save_edge_list(const char* path, uint32_t n, size_t m, const uint32_t* u,
                          const uint32_t* v, const double* w) {
  return guarded([&] {
    std::vector<fsg::Edge> e(m);
    for (size_t i = 0; i < m; ++i) e[i] = {u[i], v[i], w[i]};
    fsg::GraphBuilder b(n);
    b.adopt_sorted_unique(std::move(e));
    fsg::save_edge_list(path, b.build());
  });
}

// fsg::load_edge_list: arrays, degrees and total weight of the read graph.
int fsgref_load_edge_list(const char* path, uint32_t* n, size_t* m, uint32_t** u,
                          uint32_t** v, double** w, double** degrees, double* total) {
  return guarded([&] {
    fsg::WeightedGraph g = fsg::load_edge_list(path);
    const auto& e = g.edges();
    std::vector<uint32_t> uu(e.size()), vv(e.size());
    std::vector<double> ww(e.size());
    for (size_t i = 0; i < e.size(); ++i) {
      uu[i] = e[i].u;
      vv[i] = e[i].v;
      ww[i] = e[i].w;
    }
    *n = g.num_vertices();
    *m = e.size();
    *u = dup_vector(uu);
    *v = dup_vector(vv);
    *w = dup_vector(ww);
    *degrees = dup_vector(g.degrees());
    *total = g.total_weight();
  });
}

namespace {
fsg::WeightedGraph adopt_graph(uint32_t n, size_t m, const uint32_t* u, const uint32_t* v,
                               const double* w) {
  std::vector<fsg::Edge> e(m);
  for (size_t i = 0; i < m; ++i) e[i] = {u[i], v[i], w[i]};
  fsg::GraphBuilder b(n);
  b.adopt_sorted_unique(std::move(e));
  return b.build();
}
}  // namespace

// fsg::smallest_eigenpairs (proj/src/spectral.cpp:40-222). vectors (n*q,
// column-major) and residuals may be NULL.
int fsgref_smallest_eigenpairs(uint32_t n, size_t m, const uint32_t* u, const uint32_t* v,
                               const double* w, uint32_t q, double tol, uint64_t seed,
                               double* values, double* vectors, double* residuals,
                               uint64_t* matvecs) {
  return guarded([&] {
    fsg::WeightedGraph g = adopt_graph(n, m, u, v, w);
    fsg::EigenOptions o;
    o.tol = tol;
    o.seed = seed;
    fsg::EigenResult r = fsg::smallest_eigenpairs(g, q, o);
    std::memcpy(values, r.eigenvalues.data(), q * sizeof(double));
    if (vectors) std::memcpy(vectors, r.eigenvectors.data(), size_t(n) * q * sizeof(double));
    if (residuals) std::memcpy(residuals, r.residuals.data(), q * sizeof(double));
    if (matvecs) *matvecs = r.matvecs;
  });
}

// fsg::kmeans (spectral.cpp:257-403) on caller rows (n x dim, row-major).
int fsgref_kmeans(const double* pts, uint32_t n, uint32_t dim, uint32_t k, uint32_t restarts,
                  uint32_t max_iters, double rel_tol, uint64_t seed, uint32_t* labels,
                  double* cost, uint32_t* iterations) {
  return guarded([&] {
    fsg::KMeansOptions o;
    o.restarts = restarts;
    o.max_iters = max_iters;
    o.rel_tol = rel_tol;
    o.seed = seed;
    fsg::KMeansResult r =
        fsg::kmeans(std::vector<double>(pts, pts + size_t(n) * dim), n, dim, k, o);
    std::memcpy(labels, r.labels.labels.data(), size_t(n) * sizeof(uint32_t));
    if (cost) *cost = r.cost;
    if (iterations) *iterations = r.iterations;
  });
}

// fsg::spectral_cluster (spectral.cpp:405-419) with default options.
int fsgref_spectral_cluster(uint32_t n, size_t m, const uint32_t* u, const uint32_t* v,
                            const double* w, uint32_t k, uint64_t seed, uint32_t* labels) {
  return guarded([&] {
    fsg::WeightedGraph g = adopt_graph(n, m, u, v, w);
    fsg::ClusterLabels l = fsg::spectral_cluster(g, k, seed);
    std::memcpy(labels, l.labels.data(), size_t(n) * sizeof(uint32_t));
  });
}

}  // extern "C"
