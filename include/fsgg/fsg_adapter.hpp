// fsg_adapter.hpp — header-only C++ drop-in for the reference library.
//
// A caller of the reference `fsg` (/root/reference/proj) switches its hot
// path to the B200 by including this header instead of calling
// fsg::build_similarity_graph (proj/include/fsg/sparsifier.hpp:64-67) and
// linking libfsgg.so. Same arguments, same return type (fsg::WeightedGraph
// assembled through GraphBuilder::adopt_sorted_unique, graph.cpp:40-54), same
// exceptions (fsg::InvalidConfig / TooFewPoints / NumericError with exit
// codes 2/4, common.hpp:13-66); a device failure surfaces as fsg::Error with
// exit code 5. Requires the reference headers on the include path.
#pragma once

#include <cstdlib>
#include <string>
#include <vector>

#include "fsg/common.hpp"
#include "fsg/dataset.hpp"
#include "fsg/graph.hpp"
#include "fsg/kernel.hpp"
#include "fsg/sampler.hpp"
#include "fsg/sparsifier.hpp"
#include "fsgg.h"

namespace fsgg_adapter {

inline void throw_for(int rc, const char* where) {
  if (rc == FSGG_OK) return;
  std::string msg = std::string(where) + ": " + fsgg_last_error();
  if (rc == FSGG_ERR_CONFIG) {
    if (msg.find("n >= 2") != std::string::npos) throw fsg::TooFewPoints(msg);
    throw fsg::InvalidConfig(msg);
  }
  if (rc == FSGG_ERR_IO) throw fsg::IoError(msg);
  if (rc == FSGG_ERR_NUMERIC) throw fsg::NumericError(msg);
  throw fsg::Error(msg, rc);
}

inline fsgg_kernel to_kernel(const fsg::Kernel& k) {
  fsgg_kernel out;
  out.family = static_cast<int>(k.family());
  out.sigma = k.sigma();
  return out;
}

inline fsgg_config to_config(const fsg::SparsifierConfig& c) {
  fsgg_config out;
  fsgg_config_init(&out);
  out.C = c.C;
  out.lambda_k1_estimate = c.lambda_k1_estimate;
  out.rounds = c.rounds;
  out.epsilon = c.epsilon;
  out.log_base = c.log_base == fsg::LogBase::natural ? 1 : 0;
  out.seed = c.seed;
  return out;
}

// RAII device copy of an fsg::Dataset (fp64 coordinates rounded to fp32).
class DeviceDataset {
public:
  explicit DeviceDataset(const fsg::Dataset& ds, int device = 0) {
    throw_for(fsgg_dataset_create_f64(ds.raw().data(), ds.size(), ds.dim(),
                                      device, &h_),
              "fsgg_dataset_create_f64");
  }
  ~DeviceDataset() { fsgg_dataset_destroy(h_); }
  DeviceDataset(const DeviceDataset&) = delete;
  DeviceDataset& operator=(const DeviceDataset&) = delete;
  fsgg_dataset* get() const { return h_; }

private:
  fsgg_dataset* h_ = nullptr;
};

// Drop-in for fsg::build_similarity_graph.
inline fsg::WeightedGraph build_similarity_graph(
    const fsg::Dataset& ds, const fsg::Kernel& kernel,
    const fsg::SparsifierConfig& config, fsg::BuildReport* report = nullptr,
    std::vector<fsg::EdgeEstimate>* estimates = nullptr, int device = 0) {
  DeviceDataset dd(ds, device);
  fsgg_kernel k = to_kernel(kernel);
  fsgg_config c = to_config(config);
  fsgg_graph g;
  fsgg_report r;
  fsgg_edge_estimate* est = nullptr;
  throw_for(fsgg_build_similarity_graph(dd.get(), &k, &c, &g, &r,
                                        estimates ? &est : nullptr),
            "fsgg_build_similarity_graph");
  std::vector<fsg::Edge> edges(g.num_edges);
  for (uint64_t i = 0; i < g.num_edges; ++i) edges[i] = {g.u[i], g.v[i], g.w[i]};
  if (estimates) {
    estimates->clear();
    for (uint64_t i = 0; i < g.num_edges; ++i)
      estimates->push_back({est[i].i, est[i].j, est[i].k_ij, est[i].g_i,
                            est[i].g_j, est[i].p_hat_i_j, est[i].p_hat_j_i,
                            est[i].p_hat});
    fsgg_free(est);
  }
  const uint32_t n = g.n;
  fsgg_graph_free(&g);
  if (report) {
    report->n = r.n;
    report->rounds = r.rounds;
    report->epsilon = r.epsilon;
    report->backend = r.backend;
    report->sampled_pairs = r.sampled_pairs;
    report->self_pairs_discarded = r.self_pairs_discarded;
    report->underflow_edges_discarded = r.underflow_edges_discarded;
    report->edge_count = r.edge_count;
    report->degenerate_draws = r.degenerate_draws;
    report->estimator_build_seconds = r.estimator_build_seconds;
    report->sampling_seconds = r.sampling_seconds;
    report->degree_kde_seconds = r.degree_kde_seconds;
    report->weighting_seconds = r.weighting_seconds;
    report->total_seconds = r.total_seconds;
    report->estimator_bytes = r.estimator_bytes;
    report->graph_bytes = r.graph_bytes;
  }
  fsg::GraphBuilder builder(n, /*strict=*/true);
  builder.adopt_sorted_unique(std::move(edges));
  return builder.build();
}

// Drop-in for fsg::sample_neighbors_counted with an exact estimator.
inline std::vector<fsg::CountedNeighborSample> sample_neighbors_counted(
    const fsg::Dataset& ds, const fsg::Kernel& kernel,
    const std::vector<uint32_t>& queries, uint32_t rounds, uint64_t seed,
    fsg::SampleDiagnostics* diagnostics = nullptr, int device = 0) {
  DeviceDataset dd(ds, device);
  fsgg_kernel k = to_kernel(kernel);
  uint32_t* tri = nullptr;
  size_t count = 0;
  fsgg_sample_diag diag;
  throw_for(fsgg_sample_neighbors_counted(dd.get(), &k, queries.data(),
                                          queries.size(), rounds, seed,
                                          FSGG_RNG_REFERENCE, 0, &tri, &count,
                                          &diag),
            "fsgg_sample_neighbors_counted");
  std::vector<fsg::CountedNeighborSample> out(count);
  for (size_t i = 0; i < count; ++i)
    out[i] = {tri[3 * i], tri[3 * i + 1], tri[3 * i + 2]};
  fsgg_free(tri);
  if (diagnostics) {
    diagnostics->entries_per_level.assign(diag.entries_per_level,
                                          diag.entries_per_level + diag.nlevels);
    diagnostics->tickets_per_level.assign(diag.tickets_per_level,
                                          diag.tickets_per_level + diag.nlevels);
    diagnostics->degenerate_draws = diag.degenerate_draws;
  }
  return out;
}

}  // namespace fsgg_adapter
