// TEST INFRASTRUCTURE: links the reference library (compiled in place) AND
// libfsgg.so into one binary and runs the same call both ways, proving the
// C++ drop-in (include/fsgg/fsg_adapter.hpp) on the reference's own types.
// Exit 0 when the edge sets are identical and weights agree to 1e-5.
#include <cmath>
#include <cstdio>

#include "fsg/datasets.hpp"
#include "fsg/sparsifier.hpp"
#include "fsgg/fsg_adapter.hpp"

int main() {
  auto data = fsg::make_blobs(2000, {{-2.0, 0.0}, {2.0, 0.0}}, 0.5, 1);
  std::vector<double> p32(data.data.raw().begin(), data.data.raw().end());
  for (double& v : p32) v = static_cast<float>(v);  // the device consumes fp32
  fsg::Dataset ds(p32, 2000, 2);
  fsg::Kernel kernel(fsg::KernelFamily::gaussian, 0.5);
  fsg::SparsifierConfig cfg;
  cfg.rounds = 32;
  cfg.kde.backend = fsg::KdeBackend::exact;
  fsg::BuildReport rc, rg;
  fsg::WeightedGraph cpu = fsg::build_similarity_graph(ds, kernel, cfg, &rc);
  fsg::WeightedGraph gpu = fsgg_adapter::build_similarity_graph(ds, kernel, cfg, &rg);
  if (cpu.num_edges() != gpu.num_edges()) {
    std::printf("edge count differs: %zu vs %zu\n", cpu.num_edges(), gpu.num_edges());
    return 1;
  }
  double worst = 0.0;
  for (size_t i = 0; i < cpu.num_edges(); ++i) {
    const auto &a = cpu.edges()[i], &b = gpu.edges()[i];
    if (a.u != b.u || a.v != b.v) {
      std::printf("edge %zu differs\n", i);
      return 1;
    }
    worst = std::fmax(worst, std::fabs(a.w - b.w) / a.w);
  }
  std::printf("adapter ok: %zu edges, max weight rel diff %.3e, cpu %.3fs (%s), gpu %.3fs (%s)\n",
              cpu.num_edges(), worst, rc.total_seconds, rc.backend.c_str(), rg.total_seconds,
              rg.backend.c_str());
  return worst <= 1e-5 ? 0 : 1;
}
