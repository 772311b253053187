// Spectral clustering on a device-resident graph (spectral.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "engine.cuh"

namespace fsgg {

// Upper-triangular CSR of an undirected graph (row u holds its v > u
// neighbours) plus degrees, all device pointers.
struct SpectralGraphView {
  uint32_t n = 0;
  uint64_t m = 0;
  const uint64_t* row_ptr = nullptr;
  const uint32_t* col = nullptr;
  const double* w = nullptr;
  const double* degrees = nullptr;
};

// proj/include/fsg/spectral.hpp:11-16 and :44-49
struct EigenOpts {
  double tol = 1e-6;
  uint64_t max_matvecs = 0;
  uint32_t max_basis = 0;
  uint64_t seed = 7;
};
struct KmeansOpts {
  uint32_t restarts = 10;
  uint32_t max_iters = 300;
  double rel_tol = 1e-8;
  uint64_t seed = 7;
};

struct SpectralStats {
  uint64_t matvecs = 0;
  uint32_t ncomp = 0;
  uint32_t kmeans_iterations = 0;
  double kmeans_cost = 0.0;
  double eigen_seconds = 0.0;
  double kmeans_seconds = 0.0;
  uint64_t launches = 0;
};

// fsg::smallest_eigenpairs: q eigenvalues ascending, eigenvectors (n x q,
// column-major) left in `vectors` on the device.
void smallest_eigenpairs_dev(const SpectralGraphView& g, cudaStream_t s, uint32_t q,
                             const EigenOpts& opts, std::vector<double>& values,
                             std::vector<double>& residuals, DevBuf& vectors, SpectralStats& st);

// fsg::kmeans on device rows (n x dim, row-major); labels to host memory.
void kmeans_dev(const double* pts, uint32_t n, uint32_t dim, uint32_t k, const KmeansOpts& opts,
                cudaStream_t s, uint32_t* labels_out, double* cost_out, uint32_t* iters_out,
                SpectralStats& st);

// fsg::spectral_cluster (eigenpairs -> embedding -> k-means).
void spectral_cluster_dev(const SpectralGraphView& g, cudaStream_t s, uint32_t k, uint64_t seed,
                          const EigenOpts& eopts, const KmeansOpts& kopts, uint32_t* labels,
                          std::vector<double>* values, SpectralStats& st);

}  // namespace fsgg
