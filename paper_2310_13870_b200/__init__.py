"""B200-native KDE-driven similarity-graph sampler (arXiv 2310.13870 hot path).

Drop-in for the reference's ``fsg::build_similarity_graph`` path: the C ABI
is ``include/fsgg.h`` (libfsgg.so, hand-written sm_100a kernels); this
package is the host-side mirror of the reference interface over it.
"""
from .api import (BuildReport, Dataset, EigenOptions, EigenResult, KMeansOptions,
                  SpectralOptions, kmeans, smallest_eigenpairs, spectral_cluster, Kernel, KernelFamily, KdeBackend, KdeEstimator, LogBase,
                  RngMode, SampleDiagnostics, SparsifierConfig, WeightedGraph,
                  build_similarity_graph, build_similarity_graph_device, default_epsilon,
                  device_available, device_graph_to_host, exact_kde, load_csr, load_csv, make_estimator,
                  read_edge_list, sample_neighbors, sample_neighbors_counted,
                  sample_neighbors_counted_ex, SampleReport, RECORD_DTYPE, save_csv)
from .errors import (ConfigError, DeviceError, Error, InvalidConfig, IoError,
                     LengthMismatch, NumericError, TooFewPoints)

__all__ = [
    "EigenOptions", "EigenResult", "KMeansOptions", "SpectralOptions", "kmeans",
    "smallest_eigenpairs", "spectral_cluster", "device_graph_to_host",
    "BuildReport", "Dataset", "Kernel", "KernelFamily", "KdeBackend", "KdeEstimator", "LogBase", "RngMode",
    "SampleDiagnostics", "SparsifierConfig", "WeightedGraph", "build_similarity_graph",
    "build_similarity_graph_device", "default_epsilon", "device_available", "exact_kde",
    "load_csr", "load_csv", "save_csv", "make_estimator", "read_edge_list", "sample_neighbors", "sample_neighbors_counted",
    "sample_neighbors_counted_ex", "SampleReport", "RECORD_DTYPE", "ConfigError",
    "DeviceError", "Error", "InvalidConfig", "IoError", "LengthMismatch", "NumericError",
    "TooFewPoints",
]
