/* fsgg.h — C ABI of the B200-native KDE-driven similarity-graph sampler.
 *
 * Drop-in for the hot path of arXiv 2310.13870 as implemented by the
 * reference C++ library `fsg` (/root/reference/proj). Every entry point
 * names the reference interface it replaces (file:line). Plain pointers and
 * sizes only; no C++ or torch types cross this boundary.
 *
 * Error contract (proj/include/fsg/common.hpp:13-66): every function that
 * can fail returns FSGG_OK (0) or the reference's exit-code class —
 * 2 config (TooFewPoints, InvalidConfig, LengthMismatch), 3 I/O,
 * 4 numeric (sparsity invariant) — plus 5 for a CUDA/device failure. There
 * is no CPU fallback: without a usable sm_100 device every compute call
 * returns FSGG_ERR_DEVICE. fsgg_last_error() returns a thread-local message.
 *
 * Threading: calls are synchronous. A dataset handle owns its device,
 * stream and memory pool; do not use one handle from two threads at once.
 */
#ifndef FSGG_H
#define FSGG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

#define FSGG_OK 0
#define FSGG_ERR_CONFIG 2
#define FSGG_ERR_IO 3
#define FSGG_ERR_NUMERIC 4
#define FSGG_ERR_DEVICE 5

/* proj/include/fsg/kernel.hpp:12 KernelFamily */
#define FSGG_KERNEL_GAUSSIAN 0
#define FSGG_KERNEL_EXPONENTIAL 1
#define FSGG_KERNEL_LAPLACIAN 2

/* Routing random stream.
 * REFERENCE: the reference's keyed splitmix64 streams
 *   (proj/include/fsg/rng.hpp:11-71, keyed as in proj/src/sampler.cpp:213-216),
 *   reproduced bit-exactly, so graphs match the reference edge for edge.
 * PHILOX: counter-based Philox4x32-10 keyed by (seed, node, query, ticket);
 *   same distribution, validated by chi-squared, not edge-for-edge. */
#define FSGG_RNG_REFERENCE 0
#define FSGG_RNG_PHILOX 1

/* proj/include/fsg/kernel.hpp:21-58 (Kernel: family + bandwidth sigma). */
typedef struct fsgg_kernel {
  int family;
  double sigma;
} fsgg_kernel;

/* Mirrors fsg::SparsifierConfig (proj/include/fsg/sparsifier.hpp:14-26).
 * `epsilon` is read by the fast backend only (kde_backend below); the exact
 * backend, the default, reports epsilon 0 as the reference's does. */
typedef struct fsgg_config {
  double C;                  /* default 1 */
  double lambda_k1_estimate; /* default 1 */
  uint32_t rounds;           /* 0 = ceil(6 C log(n) / lambda) */
  double epsilon;            /* FSGG_KDE_FAST budget (0 = default_epsilon(n)) */
  int log_base;              /* 0 = log2 (default), 1 = natural */
  uint64_t seed;             /* default 1 */
  int rng_mode;              /* FSGG_RNG_REFERENCE (default) | FSGG_RNG_PHILOX */
  /* Query shard [query_begin, query_end) for multi-GPU runs; (0, 0) = all.
   * Results for a query never depend on the shard layout. */
  uint32_t query_begin;
  uint32_t query_end;
  /* 0 (default): certified pruning — a source sub-chunk whose bounding-box
   * bound is below 2^-48 of half the entry's node mass is skipped
   * (engine.cuh kPruneBits); with at most 2^20 sub-chunks per node the
   * skipped mass is below 2^-27 of the node mass, which the tie guard adds to
   * its margin, so routing decisions are unchanged. Per child sum:
   * |g - g_exact| <= (fp32 evaluation error) + 2^-27 * (node mass)
   * (tests/test_gpu_node_sums.py). 1: evaluate every kernel term (dense). */
  int dense_kde;
  /* fsg::KdeConfig::backend (proj/include/fsg/kde.hpp:20,28-30;
   * make_estimator proj/src/kde.cpp:104-129). FSGG_KDE_EXACT (the default
   * here: exact sums, the reference's exact backend edge for edge);
   * FSGG_KDE_FAST: the device analogue of the reference's (1 +- eps) fast
   * backend -- certified pruning with an epsilon-derived budget (eps =
   * `epsilon`, or default_epsilon(n) when 0; 0 < eps < 1 else
   * FSGG_ERR_CONFIG): every level skips at most eps / (depth + 1) of each
   * node's kernel mass, so each query's sampling distribution is within total
   * variation eps of the exact one and every degree g_full is within a factor
   * (1 - eps / (depth + 1)) of exact; no tie guard. Non-gaussian kernels fall
   * back to exact, as the reference does (UnsupportedKernel). FSGG_KDE_AUTO:
   * the reference's autoselect rule (fast for gaussian, d <= 3, n >= 4096).
   * The report's epsilon / backend say which ran. */
  int kde_backend;
} fsgg_config;

#define FSGG_KDE_EXACT 0
#define FSGG_KDE_FAST 1
#define FSGG_KDE_AUTO 2

/* Mirrors fsg::BuildReport (proj/include/fsg/sparsifier.hpp:40-58), plus
 * device counters. Phase times are device (CUDA event) seconds. */
typedef struct fsgg_report {
  uint32_t n;
  uint32_t rounds;
  double epsilon;
  char backend[32];
  uint64_t sampled_pairs;
  uint64_t self_pairs_discarded;
  uint64_t underflow_edges_discarded;
  uint64_t edge_count;
  uint64_t degenerate_draws;
  double estimator_build_seconds; /* node table + bounding boxes */
  double sampling_seconds;        /* level-synchronous descent */
  double degree_kde_seconds;      /* 0: fused into level 0 of the descent */
  double weighting_seconds;       /* pair collapse, weights, CSR, degrees */
  double total_seconds;
  uint64_t estimator_bytes;
  uint64_t graph_bytes;
  /* device extras */
  uint64_t kernel_evals;      /* Gaussian evaluations performed */
  uint64_t kde_tiled_evals;   /* of which in the tiled (big-node) kernel */
  double kde_tiled_seconds;   /* device time of the tiled kernel launches */
  uint32_t kde_tiled_launches;
  uint32_t levels;
  uint64_t peak_entries;
  uint32_t gpu_launches;      /* kernels launched by this call */
  uint64_t kernel_evals_performed;    /* evaluations actually executed */
  uint64_t kde_tiled_performed_evals; /* of which in the tiled kernel */
  uint64_t tie_verified_entries; /* entries re-decided on fp64 sums (tie guard) */
  uint64_t kde_root_performed_evals; /* pair evaluations of the symmetric root kernel */
  double kde_root_seconds;           /* its device time (0: one-sided root pass) */
} fsgg_report;

/* Per-edge quantities of the weighting step (sparsifier.hpp:29-38). */
typedef struct fsgg_edge_estimate {
  uint32_t i, j;
  double k_ij, g_i, g_j, p_hat_i_j, p_hat_j_i, p_hat;
} fsgg_edge_estimate;

/* Undirected graph, edges stored once with u < v, sorted by (u, v): the
 * layout of fsg::WeightedGraph (proj/include/fsg/graph.hpp:20-40), plus the
 * equivalent upper-triangular CSR row_ptr (n + 1 entries, row u holds the
 * v > u neighbours). Host memory owned by the library; release with
 * fsgg_graph_free. */
typedef struct fsgg_graph {
  uint32_t n;
  uint64_t num_edges;
  uint32_t* u;
  uint32_t* v;
  double* w;
  uint64_t* row_ptr;
  double* degrees; /* n entries, summed in the reference's order */
  double total_weight;
} fsgg_graph;

/* Same graph left in device memory (pointers valid until the next build on
 * the same dataset handle or fsgg_dataset_destroy). */
typedef struct fsgg_device_graph {
  uint32_t n;
  uint64_t num_edges;
  const uint32_t* u;
  const uint32_t* v;
  const double* w;
  const uint64_t* row_ptr;
  const double* degrees;
  double total_weight;
} fsgg_device_graph;

typedef struct fsgg_dataset fsgg_dataset;

const char* fsgg_version(void);
const char* fsgg_last_error(void);
/* 1 when a usable sm_100 device is visible, else 0. */
int fsgg_device_available(void);

void fsgg_config_init(fsgg_config* cfg);

/* proj/src/sparsifier.cpp:17-23 (SparsifierConfig::rounds_for) */
int fsgg_rounds_for(const fsgg_config* cfg, uint32_t n, uint32_t* out);
/* proj/src/kde.cpp:15-18 (default_epsilon) */
double fsgg_default_epsilon(uint32_t n, int log_base);

/* fsg::Dataset (proj/include/fsg/dataset.hpp:12-25; ctor dataset.cpp:14-23):
 * n x d row-major, index order defines the tree. Points are fp32 on the
 * device. `points_on_device` != 0 means `points` is a device pointer on
 * `device`. Validates n >= 1, d >= 1 and finiteness (InvalidConfig). */
int fsgg_dataset_create(const float* points, uint32_t n, uint32_t d,
                        int points_on_device, int device, fsgg_dataset** out);
/* Same, from fp64 host coordinates (rounded to fp32). */
int fsgg_dataset_create_f64(const double* points, uint32_t n, uint32_t d,
                            int device, fsgg_dataset** out);
/* Replace the coordinates of an existing dataset (same n, d) from host
 * memory: one host->device copy, no reallocation. */
int fsgg_dataset_upload(fsgg_dataset* ds, const float* host_points);
void fsgg_dataset_destroy(fsgg_dataset* ds);
uint32_t fsgg_dataset_size(const fsgg_dataset* ds);
uint32_t fsgg_dataset_dim(const fsgg_dataset* ds);
/* Raw device pointer of the fp32 coordinates. */
const float* fsgg_dataset_device_points(const fsgg_dataset* ds);
/* The cudaStream_t every kernel of this handle is launched on (for callers
 * that time or order work around the library with CUDA events). */
void* fsgg_dataset_stream(const fsgg_dataset* ds);

/* fsg::build_similarity_graph (proj/include/fsg/sparsifier.hpp:64-67,
 * proj/src/sparsifier.cpp:51-142). Host output. `estimates` (nullable)
 * receives a malloc'd array of num_edges records (free with fsgg_free). */
int fsgg_build_similarity_graph(fsgg_dataset* ds, const fsgg_kernel* kernel,
                                const fsgg_config* cfg, fsgg_graph* out,
                                fsgg_report* report,
                                fsgg_edge_estimate** estimates);

/* Device-resident variant (no device->host copy of the graph). */
int fsgg_build_similarity_graph_device(fsgg_dataset* ds,
                                       const fsgg_kernel* kernel,
                                       const fsgg_config* cfg,
                                       fsgg_device_graph* out,
                                       fsgg_report* report);

/* fsg::build_similarity_graph into caller host buffers (pinned memory for
 * full speed): the upper CSR (v, w: `capacity` entries, at least the number
 * of sampled unique pairs BEFORE underflow drops -- n*L always suffices --;
 * row_ptr: n+1; degrees: n) is copied out array by array
 * while the rest of the graph is still being finished, so the transfer
 * overlaps the device work. Any buffer pointer may be NULL (not copied);
 * total_weight (nullable) receives the graph's total weight. Edge u of
 * entry e is the row r with row_ptr[r] <= e < row_ptr[r+1]. */
int fsgg_build_similarity_graph_into(fsgg_dataset* ds, const fsgg_kernel* kernel,
                                     const fsgg_config* cfg, uint64_t capacity,
                                     uint32_t* v, double* w, uint64_t* row_ptr,
                                     double* degrees, uint64_t* num_edges,
                                     double* total_weight, fsgg_report* report);
/* One-call drop-in from host fp32 points to a host graph. */
int fsgg_build_similarity_graph_host(const float* points, uint32_t n,
                                     uint32_t d, const fsgg_kernel* kernel,
                                     const fsgg_config* cfg, int device,
                                     fsgg_graph* out, fsgg_report* report);

/* Copy the handle's current device graph (from the last device-resident
 * or distributed build) into host memory (free with fsgg_graph_free). */
int fsgg_device_graph_to_host(fsgg_dataset* ds, fsgg_graph* out);

/* Copy the handle's current device graph into caller-owned buffers (host
 * or device memory; any may be NULL): u, v (num_edges u32), w (num_edges
 * f64), row_ptr (n + 1 u64), degrees (n f64). With pinned (page-locked) host
 * buffers this runs at full PCIe/C2C bandwidth; completes before returning. */
int fsgg_device_graph_copy(fsgg_dataset* ds, uint32_t* u, uint32_t* v,
                           double* w, uint64_t* row_ptr, double* degrees);

void fsgg_graph_free(fsgg_graph* g);
void fsgg_free(void* p);

/* Spectral clustering on the graph (proj/include/fsg/spectral.hpp), the
 * consumer of the similarity graph, run on the device. */
typedef struct fsgg_eigen_options { /* spectral.hpp:11-16 */
  double tol;           /* 1e-6 */
  uint64_t max_matvecs; /* 0 = 50 n + 1000 */
  uint32_t max_basis;   /* 0 = auto */
  uint64_t seed;        /* 7 */
} fsgg_eigen_options;
typedef struct fsgg_kmeans_options { /* spectral.hpp:44-49 */
  uint32_t restarts;  /* 10 */
  uint32_t max_iters; /* 300 */
  double rel_tol;     /* 1e-8 */
  uint64_t seed;      /* 7 */
} fsgg_kmeans_options;
typedef struct fsgg_spectral_options {
  fsgg_eigen_options eigen;
  fsgg_kmeans_options kmeans;
} fsgg_spectral_options;
typedef struct fsgg_spectral_report {
  uint64_t matvecs;
  uint32_t components;
  uint32_t kmeans_iterations;
  double kmeans_cost;
  double eigen_seconds;
  double kmeans_seconds;
  uint64_t gpu_launches;
} fsgg_spectral_report;
void fsgg_spectral_options_init(fsgg_spectral_options* opts);

/* fsg::smallest_eigenpairs (spectral.cpp:40-222) of the normalised Laplacian
 * of the handle's current device graph (last build on `ds`): q eigenvalues
 * ascending; vectors (n x q column-major) and residuals may be NULL.
 * Isolated vertex -> FSGG_ERR_CONFIG; no convergence -> FSGG_ERR_NUMERIC. */
int fsgg_smallest_eigenpairs(fsgg_dataset* ds, uint32_t q, const fsgg_eigen_options* opts,
                             double* values, double* vectors, double* residuals,
                             uint64_t* matvecs);
/* fsg::spectral_cluster (spectral.cpp:405-419) on the handle's device graph;
 * labels: n entries in [0, k). opts may be NULL (reference defaults). */
int fsgg_spectral_cluster(fsgg_dataset* ds, uint32_t k, uint64_t seed,
                          const fsgg_spectral_options* opts, uint32_t* labels,
                          fsgg_spectral_report* report);
/* Same for a host graph (e.g. from fsgg_graph_load_text), uploaded to
 * `device` for the call. */
int fsgg_spectral_cluster_graph(const fsgg_graph* g, int device, uint32_t k, uint64_t seed,
                                const fsgg_spectral_options* opts, uint32_t* labels,
                                fsgg_spectral_report* report);
int fsgg_smallest_eigenpairs_graph(const fsgg_graph* g, int device, uint32_t q,
                                   const fsgg_eigen_options* opts, double* values,
                                   double* vectors, double* residuals, uint64_t* matvecs);
/* fsg::kmeans (spectral.cpp:257-403) on host rows (n x dim, row-major). */
int fsgg_kmeans(const double* points, uint32_t n, uint32_t dim, uint32_t k,
                const fsgg_kmeans_options* opts, int device, uint32_t* labels,
                double* cost, uint32_t* iterations);

/* Graph files (host-only; no device needed).
 * Text edge list, byte-identical to fsg::write_edge_list / save_edge_list
 * (proj/src/graph.cpp:234-241, 265-270): "n m\n" then "u v %.17g\n" per
 * edge in array order. threads = 0 uses every host core; the bytes do not
 * depend on it. */
int fsgg_graph_save_text(const char* path, uint32_t n, uint64_t num_edges,
                         const uint32_t* u, const uint32_t* v, const double* w,
                         uint32_t threads);
/* fsg::read_edge_list / load_edge_list (graph.cpp:243-263, 272-276): swaps
 * u > v, sorts unsorted input by (u, v), degrees and total weight summed in
 * the reference's order. Returns FSGG_ERR_IO for unreadable or malformed
 * files. Free with fsgg_graph_free. */
int fsgg_graph_load_text(const char* path, uint32_t threads, fsgg_graph* out);
/* Point files, fsg::load_csv / save_csv (proj/src/dataset.cpp:54-130): an
 * optional header row (first field not a number; a trailing "label" column
 * marks integer labels), comma-separated values parsed as doubles; saving
 * writes "x0,...,x{d-1}[,label]" and "%.17g" values. Rows are parsed and
 * formatted in parallel (threads = 0: every host core); files and errors do
 * not depend on the thread count. load: *points (n x d, row-major) and
 * *labels (NULL when the file has none; pass labels = NULL to skip them)
 * are freed with fsgg_free. Malformed files return FSGG_ERR_IO, non-finite
 * values FSGG_ERR_CONFIG, as the reference. */
int fsgg_csv_load(const char* path, uint32_t threads, double** points, uint32_t* n,
                  uint32_t* d, uint32_t** labels);
int fsgg_csv_save(const char* path, const double* points, uint32_t n, uint32_t d,
                  const uint32_t* labels, uint32_t threads);
/* Binary upper-triangular CSR ("FSGGCSR1", n, m, total weight, row_ptr,
 * v, w, degrees; little-endian): no text conversion either way. */
int fsgg_graph_save_csr(const char* path, const fsgg_graph* g);
int fsgg_graph_load_csr(const char* path, fsgg_graph* out);

/* fsg::SampleDiagnostics (proj/include/fsg/sampler.hpp:22-26). */
typedef struct fsgg_sample_diag {
  uint32_t nlevels;
  uint64_t entries_per_level[64];
  uint64_t tickets_per_level[64];
  uint64_t degenerate_draws;
} fsgg_sample_diag;

/* fsg::sample_neighbors_counted (proj/include/fsg/sampler.hpp:48-51,
 * proj/src/sampler.cpp:77-247). `queries` is a host array; duplicates are
 * merged as the reference does (:89-106). Output: malloc'd triples
 * (query, source, count) sorted by (query, source), 3 u32 each. */
int fsgg_sample_neighbors_counted(fsgg_dataset* ds, const fsgg_kernel* kernel,
                                  const uint32_t* queries, size_t num_queries,
                                  uint32_t rounds, uint64_t seed, int rng_mode,
                                  int dense_kde, uint32_t** triples,
                                  size_t* count, fsgg_sample_diag* diag);

/* Same descent with options and a richer report (test / diagnostics
 * entry point; the reference's closest equivalent is the recording
 * KdeEstimator wrapper its tests put around ExactKdeEstimator::eval,
 * proj/src/sampler.cpp:146-149 -> kde.cpp:38-49).
 *
 * record_sums = 1 exports, for every (node, query) entry of every level, the
 * two child sums exactly as the level's KDE kernels produced them (symmetric
 * root, root-row / block lookups, tiled or tensor-core passes, direct
 * kernels), BEFORE the tie guard re-decides near-ties on fp64 sums. It forces
 * the level-synchronous path (single-ticket walks off, which use the same
 * direct_child_sums device function as the direct kernel). Records are
 * malloc'd (free with fsgg_free); children of node [first, last) are
 * [first, first + (last - first) / 2) and [that, last) (sampler.cpp:141,200);
 * nodes of one point carry left = right = 0. */
typedef struct fsgg_entry_record {
  uint32_t level, query, first, last;
  double left, right;
} fsgg_entry_record;

typedef struct fsgg_sample_options {
  int rng_mode;      /* FSGG_RNG_REFERENCE | FSGG_RNG_PHILOX */
  int dense_kde;     /* 1: no certified pruning */
  int record_sums;   /* 1: export every entry's child sums (see above) */
  int walks;         /* 0: no single-ticket walks (1 default) */
  int kde_backend;   /* FSGG_KDE_EXACT (default) | _FAST | _AUTO, as fsgg_config */
  double epsilon;    /* fast backend budget; 0 = default_epsilon(n) */
} fsgg_sample_options;

typedef struct fsgg_sample_report {
  fsgg_sample_diag diag;
  uint64_t kernel_evals;            /* reference-equivalent Gaussian evaluations */
  uint64_t kernel_evals_performed;  /* evaluations executed on the device */
  uint64_t root_evals_performed;    /* symmetric root pass (0: it did not run) */
  uint64_t tie_verified;            /* entries re-decided on fp64 sums */
  fsgg_entry_record* records;       /* record_sums only, else NULL */
  size_t num_records;
} fsgg_sample_report;

void fsgg_sample_options_init(fsgg_sample_options* opt);
int fsgg_sample_neighbors_counted_ex(fsgg_dataset* ds, const fsgg_kernel* kernel,
                                     const uint32_t* queries, size_t num_queries,
                                     uint32_t rounds, uint64_t seed,
                                     const fsgg_sample_options* opt, uint32_t** triples,
                                     size_t* count, fsgg_sample_report* rep);

/* fsg::KdeEstimator::eval (proj/include/fsg/kde.hpp:54-58, exact backend
 * proj/src/kde.cpp:57-71): out[t] = max(sum_{j in [first,last)} k(x_t, x_j),
 * 1e-300) for a non-empty range, 0 for an empty one. Host arrays. */
int fsgg_kde_eval(fsgg_dataset* ds, const fsgg_kernel* kernel, uint32_t first,
                  uint32_t last, const uint32_t* targets, size_t m,
                  double* out);

/* ---- input side (proj/src/datasets.cpp:32-124), host generators ------ */
/* make_moons: outer arc first, keyed Box-Muller noise; fp64 output. */
int fsgg_make_moons(uint32_t n, double noise, uint64_t seed, double* points,
                    uint32_t* labels);
/* make_blobs: centers k x d, n split as evenly as possible. */
int fsgg_make_blobs(uint32_t n, const double* centers, uint32_t k, uint32_t d,
                    double stddev, uint64_t seed, double* points,
                    uint32_t* labels);
/* Harness-defined configs without a reference generator:
 * C4 synthetic image pixels (row/H, col/W, r, g, b), H x W raster, 8 seeded
 * Voronoi colour regions, noise std 0.03. */
int fsgg_make_image_features(uint32_t height, uint32_t width,
                             uint32_t regions, double noise, uint64_t seed,
                             double* points, uint32_t* labels);
/* C5 Gaussian mixture: k components in make_blobs order, centres U[0,1]^d,
 * per-component std, values clipped to [0,1]. */
int fsgg_make_gmm(uint32_t n, uint32_t d, uint32_t k, double stddev,
                  uint64_t seed, double* points, uint32_t* labels);

/* ---- input side on the device (same generators, GPU `device`) -------- */
/* Each writes the points of the host generator above straight into device
 * memory: fp64 (points64, n x d) and/or rounded to fp32 (points32, the
 * precision the descent consumes) and/or labels — any of the three may be
 * NULL; all are device pointers on `device`. log/sin/cos are correctly
 * rounded (double-double); glibc's are within 0.502 ulp, so a fp64
 * coordinate may differ from the host generator's in its last bit (~0.1% of
 * values); the fp32 arrays are identical. Blocking. Errors as the host
 * generators (2 for invalid arguments), 5 without an sm_100 device. */
int fsgg_make_moons_device(uint32_t n, double noise, uint64_t seed, int device,
                           double* points64, float* points32, uint32_t* labels);
/* centers: HOST array k x d */
int fsgg_make_blobs_device(uint32_t n, const double* centers, uint32_t k, uint32_t d,
                           double stddev, uint64_t seed, int device, double* points64,
                           float* points32, uint32_t* labels);
int fsgg_make_image_features_device(uint32_t height, uint32_t width, uint32_t regions,
                                    double noise, uint64_t seed, int device,
                                    double* points64, float* points32, uint32_t* labels);
int fsgg_make_gmm_device(uint32_t n, uint32_t d, uint32_t k, double stddev, uint64_t seed,
                         int device, double* points64, float* points32, uint32_t* labels);

/* ---- multi-GPU shard pipeline (one process per GPU) ------------------ */
/* Phase 1 on every rank: descent for queries [query_begin, query_end) of
 * cfg, producing the shard's sorted unique undirected pair keys and its
 * slice of the degree KDE g_full. Device pointers, valid until the next
 * call on this dataset. pair keys encode (u << 32) | v with u < v. */
typedef struct fsgg_shard {
  uint32_t query_begin, query_end;
  uint32_t rounds;
  uint64_t num_pairs;
  const uint64_t* pairs;   /* device */
  const double* g_full;    /* device, query_end - query_begin entries */
  uint64_t sampled_pairs;
  uint64_t self_pairs;
  uint64_t degenerate_draws;
} fsgg_shard;
int fsgg_sample_shard(fsgg_dataset* ds, const fsgg_kernel* kernel,
                      const fsgg_config* cfg, fsgg_shard* out,
                      fsgg_report* report);
/* Copy the last shard's pair keys (num_pairs u64) and g_full slice
 * (query_end - query_begin f64) into caller-owned device buffers (either
 * may be NULL); completes before returning. */
int fsgg_shard_export(fsgg_dataset* ds, uint64_t* pairs_device,
                      double* g_full_device);
/* Owner mode of the symmetric root pass (low d, multi-GPU). At the root
 * every query is a source, and the block-pair tiles between two shards
 * serve both: instead of both ranks evaluating such a tile, one computes it
 * and sends the other rank's side as a record. Sequence per rank:
 *   fsgg_shard_bounds(ds, k, world, bounds)     block-aligned query ranges
 *   fsgg_shard_root_prepare(ds, k, cfg, &n)   this shard's tiles, and n
 *       records owed to other ranks
 *   fsgg_shard_root_export(ds, dst)             copy them to a caller device
 *       buffer: 324 32-bit words each (X, Y, first point of X, |X|, then
 *       |X| <= 320 fp32 values of X's points over partner block Y), for the
 *       rank whose range holds point word[2]
 *   (caller: all-to-all of the records)
 *   fsgg_shard_root_receive(ds, recv, m)        store the m received records
 *   fsgg_sample_shard(ds, k, cfg, ...)          the descent, root tiles reused
 * Results are bit-identical to the 1-GPU build. prepare returns 0 records
 * (and every rank's descent computes its root alone) when the root pass is
 * not symmetric for this data -- a property of the dataset, so all ranks
 * agree. A range that is not block-aligned is FSGG_ERR_CONFIG (a silent
 * per-rank fallback would leave an aligned peer waiting for records). Replaces no
 * reference interface: the reference has no multi-device path
 * (SURVEY.md §2). */
/* kernel may be NULL: equal block counts; else block-aligned bounds that
 * balance a per-block cost model (root pair evaluations + descent work). */
int fsgg_shard_bounds(fsgg_dataset* ds, const fsgg_kernel* kernel, uint32_t world,
                      uint32_t* bounds_host);
int fsgg_shard_root_prepare(fsgg_dataset* ds, const fsgg_kernel* kernel,
                            const fsgg_config* cfg, uint64_t* num_records);
int fsgg_shard_root_export(fsgg_dataset* ds, uint32_t* records_device);
int fsgg_shard_root_receive(fsgg_dataset* ds, const uint32_t* records_device,
                            uint64_t num_records);
/* Phase 1 for the row-sharded finish: the descent of fsgg_sample_shard,
 * then the shard's pair keys (u << 32 | v, u < v, self samples dropped,
 * duplicates kept, unsorted) grouped by the rank owning row u under
 * `bounds` (world + 1 entries, 0 .. n, host; world <= 64): counts[r] keys for
 * rank r, in rank order, at out->pairs — ready for one all-to-all, no sort
 * on the sending side (the owner's fsgg_finish_graph sorts and dedupes).
 * out->num_pairs is their total. */
int fsgg_sample_shard_routed(fsgg_dataset* ds, const fsgg_kernel* kernel,
                             const fsgg_config* cfg, uint32_t world, const uint32_t* bounds,
                             uint64_t* counts, fsgg_shard* out, fsgg_report* report);

/* Phase 2 after the caller all-gathers g_full (n doubles, device) and the
 * shards' pair keys (concatenated, device, any order, duplicates allowed):
 * dedupe, weight, CSR and degrees exactly as the 1-GPU path. */
int fsgg_finish_graph(fsgg_dataset* ds, const fsgg_kernel* kernel,
                      uint32_t rounds, const double* g_full_device,
                      const uint64_t* pairs_device, uint64_t num_pairs,
                      fsgg_device_graph* out, fsgg_report* report);

/* Row-sharded phase 2 (each rank owns the rows [row_begin, row_end) of the
 * upper-triangular graph; parallel.py routes every pair key (u << 32 | v,
 * u < v) to the owner of u first). Call sequence per rank:
 *   fsgg_finish_graph(ds, ..., routed pairs, ...)   dedupe + weights of the
 *       rank's rows (degrees in `out` are partial: use the next two calls);
 *   fsgg_rows_transposed(ds, v, w)   the rows' (v, w), m entries, stable-sorted
 *       by v, to be routed to the owners of v;
 *   fsgg_rows_degrees(ds, v, w, n, row_begin, row_end, deg)   degrees of the
 *       rank's rows from the received (v, w) (concatenated in rank order) and
 *       its own rows — summed in exactly the 1-GPU order.
 * All pointers are device pointers on the handle's device. */
int fsgg_rows_transposed(fsgg_dataset* ds, uint32_t* v_device, double* w_device);
/* The rank's slice of the gathered graph's row_ptr: row_ptr[row_begin ..
 * row_end) of its rows plus edge_offset (the edges of the ranks before it),
 * row_end - row_begin entries (device); concatenated in rank order plus the
 * total edge count they form the global upper CSR row_ptr. */
int fsgg_rows_row_ptr(fsgg_dataset* ds, uint32_t row_begin, uint32_t row_end,
                      uint64_t edge_offset, uint64_t* row_ptr_device);
int fsgg_rows_degrees(fsgg_dataset* ds, const uint32_t* lower_v_device,
                      const double* lower_w_device, uint64_t num_lower, uint32_t row_begin,
                      uint32_t row_end, double* degrees_device);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* FSGG_H */
