/* TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
 *
 * Plain-C restatement of the reference's KDE-driven similarity-graph path
 * (arXiv 2310.13870, Algorithms 1 and 2 as implemented in
 * /root/reference/proj). Each function cites the reference file:line it
 * restates. Exact (fp64, Kahan) backend only: the reference's FGT backend
 * (proj/src/kde_fast.cpp) is out of scope.
 *
 * Pinned against the reference itself: tests/test_oracle.py checks this
 * restatement bit-for-bit against oracle/_ref/libfsgref.so (the reference's
 * own sources compiled in place) when that library is present, and against
 * the committed golden fixtures in tests/golden/ (generated from
 * oracle/_ref by tests/golden/make_golden.py) everywhere.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library. */
#ifndef FSG_ORACLE_H
#define FSG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* proj/include/fsg/rng.hpp:11-16 */
uint64_t oracle_splitmix64(uint64_t x);
/* proj/include/fsg/rng.hpp:20-27 — returns the stream key */
uint64_t oracle_rng_key(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b);
/* proj/include/fsg/rng.hpp:32-34 — draw `counter` of stream `key` */
double oracle_rng_double(uint64_t key, uint64_t counter);
/* proj/include/fsg/rng.hpp:65-71 */
uint64_t oracle_binomial(uint64_t key, uint64_t m, double p);

/* proj/tests/support.hpp:22-28 */
void oracle_random_dataset(uint32_t n, uint32_t d, uint64_t seed, double lo,
                           double hi, double* out);

/* proj/include/fsg/kernel.hpp:28-53; family 0 gaussian, 1 exponential,
 * 2 laplacian */
double oracle_kernel(int family, double sigma, const double* x,
                     const double* y, uint32_t d);

/* proj/src/kde.cpp:38-71 (ExactKdeEstimator::eval): out[t] =
 * max(kahan_sum, floor) for a non-empty range, 0 for an empty one.
 * Returns 0, or 2 on an invalid range/target (InvalidConfig). */
int oracle_kde_exact(const double* pts, uint32_t n, uint32_t d, int family,
                     double sigma, uint32_t first, uint32_t last,
                     const uint32_t* targets, size_t m, double floor_,
                     double* out);

typedef struct {
  uint32_t nlevels;
  uint64_t entries_per_level[64];
  uint64_t tickets_per_level[64];
  uint64_t degenerate_draws;
} oracle_diag;

/* proj/src/sampler.cpp:77-247 with the exact backend. Output triples
 * (query, source, count), sorted by (query, source), malloc'd into *out
 * (3 u32 per triple). When rec_* are non-NULL every child sum is recorded
 * as (first, last, query, sum), in the order the reference's
 * RecordingEstimator sees them with inline_range = 0. Returns 0 / 2. */
int oracle_sample_counted(const double* pts, uint32_t n, uint32_t d,
                          int family, double sigma, const uint32_t* queries,
                          size_t nq, uint32_t rounds, uint64_t seed,
                          uint32_t** out, size_t* count, oracle_diag* diag,
                          uint32_t** rec_first, uint32_t** rec_last,
                          uint32_t** rec_query, double** rec_sum,
                          size_t* rec_count);

/* proj/src/sparsifier.cpp:17-23 */
int oracle_rounds_for(uint32_t n, double C, double lambda, uint32_t rounds,
                      int log_base, uint32_t* out);
/* proj/src/kde.cpp:15-18 */
double oracle_default_epsilon(uint32_t n, int log_base);

/* proj/src/sparsifier.cpp:51-142 (exact backend). Edges sorted (u < v),
 * degrees as WeightedGraph computes them (proj/src/graph.cpp:14-21).
 * estimates: 8 doubles per edge (i, j, k_ij, g_i, g_j, p_i, p_j, p_hat).
 * report[8]: n, rounds, sampled_pairs, self_pairs, underflow_edges,
 * edge_count, degenerate_draws, total_weight.
 * g_full (n doubles, optional) receives the degree KDE. Returns 0/2/4. */
int oracle_build_graph(const double* pts, uint32_t n, uint32_t d, int family,
                       double sigma, uint32_t rounds, uint64_t seed,
                       size_t* m, uint32_t** u, uint32_t** v, double** w,
                       double** degrees, double** estimates, double* g_full,
                       double* report);

void oracle_free(void* p);
void oracle_set_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
