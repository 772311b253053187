/* TEST INFRASTRUCTURE ONLY — see fsg_oracle.h for scope and pinning.
 *
 * Plain-C restatement of the reference hot path. Every function names the
 * reference file:line it follows. Nothing here is on the product path. */
#include "fsg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ROUTE_TAG 0x88b4f8a3c2d1e5f7ULL /* proj/src/sampler.cpp:25 */
#define SUM_FLOOR 1e-300                /* proj/include/fsg/kde.hpp:43 */

void oracle_free(void* p) { free(p); }

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* proj/include/fsg/rng.hpp:11-16 */
uint64_t oracle_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* proj/include/fsg/rng.hpp:20-27 */
uint64_t oracle_rng_key(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
  uint64_t k = oracle_splitmix64(seed);
  k = oracle_splitmix64(k ^ oracle_splitmix64(tag ^ 0x6a09e667f3bcc909ULL));
  k = oracle_splitmix64(k ^ oracle_splitmix64(a ^ 0xbb67ae8584caa73bULL));
  k = oracle_splitmix64(k ^ oracle_splitmix64(b ^ 0x3c6ef372fe94f82bULL));
  return k;
}

/* proj/include/fsg/rng.hpp:29-34 */
double oracle_rng_double(uint64_t key, uint64_t counter) {
  return (double)(oracle_splitmix64(key + counter) >> 11) * 0x1.0p-53;
}

/* proj/include/fsg/rng.hpp:65-71: Binomial(m, p) as m Bernoulli trials */
uint64_t oracle_binomial(uint64_t key, uint64_t m, double p) {
  if (p <= 0.0) return 0;
  if (p >= 1.0) return m;
  uint64_t s = 0;
  for (uint64_t i = 0; i < m; ++i) s += oracle_rng_double(key, i) < p ? 1 : 0;
  return s;
}

/* proj/tests/support.hpp:22-28 */
void oracle_random_dataset(uint32_t n, uint32_t d, uint64_t seed, double lo,
                           double hi, double* out) {
  uint64_t key = oracle_rng_key(seed, 0x7465737464617461ULL, 0, 0);
  for (size_t i = 0; i < (size_t)n * d; ++i)
    out[i] = lo + (hi - lo) * oracle_rng_double(key, i);
}

/* Squared distance exactly as the reference BINARY evaluates it: g++ -O3
 * with an FMA-capable -march vectorises the loop of kernel.hpp:31-35
 * (products rounded, then added in order) and contracts the scalar tail
 * (the last coordinate when d is odd) into a fused multiply-add. Verified
 * bit-for-bit against oracle/_ref for d = 1..16 (tests/test_oracle.py). */
static double sq_dist_ref(const double* x, const double* y, uint32_t d) {
  double s = 0.0;
  uint32_t even = d & ~1u;
  for (uint32_t i = 0; i < even; ++i) {
    double t = x[i] - y[i];
    double p = t * t;
    s = s + p;
  }
  if (d & 1u) {
    double t = x[d - 1] - y[d - 1];
    s = fma(t, t, s);
  }
  return s;
}

/* proj/include/fsg/kernel.hpp:28-53 */
double oracle_kernel(int family, double sigma, const double* x,
                     const double* y, uint32_t d) {
  double s = 0.0;
  switch (family) {
    case 0:
      s = sq_dist_ref(x, y, d);
      return exp(-s / (sigma * sigma));
    case 1:
      s = sq_dist_ref(x, y, d);
      return exp(-sqrt(s) / sigma);
    case 2:
      for (uint32_t i = 0; i < d; ++i) s += fabs(x[i] - y[i]);
      return exp(-s / sigma);
  }
  return 0.0;
}

/* proj/src/kde.cpp:38-49 (compensated_range_sum) */
static double kahan_range(const double* pts, uint32_t d, int family,
                          double sigma, uint32_t first, uint32_t last,
                          const double* y) {
  double sum = 0.0, comp = 0.0;
  for (uint32_t j = first; j < last; ++j) {
    double term = oracle_kernel(family, sigma, y, pts + (size_t)j * d, d) - comp;
    double next = sum + term;
    comp = (next - sum) - term;
    sum = next;
  }
  return sum;
}

/* proj/src/kde.cpp:29-35, 57-71 */
int oracle_kde_exact(const double* pts, uint32_t n, uint32_t d, int family,
                     double sigma, uint32_t first, uint32_t last,
                     const uint32_t* targets, size_t m, double floor_,
                     double* out) {
  if (first > last || last > n) return 2;
  for (size_t t = 0; t < m; ++t)
    if (targets[t] >= n) return 2;
#pragma omp parallel for schedule(dynamic, 16)
  for (size_t t = 0; t < m; ++t) {
    double s = kahan_range(pts, d, family, sigma, first, last,
                           pts + (size_t)targets[t] * d);
    out[t] = last == first ? 0.0 : (s > floor_ ? s : floor_);
  }
  return 0;
}

/* proj/src/kde.cpp:15-18 */
double oracle_default_epsilon(uint32_t n, int log_base) {
  double nn = n < 2 ? 2.0 : (double)n;
  double l = log_base ? log(nn) : log2(nn);
  return 1.0 / (6.0 * (l > 1.0 ? l : 1.0));
}

/* proj/src/sparsifier.cpp:17-23 */
int oracle_rounds_for(uint32_t n, double C, double lambda, uint32_t rounds,
                      int log_base, uint32_t* out) {
  if (rounds > 0) {
    *out = rounds;
    return 0;
  }
  double nn = n < 2 ? 2.0 : (double)n;
  double l = log_base ? log(nn) : log2(nn);
  if (l < 1.0) l = 1.0;
  double r = ceil(6.0 * C * l / lambda);
  if (!(r >= 1.0) || r > 4e9) return 2;
  *out = (uint32_t)r;
  return 0;
}

typedef struct {
  uint32_t first, last, query, tickets;
} entry; /* proj/src/sampler.cpp:27-32 */

typedef struct {
  uint32_t q, s, c;
} triple;

static int cmp_u32(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}
static int cmp_triple(const void* a, const void* b) {
  const triple* x = a;
  const triple* y = b;
  if (x->q != y->q) return x->q < y->q ? -1 : 1;
  return x->s < y->s ? -1 : x->s > y->s;
}

typedef struct {
  void* p;
  size_t n, cap, elem;
} vec;
static void vec_push(vec* v, const void* x) {
  if (v->n == v->cap) {
    v->cap = v->cap ? 2 * v->cap : 1024;
    v->p = realloc(v->p, v->cap * v->elem);
  }
  memcpy((char*)v->p + v->n * v->elem, x, v->elem);
  v->n++;
}

/* proj/src/sampler.cpp:77-247 (exact backend; inline sums are the same
 * Kahan loop as the estimator, proj/src/sampler.cpp:34-45). */
int oracle_sample_counted(const double* pts, uint32_t n, uint32_t d,
                          int family, double sigma, const uint32_t* queries,
                          size_t nq, uint32_t rounds, uint64_t seed,
                          uint32_t** out, size_t* count, oracle_diag* diag,
                          uint32_t** rec_first, uint32_t** rec_last,
                          uint32_t** rec_query, double** rec_sum,
                          size_t* rec_count) {
  if (rounds == 0) return 2; /* :85 */
  for (size_t i = 0; i < nq; ++i)
    if (queries[i] >= n) return 2; /* :86-87 */

  /* :89-106 merge duplicate queries, ascending query order */
  uint32_t* sq = malloc(sizeof(uint32_t) * (nq ? nq : 1));
  memcpy(sq, queries, sizeof(uint32_t) * nq);
  qsort(sq, nq, sizeof(uint32_t), cmp_u32);
  entry* cur = malloc(sizeof(entry) * (nq ? nq : 1));
  size_t ncur = 0;
  for (size_t i = 0; i < nq;) {
    size_t j = i;
    while (j < nq && sq[j] == sq[i]) ++j;
    uint64_t t = (uint64_t)(j - i) * rounds;
    if (t > 0xffffffffULL) {
      free(sq);
      free(cur);
      return 2;
    }
    entry e = {0, n, sq[i], (uint32_t)t};
    cur[ncur++] = e;
    i = j;
  }
  free(sq);

  const int record = rec_first != NULL;
  vec rf = {0, 0, 0, 4}, rl = {0, 0, 0, 4}, rq = {0, 0, 0, 4},
      rs = {0, 0, 0, 8};
  vec res = {0, 0, 0, sizeof(triple)};
  if (diag) memset(diag, 0, sizeof(*diag));

  while (ncur > 0) { /* :117 one iteration per tree level */
    if (diag && diag->nlevels < 64) {
      uint64_t tk = 0;
      for (size_t i = 0; i < ncur; ++i) tk += cur[i].tickets;
      diag->entries_per_level[diag->nlevels] = ncur;
      diag->tickets_per_level[diag->nlevels] = tk;
      diag->nlevels++;
    }
    double* g1 = calloc(ncur, sizeof(double));
    double* g2 = calloc(ncur, sizeof(double));

    /* pass 1 (:129-182): child sums per node group */
    for (size_t i = 0; i < ncur;) {
      size_t j = i;
      while (j < ncur && cur[j].first == cur[i].first &&
             cur[j].last == cur[i].last)
        ++j;
      uint32_t first = cur[i].first, last = cur[i].last;
      uint32_t size = last - first;
      if (size > 1) {
        uint32_t mid = first + size / 2;
#pragma omp parallel for schedule(dynamic, 16)
        for (size_t t = i; t < j; ++t) {
          const double* y = pts + (size_t)cur[t].query * d;
          double a = kahan_range(pts, d, family, sigma, first, mid, y);
          double b = kahan_range(pts, d, family, sigma, mid, last, y);
          g1[t] = a > SUM_FLOOR ? a : SUM_FLOOR;
          g2[t] = b > SUM_FLOOR ? b : SUM_FLOOR;
        }
        if (record) {
          for (int side = 0; side < 2; ++side)
            for (size_t t = i; t < j; ++t) {
              uint32_t f = side ? mid : first, l = side ? last : mid;
              vec_push(&rf, &f);
              vec_push(&rl, &l);
              vec_push(&rq, &cur[t].query);
              vec_push(&rs, side ? &g2[t] : &g1[t]);
            }
        }
      }
      i = j;
    }

    /* pass 2 (:186-225): route tickets; children of one node stay grouped,
     * left children before right children. */
    entry* next = malloc(sizeof(entry) * (2 * ncur));
    entry* rbuf = malloc(sizeof(entry) * (ncur ? ncur : 1));
    size_t nnext = 0;
    for (size_t i = 0; i < ncur;) {
      size_t j = i;
      while (j < ncur && cur[j].first == cur[i].first &&
             cur[j].last == cur[i].last)
        ++j;
      uint32_t first = cur[i].first, last = cur[i].last;
      uint32_t size = last - first;
      if (size == 1) {
        for (size_t t = i; t < j; ++t) {
          triple tr = {cur[t].query, first, cur[t].tickets};
          vec_push(&res, &tr);
        }
      } else {
        uint32_t mid = first + size / 2;
        size_t nr = 0;
        for (size_t t = i; t < j; ++t) {
          double a = g1[t], b = g2[t], p;
          if (a <= SUM_FLOOR && b <= SUM_FLOOR) {
            p = 0.5;
            if (diag) diag->degenerate_draws += cur[t].tickets;
          } else {
            p = a / (a + b);
          }
          uint64_t key = oracle_rng_key(
              seed, ROUTE_TAG, ((uint64_t)first << 32) | last, cur[t].query);
          uint32_t to_left = (uint32_t)oracle_binomial(key, cur[t].tickets, p);
          if (to_left > 0) {
            entry e = {first, mid, cur[t].query, to_left};
            next[nnext++] = e;
          }
          if (to_left < cur[t].tickets) {
            entry e = {mid, last, cur[t].query, cur[t].tickets - to_left};
            rbuf[nr++] = e;
          }
        }
        memcpy(next + nnext, rbuf, nr * sizeof(entry));
        nnext += nr;
      }
      i = j;
    }
    free(rbuf);
    free(g1);
    free(g2);
    free(cur);
    cur = next;
    ncur = nnext;
  }
  free(cur);

  qsort(res.p, res.n, sizeof(triple), cmp_triple); /* :241-246 */
  *out = malloc(sizeof(uint32_t) * 3 * (res.n ? res.n : 1));
  memcpy(*out, res.p, sizeof(triple) * res.n);
  *count = res.n;
  free(res.p);
  if (record) {
    *rec_first = rf.p;
    *rec_last = rl.p;
    *rec_query = rq.p;
    *rec_sum = rs.p;
    *rec_count = rs.n;
  }
  return 0;
}

/* proj/src/sparsifier.cpp:51-142 (exact backend). */
int oracle_build_graph(const double* pts, uint32_t n, uint32_t d, int family,
                       double sigma, uint32_t rounds, uint64_t seed,
                       size_t* m, uint32_t** u, uint32_t** v, double** w,
                       double** degrees, double** estimates, double* g_full_out,
                       double* report) {
  if (n < 2) return 2;            /* :56 TooFewPoints */
  if (!(sigma > 0.0)) return 2;   /* proj/src/kernel.cpp:23-26 */
  uint32_t L;
  if (oracle_rounds_for(n, 1.0, 1.0, rounds, 0, &L)) return 2; /* :57 */

  uint32_t* all = malloc(sizeof(uint32_t) * n);
  for (uint32_t i = 0; i < n; ++i) all[i] = i;
  uint32_t* tri;
  size_t ntri;
  oracle_diag diag;
  int rc = oracle_sample_counted(pts, n, d, family, sigma, all, n, L, seed,
                                 &tri, &ntri, &diag, NULL, NULL, NULL, NULL,
                                 NULL); /* :70 */
  if (rc) {
    free(all);
    return rc;
  }
  double* g_full = malloc(sizeof(double) * n); /* :74-75 */
  oracle_kde_exact(pts, n, d, family, sigma, 0, n, all, n, SUM_FLOOR, g_full);
  free(all);

  /* :78-92 collapse directions and multiplicities */
  uint64_t* pairs = malloc(sizeof(uint64_t) * (ntri ? ntri : 1));
  size_t np = 0, self_pairs = 0;
  for (size_t i = 0; i < ntri; ++i) {
    uint32_t q = tri[3 * i], s = tri[3 * i + 1], c = tri[3 * i + 2];
    if (q == s) {
      self_pairs += c;
      continue;
    }
    uint32_t a = q < s ? q : s, b = q < s ? s : q;
    pairs[np++] = ((uint64_t)a << 32) | b;
  }
  free(tri);
  qsort(pairs, np, sizeof(uint64_t), cmp_u64);
  size_t nu = 0;
  for (size_t i = 0; i < np; ++i)
    if (nu == 0 || pairs[nu - 1] != pairs[i]) pairs[nu++] = pairs[i];

  /* :100-117 weighting */
  uint32_t* uu = malloc(sizeof(uint32_t) * (nu ? nu : 1));
  uint32_t* vv = malloc(sizeof(uint32_t) * (nu ? nu : 1));
  double* ww = malloc(sizeof(double) * (nu ? nu : 1));
  double* est = estimates ? malloc(sizeof(double) * 8 * (nu ? nu : 1)) : NULL;
  size_t ne = 0, underflow = 0;
  const double Lf = (double)L;
  for (size_t k = 0; k < nu; ++k) {
    uint32_t i = (uint32_t)(pairs[k] >> 32), j = (uint32_t)pairs[k];
    double kij = oracle_kernel(family, sigma, pts + (size_t)i * d,
                               pts + (size_t)j * d, d);
    if (!(kij >= 1e-300)) {
      ++underflow;
      continue;
    }
    double pi = Lf * kij / g_full[i];
    double pj = Lf * kij / g_full[j];
    if (pi > 1.0) pi = 1.0;
    if (pj > 1.0) pj = 1.0;
    double ph = pi + pj - pi * pj;
    uu[ne] = i;
    vv[ne] = j;
    ww[ne] = kij / ph;
    if (est) {
      double row[8] = {i, j, kij, g_full[i], g_full[j], pi, pj, ph};
      memcpy(est + 8 * ne, row, sizeof(row));
    }
    ++ne;
  }
  free(pairs);
  if (ne > (size_t)n * L) { /* :120-121 NumericError */
    free(uu);
    free(vv);
    free(ww);
    free(est);
    free(g_full);
    return 4;
  }
  /* proj/src/graph.cpp:14-21 degrees in edge order */
  double* deg = calloc(n, sizeof(double));
  double total = 0.0;
  for (size_t k = 0; k < ne; ++k) {
    deg[uu[k]] += ww[k];
    deg[vv[k]] += ww[k];
    total += ww[k];
  }
  *m = ne;
  *u = uu;
  *v = vv;
  *w = ww;
  if (degrees)
    *degrees = deg;
  else
    free(deg);
  if (estimates) *estimates = est;
  if (g_full_out) memcpy(g_full_out, g_full, sizeof(double) * n);
  free(g_full);
  if (report) {
    report[0] = n;
    report[1] = L;
    report[2] = (double)ntri;
    report[3] = (double)self_pairs;
    report[4] = (double)underflow;
    report[5] = (double)ne;
    report[6] = (double)diag.degenerate_draws;
    report[7] = total;
  }
  return 0;
}
