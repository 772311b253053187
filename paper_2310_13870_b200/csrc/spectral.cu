// Spectral clustering on the device graph: the
// consumer of the similarity graph and the pipeline of the ARI parity check.
//
// Restates proj/src/spectral.cpp:40-419 (deflated thick-restart Lanczos on
// the normalised Laplacian, row-normalised embedding, k-means++ + Lloyd)
// with the n-length work on the device:
//   * N x = x - D^-1/2 A D^-1/2 x as a warp-per-row SpMV over the graph's
//     upper CSR plus its transpose (built once by a radix sort), so every
//     row's sum has a fixed order (graph.cpp:160-188 uses 32 edge blocks);
//   * the Lanczos basis V (n x (m+1) fp64) stays in HBM; reorthogonalisation
//     is two classical Gram-Schmidt passes per step (block dots + one update
//     kernel) where the reference runs modified Gram-Schmidt, each followed
//     by projecting out the known zero eigenspace (one D^1/2 indicator per
//     connected component, components by hooking + pointer jumping);
//   * only the m x m projected matrix T is on the host (cyclic Jacobi, m is
//     40 by default), as the reference keeps it in an Eigen matrix;
//   * k-means runs its assignment, seeding scans and per-cluster sums as
//     kernels with fixed reduction orders; its few sequential random draws
//     use the reference's RngStream on the host, so seeds select the same
//     restarts.
// Start vectors use the reference's keyed normal stream (rng.hpp:47-62)
// evaluated per element on the device.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_reduce.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "engine.cuh"
#include "spectral.cuh"

namespace fsgg {
namespace {

constexpr uint64_t kLanczosTag = 0x9d3f1c6a24b8e705ULL;  // spectral.cpp:90
constexpr uint64_t kKmeansTag = 0x6b6d65616e732b2bULL;   // spectral.cpp:296
constexpr uint64_t kSpectralSeedTag = 0x73706563747261ULL;  // spectral.cpp:411
constexpr int kDotBlocks = 296;                           // 2 x 148 SMs
constexpr uint32_t kMaxK = 64;

// proj/include/fsg/rng.hpp:18-44 (host side: the handful of sequential draws)
struct HostRng {
  uint64_t key = 0, counter = 0;
  static HostRng keyed(uint64_t seed, uint64_t tag, uint64_t a = 0, uint64_t b = 0) {
    uint64_t k = splitmix64(seed);
    k = splitmix64(k ^ splitmix64(tag ^ 0x6a09e667f3bcc909ULL));
    k = splitmix64(k ^ splitmix64(a ^ 0xbb67ae8584caa73bULL));
    k = splitmix64(k ^ splitmix64(b ^ 0x3c6ef372fe94f82bULL));
    HostRng r;
    r.key = k;
    return r;
  }
  uint64_t next_u64() { return splitmix64(key + counter++); }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  uint64_t next_below(uint64_t n) {
    if (n <= 1) return 0;
    const uint64_t threshold = -n % n;
    for (;;) {
      const uint64_t r = next_u64();
      if (r >= threshold) return r % n;
    }
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

template <class F>
void cub_call(DevBuf& tmp, cudaStream_t s, F&& f) {
  size_t bytes = 0;
  FSGG_CUDA(f(static_cast<void*>(nullptr), bytes));
  tmp.ensure(bytes + 16, s);
  FSGG_CUDA(f(tmp.as<void>(), bytes));
}

// ---- kernels ---------------------------------------------------------------

__global__ void lower_keys_kernel(uint32_t n, const uint64_t* __restrict__ rp,
                                  const uint32_t* __restrict__ col, uint64_t m,
                                  unsigned long long* __restrict__ keys) {
  // one thread per row u: keys (v << 32 | u) for its upper entries
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  for (uint64_t e = rp[u]; e < rp[u + 1]; ++e)
    keys[e] = (static_cast<unsigned long long>(col[e]) << 32) | u;
}

__global__ void lower_split_kernel(const unsigned long long* __restrict__ keys, uint64_t m,
                                   uint32_t* __restrict__ lcol, uint32_t* __restrict__ lrow) {
  const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (e >= m) return;
  lcol[e] = uint32_t(keys[e]);
  lrow[e] = uint32_t(keys[e] >> 32);
}

__global__ void row_ptr_from_rows_kernel(const uint32_t* __restrict__ rows, uint64_t m,
                                         uint32_t n, uint64_t* __restrict__ rp) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x > n) return;
  uint64_t lo = 0, hi = m;  // first e with rows[e] >= x
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (rows[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  rp[x] = lo;
}

// NormalizedLaplacian ctor (graph.cpp:150-158): 1/sqrt(d), first isolated v.
__global__ void inv_sqrt_kernel(uint32_t n, const double* __restrict__ deg,
                                double* __restrict__ inv, unsigned int* __restrict__ first_bad) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const double d = deg[v];
  if (!(d > 0.0)) {
    atomicMin(first_bad, v);
    inv[v] = 0.0;
  } else {
    inv[v] = 1.0 / sqrt(d);
  }
}

// y = x - inv .* (A (inv .* x)), one warp per row over upper + lower CSR.
__global__ void lap_apply_kernel(uint32_t n, const uint64_t* __restrict__ rp,
                                 const uint32_t* __restrict__ col, const double* __restrict__ w,
                                 const uint64_t* __restrict__ lrp,
                                 const uint32_t* __restrict__ lcol,
                                 const double* __restrict__ lw, const double* __restrict__ inv,
                                 const double* __restrict__ x, double* __restrict__ y) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  double s = 0.0;
  for (uint64_t e = lrp[row] + lane; e < lrp[row + 1]; e += 32) {
    const uint32_t c = lcol[e];
    s = fma(lw[e], inv[c] * x[c], s);
  }
  for (uint64_t e = rp[row] + lane; e < rp[row + 1]; e += 32) {
    const uint32_t c = col[e];
    s = fma(w[e], inv[c] * x[c], s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = x[row] - inv[row] * s;
}

// partial[i][b] = sum over block b's rows of V[i][r] * x[r], i < J.
__global__ void coldots_kernel(const double* __restrict__ V, uint64_t ld, uint32_t n,
                               const double* __restrict__ x, double* __restrict__ partial) {
  __shared__ double red[32];
  const uint32_t i = blockIdx.y;
  const double* vi = V + i * ld;
  double s = 0.0;
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
    s = fma(vi[r], x[r], s);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) partial[size_t(i) * gridDim.x + blockIdx.x] = s;
  }
}

// out[i] = sum_b partial[i][b] (fixed order), optionally negated.
__global__ void reduce_partials_kernel(const double* __restrict__ partial, uint32_t nb,
                                       double* __restrict__ out) {
  __shared__ double red[32];
  const uint32_t i = blockIdx.x;
  double s = 0.0;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) s += partial[size_t(i) * nb + b];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) out[i] = s;
  }
}

// x[r] -= sum_{i<J} h[i] * V[i][r]
__global__ void sub_combo_kernel(const double* __restrict__ V, uint64_t ld, uint32_t n,
                                 uint32_t J, const double* __restrict__ h,
                                 double* __restrict__ x) {
  __shared__ double sh[128];
  for (uint32_t i = threadIdx.x; i < J; i += blockDim.x) sh[i] = h[i];
  __syncthreads();
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double acc = x[r];
  for (uint32_t i = 0; i < J; ++i) acc = fma(-sh[i], V[i * ld + r], acc);
  x[r] = acc;
}

__global__ void scale_copy_kernel(uint32_t n, double s, const double* __restrict__ x,
                                  double* __restrict__ y) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) y[r] = s * x[r];
}

// Y[c][r] = sum_k V[k][r] * S[k][c] (S: m x keep, column-major)
__global__ void ritz_kernel(const double* __restrict__ V, uint64_t ld, uint32_t n, uint32_t m,
                            const double* __restrict__ S, uint32_t keep,
                            double* __restrict__ Y) {
  extern __shared__ double sS[];
  for (uint32_t i = threadIdx.x; i < m * keep; i += blockDim.x) sS[i] = S[i];
  __syncthreads();
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (uint32_t c = 0; c < keep; ++c) {
    double acc = 0.0;
    for (uint32_t k = 0; k < m; ++k) acc = fma(V[k * ld + r], sS[c * m + k], acc);
    Y[c * ld + r] = acc;
  }
}

// Normals #g0 .. #g0+n-1 of RngStream(key).next_normal() (rng.hpp:47-62):
// pair p draws u1 = counter 2p, u2 = counter 2p + 1; even = r cos, odd = r sin.
__global__ void normals_kernel(uint64_t key, uint64_t g0, uint32_t n, double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t g = g0 + i, p = g >> 1;
  const double u1 = static_cast<double>(splitmix64(key + 2 * p) >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(splitmix64(key + 2 * p + 1) >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double a = 6.283185307179586476925286766559 * u2;
  out[i] = (g & 1) ? r * sin(a) : r * cos(a);
}

// ---- connected components (graph.cpp:191-230) ------------------------------
__device__ __forceinline__ uint32_t cc_find(const uint32_t* parent, uint32_t x) {
  uint32_t p = parent[x];
  while (p != x) {
    x = p;
    p = parent[x];
  }
  return x;
}

__global__ void cc_init_kernel(uint32_t n, uint32_t* parent) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) parent[v] = v;
}

__global__ void cc_hook_kernel(uint32_t n, const uint64_t* __restrict__ rp,
                               const uint32_t* __restrict__ col, uint32_t* parent,
                               int* changed) {
  const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  for (uint64_t e = rp[u]; e < rp[u + 1]; ++e) {
    uint32_t a = cc_find(parent, u), b = cc_find(parent, col[e]);
    if (a == b) continue;
    const uint32_t hi = max(a, b), lo = min(a, b);
    atomicMin(parent + hi, lo);
    *changed = 1;
  }
}

__global__ void cc_jump_kernel(uint32_t n, uint32_t* parent) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) parent[v] = cc_find(parent, v);
}

__global__ void cc_flags_kernel(uint32_t n, const uint32_t* __restrict__ root,
                                uint32_t* __restrict__ flag) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) flag[v] = root[v] == v ? 1u : 0u;
}

__global__ void cc_label_kernel(uint32_t n, const uint32_t* __restrict__ root,
                                const uint32_t* __restrict__ id, uint32_t* __restrict__ comp) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) comp[v] = id[root[v]];
}

__global__ void iota_kernel(uint32_t n, uint32_t* x) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) x[v] = v;
}

__global__ void gather_kernel(uint32_t n, const uint32_t* __restrict__ perm,
                              const double* __restrict__ a, const double* __restrict__ b,
                              double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t v = perm[i];
  out[i] = b ? a[v] * b[v] : a[v];
}

__global__ void basis_kernel(uint32_t n, const double* __restrict__ deg,
                             const uint32_t* __restrict__ comp, const double* __restrict__ vol,
                             double* __restrict__ basis) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) basis[v] = sqrt(deg[v] / vol[comp[v]]);
}

// vec -= dots[comp] * basis  (components have disjoint supports)
__global__ void project_kernel(uint32_t n, const uint32_t* __restrict__ comp,
                               const double* __restrict__ dots,
                               const double* __restrict__ basis, double* __restrict__ vec) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) vec[v] = fma(-dots[comp[v]], basis[v], vec[v]);
}

__global__ void indicator_kernel(uint32_t n, uint32_t c, const uint32_t* __restrict__ comp,
                                 const double* __restrict__ basis, double* __restrict__ out) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v < n) out[v] = comp[v] == c ? basis[v] : 0.0;
}

// spectral_embed (spectral.cpp:225-242)
__global__ void embed_kernel(uint32_t n, uint32_t k, const double* __restrict__ vecs,
                             uint64_t ld, double* __restrict__ rows) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  double norm = 0.0;
  for (uint32_t c = 0; c < k; ++c) {
    const double x = vecs[c * ld + v];
    norm += x * x;
  }
  const double inv = norm > 0.0 ? 1.0 / sqrt(norm) : 1.0;
  for (uint32_t c = 0; c < k; ++c) rows[size_t(v) * k + c] = norm > 0.0 ? vecs[c * ld + v] * inv
                                                                          : vecs[c * ld + v];
}

// ---- k-means kernels (spectral.cpp:257-403) --------------------------------
__device__ __forceinline__ double row_dist2(const double* a, const double* b, uint32_t d) {
  double s = 0.0;
  for (uint32_t i = 0; i < d; ++i) {
    const double t = a[i] - b[i];
    s += t * t;
  }
  return s;
}

__global__ void km_d2_kernel(uint32_t n, uint32_t dim, const double* __restrict__ pts,
                             const double* __restrict__ center, int init,
                             double* __restrict__ d2) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double dd = row_dist2(pts + size_t(i) * dim, center, dim);
  d2[i] = init ? dd : fmin(d2[i], dd);
}

// first i with d2[i] > 0 and prefix[i] >= r (spectral.cpp:307-316)
__global__ void km_pick_kernel(uint32_t n, const double* __restrict__ d2,
                               const double* __restrict__ prefix, double r,
                               unsigned int* __restrict__ pick) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && d2[i] > 0.0 && prefix[i] >= r) atomicMin(pick, i);
}

// first index of the maximum of d2 over points whose cluster keeps > 1
// member (mask null: all points)
__global__ void km_argmax_kernel(uint32_t n, const double* __restrict__ d2,
                                 const uint32_t* __restrict__ labels,
                                 const uint32_t* __restrict__ counts, double best,
                                 unsigned int* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (counts && counts[labels[i]] <= 1) return;
  if (d2[i] == best) atomicMin(idx, i);
}

__global__ void km_masked_kernel(uint32_t n, const double* __restrict__ d2,
                                 const uint32_t* __restrict__ labels,
                                 const uint32_t* __restrict__ counts,
                                 double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = (counts && counts[labels[i]] <= 1) ? -1.0 : d2[i];
}

__global__ void km_assign_kernel(uint32_t n, uint32_t dim, uint32_t k,
                                 const double* __restrict__ pts,
                                 const double* __restrict__ centers,
                                 uint32_t* __restrict__ labels, double* __restrict__ d2,
                                 uint32_t* __restrict__ counts) {
  extern __shared__ double sc[];
  for (uint32_t i = threadIdx.x; i < k * dim; i += blockDim.x) sc[i] = centers[i];
  __syncthreads();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* p = pts + size_t(i) * dim;
  uint32_t bestc = 0;
  double bestd = row_dist2(p, sc, dim);
  for (uint32_t c = 1; c < k; ++c) {
    const double dd = row_dist2(p, sc + c * dim, dim);
    if (dd < bestd) {
      bestd = dd;
      bestc = c;
    }
  }
  labels[i] = bestc;
  d2[i] = bestd;
  atomicAdd(counts + bestc, 1u);
}

// Per-chunk per-(cluster, coord) sums and cost, each accumulated in point
// order by one thread: partial[b][k*dim + 1].
constexpr uint32_t kKmChunk = 1024;
__global__ void km_sums_kernel(uint32_t n, uint32_t dim, uint32_t k,
                               const double* __restrict__ pts,
                               const uint32_t* __restrict__ labels,
                               const double* __restrict__ d2, double* __restrict__ partial) {
  __shared__ uint32_t sl[kKmChunk];
  const uint32_t i0 = blockIdx.x * kKmChunk, i1 = min(n, i0 + kKmChunk);
  for (uint32_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) sl[i - i0] = labels[i];
  __syncthreads();
  const uint32_t W = k * dim + 1;
  for (uint32_t j = threadIdx.x; j < W; j += blockDim.x) {
    double s = 0.0;
    if (j == W - 1) {
      for (uint32_t i = i0; i < i1; ++i) s += d2[i];
    } else {
      const uint32_t c = j / dim, a = j % dim;
      for (uint32_t i = i0; i < i1; ++i)
        if (sl[i - i0] == c) s += pts[size_t(i) * dim + a];
    }
    partial[size_t(blockIdx.x) * W + j] = s;
  }
}

__global__ void km_sums_reduce_kernel(uint32_t nb, uint32_t W, const double* __restrict__ partial,
                                      double* __restrict__ out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= W) return;
  double s = 0.0;
  for (uint32_t b = 0; b < nb; ++b) s += partial[size_t(b) * W + j];
  out[j] = s;
}

// ---- host helpers ----------------------------------------------------------

// Symmetric eigen-decomposition of the small projected matrix by cyclic
// Jacobi rotations: eigenvalues ascending, unit eigenvectors in columns
// (the contract of Eigen::SelfAdjointEigenSolver used at spectral.cpp:166).
void sym_eigen(const std::vector<double>& Tin, uint32_t m, std::vector<double>& vals,
               std::vector<double>& vecs) {
  std::vector<double> A = Tin, V(size_t(m) * m, 0.0);
  auto a = [&](uint32_t i, uint32_t j) -> double& { return A[size_t(j) * m + i]; };
  auto v = [&](uint32_t i, uint32_t j) -> double& { return V[size_t(j) * m + i]; };
  for (uint32_t i = 0; i < m; ++i) v(i, i) = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (uint32_t j = 0; j < m; ++j)
      for (uint32_t i = 0; i < m; ++i) (i == j ? diag : off) += a(i, j) * a(i, j);
    if (off == 0.0 || off <= 1e-30 * diag) break;
    for (uint32_t p = 0; p < m; ++p)
      for (uint32_t q = p + 1; q < m; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) /
                         (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (uint32_t k = 0; k < m; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (uint32_t k = 0; k < m; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
        for (uint32_t k = 0; k < m; ++k) {
          const double vkp = v(k, p), vkq = v(k, q);
          v(k, p) = c * vkp - s * vkq;
          v(k, q) = s * vkp + c * vkq;
        }
      }
  }
  std::vector<uint32_t> order(m);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t x, uint32_t y) { return a(x, x) < a(y, y); });
  vals.assign(m, 0.0);
  vecs.assign(size_t(m) * m, 0.0);
  for (uint32_t j = 0; j < m; ++j) {
    vals[j] = a(order[j], order[j]);
    for (uint32_t i = 0; i < m; ++i) vecs[size_t(j) * m + i] = v(i, order[j]);
  }
}

inline uint32_t blocks(uint64_t n, uint32_t t = 256) { return ceil_div_u32(n, t); }

// Device state of one normalised Laplacian.
struct Laplacian {
  const SpectralGraphView& g;
  cudaStream_t s;
  uint32_t n;
  DevBuf lrp, lcol, lw, inv, comp, basis, perm, seg, dots, partial, hbuf, tmp, scratch;
  uint32_t ncomp = 0;
  uint64_t launches = 0;

  Laplacian(const SpectralGraphView& gv, cudaStream_t st) : g(gv), s(st), n(gv.n) {}

  void build() {
    const uint64_t m = g.m;
    // inverse square-root degrees; isolated vertices are rejected
    inv.alloc(size_t(n) * 8, s);
    DevBuf bad(4, s);
    FSGG_CUDA(cudaMemsetAsync(bad.as<void>(), 0xff, 4, s));
    inv_sqrt_kernel<<<blocks(n), 256, 0, s>>>(n, g.degrees, inv.as<double>(),
                                              bad.as<unsigned int>());
    FSGG_LAUNCH_CHECK();
    unsigned int first_bad = 0;
    FSGG_CUDA(cudaMemcpyAsync(&first_bad, bad.as<void>(), 4, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    if (first_bad != 0xffffffffu)  // graph.cpp:154-155 (IsolatedVertex)
      throw ConfigError("vertex " + std::to_string(first_bad) + " has degree 0");

    // transposed (lower) CSR: rows v, columns u ascending
    lrp.alloc(size_t(n + 1) * 8, s);
    lcol.alloc(std::max<uint64_t>(m, 1) * 4, s);
    lw.alloc(std::max<uint64_t>(m, 1) * 8, s);
    if (m) {
      DevBuf k1(m * 8, s), k2(m * 8, s), w2(m * 8, s), rows(m * 4, s);
      lower_keys_kernel<<<blocks(n), 256, 0, s>>>(n, g.row_ptr, g.col, m,
                                                  k1.as<unsigned long long>());
      FSGG_LAUNCH_CHECK();
      FSGG_CUDA(cudaMemcpyAsync(lw.as<void>(), g.w, m * 8, cudaMemcpyDeviceToDevice, s));
      cub::DoubleBuffer<unsigned long long> dk(k1.as<unsigned long long>(),
                                               k2.as<unsigned long long>());
      cub::DoubleBuffer<double> dv(lw.as<double>(), w2.as<double>());
      cub_call(tmp, s, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, m, 0, 64, s);
      });
      if (dv.Current() != lw.as<double>())
        FSGG_CUDA(cudaMemcpyAsync(lw.as<void>(), dv.Current(), m * 8, cudaMemcpyDeviceToDevice, s));
      lower_split_kernel<<<blocks(m), 256, 0, s>>>(dk.Current(), m, lcol.as<uint32_t>(),
                                                   rows.as<uint32_t>());
      FSGG_LAUNCH_CHECK();
      row_ptr_from_rows_kernel<<<blocks(uint64_t(n) + 1), 256, 0, s>>>(
          rows.as<uint32_t>(), m, n, lrp.as<uint64_t>());
      FSGG_LAUNCH_CHECK();
      FSGG_CUDA(cudaStreamSynchronize(s));
      launches += 4;
    } else {
      FSGG_CUDA(cudaMemsetAsync(lrp.as<void>(), 0, size_t(n + 1) * 8, s));
    }
    build_components();
  }

  // Components labelled in order of their smallest vertex, exactly as the
  // reference's union-find + first-occurrence remap (graph.cpp:215-228).
  void build_components() {
    DevBuf parent(size_t(n) * 4, s), flag(size_t(n) * 4, s), id(size_t(n) * 4, s),
        changed(4, s);
    cc_init_kernel<<<blocks(n), 256, 0, s>>>(n, parent.as<uint32_t>());
    FSGG_LAUNCH_CHECK();
    for (int it = 0;; ++it) {
      int h = 0;
      FSGG_CUDA(cudaMemsetAsync(changed.as<void>(), 0, 4, s));
      cc_hook_kernel<<<blocks(n), 256, 0, s>>>(n, g.row_ptr, g.col, parent.as<uint32_t>(),
                                               changed.as<int>());
      FSGG_LAUNCH_CHECK();
      cc_jump_kernel<<<blocks(n), 256, 0, s>>>(n, parent.as<uint32_t>());
      FSGG_LAUNCH_CHECK();
      FSGG_CUDA(cudaMemcpyAsync(&h, changed.as<void>(), 4, cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      launches += 2;
      if (!h) break;
      if (it > 64 + 2 * 32) throw NumericError("connected components did not converge");
    }
    cc_flags_kernel<<<blocks(n), 256, 0, s>>>(n, parent.as<uint32_t>(), flag.as<uint32_t>());
    FSGG_LAUNCH_CHECK();
    cub_call(tmp, s, [&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, flag.as<uint32_t>(), id.as<uint32_t>(), n, s);
    });
    uint32_t last_flag = 0, last_id = 0;
    FSGG_CUDA(cudaMemcpyAsync(&last_flag, flag.as<uint32_t>() + n - 1, 4,
                              cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaMemcpyAsync(&last_id, id.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, s));
    comp.alloc(size_t(n) * 4, s);
    cc_label_kernel<<<blocks(n), 256, 0, s>>>(n, parent.as<uint32_t>(), id.as<uint32_t>(),
                                              comp.as<uint32_t>());
    FSGG_LAUNCH_CHECK();
    FSGG_CUDA(cudaStreamSynchronize(s));
    ncomp = last_id + last_flag;

    // vertices grouped by component (stable: ascending v inside each), and
    // segment offsets, for per-component reductions in vertex order
    perm.alloc(size_t(n) * 4, s);
    seg.alloc(size_t(ncomp + 1) * 8, s);
    {
      DevBuf keys2(size_t(n) * 4, s), vals(size_t(n) * 4, s), vals2(size_t(n) * 4, s);
      iota_kernel<<<blocks(n), 256, 0, s>>>(n, vals.as<uint32_t>());
      FSGG_LAUNCH_CHECK();
      FSGG_CUDA(cudaMemcpyAsync(flag.as<void>(), comp.as<void>(), size_t(n) * 4,
                                cudaMemcpyDeviceToDevice, s));
      cub::DoubleBuffer<uint32_t> dk(flag.as<uint32_t>(), keys2.as<uint32_t>());
      cub::DoubleBuffer<uint32_t> dv(vals.as<uint32_t>(), vals2.as<uint32_t>());
      int end_bit = 1;
      while (end_bit < 32 && (uint64_t(1) << end_bit) < ncomp) ++end_bit;
      cub_call(tmp, s, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, n, 0, end_bit, s);
      });
      FSGG_CUDA(cudaMemcpyAsync(perm.as<void>(), dv.Current(), size_t(n) * 4,
                                cudaMemcpyDeviceToDevice, s));
      DevBuf segrows(size_t(n) * 4, s);
      FSGG_CUDA(cudaMemcpyAsync(segrows.as<void>(), dk.Current(), size_t(n) * 4,
                                cudaMemcpyDeviceToDevice, s));
      row_ptr_from_rows_kernel<<<blocks(uint64_t(ncomp) + 1), 256, 0, s>>>(
          segrows.as<uint32_t>(), n, ncomp, seg.as<uint64_t>());
      FSGG_LAUNCH_CHECK();
      FSGG_CUDA(cudaStreamSynchronize(s));
    }
    // component volumes (degree sums in vertex order) and the D^1/2 basis
    dots.alloc(size_t(std::max<uint32_t>(ncomp, 128)) * 8, s);
    scratch.alloc(size_t(n) * 8, s);
    DevBuf vol(size_t(ncomp) * 8, s);
    gather_kernel<<<blocks(n), 256, 0, s>>>(n, perm.as<uint32_t>(), g.degrees, nullptr,
                                            scratch.as<double>());
    FSGG_LAUNCH_CHECK();
    seg_sum(scratch.as<double>(), vol.as<double>());
    basis.alloc(size_t(n) * 8, s);
    basis_kernel<<<blocks(n), 256, 0, s>>>(n, g.degrees, comp.as<uint32_t>(), vol.as<double>(),
                                           basis.as<double>());
    FSGG_LAUNCH_CHECK();
    FSGG_CUDA(cudaStreamSynchronize(s));
    partial.alloc(size_t(kDotBlocks) * 128 * 8, s);
    hbuf.alloc(128 * 8, s);
    launches += 8;
  }

  void seg_sum(const double* in, double* out) {
    const uint64_t* off = seg.as<uint64_t>();
    cub_call(tmp, s, [&](void* t, size_t& b) {
      return cub::DeviceSegmentedReduce::Sum(t, b, in, out, int(ncomp), off, off + 1, s);
    });
    launches += 1;
  }

  void apply(const double* x, double* y) {
    lap_apply_kernel<<<blocks(uint64_t(n) * 32), 256, 0, s>>>(
        n, g.row_ptr, g.col, g.w, lrp.as<uint64_t>(), lcol.as<uint32_t>(), lw.as<double>(),
        inv.as<double>(), x, y);
    FSGG_LAUNCH_CHECK();
    launches++;
  }

  // vec -= sum_c (u_c . vec) u_c  (spectral.cpp:93-98)
  void project_out(double* vec) {
    gather_kernel<<<blocks(n), 256, 0, s>>>(n, perm.as<uint32_t>(), basis.as<double>(), vec,
                                            scratch.as<double>());
    FSGG_LAUNCH_CHECK();
    seg_sum(scratch.as<double>(), dots.as<double>());
    project_kernel<<<blocks(n), 256, 0, s>>>(n, comp.as<uint32_t>(), dots.as<double>(),
                                             basis.as<double>(), vec);
    FSGG_LAUNCH_CHECK();
    launches += 2;
  }

  // h[i] = V[i] . x for i < J (device result in hbuf)
  void coldots(const double* V, uint32_t J, const double* x) {
    if (J == 0) return;
    coldots_kernel<<<dim3(kDotBlocks, J), 256, 0, s>>>(V, n, n, x, partial.as<double>());
    FSGG_LAUNCH_CHECK();
    reduce_partials_kernel<<<J, 256, 0, s>>>(partial.as<double>(), kDotBlocks,
                                             hbuf.as<double>());
    FSGG_LAUNCH_CHECK();
    launches += 2;
  }

  double dot(const double* a, const double* b) {
    coldots(a, 1, b);
    double h = 0.0;
    FSGG_CUDA(cudaMemcpyAsync(&h, hbuf.as<void>(), 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    return h;
  }

  double norm2(const double* a) { return std::sqrt(dot(a, a)); }

  // x -= V[:, :J] (V[:, :J]^T x), then the zero eigenspace (one CGS pass)
  void orth_pass(const double* V, uint32_t J, double* x) {
    if (J) {
      coldots(V, J, x);
      sub_combo_kernel<<<blocks(n), 256, 0, s>>>(V, n, n, J, hbuf.as<double>(), x);
      FSGG_LAUNCH_CHECK();
      launches++;
    }
    project_out(x);
  }

  void scale(double a, const double* x, double* y) {
    scale_copy_kernel<<<blocks(n), 256, 0, s>>>(n, a, x, y);
    FSGG_LAUNCH_CHECK();
    launches++;
  }
};

}  // namespace

void smallest_eigenpairs_dev(const SpectralGraphView& g, cudaStream_t s, uint32_t q,
                             const EigenOpts& opts, std::vector<double>& values,
                             std::vector<double>& residuals, DevBuf& vectors,
                             SpectralStats& st) {
  const double t0 = now_s();
  const uint32_t n = g.n;
  if (q == 0 || q > n) throw ConfigError("requested eigenpair count must be in [1, n]");
  if (q > 128) throw ConfigError("at most 128 eigenpairs are supported on the device");
  Laplacian L(g, s);
  L.build();
  const uint32_t ncomp = L.ncomp;
  values.assign(q, 0.0);
  residuals.assign(q, 0.0);
  vectors.alloc(size_t(n) * q * 8, s);
  double* Y = vectors.as<double>();

  // zero eigenspace: D^1/2 indicator per component (spectral.cpp:59-70)
  const uint32_t nzero = std::min(q, ncomp);
  for (uint32_t i = 0; i < nzero; ++i) {
    indicator_kernel<<<blocks(n), 256, 0, s>>>(n, i, L.comp.as<uint32_t>(), L.basis.as<double>(),
                                               Y + size_t(i) * n);
    FSGG_LAUNCH_CHECK();
    L.launches++;
  }
  uint64_t matvecs = 0;
  const uint32_t need = q - nzero;
  if (need > 0) {
    const uint32_t free_dim = n - ncomp;
    if (need > free_dim) throw ConfigError("more eigenpairs requested than the graph has");
    const uint32_t m = opts.max_basis ? std::min(opts.max_basis, free_dim)
                                      : std::min(free_dim, std::max<uint32_t>(2 * need + 24, 40));
    if (m + 1 > 128) throw ConfigError("Lanczos basis larger than 127 is not supported");
    const uint64_t budget = opts.max_matvecs ? opts.max_matvecs : uint64_t(50) * n + 1000;
    DevBuf Vb(size_t(n) * (m + 1) * 8, s), wb(size_t(n) * 8, s), Yb(size_t(n) * m * 8, s),
        Sb(size_t(m) * m * 8, s);
    double* V = Vb.as<double>();
    double* w = wb.as<double>();
    std::vector<double> T(size_t(m) * m, 0.0);
    auto t = [&](uint32_t i, uint32_t j) -> double& { return T[size_t(j) * m + i]; };
    const uint64_t key = HostRng::keyed(opts.seed, kLanczosTag).key;
    uint64_t normal_index = 0;  // position in the stream's normal sequence

    auto reorthogonalize = [&](double* vec, uint32_t upto) {  // spectral.cpp:99-107
      for (int pass = 0; pass < 2; ++pass) {
        L.project_out(vec);
        if (upto) {
          L.coldots(V, upto, vec);
          sub_combo_kernel<<<blocks(n), 256, 0, s>>>(V, n, n, upto, L.hbuf.as<double>(), vec);
          FSGG_LAUNCH_CHECK();
          L.launches++;
        }
      }
    };
    auto random_start = [&](double* vec, uint32_t upto) {  // spectral.cpp:108-120
      for (int attempt = 0; attempt < 32; ++attempt) {
        normals_kernel<<<blocks(n), 256, 0, s>>>(key, normal_index, n, vec);
        FSGG_LAUNCH_CHECK();
        L.launches++;
        normal_index += n;
        reorthogonalize(vec, upto);
        const double nn = L.norm2(vec);
        if (nn > 1e-10) {
          L.scale(1.0 / nn, vec, vec);
          return;
        }
      }
      throw NumericError("cannot seed Lanczos start vector");  // NoConvergence
    };

    uint32_t locked = 0;
    double last_beta = 0.0;
    random_start(V, 0);
    std::vector<double> theta, S;
    for (;;) {
      for (uint32_t j = locked; j < m; ++j) {  // spectral.cpp:126-164
        const double* vj = V + size_t(j) * n;
        L.apply(vj, w);
        ++matvecs;
        L.project_out(w);
        t(j, j) = L.dot(vj, w);
        for (int pass = 0; pass < 2; ++pass) L.orth_pass(V, j + 1, w);
        double beta = L.norm2(w);
        double* vnext = V + size_t(j + 1) * n;
        if (j + 1 < m) {
          if (beta > 1e-13) {
            L.scale(1.0 / beta, w, vnext);
          } else {
            beta = 0.0;
            random_start(vnext, j + 1);
          }
          t(j, j + 1) = beta;
          t(j + 1, j) = beta;
        } else {
          last_beta = beta;
          if (beta > 1e-13) {
            L.scale(1.0 / beta, w, vnext);
          } else {
            last_beta = 0.0;
            FSGG_CUDA(cudaMemsetAsync(vnext, 0, size_t(n) * 8, s));
          }
        }
      }
      sym_eigen(T, m, theta, S);
      auto sv = [&](uint32_t i, uint32_t j) { return S[size_t(j) * m + i]; };
      uint32_t converged = 0;
      for (uint32_t i = 0; i < need; ++i)
        if (std::abs(last_beta * sv(m - 1, i)) <= opts.tol) ++converged;
      if (converged >= need) {  // spectral.cpp:174-182
        FSGG_CUDA(cudaMemcpyAsync(Sb.as<void>(), S.data(), size_t(m) * need * 8,
                                  cudaMemcpyHostToDevice, s));
        ritz_kernel<<<blocks(n), 256, size_t(m) * need * 8, s>>>(V, n, n, m, Sb.as<double>(),
                                                                 need, Y + size_t(nzero) * n);
        FSGG_LAUNCH_CHECK();
        L.launches++;
        for (uint32_t i = 0; i < need; ++i) values[nzero + i] = theta[i];
        break;
      }
      if (matvecs >= budget)  // spectral.cpp:183-188
        throw NumericError("Lanczos: " + std::to_string(converged) + "/" +
                           std::to_string(need) + " pairs converged after " +
                           std::to_string(matvecs) + " matvecs (tol " +
                           std::to_string(opts.tol) + ")");
      // thick restart (spectral.cpp:189-211)
      const uint32_t keep = std::min<uint32_t>(need + 8, m - 2);
      FSGG_CUDA(cudaMemcpyAsync(Sb.as<void>(), S.data(), size_t(m) * keep * 8,
                                cudaMemcpyHostToDevice, s));
      ritz_kernel<<<blocks(n), 256, size_t(m) * keep * 8, s>>>(V, n, n, m, Sb.as<double>(), keep,
                                                               Yb.as<double>());
      FSGG_LAUNCH_CHECK();
      L.launches++;
      // residual direction V[:, m] moves to column keep, Ritz vectors to 0..keep-1
      FSGG_CUDA(cudaMemcpyAsync(V + size_t(keep) * n, V + size_t(m) * n, size_t(n) * 8,
                                cudaMemcpyDeviceToDevice, s));
      FSGG_CUDA(cudaMemcpyAsync(V, Yb.as<void>(), size_t(n) * keep * 8, cudaMemcpyDeviceToDevice,
                                s));
      double* vres = V + size_t(keep) * n;
      if (L.norm2(vres) < 0.5) random_start(vres, keep);
      std::fill(T.begin(), T.end(), 0.0);
      for (uint32_t i = 0; i < keep; ++i) {
        t(i, i) = theta[i];
        const double sc = last_beta * sv(m - 1, i);
        t(i, keep) = sc;
        t(keep, i) = sc;
      }
      locked = keep;
    }
  }
  // true residuals ||N v - lambda v|| (spectral.cpp:214-222)
  {
    DevBuf wb(size_t(n) * 8, s);
    double* w = wb.as<double>();
    for (uint32_t i = 0; i < q; ++i) {
      const double* v = Y + size_t(i) * n;
      L.apply(v, w);
      double h = values[i];
      FSGG_CUDA(cudaMemcpyAsync(L.hbuf.as<void>(), &h, 8, cudaMemcpyHostToDevice, s));
      sub_combo_kernel<<<blocks(n), 256, 0, s>>>(v, n, n, 1, L.hbuf.as<double>(), w);
      FSGG_LAUNCH_CHECK();
      L.launches++;
      residuals[i] = L.norm2(w);
    }
  }
  FSGG_CUDA(cudaStreamSynchronize(s));
  st.matvecs = matvecs;
  st.ncomp = ncomp;
  st.launches += L.launches;
  st.eigen_seconds = now_s() - t0;
}

void kmeans_dev(const double* pts, uint32_t n, uint32_t dim, uint32_t k, const KmeansOpts& opts,
                cudaStream_t s, uint32_t* labels_out, double* cost_out, uint32_t* iters_out,
                SpectralStats& st) {
  const double t0 = now_s();
  if (n == 0 || dim == 0) throw ConfigError("empty k-means input");
  if (k == 0 || k > n) throw ConfigError("k must be in [1, n]");
  if (k > kMaxK || size_t(k) * dim > 4096)
    throw ConfigError("device k-means supports k <= 64 and k * dim <= 4096");
  {  // fewer than k distinct rows -> DegenerateInput (spectral.cpp:265-272)
    std::set<std::string> distinct;
    std::vector<double> rows;
    const uint32_t chunk = 65536;
    for (uint32_t i0 = 0; i0 < n && distinct.size() < k; i0 += chunk) {
      const uint32_t c = std::min(chunk, n - i0);
      rows.resize(size_t(c) * dim);
      FSGG_CUDA(cudaMemcpyAsync(rows.data(), pts + size_t(i0) * dim, size_t(c) * dim * 8,
                                cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      for (uint32_t i = 0; i < c && distinct.size() < k; ++i)
        distinct.emplace(reinterpret_cast<const char*>(rows.data() + size_t(i) * dim),
                         dim * sizeof(double));
    }
    if (distinct.size() < k)
      throw NumericError("fewer than k distinct rows in k-means input");
  }
  uint64_t launches = 0;
  const uint32_t W = k * dim + 1;
  const uint32_t nb = ceil_div_u32(n, kKmChunk);
  DevBuf centers(size_t(k) * dim * 8, s), d2(size_t(n) * 8, s), prefix(size_t(n) * 8, s),
      labels(size_t(n) * 4, s), best_labels(size_t(n) * 4, s), counts(size_t(k) * 4, s),
      partial(size_t(nb) * W * 8, s), sums(size_t(W) * 8, s), pick(4, s), tmp, red(8, s),
      masked(size_t(n) * 8, s);
  std::vector<double> hcenters(size_t(k) * dim), hsums(W);
  std::vector<uint32_t> hcounts(k);
  double best_cost = -1.0;
  uint32_t best_iters = 0;

  auto copy_center = [&](uint32_t c, uint32_t row) {
    FSGG_CUDA(cudaMemcpyAsync(centers.as<double>() + size_t(c) * dim, pts + size_t(row) * dim,
                              dim * 8, cudaMemcpyDeviceToDevice, s));
  };
  auto d2_update = [&](uint32_t c, int init) {
    km_d2_kernel<<<blocks(n), 256, 0, s>>>(n, dim, pts, centers.as<double>() + size_t(c) * dim,
                                           init, d2.as<double>());
    FSGG_LAUNCH_CHECK();
    launches++;
  };
  // first index of the maximum of d2 (optionally among points whose cluster
  // keeps more than one member); UINT32_MAX when there is none
  auto first_argmax = [&](const uint32_t* cnt) -> uint32_t {
    km_masked_kernel<<<blocks(n), 256, 0, s>>>(n, d2.as<double>(), labels.as<uint32_t>(), cnt,
                                               masked.as<double>());
    FSGG_LAUNCH_CHECK();
    cub_call(tmp, s, [&](void* t, size_t& b) {
      return cub::DeviceReduce::Max(t, b, masked.as<double>(), red.as<double>(), n, s);
    });
    double best = 0.0;
    FSGG_CUDA(cudaMemcpyAsync(&best, red.as<void>(), 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    launches += 2;
    if (best < 0.0) return UINT32_MAX;
    FSGG_CUDA(cudaMemsetAsync(pick.as<void>(), 0xff, 4, s));
    km_argmax_kernel<<<blocks(n), 256, 0, s>>>(n, d2.as<double>(), labels.as<uint32_t>(), cnt,
                                               best, pick.as<unsigned int>());
    FSGG_LAUNCH_CHECK();
    uint32_t idx = 0;
    FSGG_CUDA(cudaMemcpyAsync(&idx, pick.as<void>(), 4, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    launches++;
    return idx;
  };

  for (uint32_t restart = 0; restart < std::max<uint32_t>(opts.restarts, 1); ++restart) {
    HostRng rng = HostRng::keyed(opts.seed, kKmeansTag, restart);
    // k-means++ seeding (spectral.cpp:299-330)
    const uint32_t c0 = static_cast<uint32_t>(rng.next_below(n));
    copy_center(0, c0);
    d2_update(0, 1);
    for (uint32_t c = 1; c < k; ++c) {
      cub_call(tmp, s, [&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, d2.as<double>(), prefix.as<double>(), n, s);
      });
      double total = 0.0;
      FSGG_CUDA(cudaMemcpyAsync(&total, prefix.as<double>() + n - 1, 8, cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      const double r = rng.next_double() * total;
      FSGG_CUDA(cudaMemsetAsync(pick.as<void>(), 0xff, 4, s));
      km_pick_kernel<<<blocks(n), 256, 0, s>>>(n, d2.as<double>(), prefix.as<double>(), r,
                                               pick.as<unsigned int>());
      FSGG_LAUNCH_CHECK();
      uint32_t p = 0;
      FSGG_CUDA(cudaMemcpyAsync(&p, pick.as<void>(), 4, cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      launches += 2;
      if (p == UINT32_MAX) p = first_argmax(nullptr);  // numerical tail
      copy_center(c, p);
      d2_update(c, 0);
    }
    // Lloyd iterations (spectral.cpp:332-389)
    double prev_cost = -1.0, cost = 0.0;
    uint32_t iters = 0;
    for (uint32_t iter = 0; iter < std::max<uint32_t>(opts.max_iters, 1); ++iter) {
      ++iters;
      FSGG_CUDA(cudaMemsetAsync(counts.as<void>(), 0, size_t(k) * 4, s));
      km_assign_kernel<<<blocks(n), 256, size_t(k) * dim * 8, s>>>(
          n, dim, k, pts, centers.as<double>(), labels.as<uint32_t>(), d2.as<double>(),
          counts.as<uint32_t>());
      FSGG_LAUNCH_CHECK();
      FSGG_CUDA(cudaMemcpyAsync(hcounts.data(), counts.as<void>(), size_t(k) * 4,
                                cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      launches++;
      bool repaired = false;
      for (uint32_t c = 0; c < k; ++c) {  // empty-cluster repair (:350-366)
        if (hcounts[c] > 0) continue;
        const uint32_t far = first_argmax(counts.as<uint32_t>());
        if (far == UINT32_MAX) continue;
        uint32_t lf = 0;
        FSGG_CUDA(cudaMemcpyAsync(&lf, labels.as<uint32_t>() + far, 4, cudaMemcpyDeviceToHost, s));
        FSGG_CUDA(cudaStreamSynchronize(s));
        hcounts[lf]--;
        hcounts[c] = 1;
        const double zero = 0.0;
        FSGG_CUDA(cudaMemcpyAsync(labels.as<uint32_t>() + far, &c, 4, cudaMemcpyHostToDevice, s));
        FSGG_CUDA(cudaMemcpyAsync(d2.as<double>() + far, &zero, 8, cudaMemcpyHostToDevice, s));
        FSGG_CUDA(cudaMemcpyAsync(counts.as<void>(), hcounts.data(), size_t(k) * 4,
                                  cudaMemcpyHostToDevice, s));
        copy_center(c, far);
        FSGG_CUDA(cudaStreamSynchronize(s));
        repaired = true;
      }
      km_sums_kernel<<<nb, 256, 0, s>>>(n, dim, k, pts, labels.as<uint32_t>(), d2.as<double>(),
                                        partial.as<double>());
      FSGG_LAUNCH_CHECK();
      km_sums_reduce_kernel<<<blocks(W), 256, 0, s>>>(nb, W, partial.as<double>(),
                                                      sums.as<double>());
      FSGG_LAUNCH_CHECK();
      FSGG_CUDA(cudaMemcpyAsync(hsums.data(), sums.as<void>(), size_t(W) * 8,
                                cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaMemcpyAsync(hcenters.data(), centers.as<void>(), size_t(k) * dim * 8,
                                cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      launches += 2;
      cost = hsums[W - 1];
      for (uint32_t c = 0; c < k; ++c) {
        if (hcounts[c] == 0) continue;
        for (uint32_t a = 0; a < dim; ++a)
          hcenters[size_t(c) * dim + a] = hsums[size_t(c) * dim + a] / hcounts[c];
      }
      FSGG_CUDA(cudaMemcpyAsync(centers.as<void>(), hcenters.data(), size_t(k) * dim * 8,
                                cudaMemcpyHostToDevice, s));
      if (!repaired && prev_cost >= 0.0 &&
          prev_cost - cost <= opts.rel_tol * std::max(prev_cost, 1e-300))
        break;
      prev_cost = cost;
    }
    if (best_cost < 0.0 || cost < best_cost) {
      best_cost = cost;
      best_iters = iters;
      FSGG_CUDA(cudaMemcpyAsync(best_labels.as<void>(), labels.as<void>(), size_t(n) * 4,
                                cudaMemcpyDeviceToDevice, s));
    }
  }
  FSGG_CUDA(cudaMemcpyAsync(labels_out, best_labels.as<void>(), size_t(n) * 4,
                            cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  if (cost_out) *cost_out = best_cost;
  if (iters_out) *iters_out = best_iters;
  st.kmeans_cost = best_cost;
  st.kmeans_iterations = best_iters;
  st.launches += launches;
  st.kmeans_seconds = now_s() - t0;
}

void spectral_cluster_dev(const SpectralGraphView& g, cudaStream_t s, uint32_t k, uint64_t seed,
                          const EigenOpts& eopts_in, const KmeansOpts& kopts_in,
                          uint32_t* labels, std::vector<double>* values, SpectralStats& st) {
  if (k < 2) throw ConfigError("spectral clustering needs k >= 2");  // spectral.cpp:408
  EigenOpts eopts = eopts_in;
  eopts.seed = splitmix64(seed ^ kSpectralSeedTag);
  std::vector<double> vals, res;
  DevBuf vecs;
  smallest_eigenpairs_dev(g, s, k, eopts, vals, res, vecs, st);
  if (values) *values = vals;
  const uint32_t n = g.n;
  DevBuf rows(size_t(n) * k * 8, s);
  embed_kernel<<<blocks(n), 256, 0, s>>>(n, k, vecs.as<double>(), n, rows.as<double>());
  FSGG_LAUNCH_CHECK();
  st.launches++;
  KmeansOpts kopts = kopts_in;
  kopts.seed = seed;
  kmeans_dev(rows.as<double>(), n, k, k, kopts, s, labels, nullptr, nullptr, st);
}

}  // namespace fsgg
