// Pair collapse, weighting and graph assembly: the device replacement of
// proj/src/sparsifier.cpp:78-121 and the WeightedGraph constructor
// (proj/src/graph.cpp:14-21).
//
//  * collapse_pairs: self samples dropped (:83-86), canonical (min, max)
//    keys (:87-89), radix sort + unique (:91-92) — compact keys of 2*ceil
//    (log2 n) bits so the sort touches only significant bits.
//  * finish_graph: k_ij in fp64 from the fp32 coordinates, underflow drop
//    (:105-109), p_i = min(L k / g_i, 1), p_hat = p_i + p_j - p_i p_j,
//    w = k / p_hat (:110-113) with the reference's operation order and no
//    FMA contraction; sparsity invariant (:120-121); degrees summed per
//    vertex in exactly the reference's edge order via a transposed CSR.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <vector>

#include "engine.cuh"

namespace fsgg {

namespace {

struct EdgeEstimateDev {  // layout of fsgg_edge_estimate
  uint32_t i, j;
  double k_ij, g_i, g_j, p_i, p_j, p_hat;
};

uint32_t index_bits(uint32_t n) {
  uint32_t b = 1;
  while (b < 32 && (1ull << b) < n) ++b;
  return b;
}

__global__ void rows_to_keys_kernel(uint32_t nq, const uint32_t* __restrict__ uq,
                                    const uint64_t* __restrict__ row_off,
                                    const uint32_t* __restrict__ row_cnt,
                                    const uint32_t* __restrict__ leaf_src,
                                    const uint32_t* __restrict__ leaf_cnt,
                                    uint32_t bits, unsigned long long* __restrict__ keys,
                                    unsigned long long* __restrict__ counters) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long self = 0, sampled = 0;
  if (r < nq) {
    const uint32_t q = uq[r], cnt = row_cnt[r];
    const uint64_t a = row_off[r], b = row_off[r + 1];
    sampled = cnt;
    for (uint64_t k = a; k < b; ++k) {
      unsigned long long key = ~0ull;
      if (k - a < cnt) {
        const uint32_t s = leaf_src[k];
        if (s == q) {
          self += leaf_cnt[k];
        } else {
          const uint32_t lo = min(q, s), hi = max(q, s);
          key = (static_cast<unsigned long long>(lo) << bits) | hi;
        }
      }
      keys[k] = key;
    }
  }
  for (int o = 16; o; o >>= 1) {
    self += __shfl_xor_sync(0xffffffffu, self, o);
    sampled += __shfl_xor_sync(0xffffffffu, sampled, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (self) atomicAdd(counters + 0, self);
    if (sampled) atomicAdd(counters + 1, sampled);
  }
}

__global__ void compact_to_public_kernel(unsigned long long* keys, uint64_t m,
                                         uint32_t bits) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const unsigned long long k = keys[i];
  const unsigned long long mask = (1ull << bits) - 1;
  keys[i] = ((k >> bits) << 32) | (k & mask);
}

__global__ void public_to_compact_kernel(const unsigned long long* in,
                                         unsigned long long* out, uint64_t m,
                                         uint32_t bits) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  const unsigned long long k = in[i];
  out[i] = ((k >> 32) << bits) | (k & 0xffffffffull);
}

// Steps 2 + 3 in one pass: k_ij once per pair, the underflow flag
// (sparsifier.cpp:105-109) and the weight (:110-113); dropped pairs are
// compacted afterwards (rare).
// kernel_f64 (common.cuh) for the 32 edges of a warp at high d: the same
// operations in the same order per edge, but the rows of the edges' second
// endpoints are staged through shared memory in 32-coordinate chunks with
// coalesced loads (lane = coordinate) and each lane then walks its own row.
// One thread per edge reading its row from global memory took 4.4 ms for
// C5's 2.2M edges x 784 coordinates (a 4-byte load per 3136-byte stride);
// the first endpoint is shared by most lanes of a warp (edges are sorted by
// u) and stays a direct load.
constexpr uint32_t kEdgeWideMinDim = 32;
__device__ __forceinline__ double kernel_f64_staged(int family, double sigma,
                                                    const float* __restrict__ pts, uint32_t d,
                                                    uint32_t i, uint32_t j, float (*ys)[33]) {
  const uint32_t lane = threadIdx.x & 31;
  const float* x = pts + size_t(i) * d;
  const uint32_t lim = family == 2 ? d : (d & ~1u);
  double s = 0.0;
  for (uint32_t k0 = 0; k0 < lim; k0 += 32) {
    const uint32_t kn = min(32u, lim - k0);
    for (int r = 0; r < 32; ++r) {
      const uint32_t jr = __shfl_sync(0xffffffffu, j, r);
      ys[r][lane] = lane < kn ? __ldg(pts + size_t(jr) * d + k0 + lane) : 0.f;
    }
    __syncwarp();
    if (family == 2) {
      for (uint32_t kk = 0; kk < kn; ++kk)
        s = __dadd_rn(s, fabs(__dsub_rn(double(__ldg(x + k0 + kk)), double(ys[lane][kk]))));
    } else {
      for (uint32_t kk = 0; kk < kn; ++kk) {
        const double t = __dsub_rn(double(__ldg(x + k0 + kk)), double(ys[lane][kk]));
        s = __dadd_rn(s, __dmul_rn(t, t));
      }
    }
    __syncwarp();
  }
  if (family == 2) return exp(-s / sigma);
  if (d & 1u) {
    const double t = __dsub_rn(double(x[d - 1]), double(__ldg(pts + size_t(j) * d + d - 1)));
    s = __fma_rn(t, t, s);
  }
  if (family == 1) return exp(-sqrt(s) / sigma);
  return exp(-s / __dmul_rn(sigma, sigma));
}

template <bool WIDE>
__global__ void edges_kernel(const unsigned long long* __restrict__ keys, uint64_t m,
                             const float* __restrict__ pts, uint32_t d, int family,
                             double sigma, double L, const double* __restrict__ g_full,
                             uint32_t* __restrict__ u, uint32_t* __restrict__ v,
                             double* __restrict__ w, EdgeEstimateDev* est,
                             unsigned char* __restrict__ keep,
                             unsigned long long* __restrict__ dropped, int write_v) {
  __shared__ unsigned long long red[8];
  __shared__ float ys[WIDE ? 8 : 1][WIDE ? 32 : 1][33];
  const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  unsigned long long drop = 0;
  double kw = 0.0;
  if constexpr (WIDE) {  // whole warps: lanes past m stage point 0
    const unsigned long long key = e < m ? keys[e] : 0ull;
    kw = kernel_f64_staged(family, sigma, pts, d, uint32_t(key >> 32), uint32_t(key),
                           ys[threadIdx.x >> 5]);
  }
  if (e < m) {
    const uint32_t i = uint32_t(keys[e] >> 32), j = uint32_t(keys[e]);
    const double k =
        WIDE ? kw : kernel_f64(family, sigma, pts + size_t(i) * d, pts + size_t(j) * d, d);
    const bool ok = k >= 1e-300;
    keep[e] = ok;
    drop = ok ? 0 : 1;
    const double gi = g_full[i], gj = g_full[j];
    const double pi = fmin(__ddiv_rn(__dmul_rn(L, k), gi), 1.0);
    const double pj = fmin(__ddiv_rn(__dmul_rn(L, k), gj), 1.0);
    const double ph = __dsub_rn(__dadd_rn(pi, pj), __dmul_rn(pi, pj));
    u[e] = i;
    if (write_v) v[e] = j;
    w[e] = __ddiv_rn(k, ph);
    if (est) est[e] = EdgeEstimateDev{i, j, k, gi, gj, pi, pj, ph};
  }
  for (int o = 16; o; o >>= 1) drop += __shfl_xor_sync(0xffffffffu, drop, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = drop;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (uint32_t k = 0; k < blockDim.x / 32; ++k) t += red[k];
    if (t) atomicAdd(dropped, t);
  }
}

// v of every edge from the sorted unique public keys (streamed output: its
// copy to the host can start before the weights exist).
__global__ void keys_to_v_kernel(const unsigned long long* __restrict__ keys, uint64_t m,
                                 uint32_t* __restrict__ v) {
  const uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (e < m) v[e] = uint32_t(keys[e]);
}

// row_ptr[x] = first edge index with key-row >= x (keys sorted).
__global__ void row_ptr_kernel(const uint32_t* __restrict__ rows, uint64_t m,
                               uint32_t n, uint64_t* __restrict__ row_ptr) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x > n) return;
  uint64_t lo = 0, hi = m;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (rows[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  row_ptr[x] = lo;
}

// Degree of x in the reference's accumulation order (graph.cpp:14-21):
// edges (u, x), u < x ascending, then edges (x, v), v ascending.
__global__ void degrees_kernel(uint32_t n, const uint64_t* __restrict__ rpt,
                               const double* __restrict__ wt,
                               const uint64_t* __restrict__ rp,
                               const double* __restrict__ w,
                               double* __restrict__ deg) {
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  double s = 0.0;
  for (uint64_t e = rpt[x]; e < rpt[x + 1]; ++e) s = __dadd_rn(s, wt[e]);
  for (uint64_t e = rp[x]; e < rp[x + 1]; ++e) s = __dadd_rn(s, w[e]);
  deg[x] = s;
}

// Degrees of rows [rb, re) of a row-sharded graph: the lower contributions
// (edges (u, x), u < x, routed here from their owners and stable-sorted by
// x: u ascending) first, then the rank's own row x — exactly the
// accumulation order of degrees_kernel on one GPU.
__global__ void rows_degrees_kernel(uint32_t rb, uint32_t re,
                                    const uint64_t* __restrict__ lrp,  // re - rb + 1
                                    const double* __restrict__ lw,
                                    const uint64_t* __restrict__ rp,   // global upper CSR
                                    const double* __restrict__ w,
                                    double* __restrict__ deg) {
  const uint32_t x = rb + blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= re) return;
  double s = 0.0;
  for (uint64_t e = lrp[x - rb]; e < lrp[x - rb + 1]; ++e) s = __dadd_rn(s, lw[e]);
  for (uint64_t e = rp[x]; e < rp[x + 1]; ++e) s = __dadd_rn(s, w[e]);
  deg[x - rb] = s;
}

// lrp[i] = first index of sorted keys with key >= rb + i (i <= re - rb)
__global__ void range_ptr_kernel(const uint32_t* __restrict__ keys, uint64_t m, uint32_t rb,
                                 uint32_t re, uint64_t* __restrict__ lrp) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > re - rb) return;
  const uint32_t x = rb + i;
  uint64_t lo = 0, hi = m;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (keys[mid] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  lrp[i] = lo;
}

template <class F>
void cub_call(DevBuf& tmp, cudaStream_t s, F&& f) {
  size_t bytes = 0;
  FSGG_CUDA(f(static_cast<void*>(nullptr), bytes));
  tmp.ensure(bytes + 16, s);
  FSGG_CUDA(f(tmp.as<void>(), bytes));
}

// Sort + unique compact keys in place; returns unique count (sentinel
// ~0 entries, if any, are dropped).
uint64_t sort_unique_compact(Dataset& ds, DevBuf& keys, uint64_t m,
                             uint32_t bits) {
  cudaStream_t s = ds.stream;
  if (m == 0) return 0;
  DevBuf& alt = ds.buf("g.alt", m * 8);
  DevBuf& tmp = ds.buf("g.tmp", 8);
  DevBuf& cnt = ds.buf("g.cnt", 16);
  cub::DoubleBuffer<unsigned long long> db(keys.as<unsigned long long>(),
                                           alt.as<unsigned long long>());
  cub_call(tmp, s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortKeys(t, b, db, m, 0, int(2 * bits), s);
  });
  unsigned long long* sorted = db.Current();
  unsigned long long* other = db.Alternate();
  cub_call(tmp, s, [&](void* t, size_t& b) {
    return cub::DeviceSelect::Unique(t, b, sorted, other, cnt.as<uint64_t>(), m, s);
  });
  ds.launches += 8;
  uint64_t u = 0;
  unsigned long long last = 0;
  FSGG_CUDA(cudaMemcpyAsync(&u, cnt.as<void>(), 8, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  if (u) {
    FSGG_CUDA(cudaMemcpyAsync(&last, other + u - 1, 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    if (last == ~0ull) --u;
  }
  if (other != keys.as<unsigned long long>()) std::swap(keys, alt);
  return u;
}

// Shard keys by the owner of row u (multi-GPU finish): destination of a
// compact key = the rank whose [bounds[r], bounds[r+1]) holds its u.
constexpr int kRouteKeyThreads = 256;
constexpr int kRouteKeyItems = 8;
constexpr uint32_t kMaxWorld = 64;

__device__ __forceinline__ uint32_t key_dest(uint32_t u, const uint32_t* sb, uint32_t world) {
  uint32_t r = 0;
  while (r + 1 < world && u >= sb[r + 1]) ++r;
  return r;
}

__global__ void __launch_bounds__(kRouteKeyThreads)
    key_dest_count_kernel(const unsigned long long* __restrict__ keys, uint64_t m, uint32_t bits,
                          const uint32_t* __restrict__ bounds, uint32_t world,
                          unsigned long long* __restrict__ counts) {
  __shared__ uint32_t sb[kMaxWorld + 1];
  __shared__ unsigned long long hist[kMaxWorld];
  for (uint32_t k = threadIdx.x; k <= world; k += blockDim.x) sb[k] = bounds[k];
  for (uint32_t k = threadIdx.x; k < world; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  // warp-aggregated: lanes with the same destination add once (most keys of
  // a tile share one, and same-address shared atomics serialise)
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t e0 = blockIdx.x * uint64_t(blockDim.x); e0 < m;
       e0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t e = e0 + threadIdx.x;
    const unsigned long long k = e < m ? keys[e] : ~0ull;
    const uint32_t dst = k != ~0ull ? key_dest(uint32_t(k >> bits), sb, world) : kMaxWorld;
    const unsigned grp = __match_any_sync(0xffffffffu, dst);
    if (dst < kMaxWorld && lane == uint32_t(__ffs(grp) - 1))
      atomicAdd(&hist[dst], static_cast<unsigned long long>(__popc(grp)));
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < world; k += blockDim.x)
    if (hist[k]) atomicAdd(counts + k, hist[k]);
}

// One tile per CTA: per-destination counts in shared memory, one global
// reservation per destination, then the public keys (u << 32 | v) written
// into their destination's range (order within it is irrelevant: the owner
// sorts what it receives).
__global__ void __launch_bounds__(kRouteKeyThreads)
    key_dest_scatter_kernel(const unsigned long long* __restrict__ keys, uint64_t m,
                            uint32_t bits, const uint32_t* __restrict__ bounds, uint32_t world,
                            unsigned long long* __restrict__ cursor,
                            unsigned long long* __restrict__ out) {
  __shared__ uint32_t sb[kMaxWorld + 1];
  __shared__ uint32_t cnt[kMaxWorld];
  __shared__ unsigned long long base[kMaxWorld];
  for (uint32_t k = threadIdx.x; k <= world; k += blockDim.x) sb[k] = bounds[k];
  const uint64_t tile = uint64_t(kRouteKeyThreads) * kRouteKeyItems;
  const unsigned long long mask = (1ull << bits) - 1;
  for (uint64_t t0 = blockIdx.x * tile; t0 < m; t0 += uint64_t(gridDim.x) * tile) {
    for (uint32_t k = threadIdx.x; k < world; k += blockDim.x) cnt[k] = 0;
    __syncthreads();
    unsigned long long key[kRouteKeyItems];
    uint32_t dst[kRouteKeyItems], slot[kRouteKeyItems];
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < kRouteKeyItems; ++j) {
      const uint64_t e = t0 + uint64_t(j) * kRouteKeyThreads + threadIdx.x;
      key[j] = e < m ? keys[e] : ~0ull;
      dst[j] = key[j] != ~0ull ? key_dest(uint32_t(key[j] >> bits), sb, world) : kMaxWorld;
      // warp-aggregated slot reservation per destination
      const unsigned grp = __match_any_sync(0xffffffffu, dst[j]);
      const uint32_t leader = __ffs(grp) - 1;
      uint32_t b0 = 0;
      if (dst[j] < kMaxWorld && lane == leader) b0 = atomicAdd(&cnt[dst[j]], uint32_t(__popc(grp)));
      b0 = __shfl_sync(0xffffffffu, b0, leader);
      slot[j] = b0 + __popc(grp & ((1u << lane) - 1u));
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < world; k += blockDim.x)
      base[k] = cnt[k] ? atomicAdd(cursor + k, static_cast<unsigned long long>(cnt[k])) : 0ull;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kRouteKeyItems; ++j)
      if (dst[j] < kMaxWorld)
        out[base[dst[j]] + slot[j]] = ((key[j] >> bits) << 32) | (key[j] & mask);
    __syncthreads();
  }
}

}  // namespace

__global__ void shifted_slice_kernel(const uint64_t* __restrict__ in, uint32_t count,
                                     uint64_t shift, uint64_t* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = in[i] + shift;
}

void rows_row_ptr(Dataset& ds, const GraphResult& g, uint32_t rb, uint32_t re,
                  uint64_t edge_offset, uint64_t* out) {
  if (re <= rb) return;
  cudaStream_t s = ds.stream;
  shifted_slice_kernel<<<ceil_div_u32(re - rb, 256), 256, 0, s>>>(
      g.row_ptr.as<uint64_t>() + rb, re - rb, edge_offset, out);
  FSGG_LAUNCH_CHECK();
  ds.launches++;
  FSGG_CUDA(cudaStreamSynchronize(s));
}

// ---- row-bucketed pair collapse (1-GPU build) ------------------------------
// A sample (q, s), s != q, is the undirected pair (min, max) and belongs to
// row min(q, s). Instead of a 40-bit radix sort of all n L pair keys, the
// partners are bucketed by row (count, scan, fill; one warp per sampled
// row, coalesced over its sources), each row's partners ranked in shared
// memory by one warp (rows hold ~L values) and deduplicated: the same sorted
// unique (u, v) list with a fraction of the memory traffic. Rows longer than
// kRowSortCap (only with rounds comparable to n) go through CUB's segmented
// sort instead.
constexpr uint32_t kRowSortCap = 512;
constexpr int kRowIdxBits = 9;  // position bits of the rank keys (kRowSortCap)
constexpr int kRowWarps = 8;

__global__ void rows_count_kernel(uint32_t nq, const uint32_t* __restrict__ uq,
                                  const uint64_t* __restrict__ row_off,
                                  const uint32_t* __restrict__ row_cnt,
                                  const uint32_t* __restrict__ leaf_src,
                                  const uint32_t* __restrict__ leaf_cnt,
                                  uint32_t* __restrict__ cnt,
                                  unsigned long long* __restrict__ counters) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long self = 0, sampled = 0;
  if (r < nq) {
    const uint32_t q = uq[r], c = row_cnt[r];
    const uint64_t a = row_off[r];
    sampled = c;
    uint32_t own = 0;  // partners above q land in q's own row: one atomic
    for (uint32_t k = 0; k < c; ++k) {
      const uint32_t s = leaf_src[a + k];
      if (s == q)
        self += leaf_cnt[a + k];
      else if (s > q)
        ++own;
      else
        atomicAdd(cnt + s, 1u);
    }
    if (own) atomicAdd(cnt + q, own);
  }
  for (int o = 16; o; o >>= 1) {
    self += __shfl_xor_sync(0xffffffffu, self, o);
    sampled += __shfl_xor_sync(0xffffffffu, sampled, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (self) atomicAdd(counters + 0, self);
    if (sampled) atomicAdd(counters + 1, sampled);
  }
}

__global__ void __launch_bounds__(256) rows_fill_kernel(
    uint32_t nq, const uint32_t* __restrict__ uq, const uint64_t* __restrict__ row_off,
    const uint32_t* __restrict__ row_cnt, const uint32_t* __restrict__ leaf_src,
    const uint32_t* __restrict__ off, uint32_t* __restrict__ fill, uint32_t* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const uint32_t r = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (r >= nq) return;
  const uint32_t q = uq[r], c = row_cnt[r];
  const uint64_t a = row_off[r];
  uint32_t own = 0;
  for (uint32_t k = lane; k < c; k += 32) own += leaf_src[a + k] > q;
  for (int o = 16; o; o >>= 1) own += __shfl_xor_sync(0xffffffffu, own, o);
  uint32_t at = 0;
  if (lane == 0 && own) at = off[q] + atomicAdd(fill + q, own);
  at = __shfl_sync(0xffffffffu, at, 0);
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t k0 = 0; k0 < c; k0 += 32) {
    const uint32_t k = k0 + lane;
    const uint32_t s = k < c ? leaf_src[a + k] : q;
    const unsigned up = __ballot_sync(0xffffffffu, s > q);
    if (s > q)
      part[at + __popc(up & lt)] = s;
    else if (s < q)
      part[off[s] + atomicAdd(fill + s, 1u)] = q;
    at += __popc(up);
  }
}

// One warp per row: partner v at position i becomes the distinct key
// (v << 9) | i, whose rank among the row's keys is its sorted position
// (rows <= kRowSortCap = 512, n <= 2^23). Each lane holds up to 8 keys in
// registers and compares them against every key of the row, read as
// broadcast uint4 from shared memory; the ranked row is deduplicated by
// neighbour comparison and written back sorted with its distinct count.
template <int K>
__device__ __forceinline__ void rank_pass(const uint32_t* x, uint32_t c4, uint32_t base,
                                          int lane, uint32_t* y) {
  uint32_t v[K], r[K];
#pragma unroll
  for (int t = 0; t < K; ++t) {
    v[t] = x[base + lane + 32 * t];
    r[t] = 0;
  }
  for (uint32_t j = 0; j < c4; j += 4) {
    const uint4 q = *reinterpret_cast<const uint4*>(x + j);
#pragma unroll
    for (int t = 0; t < K; ++t)
      r[t] += (q.x < v[t]) + (q.y < v[t]) + (q.z < v[t]) + (q.w < v[t]);
  }
#pragma unroll
  for (int t = 0; t < K; ++t)
    if (v[t] != 0xffffffffu) y[r[t]] = v[t] >> kRowIdxBits;
}

__global__ void __launch_bounds__(256) rows_sort_kernel(uint32_t n, const uint32_t* __restrict__ off,
                                                        const uint32_t* __restrict__ part,
                                                        uint32_t* __restrict__ sorted,
                                                        uint32_t* __restrict__ ucnt,
                                                        unsigned long long* __restrict__ longest) {
  __shared__ __align__(16) uint32_t sx[kRowWarps][kRowSortCap];
  __shared__ uint32_t sy[kRowWarps][kRowSortCap];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * kRowWarps + w;
  if (u > n) return;
  if (u == n) {
    if (lane == 0) ucnt[n] = 0;
    return;
  }
  const uint32_t a = off[u], c = off[u + 1] - a;
  if (c > kRowSortCap) {  // the host sorts the rows with CUB instead
    if (lane == 0) atomicMax(longest, (unsigned long long)c);
    return;
  }
  uint32_t* x = sx[w];
  uint32_t* y = sy[w];
  const uint32_t c32 = (c + 31) & ~31u;
  for (uint32_t i = lane; i < c32; i += 32)
    x[i] = i < c ? (part[a + i] << kRowIdxBits) | i : 0xffffffffu;
  __syncwarp();
  const uint32_t c4 = (c + 3) & ~3u;
  for (uint32_t base = 0; base < c; base += 256) {
    switch (min(8u, (c - base + 31) >> 5)) {
      case 1: rank_pass<1>(x, c4, base, lane, y); break;
      case 2: rank_pass<2>(x, c4, base, lane, y); break;
      case 3: rank_pass<3>(x, c4, base, lane, y); break;
      case 4: rank_pass<4>(x, c4, base, lane, y); break;
      case 5: rank_pass<5>(x, c4, base, lane, y); break;
      case 6: rank_pass<6>(x, c4, base, lane, y); break;
      case 7: rank_pass<7>(x, c4, base, lane, y); break;
      default: rank_pass<8>(x, c4, base, lane, y); break;
    }
  }
  __syncwarp();
  uint32_t distinct = 0;
  for (uint32_t i = lane; i < c; i += 32) {
    const uint32_t v = y[i];
    distinct += i == 0 || v != y[i - 1];
    sorted[a + i] = v;
  }
  for (int o = 16; o; o >>= 1) distinct += __shfl_xor_sync(0xffffffffu, distinct, o);
  if (lane == 0) ucnt[u] = distinct;
}

// distinct partners per row of a sorted segment (the CUB fallback)
__global__ void rows_unique_count_kernel(uint32_t n, const uint32_t* __restrict__ off,
                                         const uint32_t* __restrict__ part,
                                         uint32_t* __restrict__ ucnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (u > n) return;
  uint32_t k = 0;
  if (u < n)
    for (uint32_t e = off[u] + lane; e < off[u + 1]; e += 32)
      k += (e == off[u] || part[e] != part[e - 1]);
  for (int o = 16; o; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  if (lane == 0) ucnt[u] = k;
}

__global__ void __launch_bounds__(256) rows_unique_write_kernel(
    uint32_t n, const uint32_t* __restrict__ off, const uint32_t* __restrict__ sorted,
    const uint32_t* __restrict__ uoff, unsigned long long* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (u >= n) return;
  const uint32_t a = off[u], e = off[u + 1];
  uint32_t at = uoff[u];
  const unsigned lt = (1u << lane) - 1u;
  for (uint32_t i0 = a; i0 < e; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t v = i < e ? sorted[i] : 0u;
    const bool keep = i < e && (i == a || sorted[i - 1] != v);
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) keys[at + __popc(m & lt)] = (static_cast<unsigned long long>(u) << 32) | v;
    at += __popc(m);
  }
}

uint64_t collapse_pairs_routed(Dataset& ds, SampleResult& res, DevBuf& keys, uint32_t world,
                               const uint32_t* bounds_host, uint64_t* counts,
                               uint64_t* self_pairs, uint64_t* sampled_pairs) {
  if (world == 0 || world > kMaxWorld) throw ConfigError("world size must be 1..64");
  cudaStream_t s = ds.stream;
  const uint64_t cap = std::max<uint64_t>(res.total_tickets, 1);
  const uint32_t bits = index_bits(ds.n);
  DevBuf& raw = ds.buf("g.raw_keys", cap * 8);
  keys.ensure(cap * 8, s);
  DevBuf& aux = ds.buf("g.route_aux", (kMaxWorld + 2) * 4 + 2 * kMaxWorld * 8);
  uint32_t* dbounds = aux.as<uint32_t>();
  unsigned long long* dcounts =
      reinterpret_cast<unsigned long long*>(aux.as<char>() + (kMaxWorld + 1) * 4 + 4);
  unsigned long long* dcursor = dcounts + kMaxWorld;
  DevBuf& counters = ds.buf("g.counters", 16);
  FSGG_CUDA(cudaMemsetAsync(counters.as<void>(), 0, 16, s));
  FSGG_CUDA(cudaMemsetAsync(dcounts, 0, kMaxWorld * 8, s));
  FSGG_CUDA(cudaMemcpyAsync(dbounds, bounds_host, size_t(world + 1) * 4, cudaMemcpyHostToDevice,
                            s));
  rows_to_keys_kernel<<<ceil_div_u32(std::max<uint32_t>(res.nq, 1), 256), 256, 0, s>>>(
      res.nq, res.uq.as<uint32_t>(), res.row_off.as<uint64_t>(),
      res.row_cnt.as<uint32_t>(), res.leaf_src.as<uint32_t>(),
      res.leaf_cnt.as<uint32_t>(), bits, raw.as<unsigned long long>(),
      counters.as<unsigned long long>());
  const uint64_t m = res.total_tickets;
  const uint32_t grid = std::max<uint32_t>(
      1, std::min<uint32_t>(ceil_div_u32(m, uint64_t(kRouteKeyThreads) * kRouteKeyItems),
                            uint32_t(ds.num_sms) * 8));
  key_dest_count_kernel<<<grid, kRouteKeyThreads, 0, s>>>(raw.as<unsigned long long>(), m, bits,
                                                          dbounds, world, dcounts);
  FSGG_LAUNCH_CHECK();
  unsigned long long hc[2 + kMaxWorld];
  FSGG_CUDA(cudaMemcpyAsync(hc, counters.as<void>(), 16, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(hc + 2, dcounts, size_t(world) * 8, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  *self_pairs = hc[0];
  *sampled_pairs = hc[1];
  std::vector<unsigned long long> off(world);
  uint64_t total = 0;
  for (uint32_t r = 0; r < world; ++r) {
    counts[r] = hc[2 + r];
    off[r] = total;
    total += hc[2 + r];
  }
  FSGG_CUDA(cudaMemcpyAsync(dcursor, off.data(), size_t(world) * 8, cudaMemcpyHostToDevice, s));
  key_dest_scatter_kernel<<<grid, kRouteKeyThreads, 0, s>>>(
      raw.as<unsigned long long>(), m, bits, dbounds, world, dcursor,
      keys.as<unsigned long long>());
  FSGG_LAUNCH_CHECK();
  ds.launches += 3;
  return total;
}

uint64_t collapse_pairs(Dataset& ds, SampleResult& res, DevBuf& keys,
                        uint64_t* self_pairs, uint64_t* sampled_pairs) {
  cudaStream_t s = ds.stream;
  const uint32_t n = ds.n;
  const uint64_t cap = std::max<uint64_t>(res.total_tickets, 1);
  if (cap > 0xffffffffull) throw ConfigError("too many samples for 32-bit row offsets");
  keys.ensure(cap * 8, s);
  DevBuf& counters = ds.buf("g.counters", 24);
  DevBuf& cnt = ds.buf("g.row_cnt", size_t(n + 2) * 4);
  DevBuf& off = ds.buf("g.row_off", size_t(n + 2) * 4);
  DevBuf& fill = ds.buf("g.row_fill", size_t(n + 2) * 4);
  DevBuf& part = ds.buf("g.part", cap * 4);
  DevBuf& sorted = ds.buf("g.part2", cap * 4);
  DevBuf& tmp = ds.buf("g.tmp", 8);
  FSGG_CUDA(cudaMemsetAsync(counters.as<void>(), 0, 24, s));
  FSGG_CUDA(cudaMemsetAsync(cnt.as<void>(), 0, size_t(n + 2) * 4, s));
  FSGG_CUDA(cudaMemsetAsync(fill.as<void>(), 0, size_t(n + 2) * 4, s));
  const uint32_t gq = ceil_div_u32(std::max<uint32_t>(res.nq, 1), kRowWarps);
  const uint32_t gn = ceil_div_u32(uint64_t(n) + 1, kRowWarps);
  rows_count_kernel<<<ceil_div_u32(std::max<uint32_t>(res.nq, 1), 256), 256, 0, s>>>(res.nq, res.uq.as<uint32_t>(),
                                       res.row_off.as<uint64_t>(), res.row_cnt.as<uint32_t>(),
                                       res.leaf_src.as<uint32_t>(), res.leaf_cnt.as<uint32_t>(),
                                       cnt.as<uint32_t>(), counters.as<unsigned long long>());
  FSGG_LAUNCH_CHECK();
  cub_call(tmp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt.as<uint32_t>(), off.as<uint32_t>(), n + 1, s);
  });
  rows_fill_kernel<<<gq, 256, 0, s>>>(
      res.nq, res.uq.as<uint32_t>(), res.row_off.as<uint64_t>(), res.row_cnt.as<uint32_t>(),
      res.leaf_src.as<uint32_t>(), off.as<uint32_t>(), fill.as<uint32_t>(), part.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  const char* env = std::getenv("FSGG_COLLAPSE_SEGSORT");  // read per call: tests toggle it
  bool segsort = (env && env[0] == '1') || uint64_t(n) > (1ull << (32 - kRowIdxBits));
  if (!segsort) {
    rows_sort_kernel<<<gn, 256, 0, s>>>(n, off.as<uint32_t>(), part.as<uint32_t>(),
                                        sorted.as<uint32_t>(), cnt.as<uint32_t>(),
                                        counters.as<unsigned long long>() + 2);
    FSGG_LAUNCH_CHECK();
  }
  unsigned long long* hw = ds.host_words();
  FSGG_CUDA(cudaMemcpyAsync(hw, counters.as<void>(), 24, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(hw + 3, off.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  *self_pairs = hw[0];
  *sampled_pairs = hw[1];
  segsort = segsort || hw[2] > kRowSortCap;
  const uint32_t total = *reinterpret_cast<const uint32_t*>(hw + 3);
  if (total == 0) return 0;
  ds.launches += 5;
  if (segsort) {
    cub_call(tmp, s, [&](void* t, size_t& b) {
      return cub::DeviceSegmentedSort::SortKeys(t, b, part.as<uint32_t>(),
                                                sorted.as<uint32_t>(), int(total), int(n),
                                                off.as<uint32_t>(), off.as<uint32_t>() + 1, s);
    });
    rows_unique_count_kernel<<<gn, 256, 0, s>>>(n, off.as<uint32_t>(), sorted.as<uint32_t>(),
                                                cnt.as<uint32_t>());
    FSGG_LAUNCH_CHECK();
    ds.launches += 2;
  }
  cub_call(tmp, s, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt.as<uint32_t>(), fill.as<uint32_t>(), n + 1, s);
  });
  rows_unique_write_kernel<<<ceil_div_u32(n, kRowWarps), 256, 0, s>>>(
      n, off.as<uint32_t>(), sorted.as<uint32_t>(), fill.as<uint32_t>(),
      keys.as<unsigned long long>());
  FSGG_LAUNCH_CHECK();
  uint32_t* hm = reinterpret_cast<uint32_t*>(ds.host_words());
  FSGG_CUDA(cudaMemcpyAsync(hm, fill.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  return *hm;
}

// Step 4 of finish_graph (shared by the chunked finish): upper CSR,
// transposed CSR, degrees, total weight, and their host copies.
template <class After>
void finish_tail(Dataset& ds, uint32_t n, uint64_t m, uint32_t bits, GraphResult& out,
                 const HostSink* sink, After&& after, cudaStream_t cs) {
  cudaStream_t s = ds.stream;
  const uint64_t mm = std::max<uint64_t>(m, 1);
  DevBuf& tmp = ds.buf("g.tmp", 8);
  out.tv_sorted = nullptr;
  out.tw_sorted = nullptr;
  // upper CSR, transposed CSR, degrees, total weight. The transpose is a
  // stable radix sort on v alone (ceil(log2 n) bits): edges arrive in (u, v)
  // order, so each vertex's lower neighbours stay in ascending u.
  out.row_ptr.ensure(size_t(n + 1) * 8, s);
  out.degrees.ensure(size_t(n) * 8, s);
  DevBuf& rpt = ds.buf("g.rpt", size_t(n + 1) * 8);
  DevBuf& tv = ds.buf("g.tv", mm * 4);
  DevBuf& tv2 = ds.buf("g.tv2", mm * 4);
  DevBuf& wt = ds.buf("g.wt", mm * 8);
  DevBuf& wt2 = ds.buf("g.wt2", mm * 8);
  row_ptr_kernel<<<ceil_div_u32(uint64_t(n) + 1, 256), 256, 0, s>>>(
      out.u.as<uint32_t>(), m, n, out.row_ptr.as<uint64_t>());
  FSGG_LAUNCH_CHECK();
  if (sink) after(sink->row_ptr, out.row_ptr.as<void>(), (uint64_t(n) + 1) * 8);
  if (m) {
    FSGG_CUDA(cudaMemcpyAsync(tv.as<void>(), out.v.as<void>(), m * 4, cudaMemcpyDeviceToDevice, s));
    FSGG_CUDA(cudaMemcpyAsync(wt.as<void>(), out.w.as<void>(), m * 8,
                              cudaMemcpyDeviceToDevice, s));
    cub::DoubleBuffer<uint32_t> dk(tv.as<uint32_t>(), tv2.as<uint32_t>());
    cub::DoubleBuffer<double> dv(wt.as<double>(), wt2.as<double>());
    cub_call(tmp, s, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, m, 0, int(bits), s);
    });
    row_ptr_kernel<<<ceil_div_u32(uint64_t(n) + 1, 256), 256, 0, s>>>(
        dk.Current(), m, n, rpt.as<uint64_t>());
    FSGG_LAUNCH_CHECK();
    out.tv_sorted = dk.Current();
    out.tw_sorted = dv.Current();
    degrees_kernel<<<ceil_div_u32(n, 256), 256, 0, s>>>(
        n, rpt.as<uint64_t>(), dv.Current(), out.row_ptr.as<uint64_t>(),
        out.w.as<double>(), out.degrees.as<double>());
    FSGG_LAUNCH_CHECK();
    // (the sum goes to its own word: wt/wt2 hold the transposed weights that
    // rows_transposed hands out)
    DevBuf& tot = ds.buf("g.total", 8);
    cub_call(tmp, s, [&](void* t, size_t& b) {
      return cub::DeviceReduce::Sum(t, b, out.w.as<double>(), tot.as<double>(), m, s);
    });
    FSGG_CUDA(cudaMemcpyAsync(&out.total_weight, tot.as<void>(), 8,
                              cudaMemcpyDeviceToHost, s));
    ds.launches += 12;
  } else {
    FSGG_CUDA(cudaMemsetAsync(out.degrees.as<void>(), 0, size_t(n) * 8, s));
    out.total_weight = 0.0;
  }
  if (sink) {
    after(sink->degrees, out.degrees.as<void>(), size_t(n) * 8);
    FSGG_CUDA(cudaStreamSynchronize(cs));
  }
  FSGG_CUDA(cudaStreamSynchronize(s));
}


// RAII for the host-output side stream: on any throw, the copies into the
// caller's buffers are finished and the stream/event released before
// unwinding.
struct SideStream {
  cudaStream_t cs = nullptr;
  cudaEvent_t ev = nullptr;
  ~SideStream() {
    if (cs) {
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
    }
    if (ev) cudaEventDestroy(ev);
  }
};

// finish_graph over u-range chunks of unsorted keys (collapse_pairs_routed
// with one "rank" per chunk): each chunk is sorted, deduplicated and
// weighted on its own and appended, and with a HostSink its v and w go to
// the host while the next chunk is processed — the graph's 0.78 GB
// device-to-host copy (C3) starts ~1 ms after the descent instead of after a
// full 64M-key sort. The arrays are the one-pass finish's bit for bit
// (chunks are disjoint u ranges in order).
void finish_graph_chunked(Dataset& ds, const KernelSpec& ks, uint32_t rounds,
                          const double* g_full, const uint64_t* keys_in,
                          const uint64_t* chunks, uint32_t nchunks, GraphResult& out,
                          const HostSink* sink) {
  cudaStream_t s = ds.stream;
  const uint32_t n = ds.n, d = ds.d;
  const uint32_t bits = index_bits(n);
  const float* pts = ds.pts.as<float>();
  out.n = n;
  uint64_t total = 0, cmax = 1;
  for (uint32_t c = 0; c < nchunks; ++c) {
    total += chunks[c];
    cmax = std::max<uint64_t>(cmax, chunks[c]);
  }
  out.u.ensure(std::max<uint64_t>(total, 1) * 4, s);
  out.v.ensure(std::max<uint64_t>(total, 1) * 4, s);
  out.w.ensure(std::max<uint64_t>(total, 1) * 8, s);
  DevBuf& keys = ds.buf("g.keys", cmax * 8);
  DevBuf& keep = ds.buf("g.keep", cmax);
  DevBuf& tmp = ds.buf("g.tmp", 8);
  DevBuf& cnt = ds.buf("g.cnt", 16);
  SideStream side;
  cudaStream_t& cs = side.cs;
  cudaEvent_t& ev = side.ev;
  auto after = [&](void* dst, const void* src, size_t bytes) {
    if (!dst || !bytes) return;
    FSGG_CUDA(cudaEventRecord(ev, s));
    FSGG_CUDA(cudaStreamWaitEvent(cs, ev, 0));
    FSGG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, cs));
  };
  if (sink) {
    FSGG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    FSGG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  uint64_t m = 0, in = 0;
  out.underflow = 0;
  for (uint32_t c = 0; c < nchunks; ++c) {
    const uint64_t kc = chunks[c];
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(keys_in) + in;
    in += kc;
    if (kc == 0) continue;
    public_to_compact_kernel<<<ceil_div_u32(kc, 256), 256, 0, s>>>(
        src, keys.as<unsigned long long>(), kc, bits);
    FSGG_LAUNCH_CHECK();
    const uint64_t mc = sort_unique_compact(ds, keys, kc, bits);
    if (mc == 0) continue;
    compact_to_public_kernel<<<ceil_div_u32(mc, 256), 256, 0, s>>>(
        keys.as<unsigned long long>(), mc, bits);
    FSGG_LAUNCH_CHECK();
    ds.launches += 2;
    if (sink && m + mc > sink->capacity)
      throw ConfigError("host output capacity below the sampled unique pair count");
    uint32_t* uc = out.u.as<uint32_t>() + m;
    uint32_t* vc = out.v.as<uint32_t>() + m;
    double* wc = out.w.as<double>() + m;
    const bool early_v = sink && sink->v;
    if (early_v) {
      keys_to_v_kernel<<<ceil_div_u32(mc, 256), 256, 0, s>>>(keys.as<unsigned long long>(), mc,
                                                             vc);
      FSGG_LAUNCH_CHECK();
      ds.launches++;
      after(sink->v + m, vc, mc * 4);
    }
    FSGG_CUDA(cudaMemsetAsync(cnt.as<void>(), 0, 16, s));
    (d >= kEdgeWideMinDim ? edges_kernel<true> : edges_kernel<false>)<<<ceil_div_u32(mc, 256), 256, 0, s>>>(
        keys.as<unsigned long long>(), mc, pts, d, ks.family, ks.sigma, double(rounds), g_full,
        uc, vc, wc, nullptr, keep.as<unsigned char>(), cnt.as<unsigned long long>(),
        early_v ? 0 : 1);
    FSGG_LAUNCH_CHECK();
    ds.launches++;
    unsigned long long dropped = 0;
    FSGG_CUDA(cudaMemcpyAsync(&dropped, cnt.as<void>(), 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    if (dropped) {  // underflow pairs (k_ij < 1e-300): compact this chunk (stable)
      DevBuf& o4 = ds.buf("g.cu", mc * 4);
      DevBuf& o8 = ds.buf("g.cw", mc * 8);
      auto compact4 = [&](uint32_t* arr) {
        cub_call(tmp, s, [&](void* t, size_t& b) {
          return cub::DeviceSelect::Flagged(t, b, arr, keep.as<unsigned char>(),
                                            o4.as<uint32_t>(), cnt.as<uint64_t>() + 1, mc, s);
        });
        FSGG_CUDA(cudaMemcpyAsync(arr, o4.as<void>(), (mc - dropped) * 4,
                                  cudaMemcpyDeviceToDevice, s));
      };
      compact4(uc);
      compact4(vc);
      cub_call(tmp, s, [&](void* t, size_t& b) {
        return cub::DeviceSelect::Flagged(t, b, wc, keep.as<unsigned char>(), o8.as<double>(),
                                          cnt.as<uint64_t>() + 1, mc, s);
      });
      FSGG_CUDA(cudaMemcpyAsync(wc, o8.as<void>(), (mc - dropped) * 8, cudaMemcpyDeviceToDevice,
                                s));
      ds.launches += 3;
      if (early_v) after(sink->v + m, vc, (mc - dropped) * 4);  // the compacted v
    }
    if (sink) after(sink->w + m, wc, (mc - dropped) * 8);
    m += mc - dropped;
    out.underflow += dropped;
  }
  if (m > uint64_t(n) * rounds)
    throw NumericError("sparsity invariant violated: more than n*L edges");
  out.m = m;
  finish_tail(ds, n, m, bits, out, sink, after, cs);
}

void finish_graph(Dataset& ds, const KernelSpec& ks, uint32_t rounds,
                  const double* g_full, const uint64_t* keys_in, uint64_t nkeys,
                  bool keys_sorted_unique, bool want_estimates,
                  GraphResult& out, const HostSink* sink, const uint64_t* chunks,
                  uint32_t nchunks) {
  if (chunks && nchunks)
    return finish_graph_chunked(ds, ks, rounds, g_full, keys_in, chunks, nchunks, out, sink);
  cudaStream_t s = ds.stream;
  const uint32_t n = ds.n, d = ds.d;
  const uint32_t bits = index_bits(n);
  const float* pts = ds.pts.as<float>();
  out.n = n;

  // 1. canonical sorted unique public keys
  DevBuf& keys = ds.buf("g.keys", std::max<uint64_t>(nkeys, 1) * 8);
  uint64_t m = nkeys;
  if (keys_sorted_unique) {
    if (m)
      FSGG_CUDA(cudaMemcpyAsync(keys.as<void>(), keys_in, m * 8,
                                cudaMemcpyDeviceToDevice, s));
  } else if (m) {
    public_to_compact_kernel<<<ceil_div_u32(m, 256), 256, 0, s>>>(
        reinterpret_cast<const unsigned long long*>(keys_in),
        keys.as<unsigned long long>(), m, bits);
    FSGG_LAUNCH_CHECK();
    m = sort_unique_compact(ds, keys, m, bits);
    if (m) {
      compact_to_public_kernel<<<ceil_div_u32(m, 256), 256, 0, s>>>(
          keys.as<unsigned long long>(), m, bits);
      FSGG_LAUNCH_CHECK();
    }
    ds.launches += 2;
  }

  // 2 + 3. k_ij once: underflow drop (k_ij < 1e-300) and weights (+ estimates)
  DevBuf& tmp = ds.buf("g.tmp", 8);
  DevBuf& cnt = ds.buf("g.cnt", 16);
  out.underflow = 0;
  {
    const uint64_t mm0 = std::max<uint64_t>(m, 1);
    out.u.ensure(mm0 * 4, s);
    out.v.ensure(mm0 * 4, s);
    out.w.ensure(mm0 * 8, s);
    if (want_estimates) out.est.ensure(mm0 * sizeof(EdgeEstimateDev), s);
  }
  // streamed host output (HostSink): each array's device-to-host copy runs
  // on its own stream as soon as the array is final — v right away (it is
  // the keys' low word), w after the weights, row_ptr and degrees after
  // theirs — overlapping the rest of the finish
  SideStream side;
  cudaStream_t& cs = side.cs;
  cudaEvent_t& ev = side.ev;
  auto after = [&](void* dst, const void* src, size_t bytes) {
    if (!dst || !bytes) return;
    FSGG_CUDA(cudaEventRecord(ev, s));
    FSGG_CUDA(cudaStreamWaitEvent(cs, ev, 0));
    FSGG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, cs));
  };
  const bool early_v = sink && sink->v && m && m <= sink->capacity;
  if (sink) {
    // checked before underflow drops: the capacity must hold the sampled
    // unique pairs (n * L always does; fsgg.h)
    if (m > sink->capacity)
      throw ConfigError("host output capacity below the sampled unique pair count");
    FSGG_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    FSGG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (early_v) {
      keys_to_v_kernel<<<ceil_div_u32(m, 256), 256, 0, s>>>(keys.as<unsigned long long>(), m,
                                                            out.v.as<uint32_t>());
      FSGG_LAUNCH_CHECK();
      ds.launches++;
      after(sink->v, out.v.as<void>(), m * 4);
    }
  }
  if (m) {
    DevBuf& keep = ds.buf("g.keep", m);
    FSGG_CUDA(cudaMemsetAsync(cnt.as<void>(), 0, 16, s));
    (d >= kEdgeWideMinDim ? edges_kernel<true> : edges_kernel<false>)<<<ceil_div_u32(m, 256), 256, 0, s>>>(
        keys.as<unsigned long long>(), m, pts, d, ks.family, ks.sigma, double(rounds), g_full,
        out.u.as<uint32_t>(), out.v.as<uint32_t>(), out.w.as<double>(),
        want_estimates ? out.est.as<EdgeEstimateDev>() : nullptr, keep.as<unsigned char>(),
        cnt.as<unsigned long long>(), early_v ? 0 : 1);
    FSGG_LAUNCH_CHECK();
    ds.launches++;
    unsigned long long dropped = 0;
    FSGG_CUDA(cudaMemcpyAsync(&dropped, cnt.as<void>(), 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    if (dropped) {
      // compact every per-edge array by the keep flags (stable)
      auto compact = [&](DevBuf& arr, size_t elem, const char* name) {
        DevBuf& o = ds.buf(name, m * elem);
        if (elem == 4) {
          cub_call(tmp, s, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, arr.as<uint32_t>(), keep.as<unsigned char>(),
                                              o.as<uint32_t>(), cnt.as<uint64_t>() + 1, m, s);
          });
        } else if (elem == 8) {
          cub_call(tmp, s, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, arr.as<double>(), keep.as<unsigned char>(),
                                              o.as<double>(), cnt.as<uint64_t>() + 1, m, s);
          });
        } else {
          cub_call(tmp, s, [&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, arr.as<EdgeEstimateDev>(),
                                              keep.as<unsigned char>(),
                                              o.as<EdgeEstimateDev>(), cnt.as<uint64_t>() + 1,
                                              m, s);
          });
        }
        FSGG_CUDA(cudaMemcpyAsync(arr.as<void>(), o.as<void>(), (m - dropped) * elem,
                                  cudaMemcpyDeviceToDevice, s));
      };
      compact(out.u, 4, "g.cu");
      compact(out.v, 4, "g.cv");
      compact(out.w, 8, "g.cw");
      if (want_estimates) compact(out.est, sizeof(EdgeEstimateDev), "g.ce");
      ds.launches += 4;
      m -= dropped;
      out.underflow = dropped;
    }
  }
  if (m > uint64_t(n) * rounds)
    throw NumericError("sparsity invariant violated: more than n*L edges");
  out.m = m;

  if (sink) {
    // dropped underflow pairs compacted v: copy it again (after the first
    // copy on the same stream); the weights are final here
    if (!early_v || out.underflow) after(sink->v, out.v.as<void>(), m * 4);
    after(sink->w, out.w.as<void>(), m * 8);
  }

  finish_tail(ds, n, m, bits, out, sink, after, cs);
}

// ---- row-sharded finish (multi-GPU, parallel.py) ----------------------------

void rows_transposed(Dataset& ds, const GraphResult& g, uint32_t* v_out, double* w_out) {
  cudaStream_t s = ds.stream;
  const uint64_t m = g.m;
  if (m == 0) return;
  if (g.tv_sorted && g.tw_sorted) {  // the finish's own transposed order
    FSGG_CUDA(cudaMemcpyAsync(v_out, g.tv_sorted, m * 4, cudaMemcpyDeviceToDevice, s));
    FSGG_CUDA(cudaMemcpyAsync(w_out, g.tw_sorted, m * 8, cudaMemcpyDeviceToDevice, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    return;
  }
  const uint32_t bits = index_bits(ds.n);
  DevBuf& tmp = ds.buf("g.tmp", 8);
  DevBuf& k2 = ds.buf("rt.k2", m * 4);
  DevBuf& w2 = ds.buf("rt.w2", m * 8);
  FSGG_CUDA(cudaMemcpyAsync(v_out, g.v.as<void>(), m * 4, cudaMemcpyDeviceToDevice, s));
  FSGG_CUDA(cudaMemcpyAsync(w_out, g.w.as<void>(), m * 8, cudaMemcpyDeviceToDevice, s));
  cub::DoubleBuffer<uint32_t> dk(v_out, k2.as<uint32_t>());
  cub::DoubleBuffer<double> dv(w_out, w2.as<double>());
  cub_call(tmp, s, [&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, m, 0, int(bits), s);
  });
  if (dk.Current() != v_out)
    FSGG_CUDA(cudaMemcpyAsync(v_out, dk.Current(), m * 4, cudaMemcpyDeviceToDevice, s));
  if (dv.Current() != w_out)
    FSGG_CUDA(cudaMemcpyAsync(w_out, dv.Current(), m * 8, cudaMemcpyDeviceToDevice, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  ds.launches += 4;
}

void rows_degrees(Dataset& ds, const GraphResult& g, const uint32_t* lower_v,
                  const double* lower_w, uint64_t nlower, uint32_t rb, uint32_t re,
                  double* deg_out) {
  cudaStream_t s = ds.stream;
  if (re <= rb) return;
  const uint32_t bits = index_bits(ds.n);
  DevBuf& tmp = ds.buf("g.tmp", 8);
  const uint64_t nl = std::max<uint64_t>(nlower, 1);
  DevBuf& k1 = ds.buf("rd.k1", nl * 4);
  DevBuf& k2 = ds.buf("rd.k2", nl * 4);
  DevBuf& w1 = ds.buf("rd.w1", nl * 8);
  DevBuf& w2 = ds.buf("rd.w2", nl * 8);
  DevBuf& lrp = ds.buf("rd.lrp", size_t(re - rb + 1) * 8);
  const uint32_t* keys = k1.as<uint32_t>();
  const double* vals = w1.as<double>();
  if (nlower) {
    FSGG_CUDA(cudaMemcpyAsync(k1.as<void>(), lower_v, nlower * 4, cudaMemcpyDeviceToDevice, s));
    FSGG_CUDA(cudaMemcpyAsync(w1.as<void>(), lower_w, nlower * 8, cudaMemcpyDeviceToDevice, s));
    // stable: rank order (u ranges ascending) survives within each vertex
    cub::DoubleBuffer<uint32_t> dk(k1.as<uint32_t>(), k2.as<uint32_t>());
    cub::DoubleBuffer<double> dv(w1.as<double>(), w2.as<double>());
    cub_call(tmp, s, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, dk, dv, nlower, 0, int(bits), s);
    });
    keys = dk.Current();
    vals = dv.Current();
  }
  range_ptr_kernel<<<ceil_div_u32(uint64_t(re - rb) + 1, 256), 256, 0, s>>>(
      keys, nlower, rb, re, lrp.as<uint64_t>());
  FSGG_LAUNCH_CHECK();
  rows_degrees_kernel<<<ceil_div_u32(re - rb, 256), 256, 0, s>>>(
      rb, re, lrp.as<uint64_t>(), vals, g.row_ptr.as<uint64_t>(), g.w.as<double>(), deg_out);
  FSGG_LAUNCH_CHECK();
  FSGG_CUDA(cudaStreamSynchronize(s));
  ds.launches += 4;
}

}  // namespace fsgg
