// Level-synchronous tree descent: the device replacement of
// fsg::sample_neighbors_counted (proj/src/sampler.cpp:77-247).
//
// State per level is an entry list grouped by node slot (SoA: query,
// tickets, slot) with a CSR-style offset array goff over the level's 2^l
// slots, so entries of one node stay contiguous exactly like the reference's
// node groups (:131-137). One level is:
//   1. kde_level (kde.cu)      child sums g1, g2 for every entry;
//   2. route_kernel            p = g1/(g1+g2) in fp64, Binomial(t, p) as t
//                              Bernoulli trials on the reference's keyed
//                              splitmix64 stream (bit-exact) or Philox;
//                              size-1 nodes emit (query, source, count) into
//                              a per-query leaf row with an atomic slot;
//   3. one 64-bit exclusive scan of packed (has_left, has_right) flags;
//   4. scatter_kernel / goff_kernel: deterministic stable placement, left
//      children of a node before its right children (:217-222), no atomics.
#include <cub/block/block_load.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_store.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "engine.cuh"
#include "kde_math.cuh"

namespace fsgg {

namespace {

// Relative half-width (of min(p, 1-p)) of the tie guard: 5x the worst p
// error implied by the fp32 child sums' measured relative error (~1e-5).
constexpr double kTieMargin = 1e-4;
// A compute level keeps partial rows deep enough to serve this many levels.
constexpr uint32_t kServeLevels = 5;
// The root's rows are kept deeper (one pass over all n^2 pairs then serves
// every level down to nodes of ~n/2^10); FSGG_ROOT_SERVE overrides.
constexpr uint32_t kServeLevelsRoot = 9;
uint32_t root_serve_levels() {
  const char* e = std::getenv("FSGG_ROOT_SERVE");
  return e ? uint32_t(std::atoi(e)) : kServeLevelsRoot;
}

// Block-value lookups below the root rows (FSGG_BLK_LOOKUP=0 disables).
bool blk_lookup_on() {
  const char* e = std::getenv("FSGG_BLK_LOOKUP");  // read per call: tests toggle it
  return !e || std::atoi(e) != 0;
}

// Levels whose nodes all hold <= this many points are finished depth-first
// (finish.cu); FSGG_DFS_MAX overrides (0 disables).
uint32_t dfs_max_node() {
  static const uint32_t v = [] {
    const char* e = std::getenv("FSGG_DFS_MAX");
    return e ? uint32_t(std::atoi(e)) : kDfsMaxNode;
  }();
  return v;
}

// Children below nodes of this many points that hold one ticket finish as
// walks (walk.cu); FSGG_WALK_MAX overrides (0 disables).
uint32_t walk_max_node() {
  const char* e = std::getenv("FSGG_WALK_MAX");  // read per call: tests toggle it
  return e ? uint32_t(std::atoi(e)) : kWalkMaxNode;
}

// FSGG_ROUTE_FEW=0 keeps the threshold draw test at every level (tests)
bool route_few() {
  const char* e = std::getenv("FSGG_ROUTE_FEW");  // read per call: tests toggle it
  return !(e && e[0] == '0');
}

// node_link (common.cuh) for every heap slot of the tree (reference RNG).
__global__ void node_link_kernel(uint64_t nslots, const uint32_t* __restrict__ tfirst,
                                 const uint32_t* __restrict__ tlast, uint64_t prefix,
                                 uint64_t* __restrict__ out) {
  const uint64_t h = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (h < nslots) out[h] = node_link(prefix, (uint64_t(tfirst[h]) << 32) | tlast[h]);
}

// query_link (common.cuh) of every point: route_kernel reads it instead of
// computing a splitmix64 per entry (~10% of its instructions at C3's deep levels).
__global__ void query_link_kernel(uint32_t n, uint64_t* __restrict__ out) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n) out[q] = query_link(q);
}

// Range request: queries qb.., `tickets` each, leaf rows of that size.
__global__ void range_request_kernel(uint32_t qb, uint32_t nq, uint32_t tickets,
                                     uint32_t* __restrict__ uq, uint32_t* __restrict__ tk,
                                     uint64_t* __restrict__ row_off) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) {
    uq[i] = qb + i;
    tk[i] = tickets;
  }
  if (i <= nq) row_off[i] = uint64_t(i) * tickets;
}

__global__ void init_rows_kernel(const uint32_t* __restrict__ uq,
                                 uint32_t nq, uint32_t* __restrict__ qrow,
                                 uint32_t* __restrict__ eq,
                                 uint32_t* __restrict__ et,
                                 uint32_t* __restrict__ eg,
                                 const uint32_t* __restrict__ tickets) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  qrow[uq[i]] = i;
  eq[i] = uq[i];
  et[i] = tickets[i];
  eg[i] = 0;
}

// proj/src/sampler.cpp:186-225 per entry. Each thread handles kRouteUnroll
// entries (block-strided, coalesced) and issues every load of all of them
// before using any: at deep levels the kernel is a latency-bound stream of
// ~60M entries with little arithmetic.
constexpr int kRouteThreads = 256;
constexpr int kRouteUnroll = 2;
constexpr uint32_t kLeafMark = 0xffffffffu;  // tl of an entry that emitted a leaf

// Packed (has_left, has_right) for the next level's list; with `walk`, a
// child holding exactly one ticket leaves the lists for walk.cu instead.
__device__ __forceinline__ unsigned long long child_flags(uint32_t left, uint32_t t, int walk) {
  const uint32_t right = t - left;
  const bool kl = left > 0 && !(walk && left == 1);
  const bool kr = right > 0 && !(walk && right == 1);
  return (static_cast<unsigned long long>(kl) << 32) | static_cast<unsigned long long>(kr);
}

// capped at 40 registers (6 CTAs per SM, a few spills): the stream of
// entries is latency-bound and the extra warps measured 6% faster
__global__ void __launch_bounds__(kRouteThreads, 6)
    route_kernel(uint32_t E, uint32_t level, const uint32_t* __restrict__ eq,
                 const uint32_t* __restrict__ et, const uint32_t* __restrict__ eg,
                 const double* __restrict__ g1, const double* __restrict__ g2,
                 const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ tlast,
                 uint64_t key_prefix, int rng_mode, uint64_t seed,
                 const uint32_t* __restrict__ qrow, const uint64_t* __restrict__ row_off,
                 uint32_t* __restrict__ row_cnt, uint32_t* __restrict__ leaf_src,
                 uint32_t* __restrict__ leaf_cnt, uint32_t* __restrict__ tl,
                 unsigned long long* __restrict__ flags,
                 unsigned long long* __restrict__ counters, const float* __restrict__ elm,
                 const uint32_t* __restrict__ eprow, const float* __restrict__ row_mass,
                 uint32_t* __restrict__ vlist, uint32_t* __restrict__ vcount, int walk,
                 const uint64_t* __restrict__ nlink, const uint32_t* __restrict__ dE,
                 const uint64_t* __restrict__ qlink, uint64_t few_tickets) {
  constexpr int U = kRouteUnroll;
  if (dE) E = *dE;  // the level's entry count on the device (sync-free levels)
  // Deep levels hold a ticket or two per entry (C3 level 12: 1.25): there the
  // draw test is the fast walks' division-free u (a + b) - a < 0 with the same
  // margin, instead of the thresholds ceil(p 2^53) -/+ M (an fp64 division
  // and three double->integer conversions per entry). The tie guard re-decides
  // everything inside the margin on exact sums, so both forms give the
  // reference's decisions. Grid-uniform: few_tickets = the descent's tickets.
  const bool few = vlist && rng_mode == 0 && few_tickets && uint64_t(E) * 6 >= few_tickets;
  unsigned long long tsum = 0, degen = 0;
  // grid-stride over tiles of kRouteThreads * U entries (index E: sentinel)
  for (uint32_t tile = blockIdx.x; uint64_t(tile) * (kRouteThreads * U) <= E;
       tile += gridDim.x) {
  const uint32_t base = tile * (kRouteThreads * U) + threadIdx.x;
  uint32_t gi[U], q[U], t[U], f[U], l[U];
  double a[U], b[U];
  float em[U], rm[U];
  uint64_t nl[U];  // node link ^ query link
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * kRouteThreads;
    const bool ok = i < E;
    gi[u] = ok ? eg[i] : 0u;
    q[u] = ok ? eq[i] : 0u;
    t[u] = ok ? et[i] : 0u;
    a[u] = ok ? g1[i] : 0.0;
    b[u] = ok ? g2[i] : 0.0;
    em[u] = (ok && elm) ? elm[i] : 0.f;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * kRouteThreads;
    const uint64_t h = ((1ull << level) - 1) + gi[u];
    f[u] = i < E ? tfirst[h] : 0u;
    l[u] = i < E ? tlast[h] : 0u;
    nl[u] = (i < E && nlink) ? (nlink[h] ^ qlink[q[u]]) : 0ull;
    rm[u] = (i < E && row_mass) ? row_mass[eprow ? eprow[i] : i] : 0.f;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * kRouteThreads;
    if (i == E) flags[i] = 0;  // scan sentinel
    if (i >= E) continue;
    tsum += t[u];
    unsigned long long fl = 0;
    if (l[u] - f[u] == 1) {
      // :196-198 leaf: (query, source = first, count = tickets)
      const uint32_t row = qrow[q[u]];
      const uint32_t slot = atomicAdd(row_cnt + row, 1u);
      const uint64_t at = row_off[row] + slot;
      leaf_src[at] = f[u];
      leaf_cnt[at] = t[u];
      tl[i] = kLeafMark;
    } else {
      double p;
      bool verify = false;
      if (a[u] <= kSumFloor && b[u] <= kSumFloor) {  // :207-209
        p = 0.5;
        if (vlist)
          verify = true;  // degenerate by fp32 sums: decided on exact sums
        else
          degen += t[u];
      } else if (few) {
        p = -1.0;  // decided below without p
      } else {
        p = a[u] / (a[u] + b[u]);  // :211
      }
      uint32_t left = 0;
      if (p < 0.0) {
        const uint64_t key = splitmix64(nl[u]);
        const double ssum = a[u] + b[u];
        const double rel = kTieMargin * (1.0 + fmaxf(0.f, -em[u]) / 32.0);
        const double pruned =
            row_mass ? double(exp2f(rm[u] - (kPruneBits - 24.f) - em[u])) : 0.0;
        const double M = fma(rel, fmin(a[u], b[u]), (pruned + 0x1p-51) * ssum);
        bool near = false;
        for (uint32_t c = 0; c < t[u]; ++c) {
          const uint64_t m = splitmix64(key + c) >> 11;
          const double d = fma(double(m) * 0x1p-53, ssum, -a[u]);
          left += d < 0.0 ? 1u : 0u;
          near |= fabs(d) <= M;
        }
        verify |= near;
      } else if (p >= 1.0) {  // rng.hpp:66-67
        left = t[u];
      } else if (p > 0.0) {
        // u_c = (x_c >> 11) * 2^-53 < p  <=>  (x_c >> 11) < ceil(p * 2^53)
        const double P = p * 9007199254740992.0;
        const uint64_t thr = static_cast<uint64_t>(ceil(P));
        if (rng_mode == 0) {
          // RngStream::keyed(seed, kRouteTag, (first<<32)|last, query)
          const uint64_t key =
              nlink ? splitmix64(nl[u])
                    : route_key(key_prefix, (uint64_t(f[u]) << 32) | l[u], uint64_t(q[u]));
          if (vlist) {
            // Tie guard: a draw within the fp32 sums' error bound of p is
            // re-decided on fp64 sums (exact_sums_kernel), which makes the
            // output match the reference's exact backend edge for edge.
            const double rel = kTieMargin * (1.0 + fmaxf(0.f, -em[u]) / 32.0);
            // certified pruning at the compute level skipped < 2^-(B-21) of
            // the ancestor row's mass (B = kPruneBits): an absolute error on
            // p of at most this (3 bits of slack)
            const double pruned =
                row_mass ? double(exp2f(rm[u] - (kPruneBits - 24.f) - em[u])) : 0.0;
            const double M = (rel * fmin(p, 1.0 - p) + pruned) * 9007199254740992.0 + 1.0;
            const uint64_t lo = P > M ? static_cast<uint64_t>(P - M) : 0ull;
            const uint64_t hi = static_cast<uint64_t>(P + M);
            bool near = false;
            for (uint32_t c = 0; c < t[u]; ++c) {
              const uint64_t m = splitmix64(key + c) >> 11;
              left += m < thr ? 1u : 0u;
              near |= (m >= lo) & (m <= hi);
            }
            verify |= near;
          } else {
            for (uint32_t c = 0; c < t[u]; ++c)
              left += (splitmix64(key + c) >> 11) < thr ? 1u : 0u;
          }
        } else {
          const uint2 k = make_uint2(uint32_t(seed), uint32_t(seed >> 32));
          for (uint32_t c = 0; c < t[u]; c += 2) {
            const uint4 r = philox4x32(make_uint4(c >> 1, q[u], f[u], l[u]), k);
            const uint64_t x0 = (uint64_t(r.x) << 32) | r.y;
            const uint64_t x1 = (uint64_t(r.z) << 32) | r.w;
            left += (x0 >> 11) < thr ? 1u : 0u;
            if (c + 1 < t[u]) left += (x1 >> 11) < thr ? 1u : 0u;
          }
        }
      }
      tl[i] = left;
      fl = child_flags(left, t[u], walk);
      if (verify) vlist[atomicAdd(vcount, 1u)] = i;
    }
    flags[i] = fl;
  }
  }  // tiles
  // one atomic per CTA per counter (per-warp atomics on two addresses
  // serialise ~0.5M times a level at 60M entries)
  __shared__ unsigned long long red_t[kRouteThreads / 32], red_d[kRouteThreads / 32];
  for (int o = 16; o; o >>= 1) {
    tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
    degen += __shfl_xor_sync(0xffffffffu, degen, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red_t[threadIdx.x >> 5] = tsum;
    red_d[threadIdx.x >> 5] = degen;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, b = 0;
    for (int k = 0; k < kRouteThreads / 32; ++k) {
      a += red_t[k];
      b += red_d[k];
    }
    if (a) atomicAdd(counters + 0, a);
    if (b) atomicAdd(counters + 1, b);
  }
}

// fp64 child sums for the entries the tie guard flagged: one CTA per entry,
// every term in fp64 with the reference's operation order (kernel_f64),
// fixed-order block reduction. Sub-chunks (tree descendants of ~256+ points)
// whose bounding-box bound is below 2^-80 of the entry's node mass are
// skipped (total < 2^-70 of it: far below the 2^-53 resolution of the
// decision). Grid-strided over the device count: no host synchronisation.
__global__ void __launch_bounds__(256)
    exact_sums_kernel(const float* __restrict__ pts, uint32_t d, int family,
                      double sigma, float scale, uint32_t level, uint32_t depth,
                      const uint32_t* __restrict__ eq, const uint32_t* __restrict__ eg,
                      const float* __restrict__ elm, const uint32_t* __restrict__ tfirst,
                      const uint32_t* __restrict__ tlast, const float* __restrict__ tlo,
                      const float* __restrict__ thi, int has_boxes,
                      const uint32_t* __restrict__ vlist,
                      const uint32_t* __restrict__ vcount, double* __restrict__ g1,
                      double* __restrict__ g2) {
  __shared__ double red[2][256];
  __shared__ unsigned char keep[1024];
  const uint32_t cnt = *vcount;
  for (uint32_t b = blockIdx.x; b < cnt; b += gridDim.x) {
    const uint32_t i = vlist[b];
    const uint64_t h = ((1ull << level) - 1) + eg[i];
    const uint32_t f = tfirst[h], l = tlast[h], mid = f + (l - f) / 2;
    const float* xq = pts + size_t(eq[i]) * d;
    // sub-chunk depth below the node: >= 256 points each, <= 1024 of them
    uint32_t kd = 0;
    while (kd < 10 && level + kd + 1 <= depth && ((l - f) >> (kd + 1)) >= 256) ++kd;
    const uint32_t nsub = 1u << kd;
    const uint64_t hb = ((1ull << (level + kd)) - 1) + (uint64_t(eg[i]) << kd);
    const float lim_base = (elm ? elm[i] : 0.f) - 1.f - 80.f;  // log2 of the skip bound
    for (uint32_t c = threadIdx.x; c < nsub; c += blockDim.x) {
      bool k = true;
      if (has_boxes && kd > 0) {
        float acc = 0.f;
        for (uint32_t a = 0; a < d; ++a) {
          const float v = fmaxf(fmaxf(tlo[(hb + c) * d + a] - xq[a], xq[a] - thi[(hb + c) * d + a]), 0.f);
          acc = (family == 2) ? acc + v : fmaf(v, v, acc);
        }
        const float dist = family == 1 ? sqrtf(acc) : acc;
        const float sz = float(tlast[hb + c] - tfirst[hb + c]);
        k = __log2f(sz) - scale * dist >= lim_base;
      }
      keep[c] = k;
    }
    __syncthreads();
    double s0 = 0.0, s1 = 0.0;
    if (d < 32) {
      for (uint32_t c = 0; c < nsub; ++c) {
        if (!keep[c]) continue;
        const uint32_t cf = kd ? tfirst[hb + c] : f, cl = kd ? tlast[hb + c] : l;
        for (uint32_t j = cf + threadIdx.x; j < cl; j += blockDim.x) {
          const double v = kernel_f64(family, sigma, xq, pts + size_t(j) * d, d);
          if (j < mid)
            s0 += v;
          else
            s1 += v;
        }
      }
    } else {
      // high d: a thread per source, float4 loads and four independent fp64
      // accumulators (the per-tie work is a long dot-product stream; the
      // coordinate order differs from the reference's, which moves k by
      // ~1 ulp — far below the 2^-53 grid the decision is taken on)
      const uint32_t d4 = d & ~3u;
      for (uint32_t c = 0; c < nsub; ++c) {
        if (!keep[c]) continue;
        const uint32_t cf = kd ? tfirst[hb + c] : f, cl = kd ? tlast[hb + c] : l;
        for (uint32_t j = cf + threadIdx.x; j < cl; j += blockDim.x) {
          const float* xj = pts + size_t(j) * d;
          double acc[4] = {0.0, 0.0, 0.0, 0.0};
          const bool al = ((reinterpret_cast<uintptr_t>(xj) | reinterpret_cast<uintptr_t>(xq)) & 15) == 0;
          uint32_t a = 0;
          if (al) {
            for (; a < d4; a += 4) {
              const float4 u = *reinterpret_cast<const float4*>(xq + a);
              const float4 v = __ldg(reinterpret_cast<const float4*>(xj + a));
              const double t0 = double(u.x) - double(v.x), t1 = double(u.y) - double(v.y);
              const double t2 = double(u.z) - double(v.z), t3 = double(u.w) - double(v.w);
              if (family == 2) {
                acc[0] += fabs(t0); acc[1] += fabs(t1); acc[2] += fabs(t2); acc[3] += fabs(t3);
              } else {
                acc[0] = fma(t0, t0, acc[0]); acc[1] = fma(t1, t1, acc[1]);
                acc[2] = fma(t2, t2, acc[2]); acc[3] = fma(t3, t3, acc[3]);
              }
            }
          }
          for (; a < d; ++a) {
            const double t = double(xq[a]) - double(xj[a]);
            acc[a & 3] = family == 2 ? acc[a & 3] + fabs(t) : fma(t, t, acc[a & 3]);
          }
          const double part = (acc[0] + acc[1]) + (acc[2] + acc[3]);
          const double v = family == 2   ? exp(-part / sigma)
                           : family == 1 ? exp(-sqrt(part) / sigma)
                                         : exp(-part / (sigma * sigma));
          if (j < mid)
            s0 += v;
          else
            s1 += v;
        }
      }
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    __syncthreads();
    for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        red[0][threadIdx.x] += red[0][threadIdx.x + w];
        red[1][threadIdx.x] += red[1][threadIdx.x + w];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      g1[i] = fmax(red[0][0], kSumFloor);
      g2[i] = fmax(red[1][0], kSumFloor);
    }
    __syncthreads();
  }
}

// Low-d tie guard (d <= 8): exact_sums_kernel specialised on (D, family):
// unrolled coordinates, 8-byte loads for d = 2, and the exponent scaled by
// a precomputed 1/sigma^2 (1/sigma) instead of a per-term fp64 division —
// the values move by <= 1 ulp, far below the 2^-53 grid the re-decision is
// taken on.
template <int D, int FAM>
__global__ void __launch_bounds__(256)
    exact_sums_lowd_kernel(const float* __restrict__ pts, double sigma, float scale,
                           uint32_t level, uint32_t depth, const uint32_t* __restrict__ eq,
                           const uint32_t* __restrict__ eg, const float* __restrict__ elm,
                           const uint32_t* __restrict__ tfirst,
                           const uint32_t* __restrict__ tlast, const float* __restrict__ tlo,
                           const float* __restrict__ thi, int has_boxes,
                           const uint32_t* __restrict__ vlist,
                           const uint32_t* __restrict__ vcount, double* __restrict__ g1,
                           double* __restrict__ g2, uint32_t first_tie) {
  __shared__ double red[2][256];
  __shared__ unsigned char keep[1024];
  const uint32_t cnt = *vcount;
  const double inv = FAM == 0 ? 1.0 / (sigma * sigma) : 1.0 / sigma;
  for (uint32_t b = first_tie + blockIdx.x; b < cnt; b += gridDim.x) {
    const uint32_t i = vlist[b];
    const uint64_t h = ((1ull << level) - 1) + eg[i];
    const uint32_t f = tfirst[h], l = tlast[h], mid = f + (l - f) / 2;
    const float* xq = pts + size_t(eq[i]) * D;
    double q[D];
#pragma unroll
    for (int k = 0; k < D; ++k) q[k] = double(xq[k]);
    uint32_t kd = 0;
    while (kd < 10 && level + kd + 1 <= depth && ((l - f) >> (kd + 1)) >= 256) ++kd;
    const uint32_t nsub = 1u << kd;
    const uint64_t hb = ((1ull << (level + kd)) - 1) + (uint64_t(eg[i]) << kd);
    const float lim_base = (elm ? elm[i] : 0.f) - 1.f - 80.f;  // log2 of the skip bound
    for (uint32_t c = threadIdx.x; c < nsub; c += blockDim.x) {
      bool k = true;
      if (has_boxes && kd > 0) {
        float acc = 0.f;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const float v = fmaxf(fmaxf(tlo[(hb + c) * D + a] - xq[a], xq[a] - thi[(hb + c) * D + a]), 0.f);
          acc = (FAM == 2) ? acc + v : fmaf(v, v, acc);
        }
        const float dist = FAM == 1 ? sqrtf(acc) : acc;
        const float sz = float(tlast[hb + c] - tfirst[hb + c]);
        k = __log2f(sz) - scale * dist >= lim_base;
      }
      keep[c] = k;
    }
    __syncthreads();
    double s0 = 0.0, s1 = 0.0;
    for (uint32_t c = 0; c < nsub; ++c) {
      if (!keep[c]) continue;
      const uint32_t cf = kd ? tfirst[hb + c] : f, cl = kd ? tlast[hb + c] : l;
      for (uint32_t j = cf + threadIdx.x; j < cl; j += blockDim.x) {
        double x[D];
        if constexpr (D == 2) {
          const float2 v = __ldg(reinterpret_cast<const float2*>(pts) + j);
          x[0] = double(v.x);
          x[1] = double(v.y);
        } else {
#pragma unroll
          for (int a = 0; a < D; ++a) x[a] = double(__ldg(pts + size_t(j) * D + a));
        }
        double t = 0.0;
        if constexpr (FAM == 2) {
#pragma unroll
          for (int a = 0; a < D; ++a) t += fabs(q[a] - x[a]);
        } else {
#pragma unroll
          for (int a = 0; a < D; ++a) t = fma(q[a] - x[a], q[a] - x[a], t);
          if constexpr (FAM == 1) t = sqrt(t);
        }
        const double v = exp(-t * inv);
        if (j < mid)
          s0 += v;
        else
          s1 += v;
      }
    }
    red[0][threadIdx.x] = s0;
    red[1][threadIdx.x] = s1;
    __syncthreads();
    for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) {
        red[0][threadIdx.x] += red[0][threadIdx.x + w];
        red[1][threadIdx.x] += red[1][threadIdx.x + w];
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      g1[i] = fmax(red[0][0], kSumFloor);
      g2[i] = fmax(red[1][0], kSumFloor);
    }
    __syncthreads();
  }
}

// Low-d tie guard split over (tie, sub-chunk) items, one warp each: a
// level-1 tie scans a 500k-point node, and one CTA per tie left the GPU
// nearly idle at the top levels (tens to thousands of ties). Each warp sums
// its sub-chunk's fp64 terms (same terms and skip rule as
// exact_sums_lowd_kernel) lane-strided, reduces them with a fixed butterfly
// and writes one (left, right) partial; tie_finish_kernel adds the
// partials in sub-chunk order, so the result depends only on the (node,
// query). Ties beyond the partial buffer's capacity (max_ties) are left to
// exact_sums_lowd_kernel (first_tie = max_ties) — no host sync needed.
constexpr uint32_t kTieSplitItems = 1u << 22;  // partial buffer: 4M items x 2 doubles
constexpr int kTieSplitThreads = 256;

__device__ __forceinline__ uint32_t tie_sub_depth(uint32_t level, uint32_t depth, uint32_t size) {
  uint32_t kd = 0;
  while (kd < 10 && level + kd + 1 <= depth && (size >> (kd + 1)) >= 256) ++kd;
  return kd;
}

// One warp's fp64 (left, right) sums of entry i over sub-chunk c of its
// node (all lanes return the butterfly-reduced totals).
template <int D, int FAM>
__device__ __forceinline__ void tie_chunk_sums(
    const float* __restrict__ pts, double inv, float scale, uint32_t level, uint32_t depth,
    const uint32_t* __restrict__ eq, const uint32_t* __restrict__ eg,
    const float* __restrict__ elm, const uint32_t* __restrict__ tfirst,
    const uint32_t* __restrict__ tlast, const float* __restrict__ tlo,
    const float* __restrict__ thi, int has_boxes, uint32_t i, uint32_t c, double& r0,
    double& r1) {
  const uint32_t lane = threadIdx.x & 31;
  {
    const uint64_t h = ((1ull << level) - 1) + eg[i];
    const uint32_t f = tfirst[h], l = tlast[h], mid = f + (l - f) / 2;
    const uint32_t kd = tie_sub_depth(level, depth, l - f);
    double s0 = 0.0, s1 = 0.0;
    if (c < (1u << kd)) {
      const float* xq = pts + size_t(eq[i]) * D;
      const uint64_t hb = ((1ull << (level + kd)) - 1) + (uint64_t(eg[i]) << kd) + c;
      bool keep = true;
      if (has_boxes && kd > 0) {
        const float lim_base = (elm ? elm[i] : 0.f) - 1.f - 80.f;
        float acc = 0.f;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const float v = fmaxf(fmaxf(tlo[hb * D + a] - xq[a], xq[a] - thi[hb * D + a]), 0.f);
          acc = (FAM == 2) ? acc + v : fmaf(v, v, acc);
        }
        const float dist = FAM == 1 ? sqrtf(acc) : acc;
        const float sz = float(tlast[hb] - tfirst[hb]);
        keep = __log2f(sz) - scale * dist >= lim_base;
      }
      if (keep) {
        double q[D];
#pragma unroll
        for (int k = 0; k < D; ++k) q[k] = double(xq[k]);
        const uint32_t cf = kd ? tfirst[hb] : f, cl = kd ? tlast[hb] : l;
        for (uint32_t j = cf + lane; j < cl; j += 32) {
          double x[D];
          if constexpr (D == 2) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(pts) + j);
            x[0] = double(v.x);
            x[1] = double(v.y);
          } else {
#pragma unroll
            for (int a = 0; a < D; ++a) x[a] = double(__ldg(pts + size_t(j) * D + a));
          }
          double t = 0.0;
          if constexpr (FAM == 2) {
#pragma unroll
            for (int a = 0; a < D; ++a) t += fabs(q[a] - x[a]);
          } else {
#pragma unroll
            for (int a = 0; a < D; ++a) t = fma(q[a] - x[a], q[a] - x[a], t);
            if constexpr (FAM == 1) t = sqrt(t);
          }
          const double v = exp(-t * inv);
          if (j < mid)
            s0 += v;
          else
            s1 += v;
        }
      }
    }
    for (int o = 16; o; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    }
    r0 = s0;
    r1 = s1;
  }
}

template <int D, int FAM>
__global__ void __launch_bounds__(kTieSplitThreads)
    tie_split_kernel(const float* __restrict__ pts, double sigma, float scale, uint32_t level,
                     uint32_t depth, const uint32_t* __restrict__ eq,
                     const uint32_t* __restrict__ eg, const float* __restrict__ elm,
                     const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ tlast,
                     const float* __restrict__ tlo, const float* __restrict__ thi,
                     int has_boxes, const uint32_t* __restrict__ vlist,
                     const uint32_t* __restrict__ vcount, uint32_t max_chunks,
                     uint32_t max_ties, double* __restrict__ part) {
  const uint32_t ties = min(*vcount, max_ties);
  const uint64_t items = uint64_t(ties) * max_chunks;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warps = uint64_t(gridDim.x) * (kTieSplitThreads / 32);
  const double inv = FAM == 0 ? 1.0 / (sigma * sigma) : 1.0 / sigma;
  for (uint64_t it = blockIdx.x * uint64_t(kTieSplitThreads / 32) + (threadIdx.x >> 5);
       it < items; it += warps) {
    const uint32_t b = uint32_t(it / max_chunks), c = uint32_t(it % max_chunks);
    double s0, s1;
    tie_chunk_sums<D, FAM>(pts, inv, scale, level, depth, eq, eg, elm, tfirst, tlast, tlo, thi,
                           has_boxes, vlist[b], c, s0, s1);
    if (lane == 0) {
      part[it * 2] = s0;
      part[it * 2 + 1] = s1;
    }
  }
}

template <class F>
bool lowd_exact_dispatch(uint32_t d, int family, F&& f) {
  auto by_fam = [&](auto dim) {
    switch (family) {
      case 0: f(dim, std::integral_constant<int, 0>{}); return true;
      case 1: f(dim, std::integral_constant<int, 1>{}); return true;
      case 2: f(dim, std::integral_constant<int, 2>{}); return true;
      default: return false;
    }
  };
  switch (d) {
    case 1: return by_fam(std::integral_constant<int, 1>{});
    case 2: return by_fam(std::integral_constant<int, 2>{});
    case 3: return by_fam(std::integral_constant<int, 3>{});
    case 4: return by_fam(std::integral_constant<int, 4>{});
    case 5: return by_fam(std::integral_constant<int, 5>{});
    case 6: return by_fam(std::integral_constant<int, 6>{});
    case 7: return by_fam(std::integral_constant<int, 7>{});
    case 8: return by_fam(std::integral_constant<int, 8>{});
    default: return false;
  }
}

// High-d tie guard, batched: the flagged entries of one node share its
// sources, so instead of one full pass over the node per tie (C5: 70k rows x
// 784 dims per tie at the root), ties are sorted by node, cut into batches of
// kTieBatch, and each CTA streams one chunk of the node's sources once for a
// whole batch: every source row is read once (float4) and its fp64 squared
// distance to each batch query accumulated in index order over the dims
// (kernel_f64's order), exp in fp64. Per-(tie, chunk) partials are combined
// in chunk order by tie_reduce_kernel, so results are deterministic.
constexpr uint32_t kTieBatchMinDim = 32;  // below: exact_sums_kernel (pruned sub-chunks)
constexpr uint32_t kTieBatchMinNode = 1024;  // smaller nodes: one CTA per tie is cheaper
constexpr uint32_t kTieBatchMaxDim = 3200;    // fp64 batch queries in shared memory (<= 200 KiB)
constexpr int kTieBatch = 8;
constexpr uint32_t kTieChunk = 1024;
constexpr int kTieThreads = 128;

struct TieItem {
  uint32_t first;   // position of the batch's first tie in the sorted list
  uint32_t count;   // ties in the batch (<= kTieBatch)
  uint32_t src0, src1;  // source chunk [src0, src1)
  uint32_t mid;     // node split point
  uint32_t chunk;   // chunk index within the node
  uint32_t nchunks; // chunks of the node
  uint32_t pad;
};

__global__ void __launch_bounds__(kTieThreads)
    tie_batch_kernel(const float* __restrict__ pts, uint32_t d, int family, double sigma,
                     const uint32_t* __restrict__ eq, const uint32_t* __restrict__ sorted,
                     const TieItem* __restrict__ items, uint32_t max_chunks,
                     double* __restrict__ partials) {
  // the batch's queries, converted to fp64 once (a per-term F2F of every
  // batch query kept the conversion (XU) pipe saturated)
  extern __shared__ __align__(16) double tq[];  // [kTieBatch][d]
  __shared__ double red[kTieThreads / 32][kTieBatch][2];
  const TieItem it = items[blockIdx.x];
  for (uint32_t idx = threadIdx.x; idx < it.count * d; idx += blockDim.x) {
    const uint32_t t = idx / d, a = idx % d;
    tq[idx] = double(pts[size_t(eq[sorted[it.first + t]]) * d + a]);
  }
  __syncthreads();
  double s0[kTieBatch], s1[kTieBatch];
#pragma unroll
  for (int t = 0; t < kTieBatch; ++t) s0[t] = s1[t] = 0.0;
  const double inv = family == 0 ? 1.0 / (sigma * sigma) : 1.0 / sigma;
  for (uint32_t j = it.src0 + threadIdx.x; j < it.src1; j += blockDim.x) {
    const float* xj = pts + size_t(j) * d;
    double acc[kTieBatch];
#pragma unroll
    for (int t = 0; t < kTieBatch; ++t) acc[t] = 0.0;
    // four dimensions per step: one 16-byte load of the source and one
    // 16-byte (broadcast) shared-memory load per tie, then 4 fp64 terms
    // each — the scalar loop was bound by shared-memory wavefronts
    uint32_t a = 0;
    if ((d & 3u) == 0) {
      for (; a < d; a += 4) {
        const float4 x4 = __ldg(reinterpret_cast<const float4*>(xj + a));
        const double x0 = x4.x, x1 = x4.y, x2 = x4.z, x3 = x4.w;
#pragma unroll
        for (int t = 0; t < kTieBatch; ++t) {
          if (uint32_t(t) < it.count) {
            const double2 qa = *reinterpret_cast<const double2*>(tq + t * d + a);
            const double2 qb = *reinterpret_cast<const double2*>(tq + t * d + a + 2);
            const double d0 = qa.x - x0, d1 = qa.y - x1;
            const double d2 = qb.x - x2, d3 = qb.y - x3;
            if (family == 2) {
              acc[t] = acc[t] + fabs(d0);
              acc[t] = acc[t] + fabs(d1);
              acc[t] = acc[t] + fabs(d2);
              acc[t] = acc[t] + fabs(d3);
            } else {
              acc[t] = fma(d0, d0, acc[t]);
              acc[t] = fma(d1, d1, acc[t]);
              acc[t] = fma(d2, d2, acc[t]);
              acc[t] = fma(d3, d3, acc[t]);
            }
          }
        }
      }
    }
    for (; a < d; ++a) {
      const double xv = double(__ldg(xj + a));
#pragma unroll
      for (int t = 0; t < kTieBatch; ++t) {
        if (uint32_t(t) < it.count) {
          const double df = tq[t * d + a] - xv;
          acc[t] = family == 2 ? acc[t] + fabs(df) : fma(df, df, acc[t]);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kTieBatch; ++t) {
      if (uint32_t(t) < it.count) {
        const double v = family == 1 ? exp(-sqrt(acc[t]) * inv) : exp(-acc[t] * inv);
        if (j < it.mid)
          s0[t] += v;
        else
          s1[t] += v;
      }
    }
  }
  // fixed-order block reduction: warp butterflies, then warps in order
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int t = 0; t < kTieBatch; ++t) {
    double a0 = s0[t], a1 = s1[t];
    for (int o = 16; o; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if (lane == 0) {
      red[w][t][0] = a0;
      red[w][t][1] = a1;
    }
  }
  __syncthreads();
  if (threadIdx.x < it.count * 2) {
    const uint32_t t = threadIdx.x >> 1, side = threadIdx.x & 1;
    double v = 0.0;
    for (int k = 0; k < kTieThreads / 32; ++k) v += red[k][t][side];
    partials[(size_t(it.first + t) * max_chunks + it.chunk) * 2 + side] = v;
  }
}

// The same recomputation as an fp64 register-tiled product (gaussian and
// exponential kernels, d a multiple of 4): |q - x|^2 = |q|^2 + |x|^2 - 2 q.x
// with every factor an fp32 value held in fp64, so each product is exact and
// only the fp64 accumulation rounds (the direct form has the same property;
// both are the exact sum to ~1e-16 relative per term). The dot products and
// the norms accumulate over the dimensions in index order with one fma per
// term — for x = q the three agree bit for bit and the distance is exactly 0.
// A CTA takes a batch of <= 32 ties against a chunk of the node's sources:
// source tiles of 128 rows and tie rows are staged 16 dimensions at a time
// (coalesced 64-byte row pieces, converted once) and each thread keeps a
// 4 tie x 8 source block of dot products in registers: one DFMA per (tie,
// source, dimension) where tie_batch_kernel spends a DADD and a DFMA and
// re-reads every source row once per 8 ties (C5 root: 24 passes over 220 MB).
constexpr int kTgTies = 32;
constexpr int kTgSrc = 128;
constexpr int kTgK = 16;
constexpr int kTgThreads = 128;

// fp64 squared norms, dimensions in index order (thread per point, rows
// staged through shared memory so the reads stay coalesced)
__global__ void __launch_bounds__(128)
    point_norms_kernel(const float* __restrict__ pts, uint32_t n, uint32_t d,
                       double* __restrict__ xn) {
  __shared__ float tile[128][33];
  const uint32_t j0 = blockIdx.x * 128;
  double acc = 0.0;
  for (uint32_t k0 = 0; k0 < d; k0 += 32) {
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < 128 * 32; idx += 128) {
      const uint32_t r = idx >> 5, c = idx & 31;
      tile[r][c] = (j0 + r < n && k0 + c < d) ? __ldg(pts + size_t(j0 + r) * d + k0 + c) : 0.f;
    }
    __syncthreads();
    const uint32_t kc = min(32u, d - k0);
    for (uint32_t c = 0; c < kc; ++c) {
      const double v = double(tile[threadIdx.x][c]);
      acc = fma(v, v, acc);
    }
  }
  if (j0 + threadIdx.x < n) xn[j0 + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(kTgThreads)
    tie_gemm_kernel(const float* __restrict__ pts, uint32_t d, int family, double sigma,
                    const uint32_t* __restrict__ eq, const uint32_t* __restrict__ sorted,
                    const TieItem* __restrict__ items, uint32_t max_chunks,
                    const double* __restrict__ xn, double* __restrict__ partials) {
  __shared__ __align__(16) double qs[kTgK][kTgTies];
  __shared__ __align__(16) double xs[kTgK][kTgSrc + 1];
  __shared__ uint32_t qrow[kTgTies];
  const TieItem it = items[blockIdx.x];
  // warp ty holds ties 8 ty .. 8 ty + 7 (its shared-memory reads of the tie
  // rows are broadcasts), lane tx sources tx, tx + 32, tx + 64, tx + 96
  // (conflict-free 8-byte reads): 12-16 shared-memory cycles per 32 DFMA
  // (16 cycles) and warp — a 4 x 8 block with the sources in the wider
  // direction was bound by shared-memory bandwidth
  const uint32_t tid = threadIdx.x, tx = tid & 31u, ty = tid >> 5;
  if (tid < uint32_t(kTgTies)) qrow[tid] = tid < it.count ? eq[sorted[it.first + tid]] : 0xffffffffu;
  __syncthreads();
  const double inv = family == 0 ? 1.0 / (sigma * sigma) : 1.0 / sigma;
  double qn[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    const uint32_t r = qrow[8 * ty + a];
    qn[a] = r != 0xffffffffu ? xn[r] : 0.0;
  }
  double s0[8], s1[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) s0[a] = s1[a] = 0.0;
  const bool warp_on = 8 * ty < it.count;  // this warp's ties exist
  for (uint32_t j0 = it.src0; j0 < it.src1; j0 += kTgSrc) {
    double acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (uint32_t k0 = 0; k0 < d; k0 += kTgK) {
      __syncthreads();  // the previous tiles have been read
      {  // tie rows: 32 x 16 values, one float4 per thread
        const uint32_t t = tid >> 2, kq = (tid & 3u) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (qrow[t] != 0xffffffffu && k0 + kq < d)
          v = __ldg(reinterpret_cast<const float4*>(pts + size_t(qrow[t]) * d + k0 + kq));
        qs[kq][t] = double(v.x);
        qs[kq + 1][t] = double(v.y);
        qs[kq + 2][t] = double(v.z);
        qs[kq + 3][t] = double(v.w);
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {  // source rows: 128 x 16 values
        const uint32_t idx = tid + uint32_t(kTgThreads) * r;
        const uint32_t sj = idx >> 2, kq = (idx & 3u) * 4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j0 + sj < it.src1 && k0 + kq < d)
          v = __ldg(reinterpret_cast<const float4*>(pts + size_t(j0 + sj) * d + k0 + kq));
        xs[kq][sj] = double(v.x);
        xs[kq + 1][sj] = double(v.y);
        xs[kq + 2][sj] = double(v.z);
        xs[kq + 3][sj] = double(v.w);
      }
      __syncthreads();
      if (warp_on) {
#pragma unroll
        for (int kk = 0; kk < kTgK; ++kk) {
          double q[8], x[4];
#pragma unroll
          for (int a = 0; a < 8; ++a) q[a] = qs[kk][8 * ty + a];
#pragma unroll
          for (int b = 0; b < 4; ++b) x[b] = xs[kk][tx + 32 * b];
#pragma unroll
          for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(q[a], x[b], acc[a][b]);
        }
      }
    }
    if (warp_on) {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t j = j0 + tx + 32 * b;
        if (j < it.src1) {
          const double xj = xn[j];
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            if (8 * ty + a < it.count) {
              const double d2 = fmax((qn[a] + xj) - 2.0 * acc[a][b], 0.0);
              const double v = family == 1 ? exp(-sqrt(d2) * inv) : exp(-d2 * inv);
              if (j < it.mid)
                s0[a] += v;
              else
                s1[a] += v;
            }
          }
        }
      }
    }
  }
  // the warp's 32 source lanes: fixed butterfly
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    double a0 = s0[a], a1 = s1[a];
    for (int o = 16; o; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    }
    if (tx == 0 && 8 * ty + a < it.count) {
      double* p = partials + (size_t(it.first + 8 * ty + a) * max_chunks + it.chunk) * 2;
      p[0] = a0;
      p[1] = a1;
    }
  }
}

__global__ void gather_u32_kernel(uint32_t n, const uint32_t* __restrict__ idx,
                                  const uint32_t* __restrict__ src, uint32_t* __restrict__ out) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n) out[b] = src[idx[b]];
}

__global__ void node_range_kernel(uint32_t n, const uint32_t* __restrict__ slot, uint64_t hbase,
                                  const uint32_t* __restrict__ tfirst,
                                  const uint32_t* __restrict__ tlast, uint32_t* __restrict__ out) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < n) {
    out[2 * b] = tfirst[hbase + slot[b]];
    out[2 * b + 1] = tlast[hbase + slot[b]];
  }
}

__global__ void tie_reduce_kernel(uint32_t count, const uint32_t* __restrict__ sorted,
                                  const uint32_t* __restrict__ nchunks_of,
                                  uint32_t max_chunks, const double* __restrict__ partials,
                                  double* __restrict__ g1, double* __restrict__ g2) {
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= count) return;
  double a = 0.0, c = 0.0;
  for (uint32_t k = 0; k < nchunks_of[b]; ++k) {
    a += partials[(size_t(b) * max_chunks + k) * 2];
    c += partials[(size_t(b) * max_chunks + k) * 2 + 1];
  }
  const uint32_t i = sorted[b];
  g1[i] = fmax(a, kSumFloor);
  g2[i] = fmax(c, kSumFloor);
}

// Re-decide the flagged entries on the fp64 sums (reference stream).
// The tie guard's re-decision of entry i on its (now fp64) child sums
// a = g1[i], b = g2[i] (sampler.cpp:205-222 on the keyed stream).
__device__ __forceinline__ void reroute_entry(uint32_t i, uint32_t level,
                                              const uint32_t* __restrict__ eq,
                                              const uint32_t* __restrict__ et,
                                              const uint32_t* __restrict__ eg, double a,
                                              double bb, const uint32_t* __restrict__ tfirst,
                                              const uint32_t* __restrict__ tlast,
                                              uint64_t key_prefix, uint32_t* __restrict__ tl,
                                              unsigned long long* __restrict__ flags,
                                              unsigned long long* __restrict__ counters,
                                              int walk) {
  const uint64_t h = ((1ull << level) - 1) + eg[i];
  const uint32_t f = tfirst[h], l = tlast[h], q = eq[i], t = et[i];
  double p;
  if (a <= kSumFloor && bb <= kSumFloor) {
    p = 0.5;
    atomicAdd(counters + 1, static_cast<unsigned long long>(t));
  } else {
    p = a / (a + bb);
  }
  uint32_t left;
  if (p <= 0.0) {
    left = 0;
  } else if (p >= 1.0) {
    left = t;
  } else {
    const uint64_t thr = static_cast<uint64_t>(ceil(p * 9007199254740992.0));
    const uint64_t key = route_key(key_prefix, (uint64_t(f) << 32) | l, uint64_t(q));
    left = 0;
    for (uint32_t c = 0; c < t; ++c) left += (splitmix64(key + c) >> 11) < thr ? 1u : 0u;
  }
  tl[i] = left;
  flags[i] = child_flags(left, t, walk);
}

__global__ void reroute_kernel(uint32_t level, const uint32_t* __restrict__ eq,
                               const uint32_t* __restrict__ et,
                               const uint32_t* __restrict__ eg,
                               const double* __restrict__ g1,
                               const double* __restrict__ g2,
                               const uint32_t* __restrict__ tfirst,
                               const uint32_t* __restrict__ tlast, uint64_t key_prefix,
                               const uint32_t* __restrict__ vlist,
                               const uint32_t* __restrict__ vcount,
                               uint32_t* __restrict__ tl,
                               unsigned long long* __restrict__ flags,
                               unsigned long long* __restrict__ counters, int walk) {
  const uint32_t cnt = *vcount;
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < cnt;
       b += gridDim.x * blockDim.x) {
    const uint32_t i = vlist[b];
    reroute_entry(i, level, eq, et, eg, g1[i], g2[i], tfirst, tlast, key_prefix, tl, flags,
                  counters, walk);
  }
}

// Low-d tie guard, second half (replaces tie_split_reduce_kernel +
// reroute_kernel): one warp per tie adds its sub-chunk partials in
// tie_split_reduce order (lane-strided, fixed butterfly), stores the sums
// and re-decides the entry; ties past the partial buffer (max_ties) already
// hold exact_sums_lowd_kernel's sums.
__global__ void __launch_bounds__(256)
    tie_finish_kernel(uint32_t level, const uint32_t* __restrict__ eq,
                      const uint32_t* __restrict__ et, const uint32_t* __restrict__ eg,
                      double* __restrict__ g1, double* __restrict__ g2,
                      const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ tlast,
                      uint64_t key_prefix, const uint32_t* __restrict__ vlist,
                      const uint32_t* __restrict__ vcount, uint32_t max_chunks,
                      uint32_t max_ties, const double* __restrict__ part,
                      uint32_t* __restrict__ tl, unsigned long long* __restrict__ flags,
                      unsigned long long* __restrict__ counters, int walk) {
  const uint32_t ties = *vcount;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < ties;
       b += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t i = vlist[b];
    double a, c;
    if (b < max_ties) {
      a = 0.0;
      c = 0.0;
      const double* p = part + size_t(b) * max_chunks * 2;
      for (uint32_t k = lane; k < max_chunks; k += 32) {
        a += p[2 * k];
        c += p[2 * k + 1];
      }
      for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
      }
      a = fmax(a, kSumFloor);
      c = fmax(c, kSumFloor);
      if (lane == 0) {
        g1[i] = a;
        g2[i] = c;
      }
    } else {
      a = g1[i];
      c = g2[i];
    }
    if (lane == 0)
      reroute_entry(i, level, eq, et, eg, a, c, tfirst, tlast, key_prefix, tl, flags, counters,
                    walk);
  }
}

// Low-d tie guard for levels whose nodes are one sub-chunk (< 512 points):
// split, reduce and re-decision in one pass, one warp per tie. The sums are
// bit-identical to tie_split_kernel + tie_finish_kernel with one chunk (a
// single partial added to zeros).
template <int D, int FAM>
__global__ void __launch_bounds__(kTieSplitThreads)
    tie_onepass_kernel(const float* __restrict__ pts, double sigma, float scale, uint32_t level,
                       uint32_t depth, const uint32_t* __restrict__ eq,
                       const uint32_t* __restrict__ et, const uint32_t* __restrict__ eg,
                       const float* __restrict__ elm, const uint32_t* __restrict__ tfirst,
                       const uint32_t* __restrict__ tlast, const float* __restrict__ tlo,
                       const float* __restrict__ thi, int has_boxes,
                       const uint32_t* __restrict__ vlist, const uint32_t* __restrict__ vcount,
                       double* __restrict__ g1, double* __restrict__ g2, uint64_t key_prefix,
                       uint32_t* __restrict__ tl, unsigned long long* __restrict__ flags,
                       unsigned long long* __restrict__ counters, int walk) {
  const uint32_t ties = *vcount;
  const double inv = FAM == 0 ? 1.0 / (sigma * sigma) : 1.0 / sigma;
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < ties;
       b += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t i = vlist[b];
    double s0, s1;
    tie_chunk_sums<D, FAM>(pts, inv, scale, level, depth, eq, eg, elm, tfirst, tlast, tlo, thi,
                           has_boxes, i, 0, s0, s1);
    if ((threadIdx.x & 31) == 0) {
      const double a = fmax(s0, kSumFloor), c = fmax(s1, kSumFloor);
      g1[i] = a;
      g2[i] = c;
      reroute_entry(i, level, eq, et, eg, a, c, tfirst, tlast, key_prefix, tl, flags, counters,
                    walk);
    }
  }
}

// Child sums from the partial row of the entry's ancestor at the last
// compute level (row_level = level - j): that row holds the ancestor's
// descendants 2^rd wide and its pairwise-sum pyramid.
constexpr int kLookupThreads = 256;
constexpr int kLookupUnroll = 4;  // entries per thread, all loads issued first

__global__ void __launch_bounds__(kLookupThreads)
    lookup_sums_kernel(uint32_t E, uint32_t level, uint32_t j, uint32_t rd,
                       const uint32_t* __restrict__ eg, const uint32_t* __restrict__ eprow,
                       const double* __restrict__ rows, const double* __restrict__ pyr,
                       const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ tlast,
                       double* __restrict__ g1, double* __restrict__ g2,
                       unsigned long long* __restrict__ evals, const uint32_t* __restrict__ dE) {
  constexpr int U = kLookupUnroll;
  if (dE) E = *dE;
  unsigned long long ev = 0;
  for (uint32_t tile = blockIdx.x; uint64_t(tile) * (kLookupThreads * U) < E;
       tile += gridDim.x) {
  const uint32_t base = tile * (kLookupThreads * U) + threadIdx.x;
  uint32_t g[U], pr[U], size[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * kLookupThreads;
    g[u] = i < E ? eg[i] : 0u;
    pr[u] = i < E ? eprow[i] : 0u;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t h = ((1ull << level) - 1) + g[u];
    size[u] = base + u * kLookupThreads < E ? tlast[h] - tfirst[h] : 0u;
  }
  // the node is descendant idx (depth j) of the row's node; its children are
  // entries 2 idx, 2 idx + 1 at depth j + 1: the row itself at the deepest
  // level, else the row's pairwise-sum pyramid (kde.cu), else (short rows)
  // `span` consecutive buckets each
  const bool two = pyr || j + 1 == rd;
  const uint32_t span = two ? 1u : 1u << (rd - j - 1);
  double a[U], b[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    a[u] = b[u] = 0.0;
    if (size[u] >= 2) {
      const uint32_t idx = g[u] & ((1u << j) - 1u);
      const double* src = j + 1 == rd || !pyr
                              ? rows + (size_t(pr[u]) << rd) + size_t(2 * idx) * span
                              : pyr + (size_t(pr[u]) << rd) + ((2u << j) - 2u) + 2 * idx;
      if (two) {
        a[u] = src[0];
        b[u] = src[1];
      } else {
        for (uint32_t k = 0; k < span; ++k) a[u] += src[k];
        for (uint32_t k = 0; k < span; ++k) b[u] += src[span + k];
      }
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * kLookupThreads;
    if (i >= E) continue;
    if (size[u] < 2) {
      g1[i] = g2[i] = 0.0;
    } else {
      g1[i] = fmax(a[u], kSumFloor);
      g2[i] = fmax(b[u], kSumFloor);
      ev += size[u];
    }
  }
  }  // tiles
  __shared__ unsigned long long red_ev[kLookupThreads / 32];
  for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
  if ((threadIdx.x & 31) == 0) red_ev[threadIdx.x >> 5] = ev;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < kLookupThreads / 32; ++k) t += red_ev[k];
    if (t) atomicAdd(evals, t);
  }
}

// log2 of a positive normal double to fp32 accuracy: exponent field plus
// MUFU.LG2 of the mantissa. An entry's mass exponent only scales pruning
// thresholds and tie margins (which carry bits of slack); the fp64 log2 it
// replaces was ~45% of scatter_kernel's instructions.
__device__ __forceinline__ float log2_mass(double g) {
  const long long b = __double_as_longlong(g);
  const int e = int((b >> 52) & 0x7ff) - 1023;
  const float m = float(__longlong_as_double((b & 0x000fffffffffffffLL) | 0x3ff0000000000000LL));
  return float(e) + __log2f(m);
}

__device__ __forceinline__ uint32_t hiw(unsigned long long x) {
  return uint32_t(x >> 32);
}
__device__ __forceinline__ uint32_t low(unsigned long long x) {
  return uint32_t(x);
}

// Stable placement: slot g's left children occupy [A[s]+B[s], A[e]+B[s]),
// its right children [A[e]+B[s], A[e]+B[e]), where A/B are the exclusive
// prefix counts of left/right children and [s, e) = goff[g], goff[g+1].
// Each child entry also carries log2 of its node's mass (the child sum just
// computed), the lower bound the next level's pruning is certified against.
__global__ void scatter_kernel(uint32_t E, const uint32_t* __restrict__ eq,
                               const uint32_t* __restrict__ et,
                               const uint32_t* __restrict__ eg,
                               const uint32_t* __restrict__ tl,
                               const unsigned long long* __restrict__ flags,
                               const uint32_t* __restrict__ goff,
                               const unsigned long long* __restrict__ P,
                               const double* __restrict__ g1,
                               const double* __restrict__ g2,
                               uint32_t* __restrict__ neq,
                               uint32_t* __restrict__ net,
                               uint32_t* __restrict__ neg,
                               float* __restrict__ nelm,
                               const uint32_t* __restrict__ eprow,
                               uint32_t* __restrict__ neprow, int self_rows,
                               uint32_t level, uint32_t* __restrict__ wq,
                               uint32_t* __restrict__ wh, float* __restrict__ welm,
                               uint32_t* __restrict__ wcount, uint32_t* __restrict__ wrow,
                               float* __restrict__ wrm, const float* __restrict__ elm,
                               int rows2, const uint32_t* __restrict__ dE) {
  if (dE) E = *dE;
  __shared__ uint32_t wtot[8], wbase;
  for (uint32_t tile = blockIdx.x; uint64_t(tile) * blockDim.x < E; tile += gridDim.x) {
  const uint32_t i = tile * blockDim.x + threadIdx.x;
  uint32_t nw = 0, wmask = 0;  // single-ticket children handed to the walk
  uint32_t g = 0, q = 0;
  // the child sums are loaded with the entry (the walk writes below used to
  // wait for them after the reservation's barriers)
  double ga = 0.0, gb = 0.0;
  if (i < E) {
    const unsigned long long fl = flags[i];
    const uint32_t t = et[i], l = tl[i];
    g = eg[i];
    q = eq[i];
    if (l != kLeafMark) {
      ga = g1[i];
      gb = g2[i];
    }
    if (wq && l != kLeafMark) {
      wmask = (l == 1 ? 1u : 0u) | (t - l == 1 ? 2u : 0u);
      nw = __popc(wmask);
    }
    if (fl) {
      const unsigned long long Pi = P[i];
      const uint32_t prow = self_rows ? i : (eprow ? eprow[i] : 0u);
      if (hiw(fl)) {
        const uint32_t pos = hiw(Pi) + low(P[goff[g]]);
        neq[pos] = q;
        net[pos] = l;
        neg[pos] = 2 * g;
        nelm[pos] = log2_mass(ga);
        neprow[pos] = prow;
      }
      if (low(fl)) {
        const uint32_t pos = hiw(P[goff[g + 1]]) + low(Pi);
        neq[pos] = q;
        net[pos] = t - l;
        neg[pos] = 2 * g + 1;
        nelm[pos] = log2_mass(gb);
        neprow[pos] = prow;
      }
    }
  }
  if (!wq) continue;
  // CTA-aggregated reservation in the walk list: one atomic per CTA (a
  // per-warp atomic on the single counter serialised ~2M times a level).
  // Order within the list is irrelevant: walks are independent and leaves
  // land in per-query rows.
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = nw;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= uint32_t(o)) incl += y;
  }
  if (lane == 31) wtot[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (uint32_t k = 0; k < blockDim.x / 32; ++k) {
      const uint32_t c = wtot[k];
      wtot[k] = t;
      t += c;
    }
    wbase = t ? atomicAdd(wcount, t) : 0u;
  }
  __syncthreads();
  const uint32_t cta_base = wbase;
  const uint32_t warp_off = wtot[warp];
  __syncthreads();  // wtot / wbase are rewritten by the next tile
  if (nw == 0) continue;
  uint32_t pos = cta_base + warp_off + incl - nw;
  const uint32_t hbase = (1u << (level + 1)) - 1;
  // rows2: this level kept two-deep partial rows (kde.cu, per-sub-chunk
  // rows), so the walk's first child sums are in row i (walk.cu reads them
  // if no later compute level reused the rows); wrm = log2 of this entry's
  // node mass, the pruning scale of those partials
  const uint32_t rw = rows2 ? i : 0xffffffffu;
  const float rm = rows2 && elm ? elm[i] : 0.f;
  if (wmask & 1u) {
    wq[pos] = q;
    wh[pos] = hbase + 2 * g;
    welm[pos] = float(int((__double_as_longlong(ga) >> 52) & 0x7ff) - 1023);
    wrow[pos] = rw;
    wrm[pos] = rm;
    ++pos;
  }
  if (wmask & 2u) {
    wq[pos] = q;
    wh[pos] = hbase + 2 * g + 1;
    welm[pos] = float(int((__double_as_longlong(gb) >> 52) & 0x7ff) - 1023);
    wrow[pos] = rw;
    wrm[pos] = rm;
  }
  }  // tiles
}

// Exclusive scan of the E + 1 packed child flags (the last one is route's
// zero sentinel, so P[E] = the next level's (left, right) totals) with the
// entry count read on the device: one pass, decoupled look-back. Tiles are
// taken in order from a per-level counter, so every predecessor a tile waits
// on belongs to a running CTA. Tile states are (epoch << 2 | kind) words
// written after their value (kind 1: the tile's aggregate, 2: its inclusive
// prefix) with a fence in between; the epoch (level + 1) makes the words of
// earlier levels invisible, so the state array is cleared once per descent.
// The thread holding index E also writes the next level's entry count.
constexpr int kScanThreads = 256;
#ifndef FSGG_SCAN_ITEMS
#define FSGG_SCAN_ITEMS 16
#endif
#ifndef FSGG_SCAN_CTAS
#define FSGG_SCAN_CTAS 4
#endif
constexpr int kScanItems = FSGG_SCAN_ITEMS;
constexpr uint32_t kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__global__ void __launch_bounds__(kScanThreads)
    flags_scan_kernel(const uint32_t* __restrict__ dE, const unsigned long long* __restrict__ flags,
                      unsigned long long* __restrict__ P, uint32_t* __restrict__ tstate,
                      unsigned long long* __restrict__ tagg, unsigned long long* __restrict__ tinc,
                      uint32_t* __restrict__ tctr, uint32_t epoch, uint32_t* __restrict__ e_next) {
  using Load = cub::BlockLoad<unsigned long long, kScanThreads, kScanItems,
                              cub::BLOCK_LOAD_WARP_TRANSPOSE>;
  using Store = cub::BlockStore<unsigned long long, kScanThreads, kScanItems,
                                cub::BLOCK_STORE_WARP_TRANSPOSE>;
  using Scan = cub::BlockScan<unsigned long long, kScanThreads>;
  __shared__ union {
    typename Load::TempStorage load;
    typename Store::TempStorage store;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_prefix;
  const uint32_t n = *dE + 1;
  const uint32_t ntiles = (n + kScanTile - 1) / kScanTile;
  const uint32_t lane = threadIdx.x & 31;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint32_t base = tile * kScanTile;
    const uint32_t valid = min(kScanTile, n - base);
    unsigned long long v[kScanItems];
    Load(tmp.load).Load(flags + base, v, int(valid), 0ull);
    __syncthreads();
    unsigned long long agg;
    Scan(tmp.scan).ExclusiveSum(v, v, agg);
    if (threadIdx.x < 32) {
      unsigned long long excl = 0;
      if (tile == 0) {
        if (lane == 0) {
          tinc[0] = agg;
          __threadfence();
          atomicExch(tstate, (epoch << 2) | 2u);
        }
      } else {
        if (lane == 0) {
          tagg[tile] = agg;
          __threadfence();
          atomicExch(tstate + tile, (epoch << 2) | 1u);
        }
        int pred = int(tile) - 1;
        for (;;) {
          const int tt = pred - int(lane);
          uint32_t st = (epoch << 2) | 2u;
          unsigned long long val = 0;
          if (tt >= 0) {
            do {
              st = ld_volatile(tstate + tt);
            } while ((st >> 2) != epoch);
            __threadfence();
            val = (st & 3u) == 2u ? ld_volatile(tinc + tt) : ld_volatile(tagg + tt);
          }
          const unsigned inc = __ballot_sync(0xffffffffu, (st & 3u) == 2u);
          const int stop = inc ? __ffs(inc) - 1 : 31;
          unsigned long long c = int(lane) <= stop ? val : 0ull;
          for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
          excl += c;
          if (inc) break;
          pred -= 32;
        }
        if (lane == 0) {
          tinc[tile] = excl + agg;
          __threadfence();
          atomicExch(tstate + tile, (epoch << 2) | 2u);
        }
      }
      if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    const unsigned long long pre = s_prefix;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] += pre;
    // the sentinel (index n - 1 = E): its exclusive prefix is the level total
    const uint32_t last = n - 1 - base;
    if (last < kScanTile && threadIdx.x == last / kScanItems) {
      unsigned long long tot = 0;
#pragma unroll
      for (int k = 0; k < kScanItems; ++k)
        if (uint32_t(k) == last % kScanItems) tot = v[k];
      *e_next = uint32_t(tot >> 32) + uint32_t(tot);
    }
    __syncthreads();
    Store(tmp.store).Store(P + base, v, int(valid));
    __syncthreads();
  }
}

__global__ void goff_kernel(uint32_t G, const uint32_t* __restrict__ goff,
                            const unsigned long long* __restrict__ P,
                            uint32_t* __restrict__ ngoff) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < G) {
    const unsigned long long Ps = P[goff[g]], Pe = P[goff[g + 1]];
    ngoff[2 * g] = hiw(Ps) + low(Ps);
    ngoff[2 * g + 1] = hiw(Pe) + low(Ps);
  } else if (g == G) {
    const unsigned long long Pe = P[goff[G]];
    ngoff[2 * G] = hiw(Pe) + low(Pe);
  }
}

__global__ void row_ends_kernel(const uint64_t* __restrict__ row_off,
                                const uint32_t* __restrict__ row_cnt,
                                uint32_t nq, uint64_t* __restrict__ ends) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) ends[i] = row_off[i] + row_cnt[i];
}

// Sort the flagged entries by node, cut node groups into batches, one work
// item per (batch, source chunk); partial sums reduced per tie in chunk order.
void batched_tie_sums(Dataset& ds, const KernelSpec& ks, uint32_t level, const uint32_t* eq,
                      const uint32_t* eg, const uint32_t* vlist, uint32_t cnt, double* g1,
                      double* g2) {
  cudaStream_t s = ds.stream;
  const TreeTable& t = ds.tree;
  DevBuf& sorted = ds.buf("s.tie_sorted", size_t(cnt) * 4);
  DevBuf& tmp = ds.buf("s.tie_tmp", 8);
  const int bits = 32;
  size_t tb = 0;
  FSGG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, vlist, sorted.as<uint32_t>(), int(cnt), 0,
                                           bits, s));
  tmp.ensure(tb, s);
  FSGG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.as<void>(), tb, vlist, sorted.as<uint32_t>(),
                                           int(cnt), 0, bits, s));
  // entries are grouped by node slot in index order, so sorted indices are
  // grouped by node: read their slots back and build the batches on the host
  std::vector<uint32_t> slot(cnt);
  DevBuf& dslot = ds.buf("s.tie_slot", size_t(cnt) * 4);
  gather_u32_kernel<<<ceil_div_u32(cnt, 256), 256, 0, s>>>(cnt, sorted.as<uint32_t>(), eg,
                                                           dslot.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  FSGG_CUDA(cudaMemcpyAsync(slot.data(), dslot.as<void>(), size_t(cnt) * 4,
                            cudaMemcpyDeviceToHost, s));
  std::vector<uint32_t> hf(cnt), hl(cnt);
  FSGG_CUDA(cudaStreamSynchronize(s));
  // node ranges of the distinct slots
  const uint64_t hbase = (1ull << level) - 1;
  std::vector<TieItem> items;
  std::vector<uint32_t> nch(cnt, 0);
  uint32_t max_chunks = 1;
  {
    // fetch first/last for every tie's node (small: cnt entries)
    DevBuf& df = ds.buf("s.tie_f", size_t(cnt) * 8);
    node_range_kernel<<<ceil_div_u32(cnt, 256), 256, 0, s>>>(
        cnt, dslot.as<uint32_t>(), hbase, t.first.as<uint32_t>(), t.last.as<uint32_t>(),
        df.as<uint32_t>());
    FSGG_LAUNCH_CHECK();
    std::vector<uint32_t> fl(size_t(cnt) * 2);
    FSGG_CUDA(cudaMemcpyAsync(fl.data(), df.as<void>(), size_t(cnt) * 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    for (uint32_t b = 0; b < cnt; ++b) {
      hf[b] = fl[2 * b];
      hl[b] = fl[2 * b + 1];
    }
  }
  // the register-tiled product (tie_gemm_kernel) for gaussian / exponential
  // kernels and d a multiple of 4; FSGG_TIE_GEMM=0 keeps tie_batch_kernel
  const char* tg_env = std::getenv("FSGG_TIE_GEMM");  // read per call: tests toggle it
  // ... and when the level's nodes hold a few ties each (a 32-tie tile costs
  // the same with 2 ties as with 8: measured on C5, the tiles win from ~3
  // ties per node; FSGG_TIE_GEMM_MIN overrides)
  const char* tm_env = std::getenv("FSGG_TIE_GEMM_MIN");
  const uint32_t tg_min = tm_env ? uint32_t(std::atoi(tm_env)) : 3u;
  uint32_t tie_nodes = cnt ? 1 : 0;
  for (uint32_t b = 1; b < cnt; ++b) tie_nodes += slot[b] != slot[b - 1];
  const bool gemm = ks.family != 2 && (ds.d & 3u) == 0 && !(tg_env && tg_env[0] == '0') &&
                    cnt >= tg_min * tie_nodes;
  const uint32_t batch = gemm ? uint32_t(kTgTies) : uint32_t(kTieBatch);
  // source chunk: kTieChunk, shortened (to >= 128 sources) when the level's
  // batches x chunks would not give every SM several CTAs
  uint64_t batch_sources = 0;
  for (uint32_t b = 0; b < cnt;) {
    uint32_t e = b + 1;
    while (e < cnt && slot[e] == slot[b] && e - b < batch) ++e;
    batch_sources += hl[b] - hf[b];
    b = e;
  }
  const uint64_t want_items = uint64_t(ds.num_sms) * (gemm ? 4 : 16);
  uint32_t chunk_len = kTieChunk;
  while (chunk_len > 128 && batch_sources / chunk_len < want_items) chunk_len >>= 1;
  for (uint32_t b = 0; b < cnt;) {
    uint32_t e = b + 1;
    while (e < cnt && slot[e] == slot[b] && e - b < batch) ++e;
    const uint32_t f = hf[b], l = hl[b], mid = f + (l - f) / 2;
    const uint32_t chunks = std::max<uint32_t>(1, (l - f + chunk_len - 1) / chunk_len);
    max_chunks = std::max(max_chunks, chunks);
    for (uint32_t c = 0; c < chunks; ++c) {
      TieItem it;
      it.first = b;
      it.count = e - b;
      it.src0 = f + c * chunk_len;
      it.src1 = std::min(l, it.src0 + chunk_len);
      it.mid = mid;
      it.chunk = c;
      it.nchunks = chunks;
      it.pad = 0;
      items.push_back(it);
    }
    for (uint32_t k = b; k < e; ++k) nch[k] = chunks;
    b = e;
  }
  DevBuf& ditems = ds.buf("s.tie_items", items.size() * sizeof(TieItem));
  DevBuf& dnch = ds.buf("s.tie_nch", size_t(cnt) * 4);
  DevBuf& parts = ds.buf("s.tie_parts", size_t(cnt) * max_chunks * 16);
  FSGG_CUDA(cudaMemcpyAsync(ditems.as<void>(), items.data(), items.size() * sizeof(TieItem),
                            cudaMemcpyHostToDevice, s));
  FSGG_CUDA(cudaMemcpyAsync(dnch.as<void>(), nch.data(), size_t(cnt) * 4, cudaMemcpyHostToDevice, s));
  if (gemm) {
    DevBuf& xn = ds.buf("s.tie_xn", size_t(ds.n) * 8);
    if (!ds.tie_xn_ready) {  // once per point set
      point_norms_kernel<<<ceil_div_u32(ds.n, 128), 128, 0, s>>>(ds.pts.as<float>(), ds.n, ds.d,
                                                                xn.as<double>());
      FSGG_LAUNCH_CHECK();
      ds.tie_xn_ready = true;
      ds.launches++;
    }
    tie_gemm_kernel<<<uint32_t(items.size()), kTgThreads, 0, s>>>(
        ds.pts.as<float>(), ds.d, ks.family, ks.sigma, eq, sorted.as<uint32_t>(),
        ditems.as<TieItem>(), max_chunks, xn.as<double>(), parts.as<double>());
  } else {
    const size_t smem = size_t(kTieBatch) * ds.d * 8;
    FSGG_CUDA(cudaFuncSetAttribute(tie_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(std::max<size_t>(smem, 48u << 10))));
    tie_batch_kernel<<<uint32_t(items.size()), kTieThreads, smem, s>>>(
        ds.pts.as<float>(), ds.d, ks.family, ks.sigma, eq, sorted.as<uint32_t>(),
        ditems.as<TieItem>(), max_chunks, parts.as<double>());
  }
  FSGG_LAUNCH_CHECK();
  tie_reduce_kernel<<<ceil_div_u32(cnt, 128), 128, 0, s>>>(cnt, sorted.as<uint32_t>(),
                                                          dnch.as<uint32_t>(), max_chunks,
                                                          parts.as<double>(), g1, g2);
  FSGG_LAUNCH_CHECK();
  ds.launches += 5;
}

}  // namespace

// Pruning threshold (log2 units) of one descent. Exact backend: kPruneBits.
// Fast backend: a sub-chunk is skipped below 2^-B of half the entry's node
// mass and a node has <= 2^20 sub-chunks, so a level skips <= 2^(19 - B) of
// every node's mass; B = 19 + log2((depth + 1) / eps) makes that
// eps / (depth + 1) per level. Since a query reaches node N with probability
// g_N / g_full and the masses of one level's nodes add up to g_full, each
// level moves the query's sampling distribution by <= eps / (depth + 1) in
// total variation: <= eps over the whole descent.
float prune_bits_for(const SampleRequest& req, const TreeTable& t) {
  if (!(req.fast_epsilon > 0.0)) return kPruneBits;
  const double b = 19.0 + std::log2(double(t.depth + 1) / req.fast_epsilon);
  return float(std::min<double>(kPruneBits, std::max(20.0, std::ceil(b))));
}

// record_sums: one EntryRecord per entry of nodes with >= 2 points.
__global__ void record_entries_kernel(uint32_t E, uint32_t level, const uint32_t* __restrict__ eq,
                                      const uint32_t* __restrict__ eg,
                                      const uint32_t* __restrict__ tfirst,
                                      const uint32_t* __restrict__ tlast,
                                      const double* __restrict__ g1,
                                      const double* __restrict__ g2, EntryRecord* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  const uint64_t slot = (uint64_t(1) << level) - 1 + eg[i];
  EntryRecord r;
  r.level = level;
  r.query = eq[i];
  r.first = tfirst[slot];
  r.last = tlast[slot];
  const bool split = r.last - r.first >= 2;
  r.left = split ? g1[i] : 0.0;
  r.right = split ? g2[i] : 0.0;
  out[i] = r;
}

void sample_counted(Dataset& ds, const KernelSpec& ks, const SampleRequest& req_in,
                    SampleResult& out) {
  SampleRequest req_rec;
  if (req_in.record_sums) {
    req_rec = req_in;
    req_rec.walk = false;
    req_rec.dfs_finish = false;
  }
  const SampleRequest& req = req_in.record_sums ? req_rec : req_in;
  out.records.clear();
  cudaStream_t s = ds.stream;
  if (!ds.tree_valid) build_tree(ds);
  const TreeTable& t = ds.tree;
  const uint32_t nq =
      req.range ? req.range_count : static_cast<uint32_t>(req.queries.size());
  out.nq = nq;
  uint64_t total = 0;
  if (req.range) {
    if (uint64_t(req.range_begin) + nq > ds.n) throw ConfigError("query range out of bounds");
    total = uint64_t(nq) * req.range_tickets;
  } else {
    for (uint32_t x : req.tickets) total += x;
  }
  out.total_tickets = total;
  if (total > 0xffffffffull)
    throw ConfigError("total tickets exceed 2^32 - 1 (entries are 32-bit)");

  // queries, tickets, leaf row offsets: generated on the device for a range
  // request, else uploaded
  out.uq.ensure(size_t(nq) * 4 + 4, s);
  out.row_off.ensure(size_t(nq + 1) * 8, s);
  out.row_cnt.ensure(size_t(nq) * 4 + 4, s);
  out.leaf_src.ensure(total * 4 + 4, s);
  out.leaf_cnt.ensure(total * 4 + 4, s);
  DevBuf& dtk = ds.buf("s.tickets", size_t(nq) * 4 + 4);
  DevBuf& qrow = ds.buf("s.qrow", size_t(ds.n) * 4);
  if (req.range) {
    range_request_kernel<<<ceil_div_u32(uint64_t(nq) + 1, 256), 256, 0, s>>>(
        req.range_begin, nq, req.range_tickets, out.uq.as<uint32_t>(), dtk.as<uint32_t>(),
        out.row_off.as<uint64_t>());
    FSGG_LAUNCH_CHECK();
    ds.launches++;
  } else {
    std::vector<uint64_t> row_off(nq + 1, 0);
    for (uint32_t i = 0; i < nq; ++i) row_off[i + 1] = row_off[i] + req.tickets[i];
    FSGG_CUDA(cudaMemcpyAsync(out.uq.as<void>(), req.queries.data(), size_t(nq) * 4,
                              cudaMemcpyHostToDevice, s));
    FSGG_CUDA(cudaMemcpyAsync(dtk.as<void>(), req.tickets.data(), size_t(nq) * 4,
                              cudaMemcpyHostToDevice, s));
    FSGG_CUDA(cudaMemcpyAsync(out.row_off.as<void>(), row_off.data(),
                              size_t(nq + 1) * 8, cudaMemcpyHostToDevice, s));
  }
  FSGG_CUDA(cudaMemsetAsync(out.row_cnt.as<void>(), 0, size_t(nq) * 4 + 4, s));
  if (req.want_root_sums) out.groot.ensure(size_t(nq) * 8 + 8, s);

  // double-buffered entry lists, capacity = total tickets (>= entries)
  const uint64_t cap = std::max<uint64_t>(total, 1);
  DevBuf* eq[2];
  DevBuf* et[2];
  DevBuf* eg[2];
  DevBuf* elm[2];
  DevBuf* eprow[2];
  for (int b = 0; b < 2; ++b) {
    const std::string k = std::to_string(b);
    eq[b] = &ds.buf("s.eq" + k, cap * 4);
    et[b] = &ds.buf("s.et" + k, cap * 4);
    eg[b] = &ds.buf("s.eg" + k, cap * 4);
    elm[b] = &ds.buf("s.elm" + k, cap * 4);
    eprow[b] = &ds.buf("s.eprow" + k, cap * 4);
  }
  // Partial rows of the last compute level serve the following levels.
  DevBuf& row_mass = ds.buf("s.row_mass", 8);
  DevBuf& lookup_evals = ds.buf("s.lookup_evals", 8);
  FSGG_CUDA(cudaMemsetAsync(lookup_evals.as<void>(), 0, 8, s));
  if (!ds.kde_ws) ds.kde_ws = std::make_unique<KdeWorkspace>();
  ds.kde_ws->direct_evals.ensure(8, s);
  FSGG_CUDA(cudaMemsetAsync(ds.kde_ws->direct_evals.as<void>(), 0, 8, s));
  bool have_rows = false;
  // the last level that wrote ws.partials (and their depth): the walks read
  // two-deep rows only if nothing overwrote them after
  uint32_t part_level = 0, part_depth = 0;
  uint32_t row_level = 0, row_depth = 0;
  DevBuf& g1 = ds.buf("s.g1", cap * 8);
  DevBuf& g2 = ds.buf("s.g2", cap * 8);
  DevBuf& tl = ds.buf("s.tl", cap * 4);
  DevBuf& flags = ds.buf("s.flags", (cap + 1) * 8);
  DevBuf& P = ds.buf("s.scan", (cap + 1) * 8);
  const uint64_t max_slots = 1ull << t.depth;
  DevBuf* goff[2] = {&ds.buf("s.goff0", (max_slots + 1) * 4),
                     &ds.buf("s.goff1", (max_slots + 1) * 4)};
  // per-level counters (tickets, degenerate draws, tie count, spare) and the
  // entry count of every level (elog[0] = nq; the scan writes elog[l + 1]):
  // read once after the descent
  constexpr uint32_t kMaxLevelsLog = 64;
  DevBuf& lvc = ds.buf("s.lvc", kMaxLevelsLog * 4 * 8);
  DevBuf& elog = ds.buf("s.elog", (kMaxLevelsLog + 2) * 4);
  FSGG_CUDA(cudaMemsetAsync(lvc.as<void>(), 0, kMaxLevelsLog * 4 * 8, s));
  FSGG_CUDA(cudaMemsetAsync(elog.as<void>(), 0, (kMaxLevelsLog + 2) * 4, s));
  FSGG_CUDA(cudaMemcpyAsync(elog.as<void>(), &nq, 4, cudaMemcpyHostToDevice, s));
  // decoupled look-back scan state (flags_scan_kernel), cleared per descent
  const uint64_t max_tiles = (cap + 1 + kScanTile - 1) / kScanTile;
  DevBuf& tstate = ds.buf("s.scan_state", max_tiles * 4 + kMaxLevelsLog * 4);
  DevBuf& tagg = ds.buf("s.scan_agg", max_tiles * 8);
  DevBuf& tinc = ds.buf("s.scan_inc", max_tiles * 8);
  FSGG_CUDA(cudaMemsetAsync(tstate.as<void>(), 0, max_tiles * 4 + kMaxLevelsLog * 4, s));
  uint32_t* tctr = tstate.as<uint32_t>() + max_tiles;
  const bool verify = req.rng_mode == 0 && req.verify_ties;
  DevBuf& vlist = ds.buf("s.vlist", verify ? cap * 4 : 4);
  if (!ds.kde_ws) ds.kde_ws = std::make_unique<KdeWorkspace>();
  KdeWorkspace& ws = *ds.kde_ws;
  ws.prune_bits = prune_bits_for(req, t);
  // single-ticket walk list (walk.cu), filled by scatter_kernel
  const bool walk_on = req.walk && walk_supported(ds.d) && walk_max_node() > 0;
  DevBuf& wq = ds.buf("s.wq", walk_on ? cap * 4 : 4);
  DevBuf& wh = ds.buf("s.wh", walk_on ? cap * 4 : 4);
  DevBuf& welm = ds.buf("s.welm", walk_on ? cap * 4 : 4);
  DevBuf& wrow = ds.buf("s.wrow", walk_on ? cap * 4 : 4);
  DevBuf& wrm = ds.buf("s.wrm", walk_on ? cap * 4 : 4);
  DevBuf& wcount = ds.buf("s.wcount", 8);
  FSGG_CUDA(cudaMemsetAsync(wcount.as<void>(), 0, 8, s));

  init_rows_kernel<<<ceil_div_u32(std::max<uint32_t>(nq, 1), 256), 256, 0, s>>>(
      out.uq.as<uint32_t>(), nq, qrow.as<uint32_t>(), eq[0]->as<uint32_t>(),
      et[0]->as<uint32_t>(), eg[0]->as<uint32_t>(), dtk.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  ds.launches++;
  const uint32_t goff0[2] = {0, nq};
  FSGG_CUDA(cudaMemcpyAsync(goff[0]->as<void>(), goff0, 8, cudaMemcpyHostToDevice, s));

  // level-0 entries are a contiguous point range (full builds and shards)
  const bool contiguous =
      nq > 0 && (req.range || uint64_t(req.queries.back()) - req.queries.front() + 1 == nq);
  const uint32_t first_query = req.range ? req.range_begin : (nq ? req.queries.front() : 0u);
  const uint64_t prefix = route_key_prefix(req.seed);
  // per-slot node links of the keyed stream: an entry's key is then one
  // splitmix64 of (node link ^ query link) instead of three
  const uint64_t nslots = (uint64_t(2) << t.depth) - 1;
  DevBuf& nlink = ds.buf("s.nlink", req.rng_mode == 0 ? nslots * 8 : 8);
  if (req.rng_mode == 0) {
    node_link_kernel<<<ceil_div_u32(nslots, 256), 256, 0, s>>>(
        nslots, t.first.as<uint32_t>(), t.last.as<uint32_t>(), prefix, nlink.as<uint64_t>());
    FSGG_LAUNCH_CHECK();
    ds.launches++;
  }
  DevBuf& qlink = ds.buf("s.qlink", req.rng_mode == 0 ? size_t(ds.n) * 8 : 8);
  if (req.rng_mode == 0) {
    query_link_kernel<<<ceil_div_u32(ds.n, 256), 256, 0, s>>>(ds.n, qlink.as<uint64_t>());
    FSGG_LAUNCH_CHECK();
    ds.launches++;
  }
  const uint64_t* nlink_p = req.rng_mode == 0 ? nlink.as<uint64_t>() : nullptr;
  const uint64_t* qlink_p = req.rng_mode == 0 ? qlink.as<uint64_t>() : nullptr;
  // E: the current level's entry count when known on the host (E_known);
  // E_hi: an upper bound otherwise. Sync-free descent (low d): a level's
  // kernels read the count from elog on the device and grid-stride, so the
  // host only synchronises before the levels whose launch geometry needs the
  // exact count (tiled KDE levels); statistics are read once at the end.
  uint32_t E = nq;
  bool E_known = true;
  uint64_t E_hi = nq;
  int cur = 0;
  out.entries_per_level.clear();
  out.tickets_per_level.clear();
  out.degenerate_draws = 0;
  out.tie_verified = 0;
  out.kde = KdeStats{};
  out.peak_entries = 0;
  // FSGG_TRACE=1: per-level phase times (CUDA events on the launch stream)
  // and host wall time to stderr.
  const bool trace = std::getenv("FSGG_TRACE") != nullptr;
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
  if (trace)
    for (auto& e : tev) FSGG_CUDA(cudaEventCreate(&e));
  const char* sf_env = std::getenv("FSGG_SYNC_FREE");
  const bool lite = ds.d <= 8 && !trace && !req.record_sums &&
                    !(req.dfs_finish && dfs_finish_supported(ds.d) && dfs_max_node() > 0) &&
                    !(sf_env && std::atoi(sf_env) == 0);
  const uint32_t nsm = uint32_t(ds.num_sms);
  // grid of a grid-strided kernel over n items, span items per CTA
  auto grid_of = [&](uint64_t n, uint32_t span, uint32_t per_sm) {
    return uint32_t(std::max<uint64_t>(
        1, std::min<uint64_t>((n + span - 1) / span, uint64_t(nsm) * per_sm)));
  };
  uint32_t levels_run = 0;
  for (uint32_t level = 0;; ++level) {
    if (E_known && E == 0) break;
    if (level > t.depth) {
      if (E_known) throw NumericError("descent exceeded tree depth");
      break;  // sync-free: checked on the level counts below
    }
    const uint32_t G = 1u << level;
    const uint32_t* dE = elog.as<uint32_t>() + level;
    // the exact count, when the next launch needs it
    auto sync_E = [&] {
      if (E_known) return;
      uint32_t* hw = reinterpret_cast<uint32_t*>(ds.host_words());
      FSGG_CUDA(cudaMemcpyAsync(hw, dE, 4, cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      E = *hw;
      E_known = true;
      E_hi = E;
    };
    const uint32_t smax_level = uint32_t((uint64_t(ds.n) + (1ull << level) - 1) >> level);
    if (req.dfs_finish && dfs_finish_supported(ds.d) && smax_level <= dfs_max_node()) {
      if (level == 0 && req.want_root_sums) {
        // the root's sums are the degree KDE g_full: compute them first
        LevelView lv0;
        lv0.level = 0;
        lv0.num_slots = 1;
        lv0.num_entries = E;
        lv0.eq = eq[cur]->as<uint32_t>();
        lv0.eg = eg[cur]->as<uint32_t>();
        lv0.goff = goff[cur]->as<uint32_t>();
        lv0.prune = req.prune;
        lv0.prune_bits = ws.prune_bits;
        KdeStats scratch;
        kde_level(ds, ks, lv0, g1.as<double>(), g2.as<double>(), out.groot.as<double>(), ws,
                  scratch, 1, nullptr);
      }
      // every remaining level is finished depth-first per entry (finish.cu)
      DevBuf& st = ds.buf("s.dfs_stats", (4 * 64 + 1) * 8);
      FSGG_CUDA(cudaMemsetAsync(st.as<void>(), 0, (4 * 64 + 1) * 8, s));
      DfsArgs a;
      a.E = E;
      a.level = level;
      a.eq = eq[cur]->as<uint32_t>();
      a.et = et[cur]->as<uint32_t>();
      a.eg = eg[cur]->as<uint32_t>();
      a.key_prefix = prefix;
      a.seed = req.seed;
      a.rng_mode = req.rng_mode;
      a.verify = verify ? 1 : 0;
      a.qrow = qrow.as<uint32_t>();
      a.row_off = out.row_off.as<uint64_t>();
      a.row_cnt = out.row_cnt.as<uint32_t>();
      a.leaf_src = out.leaf_src.as<uint32_t>();
      a.leaf_cnt = out.leaf_cnt.as<uint32_t>();
      a.stats = st.as<unsigned long long>();
      const auto w0 = std::chrono::steady_clock::now();
      dfs_finish(ds, ks, a);
      std::vector<unsigned long long> h(4 * 64 + 1);
      FSGG_CUDA(cudaMemcpyAsync(h.data(), st.as<void>(), h.size() * 8, cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      for (uint32_t lv2 = level; lv2 < 64 && h[lv2]; ++lv2) {
        out.entries_per_level.push_back(h[lv2]);
        out.tickets_per_level.push_back(h[64 + lv2]);
        out.kde.evals += h[128 + lv2];
        out.kde.performed += h[128 + lv2];
        out.degenerate_draws += h[192 + lv2];
        out.peak_entries = std::max<uint64_t>(out.peak_entries, h[lv2]);
      }
      out.tie_verified += h[256];
      if (trace)
        std::fprintf(stderr, "fsgg levels %u..: depth-first finish of %u entries %.3fms\n",
                     level, E,
                     std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now() - w0).count());
      E = 0;
      break;
    }
    const auto wall0 = std::chrono::steady_clock::now();
    const KdeStats kde0 = out.kde;
    const bool lookup = have_rows && level - row_level < row_depth;
    // below the root rows' reach, the symmetric root's block values still
    // hold every child sum while children are unions of its blocks
    const bool blk_lookup = !lookup && have_rows && row_level == 0 && level > 0 &&
                            ws.sym_Lb > 0 && level + 1 <= ws.sym_Lb && blk_lookup_on();
    if (!lite || (!lookup && !blk_lookup && !kde_level_sync_free(ds, ks, level))) sync_E();
    if (E_known && E == 0) break;
    ++levels_run;
    const uint32_t En = E_known ? E : uint32_t(E_hi);  // grid bound
    const uint32_t* dEp = E_known ? nullptr : dE;
    if (trace) FSGG_CUDA(cudaEventRecord(tev[0], s));
    if (!lite) {
      out.entries_per_level.push_back(E);
      out.peak_entries = std::max<uint64_t>(out.peak_entries, E);
    }
    LevelView lv;
    lv.level = level;
    lv.num_slots = G;
    lv.num_entries = En;
    lv.dE = dEp;
    lv.eq = eq[cur]->as<uint32_t>();
    lv.eg = eg[cur]->as<uint32_t>();
    lv.elm = level == 0 ? nullptr : elm[cur]->as<float>();
    lv.prune = req.prune;
    lv.prune_bits = ws.prune_bits;
    lv.goff = goff[cur]->as<uint32_t>();
    if (level == 0 && contiguous) lv.qbase = first_query;
    bool self_rows = false;
    // (lookup levels accumulate their reference-equivalent evaluations on the
    // device; read once after the descent — no host sync per level)
    if (blk_lookup) {
      block_lookup_sums(ds, En, level, eq[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(),
                        g1.as<double>(), g2.as<double>(), lookup_evals.as<unsigned long long>(),
                        dEp);
    } else if (lookup) {
      lookup_sums_kernel<<<grid_of(En, kLookupThreads * kLookupUnroll, 16), kLookupThreads, 0, s>>>(
          En, level, level - row_level, row_depth, eg[cur]->as<uint32_t>(),
          eprow[cur]->as<uint32_t>(), ws.partials.as<double>(),
          ws.pyr_depth == row_depth ? ws.pyr.as<double>() : nullptr,
          t.first.as<uint32_t>(),
          t.last.as<uint32_t>(), g1.as<double>(), g2.as<double>(),
          lookup_evals.as<unsigned long long>(), dEp);
      FSGG_LAUNCH_CHECK();
      ds.launches++;
    } else {
      uint32_t rd = 0;
      kde_level(ds, ks, lv, g1.as<double>(), g2.as<double>(),
                level == 0 && req.want_root_sums ? out.groot.as<double>() : nullptr, ws,
                out.kde, level == 0 ? root_serve_levels() : kServeLevels, &rd);
      have_rows = rd > 1;
      if (rd > 0) {
        part_level = level;
        part_depth = rd;
      }
      if (have_rows) {
        self_rows = true;
        row_level = level;
        row_depth = rd;
        if (req.prune && req.verify_ties && req.rng_mode == 0) {
          row_mass.ensure(size_t(E) * 4, s);
          if (level == 0)
            FSGG_CUDA(cudaMemsetAsync(row_mass.as<void>(), 0, size_t(E) * 4, s));
          else
            FSGG_CUDA(cudaMemcpyAsync(row_mass.as<void>(), elm[cur]->as<void>(),
                                      size_t(E) * 4, cudaMemcpyDeviceToDevice, s));
        }
      }
    }

    if (req.record_sums) {
      DevBuf& rb = ds.buf("s.records", size_t(E) * sizeof(EntryRecord));
      record_entries_kernel<<<ceil_div_u32(E, 256), 256, 0, s>>>(
          E, level, eq[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(), t.first.as<uint32_t>(),
          t.last.as<uint32_t>(), g1.as<double>(), g2.as<double>(), rb.as<EntryRecord>());
      FSGG_LAUNCH_CHECK();
      const size_t o = out.records.size();
      out.records.resize(o + E);
      FSGG_CUDA(cudaMemcpyAsync(out.records.data() + o, rb.as<void>(),
                                size_t(E) * sizeof(EntryRecord), cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
    }
    if (trace) FSGG_CUDA(cudaEventRecord(tev[1], s));
    // children (level + 1) below walk_max_node points with one ticket walk
    const uint32_t smax_child =
        uint32_t((uint64_t(ds.n) + (1ull << (level + 1)) - 1) >> (level + 1));
    const int wk = walk_on && level < t.depth && smax_child <= walk_max_node() ? 1 : 0;
    unsigned long long* counters = lvc.as<unsigned long long>() + 4 * size_t(level);
    uint32_t* vcount = reinterpret_cast<uint32_t*>(counters + 2);
    route_kernel<<<grid_of(uint64_t(En) + 1, kRouteThreads * kRouteUnroll, 12),
                   kRouteThreads, 0, s>>>(
        En, level, eq[cur]->as<uint32_t>(), et[cur]->as<uint32_t>(),
        eg[cur]->as<uint32_t>(), g1.as<double>(), g2.as<double>(),
        t.first.as<uint32_t>(), t.last.as<uint32_t>(), prefix, req.rng_mode,
        req.seed, qrow.as<uint32_t>(), out.row_off.as<uint64_t>(),
        out.row_cnt.as<uint32_t>(), out.leaf_src.as<uint32_t>(),
        out.leaf_cnt.as<uint32_t>(), tl.as<uint32_t>(),
        flags.as<unsigned long long>(), counters,
        level == 0 ? nullptr : elm[cur]->as<float>(),
        self_rows ? nullptr : eprow[cur]->as<uint32_t>(),
        (have_rows && req.prune) ? row_mass.as<float>() : nullptr,
        verify ? vlist.as<uint32_t>() : nullptr, vcount, wk, nlink_p, dEp, qlink_p,
        nlink_p && route_few() ? out.total_tickets : 0ull);
    FSGG_LAUNCH_CHECK();
    if (verify && ds.d >= kTieBatchMinDim && ds.d <= kTieBatchMaxDim &&
        smax_level >= kTieBatchMinNode) {
      // high d: batched fp64 recomputation (tie_batch_kernel), then reroute
      uint32_t* hc = reinterpret_cast<uint32_t*>(ds.host_words());
      FSGG_CUDA(cudaMemcpyAsync(hc, vcount, 4, cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      const uint32_t cnt = *hc;
      if (cnt > 0) {
        batched_tie_sums(ds, ks, level, eq[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(),
                         vlist.as<uint32_t>(), cnt, g1.as<double>(), g2.as<double>());
        reroute_kernel<<<ds.num_sms, 256, 0, s>>>(
            level, eq[cur]->as<uint32_t>(), et[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(),
            g1.as<double>(), g2.as<double>(), t.first.as<uint32_t>(), t.last.as<uint32_t>(),
            prefix, ds.buf("s.tie_sorted", 4).as<uint32_t>(), vcount, tl.as<uint32_t>(),
            flags.as<unsigned long long>(), counters, wk);
        FSGG_LAUNCH_CHECK();
        ds.launches += 1;
      }
    } else if (verify) {
      const bool lowd_done = lowd_exact_dispatch(ds.d, ks.family, [&](auto dim, auto fam) {
        constexpr int D = decltype(dim)::value;
        constexpr int FAM = decltype(fam)::value;
        const float* lm = level == 0 ? nullptr : elm[cur]->as<float>();
        const int boxes = t.has_boxes && req.prune ? 1 : 0;
        // the level's largest node fixes the partial layout (sub-chunks per tie)
        uint32_t kd = 0;
        while (kd < 10 && level + kd + 1 <= t.depth && (smax_level >> (kd + 1)) >= 256) ++kd;
        const uint32_t max_chunks = 1u << kd;
        const uint32_t max_ties = kTieSplitItems / max_chunks;
        if (max_chunks == 1) {  // one pass: sums, re-decision (no partial buffer)
          tie_onepass_kernel<D, FAM><<<ds.num_sms * 8, kTieSplitThreads, 0, s>>>(
              ds.pts.as<float>(), ks.sigma, ks.scale, level, t.depth, eq[cur]->as<uint32_t>(),
              et[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(), lm, t.first.as<uint32_t>(),
              t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(), boxes,
              vlist.as<uint32_t>(), vcount, g1.as<double>(), g2.as<double>(), prefix,
              tl.as<uint32_t>(), flags.as<unsigned long long>(), counters, wk);
          ds.launches += 1;
          return;
        }
        DevBuf& part = ds.buf("s.tie_part", size_t(kTieSplitItems) * 16);
        tie_split_kernel<D, FAM><<<ds.num_sms * 8, kTieSplitThreads, 0, s>>>(
            ds.pts.as<float>(), ks.sigma, ks.scale, level, t.depth, eq[cur]->as<uint32_t>(),
            eg[cur]->as<uint32_t>(), lm, t.first.as<uint32_t>(), t.last.as<uint32_t>(),
            t.lo.as<float>(), t.hi.as<float>(), boxes, vlist.as<uint32_t>(), vcount,
            max_chunks, max_ties, part.as<double>());
        // overflow ties (more than the partial buffer holds): one CTA each,
        // launched only when the level can have that many
        if (uint64_t(En) > max_ties) {
          exact_sums_lowd_kernel<D, FAM><<<ds.num_sms * 4, 256, 0, s>>>(
              ds.pts.as<float>(), ks.sigma, ks.scale, level, t.depth, eq[cur]->as<uint32_t>(),
              eg[cur]->as<uint32_t>(), lm, t.first.as<uint32_t>(), t.last.as<uint32_t>(),
              t.lo.as<float>(), t.hi.as<float>(), boxes, vlist.as<uint32_t>(), vcount,
              g1.as<double>(), g2.as<double>(), max_ties);
          ds.launches += 1;
        }
        tie_finish_kernel<<<ds.num_sms * 4, 256, 0, s>>>(
            level, eq[cur]->as<uint32_t>(), et[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(),
            g1.as<double>(), g2.as<double>(), t.first.as<uint32_t>(), t.last.as<uint32_t>(),
            prefix, vlist.as<uint32_t>(), vcount, max_chunks, max_ties, part.as<double>(),
            tl.as<uint32_t>(), flags.as<unsigned long long>(), counters, wk);
        ds.launches += 2;
      });
      if (!lowd_done) {
        exact_sums_kernel<<<ds.num_sms * 4, 256, 0, s>>>(
            ds.pts.as<float>(), ds.d, ks.family, ks.sigma, ks.scale, level, t.depth,
            eq[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(),
            level == 0 ? nullptr : elm[cur]->as<float>(), t.first.as<uint32_t>(),
            t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(),
            t.has_boxes && req.prune ? 1 : 0, vlist.as<uint32_t>(), vcount, g1.as<double>(),
            g2.as<double>());
        FSGG_LAUNCH_CHECK();
        reroute_kernel<<<ds.num_sms, 256, 0, s>>>(
            level, eq[cur]->as<uint32_t>(), et[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(),
            g1.as<double>(), g2.as<double>(), t.first.as<uint32_t>(), t.last.as<uint32_t>(),
            prefix, vlist.as<uint32_t>(), vcount, tl.as<uint32_t>(),
            flags.as<unsigned long long>(), counters, wk);
        ds.launches += 2;
      }
      FSGG_LAUNCH_CHECK();
    }

    if (trace) FSGG_CUDA(cudaEventRecord(tev[2], s));
    if (level + 1 > kMaxLevelsLog) throw NumericError("descent exceeded the level log");
    flags_scan_kernel<<<grid_of(uint64_t(En) + 1, kScanTile, FSGG_SCAN_CTAS), kScanThreads, 0, s>>>(
        dE, flags.as<unsigned long long>(), P.as<unsigned long long>(), tstate.as<uint32_t>(),
        tagg.as<unsigned long long>(), tinc.as<unsigned long long>(), tctr + level, level + 1,
        elog.as<uint32_t>() + level + 1);
    FSGG_LAUNCH_CHECK();
    const int nxt = cur ^ 1;
    scatter_kernel<<<grid_of(En, 256, 16), 256, 0, s>>>(
        En, eq[cur]->as<uint32_t>(), et[cur]->as<uint32_t>(), eg[cur]->as<uint32_t>(),
        tl.as<uint32_t>(), flags.as<unsigned long long>(), goff[cur]->as<uint32_t>(),
        P.as<unsigned long long>(), g1.as<double>(), g2.as<double>(), eq[nxt]->as<uint32_t>(),
        et[nxt]->as<uint32_t>(), eg[nxt]->as<uint32_t>(), elm[nxt]->as<float>(),
        eprow[cur]->as<uint32_t>(), eprow[nxt]->as<uint32_t>(), self_rows ? 1 : 0, level,
        wk ? wq.as<uint32_t>() : nullptr, wh.as<uint32_t>(), welm.as<float>(),
        wcount.as<uint32_t>(), wrow.as<uint32_t>(), wrm.as<float>(),
        level == 0 ? nullptr : elm[cur]->as<float>(),
        self_rows && row_depth == 2 ? 1 : 0, dEp);
    FSGG_LAUNCH_CHECK();
    if (level < t.depth) {
      goff_kernel<<<ceil_div_u32(uint64_t(G) + 1, 256), 256, 0, s>>>(
          G, goff[cur]->as<uint32_t>(), P.as<unsigned long long>(),
          goff[nxt]->as<uint32_t>());
      FSGG_LAUNCH_CHECK();
      ds.launches++;
    }
    ds.launches += 3;
    cur = nxt;
    if (lite) {  // next level: count on the device, bounded by 2 E and the tickets
      E_known = false;
      E_hi = std::min<uint64_t>(2 * E_hi, cap);
      continue;
    }

    if (trace) FSGG_CUDA(cudaEventRecord(tev[3], s));
    unsigned long long* host = ds.host_words();
    FSGG_CUDA(cudaMemcpyAsync(host, counters, 24, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(host + 3), dE + 1, 4,
                              cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    out.tickets_per_level.push_back(host[0]);
    out.degenerate_draws += host[1];
    out.tie_verified += host[2] & 0xffffffffull;
    const uint64_t next = *reinterpret_cast<const uint32_t*>(host + 3);
    if (next > cap) throw NumericError("entry list overflow");
    if (next > 0 && level >= t.depth)
      throw NumericError("tickets remain below the deepest level");
    if (trace) {
      float ms[3];
      for (int k = 0; k < 3; ++k) FSGG_CUDA(cudaEventElapsedTime(&ms[k], tev[k], tev[k + 1]));
      const double wall = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - wall0).count();
      const uint32_t smax = uint32_t((uint64_t(ds.n) + (1ull << level) - 1) >> level);
      std::fprintf(stderr,
                   "fsgg level %2u: entries=%10u node<=%8u evals=%.3e performed=%.3e "
                   "kde=%8.3fms route=%7.3fms scan+scatter=%7.3fms wall=%8.3fms ties=%llu\n",
                   level, E, smax, double(out.kde.evals - kde0.evals),
                   double(out.kde.performed - kde0.performed), ms[0], ms[1], ms[2], wall,
                   (unsigned long long)(host[2] & 0xffffffffull));
    }
    E = static_cast<uint32_t>(next);
    E_hi = E;
  }
  if (lite) {
    // per-level statistics of the sync-free descent (one read)
    std::vector<uint32_t> hE(kMaxLevelsLog + 2);
    std::vector<unsigned long long> hc(size_t(kMaxLevelsLog) * 4);
    FSGG_CUDA(cudaMemcpyAsync(hE.data(), elog.as<void>(), hE.size() * 4, cudaMemcpyDeviceToHost,
                              s));
    FSGG_CUDA(cudaMemcpyAsync(hc.data(), lvc.as<void>(), hc.size() * 8, cudaMemcpyDeviceToHost,
                              s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    for (uint32_t l = 0; l < levels_run; ++l) {
      if (hE[l] == 0) break;
      if (hE[l] > cap) throw NumericError("entry list overflow");
      out.entries_per_level.push_back(hE[l]);
      out.peak_entries = std::max<uint64_t>(out.peak_entries, hE[l]);
      out.tickets_per_level.push_back(hc[4 * l]);
      out.degenerate_draws += hc[4 * l + 1];
      out.tie_verified += hc[4 * l + 2] & 0xffffffffull;
    }
    if (hE[levels_run] > 0) throw NumericError("tickets remain below the deepest level");
  }
  {
    // reference-equivalent work served by lookups; direct-level evaluations
    unsigned long long* ev = ds.host_words();
    FSGG_CUDA(cudaMemcpyAsync(&ev[0], lookup_evals.as<void>(), 8, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaMemcpyAsync(&ev[1], ds.kde_ws->direct_evals.as<void>(), 8,
                              cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    out.kde.evals += ev[0] + ev[1];
    out.kde.performed += ev[1];
  }
  if (walk_on) {
    uint32_t* hw = reinterpret_cast<uint32_t*>(ds.host_words());
    FSGG_CUDA(cudaMemcpyAsync(hw, wcount.as<void>(), 4, cudaMemcpyDeviceToHost, s));
    FSGG_CUDA(cudaStreamSynchronize(s));
    const uint32_t W = *hw;
    if (W > 0) {
      const auto w0 = std::chrono::steady_clock::now();
      DevBuf& st = ds.buf("s.walk_stats", 5 * 64 * 8);
      FSGG_CUDA(cudaMemsetAsync(st.as<void>(), 0, 5 * 64 * 8, s));
      WalkArgs a;
      a.W = W;
      a.wq = wq.as<uint32_t>();
      a.wh = wh.as<uint32_t>();
      a.welm = welm.as<float>();
      a.wrow = wrow.as<uint32_t>();
      a.wrm = wrm.as<float>();
      // the last compute level's two-deep rows, if no later level reused them
      a.rows = part_depth == 2 ? ws.partials.as<double>() : nullptr;
      a.rows_level = part_level;
      a.key_prefix = prefix;
      a.seed = req.seed;
      a.rng_mode = req.rng_mode;
      a.verify = verify ? 1 : 0;
      a.qrow = qrow.as<uint32_t>();
      a.row_off = out.row_off.as<uint64_t>();
      a.row_cnt = out.row_cnt.as<uint32_t>();
      a.leaf_src = out.leaf_src.as<uint32_t>();
      a.leaf_cnt = out.leaf_cnt.as<uint32_t>();
      a.stats = st.as<unsigned long long>();
      a.nlink = nlink_p;
      walk_finish(ds, ks, a);
      std::vector<unsigned long long> h(5 * 64);
      FSGG_CUDA(cudaMemcpyAsync(h.data(), st.as<void>(), h.size() * 8, cudaMemcpyDeviceToHost, s));
      FSGG_CUDA(cudaStreamSynchronize(s));
      // merge the walks' per-level tallies into the level diagnostics
      for (uint32_t lv2 = 0; lv2 < 64; ++lv2) {
        if (!h[lv2]) continue;
        if (out.entries_per_level.size() <= lv2) {
          out.entries_per_level.resize(lv2 + 1, 0);
          out.tickets_per_level.resize(lv2 + 1, 0);
        }
        out.entries_per_level[lv2] += h[lv2];
        out.tickets_per_level[lv2] += h[lv2];  // one ticket each
        out.kde.evals += h[64 + lv2];
        out.kde.performed += h[64 + lv2] - h[256 + lv2];  // minus steps read from rows
        out.degenerate_draws += h[128 + lv2];
        out.tie_verified += h[192 + lv2];
      }
      for (uint64_t e : out.entries_per_level) out.peak_entries = std::max(out.peak_entries, e);
      if (trace)
        std::fprintf(stderr, "fsgg walks: %u single-ticket walks %.3fms\n", W,
                     std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now() - w0).count());
    }
  }
  if (trace)
    for (auto& e : tev) cudaEventDestroy(e);
}

void sampled_triples_to_host(Dataset& ds, SampleResult& res,
                             std::vector<uint32_t>& triples) {
  cudaStream_t s = ds.stream;
  const uint32_t nq = res.nq;
  const uint64_t total = res.total_tickets;
  triples.clear();
  if (nq == 0 || total == 0) return;
  if (total > 0x7fffffffull) throw ConfigError("too many tickets for host output");
  DevBuf& ends = ds.buf("t.ends", size_t(nq) * 8);
  DevBuf& src_out = ds.buf("t.src", total * 4);
  DevBuf& cnt_out = ds.buf("t.cnt", total * 4);
  DevBuf& tmp = ds.buf("t.tmp", 8);
  row_ends_kernel<<<ceil_div_u32(nq, 256), 256, 0, s>>>(
      res.row_off.as<uint64_t>(), res.row_cnt.as<uint32_t>(), nq, ends.as<uint64_t>());
  FSGG_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  FSGG_CUDA(cub::DeviceSegmentedSort::SortPairs(
      nullptr, tmp_bytes, res.leaf_src.as<uint32_t>(), src_out.as<uint32_t>(),
      res.leaf_cnt.as<uint32_t>(), cnt_out.as<uint32_t>(), int(total), int(nq),
      res.row_off.as<uint64_t>(), ends.as<uint64_t>(), s));
  tmp.ensure(tmp_bytes, s);
  FSGG_CUDA(cub::DeviceSegmentedSort::SortPairs(
      tmp.as<void>(), tmp_bytes, res.leaf_src.as<uint32_t>(), src_out.as<uint32_t>(),
      res.leaf_cnt.as<uint32_t>(), cnt_out.as<uint32_t>(), int(total), int(nq),
      res.row_off.as<uint64_t>(), ends.as<uint64_t>(), s));
  ds.launches += 2;
  std::vector<uint32_t> uq(nq), cnt(nq), src(total), c(total);
  std::vector<uint64_t> off(nq + 1);
  FSGG_CUDA(cudaMemcpyAsync(uq.data(), res.uq.as<void>(), size_t(nq) * 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(cnt.data(), res.row_cnt.as<void>(), size_t(nq) * 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(off.data(), res.row_off.as<void>(), size_t(nq + 1) * 8, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(src.data(), src_out.as<void>(), total * 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(c.data(), cnt_out.as<void>(), total * 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  uint64_t m = 0;
  for (uint32_t i = 0; i < nq; ++i) m += cnt[i];
  triples.resize(m * 3);
  uint64_t at = 0;
  for (uint32_t i = 0; i < nq; ++i)
    for (uint32_t k = 0; k < cnt[i]; ++k, ++at) {
      triples[3 * at] = uq[i];
      triples[3 * at + 1] = src[off[i] + k];
      triples[3 * at + 2] = c[off[i] + k];
    }
}

}  // namespace fsgg
