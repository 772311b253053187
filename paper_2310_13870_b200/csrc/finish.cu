// Depth-first finish of the descent for small nodes.
//
// Once every node of a level holds at most kDfsMaxNode points, the
// remaining levels of proj/src/sampler.cpp:117-239 are cheaper to run per
// entry than level-synchronously: one thread takes an entry (node, query,
// tickets) and walks its subtree depth-first — child sums over the node's
// points (fp32 terms with bounding-box exponent offsets, fp64 totals), p, the
// reference's keyed Binomial(t, p), then the children with tickets — emitting
// (query, source, count) at size-1 nodes. This removes ~7 levels of
// entry-list materialisation (route, scan, scatter: ~60M entries each at
// n = 1M) while producing exactly the same samples: every routing decision
// uses the same sums/stream as the level-synchronous path, near-ties are
// re-decided on fp64 sums, and (node, query) pairs stay unique, so the
// reference's per-level diagnostics are rebuilt from per-block histograms.
#include "engine.cuh"
#include "kde_math.cuh"

namespace fsgg {
namespace {

constexpr int kDfsThreads = 128;
constexpr int kMaxLevels = 64;
constexpr int kMaxDepth = 10;  // levels below the start level (nodes <= 512)
constexpr double kTieMargin = 1e-4;  // as route_kernel (sampler.cu)

__device__ __forceinline__ uint4 philox4x32_f(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

template <int D, int FAM>
__device__ __forceinline__ double range_sum_f32(const float* __restrict__ pts,
                                                const float (&q)[D], uint32_t a,
                                                uint32_t b, float scale, float off) {
  float acc = 0.f;
  for (uint32_t j = a; j < b; ++j) {
    const float* x = pts + size_t(j) * D;
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) t = fam_acc1<FAM>(q[k] - __ldg(x + k), t);
    acc += ex2_approx(fmaf(fam_finish1<FAM>(t), -scale, off));
  }
  return off > 0.f ? double(acc) * exp2(-double(off)) : double(acc);
}

__device__ __forceinline__ double range_sum_f64(const float* __restrict__ pts, uint32_t d,
                                                int family, double sigma, const float* q,
                                                uint32_t a, uint32_t b) {
  double s = 0.0;
  for (uint32_t j = a; j < b; ++j) s += kernel_f64(family, sigma, q, pts + size_t(j) * d, d);
  return s;
}

template <int D, int FAM>
__global__ void __launch_bounds__(kDfsThreads)
    dfs_finish_kernel(const float* __restrict__ pts, uint32_t E, uint32_t level0,
                      const uint32_t* __restrict__ eq, const uint32_t* __restrict__ et,
                      const uint32_t* __restrict__ eg, const uint32_t* __restrict__ tfirst,
                      const uint32_t* __restrict__ tlast, const float* __restrict__ tlo,
                      const float* __restrict__ thi, int has_boxes, float scale, int family,
                      double sigma, uint64_t key_prefix, int rng_mode, uint64_t seed,
                      int verify, const uint32_t* __restrict__ qrow,
                      const uint64_t* __restrict__ row_off, uint32_t* __restrict__ row_cnt,
                      uint32_t* __restrict__ leaf_src, uint32_t* __restrict__ leaf_cnt,
                      unsigned long long* __restrict__ stats /* [4][kMaxLevels] */) {
  __shared__ unsigned long long s_stats[4][kMaxLevels];  // entries, tickets, evals, degen
  __shared__ unsigned long long s_ties;
  for (int k = threadIdx.x; k < 4 * kMaxLevels; k += blockDim.x) (&s_stats[0][0])[k] = 0;
  if (threadIdx.x == 0) s_ties = 0;
  __syncthreads();

  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < E) {
    const uint32_t query = eq[i];
    float qc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) qc[k] = __ldg(pts + size_t(query) * D + k);
    const uint32_t row = qrow[query];
    // explicit stack of (heap slot, tickets); depth <= log2(kDfsMaxNode) + 1
    uint32_t sh[16], st[16];
    int sp = 0;
    sh[sp] = ((1u << level0) - 1) + eg[i];
    st[sp++] = et[i];
    unsigned long long ties = 0;
    // per-thread per-level tallies (flushed once: shared-memory atomics per
    // visited node would serialise the block on a handful of addresses)
    uint32_t c_ent[kMaxDepth] = {}, c_tik[kMaxDepth] = {}, c_ev[kMaxDepth] = {},
             c_deg[kMaxDepth] = {};
    while (sp > 0) {
      --sp;
      const uint32_t h = sh[sp], t = st[sp];
      const uint32_t lev = 31 - __clz(h + 1);
      const uint32_t rl = min(lev - level0, uint32_t(kMaxDepth - 1));
      const uint32_t f = tfirst[h], l = tlast[h];
      c_ent[rl] += 1;
      c_tik[rl] += t;
      if (l - f == 1) {  // proj/src/sampler.cpp:196-198
        const uint32_t slot = atomicAdd(row_cnt + row, 1u);
        const uint64_t at = row_off[row] + slot;
        leaf_src[at] = f;
        leaf_cnt[at] = t;
        continue;
      }
      const uint32_t mid = f + (l - f) / 2;
      const uint32_t hl = 2 * h + 1, hr = 2 * h + 2;
      const float offl = has_boxes ? scale * box_dist<FAM>(qc, tlo + size_t(hl) * D,
                                                            thi + size_t(hl) * D, D)
                                   : 0.f;
      const float offr = has_boxes ? scale * box_dist<FAM>(qc, tlo + size_t(hr) * D,
                                                            thi + size_t(hr) * D, D)
                                   : 0.f;
      double a = fmax(range_sum_f32<D, FAM>(pts, qc, f, mid, scale, offl), kSumFloor);
      double b = fmax(range_sum_f32<D, FAM>(pts, qc, mid, l, scale, offr), kSumFloor);
      c_ev[rl] += l - f;
      bool exact = false;
      uint32_t left = 0;
      for (int pass = 0; pass < 2; ++pass) {
        double p;
        bool degenerate = false;
        if (a <= kSumFloor && b <= kSumFloor) {
          p = 0.5;
          degenerate = true;
        } else {
          p = a / (a + b);
        }
        bool near = degenerate && verify && !exact;
        left = 0;
        if (p >= 1.0) {
          left = t;
        } else if (p > 0.0) {
          const double P = p * 9007199254740992.0;
          const uint64_t thr = static_cast<uint64_t>(ceil(P));
          if (rng_mode == 0) {
            const uint64_t key = route_key(key_prefix, (uint64_t(f) << 32) | l, uint64_t(query));
            const double M = kTieMargin * fmin(p, 1.0 - p) * 9007199254740992.0 + 1.0;
            const uint64_t lo = P > M ? static_cast<uint64_t>(P - M) : 0ull;
            const uint64_t hi = static_cast<uint64_t>(P + M);
            for (uint32_t c = 0; c < t; ++c) {
              const uint64_t m = splitmix64(key + c) >> 11;
              left += m < thr ? 1u : 0u;
              near |= (m >= lo) & (m <= hi);
            }
          } else {
            const uint2 k = make_uint2(uint32_t(seed), uint32_t(seed >> 32));
            for (uint32_t c = 0; c < t; c += 2) {
              const uint4 r = philox4x32_f(make_uint4(c >> 1, query, f, l), k);
              left += ((uint64_t(r.x) << 32 | r.y) >> 11) < thr ? 1u : 0u;
              if (c + 1 < t) left += ((uint64_t(r.z) << 32 | r.w) >> 11) < thr ? 1u : 0u;
            }
            near = false;
          }
        }
        if (near && verify && !exact && rng_mode == 0) {
          // re-decide on fp64 sums (see route_kernel's tie guard)
          a = fmax(range_sum_f64(pts, D, family, sigma, qc, f, mid), kSumFloor);
          b = fmax(range_sum_f64(pts, D, family, sigma, qc, mid, l), kSumFloor);
          exact = true;
          ++ties;
          continue;
        }
        if (degenerate) c_deg[rl] += t;
        break;
      }
      // right pushed first so the left subtree is walked first
      if (left < t) {
        sh[sp] = hr;
        st[sp++] = t - left;
      }
      if (left > 0) {
        sh[sp] = hl;
        st[sp++] = left;
      }
    }
    if (ties) atomicAdd(&s_ties, ties);
    for (uint32_t r = 0; r < kMaxDepth && level0 + r < kMaxLevels; ++r) {
      if (!c_ent[r]) break;
      atomicAdd(&s_stats[0][level0 + r], static_cast<unsigned long long>(c_ent[r]));
      atomicAdd(&s_stats[1][level0 + r], static_cast<unsigned long long>(c_tik[r]));
      atomicAdd(&s_stats[2][level0 + r], static_cast<unsigned long long>(c_ev[r]));
      if (c_deg[r]) atomicAdd(&s_stats[3][level0 + r], static_cast<unsigned long long>(c_deg[r]));
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 4 * kMaxLevels; k += blockDim.x) {
    const unsigned long long v = (&s_stats[0][0])[k];
    if (v) atomicAdd(stats + k, v);
  }
  if (threadIdx.x == 0 && s_ties) atomicAdd(stats + 4 * kMaxLevels, s_ties);
}

template <int FAM, class F>
void by_dim(uint32_t d, F&& f) {
  switch (d) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    default: throw ConfigError("dfs finish supports d <= 8");
  }
}

}  // namespace

bool dfs_finish_supported(uint32_t d) { return d >= 1 && d <= 8; }

void dfs_finish(Dataset& ds, const KernelSpec& ks, const DfsArgs& a) {
  const TreeTable& t = ds.tree;
  cudaStream_t s = ds.stream;
  auto launch = [&](auto dim, auto fam) {
    constexpr int D = decltype(dim)::value;
    constexpr int FAM = decltype(fam)::value;
    dfs_finish_kernel<D, FAM><<<ceil_div_u32(a.E, kDfsThreads), kDfsThreads, 0, s>>>(
        ds.pts.as<float>(), a.E, a.level, a.eq, a.et, a.eg, t.first.as<uint32_t>(),
        t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(), t.has_boxes, ks.scale,
        ks.family, ks.sigma, a.key_prefix, a.rng_mode, a.seed, a.verify, a.qrow, a.row_off,
        a.row_cnt, a.leaf_src, a.leaf_cnt, a.stats);
  };
  switch (ks.family) {
    case 0: by_dim<0>(ds.d, [&](auto dim) { launch(dim, std::integral_constant<int, 0>{}); }); break;
    case 1: by_dim<1>(ds.d, [&](auto dim) { launch(dim, std::integral_constant<int, 1>{}); }); break;
    case 2: by_dim<2>(ds.d, [&](auto dim) { launch(dim, std::integral_constant<int, 2>{}); }); break;
    default: throw ConfigError("unknown kernel family");
  }
  FSGG_LAUNCH_CHECK();
  ds.launches++;
}

}  // namespace fsgg
