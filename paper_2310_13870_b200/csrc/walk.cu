// Single-ticket walks: the tail of fsg::sample_neighbors_counted
// (proj/src/sampler.cpp:117-239) for entries that hold one ticket.
//
// Below nodes of kWalkMaxNode points almost every entry carries a single
// ticket (C3: 60M entries for 64M tickets at level 14), and an entry with one
// ticket never splits: it follows one root-to-leaf path. Keeping those
// entries in the level-synchronous lists costs a route, a scan and a scatter
// pass over ~60M entries per level for a handful of arithmetic each; here
// every such entry instead becomes one thread that walks its path to the
// leaf: child sums of the current node (the same direct_child_sums as the
// level-synchronous direct kernel, so the same bits), p, the reference's
// keyed draw for counter 0, the tie guard (fp64 re-decision of draws within
// the fp32 error of p), then the chosen child. Entries with more tickets stay
// in the lists; scatter_kernel routes children with exactly one ticket here.
// Per-level counters (entries, tickets, evaluations, degenerate draws) are
// aggregated per warp by level, so the reference's diagnostics are intact.
#include "engine.cuh"
#include "kde_math.cuh"

namespace fsgg {
namespace {

constexpr int kWalkThreads = 128;
#ifndef FSGG_WALK_CTAS
#define FSGG_WALK_CTAS 16
#endif
constexpr int kMaxLevels = 64;
constexpr double kTieMargin = 1e-4;  // as route_kernel (sampler.cu)

// p = a / (a + b) with the reference's degenerate rule (sampler.cpp:205-211)
// and the draw u_0 < p on the keyed stream (rng.hpp:34-36, 66-70).
struct Decision {
  bool left, near, degenerate;
};

__device__ __forceinline__ Decision decide(double a, double b, float em, uint32_t f,
                                           uint32_t l, uint32_t q, uint64_t qlink,
                                           uint64_t key_prefix, int rng_mode, uint64_t seed,
                                           bool want_near, const uint64_t* nlink, uint64_t h,
                                           double pruned) {
  Decision d{false, false, false};
  double p;
  if (a <= kSumFloor && b <= kSumFloor) {
    p = 0.5;
    d.degenerate = true;
    d.near = want_near;  // degenerate by fp32 sums: decided on exact sums
  } else {
    p = a / (a + b);
  }
  if (p >= 1.0) {
    d.left = true;
  } else if (p > 0.0) {
    const double P = p * 9007199254740992.0;
    const uint64_t thr = static_cast<uint64_t>(ceil(P));
    uint64_t m;
    if (rng_mode == 0) {
      const uint64_t key = nlink ? splitmix64(__ldg(nlink + h) ^ qlink)
                                 : route_key_q(key_prefix, (uint64_t(f) << 32) | l, qlink);
      m = splitmix64(key) >> 11;
      if (want_near) {
        const double rel = kTieMargin * (1.0 + fmaxf(0.f, -em) / 32.0);
        const double M = (rel * fmin(p, 1.0 - p) + pruned) * 9007199254740992.0 + 1.0;
        const uint64_t lo = P > M ? static_cast<uint64_t>(P - M) : 0ull;
        const uint64_t hi = static_cast<uint64_t>(P + M);
        d.near |= (m >= lo) & (m <= hi);
      }
    } else {
      const uint4 r = philox4x32(make_uint4(0u, q, f, l),
                                 make_uint2(uint32_t(seed), uint32_t(seed >> 32)));
      m = ((uint64_t(r.x) << 32) | r.y) >> 11;
    }
    d.left = m < thr;
  }
  return d;
}

// d <= 2: capped at 32 registers (16 CTAs per SM; some spills) — the
// kernel is latency-bound on its loads (ncu: long-scoreboard stalls lead),
// and the extra warps measured faster than fewer spills (12 CTAs: 9.10 ms,
// 14-16: 8.90)
template <int D, int FAM>
__global__ void __launch_bounds__(kWalkThreads, D <= 2 ? FSGG_WALK_CTAS : 0)
    walk_kernel(const float* __restrict__ pts, uint32_t W, const uint32_t* __restrict__ wq,
                const uint32_t* __restrict__ wh, const float* __restrict__ welm,
                const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ tlast,
                const float* __restrict__ tlo, const float* __restrict__ thi, int has_boxes,
                float scale, int family, double sigma, uint64_t key_prefix, int rng_mode,
                uint64_t seed, int verify, const uint32_t* __restrict__ qrow,
                const uint64_t* __restrict__ row_off, uint32_t* __restrict__ row_cnt,
                uint32_t* __restrict__ leaf_src, uint32_t* __restrict__ leaf_cnt,
                unsigned long long* __restrict__ stats, const uint64_t* __restrict__ nlink,
                const uint32_t* __restrict__ wrow, const float* __restrict__ wrm,
                const double* __restrict__ rows, uint32_t rows_level) {
  // entries, evals, degen, ties, evals read from rows
  // 32-bit per-CTA tallies (native shared-memory atomics; 64-bit ones are
  // CAS loops): a CTA's counts per level stay far below 2^32 (at most 128
  // walks x their node sizes), widened when flushed to the global counters
  __shared__ unsigned int s_stats[5][kMaxLevels];
  for (int k = threadIdx.x; k < 5 * kMaxLevels; k += blockDim.x) (&s_stats[0][0])[k] = 0;
  __syncthreads();

  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  bool live = i < W;
  uint32_t q = 0, lev = 0;
  uint64_t h = 0;
  float em = 0.f;
  float qc[D];
  uint64_t qlink = 0;
  uint32_t row = 0xffffffffu;  // first step read from the row (see WalkArgs)
  float rmass = 0.f;
  // the node's point range: loaded once, then carried — a child is
  // [f, mid) or [mid, l) with mid = f + (l - f) / 2 (the tree's split), so
  // no step waits on a dependent load of the next node's range
  uint32_t nf = 0, nl = 0;
  if (live) {
    q = wq[i];
    qlink = query_link(q);
    h = wh[i];
    nf = tfirst[h];
    nl = tlast[h];
    em = welm[i];
    lev = 31 - __clz(uint32_t(h) + 1);
    if (rows && lev == rows_level + 1) {
      row = wrow[i];
      rmass = wrm[i];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) qc[k] = __ldg(pts + size_t(q) * D + k);
  }
  const bool check = verify && rng_mode == 0;
  while (__any_sync(0xffffffffu, live)) {
    const unsigned live_mask = __ballot_sync(0xffffffffu, live);
    if (live) {
      const uint32_t f = nf, l = nl;
      uint32_t ev = 0, dg = 0, tie = 0, sv = 0;
      const uint32_t at = lev;
      if (l - f == 1) {  // sampler.cpp:196-198: leaf (query, source, 1)
        const uint32_t row = qrow[q];
        const uint32_t slot = atomicAdd(row_cnt + row, 1u);
        const uint64_t o = row_off[row] + slot;
        leaf_src[o] = f;
        leaf_cnt[o] = 1u;
        live = false;
      } else {
        double s[2];
        double pruned = 0.0;
        ev = l - f;
        if (row != 0xffffffffu) {
          // the node's children are buckets 2 side, 2 side + 1 of the row
          // (h odd: left child of its parent); the partials skipped
          // sub-chunks below 2^-48 of half the row's node mass: the tie
          // margin takes that bound (as route_kernel's row_mass term)
          const double* r = rows + (size_t(row) << 2) + ((h & 1u) ? 0u : 2u);
          s[0] = r[0];
          s[1] = r[1];
          pruned = check ? double(exp2f(rmass - (kPruneBits - 24.f) - em)) : 0.0;
          sv = ev;
          row = 0xffffffffu;  // later steps evaluate
        } else {
          direct_child_sums<D, FAM>(pts, qc, h, f, l, tlo, thi, has_boxes, scale, s);
        }
        double a = fmax(s[0], kSumFloor), b = fmax(s[1], kSumFloor);
        Decision dc =
            decide(a, b, em, f, l, q, qlink, key_prefix, rng_mode, seed, check, nlink, h, pruned);
        if (check && dc.near) {
          // tie guard: re-decide on fp64 sums (kernel_f64, index order)
          const uint32_t mid = f + (l - f) / 2;
          const float* xq = pts + size_t(q) * D;
          double e0 = 0.0, e1 = 0.0;
          for (uint32_t j = f; j < mid; ++j) e0 += kernel_f64(family, sigma, xq, pts + size_t(j) * D, D);
          for (uint32_t j = mid; j < l; ++j) e1 += kernel_f64(family, sigma, xq, pts + size_t(j) * D, D);
          a = fmax(e0, kSumFloor);
          b = fmax(e1, kSumFloor);
          dc = decide(a, b, em, f, l, q, qlink, key_prefix, rng_mode, seed, false, nlink, h, 0.0);
          tie = 1;
        }
        dg = dc.degenerate ? 1u : 0u;
        // log2 of the chosen child's sum, to integer precision (only the tie
        // margin's far-node widening reads it)
        em = float(int((__double_as_longlong(dc.left ? a : b) >> 52) & 0x7ff) - 1023);
        h = dc.left ? 2 * h + 1 : 2 * h + 2;
        const uint32_t mid = f + (l - f) / 2;
        nf = dc.left ? f : mid;
        nl = dc.left ? mid : l;
        ++lev;
      }
      // per-level tallies, one shared-memory update per level group of the
      // warp; lanes of a warp almost always share the level (fast path)
      const uint32_t lead_at = __shfl_sync(live_mask, at, __ffs(live_mask) - 1);
      const unsigned grp = __all_sync(live_mask, at == lead_at) ? live_mask
                                                                : __match_any_sync(live_mask, at);
      const uint32_t n_ent = __popc(grp);
      const uint32_t n_ev = __reduce_add_sync(grp, ev);
      const uint32_t n_sv = __reduce_add_sync(grp, sv);
      const bool rare = __any_sync(grp, dg | tie);
      const uint32_t n_dg = rare ? __reduce_add_sync(grp, dg) : 0u;
      const uint32_t n_tie = rare ? __reduce_add_sync(grp, tie) : 0u;
      if ((threadIdx.x & 31) == uint32_t(__ffs(grp) - 1) && at < kMaxLevels) {
        atomicAdd(&s_stats[0][at], n_ent);
        if (n_ev) atomicAdd(&s_stats[1][at], n_ev);
        if (n_dg) atomicAdd(&s_stats[2][at], n_dg);
        if (n_tie) atomicAdd(&s_stats[3][at], n_tie);
        if (n_sv) atomicAdd(&s_stats[4][at], n_sv);
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 5 * kMaxLevels; k += blockDim.x) {
    const unsigned long long v = (&s_stats[0][0])[k];  // widened
    if (v) atomicAdd(stats + k, v);
  }
}

template <class F>
void walk_by_dim(uint32_t d, F&& f) {
  switch (d) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    default: throw ConfigError("walk supports d <= 8");
  }
}

}  // namespace

bool walk_supported(uint32_t d) { return d >= 1 && d <= 8; }

void walk_finish(Dataset& ds, const KernelSpec& ks, const WalkArgs& a) {
  if (a.W == 0) return;
  const TreeTable& t = ds.tree;
  cudaStream_t s = ds.stream;
  auto launch = [&](auto dim, auto fam) {
    constexpr int D = decltype(dim)::value;
    constexpr int FAM = decltype(fam)::value;
    walk_kernel<D, FAM><<<ceil_div_u32(a.W, kWalkThreads), kWalkThreads, 0, s>>>(
        ds.pts.as<float>(), a.W, a.wq, a.wh, a.welm, t.first.as<uint32_t>(),
        t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(), t.has_boxes, ks.scale,
        ks.family, ks.sigma, a.key_prefix, a.rng_mode, a.seed, a.verify, a.qrow, a.row_off,
        a.row_cnt, a.leaf_src, a.leaf_cnt, a.stats, a.nlink, a.wrow, a.wrm, a.rows,
        a.rows_level);
  };
  switch (ks.family) {
    case 0: walk_by_dim(ds.d, [&](auto dim) { launch(dim, std::integral_constant<int, 0>{}); }); break;
    case 1: walk_by_dim(ds.d, [&](auto dim) { launch(dim, std::integral_constant<int, 1>{}); }); break;
    case 2: walk_by_dim(ds.d, [&](auto dim) { launch(dim, std::integral_constant<int, 2>{}); }); break;
    default: throw ConfigError("unknown kernel family");
  }
  FSGG_LAUNCH_CHECK();
  ds.launches++;
}

}  // namespace fsgg
