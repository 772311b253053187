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
#include <algorithm>
#include <cstdlib>

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
                const double* __restrict__ rows, uint32_t rows_level,
                const uint32_t* __restrict__ widx, const uint32_t* __restrict__ wcount) {
  // entries, evals, degen, ties, evals read from rows
  // 32-bit per-CTA tallies (native shared-memory atomics; 64-bit ones are
  // CAS loops): a CTA's counts per level stay far below 2^32 (at most 128
  // walks x their node sizes), widened when flushed to the global counters
  __shared__ unsigned int s_stats[5][kMaxLevels];
  for (int k = threadIdx.x; k < 5 * kMaxLevels; k += blockDim.x) (&s_stats[0][0])[k] = 0;
  __syncthreads();

  // widx/wcount: the walks the fast kernel deferred (indices into the walk
  // list, count on the device); otherwise all W walks, one per thread
  const uint32_t count = wcount ? *wcount : W;
  for (uint32_t base = blockIdx.x * blockDim.x; base < count; base += gridDim.x * blockDim.x) {
  const uint32_t slot_t = base + threadIdx.x;
  bool live = slot_t < count;
  const uint32_t i = live ? (widx ? widx[slot_t] : slot_t) : 0u;
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
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 5 * kMaxLevels; k += blockDim.x) {
    const unsigned long long v = (&s_stats[0][0])[k];  // widened
    if (v) atomicAdd(stats + k, v);
  }
}

// ---- fast walk (reference RNG with the tie guard on) ------------------------
// With the tie guard every fp32-based decision whose draw lies within the
// sums' error of p is re-decided on exact fp64 sums, so the fast path only
// has to be (a) within the guard's margin of the exact p and (b) cheap:
//   * one exponent offset per node (its own box) instead of one per child, so
//     the two children's fp32 sums share a scale and p needs no rescaling;
//     the children are summed in one loop (two independent accumulators);
//   * no division and no float-to-integer conversions: with u = m 2^-53 the
//     draw u < a / (a + b) is u (a + b) - a < 0, and "near" is
//     |u (a + b) - a| <= rel min(a, b) + (pruned + 2^-51)(a + b) — the same
//     test as decide()'s, multiplied through by a + b;
//   * per-level tallies once per walk: a thread keeps its start level, start
//     size and the left/right bits of its path; node sizes along the path
//     follow from those, and the warp adds them up per level after the loop
//     (the per-step version spent 15% of the kernel's instructions on it).
// A walk whose step the fast path cannot take — a draw inside the margin,
// both fp32 sums zero, or an offset so large that the 1e-300 floor could
// matter — stops there: its node and mass go back into its walk-list slot and
// its index onto a deferred list, and walk_kernel (per-child offsets,
// decide(), fp64 re-decision) finishes the deferred walks afterwards (~1 in
// 10^3 at C3). The fast kernel then holds no fp64 sums and no calls.
#ifndef FSGG_WALKF_CTAS
#define FSGG_WALKF_CTAS 12
#endif
template <int D, int FAM>
__global__ void __launch_bounds__(kWalkThreads, D <= 2 ? FSGG_WALKF_CTAS : 0)
    walk_fast_kernel(const float* __restrict__ pts, uint32_t W, const uint32_t* __restrict__ wq,
                     uint32_t* __restrict__ wh, float* __restrict__ welm,
                     uint32_t* __restrict__ widx, uint32_t* __restrict__ wcount,
                     const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ tlast,
                     const float* __restrict__ tlo, const float* __restrict__ thi,
                     int has_boxes, float scale, uint64_t key_prefix,
                     const uint32_t* __restrict__ qrow,
                     const uint64_t* __restrict__ row_off, uint32_t* __restrict__ row_cnt,
                     uint32_t* __restrict__ leaf_src, uint32_t* __restrict__ leaf_cnt,
                     unsigned long long* __restrict__ stats,
                     const uint64_t* __restrict__ nlink, const uint32_t* __restrict__ wrow,
                     const float* __restrict__ wrm, const double* __restrict__ rows,
                     uint32_t rows_level) {
  __shared__ unsigned int s_stats[5][kMaxLevels];
  for (int k = threadIdx.x; k < 5 * kMaxLevels; k += blockDim.x) (&s_stats[0][0])[k] = 0;
  __syncthreads();

  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool mine = i < W;
  uint32_t q = 0, lev0 = 0xffffffffu, n0 = 0, path = 0, steps = 0, sv0 = 0;
  bool deferred = false;
  if (mine) {
    q = wq[i];
    // opaque: under the register cap the compiler otherwise recomputes the
    // query's splitmix64 at every step instead of keeping two registers
    uint64_t qlink = query_link(q);
    asm volatile("" : "+l"(qlink));
    uint64_t h = wh[i];
    uint32_t nf = tfirst[h], nl = tlast[h];
    float em = welm[i];
    lev0 = 31 - __clz(uint32_t(h) + 1);
    n0 = nl - nf;
    uint32_t row = 0xffffffffu;
    float rmass = 0.f;
    if (rows && lev0 == rows_level + 1) {
      row = wrow[i];
      rmass = wrm[i];
    }
    float qc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) qc[k] = __ldg(pts + size_t(q) * D + k);
    while (nl - nf > 1) {
      const uint32_t f = nf, l = nl, mid = f + (l - f) / 2;
      double a, b, pruned = 0.0;
      float offn = 0.f;
      bool fast;
      const bool rowstep = row != 0xffffffffu;
      if (rowstep) {
        // the node's children are buckets 2 side, 2 side + 1 of the row (see
        // walk_kernel); absolute fp64 sums
        const double* r = rows + (size_t(row) << 2) + ((h & 1u) ? 0u : 2u);
        a = fmax(r[0], kSumFloor);
        b = fmax(r[1], kSumFloor);
        pruned = double(exp2f(rmass - (kPruneBits - 24.f) - em));
        sv0 = l - f;
        row = 0xffffffffu;
        fast = a > kSumFloor || b > kSumFloor;
      } else {
        offn = has_boxes ? scale * box_dist_d<D, FAM>(qc, tlo + h * D, thi + h * D) : 0.f;
        float a0 = 0.f, a1 = 0.f;
        const uint32_t nleft = mid - f;  // the right child has nleft or nleft + 1 points
        for (uint32_t j = 0; j < nleft; ++j) {
          float t0 = 0.f, t1 = 0.f;
          if constexpr (D == 2) {
            const float2 x0 = __ldg(reinterpret_cast<const float2*>(pts) + f + j);
            const float2 x1 = __ldg(reinterpret_cast<const float2*>(pts) + mid + j);
            t0 = fam_acc1<FAM>(qc[0] - x0.x, t0);
            t0 = fam_acc1<FAM>(qc[1] - x0.y, t0);
            t1 = fam_acc1<FAM>(qc[0] - x1.x, t1);
            t1 = fam_acc1<FAM>(qc[1] - x1.y, t1);
          } else {
#pragma unroll
            for (int k = 0; k < D; ++k) {
              t0 = fam_acc1<FAM>(qc[k] - __ldg(pts + size_t(f + j) * D + k), t0);
              t1 = fam_acc1<FAM>(qc[k] - __ldg(pts + size_t(mid + j) * D + k), t1);
            }
          }
          a0 += ex2_approx(fmaf(fam_finish1<FAM>(t0), -scale, offn));
          a1 += ex2_approx(fmaf(fam_finish1<FAM>(t1), -scale, offn));
        }
        if (l - mid > nleft) {
          float t1 = 0.f;
#pragma unroll
          for (int k = 0; k < D; ++k)
            t1 = fam_acc1<FAM>(qc[k] - __ldg(pts + size_t(l - 1) * D + k), t1);
          a1 += ex2_approx(fmaf(fam_finish1<FAM>(t1), -scale, offn));
        }
        a = double(a0);
        b = double(a1);
        fast = (a0 > 0.f || a1 > 0.f) && offn < 800.f;
      }
      bool left = false;
      bool defer = !fast;
      if (fast) {
        const uint64_t key = nlink ? splitmix64(__ldg(nlink + h) ^ qlink)
                                   : route_key_q(key_prefix, (uint64_t(f) << 32) | l, qlink);
        const uint64_t m = splitmix64(key) >> 11;
        const double ssum = a + b;
        const double t = fma(double(m) * 0x1p-53, ssum, -a);
        const float rel = float(kTieMargin) * (1.f + fmaxf(0.f, -em) * (1.f / 32.f));
        const double M = fma(double(rel), fmin(a, b), (pruned + 0x1p-51) * ssum);
        left = t < 0.0;
        defer = fabs(t) <= M;  // tie guard
      }
      if (defer) {  // walk_kernel takes this walk on from here
        wh[i] = uint32_t(h);
        welm[i] = em;
        widx[atomicAdd(wcount, 1u)] = i;
        deferred = true;
        if (rowstep) sv0 = 0;  // the row step is walk_kernel's to count
        break;
      }
      if (rowstep) {  // absolute fp64 sums: exponent of the chosen double
        em = float(int((__double_as_longlong(left ? a : b) >> 52) & 0x7ff) - 1023);
      } else {
        const float c = left ? float(a) : float(b);
        em = float(int((__float_as_uint(c) >> 23) & 0xffu) - 127) - offn;
      }
      path |= (left ? 1u : 0u) << steps;
      ++steps;
      h = left ? 2 * h + 1 : 2 * h + 2;
      nf = left ? f : mid;
      nl = left ? mid : l;
    }
    if (!deferred) {  // sampler.cpp:196-198: leaf (query, source, 1)
      const uint32_t row_q = qrow[q];
      const uint32_t slot = atomicAdd(row_cnt + row_q, 1u);
      const uint64_t o = row_off[row_q] + slot;
      leaf_src[o] = nf;
      leaf_cnt[o] = 1u;
    }
  }
  // per-level tallies of the warp's walks: level lev0 + k holds the walks
  // with at least k steps (the last one is the leaf entry), evaluating their
  // k-th node's size when they step on
  {
    const unsigned grp = __match_any_sync(0xffffffffu, lev0);
    const uint32_t maxsteps = __reduce_max_sync(0xffffffffu, steps);
    const bool lead = (threadIdx.x & 31) == uint32_t(__ffs(grp) - 1);
    uint32_t nk = n0;
    for (uint32_t k = 0; k <= maxsteps; ++k) {
      // (a deferred walk's last node is walk_kernel's entry)
      const uint32_t n_ent =
          __popc(__ballot_sync(0xffffffffu, mine && k + (deferred ? 1u : 0u) <= steps) & grp);
      const uint32_t n_ev = __reduce_add_sync(grp, k < steps ? nk : 0u);
      const uint32_t at = lev0 + k;
      if (lead && n_ent && at < kMaxLevels) {
        atomicAdd(&s_stats[0][at], n_ent);
        atomicAdd(&s_stats[1][at], n_ev);
      }
      if (k == 0) {
        const uint32_t n_sv = __reduce_add_sync(grp, sv0);
        if (lead && n_sv && at < kMaxLevels) atomicAdd(&s_stats[4][at], n_sv);
      }
      nk = ((path >> k) & 1u) ? nk / 2 : nk - nk / 2;
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
  // the fast kernel relies on the tie guard (reference RNG, verify on);
  // FSGG_WALK_FAST=0 keeps the per-child-offset kernel
  const char* e = std::getenv("FSGG_WALK_FAST");  // read per call: tests toggle it
  const bool fast = a.verify && a.rng_mode == 0 && !(e && e[0] == '0');
  uint32_t *widx = nullptr, *wcount = nullptr;
  if (fast) {
    widx = ds.buf("walk.deferred", size_t(a.W) * 4).as<uint32_t>();
    wcount = ds.buf("walk.ndeferred", 4).as<uint32_t>();
    FSGG_CUDA(cudaMemsetAsync(wcount, 0, 4, s));
    ds.launches++;
  }
  auto launch = [&](auto dim, auto fam) {
    constexpr int D = decltype(dim)::value;
    constexpr int FAM = decltype(fam)::value;
    uint32_t grid = ceil_div_u32(a.W, kWalkThreads);
    if (fast) {
      walk_fast_kernel<D, FAM><<<grid, kWalkThreads, 0, s>>>(
          ds.pts.as<float>(), a.W, a.wq, const_cast<uint32_t*>(a.wh),
          const_cast<float*>(a.welm), widx, wcount, t.first.as<uint32_t>(),
          t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(), t.has_boxes, ks.scale,
          a.key_prefix, a.qrow, a.row_off, a.row_cnt, a.leaf_src, a.leaf_cnt, a.stats, a.nlink,
          a.wrow, a.wrm, a.rows, a.rows_level);
      grid = std::min<uint32_t>(grid, uint32_t(ds.num_sms) * 4);  // the deferred few
    }
    walk_kernel<D, FAM><<<grid, kWalkThreads, 0, s>>>(
        ds.pts.as<float>(), a.W, a.wq, a.wh, a.welm, t.first.as<uint32_t>(),
        t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(), t.has_boxes, ks.scale,
        ks.family, ks.sigma, a.key_prefix, a.rng_mode, a.seed, a.verify, a.qrow, a.row_off,
        a.row_cnt, a.leaf_src, a.leaf_cnt, a.stats, a.nlink, a.wrow, a.wrm, a.rows,
        a.rows_level, widx, wcount);
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
