// Fused kernel-sum ("KDE") kernels: the device replacement of the
// reference's ExactKdeEstimator::eval / compensated_range_sum
// (proj/src/kde.cpp:38-71) and of the sampler's inline sums
// (proj/src/sampler.cpp:34-73), batched over a whole tree level.
//
// For every entry (node, query) of a level the sampler needs the two child
// sums g1 = sum_{j in [first,mid)} k(x_q, x_j) and g2 over [mid, last)
// (proj/src/sampler.cpp:141-149). The n x n kernel matrix is never
// materialised: sources stream through shared memory, exponentials go
// through MUFU.EX2 and each sum is reduced in registers.
//
// Numerics (SURVEY.md §8a'):
//  * direct differences (q - x) in fp32 (the expanded ||q||^2+||x||^2-2q.x
//    form loses 1e-4 by cancellation at n = 1M), exponent in base 2;
//  * each (entry, source-chunk) pair carries an exponent offset
//    off = scale * dist(q, bbox(chunk)) <= every term's exponent, so terms
//    are evaluated as 2^(off - scale*dist) <= 1 and never flush to zero in
//    fp32 while they are representable in fp64; the chunk sum is rescaled by
//    2^-off in fp64. Algebraically exact, so the offset's own rounding does
//    not matter;
//  * fp32 accumulation within a shared-memory tile, fp64 across tiles and
//    chunks, combined in a fixed order: results depend only on (node, query),
//    never on how entries are batched or sharded across GPUs.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "engine.cuh"
#include "kde_math.cuh"

namespace fsgg {

KernelSpec make_kernel_spec(int family, double sigma) {
  KernelSpec k;
  k.family = family;
  k.sigma = sigma;
  const double log2e = 1.4426950408889634074;
  k.scale = static_cast<float>(family == 0 ? log2e / (sigma * sigma)
                                           : log2e / sigma);
  return k;
}

KdeWorkspace::~KdeWorkspace() {
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
}

namespace {

constexpr int kThreads = 128;        // low-d tiled kernel CTA
constexpr int kBE = 2 * kThreads;    // entries per low-d work item (2/thread)
constexpr int kXThreads = 128;       // high-d tiled kernel CTA
constexpr int kXBM = 64;             // entries per high-d work item
constexpr int kXBN = 64;             // sources per high-d tile
constexpr int kXBK = 16;             // dims per high-d k-step
constexpr uint32_t kChunkMin = 2048; // smallest source chunk of one item
constexpr uint64_t kMaxPartials = 2560ull << 20;  // doubles (20 GiB of the 180 GB HBM)
constexpr float kPad = 3.0e18f;      // padding coordinate: term underflows to 0
constexpr uint32_t kFlush = 256;     // fp32 run length before the fp64 flush
#ifndef FSGG_POLY_EVERY
#define FSGG_POLY_EVERY 16
#endif
// 1 in kPolyEvery exp2 on the FP32 pipe (ex2_poly2); 0 = all on MUFU
constexpr uint32_t kPolyEvery = FSGG_POLY_EVERY;
constexpr uint32_t kSubMin = 512;    // smallest sub-chunk (pruning granularity)
constexpr uint32_t kSubMinSmall = 64;  // ... for nodes below 8 * kSubMin points
constexpr uint32_t kSubMinRow = 32;    // per-sub-chunk rows: sub-chunks of >= 32 points

template <int D>
struct LowDTile {
  static constexpr int T = D <= 2 ? 2048 : (D <= 4 ? 1024 : 512);
};

__device__ __forceinline__ double rescale(double acc, float off) {
  return rescale_off(acc, off);  // kde_math.cuh
}

// Work-item -> node slot lookup: largest g with blk_off[g] <= blk.
__device__ __forceinline__ uint32_t find_slot(const uint32_t* blk_off,
                                              uint32_t num_slots,
                                              uint32_t blk) {
  uint32_t lo = 0, hi = num_slots;  // blk_off[lo] <= blk < blk_off[hi]
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (blk_off[mid] <= blk)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Sum of 2^(off - scale*dist) over the lenp staged sources (negated, each
// coordinate stored once, padded to a multiple of 4 sources) for two packed
// entries: fp32 partial sums over runs of kFlush sources, flushed into fp64
// (keeps the accumulation error ~1e-7 relative at no measurable cost).
// Four sources come in with D 16-byte loads and enter the packed operations
// as broadcast scalar operands (FADD2 R, R.F32x2, R.F32): shared-memory
// loads share the MIO queue with MUFU, the binding pipe, so a source costs a
// quarter to a half of a load instead of one.
template <int D, int FAM>
__device__ __forceinline__ void lowd_staged_sum(const float* sm, uint32_t lenp,
                                                const float2 (&q2)[D], float2 off2,
                                                float scale, double& accA, double& accB) {
  const float2 ms = make_float2(-scale, -scale);
  for (uint32_t j0 = 0; j0 < lenp; j0 += kFlush) {
    const uint32_t j1 = min(lenp, j0 + kFlush);
    float2 acc = make_float2(0.f, 0.f);
    // the four sources j .. j + 3 (j a multiple of 4)
    auto load4 = [&](uint32_t j, float (&xs)[4 * D]) {
      const float4* p = reinterpret_cast<const float4*>(sm + size_t(j) * D);
#pragma unroll
      for (int v4 = 0; v4 < D; ++v4) {
        const float4 v = p[v4];
        xs[4 * v4] = v.x;
        xs[4 * v4 + 1] = v.y;
        xs[4 * v4 + 2] = v.z;
        xs[4 * v4 + 3] = v.w;
      }
    };
    auto arg_of = [&](const float* x) {
      float2 t = fam_first<FAM>(__fadd2_rn(q2[0], make_float2(x[0], x[0])));
#pragma unroll
      for (int k = 1; k < D; ++k)
        t = fam_next<FAM>(__fadd2_rn(q2[k], make_float2(x[k], x[k])), t);
      t = fam_finish<FAM>(t);
      return __ffma2_rn(t, ms, off2);
    };
    uint32_t j = j0;
    // one source in kPolyEvery takes the FP32-pipe exp2, the rest MUFU:
    // balances the two pipes (the loop is MUFU-bound otherwise)
    static_assert(kPolyEvery % 4 == 0, "sources are loaded four at a time");
    if (kPolyEvery > 0)
      for (; j + kPolyEvery <= j1; j += kPolyEvery) {
#pragma unroll
        for (uint32_t u4 = 0; u4 < kPolyEvery; u4 += 4) {
          float xs[4 * D];
          load4(j + u4, xs);
#pragma unroll
          for (uint32_t u = 0; u < 4; ++u) {
            const float2 arg = arg_of(xs + u * D);
            if (u4 + u == kPolyEvery - 1)
              acc = __fadd2_rn(acc, ex2_poly2(arg));
            else
              acc = __fadd2_rn(acc, make_float2(ex2_approx(arg.x), ex2_approx(arg.y)));
          }
        }
      }
    for (; j < j1; j += 4) {
      float xs[4 * D];
      load4(j, xs);
#pragma unroll
      for (uint32_t u = 0; u < 4; ++u) {
        const float2 arg = arg_of(xs + u * D);
        acc = __fadd2_rn(acc, make_float2(ex2_approx(arg.x), ex2_approx(arg.y)));
      }
    }
    accA += acc.x;
    accB += acc.y;
  }
}

// Sum of 2^(off - scale*dist) over sources [cf, cl) for two packed entries;
// sources staged negated in shared memory.
template <int D, int FAM>
__device__ __forceinline__ void lowd_range_sum(
    const float* __restrict__ pts, float* sm, const float2 (&q2)[D],
    float2 off2, float scale, uint32_t cf, uint32_t cl, double& accA,
    double& accB, bool warp_skip = false) {
  constexpr int T = LowDTile<D>::T;
  for (uint32_t t0 = cf; t0 < cl; t0 += T) {
    const uint32_t len = min(uint32_t(T), cl - t0);
    const uint32_t lenp = (len + 3u) & ~3u;
    __syncthreads();
    const float* src = pts + size_t(t0) * D;
    for (uint32_t idx = threadIdx.x; idx < lenp * D; idx += blockDim.x) {
      sm[idx] = idx < len * D ? -__ldg(src + idx) : -kPad;
    }
    __syncthreads();
    if (warp_skip) continue;  // this warp's entries all prune the range
    lowd_staged_sum<D, FAM>(sm, lenp, q2, off2, scale, accA, accB);
  }
}

// ---- low-d tiled kernel (node size > direct threshold) --------------------
// One CTA = (node slot, block of <= 256 entries, child side, chunk group).
// A chunk group is one of the child's tree descendants `cdepth` levels down;
// it is walked as its descendants `sdepth` levels below the child
// ("sub-chunks", ~1-2K sources, one shared-memory tile each). Boundaries and
// bounding boxes of both come from the tree table, so they depend only on
// the node. Writes one fp64 partial per (entry, side, group).
//
// Certified pruning (prune != 0): a sub-chunk c can contribute at most
// |c| * 2^-off_c to an entry's sum (off_c = scale * dist(q, bbox(c))). It is
// skipped when that bound is below 2^-kPruneBits of half the entry's node
// mass (known from the previous level; >= 1 at the root, which holds the
// query itself). With at most 2^20 sub-chunks per node the total skipped
// mass is < 2^-27 of the node mass (kPruneBits = 48), below the fp32
// evaluation error of the sums; the tie guard adds this bound to its margin,
// so routing decisions still match the fp64 reference exactly (a draw that
// close to p is re-decided on exact sums). The whole CTA skips when all its entries agree; a warp skips
// the arithmetic when all of its entries do; a pruned sub-chunk is dropped
// from an entry's sum whether or not its CTA evaluated it.
template <int D, int FAM>
__global__ void __launch_bounds__(kThreads)
    kde_lowd_tiled_kernel(const float* __restrict__ pts,
                          const uint32_t* __restrict__ eq,
                          const float* __restrict__ elm,
                          const uint32_t* __restrict__ goff,
                          const uint32_t* __restrict__ blk_off,
                          uint32_t num_slots, uint32_t level, uint32_t cdepth,
                          uint32_t sdepth, const uint32_t* __restrict__ tfirst,
                          const uint32_t* __restrict__ tlast,
                          const float* __restrict__ tlo,
                          const float* __restrict__ thi, int has_boxes,
                          float scale, float prune_bits, double* __restrict__ partials,
                          unsigned long long* __restrict__ performed, int per_sub) {
  const bool prune = prune_bits > 0.f;
  constexpr int T = LowDTile<D>::T;
  __shared__ __align__(16) float sm[T * D];
  __shared__ unsigned long long s_done;
  const uint32_t K = 1u << cdepth;
  const uint32_t item = blockIdx.x;
  const uint32_t blk = item >> (cdepth + 1);
  const uint32_t side = (item >> cdepth) & 1u;
  const uint32_t kk = item & (K - 1);
  const uint32_t g = find_slot(blk_off, num_slots, blk);
  const uint32_t e0 = goff[g] + (blk - blk_off[g]) * kBE;
  const uint32_t e1 = min(e0 + kBE, goff[g + 1]);

  const uint32_t ia = e0 + threadIdx.x, ib = ia + kThreads;
  const bool va = ia < e1, vb = ib < e1;
  const uint32_t qa = eq[va ? ia : e0], qb = eq[vb ? ib : e0];
  float qa_c[D], qb_c[D];
  float2 q2[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    qa_c[k] = __ldg(pts + size_t(qa) * D + k);
    qb_c[k] = __ldg(pts + size_t(qb) * D + k);
    q2[k] = make_float2(qa_c[k], qb_c[k]);
  }
  // log2 of a lower bound of each entry's node mass (half the previous
  // level's exact sum; the root holds the query itself, so >= 1 there)
  const float lbA = prune ? (elm ? elm[va ? ia : e0] : 0.f) - 1.f : 0.f;
  const float lbB = prune ? (elm ? elm[vb ? ib : e0] : 0.f) - 1.f : 0.f;
  if (threadIdx.x == 0) s_done = 0;

  const uint32_t nsub = 1u << (sdepth - cdepth);
  const uint32_t ls = level + 1 + sdepth;
  const uint64_t hbase = ((1ull << ls) - 1) +
                         ((uint64_t(2 * g + side) << sdepth) + uint64_t(kk) * nsub);
  const uint32_t nvalid_warp =
      __popc(__ballot_sync(0xffffffffu, va)) + __popc(__ballot_sync(0xffffffffu, vb));
  unsigned long long done = 0;
  double accA = 0.0, accB = 0.0;
  for (uint32_t sc = 0; sc < nsub; ++sc) {
    const uint64_t h = hbase + sc;
    const uint32_t cf = tfirst[h], cl = tlast[h];
    float offA = 0.f, offB = 0.f;
    if (has_boxes) {
      offA = scale * box_dist<FAM>(qa_c, tlo + h * D, thi + h * D, D);
      offB = scale * box_dist<FAM>(qb_c, tlo + h * D, thi + h * D, D);
    }
    bool skipA = false, skipB = false;
    if (prune) {
      const float lim = __log2f(float(cl - cf)) + prune_bits;
      skipA = !va || offA > lim - lbA;
      skipB = !vb || offB > lim - lbB;
    }
    const bool skip = skipA && skipB;
    if (__syncthreads_and(skip)) continue;
    const bool wskip = __all_sync(0xffffffffu, skip);
    double sA = 0.0, sB = 0.0;
    lowd_range_sum<D, FAM>(pts, sm, q2, make_float2(offA, offB), scale, cf, cl, sA, sB,
                           wskip);
    // A pruned sub-chunk contributes nothing to that entry even when its CTA
    // evaluates it for others: each sum depends on (node, query) alone, never
    // on which entries share the CTA (so sharded and unsharded runs agree).
    const double rA = skipA ? 0.0 : rescale(sA, offA);
    const double rB = skipB ? 0.0 : rescale(sB, offB);
    if (per_sub) {  // one partial per sub-chunk: rows sdepth + 1 deep (c == 0)
      const uint32_t stride = 2u * nsub, col = side * nsub + sc;
      if (va) partials[size_t(ia) * stride + col] = rA;
      if (vb) partials[size_t(ib) * stride + col] = rB;
    }
    accA += rA;
    accB += rB;
    if (!wskip) done += uint64_t(cl - cf) * nvalid_warp;
  }
  if (!per_sub) {
    const uint32_t stride = 2u * K, col = side * K + kk;
    if (va) partials[size_t(ia) * stride + col] = accA;
    if (vb) partials[size_t(ib) * stride + col] = accB;
  }
  if (performed) {
    if ((threadIdx.x & 31) == 0 && done) atomicAdd(&s_done, done);
    __syncthreads();
    if (threadIdx.x == 0 && s_done) atomicAdd(performed, s_done);
  }
}

// ---- low-d node kernel: two-deep rows of small nodes ------------------------
// The per-sub-chunk case of the tiled kernel with one work item per (node
// slot, block of <= 256 entries) instead of one per child side (C3 level 12:
// 245-point nodes, four ~61-point sub-chunks): the node's points are staged
// once, each sub-chunk at its own 4-aligned offset, and the four sub-chunk
// sums follow without a barrier in between — half the work items (slot
// search, query gathers) and one barrier instead of seven. Sub-chunk sums,
// offsets, pruning rule and partial layout are the tiled kernel's, bit for bit.
constexpr uint32_t kNodeMax = 4 * kSubMinSmall;  // node points (2 children x 2 x < 64)

template <int D, int FAM>
__global__ void __launch_bounds__(kThreads)
    kde_lowd_node_kernel(const float* __restrict__ pts, const uint32_t* __restrict__ eq,
                         const float* __restrict__ elm, const uint32_t* __restrict__ goff,
                         const uint32_t* __restrict__ blk_off, uint32_t num_slots,
                         uint32_t level, const uint32_t* __restrict__ tfirst,
                         const uint32_t* __restrict__ tlast, const float* __restrict__ tlo,
                         const float* __restrict__ thi, int has_boxes, float scale,
                         float prune_bits, double* __restrict__ partials,
                         unsigned long long* __restrict__ performed,
                         double* __restrict__ g1, double* __restrict__ g2) {
  const bool prune = prune_bits > 0.f;
  __shared__ __align__(16) float sm[(kNodeMax + 16) * D];
  __shared__ unsigned long long s_done;
  const uint32_t blk = blockIdx.x;
  const uint32_t g = find_slot(blk_off, num_slots, blk);
  const uint32_t e0 = goff[g] + (blk - blk_off[g]) * kBE;
  const uint32_t e1 = min(e0 + kBE, goff[g + 1]);
  // sub-chunks: the node's descendants two levels down, in order
  const uint64_t hbase = ((1ull << (level + 2)) - 1) + (uint64_t(g) << 2);
  uint32_t cf[4], cl[4], so[4];
  uint32_t at = 0;
#pragma unroll
  for (int sc = 0; sc < 4; ++sc) {
    cf[sc] = tfirst[hbase + sc];
    cl[sc] = tlast[hbase + sc];
    so[sc] = at;
    at += (cl[sc] - cf[sc] + 3u) & ~3u;
  }
  if (threadIdx.x == 0) s_done = 0;
#pragma unroll
  for (int sc = 0; sc < 4; ++sc) {
    const uint32_t len = cl[sc] - cf[sc], lenp = (len + 3u) & ~3u;
    const float* src = pts + size_t(cf[sc]) * D;
    for (uint32_t idx = threadIdx.x; idx < lenp * D; idx += blockDim.x) {
      sm[so[sc] * D + idx] = idx < len * D ? -__ldg(src + idx) : -kPad;
    }
  }
  const uint32_t ia = e0 + threadIdx.x, ib = ia + kThreads;
  const bool va = ia < e1, vb = ib < e1;
  const uint32_t qa = eq[va ? ia : e0], qb = eq[vb ? ib : e0];
  float qa_c[D], qb_c[D];
  float2 q2[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    qa_c[k] = __ldg(pts + size_t(qa) * D + k);
    qb_c[k] = __ldg(pts + size_t(qb) * D + k);
    q2[k] = make_float2(qa_c[k], qb_c[k]);
  }
  const float lbA = prune ? (elm ? elm[va ? ia : e0] : 0.f) - 1.f : 0.f;
  const float lbB = prune ? (elm ? elm[vb ? ib : e0] : 0.f) - 1.f : 0.f;
  const uint32_t nvalid_warp =
      __popc(__ballot_sync(0xffffffffu, va)) + __popc(__ballot_sync(0xffffffffu, vb));
  __syncthreads();
  unsigned long long done = 0;
  double rA[4], rB[4];
#pragma unroll
  for (int sc = 0; sc < 4; ++sc) {
    const uint64_t h = hbase + sc;
    float offA = 0.f, offB = 0.f;
    if (has_boxes) {
      offA = scale * box_dist<FAM>(qa_c, tlo + h * D, thi + h * D, D);
      offB = scale * box_dist<FAM>(qb_c, tlo + h * D, thi + h * D, D);
    }
    bool skipA = false, skipB = false;
    if (prune) {
      const float lim = __log2f(float(cl[sc] - cf[sc])) + prune_bits;
      skipA = !va || offA > lim - lbA;
      skipB = !vb || offB > lim - lbB;
    }
    double sA = 0.0, sB = 0.0;
    if (!__all_sync(0xffffffffu, skipA && skipB)) {
      lowd_staged_sum<D, FAM>(sm + so[sc] * D, (cl[sc] - cf[sc] + 3u) & ~3u, q2,
                              make_float2(offA, offB), scale, sA, sB);
      done += uint64_t(cl[sc] - cf[sc]) * nvalid_warp;
    }
    rA[sc] = skipA ? 0.0 : rescale(sA, offA);
    rB[sc] = skipB ? 0.0 : rescale(sB, offB);
  }
  // the row, and the entry's child sums (finalize_kernel's: buckets added in
  // order, floored)
  if (va) {
    double2* p = reinterpret_cast<double2*>(partials + size_t(ia) * 4);
    p[0] = make_double2(rA[0], rA[1]);
    p[1] = make_double2(rA[2], rA[3]);
    g1[ia] = fmax(rA[0] + rA[1], kSumFloor);
    g2[ia] = fmax(rA[2] + rA[3], kSumFloor);
  }
  if (vb) {
    double2* p = reinterpret_cast<double2*>(partials + size_t(ib) * 4);
    p[0] = make_double2(rB[0], rB[1]);
    p[1] = make_double2(rB[2], rB[3]);
    g1[ib] = fmax(rB[0] + rB[1], kSumFloor);
    g2[ib] = fmax(rB[2] + rB[3], kSumFloor);
  }
  if (performed) {
    if ((threadIdx.x & 31) == 0 && done) atomicAdd(&s_done, done);
    __syncthreads();
    if (threadIdx.x == 0 && s_done) atomicAdd(performed, s_done);
  }
}

// ---- low-d direct kernel (small nodes: one thread per entry) --------------
template <int D, int FAM>
__global__ void __launch_bounds__(256)
    kde_lowd_direct_kernel(const float* __restrict__ pts,
                           const uint32_t* __restrict__ eq,
                           const uint32_t* __restrict__ eg, uint32_t E,
                           uint32_t level, const uint32_t* __restrict__ tfirst,
                           const uint32_t* __restrict__ tlast,
                           const float* __restrict__ tlo,
                           const float* __restrict__ thi, int has_boxes,
                           float scale, double* __restrict__ g1,
                           double* __restrict__ g2, double* __restrict__ groot,
                           const uint32_t* __restrict__ dE,
                           unsigned long long* __restrict__ evals) {
  // dE: the entry count on the device (E is then the grid's upper bound,
  // grid-strided) and the reference-equivalent evaluations are tallied here
  if (dE) E = *dE;
  unsigned long long ev = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < E; i += gridDim.x * blockDim.x) {
    const uint64_t h = ((1ull << level) - 1) + eg[i];
    const uint32_t f = tfirst[h], l = tlast[h];
    if (l - f < 2) {
      g1[i] = g2[i] = 0.0;
      continue;
    }
    ev += l - f;
    const uint32_t q = eq[i];
    float qc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) qc[k] = __ldg(pts + size_t(q) * D + k);
    double s[2];
    direct_child_sums<D, FAM>(pts, qc, h, f, l, tlo, thi, has_boxes, scale, s);
    g1[i] = fmax(s[0], kSumFloor);
    g2[i] = fmax(s[1], kSumFloor);
    if (groot) groot[i] = fmax(s[0] + s[1], kSumFloor);
  }
  if (evals) {
    for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
    if ((threadIdx.x & 31) == 0 && ev) atomicAdd(evals, ev);
  }
}

// ---- high-d tiled kernel (CUDA-core micro-tiles, direct differences) ------
// 64 entries x 64 sources per tile, k-steps of 16 dims; each thread owns a
// 4 x 8 block of (entry, source) squared distances.
template <int FAM>
__device__ __forceinline__ void xd_tile_sums(
    const float* __restrict__ pts, uint32_t d, const uint32_t* qrow,  // smem
    float (*sq)[kXBM], float (*sx)[kXBN], uint32_t cf, uint32_t cl,
    const float* off /*4 rows*/, float scale, double* racc /*4 rows*/) {
  const int tid = threadIdx.x;
  const int tr = tid >> 3;  // row group: rows tr*4 .. tr*4+3
  const int tc = tid & 7;   // cols tc*4..+3 and 32+tc*4..+3
  for (uint32_t s0 = cf; s0 < cl; s0 += kXBN) {
    const uint32_t len = min(uint32_t(kXBN), cl - s0);
    float acc[4][8];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
    for (uint32_t k0 = 0; k0 < d; k0 += kXBK) {
      __syncthreads();
      for (int idx = tid; idx < kXBK * kXBM; idx += kXThreads) {
        const int m = idx / kXBK, k = idx % kXBK;
        const uint32_t kg = k0 + k;
        sq[k][m] = kg < d ? __ldg(pts + size_t(qrow[m]) * d + kg) : 0.f;
      }
      for (int idx = tid; idx < kXBK * kXBN; idx += kXThreads) {
        const int c = idx / kXBK, k = idx % kXBK;
        const uint32_t kg = k0 + k;
        float v = 0.f;
        if (kg < d) v = c < int(len) ? -__ldg(pts + size_t(s0 + c) * d + kg) : -kPad;
        sx[k][c] = v;
      }
      __syncthreads();
#pragma unroll 4
      for (int k = 0; k < kXBK; ++k) {
        const float4 qv = *reinterpret_cast<const float4*>(&sq[k][tr * 4]);
        const float4 x0 = *reinterpret_cast<const float4*>(&sx[k][tc * 4]);
        const float4 x1 = *reinterpret_cast<const float4*>(&sx[k][32 + tc * 4]);
        const float qr[4] = {qv.x, qv.y, qv.z, qv.w};
        const float xc[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float2 qq = make_float2(qr[r], qr[r]);
#pragma unroll
          for (int c = 0; c < 8; c += 2) {
            const float2 dk = __fadd2_rn(qq, make_float2(xc[c], xc[c + 1]));
            float2 t = make_float2(acc[r][c], acc[r][c + 1]);
            t = fam_next<FAM>(dk, t);
            acc[r][c] = t.x;
            acc[r][c + 1] = t.y;
          }
        }
      }
    }
    // epilogue: exponentials and per-row sums for this source tile
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int col = c < 4 ? tc * 4 + c : 32 + tc * 4 + (c - 4);
        const float t = fam_finish1<FAM>(acc[r][c]);
        const float e = ex2_approx(fmaf(t, -scale, off[r]));
        rs += col < int(len) ? e : 0.f;
      }
      rs += __shfl_xor_sync(0xffffffffu, rs, 1);
      rs += __shfl_xor_sync(0xffffffffu, rs, 2);
      rs += __shfl_xor_sync(0xffffffffu, rs, 4);
      racc[r] += rs;
    }
  }
}

template <int FAM>
__global__ void __launch_bounds__(kXThreads)
    kde_xd_tiled_kernel(const float* __restrict__ pts, uint32_t d,
                        const uint32_t* __restrict__ eq,
                        const uint32_t* __restrict__ goff,
                        const uint32_t* __restrict__ blk_off,
                        uint32_t num_slots, uint32_t level, uint32_t cdepth,
                        const uint32_t* __restrict__ tfirst,
                        const uint32_t* __restrict__ tlast,
                        const float* __restrict__ tlo,
                        const float* __restrict__ thi, int has_boxes,
                        float scale, double* __restrict__ partials) {
  __shared__ __align__(16) float sq[kXBK][kXBM];
  __shared__ __align__(16) float sx[kXBK][kXBN];
  __shared__ uint32_t qrow[kXBM];
  __shared__ float soff[kXBM];
  const uint32_t K = 1u << cdepth;
  const uint32_t item = blockIdx.x;
  const uint32_t blk = item >> (cdepth + 1);
  const uint32_t side = (item >> cdepth) & 1u;
  const uint32_t kk = item & (K - 1);
  const uint32_t g = find_slot(blk_off, num_slots, blk);
  const uint32_t e0 = goff[g] + (blk - blk_off[g]) * kXBM;
  const uint32_t e1 = min(e0 + kXBM, goff[g + 1]);
  const uint32_t lc = level + 1 + cdepth;
  const uint64_t h = ((1ull << lc) - 1) + ((uint64_t(2 * g + side)) << cdepth) + kk;
  const uint32_t cf = tfirst[h], cl = tlast[h];
  if (threadIdx.x < kXBM) {
    const uint32_t e = e0 + threadIdx.x;
    const uint32_t q = eq[e < e1 ? e : e0];
    qrow[threadIdx.x] = q;
    float off = 0.f;
    if (has_boxes) {
      float qc[kBoxMaxDim];
      for (uint32_t k = 0; k < d; ++k) qc[k] = __ldg(pts + size_t(q) * d + k);
      off = scale * box_dist<FAM>(qc, tlo + h * d, thi + h * d, d);
    }
    soff[threadIdx.x] = off;
  }
  __syncthreads();
  const int tr = threadIdx.x >> 3;
  float off[4];
  double racc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int r = 0; r < 4; ++r) off[r] = soff[tr * 4 + r];
  xd_tile_sums<FAM>(pts, d, qrow, sq, sx, cf, cl, off, scale, racc);
  if ((threadIdx.x & 7) == 0) {
    const uint32_t stride = 2u * K, col = side * K + kk;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const uint32_t e = e0 + tr * 4 + r;
      if (e < e1) partials[size_t(e) * stride + col] = rescale(racc[r], off[r]);
    }
  }
}

// ---- high-d direct kernel: one warp per entry ------------------------------
template <int FAM>
__global__ void __launch_bounds__(256)
    kde_xd_direct_kernel(const float* __restrict__ pts, uint32_t d,
                         const uint32_t* __restrict__ eq,
                         const uint32_t* __restrict__ eg, uint32_t E,
                         uint32_t level, const uint32_t* __restrict__ tfirst,
                         const uint32_t* __restrict__ tlast,
                         const float* __restrict__ tlo,
                         const float* __restrict__ thi, int has_boxes,
                         float scale, double* __restrict__ g1,
                         double* __restrict__ g2, double* __restrict__ groot) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= E) return;
  const uint64_t h = ((1ull << level) - 1) + eg[w];
  const uint32_t f = tfirst[h], l = tlast[h];
  if (l - f < 2) {
    if (lane == 0) g1[w] = g2[w] = 0.0;
    return;
  }
  const uint32_t mid = f + (l - f) / 2;
  const float* q = pts + size_t(eq[w]) * d;
  double s[2];
  for (int side = 0; side < 2; ++side) {
    const uint64_t hc = 2 * h + 1 + side;
    const uint32_t a = side ? mid : f, b = side ? l : mid;
    float off = 0.f;
    if (has_boxes) {
      float part = 0.f;
      for (uint32_t k = lane; k < d; k += 32) {
        float v = fmaxf(fmaxf(tlo[hc * d + k] - q[k], q[k] - thi[hc * d + k]), 0.f);
        part = (FAM == 2) ? part + v : fmaf(v, v, part);
      }
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      off = scale * fam_finish1<FAM>(part);
    }
    float acc = 0.f;
    for (uint32_t j = a; j < b; ++j) {
      const float* x = pts + size_t(j) * d;
      float part = 0.f;
      for (uint32_t k = lane; k < d; k += 32) part = fam_acc1<FAM>(__ldg(q + k) - __ldg(x + k), part);
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      acc += ex2_approx(fmaf(fam_finish1<FAM>(part), -scale, off));
    }
    s[side] = rescale(acc, off);
  }
  if (lane == 0) {
    g1[w] = fmax(s[0], kSumFloor);
    g2[w] = fmax(s[1], kSumFloor);
    if (groot) groot[w] = fmax(s[0] + s[1], kSumFloor);
  }
}

// ---- level bookkeeping -----------------------------------------------------
// Per slot: work blocks (size >= 2 nodes only) and evaluations
// (entries x node size, the reference's "kernel evals").
__global__ void slot_blocks_kernel(const uint32_t* __restrict__ goff,
                                   uint32_t num_slots, uint32_t level,
                                   const uint32_t* __restrict__ tfirst,
                                   const uint32_t* __restrict__ tlast,
                                   uint32_t be, uint32_t* __restrict__ nb,
                                   unsigned long long* __restrict__ evals) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long ev = 0;
  if (g < num_slots) {
    const uint64_t h = ((1ull << level) - 1) + g;
    const uint32_t size = tlast[h] - tfirst[h];
    const uint32_t ne = goff[g + 1] - goff[g];
    const bool work = size >= 2 && ne > 0;
    if (nb) nb[g] = work ? (ne + be - 1) / be : 0;
    ev = work ? (unsigned long long)ne * size : 0ull;
  } else if (nb && g == num_slots) {
    nb[g] = 0;
  }
  for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
  if ((threadIdx.x & 31) == 0 && ev) atomicAdd(evals, ev);
}

__global__ void finalize_kernel(const double* __restrict__ partials,
                                uint32_t K, const uint32_t* __restrict__ eg,
                                uint32_t E, uint32_t level,
                                const uint32_t* __restrict__ tfirst,
                                const uint32_t* __restrict__ tlast,
                                double* __restrict__ g1,
                                double* __restrict__ g2,
                                double* __restrict__ groot) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E) return;
  const uint64_t h = ((1ull << level) - 1) + eg[i];
  if (tlast[h] - tfirst[h] < 2) {
    g1[i] = g2[i] = 0.0;
    return;
  }
  const double* p = partials + size_t(i) * 2 * K;
  double a = 0.0, b = 0.0;
  for (uint32_t k = 0; k < K; ++k) a += p[k];
  for (uint32_t k = 0; k < K; ++k) b += p[K + k];
  g1[i] = fmax(a, kSumFloor);
  g2[i] = fmax(b, kSumFloor);
  if (groot) groot[i] = fmax(a + b, kSumFloor);
}

// Pairwise-sum pyramid of each entry's partial row (rd >= 2): one warp per
// entry stages the 2^rd buckets in shared memory, writes depths rd-1 .. 1
// (fixed pairwise order) to pyr, and the two depth-1 sums as the entry's
// child sums. Lookups at the next levels then read two values per entry.
__global__ void pyramid_kernel(const double* __restrict__ partials, uint32_t rd,
                               const uint32_t* __restrict__ eg, uint32_t E, uint32_t level,
                               const uint32_t* __restrict__ tfirst,
                               const uint32_t* __restrict__ tlast, double* __restrict__ pyr,
                               double* __restrict__ g1, double* __restrict__ g2,
                               double* __restrict__ groot) {
  extern __shared__ double psm[];
  const uint32_t W = 1u << rd;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t i = blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= E) return;
  double* a = psm + size_t(warp) * 2 * W;  // level m+1 values
  double* b = a + W;                        // level m values
  const double* row = partials + (size_t(i) << rd);
  double* out = pyr + (size_t(i) << rd);
  for (uint32_t k = lane; k < W; k += 32) a[k] = row[k];
  __syncwarp();
  for (uint32_t m = rd - 1; m >= 1; --m) {
    const uint32_t cnt = 1u << m;
    for (uint32_t k = lane; k < cnt; k += 32) {
      const double v = a[2 * k] + a[2 * k + 1];
      b[k] = v;
      out[(cnt - 2) + k] = v;
    }
    __syncwarp();
    for (uint32_t k = lane; k < cnt; k += 32) a[k] = b[k];
    __syncwarp();
  }
  if (lane == 0) {
    const uint64_t h = ((1ull << level) - 1) + eg[i];
    if (tlast[h] - tfirst[h] < 2) {
      g1[i] = g2[i] = 0.0;
    } else {
      g1[i] = fmax(a[0], kSumFloor);
      g2[i] = fmax(a[1], kSumFloor);
      if (groot) groot[i] = fmax(a[0] + a[1], kSumFloor);
    }
  }
}

// ---- arbitrary-range evaluation (KdeEstimator::eval seam) -----------------
__global__ void range_box_kernel(const float* __restrict__ pts, uint32_t d,
                                 uint32_t first, uint32_t last, float* lo,
                                 float* hi) {
  // one CTA per dimension
  const uint32_t k = blockIdx.x;
  float mn = FLT_MAX, mx = -FLT_MAX;
  for (uint32_t j = first + threadIdx.x; j < last; j += blockDim.x) {
    const float v = pts[size_t(j) * d + k];
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
  __shared__ float smn[32], smx[32];
  for (int o = 16; o; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < blockDim.x / 32; ++w) {
      mn = fminf(mn, smn[w]);
      mx = fmaxf(mx, smx[w]);
    }
    lo[k] = mn;
    hi[k] = mx;
  }
}

template <int D, int FAM>
__global__ void __launch_bounds__(kThreads)
    kde_lowd_range_kernel(const float* __restrict__ pts,
                          const uint32_t* __restrict__ targets, uint32_t m,
                          uint32_t first, uint32_t last, uint32_t chunk,
                          uint32_t nchunks, const float* __restrict__ lo,
                          const float* __restrict__ hi, float scale,
                          double* __restrict__ partials) {
  constexpr int T = LowDTile<D>::T;
  __shared__ __align__(16) float sm[T * D];
  const uint32_t blk = blockIdx.x / nchunks, c = blockIdx.x % nchunks;
  const uint32_t cf = first + c * chunk, cl = min(last, cf + chunk);
  const uint32_t e0 = blk * kBE;
  const uint32_t ia = e0 + threadIdx.x, ib = ia + kThreads;
  const bool va = ia < m, vb = ib < m;
  const uint32_t qa = targets[va ? ia : e0], qb = targets[vb ? ib : e0];
  float qa_c[D], qb_c[D];
  float2 q2[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    qa_c[k] = pts[size_t(qa) * D + k];
    qb_c[k] = pts[size_t(qb) * D + k];
    q2[k] = make_float2(qa_c[k], qb_c[k]);
  }
  const float offA = scale * box_dist<FAM>(qa_c, lo, hi, D);
  const float offB = scale * box_dist<FAM>(qb_c, lo, hi, D);
  double accA = 0.0, accB = 0.0;
  lowd_range_sum<D, FAM>(pts, sm, q2, make_float2(offA, offB), scale, cf, cl,
                         accA, accB);
  if (va) partials[size_t(ia) * nchunks + c] = rescale(accA, offA);
  if (vb) partials[size_t(ib) * nchunks + c] = rescale(accB, offB);
}

template <int FAM>
__global__ void __launch_bounds__(256)
    kde_xd_range_kernel(const float* __restrict__ pts, uint32_t d,
                        const uint32_t* __restrict__ targets, uint32_t m,
                        uint32_t first, uint32_t last, uint32_t chunk,
                        uint32_t nchunks, const float* __restrict__ lo,
                        const float* __restrict__ hi, int has_box, float scale,
                        double* __restrict__ partials) {
  const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= uint64_t(m) * nchunks) return;
  const uint32_t t = w / nchunks, c = w % nchunks;
  const uint32_t a = first + c * chunk, b = min(last, a + chunk);
  const float* q = pts + size_t(targets[t]) * d;
  float off = 0.f;
  if (has_box) {
    float part = 0.f;
    for (uint32_t k = lane; k < d; k += 32) {
      float v = fmaxf(fmaxf(lo[k] - q[k], q[k] - hi[k]), 0.f);
      part = (FAM == 2) ? part + v : fmaf(v, v, part);
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    off = scale * fam_finish1<FAM>(part);
  }
  float acc = 0.f;
  for (uint32_t j = a; j < b; ++j) {
    const float* x = pts + size_t(j) * d;
    float part = 0.f;
    for (uint32_t k = lane; k < d; k += 32) part = fam_acc1<FAM>(q[k] - x[k], part);
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    acc += ex2_approx(fmaf(fam_finish1<FAM>(part), -scale, off));
  }
  if (lane == 0) partials[size_t(t) * nchunks + c] = rescale(acc, off);
}

__global__ void range_finalize_kernel(const double* __restrict__ partials,
                                      uint32_t nchunks, uint32_t m,
                                      int empty, double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (uint32_t c = 0; c < nchunks; ++c) s += partials[size_t(i) * nchunks + c];
  out[i] = empty ? 0.0 : fmax(s, kSumFloor);
}

// ---- dispatch --------------------------------------------------------------
template <int D, int FAM>
struct LowD {
  static void tiled(dim3 grid, cudaStream_t s, const float* pts,
                    const LevelView& lv, const uint32_t* blk_off,
                    uint32_t cdepth, uint32_t sdepth, const TreeTable& t,
                    float scale, double* partials,
                    unsigned long long* performed, int per_sub, bool whole_node,
                    double* g1, double* g2) {
    if (whole_node) {  // two-deep rows of small nodes: one item per entry block
      kde_lowd_node_kernel<D, FAM><<<grid.x / 2, kThreads, 0, s>>>(
          pts, lv.eq, lv.elm, lv.goff, blk_off, lv.num_slots, lv.level,
          t.first.as<uint32_t>(), t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(),
          t.has_boxes, scale, (lv.prune && t.has_boxes) ? lv.prune_bits : 0.f, partials,
          performed, g1, g2);
      return;
    }
    kde_lowd_tiled_kernel<D, FAM><<<grid, kThreads, 0, s>>>(
        pts, lv.eq, lv.elm, lv.goff, blk_off, lv.num_slots, lv.level, cdepth,
        sdepth, t.first.as<uint32_t>(), t.last.as<uint32_t>(), t.lo.as<float>(),
        t.hi.as<float>(), t.has_boxes, scale, (lv.prune && t.has_boxes) ? lv.prune_bits : 0.f, partials,
        performed, per_sub);
  }
  static void direct(cudaStream_t s, const float* pts, const LevelView& lv,
                     const TreeTable& t, float scale, double* g1, double* g2,
                     double* groot, uint32_t max_grid, unsigned long long* evals) {
    const uint32_t grid = lv.dE ? std::min(ceil_div_u32(lv.num_entries, 256), max_grid)
                                : ceil_div_u32(lv.num_entries, 256);
    kde_lowd_direct_kernel<D, FAM><<<grid, 256, 0, s>>>(
        pts, lv.eq, lv.eg, lv.num_entries, lv.level, t.first.as<uint32_t>(),
        t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(),
        t.has_boxes, scale, g1, g2, groot, lv.dE, evals);
  }
  static void range(dim3 grid, cudaStream_t s, const float* pts,
                    const uint32_t* targets, uint32_t m, uint32_t first,
                    uint32_t last, uint32_t chunk, uint32_t nchunks,
                    const float* lo, const float* hi, float scale,
                    double* partials) {
    kde_lowd_range_kernel<D, FAM><<<grid, kThreads, 0, s>>>(
        pts, targets, m, first, last, chunk, nchunks, lo, hi, scale, partials);
  }
};

template <template <int, int> class Op, int FAM>
struct ByDim {
  template <class F>
  static void run(uint32_t d, F&& f) {
    switch (d) {
      case 1: f(Op<1, FAM>{}); break;
      case 2: f(Op<2, FAM>{}); break;
      case 3: f(Op<3, FAM>{}); break;
      case 4: f(Op<4, FAM>{}); break;
      case 5: f(Op<5, FAM>{}); break;
      case 6: f(Op<6, FAM>{}); break;
      case 7: f(Op<7, FAM>{}); break;
      case 8: f(Op<8, FAM>{}); break;
      default: throw ConfigError("low-d path supports d <= 8");
    }
  }
};

template <class F>
void with_lowd(int family, uint32_t d, F&& f) {
  switch (family) {
    case 0: ByDim<LowD, 0>::run(d, f); break;
    case 1: ByDim<LowD, 1>::run(d, f); break;
    case 2: ByDim<LowD, 2>::run(d, f); break;
    default: throw ConfigError("unknown kernel family");
  }
}

template <class F>
void with_family(int family, F&& f) {
  switch (family) {
    case 0: f(std::integral_constant<int, 0>{}); break;
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    default: throw ConfigError("unknown kernel family");
  }
}

constexpr uint32_t kLowDMax = 8;
constexpr uint32_t kPyramidMinDepth = 6;  // rows of >= 64 buckets get a sum pyramid
constexpr uint32_t kTcDirectMax = 24;  // tensor-core levels: direct (warp per entry) for small nodes
uint32_t env_u32(const char* name, uint32_t dflt) {  // development overrides
  const char* e = std::getenv(name);
  return e ? uint32_t(std::atoi(e)) : dflt;
}
constexpr uint32_t kTcSubMin = 16;    // tensor-core partial buckets: >= 16 sources
constexpr uint32_t kTcChunkMin = 128; // ... work items: >= one 128-source N-tile
constexpr uint32_t kTcMaxRowDepth = 11;  // root rows serve ~10 levels (C5: 70k x 2^11 buckets)
uint32_t direct_threshold(uint32_t d) { return d <= kLowDMax ? 192u : 96u; }

}  // namespace

bool kde_level_sync_free(const Dataset& ds, const KernelSpec& ks, uint32_t level) {
  (void)ks;
  const uint32_t s_max = uint32_t((uint64_t(ds.n) + (1ull << level) - 1) >> level);
  return s_max < 2 || (ds.d <= kLowDMax && s_max <= direct_threshold(ds.d));
}

void kde_level(Dataset& ds, const KernelSpec& ks, const LevelView& lv,
               double* g1, double* g2, double* groot, KdeWorkspace& ws,
               KdeStats& stats, uint32_t serve_levels, uint32_t* row_depth) {
  const uint32_t E = lv.num_entries;
  if (row_depth) *row_depth = 0;
  if (E == 0) return;
  const uint32_t n = ds.n, d = ds.d;
  const uint32_t s_max = uint32_t((uint64_t(n) + (1ull << lv.level) - 1) >> lv.level);
  if (s_max < 2) return;  // every node is a leaf: routing emits, no sums
  cudaStream_t s = ds.stream;
  const TreeTable& t = ds.tree;
  const float* pts = ds.pts.as<float>();
  const bool lowd = d <= kLowDMax;
  const bool tc = !lowd && kde_tc_supported(ds, ks.family);
  const bool direct = s_max <= (tc ? env_u32("FSGG_TC_DIRECT", kTcDirectMax) : direct_threshold(d));
  const uint32_t be = lowd ? kBE : (tc ? 128u : uint32_t(kXBM));

  // blocks per slot + exact evaluation count of the level
  const uint32_t G = lv.num_slots;
  ws.blk_off.ensure(size_t(G + 4) * 4 + 64, s);
  uint32_t* nb = ws.blk_off.as<uint32_t>();
  unsigned long long* d_evals =
      reinterpret_cast<unsigned long long*>(nb + G + 2 + (G & 1));
  FSGG_CUDA(cudaMemsetAsync(d_evals, 0, 16, s));
  // direct levels add their evaluation count to ws.direct_evals (read once
  // by the caller after the descent: no host sync per small level); the
  // low-d direct kernel tallies it itself
  if (lv.dE && !(direct && lowd))
    throw ConfigError("device entry counts are only supported on low-d direct levels");
  if (direct) ws.direct_evals.ensure(8, s);
  if (!(direct && lowd)) {
    slot_blocks_kernel<<<ceil_div_u32(uint64_t(G) + 1, 256), 256, 0, s>>>(
        lv.goff, G, lv.level, t.first.as<uint32_t>(), t.last.as<uint32_t>(), be,
        direct ? nullptr : nb, direct ? ws.direct_evals.as<unsigned long long>() : d_evals);
    FSGG_LAUNCH_CHECK();
    ds.launches += 1;
  }

  if (direct) {
    if (lowd) {
      with_lowd(ks.family, d, [&](auto op) {
        op.direct(s, pts, lv, t, ks.scale, g1, g2, groot, uint32_t(ds.num_sms) * 16,
                  ws.direct_evals.as<unsigned long long>());
      });
    } else {
      with_family(ks.family, [&](auto fam) {
        constexpr int FAM = decltype(fam)::value;
        kde_xd_direct_kernel<FAM><<<ceil_div_u32(uint64_t(E) * 32, 256), 256, 0, s>>>(
            pts, d, lv.eq, lv.eg, E, lv.level, t.first.as<uint32_t>(),
            t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(),
            t.has_boxes, ks.scale, g1, g2, groot);
      });
    }
    FSGG_LAUNCH_CHECK();
    ds.launches += 1;
    return;
  }

  // exclusive scan of blocks per slot -> blk_off (in place, G + 1 entries)
  size_t tmp_bytes = 0;
  FSGG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, nb, nb, G + 1, s));
  ws.cub_tmp.ensure(tmp_bytes, s);
  FSGG_CUDA(cub::DeviceScan::ExclusiveSum(ws.cub_tmp.as<void>(), tmp_bytes, nb,
                                          nb, G + 1, s));
  unsigned long long* hw = ds.host_words();
  FSGG_CUDA(cudaMemcpyAsync(hw, d_evals, 8, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(hw + 1, nb + G, 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  const unsigned long long ev = hw[0];
  const uint32_t total_blocks = *reinterpret_cast<const uint32_t*>(hw + 1);
  ds.launches += 1;
  stats.evals += ev;
  stats.performed += ev;
  if (total_blocks == 0) return;

  // sub-chunk depth (pruning / tiling granularity, ~kSubMin..2*kSubMin
  // sources) and chunk-group depth c <= sd: enough independent items to fill
  // the GPU many times over, partials bounded.
  const uint32_t node_min = uint32_t(uint64_t(n) >> lv.level);
  const uint32_t child_min = node_min / 2;
  const uint64_t target_items = uint64_t(ds.num_sms) * 8 * 40;
  uint32_t sd = 0;
  // small nodes: finer sub-chunks so the partial rows can still serve the
  // next levels (pruning rarely applies there anyway)
  const uint32_t sub_min = child_min >= 8 * kSubMin ? kSubMin : kSubMinSmall;
  while ((child_min >> (sd + 1)) >= sub_min && lv.level + 2 + sd <= t.depth) ++sd;
  // c >= serve_levels - 1 keeps per-entry partials at the granularity of
  // the node's descendants c+1 levels down, so the next c levels' child sums
  // are range sums of this row (lookup_sums_kernel, sampler.cu) instead of
  // new kernel evaluations.
  uint32_t c = 0;
  int per_sub = 0;
  // rl: log2 of the partial-row width. The CUDA-core kernels write one
  // partial per work item (rl = c + 1); the tensor-core kernel splits its
  // columns at sub-chunk boundaries and writes one per sub-chunk (rl = sd + 1).
  uint32_t rl;
  if (tc) {
    sd = 0;
    // small nodes: buckets down to single points, so one tensor-core pass
    // serves every remaining level by lookups (C5 levels 12-15: the direct
    // warp-per-entry kernel re-read each 784-d query once per level)
    const uint32_t tc_sub_min = child_min >= 8 * kTcSubMin ? kTcSubMin : 1u;
    while ((child_min >> (sd + 1)) >= tc_sub_min && lv.level + 2 + sd <= t.depth &&
           sd + 1 < env_u32("FSGG_TC_ROWDEPTH", kTcMaxRowDepth) &&
           (uint64_t(E) << (sd + 2)) <= kMaxPartials)
      ++sd;
    while (c < sd && (child_min >> (c + 1)) >= kTcChunkMin &&
           (uint64_t(total_blocks) << (c + 1)) < target_items)
      ++c;
    rl = sd + 1;
  } else {
    while (c < sd && (child_min >> (c + 1)) >= (lowd ? sub_min : kChunkMin) &&
           ((uint64_t(total_blocks) << (c + 1)) < target_items || c + 1 < serve_levels) &&
           (uint64_t(E) << (c + 2)) <= kMaxPartials)
      ++c;
    rl = c + 1;
    // children of 64..127 points (C3 level 12): split each into two
    // sub-chunks and keep both partials per child (rows two levels deep,
    // same work items): the next level's child sums become lookups and a
    // walk starting below reads its first child sums from the row
    if (lowd && sd == 0 && c == 0 && child_min >= 2 * kSubMinRow &&
        child_min < 2 * kSubMinSmall && lv.level + 2 <= t.depth &&
        (uint64_t(E) << 2) <= kMaxPartials && env_u32("FSGG_SUBROWS", 1) != 0) {
      sd = 1;
      rl = 2;
      per_sub = 1;
    }
  }
  // the symmetric root pass (kde_sym.cu) writes rows at any depth up to its
  // block depth Lb (not tied to sub-chunks): as deep as serve_levels asks,
  // capped by Lb and by HBM
  const uint32_t Lb = (lowd && lv.level == 0 && lv.qbase != 0xffffffffu && lv.prune &&
                       env_u32("FSGG_SYM", 1) != 0)
                          ? sym_block_depth(ds)
                          : 0;
  if (Lb > 0) {
    // the block values (block_lookup_sums) serve every level whose children
    // are unions of blocks, so the fp64 rows only need to reach the levels
    // where a block lookup would sum many partners: kSymRootServe (measured
    // at C3: rows for levels 1-6 + block lookups for 7-11 beat rows to 8)
    if (!std::getenv("FSGG_ROOT_SERVE")) {
      serve_levels = std::min(serve_levels, kSymRootServe);
      rl = std::min(rl, serve_levels);
    }
    uint32_t want = std::min(std::max(rl, std::min(serve_levels, Lb)), Lb);
    while (want > 1 && (uint64_t(E) << (want + 1)) > kMaxPartials) --want;
    rl = want;
  }
  if (row_depth) *row_depth = rl;
  const uint32_t K = 1u << c;
  ws.partials.ensure(size_t(E) << rl << 3, s);
  double* partials = ws.partials.as<double>();
  const uint64_t items = uint64_t(total_blocks) * 2 * K;
  if (items > 0x7fffffffull) throw ConfigError("level too large for one launch");
  const dim3 grid(static_cast<uint32_t>(items));

  if (!ws.ev0) {
    FSGG_CUDA(cudaEventCreate(&ws.ev0));
    FSGG_CUDA(cudaEventCreate(&ws.ev1));
  }
  unsigned long long* d_perf = d_evals + 1;
  // two-deep rows of small nodes: the whole-node kernel, which also writes the
  // entries' child sums (per_sub implies c == 0, sd == 1; never the root)
  const bool whole_node = lowd && per_sub && Lb == 0 && !groot && node_min + 1 < kNodeMax &&
                          env_u32("FSGG_NODE_KERNEL", 1) != 0;
  uint64_t tc_sym_perf = 0;  // pair evaluations of the symmetric tensor-core root
  FSGG_CUDA(cudaMemsetAsync(d_perf, 0, 8, s));
  FSGG_CUDA(cudaEventRecord(ws.ev0, s));
  const bool sym = Lb > 0 && kde_root_symmetric(ds, ks, lv.qbase, lv.qbase + E, rl, partials,
                                                d_perf, ws.ev0, ws.ev1);
  if (Lb > 0 && !sym) throw NumericError("symmetric root pass rejected its row depth");
  if (lv.level == 0) ws.sym_Lb = sym ? Lb : 0;
  if (sym) {
    // every pair evaluated once (kde_sym.cu)
  } else if (lowd) {
    with_lowd(ks.family, d, [&](auto op) {
      // (per_sub implies c == 0, sd == 1 and nodes below 4 * kSubMinSmall points)
      op.tiled(grid, s, pts, lv, nb, c, sd, t, ks.scale, partials, d_perf, per_sub, whole_node,
               g1, g2);
    });
  } else if (tc) {
    // full build: the symmetric root (each pair once, both row sums)
    if (!kde_tc_root_symmetric(ds, ks, lv, rl, partials, &tc_sym_perf))
      kde_tc_tiled(ds, ks, lv, nb, c, sd, items, partials);
  } else {
    with_family(ks.family, [&](auto fam) {
      constexpr int FAM = decltype(fam)::value;
      kde_xd_tiled_kernel<FAM><<<grid, kXThreads, 0, s>>>(
          pts, d, lv.eq, lv.goff, nb, G, lv.level, c, t.first.as<uint32_t>(),
          t.last.as<uint32_t>(), t.lo.as<float>(), t.hi.as<float>(),
          t.has_boxes, ks.scale, partials);
    });
  }
  FSGG_LAUNCH_CHECK();
  if (!sym) FSGG_CUDA(cudaEventRecord(ws.ev1, s));  // sym: around its tile kernel
  ws.pyr_depth = 0;
  if (rl >= kPyramidMinDepth) {
    ws.pyr_depth = rl;
    ws.pyr.ensure(size_t(E) << rl << 3, s);
    const size_t per_warp = size_t(2) << rl << 3;
    const uint32_t warps = uint32_t(std::max<size_t>(1, std::min<size_t>(8, (96u << 10) / per_warp)));
    FSGG_CUDA(cudaFuncSetAttribute(pyramid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(std::max<size_t>(per_warp * warps, 48u << 10))));
    pyramid_kernel<<<ceil_div_u32(E, warps), warps * 32, per_warp * warps, s>>>(
        partials, rl, lv.eg, E, lv.level, t.first.as<uint32_t>(), t.last.as<uint32_t>(),
        ws.pyr.as<double>(), g1, g2, groot);
  } else if (!whole_node) {
    finalize_kernel<<<ceil_div_u32(E, 256), 256, 0, s>>>(
        partials, 1u << (rl - 1), lv.eg, E, lv.level, t.first.as<uint32_t>(),
        t.last.as<uint32_t>(), g1, g2, groot);
  }
  FSGG_LAUNCH_CHECK();
  ds.launches += 2;
  unsigned long long perf = tc_sym_perf ? tc_sym_perf : ev;
  if (lowd) FSGG_CUDA(cudaMemcpyAsync(&perf, d_perf, 8, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  FSGG_CUDA(cudaEventElapsedTime(&ms, ws.ev0, ws.ev1));
  if (sym) ms += float(ws.sym_prepared_seconds * 1e3);  // tiles run ahead (owner mode)
  stats.tiled_seconds += ms * 1e-3;
  if (sym || (tc && lv.level == 0)) {  // the root launch: the dominant kernel
    stats.root_seconds += ms * 1e-3;
    stats.root_performed += perf;
  }
  stats.tiled_evals += ev;
  stats.tiled_performed += perf;
  stats.performed += perf - ev;  // stats.performed was credited with ev above
  stats.tiled_launches += 1;
}

void kde_range(Dataset& ds, const KernelSpec& ks, uint32_t first,
               uint32_t last, const uint32_t* targets, uint32_t m,
               double* out) {
  if (m == 0) return;
  cudaStream_t s = ds.stream;
  const uint32_t d = ds.d;
  const float* pts = ds.pts.as<float>();
  const uint32_t len = last - first;
  const uint32_t chunk = 8192;
  const uint32_t nchunks = len == 0 ? 1 : (len + chunk - 1) / chunk;
  DevBuf box(size_t(2) * d * 4, s), partials(size_t(m) * nchunks * 8, s);
  float* lo = box.as<float>();
  float* hi = lo + d;
  const bool lowd = d <= kLowDMax;
  if (len > 0) {
    range_box_kernel<<<d, 256, 0, s>>>(pts, d, first, last, lo, hi);
    FSGG_LAUNCH_CHECK();
    ds.launches++;
    if (lowd) {
      const dim3 grid(ceil_div_u32(m, kBE) * nchunks);
      with_lowd(ks.family, d, [&](auto op) {
        op.range(grid, s, pts, targets, m, first, last, chunk, nchunks, lo, hi,
                 ks.scale, partials.as<double>());
      });
    } else {
      with_family(ks.family, [&](auto fam) {
        constexpr int FAM = decltype(fam)::value;
        kde_xd_range_kernel<FAM><<<ceil_div_u32(uint64_t(m) * nchunks * 32, 256), 256, 0, s>>>(
            pts, d, targets, m, first, last, chunk, nchunks, lo, hi,
            d <= kBoxMaxDim, ks.scale, partials.as<double>());
      });
    }
    FSGG_LAUNCH_CHECK();
    ds.launches++;
  }
  range_finalize_kernel<<<ceil_div_u32(m, 256), 256, 0, s>>>(
      partials.as<double>(), len == 0 ? 0 : nchunks, m, len == 0, out);
  FSGG_LAUNCH_CHECK();
  ds.launches++;
}

}  // namespace fsgg
