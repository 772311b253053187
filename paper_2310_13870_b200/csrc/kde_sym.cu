// Symmetric root level: the n^2 pass of the descent evaluates every pair once.
//
// At the root every query is also a source, and k(q, x) = k(x, q): the row
// sums a query needs (its partial row over the root's descendants) and the
// column sums its partner block needs come out of the same evaluations. The
// point set is cut into tree-aligned blocks (nodes at depth Lb, <= 256
// points); for every pair of blocks I <= J that is not prunable (bounding-box
// distance) one CTA evaluates the |I| x |J| tile once and writes
//   * the row sums of I's points over J  -> I's slot for partner J,
//   * the column sums of J's points over I -> J's slot for partner I,
// each as one fp32 value per point (a fixed-order sum of <= 256 terms).
// sym_rows_kernel then folds every point's partner values, in ascending
// partner order, into its fp64 bucket row (buckets = tree nodes at depth rd,
// aligned with the blocks), which is exactly the row format of the tiled
// kernels (kde.cu) — lookups and the pyramid are unchanged.
//
// Pruning per (point, partner block) keeps the tiled kernel's certified rule
// (bound below 2^-kPruneBits of half the root mass, >= 1/2): a pruned
// partner's value is dropped for that point only. Every value depends on the
// two blocks alone, so a shard (a contiguous query range) computes the tiles
// touching its blocks and gets bit-identical rows.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cfloat>
#include <vector>

#include "engine.cuh"
#include "kde_math.cuh"

namespace fsgg {
namespace {

// A tile holds up to 32 * ROWS rows in registers (ROWS per lane, 8 or 10)
// and as many sources (ROWS / 2 warps x 64). Blocks of <= 256 points take
// ROWS = 8, blocks of 257..320 points ROWS = 10 (C4: 302-point blocks at 94%
// lane use, where 256-capacity tiles of its 151-point blocks left 65% of the
// lanes on padding). P rows and records have the 320-value stride.
constexpr uint32_t kSymBlock = kSymStride;  // max points per block (320)
constexpr uint32_t kSymMinBlock = 192;

// rec/remote: in a multi-GPU shard (owner mode) one side of a cross-shard
// tile may belong to another rank; its values then go to exchange record
// `rec` instead of P (remote bit 1: I's rows, bit 2: J's columns).
struct SymTile {
  uint32_t I, J, slotI, slotJ, rec, remote;
};
// Exchange record: [X, Y, first point of X, |X|, 256 values of X's points
// over partner block Y], 32-bit words.
constexpr uint32_t kSymRecWords = kSymRecordWords;  // 4 + kSymStride

__device__ __forceinline__ float block_dist(const float* lo, const float* hi, uint32_t a,
                                            uint32_t b, uint32_t d, int family) {
  float acc = 0.f;
  for (uint32_t k = 0; k < d; ++k) {
    const float g = fmaxf(0.f, fmaxf(lo[size_t(b) * d + k] - hi[size_t(a) * d + k],
                                     lo[size_t(a) * d + k] - hi[size_t(b) * d + k]));
    acc = family == 2 ? acc + g : fmaf(g, g, acc);
  }
  return family == 1 ? sqrtf(acc) : acc;
}

// Block pair (a, b) can contribute to some point of either block.
__device__ __forceinline__ bool pair_active(const float* lo, const float* hi,
                                            const uint32_t* bf, const uint32_t* bl, uint32_t a,
                                            uint32_t b, uint32_t d, int family, float scale,
                                            float bits) {
  const float off = scale * block_dist(lo, hi, a, b, d, family);
  const float na = float(bl[a] - bf[a]), nb = float(bl[b] - bf[b]);
  return off <= __log2f(fmaxf(na, nb)) + bits;
}

__global__ void sym_count_kernel(uint32_t B, const float* __restrict__ lo,
                                 const float* __restrict__ hi, const uint32_t* __restrict__ bf,
                                 const uint32_t* __restrict__ bl, uint32_t d, int family,
                                 float scale, float bits, uint32_t* __restrict__ cnt) {
  __shared__ uint32_t red[8];
  const uint32_t I = blockIdx.x;
  uint32_t c = 0;
  for (uint32_t J = threadIdx.x; J < B; J += blockDim.x)
    c += pair_active(lo, hi, bf, bl, I, J, d, family, scale, bits) ? 1u : 0u;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) t += red[w];
    cnt[I] = t;
  }
}

// Ordered compaction of I's active partners (ascending J).
__global__ void sym_fill_kernel(uint32_t B, const float* __restrict__ lo,
                                const float* __restrict__ hi, const uint32_t* __restrict__ bf,
                                const uint32_t* __restrict__ bl, uint32_t d, int family,
                                float scale, float bits, const uint32_t* __restrict__ poff,
                                uint32_t* __restrict__ plist) {
  __shared__ uint32_t wsum[8];
  __shared__ uint32_t base;
  const uint32_t I = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) base = poff[I];
  __syncthreads();
  for (uint32_t J0 = 0; J0 < B; J0 += blockDim.x) {
    const uint32_t J = J0 + threadIdx.x;
    const bool a = J < B && pair_active(lo, hi, bf, bl, I, J, d, family, scale, bits);
    const unsigned m = __ballot_sync(0xffffffffu, a);
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (uint32_t k = 0; k < blockDim.x / 32; ++k) {
      if (k < w) before += wsum[k];
      total += wsum[k];
    }
    if (a) plist[base + before + __popc(m & ((1u << lane) - 1u))] = J;
    __syncthreads();
    if (threadIdx.x == 0) base += total;
    __syncthreads();
  }
}

// Spatial order inside each block, for batch pruning in the tile kernel.
// The blocks are the reference's index-order tree nodes (sampler.cpp:138-141):
// on C3 a block is a ~0.28 x 0.28 blob of noise around a short arc, so whole
// block pairs within the pruning radius still hold many pairs far beyond it.
// Each block's points are ordered by recursive splits — windows of 512, 256,
// ..., 16 positions, each sorted along its widest box side — so every aligned
// batch of kSymBatch positions is a small cluster with its own box (bbox).
// A tile skips a source batch whose box is beyond the pruning radius of the
// row block's box. Only the visiting order changes: sums are order-free up to
// fp32 rounding, and results go back to the points' own positions (perm).
constexpr uint32_t kSymBatch = 8;
constexpr uint32_t kSymBatches = kSymBlock / kSymBatch;  // 40
constexpr uint32_t kSymPermP = 512;                      // pow2 >= kSymBlock

__global__ void __launch_bounds__(256)
    sym_perm_kernel(const float* __restrict__ pts, uint32_t d, const uint32_t* __restrict__ bf,
                    const uint32_t* __restrict__ bl, float* __restrict__ ppts,
                    uint32_t* __restrict__ perm, float* __restrict__ bbox) {
  // key: window (6 bits) | orderable coordinate (32) | local index (9)
  __shared__ unsigned long long key[kSymPermP];
  __shared__ uint32_t wdim[kSymPermP / 16];
  const uint32_t I = blockIdx.x, f = bf[I], n = bl[I] - f;
  const uint32_t lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  uint32_t P = 16;
  while (P < n) P <<= 1;
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) key[i] = i;
  __syncthreads();
  for (uint32_t W = P; W >= 16; W >>= 1) {
    const uint32_t nw = P / W;
    for (uint32_t w = threadIdx.x >> 5; w < nw; w += nwarps) {
      float lo[kBoxMaxDim], hi[kBoxMaxDim];
      for (uint32_t k = 0; k < d; ++k) {
        lo[k] = FLT_MAX;
        hi[k] = -FLT_MAX;
      }
      for (uint32_t pos = w * W + lane; pos < w * W + W; pos += 32) {
        const uint32_t i = uint32_t(key[pos] & 511u);
        if (i < n)
          for (uint32_t k = 0; k < d; ++k) {
            const float c = pts[size_t(f + i) * d + k];
            lo[k] = fminf(lo[k], c);
            hi[k] = fmaxf(hi[k], c);
          }
      }
      uint32_t best = 0;
      float ext = -1.f;
      for (uint32_t k = 0; k < d; ++k) {
        for (int o = 16; o; o >>= 1) {
          lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
          hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
        if (hi[k] - lo[k] > ext) {
          ext = hi[k] - lo[k];
          best = k;
        }
      }
      if (lane == 0) wdim[w] = best;
    }
    __syncthreads();
    for (uint32_t pos = threadIdx.x; pos < P; pos += blockDim.x) {
      const uint32_t i = uint32_t(key[pos] & 511u), w = pos / W;
      uint32_t u = 0xffffffffu;  // absent positions sort last in their window
      if (i < n) {
        u = __float_as_uint(pts[size_t(f + i) * d + wdim[w]]);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
      }
      key[pos] = (static_cast<unsigned long long>(w) << 41) |
                 (static_cast<unsigned long long>(u) << 9) | i;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1)
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t t = threadIdx.x; t < P / 2; t += blockDim.x) {
          const uint32_t a = 2 * t - (t & (j - 1)), b = a + j;
          const unsigned long long x = key[a], y = key[b];
          if ((x > y) == ((a & k) == 0)) {
            key[a] = y;
            key[b] = x;
          }
        }
        __syncthreads();
      }
  }
  for (uint32_t pos = threadIdx.x; pos < n; pos += blockDim.x) {
    const uint32_t i = uint32_t(key[pos] & 511u);
    perm[f + pos] = i;
    for (uint32_t k = 0; k < d; ++k) ppts[size_t(f + pos) * d + k] = pts[size_t(f + i) * d + k];
  }
  for (uint32_t b = threadIdx.x; b * kSymBatch < n; b += blockDim.x) {
    float* out = bbox + (size_t(I) * kSymBatches + b) * 2 * d;
    for (uint32_t k = 0; k < d; ++k) {
      float lo = FLT_MAX, hi = -FLT_MAX;
      for (uint32_t pos = b * kSymBatch; pos < min(n, (b + 1) * kSymBatch); ++pos) {
        const float c = pts[size_t(f + uint32_t(key[pos] & 511u)) * d + k];
        lo = fminf(lo, c);
        hi = fmaxf(hi, c);
      }
      out[k] = lo;
      out[d + k] = hi;
    }
  }
}

// Tiles (I <= J) that touch the query blocks [b0, b1].
// Owner mode (multi-GPU, shard bounds on block boundaries): every tile is
// computed by exactly one rank — a tile inside the shard by it, a cross tile
// (I, J) by the owner of I when I + J is even, else by the owner of J — and
// the other rank's side travels as an exchange record.
__global__ void __launch_bounds__(128)
    sym_tiles_kernel(uint32_t B, const uint32_t* __restrict__ poff,
                     const uint32_t* __restrict__ plist, uint32_t b0, uint32_t b1,
                     const uint32_t* __restrict__ bf, const uint32_t* __restrict__ bl,
                     SymTile* __restrict__ tiles, uint32_t* __restrict__ ntiles,
                     unsigned long long* __restrict__ performed, int own,
                     uint32_t* __restrict__ nrec, uint32_t* __restrict__ records,
                     SymTile* __restrict__ xtiles) {
  __shared__ unsigned long long red[4];
  __shared__ uint32_t wcnt[4], cbase;
  const uint32_t I = blockIdx.x;
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long ev = 0;  // evaluations of this row's tiles
  for (uint32_t k0 = poff[I]; k0 < poff[I + 1]; k0 += blockDim.x) {
    const uint32_t k = k0 + threadIdx.x;
    const uint32_t J = k < poff[I + 1] ? plist[k] : 0u;
    const bool mineI = I >= b0 && I <= b1, mineJ = J >= b0 && J <= b1;
    const bool take_any = k < poff[I + 1] && J >= I &&
                          (own ? (mineI && mineJ) || (mineI && ((I + J) & 1u) == 0u) ||
                                     (mineJ && ((I + J) & 1u) == 1u)
                               : mineI || mineJ);
    // owner mode: cross-shard tiles go to their own list (record = index)
    const bool cross = take_any && own && !(mineI && mineJ);
    const bool take = take_any && !cross;
    // one reservation per CTA chunk (a per-tile atomic on one counter
    // serialises ~1.7M times at C3)
    const unsigned m = __ballot_sync(0xffffffffu, take);
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int q = 0; q < 4; ++q) {
        const uint32_t c = wcnt[q];
        wcnt[q] = t;
        t += c;
      }
      cbase = t ? atomicAdd(ntiles, t) : 0u;
    }
    __syncthreads();
    if (take_any) {
      ev += (unsigned long long)(bl[I] - bf[I]) * (bl[J] - bf[J]);
      // position of I in J's (ascending) partner list
      uint32_t lo = poff[J], hi = poff[J + 1];
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (plist[mid] < I)
          lo = mid + 1;
        else
          hi = mid;
      }
      if (cross) {  // the other block's values are exported as record `rec`
        const uint32_t remote = mineI ? 2u : 1u;
        const uint32_t rec = atomicAdd(nrec, 1u);
        const uint32_t X = mineI ? J : I, Y = mineI ? I : J;
        uint32_t* hdr = records + size_t(rec) * kSymRecWords;
        hdr[0] = X;
        hdr[1] = Y;
        hdr[2] = bf[X];
        hdr[3] = bl[X] - bf[X];
        xtiles[rec] = SymTile{I, J, k - poff[I], lo - poff[J], rec, remote};
      } else {
        tiles[cbase + wcnt[w] + __popc(m & ((1u << lane) - 1u))] =
            SymTile{I, J, k - poff[I], lo - poff[J], 0u, 0u};
      }
    }
    __syncthreads();
  }
  for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
  if (lane == 0) red[w] = ev;
  __syncthreads();
  if (threadIdx.x == 0 && performed) {
    const unsigned long long t = red[0] + red[1] + red[2] + red[3];
    if (t) atomicAdd(performed, t);
  }
}

// Expanded-form distances for the gaussian at d >= FSGG_SYM_EXP_MIN_D:
// |q - x|^2 = |q|^2 + |x|^2 - 2 q.x with the tile-relative scaled
// coordinates, so a pair costs d + 1 packed FMA-pipe operations instead of
// 2d (d FADD2 + d FMUL2/FFMA2) — the FMA pipe, not MUFU, bound the d = 5
// tile (ncu: FMA-pipe cycles 74%, XU 47%). The cancellation error is
// ~eps_f32 * (|q'|^2 + |x'|^2) in the exponent, |q'|, |x'| measured from the
// midpoint of the two blocks' boxes (the pair's own scale for the near
// pairs that carry the sums), far below the tie guard's 1e-4 margin.
// Per tile, and only when its scaled coordinates are small: max |q'|^2 +
// max |x'|^2 <= kSymExpMaxNorm over the tile's points (the error is ~7e-8 x
// that bound, relative, per term); wide blocks (sparse data, small sigma)
// keep the direct form. The choice depends on the two blocks alone
// (shard-safe).
#ifndef FSGG_SYM_EXP_MIN_D
#define FSGG_SYM_EXP_MIN_D 3
#endif
#ifndef FSGG_SYM_R10_CTAS
#define FSGG_SYM_R10_CTAS 4
#endif
#ifndef FSGG_SYM_EXP_MAX
#define FSGG_SYM_EXP_MAX 64.f
#endif
constexpr float kSymExpMaxNorm = FSGG_SYM_EXP_MAX;
// Factored form (warp-per-tile kernel, gaussian, FSGG_SYM_FACT_MIN_D <= d <=
// FSGG_SYM_FACT_MAX_D): 2^-|q' - x'|^2 = 2^-|q'|^2 * 2^-(|x'|^2 - 2 q'.x').
// The row factor leaves the row sum (one multiply per row per tile) and
// enters the column sum as the multiplicand of the accumulating FFMA2, so a
// pair costs d packed FMA-pipe operations for the exponent + 2 for the two
// sums (the expanded form: d + 3). Same tile-relative origin, same per-tile
// norm bound (on the tile's actual points) and the same error scale as the
// expanded form above (~eps_f32 * (|q'|^2 + |x'|^2) in the exponent, <= 64:
// ~5e-6 relative at worst, far inside the tie guard's 1e-4). C4 (d = 5):
// root 4.56 -> 4.39 ms.
// d <= 2 can take it too (FSGG_SYM_FACT_MIN_D = 1: 4 packed operations per
// pair instead of the direct form's 6, the tile's form decided from the two
// boxes' farthest corners, bound kSymFactMaxNorm, with no pass over the
// points) but measured no faster (21.7 vs 21.3 ms at C3 with FMA-pipe cycles
// down from 67% to 55%): that kernel is bound by the MIO queue MUFU shares
// with LDS and SHFL, not by the FMA pipe, so d <= 2 keeps the more accurate
// direct form.
#ifndef FSGG_SYM_FACT_MIN_D
#define FSGG_SYM_FACT_MIN_D 3
#endif
#ifndef FSGG_SYM_FACT_MAX_D
#define FSGG_SYM_FACT_MAX_D 6
#endif
#ifndef FSGG_SYM_FACT_MAX
#define FSGG_SYM_FACT_MAX 160.f
#endif
constexpr float kSymFactMaxNorm = FSGG_SYM_FACT_MAX;

template <int D, int FAM, int ROWS, bool OWN>
__device__ __forceinline__ void sym_tile_body(
    const float* __restrict__ pts, float cs, const SymTile* __restrict__ tiles,
    const uint32_t* __restrict__ bf, const uint32_t* __restrict__ bl,
    const float* __restrict__ lo, const float* __restrict__ hi, float scale, float bits,
    const uint32_t* __restrict__ poff, float* __restrict__ P,
    unsigned long long* __restrict__ performed, float* __restrict__ records,
    const float* __restrict__ ppts, const uint32_t* __restrict__ perm,
    const float* __restrict__ bbox) {
  constexpr int kSymRows = ROWS;
  constexpr int kSymWarps = ROWS / 2;
  constexpr uint32_t kCap = 32u * ROWS;
  constexpr bool EXP_OK = FAM == 0 && D >= FSGG_SYM_EXP_MIN_D;
  constexpr int SW = EXP_OK ? D + 1 : D;  // float2 per source in shared memory
  __shared__ __align__(16) float2 sx[kCap * SW];
  __shared__ float rowred[kSymWarps][kCap];
  __shared__ float colv[kCap];
  const SymTile tl = tiles[blockIdx.x];
  const uint32_t fi = bf[tl.I], ni = bl[tl.I] - fi;
  const uint32_t fj = bf[tl.J], nj = bl[tl.J] - fj;
  // Coordinates relative to I's first point, scaled by cs (sqrt(scale) for
  // the gaussian, scale otherwise): the exponent of a pair is then -dist'
  // itself (MUFU takes the negation for free) — one packed multiply per pair
  // less on the FMA pipe, which shares the binding with the XU pipe. The
  // local origin keeps the scaled values small (pre-scaling absolute
  // coordinates lost accuracy for data far from the origin).
  // (expanded form: origin midway between the two blocks' box centres, which
  // keeps |q'|^2 + |x'|^2 — the scale of its cancellation error — near the
  // pair distances themselves)
  float c0[D];
  if constexpr (EXP_OK) {
#pragma unroll
    for (int k = 0; k < D; ++k)
      c0[k] = 0.25f * ((__ldg(lo + size_t(tl.I) * D + k) + __ldg(hi + size_t(tl.I) * D + k)) +
                       (__ldg(lo + size_t(tl.J) * D + k) + __ldg(hi + size_t(tl.J) * D + k)));
  } else {
#pragma unroll
    for (int k = 0; k < D; ++k) c0[k] = __ldg(pts + size_t(fi) * D + k);
  }
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // sources of J; slots past nj sit far away (their terms underflow to 0),
  // so the unrolled source loop needs no guard.
  // Direct form: -x' duplicated. Expanded-capable kernels store -2 x'
  // (the direct form takes -x' = 0.5 * (-2 x') exactly through one FFMA2)
  // and |x'|^2 (absent: x' = 1e18, |x'|^2 = 1e30); the largest norms of the
  // two blocks, gathered on the way, decide the form.
  __shared__ float s_max[2][kCap / 32];
  float mi = 0.f, mj = 0.f;
  if constexpr (EXP_OK) {
    for (uint32_t j = threadIdx.x; j < kCap; j += blockDim.x) {
      float nrm = 1e30f;
      float xv[D];
#pragma unroll
      for (int k = 0; k < D; ++k) xv[k] = 1e18f;
      if (j < nj) {
        nrm = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          xv[k] = (__ldg(ppts + size_t(fj + j) * D + k) - c0[k]) * cs;
          nrm = fmaf(xv[k], xv[k], nrm);
        }
        mj = fmaxf(mj, nrm);
      }
#pragma unroll
      for (int k = 0; k < D; ++k) sx[j * SW + k] = make_float2(-2.f * xv[k], -2.f * xv[k]);
      sx[j * SW + D] = make_float2(nrm, nrm);
    }
  } else {
    for (uint32_t idx = threadIdx.x; idx < kCap * D; idx += blockDim.x) {
      const float v =
          idx < nj * D ? -((__ldg(ppts + size_t(fj) * D + idx) - c0[idx % D]) * cs) : -1e18f;
      sx[idx] = make_float2(v, v);
    }
  }
  // this lane's rows (points of I) as packed pairs; absent rows far away
  float2 q2[kSymRows / 2][D];
  float2 qn[EXP_OK ? kSymRows / 2 : 1];  // expanded form: |q'|^2 of each row pair
#pragma unroll
  for (int p = 0; p < kSymRows / 2; ++p) {
    const uint32_t r0 = lane * kSymRows + 2 * p, r1 = r0 + 1;
    float na = 0.f, nb = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const float a = r0 < ni ? (__ldg(pts + size_t(fi + r0) * D + k) - c0[k]) * cs : 1e18f;
      const float b = r1 < ni ? (__ldg(pts + size_t(fi + r1) * D + k) - c0[k]) * cs : 1e18f;
      q2[p][k] = make_float2(a, b);
      na = fmaf(a, a, na);
      nb = fmaf(b, b, nb);
    }
    if constexpr (EXP_OK) {
      qn[p] = make_float2(r0 < ni ? na : 1e30f, r1 < ni ? nb : 1e30f);
      if (r0 < ni) mi = fmaxf(mi, na);
      if (r1 < ni) mi = fmaxf(mi, nb);
    }
  }
  if constexpr (EXP_OK) {
    for (int o = 16; o; o >>= 1) {
      mi = fmaxf(mi, __shfl_xor_sync(0xffffffffu, mi, o));
      mj = fmaxf(mj, __shfl_xor_sync(0xffffffffu, mj, o));
    }
    if (lane == 0) {
      s_max[0][w] = mi;
      s_max[1][w] = mj;
    }
  }
  // source batches of J beyond the pruning radius of I's box: a row of I
  // loses < nj 2^-thr <= 2^-bits over all of J's skipped batches and a
  // source of J < ni 2^-thr, the same bound as a pruned block pair
  __shared__ uint32_t s_skip[2];
  if (threadIdx.x < 64) {
    const uint32_t b = threadIdx.x;
    bool sk = false;
    if (tl.I != tl.J && b * kSymBatch < nj) {
      const float* bx = bbox + (size_t(tl.J) * kSymBatches + b) * 2 * D;
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float g = fmaxf(0.f, fmaxf(__ldg(bx + k) - __ldg(hi + size_t(tl.I) * D + k),
                                         __ldg(lo + size_t(tl.I) * D + k) - __ldg(bx + D + k)));
        acc = FAM == 2 ? acc + g : fmaf(g, g, acc);
      }
      sk = scale * fam_finish1<FAM>(acc) > bits + __log2f(float(max(ni, nj)));
    }
    const unsigned m = __ballot_sync(0xffffffffu, sk);
    if (lane == 0) s_skip[w] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0 && performed) {  // pair evaluations this tile executes
    uint32_t kept = nj;
    for (uint32_t b = 0; b * kSymBatch < nj; ++b)
      if ((s_skip[b >> 5] >> (b & 31)) & 1u) kept -= min(kSymBatch, nj - b * kSymBatch);
    if (kept) atomicAdd(performed, (unsigned long long)ni * kept);
  }
  bool use_exp = false;
  if constexpr (EXP_OK) {
    mi = mj = 0.f;
#pragma unroll
    for (int k = 0; k < kSymWarps; ++k) {
      mi = fmaxf(mi, s_max[0][k]);
      mj = fmaxf(mj, s_max[1][k]);
    }
    use_exp = mi + mj <= kSymExpMaxNorm;
  }
  float2 racc[kSymRows / 2];
#pragma unroll
  for (int p = 0; p < kSymRows / 2; ++p) racc[p] = make_float2(0.f, 0.f);
  // warp w: batches of 8 sources (w, w + warps, ...): 8 column partials
  // per lane (not 32) keep the kernel at 62 registers, 8 CTAs per SM — the
  // extra shuffles cost less than the occupancy buys (32: 30.0 ms, 16: 29.6,
  // 8: 28.9, 4: 30.1 on C3)
  auto tile_loop = [&](auto exp_tag) {
  constexpr bool EXP = decltype(exp_tag)::value;
  // batches dealt round-robin: skipped batches cluster in the spatial order,
  // so contiguous ranges would leave some warps idle while others work
  for (uint32_t jb = w * 8; jb < nj; jb += 8 * kSymWarps) {
    if ((s_skip[jb >> 8] >> ((jb >> 3) & 31)) & 1u) {
      if (lane < 8 && jb + lane < nj) colv[jb + lane] = 0.f;
      continue;
    }
    float c[8];  // this lane's 8-row partial of each source's column sum
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      const float2* x = sx + (jb + jj) * SW;
      float2 es = make_float2(0.f, 0.f);
#pragma unroll
      for (int p = 0; p < kSymRows / 2; ++p) {
        float2 t;
        if constexpr (EXP) {
          t = __fadd2_rn(qn[p], x[D]);
#pragma unroll
          for (int k = 0; k < D; ++k) t = __ffma2_rn(q2[p][k], x[k], t);
        } else if constexpr (EXP_OK) {  // -x' = 0.5 * (-2 x'), exactly
          const float2 h = make_float2(0.5f, 0.5f);
          t = fam_first<FAM>(__ffma2_rn(h, x[0], q2[p][0]));
#pragma unroll
          for (int k = 1; k < D; ++k) t = fam_next<FAM>(__ffma2_rn(h, x[k], q2[p][k]), t);
          t = fam_finish<FAM>(t);
        } else {
          t = fam_first<FAM>(__fadd2_rn(q2[p][0], x[0]));
#pragma unroll
          for (int k = 1; k < D; ++k) t = fam_next<FAM>(__fadd2_rn(q2[p][k], x[k]), t);
          t = fam_finish<FAM>(t);
        }
        const float2 e = make_float2(ex2_approx(-t.x), ex2_approx(-t.y));
        racc[p] = __fadd2_rn(racc[p], e);
        es = p == 0 ? e : __fadd2_rn(es, e);
      }
      c[jj] = es.x + es.y;
    }
    // fold lanes l ^ 16 and l ^ 8, then a butterfly transpose-reduction over
    // 8 lanes: afterwards lane l holds the column sum of source jb + (l & 7)
    // over all 32 lanes (23 shuffles for 8 sources)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] += __shfl_xor_sync(0xffffffffu, c[i], 16);
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] += __shfl_xor_sync(0xffffffffu, c[i], 8);
#pragma unroll
    for (int st = 4; st >= 1; st >>= 1) {
      const bool up = (lane & st) != 0;
#pragma unroll
      for (int i = 0; i < st; ++i) {
        const float keep = up ? c[i + st] : c[i];
        const float send = up ? c[i] : c[i + st];
        c[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
      }
    }
    if (lane < 8 && jb + lane < nj) colv[jb + lane] = c[0];
  }
  };
  if constexpr (EXP_OK) {
    if (use_exp)
      tile_loop(std::true_type{});
    else
      tile_loop(std::false_type{});
  } else {
    tile_loop(std::false_type{});
  }
#pragma unroll
  for (int p = 0; p < kSymRows / 2; ++p) {
    rowred[w][lane * kSymRows + 2 * p] = racc[p].x;
    rowred[w][lane * kSymRows + 2 * p + 1] = racc[p].y;
  }
  __syncthreads();
  // destinations: this shard's P slots, or an exchange record (owner mode;
  // a separate instantiation: the single-GPU kernel keeps its 80 registers)
  float* rdst = P + (size_t(poff[tl.I]) + tl.slotI) * kCap;
  float* cdst = P + (size_t(poff[tl.J]) + tl.slotJ) * kCap;
  if constexpr (OWN) {
    if (tl.remote & 1u) rdst = records + size_t(tl.rec) * kSymRecWords + 4;
    if (tl.remote & 2u) cdst = records + size_t(tl.rec) * kSymRecWords + 4;
  }
  // rows of I over J, columns of J over I (the diagonal tile has rows only);
  // a point that prunes the partner block drops its value
  for (uint32_t t = threadIdx.x; t < ni; t += blockDim.x) {
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < kSymWarps; ++k) v += rowred[k][t];
    float q[D];
#pragma unroll
    for (int k = 0; k < D; ++k) q[k] = __ldg(pts + size_t(fi + t) * D + k);
    const float off = scale * box_dist<FAM>(q, lo + size_t(tl.J) * D, hi + size_t(tl.J) * D, D);
    if (off > __log2f(float(nj)) + bits) v = 0.f;
    rdst[t] = v;
  }
  if (tl.I != tl.J) {
    for (uint32_t t = threadIdx.x; t < nj; t += blockDim.x) {
      float v = colv[t];
      float x[D];
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = __ldg(ppts + size_t(fj + t) * D + k);
      const float off = scale * box_dist<FAM>(x, lo + size_t(tl.I) * D, hi + size_t(tl.I) * D, D);
      if (off > __log2f(float(ni)) + bits) v = 0.f;
      cdst[__ldg(perm + fj + t)] = v;
    }
  }
}

// The kernel for a shard's own tiles (80 registers at d = 2, 6 CTAs per SM)
// and the one for owner-mode cross-shard tiles (one side exported).
template <int D, int FAM, int ROWS>
__global__ void __launch_bounds__(ROWS * 16, ROWS == 10 ? FSGG_SYM_R10_CTAS : 0)
    sym_tile_kernel(const float* __restrict__ pts, float cs,
                    const SymTile* __restrict__ tiles,
                    const uint32_t* __restrict__ bf, const uint32_t* __restrict__ bl,
                    const float* __restrict__ lo, const float* __restrict__ hi, float scale,
                    float bits, const uint32_t* __restrict__ poff, float* __restrict__ P,
                    unsigned long long* __restrict__ performed, float* __restrict__ records,
                    const float* __restrict__ ppts, const uint32_t* __restrict__ perm,
                    const float* __restrict__ bbox) {
  sym_tile_body<D, FAM, ROWS, false>(pts, cs, tiles, bf, bl, lo, hi, scale, bits, poff, P,
                                     performed, records, ppts, perm, bbox);
}
template <int D, int FAM, int ROWS>
__global__ void __launch_bounds__(ROWS * 16, ROWS == 10 ? FSGG_SYM_R10_CTAS : 0)
    sym_tile_own_kernel(const float* __restrict__ pts, float cs,
                        const SymTile* __restrict__ tiles,
                        const uint32_t* __restrict__ bf, const uint32_t* __restrict__ bl,
                        const float* __restrict__ lo, const float* __restrict__ hi,
                        float scale, float bits, const uint32_t* __restrict__ poff,
                        float* __restrict__ P, unsigned long long* __restrict__ performed,
                        float* __restrict__ records, const float* __restrict__ ppts,
                        const uint32_t* __restrict__ perm, const float* __restrict__ bbox) {
  sym_tile_body<D, FAM, ROWS, true>(pts, cs, tiles, bf, bl, lo, hi, scale, bits, poff, P,
                                    performed, records, ppts, perm, bbox);
}

// Warp-per-tile variant for d <= 2 (C2/C3: the headline path). One warp
// evaluates a whole tile on its own — its 32 lanes hold all 32 * ROWS rows of
// I, the sources of J sit in the warp's private shared-memory slice — so a
// tile needs no CTA barrier and no cross-warp row reduction, and the warps
// of an SM run at 32 independent phases instead of 8 lock-stepped groups of
// 4 (the CTA-per-tile kernel lost ~1 issue slot in 12 to barrier stalls once
// batch pruning made its warps' shares uneven: XU 83% -> 72%). Warps are
// persistent and take tiles in list order from a device counter, so a warp
// that drew heavily pruned tiles simply takes more of them. A row's value is
// the fp32 sum over J's kept batches in batch order; it depends on the two
// blocks alone (deterministic, shard-safe).
constexpr int kWtWarps = 4;

// Sources of J staged per warp: all of them for d <= 2, else stages of
// kWtStage<..> sources (<= 8 KiB of shared memory per warp) — the warp fills
// its own slice, so staging costs nothing but the loop.
template <int SW, uint32_t CAP, uint32_t BYTES = 8192u>
constexpr uint32_t wt_stage() {
  const uint32_t fit = (BYTES / (SW * 4u)) & ~7u;
  return fit < CAP ? fit : CAP;
}

template <int D, int FAM, int ROWS, bool OWN>
__device__ __forceinline__ void sym_wtile_body(
    const float* __restrict__ pts, float cs, const SymTile* __restrict__ tiles,
    uint32_t ntiles, uint32_t* __restrict__ next, const uint32_t* __restrict__ bf,
    const uint32_t* __restrict__ bl, const float* __restrict__ lo,
    const float* __restrict__ hi, float scale, float bits,
    const uint32_t* __restrict__ poff, float* __restrict__ P,
    unsigned long long* __restrict__ performed, float* __restrict__ records,
    const float* __restrict__ ppts, const uint32_t* __restrict__ perm,
    const float* __restrict__ bbox) {
  constexpr uint32_t kCap = 32u * ROWS;
  constexpr bool FACT =
      FAM == 0 && D >= FSGG_SYM_FACT_MIN_D && D <= FSGG_SYM_FACT_MAX_D;  // factored form
  constexpr bool EXP_OK = FACT || (FAM == 0 && D >= FSGG_SYM_EXP_MIN_D);
  // Words per source in shared memory, padded to an even count so that a
  // pair of sources is a whole number of 16-byte loads. Each word is stored
  // once: the packed operations take it as a broadcast scalar operand
  // (FADD2 R, R.F32x2, R.F32), so no duplicated (v, v) pairs are staged —
  // shared-memory loads share the MIO queue with MUFU, the binding pipe.
  constexpr int SW = ((EXP_OK ? D + 1 : D) + 1) & ~1;
  // d <= 2 holds 8 CTAs per SM: 4 KiB of sources per warp (two stages per tile
  // in the factored form's 3-word format)
  constexpr uint32_t SC = wt_stage<SW, kCap, (D <= 2 ? 4096u : 8192u)>();
  static_assert(SC * SW >= kCap, "the stage buffer doubles as the row buffer");
  __shared__ __align__(16) float sx_all[kWtWarps][SC * SW];
  __shared__ float colv_all[kWtWarps][kCap];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* sx = sx_all[w];
  float* colv = colv_all[w];
  float* rowv = sx;  // reused after the tile loop
  unsigned long long ev = 0;                   // pair evaluations of this warp's tiles
  for (;;) {
    uint32_t ti = 0;
    if (lane == 0) ti = atomicAdd(next, 1u);
    ti = __shfl_sync(0xffffffffu, ti, 0);
    if (ti >= ntiles) break;
    const SymTile tl = tiles[ti];
    const uint32_t fi = __ldg(bf + tl.I), ni = __ldg(bl + tl.I) - fi;
    const uint32_t fj = __ldg(bf + tl.J), nj = __ldg(bl + tl.J) - fj;
    // coordinates relative to I's first point (expanded form: the midpoint of
    // the two blocks' box centres), pre-scaled (see sym_tile_body)
    float c0[D];
    if constexpr (EXP_OK) {
#pragma unroll
      for (int k = 0; k < D; ++k)
        c0[k] = 0.25f * ((__ldg(lo + size_t(tl.I) * D + k) + __ldg(hi + size_t(tl.I) * D + k)) +
                         (__ldg(lo + size_t(tl.J) * D + k) + __ldg(hi + size_t(tl.J) * D + k)));
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) c0[k] = __ldg(pts + size_t(fi) * D + k);
    }
    float2 q2[ROWS / 2][D];
    // expanded form: |q'|^2 of each row pair; factored form: the rows'
    // factors 2^-|q'|^2 (direct tiles: 1), 0 for an absent row
    float2 qn[EXP_OK ? ROWS / 2 : 1];
    float mi = 0.f, mj = 0.f;
    // an absent row sits far away; in the factored form at the origin with
    // factor 0 (its exponent must stay finite)
    constexpr float kAbsent = FACT ? 0.f : 1e18f;
#pragma unroll
    for (int p = 0; p < ROWS / 2; ++p) {
      const uint32_t r0 = lane * ROWS + 2 * p, r1 = r0 + 1;
      float na = 0.f, nb = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float a = r0 < ni ? (__ldg(pts + size_t(fi + r0) * D + k) - c0[k]) * cs : kAbsent;
        const float b = r1 < ni ? (__ldg(pts + size_t(fi + r1) * D + k) - c0[k]) * cs : kAbsent;
        q2[p][k] = make_float2(a, b);
        na = fmaf(a, a, na);
        nb = fmaf(b, b, nb);
      }
      if constexpr (EXP_OK) {
        qn[p] = make_float2(r0 < ni ? na : 1e30f, r1 < ni ? nb : 1e30f);
        if (r0 < ni) mi = fmaxf(mi, na);
        if (r1 < ni) mi = fmaxf(mi, nb);
      }
    }
    bool use_exp = false;
    if constexpr (FACT && D <= 2) {
      // the form is the tile's: the scaled norms of its two boxes' farthest
      // corners from the origin (no pass over the points)
      float bi = 0.f, bj = 0.f;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const float li = __ldg(lo + size_t(tl.I) * D + k), hi_ = __ldg(hi + size_t(tl.I) * D + k);
        const float lj = __ldg(lo + size_t(tl.J) * D + k), hj = __ldg(hi + size_t(tl.J) * D + k);
        const float ai = fmaxf(fabsf(li - c0[k]), fabsf(hi_ - c0[k])) * cs;
        const float aj = fmaxf(fabsf(lj - c0[k]), fabsf(hj - c0[k])) * cs;
        bi = fmaf(ai, ai, bi);
        bj = fmaf(aj, aj, bj);
      }
      use_exp = bi + bj <= kSymFactMaxNorm;
#pragma unroll
      for (int p = 0; p < ROWS / 2; ++p) {
        const uint32_t r0 = lane * ROWS + 2 * p, r1 = r0 + 1;
        qn[p] = make_float2(r0 < ni ? (use_exp ? ex2_approx(-qn[p].x) : 1.f) : 0.f,
                            r1 < ni ? (use_exp ? ex2_approx(-qn[p].y) : 1.f) : 0.f);
      }
    } else if constexpr (EXP_OK) {
      // the form is the tile's: largest scaled norms of its two blocks
      for (uint32_t j = lane; j < nj; j += 32) {
        float nrm = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float xv = (__ldg(ppts + size_t(fj + j) * D + k) - c0[k]) * cs;
          nrm = fmaf(xv, xv, nrm);
        }
        mj = fmaxf(mj, nrm);
      }
      for (int o = 16; o; o >>= 1) {
        mi = fmaxf(mi, __shfl_xor_sync(0xffffffffu, mi, o));
        mj = fmaxf(mj, __shfl_xor_sync(0xffffffffu, mj, o));
      }
      use_exp = mi + mj <= kSymExpMaxNorm;
      if constexpr (FACT) {
#pragma unroll
        for (int p = 0; p < ROWS / 2; ++p) {
          const uint32_t r0 = lane * ROWS + 2 * p, r1 = r0 + 1;
          qn[p] = make_float2(r0 < ni ? (use_exp ? ex2_approx(-qn[p].x) : 1.f) : 0.f,
                              r1 < ni ? (use_exp ? ex2_approx(-qn[p].y) : 1.f) : 0.f);
        }
      }
    }
    // source batches of J beyond the pruning radius of I's box (sym_tile_body)
    uint32_t skip[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t b = lane + 32u * h;
      bool sk = false;
      if (tl.I != tl.J && b * kSymBatch < nj) {
        const float* bx = bbox + (size_t(tl.J) * kSymBatches + b) * 2 * D;
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < D; ++k) {
          const float g = fmaxf(0.f, fmaxf(__ldg(bx + k) - __ldg(hi + size_t(tl.I) * D + k),
                                           __ldg(lo + size_t(tl.I) * D + k) - __ldg(bx + D + k)));
          acc = FAM == 2 ? acc + g : fmaf(g, g, acc);
        }
        sk = scale * fam_finish1<FAM>(acc) > bits + __log2f(float(max(ni, nj)));
      }
      skip[h] = __ballot_sync(0xffffffffu, sk);
    }
    {
      const uint32_t lb = (nj - 1u) >> 3;  // the last batch may be partial
      uint32_t dropped = 8u * (__popc(skip[0]) + __popc(skip[1]));
      if ((skip[lb >> 5] >> (lb & 31)) & 1u) dropped -= 8u * (lb + 1u) - nj;
      ev += (unsigned long long)ni * (nj - dropped);
    }
    float2 racc[ROWS / 2];
#pragma unroll
    for (int p = 0; p < ROWS / 2; ++p) racc[p] = make_float2(0.f, 0.f);
    auto stage_loop = [&](auto exp_tag, uint32_t s0, uint32_t s1) {
      constexpr bool EXP = decltype(exp_tag)::value;
      for (uint32_t jb = s0; jb < s1; jb += 8) {
        if ((skip[jb >> 8] >> ((jb >> 3) & 31)) & 1u) {
          if (lane < 8 && jb + lane < nj) colv[jb + lane] = 0.f;
          continue;
        }
        float c[8];  // this lane's ROWS-row partial of each source's column sum
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          // the words of sources jj and jj ^ 1 come in together (16-byte
          // loads; the unrolled loop keeps one copy per pair)
          float xw[2 * SW];
          {
            const float4* src = reinterpret_cast<const float4*>(sx + (jb - s0 + (jj & ~1)) * SW);
#pragma unroll
            for (int v4 = 0; v4 < SW / 2; ++v4) {
              const float4 v = src[v4];
              xw[4 * v4] = v.x;
              xw[4 * v4 + 1] = v.y;
              xw[4 * v4 + 2] = v.z;
              xw[4 * v4 + 3] = v.w;
            }
          }
          float2 x[SW];
#pragma unroll
          for (int k = 0; k < SW; ++k)
            x[k] = make_float2(xw[(jj & 1) * SW + k], xw[(jj & 1) * SW + k]);
          float2 es = make_float2(0.f, 0.f);
#pragma unroll
          for (int p = 0; p < ROWS / 2; ++p) {
            float2 t;
            if constexpr (EXP && FACT) {  // |x'|^2 - 2 q'.x'
              t = __ffma2_rn(q2[p][0], x[0], x[D]);
#pragma unroll
              for (int k = 1; k < D; ++k) t = __ffma2_rn(q2[p][k], x[k], t);
            } else if constexpr (EXP) {
              t = __fadd2_rn(qn[p], x[D]);
#pragma unroll
              for (int k = 0; k < D; ++k) t = __ffma2_rn(q2[p][k], x[k], t);
            } else if constexpr (EXP_OK) {  // -x' = 0.5 * (-2 x'), exactly
              const float2 h = make_float2(0.5f, 0.5f);
              t = fam_first<FAM>(__ffma2_rn(h, x[0], q2[p][0]));
#pragma unroll
              for (int k = 1; k < D; ++k) t = fam_next<FAM>(__ffma2_rn(h, x[k], q2[p][k]), t);
              t = fam_finish<FAM>(t);
            } else {
              t = fam_first<FAM>(__fadd2_rn(q2[p][0], x[0]));
#pragma unroll
              for (int k = 1; k < D; ++k) t = fam_next<FAM>(__fadd2_rn(q2[p][k], x[k]), t);
              t = fam_finish<FAM>(t);
            }
            const float2 e = make_float2(ex2_approx(-t.x), ex2_approx(-t.y));
            racc[p] = __fadd2_rn(racc[p], e);
            if constexpr (FACT)
              es = p == 0 ? __fmul2_rn(e, qn[0]) : __ffma2_rn(e, qn[p], es);
            else
              es = p == 0 ? e : __fadd2_rn(es, e);
          }
          c[jj] = es.x + es.y;
        }
        // transpose-reduction butterfly over lane bits 4, 3, 2 (each stage
        // keeps half of the values and sends the other half: 4 + 2 + 1
        // shuffles), then two plain folds: the four lanes with
        // lane >> 2 == s end with the column sum of source jb + bitrev3(s)
#pragma unroll
        for (int st = 16, h = 4; h >= 1; st >>= 1, h >>= 1) {
          const bool up = (lane & st) != 0;
#pragma unroll
          for (int i = 0; i < h; ++i) {
            const float keep = up ? c[i + h] : c[i];
            const float send = up ? c[i] : c[i + h];
            c[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
          }
        }
        c[0] += __shfl_xor_sync(0xffffffffu, c[0], 2);
        c[0] += __shfl_xor_sync(0xffffffffu, c[0], 1);
        {
          const uint32_t sj = jb + ((lane >> 4) & 1u) * 4u + ((lane >> 3) & 1u) * 2u +
                              ((lane >> 2) & 1u);
          if ((lane & 3u) == 0 && sj < nj) colv[sj] = c[0];
        }
      }
    };
    const uint32_t njp = (nj + 7u) & ~7u;  // whole batches; slots past nj far away
    for (uint32_t s0 = 0; s0 < njp; s0 += SC) {
      const uint32_t s1 = min(njp, s0 + SC);
      if (s0) __syncwarp();  // the previous stage has been read
      if constexpr (EXP_OK) {
        // -2 x' and |x'|^2 (absent: x' = 1e18, |x'|^2 = 1e30): the direct form
        // takes -x' = 0.5 * (-2 x') exactly through one FFMA2
        for (uint32_t j = s0 + lane; j < s1; j += 32) {
          float nrm = 1e30f;
          float xv[D];
#pragma unroll
          for (int k = 0; k < D; ++k) xv[k] = 1e18f;
          if (j < nj) {
            nrm = 0.f;
#pragma unroll
            for (int k = 0; k < D; ++k) {
              xv[k] = (__ldg(ppts + size_t(fj + j) * D + k) - c0[k]) * cs;
              nrm = fmaf(xv[k], xv[k], nrm);
            }
          }
#pragma unroll
          for (int k = 0; k < D; ++k) sx[(j - s0) * SW + k] = -2.f * xv[k];
          sx[(j - s0) * SW + D] = nrm;
        }
      } else {
        for (uint32_t idx = s0 * D + lane; idx < s1 * D; idx += 32) {
          const float v =
              idx < nj * D ? -((__ldg(ppts + size_t(fj) * D + idx) - c0[idx % D]) * cs) : -1e18f;
          if constexpr (SW == D)
            sx[idx - s0 * D] = v;
          else
            sx[(idx / D - s0) * SW + idx % D] = v;
        }
      }
      __syncwarp();
      if constexpr (EXP_OK) {
        if (use_exp)
          stage_loop(std::true_type{}, s0, s1);
        else
          stage_loop(std::false_type{}, s0, s1);
      } else {
        stage_loop(std::false_type{}, s0, s1);
      }
    }
    __syncwarp();
#pragma unroll
    for (int p = 0; p < ROWS / 2; ++p) {
      if constexpr (FACT) racc[p] = __fmul2_rn(racc[p], qn[p]);
      rowv[lane * ROWS + 2 * p] = racc[p].x;
      rowv[lane * ROWS + 2 * p + 1] = racc[p].y;
    }
    __syncwarp();
    float* rdst = P + (size_t(poff[tl.I]) + tl.slotI) * kCap;
    float* cdst = P + (size_t(poff[tl.J]) + tl.slotJ) * kCap;
    if constexpr (OWN) {
      if (tl.remote & 1u) rdst = records + size_t(tl.rec) * kSymRecWords + 4;
      if (tl.remote & 2u) cdst = records + size_t(tl.rec) * kSymRecWords + 4;
    }
    // a point that prunes the partner block drops its value
    for (uint32_t t = lane; t < ni; t += 32) {
      float q[D];
#pragma unroll
      for (int k = 0; k < D; ++k) q[k] = __ldg(pts + size_t(fi + t) * D + k);
      const float off = scale * box_dist<FAM>(q, lo + size_t(tl.J) * D, hi + size_t(tl.J) * D, D);
      rdst[t] = off > __log2f(float(nj)) + bits ? 0.f : rowv[t];
    }
    if (tl.I != tl.J) {
      for (uint32_t t = lane; t < nj; t += 32) {
        float x[D];
#pragma unroll
        for (int k = 0; k < D; ++k) x[k] = __ldg(ppts + size_t(fj + t) * D + k);
        const float off =
            scale * box_dist<FAM>(x, lo + size_t(tl.I) * D, hi + size_t(tl.I) * D, D);
        cdst[__ldg(perm + fj + t)] = off > __log2f(float(ni)) + bits ? 0.f : colv[t];
      }
    }
    __syncwarp();  // rowv/colv are refilled by the next tile
  }
  if (performed) {
    if (lane == 0 && ev) atomicAdd(performed, ev);
  }
}

#ifndef FSGG_WT_CTAS_HID
#define FSGG_WT_CTAS_HID 5
#endif
template <int D, int ROWS>
constexpr int wt_ctas() {
  return D <= 2 ? (ROWS == 8 ? 8 : 6) : (ROWS == 8 ? 6 : FSGG_WT_CTAS_HID);
}
#define FSGG_WT_ARGS                                                                          \
  const float *__restrict__ pts, float cs, const SymTile *__restrict__ tiles, uint32_t ntiles, \
      uint32_t *__restrict__ next, const uint32_t *__restrict__ bf,                            \
      const uint32_t *__restrict__ bl, const float *__restrict__ lo,                           \
      const float *__restrict__ hi, float scale, float bits, const uint32_t *__restrict__ poff, \
      float *__restrict__ P, unsigned long long *__restrict__ performed,                       \
      float *__restrict__ records, const float *__restrict__ ppts,                             \
      const uint32_t *__restrict__ perm, const float *__restrict__ bbox
template <int D, int FAM, int ROWS>
__global__ void __launch_bounds__(kWtWarps * 32, wt_ctas<D, ROWS>())
    sym_wtile_kernel(FSGG_WT_ARGS) {
  sym_wtile_body<D, FAM, ROWS, false>(pts, cs, tiles, ntiles, next, bf, bl, lo, hi, scale, bits,
                                      poff, P, performed, records, ppts, perm, bbox);
}
template <int D, int FAM, int ROWS>
__global__ void __launch_bounds__(kWtWarps * 32, wt_ctas<D, ROWS>())
    sym_wtile_own_kernel(FSGG_WT_ARGS) {
  sym_wtile_body<D, FAM, ROWS, true>(pts, cs, tiles, ntiles, next, bf, bl, lo, hi, scale, bits,
                                     poff, P, performed, records, ppts, perm, bbox);
}
#undef FSGG_WT_ARGS

// Fold each point's partner values, in ascending partner order, into its
// fp64 bucket row (bucket of partner J = J >> shift).
constexpr uint32_t kSymBucketChunk = 16;  // 16 x 257 fp64 = 32 KiB of shared memory
__global__ void __launch_bounds__(kSymBlock)
    sym_rows_kernel(const float* __restrict__ P, const uint32_t* __restrict__ poff,
                    const uint32_t* __restrict__ plist, const uint32_t* __restrict__ bf,
                    const uint32_t* __restrict__ bl, uint32_t blk0, uint32_t shift,
                    uint32_t rd, uint32_t qb, uint32_t qe, double* __restrict__ rows,
                    uint32_t ps) {
  // acc[c][t]: point t's sum for bucket b0 + c (row stride 257: conflict-free
  // when the store pass below reads it column-wise)
  __shared__ double acc[kSymBucketChunk][kSymBlock + 1];
  const uint32_t I = blk0 + blockIdx.x;
  const uint32_t f = bf[I], ni = bl[I] - f;
  const uint32_t t = threadIdx.x;
  const uint32_t W = 1u << rd;
  const uint32_t p0 = poff[I], p1 = poff[I + 1];
  // points of this block that are queries of this call
  const uint32_t t0 = qb > f ? min(qb - f, ni) : 0u;
  const uint32_t t1 = qe > f ? min(qe - f, ni) : 0u;
  uint32_t k = p0;
  for (uint32_t b0 = 0; b0 < W; b0 += kSymBucketChunk) {
#pragma unroll
    for (uint32_t c = 0; c < kSymBucketChunk; ++c) acc[c][t] = 0.0;
    // partners in ascending order, 8 loads in flight per thread (one
    // dependent load per partner left the kernel latency-bound)
    const uint32_t bend = b0 + kSymBucketChunk;
    while (k < p1) {
      constexpr int kB = 8;
      uint32_t cb[kB];
      float v[kB];
      uint32_t take = 0;
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        cb[j] = k + j < p1 ? (__ldg(plist + k + j) >> shift) : 0xffffffffu;
        take += cb[j] < bend ? 1u : 0u;  // a prefix: partners are sorted
      }
#pragma unroll
      for (int j = 0; j < kB; ++j)
        v[j] = (cb[j] < bend && t < ni) ? __ldg(P + size_t(k + j) * ps + t) : 0.f;
#pragma unroll
      for (int j = 0; j < kB; ++j)
        if (cb[j] < bend && t < ni) acc[cb[j] - b0][t] += double(v[j]);
      k += take;
      if (take < uint32_t(kB)) break;
    }
    __syncthreads();
    // coalesced store: consecutive threads write consecutive buckets of a point
    const uint32_t cmax = min(kSymBucketChunk, W - b0);
    for (uint32_t idx = t; idx < (t1 - t0) * cmax; idx += blockDim.x) {
      const uint32_t pt = t0 + idx / cmax, c = idx % cmax;
      rows[(size_t(f + pt - qb) << rd) + b0 + c] = acc[c][pt];
    }
    __syncthreads();
  }
}

// Received exchange records into P: X's slot for partner Y.
__global__ void sym_receive_kernel(const uint32_t* __restrict__ records,
                                   const uint32_t* __restrict__ poff,
                                   const uint32_t* __restrict__ plist, float* __restrict__ P,
                                   uint32_t ps) {
  const uint32_t* r = records + size_t(blockIdx.x) * kSymRecWords;
  const uint32_t X = r[0], Y = r[1], nx = r[3];
  uint32_t lo = poff[X], hi = poff[X + 1];
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (plist[mid] < Y)
      lo = mid + 1;
    else
      hi = mid;
  }
  for (uint32_t t = threadIdx.x; t < nx; t += blockDim.x)
    P[size_t(lo) * ps + t] = __uint_as_float(r[4 + t]);
}

// Block index of every point (blocks are the depth-Lb tree nodes).
__global__ void sym_qblock_kernel(const uint32_t* __restrict__ bf,
                                  const uint32_t* __restrict__ bl,
                                  uint32_t* __restrict__ qblk) {
  const uint32_t I = blockIdx.x;
  for (uint32_t p = bf[I] + threadIdx.x; p < bl[I]; p += blockDim.x) qblk[p] = I;
}

// pos[I - b0][J] = position of the first partner >= J in I's ascending
// partner list (J = 0..B), for the query blocks I in [b0, b0 + gridDim.x):
// a lookup then finds the partner run of any block range with three
// independent loads instead of a binary search.
constexpr uint32_t kSymPosMaxBlocks = 8192;  // table (B + 1)^2 x 4 bytes <= 256 MiB
__global__ void sym_pos_kernel(uint32_t B, uint32_t b0, const uint32_t* __restrict__ poff,
                               const uint32_t* __restrict__ plist, uint32_t* __restrict__ pos) {
  const uint32_t I = b0 + blockIdx.x;
  uint32_t* row = pos + size_t(blockIdx.x) * (B + 1);
  const uint32_t p0 = poff[I], p1 = poff[I + 1];
  for (uint32_t k = p0 + threadIdx.x; k < p1; k += blockDim.x) {
    const uint32_t from = k == p0 ? 0u : plist[k - 1] + 1;
    for (uint32_t J = from; J <= plist[k]; ++J) row[J] = k;
  }
  const uint32_t tail = p1 > p0 ? plist[p1 - 1] + 1 : 0u;
  for (uint32_t J = tail + threadIdx.x; J <= B; J += blockDim.x) row[J] = p1;
}

// One thread per entry, kBlkUnroll entries per thread (all loads first). The
// node's blocks are [B0, B1) (heap slot g at `level` covers blocks
// g << (Lb - level) ...); q's partners in that run are a contiguous range of
// its block's ascending partner list: one lower_bound for B0, then a forward
// scan that sums the values of the left half [B0, Bm) and the right half
// [Bm, B1) in partner order (fp64), exactly the values the root rows fold.
constexpr int kBlkThreads = 256;
constexpr int kBlkUnroll = 2;
__global__ void __launch_bounds__(kBlkThreads)
    block_lookup_kernel(uint32_t E, uint32_t level, uint32_t Lb,
                        const uint32_t* __restrict__ eq, const uint32_t* __restrict__ eg,
                        const uint32_t* __restrict__ qblk, const uint32_t* __restrict__ bf,
                        const uint32_t* __restrict__ poff, const uint32_t* __restrict__ plist,
                        const float* __restrict__ P, const uint32_t* __restrict__ tfirst,
                        const uint32_t* __restrict__ tlast, const uint32_t* __restrict__ pos,
                        uint32_t b0, uint32_t ps, double* __restrict__ g1,
                        double* __restrict__ g2, unsigned long long* __restrict__ evals,
                        const uint32_t* __restrict__ dE) {
  constexpr int U = kBlkUnroll;
  if (dE) E = *dE;  // sync-free levels: the count is on the device
  const uint32_t sh = Lb - level;
  unsigned long long ev = 0;
  for (uint32_t tile = blockIdx.x; uint64_t(tile) * (kBlkThreads * U) < E; tile += gridDim.x) {
  const uint32_t base = tile * (kBlkThreads * U) + threadIdx.x;
  uint32_t q[U], g[U], I[U], size[U], k[U], k1[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * kBlkThreads;
    q[u] = i < E ? eq[i] : 0u;
    g[u] = i < E ? eg[i] : 0u;
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint64_t h = ((1ull << level) - 1) + g[u];
    size[u] = base + u * kBlkThreads < E ? tlast[h] - tfirst[h] : 0u;
    I[u] = qblk[q[u]];
    k[u] = poff[I[u]];
    k1[u] = poff[I[u] + 1];
  }
  double a[U], b[U];
  if (pos) {  // partner runs from the position table
    const uint32_t W = (1u << Lb) + 1;
    uint32_t km[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      k[u] = km[u] = k1[u] = 0;
      if (base + u * kBlkThreads < E) {  // (a padding lane's query 0 may precede b0)
        const uint32_t* row = pos + size_t(I[u] - b0) * W;
        const uint32_t B0 = g[u] << sh;
        k[u] = row[B0];
        km[u] = row[B0 + (1u << (sh - 1))];
        k1[u] = row[B0 + (1u << sh)];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = b[u] = 0.0;
      const float* pv = P + (q[u] - bf[I[u]]);
      // 4 loads in flight; absent ones add +0 (the sums keep their bits)
      for (uint32_t kk = k[u]; kk < km[u]; kk += 4) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = kk + j < km[u] ? __ldg(pv + size_t(kk + j) * ps) : 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) a[u] += double(v[j]);
      }
      for (uint32_t kk = km[u]; kk < k1[u]; kk += 4) {
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = kk + j < k1[u] ? __ldg(pv + size_t(kk + j) * ps) : 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) b[u] += double(v[j]);
      }
    }
  } else
#pragma unroll
  for (int u = 0; u < U; ++u) {
    a[u] = b[u] = 0.0;
    const uint32_t B0 = g[u] << sh, Bm = B0 + (1u << (sh - 1)), B1 = B0 + (1u << sh);
    // lower_bound(B0) in plist[k, k1)
    uint32_t lo = k[u], hi = k1[u];
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(plist + mid) < B0)
        lo = mid + 1;
      else
        hi = mid;
    }
    const uint32_t t = q[u] - bf[I[u]];
    for (uint32_t kk = lo; kk < k1[u]; ++kk) {
      const uint32_t J = __ldg(plist + kk);
      if (J >= B1) break;
      const double v = double(__ldg(P + size_t(kk) * ps + t));
      if (J < Bm)
        a[u] += v;
      else
        b[u] += v;
    }
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const uint32_t i = base + u * kBlkThreads;
    if (i >= E) continue;
    g1[i] = fmax(a[u], kSumFloor);
    g2[i] = fmax(b[u], kSumFloor);
    ev += size[u];
  }
  }  // tiles
  __shared__ unsigned long long red[kBlkThreads / 32];
  for (int o = 16; o; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ev;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int w = 0; w < kBlkThreads / 32; ++w) tot += red[w];
    if (tot) atomicAdd(evals, tot);
  }
}

template <class F>
void sym_by_dim(uint32_t d, F&& f) {
  switch (d) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 3: f(std::integral_constant<int, 3>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 5: f(std::integral_constant<int, 5>{}); break;
    case 6: f(std::integral_constant<int, 6>{}); break;
    case 7: f(std::integral_constant<int, 7>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    default: throw ConfigError("symmetric root supports d <= 8");
  }
}

}  // namespace

uint32_t sym_block_depth(const Dataset& ds) {
  const TreeTable& t = ds.tree;
  if (ds.d < 1 || ds.d > 8 || !t.has_boxes) return 0;
  // blocks: tree nodes at depth Lb with <= 320 points (<= 256 for d > 6:
  // 10-row lanes would spill)
  const uint32_t cap = ds.d <= 6 ? kSymBlock : 256u;
  uint32_t Lb = 0;
  while (((uint64_t(ds.n) + (1ull << Lb) - 1) >> Lb) > cap) ++Lb;
  if (Lb == 0 || Lb > t.depth || Lb > 20) return 0;
  // tiles hold 256 (or 320) rows in registers: smaller blocks leave lanes
  // idle (151-point blocks measured slower than the one-sided tiled kernel)
  if ((uint64_t(ds.n) >> Lb) < kSymMinBlock) return 0;
  return Lb;
}

// Rows per lane of the tile kernel for this dataset's blocks.
int sym_rows_per_lane(const Dataset& ds, uint32_t Lb) {
  return ((uint64_t(ds.n) + (1ull << Lb) - 1) >> Lb) > 256 ? 10 : 8;
}
// Values per (block, partner) slot of P: the tile capacity.
uint32_t sym_pstride(const Dataset& ds, uint32_t Lb) { return 32u * sym_rows_per_lane(ds, Lb); }

namespace {

// Count / fill the partner lists, build the tile list of the query blocks
// [b0, b1] and run the tile kernel. own: owner mode (multi-GPU exchange);
// remote sides go to "sym.rec" records (*nrec of them).
void sym_tile_pass(Dataset& ds, const KernelSpec& ks, uint32_t qb, uint32_t qe, bool own,
                   unsigned long long* d_performed, cudaEvent_t ev0, cudaEvent_t ev1,
                   uint32_t* b0_out, uint32_t* b1_out, uint32_t* nrec_out) {
  const TreeTable& t = ds.tree;
  const uint32_t Lb = sym_block_depth(ds);
  cudaStream_t s = ds.stream;
  const uint32_t B = 1u << Lb;
  const uint64_t hb = uint64_t(B) - 1;
  const uint32_t* bf = t.first.as<uint32_t>() + hb;
  const uint32_t* bl = t.last.as<uint32_t>() + hb;
  const float* lo = t.lo.as<float>() + hb * ds.d;
  const float* hi = t.hi.as<float>() + hb * ds.d;
  // half the root mass (>= 1/2); the call's threshold (kPruneBits, or the
  // fast backend's)
  const float bits = (ds.kde_ws ? ds.kde_ws->prune_bits : kPruneBits) + 1.f;

  DevBuf& cnt = ds.buf("sym.cnt", size_t(B + 1) * 4);
  DevBuf& poff = ds.buf("sym.poff", size_t(B + 1) * 4);
  DevBuf& tmp = ds.buf("sym.tmp", 8);
  sym_count_kernel<<<B, 256, 0, s>>>(B, lo, hi, bf, bl, ds.d, ks.family, ks.scale, bits,
                                     cnt.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  FSGG_CUDA(cudaMemsetAsync(cnt.as<uint32_t>() + B, 0, 4, s));
  size_t tb = 0;
  FSGG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<uint32_t>(), poff.as<uint32_t>(),
                                          B + 1, s));
  tmp.ensure(tb, s);
  FSGG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.as<void>(), tb, cnt.as<uint32_t>(),
                                          poff.as<uint32_t>(), B + 1, s));
  uint32_t npart = 0;
  FSGG_CUDA(cudaMemcpyAsync(&npart, poff.as<uint32_t>() + B, 4, cudaMemcpyDeviceToHost, s));
  // query blocks: the blocks holding points qb and qe - 1
  std::vector<uint32_t> hbf(B), hbl(B);
  FSGG_CUDA(cudaMemcpyAsync(hbf.data(), bf, size_t(B) * 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(hbl.data(), bl, size_t(B) * 4, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  uint32_t b0 = 0, b1 = B - 1;
  while (b0 < B && hbl[b0] <= qb) ++b0;
  while (b1 > 0 && hbf[b1] >= qe) --b1;
  DevBuf& plist = ds.buf("sym.plist", size_t(npart) * 4 + 4);
  sym_fill_kernel<<<B, 256, 0, s>>>(B, lo, hi, bf, bl, ds.d, ks.family, ks.scale, bits,
                                    poff.as<uint32_t>(), plist.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  DevBuf& tiles = ds.buf("sym.tiles", size_t(npart) * sizeof(SymTile) + 16);
  // [tiles, cross tiles, the warp-per-tile kernels' two take counters]
  DevBuf& ntiles = ds.buf("sym.ntiles", 16);
  FSGG_CUDA(cudaMemsetAsync(ntiles.as<void>(), 0, 16, s));
  // a cross tile has one remote side: at most half the partner slots
  DevBuf& rec = ds.buf("sym.rec", own ? (size_t(npart) / 2 + 1) * kSymRecWords * 4 : 4);
  DevBuf& xtiles = ds.buf("sym.xtiles", own ? (size_t(npart) / 2 + 1) * sizeof(SymTile) : 16);
  sym_tiles_kernel<<<B, 128, 0, s>>>(B, poff.as<uint32_t>(), plist.as<uint32_t>(), b0, b1, bf,
                                     bl, tiles.as<SymTile>(), ntiles.as<uint32_t>(),
                                     nullptr, own ? 1 : 0, ntiles.as<uint32_t>() + 1,
                                     rec.as<uint32_t>(), xtiles.as<SymTile>());
  FSGG_LAUNCH_CHECK();
  uint32_t nt2[2] = {0, 0};
  FSGG_CUDA(cudaMemcpyAsync(nt2, ntiles.as<void>(), 8, cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  const uint32_t nt = nt2[0], nx = own ? nt2[1] : 0;
  DevBuf& P = ds.buf("sym.P", size_t(npart) * sym_pstride(ds, Lb) * 4 + 4);
  DevBuf& ppts = ds.buf("sym.ppts", size_t(ds.n) * ds.d * 4);
  DevBuf& perm = ds.buf("sym.perm", size_t(ds.n) * 4);
  DevBuf& bbox = ds.buf("sym.bbox", size_t(B) * kSymBatches * 2 * ds.d * 4);
  sym_perm_kernel<<<B, 256, 0, s>>>(ds.pts.as<float>(), ds.d, bf, bl, ppts.as<float>(),
                                    perm.as<uint32_t>(), bbox.as<float>());
  FSGG_LAUNCH_CHECK();
  ds.launches++;
  if (ev0) FSGG_CUDA(cudaEventRecord(ev0, s));
  // the shard's own tiles with the single-GPU kernel, then (owner mode) the
  // cross-shard tiles with the kernel that exports one side
  const int rows = sym_rows_per_lane(ds, Lb);
  const float cs = ks.family == 0 ? sqrtf(ks.scale) : ks.scale;
  // FSGG_SYM_WPT: 0 CTA-per-tile kernels, 1 warp-per-tile for d <= 2, 2 for d <= 6
  static const int wpt = [] {
    const char* e = std::getenv("FSGG_SYM_WPT");
    return e ? std::atoi(e) : 2;
  }();
  for (int pass = 0; pass < 2; ++pass) {
    const uint32_t cnt = pass == 0 ? nt : nx;
    if (cnt == 0) continue;
    const SymTile* tl = pass == 0 ? tiles.as<SymTile>() : xtiles.as<SymTile>();
    sym_by_dim(ds.d, [&](auto dim) {
      constexpr int D = decltype(dim)::value;
      // persistent warp-per-tile kernel, tiles taken from a counter
      if constexpr (D <= 6) {
        if (wpt >= 2 || (wpt == 1 && D <= 2)) {
          auto wlaunch = [&](auto kern) {
            int per_sm = 0;
            FSGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                                    kWtWarps * 32, 0));
            const uint32_t grid = std::min<uint32_t>(
                (cnt + kWtWarps - 1) / kWtWarps, uint32_t(std::max(per_sm, 1)) * uint32_t(ds.num_sms));
            kern<<<grid, kWtWarps * 32, 0, s>>>(
                ds.pts.as<float>(), cs, tl, cnt, ntiles.as<uint32_t>() + 2 + pass, bf, bl, lo,
                hi, ks.scale, bits, poff.as<uint32_t>(), P.as<float>(), d_performed,
                rec.as<float>(), ppts.as<float>(), perm.as<uint32_t>(), bbox.as<float>());
          };
          auto wby_rows = [&](auto fam) {
            constexpr int FAM = decltype(fam)::value;
            if (rows == 10)
              return pass ? wlaunch(sym_wtile_own_kernel<D, FAM, 10>)
                          : wlaunch(sym_wtile_kernel<D, FAM, 10>);
            pass ? wlaunch(sym_wtile_own_kernel<D, FAM, 8>)
                 : wlaunch(sym_wtile_kernel<D, FAM, 8>);
          };
          switch (ks.family) {
            case 0: wby_rows(std::integral_constant<int, 0>{}); break;
            case 1: wby_rows(std::integral_constant<int, 1>{}); break;
            default: wby_rows(std::integral_constant<int, 2>{}); break;
          }
          return;
        }
      }
      auto launch = [&](auto kern, int threads) {
        kern<<<cnt, threads, 0, s>>>(ds.pts.as<float>(), cs, tl, bf, bl, lo, hi,
                                     ks.scale, bits,
                                     poff.as<uint32_t>(), P.as<float>(), d_performed,
                                     rec.as<float>(), ppts.as<float>(), perm.as<uint32_t>(),
                                     bbox.as<float>());
      };
      auto by_rows = [&](auto fam) {
        constexpr int FAM = decltype(fam)::value;
        if constexpr (D <= 6) {
          if (rows == 10)
            return pass ? launch(sym_tile_own_kernel<D, FAM, 10>, 160)
                        : launch(sym_tile_kernel<D, FAM, 10>, 160);
        }
        pass ? launch(sym_tile_own_kernel<D, FAM, 8>, 128)
             : launch(sym_tile_kernel<D, FAM, 8>, 128);
      };
      switch (ks.family) {
        case 0: by_rows(std::integral_constant<int, 0>{}); break;
        case 1: by_rows(std::integral_constant<int, 1>{}); break;
        default: by_rows(std::integral_constant<int, 2>{}); break;
      }
    });
    FSGG_LAUNCH_CHECK();
  }
  if (ev1) FSGG_CUDA(cudaEventRecord(ev1, s));
  ds.launches += 4;
  *b0_out = b0;
  *b1_out = b1;
  *nrec_out = own ? nt2[1] : 0;
}

}  // namespace

bool sym_shard_prepare(Dataset& ds, const KernelSpec& ks, uint32_t qb, uint32_t qe,
                       uint32_t* num_records, const uint32_t** records) {
  *num_records = 0;
  *records = nullptr;
  if (!ds.kde_ws) ds.kde_ws = std::make_unique<KdeWorkspace>();
  KdeWorkspace& ws = *ds.kde_ws;
  ws.sym_ready = false;
  const uint32_t Lb = sym_block_depth(ds);
  if (Lb == 0 || qe <= qb) return false;
  // owner mode needs block-aligned shard bounds (every block on one rank)
  const TreeTable& t = ds.tree;
  const uint64_t hb = (uint64_t(1) << Lb) - 1;
  std::vector<uint32_t> hbf(size_t(1) << Lb);
  FSGG_CUDA(cudaMemcpyAsync(hbf.data(), t.first.as<uint32_t>() + hb, hbf.size() * 4,
                            cudaMemcpyDeviceToHost, ds.stream));
  FSGG_CUDA(cudaStreamSynchronize(ds.stream));
  const bool qb_ok = std::binary_search(hbf.begin(), hbf.end(), qb);
  const bool qe_ok = qe == ds.n || std::binary_search(hbf.begin(), hbf.end(), qe);
  // Not a silent fallback: a peer whose bounds are aligned would run owner
  // mode and wait for records this rank never sends (its sym.P slots would
  // keep an earlier build's values).
  if (!qb_ok || !qe_ok)
    throw ConfigError("shard bounds must sit on symmetric-root block boundaries "
                      "(use fsgg_shard_bounds)");
  if (!ws.ev0) {
    FSGG_CUDA(cudaEventCreate(&ws.ev0));
    FSGG_CUDA(cudaEventCreate(&ws.ev1));
  }
  DevBuf& perf = ds.buf("sym.perf", 8);
  FSGG_CUDA(cudaMemsetAsync(perf.as<void>(), 0, 8, ds.stream));
  uint32_t b0 = 0, b1 = 0, nrec = 0;
  sym_tile_pass(ds, ks, qb, qe, true, perf.as<unsigned long long>(), ws.ev0, ws.ev1, &b0, &b1,
                &nrec);
  FSGG_CUDA(cudaStreamSynchronize(ds.stream));
  float ms = 0.f;
  FSGG_CUDA(cudaEventElapsedTime(&ms, ws.ev0, ws.ev1));
  ws.sym_ready = true;
  ws.sym_ready_qb = qb;
  ws.sym_ready_qe = qe;
  ws.sym_ready_scale = ks.scale;
  ws.sym_ready_family = ks.family;
  ws.sym_ready_bits = ws.prune_bits;
  ws.sym_ready_b0 = b0;
  ws.sym_ready_b1 = b1;
  ws.sym_ready_seconds = ms * 1e-3;
  *num_records = nrec;
  *records = ds.buf("sym.rec", 4).as<uint32_t>();
  return true;
}

void sym_shard_receive(Dataset& ds, const uint32_t* records, uint32_t num_records) {
  if (!ds.kde_ws || !ds.kde_ws->sym_ready) throw ConfigError("no prepared symmetric root");
  if (num_records == 0) return;
  sym_receive_kernel<<<num_records, 256, 0, ds.stream>>>(
      records, ds.buf("sym.poff", 4).as<uint32_t>(), ds.buf("sym.plist", 4).as<uint32_t>(),
      ds.buf("sym.P", 4).as<float>(), sym_pstride(ds, sym_block_depth(ds)));
  FSGG_LAUNCH_CHECK();
  ds.launches++;
}

bool kde_root_symmetric(Dataset& ds, const KernelSpec& ks, uint32_t qb, uint32_t qe,
                        uint32_t rd, double* rows, unsigned long long* d_performed,
                        cudaEvent_t ev0, cudaEvent_t ev1) {
  const TreeTable& t = ds.tree;
  const uint32_t Lb = sym_block_depth(ds);
  if (Lb == 0 || Lb < rd) return false;
  cudaStream_t s = ds.stream;
  const uint32_t B = 1u << Lb;
  const uint64_t hb = uint64_t(B) - 1;
  const uint32_t* bf = t.first.as<uint32_t>() + hb;
  const uint32_t* bl = t.last.as<uint32_t>() + hb;
  KdeWorkspace& ws = *ds.kde_ws;
  uint32_t b0 = 0, b1 = 0, nrec = 0;
  ws.sym_prepared_seconds = 0.0;
  if (ws.sym_ready && ws.sym_ready_qb == qb && ws.sym_ready_qe == qe &&
      ws.sym_ready_scale == ks.scale && ws.sym_ready_family == ks.family &&
      ws.sym_ready_bits == ws.prune_bits) {
    // tiles already computed by sym_shard_prepare (+ received records)
    b0 = ws.sym_ready_b0;
    b1 = ws.sym_ready_b1;
    FSGG_CUDA(cudaMemcpyAsync(d_performed, ds.buf("sym.perf", 8).as<void>(), 8,
                              cudaMemcpyDeviceToDevice, s));
    if (ev0) FSGG_CUDA(cudaEventRecord(ev0, s));
    if (ev1) FSGG_CUDA(cudaEventRecord(ev1, s));
    ws.sym_prepared_seconds = ws.sym_ready_seconds;
  } else {
    sym_tile_pass(ds, ks, qb, qe, false, d_performed, ev0, ev1, &b0, &b1, &nrec);
  }
  ws.sym_ready = false;
  DevBuf& poff = ds.buf("sym.poff", 4);
  DevBuf& plist = ds.buf("sym.plist", 4);
  DevBuf& P = ds.buf("sym.P", 4);
  ds.kde_ws->sym_b0 = b0;
  ds.kde_ws->sym_pos = B <= kSymPosMaxBlocks && b0 <= b1;
  if (ds.kde_ws->sym_pos) {
    DevBuf& pos = ds.buf("sym.pos", size_t(b1 - b0 + 1) * (B + 1) * 4);
    sym_pos_kernel<<<b1 - b0 + 1, 256, 0, s>>>(B, b0, poff.as<uint32_t>(), plist.as<uint32_t>(),
                                              pos.as<uint32_t>());
    FSGG_LAUNCH_CHECK();
    ds.launches++;
  }
  DevBuf& qblk = ds.buf("sym.qblk", size_t(ds.n) * 4);
  sym_qblock_kernel<<<B, 256, 0, s>>>(bf, bl, qblk.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  ds.launches++;
  if (b0 <= b1) {
    sym_rows_kernel<<<b1 - b0 + 1, kSymBlock, 0, s>>>(P.as<float>(), poff.as<uint32_t>(),
                                                     plist.as<uint32_t>(), bf, bl, b0,
                                                     Lb - rd, rd, qb, qe, rows,
                                                     sym_pstride(ds, Lb));
    FSGG_LAUNCH_CHECK();
    ds.launches++;
  }
  return true;
}

// Cost model of a shard (measured on C3): a root pair evaluation costs
// ~6.6e-6 of the descent work of one query; a block's root cost is half its
// pair evaluations (cross tiles are split between the two owners).
constexpr double kRootPairPerQuery = 6.6e-6;

void sym_shard_bounds(Dataset& ds, const KernelSpec* ks, uint32_t world, uint32_t* bounds) {
  const uint32_t Lb = sym_block_depth(ds);
  for (uint32_t r = 0; r <= world; ++r) bounds[r] = uint32_t(uint64_t(ds.n) * r / world);
  if (Lb == 0) return;
  const uint32_t B = 1u << Lb;
  const uint64_t hb = uint64_t(B) - 1;
  std::vector<uint32_t> hbf(B), hbl(B), cnt(B, 0);
  FSGG_CUDA(cudaMemcpyAsync(hbf.data(), ds.tree.first.as<uint32_t>() + hb, size_t(B) * 4,
                            cudaMemcpyDeviceToHost, ds.stream));
  FSGG_CUDA(cudaMemcpyAsync(hbl.data(), ds.tree.last.as<uint32_t>() + hb, size_t(B) * 4,
                            cudaMemcpyDeviceToHost, ds.stream));
  if (ks) {  // active partners per block (the root pass's own count kernel)
    DevBuf& c = ds.buf("sym.cnt", size_t(B + 1) * 4);
    sym_count_kernel<<<B, 256, 0, ds.stream>>>(
        B, ds.tree.lo.as<float>() + hb * ds.d, ds.tree.hi.as<float>() + hb * ds.d,
        ds.tree.first.as<uint32_t>() + hb, ds.tree.last.as<uint32_t>() + hb, ds.d, ks->family,
        ks->scale, (ds.kde_ws ? ds.kde_ws->prune_bits : kPruneBits) + 1.f, c.as<uint32_t>());
    FSGG_LAUNCH_CHECK();
    FSGG_CUDA(cudaMemcpyAsync(cnt.data(), c.as<void>(), size_t(B) * 4, cudaMemcpyDeviceToHost,
                              ds.stream));
  }
  FSGG_CUDA(cudaStreamSynchronize(ds.stream));
  // cumulative cost over blocks; rank r starts at the first block whose
  // prefix reaches r/world of the total (equal block counts without ks)
  const double per_block = double(ds.n) / B;
  std::vector<double> pre(B + 1, 0.0);
  for (uint32_t I = 0; I < B; ++I) {
    const double sz = double(hbl[I] - hbf[I]);
    pre[I + 1] = pre[I] + sz * (1.0 + kRootPairPerQuery * 0.5 * cnt[I] * per_block);
  }
  uint32_t I = 0;
  for (uint32_t r = 1; r < world; ++r) {
    const double target = pre[B] * r / world;
    while (I < B && pre[I + 1] <= target) ++I;
    // nearer of the two block boundaries around the target
    const uint32_t cut = (I < B && target - pre[I] > pre[I + 1] - target) ? I + 1 : I;
    bounds[r] = cut < B ? hbf[cut] : ds.n;
  }
  bounds[0] = 0;
  bounds[world] = ds.n;
  for (uint32_t r = 1; r <= world; ++r) bounds[r] = std::max(bounds[r], bounds[r - 1]);
}

void block_lookup_sums(Dataset& ds, uint32_t E, uint32_t level, const uint32_t* eq,
                       const uint32_t* eg, double* g1, double* g2,
                       unsigned long long* evals, const uint32_t* dE) {
  const uint32_t Lb = ds.kde_ws ? ds.kde_ws->sym_Lb : 0;
  if (Lb == 0 || level == 0 || level + 1 > Lb) throw NumericError("no symmetric block values");
  if (E == 0) return;
  const TreeTable& t = ds.tree;
  const uint64_t hb = (uint64_t(1) << Lb) - 1;
  cudaStream_t s = ds.stream;
  // E: the entry count, or with dE its upper bound (grid-strided)
  const uint32_t grid = std::min<uint32_t>(ceil_div_u32(E, kBlkThreads * kBlkUnroll),
                                           uint32_t(ds.num_sms) * 16);
  block_lookup_kernel<<<grid, kBlkThreads, 0, s>>>(
      E, level, Lb, eq, eg, ds.buf("sym.qblk", 4).as<uint32_t>(), t.first.as<uint32_t>() + hb,
      ds.buf("sym.poff", 4).as<uint32_t>(), ds.buf("sym.plist", 4).as<uint32_t>(),
      ds.buf("sym.P", 4).as<float>(), t.first.as<uint32_t>(), t.last.as<uint32_t>(),
      ds.kde_ws->sym_pos ? ds.buf("sym.pos", 4).as<uint32_t>() : nullptr, ds.kde_ws->sym_b0,
      sym_pstride(ds, Lb), g1,
      g2, evals, dE);
  FSGG_LAUNCH_CHECK();
  ds.launches++;
}

}  // namespace fsgg
