// Tensor-core child sums for high-dimensional data (d >= kTcMinDim):
// tcgen05.mma kind::tf32 with TMEM accumulators, TMA-fed sources and
// error-compensated 3xTF32, replacing the CUDA-core kde_xd_tiled_kernel.
//
// For a block of 128 entries (queries q_m, gathered) against a source range
// (x_n, contiguous) the kernel forms S = Q X^T on the tensor cores,
//   S ~= Qhi Xhi^T + Qhi Xlo^T + Qlo Xhi^T     (hi = tf32(x), lo = tf32(x - hi))
// which keeps fp32-level accuracy (SURVEY.md §8a': 1.1e-8 vs 4.4e-5 for
// 1xTF32), then in the epilogue d2 = |q|^2 + |x|^2 - 2 S, arg = -scale * d2
// (gaussian) or -scale * sqrt(d2) (exponential), one MUFU.EX2 per element and
// a per-row running sum — the n x n matrix never leaves TMEM/registers.
//
// CTA = 8 warps, warp-specialised:
//   warp 0     TMA producer: source tiles Xhi/Xlo (128 rows x 32 fp32, SW128)
//   warp 1     TMEM allocator + single-thread MMA issuer
//   warps 2-3  query gather: cp.async of Qhi/Qlo rows into the SW128 layout
//   warps 4-7  epilogue: tcgen05.ld of the 128 x 128 fp32 accumulator
// Pipelines: 3-stage smem ring (full/empty mbarriers), double-buffered TMEM
// accumulator (tfull/tempty) so the epilogue of N-tile t overlaps the MMAs of
// N-tile t+1.
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "engine.cuh"

namespace fsgg {
namespace {

constexpr int kTcM = 128;       // entries per work item = TMEM lanes
constexpr int kTcN = 128;       // sources per N-tile
constexpr int kTcKB = 32;       // fp32 per K-block: one 128-byte SW128 row
constexpr int kTcStages = 3;
constexpr int kTcThreads = 256;
constexpr int kTileBytes = kTcM * kTcKB * 4;            // 16 KiB (A or B, hi or lo)
constexpr int kStageBytes = 4 * kTileBytes;             // Ahi, Alo, Bhi, Blo
constexpr int kSmemBytes = kTcStages * kStageBytes + 1024 + 512;
constexpr uint32_t kTmemCols = 256;                     // 2 x 128-column accumulators
constexpr uint32_t kTcGroup = 64;                       // entry blocks per L2 group
constexpr int kRing = 8;          // work-item ring (persistent kernel)
constexpr int kRingReaders = 6;   // MMA thread, query warp, 4 epilogue warps

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// TMA row gather (sm_100a): four rows of a 2-D tensor (box {32 fp32, 1 row})
// at arbitrary row indices land as four consecutive 128-byte rows at dst,
// swizzled by their shared-memory address like a regular SW128 tile.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int col, int r0, int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// K-major, 128-byte-swizzled shared-memory matrix descriptor (sm100 UMMA):
// start >> 4 [0,14), LBO >> 4 [16,30) (unused for SW128 K-major: 1),
// SBO >> 4 [32,46) = 1024 B between 8-row groups, version 1 [46,48),
// layout type SWIZZLE_128B = 2 [61,64).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 128.
constexpr uint32_t kIdesc = (1u << 4)            // c_format F32
                            | (2u << 7)          // a_format TF32
                            | (2u << 10)         // b_format TF32
                            | (uint32_t(kTcN >> 3) << 17) | (uint32_t(kTcM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

// hi = tf32(x) (round to nearest), lo = tf32(x - hi); both stored as fp32
// bit patterns in row-major n x d_pad arrays (padding columns are 0), plus
// |x|^2 accumulated in fp64 and rounded once.
// Per-dimension mean (fixed-order fp64 reduction, one CTA per dimension).
// Centring leaves every pairwise distance unchanged but shrinks |x|^2 and
// the dot products, which is what limits d2 = |q|^2 + |x|^2 - 2 q.x: the
// tensor cores' fp32 accumulation (not IEEE round-to-nearest across the K
// steps) loses ~1e-5 of |S| on uncentred [0,1]^784 data, <1e-7 centred.
__global__ void tc_mean_kernel(const float* __restrict__ pts, uint32_t n, uint32_t d,
                               float* __restrict__ mean) {
  const uint32_t k = blockIdx.x;
  double acc = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) acc += pts[size_t(i) * d + k];
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) mean[k] = float(red[0] / n);
}

__global__ void tc_split_kernel(const float* __restrict__ pts, uint32_t n, uint32_t d,
                                uint32_t d_pad, const float* __restrict__ mean,
                                float* __restrict__ hi, float* __restrict__ lo,
                                float* __restrict__ norm) {
  const uint32_t row = blockIdx.x;
  if (row >= n) return;
  double acc = 0.0;
  for (uint32_t k = threadIdx.x; k < d_pad; k += blockDim.x) {
    float h = 0.f, l = 0.f;
    if (k < d) {
      const float x = pts[size_t(row) * d + k] - mean[k];
      uint32_t hb;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x));
      h = __uint_as_float(hb);
      uint32_t lb;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(x - h));
      l = __uint_as_float(lb);
      acc += double(x) * double(x);
    }
    hi[size_t(row) * d_pad + k] = h;
    lo[size_t(row) * d_pad + k] = l;
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) norm[row] = float(red[0]);
}

// Work item: (entry block, side, chunk group), visited in groups of
// kTcGroup entry blocks x all source groups so the concurrent CTAs share
// their query and source tiles through L2 (the hi/lo copies of C5 are
// 440 MB; with a block-major order every CTA streams its sources from
// DRAM). whole: nodes of <= kTcN points take one item per (entry block,
// node), both children in one N tile (each query tile gathered once).
struct TcItem {
  uint32_t g, side, kk, e0, e1, cf, cl, ntiles;
};

__device__ __forceinline__ TcItem tc_item(uint32_t item, uint32_t cdepth, int whole,
                                          uint32_t total_blocks, uint32_t num_slots,
                                          uint32_t level, const uint32_t* __restrict__ goff,
                                          const uint32_t* __restrict__ blk_off,
                                          const uint32_t* __restrict__ tfirst,
                                          const uint32_t* __restrict__ tlast) {
  TcItem it;
  const uint32_t K = 1u << cdepth;
  const uint32_t cols = whole ? 1u : 2u * K;
  const uint32_t grp = item / (kTcGroup * cols);
  const uint32_t r = item - grp * (kTcGroup * cols);
  const uint32_t gsize = min(uint32_t(kTcGroup), total_blocks - grp * kTcGroup);
  const uint32_t blk = grp * kTcGroup + r % gsize;
  const uint32_t col = r / gsize;
  it.side = whole ? 0u : col >> cdepth;
  it.kk = whole ? 0u : col & (K - 1);
  uint32_t lo_ = 0, hi_ = num_slots;
  while (hi_ - lo_ > 1) {
    const uint32_t mid = (lo_ + hi_) >> 1;
    if (blk_off[mid] <= blk) lo_ = mid; else hi_ = mid;
  }
  it.g = lo_;
  it.e0 = goff[it.g] + (blk - blk_off[it.g]) * kTcM;
  it.e1 = min(it.e0 + uint32_t(kTcM), goff[it.g + 1]);
  const uint32_t lc = level + 1 + cdepth;
  const uint64_t h = whole ? ((1ull << level) - 1) + it.g
                           : ((1ull << lc) - 1) + ((uint64_t(2 * it.g + it.side)) << cdepth) + it.kk;
  it.cf = tfirst[h];
  it.cl = tlast[h];
  it.ntiles = (it.cl - it.cf + kTcN - 1) / kTcN;
  return it;
}

// Persistent: one CTA per SM walks the items blockIdx.x, + gridDim.x, ...;
// the smem ring, the TMEM double buffer and their barrier phases run on
// across items, so the next item's loads and MMAs overlap this item's
// epilogue (one CTA per item left a pipeline fill and drain per ~4 N-tiles).
template <int FAM>
__global__ void __launch_bounds__(kTcThreads, 1)
    kde_tc_kernel(const __grid_constant__ CUtensorMap map_hi,
                  const __grid_constant__ CUtensorMap map_lo,
                  const __grid_constant__ CUtensorMap gmap_hi,
                  const __grid_constant__ CUtensorMap gmap_lo, const float* __restrict__ qhi_g,
                  const float* __restrict__ qlo_g, const float* __restrict__ norm,
                  uint32_t d_pad, const uint32_t* __restrict__ eq,
                  const uint32_t* __restrict__ goff, const uint32_t* __restrict__ blk_off,
                  uint32_t num_slots, uint32_t total_blocks, uint32_t level, uint32_t cdepth,
                  uint32_t sdepth,
                  const uint32_t* __restrict__ tfirst, const uint32_t* __restrict__ tlast,
                  float scale, double* __restrict__ partials, int terms, int whole,
                  uint32_t items, uint32_t* __restrict__ next_item) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTcStages * kStageBytes);
  uint64_t* full = bars;                   // [kTcStages]
  uint64_t* empty = bars + kTcStages;      // [kTcStages]
  uint64_t* tfull = bars + 2 * kTcStages;  // [2]
  uint64_t* tempty = tfull + 2;            // [2]
  uint64_t* ring_full = tempty + 2;           // [kRing]
  uint64_t* ring_empty = ring_full + kRing;   // [kRing]
  uint32_t* ring = reinterpret_cast<uint32_t*>(ring_empty + kRing);  // [kRing]
  uint32_t* tmem_slot = ring + kRing;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t kblocks = d_pad / kTcKB;
  // Items are handed out in order by a global counter (the producer thread
  // fetches, the other roles read them from a small smem ring): the active
  // items of all CTAs stay a compact window, which is what lets them share
  // query and source tiles in L2 (a static stride let CTAs drift apart:
  // 4x the DRAM reads).
  auto next = [&](uint32_t k) -> uint32_t {  // consumers: k-th item of this CTA
    const uint32_t slot = k % kRing;
    mbar_wait(&ring_full[slot], (k / kRing) & 1u);
    return ring[slot];
  };
  auto release = [&](uint32_t k) { mbar_arrive(&ring_empty[k % kRing]); };
  auto item_at = [&](uint32_t item) {
    return tc_item(item, cdepth, whole, total_blocks, num_slots, level, goff, blk_off, tfirst,
                   tlast);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 2);  // producer (sources) + gather warp (queries)
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 128);
    }
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&ring_full[r], 1);
      mbar_init(&ring_empty[r], kRingReaders);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&gmap_hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&gmap_lo)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer: source tiles ------------------------------------
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t slot = k % kRing;
        mbar_wait(&ring_empty[slot], ((k / kRing) & 1u) ^ 1u);
        const uint32_t item = atomicAdd(next_item, 1u);
        ring[slot] = item;
        mbar_arrive(&ring_full[slot]);  // release: the ring write is visible
        if (item >= items) break;
        const TcItem w = item_at(item);
        const uint32_t total = w.ntiles * kblocks;
        for (uint32_t j = 0; j < total; ++j, ++it) {
          const uint32_t s = it % kTcStages, ph = (it / kTcStages) & 1u;
          const uint32_t tile = j / kblocks, kb = j % kblocks;
          mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* st = smem + s * kStageBytes;
          mbar_arrive_expect_tx(&full[s], 2 * kTileBytes);
          const int row = int(w.cf + tile * kTcN), col = int(kb * kTcKB);
          tma_load_2d(st + 2 * kTileBytes, &map_hi, &full[s], col, row);
          tma_load_2d(st + 3 * kTileBytes, &map_lo, &full[s], col, row);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer --------------------------------------------------------
    if (lane == 0) {
      uint32_t it = 0, tg = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t item = next(k);
        release(k);
        if (item >= items) break;
        const TcItem w = item_at(item);
        for (uint32_t tile = 0; tile < w.ntiles; ++tile, ++tg) {
          const uint32_t buf = tg & 1u;
          mbar_wait(&tempty[buf], ((tg >> 1) & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t tacc = tmem_base + buf * kTcN;
          for (uint32_t kb = 0; kb < kblocks; ++kb, ++it) {
            const uint32_t s = it % kTcStages, ph = (it / kTcStages) & 1u;
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t base = smem_u32(smem + s * kStageBytes);
#pragma unroll
            for (int ks = 0; ks < kTcKB / 8; ++ks) {
              const uint32_t off = ks * 32;  // 8 tf32 = 32 bytes along K
              const uint64_t a_hi = sw128_desc(base + off);
              const uint64_t a_lo = sw128_desc(base + kTileBytes + off);
              const uint64_t b_hi = sw128_desc(base + 2 * kTileBytes + off);
              const uint64_t b_lo = sw128_desc(base + 3 * kTileBytes + off);
              mma_tf32(tacc, a_hi, b_hi, (kb | ks) != 0);
              if (terms & 1) mma_tf32(tacc, a_hi, b_lo, 1);
              if (terms & 2) mma_tf32(tacc, a_lo, b_hi, 1);
            }
            mma_commit(&empty[s]);
          }
          mma_commit(&tfull[buf]);
        }
      }
    }
  } else if (warp < 4) {
    // ---- query tiles (warp 2): one TMA box when the block's queries are
    // consecutive (always at the root of a full build), else TMA gather4 —
    // lane l brings rows 4l..4l+3 ----------------------------------------
    if (warp == 2) {
      uint32_t it = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t item = next(k);
        __syncwarp();
        if (lane == 0) release(k);
        if (item >= items) break;
        const TcItem w = item_at(item);
        const uint32_t total = w.ntiles * kblocks;
        int rows[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t e = w.e0 + 4 * lane + j;
          rows[j] = int(eq[e < w.e1 ? e : w.e0]);
        }
        // queries of a block are sorted and distinct; consecutive point
        // indices make the tile a plain box
        const uint32_t q0 = eq[w.e0];
        const bool contig = eq[w.e1 - 1] == q0 + (w.e1 - 1 - w.e0);
        for (uint32_t j = 0; j < total; ++j, ++it) {
          const uint32_t s = it % kTcStages, ph = (it / kTcStages) & 1u;
          const int col = int((j % kblocks) * kTcKB);
          mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* st = smem + s * kStageBytes;
          if (lane == 0) mbar_arrive_expect_tx(&full[s], 2 * kTileBytes);
          __syncwarp();
          if (contig) {
            if (lane == 0) {
              tma_load_2d(st, &map_hi, &full[s], col, int(q0));
              tma_load_2d(st + kTileBytes, &map_lo, &full[s], col, int(q0));
            }
          } else {
            tma_gather4(st + lane * 512, &gmap_hi, &full[s], col, rows[0], rows[1], rows[2],
                        rows[3]);
            tma_gather4(st + kTileBytes + lane * 512, &gmap_lo, &full[s], col, rows[0], rows[1],
                        rows[2], rows[3]);
          }
        }
      }
    }
  } else {
    // ---- epilogue (128 threads = TMEM lanes) -------------------------------
    // Columns are split at the sub-chunk boundaries (tree descendants
    // sdepth levels below the child); one fp64 partial per sub-chunk.
    const uint32_t ew = warp & 3;               // TMEM lane group of this warp
    const uint32_t row = ew * 32 + lane;        // accumulator row = entry
    uint32_t tg = 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t item = next(k);
      __syncwarp();
      if (lane == 0) release(k);
      if (item >= items) break;
      const TcItem w = item_at(item);
      const uint32_t e = w.e0 + row;
      const float qn = norm[eq[e < w.e1 ? e : w.e0]];
      const uint32_t nsub = 1u << (sdepth - cdepth);
      const uint64_t hs = ((1ull << (level + 1 + sdepth)) - 1) +
                          ((uint64_t(2 * w.g + w.side)) << sdepth) + uint64_t(w.kk) * nsub;
      double* prow =
          partials + (size_t(e) << (sdepth + 1)) + (w.side << sdepth) + w.kk * nsub;
      uint32_t b = 0, bend = tlast[hs];
      double racc = 0.0;
      for (uint32_t tile = 0; tile < w.ntiles; ++tile, ++tg) {
        const uint32_t buf = tg & 1u;
        mbar_wait(&tfull[buf], (tg >> 1) & 1u);
        tc_fence_after();
        const uint32_t n0 = w.cf + tile * kTcN;
        const uint32_t valid = min(uint32_t(kTcN), w.cl - n0);
        float acc = 0.f;
#pragma unroll
        for (int chunk = 0; chunk < kTcN / 32; ++chunk) {
          float v[32];
          tmem_ld32(tmem_base + ((ew * 32) << 16) + buf * kTcN + chunk * 32, v);
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const uint32_t col = chunk * 32 + k;
            if (col < valid) {  // uniform across the warp
              while (n0 + col >= bend) {  // next sub-chunk (uniform)
                if (e < w.e1) prow[b] = racc + acc;
                racc = 0.0;
                acc = 0.f;
                bend = tlast[hs + (++b)];
              }
              const float xn = __ldg(norm + n0 + col);
              float d2 = fmaxf(fmaf(-2.f, v[k], qn + xn), 0.f);
              if constexpr (FAM == 1) d2 = sqrtf(d2);
              acc += ex2_approx(-scale * d2);
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);
        racc += acc;
      }
      if (e < w.e1) prow[b] = racc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// ---- symmetric root (level 0 of a full build, d >= kTcMinDim) ------------
// Every pair once: the points are cut into 128-point tiles on a fixed grid
// and each tile pair I <= J is evaluated once. A work item is (query tile I,
// super-tiles [S0, S1)), super-tile S = source tiles {2S, 2S + 1}: each MMA
// is 128 x 256 with 16-wide K blocks in 64-byte-swizzled rows, so a 48 KiB
// stage carries twice the MMA work of a 128-wide 64 KiB one and four stages
// fit. Per half of a super-tile the pairing rule picks full (rows and
// columns), diagonal (rows only: the diagonal tile's rows hold both
// directions) or skipped (J < I: the pair belongs to the item of tile J).
// The epilogue of each accumulator yields
//   * row sums (I's points over the sources), split at the sources' bucket
//     boundaries — warps 4-7, and
//   * column sums (the full halves' points over I's points), split at I's
//     bucket boundaries — warps 8-11: per warp a masked butterfly
//     transpose-reduction for each bucket among its 32 rows, then the four
//     warps' partials added in warp order through shared memory.
// Both groups read the accumulator from TMEM and evaluate the same
// exponentials (same instructions, same bits), so the column side's
// cross-lane reductions run beside the row side. The epilogue bodies are
// kept compact (exponentials, then predicated per-bucket sums): a
// per-column boundary loop unrolled 32x made the code large enough to evict
// the MMA warp's instructions (root 19.6 -> 15.4 ms at C5).
// Buckets are the root row's tree nodes at depth rl (16..128 points, so a
// bucket meets at most two 128-point tiles): a bucket complete within an
// item is stored, the two parts of a straddling bucket are added to the
// zeroed row with fp64 atomics — two addends, so the sum is the same in
// either order. Every value depends on its tiles only: deterministic, and
// it halves the tensor-core work of the n^2 pass.
#ifndef FSGG_TC_SYM_GI
#define FSGG_TC_SYM_GI 32
#endif
constexpr uint32_t kTcSymGI = FSGG_TC_SYM_GI;   // tiles per side of an L2 block of items
constexpr int kTcSymMaxSegW = 3;    // buckets among a warp's 32 rows (>= 16 points each)
constexpr int kTcSymThreads = 384;  // the one-sided kernel's 8 roles + 4 column warps
constexpr int kTcSymRingReaders = 10;  // MMA thread, query warp, 8 epilogue warps

__device__ __forceinline__ void flush_bucket(double* __restrict__ prow, uint32_t b, float acc,
                                             bool whole) {
  if (whole)
    prow[b] = double(acc);
  else
    atomicAdd(prow + b, double(acc));
}

constexpr int kS2N = 256;                  // sources per MMA (two tiles)
constexpr int kS2KB = 16;                  // fp32 per K-block: one 64-byte row
constexpr int kS2Stages = 4;
constexpr int kS2ATile = kTcM * kS2KB * 4;    // 8 KiB (A hi or lo)
constexpr int kS2BTile = kS2N * kS2KB * 4;    // 16 KiB (B hi or lo)
constexpr int kS2Stage = 2 * kS2ATile + 2 * kS2BTile;  // 48 KiB
constexpr uint32_t kS2TmemCols = 512;      // 2 x 256-column accumulators
constexpr uint32_t kS2R = 4;               // super-tiles per work item
constexpr int kSmemS2Bytes = kS2Stages * kS2Stage + 1024 + 4 * 3 * kS2N * 4 + 16 + 1024;

// K-major, 64-byte-swizzled shared-memory matrix descriptor: SBO = 512 B
// between 8-row groups, layout type SWIZZLE_64B = 4.
__device__ __forceinline__ uint64_t sw64_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fff);
  d |= uint64_t(1) << 16;
  d |= uint64_t(512 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;
  return d;
}
constexpr uint32_t kIdescS2 = (1u << 4) | (2u << 7) | (2u << 10) |
                              (uint32_t(kS2N >> 3) << 17) | (uint32_t(kTcM >> 4) << 24);
__device__ __forceinline__ void mma_tf32_n256(uint32_t tmem_d, uint64_t da, uint64_t db,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdescS2), "r"(accumulate)
      : "memory");
}

// half mode of super-tile S for query tile I: 0 skipped, 1 diagonal, 2 full
__device__ __forceinline__ uint32_t s2_mode(uint32_t I, uint32_t J, uint32_t T) {
  if (J >= T || J < I) return 0u;
  return J == I ? 1u : 2u;
}

template <int FAM>
__global__ void __launch_bounds__(kTcSymThreads, 1)
    kde_tc_sym256_kernel(const __grid_constant__ CUtensorMap amap_hi,
                         const __grid_constant__ CUtensorMap amap_lo,
                         const __grid_constant__ CUtensorMap bmap_hi,
                         const __grid_constant__ CUtensorMap bmap_lo,
                         const float* __restrict__ norm, uint32_t d_pad, uint32_t n,
                         const uint32_t* __restrict__ sitems, uint32_t items,
                         uint32_t* __restrict__ next_item, const uint32_t* __restrict__ tile_b0,
                         const uint32_t* __restrict__ bfirst, const uint32_t* __restrict__ blast,
                         uint32_t rl, float scale, double* __restrict__ partials, int terms) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kS2Stages * kS2Stage);
  uint64_t* full = bars;
  uint64_t* empty = bars + kS2Stages;
  uint64_t* tfull = bars + 2 * kS2Stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* ring_full = tempty + 2;
  uint64_t* ring_empty = ring_full + kRing;
  uint32_t* ring = reinterpret_cast<uint32_t*>(ring_empty + kRing);
  uint32_t* tmem_slot = ring + kRing;
  float* colpart = reinterpret_cast<float*>(smem + kS2Stages * kS2Stage + 1024);
  uint32_t* wfirst = reinterpret_cast<uint32_t*>(colpart + 4 * kTcSymMaxSegW * kS2N);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t kblocks = d_pad / kS2KB;
  const uint32_t T = (n + kTcM - 1) / kTcM;
  auto next = [&](uint32_t k) -> uint32_t {
    const uint32_t slot = k % kRing;
    mbar_wait(&ring_full[slot], (k / kRing) & 1u);
    return ring[slot];
  };
  auto release = [&](uint32_t k) { mbar_arrive(&ring_empty[k % kRing]); };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kS2Stages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256);
    }
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&ring_full[r], 1);
      mbar_init(&ring_empty[r], kTcSymRingReaders);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kS2TmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap_hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&amap_lo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap_hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&bmap_lo)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---- TMA producer: 256-row source super-tiles --------------------------
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t slot = k % kRing;
        mbar_wait(&ring_empty[slot], ((k / kRing) & 1u) ^ 1u);
        const uint32_t item = atomicAdd(next_item, 1u);
        ring[slot] = item;
        mbar_arrive(&ring_full[slot]);
        if (item >= items) break;
        const uint32_t S0 = sitems[3 * item + 1], S1 = sitems[3 * item + 2];
        const uint32_t total = (S1 - S0) * kblocks;
        for (uint32_t j = 0; j < total; ++j, ++it) {
          const uint32_t s = it % kS2Stages, ph = (it / kS2Stages) & 1u;
          const uint32_t st_ = j / kblocks, kb = j % kblocks;
          mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* st = smem + s * kS2Stage;
          mbar_arrive_expect_tx(&full[s], 2 * kS2BTile);
          const int row = int((S0 + st_) * kS2N), col = int(kb * kS2KB);
          tma_load_2d(st + 2 * kS2ATile, &bmap_hi, &full[s], col, row);
          tma_load_2d(st + 2 * kS2ATile + kS2BTile, &bmap_lo, &full[s], col, row);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ----------------------------------------------------------
    if (lane == 0) {
      uint32_t it = 0, tg = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t item = next(k);
        release(k);
        if (item >= items) break;
        const uint32_t nt = sitems[3 * item + 2] - sitems[3 * item + 1];
        for (uint32_t tile = 0; tile < nt; ++tile, ++tg) {
          const uint32_t buf = tg & 1u;
          mbar_wait(&tempty[buf], ((tg >> 1) & 1u) ^ 1u);
          tc_fence_after();
          const uint32_t tacc = tmem_base + buf * kS2N;
          for (uint32_t kb = 0; kb < kblocks; ++kb, ++it) {
            const uint32_t s = it % kS2Stages, ph = (it / kS2Stages) & 1u;
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t base = smem_u32(smem + s * kS2Stage);
#pragma unroll
            for (int ks = 0; ks < kS2KB / 8; ++ks) {
              const uint32_t off = ks * 32;
              const uint64_t a_hi = sw64_desc(base + off);
              const uint64_t a_lo = sw64_desc(base + kS2ATile + off);
              const uint64_t b_hi = sw64_desc(base + 2 * kS2ATile + off);
              const uint64_t b_lo = sw64_desc(base + 2 * kS2ATile + kS2BTile + off);
              mma_tf32_n256(tacc, a_hi, b_hi, (kb | ks) != 0);
              if (terms & 1) mma_tf32_n256(tacc, a_hi, b_lo, 1);
              if (terms & 2) mma_tf32_n256(tacc, a_lo, b_hi, 1);
            }
            mma_commit(&empty[s]);
          }
          mma_commit(&tfull[buf]);
        }
      }
    }
  } else if (warp < 4) {
    // ---- query tile I (one TMA box per K-block and super-tile) -------------
    if (warp == 2) {
      uint32_t it = 0;
      for (uint32_t k = 0;; ++k) {
        const uint32_t item = next(k);
        __syncwarp();
        if (lane == 0) release(k);
        if (item >= items) break;
        const uint32_t I = sitems[3 * item];
        const uint32_t total = (sitems[3 * item + 2] - sitems[3 * item + 1]) * kblocks;
        for (uint32_t j = 0; j < total; ++j, ++it) {
          const uint32_t s = it % kS2Stages, ph = (it / kS2Stages) & 1u;
          const int col = int((j % kblocks) * kS2KB);
          mbar_wait(&empty[s], ph ^ 1u);
          unsigned char* st = smem + s * kS2Stage;
          if (lane == 0) {
            mbar_arrive_expect_tx(&full[s], 2 * kS2ATile);
            tma_load_2d(st, &amap_hi, &full[s], col, int(I * kTcM));
            tma_load_2d(st + kS2ATile, &amap_lo, &full[s], col, int(I * kTcM));
          }
          __syncwarp();
        }
      }
    }
  } else if (warp < 8) {
    // ---- row side (warps 4-7) ---------------------------------------------
    const uint32_t ew = warp & 3;
    const uint32_t row = ew * 32 + lane;
    uint32_t tg = 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t item = next(k);
      __syncwarp();
      if (lane == 0) release(k);
      if (item >= items) break;
      const uint32_t I = sitems[3 * item], S0 = sitems[3 * item + 1],
                     S1 = sitems[3 * item + 2];
      const uint32_t q = I * kTcM + row;
      const bool qv = q < n;
      const float qn = norm[qv ? q : n - 1];
      double* prow = partials + (size_t(q) << rl);
      for (uint32_t S = S0; S < S1; ++S, ++tg) {
        const uint32_t buf = tg & 1u;
        mbar_wait(&tfull[buf], (tg >> 1) & 1u);
        tc_fence_after();
        const uint32_t n0 = S * kS2N;
        // row-valid columns: [c0, c1) (half 0 skipped when its tile precedes I)
        const uint32_t c0 = s2_mode(I, 2 * S, T) ? 0u : uint32_t(kTcN);
        const uint32_t c1 = min(uint32_t(kS2N), n - n0);
        uint32_t b = tile_b0[(n0 + c0) / kTcM], bend = blast[b];
        float acc = 0.f;
        // compact body: the chunk's exponentials first (no branches), then
        // its bucket segments (<= 3, bucket >= 16 points) as predicated sums
        // — a per-column boundary loop unrolled 32x made the epilogue code
        // large enough to evict the MMA warp's instructions
#pragma unroll 1
        for (int chunk = int(c0 / 32); chunk < kS2N / 32; ++chunk) {
          float v[32];
          tmem_ld32(tmem_base + ((ew * 32) << 16) + buf * kS2N + chunk * 32, v);
          const uint32_t cb = chunk * 32;
#pragma unroll
          for (int kk = 0; kk < 32; ++kk) {
            const float xn = __ldg(norm + n0 + min(cb + kk, c1 - 1));
            float d2 = fmaxf(fmaf(-2.f, v[kk], qn + xn), 0.f);
            if constexpr (FAM == 1) d2 = sqrtf(d2);
            v[kk] = cb + kk < c1 ? ex2_approx(-scale * d2) : 0.f;
          }
          uint32_t lo = cb;  // this chunk's columns [lo, min(cb + 32, c1))
          const uint32_t hi = min(cb + 32u, c1);
          while (lo < hi) {  // uniform
            const uint32_t end = min(hi, bend - n0);
#pragma unroll
            for (int kk = 0; kk < 32; ++kk)
              acc += (cb + kk >= lo && cb + kk < end) ? v[kk] : 0.f;
            lo = end;
            if (lo == bend - n0 && lo < c1) {  // bucket complete
              if (qv) flush_bucket(prow, b, acc, bfirst[b] >= n0 + c0);
              acc = 0.f;
              bend = blast[++b];
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);
        if (qv) flush_bucket(prow, b, acc, bfirst[b] >= n0 + c0 && bend <= n0 + c1);
      }
    }
  } else {
    // ---- column side (warps 8-11): the full halves' points over I's buckets
    const uint32_t ew = warp & 3;
    const uint32_t row = ew * 32 + lane;
    uint32_t tg = 0;
    for (uint32_t k = 0;; ++k) {
      const uint32_t item = next(k);
      __syncwarp();
      if (lane == 0) release(k);
      if (item >= items) break;
      const uint32_t I = sitems[3 * item], S0 = sitems[3 * item + 1],
                     S1 = sitems[3 * item + 2];
      const uint32_t q0 = I * kTcM, q = q0 + row;
      const bool qv = q < n;
      const uint32_t qend = min(q0 + uint32_t(kTcM), n);
      const float qn = norm[qv ? q : n - 1];
      uint32_t bq = tile_b0[I];
      const uint32_t qq = qv ? q : n - 1;
      while (blast[bq] <= qq) ++bq;
      const uint32_t bw = __shfl_sync(0xffffffffu, bq, 0);
      const uint32_t nsw = __shfl_sync(0xffffffffu, bq, 31) - bw + 1;
      const uint32_t bI0 = tile_b0[I];
      uint32_t bIend = bI0;
      while (bIend < (1u << rl) && bfirst[bIend] < qend) ++bIend;
      for (uint32_t S = S0; S < S1; ++S, ++tg) {
        const uint32_t buf = tg & 1u;
        const uint32_t m0 = s2_mode(I, 2 * S, T), m1 = s2_mode(I, 2 * S + 1, T);
        mbar_wait(&tfull[buf], (tg >> 1) & 1u);
        tc_fence_after();
        const uint32_t n0 = S * kS2N;
        const uint32_t c1 = min(uint32_t(kS2N), n - n0);
        if (m0 == 2 || m1 == 2) {
#pragma unroll 1
          for (int chunk = 0; chunk < kS2N / 32; ++chunk) {
            if ((chunk < 4 ? m0 : m1) != 2) continue;  // uniform
            float v[32];
            tmem_ld32(tmem_base + ((ew * 32) << 16) + buf * kS2N + chunk * 32, v);
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) {
              const uint32_t col = chunk * 32 + kk;
              float e = 0.f;
              if (col < c1) {
                const float xn = __ldg(norm + n0 + col);
                float d2 = fmaxf(fmaf(-2.f, v[kk], qn + xn), 0.f);
                if constexpr (FAM == 1) d2 = sqrtf(d2);
                e = ex2_approx(-scale * d2);
              }
              v[kk] = qv ? e : 0.f;
            }
            for (uint32_t sgm = 0; sgm < nsw; ++sgm) {
              float c[32];
              const bool mine = bq == bw + sgm;
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) c[kk] = mine ? v[kk] : 0.f;
#pragma unroll
              for (int st = 16; st >= 1; st >>= 1) {
                const bool up = (lane & st) != 0;
#pragma unroll
                for (int i = 0; i < st; ++i) {
                  const float keep = up ? c[i + st] : c[i];
                  const float send = up ? c[i] : c[i + st];
                  c[i] = keep + __shfl_xor_sync(0xffffffffu, send, st);
                }
              }
              colpart[(ew * kTcSymMaxSegW + sgm) * kS2N + chunk * 32 + lane] = c[0];
            }
          }
        }
        tc_fence_before();
        mbar_arrive(&tempty[buf]);
        if (!(m0 == 2 || m1 == 2)) continue;
        if (lane == 0) wfirst[ew] = bw;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // threads: columns row and row + 128 of the full halves
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t ct = row + 128u * h;
          if ((h ? m1 : m0) != 2 || ct >= c1) continue;
          double* xrow = partials + (size_t(n0 + ct) << rl);
          for (uint32_t bb = bI0; bb < bIend; ++bb) {
            const uint32_t lo = bfirst[bb], hi = blast[bb];
            float sum = 0.f;
#pragma unroll
            for (uint32_t w = 0; w < 4; ++w) {
              const uint32_t r0 = q0 + 32 * w;
              const uint32_t r1 = min(r0 + 32, qend);
              if (r0 < qend && hi > r0 && lo < r1)
                sum += colpart[(w * kTcSymMaxSegW + (bb - wfirst[w])) * kS2N + ct];
            }
            flush_bucket(xrow, bb, sum, lo >= q0 && hi <= qend);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kS2TmemCols)
                 : "memory");
  }
}

// ---- host: tensor maps -------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw DeviceError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

void make_map(CUtensorMap* map, float* base, uint32_t n, uint32_t d_pad, uint32_t box_rows,
              uint32_t box_cols = kTcKB,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  const cuuint64_t dims[2] = {d_pad, n};
  const cuuint64_t strides[1] = {cuuint64_t(d_pad) * 4};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw DeviceError("cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

struct TcState {
  uint32_t d_pad = 0;
  CUtensorMap map_hi, map_lo;    // 128-row boxes (sources, contiguous queries)
  CUtensorMap gmap_hi, gmap_lo;  // 1-row boxes for tile::gather4
  // symmetric 256-wide root: 16-wide K blocks, 64-byte swizzle
  CUtensorMap amap_hi, amap_lo;  // 128-row query boxes
  CUtensorMap bmap_hi, bmap_lo;  // 256-row source boxes
};

TcState& tc_state(Dataset& ds) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (!ds.tc_ready) {
    const uint32_t d_pad = (ds.d + kTcKB - 1) / kTcKB * kTcKB;
    DevBuf& hi = ds.buf("tc.hi", size_t(ds.n) * d_pad * 4);
    DevBuf& lo = ds.buf("tc.lo", size_t(ds.n) * d_pad * 4);
    DevBuf& nrm = ds.buf("tc.norm", size_t(ds.n) * 4);
    DevBuf& mean = ds.buf("tc.mean", size_t(ds.d) * 4);
    tc_mean_kernel<<<ds.d, 256, 0, ds.stream>>>(ds.pts.as<float>(), ds.n, ds.d,
                                                mean.as<float>());
    FSGG_LAUNCH_CHECK();
    tc_split_kernel<<<ds.n, 256, 0, ds.stream>>>(ds.pts.as<float>(), ds.n, ds.d, d_pad,
                                                 mean.as<float>(), hi.as<float>(),
                                                 lo.as<float>(), nrm.as<float>());
    FSGG_LAUNCH_CHECK();
    ds.launches += 2;
    auto* st = reinterpret_cast<TcState*>(ds.tc_blob);
    st->d_pad = d_pad;
    make_map(&st->map_hi, hi.as<float>(), ds.n, d_pad, kTcN);
    make_map(&st->map_lo, lo.as<float>(), ds.n, d_pad, kTcN);
    make_map(&st->gmap_hi, hi.as<float>(), ds.n, d_pad, 1);
    make_map(&st->gmap_lo, lo.as<float>(), ds.n, d_pad, 1);
    make_map(&st->amap_hi, hi.as<float>(), ds.n, d_pad, kTcM, kS2KB, CU_TENSOR_MAP_SWIZZLE_64B);
    make_map(&st->amap_lo, lo.as<float>(), ds.n, d_pad, kTcM, kS2KB, CU_TENSOR_MAP_SWIZZLE_64B);
    make_map(&st->bmap_hi, hi.as<float>(), ds.n, d_pad, kS2N, kS2KB, CU_TENSOR_MAP_SWIZZLE_64B);
    make_map(&st->bmap_lo, lo.as<float>(), ds.n, d_pad, kS2N, kS2KB, CU_TENSOR_MAP_SWIZZLE_64B);
    ds.tc_ready = true;
  }
  return *reinterpret_cast<TcState*>(ds.tc_blob);
}

}  // namespace

static_assert(sizeof(TcState) <= sizeof(Dataset::tc_blob), "tc_blob too small");

// FSGG_TC_TERMS (debug): bit 0 = Qhi*Xlo, bit 1 = Qlo*Xhi (default 3 = 3xTF32)
int tc_terms() {
  static const int v = [] {
    const char* e = std::getenv("FSGG_TC_TERMS");
    return e ? std::atoi(e) : 3;
  }();
  return v;
}

bool kde_tc_supported(const Dataset& ds, int family) {
  static const bool enabled = [] {
    const char* e = std::getenv("FSGG_TC");
    return !(e && e[0] == '0');
  }();
  return enabled && ds.d >= kTcMinDim && family != 2;
}

// Symmetric root (kde_tc_sym256_kernel) for a full build's level 0: partials
// (n rows of 2^rl fp64 buckets) zeroed and filled; returns false (nothing
// launched) when the layout does not fit it (a query shard, buckets outside
// 16..128 points) or FSGG_TC_SYM=0.
bool kde_tc_root_symmetric(Dataset& ds, const KernelSpec& ks, const LevelView& lv, uint32_t rl,
                           double* partials, uint64_t* performed) {
  const char* env = std::getenv("FSGG_TC_SYM");  // read per call: tests toggle it
  const bool enabled = !(env && env[0] == '0');
  const uint32_t n = ds.n;
  if (!enabled || lv.level != 0 || lv.dE || lv.qbase != 0 || lv.num_entries != n || rl == 0 ||
      rl > 16 || rl > ds.tree.depth)
    return false;
  const TreeTable& t = ds.tree;
  cudaStream_t s = ds.stream;
  const uint32_t nb = 1u << rl;
  const uint64_t hb = (uint64_t(1) << rl) - 1;
  std::vector<uint32_t> bf(nb), bl(nb);
  FSGG_CUDA(cudaMemcpyAsync(bf.data(), t.first.as<uint32_t>() + hb, size_t(nb) * 4,
                            cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaMemcpyAsync(bl.data(), t.last.as<uint32_t>() + hb, size_t(nb) * 4,
                            cudaMemcpyDeviceToHost, s));
  FSGG_CUDA(cudaStreamSynchronize(s));
  for (uint32_t b = 0; b < nb; ++b) {
    const uint32_t sz = bl[b] - bf[b];
    if (sz < 16 || sz > uint32_t(kTcN)) return false;  // segments per warp / per tile
  }
  TcState& st = tc_state(ds);
  const uint32_t T = (n + kTcM - 1) / kTcM;
  std::vector<uint32_t> b0(T);
  for (uint32_t tt = 0, b = 0; tt < T; ++tt) {
    while (bl[b] <= tt * uint32_t(kTcM)) ++b;
    b0[tt] = b;
  }
  // items (I, J0, J1), J0 >= I, in blocks of kTcSymGI x kTcSymGI tiles: the
  // items of one block (about one wave of CTAs) read kTcSymGI query and
  // kTcSymGI source tiles (2 x 26 MB at C5), which stay in L2 (an order by
  // query tile alone read 81 GB from DRAM per launch). The 256-wide kernel
  // takes (I, S0, S1) over super-tiles S = {2S, 2S + 1}, S >= I / 2.
  std::vector<uint32_t> it;
  uint64_t perf = 0;
  const uint32_t TS = (T + 1) / 2;
  for (uint32_t a0 = 0; a0 < T; a0 += kTcSymGI) {
    const uint32_t a1 = std::min(T, a0 + kTcSymGI);
    for (uint32_t c0 = a0 / 2; c0 < TS; c0 += kTcSymGI / 2) {
      const uint32_t c1 = std::min(TS, c0 + kTcSymGI / 2);
      for (uint32_t I = a0; I < a1; ++I)
        for (uint32_t S0 = std::max(I / 2, c0); S0 < c1; S0 += kS2R) {
          it.push_back(I);
          it.push_back(S0);
          it.push_back(std::min(c1, S0 + kS2R));
        }
    }
  }
  for (uint32_t I = 0; I < T; ++I) {
    const uint64_t rows = std::min<uint64_t>(kTcM, n - uint64_t(I) * kTcM);
    perf += rows * (uint64_t(n) - uint64_t(I) * kTcM);
  }
  const uint32_t items = uint32_t(it.size() / 3);
  DevBuf& ditems = ds.buf("tc.sym_items", it.size() * 4);
  DevBuf& db0 = ds.buf("tc.sym_b0", size_t(T) * 4);
  FSGG_CUDA(cudaMemcpyAsync(ditems.as<void>(), it.data(), it.size() * 4, cudaMemcpyHostToDevice,
                            s));
  FSGG_CUDA(cudaMemcpyAsync(db0.as<void>(), b0.data(), size_t(T) * 4, cudaMemcpyHostToDevice, s));
  FSGG_CUDA(cudaMemsetAsync(partials, 0, (size_t(n) << rl) * 8, s));
  static bool attr[64] = {};
  if (ds.device < 64 && !attr[ds.device]) {
    FSGG_CUDA(cudaFuncSetAttribute(kde_tc_sym256_kernel<0>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemS2Bytes));
    FSGG_CUDA(cudaFuncSetAttribute(kde_tc_sym256_kernel<1>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemS2Bytes));
    attr[ds.device] = true;
  }
  DevBuf& counter = ds.buf("tc.next_item", 8);
  FSGG_CUDA(cudaMemsetAsync(counter.as<void>(), 0, 4, s));
  const uint32_t grid = std::min<uint32_t>(items, uint32_t(ds.num_sms));
  auto kern = ks.family == 1 ? kde_tc_sym256_kernel<1> : kde_tc_sym256_kernel<0>;
  kern<<<grid, kTcSymThreads, kSmemS2Bytes, s>>>(
      st.amap_hi, st.amap_lo, st.bmap_hi, st.bmap_lo, ds.buf("tc.norm", 8).as<float>(),
      st.d_pad, n, ditems.as<uint32_t>(), items, counter.as<uint32_t>(), db0.as<uint32_t>(),
      t.first.as<uint32_t>() + hb, t.last.as<uint32_t>() + hb, rl, ks.scale, partials,
      tc_terms());
  FSGG_LAUNCH_CHECK();
  ds.launches++;
  if (performed) *performed = perf;
  return true;
}

void kde_tc_tiled(Dataset& ds, const KernelSpec& ks, const LevelView& lv,
                  const uint32_t* blk_off, uint32_t cdepth, uint32_t sdepth, uint64_t items,
                  double* partials) {
  TcState& st = tc_state(ds);
  const TreeTable& t = ds.tree;
  static bool attr[64] = {};
  auto kern = ks.family == 1 ? kde_tc_kernel<1> : kde_tc_kernel<0>;
  if (ds.device < 64 && !attr[ds.device]) {
    FSGG_CUDA(cudaFuncSetAttribute(kde_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSmemBytes));
    FSGG_CUDA(cudaFuncSetAttribute(kde_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kSmemBytes));
    attr[ds.device] = true;
  }
  const uint32_t s_max = uint32_t((uint64_t(ds.n) + (1ull << lv.level) - 1) >> lv.level);
  const int whole = cdepth == 0 && s_max <= uint32_t(kTcN) ? 1 : 0;
  const uint64_t nitems = whole ? items / 2 : items;
  const uint32_t grid = uint32_t(std::min<uint64_t>(nitems, uint64_t(ds.num_sms)));
  DevBuf& counter = ds.buf("tc.next_item", 8);
  FSGG_CUDA(cudaMemsetAsync(counter.as<void>(), 0, 4, ds.stream));
  kern<<<dim3(grid), kTcThreads, kSmemBytes, ds.stream>>>(
      st.map_hi, st.map_lo, st.gmap_hi, st.gmap_lo, ds.buf("tc.hi", 8).as<float>(), ds.buf("tc.lo", 8).as<float>(),
      ds.buf("tc.norm", 8).as<float>(), st.d_pad, lv.eq, lv.goff, blk_off, lv.num_slots,
      static_cast<uint32_t>(items >> (cdepth + 1)), lv.level, cdepth, sdepth, t.first.as<uint32_t>(), t.last.as<uint32_t>(), ks.scale, partials,
      tc_terms(), whole, static_cast<uint32_t>(nitems), counter.as<uint32_t>());
  FSGG_LAUNCH_CHECK();
  ds.launches++;
}

}  // namespace fsgg
