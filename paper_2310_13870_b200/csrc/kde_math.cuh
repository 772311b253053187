// Kernel-family arithmetic shared by the KDE kernels (kde.cu), the
// depth-first finish kernel (finish.cu) and the single-ticket walk (walk.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace fsgg {

// ---- kernel-family arithmetic (proj/include/fsg/kernel.hpp:28-53) ---------
// FAM 0 gaussian: dist = sum dk^2; 1 exponential: sqrt(sum dk^2);
// 2 laplacian: sum |dk|.
template <int FAM>
__device__ __forceinline__ float2 fam_first(float2 dk) {
  if constexpr (FAM == 2) return make_float2(fabsf(dk.x), fabsf(dk.y));
  return __fmul2_rn(dk, dk);
}
template <int FAM>
__device__ __forceinline__ float2 fam_next(float2 dk, float2 t) {
  if constexpr (FAM == 2)
    return __fadd2_rn(t, make_float2(fabsf(dk.x), fabsf(dk.y)));
  return __ffma2_rn(dk, dk, t);
}
template <int FAM>
__device__ __forceinline__ float2 fam_finish(float2 t) {
  if constexpr (FAM == 1) return make_float2(sqrtf(t.x), sqrtf(t.y));
  return t;
}
template <int FAM>
__device__ __forceinline__ float fam_acc1(float dk, float t) {
  if constexpr (FAM == 2) return t + fabsf(dk);
  return fmaf(dk, dk, t);
}
template <int FAM>
__device__ __forceinline__ float fam_finish1(float t) {
  if constexpr (FAM == 1) return sqrtf(t);
  return t;
}

// Lower bound of dist(q, box) for the exponent offset.
template <int FAM>
__device__ __forceinline__ float box_dist(const float* q, const float* lo,
                                          const float* hi, uint32_t d) {
  float acc = 0.f;
  for (uint32_t k = 0; k < d; ++k) {
    float v = fmaxf(fmaxf(lo[k] - q[k], q[k] - hi[k]), 0.f);
    acc = (FAM == 2) ? acc + v : fmaf(v, v, acc);
  }
  return fam_finish1<FAM>(acc);
}

// box_dist with a compile-time dimension (8-byte box loads for d = 2).
template <int D, int FAM>
__device__ __forceinline__ float box_dist_d(const float (&q)[D], const float* lo,
                                            const float* hi) {
  if constexpr (D == 2) {
    const float2 l = __ldg(reinterpret_cast<const float2*>(lo));
    const float2 h = __ldg(reinterpret_cast<const float2*>(hi));
    const float v0 = fmaxf(fmaxf(l.x - q[0], q[0] - h.x), 0.f);
    const float v1 = fmaxf(fmaxf(l.y - q[1], q[1] - h.y), 0.f);
    const float acc = (FAM == 2) ? v0 + v1 : fmaf(v1, v1, v0 * v0);
    return fam_finish1<FAM>(acc);
  } else {
    return box_dist<FAM>(q, lo, hi, D);
  }
}

// Rescale an fp32 sum of offset terms 2^(off - scale*dist) back to k units.
// 2^-off = 2^-j * 2^-(off - j) with j = floor(off): an exact power of two
// times a MUFU ex2 of a value in (-1, 0] (rel. error ~1e-7, the order of the
// fp32 terms themselves) instead of an fp64 exp2 per child.
__device__ __forceinline__ double rescale_off(double acc, float off) {
  if (!(off > 0.f)) return acc;
  const float j = floorf(off);
  const double m = acc * static_cast<double>(ex2_approx(j - off));
  // 2^-j built from its exponent bits: the same bits as ldexp(m, -j) (an
  // exact power-of-two scaling), without the library call
  if (j > 1022.f) return ldexp(m, -static_cast<int>(j));
  return m * __hiloint2double((1023 - static_cast<int>(j)) << 20, 0);
}

// Child sums of a small node (heap index h, points [f, l), l - f >= 2) for
// one query, one thread: fp32 terms with the child's bounding-box exponent
// offset, fp32 accumulation in index order, fp64 rescale. Shared by the
// direct KDE kernel and the walk so both produce the same bits.
template <int D, int FAM>
__device__ __forceinline__ void direct_child_sums(const float* __restrict__ pts,
                                                  const float (&qc)[D], uint64_t h,
                                                  uint32_t f, uint32_t l,
                                                  const float* __restrict__ tlo,
                                                  const float* __restrict__ thi,
                                                  int has_boxes, float scale, double (&s)[2]) {
  const uint32_t mid = f + (l - f) / 2;
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const uint64_t hc = 2 * h + 1 + side;
    const uint32_t a = side ? mid : f, b = side ? l : mid;
    const float off = has_boxes ? scale * box_dist_d<D, FAM>(qc, tlo + hc * D, thi + hc * D) : 0.f;
    float acc = 0.f;
    for (uint32_t j = a; j < b; ++j) {
      float t = 0.f;
      if constexpr (D == 2) {  // one 8-byte load per point
        const float2 x = __ldg(reinterpret_cast<const float2*>(pts) + j);
        t = fam_acc1<FAM>(qc[0] - x.x, t);
        t = fam_acc1<FAM>(qc[1] - x.y, t);
      } else {
        const float* x = pts + size_t(j) * D;
#pragma unroll
        for (int k = 0; k < D; ++k) t = fam_acc1<FAM>(qc[k] - __ldg(x + k), t);
      }
      t = fam_finish1<FAM>(t);
      acc += ex2_approx(fmaf(t, -scale, off));
    }
    s[side] = rescale_off(acc, off);
  }
}

// Philox4x32-10 (Salmon et al. 2011), for rng_mode = PHILOX.
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k) {
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


}  // namespace fsgg
