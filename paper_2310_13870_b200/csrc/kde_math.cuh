// Kernel-family arithmetic shared by the KDE kernels (kde.cu) and the
// depth-first finish kernel (finish.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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


}  // namespace fsgg
