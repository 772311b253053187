// Shared device/host helpers for the fsgg sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

namespace fsgg {

// Error classes carrying the reference's exit codes
// (proj/include/fsg/common.hpp:13-66) plus 5 for device failures.
struct Error : std::runtime_error {
  int code;
  Error(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};
struct ConfigError : Error {
  explicit ConfigError(const std::string& m) : Error(m, 2) {}
};
struct NumericError : Error {
  explicit NumericError(const std::string& m) : Error(m, 4) {}
};
struct DeviceError : Error {
  explicit DeviceError(const std::string& m) : Error(m, 5) {}
};

#define FSGG_CUDA(expr)                                                    \
  do {                                                                     \
    cudaError_t _e = (expr);                                               \
    if (_e != cudaSuccess)                                                 \
      throw ::fsgg::DeviceError(std::string(#expr) + ": " +                \
                                cudaGetErrorString(_e) + " (" __FILE__ ":" \
                                + std::to_string(__LINE__) + ")");         \
  } while (0)

#define FSGG_LAUNCH_CHECK() FSGG_CUDA(cudaGetLastError())

constexpr double kSumFloor = 1e-300;                 // kde.hpp:43
constexpr uint64_t kRouteTag = 0x88b4f8a3c2d1e5f7ULL;  // sampler.cpp:25

// proj/include/fsg/rng.hpp:11-16
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// First two links of RngStream::keyed (rng.hpp:22-23) depend only on
// (seed, tag); the host folds them once per build.
inline uint64_t route_key_prefix(uint64_t seed) {
  uint64_t k = splitmix64(seed);
  return splitmix64(k ^ splitmix64(kRouteTag ^ 0x6a09e667f3bcc909ULL));
}

// Remaining links (rng.hpp:24-25) for a = (first << 32) | last, b = query.
__host__ __device__ __forceinline__ uint64_t route_key(uint64_t prefix,
                                                       uint64_t a,
                                                       uint64_t b) {
  uint64_t k = splitmix64(prefix ^ splitmix64(a ^ 0xbb67ae8584caa73bULL));
  return splitmix64(k ^ splitmix64(b ^ 0x3c6ef372fe94f82bULL));
}
// Same key with the query's link splitmix64(b ^ ...) precomputed (a walk
// keeps its query for every node it visits).
__host__ __device__ __forceinline__ uint64_t query_link(uint64_t b) {
  return splitmix64(b ^ 0x3c6ef372fe94f82bULL);
}
// The node's link splitmix64(prefix ^ splitmix64(a ^ ...)) of route_key: a
// function of (seed, node) alone, tabulated once per build per tree slot
// (node_link_kernel, sampler.cu), so an entry's key is
// splitmix64(node_link ^ query_link).
__host__ __device__ __forceinline__ uint64_t node_link(uint64_t prefix, uint64_t a) {
  return splitmix64(prefix ^ splitmix64(a ^ 0xbb67ae8584caa73bULL));
}
__host__ __device__ __forceinline__ uint64_t route_key_q(uint64_t prefix, uint64_t a,
                                                         uint64_t qlink) {
  return splitmix64(splitmix64(prefix ^ splitmix64(a ^ 0xbb67ae8584caa73bULL)) ^ qlink);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

#ifdef __CUDACC__
// 2^x for a pair of x <= 0 on the FP32 pipe instead of MUFU (FA4-style
// offload): x = j + f with j = rint(x) (1.5*2^23 magic add), 2^f on
// [-1/2, 1/2] by a degree-5 minimax polynomial (max rel. error 2.4e-7 in
// fp32, the same order as ex2.approx), then j added to the exponent field.
// Arguments are clamped at -125 (MUFU's .ftz result there is 0; this one is
// < 2^-124: both negligible against the pruning bound).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 r = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(x, make_float2(-r.x, -r.y));
  float2 p = make_float2(0.0013277226826176047f, 0.0013277226826176047f);
  p = __ffma2_rn(p, f, make_float2(0.009675547480583191f, 0.009675547480583191f));
  p = __ffma2_rn(p, f, make_float2(0.0555071085691452f, 0.0555071085691452f));
  p = __ffma2_rn(p, f, make_float2(0.24022120237350464f, 0.24022120237350464f));
  p = __ffma2_rn(p, f, make_float2(0.6931469440460205f, 0.6931469440460205f));
  p = __ffma2_rn(p, f, make_float2(1.0000001192092896f, 1.0000001192092896f));
  // low bits of t hold j; (bits(t) << 23) == (j << 23) mod 2^32
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}
#endif

#ifdef __CUDACC__
// fp64 kernel value, same operation order as proj/include/fsg/kernel.hpp:28-53.
__device__ __forceinline__ double kernel_f64(int family, double sigma,
                                             const float* x, const float* y,
                                             uint32_t d) {
  double s = 0.0;
  if (family == 2) {
    for (uint32_t k = 0; k < d; ++k)
      s = __dadd_rn(s, fabs(__dsub_rn(double(x[k]), double(y[k]))));
    return exp(-s / sigma);
  }
  // Products rounded and added in order; the last coordinate of an odd d is
  // fused, as the reference binary's vectorised loop does (see
  // oracle/fsg_oracle.c: sq_dist_ref).
  const uint32_t even = d & ~1u;
  for (uint32_t k = 0; k < even; ++k) {
    const double t = __dsub_rn(double(x[k]), double(y[k]));
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  if (d & 1u) {
    const double t = __dsub_rn(double(x[d - 1]), double(y[d - 1]));
    s = __fma_rn(t, t, s);
  }
  if (family == 1) return exp(-sqrt(s) / sigma);
  return exp(-s / __dmul_rn(sigma, sigma));
}
#endif

inline uint32_t ceil_div_u32(uint64_t a, uint64_t b) {
  return static_cast<uint32_t>((a + b - 1) / b);
}

}  // namespace fsgg
