// Input side of the path: seeded generators for the
// benchmark configurations.
//
//  * make_moons / make_blobs restate proj/src/datasets.cpp:20-124 with the
//    reference's keyed splitmix64 streams and Box-Muller normals
//    (proj/include/fsg/rng.hpp:20-62). Same libm calls in the same order,
//    so on the same host they produce bit-identical fp64 coordinates (the
//    tests check this against the reference build).
//  * make_image_features / make_gmm define configs C4/C5, which have no
//    reference generator; BSDS images and MNIST-like data are
//    not available offline, so seeded synthetic stand-ins with the stated
//    shapes and value distributions are used instead.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/fsgg.h"
#include "common.cuh"

namespace fsgg {
namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr uint64_t kMoonsTag = 0x6d6f6f6e73ULL;
constexpr uint64_t kBlobsTag = 0x626c6f6273ULL;
constexpr uint64_t kImageTag = 0x696d616765ULL;   // "image"
constexpr uint64_t kImageNoiseTag = 0x696d676e6fULL;
constexpr uint64_t kGmmTag = 0x676d6dULL;         // "gmm"
constexpr uint64_t kGmmNoiseTag = 0x676d6d6eULL;

// Keyed counter-based stream (proj/include/fsg/rng.hpp:18-79).
class Stream {
public:
  Stream(uint64_t seed, uint64_t tag, uint64_t a = 0, uint64_t b = 0) {
    uint64_t k = splitmix64(seed);
    k = splitmix64(k ^ splitmix64(tag ^ 0x6a09e667f3bcc909ULL));
    k = splitmix64(k ^ splitmix64(a ^ 0xbb67ae8584caa73bULL));
    k = splitmix64(k ^ splitmix64(b ^ 0x3c6ef372fe94f82bULL));
    key_ = k;
  }
  uint64_t next_u64() { return splitmix64(key_ + counter_++); }
  double next_double() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_normal() {
    if (have_) {
      have_ = false;
      return cached_;
    }
    double u1, u2;
    do {
      u1 = next_double();
    } while (u1 <= 0.0);
    u2 = next_double();
    double r = std::sqrt(-2.0 * std::log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    cached_ = r * std::sin(a);
    have_ = true;
    return r * std::cos(a);
  }

private:
  uint64_t key_ = 0, counter_ = 0;
  double cached_ = 0.0;
  bool have_ = false;
};

// proj/src/datasets.cpp:20-28
void add_noise(double* pts, uint32_t n, uint32_t d, double stddev,
               uint64_t seed, uint64_t tag) {
  if (stddev == 0.0) return;
  for (uint32_t i = 0; i < n; ++i) {
    Stream s(seed, tag, i);
    // The reference build (g++ -O3, FMA-capable -march) contracts this
    // update into a fused multiply-add; spell it out so the result does not
    // depend on our own compile flags.
    for (uint32_t c = 0; c < d; ++c) {
      double& p = pts[size_t(i) * d + c];
      p = std::fma(stddev, s.next_normal(), p);
    }
  }
}

}  // namespace
}  // namespace fsgg

using fsgg::Stream;

extern "C" int fsgg_make_moons(uint32_t n, double noise, uint64_t seed,
                               double* pts, uint32_t* labels) {
  if (n < 2 || noise < 0.0 || !pts) return FSGG_ERR_CONFIG;  // datasets.cpp:33-34
  const uint32_t n_out = n / 2, n_in = n - n_out;
  for (uint32_t i = 0; i < n_out; ++i) {
    double t = n_out > 1 ? fsgg::kPi * i / (n_out - 1) : 0.0;
    pts[size_t(i) * 2] = std::cos(t);
    pts[size_t(i) * 2 + 1] = std::sin(t);
    if (labels) labels[i] = 0;
  }
  for (uint32_t i = 0; i < n_in; ++i) {
    double t = n_in > 1 ? fsgg::kPi * i / (n_in - 1) : 0.0;
    size_t at = size_t(n_out + i) * 2;
    pts[at] = 1.0 - std::cos(t);
    pts[at + 1] = 1.0 - std::sin(t) - 0.5;
    if (labels) labels[n_out + i] = 1;
  }
  fsgg::add_noise(pts, n, 2, noise, seed, fsgg::kMoonsTag);
  return FSGG_OK;
}

extern "C" int fsgg_make_blobs(uint32_t n, const double* centers, uint32_t k,
                               uint32_t d, double stddev, uint64_t seed,
                               double* pts, uint32_t* labels) {
  if (k == 0 || n < k || stddev < 0.0 || d == 0 || !pts || !centers)
    return FSGG_ERR_CONFIG;  // datasets.cpp:71-80
  uint32_t at = 0;
  for (uint32_t c = 0; c < k; ++c) {
    uint32_t cnt = n / k + (c < n % k ? 1 : 0);
    for (uint32_t i = 0; i < cnt; ++i, ++at) {
      for (uint32_t a = 0; a < d; ++a) pts[size_t(at) * d + a] = centers[size_t(c) * d + a];
      if (labels) labels[at] = c;
    }
  }
  fsgg::add_noise(pts, n, d, stddev, seed, fsgg::kBlobsTag);
  return FSGG_OK;
}

extern "C" int fsgg_make_image_features(uint32_t height, uint32_t width,
                                        uint32_t regions, double noise,
                                        uint64_t seed, double* pts,
                                        uint32_t* labels) {
  if (height == 0 || width == 0 || regions == 0 || noise < 0.0 || !pts)
    return FSGG_ERR_CONFIG;
  // Voronoi sites in normalised (row, col) space and one colour per region.
  Stream rs(seed, fsgg::kImageTag);
  std::vector<double> site(size_t(regions) * 2), colour(size_t(regions) * 3);
  for (uint32_t r = 0; r < regions; ++r) {
    site[2 * r] = rs.next_double();
    site[2 * r + 1] = rs.next_double();
    for (int c = 0; c < 3; ++c) colour[3 * r + c] = rs.next_double();
  }
  for (uint32_t row = 0; row < height; ++row) {
    for (uint32_t col = 0; col < width; ++col) {
      const uint32_t i = row * width + col;
      const double y = double(row) / height, x = double(col) / width;
      uint32_t best = 0;
      double bd = 1e300;
      for (uint32_t r = 0; r < regions; ++r) {
        double dy = y - site[2 * r], dx = x - site[2 * r + 1];
        double dd = dy * dy + dx * dx;
        if (dd < bd) {
          bd = dd;
          best = r;
        }
      }
      Stream ns(seed, fsgg::kImageNoiseTag, i);
      double* p = pts + size_t(i) * 5;
      p[0] = y;
      p[1] = x;
      for (int c = 0; c < 3; ++c) p[2 + c] = std::fma(noise, ns.next_normal(), colour[3 * best + c]);
      if (labels) labels[i] = best;
    }
  }
  return FSGG_OK;
}

extern "C" int fsgg_make_gmm(uint32_t n, uint32_t d, uint32_t k, double stddev,
                             uint64_t seed, double* pts, uint32_t* labels) {
  if (k == 0 || n < k || d == 0 || stddev < 0.0 || !pts) return FSGG_ERR_CONFIG;
  Stream cs(seed, fsgg::kGmmTag);
  std::vector<double> centers(size_t(k) * d);
  for (auto& v : centers) v = cs.next_double();
  uint32_t at = 0;
  for (uint32_t c = 0; c < k; ++c) {
    uint32_t cnt = n / k + (c < n % k ? 1 : 0);
    for (uint32_t i = 0; i < cnt; ++i, ++at) {
      Stream ns(seed, fsgg::kGmmNoiseTag, at);
      for (uint32_t a = 0; a < d; ++a) {
        double v = std::fma(stddev, ns.next_normal(), centers[size_t(c) * d + a]);
        pts[size_t(at) * d + a] = std::min(1.0, std::max(0.0, v));
      }
      if (labels) labels[at] = c;
    }
  }
  return FSGG_OK;
}
