// Test helper (CPU suite): the device generators' double-double math
// (paper_2310_13870_b200/csrc/ddmath.cuh) compiled for the host.
//   ddmath_driver fn      reads doubles (hex) from stdin, prints fn(x) for
//                         fn in {log, sin, cos} as hex, one per line
//   ddmath_driver moons n noise seed
//                         make_moons (proj/src/datasets.cpp:32-55) with the
//                         dd functions; prints the fp64 coordinates as hex
//   ddmath_driver glibc N   counts dd vs glibc mismatches over N Box-Muller
//                         arguments (log u1, sin/cos 2 pi u2)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ddmath.cuh"

namespace {
uint64_t sm64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
struct Stream {  // proj/include/fsg/rng.hpp:20-62 with the dd functions
  uint64_t key, c = 0;
  bool have = false;
  double cached = 0;
  Stream(uint64_t seed, uint64_t tag, uint64_t a) {
    uint64_t k = sm64(seed);
    k = sm64(k ^ sm64(tag ^ 0x6a09e667f3bcc909ULL));
    k = sm64(k ^ sm64(a ^ 0xbb67ae8584caa73bULL));
    key = sm64(k ^ sm64(0x3c6ef372fe94f82bULL));
  }
  double next_double() { return double(sm64(key + c++) >> 11) * 0x1.0p-53; }
  double next_normal() {
    if (have) {
      have = false;
      return cached;
    }
    double u1, u2;
    do u1 = next_double(); while (u1 <= 0.0);
    u2 = next_double();
    const double r = std::sqrt(-2.0 * fsgg::dd::log_cr(u1));
    double s, co;
    fsgg::dd::sincos_cr(6.283185307179586476925286766559 * u2, &s, &co);
    cached = r * s;
    have = true;
    return r * co;
  }
};
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  const char* mode = argv[1];
  if (!std::strcmp(mode, "moons")) {
    const uint32_t n = std::strtoul(argv[2], nullptr, 10);
    const double noise = std::strtod(argv[3], nullptr);
    const uint64_t seed = std::strtoull(argv[4], nullptr, 10);
    const uint32_t no = n / 2, ni = n - no;
    const double kPi = 3.14159265358979323846;
    std::vector<double> p(size_t(n) * 2);
    for (uint32_t i = 0; i < n; ++i) {
      const bool outer = i < no;
      const uint32_t j = outer ? i : i - no, m = outer ? no : ni;
      const double t = m > 1 ? kPi * j / (m - 1) : 0.0;
      double s, c;
      fsgg::dd::sincos_cr(t, &s, &c);
      p[2 * size_t(i)] = outer ? c : 1.0 - c;
      p[2 * size_t(i) + 1] = outer ? s : 1.0 - s - 0.5;
      if (noise != 0.0) {
        Stream st(seed, 0x6d6f6f6e73ULL, i);
        for (int k = 0; k < 2; ++k) p[2 * size_t(i) + k] = std::fma(noise, st.next_normal(), p[2 * size_t(i) + k]);
      }
    }
    std::fwrite(p.data(), 8, p.size(), stdout);
    return 0;
  }
  if (!std::strcmp(mode, "glibc")) {
    const long N = std::atol(argv[2]);
    long bl = 0, bs = 0, bc = 0;
    for (long i = 0; i < N; ++i) {
      uint64_t k = sm64(i) >> 11;
      if (!k) k = 1;
      const double u = double(k) * 0x1.0p-53;
      const double a = std::log(u), b = fsgg::dd::log_cr(u);
      bl += std::memcmp(&a, &b, 8) != 0;
      const double t = 6.283185307179586476925286766559 * (double(sm64(i + N) >> 11) * 0x1.0p-53);
      double s, c;
      fsgg::dd::sincos_cr(t, &s, &c);
      const double s0 = std::sin(t), c0 = std::cos(t);
      bs += std::memcmp(&s, &s0, 8) != 0;
      bc += std::memcmp(&c, &c0, 8) != 0;
    }
    std::printf("%ld %ld %ld\n", bl, bs, bc);
    return 0;
  }
  double x;
  char buf[64];
  while (std::scanf("%63s", buf) == 1) {
    x = std::strtod(buf, nullptr);
    double y = 0, s, c;
    if (!std::strcmp(mode, "log")) y = fsgg::dd::log_cr(x);
    else {
      fsgg::dd::sincos_cr(x, &s, &c);
      y = !std::strcmp(mode, "sin") ? s : c;
    }
    std::printf("%a\n", y);
  }
  return 0;
}
