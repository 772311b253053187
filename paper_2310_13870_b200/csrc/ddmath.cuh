// Correctly rounded log, sin and cos in double-double arithmetic, for the
// device-side dataset generators (datasets_dev.cu).
//
// The reference draws its points with glibc's log/sin/cos
// (proj/include/fsg/rng.hpp:47-62 Box-Muller, proj/src/datasets.cpp:38-50
// the moons' arcs). glibc returns the correctly rounded double for these
// functions on the argument ranges the generators use; CUDA's libdevice
// versions are accurate to 1-2 ulp, which would change a few low bits per
// million points. Here every function is evaluated to ~2^-100 relative
// accuracy in double-double (pairs hi + lo of doubles, error-free
// transformations built on fma) and rounded once, so the device generators
// reproduce the host's bits. Header-only and __host__ __device__: the CPU
// suite compiles the same code with g++ (-ffp-contract=off) and checks it
// against glibc on millions of arguments (tests/test_ddmath.py).
//
// Device code must not let nvcc contract a*b+c, which would break the
// error-free transformations: every operation goes through the explicitly
// rounded intrinsics.
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define FSGG_HD __host__ __device__ __forceinline__
#else
#define FSGG_HD inline
#endif

namespace fsgg {
namespace dd {

#if defined(__CUDA_ARCH__)
FSGG_HD double add(double a, double b) { return __dadd_rn(a, b); }
FSGG_HD double sub(double a, double b) { return __dsub_rn(a, b); }
FSGG_HD double mul(double a, double b) { return __dmul_rn(a, b); }
FSGG_HD double div(double a, double b) { return __ddiv_rn(a, b); }
FSGG_HD double fmaf64(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
// host: compiled with -ffp-contract=off (no implicit contraction)
FSGG_HD double add(double a, double b) { return a + b; }
FSGG_HD double sub(double a, double b) { return a - b; }
FSGG_HD double mul(double a, double b) { return a * b; }
FSGG_HD double div(double a, double b) { return a / b; }
FSGG_HD double fmaf64(double a, double b, double c) { return fma(a, b, c); }
#endif

struct DD {
  double hi, lo;
};

FSGG_HD DD two_sum(double a, double b) {
  const double s = add(a, b);
  const double bb = sub(s, a);
  const double e = add(sub(a, sub(s, bb)), sub(b, bb));
  return {s, e};
}
FSGG_HD DD quick_two_sum(double a, double b) {  // |a| >= |b|
  const double s = add(a, b);
  return {s, sub(b, sub(s, a))};
}
FSGG_HD DD two_prod(double a, double b) {
  const double p = mul(a, b);
  return {p, fmaf64(a, b, -p)};
}
FSGG_HD DD neg(DD x) { return {-x.hi, -x.lo}; }
FSGG_HD DD add(DD x, DD y) {  // accurate (IEEE-style) double-double sum
  DD s = two_sum(x.hi, y.hi);
  const DD t = two_sum(x.lo, y.lo);
  s.lo = add(s.lo, t.hi);
  s = quick_two_sum(s.hi, s.lo);
  s.lo = add(s.lo, t.lo);
  return quick_two_sum(s.hi, s.lo);
}
FSGG_HD DD mul(DD x, DD y) {
  DD p = two_prod(x.hi, y.hi);
  p.lo = fmaf64(x.hi, y.lo, p.lo);
  p.lo = fmaf64(x.lo, y.hi, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
FSGG_HD DD mul(DD x, double d) {
  DD p = two_prod(x.hi, d);
  p.lo = fmaf64(x.lo, d, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
FSGG_HD DD div(DD x, DD y) {
  const double q1 = div(x.hi, y.hi);
  DD r = add(x, neg(mul(y, q1)));
  const double q2 = div(r.hi, y.hi);
  r = add(r, neg(mul(y, q2)));
  const double q3 = div(r.hi, y.hi);
  DD q = quick_two_sum(q1, q2);
  return add(q, DD{q3, 0.0});
}

// 1/n! (n = 0..29) and 1/(2k+1) (k = 0..22) as double-doubles (hi, lo),
// computed to 80 digits with Python's decimal module.
#define FSGG_DD(h, l) DD{h, l}
FSGG_HD DD inv_fact(int n) {
  switch (n) {
    case 0: case 1: return FSGG_DD(1.0, 0.0);
    case 2: return FSGG_DD(0x1.0000000000000p-1, 0.0);
    case 3: return FSGG_DD(0x1.5555555555555p-3, 0x1.5555555555555p-57);
    case 4: return FSGG_DD(0x1.5555555555555p-5, 0x1.5555555555555p-59);
    case 5: return FSGG_DD(0x1.1111111111111p-7, 0x1.1111111111111p-63);
    case 6: return FSGG_DD(0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65);
    case 7: return FSGG_DD(0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73);
    case 8: return FSGG_DD(0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76);
    case 9: return FSGG_DD(0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73);
    case 10: return FSGG_DD(0x1.27e4fb7789f5cp-22, 0x1.cbbc05b4fa99ap-76);
    case 11: return FSGG_DD(0x1.ae64567f544e4p-26, -0x1.c062e06d1f209p-80);
    case 12: return FSGG_DD(0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83);
    case 13: return FSGG_DD(0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87);
    case 14: return FSGG_DD(0x1.93974a8c07c9dp-37, 0x1.05d6f8a2efd1fp-92);
    case 15: return FSGG_DD(0x1.ae7f3e733b81fp-41, 0x1.1d8656b0ee8cbp-97);
    case 16: return FSGG_DD(0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101);
    case 17: return FSGG_DD(0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103);
    case 18: return FSGG_DD(0x1.6827863b97d97p-53, 0x1.eec01221a8b0bp-107);
    case 19: return FSGG_DD(0x1.2f49b46814157p-57, 0x1.2650f61dbdcb4p-112);
    case 20: return FSGG_DD(0x1.e542ba4020225p-62, 0x1.ea72b4afe3c2fp-120);
    case 21: return FSGG_DD(0x1.71b8ef6dcf572p-66, -0x1.d043ae40c4647p-120);
    case 22: return FSGG_DD(0x1.0ce396db7f853p-70, -0x1.aebcdbd20331cp-124);
    case 23: return FSGG_DD(0x1.761b41316381ap-75, -0x1.3423c7d91404fp-130);
    case 24: return FSGG_DD(0x1.f2cf01972f578p-80, -0x1.9ada5fcc1ab14p-135);
    case 25: return FSGG_DD(0x1.3f3ccdd165fa9p-84, -0x1.58ddadf344487p-139);
    case 26: return FSGG_DD(0x1.88e85fc6a4e5ap-89, -0x1.71c37ebd16540p-143);
    case 27: return FSGG_DD(0x1.d1ab1c2dccea3p-94, 0x1.054d0c78aea14p-149);
    case 28: return FSGG_DD(0x1.0a18a2635085dp-98, 0x1.b9e2e28e1aa54p-153);
    default: return FSGG_DD(0x1.259f98b4358adp-103, 0x1.eaf8c39dd9bc5p-157);  // 29
  }
}
FSGG_HD DD inv_odd(int k) {  // 1 / (2k + 1)
  switch (k) {
    case 0: return FSGG_DD(1.0, 0.0);
    case 1: return FSGG_DD(0x1.5555555555555p-2, 0x1.5555555555555p-56);
    case 2: return FSGG_DD(0x1.999999999999ap-3, -0x1.999999999999ap-57);
    case 3: return FSGG_DD(0x1.2492492492492p-3, 0x1.2492492492492p-57);
    case 4: return FSGG_DD(0x1.c71c71c71c71cp-4, 0x1.c71c71c71c71cp-58);
    case 5: return FSGG_DD(0x1.745d1745d1746p-4, -0x1.745d1745d1746p-59);
    case 6: return FSGG_DD(0x1.3b13b13b13b14p-4, -0x1.3b13b13b13b14p-58);
    case 7: return FSGG_DD(0x1.1111111111111p-4, 0x1.1111111111111p-60);
    case 8: return FSGG_DD(0x1.e1e1e1e1e1e1ep-5, 0x1.e1e1e1e1e1e1ep-61);
    case 9: return FSGG_DD(0x1.af286bca1af28p-5, 0x1.af286bca1af28p-59);
    case 10: return FSGG_DD(0x1.8618618618618p-5, 0x1.8618618618618p-59);
    case 11: return FSGG_DD(0x1.642c8590b2164p-5, 0x1.642c8590b2164p-60);
    case 12: return FSGG_DD(0x1.47ae147ae147bp-5, -0x1.eb851eb851eb8p-61);
    case 13: return FSGG_DD(0x1.2f684bda12f68p-5, 0x1.2f684bda12f68p-59);
    case 14: return FSGG_DD(0x1.1a7b9611a7b96p-5, 0x1.1a7b9611a7b96p-61);
    case 15: return FSGG_DD(0x1.0842108421084p-5, 0x1.0842108421084p-60);
    case 16: return FSGG_DD(0x1.f07c1f07c1f08p-6, -0x1.f07c1f07c1f08p-61);
    case 17: return FSGG_DD(0x1.d41d41d41d41dp-6, 0x1.0750750750750p-60);
    case 18: return FSGG_DD(0x1.bacf914c1bad0p-6, -0x1.bacf914c1bad0p-60);
    case 19: return FSGG_DD(0x1.a41a41a41a41ap-6, 0x1.0690690690690p-60);
    case 20: return FSGG_DD(0x1.8f9c18f9c18fap-6, -0x1.f3831f3831f38p-61);
    case 21: return FSGG_DD(0x1.7d05f417d05f4p-6, 0x1.7d05f417d05f4p-62);
    default: return FSGG_DD(0x1.6c16c16c16c17p-6, -0x1.f49f49f49f49fp-61);  // 22
  }
}
#undef FSGG_DD

constexpr double kLn2Hi = 0x1.62e42fefa39efp-1, kLn2Lo = 0x1.abc9e3b39803fp-56;
// pi/2 as a triple-double
constexpr double kPio2A = 0x1.921fb54442d18p+0, kPio2B = 0x1.1a62633145c07p-54,
                 kPio2C = -0x1.f1976b7ed8fbcp-110;

// log(x) for finite x > 0, correctly rounded (to ~2^-100 relative before the
// final rounding). x = m 2^e with m in [sqrt(1/2), sqrt(2)); log m =
// 2 atanh(s), s = (m - 1)/(m + 1), |s| <= 0.1716, series to s^45.
FSGG_HD double log_cr(double x) {
  int e = 0;
  double m = frexp(x, &e);  // m in [1/2, 1)
  if (m < 0x1.6a09e667f3bcdp-1) {  // below sqrt(1/2): scale into [sqrt(1/2), 1)
    m = mul(m, 2.0);
    e -= 1;
  }
  // m in [sqrt(1/2), sqrt(2)) after the scaling above (exact)
  const double num = sub(m, 1.0);  // exact (Sterbenz)
  const DD den = two_sum(m, 1.0);
  const DD s = div(DD{num, 0.0}, den);
  const DD s2 = mul(s, s);
  DD p = inv_odd(22);
  for (int k = 21; k >= 0; --k) p = add(mul(p, s2), inv_odd(k));
  DD l = mul(s, p);
  l.hi = mul(l.hi, 2.0);
  l.lo = mul(l.lo, 2.0);
  const DD el = add(two_prod(double(e), kLn2Hi), two_prod(double(e), kLn2Lo));
  const DD r = add(el, l);
  return add(r.hi, r.lo);
}

// sin(x), cos(x) for finite |x| <= 8, correctly rounded (same sense as
// log_cr). x = q pi/2 + r, |r| <= pi/4, r in double-double from a
// triple-double pi/2; Taylor series to r^29 / 29!.
FSGG_HD void sincos_cr(double x, double* sn, double* cs) {
  const double q = rint(mul(x, 0x1.45f306dc9c883p-1));  // x * 2/pi
  // r = x - q (A + B + C): q A, q B as exact products
  DD r = two_sum(x, -two_prod(q, kPio2A).hi);
  r = add(r, DD{-two_prod(q, kPio2A).lo, 0.0});
  r = add(r, neg(two_prod(q, kPio2B)));
  r = add(r, DD{-mul(q, kPio2C), 0.0});
  const DD nr2 = neg(mul(r, r));
  DD S = inv_fact(29), C = inv_fact(28);
  for (int k = 13; k >= 0; --k) {
    S = add(mul(S, nr2), inv_fact(2 * k + 1));
    C = add(mul(C, nr2), inv_fact(2 * k));
  }
  S = mul(S, r);
  const double s = add(S.hi, S.lo), c = add(C.hi, C.lo);
  switch (int(q) & 3) {
    case 0: *sn = s; *cs = c; break;
    case 1: *sn = c; *cs = -s; break;
    case 2: *sn = -s; *cs = -c; break;
    default: *sn = -c; *cs = s; break;
  }
}

}  // namespace dd
}  // namespace fsgg
