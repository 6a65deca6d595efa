// Device arithmetic that reproduces the reference's x86-64 GCC 13 floating
// point program bit for bit: every operation is an explicit round-to-nearest
// intrinsic (no FMA contraction; the reference build has none).
//
//   complex multiply   (ac - bd, ad + bc)            libstdc++ inline, complex3.hpp:80/88
//   complex divide     libgcc __divdc3 (GCC >= 12 scaled Smith)   complex3.cpp:43-47
//   Mat3c * Vec3c      r[i] = ((0 + m0 x0) + m1 x1) + m2 x2       complex3.hpp:85-90
//   Mat3c * Mat3c      skip exact-zero left entries               complex3.hpp:76-84
//   masked_inverse     Gauss-Jordan, partial pivoting on cabs     complex3.cpp:9-61
#pragma once

#include <cfloat>
#include <cstdint>

#if defined(__CUDACC__)
#define KR_HD __host__ __device__ __forceinline__
#else
#define KR_HD inline
#endif

namespace kronred::b200::dev {

#if defined(__CUDA_ARCH__)
KR_HD double dadd(double a, double b) { return __dadd_rn(a, b); }
KR_HD double dsub(double a, double b) { return __dsub_rn(a, b); }
KR_HD double dmul(double a, double b) { return __dmul_rn(a, b); }
KR_HD double ddiv(double a, double b) { return __ddiv_rn(a, b); }
KR_HD double dsqrt(double a) { return __dsqrt_rn(a); }
#else
KR_HD double dadd(double a, double b) { return a + b; }
KR_HD double dsub(double a, double b) { return a - b; }
KR_HD double dmul(double a, double b) { return a * b; }
KR_HD double ddiv(double a, double b) { return a / b; }
KR_HD double dsqrt(double a) { return __builtin_sqrt(a); }
#endif

struct C2 {
  double x, y;
};

KR_HD C2 cadd(C2 a, C2 b) { return {dadd(a.x, b.x), dadd(a.y, b.y)}; }
KR_HD C2 csub(C2 a, C2 b) { return {dsub(a.x, b.x), dsub(a.y, b.y)}; }
KR_HD C2 cmul(C2 a, C2 b) {
  return {dsub(dmul(a.x, b.x), dmul(a.y, b.y)), dadd(dmul(a.x, b.y), dmul(a.y, b.x))};
}
KR_HD bool cis0(C2 a) { return a.x == 0.0 && a.y == 0.0; }

// libgcc2.c __divdc3 as shipped with GCC 13 (RBIG = DBL_MAX/2, RMIN = DBL_MIN,
// RMIN2 = DBL_EPSILON, RMINSCAL = 1/DBL_EPSILON, RMAX2 = RBIG*RMIN2).
KR_HD C2 cdiv(C2 num, C2 den) {
  double a = num.x, b = num.y, c = den.x, d = den.y;
  const double RBIG = DBL_MAX / 2.0, RMIN = DBL_MIN, RMIN2 = DBL_EPSILON;
  const double RMINSCAL = 1.0 / DBL_EPSILON, RMAX2 = RBIG * RMIN2;
  double denom, ratio, x, y;
  auto fab = [](double v) { return v < 0 ? -v : (v == 0 ? 0.0 : v); };
  if (fab(c) < fab(d)) {
    if (fab(d) >= RBIG) {
      a = ddiv(a, 2.0); b = ddiv(b, 2.0); c = ddiv(c, 2.0); d = ddiv(d, 2.0);
    }
    if (fab(d) < RMIN2) {
      a = dmul(a, RMINSCAL); b = dmul(b, RMINSCAL); c = dmul(c, RMINSCAL); d = dmul(d, RMINSCAL);
    } else if (((fab(a) < RMIN) && (fab(b) < RMAX2) && (fab(d) < RMAX2)) ||
               ((fab(b) < RMIN) && (fab(a) < RMAX2) && (fab(d) < RMAX2))) {
      a = dmul(a, RMINSCAL); b = dmul(b, RMINSCAL); c = dmul(c, RMINSCAL); d = dmul(d, RMINSCAL);
    }
    ratio = ddiv(c, d);
    denom = dadd(dmul(c, ratio), d);
    if (fab(ratio) > RMIN) {
      x = ddiv(dadd(dmul(a, ratio), b), denom);
      y = ddiv(dsub(dmul(b, ratio), a), denom);
    } else {
      x = ddiv(dadd(dmul(c, ddiv(a, d)), b), denom);
      y = ddiv(dsub(dmul(c, ddiv(b, d)), a), denom);
    }
  } else {
    if (fab(c) >= RBIG) {
      a = ddiv(a, 2.0); b = ddiv(b, 2.0); c = ddiv(c, 2.0); d = ddiv(d, 2.0);
    }
    if (fab(c) < RMIN2) {
      a = dmul(a, RMINSCAL); b = dmul(b, RMINSCAL); c = dmul(c, RMINSCAL); d = dmul(d, RMINSCAL);
    } else if (((fab(a) < RMIN) && (fab(b) < RMAX2) && (fab(c) < RMAX2)) ||
               ((fab(b) < RMIN) && (fab(a) < RMAX2) && (fab(c) < RMAX2))) {
      a = dmul(a, RMINSCAL); b = dmul(b, RMINSCAL); c = dmul(c, RMINSCAL); d = dmul(d, RMINSCAL);
    }
    ratio = ddiv(d, c);
    denom = dadd(dmul(d, ratio), c);
    if (fab(ratio) > RMIN) {
      x = ddiv(dadd(dmul(b, ratio), a), denom);
      y = ddiv(dsub(b, dmul(a, ratio)), denom);
    } else {
      x = ddiv(dadd(a, dmul(d, ddiv(b, c))), denom);
      y = ddiv(dsub(b, dmul(d, ddiv(a, c))), denom);
    }
  }
  if (x != x && y != y) {
    const double inf = __builtin_huge_val();
    auto isinf_ = [](double v) { return v == __builtin_huge_val() || v == -__builtin_huge_val(); };
    auto isnan_ = [](double v) { return v != v; };
    auto isfin_ = [&](double v) { return !isnan_(v) && !isinf_(v); };
    auto csign = [](double mag, double sgn) { return __builtin_copysign(mag, sgn); };
    if (c == 0.0 && d == 0.0 && (!isnan_(a) || !isnan_(b))) {
      x = dmul(csign(inf, c), a);
      y = dmul(csign(inf, c), b);
    } else if ((isinf_(a) || isinf_(b)) && isfin_(c) && isfin_(d)) {
      a = csign(isinf_(a) ? 1.0 : 0.0, a);
      b = csign(isinf_(b) ? 1.0 : 0.0, b);
      x = dmul(inf, dadd(dmul(a, c), dmul(b, d)));
      y = dmul(inf, dsub(dmul(b, c), dmul(a, d)));
    } else if ((isinf_(c) || isinf_(d)) && isfin_(a) && isfin_(b)) {
      c = csign(isinf_(c) ? 1.0 : 0.0, c);
      d = csign(isinf_(d) ? 1.0 : 0.0, d);
      x = dmul(0.0, dadd(dmul(a, c), dmul(b, d)));
      y = dmul(0.0, dsub(dmul(b, c), dmul(a, d)));
    }
  }
  return {x, y};
}

}  // namespace kronred::b200::dev
