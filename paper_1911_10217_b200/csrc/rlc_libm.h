// rlc_libm.h -- bit-exact restatement of the host C library's double sin/cos
// for the cosine-hemisphere sampler of multi-bounce paths
// (proj/include/rlcuts/math.hpp:101-107 calls std::cos / std::sin).
//
// glibc's sin/cos are not correctly rounded (about 0.25% of results in
// [0, 2pi) differ from the correctly rounded value), so a device sin/cos of
// any accuracy would not reproduce the reference's bounce directions.  This
// header restates the algorithm glibc 2.39 ships (IBM Accurate Mathematical
// Library, sysdeps/ieee754/dbl-64/s_sin.c with the multi-precision slow
// paths removed in 2.28): table-driven sin/cos for |x| < 0.855469, the pi/2
// reflection up to 2.426265, and a three-part Cody-Waite reduction beyond,
// with a Taylor polynomial for small reduced arguments.  The table is
// rlc_sincostab.h (gen_sincostab.py).
//
// x86-64 glibc dispatches between two builds of that source: __sin_fma /
// __cos_fma (compiled with -mfma, where GCC contracts every multiply whose
// only consumers are adds into an FMA) and the SSE2 build (no contraction).
// mad() reproduces exactly those contractions; Variant selects the build the
// host libm uses (probed at context creation, rlc_capi.cpp).  Verified
// bit-identical to the host libm on 4e8 random sampler angles per variant
// (the SSE2 build forced with GLIBC_TUNABLES=glibc.cpu.hwcaps=-AVX2,-FMA)
// and on every angle within 1e6 ulps of the multiples of pi/4.
//
// Domain: |x| < 105414350 (the sampler's phi = 2 pi u2 lies in [0, 2 pi)).
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

#include "rlc_common.h"

namespace rlc {
namespace libm {

enum Variant : int { kUnknown = -1, kSse2 = 0, kFma = 1 };

struct Ctx {
  const double* tab;  // rlc_sincostab.h, 440 doubles
  bool fma;           // Variant kFma
};

RLC_HD double mad(const Ctx& c, double a, double b, double x) {
  return c.fma ? fma(a, b, x) : a * b + x;  // built without contraction (--fmad=false)
}

RLC_HD uint64_t bits_of(double x) {
#ifdef __CUDA_ARCH__
  return uint64_t(__double_as_longlong(x));
#else
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
#endif
}

RLC_HD uint32_t hi_word(double x) { return uint32_t(bits_of(x) >> 32); }
RLC_HD uint32_t lo_word(double x) { return uint32_t(bits_of(x)); }

// s_sin.c constants (usncs.h); pp4 and hp1 re-derived from a 300-bit pi.
constexpr double s1 = -0x1.5555555555555p-3, s2 = 0x1.1111111110ecep-7,
                 s3 = -0x1.a01a019db08b8p-13, s4 = 0x1.71de27b9a7ed9p-19,
                 s5 = -0x1.addffc2fcdf59p-26;
constexpr double sn3 = -1.66666666666664880952546298448555E-01,
                 sn5 = 8.33333214285722277379541354343671E-03,
                 cs2 = 4.99999999999999999999950396842453E-01,
                 cs4 = -4.16666666666664434524222570944589E-02,
                 cs6 = 1.38888874007937613028114285595617E-03;
constexpr double big = 0x1.8p45, hp0 = 0x1.921fb54442d18p0, hp1 = 0x1.1a62633145c07p-54,
                 mp1 = 0x1.921fb58p0, mp2 = -0x1.dde973cp-27, pp3 = -0x1.cb3b398p-55,
                 pp4 = -0x1.d747f23e32ed7p-83, hpinv = 0x1.45f306dc9c883p-1,
                 toint = 0x1.8p52;

// TAYLOR_SIN: a + ((P(xx) a - da/2) xx + da)
RLC_HD double taylor_sin(const Ctx& c, double xx, double a, double da) {
  double p = mad(c, s5, xx, s4);
  p = mad(c, p, xx, s3);
  p = mad(c, p, xx, s2);
  p = mad(c, p, xx, s1);
  double t = mad(c, p, a, -(0.5 * da));
  t = mad(c, t, xx, da);
  return a + t;
}

RLC_HD double do_cos(const Ctx& c, double x, double dx) {
  if (x < 0) dx = -dx;
  const double u = big + fabs(x);
  x = fabs(x) - (u - big) + dx;
  const double xx = x * x;
  const double s = mad(c, x * xx, mad(c, xx, sn5, sn3), x);
  const double cc = xx * mad(c, xx, mad(c, xx, cs6, cs4), cs2);
  const double* e = c.tab + (lo_word(u) << 2);
  const double sn = e[0], ssn = e[1], cs = e[2], ccs = e[3];
  double cor = mad(c, -s, ssn, ccs);
  cor = mad(c, -cs, cc, cor);
  cor = mad(c, -sn, s, cor);
  return cs + cor;
}

RLC_HD double do_sin(const Ctx& c, double x, double dx) {
  const double xold = x;
  if (fabs(x) < 0.126) return taylor_sin(c, x * x, x, dx);
  if (x <= 0) dx = -dx;
  const double u = big + fabs(x);
  x = fabs(x) - (u - big);
  const double xx = x * x;
  const double s = x + mad(c, x * xx, mad(c, xx, sn5, sn3), dx);
  const double cc = mad(c, x, dx, xx * mad(c, xx, mad(c, xx, cs6, cs4), cs2));
  const double* e = c.tab + (lo_word(u) << 2);
  const double sn = e[0], ssn = e[1], cs = e[2], ccs = e[3];
  double cor = mad(c, s, ccs, ssn);
  cor = mad(c, -sn, cc, cor);
  cor = mad(c, cs, s, cor);
  return copysign(sn + cor, xold);
}

RLC_HD int reduce_sincos(const Ctx& c, double x, double* a, double* da) {
  const double t = mad(c, x, hpinv, toint);
  const double xn = t - toint;
  const double y = mad(c, -xn, mp2, mad(c, -xn, mp1, x));
  const int n = int(lo_word(t) & 3u);
  const double t2 = mad(c, -xn, pp3, y);
  double db = mad(c, -xn, pp3, y - t2);
  const double b = mad(c, -xn, pp4, t2);
  db += mad(c, -xn, pp4, t2 - b);
  *a = b;
  *da = db;
  return n;
}

RLC_HD double do_sincos(const Ctx& c, double a, double da, int n) {
  const double r = (n & 1) ? do_cos(c, a, da) : do_sin(c, a, da);
  return (n & 2) ? -r : r;
}

RLC_HD double sin(const Ctx& c, double x) {
  const uint32_t k = hi_word(x) & 0x7fffffffu;
  if (k < 0x3e500000u) return x;
  if (k < 0x3feb6000u) return do_sin(c, x, 0);
  if (k < 0x400368fdu) return copysign(do_cos(c, hp0 - fabs(x), hp1), x);
  double a, da;
  const int n = reduce_sincos(c, x, &a, &da);
  return do_sincos(c, a, da, n);
}

RLC_HD double cos(const Ctx& c, double x) {
  const uint32_t k = hi_word(x) & 0x7fffffffu;
  if (k < 0x3e400000u) return 1.0;
  if (k < 0x3feb6000u) return do_cos(c, x, 0);
  if (k < 0x400368fdu) {
    const double y = hp0 - fabs(x);
    const double a = y + hp1;
    const double da = (y - a) + hp1;
    return do_sin(c, a, da);
  }
  double a, da;
  const int n = reduce_sincos(c, x, &a, &da);
  return do_sincos(c, a, da, n + 1);
}

}  // namespace libm
}  // namespace rlc
