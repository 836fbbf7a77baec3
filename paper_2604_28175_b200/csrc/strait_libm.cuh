// strait_libm.cuh — device exp / log / pow that return the SAME bits as the
// host libm the reference runs on (glibc 2.39, x86-64 FMA variants
// __exp_fma / __log_fma / __pow_fma, which CPython's math.exp / math.log /
// float.__pow__ call: predictor.py:136-137,181-184,289-293, oracle.py:73).
//
// These are restatements of the published ARM optimized-routines algorithms
// that glibc ships (sysdeps/ieee754/dbl-64/e_exp.c, e_log.c, e_pow.c) with
// the data tables of strait_libm_tables.cuh, and with every multiply-add
// fused exactly where the x86-64 FMA build fuses it (read from the
// disassembly; marked "fma" below) and nowhere else.  The library is built
// with --fmad=false, so every other `a * b + c` rounds twice, as on the host.
// errno / floating-point exception side effects are not reproduced (the
// reference never reads them).
#pragma once

#include <stdint.h>

#include "strait_libm_tables.cuh"

namespace strait {
namespace glibc {

__device__ __forceinline__ double as_d(uint64_t u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ uint64_t as_u(double d) { return (uint64_t)__double_as_longlong(d); }
__device__ __forceinline__ uint32_t top12(double x) { return (uint32_t)(as_u(x) >> 52); }

constexpr uint32_t kExpBits = 7;
constexpr uint64_t kN = 1u << kExpBits;

// e_exp.c specialcase: k is large, scale = 2^k might over/underflow
__device__ __forceinline__ double exp_special(double tmp, uint64_t sbits, uint64_t ki, bool pow_sign) {
  if ((ki & 0x80000000u) == 0) {  // k > 0: exponent of scale might have overflowed by <= 460
    sbits -= 1009ull << 52;
    const double scale = as_d(sbits);
    return 0x1p1009 * __fma_rn(scale, tmp, scale);
  }
  sbits += 1022ull << 52;  // k < 0: careful in the subnormal range
  const double scale = as_d(sbits);
  const double st = scale * tmp;  // not fused here (mul, then add)
  double y = scale + st;
  if (pow_sign ? fabs(y) < 1.0 : y < 1.0) {
    const double one = (pow_sign && y < 0.0) ? -1.0 : 1.0;
    double lo = scale - y + st;
    const double hi = one + y;
    lo = one - hi + y + lo;
    y = (hi + lo) - one;
    if (y == 0.0) y = pow_sign ? as_d(sbits & 0x8000000000000000ull) : 0.0;
  }
  return 0x1p-1022 * y;
}

// exp core shared by exp() and pow(): 2^(k/N) * exp(r), |r| <= ln2/2N
// `tab` = __exp_data.tab as 128 (tail, sbits) pairs: the global copy, or a
// shared-memory copy staged by a kernel that calls exp in its hot loop.
template <bool POW>
__device__ __forceinline__ double exp_core(double x, double xtail, uint64_t sign_bias, uint32_t abstop,
                                           const ulonglong2* tab) {
  constexpr double InvLn2N = kExpInvLn2N, Shift = kExpShift;
  constexpr double NegLn2hiN = kExpNegLn2hiN, NegLn2loN = kExpNegLn2loN;
  constexpr double C2 = kExpC2, C3 = kExpC3, C4 = kExpC4, C5 = kExpC5;
  double kd = __fma_rn(x, InvLn2N, Shift);  // fma: z = InvLn2N * x; kd = z + Shift
  const uint64_t ki = as_u(kd);
  kd -= Shift;
  double r = __fma_rn(kd, NegLn2hiN, x);  // fma
  r = __fma_rn(kd, NegLn2loN, r);         // fma
  if (POW) r = xtail + r;                 // pow's exp_inline: r += xtail
  const uint64_t top = (ki + sign_bias) << (52 - kExpBits);
  const ulonglong2 te = tab[ki % kN];  // one 16-B load
  const double tail = as_d(te.x);
  const uint64_t sbits = te.y + top;
  const double r2 = r * r;
  const double p23 = __fma_rn(r, C3, C2);       // fma
  const double p45 = __fma_rn(r, C5, C4);       // fma
  double tmp = __fma_rn(p23, r2, r + tail);     // fma: tail + r + r2 * (C2 + r * C3)
  tmp = __fma_rn(p45, r2 * r2, tmp);            // fma: ... + r2 * r2 * (C4 + r * C5)
  if (abstop == 0) return exp_special(tmp, sbits, ki, POW);
  const double scale = as_d(sbits);
  return __fma_rn(tmp, scale, scale);  // fma: scale + scale * tmp
}

__device__ __forceinline__ const ulonglong2* exp_table() { return reinterpret_cast<const ulonglong2*>(kExpTab); }

// exp()'s common path with no branch: equal to exp(x) whenever x needs none of
// its special cases (2^-54 <= |x| < 512), which is flagged in `special`
// otherwise (the value is then meaningless and must be discarded).  Two calls
// in one basic block interleave; callers recompute the rare special inputs.
__device__ __forceinline__ double exp_common(double x, const ulonglong2* tab, bool& special) {
  const uint32_t abstop = top12(x) & 0x7ff;
  special |= abstop - 0x3c9u >= 0x408u - 0x3c9u;
  constexpr double InvLn2N = kExpInvLn2N, Shift = kExpShift;
  constexpr double NegLn2hiN = kExpNegLn2hiN, NegLn2loN = kExpNegLn2loN;
  constexpr double C2 = kExpC2, C3 = kExpC3, C4 = kExpC4, C5 = kExpC5;
  double kd = __fma_rn(x, InvLn2N, Shift);  // the exp_core<false> sequence, line for line
  const uint64_t ki = as_u(kd);
  kd -= Shift;
  double r = __fma_rn(kd, NegLn2hiN, x);
  r = __fma_rn(kd, NegLn2loN, r);
  const uint64_t top = ki << (52 - kExpBits);
  const ulonglong2 te = tab[ki % kN];
  const double tail = as_d(te.x);
  const uint64_t sbits = te.y + top;
  const double r2 = r * r;
  const double p23 = __fma_rn(r, C3, C2);
  const double p45 = __fma_rn(r, C5, C4);
  double tmp = __fma_rn(p23, r2, r + tail);
  tmp = __fma_rn(p45, r2 * r2, tmp);
  const double scale = as_d(sbits);
  return __fma_rn(tmp, scale, scale);
}

// math.exp (e_exp.c __exp, FMA build)
__device__ __forceinline__ double exp(double x, const ulonglong2* tab = exp_table()) {
  uint32_t abstop = top12(x) & 0x7ff;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {  // |x| < 2^-54, |x| >= 512, inf or nan
    if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x;
    if (abstop >= 0x409u) {
      if (as_u(x) == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return 1.0 + x;
      return (as_u(x) >> 63) ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
    }
    abstop = 0;  // large finite x: special-cased in the core
  }
  return exp_core<false>(x, 0.0, 0, abstop, tab);
}

// math.log (e_log.c __log, FMA build)
__device__ __forceinline__ double log(double x) {
  uint64_t ix = as_u(x);
  const uint32_t top = (uint32_t)(ix >> 48);
  const uint64_t LO = 0x3fee000000000000ull;  // asuint64(1.0 - 0x1p-4)
  if (ix - LO < 0x3ff1090000000000ull - LO) {  // close to 1.0
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = x - 1.0;
    const double r2 = r * r;
    const double r3 = r * r2;
    const double B0 = kLogB0;
    double p = __fma_rn(r, kLogB8, kLogB7);           // B7 + r*B8
    p = __fma_rn(r2, kLogB9, p);                                 // + r2*B9
    p = __fma_rn(r3, kLogB10, p);                                 // + r3*B10
    const double q4 = __fma_rn(r2, kLogB6, __fma_rn(r, kLogB5, kLogB4));
    p = __fma_rn(p, r3, q4);                                               // B4 + r*B5 + r2*B6 + r3*(...)
    const double q1 = __fma_rn(r2, kLogB3, __fma_rn(r, kLogB2, kLogB1));
    p = __fma_rn(p, r3, q1);                                               // B1 + r*B2 + r2*B3 + r3*(...)
    const double rhi = __fma_rn(-0x1p27, r, __fma_rn(r, 0x1p27, r));     // w = r*2^27; rhi = r + w - w
    const double rlo = r - rhi;
    const double rr = rhi * rhi;
    const double hi = __fma_rn(rr, B0, r);                                 // fma: w = rhi*rhi*B0; hi = r + w
    double lo = __fma_rn(rr, B0, r - hi);                                  // fma: lo = r - hi + w
    lo = __fma_rn(B0 * rlo, r + rhi, lo);                                  // fma: lo += B0*rlo*(rhi + r)
    const double y = __fma_rn(p, r3, lo);                                  // fma: y = r3*p; y += lo
    return hi + y;
  }
  if (top - 0x0010u >= 0x7ff0u - 0x0010u) {  // x < 0x1p-1022, or inf / nan / negative
    if (2 * ix == 0) return __longlong_as_double(0xfff0000000000000LL);  // -inf (divbyzero)
    if (ix == 0x7ff0000000000000ull) return x;
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return __longlong_as_double(0x7ff8000000000000LL);
    ix = as_u(x * 0x1p52) - (52ull << 52);  // subnormal: normalize
  }
  const uint64_t OFF = 0x3fe6000000000000ull;
  const uint64_t tmp = ix - OFF;
  const int i = (int)((tmp >> 45) % 128);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffull << 52));
  const double2 tl = __ldg(reinterpret_cast<const double2*>(kLogTab) + i);  // (invc, logc)
  const double invc = tl.x, logc = tl.y;
  const double z = as_d(iz);
  const double kd = (double)k;
  const double r = __fma_rn(z, invc, -1.0);                     // fma (__FP_FAST_FMA path)
  const double w = __fma_rn(kd, kLogLn2hi, logc);          // fma: kd*Ln2hi + logc
  const double hi = r + w;
  double lo = w - hi + r;
  lo = __fma_rn(kd, kLogLn2lo, lo);                        // fma: + kd*Ln2lo
  const double r2 = r * r;
  const double a12 = __fma_rn(r, kLogA2, kLogA1);  // A1 + r*A2
  const double a34 = __fma_rn(r, kLogA4, kLogA3);  // A3 + r*A4
  const double lo2 = __fma_rn(r2, kLogA0, lo);              // lo + r2*A0
  const double poly = __fma_rn(a34, r2, a12);                        // A1 + r*A2 + r2*(A3 + r*A4)
  return __fma_rn(r * r2, poly, lo2) + hi;
}

// e_pow.c log_inline: log(x) as hi + tail with ~64 bits of precision
__device__ __forceinline__ double pow_log(uint64_t ix, double& tail) {
  const uint64_t OFF = 0x3fe6955500000000ull;
  const uint64_t tmp = ix - OFF;
  const int i = (int)((tmp >> 45) % 128);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffull << 52));
  const double z = as_d(iz);
  const double kd = (double)k;
  const double2 ta = __ldg(reinterpret_cast<const double2*>(kPowTab) + 2 * i);      // (invc, pad)
  const double2 tb = __ldg(reinterpret_cast<const double2*>(kPowTab) + 2 * i + 1);  // (logc, logctail)
  const double invc = ta.x, logc = tb.x, logctail = tb.y;
  const double r = __fma_rn(z, invc, -1.0);                     // fma
  const double t1 = __fma_rn(kd, kPowLn2hi, logc);         // fma: kd*Ln2hi + logc
  const double t2 = r + t1;
  const double lo1 = __fma_rn(kd, kPowLn2lo, logctail);    // fma: kd*Ln2lo + logctail
  const double lo2 = t1 - t2 + r;
  const double ar = r * kPowA0;  // A[0] * r
  const double ar2 = r * ar;
  const double ar3 = r * ar2;
  const double hi = t2 + ar2;
  const double lo3 = __fma_rn(ar, r, -ar2);  // fma
  const double lo4 = t2 - hi + ar2;
  const double a12 = __fma_rn(r, kPowA2, kPowA1);  // A1 + r*A2
  const double a34 = __fma_rn(r, kPowA4, kPowA3);  // A3 + r*A4
  const double a56 = __fma_rn(r, kPowA6, kPowA5);  // A5 + r*A6
  const double q = __fma_rn(ar2, __fma_rn(a56, ar2, a34), a12);      // A1 + r*A2 + ar2*(A3 + r*A4 + ar2*(A5 + r*A6))
  const double lo = __fma_rn(ar3, q, lo1 + lo2 + lo3 + lo4);          // fma: lo1 + lo2 + lo3 + lo4 + ar3*q
  const double y = hi + lo;
  tail = hi - y + lo;
  return y;
}

// 0 not an integer, 1 odd integer, 2 even integer (iy: non-zero finite)
__device__ __forceinline__ int checkint(uint64_t iy) {
  const int e = (int)(iy >> 52 & 0x7ff);
  if (e < 0x3ff) return 0;
  if (e > 0x3ff + 52) return 2;
  if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
  if (iy & (1ull << (0x3ff + 52 - e))) return 1;
  return 2;
}
__device__ __forceinline__ bool zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * 0x7ff0000000000000ull - 1; }

// float.__pow__ for finite floats (e_pow.c __pow, FMA build)
__device__ __forceinline__ double pow(double x, double y) {
  const double INF = __longlong_as_double(0x7ff0000000000000LL);
  uint64_t sign_bias = 0;
  uint64_t ix = as_u(x);
  const uint64_t iy = as_u(y);
  uint32_t topx = top12(x);
  const uint32_t topy = top12(y);
  if (topx - 0x001u >= 0x7ffu - 0x001u || (topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
    if (zeroinfnan(iy)) {
      if (2 * iy == 0) return 1.0;
      if (ix == 0x3ff0000000000000ull) return 1.0;
      if (2 * ix > 2 * 0x7ff0000000000000ull || 2 * iy > 2 * 0x7ff0000000000000ull) return x + y;
      if (2 * ix == 2 * 0x3ff0000000000000ull) return 1.0;
      if ((2 * ix < 2 * 0x3ff0000000000000ull) == !(iy >> 63)) return 0.0;
      return y * y;
    }
    if (zeroinfnan(ix)) {
      double x2 = x * x;
      if ((ix >> 63) && checkint(iy) == 1) x2 = -x2;
      return (iy >> 63) ? 1.0 / x2 : x2;
    }
    if (ix >> 63) {  // finite x < 0
      const int yint = checkint(iy);
      if (yint == 0) return __longlong_as_double(0x7ff8000000000000LL);
      if (yint == 1) sign_bias = 0x800ull << kExpBits;
      ix &= 0x7fffffffffffffffull;
      topx &= 0x7ff;
    }
    if ((topy & 0x7ffu) - 0x3beu >= 0x43eu - 0x3beu) {
      if (ix == 0x3ff0000000000000ull) return 1.0;
      if ((topy & 0x7ffu) < 0x3beu) return ix > 0x3ff0000000000000ull ? 1.0 + y : 1.0 - y;
      return (ix > 0x3ff0000000000000ull) == (topy < 0x800u) ? INF : 0.0;
    }
    if (topx == 0) ix = (as_u(x * 0x1p52) & 0x7fffffffffffffffull) - (52ull << 52);  // subnormal x
  }
  double lo;
  const double hi = pow_log(ix, lo);
  const double ehi = y * hi;
  const double elo = __fma_rn(y, lo, __fma_rn(hi, y, -ehi));  // fma: y*lo + fma(y, hi, -ehi)
  // exp_inline(ehi, elo, sign_bias)
  uint32_t abstop = top12(ehi) & 0x7ff;
  if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
    if ((int32_t)(abstop - 0x3c9u) < 0) {
      const double one = 1.0 + ehi;
      return sign_bias ? -one : one;
    }
    if (abstop >= 0x409u) {
      const double big = (as_u(ehi) >> 63) ? 0.0 : INF;
      return sign_bias ? -big : big;
    }
    abstop = 0;
  }
  return exp_core<true>(ehi, elo, sign_bias, abstop, exp_table());
}

// math.log1p / numpy's npy_log1p (s_log1p.c, fdlibm algorithm; glibc's FMA
// build __log1p_fma).  Used by numpy's ziggurat tails (distributions.c).
__device__ __forceinline__ double set_high(double u, uint32_t hi) {
  return as_d(((uint64_t)hi << 32) | (as_u(u) & 0xffffffffull));
}
__device__ __forceinline__ double log1p(double x) {
  constexpr double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
  constexpr double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2, Lp3 = 0x1.2492494229359p-2;
  constexpr double Lp4 = 0x1.c71c51d8e78afp-3, Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3;
  constexpr double Lp7 = 0x1.2f112df3e5244p-3;
  const int32_t hx = (int32_t)(as_u(x) >> 32);
  const uint32_t ax = (uint32_t)hx & 0x7fffffffu;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {                           // x < 0.41422
    if (ax >= 0x3ff00000u) {                       // x <= -1
      if (x == -1.0) return __longlong_as_double(0xfff0000000000000LL);
      return __longlong_as_double(0x7ff8000000000000LL);
    }
    if (ax < 0x3e200000u) {                        // |x| < 2^-29
      if (ax < 0x3c900000u) return x;              // |x| < 2^-54
      return __fma_rn(-(x * x), 0.5, x);           // fma: x - x*x*0.5
    }
    if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx > 0x7fefffff) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = (int)(as_u(u) >> 32);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);  // correction term
      c = __ddiv_rn(c, u);
    } else {
      u = x;
      hu = (int)(as_u(u) >> 32);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = set_high(u, (uint32_t)hu | 0x3ff00000u);  // normalize u
    } else {
      k += 1;
      u = set_high(u, (uint32_t)hu | 0x3fe00000u);  // normalize u/2
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = (f * 0.5) * f;
  const double kd = (double)k;
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return __fma_rn(kd, ln2_hi, __fma_rn(kd, ln2_lo, c));  // fma x2: c += k*ln2_lo; k*ln2_hi + c
    }
    const double R = __fma_rn(-f, 0x1.5555555555555p-1, 1.0) * hfsq;  // fma: hfsq*(1.0 - 0.666..*f)
    if (k == 0) return f - R;
    return __fma_rn(kd, ln2_hi, -((R - __fma_rn(kd, ln2_lo, c)) - f));
  }
  const double s = __ddiv_rn(f, f + 2.0);
  const double z = s * s;
  const double R2 = __fma_rn(z, Lp3, Lp2), R3 = __fma_rn(z, Lp5, Lp4), R4 = __fma_rn(z, Lp7, Lp6);
  const double z2 = z * z, z4 = z2 * z2, z6 = z2 * z4;
  double R = __fma_rn(z, Lp1, z2 * R2);  // fma: R1 + z2*R2, R1 = z*Lp1
  R = __fma_rn(z4, R3, R);
  R = __fma_rn(z6, R4, R);
  const double q = (R + hfsq) * s;  // s*(hfsq+R)
  if (k == 0) return f - (hfsq - q);
  const double w = __fma_rn(kd, ln2_lo, c) + q;
  return __fma_rn(kd, ln2_hi, -((hfsq - w) - f));  // fmsub: k*ln2_hi - ((hfsq - (...)) - f)
}

}  // namespace glibc
}  // namespace strait
