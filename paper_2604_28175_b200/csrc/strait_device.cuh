// strait_device.cuh — binary64 device arithmetic of the Strait estimator.
//
// Every helper restates one reference function (file:line under
// /root/reference/pkg/src/infersim) in its exact left-to-right evaluation
// order.  The library is compiled with --fmad=false -prec-div=true
// -prec-sqrt=true so that each `a * b + c` below rounds twice, like CPython.
// exp/log/pow are restatements of the reference host's glibc routines
// (strait_libm.cuh), so results are bit-identical to the reference.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/strait.h"
#include "strait_libm.cuh"

namespace strait {

// exp / log / pow with the reference host's bits (strait_libm.cuh).  Build with
// -DSTRAIT_LIBM=0 to use libdevice instead (<= 1-2 ulp, for A/B timing only).
#ifndef STRAIT_LIBM
#define STRAIT_LIBM 1
#endif
#if STRAIT_LIBM
__device__ __forceinline__ double dexp(double x, const ulonglong2* tab = glibc::exp_table()) {
  return glibc::exp(x, tab);
}
__device__ __forceinline__ double dlog(double x) { return glibc::log(x); }
__device__ __forceinline__ double dpow(double x, double y) { return glibc::pow(x, y); }
#else
__device__ __forceinline__ double dexp(double x, const ulonglong2* = nullptr) { return ::exp(x); }
__device__ __forceinline__ double dlog(double x) { return ::log(x); }
__device__ __forceinline__ double dpow(double x, double y) { return ::pow(x, y); }
#endif

constexpr double kLogSaturate = 500.0;  // predictor.py:27 _LOG_SATURATE
constexpr int kMaxM = STRAIT_MAX_METRICS;
constexpr int kMaxP = STRAIT_MAX_METRICS + 7;

// CPython builtin max(a, b) / min(a, b): first-wins, NaN-propagating.
__host__ __device__ __forceinline__ double py_max(double a, double b) { return (b > a) ? b : a; }
__host__ __device__ __forceinline__ double py_min(double a, double b) { return (b < a) ? b : a; }

// q[i] = a[i] / b for i < N, each the correctly rounded binary64 quotient (as
// __ddiv_rn), with ONE divisor: the reciprocal is formed once (rcp.approx +
// two Newton steps), each quotient gets one Markstein step, and each is then
// CERTIFIED exactly — the residual r = a - q*b is exact (FMA, operands in
// range), and |r| < ulp(q)/2 * |b| with q not a power of two proves q is the
// nearest binary64 to a/b.  Any operand out of range, any tie or any failed
// certificate sends all N to __ddiv_rn.  Straight-line in the common case, so
// the N quotients overlap (N sequential __ddiv_rn do not: each carries its
// slow-path branch).
template <int N>
__device__ __forceinline__ void div_shared(const double (&a)[N], double b, double (&q)[N]) {
  const double ab = fabs(b);
  bool ok = ab >= 0x1p-400 && ab <= 0x1p400;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = __fma_rn(-b, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-b, r, 1.0);
  r = __fma_rn(r, e, r);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const double q0 = a[i] * r;
    const double q1 = __fma_rn(__fma_rn(-b, q0, a[i]), r, q0);
    const double res = __fma_rn(-b, q1, a[i]);  // a - q1*b, exact
    const unsigned long long qb = (unsigned long long)__double_as_longlong(q1);
    const int ex = (int)((qb >> 52) & 0x7ff);
    // |q1| in [2^-400, 2^400] and not a power of two (its lower neighbour is a full ulp away)
    ok = ok && ex >= 1023 - 400 && ex <= 1023 + 400 && (qb & 0xfffffffffffffull) != 0;
    const double half_ulp = __longlong_as_double((long long)((unsigned long long)(ex - 53) << 52));
    ok = ok && fabs(res) < half_ulp * ab;
    q[i] = q1;
  }
  if (!ok) {
#pragma unroll
    for (int i = 0; i < N; ++i) q[i] = __ddiv_rn(a[i], b);
  }
}

// Transcendental policy of the predictor: inlined (default), or routed by a
// kernel to shared out-of-line copies (MathT with the same static members).
struct InlineMath {
  static constexpr bool kInline = true;  // exp is inlined: two effects may interleave (Pred::effect2)
  static __device__ __forceinline__ double exp(double x, const ulonglong2* tab) { return dexp(x, tab); }
  static __device__ __forceinline__ double log(double x) { return dlog(x); }
};

// Parameters of one predictor, staged in registers/shared memory by callers.
template <int NM, typename MathT = InlineMath>
struct Pred {
  double scale, offset, log_base;  // log_base = math.log(params.base), hoisted (same value per call)
  double w[NM];
  double w_cmp, w_mem;
  double coeff[2];  // [HIGH, LOW]
  double cap;
  const ulonglong2* etab;  // exp table (global, or a kernel's shared-memory copy)

  __device__ __forceinline__ void load(const double* __restrict__ P, double effect_cap) {
    scale = P[0];
    log_base = MathT::log(P[1]);
    offset = P[2];
#pragma unroll
    for (int i = 0; i < NM; ++i) w[i] = P[3 + i];
    w_cmp = P[3 + NM];
    w_mem = P[4 + NM];
    coeff[0] = P[5 + NM];
    coeff[1] = P[6 + NM];
    cap = effect_cap;
#if STRAIT_LIBM
    etab = glibc::exp_table();
#endif
  }

  // predictor.py:161-176 pressure_exponent — self terms first, then metrics.
  __device__ __forceinline__ double exponent(const double (&a)[NM], double cmp, double mem) const {
    double x = w_cmp * cmp + w_mem * mem;
#pragma unroll
    for (int i = 0; i < NM; ++i) x += w[i] * a[i];
    return x;
  }

  // predictor.py:179-195 _raw_effect + kernel_effect.
  __device__ __forceinline__ double effect(double x, bool& saturated) const {
    const double z = x * log_base;
    if (z > kLogSaturate) {
      saturated = true;
      return cap;
    }
    const double inner = scale * MathT::exp(z, etab) + offset;
    saturated = inner >= cap;
    if (saturated) return cap;
    return py_min(py_max(inner, 0.0), cap);
  }

  // predictor.py:198-216 interference_degree(kernel_effect(pressure_exponent(...))).
  __device__ __forceinline__ double predict(const double (&a)[NM], double cmp, double mem, int prio,
                                            bool& saturated) const {
    const double x = exponent(a, cmp, mem);
    const double eff = effect(x, saturated);
    return 1.0 + eff * (prio == 0 ? coeff[0] : coeff[1]);
  }
  __device__ __forceinline__ double predict(const double (&a)[NM], double cmp, double mem,
                                            int prio) const {
    bool s;
    return predict(a, cmp, mem, prio, s);
  }
  // exp(z1), exp(z2) as one block (interleaved chains); bit-identical to two exp calls
  __device__ __forceinline__ void exp2v(double z1, double z2, double& e1, double& e2) const {
#if STRAIT_LIBM
    bool special = false;
    e1 = glibc::exp_common(z1, etab, special);
    e2 = glibc::exp_common(z2, etab, special);
    if (!special) return;
#endif
    e1 = MathT::exp(z1, etab);
    e2 = MathT::exp(z2, etab);
  }
  // Two kernel_effect()s as one block, so their exp chains interleave when exp
  // is inlined (bit-identical to two effect() calls; the inputs that need the
  // saturation or exp()'s special cases take effect() itself).
  __device__ __forceinline__ void effect2(double x1, double x2, double& e1, double& e2) const {
#if STRAIT_LIBM
    if constexpr (MathT::kInline) {
      const double z1 = x1 * log_base, z2 = x2 * log_base;
      bool special = z1 > kLogSaturate || z2 > kLogSaturate;
      const double p1 = glibc::exp_common(z1, etab, special), p2 = glibc::exp_common(z2, etab, special);
      if (!special) {
        const double in1 = scale * p1 + offset, in2 = scale * p2 + offset;
        e1 = in1 >= cap ? cap : py_min(py_max(in1, 0.0), cap);
        e2 = in2 >= cap ? cap : py_min(py_max(in2, 0.0), cap);
        return;
      }
    }
#endif
    bool s;
    e1 = effect(x1, s);
    e2 = effect(x2, s);
  }
#if STRAIT_LIBM
  // Two predictions for the same self terms and priority (a running entry's
  // intf_cur and intf_new) as one straight-line block, so their dependent
  // chains interleave.  Bit-identical to two predict() calls: the same
  // operations in the same order; the inputs that need exp()'s special cases
  // or the z > 500 saturation take predict() itself.
  __device__ __forceinline__ void predict2(const double (&a1)[NM], const double (&a2)[NM], double cmp, double mem,
                                           int prio, double& out1, double& out2) const {
    const double x1 = exponent(a1, cmp, mem), x2 = exponent(a2, cmp, mem);
    const double z1 = x1 * log_base, z2 = x2 * log_base;
    bool special = z1 > kLogSaturate || z2 > kLogSaturate;
    const double e1 = glibc::exp_common(z1, etab, special), e2 = glibc::exp_common(z2, etab, special);
    if (special) {
      out1 = predict(a1, cmp, mem, prio);
      out2 = predict(a2, cmp, mem, prio);
      return;
    }
    const double in1 = scale * e1 + offset, in2 = scale * e2 + offset;
    const double f1 = in1 >= cap ? cap : py_min(py_max(in1, 0.0), cap);
    const double f2 = in2 >= cap ? cap : py_min(py_max(in2, 0.0), cap);
    const double cf = prio == 0 ? coeff[0] : coeff[1];
    out1 = 1.0 + f1 * cf;
    out2 = 1.0 + f2 * cf;
  }
#endif
};

// Runtime-NM dispatch: instantiate `F<NM>` for NM = 1..8.
#define STRAIT_DISPATCH_NM(nm, F, ...)                 \
  switch (nm) {                                        \
    case 1: F<1>(__VA_ARGS__); break;                  \
    case 2: F<2>(__VA_ARGS__); break;                  \
    case 3: F<3>(__VA_ARGS__); break;                  \
    case 4: F<4>(__VA_ARGS__); break;                  \
    case 5: F<5>(__VA_ARGS__); break;                  \
    case 6: F<6>(__VA_ARGS__); break;                  \
    case 7: F<7>(__VA_ARGS__); break;                  \
    case 8: F<8>(__VA_ARGS__); break;                  \
    default: break;                                    \
  }

}  // namespace strait
