// strait_refit.cuh — the online refit (R14-R16) as one warp.
//
// Restates InterferencePredictor.update (predictor.py:345-363) applied to a
// sequence of FeedbackSamples strictly in order: lane k owns parameter k of
// the canonical vector (predictor.py:64-77) together with its Adam moments.
// Per sample every lane recomputes the prediction under the CURRENT
// parameters (predictor.py:271-300), lane k forms dLoss/dtheta_k
// (loss_gradient + huber_grad, :303-309, :155-158), a warp vote implements the
// non-finite skip (:352-353), then adam_step (:124-145) with the other class's
// coefficient inactive and enforce_floors (:98-102).
#pragma once

#include "strait_device.cuh"

namespace strait {

template <int NM>
__device__ void refit_warp(const StraitRefitArgs& a, double* sP /* shared, >= NM+7 */) {
  constexpr int NP = NM + 7;
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const bool owner = lane < NP;
  double p = owner ? a.state[lane] : 0.0;
  double m = owner ? a.state[NP + lane] : 0.0;
  double v = owner ? a.state[2 * NP + lane] : 0.0;
  int64_t step = *a.step;
  const double cap = a.effect_cap, delta = a.huber_delta;
  const double b1 = a.beta1, b2 = a.beta2, lr = a.learning_rate, eps = a.eps;
  const double omb1 = 1.0 - b1, omb2 = 1.0 - b2;  // (1.0 - b1), (1.0 - b2) as in adam_step
  if (owner) sP[lane] = p;
  __syncwarp();

  for (int64_t i = 0; i < a.n; ++i) {
    // sample inputs (independent of the parameter chain; the compiler hoists them)
    double tw[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) tw[k] = a.twa[k * a.n + i];
    const double cmp = a.self_cmp[i], mem = a.self_mem[i], actual = a.actual[i];
    const int prio = a.prio[i];

    // prediction under current parameters (predictor.py:276-283)
    const double scale = sP[0], base = sP[1], offset = sP[2];
    double x = sP[3 + NM] * cmp + sP[4 + NM] * mem;
#pragma unroll
    for (int k = 0; k < NM; ++k) x += sP[3 + k] * tw[k];
    const double log_b = dlog(base);
    const double z = x * log_b;
    bool saturated;
    double inner, pow_bx = 0.0;
    if (z > kLogSaturate) {
      saturated = true;
      inner = __longlong_as_double(0x7ff0000000000000LL);  // math.inf
    } else {
      pow_bx = dexp(z);
      inner = scale * pow_bx + offset;
      saturated = inner >= cap;
    }
    const double eff = saturated ? cap : py_min(py_max(inner, 0.0), cap);
    const int own = NM + (prio == 0 ? 5 : 6), other = NM + (prio == 0 ? 6 : 5);
    const double cf = sP[own];
    const double predicted = 1.0 + eff * cf;

    // d(prediction)/d(theta_lane) (predictor.py:285-299)
    double d = 0.0;
    const bool clamp_active = saturated || inner <= 0.0 || inner >= cap;
    if (!clamp_active && owner) {
      const double zz = scale * pow_bx;
      if (lane == 0) d = pow_bx * cf;
      else if (lane == 1) d = scale * x * dexp((x - 1.0) * log_b) * cf;
      else if (lane == 2) d = cf;
      else if (lane < 3 + NM) {
        double ai = 0.0;
#pragma unroll
        for (int k = 0; k < NM; ++k)
          if (lane == 3 + k) ai = tw[k];
        d = zz * log_b * ai * cf;
      } else if (lane == 3 + NM) d = zz * log_b * cmp * cf;
      else if (lane == 4 + NM) d = zz * log_b * mem * cf;
    }
    if (lane == own) d = eff;

    const double residual = predicted - actual;
    const double g = fabs(residual) <= delta ? residual : (residual > 0 ? delta : -delta);
    const double gk = g * d;
    const bool finite = __all_sync(full, !owner || isfinite(gk)) && isfinite(residual);

    if (lane == 0) {
      if (a.out_predicted) a.out_predicted[i] = predicted;
      if (a.out_residual) a.out_residual[i] = residual;
      if (a.out_flags) a.out_flags[i] = (uint8_t)((finite ? 0 : 1) | (saturated ? 2 : 0));
    }
    if (!finite) continue;  // UpdateResult(skipped=True): no step

    ++step;
    const double bc1 = step <= a.n_bc ? a.bc1[step - 1] : 1.0;
    const double bc2 = step <= a.n_bc ? a.bc2[step - 1] : 1.0;
    if (owner && lane != other) {
      m = b1 * m + omb1 * gk;
      v = b2 * v + omb2 * gk * gk;
      const double m_hat = m / bc1;
      const double v_hat = v / bc2;
      p -= lr * m_hat / (sqrt(v_hat) + eps);
      if (lane == 0) p = py_max(p, 1e-6);        // MIN_SCALE
      if (lane == 1) p = py_max(p, 1.0 + 1e-6);  // MIN_BASE
    }
    if (lane == NM + 5 || lane == NM + 6) p = py_max(p, 1e-6);  // MIN_PRIORITY_COEFF (both classes)
    __syncwarp();
    if (owner) sP[lane] = p;
    __syncwarp();
  }
  if (owner) {
    a.state[lane] = p;
    a.state[NP + lane] = m;
    a.state[2 * NP + lane] = v;
  }
  if (lane == 0) *a.step = step;
}

}  // namespace strait
