// strait_predictor.cu — the refit's building blocks as standalone entry points:
// loss_gradient (predictor.py:271-309) for many samples under one parameter
// vector, one adam_step (predictor.py:124-145) and the Huber pieces
// (:148-158).  strait_refit fuses the same arithmetic, sample after sample, in
// one warp (strait_refit.cuh); these serve the reference's function-level API.
#include <cuda_runtime.h>

#include "strait_capi.cuh"
#include "strait_device.cuh"

namespace {

using strait::py_max;
using strait::py_min;

template <int NM>
__global__ void loss_grad_kernel(const double* __restrict__ P, double cap, double delta, const double* __restrict__ twa,
                                 const double* __restrict__ cmp_, const double* __restrict__ mem_,
                                 const int8_t* __restrict__ prio_, const double* __restrict__ actual_, int64_t n,
                                 double* __restrict__ out_pred, double* __restrict__ out_res,
                                 uint8_t* __restrict__ out_sat, double* __restrict__ out_grad) {
  constexpr int NP = NM + 7;
  const double scale = P[0], base = P[1], offset = P[2];
  const double log_b = strait::dlog(base);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double tw[NM];
#pragma unroll
    for (int k = 0; k < NM; ++k) tw[k] = twa[k * n + i];
    const double cmp = cmp_[i], mem = mem_[i];
    const int prio = prio_[i];
    double x = P[3 + NM] * cmp + P[4 + NM] * mem;  // pressure_exponent: self terms first
#pragma unroll
    for (int k = 0; k < NM; ++k) x += P[3 + k] * tw[k];
    const double z = x * log_b;  // _raw_effect
    bool saturated;
    double inner, pow_bx = 0.0;
    if (z > strait::kLogSaturate) {
      saturated = true;
      inner = __longlong_as_double(0x7ff0000000000000LL);
    } else {
      pow_bx = strait::dexp(z);
      inner = scale * pow_bx + offset;
      saturated = inner >= cap;
    }
    const double eff = saturated ? cap : py_min(py_max(inner, 0.0), cap);
    const int own = NM + (prio == 0 ? 5 : 6);
    const double cf = P[own];
    const double predicted = 1.0 + eff * cf;
    const double residual = predicted - actual_[i];
    const double g = fabs(residual) <= delta ? residual : (residual > 0 ? delta : -delta);  // huber_grad
    double d[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) d[k] = 0.0;
    if (!(saturated || inner <= 0.0 || inner >= cap)) {  // _prediction_gradient, unclamped
      const double zz = scale * pow_bx;
      d[0] = pow_bx * cf;
      d[1] = scale * x * strait::dexp((x - 1.0) * log_b) * cf;
      d[2] = cf;
#pragma unroll
      for (int k = 0; k < NM; ++k) d[3 + k] = zz * log_b * tw[k] * cf;
      d[3 + NM] = zz * log_b * cmp * cf;
      d[4 + NM] = zz * log_b * mem * cf;
    }
    d[own] = eff;
#pragma unroll
    for (int k = 0; k < NP; ++k) out_grad[k * n + i] = g * d[k];
    out_pred[i] = predicted;
    out_res[i] = residual;
    if (out_sat) out_sat[i] = saturated;
  }
}

template <int NM>
void launch_loss_grad(const double* P, double cap, double delta, const double* twa, const double* cmp,
                      const double* mem, const int8_t* prio, const double* actual, int64_t n, double* pred,
                      double* res, uint8_t* sat, double* grad, cudaStream_t st) {
  const int64_t b = (n + 127) / 128;
  loss_grad_kernel<NM><<<(unsigned)(b < 4096 ? b : 4096), 128, 0, st>>>(P, cap, delta, twa, cmp, mem, prio, actual,
                                                                        n, pred, res, sat, grad);
}

__global__ void adam_kernel(double* __restrict__ values, double* __restrict__ m, double* __restrict__ v,
                            const double* __restrict__ grads, const uint8_t* __restrict__ active, int n, double bc1,
                            double bc2, double lr, double b1, double b2, double eps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || (active && !active[i])) return;  // inactive: value and moments untouched
  const double g = grads[i];
  m[i] = b1 * m[i] + (1.0 - b1) * g;
  v[i] = b2 * v[i] + (1.0 - b2) * g * g;
  const double m_hat = m[i] / bc1;
  const double v_hat = v[i] / bc2;
  values[i] -= lr * m_hat / (sqrt(v_hat) + eps);
}

__global__ void huber_kernel(const double* __restrict__ r, double delta, int64_t n, double* __restrict__ loss,
                             double* __restrict__ grad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = r[i], a = fabs(x);
    if (loss) loss[i] = a <= delta ? 0.5 * x * x : delta * (a - 0.5 * delta);
    if (grad) grad[i] = a <= delta ? x : (x > 0 ? delta : -delta);
  }
}

}  // namespace

extern "C" int strait_loss_gradient(const double* params, int32_t n_metrics, double effect_cap, double huber_delta,
                                    const double* twa, const double* self_cmp, const double* self_mem,
                                    const int8_t* prio, const double* actual, int64_t n, double* out_predicted,
                                    double* out_residual, uint8_t* out_saturated, double* out_grad, void* stream) {
  if (n_metrics < 1 || n_metrics > STRAIT_MAX_METRICS || n < 0)
    return strait::set_error(STRAIT_EINVAL, "strait_loss_gradient: bad arguments");
  if (!n) return STRAIT_OK;
  if (!params || !twa || !self_cmp || !self_mem || !prio || !actual || !out_predicted || !out_residual || !out_grad)
    return strait::set_error(STRAIT_EINVAL, "strait_loss_gradient: null buffer");
  STRAIT_DISPATCH_NM(n_metrics, launch_loss_grad, params, effect_cap, huber_delta, twa, self_cmp, self_mem, prio,
                     actual, n, out_predicted, out_residual, out_saturated, out_grad, (cudaStream_t)stream);
  return strait::check_launch("strait_loss_gradient");
}

extern "C" int strait_adam_step(double* values, double* m, double* v, const double* grads, const uint8_t* active,
                                int32_t n, double bc1, double bc2, double learning_rate, double beta1, double beta2,
                                double eps, void* stream) {
  if (n < 0) return strait::set_error(STRAIT_EINVAL, "strait_adam_step: n < 0");
  if (!n) return STRAIT_OK;
  if (!values || !m || !v || !grads) return strait::set_error(STRAIT_EINVAL, "strait_adam_step: null buffer");
  adam_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(values, m, v, grads, active, n, bc1, bc2,
                                                                 learning_rate, beta1, beta2, eps);
  return strait::check_launch("strait_adam_step");
}

extern "C" int strait_huber(const double* residual, double delta, int64_t n, double* out_loss, double* out_grad,
                            void* stream) {
  if (n < 0 || (n && !residual)) return strait::set_error(STRAIT_EINVAL, "strait_huber: bad arguments");
  if (!n) return STRAIT_OK;
  const int64_t b = (n + 255) / 256;
  huber_kernel<<<(unsigned)(b < 4096 ? b : 4096), 256, 0, (cudaStream_t)stream>>>(residual, delta, n, out_loss,
                                                                                   out_grad);
  return strait::check_launch("strait_huber");
}
