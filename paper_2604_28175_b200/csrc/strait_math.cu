// strait_math.cu — elementwise device exp / log / pow (strait_libm.cuh), the
// transcendental functions of the estimator (predictor.py:181-184,289-293)
// and the ground truth (oracle.py:73), exported so their bit-identity with the
// host libm can be checked directly (tests/test_libm_gpu.py).
#include <cuda_runtime.h>

#include "strait_capi.cuh"
#include "strait_device.cuh"

namespace {
__global__ void math_kernel(int fn, const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                            double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = x[i];
    if (fn == 4) {  // the certified shared-divisor quotient (strait_device.cuh div_shared), one element
      double num[1] = {a}, q[1];
      strait::div_shared(num, y[i], q);
      out[i] = q[0];
      continue;
    }
    out[i] = fn == 0 ? strait::dexp(a) : fn == 1 ? strait::dlog(a) : fn == 2 ? strait::dpow(a, y[i])
                                                                  : strait::glibc::log1p(a);
  }
}

// ground_truth_slowdown (oracle.py:55-77), one element per thread; the
// expression order is Python's (no FMA contraction: --fmad=false)
__global__ void gt_kernel(const StraitGroundTruth gt, const double* __restrict__ co, const double* __restrict__ cmp,
                          const double* __restrict__ mem, const int8_t* __restrict__ prio,
                          const double* __restrict__ noise, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double x = gt.w_cmp * cmp[i] + gt.w_mem * mem[i];
    for (int k = 0; k < gt.n_metrics; ++k) x += gt.w[k] * co[k * n + i];
    double effect = gt.family == 0 ? gt.scale * strait::dpow(gt.base, x) + gt.offset : gt.scale * x * x + gt.offset;
    effect = strait::py_max(0.0, effect);
    const double f = prio[i] == 0 ? gt.pf_high : gt.pf_low;
    out[i] = 1.0 + effect * f * (noise ? noise[i] : 1.0);
  }
}
}  // namespace

extern "C" int strait_gt_slowdown(const StraitGroundTruth* gt, const double* co, const double* cmp, const double* mem,
                                  const int8_t* prio, const double* noise, int64_t n, double* out, void* stream) {
  if (!gt || n < 0 || gt->n_metrics < 1 || gt->n_metrics > STRAIT_MAX_METRICS || (gt->family != 0 && gt->family != 1))
    return strait::set_error(STRAIT_EINVAL, "strait_gt_slowdown: bad arguments");
  if (!n) return STRAIT_OK;
  if (!co || !cmp || !mem || !prio || !out) return strait::set_error(STRAIT_EINVAL, "strait_gt_slowdown: null buffer");
  const int64_t blocks64 = (n + 255) / 256;
  const unsigned blocks = (unsigned)(blocks64 < 4096 ? blocks64 : 4096);
  gt_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*gt, co, cmp, mem, prio, noise, n, out);
  return strait::check_launch("strait_gt_slowdown");
}

extern "C" int strait_math(int32_t fn, const double* x, const double* y, int64_t n, double* out, void* stream) {
  if (fn < 0 || fn > 4 || n < 0 || (n && (!x || !out || ((fn == 2 || fn == 4) && !y))))
    return strait::set_error(STRAIT_EINVAL, "strait_math: bad arguments");
  if (!n) return STRAIT_OK;
  const int64_t blocks64 = (n + 255) / 256;
  const unsigned blocks = (unsigned)(blocks64 < 4096 ? blocks64 : 4096);
  math_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(fn, x, y, n, out);
  return strait::check_launch("strait_math");
}
