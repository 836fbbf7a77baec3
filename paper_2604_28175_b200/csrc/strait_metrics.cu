// strait_metrics.cu — compute_metrics (metrics.py:88-158) of finished replays on
// the device: class counts and windowed goodput (one CTA per replay), exact
// nearest-rank percentiles by MSB-first radix SELECT on the value bits (one
// CTA per replay and series; 8 passes of 8-bit digit histograms, three ranks
// at once), and the per-batch error series.
#include <cuda_runtime.h>
#include <math.h>

#include "../../include/strait_replay.h"
#include "strait_capi.cuh"

namespace {

constexpr int kThreads = 256;

// CPython float floor division (Objects/floatobject.c float_floor_div via
// float_divmod) for the goodput window index `completion // window_ms`.
__device__ __forceinline__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = __ddiv_rn(vx - mod, wx);
  if (mod) {
    if ((wx < 0) != (mod < 0)) {
      mod += wx;
      div -= 1.0;
    }
  }
  double floordiv;
  if (div) {
    floordiv = floor(div);
    if (div - floordiv > 0.5) floordiv += 1.0;
  } else {
    floordiv = copysign(0.0, __ddiv_rn(vx, wx));
  }
  return floordiv;
}

__global__ void counts_kernel(const StraitMetricsArgs a) {
  const int64_t r = blockIdx.x;
  const int64_t lo = a.req_off[r], hi = a.req_off[r + 1];
  const int W = a.max_windows;
  __shared__ unsigned long long cnt[2][4];
  __shared__ int glen[2];
  __shared__ int flags;
  if (threadIdx.x < 8) cnt[threadIdx.x / 4][threadIdx.x % 4] = 0;
  if (threadIdx.x < 2) glen[threadIdx.x] = 0;
  if (threadIdx.x == 0) flags = 0;
  for (int64_t i = threadIdx.x; i < 2 * (int64_t)W; i += blockDim.x) a.goodput[r * 2 * W + i] = 0;
  __syncthreads();
  const double wms = a.window_ms[r];
  for (int64_t g = lo + threadIdx.x; g < hi; g += blockDim.x) {
    const int c = a.model_prio[a.arr_model[g]] == 0 ? 0 : 1;
    const int st = a.req_status[g];
    atomicAdd(&cnt[c][0], 1ull);  // arrivals
    if (st == 2) {                // dropped counts as a violation (metrics.py:107-110)
      atomicAdd(&cnt[c][2], 1ull);
      atomicAdd(&cnt[c][3], 1ull);
    } else if (st == 0) {         // completion "" => partial report
      atomicOr(&flags, 1);
    } else {
      atomicAdd(&cnt[c][1], 1ull);
      if (a.req_violated[g]) {
        atomicAdd(&cnt[c][3], 1ull);
      } else {
        const double w = py_floordiv(a.req_completion[g], wms);
        const long long wi = (long long)w;
        if (wi >= 0 && wi < W) {
          atomicAdd((unsigned long long*)&a.goodput[(r * 2 + c) * W + wi], 1ull);
          atomicMax(&glen[c], (int)wi + 1);
        } else {
          atomicOr(&flags, 2);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < 8) a.class_counts[r * 8 + threadIdx.x] = (int64_t)cnt[threadIdx.x / 4][threadIdx.x % 4];
  if (threadIdx.x < 2) a.goodput_len[r * 2 + threadIdx.x] = glen[threadIdx.x];
  if (threadIdx.x == 0) a.partial[r] = (uint8_t)flags;
}

// value of element i of series s of replay r (false if i is not in the series)
__device__ __forceinline__ bool series_value(const StraitMetricsArgs& a, int64_t r, int s, int64_t i, double& v) {
  const int64_t lo = a.req_off[r];
  if (s < 2) {
    const int64_t g = lo + i;
    if (a.req_status[g] != 1 || (a.model_prio[a.arr_model[g]] == 0 ? 0 : 1) != s) return false;
    v = a.req_completion[g] - a.arr_time[g];  // row["latency"] (simulation.py:259-276)
    return true;
  }
  const int64_t b = lo + i;
  if (s == 2) {
    const double act = a.fb_actual[b];
    v = fabs(__ddiv_rn(a.fb_predicted[b] - act, act));
  } else if (s == 3) {
    const double act = a.b_completion[b] - a.b_front[b];  // actual_latency
    v = fabs(__ddiv_rn(a.dec_est_latency[b] - act, act));
  } else {
    const double iso = a.kernel_table[(int64_t)a.dec_model[b] * a.table_stride + a.dec_size[b] - 1];
    v = __ddiv_rn(fabs((a.b_kernel_end[b] - a.b_kernel_start[b]) - iso), iso);
  }
  return true;
}

// order-preserving map of binary64 onto uint64
__device__ __forceinline__ unsigned long long okey(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double okey_inv(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void select_kernel(const StraitMetricsArgs a) {
  const int64_t r = blockIdx.x;
  const int s = blockIdx.y;
  const int64_t n_elem = s < 2 ? a.req_off[r + 1] - a.req_off[r] : a.counters[r * STRAIT_RC_N + STRAIT_RC_COMPLETED];
  __shared__ unsigned int hist[3][256];
  __shared__ unsigned long long count, prefix[3];
  __shared__ long long rank[3];
  if (threadIdx.x == 0) count = 0;
  __syncthreads();
  unsigned long long local = 0;
  for (int64_t i = threadIdx.x; i < n_elem; i += blockDim.x) {
    double v;
    local += series_value(a, r, s, i, v);
  }
  atomicAdd(&count, local);
  __syncthreads();
  const long long n = (long long)count;
  double* out = a.pct + (r * STRAIT_MS_N + s) * 3;
  if (threadIdx.x == 0) a.series_count[r * STRAIT_MS_N + s] = n;
  if (n == 0) {
    if (threadIdx.x < 3) out[threadIdx.x] = __longlong_as_double(0x7ff8000000000000LL);
    return;
  }
  if (threadIdx.x < 3) {  // nearest_rank: max(1, ceil(pct / 100 * n)), clipped to n (metrics.py:16-22)
    const double pct = threadIdx.x == 0 ? 50.0 : threadIdx.x == 1 ? 95.0 : 99.0;
    long long k = (long long)ceil(__dmul_rn(__ddiv_rn(pct, 100.0), (double)n));
    if (k < 1) k = 1;
    if (k > n) k = n;
    rank[threadIdx.x] = k;
    prefix[threadIdx.x] = 0;
  }
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < n_elem; i += blockDim.x) {
      double v;
      if (!series_value(a, r, s, i, v)) continue;
      const unsigned long long k = okey(v);
      const unsigned d = (unsigned)(k >> shift) & 255u;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (pass == 0 || (k >> (shift + 8)) == (prefix[j] >> (shift + 8))) atomicAdd(&hist[j][d], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      const int j = threadIdx.x;
      long long k = rank[j], cum = 0;
      int d = 0;
      for (; d < 255; ++d) {
        if (cum + hist[j][d] >= k) break;
        cum += hist[j][d];
      }
      rank[j] = k - cum;
      prefix[j] |= (unsigned long long)d << shift;
    }
    __syncthreads();
  }
  if (threadIdx.x < 3) out[threadIdx.x] = okey_inv(prefix[threadIdx.x]);
}

__global__ void series_kernel(const StraitMetricsArgs a) {
  const int64_t r = blockIdx.x;
  const int64_t lo = a.req_off[r];
  const int64_t nb = a.counters[r * STRAIT_RC_N + STRAIT_RC_COMPLETED];
  for (int64_t b = lo + threadIdx.x; b < lo + nb; b += blockDim.x) {
    const double act = a.fb_actual[b];
    if (a.intf_error) a.intf_error[b] = __ddiv_rn(a.fb_predicted[b] - act, act);
    const double lat = a.b_completion[b] - a.b_front[b];
    if (a.latency_error) a.latency_error[b] = __ddiv_rn(a.dec_est_latency[b] - lat, lat);
    const double iso = a.kernel_table[(int64_t)a.dec_model[b] * a.table_stride + a.dec_size[b] - 1];
    if (a.kernel_overhead) a.kernel_overhead[b] = __ddiv_rn(fabs((a.b_kernel_end[b] - a.b_kernel_start[b]) - iso), iso);
  }
}

}  // namespace

extern "C" int strait_replay_metrics(const StraitMetricsArgs* a, void* stream) {
  using namespace strait;
  if (!a || a->n_replays < 0 || a->max_windows < 1 || a->table_stride < 1)
    return set_error(STRAIT_EINVAL, "strait_replay_metrics: bad arguments");
  if (!a->n_replays) return STRAIT_OK;
  const void* need[] = {a->window_ms, a->req_off, a->arr_time, a->arr_model, a->model_prio, a->req_status,
                        a->req_violated, a->req_completion, a->counters, a->dec_model, a->dec_size,
                        a->dec_est_latency, a->b_front, a->b_kernel_start, a->b_kernel_end, a->b_completion,
                        a->fb_predicted, a->fb_actual, a->kernel_table, a->class_counts, a->partial, a->pct,
                        a->series_count, a->goodput, a->goodput_len};
  for (const void* p : need)
    if (!p) return set_error(STRAIT_EINVAL, "strait_replay_metrics: null buffer");
  cudaStream_t st = (cudaStream_t)stream;
  counts_kernel<<<a->n_replays, kThreads, 0, st>>>(*a);
  if (int rc = check_launch("strait_replay_metrics/counts")) return rc;
  select_kernel<<<dim3(a->n_replays, STRAIT_MS_N), kThreads, 0, st>>>(*a);
  if (int rc = check_launch("strait_replay_metrics/select")) return rc;
  if (a->intf_error || a->latency_error || a->kernel_overhead) {
    series_kernel<<<a->n_replays, kThreads, 0, st>>>(*a);
    if (int rc = check_launch("strait_replay_metrics/series")) return rc;
  }
  return STRAIT_OK;
}
