// strait_workload.cu — on-device generation of the reference's arrival and
// noise streams (include/strait_replay.h, "On-device workload generation"):
// one thread per numpy Generator stream (a stream is inherently sequential:
// the ziggurat consumes a data-dependent number of draws), then an
// event-order merge with one thread per arrival (binary search in every
// other model's sorted segment).
#include <cuda_runtime.h>
#include <math.h>

#include "../../include/strait_replay.h"
#include "strait_capi.cuh"
#include "strait_rng.cuh"

namespace {

using strait::rng::Pcg64;

// gen_poisson / gen_uniform / noise of one stream; writes when out != nullptr
__device__ int64_t run_stream(const StraitStreamSpec& sp, double* out) {
  if (sp.mode == STRAIT_STREAM_NOISE) {
    Pcg64 r;
    r.seed(sp.entropy, sp.n_entropy);
    if (out)
      for (int64_t i = 0; i < sp.n_draws; ++i) out[i] = strait::glibc::exp(0.0 + sp.sigma * strait::rng::std_normal(r));
    return sp.n_draws;
  }
  if (sp.mode == STRAIT_STREAM_UNIFORM) {  // workload.py:38-50
    if (sp.rate_per_s <= 0) return 0;
    const double gap = __ddiv_rn(1000.0, sp.rate_per_s);
    const int64_t count = (int64_t)ceil(__ddiv_rn(sp.span_ms, gap));
    int64_t n = 0;
    for (int64_t k = 0; k <= count; ++k) {
      const double t = (double)k * gap;
      if (t < sp.span_ms) {
        if (out) out[n] = sp.offset_ms + t;
        ++n;
      }
    }
    return n;
  }
  // gen_poisson (workload.py:19-35)
  if (sp.rate_per_s == 0 || sp.span_ms <= 0) return 0;
  Pcg64 r;
  r.seed(sp.entropy, sp.n_entropy);
  const double mean_gap = __ddiv_rn(1000.0, sp.rate_per_s);
  double t = 0.0;
  int64_t n = 0;
  for (;;) {
    t += mean_gap * strait::rng::std_exponential(r);
    if (t >= sp.span_ms) return n;
    if (out) out[n] = sp.offset_ms == 0.0 ? t : sp.offset_ms + t;  // load_trace: start + t
    ++n;
  }
}

__global__ void count_kernel(const StraitStreamSpec* specs, int64_t n, int64_t* counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    counts[i] = run_stream(specs[i], nullptr);
}

__global__ void fill_kernel(const StraitStreamSpec* specs, int64_t n, const int64_t* offsets, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    run_stream(specs[i], out + offsets[i]);
}

// first index in [lo, hi) with a[i] > t (upper) or a[i] >= t (lower)
__device__ __forceinline__ int64_t bound(const double* a, int64_t lo, int64_t hi, double t, bool upper) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const double v = a[mid];
    if (upper ? !(t < v) : (v < t)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void order_kernel(int32_t R, int32_t M, const int64_t* mr_off, const double* mm, double* arr_time,
                             int16_t* arr_model, int32_t* model_req) {
  const int64_t N = mr_off[(int64_t)R * M];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
    // segment (r, m) holding e: upper_bound over the R*M+1 offsets, minus one
    int64_t lo = 0, hi = (int64_t)R * M;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (mr_off[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    int64_t seg = lo;
    while (seg + 1 <= (int64_t)R * M && mr_off[seg + 1] <= e) ++seg;  // skip empty segments
    const int64_t r = seg / M;
    const int m = (int)(seg - r * M);
    const double t = mm[e];
    int64_t pos = e - mr_off[seg];
    for (int mm2 = 0; mm2 < M; ++mm2) {
      if (mm2 == m) continue;
      const int64_t a = mr_off[r * M + mm2], b = mr_off[r * M + mm2 + 1];
      pos += bound(mm, a, b, t, mm2 < m) - a;  // earlier models win ties (push order)
    }
    const int64_t g = mr_off[r * M] + pos;
    arr_time[g] = t;
    arr_model[g] = (int16_t)m;
    model_req[e] = (int32_t)g;
  }
}

__global__ void draws_kernel(const uint64_t* entropy, int32_t n_entropy, int32_t kind, double loc, double scale,
                             int64_t n, double* out) {
  if (threadIdx.x || blockIdx.x) return;
  uint64_t ent[3];
  for (int i = 0; i < n_entropy; ++i) ent[i] = entropy[i];
  Pcg64 r;
  r.seed(ent, n_entropy);
  for (int64_t i = 0; i < n; ++i) {
    if (kind == 0) out[i] = scale * strait::rng::std_exponential(r);
    else if (kind == 1) out[i] = loc + scale * strait::rng::std_normal(r);
    else out[i] = __longlong_as_double((long long)r.next64());
  }
}

unsigned grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < 1 ? 1 : (b > 65535 ? 65535 : b));
}

}  // namespace

extern "C" int strait_stream_count(const StraitStreamSpec* specs, int64_t n, int64_t* counts, void* stream) {
  if (n < 0 || (n && (!specs || !counts))) return strait::set_error(STRAIT_EINVAL, "strait_stream_count: bad args");
  if (!n) return STRAIT_OK;
  count_kernel<<<grid_for(n, 64), 64, 0, (cudaStream_t)stream>>>(specs, n, counts);
  return strait::check_launch("strait_stream_count");
}

extern "C" int strait_stream_fill(const StraitStreamSpec* specs, int64_t n, const int64_t* offsets, double* out,
                                  void* stream) {
  if (n < 0 || (n && (!specs || !offsets || !out)))
    return strait::set_error(STRAIT_EINVAL, "strait_stream_fill: bad args");
  if (!n) return STRAIT_OK;
  fill_kernel<<<grid_for(n, 64), 64, 0, (cudaStream_t)stream>>>(specs, n, offsets, out);
  return strait::check_launch("strait_stream_fill");
}

extern "C" int strait_arrival_order(int32_t R, int32_t M, const int64_t* mr_off, const double* mm, double* arr_time,
                                    int16_t* arr_model, int32_t* model_req, void* stream) {
  if (R < 0 || M < 1 || !mr_off || !mm || !arr_time || !arr_model || !model_req)
    return strait::set_error(STRAIT_EINVAL, "strait_arrival_order: bad args");
  if (!R) return STRAIT_OK;
  order_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(R, M, mr_off, mm, arr_time, arr_model, model_req);
  return strait::check_launch("strait_arrival_order");
}

extern "C" int strait_rng_draws(const uint64_t* entropy, int32_t n_entropy, int32_t kind, double loc, double scale,
                                int64_t n, double* out, void* stream) {
  if (!entropy || n_entropy < 1 || n_entropy > 3 || kind < 0 || kind > 2 || n < 0 || (n && !out))
    return strait::set_error(STRAIT_EINVAL, "strait_rng_draws: bad args");
  if (!n) return STRAIT_OK;
  draws_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(entropy, n_entropy, kind, loc, scale, n, out);
  return strait::check_launch("strait_rng_draws");
}
