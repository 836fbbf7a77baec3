// strait_node.cuh — the object-API runtime record (include/strait_node.h):
// accessors and the bookkeeping steps, written once as __host__ __device__
// code over the flat record.  Each step restates one reference method in its
// exact floating-point order (file:line under /root/reference/pkg/src/infersim).
#pragma once

#include <stdint.h>

#include "../../include/strait_node.h"

namespace strait {
namespace node {

__host__ __device__ __forceinline__ StraitGpuHdr* hdr(void* r) { return (StraitGpuHdr*)r; }
__host__ __device__ __forceinline__ const StraitGpuHdr* hdr(const void* r) { return (const StraitGpuHdr*)r; }
__host__ __device__ __forceinline__ StraitNodeEntry* entries(void* r) {
  return (StraitNodeEntry*)((char*)r + sizeof(StraitGpuHdr));
}
__host__ __device__ __forceinline__ const StraitNodeEntry* entries(const void* r) {
  return (const StraitNodeEntry*)((const char*)r + sizeof(StraitGpuHdr));
}
__host__ __device__ __forceinline__ double* ring(void* r) {
  return (double*)((char*)r + sizeof(StraitGpuHdr) + sizeof(StraitNodeEntry) * (size_t)hdr(r)->slot_cap);
}
__host__ __device__ __forceinline__ int64_t record_bytes(int slot_cap, int ring_cap) {
  return (int64_t)sizeof(StraitGpuHdr) + (int64_t)sizeof(StraitNodeEntry) * slot_cap + 8LL * ring_cap;
}

// CPython max(a, b) / min(a, b) on floats: the first argument wins unless the
// second compares greater (smaller).
__host__ __device__ __forceinline__ double fmax_py(double a, double b) { return b > a ? b : a; }
__host__ __device__ __forceinline__ double fmin_py(double a, double b) { return b < a ? b : a; }

// ---------------------------------------------------------------- timeline
// ThroughputTimeline.record (domain.py:237-248) in running-integral form: the
// closed segment's v * d is added when it closes, in the reference loop's
// order, so the TWA below repeats its sums exactly.
__host__ __device__ inline int tl_record(StraitNodeEntry& e, int nm, double now, const double* v) {
  if (e.tl_n == 0) {
    for (int m = 0; m < nm; ++m) {
      e.tl_acc[m] = 0.0;
      e.tl_v[m] = v[m];
    }
    e.tl_t0 = e.tl_tlast = now;
    e.tl_n = 1;
    return STRAIT_OK;
  }
  if (now < e.tl_tlast) return STRAIT_EORDER;
  if (now == e.tl_tlast) {  // collapse onto the later value
    for (int m = 0; m < nm; ++m) e.tl_v[m] = v[m];
    return STRAIT_OK;
  }
  const double d = now - e.tl_tlast;
  for (int m = 0; m < nm; ++m) {
    e.tl_acc[m] = e.tl_acc[m] + e.tl_v[m] * d;
    e.tl_v[m] = v[m];
  }
  e.tl_tlast = now;
  e.tl_n += 1;
  return STRAIT_OK;
}

// time_weighted_average (domain.py:250-264): 1 = no samples, 2 = end before the
// last sample (both ValueError in the reference), else 0.
__host__ __device__ inline int tl_twa(const StraitNodeEntry& e, int nm, double end, double* out) {
  if (e.tl_n == 0) return 1;
  if (end < e.tl_tlast) return 2;
  const double total = end - e.tl_t0;
  if (total <= 0.0) {
    for (int m = 0; m < nm; ++m) out[m] = e.tl_v[m];
    return 0;
  }
  const double d = end - e.tl_tlast;
  for (int m = 0; m < nm; ++m) out[m] = (e.tl_acc[m] + e.tl_v[m] * d) / total;
  return 0;
}

// ---------------------------------------------------------------- aggregates
// _recompute_aggregate (runtime.py:104-109): per metric, a sum from 0.0 in list order.
__host__ __device__ inline void recompute(void* r) {
  StraitGpuHdr* h = hdr(r);
  const StraitNodeEntry* e = entries(r);
  for (int m = 0; m < h->n_metrics; ++m) {
    double s = 0.0;
    for (int i = 0; i < h->n_running; ++i) s += e[i].contrib[m];
    h->agg[m] = s;
  }
}

// low_priority_aggregate (runtime.py:115-122)
__host__ __device__ inline void lp_aggregate(const void* r, double* out) {
  const StraitGpuHdr* h = hdr(r);
  const StraitNodeEntry* e = entries(r);
  for (int m = 0; m < h->n_metrics; ++m) {
    double s = 0.0;
    for (int i = 0; i < h->n_running; ++i)
      if (e[i].prio == 1) s += e[i].contrib[m];
    out[m] = s;
  }
}

// every running entry records aggregate_excluding(entry) at `now` (runtime.py:129-130,140-141)
__host__ __device__ inline int restamp(void* r, double now) {
  StraitGpuHdr* h = hdr(r);
  StraitNodeEntry* e = entries(r);
  double ex[STRAIT_MAX_METRICS];
  for (int i = 0; i < h->n_running; ++i) {
    for (int m = 0; m < h->n_metrics; ++m) ex[m] = h->agg[m] - e[i].contrib[m];
    const int st = tl_record(e[i], h->n_metrics, now, ex);
    if (st != STRAIT_OK) return st;
  }
  return STRAIT_OK;
}

}  // namespace node
}  // namespace strait
