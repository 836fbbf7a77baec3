// strait_expand.cu — rebuild the profile-derived fields of a sweep snapshot
// from profile-row indices (include/strait.h, strait_sweep_expand).  The
// aggregates are the reference's list-order sums from 0.0 over the running
// prefix of the slots (runtime.py:104-122), so the expanded SoA is
// bit-identical to one exported field by field.
#include <cuda_runtime.h>

#include "../../include/strait.h"
#include "strait_capi.cuh"

namespace {

template <int NM>
__global__ void expand_kernel(const StraitSweepExpandArgs e, const StraitSweepArgs a) {
  const int64_t S = a.n_segments, P = S * a.gpus_per_segment, C = a.n_slots, T = P * C;
  const int64_t R = e.n_rows;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double* ec = const_cast<double*>(a.ent_contrib);
  for (int64_t t = i0; t < T; t += stride) {  // co-runner rows
    const int row = e.ent_row[t];
#pragma unroll
    for (int m = 0; m < NM; ++m) ec[m * T + t] = __ldg(&e.thr[m * R + row]);
    const_cast<double*>(a.ent_self_cmp)[t] = __ldg(&e.self_cmp[row]);
    const_cast<double*>(a.ent_self_mem)[t] = __ldg(&e.self_mem[row]);
    const_cast<double*>(a.ent_t_kernel)[t] = __ldg(&e.kernel[row]);
    const_cast<int8_t*>(a.ent_prio)[t] = __ldg(&e.prio[row / e.table_stride]);
  }
  for (int64_t p = i0; p < P; p += stride) {  // aggregates over the running prefix, list order from 0.0
    const int n = a.gpu_n_running[p];
    double agg[NM], lp[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) agg[m] = lp[m] = 0.0;
    for (int c = 0; c < n && c < C; ++c) {
      const int row = e.ent_row[p * C + c];
      const bool low = __ldg(&e.prio[row / e.table_stride]) == 1;
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        const double v = __ldg(&e.thr[m * R + row]);
        agg[m] += v;
        if (low) lp[m] += v;
      }
    }
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const_cast<double*>(a.gpu_agg)[m * P + p] = agg[m];
      const_cast<double*>(a.gpu_lp_agg)[m * P + p] = lp[m];
    }
  }
  for (int64_t s = i0; s < S; s += stride) {  // candidate rows
    const int row = e.cand_row[s];
    const int model = row / e.table_stride;
#pragma unroll
    for (int m = 0; m < NM; ++m) const_cast<double*>(a.cand_contrib)[m * S + s] = __ldg(&e.thr[m * R + row]);
    const_cast<double*>(a.cand_self_cmp)[s] = __ldg(&e.self_cmp[row]);
    const_cast<double*>(a.cand_self_mem)[s] = __ldg(&e.self_mem[row]);
    const_cast<double*>(a.cand_total)[s] = __ldg(&e.total[row]);
    const_cast<double*>(a.cand_kernel)[s] = __ldg(&e.kernel[row]);
    const_cast<double*>(a.cand_deadline)[s] = __ldg(&e.deadline[model]);
    const_cast<int8_t*>(a.cand_prio)[s] = __ldg(&e.prio[model]);
  }
}

}  // namespace

extern "C" int strait_sweep_expand(const StraitSweepExpandArgs* e, const StraitSweepArgs* a, void* stream) {
  if (!e || !a || a->n_metrics < 1 || a->n_metrics > STRAIT_MAX_METRICS || e->table_stride < 1 || e->n_rows < 1 ||
      !e->thr || !e->self_cmp || !e->self_mem || !e->kernel || !e->total || !e->deadline || !e->prio ||
      !e->ent_row || !e->cand_row)
    return strait::set_error(STRAIT_EINVAL, "strait_sweep_expand: bad arguments");
  const unsigned grid = 148 * 8;
  cudaStream_t st = (cudaStream_t)stream;
  switch (a->n_metrics) {
    case 1: expand_kernel<1><<<grid, 256, 0, st>>>(*e, *a); break;
    case 2: expand_kernel<2><<<grid, 256, 0, st>>>(*e, *a); break;
    case 3: expand_kernel<3><<<grid, 256, 0, st>>>(*e, *a); break;
    case 4: expand_kernel<4><<<grid, 256, 0, st>>>(*e, *a); break;
    case 5: expand_kernel<5><<<grid, 256, 0, st>>>(*e, *a); break;
    case 6: expand_kernel<6><<<grid, 256, 0, st>>>(*e, *a); break;
    case 7: expand_kernel<7><<<grid, 256, 0, st>>>(*e, *a); break;
    default: expand_kernel<8><<<grid, 256, 0, st>>>(*e, *a); break;
  }
  return strait::check_launch("strait_sweep_expand");
}
