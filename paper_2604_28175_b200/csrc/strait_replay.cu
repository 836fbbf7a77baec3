// strait_replay.cu — C-ABI of the device trace-replay engine
// (include/strait_replay.h): argument validation, launch geometry, dispatch
// on the metric count.  The engine is strait_replay_impl.cuh; one
// instantiation per metric count lives in strait_replay_nm<k>.cu so they
// compile in parallel.
#include <cuda_runtime.h>

#include <cstdlib>

#include "strait_capi.cuh"
#include "strait_replay_impl.cuh"

namespace {

constexpr size_t kSmemBudget = 200 * 1024;  // per CTA, of the 227 KB opt-in maximum
constexpr int kMaxWarpsPerCta = 4;

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

}  // namespace

namespace strait {
namespace rp {
bool replay_cta_enabled(bool wide) {
  const char* e = getenv("STRAIT_REPLAY_NW");
  if (e && atoi(e) == 1) return false;
  if (e && atoi(e) > 1) return true;
  return wide;
}
int replay_occupancy(int64_t n_replays, int wpc) {
  if (const char* e = getenv("STRAIT_REPLAY_OCC")) return atoi(e) >= 4 ? 4 : 1;
  return n_replays > (int64_t)sm_count() * 2 * wpc ? 4 : 1;
}
}  // namespace rp
}  // namespace strait

extern "C" int64_t strait_replay_smem_bytes(int32_t n_gpus, int32_t concurrency_limit, int32_t n_models,
                                            int32_t n_metrics) {
  using namespace strait::rp;
  if (n_gpus < 1 || concurrency_limit < 1 || concurrency_limit > kMaxConc || n_models < 1 ||
      n_models > kMaxModels || n_metrics < 1 || n_metrics > STRAIT_MAX_METRICS)
    return 0;
  const Layout L(n_gpus, concurrency_limit, n_models, n_metrics);
  return L.bytes <= kSmemBudget ? (int64_t)L.bytes : 0;
}

extern "C" int strait_replay(const StraitReplayArgs* a, void* stream) {
  using namespace strait;
  using namespace strait::rp;
  if (!a) return set_error(STRAIT_EINVAL, "strait_replay: null args");
  if (a->n_replays < 0) return set_error(STRAIT_EINVAL, "strait_replay: n_replays < 0");
  if (a->n_replays == 0) return STRAIT_OK;
  const StraitReplayModels& md = a->models;
  if (md.n_metrics < 1 || md.n_metrics > STRAIT_MAX_METRICS)
    return set_error(STRAIT_EINVAL, "strait_replay: n_metrics %d outside 1..%d", md.n_metrics, STRAIT_MAX_METRICS);
  if (md.n_models < 1 || md.n_models > kMaxModels)
    return set_error(STRAIT_EINVAL, "strait_replay: n_models %d outside 1..%d", md.n_models, kMaxModels);
  if (md.stride < 1 || md.stride > kMaxBatch)
    return set_error(STRAIT_EINVAL, "strait_replay: table stride %d outside 1..%d", md.stride, kMaxBatch);
  if (a->max_concurrency < 1 || a->max_concurrency > kMaxConc)
    return set_error(STRAIT_EINVAL, "strait_replay: concurrency_limit %d outside 1..%d", a->max_concurrency,
                     kMaxConc);
  if (a->max_gpus < 1) return set_error(STRAIT_EINVAL, "strait_replay: max_gpus < 1");
  int64_t per_warp = strait_replay_smem_bytes(a->max_gpus, a->max_concurrency, md.n_models, md.n_metrics);
  // a geometry past the one-warp budget still runs as one replay per CTA (up to the 227 KB opt-in maximum)
  const bool cta_only = !per_warp && a->n_replays <= (int64_t)sm_count() && cta_replay_smem(*a);
  if (!per_warp && !cta_only)
    return set_error(STRAIT_EINVAL, "strait_replay: %d GPUs x %d slots x %d models needs more than %zu B on chip",
                     a->max_gpus, a->max_concurrency, md.n_models, kSmemBudget);
  if (cta_only) per_warp = (int64_t)cta_replay_smem(*a);
  const void* need[] = {a->cfg, a->req_off, a->arr_time, a->arr_model, a->model_req, a->mr_off, a->noise,
                        a->bc1, a->bc2, a->pred_state, a->pred_step, a->req_status, a->req_violated,
                        a->req_completion, a->req_batch, a->dec_time, a->dec_pass, a->dec_model, a->dec_size,
                        a->dec_gpu, a->dec_est_latency, a->dec_intf, a->b_front, a->b_transfer_start,
                        a->b_transfer_end, a->b_kernel_start, a->b_kernel_end, a->b_completion, a->b_work,
                        a->b_done_order, a->fb_predicted, a->fb_actual, a->fb_residual, a->fb_flags,
                        a->counters, md.max_batch, md.prio, md.deadline, md.timeout, md.total, md.transfer,
                        md.kernel, md.self_cmp, md.self_mem, md.throughput};
  for (const void* p : need)
    if (!p) return set_error(STRAIT_EINVAL, "strait_replay: null buffer");
  if (a->cap_rows_max > 0 && (!a->cap_time || !a->cap_gpu || !a->cap_pct))
    return set_error(STRAIT_EINVAL, "strait_replay: null cap-row buffer");
  if (a->trace && a->trace_max < 0) return set_error(STRAIT_EINVAL, "strait_replay: trace_max < 0");
  // warps per CTA: enough CTAs to cover the SMs first, then pack up to the smem budget
  int wpc = (int)(kSmemBudget / per_warp);
  if (wpc > kMaxWarpsPerCta) wpc = kMaxWarpsPerCta;
  const int64_t want = (a->n_replays + sm_count() - 1) / sm_count();
  if (want < wpc) wpc = (int)(want < 1 ? 1 : want);
  // variant: the latency kernel while every replay is resident (2 CTAs x 4 warps per
  // SM), then one warp per CTA so the hardware spreads the (heaviest-first ordered)
  // replays over SMs and sub-partitions; past that, the 16-replays-per-SM kernel
  // a traced launch (event log) always runs the latency variant with the log compiled in
  int minb = a->trace ? 0 : replay_occupancy(a->n_replays, wpc);
  if (minb < 4 || cta_only) wpc = 1;
  if (cta_only) minb = a->trace ? 3 : 2;
  // at most one replay per SM and more running-batch slots than a warp has lanes (C5's 64 GPUs):
  // a CTA of kCtaWarps warps per replay (STRAIT_REPLAY_NW=8 forces it, =1 disables it)
  if (minb == 1 && a->n_replays <= (int64_t)sm_count() && cta_replay_smem(*a) &&
      replay_cta_enabled((int64_t)a->max_gpus * a->max_concurrency > 32))
    minb = 2;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = STRAIT_EINVAL;
  switch (md.n_metrics) {
    case 1: rc = launch_replay<1>(*a, st, wpc, per_warp, minb); break;
    case 2: rc = launch_replay<2>(*a, st, wpc, per_warp, minb); break;
    case 3: rc = launch_replay<3>(*a, st, wpc, per_warp, minb); break;
    case 4: rc = launch_replay<4>(*a, st, wpc, per_warp, minb); break;
    case 5: rc = launch_replay<5>(*a, st, wpc, per_warp, minb); break;
    case 6: rc = launch_replay<6>(*a, st, wpc, per_warp, minb); break;
    case 7: rc = launch_replay<7>(*a, st, wpc, per_warp, minb); break;
    case 8: rc = launch_replay<8>(*a, st, wpc, per_warp, minb); break;
  }
  return rc;
}

#if STRAIT_REPLAY_PROFILE
namespace strait {
namespace rp {
__device__ unsigned long long g_replay_prof[RPF_N];
__device__ unsigned long long g_cta_warp[3][16];
}  // namespace rp
}  // namespace strait
/* diagnostic build only: per-warp CTA propose-job timestamps (wake, phase-A end, phase-B end) summed */
extern "C" int strait_replay_cta_profile(unsigned long long* out) {
  using namespace strait::rp;
  unsigned long long zero[48] = {};
  if (cudaMemcpyFromSymbol(out, g_cta_warp, sizeof zero) != cudaSuccess ||
      cudaMemcpyToSymbol(g_cta_warp, zero, sizeof zero) != cudaSuccess)
    return strait::set_error(STRAIT_ECUDA, "strait_replay_cta_profile: copy failed");
  return 48;
}
/* diagnostic build only: accumulated engine cycles per phase since the last call (then reset) */
extern "C" int strait_replay_profile(unsigned long long* out) {
  using namespace strait::rp;
  unsigned long long zero[RPF_N] = {};
  if (cudaMemcpyFromSymbol(out, g_replay_prof, sizeof zero) != cudaSuccess ||
      cudaMemcpyToSymbol(g_replay_prof, zero, sizeof zero) != cudaSuccess)
    return strait::set_error(STRAIT_ECUDA, "strait_replay_profile: copy failed");
  return RPF_N;
}
#endif
