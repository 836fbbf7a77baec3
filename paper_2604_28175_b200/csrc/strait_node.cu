// strait_node.cu — the object-API runtime (include/strait_node.h).
//
// Host entry points: O(concurrency) bookkeeping on the caller-owned records
// (link FIFO, AIMD cap, running list with list-order aggregates, timelines).
// Device entry point: strait_node_propose, PredictivePolicy.propose
// (scheduler.py:257-285) over the records of a node in one launch.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstring>

#include "strait_capi.cuh"
#include "strait_device.cuh"
#include "strait_node.cuh"

using namespace strait;
using namespace strait::node;

// ============================================================================ host entries

extern "C" int64_t strait_node_record_bytes(int32_t slot_cap, int32_t ring_cap) {
  return record_bytes(slot_cap, ring_cap);
}

extern "C" void* strait_node_device_address(void* host_ptr) {
  void* d = nullptr;
  const cudaError_t e = cudaHostGetDevicePointer(&d, host_ptr, 0);
  if (e != cudaSuccess) {
    set_error(STRAIT_ECUDA, "record is not device-mapped page-locked memory: %s", cudaGetErrorString(e));
    return nullptr;
  }
  return d;
}

extern "C" double strait_link_delay(const void* rec, double now) {
  return fmax_py(0.0, hdr(rec)->t_available - now);  // pcie.py:21-23
}

extern "C" int strait_link_reserve(void* rec, double now, double duration, double* out_start, double* out_end) {
  StraitGpuHdr* h = hdr(rec);
  if (duration <= 0) return set_error(STRAIT_EINVAL, "transfer duration must be positive, got %.17g", duration);
  if (h->ring_len == h->ring_cap) return set_error(STRAIT_ENOSPC, "pending-transfer ring full");
  const double start = fmax_py(now, h->t_available);  // pcie.py:30-34
  const double end = start + duration;
  h->t_available = end;
  int tail = h->ring_head + h->ring_len;
  if (tail >= h->ring_cap) tail -= h->ring_cap;
  ring(rec)[tail] = end;
  h->ring_len += 1;
  if (out_start) *out_start = start;
  if (out_end) *out_end = end;
  return STRAIT_OK;
}

extern "C" int strait_link_calibrate(void* rec, double actual_end) {
  StraitGpuHdr* h = hdr(rec);
  if (h->ring_len == 0) return set_error(STRAIT_EINVAL, "no outstanding transfer to calibrate");
  double* q = ring(rec);
  const double predicted = q[h->ring_head];
  h->ring_head = h->ring_head + 1 == h->ring_cap ? 0 : h->ring_head + 1;
  h->ring_len -= 1;
  if (h->ring_len == 0) {  // nothing reserved after it: replace the estimate (pcie.py:45-47)
    h->t_available = actual_end;
    return STRAIT_OK;
  }
  const double offset = actual_end - predicted;
  if (offset == 0.0) return STRAIT_OK;
  h->t_available += offset;  // shift the estimate and every later predicted end (pcie.py:48-53)
  for (int i = 0, j = h->ring_head; i < h->ring_len; ++i, j = (j + 1 == h->ring_cap ? 0 : j + 1))
    q[j] = q[j] + offset;
  return STRAIT_OK;
}

extern "C" int strait_aimd_advance(void* rec, double now) {
  StraitGpuHdr* h = hdr(rec);
  if (now < h->aimd_last_tick)
    return set_error(STRAIT_EINVAL, "aimd tick moving backwards: %.17g < %.17g", now, h->aimd_last_tick);
  const double whole = std::floor((now - h->aimd_last_tick) / h->aimd_interval);  // runtime.py:30-35
  if (!(whole > 0)) return STRAIT_OK;
  h->cap_pct = fmin_py(h->aimd_ceiling, h->cap_pct + whole * h->aimd_increase);
  h->aimd_last_tick += whole * h->aimd_interval;
  return STRAIT_OK;
}

extern "C" void strait_aimd_reset(void* rec) { hdr(rec)->cap_pct = hdr(rec)->aimd_floor; }

extern "C" int strait_nodes_tick(void* const* recs, int32_t n, double now) {
  for (int i = 0; i < n; ++i) {
    const int st = strait_aimd_advance(recs[i], now);
    if (st != STRAIT_OK) return st;
  }
  return STRAIT_OK;
}

static inline int check_pos(const void* rec, int32_t pos) {
  if (pos < 0 || pos >= hdr(rec)->n_running) return set_error(STRAIT_EINVAL, "no running entry at %d", pos);
  return STRAIT_OK;
}

extern "C" int strait_entry_tl_record(StraitNodeEntry* e, int32_t nm, double now, const double* value) {
  const double last = e->tl_tlast;
  const int st = tl_record(*e, nm, now, value);
  if (st == STRAIT_EORDER)
    return set_error(st, "timeline sample at %.17g precedes last sample at %.17g", now, last);
  return st;
}

static int twa_status(int st, const StraitNodeEntry& e, double end) {
  if (st == 1) return set_error(STRAIT_EINVAL, "no samples");
  if (st == 2) return set_error(STRAIT_EINVAL, "end_time %.17g precedes last sample at %.17g", end, e.tl_tlast);
  return STRAIT_OK;
}

extern "C" int strait_entry_tl_twa(const StraitNodeEntry* e, int32_t nm, double end, double* out) {
  return twa_status(tl_twa(*e, nm, end, out), *e, end);
}

extern "C" int strait_node_excluding(const void* rec, int32_t pos, double* out) {
  if (check_pos(rec, pos)) return STRAIT_EINVAL;
  const StraitGpuHdr* h = hdr(rec);
  const StraitNodeEntry& e = entries(rec)[pos];
  for (int m = 0; m < h->n_metrics; ++m) out[m] = h->agg[m] - e.contrib[m];  // runtime.py:111-113
  return STRAIT_OK;
}

extern "C" void strait_node_lp_aggregate(const void* rec, double* out) { lp_aggregate(rec, out); }

extern "C" int32_t strait_node_find(const void* rec, int32_t handle) {
  const StraitGpuHdr* h = hdr(rec);
  const StraitNodeEntry* e = entries(rec);
  for (int i = 0; i < h->n_running; ++i)
    if (e[i].handle == handle) return i;
  return -1;
}

static int restamp_status(void* rec, double now) {
  const int st = restamp(rec, now);
  if (st == STRAIT_EORDER) return set_error(st, "timeline sample at %.17g precedes a running entry's last sample", now);
  return st;
}

extern "C" int strait_node_detach(void* rec, int32_t handle, StraitNodeEntry* out_removed) {
  StraitGpuHdr* h = hdr(rec);
  const int pos = strait_node_find(rec, handle);
  if (pos < 0) return set_error(STRAIT_ERUNTIME, "gpu %d: batch is not running here", h->gpu_id);
  StraitNodeEntry* e = entries(rec);
  if (out_removed) *out_removed = e[pos];
  for (int i = pos; i + 1 < h->n_running; ++i) e[i] = e[i + 1];
  h->n_running -= 1;
  return STRAIT_OK;
}

extern "C" int strait_node_attach(void* rec, const StraitNodeEntry* entry) {
  StraitGpuHdr* h = hdr(rec);
  if (h->n_running >= h->slot_cap) return set_error(STRAIT_ENOSPC, "entry slots full");
  entries(rec)[h->n_running] = *entry;
  h->n_running += 1;
  return STRAIT_OK;
}

extern "C" int strait_node_add(void* rec, const StraitNodeEntry* entry, double now) {
  StraitGpuHdr* h = hdr(rec);
  if (h->n_running >= h->concurrency_limit)  // runtime.py:125-126
    return set_error(STRAIT_ERUNTIME, "gpu %d: concurrency limit exceeded", h->gpu_id);
  if (h->n_running >= h->slot_cap) return set_error(STRAIT_ENOSPC, "entry slots full");
  entries(rec)[h->n_running] = *entry;
  h->n_running += 1;
  recompute(rec);
  return restamp_status(rec, now);
}

extern "C" int strait_node_remove(void* rec, int32_t handle, double now, StraitNodeEntry* out_removed) {
  const int st = strait_node_detach(rec, handle, out_removed);  // list order of the survivors kept
  if (st != STRAIT_OK) return st;
  recompute(rec);
  return restamp_status(rec, now);
}

extern "C" int strait_node_submit(void* rec, StraitNodeEntry* entry, double transfer_ms, double now,
                                  double* out_start, double* out_end) {
  StraitGpuHdr* h = hdr(rec);
  // capacity first (the caller grows the record and retries: not observable); then, as
  // submit_plan, reserve the link and add the entry — a full GPU raises after the reservation
  if (h->n_running >= h->slot_cap && h->n_running < h->concurrency_limit)
    return set_error(STRAIT_ENOSPC, "entry slots full");
  double start, end;
  const int st = strait_link_reserve(rec, now, transfer_ms, &start, &end);
  if (st != STRAIT_OK) return st;
  entry->kstart_est = end;  // scheduler.py:321 kernel_start_estimate = transfer end
  if (out_start) *out_start = start;
  if (out_end) *out_end = end;
  return strait_node_add(rec, entry, now);
}

extern "C" int strait_node_start(void* rec, int32_t handle, double now) {
  const int pos = strait_node_find(rec, handle);
  if (pos < 0) return set_error(STRAIT_ERUNTIME, "gpu %d: batch is not running here", hdr(rec)->gpu_id);
  int st = strait_link_calibrate(rec, now);  // simulation.py:382: measured end == now in simulation
  if (st != STRAIT_OK) return st;
  StraitNodeEntry& e = entries(rec)[pos];
  e.kernel_start = now;
  e.started = 1;
  double ex[STRAIT_MAX_METRICS];
  strait_node_excluding(rec, pos, ex);
  e.tl_n = 0;  // a fresh timeline [(now, aggregate_excluding(entry))] (simulation.py:387)
  tl_record(e, hdr(rec)->n_metrics, now, ex);
  return STRAIT_OK;
}

extern "C" int strait_node_complete(void* rec, int32_t handle, double now, double* out_twa,
                                    StraitNodeEntry* out_removed) {
  const int pos = strait_node_find(rec, handle);
  if (pos < 0) return set_error(STRAIT_ERUNTIME, "gpu %d: batch is not running here", hdr(rec)->gpu_id);
  const StraitNodeEntry& e = entries(rec)[pos];
  const int st = twa_status(tl_twa(e, hdr(rec)->n_metrics, now, out_twa), e, now);  // scheduler.py:335
  if (st != STRAIT_OK) return st;
  return strait_node_remove(rec, handle, now, out_removed);
}

// ============================================================================ device propose

namespace {

constexpr int kProposeThreads = 256;

__device__ __forceinline__ double nan_d() { return __longlong_as_double(0x7ff8000000000000LL); }

// Dynamic shared memory of one propose: per-(size, GPU) results, per-size
// argmin, then (optionally) the staged records.
struct ProposeLayout {
  size_t lat, intf, seg_lat, seg_intf, seg_gpu, flags, recs, bytes;
  __host__ __device__ ProposeLayout(int K, int G, int stage_stride) {
    const size_t KG = (size_t)K * G;
    lat = 0;
    intf = lat + 8 * KG;
    seg_lat = intf + 8 * KG;
    seg_intf = seg_lat + 8 * (size_t)K;
    seg_gpu = seg_intf + 8 * (size_t)K;
    flags = seg_gpu + 4 * (size_t)K;
    recs = (flags + KG + 15) & ~(size_t)15;
    bytes = recs + (size_t)stage_stride * G;
  }
};

// check_violate (scheduler.py:118-161) + check_meet (:164-185) of candidate
// size k on record `r`.  Returns the STRAIT_PAIR_* flags; err_pos >= 0 when a
// running entry's timeline read raises (ValueError) before a verdict.
template <int NM>
__device__ uint8_t eval_pair(const StraitProposeArgs& a, const Pred<NM>& pr, const void* r, int k, double& lat,
                             double& intf, int& err_pos, int& err_kind) {
  const StraitGpuHdr* h = hdr(r);
  const StraitNodeEntry* ent = entries(r);
  const int K = a.k_max, kk = k - 1;
  const double now = a.now;
  lat = intf = nan_d();
  err_pos = -1;
  err_kind = 0;
  const bool has_slot = h->n_running < h->concurrency_limit;  // runtime.py:101-102
  // best_for skips a full GPU; check_violate / check_meet called on their own
  // (fixed_size) answer regardless, like the reference functions
  if (!has_slot && a.fixed_size == 0) return 0;
  uint8_t flags = has_slot ? STRAIT_PAIR_HAS_SLOT : 0;
  double add[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) add[m] = a.cand_contrib[m * K + kk];
  bool violate = false;
  if (a.use_violate) {
    if (a.cand_prio == 1) {  // LOW candidate against the AIMD cap (scheduler.py:129-135)
      const double cap = h->cap_pct / 100.0;
      double lp[NM];
      lp_aggregate(r, lp);
#pragma unroll
      for (int m = 0; m < NM; ++m)
        if (lp[m] + add[m] > cap) violate = true;
    }
    for (int j = 0; !violate && j < h->n_running; ++j) {
      const StraitNodeEntry& e = ent[j];
      if (e.prio > a.cand_prio) continue;  // lower priority than the candidate: may be sacrificed
      double nagg[NM], tw[NM];
#pragma unroll
      for (int m = 0; m < NM; ++m) nagg[m] = h->agg[m] - e.contrib[m] + add[m];
      const double intf_new = pr.predict(nagg, e.self_cmp, e.self_mem, e.prio);
      const double ks = e.started ? e.kernel_start : e.kstart_est;
      const int st = tl_twa(e, NM, now, tw);
      if (st) {
        err_pos = j;
        err_kind = st;
        return flags;
      }
      const double intf_cur = pr.predict(tw, e.self_cmp, e.self_mem, e.prio);
      const double elapsed = py_max(0.0, now - ks);
      const double denom = intf_cur * e.t_kernel;
      const double progress = denom > 0 ? py_min(1.0, elapsed / denom) : 1.0;
      const double remaining = (1.0 - progress) * e.t_kernel * intf_new;
      if (py_max(now, ks) + remaining > e.deadline_abs) violate = true;
    }
    if (violate) flags |= STRAIT_PAIR_VIOLATE;
  }
  double assumed[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) assumed[m] = 0.5 * h->agg[m];
  intf = pr.predict(assumed, a.cand_self_cmp[kk], a.cand_self_mem[kk], a.cand_prio);
  // _latency_parts (scheduler.py:106-114): ((total + pcie delay) + kernel delay) + queueing
  lat = a.cand_total[kk] + py_max(0.0, h->t_available - now) + (intf - 1.0) * a.cand_kernel[kk] +
        (now - a.front_arrival);
  const bool ok = lat <= a.deadline_ms;
  if (ok) flags |= STRAIT_PAIR_MEET;
  if (has_slot && !(a.use_violate && violate) && !(a.use_meet && !ok)) flags |= STRAIT_PAIR_FEASIBLE;
  return flags;
}

template <int NM>
__global__ void __launch_bounds__(kProposeThreads) node_propose_kernel(const StraitProposeArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Pred<NM> pr;
  __shared__ int s_err_k;
  const int G = a.n_gpus, K = a.k_max, tid = threadIdx.x;
  const ProposeLayout L(K, G, a.stage_stride);
  double* s_lat = (double*)(smem + L.lat);
  double* s_intf = (double*)(smem + L.intf);
  double* s_seg_lat = (double*)(smem + L.seg_lat);
  double* s_seg_intf = (double*)(smem + L.seg_intf);
  int* s_seg_gpu = (int*)(smem + L.seg_gpu);
  uint8_t* s_flags = (uint8_t*)(smem + L.flags);
  if (tid == 0) {
    pr.load(a.params, a.effect_cap);
    s_err_k = INT_MAX;
  }
  // ---- stage each record's header + live entries (one pass over the page-locked
  //      records: all loads in flight together, then the stores)
  const bool staged = a.stage_stride > 0;
  if (staged) {
    __shared__ int s_words[1024];
    for (int g = tid; g < G; g += kProposeThreads)
      s_words[g] = (int)((sizeof(StraitGpuHdr) + sizeof(StraitNodeEntry) * hdr(a.recs[g])->n_running) / 8);
    __syncthreads();
    const int wpr = a.stage_stride / 8;
    constexpr int kBatch = 8;
    for (int base = tid; base < G * wpr; base += kProposeThreads * kBatch) {
      double v[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int q = base + u * kProposeThreads, g = q / wpr, w = q - g * wpr;
        v[u] = (q < G * wpr && w < s_words[g]) ? ((const double*)a.recs[g])[w] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int q = base + u * kProposeThreads;
        if (q < G * wpr) ((double*)(smem + L.recs))[q] = v[u];
      }
    }
  }
  __syncthreads();
  auto rec = [&](int g) -> const void* {
    return staged ? (const void*)(smem + L.recs + (size_t)g * a.stage_stride) : a.recs[g];
  };

  // ---- every (size, GPU) pair: has_slot / check_violate / check_meet
  const int k_lo = a.fixed_size > 0 ? a.fixed_size : 1;
  const int nk = a.fixed_size > 0 ? 1 : K;
  for (int p = tid; p < nk * G; p += kProposeThreads) {
    const int k = k_lo + p / G, g = p % G;
    const int q = (k - 1) * G + g;
    int ep, ek;
    s_flags[q] = eval_pair<NM>(a, pr, rec(g), k, s_lat[q], s_intf[q], ep, ek);
    if (ep >= 0) atomicMin(&s_err_k, k);
  }
  __syncthreads();

  // ---- best_for per size: GPUs in list order, replaced when (latency, gpu_id)
  //      is smaller as a Python tuple (first unequal element decides; NaN never wins)
  for (int kk = tid; kk < nk; kk += kProposeThreads) {
    const int k = k_lo + kk;
    int best = -1, bid = 0;
    double bl = 0.0;
    for (int g = 0; g < G; ++g) {
      const int q = (k - 1) * G + g;
      if (!(s_flags[q] & STRAIT_PAIR_FEASIBLE)) continue;
      const double l = s_lat[q];
      const int id = hdr(rec(g))->gpu_id;
      if (best < 0 || (l == bl ? id < bid : l < bl)) {
        best = g;
        bl = l;
        bid = id;
      }
    }
    s_seg_gpu[k - 1] = best;
    s_seg_lat[k - 1] = best >= 0 ? s_lat[(k - 1) * G + best] : nan_d();
    s_seg_intf[k - 1] = best >= 0 ? s_intf[(k - 1) * G + best] : nan_d();
  }
  __syncthreads();

  // ---- outputs the caller asked for
  for (int p = tid; p < nk * G; p += kProposeThreads) {
    const int q = (k_lo - 1) * G + p;
    if (a.pair_flags) a.pair_flags[q] = s_flags[q];
    if (a.pair_latency) a.pair_latency[q] = s_lat[q];
    if (a.pair_intf) a.pair_intf[q] = s_intf[q];
  }
  for (int kk = tid; kk < nk; kk += kProposeThreads) {
    const int i = k_lo - 1 + kk;
    if (a.seg_gpu) a.seg_gpu[i] = s_seg_gpu[i];
    if (a.seg_latency) a.seg_latency[i] = s_seg_lat[i];
    if (a.seg_intf) a.seg_intf[i] = s_seg_intf[i];
  }

  // ---- largest_feasible's probe sequence (scheduler.py:78-90) over the memoised best_for
  if (tid == 0) {
    StraitProposeOut o;
    o.status = STRAIT_OK;
    o.size = 0;
    o.gpu_index = o.err_gpu = o.err_pos = -1;
    o.err_kind = o.probes = o.pad = 0;
    o.latency = o.intf = nan_d();
    int lo = k_lo, hi = k_lo + nk - 1, best = 0;
    while (lo <= hi) {
      const int mid = a.fixed_size > 0 ? a.fixed_size : (lo + hi) / 2;
      o.probes += 1;
      if (mid >= s_err_k) {  // best_for(mid) reads a malformed entry: the reference raises there
        for (int g = 0; g < G; ++g) {
          double lat, intf;
          int ep, ek;
          eval_pair<NM>(a, pr, rec(g), mid, lat, intf, ep, ek);
          if (ep >= 0) {
            o.status = STRAIT_EINVAL;
            o.err_gpu = g;
            o.err_pos = ep;
            o.err_kind = ek;
            break;
          }
        }
        if (o.status != STRAIT_OK) break;
      }
      if (s_seg_gpu[mid - 1] >= 0) {
        best = mid;
        lo = mid + 1;
      } else {
        hi = mid - 1;
      }
      if (a.fixed_size > 0) break;
    }
    if (o.status == STRAIT_OK && best > 0) {
      o.size = best;
      o.gpu_index = s_seg_gpu[best - 1];
      o.latency = s_seg_lat[best - 1];
      o.intf = s_seg_intf[best - 1];
    }
    *a.out = o;
  }
}

template <int NM>
int launch_propose(const StraitProposeArgs& a, cudaStream_t s) {
  const ProposeLayout L(a.k_max, a.n_gpus, a.stage_stride);
  if (L.bytes > 200 * 1024)
    return set_error(STRAIT_EINVAL, "propose over %d sizes x %d GPUs needs %zu B of shared memory", a.k_max,
                     a.n_gpus, L.bytes);
  if (L.bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(node_propose_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L.bytes);
    if (e != cudaSuccess) return set_error(STRAIT_ECUDA, "propose smem: %s", cudaGetErrorString(e));
  }
  node_propose_kernel<NM><<<1, kProposeThreads, L.bytes, s>>>(a);
  return check_launch("strait_node_propose");
}

}  // namespace

extern "C" int64_t strait_node_propose_smem(int32_t k_max, int32_t n_gpus, int32_t stage_stride) {
  return (int64_t)ProposeLayout(k_max, n_gpus, stage_stride).bytes;
}

extern "C" int strait_node_propose(const StraitProposeArgs* args, void* stream) {
  if (!args) return set_error(STRAIT_EINVAL, "null args");
  const StraitProposeArgs& a = *args;
  if (a.n_metrics < 1 || a.n_metrics > STRAIT_MAX_METRICS)
    return set_error(STRAIT_EINVAL, "n_metrics %d outside 1..%d", a.n_metrics, STRAIT_MAX_METRICS);
  if (a.n_gpus < 1 || a.k_max < 1) return set_error(STRAIT_EINVAL, "empty propose (%d GPUs, k_max %d)", a.n_gpus, a.k_max);
  if (a.fixed_size > a.k_max) return set_error(STRAIT_EINVAL, "fixed size %d > k_max %d", a.fixed_size, a.k_max);
  if (a.stage_stride % 8 || (a.stage_stride > 0 && a.n_gpus > 1024))
    return set_error(STRAIT_EINVAL, "bad stage stride %d for %d GPUs", a.stage_stride, a.n_gpus);
  if (!a.recs || !a.out || !a.params) return set_error(STRAIT_EINVAL, "null propose buffer");
  cudaStream_t s = (cudaStream_t)stream;
  switch (a.n_metrics) {
    case 1: return launch_propose<1>(a, s);
    case 2: return launch_propose<2>(a, s);
    case 3: return launch_propose<3>(a, s);
    case 4: return launch_propose<4>(a, s);
    case 5: return launch_propose<5>(a, s);
    case 6: return launch_propose<6>(a, s);
    case 7: return launch_propose<7>(a, s);
    default: return launch_propose<8>(a, s);
  }
}
