/*
 * strait_node.h — C-ABI of the object-API runtime state: one flat, fixed-layout
 * record per simulated GPU that holds what the reference keeps in three Python
 * objects, plus the entry points that mutate it and the one-launch device
 * propose that reads it in place.
 *
 *   GpuRuntimeState  runtime.py:82-141  running list, aggregates, has_slot
 *   PcieLinkState    pcie.py:13-53      t_available + FIFO of pending transfer ends
 *   AimdState        runtime.py:13-40   LP cap, additive increase, reset
 *   RunningTaskEntry runtime.py:53-72   one running batch + its ThroughputTimeline
 *                                       (domain.py:217-264, kept in running-integral
 *                                       form: t0, t_last, v_last, acc)
 *
 * Record layout (byte offsets; every field naturally aligned):
 *   [StraitGpuHdr][StraitNodeEntry x hdr.slot_cap][double ring[hdr.ring_cap]]
 * Entries are kept in the reference's list order (entry i = running[i]).
 * The pending ring holds the link's FIFO: ring[(ring_head + i) % ring_cap],
 * i < ring_len.
 *
 * Ownership and memory.  The caller allocates records (page-locked host memory
 * on a CUDA box, so that strait_node_propose reads them in place over the
 * unified address space with no staging copy).  The strait_node_* mutators are
 * O(concurrency) host bookkeeping executed in the caller's thread — the same
 * ownership model as the reference, whose caller owns and mutates these objects
 * between passes (SURVEY §8(b) "Ownership").  All scheduling arithmetic on the
 * records (timeline TWA, predictions, check_violate / check_meet projections,
 * best_for argmin, the binary search) runs on the device in strait_node_propose.
 *
 * Errors: STRAIT_EINVAL -> ValueError, STRAIT_ERUNTIME -> RuntimeError,
 * STRAIT_EORDER -> SimulationOrderError (strait.h), STRAIT_ENOSPC: the ring is
 * full, the caller grows the record and retries (not an error of the reference).
 */
#ifndef STRAIT_NODE_H
#define STRAIT_NODE_H

#include <stdint.h>

#include "strait.h"

#ifdef __cplusplus
extern "C" {
#endif

#define STRAIT_ENOSPC 5

typedef struct StraitGpuHdr {
  int32_t gpu_id;
  int32_t n_metrics;
  int32_t concurrency_limit;
  int32_t n_running; /* len(running) */
  int32_t slot_cap;  /* entries allocated after the header */
  int32_t ring_cap;  /* pending-transfer ring capacity */
  int32_t ring_head;
  int32_t ring_len;  /* len(pending) */
  double t_available;  /* pcie.py:18 */
  double cap_pct;      /* runtime.py:23-28 AimdState fields */
  double aimd_floor;
  double aimd_ceiling;
  double aimd_increase;
  double aimd_interval;
  double aimd_last_tick;
  double reserved;
  double agg[STRAIT_MAX_METRICS]; /* aggregate_throughput (list-order sum, runtime.py:104-109) */
} StraitGpuHdr;

typedef struct StraitNodeEntry {
  double contrib[STRAIT_MAX_METRICS]; /* contribution */
  double tl_v[STRAIT_MAX_METRICS];    /* timeline: last recorded value */
  double tl_acc[STRAIT_MAX_METRICS];  /* timeline: sum_i v_i * (t_{i+1} - t_i) over closed segments */
  double self_cmp, self_mem, t_kernel, deadline_abs, kstart_est;
  double kernel_start; /* batch.kernel_start, meaningful when started */
  double intf_pred;
  double tl_t0, tl_tlast;
  int32_t prio;    /* 0 HIGH, 1 LOW (batch.priority) */
  int32_t started; /* kernel_started */
  int32_t tl_n;    /* number of timeline samples */
  int32_t handle;  /* caller's identity of the entry (list.remove is by identity) */
} StraitNodeEntry;

/* bytes of one record with `slot_cap` entries and `ring_cap` ring slots */
int64_t strait_node_record_bytes(int32_t slot_cap, int32_t ring_cap);

/* device address of a page-locked host record (cudaHostGetDevicePointer), NULL
 * with strait_last_error() set if the memory is not device-mapped */
void *strait_node_device_address(void *host_ptr);

/* ---- PcieLinkState (pcie.py:13-53) ---- */
/* estimate_delay (Eq.2): max(0, t_available - now) */
double strait_link_delay(const void *rec, double now);
/* reserve (Eq.3): start = max(now, t_available); end = start + duration; appends end.
 * EINVAL for duration <= 0 (pcie.py:28-29); ENOSPC when the ring is full. */
int strait_link_reserve(void *rec, double now, double duration, double *out_start, double *out_end);
/* calibrate: pops the oldest pending end; EINVAL with nothing pending (pcie.py:43-44) */
int strait_link_calibrate(void *rec, double actual_end);

/* ---- AimdState (runtime.py:13-40) ---- */
/* advance: EINVAL when now < last_tick */
int strait_aimd_advance(void *rec, double now);
void strait_aimd_reset(void *rec);

/* ---- ThroughputTimeline of one entry (domain.py:237-264), wherever the entry lives
 *      (a record slot or the caller's detached copy) ---- */
/* record: EORDER if now precedes the last sample; equal time replaces the value */
int strait_entry_tl_record(StraitNodeEntry *entry, int32_t n_metrics, double now, const double *value);
/* time_weighted_average into out[n_metrics]: EINVAL with no samples or end before the last sample */
int strait_entry_tl_twa(const StraitNodeEntry *entry, int32_t n_metrics, double end, double *out);

/* ---- GpuRuntimeState (runtime.py:82-141) ---- */
/* aggregate_excluding(running[pos]) and low_priority_aggregate(), into out[n_metrics] */
int strait_node_excluding(const void *rec, int32_t pos, double *out);
void strait_node_lp_aggregate(const void *rec, double *out);
/* add_entry: appends `entry` (its timeline fields as the caller built them),
 * recomputes the aggregate in list order and records agg - contrib on every
 * running entry's timeline at `now`.  ERUNTIME when no slot is free
 * (runtime.py:125-126); ENOSPC when slot_cap is exhausted (caller grows). */
int strait_node_add(void *rec, const StraitNodeEntry *entry, double now);
/* remove_entry by handle, same recompute + restamp.  ERUNTIME when the handle
 * is not running here (runtime.py:135-138).  out_removed (nullable) receives
 * the removed entry. */
int strait_node_remove(void *rec, int32_t handle, double now, StraitNodeEntry *out_removed);
/* position of `handle` in the running list, or -1 */
int32_t strait_node_find(const void *rec, int32_t handle);
/* raw list operations with no recompute or restamp (a caller editing `running`
 * directly, e.g. list.clear() / list.remove()): detach copies the entry out and
 * closes the gap (ERUNTIME if absent); attach appends (ENOSPC when slots are full) */
int strait_node_detach(void *rec, int32_t handle, StraitNodeEntry *out_removed);
int strait_node_attach(void *rec, const StraitNodeEntry *entry);

/* ---- composite steps of the scheduling loop ---- */
/* submit_plan's runtime half (scheduler.py:309-323): reserve the link for
 * `transfer_ms` at `now`, set the entry's kernel_start_estimate to the transfer
 * end, then add_entry.  out_start/out_end receive the reservation. */
int strait_node_submit(void *rec, StraitNodeEntry *entry, double transfer_ms, double now, double *out_start,
                       double *out_end);
/* the transfer-complete step (simulation.py:379-388): calibrate(now), mark the
 * entry started at `now`, reset its timeline to [(now, aggregate_excluding)] */
int strait_node_start(void *rec, int32_t handle, double now);
/* complete_batch's runtime half (scheduler.py:327-352): TWA of the entry's
 * timeline at `now` into out_twa[n_metrics], then remove_entry */
int strait_node_complete(void *rec, int32_t handle, double now, double *out_twa, StraitNodeEntry *out_removed);
/* AIMD tick over n records (simulation.py:462-467) / reset (HP violation) */
int strait_nodes_tick(void *const *recs, int32_t n, double now);

/*
 * PredictivePolicy.propose (scheduler.py:257-285) in ONE device launch over the
 * records of `n_gpus` GPUs in the caller's list order: for every size
 * k = 1..k_max and GPU g, has_slot / check_violate (LP cap + the projection of
 * every running entry, each with its timeline TWA) / check_meet, then best_for's
 * (latency, gpu_id) argmin per size and largest_feasible's probe sequence.
 * `recs` is a device-readable array of n_gpus record pointers (page-locked host
 * records are read in place).  The candidate's profile rows for sizes 1..k_max
 * are metric-major: cand_contrib[m * k_max + (k-1)].
 * Output (device-writable, e.g. page-locked host; every array but `out` nullable):
 *   out->size (0 = no feasible size), gpu_index (into recs), latency, intf;
 *   per size k: seg_gpu[k-1] (-1 none), seg_latency, seg_intf;
 *   per (k, g): pair_flags[(k-1) * n_gpus + g] (STRAIT_PAIR_* bits), pair_latency, pair_intf.
 * A malformed running entry (no timeline samples, or now before its last
 * sample) is reported like the reference, which raises in check_violate's
 * timeline read on the first probed size that evaluates it: out->status =
 * STRAIT_EINVAL with out->err_gpu / out->err_pos set.
 */
typedef struct StraitProposeOut {
  int32_t status, size, gpu_index, err_gpu;
  int32_t err_pos, err_kind, probes, pad;
  double latency, intf;
} StraitProposeOut;

typedef struct StraitProposeArgs {
  int32_t n_metrics, n_gpus, k_max, cand_prio;
  int32_t use_violate, use_meet;
  int32_t fixed_size;   /* > 0: evaluate that size only, no search, and evaluate full GPUs too
                           (the standalone check_violate / check_meet) */
  int32_t stage_stride; /* > 0: bytes per record slot when the records are staged in shared memory
                           (>= header + n_running entries, multiple of 8); 0: read them in place */
  double now, effect_cap, deadline_ms, front_arrival;
  const double *params; /* [n_metrics + 7] */
  const void *const *recs;
  const double *cand_contrib, *cand_self_cmp, *cand_self_mem, *cand_total, *cand_kernel; /* [.. k_max] */
  uint8_t *pair_flags;
  double *pair_latency, *pair_intf;
  int32_t *seg_gpu;
  double *seg_latency, *seg_intf;
  StraitProposeOut *out;
} StraitProposeArgs;

int strait_node_propose(const StraitProposeArgs *args, void *stream);
/* dynamic shared memory one propose launch needs (the caller picks stage_stride = 0
 * when staging would not fit); > 200 KiB is refused with EINVAL */
int64_t strait_node_propose_smem(int32_t k_max, int32_t n_gpus, int32_t stage_stride);

#ifdef __cplusplus
}
#endif
#endif
