/*
 * strait.h — C-ABI of the B200 (sm_100a) estimator + dispatch path of Strait
 * (arXiv 2604.28175).  This is the drop-in boundary: the Python host mirror in
 * paper_2604_28175_b200/ binds these symbols with ctypes, and any other host
 * (C++, cgo, JNI) can bind them the same way.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers owned by the caller, laid out as
 *    structure-of-arrays (SoA).  Per-metric arrays are metric-major:
 *    a[m * n + i] holds metric m of element i.
 *  - All arithmetic is IEEE binary64, evaluated in the reference's
 *    left-to-right order with no FMA contraction.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call
 *    is stream-ordered and asynchronous; the library never frees or retains
 *    a caller pointer past the call.
 *  - Return value: STRAIT_OK or an error code; strait_last_error() returns a
 *    thread-local message.  Per-element conditions that the reference does
 *    not raise on (saturated effect, skipped non-finite refit) are reported
 *    through output flag arrays, never as errors.
 *
 * Predictor parameter vector P (length n_metrics + 7), the reference's
 * canonical flat layout (predictor.py:64-77):
 *   [scale, base, offset, w_0 .. w_{n-1}, w_cmp, w_mem, coeff_high, coeff_low]
 * Priority codes: 0 = HIGH, 1 = LOW (domain.py:17-21).
 */
#ifndef STRAIT_H
#define STRAIT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STRAIT_ABI_VERSION 2

/* error codes; the Python mirror maps them to the reference's exceptions */
#define STRAIT_OK 0
#define STRAIT_EINVAL 1   /* ValueError            (predictor.py:169-172, domain.py:102-105, pcie.py:28-29) */
#define STRAIT_ERUNTIME 2 /* RuntimeError          (runtime.py:125-126,135-138)                          */
#define STRAIT_EORDER 3   /* SimulationOrderError  (domain.py:241-242, simulation.py:61-66,491-494)      */
#define STRAIT_ECUDA 4    /* CUDA launch / runtime failure                                              */

#define STRAIT_MAX_METRICS 8

/* pair_flags bits written by strait_sweep */
#define STRAIT_PAIR_HAS_SLOT 1u /* len(running) < concurrency_limit      (runtime.py:101-102)  */
#define STRAIT_PAIR_VIOLATE 2u  /* check_violate(...) is True             (scheduler.py:118-161) */
#define STRAIT_PAIR_MEET 4u     /* check_meet(...)[0] is True             (scheduler.py:164-185) */
#define STRAIT_PAIR_FEASIBLE 8u /* admitted by best_for under the flags   (scheduler.py:263-280) */

int strait_abi_version(void);
/* sizeof of each ABI struct, so bindings can verify their mirrors (HOST only):
 * 0 StraitSweepArgs, 1 StraitSweepExpandArgs, 2 StraitRefitArgs, 3 StraitReplayModels,
 * 4 StraitReplayConfig, 5 StraitReplayArgs, 6 StraitTraceRec, 7 StraitMetricsArgs,
 * 8 StraitStreamSpec, 9 StraitGroundTruth, 10 StraitGpuHdr, 11 StraitNodeEntry, 12 StraitProposeArgs,
 * 13 StraitProposeOut (strait_node.h); -1 for an unknown id */
int64_t strait_struct_size(int32_t id);
const char *strait_last_error(void);
/* number of device kernels this library launched since load (evidence counter) */
int64_t strait_kernel_launches(void);
/* which sweep kernel the last strait_sweep/strait_round used:
 * 1 synchronous, 2 bulk-copy pipeline, 3 tensor-map pipeline */
int strait_last_sweep_path(void);

/*
 * Elementwise device math with the reference host's bits: fn 0 exp(x),
 * 1 log(x), 2 pow(x, y), 3 log1p(x) — restatements of glibc 2.39's
 * exp/log/pow/log1p (the libm behind CPython's math.exp, math.log and
 * float.__pow__, which predictor.py:136-137,181-184,289-293 and oracle.py:73
 * call, and behind numpy's ziggurat tails).  fn 4 is x / y through the
 * engine's certified shared-divisor division (must equal IEEE division).
 * y may be NULL unless fn == 2 or 4.
 */
int strait_math(int32_t fn, const double *x, const double *y, int64_t n, double *out, void *stream);

/* loss_gradient (predictor.py:271-309) of n independent samples under ONE
 * parameter vector params[n_metrics + 7]: out_grad is [n_metrics + 7][n]
 * (huber_grad(residual) * d(prediction)/d(theta), the inactive coefficient 0).
 * out_saturated is nullable. */
int strait_loss_gradient(const double *params, int32_t n_metrics, double effect_cap, double huber_delta,
                         const double *twa, const double *self_cmp, const double *self_mem, const int8_t *prio,
                         const double *actual, int64_t n, double *out_predicted, double *out_residual,
                         uint8_t *out_saturated, double *out_grad, void *stream);
/* One adam_step (predictor.py:124-145) over n entries in place, after the
 * caller advanced opt.step to t: bc1 = 1 - beta1**t, bc2 = 1 - beta2**t.
 * active is nullable; inactive entries keep value and moments. */
int strait_adam_step(double *values, double *m, double *v, const double *grads, const uint8_t *active, int32_t n,
                     double bc1, double bc2, double learning_rate, double beta1, double beta2, double eps,
                     void *stream);
/* huber_loss / huber_grad (predictor.py:148-158); either output nullable. */
int strait_huber(const double *residual, double delta, int64_t n, double *out_loss, double *out_grad, void *stream);

/* Hidden ground-truth slowdown of the simulated GPUs (oracle.py:18-77): */
typedef struct StraitGroundTruth {
  int32_t family;     /* 0 exponential (scale * base**x + offset), 1 quadratic (scale * x*x + offset) */
  int32_t n_metrics;  /* == len(weights) */
  double scale, base, offset, w_cmp, w_mem;
  double pf_high, pf_low; /* priority_factor */
  double w[STRAIT_MAX_METRICS];
} StraitGroundTruth;
/* out[i] = ground_truth_slowdown(gt, colocated[:, i], self_cmp[i], self_mem[i], prio[i], noise[i])
 * (oracle.py:55-77): x = w_cmp*cmp + w_mem*mem, then x += w_k*a_k in metric order;
 * 1 + max(0, effect) * priority_factor * noise.  colocated is [n_metrics][n];
 * noise is nullable (1.0).  Replaces ground_truth_slowdown (oracle.py:55-77). */
int strait_gt_slowdown(const StraitGroundTruth *gt, const double *colocated, const double *self_cmp,
                       const double *self_mem, const int8_t *prio, const double *noise, int64_t n, double *out,
                       void *stream);

/*
 * R1-R3: batched predict_interference (predictor.py:208-216).
 *   coloc [n_metrics][n], self_cmp[n], self_mem[n], prio[n] -> out_intf[n],
 *   out_saturated[n] (the _raw_effect saturation flag, predictor.py:179-185;
 *   may be NULL).
 */
int strait_predict(const double *params, int32_t n_metrics, double effect_cap,
                   const double *coloc, const double *self_cmp, const double *self_mem,
                   const int8_t *prio, int64_t n, double *out_intf, uint8_t *out_saturated,
                   void *stream);

/*
 * R1-R3 with the intermediate terms: out_exponent[n] = pressure_exponent
 * (predictor.py:161-176), out_effect[n] = kernel_effect (:188-195),
 * out_intf[n] = interference_degree (:198-200).  Any output may be NULL.
 */
int strait_predict_parts(const double *params, int32_t n_metrics, double effect_cap,
                         const double *coloc, const double *self_cmp, const double *self_mem,
                         const int8_t *prio, int64_t n, double *out_exponent, double *out_effect,
                         double *out_intf, uint8_t *out_saturated, void *stream);

/*
 * R2: kernel_effect (predictor.py:188-195) of given exponents x[n].
 */
int strait_kernel_effect(const double *params, int32_t n_metrics, double effect_cap, const double *x,
                         int64_t n, double *out_effect, uint8_t *out_saturated, void *stream);

/*
 * R4: batched estimate_latency (predictor.py:219-242 == scheduler.py:93-115):
 *   ((total + max(0, t_avail - now)) + (intf - 1) * kernel) + (now - front)
 * with intf = predict(assumed, self_cmp, self_mem, prio).  `now` is per element.
 * out_intf may be NULL.
 */
int strait_estimate_latency(const double *params, int32_t n_metrics, double effect_cap,
                            const double *assumed, const double *self_cmp, const double *self_mem,
                            const int8_t *prio, const double *total, const double *kernel,
                            const double *t_avail, const double *front, const double *now,
                            int64_t n, double *out_latency, double *out_intf, void *stream);

/*
 * R6: ThroughputTimeline.time_weighted_average (domain.py:249-264) for n
 * step-hold timelines in running-integral form: t0 = times[0], t_last =
 * times[-1], v_last[nm][n] = values[-1], acc[nm][n] = sum over closed segments
 * of v_i * (t_{i+1} - t_i) accumulated in sample order.  Output
 *   twa = v_last                                      if end - t0 <= 0
 *       = (acc + v_last * (end - t_last)) / (end - t0) otherwise
 * which is the reference loop's exact operation sequence.  Caller guarantees
 * end >= t_last (the reference raises ValueError otherwise).
 */
int strait_twa(int32_t n_metrics, const double *t0, const double *t_last, const double *v_last,
               const double *acc, const double *end, int64_t n, double *out_twa, void *stream);

/*
 * R1-R4, R9-R11: the candidate sweep.  A *segment* is one candidate batch
 * (model at size k, front enqueue time) scored against `gpus_per_segment`
 * GPU states (*pairs*), each with `n_slots` co-runner slots (*triples*) of
 * which the first n_running are live (list order of GpuRuntimeState.running).
 *   pair   p = seg * gpus_per_segment + g   (g doubles as the gpu_id tie-break)
 *   triple t = p * n_slots + c
 * For every pair: has_slot, check_violate (LP cap + projection of every
 * equal-or-higher-priority co-runner), check_meet; per segment the
 * lexicographic (latency, gpu_id) argmin over admitted pairs (best_for).
 * n_slots must be a power of two <= 32 and >= every n_running.
 */
typedef struct StraitSweepArgs {
  int32_t n_metrics;         /* 1..STRAIT_MAX_METRICS */
  int32_t n_slots;           /* C: co-runner slots per pair */
  int32_t gpus_per_segment;  /* G */
  int32_t concurrency_limit; /* GpuRuntimeState.concurrency_limit */
  int64_t n_segments;
  double now;
  double effect_cap;         /* PredictorParams.effect_cap */
  int32_t use_violate;       /* PredictivePolicy.use_violate */
  int32_t use_meet;          /* PredictivePolicy.use_meet */
  const double *params;      /* [n_metrics + 7] */
  /* candidate (segment) SoA: profile row at size k */
  const double *cand_contrib;  /* [nm][S] throughput_at(k) */
  const double *cand_self_cmp; /* [S] */
  const double *cand_self_mem; /* [S] */
  const double *cand_total;    /* [S] total_latency_ms(k) */
  const double *cand_kernel;   /* [S] kernel_latency_ms(k) */
  const double *cand_deadline; /* [S] profile.deadline_ms (relative) */
  const double *cand_front;    /* [S] front request arrival_time */
  const int8_t *cand_prio;     /* [S] */
  /* GPU (pair) SoA */
  const double *gpu_agg;       /* [nm][P] aggregate_throughput */
  const double *gpu_lp_agg;    /* [nm][P] low_priority_aggregate() */
  const double *gpu_cap_pct;   /* [P] aimd.cap_pct */
  const double *gpu_t_avail;   /* [P] pcie.t_available */
  const int8_t *gpu_n_running; /* [P] len(running) */
  /* co-runner (triple) SoA */
  const double *ent_contrib;      /* [nm][T] entry.contribution */
  const double *ent_twa;          /* [nm][T] entry.timeline.time_weighted_average(now) */
  const double *ent_self_cmp;     /* [T] */
  const double *ent_self_mem;     /* [T] */
  const double *ent_t_kernel;     /* [T] kernel_latency_ms */
  const double *ent_deadline_abs; /* [T] */
  const double *ent_kstart;       /* [T] kernel_start if started else kernel_start_estimate */
  const int8_t *ent_prio;         /* [T] */
  /* outputs; pair_* may be NULL */
  uint8_t *pair_flags;  /* [P] STRAIT_PAIR_* bits */
  double *pair_latency; /* [P] check_meet latency (NaN when no slot) */
  double *pair_intf;    /* [P] check_meet intf   (NaN when no slot) */
  int32_t *seg_gpu;     /* [S] best gpu index g, -1 if none (best_for(k) is None) */
  double *seg_latency;  /* [S] BatchPlan.est_latency (NaN if none) */
  double *seg_intf;     /* [S] BatchPlan.intf_pred  (NaN if none) */
} StraitSweepArgs;

int strait_sweep(const StraitSweepArgs *args, void *stream);

/*
 * Profile-indexed snapshots for strait_sweep.  Every co-runner's contribution,
 * self_compute / self_memory and isolated kernel latency is its profile row at
 * (model, size) (submit_plan, scheduler.py:295-324), the candidate's likewise,
 * and a GPU's aggregate / LP aggregate are list-order sums of its running
 * entries' contributions (runtime.py:104-122).  A host can therefore ship only
 * row indices plus the non-derived fields; this call fills the derived fields
 * of `target` (ent_contrib, ent_self_cmp, ent_self_mem, ent_t_kernel, ent_prio,
 * gpu_agg, gpu_lp_agg, cand_contrib, cand_self_cmp, cand_self_mem, cand_total,
 * cand_kernel, cand_deadline, cand_prio) exactly as the reference objects hold
 * them.  row = model * table_stride + size - 1.
 */
typedef struct StraitSweepExpandArgs {
  int32_t table_stride; /* profile rows per model (max batch size) */
  int32_t pad;
  const double *thr;      /* [nm][rows] throughput_at(size) */
  const double *self_cmp; /* [rows] */
  const double *self_mem; /* [rows] */
  const double *kernel;   /* [rows] kernel_latency_ms */
  const double *total;    /* [rows] total_latency_ms */
  const double *deadline; /* [models] deadline_ms */
  const int8_t *prio;     /* [models] */
  const int16_t *ent_row; /* [T] */
  const int16_t *cand_row; /* [S] */
  int64_t n_rows;
} StraitSweepExpandArgs;

int strait_sweep_expand(const StraitSweepExpandArgs *e, const StraitSweepArgs *target, void *stream);

/*
 * R14-R16: sequential online refit, InterferencePredictor.update applied to
 * n samples in order (predictor.py:345-363): Huber-loss gradient under the
 * current parameters, non-finite skip, Adam with the other class's
 * coefficient inactive, parameter floors.
 *   state: [3 * (n_metrics + 7)] = params | adam m | adam v   (updated in place)
 *   step:  [1] Adam step counter                               (updated in place)
 *   bc1/bc2: host-computed tables of 1 - beta**t for t = 1..n_bc (the
 *     reference's float pow, predictor.py:136-137); steps past the table use
 *     1.0, which is exact once beta**t < 2**-54.
 *   samples: twa [nm][n], self_cmp[n], self_mem[n], prio[n], actual[n]
 *   outputs (nullable): predicted[n], residual[n],
 *     flags[n] (bit0 skipped, bit1 saturated)   (UpdateResult, predictor.py:263-268)
 */
typedef struct StraitRefitArgs {
  int32_t n_metrics;
  int32_t n_bc;
  int64_t n;
  double effect_cap, learning_rate, beta1, beta2, eps, huber_delta;
  double *state;
  int64_t *step;
  const double *bc1, *bc2;
  const double *twa, *self_cmp, *self_mem, *actual;
  const int8_t *prio;
  double *out_predicted, *out_residual;
  uint8_t *out_flags;
} StraitRefitArgs;

int strait_refit(const StraitRefitArgs *args, void *stream);

/*
 * One scheduling round of the candidate-sweep microbench: strait_sweep under
 * the params in sweep->params, fused in ONE launch with strait_refit over this
 * round's feedback samples (block 0 runs the serial Adam chain while the other
 * blocks stream the sweep).  refit->state must not alias sweep->params; the
 * refit result is the next round's parameter vector.
 */
int strait_round(const StraitSweepArgs *sweep, const StraitRefitArgs *refit, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* STRAIT_H */
