/*
 * strait_replay_oracle.c — CPU ORACLE of the trace replay (test infrastructure,
 * NOT product code).
 *
 * A literal C restatement of infersim's discrete-event simulator
 * (/root/reference/pkg/src/infersim/simulation.py:122-513) driving the
 * PredictivePolicy (scheduler.py:229-378) with the InterferencePredictor
 * (predictor.py) and the hidden ground truth (oracle.py:55-77): a binary heap
 * of (time, kind, seq, payload) with lazy deletion of stale events, list-order
 * running sets, per-entry step-hold timelines integrated by the reference's
 * loop, general early-drop filtering.  With glibc libm and -ffp-contract=off
 * it reproduces the reference bit for bit (tests/test_replay_oracle.py against
 * golden replays produced by the reference itself).  Inputs/outputs use the
 * device ABI (include/strait_replay.h) so the oracle checks the CUDA engine on
 * identical buffers.  Replays of a batch run on OpenMP threads (the analogue of
 * `infersim sweep --jobs N`, cli.py:76-80).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/strait_replay.h"

#define EV_KC 0 /* simulation.py:28-33 */
#define EV_TC 1
#define EV_ARR 2
#define EV_TO 3
#define EV_TICK 4
#define WORK_EPS 1e-9
#define MAXM STRAIT_MAX_METRICS
#define MAXP (STRAIT_MAX_METRICS + 7)

static inline double py_max(double a, double b) { return (b > a) ? b : a; }
static inline double py_min(double a, double b) { return (b < a) ? b : a; }

typedef struct {
  double time;
  int kind;
  int64_t seq;
  int64_t a, b;
} Ev;

typedef struct {
  Ev *v;
  int64_t n, cap;
} Heap;

static int ev_less(const Ev *x, const Ev *y) {
  if (x->time != y->time) return x->time < y->time;
  if (x->kind != y->kind) return x->kind < y->kind;
  return x->seq < y->seq;
}

static void heap_push(Heap *h, Ev e) {
  if (h->n == h->cap) {
    h->cap = h->cap ? 2 * h->cap : 1024;
    h->v = realloc(h->v, h->cap * sizeof(Ev));
  }
  int64_t i = h->n++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (!ev_less(&e, &h->v[p])) break;
    h->v[i] = h->v[p];
    i = p;
  }
  h->v[i] = e;
}

static Ev heap_pop(Heap *h) {
  Ev top = h->v[0], last = h->v[--h->n];
  int64_t i = 0;
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, m = i;
    const Ev *best = &last;
    if (l < h->n && ev_less(&h->v[l], best)) m = l, best = &h->v[l];
    if (r < h->n && ev_less(&h->v[r], best)) m = r, best = &h->v[r];
    if (m == i) break;
    h->v[i] = h->v[m];
    i = m;
  }
  if (h->n) h->v[i] = last;
  return top;
}

/* ThroughputTimeline (domain.py:217-264) */
typedef struct {
  double *t, *v; /* v[i*nm + k] */
  int n, cap;
} Timeline;

static void tl_clear(Timeline *tl) { tl->n = 0; }
static int tl_record(Timeline *tl, int nm, double now, const double *vec) {
  if (tl->n) {
    double last = tl->t[tl->n - 1];
    if (now < last) return STRAIT_EORDER;
    if (now == last) {
      memcpy(tl->v + (size_t)(tl->n - 1) * nm, vec, nm * sizeof(double));
      return 0;
    }
  }
  if (tl->n == tl->cap) {
    tl->cap = tl->cap ? 2 * tl->cap : 8;
    tl->t = realloc(tl->t, tl->cap * sizeof(double));
    tl->v = realloc(tl->v, (size_t)tl->cap * nm * sizeof(double));
  }
  tl->t[tl->n] = now;
  memcpy(tl->v + (size_t)tl->n * nm, vec, nm * sizeof(double));
  tl->n++;
  return 0;
}
static void tl_twa(const Timeline *tl, int nm, double end, double *out) {
  double total = end - tl->t[0];
  if (total <= 0.0) {
    memcpy(out, tl->v + (size_t)(tl->n - 1) * nm, nm * sizeof(double));
    return;
  }
  double acc[MAXM];
  for (int k = 0; k < nm; ++k) acc[k] = 0.0;
  for (int i = 0; i < tl->n; ++i) {
    double hold = i + 1 < tl->n ? tl->t[i + 1] : end;
    double d = hold - tl->t[i];
    for (int k = 0; k < nm; ++k) acc[k] += tl->v[(size_t)i * nm + k] * d;
  }
  for (int k = 0; k < nm; ++k) out[k] = acc[k] / total;
}

typedef struct { /* RunningTaskEntry + Batch + ExecutionState of one batch */
  int model, size, prio, gpu;
  int64_t req0; /* position in the model's queue storage of the first request */
  double deadline_abs, intf_predicted, kernel_start_estimate, kernel_start;
  int kernel_started;
  Timeline tl;
  double remaining, slowdown, noise, last_update;
  int64_t version;
  int has_exec, live;
  double work;
} Entry;

typedef struct {
  int running[64];
  int n_running;
  double agg[MAXM];
  double t_avail;
  double pending[64];
  int p_head, p_n;
  double cap_pct, last_tick;
} Gpu;

typedef struct {
  const StraitReplayArgs *A;
  const StraitReplayConfig *cfg;
  int64_t r, base, N;
  int nm, M, B, np;
  Heap heap;
  int64_t seq, batch_seq, pass_seq, resolved, done_order;
  Gpu *gpus;
  Entry *ent;              /* by batch id */
  int64_t *q_store;        /* per model: global request indices (mutable copy) */
  int64_t *q_head, *q_tail, *q_beg;
  int64_t *front_gen, *timeout_gen;
  double P[MAXP], Mv[MAXP], Vv[MAXP];
  int64_t step;
  int lp_allowance;   /* ReactiveState (baselines.py:81-110) */
  double last_reset;
  int err;
  int64_t *cnt;
} Sim;

#define MTAB(arr, m, k) (S->A->models.arr[(int64_t)(m) * S->B + (k) - 1])

static double thr(const Sim *S, int m, int k, int i) {
  return S->A->models.throughput[(int64_t)i * S->M * S->B + (int64_t)m * S->B + k - 1];
}

static void set_err(Sim *S, int e) {
  if (!S->err) S->err = e;
}

static void push(Sim *S, double t, int kind, int64_t a, int64_t b) {
  Ev e = {t, kind, ++S->seq, a, b};
  heap_push(&S->heap, e);
}

/* ---------------------------------------------------------------- predictor (predictor.py) */
static double pred_predict(const Sim *S, const double *coloc, double cmp, double mem, int prio, int *sat,
                           double *inner_out, double *x_out) {
  const int nm = S->nm;
  const double *P = S->P;
  double x = P[3 + nm] * cmp + P[4 + nm] * mem;
  for (int i = 0; i < nm; ++i) x += P[3 + i] * coloc[i];
  double z = x * log(P[1]);
  double inner;
  if (z > 500.0) {
    *sat = 1;
    inner = INFINITY;
  } else {
    inner = P[0] * exp(z) + P[2];
    *sat = inner >= S->cfg->effect_cap;
  }
  double eff = *sat ? S->cfg->effect_cap : py_min(py_max(inner, 0.0), S->cfg->effect_cap);
  if (inner_out) *inner_out = inner;
  if (x_out) *x_out = x;
  return 1.0 + eff * P[nm + (prio == 0 ? 5 : 6)];
}

static double predict(const Sim *S, const double *coloc, double cmp, double mem, int prio) {
  int sat;
  return pred_predict(S, coloc, cmp, mem, prio, &sat, NULL, NULL);
}

/* InterferencePredictor.update (predictor.py:345-363) */
static void pred_update(Sim *S, const double *twa, double cmp, double mem, int prio, double actual,
                        double *predicted, double *residual, int *skipped, int *saturated) {
  const int nm = S->nm, np = S->np;
  double *P = S->P;
  const double cap = S->cfg->effect_cap;
  int sat;
  double inner, x;
  double pred = pred_predict(S, twa, cmp, mem, prio, &sat, &inner, &x);
  double eff = sat ? cap : py_min(py_max(inner, 0.0), cap);
  double cf = P[nm + (prio == 0 ? 5 : 6)];
  double grad[MAXP];
  for (int k = 0; k < np; ++k) grad[k] = 0.0;
  if (!(sat || inner <= 0.0 || inner >= cap)) {
    double pow_bx = exp(x * log(P[1]));
    double z = P[0] * pow_bx;
    double log_b = log(P[1]);
    grad[0] = pow_bx * cf;
    grad[1] = P[0] * x * exp((x - 1.0) * log_b) * cf;
    grad[2] = cf;
    for (int i = 0; i < nm; ++i) grad[3 + i] = z * log_b * twa[i] * cf;
    grad[3 + nm] = z * log_b * cmp * cf;
    grad[4 + nm] = z * log_b * mem * cf;
  }
  int own = nm + (prio == 0 ? 5 : 6), other = nm + (prio == 0 ? 6 : 5);
  grad[own] = eff;
  double res = pred - actual;
  double delta = S->cfg->huber_delta;
  double g = fabs(res) <= delta ? res : (res > 0 ? delta : -delta);
  int finite = isfinite(res);
  for (int k = 0; k < np; ++k) {
    grad[k] = g * grad[k];
    if (!isfinite(grad[k])) finite = 0;
  }
  *predicted = pred;
  *residual = res;
  *saturated = sat;
  *skipped = !finite && !S->cfg->refit_frozen;
  if (!finite || S->cfg->refit_frozen) return; /* frozen update(): loss terms only, never steps */
  int64_t t = ++S->step;
  double b1 = S->cfg->beta1, b2 = S->cfg->beta2;
  double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
  for (int k = 0; k < np; ++k) {
    if (k == other) continue;
    S->Mv[k] = b1 * S->Mv[k] + (1.0 - b1) * grad[k];
    S->Vv[k] = b2 * S->Vv[k] + (1.0 - b2) * grad[k] * grad[k];
    double m_hat = S->Mv[k] / bc1, v_hat = S->Vv[k] / bc2;
    P[k] -= S->cfg->learning_rate * m_hat / (sqrt(v_hat) + S->cfg->eps);
  }
  P[0] = py_max(P[0], 1e-6);
  P[1] = py_max(P[1], 1.0 + 1e-6);
  P[nm + 5] = py_max(P[nm + 5], 1e-6);
  P[nm + 6] = py_max(P[nm + 6], 1e-6);
}

/* ---------------------------------------------------------------- runtime (runtime.py) */
static void cap_row(Sim *S, double t, int g) {
  int64_t n = S->cnt[STRAIT_RC_CAP_ROWS]++;
  if (n < S->A->cap_rows_max) {
    int64_t o = S->r * S->A->cap_rows_max + n;
    S->A->cap_time[o] = t;
    S->A->cap_gpu[o] = (int16_t)g;
    S->A->cap_pct[o] = S->gpus[g].cap_pct;
  }
}

static void recompute_aggregate(Sim *S, Gpu *g) {
  for (int i = 0; i < S->nm; ++i) g->agg[i] = 0.0;
  for (int j = 0; j < g->n_running; ++j) {
    const Entry *e = &S->ent[g->running[j]];
    for (int i = 0; i < S->nm; ++i) g->agg[i] += thr(S, e->model, e->size, i);
  }
}

static void aggregate_excluding(const Sim *S, const Gpu *g, const Entry *e, double *out) {
  for (int i = 0; i < S->nm; ++i) out[i] = g->agg[i] - thr(S, e->model, e->size, i);
}

static void stamp_all(Sim *S, Gpu *g, double now) {
  for (int j = 0; j < g->n_running; ++j) {
    Entry *e = &S->ent[g->running[j]];
    double v[MAXM];
    aggregate_excluding(S, g, e, v);
    if (tl_record(&e->tl, S->nm, now, v)) set_err(S, STRAIT_EORDER);
  }
}

/* ---------------------------------------------------------------- ground truth (oracle.py:55-77) */
static double gt_slowdown(const Sim *S, const Gpu *g, const Entry *e) {
  const StraitReplayConfig *c = S->cfg;
  double a[MAXM];
  aggregate_excluding(S, g, e, a);
  double cmp = MTAB(self_cmp, e->model, e->size), mem = MTAB(self_mem, e->model, e->size);
  double x = c->gt_w_cmp * cmp + c->gt_w_mem * mem;
  for (int i = 0; i < S->nm; ++i) x += c->gt_w[i] * a[i];
  double effect = c->gt_family == 0 ? c->gt_scale * pow(c->gt_base, x) + c->gt_offset
                                    : c->gt_scale * x * x + c->gt_offset;
  effect = py_max(0.0, effect);
  return 1.0 + effect * (e->prio == 0 ? c->gt_pf_high : c->gt_pf_low) * e->noise;
}

/* ExecutionState (simulation.py:38-83) */
static void ex_consume(Sim *S, Entry *e, double now) {
  double d = now - e->last_update;
  if (d < 0) set_err(S, STRAIT_EORDER);
  if (d > 0) {
    e->work += d / e->slowdown;
    e->remaining -= d / e->slowdown;
    if (e->remaining < -WORK_EPS) set_err(S, STRAIT_EORDER);
    if (e->remaining < 0.0) e->remaining = 0.0;
  }
  e->last_update = now;
}
static double ex_eta(const Entry *e) { return e->last_update + e->remaining * e->slowdown; }

static void recompute(Sim *S, int gi, double now) { /* simulation.py:290-297 */
  Gpu *g = &S->gpus[gi];
  for (int j = 0; j < g->n_running; ++j) {
    int bid = g->running[j];
    Entry *e = &S->ent[bid];
    if (!e->kernel_started) continue;
    ex_consume(S, e, now);
    e->slowdown = gt_slowdown(S, g, e);
    e->version++;
    push(S, ex_eta(e), EV_KC, bid, e->version);
  }
}

/* ---------------------------------------------------------------- dispatch (scheduler.py) */
static int64_t q_len(const Sim *S, int m) { return S->q_tail[m] - S->q_head[m]; }
static double req_arr(const Sim *S, int64_t gi) { return S->A->arr_time[gi]; }
static double req_deadline(const Sim *S, int m, int64_t gi) { return req_arr(S, gi) + S->A->models.deadline[m]; }

/* ReactiveState.catch_up (baselines.py:99-104) */
static void reactive_catch_up(Sim *S, double now) {
  const double period = S->cfg->reactive_period;
  if (now - S->last_reset >= period) {
    double periods = floor((now - S->last_reset) / period);
    S->lp_allowance = S->cfg->reactive_default;
    S->last_reset += periods * period;
  }
}

static void signal_hp_violation(Sim *S, int gpu_id, double now) { /* simulation.py:223-229 */
  if (S->cfg->policy != STRAIT_POLICY_PREDICTIVE) {
    /* baselines: TemporalPolicy / StaticSpatialPolicy inherit the no-op
     * on_hp_violation (scheduler.py:225-226); ReactiveSpatialPolicy shrinks the
     * LP allowance (baselines.py:131-133, 106-107).  AIMD caps never change. */
    if (S->cfg->policy == STRAIT_POLICY_REACTIVE) {
      reactive_catch_up(S, now);
      int a = S->lp_allowance - 1;
      S->lp_allowance = a > S->cfg->reactive_min ? a : S->cfg->reactive_min;
    }
    return;
  }
  for (int g = 0; g < S->cfg->n_gpus; ++g) {
    if (gpu_id >= 0 && g != gpu_id) continue;
    double old = S->gpus[g].cap_pct;
    S->gpus[g].cap_pct = S->cfg->aimd_floor;
    if (S->gpus[g].cap_pct != old) cap_row(S, now, g);
  }
}

static void resolve_dropped(Sim *S, int m, int64_t gi) {
  S->A->req_status[gi] = 2;
  S->A->req_violated[gi] = 1;
  S->A->req_completion[gi] = NAN;
  S->A->req_batch[gi] = -1;
  S->resolved++;
  if (S->A->models.prio[m] == 0) S->cnt[STRAIT_RC_HP_DROP]++, S->cnt[STRAIT_RC_HP_VIOL]++;
  else S->cnt[STRAIT_RC_LP_DROP]++, S->cnt[STRAIT_RC_LP_VIOL]++;
}

/* early_drop (scheduler.py:65-75): general order-preserving filter.  Survivors
 * are packed towards the tail so the window stays contiguous with the
 * not-yet-arrived requests that follow it in q_store. */
static void early_drop(Sim *S, int m, double now) {
  double floor_latency = MTAB(total, m, 1);
  int64_t h = S->q_head[m], t = S->q_tail[m], ndrop = 0;
  if (h == t) return;
  int64_t old_front = S->q_store[h];
  for (int64_t i = h; i < t; ++i)
    if (req_deadline(S, m, S->q_store[i]) - now < floor_latency) ndrop++;
  if (!ndrop) return;
  for (int64_t i = h; i < t; ++i) {
    int64_t gi = S->q_store[i];
    if (req_deadline(S, m, gi) - now < floor_latency) resolve_dropped(S, m, gi);
  }
  int64_t w = t;
  for (int64_t i = t - 1; i >= h; --i) {
    int64_t gi = S->q_store[i];
    if (!(req_deadline(S, m, gi) - now < floor_latency)) S->q_store[--w] = gi;
  }
  S->q_head[m] = w;
  if (S->q_tail[m] == S->q_head[m] || S->q_store[S->q_head[m]] != old_front) S->front_gen[m]++;
  if (S->A->models.prio[m] == 0) signal_hp_violation(S, -1, now);
}

typedef struct {
  int ok;
  int gpu;
  double lat, intf;
} Plan;

static int check_violate(Sim *S, const Gpu *g, int m, int k, double now) {
  int cprio = S->A->models.prio[m];
  if (cprio == 1) {
    double capf = g->cap_pct / 100.0;
    double lp[MAXM];
    for (int i = 0; i < S->nm; ++i) lp[i] = 0.0;
    for (int j = 0; j < g->n_running; ++j) {
      const Entry *e = &S->ent[g->running[j]];
      if (e->prio == 1)
        for (int i = 0; i < S->nm; ++i) lp[i] += thr(S, e->model, e->size, i);
    }
    for (int i = 0; i < S->nm; ++i)
      if (lp[i] + thr(S, m, k, i) > capf) return 1;
  }
  for (int j = 0; j < g->n_running; ++j) {
    const Entry *e = &S->ent[g->running[j]];
    if (e->prio > cprio) continue;
    double nagg[MAXM], twa[MAXM];
    for (int i = 0; i < S->nm; ++i) nagg[i] = g->agg[i] - thr(S, e->model, e->size, i) + thr(S, m, k, i);
    double cmp = MTAB(self_cmp, e->model, e->size), mem = MTAB(self_mem, e->model, e->size);
    double intf_new = predict(S, nagg, cmp, mem, e->prio);
    double ks = e->kernel_started ? e->kernel_start : e->kernel_start_estimate;
    tl_twa(&e->tl, S->nm, now, twa);
    double intf_cur = predict(S, twa, cmp, mem, e->prio);
    double tk = MTAB(kernel, e->model, e->size);
    double elapsed = py_max(0.0, now - ks);
    double denom = intf_cur * tk;
    double progress = denom > 0 ? py_min(1.0, elapsed / denom) : 1.0;
    double remaining = (1.0 - progress) * tk * intf_new;
    double projected = py_max(now, ks) + remaining;
    if (projected > e->deadline_abs) return 1;
  }
  return 0;
}

static void check_meet(Sim *S, const Gpu *g, int m, int k, double front, double now, int *ok, double *lat,
                       double *intf) {
  double assumed[MAXM];
  for (int i = 0; i < S->nm; ++i) assumed[i] = 0.5 * g->agg[i];
  *intf = predict(S, assumed, MTAB(self_cmp, m, k), MTAB(self_mem, m, k), S->A->models.prio[m]);
  *lat = MTAB(total, m, k) + py_max(0.0, g->t_avail - now) + (*intf - 1.0) * MTAB(kernel, m, k) + (now - front);
  *ok = *lat <= S->A->models.deadline[m];
}

static Plan best_for(Sim *S, int m, int k, double front, double now) {
  Plan best = {0, -1, 0, 0};
  for (int gi = 0; gi < S->cfg->n_gpus; ++gi) {
    const Gpu *g = &S->gpus[gi];
    if (!(g->n_running < S->cfg->concurrency_limit)) continue;
    if (S->cfg->use_violate && check_violate(S, g, m, k, now)) continue;
    int ok;
    double lat, intf;
    check_meet(S, g, m, k, front, now, &ok, &lat, &intf);
    if (S->cfg->use_meet && !ok) continue;
    if (!best.ok || lat < best.lat) best = (Plan){1, gi, lat, intf};
  }
  return best;
}

/* _isolated_latency_plan (baselines.py:34-37): est = (now - front) + total(size), intf 1.0 */
static Plan isolated_plan(Sim *S, int m, int gpu, int size, double now) {
  double front = req_arr(S, S->q_store[S->q_head[m]]);
  Plan p = {size, gpu, (now - front) + MTAB(total, m, size), 1.0};
  return p;
}

/* the baselines' propose (baselines.py:40-128); returns size in .ok, 0 = None */
static Plan propose_baseline(Sim *S, int m, double now) {
  Plan none = {0, -1, 0, 0};
  const int G = S->cfg->n_gpus, pol = S->cfg->policy;
  int64_t len = q_len(S, m);
  int kmax = (int)(len < S->A->models.max_batch[m] ? len : S->A->models.max_batch[m]);
  if (pol == STRAIT_POLICY_TEMPORAL) { /* first idle GPU, largest isolated-feasible size */
    int idle = -1;
    for (int g = 0; g < G && idle < 0; ++g)
      if (S->gpus[g].n_running == 0) idle = g;
    if (idle < 0) return none;
    double deadline = req_deadline(S, m, S->q_store[S->q_head[m]]);
    int lo = 1, hi = kmax, best = 0;
    while (lo <= hi) {
      int mid = (lo + hi) / 2;
      if (now + MTAB(total, m, mid) <= deadline) best = mid, lo = mid + 1;
      else hi = mid - 1;
    }
    return best ? isolated_plan(S, m, idle, best, now) : none;
  }
  /* static / reactive: min (len(running), gpu_id) over the open GPUs; size = everything buffered */
  int prio = S->A->models.prio[m];
  int bound = prio == 1 ? S->lp_allowance : S->cfg->reactive_hp_bound;
  int cap = S->cfg->static_cap < S->cfg->concurrency_limit ? S->cfg->static_cap : S->cfg->concurrency_limit;
  int best = -1;
  for (int g = 0; g < G; ++g) {
    const Gpu *gp = &S->gpus[g];
    int open;
    if (pol == STRAIT_POLICY_STATIC) open = gp->n_running < cap;
    else {
      int count = 0;
      for (int j = 0; j < gp->n_running; ++j) count += S->ent[gp->running[j]].prio == prio;
      open = gp->n_running < S->cfg->concurrency_limit && count < bound;
    }
    if (open && (best < 0 || gp->n_running < S->gpus[best].n_running)) best = g;
  }
  return best < 0 ? none : isolated_plan(S, m, best, kmax, now);
}

static Plan propose(Sim *S, int m, double now) { /* scheduler.py:257-285 */
  if (S->cfg->policy != STRAIT_POLICY_PREDICTIVE) return propose_baseline(S, m, now);
  double front = req_arr(S, S->q_store[S->q_head[m]]);
  int64_t len = q_len(S, m);
  int kmax = (int)(len < S->A->models.max_batch[m] ? len : S->A->models.max_batch[m]);
  Plan cache[65];
  int have[65];
  memset(have, 0, sizeof have);
  int lo = 1, hi = kmax, bestk = 0;
  while (lo <= hi) {
    int mid = (lo + hi) / 2;
    if (!have[mid]) cache[mid] = best_for(S, m, mid, front, now), have[mid] = 1;
    if (cache[mid].ok) bestk = mid, lo = mid + 1;
    else hi = mid - 1;
  }
  Plan p = {0, -1, 0, 0};
  if (bestk) {
    if (!have[bestk]) cache[bestk] = best_for(S, m, bestk, front, now);
    p = cache[bestk];
    p.gpu = p.ok ? p.gpu : -1;
    p.ok = bestk; /* reuse ok as the chosen size */
  }
  return p;
}

static void submit(Sim *S, int m, int k, const Plan *plan, double now, int64_t pass_id) {
  const StraitReplayArgs *A = S->A;
  int64_t bid = S->batch_seq++;
  int64_t h = S->q_head[m];
  S->q_head[m] += k; /* pop_front(k) */
  S->front_gen[m]++;
  Entry *e = &S->ent[bid];
  memset(e, 0, sizeof *e);
  e->model = m, e->size = k, e->prio = A->models.prio[m], e->gpu = plan->gpu, e->req0 = h;
  Gpu *g = &S->gpus[plan->gpu];
  double d = MTAB(transfer, m, k);
  if (d <= 0) set_err(S, STRAIT_EINVAL);
  double start = py_max(now, g->t_avail), end = start + d; /* pcie.py:25-34 */
  g->t_avail = end;
  g->pending[(g->p_head + g->p_n++) % 64] = end;
  int64_t first = S->q_store[h];
  e->deadline_abs = req_deadline(S, m, first);
  e->intf_predicted = plan->intf;
  e->kernel_start_estimate = end;
  e->live = 1;
  if (g->n_running >= S->cfg->concurrency_limit) set_err(S, STRAIT_ERUNTIME);
  g->running[g->n_running++] = (int)bid;
  recompute_aggregate(S, g);
  stamp_all(S, g, now);
  double noise = 1.0;
  if (S->cfg->has_noise) noise = A->noise[S->base + bid];
  e->remaining = MTAB(kernel, m, k), e->noise = noise, e->slowdown = 1.0, e->has_exec = 1;
  push(S, end, EV_TC, bid, 0);
  recompute(S, plan->gpu, now);
  int64_t o = S->base + bid;
  A->dec_time[o] = now, A->dec_pass[o] = (int32_t)pass_id, A->dec_model[o] = (int16_t)m;
  A->dec_size[o] = (int8_t)k, A->dec_gpu[o] = (int16_t)plan->gpu;
  A->dec_est_latency[o] = plan->lat, A->dec_intf[o] = plan->intf;
  A->b_front[o] = req_arr(S, first), A->b_transfer_start[o] = start, A->b_transfer_end[o] = end;
  S->cnt[STRAIT_RC_BATCHES]++;
}

static void ensure_timeout(Sim *S, int m, double now) { /* simulation.py:231-238 */
  if (!q_len(S, m)) return;
  if (S->timeout_gen[m] == S->front_gen[m]) return;
  double t = py_max(now, req_arr(S, S->q_store[S->q_head[m]]) + S->A->models.timeout[m]);
  push(S, t, EV_TO, m, S->front_gen[m]);
  S->timeout_gen[m] = S->front_gen[m];
}

static void do_pass(Sim *S, double now) { /* simulation.py:301-361 + scheduler.py:355-378 */
  int64_t pass_id = ++S->pass_seq;
  S->cnt[STRAIT_RC_PASSES]++;
  if (S->cfg->policy == STRAIT_POLICY_REACTIVE) reactive_catch_up(S, now); /* begin_pass */
  int order[256], n = 0;
  for (int m = 0; m < S->M; ++m)
    if (q_len(S, m)) order[n++] = m;
  /* stable insertion sort by (priority, front arrival, model_id) (scheduler.py:249-255) */
  for (int i = 1; i < n; ++i) {
    int x = order[i], j = i - 1;
    double fx = req_arr(S, S->q_store[S->q_head[x]]);
    int px = S->cfg->use_priority_order ? S->A->models.prio[x] : 0;
    while (j >= 0) {
      int y = order[j];
      double fy = req_arr(S, S->q_store[S->q_head[y]]);
      int py = S->cfg->use_priority_order ? S->A->models.prio[y] : 0;
      int less = px != py ? px < py : (fx != fy ? fx < fy : x < y);
      if (!less) break;
      order[j + 1] = y;
      j--;
    }
    order[j + 1] = x;
  }
  for (int i = 0; i < n; ++i) {
    int m = order[i];
    early_drop(S, m, now);
    int64_t len = q_len(S, m);
    if (!len) continue;
    double front = req_arr(S, S->q_store[S->q_head[m]]);
    int eligible = len >= S->A->models.max_batch[m] || now >= front + S->A->models.timeout[m];
    if (!eligible) continue;
    Plan p = propose(S, m, now);
    if (!p.ok) continue;
    int k = p.ok;
    submit(S, m, k, &p, now, pass_id);
  }
  for (int m = 0; m < S->M; ++m) ensure_timeout(S, m, now);
}

/* ---------------------------------------------------------------- handlers */
static void on_arrival(Sim *S, int64_t gi, double now) {
  int m = S->A->arr_model[gi];
  S->q_tail[m]++; /* queue.push: the next request of model m in k order */
  if (S->q_store[S->q_tail[m] - 1] != gi) set_err(S, STRAIT_EINVAL);
  if (q_len(S, m) == 1) S->front_gen[m]++;
  if (q_len(S, m) == S->A->models.max_batch[m]) do_pass(S, now);
  ensure_timeout(S, m, now);
}

static void on_timeout(Sim *S, int m, int64_t gen, double now) {
  if (q_len(S, m) && gen == S->front_gen[m]) do_pass(S, now);
}

static void on_transfer_complete(Sim *S, int64_t bid, double now) {
  Entry *e = &S->ent[bid];
  Gpu *g = &S->gpus[e->gpu];
  if (!g->p_n) set_err(S, STRAIT_EINVAL); /* pcie.calibrate (pcie.py:36-53) */
  double predicted = g->pending[g->p_head];
  g->p_head = (g->p_head + 1) % 64, g->p_n--;
  if (!g->p_n) g->t_avail = now;
  else {
    double off = now - predicted;
    if (off != 0.0) {
      g->t_avail += off;
      for (int i = 0; i < g->p_n; ++i) g->pending[(g->p_head + i) % 64] += off;
    }
  }
  e->kernel_start = now, e->kernel_started = 1, e->kernel_start_estimate = now;
  tl_clear(&e->tl);
  double v[MAXM];
  aggregate_excluding(S, g, e, v);
  tl_record(&e->tl, S->nm, now, v);
  e->slowdown = gt_slowdown(S, g, e);
  e->last_update = now;
  push(S, ex_eta(e), EV_KC, bid, e->version);
  S->A->b_kernel_start[S->base + bid] = now;
}

static void on_kernel_complete(Sim *S, int64_t bid, int64_t version, double now) {
  Entry *e = &S->ent[bid];
  if (!e->live || !e->has_exec || version != e->version) return; /* stale */
  const StraitReplayArgs *A = S->A;
  Gpu *g = &S->gpus[e->gpu];
  ex_consume(S, e, now);
  double measured = now - e->kernel_start;
  int m = e->model, k = e->size;
  double completion = now + (MTAB(total, m, k) - MTAB(transfer, m, k) - MTAB(kernel, m, k));
  int any_violated = 0;
  for (int i = 0; i < k; ++i) {
    int64_t gi = S->q_store[e->req0 + i];
    int viol = completion > req_deadline(S, m, gi);
    A->req_status[gi] = 1, A->req_violated[gi] = (uint8_t)viol, A->req_completion[gi] = completion;
    A->req_batch[gi] = (int32_t)bid;
    S->resolved++;
    if (viol) {
      any_violated = 1;
      S->cnt[e->prio == 0 ? STRAIT_RC_HP_VIOL : STRAIT_RC_LP_VIOL]++;
    }
  }
  /* complete_batch (scheduler.py:327-352) */
  double twa[MAXM];
  tl_twa(&e->tl, S->nm, now, twa);
  double tk = MTAB(kernel, m, k);
  double actual = measured / tk;
  if (!(actual > 0)) set_err(S, STRAIT_EINVAL);
  int j = 0;
  while (j < g->n_running && g->running[j] != bid) j++;
  if (j == g->n_running) set_err(S, STRAIT_ERUNTIME);
  for (; j + 1 < g->n_running; ++j) g->running[j] = g->running[j + 1];
  g->n_running--;
  recompute_aggregate(S, g);
  stamp_all(S, g, now);
  double pred, res;
  int skipped, sat;
  pred_update(S, twa, MTAB(self_cmp, m, k), MTAB(self_mem, m, k), e->prio, actual, &pred, &res, &skipped, &sat);
  int64_t o = S->base + bid;
  A->fb_predicted[o] = pred, A->fb_actual[o] = actual, A->fb_residual[o] = res;
  A->fb_flags[o] = (uint8_t)((skipped ? 1 : 0) | (sat ? 2 : 0));
  A->b_kernel_end[o] = now, A->b_completion[o] = completion, A->b_work[o] = e->work;
  A->b_done_order[o] = (int32_t)S->done_order++;
  S->cnt[STRAIT_RC_COMPLETED]++;
  e->live = 0;
  recompute(S, e->gpu, now);
  if (e->prio == 0 && any_violated) signal_hp_violation(S, e->gpu, now);
  do_pass(S, now);
}

static void on_tick(Sim *S, double now) {
  for (int gi = 0; gi < S->cfg->n_gpus; ++gi) { /* AimdState.advance (runtime.py:26-34) */
    Gpu *g = &S->gpus[gi];
    double old = g->cap_pct;
    if (now < g->last_tick) set_err(S, STRAIT_EINVAL);
    double whole = floor((now - g->last_tick) / S->cfg->aimd_interval);
    if (whole > 0) {
      g->cap_pct = py_min(S->cfg->aimd_ceiling, g->cap_pct + whole * S->cfg->aimd_increase);
      g->last_tick += whole * S->cfg->aimd_interval;
    }
    if (g->cap_pct != old) cap_row(S, now, gi);
  }
  do_pass(S, now);
  if (S->resolved < S->N) push(S, now + S->cfg->aimd_interval, EV_TICK, 0, 0);
}

static int run_one(const StraitReplayArgs *A, int64_t r) {
  Sim S_, *S = &S_;
  memset(S, 0, sizeof *S);
  S->A = A, S->cfg = &A->cfg[r], S->r = r;
  S->base = A->req_off[r], S->N = A->req_off[r + 1] - S->base;
  S->nm = A->models.n_metrics, S->M = A->models.n_models, S->B = A->models.stride, S->np = S->nm + 7;
  S->cnt = A->counters + r * STRAIT_RC_N;
  memset(S->cnt, 0, STRAIT_RC_N * sizeof(int64_t));
  const double *st = A->pred_state + r * 3 * S->np;
  memcpy(S->P, st, S->np * sizeof(double));
  memcpy(S->Mv, st + S->np, S->np * sizeof(double));
  memcpy(S->Vv, st + 2 * S->np, S->np * sizeof(double));
  S->step = A->pred_step[r];
  S->lp_allowance = S->cfg->reactive_default;
  S->last_reset = 0.0;
  int G = S->cfg->n_gpus;
  S->gpus = calloc(G, sizeof(Gpu));
  for (int g = 0; g < G; ++g) S->gpus[g].cap_pct = S->cfg->aimd_floor;
  S->ent = calloc(S->N > 0 ? S->N : 1, sizeof(Entry));
  int M = S->M;
  S->q_store = malloc((S->N > 0 ? S->N : 1) * sizeof(int64_t));
  S->q_head = calloc(M, 8), S->q_tail = calloc(M, 8), S->q_beg = calloc(M, 8);
  S->front_gen = calloc(M, 8), S->timeout_gen = malloc(M * 8);
  int64_t pos = 0;
  for (int m = 0; m < M; ++m) {
    int64_t b = A->mr_off[r * M + m], e = A->mr_off[r * M + m + 1];
    S->q_head[m] = S->q_tail[m] = S->q_beg[m] = pos;
    for (int64_t i = b; i < e; ++i) S->q_store[pos++] = A->model_req[i];
    S->timeout_gen[m] = -1;
  }
  for (int64_t i = 0; i < S->N; ++i) {
    int m = A->arr_model[S->base + i];
    A->req_status[S->base + i] = 0;
    S->cnt[A->models.prio[m] == 0 ? STRAIT_RC_HP_ARR : STRAIT_RC_LP_ARR]++;
  }
  /* arrivals pushed model-sorted in k order (simulation.py:184-194) */
  for (int m = 0; m < M; ++m)
    for (int64_t i = A->mr_off[r * M + m]; i < A->mr_off[r * M + m + 1]; ++i)
      push(S, A->arr_time[A->model_req[i]], EV_ARR, A->model_req[i], 0);
  for (int g = 0; g < G; ++g) cap_row(S, 0.0, g);
  if (S->N) push(S, S->cfg->aimd_interval, EV_TICK, 0, 0);
  while (S->heap.n && !S->err) {
    Ev e = heap_pop(&S->heap);
    switch (e.kind) {
      case EV_KC: on_kernel_complete(S, e.a, e.b, e.time); break;
      case EV_TC: on_transfer_complete(S, e.a, e.time); break;
      case EV_ARR: on_arrival(S, e.a, e.time); break;
      case EV_TO: on_timeout(S, (int)e.a, e.b, e.time); break;
      default: on_tick(S, e.time); break;
    }
    S->cnt[STRAIT_RC_EVENTS]++;
  }
  if (!S->err && S->resolved != S->N) S->err = STRAIT_EORDER;
  S->cnt[STRAIT_RC_ERROR] = S->err;
  S->cnt[STRAIT_RC_RESOLVED] = S->resolved;
  double *so = A->pred_state + r * 3 * S->np;
  memcpy(so, S->P, S->np * sizeof(double));
  memcpy(so + S->np, S->Mv, S->np * sizeof(double));
  memcpy(so + 2 * S->np, S->Vv, S->np * sizeof(double));
  A->pred_step[r] = S->step;
  for (int64_t i = 0; i < S->N; ++i) free(S->ent[i].tl.t), free(S->ent[i].tl.v);
  free(S->ent), free(S->gpus), free(S->q_store), free(S->q_head), free(S->q_tail), free(S->q_beg);
  free(S->front_gen), free(S->timeout_gen), free(S->heap.v);
  return S->err;
}

int oracle_replay(const StraitReplayArgs *A, int n_threads) {
  int err = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads > 0 ? n_threads : 1) reduction(| : err)
  for (int64_t r = 0; r < A->n_replays; ++r) err |= run_one(A, r);
  return err;
}
