/*
 * strait_oracle.c — CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference `infersim` hot path
 * (/root/reference/pkg/src/infersim), used only by tests/, by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
 * --impl reference leg.  The product path (paper_2604_28175_b200) never links
 * or calls this file.
 *
 * Every function mirrors the reference's arithmetic in its exact
 * left-to-right order with glibc libm (exp/log/pow/sqrt are the same calls
 * CPython's math module and float.__pow__ make), compiled with
 * -ffp-contract=off, so results are bit-identical to the reference on the
 * same inputs.  This is pinned by tests/test_oracle.py against golden vectors
 * produced by importing the reference itself (tests/golden/gen_golden.py).
 *
 * Python semantics mirrored exactly:
 *  - builtin max(a, b) returns b iff b > a, else a; min(a, b) returns b iff
 *    b < a (first-wins, NaN-propagating as in CPython) — see py_max/py_min.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/strait.h"

#define LOG_SATURATE 500.0 /* predictor.py:27 */

static inline double py_max(double a, double b) { return (b > a) ? b : a; }
static inline double py_min(double a, double b) { return (b < a) ? b : a; }

/* predictor.py:161-176 pressure_exponent: self terms first, then metrics */
static double pressure_exponent(const double *P, int nm, const double *coloc, int64_t stride,
                                double cmp, double mem) {
  double x = P[3 + nm] * cmp + P[4 + nm] * mem;
  for (int i = 0; i < nm; ++i) x += P[3 + i] * coloc[(int64_t)i * stride];
  return x;
}

/* predictor.py:179-185 _raw_effect -> (inner, saturated) */
static double raw_effect(const double *P, double cap, double x, int *saturated) {
  double z = x * log(P[1]);
  if (z > LOG_SATURATE) {
    *saturated = 1;
    return INFINITY;
  }
  double inner = P[0] * exp(z) + P[2];
  *saturated = inner >= cap;
  return inner;
}

/* predictor.py:188-195 kernel_effect */
static double kernel_effect(const double *P, double cap, double x, int *saturated) {
  double inner = raw_effect(P, cap, x, saturated);
  if (*saturated) return cap;
  return py_min(py_max(inner, 0.0), cap);
}

/* predictor.py:95-96 coeff_index; 198-200 interference_degree */
static inline double coeff(const double *P, int nm, int prio) { return P[nm + (prio == 0 ? 5 : 6)]; }

/* predictor.py:208-216 predict_interference */
static double predict(const double *P, int nm, double cap, const double *coloc, int64_t stride,
                      double cmp, double mem, int prio, int *saturated) {
  double x = pressure_exponent(P, nm, coloc, stride, cmp, mem);
  double eff = kernel_effect(P, cap, x, saturated);
  return 1.0 + eff * coeff(P, nm, prio);
}

int oracle_predict(const double *P, int32_t nm, double cap, const double *coloc,
                   const double *self_cmp, const double *self_mem, const int8_t *prio, int64_t n,
                   double *out, uint8_t *sat) {
  for (int64_t i = 0; i < n; ++i) {
    int s = 0;
    out[i] = predict(P, nm, cap, coloc + i, n, self_cmp[i], self_mem[i], prio[i], &s);
    if (sat) sat[i] = (uint8_t)s;
  }
  return 0;
}

/* predictor.py:219-242 estimate_latency (== scheduler.py:93-115 _latency_parts) */
int oracle_estimate_latency(const double *P, int32_t nm, double cap, const double *assumed,
                            const double *self_cmp, const double *self_mem, const int8_t *prio,
                            const double *total, const double *kernel, const double *t_avail,
                            const double *front, const double *now, int64_t n, double *out_lat,
                            double *out_intf) {
  for (int64_t i = 0; i < n; ++i) {
    int s = 0;
    double intf = predict(P, nm, cap, assumed + i, n, self_cmp[i], self_mem[i], prio[i], &s);
    double wait = py_max(0.0, t_avail[i] - now[i]); /* pcie.py:21-23 */
    double delay = (intf - 1.0) * kernel[i];        /* predictor.py:203-205 */
    out_lat[i] = total[i] + wait + delay + (now[i] - front[i]);
    if (out_intf) out_intf[i] = intf;
  }
  return 0;
}

/*
 * scheduler.py:118-161 check_violate, 164-185 check_meet, 263-280 best_for,
 * evaluated on the SoA snapshot of StraitSweepArgs (host pointers here).
 */
static void sweep_segment(const StraitSweepArgs *a, int64_t s) {
  const int nm = a->n_metrics, C = a->n_slots, G = a->gpus_per_segment;
  const int64_t S = a->n_segments, Pn = S * G, Tn = Pn * C;
  const double *P = a->params;
  const double now = a->now, cap = a->effect_cap;
  const int cprio = a->cand_prio[s];
  double add[STRAIT_MAX_METRICS];
  for (int m = 0; m < nm; ++m) add[m] = a->cand_contrib[(int64_t)m * S + s];
  int best_g = -1;
  double best_lat = NAN, best_intf = NAN;
  for (int g = 0; g < G; ++g) {
    int64_t p = s * G + g;
    int nrun = a->gpu_n_running[p];
    uint8_t flags = 0;
    double lat = NAN, intf = NAN;
    if (nrun < a->concurrency_limit) { /* runtime.py:101-102 has_slot */
      flags |= STRAIT_PAIR_HAS_SLOT;
      int violate = 0;
      if (cprio == 1) { /* LOW candidate: AIMD cap, scheduler.py:130-135 */
        double capf = a->gpu_cap_pct[p] / 100.0; /* runtime.py:39-40 */
        for (int m = 0; m < nm; ++m)
          if (a->gpu_lp_agg[(int64_t)m * Pn + p] + add[m] > capf) violate = 1;
      }
      for (int c = 0; c < nrun && !violate; ++c) {
        int64_t t = p * C + c;
        int eprio = a->ent_prio[t];
        if (eprio > cprio) continue; /* lower priority: may be sacrificed */
        double nagg[STRAIT_MAX_METRICS], twa[STRAIT_MAX_METRICS];
        for (int m = 0; m < nm; ++m) {
          nagg[m] = a->gpu_agg[(int64_t)m * Pn + p] - a->ent_contrib[(int64_t)m * Tn + t] + add[m];
          twa[m] = a->ent_twa[(int64_t)m * Tn + t];
        }
        int sat;
        double intf_new = predict(P, nm, cap, nagg, 1, a->ent_self_cmp[t], a->ent_self_mem[t], eprio, &sat);
        double ks = a->ent_kstart[t];
        double intf_cur = predict(P, nm, cap, twa, 1, a->ent_self_cmp[t], a->ent_self_mem[t], eprio, &sat);
        double tk = a->ent_t_kernel[t];
        double elapsed = py_max(0.0, now - ks);
        double denom = intf_cur * tk;
        double progress = denom > 0 ? py_min(1.0, elapsed / denom) : 1.0;
        double remaining = (1.0 - progress) * tk * intf_new;
        double projected = py_max(now, ks) + remaining;
        if (projected > a->ent_deadline_abs[t]) violate = 1;
      }
      if (violate) flags |= STRAIT_PAIR_VIOLATE;
      /* check_meet: assumed = 0.5 * agg */
      double assumed[STRAIT_MAX_METRICS];
      for (int m = 0; m < nm; ++m) assumed[m] = 0.5 * a->gpu_agg[(int64_t)m * Pn + p];
      int sat;
      intf = predict(P, nm, cap, assumed, 1, a->cand_self_cmp[s], a->cand_self_mem[s], cprio, &sat);
      lat = a->cand_total[s] + py_max(0.0, a->gpu_t_avail[p] - now) + (intf - 1.0) * a->cand_kernel[s] +
            (now - a->cand_front[s]);
      int ok = lat <= a->cand_deadline[s];
      if (ok) flags |= STRAIT_PAIR_MEET;
      int admitted = !(a->use_violate && violate) && !(a->use_meet && !ok);
      if (admitted) {
        flags |= STRAIT_PAIR_FEASIBLE;
        /* (latency, gpu_id) < (best.est_latency, best.gpu_id), scheduler.py:277 */
        if (best_g < 0 || lat < best_lat || (!(best_lat < lat) && lat == best_lat && g < best_g)) {
          best_g = g;
          best_lat = lat;
          best_intf = intf;
        }
      }
    }
    if (a->pair_flags) a->pair_flags[p] = flags;
    if (a->pair_latency) a->pair_latency[p] = lat;
    if (a->pair_intf) a->pair_intf[p] = intf;
  }
  a->seg_gpu[s] = best_g;
  a->seg_latency[s] = best_lat;
  a->seg_intf[s] = best_intf;
}

int oracle_sweep(const StraitSweepArgs *a, int n_threads, int64_t seg_begin, int64_t seg_end) {
  if (seg_end < 0) seg_end = a->n_segments;
#pragma omp parallel for schedule(static) num_threads(n_threads > 0 ? n_threads : 1)
  for (int64_t s = seg_begin; s < seg_end; ++s) sweep_segment(a, s);
  return 0;
}

/*
 * predictor.py:271-300 _prediction_gradient, 303-309 loss_gradient,
 * 155-158 huber_grad, 124-145 adam_step, 345-363 update, 98-102 enforce_floors.
 * bc1/bc2 are recomputed with pow exactly as the reference does (b1**t).
 */
int oracle_refit(const StraitRefitArgs *a) {
  const int nm = a->n_metrics, np = nm + 7;
  double *P = a->state, *M = a->state + np, *V = a->state + 2 * np;
  const double cap = a->effect_cap, delta = a->huber_delta;
  for (int64_t i = 0; i < a->n; ++i) {
    const double cmp = a->self_cmp[i], mem = a->self_mem[i];
    const int prio = a->prio[i];
    double x = pressure_exponent(P, nm, a->twa + i, a->n, cmp, mem);
    int saturated = 0;
    double inner = raw_effect(P, cap, x, &saturated);
    double eff = saturated ? cap : py_min(py_max(inner, 0.0), cap);
    double cf = coeff(P, nm, prio);
    double predicted = 1.0 + eff * cf;
    double grad[STRAIT_MAX_METRICS + 7];
    for (int k = 0; k < np; ++k) grad[k] = 0.0;
    int clamp_active = saturated || inner <= 0.0 || inner >= cap;
    if (!clamp_active) {
      double pow_bx = exp(x * log(P[1]));
      double z = P[0] * pow_bx;
      double log_b = log(P[1]);
      grad[0] = pow_bx * cf;
      grad[1] = P[0] * x * exp((x - 1.0) * log_b) * cf;
      grad[2] = cf;
      for (int m = 0; m < nm; ++m) grad[3 + m] = z * log_b * a->twa[(int64_t)m * a->n + i] * cf;
      grad[3 + nm] = z * log_b * cmp * cf;
      grad[4 + nm] = z * log_b * mem * cf;
    }
    int own = nm + (prio == 0 ? 5 : 6), other = nm + (prio == 0 ? 6 : 5);
    grad[own] = eff;
    double residual = predicted - a->actual[i];
    double g = fabs(residual) <= delta ? residual : (residual > 0 ? delta : -delta);
    int finite = isfinite(residual);
    for (int k = 0; k < np; ++k) {
      grad[k] = g * grad[k];
      if (!isfinite(grad[k])) finite = 0;
    }
    if (a->out_predicted) a->out_predicted[i] = predicted;
    if (a->out_residual) a->out_residual[i] = residual;
    if (a->out_flags) a->out_flags[i] = (uint8_t)((finite ? 0 : 1) | (saturated ? 2 : 0));
    if (!finite) continue;
    int64_t t = ++(*a->step);
    double b1 = a->beta1, b2 = a->beta2;
    double bc1 = 1.0 - pow(b1, (double)t);
    double bc2 = 1.0 - pow(b2, (double)t);
    for (int k = 0; k < np; ++k) {
      if (k == other) continue;
      M[k] = b1 * M[k] + (1.0 - b1) * grad[k];
      V[k] = b2 * V[k] + (1.0 - b2) * grad[k] * grad[k];
      double m_hat = M[k] / bc1;
      double v_hat = V[k] / bc2;
      P[k] -= a->learning_rate * m_hat / (sqrt(v_hat) + a->eps);
    }
    P[0] = py_max(P[0], 1e-6);       /* MIN_SCALE */
    P[1] = py_max(P[1], 1.0 + 1e-6); /* MIN_BASE */
    P[nm + 5] = py_max(P[nm + 5], 1e-6);
    P[nm + 6] = py_max(P[nm + 6], 1e-6);
  }
  return 0;
}

/* simulation.py:309-311: the per-batch noise factor math.exp(normal(0, sigma)),
 * applied to host-drawn normals with glibc exp (the same call as math.exp). */
void oracle_exp(const double *z, double *out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = exp(z[i]);
}
