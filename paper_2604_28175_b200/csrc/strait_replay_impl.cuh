// strait_replay_impl.cuh — the device trace-replay engine (R5-R21): whole
// discrete-event replays of the Strait scheduler, the replay's entire mutable
// state resident in shared memory.  One warp per replay (replay sweeps, narrow
// nodes), or one CTA of 8 warps per replay for wide nodes: a master warp runs
// the event loop and the helper warps join its wide steps (Sim<..., NW>).
// Instantiated once per metric count in strait_replay_nm*.cu.
//
// Restates /root/reference/pkg/src/infersim/simulation.py:122-513 driving
// PredictivePolicy (scheduler.py:229-378), InterferencePredictor
// (predictor.py:161-363), PcieLinkState (pcie.py:13-53), GpuRuntimeState +
// AimdState (runtime.py:13-141), ThroughputTimeline (domain.py:217-264) and
// the hidden ground truth (oracle.py:55-77).
//
// B200 design (not the reference's structure):
//  * No event heap.  Every live event of a replay has a fixed home: each
//    running-batch slot holds at most ONE pending event (its transfer-complete
//    or its latest kernel-complete; older kernel-completes are exactly the
//    reference's stale, version-superseded events), each model queue holds its
//    latest batch timeout, plus one AIMD tick and the head of the pre-sorted
//    arrival stream.  The next event is a warp-wide lexicographic argmin over
//    these <= G*C + M + 2 candidates on the reference's (time, kind, seq) key,
//    with seq assigned in the reference's push order, so pops happen in the
//    reference's order and stale events never exist.
//  * Timelines are kept in running-integral form (t0, t_last, v_last, acc):
//    the same additions in the same order as the reference loop
//    (domain.py:249-264), O(1) memory per running batch.
//  * Lane-parallel: the pass's queue ordering (rank sort), early drop
//    (ballot over the queue prefix), best_for (lane per GPU), recompute and
//    timeline stamping (lane per running entry), the aggregate (lane per
//    metric), the refit (lane per parameter, predictor.py:345-363), cap rows
//    (ballot-ordered).  Everything else is uniform scalar code executed by all
//    lanes; shared-memory scalars are written by lane 0 followed by __syncwarp.
//  * Binary64 throughout, --fmad=false, left-to-right evaluation as the
//    reference, exp/log/pow restated from the reference host's glibc
//    (strait_libm.cuh): results are bit-identical to the reference.
//  * Specialised instantiations, because the engine is instruction-cache and
//    latency bound and every instruction removed pays.  These are MINB
//    (latency / throughput register budgets), TR (event log compiled in or
//    out), LEAN (predictive-only batches whose proposes all take the
//    all-sizes path) and GEOM (the 4 GPU x 4 slot x 6 model geometry as
//    constants, so every field offset is an immediate).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/strait_replay.h"
#include "strait_capi.cuh"

#include "strait_device.cuh"

namespace strait {
namespace rp {

// Cycle accounting of the engine's phases (diagnostic build only:
// -DSTRAIT_REPLAY_PROFILE=1, scripts/replay_profile.py); compiled out otherwise.
#ifndef STRAIT_REPLAY_PROFILE
#define STRAIT_REPLAY_PROFILE 0
#endif
#if STRAIT_REPLAY_PROFILE
enum { RPF_SELECT, RPF_ARRIVAL, RPF_RANK, RPF_DROP, RPF_ELIG, RPF_PROPOSE, RPF_SUBMIT, RPF_ICUR, RPF_TIMEOUTS,
       RPF_TC, RPF_KC_PRE, RPF_KC_UPDATE, RPF_KC_POST, RPF_TICK, RPF_POST, RPF_TOTAL,
       RPF_N_QUEUES, RPF_N_ELIGIBLE, RPF_N_PROPOSE_WIDE, RPF_N_SUBMIT, RPF_N_ICUR_ALL, RPF_SUM_KMAX, RPF_N_NOSLOT,
       RPF_SUM_ENTRIES, RPF_CTA_A, RPF_CTA_B, RPF_CTA_M, RPF_N_CTA, RPF_CTA_PA, RPF_CTA_PB, RPF_CTA_J, RPF_N };
#define RP_CNT(i) (++prof[i])
extern __device__ unsigned long long g_replay_prof[RPF_N];
extern __device__ unsigned long long g_cta_warp[3][16];  // per warp: wake, phase-A end, phase-B end (- post)
#define RP_T(v) const long long v = clock64()
#define RP_ADD(i, v) (prof[i] += clock64() - (v))
#else
#define RP_T(v)
#define RP_ADD(i, v)
#define RP_CNT(i)
#endif

// Two math policies.  The latency variant (few replays, one warp each: C2,
// C4's longest replays bound the launch) inlines everything.  The throughput
// variant (16 replays per SM) is instruction-cache bound — 16 warps at
// different points of the hot loop — so exp, log, pow and the IEEE division
// get ONE out-of-line copy each.  Both return identical bits.
static __device__ __noinline__ double rp_exp(double x) { return dexp(x); }
static __device__ __noinline__ double rp_log(double x) { return dlog(x); }
static __device__ __noinline__ double rp_pow(double x, double y) { return dpow(x, y); }
static __device__ __noinline__ double rp_div(double a, double b) { return __ddiv_rn(a, b); }

struct OutlineMath {
  static constexpr bool kInline = false;
  static __device__ __forceinline__ double exp(double x, const ulonglong2*) { return rp_exp(x); }
  static __device__ __forceinline__ double log(double x) { return rp_log(x); }
  static __device__ __forceinline__ double pow(double x, double y) { return rp_pow(x, y); }
  static __device__ __forceinline__ double div(double a, double b) { return rp_div(a, b); }
};
struct FullInlineMath : InlineMath {
  static __device__ __forceinline__ double exp(double x, const ulonglong2* tab) { return dexp(x, tab); }
  static __device__ __forceinline__ double pow(double x, double y) { return dpow(x, y); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};

constexpr int kKC = 0, kTC = 1, kARR = 2, kTO = 3, kTICK = 4;  // simulation.py:28-33 tie ranks
constexpr double kWorkEps = 1e-9;                               // simulation.py:35
constexpr unsigned long long kNoKey = ~0ULL;
#ifndef STRAIT_CTA_PROBE_ITEMS
#define STRAIT_CTA_PROBE_ITEMS 2  // CTA propose: probe-by-probe jobs above this many items per thread
#endif
constexpr int kMaxConc = 32;  // lane-per-list-position steps (recompute, restamp, intf_cur of a GPU)
constexpr int kMaxModels = 64;
constexpr int kMaxBatch = 64;
constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ __forceinline__ size_t al(size_t x) { return (x + 15) & ~(size_t)15; }

// Shared-memory layout of one replay (one warp), grouped field arrays so the
// engine needs only a handful of base pointers.  Slot s = g * C + j is
// running-batch slot j of GPU g (G, C = the launch's maximum geometry);
// per-GPU fields are [field][G] so lanes over GPUs touch consecutive words.
// Slot double fields (SD_*), then four NM-vectors: timeline value, timeline
// integral, the entry's contribution and aggregate_excluding(entry):
// SD_X0 / SD_RB / SD_ST: the k-independent parts of a co-runner's projection,
// refreshed with intf_cur (icur_slot)
enum { SD_DL, SD_KS, SD_T0, SD_TL, SD_REM, SD_SLOW, SD_NOISE, SD_LAST, SD_WORK, SD_RB, SD_X0, SD_ST, SD_CMP, SD_MEM,
       SD_TK, SD_VL };
enum { SI_BID, SI_REQ0, SI_GPU, SI_J, SI_N };  // SI_GPU / SI_J: s / C and s % C, precomputed
enum { SB_MODEL, SB_SIZE, SB_PRIO, SB_STARTED, SB_LIVE, SB_TLEN, SB_N };
// GD_CAPF = cap_fraction() = cap_pct / 100 (runtime.py:39-40), refreshed wherever the cap changes
enum { GD_TAV, GD_CAP, GD_TICK, GD_CAPF, GD_AGG };  // then NM aggregates, NM LP aggregates, C pending reservations
enum { GI_NRUN, GI_PHEAD, GI_PN, GI_N };
enum { QI_HEAD, QI_TAIL, QI_FGEN, QI_TGEN, QI_EGEN, QI_ORD, QI_N };

// Job block of a CTA-per-replay launch (NW > 1 warps per replay, below): the
// master warp posts one of these, the helper warps read it after barrier 1.
enum { JOB_EXIT, JOB_ICUR, JOB_PROPOSE };
struct Job {
  int kind, m, kmax, cprio, k0, pad;
  double now, dl, front;
  long long t0;  // profiling build: the master's clock at the post
};
// one warp's partial of a reduction: a size's best GPU over a chunk of 32 GPUs
struct Part {
  double t, x;  // latency, interference of the chunk's best GPU
  int g, pad;   // its gpu_id, -1 if none feasible
};

struct Layout {
  int G, C, M, NM, S, NE;
  size_t P, sd, gd, ed, ek, qd, qf, sl, si, gi, qi, sb, go, qb, bytes;
  // CTA-per-replay scratch (nw > 1 only): job, per-(size, GPU, co-runner) violate
  // bits, per-(size, GPU) meet results, per-warp reduction partials
  size_t jb, pv, plat, pintf, pm, part;
  __host__ __device__ static int sd_fields(int nm) { return SD_VL + 4 * nm; }
  __host__ __device__ static int gd_fields(int nm, int c) { return GD_AGG + 2 * nm + c; }
  // items of the CTA propose: sizes (<= 32) x GPUs x (co-runner slots + the meet)
  __host__ __device__ static int cta_sizes(int b) { return b < 32 ? b : 32; }
  __host__ __device__ static int cta_chunks(int g) { return g <= 32 ? 1 : (g + 31) / 32; }
  __host__ __device__ Layout(int g, int c, int m, int nm, int nw = 1, int b = 0) : G(g), C(c), M(m), NM(nm) {
    S = G * C;
    NE = S + M + 2;
    size_t o = 0;
    auto take = [&](size_t n) {
      size_t r = o;
      o = al(o + n);
      return r;
    };
    P = take(8 * (NM + 8));  // params, then log(base) for the helper warps
    sd = take(8 * (size_t)sd_fields(NM) * S);
    gd = take(8 * (size_t)gd_fields(NM, C) * G);
    ed = take(8 * (size_t)NE);
    ek = take(8 * (size_t)NE);
    qd = take(8 * (size_t)M);
    qf = take(8 * (size_t)M);
    sl = take(4 * (size_t)S);  // scratch slot list (icur_all)
    si = take(4 * (size_t)SI_N * S);
    gi = take(4 * (size_t)GI_N * G);
    qi = take(4 * (size_t)QI_N * M);
    sb = take((size_t)SB_N * S);
    go = take((size_t)C * G);
    qb = take((size_t)M);
    jb = pv = plat = pintf = pm = part = 0;
    if (nw > 1) {
      const size_t kg = (size_t)cta_sizes(b) * G;
      jb = take(sizeof(Job));
      pv = take(kg * (C + 1));
      plat = take(8 * kg);
      pintf = take(8 * kg);
      pm = take(kg);
      const size_t np = (size_t)cta_sizes(b) * cta_chunks(G);
      part = take(sizeof(Part) * np);
    }
    bytes = o;
  }
};

// Replay geometry: launch-wide layout strides (max GPUs G, max concurrency C,
// models M; S = G*C slots, NE = S + M + 2 event homes) and this replay's
// n_gpus / concurrency_limit.  GEOM 0 keeps them at run time; GEOM 1 is the
// overload.yaml / BASELINE C2 / C4 geometry (4 GPUs x 4 slots, 6 models, every
// replay at the maxima) as compile-time constants, so every shared-memory
// field offset folds into an immediate (a ~20 % smaller, faster kernel).
template <int GEOM>
struct Geom {
  int G, C, M, S, NE, NG, CONC, B;  // B: profile-table stride (max batch size)
  __device__ __forceinline__ bool set_geom(const Layout& L, const StraitReplayConfig* cf, int stride) {
    G = L.G, C = L.C, M = L.M, S = L.S, NE = L.NE, NG = cf->n_gpus, CONC = cf->concurrency_limit, B = stride;
    return true;
  }
};
template <>
struct Geom<1> {
  static constexpr int G = 4, C = 4, M = 6, S = 16, NE = 24, NG = 4, CONC = 4;
  int B;
  __device__ __forceinline__ bool set_geom(const Layout& L, const StraitReplayConfig* cf, int stride) {
    B = stride;
    return L.G == G && L.C == C && L.M == M && cf->n_gpus == NG && cf->concurrency_limit == CONC;
  }
};
// GEOM 2: GEOM 1 with the table stride (max batch 8) fixed too.  The latency
// kernel gains (+2-3 %); the 128-register throughput kernel allocates worse
// with it (-9 %), so that one keeps GEOM 1.
template <>
struct Geom<2> {
  static constexpr int G = 4, C = 4, M = 6, S = 16, NE = 24, NG = 4, CONC = 4, B = 8;
  __device__ __forceinline__ bool set_geom(const Layout& L, const StraitReplayConfig* cf, int stride) const {
    return L.G == G && L.C == C && L.M == M && cf->n_gpus == NG && cf->concurrency_limit == CONC && stride == B;
  }
};

// GEOM 3: the BASELINE C5 geometry (64 GPUs x 4 slots, 20 models), every replay
// at the maxima.
template <>
struct Geom<3> {
  static constexpr int G = 64, C = 4, M = 20, S = 256, NE = 278, NG = 64, CONC = 4;
  int B;
  __device__ __forceinline__ bool set_geom(const Layout& L, const StraitReplayConfig* cf, int stride) {
    B = stride;
    return L.G == G && L.C == C && L.M == M && cf->n_gpus == NG && cf->concurrency_limit == CONC;
  }
};

// NW = warps per replay.  NW = 1: one warp runs the whole replay.  NW > 1 (one
// replay per CTA, for single replays and few-replay launches): warp 0 (the
// master) runs the event loop exactly as with NW = 1; at the wide steps —
// intf_cur of every running entry and a propose's (size, GPU, co-runner)
// projections and meets — it posts a Job and
// the NW - 1 helper warps, parked on named barrier 1, join it.  Every job reads
// the replay state and writes only per-item scratch (or per-slot caches that
// no other item touches); barrier 2 ends it.  Same arithmetic, same bits.
// ILP: eval_pair evaluates check_meet and the co-runner projections two exp
// chains at a time (Pred::effect2) — the lower latency for single replays; a
// launch with several replays per SM keeps the smaller one-chain code, which
// the instruction cache rewards there, and so do the generic CTA-layout
// kernels, whose proposes run as jobs (eval_pair only for batches past 32
// sizes) and whose 256 threads leave at most 255 registers (the C5-geometry
// CTA kernel measured faster with it, spills included).
template <int NM, typename MathT, bool TR, bool LEAN, int GEOM, int NW = 1, bool ILP = true>
struct Sim : Geom<GEOM> {
  using Geom<GEOM>::G;
  using Geom<GEOM>::C;
  using Geom<GEOM>::M;
  using Geom<GEOM>::S;
  using Geom<GEOM>::NE;
  using Geom<GEOM>::NG;
  using Geom<GEOM>::CONC;
  using Geom<GEOM>::B;
  static constexpr int NP = NM + 7;
  static constexpr int SD_ACC = SD_VL + NM;   // timeline integral
  static constexpr int SD_CON = SD_VL + 2 * NM;  // entry.contribution (throughput_at(size))
  static constexpr int SD_AEX = SD_VL + 3 * NM;  // aggregate_excluding(entry) as last stamped
  static constexpr int GD_LPA = GD_AGG + NM;     // low_priority_aggregate()
  static constexpr int GD_PEND = GD_AGG + 2 * NM;
  static constexpr bool CTA = NW > 1;
  static constexpr int NT = NW * 32;
  // ---- launch-wide inputs
  const StraitReplayArgs* A;
  const StraitReplayConfig* cf;
  int lane;
  int w;  // warp of the replay's CTA (0 = master); 0 when NW = 1
  // CTA scratch (Layout::jb ...)
  Job* jb;
  uint8_t *pv, *pm;
  double *plat, *pintf;
  Part* part;
  int64_t r, base, N;     // request range [base, base + N)
  // ---- shared-memory state: grouped field arrays of this warp's slice
  double *P, *sd, *gd, *ed, *qd;
  double* qf;  // front arrival time of each non-empty queue (cache of arr(model_req[head]))
  int* slist;  // scratch list of slots
  unsigned long long* ek;
  int *si, *gi, *qi;
  int8_t *sb, *go, *qb;
  // ---- uniform scalar state (identical in every lane)
  Pred<NM, MathT> pr;
  double adam_m, adam_v;  // lane-owned Adam moments (lane k owns parameter k)
  int64_t step;
  unsigned long long seq;
  int batch_seq, pass_seq, done_order, err;
  int lp_allowance;   // ReactiveState (baselines.py:81-110)
  double last_reset;
  int64_t next_arr, resolved;
  double my_dl, my_floor, my_to;  // lane m < 32: model m's deadline, total(1), batch timeout
  int my_maxb;                    // and max batch size
  int64_t pf_q, pf_g;  // the last arrival's queue-order check, settled at the next arrival / the end
  int pf_m;            // model of the next arrival
  double pf_t2;        // time of the arrival after the next
  int64_t c_batches, c_completed, c_passes, c_cap_rows, c_events, c_hp_viol, c_lp_viol, c_hp_drop, c_lp_drop;
  int64_t c_trace;  // trace records produced (TR)
#if STRAIT_REPLAY_PROFILE
  mutable long long prof[RPF_N];
#endif

  // ------------------------------------------------------------ accessors
  __device__ __forceinline__ double& SD(int f, int s) const { return sd[f * S + s]; }
  __device__ __forceinline__ int& SI(int f, int s) const { return si[f * S + s]; }
  __device__ __forceinline__ int8_t& SB(int f, int s) const { return sb[f * S + s]; }
  __device__ __forceinline__ double& GD(int f, int g) const { return gd[f * G + g]; }
  __device__ __forceinline__ int& GI(int f, int g) const { return gi[f * G + g]; }
  __device__ __forceinline__ int& QI(int f, int m) const { return qi[f * M + m]; }
  __device__ __forceinline__ int8_t& ORD(int p, int g) const { return go[p * G + g]; }
  // GPU-major: a GPU's running batches are adjacent words, so lanes over one GPU's
  // list positions (recompute, restamp, intf_cur) and the CTA's (GPU, co-runner)
  // items read distinct shared-memory banks
  __device__ __forceinline__ int slot(int g, int j) const { return g * C + j; }
  __device__ __forceinline__ int slot_at(int g, int p) const { return slot(g, ORD(p, g)); }

  __device__ __forceinline__ void sync() const { __syncwarp(); }
  // named barrier over the replay's NW warps (ids 1-3; 0 is __syncthreads).  The
  // master and the helpers reach it from different code locations, so it is the
  // non-.aligned form (bar.sync is barrier.sync.aligned).
  __device__ __forceinline__ void cta_bar(int id) const {
    asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(NT) : "memory");
  }
  // master: the job fields were written by lane 0; wake the helpers.  (Measured
  // and reverted: a generation counter the parked helpers poll in shared memory
  // instead of barrier 1 — they still issue ~400 cycles after the post, and the
  // polling slows the master: C5 134 k vs 140 k req/s.)
  __device__ __forceinline__ void post_job() const {
    __syncwarp();
    cta_bar(1);
  }
  // helpers: the predictor as the master holds it (P + log(base) in shared memory)
  __device__ __forceinline__ void load_shared_pred() {
    pr.scale = P[0];
    pr.log_base = P[NP];
    pr.offset = P[2];
#pragma unroll
    for (int i = 0; i < NM; ++i) pr.w[i] = P[3 + i];
    pr.w_cmp = P[3 + NM];
    pr.w_mem = P[4 + NM];
    pr.coeff[0] = P[5 + NM];
    pr.coeff[1] = P[6 + NM];
    pr.cap = cf->effect_cap;
#if STRAIT_LIBM
    pr.etab = glibc::exp_table();
#endif
  }
  // master: (re)load the predictor from P and publish log(base) to the helpers
  __device__ __forceinline__ void load_pred() {
    pr.load(P, cf->effect_cap);
    if constexpr (CTA) {
      if (lane == 0) P[NP] = pr.log_base;
      __syncwarp();
    }
  }
  // Uniform scalar store: every lane computed v; lane 0 writes it after the warp
  // has finished its earlier reads of shared state (write-after-read).  Readers
  // of the new value come after a sync() (read-after-write).
  template <typename T>
  __device__ __forceinline__ void put(T& ref, T v) const {
    __syncwarp();
    if (lane == 0) ref = v;
  }
  __device__ __forceinline__ void fail(int code) {
    if (!err) err = code;
  }
  __device__ __forceinline__ void fail_any(bool bad, int code) {
    if (__any_sync(kFull, bad)) fail(code);
  }
  // profile tables (domain.py:52-105), size k in 1..max_batch
  __device__ __forceinline__ int64_t ti(int m, int k) const { return (int64_t)m * B + k - 1; }
  __device__ __forceinline__ double thr(int m, int k, int i) const {
    return __ldg(&A->models.throughput[(int64_t)i * M * B + ti(m, k)]);
  }
  __device__ __forceinline__ double tab_total(int m, int k) const { return __ldg(&A->models.total[ti(m, k)]); }
  __device__ __forceinline__ double tab_transfer(int m, int k) const { return __ldg(&A->models.transfer[ti(m, k)]); }
  __device__ __forceinline__ double tab_kernel(int m, int k) const { return __ldg(&A->models.kernel[ti(m, k)]); }
  __device__ __forceinline__ double tab_cmp(int m, int k) const { return __ldg(&A->models.self_cmp[ti(m, k)]); }
  __device__ __forceinline__ double tab_mem(int m, int k) const { return __ldg(&A->models.self_mem[ti(m, k)]); }
  __device__ __forceinline__ int mprio(int m) const { return __ldg(&A->models.prio[m]); }
  __device__ __forceinline__ double mdeadline(int m) const { return __ldg(&A->models.deadline[m]); }
  __device__ __forceinline__ double mtimeout(int m) const { return __ldg(&A->models.timeout[m]); }
  __device__ __forceinline__ int mmaxb(int m) const { return __ldg(&A->models.max_batch[m]); }
  __device__ __forceinline__ int64_t req_at(int pos) const { return __ldg(&A->model_req[pos]); }
  __device__ __forceinline__ double arr(int64_t gidx) const { return __ldg(&A->arr_time[gidx]); }
  // LEAN: a predictive-only batch whose proposes all fit the all-sizes-at-once
  // path (max batch x pow2ceil(max GPUs) <= 32): the baseline policies and the
  // probe-by-probe propose compile out, a smaller kernel for the instruction cache
  __device__ __forceinline__ int policy() const { return LEAN ? STRAIT_POLICY_PREDICTIVE : cf->policy; }
  __device__ __forceinline__ int q_len(int m) const { return QI(QI_TAIL, m) - QI(QI_HEAD, m); }
  __device__ __forceinline__ double front_arrival(int m) const { return qf[m]; }

  __device__ __forceinline__ void push_event(int i, double t, int kind) {  // Simulation._push (simulation.py:202-205)
    ++seq;
    put(ed[i], t);
    put(ek[i], ((unsigned long long)kind << 56) | seq);
  }
  __device__ __forceinline__ void clear_event(int i) {
    put(ed[i], __longlong_as_double(0x7ff0000000000000LL));
    put(ek[i], kNoKey);
  }

  __device__ __forceinline__ void cap_row_at(int64_t n, double t, int g, double pct) const {
    if (n < A->cap_rows_max) {
      const int64_t o = r * A->cap_rows_max + n;
      A->cap_time[o] = t;
      A->cap_gpu[o] = (int16_t)g;
      A->cap_pct[o] = pct;
    }
  }

  // Simulation._trace (simulation.py:207-218), TR only: record i of this replay's log
  __device__ __forceinline__ void trace_put(int64_t i, int ev, double t, int gpu, int bid, int64_t req, int size,
                                            double x0, double x1, double x2) const {
    if (i < A->trace_max) {
      StraitTraceRec* o = A->trace + r * (int64_t)A->trace_max + i;
      o->time = t;
      o->x[0] = x0;
      o->x[1] = x1;
      o->x[2] = x2;
      o->request = req;
      o->batch = bid;
      o->gpu = (int16_t)gpu;
      o->event = (int8_t)ev;
      o->size = (int8_t)size;
    }
  }
  // one record with uniform fields, written by lane 0
  __device__ __forceinline__ void trace1(int ev, double t, int gpu = -1, int bid = -1, int64_t req = -1, int size = 0,
                                         double x0 = 0.0, double x1 = 0.0, double x2 = 0.0) {
    if constexpr (TR) {
      if (lane == 0) trace_put(c_trace, ev, t, gpu, bid, req, size, x0, x1, x2);
      ++c_trace;
    }
  }

  // ------------------------------------------------------------ timelines (domain.py:237-264)
  // lane-local: called by the one lane that owns slot s
  __device__ __forceinline__ bool tl_record(int s, double now, const double (&v)[NM]) const {
    if (SB(SB_TLEN, s)) {
      const double last = SD(SD_TL, s);
      if (now < last) return false;  // SimulationOrderError
      if (now == last) {             // same timestamp: replace the last sample
#pragma unroll
        for (int i = 0; i < NM; ++i) SD(SD_VL + i, s) = v[i];
        return true;
      }
      const double d = now - last;  // closes segment [last, now) of the held value
#pragma unroll
      for (int i = 0; i < NM; ++i) SD(SD_ACC + i, s) = SD(SD_ACC + i, s) + SD(SD_VL + i, s) * d;
      SD(SD_TL, s) = now;
#pragma unroll
      for (int i = 0; i < NM; ++i) SD(SD_VL + i, s) = v[i];
      return true;
    }
    SB(SB_TLEN, s) = 1;
    SD(SD_T0, s) = now;
    SD(SD_TL, s) = now;
#pragma unroll
    for (int i = 0; i < NM; ++i) {
      SD(SD_VL + i, s) = v[i];
      SD(SD_ACC + i, s) = 0.0;
    }
    return true;
  }
  __device__ __forceinline__ void tl_twa(int s, double end, double (&out)[NM]) const {
    const double total = end - SD(SD_T0, s);
    if (total <= 0.0) {
#pragma unroll
      for (int i = 0; i < NM; ++i) out[i] = SD(SD_VL + i, s);
      return;
    }
    const double d = end - SD(SD_TL, s);
    if constexpr (MathT::kInline) {  // the NM quotients by one total overlap (div_shared)
      double num[NM];
#pragma unroll
      for (int i = 0; i < NM; ++i) num[i] = SD(SD_ACC + i, s) + SD(SD_VL + i, s) * d;
      div_shared(num, total, out);
    } else {
#pragma unroll
      for (int i = 0; i < NM; ++i) out[i] = MathT::div(SD(SD_ACC + i, s) + SD(SD_VL + i, s) * d, total);
    }
  }

  // ------------------------------------------------------------ runtime (runtime.py:104-141)
  // aggregate_throughput and low_priority_aggregate(): sums of contributions in
  // running-list order from 0.0 (runtime.py:104-109,116-122); lane i owns metric i
  __device__ __forceinline__ void recompute_aggregate(int g) {
    if (lane < NM) {
      double a = 0.0, lp = 0.0;
      const int n = GI(GI_NRUN, g);
#pragma unroll 1
      for (int p = 0; p < n; ++p) {
        const int s = slot_at(g, p);
        const double c = SD(SD_CON + lane, s);
        a += c;
        if (SB(SB_PRIO, s) == 1) lp += c;
      }
      GD(GD_AGG + lane, g) = a;
      GD(GD_LPA + lane, g) = lp;
    }
    sync();
  }
  // every running entry records aggregate_excluding(self) at now; lane p owns list position p
  __device__ __forceinline__ void stamp_all(int g, double now) {
    bool bad = false;
    if (lane < GI(GI_NRUN, g)) {
      const int s = slot_at(g, lane);
      double v[NM];
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        v[i] = GD(GD_AGG + i, g) - SD(SD_CON + i, s);  // aggregate_excluding (runtime.py:111-114)
        SD(SD_AEX + i, s) = v[i];
      }
      bad = !tl_record(s, now, v);
    }
    sync();
    fail_any(bad, STRAIT_EORDER);
  }

  // ------------------------------------------------------------ ground truth (oracle.py:55-77)
  __device__ __forceinline__ double gt_slowdown(int s) const {
    double x = cf->gt_w_cmp * SD(SD_CMP, s) + cf->gt_w_mem * SD(SD_MEM, s);
#pragma unroll
    for (int i = 0; i < NM; ++i) x += cf->gt_w[i] * SD(SD_AEX + i, s);
    double effect = cf->gt_family == 0 ? cf->gt_scale * MathT::pow(cf->gt_base, x) + cf->gt_offset
                                       : cf->gt_scale * x * x + cf->gt_offset;
    effect = py_max(0.0, effect);
    return 1.0 + effect * (SB(SB_PRIO, s) == 0 ? cf->gt_pf_high : cf->gt_pf_low) * SD(SD_NOISE, s);
  }

  // ExecutionState.advance (simulation.py:54-70); lane-local
  __device__ __forceinline__ bool ex_consume(int s, double now) const {
    const double d = now - SD(SD_LAST, s);
    bool ok = !(d < 0);
    if (d > 0) {
      const double slow = SD(SD_SLOW, s);
      const double q = MathT::div(d, slow);  // the reference divides twice; same value
      SD(SD_WORK, s) = SD(SD_WORK, s) + q;
      double rem = SD(SD_REM, s) - q;
      if (rem < -kWorkEps) ok = false;
      if (rem < 0.0) rem = 0.0;
      SD(SD_REM, s) = rem;
    }
    SD(SD_LAST, s) = now;
    return ok;
  }

  // Simulation._recompute (simulation.py:290-297): every STARTED entry of GPU g
  // integrates its work so far, takes the new ground-truth slowdown and
  // re-pushes its kernel-complete (fresh seq, list order).  Lane p = position p.
  __device__ __forceinline__ void recompute(int g, double now) {
    const int n = GI(GI_NRUN, g);
    int s = -1;
    bool started = false, ok = true;
    double eta = 0.0;
    double seg_d = 0.0, seg_slow = 0.0;
    if (lane < n) {
      s = slot_at(g, lane);
      started = SB(SB_STARTED, s);
      if (started) {
        seg_d = now - SD(SD_LAST, s);
        seg_slow = SD(SD_SLOW, s);
        ok = ex_consume(s, now);
        const double slow = gt_slowdown(s);
        SD(SD_SLOW, s) = slow;
        eta = SD(SD_LAST, s) + SD(SD_REM, s) * slow;
      }
    }
    const unsigned mask = __ballot_sync(kFull, started);
    if (started) {
      const unsigned long long q = seq + 1 + __popc(mask & ((1u << lane) - 1));
      ed[s] = eta;
      ek[s] = ((unsigned long long)kKC << 56) | q;
    }
    seq += __popc(mask);
    if constexpr (TR) {  // ExecutionState.segments: (d, slowdown) for every d > 0 advance
      const bool seg = started && seg_d > 0;
      const unsigned sm = __ballot_sync(kFull, seg);
      if (seg)
        trace_put(c_trace + __popc(sm & ((1u << lane) - 1)), STRAIT_TR_SEGMENT, now, g, SI(SI_BID, s), -1, 0, seg_d,
                  seg_slow, 0.0);
      c_trace += __popc(sm);
    }
    sync();
    fail_any(!ok, STRAIT_EORDER);
  }

  // ReactiveState.catch_up (baselines.py:99-104)
  __device__ __forceinline__ void reactive_catch_up(double now) {
    const double period = cf->reactive_period;
    if (now - last_reset >= period) {
      const double periods = floor(MathT::div(now - last_reset, period));
      lp_allowance = cf->reactive_default;
      last_reset += periods * period;
    }
  }

  // _signal_hp_violation (simulation.py:223-229) -> policy.on_hp_violation:
  // AimdState.reset for the predictive policy (scheduler.py:287-292), the
  // reactive allowance for ReactiveSpatialPolicy (baselines.py:131-133), a
  // no-op for the other baselines (scheduler.py:225-226).
  __device__ __forceinline__ void signal_hp(int gpu_id, double now) {
    if (policy() != STRAIT_POLICY_PREDICTIVE) {
      if (policy() == STRAIT_POLICY_REACTIVE) {
        reactive_catch_up(now);
        lp_allowance = max(cf->reactive_min, lp_allowance - 1);
      }
      return;
    }
    for (int g0 = 0; g0 < NG; g0 += 32) {
      const int g = g0 + lane;
      bool changed = false;
      double cap = 0.0;
      if (g < NG && (gpu_id < 0 || g == gpu_id)) {
        const double old = GD(GD_CAP, g);
        cap = cf->aimd_floor;
        GD(GD_CAP, g) = cap;
        GD(GD_CAPF, g) = MathT::div(cap, 100.0);
        changed = cap != old;
      }
      const unsigned mask = __ballot_sync(kFull, changed);
      if (changed) cap_row_at(c_cap_rows + __popc(mask & ((1u << lane) - 1)), now, g, cap);
      c_cap_rows += __popc(mask);
      if constexpr (TR) {  // "aimd_reset" rows, GPU order (simulation.py:226-229)
        if (changed) trace_put(c_trace + __popc(mask & ((1u << lane) - 1)), STRAIT_TR_RESET, now, g, -1, -1, 0, cap, 0.0, 0.0);
        c_trace += __popc(mask);
      }
    }
    sync();
  }

  // ------------------------------------------------------------ predictor (predictor.py)
  // InterferencePredictor.update (predictor.py:345-363) for one sample, all lanes;
  // lane k owns parameter k and its Adam moments.
  __device__ __forceinline__ void update(const double (&tw)[NM], double cmp, double mem, int prio, double actual,
                                         double& predicted, double& residual, bool& skipped, bool& saturated) {
    const bool owner = lane < NP;
    const double cap = pr.cap;
    const double x = pr.exponent(tw, cmp, mem);
    const double z = x * pr.log_base;
    double inner, pow_bx = 0.0, pow_bx1 = 0.0;  // b^x, and b^(x-1) for lane 1's gradient term
    if (z > kLogSaturate) {
      saturated = true;
      inner = __longlong_as_double(0x7ff0000000000000LL);
    } else {
      if constexpr (MathT::kInline) {  // both exps as one block, on every lane (no divergent exp)
        pr.exp2v(z, (x - 1.0) * pr.log_base, pow_bx, pow_bx1);
      } else {
        pow_bx = MathT::exp(z, pr.etab);
      }
      inner = pr.scale * pow_bx + pr.offset;
      saturated = inner >= cap;
    }
    const double eff = saturated ? cap : py_min(py_max(inner, 0.0), cap);
    const int own = NM + (prio == 0 ? 5 : 6), other = NM + (prio == 0 ? 6 : 5);
    const double cfc = prio == 0 ? pr.coeff[0] : pr.coeff[1];
    predicted = 1.0 + eff * cfc;
    double d = 0.0;
    const bool clamp_active = saturated || inner <= 0.0 || inner >= cap;
    if (!clamp_active && owner) {  // _prediction_gradient (predictor.py:285-299)
      const double log_b = pr.log_base;
      const double zz = pr.scale * pow_bx;
      if (lane == 0) d = pow_bx * cfc;
      else if (lane == 1) d = pr.scale * x * (MathT::kInline ? pow_bx1 : MathT::exp((x - 1.0) * log_b, pr.etab)) * cfc;
      else if (lane == 2) d = cfc;
      else if (lane < 3 + NM) {
        double ai = 0.0;
#pragma unroll
        for (int k = 0; k < NM; ++k)
          if (lane == 3 + k) ai = tw[k];
        d = zz * log_b * ai * cfc;
      } else if (lane == 3 + NM) d = zz * log_b * cmp * cfc;
      else if (lane == 4 + NM) d = zz * log_b * mem * cfc;
    }
    if (lane == own) d = eff;
    residual = predicted - actual;
    const double delta = cf->huber_delta;  // huber_grad (predictor.py:155-158)
    const double gh = fabs(residual) <= delta ? residual : (residual > 0 ? delta : -delta);
    const double gk = gh * d;
    const bool finite = __all_sync(kFull, !owner || isfinite(gk)) && isfinite(residual);
    skipped = !finite && !cf->refit_frozen;
    // UpdateResult(skipped=True); a frozen update() returns the loss terms and never steps
    if (!finite || cf->refit_frozen) return;
    ++step;               // adam_step (predictor.py:124-145)
    const double bc1 = step <= A->n_bc ? __ldg(&A->bc1[step - 1]) : 1.0;
    const double bc2 = step <= A->n_bc ? __ldg(&A->bc2[step - 1]) : 1.0;
    const double b1 = cf->beta1, b2 = cf->beta2;
    double p = owner ? P[lane] : 0.0;
    if (owner && lane != other) {
      adam_m = b1 * adam_m + (1.0 - b1) * gk;
      adam_v = b2 * adam_v + (1.0 - b2) * gk * gk;
      const double m_hat = MathT::div(adam_m, bc1);
      const double v_hat = MathT::div(adam_v, bc2);
      p -= MathT::div(cf->learning_rate * m_hat, sqrt(v_hat) + cf->eps);
      if (lane == 0) p = py_max(p, 1e-6);        // enforce_floors (predictor.py:98-102)
      if (lane == 1) p = py_max(p, 1.0 + 1e-6);
    }
    if (lane == NM + 5 || lane == NM + 6) p = py_max(p, 1e-6);
    sync();
    if (owner) P[lane] = p;
    sync();
    load_pred();
  }

  // ------------------------------------------------------------ dispatch (scheduler.py)
  // intf_cur of every running entry = predict(timeline TWA at now) under the
  // current params (scheduler.py:150-153): a function of (entry timeline, now,
  // params) only, so it is evaluated once per pass (lane per slot) and
  // re-evaluated for a GPU's entries after a submission stamps their timelines.
  // Everything of the projection (scheduler.py:150-160) that does not depend on
  // the candidate is cached with it: x0 = w_cmp*cmp + w_mem*mem (the first
  // step of pressure_exponent), rb = (1 - progress) * t_kernel and
  // st = max(now, kernel start); per candidate only intf_new remains.
  __device__ __forceinline__ void icur_slot(int s, double now) const {
    double tw[NM];
    tl_twa(s, now, tw);
    const double cmp = SD(SD_CMP, s), mem = SD(SD_MEM, s);
    const double intf_cur = pr.predict(tw, cmp, mem, SB(SB_PRIO, s));
    const double ks = SD(SD_KS, s), tk = SD(SD_TK, s);
    const double elapsed = py_max(0.0, now - ks);
    const double denom = intf_cur * tk;
    const double progress = denom > 0 ? py_min(1.0, MathT::div(elapsed, denom)) : 1.0;
    SD(SD_RB, s) = (1.0 - progress) * tk;
    SD(SD_ST, s) = py_max(now, ks);
    SD(SD_X0, s) = pr.w_cmp * cmp + pr.w_mem * mem;
  }
  // intf_cur is read only by check_violate of GPUs that have a free slot
  // (has_slot is tested first), so only their entries are evaluated: the
  // slots are compacted into a list and processed 32 at a time
  __device__ __forceinline__ void icur_all(double now) const {
    if constexpr (CTA) {
      if (S > 32) {  // one slot per thread of the CTA
        if (lane == 0) {
          jb->kind = JOB_ICUR;
          jb->now = now;
        }
        post_job();
        job_icur(now);
        return;
      }
    }
    int count = 0;
    for (int s0 = 0; s0 < S; s0 += 32) {
      const int s = s0 + lane;
      const bool need = s < S && SB(SB_LIVE, s) && GI(GI_NRUN, SI(SI_GPU, s)) < CONC;
      const unsigned m = __ballot_sync(kFull, need);
      if (need) slist[count + __popc(m & ((1u << lane) - 1))] = s;
      count += __popc(m);
    }
    __syncwarp();
    for (int i = lane; i < count; i += 32) icur_slot(slist[i], now);
    __syncwarp();
  }
  __device__ __forceinline__ void icur_gpu(int g, double now) const {
    if (lane < GI(GI_NRUN, g)) icur_slot(slot_at(g, lane), now);
    __syncwarp();
  }
  // JOB_ICUR (every warp of the CTA): intf_cur of the entries whose GPU has a free slot
  __device__ __forceinline__ void job_icur(double now) const {
    for (int s = w * 32 + lane; s < S; s += NT)
      if (SB(SB_LIVE, s) && GI(GI_NRUN, SI(SI_GPU, s)) < CONC) icur_slot(s, now);
    cta_bar(2);
  }

  // the candidate batch (model m at size k): profile row at k (domain.py:52-105)
  struct Cand {
    double c[NM];
    double cmp, mem, total, kern;
  };
  __device__ __forceinline__ void load_cand(int m, int k, Cand& cd) const {
#pragma unroll
    for (int i = 0; i < NM; ++i) cd.c[i] = thr(m, k, i);
    cd.cmp = tab_cmp(m, k);
    cd.mem = tab_mem(m, k);
    cd.total = tab_total(m, k);
    cd.kern = tab_kernel(m, k);
  }

  // check_violate (scheduler.py:118-161) of the candidate on GPU g; lane-local.
  __device__ __forceinline__ bool violate(int g, const Cand& cd, int cprio, double now) const {
    if (cprio == 1) {  // LOW: LP aggregate + contribution vs the AIMD cap (:130-135)
      const double capf = GD(GD_CAPF, g);
#pragma unroll
      for (int i = 0; i < NM; ++i)
        if (GD(GD_LPA + i, g) + cd.c[i] > capf) return true;
    }
    const int n = GI(GI_NRUN, g);
    for (int p = 0; p < n; ++p) {  // projection of every equal-or-higher-priority co-runner (:137-160)
      const int s = slot_at(g, p);
      const int ep = SB(SB_PRIO, s);
      if (ep > cprio) continue;
      if (projection(s, cd, ep) > SD(SD_DL, s)) return true;
    }
    return false;
  }
  // projected completion of co-runner s if the candidate joins (scheduler.py:150-159):
  // max(now, ks) + ((1 - progress) * t_kernel) * intf_new
  __device__ __forceinline__ double projection(int s, const Cand& cd, int ep) const {
    double x = SD(SD_X0, s);  // pressure_exponent of (agg - e.contrib) + add, self terms first
#pragma unroll
    for (int i = 0; i < NM; ++i) x += pr.w[i] * (SD(SD_AEX + i, s) + cd.c[i]);
    bool sat;
    const double intf_new = 1.0 + pr.effect(x, sat) * (ep == 0 ? pr.coeff[0] : pr.coeff[1]);
    return SD(SD_ST, s) + SD(SD_RB, s) * intf_new;
  }

  // pressure_exponent of (agg - e.contrib) + add for co-runner s (scheduler.py:150-153)
  __device__ __forceinline__ double proj_x(int s, const Cand& cd) const {
    double x = SD(SD_X0, s);  // self terms first (cached with intf_cur)
#pragma unroll
    for (int i = 0; i < NM; ++i) x += pr.w[i] * (SD(SD_AEX + i, s) + cd.c[i]);
    return x;
  }
  // max(now, ks) + ((1 - progress) * t_kernel) * intf_new > deadline (scheduler.py:154-160)
  __device__ __forceinline__ bool proj_late(int s, double eff, int ep) const {
    const double intf_new = 1.0 + eff * (ep == 0 ? pr.coeff[0] : pr.coeff[1]);
    return SD(SD_ST, s) + SD(SD_RB, s) * intf_new > SD(SD_DL, s);
  }

  // one (size, GPU) pair of best_for (scheduler.py:263-280): has_slot, violate, meet.
  // With exp inlined, check_meet's prediction and the co-runner projections are
  // evaluated two chains at a time ((meet, c0), (c1, c2), (c3, -), ...), stopping
  // at the first violating pair of chains: check_violate's boolean and the meet
  // are pure, so the result is the sequential one.
  __device__ __forceinline__ bool eval_pair(int g, const Cand& cd, int cprio, double dl, double front, double now,
                                            double& lat, double& intf) const {
    const int n = GI(GI_NRUN, g);
    if (!(n < CONC)) return false;  // has_slot (runtime.py:101-102)
    double assumed[NM];  // check_meet (scheduler.py:164-185): half the aggregate
#pragma unroll
    for (int i = 0; i < NM; ++i) assumed[i] = 0.5 * GD(GD_AGG + i, g);
    if constexpr (MathT::kInline && ILP) {
      if (cf->use_violate && cprio == 1) {  // LOW: LP aggregate + contribution vs the AIMD cap (:130-135)
        const double capf = GD(GD_CAPF, g);
#pragma unroll
        for (int i = 0; i < NM; ++i)
          if (GD(GD_LPA + i, g) + cd.c[i] > capf) return false;
      }
      const bool uv = cf->use_violate;
      if (n == 0) {
        intf = pr.predict(assumed, cd.cmp, cd.mem, cprio);
      } else {  // (meet, co-runner 0)
        const int s0 = slot_at(g, 0);
        const int ep0 = SB(SB_PRIO, s0);
        double em, e0;
        pr.effect2(pr.exponent(assumed, cd.cmp, cd.mem), proj_x(s0, cd), em, e0);
        intf = 1.0 + em * (cprio == 0 ? pr.coeff[0] : pr.coeff[1]);
        if (uv && ep0 <= cprio && proj_late(s0, e0, ep0)) return false;
      }
      for (int p = 1; p < n; p += 2) {  // (c1, c2), (c3, c4), ...
        const int sa = slot_at(g, p), sb = p + 1 < n ? slot_at(g, p + 1) : sa;
        const int ea = SB(SB_PRIO, sa), eb = SB(SB_PRIO, sb);
        double fa, fb;
        pr.effect2(proj_x(sa, cd), proj_x(sb, cd), fa, fb);
        if (uv && ((ea <= cprio && proj_late(sa, fa, ea)) || (p + 1 < n && eb <= cprio && proj_late(sb, fb, eb))))
          return false;
      }
    } else {
      if (cf->use_violate && violate(g, cd, cprio, now)) return false;
      intf = pr.predict(assumed, cd.cmp, cd.mem, cprio);
    }
    lat = cd.total + py_max(0.0, GD(GD_TAV, g) - now) + (intf - 1.0) * cd.kern + (now - front);
    return !(cf->use_meet && !(lat <= dl));
  }

  struct Plan {
    bool ok;
    int gpu;
    double lat, intf;
  };

  // lexicographic (latency, gpu_id) argmin across the warp (best_for's tie-break)
  // as three 32-bit warp reductions on an order-preserving image of the latency
  // (-0 folded onto +0, so equal latencies tie on gpu_id as in the scan), then
  // the winner's fields
  __device__ __forceinline__ Plan warp_best(bool found, int bg, double bl, double bi) const {
    unsigned long long lb = (unsigned long long)__double_as_longlong(bl == 0.0 ? 0.0 : bl);
    lb = (lb >> 63) ? ~lb : lb | 0x8000000000000000ull;
    const unsigned h = found ? (unsigned)(lb >> 32) : ~0u, lo = found ? (unsigned)lb : ~0u;
    const unsigned m0 = __reduce_min_sync(kFull, h);
    bool c = found && h == m0;
    const unsigned m1 = __reduce_min_sync(kFull, c ? lo : ~0u);
    c = c && lo == m1;
    const unsigned m2 = __reduce_min_sync(kFull, c ? (unsigned)bg : ~0u);
    c = c && (unsigned)bg == m2;
    const unsigned who = __ballot_sync(kFull, c);
    const int src = who ? __ffs(who) - 1 : 0;
    return Plan{who != 0, __shfl_sync(kFull, bg, src), __shfl_sync(kFull, bl, src), __shfl_sync(kFull, bi, src)};
  }

  // best_for(k) with lanes over GPUs
  __device__ __forceinline__ Plan best_for(int m, int k, int cprio, double dl, double front, double now) const {
    Cand cd;
    load_cand(m, k, cd);
    bool found = false;
    int bg = 0x7fffffff;
    double bl = 0.0, bi = 0.0;
    for (int g = lane; g < NG; g += 32) {
      double lat, intf;
      if (eval_pair(g, cd, cprio, dl, front, now, lat, intf) && (!found || lat < bl)) {
        found = true;
        bg = g;
        bl = lat;
        bi = intf;
      }
    }
    return warp_best(found, bg, bl, bi);
  }

  // The baselines' propose (baselines.py:34-128): placement by occupancy only,
  // BatchPlan(est = (now - front) + total(size), intf = 1.0).
  __device__ __forceinline__ int propose_baseline(int m, double now, Plan& plan) const {
    const double front = front_arrival(m);
    const int kmax = min(q_len(m), mmaxb(m));
    const int pol = policy();
    int gpu = -1, size = kmax;
    if (pol == STRAIT_POLICY_TEMPORAL) {  // first idle GPU; largest size meeting the front deadline
      for (int g0 = 0; g0 < NG && gpu < 0; g0 += 32) {
        const unsigned idle = __ballot_sync(kFull, g0 + lane < NG && GI(GI_NRUN, g0 + lane) == 0);
        if (idle) gpu = g0 + __ffs(idle) - 1;
      }
      if (gpu < 0) return 0;
      const double deadline = front + mdeadline(m);
      int lo = 1, hi = kmax;
      size = 0;
      while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        if (now + tab_total(m, mid) <= deadline) size = mid, lo = mid + 1;
        else hi = mid - 1;
      }
      if (!size) return 0;
    } else {  // static / reactive: min (len(running), gpu_id) over the open GPUs
      const int prio = mprio(m);
      const int bound = prio == 1 ? lp_allowance : cf->reactive_hp_bound;
      const int cap = min(cf->static_cap, CONC);
      unsigned best = ~0u;
      for (int g0 = 0; g0 < NG; g0 += 32) {
        const int g = g0 + lane;
        unsigned key = ~0u;
        if (g < NG) {
          const int n = GI(GI_NRUN, g);
          bool open;
          if (pol == STRAIT_POLICY_STATIC) {
            open = n < cap;
          } else {
            int count = 0;
            for (int p = 0; p < n; ++p) count += SB(SB_PRIO, slot_at(g, p)) == prio;
            open = n < CONC && count < bound;
          }
          if (open) key = ((unsigned)n << 16) | (unsigned)g;
        }
        best = min(best, __reduce_min_sync(kFull, key));
      }
      if (best == ~0u) return 0;
      gpu = (int)(best & 0xffffu);
    }
    plan = Plan{true, gpu, (now - front) + tab_total(m, size), 1.0};
    return size;
  }

  // (Measured and reverted: the jobs as out-of-line calls, so master and helpers
  // share one copy of the code — call-boundary spills doubled a job's time; and
  // the exp table in shared memory — no change, its lookups already hit L1.)
  //
  // JOB_PROPOSE (every warp of the CTA): PredictivePolicy.propose's whole
  // (size x GPU x co-runner) search for queue m.
  //  A. items (k, g, c): c < CONC is check_violate's projection of running entry
  //     c of GPU g (scheduler.py:137-160), c == CONC the pair's LP-cap test
  //     (:130-135) and check_meet (:164-185) — independent chains, one per thread;
  //  B. pairs (k, g): has_slot, the OR of the pair's projections, the meet, then
  //     each size's lexicographic (latency, gpu_id) argmin over its GPUs within
  //     the warp (segments of W lanes, W = pow2ceil(n_gpus) clipped to 32); a warp
  //     chunk's winner goes to part[(k - 1) * chunks + g / 32].
  // check_violate's early exit and co-runner order do not change its boolean,
  // and best_for is pure, so evaluating sizes the search never probes changes
  // nothing.  The job covers sizes k0 + 1 .. k0 + kmax.
  __device__ __forceinline__ void job_propose(int m, int k0, int kmax, int cprio, double dl, double front,
                                              double now) const {
    const int C1 = CONC + 1;
    const int t = w * 32 + lane;
    // Phase A in rounds of NT: thread t takes projection item r0 + t (items
    // (k, g, c), from thread 0 up) and meet item r0 + NT - 1 - t (items (k, g),
    // from the last thread down), and evaluates both effects as one block
    // (Pred::effect2, the exp chains interleave); an absent item computes a
    // dummy exponent whose result is discarded, so the warps stay on one path.
    RP_T(t_pa);
    const bool uv = cf->use_violate;
    const int ni = uv ? kmax * NG * CONC : 0;
    const int np2 = kmax * NG;
    for (int r0 = 0; r0 < ni || r0 < np2; r0 += NT) {  // warp-uniform trip count
      const int i = r0 + t, pg2 = r0 + NT - 1 - t;
      bool hp = false, hm = false;
      int s = 0, ep = 0, pgi = 0, ci = 0, g2 = 0;
      double xp = 1.0, xm = 1.0;
      if (i < ni) {  // A1: check_violate's projection of the entry in slot ci of GPU g (scheduler.py:137-160)
        // items walk a GPU's slots, not its list positions: check_violate's
        // boolean is an OR over the running entries, so the order is immaterial,
        // and the slot's fields load without first reading the running list
        pgi = i / CONC, ci = i - pgi * CONC;
        const int kq = pgi / NG, g = pgi - kq * NG;
        s = slot(g, ci);
        const int n = GI(GI_NRUN, g);
        const bool live = SB(SB_LIVE, s);
        ep = SB(SB_PRIO, s);
        if (n < CONC) {  // else has_slot fails: phase B never reads this pair's items
          if (live && ep <= cprio) {
            Cand cd;
#pragma unroll
            for (int q = 0; q < NM; ++q) cd.c[q] = thr(m, k0 + kq + 1, q);
            xp = proj_x(s, cd);
            hp = true;
          } else {
            pv[pgi * C1 + ci] = 0;
          }
        }
      }
      Cand cm;
      bool capv = false;
      if (pg2 >= 0 && pg2 < np2) {  // A2: the pair's LP-cap test (:130-135) and check_meet (:164-185)
        const int kq = pg2 / NG;
        g2 = pg2 - kq * NG;
        if (GI(GI_NRUN, g2) < CONC) {
          load_cand(m, k0 + kq + 1, cm);
          if (cprio == 1) {
            const double capf = GD(GD_CAPF, g2);
#pragma unroll
            for (int q = 0; q < NM; ++q) capv |= GD(GD_LPA + q, g2) + cm.c[q] > capf;
          }
          double assumed[NM];
#pragma unroll
          for (int q = 0; q < NM; ++q) assumed[q] = 0.5 * GD(GD_AGG + q, g2);
          xm = pr.exponent(assumed, cm.cmp, cm.mem);
          hm = true;
        }
      }
      double fp, fm;
      pr.effect2(xp, xm, fp, fm);
      if (hp) pv[pgi * C1 + ci] = proj_late(s, fp, ep);
      if (hm) {
        const double intf = 1.0 + fm * (cprio == 0 ? pr.coeff[0] : pr.coeff[1]);
        const double lat = cm.total + py_max(0.0, GD(GD_TAV, g2) - now) + (intf - 1.0) * cm.kern + (now - front);
        pm[pg2] = (uint8_t)((lat <= dl ? 1 : 0) | (capv ? 2 : 0));
        plat[pg2] = lat;
        pintf[pg2] = intf;
      }
    }
    if (w == 0) RP_ADD(RPF_CTA_PA, t_pa);  // the master's own phase-A items
#if STRAIT_REPLAY_PROFILE
    if (lane == 0) {
      atomicAdd(&g_cta_warp[0][w], (unsigned long long)(t_pa - jb->t0));
      atomicAdd(&g_cta_warp[1][w], (unsigned long long)(clock64() - jb->t0));
    }
#endif
    RP_T(t_b);
    cta_bar(3);
    if (w == 0) RP_ADD(RPF_CTA_B, t_b);  // the master's wait at the end of phase A
    RP_T(t_pb);
    const int lw = NG <= 1 ? 0 : 32 - __clz(NG - 1);
    const int W = 1 << lw, seg = W < 32 ? W : 32, nch = Layout::cta_chunks(NG);
    const int np = kmax << lw;
    for (int b0 = w * 32; b0 < np; b0 += NT) {  // warp-uniform trip count
      const int p = b0 + lane, kq = p >> lw, g = p & (W - 1);
      bool found = false;
      int bg = g;
      double bl = 0.0, bi = 0.0;
      if (kq < kmax && g < NG && GI(GI_NRUN, g) < CONC) {
        const int pg = kq * NG + g;
        const int f = pm[pg];
        bool viol = false;
        if (cf->use_violate) {
          viol = (f & 2) != 0;
          for (int c = 0; c < CONC; ++c) viol |= pv[pg * C1 + c] != 0;
        }
        found = !viol && !(cf->use_meet && !(f & 1));
        bl = plat[pg];
        bi = pintf[pg];
      }
      if (seg == 32) {  // a whole warp is one size's chunk of 32 GPUs
        const Plan b = warp_best(found, bg, bl, bi);
        found = b.ok, bg = b.gpu, bl = b.lat, bi = b.intf;
      } else {
        for (int off = seg >> 1; off; off >>= 1) {
          const bool f2 = __shfl_xor_sync(kFull, found, off);
          const int g2 = __shfl_xor_sync(kFull, bg, off);
          const double l2 = __shfl_xor_sync(kFull, bl, off);
          const double i2 = __shfl_xor_sync(kFull, bi, off);
          if (f2 && (!found || l2 < bl || (l2 == bl && g2 < bg))) {
            found = true;
            bg = g2;
            bl = l2;
            bi = i2;
          }
        }
      }
      if ((lane & (seg - 1)) == 0 && kq < kmax) part[kq * nch + (g >> 5)] = Part{bl, bi, found ? bg : -1, 0};
    }
    if (w == 0) RP_ADD(RPF_CTA_PB, t_pb);  // the master's phase-B pairs
#if STRAIT_REPLAY_PROFILE
    if (lane == 0) atomicAdd(&g_cta_warp[2][w], (unsigned long long)(clock64() - jb->t0));
#endif
    RP_T(t_j);
    cta_bar(2);
    if (w == 0) RP_ADD(RPF_CTA_J, t_j);  // the master's wait at the join
  }
  // master side of JOB_PROPOSE: post it for sizes k0 + 1 .. k0 + kcnt and take part in it
  __device__ __forceinline__ void run_propose_job(int m, int k0, int kcnt, int cprio, double dl, double front,
                                                  double now) {
#if STRAIT_REPLAY_PROFILE
    if (lane == 0) *jb = Job{JOB_PROPOSE, m, kcnt, cprio, k0, 0, now, dl, front, clock64()};
#else
    if (lane == 0) *jb = Job{JOB_PROPOSE, m, kcnt, cprio, k0, 0, now, dl, front, 0};
#endif
    RP_T(t_a);
    post_job();
    job_propose(m, k0, kcnt, cprio, dl, front, now);
    RP_ADD(RPF_CTA_A, t_a);  // post + phases A and B (barrier-bound: the slowest warp)
    RP_CNT(RPF_N_CTA);
  }
  // best of size index kq over its warp chunks, in GPU order (best_for's tie-break)
  __device__ __forceinline__ bool size_best(int kq, int nch, int& bg, double& bl, double& bi) const {
    bool found = false;
    for (int ch = 0; ch < nch; ++ch) {
      const Part q = part[kq * nch + ch];
      if (q.g >= 0 && (!found || q.t < bl || (q.t == bl && q.g < bg))) {
        found = true;
        bg = q.g;
        bl = q.t;
        bi = q.x;
      }
    }
    return found;
  }
  // PredictivePolicy.propose on the CTA.  When the (size x GPU x co-runner)
  // items of every size fit in two passes of the CTA, one job evaluates all
  // sizes and the binary search's probes are replayed on the feasibility bits
  // (lane k - 1 holds size k).  Otherwise (C5's 64 GPUs) each probe is one job
  // over its GPUs x co-runners, ~1 item per thread, in the search's order.
  __device__ __forceinline__ int propose_cta(int m, int kmax, double now, Plan& plan) {
    const double front = front_arrival(m);
    const int cprio = mprio(m);
    const double dl = mdeadline(m);
    const int nch = Layout::cta_chunks(NG);
    int lo = 1, hi = kmax, bestk = 0;
    if (kmax * NG * (CONC + 1) > STRAIT_CTA_PROBE_ITEMS * NT) {
      while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        run_propose_job(m, mid - 1, 1, cprio, dl, front, now);
        int bg = 0;
        double bl = 0.0, bi = 0.0;
        if (size_best(0, nch, bg, bl, bi)) {
          bestk = mid;
          plan = Plan{true, bg, bl, bi};
          lo = mid + 1;
        } else {
          hi = mid - 1;
        }
      }
      return bestk;
    }
    run_propose_job(m, 0, kmax, cprio, dl, front, now);
    RP_T(t_m);
    bool found = false;
    int bg = 0;
    double bl = 0.0, bi = 0.0;
    if (lane < kmax) found = size_best(lane, nch, bg, bl, bi);
    const unsigned feas = __ballot_sync(kFull, found);  // bit k - 1: best_for(k) is not None
    while (lo <= hi) {
      const int mid = (lo + hi) / 2;
      if (feas >> (mid - 1) & 1u) {
        bestk = mid;
        lo = mid + 1;
      } else {
        hi = mid - 1;
      }
    }
    if (bestk) {
      const int src = bestk - 1;
      plan = Plan{true, __shfl_sync(kFull, bg, src), __shfl_sync(kFull, bl, src), __shfl_sync(kFull, bi, src)};
    }
    RP_ADD(RPF_CTA_M, t_m);
    return bestk;
  }

  // PredictivePolicy.propose (scheduler.py:257-285) + largest_feasible (:78-90).
  // When every size fits in the warp (kmax segments of W = pow2ceil(n_gpus)
  // lanes), all sizes are evaluated at once (lane = (k - 1) * W + g; best_for
  // is pure, so evaluating sizes the search never probes changes nothing),
  // each size's argmin is a segmented butterfly, and the binary search's exact
  // probe sequence is replayed on the feasibility bits.  Otherwise sizes are probed one at a
  // time with lanes over GPUs.  Probes never repeat, so the reference's memo
  // reduces to the plan of the last feasible probe.
  __device__ __forceinline__ int propose(int m, double now, Plan& plan) {
    const double front = front_arrival(m);
    const int kmax = min(q_len(m), mmaxb(m));
    if constexpr (CTA)
      if (kmax <= 32) return propose_cta(m, kmax, now, plan);
    const int cprio = mprio(m);
    const double dl = mdeadline(m);
    int lo = 1, hi = kmax, bestk = 0;
    // segment width: next power of two >= n_gpus
    const int lw = NG <= 1 ? 0 : 32 - __clz(NG - 1);
    if ((kmax << lw) <= 32) {
      RP_CNT(RPF_N_PROPOSE_WIDE);
#if STRAIT_REPLAY_PROFILE
      prof[RPF_SUM_KMAX] += kmax;
      {
        bool any = false;
        int ne = 0;
        for (int g = 0; g < NG; ++g) any |= GI(GI_NRUN, g) < CONC, ne += GI(GI_NRUN, g);
        prof[RPF_N_NOSLOT] += !any;
        prof[RPF_SUM_ENTRIES] += ne;
      }
#endif
      const int W = 1 << lw;
      const int k = (lane >> lw) + 1, g = lane & (W - 1);
      bool found = false;
      int bg = g;
      double bl = 0.0, bi = 0.0;
      if (k <= kmax && g < NG) {
        Cand cd;
        load_cand(m, k, cd);
        found = eval_pair(g, cd, cprio, dl, front, now, bl, bi);
      }
      // best_for(k) is not None iff some lane of size k's W-lane segment found a
      // pair: the binary search's probes run on those bits, and only the chosen
      // size's (latency, gpu_id) argmin is reduced (warp reductions over the
      // segment's lanes)
      const unsigned fb = __ballot_sync(kFull, found);
      const unsigned segmask = W == 32 ? ~0u : (1u << W) - 1;
      while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        if (fb >> ((mid - 1) << lw) & segmask) {
          bestk = mid;
          lo = mid + 1;
        } else {
          hi = mid - 1;
        }
      }
      if (bestk) plan = warp_best(found && k == bestk, bg, bl, bi);
      return bestk;
    }
    if constexpr (LEAN) {  // the launcher chose LEAN for a geometry that cannot reach here
      fail(STRAIT_EINVAL);
      return 0;
    } else {
      while (lo <= hi) {
        const int mid = (lo + hi) / 2;
        const Plan p = best_for(m, mid, cprio, dl, front, now);
        if (p.ok) {
          bestk = mid;
          plan = p;
          lo = mid + 1;
        } else {
          hi = mid - 1;
        }
      }
      return bestk;
    }
  }

  // early_drop (scheduler.py:65-75).  deadline_abs - now is monotone in queue
  // order (FIFO of nondecreasing arrival times plus a per-model deadline_ms, and
  // rounding is monotone), so the dropped set is always a prefix of the queue.
  __device__ __forceinline__ void early_drop(int m, double now) {
    const int h = QI(QI_HEAD, m), t = QI(QI_TAIL, m);
    if (h == t) return;
    const double floor_latency = tab_total(m, 1), dl = mdeadline(m);
    if (!((qf[m] + dl) - now < floor_latency)) return;  // the front stays, hence all stay (prefix)
    int ndrop = 0;
    for (int b = h; b < t; b += 32) {
      const int p = b + lane;
      const bool drop = p < t && (arr(req_at(p)) + dl) - now < floor_latency;
      const unsigned mask = __ballot_sync(kFull, drop);
      if (mask == kFull) {
        ndrop += 32;
        continue;
      }
      ndrop += __ffs(~mask) - 1;
      break;
    }
    if (!ndrop) return;
    for (int i = lane; i < ndrop; i += 32) {  // request rows of the dropped (simulation.py:240-257)
      const int64_t gidx = req_at(h + i);
      A->req_status[gidx] = 2;
      A->req_violated[gidx] = 1;
      A->req_completion[gidx] = __longlong_as_double(0x7ff8000000000000LL);
      A->req_batch[gidx] = -1;
    }
    if constexpr (TR) {  // "drop" rows in queue order (simulation.py:353-355)
      for (int i = lane; i < ndrop; i += 32) trace_put(c_trace + i, STRAIT_TR_DROP, now, -1, -1, req_at(h + i), 0, 0.0, 0.0, 0.0);
      c_trace += ndrop;
    }
    resolved += ndrop;
    if (mprio(m) == 0) c_hp_drop += ndrop, c_hp_viol += ndrop;
    else c_lp_drop += ndrop, c_lp_viol += ndrop;
    put(QI(QI_HEAD, m), h + ndrop);
    put(QI(QI_FGEN, m), QI(QI_FGEN, m) + 1);
    if (h + ndrop < t) put(qf[m], arr(req_at(h + ndrop)));
    sync();
    if (mprio(m) == 0) signal_hp(-1, now);  // simulation.py:352-357
  }

  // submit_plan (scheduler.py:295-324) + Simulation on_submit (simulation.py:305-350)
  __device__ __forceinline__ void submit(int m, int k, const Plan& plan, double now, int pass_id) {
    const int bid = batch_seq++;
    const int g = plan.gpu;
    const int h = QI(QI_HEAD, m);
    const int n = GI(GI_NRUN, g);
    int j = 0;
    while (j < C && SB(SB_LIVE, slot(g, j))) ++j;
    if (j >= C || n >= CONC) {  // GpuRuntimeState.add_entry (runtime.py:125-126)
      fail(STRAIT_ERUNTIME);
      return;
    }
    const int s = slot(g, j);
    const double d = tab_transfer(m, k);
    if (!(d > 0)) fail(STRAIT_EINVAL);  // PcieLinkState.reserve (pcie.py:28-29)
    const double start = py_max(now, GD(GD_TAV, g)), end = start + d;
    const double front = qf[m];
    const double next_front = h + k < QI(QI_TAIL, m) ? arr(req_at(h + k)) : 0.0;
    const double noise = cf->has_noise ? __ldg(&A->noise[base + bid]) : 1.0;  // simulation.py:309-311
    sync();
    if (lane == 0) {
      QI(QI_HEAD, m) = h + k;  // TaskQueue.pop_front
      qf[m] = next_front;
      QI(QI_FGEN, m) = QI(QI_FGEN, m) + 1;
      GD(GD_TAV, g) = end;
      const int tailp = GI(GI_PHEAD, g) + GI(GI_PN, g);  // < 2C: ring index without a division
      GD(GD_PEND + (tailp >= C ? tailp - C : tailp), g) = end;
      GI(GI_PN, g) = GI(GI_PN, g) + 1;
      SB(SB_MODEL, s) = (int8_t)m;
      SB(SB_SIZE, s) = (int8_t)k;
      SB(SB_PRIO, s) = (int8_t)mprio(m);
      SB(SB_STARTED, s) = 0;
      SB(SB_LIVE, s) = 1;
      SB(SB_TLEN, s) = 0;
      SI(SI_BID, s) = bid;
      SI(SI_REQ0, s) = h;
#pragma unroll
      for (int i = 0; i < NM; ++i) SD(SD_CON + i, s) = thr(m, k, i);
      SD(SD_CMP, s) = tab_cmp(m, k);
      SD(SD_MEM, s) = tab_mem(m, k);
      SD(SD_TK, s) = tab_kernel(m, k);
      SD(SD_DL, s) = front + mdeadline(m);
      SD(SD_KS, s) = end;  // kernel_start_estimate
      SD(SD_REM, s) = tab_kernel(m, k);
      SD(SD_SLOW, s) = 1.0;
      SD(SD_NOISE, s) = noise;
      SD(SD_LAST, s) = 0.0;
      SD(SD_WORK, s) = 0.0;
      ORD(n, g) = (int8_t)j;
      GI(GI_NRUN, g) = n + 1;
    }
    sync();
    recompute_aggregate(g);
    stamp_all(g, now);
    push_event(s, end, kTC);
    sync();
    recompute(g, now);
    trace1(STRAIT_TR_SUBMIT, now, g, bid, -1, k, start, end, plan.lat);  // simulation.py:321-328
    if (lane == 0) {
      const int64_t o = base + bid;
      A->dec_time[o] = now;
      A->dec_pass[o] = pass_id;
      A->dec_model[o] = (int16_t)m;
      A->dec_size[o] = (int8_t)k;
      A->dec_gpu[o] = (int16_t)g;
      A->dec_est_latency[o] = plan.lat;
      A->dec_intf[o] = plan.intf;
      A->b_front[o] = front;
      A->b_transfer_start[o] = start;
      A->b_transfer_end[o] = end;
    }
    ++c_batches;
  }

  __device__ __forceinline__ bool has_any_slot() const {
    bool any = false;
    for (int g0 = 0; g0 < NG; g0 += 32) any |= __any_sync(kFull, g0 + lane < NG && GI(GI_NRUN, g0 + lane) < CONC);
    return any;
  }

  // _ensure_timeout for one model (simulation.py:231-238)
  __device__ __forceinline__ void ensure_timeout(int m, double now) {
    if (!q_len(m) || QI(QI_TGEN, m) == QI(QI_FGEN, m)) return;
    const double t = py_max(now, front_arrival(m) + mtimeout(m));
    const int gen = QI(QI_FGEN, m);
    push_event(S + m, t, kTO);
    put(QI(QI_EGEN, m), gen);
    put(QI(QI_TGEN, m), gen);
    sync();
  }

  // _ensure_timeout for every queue in model order (simulation.py:360-361)
  __device__ __forceinline__ void ensure_timeouts(double now) {
    RP_T(t_to);
    for (int m0 = 0; m0 < M; m0 += 32) {
      const int m = m0 + lane;
      const bool need = m < M && q_len(m) > 0 && QI(QI_TGEN, m) != QI(QI_FGEN, m);
      const unsigned mask = __ballot_sync(kFull, need);
      if (need) {
        const unsigned long long q = seq + 1 + __popc(mask & ((1u << lane) - 1));
        ed[S + m] = py_max(now, front_arrival(m) + mtimeout(m));
        ek[S + m] = ((unsigned long long)kTO << 56) | q;
        QI(QI_EGEN, m) = QI(QI_FGEN, m);
        QI(QI_TGEN, m) = QI(QI_FGEN, m);
      }
      seq += __popc(mask);
    }
    sync();
    RP_ADD(RPF_TIMEOUTS, t_to);
  }

  // Simulation._pass (simulation.py:301-361) + run_scheduling_pass (scheduler.py:355-378)
  __device__ __forceinline__ void do_pass(double now) {
    const int pass_id = ++pass_seq;
    ++c_passes;
    if (policy() == STRAIT_POLICY_REACTIVE) reactive_catch_up(now);  // begin_pass (baselines.py:113-114)
    // The queues this pass acts on: a front that early_drop removes, or an
    // eligible queue (TaskQueue.eligible).  A queue's front and length change
    // only when the pass reaches that queue (its own drop / submission), so both
    // tests give at the pass start what they give when the loop reaches it; a
    // ready queue in neither set is a no-op of the loop and is skipped.
    RP_T(t_rank);
    unsigned long long act = 0, dropm = 0;
    for (int m0 = 0; m0 < M; m0 += 32) {
      const int m = m0 + lane;
      bool d = false, e = false;
      if (m < M) {
        const int len = q_len(m);
        if (len) {
          const double fr = front_arrival(m);
          // lane m's model constants stay in registers (M <= 32, loaded once in run())
          const double mdl = m0 == 0 ? my_dl : mdeadline(m), mfl = m0 == 0 ? my_floor : tab_total(m, 1);
          const double mto = m0 == 0 ? my_to : mtimeout(m);
          const int mmb = m0 == 0 ? my_maxb : mmaxb(m);
          d = (fr + mdl) - now < mfl;  // early_drop's front test (scheduler.py:65-75)
          e = len >= mmb || now >= fr + mto;
        }
      }
      dropm |= (unsigned long long)__ballot_sync(kFull, d) << m0;
      act |= (unsigned long long)__ballot_sync(kFull, d || e) << m0;
    }
    RP_ADD(RPF_RANK, t_rank);
    if (act) pass_queues(now, act, dropm, pass_id);
    ensure_timeouts(now);
  }

  // the acted-on queues of a pass, in queue order: early drop, then at most one
  // submission per eligible queue (run_scheduling_pass, scheduler.py:355-378)
  __device__ __forceinline__ void pass_queues(double now, unsigned long long act, unsigned long long dropm,
                                              int pass_id) {
    RP_T(t_rank);
    const bool predictive = policy() == STRAIT_POLICY_PREDICTIVE;
    // queue_order (scheduler.py:249-255): stable sort of the acted-on ready
    // queues by (priority, front arrival, model_id) — the order their subset
    // has in the sort of all ready queues — as a lane-parallel rank sort.
    // key = priority in the top bit | bit pattern of the (>= 0) front arrival.
    const bool use_prio = cf->use_priority_order;
    const int n = __popcll(act);
    if (M <= 32) {  // keys in registers, broadcast by shuffles
      const bool on = lane < M && (act >> lane & 1);
      const unsigned long long km =
          on ? ((unsigned long long)(use_prio ? mprio(lane) : 0) << 63) |
                   (unsigned long long)__double_as_longlong(front_arrival(lane))
             : kNoKey;
      int rank = 0;
#pragma unroll 4
      for (int j = 0; j < M; ++j) {
        const unsigned long long kj = __shfl_sync(kFull, km, j);
        rank += kj < km || (kj == km && j < lane);
      }
      __syncwarp();
      if (on) QI(QI_ORD, rank) = lane;
    } else {
      unsigned long long* qk = reinterpret_cast<unsigned long long*>(qd);
      for (int m = lane; m < M; m += 32)
        qk[m] = act >> m & 1 ? ((unsigned long long)(use_prio ? mprio(m) : 0) << 63) |
                                   (unsigned long long)__double_as_longlong(front_arrival(m))
                             : kNoKey;
      sync();
      for (int m = lane; m < M; m += 32) {
        const unsigned long long km = qk[m];
        if (km != kNoKey) {
          int rank = 0;
#pragma unroll 1
          for (int j = 0; j < M; ++j) {
            const unsigned long long kj = qk[j];
            rank += kj < km || (kj == km && j < m);
          }
          QI(QI_ORD, rank) = m;
        }
      }
    }
    sync();
    RP_ADD(RPF_RANK, t_rank);
    bool icur_ready = false;
    // No GPU with a free slot => no policy can place anything (has_slot fails for
    // every pair; the baselines need len(running) < cap <= limit too), so the
    // pass only drops: proposes and intf_cur are skipped until a slot exists.
    bool any_slot = has_any_slot();
    for (int i = 0; i < n && !err; ++i) {
      const int m = QI(QI_ORD, i);
      RP_T(t_drop);
      RP_CNT(RPF_N_QUEUES);
      if (dropm >> m & 1) early_drop(m, now);
      RP_ADD(RPF_DROP, t_drop);
      RP_T(t_elig);
      const int len = q_len(m);
      if (!len) continue;
      // TaskQueue.eligible: known from the pass start unless the drop moved the front
      if ((dropm >> m & 1) && !(len >= mmaxb(m) || now >= front_arrival(m) + mtimeout(m))) continue;
      RP_CNT(RPF_N_ELIGIBLE);
      if (!any_slot) continue;
      if (predictive && !icur_ready) {
        RP_CNT(RPF_N_ICUR_ALL);
        icur_all(now);
        icur_ready = true;
      }
      RP_ADD(RPF_ELIG, t_elig);
      RP_T(t_prop);
      Plan plan;
      const int k = predictive ? propose(m, now, plan) : propose_baseline(m, now, plan);
      RP_ADD(RPF_PROPOSE, t_prop);
      if (!k) continue;
      RP_T(t_sub);
      RP_CNT(RPF_N_SUBMIT);
      submit(m, k, plan, now, pass_id);
      RP_ADD(RPF_SUBMIT, t_sub);
      RP_T(t_icur);
      if (predictive) icur_gpu(plan.gpu, now);
      RP_ADD(RPF_ICUR, t_icur);
      any_slot = has_any_slot();
    }
  }

  // ------------------------------------------------------------ event handlers
  __device__ __forceinline__ void on_transfer_complete(int s, double now) {  // simulation.py:378-394
    const int g = SI(SI_GPU, s);
    const int pn = GI(GI_PN, g);
    if (pn <= 0) {  // PcieLinkState.calibrate with nothing pending (pcie.py:43-44)
      fail(STRAIT_EINVAL);
      return;
    }
    sync();
    if (lane == 0) {
      // calibrate (pcie.py:36-53): FIFO => the oldest reservation is this batch's
      const int ph = GI(GI_PHEAD, g);
      const double predicted = GD(GD_PEND + ph, g);
      const int nph = ph + 1 == C ? 0 : ph + 1, npn = pn - 1;
      GI(GI_PHEAD, g) = nph;
      GI(GI_PN, g) = npn;
      if (!npn) {
        GD(GD_TAV, g) = now;
      } else {
        const double off = now - predicted;
        if (off != 0.0) {
          GD(GD_TAV, g) = GD(GD_TAV, g) + off;
#pragma unroll 1
          for (int i = 0; i < npn; ++i) {
            const int q = nph + i >= C ? nph + i - C : nph + i;
            GD(GD_PEND + q, g) = GD(GD_PEND + q, g) + off;
          }
        }
      }
      SB(SB_STARTED, s) = 1;
      SD(SD_KS, s) = now;  // kernel_start (and kernel_start_estimate)
      SB(SB_TLEN, s) = 0;  // timeline reset to the kernel window
      double v[NM];  // timeline reset to [(now, aggregate_excluding(entry))]
#pragma unroll
      for (int i = 0; i < NM; ++i) v[i] = SD(SD_AEX + i, s);
      tl_record(s, now, v);
      SD(SD_SLOW, s) = gt_slowdown(s);
      SD(SD_LAST, s) = now;
      A->b_kernel_start[base + SI(SI_BID, s)] = now;
    }
    sync();
    push_event(s, SD(SD_LAST, s) + SD(SD_REM, s) * SD(SD_SLOW, s), kKC);
    trace1(STRAIT_TR_KSTART, now, g, SI(SI_BID, s), -1, 0, SD(SD_SLOW, s));  // simulation.py:391-394
    sync();
  }

  // simulation.py:396-460 (+ complete_batch, scheduler.py:327-352)
  __device__ __forceinline__ void on_kernel_complete(int s, double now) {
    const int g = SI(SI_GPU, s), j = SI(SI_J, s);
    const int m = SB(SB_MODEL, s), k = SB(SB_SIZE, s), prio = SB(SB_PRIO, s);
    const int bid = SI(SI_BID, s), req0 = SI(SI_REQ0, s);
    bool ok = true;
    const double seg_d = now - SD(SD_LAST, s), seg_slow = SD(SD_SLOW, s);
    sync();
    if (lane == 0) ok = ex_consume(s, now);
    if (seg_d > 0) trace1(STRAIT_TR_SEGMENT, now, g, bid, -1, 0, seg_d, seg_slow);  // ExecutionState.finish
    fail_any(!ok, STRAIT_EORDER);
    sync();
    const double measured = now - SD(SD_KS, s);
    const double completion = now + (tab_total(m, k) - tab_transfer(m, k) - tab_kernel(m, k));
    const double dl = mdeadline(m);
    int nviol = 0;
    for (int i0 = 0; i0 < k; i0 += 32) {
      const int i = i0 + lane;
      bool viol = false;
      if (i < k) {
        const int64_t gidx = req_at(req0 + i);
        viol = completion > arr(gidx) + dl;
        A->req_status[gidx] = 1;
        A->req_violated[gidx] = (uint8_t)viol;
        A->req_completion[gidx] = completion;
        A->req_batch[gidx] = bid;
      }
      nviol += __popc(__ballot_sync(kFull, viol));
    }
    resolved += k;
    if (prio == 0) c_hp_viol += nviol;
    else c_lp_viol += nviol;
    double tw[NM];
    tl_twa(s, now, tw);
    const double tk = tab_kernel(m, k);
    const double actual = MathT::div(measured, tk);
    if (!(actual > 0)) fail(STRAIT_EINVAL);
    // GpuRuntimeState.remove_entry (runtime.py:132-141): shift the running list
    const int n = GI(GI_NRUN, g);
    int pos = 0;
    while (pos < n && ORD(pos, g) != j) ++pos;
    if (pos == n) fail(STRAIT_ERUNTIME);
    const double work = SD(SD_WORK, s);
    sync();
    if (lane == 0) {
      for (int p = pos; p + 1 < n; ++p) ORD(p, g) = ORD(p + 1, g);
      GI(GI_NRUN, g) = n - 1;
      SB(SB_LIVE, s) = 0;
    }
    clear_event(s);
    sync();
    recompute_aggregate(g);
    stamp_all(g, now);
    double predicted, residual;
    bool skipped, saturated;
    RP_T(t_upd);
    update(tw, tab_cmp(m, k), tab_mem(m, k), prio, actual, predicted, residual, skipped, saturated);
    RP_ADD(RPF_KC_UPDATE, t_upd);
    if (lane == 0) {
      const int64_t o = base + bid;
      A->fb_predicted[o] = predicted;
      A->fb_actual[o] = actual;
      A->fb_residual[o] = residual;
      A->fb_flags[o] = (uint8_t)((skipped ? 1 : 0) | (saturated ? 2 : 0));
      A->b_kernel_end[o] = now;
      A->b_completion[o] = completion;
      A->b_work[o] = work;
      A->b_done_order[o] = done_order;
    }
    ++done_order;
    ++c_completed;
    recompute(g, now);
    trace1(STRAIT_TR_KDONE, now, g, bid, -1, 0, measured, actual);  // simulation.py:454-457
    if (prio == 0 && nviol) signal_hp(g, now);  // simulation.py:458-459
  }

  __device__ __forceinline__ void on_tick_advance(double now) {  // AimdState.advance (runtime.py:26-34)
    bool bad = false;
    for (int g0 = 0; g0 < NG; g0 += 32) {
      const int g = g0 + lane;
      bool changed = false;
      double cap = 0.0;
      if (g < NG) {
        const double old = GD(GD_CAP, g), last = GD(GD_TICK, g);
        if (now < last) bad = true;
        const double whole = floor(MathT::div(now - last, cf->aimd_interval));
        cap = old;
        if (whole > 0) {
          cap = py_min(cf->aimd_ceiling, old + whole * cf->aimd_increase);
          GD(GD_CAP, g) = cap;
          GD(GD_CAPF, g) = MathT::div(cap, 100.0);
          GD(GD_TICK, g) = last + whole * cf->aimd_interval;
        }
        changed = cap != old;
      }
      const unsigned mask = __ballot_sync(kFull, changed);
      if (changed) cap_row_at(c_cap_rows + __popc(mask & ((1u << lane) - 1)), now, g, cap);
      c_cap_rows += __popc(mask);
    }
    sync();
    fail_any(bad, STRAIT_EINVAL);
  }

  // ------------------------------------------------------------ next event
  // this thread's share of the event homes: i = first, first + step, ...
  __device__ __forceinline__ void scan_homes(int first, int step, double& bt, unsigned long long& bk, int& bi) const {
#pragma unroll 4
    for (int i = first; i < NE; i += step) {
      const double t = ed[i];
      const unsigned long long kk = ek[i];
      if (t < bt || (t == bt && kk < bk)) bt = t, bk = kk, bi = i;
    }
  }
  // across lanes: event times are >= 0, so their bit patterns order like the
  // values; a 128-bit (time, key) minimum as four 32-bit warp reductions.
  // Leaves the minimum and its home in every lane.
  __device__ __forceinline__ void warp_min_event(double& bt, unsigned long long& bk, int& bi) const {
    const unsigned long long tb = (unsigned long long)__double_as_longlong(bt);
    const unsigned w0 = (unsigned)(tb >> 32), w1 = (unsigned)tb, w2 = (unsigned)(bk >> 32), w3 = (unsigned)bk;
    const unsigned m0 = __reduce_min_sync(kFull, w0);
    bool c = w0 == m0;
    const unsigned m1 = __reduce_min_sync(kFull, c ? w1 : ~0u);
    c = c && w1 == m1;
    const unsigned m2 = __reduce_min_sync(kFull, c ? w2 : ~0u);
    c = c && w2 == m2;
    const unsigned m3 = __reduce_min_sync(kFull, c ? w3 : ~0u);
    c = c && w3 == m3;
    bk = ((unsigned long long)m2 << 32) | m3;
    bt = __longlong_as_double((long long)(((unsigned long long)m0 << 32) | m1));
    bi = __shfl_sync(kFull, bi, __ffs(__ballot_sync(kFull, c)) - 1);
  }
  // helper warps (NW > 1): parked on barrier 1 until the master posts a job
  __device__ void helper_loop() {
    for (;;) {
      cta_bar(1);
      const int kind = jb->kind;
      if (kind == JOB_EXIT) return;
      const double now = jb->now;
      load_shared_pred();
      if (kind == JOB_ICUR) job_icur(now);
      else job_propose(jb->m, jb->k0, jb->kmax, jb->cprio, jb->dl, jb->front, now);
    }
  }

  // ------------------------------------------------------------ main loop (simulation.py:475-513)
  __device__ __forceinline__ void run() {
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    const int np = NP;
    const double* st = A->pred_state + r * 3 * np;
    if (lane < np) P[lane] = st[lane];
    adam_m = lane < np ? st[np + lane] : 0.0;
    adam_v = lane < np ? st[2 * np + lane] : 0.0;
    step = A->pred_step[r];
    for (int g = lane; g < G; g += 32) {
      GD(GD_TAV, g) = 0.0;
      GD(GD_CAP, g) = cf->aimd_floor;
      GD(GD_CAPF, g) = MathT::div(cf->aimd_floor, 100.0);
      GD(GD_TICK, g) = 0.0;
      GI(GI_NRUN, g) = 0;
      GI(GI_PHEAD, g) = 0;
      GI(GI_PN, g) = 0;
#pragma unroll
      for (int i = 0; i < NM; ++i) GD(GD_AGG + i, g) = GD(GD_LPA + i, g) = 0.0;
    }
    for (int s = lane; s < S; s += 32) {
      SB(SB_LIVE, s) = 0;
      SI(SI_GPU, s) = s / C;
      SI(SI_J, s) = s % C;
    }
    for (int i = lane; i < NE; i += 32) {
      ed[i] = INF;
      ek[i] = kNoKey;
    }
    int64_t hp_arr = 0, lp_arr = 0;
    for (int m = lane; m < M; m += 32) {
      const int64_t b = A->mr_off[r * M + m], e = A->mr_off[r * M + m + 1];
      QI(QI_HEAD, m) = QI(QI_TAIL, m) = (int)b;
      QI(QI_FGEN, m) = 0;
      QI(QI_TGEN, m) = -1;
      QI(QI_EGEN, m) = 0;
      if (mprio(m) == 0) hp_arr += e - b;
      else lp_arr += e - b;
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      hp_arr += __shfl_xor_sync(kFull, hp_arr, off);
      lp_arr += __shfl_xor_sync(kFull, lp_arr, off);
    }
#pragma unroll 1
    for (int64_t i = lane; i < N; i += 32) A->req_status[base + i] = 0;
    for (int g = lane; g < NG; g += 32) cap_row_at(g, 0.0, g, cf->aimd_floor);  // simulation.py:196-197
    sync();
    load_pred();
    c_cap_rows = NG;
    seq = (unsigned long long)N;  // the arrivals took seq 1..N (simulation.py:184-194)
    next_arr = 0;
    my_dl = lane < M ? mdeadline(lane) : 0.0;
    my_floor = lane < M ? tab_total(lane, 1) : 0.0;
    my_to = lane < M ? mtimeout(lane) : 0.0;
    my_maxb = lane < M ? mmaxb(lane) : 0;
    pf_q = pf_g = 0;
    pf_m = N ? (int)__ldg(&A->arr_model[base]) : 0;
    pf_t2 = N > 1 ? arr(base + 1) : INF;
    if (N) {
      push_event(S + M, cf->aimd_interval, kTICK);
      put(ed[S + M + 1], arr(base));
      put(ek[S + M + 1], (unsigned long long)kARR << 56);
    }
    sync();

    if (LEAN && cf->policy != STRAIT_POLICY_PREDICTIVE) err = STRAIT_EINVAL;  // args.policies was wrong
#if STRAIT_REPLAY_PROFILE
    for (int i = 0; i < RPF_N; ++i) prof[i] = 0;
    RP_T(t_all);
#endif
    while (!err) {
      RP_T(t_sel);
      // next event: lexicographic argmin of (time, kind << 56 | seq) over all homes
      double bt = INF;
      unsigned long long bk = kNoKey;
      int bi = -1;
      // (the CTA layout scans on the master too: with the scan unrolled, a scan
      // job's wake-up costs what splitting the homes saves)
      scan_homes(lane, 32, bt, bk, bi);
      warp_min_event(bt, bk, bi);
      if (bk == kNoKey) break;
      sync();  // the scan's reads of the event homes complete before any handler writes them
      RP_ADD(RPF_SELECT, t_sel);
      RP_T(t_h);
      const int kind = (int)(bk >> 56);
      const double now = bt;
      ++c_events;
      // each handler's pre-pass part, at most one pass, then the post-pass part,
      // so the pass is instantiated once
      bool pass = false;
      int post_timeout = -1;
      bool post_tick = false;
      if (kind == kARR) {  // _on_arrival (simulation.py:365-371)
        // the arrival stream is read one arrival ahead (pf_m, pf_t2), and the
        // queue-order check of the previous arrival is settled now, so no
        // global load is waited on here
        if (pf_q != pf_g) fail(STRAIT_EINVAL);  // per-model arrivals must pop in k order
        const int64_t gidx = base + next_arr;
        const int m = pf_m;
        ++next_arr;
        put(ed[S + M + 1], next_arr < N ? pf_t2 : INF);
        put(ek[S + M + 1], next_arr < N ? (unsigned long long)kARR << 56 : kNoKey);
        pf_m = next_arr < N ? (int)__ldg(&A->arr_model[base + next_arr]) : 0;
        pf_t2 = next_arr + 1 < N ? arr(base + next_arr + 1) : INF;
        const int t = QI(QI_TAIL, m);
        pf_q = req_at(t);
        pf_g = gidx;
        put(QI(QI_TAIL, m), t + 1);
        if (t + 1 - QI(QI_HEAD, m) == 1) {  // TaskQueue.push into an empty queue: new front
          put(QI(QI_FGEN, m), QI(QI_FGEN, m) + 1);
          put(qf[m], now);
        }
        trace1(STRAIT_TR_ARRIVAL, now, -1, -1, gidx);  // simulation.py:368
        sync();
        pass = q_len(m) == mmaxb(m);
        post_timeout = m;
        RP_ADD(RPF_ARRIVAL, t_h);
      } else if (kind == kKC) {
        on_kernel_complete(bi, now);
        pass = true;
        RP_ADD(RPF_KC_PRE, t_h);
      } else if (kind == kTC) {
        on_transfer_complete(bi, now);
        RP_ADD(RPF_TC, t_h);
      } else if (kind == kTO) {  // _on_timeout (simulation.py:373-376)
        const int m = bi - S;
        const int gen = QI(QI_EGEN, m);
        clear_event(bi);
        sync();
        pass = q_len(m) && gen == QI(QI_FGEN, m);
      } else {  // _on_tick (simulation.py:462-471)
        clear_event(bi);
        sync();
        on_tick_advance(now);
        trace1(STRAIT_TR_TICK, now);  // simulation.py:468
        pass = true;
        post_tick = true;
        RP_ADD(RPF_TICK, t_h);
      }
      if (pass && !err) do_pass(now);
      RP_T(t_post);
      if (post_timeout >= 0) ensure_timeout(post_timeout, now);
      if (post_tick && resolved < N) {
        push_event(S + M, now + cf->aimd_interval, kTICK);
        sync();
      }
      RP_ADD(RPF_POST, t_post);
    }
    if constexpr (CTA) {  // release the helper warps (the loop's only exit is above)
      if (lane == 0) jb->kind = JOB_EXIT;
      post_job();
    }
#if STRAIT_REPLAY_PROFILE
    RP_ADD(RPF_TOTAL, t_all);
    if (lane == 0)
      for (int i = 0; i < RPF_N; ++i) atomicAdd(&g_replay_prof[i], (unsigned long long)prof[i]);
#endif
    if (pf_q != pf_g) fail(STRAIT_EINVAL);  // the last arrival's queue-order check
    if (!err && resolved != N) err = STRAIT_EORDER;  // unresolved requests (simulation.py:491-494)
    sync();
    double* so = A->pred_state + r * 3 * np;
    if (lane < np) {
      so[lane] = P[lane];
      so[np + lane] = adam_m;
      so[2 * np + lane] = adam_v;
    }
    if (lane == 0) {
      A->pred_step[r] = step;
      int64_t* c = A->counters + r * STRAIT_RC_N;
      for (int i = 0; i < STRAIT_RC_N; ++i) c[i] = 0;
      c[STRAIT_RC_ERROR] = err;
      c[STRAIT_RC_BATCHES] = c_batches;
      c[STRAIT_RC_COMPLETED] = c_completed;
      c[STRAIT_RC_PASSES] = c_passes;
      c[STRAIT_RC_CAP_ROWS] = c_cap_rows;
      c[STRAIT_RC_EVENTS] = c_events;
      c[STRAIT_RC_HP_ARR] = hp_arr;
      c[STRAIT_RC_LP_ARR] = lp_arr;
      c[STRAIT_RC_HP_VIOL] = c_hp_viol;
      c[STRAIT_RC_LP_VIOL] = c_lp_viol;
      c[STRAIT_RC_HP_DROP] = c_hp_drop;
      c[STRAIT_RC_LP_DROP] = c_lp_drop;
      c[STRAIT_RC_RESOLVED] = resolved;
      c[STRAIT_RC_TRACE] = c_trace;
    }
  }
};

// MINB = minimum resident CTAs of 4 warps per SM: 1 lets ptxas keep the whole
// replay state in registers (latency: few replays), 4 caps it at 128 registers
// for 16 resident replays per SM (throughput: replay sweeps).
// NW = 1: up to wpc replays per CTA, one warp each.  NW > 1: one replay per
// CTA of NW warps (warp 0 the master, the others helpers).
template <int NM, int MINB, bool TR, bool LEAN, int GEOM, int NW, bool ILP = true>
__global__ void __launch_bounds__(NW > 1 ? 32 * NW : 128, MINB)
    replay_kernel(const __grid_constant__ StraitReplayArgs a, int wpc) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int w = threadIdx.x >> 5;
  const int64_t slot_w = NW > 1 ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * wpc + w;
  if (slot_w >= a.n_replays) return;
  const int64_t r = a.order ? (int64_t)a.order[slot_w] : slot_w;
  const Layout L(a.max_gpus, a.max_concurrency, a.models.n_models, NM, NW, a.models.stride);
  unsigned char* base = NW > 1 ? smem : smem + (size_t)w * L.bytes;
  Sim<NM, typename std::conditional<(MINB >= 4), OutlineMath, FullInlineMath>::type, TR, LEAN, GEOM, NW, ILP> S;
  S.A = &a;
  S.cf = a.cfg + r;
  S.lane = threadIdx.x & 31;
  S.w = NW > 1 ? w : 0;
  S.r = r;
  if (!S.set_geom(L, S.cf, a.models.stride)) {  // the launcher chose a fixed geometry this replay does not have
    if (S.lane == 0 && S.w == 0) {
      int64_t* c = a.counters + r * STRAIT_RC_N;
      for (int i = 0; i < STRAIT_RC_N; ++i) c[i] = 0;
      c[STRAIT_RC_ERROR] = STRAIT_EINVAL;
    }
    return;  // uniform over the CTA when NW > 1: no helper is left parked
  }
  S.base = a.req_off[r];
  S.N = a.req_off[r + 1] - S.base;
  S.P = (double*)(base + L.P);
  S.sd = (double*)(base + L.sd);
  S.gd = (double*)(base + L.gd);
  S.ed = (double*)(base + L.ed);
  S.ek = (unsigned long long*)(base + L.ek);
  S.qd = (double*)(base + L.qd);
  S.qf = (double*)(base + L.qf);
  S.slist = (int*)(base + L.sl);
  S.si = (int*)(base + L.si);
  S.gi = (int*)(base + L.gi);
  S.qi = (int*)(base + L.qi);
  S.sb = (int8_t*)(base + L.sb);
  S.go = (int8_t*)(base + L.go);
  S.qb = (int8_t*)(base + L.qb);
  S.jb = (Job*)(base + L.jb);
  S.pv = (uint8_t*)(base + L.pv);
  S.pm = (uint8_t*)(base + L.pm);
  S.plat = (double*)(base + L.plat);
  S.pintf = (double*)(base + L.pintf);
  S.part = (Part*)(base + L.part);
  if (NW > 1 && w > 0) {
    S.helper_loop();
    return;
  }
  S.batch_seq = S.pass_seq = S.done_order = S.err = 0;
  S.lp_allowance = S.cf->reactive_default;
  S.last_reset = 0.0;
  S.resolved = 0;
  S.c_batches = S.c_completed = S.c_passes = S.c_events = S.c_trace = 0;
  S.c_hp_viol = S.c_lp_viol = S.c_hp_drop = S.c_lp_drop = 0;
  S.run();
}

// LEAN instantiations: a predictive-only batch (args.policies) whose largest
// batch size x pow2ceil(max GPUs) fits one warp, so every propose takes the
// all-sizes-at-once path
inline bool lean_batch(const StraitReplayArgs& a) {
  const int g = a.max_gpus, lw = g <= 1 ? 0 : 32 - __builtin_clz((unsigned)(g - 1));
  return a.policies == (1 << STRAIT_POLICY_PREDICTIVE) && ((int64_t)a.models.stride << lw) <= 32;
}

// GEOM 1 instantiations: every replay has 4 GPUs x 4 slots and 6 models
// (args.uniform: each replay at the launch maxima)
inline bool overload_geometry(const StraitReplayArgs& a) {
  return a.uniform && a.max_gpus == 4 && a.max_concurrency == 4 && a.models.n_models == 6;
}

inline bool c5_geometry(const StraitReplayArgs& a) {
  return a.uniform && a.max_gpus == 64 && a.max_concurrency == 4 && a.models.n_models == 20;
}

// host side: launch one instantiation (explicitly specialised in strait_replay_nm*.cu);
// minb = 4 selects the 128-register throughput variant, 0 the traced latency variant,
// 2 the CTA-per-replay latency variant (kCtaWarps warps per replay), 3 its traced
// form (geometries past the one-warp shared-memory budget), else the one-warp
// latency variant
constexpr int kCtaWarps = 8;

inline int sm_count_cached() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        n <= 0)
      n = 148;
  }
  return n;
}

template <int NM>
int launch_replay(const StraitReplayArgs& a, cudaStream_t st, int wpc, size_t smem_per_warp, int minb);

// shared memory of one CTA-per-replay replay (0: more than the opt-in maximum)
inline size_t cta_replay_smem(const StraitReplayArgs& a) {
  const size_t b = Layout(a.max_gpus, a.max_concurrency, a.models.n_models, a.models.n_metrics, kCtaWarps,
                          a.models.stride).bytes;
  return b <= 227 * 1024 ? b : 0;
}

template <int NM, int MINB, bool TR, bool LEAN, int GEOM, int NW = 1, bool ILP = true>
int launch_replay_occ(const StraitReplayArgs& a, cudaStream_t st, int wpc, size_t smem_per_warp) {
  const size_t smem = NW > 1 ? cta_replay_smem(a) : smem_per_warp * wpc;
  auto* k = replay_kernel<NM, MINB, TR, LEAN, GEOM, NW, ILP>;
  if (!smem || cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return set_error(STRAIT_ECUDA, "strait_replay: cannot reserve %zu B of shared memory", smem);
  const unsigned grid = NW > 1 ? (unsigned)a.n_replays : (unsigned)((a.n_replays + wpc - 1) / wpc);
  k<<<grid, NW > 1 ? 32 * NW : 32 * wpc, smem, st>>>(a, wpc);
  return check_launch("strait_replay");
}

#define STRAIT_INSTANTIATE_REPLAY(NMV)                                                                            \
  template <>                                                                                                     \
  int launch_replay<NMV>(const StraitReplayArgs& a, cudaStream_t st, int wpc, size_t smem_per_warp, int minb) { \
    const bool po = lean_batch(a);                                                                                \
    if (minb == 3) /* traced, geometry past the one-warp budget: CTA per replay with the event log */           \
      return launch_replay_occ<NMV, 1, true, false, 0, kCtaWarps, false>(a, st, wpc, smem_per_warp);                    \
    if (minb == 2) { /* CTA per replay: single replays and few-replay launches */                                \
      if constexpr (NMV == 5) {                                                                                   \
        if (c5_geometry(a)) return launch_replay_occ<NMV, 1, false, false, 3, kCtaWarps>(a, st, wpc, smem_per_warp); \
        if (po && overload_geometry(a) && a.models.stride == 8)                                                   \
          return launch_replay_occ<NMV, 1, false, true, 2, kCtaWarps, false>(a, st, wpc, smem_per_warp);                \
      }                                                                                                           \
      return po ? launch_replay_occ<NMV, 1, false, true, 0, kCtaWarps, false>(a, st, wpc, smem_per_warp)                \
                : launch_replay_occ<NMV, 1, false, false, 0, kCtaWarps, false>(a, st, wpc, smem_per_warp);              \
    }                                                                                                             \
    if constexpr (NMV == 5) /* traced: run() / Simulation.run() of the overload geometry */                     \
      if (minb == 0 && po && overload_geometry(a) && a.models.stride == 8)                                       \
        return launch_replay_occ<NMV, 1, true, true, 2>(a, st, wpc, smem_per_warp);                             \
    if (minb == 0) return launch_replay_occ<NMV, 1, true, false, 0>(a, st, wpc, smem_per_warp);                  \
    if constexpr (NMV == 5)                                                                                       \
      if (minb == 1 && c5_geometry(a)) return launch_replay_occ<NMV, 1, false, false, 3>(a, st, wpc, smem_per_warp); \
    if constexpr (NMV == 5)                                                                                       \
      if (po && overload_geometry(a))                                                                             \
        return minb >= 4 ? launch_replay_occ<NMV, 4, false, true, 1>(a, st, wpc, smem_per_warp)                  \
                         : a.models.stride == 8 ? (a.n_replays > sm_count_cached() ? launch_replay_occ<NMV, 1, false, true, 2, 1, false>(a, st, wpc, smem_per_warp) : launch_replay_occ<NMV, 1, false, true, 2>(a, st, wpc, smem_per_warp)) \
                                                : launch_replay_occ<NMV, 1, false, true, 1>(a, st, wpc, smem_per_warp); \
    if (minb >= 4)                                                                                                \
      return po ? launch_replay_occ<NMV, 4, false, true, 0>(a, st, wpc, smem_per_warp)                           \
                : launch_replay_occ<NMV, 4, false, false, 0>(a, st, wpc, smem_per_warp);                         \
    return po ? launch_replay_occ<NMV, 1, false, true, 0>(a, st, wpc, smem_per_warp)                             \
              : launch_replay_occ<NMV, 1, false, false, 0>(a, st, wpc, smem_per_warp);                           \
  }

}  // namespace rp
}  // namespace strait
