// strait_sweep.cu — the candidate sweep (R1-R4, R9-R11) and the batched
// estimator entry points (R1-R4), plus the fused sweep+refit round.
//
// Layout (see include/strait.h): one THREAD per (candidate, GPU, co-runner)
// triple, the n_slots threads of a (candidate, GPU) pair are adjacent lanes.
// Every thread issues all of its SoA loads up front (coalesced: consecutive
// lanes read consecutive doubles of each field array), so a CTA keeps
// ~16 independent 8-byte loads per thread in flight — the sweep is HBM-bound
// (~0.5 flop/byte) and the design goal is bytes in flight, not FLOPs.
//   1. triple:  check_violate's per-entry projection (scheduler.py:137-160)
//   2. pair:    OR over the pair's lanes (__shfl_xor), LP-cap check
//               (scheduler.py:130-135), check_meet (:164-185) on the leader lane
//   3. segment: best_for's lexicographic (latency, gpu_id) argmin over the
//               segment's pairs (:263-280), one warp per segment over shared memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>

#include "strait_capi.cuh"
#include "strait_device.cuh"
#include "strait_ptx.cuh"
#include "strait_refit.cuh"

namespace strait {

constexpr int kSweepThreads = 256;       // compute threads per CTA (one per triple)
constexpr int kMaxStages = 4;
constexpr int kMaxGroups = 2;  // consumer groups of 8 warps (named barriers 1 .. 10)
// an upper bound of RN(cap / 100) for cap >= 0: RN(cap * kCapFractionHi) exceeds
// cap / 100 by a relative ~2^-40, far above the two roundings (each <= 2^-53)
constexpr double kCapFractionHi = 0.01 * (1.0 + 0x1p-40);

// A *tile* is the unit one CTA processes at a time: `spb` consecutive segments
// (all of their pairs and triples), contiguous in every SoA field array.
struct TileGeom {
  int G, C, span, spb, TT, TP;  // TT triples / TP pairs per tile
  __host__ __device__ TileGeom(int g, int c) : G(g), C(c) {
    span = G * C;
    spb = span <= kSweepThreads ? kSweepThreads / span : 1;
    TT = spb * span;
    TP = spb * G;
  }
};

__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) { return (x + a - 1) & ~(a - 1); }

// Byte layout of one pipeline stage in shared memory.  Triple fields are
// metric-major [field][TT]; pair fields [field][TP]; candidate values
// [field][spb].  The same layout serves the synchronous kernel (pair/cand
// only) and the TMA pipeline (everything, filled by cp.async.bulk).
template <int NM>
struct StageLayout {
  static constexpr int kEntF = 2 * NM + 5;   // contrib[NM], twa[NM], cmp, mem, t_kernel, deadline_abs, kstart
  static constexpr int kPairF = 2 * NM + 2;  // agg[NM], lp_agg[NM], cap_pct, t_avail
  static constexpr int kCandF = NM + 6;      // contrib[NM], cmp, mem, total, kernel, front, deadline
  size_t ent, eprio, pair, nrun, cand, cprio, bytes, tx_bytes;
  __host__ __device__ StageLayout(const TileGeom& t) {
    ent = 0;
    eprio = ent + (size_t)kEntF * t.TT * 8;
    pair = align_up(eprio + t.TT, 128);  // TMA tensor-copy destination
    nrun = pair + (size_t)kPairF * t.TP * 8;
    cand = align_up(nrun + t.TP, 16);
    cprio = cand + (size_t)kCandF * t.spb * 8;
    bytes = align_up(cprio + 4 * t.spb, 128);  // TMA path stores the aligned 4-byte word holding each prio
    tx_bytes = (size_t)kEntF * t.TT * 8 + t.TT + (size_t)kPairF * t.TP * 8 + t.TP;
  }
};

// Per-CTA (not per-stage) scratch after the stages: pair results + predictor.
template <int NM>
struct CtaLayout {
  size_t lat, intf, adm, pred, bars, refit, bytes;
  __host__ __device__ CtaLayout(const TileGeom& t, const StageLayout<NM>& sl, int nstages) {
    lat = sl.bytes * nstages;
    intf = lat + (size_t)t.TP * 8;
    adm = intf + (size_t)t.TP * 8;
    pred = align_up(adm + t.TP, 16);
    bars = align_up(pred + sizeof(Pred<NM>), 16);
    refit = bars + 8 * kMaxStages;
    bytes = refit + 8 * kMaxP;
  }
};

// best_for's scan: the first admitted pair seeds `best`; a later pair replaces
// it iff its latency is strictly smaller (scheduler.py:277, GPUs in id order).
// Equivalent reducible form: if the first admitted latency is NaN it wins;
// otherwise NaN latencies never win and the argmin takes the smallest g on ties.
struct ArgminKey {
  int first_g;       // smallest admitted g (INT_MAX if none)
  double first_lat;  // its latency
  int best_g;        // argmin over admitted non-NaN latencies, ties -> smaller g
  double best_lat;
};

__device__ __forceinline__ ArgminKey argmin_combine(ArgminKey a, const ArgminKey& b) {
  if (b.first_g < a.first_g) {
    a.first_g = b.first_g;
    a.first_lat = b.first_lat;
  }
  if (b.best_g != INT_MAX &&
      (a.best_g == INT_MAX || b.best_lat < a.best_lat || (b.best_lat == a.best_lat && b.best_g < a.best_g))) {
    a.best_g = b.best_g;
    a.best_lat = b.best_lat;
  }
  return a;
}

__device__ __forceinline__ ArgminKey argmin_warp(ArgminKey k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgminKey other;
    other.first_g = __shfl_xor_sync(0xffffffffu, k.first_g, o);
    other.first_lat = __shfl_xor_sync(0xffffffffu, k.first_lat, o);
    other.best_g = __shfl_xor_sync(0xffffffffu, k.best_g, o);
    other.best_lat = __shfl_xor_sync(0xffffffffu, k.best_lat, o);
    k = argmin_combine(k, other);
  }
  return k;
}

// Triple operands of one thread.
template <int NM>
struct TripleRegs {
  double ec[NM], tw[NM];
  double cmp, mem, tk, dl, ks;
  int prio;
};

// Compute one tile whose pair/candidate operands are staged at `stage`, for
// the triple held in `e` (thread-local index `local` within the tile).  Ends
// with the segment argmin; contains two group barriers.
template <int NM, int C>
__device__ __forceinline__ void tile_compute(const StraitSweepArgs& a, const TileGeom& tg,
                                             const StageLayout<NM>& L, const CtaLayout<NM>& CL,
                                             unsigned char* smem, unsigned char* stage, int64_t seg0,
                                             const TripleRegs<NM>& e) {
  const int tid = threadIdx.x;
  const int G = tg.G, TP = tg.TP, spb = tg.spb;
  const int64_t S = a.n_segments;
  const int nseg = (int)((S - seg0) < spb ? (S - seg0) : spb);
  const bool active = tid < nseg * tg.span;
  const int sl = active ? tid / tg.span : 0;
  const int r = tid - sl * tg.span;
  const int g = r / C;
  const int c = r - g * C;
  const int pl = sl * G + g;
  const double now = a.now;
  const double* pair = (const double*)(stage + L.pair);
  const int8_t* nrun_s = (const int8_t*)(stage + L.nrun);
  const double* cand = (const double*)(stage + L.cand);
  const int8_t* cprio_s = (const int8_t*)(stage + L.cprio);
  const Pred<NM>& pr = *(const Pred<NM>*)(smem + CL.pred);
  double* s_lat = (double*)(smem + CL.lat);
  double* s_intf = (double*)(smem + CL.intf);
  uint8_t* s_adm = (uint8_t*)(smem + CL.adm);

  // ---- 1. triple: projection of one running entry (scheduler.py:137-160) ----
  const int nrun = active ? nrun_s[pl] : 0;
  const int cprio = active ? cprio_s[sl] : 0;
  // the LOW candidate's AIMD-cap test answers check_violate before any co-runner is read (scheduler.py:129-135)
  bool capv = false;
  if (active && cprio == 1) {
    const double cap_fraction = pair[(2 * NM) * TP + pl] / 100.0;
#pragma unroll
    for (int m = 0; m < NM; ++m) capv |= pair[(NM + m) * TP + pl] + cand[m * spb + sl] > cap_fraction;
  }
  bool viol = false;
  if (active && c < nrun && e.prio <= cprio && !capv) {
    // current progress under the time-weighted co-location (R6 input)
    const double intf_cur = pr.predict(e.tw, e.cmp, e.mem, e.prio);
    const double elapsed = py_max(0.0, now - e.ks);
    const double denom = intf_cur * e.tk;
    const double progress = denom > 0 ? py_min(1.0, elapsed / denom) : 1.0;
    double nagg[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) nagg[m] = pair[m * TP + pl] - e.ec[m] + cand[m * spb + sl];
    const double intf_new = pr.predict(nagg, e.cmp, e.mem, e.prio);
    const double remaining = (1.0 - progress) * e.tk * intf_new;
    const double projected = py_max(now, e.ks) + remaining;
    viol = projected > e.dl;
  }

  // ---- 2. pair: OR over the C lanes, LP cap + check_meet on the leader lane ----
  unsigned vbits = viol ? 1u : 0u;
#pragma unroll
  for (int o = C / 2; o > 0; o >>= 1) vbits |= __shfl_xor_sync(0xffffffffu, vbits, o, C);
  if (active && c == 0) {
    uint8_t flags = 0;
    double lat = __longlong_as_double(0x7ff8000000000000LL), intf = lat;  // NaN
    bool admitted = false;
    if (nrun < a.concurrency_limit) {  // runtime.py:101-102 has_slot
      flags |= STRAIT_PAIR_HAS_SLOT;
      bool violate = vbits != 0;
      if (cprio == 1) {  // LOW candidate vs the AIMD cap (scheduler.py:130-135)
        const double cap_fraction = pair[(2 * NM) * TP + pl] / 100.0;  // runtime.py:39-40
#pragma unroll
        for (int m = 0; m < NM; ++m)
          if (pair[(NM + m) * TP + pl] + cand[m * spb + sl] > cap_fraction) violate = true;
      }
      if (violate) flags |= STRAIT_PAIR_VIOLATE;
      double assumed[NM];  // check_meet: half the GPU aggregate (scheduler.py:178)
#pragma unroll
      for (int m = 0; m < NM; ++m) assumed[m] = 0.5 * pair[m * TP + pl];
      intf = pr.predict(assumed, cand[(NM + 0) * spb + sl], cand[(NM + 1) * spb + sl], cprio);
      const double wait = py_max(0.0, pair[(2 * NM + 1) * TP + pl] - now);  // pcie.py:21-23
      lat = cand[(NM + 2) * spb + sl] + wait + (intf - 1.0) * cand[(NM + 3) * spb + sl] +
            (now - cand[(NM + 4) * spb + sl]);
      const bool ok = lat <= cand[(NM + 5) * spb + sl];
      if (ok) flags |= STRAIT_PAIR_MEET;
      admitted = !(a.use_violate && violate) && !(a.use_meet && !ok);
      if (admitted) flags |= STRAIT_PAIR_FEASIBLE;
    }
    const int64_t p = seg0 * G + pl;
    if (a.pair_flags) a.pair_flags[p] = flags;
    if (a.pair_latency) __stcs(a.pair_latency + p, lat);
    if (a.pair_intf) __stcs(a.pair_intf + p, intf);
    s_lat[pl] = lat;
    s_intf[pl] = intf;
    s_adm[pl] = admitted;
  }
  group_sync(kSweepThreads);

  // ---- 3. segment: best_for argmin, one warp per segment ----
  const int warp = tid >> 5, lane = tid & 31;
  for (int q = warp; q < nseg; q += kSweepThreads / 32) {
    ArgminKey k{INT_MAX, 0.0, INT_MAX, 0.0};
    for (int gg = lane; gg < G; gg += 32) {
      const int qp = q * G + gg;
      if (!s_adm[qp]) continue;
      const double lt = s_lat[qp];
      ArgminKey en{gg, lt, INT_MAX, 0.0};
      if (!isnan(lt)) {
        en.best_g = gg;
        en.best_lat = lt;
      }
      k = argmin_combine(k, en);
    }
    k = argmin_warp(k);
    if (lane == 0) {
      const int64_t s = seg0 + q;
      int bg = -1;
      if (k.first_g != INT_MAX) bg = isnan(k.first_lat) ? k.first_g : k.best_g;
      const double nan = __longlong_as_double(0x7ff8000000000000LL);
      a.seg_gpu[s] = bg;
      a.seg_latency[s] = bg >= 0 ? s_lat[q * G + bg] : nan;
      a.seg_intf[s] = bg >= 0 ? s_intf[q * G + bg] : nan;
    }
  }
  group_sync(kSweepThreads);  // stage + pair results free for reuse
}

// Candidate value v of field f for segment s (global, read-only path).
template <int NM>
__device__ __forceinline__ double cand_field(const StraitSweepArgs& a, int f, int64_t s) {
  if (f < NM) return __ldg(a.cand_contrib + f * a.n_segments + s);
  switch (f - NM) {
    case 0: return __ldg(a.cand_self_cmp + s);
    case 1: return __ldg(a.cand_self_mem + s);
    case 2: return __ldg(a.cand_total + s);
    case 3: return __ldg(a.cand_kernel + s);
    case 4: return __ldg(a.cand_front + s);
    default: return __ldg(a.cand_deadline + s);
  }
}

// Cooperative synchronous staging of the tile's pair + candidate operands.
template <int NM>
__device__ __forceinline__ void stage_pairs_sync(const StraitSweepArgs& a, const TileGeom& tg,
                                                 const StageLayout<NM>& L, unsigned char* stage, int64_t seg0) {
  const int64_t S = a.n_segments, Pn = S * tg.G;
  const int nseg = (int)((S - seg0) < tg.spb ? (S - seg0) : tg.spb);
  const int npair = nseg * tg.G, TP = tg.TP, spb = tg.spb;
  double* pair = (double*)(stage + L.pair);
  int8_t* nrun = (int8_t*)(stage + L.nrun);
  double* cand = (double*)(stage + L.cand);
  int8_t* cprio = (int8_t*)(stage + L.cprio);
  const int64_t p0 = seg0 * tg.G;
  for (int q = threadIdx.x; q < npair; q += kSweepThreads) {
    const int64_t p = p0 + q;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      pair[m * TP + q] = __ldcs(a.gpu_agg + m * Pn + p);
      pair[(NM + m) * TP + q] = __ldcs(a.gpu_lp_agg + m * Pn + p);
    }
    pair[(2 * NM) * TP + q] = __ldcs(a.gpu_cap_pct + p);
    pair[(2 * NM + 1) * TP + q] = __ldcs(a.gpu_t_avail + p);
    nrun[q] = __ldcs(a.gpu_n_running + p);
  }
  for (int q = threadIdx.x; q < nseg * StageLayout<NM>::kCandF; q += kSweepThreads) {
    const int f = q / nseg, sl = q - f * nseg;
    cand[f * spb + sl] = cand_field<NM>(a, f, seg0 + sl);
  }
  for (int q = threadIdx.x; q < nseg; q += kSweepThreads) cprio[q] = __ldg(a.cand_prio + seg0 + q);
}

template <int NM>
__device__ __forceinline__ void load_triple_global(const StraitSweepArgs& a, int64_t t, TripleRegs<NM>& e) {
  const int64_t Tn = a.n_segments * a.gpus_per_segment * a.n_slots;
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    e.ec[m] = __ldcs(a.ent_contrib + m * Tn + t);
    e.tw[m] = __ldcs(a.ent_twa + m * Tn + t);
  }
  e.cmp = __ldcs(a.ent_self_cmp + t);
  e.mem = __ldcs(a.ent_self_mem + t);
  e.tk = __ldcs(a.ent_t_kernel + t);
  e.dl = __ldcs(a.ent_deadline_abs + t);
  e.ks = __ldcs(a.ent_kstart + t);
  e.prio = __ldcs(a.ent_prio + t);
}

// ============================================================== synchronous kernel
// General geometry (any G, power-of-two C).  Grid = one CTA per tile; each
// thread loads its triple into registers while the CTA stages pair/candidate
// operands into shared memory.
template <int NM, int C>
__global__ void __launch_bounds__(kSweepThreads + 32, 2)
    sweep_sync_kernel(const StraitSweepArgs a, const StraitRefitArgs r, int with_refit) {
  extern __shared__ __align__(128) unsigned char smem[];
  const TileGeom tg(a.gpus_per_segment, C);
  const StageLayout<NM> L(tg);
  const CtaLayout<NM> CL(tg, L, 1);
  if (threadIdx.x >= kSweepThreads) {  // the optional refit warp of CTA 0
    if (with_refit && blockIdx.x == 0) refit_warp<NM>(r, (double*)(smem + CL.refit));
    return;
  }
  const int64_t seg0 = (int64_t)blockIdx.x * tg.spb;
  const int64_t S = a.n_segments;
  const int nseg = (int)((S - seg0) < tg.spb ? (S - seg0) : tg.spb);
  if (threadIdx.x == 0) ((Pred<NM>*)(smem + CL.pred))->load(a.params, a.effect_cap);
  TripleRegs<NM> e;
  e.prio = 0;
  if ((int)threadIdx.x < nseg * tg.span) load_triple_global<NM>(a, seg0 * tg.span + threadIdx.x, e);
  stage_pairs_sync<NM>(a, tg, L, smem, seg0);
  group_sync(kSweepThreads);
  tile_compute<NM, C>(a, tg, L, CL, smem, smem, seg0, e);
}

// ============================================================== warp-specialized TMA pipeline
// Persistent CTAs walk the tiles blockIdx.x, +gridDim.x, ...  Roles:
//   * producer warp: for every tile waits the stage's EMPTY barrier, posts the
//     tile's byte count on its FULL barrier and issues one cp.async.bulk per
//     SoA field chunk (one lane per chunk); candidate values (8 bytes per
//     field, below the bulk-copy granule) ride one tile ahead in registers and
//     are stored into the stage before the producer arrives on FULL.
//   * `groups` x 8 consumer warps: group q takes every groups-th tile; a warp
//     owns 32 consecutive triples of the tile.  No CTA-wide barriers: each warp
//     computes its triples, ORs pairs with shuffles, writes pair results into
//     the stage, and the LAST warp of the tile to finish (shared atomic
//     counter) runs best_for's argmin for the tile's segments.  Each warp then
//     releases the stage (EMPTY arrive, 8 per tile).
//   * optional refit warp (CTA 0 only): the serial Adam chain of strait_round.
// One bulk copy of a tile: src = src0 + tile * stride, into stage + dst.
struct BulkCopy {
  const char* src0;
  int64_t stride;
  uint32_t dst, bytes;
};

template <int NM>
struct WsLayout {
  StageLayout<NM> st;
  size_t res_lat, res_intf, res_adm, res_viol, cnt, stage_bytes;
  size_t pred, full, empty, refit, copies, etab, bytes;
  __host__ __device__ WsLayout(const TileGeom& t, int nstages) : st(t) {
    res_lat = st.bytes;
    res_intf = res_lat + (size_t)t.TP * 8;
    res_adm = res_intf + (size_t)t.TP * 8;
    res_viol = res_adm + t.TP;  // per pair: some co-runner projection violates (phase 1)
    cnt = align_up(res_viol + t.TP, 16);
    stage_bytes = align_up(cnt + 16, 128);
    pred = stage_bytes * nstages;
    full = align_up(pred + sizeof(Pred<NM>), 16);
    empty = full + 8 * kMaxStages;
    refit = empty + 8 * kMaxStages;
    copies = align_up(refit + 8 * kMaxP, 16);
    etab = align_up(copies + sizeof(BulkCopy) * (4 * kMaxM + 9), 16);
    bytes = etab + 128 * 16;  // shared copy of the exp table (strait_libm.cuh)
  }
};

constexpr int kWsMaxStages = kMaxStages;

template <int NM>
__device__ __forceinline__ int n_bulk_copies() { return (2 * NM + 5) + 1 + (2 * NM + 2) + 1; }

// Table of the tile's bulk copies (built once per CTA): every SoA field chunk
// of a tile is contiguous, so copy i of tile t is src0_i + t * stride_i.
template <int NM, int C>
__device__ __forceinline__ int build_copy_table(const StraitSweepArgs& a, const TileGeom& tg, const StageLayout<NM>& L,
                                                BulkCopy* tab) {
  const int64_t S = a.n_segments, Pn = S * tg.G, Tn = Pn * C;
  const uint32_t tb = tg.TT * 8, pb = tg.TP * 8;
  int n = 0;
  auto add = [&](const void* base, int64_t stride, size_t dst, uint32_t bytes) {
    tab[n++] = BulkCopy{(const char*)base, stride, (uint32_t)dst, bytes};
  };
  for (int m = 0; m < NM; ++m) add(a.ent_contrib + m * Tn, tb, L.ent + (size_t)m * tb, tb);
  for (int m = 0; m < NM; ++m) add(a.ent_twa + m * Tn, tb, L.ent + (size_t)(NM + m) * tb, tb);
  const double* ef[5] = {a.ent_self_cmp, a.ent_self_mem, a.ent_t_kernel, a.ent_deadline_abs, a.ent_kstart};
  for (int j = 0; j < 5; ++j) add(ef[j], tb, L.ent + (size_t)(2 * NM + j) * tb, tb);
  add(a.ent_prio, tg.TT, L.eprio, tg.TT);
  for (int m = 0; m < NM; ++m) add(a.gpu_agg + m * Pn, pb, L.pair + (size_t)m * pb, pb);
  for (int m = 0; m < NM; ++m) add(a.gpu_lp_agg + m * Pn, pb, L.pair + (size_t)(NM + m) * pb, pb);
  add(a.gpu_cap_pct, pb, L.pair + (size_t)(2 * NM) * pb, pb);
  add(a.gpu_t_avail, pb, L.pair + (size_t)(2 * NM + 1) * pb, pb);
  add(a.gpu_n_running, tg.TP, L.nrun, tg.TP);
  return n;
}

// SG != 0 fixes gpus_per_segment at compile time (SG * C == 256: one segment per
// tile) so every shared-memory offset folds into an immediate.
template <int NM, int C, int SG>
__global__ void __launch_bounds__(32 * (8 * kMaxGroups + 2), 1)
    sweep_ws_kernel(const StraitSweepArgs a, const StraitRefitArgs r, int with_refit, int nstages, int groups,
                    int diag, const __grid_constant__ CUtensorMap ent_map,
                    const __grid_constant__ CUtensorMap pair_map, int use_tmap) {
  extern __shared__ __align__(128) unsigned char smem[];
#if !STRAIT_SWEEP_DIAG_BUILD
  diag = 0;  // the timing diagnostics (STRAIT_SWEEP_DIAG) exist only in a -DSTRAIT_SWEEP_DIAG_BUILD=1 build
#endif
  const TileGeom tg(SG ? SG : a.gpus_per_segment, C);
  const WsLayout<NM> W(tg, nstages);
  const StageLayout<NM>& L = W.st;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_cons = 8 * groups;
  const int64_t ntiles = a.n_segments / tg.spb;
  uint64_t* full = (uint64_t*)(smem + W.full);
  uint64_t* empty = (uint64_t*)(smem + W.empty);
  const int ncand = tg.spb * StageLayout<NM>::kCandF;

  BulkCopy* ctab = (BulkCopy*)(smem + W.copies);
  ulonglong2* etab = (ulonglong2*)(smem + W.etab);
  for (int i = threadIdx.x; i < 128; i += blockDim.x) etab[i] = __ldg((const ulonglong2*)glibc::kExpTab + i);
  if (threadIdx.x == 0) {
    ((Pred<NM>*)(smem + W.pred))->load(a.params, a.effect_cap);
#if STRAIT_LIBM
    ((Pred<NM>*)(smem + W.pred))->etab = etab;
#endif
    build_copy_table<NM, C>(a, tg, L, ctab);
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 32);  // the producer warp's cp.async arrivals; bulk bytes via expect_tx
      mbar_init(&empty[s], 8);
      *(int*)(smem + s * W.stage_bytes + W.cnt) = 0;
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == n_cons + 1) {  // ---------------------------------------------- refit warp
    if (with_refit && blockIdx.x == 0) refit_warp<NM>(r, (double*)(smem + W.refit));
    return;
  }
  if (warp == n_cons) {  // ------------------------------------------------- producer warp
    const uint64_t pol = l2_evict_first_policy();
    if (use_tmap && lane == 0) {
      prefetch_tmap(&ent_map);
      prefetch_tmap(&pair_map);
    }
    int64_t tile = blockIdx.x;
    // stage index and ring pass kept incrementally (a 64-bit k % nstages costs ~26 instructions)
    int st = 0;
    uint32_t use = 0;
    for (int64_t k = 0; tile < ntiles; ++k, tile += gridDim.x, st = st + 1 < nstages ? st + 1 : (++use, 0)) {
      unsigned char* stage = smem + st * W.stage_bytes;
      mbar_wait(&empty[st], (use & 1) ^ 1);
      if ((diag & 4) && k >= nstages) {
        // diagnostic: compute only — after the first fill the stages keep their data
      } else if (lane == 0 && use_tmap) {
        // packed SoA: two 2-D boxes ([2NM+5] x TT triple fields, [2NM+2] x TP pair fields) + 2 byte arrays
        mbar_expect_tx(&full[st], (uint32_t)L.tx_bytes);
        tma_2d_g2s(stage + L.ent, &ent_map, (int)(tile * tg.TT), 0, &full[st], pol);
        tma_2d_g2s(stage + L.pair, &pair_map, (int)(tile * tg.TP), 0, &full[st], pol);
        const BulkCopy& e = ctab[2 * NM + 5];
        bulk_g2s(stage + e.dst, e.src0 + tile * e.stride, e.bytes, &full[st], pol);
        const BulkCopy& n = ctab[n_bulk_copies<NM>() - 1];
        bulk_g2s(stage + n.dst, n.src0 + tile * n.stride, n.bytes, &full[st], pol);
      } else if (lane == 0) {
        mbar_expect_tx(&full[st], (uint32_t)L.tx_bytes);
        for (int i = 0; i < n_bulk_copies<NM>(); ++i) {
          const BulkCopy cp = ctab[i];
          if (diag & 1) bulk_g2s_nohint(stage + cp.dst, cp.src0 + tile * cp.stride, cp.bytes, &full[st]);
          else bulk_g2s(stage + cp.dst, cp.src0 + tile * cp.stride, cp.bytes, &full[st], pol);
        }
      }
      // candidate values (8 B per field and segment) and the aligned words holding the priorities
      for (int i = lane; i < ncand + tg.spb; i += 32) {
        if (i < ncand) {
          const int f = i / tg.spb, sl = i - f * tg.spb;
          const int64_t s = tile * tg.spb + sl;
          const double* src = f < NM ? a.cand_contrib + f * a.n_segments + s
                            : f == NM ? a.cand_self_cmp + s : f == NM + 1 ? a.cand_self_mem + s
                            : f == NM + 2 ? a.cand_total + s : f == NM + 3 ? a.cand_kernel + s
                            : f == NM + 4 ? a.cand_front + s : a.cand_deadline + s;
          cp_async_8((double*)(stage + L.cand) + i, src);
        } else {
          const int64_t s = tile * tg.spb + (i - ncand);
          cp_async_4((uint32_t*)(stage + L.cprio) + (i - ncand), a.cand_prio + (s & ~int64_t(3)));
        }
      }
      cp_async_mbar_arrive_noinc(&full[st]);  // one of the 32 expected arrivals per phase
    }
    return;
  }

  // ------------------------------------------------------------------------ consumer warps
  const int group = warp >> 3, wg = warp & 7;
  const int local = wg * 32 + lane;  // triple within the tile
  const bool active = local < tg.TT;
  const int sl = active ? local / tg.span : 0;
  const int rr = local - sl * tg.span;
  const int g = rr / C;
  const int c = rr - g * C;
  const int pl = sl * tg.G + g;
  const int TP = tg.TP, TT = tg.TT, spb = tg.spb, G = tg.G;
  const double now = a.now;
  const Pred<NM> pr = *(const Pred<NM>*)(smem + W.pred);  // in registers for the tile loop
  const double nan = __longlong_as_double(0x7ff8000000000000LL);

  int64_t tile = blockIdx.x + (int64_t)group * gridDim.x;
  const int64_t tile_step = (int64_t)groups * gridDim.x;
  // st = k % nstages and use = k / nstages for k = group, group + groups, ...,
  // kept incrementally (groups <= nstages: at most one wrap per step)
  int st = group % nstages;
  uint32_t use = (uint32_t)(group / nstages);
  for (; tile < ntiles;
       tile += tile_step, st = st + groups < nstages ? st + groups : (++use, st + groups - nstages)) {
    unsigned char* stage = smem + st * W.stage_bytes;
    mbar_wait(&full[st], use & 1);
    if (diag & 2) {  // diagnostic: data movement only
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      continue;
    }

    const double* ent = (const double*)(stage + L.ent);
    const double* pair = (const double*)(stage + L.pair);
    const double* cand = (const double*)(stage + L.cand);
    double* s_lat = (double*)(stage + W.res_lat);
    double* s_intf = (double*)(stage + W.res_intf);
    uint8_t* s_adm = (uint8_t*)(stage + W.res_adm);

    // ---- 1. triple projection (scheduler.py:137-160) ----
    const int nrun = active ? ((const int8_t*)(stage + L.nrun))[pl] : 0;
    const int cprio = active ? ((const int8_t*)(stage + L.cprio))[4 * sl + (int)((tile * spb + sl) & 3)] : 0;
    const int eprio = active ? ((const int8_t*)(stage + L.eprio))[local] : 0;
    // check_violate answers True at the LOW candidate's AIMD-cap test before it
    // reads any co-runner (scheduler.py:129-135): such pairs project nothing.
    // This test only skips work, so it may be conservative: it compares against
    // an upper bound of cap_pct / 100 (one multiply, not a division on the path
    // to the projection); the pair lanes below apply the exact test, and the
    // pair's flag is the exact test OR the projections.
    bool capv = false;
    if (active && cprio == 1) {
      const double cap = pair[(2 * NM) * TP + pl];
      const double cap_hi = cap >= 0.0 ? cap * kCapFractionHi : __longlong_as_double(0x7ff8000000000000LL);
#pragma unroll
      for (int m = 0; m < NM; ++m) capv |= pair[(NM + m) * TP + pl] + cand[m * spb + sl] > cap_hi;
    }
    bool viol = false;
    if (active && c < nrun && eprio <= cprio && !capv && !(diag & 8)) {  // diag 8: skip the projections (timing only)
      double tw[NM], nagg[NM];
#pragma unroll
      for (int m = 0; m < NM; ++m) tw[m] = ent[(NM + m) * TT + local];
      const double cmp = ent[(2 * NM + 0) * TT + local], mem = ent[(2 * NM + 1) * TT + local];
      const double tk = ent[(2 * NM + 2) * TT + local], ks = ent[(2 * NM + 4) * TT + local];
#pragma unroll
      for (int m = 0; m < NM; ++m) nagg[m] = pair[m * TP + pl] - ent[m * TT + local] + cand[m * spb + sl];
      double intf_cur, intf_new;  // current progress under the TWA co-location; the candidate joining
#if STRAIT_LIBM
      pr.predict2(tw, nagg, cmp, mem, eprio, intf_cur, intf_new);
#else
      intf_cur = pr.predict(tw, cmp, mem, eprio);
      intf_new = pr.predict(nagg, cmp, mem, eprio);
#endif
      const double elapsed = py_max(0.0, now - ks);
      const double denom = intf_cur * tk;
      const double progress = denom > 0 ? py_min(1.0, elapsed / denom) : 1.0;
      const double remaining = (1.0 - progress) * tk * intf_new;
      const double projected = py_max(now, ks) + remaining;
      viol = projected > ent[(2 * NM + 3) * TT + local];
    }
    unsigned vbits = viol ? 1u : 0u;
#pragma unroll
    for (int o = C / 2; o > 0; o >>= 1) vbits |= __shfl_xor_sync(0xffffffffu, vbits, o, C);
    uint8_t* s_viol = (uint8_t*)(stage + W.res_viol);
    if (active && c == 0) s_viol[pl] = vbits != 0;
    // The tile's projections are published on a named barrier of the group's 8
    // consumer warps. Only the pair warps wait on it (bar.sync); the others
    // arrive (bar.arrive), release the stage and go on to their next tile, so the
    // pair / argmin phases of tile k overlap the projections of tile k+1. There is
    // one barrier per (group, stage): a stage, and with it its barrier, is reused
    // only after every warp has released it, so arrivals never mix generations.
    const int npw = (TP + 31) >> 5;
    const int bar1 = 1 + group * kMaxStages + st;
    if (wg >= npw) {
      asm volatile("bar.arrive %0, %1;" ::"r"(bar1), "r"(8 * 32) : "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      continue;
    }

    // ---- 2. pair: LP cap + check_meet, one lane per pair on the first ceil(TP/32) warps ----
    // Neither reads the projections, so the pair lanes run both BEFORE waiting
    // for the tile's projections (the wait is then mostly hidden), then read the
    // projections' violate bits and release the stage: the producer refills it
    // while the argmin runs (it only touches the stage's result area, which TMA
    // never writes and which only these warps use, in tile order).
    {
      const int pp = wg * 32 + lane;
      const bool pact = pp < TP;
      const int psl = pact ? pp / G : 0;
      int pn = 0, pprio = 0;
      bool capx = false, ok = false;
      double lat = nan, intf = nan;
      if (pact) {
        pn = ((const int8_t*)(stage + L.nrun))[pp];
        pprio = ((const int8_t*)(stage + L.cprio))[4 * psl + (int)((tile * spb + psl) & 3)];
        if (pprio == 1) {  // LOW candidate vs the AIMD cap (scheduler.py:130-135), exact
          const double cap_fraction = pair[(2 * NM) * TP + pp] / 100.0;  // runtime.py:39-40
#pragma unroll
          for (int m = 0; m < NM; ++m)
            if (pair[(NM + m) * TP + pp] + cand[m * spb + psl] > cap_fraction) capx = true;
        }
        if (pn < a.concurrency_limit) {  // has_slot (runtime.py:101-102), then check_meet
          double assumed[NM];  // half the GPU aggregate (scheduler.py:178)
#pragma unroll
          for (int m = 0; m < NM; ++m) assumed[m] = 0.5 * pair[m * TP + pp];
          const double cmp = cand[(NM + 0) * spb + psl], mem = cand[(NM + 1) * spb + psl];
          intf = (diag & 16) ? assumed[0]  // diag 16: skip check_meet's prediction (timing only)
                             : pr.predict(assumed, cmp, mem, pprio);
          const double wait = py_max(0.0, pair[(2 * NM + 1) * TP + pp] - now);  // pcie.py:21-23
          lat = cand[(NM + 2) * spb + psl] + wait + (intf - 1.0) * cand[(NM + 3) * spb + psl] +
                (now - cand[(NM + 4) * spb + psl]);
          ok = lat <= cand[(NM + 5) * spb + psl];
        }
      }
      asm volatile("bar.sync %0, %1;" ::"r"(bar1), "r"(8 * 32) : "memory");  // the tile's projections
      const bool violate = pact && (capx || s_viol[pp] != 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);  // the TMA region of this stage is free
      if (pact) {
        uint8_t flags = 0;
        bool admitted = false;
        if (pn < a.concurrency_limit) {
          flags |= STRAIT_PAIR_HAS_SLOT;
          if (violate) flags |= STRAIT_PAIR_VIOLATE;
          if (ok) flags |= STRAIT_PAIR_MEET;
          admitted = !(a.use_violate && violate) && !(a.use_meet && !ok);
          if (admitted) flags |= STRAIT_PAIR_FEASIBLE;
        }
        const int64_t p = tile * TP + pp;
        if (a.pair_flags) a.pair_flags[p] = flags;
        if (a.pair_latency) __stcs(a.pair_latency + p, lat);
        if (a.pair_intf) __stcs(a.pair_intf + p, intf);
        s_lat[pp] = lat;
        s_intf[pp] = intf;
        s_adm[pp] = admitted;
      }
      if (npw > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + kMaxGroups * kMaxStages + group), "r"(npw * 32) : "memory");
    }

    // ---- 3. warp 0: best_for argmin per segment ----
    const int last = wg == 0;
    if (last) {
      for (int q = 0; q < spb; ++q) {
        ArgminKey key{INT_MAX, 0.0, INT_MAX, 0.0};
        for (int gg = lane; gg < G; gg += 32) {
          const int qp = q * G + gg;
          if (!s_adm[qp]) continue;
          const double lt = s_lat[qp];
          ArgminKey en{gg, lt, INT_MAX, 0.0};
          if (!isnan(lt)) {
            en.best_g = gg;
            en.best_lat = lt;
          }
          key = argmin_combine(key, en);
        }
        key = argmin_warp(key);
        if (lane == 0) {
          const int64_t s = tile * spb + q;
          int bg = -1;
          if (key.first_g != INT_MAX) bg = isnan(key.first_lat) ? key.first_g : key.best_g;
          a.seg_gpu[s] = bg;
          a.seg_latency[s] = bg >= 0 ? s_lat[q * G + bg] : nan;
          a.seg_intf[s] = bg >= 0 ? s_intf[q * G + bg] : nan;
        }
      }
    }
    // (the stage was released before the meet predictions; the result area is
    // next written by these same warps, for tile + nstages, in program order)
    __syncwarp();
  }
}

template <int NM>
__global__ void refit_kernel(const StraitRefitArgs r) {
  __shared__ double sP[kMaxP];
  refit_warp<NM>(r, sP);
}

template <int NM>
__global__ void predict_kernel(const double* __restrict__ P, double cap, const double* __restrict__ coloc,
                               const double* __restrict__ cmp, const double* __restrict__ mem,
                               const int8_t* __restrict__ prio, int64_t n, double* __restrict__ out_x,
                               double* __restrict__ out_eff, double* __restrict__ out,
                               uint8_t* __restrict__ sat) {
  Pred<NM> pr;
  pr.load(P, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double a[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) a[m] = coloc[m * n + i];
    const int p = prio[i];
    bool s;
    const double x = pr.exponent(a, cmp[i], mem[i]);
    const double eff = pr.effect(x, s);
    if (out_x) out_x[i] = x;
    if (out_eff) out_eff[i] = eff;
    if (out) out[i] = 1.0 + eff * (p == 0 ? pr.coeff[0] : pr.coeff[1]);
    if (sat) sat[i] = s;
  }
}

template <int NM>
__global__ void latency_kernel(const double* __restrict__ P, double cap, const double* __restrict__ assumed,
                               const double* __restrict__ cmp, const double* __restrict__ mem,
                               const int8_t* __restrict__ prio, const double* __restrict__ total,
                               const double* __restrict__ kernel, const double* __restrict__ t_avail,
                               const double* __restrict__ front, const double* __restrict__ now, int64_t n,
                               double* __restrict__ out_lat, double* __restrict__ out_intf) {
  Pred<NM> pr;
  pr.load(P, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double a[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) a[m] = assumed[m * n + i];
    const double intf = pr.predict(a, cmp[i], mem[i], prio[i]);
    const double t = now[i];
    out_lat[i] = total[i] + py_max(0.0, t_avail[i] - t) + (intf - 1.0) * kernel[i] + (t - front[i]);
    if (out_intf) out_intf[i] = intf;
  }
}

template <int NM>
__global__ void effect_kernel(const double* __restrict__ P, double cap, const double* __restrict__ x, int64_t n,
                              double* __restrict__ out, uint8_t* __restrict__ sat) {
  Pred<NM> pr;
  pr.load(P, cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    bool s;
    out[i] = pr.effect(x[i], s);
    if (sat) sat[i] = s;
  }
}

template <int NM>
__global__ void twa_kernel(const double* __restrict__ t0, const double* __restrict__ tl,
                           const double* __restrict__ vl, const double* __restrict__ acc,
                           const double* __restrict__ end, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double e = end[i];
    const double total = e - t0[i];
    const double d = e - tl[i];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const double v = vl[m * n + i];
      out[m * n + i] = total <= 0.0 ? v : (acc[m * n + i] + v * d) / total;
    }
  }
}

// ----------------------------------------------------------------------------- launchers

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

// TMA eligibility: whole tiles, 16-byte aligned chunk offsets and sizes.
static bool tma_eligible(const StraitSweepArgs& a, const TileGeom& tg) {
  if (a.n_segments % tg.spb || a.n_segments % 4) return false;
  if (!aligned16(a.cand_prio)) return false;
  if (tg.TT % 16 || tg.TP % 16) return false;
  const void* ptrs[] = {a.ent_contrib, a.ent_twa, a.ent_self_cmp, a.ent_self_mem, a.ent_t_kernel,
                        a.ent_deadline_abs, a.ent_kstart, a.ent_prio, a.gpu_agg, a.gpu_lp_agg,
                        a.gpu_cap_pct, a.gpu_t_avail, a.gpu_n_running};
  for (const void* q : ptrs)
    if (!aligned16(q)) return false;
  return true;
}

static int g_last_sweep_path = 0;  // 1 sync, 2 bulk-copy pipeline, 3 tensor-map pipeline

static PFN_cuTensorMapEncodeTiled encode_fn() {
  static PFN_cuTensorMapEncodeTiled fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled)p;
  }
  return fn;
}

// Rows base, base + stride, ... (nrows arrays of `n` doubles) as one 2-D tensor map with a
// box of `box` columns x nrows rows.  Returns false if the arrays are not uniformly packed.
static bool encode_rows(CUtensorMap* map, const double* const* rows, int nrows, int64_t n, int box) {
  const int64_t stride = rows[1] - rows[0];
  if (stride < n || n >= (1LL << 31)) return false;
  for (int i = 1; i < nrows; ++i)
    if (rows[i] - rows[i - 1] != stride) return false;
  if (((uintptr_t)rows[0] & 15) || (stride * 8) % 16) return false;
  PFN_cuTensorMapEncodeTiled enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)nrows};
  cuuint64_t strides[1] = {(cuuint64_t)(stride * 8)};
  cuuint32_t boxd[2] = {(cuuint32_t)box, (cuuint32_t)nrows};
  cuuint32_t es[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)rows[0], dims, strides, boxd, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NM>
static bool packed_tensor_maps(const StraitSweepArgs& a, const TileGeom& tg, CUtensorMap* ent, CUtensorMap* pair) {
  const int64_t Pn = a.n_segments * tg.G, Tn = Pn * tg.C;
  const double* er[2 * NM + 5];
  for (int m = 0; m < NM; ++m) er[m] = a.ent_contrib + m * Tn, er[NM + m] = a.ent_twa + m * Tn;
  er[2 * NM] = a.ent_self_cmp, er[2 * NM + 1] = a.ent_self_mem, er[2 * NM + 2] = a.ent_t_kernel;
  er[2 * NM + 3] = a.ent_deadline_abs, er[2 * NM + 4] = a.ent_kstart;
  // the metric-major fields are themselves rows of stride Tn: require one uniform stride
  const double* pr[2 * NM + 2];
  for (int m = 0; m < NM; ++m) pr[m] = a.gpu_agg + m * Pn, pr[NM + m] = a.gpu_lp_agg + m * Pn;
  pr[2 * NM] = a.gpu_cap_pct, pr[2 * NM + 1] = a.gpu_t_avail;
  return encode_rows(ent, er, 2 * NM + 5, Tn, tg.TT) && encode_rows(pair, pr, 2 * NM + 2, Pn, tg.TP);
}

template <int NM, int C>
static int launch_sweep_c(const StraitSweepArgs& a, cudaStream_t st, const StraitRefitArgs* r) {
  const TileGeom tg(a.gpus_per_segment, C);
  const StageLayout<NM> L(tg);
  const int with_refit = r ? 1 : 0;
  StraitRefitArgs rr = r ? *r : StraitRefitArgs{};
  const int force = env_int("STRAIT_SWEEP_PATH", 0);  // 0 auto, 1 sync, 3 bulk copies without tensor maps
  const bool use_tma = force == 1 ? false : tma_eligible(a, tg);
  if (use_tma) {
    int groups = env_int("STRAIT_SWEEP_GROUPS", 1);
    groups = groups < 1 ? 1 : (groups > kMaxGroups ? kMaxGroups : groups);
    int ns = env_int("STRAIT_SWEEP_STAGES", 2);
    ns = ns < 2 ? 2 : (ns > kWsMaxStages ? kWsMaxStages : ns);
    const WsLayout<NM> WL(tg, ns);
    const size_t smem = WL.bytes;
    auto kern = sweep_ws_kernel<NM, C, 0>;
    if constexpr (NM == 5) {  // the profiled shape: static one-segment tiles
      if (tg.span == 256) kern = sweep_ws_kernel<NM, C, 256 / C>;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return set_error(STRAIT_ECUDA, "strait_sweep: %zu B shared memory per CTA unavailable", smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    const int threads = 32 * (8 * groups + 2);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (occ < 1) occ = 1;
    const int64_t ntiles = a.n_segments / tg.spb;
    int64_t grid = (int64_t)sm_count() * occ;
    const int cap = env_int("STRAIT_SWEEP_GRID", 0);
    if (cap > 0 && cap < grid) grid = cap;
    if (grid > ntiles) grid = ntiles;
    if (grid < 1) grid = 1;
    CUtensorMap ent_map, pair_map;
    memset(&ent_map, 0, sizeof ent_map);
    memset(&pair_map, 0, sizeof pair_map);
    const int use_tmap = force != 3 && packed_tensor_maps<NM>(a, tg, &ent_map, &pair_map) ? 1 : 0;
    kern<<<(unsigned)grid, threads, smem, st>>>(a, rr, with_refit, ns, groups, env_int("STRAIT_SWEEP_DIAG", 0),
                                                ent_map, pair_map, use_tmap);
    g_last_sweep_path = use_tmap ? 3 : 2;
  } else {
    const CtaLayout<NM> CL(tg, L, 1);
    const size_t smem = CL.bytes;
    auto kern = sweep_sync_kernel<NM, C>;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return set_error(STRAIT_ECUDA, "strait_sweep: %zu B shared memory per CTA unavailable", smem);
    int64_t grid = (a.n_segments + tg.spb - 1) / tg.spb;
    if (with_refit && grid < 1) grid = 1;
    kern<<<(unsigned)grid, kSweepThreads + (with_refit ? 32 : 0), smem, st>>>(a, rr, with_refit);
    g_last_sweep_path = 1;
  }
  return STRAIT_OK;
}

template <int NM>
static void launch_sweep_nm(const StraitSweepArgs& a, cudaStream_t st, const StraitRefitArgs* r, int* rc) {
  switch (a.n_slots) {
    case 1: *rc = launch_sweep_c<NM, 1>(a, st, r); break;
    case 2: *rc = launch_sweep_c<NM, 2>(a, st, r); break;
    case 4: *rc = launch_sweep_c<NM, 4>(a, st, r); break;
    case 8: *rc = launch_sweep_c<NM, 8>(a, st, r); break;
    case 16: *rc = launch_sweep_c<NM, 16>(a, st, r); break;
    case 32: *rc = launch_sweep_c<NM, 32>(a, st, r); break;
    default: *rc = set_error(STRAIT_EINVAL, "bad n_slots"); break;
  }
}

static int validate_sweep(const StraitSweepArgs* a) {
  if (!a) return set_error(STRAIT_EINVAL, "sweep args is NULL");
  if (a->n_metrics < 1 || a->n_metrics > STRAIT_MAX_METRICS)
    return set_error(STRAIT_EINVAL, "aggregate throughput has %d metrics, supported 1..%d", a->n_metrics,
                     STRAIT_MAX_METRICS);
  const int C = a->n_slots;
  if (C < 1 || C > 32 || (C & (C - 1)))
    return set_error(STRAIT_EINVAL, "n_slots must be a power of two <= 32, got %d", C);
  if (a->gpus_per_segment < 1) return set_error(STRAIT_EINVAL, "gpus_per_segment must be >= 1");
  if ((int64_t)a->gpus_per_segment * C > kSweepThreads)
    return set_error(STRAIT_EINVAL, "gpus_per_segment * n_slots must be <= %d, got %d * %d", kSweepThreads,
                     a->gpus_per_segment, C);
  if (a->n_segments < 0) return set_error(STRAIT_EINVAL, "n_segments must be >= 0");
  if (!a->params || !a->seg_gpu || !a->seg_latency || !a->seg_intf)
    return set_error(STRAIT_EINVAL, "params and seg_* outputs are required");
  return STRAIT_OK;
}

static int validate_refit(const StraitRefitArgs* r) {
  if (!r) return set_error(STRAIT_EINVAL, "refit args is NULL");
  if (r->n_metrics < 1 || r->n_metrics > STRAIT_MAX_METRICS)
    return set_error(STRAIT_EINVAL, "expected 1..%d metrics, got %d", STRAIT_MAX_METRICS, r->n_metrics);
  if (r->n < 0 || !r->state || !r->step) return set_error(STRAIT_EINVAL, "refit state/step required");
  if (r->n_bc < 0 || (r->n_bc > 0 && (!r->bc1 || !r->bc2)))
    return set_error(STRAIT_EINVAL, "bias-correction tables required");
  return STRAIT_OK;
}

template <int NM>
static void launch_refit_nm(const StraitRefitArgs& r, cudaStream_t st) {
  refit_kernel<NM><<<1, 32, 0, st>>>(r);
}

static unsigned ew_grid(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

template <int NM>
static void launch_predict_nm(const double* P, double cap, const double* coloc, const double* cmp,
                              const double* mem, const int8_t* prio, int64_t n, double* out_x, double* out_eff,
                              double* out, uint8_t* sat, cudaStream_t st) {
  predict_kernel<NM><<<ew_grid(n), 256, 0, st>>>(P, cap, coloc, cmp, mem, prio, n, out_x, out_eff, out, sat);
}

template <int NM>
static void launch_latency_nm(const double* P, double cap, const double* assumed, const double* cmp,
                              const double* mem, const int8_t* prio, const double* total, const double* kernel,
                              const double* t_avail, const double* front, const double* now, int64_t n,
                              double* out_lat, double* out_intf, cudaStream_t st) {
  latency_kernel<NM><<<ew_grid(n), 256, 0, st>>>(P, cap, assumed, cmp, mem, prio, total, kernel, t_avail,
                                                  front, now, n, out_lat, out_intf);
}

}  // namespace strait

using namespace strait;

extern "C" int strait_sweep(const StraitSweepArgs* a, void* stream) {
  if (int e = validate_sweep(a)) return e;
  if (a->n_segments == 0) return STRAIT_OK;
  int rc = STRAIT_OK;
  STRAIT_DISPATCH_NM(a->n_metrics, launch_sweep_nm, *a, (cudaStream_t)stream, nullptr, &rc);
  if (rc) return rc;
  return check_launch("strait_sweep");
}

extern "C" int strait_round(const StraitSweepArgs* a, const StraitRefitArgs* r, void* stream) {
  if (int e = validate_sweep(a)) return e;
  if (int e = validate_refit(r)) return e;
  if (r->n_metrics != a->n_metrics) return set_error(STRAIT_EINVAL, "sweep/refit metric count mismatch");
  if ((const void*)r->state == (const void*)a->params)
    return set_error(STRAIT_EINVAL, "refit state must not alias the sweep parameters");
  int rc = STRAIT_OK;
  STRAIT_DISPATCH_NM(a->n_metrics, launch_sweep_nm, *a, (cudaStream_t)stream, r, &rc);
  if (rc) return rc;
  return check_launch("strait_round");
}

extern "C" int strait_refit(const StraitRefitArgs* r, void* stream) {
  if (int e = validate_refit(r)) return e;
  if (r->n == 0) return STRAIT_OK;
  STRAIT_DISPATCH_NM(r->n_metrics, launch_refit_nm, *r, (cudaStream_t)stream);
  return check_launch("strait_refit");
}

extern "C" int strait_predict(const double* params, int32_t nm, double cap, const double* coloc,
                              const double* self_cmp, const double* self_mem, const int8_t* prio, int64_t n,
                              double* out, uint8_t* sat, void* stream) {
  if (nm < 1 || nm > STRAIT_MAX_METRICS)
    return set_error(STRAIT_EINVAL, "aggregate throughput has %d metrics, supported 1..%d", nm, STRAIT_MAX_METRICS);
  if (n < 0) return set_error(STRAIT_EINVAL, "n must be >= 0");
  if (n == 0) return STRAIT_OK;
  STRAIT_DISPATCH_NM(nm, launch_predict_nm, params, cap, coloc, self_cmp, self_mem, prio, n, nullptr, nullptr,
                     out, sat, (cudaStream_t)stream);
  return check_launch("strait_predict");
}

template <int NM>
static void launch_effect_nm(const double* P, double cap, const double* x, int64_t n, double* out, uint8_t* sat,
                             cudaStream_t st) {
  effect_kernel<NM><<<ew_grid(n), 256, 0, st>>>(P, cap, x, n, out, sat);
}

extern "C" int strait_kernel_effect(const double* params, int32_t nm, double cap, const double* x, int64_t n,
                                    double* out, uint8_t* sat, void* stream) {
  if (nm < 1 || nm > STRAIT_MAX_METRICS) return set_error(STRAIT_EINVAL, "bad metric count %d", nm);
  if (n < 0) return set_error(STRAIT_EINVAL, "n must be >= 0");
  if (n == 0) return STRAIT_OK;
  STRAIT_DISPATCH_NM(nm, launch_effect_nm, params, cap, x, n, out, sat, (cudaStream_t)stream);
  return check_launch("strait_kernel_effect");
}

template <int NM>
static void launch_twa_nm(const double* t0, const double* tl, const double* vl, const double* acc, const double* end,
                          int64_t n, double* out, cudaStream_t st) {
  twa_kernel<NM><<<ew_grid(n), 256, 0, st>>>(t0, tl, vl, acc, end, n, out);
}

extern "C" int strait_twa(int32_t nm, const double* t0, const double* tl, const double* vl, const double* acc,
                          const double* end, int64_t n, double* out, void* stream) {
  if (nm < 1 || nm > STRAIT_MAX_METRICS) return set_error(STRAIT_EINVAL, "bad metric count %d", nm);
  if (n < 0) return set_error(STRAIT_EINVAL, "n must be >= 0");
  if (n == 0) return STRAIT_OK;
  STRAIT_DISPATCH_NM(nm, launch_twa_nm, t0, tl, vl, acc, end, n, out, (cudaStream_t)stream);
  return check_launch("strait_twa");
}

extern "C" int strait_predict_parts(const double* params, int32_t nm, double cap, const double* coloc,
                                    const double* self_cmp, const double* self_mem, const int8_t* prio, int64_t n,
                                    double* out_x, double* out_eff, double* out, uint8_t* sat, void* stream) {
  if (nm < 1 || nm > STRAIT_MAX_METRICS)
    return set_error(STRAIT_EINVAL, "aggregate throughput has %d metrics, supported 1..%d", nm, STRAIT_MAX_METRICS);
  if (n < 0) return set_error(STRAIT_EINVAL, "n must be >= 0");
  if (n == 0) return STRAIT_OK;
  STRAIT_DISPATCH_NM(nm, launch_predict_nm, params, cap, coloc, self_cmp, self_mem, prio, n, out_x, out_eff, out,
                     sat, (cudaStream_t)stream);
  return check_launch("strait_predict_parts");
}

extern "C" int strait_estimate_latency(const double* params, int32_t nm, double cap, const double* assumed,
                                       const double* self_cmp, const double* self_mem, const int8_t* prio,
                                       const double* total, const double* kernel, const double* t_avail,
                                       const double* front, const double* now, int64_t n, double* out_lat,
                                       double* out_intf, void* stream) {
  if (nm < 1 || nm > STRAIT_MAX_METRICS)
    return set_error(STRAIT_EINVAL, "aggregate throughput has %d metrics, supported 1..%d", nm, STRAIT_MAX_METRICS);
  if (n < 0) return set_error(STRAIT_EINVAL, "n must be >= 0");
  if (n == 0) return STRAIT_OK;
  STRAIT_DISPATCH_NM(nm, launch_latency_nm, params, cap, assumed, self_cmp, self_mem, prio, total, kernel,
                     t_avail, front, now, n, out_lat, out_intf, (cudaStream_t)stream);
  return check_launch("strait_estimate_latency");
}

extern "C" int strait_last_sweep_path(void) { return g_last_sweep_path; }
