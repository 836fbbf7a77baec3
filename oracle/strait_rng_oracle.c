/*
 * strait_rng_oracle.c — CPU ORACLE (test infrastructure, NOT product code) of
 * the reference's random streams, restating numpy 2.3's algorithms so the
 * device workload generator can be checked draw for draw:
 *   - SeedSequence (numpy/random/bit_generator.pyx: mix_entropy, generate_state)
 *     seeded the way the reference seeds it: SeedSequence([seed, model_index])
 *     per model (workload.py:147-152), [seed, index, minute] per trace minute
 *     (workload.py:75-104), [seed, 1_000_003] for the batch noise
 *     (simulation.py:163);
 *   - PCG64 (XSL-RR 128/64, pcg64.h) seeded from generate_state(4, uint64);
 *   - random_standard_exponential / random_standard_normal (ziggurat,
 *     distributions.c) with the tables of scripts/gen_rng_tables.py and the
 *     host libm's exp / log1p (what numpy calls);
 *   - gen_poisson (workload.py:19-35): t += scale * exponential until t >= duration.
 * Pinned against numpy itself by tests/test_rng.py.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "rng_tables.h"

typedef unsigned __int128 u128;
static const u128 PCG_MULT = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;

/* ---------------------------------------------------------------- SeedSequence */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_XSHIFT 16

static uint32_t ss_hashmix(uint32_t value, uint32_t *hash_const) {
  value ^= *hash_const;
  *hash_const *= SS_MULT_A;
  value *= *hash_const;
  value ^= value >> SS_XSHIFT;
  return value;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> SS_XSHIFT;
  return r;
}

/* entropy: non-negative integers < 2^64, each coerced to 1 or 2 little-endian uint32 words */
void oracle_seedseq_state(const uint64_t *entropy, int n_entropy, uint64_t out[4]) {
  uint32_t words[64];
  int nw = 0;
  for (int i = 0; i < n_entropy; ++i) {
    uint64_t v = entropy[i];
    words[nw++] = (uint32_t)v;
    if (v >> 32) words[nw++] = (uint32_t)(v >> 32);
  }
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < nw ? words[i] : 0u, &hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < nw; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], &hc));
  uint32_t st[8];
  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> SS_XSHIFT;
    st[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
}

/* ---------------------------------------------------------------- PCG64 */
typedef struct {
  u128 state, inc;
} Pcg64;

static void pcg_step(Pcg64 *r) { r->state = r->state * PCG_MULT + r->inc; }
static void pcg_seed(Pcg64 *r, const uint64_t v[4]) {
  u128 initstate = ((u128)v[0] << 64) | v[1], initseq = ((u128)v[2] << 64) | v[3];
  r->state = 0;
  r->inc = (initseq << 1) | 1;
  pcg_step(r);
  r->state += initstate;
  pcg_step(r);
}
static uint64_t pcg_next64(Pcg64 *r) {
  pcg_step(r);
  uint64_t x = (uint64_t)(r->state >> 64) ^ (uint64_t)r->state;
  unsigned rot = (unsigned)(r->state >> 122);
  return (x >> rot) | (x << ((64 - rot) & 63));
}
static double next_double(Pcg64 *r) { return (double)(pcg_next64(r) >> 11) * (1.0 / 9007199254740992.0); }

static double d(uint64_t u) {
  double x;
  memcpy(&x, &u, 8);
  return x;
}

static const double ziggurat_nor_r = 3.6541528853610087963519472518;
static const double ziggurat_nor_inv_r = 0.27366123732975827203338247596;
static const double ziggurat_exp_r = 7.6971174701310497140446280481;

static double std_exponential(Pcg64 *r) {
  for (;;) {
    uint64_t ri = pcg_next64(r);
    ri >>= 3;
    uint8_t idx = ri & 0xFF;
    ri >>= 8;
    double x = (double)ri * d(zig_we[idx]);
    if (ri < zig_ke[idx]) return x;
    if (idx == 0) return ziggurat_exp_r - log1p(-next_double(r));
    if ((d(zig_fe[idx - 1]) - d(zig_fe[idx])) * next_double(r) + d(zig_fe[idx]) < exp(-x)) return x;
  }
}

static double std_normal(Pcg64 *r) {
  for (;;) {
    uint64_t rr = pcg_next64(r);
    int idx = rr & 0xff;
    rr >>= 8;
    int sign = rr & 0x1;
    uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * d(zig_wi[idx]);
    if (sign & 0x1) x = -x;
    if (rabs < zig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -ziggurat_nor_inv_r * log1p(-next_double(r));
        double yy = -log1p(-next_double(r));
        if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(ziggurat_nor_r + xx) : ziggurat_nor_r + xx;
      }
    } else {
      if (((d(zig_fi[idx - 1]) - d(zig_fi[idx])) * next_double(r) + d(zig_fi[idx])) < exp(-0.5 * x * x)) return x;
    }
  }
}

/* ---------------------------------------------------------------- entry points (ctypes) */
void oracle_rng_raw(const uint64_t *entropy, int n_entropy, int64_t n, uint64_t *out) {
  uint64_t st[4];
  Pcg64 r;
  oracle_seedseq_state(entropy, n_entropy, st);
  pcg_seed(&r, st);
  for (int64_t i = 0; i < n; ++i) out[i] = pcg_next64(&r);
}

/* kind 0: scale * standard_exponential, 1: loc + scale * standard_normal */
void oracle_rng_draws(const uint64_t *entropy, int n_entropy, int kind, double loc, double scale, int64_t n,
                      double *out) {
  uint64_t st[4];
  Pcg64 r;
  oracle_seedseq_state(entropy, n_entropy, st);
  pcg_seed(&r, st);
  for (int64_t i = 0; i < n; ++i) out[i] = kind == 0 ? scale * std_exponential(&r) : loc + scale * std_normal(&r);
}

/* gen_poisson (workload.py:19-35); returns the count, writes up to cap times */
int64_t oracle_gen_poisson(const uint64_t *entropy, int n_entropy, double rate_per_s, double duration_ms,
                           double *out, int64_t cap) {
  if (rate_per_s == 0 || duration_ms <= 0) return 0;
  uint64_t st[4];
  Pcg64 r;
  oracle_seedseq_state(entropy, n_entropy, st);
  pcg_seed(&r, st);
  const double mean_gap = 1000.0 / rate_per_s;
  double t = 0.0;
  int64_t n = 0;
  for (;;) {
    t += mean_gap * std_exponential(&r);
    if (t >= duration_ms) return n;
    if (n < cap) out[n] = t;
    n++;
  }
}
