// strait_rng.cuh — the reference's random streams on the device, draw for draw
// identical to numpy 2.3 (the generator behind workload.py:19-152 and the
// batch noise, simulation.py:163,309-311):
//   SeedSequence (mix_entropy + generate_state(4, uint64)) -> PCG64 XSL-RR
//   128/64 -> ziggurat standard exponential / normal (distributions.c) with
//   numpy's tables (strait_rng_tables.cuh) and the reference host's exp/log1p
//   (strait_libm.cuh).  numpy's distribution code is built without FMA, so the
//   library's --fmad=false gives the same roundings.
#pragma once

#include <stdint.h>

#include "strait_libm.cuh"
#include "strait_rng_tables.cuh"

namespace strait {
namespace rng {

typedef unsigned __int128 u128;

// SeedSequence(entropy).generate_state(4, np.uint64); entropy words < 2^64
__device__ __forceinline__ void seedseq_state(const uint64_t* entropy, int n_entropy, uint64_t out[4]) {
  constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
  uint32_t words[8];
  int nw = 0;
  for (int i = 0; i < n_entropy && nw < 8; ++i) {
    const uint64_t v = entropy[i];
    words[nw++] = (uint32_t)v;
    if ((v >> 32) && nw < 8) words[nw++] = (uint32_t)(v >> 32);
  }
  uint32_t hc = INIT_A;
  auto hashmix = [&](uint32_t value) {
    value ^= hc;
    hc *= MULT_A;
    value *= hc;
    value ^= value >> 16;
    return value;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = MIX_L * x - MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nw ? words[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < nw; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(words[s]));
  uint32_t hb = INIT_B, st[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)st[2 * i] | ((uint64_t)st[2 * i + 1] << 32);
}

struct Pcg64 {
  u128 state, inc;
  __device__ __forceinline__ void step() {
    const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    state = state * mult + inc;
  }
  // numpy PCG64(SeedSequence): pcg64_set_seed(state = v[0]:v[1], inc = v[2]:v[3])
  __device__ __forceinline__ void seed(const uint64_t* entropy, int n_entropy) {
    uint64_t v[4];
    seedseq_state(entropy, n_entropy, v);
    state = 0;
    inc = ((((u128)v[2] << 64) | v[3]) << 1) | 1;
    step();
    state += ((u128)v[0] << 64) | v[1];
    step();
  }
  __device__ __forceinline__ uint64_t next64() {
    step();
    const uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    const unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  __device__ __forceinline__ double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
};

__device__ __forceinline__ double tab(const uint64_t* t, int i) { return __longlong_as_double((long long)__ldg(&t[i])); }

// random_standard_exponential (distributions.c)
__device__ __forceinline__ double std_exponential(Pcg64& r) {
  constexpr double ziggurat_exp_r = 7.6971174701310497140446280481;
  for (;;) {
    uint64_t ri = r.next64();
    ri >>= 3;
    const int idx = (int)(ri & 0xFF);
    ri >>= 8;
    const double x = (double)ri * tab(zig::kWe, idx);
    if (ri < __ldg(&zig::kKe[idx])) return x;
    if (idx == 0) return ziggurat_exp_r - glibc::log1p(-r.next_double());
    if ((tab(zig::kFe, idx - 1) - tab(zig::kFe, idx)) * r.next_double() + tab(zig::kFe, idx) < glibc::exp(-x))
      return x;
  }
}

// random_standard_normal (distributions.c)
__device__ __forceinline__ double std_normal(Pcg64& r) {
  constexpr double ziggurat_nor_r = 3.6541528853610087963519472518;
  constexpr double ziggurat_nor_inv_r = 0.27366123732975827203338247596;
  for (;;) {
    uint64_t rr = r.next64();
    const int idx = (int)(rr & 0xff);
    rr >>= 8;
    const int sign = (int)(rr & 0x1);
    const uint64_t rabs = (rr >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * tab(zig::kWi, idx);
    if (sign & 0x1) x = -x;
    if (rabs < __ldg(&zig::kKi[idx])) return x;
    if (idx == 0) {
      for (;;) {
        const double xx = -ziggurat_nor_inv_r * glibc::log1p(-r.next_double());
        const double yy = -glibc::log1p(-r.next_double());
        if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(ziggurat_nor_r + xx) : ziggurat_nor_r + xx;
      }
    } else {
      if (((tab(zig::kFi, idx - 1) - tab(zig::kFi, idx)) * r.next_double() + tab(zig::kFi, idx)) <
          glibc::exp(-0.5 * x * x))
        return x;
    }
  }
}

}  // namespace rng
}  // namespace strait
