// numpy-exact random streams on the device.
//
// The reference draws all randomness through numpy (embedding.py:56-57
// default_rng([seed, node]).choice; policy.py:235/288 default_rng(seed).random).
// These are the published numpy algorithms (SeedSequence hash mixing, PCG64
// XSL-RR 128/64 "step then output", Lemire bounded draws from the buffered
// next_uint32, Floyd's sampling without replacement), written as __host__
// __device__ functions so every GPU thread can regenerate exactly the draw the
// reference would consume at its position in the stream (PCG64 jump-ahead).
// Spec + tests: oracle/rng.py, tests/test_oracle_golden.py.
#pragma once
#include <stdint.h>

namespace go {

typedef unsigned __int128 u128;

struct SeedSeqConst {
  static constexpr uint32_t INIT_A = 0x43B0D7E5u, MULT_A = 0x931E8875u;
  static constexpr uint32_t INIT_B = 0x8B51F9DDu, MULT_B = 0x58F38DEDu;
  static constexpr uint32_t MIX_L = 0xCA01F9DDu, MIX_R = 0x4973F715u;
};

// Entropy words of a non-negative integer < 2**64, little-endian 32-bit words
// (bit_generator.pyx _int_to_uint32_array): 0 -> [0].
__host__ __device__ inline int int_words(uint64_t x, uint32_t* w) {
  if (x == 0) {
    w[0] = 0;
    return 1;
  }
  int k = 0;
  while (x) {
    w[k++] = (uint32_t)(x & 0xFFFFFFFFu);
    x >>= 32;
  }
  return k;
}

// SeedSequence(entropy).generate_state(4, uint64) for an entropy word list of
// length <= 8 (we only need [seed] and [seed, node]).
__host__ __device__ inline void seedseq_state4(const uint32_t* ent, int nent, uint64_t out[4]) {
  uint32_t hc = SeedSeqConst::INIT_A;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= SeedSeqConst::MULT_A;
    v *= hc;
    v ^= v >> 16;
    return v;
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = SeedSeqConst::MIX_L * x - SeedSeqConst::MIX_R * y;
    r ^= r >> 16;
    return r;
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nent ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  for (int s = 4; s < nent; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s]));
  uint32_t hb = SeedSeqConst::INIT_B;
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= SeedSeqConst::MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

struct Pcg64 {
  u128 state, inc;
  bool has32;
  uint32_t buf32;

  __host__ __device__ static u128 mult() {
    return ((u128)2549297995355413924ull << 64) | (u128)4865540595714422341ull;
  }

  // PCG64(SeedSequence(entropy)) initial state (pcg64.pyx / pcg64_set_seed).
  __host__ __device__ void seed_words(const uint32_t* ent, int nent) {
    uint64_t s[4];
    seedseq_state4(ent, nent, s);
    u128 initstate = ((u128)s[0] << 64) | s[1];
    u128 initseq = ((u128)s[2] << 64) | s[3];
    inc = (initseq << 1) | 1;
    state = 0;
    step();
    state += initstate;
    step();
    has32 = false;
    buf32 = 0;
  }
  __host__ __device__ void seed1(uint64_t seed) {
    uint32_t w[2];
    int k = int_words(seed, w);
    seed_words(w, k);
  }
  __host__ __device__ void seed2(uint64_t a, uint64_t b) {
    uint32_t w[4];
    int k = int_words(a, w);
    k += int_words(b, w + k);
    seed_words(w, k);
  }
  __host__ __device__ void step() { state = state * mult() + inc; }
  __host__ __device__ static uint64_t output(u128 st) {
    uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
    unsigned rot = (unsigned)(hi >> 58);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  __host__ __device__ uint64_t next64() {
    step();
    return output(state);
  }
  __host__ __device__ uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    uint64_t v = next64();
    has32 = true;
    buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  __host__ __device__ double random() {
    return (double)(next64() >> 11) * (1.0 / 9007199254740992.0);
  }
  // Jump ahead `delta` steps (pcg64_advance / LCG power by squaring).
  __host__ __device__ void advance(uint64_t delta) {
    u128 acc_m = 1, acc_p = 0, cur_m = mult(), cur_p = inc;
    while (delta) {
      if (delta & 1) {
        acc_m *= cur_m;
        acc_p = acc_p * cur_m + cur_p;
      }
      cur_p = (cur_m + 1) * cur_p;
      cur_m *= cur_m;
      delta >>= 1;
    }
    state = acc_m * state + acc_p;
  }
  // random_bounded_uint64(off=0, rng, mask=0, use_masked=false), rng < 2**32:
  // buffered Lemire on next_uint32 (distributions.c).
  __host__ __device__ uint32_t bounded(uint32_t rng) {
    if (rng == 0) return 0;
    if (rng == 0xFFFFFFFFu) return next32();
    uint32_t rng_excl = rng + 1;
    uint64_t m = (uint64_t)next32() * rng_excl;
    uint32_t left = (uint32_t)m;
    if (left < rng_excl) {
      uint32_t threshold = (0xFFFFFFFFu - rng) % rng_excl;
      while (left < threshold) {
        m = (uint64_t)next32() * rng_excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

}  // namespace go
