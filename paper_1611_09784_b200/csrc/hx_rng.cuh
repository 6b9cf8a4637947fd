// Bit-exact port of numpy's SeedSequence -> PCG64 -> Generator.random() draw used by the reference
// vacancy sampler (disorder.py:66-68, :79).  Third-party algorithm (numpy 2.3.5, not vendored in the
// reference): SeedSequence pool mixing (pool size 4, hashmix/mix constants), generate_state(4, uint64),
// PCG64 "setseq" seeding (state = 0; step; state += initstate; step), XSL-RR 128/64 output after each
// step, random() = (next64 >> 11) * 2^-53.  Pinned against numpy in tests/test_boundary.py (rng draws, masks) and tests/test_device_pipeline_gpu.py (device sampler).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define HX_HD __host__ __device__ __forceinline__
#else
#define HX_HD inline
#endif

namespace hx {

struct u128 {
  uint64_t hi, lo;
};

HX_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

HX_HD u128 mul128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo * b.lo;
  r.hi = mulhi64(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
  return r;
}

HX_HD u128 add128(u128 a, u128 b) {
  u128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1u : 0u);
  return r;
}

// numpy SeedSequence word coercion of a non-negative integer (little-endian 32-bit words; 0 -> [0]).
HX_HD int words32(uint64_t x, uint32_t* w) {
  if (x == 0) {
    w[0] = 0;
    return 1;
  }
  int n = 0;
  while (x) {
    w[n++] = (uint32_t)(x & 0xFFFFFFFFu);
    x >>= 32;
  }
  return n;
}

struct SeedHash {
  uint32_t hc;
  HX_HD uint32_t hashmix(uint32_t v) {
    v ^= hc;
    hc *= 0x931E8875u;
    v *= hc;
    v ^= v >> 16;
    return v;
  }
};

HX_HD uint32_t seed_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
  return r ^ (r >> 16);
}

// generate_state(4, uint64) of SeedSequence(seed, spawn_key=(level, rep)).
HX_HD void seedseq_state4(uint64_t seed, uint64_t level, uint64_t rep, uint64_t out[4]) {
  uint32_t ent[12];
  int ne = words32(seed, ent);
  // spawn_key present: pad run entropy to the pool size with zeros
  while (ne < 4) ent[ne++] = 0;
  ne += words32(level, ent + ne);
  ne += words32(rep, ent + ne);
  SeedHash h{0x43B0D7E5u};
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = h.hashmix(i < ne ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = seed_mix(pool[d], h.hashmix(pool[s]));
  for (int s = 4; s < ne; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = seed_mix(pool[d], h.hashmix(ent[s]));
  uint32_t hb = 0x8B51F9DDu;
  uint32_t w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= 0x58F38DEDu;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; ++i) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

struct Pcg64 {
  u128 state, inc;
  static constexpr uint64_t MUL_HI = 0x2360ED051FC65DA4ull;
  static constexpr uint64_t MUL_LO = 0x4385DF649FCCF645ull;
  HX_HD void step() { state = add128(mul128(state, u128{MUL_HI, MUL_LO}), inc); }
  HX_HD void seed(const uint64_t s[4]) {
    u128 initstate{s[0], s[1]};
    u128 seq{s[2], s[3]};
    inc.hi = (seq.hi << 1) | (seq.lo >> 63);
    inc.lo = (seq.lo << 1) | 1u;
    state = u128{0, 0};
    step();
    state = add128(state, initstate);
    step();
  }
  HX_HD uint64_t next64() {
    step();
    uint64_t x = state.hi ^ state.lo;
    unsigned r = (unsigned)(state.hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
  }
  HX_HD double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
};

}  // namespace hx
