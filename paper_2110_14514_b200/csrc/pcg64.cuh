// numpy-compatible keyed RNG: SeedSequence -> PCG64 (XSL-RR 128/64) -> bounded
// 32-bit Lemire draws, restated so the GPU sampler reproduces the reference's
// draws bit-exactly.
//
// Reference call sites: rng_at  pkg/src/ogcp/sampling.py:39-42
//                       integers(0, eta, p)        sampling.py:125
//                       integers(0, dims, (n, d))  sampling.py:138
// Third-party algorithm (numpy 2.3.5, un-vendored): SeedSequence
// (numpy/random/bit_generator.pyx), PCG64 (numpy/random/src/pcg64/pcg64.h),
// random_bounded_uint64[_fill] + buffered_bounded_lemire_uint32
// (numpy/random/src/distributions/distributions.c).  Restatement: SURVEY.md App. A.
//
// Counter-based view used on the device: a fresh Generator is a stream of
// 32-bit words; word w is the low (w even) / high (w odd) half of PCG64 output
// number w>>1, and output o is XSL-RR of the LCG state after o+1 steps.  The
// LCG jump-ahead s_n = A_n*s_0 + inc*B_n makes every word addressable.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define OGCP_HD __host__ __device__ __forceinline__
#else
#define OGCP_HD inline
#endif

namespace ogcp {

typedef unsigned __int128 u128;

OGCP_HD u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

OGCP_HD uint64_t rotr64(uint64_t v, unsigned r) {
  return (v >> r) | (v << ((-r) & 63u));
}

// XSL-RR output of a 128-bit state (pcg_output_xsl_rr_128_64).
OGCP_HD uint64_t pcg_output(u128 state) {
  return rotr64((uint64_t)(state >> 64) ^ (uint64_t)state, (unsigned)(state >> 122));
}

struct Pcg64 {
  u128 state;
  u128 inc;
};

// pcg_setseq_128_srandom_r: state=0, inc=(initseq<<1)|1, step, +=initstate, step.
OGCP_HD Pcg64 pcg_seed(u128 initstate, u128 initseq) {
  Pcg64 g;
  g.inc = (initseq << 1) | (u128)1;
  g.state = 0;
  g.state = g.state * pcg_mult() + g.inc;
  g.state += initstate;
  g.state = g.state * pcg_mult() + g.inc;
  return g;
}

// Jump coefficients: after n steps, state = A*state0 + inc*B.
struct Jump {
  u128 A, B;
};

OGCP_HD Jump jump_identity() { Jump j; j.A = 1; j.B = 0; return j; }

// compose: first x then y.
OGCP_HD Jump jump_compose(Jump x, Jump y) {
  Jump r;
  r.A = x.A * y.A;
  r.B = x.B * y.A + y.B;
  return r;
}

// Jump by n steps via binary powers (host or device; ~log2(n) 128-bit mults).
OGCP_HD Jump jump_pow(uint64_t n) {
  Jump acc = jump_identity();
  Jump cur; cur.A = pcg_mult(); cur.B = 1;
  while (n) {
    if (n & 1ull) acc = jump_compose(acc, cur);
    cur = jump_compose(cur, cur);
    n >>= 1;
  }
  return acc;
}

OGCP_HD u128 jump_apply(Jump j, const Pcg64& g) { return j.A * g.state + g.inc * j.B; }

// ---------------------------------------------------------------------------
// SeedSequence (pool size 4) -> generate_state(4, uint64) -> PCG64 seeding.
// entropy words: uint32 little-endian words of `seed`; spawn_key elements each
// contribute their uint32 words; run entropy is zero-padded to 4 words when a
// spawn key is present.
// ---------------------------------------------------------------------------
static inline int seedseq_words_of(uint64_t v, uint32_t* out) {
  if (v == 0) { out[0] = 0; return 1; }
  int n = 0;
  while (v) { out[n++] = (uint32_t)(v & 0xffffffffu); v >>= 32; }
  return n;
}

static inline uint32_t seedseq_hashmix(uint32_t value, uint32_t* hash_const) {
  value ^= *hash_const;
  *hash_const *= 0x931e8875u;
  value *= *hash_const;
  value ^= value >> 16;
  return value;
}

static inline uint32_t seedseq_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
  r ^= r >> 16;
  return r;
}

// Returns PCG64 seeded exactly as np.random.default_rng(SeedSequence(seed, spawn_key=key)).
// key elements must be >= 0 (numpy rejects negatives).
static inline Pcg64 seedseq_pcg64(uint64_t seed, const uint64_t* key, int nkey) {
  uint32_t ent[64];
  int n = seedseq_words_of(seed, ent);
  if (nkey > 0) {
    while (n < 4) ent[n++] = 0;
    for (int i = 0; i < nkey && n < 60; ++i) n += seedseq_words_of(key[i], ent + n);
  }
  uint32_t pool[4];
  uint32_t hc = 0x43b0d7e5u;
  for (int i = 0; i < 4; ++i) pool[i] = seedseq_hashmix(i < n ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = seedseq_mix(pool[d], seedseq_hashmix(pool[s], &hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = seedseq_mix(pool[d], seedseq_hashmix(ent[s], &hc));
  uint32_t words[8];
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= 0x58f38dedu;
    v *= hb;
    v ^= v >> 16;
    words[i] = v;
  }
  uint64_t s64[4];
  for (int i = 0; i < 4; ++i) s64[i] = (uint64_t)words[2 * i] | ((uint64_t)words[2 * i + 1] << 32);
  u128 initstate = ((u128)s64[0] << 64) | s64[1];
  u128 initseq = ((u128)s64[2] << 64) | s64[3];
  return pcg_seed(initstate, initseq);
}

// Lemire acceptance for range n = high-low (n >= 2, n <= 2^32-1):
// m = word*n; accept iff (uint32)m >= (2^32 mod n); value = m>>32.
OGCP_HD uint32_t lemire_threshold(uint32_t n) {
  return (uint32_t)((0x100000000ull) % (uint64_t)n);
}

// Sequential host-side stream (has_uint32 half-word buffer semantics).
struct HostStream {
  Pcg64 g;
  int has_half;
  uint32_t half;
  uint64_t words;  // words consumed so far
  OGCP_HD uint32_t next32() {
    ++words;
    if (has_half) { has_half = 0; return half; }
    g.state = g.state * pcg_mult() + g.inc;
    uint64_t o = pcg_output(g.state);
    has_half = 1;
    half = (uint32_t)(o >> 32);
    return (uint32_t)o;
  }
  // integers(0, n) for 1 <= n <= 2^32-1 (n == 1 consumes nothing).
  OGCP_HD uint32_t bounded(uint32_t n) {
    if (n <= 1) return 0;
    uint32_t thr = lemire_threshold(n);
    for (;;) {
      uint64_t m = (uint64_t)next32() * n;
      if ((uint32_t)m >= thr) return (uint32_t)(m >> 32);
    }
  }
};

}  // namespace ogcp
