// Membership hash over 64-bit linear keys (replaces the sorted-key
// searchsorted of tensor.py:163-169).  Open addressing, linear probing,
// power-of-two table at load <= 0.5; an absent key costs ~1.5 probes.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace ogcp {

constexpr unsigned long long kEmptyKey = ~0ull;

struct Dims {
  long long d[kMaxModes];
};
struct Strides {
  uint64_t s[kMaxModes];
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// Returns false when the key was already present (duplicate coordinate).
__device__ __forceinline__ bool hash_insert(unsigned long long* table, uint64_t mask, uint64_t key) {
  uint64_t slot = mix64(key) & mask;
  for (;;) {
    unsigned long long prev = atomicCAS(table + slot, kEmptyKey, (unsigned long long)key);
    if (prev == kEmptyKey) return true;
    if (prev == key) return false;
    slot = (slot + 1) & mask;
  }
}

// Membership prefilter: a word-blocked Bloom filter over the same keys -- the
// high half of the mixed key picks one 32-bit word, its low 15 bits set three
// bits in that word (one load per probe; a clear bit proves absence).  fmask =
// filter bits - 1.
__device__ __forceinline__ uint64_t filter_word(uint64_t h, uint64_t fmask) { return (h >> 32) & (fmask >> 5); }
__device__ __forceinline__ uint32_t filter_bits(uint64_t h) {
  return (1u << (h & 31)) | (1u << ((h >> 5) & 31)) | (1u << ((h >> 10) & 31));
}
__device__ __forceinline__ bool filter_may_contain(const unsigned int* __restrict__ filter, uint64_t fmask,
                                                   uint64_t h) {
  const uint32_t b = filter_bits(h);
  return (__ldg(filter + filter_word(h, fmask)) & b) == b;
}

__device__ __forceinline__ bool hash_contains(const unsigned long long* __restrict__ table, uint64_t mask,
                                              uint64_t key) {
  uint64_t slot = mix64(key) & mask;
  for (;;) {
    unsigned long long k = __ldg(table + slot);
    if (k == key) return true;
    if (k == kEmptyKey) return false;
    slot = (slot + 1) & mask;
  }
}

}  // namespace ogcp
