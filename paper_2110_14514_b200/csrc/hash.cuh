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

// Bit of the membership prefilter (a one-hash Bloom bitmap over the same keys):
// the high half of the mixed key, independent of the table's low-bit slot.
__device__ __forceinline__ uint64_t filter_bit(uint64_t h, uint64_t fmask) { return (h >> 32) & fmask; }

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
