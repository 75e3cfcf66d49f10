// Multi-GPU plumbing of the sample-sharded solves.
#pragma once
#include "common.cuh"

namespace ogcp {

// In-place sums across the context's ranks on the context stream (no-ops for world == 1).
void comm_allreduce_sum(Ctx* ctx, float* p, size_t n);
void comm_allreduce_sum(Ctx* ctx, double* p, size_t n);
// Make the device error word identical on every rank (min of first codes, OR of bits),
// so every rank takes the same accept / reject / raise decision.
void comm_sync_flags(Ctx* ctx);
void comm_init(Ctx* ctx, const uint8_t* id, int rank, int world);
void comm_unique_id(uint8_t* out128);
void comm_destroy(Ctx* ctx);
int comm_selftest(Ctx* ctx);

}  // namespace ogcp
