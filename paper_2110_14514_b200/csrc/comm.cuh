// Multi-GPU plumbing of the sample-sharded solves.
#pragma once
#include "common.cuh"

namespace ogcp {

// In-place sums across the context's ranks on the context stream (no-ops for world == 1).
void comm_allreduce_sum(Ctx* ctx, float* p, size_t n);
void comm_allreduce_sum(Ctx* ctx, double* p, size_t n);
// Rank r's contiguous share [lo, hi) of `rows` rows.
void comm_row_range(int64_t rows, int rank, int world, int64_t* lo, int64_t* hi);
// Row-owner collectives over nbuf row-major [rows[k] x ldr] fp32 buffers (no-ops without a
// communicator): reduce sums every rank's copy of rows [lo_r, hi_r) onto rank r;
// gather broadcasts each owner's rows to every rank.
void comm_reduce_rows(Ctx* ctx, float* const* bufs, const int64_t* rows, int nbuf, int ldr);
void comm_gather_rows(Ctx* ctx, float* const* bufs, const int64_t* rows, int nbuf, int ldr);
// Make the device error word identical on every rank (min of first codes, OR of bits),
// so every rank takes the same accept / reject / raise decision.
void comm_sync_flags(Ctx* ctx);
// Sharded-draw exchanges on the draw communicator (ctx->comm_draw) and ctx->stream:
// in-place all-gather of per-rank slots of `bytes` each; in-place reduce-scatter of
// uint32 sums (chunk r of `words` words lands on rank r); uint64 sum all-reduce.
// begin/end bracket one NCCL group.
void comm_draw_group(Ctx* ctx, bool begin);
void comm_draw_allgather(Ctx* ctx, void* buf, size_t bytes);
void comm_draw_reduce_scatter_u32(Ctx* ctx, uint32_t* buf, size_t words);
void comm_draw_allreduce_u64(Ctx* ctx, unsigned long long* buf, size_t n);
// Timing shard simulation (no communicator): enqueue a stand-in for a collective that
// moves `moved` bytes per rank -- its modeled time on the SMs an NCCL kernel holds.
void comm_standin(Ctx* ctx, double moved);
void comm_init(Ctx* ctx, const uint8_t* id, int rank, int world);
void comm_unique_id(uint8_t* out128);
void comm_destroy(Ctx* ctx);
int comm_selftest(Ctx* ctx);

}  // namespace ogcp
