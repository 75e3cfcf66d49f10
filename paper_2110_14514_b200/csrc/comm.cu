// NCCL communicator for the sample-sharded solves.  NCCL is loaded with dlopen
// (libnccl.so.2 -- the copy torch already mapped, or the system one), so the
// engine library itself has no link-time NCCL dependency; the unique id is
// exchanged by the caller (torch.distributed broadcast, 128 bytes).
//
// Per factor iteration the ranks exchange the d factor-gradient matrices: for
// small models one allreduce over the contiguous gradient buffer, then Adam runs
// replicated on identical inputs; otherwise each rank owns a contiguous 1/N of
// every mode's rows -- the gradient rows are reduced onto their owner, the owner
// runs the row Adam (K5) on them alone and broadcasts the new factor rows, so
// the factors stay bitwise identical across ranks.  Per weight iteration the
// R-vector gradient is allreduced; per objective evaluation one fp64 partial;
// per epoch the error word.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "comm.cuh"

namespace ogcp {

namespace {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) return;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(a.lib, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(a.lib, "ncclCommInitRank"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(a.lib, "ncclAllReduce"));
    a.Reduce = reinterpret_cast<decltype(a.Reduce)>(dlsym(a.lib, "ncclReduce"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(dlsym(a.lib, "ncclBroadcast"));
    a.ReduceScatter = reinterpret_cast<decltype(a.ReduceScatter)>(dlsym(a.lib, "ncclReduceScatter"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(a.lib, "ncclAllGather"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.lib, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.lib, "ncclGroupEnd"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.lib, "ncclCommDestroy"));
    a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(dlsym(a.lib, "ncclCommSplit"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(a.lib, "ncclGetErrorString"));
  });
  if (!a.lib || !a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.Reduce || !a.Broadcast || !a.GroupStart ||
      !a.GroupEnd || !a.ReduceScatter || !a.AllGather)
    throw Error(OGCP_E_INTERNAL, "NCCL (libnccl.so.2) is not available for the multi-GPU path");
  return a;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(OGCP_E_CUDA, std::string(what) + ": " + (api().GetErrorString ? api().GetErrorString(r) : "nccl"));
}

__global__ void k_flags_pack(const DevFlags* f, long long* pk) {
  if (threadIdx.x || blockIdx.x) return;
  for (int i = 0; i < 4; ++i) pk[i] = f->first_code[i];
  pk[4] = (f->data_bits & 1u) ? 1 : 0;
  pk[5] = (f->data_bits & 2u) ? 1 : 0;
  pk[6] = (f->data_bits & kMergeOverflowBit) ? 1 : 0;
  pk[7] = 0;
}

__global__ void k_flags_unpack(DevFlags* f, const long long* pk) {
  if (threadIdx.x || blockIdx.x) return;
  for (int i = 0; i < 4; ++i) f->first_code[i] = pk[i];
  f->data_bits = (pk[4] ? 1u : 0u) | (pk[5] ? 2u : 0u) | (pk[6] ? kMergeOverflowBit : 0u);
}

// Timing shard simulation: a collective's stand-in -- kStandinCtas CTAs (the SMs an
// NCCL ring / NVLS kernel holds) spin on the global timer for the modeled time.
constexpr int kStandinCtas = 24;
__global__ void k_comm_standin(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(256);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

}  // namespace

// Modeled time of a collective moving `moved` bytes per rank (ring schedule:
// all-reduce 2 (N-1)/N of the buffer, reduce-scatter / all-gather (N-1)/N of the
// full buffer) plus a fixed latency; enqueued as k_comm_standin in a timing shard
// simulation, nothing otherwise.
void comm_standin(Ctx* ctx, double moved) {
  if (!ctx->shard_sim || !ctx->shard_sim_timing || ctx->world <= 1) return;
  const double ns = ctx->sim_lat_us * 1e3 + moved / (ctx->sim_bus_gbs * 1e9) * 1e9;
  k_comm_standin<<<kStandinCtas, 32, 0, ctx->stream>>>((unsigned long long)ns);
  ctx->count();
}

static double ring_share(const Ctx* ctx) { return (double)(ctx->world - 1) / ctx->world; }

// (no communicator with world > 1: single-process shard simulation, sums are the caller's)
void comm_allreduce_sum(Ctx* ctx, float* p, size_t n) {
  if (ctx->world <= 1 || n == 0) return;
  if (!ctx->comm) return comm_standin(ctx, 2.0 * ring_share(ctx) * 4.0 * n);
  nccl_check(api().AllReduce(p, p, n, ncclFloat32, ncclSum, (ncclComm_t)ctx->comm, ctx->stream), "ncclAllReduce");
}

void comm_allreduce_sum(Ctx* ctx, double* p, size_t n) {
  if (ctx->world <= 1 || n == 0) return;
  if (!ctx->comm) return comm_standin(ctx, 2.0 * ring_share(ctx) * 8.0 * n);
  nccl_check(api().AllReduce(p, p, n, ncclFloat64, ncclSum, (ncclComm_t)ctx->comm, ctx->stream), "ncclAllReduce");
}

void comm_row_range(int64_t rows, int rank, int world, int64_t* lo, int64_t* hi) {
  *lo = rows * rank / world;
  *hi = rows * (rank + 1) / world;
}

// Owner-computes row blocks.  Rank r owns rows [lo_r, hi_r) of every buffer
// (comm_row_range).  A buffer whose row count divides by the world size has equal
// blocks, so its reduction onto the owners is one in-place ncclReduceScatter and
// the return trip one in-place ncclAllGather -- the collectives NCCL runs
// ring/NVLS-optimal on NVSwitch (every c4 mode: 1e6 and 1e3 rows at N = 2/4/8).
// Other buffers fall back to one in-place ncclReduce / ncclBroadcast per owner.
// Both forms move the bytes of one allreduce but leave the row update between
// them to the owner alone; all calls of a step go out as one NCCL group.
static void rows_group(Ctx* ctx, float* const* bufs, const int64_t* rows, int nbuf, int ldr, bool reduce) {
  if (ctx->world <= 1) return;
  if (!ctx->comm) {
    double bytes = 0.0;
    for (int k = 0; k < nbuf; ++k) bytes += (double)rows[k] * ldr * 4.0;
    return comm_standin(ctx, ring_share(ctx) * bytes);
  }
  NcclApi& a = api();
  ncclComm_t comm = (ncclComm_t)ctx->comm;
  const int W = ctx->world;
  nccl_check(a.GroupStart(), "ncclGroupStart");
  for (int k = 0; k < nbuf; ++k) {
    if (rows[k] % W == 0) {
      const size_t blk = (size_t)(rows[k] / W) * ldr;
      float* own = bufs[k] + blk * ctx->rank;
      if (reduce)
        nccl_check(a.ReduceScatter(bufs[k], own, blk, ncclFloat32, ncclSum, comm, ctx->stream), "ncclReduceScatter");
      else
        nccl_check(a.AllGather(own, bufs[k], blk, ncclFloat32, comm, ctx->stream), "ncclAllGather");
      continue;
    }
    for (int r = 0; r < W; ++r) {
      int64_t lo, hi;
      comm_row_range(rows[k], r, W, &lo, &hi);
      if (hi <= lo) continue;
      float* p = bufs[k] + (size_t)lo * ldr;
      const size_t n = (size_t)(hi - lo) * ldr;
      if (reduce) nccl_check(a.Reduce(p, p, n, ncclFloat32, ncclSum, r, comm, ctx->stream), "ncclReduce");
      else nccl_check(a.Broadcast(p, p, n, ncclFloat32, r, comm, ctx->stream), "ncclBroadcast");
    }
  }
  nccl_check(a.GroupEnd(), "ncclGroupEnd");
}

void comm_reduce_rows(Ctx* ctx, float* const* bufs, const int64_t* rows, int nbuf, int ldr) {
  rows_group(ctx, bufs, rows, nbuf, ldr, true);
}

void comm_gather_rows(Ctx* ctx, float* const* bufs, const int64_t* rows, int nbuf, int ldr) {
  rows_group(ctx, bufs, rows, nbuf, ldr, false);
}

void comm_sync_flags(Ctx* ctx) {
  if (ctx->world <= 1) return;
  if (!ctx->comm) return comm_standin(ctx, 0.0);
  long long* pk = static_cast<long long*>(ctx->flagpack.ensure(8 * sizeof(long long)));
  k_flags_pack<<<1, 1, 0, ctx->stream>>>(ctx->flags.as<DevFlags>(), pk);
  nccl_check(api().AllReduce(pk, pk, 4, ncclInt64, ncclMin, (ncclComm_t)ctx->comm, ctx->stream), "ncclAllReduce");
  nccl_check(api().AllReduce(pk + 4, pk + 4, 4, ncclInt64, ncclMax, (ncclComm_t)ctx->comm, ctx->stream),
             "ncclAllReduce");
  k_flags_unpack<<<1, 1, 0, ctx->stream>>>(ctx->flags.as<DevFlags>(), pk);
  ctx->count(2);
  check_launch();
}

// ---- sharded draws (sampler.cu shard_draw_enqueue): a second communicator, so the
// draw's collectives on the side stream never interleave with the solve's on the
// context stream within one communicator
void comm_draw_group(Ctx* ctx, bool begin) {
  if (!ctx->comm_draw) return;  // (no stand-in: the group's members stand in for themselves)
  nccl_check(begin ? api().GroupStart() : api().GroupEnd(), "ncclGroup");
}

void comm_draw_allgather(Ctx* ctx, void* buf, size_t bytes) {
  if (bytes == 0) return;
  if (!ctx->comm_draw) return comm_standin(ctx, ring_share(ctx) * bytes * ctx->world);
  char* b = static_cast<char*>(buf);
  nccl_check(api().AllGather(b + bytes * ctx->rank, b, bytes, ncclUint8, (ncclComm_t)ctx->comm_draw, ctx->stream),
             "ncclAllGather");
}

void comm_draw_reduce_scatter_u32(Ctx* ctx, uint32_t* buf, size_t words) {
  if (words == 0) return;
  if (!ctx->comm_draw) return comm_standin(ctx, ring_share(ctx) * 4.0 * words * ctx->world);
  nccl_check(api().ReduceScatter(buf, buf + words * ctx->rank, words, ncclUint32, ncclSum,
                                 (ncclComm_t)ctx->comm_draw, ctx->stream),
             "ncclReduceScatter");
}

void comm_draw_allreduce_u64(Ctx* ctx, unsigned long long* buf, size_t n) {
  if (n == 0) return;
  if (!ctx->comm_draw) return comm_standin(ctx, 2.0 * ring_share(ctx) * 8.0 * n);
  nccl_check(api().AllReduce(buf, buf, n, ncclUint64, ncclSum, (ncclComm_t)ctx->comm_draw, ctx->stream),
             "ncclAllReduce");
}

void comm_init(Ctx* ctx, const uint8_t* id, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(OGCP_E_USAGE, "bad rank / world size");
  if (world == 1) {
    ctx->rank = 0;
    ctx->world = 1;
    return;
  }
  ncclUniqueId uid;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm;
  OGCP_CUDA(cudaSetDevice(ctx->device));
  nccl_check(api().CommInitRank(&comm, world, uid, rank), "ncclCommInitRank");
  ctx->comm = comm;
  ctx->comm_draw = nullptr;  // without ncclCommSplit (NCCL < 2.18) the draws stay replicated
  if (api().CommSplit) {
    ncclComm_t dc = nullptr;
    nccl_check(api().CommSplit(comm, 0, rank, &dc, nullptr), "ncclCommSplit");
    ctx->comm_draw = dc;
  }
  ctx->rank = rank;
  ctx->world = world;
}

void comm_unique_id(uint8_t* out) {
  ncclUniqueId uid;
  nccl_check(api().GetUniqueId(&uid), "ncclGetUniqueId");
  memcpy(out, &uid, sizeof(uid));
}

// One-rank communicator round trip through every collective the solves use
// (fp32 / fp64 sum, int64 min / max, grouped fp32 row reduce / broadcast / reduce-scatter /
// all-gather): checks the dlopen'd NCCL entry points and
// their signatures on a single GPU.  Returns the number of mismatches.
int comm_selftest(Ctx* ctx) {
  OGCP_CUDA(cudaSetDevice(ctx->device));
  ncclUniqueId uid;
  nccl_check(api().GetUniqueId(&uid), "ncclGetUniqueId");
  ncclComm_t comm;
  nccl_check(api().CommInitRank(&comm, 1, uid, 0), "ncclCommInitRank");
  DevBuf buf;
  char* d = static_cast<char*>(buf.ensure(512));
  const float hf[4] = {1.5f, -2.f, 3.25f, 0.f};
  const double hd[2] = {1e300, -7.5};
  const long long hl[4] = {5, -3, 1LL << 40, 0};
  OGCP_CUDA(cudaMemcpy(d, hf, sizeof(hf), cudaMemcpyHostToDevice));
  OGCP_CUDA(cudaMemcpy(d + 64, hd, sizeof(hd), cudaMemcpyHostToDevice));
  OGCP_CUDA(cudaMemcpy(d + 128, hl, sizeof(hl), cudaMemcpyHostToDevice));
  cudaStream_t st = ctx->stream;
  nccl_check(api().AllReduce(d, d, 4, ncclFloat32, ncclSum, comm, st), "ncclAllReduce");
  nccl_check(api().AllReduce(d + 64, d + 64, 2, ncclFloat64, ncclSum, comm, st), "ncclAllReduce");
  nccl_check(api().AllReduce(d + 128, d + 128, 2, ncclInt64, ncclMin, comm, st), "ncclAllReduce");
  nccl_check(api().AllReduce(d + 144, d + 144, 2, ncclInt64, ncclMax, comm, st), "ncclAllReduce");
  nccl_check(api().GroupStart(), "ncclGroupStart");
  nccl_check(api().Reduce(d, d, 2, ncclFloat32, ncclSum, 0, comm, st), "ncclReduce");
  nccl_check(api().Broadcast(d + 8, d + 8, 2, ncclFloat32, 0, comm, st), "ncclBroadcast");
  nccl_check(api().ReduceScatter(d, d, 2, ncclFloat32, ncclSum, comm, st), "ncclReduceScatter");
  nccl_check(api().AllGather(d + 8, d + 8, 2, ncclFloat32, comm, st), "ncclAllGather");
  nccl_check(api().GroupEnd(), "ncclGroupEnd");
  // the sharded draws' collectives on a split communicator: uint8 all-gather,
  // uint32 reduce-scatter and uint64 all-reduce (one group)
  ncclComm_t dc = nullptr;
  const uint32_t hu[2] = {0x12345678u, 7u};
  const unsigned long long hq[2] = {1ull << 40, 3ull};
  OGCP_CUDA(cudaMemcpy(d + 192, hu, sizeof(hu), cudaMemcpyHostToDevice));
  OGCP_CUDA(cudaMemcpy(d + 208, hq, sizeof(hq), cudaMemcpyHostToDevice));
  if (api().CommSplit) {
    nccl_check(api().CommSplit(comm, 0, 0, &dc, nullptr), "ncclCommSplit");
    nccl_check(api().GroupStart(), "ncclGroupStart");
    nccl_check(api().AllGather(d + 192, d + 192, 4, ncclUint8, dc, st), "ncclAllGather");
    nccl_check(api().ReduceScatter(d + 192, d + 192, 2, ncclUint32, ncclSum, dc, st), "ncclReduceScatter");
    nccl_check(api().AllReduce(d + 208, d + 208, 2, ncclUint64, ncclSum, dc, st), "ncclAllReduce");
    nccl_check(api().GroupEnd(), "ncclGroupEnd");
  }
  OGCP_CUDA(cudaStreamSynchronize(st));
  uint32_t ru[2];
  unsigned long long rq[2];
  OGCP_CUDA(cudaMemcpy(ru, d + 192, sizeof(ru), cudaMemcpyDeviceToHost));
  OGCP_CUDA(cudaMemcpy(rq, d + 208, sizeof(rq), cudaMemcpyDeviceToHost));
  if (dc && api().CommDestroy) api().CommDestroy(dc);
  float rf[4];
  double rd[2];
  long long rl[4];
  OGCP_CUDA(cudaMemcpy(rf, d, sizeof(rf), cudaMemcpyDeviceToHost));
  OGCP_CUDA(cudaMemcpy(rd, d + 64, sizeof(rd), cudaMemcpyDeviceToHost));
  OGCP_CUDA(cudaMemcpy(rl, d + 128, sizeof(rl), cudaMemcpyDeviceToHost));
  if (api().CommDestroy) api().CommDestroy(comm);
  int bad = 0;
  for (int i = 0; i < 4; ++i) bad += rf[i] != hf[i];
  for (int i = 0; i < 2; ++i) bad += rd[i] != hd[i];
  for (int i = 0; i < 4; ++i) bad += rl[i] != hl[i];
  for (int i = 0; i < 2; ++i) bad += ru[i] != hu[i];
  for (int i = 0; i < 2; ++i) bad += rq[i] != hq[i];
  bad += api().CommSplit ? 0 : 1;  // the sharded draws need a second communicator
  return bad;
}

void comm_destroy(Ctx* ctx) {
  if (ctx->comm_draw && api().CommDestroy) api().CommDestroy((ncclComm_t)ctx->comm_draw);
  ctx->comm_draw = nullptr;
  if (ctx->comm && api().CommDestroy) api().CommDestroy((ncclComm_t)ctx->comm);
  ctx->comm = nullptr;
  ctx->world = 1;
  ctx->rank = 0;
}

}  // namespace ogcp
