// Internal engine structures shared by the kernels and the host runtime.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ogcp_b200.h"
#include "pcg64.cuh"

namespace ogcp {

constexpr int kMaxModes = 8;
constexpr int kNumSMs = 148;

// Engine error carrying the ABI status code (mirrors exceptions.py).
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define OGCP_CUDA(call)                                                                \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::ogcp::Error(OGCP_E_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                           " at " __FILE__ ":" + std::to_string(__LINE__)); \
  } while (0)

// Allocations come from the device's stream-ordered memory pool with an
// unbounded release threshold: a slice's multi-GB buffers freed at the end of a
// step are handed to the next slice without another trip through the driver
// (plain cudaMalloc/cudaFree of GB-sized blocks measured 10-700 ms per slice).
// The allocation is complete before ensure() returns, so any stream may use it;
// release() waits for the device first, like cudaFree.
cudaStream_t alloc_stream();

// Device buffer owned by the engine (slices, scratch).
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) {
      cudaDeviceSynchronize();
      cudaFreeAsync(ptr, alloc_stream());
    }
    ptr = nullptr;
    bytes = 0;
  }
  // Grow-only; contents are not preserved.
  void* ensure(size_t b) {
    if (b <= bytes && ptr) return ptr;
    release();
    size_t nb = b < 256 ? 256 : b;
    OGCP_CUDA(cudaMallocAsync(&ptr, nb, alloc_stream()));
    OGCP_CUDA(cudaStreamSynchronize(alloc_stream()));
    bytes = nb;
    return ptr;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(ptr); }
};

// Record layout of one stored nonzero in HBM: ndim int32 coordinates followed
// by the float32 value, padded to 16 B (ndim <= 3) or 32 B (ndim <= 7).
inline int record_ints(int ndim) { return ndim + 1 <= 4 ? 4 : 8; }

// Device-side error/event word.  Codes are event*4 + sub with sub 0 = draw,
// 1 = loss-domain check, 2 = non-finite iterate, so the smallest code is the
// error the reference would have raised first (solvers.py:243-254, 337-355).
struct DevFlags {
  long long first_code[4];   // [0] sampling error, [1] data error, [2] divergence, [3] shortfall
  unsigned int data_bits;    // bit0 non-finite m, bit1 m < 0
  unsigned int pad;
};

enum : int { kFlagSampling = 0, kFlagData = 1, kFlagDiverge = 2, kFlagShortfall = 3 };
constexpr unsigned kMergeOverflowBit = 0x80000000u;  // DevFlags::data_bits: a merged-draw counter wrapped
constexpr long long kNoEvent = 0x7fffffffffffffffLL;

struct Slice {
  int ndim = 0;
  int64_t dims[kMaxModes] = {0};
  int64_t nnz = 0;
  bool omega_fits = true;   // omega < 2^63
  int64_t omega = 0;
  double omega_d = 0;
  double frob_sq = 0;
  bool x_negative = false;  // any stored value < 0   (poisson domain, losses.py:52)
  bool x_nonbinary = false; // any stored value not in {0,1} (losses.py:54)
  int rec_ints = 4;
  DevBuf records;           // nnz * rec_ints int32
  DevBuf hash;              // table_size uint64 linear keys, ~0 = empty
  uint64_t table_mask = 0;
  // Prefilter for large slices: a word-blocked Bloom filter (hash.cuh
  // filter_may_contain); a clear bit proves absence without touching the
  // (DRAM-resident) table.  <= 64 MB so it stays in L2 while the zero candidates
  // are probed.
  DevBuf filter;
  uint64_t filter_mask = 0;  // 0: no prefilter
  uint64_t strides[kMaxModes] = {0};
  // Bucketed copy for merged (count-form) sample sets: positions ordered by
  // (row bucket of bucket_mode, ordinal), perm[pos] = ordinal, rec_b[pos] =
  // records[perm[pos]].  A merged set walked in position order touches one
  // 1/nbuckets slice of the bucket mode's factor and gradient rows at a time,
  // which then stay L2-resident; within a bucket mode-0 order is kept.
  int bucket_mode = -1, nbuckets = 0;
  int64_t bucket_olo = 0, bucket_ohi = 0;  // ordinal range covered (a rank's share in a multi-GPU solve)
  DevBuf perm, rec_b;
};

// Per-kernel-class CUDA-event timing on the context stream (bench evidence).
enum : int { kProfDraw = 0, kProfSgrad, kProfWgrad, kProfObjective, kProfGram, kProfUpdate, kProfIngest,
             kProfClasses };

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[kProfClasses];
  double total_ms[kProfClasses] = {0};
  int64_t count[kProfClasses] = {0};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) throw Error(OGCP_E_CUDA, "cudaEventCreate failed");
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void resolve() {
    for (int c = 0; c < kProfClasses; ++c) {
      for (auto& pr : pending[c]) {
        cudaEventSynchronize(pr.second);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pr.first, pr.second);
        total_ms[c] += ms;
        count[c] += 1;
        pool.push_back(pr.first);
        pool.push_back(pr.second);
      }
      pending[c].clear();
    }
  }
  void reset() {
    resolve();
    for (int c = 0; c < kProfClasses; ++c) { total_ms[c] = 0; count[c] = 0; }
  }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  Profiler prof;
  bool shard_sim = false;       // rank/world set without a communicator (single-process tests of the shard logic)
  double slack = 1.0;           // sampler over-provisioning multiplier (grows on shortfall)
  bool merge_draws = true;      // merged (count) form of dense nonzero draws in the solves
  // Two-pass scatter for merged sets with a large random-access mode.  Off: on
  // c4 it measured 19.2 ms vs 10.2 ms for the fused pass (profiles/), the second
  // pass repeating the gather latency chain without saving enough traffic.
  bool split_scatter = false;
  DevBuf wticket_buf;           // fused weight step: last-block ticket (0 between launches)
  unsigned int* wticket() {
    if (!wticket_buf.ptr) {
      wticket_buf.ensure(64);
      OGCP_CUDA(cudaMemset(wticket_buf.ptr, 0, 64));
    }
    return wticket_buf.as<unsigned int>();
  }
  bool deterministic = false;   // small models: fixed-order (bitwise reproducible) K3 scatter
  DevBuf det_partials;
  bool umma_gram = true;        // ldr 64 / 128 Grams on tcgen05 / TMEM (gram_umma.cuh)
  bool batch_draws = true;      // small draws: every draw of a solver epoch made at its start (one launch per pass)
  int sort_zeros = 0;           // bucketed merged draws: zero rows sorted by (bucket, mode-0 row) [1] or
                                // by bucket only [2];
                                // off: c4 measured +0.5 ms per draw for -0.3 ms of k_sgrad
  bool lean_walks = false;      // walk3.cuh kernels for merged 3-way sets (register-pipelined)
  bool tma_walks = true;        // walk_tma.cuh K3 walk for merged 3-way sets (TMA gather4, warp-specialised)
  bool tma_a2_resident = false; // TMA walks: a mode-2 factor <= 128 KB resident in shared memory (8 stages
                                // then fit: c4 measured 7.55 -> 7.79 ms, fewer rows in flight)
  bool tma_wgrad = false;       // walk_tma.cuh weight-gradient walk (measured slower than the generic one)
  bool buckets = true;          // bucketed layout for merged sets of large slices (OGCP_OPT_BUCKETS)
  int buckets_force = 0;        // > 1: always bucket, with this many buckets (tests)
  DevBuf ybuf;                  // per-sample y of the split scatter
  // multi-GPU: NCCL communicator over the ranks that share one stream of slices
  void* comm = nullptr;         // ncclComm_t
  void* comm_draw = nullptr;    // ncclComm_t split from comm: the sharded draws' exchanges (side stream)
  bool shard_draws = true;      // multi-GPU merged draws sharded by word range (sampler.cu shard_draw_enqueue)
  bool shard_sim_timing = false;  // timing shard simulation: draws' exchanges stood in by this rank's own
                                  // slots, every collective by a stand-in kernel for its modeled duration
  double sim_bus_gbs = 700.0;     // stand-in collectives: NVLink bus bandwidth per GPU
  double sim_lat_us = 15.0;       // ... and per-collective latency
  int rank = 0, world = 1;
  DevBuf flagpack;
  // scratch
  DevBuf flags;                 // DevFlags
  DevBuf draw_a, draw_b, draw_c, draw_d, draw_e;   // sampler scratch
  DevBuf scalars;               // small device scalars (int64 x 16)
  DevBuf partials;              // reduction partials (double)
  DevBuf gram;                  // gram scratch
  DevBuf hist;                  // history coefficient matrices
  DevBuf wsolve;                // weight-solve state
  DevBuf grads;                 // factor-gradient buffers
  DevBuf grad_ord, grad_zero;   // gradient sample set
  DevBuf obj_ord, obj_zero;     // objective sample set
  DevBuf window;                // window matrix / vectors
  DevBuf iota;                  // 0..iota_n-1 ordinals: "every stored nonzero once" sample sets
  int64_t iota_n = 0;
  DevBuf dense;                 // dense-Gaussian terms: b[ldr], s[ldr] (double)
  DevBuf pinned_dummy;
  double* host_scalars = nullptr;  // pinned host mirror
  DevFlags* host_flags = nullptr;  // pinned
  void count(int n = 1) { launches += n; }
};
// Restores ctx->slack when a retry loop ends: the over-provisioning raised by a
// draw shortfall applies to the retried draw/epoch only, not to every later one.
struct SlackScope {
  Ctx* ctx;
  double saved;
  explicit SlackScope(Ctx* c) : ctx(c), saved(c->slack) {}
  ~SlackScope() { ctx->slack = saved; }
};


// RAII event bracket around the launches of one kernel class.
struct ProfScope {
  Ctx* ctx;
  int cls;
  cudaEvent_t start = nullptr;
  ProfScope(Ctx* c, int k) : ctx(c), cls(k) {
    if (ctx->prof.on) {
      start = ctx->prof.get();
      cudaEventRecord(start, ctx->stream);
    }
  }
  ~ProfScope() {
    if (start) {
      cudaEvent_t end = ctx->prof.get();
      cudaEventRecord(end, ctx->stream);
      ctx->prof.pending[cls].emplace_back(start, end);
    }
  }
};

inline void check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(OGCP_E_CUDA, std::string("kernel launch failed: ") + cudaGetErrorString(e));
}

inline int ceil_div_i(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace ogcp
