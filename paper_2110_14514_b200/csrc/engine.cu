#include <chrono>
// Native runtime of the engine: context, slices, the per-slice solvers and
// the extern "C" boundary declared in include/ogcp_b200.h.
//
// The solver loops (solve_weights solvers.py:197-268, solve_factors
// solvers.py:290-368) run on the host and enqueue every iteration on the
// context stream without synchronising; the host synchronises once per epoch
// to read the objective estimate and the device error word, then applies the
// reference gate (fest > fest_old rejects, ties accept) with the reference's
// Adam accept/reject semantics (adam.py:83-94).
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "comm.cuh"
#include "common.cuh"
#include "compute.cuh"
#include "hash.cuh"
#include "sampler.cuh"

namespace ogcp {

template <class CT, class VT>
Slice* slice_create_impl(Ctx* ctx, int ndim, const int64_t* dims, int64_t nnz, const CT* subs, const VT* vals,
                         int allow_zero);
int64_t gradient_tensor_impl(Ctx* ctx, const SamplesP& S, const ModelP& M, const double* w_dev, const LossP& L,
                             const Strides& st, int32_t* ycoords, double* yvals, unsigned int* bad_host);
void segment_layout_impl(Ctx* ctx, const int32_t* coords, int64_t n, int ndim, int mode, int64_t dim, int32_t* perm,
                         int64_t* offsets);
void slice_contains_impl(Ctx* ctx, const Slice* s, const int64_t* subs, int64_t n, uint8_t* hit);
void iota_enqueue(Ctx* ctx, int32_t* p, int64_t n);
void slice_bucket_layout(Ctx* ctx, Slice* X, int mode, int nb, int64_t olo, int64_t ohi);

static thread_local std::string g_last_error;

cudaStream_t alloc_stream() {
  static thread_local cudaStream_t st = [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaStream_t s = nullptr;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    return s;
  }();
  return st;
}

// OGCP_DEBUG_TIMING=1: host wall time of the named scope on stderr (diagnostics only)
struct DbgTimer {
  const char* name;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit DbgTimer(const char* n) : name(n) {}
  ~DbgTimer() {
    static const bool on = getenv("OGCP_DEBUG_TIMING") != nullptr;
    if (on)
      fprintf(stderr, "[timing] %s %.1f ms\n", name,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

static const char* kind_name(int k) {
  return k == OGCP_GAUSSIAN ? "gaussian" : (k == OGCP_POISSON ? "poisson" : "bernoulli");
}

// --------------------------------------------------------------------- flags
static void reset_flags(Ctx* ctx) {
  DevFlags f;
  for (int i = 0; i < 4; ++i) f.first_code[i] = kNoEvent;
  f.data_bits = 0;
  f.pad = 0;
  *ctx->host_flags = f;
  OGCP_CUDA(cudaMemcpyAsync(ctx->flags.ptr, ctx->host_flags, sizeof(DevFlags), cudaMemcpyHostToDevice, ctx->stream));
}

static void fetch_flags(Ctx* ctx) {
  OGCP_CUDA(cudaMemcpyAsync(ctx->host_flags, ctx->flags.ptr, sizeof(DevFlags), cudaMemcpyDeviceToHost, ctx->stream));
}

struct DrawCtx {
  const Slice* X;
  double budget_q_mult = 1000.0;
};

static std::string fmt_g4(double v) {
  char buf[64];
  snprintf(buf, sizeof(buf), "%.4g", v);
  return buf;
}

static int64_t budget_of(int64_t q, int64_t max_rejects) {
  return max_rejects < 0 ? (q ? 1000 * q : 0) : max_rejects;
}

static void precheck_draw(const Slice* X, int64_t p, int64_t q) {
  if (p > 0 && X->nnz == 0) throw Error(OGCP_E_SAMPLING, "cannot draw nonzero samples: slice has no nonzeros");
  if (q > 0 && X->omega == X->nnz) throw Error(OGCP_E_SAMPLING, "cannot draw zero samples: tensor has no zeros");
}

// Outcome of an enqueued batch of events, read after a synchronisation.
// Returns 0 (clean), 1 (shortfall: redo with more candidates) or throws.
static int check_flags(Ctx* ctx, const Slice* X, int kind, int64_t budget, const std::string& what, int64_t t) {
  const DevFlags& f = *ctx->host_flags;
  if (f.data_bits & kMergeOverflowBit) return 2;  // redo without merging the draws
  long long e_min = kNoEvent;
  int which = -1;
  for (int i = 0; i < 3; ++i)
    if (f.first_code[i] < e_min) { e_min = f.first_code[i]; which = i; }
  if (f.first_code[kFlagShortfall] <= e_min && f.first_code[kFlagShortfall] != kNoEvent) return 1;
  if (which < 0) return 0;
  if (which == kFlagSampling)
    throw Error(OGCP_E_SAMPLING, "zero sampling exhausted " + std::to_string(budget) +
                                     " rejects; nonzero density is " + fmt_g4((double)X->nnz / X->omega_d) +
                                     ", set the zero sample count to 0 for dense data");
  if (which == kFlagData) {
    if (f.data_bits & 1u) throw Error(OGCP_E_DATA, std::string(kind_name(kind)) + " loss: non-finite input");
    throw Error(OGCP_E_DATA, std::string(kind_name(kind)) + " loss requires m >= 0");
  }
  throw Error(OGCP_E_DIVERGENCE,
              what + " produced non-finite values at slice " + std::to_string(t) + "; lower the learning rate");
}

static void x_domain_check(const Slice* X, int kind) {
  if (kind == OGCP_IDENTITY) return;
  if (kind == OGCP_POISSON && X->x_negative) throw Error(OGCP_E_DATA, "poisson loss requires x >= 0");
  if (kind == OGCP_BERNOULLI && X->x_nonbinary) throw Error(OGCP_E_DATA, "bernoulli loss requires x in {0, 1}");
}

// ------------------------------------------------------------- model helpers
static ModelP model_of(const ogcp_model* m) {
  if (!m || m->ndim < 1 || m->ndim > 7) throw Error(OGCP_E_USAGE, "model must have 1..7 modes");
  if (m->rank < 1) throw Error(OGCP_E_USAGE, "rank must be >= 1");
  if (m->ldr != ogcp_padded_rank(m->rank))
    throw Error(OGCP_E_USAGE, "model ldr must equal ogcp_padded_rank(rank)");
  ModelP M;
  M.ndim = m->ndim;
  M.rank = m->rank;
  M.ldr = m->ldr;
  for (int k = 0; k < kMaxModes; ++k) {
    M.A[k] = k < m->ndim ? m->factors[k] : nullptr;
    M.dims[k] = k < m->ndim ? m->dims[k] : 1;
  }
  return M;
}

static void check_model_slice(const ModelP& M, const Slice* X) {
  if (M.ndim != X->ndim)
    throw Error(OGCP_E_DATA, "tensor has " + std::to_string(X->ndim) + " modes but " + std::to_string(M.ndim) +
                                 " factors given");
  for (int k = 0; k < M.ndim; ++k)
    if (M.dims[k] != X->dims[k])
      throw Error(OGCP_E_DATA, "factor " + std::to_string(k) + " has " + std::to_string(M.dims[k]) +
                                   " rows, tensor dim is " + std::to_string(X->dims[k]));
}

static LossP loss_of(const ogcp_loss* l) {
  if (!l || l->kind < 0 || l->kind > 3) throw Error(OGCP_E_DATA, "unknown loss kind");
  if (!(l->eps > 0)) throw Error(OGCP_E_DATA, "eps must be positive");
  LossP L;
  L.kind = l->kind;
  L.eps = (float)l->eps;
  L.eps_d = l->eps;
  return L;
}

static SamplesP samples_of(const Slice* X, const int32_t* ord, int64_t p, const int32_t* z, int64_t q) {
  SamplesP S;
  S.ord = ord;
  S.p = p;
  S.zsub = z;
  S.q = q;
  S.rec = X->records.as<int>();
  S.rec_ints = X->rec_ints;
  S.nz_scale = p ? (double)X->nnz / (double)p : 0.0;
  S.zero_scale = q ? (X->omega_d - (double)X->nnz) / (double)q : 0.0;
  if (X->omega_fits && q) S.zero_scale = (double)(X->omega - X->nnz) / (double)q;
  S.p_dev = nullptr;
  S.cnt = nullptr;
  S.q_dev = nullptr;
  S.shard_rank = 0;
  S.shard_world = 1;
  S.semi = 0;
  S.chunk_shift = 0;
  S.zshard = 0;
  return S;
}

// Semi-stratified extension: uniform stratum scale omega/q, nonzero draws corrected by -g(0, m).
static SamplesP semi_of(const Slice* X, SamplesP S, bool semi) {
  if (!semi) return S;
  S.semi = 1;
  S.zero_scale = S.q ? X->omega_d / (double)S.q : 0.0;
  if (X->omega_fits && S.q) S.zero_scale = (double)X->omega / (double)S.q;
  return S;
}

// Multi-GPU merged draws: rank r owns the r-th chunk of whole nibble words of the
// nonzero ordinals (shard_owner_range: [8 cw r, 8 cw (r+1)), cw = ceil(eta / 8 / N))
// and evaluates every merged sample there, plus its share of the zero rows.
static void owned_range(const Ctx* ctx, const Slice* X, int64_t* olo, int64_t* ohi) {
  if (ctx->world <= 1) {
    *olo = 0;
    *ohi = X->nnz;
    return;
  }
  shard_owner_range(X->nnz, ctx->rank, ctx->world, olo, ohi);
}

// Solve-time sample sets are evaluated sharded across the context's ranks.
static SamplesP sharded(const Ctx* ctx, SamplesP S) {
  S.shard_rank = ctx->rank;
  S.shard_world = ctx->world;
  return S;
}

// Ordinals 0..n-1 on the device (grown lazily, kept on the context).
static const int32_t* iota_of(Ctx* ctx, int64_t n) {
  if (n > ctx->iota_n) {
    ctx->iota.ensure((size_t)std::max<int64_t>(n, 1) * 4);
    iota_enqueue(ctx, ctx->iota.as<int32_t>(), n);
    ctx->iota_n = n;
  }
  return ctx->iota.as<int32_t>();
}

// Every stored nonzero once with value weight `scale` (exact / dense-Gaussian terms),
// sharded across the context's ranks.
static SamplesP all_nonzeros(Ctx* ctx, const Slice* X, double scale) {
  SamplesP S = samples_of(X, X->nnz ? iota_of(ctx, X->nnz) : nullptr, X->nnz, nullptr, 0);
  S.nz_scale = scale;
  return sharded(ctx, S);
}

// gradient_mode (solvers.py:110-124): "dense-gaussian" only with the Gaussian loss.
static bool dense_mode(const ogcp_solver_config* cfg, int loss_kind) {
  if (cfg->gradient_mode == 0) return false;
  if (cfg->gradient_mode != 1) throw Error(OGCP_E_USAGE, "unknown gradient mode");
  if (loss_kind != OGCP_GAUSSIAN) throw Error(OGCP_E_DATA, "gradient_mode 'dense-gaussian' requires gaussian loss");
  return true;
}

// ctx->dense = [b (ldr) | s (ldr)] doubles; returns the device s after uploading w.
static double* dense_upload_s(Ctx* ctx, const double* w, int rank, int ldr) {
  ctx->dense.ensure((size_t)2 * ldr * 8);
  std::vector<double> h(ldr, 0.0);
  for (int r = 0; r < rank; ++r) h[r] = w[r];
  double* s = ctx->dense.as<double>() + ldr;
  OGCP_CUDA(cudaMemcpyAsync(s, h.data(), ldr * 8, cudaMemcpyHostToDevice, ctx->stream));
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  return s;
}

static void upload_weights(Ctx* ctx, const double* w, int rank, int ldr, float* s_f) {
  std::vector<float> h(ldr, 0.0f);
  for (int r = 0; r < rank; ++r) h[r] = (float)w[r];
  OGCP_CUDA(cudaMemcpyAsync(s_f, h.data(), ldr * 4, cudaMemcpyHostToDevice, ctx->stream));
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
}

// resolve_counts (sampling.py:71-77)
static void resolve_counts(int64_t nonzeros, int64_t zeros, const Slice* X, int64_t* p, int64_t* q) {
  *p = nonzeros < 0 ? X->nnz : nonzeros;
  if (X->nnz == 0) *p = 0;
  *q = zeros;
}

struct SampleBufs {
  DevBuf ord, zero;
  DrawScratch scr;
  MergedDraw md;
  bool merged = false;
  bool owned = false;  // multi-GPU: the merged nonzero part is this rank's own ordinal range
  bool word_sharded = false;  // multi-GPU: drawn by word range (shard_draw_enqueue); zero rows rank-local
  ShardScratch sh;
  bool semi = false;  // semi-stratified extension
  const int32_t* zsub = nullptr;   // where the last draw left the zero coordinates
  const long long* q_dev = nullptr;  // lazy zero layout row count (device)
  int64_t p = 0, q = 0;
  void size(int64_t p_, int64_t q_, int ndim, bool merged_ = false) {
    p = p_;
    q = q_;
    merged = merged_;
    if (!merged) ord.ensure((size_t)std::max<int64_t>(p, 1) * 4);
    zero.ensure((size_t)std::max<int64_t>(q, 1) * ndim * 4);
  }
  // Enqueue the draw of this buffer set and return its device sample set.
  SamplesP draw(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t budget, long long code) {
    int64_t olo = 0, ohi = X->nnz;
    owned_range(ctx, X, &olo, &ohi);
    md.perm = (merged && ctx->buckets && X->bucket_mode >= 0 && X->bucket_olo == olo && X->bucket_ohi == ohi)
                  ? X->perm.as<int32_t>()
                  : nullptr;
    md.olo = ctx->world > 1 ? (uint32_t)olo : 0u;
    md.ohi = ctx->world > 1 ? (uint32_t)ohi : 0u;
    owned = merged && ctx->world > 1;
    word_sharded = owned && shard_draw_eligible(ctx, X, p, q, semi);
    const DrawOut o = word_sharded ? shard_draw_enqueue(ctx, X, g, p, q, budget, code, md, sh)
                                   : draw_enqueue(ctx, X, g, p, q, budget, merged ? nullptr : ord.as<int32_t>(),
                                                  zero.as<int32_t>(), code, scr, merged ? &md : nullptr,
                                                  /*lazy=*/true, semi);
    zsub = o.zsub;
    q_dev = o.q_dev;
    return sample_set(X);
  }
  SamplesP sample_set(const Slice* X) const;
};

SamplesP SampleBufs::sample_set(const Slice* X) const {
  if (!merged) {
    SamplesP S = semi_of(X, samples_of(X, ord.as<int32_t>(), p, zsub, q), semi);
    S.q_dev = q_dev;
    return S;
  }
  SamplesP S = semi_of(X, samples_of(X, md.ord.as<int32_t>(), p, zsub, q), semi);
  S.q_dev = q_dev;
  S.zshard = word_sharded ? 2 : (owned ? 1 : 0);
  if (md.perm) {  // positions into the bucketed copy, walked in round-robin chunks
    S.rec = X->rec_b.as<int>();
    S.chunk_shift = 3;  // 8 batches per chunk (measured flat for shifts 2..6 on c4)
  }
  S.p = std::min<int64_t>(p, X->nnz);  // upper bound of the distinct count
  S.p_dev = md.count;
  S.cnt = md.cnt.as<uint8_t>();
  return S;                            // nz_scale stays eta / p (p draws)
}

// Two-deep draw pipeline.  A draw depends only on the slice and its key, never on
// the iterate, so the draw of iteration it+1 is enqueued on a side stream before
// iteration it's evaluation is enqueued on the context stream and overlaps it.
// The side stream first waits for everything already enqueued on the context
// stream (which includes the last reader of the buffer set it refills).
struct DrawPipe {
  SampleBufs buf[2];
  SamplesP S[2];
  cudaStream_t side = nullptr;
  cudaEvent_t go = nullptr, done[2] = {nullptr, nullptr};
  void init() {
    if (side) return;
    int lo = 0, hi = 0;  // the prefetching draws take the lower priority: they fill gaps
    OGCP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    (void)hi;
    OGCP_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, lo));
    OGCP_CUDA(cudaEventCreateWithFlags(&go, cudaEventDisableTiming));
    for (auto& e : done) OGCP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  void size(int64_t p, int64_t q, int ndim, bool merged, bool semi) {
    for (auto& b : buf) {
      b.size(p, q, ndim, merged);
      b.semi = semi;
    }
  }
  bool merged() const { return buf[0].merged; }
  // Batched epochs (small draws): every draw of the epoch made at its start in one
  // launch per pass (sampler.cu draw_batch_enqueue); issue() is then a no-op and
  // take() hands out the epoch's draws in order.
  DrawBatchSet batch;
  bool batched = false;
  int bnext = 0;
  const Slice* bX = nullptr;
  template <class KeyFn>
  void begin_epoch(Ctx* ctx, const Slice* X, KeyFn key_of, int iters, int64_t budget, long long code0) {
    batched = false;
    const SampleBufs& b0 = buf[0];
    if (!merged() && ctx->batch_draws && iters > 1 && ctx->world == 1 &&
        draw_batch_eligible(ctx, X, b0.p, b0.q, budget, b0.semi)) {
      std::vector<Pcg64> gens(iters);
      for (int it = 0; it < iters; ++it) gens[it] = key_of(it);
      draw_batch_enqueue(ctx, X, gens.data(), iters, b0.p, b0.q, budget, code0, 4, batch);
      batched = true;
      bnext = 0;
      bX = X;
      return;
    }
    issue(ctx, X, key_of(0), budget, code0, 0);
  }
  void issue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t budget, long long code, int slot) {
    if (batched) return;
    init();
    const cudaStream_t main = ctx->stream;
    OGCP_CUDA(cudaEventRecord(go, main));
    OGCP_CUDA(cudaStreamWaitEvent(side, go, 0));
    ctx->stream = side;
    try {
      S[slot] = buf[slot].draw(ctx, X, g, budget, code);
    } catch (...) {
      ctx->stream = main;
      throw;
    }
    ctx->stream = main;
    OGCP_CUDA(cudaEventRecord(done[slot], side));
  }
  SamplesP take(Ctx* ctx, int slot) {
    if (batched) {
      const int b = bnext++;
      const int32_t* ord = batch.p ? batch.ord.as<int32_t>() + (int64_t)b * batch.p : nullptr;
      const int32_t* zs = batch.q ? batch.cand.as<int32_t>() + (int64_t)b * batch.rows_max * bX->ndim : nullptr;
      SamplesP Sb = semi_of(bX, samples_of(bX, ord, batch.p, zs, batch.q), buf[0].semi);
      Sb.q_dev = batch.q ? batch.scal.as<long long>() + (int64_t)b * 16 + 8 : nullptr;  // lazy layout row count
      return Sb;
    }
    OGCP_CUDA(cudaStreamWaitEvent(ctx->stream, done[slot], 0));
    return S[slot];
  }
};

// Merged (count) form pays off when the nonzero draws cover the slice densely
// (p = "all" draws eta with replacement, sampling.py:71-77, 125).
static bool use_merged(const Ctx* ctx, const Slice* X, int64_t p) {
  // 4-bit counters: with p <= 1.25 eta a counter reaches 16 with probability
  // ~5e-13 per ordinal; the count-sum check catches it and the epoch is redone.
  return ctx->merge_draws && X->nnz >= 65536 && p >= X->nnz / 8 && p <= X->nnz + X->nnz / 4;
}

// Bucketed layout for merged sets (Slice::perm): the largest mode k >= 1 whose
// factor + gradient rows (2 dims[k] ldr 4 B) exceed 48 MB is cut into
// power-of-two row buckets of <= 64 MB, so each bucket's rows stay L2-resident
// while the set's positions inside it are walked.  Built once per slice.
static void prepare_buckets(Ctx* ctx, const Slice* Xc, int ldr) {
  Slice* X = const_cast<Slice*>(Xc);
  if (!ctx->buckets || X->ndim < 2) return;
  int mode = -1;
  double ws = 0.0;
  for (int k = 1; k < X->ndim; ++k) {
    const double w = 2.0 * (double)X->dims[k] * ldr * 4.0;
    if (w > ws) {
      ws = w;
      mode = k;
    }
  }
  int nb = 2;
  if (ctx->buckets_force > 1) {
    nb = ctx->buckets_force;
  } else {
    if (ws <= 48e6) return;
    while (nb < 256 && ws / nb > 64e6) nb <<= 1;  // c4 (256 MB): 4 buckets, measured better than 2 or 8
  }
  int64_t olo = 0, ohi = X->nnz;
  owned_range(ctx, X, &olo, &ohi);
  if (X->bucket_mode == mode && X->nbuckets == nb && X->bucket_olo == olo && X->bucket_ohi == ohi) return;
  const auto t0 = std::chrono::steady_clock::now();
  slice_bucket_layout(ctx, X, mode, nb, olo, ohi);
  if (getenv("OGCP_DEBUG_TIMING"))
    fprintf(stderr, "bucket layout %.1f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
}

// Synchronous draw with shortfall retry (used for objective sets).
static void draw_sync(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t max_rejects,
                      SampleBufs& b, bool semi = false) {
  DbgTimer dt("draw_sync");
  precheck_draw(X, p, semi ? 0 : q);
  b.size(p, q, X->ndim);
  b.semi = semi;
  const int64_t budget = budget_of(q, max_rejects);
  SlackScope slack_scope(ctx);  // a shortfall raises the slack for this retry only
  for (int attempt = 0;; ++attempt) {
    reset_flags(ctx);
    const DrawOut o = draw_enqueue(ctx, X, g, p, q, budget, b.ord.as<int32_t>(), b.zero.as<int32_t>(), 0, b.scr,
                                   nullptr, /*lazy=*/true, semi);
    b.zsub = o.zsub;
    b.q_dev = o.q_dev;
    fetch_flags(ctx);
    OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
    int r = check_flags(ctx, X, OGCP_GAUSSIAN, budget, "draw", 0);
    if (r == 0) break;
    ctx->slack *= 4.0;
    if (attempt > 8) throw Error(OGCP_E_INTERNAL, "sampler could not provision enough candidates");
  }
}

static Pcg64 keyed(uint64_t seed, std::initializer_list<int64_t> key) {
  uint64_t k[8];
  int n = 0;
  for (int64_t v : key) k[n++] = (uint64_t)v;
  return seedseq_pcg64(seed, k, n);
}

// Grams for history/regularisation: per mode P_m = A_m'A_m, C_m = Aold_m'A_m.
struct HistBufs {
  DevBuf P, C, Poo, S, Ws, coef, out, Mk, Nk, scratch, part, tmp;
};

// Small models: every mode in one launch (see compute.cuh kSmallRows).
static bool small_model(const ModelP& M) {
  if (M.ldr > 32) return false;
  for (int k = 0; k < M.ndim; ++k)
    if (M.dims[k] > kSmallRows) return false;
  return true;
}

// Multi-GPU factor solves of models past the small-model size split K5 by rows:
// rank r updates a contiguous 1/N of every mode's rows.  Also
// active in shard simulation, where rank r's share is all that runs.
static bool row_sharded(const Ctx* ctx, const ModelP& M) { return ctx->world > 1 && !small_model(M); }

// Rows [lo, hi) of mode k this rank's Gram partials cover: all of them, or the
// owned block when `shard` (the factor solves' per-iteration Grams of a
// row-sharded solve; the partials are then all-reduced, 2dR^2 fp64).  An empty block zero-fills its outputs and returns false.
static bool gram_rows(Ctx* ctx, const ModelP& M, bool shard, int k, int64_t* lo, int64_t* hi, double* o1,
                      double* o2) {
  *lo = 0;
  *hi = M.dims[k];
  if (shard) comm_row_range(M.dims[k], ctx->rank, ctx->world, lo, hi);
  if (*hi > *lo) return true;
  const size_t b = (size_t)M.rank * M.rank * 8;
  OGCP_CUDA(cudaMemsetAsync(o1, 0, b, ctx->stream));
  if (o2) OGCP_CUDA(cudaMemsetAsync(o2, 0, b, ctx->stream));
  return false;
}

static void grams_enqueue(Ctx* ctx, const ModelP& M, float* const* other, double* out_per_mode, HistBufs& hb,
                          bool self, bool shard_rows = false) {
  const int RR = M.rank * M.rank;
  if (small_model(M)) {
    SmallGrams g{};
    for (int k = 0; k < M.ndim; ++k) {
      g.A[k] = M.A[k];
      g.B1[k] = self ? M.A[k] : other[k];
      g.rows[k] = M.dims[k];
    }
    gram_small_enqueue(ctx, g, M.ndim, M.rank, M.ldr, out_per_mode, nullptr);
    return;
  }
  const bool shard = shard_rows && row_sharded(ctx, M);
  for (int k = 0; k < M.ndim; ++k) {
    int64_t lo, hi;
    double* o = out_per_mode + (int64_t)k * RR;
    if (!gram_rows(ctx, M, shard, k, &lo, &hi, o, nullptr)) continue;
    const size_t off = (size_t)lo * M.ldr;
    const float* A = M.A[k] + off;
    const float* B = (self ? M.A[k] : other[k]) + off;
    gram_enqueue(ctx, A, B, hi - lo, M.rank, M.ldr, o, hb.scratch);
  }
  if (shard) comm_allreduce_sum(ctx, out_per_mode, (size_t)M.ndim * RR);
}

// P_m = A_m'A_m and C_m = Aold_m'A_m for every mode, one pass over each A_m.
static void grams_pc_enqueue(Ctx* ctx, const ModelP& M, float* const* old, HistBufs& hb, bool shard_rows = false) {
  const int RR = M.rank * M.rank;
  if (small_model(M)) {
    SmallGrams g{};
    for (int k = 0; k < M.ndim; ++k) {
      g.A[k] = M.A[k];
      g.B1[k] = M.A[k];
      g.B2[k] = old[k];
      g.rows[k] = M.dims[k];
    }
    gram_small_enqueue(ctx, g, M.ndim, M.rank, M.ldr, hb.P.as<double>(), hb.C.as<double>());
    return;
  }
  const bool shard = shard_rows && row_sharded(ctx, M);
  for (int k = 0; k < M.ndim; ++k) {
    int64_t lo, hi;
    double* oP = hb.P.as<double>() + (int64_t)k * RR;
    double* oC = hb.C.as<double>() + (int64_t)k * RR;
    if (!gram_rows(ctx, M, shard, k, &lo, &hi, oP, oC)) continue;
    const size_t off = (size_t)lo * M.ldr;
    gram2_enqueue(ctx, M.A[k] + off, old[k] + off, hi - lo, M.rank, M.ldr, oP, oC, hb.scratch);
  }
  if (shard) {
    comm_allreduce_sum(ctx, hb.P.as<double>(), (size_t)M.ndim * RR);
    comm_allreduce_sum(ctx, hb.C.as<double>(), (size_t)M.ndim * RR);
  }
}

// Device objective for a fixed sample set: returns data term + history + regs.
struct ObjectiveParts {
  double data = 0, hist = 0, trace = 0;
};

static long long code_of(long long ev, int sub) { return ev * 4 + sub; }

static const LossP kIdentityLoss = {OGCP_IDENTITY, 1e-10f, 1e-10};

// sum over (i, j) of s_i s_j prod_m P_m[i][j]: ||M||^2 of the model (kernels.py:143-145).
static double model_sq_host(const std::vector<double>& P, int ndim, int R, const double* s) {
  const size_t RR = (size_t)R * R;
  double acc = 0.0;
  for (int i = 0; i < R; ++i) {
    double row = 0.0;
    for (int j = 0; j < R; ++j) {
      double g = 1.0;
      for (int m = 0; m < ndim; ++m) g *= P[m * RR + (size_t)i * R + j];
      row += g * s[j];
    }
    acc += s[i] * row;
  }
  return acc;
}

struct FactorWork {
  DevBuf grads;
  HistBufs hb;
  SampleBufs obj;
  DrawPipe grad;
};

static FactorWork& factor_work() {
  static thread_local FactorWork w;
  return w;
}

static void hist_alloc(HistBufs& hb, int ndim, int R) {
  const size_t RR = (size_t)R * R;
  hb.P.ensure(ndim * RR * 8);
  hb.C.ensure(ndim * RR * 8);
  hb.Poo.ensure(ndim * RR * 8);
  hb.S.ensure(RR * 8);
  hb.Mk.ensure(ndim * RR * 4);
  hb.Nk.ensure(ndim * RR * 4);
}

// ============================================================= solve_weights
static void solve_weights_impl(Ctx* ctx, const Slice* X, const ogcp_solver_config* cfg, const ogcp_loss* loss,
                               int64_t t, const ogcp_model* mdl, const double* s_init, double* s_out,
                               ogcp_trace* trace) {
  ModelP M = model_of(mdl);
  check_model_slice(M, X);
  LossP L = loss_of(loss);
  const int R = M.rank, ldr = M.ldr;
  const uint64_t seed = cfg->samples.seed;
  cudaStream_t st = ctx->stream;
  // state: s u v s_o u_o v_o (double ldr each) + s_f float ldr
  ctx->wsolve.ensure((size_t)ldr * (6 * 8 + 4));
  double* ws = ctx->wsolve.as<double>();
  float* s_f = reinterpret_cast<float*>(ws + 6 * ldr);
  std::vector<double> h(6 * ldr, 0.0);
  std::vector<double> s(R, 0.0);
  if (cfg->warm_start_weights && s_init)
    for (int r = 0; r < R; ++r) s[r] = s_init[r];
  for (int r = 0; r < R; ++r) {
    h[r] = s[r];
    h[3 * ldr + r] = s[r];  // snapshot of the entry state (solvers.py:217-218)
  }
  OGCP_CUDA(cudaMemcpyAsync(ws, h.data(), 6 * ldr * 8, cudaMemcpyHostToDevice, st));
  upload_weights(ctx, s.data(), R, ldr, s_f);
  double rate = cfg->rate_weights;

  int64_t po, qo, p, q;
  resolve_counts(cfg->samples.obj_nonzeros, cfg->samples.obj_zeros, X, &po, &qo);
  resolve_counts(cfg->samples.grad_nonzeros, cfg->samples.grad_zeros, X, &p, &q);
  static thread_local SampleBufs obj;
  static thread_local DrawPipe grad;
  const bool dense = dense_mode(cfg, L.kind);
  SamplesP So{};
  int64_t budget = 0;
  if (!dense) {
    if (po > 0 || p > 0) x_domain_check(X, L.kind);
    const bool semi = cfg->samples.semi_stratified != 0;
    draw_sync(ctx, X, keyed(seed, {t, 2}), po, qo, cfg->samples.max_rejects, obj, semi);
    So = sharded(ctx, obj.sample_set(X));
    precheck_draw(X, p, semi ? 0 : q);
    grad.size(p, q, X->ndim, p > 0 && use_merged(ctx, X, p), semi);
    if (grad.merged()) prepare_buckets(ctx, X, M.ldr);
    budget = budget_of(q, cfg->samples.max_rejects);
  }
  ctx->partials.ensure((size_t)kNumSMs * 8 * ldr * 8 + 64);
  double* part = ctx->partials.as<double>();
  ctx->scalars.ensure(64 * 8 + ldr * 8);
  double* dsc = ctx->scalars.as<double>();
  double* gsum = dsc + 64;  // multi-GPU: the R-vector gradient summed across ranks
  double* hsc = ctx->host_scalars;

  // dense-Gaussian (solvers.py:182-185, 220-224): with the factors fixed the
  // Grams and b = Z' vec(X) are constant, so each step is an R-vector update
  // and the objective ||X||^2 - 2 s'b + s'(hadamard P)s + (mu/2)||s||^2.
  std::vector<double> Ph, bh(R, 0.0);
  double* bdev = nullptr;
  HistBufs* hb = nullptr;
  if (dense) {
    hb = &factor_work().hb;
    hist_alloc(*hb, M.ndim, R);
    grams_enqueue(ctx, M, nullptr, hb->P.as<double>(), *hb, true);
    ctx->dense.ensure((size_t)2 * ldr * 8);
    bdev = ctx->dense.as<double>();
    const SamplesP Sx = all_nonzeros(ctx, X, 1.0);
    const int nb = wgrad_enqueue(ctx, Sx, M, s_f, kIdentityLoss, part, code_of(0, 1));
    sum_partials_enqueue(ctx, part, nb, ldr, bdev);
    if (Sx.shard_world > 1) comm_allreduce_sum(ctx, bdev, (size_t)ldr);
    Ph.resize((size_t)M.ndim * R * R);
    OGCP_CUDA(cudaMemcpyAsync(Ph.data(), hb->P.ptr, Ph.size() * 8, cudaMemcpyDeviceToHost, st));
    OGCP_CUDA(cudaMemcpyAsync(bh.data(), bdev, R * 8, cudaMemcpyDeviceToHost, st));
    OGCP_CUDA(cudaStreamSynchronize(st));
  }

  long long ev = 1;
  auto fest_fn = [&]() -> double {
    if (dense) {
      OGCP_CUDA(cudaMemcpyAsync(hsc + 8, ws, R * 8, cudaMemcpyDeviceToHost, st));
      OGCP_CUDA(cudaStreamSynchronize(st));
      const double* sv = hsc + 8;
      double sb = 0.0, ss = 0.0;
      for (int r = 0; r < R; ++r) {
        sb += sv[r] * bh[r];
        ss += sv[r] * sv[r];
      }
      return X->frob_sq - 2.0 * sb + model_sq_host(Ph, M.ndim, R, sv) + 0.5 * cfg->reg_weights * ss;
    }
    reset_flags(ctx);
    const long long c = code_of(ev++, 1);
    int nb = objective_enqueue(ctx, So, M, s_f, L, part, c);
    sum_partials_enqueue(ctx, part, nb, 1, dsc);
    comm_allreduce_sum(ctx, dsc, 1);
    OGCP_CUDA(cudaMemcpyAsync(hsc, dsc, 8, cudaMemcpyDeviceToHost, st));
    OGCP_CUDA(cudaMemcpyAsync(hsc + 8, ws, R * 8, cudaMemcpyDeviceToHost, st));
    comm_sync_flags(ctx);
    fetch_flags(ctx);
    OGCP_CUDA(cudaStreamSynchronize(st));
    check_flags(ctx, X, L.kind, budget, "temporal weight solve", t);
    double val = hsc[0];
    if (cfg->reg_weights) {
      double ss = 0.0;
      for (int r = 0; r < R; ++r) ss += hsc[8 + r] * hsc[8 + r];
      val += 0.5 * cfg->reg_weights * ss;
    }
    return val;
  };

  double fest = fest_fn();
  std::vector<double> objv{fest};
  int64_t i = 0;
  int epochs = 0, rejections = 0;
  for (int epoch = 0; epoch < cfg->max_epochs_weights; ++epoch) {
    if (!(fest > cfg->tol_weights)) break;
    const double fold = fest;
    SlackScope slack_scope(ctx);  // a shortfall raises the slack for this retry only
    for (int attempt = 0;; ++attempt) {
      reset_flags(ctx);
      const long long ev0 = ev;
      if (!dense)
        grad.begin_epoch(ctx, X, [&](int it) { return keyed(seed, {t, 1, epoch, it}); }, cfg->iters_weights, budget,
                         code_of(ev0, 0));
      for (int it = 0; it < cfg->iters_weights; ++it) {
        const long long e = ev++;
        const int64_t cnt = i + it + 1;
        const double rate_i = rate * std::sqrt(1.0 - std::pow(cfg->beta2, (double)cnt)) /
                              (1.0 - std::pow(cfg->beta1, (double)cnt));
        if (dense) {
          dense_wgrad_enqueue(ctx, M.ndim, R, ldr, hb->P.as<double>(), bdev, ws, part);
          weight_step_enqueue(ctx, part, 1, R, ldr, ws, s_f, cfg->reg_weights, rate_i, cfg->beta1, cfg->beta2,
                              cfg->adam_eps, cfg->lower_bound, code_of(e, 2));
          continue;
        }
        if (it + 1 < cfg->iters_weights)
          grad.issue(ctx, X, keyed(seed, {t, 1, epoch, it + 1}), budget, code_of(e + 1, 0), (it + 1) & 1);
        SamplesP Sg = sharded(ctx, grad.take(ctx, it & 1));
        // one GPU: the weight step runs in the tail of the K2w launch (last block)
        WStep wstep{R, ldr, ws, s_f, cfg->reg_weights, rate_i, cfg->beta1, cfg->beta2, cfg->adam_eps,
                    cfg->lower_bound, code_of(e, 2), ctx->wticket()};
        bool stepped = false;
        int nb = wgrad_enqueue(ctx, Sg, M, s_f, L, part, code_of(e, 1), ctx->world == 1 ? &wstep : nullptr, &stepped);
        if (stepped) continue;
        const double* gparts = part;
        if (ctx->world > 1) {  // sum the shard gradients across ranks, then the replicated step
          sum_partials_enqueue(ctx, part, nb, ldr, gsum);
          comm_allreduce_sum(ctx, gsum, (size_t)ldr);
          gparts = gsum;
          nb = 1;
        }
        weight_step_enqueue(ctx, gparts, nb, R, ldr, ws, s_f, cfg->reg_weights, rate_i, cfg->beta1, cfg->beta2,
                            cfg->adam_eps, cfg->lower_bound, code_of(e, 2));
      }
      comm_sync_flags(ctx);
      fetch_flags(ctx);
      OGCP_CUDA(cudaStreamSynchronize(st));
      int r = check_flags(ctx, X, L.kind, budget, "temporal weight solve", t);
      if (r == 0) break;
      // shortfall: restore the epoch-start snapshot and redo with more candidates
      // (r == 2: a merged-draw counter wrapped; redo with per-draw evaluation)
      if (r == 2) grad.size(p, q, X->ndim, false, cfg->samples.semi_stratified != 0);
      else ctx->slack *= 4.0;
      OGCP_CUDA(cudaMemcpyAsync(ws, ws + 3 * ldr, 3 * ldr * 8, cudaMemcpyDeviceToDevice, st));
      OGCP_CUDA(cudaMemcpyAsync(hsc, ws, ldr * 8, cudaMemcpyDeviceToHost, st));
      OGCP_CUDA(cudaStreamSynchronize(st));
      upload_weights(ctx, hsc, R, ldr, s_f);
      ev = ev0;
      if (attempt > 8) throw Error(OGCP_E_INTERNAL, "sampler could not provision enough candidates");
    }
    i += cfg->iters_weights;
    fest = fest_fn();
    if (!std::isfinite(fest))
      throw Error(OGCP_E_DIVERGENCE, "temporal weight solve diverged at slice " + std::to_string(t));
    if (fest > fold) {
      // reject: restore u, v, s and decay the rate (adam.py:91-94)
      OGCP_CUDA(cudaMemcpyAsync(ws, ws + 3 * ldr, 3 * ldr * 8, cudaMemcpyDeviceToDevice, st));
      rate *= cfg->rate_decay;
      fest = fold;
      i -= cfg->iters_weights;
      ++rejections;
    } else {
      OGCP_CUDA(cudaMemcpyAsync(ws + 3 * ldr, ws, 3 * ldr * 8, cudaMemcpyDeviceToDevice, st));
    }
    OGCP_CUDA(cudaMemcpyAsync(hsc, ws, ldr * 8, cudaMemcpyDeviceToHost, st));
    OGCP_CUDA(cudaStreamSynchronize(st));
    upload_weights(ctx, hsc, R, ldr, s_f);
    ++epochs;
    objv.push_back(fest);
  }
  OGCP_CUDA(cudaMemcpyAsync(hsc, ws, ldr * 8, cudaMemcpyDeviceToHost, st));
  OGCP_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < R; ++r) s_out[r] = hsc[r];
  if (trace) {
    trace->n_objective = 0;
    for (size_t j = 0; j < objv.size() && (int)j <= cfg->max_epochs_weights; ++j)
      trace->objective[trace->n_objective++] = objv[j];
    trace->epochs = epochs;
    trace->rejections = rejections;
  }
}

// ============================================================= solve_factors

static void window_upload(Ctx* ctx, HistBufs& hb, int R, const double* window_s, const int64_t* window_ids, int H,
                          double decay, int64_t t) {
  hb.Ws.ensure((size_t)std::max(H, 1) * R * 8);
  hb.coef.ensure((size_t)std::max(H, 1) * 8);
  std::vector<double> coef(std::max(H, 1), 0.0);
  for (int h = 0; h < H; ++h) coef[h] = std::pow(decay, (double)(t - window_ids[h]));
  if (H > 0) OGCP_CUDA(cudaMemcpyAsync(hb.Ws.ptr, window_s, (size_t)H * R * 8, cudaMemcpyHostToDevice, ctx->stream));
  OGCP_CUDA(cudaMemcpyAsync(hb.coef.ptr, coef.data(), coef.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
}

__global__ void k_window_matrix(int R, int H, const double* __restrict__ Ws, const double* __restrict__ coef,
                                double* __restrict__ S) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int i = e / R, j = e % R;
    double acc = 0.0;
    for (int h = 0; h < H; ++h) acc += coef[h] * (Ws[(int64_t)h * R + i] * Ws[(int64_t)h * R + j]);
    S[e] = acc;
  }
}

__global__ void k_trace_sum(int ndim, int R, const double* __restrict__ P, double* __restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  double t = 0.0;
  for (int m = 0; m < ndim; ++m)
    for (int i = 0; i < R; ++i) t += P[(int64_t)m * R * R + i * R + i];
  *out = t;
}

// F(factors) = data term on the fixed objective set + (w/2) history + (lambda/2) sum ||A||^2.
// dense_s (host weights) selects the exact Gaussian residual ||X||^2 - 2<X,M> + ||M||^2
// (kernels.py:135-146) as the data term instead of the sampled estimate.
static double factor_objective(Ctx* ctx, const Slice* X, const SamplesP& So, const ModelP& M, const float* s_f,
                               const LossP& L, float* const* old_factors, int H, const ogcp_solver_config* cfg,
                               HistBufs& hb, long long code, int64_t budget, int64_t t,
                               const char* what = "factor solve", const double* dense_s = nullptr) {
  cudaStream_t st = ctx->stream;
  const int RR = M.rank * M.rank;
  double* part = ctx->partials.as<double>();
  double* dsc = ctx->scalars.as<double>();
  double* hsc = ctx->host_scalars;
  const bool dense = dense_s != nullptr;
  reset_flags(ctx);
  const SamplesP S = dense ? all_nonzeros(ctx, X, 1.0) : So;
  int nb = objective_enqueue(ctx, S, M, s_f, dense ? kIdentityLoss : L, part, code);
  sum_partials_enqueue(ctx, part, nb, 1, dsc);
  const bool collective = S.shard_world > 1;
  if (collective) comm_allreduce_sum(ctx, dsc, 1);  // the data term is per-shard; Grams are replicated
  const bool hist = cfg->hist_weight != 0.0 && H > 0;
  const bool reg = cfg->reg_factors != 0.0;
  std::vector<double> Ph;
  if (hist || reg || dense) {
    if (hist) grams_pc_enqueue(ctx, M, old_factors, hb, collective);
    else grams_enqueue(ctx, M, nullptr, hb.P.as<double>(), hb, true, collective);
    if (reg) {
      k_trace_sum<<<1, 1, 0, st>>>(M.ndim, M.rank, hb.P.as<double>(), dsc + 2);
      ctx->count();
    }
    if (hist) {
      hist_penalty_enqueue(ctx, M.ndim, M.rank, hb.Poo.as<double>(), hb.C.as<double>(), hb.P.as<double>(),
                           hb.Ws.as<double>(), hb.coef.as<double>(), H, dsc + 1);
    }
    if (dense) {
      Ph.resize((size_t)M.ndim * RR);
      OGCP_CUDA(cudaMemcpyAsync(Ph.data(), hb.P.ptr, Ph.size() * 8, cudaMemcpyDeviceToHost, st));
    }
  }
  OGCP_CUDA(cudaMemcpyAsync(hsc, dsc, 3 * 8, cudaMemcpyDeviceToHost, st));
  if (collective) comm_sync_flags(ctx);
  fetch_flags(ctx);
  OGCP_CUDA(cudaStreamSynchronize(st));
  check_flags(ctx, X, L.kind, budget, what, t);
  double val = hsc[0];
  if (dense) val = X->frob_sq - 2.0 * hsc[0] + model_sq_host(Ph, M.ndim, M.rank, dense_s);
  if (hist) val += 0.5 * cfg->hist_weight * hsc[1];
  if (reg) val += 0.5 * cfg->reg_factors * hsc[2];
  return val;
}

static void adam_epoch(Ctx* ctx, const ModelP& M, float* const* A, ogcp_adam_state* ad, bool passed) {
  for (int k = 0; k < M.ndim; ++k) {
    const size_t b = (size_t)M.dims[k] * M.ldr * 4;
    if (passed) {
      OGCP_CUDA(cudaMemcpyAsync(ad->u_o[k], ad->u[k], b, cudaMemcpyDeviceToDevice, ctx->stream));
      OGCP_CUDA(cudaMemcpyAsync(ad->v_o[k], ad->v[k], b, cudaMemcpyDeviceToDevice, ctx->stream));
      OGCP_CUDA(cudaMemcpyAsync(ad->a_o[k], A[k], b, cudaMemcpyDeviceToDevice, ctx->stream));
    } else {
      OGCP_CUDA(cudaMemcpyAsync(ad->u[k], ad->u_o[k], b, cudaMemcpyDeviceToDevice, ctx->stream));
      OGCP_CUDA(cudaMemcpyAsync(ad->v[k], ad->v_o[k], b, cudaMemcpyDeviceToDevice, ctx->stream));
      OGCP_CUDA(cudaMemcpyAsync(A[k], ad->a_o[k], b, cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
}

// One factor iteration: draw -> K2/K3 -> (K4 Grams -> coefficients) -> K5 per mode.
// dense_s (device double weights) selects the exact Gaussian gradient
// 2 (A_k (Gamma_k o s s') - mttkrp(X, k) diag(s)) (kernels.py:117-132): the
// scatter runs over every stored nonzero with y = -2 x and the model term
// joins the history coefficients of K5.
static void factor_iteration(Ctx* ctx, const Slice* X, const ModelP& M, float* const* A, const float* s_f,
                             const LossP& L, float* const* old_factors, bool hist, const ogcp_solver_config* cfg,
                             ogcp_adam_state* ad, double rate_i, const SamplesP* Sdrawn, FactorWork& W,
                             long long ev, const double* dense_s = nullptr) {
  const int RR = M.rank * M.rank;
  const bool dense = dense_s != nullptr;
  float* gp[kMaxModes];
  size_t off = 0;
  for (int k = 0; k < M.ndim; ++k) {
    gp[k] = W.grads.as<float>() + off;
    off += (size_t)M.dims[k] * M.ldr;
  }
  if (dense) {
    sgrad_enqueue(ctx, all_nonzeros(ctx, X, -2.0), M, s_f, kIdentityLoss, gp, code_of(ev, 1));
  } else {
    sgrad_enqueue(ctx, *Sdrawn, M, s_f, L, gp, code_of(ev, 1));
  }
  // multi-GPU: sum of the shard gradients -- all of it for small models (replicated
  // K5), else each mode's row block onto its owner (owner-computes K5)
  const bool rowshard = row_sharded(ctx, M);
  if (rowshard) comm_reduce_rows(ctx, gp, M.dims, M.ndim, M.ldr);
  else comm_allreduce_sum(ctx, W.grads.as<float>(), off);
  const bool coeffs = hist || dense;
  if (coeffs && hist && small_model(M) && !rowshard) {
    // small models: the history coefficients run in the tail of the Gram launch
    SmallGrams g{};
    for (int k = 0; k < M.ndim; ++k) {
      g.A[k] = M.A[k];
      g.B1[k] = M.A[k];
      g.B2[k] = old_factors[k];
      g.rows[k] = M.dims[k];
    }
    CoeffTail tail{W.hb.S.as<double>(), cfg->hist_weight, dense_s, 2.0, W.hb.Mk.as<float>(), W.hb.Nk.as<float>(),
                   ctx->wticket() + 2};
    gram_small_enqueue(ctx, g, M.ndim, M.rank, M.ldr, W.hb.P.as<double>(), W.hb.C.as<double>(), &tail);
  } else if (coeffs) {
    if (hist) grams_pc_enqueue(ctx, M, old_factors, W.hb, true);
    else grams_enqueue(ctx, M, nullptr, W.hb.P.as<double>(), W.hb, true, true);
    hist_coeffs_enqueue(ctx, M.ndim, M.rank, W.hb.P.as<double>(), hist ? W.hb.C.as<double>() : nullptr,
                        hist ? W.hb.S.as<double>() : nullptr, cfg->hist_weight, W.hb.Mk.as<float>(),
                        W.hb.Nk.as<float>(), dense_s, 2.0);
  }
  if (small_model(M)) {  // every mode in one launch
    K5Modes km{};
    for (int k = 0; k < M.ndim; ++k) {
      km.A[k] = A[k];
      km.Aold[k] = hist ? old_factors[k] : nullptr;
      km.G[k] = gp[k];
      km.u[k] = ad->u[k];
      km.v[k] = ad->v[k];
      km.Mk[k] = coeffs ? W.hb.Mk.as<float>() + (size_t)k * RR : nullptr;
      km.Nk[k] = coeffs ? W.hb.Nk.as<float>() + (size_t)k * RR : nullptr;
      km.rows[k] = M.dims[k];
    }
    factor_update_modes_enqueue(ctx, km, M.ndim, M.rank, M.ldr, cfg->reg_factors, rate_i, cfg->beta1, cfg->beta2,
                                cfg->adam_eps, cfg->lower_bound, code_of(ev, 2));
    return;
  }
  for (int k = 0; k < M.ndim; ++k) {
    int64_t lo = 0, hi = M.dims[k];
    if (rowshard) comm_row_range(M.dims[k], ctx->rank, ctx->world, &lo, &hi);
    const size_t o = (size_t)lo * M.ldr;
    factor_update_enqueue(ctx, hi - lo, M.rank, M.ldr, A[k] + o, hist ? old_factors[k] + o : nullptr, gp[k] + o,
                          ad->u[k] + o, ad->v[k] + o, coeffs ? W.hb.Mk.as<float>() + (size_t)k * RR : nullptr,
                          coeffs ? W.hb.Nk.as<float>() + (size_t)k * RR : nullptr, cfg->reg_factors, rate_i,
                          cfg->beta1, cfg->beta2, cfg->adam_eps, cfg->lower_bound, code_of(ev, 2));
  }
  if (rowshard) comm_gather_rows(ctx, A, M.dims, M.ndim, M.ldr);  // every rank gets the new factors
}



static void solve_factors_impl(Ctx* ctx, const Slice* X, const ogcp_solver_config* cfg, const ogcp_loss* loss,
                               int64_t t, const ogcp_model* mdl, float* const* old_factors, const double* weights,
                               const double* window_s, const int64_t* window_ids, int H, ogcp_adam_state* ad,
                               int64_t* iteration, ogcp_trace* trace) {
  ModelP M = model_of(mdl);
  check_model_slice(M, X);
  LossP L = loss_of(loss);
  cudaStream_t st = ctx->stream;
  const uint64_t seed = cfg->samples.seed;
  FactorWork& W = factor_work();
  float* const* A = mdl->factors;
  ctx->wsolve.ensure((size_t)M.ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * M.ldr);
  upload_weights(ctx, weights, M.rank, M.ldr, s_f);
  ctx->partials.ensure((size_t)kNumSMs * 8 * M.ldr * 8 + 64);
  ctx->scalars.ensure(64 * 8);
  size_t gtot = 0;
  for (int k = 0; k < M.ndim; ++k) gtot += (size_t)M.dims[k] * M.ldr;
  W.grads.ensure(gtot * 4);
  hist_alloc(W.hb, M.ndim, M.rank);
  const bool dense = dense_mode(cfg, L.kind);
  const double* s_dev = dense ? dense_upload_s(ctx, weights, M.rank, M.ldr) : nullptr;
  const bool hist = cfg->hist_weight != 0.0 && H > 0;
  if (hist && !old_factors) throw Error(OGCP_E_DATA, "history terms require the previous-step factors");
  window_upload(ctx, W.hb, M.rank, window_s, window_ids, H, cfg->hist_decay, t);
  if (hist) {
    k_window_matrix<<<1, 256, 0, st>>>(M.rank, H, W.hb.Ws.as<double>(), W.hb.coef.as<double>(), W.hb.S.as<double>());
    ctx->count();
    // Poo = Aold'Aold, constant during the solve
    for (int k = 0; k < M.ndim; ++k)
      gram_enqueue(ctx, old_factors[k], old_factors[k], M.dims[k], M.rank, M.ldr,
                   W.hb.Poo.as<double>() + (size_t)k * M.rank * M.rank, W.hb.scratch);
  }
  // entry snapshot (solvers.py:303-305)
  adam_epoch(ctx, M, A, ad, true);

  int64_t po, qo, p, q;
  resolve_counts(cfg->samples.obj_nonzeros, cfg->samples.obj_zeros, X, &po, &qo);
  resolve_counts(cfg->samples.grad_nonzeros, cfg->samples.grad_zeros, X, &p, &q);
  SamplesP So{};
  int64_t budget = 0;
  if (!dense) {  // the dense-Gaussian solve draws nothing (solvers.py:310-329)
    if (po > 0 || p > 0) x_domain_check(X, L.kind);
    const bool semi = cfg->samples.semi_stratified != 0;
    draw_sync(ctx, X, keyed(seed, {t, 4}), po, qo, cfg->samples.max_rejects, W.obj, semi);
    So = sharded(ctx, W.obj.sample_set(X));
    precheck_draw(X, p, semi ? 0 : q);
    W.grad.size(p, q, X->ndim, p > 0 && use_merged(ctx, X, p), semi);
    if (W.grad.merged()) prepare_buckets(ctx, X, M.ldr);
    budget = budget_of(q, cfg->samples.max_rejects);
  }
  const double* dense_w = dense ? weights : nullptr;

  long long ev = 1;
  double fest = factor_objective(ctx, X, So, M, s_f, L, old_factors, H, cfg, W.hb, code_of(ev++, 1), budget, t,
                                 "factor solve", dense_w);
  std::vector<double> objv{fest};
  int64_t iter = *iteration;
  int epochs = 0, rejections = 0;
  for (int epoch = 0; epoch < cfg->max_epochs_factors; ++epoch) {
    if (!(fest > cfg->tol_factors)) break;
    const double fold = fest;
    SlackScope slack_scope(ctx);  // a shortfall raises the slack for this retry only
    for (int attempt = 0;; ++attempt) {
      reset_flags(ctx);
      const long long ev0 = ev;
      if (!dense)
        W.grad.begin_epoch(ctx, X, [&](int it) { return keyed(seed, {t, 3, epoch, it}); }, cfg->iters_factors,
                           budget, code_of(ev0, 0));
      for (int it = 0; it < cfg->iters_factors; ++it) {
        const int64_t cnt = iter + it + 1;
        const double rate_i = ad->rate * std::sqrt(1.0 - std::pow(cfg->beta2, (double)cnt)) /
                              (1.0 - std::pow(cfg->beta1, (double)cnt));
        SamplesP Sg{};
        if (!dense) {
          if (it + 1 < cfg->iters_factors)
            W.grad.issue(ctx, X, keyed(seed, {t, 3, epoch, it + 1}), budget, code_of(ev + 1, 0), (it + 1) & 1);
          Sg = sharded(ctx, W.grad.take(ctx, it & 1));
        }
        factor_iteration(ctx, X, M, A, s_f, L, old_factors, hist, cfg, ad, rate_i, &Sg, W, ev++,
                         dense ? s_dev : nullptr);
      }
      comm_sync_flags(ctx);
      fetch_flags(ctx);
      OGCP_CUDA(cudaStreamSynchronize(st));
      int r = check_flags(ctx, X, L.kind, budget, "factor solve", t);
      if (r == 0) break;
      if (r == 2) W.grad.size(p, q, X->ndim, false, cfg->samples.semi_stratified != 0);
      else ctx->slack *= 4.0;
      adam_epoch(ctx, M, A, ad, false);  // restore the epoch-start state (no rate decay)
      ev = ev0;
      if (attempt > 8) throw Error(OGCP_E_INTERNAL, "sampler could not provision enough candidates");
    }
    iter += cfg->iters_factors;
    fest = factor_objective(ctx, X, So, M, s_f, L, old_factors, H, cfg, W.hb, code_of(ev++, 1), budget, t,
                            "factor solve", dense_w);
    if (!std::isfinite(fest)) throw Error(OGCP_E_DIVERGENCE, "factor solve diverged at slice " + std::to_string(t));
    if (fest > fold) {
      adam_epoch(ctx, M, A, ad, false);
      ad->rate *= cfg->rate_decay;
      fest = fold;
      iter -= cfg->iters_factors;
      ++rejections;
    } else {
      adam_epoch(ctx, M, A, ad, true);
    }
    ++epochs;
    objv.push_back(fest);
  }
  if (row_sharded(ctx, M)) {  // owners hold their rows' Adam moments: leave every rank the full state
    comm_gather_rows(ctx, ad->u, M.dims, M.ndim, M.ldr);
    comm_gather_rows(ctx, ad->v, M.dims, M.ndim, M.ldr);
  }
  OGCP_CUDA(cudaStreamSynchronize(st));
  *iteration = iter;
  if (trace) {
    trace->n_objective = 0;
    for (size_t j = 0; j < objv.size() && (int)j <= cfg->max_epochs_factors; ++j)
      trace->objective[trace->n_objective++] = objv[j];
    trace->epochs = epochs;
    trace->rejections = rejections;
  }
}

// ============================================================== solve_static
// Static GCP-SGD over weights and every factor jointly (solvers.py:371-493):
// one draw per iteration feeds both the factor scatter (K3) and the weight
// MTTKRP (K3w); the weights keep the fp64 temporal-row Adam, the factors the
// fp32 row Adam, both on one step counter and one (decaying) rate.
static void solve_static_impl(Ctx* ctx, const Slice* X, const ogcp_solver_config* cfg, const ogcp_loss* loss,
                              int64_t seed_key, const ogcp_model* mdl, double* weights, ogcp_adam_state* ad,
                              int32_t max_epochs, int32_t iters, double tol, ogcp_trace* trace) {
  ModelP M = model_of(mdl);
  check_model_slice(M, X);
  LossP L = loss_of(loss);
  const int R = M.rank, ldr = M.ldr;
  cudaStream_t st = ctx->stream;
  const uint64_t seed = cfg->samples.seed;
  FactorWork& W = factor_work();
  float* const* A = mdl->factors;
  // weight state: s u v s_o u_o v_o (double ldr each) + s_f float ldr; u = v = 0
  ctx->wsolve.ensure((size_t)ldr * (6 * 8 + 4));
  double* ws = ctx->wsolve.as<double>();
  float* s_f = reinterpret_cast<float*>(ws + 6 * ldr);
  {
    std::vector<double> h(6 * ldr, 0.0);
    for (int r = 0; r < R; ++r) h[r] = h[3 * ldr + r] = weights[r];
    OGCP_CUDA(cudaMemcpyAsync(ws, h.data(), 6 * ldr * 8, cudaMemcpyHostToDevice, st));
    upload_weights(ctx, weights, R, ldr, s_f);
  }
  ctx->partials.ensure((size_t)kNumSMs * 8 * ldr * 8 + 64);
  ctx->scalars.ensure(64 * 8 + ldr * 8);
  double* part = ctx->partials.as<double>();
  double* gsum = ctx->scalars.as<double>() + 64;
  double* hsc = ctx->host_scalars;
  size_t gtot = 0;
  for (int k = 0; k < M.ndim; ++k) gtot += (size_t)M.dims[k] * ldr;
  W.grads.ensure(gtot * 4);
  hist_alloc(W.hb, M.ndim, R);
  adam_epoch(ctx, M, A, ad, true);  // adam.update(variables, True) at entry

  int64_t po, qo, p, q;
  resolve_counts(cfg->samples.obj_nonzeros, cfg->samples.obj_zeros, X, &po, &qo);
  resolve_counts(cfg->samples.grad_nonzeros, cfg->samples.grad_zeros, X, &p, &q);
  const bool dense = dense_mode(cfg, L.kind);
  SamplesP So{};
  int64_t budget = 0;
  if (!dense) {
    if (po > 0 || p > 0) x_domain_check(X, L.kind);
    const bool semi = cfg->samples.semi_stratified != 0;
    draw_sync(ctx, X, keyed(seed, {seed_key, 8}), po, qo, cfg->samples.max_rejects, W.obj, semi);
    So = sharded(ctx, W.obj.sample_set(X));
    precheck_draw(X, p, semi ? 0 : q);
    W.grad.size(p, q, X->ndim, p > 0 && use_merged(ctx, X, p), semi);
    if (W.grad.merged()) prepare_buckets(ctx, X, M.ldr);
    budget = budget_of(q, cfg->samples.max_rejects);
  }
  const char* what = "static solve";
  double* bdev = nullptr;
  if (dense) {
    ctx->dense.ensure((size_t)2 * ldr * 8);
    bdev = ctx->dense.as<double>();
  }

  long long ev = 1;
  std::vector<double> cur_w(R);
  auto fest_fn = [&]() -> double {
    OGCP_CUDA(cudaMemcpyAsync(hsc + 8, ws, R * 8, cudaMemcpyDeviceToHost, st));
    OGCP_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < R; ++r) cur_w[r] = hsc[8 + r];
    double v = factor_objective(ctx, X, So, M, s_f, L, nullptr, 0, cfg, W.hb, code_of(ev++, 1), budget, seed_key,
                                what, dense ? cur_w.data() : nullptr);
    if (cfg->reg_weights) {
      double ss = 0.0;
      for (int r = 0; r < R; ++r) ss += cur_w[r] * cur_w[r];
      v += 0.5 * cfg->reg_weights * ss;
    }
    return v;
  };
  auto weights_epoch = [&](bool passed) {
    if (passed) OGCP_CUDA(cudaMemcpyAsync(ws + 3 * ldr, ws, 3 * ldr * 8, cudaMemcpyDeviceToDevice, st));
    else OGCP_CUDA(cudaMemcpyAsync(ws, ws + 3 * ldr, 3 * ldr * 8, cudaMemcpyDeviceToDevice, st));
    OGCP_CUDA(cudaMemcpyAsync(hsc, ws, ldr * 8, cudaMemcpyDeviceToHost, st));
    OGCP_CUDA(cudaStreamSynchronize(st));
    upload_weights(ctx, hsc, R, ldr, s_f);
  };

  double fest = fest_fn();
  std::vector<double> objv{fest};
  int64_t iter = 0;
  int epochs = 0, rejections = 0;
  float* gp[kMaxModes];
  {
    size_t off = 0;
    for (int k = 0; k < M.ndim; ++k) {
      gp[k] = W.grads.as<float>() + off;
      off += (size_t)M.dims[k] * ldr;
    }
  }
  for (int epoch = 0; epoch < max_epochs; ++epoch) {
    if (!(fest > tol)) break;
    const double fold = fest;
    SlackScope slack_scope(ctx);  // a shortfall raises the slack for this retry only
    for (int attempt = 0;; ++attempt) {
      reset_flags(ctx);
      const long long ev0 = ev;
      if (!dense)
        W.grad.begin_epoch(ctx, X, [&](int it) { return keyed(seed, {seed_key, 7, epoch, it}); }, iters, budget,
                           code_of(ev0, 0));
      for (int it = 0; it < iters; ++it) {
        const long long e = ev++;
        const int64_t cnt = iter + it + 1;
        const double rate_i = ad->rate * std::sqrt(1.0 - std::pow(cfg->beta2, (double)cnt)) /
                              (1.0 - std::pow(cfg->beta1, (double)cnt));
        if (dense) {
          // exact Gaussian gradients (solvers.py:473-478) at the current iterate
          grams_enqueue(ctx, M, nullptr, W.hb.P.as<double>(), W.hb, true);
          const SamplesP Sx = all_nonzeros(ctx, X, 1.0);
          const int nbx = wgrad_enqueue(ctx, Sx, M, s_f, kIdentityLoss, part, code_of(e, 1));
          sum_partials_enqueue(ctx, part, nbx, ldr, bdev);
          if (Sx.shard_world > 1) comm_allreduce_sum(ctx, bdev, (size_t)ldr);
          hist_coeffs_enqueue(ctx, M.ndim, R, W.hb.P.as<double>(), nullptr, nullptr, 0.0, W.hb.Mk.as<float>(),
                              W.hb.Nk.as<float>(), ws, 2.0);
          sgrad_enqueue(ctx, all_nonzeros(ctx, X, -2.0), M, s_f, kIdentityLoss, gp, code_of(e, 1));
          comm_allreduce_sum(ctx, W.grads.as<float>(), gtot);
          dense_wgrad_enqueue(ctx, M.ndim, R, ldr, W.hb.P.as<double>(), bdev, ws, part);
          weight_step_enqueue(ctx, part, 1, R, ldr, ws, s_f, cfg->reg_weights, rate_i, cfg->beta1, cfg->beta2,
                              cfg->adam_eps, cfg->lower_bound, code_of(e, 2));
          const int RR = R * R;
          for (int k = 0; k < M.ndim; ++k)
            factor_update_enqueue(ctx, M.dims[k], R, ldr, A[k], nullptr, gp[k], ad->u[k], ad->v[k],
                                  W.hb.Mk.as<float>() + (size_t)k * RR, W.hb.Nk.as<float>() + (size_t)k * RR,
                                  cfg->reg_factors, rate_i, cfg->beta1, cfg->beta2, cfg->adam_eps, cfg->lower_bound,
                                  code_of(e, 2));
          continue;
        }
        if (it + 1 < iters)
          W.grad.issue(ctx, X, keyed(seed, {seed_key, 7, epoch, it + 1}), budget, code_of(e + 1, 0), (it + 1) & 1);
        SamplesP Sg = sharded(ctx, W.grad.take(ctx, it & 1));
        // both gradients at the current iterate, before either update
        sgrad_enqueue(ctx, Sg, M, s_f, L, gp, code_of(e, 1));
        int nb = wgrad_enqueue(ctx, Sg, M, s_f, L, part, code_of(e, 1));
        comm_allreduce_sum(ctx, W.grads.as<float>(), gtot);
        const double* gparts = part;
        if (ctx->world > 1) {
          sum_partials_enqueue(ctx, part, nb, ldr, gsum);
          comm_allreduce_sum(ctx, gsum, (size_t)ldr);
          gparts = gsum;
          nb = 1;
        }
        weight_step_enqueue(ctx, gparts, nb, R, ldr, ws, s_f, cfg->reg_weights, rate_i, cfg->beta1, cfg->beta2,
                            cfg->adam_eps, cfg->lower_bound, code_of(e, 2));
        for (int k = 0; k < M.ndim; ++k)
          factor_update_enqueue(ctx, M.dims[k], R, ldr, A[k], nullptr, gp[k], ad->u[k], ad->v[k], nullptr, nullptr,
                                cfg->reg_factors, rate_i, cfg->beta1, cfg->beta2, cfg->adam_eps, cfg->lower_bound,
                                code_of(e, 2));
      }
      comm_sync_flags(ctx);
      fetch_flags(ctx);
      OGCP_CUDA(cudaStreamSynchronize(st));
      int r = check_flags(ctx, X, L.kind, budget, what, seed_key);
      if (r == 0) break;
      if (r == 2) W.grad.size(p, q, X->ndim, false, cfg->samples.semi_stratified != 0);
      else ctx->slack *= 4.0;
      adam_epoch(ctx, M, A, ad, false);
      weights_epoch(false);
      ev = ev0;
      if (attempt > 8) throw Error(OGCP_E_INTERNAL, "sampler could not provision enough candidates");
    }
    iter += iters;
    fest = fest_fn();
    if (!std::isfinite(fest)) throw Error(OGCP_E_DIVERGENCE, "static solve diverged");
    if (fest > fold) {
      adam_epoch(ctx, M, A, ad, false);
      weights_epoch(false);
      ad->rate *= cfg->rate_decay;
      fest = fold;
      iter -= iters;
      ++rejections;
    } else {
      adam_epoch(ctx, M, A, ad, true);
      weights_epoch(true);
    }
    ++epochs;
    objv.push_back(fest);
  }
  OGCP_CUDA(cudaMemcpyAsync(hsc, ws, ldr * 8, cudaMemcpyDeviceToHost, st));
  OGCP_CUDA(cudaStreamSynchronize(st));
  for (int r = 0; r < R; ++r) weights[r] = hsc[r];
  if (trace) {
    trace->n_objective = 0;
    for (size_t j = 0; j < objv.size() && (int)j <= max_epochs; ++j)
      trace->objective[trace->n_objective++] = objv[j];
    trace->epochs = epochs;
    trace->rejections = rejections;
  }
}

// G += lambda A + (A Mk - Aold Nk): the K5 kernel on scratch moments with beta1 = 0
// and rate 0, so its first moment u' = g is the assembled gradient.
static void assemble_grads(Ctx* ctx, const ModelP& M, float* const* old_factors, float* const* grads, const float* Mk,
                           const float* Nk, double reg_factors, HistBufs& hb) {
  const int RR = M.rank * M.rank;
  for (int k = 0; k < M.ndim; ++k) {
    const size_t n = (size_t)M.dims[k] * M.ldr;
    hb.tmp.ensure(n * 3 * 4);
    float* u = hb.tmp.as<float>();
    float* v = u + n;
    float* a = v + n;
    OGCP_CUDA(cudaMemsetAsync(u, 0, n * 4, ctx->stream));
    OGCP_CUDA(cudaMemsetAsync(v, 0, n * 4, ctx->stream));
    OGCP_CUDA(cudaMemcpyAsync(a, M.A[k], n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    factor_update_enqueue(ctx, M.dims[k], M.rank, M.ldr, a, old_factors ? old_factors[k] : nullptr, grads[k], u, v,
                          Mk ? Mk + (size_t)k * RR : nullptr, Nk ? Nk + (size_t)k * RR : nullptr, reg_factors, 0.0,
                          0.0, 0.0, 1.0, -INFINITY, code_of(1, 2));
    OGCP_CUDA(cudaMemcpyAsync(grads[k], u, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  }
}

// Per-mode Grams (host [ndim][R][R]) and b = Z' vec(X) (host [R]) at the model.
static void dense_gamma_b(Ctx* ctx, const Slice* X, const ModelP& M, const float* s_f, HistBufs& hb,
                          std::vector<double>& Ph, std::vector<double>& bh) {
  grams_enqueue(ctx, M, nullptr, hb.P.as<double>(), hb, true);
  ctx->dense.ensure((size_t)2 * M.ldr * 8);
  double* bdev = ctx->dense.as<double>();
  double* part = ctx->partials.as<double>();
  const SamplesP Sx = all_nonzeros(ctx, X, 1.0);
  const int nb = wgrad_enqueue(ctx, Sx, M, s_f, kIdentityLoss, part, code_of(1, 1));
  sum_partials_enqueue(ctx, part, nb, M.ldr, bdev);
  if (Sx.shard_world > 1) comm_allreduce_sum(ctx, bdev, (size_t)M.ldr);
  Ph.resize((size_t)M.ndim * M.rank * M.rank);
  bh.resize(M.rank);
  OGCP_CUDA(cudaMemcpyAsync(Ph.data(), hb.P.ptr, Ph.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  OGCP_CUDA(cudaMemcpyAsync(bh.data(), bdev, M.rank * 8, cudaMemcpyDeviceToHost, ctx->stream));
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace ogcp

// ===================================================================== C ABI
using namespace ogcp;

struct ogcp_ctx : Ctx {};
struct ogcp_slice : Slice {};

#define OGCP_API_BEGIN try {
#define OGCP_API_END                                  \
  return OGCP_OK;                                     \
  }                                                   \
  catch (const ogcp::Error& e) {                      \
    g_last_error = e.what();                          \
    return e.code;                                    \
  }                                                   \
  catch (const std::exception& e) {                   \
    g_last_error = e.what();                          \
    return OGCP_E_INTERNAL;                           \
  }

extern "C" {

int ogcp_abi_version(void) { return OGCP_ABI_VERSION; }

const char* ogcp_last_error(void) { return g_last_error.c_str(); }

int32_t ogcp_padded_rank(int32_t rank) {
  int32_t l = 4;
  while (l < rank) l <<= 1;
  return l;
}

int ogcp_rng_state(uint64_t seed, const int64_t* key, int32_t nkey, uint64_t out[4]) {
  OGCP_API_BEGIN
  if (nkey < 0 || nkey > 16) throw Error(OGCP_E_USAGE, "key too long");
  uint64_t k[16];
  for (int i = 0; i < nkey; ++i) {
    if (key[i] < 0) throw Error(OGCP_E_USAGE, "key elements must be >= 0");
    k[i] = (uint64_t)key[i];
  }
  Pcg64 g = seedseq_pcg64(seed, k, nkey);
  out[0] = (uint64_t)(g.state >> 64);
  out[1] = (uint64_t)g.state;
  out[2] = (uint64_t)(g.inc >> 64);
  out[3] = (uint64_t)g.inc;
  OGCP_API_END
}

int ogcp_rng_integers(uint64_t seed, const int64_t* key, int32_t nkey, const int64_t* highs, int32_t nhigh, int64_t n,
                      int64_t* out) {
  OGCP_API_BEGIN
  if (nkey < 0 || nkey > 16 || nhigh < 1) throw Error(OGCP_E_USAGE, "bad key or bounds");
  uint64_t k[16];
  for (int i = 0; i < nkey; ++i) k[i] = (uint64_t)key[i];
  HostStream hs;
  hs.g = seedseq_pcg64(seed, k, nkey);
  hs.has_half = 0;
  hs.half = 0;
  hs.words = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t hi = highs[i % nhigh];
    if (hi < 1 || hi > 0xffffffffLL) throw Error(OGCP_E_USAGE, "bounds must lie in [1, 2^32)");
    out[i] = (int64_t)hs.bounded((uint32_t)hi);
  }
  OGCP_API_END
}

int ogcp_ctx_create(int32_t device, void* cuda_stream, ogcp_ctx** out) {
  OGCP_API_BEGIN
  OGCP_CUDA(cudaSetDevice(device));
  std::unique_ptr<ogcp_ctx> c(new ogcp_ctx());
  c->device = device;
  c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  c->flags.ensure(sizeof(DevFlags));
  OGCP_CUDA(cudaMallocHost((void**)&c->host_scalars, 1024 * 8));
  OGCP_CUDA(cudaMallocHost((void**)&c->host_flags, sizeof(DevFlags)));
  init_jump_table();
  *out = c.release();
  OGCP_API_END
}

int ogcp_ctx_destroy(ogcp_ctx* ctx) {
  OGCP_API_BEGIN
  if (ctx) {
    cudaStreamSynchronize(ctx->stream);
    comm_destroy(ctx);
    if (ctx->host_scalars) cudaFreeHost(ctx->host_scalars);
    if (ctx->host_flags) cudaFreeHost(ctx->host_flags);
    delete ctx;
  }
  OGCP_API_END
}

int ogcp_ctx_set_stream(ogcp_ctx* ctx, void* cuda_stream) {
  OGCP_API_BEGIN
  ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  OGCP_API_END
}

int64_t ogcp_ctx_launches(const ogcp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int ogcp_ctx_profile_enable(ogcp_ctx* ctx, int32_t on) {
  OGCP_API_BEGIN
  ctx->prof.on = on != 0;
  OGCP_API_END
}

int ogcp_ctx_profile_read(ogcp_ctx* ctx, int32_t cls, int64_t* brackets, double* total_ms) {
  OGCP_API_BEGIN
  if (cls < 0 || cls >= kProfClasses) throw Error(OGCP_E_USAGE, "bad profile class");
  ctx->prof.resolve();
  *brackets = ctx->prof.count[cls];
  *total_ms = ctx->prof.total_ms[cls];
  OGCP_API_END
}

int ogcp_ctx_profile_reset(ogcp_ctx* ctx) {
  OGCP_API_BEGIN
  ctx->prof.reset();
  OGCP_API_END
}

int ogcp_gradient_tensor(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev, int64_t p,
                         const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m, const double* weights,
                         const ogcp_loss* loss, int32_t* coords_out, double* vals_out, int64_t* n_out) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  check_model_slice(M, s);
  LossP L = loss_of(loss);
  if (p > 0) x_domain_check(s, L.kind);
  SamplesP S = samples_of(s, ordinals_dev, p, zero_subs_dev, q);
  static thread_local DevBuf wdev;
  wdev.ensure((size_t)M.rank * 8);
  OGCP_CUDA(cudaMemcpyAsync(wdev.ptr, weights, (size_t)M.rank * 8, cudaMemcpyHostToDevice, ctx->stream));
  Strides st;
  for (int k = 0; k < kMaxModes; ++k) st.s[k] = k < s->ndim ? s->strides[k] : 0;
  unsigned int bad = 0;
  *n_out = gradient_tensor_impl(ctx, S, M, wdev.as<double>(), L, st, coords_out, vals_out, &bad);
  if (bad & 1u) throw Error(OGCP_E_DATA, std::string(kind_name(L.kind)) + " loss: non-finite input");
  if (bad & 2u) throw Error(OGCP_E_DATA, std::string(kind_name(L.kind)) + " loss requires m >= 0");
  OGCP_API_END
}

int ogcp_segment_layout(ogcp_ctx* ctx, const int32_t* coords_dev, int64_t n, int32_t ndim, int32_t mode, int64_t dim,
                        int32_t* perm_out, int64_t* offsets_out) {
  OGCP_API_BEGIN
  if (mode < 0 || mode >= ndim) throw Error(OGCP_E_USAGE, "mode out of range");
  segment_layout_impl(ctx, coords_dev, n, ndim, mode, dim, perm_out, offsets_out);
  OGCP_API_END
}

int ogcp_nccl_unique_id(uint8_t out[128]) {
  OGCP_API_BEGIN
  comm_unique_id(out);
  OGCP_API_END
}

int ogcp_ctx_init_comm(ogcp_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t world) {
  OGCP_API_BEGIN
  comm_init(ctx, id, rank, world);
  OGCP_API_END
}

int ogcp_ctx_set_option(ogcp_ctx* ctx, int32_t option, int64_t value) {
  OGCP_API_BEGIN
  if (option == OGCP_OPT_MERGE_DRAWS) ctx->merge_draws = value != 0;
  else if (option == OGCP_OPT_SPLIT_SCATTER) ctx->split_scatter = value != 0;
  else if (option == OGCP_OPT_SORT_ZEROS) ctx->sort_zeros = (int)std::min<int64_t>(std::max<int64_t>(value, 0), 2);
  else if (option == OGCP_OPT_BATCH_DRAWS) ctx->batch_draws = value != 0;
  else if (option == OGCP_OPT_UMMA_GRAM) ctx->umma_gram = value != 0;
  else if (option == OGCP_OPT_DETERMINISTIC) ctx->deterministic = value != 0;
  else if (option == OGCP_OPT_LEAN_WALKS) ctx->lean_walks = value != 0;
  else if (option == OGCP_OPT_SHARD_DRAWS) ctx->shard_draws = value != 0;
  else if (option == OGCP_OPT_TMA_WALKS) {
    ctx->tma_walks = (value & 1) != 0;
    ctx->tma_wgrad = (value & 2) != 0;
    ctx->tma_a2_resident = (value & 4) != 0;
  }
  else if (option == OGCP_OPT_SHARD_SIM) {
    if (ctx->comm) throw Error(OGCP_E_USAGE, "shard simulation needs a context without a communicator");
    const int r = (int)(value & 0xffff), w = (int)((value >> 16) & 0xffff);
    ctx->shard_sim_timing = ((value >> 32) & 1) != 0;
    if (w < 1 || r >= w) {
      ctx->rank = 0;
      ctx->world = 1;
      ctx->shard_sim = false;
      ctx->shard_sim_timing = false;
    } else {
      ctx->rank = r;
      ctx->world = w;
      ctx->shard_sim = w > 1;
    }
  } else if (option == OGCP_OPT_BUCKETS) {
    ctx->buckets = value != 0;
    ctx->buckets_force = value > 1 ? (int)std::min<int64_t>(value, 256) : 0;
  }
  else throw Error(OGCP_E_USAGE, "unknown option");
  OGCP_API_END
}

int ogcp_slice_create(ogcp_ctx* ctx, int32_t ndim, const int64_t* dims, int64_t nnz, const int64_t* subs0_dev,
                      const double* vals_dev, int32_t allow_zero, ogcp_slice** out) {
  OGCP_API_BEGIN
  Slice* s = slice_create_impl<int64_t, double>(ctx, ndim, dims, nnz, subs0_dev, vals_dev, allow_zero);
  *out = static_cast<ogcp_slice*>(s);
  OGCP_API_END
}

int ogcp_slice_create_i32(ogcp_ctx* ctx, int32_t ndim, const int64_t* dims, int64_t nnz, const int32_t* subs0_dev,
                          const float* vals_dev, int32_t allow_zero, ogcp_slice** out) {
  OGCP_API_BEGIN
  Slice* s = slice_create_impl<int32_t, float>(ctx, ndim, dims, nnz, subs0_dev, vals_dev, allow_zero);
  *out = static_cast<ogcp_slice*>(s);
  OGCP_API_END
}

int ogcp_slice_destroy(ogcp_slice* s) {
  OGCP_API_BEGIN
  delete static_cast<Slice*>(s);
  OGCP_API_END
}

int ogcp_slice_info(const ogcp_slice* s, int64_t* nnz, int64_t* omega, double* frob) {
  OGCP_API_BEGIN
  if (nnz) *nnz = s->nnz;
  if (omega) *omega = s->omega;
  if (frob) *frob = s->frob_sq;
  OGCP_API_END
}

int ogcp_slice_contains(ogcp_ctx* ctx, const ogcp_slice* s, const int64_t* subs0_dev, int64_t n, uint8_t* hit_dev) {
  OGCP_API_BEGIN
  slice_contains_impl(ctx, s, subs0_dev, n, hit_dev);
  OGCP_API_END
}

int ogcp_draw_samples(ogcp_ctx* ctx, const ogcp_slice* s, uint64_t seed, const int64_t* key, int32_t nkey, int64_t p,
                      int64_t q, int64_t max_rejects, int32_t* ordinals_dev, int32_t* zero_subs_dev) {
  return ogcp_draw_samples_ex(ctx, s, seed, key, nkey, p, q, max_rejects, 0, ordinals_dev, zero_subs_dev);
}

int ogcp_draw_samples_ex(ogcp_ctx* ctx, const ogcp_slice* s, uint64_t seed, const int64_t* key, int32_t nkey,
                         int64_t p, int64_t q, int64_t max_rejects, int32_t flags, int32_t* ordinals_dev,
                         int32_t* zero_subs_dev) {
  OGCP_API_BEGIN
  if (p < 0 || q < 0) throw Error(OGCP_E_USAGE, "counts must be >= 0");
  const bool semi = (flags & 1) != 0;
  uint64_t k[16];
  if (nkey < 0 || nkey > 16) throw Error(OGCP_E_USAGE, "key too long");
  for (int i = 0; i < nkey; ++i) k[i] = (uint64_t)key[i];
  Pcg64 g = seedseq_pcg64(seed, k, nkey);
  precheck_draw(s, p, semi ? 0 : q);
  const int64_t budget = budget_of(q, max_rejects);
  static thread_local DrawScratch scr;
  SlackScope slack_scope(ctx);  // a shortfall raises the slack for this retry only
  for (int attempt = 0;; ++attempt) {
    reset_flags(ctx);
    const int32_t* z =
        draw_enqueue(ctx, s, g, p, q, budget, ordinals_dev, zero_subs_dev, 0, scr, nullptr, false, semi).zsub;
    if (q > 0 && z != zero_subs_dev)
      OGCP_CUDA(cudaMemcpyAsync(zero_subs_dev, z, (size_t)q * s->ndim * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    fetch_flags(ctx);
    OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
    if (check_flags(ctx, s, OGCP_GAUSSIAN, budget, "draw", 0) == 0) break;
    ctx->slack *= 4.0;
    if (attempt > 8) throw Error(OGCP_E_INTERNAL, "sampler could not provision enough candidates");
  }
  OGCP_API_END
}

int ogcp_sampled_gradient(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev, int64_t p,
                          const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m, const double* weights,
                          const ogcp_loss* loss, float* const* grads_dev, double* gw_dev) {
  return ogcp_sampled_gradient_ex(ctx, s, ordinals_dev, p, zero_subs_dev, q, m, weights, loss, 0, grads_dev, gw_dev);
}

int ogcp_sampled_gradient_ex(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev, int64_t p,
                             const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m, const double* weights,
                             const ogcp_loss* loss, int32_t flags, float* const* grads_dev, double* gw_dev) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  check_model_slice(M, s);
  LossP L = loss_of(loss);
  if (p > 0) x_domain_check(s, L.kind);
  ctx->wsolve.ensure((size_t)M.ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * M.ldr);
  upload_weights(ctx, weights, M.rank, M.ldr, s_f);
  SamplesP S = semi_of(s, samples_of(s, ordinals_dev, p, zero_subs_dev, q), (flags & 1) != 0);
  reset_flags(ctx);
  if (grads_dev) sgrad_enqueue(ctx, S, M, s_f, L, grads_dev, code_of(1, 1));
  if (gw_dev) {
    ctx->partials.ensure((size_t)kNumSMs * 8 * M.ldr * 8 + 64);
    ctx->scalars.ensure(64 * 8 + M.ldr * 8);
    int nb = wgrad_enqueue(ctx, S, M, s_f, L, ctx->partials.as<double>(), code_of(1, 1));
    sum_partials_enqueue(ctx, ctx->partials.as<double>(), nb, M.ldr, ctx->scalars.as<double>() + 64);
    OGCP_CUDA(cudaMemcpyAsync(gw_dev, ctx->scalars.as<double>() + 64, M.rank * 8, cudaMemcpyDeviceToDevice,
                              ctx->stream));
  }
  fetch_flags(ctx);
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  check_flags(ctx, s, L.kind, 0, "gradient", 0);
  OGCP_API_END
}

int ogcp_factor_gradients(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev, int64_t p,
                          const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m, float* const* old_factors,
                          const double* weights, const ogcp_loss* loss, const double* window_s,
                          const int64_t* window_ids, int32_t H, double hist_weight, double hist_decay, int64_t t,
                          double reg_factors, float* const* grads_dev) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  check_model_slice(M, s);
  LossP L = loss_of(loss);
  if (p > 0) x_domain_check(s, L.kind);
  ctx->wsolve.ensure((size_t)M.ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * M.ldr);
  upload_weights(ctx, weights, M.rank, M.ldr, s_f);
  SamplesP S = samples_of(s, ordinals_dev, p, zero_subs_dev, q);
  FactorWork& W = factor_work();
  hist_alloc(W.hb, M.ndim, M.rank);
  const bool hist = hist_weight != 0.0 && H > 0;
  if (hist && !old_factors) throw Error(OGCP_E_DATA, "history terms require the previous-step factors");
  reset_flags(ctx);
  sgrad_enqueue(ctx, S, M, s_f, L, grads_dev, code_of(1, 1));
  window_upload(ctx, W.hb, M.rank, window_s, window_ids, H, hist_decay, t);
  const int RR = M.rank * M.rank;
  if (hist) {
    k_window_matrix<<<1, 256, 0, ctx->stream>>>(M.rank, H, W.hb.Ws.as<double>(), W.hb.coef.as<double>(),
                                                W.hb.S.as<double>());
    ctx->count();
    grams_pc_enqueue(ctx, M, old_factors, W.hb);
    hist_coeffs_enqueue(ctx, M.ndim, M.rank, W.hb.P.as<double>(), W.hb.C.as<double>(), W.hb.S.as<double>(),
                        hist_weight, W.hb.Mk.as<float>(), W.hb.Nk.as<float>());
  }
  assemble_grads(ctx, M, hist ? old_factors : nullptr, grads_dev, hist ? W.hb.Mk.as<float>() : nullptr,
                 hist ? W.hb.Nk.as<float>() : nullptr, reg_factors, W.hb);
  fetch_flags(ctx);
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  check_flags(ctx, s, L.kind, 0, "gradient", t);
  OGCP_API_END
}

int ogcp_dense_gaussian_gradients(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m,
                                  float* const* old_factors, const double* weights, const double* window_s,
                                  const int64_t* window_ids, int32_t H, double hist_weight, double hist_decay,
                                  int64_t t, double reg_factors, double reg_weights, float* const* grads_dev,
                                  double* weight_grad) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  check_model_slice(M, s);
  const int R = M.rank, ldr = M.ldr;
  ctx->wsolve.ensure((size_t)ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * ldr);
  upload_weights(ctx, weights, R, ldr, s_f);
  const double* s_dev = dense_upload_s(ctx, weights, R, ldr);
  ctx->partials.ensure((size_t)kNumSMs * 8 * ldr * 8 + 64);
  FactorWork& W = factor_work();
  hist_alloc(W.hb, M.ndim, R);
  const bool hist = hist_weight != 0.0 && H > 0;
  if (hist && !old_factors) throw Error(OGCP_E_DATA, "history terms require the previous-step factors");
  reset_flags(ctx);
  if (grads_dev) {
    sgrad_enqueue(ctx, all_nonzeros(ctx, s, -2.0), M, s_f, kIdentityLoss, grads_dev, code_of(1, 1));
    window_upload(ctx, W.hb, R, window_s, window_ids, H, hist_decay, t);
    if (hist) {
      k_window_matrix<<<1, 256, 0, ctx->stream>>>(R, H, W.hb.Ws.as<double>(), W.hb.coef.as<double>(),
                                                  W.hb.S.as<double>());
      ctx->count();
      grams_pc_enqueue(ctx, M, old_factors, W.hb);
    } else {
      grams_enqueue(ctx, M, nullptr, W.hb.P.as<double>(), W.hb, true);
    }
    hist_coeffs_enqueue(ctx, M.ndim, R, W.hb.P.as<double>(), hist ? W.hb.C.as<double>() : nullptr,
                        hist ? W.hb.S.as<double>() : nullptr, hist_weight, W.hb.Mk.as<float>(), W.hb.Nk.as<float>(),
                        s_dev, 2.0);
    assemble_grads(ctx, M, hist ? old_factors : nullptr, grads_dev, W.hb.Mk.as<float>(), W.hb.Nk.as<float>(),
                   reg_factors, W.hb);
  }
  if (weight_grad) {
    std::vector<double> Ph, bh;
    dense_gamma_b(ctx, s, M, s_f, W.hb, Ph, bh);
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      for (int j = 0; j < R; ++j) {
        double g = 1.0;
        for (int k = 0; k < M.ndim; ++k) g *= Ph[(size_t)k * R * R + (size_t)r * R + j];
        acc += g * weights[j];
      }
      weight_grad[r] = 2.0 * (acc - bh[r]) + reg_weights * weights[r];
    }
  }
  fetch_flags(ctx);
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  check_flags(ctx, s, OGCP_GAUSSIAN, 0, "gradient", t);
  OGCP_API_END
}

int ogcp_gaussian_residual(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m, const double* weights,
                           double* out) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  check_model_slice(M, s);
  ctx->wsolve.ensure((size_t)M.ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * M.ldr);
  upload_weights(ctx, weights, M.rank, M.ldr, s_f);
  ctx->partials.ensure((size_t)kNumSMs * 8 * M.ldr * 8 + 64);
  ctx->scalars.ensure(64 * 8);
  FactorWork& W = factor_work();
  hist_alloc(W.hb, M.ndim, M.rank);
  ogcp_solver_config cfg{};
  *out = factor_objective(ctx, s, SamplesP{}, M, s_f, kIdentityLoss, nullptr, 0, &cfg, W.hb, code_of(1, 1), 0, 0,
                          "gaussian residual", weights);
  OGCP_API_END
}

int ogcp_solve_weights_ls(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m, double reg_weights,
                          double* s_out) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  check_model_slice(M, s);
  const int R = M.rank;
  ctx->wsolve.ensure((size_t)M.ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * M.ldr);
  std::vector<double> zeros(R, 0.0);
  upload_weights(ctx, zeros.data(), R, M.ldr, s_f);
  ctx->partials.ensure((size_t)kNumSMs * 8 * M.ldr * 8 + 64);
  FactorWork& W = factor_work();
  hist_alloc(W.hb, M.ndim, R);
  reset_flags(ctx);
  std::vector<double> Ph, bh;
  dense_gamma_b(ctx, s, M, s_f, W.hb, Ph, bh);
  // (hadamard_k Gram_k + mu I) s = b by LU with partial pivoting (LAPACK gesv);
  // an exactly zero pivot is the singular system numpy.linalg.solve rejects.
  std::vector<double> a((size_t)R * R);
  for (int i = 0; i < R; ++i)
    for (int j = 0; j < R; ++j) {
      double g = 1.0;
      for (int k = 0; k < M.ndim; ++k) g *= Ph[(size_t)k * R * R + (size_t)i * R + j];
      a[(size_t)i * R + j] = g + (i == j ? reg_weights : 0.0);
    }
  std::vector<double> x = bh;
  for (int c = 0; c < R; ++c) {
    int piv = c;
    for (int r = c + 1; r < R; ++r)
      if (std::fabs(a[(size_t)r * R + c]) > std::fabs(a[(size_t)piv * R + c])) piv = r;
    if (a[(size_t)piv * R + c] == 0.0)
      throw Error(OGCP_E_DATA,
                  "temporal least-squares system is singular; set a positive weight regularization (mu)");
    if (piv != c) {
      for (int j = 0; j < R; ++j) std::swap(a[(size_t)c * R + j], a[(size_t)piv * R + j]);
      std::swap(x[c], x[piv]);
    }
    for (int r = c + 1; r < R; ++r) {
      const double f = a[(size_t)r * R + c] / a[(size_t)c * R + c];
      if (f == 0.0) continue;
      for (int j = c; j < R; ++j) a[(size_t)r * R + j] -= f * a[(size_t)c * R + j];
      x[r] -= f * x[c];
    }
  }
  for (int r = R - 1; r >= 0; --r) {
    double acc = x[r];
    for (int j = r + 1; j < R; ++j) acc -= a[(size_t)r * R + j] * x[j];
    x[r] = acc / a[(size_t)r * R + r];
  }
  for (int r = 0; r < R; ++r) s_out[r] = x[r];
  OGCP_API_END
}

int ogcp_estimate_objective(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev, int64_t p,
                            const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m, float* const* old_factors,
                            const double* weights, const ogcp_loss* loss, const double* window_s,
                            const int64_t* window_ids, int32_t H, double hist_weight, double hist_decay, int64_t t,
                            double reg_factors, double reg_weights, double* out) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  check_model_slice(M, s);
  LossP L = loss_of(loss);
  if (p > 0) x_domain_check(s, L.kind);
  ctx->wsolve.ensure((size_t)M.ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * M.ldr);
  upload_weights(ctx, weights, M.rank, M.ldr, s_f);
  ctx->partials.ensure((size_t)kNumSMs * 8 * M.ldr * 8 + 64);
  ctx->scalars.ensure(64 * 8);
  SamplesP S = samples_of(s, ordinals_dev, p, zero_subs_dev, q);
  FactorWork& W = factor_work();
  hist_alloc(W.hb, M.ndim, M.rank);
  const bool hist = hist_weight != 0.0 && H > 0;
  if (hist && !old_factors) throw Error(OGCP_E_DATA, "history terms require the previous-step factors");
  window_upload(ctx, W.hb, M.rank, window_s, window_ids, H, hist_decay, t);
  if (hist)
    for (int k = 0; k < M.ndim; ++k)
      gram_enqueue(ctx, old_factors[k], old_factors[k], M.dims[k], M.rank, M.ldr,
                   W.hb.Poo.as<double>() + (size_t)k * M.rank * M.rank, W.hb.scratch);
  ogcp_solver_config cfg{};
  cfg.hist_weight = hist_weight;
  cfg.hist_decay = hist_decay;
  cfg.reg_factors = reg_factors;
  double v = factor_objective(ctx, s, S, M, s_f, L, old_factors, hist ? H : 0, &cfg, W.hb, code_of(1, 1), 0, t);
  if (reg_weights) {
    double ss = 0.0;
    for (int r = 0; r < M.rank; ++r) ss += weights[r] * weights[r];
    v += 0.5 * reg_weights * ss;
  }
  *out = v;
  OGCP_API_END
}

int ogcp_gram(ogcp_ctx* ctx, const ogcp_model* m, float* const* other, int32_t skip, double* out) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  const int RR = M.rank * M.rank;
  FactorWork& W = factor_work();
  hist_alloc(W.hb, M.ndim, M.rank);
  grams_enqueue(ctx, M, other, W.hb.P.as<double>(), W.hb, other == nullptr);
  std::vector<double> h((size_t)M.ndim * RR);
  OGCP_CUDA(cudaMemcpyAsync(h.data(), W.hb.P.ptr, h.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  bool any = false;
  for (int e = 0; e < RR; ++e) out[e] = 1.0;
  for (int k = 0; k < M.ndim; ++k) {
    if (k == skip) continue;
    any = true;
    for (int e = 0; e < RR; ++e) out[e] *= h[(size_t)k * RR + e];
  }
  if (!any) throw Error(OGCP_E_DATA, "gram over zero modes is undefined");
  OGCP_API_END
}

int ogcp_adam_step(ogcp_ctx* ctx, const ogcp_model* m, float* const* grads, ogcp_adam_state* st, double beta1,
                   double beta2, double eps, double lower_bound, int64_t step_count) {
  OGCP_API_BEGIN
  if (step_count < 1) throw Error(OGCP_E_DATA, "step_count is 1-based and must be >= 1");
  ModelP M = model_of(m);
  const double rate_i =
      st->rate * std::sqrt(1.0 - std::pow(beta2, (double)step_count)) / (1.0 - std::pow(beta1, (double)step_count));
  reset_flags(ctx);
  for (int k = 0; k < M.ndim; ++k)
    factor_update_enqueue(ctx, M.dims[k], M.rank, M.ldr, m->factors[k], nullptr, grads[k], st->u[k], st->v[k],
                          nullptr, nullptr, 0.0, rate_i, beta1, beta2, eps, lower_bound, code_of(1, 2));
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  OGCP_API_END
}

int ogcp_adam_update(ogcp_ctx* ctx, const ogcp_model* m, ogcp_adam_state* st, int32_t passed, double rate_decay) {
  OGCP_API_BEGIN
  ModelP M = model_of(m);
  adam_epoch(ctx, M, m->factors, st, passed != 0);
  if (!passed) st->rate *= rate_decay;
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  OGCP_API_END
}

int ogcp_solve_weights(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_solver_config* cfg, const ogcp_loss* loss,
                       int64_t t, const ogcp_model* m, const double* s_init, double* s_out, ogcp_trace* trace) {
  OGCP_API_BEGIN
  DbgTimer dt("solve_weights");
  solve_weights_impl(ctx, s, cfg, loss, t, m, s_init, s_out, trace);
  OGCP_API_END
}

int ogcp_solve_factors(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_solver_config* cfg, const ogcp_loss* loss,
                       int64_t t, const ogcp_model* m, float* const* old_factors, const double* weights,
                       const double* window_s, const int64_t* window_ids, int32_t H, ogcp_adam_state* adam,
                       int64_t* iteration, ogcp_trace* trace) {
  OGCP_API_BEGIN
  DbgTimer dt("solve_factors");
  solve_factors_impl(ctx, s, cfg, loss, t, m, old_factors, weights, window_s, window_ids, H, adam, iteration, trace);
  OGCP_API_END
}

int ogcp_solve_static(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_solver_config* cfg, const ogcp_loss* loss,
                      int64_t seed_key, const ogcp_model* m, double* weights, ogcp_adam_state* adam,
                      int32_t max_epochs, int32_t iters, double tol, ogcp_trace* trace) {
  OGCP_API_BEGIN
  if (max_epochs < 0 || iters < 1) throw Error(OGCP_E_USAGE, "epoch and iteration counts must be >= 1");
  solve_static_impl(ctx, s, cfg, loss, seed_key, m, weights, adam, max_epochs, iters, tol, trace);
  OGCP_API_END
}

int ogcp_comm_selftest(ogcp_ctx* ctx, int32_t* mismatches) {
  OGCP_API_BEGIN
  *mismatches = comm_selftest(ctx);
  OGCP_API_END
}

int ogcp_debug_solve_draw(ogcp_ctx* ctx, const ogcp_slice* s, uint64_t seed, const int64_t* key, int32_t nkey,
                          int64_t p, int64_t q, int64_t max_rejects, int32_t ldr, int64_t cap_nz, int32_t* ord_out,
                          uint8_t* cnt_out, int64_t* n_nz, int64_t cap_zero, int32_t* zero_out, int64_t* n_zero) {
  OGCP_API_BEGIN
  const Slice* X = s;
  if (p < 0) p = X->nnz;
  if (X->nnz == 0) p = 0;
  static thread_local SampleBufs b;
  precheck_draw(X, p, q);
  b.size(p, q, X->ndim, p > 0 && use_merged(ctx, X, p));
  b.semi = false;
  if (b.merged) prepare_buckets(ctx, X, ldr);
  const int64_t budget = budget_of(q, max_rejects);
  if (nkey > 8) throw Error(OGCP_E_USAGE, "at most 8 key words");
  uint64_t k[8];
  for (int i = 0; i < nkey; ++i) k[i] = (uint64_t)key[i];
  reset_flags(ctx);
  const SamplesP S = sharded(ctx, b.draw(ctx, X, seedseq_pcg64(seed, k, nkey), budget, code_of(1, 0)));
  fetch_flags(ctx);
  OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (check_flags(ctx, X, OGCP_GAUSSIAN, budget, "draw", 0) != 0)
    throw Error(OGCP_E_INTERNAL, "draw shortfall or counter overflow (retry with more slack)");
  // the samples this rank's SampleStream walks (compute.cu SampleStream::init)
  int64_t pn = S.p;
  if (S.p_dev) OGCP_CUDA(cudaMemcpy(&pn, S.p_dev, 8, cudaMemcpyDeviceToHost));
  int64_t zrows = S.q;
  if (S.q_dev) OGCP_CUDA(cudaMemcpy(&zrows, S.q_dev, 8, cudaMemcpyDeviceToHost));
  const int64_t total = pn + zrows;
  int64_t nlo = 0, nhi = pn, zlo = 0, zhi = zrows;
  if (S.shard_world > 1 && S.zshard == 2) {
    // rank-local zero rows (word-sharded draw): all of them
  } else if (S.shard_world > 1 && S.zshard) {
    zlo = zrows * S.shard_rank / S.shard_world;
    zhi = zrows * (S.shard_rank + 1) / S.shard_world;
  } else if (S.shard_world > 1) {
    const int64_t lo = total * S.shard_rank / S.shard_world, hi = total * (S.shard_rank + 1) / S.shard_world;
    nlo = std::min(lo, pn);
    nhi = std::min(hi, pn);
    zlo = std::max<int64_t>(lo - pn, 0);
    zhi = std::max<int64_t>(hi - pn, 0);
  }
  std::vector<int32_t> ord(std::max<int64_t>(nhi - nlo, 0));
  std::vector<uint8_t> cnt(ord.size(), 1);
  if (!ord.empty()) {
    OGCP_CUDA(cudaMemcpy(ord.data(), S.ord + nlo, ord.size() * 4, cudaMemcpyDeviceToHost));
    if (S.cnt) OGCP_CUDA(cudaMemcpy(cnt.data(), S.cnt + nlo, ord.size(), cudaMemcpyDeviceToHost));
  }
  if (b.merged && b.md.perm) {  // positions of the bucketed copy -> ordinals
    std::vector<int32_t> perm(X->bucket_ohi - X->bucket_olo);
    OGCP_CUDA(cudaMemcpy(perm.data(), b.md.perm, perm.size() * 4, cudaMemcpyDeviceToHost));
    for (auto& o : ord) o = perm[o];
  }
  if ((int64_t)ord.size() > cap_nz) throw Error(OGCP_E_USAGE, "nonzero output capacity too small");
  std::copy(ord.begin(), ord.end(), ord_out);
  std::copy(cnt.begin(), cnt.end(), cnt_out);
  *n_nz = (int64_t)ord.size();
  const int d = X->ndim;
  std::vector<int32_t> z((size_t)std::max<int64_t>(zhi - zlo, 0) * d);
  if (!z.empty()) OGCP_CUDA(cudaMemcpy(z.data(), S.zsub + zlo * d, z.size() * 4, cudaMemcpyDeviceToHost));
  int64_t nz = 0;
  for (int64_t r = 0; r < zhi - zlo; ++r) {
    if (z[r * d] < 0) continue;  // rejected candidate of the lazy layout
    if (nz >= cap_zero) throw Error(OGCP_E_USAGE, "zero output capacity too small");
    std::copy(z.begin() + r * d, z.begin() + (r + 1) * d, zero_out + nz * d);
    ++nz;
  }
  *n_zero = nz;
  OGCP_API_END
}

int ogcp_local_loss(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m, const double* weights,
                    const ogcp_loss* loss, int32_t mode, int64_t p, int64_t q, uint64_t seed, const int64_t* key,
                    int32_t nkey, int64_t max_rejects, int64_t max_elements, double* out, int32_t* normalized) {
  OGCP_API_BEGIN
  DbgTimer dt("local_loss");
  ModelP M = model_of(m);
  if (M.ndim != s->ndim) throw Error(OGCP_E_DATA, "dims differ");
  for (int k = 0; k < M.ndim; ++k)
    if (M.dims[k] != s->dims[k]) throw Error(OGCP_E_DATA, "dims differ");
  LossP L = loss_of(loss);
  ctx->wsolve.ensure((size_t)M.ldr * (6 * 8 + 4));
  float* s_f = reinterpret_cast<float*>(ctx->wsolve.as<double>() + 6 * M.ldr);
  upload_weights(ctx, weights, M.rank, M.ldr, s_f);
  ctx->partials.ensure((size_t)kNumSMs * 8 * M.ldr * 8 + 64);
  ctx->scalars.ensure(64 * 8);
  double* part = ctx->partials.as<double>();
  double* dsc = ctx->scalars.as<double>();
  double total = 0.0;
  if (mode == 0) {
    if (!s->omega_fits || s->omega > max_elements)
      throw Error(OGCP_E_DATA, "exact local loss over " + std::to_string(s->omega) + " cells exceeds cap " +
                                   std::to_string(max_elements) + "; use sampled mode");
    if (s->nnz > 0) x_domain_check(s, L.kind);
    reset_flags(ctx);
    int nb = exact_cells_enqueue(ctx, M, s_f, L, s->omega, part, code_of(1, 1));
    sum_partials_enqueue(ctx, part, nb, 1, dsc);
    SamplesP S = samples_of(s, nullptr, 0, nullptr, 0);
    if (s->nnz > 0) {
      S = samples_of(s, iota_of(ctx, s->nnz), s->nnz, nullptr, 0);  // every stored entry once
      int nb2 = exact_nz_enqueue(ctx, S, M, s_f, L, part + nb, code_of(1, 1));
      sum_partials_enqueue(ctx, part + nb, nb2, 1, dsc + 1);
    } else {
      OGCP_CUDA(cudaMemsetAsync(dsc + 1, 0, 8, ctx->stream));
    }
    OGCP_CUDA(cudaMemcpyAsync(ctx->host_scalars, dsc, 16, cudaMemcpyDeviceToHost, ctx->stream));
    fetch_flags(ctx);
    OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
    check_flags(ctx, s, L.kind, 0, "local loss", 0);
    total = ctx->host_scalars[0] + ctx->host_scalars[1];
  } else {
    int64_t pp, qq;
    resolve_counts(p, q, s, &pp, &qq);
    if (pp > 0) x_domain_check(s, L.kind);
    uint64_t k[16];
    for (int i = 0; i < nkey; ++i) k[i] = (uint64_t)key[i];
    static thread_local SampleBufs b;
    draw_sync(ctx, s, seedseq_pcg64(seed, k, nkey), pp, qq, max_rejects, b);
    SamplesP S = b.sample_set(s);
    reset_flags(ctx);
    int nb = objective_enqueue(ctx, S, M, s_f, L, part, code_of(1, 1));
    sum_partials_enqueue(ctx, part, nb, 1, dsc);
    OGCP_CUDA(cudaMemcpyAsync(ctx->host_scalars, dsc, 8, cudaMemcpyDeviceToHost, ctx->stream));
    fetch_flags(ctx);
    OGCP_CUDA(cudaStreamSynchronize(ctx->stream));
    check_flags(ctx, s, L.kind, 0, "local loss", 0);
    total = ctx->host_scalars[0];
  }
  if (s->frob_sq > 0) {
    *out = total / s->frob_sq;
    *normalized = 1;
  } else {
    *out = total;
    *normalized = 0;
  }
  OGCP_API_END
}

}  // extern "C"
