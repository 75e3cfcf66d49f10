/*
 * ogcp_b200 -- B200-native (sm_100a) engine for the OnlineGCP per-slice solve.
 *
 * C ABI: plain pointers and sizes, no torch types.  Device pointers are raw
 * CUDA device addresses owned by the caller unless stated otherwise; the
 * context owns only scratch.  Every call is enqueued on the context's CUDA
 * stream; calls that return scalars or status synchronize that stream.
 *
 * The reference (pkg/src/ogcp, pure Python/numpy) has no FFI: these entry
 * points replace its Python functions one for one, and the Python package
 * paper_2110_14514_b200 re-exports the reference names on top of them (see
 * INTEGRATION.md for the ctypes binding).  Each declaration cites the
 * reference interface it replaces.
 *
 * Status codes mirror the reference exception hierarchy (exceptions.py:7-20,
 * CLI exit codes cli.py:420-425): DataError=3, DivergenceError=4,
 * SamplingError=5 (a DataError subclass in Python).
 */
#ifndef OGCP_B200_H
#define OGCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OGCP_ABI_VERSION 2

enum {
  OGCP_OK = 0,
  OGCP_E_INTERNAL = 1,
  OGCP_E_USAGE = 2,
  OGCP_E_DATA = 3,        /* exceptions.py:11 DataError */
  OGCP_E_DIVERGENCE = 4,  /* exceptions.py:19 DivergenceError */
  OGCP_E_SAMPLING = 5,    /* exceptions.py:15 SamplingError (subclass of DataError) */
  OGCP_E_CUDA = 6
};

/* losses.py:24 KINDS */
enum { OGCP_GAUSSIAN = 0, OGCP_POISSON = 1, OGCP_BERNOULLI = 2,
       /* gradient-tensor mode: y = x (apply MTTKRP to a given sparse tensor Y,
        * kernels.py:33-72); no model evaluation, no domain checks */
       OGCP_IDENTITY = 3 };

typedef struct ogcp_ctx ogcp_ctx;      /* one per (stream, device); owns scratch, not thread-safe */
typedef struct ogcp_slice ogcp_slice;  /* a device-resident validated COO slice + membership hash */

/* losses.py:27-38 LossFunction(kind, eps) */
typedef struct {
  int32_t kind;
  double eps;
} ogcp_loss;

/* sampling.py:45-54 SamplerConfig; a count < 0 means None ("all" nonzeros);
 * max_rejects < 0 means None (1000*q at draw time). */
typedef struct {
  int64_t grad_nonzeros;
  int64_t grad_zeros;
  int64_t obj_nonzeros;
  int64_t obj_zeros;
  uint64_t seed;
  int64_t max_rejects;
  /* Extension (not in the reference; BASELINE configs[2]):
   * semi-stratified estimator -- nonzero stratum (eta/p)(g(x,m) - g(0,m)),
   * uniform stratum (omega/q) g(0,m) over the whole box, no rejection. */
  int32_t semi_stratified;
} ogcp_sampler_config;

/* solvers.py:40-69 SolverConfig;
 * lower_bound is already resolved against the loss (solvers.py:86-87). */
typedef struct {
  double tol_weights, tol_factors;
  int32_t max_epochs_weights, max_epochs_factors;
  int32_t iters_weights, iters_factors;
  double reg_factors, reg_weights, hist_weight, hist_decay;
  int32_t warm_start_weights;
  double rate_weights, rate_factors, beta1, beta2, adam_eps, rate_decay;
  double lower_bound;
  ogcp_sampler_config samples;
  int32_t gradient_mode;    /* 0 "sampled", 1 "dense-gaussian" (solvers.py:35, 145-185) */
  int32_t temporal_solver;  /* 0 "sgd", 1 "least-squares" (solvers.py:34, 271-288; streaming.py:168-176) */
} ogcp_solver_config;

/* A CP model bound to caller-owned device buffers.  factors[k] is a row-major
 * dims[k] x ldr float32 matrix whose first `rank` columns are the factor and
 * whose padding columns are zero (ldr is a multiple of 4, see ogcp_padded_rank). */
typedef struct {
  int32_t ndim;
  int32_t rank;
  int32_t ldr;
  const int64_t* dims;     /* host, [ndim] */
  float* const* factors;   /* host array of ndim device pointers */
} ogcp_model;

/* Persistent factor Adam (adam.py:20-109): device buffers shaped like the
 * factors; rate is read and written back (rejections decay it). */
typedef struct {
  float* const* u;
  float* const* v;
  float* const* u_o;
  float* const* v_o;
  float* const* a_o;
  double rate;
} ogcp_adam_state;

/* solvers.py:94-100 EpochTrace; objective[] must hold max_epochs+1 doubles. */
typedef struct {
  double* objective;
  int32_t n_objective;
  int32_t epochs;
  int32_t rejections;
} ogcp_trace;

/* ------------------------------------------------------------------ misc */
int ogcp_abi_version(void);
/* Message of the last failing call on this thread (empty if none). */
const char* ogcp_last_error(void);
/* Padded row stride the kernels require for a given rank. */
int32_t ogcp_padded_rank(int32_t rank);

/* Keyed generator state, sampling.py:39-42 rng_at(seed, *key): the PCG64 state
 * and increment as {state_hi, state_lo, inc_hi, inc_lo}.  Host only. */
int ogcp_rng_state(uint64_t seed, const int64_t* key, int32_t nkey, uint64_t out[4]);
/* Host restatement of Generator.integers(0, highs[j % nhigh]) for n draws on the
 * keyed stream (sampling.py:125, 138; streaming.py:51).  Host only. */
int ogcp_rng_integers(uint64_t seed, const int64_t* key, int32_t nkey, const int64_t* highs,
                      int32_t nhigh, int64_t n, int64_t* out);

/* --------------------------------------------------------------- context */
int ogcp_ctx_create(int32_t device, void* cuda_stream, ogcp_ctx** out);
int ogcp_ctx_destroy(ogcp_ctx* ctx);
int ogcp_ctx_set_stream(ogcp_ctx* ctx, void* cuda_stream);
/* Number of kernels this context has launched so far. */
int64_t ogcp_ctx_launches(const ogcp_ctx* ctx);
/* CUDA-event timing per kernel class on the context stream (measurement):
 * classes 0 draw (K1), 1 eval+scatter (K2/K3), 2 weight gradient, 3 objective (K6),
 * 4 Gram (K4), 5 fused update (K5 / weight Adam), 6 ingest (K0). */
int ogcp_ctx_profile_enable(ogcp_ctx* ctx, int32_t on);
/* Resolves pending events (synchronizes) and returns the accumulated bracket
 * count and milliseconds of one class. */
int ogcp_ctx_profile_read(ogcp_ctx* ctx, int32_t cls, int64_t* brackets, double* total_ms);
int ogcp_ctx_profile_reset(ogcp_ctx* ctx);
/* Engine options.  OGCP_OPT_MERGE_DRAWS (default 1): in the solves, merge dense
 * nonzero draws (p >= eta/8) into distinct ordinals with multiplicities before
 * evaluation -- the same merge sampled_gradient_tensor performs
 * (sampling.py:233-237); 0 evaluates every draw separately. */
/* OGCP_OPT_SPLIT_SCATTER (default 0): for merged sets, scatter the largest
 * random-access mode in a second pass from stored per-sample values.
 * OGCP_OPT_BUCKETS (default 1): walk merged sets of slices with a large
 * random-access mode in row-bucket order (Slice bucketed copy, built once per
 * slice) so the bucket's factor/gradient rows stay L2-resident; a value k > 1
 * forces k buckets on every merged solve (tests). */
/* OGCP_OPT_SHARD_SIM: value = rank | world << 16 | timing << 32 on a context
 * without a communicator -- the solves then run rank `rank`'s share of a
 * world-`world` multi-GPU solve with the collectives skipped (single-process
 * tests of the shard partition); world 1 (or 0) restores the single-GPU context.
 * timing = 1: a timing simulation -- every collective is replaced by a stand-in
 * kernel holding 24 SMs for its modeled time (15 us + ring bytes at 700 GB/s) and
 * the sharded draws run only this rank's part, its own slots standing in for the
 * other ranks' (results then inexact; for projections only). */
/* OGCP_OPT_SORT_ZEROS (default 0): in a bucketed merged solve, the accepted zero
 * rows of every draw are sorted (stable radix sort) by (row bucket, mode-0 row) so
 * the zero part of the walk meets the same L2-resident bucket rows and streams
 * mode 0 in order like the nonzero part; 0 keeps the draw order (lazy layout). */
enum { OGCP_OPT_MERGE_DRAWS = 1, OGCP_OPT_SPLIT_SCATTER = 2, OGCP_OPT_BUCKETS = 3, OGCP_OPT_SHARD_SIM = 4,
       OGCP_OPT_SORT_ZEROS = 5, OGCP_OPT_LEAN_WALKS = 6, OGCP_OPT_TMA_WALKS = 7,
       OGCP_OPT_BATCH_DRAWS = 8, OGCP_OPT_UMMA_GRAM = 9, OGCP_OPT_DETERMINISTIC = 10,
       OGCP_OPT_SHARD_DRAWS = 11 };
/* OGCP_OPT_SHARD_DRAWS (default 1): in a multi-GPU solve the merged
 * gradient draws of slices whose modes all exceed 1 are sharded by RNG word
 * range -- each rank generates 1/world of the words; tile maps, per-rank zero-row
 * records and the nibble counters (reduce-scattered to the ordinal owners) are
 * exchanged on a second communicator -- so no rank replays the whole stream; 0
 * keeps every rank generating every word.  In an exact shard simulation
 * (OGCP_OPT_SHARD_SIM) every rank's part runs on this GPU in lock step with exact
 * device-side stand-ins for the exchanges. */
/* OGCP_OPT_DETERMINISTIC (default 0): for small models (sum of mode sizes x ldr
 * <= 4096, one GPU) the factor-gradient scatter adds in a fixed order (per-warp
 * shared-memory copies, groups in turn, fixed-order block and grid sums), so a
 * same-seed stream is bitwise reproducible; large models keep the 16-byte vector
 * reductions (run-to-run differences in the last bits). */
/* OGCP_OPT_UMMA_GRAM (default 1): history Grams of large factors with ldr 32 / 64 /
 * 128 on the tcgen05 tensor cores with TMEM accumulators (csrc/gram_umma.cuh;
 * ldr 32 packs both Grams of two row sub-chunks into one MMA); 0 keeps the
 * mma.sync split-TF32 kernel. */
/* OGCP_OPT_BATCH_DRAWS (default 1): small per-draw sample sets (the c1 / c2
 * shapes) -- all tau draws of a solver epoch are made at the epoch's start,
 * one launch per sampler pass with one block per draw, instead of one draw
 * per iteration on the side stream. */
/* OGCP_OPT_TMA_WALKS (default 1): bit 0 -- the K3 walk of merged sample sets of
 * 3-way slices (ldr 16 / 32) runs in warp-specialised kernels whose factor-row
 * gathers are TMA tile::gather4 loads into a 16-stage shared-memory ring
 * (csrc/walk_tma.cuh); bit 1 -- the weight-gradient walk too (off by default:
 * measured slower than the generic kernel at c4); bit 2 -- keep a small
 * (<= 128 KB) mode-2 factor resident in shared memory (off by default: the
 * ring then holds 8 stages instead of 16, measured slower at c4).
 * OGCP_OPT_LEAN_WALKS (default 0; used when TMA walks are off): merged sample sets of 3-way slices
 * are evaluated by the specialised walk kernels (csrc/walk3.cuh, ldr 16 / 32); 0 uses the
 * generic sample kernels. */
int ogcp_ctx_set_option(ogcp_ctx* ctx, int32_t option, int64_t value);

/* Multi-GPU (the reference is single-process): the
 * ranks that share one stream each hold the slice and the model; the solves
 * evaluate each rank's contiguous 1/world of every sample set and sum the
 * factor gradients, the temporal-row gradient and the objective with NCCL
 * (loaded at run time).  Rank 0 creates the id, the caller broadcasts it. */
int ogcp_nccl_unique_id(uint8_t out[128]);
int ogcp_ctx_init_comm(ogcp_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t world);

/* ----------------------------------------------------------------- slice */
/* SparseTensor.from_zero_based (tensor.py:75-119): validates bounds,
 * finiteness, stored zeros (unless allow_zero) and duplicates with the
 * reference's messages, then builds the AoS records and the membership hash.
 * subs0_dev: int64 [nnz x ndim] row-major, vals_dev: float64 [nnz]. */
int ogcp_slice_create(ogcp_ctx* ctx, int32_t ndim, const int64_t* dims, int64_t nnz,
                      const int64_t* subs0_dev, const double* vals_dev, int32_t allow_zero,
                      ogcp_slice** out);
/* Same from int32 coordinates and float32 values (device generators). */
int ogcp_slice_create_i32(ogcp_ctx* ctx, int32_t ndim, const int64_t* dims, int64_t nnz,
                          const int32_t* subs0_dev, const float* vals_dev, int32_t allow_zero,
                          ogcp_slice** out);
int ogcp_slice_destroy(ogcp_slice* s);
/* nnz (eta), num_cells (omega, as double and exact int64 when < 2^63),
 * frobenius_sq (tensor.py:138-141). */
int ogcp_slice_info(const ogcp_slice* s, int64_t* nnz, int64_t* omega, double* frobenius_sq);
/* SparseTensor.contains_linear (tensor.py:163-169) for device coords [n x ndim] int64. */
int ogcp_slice_contains(ogcp_ctx* ctx, const ogcp_slice* s, const int64_t* subs0_dev, int64_t n,
                        uint8_t* hit_dev);

/* --------------------------------------------------------------- sampler */
/* draw_samples (sampling.py:108-153) on rng_at(seed, *key): bit-exact nonzero
 * ordinals [p] and zero coordinates [q x ndim] (int32, device). */
int ogcp_draw_samples(ogcp_ctx* ctx, const ogcp_slice* s, uint64_t seed, const int64_t* key,
                      int32_t nkey, int64_t p, int64_t q, int64_t max_rejects,
                      int32_t* ordinals_dev, int32_t* zero_subs_dev);
/* flags bit 0: semi-stratified draw (q uniform cells, no rejection). */
int ogcp_draw_samples_ex(ogcp_ctx* ctx, const ogcp_slice* s, uint64_t seed, const int64_t* key,
                         int32_t nkey, int64_t p, int64_t q, int64_t max_rejects, int32_t flags,
                         int32_t* ordinals_dev, int32_t* zero_subs_dev);

/* ------------------------------------------------------------- estimators */
/* Data part of factor_gradients (solvers.py:139-140 = sampled_mttkrp(Y,k)*s,
 * kernels.py:33-56) and weight_gradient_mttkrp (kernels.py:59-72) for the
 * sampled gradient tensor Y of sampled_gradient_tensor (sampling.py:209-239),
 * given the replayed sample set.  grads_dev (nullable) receives per-mode
 * dims[k] x ldr float32; gw_dev (nullable) receives rank float64. */
int ogcp_sampled_gradient(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev,
                          int64_t p, const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m,
                          const double* weights, const ogcp_loss* loss, float* const* grads_dev,
                          double* gw_dev);

/* flags bit 0: the sample set is a semi-stratified one (ogcp_draw_samples_ex). */
int ogcp_sampled_gradient_ex(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev,
                             int64_t p, const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m,
                             const double* weights, const ogcp_loss* loss, int32_t flags,
                             float* const* grads_dev, double* gw_dev);

/* sampled_gradient_tensor (sampling.py:209-239) in parity form: the merged Y of
 * a replayed sample set, bit-exact in layout -- unique coordinates in
 * ascending linear order (np.unique), each taken from its first draw, values
 * summed in draw order (np.bincount) in fp64.  coords_out: device int32
 * [(p+q) x ndim], vals_out: device fp64 [p+q]; *n_out = number of entries. */
int ogcp_gradient_tensor(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev, int64_t p,
                         const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m, const double* weights,
                         const ogcp_loss* loss, int32_t* coords_out, double* vals_out, int64_t* n_out);
/* Row-segment layout of mode `mode` of a COO coordinate list (device int32
 * [n x ndim]): perm_out = stable argsort of column `mode`
 * (np.argsort(..., kind="stable")), offsets_out[r] = start of row r, r = 0..dim
 * (cumsum of bincount) -- the layout a sort-by-row MTTKRP walks. */
int ogcp_segment_layout(ogcp_ctx* ctx, const int32_t* coords_dev, int64_t n, int32_t ndim, int32_t mode,
                        int64_t dim, int32_t* perm_out, int64_t* offsets_out);

/* Full factor_gradients (solvers.py:127-142, 159-179): data term + lambda*A
 * + history Gram term.  old_factors may be NULL when H == 0 or hist_weight == 0.
 * window_s is host [H x rank] float64, window_ids host [H]. */
int ogcp_factor_gradients(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev,
                          int64_t p, const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m,
                          float* const* old_factors, const double* weights, const ogcp_loss* loss,
                          const double* window_s, const int64_t* window_ids, int32_t H,
                          double hist_weight, double hist_decay, int64_t t, double reg_factors,
                          float* const* grads_dev);

/* estimate_objective (sampling.py:177-206) on a replayed sample set. */
int ogcp_estimate_objective(ogcp_ctx* ctx, const ogcp_slice* s, const int32_t* ordinals_dev,
                            int64_t p, const int32_t* zero_subs_dev, int64_t q, const ogcp_model* m,
                            float* const* old_factors, const double* weights, const ogcp_loss* loss,
                            const double* window_s, const int64_t* window_ids, int32_t H,
                            double hist_weight, double hist_decay, int64_t t, double reg_factors,
                            double reg_weights, double* out);

/* gram (kernels.py:75-98): hadamard over modes != skip of B_m' A_m, B = other
 * (nullable -> A).  skip < 0 means all modes.  out: host [rank x rank] float64. */
int ogcp_gram(ogcp_ctx* ctx, const ogcp_model* m, float* const* other, int32_t skip, double* out);

/* Adam.step (adam.py:51-81) on device buffers shaped like the model. */
int ogcp_adam_step(ogcp_ctx* ctx, const ogcp_model* m, float* const* grads, ogcp_adam_state* st,
                   double beta1, double beta2, double eps, double lower_bound, int64_t step_count);
/* Adam.update (adam.py:83-94): accept snapshots, reject restores + decays rate. */
int ogcp_adam_update(ogcp_ctx* ctx, const ogcp_model* m, ogcp_adam_state* st, int32_t passed,
                     double rate_decay);

/* ---------------------------------------------------------------- solves */
/* solve_weights (solvers.py:197-268): temporal-row GCP-SGD with the factors
 * fixed; s_init host [rank] (nullable), s_out host [rank]. */
int ogcp_solve_weights(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_solver_config* cfg,
                       const ogcp_loss* loss, int64_t t, const ogcp_model* m,
                       const double* s_init, double* s_out, ogcp_trace* trace);

/* solve_factors (solvers.py:290-368): factor GCP-SGD with the weights fixed,
 * persistent Adam and counter.  m->factors are updated in place. */
int ogcp_solve_factors(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_solver_config* cfg,
                       const ogcp_loss* loss, int64_t t, const ogcp_model* m,
                       float* const* old_factors, const double* weights, const double* window_s,
                       const int64_t* window_ids, int32_t H, ogcp_adam_state* adam,
                       int64_t* iteration, ogcp_trace* trace);

/* solve_static (solvers.py:371-493, sampled mode, one restart): joint GCP-SGD
 * over the weights and every factor of a (d+1)-way block, keyed (seed,
 * seed_key, PHASE_STATIC_*).  m->factors (device, updated in place) hold the
 * initial factors, weights (host [rank], in/out) the initial weights; adam
 * holds zeroed factor moments and the rate (decayed on rejections).  The
 * epoch loop runs max_epochs x iters at tolerance tol. */
int ogcp_solve_static(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_solver_config* cfg,
                      const ogcp_loss* loss, int64_t seed_key, const ogcp_model* m, double* weights,
                      ogcp_adam_state* adam, int32_t max_epochs, int32_t iters, double tol,
                      ogcp_trace* trace);

/* ------------------------------------------------ Gaussian special cases */
/* solve_weights_least_squares (solvers.py:271-288): (hadamard_k Gram_k + mu I) s
 * = Z' vec(X) over the stored entries; s_out host [rank].  An exactly singular
 * system is OGCP_E_DATA. */
int ogcp_solve_weights_ls(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m, double reg_weights,
                          double* s_out);

/* gaussian_sum_sq_residual (kernels.py:135-146): sum over every cell of (x - m)^2
 * = ||X||^2 - 2 <X, M> + ||M||^2.  weights host [rank]. */
int ogcp_gaussian_residual(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m, const double* weights,
                           double* out);

/* dense_gaussian_factor_gradients (solvers.py:145-156) into grads_dev (nullable,
 * device, model layout) and _dense_gaussian_weight_gradient (solvers.py:182-185)
 * into weight_grad (nullable, host [rank]). */
int ogcp_dense_gaussian_gradients(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m,
                                  float* const* old_factors, const double* weights, const double* window_s,
                                  const int64_t* window_ids, int32_t H, double hist_weight, double hist_decay,
                                  int64_t t, double reg_factors, double reg_weights, float* const* grads_dev,
                                  double* weight_grad);

/* Diagnostics: a one-rank NCCL communicator round trip through every collective
 * the multi-GPU solves use (checks the run-time loaded libnccl.so.2 on one GPU). */
int ogcp_comm_selftest(ogcp_ctx* ctx, int32_t* mismatches);

/* Diagnostics: the gradient sample set a solve iteration would evaluate on
 * this context (merged/bucketed form and multi-GPU share included), keyed
 * rng_at(seed, *key): this rank's nonzero ordinals with multiplicities and its
 * accepted zero rows.  Used by the tests of the shard partition. */
int ogcp_debug_solve_draw(ogcp_ctx* ctx, const ogcp_slice* s, uint64_t seed, const int64_t* key, int32_t nkey,
                          int64_t p, int64_t q, int64_t max_rejects, int32_t ldr, int64_t cap_nz, int32_t* ord_out,
                          uint8_t* cnt_out, int64_t* n_nz, int64_t cap_zero, int32_t* zero_out, int64_t* n_zero);

/* local_loss (metrics.py:36-70): mode 0 exact (every cell, <= max_elements),
 * mode 1 sampled on rng_at(seed, *key) with (p, q) (p < 0: all nonzeros).
 * Returns the loss total divided by ||X||^2 when that is > 0; *normalized says which. */
int ogcp_local_loss(ogcp_ctx* ctx, const ogcp_slice* s, const ogcp_model* m, const double* weights,
                    const ogcp_loss* loss, int32_t mode, int64_t p, int64_t q, uint64_t seed,
                    const int64_t* key, int32_t nkey, int64_t max_rejects, int64_t max_elements,
                    double* out, int32_t* normalized);

#ifdef __cplusplus
}
#endif
#endif /* OGCP_B200_H */
