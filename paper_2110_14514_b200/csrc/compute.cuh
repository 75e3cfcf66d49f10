#pragma once
#include "common.cuh"

namespace ogcp {

// One sample set on the device: p nonzero ordinals into the slice records and
// q zero coordinates (int32 [q x ndim]); scales per sampling.py:99-105.
// Merged (count) form: ord holds the distinct drawn ordinals in ascending
// order, cnt their multiplicities, and the distinct count lives on the device
// (p_dev); p is then an upper bound used only for launch sizing.  nz_scale is
// always eta / (number of draws).
struct SamplesP {
  const int32_t* ord;
  int64_t p;
  const int32_t* zsub;
  int64_t q;
  const int* rec;
  int rec_ints;
  double nz_scale, zero_scale;
  const long long* p_dev;   // nullable: distinct nonzero count (merged form)
  const uint8_t* cnt;       // nullable: multiplicity per merged nonzero
  const long long* q_dev;   // nullable: lazy zero layout, rows [0, *q_dev) with -1-flagged rows skipped
  int shard_rank, shard_world;  // multi-GPU: this rank evaluates its contiguous 1/world of the samples
  int semi;                 // semi-stratified estimator: nonzero draws use g(x,m) - g(0,m); zero_scale = omega/q
  int chunk_shift;          // bucketed merged set: warps walk chunks of 2^chunk_shift batches round-robin
  int zshard;               // multi-GPU merged set: the nonzero part is rank-owned; zero rows split
                            // (1: a contiguous 1/world of [0, *q_dev)) or already rank-local (2: all of them)
};

struct GradPtrs {
  float* g[kMaxModes];
};

struct ModelP {
  const float* A[kMaxModes];
  int ndim, rank, ldr;
  int64_t dims[kMaxModes];
};

struct LossP {
  int kind;
  float eps;
  double eps_d;
};

// K2+K3: data term of every factor gradient, grads[k] = mttkrp(Y,k)*diag(s)
// (zeroed and written).  s_f: float [ldr] weights (padding zero).
void sgrad_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                   float* const* grads, long long code);
// Temporal-row Adam step (k_weight_step's arithmetic) fused into the tail of a
// K2w launch: the last block to finish sums the block partials in block order
// and updates the R-vector state.  ticket: a device counter that is 0 between
// launches (the last block resets it).
struct WStep {
  int rank, ldr;
  double* ws;
  float* s_f;
  double mu, rate_i, b1, b2, eps, lower;
  long long code;
  unsigned int* ticket;
};
// K2 (weight solve): per-block partial sums of Z'vec(Y) into partials [nblk x ldr] double.
// With `step`, the walk kernel also applies the weight step when it can (*stepped
// tells whether it did; otherwise the caller runs weight_step_enqueue).
int wgrad_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                  double* partials, long long code, const WStep* step = nullptr, bool* stepped = nullptr);
// K6: per-block partial sums of scale*f(x,m) into partials; returns the block count.
int objective_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                      double* partials, long long code);
// Sum nblk partial vectors of length len (fixed order) into out.
void sum_partials_enqueue(Ctx* ctx, const double* partials, int nblk, int len, double* out);
// K4: out[R x R] = B' A over rows (fp64 accumulation), A/B rows x ldr.
void gram_enqueue(Ctx* ctx, const float* A, const float* B, int64_t rows, int rank, int ldr, double* out,
                  DevBuf& scratch);
// K4 pair: outP = A'A and (B != nullptr) outC = B'A in one pass over the rows.
void gram2_enqueue(Ctx* ctx, const float* A, const float* B, int64_t rows, int rank, int ldr, double* outP,
                   double* outC, DevBuf& scratch);
// History coefficients: Mk = w*(hadamard_{m!=k} P_m) o S, Nk = w*(hadamard_{m!=k} C_m) o S  (float [d][R][R]).
// Dense-Gaussian model term: Mk += extra * Gamma_k o s s' (s: device double [R], nullable); C / S nullable.
void hist_coeffs_enqueue(Ctx* ctx, int ndim, int rank, const double* P, const double* C, const double* S,
                         double w, float* Mk, float* Nk, const double* s = nullptr, double extra = 0.0);
// Dense-Gaussian weight gradient 2((hadamard_m P_m) s - b) into out[ldr] (one block).
void dense_wgrad_enqueue(Ctx* ctx, int ndim, int rank, int ldr, const double* P, const double* b, const double* s,
                         double* out);
// Small models (every mode <= kSmallRows rows, ldr <= 32): all modes in one launch.
constexpr int64_t kSmallRows = 4096;
struct SmallGrams {
  const float* A[kMaxModes];
  const float* B1[kMaxModes];
  const float* B2[kMaxModes];  // nullable
  int64_t rows[kMaxModes];
};
// Optional tail of the small-model Gram launch: the last mode-block to finish
// also computes the history coefficients of every mode (k_hist_coeffs' arithmetic).
struct CoeffTail {
  const double* S;   // nullable
  double w;
  const double* s;   // nullable (dense-Gaussian model term)
  double extra;
  float* Mk;
  float* Nk;
  unsigned int* ticket;  // nullptr: no tail
};
void gram_small_enqueue(Ctx* ctx, const SmallGrams& g, int ndim, int rank, int ldr, double* out1, double* out2,
                        const CoeffTail* tail = nullptr);
struct K5Modes {
  float* A[kMaxModes];
  const float* Aold[kMaxModes];
  const float* G[kMaxModes];
  float* u[kMaxModes];
  float* v[kMaxModes];
  const float* Mk[kMaxModes];
  const float* Nk[kMaxModes];
  int64_t rows[kMaxModes];
};
void factor_update_modes_enqueue(Ctx* ctx, const K5Modes& m, int ndim, int rank, int ldr, double reg, double rate_i,
                                 double beta1, double beta2, double eps, double lower, long long code);
// K5: g = G + lambda*A + (A Mk - Aold Nk) ; Adam ; clamp ; isfinite  (one mode).
void factor_update_enqueue(Ctx* ctx, int64_t rows, int rank, int ldr, float* A, const float* Aold,
                           const float* G, float* u, float* v, const float* Mk, const float* Nk,
                           double reg, double rate_i, double beta1, double beta2, double eps, double lower,
                           long long code);
// Weight solve step: g = sum(partials) + mu*s ; Adam on the R-vector (double) ; s_f refresh.
void weight_step_enqueue(Ctx* ctx, const double* partials, int nblk, int rank, int ldr, double* wstate,
                         float* s_f, double mu, double rate_i, double beta1, double beta2, double eps,
                         double lower, long long code);
// Objective finalisation on device: data partials + window quad forms + regularizers.
void hist_penalty_enqueue(Ctx* ctx, int ndim, int rank, const double* Poo, const double* Pon,
                          const double* Pnn, const double* window_s, const double* window_coef, int H,
                          double* out);
// Exact loss over every cell (metrics.py:50-57) : partial sums.
int exact_cells_enqueue(Ctx* ctx, const ModelP& M, const float* s_f, const LossP& L, int64_t omega,
                        double* partials, long long code);
int exact_nz_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                     double* partials, long long code);

}  // namespace ogcp
