// K2..K6: sampled-entry model evaluation, loss/derivative, sampled-MTTKRP
// scatter, weight gradient, objective, Gram, history and fused Adam.
//
// Thread mapping for the sample kernels: a group of G lanes serves one sample;
// lane gl owns the float4 chunks v*G+gl (v < V) of every factor row, so the
// d row gathers of a sample are G*16-byte contiguous 128-bit loads (one 128 B
// line per row at R = 32), the Hadamard product and the dot with s stay in
// registers and m is reduced with log2(G) xor-shuffles.  Each group works on
// U samples at a time and issues the three dependent gather stages
// (ordinal -> record -> factor rows) for all U before using any of them, so a
// warp keeps 3*U*SPW independent 128-bit loads in flight.
//
// Reference: model_values tensor.py:203-211; LossFunction losses.py:58-78;
// sampled_mttkrp kernels.py:33-56 (times s, solvers.py:139-140);
// weight_gradient_mttkrp kernels.py:59-72; estimate_objective
// sampling.py:177-206; gram kernels.py:75-98; _add_reg_and_history
// solvers.py:159-179; Adam.step adam.py:51-81; _ensure_finite solvers.py:188-194.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <unordered_map>

#include "common.cuh"
#include "compute.cuh"

namespace ogcp {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;
// minimum resident CTAs per SM for the sample kernels (register budget); tuned on B200
#ifndef OGCP_SGRAD_MINB
#define OGCP_SGRAD_MINB 1
#endif
#ifndef OGCP_WGRAD_MINB
#define OGCP_WGRAD_MINB 2
#endif

template <int D>
struct ND {
  static constexpr int v = D > 0 ? D : 7;
};

__device__ __forceinline__ float4 mul4(float4 a, float4 b) {
  return make_float4(a.x * b.x, a.y * b.y, a.z * b.z, a.w * b.w);
}
__device__ __forceinline__ float dot4(float4 a, float4 b) { return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w; }

__device__ __forceinline__ void red_add_v4(float* addr, float4 v) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

// d f/d m (losses.py:69-78) in fp32.
__device__ __forceinline__ float dloss(int kind, float x, float m, float eps) {
  if (kind == OGCP_IDENTITY) return x;
  if (kind == OGCP_GAUSSIAN) return 2.0f * (m - x);
  if (kind == OGCP_POISSON) return 1.0f - x / (m + eps);
  return 1.0f / (m + 1.0f) - x / (m + eps);
}
// f (losses.py:58-67) in fp64.
// IDENTITY gives the cross term x*m of the exact Gaussian residual (kernels.py:143).
__device__ __forceinline__ double floss(int kind, double x, double m, double eps) {
  if (kind == OGCP_IDENTITY) return x * m;
  if (kind == OGCP_GAUSSIAN) return (x - m) * (x - m);
  if (kind == OGCP_POISSON) return m - x * log(m + eps);
  return log(m + 1.0) - x * log(m + eps);
}
__device__ __forceinline__ unsigned domain_bits(int kind, float m) {
  unsigned b = 0;
  if (kind == OGCP_IDENTITY) return 0u;
  if (!isfinite(m)) b |= 1u;
  if (kind != OGCP_GAUSSIAN && m < 0.0f) b |= 2u;
  return b;
}

__device__ __forceinline__ void report(DevFlags* f, int which, long long code, unsigned bits) {
  atomicMin(&f->first_code[which], code);
  if (bits) atomicOr(&f->data_bits, bits);
}

template <int D, int V>
struct Sample {
  int idx[ND<D>::v];
  float4 a[ND<D>::v][V];
  float x;
  float scale;
  float cnt;  // multiplicity of a merged nonzero (1 otherwise)
  int64_t n;  // index in the sample set
  bool nz;
};

// Software-pipelined sample stream.  A warp walks batches of SPW*U samples with
// a grid stride; while the factor rows of batch b are in flight, the records
// (or zero coordinates) of batch b+stride and the ordinals of batch b+2*stride
// are already being fetched, so the three dependent gathers of a sample
// (ordinal -> record -> rows) overlap across batches instead of serialising.
template <int D, int G, int V, int U>
struct SampleStream {
  static constexpr int NDm = ND<D>::v;
  static constexpr int SPW = 32 / G;
  static constexpr int SPB = SPW * U;
  static constexpr int RI = (D > 0 && D <= 3) ? 4 : 8;
  SamplesP S;
  const ModelP* M;
  int64_t p, total, b, end;
  int64_t zoff;  // walk index m >= p maps to sample p + zoff + (m - p) (zero-row share of a rank)
  int lane, gl, nd;
  int skip = -1;  // mode whose rows are not gathered (split scatter, pass 2)
  int oB[U];
  float cB[U], cC[U];
  int tC[U][RI];

  __device__ __forceinline__ int64_t nidx(int64_t base, int u) const { return base + u * SPW + lane / G; }

  __device__ __forceinline__ void load_ord(int64_t base, int (&o)[U], float (&c)[U]) const {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t n = nidx(base, u);
      const bool nz = n < p && n < end;
      o[u] = nz ? __ldg(S.ord + n) : 0;
      c[u] = (S.cnt && nz) ? (float)__ldg(S.cnt + n) : 1.0f;
    }
  }

  __device__ __forceinline__ void load_rec(int64_t base, const int (&o)[U], int (&t)[U][RI]) const {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t n = nidx(base, u);
#pragma unroll
      for (int k = 0; k < RI; ++k) t[u][k] = 0;
      if (n >= end) continue;
      if (n < p) {
        const int4* r = reinterpret_cast<const int4*>(S.rec + (int64_t)o[u] * S.rec_ints);
        const int4 v0 = __ldg(r);
        t[u][0] = v0.x; t[u][1] = v0.y; t[u][2] = v0.z; t[u][3] = v0.w;
        if (RI == 8 && S.rec_ints == 8) {
          const int4 v1 = __ldg(r + 1);
          t[u][RI > 4 ? 4 : 0] = v1.x; t[u][RI > 4 ? 5 : 1] = v1.y;
          t[u][RI > 4 ? 6 : 2] = v1.z; t[u][RI > 4 ? 7 : 3] = v1.w;
        }
      } else {
        const int32_t* z = S.zsub + (n + zoff - p) * nd;
#pragma unroll
        for (int k = 0; k < NDm; ++k)
          if (k < nd) t[u][k] = __ldg(z + k);
      }
    }
  }

  // Walk order.  contiguous = true: warp w walks its own contiguous range of
  // samples (keeps the ordinal order of a merged sample set, so consecutive
  // samples of a group share mode-0 rows).  Otherwise warps take chunks of
  // 2^S.chunk_shift batches round-robin (shift 0: plain grid-stride batches), so
  // the warps in flight stay inside a narrow window of the set -- one row bucket
  // of a bucketed merged set, whose rows then stay in L2.
  int64_t lo_, warp_, nwarps_, t_ = 0;
  int64_t stride_ = 0, b1_ = 0, b2_ = 0;  // unchunked walks: fixed stride, next two batch bases
  int cshift = 0;
  bool contig = false;
  __device__ __forceinline__ int64_t base_of(int64_t t) const {
    const int64_t chunk = t >> cshift;
    const int64_t within = t & ((1 << cshift) - 1);
    return lo_ + (((warp_ + chunk * nwarps_) << cshift) + within) * SPB;
  }

  __device__ __forceinline__ void init(const SamplesP& S_, const ModelP& M_, int lane_, int64_t warp,
                                       int64_t nwarps, bool contiguous = false) {
    S = S_;
    M = &M_;
    p = S.p_dev ? (int64_t)*S.p_dev : S.p;
    total = p + (S.q_dev ? (int64_t)*S.q_dev : S.q);
    lane = lane_;
    gl = lane & (G - 1);
    nd = D > 0 ? D : M_.ndim;
    int64_t lo = 0, hi = total;
    zoff = 0;
    if (S.shard_world > 1 && S.zshard == 2) {
      // word-sharded draw: rank-owned merged nonzeros and rank-local zero rows, all of them
    } else if (S.shard_world > 1 && S.zshard == 1) {  // rank-owned merged nonzeros + a contiguous share of the zero rows
      const int64_t zrows = total - p;
      const int64_t zlo = zrows * S.shard_rank / S.shard_world, zhi = zrows * (S.shard_rank + 1) / S.shard_world;
      hi = p + (zhi - zlo);
      zoff = zlo;
    } else if (S.shard_world > 1) {  // sample-sharded multi-GPU solve: this rank's contiguous share
      lo = total * S.shard_rank / S.shard_world;
      hi = total * (S.shard_rank + 1) / S.shard_world;
    }
    contig = contiguous;
    warp_ = warp;
    nwarps_ = nwarps;
    if (contiguous) {
      const int64_t per = ((hi - lo + nwarps - 1) / nwarps + SPB - 1) / SPB * SPB;
      b = lo + warp * per;
      end = min(hi, b + per);
      stride_ = SPB;
    } else {
      lo_ = lo;
      cshift = S.chunk_shift;
      end = hi;
      b = base_of(0);
      stride_ = cshift ? 0 : nwarps * SPB;
      if (cshift) {
        b1_ = base_of(1);
        b2_ = base_of(2);
      }
    }
    if (stride_) {
      b1_ = b + stride_;
      b2_ = b + 2 * stride_;
    }
    int o0[U];
    float c0[U];
    load_ord(b, o0, c0);
    load_rec(b, o0, tC);
#pragma unroll
    for (int u = 0; u < U; ++u) cC[u] = c0[u];
    load_ord(b1_, oB, cB);
  }

  // Fill the per-sample fields of the current batch except the factor rows.
  __device__ __forceinline__ void meta(Sample<D, V> (&s)[U], bool (&valid)[U]) const {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t n = nidx(b, u);
      s[u].nz = n < p;
      valid[u] = n < end && (s[u].nz || tC[u][0] >= 0);  // -1: rejected candidate (lazy zero layout)
      s[u].scale = s[u].nz ? (float)S.nz_scale * cC[u] : (float)S.zero_scale;
      s[u].cnt = s[u].nz ? cC[u] : 1.0f;
      float x = 0.0f;
      if (D > 0) x = __int_as_float(tC[u][D < RI ? D : 0]);
      else {
#pragma unroll
        for (int k = 0; k < RI; ++k)
          if (k == nd) x = __int_as_float(tC[u][k]);
      }
      s[u].x = s[u].nz ? x : 0.0f;
      s[u].n = s[u].nz ? n : n + zoff;
#pragma unroll
      for (int k = 0; k < NDm; ++k) s[u].idx[k] = tC[u][k < RI ? k : 0];
    }
  }

  // Move the ordinal/record stages one batch forward.
  __device__ __forceinline__ void advance() {
    // stage 2 for the next batch, stage 1 for the one after
    int tB[U][RI];
    load_rec(b1_, oB, tB);
#pragma unroll
    for (int u = 0; u < U; ++u) cC[u] = cB[u];
    load_ord(b2_, oB, cB);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < RI; ++k) tC[u][k] = tB[u][k];
    b = b1_;
    b1_ = b2_;
    b2_ = stride_ ? b2_ + stride_ : base_of(++t_ + 2);
  }

  // Issue the row gathers of the current batch (and the next batches' earlier
  // stages); returns false when the warp has no batch left.
  __device__ __forceinline__ bool next(Sample<D, V> (&s)[U], bool (&valid)[U]) {
    if (b >= end) return false;
    meta(s, valid);
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int k = 0; k < NDm; ++k) {
        if (k < nd && k != skip) {
          const float4* row = reinterpret_cast<const float4*>(M->A[k] + (int64_t)s[u].idx[k] * M->ldr);
#pragma unroll
          for (int v = 0; v < V; ++v)
            s[u].a[k][v] = valid[u] ? __ldg(row + v * G + gl) : make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) s[u].a[k][v] = make_float4(1.f, 1.f, 1.f, 1.f);
        }
      }
    }
    advance();
    return true;
  }
};

template <int D, int G, int V>
__device__ __forceinline__ float model_value(const Sample<D, V>& s, const float4* s4) {
  constexpr int NDm = ND<D>::v;
  float part = 0.0f;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    float4 pr = s.a[0][v];
#pragma unroll
    for (int k = 1; k < NDm; ++k) pr = mul4(pr, s.a[k][v]);
    part += dot4(pr, s4[v]);
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
  return part;
}

// ------------------------------------------------------------------ K2+K3
// Small modes (dims*ldr*4 bytes within the shared-memory budget) are
// privatised per CTA and flushed once; large modes use 16-byte vector
// reductions (REDG.F32x4) into L2.
struct PrivP {
  int nmodes;
  int mode[kMaxModes];
  int64_t off[kMaxModes];  // float offset in dynamic smem
  int64_t len[kMaxModes];  // floats
};

// SEG: the sample set is a merged (ordinal-sorted) one walked in contiguous
// per-warp ranges; each lane group accumulates its mode-0 contributions in
// registers while consecutive samples share the mode-0 row and issues one
// reduction per row segment (sort-by-row segmented reduction for mode 0).
//
// split >= 0 (split scatter, pass 1): mode `split` is not scattered here; the
// sample's y is stored in ybuf[n] for k_sgrad_split.
template <int D, int G, int V, int U, bool SEG>
__global__ void __launch_bounds__(kThreads, OGCP_SGRAD_MINB) k_sgrad(SamplesP S, ModelP M, const float* __restrict__ s_f, LossP L,
                                                    GradPtrs GP, PrivP PV, DevFlags* flags, long long code,
                                                    int split, float* __restrict__ ybuf) {
  extern __shared__ float smem[];
  constexpr int NDm = ND<D>::v;
  const int nd = D > 0 ? D : M.ndim;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  const int64_t plen = PV.nmodes ? PV.off[PV.nmodes - 1] + PV.len[PV.nmodes - 1] : 0;
  for (int64_t i = threadIdx.x; i < plen; i += blockDim.x) smem[i] = 0.0f;
  __syncthreads();
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * G + gl);
  int priv_slot[NDm];
#pragma unroll
  for (int k = 0; k < NDm; ++k) {
    priv_slot[k] = -1;
#pragma unroll
    for (int j = 0; j < kMaxModes; ++j)
      if (j < PV.nmodes && PV.mode[j] == k) priv_slot[k] = j;
  }
  const int64_t total = S.p + S.q;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bits = 0;
  SampleStream<D, G, V, U> stream;
  stream.init(S, M, lane, warp, nwarps, SEG && S.chunk_shift == 0);
  Sample<D, V> s[U];
  bool valid[U];
  const bool seg0 = SEG && priv_slot[0] < 0;
  int seg_row = -1;
  float4 seg_acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) seg_acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  while (stream.next(s, valid)) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float m = model_value<D, G, V>(s[u], s4);
      if (valid[u]) {
        bits |= domain_bits(L.kind, m);
        float y = dloss(L.kind, s[u].x, m, L.eps);
        if (S.semi && s[u].nz) y -= dloss(L.kind, 0.0f, m, L.eps);  // semi-stratified nonzero stratum
        y *= s[u].scale;
        if (split >= 0 && gl == 0) ybuf[s[u].n] = y;
        if (seg0 && s[u].idx[0] != seg_row) {
          if (seg_row >= 0) {
#pragma unroll
            for (int v = 0; v < V; ++v) red_add_v4(GP.g[0] + (int64_t)seg_row * M.ldr + (v * G + gl) * 4, seg_acc[v]);
          }
          seg_row = s[u].idx[0];
#pragma unroll
          for (int v = 0; v < V; ++v) seg_acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < NDm; ++k) {
          if (k >= nd) break;
          if (k == split) continue;
#pragma unroll
          for (int v = 0; v < V; ++v) {
            float4 c = make_float4(y * s4[v].x, y * s4[v].y, y * s4[v].z, y * s4[v].w);
#pragma unroll
            for (int j = 0; j < NDm; ++j)
              if (j != k && j < nd) c = mul4(c, s[u].a[j][v]);
            const int64_t off = (int64_t)s[u].idx[k] * M.ldr + (v * G + gl) * 4;
            if (k == 0 && seg0) {
              seg_acc[v].x += c.x;
              seg_acc[v].y += c.y;
              seg_acc[v].z += c.z;
              seg_acc[v].w += c.w;
            } else if (priv_slot[k] >= 0) {
              float* p = smem + PV.off[priv_slot[k]] + off;
              atomicAdd(p + 0, c.x);
              atomicAdd(p + 1, c.y);
              atomicAdd(p + 2, c.z);
              atomicAdd(p + 3, c.w);
            } else {
              red_add_v4(GP.g[k] + off, c);
            }
          }
        }
      }
    }
  }
  if (seg0 && seg_row >= 0) {
#pragma unroll
    for (int v = 0; v < V; ++v) red_add_v4(GP.g[0] + (int64_t)seg_row * M.ldr + (v * G + gl) * 4, seg_acc[v]);
  }
  if (bits) report(flags, kFlagData, code, bits);
  if (PV.nmodes) {
    __syncthreads();
    for (int j = 0; j < PV.nmodes; ++j) {
      const float4* src = reinterpret_cast<const float4*>(smem + PV.off[j]);
      float* dst = GP.g[PV.mode[j]];
      for (int64_t i = threadIdx.x; i < PV.len[j] / 4; i += blockDim.x) {
        float4 c = src[i];
        if (c.x != 0.f || c.y != 0.f || c.z != 0.f || c.w != 0.f) red_add_v4(dst + i * 4, c);
      }
    }
  }
}

// Split scatter, pass 2: the contributions of mode `split` from the stored y,
// without that mode's row gathers; run separately so the 16-byte reductions
// into G_split meet an L2 that holds G_split instead of the gathered rows.
template <int D, int G, int V, int U>
__global__ void __launch_bounds__(kThreads) k_sgrad_split(SamplesP S, ModelP M, const float* __restrict__ s_f,
                                                          const float* __restrict__ ybuf, float* __restrict__ Gs,
                                                          int split) {
  constexpr int NDm = ND<D>::v;
  const int nd = D > 0 ? D : M.ndim;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * G + gl);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  SampleStream<D, G, V, U> stream;
  stream.skip = split;
  stream.init(S, M, lane, warp, nwarps, S.cnt != nullptr && S.chunk_shift == 0);
  Sample<D, V> s[U];
  bool valid[U];
  while (stream.next(s, valid)) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!valid[u]) continue;
      const float y = __ldg(ybuf + s[u].n);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float4 c = make_float4(y * s4[v].x, y * s4[v].y, y * s4[v].z, y * s4[v].w);
#pragma unroll
        for (int j = 0; j < NDm; ++j)
          if (j != split && j < nd) c = mul4(c, s[u].a[j][v]);
        red_add_v4(Gs + (int64_t)s[u].idx[split] * M.ldr + (v * G + gl) * 4, c);
      }
    }
  }
}

// Temporal-row Adam step (adam.py:51-81 on the R-vector, fp64) of entry r < ldr
// given its summed gradient g (without the mu term).
__device__ __forceinline__ void weight_step_apply(int r, double g, int rank, int ldr, double* ws, float* s_f,
                                                  double mu, double rate_i, double b1, double b2, double eps,
                                                  double lower, DevFlags* flags, long long code) {
  if (r >= rank) {
    s_f[r] = 0.f;
    return;
  }
  double s = ws[r];
  g += mu * s;
  double u = b1 * ws[ldr + r] + (1.0 - b1) * g;
  double v = b2 * ws[2 * ldr + r] + (1.0 - b2) * g * g;
  double sn = s - rate_i * u / (sqrt(v) + eps);
  if (sn < lower) sn = lower;
  ws[r] = sn;
  ws[ldr + r] = u;
  ws[2 * ldr + r] = v;
  s_f[r] = (float)sn;
  // the sample kernels evaluate in fp32: an iterate beyond fp32 range has diverged for this engine
  if (!isfinite(sn) || !isfinite((float)sn)) report(flags, kFlagDiverge, code, 0);
}

// Thread r < ldr sums column r of the nblk block partials in block order (deterministic).
__device__ __forceinline__ void weight_step_body(const double* partials, int nblk, int rank, int ldr, double* ws,
                                                 float* s_f, double mu, double rate_i, double b1, double b2,
                                                 double eps, double lower, DevFlags* flags, long long code) {
  const int r = threadIdx.x;
  if (r >= ldr) return;
  double g = 0.0;
  for (int b = 0; b < nblk; ++b) g += partials[(int64_t)b * ldr + r];
  weight_step_apply(r, g, rank, ldr, ws, s_f, mu, rate_i, b1, b2, eps, lower, flags, code);
}

// ------------------------------------------------------------------ K2 (weights)
template <int D, int G, int V, int U>
__global__ void __launch_bounds__(kThreads, OGCP_WGRAD_MINB) k_wgrad(SamplesP S, ModelP M, const float* __restrict__ s_f, LossP L,
                                                    double* __restrict__ partials, DevFlags* flags, long long code,
                                                    WStep step) {
  __shared__ double red[kThreads / 32][4 * V * G];
  constexpr int NDm = ND<D>::v;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * G + gl);
  double acc[V][4];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v][0] = acc[v][1] = acc[v][2] = acc[v][3] = 0.0;
  const int64_t total = S.p + S.q;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bits = 0;
  SampleStream<D, G, V, U> stream;
  stream.init(S, M, lane, warp, nwarps, S.cnt != nullptr && S.chunk_shift == 0);
  Sample<D, V> s[U];
  bool valid[U];
  while (stream.next(s, valid)) {
    float4 part[V];
#pragma unroll
    for (int v = 0; v < V; ++v) part[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float m = model_value<D, G, V>(s[u], s4);
      if (valid[u]) {
        bits |= domain_bits(L.kind, m);
        float y = dloss(L.kind, s[u].x, m, L.eps);
        if (S.semi && s[u].nz) y -= dloss(L.kind, 0.0f, m, L.eps);  // semi-stratified nonzero stratum
        y *= s[u].scale;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          float4 pr = s[u].a[0][v];
#pragma unroll
          for (int k = 1; k < NDm; ++k) pr = mul4(pr, s[u].a[k][v]);
          part[v].x += y * pr.x;
          part[v].y += y * pr.y;
          part[v].z += y * pr.z;
          part[v].w += y * pr.w;
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      acc[v][0] += (double)part[v].x;
      acc[v][1] += (double)part[v].y;
      acc[v][2] += (double)part[v].z;
      acc[v][3] += (double)part[v].w;
    }
  }
  if (bits) report(flags, kFlagData, code, bits);
  // reduce lanes with the same gl (fixed order), then warps in order
#pragma unroll
  for (int o = G; o < 32; o <<= 1)
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[v][e] += __shfl_xor_sync(kFull, acc[v][e], o);
  const int w = threadIdx.x >> 5;
  if (lane < G) {
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int e = 0; e < 4; ++e) red[w][(v * G + lane) * 4 + e] = acc[v][e];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 4 * V * G; c += blockDim.x) {
    double t = 0.0;
    for (int j = 0; j < kThreads / 32; ++j) t += red[j][c];
    partials[blockIdx.x * (int64_t)(4 * V * G) + c] = t;
  }
  if (step.ticket) {  // fused weight step: the last block to finish applies it
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(step.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) {
      // all threads of the last block sum the partials: thread t takes column t % ldr of
      // every J-th block (J = blockDim / ldr), then the J sums combine in fixed order
      __shared__ double colsum[kThreads];
      __threadfence();
      const int ldr = step.ldr;
      const int J = kThreads / ldr;
      const int t = threadIdx.x, r = t % ldr, j = t / ldr;
      double a = 0.0;
      if (j < J)
        for (int b = j; b < (int)gridDim.x; b += J) a += partials[(int64_t)b * ldr + r];
      colsum[t] = a;
      __syncthreads();
      if (t < ldr) {
        double g = 0.0;
        for (int jj = 0; jj < J; ++jj) g += colsum[jj * ldr + t];
        weight_step_apply(t, g, step.rank, ldr, step.ws, step.s_f, step.mu, step.rate_i, step.b1, step.b2, step.eps,
                          step.lower, flags, step.code);
      }
      if (threadIdx.x == 0) *step.ticket = 0u;
    }
  }
}

// ------------------------------------------------------------------ K6
// MODE 0: sum scale * f(x, m) (objective); MODE 1: sum f(x,m) - f(0,m) (exact-loss nonzero correction).
template <int D, int G, int V, int U, int MODE>
__global__ void __launch_bounds__(kThreads) k_objective(SamplesP S, ModelP M, const float* __restrict__ s_f,
                                                        LossP L, double* __restrict__ partials, DevFlags* flags,
                                                        long long code) {
  __shared__ double red[kThreads / 32];
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * G + gl);
  double acc_nz = 0.0, acc_z = 0.0;
  const int64_t total = S.p + S.q;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bits = 0;
  SampleStream<D, G, V, U> stream;
  stream.init(S, M, lane, warp, nwarps, S.cnt != nullptr && S.chunk_shift == 0);
  Sample<D, V> s[U];
  bool valid[U];
  while (stream.next(s, valid)) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const float m = model_value<D, G, V>(s[u], s4);
      if (valid[u] && gl == 0) {
        bits |= domain_bits(L.kind, m);
        double f = floss(L.kind, (double)s[u].x, (double)m, L.eps_d);
        if (MODE == 1 || (S.semi && s[u].nz)) f -= floss(L.kind, 0.0, (double)m, L.eps_d);
        if (s[u].nz) acc_nz += f * (double)s[u].cnt;
        else acc_z += f;
      }
    }
  }
  if (bits) report(flags, kFlagData, code, bits);
  double acc = MODE == 0 ? acc_nz * S.nz_scale + acc_z * S.zero_scale : acc_nz + acc_z;
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int j = 0; j < kThreads / 32; ++j) t += red[j];
    partials[blockIdx.x] = t;
  }
}

// Exact loss: f(0, m) over every cell of the box (cells enumerated in odometer order).
__global__ void __launch_bounds__(kThreads) k_exact_cells(ModelP M, const float* __restrict__ s_f, LossP L,
                                                          int64_t omega, double* __restrict__ partials,
                                                          DevFlags* flags, long long code) {
  __shared__ double red[kThreads / 32];
  double acc = 0.0;
  unsigned bits = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < omega; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = c;
    int idx[kMaxModes];
    for (int k = M.ndim - 1; k >= 0; --k) {
      idx[k] = (int)(rem % M.dims[k]);
      rem /= M.dims[k];
    }
    float m = 0.0f;
    for (int r = 0; r < M.rank; ++r) {
      float pr = s_f[r];
      for (int k = 0; k < M.ndim; ++k) pr *= M.A[k][(int64_t)idx[k] * M.ldr + r];
      m += pr;
    }
    bits |= domain_bits(L.kind, m);
    acc += floss(L.kind, 0.0, (double)m, L.eps_d);
  }
  if (bits) report(flags, kFlagData, code, bits);
  const int lane = threadIdx.x & 31;
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int j = 0; j < kThreads / 32; ++j) t += red[j];
    partials[blockIdx.x] = t;
  }
}

// Fixed-order column sums of block partials, spread over threads: a 256-thread
// block takes 32 columns x 8 segments; segment s sums blocks s, s + 8, ... in
// order (two interleaved accumulators), then the 8 segment sums combine in order.
// The order depends only on nblk, so the result is deterministic; a column's
// chain is nblk / 16 loads long instead of nblk.
constexpr int kColSumSegs = 8;
template <typename T>
__device__ __forceinline__ double seg_colsum(const T* __restrict__ p, int nblk, int64_t stride, int64_t off,
                                             int seg) {
  double t0 = 0.0, t1 = 0.0;
  int b = seg;
  for (; b + kColSumSegs < nblk; b += 2 * kColSumSegs) {
    t0 += (double)__ldg(p + (int64_t)b * stride + off);
    t1 += (double)__ldg(p + (int64_t)(b + kColSumSegs) * stride + off);
  }
  if (b < nblk) t0 += (double)__ldg(p + (int64_t)b * stride + off);
  return t0 + t1;
}

__global__ void __launch_bounds__(256) k_sum_partials_vec(const double* __restrict__ p, int nblk, int len,
                                                          double* __restrict__ out) {
  __shared__ double seg[kColSumSegs][32];
  const int lane = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  seg[sg][lane] = c < len ? seg_colsum(p, nblk, len, c, sg) : 0.0;
  __syncthreads();
  if (sg == 0 && c < len) {
    double t = 0.0;
    for (int j = 0; j < kColSumSegs; ++j) t += seg[j][lane];
    out[c] = t;
  }
}

// ------------------------------------------------------------------ K4 Gram
// P = A'A and (optionally) C = B'A in one pass over the rows.  Work item =
// (gram, 4x4 sub-block); a thread accumulates its sub-blocks over a row group
// in fp32 per 32-row tile and in fp64 across tiles; row groups are reduced in
// fixed order in shared memory, blocks by the finalize kernel.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int kGramTile = 32;
constexpr int kGramIPT = 2;
__global__ void __launch_bounds__(kThreads) k_gram2(const float* __restrict__ A, const float* __restrict__ B,
                                                    int64_t rows, int ldr, int ngram, int item0, int nitems_pass,
                                                    int64_t rows_per_block, double* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char gsm[];
  float* sa = reinterpret_cast<float*>(gsm);
  const int nsb = ldr / 4;
  const int nsub = nsb * nsb;
  const int nitems = ngram * nsub;
  // thread -> (items, row group)
  int nrg = 1, item_base = threadIdx.x;
  if (nitems_pass < kThreads) {
    nrg = kThreads / nitems_pass;
    item_base = threadIdx.x % nitems_pass;
  }
  const int rg = nitems_pass < kThreads ? threadIdx.x / nitems_pass : 0;
  const bool active = rg < nrg;
  int gi[kGramIPT], bi[kGramIPT], bj[kGramIPT];
  bool on[kGramIPT];
#pragma unroll
  for (int t = 0; t < kGramIPT; ++t) {
    const int it = item0 + item_base + t * kThreads;
    on[t] = active && (item_base + t * kThreads) < nitems_pass && it < nitems;
    const int itc = on[t] ? it : 0;
    gi[t] = itc / nsub;
    bi[t] = (itc % nsub) / nsb;
    bj[t] = (itc % nsub) % nsb;
  }
  double dacc[kGramIPT][16];
#pragma unroll
  for (int t = 0; t < kGramIPT; ++t)
#pragma unroll
    for (int e = 0; e < 16; ++e) dacc[t][e] = 0.0;
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  const bool has_b = ngram > 1;
  // double-buffered tiles: the cp.async copy of tile k+1 overlaps the FMAs on tile k
  const int tile_f = kGramTile * ldr;
  auto stage = [&](int64_t rb, int buf) {
    const int nr = (int)min((int64_t)kGramTile, r1 - rb);
    const int nv = nr * ldr / 4;
    float4* da = reinterpret_cast<float4*>(sa + buf * 2 * tile_f);
    float4* db = reinterpret_cast<float4*>(sa + buf * 2 * tile_f + tile_f);
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
      cp_async16(da + i, reinterpret_cast<const float4*>(A + rb * ldr) + i);
      if (has_b) cp_async16(db + i, reinterpret_cast<const float4*>(B + rb * ldr) + i);
    }
  };
  if (r0 < r1) stage(r0, 0);
  cp_async_commit();
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += kGramTile, buf ^= 1) {
    const int nr = (int)min((int64_t)kGramTile, r1 - rb);
    if (rb + kGramTile < r1) stage(rb + kGramTile, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const float* ta = sa + buf * 2 * tile_f;
    const float* tb = ta + tile_f;
#pragma unroll
    for (int t = 0; t < kGramIPT; ++t) {
      if (!on[t]) continue;
      float acc[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) acc[e] = 0.f;
      const float* lhs = gi[t] == 0 ? ta : tb;
      for (int r = rg; r < nr; r += nrg) {
        const float4 l = reinterpret_cast<const float4*>(lhs + r * ldr)[bi[t]];
        const float4 a = reinterpret_cast<const float4*>(ta + r * ldr)[bj[t]];
        const float lv[4] = {l.x, l.y, l.z, l.w};
        const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[ii * 4 + jj] += lv[ii] * av[jj];
      }
#pragma unroll
      for (int e = 0; e < 16; ++e) dacc[t][e] += (double)acc[e];
    }
    __syncthreads();  // this buffer is refilled by the next iteration's stage
  }
  // reduce row groups in fixed order through shared memory
  __syncthreads();
  double* red = reinterpret_cast<double*>(gsm);
  const int LL = ldr * ldr;
#pragma unroll
  for (int t = 0; t < kGramIPT; ++t) {
    if (nrg > 1 && on[t]) {
#pragma unroll
      for (int e = 0; e < 16; ++e) red[(rg * nitems_pass + item_base) * 16 + e] = dacc[t][e];
    }
  }
  if (nrg > 1) __syncthreads();
#pragma unroll
  for (int t = 0; t < kGramIPT; ++t) {
    if (!on[t] || rg != 0) continue;
    double v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = dacc[t][e];
    for (int g2 = 1; g2 < nrg; ++g2)
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] += red[(g2 * nitems_pass + item_base) * 16 + e];
    double* out = partials + ((int64_t)blockIdx.x * ngram + gi[t]) * LL;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii)
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) out[(bi[t] * 4 + ii) * ldr + bj[t] * 4 + jj] = v[ii * 4 + jj];
  }
}

// ---- K4 on tensor cores for ldr 64 / 128 (the Grams are
// [R x rows] x [rows x R] products with arithmetic intensity growing with R).
// mma.sync m16n8k8 TF32 with the 3-term split x = hi + lo (hi = tf32(x),
// lo = tf32(x - hi)): hi*hi + hi*lo + lo*hi keeps fp32-level accuracy.  Warp w
// owns one 16-row block of the output (i) and JPW 8-column blocks (j); row tiles
// of A (and B = A_old) are double-buffered in padded shared memory (stride
// LDR + 8: conflict-free fragment loads).  fp32 accumulation over a CTA's rows,
// fp64 across CTAs (k_gram_finalize, fixed order).
__device__ __forceinline__ uint32_t tf32_of(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

constexpr int kGramTcRows = 32;
// rows per staged tile: ldr 32 rows are short, so a longer tile (and two CTAs
// per SM, see gram2_enqueue) keeps enough bytes in flight per SM
__host__ __device__ constexpr int gram_tc_rows(int ldr) { return ldr == 32 ? 128 : kGramTcRows; }
template <int LDR>
__global__ void __launch_bounds__(kThreads, 1) k_gram_tc(const float* __restrict__ A, const float* __restrict__ B,
                                                         int64_t rows, int64_t rows_per_block, int ngram,
                                                         double* __restrict__ partials) {
  constexpr int TR = gram_tc_rows(LDR);
  constexpr int LDP = LDR + 8;
  constexpr int IB = LDR / 16, JB = LDR / 8;
  constexpr int WPI = 8 / IB;        // warps per i-block
  constexpr int JPW = JB / WPI;      // j-blocks per warp
  constexpr int TILE = TR * LDP;
  extern __shared__ __align__(16) float gts[];  // [2 buffers][A tile, B tile]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int i0 = (w / WPI) * 16;
  const int jb0 = (w % WPI) * JPW;
  const bool has_b = ngram > 1;
  float acc[2][JPW][4];
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int j = 0; j < JPW; ++j) acc[g][j][0] = acc[g][j][1] = acc[g][j][2] = acc[g][j][3] = 0.f;
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  auto stage = [&](int64_t rb, int buf) {
    float* da = gts + buf * 2 * TILE;
    float* db = da + TILE;
    for (int e = threadIdx.x; e < TR * (LDR / 4); e += blockDim.x) {
      const int rr = e / (LDR / 4), c4 = e % (LDR / 4);
      const int64_t row = rb + rr;
      float* pa = da + rr * LDP + c4 * 4;
      float* pb = db + rr * LDP + c4 * 4;
      if (row < r1) {
        cp_async16(pa, A + row * LDR + c4 * 4);
        if (has_b) cp_async16(pb, B + row * LDR + c4 * 4);
      } else {
        *reinterpret_cast<float4*>(pa) = make_float4(0.f, 0.f, 0.f, 0.f);
        if (has_b) *reinterpret_cast<float4*>(pb) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  if (r0 < r1) stage(r0, 0);
  cp_async_commit();
  int buf = 0;
  for (int64_t rb = r0; rb < r1; rb += TR, buf ^= 1) {
    if (rb + TR < r1) stage(rb + TR, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const float* ta = gts + buf * 2 * TILE;
    const float* tb = ta + TILE;
#pragma unroll
    for (int k0 = 0; k0 < TR; k0 += 8) {
      // operand "A" of the MMA: L^T (16 x 8) from L = A (P) or B (C); operand "B": A (8 x 8)
      uint32_t ah[2][4], al[2][4];
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        if (g == 1 && !has_b) break;
        const float* L = g == 0 ? ta : tb;
        const float x[4] = {L[(k0 + tig) * LDP + i0 + gid], L[(k0 + tig) * LDP + i0 + gid + 8],
                            L[(k0 + tig + 4) * LDP + i0 + gid], L[(k0 + tig + 4) * LDP + i0 + gid + 8]};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ah[g][q] = tf32_of(x[q]);
          al[g][q] = tf32_of(x[q] - __uint_as_float(ah[g][q]));
        }
      }
#pragma unroll
      for (int jj = 0; jj < JPW; ++jj) {
        const int j0 = (jb0 + jj) * 8;
        const float y0 = ta[(k0 + tig) * LDP + j0 + gid], y1 = ta[(k0 + tig + 4) * LDP + j0 + gid];
        const uint32_t bh[2] = {tf32_of(y0), tf32_of(y1)};
        const uint32_t bl[2] = {tf32_of(y0 - __uint_as_float(bh[0])), tf32_of(y1 - __uint_as_float(bh[1]))};
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          if (g == 1 && !has_b) break;
          mma_tf32(acc[g][jj], al[g], bh);
          mma_tf32(acc[g][jj], ah[g], bl);
          mma_tf32(acc[g][jj], ah[g], bh);
        }
      }
    }
    __syncthreads();  // this buffer is refilled by the next iteration's stage
  }
  const int LL = LDR * LDR;
#pragma unroll
  for (int g = 0; g < 2; ++g) {
    if (g >= ngram) break;
    double* out = partials + ((int64_t)blockIdx.x * ngram + g) * LL;
#pragma unroll
    for (int jj = 0; jj < JPW; ++jj) {
      const int j = (jb0 + jj) * 8 + 2 * tig;
      out[(i0 + gid) * LDR + j] = acc[g][jj][0];
      out[(i0 + gid) * LDR + j + 1] = acc[g][jj][1];
      out[(i0 + gid + 8) * LDR + j] = acc[g][jj][2];
      out[(i0 + gid + 8) * LDR + j + 1] = acc[g][jj][3];
    }
  }
}

// Grams of every mode of a small model in one launch (blockIdx.y = mode), fp64
// sums straight into the outputs: out1_k = B1_k' A_k, out2_k = B2_k' A_k (B2 nullable).
// Rows are staged through shared memory 64 at a time (coalesced), and every
// thread keeps two independent fp64 partial sums per entry, so the loop runs on
// shared-memory latency instead of a dependent global load per row (c2: 41 us ->
// a few us per launch; the Grams were the longest kernel of a c2 iteration).
constexpr int kGramSmallRows = 64;
__device__ __forceinline__ void hist_coeffs_body(int ndim, int rank, const double* P, const double* C,
                                                 const double* S, double w, const double* s, double extra, float* Mk,
                                                 float* Nk) {
  const int RR = rank * rank;
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    const double se = S ? w * S[e] : 0.0;
    const double me = se + (s ? extra * s[e / rank] * s[e % rank] : 0.0);
    for (int k = 0; k < ndim; ++k) {
      double gp = 1.0, gc = 1.0;
      for (int m = 0; m < ndim; ++m) {
        if (m == k) continue;
        gp *= P[(int64_t)m * RR + e];
        if (C) gc *= C[(int64_t)m * RR + e];
      }
      Mk[(int64_t)k * RR + e] = (float)(gp * me);
      Nk[(int64_t)k * RR + e] = C ? (float)(gc * se) : 0.f;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_gram_small(SmallGrams g, int rank, int ldr, double* __restrict__ out1,
                                                         double* __restrict__ out2, CoeffTail tail) {
  __shared__ float sA[kGramSmallRows * 32], sB1[kGramSmallRows * 32], sB2[kGramSmallRows * 32];
  const int k = blockIdx.y;
  const int RR = rank * rank;
  const float* A = g.A[k];
  const float* B1 = g.B1[k];
  const float* B2 = g.B2[k];
  const int64_t rows = g.rows[k];
  // ldr <= 32 on this path (small models); entries e = threadIdx.x + kThreads * t
  constexpr int kMaxPer = (32 * 32 + kThreads - 1) / kThreads;
  double s1[kMaxPer][2], s2[kMaxPer][2];
#pragma unroll
  for (int t = 0; t < kMaxPer; ++t) s1[t][0] = s1[t][1] = s2[t][0] = s2[t][1] = 0.0;
  for (int64_t r0 = 0; r0 < rows; r0 += kGramSmallRows) {
    const int nr = (int)min((int64_t)kGramSmallRows, rows - r0);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * ldr; e += blockDim.x) {
      sA[e] = A[r0 * ldr + e];
      sB1[e] = B1[r0 * ldr + e];
      if (B2) sB2[e] = B2[r0 * ldr + e];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < kMaxPer; ++t) {
      const int e = threadIdx.x + kThreads * t;
      if (e >= RR) continue;
      const int i = e / rank, j = e % rank;
      int r = 0;
      for (; r + 1 < nr; r += 2) {
        const double a0 = sA[r * ldr + j], a1 = sA[(r + 1) * ldr + j];
        s1[t][0] += (double)sB1[r * ldr + i] * a0;
        s1[t][1] += (double)sB1[(r + 1) * ldr + i] * a1;
        if (B2) {
          s2[t][0] += (double)sB2[r * ldr + i] * a0;
          s2[t][1] += (double)sB2[(r + 1) * ldr + i] * a1;
        }
      }
      if (r < nr) {
        const double a0 = sA[r * ldr + j];
        s1[t][0] += (double)sB1[r * ldr + i] * a0;
        if (B2) s2[t][0] += (double)sB2[r * ldr + i] * a0;
      }
    }
  }
#pragma unroll
  for (int t = 0; t < kMaxPer; ++t) {
    const int e = threadIdx.x + kThreads * t;
    if (e >= RR) continue;
    out1[(int64_t)k * RR + e] = s1[t][0] + s1[t][1];
    if (B2) out2[(int64_t)k * RR + e] = s2[t][0] + s2[t][1];
  }
  if (tail.ticket) {  // the last mode-block also computes every mode's history coefficients
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(tail.ticket, 1u) == gridDim.y - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    hist_coeffs_body(gridDim.y, rank, out1, out2, tail.S, tail.w, tail.s, tail.extra, tail.Mk, tail.Nk);
    if (threadIdx.x == 0) *tail.ticket = 0u;
  }
}

// Small models with ndim x R^2 <= 1024 whose rows fit in shared memory: every
// mode's Grams in ONE block of 1024 threads.  All modes' rows are staged in one
// coalesced pass (a single dependent round trip to L2), thread = (mode, row
// group, entry) sums its interleaved row group from shared memory, the groups
// combine in fixed order, and the history coefficients follow from the
// shared-memory Grams after a block barrier -- no cross-block ticket or
// grid-wide fence.
constexpr int kGramOneThreads = 1024;
constexpr size_t kGramOneRowSmem = 160 * 1024;  // staged rows (floats) at most
__global__ void __launch_bounds__(kGramOneThreads) k_gram_small_one(SmallGrams g, int ndim, int rank, int ldr,
                                                                    double* __restrict__ out1,
                                                                    double* __restrict__ out2, CoeffTail tail) {
  extern __shared__ float rs[];  // per mode: A [rows x ldr], B1, B2 (if any)
  __shared__ double red1[kGramOneThreads], red2[kGramOneThreads];
  __shared__ double P[kGramOneThreads], C[kGramOneThreads];
  const int RR = rank * rank;
  const int groups = max(1, min(kGramOneThreads / (ndim * RR), 64));
  const int t = threadIdx.x;
  const bool B2 = g.B2[0] != nullptr;
  const int nmat = B2 ? 3 : 2;
  int64_t off[kMaxModes];
  int64_t o = 0;
  for (int k = 0; k < ndim; ++k) {
    off[k] = o;
    const int64_t n = g.rows[k] * ldr;
    for (int64_t x = t; x < n; x += blockDim.x) {
      rs[o + x] = __ldg(g.A[k] + x);
      rs[o + n + x] = __ldg(g.B1[k] + x);
      if (B2) rs[o + 2 * n + x] = __ldg(g.B2[k] + x);
    }
    o += nmat * n;
  }
  __syncthreads();
  const int e = t % RR, kg = t / RR, k = kg / groups, grp = kg % groups;
  const int i = e / rank, j = e % rank;
  double s1 = 0.0, s2 = 0.0;
  if (k < ndim) {
    const int64_t rows = g.rows[k], n = rows * ldr;
    const float* A = rs + off[k];
    const float* B1 = A + n;
    const float* Bo = A + 2 * n;
    for (int64_t r = grp; r < rows; r += groups) {
      const double a = A[r * ldr + j];
      s1 += (double)B1[r * ldr + i] * a;
      if (B2) s2 += (double)Bo[r * ldr + i] * a;
    }
  }
  red1[t] = s1;
  red2[t] = s2;
  __syncthreads();
  if (t < ndim * RR) {
    const int kk = t / RR, ee = t % RR;
    double a1 = 0.0, a2 = 0.0;
    for (int q = 0; q < groups; ++q) {
      a1 += red1[(kk * groups + q) * RR + ee];
      a2 += red2[(kk * groups + q) * RR + ee];
    }
    P[t] = a1;
    C[t] = a2;
    out1[t] = a1;
    if (B2) out2[t] = a2;
  }
  if (tail.ticket) {  // every mode's history coefficients (k_hist_coeffs' arithmetic)
    __syncthreads();
    hist_coeffs_body(ndim, rank, P, B2 ? C : nullptr, tail.S, tail.w, tail.s, tail.extra, tail.Mk, tail.Nk);
  }
}

void gram_small_enqueue(Ctx* ctx, const SmallGrams& g, int ndim, int rank, int ldr, double* out1, double* out2,
                        const CoeffTail* tail) {
  ProfScope prof_scope(ctx, kProfGram);
  CoeffTail t{};
  if (tail) t = *tail;
  size_t rows_bytes = 0;
  for (int k = 0; k < ndim; ++k) rows_bytes += (size_t)g.rows[k] * ldr * 4 * (g.B2[0] ? 3 : 2);
  if (ndim * rank * rank <= kGramOneThreads && rows_bytes <= kGramOneRowSmem) {
    static thread_local bool attr = false;  // static 32 KB + staged rows may pass 48 KB in total
    if (!attr) {
      OGCP_CUDA(cudaFuncSetAttribute(k_gram_small_one, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kGramOneRowSmem));
      attr = true;
    }
    k_gram_small_one<<<1, kGramOneThreads, rows_bytes, ctx->stream>>>(g, ndim, rank, ldr, out1, out2, t);
  } else {
    k_gram_small<<<dim3(1, ndim), kThreads, 0, ctx->stream>>>(g, rank, ldr, out1, out2, t);
  }
  ctx->count();
  check_launch();
}

// Sum block partials (fixed order) and extract the rank x rank blocks.
template <typename T>
__global__ void __launch_bounds__(256) k_gram_finalize(const T* __restrict__ partials, int nblk, int ngram, int ldr,
                                                       int rank, double* __restrict__ outP,
                                                       double* __restrict__ outC) {
  // 32 entries x 8 fixed-order segments per block (seg_colsum)
  __shared__ double seg[kColSumSegs][32];
  const int LL = ldr * ldr;
  const int lane = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const bool live = e < ngram * rank * rank;
  const int g = live ? e / (rank * rank) : 0;
  const int ij = live ? e % (rank * rank) : 0;
  const int i = ij / rank, j = ij % rank;
  seg[sg][lane] = live ? seg_colsum(partials, nblk, (int64_t)ngram * LL, (int64_t)g * LL + i * ldr + j, sg) : 0.0;
  __syncthreads();
  if (sg == 0 && live) {
    double t = 0.0;
    for (int k = 0; k < kColSumSegs; ++k) t += seg[k][lane];
    (g == 0 ? outP : outC)[ij] = t;
  }
}

// ------------------------------------------------------------------ history coefficients
// Mk = Gamma_k o (w S + extra s s'), Nk = Gamma^_k o (w S): the history term
// (solvers.py:159-179) plus, for the dense-Gaussian gradient, its model term
// 2 A_k (Gamma_k o s s') (kernels.py:117-132).  C / S / s may be null.
__global__ void k_hist_coeffs(int ndim, int rank, const double* __restrict__ P, const double* __restrict__ C,
                              const double* __restrict__ S, double w, const double* __restrict__ s, double extra,
                              float* __restrict__ Mk, float* __restrict__ Nk) {
  hist_coeffs_body(ndim, rank, P, C, S, w, s, extra, Mk, Nk);
}

// Dense-Gaussian weight gradient without the mu term (solvers.py:182-185):
// out[r] = 2 ((hadamard_m P_m) s - b)[r]; weight_step adds mu s.
__global__ void k_dense_wgrad(int ndim, int rank, int ldr, const double* __restrict__ P,
                              const double* __restrict__ b, const double* __restrict__ s, double* __restrict__ out) {
  const int r = threadIdx.x;
  if (r >= ldr) return;
  if (r >= rank) {
    out[r] = 0.0;
    return;
  }
  const int RR = rank * rank;
  double acc = 0.0;
  for (int j = 0; j < rank; ++j) {
    double g = 1.0;
    for (int m = 0; m < ndim; ++m) g *= P[(int64_t)m * RR + r * rank + j];
    acc += g * s[j];
  }
  out[r] = 2.0 * (acc - b[r]);
}

// ------------------------------------------------------------------ K5
// g = G + lambda*a + (A Mk - Aold Nk)[row]; Adam in fp32 (the storage
// precision) with 1-beta passed from fp64; the clamp keeps NaN so the
// _ensure_finite semantics (solvers.py:188-194) are preserved.
__device__ __forceinline__ bool adam_elem(float* __restrict__ A, float* __restrict__ u, float* __restrict__ v,
                                          int64_t at, float a, float gval, float b1, float omb1, float b2,
                                          float omb2, float rate_i, float eps, float lower) {
  const float un = b1 * u[at] + omb1 * gval;
  const float vn = b2 * v[at] + (omb2 * gval) * gval;
  float an = a - rate_i * un / (sqrtf(vn) + eps);
  if (an < lower) an = lower;
  u[at] = un;
  v[at] = vn;
  A[at] = an;
  return isfinite(an);
}

// Adam update of one element from values already in registers (u, v loaded
// with the row); same arithmetic as adam_elem.
__device__ __forceinline__ bool adam_regs(float* __restrict__ A, float* __restrict__ u, float* __restrict__ v,
                                          int64_t at, float a, float gval, float uo, float vo, float b1, float omb1,
                                          float b2, float omb2, float rate_i, float eps, float lower) {
  const float un = b1 * uo + omb1 * gval;
  const float vn = b2 * vo + (omb2 * gval) * gval;
  float an = a - rate_i * un / (sqrtf(vn) + eps);
  if (an < lower) an = lower;
  u[at] = un;
  v[at] = vn;
  A[at] = an;
  return isfinite(an);
}

// rank <= 32: one group of GR lanes per row, lane c owns column c; Mk and Nk
// are staged in shared memory (lane c reads column c, conflict-free) and rows
// of A / Aold reach the group through a per-warp shared-memory stage read as
// float4 broadcasts (GR < 4: shuffles).  RPI rows per group
// per pass with all five row streams (A, Aold, G, u, v) issued before any use:
// one memory round trip per pass, and the small register footprint keeps
// enough CTAs resident to cover the HBM latency.
// K5 tuning (c4, measured): 4 rows per group pass, history loop unrolled by 8,
// >= 3 CTAs per SM (80 registers, no spills): 0.27 -> 0.21 ms per launch;
// float4 broadcasts from the row stage instead of 2 GR shuffles per row: the
// c4 average per launch 0.275 -> 0.189 ms (the shuffle form was MIO-bound).
constexpr int kK5Rows = 4;
constexpr int kK5Unroll = 8;
template <int GR>
__device__ __forceinline__ void factor_update_rows(int64_t rows, int rank, int ldr, float* __restrict__ A,
                                                   const float* __restrict__ Aold, const float* __restrict__ G,
                                                   float* __restrict__ u, float* __restrict__ v,
                                                   const float* __restrict__ Mk, const float* __restrict__ Nk,
                                                   float reg, float rate_i, float b1, float omb1, float b2,
                                                   float omb2, float eps, float lower, DevFlags* flags,
                                                   long long code) {
  constexpr int RPI = kK5Rows;
  const bool hist = Mk != nullptr;
  const bool has_old = hist && Aold != nullptr;  // dense-Gaussian model term without history
  const int lane = threadIdx.x & 31;
  const int c = lane & (GR - 1);
  const bool col_on = c < rank;
  __shared__ float sm_m[GR * GR], sm_n[GR * GR];
  __shared__ __align__(16) float sm_rows[(kThreads / 32) * 2 * RPI * 32];
  if (hist) {
    for (int e = threadIdx.x; e < GR * GR; e += blockDim.x) {
      const int r = e / GR, cc = e % GR;
      const bool in = r < rank && cc < rank;
      sm_m[e] = in ? Mk[r * rank + cc] : 0.f;
      sm_n[e] = (in && has_old) ? Nk[r * rank + cc] : 0.f;
    }
  }
  __syncthreads();
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GR;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / GR;
  bool bad = false;
  const int64_t span = ngrp * RPI;
  const int64_t rows_pad = ((rows + span - 1) / span) * span;
  for (int64_t i0 = grp * RPI; i0 < rows_pad; i0 += span) {
    float a[RPI], ao[RPI], gv[RPI], uo[RPI], vo[RPI];
    bool ok[RPI];
#pragma unroll
    for (int q = 0; q < RPI; ++q) {
      const int64_t i = i0 + q;
      ok[q] = i < rows && col_on;
      const int64_t at = i * ldr + c;
      a[q] = ok[q] ? A[at] : 0.f;
      ao[q] = (ok[q] && has_old) ? __ldg(Aold + at) : 0.f;
      gv[q] = ok[q] ? __ldg(G + at) : 0.f;
      uo[q] = ok[q] ? u[at] : 0.f;
      vo[q] = ok[q] ? v[at] : 0.f;
    }
    if (hist && GR >= 4) {
      // rows staged per warp in shared memory, read back as float4 broadcasts:
      // 2 GR / 4 LDS.128 per row instead of 2 GR shuffles (K5 was MIO-bound)
      const int w = threadIdx.x >> 5;
      const int gb = lane & ~(GR - 1);  // first lane of this row group
      float* sa = sm_rows + (size_t)w * (2 * RPI * 32);
      float* so = sa + RPI * 32;
#pragma unroll
      for (int q = 0; q < RPI; ++q) {
        sa[q * 32 + lane] = a[q];
        if (has_old) so[q * 32 + lane] = ao[q];
      }
      __syncwarp();
      float h[RPI];
#pragma unroll
      for (int q = 0; q < RPI; ++q) h[q] = 0.f;
#pragma unroll 2
      for (int r4 = 0; r4 < GR / 4; ++r4) {
        float mr[4], nr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mr[j] = sm_m[(4 * r4 + j) * GR + c];
          nr[j] = sm_n[(4 * r4 + j) * GR + c];
        }
#pragma unroll
        for (int q = 0; q < RPI; ++q) {
          const float4 av = *reinterpret_cast<const float4*>(sa + q * 32 + gb + 4 * r4);
          h[q] += av.x * mr[0] + av.y * mr[1] + av.z * mr[2] + av.w * mr[3];
          if (has_old) {
            const float4 ov = *reinterpret_cast<const float4*>(so + q * 32 + gb + 4 * r4);
            h[q] -= ov.x * nr[0] + ov.y * nr[1] + ov.z * nr[2] + ov.w * nr[3];
          }
        }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < RPI; ++q) gv[q] += h[q];
    } else if (hist) {
      float h[RPI];
#pragma unroll
      for (int q = 0; q < RPI; ++q) h[q] = 0.f;
#pragma unroll kK5Unroll
      for (int r = 0; r < GR; ++r) {
        const float mr = sm_m[r * GR + c];
        const float nr = sm_n[r * GR + c];
#pragma unroll
        for (int q = 0; q < RPI; ++q) {
          const float ar = __shfl_sync(kFull, a[q], r, GR);
          h[q] += ar * mr;
          if (has_old) {
            const float aor = __shfl_sync(kFull, ao[q], r, GR);
            h[q] -= aor * nr;
          }
        }
      }
#pragma unroll
      for (int q = 0; q < RPI; ++q) gv[q] += h[q];
    }
#pragma unroll
    for (int q = 0; q < RPI; ++q)
      if (ok[q] && !adam_regs(A, u, v, (i0 + q) * ldr + c, a[q], gv[q] + reg * a[q], uo[q], vo[q], b1, omb1, b2,
                              omb2, rate_i, eps, lower))
        bad = true;
  }
  if (bad) report(flags, kFlagDiverge, code, 0);
}

template <int GR>
__global__ void __launch_bounds__(kThreads, 3) k_factor_update(int64_t rows, int rank, int ldr, float* __restrict__ A,
                                                            const float* __restrict__ Aold,
                                                            const float* __restrict__ G, float* __restrict__ u,
                                                            float* __restrict__ v, const float* __restrict__ Mk,
                                                            const float* __restrict__ Nk, float reg, float rate_i,
                                                            float b1, float omb1, float b2, float omb2, float eps,
                                                            float lower, DevFlags* flags, long long code) {
  factor_update_rows<GR>(rows, rank, ldr, A, Aold, G, u, v, Mk, Nk, reg, rate_i, b1, omb1, b2, omb2, eps, lower,
                         flags, code);
}

// Every mode of a small model in one launch (blockIdx.y = mode): the c1/c2
// shapes are launch-bound, one K5 launch per mode cost more than the update.
template <int GR>
__global__ void __launch_bounds__(kThreads, 3) k_factor_update_modes(K5Modes m, int rank, int ldr, float reg,
                                                                  float rate_i, float b1, float omb1, float b2,
                                                                  float omb2, float eps, float lower,
                                                                  DevFlags* flags, long long code) {
  const int k = blockIdx.y;
  factor_update_rows<GR>(m.rows[k], rank, ldr, m.A[k], m.Aold[k], m.G[k], m.u[k], m.v[k], m.Mk[k], m.Nk[k], reg,
                         rate_i, b1, omb1, b2, omb2, eps, lower, flags, code);
}

// 32 < rank <= 128 with history / model terms: the apply H = A Mk - Aold Nk is
// an [rows x R] x [R x R] product, so it is register-tiled: a CTA stages Mk, Nk
// (R x R) once and a 32-row tile of A / Aold per pass in shared memory; thread
// (warp w, lane l) owns rows 4w..4w+3 and columns CPT*l..CPT*l+CPT-1 (CPT = LDR/32),
// reading A / Aold rows as broadcasts and Mk / Nk rows as contiguous vectors,
// then applies reg + Adam to its 4 x CPT elements (coalesced row segments).
constexpr int kK5TileRows = 32;
template <int LDR>
__global__ void __launch_bounds__(kThreads) k_factor_update_tiled(int64_t rows, int rank, float* __restrict__ A,
                                                                  const float* __restrict__ Aold,
                                                                  const float* __restrict__ G, float* __restrict__ u,
                                                                  float* __restrict__ v, const float* __restrict__ Mk,
                                                                  const float* __restrict__ Nk, float reg,
                                                                  float rate_i, float b1, float omb1, float b2,
                                                                  float omb2, float eps, float lower, DevFlags* flags,
                                                                  long long code) {
  constexpr int CPT = LDR / 32;
  constexpr int TR = kK5TileRows;
  extern __shared__ __align__(16) float k5s[];
  float* sm = k5s;                 // [LDR][LDR] Mk (zero padded)
  float* sn = sm + LDR * LDR;      // [LDR][LDR] Nk
  float* tiles = sn + LDR * LDR;   // 2 buffers x {A tile, Aold tile} [TR][LDR]
  const bool has_old = Aold != nullptr;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c0 = lane * CPT;
  const int64_t ntiles = (rows + TR - 1) / TR;
  // rows of tile t into buffer b by cp.async (A and Aold); rows past the end are zeroed
  auto stage = [&](int64_t tile, int b) {
    float* ta = tiles + b * 2 * TR * LDR;
    float* to = ta + TR * LDR;
    const int64_t r0 = tile * TR;
    for (int e = threadIdx.x; e < TR * LDR / 4; e += blockDim.x) {
      const int rr = e / (LDR / 4);
      const int64_t at = (r0 + rr) * LDR + (e % (LDR / 4)) * 4;
      if (r0 + rr < rows) {
        cp_async16(ta + e * 4, A + at);
        if (has_old) cp_async16(to + e * 4, Aold + at);
        else reinterpret_cast<float4*>(to)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        reinterpret_cast<float4*>(ta)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        reinterpret_cast<float4*>(to)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  if (blockIdx.x < ntiles) stage(blockIdx.x, 0);
  cp_async_commit();
  for (int e = threadIdx.x; e < LDR * LDR; e += blockDim.x) {
    const int r = e / LDR, c = e % LDR;
    const bool in = r < rank && c < rank;
    sm[e] = in ? Mk[r * rank + c] : 0.f;
    sn[e] = (in && has_old) ? Nk[r * rank + c] : 0.f;
  }
  bool bad = false;
  int buf = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, buf ^= 1) {
    const int64_t r0 = tile * TR;
    if (tile + gridDim.x < ntiles) stage(tile + gridDim.x, buf ^ 1);
    cp_async_commit();
    // this thread's G / u / v elements, fetched while the tile lands and the product runs
    float gq[4][CPT], uq[4][CPT], vq[4][CPT];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = r0 + w * 4 + i;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const bool ok = row < rows && c0 + j < rank;
        const int64_t at = row * LDR + c0 + j;
        gq[i][j] = ok ? __ldg(G + at) : 0.f;
        uq[i][j] = ok ? u[at] : 0.f;
        vq[i][j] = ok ? v[at] : 0.f;
      }
    }
    cp_async_wait<1>();
    __syncthreads();  // tile `buf` (and Mk / Nk on the first pass) visible to all
    const float* sa = tiles + buf * 2 * TR * LDR;
    const float* so = sa + TR * LDR;
    float h[4][CPT];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < CPT; ++j) h[i][j] = 0.f;
#pragma unroll 4
    for (int k = 0; k < LDR; ++k) {
      float mr[CPT], nr[CPT];
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        mr[j] = sm[k * LDR + c0 + j];
        nr[j] = sn[k * LDR + c0 + j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float a = sa[(w * 4 + i) * LDR + k];
        const float ao = so[(w * 4 + i) * LDR + k];
#pragma unroll
        for (int j = 0; j < CPT; ++j) h[i][j] += a * mr[j] - ao * nr[j];
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = r0 + w * 4 + i;
      if (row >= rows) continue;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int c = c0 + j;
        if (c >= rank) continue;
        const float a = sa[(w * 4 + i) * LDR + c];
        const float g = gq[i][j] + reg * a + h[i][j];
        if (!adam_regs(A, u, v, row * LDR + c, a, g, uq[i][j], vq[i][j], b1, omb1, b2, omb2, rate_i, eps, lower))
          bad = true;
      }
    }
    __syncthreads();  // buffer `buf` is restaged two tiles later
  }
  if (bad) report(flags, kFlagDiverge, code, 0);
}

// rank > 32: one warp per row, CPL columns per lane, Mk / Nk in shared memory.
template <int CPL>
__global__ void __launch_bounds__(kThreads) k_factor_update_wide(int64_t rows, int rank, int ldr,
                                                                 float* __restrict__ A,
                                                                 const float* __restrict__ Aold,
                                                                 const float* __restrict__ G, float* __restrict__ u,
                                                                 float* __restrict__ v, const float* __restrict__ Mk,
                                                                 const float* __restrict__ Nk, float reg,
                                                                 float rate_i, float b1, float omb1, float b2,
                                                                 float omb2, float eps, float lower, DevFlags* flags,
                                                                 long long code, int stage) {
  extern __shared__ float sm[];
  const bool hist = Mk != nullptr;
  const bool has_old = hist && Aold != nullptr;
  const int RR = rank * rank;
  if (hist && stage) {  // Mk / Nk staged in shared memory when they fit, else read through L1/L2
    for (int i = threadIdx.x; i < RR; i += blockDim.x) {
      sm[i] = Mk[i];
      sm[RR + i] = Nk[i];
    }
  }
  __syncthreads();
  const float* mm = stage ? sm : Mk;
  const float* nn = stage ? sm + RR : Nk;
  const int lane = threadIdx.x & 31;
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / 32;
  bool bad = false;
  const int64_t rows_pad = ((rows + ngrp - 1) / ngrp) * ngrp;
  for (int64_t i = grp; i < rows_pad; i += ngrp) {
    const bool valid = i < rows;
    float a[CPL], ao[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int cc = lane + j * 32;
      a[j] = (cc < rank && valid) ? A[i * ldr + cc] : 0.f;
      ao[j] = (has_old && cc < rank && valid) ? Aold[i * ldr + cc] : 0.f;
    }
    float h[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) h[j] = 0.f;
    if (hist) {
#pragma unroll
      for (int jj = 0; jj < CPL; ++jj) {
        for (int src = 0; src < 32; ++src) {
          const int r = jj * 32 + src;
          const float ar = __shfl_sync(kFull, a[jj], src);
          const float aor = __shfl_sync(kFull, ao[jj], src);
          if (r < rank) {
#pragma unroll
            for (int j = 0; j < CPL; ++j) {
              const int cc = lane + j * 32;
              if (cc < rank) h[j] += ar * mm[r * rank + cc] - aor * nn[r * rank + cc];
            }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int cc = lane + j * 32;
      if (!valid || cc >= rank) continue;
      const int64_t at = i * ldr + cc;
      if (!adam_elem(A, u, v, at, a[j], G[at] + reg * a[j] + h[j], b1, omb1, b2, omb2, rate_i, eps, lower))
        bad = true;
    }
  }
  if (bad) report(flags, kFlagDiverge, code, 0);
}

// ------------------------------------------------------------------ weight step
// wstate layout (double): s[ldr] u[ldr] v[ldr] s_o[ldr] u_o[ldr] v_o[ldr]
__global__ void k_weight_step(const double* __restrict__ partials, int nblk, int rank, int ldr,
                              double* __restrict__ ws, float* __restrict__ s_f, double mu, double rate_i, double b1,
                              double b2, double eps, double lower, DevFlags* flags, long long code) {
  weight_step_body(partials, nblk, rank, ldr, ws, s_f, mu, rate_i, b1, b2, eps, lower, flags, code);
}

// ------------------------------------------------------------------ history penalty
// out[0] = sum_h coef_h * max(s_h' Q s_h, 0), Q = Poo - (Pon + Pon') + Pnn (all-mode Grams).
__global__ void k_hist_penalty(int ndim, int rank, const double* __restrict__ Poo, const double* __restrict__ Pon,
                               const double* __restrict__ Pnn, const double* __restrict__ Ws,
                               const double* __restrict__ coef, int H, double* __restrict__ out,
                               double* __restrict__ qglobal) {
  extern __shared__ double qs[];
  double* q = qglobal ? qglobal : qs;  // Q in shared memory when it fits (R <= 160)
  const int RR = rank * rank;
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    const int i = e / rank, j = e % rank;
    const int et = j * rank + i;
    double oo = 1.0, on = 1.0, no = 1.0, nn = 1.0;
    for (int m = 0; m < ndim; ++m) {
      oo *= Poo[(int64_t)m * RR + e];
      on *= Pon[(int64_t)m * RR + e];
      no *= Pon[(int64_t)m * RR + et];
      nn *= Pnn[(int64_t)m * RR + e];
    }
    q[e] = oo - (on + no) + nn;
  }
  __syncthreads();
  __shared__ double red[32];
  double tot = 0.0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  double wsum = 0.0;
  for (int h = w; h < H; h += nw) {
    const double* s = Ws + (int64_t)h * rank;
    double part = 0.0;
    for (int e = lane; e < RR; e += 32) part += s[e / rank] * q[e] * s[e % rank];
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(kFull, part, o);
    wsum += coef[h] * fmax(part, 0.0);
  }
  if (lane == 0) red[w] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 0; j < nw; ++j) tot += red[j];
    *out = tot;
  }
}

// ==================================================================== host side
template <int N>
using IC = std::integral_constant<int, N>;

// Lane layout per kernel kind (G lanes per sample, V float4 chunks per lane, U
// samples per group per pass), measured on B200 at R = 32 (profiles/): the
// scatter kernel prefers 8 lanes x 1 chunk (one 16-byte reduction per lane per
// mode), the reductions (weight gradient, objective) prefer 4 lanes x 2 chunks
// (half the per-sample scalar work per warp instruction).  U = 2 keeps the
// pipelined gathers below ~130 registers.
#include "walk3.cuh"
#include "walk_tma.cuh"
#include "gram_umma.cuh"

enum class Layout { Scatter, Reduce };

template <class F>
static void dispatch_layout(Layout kind, int ndim, int ldr, F&& f) {
  auto by_ldr = [&](auto Dc) {
    if (kind == Layout::Scatter) {
      switch (ldr) {
        case 4: f(Dc, IC<1>(), IC<1>(), IC<2>()); break;
        case 8: f(Dc, IC<2>(), IC<1>(), IC<2>()); break;
        case 16: f(Dc, IC<4>(), IC<1>(), IC<2>()); break;  // measured best of (4,1,2) (2,2,1) (2,2,2) on c3
        // ldr 32: 4 lanes x 2 float4 per row, 8 samples per warp instruction (halves the
        // per-sample index/address work against 8 lanes x 1 float4; c4: 9.04 -> 8.62 ms)
        case 32: f(Dc, IC<4>(), IC<2>(), IC<1>()); break;
        case 64: f(Dc, IC<16>(), IC<1>(), IC<2>()); break;
        case 128: f(Dc, IC<32>(), IC<1>(), IC<2>()); break;
        case 256: f(Dc, IC<32>(), IC<2>(), IC<1>()); break;
        default: throw Error(OGCP_E_USAGE, "unsupported padded rank " + std::to_string(ldr));
      }
    } else {
      switch (ldr) {
        case 4: f(Dc, IC<1>(), IC<1>(), IC<2>()); break;
        case 8: f(Dc, IC<2>(), IC<1>(), IC<2>()); break;
        case 16: f(Dc, IC<4>(), IC<1>(), IC<2>()); break;
        case 32: f(Dc, IC<4>(), IC<2>(), IC<2>()); break;  // measured best of (4,2,1) (2,4,1) (8,1,2) on c4
        case 64: f(Dc, IC<8>(), IC<2>(), IC<2>()); break;
        case 128: f(Dc, IC<16>(), IC<2>(), IC<2>()); break;
        case 256: f(Dc, IC<32>(), IC<2>(), IC<1>()); break;
        default: throw Error(OGCP_E_USAGE, "unsupported padded rank " + std::to_string(ldr));
      }
    }
  };
  switch (ndim) {
    case 2: by_ldr(IC<2>()); break;
    case 3: by_ldr(IC<3>()); break;
    case 4: by_ldr(IC<4>()); break;
    default: by_ldr(IC<0>()); break;
  }
}

// Opt a kernel into `smem` bytes of dynamic shared memory (> 48 KB), once per size.
template <class K>
static void allow_smem(K kern, size_t smem) {
  if (smem <= 48 * 1024) return;
  static thread_local std::unordered_map<const void*, size_t> done;
  size_t& have = done[(const void*)kern];
  if (have >= smem) return;
  OGCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  have = smem;
}

// Resident blocks per SM of a kernel at kThreads threads and `smem` dynamic bytes,
// cached per (kernel, smem): the occupancy query is a host API call, and the small
// streams (c1/c2) launch kernels every few microseconds.
template <class K>
static int occupancy(K kern, size_t smem) {
  static thread_local std::unordered_map<uint64_t, int> cache;
  const uint64_t key = (uint64_t)(uintptr_t)(const void*)kern * 1000003ull ^ (uint64_t)smem;
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  OGCP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
  cache.emplace(key, per_sm);
  return per_sm;
}

// Grid for a grid-stride sample kernel: enough blocks to cover the samples once,
// capped at the number that can be co-resident (occupancy API).
template <class K>
static int sample_grid(K kern, size_t smem, int64_t total, int G, int U) {
  const int per_sm = std::max(occupancy(kern, smem), 1);
  const int64_t per_block = (int64_t)(kThreads / G) * U;
  const int64_t need = (total + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)kNumSMs * per_sm));
}

// ------------------------------------------------------------------ K3, deterministic (small models)
// Bitwise run-to-run reproducible sampled MTTKRP for small models (every mode's
// gradient fits a per-warp shared-memory copy): block b takes a fixed contiguous
// range of the samples, warp w a fixed sub-range; a group of G lanes (one float4
// each, G = ldr / 4) evaluates one sample, and the groups of a warp add their
// contributions to the warp's private copy one group at a time (fixed order, no
// atomics).  The block sums its warps' copies in warp order into a block partial;
// the last block to finish (ticket) sums the partials in block order into G.
// Every float addition has a fixed order, so the same sample set gives the same
// bits -- the reference's same-seed bitwise trajectories (tests/test_streaming.py:
// 222-238 there) hold for these shapes.  Reference: sampled_mttkrp kernels.py:33-56.
constexpr int kDetThreads = 256;
constexpr int64_t kDetMaxFloats = 4096;  // per-warp copy: sum_k dims[k] * ldr floats (16 KB)

struct DetP {
  int64_t off[kMaxModes];  // float offset of mode k inside a gradient copy
  int64_t len;             // floats of one copy
  unsigned int* ticket;
  float* partials;         // [gridDim.x x len]
};

template <int G>
__global__ void __launch_bounds__(kDetThreads) k_sgrad_det(SamplesP S, ModelP M, const float* __restrict__ s_f,
                                                          LossP L, GradPtrs GP, DetP D, DevFlags* flags,
                                                          long long code) {
  extern __shared__ float wacc[];  // [8 warps][D.len]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / G, gl = lane % G;
  constexpr int kGroups = 32 / G;
  const int nd = M.ndim, ldr = M.ldr;
  float* mine = wacc + (int64_t)warp * D.len;
  for (int64_t e = lane; e < D.len; e += 32) mine[e] = 0.f;
  __syncwarp();
  const float4 s4 = gl * 4 < ldr ? __ldg(reinterpret_cast<const float4*>(s_f) + gl) : make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t p = S.p_dev ? (int64_t)*S.p_dev : S.p;
  const int64_t total = p + (S.q_dev ? (int64_t)*S.q_dev : S.q);
  const int64_t per_blk = (total + gridDim.x - 1) / gridDim.x;
  const int64_t blo = blockIdx.x * per_blk, bhi = min(total, blo + per_blk);
  const int64_t per_w = (bhi - blo + (kDetThreads / 32) - 1) / (kDetThreads / 32);
  const int64_t wlo = blo + warp * per_w, whi = min(bhi, wlo + per_w);
  unsigned bits = 0;
  for (int64_t base = wlo; base < whi; base += kGroups) {
    const int64_t n = base + grp;
    bool valid = n < whi;
    int idx[kMaxModes];
    float x = 0.f, scale = 0.f;
    bool nz = false;
    if (valid) {
      if (n < p) {
        nz = true;
        const int o = __ldg(S.ord + n);
        const int* r = S.rec + (int64_t)o * S.rec_ints;
        for (int k = 0; k < nd; ++k) idx[k] = __ldg(r + k);
        x = __int_as_float(__ldg(r + nd));
        scale = (float)S.nz_scale * (S.cnt ? (float)__ldg(S.cnt + n) : 1.0f);
      } else {
        const int32_t* z = S.zsub + (n - p) * nd;
        for (int k = 0; k < nd; ++k) idx[k] = __ldg(z + k);
        valid = idx[0] >= 0;  // lazy layout: a rejected candidate
        scale = (float)S.zero_scale;
      }
    }
    float4 a[kMaxModes];
    float4 pr = make_float4(1.f, 1.f, 1.f, 1.f);
    for (int k = 0; k < nd; ++k) {
      a[k] = (valid && gl * 4 < ldr) ? __ldg(reinterpret_cast<const float4*>(M.A[k] + (int64_t)idx[k] * ldr) + gl)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
      pr = mul4(pr, a[k]);
    }
    float m = dot4(pr, s4);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) m += __shfl_xor_sync(kFull, m, o);
    float y = 0.f;
    if (valid) {
      bits |= domain_bits(L.kind, m);
      y = dloss(L.kind, nz ? x : 0.f, m, L.eps);
      if (S.semi && nz) y -= dloss(L.kind, 0.0f, m, L.eps);
      y *= scale;
    }
    // groups add in fixed order
    for (int g2 = 0; g2 < kGroups; ++g2) {
      if (grp == g2 && valid && gl * 4 < ldr) {
        for (int k = 0; k < nd; ++k) {
          float4 c = make_float4(y * s4.x, y * s4.y, y * s4.z, y * s4.w);
          for (int j = 0; j < nd; ++j)
            if (j != k) c = mul4(c, a[j]);
          float* dst = mine + D.off[k] + (int64_t)idx[k] * ldr + gl * 4;
          dst[0] += c.x;
          dst[1] += c.y;
          dst[2] += c.z;
          dst[3] += c.w;
        }
      }
      __syncwarp();
    }
  }
  if (bits) report(flags, kFlagData, code, bits);
  __syncthreads();
  float* part = D.partials + (int64_t)blockIdx.x * D.len;
  for (int64_t e = threadIdx.x; e < D.len; e += blockDim.x) {
    float t = 0.f;
    for (int w = 0; w < kDetThreads / 32; ++w) t += wacc[(int64_t)w * D.len + e];
    part[e] = t;
  }
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(D.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int64_t e = threadIdx.x; e < D.len; e += blockDim.x) {
    float t = 0.f;
    for (int b = 0; b < (int)gridDim.x; ++b) t += D.partials[(int64_t)b * D.len + e];
    int k = 0;
    while (k + 1 < nd && e >= D.off[k + 1]) ++k;
    GP.g[k][e - D.off[k]] = t;
  }
  if (threadIdx.x == 0) *D.ticket = 0u;
}

// Launch the deterministic scatter when the model is small enough; false otherwise.
static bool sgrad_det_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                              const GradPtrs& GP, long long code) {
  if (!ctx->deterministic || S.shard_world > 1 || M.ldr > 32 || M.ndim > kMaxModes) return false;
  DetP D{};
  int64_t len = 0;
  for (int k = 0; k < M.ndim; ++k) {
    D.off[k] = len;
    len += M.dims[k] * M.ldr;
  }
  if (len > kDetMaxFloats) return false;
  D.len = len;
  const int64_t total = S.p + S.q;
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 64));
  D.partials = static_cast<float*>(ctx->det_partials.ensure((size_t)nblk * len * 4));
  D.ticket = ctx->wticket() + 1;  // second counter of the ticket buffer (0 between launches)
  const size_t smem = (size_t)(kDetThreads / 32) * len * 4;
  auto go = [&](auto kern) {
    allow_smem(kern, smem);
    kern<<<nblk, kDetThreads, smem, ctx->stream>>>(S, M, s_f, L, GP, D, ctx->flags.as<DevFlags>(), code);
  };
  switch (M.ldr) {
    case 4: go(k_sgrad_det<1>); break;
    case 8: go(k_sgrad_det<2>); break;
    case 16: go(k_sgrad_det<4>); break;
    default: go(k_sgrad_det<8>); break;
  }
  ctx->count();
  check_launch();
  return true;
}

// The lean 3-way walks (walk3.cuh) serve merged sets of 3-way slices at ldr 16 / 32
// (at ldr 64 the double-buffered rows exceed the register budget).
static bool lean_walk(const Ctx* ctx, const SamplesP& S, const ModelP& M) {
  return (ctx->lean_walks || ctx->tma_walks) && M.ndim == 3 && S.cnt != nullptr && S.rec_ints == 4 && !S.semi &&
         (M.ldr == 16 || M.ldr == 32) && (S.shard_world <= 1 || S.zshard);
}

template <bool ZERO>
static walk3::Walk<ZERO> walk_of(const SamplesP& S) {
  walk3::Walk<ZERO> W;
  W.pos = S.ord;
  W.cnt = S.cnt;
  W.rec = S.rec;
  W.zsub = S.zsub;
  W.n_dev = ZERO ? S.q_dev : S.p_dev;
  W.n_host = ZERO ? S.q : S.p;
  W.shard_rank = S.shard_rank;
  W.shard_world = ZERO && S.zshard == 1 ? S.shard_world : 1;
  return W;
}

// Launch a lean walk kernel over an (upper-bound) entry count; returns the grid.
template <class K, class... A>
static int lean_launch(Ctx* ctx, K kern, int64_t n_est, A... args) {
  const int per_sm = std::max(occupancy(kern, 0), 1);
  const int64_t need = (n_est + (kThreads / 32) * walk3::kChunk - 1) / ((kThreads / 32) * walk3::kChunk);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)kNumSMs * per_sm));
  kern<<<grid, kThreads, 0, ctx->stream>>>(args...);
  ctx->count();
  return grid;
}

template <int V>
static void sgrad3_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                           const GradPtrs& GP, long long code) {
  DevFlags* fl = ctx->flags.as<DevFlags>();
  if (S.p > 0)
    lean_launch(ctx, walk3::k_sgrad3<V, false>, S.p, walk_of<false>(S), M, s_f, L, (float)S.nz_scale, GP, fl, code);
  if (S.q > 0) {
    const int64_t zest = S.q_dev ? S.q + S.q / 64 + 1024 : S.q;
    lean_launch(ctx, walk3::k_sgrad3<V, true>, zest / std::max(S.zshard ? S.shard_world : 1, 1), walk_of<true>(S),
                M, s_f, L, (float)S.zero_scale, GP, fl, code);
  }
}

template <int V>
static int wgrad3_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                          double* partials, long long code) {
  DevFlags* fl = ctx->flags.as<DevFlags>();
  int nb = 0;
  if (S.p > 0)
    nb += lean_launch(ctx, walk3::k_wgrad3<V, false>, S.p, walk_of<false>(S), M, s_f, L, (float)S.nz_scale,
                      partials, fl, code);
  if (S.q > 0) {
    const int64_t zest = S.q_dev ? S.q + S.q / 64 + 1024 : S.q;
    nb += lean_launch(ctx, walk3::k_wgrad3<V, true>, zest / std::max(S.zshard ? S.shard_world : 1, 1),
                      walk_of<true>(S), M, s_f, L, (float)S.zero_scale, partials + (int64_t)nb * M.ldr, fl, code);
  }
  return std::max(nb, 1);
}

// ---- TMA-fed walks (walk_tma.cuh): tensor maps of the three factor matrices
static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    OGCP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error(OGCP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [rows x ldr] fp32 rows, box {ldr, 1}: the unit of a tile::gather4 row gather.
static CUtensorMap row_map(const float* A, int64_t rows, int ldr) {
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)ldr, (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t gstride[1] = {(cuuint64_t)ldr * 4};
  cuuint32_t box[2] = {(cuuint32_t)ldr, 1};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = tmap_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), gdim, gstride, box,
                                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(OGCP_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return tm;
}

template <int V, int MODE, bool ZERO, bool A2S>
static int tma_launch_as(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L, float scale,
                         const GradPtrs& GP, double* partials, long long code) {
  auto kern = walkt::k_walk_tma<V, MODE, ZERO, A2S>;
  using SL = walkt::StageLayout<V, A2S>;
  const int64_t a2 = A2S ? (M.dims[2] * (int64_t)SL::kRowBytes + 127) / 128 * 128 : 0;
  const int smem = (int)(SL::kSmemFixed + a2);
  static thread_local int attr = 0;
  if (smem > attr) {
    OGCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = smem;
  }
  walkt::Maps maps;
  for (int k = 0; k < 3; ++k) maps.a[k] = row_map(M.A[k], M.dims[k], M.ldr);
  kern<<<kNumSMs, walkt::kThreadsT, smem, ctx->stream>>>(maps, walk_of<ZERO>(S), M, s_f, L, scale, GP, partials,
                                                          ctx->flags.as<DevFlags>(), code);
  ctx->count();
  return kNumSMs;
}

// The mode-2 factor stays resident in shared memory when it fits (walk_tma.cuh A2S).
template <int V, int MODE, bool ZERO>
static int tma_launch(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L, float scale,
                      const GradPtrs& GP, double* partials, long long code) {
  using SL = walkt::StageLayout<V, true>;
  const int64_t a2 = M.dims[2] * (int64_t)SL::kRowBytes;
  if (ctx->tma_a2_resident && a2 <= walkt::kA2Max && SL::kSmemFixed + (a2 + 127) / 128 * 128 <= 227 * 1024)
    return tma_launch_as<V, MODE, ZERO, true>(ctx, S, M, s_f, L, scale, GP, partials, code);
  return tma_launch_as<V, MODE, ZERO, false>(ctx, S, M, s_f, L, scale, GP, partials, code);
}

template <int V>
static void sgrad_tma_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                              const GradPtrs& GP, long long code) {
  if (S.p > 0) tma_launch<V, 0, false>(ctx, S, M, s_f, L, (float)S.nz_scale, GP, nullptr, code);
  if (S.q > 0) tma_launch<V, 0, true>(ctx, S, M, s_f, L, (float)S.zero_scale, GP, nullptr, code);
}

template <int V>
static int wgrad_tma_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                             double* partials, long long code) {
  GradPtrs none{};
  int nb = 0;
  if (S.p > 0) nb += tma_launch<V, 1, false>(ctx, S, M, s_f, L, (float)S.nz_scale, none, partials, code);
  if (S.q > 0)
    nb += tma_launch<V, 1, true>(ctx, S, M, s_f, L, (float)S.zero_scale, none, partials + (int64_t)nb * M.ldr, code);
  return std::max(nb, 1);
}

void sgrad_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                   float* const* grads, long long code) {
  GradPtrs GP;
  for (int k = 0; k < kMaxModes; ++k) GP.g[k] = k < M.ndim ? grads[k] : nullptr;
  // zero the outputs: one memset when the per-mode buffers are contiguous
  bool contiguous = true;
  size_t tot_bytes = 0;
  for (int k = 0; k < M.ndim; ++k) {
    if (grads[k] != grads[0] + tot_bytes / 4) contiguous = false;
    tot_bytes += (size_t)M.dims[k] * M.ldr * 4;
  }
  if (contiguous) {
    OGCP_CUDA(cudaMemsetAsync(grads[0], 0, tot_bytes, ctx->stream));
  } else {
    for (int k = 0; k < M.ndim; ++k)
      OGCP_CUDA(cudaMemsetAsync(grads[k], 0, (size_t)M.dims[k] * M.ldr * 4, ctx->stream));
  }
  const int64_t total = S.p + S.q;
  if (total == 0) return;
  {
    ProfScope prof_scope(ctx, kProfSgrad);
    if (sgrad_det_enqueue(ctx, S, M, s_f, L, GP, code)) return;
  }
  // privatise small modes in shared memory when the per-CTA flush is cheap
  PrivP PV;
  PV.nmodes = 0;
  int64_t used = 0;
  const int64_t budget = 96 * 1024 / 4;
  for (int k = 0; k < M.ndim; ++k) {
    const int64_t len = M.dims[k] * M.ldr;
    const int64_t est_grid = std::min<int64_t>((total * (M.ldr / 4) + kThreads - 1) / kThreads, kNumSMs * 2);
    if (used + len <= budget && est_grid * len * 2 <= total * (int64_t)M.ldr) {
      PV.mode[PV.nmodes] = k;
      PV.off[PV.nmodes] = used;
      PV.len[PV.nmodes] = len;
      ++PV.nmodes;
      used += len;
    }
  }
  const size_t smem = (size_t)used * 4;
  // Split scatter for merged sets whose largest random-access gradient (a mode
  // other than the segmented mode 0) is too big to share L2 with the gathers.
  int split = -1;
  if (S.cnt && ctx->split_scatter) {
    int64_t best = 0;
    for (int k = 1; k < M.ndim; ++k) {
      bool priv = false;
      for (int j = 0; j < PV.nmodes; ++j) priv = priv || PV.mode[j] == k;
      const int64_t bytes = M.dims[k] * M.ldr * 4;
      if (!priv && bytes >= (int64_t)32 << 20 && bytes > best) {
        best = bytes;
        split = k;
      }
    }
  }
  if (PV.nmodes == 0 && split < 0 && lean_walk(ctx, S, M)) {
    ProfScope prof_scope(ctx, kProfSgrad);
    if (ctx->tma_walks) {
      if (M.ldr == 16) sgrad_tma_enqueue<1>(ctx, S, M, s_f, L, GP, code);
      else sgrad_tma_enqueue<2>(ctx, S, M, s_f, L, GP, code);
    } else if (M.ldr == 16) {
      sgrad3_enqueue<1>(ctx, S, M, s_f, L, GP, code);
    } else {
      sgrad3_enqueue<2>(ctx, S, M, s_f, L, GP, code);
    }
    check_launch();
    return;
  }
  float* ybuf = split >= 0 ? static_cast<float*>(ctx->ybuf.ensure((size_t)total * 4)) : nullptr;
  ProfScope prof_scope(ctx, kProfSgrad);
  dispatch_layout(Layout::Scatter, M.ndim, M.ldr, [&](auto Dc, auto Gc, auto Vc, auto Uc) {
    constexpr int D = decltype(Dc)::value, G = decltype(Gc)::value, V = decltype(Vc)::value;
    constexpr int U = decltype(Uc)::value;
    auto launch = [&](auto kern) {
      allow_smem(kern, smem);
      const int grid = sample_grid(kern, smem, total, G, U);
      kern<<<grid, kThreads, smem, ctx->stream>>>(S, M, s_f, L, GP, PV, ctx->flags.as<DevFlags>(), code, split,
                                                  ybuf);
    };
    if (S.cnt) launch(k_sgrad<D, G, V, U, true>);
    else launch(k_sgrad<D, G, V, U, false>);
    if (split >= 0) {
      auto kern2 = k_sgrad_split<D, G, V, U>;
      const int grid2 = sample_grid(kern2, 0, total, G, U);
      kern2<<<grid2, kThreads, 0, ctx->stream>>>(S, M, s_f, ybuf, GP.g[split], split);
      ctx->count();
    }
  });
  ctx->count();
  check_launch();
}

int wgrad_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                  double* partials, long long code, const WStep* step, bool* stepped) {
  if (stepped) *stepped = false;
  const int64_t total = S.p + S.q;
  int grid = 1;
  ProfScope prof_scope(ctx, kProfWgrad);
  if (lean_walk(ctx, S, M) && (ctx->lean_walks || ctx->tma_wgrad) && total > 0) {
    // the weight walk has no scatter; its register-fed generic kernel measured faster than
    // the TMA walk at c4 (3.3 vs 4.6 ms), so ctx->tma_walks only selects the K3 walk
    if (ctx->tma_wgrad) grid = M.ldr == 16 ? wgrad_tma_enqueue<1>(ctx, S, M, s_f, L, partials, code)
                                           : wgrad_tma_enqueue<2>(ctx, S, M, s_f, L, partials, code);
    else if (M.ldr == 16) grid = wgrad3_enqueue<1>(ctx, S, M, s_f, L, partials, code);
    else grid = wgrad3_enqueue<2>(ctx, S, M, s_f, L, partials, code);
    check_launch();
    return grid;
  }
  dispatch_layout(Layout::Reduce, M.ndim, M.ldr, [&](auto Dc, auto Gc, auto Vc, auto Uc) {
    constexpr int D = decltype(Dc)::value, G = decltype(Gc)::value, V = decltype(Vc)::value;
    constexpr int U = decltype(Uc)::value;
    auto kern = k_wgrad<D, G, V, U>;
    grid = sample_grid(kern, 0, std::max<int64_t>(total, 1), G, U);
    WStep ws{};
    if (step && step->ldr <= kThreads) {
      ws = *step;
      if (stepped) *stepped = true;
    }
    kern<<<grid, kThreads, 0, ctx->stream>>>(S, M, s_f, L, partials, ctx->flags.as<DevFlags>(), code, ws);
  });
  ctx->count();
  check_launch();
  return grid;
}

template <int MODE>
static int objective_like(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                          double* partials, long long code) {
  const int64_t total = S.p + S.q;
  int grid = 1;
  ProfScope prof_scope(ctx, kProfObjective);
  dispatch_layout(Layout::Reduce, M.ndim, M.ldr, [&](auto Dc, auto Gc, auto Vc, auto Uc) {
    constexpr int D = decltype(Dc)::value, G = decltype(Gc)::value, V = decltype(Vc)::value;
    constexpr int U = decltype(Uc)::value;
    auto kern = k_objective<D, G, V, U, MODE>;
    grid = sample_grid(kern, 0, std::max<int64_t>(total, 1), G, U);
    kern<<<grid, kThreads, 0, ctx->stream>>>(S, M, s_f, L, partials, ctx->flags.as<DevFlags>(), code);
  });
  ctx->count();
  check_launch();
  return grid;
}

int objective_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                      double* partials, long long code) {
  return objective_like<0>(ctx, S, M, s_f, L, partials, code);
}

int exact_nz_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                     double* partials, long long code) {
  return objective_like<1>(ctx, S, M, s_f, L, partials, code);
}

int exact_cells_enqueue(Ctx* ctx, const ModelP& M, const float* s_f, const LossP& L, int64_t omega,
                        double* partials, long long code) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((omega + kThreads - 1) / kThreads, kNumSMs * 4));
  k_exact_cells<<<grid, kThreads, 0, ctx->stream>>>(M, s_f, L, omega, partials, ctx->flags.as<DevFlags>(), code);
  ctx->count();
  check_launch();
  return grid;
}

void sum_partials_enqueue(Ctx* ctx, const double* partials, int nblk, int len, double* out) {
  k_sum_partials_vec<<<std::max(1, ceil_div_i(len, 32)), 256, 0, ctx->stream>>>(partials, nblk, len,
                                                                                               out);
  ctx->count();
  check_launch();
}

// [rows x ldr] fp32 in raw row tiles of {ldr, 32 rows} (the UMMA Gram's converter
// warps transpose them into its K-major operand tiles, gram_umma.cuh).
static CUtensorMap gram_tile_map(const float* A, int64_t rows, int ldr) {
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)ldr, (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t gstride[1] = {(cuuint64_t)ldr * 4};
  cuuint32_t box[2] = {(cuuint32_t)ldr, (cuuint32_t)umma::kRows};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = tmap_encoder()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(A), gdim, gstride, box,
                                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(OGCP_E_CUDA, "cuTensorMapEncodeTiled (Gram tiles) failed (" + std::to_string((int)r) + ")");
  return tm;
}

void gram2_enqueue(Ctx* ctx, const float* A, const float* B, int64_t rows, int rank, int ldr, double* outP,
                   double* outC, DevBuf& scratch) {
  const int ngram = B ? 2 : 1;
  if (ldr == 32 && ctx->umma_gram && rows > 0) {  // tcgen05 / TMEM, packed 64-row chunks (gram_umma.cuh)
    const int64_t nchunks = (rows + umma::kRows32 - 1) / umma::kRows32;
    const int nblk = (int)std::min<int64_t>(nchunks, kNumSMs);
    scratch.ensure((size_t)2 * nblk * ngram * 32 * 32 * 4);  // two sub-chunk partials per CTA
    umma::GramMaps maps;
    maps.a = gram_tile_map(A, rows, ldr);
    maps.b = B ? gram_tile_map(B, rows, ldr) : maps.a;
    static thread_local bool attr32 = false;
    if (!attr32) {
      OGCP_CUDA(cudaFuncSetAttribute(umma::k_gram_umma32, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     umma::kSmem32));
      attr32 = true;
    }
    ProfScope prof_scope(ctx, kProfGram);
    umma::k_gram_umma32<<<nblk, umma::kThreadsG, umma::kSmem32, ctx->stream>>>(maps, rows, ngram,
                                                                               scratch.as<float>());
    ctx->count();
    k_gram_finalize<float><<<std::max(1, ceil_div_i((int64_t)ngram * rank * rank, 32)), 256, 0, ctx->stream>>>(
        scratch.as<float>(), 2 * nblk, ngram, ldr, rank, outP, outC);
    ctx->count();
    check_launch();
    return;
  }
  if ((ldr == 64 || ldr == 128) && ctx->umma_gram && rows > 0) {  // tcgen05 / TMEM path (gram_umma.cuh)
    const int64_t nchunks = (rows + umma::kRows - 1) / umma::kRows;
    const int nblk = (int)std::min<int64_t>(nchunks, kNumSMs);
    scratch.ensure((size_t)nblk * ngram * ldr * ldr * 4);  // fp32 CTA partials (the TMEM accumulators)
    umma::GramMaps maps;
    maps.a = gram_tile_map(A, rows, ldr);
    maps.b = B ? gram_tile_map(B, rows, ldr) : maps.a;
    auto kern = ldr == 64 ? umma::k_gram_umma<64> : umma::k_gram_umma<128>;
    static thread_local bool attr64 = false, attr128 = false;
    bool& attr = ldr == 64 ? attr64 : attr128;
    if (!attr) {
      OGCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, umma::kSmemG));
      attr = true;
    }
    ProfScope prof_scope(ctx, kProfGram);
    kern<<<nblk, umma::kThreadsG, umma::kSmemG, ctx->stream>>>(maps, rows, ngram, scratch.as<float>());
    ctx->count();
    k_gram_finalize<float><<<std::max(1, ceil_div_i((int64_t)ngram * rank * rank, 32)), 256, 0, ctx->stream>>>(
        scratch.as<float>(), nblk, ngram, ldr, rank, outP, outC);
    ctx->count();
    check_launch();
    return;
  }
  if (ldr == 32 || ldr == 64 || ldr == 128) {  // tensor-core path (mma.sync, split-TF32)
    // ldr 32: two CTAs per SM (80 KB of tiles each) to cover the load latency
    const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64, kNumSMs * (ldr == 32 ? 2 : 1)));
    const int64_t rpb = (rows + nblk - 1) / nblk;
    scratch.ensure((size_t)nblk * ngram * ldr * ldr * 8);
    const size_t smem = (size_t)2 * 2 * gram_tc_rows(ldr) * (ldr + 8) * 4;
    auto go = [&](auto kern) {
      allow_smem(kern, smem);
      ProfScope prof_scope(ctx, kProfGram);
      kern<<<nblk, kThreads, smem, ctx->stream>>>(A, B ? B : A, rows, rpb, ngram, scratch.as<double>());
      ctx->count();
      k_gram_finalize<double><<<std::max(1, ceil_div_i((int64_t)ngram * rank * rank, 32)), 256, 0,
                        ctx->stream>>>(scratch.as<double>(), nblk, ngram, ldr, rank, outP, outC);
      ctx->count();
      check_launch();
    };
    if (ldr == 32) go(k_gram_tc<32>);
    else if (ldr == 64) go(k_gram_tc<64>);
    else go(k_gram_tc<128>);
    return;
  }
  const int nsub = (ldr / 4) * (ldr / 4);
  const int nitems = ngram * nsub;
  const int per_pass = kGramIPT * kThreads;
  int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 127) / 128, kNumSMs * 2));
  const int64_t rpb = (rows + nblk - 1) / nblk;
  nblk = (int)std::max<int64_t>(1, (rows + rpb - 1) / rpb);
  scratch.ensure((size_t)nblk * ngram * ldr * ldr * 8);
  size_t smem = (size_t)4 * kGramTile * ldr * 4;  // two buffers x (A tile, B tile)
  smem = std::max(smem, (size_t)kThreads * 16 * 8);
  allow_smem(k_gram2, smem);
  ProfScope prof_scope(ctx, kProfGram);
  for (int item0 = 0; item0 < nitems; item0 += per_pass) {
    const int n_pass = std::min(per_pass, nitems - item0);
    // for small passes each thread owns one item and row groups split the rows
    const int npass_items = n_pass <= kThreads ? n_pass : n_pass;
    k_gram2<<<nblk, kThreads, smem, ctx->stream>>>(A, B ? B : A, rows, ldr, ngram, item0, npass_items, rpb,
                                                   scratch.as<double>());
    ctx->count();
  }
  k_gram_finalize<double><<<std::max(1, ceil_div_i((int64_t)ngram * rank * rank, 32)), 256, 0,
                    ctx->stream>>>(scratch.as<double>(), nblk, ngram, ldr, rank, outP, outC);
  ctx->count();
  check_launch();
}

void gram_enqueue(Ctx* ctx, const float* A, const float* B, int64_t rows, int rank, int ldr, double* out,
                  DevBuf& scratch) {
  // out = B'A : run the pair kernel with (A, B) and keep the cross Gram
  if (A == B) {
    gram2_enqueue(ctx, A, nullptr, rows, rank, ldr, out, nullptr, scratch);
  } else {
    static thread_local DevBuf tmp;
    tmp.ensure((size_t)rank * rank * 8);
    gram2_enqueue(ctx, A, B, rows, rank, ldr, tmp.as<double>(), out, scratch);
  }
}

void hist_coeffs_enqueue(Ctx* ctx, int ndim, int rank, const double* P, const double* C, const double* S,
                         double w, float* Mk, float* Nk, const double* s, double extra) {
  k_hist_coeffs<<<1, 256, 0, ctx->stream>>>(ndim, rank, P, C, S, w, s, extra, Mk, Nk);
  ctx->count();
  check_launch();
}

void dense_wgrad_enqueue(Ctx* ctx, int ndim, int rank, int ldr, const double* P, const double* b, const double* s,
                         double* out) {
  k_dense_wgrad<<<1, ldr, 0, ctx->stream>>>(ndim, rank, ldr, P, b, s, out);
  ctx->count();
  check_launch();
}

void factor_update_modes_enqueue(Ctx* ctx, const K5Modes& m, int ndim, int rank, int ldr, double reg, double rate_i,
                                 double beta1, double beta2, double eps, double lower, long long code) {
  ProfScope prof_scope(ctx, kProfUpdate);
  const float fb1 = (float)beta1, fomb1 = (float)(1.0 - beta1), fb2 = (float)beta2, fomb2 = (float)(1.0 - beta2);
  int64_t rmax = 1;
  for (int k = 0; k < ndim; ++k) rmax = std::max<int64_t>(rmax, m.rows[k]);
  int GR = 1;
  while (GR < rank) GR <<= 1;
  auto launch = [&](auto kern) {
    const int64_t rows_per_block = (kThreads / GR) * kK5Rows;
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((rmax + rows_per_block - 1) / rows_per_block,
                                                                (int64_t)kNumSMs * 3));
    kern<<<dim3(gx, ndim), kThreads, 0, ctx->stream>>>(m, rank, ldr, (float)reg, (float)rate_i, fb1, fomb1, fb2,
                                                         fomb2, (float)eps, (float)lower, ctx->flags.as<DevFlags>(),
                                                         code);
  };
  switch (GR) {
    case 1: launch(k_factor_update_modes<1>); break;
    case 2: launch(k_factor_update_modes<2>); break;
    case 4: launch(k_factor_update_modes<4>); break;
    case 8: launch(k_factor_update_modes<8>); break;
    case 16: launch(k_factor_update_modes<16>); break;
    default: launch(k_factor_update_modes<32>); break;
  }
  ctx->count();
  check_launch();
}

void factor_update_enqueue(Ctx* ctx, int64_t rows, int rank, int ldr, float* A, const float* Aold,
                           const float* G, float* u, float* v, const float* Mk, const float* Nk,
                           double reg, double rate_i, double beta1, double beta2, double eps, double lower,
                           long long code) {
  if (rows <= 0) return;
  ProfScope prof_scope(ctx, kProfUpdate);
  const float fb1 = (float)beta1, fomb1 = (float)(1.0 - beta1), fb2 = (float)beta2, fomb2 = (float)(1.0 - beta2);
  if (rank <= 32) {
    int GR = 1;
    while (GR < rank) GR <<= 1;
    auto launch = [&](auto kern) {
      const int per_sm = occupancy(kern, 0);
      const int64_t rows_per_block = (kThreads / GR) * kK5Rows;
      const int grid = (int)std::max<int64_t>(
          1, std::min<int64_t>((rows + rows_per_block - 1) / rows_per_block, (int64_t)kNumSMs * std::max(per_sm, 1)));
      kern<<<grid, kThreads, 0, ctx->stream>>>(rows, rank, ldr, A, Aold, G, u, v, Mk, Nk, (float)reg, (float)rate_i,
                                               fb1, fomb1, fb2, fomb2, (float)eps, (float)lower,
                                               ctx->flags.as<DevFlags>(), code);
    };
    switch (GR) {
      case 1: launch(k_factor_update<1>); break;
      case 2: launch(k_factor_update<2>); break;
      case 4: launch(k_factor_update<4>); break;
      case 8: launch(k_factor_update<8>); break;
      case 16: launch(k_factor_update<16>); break;
      default: launch(k_factor_update<32>); break;
    }
  } else if (Mk && ldr <= 128) {
    auto launch = [&](auto kern, int L) {
      const size_t smem = ((size_t)2 * L * L + (size_t)4 * kK5TileRows * L) * 4;
      allow_smem(kern, smem);
      const int per_sm = occupancy(kern, smem);
      const int64_t tiles = (rows + kK5TileRows - 1) / kK5TileRows;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)kNumSMs * std::max(per_sm, 1)));
      kern<<<grid, kThreads, smem, ctx->stream>>>(rows, rank, A, Aold, G, u, v, Mk, Nk, (float)reg, (float)rate_i,
                                                  fb1, fomb1, fb2, fomb2, (float)eps, (float)lower,
                                                  ctx->flags.as<DevFlags>(), code);
    };
    if (ldr <= 64) launch(k_factor_update_tiled<64>, 64);
    else launch(k_factor_update_tiled<128>, 128);
  } else {
    const size_t need = Mk ? (size_t)2 * rank * rank * 4 : 0;
    const bool stage = need > 0 && need <= 200 * 1024;
    const size_t smem = stage ? need : 0;
    auto launch = [&](auto kern) {
      allow_smem(kern, smem);
      const int64_t groups = kThreads / 32;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + groups - 1) / groups, kNumSMs * 4));
      kern<<<grid, kThreads, smem, ctx->stream>>>(rows, rank, ldr, A, Aold, G, u, v, Mk, Nk, (float)reg,
                                                  (float)rate_i, fb1, fomb1, fb2, fomb2, (float)eps, (float)lower,
                                                  ctx->flags.as<DevFlags>(), code, stage ? 1 : 0);
    };
    if (rank <= 64) launch(k_factor_update_wide<2>);
    else if (rank <= 128) launch(k_factor_update_wide<4>);
    else launch(k_factor_update_wide<8>);
  }
  ctx->count();
  check_launch();
}

void weight_step_enqueue(Ctx* ctx, const double* partials, int nblk, int rank, int ldr, double* wstate, float* s_f,
                         double mu, double rate_i, double beta1, double beta2, double eps, double lower,
                         long long code) {
  ProfScope prof_scope(ctx, kProfUpdate);
  k_weight_step<<<1, ldr, 0, ctx->stream>>>(partials, nblk, rank, ldr, wstate, s_f, mu, rate_i, beta1, beta2, eps,
                                            lower, ctx->flags.as<DevFlags>(), code);
  ctx->count();
  check_launch();
}

void hist_penalty_enqueue(Ctx* ctx, int ndim, int rank, const double* Poo, const double* Pon, const double* Pnn,
                          const double* window_s, const double* window_coef, int H, double* out) {
  const size_t need = (size_t)rank * rank * 8;
  double* qglobal = nullptr;
  size_t smem = need;
  if (need > 200 * 1024) {
    static thread_local DevBuf qbuf;
    qglobal = static_cast<double*>(qbuf.ensure(need));
    smem = 0;
  }
  allow_smem(k_hist_penalty, smem);
  k_hist_penalty<<<1, 256, smem, ctx->stream>>>(ndim, rank, Poo, Pon, Pnn, window_s, window_coef, H, out, qglobal);
  ctx->count();
  check_launch();
}

}  // namespace ogcp
