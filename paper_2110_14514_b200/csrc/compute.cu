// K2..K6: sampled-entry model evaluation, loss/derivative, sampled-MTTKRP
// scatter, weight gradient, objective, Gram, history and fused Adam.
//
// Thread mapping for the sample kernels: a group of G lanes serves one sample;
// lane gl owns the float4 chunks v*G+gl (v < V) of every factor row, so the
// d row gathers of a sample are G*16-byte contiguous 128-bit loads (one 128 B
// line per row at R = 32), the Hadamard product and the dot with s stay in
// registers and m is reduced with log2(G) xor-shuffles.
//
// Reference: model_values tensor.py:203-211; LossFunction losses.py:58-78;
// sampled_mttkrp kernels.py:33-56 (times s, solvers.py:139-140);
// weight_gradient_mttkrp kernels.py:59-72; estimate_objective
// sampling.py:177-206; gram kernels.py:75-98; _add_reg_and_history
// solvers.py:159-179; Adam.step adam.py:51-81; _ensure_finite solvers.py:188-194.
#include <algorithm>

#include "common.cuh"
#include "compute.cuh"

namespace ogcp {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;

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
__device__ __forceinline__ double floss(int kind, double x, double m, double eps) {
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
};

// Load coordinates, value and the d factor-row chunks of sample n.
template <int D, int G, int V>
__device__ __forceinline__ void gather(int64_t n, bool valid, const SamplesP& S, const ModelP& M, int gl,
                                       Sample<D, V>& s) {
  constexpr int NDm = ND<D>::v;
  const int nd = D > 0 ? D : M.ndim;
  int t[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) t[k] = 0;
  s.x = 0.0f;
  s.scale = 0.0f;
  if (valid) {
    if (n < S.p) {
      const int o = __ldg(S.ord + n);
      const int4* r = reinterpret_cast<const int4*>(S.rec + (int64_t)o * S.rec_ints);
      int4 v0 = __ldg(r);
      t[0] = v0.x; t[1] = v0.y; t[2] = v0.z; t[3] = v0.w;
      if (D == 0 || D > 3) {
        if (S.rec_ints == 8) {
          int4 v1 = __ldg(r + 1);
          t[4] = v1.x; t[5] = v1.y; t[6] = v1.z; t[7] = v1.w;
        }
      }
      if (D > 0) s.x = __int_as_float(t[D]);
      else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k == nd) s.x = __int_as_float(t[k]);
      }
      s.scale = (float)S.nz_scale;
    } else {
      const int32_t* z = S.zsub + (n - S.p) * nd;
#pragma unroll
      for (int k = 0; k < NDm; ++k)
        if (k < nd) t[k] = __ldg(z + k);
      s.scale = (float)S.zero_scale;
    }
  }
#pragma unroll
  for (int k = 0; k < NDm; ++k) {
    s.idx[k] = t[k];
    if (k < nd) {
      const float4* row = reinterpret_cast<const float4*>(M.A[k] + (int64_t)t[k] * M.ldr);
#pragma unroll
      for (int v = 0; v < V; ++v) s.a[k][v] = valid ? __ldg(row + v * G + gl) : make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) s.a[k][v] = make_float4(1.f, 1.f, 1.f, 1.f);
    }
  }
}

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

template <int D, int G, int V>
__global__ void __launch_bounds__(kThreads) k_sgrad(SamplesP S, ModelP M, const float* __restrict__ s_f, LossP L,
                                                    GradPtrs GP, PrivP PV,
                                                    DevFlags* flags, long long code) {
  extern __shared__ float smem[];
  constexpr int NDm = ND<D>::v;
  const int nd = D > 0 ? D : M.ndim;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  for (int64_t i = threadIdx.x; i < (PV.nmodes ? PV.off[PV.nmodes - 1] + PV.len[PV.nmodes - 1] : 0); i += blockDim.x)
    smem[i] = 0.0f;
  __syncthreads();
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * G + gl);
  int priv_slot[NDm];
#pragma unroll
  for (int k = 0; k < NDm; ++k) {
    priv_slot[k] = -1;
    for (int j = 0; j < PV.nmodes; ++j)
      if (PV.mode[j] == k) priv_slot[k] = j;
  }
  const int64_t total = S.p + S.q;
  constexpr int SPW = 32 / G;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bits = 0;
  for (int64_t base = warp * SPW; base < total; base += nwarps * SPW) {
    const int64_t n = base + lane / G;
    const bool valid = n < total;
    Sample<D, V> s;
    gather<D, G, V>(n, valid, S, M, gl, s);
    const float m = model_value<D, G, V>(s, s4);
    if (!valid) continue;
    bits |= domain_bits(L.kind, m);
    const float y = s.scale * dloss(L.kind, s.x, m, L.eps);
#pragma unroll
    for (int k = 0; k < NDm; ++k) {
      if (k >= nd) break;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float4 c = make_float4(y * s4[v].x, y * s4[v].y, y * s4[v].z, y * s4[v].w);
#pragma unroll
        for (int j = 0; j < NDm; ++j)
          if (j != k && j < nd) c = mul4(c, s.a[j][v]);
        const int64_t off = (int64_t)s.idx[k] * M.ldr + (v * G + gl) * 4;
        if (priv_slot[k] >= 0) {
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

// ------------------------------------------------------------------ K2 (weights)
template <int D, int G, int V>
__global__ void __launch_bounds__(kThreads) k_wgrad(SamplesP S, ModelP M, const float* __restrict__ s_f, LossP L,
                                                    double* __restrict__ partials, DevFlags* flags, long long code) {
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
  constexpr int SPW = 32 / G;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bits = 0;
  for (int64_t base = warp * SPW; base < total; base += nwarps * SPW) {
    const int64_t n = base + lane / G;
    const bool valid = n < total;
    Sample<D, V> s;
    gather<D, G, V>(n, valid, S, M, gl, s);
    const float m = model_value<D, G, V>(s, s4);
    if (!valid) continue;
    bits |= domain_bits(L.kind, m);
    const float y = s.scale * dloss(L.kind, s.x, m, L.eps);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float4 pr = s.a[0][v];
#pragma unroll
      for (int k = 1; k < NDm; ++k) pr = mul4(pr, s.a[k][v]);
      acc[v][0] += (double)(y * pr.x);
      acc[v][1] += (double)(y * pr.y);
      acc[v][2] += (double)(y * pr.z);
      acc[v][3] += (double)(y * pr.w);
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
}

// ------------------------------------------------------------------ K6
template <int D, int G, int V>
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
  constexpr int SPW = 32 / G;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bits = 0;
  for (int64_t base = warp * SPW; base < total; base += nwarps * SPW) {
    const int64_t n = base + lane / G;
    const bool valid = n < total;
    Sample<D, V> s;
    gather<D, G, V>(n, valid, S, M, gl, s);
    const float m = model_value<D, G, V>(s, s4);
    if (!valid || gl != 0) continue;
    bits |= domain_bits(L.kind, m);
    const double f = floss(L.kind, (double)s.x, (double)m, L.eps_d);
    if (n < S.p) acc_nz += f;
    else acc_z += f;
  }
  if (bits) report(flags, kFlagData, code, bits);
  double acc = acc_nz * S.nz_scale + acc_z * S.zero_scale;
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int j = 0; j < kThreads / 32; ++j) t += red[j];
    partials[blockIdx.x] = t;
  }
}

// Exact loss: nonzero correction f(x,m) - f(0,m) over every stored entry.
template <int D, int G, int V>
__global__ void __launch_bounds__(kThreads) k_exact_nz(SamplesP S, ModelP M, const float* __restrict__ s_f,
                                                       LossP L, double* __restrict__ partials, DevFlags* flags,
                                                       long long code) {
  __shared__ double red[kThreads / 32];
  const int lane = threadIdx.x & 31;
  const int gl = lane & (G - 1);
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * G + gl);
  double acc = 0.0;
  const int64_t total = S.p;
  constexpr int SPW = 32 / G;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned bits = 0;
  for (int64_t base = warp * SPW; base < total; base += nwarps * SPW) {
    const int64_t n = base + lane / G;
    const bool valid = n < total;
    Sample<D, V> s;
    gather<D, G, V>(n, valid, S, M, gl, s);
    const float m = model_value<D, G, V>(s, s4);
    if (!valid || gl != 0) continue;
    bits |= domain_bits(L.kind, m);
    acc += floss(L.kind, (double)s.x, (double)m, L.eps_d) - floss(L.kind, 0.0, (double)m, L.eps_d);
  }
  if (bits) report(flags, kFlagData, code, bits);
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

__global__ void k_sum_partials_vec(const double* __restrict__ p, int nblk, int len, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < len; c += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int b = 0; b < nblk; ++b) t += p[(int64_t)b * len + c];
    out[c] = t;
  }
}

// ------------------------------------------------------------------ K4 Gram
// out = B' A (R x R) ; each block reduces a row range in fp32 tiles of kGramTile
// rows and accumulates tiles in fp64; partials summed in block order.
constexpr int kGramTile = 32;
__global__ void __launch_bounds__(kThreads) k_gram(const float* __restrict__ A, const float* __restrict__ B,
                                                   int64_t rows, int rank, int ldr, int64_t rows_per_block,
                                                   double* __restrict__ partials) {
  extern __shared__ float sm[];
  float* sa = sm;
  float* sb = sm + kGramTile * ldr;
  const int RR = rank * rank;
  const int64_t r0 = blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  for (int e0 = 0; e0 < RR; e0 += 16 * kThreads) {
    double acc[16];
    int ei[16], ej[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      int e = e0 + t * kThreads + threadIdx.x;
      acc[t] = 0.0;
      ei[t] = e < RR ? e / rank : -1;
      ej[t] = e < RR ? e % rank : 0;
    }
    for (int64_t rb = r0; rb < r1; rb += kGramTile) {
      const int nr = (int)min((int64_t)kGramTile, r1 - rb);
      __syncthreads();
      for (int i = threadIdx.x; i < nr * ldr; i += blockDim.x) {
        sa[i] = A[rb * ldr + i];
        sb[i] = B[rb * ldr + i];
      }
      __syncthreads();
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        if (ei[t] < 0) continue;
        float f = 0.0f;
        for (int r = 0; r < nr; ++r) f += sb[r * ldr + ei[t]] * sa[r * ldr + ej[t]];
        acc[t] += (double)f;
      }
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      int e = e0 + t * kThreads + threadIdx.x;
      if (e < RR) partials[blockIdx.x * (int64_t)RR + e] = acc[t];
    }
  }
}

// ------------------------------------------------------------------ history coefficients
__global__ void k_hist_coeffs(int ndim, int rank, const double* __restrict__ P, const double* __restrict__ C,
                              const double* __restrict__ S, double w, float* __restrict__ Mk,
                              float* __restrict__ Nk) {
  const int RR = rank * rank;
  for (int e = threadIdx.x; e < RR; e += blockDim.x) {
    for (int k = 0; k < ndim; ++k) {
      double gp = 1.0, gc = 1.0;
      for (int m = 0; m < ndim; ++m) {
        if (m == k) continue;
        gp *= P[(int64_t)m * RR + e];
        gc *= C[(int64_t)m * RR + e];
      }
      Mk[(int64_t)k * RR + e] = (float)(w * gp * S[e]);
      Nk[(int64_t)k * RR + e] = (float)(w * gc * S[e]);
    }
  }
}

// ------------------------------------------------------------------ K5
// One warp-group of GR lanes per row; columns c = gl + j*GR.
template <int GR>
__global__ void __launch_bounds__(kThreads) k_factor_update(int64_t rows, int rank, int ldr, float* __restrict__ A,
                                                            const float* __restrict__ Aold,
                                                            const float* __restrict__ G, float* __restrict__ u,
                                                            float* __restrict__ v, const float* __restrict__ Mk,
                                                            const float* __restrict__ Nk, double reg, double rate_i,
                                                            double b1, double b2, double eps, double lower,
                                                            DevFlags* flags, long long code) {
  extern __shared__ float sm[];
  const bool hist = Mk != nullptr;
  const int RR = rank * rank;
  if (hist) {
    for (int i = threadIdx.x; i < RR; i += blockDim.x) {
      sm[i] = Mk[i];
      sm[RR + i] = Nk[i];
    }
  }
  __syncthreads();
  constexpr int CPL = GR < 32 ? 1 : 8;  // columns per lane (rank <= GR, or <= 256 at GR = 32)
  const int lane = threadIdx.x & 31;
  const int gl = lane & (GR - 1);
  const int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / GR;
  const int64_t ngrp = ((int64_t)gridDim.x * blockDim.x) / GR;
  const int ncpl = (rank + GR - 1) / GR;
  bool bad = false;
  const int64_t rows_pad = ((rows + ngrp - 1) / ngrp) * ngrp;
  for (int64_t i = grp; i < rows_pad; i += ngrp) {
    const bool valid = i < rows;
    float a[CPL], ao[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c = gl + j * GR;
      a[j] = (j < ncpl && c < rank && valid) ? A[i * ldr + c] : 0.f;
      ao[j] = (hist && j < ncpl && c < rank && valid) ? Aold[i * ldr + c] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c = gl + j * GR;
      if (j >= ncpl) break;
      float hsum = 0.0f;
      if (hist) {
        // (A Mk)[c] - (Aold Nk)[c] = sum_r a[r] Mk[r][c] - ao[r] Nk[r][c]
        for (int r = 0; r < rank; ++r) {
          const int src = r % GR, slot = r / GR;
          float ar = 0.f, aor = 0.f;
#pragma unroll
          for (int jj = 0; jj < CPL; ++jj)
            if (jj == slot) {
              ar = __shfl_sync(kFull, a[jj], src, GR);
              aor = __shfl_sync(kFull, ao[jj], src, GR);
            }
          if (c < rank) hsum += ar * sm[r * rank + c] - aor * sm[RR + r * rank + c];
        }
      }
      if (!valid || c >= rank) continue;
      const int64_t at = i * ldr + c;
      const double g = (double)G[at] + reg * (double)a[j] + (double)hsum;
      const double un = b1 * (double)u[at] + (1.0 - b1) * g;
      const double vn = b2 * (double)v[at] + (1.0 - b2) * g * g;
      double an = (double)a[j] - rate_i * un / (sqrt(vn) + eps);
      an = fmax(an, lower);
      const float af = (float)an;
      u[at] = (float)un;
      v[at] = (float)vn;
      A[at] = af;
      if (!isfinite(af)) bad = true;
    }
  }
  if (bad) report(flags, kFlagDiverge, code, 0);
}

// ------------------------------------------------------------------ weight step
// wstate layout (double): s[ldr] u[ldr] v[ldr] s_o[ldr] u_o[ldr] v_o[ldr]
__global__ void k_weight_step(const double* __restrict__ partials, int nblk, int rank, int ldr,
                              double* __restrict__ ws, float* __restrict__ s_f, double mu, double rate_i, double b1,
                              double b2, double eps, double lower, DevFlags* flags, long long code) {
  const int r = threadIdx.x;
  if (r >= ldr) return;
  if (r >= rank) {
    s_f[r] = 0.f;
    return;
  }
  double g = 0.0;
  for (int b = 0; b < nblk; ++b) g += partials[(int64_t)b * ldr + r];
  double s = ws[r];
  g += mu * s;
  double u = b1 * ws[ldr + r] + (1.0 - b1) * g;
  double v = b2 * ws[2 * ldr + r] + (1.0 - b2) * g * g;
  double sn = fmax(s - rate_i * u / (sqrt(v) + eps), lower);
  ws[r] = sn;
  ws[ldr + r] = u;
  ws[2 * ldr + r] = v;
  s_f[r] = (float)sn;
  if (!isfinite(sn)) report(flags, kFlagDiverge, code, 0);
}

// ------------------------------------------------------------------ history penalty
// out[0] = sum_h coef_h * max(s_h' Q s_h, 0), Q = Poo - (Pon + Pon') + Pnn (all-mode Grams).
__global__ void k_hist_penalty(int ndim, int rank, const double* __restrict__ Poo, const double* __restrict__ Pon,
                               const double* __restrict__ Pnn, const double* __restrict__ Ws,
                               const double* __restrict__ coef, int H, double* __restrict__ out) {
  extern __shared__ double q[];
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
  // one warp per window entry, fixed order of accumulation per warp then warps in order
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
template <class F>
static void dispatch_dgv(int ndim, int ldr, F&& f);

#define OGCP_DISPATCH_LDR(D)                                        \
  switch (ldr) {                                                    \
    case 4: f(std::integral_constant<int, D>(), std::integral_constant<int, 1>(), std::integral_constant<int, 1>()); break;  \
    case 8: f(std::integral_constant<int, D>(), std::integral_constant<int, 2>(), std::integral_constant<int, 1>()); break;  \
    case 16: f(std::integral_constant<int, D>(), std::integral_constant<int, 4>(), std::integral_constant<int, 1>()); break; \
    case 32: f(std::integral_constant<int, D>(), std::integral_constant<int, 8>(), std::integral_constant<int, 1>()); break; \
    case 64: f(std::integral_constant<int, D>(), std::integral_constant<int, 16>(), std::integral_constant<int, 1>()); break; \
    case 128: f(std::integral_constant<int, D>(), std::integral_constant<int, 32>(), std::integral_constant<int, 1>()); break; \
    case 256: f(std::integral_constant<int, D>(), std::integral_constant<int, 32>(), std::integral_constant<int, 2>()); break; \
    default: throw Error(OGCP_E_USAGE, "unsupported padded rank " + std::to_string(ldr));                  \
  }

template <class F>
static void dispatch_dgv(int ndim, int ldr, F&& f) {
  switch (ndim) {
    case 2: OGCP_DISPATCH_LDR(2); break;
    case 3: OGCP_DISPATCH_LDR(3); break;
    case 4: OGCP_DISPATCH_LDR(4); break;
    default: OGCP_DISPATCH_LDR(0); break;
  }
}

static int sample_grid(int64_t total, int G, int per_sm) {
  const int64_t groups_per_block = kThreads / G;
  const int64_t need = (total + groups_per_block - 1) / groups_per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)kNumSMs * per_sm));
}

void sgrad_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                   float* const* grads, long long code) {
  GradPtrs GP;
  for (int k = 0; k < kMaxModes; ++k) GP.g[k] = k < M.ndim ? grads[k] : nullptr;
  for (int k = 0; k < M.ndim; ++k)
    OGCP_CUDA(cudaMemsetAsync(grads[k], 0, (size_t)M.dims[k] * M.ldr * 4, ctx->stream));
  const int64_t total = S.p + S.q;
  if (total == 0) return;
  // privatise small modes in shared memory
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
  ProfScope prof_scope(ctx, kProfSgrad);
  dispatch_dgv(M.ndim, M.ldr, [&](auto Dc, auto Gc, auto Vc) {
    constexpr int D = decltype(Dc)::value, G = decltype(Gc)::value, V = decltype(Vc)::value;
    auto kern = k_sgrad<D, G, V>;
    if (smem > 48 * 1024) OGCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int per_sm = smem > 0 ? std::max(1, (int)(200 * 1024 / std::max<size_t>(smem, 1))) : 8;
    const int grid = sample_grid(total, G, std::min(per_sm, 8));
    kern<<<grid, kThreads, smem, ctx->stream>>>(S, M, s_f, L, GP, PV, ctx->flags.as<DevFlags>(), code);
  });
  ctx->count();
  check_launch();
}

int wgrad_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                  double* partials, long long code) {
  const int64_t total = S.p + S.q;
  int grid = 1;
  ProfScope prof_scope(ctx, kProfWgrad);
  dispatch_dgv(M.ndim, M.ldr, [&](auto Dc, auto Gc, auto Vc) {
    constexpr int D = decltype(Dc)::value, G = decltype(Gc)::value, V = decltype(Vc)::value;
    grid = sample_grid(std::max<int64_t>(total, 1), G, 4);
    k_wgrad<D, G, V><<<grid, kThreads, 0, ctx->stream>>>(S, M, s_f, L, partials, ctx->flags.as<DevFlags>(), code);
  });
  ctx->count();
  check_launch();
  return grid;
}

int objective_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                      double* partials, long long code) {
  const int64_t total = S.p + S.q;
  int grid = 1;
  dispatch_dgv(M.ndim, M.ldr, [&](auto Dc, auto Gc, auto Vc) {
    constexpr int D = decltype(Dc)::value, G = decltype(Gc)::value, V = decltype(Vc)::value;
    grid = sample_grid(std::max<int64_t>(total, 1), G, 4);
    ProfScope prof_scope(ctx, kProfObjective);
    k_objective<D, G, V><<<grid, kThreads, 0, ctx->stream>>>(S, M, s_f, L, partials, ctx->flags.as<DevFlags>(),
                                                             code);
  });
  ctx->count();
  check_launch();
  return grid;
}

int exact_nz_enqueue(Ctx* ctx, const SamplesP& S, const ModelP& M, const float* s_f, const LossP& L,
                     double* partials, long long code) {
  int grid = 1;
  dispatch_dgv(M.ndim, M.ldr, [&](auto Dc, auto Gc, auto Vc) {
    constexpr int D = decltype(Dc)::value, G = decltype(Gc)::value, V = decltype(Vc)::value;
    grid = sample_grid(std::max<int64_t>(S.p, 1), G, 4);
    k_exact_nz<D, G, V><<<grid, kThreads, 0, ctx->stream>>>(S, M, s_f, L, partials, ctx->flags.as<DevFlags>(),
                                                            code);
  });
  ctx->count();
  check_launch();
  return grid;
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
  k_sum_partials_vec<<<std::max(1, std::min(ceil_div_i(len, 256), 64)), 256, 0, ctx->stream>>>(partials, nblk, len,
                                                                                               out);
  ctx->count();
  check_launch();
}

void gram_enqueue(Ctx* ctx, const float* A, const float* B, int64_t rows, int rank, int ldr, double* out,
                  DevBuf& scratch) {
  const int RR = rank * rank;
  int nblk = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, kNumSMs * 2));
  const int64_t rpb = (rows + nblk - 1) / nblk;
  nblk = (int)std::max<int64_t>(1, (rows + rpb - 1) / rpb);
  scratch.ensure((size_t)nblk * RR * 8);
  const size_t smem = (size_t)2 * kGramTile * ldr * 4;
  if (smem > 48 * 1024) OGCP_CUDA(cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfScope prof_scope(ctx, kProfGram);
  k_gram<<<nblk, kThreads, smem, ctx->stream>>>(A, B, rows, rank, ldr, rpb, scratch.as<double>());
  ctx->count();
  check_launch();
  sum_partials_enqueue(ctx, scratch.as<double>(), nblk, RR, out);
}

void hist_coeffs_enqueue(Ctx* ctx, int ndim, int rank, const double* P, const double* C, const double* S,
                         double w, float* Mk, float* Nk) {
  k_hist_coeffs<<<1, 256, 0, ctx->stream>>>(ndim, rank, P, C, S, w, Mk, Nk);
  ctx->count();
  check_launch();
}

void factor_update_enqueue(Ctx* ctx, int64_t rows, int rank, int ldr, float* A, const float* Aold,
                           const float* G, float* u, float* v, const float* Mk, const float* Nk,
                           double reg, double rate_i, double beta1, double beta2, double eps, double lower,
                           long long code) {
  if (rows <= 0) return;
  const size_t smem = Mk ? (size_t)2 * rank * rank * 4 : 0;
  int GR = 1;
  while (GR < rank && GR < 32) GR <<= 1;
  ProfScope prof_scope(ctx, kProfUpdate);
  auto launch = [&](auto kern) {
    if (smem > 48 * 1024) OGCP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t groups = kThreads / GR;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + groups - 1) / groups, kNumSMs * 8));
    kern<<<grid, kThreads, smem, ctx->stream>>>(rows, rank, ldr, A, Aold, G, u, v, Mk, Nk, reg, rate_i, beta1, beta2,
                                                eps, lower, ctx->flags.as<DevFlags>(), code);
  };
  switch (GR) {
    case 1: launch(k_factor_update<1>); break;
    case 2: launch(k_factor_update<2>); break;
    case 4: launch(k_factor_update<4>); break;
    case 8: launch(k_factor_update<8>); break;
    case 16: launch(k_factor_update<16>); break;
    default: launch(k_factor_update<32>); break;
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
  const size_t smem = (size_t)rank * rank * 8;
  if (smem > 48 * 1024)
    OGCP_CUDA(cudaFuncSetAttribute(k_hist_penalty, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_hist_penalty<<<1, 256, smem, ctx->stream>>>(ndim, rank, Poo, Pon, Pnn, window_s, window_coef, H, out);
  ctx->count();
  check_launch();
}

}  // namespace ogcp
