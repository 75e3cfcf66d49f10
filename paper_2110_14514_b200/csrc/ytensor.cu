// Parity mode of the merged sampled gradient tensor Y (sampled_gradient_tensor,
// sampling.py:209-239) and of its per-mode row-segment layout.
//
// The solves never build Y (MTTKRP is linear in Y, so the fused kernels scatter
// per draw or per merged nonzero).  For parity checks and for callers of the
// reference's fine-grained API this file reproduces Y's layout bit-exactly:
// draws are keyed by their 64-bit linear index and stably radix-sorted (CUB),
// so each run of equal keys keeps draw order -- its head is np.unique's
// first occurrence and its sum is np.bincount's summation order.  The
// segment layout of mode k is the stable argsort of Y's k-th coordinates plus
// the row offsets (cumsum of bincount) that a sort-by-row MTTKRP walks.
#include <cub/cub.cuh>

#include "common.cuh"
#include "compute.cuh"
#include "hash.cuh"

namespace ogcp {

// Per draw: coordinates, linear key, and y = scale * f'(x, m) in fp64.
__global__ void k_draw_values(SamplesP S, ModelP M, const double* __restrict__ w, LossP L, Strides st,
                              unsigned long long* __restrict__ keys, int32_t* __restrict__ idx,
                              int32_t* __restrict__ coords, double* __restrict__ y,
                              unsigned int* __restrict__ bad) {
  const int64_t total = S.p + S.q;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < total; n += (int64_t)gridDim.x * blockDim.x) {
    int c[kMaxModes];
    double x = 0.0, scale;
    if (n < S.p) {
      const int* r = S.rec + (int64_t)S.ord[n] * S.rec_ints;
      for (int k = 0; k < M.ndim; ++k) c[k] = r[k];
      x = (double)__int_as_float(r[M.ndim]);
      scale = S.nz_scale;
    } else {
      for (int k = 0; k < M.ndim; ++k) c[k] = S.zsub[(n - S.p) * M.ndim + k];
      scale = S.zero_scale;
    }
    double m = 0.0;
    for (int j = 0; j < M.rank; ++j) {
      double pr = w[j];
      for (int k = 0; k < M.ndim; ++k) pr *= (double)M.A[k][(int64_t)c[k] * M.ldr + j];
      m += pr;
    }
    double d;
    if (L.kind == OGCP_GAUSSIAN) d = 2.0 * (m - x);
    else if (L.kind == OGCP_POISSON) d = 1.0 - x / (m + L.eps_d);
    else d = 1.0 / (m + 1.0) - x / (m + L.eps_d);
    if (!isfinite(m)) atomicOr(bad, 1u);
    if (L.kind != OGCP_GAUSSIAN && m < 0.0) atomicOr(bad, 2u);
    uint64_t key = 0;
    for (int k = 0; k < M.ndim; ++k) {
      key += (uint64_t)(uint32_t)c[k] * st.s[k];
      coords[n * M.ndim + k] = c[k];
    }
    keys[n] = key;
    idx[n] = (int32_t)n;
    y[n] = scale * d;
  }
}

__global__ void k_run_heads(const unsigned long long* __restrict__ k, int64_t n, int32_t* __restrict__ head) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// pos = inclusive scan of heads; run u starts at the i with head[i] and pos[i] == u + 1.
__global__ void k_run_merge(const unsigned long long* __restrict__ k, const int32_t* __restrict__ sidx,
                            const int32_t* __restrict__ head, const int32_t* __restrict__ pos, int64_t n, int ndim,
                            const int32_t* __restrict__ coords, const double* __restrict__ y,
                            int32_t* __restrict__ ycoords, double* __restrict__ yvals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!head[i]) continue;
    const int64_t u = pos[i] - 1;
    double s = 0.0;
    for (int64_t j = i; j < n && (j == i || k[j] == k[i]); ++j) s += y[sidx[j]];
    const int32_t first = sidx[i];  // stable sort: earliest draw of this coordinate
    for (int d = 0; d < ndim; ++d) ycoords[u * ndim + d] = coords[(int64_t)first * ndim + d];
    yvals[u] = s;
  }
}

__global__ void k_iota32(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)i;
}

__global__ void k_column(const int32_t* __restrict__ coords, int64_t n, int ndim, int mode, int32_t* __restrict__ col) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    col[i] = coords[i * ndim + mode];
}

// offsets[r] = first position whose sorted row index >= r (r = 0..dim).
__global__ void k_row_offsets(const int32_t* __restrict__ sorted_rows, int64_t n, int64_t dim,
                              int64_t* __restrict__ offsets) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= dim; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (sorted_rows[mid] < r) lo = mid + 1;
      else hi = mid;
    }
    offsets[r] = lo;
  }
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, kNumSMs * 8)); }

void iota_enqueue(Ctx* ctx, int32_t* p, int64_t n) {
  k_iota32<<<grid_for(n), 256, 0, ctx->stream>>>(p, n);
  ctx->count();
  check_launch();
}

// ---------------------------------------------------------- bucketed layout
__global__ void k_bucket_keys(const int* __restrict__ rec, int rec_ints, int mode, long long dim, int nb, int64_t n,
                              uint8_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = (uint8_t)(((long long)rec[i * rec_ints + mode] * nb) / dim);
}

__global__ void k_add32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] += v;
}

__global__ void k_gather_records(const int4* __restrict__ rec, int vec_per_rec, const int32_t* __restrict__ perm,
                                 int64_t n, int4* __restrict__ out) {
  const int64_t total = n * vec_per_rec;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / vec_per_rec;
    const int v = (int)(e - i * vec_per_rec);
    out[e] = __ldg(rec + (int64_t)__ldg(perm + i) * vec_per_rec + v);
  }
}

void slice_bucket_layout(Ctx* ctx, Slice* X, int mode, int nb, int64_t olo, int64_t ohi) {
  const int64_t n = ohi - olo;  // the ordinals [olo, ohi) this rank owns (the whole slice on one GPU)
  cudaStream_t s = ctx->stream;
  int bits = 0;
  while ((1 << bits) < nb) ++bits;
  DevBuf keys, keys_s, iota, cub_tmp;
  keys.ensure(n);
  keys_s.ensure(n);
  iota.ensure(n * 4);
  X->perm.ensure(n * 4);
  X->rec_b.ensure((size_t)n * X->rec_ints * 4);
  k_bucket_keys<<<grid_for(n), 256, 0, s>>>(X->records.as<int>() + olo * X->rec_ints, X->rec_ints, mode,
                                            (long long)X->dims[mode], nb, n, keys.as<uint8_t>());
  k_iota32<<<grid_for(n), 256, 0, s>>>(iota.as<int32_t>(), n);
  if (olo) k_add32<<<grid_for(n), 256, 0, s>>>(iota.as<int32_t>(), n, (int32_t)olo);
  size_t tb = 0;
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint8_t>(), keys_s.as<uint8_t>(),
                                            iota.as<int32_t>(), X->perm.as<int32_t>(), (int)n, 0, bits, s));
  cub_tmp.ensure(tb);
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp.ptr, tb, keys.as<uint8_t>(), keys_s.as<uint8_t>(),
                                            iota.as<int32_t>(), X->perm.as<int32_t>(), (int)n, 0, bits, s));
  const int vpr = X->rec_ints / 4;
  k_gather_records<<<grid_for(n * vpr), 256, 0, s>>>(reinterpret_cast<const int4*>(X->records.ptr), vpr,
                                                     X->perm.as<int32_t>(), n, reinterpret_cast<int4*>(X->rec_b.ptr));
  ctx->count(4);
  check_launch();
  OGCP_CUDA(cudaStreamSynchronize(s));  // scratch buffers are released on return
  X->bucket_mode = mode;
  X->nbuckets = nb;
  X->bucket_olo = olo;
  X->bucket_ohi = ohi;
}

struct YScratch {
  DevBuf keys, keys_s, idx, idx_s, coords, y, head, pos, cub, bad, cols, cols_s;
};

static YScratch& yscratch() {
  static thread_local YScratch s;
  return s;
}

int64_t gradient_tensor_impl(Ctx* ctx, const SamplesP& S, const ModelP& M, const double* w_dev, const LossP& L,
                             const Strides& st, int32_t* ycoords, double* yvals, unsigned int* bad_host) {
  const int64_t n = S.p + S.q;
  if (n == 0) return 0;
  YScratch& Y = yscratch();
  cudaStream_t s = ctx->stream;
  auto* keys = static_cast<unsigned long long*>(Y.keys.ensure(n * 8));
  auto* keys_s = static_cast<unsigned long long*>(Y.keys_s.ensure(n * 8));
  auto* idx = static_cast<int32_t*>(Y.idx.ensure(n * 4));
  auto* idx_s = static_cast<int32_t*>(Y.idx_s.ensure(n * 4));
  auto* coords = static_cast<int32_t*>(Y.coords.ensure(n * M.ndim * 4));
  auto* y = static_cast<double*>(Y.y.ensure(n * 8));
  auto* head = static_cast<int32_t*>(Y.head.ensure(n * 4));
  auto* pos = static_cast<int32_t*>(Y.pos.ensure(n * 4));
  auto* bad = static_cast<unsigned int*>(Y.bad.ensure(4));
  OGCP_CUDA(cudaMemsetAsync(bad, 0, 4, s));
  k_draw_values<<<grid_for(n), 256, 0, s>>>(S, M, w_dev, L, st, keys, idx, coords, y, bad);
  size_t tb = 0;
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_s, idx, idx_s, (int)n, 0, 64, s));
  void* tmp = Y.cub.ensure(tb);
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_s, idx, idx_s, (int)n, 0, 64, s));
  k_run_heads<<<grid_for(n), 256, 0, s>>>(keys_s, n, head);
  size_t tb2 = 0;
  OGCP_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb2, head, pos, (int)n, s));
  tmp = Y.cub.ensure(std::max(tb, tb2));
  OGCP_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb2, head, pos, (int)n, s));
  k_run_merge<<<grid_for(n), 256, 0, s>>>(keys_s, idx_s, head, pos, n, M.ndim, coords, y, ycoords, yvals);
  ctx->count(4);
  check_launch();
  int32_t nu = 0;
  OGCP_CUDA(cudaMemcpyAsync(&nu, pos + n - 1, 4, cudaMemcpyDeviceToHost, s));
  OGCP_CUDA(cudaMemcpyAsync(bad_host, bad, 4, cudaMemcpyDeviceToHost, s));
  OGCP_CUDA(cudaStreamSynchronize(s));
  return nu;
}

void segment_layout_impl(Ctx* ctx, const int32_t* coords, int64_t n, int ndim, int mode, int64_t dim, int32_t* perm,
                         int64_t* offsets) {
  cudaStream_t s = ctx->stream;
  YScratch& Y = yscratch();
  if (n == 0) {
    OGCP_CUDA(cudaMemsetAsync(offsets, 0, (dim + 1) * 8, s));
    OGCP_CUDA(cudaStreamSynchronize(s));
    return;
  }
  auto* col = static_cast<int32_t*>(Y.cols.ensure(n * 4));
  auto* col_s = static_cast<int32_t*>(Y.cols_s.ensure(n * 4));
  auto* iota = static_cast<int32_t*>(Y.idx.ensure(n * 4));
  k_column<<<grid_for(n), 256, 0, s>>>(coords, n, ndim, mode, col);
  k_iota32<<<grid_for(n), 256, 0, s>>>(iota, n);
  int bits = 1;
  while ((1ll << bits) <= dim) ++bits;
  size_t tb = 0;
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, col, col_s, iota, perm, (int)n, 0, bits, s));
  void* tmp = Y.cub.ensure(tb);
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, col, col_s, iota, perm, (int)n, 0, bits, s));
  k_row_offsets<<<grid_for(dim + 1), 256, 0, s>>>(col_s, n, dim, offsets);
  ctx->count(3);
  check_launch();
  OGCP_CUDA(cudaStreamSynchronize(s));
}

}  // namespace ogcp
