// K0 ingest: validate a COO slice, write the AoS records and build the
// membership hash (SparseTensor construction, tensor.py:63-119; membership
// contains_linear, tensor.py:163-169).
//
// HBM layout
//   records : nnz x {ndim int32 coords, float32 value} padded to 16/32 B, stored
//             in the caller's entry order (nonzero ordinals index this array).
//   hash    : open-addressing table of 64-bit linear keys (mode 0 most
//             significant, tensor.py:33-38), load <= 0.5, linear probing.
#include <cstdio>
#include <sstream>

#include "common.cuh"
#include "hash.cuh"

namespace ogcp {

struct IngestOut {
  unsigned long long bad_entry;   // min entry index with an out-of-bounds coordinate
  unsigned long long dup_key;     // min duplicated linear key
  unsigned int nonfinite, zero, negative, nonbinary;
};

template <class CT, class VT>
__global__ void k_ingest(int ndim, int64_t nnz, const CT* __restrict__ subs, const VT* __restrict__ vals,
                         Dims dims, int rec_ints, int allow_zero, int* __restrict__ rec,
                         IngestOut* out, double* __restrict__ frob_partials) {
  __shared__ double red[32];
  double fs = 0.0;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nnz;
       n += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    int c32[kMaxModes];
#pragma unroll
    for (int k = 0; k < kMaxModes; ++k) {
      if (k < ndim) {
        long long c = (long long)subs[n * ndim + k];
        ok = ok && c >= 0 && c < dims.d[k];
        c32[k] = (int)c;
      }
    }
    double v = (double)vals[n];
    if (!ok) atomicMin(&out->bad_entry, (unsigned long long)n);
    if (!isfinite(v)) atomicOr(&out->nonfinite, 1u);
    if (v == 0.0 && !allow_zero) atomicOr(&out->zero, 1u);
    if (v < 0.0) atomicOr(&out->negative, 1u);
    if (v != 0.0 && v != 1.0) atomicOr(&out->nonbinary, 1u);
    fs += v * v;
    int* r = rec + n * rec_ints;
    for (int k = 0; k < rec_ints; ++k) {
      int val = 0;
      if (k < ndim) val = ok ? c32[k] : 0;
      else if (k == ndim) val = __float_as_int((float)v);
      r[k] = val;
    }
  }
  // deterministic block reduction of ||X||^2 (tensor.py:138-141)
  for (int o = 16; o; o >>= 1) fs += __shfl_xor_sync(0xffffffffu, fs, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = fs;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) frob_partials[blockIdx.x] = t;
  }
}

__global__ void k_hash_insert(int ndim, int64_t nnz, const int* __restrict__ rec, int rec_ints,
                              Strides st, unsigned long long* __restrict__ table, uint64_t mask,
                              IngestOut* out, unsigned int* __restrict__ filter, uint64_t fmask) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nnz;
       n += (int64_t)gridDim.x * blockDim.x) {
    const int* r = rec + n * rec_ints;
    uint64_t key = 0;
    for (int k = 0; k < ndim; ++k) key += (uint64_t)(uint32_t)r[k] * st.s[k];
    if (!hash_insert(table, mask, key)) atomicMin(&out->dup_key, (unsigned long long)key);
    if (filter) {
      const uint64_t h = mix64(key);
      atomicOr(filter + filter_word(h, fmask), filter_bits(h));
    }
  }
}

__global__ void k_sum_partials(const double* p, int n, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += p[i];
    *out = s;
  }
}

__global__ void k_fill_u64(unsigned long long* p, int64_t n, unsigned long long v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

static std::string tuple_str(const int64_t* v, int n, int64_t add) {
  std::ostringstream os;
  os << "(";
  for (int i = 0; i < n; ++i) {
    os << (v[i] + add);
    if (n == 1) os << ",";
    else if (i + 1 < n) os << ", ";
  }
  os << ")";
  return os.str();
}

template <class CT, class VT>
Slice* slice_create_impl(Ctx* ctx, int ndim, const int64_t* dims, int64_t nnz, const CT* subs,
                         const VT* vals, int allow_zero) {
  if (ndim < 1 || ndim > 7) throw Error(OGCP_E_USAGE, "ogcp_b200 supports 1..7 modes");
  // _check_dims (tensor.py:19-30)
  unsigned __int128 total = 1;
  bool overflow = false;
  for (int k = 0; k < ndim; ++k) {
    if (dims[k] <= 0) throw Error(OGCP_E_DATA, "dims must be positive integers, got " + tuple_str(dims, ndim, 0));
    total *= (unsigned __int128)dims[k];
    if (total > (unsigned __int128)0x7fffffffffffffffULL) overflow = true;
  }
  if (overflow)
    throw Error(OGCP_E_DATA, "index space of size prod" + tuple_str(dims, ndim, 0) +
                                 " exceeds 2**63-1; cannot linearize");
  for (int k = 0; k < ndim; ++k)
    if (dims[k] > 0x7fffffffLL) throw Error(OGCP_E_USAGE, "ogcp_b200 supports mode sizes < 2^31");
  if (nnz >= 0x7fffffffLL) throw Error(OGCP_E_USAGE, "ogcp_b200 supports < 2^31 stored entries per slice");

  Slice* s = new Slice();
  try {
    s->ndim = ndim;
    for (int k = 0; k < ndim; ++k) s->dims[k] = dims[k];
    s->nnz = nnz;
    s->omega = (int64_t)total;
    s->omega_d = (double)total;
    s->rec_ints = record_ints(ndim);
    uint64_t st = 1;
    for (int k = ndim - 1; k >= 0; --k) { s->strides[k] = st; st *= (uint64_t)dims[k]; }
    uint64_t tsize = 1024;
    while (tsize < 2 * (uint64_t)nnz) tsize <<= 1;
    s->table_mask = tsize - 1;
    s->records.ensure((size_t)(nnz > 0 ? nnz : 1) * s->rec_ints * 4);
    s->hash.ensure(tsize * 8);
    cudaStream_t str = ctx->stream;

    DevBuf scratch;
    const int threads = 256;
    int blocks = (int)std::min<int64_t>(std::max<int64_t>(ceil_div_i(nnz, threads), 1), kNumSMs * 8);
    scratch.ensure(sizeof(IngestOut) + 8 * (blocks + 2));
    IngestOut init{~0ull, ~0ull, 0, 0, 0, 0};
    OGCP_CUDA(cudaMemcpyAsync(scratch.ptr, &init, sizeof(init), cudaMemcpyHostToDevice, str));
    double* partials = reinterpret_cast<double*>(scratch.as<char>() + sizeof(IngestOut));
    Dims dd;
    Strides ss;
    for (int k = 0; k < kMaxModes; ++k) {
      dd.d[k] = k < ndim ? dims[k] : 1;
      ss.s[k] = k < ndim ? s->strides[k] : 0;
    }
    k_fill_u64<<<kNumSMs * 4, 256, 0, str>>>(s->hash.as<unsigned long long>(), (int64_t)tsize, kEmptyKey);
    ctx->count();
    k_ingest<CT, VT><<<blocks, threads, 0, str>>>(ndim, nnz, subs, vals, dd, s->rec_ints, allow_zero,
                                                   s->records.as<int>(), scratch.as<IngestOut>(), partials);
    ctx->count();
    k_sum_partials<<<1, 32, 0, str>>>(partials, blocks, partials + blocks);
    ctx->count();
    check_launch();
    IngestOut res;
    double frob;
    OGCP_CUDA(cudaMemcpyAsync(&res, scratch.ptr, sizeof(res), cudaMemcpyDeviceToHost, str));
    OGCP_CUDA(cudaMemcpyAsync(&frob, partials + blocks, 8, cudaMemcpyDeviceToHost, str));
    OGCP_CUDA(cudaStreamSynchronize(str));
    if (res.bad_entry != ~0ull) {
      std::vector<CT> row(ndim);
      OGCP_CUDA(cudaMemcpy(row.data(), subs + res.bad_entry * ndim, sizeof(CT) * ndim, cudaMemcpyDeviceToHost));
      std::vector<int64_t> r64(row.begin(), row.end());
      throw Error(OGCP_E_DATA, "entry " + std::to_string(res.bad_entry) + ": coordinate " +
                                   tuple_str(r64.data(), ndim, 1) + " out of bounds for dims " +
                                   tuple_str(dims, ndim, 0));
    }
    if (res.nonfinite) throw Error(OGCP_E_DATA, "stored values must be finite");
    if (res.zero) throw Error(OGCP_E_DATA, "stored values of exactly 0 are disallowed (zeros are implicit)");
    s->frob_sq = frob;
    s->x_negative = res.negative != 0;
    s->x_nonbinary = res.nonbinary != 0;
    if (nnz > 0) {
      s->filter_mask = 0;
      // prefilter (hash.cuh): >= 5 bits per key, at most 2^29 bits (64 MB, L2-resident while
      // the zero candidates are probed; c4: 1e8 keys, 5.4 bits per key -> ~10% of the absent
      // candidates still reach the table, against 31% for the earlier one-hash 32 MB bitmap)
      if (nnz >= (int64_t)1 << 20) {
        uint64_t fbits = 1 << 20;
        while (fbits < 5 * (uint64_t)nnz && fbits < ((uint64_t)1 << 29)) fbits <<= 1;
        s->filter.ensure(fbits / 8);
        OGCP_CUDA(cudaMemsetAsync(s->filter.ptr, 0, fbits / 8, str));
        s->filter_mask = fbits - 1;
      }
      k_hash_insert<<<blocks, threads, 0, str>>>(ndim, nnz, s->records.as<int>(), s->rec_ints, ss,
                                                 s->hash.as<unsigned long long>(), s->table_mask,
                                                 scratch.as<IngestOut>(),
                                                 s->filter_mask ? s->filter.as<unsigned int>() : nullptr,
                                                 s->filter_mask);
      ctx->count();
      check_launch();
      OGCP_CUDA(cudaMemcpyAsync(&res, scratch.ptr, sizeof(res), cudaMemcpyDeviceToHost, str));
      OGCP_CUDA(cudaStreamSynchronize(str));
      if (res.dup_key != ~0ull) {
        int64_t c[kMaxModes];
        uint64_t rem = res.dup_key;
        for (int k = 0; k < ndim; ++k) { c[k] = (int64_t)(rem / s->strides[k]); rem %= s->strides[k]; }
        throw Error(OGCP_E_DATA, "duplicate coordinate " + tuple_str(c, ndim, 1) + " in entry list");
      }
    }
  } catch (...) {
    delete s;
    throw;
  }
  return s;
}

template Slice* slice_create_impl<int64_t, double>(Ctx*, int, const int64_t*, int64_t, const int64_t*,
                                                   const double*, int);
template Slice* slice_create_impl<int32_t, float>(Ctx*, int, const int64_t*, int64_t, const int32_t*,
                                                  const float*, int);

__global__ void k_contains(int ndim, int64_t n, const int64_t* __restrict__ subs, Strides st, Dims dims,
                           const unsigned long long* __restrict__ table, uint64_t mask, uint8_t* hit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key = 0;
    for (int k = 0; k < ndim; ++k) key += (uint64_t)subs[i * ndim + k] * st.s[k];
    hit[i] = hash_contains(table, mask, key) ? 1 : 0;
  }
}

void slice_contains_impl(Ctx* ctx, const Slice* s, const int64_t* subs, int64_t n, uint8_t* hit) {
  if (n <= 0) return;
  Strides ss;
  Dims dd;
  for (int k = 0; k < kMaxModes; ++k) {
    ss.s[k] = k < s->ndim ? s->strides[k] : 0;
    dd.d[k] = k < s->ndim ? s->dims[k] : 1;
  }
  int blocks = std::min(ceil_div_i(n, 256), kNumSMs * 8);
  k_contains<<<blocks, 256, 0, ctx->stream>>>(s->ndim, n, subs, ss, dd, s->hash.as<unsigned long long>(),
                                               s->table_mask, hit);
  ctx->count();
  check_launch();
}

}  // namespace ogcp
