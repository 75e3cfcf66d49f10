// Lean sample walks for the dominant shape: 3-way slices whose gradient sample
// set is a merged, row-bucketed nonzero set (positions into Slice::rec_b with
// multiplicities, SamplesP::chunk_shift == 3) plus the zero stratum.  Included
// by compute.cu after the shared device helpers (mul4, dot4, dloss, ...).
//
// The generic k_sgrad / k_wgrad serve every layout (d modes, plain / merged /
// sharded / semi-stratified sets, privatised modes, split scatter) through
// per-sample runtime branches; at c4 that bookkeeping is ~390 warp
// instructions per batch of 8 samples and the kernels issue on ~45% of the
// cycles (ncu, profiles/r02_*).  These kernels fix d = 3 and the walk:
//
// * A warp takes chunks of 64 consecutive walk entries round-robin (the
//   bucketed walk of SampleStream with chunk_shift 3: all warps in flight stay
//   inside one row bucket, whose mode-1 rows then stay L2-resident).  Group g
//   (4 lanes) owns entries 8g .. 8g+7 of a chunk -- consecutive entries, so
//   mode-0 rows repeat within a group and its mode-0 contributions are summed
//   in registers per row segment (sort-by-row segmented reduction for mode 0).
// * The chunk's metadata (position, multiplicity, record) is loaded by all 32
//   lanes at once, two entries per lane arranged so that for sub-batch j every
//   group reads its sample from a lane of its own group: one shuffle per field.
// * Factor rows are double-buffered in registers: the rows of sub-batch j+1 are
//   in flight while sub-batch j is evaluated; the next chunk's metadata is
//   fetched two stages ahead.
// * Mode-1 rows and records are streamed with L1::no_allocate, so the L1 keeps
//   the rows that are reused (mode 0 within a segment, the small mode 2).
// * The zero stratum is a second launch of the same kernel over the zero rows.
//
// Reference: model_values tensor.py:203-211; LossFunction.deriv losses.py:69-78;
// sampled_mttkrp kernels.py:33-56 (x s, solvers.py:139-140);
// weight_gradient_mttkrp kernels.py:59-72; scales sampling.py:99-105.

namespace walk3 {

constexpr int kChunk = 64;  // walk entries per warp chunk (8 sub-batches of 8 samples)

__device__ __forceinline__ float4 ld_stream(const float* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int4 ld_stream_i4(const int* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Entry of chunk c held by this lane in set k (k = 0, 1): sub-batch j of group g
// is entry 8g + j, which set j>>2 holds in lane 4g + (j & 3).
__device__ __forceinline__ int64_t entry_of(int64_t c, int lane, int k) {
  return c * kChunk + 8 * (lane >> 2) + 4 * k + (lane & 3);
}

// Walk description: ZERO = false -> merged nonzeros [0, n); true -> zero rows
// [zlo, zlo + n) of this rank's share.  The counts live on the device (the
// merged distinct count, the lazy layout's row count), so every launch resolves
// them first (resolve()).
template <bool ZERO>
struct Walk {
  const int32_t* pos;    // nonzero: positions into rec
  const uint8_t* cnt;    // nonzero: multiplicities
  const int* rec;        // nonzero: 4-int records {i0, i1, i2, x}
  const int32_t* zsub;   // zero: rows [.. x 3], first coordinate -1 = rejected candidate
  const long long* n_dev;  // nullable: entry count on the device
  int64_t n_host;
  int shard_rank, shard_world;  // zero walk of a multi-GPU merged solve: this rank's contiguous share
  int64_t zlo = 0, n = 0;
  __device__ __forceinline__ void resolve() {
    const int64_t total = n_dev ? (int64_t)*n_dev : n_host;
    if (ZERO && shard_world > 1) {
      zlo = total * shard_rank / shard_world;
      n = total * (shard_rank + 1) / shard_world - zlo;
    } else {
      zlo = 0;
      n = total;
    }
  }
  __device__ __forceinline__ void load_head(int64_t c, int lane, int (&p)[2], float (&m)[2]) const {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int64_t e = entry_of(c, lane, k);
      if (ZERO) {
        p[k] = e < n ? 0 : -1;
        m[k] = 1.0f;
      } else {
        p[k] = e < n ? __ldg(pos + e) : -1;
        m[k] = e < n ? (float)__ldg(cnt + e) : 0.0f;
      }
    }
  }
  __device__ __forceinline__ void load_rec(int64_t c, int lane, const int (&p)[2], int4 (&r)[2]) const {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (p[k] < 0) {
        r[k] = make_int4(-1, 0, 0, 0);
      } else if (ZERO) {
        const int32_t* z = zsub + (zlo + entry_of(c, lane, k)) * 3;
        r[k] = make_int4(__ldg(z), __ldg(z + 1), __ldg(z + 2), 0);
      } else {
        r[k] = ld_stream_i4(rec + (int64_t)p[k] * 4);
      }
    }
  }
};

template <int V>
struct Rows {
  float4 a[3][V];
};

// One sample of a sub-batch, broadcast to its group.
struct Smp {
  int i0, i1, i2;
  float x, mult;
  bool valid;
};

template <int J>
__device__ __forceinline__ Smp pick(const int4 (&r)[2], const float (&m)[2], int lane) {
  constexpr int k = J >> 2;
  const int src = (lane & ~3) | (J & 3);
  Smp s;
  s.i0 = __shfl_sync(kFull, r[k].x, src);
  s.i1 = __shfl_sync(kFull, r[k].y, src);
  s.i2 = __shfl_sync(kFull, r[k].z, src);
  s.x = __int_as_float(__shfl_sync(kFull, r[k].w, src));
  s.mult = __shfl_sync(kFull, m[k], src);
  s.valid = s.i0 >= 0;
  return s;
}

template <int V>
__device__ __forceinline__ void load_rows(const ModelP& M, const Smp& s, int gl, Rows<V>& R) {
  const int ldr = 16 * V;
  const float4* r0 = reinterpret_cast<const float4*>(M.A[0] + (int64_t)s.i0 * ldr);
  const float* r1 = M.A[1] + (int64_t)s.i1 * ldr;
  const float4* r2 = reinterpret_cast<const float4*>(M.A[2] + (int64_t)s.i2 * ldr);
#pragma unroll
  for (int v = 0; v < V; ++v) {
    if (s.valid) {
      R.a[0][v] = __ldg(r0 + v * 4 + gl);
      R.a[1][v] = ld_stream(r1 + (v * 4 + gl) * 4);
      R.a[2][v] = __ldg(r2 + v * 4 + gl);
    } else {
      R.a[0][v] = R.a[1][v] = R.a[2][v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// y = scale * d f / d m at the sample, m = <a0 o a1 o a2, s> (group-reduced).
template <int V>
__device__ __forceinline__ float sample_y(const Rows<V>& R, const float4 (&s4)[V], const Smp& s, const LossP& L,
                                          float scale, unsigned& bits, float4 (&p01)[V]) {
  float part = 0.0f;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    p01[v] = mul4(R.a[0][v], R.a[1][v]);
    part += dot4(mul4(p01[v], R.a[2][v]), s4[v]);
  }
  part += __shfl_xor_sync(kFull, part, 1);
  part += __shfl_xor_sync(kFull, part, 2);
  if (!s.valid) return 0.0f;
  bits |= domain_bits(L.kind, part);
  return dloss(L.kind, s.x, part, L.eps) * scale;
}

// ---------------------------------------------------------------- K2+K3
template <int V, bool ZERO>
__global__ void __launch_bounds__(kThreads, 2) k_sgrad3(Walk<ZERO> W, ModelP M, const float* __restrict__ s_f,
                                                       LossP L, float scale, GradPtrs GP, DevFlags* flags,
                                                       long long code) {
  const int lane = threadIdx.x & 31;
  const int gl = lane & 3;
  const int ldr = 16 * V;
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * 4 + gl);
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  W.resolve();
  const int64_t nchunks = (W.n + kChunk - 1) / kChunk;
  unsigned bits = 0;
  int seg_row = -1;
  float4 seg[V];
#pragma unroll
  for (int v = 0; v < V; ++v) seg[v] = make_float4(0.f, 0.f, 0.f, 0.f);

  auto scatter = [&](const Smp& s, const Rows<V>& R) {
    float4 p01[V];
    const float y = sample_y<V>(R, s4, s, L, ZERO ? scale : scale * s.mult, bits, p01);
    if (!s.valid) return;
    if (s.i0 != seg_row) {
      if (seg_row >= 0) {
#pragma unroll
        for (int v = 0; v < V; ++v) red_add_v4(GP.g[0] + (int64_t)seg_row * ldr + (v * 4 + gl) * 4, seg[v]);
      }
      seg_row = s.i0;
#pragma unroll
      for (int v = 0; v < V; ++v) seg[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float* g1 = GP.g[1] + (int64_t)s.i1 * ldr;
    float* g2 = GP.g[2] + (int64_t)s.i2 * ldr;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float4 ys = make_float4(y * s4[v].x, y * s4[v].y, y * s4[v].z, y * s4[v].w);
      const float4 t = mul4(ys, R.a[2][v]);   // y s o a2
      const float4 c0 = mul4(t, R.a[1][v]);   // mode 0: y s o a1 o a2
      seg[v].x += c0.x;
      seg[v].y += c0.y;
      seg[v].z += c0.z;
      seg[v].w += c0.w;
      red_add_v4(g1 + (v * 4 + gl) * 4, mul4(t, R.a[0][v]));  // mode 1: y s o a0 o a2
      red_add_v4(g2 + (v * 4 + gl) * 4, mul4(ys, p01[v]));    // mode 2: y s o a0 o a1
    }
  };

  int64_t c = warp;
  int pos[2];
  float mult[2], mult_n[2];
  int4 rec[2], rec_n[2];
  if (c < nchunks) {
    W.load_head(c, lane, pos, mult);
    W.load_rec(c, lane, pos, rec);
  }
  Rows<V> Ra, Rb;
  Smp sa, sb;
  if (c < nchunks) {
    sa = pick<0>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
  }
  for (; c < nchunks; c += nwarps) {
    const int64_t cn = c + nwarps;
    const bool more = cn < nchunks;
    if (more) W.load_head(cn, lane, pos, mult_n);
    // sub-batches 0..7, rows of the next sub-batch in flight while this one is evaluated
    sb = pick<1>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    scatter(sa, Ra);
    sa = pick<2>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
    scatter(sb, Rb);
    sb = pick<3>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    scatter(sa, Ra);
    if (more) W.load_rec(cn, lane, pos, rec_n);
    sa = pick<4>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
    scatter(sb, Rb);
    sb = pick<5>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    scatter(sa, Ra);
    sa = pick<6>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
    scatter(sb, Rb);
    sb = pick<7>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    scatter(sa, Ra);
    if (more) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        rec[k] = rec_n[k];
        mult[k] = mult_n[k];
      }
      sa = pick<0>(rec, mult, lane);
      load_rows<V>(M, sa, gl, Ra);
    }
    scatter(sb, Rb);
  }
  if (seg_row >= 0) {
#pragma unroll
    for (int v = 0; v < V; ++v) red_add_v4(GP.g[0] + (int64_t)seg_row * ldr + (v * 4 + gl) * 4, seg[v]);
  }
  if (bits) report(flags, kFlagData, code, bits);
}

// ---------------------------------------------------------------- K2 (weights)
// Z' vec(Y): per-lane fp32 sums per chunk, fp64 across chunks, then lanes with
// the same columns and the block's warps in fixed order (deterministic).
template <int V, bool ZERO>
__global__ void __launch_bounds__(kThreads, 2) k_wgrad3(Walk<ZERO> W, ModelP M, const float* __restrict__ s_f,
                                                       LossP L, float scale, double* __restrict__ partials,
                                                       DevFlags* flags, long long code) {
  __shared__ double red[kThreads / 32][16 * V];
  const int lane = threadIdx.x & 31;
  const int gl = lane & 3;
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * 4 + gl);
  double acc[V][4];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v][0] = acc[v][1] = acc[v][2] = acc[v][3] = 0.0;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  W.resolve();
  const int64_t nchunks = (W.n + kChunk - 1) / kChunk;
  unsigned bits = 0;
  float4 part[V];
#pragma unroll
  for (int v = 0; v < V; ++v) part[v] = make_float4(0.f, 0.f, 0.f, 0.f);

  auto accumulate = [&](const Smp& s, const Rows<V>& R) {
    float4 p01[V];
    const float y = sample_y<V>(R, s4, s, L, ZERO ? scale : scale * s.mult, bits, p01);
    if (!s.valid) return;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const float4 pr = mul4(p01[v], R.a[2][v]);
      part[v].x += y * pr.x;
      part[v].y += y * pr.y;
      part[v].z += y * pr.z;
      part[v].w += y * pr.w;
    }
  };

  int64_t c = warp;
  int pos[2];
  float mult[2], mult_n[2];
  int4 rec[2], rec_n[2];
  if (c < nchunks) {
    W.load_head(c, lane, pos, mult);
    W.load_rec(c, lane, pos, rec);
  }
  Rows<V> Ra, Rb;
  Smp sa, sb;
  if (c < nchunks) {
    sa = pick<0>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
  }
  for (; c < nchunks; c += nwarps) {
    const int64_t cn = c + nwarps;
    const bool more = cn < nchunks;
    if (more) W.load_head(cn, lane, pos, mult_n);
    sb = pick<1>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    accumulate(sa, Ra);
    sa = pick<2>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
    accumulate(sb, Rb);
    sb = pick<3>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    accumulate(sa, Ra);
    if (more) W.load_rec(cn, lane, pos, rec_n);
    sa = pick<4>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
    accumulate(sb, Rb);
    sb = pick<5>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    accumulate(sa, Ra);
    sa = pick<6>(rec, mult, lane);
    load_rows<V>(M, sa, gl, Ra);
    accumulate(sb, Rb);
    sb = pick<7>(rec, mult, lane);
    load_rows<V>(M, sb, gl, Rb);
    accumulate(sa, Ra);
    if (more) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        rec[k] = rec_n[k];
        mult[k] = mult_n[k];
      }
      sa = pick<0>(rec, mult, lane);
      load_rows<V>(M, sa, gl, Ra);
    }
    accumulate(sb, Rb);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      acc[v][0] += (double)part[v].x;
      acc[v][1] += (double)part[v].y;
      acc[v][2] += (double)part[v].z;
      acc[v][3] += (double)part[v].w;
      part[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (bits) report(flags, kFlagData, code, bits);
#pragma unroll
  for (int o = 4; o < 32; o <<= 1)
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[v][e] += __shfl_xor_sync(kFull, acc[v][e], o);
  const int w = threadIdx.x >> 5;
  if (lane < 4) {
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
      for (int e = 0; e < 4; ++e) red[w][(v * 4 + lane) * 4 + e] = acc[v][e];
  }
  __syncthreads();
  for (int c2 = threadIdx.x; c2 < 16 * V; c2 += blockDim.x) {
    double t = 0.0;
    for (int j = 0; j < kThreads / 32; ++j) t += red[j][c2];
    partials[blockIdx.x * (int64_t)(16 * V) + c2] = t;
  }
}

}  // namespace walk3
