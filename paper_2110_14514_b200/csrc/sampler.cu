// K1 sampler: bit-exact, counter-based replay of the reference's stratified
// draws (draw_samples, sampling.py:108-153) on the GPU.
//
// A keyed Generator (rng_at, sampling.py:39-42) is a stream of 32-bit words
// (pcg64.cuh).  Each bounded draw integers(0, n) consumes words until one
// passes the Lemire test; the array-bound call integers(0, dims, (rows, d))
// cycles through the word-consuming columns in row-major order.  A word's
// acceptance depends on which column it serves, so the stream is cut into
// chunks of kChunkWords words and every chunk is summarised by a map
// "start column c -> number of elements emitted" (NCOL entries).  Maps compose
// associatively, so one parallel scan gives every chunk its start column and
// output offset, and a second pass re-generates the words and writes the
// accepted values in place.  The nonzero stratum is the NCOL = 1 case.
//
// Zero stratum (sampling.py:133-150): rejection rounds of `need` candidate
// rows continue the same word stream, so the accepted zeros are exactly the
// first q candidate rows that miss the nonzero set, and the budget test
// "rejected > budget" fires iff more than `budget` hits precede the q-th miss.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "hash.cuh"
#include "sampler.cuh"

namespace ogcp {

constexpr int kChunkWords = 128;   // words per thread-chunk (CW)
constexpr int kScanThreads = 256;  // chunks per block
constexpr int kMaxCols = 7;

struct JumpTable {
  u128 A[64];
  u128 B[64];
};
__constant__ JumpTable c_jump;

void init_jump_table() {
  static bool done[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && done[dev]) return;
  JumpTable h;
  Jump cur;
  cur.A = pcg_mult();
  cur.B = 1;
  for (int k = 0; k < 64; ++k) {
    h.A[k] = cur.A;
    h.B[k] = cur.B;
    cur = jump_compose(cur, cur);
  }
  OGCP_CUDA(cudaMemcpyToSymbol(c_jump, &h, sizeof(h)));
  if (dev >= 0 && dev < 64) done[dev] = true;
}

struct StreamSpec {
  unsigned long long st_hi, st_lo, inc_hi, inc_lo;
  int ncol;
  uint32_t n[kMaxCols];
  uint32_t thr[kMaxCols];
};

// Word generator positioned at word index w of a fresh Generator.
struct WordGen {
  u128 st, inc;
  uint64_t out;
  int half;
  __device__ __forceinline__ void init(const StreamSpec& sp, uint64_t w) {
    u128 s0 = ((u128)sp.st_hi << 64) | sp.st_lo;
    inc = ((u128)sp.inc_hi << 64) | sp.inc_lo;
    uint64_t n = (w >> 1) + 1;  // state after output (w>>1) = n steps
    u128 A = 1, B = 0;
    for (int k = 0; n; ++k, n >>= 1)
      if (n & 1ull) {
        A = A * c_jump.A[k];
        B = B * c_jump.A[k] + c_jump.B[k];
      }
    st = A * s0 + inc * B;
    out = pcg_output(st);
    half = (int)(w & 1ull);
  }
  __device__ __forceinline__ uint32_t next() {
    uint32_t r;
    if (half) {
      r = (uint32_t)(out >> 32);
      st = st * pcg_mult() + inc;
      out = pcg_output(st);
    } else {
      r = (uint32_t)out;
    }
    half ^= 1;
    return r;
  }
};

template <int NCOL>
struct Map {
  uint32_t c[NCOL];
};

// f then g
template <int NCOL>
__device__ __forceinline__ Map<NCOL> compose(const Map<NCOL>& f, const Map<NCOL>& g) {
  Map<NCOL> h;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    uint32_t adv = f.c[c];
    int cc = (int)((c + adv) % NCOL);
    uint32_t gv = g.c[0];
#pragma unroll
    for (int j = 1; j < NCOL; ++j)
      if (j == cc) gv = g.c[j];
    h.c[c] = adv + gv;
  }
  return h;
}

template <int NCOL>
__device__ __forceinline__ Map<NCOL> identity_map() {
  Map<NCOL> m;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) m.c[c] = 0;
  return m;
}

// Block-wide scan of maps (Hillis-Steele over kScanThreads threads).
template <int NCOL>
__device__ void block_scan_maps(Map<NCOL> mine, Map<NCOL>& excl, Map<NCOL>& agg) {
  __shared__ uint32_t buf[2][kScanThreads][NCOL];
  int tid = threadIdx.x;
  int cur = 0;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) buf[0][tid][c] = mine.c[c];
  __syncthreads();
  for (int off = 1; off < kScanThreads; off <<= 1) {
    Map<NCOL> me, other;
#pragma unroll
    for (int c = 0; c < NCOL; ++c) me.c[c] = buf[cur][tid][c];
    if (tid >= off) {
#pragma unroll
      for (int c = 0; c < NCOL; ++c) other.c[c] = buf[cur][tid - off][c];
      me = compose<NCOL>(other, me);
    }
#pragma unroll
    for (int c = 0; c < NCOL; ++c) buf[cur ^ 1][tid][c] = me.c[c];
    cur ^= 1;
    __syncthreads();
  }
  if (tid == 0) excl = identity_map<NCOL>();
  else {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) excl.c[c] = buf[cur][tid - 1][c];
  }
#pragma unroll
  for (int c = 0; c < NCOL; ++c) agg.c[c] = buf[cur][kScanThreads - 1][c];
  __syncthreads();
}

__device__ __forceinline__ uint64_t start_word(const long long* w0p, int64_t chunk) {
  return (uint64_t)(w0p ? *w0p : 0) + (uint64_t)chunk * kChunkWords;
}

// Pass 1: per-chunk maps + per-block aggregate maps.
template <int NCOL>
__global__ void __launch_bounds__(kScanThreads) k_draw_count(StreamSpec sp, const long long* w0p, int64_t nchunks,
                                                             uint8_t* __restrict__ tmaps,
                                                             uint32_t* __restrict__ bagg) {
  int64_t chunk = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  Map<NCOL> m = identity_map<NCOL>();
  if (chunk < nchunks) {
    WordGen g;
    g.init(sp, start_word(w0p, chunk));
    int col[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) col[c] = c;
    for (int i = 0; i < kChunkWords; ++i) {
      uint32_t w = g.next();
#pragma unroll
      for (int c = 0; c < NCOL; ++c) {
        int cc = col[c];
        uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
        for (int j = 1; j < NCOL; ++j)
          if (j == cc) { n = sp.n[j]; thr = sp.thr[j]; }
        uint64_t prod = (uint64_t)w * n;
        if ((uint32_t)prod >= thr) {
          m.c[c] += 1;
          col[c] = cc + 1 == NCOL ? 0 : cc + 1;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NCOL; ++c) tmaps[chunk * NCOL + c] = (uint8_t)m.c[c];
  }
  Map<NCOL> excl, agg;
  block_scan_maps<NCOL>(m, excl, agg);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) bagg[blockIdx.x * (int64_t)NCOL + c] = agg.c[c];
  }
}

// Pass 2: exclusive scan of block aggregates (one block, tiles of kScanThreads)
// -> per-block start (column, element offset); total elements emitted.
template <int NCOL>
__global__ void __launch_bounds__(kScanThreads) k_draw_scan_blocks(const uint32_t* __restrict__ bagg, int64_t nblocks,
                                                                   long long* __restrict__ bstart,
                                                                   long long* __restrict__ total_out) {
  __shared__ long long carry_elem;
  __shared__ int carry_col;
  if (threadIdx.x == 0) { carry_elem = 0; carry_col = 0; }
  __syncthreads();
  for (int64_t base = 0; base < nblocks; base += kScanThreads) {
    int64_t b = base + threadIdx.x;
    Map<NCOL> m = identity_map<NCOL>();
    if (b < nblocks) {
#pragma unroll
      for (int c = 0; c < NCOL; ++c) m.c[c] = bagg[b * NCOL + c];
    }
    Map<NCOL> excl, agg;
    block_scan_maps<NCOL>(m, excl, agg);
    long long ce = carry_elem;
    int cc = carry_col;
    if (b < nblocks) {
      uint32_t adv = excl.c[0];
#pragma unroll
      for (int j = 1; j < NCOL; ++j)
        if (j == cc) adv = excl.c[j];
      bstart[b * 2 + 0] = (cc + adv) % NCOL;
      bstart[b * 2 + 1] = ce + adv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t adv = agg.c[0];
#pragma unroll
      for (int j = 1; j < NCOL; ++j)
        if (j == cc) adv = agg.c[j];
      carry_elem = ce + adv;
      carry_col = (int)((cc + adv) % NCOL);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = carry_elem;
}

// Pass 3: re-generate the words and write accepted values at their offsets.
// NCOL == 1 (nonzero stratum): out[e] = value, end word of element target-1.
// NCOL  > 1 (zero candidates):  out[e] = value (row-major [row][NCOL]).
template <int NCOL>
__global__ void __launch_bounds__(kScanThreads) k_draw_write(StreamSpec sp, const long long* w0p, int64_t nchunks,
                                                             const uint8_t* __restrict__ tmaps,
                                                             const long long* __restrict__ bstart,
                                                             int64_t target, int32_t* __restrict__ out,
                                                             long long* __restrict__ end_word) {
  int64_t chunk = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  Map<NCOL> m = identity_map<NCOL>();
  if (chunk < nchunks) {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) m.c[c] = tmaps[chunk * NCOL + c];
  }
  Map<NCOL> excl, agg;
  block_scan_maps<NCOL>(m, excl, agg);
  if (chunk >= nchunks) return;
  int bcol = (int)bstart[blockIdx.x * 2 + 0];
  long long e = bstart[blockIdx.x * 2 + 1];
  uint32_t adv = excl.c[0];
#pragma unroll
  for (int j = 1; j < NCOL; ++j)
    if (j == bcol) adv = excl.c[j];
  e += adv;
  int col = (int)((bcol + adv) % NCOL);
  if (e >= target) return;
  uint64_t w = start_word(w0p, chunk);
  WordGen g;
  g.init(sp, w);
  for (int i = 0; i < kChunkWords && e < target; ++i, ++w) {
    uint32_t word = g.next();
    uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
    for (int j = 1; j < NCOL; ++j)
      if (j == col) { n = sp.n[j]; thr = sp.thr[j]; }
    uint64_t prod = (uint64_t)word * n;
    if ((uint32_t)prod >= thr) {
      out[e] = (int32_t)(prod >> 32);
      if (e == target - 1 && end_word) *end_word = (long long)(w + 1);
      ++e;
      col = col + 1 == NCOL ? 0 : col + 1;
    }
  }
}

// Zero stratum: hit test of candidate rows against the nonzero hash; per-block
// miss counts.
__device__ __forceinline__ void assemble_row(const int32_t* __restrict__ cand, int64_t r, int ncol,
                                             const int* colmap, int ndim, int32_t* c) {
  for (int k = 0; k < ndim; ++k) c[k] = colmap[k] < 0 ? 0 : cand[r * ncol + colmap[k]];
}

struct ZeroSpec {
  int ndim, ncol;
  int colmap[kMaxModes];
  Strides st;
};

__global__ void __launch_bounds__(kScanThreads) k_zero_hits(ZeroSpec zs, const int32_t* __restrict__ cand,
                                                            const long long* __restrict__ elems_avail,
                                                            int64_t rows_max,
                                                            const unsigned long long* __restrict__ table,
                                                            uint64_t mask, uint8_t* __restrict__ miss,
                                                            uint32_t* __restrict__ bcount) {
  int64_t r = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  int64_t rows = zs.ncol ? min(rows_max, (int64_t)(*elems_avail / zs.ncol)) : rows_max;
  uint32_t ms = 0;
  if (r < rows) {
    int32_t c[kMaxModes];
    assemble_row(cand, r, zs.ncol, zs.colmap, zs.ndim, c);
    uint64_t key = 0;
    for (int k = 0; k < zs.ndim; ++k) key += (uint64_t)(uint32_t)c[k] * zs.st.s[k];
    ms = table ? (hash_contains(table, mask, key) ? 0u : 1u) : 1u;
  }
  if (r < rows_max) miss[r] = (uint8_t)ms;
  uint32_t tot = __syncthreads_count(ms);
  if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_zero_scan(const uint32_t* __restrict__ bcount, int64_t nblocks,
                                                            long long* __restrict__ boff,
                                                            long long* __restrict__ total) {
  __shared__ long long carry;
  __shared__ long long tmp[kScanThreads];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nblocks; base += kScanThreads) {
    int64_t b = base + threadIdx.x;
    long long v = b < nblocks ? bcount[b] : 0;
    tmp[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < kScanThreads; off <<= 1) {
      long long o = threadIdx.x >= off ? tmp[threadIdx.x - off] : 0;
      __syncthreads();
      tmp[threadIdx.x] += o;
      __syncthreads();
    }
    if (b < nblocks) boff[b] = carry + tmp[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += tmp[kScanThreads - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Compact the first q misses into zero_subs (int32 [q x ndim]); the thread that
// writes miss number q-1 records how many hits preceded it.
__global__ void __launch_bounds__(kScanThreads) k_zero_compact(ZeroSpec zs, const int32_t* __restrict__ cand,
                                                               int64_t rows_max, const uint8_t* __restrict__ miss,
                                                               const long long* __restrict__ boff, int64_t q,
                                                               int32_t* __restrict__ zero_subs,
                                                               long long* __restrict__ hits_before) {
  __shared__ uint32_t tmp[kScanThreads];
  int64_t r = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  uint32_t ms = r < rows_max ? miss[r] : 0;
  tmp[threadIdx.x] = ms;
  __syncthreads();
  for (int off = 1; off < kScanThreads; off <<= 1) {
    uint32_t o = threadIdx.x >= off ? tmp[threadIdx.x - off] : 0;
    __syncthreads();
    tmp[threadIdx.x] += o;
    __syncthreads();
  }
  if (!ms) return;
  long long rank = boff[blockIdx.x] + tmp[threadIdx.x] - 1;
  if (rank >= q) return;
  int32_t c[kMaxModes];
  assemble_row(cand, r, zs.ncol, zs.colmap, zs.ndim, c);
  for (int k = 0; k < zs.ndim; ++k) zero_subs[rank * zs.ndim + k] = c[k];
  if (rank == q - 1) *hits_before = (long long)(r - rank);
}

// Final status: shortfall (need more candidates) or budget exhaustion.
__global__ void k_draw_status(int64_t p, const long long* nz_avail, int64_t q, const long long* z_misses,
                              const long long* z_rows_total, int64_t rows_max, int ncol,
                              const long long* z_elems, const long long* hits_before, long long budget,
                              long long code, DevFlags* flags) {
  if (threadIdx.x || blockIdx.x) return;
  bool shortfall = false, exhausted = false;
  if (p > 0 && nz_avail && *nz_avail < p) shortfall = true;
  if (q > 0) {
    long long rows = ncol ? min((long long)rows_max, *z_elems / ncol) : rows_max;
    long long misses = *z_misses;
    if (misses >= q) {
      if (*hits_before > budget) exhausted = true;
    } else {
      long long hits = rows - misses;
      if (hits > budget) exhausted = true;
      else shortfall = true;
    }
  }
  (void)z_rows_total;
  if (exhausted) atomicMin(&flags->first_code[kFlagSampling], code);
  else if (shortfall) atomicMin(&flags->first_code[kFlagShortfall], code);
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_set_ll(long long* p, long long v) { *p = v; }

template <int NCOL>
static void run_stream(Ctx* ctx, const StreamSpec& sp, const long long* w0, int64_t target, int64_t words,
                       int32_t* out, long long* end_word, long long* elems_total, DrawScratch& scr) {
  int64_t nchunks = std::max<int64_t>(1, (words + kChunkWords - 1) / kChunkWords);
  int64_t nblocks = (nchunks + kScanThreads - 1) / kScanThreads;
  uint8_t* tmaps = scr.tmaps.as<uint8_t>();
  scr.tmaps.ensure((size_t)nchunks * NCOL);
  tmaps = scr.tmaps.as<uint8_t>();
  scr.bagg.ensure((size_t)nblocks * NCOL * 4);
  scr.bstart.ensure((size_t)nblocks * 16);
  cudaStream_t s = ctx->stream;
  k_draw_count<NCOL><<<(unsigned)nblocks, kScanThreads, 0, s>>>(sp, w0, nchunks, tmaps, scr.bagg.as<uint32_t>());
  k_draw_scan_blocks<NCOL><<<1, kScanThreads, 0, s>>>(scr.bagg.as<uint32_t>(), nblocks,
                                                      scr.bstart.as<long long>(), elems_total);
  k_draw_write<NCOL><<<(unsigned)nblocks, kScanThreads, 0, s>>>(sp, w0, nchunks, tmaps,
                                                                scr.bstart.as<long long>(), target, out, end_word);
  ctx->count(3);
  check_launch();
}

static void run_stream_dispatch(int ncol, Ctx* ctx, const StreamSpec& sp, const long long* w0, int64_t target,
                                int64_t words, int32_t* out, long long* end_word, long long* elems_total,
                                DrawScratch& scr) {
  switch (ncol) {
    case 1: run_stream<1>(ctx, sp, w0, target, words, out, end_word, elems_total, scr); break;
    case 2: run_stream<2>(ctx, sp, w0, target, words, out, end_word, elems_total, scr); break;
    case 3: run_stream<3>(ctx, sp, w0, target, words, out, end_word, elems_total, scr); break;
    case 4: run_stream<4>(ctx, sp, w0, target, words, out, end_word, elems_total, scr); break;
    case 5: run_stream<5>(ctx, sp, w0, target, words, out, end_word, elems_total, scr); break;
    case 6: run_stream<6>(ctx, sp, w0, target, words, out, end_word, elems_total, scr); break;
    case 7: run_stream<7>(ctx, sp, w0, target, words, out, end_word, elems_total, scr); break;
    default: throw Error(OGCP_E_USAGE, "too many modes for the sampler");
  }
}

static double reject_rate(uint32_t n) { return (double)lemire_threshold(n) / 4294967296.0; }

// Enqueue one stratified draw.  ordinals: int32 [p]; zero_subs: int32 [q x ndim].
// code: event code (event*4) recorded on sampling errors / shortfall.
void draw_enqueue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget,
                  int32_t* ordinals, int32_t* zero_subs, long long code, DrawScratch& scr) {
  init_jump_table();
  ProfScope prof_scope(ctx, kProfDraw);
  const int d = X->ndim;
  const int64_t eta = X->nnz;
  cudaStream_t s = ctx->stream;
  scr.scal.ensure(16 * 8);
  long long* sc = scr.scal.as<long long>();
  long long* nz_end = sc + 0;
  long long* nz_avail = sc + 1;
  long long* z_elems = sc + 2;
  long long* z_misses = sc + 3;
  long long* z_hits_before = sc + 4;
  OGCP_CUDA(cudaMemsetAsync(sc, 0, 16 * 8, s));
  StreamSpec sp;
  sp.st_hi = (unsigned long long)(g.state >> 64);
  sp.st_lo = (unsigned long long)g.state;
  sp.inc_hi = (unsigned long long)(g.inc >> 64);
  sp.inc_lo = (unsigned long long)g.inc;
  const double slack = ctx->slack;

  // ---- nonzero stratum: integers(0, eta, size=p)  (sampling.py:125)
  bool nz_stream = false;
  if (p > 0) {
    if (eta == 1) {
      k_fill_i32<<<std::min(ceil_div_i(p, 256), kNumSMs * 4), 256, 0, s>>>(ordinals, p, 0);
      ctx->count();
    } else {
      sp.ncol = 1;
      sp.n[0] = (uint32_t)eta;
      sp.thr[0] = lemire_threshold((uint32_t)eta);
      double r = reject_rate((uint32_t)eta);
      double exp_words = (double)p / (1.0 - r);
      double sd = std::sqrt((double)p * r) / (1.0 - r);
      int64_t words = (int64_t)((exp_words + 10.0 * sd + 2048.0) * slack);
      run_stream_dispatch(1, ctx, sp, nullptr, p, words, ordinals, nz_end, nz_avail, scr);
      nz_stream = true;
    }
  }

  // ---- zero stratum: rounds of integers(0, dims, (need, d)) + rejection (sampling.py:133-150)
  int ncol = 0;
  ZeroSpec zs;
  zs.ndim = d;
  for (int k = 0; k < kMaxModes; ++k) {
    zs.colmap[k] = -1;
    zs.st.s[k] = k < d ? X->strides[k] : 0;
  }
  int64_t rows_max = 0;
  if (q > 0) {
    double rmax = 0.0;
    for (int k = 0; k < d; ++k)
      if (X->dims[k] > 1) {
        sp.n[ncol] = (uint32_t)X->dims[k];
        sp.thr[ncol] = lemire_threshold((uint32_t)X->dims[k]);
        rmax = std::max(rmax, reject_rate((uint32_t)X->dims[k]));
        zs.colmap[k] = ncol++;
      }
    zs.ncol = ncol;
    sp.ncol = ncol;
    double rho = X->omega_d > 0 ? (double)eta / X->omega_d : 0.0;
    double exp_rows = rho < 1.0 ? (double)q / (1.0 - rho) : 1e30;
    double sd_rows = rho < 1.0 ? std::sqrt((double)q * rho) / (1.0 - rho) : 1e30;
    double want = (exp_rows + 10.0 * sd_rows + 64.0) * slack;
    double cap = (double)q + (double)budget + 1.0;
    rows_max = (int64_t)std::min(want, cap);
    if (rows_max < q) rows_max = q;
    scr.miss.ensure((size_t)rows_max);
    int64_t zblocks = (rows_max + kScanThreads - 1) / kScanThreads;
    scr.zcount.ensure((size_t)zblocks * 4);
    scr.zoff.ensure((size_t)zblocks * 8);
    const unsigned long long* table = eta > 0 ? X->hash.as<unsigned long long>() : nullptr;
    if (ncol > 0) {
      int64_t target = rows_max * ncol;
      scr.cand.ensure((size_t)target * 4);
      double exp_words = (double)target / (1.0 - rmax);
      double sd = std::sqrt((double)target * rmax) / (1.0 - rmax);
      int64_t words = (int64_t)((exp_words + 10.0 * sd + 2048.0) * slack);
      const long long* w0 = nz_stream ? nz_end : nullptr;
      run_stream_dispatch(ncol, ctx, sp, w0, target, words, scr.cand.as<int32_t>(), nullptr, z_elems, scr);
    } else {
      // every mode has size 1: each candidate is the origin and no words are consumed
      k_set_ll<<<1, 1, 0, s>>>(z_elems, 0);
      ctx->count();
    }
    k_zero_hits<<<(unsigned)zblocks, kScanThreads, 0, s>>>(zs, scr.cand.as<int32_t>(), z_elems, rows_max, table,
                                                           X->table_mask, scr.miss.as<uint8_t>(),
                                                           scr.zcount.as<uint32_t>());
    k_zero_scan<<<1, kScanThreads, 0, s>>>(scr.zcount.as<uint32_t>(), zblocks, scr.zoff.as<long long>(), z_misses);
    k_zero_compact<<<(unsigned)zblocks, kScanThreads, 0, s>>>(zs, scr.cand.as<int32_t>(), rows_max,
                                                              scr.miss.as<uint8_t>(), scr.zoff.as<long long>(), q,
                                                              zero_subs, z_hits_before);
    ctx->count(3);
  }
  k_draw_status<<<1, 1, 0, s>>>(nz_stream ? p : 0, nz_avail, q, z_misses, nullptr, rows_max, ncol, z_elems,
                                z_hits_before, (long long)budget, code, ctx->flags.as<DevFlags>());
  ctx->count();
  check_launch();
}

}  // namespace ogcp
