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
// accepted values.  The nonzero stratum is the NCOL = 1 case.
//
// Each block covers kScanThreads consecutive chunks.  Its first thread jumps
// the LCG to the block's first word (O(log n) 128-bit multiply-adds against a
// power-of-two table); every thread then applies a precomputed local jump of
// tid*kChunkWords/2 steps.  Accepted values are staged in shared memory and
// written to HBM with coalesced stores.
//
// Zero stratum (sampling.py:133-150): rejection rounds of `need` candidate
// rows continue the same word stream, so the accepted zeros are exactly the
// first q candidate rows that miss the nonzero set, and the budget test
// "rejected > budget" fires iff more than `budget` hits precede the q-th miss.
#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include <cub/cub.cuh>

#include "common.cuh"
#include "hash.cuh"
#include "sampler.cuh"
#include "comm.cuh"

namespace ogcp {

constexpr int kChunkWords = 32;    // words per thread-chunk
constexpr int kScanThreads = 256;  // chunks per block
constexpr int kBlockWords = kChunkWords * kScanThreads;
constexpr int kMaxCols = 7;
constexpr int kRowsPerThread = 8;  // zero-candidate rows per thread in the hit/compact passes
constexpr int kRowsPerBlock = kRowsPerThread * kScanThreads;

struct JumpTable {
  u128 A[64];
  u128 B[64];
};
__constant__ JumpTable c_jump;
// local jumps by t * kChunkWords/2 LCG steps, t < kScanThreads
__device__ u128 g_local_A[kScanThreads];
__device__ u128 g_local_B[kScanThreads];

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
  std::vector<u128> la(kScanThreads), lb(kScanThreads);
  for (int t = 0; t < kScanThreads; ++t) {
    Jump j = jump_pow((uint64_t)t * (kChunkWords / 2));
    la[t] = j.A;
    lb[t] = j.B;
  }
  OGCP_CUDA(cudaMemcpyToSymbol(g_local_A, la.data(), sizeof(u128) * kScanThreads));
  OGCP_CUDA(cudaMemcpyToSymbol(g_local_B, lb.data(), sizeof(u128) * kScanThreads));
  if (dev >= 0 && dev < 64) done[dev] = true;
}

struct StreamSpec {
  unsigned long long st_hi, st_lo, inc_hi, inc_lo;
  int ncol;
  uint32_t n[kMaxCols];
  uint32_t thr[kMaxCols];
};

// LCG state after `steps` steps from the seeded state (power-of-two table).
__device__ __forceinline__ u128 state_after(const StreamSpec& sp, uint64_t steps) {
  const u128 s0 = ((u128)sp.st_hi << 64) | sp.st_lo;
  const u128 inc = ((u128)sp.inc_hi << 64) | sp.inc_lo;
  u128 A = 1, B = 0;
  for (int k = 0; steps; ++k, steps >>= 1)
    if (steps & 1ull) {
      A = A * c_jump.A[k];
      B = B * c_jump.A[k] + c_jump.B[k];
    }
  return A * s0 + inc * B;
}

// Word generator for this thread's chunk.  Block base state is computed once
// per block (thread 0) and shared; the thread applies its local jump.
struct WordGen {
  u128 st, inc;
  uint64_t out;
  int half;
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

__device__ __forceinline__ uint64_t tile_word0(const long long* w0p, int64_t tile) {
  return (uint64_t)(w0p ? *w0p : 0) + (uint64_t)tile * kBlockWords;
}
__device__ __forceinline__ uint64_t block_word0(const long long* w0p) { return tile_word0(w0p, blockIdx.x); }

// All threads of the block call this (contains __syncthreads).  Tile `tile` of the
// stream = words [tile * kBlockWords, (tile + 1) * kBlockWords) after w0.
__device__ __forceinline__ WordGen tile_wordgen(const StreamSpec& sp, const long long* w0p, int64_t tile) {
  __shared__ unsigned long long base[2];
  const uint64_t wb = tile_word0(w0p, tile);
  if (threadIdx.x == 0) {
    const u128 s = state_after(sp, (wb >> 1) + 1);
    base[0] = (unsigned long long)(s >> 64);
    base[1] = (unsigned long long)s;
  }
  __syncthreads();
  WordGen g;
  g.inc = ((u128)sp.inc_hi << 64) | sp.inc_lo;
  const u128 sb = ((u128)base[0] << 64) | base[1];
  const u128 A = g_local_A[threadIdx.x], B = g_local_B[threadIdx.x];
  g.st = A * sb + g.inc * B;
  g.out = pcg_output(g.st);
  g.half = (int)(wb & 1ull);  // chunk starts share the block's word parity (kChunkWords even)
  return g;
}
__device__ __forceinline__ WordGen block_wordgen(const StreamSpec& sp, const long long* w0p) {
  return tile_wordgen(sp, w0p, blockIdx.x);
}

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

template <int NCOL>
__device__ __forceinline__ Map<NCOL> shfl_up_map(const Map<NCOL>& m, int d) {
  Map<NCOL> r;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) r.c[c] = __shfl_up_sync(0xffffffffu, m.c[c], d);
  return r;
}

// Block-wide exclusive scan of maps: warp shuffles, then one warp scans the
// 8 warp aggregates.
template <int NCOL>
__device__ void block_scan_maps(Map<NCOL> mine, Map<NCOL>& excl, Map<NCOL>& agg) {
  __shared__ uint32_t wagg[kScanThreads / 32][NCOL];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Map<NCOL> inc = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Map<NCOL> o = shfl_up_map<NCOL>(inc, d);
    if (lane >= d) inc = compose<NCOL>(o, inc);
  }
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) wagg[w][c] = inc.c[c];
  }
  __syncthreads();
  // prefix over preceding warps (at most 7 compositions)
  Map<NCOL> pre = identity_map<NCOL>();
  for (int j = 0; j < w; ++j) {
    Map<NCOL> a;
#pragma unroll
    for (int c = 0; c < NCOL; ++c) a.c[c] = wagg[j][c];
    pre = compose<NCOL>(pre, a);
  }
  Map<NCOL> incl = compose<NCOL>(pre, inc);
  // exclusive = incl of lane-1 within the block
  Map<NCOL> prev = shfl_up_map<NCOL>(incl, 1);
  excl = lane == 0 ? pre : prev;
  Map<NCOL> tot = identity_map<NCOL>();
  for (int j = 0; j < kScanThreads / 32; ++j) {
    Map<NCOL> a;
#pragma unroll
    for (int c = 0; c < NCOL; ++c) a.c[c] = wagg[j][c];
    tot = compose<NCOL>(tot, a);
  }
  agg = tot;
  __syncthreads();
}

template <int NCOL>
__device__ __forceinline__ uint32_t map_at(const Map<NCOL>& m, int c) {
  uint32_t v = m.c[0];
#pragma unroll
  for (int j = 1; j < NCOL; ++j)
    if (j == c) v = m.c[j];
  return v;
}

// Pass 1: per-chunk maps + per-block aggregate maps.  Block b covers tile b0 + b
// of the stream (b0 > 0: a word-range shard); tmaps are indexed by the launch's
// own chunks, bagg by tile.
template <int NCOL>
__global__ void __launch_bounds__(kScanThreads) k_draw_count(StreamSpec sp, const long long* w0p, int64_t nchunks,
                                                             uint8_t* __restrict__ tmaps,
                                                             uint32_t* __restrict__ bagg, int64_t b0 = 0) {
  const int64_t tile = b0 + blockIdx.x;
  const int64_t chunk = tile * kScanThreads + threadIdx.x;
  const int64_t lchunk = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  WordGen g = tile_wordgen(sp, w0p, tile);
  Map<NCOL> m = identity_map<NCOL>();
  if (chunk < nchunks) {
    // Fast path (NCOL > 1): a word that passes every column's Lemire test is
    // accepted whichever column it serves, so a chunk of such words emits
    // kChunkWords elements from every start column.  Rejections are rare for
    // large modes (c4: 2^32 mod 1e6 / 2^32 = 2.3e-4 per word), so nearly every
    // chunk takes this path; the rest re-generate their words and run the
    // per-start-column state machine.
    bool fast = false;
    if (NCOL > 1) {
      const WordGen g0 = g;
      bool all = true;
#pragma unroll 4
      for (int i = 0; i < kChunkWords; ++i) {
        const uint32_t w = g.next();
#pragma unroll
        for (int c = 0; c < NCOL; ++c) all &= (uint32_t)((uint64_t)w * sp.n[c]) >= sp.thr[c];
      }
      if (all) {
#pragma unroll
        for (int c = 0; c < NCOL; ++c) m.c[c] = kChunkWords;
        fast = true;
      } else {
        g = g0;
      }
    }
    if (!fast) {
      int col[NCOL];
#pragma unroll
      for (int c = 0; c < NCOL; ++c) col[c] = c;
#pragma unroll 4
      for (int i = 0; i < kChunkWords; ++i) {
        const uint32_t w = g.next();
#pragma unroll
        for (int c = 0; c < NCOL; ++c) {
          const int cc = col[c];
          uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
          for (int j = 1; j < NCOL; ++j)
            if (j == cc) { n = sp.n[j]; thr = sp.thr[j]; }
          const uint64_t prod = (uint64_t)w * n;
          if ((uint32_t)prod >= thr) {
            m.c[c] += 1;
            col[c] = cc + 1 == NCOL ? 0 : cc + 1;
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NCOL; ++c) tmaps[lchunk * NCOL + c] = (uint8_t)m.c[c];
  }
  Map<NCOL> excl, agg;
  block_scan_maps<NCOL>(m, excl, agg);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) bagg[tile * NCOL + c] = agg.c[c];
  }
}

// Pass 2 (one block of 1024 threads, one pass): thread t composes the maps of its
// run of ceil(nblocks / 1024) consecutive tiles, a block scan of the run maps
// (64-bit counts) gives every run its start (column, element), and each thread
// then steps through its tiles writing their starts (the column after E
// elements is E mod NCOL) -- one sweep, not nblocks / 256 dependent block scans.
constexpr int kScanTilesThreads = 1024;
template <int NCOL>
struct Map64 {
  unsigned long long c[NCOL];
};
template <int NCOL>
__device__ __forceinline__ Map64<NCOL> compose64(const Map64<NCOL>& f, const Map64<NCOL>& g) {
  Map64<NCOL> h;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    const unsigned long long adv = f.c[c];
    const int cc = (int)((c + adv) % NCOL);
    unsigned long long gv = g.c[0];
#pragma unroll
    for (int j = 1; j < NCOL; ++j)
      if (j == cc) gv = g.c[j];
    h.c[c] = adv + gv;
  }
  return h;
}

template <int NCOL>
__global__ void __launch_bounds__(kScanTilesThreads) k_draw_scan_tiles(const uint32_t* __restrict__ bagg,
                                                                       int64_t nblocks, long long* __restrict__ bstart,
                                                                       long long* __restrict__ total_out) {
  __shared__ unsigned long long wagg[kScanTilesThreads / 32][NCOL];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t per = (nblocks + kScanTilesThreads - 1) / kScanTilesThreads;
  const int64_t b0 = min((int64_t)t * per, nblocks), b1 = min(b0 + per, nblocks);
  Map64<NCOL> m;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) m.c[c] = 0;
  for (int64_t b = b0; b < b1; ++b) {
    Map64<NCOL> tm;
#pragma unroll
    for (int c = 0; c < NCOL; ++c) tm.c[c] = __ldg(bagg + b * NCOL + c);
    m = compose64<NCOL>(m, tm);
  }
  Map64<NCOL> inc = m;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Map64<NCOL> o;
#pragma unroll
    for (int c = 0; c < NCOL; ++c) o.c[c] = __shfl_up_sync(0xffffffffu, inc.c[c], d);
    if (lane >= d) inc = compose64<NCOL>(o, inc);
  }
  if (lane == 31) {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) wagg[w][c] = inc.c[c];
  }
  __syncthreads();
  Map64<NCOL> pre;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) pre.c[c] = 0;
  for (int j = 0; j < w; ++j) {
    Map64<NCOL> a;
#pragma unroll
    for (int c = 0; c < NCOL; ++c) a.c[c] = wagg[j][c];
    pre = compose64<NCOL>(pre, a);
  }
  Map64<NCOL> prev;
#pragma unroll
  for (int c = 0; c < NCOL; ++c) prev.c[c] = __shfl_up_sync(0xffffffffu, inc.c[c], 1);
  const Map64<NCOL> excl = lane == 0 ? pre : compose64<NCOL>(pre, prev);
  unsigned long long elem = excl.c[0];  // from column 0 at the stream start
  int col = (int)(elem % NCOL);
  for (int64_t b = b0; b < b1; ++b) {
    bstart[b * 2 + 0] = col;
    bstart[b * 2 + 1] = (long long)elem;
    uint32_t adv = __ldg(bagg + b * NCOL);
#pragma unroll
    for (int j = 1; j < NCOL; ++j)
      if (j == col) adv = __ldg(bagg + b * NCOL + j);
    elem += adv;
    col = (int)((col + adv) % NCOL);
  }
  if (t == kScanTilesThreads - 1) *total_out = (long long)elem;
}

// Pass 3: re-generate the words, stage accepted values in shared memory and
// write the block's contiguous output range with coalesced stores.
// NCOL == 1 (nonzero stratum): out[e] = value; records the end word of element target-1.
// NCOL  > 1 (zero candidates):  out[e] = value (row-major [row][NCOL]).
//
// Word-range shards (sharded draws, below): b0 is the first tile of this rank's
// range; lim_dev (nullable) lowers the element limit to *lim_dev and shift_dev
// (nullable) writes element e at out[e - *shift_dev], dropping e < *shift_dev;
// owned may be null (the sharded draw certifies its counters from their sums).
template <int NCOL>
__global__ void __launch_bounds__(kScanThreads) k_draw_write(StreamSpec sp, const long long* w0p, int64_t nchunks,
                                                             const uint8_t* __restrict__ tmaps,
                                                             const long long* __restrict__ bstart,
                                                             int64_t target, int32_t* __restrict__ out,
                                                             long long* __restrict__ end_word,
                                                             uint32_t* __restrict__ hist, DevFlags* flags,
                                                             uint32_t olo, uint32_t ohi,
                                                             unsigned long long* __restrict__ owned,
                                                             int64_t b0 = 0, const long long* lim_dev = nullptr,
                                                             const long long* shift_dev = nullptr) {
  extern __shared__ int32_t stage[];  // kBlockWords int32 (draw_stage_smem)
  uint32_t mine = 0;  // merged form: accepted draws landing in this rank's ordinal range [olo, ohi)
  const int64_t tile = b0 + blockIdx.x;
  const int64_t chunk = tile * kScanThreads + threadIdx.x;
  const int64_t lchunk = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  WordGen g = tile_wordgen(sp, w0p, tile);
  if (lim_dev) target = min((long long)target, *lim_dev);
  const long long shift = shift_dev ? *shift_dev : 0;
  Map<NCOL> m = identity_map<NCOL>();
  if (chunk < nchunks) {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) m.c[c] = tmaps[lchunk * NCOL + c];
  }
  Map<NCOL> excl, agg;
  block_scan_maps<NCOL>(m, excl, agg);
  const int bcol = (int)bstart[tile * 2 + 0];
  const long long eb = bstart[tile * 2 + 1];
  const uint32_t adv = map_at<NCOL>(excl, bcol);
  const long long nblk = map_at<NCOL>(agg, bcol);
  int col = (int)((bcol + adv) % NCOL);
  long long e = eb + adv;
  int rel = (int)adv;
  if (chunk < nchunks && e < target) {
    uint64_t w = tile_word0(w0p, tile) + (uint64_t)threadIdx.x * kChunkWords;
    for (int i = 0; i < kChunkWords && e < target; ++i, ++w) {
      const uint32_t word = g.next();
      uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
      for (int j = 1; j < NCOL; ++j)
        if (j == col) { n = sp.n[j]; thr = sp.thr[j]; }
      const uint64_t prod = (uint64_t)word * n;
      if ((uint32_t)prod >= thr) {
        const uint32_t val = (uint32_t)(prod >> 32);
        if (hist) {  // merged form: 4-bit counters (a wrap is caught by the count-sum check)
          if (val >= olo && val < ohi) {
            const uint32_t o = val - olo;
            atomicAdd(hist + (o >> 3), 1u << ((o & 7u) << 2));
            ++mine;
          }
        } else {
          stage[rel++] = (int32_t)val;
        }
        if (e == target - 1 && end_word) *end_word = (long long)(w + 1);
        ++e;
        col = col + 1 == NCOL ? 0 : col + 1;
      }
    }
  }
  if (hist) {
    if (!owned) return;
#pragma unroll
    for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(owned, (unsigned long long)mine);
    return;
  }
  __syncthreads();
  const long long lim = min((long long)nblk, (long long)target - eb);
  for (long long i = threadIdx.x; i < lim; i += kScanThreads)
    if (eb + i >= shift) out[eb + i - shift] = stage[i];
}

struct ZeroSpec {
  int ndim, ncol;
  int colmap[kMaxModes];
  Strides st;
};

__device__ __forceinline__ int64_t zero_rows_avail(const ZeroSpec& zs, const long long* elems_avail,
                                                   int64_t rows_max) {
  return zs.ncol ? min(rows_max, (int64_t)(*elems_avail / zs.ncol)) : rows_max;
}

// Zero stratum, pass A: hit test of kRowsPerThread consecutive candidate rows
// per thread against the nonzero hash; per-thread miss mask, per-block miss count.
__global__ void __launch_bounds__(kScanThreads) k_zero_hits(ZeroSpec zs, const int32_t* __restrict__ cand,
                                                            const long long* __restrict__ elems_avail,
                                                            int64_t rows_max,
                                                            const unsigned long long* __restrict__ table,
                                                            uint64_t mask, uint8_t* __restrict__ miss,
                                                            uint32_t* __restrict__ bcount, int64_t q,
                                                            unsigned long long* __restrict__ hit_in_q,
                                                            int mark_hits, const unsigned int* __restrict__ filter,
                                                            uint64_t fmask) {
  const int64_t rows = zero_rows_avail(zs, elems_avail, rows_max);
  const int64_t t = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  const int64_t r0 = t * kRowsPerThread;
  uint32_t bits = 0;
  uint64_t key[kRowsPerThread];
  bool live[kRowsPerThread];
#pragma unroll
  for (int j = 0; j < kRowsPerThread; ++j) {
    const int64_t r = r0 + j;
    live[j] = r < rows;
    key[j] = 0;
    if (live[j])
      for (int k = 0; k < zs.ndim; ++k) {
        const int cm = zs.colmap[k];
        const uint32_t c = cm < 0 ? 0u : (uint32_t)__ldg(cand + r * zs.ncol + cm);
        key[j] += (uint64_t)c * zs.st.s[k];
      }
  }
#pragma unroll
  for (int j = 0; j < kRowsPerThread; ++j) {
    if (!live[j]) continue;
    bool present = false;
    if (table) {
      present = true;
      if (filter) present = filter_may_contain(filter, fmask, mix64(key[j]));  // a clear bit proves absence
      if (present) present = hash_contains(table, mask, key[j]);
    }
    if (!present) bits |= 1u << j;
  }
  if (r0 < rows_max) miss[t] = (uint8_t)bits;
  if (hit_in_q) {  // any of the first q candidate rows not a miss -> the slow (compacting) path
    bool hit = false;
#pragma unroll
    for (int j = 0; j < kRowsPerThread; ++j)
      if (r0 + j < q && !((bits >> j) & 1u)) hit = true;
    if (hit) atomicOr(hit_in_q, 1ull);
  }
  if (mark_hits) {  // lazy layout: a hit row keeps its slot, flagged by coordinate -1
#pragma unroll
    for (int j = 0; j < kRowsPerThread; ++j)
      if (live[j] && !((bits >> j) & 1u)) const_cast<int32_t*>(cand)[(r0 + j) * zs.ncol] = -1;
  }
  const int cnt = __popc(bits);
  __shared__ uint32_t wsum[kScanThreads / 32];
  int v = cnt;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int j = 0; j < kScanThreads / 32; ++j) s += wsum[j];
    bcount[blockIdx.x] = s;
  }
}

// Batched small draws (DrawBatchSet): block b of a batch launch runs draw b --
// its own StreamSpec, outputs, scalar block and event code offset by b strides.
// A plain launch (gridDim 1, specs null) is a single draw.
struct DrawBatch {
  const StreamSpec* specs;  // nullable: the kernel's own StreamSpec
  int64_t out_stride;       // output elements between consecutive draws
  int64_t scal_stride;      // long longs between consecutive draws' scalar blocks
  long long code_stride;    // event-code step between consecutive draws
};

// Small zero strata (lazy layout): hit test + flagging, the miss scan and the
// q-th-miss search of passes A / B / locate in one block walking the rows in
// order; it stops at the tile holding the q-th miss.
__global__ void __launch_bounds__(kScanThreads) k_zero_fused(ZeroSpec zs, int32_t* __restrict__ cand,
                                                             const long long* __restrict__ elems_avail,
                                                             int64_t rows_max,
                                                             const unsigned long long* __restrict__ table,
                                                             uint64_t mask, const unsigned int* __restrict__ filter,
                                                             uint64_t fmask, int64_t q, long long* __restrict__ rows_used,
                                                             long long* __restrict__ hits_before,
                                                             long long* __restrict__ misses_out, int64_t p,
                                                             const long long* __restrict__ nz_avail, long long budget,
                                                             long long code, DevFlags* flags, DrawBatch B) {
  __shared__ long long carry;
  __shared__ int found;
  {
    const int64_t bi = blockIdx.x;
    cand += bi * B.out_stride;
    const int64_t so = bi * B.scal_stride;
    elems_avail += so;
    rows_used += so;
    hits_before += so;
    misses_out += so;
    if (nz_avail) nz_avail += so;
    code += bi * B.code_stride;
  }
  __shared__ int wsum[kScanThreads / 32];
  if (threadIdx.x == 0) {
    carry = 0;
    found = 0;
  }
  __syncthreads();
  const int64_t rows = zero_rows_avail(zs, elems_avail, rows_max);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < rows_max; base += kRowsPerBlock) {
    const int64_t r0 = base + (int64_t)threadIdx.x * kRowsPerThread;
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < kRowsPerThread; ++j) {
      const int64_t r = r0 + j;
      if (r >= rows) continue;
      uint64_t key = 0;
      for (int k = 0; k < zs.ndim; ++k) {
        const int cm = zs.colmap[k];
        const uint32_t c = cm < 0 ? 0u : (uint32_t)cand[r * zs.ncol + cm];
        key += (uint64_t)c * zs.st.s[k];
      }
      bool present = false;
      if (table) {
        present = true;
        if (filter) present = filter_may_contain(filter, fmask, mix64(key));
        if (present) present = hash_contains(table, mask, key);
      }
      if (present) cand[r * zs.ncol] = -1;  // lazy layout: a hit keeps its slot, flagged
      else bits |= 1u << j;
    }
    const int cnt = __popc(bits);
    int inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int pre = 0, tot = 0;
    for (int j = 0; j < kScanThreads / 32; ++j) {
      if (j < w) pre += wsum[j];
      tot += wsum[j];
    }
    const long long c0 = carry;
    long long rank = c0 + pre + inc - cnt;
    for (int j = 0; j < kRowsPerThread; ++j) {
      if (!(bits & (1u << j))) continue;
      if (rank == q - 1) {
        *rows_used = r0 + j + 1;
        *hits_before = (r0 + j) - (q - 1);
        found = 1;
      }
      ++rank;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + tot;
    __syncthreads();
    if (found) break;
  }
  if (threadIdx.x == 0) {  // k_draw_status, folded
    *misses_out = carry;
    if (!found) *rows_used = rows_max;
    bool shortfall = p > 0 && nz_avail && *nz_avail < p, exhausted = false;
    if (carry >= q) {
      if (*hits_before > budget) exhausted = true;
    } else if (rows - carry > budget) {
      exhausted = true;
    } else {
      shortfall = true;
    }
    if (exhausted) atomicMin(&flags->first_code[kFlagSampling], code);
    else if (shortfall) atomicMin(&flags->first_code[kFlagShortfall], code);
  }
}

// Pass B: exclusive scan of per-block miss counts (one block of 1024 threads).
__global__ void __launch_bounds__(1024) k_zero_scan(const uint32_t* __restrict__ bcount, int64_t nblocks,
                                                    long long* __restrict__ boff, long long* __restrict__ total) {
  __shared__ long long wsum[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < nblocks; base += 1024) {
    const int64_t b = base + threadIdx.x;
    const long long v = b < nblocks ? bcount[b] : 0;
    long long inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const long long o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    long long pre = 0;
    for (int j = 0; j < w; ++j) pre += wsum[j];
    if (b < nblocks) boff[b] = carry + pre + inc - v;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long s = 0;
      for (int j = 0; j < 32; ++j) s += wsum[j];
      carry += s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Pass C: compact the first q misses into zero_subs (int32 [q x ndim]) through
// a shared-memory stage; the writer of miss number q-1 records how many hits
// preceded it (the reference's rejection count at its last round).
__global__ void __launch_bounds__(kScanThreads) k_zero_compact(ZeroSpec zs, const int32_t* __restrict__ cand,
                                                               int64_t rows_max, const uint8_t* __restrict__ miss,
                                                               const long long* __restrict__ boff, int64_t q,
                                                               int32_t* __restrict__ zero_subs,
                                                               long long* __restrict__ hits_before,
                                                               const unsigned long long* __restrict__ hit_in_q) {
  extern __shared__ int32_t zstage[];
  __shared__ int wsum[kScanThreads / 32];
  // fast path: the first q candidates all miss, so the candidate buffer already
  // holds the accepted zeros in order and nothing precedes the q-th miss
  if (hit_in_q && *hit_in_q == 0ull) return;
  const int64_t t = blockIdx.x * (int64_t)kScanThreads + threadIdx.x;
  const int64_t r0 = t * kRowsPerThread;
  const uint32_t bits = r0 < rows_max ? miss[t] : 0u;
  const int cnt = __popc(bits);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  int pre = 0;
  for (int j = 0; j < w; ++j) pre += wsum[j];
  int blk_total = 0;
  for (int j = 0; j < kScanThreads / 32; ++j) blk_total += wsum[j];
  const long long bo = boff[blockIdx.x];
  int rel = pre + inc - cnt;
  const int nd = zs.ndim;
  for (int j = 0; j < kRowsPerThread; ++j) {
    if (!(bits & (1u << j))) continue;
    const long long rank = bo + rel;
    if (rank < q) {
      const int64_t r = r0 + j;
      for (int k = 0; k < nd; ++k) {
        const int cm = zs.colmap[k];
        zstage[rel * nd + k] = cm < 0 ? 0 : __ldg(cand + r * zs.ncol + cm);
      }
      if (rank == q - 1) *hits_before = (long long)(r - rank);
    }
    ++rel;
  }
  __syncthreads();
  const long long nrows = max(0LL, min((long long)blk_total, q - bo));
  for (long long i = threadIdx.x; i < nrows * nd; i += kScanThreads) zero_subs[bo * nd + i] = zstage[i];
}

// Lazy layout: locate the q-th miss.  The accepted zeros are then candidate rows
// [0, R) minus the rows flagged -1, R = row of the q-th miss + 1, and the
// reference's rejection count at its last round is R - q (sampling.py:137-150).
// (a __device__ body: the sharded draw's cut runs it with a device-side q; all
// threads of the block call it, row_base shifts the reported hit count)
__device__ void zero_locate_body(const uint32_t* __restrict__ bcount, const long long* __restrict__ boff,
                                 int64_t nblocks, const uint8_t* __restrict__ miss, int64_t rows_max, int64_t q,
                                 long long* __restrict__ rows_used, long long* __restrict__ hits_before,
                                 long long row_base, long long q_global) {
  __shared__ int64_t sb;
  __shared__ int wsum[kScanThreads / 32];
  if (threadIdx.x == 0) {
    // last block whose exclusive offset is <= q-1
    int64_t lo = 0, hi = nblocks - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (boff[mid] <= q - 1) lo = mid;
      else hi = mid - 1;
    }
    sb = (boff[lo] + (long long)bcount[lo] > q - 1) ? lo : -1;
    if (sb < 0) *rows_used = rows_max;  // fewer than q misses: the status pass reports it
  }
  __syncthreads();
  if (sb < 0) return;
  const int64_t t = sb * kScanThreads + threadIdx.x;
  const int64_t r0 = t * kRowsPerThread;
  const uint32_t bits = r0 < rows_max ? miss[t] : 0u;
  const int cnt = __popc(bits);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int inc = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[w] = inc;
  __syncthreads();
  int pre = 0;
  for (int j = 0; j < w; ++j) pre += wsum[j];
  const long long target = q - 1 - boff[sb];  // rank of the q-th miss within the block
  long long rank = pre + inc - cnt;
  for (int j = 0; j < kRowsPerThread; ++j) {
    if (!(bits & (1u << j))) continue;
    if (rank == target) {
      *rows_used = r0 + j + 1;
      *hits_before = (row_base + r0 + j) - (q_global - 1);
    }
    ++rank;
  }
}

__global__ void __launch_bounds__(kScanThreads) k_zero_locate(const uint32_t* __restrict__ bcount,
                                                              const long long* __restrict__ boff, int64_t nblocks,
                                                              const uint8_t* __restrict__ miss, int64_t rows_max,
                                                              int64_t q, long long* __restrict__ rows_used,
                                                              long long* __restrict__ hits_before) {
  zero_locate_body(bcount, boff, nblocks, miss, rows_max, q, rows_used, hits_before, 0, q);
}

// Semi-stratified uniform stratum with size-1 modes: [row][ncol] -> [row][d] (zeros inserted).
__global__ void k_expand_rows(ZeroSpec zs, const int32_t* __restrict__ cand, int64_t rows, int32_t* __restrict__ out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < zs.ndim; ++k) out[r * zs.ndim + k] = zs.colmap[k] < 0 ? 0 : cand[r * zs.ncol + zs.colmap[k]];
}

__global__ void k_semi_status(int64_t p, const long long* nz_avail, long long need_elems, const long long* z_elems,
                              long long code, DevFlags* flags) {
  if (threadIdx.x || blockIdx.x) return;
  const bool short_nz = p > 0 && nz_avail && *nz_avail < p;
  const bool short_z = need_elems > 0 && *z_elems < need_elems;
  if (short_nz || short_z) atomicMin(&flags->first_code[kFlagShortfall], code);
}

// Slow path of the in-place layout: copy the compacted zeros back over the candidates.
__global__ void k_zero_copyback(const unsigned long long* __restrict__ hit_in_q, const int32_t* __restrict__ src,
                                int32_t* __restrict__ dst, int64_t n) {
  if (*hit_in_q == 0ull) return;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Final status: shortfall (need more candidates) or budget exhaustion.
__global__ void k_draw_status(int64_t p, const long long* nz_avail, int64_t q, const long long* z_misses,
                              int64_t rows_max, int ncol, const long long* z_elems, const long long* hits_before,
                              long long budget, long long code, DevFlags* flags) {
  if (threadIdx.x || blockIdx.x) return;
  bool shortfall = false, exhausted = false;
  if (p > 0 && nz_avail && *nz_avail < p) shortfall = true;
  if (q > 0) {
    const long long rows = ncol ? min((long long)rows_max, *z_elems / ncol) : rows_max;
    const long long misses = *z_misses;
    if (misses >= q) {
      if (*hits_before > budget) exhausted = true;
    } else {
      const long long hits = rows - misses;
      if (hits > budget) exhausted = true;
      else shortfall = true;
    }
  }
  if (exhausted) atomicMin(&flags->first_code[kFlagSampling], code);
  else if (shortfall) atomicMin(&flags->first_code[kFlagShortfall], code);
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_set_ll(long long* p, long long v) { *p = v; }

// Merged nonzero stratum: ordinals with a nonzero byte counter, in ascending
// order, with their multiplicities (the np.unique + bincount merge of
// sampled_gradient_tensor, sampling.py:233-237, restricted to the nonzero
// stratum).  Pass 1 counts per block, pass 2 (k_zero_scan) scans, pass 3 writes.
// Counters are 4-bit nibbles, 8 per word: at c4 the 1e8 counters take 50 MB and
// stay L2-resident while the draw's atomics land on them.
constexpr int kHistWordsPerThread = 4;
constexpr int kHistPerBlock = kHistWordsPerThread * 8 * kScanThreads;

__device__ __forceinline__ int bytes_nonzero(uint32_t w) {  // nonzero nibbles
  int c = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) c += ((w >> (4 * b)) & 0xfu) != 0;
  return c;
}

__device__ __forceinline__ uint32_t bytes_sum(uint32_t w) {  // sum of nibbles
  uint32_t s = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b) s += (w >> (4 * b)) & 0xfu;
  return s;
}

// Per-block count of nonzero counters, plus the sum of all counters: a wrapped
// byte loses 256 from that sum, so sum == p certifies the counts exactly.
__global__ void __launch_bounds__(kScanThreads) k_hist_count(const uint32_t* __restrict__ hist, int64_t nwords,
                                                             uint32_t* __restrict__ bcount,
                                                             unsigned long long* __restrict__ cnt_sum) {
  const int64_t w0 = (blockIdx.x * (int64_t)kScanThreads + threadIdx.x) * kHistWordsPerThread;
  int c = 0;
  uint32_t sum = 0;
#pragma unroll
  for (int j = 0; j < kHistWordsPerThread; ++j)
    if (w0 + j < nwords) {
      const uint32_t w = __ldg(hist + w0 + j);
      c += bytes_nonzero(w);
      sum += bytes_sum(w);
    }
  __shared__ int wsum[kScanThreads / 32];
  __shared__ uint32_t ssum[kScanThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, o);
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    wsum[threadIdx.x >> 5] = c;
    ssum[threadIdx.x >> 5] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    unsigned long long t = 0;
    for (int j = 0; j < kScanThreads / 32; ++j) {
      s += wsum[j];
      t += ssum[j];
    }
    bcount[blockIdx.x] = (uint32_t)s;
    atomicAdd(cnt_sum, t);
  }
}

// Σ counters must equal the draws that landed in this rank's range (all p on one GPU).
__global__ void k_hist_verify(const unsigned long long* __restrict__ cnt_sum,
                              const unsigned long long* __restrict__ owned, DevFlags* flags) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && *cnt_sum != *owned) atomicOr(&flags->data_bits, kMergeOverflowBit);
}

__global__ void __launch_bounds__(kScanThreads) k_hist_write(const uint32_t* __restrict__ hist, int64_t nwords,
                                                             int64_t eta, const long long* __restrict__ boff,
                                                             int32_t* __restrict__ ord, uint8_t* __restrict__ cnt,
                                                             int32_t obase) {
  const int64_t w0 = (blockIdx.x * (int64_t)kScanThreads + threadIdx.x) * kHistWordsPerThread;
  uint32_t w[kHistWordsPerThread];
  int c = 0;
#pragma unroll
  for (int j = 0; j < kHistWordsPerThread; ++j) {
    w[j] = w0 + j < nwords ? __ldg(hist + w0 + j) : 0u;
    c += bytes_nonzero(w[j]);
  }
  __shared__ int wsum[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  int inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) wsum[wi] = inc;
  __syncthreads();
  int pre = 0, tot = 0;
  for (int j = 0; j < kScanThreads / 32; ++j) {
    if (j < wi) pre += wsum[j];
    tot += wsum[j];
  }
  // stage the block's entries in shared memory, then write them coalesced
  __shared__ int32_t s_ord[kHistPerBlock];
  __shared__ uint8_t s_cnt[kHistPerBlock];
  int rel = pre + inc - c;
#pragma unroll
  for (int j = 0; j < kHistWordsPerThread; ++j)
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t v = (w[j] >> (4 * b)) & 0xfu;
      if (v) {
        s_ord[rel] = obase + (int32_t)((w0 + j) * 8 + b);
        s_cnt[rel] = (uint8_t)v;
        ++rel;
      }
    }
  __syncthreads();
  const long long base = boff[blockIdx.x];
  for (int i = threadIdx.x; i < tot; i += kScanThreads) {
    ord[base + i] = s_ord[i];
    cnt[base + i] = s_cnt[i];
  }
  (void)eta;
}

// Gather the ordinal-indexed counters into position order (perm[pos] = ordinal):
// one output word = 8 consecutive positions; the counter reads are random but
// hit the L2-resident histogram.
__global__ void k_hist_permute(const uint32_t* __restrict__ hist, const int32_t* __restrict__ perm, int64_t eta,
                               int64_t nwords, uint32_t* __restrict__ pnib, int32_t olo) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p0 = w * 8;
    int32_t o[8];
    if (p0 + 8 <= eta) {
      const int4 a = __ldg(reinterpret_cast<const int4*>(perm + p0));
      const int4 b = __ldg(reinterpret_cast<const int4*>(perm + p0) + 1);
      o[0] = a.x - olo; o[1] = a.y - olo; o[2] = a.z - olo; o[3] = a.w - olo;
      o[4] = b.x - olo; o[5] = b.y - olo; o[6] = b.z - olo; o[7] = b.w - olo;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] = p0 + j < eta ? __ldg(perm + p0 + j) - olo : -1;
    }
    uint32_t out = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (o[j] >= 0) out |= ((__ldg(hist + (o[j] >> 3)) >> (4 * (o[j] & 7))) & 0xfu) << (4 * j);
    pnib[w] = out;
  }
}

// Small draws (c1/c2 shapes): passes 1-3 fused in one block that walks the tiles
// in order with a running (column, element) carry -- the same chunk maps, scan
// and staged write as above, in one launch instead of three.
constexpr int64_t kFusedMaxTiles = 16;
template <int NCOL>
__global__ void __launch_bounds__(kScanThreads) k_draw_fused(StreamSpec sp, const long long* w0p, int64_t nchunks,
                                                             int64_t target, int32_t* __restrict__ out,
                                                             long long* __restrict__ end_word,
                                                             long long* __restrict__ elems_total, DevFlags* report,
                                                             long long code, long long* __restrict__ clear,
                                                             DrawBatch B) {
  __shared__ int32_t stage[kBlockWords];
  {
    const int64_t bi = blockIdx.x;
    if (B.specs) sp = B.specs[bi];
    out += bi * B.out_stride;
    const int64_t so = bi * B.scal_stride;
    if (w0p) w0p += so;
    if (end_word) end_word += so;
    elems_total += so;
    if (clear) clear += so;
    code += bi * B.code_stride;
  }
  __shared__ long long carry_e;
  __shared__ int carry_c;
  if (threadIdx.x == 0) {
    carry_e = 0;
    carry_c = 0;
  }
  if (clear && threadIdx.x < 16) clear[threadIdx.x] = 0;  // the draw's scalars (instead of a memset)
  const int64_t ntiles = (nchunks + kScanThreads - 1) / kScanThreads;
  for (int64_t tile = 0; tile < ntiles; ++tile) {
    const int64_t chunk = tile * kScanThreads + threadIdx.x;
    WordGen g = tile_wordgen(sp, w0p, tile);  // syncs: carry from the previous tile is visible
    const WordGen g0 = g;
    Map<NCOL> m = identity_map<NCOL>();
    if (chunk < nchunks) {
      int col[NCOL];
#pragma unroll
      for (int c = 0; c < NCOL; ++c) col[c] = c;
      for (int i = 0; i < kChunkWords; ++i) {
        const uint32_t w = g.next();
#pragma unroll
        for (int c = 0; c < NCOL; ++c) {
          const int cc = col[c];
          uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
          for (int j = 1; j < NCOL; ++j)
            if (j == cc) { n = sp.n[j]; thr = sp.thr[j]; }
          if ((uint32_t)((uint64_t)w * n) >= thr) {
            m.c[c] += 1;
            col[c] = cc + 1 == NCOL ? 0 : cc + 1;
          }
        }
      }
    }
    Map<NCOL> excl, agg;
    block_scan_maps<NCOL>(m, excl, agg);
    const int bcol = carry_c;
    const long long eb = carry_e;
    const uint32_t adv = map_at<NCOL>(excl, bcol);
    const long long nblk = map_at<NCOL>(agg, bcol);
    int col = (int)((bcol + adv) % NCOL);
    long long e = eb + adv;
    int rel = (int)adv;
    if (chunk < nchunks && e < target) {
      g = g0;
      uint64_t w = tile_word0(w0p, tile) + (uint64_t)threadIdx.x * kChunkWords;
      for (int i = 0; i < kChunkWords && e < target; ++i, ++w) {
        const uint32_t word = g.next();
        uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
        for (int j = 1; j < NCOL; ++j)
          if (j == col) { n = sp.n[j]; thr = sp.thr[j]; }
        const uint64_t prod = (uint64_t)word * n;
        if ((uint32_t)prod >= thr) {
          stage[rel++] = (int32_t)(prod >> 32);
          if (e == target - 1 && end_word) *end_word = (long long)(w + 1);
          ++e;
          col = col + 1 == NCOL ? 0 : col + 1;
        }
      }
    }
    __syncthreads();
    const long long lim = min(nblk, (long long)target - eb);
    for (long long i = threadIdx.x; i < lim; i += kScanThreads) out[eb + i] = stage[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      carry_e = eb + nblk;
      carry_c = (int)((bcol + nblk) % NCOL);
    }
    if (eb + nblk >= target) break;  // every element the draw uses is written
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *elems_total = carry_e;
    if (report && carry_e < target) atomicMin(&report->first_code[kFlagShortfall], code);  // k_draw_status, folded
  }
}

// ---- merged form of the nonzero stratum: one generating pass, then a trim.
// The counters do not care about element order, so a single pass over the
// tiles counts every tile's accepted words (for the scan) and histograms them
// at once; the provisioning slack past element p - 1 (a couple of tiles at
// slack 1) is then taken back out by k_draw_trim, which re-generates only the
// tiles from the one holding element p - 1.  Saves the separate counting pass.
__global__ void __launch_bounds__(kScanThreads) k_draw_count_hist(StreamSpec sp, const long long* w0p,
                                                                  int64_t nchunks, uint32_t* __restrict__ bagg,
                                                                  int64_t b0, uint32_t* __restrict__ hist,
                                                                  uint32_t olo, uint32_t ohi,
                                                                  unsigned long long* __restrict__ owned) {
  const int64_t tile = b0 + blockIdx.x;
  const int64_t chunk = tile * kScanThreads + threadIdx.x;
  WordGen g = tile_wordgen(sp, w0p, tile);
  uint32_t cnt = 0, mine = 0;
  if (chunk < nchunks) {
    const uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll 4
    for (int i = 0; i < kChunkWords; ++i) {
      const uint64_t prod = (uint64_t)g.next() * n;
      if ((uint32_t)prod >= thr) {
        ++cnt;
        const uint32_t val = (uint32_t)(prod >> 32);
        if (val >= olo && val < ohi) {
          const uint32_t o = val - olo;
          atomicAdd(hist + (o >> 3), 1u << ((o & 7u) << 2));
          ++mine;
        }
      }
    }
  }
  __shared__ uint32_t wsum[kScanThreads / 32];
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    mine += __shfl_xor_sync(0xffffffffu, mine, o);
  }
  if ((threadIdx.x & 31) == 0) {
    wsum[threadIdx.x >> 5] = cnt;
    if (owned && mine) atomicAdd(owned, (unsigned long long)mine);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int j = 0; j < kScanThreads / 32; ++j) t += wsum[j];
    bagg[tile] = t;
  }
}

// Take the accepted words at element >= target out of the counters again, over
// this caller's tiles [b_lo, b_hi) from the tile holding element target - 1 on
// (grid-stride over those tiles), and record the end word of element target - 1
// (end_word nullable).  Nothing to do if the stream fell short of target.
__global__ void __launch_bounds__(kScanThreads) k_draw_trim(StreamSpec sp, const long long* w0p, int64_t nchunks,
                                                            const long long* __restrict__ bstart, int64_t nblocks,
                                                            const long long* __restrict__ total, int64_t target,
                                                            int64_t b_lo, int64_t b_hi, uint32_t* __restrict__ hist,
                                                            uint32_t olo, uint32_t ohi,
                                                            unsigned long long* __restrict__ owned,
                                                            long long* __restrict__ end_word) {
  __shared__ long long tb;
  __shared__ uint32_t wsum[kScanThreads / 32];
  if (threadIdx.x == 0) {
    tb = -1;
    if (target > 0 && *total >= target) {
      int64_t lo = 0, hi = nblocks - 1;  // last tile whose first element is <= target-1
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (bstart[mid * 2 + 1] <= target - 1) lo = mid;
        else hi = mid - 1;
      }
      tb = lo;
    }
  }
  __syncthreads();
  if (tb < 0) return;
  const uint32_t n = sp.n[0], thr = sp.thr[0];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t tile = max((int64_t)tb, b_lo) + blockIdx.x; tile < b_hi; tile += gridDim.x) {
    const int64_t chunk = tile * kScanThreads + threadIdx.x;
    WordGen g = tile_wordgen(sp, w0p, tile);
    WordGen g0 = g;
    uint32_t cnt = 0;
    if (chunk < nchunks)
      for (int i = 0; i < kChunkWords; ++i)
        if ((uint32_t)((uint64_t)g.next() * n) >= thr) ++cnt;
    uint32_t inc = cnt;  // block exclusive scan of the chunk counts
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t pre = 0;
    for (int j = 0; j < w; ++j) pre += wsum[j];
    __syncthreads();
    long long e = bstart[tile * 2 + 1] + pre + inc - cnt;
    uint32_t back = 0;
    if (chunk < nchunks && e + cnt > target - 1) {
      uint64_t wi = tile_word0(w0p, tile) + (uint64_t)threadIdx.x * kChunkWords;
      for (int i = 0; i < kChunkWords; ++i, ++wi) {
        const uint64_t prod = (uint64_t)g0.next() * n;
        if ((uint32_t)prod < thr) continue;
        if (e == target - 1 && end_word) *end_word = (long long)(wi + 1);
        if (e >= target) {
          const uint32_t val = (uint32_t)(prod >> 32);
          if (val >= olo && val < ohi) {
            const uint32_t o = val - olo;
            atomicSub(hist + (o >> 3), 1u << ((o & 7u) << 2));
            ++back;
          }
        }
        ++e;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) back += __shfl_xor_sync(0xffffffffu, back, o);
    if (lane == 0 && back && owned) atomicAdd(owned, (unsigned long long)(-(long long)back));
  }
}

// Shared memory of a write / counter pass: the output stage's footprint even in
// the merged form, which does not use it -- a lean counter pass squeezes in
// beside the walk kernels and slows them more than it gains (c4: 1414 vs 1392 ms
// per step at N = 1, 241 vs 230 ms in the N = 8 projection; the fused counter
// pass likewise 1394 vs 1376 without the footprint).
static int draw_stage_smem(bool /*merged_form*/) { return kBlockWords * 4; }

template <int NCOL>
static void run_stream(Ctx* ctx, const StreamSpec& sp, const long long* w0, int64_t target, int64_t words,
                       int32_t* out, long long* end_word, long long* elems_total, DrawScratch& scr,
                       uint32_t* hist = nullptr, uint32_t olo = 0, uint32_t ohi = 0,
                       unsigned long long* owned = nullptr, DevFlags* report = nullptr, long long code = 0,
                       bool* fused = nullptr, long long* clear = nullptr) {
  const int64_t nchunks = std::max<int64_t>(1, (words + kChunkWords - 1) / kChunkWords);
  const int64_t nblocks = (nchunks + kScanThreads - 1) / kScanThreads;
  if (fused) *fused = false;
  if (!hist && nblocks <= kFusedMaxTiles) {
    k_draw_fused<NCOL><<<1, kScanThreads, 0, ctx->stream>>>(sp, w0, nchunks, target, out, end_word, elems_total,
                                                            report, code, clear, DrawBatch{nullptr, 0, 0, 0});
    ctx->count();
    check_launch();
    if (fused) *fused = true;
    return;
  }
  scr.tmaps.ensure((size_t)nblocks * kScanThreads * NCOL);
  scr.bagg.ensure((size_t)nblocks * NCOL * 4);
  scr.bstart.ensure((size_t)nblocks * 16);
  cudaStream_t s = ctx->stream;
  k_draw_count<NCOL><<<(unsigned)nblocks, kScanThreads, 0, s>>>(sp, w0, nchunks, scr.tmaps.as<uint8_t>(),
                                                               scr.bagg.as<uint32_t>());
  k_draw_scan_tiles<NCOL><<<1, kScanTilesThreads, 0, s>>>(scr.bagg.as<uint32_t>(), nblocks, scr.bstart.as<long long>(),
                                                      elems_total);
  k_draw_write<NCOL><<<(unsigned)nblocks, kScanThreads, draw_stage_smem(hist != nullptr), s>>>(sp, w0, nchunks,
                                                                                              scr.tmaps.as<uint8_t>(),
                                                               scr.bstart.as<long long>(), target, out, end_word,
                                                               hist, ctx->flags.as<DevFlags>(), olo, ohi, owned);
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

// Sorted zero stratum (bucketed merged solves).  Key of candidate row r =
// (row bucket of its bucket-mode coordinate) << b0 | (mode-0 row >> s0), the
// order of the bucketed nonzero walk (Slice::perm); rejected candidates (first
// coordinate -1) and rows past the q-th miss get the sentinel 1 << kb, so a
// stable radix sort on kb + 1 bits lists the q accepted rows first, in
// (bucket, mode-0 row, draw) order -- a fixed permutation of the reference's
// zero set, so the walk (and its float sums) stays deterministic.
__global__ void k_zero_sort_keys(const int32_t* __restrict__ cand, int ndim, int64_t rows,
                                 const long long* __restrict__ q_rows, int bmode, long long bdim, int nb, int b0,
                                 int s0, int kb, uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t R = *q_rows;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t* c = cand + i * ndim;
    const int32_t c0 = c[0];
    uint32_t key = 1u << kb;
    if (i < R && c0 >= 0) {
      const uint32_t b = (uint32_t)(((long long)c[bmode] * nb) / bdim);
      key = (b << b0) | ((uint32_t)c0 >> s0);
    }
    keys[i] = key;
    vals[i] = (int32_t)i;
  }
}

__global__ void k_zero_sorted_gather(const int32_t* __restrict__ cand, int ndim, const int32_t* __restrict__ idx,
                                     int64_t q, int32_t* __restrict__ out) {
  const int64_t total = q * ndim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / ndim;
    out[e] = __ldg(cand + (int64_t)__ldg(idx + j) * ndim + (e - j * ndim));
  }
}

static int bits_for(int64_t n) {  // bits to hold values 0 .. n-1
  int b = 0;
  while (b < 62 && ((int64_t)1 << b) < n) ++b;
  return b;
}

// Sort the lazy layout's accepted zero rows into the bucketed walk order (see
// k_zero_sort_keys); returns the [q x ndim] sorted rows in scr.zsorted.
static const int32_t* sort_zero_rows(Ctx* ctx, const Slice* X, DrawScratch& scr, int64_t rows, int64_t q,
                                     const long long* q_rows) {
  cudaStream_t s = ctx->stream;
  const int d = X->ndim;
  const int nbb = bits_for(X->nbuckets);
  const int i0b = bits_for(X->dims[0]);
  // sort_zeros 2: bucket only (a one-digit radix pass); 1: bucket, then mode-0 row
  const int b0 = ctx->sort_zeros == 2 ? 0 : std::min(i0b, 30 - nbb);
  const int s0 = i0b - b0;
  const int kb = nbb + b0;
  scr.zkey.ensure((size_t)rows * 4);
  scr.zkey_s.ensure((size_t)rows * 4);
  scr.zval.ensure((size_t)rows * 4);
  scr.zval_s.ensure((size_t)rows * 4);
  scr.zsorted.ensure((size_t)std::max<int64_t>(q, 1) * d * 4);
  const int grid = (int)std::min<int64_t>((rows + 255) / 256, (int64_t)kNumSMs * 8);
  k_zero_sort_keys<<<grid, 256, 0, s>>>(scr.cand.as<int32_t>(), d, rows, q_rows, X->bucket_mode,
                                        (long long)X->dims[X->bucket_mode], X->nbuckets, b0, s0, kb,
                                        scr.zkey.as<uint32_t>(), scr.zval.as<int32_t>());
  size_t tb = 0;
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, scr.zkey.as<uint32_t>(), scr.zkey_s.as<uint32_t>(),
                                            scr.zval.as<int32_t>(), scr.zval_s.as<int32_t>(), (int)rows, 0, kb + 1,
                                            s));
  scr.ztmp.ensure(tb);
  OGCP_CUDA(cub::DeviceRadixSort::SortPairs(scr.ztmp.ptr, tb, scr.zkey.as<uint32_t>(), scr.zkey_s.as<uint32_t>(),
                                            scr.zval.as<int32_t>(), scr.zval_s.as<int32_t>(), (int)rows, 0, kb + 1,
                                            s));
  const int ggrid = (int)std::min<int64_t>((q * d + 255) / 256, (int64_t)kNumSMs * 8);
  k_zero_sorted_gather<<<ggrid, 256, 0, s>>>(scr.cand.as<int32_t>(), d, scr.zval_s.as<int32_t>(), q,
                                             scr.zsorted.as<int32_t>());
  ctx->count(2 + (kb + 8) / 8);
  return scr.zsorted.as<int32_t>();
}

// Merged form, second half: the 4-bit counters of ordinals [olo, olo + own) ->
// (ordinal or bucketed position, multiplicity) in ascending order, certified by
// Σ counters = *owned (the draws that landed in the range); the distinct count
// lands in sc[5] (merged->count), the counter sum in sc[7].
static void merged_compact(Ctx* ctx, MergedDraw* merged, const uint32_t* counters, uint32_t olo, int64_t own,
                           const unsigned long long* owned, long long* sc,
                           unsigned long long* cnt_sum_out = nullptr) {
  cudaStream_t s = ctx->stream;
  const int64_t nwords = (own + 7) / 8;
  // (the caller sized merged->ord / cnt for min(p, own) entries)
  if (merged->perm) {  // emit in the slice's bucketed position order
    merged->pnib.ensure((size_t)std::max<int64_t>(nwords, 1) * 4);
    k_hist_permute<<<std::max<int64_t>(1, std::min<int64_t>((nwords + 255) / 256, kNumSMs * 16)), 256, 0, s>>>(
        counters, merged->perm, own, nwords, merged->pnib.as<uint32_t>(), (int32_t)olo);
    ctx->count();
    counters = merged->pnib.as<uint32_t>();
  }
  const int64_t hblocks = std::max<int64_t>(1, (nwords + (int64_t)kHistWordsPerThread * kScanThreads - 1) /
                                                   ((int64_t)kHistWordsPerThread * kScanThreads));
  merged->bcount.ensure((size_t)hblocks * 4);
  merged->boff.ensure((size_t)hblocks * 8);
  unsigned long long* cnt_sum = cnt_sum_out ? cnt_sum_out : reinterpret_cast<unsigned long long*>(sc + 7);
  k_hist_count<<<(unsigned)hblocks, kScanThreads, 0, s>>>(counters, nwords, merged->bcount.as<uint32_t>(), cnt_sum);
  if (owned) {
    k_hist_verify<<<1, 32, 0, s>>>(cnt_sum, owned, ctx->flags.as<DevFlags>());
    ctx->count();
  }
  k_zero_scan<<<1, 1024, 0, s>>>(merged->bcount.as<uint32_t>(), hblocks, merged->boff.as<long long>(), sc + 5);
  // positions (bucketed copy) are local; unbucketed ordinals are global
  k_hist_write<<<(unsigned)hblocks, kScanThreads, 0, s>>>(counters, nwords, own, merged->boff.as<long long>(),
                                                          merged->ord.as<int32_t>(), merged->cnt.as<uint8_t>(),
                                                          merged->perm ? 0 : (int32_t)olo);
  ctx->count(3);
  merged->count = sc + 5;
}

// Enqueue one stratified draw.  ordinals: int32 [p]; zero_subs: int32 [q x ndim].
// code: event code (event*4) recorded on sampling errors / shortfall.
DrawOut draw_enqueue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget,
                     int32_t* ordinals, int32_t* zero_subs, long long code, DrawScratch& scr, MergedDraw* merged,
                     bool lazy, bool semi) {
  DrawOut out;
  out.zsub = zero_subs;
  out.q_dev = nullptr;
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
  // the draw's scalars start at zero: a memset, or the first (fused) kernel clears them
  bool clear_in_kernel = false;
  if (!merged && p > 0 && eta > 1) {
    const double r = reject_rate((uint32_t)eta);
    const double w = ((double)p / (1.0 - r) + 10.0 * std::sqrt((double)p * r) / (1.0 - r) + 2048.0) * ctx->slack;
    const int64_t nchunks = std::max<int64_t>(1, ((int64_t)w + kChunkWords - 1) / kChunkWords);
    clear_in_kernel = (nchunks + kScanThreads - 1) / kScanThreads <= kFusedMaxTiles;
  }
  if (!clear_in_kernel) OGCP_CUDA(cudaMemsetAsync(sc, 0, 16 * 8, s));
  StreamSpec sp;
  sp.st_hi = (unsigned long long)(g.state >> 64);
  sp.st_lo = (unsigned long long)g.state;
  sp.inc_hi = (unsigned long long)(g.inc >> 64);
  sp.inc_lo = (unsigned long long)g.inc;
  const double slack = ctx->slack;

  // ---- nonzero stratum: integers(0, eta, size=p)  (sampling.py:125)
  bool nz_stream = false;
  bool nz_self_reported = false;
  if (merged && (p == 0 || eta < 2)) throw Error(OGCP_E_INTERNAL, "merged draw needs p > 0 and eta > 1");
  if (p > 0) {
    if (eta == 1) {
      k_fill_i32<<<std::min(ceil_div_i(p, 256), kNumSMs * 4), 256, 0, s>>>(ordinals, p, 0);
      ctx->count();
    } else {
      sp.ncol = 1;
      sp.n[0] = (uint32_t)eta;
      sp.thr[0] = lemire_threshold((uint32_t)eta);
      const double r = reject_rate((uint32_t)eta);
      const double exp_words = (double)p / (1.0 - r);
      const double sd = std::sqrt((double)p * r) / (1.0 - r);
      const int64_t words = (int64_t)((exp_words + 10.0 * sd + 2048.0) * slack);
      if (merged) {
        // counters for this rank's ordinal range [olo, ohi) (the whole slice on one GPU)
        const uint32_t olo = merged->ohi ? merged->olo : 0u;
        const uint32_t ohi = merged->ohi ? merged->ohi : (uint32_t)eta;
        const int64_t own = (int64_t)ohi - olo;
        const int64_t nwords = (own + 7) / 8;
        merged->hist.ensure((size_t)std::max<int64_t>(nwords, 1) * 4);
        merged->ord.ensure((size_t)std::max<int64_t>(std::min(p, own), 1) * 4);
        merged->cnt.ensure((size_t)std::max<int64_t>(std::min(p, own), 1));
        OGCP_CUDA(cudaMemsetAsync(merged->hist.ptr, 0, (size_t)std::max<int64_t>(nwords, 1) * 4, s));
        unsigned long long* owned = reinterpret_cast<unsigned long long*>(sc + 9);
        // one generating pass (count + counters), the tile scan, the trim of the slack
        const int64_t nchunks = std::max<int64_t>(1, (words + kChunkWords - 1) / kChunkWords);
        const int64_t nblocks = (nchunks + kScanThreads - 1) / kScanThreads;
        scr.bagg.ensure((size_t)nblocks * 4);
        scr.bstart.ensure((size_t)nblocks * 16);
        k_draw_count_hist<<<(unsigned)nblocks, kScanThreads, draw_stage_smem(true), s>>>(
            sp, nullptr, nchunks, scr.bagg.as<uint32_t>(), 0, merged->hist.as<uint32_t>(), olo, ohi, owned);
        k_draw_scan_tiles<1><<<1, kScanTilesThreads, 0, s>>>(scr.bagg.as<uint32_t>(), nblocks,
                                                             scr.bstart.as<long long>(), nz_avail);
        k_draw_trim<<<kNumSMs, kScanThreads, 0, s>>>(sp, nullptr, nchunks, scr.bstart.as<long long>(), nblocks,
                                                     nz_avail, p, 0, nblocks, merged->hist.as<uint32_t>(), olo, ohi,
                                                     owned, nz_end);
        ctx->count(3);
        check_launch();
        merged_compact(ctx, merged, merged->hist.as<uint32_t>(), olo, own, owned, sc);
      } else {
        // q == 0: nothing follows, so the fused pass reports its own shortfall
        run_stream<1>(ctx, sp, nullptr, p, words, ordinals, nz_end, nz_avail, scr, nullptr, 0, 0, nullptr,
                      q == 0 ? ctx->flags.as<DevFlags>() : nullptr, code, &nz_self_reported,
                      clear_in_kernel ? sc : nullptr);
        if (clear_in_kernel && !nz_self_reported) throw Error(OGCP_E_INTERNAL, "fused draw expected");
        if (q != 0) nz_self_reported = false;
      }
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
    if (semi) {
      // semi-stratified: the first q uniform cells of the box, no rejection
      if (ncol > 0) {
        const int64_t target = q * ncol;
        scr.cand.ensure((size_t)target * 4);
        const double exp_words = (double)target / (1.0 - rmax);
        const double sd = std::sqrt((double)target * rmax) / (1.0 - rmax);
        const int64_t words = (int64_t)((exp_words + 10.0 * sd + 2048.0) * slack);
        const long long* w0 = nz_stream ? nz_end : nullptr;
        run_stream_dispatch(ncol, ctx, sp, w0, target, words, scr.cand.as<int32_t>(), nullptr, z_elems, scr);
      } else {
        k_set_ll<<<1, 1, 0, s>>>(z_elems, 0);
        ctx->count();
      }
      if (ncol == d) {
        out.zsub = scr.cand.as<int32_t>();
      } else {
        k_expand_rows<<<std::min(ceil_div_i(q, 256), kNumSMs * 4), 256, 0, s>>>(zs, scr.cand.as<int32_t>(), q,
                                                                               zero_subs);
        ctx->count();
      }
      k_semi_status<<<1, 1, 0, s>>>(nz_stream ? p : 0, nz_avail, (long long)q * ncol, z_elems, code,
                                    ctx->flags.as<DevFlags>());
      ctx->count();
      check_launch();
      return out;
    }
    const double rho = X->omega_d > 0 ? (double)eta / X->omega_d : 0.0;
    const double exp_rows = rho < 1.0 ? (double)q / (1.0 - rho) : 1e30;
    const double sd_rows = rho < 1.0 ? std::sqrt((double)q * rho) / (1.0 - rho) : 1e30;
    const double want = (exp_rows + 10.0 * sd_rows + 64.0) * slack;
    const double cap = (double)q + (double)budget + 1.0;
    rows_max = (int64_t)std::min(want, cap);
    if (rows_max < q) rows_max = q;
    const int64_t nthreads = (rows_max + kRowsPerThread - 1) / kRowsPerThread;
    const int64_t zblocks = (nthreads + kScanThreads - 1) / kScanThreads;
    scr.miss.ensure((size_t)zblocks * kScanThreads);
    scr.zcount.ensure((size_t)zblocks * 4);
    scr.zoff.ensure((size_t)zblocks * 8);
    const unsigned long long* table = eta > 0 ? X->hash.as<unsigned long long>() : nullptr;
    if (ncol > 0) {
      const int64_t target = rows_max * ncol;
      scr.cand.ensure((size_t)target * 4);
      const double exp_words = (double)target / (1.0 - rmax);
      const double sd = std::sqrt((double)target * rmax) / (1.0 - rmax);
      const int64_t words = (int64_t)((exp_words + 10.0 * sd + 2048.0) * slack);
      const long long* w0 = nz_stream ? nz_end : nullptr;
      run_stream_dispatch(ncol, ctx, sp, w0, target, words, scr.cand.as<int32_t>(), nullptr, z_elems, scr);
    } else {
      // every mode has size 1: each candidate is the origin and no words are consumed
      k_set_ll<<<1, 1, 0, s>>>(z_elems, 0);
      ctx->count();
    }
    // In-place layout when no mode has size 1: the candidate rows are already
    // [row][d] coordinates, so when the first q candidates all miss (the usual
    // case for sparse slices) they are the accepted zeros and no compaction runs.
    const bool in_place = ncol == d;
    const bool mark = lazy && in_place;
    if (mark && rows_max <= kFusedMaxTiles * kRowsPerBlock) {  // small stratum: one fused block
      k_zero_fused<<<1, kScanThreads, 0, s>>>(zs, scr.cand.as<int32_t>(), z_elems, rows_max, table, X->table_mask,
                                              X->filter_mask ? X->filter.as<unsigned int>() : nullptr,
                                              X->filter_mask, q, sc + 8, z_hits_before, z_misses,
                                              nz_stream ? p : 0, nz_avail, (long long)budget, code,
                                              ctx->flags.as<DevFlags>(), DrawBatch{nullptr, 0, 0, 0});
      ctx->count();
      check_launch();
      out.zsub = scr.cand.as<int32_t>();
      out.q_dev = sc + 8;
      return out;
    }
    unsigned long long* hit_in_q =
        (in_place && !lazy) ? reinterpret_cast<unsigned long long*>(sc + 6) : nullptr;
    k_zero_hits<<<(unsigned)zblocks, kScanThreads, 0, s>>>(zs, scr.cand.as<int32_t>(), z_elems, rows_max, table,
                                                           X->table_mask, scr.miss.as<uint8_t>(),
                                                           scr.zcount.as<uint32_t>(), q, hit_in_q, mark ? 1 : 0,
                                                           X->filter_mask ? X->filter.as<unsigned int>() : nullptr,
                                                           X->filter_mask);
    k_zero_scan<<<1, 1024, 0, s>>>(scr.zcount.as<uint32_t>(), zblocks, scr.zoff.as<long long>(), z_misses);
    ctx->count(2);
    if (mark) {
      // lazy layout: the kernels walk candidate rows [0, R) and skip the flagged hits
      k_zero_locate<<<1, kScanThreads, 0, s>>>(scr.zcount.as<uint32_t>(), scr.zoff.as<long long>(), zblocks,
                                               scr.miss.as<uint8_t>(), rows_max, q, sc + 8, z_hits_before);
      ctx->count();
      if (merged && merged->perm && ctx->sort_zeros > 0 && X->bucket_mode > 0 && q >= 65536 && rows_max < INT32_MAX) {
        out.zsub = sort_zero_rows(ctx, X, scr, rows_max, q, sc + 8);  // exactly q rows, walk order
        out.q_dev = nullptr;
      } else {
        out.zsub = scr.cand.as<int32_t>();
        out.q_dev = sc + 8;
      }
    } else {
      const size_t smem = (size_t)kRowsPerBlock * d * 4;
      if (smem > 48 * 1024)
        OGCP_CUDA(cudaFuncSetAttribute(k_zero_compact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_zero_compact<<<(unsigned)zblocks, kScanThreads, smem, s>>>(zs, scr.cand.as<int32_t>(), rows_max,
                                                                   scr.miss.as<uint8_t>(), scr.zoff.as<long long>(),
                                                                   q, zero_subs, z_hits_before, hit_in_q);
      ctx->count();
      if (in_place) {
        k_zero_copyback<<<std::min(ceil_div_i(q * d, 256), kNumSMs * 4), 256, 0, s>>>(hit_in_q, zero_subs,
                                                                                     scr.cand.as<int32_t>(), q * d);
        ctx->count();
        out.zsub = scr.cand.as<int32_t>();
      }
    }
  }
  if (q == 0 && (!nz_stream || nz_self_reported)) return out;  // nothing left to check
  k_draw_status<<<1, 1, 0, s>>>(nz_stream ? p : 0, nz_avail, q, z_misses, rows_max, ncol, z_elems, z_hits_before,
                                (long long)budget, code, ctx->flags.as<DevFlags>());
  ctx->count();
  check_launch();
  return out;
}

// ---------------------------------------------------------------------------
// Word-range sharded merged draws (multi-GPU; sampler.cuh ShardScratch).  Rank r
// of N generates the stream tiles [r S, (r + 1) S), S = ceil(tiles / N), of both
// strata; everything a rank needs from the others is small (per-tile aggregate
// maps, per-rank zero-row records) except the nibble counters, which are
// reduce-scattered to the ordinal owners (eta / 2 bytes in total).

// Per-chunk map of the words of one thread's chunk (the counting loop of k_draw_count).
template <int NCOL>
__device__ __forceinline__ Map<NCOL> chunk_map(WordGen& g, const StreamSpec& sp) {
  Map<NCOL> m = identity_map<NCOL>();
  int col[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) col[c] = c;
#pragma unroll 4
  for (int i = 0; i < kChunkWords; ++i) {
    const uint32_t w = g.next();
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const int cc = col[c];
      uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
      for (int j = 1; j < NCOL; ++j)
        if (j == cc) { n = sp.n[j]; thr = sp.thr[j]; }
      if ((uint32_t)((uint64_t)w * n) >= thr) {
        m.c[c] += 1;
        col[c] = cc + 1 == NCOL ? 0 : cc + 1;
      }
    }
  }
  return m;
}

// The word after element target-1 of the stream (what k_draw_write records as
// end_word), found by re-generating the one tile that holds it.
template <int NCOL>
__global__ void __launch_bounds__(kScanThreads) k_draw_locate_end(StreamSpec sp, const long long* w0p, int64_t nchunks,
                                                                  const long long* __restrict__ bstart,
                                                                  int64_t nblocks, const long long* __restrict__ total,
                                                                  int64_t target, long long* __restrict__ end_word) {
  __shared__ long long tb;
  if (threadIdx.x == 0) {
    tb = -1;
    if (target > 0 && *total >= target) {
      int64_t lo = 0, hi = nblocks - 1;  // last tile whose first element is <= target-1
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (bstart[mid * 2 + 1] <= target - 1) lo = mid;
        else hi = mid - 1;
      }
      tb = lo;
    }
  }
  __syncthreads();
  if (tb < 0) return;
  const int64_t tile = tb;
  const int64_t chunk = tile * kScanThreads + threadIdx.x;
  WordGen g = tile_wordgen(sp, w0p, tile);
  WordGen g0 = g;
  Map<NCOL> m = identity_map<NCOL>();
  if (chunk < nchunks) m = chunk_map<NCOL>(g, sp);
  Map<NCOL> excl, agg;
  block_scan_maps<NCOL>(m, excl, agg);
  const int bcol = (int)bstart[tile * 2 + 0];
  const uint32_t adv = map_at<NCOL>(excl, bcol);
  int col = (int)((bcol + adv) % NCOL);
  long long e = bstart[tile * 2 + 1] + adv;
  if (chunk >= nchunks || e > target - 1) return;
  uint64_t w = tile_word0(w0p, tile) + (uint64_t)threadIdx.x * kChunkWords;
  for (int i = 0; i < kChunkWords && e < target; ++i, ++w) {
    const uint32_t word = g0.next();
    uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
    for (int j = 1; j < NCOL; ++j)
      if (j == col) { n = sp.n[j]; thr = sp.thr[j]; }
    if ((uint32_t)((uint64_t)word * n) >= thr) {
      if (e == target - 1) *end_word = (long long)(w + 1);
      ++e;
      col = col + 1 == NCOL ? 0 : col + 1;
    }
  }
}

// This rank's zero candidate rows: the rows whose first element lies in its
// element range [E(r S), E((r + 1) S)) (complete rows only, clipped to the
// provisioned target).  zr: [0] first row, [1] end row, [2] local elements,
// [3] element shift (ncol x first row), [4] element limit (ncol x end row),
// [5] end of its own element range, [6] first tile after its range.
__global__ void k_zshard_range(const long long* __restrict__ bst, int64_t nblocks, const long long* __restrict__ total,
                               int64_t target, int64_t slot, int rank, int world, int ncol, long long* __restrict__ zr,
                               long long* __restrict__ rec_rows) {
  if (threadIdx.x || blockIdx.x) return;
  const long long tlim = min(*total, (long long)target);
  const int64_t blo = (int64_t)rank * slot, bhi = min((int64_t)(rank + 1) * slot, nblocks);
  const long long elo = blo < nblocks ? min(bst[blo * 2 + 1], tlim) : tlim;
  const long long ehi = (rank == world - 1 || bhi >= nblocks) ? tlim : min(bst[bhi * 2 + 1], tlim);
  const long long rows_all = tlim / ncol;
  long long rhi = rank == world - 1 ? rows_all : min((ehi + ncol - 1) / ncol, rows_all);
  long long rlo = min(min((elo + ncol - 1) / ncol, rows_all), rhi);
  zr[0] = rlo;
  zr[1] = rhi;
  zr[2] = (rhi - rlo) * ncol;
  zr[3] = rlo * ncol;
  zr[4] = rhi * ncol;
  zr[5] = ehi;
  zr[6] = bhi;
  *rec_rows = rhi - rlo;
}

// The elements of this rank's last row past its own tiles (< ncol of them, the
// first accepted words of the next tile).
template <int NCOL>
__global__ void k_zshard_tail(StreamSpec sp, const long long* w0p, const long long* __restrict__ bst, int64_t nblocks,
                              const long long* __restrict__ zr, int32_t* __restrict__ out) {
  const long long lim = zr[4], ehi = zr[5], shift = zr[3];
  const int64_t tile = zr[6];
  if (zr[1] <= zr[0] || lim <= ehi || tile >= nblocks) return;
  WordGen g = tile_wordgen(sp, w0p, tile);  // thread 0's chunk starts at the tile's first word
  if (threadIdx.x != 0) return;
  int col = (int)bst[tile * 2 + 0];
  long long e = bst[tile * 2 + 1];
  while (e < lim) {
    const uint32_t word = g.next();
    uint32_t n = sp.n[0], thr = sp.thr[0];
#pragma unroll
    for (int j = 1; j < NCOL; ++j)
      if (j == col) { n = sp.n[j]; thr = sp.thr[j]; }
    const uint64_t prod = (uint64_t)word * n;
    if ((uint32_t)prod >= thr) {
      if (e >= shift) out[e - shift] = (int32_t)(prod >> 32);
      ++e;
      col = col + 1 == NCOL ? 0 : col + 1;
    }
  }
}

// Locate the q-th miss from the all-gathered (misses, rows) records: the rank
// holding it finds its local row (rows_used = local row + 1, hits_before = the
// reference's rejection count); ranks before it use all their rows, ranks after
// it none.  Status as k_draw_status: a nonzero shortfall asks for a retry; with
// fewer than q misses in all ranks' rows, more than `budget` hits is the
// reference's SamplingError, else a shortfall.
// The records also carry every owner's counter sum: all of them together must
// be p (a wrapped nibble loses 16), else the merge-overflow bit sends the epoch
// back to per-draw evaluation, as k_hist_verify does on one GPU (check_counts 0:
// timing simulation, whose stand-in records do not add up).
constexpr int kZrec = 3;  // (misses, rows, counter sum) per rank
__global__ void __launch_bounds__(kScanThreads) k_zshard_cut(
    const long long* __restrict__ rec, int world, int rank, int64_t q, long long budget,
    const long long* __restrict__ zr, const uint32_t* __restrict__ bcount, const long long* __restrict__ boff,
    int64_t nblocks, const uint8_t* __restrict__ miss, int64_t lrows_max, long long* __restrict__ rows_used,
    long long* __restrict__ hits_before, const long long* __restrict__ nz_avail, int64_t p, long long code,
    int check_counts, DevFlags* flags) {
  __shared__ long long t_loc;
  __shared__ int holds;
  const bool nz_short = p > 0 && *nz_avail < p;
  if (threadIdx.x == 0) {
    long long before = 0, mt = 0, nt = 0;
    unsigned long long drawn = 0;
    for (int s = 0; s < world; ++s) {
      if (s < rank) before += rec[kZrec * s];
      mt += rec[kZrec * s];
      nt += rec[kZrec * s + 1];
      drawn += (unsigned long long)rec[kZrec * s + 2];
    }
    if (check_counts && !nz_short && drawn != (unsigned long long)p) atomicOr(&flags->data_bits, kMergeOverflowBit);
    const long long mine = rec[kZrec * rank], rows = rec[kZrec * rank + 1];
    const long long t = q - before;
    *hits_before = 0;
    holds = 0;
    if (t <= 0) *rows_used = 0;
    else if (t > mine) *rows_used = rows;
    else holds = 1;
    t_loc = t;
    bool exhausted = false, shortfall = nz_short;
    if (!nz_short && mt < q) {
      if (nt - mt > budget) exhausted = true;
      else shortfall = true;
    }
    if (exhausted) atomicMin(&flags->first_code[kFlagSampling], code);
    else if (shortfall) atomicMin(&flags->first_code[kFlagShortfall], code);
  }
  __syncthreads();
  if (!holds) return;
  zero_locate_body(bcount, boff, nblocks, miss, lrows_max, t_loc, rows_used, hits_before, zr[0], q);
  __syncthreads();
  if (threadIdx.x == 0 && !nz_short && *hits_before > budget) atomicMin(&flags->first_code[kFlagSampling], code);
}

template <typename T>
__global__ void k_add_into(T* __restrict__ dst, const T* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

void shard_owner_range(int64_t eta, int rank, int world, int64_t* olo, int64_t* ohi) {
  const int64_t cw = ((eta + 7) / 8 + world - 1) / world;
  *olo = std::min<int64_t>(8 * cw * rank, eta);
  *ohi = std::min<int64_t>(8 * cw * (rank + 1), eta);
}

bool shard_draw_eligible(const Ctx* ctx, const Slice* X, int64_t p, int64_t q, bool semi) {
  if (!ctx->shard_draws || ctx->world < 2) return false;
  if (!ctx->comm_draw && !ctx->shard_sim) return false;
  if (semi || p <= 0 || q <= 0 || X->nnz < 2 || X->ndim > kMaxCols) return false;
  for (int k = 0; k < X->ndim; ++k)
    if (X->dims[k] < 2) return false;  // the in-place lazy layout (every mode consumes words)
  return true;
}

namespace {

struct ShardPlan {
  int world = 1, ncol = 0;
  int64_t eta = 0, p = 0, q = 0, budget = 0;
  StreamSpec spn, spz;
  ZeroSpec zs;
  int64_t n_nchunks = 0, n_nblocks = 0, n_slot = 0;
  int64_t z_nchunks = 0, z_nblocks = 0, z_slot = 0, z_target = 0;
  int64_t lrows_max = 0, lzblocks = 0, cw = 0;
};

ShardPlan shard_plan(const Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget) {
  ShardPlan pl;
  const int W = ctx->world;
  const int d = X->ndim;
  pl.world = W;
  pl.eta = X->nnz;
  pl.p = p;
  pl.q = q;
  pl.budget = budget;
  StreamSpec sp;
  sp.st_hi = (unsigned long long)(g.state >> 64);
  sp.st_lo = (unsigned long long)g.state;
  sp.inc_hi = (unsigned long long)(g.inc >> 64);
  sp.inc_lo = (unsigned long long)g.inc;
  const double slack = ctx->slack;
  // nonzero stratum: integers(0, eta, size=p), words provisioned as draw_enqueue does
  pl.spn = sp;
  pl.spn.ncol = 1;
  pl.spn.n[0] = (uint32_t)pl.eta;
  pl.spn.thr[0] = lemire_threshold((uint32_t)pl.eta);
  {
    const double r = reject_rate((uint32_t)pl.eta);
    const int64_t words = (int64_t)(((double)p / (1.0 - r) + 10.0 * std::sqrt((double)p * r) / (1.0 - r) + 2048.0) *
                                    slack);
    pl.n_nchunks = std::max<int64_t>(1, (words + kChunkWords - 1) / kChunkWords);
    pl.n_nblocks = (pl.n_nchunks + kScanThreads - 1) / kScanThreads;
    pl.n_slot = (pl.n_nblocks + W - 1) / W;
  }
  pl.cw = ((pl.eta + 7) / 8 + W - 1) / W;
  // zero stratum: candidate rows as draw_enqueue provisions them (every mode consumes words)
  pl.spz = sp;
  pl.ncol = d;
  pl.spz.ncol = d;
  pl.zs.ndim = d;
  pl.zs.ncol = d;
  double rmax = 0.0;
  for (int k = 0; k < kMaxModes; ++k) {
    pl.zs.colmap[k] = k < d ? k : -1;
    pl.zs.st.s[k] = k < d ? X->strides[k] : 0;
  }
  for (int k = 0; k < d; ++k) {
    pl.spz.n[k] = (uint32_t)X->dims[k];
    pl.spz.thr[k] = lemire_threshold((uint32_t)X->dims[k]);
    rmax = std::max(rmax, reject_rate((uint32_t)X->dims[k]));
  }
  const double rho = X->omega_d > 0 ? (double)pl.eta / X->omega_d : 0.0;
  const double exp_rows = rho < 1.0 ? (double)q / (1.0 - rho) : 1e30;
  const double sd_rows = rho < 1.0 ? std::sqrt((double)q * rho) / (1.0 - rho) : 1e30;
  const double want = (exp_rows + 10.0 * sd_rows + 64.0) * slack;
  const double cap = (double)q + (double)budget + 1.0;
  int64_t rows_max = (int64_t)std::min(want, cap);
  if (rows_max < q) rows_max = q;
  pl.z_target = rows_max * d;
  {
    const double exp_words = (double)pl.z_target / (1.0 - rmax);
    const double sd = std::sqrt((double)pl.z_target * rmax) / (1.0 - rmax);
    const int64_t words = (int64_t)((exp_words + 10.0 * sd + 2048.0) * slack);
    pl.z_nchunks = std::max<int64_t>(1, (words + kChunkWords - 1) / kChunkWords);
    pl.z_nblocks = (pl.z_nchunks + kScanThreads - 1) / kScanThreads;
    pl.z_slot = (pl.z_nblocks + W - 1) / W;
  }
  // a rank's rows start in its own elements: at most (its words) / d + 1 of them
  pl.lrows_max = std::min<int64_t>(rows_max, pl.z_slot * (int64_t)kBlockWords / d + 1);
  pl.lzblocks = ((pl.lrows_max + kRowsPerThread - 1) / kRowsPerThread + kScanThreads - 1) / kScanThreads;
  return pl;
}

void shard_alloc(const ShardPlan& pl, ShardScratch& sh, int d) {
  const int W = pl.world;
  sh.tm_z.ensure((size_t)pl.z_slot * kScanThreads * pl.ncol);
  sh.bagg_nz.ensure((size_t)W * pl.n_slot * 4);
  sh.bagg_z.ensure((size_t)W * pl.z_slot * pl.ncol * 4);
  sh.bst_nz.ensure((size_t)pl.n_nblocks * 16);
  sh.bst_z.ensure((size_t)pl.z_nblocks * 16);
  sh.hist.ensure((size_t)W * pl.cw * 4);
  sh.zrec.ensure((size_t)W * kZrec * 8);
  sh.scal.ensure(16 * 8);
  sh.cand.ensure((size_t)std::max<int64_t>(pl.lrows_max, 1) * d * 4);
  sh.miss.ensure((size_t)pl.lzblocks * kScanThreads);
  sh.zcount.ensure((size_t)pl.lzblocks * 4);
  sh.zoff.ensure((size_t)pl.lzblocks * 8);
}

template <int NCOL>
void zero_tiles(Ctx* ctx, const ShardPlan& pl, ShardScratch& sh, int r, bool count) {
  cudaStream_t s = ctx->stream;
  const int64_t b0 = (int64_t)r * pl.z_slot;
  const int64_t nt = std::max<int64_t>(0, std::min(pl.z_slot, pl.z_nblocks - b0));
  long long* sc = sh.scal.as<long long>();
  if (count) {
    if (nt > 0) {
      k_draw_count<NCOL><<<(unsigned)nt, kScanThreads, 0, s>>>(pl.spz, sc + 0, pl.z_nchunks, sh.tm_z.as<uint8_t>(),
                                                              sh.bagg_z.as<uint32_t>(), b0);
      ctx->count();
    }
    return;
  }
  k_draw_scan_tiles<NCOL><<<1, kScanTilesThreads, 0, s>>>(sh.bagg_z.as<uint32_t>(), pl.z_nblocks, sh.bst_z.as<long long>(),
                                                      sc + 2);
  k_zshard_range<<<1, 1, 0, s>>>(sh.bst_z.as<long long>(), pl.z_nblocks, sc + 2, pl.z_target, pl.z_slot, r, pl.world,
                                 NCOL, sc + 9, sh.zrec.as<long long>() + kZrec * r + 1);
  ctx->count(2);
  if (nt > 0) {
    k_draw_write<NCOL><<<(unsigned)nt, kScanThreads, kBlockWords * 4, s>>>(
        pl.spz, sc + 0, pl.z_nchunks, sh.tm_z.as<uint8_t>(), sh.bst_z.as<long long>(), pl.z_target,
        sh.cand.as<int32_t>(), nullptr, nullptr, ctx->flags.as<DevFlags>(), 0u, 0u, nullptr, b0, sc + 13, sc + 12);
    ctx->count();
  }
  k_zshard_tail<NCOL><<<1, 32, 0, s>>>(pl.spz, sc + 0, sh.bst_z.as<long long>(), pl.z_nblocks, sc + 9,
                                       sh.cand.as<int32_t>());
  ctx->count();
}

void zero_tiles_any(Ctx* ctx, const ShardPlan& pl, ShardScratch& sh, int r, bool count) {
  switch (pl.ncol) {
    case 2: zero_tiles<2>(ctx, pl, sh, r, count); break;
    case 3: zero_tiles<3>(ctx, pl, sh, r, count); break;
    case 4: zero_tiles<4>(ctx, pl, sh, r, count); break;
    case 5: zero_tiles<5>(ctx, pl, sh, r, count); break;
    case 6: zero_tiles<6>(ctx, pl, sh, r, count); break;
    case 7: zero_tiles<7>(ctx, pl, sh, r, count); break;
    default: throw Error(OGCP_E_INTERNAL, "sharded draw: unsupported mode count");
  }
}

// Rank r's part before the first exchange: the nonzero tiles' maps.
void phase_count(Ctx* ctx, const ShardPlan& pl, ShardScratch& sh, int r) {
  cudaStream_t s = ctx->stream;
  OGCP_CUDA(cudaMemsetAsync(sh.scal.ptr, 0, 16 * 8, s));
  OGCP_CUDA(cudaMemsetAsync(sh.zrec.ptr, 0, (size_t)pl.world * kZrec * 8, s));
  OGCP_CUDA(cudaMemsetAsync(sh.hist.ptr, 0, (size_t)pl.world * pl.cw * 4, s));
  const int64_t b0 = (int64_t)r * pl.n_slot;
  const int64_t nt = std::max<int64_t>(0, std::min(pl.n_slot, pl.n_nblocks - b0));
  if (nt > 0) {  // its tiles' counts and its draws into counters over all ordinals, one pass
    k_draw_count_hist<<<(unsigned)nt, kScanThreads, draw_stage_smem(true), s>>>(pl.spn, nullptr, pl.n_nchunks,
                                                                                 sh.bagg_nz.as<uint32_t>(),
                                                            b0, sh.hist.as<uint32_t>(), 0u, (uint32_t)pl.eta,
                                                            nullptr);
    ctx->count();
  }
}

// After the map all-gather: the stream scan, the nonzero end word, this rank's
// counters over all ordinals, and the zero stream's tile maps.
void phase_write(Ctx* ctx, const ShardPlan& pl, ShardScratch& sh, int r) {
  cudaStream_t s = ctx->stream;
  long long* sc = sh.scal.as<long long>();
  k_draw_scan_tiles<1><<<1, kScanTilesThreads, 0, s>>>(sh.bagg_nz.as<uint32_t>(), pl.n_nblocks, sh.bst_nz.as<long long>(),
                                                   sc + 1);
  k_draw_locate_end<1><<<1, kScanThreads, 0, s>>>(pl.spn, nullptr, pl.n_nchunks, sh.bst_nz.as<long long>(),
                                                  pl.n_nblocks, sc + 1, pl.p, sc + 0);
  ctx->count(2);
  const int64_t b0 = (int64_t)r * pl.n_slot;
  const int64_t b1 = std::min(b0 + pl.n_slot, pl.n_nblocks);
  if (b1 > b0) {  // the slack past element p - 1, if in its tiles
    k_draw_trim<<<4, kScanThreads, 0, s>>>(pl.spn, nullptr, pl.n_nchunks, sh.bst_nz.as<long long>(), pl.n_nblocks,
                                           sc + 1, pl.p, b0, b1, sh.hist.as<uint32_t>(), 0u, (uint32_t)pl.eta, nullptr,
                                           nullptr);
    ctx->count();
  }
  zero_tiles_any(ctx, pl, sh, r, /*count=*/true);
  check_launch();
}

// After the counter reduce-scatter and the zero maps' all-gather: this rank's zero
// candidate rows and their hit test (and, for the calling rank, the compaction of
// its merged nonzeros).
void phase_zero(Ctx* ctx, const ShardPlan& pl, ShardScratch& sh, int r, const Slice* X) {
  cudaStream_t s = ctx->stream;
  long long* sc = sh.scal.as<long long>();
  zero_tiles_any(ctx, pl, sh, r, /*count=*/false);
  k_zero_hits<<<(unsigned)pl.lzblocks, kScanThreads, 0, s>>>(
      pl.zs, sh.cand.as<int32_t>(), sc + 11, pl.lrows_max, X->hash.as<unsigned long long>(), X->table_mask,
      sh.miss.as<uint8_t>(), sh.zcount.as<uint32_t>(), 0, nullptr, 1,
      X->filter_mask ? X->filter.as<unsigned int>() : nullptr, X->filter_mask);
  k_zero_scan<<<1, 1024, 0, s>>>(sh.zcount.as<uint32_t>(), pl.lzblocks, sh.zoff.as<long long>(),
                                 sh.zrec.as<long long>() + kZrec * r);
  ctx->count(2);
  check_launch();
}

enum class XMode { nccl, emulate, replicate };

__global__ void k_replicate_slot(uint8_t* __restrict__ buf, int64_t bytes, int r, int world) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < bytes * world;
       i += (int64_t)gridDim.x * blockDim.x)
    if (i / bytes != r) buf[i] = buf[(int64_t)r * bytes + i % bytes];
}

// All-gather of per-rank slots of `bytes`: NCCL, the other ranks' buffers (exact
// simulation), or this rank's own slot standing in for the others (timing
// simulation, plus the collective's stand-in kernel).
void xchg_allgather(Ctx* ctx, XMode xm, std::vector<ShardScratch*>& st, DevBuf ShardScratch::*mb, size_t bytes) {
  const int W = ctx->world, R = ctx->rank;
  if (xm == XMode::nccl) {
    comm_draw_allgather(ctx, (st[R]->*mb).ptr, bytes);
    return;
  }
  if (xm == XMode::replicate) {
    const int64_t n = (int64_t)bytes * W;
    k_replicate_slot<<<(unsigned)std::min<int64_t>((n + 255) / 256, kNumSMs * 4), 256, 0, ctx->stream>>>(
        static_cast<uint8_t*>((st[R]->*mb).ptr), (int64_t)bytes, R, W);
    ctx->count();
    comm_draw_allgather(ctx, nullptr, bytes);  // no draw communicator: the stand-in
    return;
  }
  for (int s = 0; s < W; ++s) {
    if (!st[s]) continue;
    char* dst = static_cast<char*>((st[s]->*mb).ptr);
    for (int o = 0; o < W; ++o) {
      if (o == s) continue;
      const char* src = st[o] ? static_cast<const char*>((st[o]->*mb).ptr) + o * bytes : dst + s * bytes;
      OGCP_CUDA(cudaMemcpyAsync(dst + o * bytes, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    }
  }
}

}  // namespace

DrawOut shard_draw_enqueue(Ctx* ctx, const Slice* X, const Pcg64& g, int64_t p, int64_t q, int64_t budget,
                           long long code, MergedDraw& md, ShardScratch& sh) {
  init_jump_table();
  ProfScope prof_scope(ctx, kProfDraw);
  const ShardPlan pl = shard_plan(ctx, X, g, p, q, budget);
  const int W = ctx->world, R = ctx->rank, d = X->ndim;
  cudaStream_t s = ctx->stream;
  const XMode xm = ctx->comm_draw ? XMode::nccl : (ctx->shard_sim_timing ? XMode::replicate : XMode::emulate);
  static thread_local std::vector<std::unique_ptr<ShardScratch>> emu;  // the other ranks' state (exact simulation)
  std::vector<ShardScratch*> st(W, nullptr);
  st[R] = &sh;
  if (xm == XMode::emulate) {
    if ((int)emu.size() < W) emu.resize(W);
    for (int r = 0; r < W; ++r)
      if (r != R) {
        if (!emu[r]) emu[r].reset(new ShardScratch);
        st[r] = emu[r].get();
      }
  }
  for (int r = 0; r < W; ++r)
    if (st[r]) shard_alloc(pl, *st[r], d);
  // 1. nonzero tile maps -> all-gather
  for (int r = 0; r < W; ++r)
    if (st[r]) phase_count(ctx, pl, *st[r], r);
  xchg_allgather(ctx, xm, st, &ShardScratch::bagg_nz, (size_t)pl.n_slot * 4);
  // 2. scan, end word, counters over all ordinals, zero tile maps -> reduce-scatter the
  //    counters, all-reduce the per-owner draw counts, all-gather the zero maps (one group)
  for (int r = 0; r < W; ++r)
    if (st[r]) phase_write(ctx, pl, *st[r], r);
  if (xm == XMode::nccl) {
    comm_draw_group(ctx, true);
    comm_draw_reduce_scatter_u32(ctx, sh.hist.as<uint32_t>(), (size_t)pl.cw);
    comm_draw_allgather(ctx, sh.bagg_z.ptr, (size_t)pl.z_slot * pl.ncol * 4);
    comm_draw_group(ctx, false);
  } else {
    if (xm == XMode::replicate) comm_draw_reduce_scatter_u32(ctx, nullptr, (size_t)pl.cw);  // the stand-in
    if (xm == XMode::emulate)  // every rank's chunk summed over the ranks (the reduce-scatter)
      for (int r = 0; r < W; ++r)
        for (int o = 0; o < W; ++o) {
          if (o == r) continue;
          k_add_into<uint32_t><<<kNumSMs * 4, 256, 0, s>>>(st[r]->hist.as<uint32_t>() + (size_t)r * pl.cw,
                                                           st[o]->hist.as<uint32_t>() + (size_t)r * pl.cw, pl.cw);
          ctx->count();
        }
    xchg_allgather(ctx, xm, st, &ShardScratch::bagg_z, (size_t)pl.z_slot * pl.ncol * 4);
  }
  // 3. this rank's merged nonzeros (owner range) from the summed counters; every
  //    rank's counter sum goes into its zero-row record for the cut's count check
  int64_t olo, ohi;
  shard_owner_range(pl.eta, R, W, &olo, &ohi);
  const int64_t own = ohi - olo;
  md.ord.ensure((size_t)std::max<int64_t>(std::min(p, own), 1) * 4);
  md.cnt.ensure((size_t)std::max<int64_t>(std::min(p, own), 1));
  long long* sc = sh.scal.as<long long>();
  merged_compact(ctx, &md, sh.hist.as<uint32_t>() + (size_t)R * pl.cw, (uint32_t)olo, own, nullptr, sc,
                 reinterpret_cast<unsigned long long*>(sh.zrec.as<long long>() + kZrec * R + 2));
  for (int r = 0; r < W; ++r) {
    if (r == R || !st[r]) continue;
    int64_t lo, hi;
    shard_owner_range(pl.eta, r, W, &lo, &hi);
    const int64_t nwords = (hi - lo + 7) / 8;
    const int64_t hblocks = std::max<int64_t>(1, (nwords + (int64_t)kHistWordsPerThread * kScanThreads - 1) /
                                                     ((int64_t)kHistWordsPerThread * kScanThreads));
    st[r]->zcount.ensure((size_t)hblocks * 4);
    k_hist_count<<<(unsigned)hblocks, kScanThreads, 0, s>>>(
        st[r]->hist.as<uint32_t>() + (size_t)r * pl.cw, nwords, st[r]->zcount.as<uint32_t>(),
        reinterpret_cast<unsigned long long*>(st[r]->zrec.as<long long>() + kZrec * r + 2));
    ctx->count();
  }
  // 4. zero rows -> all-gather the (misses, rows) records -> the cut
  for (int r = 0; r < W; ++r)
    if (st[r]) phase_zero(ctx, pl, *st[r], r, X);
  xchg_allgather(ctx, xm, st, &ShardScratch::zrec, kZrec * 8);
  k_zshard_cut<<<1, kScanThreads, 0, s>>>(sh.zrec.as<long long>(), W, R, q, (long long)budget, sc + 9,
                                          sh.zcount.as<uint32_t>(), sh.zoff.as<long long>(), pl.lzblocks,
                                          sh.miss.as<uint8_t>(), pl.lrows_max, sc + 8, sc + 4, sc + 1, p, code,
                                          xm == XMode::replicate ? 0 : 1, ctx->flags.as<DevFlags>());
  ctx->count();
  check_launch();
  DrawOut out;
  out.zsub = sh.cand.as<int32_t>();
  out.q_dev = sc + 8;
  return out;
}


// ---------------------------------------------------------------------------
// Batched small draws: every draw of a solver epoch (tau keyed generators,
// rng_at(seed, t, phase, epoch, it) for it < tau) in one launch per pass, one
// block per draw.  A draw depends only on the slice and its key (never on the
// iterate), so the epoch's draws can all be made before its first iteration;
// for the c1 / c2 shapes each draw is a chain of single-block kernels whose
// latency (~40 us at c2) otherwise sits on every iteration's critical path.
bool draw_batch_eligible(const Ctx* ctx, const Slice* X, int64_t p, int64_t q, int64_t budget, bool semi) {
  if (semi || X->ndim > kMaxModes) return false;
  if (p > 0 && X->nnz < 2) return false;
  const double slack = ctx->slack;
  if (p > 0) {
    const double r = reject_rate((uint32_t)X->nnz);
    const double w = ((double)p / (1.0 - r) + 10.0 * std::sqrt((double)p * r) / (1.0 - r) + 2048.0) * slack;
    const int64_t nchunks = std::max<int64_t>(1, ((int64_t)w + kChunkWords - 1) / kChunkWords);
    if ((nchunks + kScanThreads - 1) / kScanThreads > kFusedMaxTiles) return false;
  }
  if (q > 0) {
    for (int k = 0; k < X->ndim; ++k)
      if (X->dims[k] < 2) return false;  // the lazy in-place layout needs every mode to consume words
    const double rho = X->omega_d > 0 ? (double)X->nnz / X->omega_d : 0.0;
    if (rho >= 0.5) return false;
    const double rows = ((double)q / (1.0 - rho) + 10.0 * std::sqrt((double)q * rho) / (1.0 - rho) + 64.0) * slack;
    if (std::min(rows, (double)q + (double)budget + 1.0) > (double)kFusedMaxTiles * kRowsPerBlock) return false;
    double rmax = 0.0;
    for (int k = 0; k < X->ndim; ++k) rmax = std::max(rmax, reject_rate((uint32_t)X->dims[k]));
    const double target = rows * X->ndim;
    const double w = (target / (1.0 - rmax) + 10.0 * std::sqrt(target * rmax) / (1.0 - rmax) + 2048.0) * slack;
    const int64_t nchunks = std::max<int64_t>(1, ((int64_t)w + kChunkWords - 1) / kChunkWords);
    if ((nchunks + kScanThreads - 1) / kScanThreads > kFusedMaxTiles) return false;
  }
  return p > 0 || q > 0;
}

void draw_batch_enqueue(Ctx* ctx, const Slice* X, const Pcg64* gens, int n, int64_t p, int64_t q, int64_t budget,
                        long long code0, long long code_stride, DrawBatchSet& B) {
  init_jump_table();
  ProfScope prof_scope(ctx, kProfDraw);
  cudaStream_t s = ctx->stream;
  const int d = X->ndim;
  const double slack = ctx->slack;
  B.n = n;
  B.p = p;
  B.q = q;
  constexpr int64_t kScal = 16;
  B.scal.ensure((size_t)n * kScal * 8);
  OGCP_CUDA(cudaMemsetAsync(B.scal.ptr, 0, (size_t)n * kScal * 8, s));
  long long* sc = B.scal.as<long long>();
  std::vector<StreamSpec> hs(n);
  for (int b = 0; b < n; ++b) {
    hs[b].st_hi = (unsigned long long)(gens[b].state >> 64);
    hs[b].st_lo = (unsigned long long)gens[b].state;
    hs[b].inc_hi = (unsigned long long)(gens[b].inc >> 64);
    hs[b].inc_lo = (unsigned long long)gens[b].inc;
  }
  // nonzero stratum: integers(0, eta, p) per draw
  if (p > 0) {
    StreamSpec sp = hs[0];
    sp.ncol = 1;
    sp.n[0] = (uint32_t)X->nnz;
    sp.thr[0] = lemire_threshold((uint32_t)X->nnz);
    for (auto& h : hs) {
      h.ncol = sp.ncol;
      h.n[0] = sp.n[0];
      h.thr[0] = sp.thr[0];
    }
    B.specs.ensure((size_t)n * sizeof(StreamSpec));
    OGCP_CUDA(cudaMemcpyAsync(B.specs.ptr, hs.data(), (size_t)n * sizeof(StreamSpec), cudaMemcpyHostToDevice, s));
    const double r = reject_rate((uint32_t)X->nnz);
    const double w = ((double)p / (1.0 - r) + 10.0 * std::sqrt((double)p * r) / (1.0 - r) + 2048.0) * slack;
    const int64_t nchunks = std::max<int64_t>(1, ((int64_t)w + kChunkWords - 1) / kChunkWords);
    B.ord.ensure((size_t)n * p * 4);
    // q == 0: nothing follows, so the nonzero pass reports its own shortfall
    k_draw_fused<1><<<n, kScanThreads, 0, s>>>(sp, nullptr, nchunks, p, B.ord.as<int32_t>(), sc + 0, sc + 1,
                                               q == 0 ? ctx->flags.as<DevFlags>() : nullptr, code0, nullptr,
                                               DrawBatch{B.specs.as<StreamSpec>(), p, kScal, code_stride});
    ctx->count();
  }
  B.rows_max = 0;
  if (q > 0) {
    ZeroSpec zs;
    zs.ndim = d;
    StreamSpec sp;
    int ncol = 0;
    double rmax = 0.0;
    for (int k = 0; k < kMaxModes; ++k) {
      zs.colmap[k] = -1;
      zs.st.s[k] = k < d ? X->strides[k] : 0;
    }
    for (int k = 0; k < d; ++k) {
      sp.n[ncol] = (uint32_t)X->dims[k];
      sp.thr[ncol] = lemire_threshold((uint32_t)X->dims[k]);
      rmax = std::max(rmax, reject_rate((uint32_t)X->dims[k]));
      zs.colmap[k] = ncol++;
    }
    zs.ncol = ncol;
    sp.ncol = ncol;
    for (auto& h : hs) {
      h.ncol = sp.ncol;
      for (int c = 0; c < ncol; ++c) {
        h.n[c] = sp.n[c];
        h.thr[c] = sp.thr[c];
      }
    }
    B.zspecs.ensure((size_t)n * sizeof(StreamSpec));
    OGCP_CUDA(cudaMemcpyAsync(B.zspecs.ptr, hs.data(), (size_t)n * sizeof(StreamSpec), cudaMemcpyHostToDevice, s));
    const double rho = X->omega_d > 0 ? (double)X->nnz / X->omega_d : 0.0;
    const double want = ((double)q / (1.0 - rho) + 10.0 * std::sqrt((double)q * rho) / (1.0 - rho) + 64.0) * slack;
    int64_t rows_max = (int64_t)std::min(want, (double)q + (double)budget + 1.0);
    if (rows_max < q) rows_max = q;
    B.rows_max = rows_max;
    const int64_t target = rows_max * ncol;
    const double exp_words = (double)target / (1.0 - rmax);
    const double sd = std::sqrt((double)target * rmax) / (1.0 - rmax);
    const int64_t words = (int64_t)((exp_words + 10.0 * sd + 2048.0) * slack);
    const int64_t nchunks = std::max<int64_t>(1, (words + kChunkWords - 1) / kChunkWords);
    B.cand.ensure((size_t)n * target * 4);
    const DrawBatch zb{B.zspecs.as<StreamSpec>(), target, kScal, code_stride};
    auto launch = [&](auto kern) {
      kern<<<n, kScanThreads, 0, s>>>(sp, p > 0 ? sc + 0 : nullptr, nchunks, target, B.cand.as<int32_t>(), nullptr,
                                      sc + 2, nullptr, code0, nullptr, zb);
    };
    switch (ncol) {
      case 2: launch(k_draw_fused<2>); break;
      case 3: launch(k_draw_fused<3>); break;
      case 4: launch(k_draw_fused<4>); break;
      case 5: launch(k_draw_fused<5>); break;
      case 6: launch(k_draw_fused<6>); break;
      case 7: launch(k_draw_fused<7>); break;
      default: throw Error(OGCP_E_USAGE, "batched draws need 2..7 modes");
    }
    const unsigned long long* table = X->nnz > 0 ? X->hash.as<unsigned long long>() : nullptr;
    k_zero_fused<<<n, kScanThreads, 0, s>>>(zs, B.cand.as<int32_t>(), sc + 2, rows_max, table, X->table_mask,
                                            X->filter_mask ? X->filter.as<unsigned int>() : nullptr, X->filter_mask, q,
                                            sc + 8, sc + 4, sc + 3, p, p > 0 ? sc + 1 : nullptr, (long long)budget,
                                            code0, ctx->flags.as<DevFlags>(), zb);
    ctx->count(2);
  }
  check_launch();
}

}  // namespace ogcp
