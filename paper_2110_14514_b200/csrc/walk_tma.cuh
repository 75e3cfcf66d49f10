// TMA-fed sample walks (sm_100a): the merged nonzero set and the zero stratum of
// a 3-way slice, evaluated by warp-specialised CTAs whose factor-row gathers are
// issued by the Tensor Memory Accelerator.  Included by compute.cu after
// walk3.cuh (shares its Walk descriptor and loss helpers).
//
// Why: the register-pipelined walks keep one or two 8-sample batches of rows in
// flight per warp; with 16 warps per SM that is ~128 samples of gathers per SM,
// and ncu shows them long-scoreboard bound at ~55% of L2 throughput.  Here the
// rows of 16 stages x 32 samples (512 samples, ~200 KB) are in flight per SM
// without costing registers:
//
// * 8 producer warps fetch each tile's metadata (position -> record, or the
//   zero row) with a register pipeline two tiles deep per stage, write it to the
//   stage and issue the row gathers as cp.async.bulk.tensor.2d ... tile::gather4
//   (four 128-byte factor rows per instruction, UTMALDG.2D.GATHER4), completing
//   on the stage's mbarrier with an expect_tx byte count.  Mode-0 rows are
//   gathered once per distinct row of the tile (the bucketed walk is sorted by
//   mode-0 row, so runs of equal rows are the rule).  Optionally (A2S) a mode-2
//   factor of at most 128 KB -- the 1000-row mode at c4 -- stays resident in
//   shared memory instead of being gathered; only 8 stages then fit beside it,
//   which measured slower (c4 K3 walk 7.55 -> 7.79 ms although its L2 bytes drop
//   from 69 to 58 GB), so it is off by default.
// * 8 consumer warps wait on the stage, read rows and metadata from shared
//   memory (no global latency on their critical path), evaluate y and either
//   scatter the sampled-MTTKRP contributions (K3: mode 0 summed per row segment
//   in registers, modes 1/2 by 16-byte vector reductions into L2; sending them
//   as TMA bulk reductions from the stage instead, cp.reduce.async.bulk add.f32,
//   measured slower: 7.4 -> 9.5 ms at c4) or
//   accumulate the weight gradient (K2w, fixed-order fp64 reduction), then
//   release the stage to its producer through a second mbarrier.
// * Tiles are dealt to CTAs round-robin (tile t of CTA b is b + t * gridDim),
//   so all SMs stay inside the same window of the bucketed walk and the
//   bucket's mode-1 rows stay L2-resident.
//
// The tile -> producer -> stage -> consumer assignment is static, so the weight
// gradient's summation order is fixed (deterministic); the K3 reductions into
// modes 1 and 2 are float atomics (order-dependent in the last bits).

#ifndef OGCP_TMA_STAGES
#define OGCP_TMA_STAGES 16  // multiple of 8 (producer / consumer warps); fewer stages leave SM room for the draw
#endif

namespace walkt {

constexpr int kT = 32;          // samples per stage (tile)
constexpr int kProducers = 8;   // producer warps
constexpr int kConsumers = 8;   // consumer warps
constexpr int kThreadsT = 32 * (kProducers + kConsumers);
constexpr int kA2Max = 128 * 1024;  // largest mode-2 factor kept resident in shared memory (bytes)

// A2S: the mode-2 factor (<= kA2Max bytes, the 1000-row mode at c4) is copied into
// shared memory once per launch and only modes 0 and 1 are gathered per tile.
template <int V, bool A2S>
struct StageLayout {
  static constexpr int kLdr = 16 * V;
  static constexpr int kRowBytes = kLdr * 4;
  static constexpr int kModes = A2S ? 2 : 3;                          // gathered modes
  static constexpr int kRowsBytes = kModes * kT * kRowBytes;          // rows[mode][slot][ldr]
  static constexpr int kMetaBytes = 7 * kT * 4;                       // i0 i1 i2 x mult slot0 uniq0
  static constexpr int kBytes = (kRowsBytes + kMetaBytes + 127) / 128 * 128;
  static constexpr int kStages = A2S ? 8 : OGCP_TMA_STAGES;           // smem ring depth
  static constexpr int kA2Off = kStages * kBytes;                     // resident mode-2 rows
  static constexpr int kSmemFixed = kStages * kBytes + 2 * kStages * 8 + 128;  // + barriers + alignment slack
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const uint32_t a = smem_u32(bar);
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// Four rows (r0..r3) of a [rows x ldr] fp32 tensor map -> 4 consecutive rows at dst.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
      : "memory");
}

struct Maps {
  CUtensorMap a[3];
};

// MODE 0: K2+K3 scatter into GP; MODE 1: K2w weight-gradient partials.
template <int V, int MODE, bool ZERO, bool A2S>
__global__ void __launch_bounds__(kThreadsT, 1)
    k_walk_tma(const __grid_constant__ Maps maps, walk3::Walk<ZERO> W, ModelP M, const float* __restrict__ s_f,
               LossP L, float scale, GradPtrs GP, double* __restrict__ partials, DevFlags* flags, long long code) {
  using SL = StageLayout<V, A2S>;
  constexpr int kStages = SL::kStages;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~(uintptr_t)127);
  float4* a2s = reinterpret_cast<float4*>(smem + SL::kA2Off);  // A2S: resident mode-2 rows
  const int64_t a2_bytes = A2S ? M.dims[2] * (int64_t)SL::kRowBytes : 0;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SL::kA2Off + ((a2_bytes + 127) & ~(int64_t)127));
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (A2S) {
    const float4* src = reinterpret_cast<const float4*>(M.A[2]);
    for (int64_t e = threadIdx.x; e < a2_bytes / 16; e += blockDim.x) a2s[e] = __ldg(src + e);
  }
  __syncthreads();
  W.resolve();
  const int64_t ntiles = (W.n + kT - 1) / kT;
  const int64_t G = gridDim.x, b = blockIdx.x;
  const int64_t my_tiles = ntiles > b ? (ntiles - b + G - 1) / G : 0;  // tile i of this CTA: b + i * G

  if (warp < kProducers) {
    // ------------------------------------------------------------ producers
    const int p = warp;
    auto tile_of = [&](int64_t k) -> int64_t { return p + k * kProducers; };  // k-th tile (CTA-local index)
    const int64_t nk = my_tiles > p ? (my_tiles - p + kProducers - 1) / kProducers : 0;
    // stage A: the entry's position (+ multiplicity); stage B: its record
    auto head = [&](int64_t k, int& pos, float& mult) {
      pos = -1;
      mult = 0.0f;
      if (k >= nk) return;
      const int64_t e = (b + tile_of(k) * G) * kT + lane;
      if (e >= W.n) return;
      if (ZERO) {
        pos = 0;
        mult = 1.0f;
      } else {
        pos = __ldg(W.pos + e);
        mult = (float)__ldg(W.cnt + e);
      }
    };
    auto record = [&](int64_t k, int pos) -> int4 {
      if (pos < 0) return make_int4(-1, 0, 0, 0);
      if (ZERO) {
        const int64_t e = (b + tile_of(k) * G) * kT + lane;
        const int32_t* z = W.zsub + (W.zlo + e) * 3;
        return make_int4(__ldg(z), __ldg(z + 1), __ldg(z + 2), 0);
      }
      return walk3::ld_stream_i4(W.rec + (int64_t)pos * 4);
    };
    // two-tile lead for both stages: the head of tile k+4 and the record of tile
    // k+2 are in flight while tile k's stage is filled
    int pq0, pq1;      // heads of tiles k+2, k+3
    float mq[4];       // multiplicities of tiles k .. k+3
    int4 rq0, rq1;     // records of tiles k, k+1
    {
      int p0, p1;
      head(0, p0, mq[0]);
      head(1, p1, mq[1]);
      head(2, pq0, mq[2]);
      head(3, pq1, mq[3]);
      rq0 = record(0, p0);
      rq1 = record(1, p1);
    }
    for (int64_t k = 0; k < nk; ++k) {
      int pn;
      float mn;
      head(k + 4, pn, mn);
      const int4 rn = record(k + 2, pq0);
      // ---- fill the stage of tile k
      const int64_t i = tile_of(k);
      const int s = (int)(i % kStages);
      const int64_t u = i / kStages;
      if (u > 0) mbar_wait(empty + s, (unsigned)((u - 1) & 1));
      unsigned char* st = smem + s * SL::kBytes;
      int* meta = reinterpret_cast<int*>(st + SL::kRowsBytes);
      const bool valid = rq0.x >= 0;
      const int r0 = valid ? rq0.x : 0, r1 = valid ? rq0.y : 0, r2 = valid ? rq0.z : 0;
      // mode 0: consecutive samples of the bucketed walk share their mode-0 row, so
      // only the distinct rows of the tile are gathered (slot = rank of the row)
      const int prev = __shfl_up_sync(kFull, r0, 1);
      const unsigned heads = __ballot_sync(kFull, lane == 0 || r0 != prev);
      const int slot = __popc(heads & (0xffffffffu >> (31 - lane))) - 1;
      const int nuniq = __popc(heads);
      meta[lane] = rq0.x;
      meta[kT + lane] = rq0.y;
      meta[2 * kT + lane] = rq0.z;
      meta[3 * kT + lane] = rq0.w;
      reinterpret_cast<float*>(meta)[4 * kT + lane] = mq[0];
      meta[5 * kT + lane] = slot;
      if (heads >> lane & 1u) meta[6 * kT + slot] = r0;
      __syncwarp();
      const int nq0 = (nuniq + 3) >> 2;  // gather4 instructions for mode 0
      if (lane == 0)
        mbar_arrive_tx(full + s, (unsigned)((4 * nq0 + (SL::kModes - 1) * kT) * SL::kRowBytes));
      __syncwarp();
      if (lane < nq0) {  // mode 0: slots 4 lane .. 4 lane + 3 (the last group padded with the last row)
        const int* u = meta + 6 * kT;
        const int j0 = 4 * lane;
        tma_gather4(st + j0 * SL::kRowBytes, &maps.a[0], u[j0], u[min(j0 + 1, nuniq - 1)], u[min(j0 + 2, nuniq - 1)],
                    u[min(j0 + 3, nuniq - 1)], full + s);
      }
      // modes 1 (and 2): lane l < 8 (16) gathers samples 4q .. 4q+3 of mode 1 + (l >> 3)
      const int q = lane & 7, m = 1 + (lane >> 3);
      int g[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int src = 4 * q + j;
        const int v1 = __shfl_sync(kFull, r1, src), v2 = __shfl_sync(kFull, r2, src);
        g[j] = m == 1 ? v1 : v2;
      }
      if (lane < 8 * (SL::kModes - 1))
        tma_gather4(st + (m * kT + 4 * q) * SL::kRowBytes, &maps.a[m], g[0], g[1], g[2], g[3], full + s);
      rq0 = rq1;
      rq1 = rn;
      pq0 = pq1;
      pq1 = pn;
      mq[0] = mq[1];
      mq[1] = mq[2];
      mq[2] = mq[3];
      mq[3] = mn;
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int c = warp - kProducers;
  const int gl = lane & 3, grp = lane >> 2;
  const int ldr = SL::kLdr;
  float4 s4[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s4[v] = __ldg(reinterpret_cast<const float4*>(s_f) + v * 4 + gl);
  unsigned bits = 0;
  double acc[V][4];
  float4 part[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    acc[v][0] = acc[v][1] = acc[v][2] = acc[v][3] = 0.0;
    part[v] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  for (int64_t i = c; i < my_tiles; i += kConsumers) {
    const int s = (int)(i % kStages);
    mbar_wait(full + s, (unsigned)((i / kStages) & 1));
    const unsigned char* st = smem + s * SL::kBytes;
    const int* meta = reinterpret_cast<const int*>(st + SL::kRowsBytes);
    const float4* rows = reinterpret_cast<const float4*>(st);
    int seg_row = -1;
    float4 seg[V];
#pragma unroll
    for (int v = 0; v < V; ++v) seg[v] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int smp = 4 * grp + j;
      const int i0 = meta[smp], i1 = meta[kT + smp], i2 = meta[2 * kT + smp];
      const float x = __int_as_float(meta[3 * kT + smp]);
      const float mult = reinterpret_cast<const float*>(meta)[4 * kT + smp];
      const int slot = meta[5 * kT + smp];
      const bool valid = i0 >= 0;
      float4 a0[V], a1[V], a2[V], p01[V];
      float mpart = 0.0f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        a0[v] = rows[slot * (ldr / 4) + v * 4 + gl];
        a1[v] = rows[(1 * kT + smp) * (ldr / 4) + v * 4 + gl];
        a2[v] = A2S ? a2s[(valid ? i2 : 0) * (ldr / 4) + v * 4 + gl] : rows[(2 * kT + smp) * (ldr / 4) + v * 4 + gl];
        p01[v] = mul4(a0[v], a1[v]);
        mpart += dot4(mul4(p01[v], a2[v]), s4[v]);
      }
      mpart += __shfl_xor_sync(kFull, mpart, 1);
      mpart += __shfl_xor_sync(kFull, mpart, 2);
      if (!valid) continue;
      bits |= domain_bits(L.kind, mpart);
      const float y = dloss(L.kind, x, mpart, L.eps) * (ZERO ? scale : scale * mult);
      if (MODE == 0) {
        if (i0 != seg_row) {
          if (seg_row >= 0) {
#pragma unroll
            for (int v = 0; v < V; ++v) red_add_v4(GP.g[0] + (int64_t)seg_row * ldr + (v * 4 + gl) * 4, seg[v]);
          }
          seg_row = i0;
#pragma unroll
          for (int v = 0; v < V; ++v) seg[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float* g1 = GP.g[1] + (int64_t)i1 * ldr;
        float* g2 = GP.g[2] + (int64_t)i2 * ldr;
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float4 ys = make_float4(y * s4[v].x, y * s4[v].y, y * s4[v].z, y * s4[v].w);
          const float4 t = mul4(ys, a2[v]);
          const float4 c0 = mul4(t, a1[v]);
          seg[v].x += c0.x;
          seg[v].y += c0.y;
          seg[v].z += c0.z;
          seg[v].w += c0.w;
          red_add_v4(g1 + (v * 4 + gl) * 4, mul4(t, a0[v]));
          red_add_v4(g2 + (v * 4 + gl) * 4, mul4(ys, p01[v]));
        }
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float4 pr = mul4(p01[v], a2[v]);
          part[v].x += y * pr.x;
          part[v].y += y * pr.y;
          part[v].z += y * pr.z;
          part[v].w += y * pr.w;
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + s);  // the stage's rows and metadata are consumed
    if (MODE == 0) {
      if (seg_row >= 0) {
#pragma unroll
        for (int v = 0; v < V; ++v) red_add_v4(GP.g[0] + (int64_t)seg_row * ldr + (v * 4 + gl) * 4, seg[v]);
      }
    } else {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        acc[v][0] += (double)part[v].x;
        acc[v][1] += (double)part[v].y;
        acc[v][2] += (double)part[v].z;
        acc[v][3] += (double)part[v].w;
        part[v] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  if (bits) report(flags, kFlagData, code, bits);
  if (MODE == 1) {
    // lanes with the same columns, then the consumer warps in fixed order
#pragma unroll
    for (int o = 4; o < 32; o <<= 1)
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[v][e] += __shfl_xor_sync(kFull, acc[v][e], o);
    // reuse stage 0's row area (all stages are consumed once every consumer is past its loop)
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumers) : "memory");
    double* red = reinterpret_cast<double*>(smem);
    if (lane < 4) {
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int e = 0; e < 4; ++e) red[c * 16 * V + (v * 4 + lane) * 4 + e] = acc[v][e];
    }
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kConsumers) : "memory");
    for (int col = threadIdx.x - 32 * kProducers; col < 16 * V; col += 32 * kConsumers) {
      double t = 0.0;
      for (int j = 0; j < kConsumers; ++j) t += red[j * 16 * V + col];
      partials[blockIdx.x * (int64_t)(16 * V) + col] = t;
    }
  }
}

}  // namespace walkt
