// K4 on the 5th-generation tensor cores (tcgen05 / TMEM, sm_100a): the history
// Grams P = A'A and C = B'A (B = A_old) of a factor matrix with ldr 64 / 128
// (k_gram_umma) and ldr 32 (k_gram_umma32, below)
// (reference gram kernels.py:75-98, _add_reg_and_history
// solvers.py:159-179).  Included by compute.cu.
//
// Shape: D[M x N] += X[M x K] Y[K x N] with X = A' (or B'), Y = A, K = rows.
// kind::tf32 takes K-major shared-memory operands only (an MN-major tf32 operand
// reads as zeros on this B200 -- measured, scripts/probes/probe_umma2.cu), so the
// converter warps write each 32-row chunk transposed: T[i][k] = A[k][i], 128
// rows i of 128 B (32 k's), in the canonical K-major SWIZZLE_128B layout (8-row
// 1024 B atoms, 16-byte chunk index XOR row % 8).  T serves as both operands of
// P (X = T_A as M x K, Y = T_A as N x K) and, with T_B, of C.  M = 128 (ldr 64
// leaves rows 64..127 of T zero), N = ldr; P and C accumulate in TMEM (fp32,
// columns [0,128) and [128,256)) over all of a CTA's rows; CTAs write their fp32
// accumulators as partials that k_gram_finalize sums in fp64 in block order
// (deterministic).
//
// Accuracy: x = hi + lo (hi, lo TF32-rounded, cvt.rna.tf32) and each product is
// hi*hi + hi*lo + lo*hi (three MMAs), fp32-level like the mma.sync kernel.
//
// Pipeline (one CTA per SM, 2 stages of 32 rows):
//   warp 0    TMA producer: the raw [32 x ldr] row tiles of A (and B), expect_tx;
//   warps 2-9 converters: split + transpose into T_hi / T_lo (16-byte chunks),
//             fence.proxy.async, arrive; warps 2-5 then run the TMEM -> fp64
//             epilogue (tcgen05.ld 32x32b, one TMEM lane quadrant each);
//   warp 1    MMA issuer (one thread): 4 K-steps x 3 (or 6) tcgen05.mma per stage
//             (the K-step advances the descriptor start by 32 B inside the atom),
//             tcgen05.commit -> the stage's empty barrier.

namespace umma {

constexpr int kRows = 32;                    // rows (K) per stage
constexpr int kStagesG = 2;
constexpr int kTile = 128 * 128;             // one transposed operand tile: 128 rows (i) x 128 B (32 k's)
constexpr int kRaw = kRows * 128 * 4;        // one raw [32 x ldr] tile (ldr <= 128)
constexpr int kStageBytes = 2 * kRaw + 4 * kTile;  // raw A, raw B, T_A hi, T_A lo, T_B hi, T_B lo
constexpr int kThreadsG = 320;               // 10 warps: TMA, MMA, 8 converters (4 of them run the epilogue)
constexpr int kSmemG = kStagesG * kStageBytes + 1024 + 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_box(void* dst, const CUtensorMap* tm, int c0, int r0, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(tm), "r"(c0), "r"(r0), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// Canonical K-major SWIZZLE_128B smem descriptor (version 1, layout type 2):
// 8-row groups 1024 B apart (SBO); LBO unused for swizzled K-major.
__device__ __forceinline__ uint64_t k_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N.
__host__ __device__ constexpr uint32_t idesc_tf32(int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// Byte offset of element (row i, k) in a K-major SWIZZLE_128B tile of 128-byte rows.
__device__ __forceinline__ uint32_t swz(int i, int k) {
  return (uint32_t)((i >> 3) * 1024 + (i & 7) * 128 + ((((k >> 2) ^ (i & 7)) & 7) << 4) + (k & 3) * 4);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

struct GramMaps {
  CUtensorMap a, b;
};

template <int LDR>
__global__ void __launch_bounds__(kThreadsG, 1)
    k_gram_umma(const __grid_constant__ GramMaps maps, int64_t rows, int ngram, float* __restrict__ partials) {
  static_assert(LDR == 64 || LDR == 128, "UMMA Gram: ldr 64 or 128");
  extern __shared__ __align__(1024) unsigned char g_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(g_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kStagesG * kStageBytes);
  uint64_t* conv = full + kStagesG;
  uint64_t* empty = conv + kStagesG;
  uint64_t* done = empty + kStagesG;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool two = ngram == 2;
  const int64_t nchunks = (rows + kRows - 1) / kRows;
  const int64_t G = gridDim.x, bi = blockIdx.x;
  const int64_t my = nchunks > bi ? (nchunks - bi + G - 1) / G : 0;
  // stage s: raw A | raw B | T_A hi | T_A lo | T_B hi | T_B lo
  auto raw = [&](int s, int t) { return sm + s * kStageBytes + t * kRaw; };
  auto tt = [&](int s, int t, int lo) { return sm + s * kStageBytes + 2 * kRaw + (2 * t + lo) * kTile; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStagesG; ++s) {
      bar_init(full + s, 1);
      bar_init(conv + s, 8);
      bar_init(empty + s, 1);
    }
    bar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (LDR < 128) {  // rows i >= ldr of every T tile stay zero (M is padded to 128)
    for (int s = 0; s < kStagesG; ++s)
      for (int t = 0; t < 2; ++t)
        for (int lo = 0; lo < 2; ++lo) {
          float4* z = reinterpret_cast<float4*>(tt(s, t, lo) + LDR * 128);
          for (int e = threadIdx.x; e < (128 - LDR) * 128 / 16; e += blockDim.x) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
  }
  if (warp == 1) {  // TMEM: P in columns [0, 128), C in [128, 256)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the zeroed rows, for the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int64_t k = 0; k < my; ++k) {
        const int s = (int)(k % kStagesG);
        const int64_t u = k / kStagesG;
        if (u > 0) bar_wait(empty + s, (unsigned)((u - 1) & 1));
        const int r0 = (int)((bi + k * G) * kRows);
        bar_arrive_tx(full + s, (unsigned)(kRows * LDR * 4 * (two ? 2 : 1)));
        tma_box(raw(s, 0), &maps.a, 0, r0, full + s);
        if (two) tma_box(raw(s, 1), &maps.b, 0, r0, full + s);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(LDR);
      for (int64_t k = 0; k < my; ++k) {
        const int s = (int)(k % kStagesG);
        bar_wait(conv + s, (unsigned)((k / kStagesG) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ahi = su32(tt(s, 0, 0)), alo = su32(tt(s, 0, 1));
        const uint32_t bhi = su32(tt(s, 1, 0)), blo = su32(tt(s, 1, 1));
#pragma unroll
        for (int g = 0; g < kRows / 8; ++g) {
          const uint32_t o = g * 32;  // K-step of 8 tf32 = 32 bytes inside the 128-byte swizzle atom
          const uint32_t acc = (k > 0 || g > 0) ? 1u : 0u;
          // P += Ahi'Ahi + Ahi'Alo + Alo'Ahi
          mma_tf32(tmem, k_desc(ahi + o), k_desc(ahi + o), idesc, acc);
          mma_tf32(tmem, k_desc(ahi + o), k_desc(alo + o), idesc, 1u);
          mma_tf32(tmem, k_desc(alo + o), k_desc(ahi + o), idesc, 1u);
          if (two) {  // C += Bhi'Ahi + Bhi'Alo + Blo'Ahi
            mma_tf32(tmem + 128, k_desc(bhi + o), k_desc(ahi + o), idesc, acc);
            mma_tf32(tmem + 128, k_desc(bhi + o), k_desc(alo + o), idesc, 1u);
            mma_tf32(tmem + 128, k_desc(blo + o), k_desc(ahi + o), idesc, 1u);
          }
        }
        mma_commit(empty + s);  // the stage may be refilled once these MMAs have read it
      }
      mma_commit(done);  // all accumulations complete
    }
  } else {
    // ---------------------------------------------------------------- converters (warps 2-9)
    // thread -> (row i, 4 consecutive k): 4 raw loads down a column (lanes take
    // consecutive i: conflict-free), one 16-byte swizzled chunk of T_hi and of T_lo
    const int ct = threadIdx.x - 64;  // 0 .. 255
    for (int64_t k = 0; k < my; ++k) {
      const int s = (int)(k % kStagesG);
      bar_wait(full + s, (unsigned)((k / kStagesG) & 1));
      for (int t = 0; t < (two ? 2 : 1); ++t) {
        const float* x = reinterpret_cast<const float*>(raw(s, t));
        unsigned char* hi = tt(s, t, 0);
        unsigned char* lo = tt(s, t, 1);
        for (int e = ct; e < (kRows / 4) * LDR; e += 256) {
          const int k4 = e / LDR, i = e - k4 * LDR;
          float v[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) v[j] = x[(4 * k4 + j) * LDR + i];
          float4 h, l;
          h.x = rna_tf32(v[0]); l.x = rna_tf32(v[0] - h.x);
          h.y = rna_tf32(v[1]); l.y = rna_tf32(v[1] - h.y);
          h.z = rna_tf32(v[2]); l.z = rna_tf32(v[2] - h.z);
          h.w = rna_tf32(v[3]); l.w = rna_tf32(v[3] - h.w);
          const uint32_t off = swz(i, 4 * k4);
          *reinterpret_cast<float4*>(hi + off) = h;
          *reinterpret_cast<float4*>(lo + off) = l;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> tensor core
      __syncwarp();
      if (lane == 0) bar_arrive(conv + s);
    }
    if (warp < 6) {  // warps 2-5, one per TMEM lane quadrant, run the epilogue
      // ---------------------------------------------------------------- epilogue: TMEM -> fp64 partials
      bar_wait(done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int q = warp & 3;       // TMEM lane quadrant this warp may read
      const int m = 32 * q + lane;  // output row (i)
      for (int gsel = 0; gsel < ngram; ++gsel) {
        for (int c0 = 0; c0 < LDR; c0 += 32) {
          uint32_t r[32];
          const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(gsel * 128 + c0);
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
              "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (m < LDR) {
            float4* out = reinterpret_cast<float4*>(partials + ((int64_t)bi * ngram + gsel) * LDR * LDR +
                                                    (int64_t)m * LDR + c0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              out[j] = my > 0 ? make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                            __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// ---------------------------------------------------------------------------
// ldr 32.  A 128-row transposed tile holds four 32-row operands, so one MMA can
// serve two 32-row sub-chunks of rows and both Grams: X = [A1'; A2'; B1'; B2']
// (sub-chunks 1, 2 of a 64-row chunk), Y = X rows 0-63 = [A1'; A2'] read as the
// N = 64 x K operand, and D[128 x 64] = X Y' holds A1'A1 (lanes 0-31, columns
// 0-31), A2'A2 (lanes 32-63, columns 32-63), B1'A1 (lanes 64-95, columns 0-31)
// and B2'A2 (lanes 96-127, columns 32-63); the off-diagonal blocks pair rows of
// different sub-chunks and are never read.  Three split-TF32 MMAs per K-step for
// 64 rows of both Grams, no zero padding in the tile.  The raw-tile ring is
// decoupled from the transposed ring: the TMA warp runs kRawRing chunks ahead
// (64 KB in flight per SM), converters move a chunk into one of kTRing transposed
// stages and free its raw stage at once, the MMA warp drains the transposed ring.
// Barriers: rfull / rempty (TMA <-> converters), tfull / tempty (converters <->
// MMA; tempty by tcgen05.commit).  CTA partials: [2 sub-chunks][ngram][32 x 32].
constexpr int kRows32 = 64;              // rows per chunk (two 32-row sub-chunks)
#ifndef OGCP_G32_TRING
#define OGCP_G32_TRING 4
#endif
#ifndef OGCP_G32_RRING
#define OGCP_G32_RRING 4
#endif
constexpr int kRawRing = OGCP_G32_RRING;
constexpr int kTRing = OGCP_G32_TRING;
constexpr int kRaw32 = kRows32 * 32 * 4; // one raw [64 x 32] operand tile
constexpr int kTStage = 2 * kTile;       // X hi, X lo
constexpr int kSmem32 = kTRing * kTStage + kRawRing * 2 * kRaw32 + 1024 + 512;

__global__ void __launch_bounds__(kThreadsG, 1)
    k_gram_umma32(const __grid_constant__ GramMaps maps, int64_t rows, int ngram, float* __restrict__ partials) {
  constexpr int LDR = 32;
  extern __shared__ __align__(1024) unsigned char g_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(g_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* tbase = sm;                         // kTRing transposed stages (1024-aligned)
  unsigned char* rbase = sm + kTRing * kTStage;      // kRawRing raw stages
  uint64_t* rfull = reinterpret_cast<uint64_t*>(rbase + kRawRing * 2 * kRaw32);
  uint64_t* rempty = rfull + kRawRing;
  uint64_t* tfull = rempty + kRawRing;
  uint64_t* tempty = tfull + kTRing;
  uint64_t* done = tempty + kTRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool two = ngram == 2;
  const int64_t nchunks = (rows + kRows32 - 1) / kRows32;
  const int64_t G = gridDim.x, bi = blockIdx.x;
  const int64_t my = nchunks > bi ? (nchunks - bi + G - 1) / G : 0;
  auto raw = [&](int s, int t) { return rbase + (2 * s + t) * kRaw32; };
  auto tx = [&](int j, int lo) { return tbase + j * kTStage + lo * kTile; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRawRing; ++s) {
      bar_init(rfull + s, 1);
      bar_init(rempty + s, 8);
    }
    for (int j = 0; j < kTRing; ++j) {
      bar_init(tfull + j, 8);
      bar_init(tempty + j, 1);
    }
    bar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!two) {  // no second operand: rows 64-127 of every X tile stay zero
    for (int j = 0; j < kTRing; ++j)
      for (int lo = 0; lo < 2; ++lo) {
        float4* z = reinterpret_cast<float4*>(tx(j, lo) + 64 * 128);
        for (int e = threadIdx.x; e < 64 * 128 / 16; e += blockDim.x) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
  }
  if (warp == 1) {  // TMEM: D[128 x 64] in columns [0, 64)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      for (int64_t k = 0; k < my; ++k) {
        const int s = (int)(k % kRawRing);
        const int64_t u = k / kRawRing;
        if (u > 0) bar_wait(rempty + s, (unsigned)((u - 1) & 1));
        const int r0 = (int)((bi + k * G) * kRows32);
        bar_arrive_tx(rfull + s, (unsigned)(kRows32 * LDR * 4 * (two ? 2 : 1)));
        for (int h = 0; h < 2; ++h) {  // two {32 x 32-row} boxes per operand
          tma_box(raw(s, 0) + h * kRows * LDR * 4, &maps.a, 0, r0 + h * kRows, rfull + s);
          if (two) tma_box(raw(s, 1) + h * kRows * LDR * 4, &maps.b, 0, r0 + h * kRows, rfull + s);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(64);
      for (int64_t k = 0; k < my; ++k) {
        const int j = (int)(k % kTRing);
        bar_wait(tfull + j, (unsigned)((k / kTRing) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t xhi = su32(tx(j, 0)), xlo = su32(tx(j, 1));
#pragma unroll
        for (int g = 0; g < kRows / 8; ++g) {
          const uint32_t o = g * 32;  // K-step of 8 tf32 = 32 bytes inside the 128-byte swizzle atom
          const uint32_t acc = (k > 0 || g > 0) ? 1u : 0u;
          // D += Xhi Yhi + Xhi Ylo + Xlo Yhi, Y = rows 0-63 of X
          mma_tf32(tmem, k_desc(xhi + o), k_desc(xhi + o), idesc, acc);
          mma_tf32(tmem, k_desc(xhi + o), k_desc(xlo + o), idesc, 1u);
          mma_tf32(tmem, k_desc(xlo + o), k_desc(xhi + o), idesc, 1u);
        }
        mma_commit(tempty + j);  // the transposed stage may be rewritten once these MMAs have read it
      }
      mma_commit(done);
    }
  } else {
    // ---------------------------------------------------------------- converters (warps 2-9)
    // thread -> (k4, i): for sub-chunk h and operand t, rows 4 k4 .. 4 k4 + 3 of
    // column i -> one 16-byte swizzled chunk of X hi / lo in row 64 t + 32 h + i
    const int ct = threadIdx.x - 64;
    const int k4 = ct >> 5, i = ct & 31;
    for (int64_t k = 0; k < my; ++k) {
      const int s = (int)(k % kRawRing), j = (int)(k % kTRing);
      bar_wait(rfull + s, (unsigned)((k / kRawRing) & 1));
      float v[2][2][4];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (t == 1 && !two) break;
        const float* x = reinterpret_cast<const float*>(raw(s, t));
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 4; ++q) v[t][h][q] = x[(32 * h + 4 * k4 + q) * LDR + i];
      }
      __syncwarp();
      if (lane == 0) bar_arrive(rempty + s);  // the raw stage is in registers: the TMA may refill it
      if (k >= kTRing) bar_wait(tempty + j, (unsigned)(((k / kTRing) - 1) & 1));
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (t == 1 && !two) break;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float4 hv, lv;
          hv.x = rna_tf32(v[t][h][0]); lv.x = rna_tf32(v[t][h][0] - hv.x);
          hv.y = rna_tf32(v[t][h][1]); lv.y = rna_tf32(v[t][h][1] - hv.y);
          hv.z = rna_tf32(v[t][h][2]); lv.z = rna_tf32(v[t][h][2] - hv.z);
          hv.w = rna_tf32(v[t][h][3]); lv.w = rna_tf32(v[t][h][3] - hv.w);
          const uint32_t off = swz(64 * t + 32 * h + i, 4 * k4);
          *reinterpret_cast<float4*>(tx(j, 0) + off) = hv;
          *reinterpret_cast<float4*>(tx(j, 1) + off) = lv;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(tfull + j);
    }
    if (warp < 6) {  // warps 2-5: TMEM lane quadrant q = warp % 4 holds sub-chunk q % 2 of gram q / 2
      const int q = warp & 3;
      const int sub = q & 1, gsel = q >> 1;
      if (gsel < ngram) {
        bar_wait(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        uint32_t r[32];
        const uint32_t taddr = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * sub);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float4* out = reinterpret_cast<float4*>(partials + (((int64_t)bi * 2 + sub) * ngram + gsel) * LDR * LDR +
                                                (int64_t)lane * LDR);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          out[jj] = my > 0 ? make_float4(__uint_as_float(r[4 * jj]), __uint_as_float(r[4 * jj + 1]),
                                         __uint_as_float(r[4 * jj + 2]), __uint_as_float(r[4 * jj + 3]))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

}  // namespace umma
