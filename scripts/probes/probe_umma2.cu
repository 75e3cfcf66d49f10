// Minimal tcgen05 probe: one CTA, A = B = ones-like 32x128 tile in smem (no TMA, no swizzle
// issues: SWIZZLE_NONE canonical), M=128 N=128 K=8, then dump TMEM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(float* out, int mode) {
  __shared__ __align__(1024) float tile[4 * 1024];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // fill: tile[k][m] = 1 for SW128 layout we write logically via swizzle formula
  for (int e = threadIdx.x; e < 8 * 128; e += blockDim.x) {
    const int kk = e / 128, m = e % 128;
    const int blk = m / 32, within = m % 32;  // 32-float (128 B) blocks, 8 rows each 128 B
    const int chunk = within / 4, sub = within % 4;
    const int sw = chunk ^ (kk & 7);
    tile[blk * 1024 + kk * 32 + sw * 4 + sub] = (mode == 3) ? __uint_as_float(0x3f803f80u) : (mode == 0 || mode >= 4) ? 1.0f : (float)(m + 1);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = su32(tile);
    const uint64_t desc = (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(4096 >> 4) << 16) |
                          ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) |
                           ((128u >> 4) << 24);
    printf("tmem %x desc %016llx idesc %08x\n", tmem, (unsigned long long)desc, idesc);
    if (mode == 4) {  // tf32, K-major A and B (bits 15/16 clear)
      const uint32_t idk = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   ::"r"(tmem), "l"(desc), "l"(desc), "r"(idk), "r"(0u) : "memory");
    } else if (mode == 5) {  // tf32, MN-major A only
      const uint32_t idk = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   ::"r"(tmem), "l"(desc), "l"(desc), "r"(idk), "r"(0u) : "memory");
    } else if (mode == 3) {  // bf16 ones (0x3f80) in the same bytes: kind::f16, K = 16 -> expect 16
      const uint32_t idesc16 = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) | ((128u >> 3) << 17) |
                               ((128u >> 4) << 24);
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                   ::"r"(tmem), "l"(desc), "l"(desc), "r"(idesc16), "r"(0u) : "memory");
    } else {
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   ::"r"(tmem), "l"(desc), "l"(desc), "r"(idesc), "r"(0u) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  unsigned done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(su32(&bar)), "r"(0u) : "memory");
  } while (!done);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[4];
  const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16);
  if (mode == 2) {  // st/ld round trip of known values (columns 0..3)
    uint32_t w0 = __float_as_uint(100.f + threadIdx.x), w1 = __float_as_uint(1.f), w2 = __float_as_uint(2.f), w3 = __float_as_uint(3.f);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(w0), "r"(w1), "r"(w2), "r"(w3) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 4; ++j) out[(32 * warp + lane) * 4 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

int main() {
  float* d; cudaMalloc(&d, 128 * 4 * 4);
  for (int mode = 0; mode < 6; ++mode) {
    cudaMemset(d, 0xff, 128 * 16);
    k<<<1, 128>>>(d, mode);
    printf("mode %d kernel: %s\n", mode, cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<float> h(128 * 4);
    cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
    printf("row0: %g %g %g %g | row5: %g %g | row127: %g %g (expect mode0: 8; mode1: 8*(m+1)*(n+1))\n", h[0], h[1], h[2], h[3], h[20], h[21], h[508], h[509]);
  }
  return 0;
}
