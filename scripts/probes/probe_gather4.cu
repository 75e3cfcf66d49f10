// Probe of the TMA row gather (cp.async.bulk.tensor.2d ... tile::gather4) on the
// B200: a [rows x 32] fp32 matrix, boxes {32, 1}; four rows per instruction land
// in shared memory as four consecutive 128-byte rows.  Prints mismatches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe scripts/probe_gather4.cu && /tmp/probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

__global__ void k_probe(const __grid_constant__ CUtensorMap tm, const int* idx, float* out, int ngroups, int box1) {
  __shared__ alignas(128) float buf[4 * 4 * 32];
  __shared__ alignas(8) unsigned long long bar;
  const unsigned dst = (unsigned)__cvta_generic_to_shared(buf);
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&bar);
  for (int g = 0; g < ngroups; ++g) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned bytes = 4u * 32u * 4u * (unsigned)box1;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4, %5, %6}], [%7];" ::"r"(dst),
          "l"(&tm), "r"(0), "r"(idx[4 * g]), "r"(idx[4 * g + 1]), "r"(idx[4 * g + 2]), "r"(idx[4 * g + 3]), "r"(mb)
          : "memory");
    }
    unsigned done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(mb), "r"(0u)
          : "memory");
    }
    for (int i = threadIdx.x; i < 4 * 32 * box1; i += blockDim.x) out[g * 4 * 32 * box1 + i] = buf[i];
    __syncthreads();
  }
}

int main() {
  const int rows = 1000, cols = 32;
  std::vector<float> h(rows * cols);
  for (int i = 0; i < rows * cols; ++i) h[i] = (float)i;
  float* d;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  std::vector<int> idx = {5, 999, 0, 17, 3, 3, 500, 2};
  int* didx;
  cudaMalloc(&didx, idx.size() * 4);
  cudaMemcpy(didx, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  for (int box1 : {1, 4}) {
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstride[1] = {(cuuint64_t)cols * 4};
    cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)box1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gdim, gstride, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("box1=%d encode rc=%d\n", box1, (int)r);
    if (r != CUDA_SUCCESS) continue;
    float* dout;
    const int n = 2 * 4 * 32 * box1;
    cudaMalloc(&dout, n * 4);
    cudaMemset(dout, 0xff, n * 4);
    k_probe<<<1, 128>>>(tm, didx, dout, 2, box1);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> o(n);
    cudaMemcpy(o.data(), dout, n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int g = 0; g < 2; ++g)
      for (int rr = 0; rr < 4; ++rr)
        for (int c = 0; c < cols; ++c) {
          const float want = (float)(idx[4 * g + rr] * cols + c);
          const float got = o[g * 4 * 32 * box1 + rr * 32 + c];
          if (got != want) ++bad;
        }
    printf("  rows-as-gathered mismatches: %d (first row: %g %g ... expect %g)\n", bad, o[0], o[1],
           (float)(idx[0] * cols));
    cudaFree(dout);
  }
  return 0;
}
