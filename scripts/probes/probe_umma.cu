// Standalone probe of the tcgen05 Gram kernel (csrc/gram_umma.cuh) on one 32-row chunk.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2110_14514_b200/csrc -o /tmp/pu scripts/probes/probe_umma.cu && /tmp/pu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
namespace ogcp {}
#include "gram_umma.cuh"
using namespace ogcp;

int main() {
  const int LDR = 128, rows = 64;
  std::vector<float> h(rows * LDR);
  for (int i = 0; i < rows * LDR; ++i) h[i] = (float)((i * 37 % 101) - 50) / 50.f;
  float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  umma::GramMaps maps;
  cuuint64_t gdim[2] = {(cuuint64_t)LDR, (cuuint64_t)rows}; cuuint64_t gs[1] = {(cuuint64_t)LDR * 4};
  cuuint32_t box[2] = {(cuuint32_t)LDR, 32}; cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&maps.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gdim, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  maps.b = maps.a;
  float* part; cudaMalloc(&part, 2 * LDR * LDR * 4); cudaMemset(part, 0xff, 2 * LDR * LDR * 4);
  cudaFuncSetAttribute(umma::k_gram_umma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, umma::kSmemG);
  umma::k_gram_umma<128><<<1, umma::kThreadsG, umma::kSmemG>>>(maps, rows, 1, part);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> o(LDR * LDR);
  cudaMemcpy(o.data(), part, o.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, nrm = 0;
  for (int i = 0; i < LDR; ++i) for (int j = 0; j < LDR; ++j) {
    double w = 0; for (int k = 0; k < rows; ++k) w += (double)h[k * LDR + i] * h[k * LDR + j];
    err += (o[i * LDR + j] - w) * (o[i * LDR + j] - w); nrm += w * w;
  }
  printf("rel err %.3e; o[0][0..3] %g %g %g %g\n", sqrt(err / nrm), o[0], o[1], o[2], o[3]);
  double w00 = 0; for (int k = 0; k < rows; ++k) w00 += (double)h[k * LDR] * h[k * LDR];
  printf("want[0][0] %g; o[5][7] %g\n", w00, o[5 * LDR + 7]);
  return 0;
}
