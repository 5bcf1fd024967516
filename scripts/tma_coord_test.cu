// Feasibility test (not product code): TMA tensor load (fp64, box 6x5x5, tensor 14x13x13) for
// every origin in {0, 1, 4, 7, 10}^3; reports the origins that fault.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap t, int x, int y, int z) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(1200u) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(buf)),
        "l"(&t), "r"(x), "r"(y), "r"(z), "r"(sb)
        : "memory");
    asm volatile("{\n .reg .pred P;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W;\n}\n" ::"r"(sb) : "memory");
  }
}
int main() {
  double* d;
  cudaMalloc(&d, 14 * 13 * 13 * 8);
  EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap t;
  cuuint64_t dims[3] = {14, 13, 13}; cuuint64_t strides[2] = {14 * 8, 14 * 13 * 8};
  cuuint32_t box[3] = {6, 5, 5}, es[3] = {1, 1, 1};
  enc(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int cs[5] = {0, 1, 4, 7, 10};
  for (int a = 0; a < 5; ++a)
    for (int b = 0; b < 5; ++b)
      for (int c = 0; c < 5; ++c) {
        k<<<1, 32>>>(t, cs[a], cs[b], cs[c]);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("FAULT at origin %d %d %d: %s\n", cs[a], cs[b], cs[c], cudaGetErrorString(e)); return 1; }
      }
  printf("all origins ok\n");
  return 0;
}
