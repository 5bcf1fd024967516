// Feasibility test (not product code): TMA tensor load into DYNAMIC shared memory at a large
// offset, descriptor as __grid_constant__ param (mode 0) or in global memory (mode 1).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const __grid_constant__ CUtensorMap tp, const CUtensorMap* tg, int mode, int ofs, double* out,
                  const int* coords) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)sm;
  double* buf = (double*)(sm + ofs);
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const CUtensorMap* t = mode == 0 ? &tp : tg;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(1200u) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(buf)),
        "l"(t), "r"(coords[0]), "r"(coords[1]), "r"(coords[2]), "r"(sb)
        : "memory");
  }
  asm volatile("{\n .reg .pred P;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W;\n}\n" ::"r"(sb) : "memory");
  for (int i = threadIdx.x; i < 150; i += blockDim.x) out[i] = buf[i];
}
int main() {
  double* d; double* out; CUtensorMap* tg; int* co;
  cudaMalloc(&co, 12); int hc[3] = {4, 0, 0}; cudaMemcpy(co, hc, 12, cudaMemcpyHostToDevice);
  std::vector<double> h(14 * 13 * 13);
  for (size_t i = 0; i < h.size(); ++i) h[i] = i;
  cudaMalloc(&d, h.size() * 8); cudaMalloc(&out, 150 * 8); cudaMalloc(&tg, sizeof(CUtensorMap));
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap t;
  cuuint64_t dims[3] = {14, 13, 13}; cuuint64_t strides[2] = {14 * 8, 14 * 13 * 8};
  cuuint32_t box[3] = {6, 5, 5}, es[3] = {1, 1, 1};
  printf("encode %d\n", (int)enc(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
  cudaMemcpy(tg, &t, sizeof t, cudaMemcpyHostToDevice);
  { const unsigned long long* w = (const unsigned long long*)&t; printf("tmap:"); for (int k = 0; k < 16; ++k) printf(" %llx", w[k]); printf("\nbase %p\n", (void*)d); }
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int ofs : {128, 1024, 65536, 111360}) {
      k<<<1, 320, ofs + 2048>>>(t, tg, mode, ofs, out, co);
      cudaError_t e = cudaDeviceSynchronize();
      printf("mode %d ofs %6d: %s\n", mode, ofs, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  return 0;
}
