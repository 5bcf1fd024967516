// Feasibility test (not product code): is cp.reduce.async.bulk.tensor .add (fp64) atomic per
// element under contention?  Every CTA reduce-adds a box of ones REPS times at the same origin.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
constexpr int BX = 14, BY = 13, BZ = 13, REPS = 50;
__global__ void k(const __grid_constant__ CUtensorMap t, int off) {
  __shared__ __align__(128) double buf[BZ * BY * BX];
  for (int i = threadIdx.x; i < BZ * BY * BX; i += blockDim.x) buf[i] = 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0)
    for (int r = 0; r < REPS; ++r) {
      const int x0 = (blockIdx.x % 3) * off;   // partially overlapping boxes
      asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&t),
                   "r"(x0), "r"(0), "r"(0), "r"((uint32_t)__cvta_generic_to_shared(buf)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
int main() {
  const int L = 32, G = 148 * 6;
  double* d;
  cudaMalloc(&d, L * L * L * 8);
  cudaMemset(d, 0, L * L * L * 8);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap t;
  cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)L, (cuuint64_t)L};
  cuuint64_t strides[2] = {(cuuint64_t)L * 8, (cuuint64_t)L * L * 8};
  cuuint32_t box[3] = {BX, BY, BZ}, es[3] = {1, 1, 1};
  enc(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  k<<<G, 128>>>(t, 4);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<double> h(L * L * L);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  long bad = 0, cnt = 0;
  for (int z = 0; z < L; ++z)
    for (int y = 0; y < L; ++y)
      for (int x = 0; x < L; ++x) {
        double want = 0;
        if (y < BY && z < BZ)
          for (int b = 0; b < 3; ++b) {
            int x0 = b * 4;
            if (x >= x0 && x < x0 + BX) want += (double)REPS * (G / 3);
          }
        if (h[(z * L + y) * L + x] != want) ++bad;
        cnt += want > 0;
      }
  printf("atomicity: %ld mismatching of %ld touched elements\n", bad, cnt);
  return 0;
}
