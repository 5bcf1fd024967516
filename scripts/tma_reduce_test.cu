// Feasibility test (not product code): TMA tensor load of a 3D box of fp64 with out-of-bounds
// zero fill, and TMA tensor reduce-add (cp.reduce.async.bulk.tensor ... .add) of fp64 back into
// global memory.  nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tma_reduce_test tma_reduce_test.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int BX = 14, BY = 13, BZ = 13;

__global__ void k(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, int x0, int y0, int z0,
                  double* dbg, int mode) {
  __shared__ __align__(128) double buf[BZ * BY * BX];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t sbuf = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"((unsigned)sizeof(buf)) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            sbuf),
        "l"(&tin), "r"(x0), "r"(y0), "r"(z0), "r"(sb)
        : "memory");
  }
  asm volatile(
      "{\n .reg .pred P;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W;\n}\n" ::"r"(sb)
      : "memory");
  for (int i = threadIdx.x; i < BZ * BY * BX; i += blockDim.x) { dbg[i] = buf[i]; buf[i] = 1.0; }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && mode == 1) {   // tensor reduce-add
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     &tout),
                 "r"(x0), "r"(y0), "r"(z0), "r"(sbuf)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (threadIdx.x == 0 && mode == 2) {   // plain tensor store
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tout),
                 "r"(x0), "r"(y0), "r"(z0), "r"(sbuf)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int L = 30;   // array L^3 doubles
  std::vector<double> h(L * L * L);
  for (int i = 0; i < L * L * L; ++i) h[i] = i;
  double *din, *dout, *dbg;
  cudaMalloc(&din, h.size() * 8);
  cudaMalloc(&dout, h.size() * 8);
  cudaMalloc(&dbg, BX * BY * BZ * 8);
  cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dout, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no encode fn\n"); return 1; }
  CUtensorMap tin, tout;
  cuuint64_t dims[3] = {(cuuint64_t)L, (cuuint64_t)L, (cuuint64_t)L};
  cuuint64_t strides[2] = {(cuuint64_t)L * 8, (cuuint64_t)L * L * 8};
  cuuint32_t box[3] = {BX, BY, BZ}, es[3] = {1, 1, 1};
  CUresult r1 = enc(&tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, din, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dout, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  const int x0 = -3, y0 = 20, z0 = 5;   // partially out of bounds in x and y
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemcpy(dout, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    k<<<1, 128>>>(tin, tout, x0, y0, z0, dbg, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d kernel: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  cudaMemcpy(dout, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  k<<<1, 128>>>(tin, tout, x0, y0, z0, dbg, 1);
  cudaDeviceSynchronize();
  std::vector<double> b(BX * BY * BZ), o(h.size());
  cudaMemcpy(b.data(), dbg, b.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int z = 0; z < BZ; ++z)
    for (int y = 0; y < BY; ++y)
      for (int x = 0; x < BX; ++x) {
        int gx = x0 + x, gy = y0 + y, gz = z0 + z;
        bool in = gx >= 0 && gx < L && gy >= 0 && gy < L && gz >= 0 && gz < L;
        double want = in ? h[(gz * L + gy) * L + gx] : 0.0;
        if (b[(z * BY + y) * BX + x] != want) ++bad;
      }
  printf("load mismatches: %d\n", bad);
  int bad2 = 0, touched = 0;
  for (int gz = 0; gz < L; ++gz)
    for (int gy = 0; gy < L; ++gy)
      for (int gx = 0; gx < L; ++gx) {
        bool inbox = gx >= x0 && gx < x0 + BX && gy >= y0 && gy < y0 + BY && gz >= z0 && gz < z0 + BZ;
        double want = h[(gz * L + gy) * L + gx] + (inbox ? 1.0 : 0.0);
        touched += inbox;
        if (o[(gz * L + gy) * L + gx] != want) ++bad2;
      }
  printf("reduce-add mismatches: %d (in-bounds box elements %d)\n", bad2, touched);
  return 0;
}
