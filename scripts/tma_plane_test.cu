// Feasibility test (not product code): TMA tensor load + reduce-add of thin "plane" boxes
// (2,5,5), (6,1,5), (6,5,1) from a padded fp64 array (10 x 10 x 10), incl. high-side OOB.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void k(const CUtensorMap* tin, const CUtensorMap* tout, int x, int y, int z, unsigned bytes, double* out) {
  __shared__ __align__(128) double buf[512];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar), sbuf = (uint32_t)__cvta_generic_to_shared(buf);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(sbuf),
                 "l"(tin), "r"(x), "r"(y), "r"(z), "r"(sb) : "memory");
    asm volatile("{\n .reg .pred P;\n W:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n @!P bra W;\n}\n" ::"r"(sb) : "memory");
    for (unsigned i = 0; i < bytes / 8; ++i) out[i] = buf[i];
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tout), "r"(x),
                 "r"(y), "r"(z), "r"(sbuf) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
int main() {
  const int L = 10;
  std::vector<double> h(L * L * L);
  for (int i = 0; i < L * L * L; ++i) h[i] = i;
  double *din, *dout, *dbuf;
  CUtensorMap *tin, *tout;
  cudaMalloc(&din, h.size() * 8); cudaMalloc(&dout, h.size() * 8); cudaMalloc(&dbuf, 4096); cudaMalloc(&tin, 128); cudaMalloc(&tout, 128);
  cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  struct C { int bx, by, bz, x, y, z; } cs[] = {{2, 5, 5, 2, 3, 3}, {6, 1, 5, 0, 3, 3}, {6, 5, 1, 4, 2, 3}, {2, 5, 5, 8, 6, 6}, {6, 1, 5, 6, 6, 6}};
  for (auto& c : cs) {
    CUtensorMap a, b;
    cuuint64_t dims[3] = {L, L, L}; cuuint64_t st[2] = {L * 8, L * L * 8};
    cuuint32_t box[3] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, (cuuint32_t)c.bz}, es[3] = {1, 1, 1};
    enc(&a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, din, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&b, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dout, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaMemcpy(tin, &a, 128, cudaMemcpyHostToDevice); cudaMemcpy(tout, &b, 128, cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, h.size() * 8);
    const unsigned bytes = c.bx * c.by * c.bz * 8;
    k<<<1, 32>>>(tin, tout, c.x, c.y, c.z, bytes, dbuf);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> o(bytes / 8), g(h.size());
    cudaMemcpy(o.data(), dbuf, bytes, cudaMemcpyDeviceToHost);
    cudaMemcpy(g.data(), dout, h.size() * 8, cudaMemcpyDeviceToHost);
    int bad = 0, bad2 = 0;
    for (int z = 0; z < c.bz; ++z) for (int y = 0; y < c.by; ++y) for (int x = 0; x < c.bx; ++x) {
      const int gx = c.x + x, gy = c.y + y, gz = c.z + z;
      const bool in = gx < L && gy < L && gz < L;
      const double want = in ? h[(gz * L + gy) * L + gx] : 0.0;
      if (o[(z * c.by + y) * c.bx + x] != want) ++bad;
    }
    for (int z = 0; z < L; ++z) for (int y = 0; y < L; ++y) for (int x = 0; x < L; ++x) {
      const bool inb = x >= c.x && x < c.x + c.bx && y >= c.y && y < c.y + c.by && z >= c.z && z < c.z + c.bz;
      if (g[(z * L + y) * L + x] != (inb ? h[(z * L + y) * L + x] : 0.0)) ++bad2;
    }
    printf("box %dx%dx%d at (%d,%d,%d): %s, load mismatches %d, reduce mismatches %d\n", c.bx, c.by, c.bz, c.x, c.y, c.z, cudaGetErrorString(e), bad, bad2);
  }
  return 0;
}
