// standalone test of the TMA bulk-copy ring used by patch_solve.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>
constexpr int NC = 8, NS = 4, NTHR = (NC + 1) * 32;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory"); }
__global__ void __launch_bounds__(NTHR) k(const double* tiles, int ntiles, double* out, int mode) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + NS;
  double* ring = reinterpret_cast<double*>(smraw + 128);
  int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) { for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC); }
    if (mode & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) for (int t = 0; t < ntiles; ++t) { int s = t % NS; if (t >= NS) mbar_wait(&empty[s], ((t / NS) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], 8192u); bulk_g2s(ring + s * 1024, tiles + (size_t)blockIdx.x * ntiles * 1024 + (size_t)t * 1024, 8192u, &full[s]); }
    return;
  }
  double acc = 0;
  for (int t = 0; t < ntiles; ++t) { int s = t % NS; mbar_wait(&full[s], (t / NS) & 1);
    for (int c = 0; c < 4; ++c) acc += ring[s * 1024 + lane * 32 + 4 * warp + c];
    __syncwarp(); if (lane == 0) mbar_arrive(&empty[s]); }
  out[blockIdx.x * 256 + tid] = acc;
  if (mode & 2) asm volatile("bar.sync 1, 256;" ::: "memory");
}
int main() {
  int nb = 1000, nt = 55;
  double *t, *o; cudaMalloc(&t, (size_t)nb * nt * 8192); cudaMalloc(&o, nb * 256 * 8);
  cudaMemset(t, 0, (size_t)nb * nt * 8192);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 4; ++mode) {
    k<<<nb, NTHR, 128 + NS * 8192 + 40000>>>(t, nt, o, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
