// Microbenchmark of the patch kernel's streaming skeleton (producer warp + bulk copies into a
// shared-memory ring with full/empty mbarriers; consumer warps only wait, touch and release).
// Measures the achievable HBM -> SMEM stream rate per design knob:
//   piece bytes, misalignment of the source, an extra small "meta" copy per piece read by every
//   CTA from the same L2 lines, ring size, CTAs per SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_bench stream_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NC = 8, NT = NC * 32, NTHR = NT + 32, NDESC = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}\n" ::"r"(
                   smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

__global__ void __launch_bounds__(NTHR) stream_kernel(const char* src, const char* meta, long long per_cta, int piece, int mbytes,
                                                      int misalign, uint32_t cap, double* sink, int ncopy, int jump) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + NDESC;
  int* slot_ofs = (int*)(empty + NDESC);
  unsigned char* ring = sm + 512;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < NDESC; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long npieces = per_cta / piece;
  const char* base = src + (long long)blockIdx.x * (per_cta + 4096) + misalign;
  if (warp == NC) {
    if (lane) return;
    uint32_t H = 0, vs_of[NDESC];
    int rel = 0;
    for (int j = 0; j < npieces; ++j) {
      const uint32_t tot = piece + mbytes;
      uint32_t off = H % cap;
      if (off + tot > cap) H += cap - off;
      const uint32_t vs = H;
      H += tot;
      while (rel < j && (j - rel >= NDESC || H - vs_of[rel % NDESC] > cap)) {
        mbar_wait(&empty[rel % NDESC], (rel / NDESC) & 1);
        ++rel;
      }
      const int sl = j % NDESC;
      vs_of[sl] = vs;
      slot_ofs[sl] = vs % cap;
      mbar_arrive_expect_tx(&full[sl], tot);
      if (mbytes) bulk_g2s(ring + vs % cap, meta + (j % 64) * mbytes, mbytes, &full[sl]);
      const int part = piece / ncopy;
      const char* src_j = base + (long long)j * piece;
      if (jump) {   // blocks of `jump` pieces at pseudo-random block positions of the whole buffer
        const long long blk = j / jump, nblk = (per_cta * gridDim.x) / ((long long)jump * piece);
        const long long pick = (blk * 7919LL + blockIdx.x * 104729LL) % nblk;
        src_j = src + pick * jump * piece + (long long)(j % jump) * piece;
      }
      for (int k = 0; k < ncopy; ++k)
        bulk_g2s(ring + vs % cap + mbytes + k * part, src_j + k * part, part, &full[sl]);
    }
    return;
  }
  double acc = 0;
  for (int j = 0; j < npieces; ++j) {
    mbar_wait(&full[j % NDESC], (j / NDESC) & 1);
    const double* p = (const double*)(ring + slot_ofs[j % NDESC] + mbytes);
    acc += p[tid];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[j % NDESC]);
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main(int argc, char** argv) {
  const long long total = 16LL << 30;
  char* src;
  char* meta;
  double* sink;
  cudaMalloc(&src, total + (1 << 24));
  cudaMalloc(&meta, 1 << 20);
  cudaMalloc(&sink, 64);
  cudaMemset(src, 1, total + (1 << 24));
  cudaMemset(meta, 0, 1 << 20);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  struct Cfg { int ctas_per_sm, ring_kb, piece, mbytes, misalign, ncopy, jump; } cfgs[] = {
      {2, 56, 16384, 0, 0, 1, 0},   {3, 45, 16384, 0, 0, 1, 0},  {3, 45, 16384, 32, 0, 1, 0}, {3, 45, 16384, 32, 0, 1, 35},
      {2, 56, 16384, 32, 0, 1, 35}, {2, 84, 16384, 32, 0, 1, 35}, {3, 45, 8192, 32, 0, 1, 70}, {2, 56, 16384, 0, 0, 1, 35},
  };
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (auto& c : cfgs) {
    const int grid = nsm * c.ctas_per_sm;
    const long long per_cta = (total / grid) / c.piece * c.piece - 8192;
    const size_t smem = 512 + (size_t)c.ring_kb * 1024;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      stream_kernel<<<grid, NTHR, smem>>>(src, meta, per_cta, c.piece, c.mbytes, c.misalign, c.ring_kb * 1024, sink, c.ncopy, c.jump);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 2)
        printf("ctas/SM %d ring %3d KB piece %5d meta %4d misalign %2d copies %d jump %d : %7.1f GB/s  (%s)\n", c.ctas_per_sm, c.ring_kb, c.piece,
               c.mbytes, c.misalign, c.ncopy, c.jump, (double)per_cta * grid / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
