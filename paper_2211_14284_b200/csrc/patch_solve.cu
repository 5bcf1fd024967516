// Batched star-patch solve: one CTA per patch of one colour.
//
//   gather   v = R_i r                                   (structured offsets per class)
//   forward  per elimination level: y_E = L_E^{-1} v_E (pivot blocks <= 3x3),  v_R -= M y_E
//   final    x_F = S_F^{-1} v_F, S_F^{-1} stored as 32x32 tiles of the lower block triangle and
//            streamed HBM -> shared memory by a producer warp with TMA bulk copies
//            (cp.async.bulk + mbarrier ring); consumer warps do the symmetric tile GEMV
//            (row sums and transposed column sums, bank-conflict-free by the stored swizzle)
//            -- or, for ICC-SC, level-scheduled sparse triangular solves
//   backward per level in reverse: x_E = L_E^{-T}(y_E - M^T x_R)
//   scatter  u += omega R_i^T x                          (patches of a colour are disjoint)
// The elimination is the Cholesky factorization of the patch matrix with the eliminated sets
// first (exact for the Cholesky family), so x = A_i^{-1} R_i r up to rounding.
#include "kernels.cuh"

namespace rm {

namespace {

constexpr int NC = 8;        // consumer warps
constexpr int NS = 4;        // TMA ring stages (8 KB each)
constexpr int NTHR = (NC + 1) * 32;

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
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
// barrier among the consumer warps only (the producer warp never joins)
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(NC * 32) : "memory"); }

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

}  // namespace

__global__ void __launch_bounds__(NTHR) patch_solve_kernel(const DClass* __restrict__ classes,
                                                           const int* __restrict__ pclass,
                                                           const long long* __restrict__ pbase,
                                                           const long long* __restrict__ pvals,
                                                           const double* __restrict__ vals,
                                                           const double* __restrict__ r, double* __restrict__ u,
                                                           double omega) {
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + NS;
  double* ring = reinterpret_cast<double*>(smraw + 128);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pi = blockIdx.x;
  const DClass& C = classes[pclass[pi]];
  const int n = C.n;
  const double* V = vals + pvals[pi];
  const int m = C.m, f0 = n - m;
  const int T = (m + 31) >> 5;
  const int ntiles = (C.final_kind == 0) ? T * (T + 1) / 2 : 0;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NC); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // ------------------------------------------------------------------ producer warp
  if (warp == NC) {
    if (lane == 0) {
      const double* tiles = V + C.vofs_final;
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % NS;
        if (t >= NS) mbar_wait(&empty[s], ((t / NS) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], 8192u);
        bulk_g2s(ring + s * 1024, tiles + (size_t)t * 1024, 8192u, &full[s]);
      }
    }
    return;
  }
  // ------------------------------------------------------------------ consumers
  constexpr int NT = NC * 32;
  double* v = ring + NS * 1024;
  double* aux = v + ((n + 1) & ~1);
  const long long b0 = pbase[3 * pi], b1 = pbase[3 * pi + 1], b2 = pbase[3 * pi + 2];
  const int* offs = C.offs;
  const unsigned char* comp = C.comp;
  for (int t = tid; t < n; t += NT) {
    const int c = comp[t];
    const long long base = c == 0 ? b0 : (c == 1 ? b1 : b2);
    v[t] = r[base + offs[t]];
  }
  csync();
  // ---- forward eliminations
  const int nlev = C.nlev;
  for (int l = 0; l < nlev; ++l) {
    {
      const DBlocks& Bk = C.lev[l].blk;
      const double* Bv = V + Bk.vofs;
      const int nb = Bk.nblk;
      for (int i = tid; i < nb; i += NT) {
        const int m0 = __ldg(Bk.mem + i);
        const double y0 = v[m0] * __ldcs(Bv + i);
        v[m0] = y0;
        if (Bk.bs > 1) {
          const int m1 = __ldg(Bk.mem + nb + i);
          if (m1 != 0xFFFF) {
            const double y1 = (v[m1] - __ldcs(Bv + nb + i) * y0) * __ldcs(Bv + 2 * nb + i);
            v[m1] = y1;
            if (Bk.bs > 2) {
              const int m2 = __ldg(Bk.mem + 2 * nb + i);
              if (m2 != 0xFFFF)
                v[m2] = (v[m2] - __ldcs(Bv + 3 * nb + i) * y0 - __ldcs(Bv + 4 * nb + i) * y1) * __ldcs(Bv + 5 * nb + i);
            }
          }
        }
      }
      csync();
    }
    const DSliced& W = C.lev[l].w;
    const double* Wv = V + W.vofs;
    for (int s = warp; s < W.nslices; s += NC) {
      const int row = s * 32 + lane;
      const int w = __ldg(W.sw + s), o = __ldg(W.soff + s);
      double acc = 0.0;
      int kk = 0;
      for (; kk + 4 <= w; kk += 4) {
        const int e = o + kk * 32 + lane;
        const double a0 = __ldcs(Wv + e), a1 = __ldcs(Wv + e + 32), a2 = __ldcs(Wv + e + 64), a3 = __ldcs(Wv + e + 96);
        const int c0 = __ldg(W.cols + e), c1 = __ldg(W.cols + e + 32), c2 = __ldg(W.cols + e + 64), c3 = __ldg(W.cols + e + 96);
        acc += a0 * v[c0] + a1 * v[c1] + a2 * v[c2] + a3 * v[c3];
      }
      for (; kk < w; ++kk) {
        const int e = o + kk * 32 + lane;
        acc += __ldcs(Wv + e) * v[__ldg(W.cols + e)];
      }
      if (row < W.nrows) v[W.r0 + row] -= acc;
    }
    csync();
  }
  // ---- final Schur block
  if (C.final_kind == 0) {
    if (m > 0) {
      const int mpad = 32 * T;
      double* g = aux;            // padded copy of v_F
      double* parts = aux + mpad; // per-warp partial results
      for (int j = tid; j < mpad; j += NT) g[j] = (j < m) ? v[f0 + j] : 0.0;
      for (int j = lane; j < mpad; j += 32) parts[warp * mpad + j] = 0.0;
      csync();
      // every consumer warp takes part in every tile (tiles are consumed in order, so each
      // mbarrier phase is awaited only after the previous phase of that stage completed):
      // warp w covers tile columns 4w..4w+3 for the row sums and tile rows 4w..4w+3 for the
      // transposed column sums; lane = row (resp. column); partial sums stay per warp.
      double* mypart = parts + warp * mpad;
      int I = 0, J = 0;
      for (int t = 0; t < ntiles; ++t) {
        const int s = t % NS;
        mbar_wait(&full[s], (t / NS) & 1);
        const double* tile = ring + s * 1024;
        const double* gJ = g + 32 * J + 4 * warp;
        const double* gI = g + 32 * I + 4 * warp;
        double racc = 0.0, cacc = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int c = 4 * warp + q;
          racc += tile[lane * 32 + ((c + lane) & 31)] * gJ[q];
          cacc += tile[c * 32 + ((lane + c) & 31)] * gI[q];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        mypart[32 * I + lane] += racc;
        if (I != J) mypart[32 * J + lane] += cacc;
        if (++J > I) { ++I; J = 0; }
      }
      csync();
      for (int j = tid; j < m; j += NT) {
        double x = 0.0;
#pragma unroll
        for (int w = 0; w < NC; ++w) x += parts[w * mpad + j];
        v[f0 + j] = x;
      }
      csync();
    }
  } else {
    // ICC(0): forward rows of L by levels, backward rows of L^T by levels; diagonal stored inverted
    const double* Lv = V + C.vofs_final;
    const double* LTv = Lv + C.icc_nnz;
    double* y = v + f0;
    for (int l = 0; l < C.icc_nlev; ++l) {
      const int a0 = C.icc_lptr[l], a1 = C.icc_lptr[l + 1];
      for (int q = a0 + tid; q < a1; q += NT) {
        const int a = C.icc_lrows[q];
        const int t0 = C.icc_rowptr[a], t1 = C.icc_rowptr[a + 1] - 1;
        double s = y[a];
        for (int t = t0; t < t1; ++t) s -= Lv[t] * y[C.icc_col[t]];
        y[a] = s * Lv[t1];
      }
      csync();
    }
    for (int l = 0; l < C.icct_nlev; ++l) {
      const int a0 = C.icct_lptr[l], a1 = C.icct_lptr[l + 1];
      for (int q = a0 + tid; q < a1; q += NT) {
        const int b = C.icct_lrows[q];
        const int t0 = C.icct_rowptr[b], t1 = C.icct_rowptr[b + 1];
        double s = y[b];
        for (int t = t0 + 1; t < t1; ++t) s -= LTv[t] * y[C.icct_col[t]];
        y[b] = s * LTv[t0];
      }
      csync();
    }
  }
  // ---- backward substitution: x_E = L^{-T} (y_E - M^T x_R)
  for (int l = nlev - 1; l >= 0; --l) {
    const DLevel& L = C.lev[l];
    const DSliced& WT = L.wt;
    const double* Tv = V + WT.vofs;
    for (int s = warp; s < WT.nslices; s += NC) {
      const int row = s * 32 + lane;
      double acc = (row < WT.nrows) ? v[L.e0 + row] : 0.0;
      const int w = __ldg(WT.sw + s), o = __ldg(WT.soff + s);
      int kk = 0;
      for (; kk + 4 <= w; kk += 4) {
        const int e = o + kk * 32 + lane;
        const double a0 = __ldcs(Tv + e), a1 = __ldcs(Tv + e + 32), a2 = __ldcs(Tv + e + 64), a3 = __ldcs(Tv + e + 96);
        const int c0 = __ldg(WT.cols + e), c1 = __ldg(WT.cols + e + 32), c2 = __ldg(WT.cols + e + 64), c3 = __ldg(WT.cols + e + 96);
        acc -= a0 * v[c0] + a1 * v[c1] + a2 * v[c2] + a3 * v[c3];
      }
      for (; kk < w; ++kk) {
        const int e = o + kk * 32 + lane;
        acc -= __ldcs(Tv + e) * v[__ldg(WT.cols + e)];
      }
      if (row < WT.nrows) aux[row] = acc;
    }
    csync();
    {
      const DBlocks& Bk = L.blk;
      const double* Bv = V + Bk.vofs;
      const int nb = Bk.nblk;
      for (int i = tid; i < nb; i += NT) {
        const int m0 = __ldg(Bk.mem + i);
        if (Bk.bs == 1) {
          v[m0] = aux[m0 - L.e0] * __ldcs(Bv + i);
          continue;
        }
        const int m1 = __ldg(Bk.mem + nb + i);
        const int m2 = (Bk.bs > 2) ? __ldg(Bk.mem + 2 * nb + i) : 0xFFFF;
        double x2 = 0.0, x1 = 0.0;
        if (m2 != 0xFFFF) { x2 = aux[m2 - L.e0] * __ldcs(Bv + 5 * nb + i); v[m2] = x2; }
        if (m1 != 0xFFFF) {
          x1 = aux[m1 - L.e0];
          if (m2 != 0xFFFF) x1 -= __ldcs(Bv + 4 * nb + i) * x2;
          x1 *= __ldcs(Bv + 2 * nb + i);
          v[m1] = x1;
        }
        double x0 = aux[m0 - L.e0];
        if (m1 != 0xFFFF) x0 -= __ldcs(Bv + nb + i) * x1;
        if (m2 != 0xFFFF) x0 -= __ldcs(Bv + 3 * nb + i) * x2;
        v[m0] = x0 * __ldcs(Bv + i);
      }
    }
    csync();
  }
  // ---- scatter-add omega * R_i^T x
  for (int t = tid; t < n; t += NT) {
    const int c = comp[t];
    const long long base = c == 0 ? b0 : (c == 1 ? b1 : b2);
    double* up = u + base + offs[t];
    *up += omega * v[t];
  }
}

size_t patch_solve_smem_bytes(int n, int max_aux) {
  return 128 + (size_t)NS * 8192 + (size_t)(((n + 1) & ~1) + max_aux) * sizeof(double);
}

cudaError_t launch_patch_solve(const DClass* classes, const int* pclass, const long long* pbase,
                               const long long* pvals, const double* vals, const double* r, double* u,
                               double omega, int npatch, size_t smem, cudaStream_t st) {
  if (npatch <= 0) return cudaSuccess;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(patch_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  patch_solve_kernel<<<npatch, NTHR, smem, st>>>(classes, pclass, pbase, pvals, vals, r, u, omega);
  return cudaGetLastError();
}

}  // namespace rm
