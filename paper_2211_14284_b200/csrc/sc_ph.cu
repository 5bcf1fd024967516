// Statically condensed Pavarino-Hiptmair relaxation (SC-PH; eq:sc-ph, eq:schur,
// eq:sc-asm-hiptmair), k = 1, 2 on Cartesian cells:
//   c = R_I^T A_II^{-1} R_I r + R_G^T S_PH^{-1} R_G r,   R_G = [-A_GI A_II^{-1}, I],
//   S_PH^{-1} = sum_i R~_i^T S_i^{-1} R~_i + D~ (sum_j R~_j^T B~_j^{-1} R~_j) D~^T.
// The star solves S_i^{-1} / B~_j^{-1} are the k-star / (k-1)-star patch programs run on interface-only
// input with their interior corrections dropped (eq:LDU: their interface part is the interface
// Schur complement solve; patches.cpp SetupInput::interface_only).  This file holds the pieces
// around them:
//   scph_interior_solve  y = A_II^{-1} x_I: per cell the interior DoFs form blocks <= 3x3 (remark
//                        P:1061-1066), assembled from alpha K + beta M and solved by Cholesky
//   scph_vec             the interface / interior masks and the final combine
#include <algorithm>

#include "kernels.cuh"

namespace rm {

namespace {

__device__ __forceinline__ long long scph_gidx(const ScPhParams& P, int code, int cx, int cy, int cz) {
  const int m = code >> 24, c = (code >> 16) & 0xFF, b = (code >> 8) & 0xFF, a = code & 0xFF;
  return P.off[m] + ((long long)(cz * P.p + c) * P.len[m][1] + (cy * P.p + b)) * P.len[m][0] + (cx * P.p + a);
}

__global__ void scph_interior_solve_kernel(ScPhParams P, const double* alpha, const double* beta, int coef_const,
                                           const int* cell_set, const int* bmem, const double* bK, const double* bM,
                                           const double* x, double* y) {
  const long long ncell = (long long)P.n[0] * P.n[1] * P.n[2];
  const long long total = ncell * P.nblk;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long K = t / P.nblk;
    const int b = (int)(t - K * P.nblk);
    const int cx = (int)(K % P.n[0]), cy = (int)((K / P.n[0]) % P.n[1]), cz = (int)(K / ((long long)P.n[0] * P.n[1]));
    const double al = coef_const ? alpha[0] : alpha[K], be = coef_const ? beta[0] : beta[K];
    const long long so = ((long long)cell_set[K] * P.nblk + b) * 6;
    const int* mem = bmem + 3 * b;
    int bs = 0;
    long long g[3];
    double v[3];
    for (int j = 0; j < 3; ++j)
      if (mem[j] >= 0) { g[bs] = scph_gidx(P, mem[j], cx, cy, cz); v[bs] = x[g[bs]]; ++bs; }
    double L[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int i = 0, q = 0; i < 3; ++i)
      for (int j = 0; j <= i; ++j, ++q) L[i][j] = al * bK[so + q] + be * bM[so + q];
    for (int j = 0; j < bs; ++j) {   // Cholesky in place (lower)
      double d = L[j][j];
      for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k];
      L[j][j] = sqrt(d);
      for (int i = j + 1; i < bs; ++i) {
        double s = L[i][j];
        for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
        L[i][j] = s / L[j][j];
      }
    }
    for (int j = 0; j < bs; ++j) {
      double s = v[j];
      for (int k = 0; k < j; ++k) s -= L[j][k] * v[k];
      v[j] = s / L[j][j];
    }
    for (int j = bs - 1; j >= 0; --j) {
      double s = v[j];
      for (int k = j + 1; k < bs; ++k) s -= L[k][j] * v[k];
      v[j] = s / L[j][j];
    }
    for (int j = 0; j < bs; ++j) y[g[j]] = v[j];
  }
}

// mode 0: out = interior ? 0 : a - b        (R_G r from r and A (A_II^{-1} r_I))
// mode 1: out = interior ? 0 : out          (keep the interface part: D~ = D_GG)
// mode 2: out += omega (interior ? a - b : c)   (u += omega c, c_I = y_I - A_II^{-1} (A c_G)_I)
__global__ void scph_vec_kernel(ScPhParams P, int mode, const double* a, const double* b, const double* c, double* out,
                                double omega) {
  const long long n = P.off[P.ncomp];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int m = 0;
    while (m + 1 < P.ncomp && i >= P.off[m + 1]) ++m;
    long long r = i - P.off[m];
    const long long ix = r % P.len[m][0];
    r /= P.len[m][0];
    const long long iy = r % P.len[m][1], iz = r / P.len[m][1];
    bool interior = true;
    const long long idx[3] = {ix, iy, iz};
    for (int d = 0; d < 3; ++d)
      if (P.fam[m][d] == 0 && idx[d] % P.p == 0) interior = false;
    if (mode == 0) out[i] = interior ? 0.0 : a[i] - b[i];
    else if (mode == 1) { if (interior) out[i] = 0.0; }
    else out[i] += omega * (interior ? a[i] - b[i] : c[i]);
  }
}

}  // namespace

cudaError_t launch_scph_interior_solve(const ScPhParams& P, const double* alpha, const double* beta, int coef_const,
                                       const int* cell_set, const int* bmem, const double* bK, const double* bM,
                                       const double* x, double* y, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(y, 0, P.off[P.ncomp] * sizeof(double), st);
  if (e != cudaSuccess) return e;
  const long long total = (long long)P.n[0] * P.n[1] * P.n[2] * P.nblk;
  if (total == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 16);
  scph_interior_solve_kernel<<<grid, 256, 0, st>>>(P, alpha, beta, coef_const, cell_set, bmem, bK, bM, x, y);
  return cudaGetLastError();
}

cudaError_t launch_scph_vec(const ScPhParams& P, int mode, const double* a, const double* b, const double* c,
                            double* out, double omega, cudaStream_t st) {
  const long long n = P.off[P.ncomp];
  if (n == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
  scph_vec_kernel<<<grid, 256, 0, st>>>(P, mode, a, b, c, out, omega);
  return cudaGetLastError();
}

}  // namespace rm
