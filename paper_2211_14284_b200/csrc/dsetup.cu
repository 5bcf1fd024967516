// Device-resident numeric setup (PAPER.md P:1131-1151 for the factorizations,
// P:732-742 for the auxiliary operator, P:1585-1596 for why setup time matters).
//
// The host builds only the SYMBOLIC side (star classes, elimination programs, stream layout and the
// per-class NumProg of patches.hpp); every number of the patch factors is produced here:
//   aux_diag_kernel      trilinear cells: the four sum-factorised diagonals of P_K (geometry at the
//                        GLL points, contracted z-plane by z-plane), one CTA per cell
//   aux_entries_kernel   P_K entries = fixed linear map of the diagonals (model.hpp AuxTables)
//   sc_cell_data_kernel  static condensation: interior inverse diagonal, couplings / weights
//   factor_kernel        one CTA per distinct value block: assemble A_i (or P_i) on the class
//                        pattern, level-0 pivot blocks, the interface Schur complement, then a dense
//                        CTA-wide Cholesky (exact programs; the final block's inverse from L_FF) or
//                        level-scheduled ICC(0) with the G7 restart (ICC-SC), and the canonical ->
//                        stream permutation straight into the HBM value block.
// Values equal the host factorization up to rounding (same operations, same term order in the
// assembly and the Schur sums; the interface elimination runs as one dense Cholesky instead of
// sparse levels + a dense final block, which is the same elimination in exact arithmetic).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "dsetup.hpp"

namespace rm {
namespace {

constexpr int NT = 256;   // threads per factor CTA

struct DNum {   // one class (device pointers into the concatenated int buffer)
  int n, nI, nG, m, nnzP, final_kind, nb0, bs0, nrec, nw0, ntgt, icc_nnz, icc_nlev;
  long long blk0_vofs, vofs_final, ncanon, nvals;
  const int *asm_ptr, *asm_src, *pdiag, *b0, *nbr, *w0, *st_idx, *st_csr, *st_ptr, *st_src, *rec;
  const int *icc_rowptr, *icc_col, *icc_lptr, *icc_lrows, *icct_src, *smap;
};

struct FArgs {
  const DNum* progs;
  const int* fclass;
  const int* fcells;
  const long long* fdst;
  int nf, ne, cart;
  const double *cset_k, *cset_m, *alpha, *beta, *cent;
  const int* cell_set;
  double* vals;
  double* scratch;
  long long sP, sM, sS, sY, sC, stride;   // scratch offsets (doubles) inside one CTA's slice
  unsigned long long* sigma_bits;
  int* err;                               // [0] = 1 + block of the first failure, [1] = stage code
};

struct Tiles {
  double A[32][33], B[32][33], R[32][33], D[32][33];
  int flag;
};

// T[r][c] = trans ? X[(r0 + c) * ld + c0 + r] : X[(r0 + r) * ld + c0 + c], zero outside rows < rmax, cols < cmax
// (source coordinates relative to r0 / c0)
__device__ void tile_load(double (*T)[33], const double* X, long long ld, int r0, int c0, int rmax, int cmax, bool trans) {
  for (int k = threadIdx.x; k < 1024; k += NT) {
    const int a = k & 31, b = k >> 5;   // a: fastest source index (coalesced)
    if (!trans) {
      const bool ok = b < rmax && a < cmax;
      T[b][a] = ok ? X[(long long)(r0 + b) * ld + c0 + a] : 0.0;
    } else {
      const bool ok = b < rmax && a < cmax;   // source row r0 + b, column c0 + a -> T[a][b]
      T[a][b] = ok ? X[(long long)(r0 + b) * ld + c0 + a] : 0.0;
    }
  }
}

// acc[4] (rows tr, tr+16; cols tc, tc+16) += sum_k A[row][k] * B[col][k]
__device__ __forceinline__ void tile_mma(const Tiles& t, double acc[4], int kb) {
  const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
#pragma unroll 8
  for (int k = 0; k < kb; ++k) {
    const double a0 = t.A[tr][k], a1 = t.A[tr + 16][k], b0 = t.B[tc][k], b1 = t.B[tc + 16][k];
    acc[0] = fma(a0, b0, acc[0]);
    acc[1] = fma(a0, b1, acc[1]);
    acc[2] = fma(a1, b0, acc[2]);
    acc[3] = fma(a1, b1, acc[3]);
  }
}

// Dense right-looking Cholesky of the lower triangle of S (N x N, row-major, leading dim ld), in
// place, by the whole CTA.  Returns false on a non-positive pivot.
__device__ bool cta_cholesky(double* S, int N, long long ld, Tiles& t) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) t.flag = 0;
  __syncthreads();
  for (int k0 = 0; k0 < N; k0 += 32) {
    const int kb = min(32, N - k0);
    if (warp == 0) {
      for (int c = 0; c < kb; ++c) t.D[c][lane] = (lane < kb) ? S[(long long)(k0 + c) * ld + k0 + lane] : 0.0;
      __syncwarp();
      for (int j = 0; j < kb; ++j) {
        if (lane == j) {
          const double d = t.D[j][j];
          if (!(d > 0)) t.flag = 1;
          t.D[j][j] = d > 0 ? sqrt(d) : 1.0;
        }
        __syncwarp();
        if (lane > j && lane < kb) t.D[lane][j] /= t.D[j][j];
        __syncwarp();
        if (lane > j && lane < kb)
          for (int c = j + 1; c <= lane; ++c) t.D[lane][c] -= t.D[lane][j] * t.D[c][j];
        __syncwarp();
      }
      for (int c = 0; c < kb; ++c)
        if (lane >= c && lane < kb) S[(long long)(k0 + lane) * ld + k0 + c] = t.D[lane][c];
    }
    __syncthreads();
    const int r0 = k0 + kb, nr = N - r0;
    if (nr <= 0) break;
    // panel: L_iK = S_iK L_KK^{-T}, 32 rows at a time (lane = row, columns through shared memory)
    for (int i0 = 0; i0 < nr; i0 += 32) {
      const int rows = min(32, nr - i0);
      tile_load(t.A, S, ld, r0 + i0, k0, rows, kb, false);
      __syncthreads();
      if (warp == 0 && lane < rows) {
        for (int c = 0; c < kb; ++c) {
          double v = t.A[lane][c];
          for (int j = 0; j < c; ++j) v -= t.A[lane][j] * t.D[c][j];
          t.A[lane][c] = v / t.D[c][c];
        }
      }
      __syncthreads();
      for (int k = threadIdx.x; k < 1024; k += NT) {
        const int a = k & 31, b = k >> 5;
        if (b < rows && a < kb) S[(long long)(r0 + i0 + b) * ld + k0 + a] = t.A[b][a];
      }
      __syncthreads();
    }
    // trailing update S_IJ -= L_IK L_JK^T over tiles I >= J of the trailing block
    const int nt = (nr + 31) / 32;
    for (int I = 0; I < nt; ++I) {
      const int ri = min(32, nr - 32 * I);
      tile_load(t.A, S, ld, r0 + 32 * I, k0, ri, kb, false);
      for (int J = 0; J <= I; ++J) {
        const int rj = min(32, nr - 32 * J);
        tile_load(t.B, S, ld, r0 + 32 * J, k0, rj, kb, false);
        __syncthreads();
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        tile_mma(t, acc, kb);
        const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = tr + 16 * (q >> 1), c = tc + 16 * (q & 1);
          if (r < ri && c < rj && (I != J || c <= r)) S[(long long)(r0 + 32 * I + r) * ld + r0 + 32 * J + c] -= acc[q];
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  return t.flag == 0;
}

// canonical tiles of the inverse of the final block F = L_FF L_FF^T (L_FF = trailing m x m of the
// factor in S): Y = L_FF^{-1}, Finv_IJ = sum_{K >= I} Y_KI^T Y_KJ.
__device__ void cta_final_inverse(const double* S, long long ld, int g0, int m, double* Y, double* canon, long long vofs,
                                  Tiles& t) {
  const int T = (m + 31) / 32;
  const long long ly = 32LL * T;
  const double* L = S + (long long)g0 * ld + g0;
  const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;
  for (int J = 0; J < T; ++J)
    for (int I = J; I < T; ++I) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int K = J; K < I; ++K) {
        tile_load(t.A, L, ld, 32 * I, 32 * K, min(32, m - 32 * I), min(32, m - 32 * K), false);
        tile_load(t.B, Y, ly, 32 * K, 32 * J, 32, 32, true);   // B[c][k] = Y[32K + k][32J + c]
        __syncthreads();
        tile_mma(t, acc, 32);
        __syncthreads();
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = tr + 16 * (q >> 1), c = tc + 16 * (q & 1);
        t.R[r][c] = ((I == J && r == c) ? 1.0 : 0.0) - acc[q];
      }
      tile_load(t.D, L, ld, 32 * I, 32 * I, min(32, m - 32 * I), min(32, m - 32 * I), false);
      __syncthreads();
      if (threadIdx.x < 32) {   // L_II X = R, column c per lane
        const int c = threadIdx.x;
        const int ri = min(32, m - 32 * I);
        for (int r = 0; r < 32; ++r) {
          double v = t.R[r][c];
          if (r < ri) {
            for (int j = 0; j < r; ++j) v -= t.D[r][j] * t.R[j][c];
            v /= t.D[r][r];
          } else {
            v = 0.0;
          }
          t.R[r][c] = v;
        }
      }
      __syncthreads();
      for (int k = threadIdx.x; k < 1024; k += NT) {
        const int a = k & 31, b = k >> 5;
        Y[(32LL * I + b) * ly + 32 * J + a] = t.R[b][a];
      }
      __syncthreads();
    }
  for (int I = 0; I < T; ++I)
    for (int J = 0; J <= I; ++J) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int K = I; K < T; ++K) {
        tile_load(t.A, Y, ly, 32 * K, 32 * I, 32, 32, true);   // A[r][k] = Y[32K + k][32I + r]
        tile_load(t.B, Y, ly, 32 * K, 32 * J, 32, 32, true);
        __syncthreads();
        tile_mma(t, acc, 32);
        __syncthreads();
      }
      double* o = canon + vofs + (long long)(I * (I + 1) / 2 + J) * 1024;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = tr + 16 * (q >> 1), c = tc + 16 * (q & 1);
        const int i = 32 * I + r, j = 32 * J + c;
        o[r * 32 + ((c + r) & 31)] = (i < m && j < m) ? acc[q] : 0.0;
      }
    }
  __syncthreads();
}

__global__ void __launch_bounds__(NT) factor_kernel(FArgs a) {
  __shared__ Tiles t;
  __shared__ int fail;
  double* scr = a.scratch + (long long)blockIdx.x * a.stride;
  double* Pv = scr + a.sP;
  double* M = scr + a.sM;
  double* S = scr + a.sS;
  double* Y = scr + a.sY;
  double* C = scr + a.sC;
  for (int f = blockIdx.x; f < a.nf; f += gridDim.x) {
    const DNum& g = a.progs[a.fclass[f]];
    const int* cells = a.fcells + (long long)f * kMaxSlots;
    const bool icc = g.final_kind == 1;
    double shift = 0.0;
    for (;;) {
      if (threadIdx.x == 0) fail = 0;
      // ---- assembly of the patch matrix on the class pattern (factor_patch order)
      for (int e = threadIdx.x; e < g.nnzP; e += NT) {
        double v = 0.0;
        for (int k = g.asm_ptr[e]; k < g.asm_ptr[e + 1]; ++k) {
          const int src = g.asm_src[k];
          const int s = src / a.ne, tt = src - s * a.ne;
          const int cell = cells[s];
          if (a.cart) {
            const long long so = (long long)a.cell_set[cell] * a.ne + tt;
            v += a.alpha[cell] * a.cset_k[so] + a.beta[cell] * a.cset_m[so];
          } else {
            v += a.cent[(long long)cell * a.ne + tt];
          }
        }
        Pv[e] = v;
      }
      for (long long c = threadIdx.x; c < g.ncanon; c += NT) C[c] = 0.0;
      const long long ns = icc ? g.icc_nnz : (long long)g.nG * g.nG;
      for (long long c = threadIdx.x; c < ns; c += NT) S[c] = 0.0;
      __syncthreads();
      if (shift != 0.0)
        for (int i = threadIdx.x; i < g.n; i += NT) Pv[g.pdiag[i]] *= (1.0 + shift);
      __syncthreads();
      // ---- level 0: pivot blocks (<= 3x3), M = L^{-1} P_{b,r}, W^ = L^{-T} M, W = P_RE
      for (int bi = threadIdx.x; bi < g.nb0; bi += NT) {
        const int* rc = g.b0 + 12 * bi;
        const int bs = rc[0];
        double Lm[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
        auto lp = [&](int i, int j) -> double { const int x = rc[4 + i * (i + 1) / 2 + j]; return x < 0 ? 0.0 : Pv[x]; };
        bool ok = true;
        for (int j = 0; j < bs; ++j) {
          double d = lp(j, j);
          for (int k = 0; k < j; ++k) d -= Lm[j][k] * Lm[j][k];
          if (!(d > 0)) { ok = false; d = 1.0; }
          Lm[j][j] = sqrt(d);
          for (int i = j + 1; i < bs; ++i) {
            double s = lp(i, j);
            for (int k = 0; k < j; ++k) s -= Lm[i][k] * Lm[j][k];
            Lm[i][j] = s / Lm[j][j];
          }
        }
        if (!ok) fail = 1;
        for (int r = 0, slot = 0; r < g.bs0; ++r)
          for (int c = 0; c <= r; ++c, ++slot) {
            double v = (r < bs) ? Lm[r][c] : 0.0;
            if (r == c) v = (r < bs) ? 1.0 / v : 0.0;
            C[g.blk0_vofs + (long long)slot * g.nb0 + bi] = v;
          }
        for (int k = rc[10]; k < rc[11]; ++k) {
          const int* nr = g.nbr + 7 * k;
          double y[3] = {0.0, 0.0, 0.0}, z[3] = {0.0, 0.0, 0.0};
          for (int j = 0; j < bs; ++j) {
            double s = nr[1 + j] < 0 ? 0.0 : Pv[nr[1 + j]];
            for (int kk = 0; kk < j; ++kk) s -= Lm[j][kk] * y[kk];
            y[j] = s / Lm[j][j];
          }
          M[3LL * k + 0] = y[0]; M[3LL * k + 1] = y[1]; M[3LL * k + 2] = y[2];
          for (int j = bs - 1; j >= 0; --j) {
            double s = y[j];
            for (int kk = j + 1; kk < bs; ++kk) s -= Lm[kk][j] * z[kk];
            z[j] = s / Lm[j][j];
            C[nr[4 + j]] = z[j];
          }
        }
      }
      for (int i = threadIdx.x; i < g.nw0; i += NT) {
        const int x = g.w0[2 * i + 1];
        C[g.w0[2 * i]] = x < 0 ? 0.0 : Pv[x];
      }
      __syncthreads();
      // ---- interface Schur complement S = P_GG - sum_b M_b M_b^T (lower), targets in parallel
      for (int q = threadIdx.x; q < g.ntgt; q += NT) {
        const int x = g.st_csr[q];
        double v = x < 0 ? 0.0 : Pv[x];
        for (int k = g.st_ptr[q]; k < g.st_ptr[q + 1]; ++k) {
          const double* ma = M + 3LL * g.st_src[2 * k];
          const double* mc = M + 3LL * g.st_src[2 * k + 1];
          v -= ma[0] * mc[0] + ma[1] * mc[1] + ma[2] * mc[2];
        }
        S[g.st_idx[q]] = v;
      }
      __syncthreads();
      bool ok = fail == 0;
      if (!icc) {
        // ---- exact: dense Cholesky of S in position order; levels >= 1 read off L; final inverse
        if (g.nG > 0 && !cta_cholesky(S, g.nG, g.nG, t)) ok = false;
        if (ok) {
          for (int i = threadIdx.x; i < g.nrec; i += NT) {
            const int* r = g.rec + 4 * i;
            const double lab = S[(long long)r[2] * g.nG + r[3]], lbb = S[(long long)r[3] * g.nG + r[3]];
            C[r[0]] = r[1] == 0 ? 1.0 / lbb : (r[1] == 1 ? lab * lbb : lab / lbb);
          }
          if (g.m > 0) cta_final_inverse(S, g.nG, g.nG - g.m, g.m, Y, C, g.vofs_final, t);
        }
      } else if (ok) {
        // ---- ICC(0) on the final pattern, up-looking rows in level order (rows of one level are
        // independent), in place: S holds F on entry and L on exit
        for (int lv = 0; lv < g.icc_nlev; ++lv) {
          for (int q = g.icc_lptr[lv] + threadIdx.x; q < g.icc_lptr[lv + 1]; q += NT) {
            const int ra = g.icc_lrows[q];
            const int a0 = g.icc_rowptr[ra], a1 = g.icc_rowptr[ra + 1];
            for (int tt = a0; tt < a1; ++tt) {
              const int b = g.icc_col[tt];
              double s = S[tt];
              int ia = a0, ib = g.icc_rowptr[b];
              const int eb = g.icc_rowptr[b + 1] - 1;
              while (ia < tt && ib < eb) {
                const int ca = g.icc_col[ia], cb = g.icc_col[ib];
                if (ca == cb) { s -= S[ia] * S[ib]; ++ia; ++ib; }
                else if (ca < cb) ++ia; else ++ib;
              }
              if (b == ra) {
                if (!(s > 0)) { fail = 1; s = 1.0; }
                S[tt] = sqrt(s);
              } else {
                S[tt] = s / S[g.icc_rowptr[b + 1] - 1];
              }
            }
          }
          __syncthreads();
        }
        ok = fail == 0;
        if (ok) {
          double* o = C + g.vofs_final;
          for (int ra = threadIdx.x; ra < g.m; ra += NT)
            for (int tt = g.icc_rowptr[ra]; tt < g.icc_rowptr[ra + 1]; ++tt)
              o[tt] = (tt == g.icc_rowptr[ra + 1] - 1) ? 1.0 / S[tt] : S[tt];
          __syncthreads();
          for (int tt = threadIdx.x; tt < g.icc_nnz; tt += NT) o[g.icc_nnz + tt] = o[g.icct_src[tt]];
        }
      }
      __syncthreads();
      if (ok) break;
      // breakdown: reading G7 restart (ICC-SC only): P + sigma diag(P), sigma = 1e-10 doubling to 1e-2
      shift = (shift == 0.0) ? 1e-10 : 2.0 * shift;
      if (!icc || shift > 1e-2) {
        if (threadIdx.x == 0 && atomicCAS(a.err, 0, 1 + f) == 0) a.err[1] = icc ? 2 : 1;
        break;
      }
      __syncthreads();
    }
    if (shift > 0.0 && threadIdx.x == 0) atomicMax(a.sigma_bits, (unsigned long long)__double_as_longlong(shift));
    // ---- canonical -> stream block in HBM
    double* out = a.vals + a.fdst[f];
    for (long long k = threadIdx.x; k < g.nvals; k += NT) {
      const int c = g.smap[k];
      out[k] = c >= 0 ? C[c] : (c == -1 ? 0.0 : 0.5 * C[-2 - c]);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ trilinear cells
struct AuxDev {
  int p, nq, ndiag, off[4];
  const double *xq, *wq, *sb2, *r2;
};

// diagonals of one cell: per z quadrature plane W0, W1[3] at the nq^2 points, contracted in x,
// then y, accumulated into the z sum (aux_cell_diagonals' order: x, y, then z ascending)
__global__ void __launch_bounds__(256) aux_diag_kernel(AuxDev T, const double* coords, int nx, int ny, int nz,
                                                       const double* alpha, const double* beta, double* diag) {
  extern __shared__ double sm[];
  const int p = T.p, n = p + 1, nq = T.nq;
  const long long K = blockIdx.x;
  const int cx = (int)(K % nx), cy = (int)((K / nx) % ny), cz = (int)(K / ((long long)nx * ny));
  double* W = sm;                        // [4][nq][nq]
  double* A = W + 4 * nq * nq;           // [4][nq][n]
  double* Bq = A + 4 * nq * n;           // [4][n][n]
  double* out = Bq + 4 * n * n;          // [ndiag]
  __shared__ double Xc[8][3];
  if (threadIdx.x < 24) {
    const int v = threadIdx.x / 3, i = threadIdx.x % 3;
    const int az = v >> 2, ay = (v >> 1) & 1, ax = v & 1;
    Xc[v][i] = coords[(((long long)(cz + az) * (ny + 1) + (cy + ay)) * (nx + 1) + (cx + ax)) * 3 + i];
  }
  for (int i = threadIdx.x; i < T.ndiag; i += blockDim.x) out[i] = 0.0;
  const double al = alpha[K], be = beta[K];
  __syncthreads();
  // per-array extents (x, y, z): d0 (n,n,n); d1x (p,n,n); d1y (n,p,n); d1z (n,n,p)
  for (int qz = 0; qz < nq; ++qz) {
    for (int q = threadIdx.x; q < nq * nq; q += blockDim.x) {
      const int qy = q / nq, qx = q % nq;
      const double tq[3] = {T.xq[qx], T.xq[qy], T.xq[qz]};
      double phi[3][2], dphi[3][2];
      for (int d = 0; d < 3; ++d) { phi[d][0] = 0.5 * (1 - tq[d]); phi[d][1] = 0.5 * (1 + tq[d]); dphi[d][0] = -0.5; dphi[d][1] = 0.5; }
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
      for (int az = 0; az < 2; ++az)
        for (int ay = 0; ay < 2; ++ay)
          for (int ax = 0; ax < 2; ++ax) {
            const double* X = Xc[az * 4 + ay * 2 + ax];
            const double f0 = dphi[0][ax] * phi[1][ay] * phi[2][az];
            const double f1 = phi[0][ax] * dphi[1][ay] * phi[2][az];
            const double f2 = phi[0][ax] * phi[1][ay] * dphi[2][az];
            for (int i = 0; i < 3; ++i) { J[i][0] += X[i] * f0; J[i][1] += X[i] * f1; J[i][2] += X[i] * f2; }
          }
      const double dJ = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                        J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      double Ji[3][3];
      Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / dJ;
      Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / dJ;
      Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / dJ;
      Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / dJ;
      Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / dJ;
      Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / dJ;
      Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / dJ;
      Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / dJ;
      Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / dJ;
      const double w = T.wq[qx] * T.wq[qy] * T.wq[qz] * dJ;
      W[q] = w * be;
      for (int m = 0; m < 3; ++m) {
        const double jj = Ji[m][0] * Ji[m][0] + Ji[m][1] * Ji[m][1] + Ji[m][2] * Ji[m][2];
        W[(1 + m) * nq * nq + q] = w * al * jj;
      }
    }
    __syncthreads();
    // x contraction: A[m][qy][i] = sum_qx Tx[qx][i] W[m][qy][qx]
    for (int q = threadIdx.x; q < 4 * nq * n; q += blockDim.x) {
      const int m = q / (nq * n), rem = q % (nq * n), qy = rem / n, i = rem % n;
      const int nxm = (m == 1) ? p : n;
      if (i >= nxm) continue;
      const double* Tx = (m == 1) ? T.r2 : T.sb2;
      double acc = 0.0;
      for (int qx = 0; qx < nq; ++qx) acc += Tx[qx * nxm + i] * W[m * nq * nq + qy * nq + qx];
      A[(m * nq + qy) * n + i] = acc;
    }
    __syncthreads();
    // y contraction: Bq[m][j][i] = sum_qy Ty[qy][j] A[m][qy][i]
    for (int q = threadIdx.x; q < 4 * n * n; q += blockDim.x) {
      const int m = q / (n * n), j = (q / n) % n, i = q % n;
      const int nxm = (m == 1) ? p : n, nym = (m == 2) ? p : n;
      if (i >= nxm || j >= nym) continue;
      const double* Ty = (m == 2) ? T.r2 : T.sb2;
      double acc = 0.0;
      for (int qy = 0; qy < nq; ++qy) acc += Ty[qy * nym + j] * A[(m * nq + qy) * n + i];
      Bq[(m * n + j) * n + i] = acc;
    }
    __syncthreads();
    // z accumulation: out[m][l][j][i] += Tz[qz][l] Bq[m][j][i]
    for (int m = 0; m < 4; ++m) {
      const int nxm = (m == 1) ? p : n, nym = (m == 2) ? p : n, nzm = (m == 3) ? p : n;
      const double* Tz = (m == 3) ? T.r2 : T.sb2;
      double* o = out + T.off[m];
      for (int q = threadIdx.x; q < nzm * nym * nxm; q += blockDim.x) {
        const int l = q / (nym * nxm), j = (q / nxm) % nym, i = q % nxm;
        o[q] += Tz[qz * nzm + l] * Bq[(m * n + j) * n + i];
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < T.ndiag; i += blockDim.x) diag[K * T.ndiag + i] = out[i];
}

__global__ void __launch_bounds__(256) aux_entries_kernel(const double* diag, int ndiag, const int* tptr, const int* tg,
                                                          const double* ta, const double* tc, int ne, double* cent) {
  extern __shared__ double dsh[];
  const long long K = blockIdx.x;
  for (int i = threadIdx.x; i < ndiag; i += blockDim.x) dsh[i] = diag[K * ndiag + i];
  __syncthreads();
  for (int t = threadIdx.x; t < ne; t += blockDim.x) {
    double acc = 0.0;
    for (int k = tptr[t]; k < tptr[t + 1]; ++k) acc += ta[k] * dsh[tg[k]] * tc[k];
    cent[K * ne + t] = acc;
  }
}

// per cell and interior DoF I: sc_dinv = 1 / A_II; Cartesian couplings sc_c[K][f][I]; trilinear
// weights sc_w[K][m][I] (the interior values of the stiffness diagonals)
__global__ void sc_cell_data_kernel(long long ncell, int ni, int ne, int cart, const int* cell_set, const double* cset_k,
                                    const double* cset_m, const double* alpha, const double* beta, const double* cent,
                                    const double* diag, int ndiag, const int* tdiag, const int* tface, const int* widx,
                                    double* sc_dinv, double* sc_c, double* sc_w) {
  const long long total = ncell * ni;
  for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total; x += (long long)gridDim.x * blockDim.x) {
    const long long K = x / ni;
    const int I = (int)(x % ni);
    auto entry = [&](int t) -> double {
      if (cart) {
        const long long so = (long long)cell_set[K] * ne + t;
        return alpha[K] * cset_k[so] + beta[K] * cset_m[so];
      }
      return cent[K * ne + t];
    };
    sc_dinv[K * ni + I] = 1.0 / entry(tdiag[I]);
    if (cart) {
      for (int f = 0; f < 6; ++f) {
        const int t = tface[6 * I + f];
        sc_c[(K * 6 + f) * ni + I] = t < 0 ? 0.0 : entry(t);
      }
    } else {
      for (int m = 0; m < 3; ++m) sc_w[(K * 3 + m) * ni + I] = diag[K * ndiag + widx[3 * I + m]];
    }
  }
}

#define DS_CK(x)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("device setup: ") + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  std::vector<void*> ptrs;
  ~DevBuf() { for (void* p : ptrs) cudaFree(p); }
  template <class T>
  T* up(const std::vector<T>& v, cudaStream_t st) {
    if (v.empty()) return nullptr;
    void* p = nullptr;
    DS_CK(cudaMalloc(&p, v.size() * sizeof(T)));
    ptrs.push_back(p);
    DS_CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return static_cast<T*>(p);
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    DS_CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

}  // namespace

void device_numeric_setup(const PatchFamily& P, const std::vector<long long>& fdst, double* vals, double* sc_dinv,
                          double* sc_c, double* sc_w, cudaStream_t st, double* sigma_max) {
  if (!P.deferred) throw std::runtime_error("device setup: family was not built with defer_numeric");
  const int nf = (int)P.fclass.size();
  const Space& sp = P.sp;
  const long long ncell = (long long)sp.n[0] * sp.n[1] * sp.n[2];
  const int ne = (int)P.cell_rows.size();
  DevBuf buf;
  // ---- per-cell entries (trilinear: diagonals on the device, then the entry map)
  const double* d_alpha = buf.up(P.cell_alpha, st);
  const double* d_beta = buf.up(P.cell_beta, st);
  const double *d_ck = nullptr, *d_cm = nullptr, *d_cent = nullptr, *d_diag = nullptr;
  const int* d_cset = nullptr;
  int ndiag = 0;
  if (P.cartesian) {
    d_ck = buf.up(P.cset_k, st);
    d_cm = buf.up(P.cset_m, st);
    d_cset = buf.up(P.cell_set, st);
  } else {
    const AuxTables& T = aux_tables(sp.p);
    if ((int)T.row.size() != ne) throw std::runtime_error("device setup: auxiliary pattern mismatch");
    AuxDev ad{};
    ad.p = T.p; ad.nq = T.nq; ad.ndiag = T.ndiag;
    for (int i = 0; i < 4; ++i) ad.off[i] = T.off[i];
    ad.xq = buf.up(T.xq, st); ad.wq = buf.up(T.wq, st); ad.sb2 = buf.up(T.sb2, st); ad.r2 = buf.up(T.r2, st);
    ndiag = T.ndiag;
    double* dg = buf.alloc<double>((size_t)ncell * ndiag);
    const double* dco = buf.up(P.coords, st);
    const int n = sp.p + 1;
    const size_t smem = (size_t)(4 * T.nq * T.nq + 4 * T.nq * n + 4 * n * n + T.ndiag) * sizeof(double);
    DS_CK(cudaFuncSetAttribute(aux_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (ncell > 0)
      aux_diag_kernel<<<(unsigned)ncell, 256, smem, st>>>(ad, dco, sp.n[0], sp.n[1], sp.n[2], d_alpha, d_beta, dg);
    DS_CK(cudaGetLastError());
    double* ce = buf.alloc<double>((size_t)ncell * ne);
    const size_t smem2 = (size_t)T.ndiag * sizeof(double);
    DS_CK(cudaFuncSetAttribute(aux_entries_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
    if (ncell > 0)
      aux_entries_kernel<<<(unsigned)ncell, 256, smem2, st>>>(dg, T.ndiag, buf.up(T.tptr, st), buf.up(T.tg, st),
                                                               buf.up(T.ta, st), buf.up(T.tc, st), ne, ce);
    DS_CK(cudaGetLastError());
    d_cent = ce;
    d_diag = dg;
  }
  // ---- static-condensation cell data
  if (sc_dinv) {
    const int p = sp.p, P1 = p + 1, pm = p - 1, ni = pm * pm * pm;
    std::vector<int> tdiag(ni, -1), tface(6 * (size_t)ni, -1), widx(3 * (size_t)ni, 0);
    for (int t = 0; t < ne; ++t) {
      const int r = P.cell_rows[t], c = P.cell_cols[t];
      const int ra = r % P1, rb = (r / P1) % P1, rc = r / (P1 * P1);
      if (ra == 0 || ra == p || rb == 0 || rb == p || rc == 0 || rc == p) continue;
      const int I = ((rc - 1) * pm + (rb - 1)) * pm + (ra - 1);
      const int ca = c % P1, cb = (c / P1) % P1, cc = c / (P1 * P1);
      if (c == r) { tdiag[I] = t; continue; }
      int face = -1;
      if (cb == rb && cc == rc && (ca == 0 || ca == p)) face = ca == 0 ? 0 : 1;
      else if (ca == ra && cc == rc && (cb == 0 || cb == p)) face = cb == 0 ? 2 : 3;
      else if (ca == ra && cb == rb && (cc == 0 || cc == p)) face = cc == 0 ? 4 : 5;
      if (face >= 0) tface[6 * (size_t)I + face] = t;
    }
    for (int I = 0; I < ni; ++I)
      if (tdiag[I] < 0) throw std::runtime_error("device setup: interior diagonal missing");
    if (!P.cartesian) {
      const AuxTables& T = aux_tables(p);
      const int n = P1;
      for (int k = 1; k < p; ++k)
        for (int j = 1; j < p; ++j)
          for (int i = 1; i < p; ++i) {
            const int I = ((k - 1) * pm + (j - 1)) * pm + (i - 1);
            widx[3 * I + 0] = T.off[1] + (k * n + j) * p + i;
            widx[3 * I + 1] = T.off[2] + (k * p + j) * n + i;
            widx[3 * I + 2] = T.off[3] + (k * n + j) * n + i;
          }
    }
    if (ncell > 0 && ni > 0)
      sc_cell_data_kernel<<<1184, 256, 0, st>>>(ncell, ni, ne, P.cartesian ? 1 : 0, d_cset, d_ck, d_cm, d_alpha, d_beta,
                                                d_cent, d_diag, ndiag, buf.up(tdiag, st), buf.up(tface, st),
                                                buf.up(widx, st), sc_dinv, sc_c, sc_w);
    DS_CK(cudaGetLastError());
  }
  if (nf == 0) { DS_CK(cudaStreamSynchronize(st)); return; }
  // ---- numeric programs of the classes used by some block
  std::vector<char> used(P.classes.size(), 0);
  for (int c : P.fclass) used[c] = 1;
  std::vector<NumProg> progs(P.classes.size());
  std::vector<int> ibuf;
  struct Ofs { long long o[17]; };
  std::vector<Ofs> ofs(P.classes.size());
  long long sP = 0, sM = 0, sS = 0, sY = 0, sC = 0;
  for (size_t c = 0; c < P.classes.size(); ++c) {
    if (!used[c]) continue;
    NumProg& g = progs[c];
    build_numeric_program(P.classes[c], P.cell_rows, P.cell_cols, g);
    const std::vector<int>* arrs[17] = {&g.asm_ptr, &g.asm_src, &g.pdiag, &g.b0, &g.nbr, &g.w0, &g.st_idx, &g.st_csr,
                                        &g.st_ptr, &g.st_src, &g.rec, &g.icc_rowptr, &g.icc_col, &g.icc_lptr,
                                        &g.icc_lrows, &g.icct_src, &g.smap};
    for (int k = 0; k < 17; ++k) {
      ofs[c].o[k] = (long long)ibuf.size();
      ibuf.insert(ibuf.end(), arrs[k]->begin(), arrs[k]->end());
      ibuf.resize((ibuf.size() + 3) & ~size_t(3));
    }
    const long long icc_nnz = g.icc_rowptr.empty() ? 0 : g.icc_rowptr.back();
    sP = std::max<long long>(sP, g.nnzP);
    sM = std::max<long long>(sM, 3LL * (long long)(g.nbr.size() / 7));
    sS = std::max<long long>(sS, g.final_kind == FINAL_ICC ? icc_nnz : (long long)g.nG * g.nG);
    if (g.final_kind != FINAL_ICC && g.m > 0) sY = std::max<long long>(sY, 1024LL * ((g.m + 31) / 32) * ((g.m + 31) / 32));
    sC = std::max<long long>(sC, g.ncanon);
  }
  const int* d_ibuf = buf.up(ibuf, st);
  std::vector<DNum> hd(P.classes.size());
  for (size_t c = 0; c < P.classes.size(); ++c) {
    DNum& d = hd[c];
    std::memset(&d, 0, sizeof d);
    if (!used[c]) continue;
    const NumProg& g = progs[c];
    d.n = g.n; d.nI = g.nI; d.nG = g.nG; d.m = g.m; d.nnzP = g.nnzP; d.final_kind = g.final_kind;
    d.nb0 = g.nb0; d.bs0 = g.bs0; d.nrec = (int)(g.rec.size() / 4); d.nw0 = (int)(g.w0.size() / 2);
    d.ntgt = (int)g.st_idx.size();
    d.icc_nnz = g.icc_rowptr.empty() ? 0 : g.icc_rowptr.back();
    d.icc_nlev = g.icc_lptr.empty() ? 0 : (int)g.icc_lptr.size() - 1;
    d.blk0_vofs = g.blk0_vofs; d.vofs_final = g.vofs_final; d.ncanon = g.ncanon; d.nvals = g.nvals;
    const int** ptrs[17] = {&d.asm_ptr, &d.asm_src, &d.pdiag, &d.b0, &d.nbr, &d.w0, &d.st_idx, &d.st_csr,
                            &d.st_ptr, &d.st_src, &d.rec, &d.icc_rowptr, &d.icc_col, &d.icc_lptr,
                            &d.icc_lrows, &d.icct_src, &d.smap};
    for (int k = 0; k < 17; ++k) *ptrs[k] = d_ibuf + ofs[c].o[k];
  }
  // ---- scratch: one slice per CTA, grid bounded by ~4 GB of scratch
  auto al = [](long long x) { return (x + 31) & ~31LL; };
  FArgs a{};
  a.sP = 0; a.sM = al(sP); a.sS = a.sM + al(sM); a.sY = a.sS + al(sS); a.sC = a.sY + al(sY);
  a.stride = a.sC + al(sC);
  int dev = 0, nsm = 148;
  DS_CK(cudaGetDevice(&dev));
  DS_CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  long long grid = std::min<long long>(nf, 4LL * nsm);
  grid = std::max<long long>(1, std::min<long long>(grid, (4LL << 30) / (8 * a.stride)));
  a.scratch = buf.alloc<double>((size_t)(grid * a.stride));
  a.progs = buf.up(hd, st);
  a.fclass = buf.up(P.fclass, st);
  a.fcells = buf.up(P.fcells, st);
  a.fdst = buf.up(fdst, st);
  a.nf = nf; a.ne = ne; a.cart = P.cartesian ? 1 : 0;
  a.cset_k = d_ck; a.cset_m = d_cm; a.cell_set = d_cset; a.alpha = d_alpha; a.beta = d_beta; a.cent = d_cent;
  a.vals = vals;
  a.sigma_bits = buf.alloc<unsigned long long>(1);
  a.err = buf.alloc<int>(2);
  DS_CK(cudaMemsetAsync(a.sigma_bits, 0, sizeof(unsigned long long), st));
  DS_CK(cudaMemsetAsync(a.err, 0, 2 * sizeof(int), st));
  factor_kernel<<<(unsigned)grid, NT, 0, st>>>(a);
  DS_CK(cudaGetLastError());
  int herr[2] = {0, 0};
  unsigned long long sb = 0;
  DS_CK(cudaMemcpyAsync(herr, a.err, sizeof herr, cudaMemcpyDeviceToHost, st));
  DS_CK(cudaMemcpyAsync(&sb, a.sigma_bits, sizeof sb, cudaMemcpyDeviceToHost, st));
  DS_CK(cudaStreamSynchronize(st));
  if (herr[0] != 0) {
    char msg[200];
    snprintf(msg, sizeof msg, "device setup: %s in value block %d", herr[1] == 2 ? "icc breakdown beyond sigma = 1e-2"
                                                                               : "non-positive pivot (exact factorization)",
             herr[0] - 1);
    throw NumericError(msg);
  }
  double sg = 0.0;
  std::memcpy(&sg, &sb, sizeof sg);
  if (sigma_max) *sigma_max = sg;
}

}  // namespace rm
