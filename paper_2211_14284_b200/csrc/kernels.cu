// sm_100a kernels of the relaxation sweep.
//
//  apply_cartesian_kernel  r = f - A u (or A u), matrix-free, output-stationary gather form of the
//                          sum-factorised cell operator eq:sum-factorization: every
//                          output DoF sums the Kronecker terms of the <= 8 cells that contain it;
//                          deterministic (no atomics), one thread per DoF, coalesced in x.
//  patch_solve_kernel      one CTA per star patch: gather R_i r into shared memory,
//                          block elimination (level 0 = cell interiors; independent-set
//                          levels), final Schur block by a packed symmetric inverse (exact
//                          Cholesky family) or level-scheduled ICC(0) triangular solves (ICC-SC,
//                          P:1142-1151), back substitution, scatter-add omega * R_i^T x into u.
//                          Patches of one colour never overlap, so plain read-modify-write is safe
//                          and the sweep is bitwise deterministic.
//  hiptmair_DT / _D_add    t = D^T r and u += omega D s for the Pavarino-Hiptmair potential stage
//                          (eq:asm-hiptmair P:961-975) with D the Kronecker-tabulated d^{k-1}.
//  axpby / dot / pcg_*     PCG vector kernels, fp64, deterministic reductions.
#include "kernels.cuh"

#include <cstdio>

namespace rm {

enum { FAM_P_ = 0, FAM_D_ = 1 };

__device__ __forceinline__ bool is_constrained_idx(int fam, long long idx, long long last, unsigned gamma_d, int d) {
  if (fam != FAM_P_) return false;
  if (idx == 0 && (gamma_d & (1u << (2 * d)))) return true;
  if (idx == last && (gamma_d & (1u << (2 * d + 1)))) return true;
  return false;
}

__device__ __forceinline__ int cells_of(long long I, int fam, int p, int ncell, int* c, int* a) {
  if (fam == FAM_D_) { c[0] = (int)(I / p); a[0] = (int)(I % p); return 1; }
  long long q = I / p;
  int r = (int)(I % p);
  if (r != 0) { c[0] = (int)q; a[0] = r; return 1; }
  int cnt = 0;
  if (q - 1 >= 0) { c[cnt] = (int)q - 1; a[cnt] = p; ++cnt; }
  if (q < ncell) { c[cnt] = (int)q; a[cnt] = 0; ++cnt; }
  return cnt;
}

// hpow layout: for direction d, exponent e in [-3,3]: hpow[hoff[d] + (e+3)*n[d] + cell]
__global__ void __launch_bounds__(256) apply_cartesian_kernel(const __grid_constant__ OpParams op,
                                                               const double* __restrict__ alpha,
                                                               const double* __restrict__ beta, int coef_const,
                                                               const double* __restrict__ hpow,
                                                               const double* __restrict__ u,
                                                               const double* __restrict__ f,
                                                               double* __restrict__ out, long long ndof) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ndof) return;
  int m = 0;
  while (m + 1 < op.ncomp && g >= op.off[m + 1]) ++m;
  const long long rr = g - op.off[m];
  const long long Lx = op.len[m][0], Ly = op.len[m][1];
  const long long idx[3] = {rr % Lx, (rr / Lx) % Ly, rr / (Lx * Ly)};
  const int p = op.p;
  for (int d = 0; d < 3; ++d)
    if (is_constrained_idx(op.fam[m][d], idx[d], (long long)op.n[d] * p, op.gamma_d, d)) { out[g] = 0.0; return; }
  int cc[3][2], aa[3][2], nc[3];
  for (int d = 0; d < 3; ++d) nc[d] = cells_of(idx[d], op.fam[m][d], p, op.n[d], cc[d], aa[d]);
  const int hoff[3] = {0, 7 * op.n[0], 7 * (op.n[0] + op.n[1])};
  double acc = 0.0;
  for (int t = 0; t < op.nterms; ++t) {
    const OpTerm& T = op.terms[t];
    if (T.mout != m) continue;
    const int mi = T.min;
    const long long Lxi = op.len[mi][0], Lyi = op.len[mi][1];
    const int mx = T.mat[0], my = T.mat[1], mz = T.mat[2];
    const int fx = op.fam[mi][0], fy = op.fam[mi][1], fz = op.fam[mi][2];
    const double* ub = u + op.off[mi];
    for (int kz = 0; kz < nc[2]; ++kz)
      for (int ky = 0; ky < nc[1]; ++ky)
        for (int kx = 0; kx < nc[0]; ++kx) {
          const int cx = cc[0][kx], cy = cc[1][ky], cz = cc[2][kz];
          const long long cell = ((long long)cz * op.n[1] + cy) * op.n[0] + cx;
          double scale = T.c * (T.coef == 0 ? (coef_const ? alpha[0] : alpha[cell]) : (coef_const ? beta[0] : beta[cell]));
          scale *= hpow[hoff[0] + (T.hexp[0] + 3) * op.n[0] + cx];
          scale *= hpow[hoff[1] + (T.hexp[1] + 3) * op.n[1] + cy];
          scale *= hpow[hoff[2] + (T.hexp[2] + 3) * op.n[2] + cz];
          const int ax = aa[0][kx], ay = aa[1][ky], az = aa[2][kz];
          double s = 0.0;
          for (int ez = op.rowptr[mz][az]; ez < op.rowptr[mz][az + 1]; ++ez) {
            const long long Iz = (long long)cz * p + op.col[mz][ez];
            if (is_constrained_idx(fz, Iz, (long long)op.n[2] * p, op.gamma_d, 2)) continue;
            const double vz = op.val[mz][ez];
            double sy = 0.0;
            for (int ey = op.rowptr[my][ay]; ey < op.rowptr[my][ay + 1]; ++ey) {
              const long long Iy = (long long)cy * p + op.col[my][ey];
              if (is_constrained_idx(fy, Iy, (long long)op.n[1] * p, op.gamma_d, 1)) continue;
              const double* urow = ub + (Iz * Lyi + Iy) * Lxi + (long long)cx * p;
              double sx = 0.0;
              for (int ex = op.rowptr[mx][ax]; ex < op.rowptr[mx][ax + 1]; ++ex) {
                const int cxl = op.col[mx][ex];
                if (is_constrained_idx(fx, (long long)cx * p + cxl, (long long)op.n[0] * p, op.gamma_d, 0)) continue;
                sx += op.val[mx][ex] * __ldg(urow + cxl);
              }
              sy += op.val[my][ey] * sx;
            }
            s += vz * sy;
          }
          acc += scale * s;
        }
  }
  out[g] = f ? (f[g] - acc) : acc;
}

cudaError_t launch_apply_cartesian(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                                   const double* hpow, const double* u, const double* f, double* out,
                                   long long ndof, cudaStream_t st) {
  const int T = 256;
  const long long B = (ndof + T - 1) / T;
  apply_cartesian_kernel<<<(unsigned)B, T, 0, st>>>(op, alpha, beta, coef_const, hpow, u, f, out, ndof);
  return cudaGetLastError();
}

// ====================================================================== patch solve
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int NT, int MAXT>
__global__ void __launch_bounds__(NT) patch_solve_kernel(const DClass* __restrict__ classes,
                                                        const int* __restrict__ pclass,
                                                        const long long* __restrict__ pbase,
                                                        const long long* __restrict__ pvals,
                                                        const double* __restrict__ vals,
                                                        const double* __restrict__ r, double* __restrict__ u,
                                                        double omega) {
  extern __shared__ double sm[];
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pi = blockIdx.x;
  const DClass& C = classes[pclass[pi]];
  const int n = C.n;
  double* v = sm;
  double* aux = sm + n;
  const long long b0 = pbase[3 * pi], b1 = pbase[3 * pi + 1], b2 = pbase[3 * pi + 2];
  const double* V = vals + pvals[pi];
  const int* offs = C.offs;
  const unsigned char* comp = C.comp;
  // ---- gather b = R_i r
  for (int t = tid; t < n; t += NT) {
    const int c = comp[t];
    const long long base = c == 0 ? b0 : (c == 1 ? b1 : b2);
    v[t] = r[base + offs[t]];
  }
  __syncthreads();
  // ---- forward eliminations: v_R -= W v_E
  const int nlev = C.nlev;
  for (int l = 0; l < nlev; ++l) {
    {   // y_E = L^{-1} v_E, thread per pivot block (<= 3x3, diagonal stored inverted)
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
      __syncthreads();
    }
    const DSliced& W = C.lev[l].w;
    const double* Wv = V + W.vofs;
    for (int s = warp; s < W.nslices; s += NW) {
      const int row = s * 32 + lane;
      const int w = __ldg(W.sw + s), o = __ldg(W.soff + s);
      double acc = 0.0;
      for (int kk = 0; kk < w; ++kk) {
        const int e = o + kk * 32 + lane;
        acc += __ldcs(Wv + e) * v[__ldg(W.cols + e)];
      }
      if (row < W.nrows) v[W.r0 + row] -= acc;
    }
    __syncthreads();
  }
  // ---- final Schur block
  const int m = C.m, f0 = n - m;
  if (C.final_kind == 0) {
    double vr[MAXT], cp[MAXT];
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const int j = lane + 32 * t;
      vr[t] = (j < m) ? v[f0 + j] : 0.0;
      cp[t] = 0.0;
    }
    double* rowsum = aux;
    double* parts = aux + m;
    const double* Sv = V + C.vofs_final;
    for (int i = warp; i < m; i += NW) {
      const double* row = Sv + (long long)i * (i + 1) / 2;
      const double vi = v[f0 + i];
      double racc = 0.0;
      double sv[MAXT];
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        const int j = lane + 32 * t;
        sv[t] = (j <= i) ? __ldcs(row + j) : 0.0;
      }
#pragma unroll
      for (int t = 0; t < MAXT; ++t) {
        const int j = lane + 32 * t;
        racc += sv[t] * vr[t];
        if (j < i) cp[t] += sv[t] * vi;
      }
      racc = warp_sum(racc);
      if (lane == 0) rowsum[i] = racc;
    }
#pragma unroll
    for (int t = 0; t < MAXT; ++t) {
      const int j = lane + 32 * t;
      if (j < m) parts[warp * m + j] = cp[t];
    }
    __syncthreads();
    for (int j = tid; j < m; j += NT) {
      double x = rowsum[j];
#pragma unroll
      for (int w = 0; w < NW; ++w) x += parts[w * m + j];
      v[f0 + j] = x;
    }
    __syncthreads();
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
      __syncthreads();
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
      __syncthreads();
    }
  }
  // ---- backward substitution: x_E = L^{-T} (y_E - M^T x_R)
  for (int l = nlev - 1; l >= 0; --l) {
    const DLevel& L = C.lev[l];
    const DSliced& WT = L.wt;
    const double* Tv = V + WT.vofs;
    for (int s = warp; s < WT.nslices; s += NW) {
      const int row = s * 32 + lane;
      double acc = (row < WT.nrows) ? v[L.e0 + row] : 0.0;
      const int w = __ldg(WT.sw + s), o = __ldg(WT.soff + s);
      for (int kk = 0; kk < w; ++kk) {
        const int e = o + kk * 32 + lane;
        acc -= __ldcs(Tv + e) * v[__ldg(WT.cols + e)];
      }
      if (row < WT.nrows) aux[row] = acc;
    }
    __syncthreads();
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
    __syncthreads();
  }
  // ---- scatter-add omega * R_i^T x
  for (int t = tid; t < n; t += NT) {
    const int c = comp[t];
    const long long base = c == 0 ? b0 : (c == 1 ? b1 : b2);
    double* up = u + base + offs[t];
    *up += omega * v[t];
  }
}

template <int MAXT>
static cudaError_t launch_ps(const DClass* classes, const int* pclass, const long long* pbase, const long long* pvals,
                             const double* vals, const double* r, double* u, double omega, int npatch,
                             size_t smem, cudaStream_t st) {
  auto kern = patch_solve_kernel<256, MAXT>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<npatch, 256, smem, st>>>(classes, pclass, pbase, pvals, vals, r, u, omega);
  return cudaGetLastError();
}

cudaError_t launch_patch_solve(const DClass* classes, const int* pclass, const long long* pbase,
                               const long long* pvals, const double* vals, const double* r, double* u,
                               double omega, int npatch, int maxT, size_t smem, cudaStream_t st) {
  if (npatch <= 0) return cudaSuccess;
  if (maxT <= 2) return launch_ps<2>(classes, pclass, pbase, pvals, vals, r, u, omega, npatch, smem, st);
  if (maxT <= 4) return launch_ps<4>(classes, pclass, pbase, pvals, vals, r, u, omega, npatch, smem, st);
  if (maxT <= 8) return launch_ps<8>(classes, pclass, pbase, pvals, vals, r, u, omega, npatch, smem, st);
  if (maxT <= 16) return launch_ps<16>(classes, pclass, pbase, pvals, vals, r, u, omega, npatch, smem, st);
  if (maxT <= 32) return launch_ps<32>(classes, pclass, pbase, pvals, vals, r, u, omega, npatch, smem, st);
  return cudaErrorInvalidValue;
}

// ====================================================================== Hiptmair D, D^T
// contributions of d^{k-1} (standard curl): target comp n <- sum sigma * d_e s_m
struct HipContrib { int n, m, e, sigma; };
__constant__ HipContrib c_grad[3] = {{0, 0, 0, 1}, {1, 0, 1, 1}, {2, 0, 2, 1}};
__constant__ HipContrib c_curl[6] = {{0, 2, 1, 1}, {0, 1, 2, -1}, {1, 0, 2, 1}, {1, 2, 0, -1}, {2, 1, 0, 1}, {2, 0, 1, -1}};

struct HipParams {
  int kpot;                 // form degree of the potential space (k - 1)
  int p, n[3];
  int fam_pot[3][3], fam_pri[3][3];
  long long len_pot[3][3], len_pri[3][3];
  long long off_pot[4], off_pri[4];
  int ncomp_pot, ncomp_pri;
  unsigned gamma_d;
  double D[RM_MAXP1 * RM_MAXP1];   // p x (p+1) row-major
};

__device__ __forceinline__ void decode(long long g, int ncomp, const long long* off, const long long (*len)[3],
                                       int& m, long long* idx) {
  m = 0;
  while (m + 1 < ncomp && g >= off[m + 1]) ++m;
  const long long rr = g - off[m];
  idx[0] = rr % len[m][0];
  idx[1] = (rr / len[m][0]) % len[m][1];
  idx[2] = rr / (len[m][0] * len[m][1]);
}

// t = D^T r on the potential space (zero on constrained potential DoFs)
__global__ void hiptmair_DT_kernel(const __grid_constant__ HipParams hp, const double* __restrict__ r,
                                   double* __restrict__ t, long long npot) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npot) return;
  int m;
  long long idx[3];
  decode(g, hp.ncomp_pot, hp.off_pot, hp.len_pot, m, idx);
  const int p = hp.p;
  for (int d = 0; d < 3; ++d)
    if (is_constrained_idx(hp.fam_pot[m][d], idx[d], (long long)hp.n[d] * p, hp.gamma_d, d)) { t[g] = 0.0; return; }
  const HipContrib* L = hp.kpot == 0 ? c_grad : c_curl;
  const int nL = hp.kpot == 0 ? 3 : 6;
  double acc = 0.0;
  for (int q = 0; q < nL; ++q) {
    if (L[q].m != m) continue;
    const int n = L[q].n, e = L[q].e;
    // (D^T r)_I along e: I is a P index in direction e; cells containing I; r_n index c p + a (DP)
    int cc[2], aa[2];
    const int nc = cells_of(idx[e], FAM_P_, p, hp.n[e], cc, aa);
    double s = 0.0;
    for (int k = 0; k < nc; ++k) {
      long long j[3] = {idx[0], idx[1], idx[2]};
      for (int a = 0; a < p; ++a) {
        j[e] = (long long)cc[k] * p + a;
        const double dv = hp.D[a * (p + 1) + aa[k]];
        if (dv == 0.0) continue;
        s += dv * r[hp.off_pri[n] + (j[2] * hp.len_pri[n][1] + j[1]) * hp.len_pri[n][0] + j[0]];
      }
    }
    acc += L[q].sigma * s;
  }
  t[g] = acc;
}

// u += omega * D s on the primal space (zero contribution on constrained primal DoFs)
__global__ void hiptmair_D_add_kernel(const __grid_constant__ HipParams hp, const double* __restrict__ s,
                                      double* __restrict__ u, double omega, long long npri) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npri) return;
  int n;
  long long idx[3];
  decode(g, hp.ncomp_pri, hp.off_pri, hp.len_pri, n, idx);
  const int p = hp.p;
  for (int d = 0; d < 3; ++d)
    if (is_constrained_idx(hp.fam_pri[n][d], idx[d], (long long)hp.n[d] * p, hp.gamma_d, d)) return;
  const HipContrib* L = hp.kpot == 0 ? c_grad : c_curl;
  const int nL = hp.kpot == 0 ? 3 : 6;
  double acc = 0.0;
  for (int q = 0; q < nL; ++q) {
    if (L[q].n != n) continue;
    const int m = L[q].m, e = L[q].e;
    // (d_e s_m)_I : I is a DP index along e in cell c = I / p, a = I % p
    const int c = (int)(idx[e] / p), a = (int)(idx[e] % p);
    long long j[3] = {idx[0], idx[1], idx[2]};
    double sum = 0.0;
    for (int i = 0; i <= p; ++i) {
      const double dv = hp.D[a * (p + 1) + i];
      if (dv == 0.0) continue;
      j[e] = (long long)c * p + i;
      sum += dv * s[hp.off_pot[m] + (j[2] * hp.len_pot[m][1] + j[1]) * hp.len_pot[m][0] + j[0]];
    }
    acc += L[q].sigma * sum;
  }
  u[g] += omega * acc;
}

static HipParams make_hip(int k, int p, const int* n, unsigned gamma_d, const double* Dh) {
  static const int FAMS[4][3][3] = {
      {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
      {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
      {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{1, 1, 1}, {0, 0, 0}, {0, 0, 0}},
  };
  HipParams hp{};
  hp.kpot = k - 1; hp.p = p;
  for (int d = 0; d < 3; ++d) hp.n[d] = n[d];
  hp.ncomp_pot = (k - 1 == 0) ? 1 : 3;
  hp.ncomp_pri = (k == 0 || k == 3) ? 1 : 3;
  hp.gamma_d = gamma_d;
  long long o1 = 0, o2 = 0;
  for (int m = 0; m < 3; ++m) {
    hp.off_pot[m] = o1; hp.off_pri[m] = o2;
    long long s1 = 1, s2 = 1;
    for (int d = 0; d < 3; ++d) {
      hp.fam_pot[m][d] = FAMS[k - 1][m][d];
      hp.fam_pri[m][d] = FAMS[k][m][d];
      hp.len_pot[m][d] = hp.fam_pot[m][d] == 0 ? (long long)n[d] * p + 1 : (long long)n[d] * p;
      hp.len_pri[m][d] = hp.fam_pri[m][d] == 0 ? (long long)n[d] * p + 1 : (long long)n[d] * p;
      s1 *= hp.len_pot[m][d]; s2 *= hp.len_pri[m][d];
    }
    if (m < hp.ncomp_pot) o1 += s1;
    if (m < hp.ncomp_pri) o2 += s2;
  }
  hp.off_pot[3] = o1; hp.off_pri[3] = o2;
  for (int i = 0; i < p * (p + 1); ++i) hp.D[i] = Dh[i];
  return hp;
}

cudaError_t launch_hiptmair_DT(int k, int p, const int* n, unsigned gamma_d, const double* Dh, const double* r,
                               double* t, cudaStream_t st) {
  HipParams hp = make_hip(k, p, n, gamma_d, Dh);
  const long long N = hp.off_pot[hp.ncomp_pot];
  hiptmair_DT_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(hp, r, t, N);
  return cudaGetLastError();
}

cudaError_t launch_hiptmair_D_add(int k, int p, const int* n, unsigned gamma_d, const double* Dh, const double* s,
                                  double* u, double omega, cudaStream_t st) {
  HipParams hp = make_hip(k, p, n, gamma_d, Dh);
  const long long N = hp.off_pri[hp.ncomp_pri];
  hiptmair_D_add_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(hp, s, u, omega, N);
  return cudaGetLastError();
}

// ====================================================================== vector kernels
__global__ void axpby_kernel(long long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}
cudaError_t launch_axpby(long long n, double a, const double* x, double b, double* y, cudaStream_t st) {
  axpby_kernel<<<148 * 8, 256, 0, st>>>(n, a, x, b, y);
  return cudaGetLastError();
}

#define RM_DOT_BLOCKS 592
__global__ void dot_stage1(long long n, const double* __restrict__ x, const double* __restrict__ y, double* partial) {
  __shared__ double sh[8];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += x[i] * y[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < 8 ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}
__global__ void dot_stage2(const double* partial, int nb, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) *out = t;
  }
}
cudaError_t launch_dot(long long n, const double* x, const double* y, double* partial, double* out, cudaStream_t st) {
  dot_stage1<<<RM_DOT_BLOCKS, 256, 0, st>>>(n, x, y, partial);
  dot_stage2<<<1, 256, 0, st>>>(partial, RM_DOT_BLOCKS, out);
  return cudaGetLastError();
}

// x += a p ; r -= a q  with a = num/den read on device
__global__ void pcg_update_kernel(long long n, const double* num, const double* den, const double* __restrict__ p,
                                  const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r) {
  const double a = *num / *den;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    r[i] -= a * q[i];
  }
}
cudaError_t launch_pcg_update(long long n, const double* num, const double* den, const double* p, const double* q,
                              double* x, double* r, cudaStream_t st) {
  pcg_update_kernel<<<148 * 8, 256, 0, st>>>(n, num, den, p, q, x, r);
  return cudaGetLastError();
}
// p = z + (rz_new/rz_old) p
__global__ void pcg_pupdate_kernel(long long n, const double* rzn, const double* rzo, const double* __restrict__ z,
                                   double* __restrict__ p) {
  const double b = *rzn / *rzo;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + b * p[i];
}
cudaError_t launch_pcg_pupdate(long long n, const double* rz_new, const double* rz_old, const double* z, double* p,
                               cudaStream_t st) {
  pcg_pupdate_kernel<<<148 * 8, 256, 0, st>>>(n, rz_new, rz_old, z, p);
  return cudaGetLastError();
}

}  // namespace rm
