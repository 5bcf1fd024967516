// Matrix-free Cartesian H(curl) / H(div) operator (k = 1, 2):
// r = f - A u or v = A u with, on an axis-aligned box (eq:sum-factorization P:690-699, pullbacks
// P:640-648, detJ = hx hy hz / 8),
//   k = 1:  A_K u = beta M^1 u + alpha C^T M^2 C u     (C = the reference curl, standard sign, G17)
//   k = 2:  A_K u = beta M^2 u + alpha D^T M^3 D u     (D = the reference divergence)
// with M^1_m = 0.5 hx hy hz / h_m^2 (B-hat on the P directions of NCE comp m, identity on its DP
// direction), M^2_n = 2 h_n^2 / (hx hy hz) (B-hat along n, identity elsewhere), M^3 = 8 / (hx hy hz).
//
// In the FDM basis every 1D factor is (nearly) diagonal: B-hat = diag + the (0,p) corner, D-hat
// row a = entries at columns 0, p and a (eq:gradbasis), so C, D, C^T, D^T and the masses are
// POINTWISE maps with <= 4 reads each, except D-hat^T onto the two vertex indices (a p-term sum).
// One CTA per cell: the cell's u in shared memory, then 3 (k = 1) / 2 (k = 2) pointwise stages
// with one barrier each -- O(p^3) per cell, no line loops.  Output: one launch over all cells
// (no colours); entries interior to the cell (in every P direction) are final and stored
// directly as f - A u; skeleton entries go to the per-cell buffer and kform_gather_rows_kernel sums
// the <= 4 cell contributions of each in a fixed order (bitwise deterministic).
#include "kernels.cuh"

namespace rm {

namespace {

constexpr int KF_THREADS = 128;   // measured per apply: 64 -> 0.36 / 0.42 ms, 128 -> 0.26 / 0.26 ms, 256 -> 0.29 / 0.28 ms (cfg3 / cfg4)

// (D-hat x)_a along a line with stride s (source: P + 1 entries)
template <int P>
__device__ __forceinline__ double dline(const double* __restrict__ sD, const double* x, int s, int a) {
  constexpr int N = P + 1;
  double v = sD[a * N] * x[0] + sD[a * N + P] * x[P * s];
  if (a >= 1) v += sD[a * N + a] * x[a * s];
  return v;
}
// (D-hat^T y)_j along a line with stride s (source: P entries)
template <int P>
__device__ __forceinline__ double dtline(const double* __restrict__ sD, const double* y, int s, int j) {
  constexpr int N = P + 1;
  if (j >= 1 && j < P) return sD[j * N + j] * y[j * s];
  double v = 0.0;
#pragma unroll
  for (int a = 0; a < P; ++a) v += sD[a * N + j] * y[a * s];
  return v;
}
// (B-hat x)_i along a line with stride s (source: P + 1 entries)
template <int P>
__device__ __forceinline__ double bline(const double* __restrict__ sB, const double* x, int s, int i) {
  constexpr int N = P + 1;
  if (i >= 1 && i < P) return sB[i * N + i] * x[i * s];
  return sB[i * N] * x[0] + sB[i * N + P] * x[P * s];
}
// (B-hat (x) B-hat) on a 2D slice: directions with strides s1, s2, output indices i1, i2
template <int P>
__device__ __forceinline__ double bb(const double* __restrict__ sB, const double* x, int s1, int i1, int s2, int i2) {
  constexpr int N = P + 1;
  const bool c1 = i1 == 0 || i1 == P, c2 = i2 == 0 || i2 == P;
  const double* x0 = x - i1 * s1 - i2 * s2;   // line origin
  if (!c1 && !c2) return sB[i1 * N + i1] * sB[i2 * N + i2] * x[0];
  if (!c1) return sB[i1 * N + i1] * bline<P>(sB, x0 + i1 * s1, s2, i2);
  if (!c2) return sB[i2 * N + i2] * bline<P>(sB, x0 + i2 * s2, s1, i1);
  return sB[i1 * N] * bline<P>(sB, x0, s2, i2) + sB[i1 * N + P] * bline<P>(sB, x0 + P * s1, s2, i2);
}

struct CellCtx {
  int cx, cy, cz;
  double al, be, hx, hy, hz;
  unsigned clo, chi;   // bit d: the cell's low / high face in direction d lies on a Gamma_D plane
};

__device__ __forceinline__ CellCtx cell_ctx(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                                            const double* hpow, int cell) {
  CellCtx c;
  c.cx = cell % op.n[0];
  c.cy = (cell / op.n[0]) % op.n[1];
  c.cz = cell / (op.n[0] * op.n[1]);
  c.al = coef_const ? alpha[0] : alpha[cell];
  c.be = coef_const ? beta[0] : beta[cell];
  c.hx = hpow[4 * op.n[0] + c.cx];
  c.hy = hpow[7 * op.n[0] + 4 * op.n[1] + c.cy];
  c.hz = hpow[7 * (op.n[0] + op.n[1]) + 4 * op.n[2] + c.cz];
  const int cc[3] = {c.cx, c.cy, c.cz};
  c.clo = c.chi = 0;
  for (int d = 0; d < 3; ++d) {
    if (cc[d] == 0 && (op.gamma_d & (1u << (2 * d)))) c.clo |= 1u << d;
    if (cc[d] == op.n[d] - 1 && (op.gamma_d & (1u << (2 * d + 1)))) c.chi |= 1u << d;
  }
  return c;
}

// 64-bit global index of the cell window's origin in component m (32-bit offsets inside)
__device__ __forceinline__ long long comp_base(const OpParams& op, int m, const CellCtx& c) {
  const int p = op.p;
  return op.off[m] + ((long long)(c.cz * p) * op.len[m][1] + c.cy * p) * op.len[m][0] + c.cx * p;
}

// gathers one component of the cell window (local dims LX, LY, LZ; P-family mask FP: bit d set
// for a P direction) into shared memory, constrained entries read as 0
template <int P, int LX, int LY, int LZ, int FP>
__device__ __forceinline__ void load_comp(const OpParams& op, int m, const CellCtx& c, const double* __restrict__ u,
                                          double* dst) {
  const double* ub = u + comp_base(op, m, c);
  const int Lx = (int)op.len[m][0], Lxy = (int)(op.len[m][0] * op.len[m][1]);
  constexpr int TOT = LX * LY * LZ;
  const unsigned lo = c.clo & FP, hi = c.chi & FP;
  for (int l = threadIdx.x; l < TOT; l += KF_THREADS) {
    const int a = l % LX, b = (l / LX) % LY, cc = l / (LX * LY);
    bool con = false;
    if (lo | hi) {
      con = ((lo & 1) && a == 0) || ((hi & 1) && a == P) || ((lo & 2) && b == 0) || ((hi & 2) && b == P) ||
            ((lo & 4) && cc == 0) || ((hi & 4) && cc == P);
    }
    dst[l] = con ? 0.0 : __ldg(ub + cc * Lxy + b * Lx + a);
  }
}

// stores one output entry: interior entries final (out = f + sign v), skeleton ones to the buffer
// (a cell-interior entry is never constrained: Gamma_D planes are cell faces)
__device__ __forceinline__ void store_entry(const OpParams& op, long long base, int m, int a, int b, int cc, bool skel,
                                            int cell, int nloc, int l, double v, const double* __restrict__ f,
                                            double* __restrict__ out, double* __restrict__ cellbuf, double sign) {
  if (skel) {
    cellbuf[(long long)cell * nloc + l] = v;
    return;
  }
  const long long g = base + cc * (int)(op.len[m][0] * op.len[m][1]) + b * (int)op.len[m][0] + a;
  out[g] = (f ? __ldg(f + g) : 0.0) + sign * v;
}

template <int P>
__global__ void __launch_bounds__(KF_THREADS) apply_nce_kernel(const __grid_constant__ OpParams op,
                                                                const double* __restrict__ alpha,
                                                                const double* __restrict__ beta, int coef_const,
                                                                const double* __restrict__ hpow,
                                                                const double* __restrict__ u,
                                                                const double* __restrict__ f, double* __restrict__ out,
                                                                double* __restrict__ cellbuf, double sign) {
  constexpr int N = P + 1, NC = P * N * N, NF = N * P * P;
  extern __shared__ double sm[];
  double* sB = sm;             // N x N
  double* sD = sB + N * N;     // P x N
  double* U = sD + P * N;      // 3 NC   NCE comps: x (P,N,N), y (N,P,N), z (N,N,P)
  double* W = U + 3 * NC;      // 3 NF   NCF comps: x (N,P,P), y (P,N,P), z (P,P,N)
  double* W2 = W + 3 * NF;     // 3 NF
  const int cell = blockIdx.x;
  const CellCtx c = cell_ctx(op, alpha, beta, coef_const, hpow, cell);
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) sB[i] = op.Bh[i];
  for (int i = threadIdx.x; i < P * N; i += blockDim.x) sD[i] = op.Dh[i];
  load_comp<P, P, N, N, 6>(op, 0, c, u, U);
  load_comp<P, N, P, N, 5>(op, 1, c, u, U + NC);
  load_comp<P, N, N, P, 3>(op, 2, c, u, U + 2 * NC);
  __syncthreads();
  const double* Ux = U;
  const double* Uy = U + NC;
  const double* Uz = U + 2 * NC;
  // curl: w_x = D_y u_z - D_z u_y, w_y = D_z u_x - D_x u_z, w_z = D_x u_y - D_y u_x
  for (int l = threadIdx.x; l < 3 * NF; l += blockDim.x) {
    const int n = l / NF, r = l - n * NF;
    double w;
    if (n == 0) {          // (N,P,P): a < N, b < P, cc < P
      const int a = r % N, b = (r / N) % P, cc = r / (N * P);
      w = dline<P>(sD, Uz + (cc * N) * N + a, N, b) - dline<P>(sD, Uy + b * N + a, P * N, cc);
    } else if (n == 1) {   // (P,N,P)
      const int a = r % P, b = (r / P) % N, cc = r / (P * N);
      w = dline<P>(sD, Ux + b * P + a, N * P, cc) - dline<P>(sD, Uz + (cc * N + b) * N, 1, a);
    } else {               // (P,P,N)
      const int a = r % P, b = (r / P) % P, cc = r / (P * P);
      w = dline<P>(sD, Uy + (cc * P + b) * N, 1, a) - dline<P>(sD, Ux + (cc * N) * P + a, P, b);
    }
    W[l] = w;
  }
  __syncthreads();
  // W2 = alpha M^2 W: B-hat along the P direction of each NCF component
  {
    const double hv = c.hx * c.hy * c.hz;
    const double s2[3] = {2.0 * c.hx * c.hx / hv, 2.0 * c.hy * c.hy / hv, 2.0 * c.hz * c.hz / hv};
    for (int l = threadIdx.x; l < 3 * NF; l += blockDim.x) {
      const int n = l / NF, r = l - n * NF;
      double w;
      if (n == 0) {
        const int a = r % N;
        w = bline<P>(sB, W + l - a, 1, a);
      } else if (n == 1) {
        const int b = (r / P) % N;
        w = bline<P>(sB, W + l - b * P, P, b);
      } else {
        const int cc = r / (P * P);
        w = bline<P>(sB, W + l - cc * P * P, P * P, cc);
      }
      W2[l] = c.al * s2[n] * w;
    }
  }
  __syncthreads();
  // v = beta M^1 u + C^T W2
  const double hv = c.hx * c.hy * c.hz;
  const double s1[3] = {0.5 * hv / (c.hx * c.hx), 0.5 * hv / (c.hy * c.hy), 0.5 * hv / (c.hz * c.hz)};
  const double* Wx = W2;
  const double* Wy = W2 + NF;
  const double* Wz = W2 + 2 * NF;
  constexpr int nloc = 3 * NC;
  const long long base[3] = {comp_base(op, 0, c), comp_base(op, 1, c), comp_base(op, 2, c)};
  for (int l = threadIdx.x; l < 3 * NC; l += blockDim.x) {
    const int m = l / NC, r = l - m * NC;
    double v;
    int a, b, cc;
    bool skel;
    if (m == 0) {          // (P,N,N): P dirs y, z
      a = r % P; b = (r / P) % N; cc = r / (P * N);
      v = c.be * s1[0] * bb<P>(sB, Ux + r, P, b, P * N, cc);
      v += dtline<P>(sD, Wy + (b * P) + a, N * P, cc) - dtline<P>(sD, Wz + (cc * P) * P + a, P, b);
      skel = b == 0 || b == P || cc == 0 || cc == P;
    } else if (m == 1) {   // (N,P,N): P dirs x, z
      a = r % N; b = (r / N) % P; cc = r / (N * P);
      v = c.be * s1[1] * bb<P>(sB, Uy + r, 1, a, N * P, cc);
      v += dtline<P>(sD, Wz + (cc * P + b) * P, 1, a) - dtline<P>(sD, Wx + b * N + a, P * N, cc);
      skel = a == 0 || a == P || cc == 0 || cc == P;
    } else {               // (N,N,P): P dirs x, y
      a = r % N; b = (r / N) % N; cc = r / (N * N);
      v = c.be * s1[2] * bb<P>(sB, Uz + r, 1, a, N, b);
      v += dtline<P>(sD, Wx + (cc * P) * N + a, N, b) - dtline<P>(sD, Wy + (cc * N + b) * P, 1, a);
      skel = a == 0 || a == P || b == 0 || b == P;
    }
    store_entry(op, base[m], m, a, b, cc, skel, cell, nloc, l, v, f, out, cellbuf, sign);
  }
}

template <int P>
__global__ void __launch_bounds__(KF_THREADS) apply_ncf_kernel(const __grid_constant__ OpParams op,
                                                                const double* __restrict__ alpha,
                                                                const double* __restrict__ beta, int coef_const,
                                                                const double* __restrict__ hpow,
                                                                const double* __restrict__ u,
                                                                const double* __restrict__ f, double* __restrict__ out,
                                                                double* __restrict__ cellbuf, double sign) {
  constexpr int N = P + 1, NF = N * P * P, N3 = P * P * P;
  extern __shared__ double sm[];
  double* sB = sm;
  double* sD = sB + N * N;
  double* U = sD + P * N;      // 3 NF: x (N,P,P), y (P,N,P), z (P,P,N)
  double* Dv = U + 3 * NF;     // P^3
  const int cell = blockIdx.x;
  const CellCtx c = cell_ctx(op, alpha, beta, coef_const, hpow, cell);
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) sB[i] = op.Bh[i];
  for (int i = threadIdx.x; i < P * N; i += blockDim.x) sD[i] = op.Dh[i];
  load_comp<P, N, P, P, 1>(op, 0, c, u, U);
  load_comp<P, P, N, P, 2>(op, 1, c, u, U + NF);
  load_comp<P, P, P, N, 4>(op, 2, c, u, U + 2 * NF);
  __syncthreads();
  const double* Ux = U;
  const double* Uy = U + NF;
  const double* Uz = U + 2 * NF;
  const double hv = c.hx * c.hy * c.hz;
  // d' = alpha M^3 (D_x u_x + D_y u_y + D_z u_z)
  {
    const double s3 = c.al * 8.0 / hv;
    for (int l = threadIdx.x; l < N3; l += blockDim.x) {
      const int a = l % P, b = (l / P) % P, cc = l / (P * P);
      const double d = dline<P>(sD, Ux + (cc * P + b) * N, 1, a) + dline<P>(sD, Uy + (cc * N) * P + a, P, b) +
                       dline<P>(sD, Uz + b * P + a, P * P, cc);
      Dv[l] = s3 * d;
    }
  }
  __syncthreads();
  const double s2[3] = {2.0 * c.hx * c.hx / hv, 2.0 * c.hy * c.hy / hv, 2.0 * c.hz * c.hz / hv};
  constexpr int nloc = 3 * NF;
  const long long base[3] = {comp_base(op, 0, c), comp_base(op, 1, c), comp_base(op, 2, c)};
  for (int l = threadIdx.x; l < 3 * NF; l += blockDim.x) {
    const int m = l / NF, r = l - m * NF;
    double v;
    int a, b, cc;
    bool skel;
    if (m == 0) {          // (N,P,P): P dir x
      a = r % N; b = (r / N) % P; cc = r / (N * P);
      v = c.be * s2[0] * bline<P>(sB, Ux + r - a, 1, a) + dtline<P>(sD, Dv + (cc * P + b) * P, 1, a);
      skel = a == 0 || a == P;
    } else if (m == 1) {   // (P,N,P): P dir y
      a = r % P; b = (r / P) % N; cc = r / (P * N);
      v = c.be * s2[1] * bline<P>(sB, Uy + r - b * P, P, b) + dtline<P>(sD, Dv + (cc * P) * P + a, P, b);
      skel = b == 0 || b == P;
    } else {               // (P,P,N): P dir z
      a = r % P; b = (r / P) % P; cc = r / (P * P);
      v = c.be * s2[2] * bline<P>(sB, Uz + r - cc * P * P, P * P, cc) + dtline<P>(sD, Dv + b * P + a, P * P, cc);
      skel = cc == 0 || cc == P;
    }
    store_entry(op, base[m], m, a, b, cc, skel, cell, nloc, l, v, f, out, cellbuf, sign);
  }
}

// (A-hat x)_i along a line with stride s: interior rows (0, i, p), vertex rows full (eq:fdmbasis)
template <int P>
__device__ __forceinline__ double aline(const double* __restrict__ sA, const double* x, int s, int i) {
  constexpr int N = P + 1;
  if (i >= 1 && i < P) return sA[i * N] * x[0] + sA[i * N + i] * x[i * s] + sA[i * N + P] * x[P * s];
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) v += sA[i * N + j] * x[j * s];
  return v;
}

// H(grad), Cartesian (k = 0): A_K u = beta s_M (B B B) u + alpha sum_d s_d (A-hat along d, B-hat
// across), in three pointwise stages on the cell window (x: B u, A u; y: B (Bu), A (Bu), B (Au)
// combined into Q = beta s_M B B u + alpha (s_x B A u + s_y A B u); z: v = B_z Q + alpha s_z A_z (B B u)).
// One CTA per cell, ONE launch over all cells; interior entries final (out = f + sign v, padded
// x-stride ldx), skeleton entries to the cell buffer, summed by kform_gather_rows_kernel.
template <int P>
__global__ void __launch_bounds__(KF_THREADS) apply_q_pw_kernel(const __grid_constant__ OpParams op,
                                                                 const double* __restrict__ alpha,
                                                                 const double* __restrict__ beta, int coef_const,
                                                                 const double* __restrict__ hpow,
                                                                 const double* __restrict__ u,
                                                                 const double* __restrict__ f, double* __restrict__ out,
                                                                 long long ldx, double* __restrict__ cellbuf,
                                                                 double sign) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  extern __shared__ double sm[];
  double* sB = sm;
  double* sA = sB + N2;
  double* U = sA + N2;
  double* X1 = U + N3;
  double* X2 = X1 + N3;
  double* Y1 = X2 + N3;
  double* Q = U;   // U is dead after the x stage
  const int cell = blockIdx.x;
  const CellCtx c = cell_ctx(op, alpha, beta, coef_const, hpow, cell);
  for (int i = threadIdx.x; i < N2; i += blockDim.x) { sB[i] = op.Bh[i]; sA[i] = op.Ah[i]; }
  load_comp<P, N, N, N, 7>(op, 0, c, u, U);
  __syncthreads();
  for (int l = threadIdx.x; l < N3; l += KF_THREADS) {
    const int a = l % N;
    X1[l] = bline<P>(sB, U + l - a, 1, a);
    X2[l] = aline<P>(sA, U + l - a, 1, a);
  }
  __syncthreads();
  const double hv = c.hx * c.hy * c.hz;
  const double sM = c.be * hv * 0.125, sx = c.al * c.hy * c.hz / (2.0 * c.hx), sy = c.al * c.hx * c.hz / (2.0 * c.hy),
               sz = c.al * c.hx * c.hy / (2.0 * c.hz);
  for (int l = threadIdx.x; l < N3; l += KF_THREADS) {
    const int b = (l / N) % N;
    const double* x1 = X1 + l - b * N;
    const double y1 = bline<P>(sB, x1, N, b);
    const double y2 = aline<P>(sA, x1, N, b);
    const double y3 = bline<P>(sB, X2 + l - b * N, N, b);
    Y1[l] = y1;
    Q[l] = sM * y1 + sx * y3 + sy * y2;
  }
  __syncthreads();
  const long long Lx = op.len[0][0], Ly = op.len[0][1];
  const long long ox = (long long)c.cx * P, oy = (long long)c.cy * P, oz = (long long)c.cz * P;
  for (int l = threadIdx.x; l < N3; l += KF_THREADS) {
    const int a = l % N, b = (l / N) % N, cc = l / N2;
    const double v = bline<P>(sB, Q + l - cc * N2, N2, cc) + sz * aline<P>(sA, Y1 + l - cc * N2, N2, cc);
    if (a == 0 || a == P || b == 0 || b == P || cc == 0 || cc == P) {
      cellbuf[(long long)cell * N3 + l] = v;
    } else {   // interior of the cell: never constrained
      const long long row = (oz + cc) * Ly + oy + b;
      out[row * ldx + ox + a] = (f ? __ldg(f + row * Lx + ox + a) : 0.0) + sign * v;
    }
  }
}

// out[g] = f[g] + sign * sum over the <= 4 cells carrying skeleton DoF g of their buffered
// contributions (cells in z, y, x order); constrained entries 0; cell-interior entries were
// stored by the apply kernel and are left alone.
// The same sums, row by row: one (y, z) row of one component per warp, SKELETON entries only
// (the apply kernels store the cell-interior entries final, out = f + sign A_K u).  A row whose y
// and z indices are both cell-interior visits only its x-boundary entries (x in the P family) or
// nothing (x in the DP family); the per-DoF divisions and the interior passes of the one-thread-
// per-DoF gather are gone.  Same addends in the same order (cells in z, y, x order): bitwise equal.
__device__ __forceinline__ void kf_dir(int idx, bool P_, int p, int n, unsigned gam, int d, int& c0, int& a0, int& two,
                                       bool& skel, bool& con) {
  const int cc = idx / p, aa = idx - cc * p;
  two = 0;
  skel = false;
  con = false;
  if (P_ && aa == 0) {
    skel = true;
    if (cc == 0) { c0 = 0; a0 = 0; }
    else if (cc == n) { c0 = cc - 1; a0 = p; }
    else { c0 = cc - 1; a0 = p; two = 1; }
    con = (cc == 0 && (gam & (1u << (2 * d)))) || (cc == n && (gam & (2u << (2 * d))));
  } else {
    c0 = cc; a0 = aa;
  }
}

__global__ void kform_gather_rows_kernel(const __grid_constant__ OpParams op, const double* __restrict__ cellbuf,
                                         const double* __restrict__ f, double* __restrict__ out, double sign, int nloc,
                                         long long ldx) {
  const int p = op.p, lane = threadIdx.x & 31;
  const int wstride = gridDim.x * (blockDim.x >> 5);
  int rows_before = 0, lo = 0;
  for (int m = 0; m < op.ncomp; ++m) {
    const int Lx = (int)op.len[m][0], Ly = (int)op.len[m][1], Lz = (int)op.len[m][2], nrow = Ly * Lz;
    const bool Px = op.fam[m][0] == 0, Py = op.fam[m][1] == 0, Pz = op.fam[m][2] == 0;
    const int ls0 = Px ? p + 1 : p, ls1 = Py ? p + 1 : p, ls2 = Pz ? p + 1 : p;
    for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) - rows_before; r < nrow; r += wstride) {
      if (r < 0) continue;
      const int iy = r % Ly, iz = r / Ly;
      int cy0, ay0, twy, cz0, az0, twz;
      bool sy, sz, cy, cz;
      kf_dir(iy, Py, p, op.n[1], op.gamma_d, 1, cy0, ay0, twy, sy, cy);
      kf_dir(iz, Pz, p, op.n[2], op.gamma_d, 2, cz0, az0, twz, sz, cz);
      const bool rskel = sy || sz, rcons = cy || cz;
      if (!rskel && !Px) continue;   // no skeleton entry in this row
      const int cnt = rskel ? Lx : op.n[0] + 1;
      const long long fb = op.off[m] + (long long)r * Lx;
      const long long ob = ldx > 0 ? (long long)r * ldx : fb;
      for (int t = lane; t < cnt; t += 32) {
        const int ix = rskel ? t : t * p;
        int cx0, ax0, twx;
        bool sx, cxn;
        kf_dir(ix, Px, p, op.n[0], op.gamma_d, 0, cx0, ax0, twx, sx, cxn);
        if (rcons || cxn) { out[ob + ix] = 0.0; continue; }
        double s = 0.0;
        for (int kz = 0; kz <= twz; ++kz)
          for (int ky = 0; ky <= twy; ++ky)
            for (int kx = 0; kx <= twx; ++kx) {
              const int cx = cx0 + kx, ax = kx ? 0 : ax0;
              const int cyy = cy0 + ky, ay = ky ? 0 : ay0;
              const int czz = cz0 + kz, az = kz ? 0 : az0;
              const long long cell = ((long long)czz * op.n[1] + cyy) * op.n[0] + cx;
              s += cellbuf[cell * nloc + lo + (az * ls1 + ay) * ls0 + ax];
            }
        out[ob + ix] = (f ? f[fb + ix] : 0.0) + sign * s;
      }
    }
    rows_before += nrow;
    lo += ls0 * ls1 * ls2;
  }
}

template <int P>
cudaError_t launch_kform_p(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                           const double* hpow, const double* u, const double* f, double* out, double* cellbuf,
                           double sign, cudaStream_t st) {
  constexpr int N = P + 1;
  const int ncell = op.n[0] * op.n[1] * op.n[2];
  if (op.k == 0) {
    const size_t smem = sizeof(double) * (size_t)(2 * N * N + 4 * N * N * N);
    static bool set = false;
    if (!set && smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(apply_q_pw_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    set = true;
    const long long ldx = op.ldx_out > 0 ? op.ldx_out : op.len[0][0];
    apply_q_pw_kernel<P><<<ncell, KF_THREADS, smem, st>>>(op, alpha, beta, coef_const, hpow, u, f, out, ldx, cellbuf, sign);
  } else if (op.k == 1) {
    const size_t smem = sizeof(double) * (size_t)(N * N + P * N + 3 * P * N * N + 6 * N * P * P);
    static bool set = false;
    if (!set && smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(apply_nce_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    set = true;
    apply_nce_kernel<P><<<ncell, KF_THREADS, smem, st>>>(op, alpha, beta, coef_const, hpow, u, f, out, cellbuf, sign);
  } else {
    const size_t smem = sizeof(double) * (size_t)(N * N + P * N + 3 * N * P * P + P * P * P);
    static bool set = false;
    if (!set && smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(apply_ncf_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    set = true;
    apply_ncf_kernel<P><<<ncell, KF_THREADS, smem, st>>>(op, alpha, beta, coef_const, hpow, u, f, out, cellbuf, sign);
  }
  return cudaGetLastError();
}

}  // namespace

size_t kform_cellbuf_doubles(int k, int p, const int* n) {
  const size_t nloc = k == 0 ? (size_t)(p + 1) * (p + 1) * (p + 1)
                             : (k == 1 ? 3 * (size_t)p * (p + 1) * (p + 1) : 3 * (size_t)(p + 1) * p * p);
  return nloc * (size_t)n[0] * n[1] * n[2];
}

cudaError_t launch_apply_kform(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                               const double* hpow, const double* u, const double* f, double* out, long long ndof,
                               double* cellbuf, cudaStream_t st, int* nlaunch, const KTimer* kt) {
  const double sign = f ? -1.0 : 1.0;
  if (op.k < 0 || op.k > 2) return cudaErrorInvalidValue;
  if (kt) kt->begin(kt->arg);
  cudaError_t e;
  switch (op.p) {
#define RM_KF(PP) case PP: e = launch_kform_p<PP>(op, alpha, beta, coef_const, hpow, u, f, out, cellbuf, sign, st); break;
    RM_KF(1) RM_KF(2) RM_KF(3) RM_KF(4) RM_KF(5) RM_KF(6) RM_KF(7) RM_KF(8)
    RM_KF(9) RM_KF(10) RM_KF(11) RM_KF(12) RM_KF(13) RM_KF(14) RM_KF(15)
#undef RM_KF
    default: e = cudaErrorInvalidValue;
  }
  if (kt) kt->end(kt->arg);
  if (e != cudaSuccess) return e;
  const int p = op.p;
  const int nloc = op.k == 0 ? (p + 1) * (p + 1) * (p + 1) : (op.k == 1 ? 3 * p * (p + 1) * (p + 1) : 3 * (p + 1) * p * p);
  kform_gather_rows_kernel<<<148 * 16, 256, 0, st>>>(op, cellbuf, f, out, sign, nloc, op.k == 0 ? op.ldx_out : 0);
  (void)ndof;
  if (nlaunch) *nlaunch = 2;
  return cudaGetLastError();
}

}  // namespace rm
