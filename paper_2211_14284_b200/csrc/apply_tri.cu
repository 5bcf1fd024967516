// Matrix-free H(grad) operator on TRILINEAR cells:
//   [A_K u]_i = sum_q w_q |det J| ( beta psi_i u_h + alpha (J^{-T} grad psi_i) . (J^{-T} grad u_h) )
// with the FDM basis psi (tensor products of s-hat_j), the trilinear map F_K of the
// cell's 8 vertices and n_q = ceil(3(p+1)/2) GLL points per direction (reading G1).
//
// Sum factorisation, one CTA per cell, the n_q quadrature planes in z processed in batches of
// ZB = 4.  The y and x contractions are small dense GEMMs (24 x 16 x 16 per plane and field) and
// run on the FP64 tensor cores (mma.sync m8n8k4 f64, SASS DMMA): the 1D tables S, D are held in
// registers as fragments, the data operands come from shared memory in conflict-free layouts.
//   forward   z (per thread line, DFMA): Az = S_z u, Bz = D_z u
//             y (DMMA): AS = S_y Az, AD = D_y Az, BS = S_y Bz
//             x (DMMA): u_q = S_x AS, g = (D_x AS, S_x AD, S_x BS)
//   pointwise on the accumulator fragments: t = beta w |J| u_q,
//             h = alpha w |J|^{-1} adj(J) adj(J)^T g   (geometry from the trilinear coefficients)
//   backward  x (DMMA): P1 = S_x^T t + D_x^T h_x, P2 = S_x^T h_y, P3 = S_x^T h_z
//             y (DMMA): Q1 = S_y^T P1 + D_y^T P2, Q2 = S_y^T P3
//             z (per thread line, DFMA): out += S_z^T Q1 + D_z^T Q2
// Tables are zero-padded to 16 coefficients x 24 points, so every p <= 15 uses the same kernel
// (padded rows contribute exact zeros).  Each CTA writes its cell's local result to a cell
// buffer; tri_gather_kernel then sums, per DoF and in a fixed order, the <= 8 cell
// contributions: no colouring, one launch over all cells, bitwise deterministic.
#include "kernels.cuh"

namespace rm {

namespace {

constexpr int TRI_THREADS = 256;
constexpr int K1 = 16;    // coefficients per direction (padded)
constexpr int NQP = 24;   // quadrature points per direction (padded)
constexpr int ZB = 4;     // z planes per batch
// shared memory (doubles)
constexpr int XS_AZ = 20, SZ_AZ = K1 * XS_AZ;      // Az/Bz plane, [x][y] (y contiguous)
constexpr int XS_Q = 17, SZ_Q = K1 * XS_Q;         // Q1/Q2 plane, [x][y]
constexpr int XS_AS = 20, SZ_AS = NQP * XS_AS;     // AS/AD/BS plane, [yq][x]
constexpr int XS_TH = 28, SZ_TH = NQP * XS_TH;     // T/HX/HY/HZ plane, [yq][xq]
constexpr int XS_P = 28, SZ_P = K1 * XS_P;         // P1/P2/P3 plane, [x][yq]
constexpr int O_SG = 0, O_DG = O_SG + NQP * K1, O_XQ = O_DG + NQP * K1, O_WQ = O_XQ + NQP, O_GC = O_WQ + NQP,
              O_U = O_GC + 24, O_OUT = O_U + K1 * K1 * K1, O_R1 = O_OUT + K1 * K1 * K1;
constexpr int R1_SIZE = ZB * 4 * SZ_TH;   // T/H (largest); Az/Bz at [0, 2560), Q at [2560, 4736)
constexpr int O_Q = ZB * 2 * SZ_AZ;
constexpr int O_R2 = O_R1 + R1_SIZE;
constexpr int R2_SIZE = ZB * 3 * SZ_AS;   // AS (largest); P aliases it
constexpr size_t TRI_SMEM = sizeof(double) * (O_R2 + R2_SIZE);
static_assert(O_Q + ZB * 2 * SZ_Q <= R1_SIZE, "R1 layout");
static_assert(ZB * 3 * SZ_P <= R2_SIZE, "R2 layout");
static_assert(TRI_SMEM <= 227 * 1024, "shared memory");

__device__ __forceinline__ bool tri_cons(long long idx, long long last, unsigned gamma_d, int d) {
  if (idx == 0 && (gamma_d & (1u << (2 * d)))) return true;
  if (idx == last && (gamma_d & (1u << (2 * d + 1)))) return true;
  return false;
}

// D(8x8) += A(8x4, row) B(4x8, col); lane l: a = A[l/4][l%4], b = B[l%4][l/4],
// c0/c1 = C[l/4][2(l%4) + 0/1]
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double pick2(const double a0, const double a1, int i) { return i ? a1 : a0; }
__device__ __forceinline__ double pick3(const double a0, const double a1, const double a2, int i) {
  return i == 0 ? a0 : (i == 1 ? a1 : a2);
}

}  // namespace

__global__ void __launch_bounds__(TRI_THREADS, 1) apply_tri_kernel(const __grid_constant__ TriParams tp,
                                                                    const double* __restrict__ tabs,
                                                                    const double* __restrict__ X,
                                                                    const double* __restrict__ alpha,
                                                                    const double* __restrict__ beta, int coef_const,
                                                                    const double* __restrict__ u,
                                                                    double* __restrict__ cellbuf) {
  extern __shared__ __align__(16) double sm[];
  const int P1 = tp.p + 1, NQ = tp.nq, p = tp.p;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int l4 = lane >> 2, lm = lane & 3;
  double* SG = sm + O_SG;   // [q][j], zero padded
  double* DG = sm + O_DG;
  double* XQ = sm + O_XQ;
  double* WQ = sm + O_WQ;
  double* GC = sm + O_GC;   // trilinear coefficients [monomial][coord]
  double* U = sm + O_U;     // [z][y][x]
  double* OUT = sm + O_OUT; // [z][y][x], the cell's result (each thread owns its (y, x) line)
  double* R1 = sm + O_R1;
  double* R2 = sm + O_R2;
  for (int i = t; i < NQP * K1; i += TRI_THREADS) {
    const int q = i / K1, j = i % K1;
    const bool in = q < NQ && j < P1;
    SG[i] = in ? tabs[q * P1 + j] : 0.0;
    DG[i] = in ? tabs[NQ * P1 + q * P1 + j] : 0.0;
  }
  if (t < NQP) {
    XQ[t] = t < NQ ? tabs[2 * NQ * P1 + t] : 0.0;
    WQ[t] = t < NQ ? tabs[2 * NQ * P1 + NQ + t] : 0.0;
  }
  const long long cell = blockIdx.x;
  const int cx = (int)(cell % tp.n[0]), cy = (int)((cell / tp.n[0]) % tp.n[1]), cz = (int)(cell / ((long long)tp.n[0] * tp.n[1]));
  if (t < 24) {
    // x(xi, eta, zeta) = sum_a X_a prod_d (1 + s_ad xi_d) / 2 = sum_m GC[m] mono_m,
    // monomials m: 1, xi, eta, zeta, xi eta, xi zeta, eta zeta, xi eta zeta
    const int m = t / 3, i = t % 3;
    const int ex = (m == 1 || m == 4 || m == 5 || m == 7), ey = (m == 2 || m == 4 || m == 6 || m == 7),
              ez = (m == 3 || m == 5 || m == 6 || m == 7);
    double s = 0.0;
    for (int a = 0; a < 8; ++a) {
      const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
      const double xa = X[(((long long)(cz + az) * (tp.n[1] + 1) + (cy + ay)) * (tp.n[0] + 1) + (cx + ax)) * 3 + i];
      const double sg = ((ex && !ax) ? -1.0 : 1.0) * ((ey && !ay) ? -1.0 : 1.0) * ((ez && !az) ? -1.0 : 1.0);
      s += sg * xa;
    }
    GC[m * 3 + i] = 0.125 * s;
  }
  const double al = coef_const ? alpha[0] : alpha[cell];
  const double be = coef_const ? beta[0] : beta[cell];
  const long long lastx = (long long)tp.n[0] * p, lasty = (long long)tp.n[1] * p, lastz = (long long)tp.n[2] * p;
  // coefficients of the cell (constrained entries read as zero), [z][y][x]
  for (int i = t; i < K1 * K1 * K1; i += TRI_THREADS) {
    const int z = i >> 8, y = (i >> 4) & 15, x = i & 15;
    double v = 0.0;
    if (x < P1 && y < P1 && z < P1) {
      const long long gx = (long long)cx * p + x, gy = (long long)cy * p + y, gz = (long long)cz * p + z;
      if (!tri_cons(gx, lastx, tp.gamma_d, 0) && !tri_cons(gy, lasty, tp.gamma_d, 1) && !tri_cons(gz, lastz, tp.gamma_d, 2))
        v = __ldg(u + (gz * tp.Ly + gy) * tp.Lx + gx);
    }
    U[i] = v;
    OUT[i] = 0.0;
  }
  __syncthreads();
  // table fragments: fa[m][k] = T[8m + l/4][4k + l%4] (A pattern), ft[k][n] = T[4k + l%4][8n + l/4]
  double faS[3][4], faD[3][4], ftS[6][2], ftD[6][2];
#pragma unroll
  for (int m = 0; m < 3; ++m)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      faS[m][k] = SG[(8 * m + l4) * K1 + 4 * k + lm];
      faD[m][k] = DG[(8 * m + l4) * K1 + 4 * k + lm];
    }
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      ftS[k][n] = SG[(4 * k + lm) * K1 + 8 * n + l4];
      ftD[k][n] = DG[(4 * k + lm) * K1 + 8 * n + l4];
    }
  const int lx = t & 15, ly = t >> 4;   // per-thread line (y, x)
  const int nb = (NQ + ZB - 1) / ZB;

  auto forward_z = [&](int b) {   // Az/Bz of the batch's planes, stored [x][y]
    double a[ZB], c[ZB];
#pragma unroll
    for (int pl = 0; pl < ZB; ++pl) a[pl] = c[pl] = 0.0;
#pragma unroll
    for (int z = 0; z < K1; ++z) {
      const double uz = U[z * 256 + t];
#pragma unroll
      for (int pl = 0; pl < ZB; ++pl) {
        const int zq = b * ZB + pl;
        a[pl] = fma(SG[zq * K1 + z], uz, a[pl]);
        c[pl] = fma(DG[zq * K1 + z], uz, c[pl]);
      }
    }
#pragma unroll
    for (int pl = 0; pl < ZB; ++pl) {
      R1[(pl * 2 + 0) * SZ_AZ + lx * XS_AZ + ly] = a[pl];
      R1[(pl * 2 + 1) * SZ_AZ + lx * XS_AZ + ly] = c[pl];
    }
  };
  auto backward_z = [&](int b) {
    double q1[ZB], q2[ZB];
#pragma unroll
    for (int pl = 0; pl < ZB; ++pl) {
      q1[pl] = R1[O_Q + (pl * 2 + 0) * SZ_Q + lx * XS_Q + ly];
      q2[pl] = R1[O_Q + (pl * 2 + 1) * SZ_Q + lx * XS_Q + ly];
    }
#pragma unroll 4
    for (int z = 0; z < K1; ++z) {
      double o = OUT[z * 256 + t];
#pragma unroll
      for (int pl = 0; pl < ZB; ++pl) {
        const int zq = b * ZB + pl;
        o = fma(SG[zq * K1 + z], q1[pl], fma(DG[zq * K1 + z], q2[pl], o));
      }
      OUT[z * 256 + t] = o;
    }
  };

  forward_z(0);
  __syncthreads();
  for (int b = 0; b < nb; ++b) {
    // ---- forward y: warp w -> plane w/2, x tile w%2; all three yq tiles, fields AS, AD, BS
    {
      const int pl = w >> 1, nt = w & 1;
      double cS[3][2] = {}, cD[3][2] = {}, cB[3][2] = {};
      const double* az = R1 + (pl * 2 + 0) * SZ_AZ + (8 * nt + l4) * XS_AZ + lm;
      const double* bz = R1 + (pl * 2 + 1) * SZ_AZ + (8 * nt + l4) * XS_AZ + lm;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double ba = az[4 * k], bb = bz[4 * k];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
          dmma(cS[m], faS[m][k], ba);
          dmma(cD[m], faD[m][k], ba);
          dmma(cB[m], faS[m][k], bb);
        }
      }
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int o = (8 * m + l4) * XS_AS + 8 * nt + 2 * lm;
        *reinterpret_cast<double2*>(R2 + (pl * 3 + 0) * SZ_AS + o) = make_double2(cS[m][0], cS[m][1]);
        *reinterpret_cast<double2*>(R2 + (pl * 3 + 1) * SZ_AS + o) = make_double2(cD[m][0], cD[m][1]);
        *reinterpret_cast<double2*>(R2 + (pl * 3 + 2) * SZ_AS + o) = make_double2(cB[m][0], cB[m][1]);
      }
    }
    __syncthreads();
    // ---- forward x + pointwise: 36 (plane, yq tile, xq tile) jobs over 8 warps
    for (int j = w; j < ZB * 9; j += 8) {
      const int pl = j / 9, mt = (j % 9) / 3, nt = j % 3;
      const int zq = b * ZB + pl;
      double cu[2] = {}, c0[2] = {}, c1[2] = {}, c2[2] = {};
      const double* as = R2 + (pl * 3 + 0) * SZ_AS + (8 * mt + l4) * XS_AS + lm;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double aS = as[4 * k], aD = as[SZ_AS + 4 * k], aB = as[2 * SZ_AS + 4 * k];
        const double bS = pick3(faS[0][k], faS[1][k], faS[2][k], nt), bD = pick3(faD[0][k], faD[1][k], faD[2][k], nt);
        dmma(cu, aS, bS);
        dmma(c0, aS, bD);
        dmma(c1, aD, bS);
        dmma(c2, aB, bS);
      }
      // pointwise at (zq, yq, xq + i), i = 0, 1
      const int yq = 8 * mt + l4, xq0 = 8 * nt + 2 * lm;
      const double ze = XQ[zq], et = XQ[yq];
      const double wzy = WQ[zq] * WQ[yq];
      double Jx[3], Jya[3], Jyb[3], Jza[3], Jzb[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double g1 = GC[3 + i], g2 = GC[6 + i], g3 = GC[9 + i], g4 = GC[12 + i], g5 = GC[15 + i], g6 = GC[18 + i],
                     g7 = GC[21 + i];
        Jx[i] = fma(fma(g7, ze, g4), et, fma(g5, ze, g1));   // d/dxi: const along xi
        Jya[i] = fma(g6, ze, g2);                             // d/deta = Jya + Jyb xi
        Jyb[i] = fma(g7, ze, g4);
        Jza[i] = fma(g6, et, g3);                             // d/dzeta = Jza + Jzb xi
        Jzb[i] = fma(g7, et, g5);
      }
      double tv[2], hx[2], hy[2], hz[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int xq = xq0 + e;
        const double xi = XQ[xq];
        double J[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          J[i][0] = Jx[i];
          J[i][1] = fma(Jyb[i], xi, Jya[i]);
          J[i][2] = fma(Jzb[i], xi, Jza[i]);
        }
        // adj(J): J^{-1} = adj / det
        const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], c01 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                     c02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
        const double c10 = J[1][2] * J[2][0] - J[1][0] * J[2][2], c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0],
                     c12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
        const double c20 = J[1][0] * J[2][1] - J[1][1] * J[2][0], c21 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                     c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        const double det = J[0][0] * c00 + J[0][1] * c10 + J[0][2] * c20;
        const double wgt = wzy * WQ[xq];
        const double ad = fabs(det);
        const double k = al * wgt * __drcp_rn(ad);
        const double g0 = c0[e], g1 = c1[e], g2 = c2[e];
        // h = k adj adj^T g: v = adj^T g (columns of adj dotted with g), h = k adj v
        const double v0 = c00 * g0 + c10 * g1 + c20 * g2, v1 = c01 * g0 + c11 * g1 + c21 * g2,
                     v2 = c02 * g0 + c12 * g1 + c22 * g2;
        hx[e] = k * (c00 * v0 + c01 * v1 + c02 * v2);
        hy[e] = k * (c10 * v0 + c11 * v1 + c12 * v2);
        hz[e] = k * (c20 * v0 + c21 * v1 + c22 * v2);
        tv[e] = be * wgt * ad * cu[e];
      }
      const int o = yq * XS_TH + xq0;
      *reinterpret_cast<double2*>(R1 + (pl * 4 + 0) * SZ_TH + o) = make_double2(tv[0], tv[1]);
      *reinterpret_cast<double2*>(R1 + (pl * 4 + 1) * SZ_TH + o) = make_double2(hx[0], hx[1]);
      *reinterpret_cast<double2*>(R1 + (pl * 4 + 2) * SZ_TH + o) = make_double2(hy[0], hy[1]);
      *reinterpret_cast<double2*>(R1 + (pl * 4 + 3) * SZ_TH + o) = make_double2(hz[0], hz[1]);
    }
    __syncthreads();
    // ---- backward x: 24 (plane, yq tile, x tile) jobs; P stored [x][yq]
#pragma unroll 1
    for (int j = w; j < ZB * 6; j += 8) {
      const int pl = j / 6, mt = (j % 6) >> 1, nt = j & 1;
      double p1[2] = {}, p2[2] = {}, p3[2] = {};
      const double* th = R1 + (pl * 4) * SZ_TH + (8 * mt + l4) * XS_TH + lm;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double aT = th[4 * k], aX = th[SZ_TH + 4 * k], aY = th[2 * SZ_TH + 4 * k], aZ = th[3 * SZ_TH + 4 * k];
        const double bS = pick2(ftS[k][0], ftS[k][1], nt), bD = pick2(ftD[k][0], ftD[k][1], nt);
        dmma(p1, aT, bS);
        dmma(p1, aX, bD);
        dmma(p2, aY, bS);
        dmma(p3, aZ, bS);
      }
      const int yq = 8 * mt + l4, x0 = 8 * nt + 2 * lm;
      double* P = R2 + (pl * 3) * SZ_P + yq;
      P[x0 * XS_P] = p1[0];
      P[(x0 + 1) * XS_P] = p1[1];
      P[SZ_P + x0 * XS_P] = p2[0];
      P[SZ_P + (x0 + 1) * XS_P] = p2[1];
      P[2 * SZ_P + x0 * XS_P] = p3[0];
      P[2 * SZ_P + (x0 + 1) * XS_P] = p3[1];
    }
    __syncthreads();
    // ---- backward y: 16 (plane, y tile, x tile) jobs; Q stored [x][y]
#pragma unroll 1
    for (int j = w; j < ZB * 4; j += 8) {
      const int pl = j >> 2, mt = (j >> 1) & 1, nt = j & 1;
      double q1[2] = {}, q2[2] = {};
      const double* P = R2 + (pl * 3) * SZ_P + (8 * nt + l4) * XS_P + lm;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double b1 = P[4 * k], b2 = P[SZ_P + 4 * k], b3 = P[2 * SZ_P + 4 * k];
        const double aS = pick2(ftS[k][0], ftS[k][1], mt), aD = pick2(ftD[k][0], ftD[k][1], mt);
        dmma(q1, aS, b1);
        dmma(q1, aD, b2);
        dmma(q2, aS, b3);
      }
      const int y = 8 * mt + l4, x0 = 8 * nt + 2 * lm;
      double* Q = R1 + O_Q + (pl * 2) * SZ_Q + y;
      Q[x0 * XS_Q] = q1[0];
      Q[(x0 + 1) * XS_Q] = q1[1];
      Q[SZ_Q + x0 * XS_Q] = q2[0];
      Q[SZ_Q + (x0 + 1) * XS_Q] = q2[1];
    }
    __syncthreads();
    // ---- backward z of this batch, forward z of the next (disjoint parts of R1)
    backward_z(b);
    if (b + 1 < nb) forward_z(b + 1);
    __syncthreads();
  }
  // local result of the cell, [z][y][x] with stride P1
  if (lx < P1 && ly < P1) {
    double* o = cellbuf + cell * P1 * P1 * P1 + ly * P1 + lx;
    for (int z = 0; z < P1; ++z) o[z * P1 * P1] = OUT[z * 256 + t];
  }
}

// out[g] = f[g] (or 0) + sign * sum over the cells containing g of their local result;
// constrained entries 0.  Fixed summation order (cells ascending in z, y, x): deterministic.
__global__ void tri_gather_kernel(const __grid_constant__ TriParams tp, const double* __restrict__ cellbuf,
                                  const double* __restrict__ f, double* __restrict__ out, double sign) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nd = tp.Lx * tp.Ly * tp.Lz;
  if (g >= nd) return;
  const int p = tp.p, P1 = p + 1;
  const long long gx = g % tp.Lx, gy = (g / tp.Lx) % tp.Ly, gz = g / (tp.Lx * tp.Ly);
  const long long lastx = (long long)tp.n[0] * p, lasty = (long long)tp.n[1] * p, lastz = (long long)tp.n[2] * p;
  if (tri_cons(gx, lastx, tp.gamma_d, 0) || tri_cons(gy, lasty, tp.gamma_d, 1) || tri_cons(gz, lastz, tp.gamma_d, 2)) {
    out[g] = 0.0;
    return;
  }
  int c[3][2], a[3][2], nc[3];
  const long long gg[3] = {gx, gy, gz};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int i = (int)gg[d];
    int cc = i / p;
    if (cc >= tp.n[d]) cc = tp.n[d] - 1;
    const int aa = i - cc * p;
    nc[d] = 0;
    if (aa == 0 && cc > 0) { c[d][nc[d]] = cc - 1; a[d][nc[d]] = p; ++nc[d]; }
    c[d][nc[d]] = cc; a[d][nc[d]] = aa; ++nc[d];
  }
  double s = 0.0;
  for (int kz = 0; kz < nc[2]; ++kz)
    for (int ky = 0; ky < nc[1]; ++ky)
      for (int kx = 0; kx < nc[0]; ++kx) {
        const long long cell = ((long long)c[2][kz] * tp.n[1] + c[1][ky]) * tp.n[0] + c[0][kx];
        s += cellbuf[cell * P1 * P1 * P1 + (a[2][kz] * P1 + a[1][ky]) * P1 + a[0][kx]];
      }
  out[g] = (f ? f[g] : 0.0) + sign * s;
}

cudaError_t launch_apply_trilinear(const TriParams& tp, const double* tabs, const double* X, const double* alpha,
                                   const double* beta, int coef_const, const double* u, const double* f, double* out,
                                   double sign, double* cellbuf, cudaStream_t st, int* nlaunch) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(apply_tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRI_SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (tp.p + 1 > K1 || tp.nq > NQP) return cudaErrorInvalidValue;
  const long long ncell = (long long)tp.n[0] * tp.n[1] * tp.n[2];
  const long long nd = tp.Lx * tp.Ly * tp.Lz;
  if (ncell <= 0) return cudaSuccess;
  apply_tri_kernel<<<(unsigned)ncell, TRI_THREADS, TRI_SMEM, st>>>(tp, tabs, X, alpha, beta, coef_const, u, cellbuf);
  tri_gather_kernel<<<(unsigned)((nd + 255) / 256), 256, 0, st>>>(tp, cellbuf, f, out, sign);
  if (nlaunch) *nlaunch += 2;
  return cudaGetLastError();
}

size_t tri_cellbuf_doubles(const TriParams& tp) {
  return (size_t)tp.n[0] * tp.n[1] * tp.n[2] * (tp.p + 1) * (tp.p + 1) * (tp.p + 1);
}

}  // namespace rm
