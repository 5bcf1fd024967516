// Matrix-free H(grad) operator on TRILINEAR cells:
//   [A_K u]_i = sum_q w_q |det J| ( beta psi_i u_h + alpha (J^{-T} grad psi_i) . (J^{-T} grad u_h) )
// with the FDM basis psi (tensor products of s-hat_j), the trilinear map F_K of the
// cell's 8 vertices and n_q = ceil(3(p+1)/2) GLL points per direction (reading G1).
// Sum factorisation, one CTA per cell, pipelined over the n_q quadrature planes in z:
//   forward   u (p+1)^3 -> per plane zq: (S_z u, D_z u) -> y stage -> x stage: u_q, grad-hat u_q
//   pointwise t = beta w |J| u_q,  h = alpha w |J| (J^T J)^{-1} grad-hat u_q   (geometry recomputed
//             from the vertices at every point: no stored geometric factors)
//   backward  x stage -> y stage -> z stage accumulated into the thread's registers
// Thread t = (y, x) owns the coefficient line u[.][y][x] and the output line out[.][y][x] in
// registers; the 1D tables are read as shared-memory broadcasts or conflict-free rows.  FP64
// bound (~6 MFLOP per cell at p = 15).  Cells of one parity colour share no DoF, so the output is
// a plain read-modify-write (8 colour launches, deterministic), like the Cartesian apply.
#include "kernels.cuh"

namespace rm {

namespace {

constexpr int TRI_THREADS = 256;
constexpr int MP1 = RM_MAXP1;   // 16
constexpr int MQ = 24;          // n_q for p = 15
constexpr size_t TRI_SMEM =
    sizeof(double) * (4 * MQ * MP1 + 2 * MQ + 24 + 2 * MP1 * MP1 + 3 * MQ * MP1 + 4 * MQ * MQ + 3 * MQ * MP1);

__device__ __forceinline__ bool tri_cons(long long idx, long long last, unsigned gamma_d, int d) {
  if (idx == 0 && (gamma_d & (1u << (2 * d)))) return true;
  if (idx == last && (gamma_d & (1u << (2 * d + 1)))) return true;
  return false;
}

}  // namespace

__global__ void __launch_bounds__(TRI_THREADS, 1) apply_tri_kernel(const __grid_constant__ TriParams tp,
                                                                    const double* __restrict__ tabs,
                                                                    const double* __restrict__ X,
                                                                    const double* __restrict__ alpha,
                                                                    const double* __restrict__ beta, int coef_const,
                                                                    const double* __restrict__ u,
                                                                    double* __restrict__ out, double sign, int px,
                                                                    int py, int pz) {
  const int P1 = tp.p + 1, NQ = tp.nq, p = tp.p;
  extern __shared__ double tsm[];
  double* S = tsm;                 // [q][j]
  double* D = S + MQ * MP1;
  double* St = D + MQ * MP1;       // [j][q]
  double* Dt = St + MP1 * MQ;
  double* xq = Dt + MP1 * MQ;
  double* wq = xq + MQ;
  double* vx = wq + MQ;            // 8 vertices x 3
  double* Az = vx + 24;
  double* Bz = Az + MP1 * MP1;
  double* AS = Bz + MP1 * MP1;
  double* AD = AS + MQ * MP1;
  double* BS = AD + MQ * MP1;
  double* T = BS + MQ * MP1;
  double* HX = T + MQ * MQ;
  double* HY = HX + MQ * MQ;
  double* HZ = HY + MQ * MQ;
  double* P1s = HZ + MQ * MQ;
  double* P2s = P1s + MQ * MP1;
  double* P3s = P2s + MQ * MP1;
  const int t = threadIdx.x;
  for (int i = t; i < NQ * P1; i += TRI_THREADS) {
    const int q = i / P1, j = i % P1;
    S[i] = tabs[i];
    D[i] = tabs[NQ * P1 + i];
    St[j * NQ + q] = S[i];
    Dt[j * NQ + q] = D[i];
  }
  if (t < NQ) { xq[t] = tabs[2 * NQ * P1 + t]; wq[t] = tabs[2 * NQ * P1 + NQ + t]; }
  // the cell of this CTA (colour (px, py, pz))
  const int ncx = (tp.n[0] - px + 1) / 2, ncy = (tp.n[1] - py + 1) / 2;
  const long long cw = blockIdx.x;
  const int cx = px + 2 * (int)(cw % ncx), cy = py + 2 * (int)((cw / ncx) % ncy), cz = pz + 2 * (int)(cw / ((long long)ncx * ncy));
  if (t < 24) {   // vertex (az, ay, ax), coordinate i
    const int a = t / 3, i = t % 3;
    const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
    vx[t] = X[(((long long)(cz + az) * (tp.n[1] + 1) + (cy + ay)) * (tp.n[0] + 1) + (cx + ax)) * 3 + i];
  }
  const long long cell = ((long long)cz * tp.n[1] + cy) * tp.n[0] + cx;
  const double al = coef_const ? alpha[0] : alpha[cell];
  const double be = coef_const ? beta[0] : beta[cell];
  const long long lastx = (long long)tp.n[0] * p, lasty = (long long)tp.n[1] * p, lastz = (long long)tp.n[2] * p;
  // coefficient line of thread t = (y, x): u[z][y][x], z = 0..p (constrained entries read as 0)
  const bool line = t < P1 * P1;
  const int ly = t / P1, lx = t % P1;
  const long long gx = (long long)cx * p + lx, gy = (long long)cy * p + ly;
  const bool conxy = line && (tri_cons(gx, lastx, tp.gamma_d, 0) || tri_cons(gy, lasty, tp.gamma_d, 1));
  double ureg[MP1], oreg[MP1];
#pragma unroll
  for (int z = 0; z < MP1; ++z) {
    ureg[z] = 0.0;
    oreg[z] = 0.0;
    if (line && z < P1 && !conxy) {
      const long long gz = (long long)cz * p + z;
      if (!tri_cons(gz, lastz, tp.gamma_d, 2)) ureg[z] = __ldg(u + (gz * tp.Ly + gy) * tp.Lx + gx);
    }
  }
  __syncthreads();
  for (int zq = 0; zq < NQ; ++zq) {
    // ---- forward z: Az = S_z u, Bz = D_z u on this plane (registers x broadcast table rows)
    if (line) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int z = 0; z < MP1; ++z)
        if (z < P1) { a = fma(S[zq * P1 + z], ureg[z], a); b = fma(D[zq * P1 + z], ureg[z], b); }
      Az[t] = a;
      Bz[t] = b;
    }
    __syncthreads();
    // ---- forward y: AS = S_y Az, AD = D_y Az, BS = S_y Bz   (outputs (yq, x))
    for (int o = t; o < NQ * P1; o += TRI_THREADS) {
      const int yq = o / P1, x = o % P1;
      double as = 0.0, ad = 0.0, bs = 0.0;
      for (int y = 0; y < P1; ++y) {
        const double s = S[yq * P1 + y], d = D[yq * P1 + y], az = Az[y * P1 + x];
        as = fma(s, az, as);
        ad = fma(d, az, ad);
        bs = fma(s, Bz[y * P1 + x], bs);
      }
      AS[o] = as;
      AD[o] = ad;
      BS[o] = bs;
    }
    __syncthreads();
    // ---- forward x + pointwise geometry (points (yq, xq))
    const double zt = xq[zq];
    for (int o = t; o < NQ * NQ; o += TRI_THREADS) {
      const int yq = o / NQ, xqi = o % NQ;
      double uq = 0.0, g0 = 0.0, g1 = 0.0, g2 = 0.0;
      for (int x = 0; x < P1; ++x) {
        const double s = St[x * NQ + xqi], d = Dt[x * NQ + xqi];
        const double as = AS[yq * P1 + x];
        uq = fma(s, as, uq);
        g0 = fma(d, as, g0);
        g1 = fma(s, AD[yq * P1 + x], g1);
        g2 = fma(s, BS[yq * P1 + x], g2);
      }
      // trilinear Jacobian J[i][d] = d x_i / d xhat_d at (xhat, yhat, zhat)
      const double xt = xq[xqi], yt = xq[yq];
      const double ph[3][2] = {{0.5 * (1 - xt), 0.5 * (1 + xt)}, {0.5 * (1 - yt), 0.5 * (1 + yt)}, {0.5 * (1 - zt), 0.5 * (1 + zt)}};
      double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
        const double dx = (ax ? 0.5 : -0.5) * ph[1][ay] * ph[2][az];
        const double dy = ph[0][ax] * (ay ? 0.5 : -0.5) * ph[2][az];
        const double dz = ph[0][ax] * ph[1][ay] * (az ? 0.5 : -0.5);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const double xa = vx[a * 3 + i];
          J[i][0] = fma(xa, dx, J[i][0]);
          J[i][1] = fma(xa, dy, J[i][1]);
          J[i][2] = fma(xa, dz, J[i][2]);
        }
      }
      // cofactors: J^{-1} = adj(J) / det J;  C = J^{-1} J^{-T} = adj adj^T / det^2
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], c01 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                   c02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
      const double c10 = J[1][2] * J[2][0] - J[1][0] * J[2][2], c11 = J[0][0] * J[2][2] - J[0][2] * J[2][0],
                   c12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
      const double c20 = J[1][0] * J[2][1] - J[1][1] * J[2][0], c21 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                   c22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      const double det = J[0][0] * c00 + J[0][1] * c10 + J[0][2] * c20;   // adj rows: inv = [c..] / det
      const double w = wq[xqi] * wq[yq] * wq[zq];
      const double wd = w * fabs(det);
      // K = alpha w |det| (adj adj^T) / det^2, adj = [[c00 c01 c02], [c10 c11 c12], [c20 c21 c22]]
      const double k = al * wd / (det * det);
      const double K00 = k * (c00 * c00 + c01 * c01 + c02 * c02), K01 = k * (c00 * c10 + c01 * c11 + c02 * c12),
                   K02 = k * (c00 * c20 + c01 * c21 + c02 * c22), K11 = k * (c10 * c10 + c11 * c11 + c12 * c12),
                   K12 = k * (c10 * c20 + c11 * c21 + c12 * c22), K22 = k * (c20 * c20 + c21 * c21 + c22 * c22);
      T[o] = be * wd * uq;
      HX[o] = K00 * g0 + K01 * g1 + K02 * g2;
      HY[o] = K01 * g0 + K11 * g1 + K12 * g2;
      HZ[o] = K02 * g0 + K12 * g1 + K22 * g2;
    }
    __syncthreads();
    // ---- backward x: P1 = S_x^T T + D_x^T HX, P2 = S_x^T HY, P3 = S_x^T HZ   (outputs (yq, x))
    for (int o = t; o < NQ * P1; o += TRI_THREADS) {
      const int yq = o / P1, x = o % P1;
      double a1 = 0.0, a2 = 0.0, a3 = 0.0;
      for (int q = 0; q < NQ; ++q) {
        const double s = S[q * P1 + x], d = D[q * P1 + x];
        const int pt = yq * NQ + q;
        a1 = fma(s, T[pt], fma(d, HX[pt], a1));
        a2 = fma(s, HY[pt], a2);
        a3 = fma(s, HZ[pt], a3);
      }
      P1s[o] = a1;
      P2s[o] = a2;
      P3s[o] = a3;
    }
    __syncthreads();
    // ---- backward y (thread (y, x)): Q1 = S_y^T P1 + D_y^T P2, Q2 = S_y^T P3; backward z into registers
    if (line) {
      double q1 = 0.0, q2 = 0.0;
      for (int q = 0; q < NQ; ++q) {
        const double s = S[q * P1 + ly], d = D[q * P1 + ly];
        q1 = fma(s, P1s[q * P1 + lx], fma(d, P2s[q * P1 + lx], q1));
        q2 = fma(s, P3s[q * P1 + lx], q2);
      }
#pragma unroll
      for (int z = 0; z < MP1; ++z)
        if (z < P1) oreg[z] = fma(S[zq * P1 + z], q1, fma(D[zq * P1 + z], q2, oreg[z]));
    }
    __syncthreads();
  }
  if (line && !conxy) {
#pragma unroll
    for (int z = 0; z < MP1; ++z) {
      if (z >= P1) continue;
      const long long gz = (long long)cz * p + z;
      if (tri_cons(gz, lastz, tp.gamma_d, 2)) continue;
      out[(gz * tp.Ly + gy) * tp.Lx + gx] += sign * oreg[z];
    }
  }
}

cudaError_t launch_apply_trilinear(const TriParams& tp, const double* tabs, const double* X, const double* alpha,
                                   const double* beta, int coef_const, const double* u, double* out, double sign,
                                   cudaStream_t st, int* nlaunch) {
  int nl = 0;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(apply_tri_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRI_SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  for (int pz = 0; pz < 2; ++pz)
    for (int py = 0; py < 2; ++py)
      for (int px = 0; px < 2; ++px) {
        const long long ncell = (long long)((tp.n[0] - px + 1) / 2) * ((tp.n[1] - py + 1) / 2) * ((tp.n[2] - pz + 1) / 2);
        if (ncell <= 0) continue;
        apply_tri_kernel<<<(unsigned)ncell, TRI_THREADS, TRI_SMEM, st>>>(tp, tabs, X, alpha, beta, coef_const, u, out, sign, px,
                                                                  py, pz);
        ++nl;
      }
  if (nlaunch) *nlaunch += nl;
  return cudaGetLastError();
}

}  // namespace rm
