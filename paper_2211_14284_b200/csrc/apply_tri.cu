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
#include <algorithm>

#include "kernels.cuh"

namespace rm {

namespace {

constexpr int TRI_THREADS = 384;   // 12 warps = 4 planes x 3 yq tiles per batch
constexpr int TRI_WARPS = TRI_THREADS / 32;
constexpr int K1 = 16;    // coefficients per direction (padded)
constexpr int NQP = 24;   // quadrature points per direction (padded)
constexpr int ZB = 4;     // z planes per batch
// shared memory (doubles); strides / XOR swizzles chosen for conflict-free fragment access
// (layouts found by an exhaustive search over strides and XOR swizzles: the fragment loads AND
// the fragment stores of every buffer below are bank-conflict free)
constexpr int XS_AS = 16, SZ_ASF = 8 * XS_AS;   // warp rows AS/AD/BS [f][r][x ^ h_as(r)]
constexpr int XS_TH = 24, SZ_THF = 8 * XS_TH;   // warp rows T/HX/HY/HZ [f][r][xq ^ h_th(r)]
constexpr int WR_SIZE = 4 * SZ_THF;             // per-warp region (T/H rows; AS rows alias it)
constexpr int XS_P = 32, SZ_P = K1 * XS_P;      // P1/P2/P3 plane [x][yq ^ h_p(x)]
constexpr int XS_Q = 18, SZ_Q = K1 * XS_Q; // Q1/Q2 plane [x][y] (fragment stores: stride = 2 mod 16)
constexpr int O_SG = 0, O_DG = O_SG + NQP * K1, O_XQ = O_DG + NQP * K1, O_WQ = O_XQ + NQP, O_GC = O_WQ + NQP,
              O_FA = O_GC + 24, O_FT = O_FA + 2 * 3 * 4 * 32, O_U = O_FT + 2 * 6 * 2 * 32, O_OUT = O_U + 4096,
              O_AZ = O_OUT + 4096, O_WR = O_AZ + ZB * 2 * 256, O_P = O_WR + TRI_WARPS * WR_SIZE,
              O_VX = O_P + ZB * 3 * SZ_P, O_FX = O_VX + 28, O_FB = O_FX + 2 * 2 * 2 * 2 * 32,
              O_END = O_FB + 2 * 2 * 3 * 32;
// even / odd x path (TriParams::eo): forward-x B fragments [S/D][E/O][n tile][k][lane] of the 12 x 8
// tables, backward-x B fragments [S/D][E/O][k][lane]; pointwise output rows [8 combos][8][XE]
constexpr int XE = 12;
constexpr size_t TRI_SMEM = sizeof(double) * O_END;
static_assert(ZB * 2 * SZ_Q <= TRI_WARPS * WR_SIZE, "Q aliases the warp regions");
static_assert(TRI_SMEM <= 232448, "shared memory");
static_assert(ZB == 4 && TRI_WARPS == 12, "job tables below assume 4 planes and 12 warps");

// [x][y] planes of 16 x 16 with the y index XOR-swizzled: lanes along y (z stages) and the
// B-fragment pattern (x = 8n + l/4, y = 4k + l%4) are both conflict-free
__device__ __forceinline__ int sw16(int x, int y) { return x * 16 + (y ^ (4 * (x & 3))); }
__device__ __forceinline__ int swu(int x, int y) { return x * 16 + (y ^ x); }   // U / OUT planes
__device__ __forceinline__ int h_as(int r) { return 8 * (r & 1) + 4 * ((r >> 1) & 1); }
__device__ __forceinline__ int h_th(int r) { return 4 * ((r >> 1) & 1); }
__device__ __forceinline__ int h_p(int x) { return (5 * x) & 28; }

__device__ __forceinline__ bool tri_cons(long long idx, long long last, unsigned gamma_d, int d) {
  if (idx == 0 && (gamma_d & (1u << (2 * d)))) return true;
  if (idx == last && (gamma_d & (1u << (2 * d + 1)))) return true;
  return false;
}

// 8-byte global -> shared async copy, zero-filled when !valid (Dirichlet entries, padding)
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// D(8x8) += A(8x4, row) B(4x8, col); lane l: a = A[l/4][l%4], b = B[l%4][l/4],
// c0/c1 = C[l/4][2(l%4) + 0/1]
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

}  // namespace

template <bool EO>
__global__ void __launch_bounds__(TRI_THREADS, 1) apply_tri_kernel(const __grid_constant__ TriParams tp,
                                                                    const double* __restrict__ tabs,
                                                                    const double* __restrict__ X,
                                                                    const double* __restrict__ alpha,
                                                                    const double* __restrict__ beta, int coef_const,
                                                                    const double* __restrict__ u,
                                                                    const double* __restrict__ f,
                                                                    double* __restrict__ out, double sign,
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
  double* FA = sm + O_FA;   // fragments T[8m + l/4][4k + l%4], [S/D][m][k][lane]
  double* FT = sm + O_FT;   // fragments T[4k + l%4][8n + l/4], [S/D][k][n][lane]
  double* U = sm + O_U;     // [z] swu(x, y)
  double* OUT = sm + O_OUT; // [z] swu(x, y): the cell's result
  double* AZ = sm + O_AZ;   // [plane][Az/Bz] sw16(x, y)
  double* WRg = sm + O_WR + w * WR_SIZE;   // this warp's rows
  double* PP = sm + O_P;    // [plane][P1/P2/P3] [x][yq]
  double* QQ = sm + O_WR;   // [plane][Q1/Q2] [x][y] (aliases the warp regions)
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
  double* VX = sm + O_VX;   // prefetched vertices [a][i] (24), alpha, beta of the next cell
  const long long ncell = (long long)tp.n[0] * tp.n[1] * tp.n[2];
  const long long lastx = (long long)tp.n[0] * p, lasty = (long long)tp.n[1] * p, lastz = (long long)tp.n[2] * p;
  // async prefetch of a cell's coefficients (constrained entries zero-filled) into U[z] swu(x, y),
  // its 8 vertices and its coefficients into VX
  auto prefetch = [&](long long c) {
    const int cx = (int)(c % tp.n[0]), cy = (int)((c / tp.n[0]) % tp.n[1]), cz = (int)(c / ((long long)tp.n[0] * tp.n[1]));
    for (int i = t; i < K1 * K1 * K1; i += TRI_THREADS) {
      const int z = i >> 8, y = (i >> 4) & 15, x = i & 15;
      const long long gx = (long long)cx * p + x, gy = (long long)cy * p + y, gz = (long long)cz * p + z;
      const bool ok = x < P1 && y < P1 && z < P1 && !tri_cons(gx, lastx, tp.gamma_d, 0) &&
                      !tri_cons(gy, lasty, tp.gamma_d, 1) && !tri_cons(gz, lastz, tp.gamma_d, 2);
      cp_async8(U + z * 256 + swu(x, y), ok ? u + (gz * tp.Ly + gy) * tp.Lx + gx : u, ok);
    }
    if (t < 24) {
      const int a = t / 3, i = t % 3, ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
      cp_async8(VX + t, X + (((long long)(cz + az) * (tp.n[1] + 1) + (cy + ay)) * (tp.n[0] + 1) + (cx + ax)) * 3 + i, true);
    } else if (t == 24) {
      cp_async8(VX + 24, coef_const ? alpha : alpha + c, true);
    } else if (t == 25) {
      cp_async8(VX + 25, coef_const ? beta : beta + c, true);
    }
    cp_async_commit();
  };
  for (int i = t; i < 4096; i += TRI_THREADS) OUT[i] = 0.0;
  if ((long long)blockIdx.x < ncell) prefetch(blockIdx.x);
  __syncthreads();
  for (int i = t; i < 2 * 3 * 4 * 32; i += TRI_THREADS) {
    const int f = i / 384, m = (i / 128) % 3, k = (i / 32) & 3, l = i & 31;
    FA[i] = (f ? DG : SG)[(8 * m + (l >> 2)) * K1 + 4 * k + (l & 3)];
  }
  for (int i = t; i < 2 * 6 * 2 * 32; i += TRI_THREADS) {
    const int f = i / 384, k = (i / 64) % 6, n = (i / 32) & 1, l = i & 31;
    FT[i] = (f ? DG : SG)[(4 * k + (l & 3)) * K1 + 8 * n + (l >> 2)];
  }
  auto fa = [&](int f, int m, int k) { return FA[((f * 3 + m) * 4 + k) * 32 + lane]; };
  auto ft = [&](int f, int k, int n) { return FT[((f * 6 + k) * 2 + n) * 32 + lane]; };
  double* FX = sm + O_FX;
  double* FB = sm + O_FB;
  if (EO) {
    const double* T4 = tabs + 2 * NQ * P1 + 2 * NQ;   // S_E, S_O, D_E, D_O [r][e], 12 x 8 each
    for (int i = t; i < 2 * 2 * 2 * 2 * 32; i += TRI_THREADS) {   // forward x: B[e = 4k + l%4][r = 8nt + l/4]
      const int f = i >> 8, eo = (i >> 7) & 1, nt = (i >> 6) & 1, k = (i >> 5) & 1, l = i & 31;
      const int r = 8 * nt + (l >> 2), e = 4 * k + (l & 3);
      FX[i] = r < tp.ne ? T4[(2 * f + eo) * 96 + r * 8 + e] : 0.0;
    }
    for (int i = t; i < 2 * 2 * 3 * 32; i += TRI_THREADS) {       // backward x: B[r = 4k + l%4][e = l/4]
      const int f = i / 192, eo = (i / 96) & 1, k = (i >> 5) % 3, l = i & 31;
      const int r = 4 * k + (l & 3), e = l >> 2;
      FB[i] = r < tp.ne ? T4[(2 * f + eo) * 96 + r * 8 + e] : 0.0;
    }
  }
  __shared__ int XPOS[16];   // EO: even / odd position of each interior x index
  if (EO && t < 16) {
    int q = 0;
    for (int pos = 1; pos < 16; ++pos)
      if (pos != 8 && tp.xsig[pos] == t) q = pos;
    XPOS[t] = q;
  }
  auto fx = [&](int f, int eo, int nt, int k) { return FX[(((f * 2 + eo) * 2 + nt) * 2 + k) * 32 + lane]; };
  auto fb = [&](int f, int eo, int k) { return FB[((f * 2 + eo) * 3 + k) * 32 + lane]; };
  const int ly = t & 15, lx = t >> 4;   // per-thread line (x, y), y fastest (threads < 256)
  const bool zline = t < K1 * K1;
  const int nb = (NQ + ZB - 1) / ZB;

  auto forward_z = [&](int b) {   // Az/Bz of the batch's planes
    if (!zline) return;
    double a[ZB], c[ZB];
#pragma unroll
    for (int pl = 0; pl < ZB; ++pl) a[pl] = c[pl] = 0.0;
#pragma unroll
    for (int z = 0; z < K1; ++z) {
      const double uz = U[z * 256 + swu(lx, ly)];
#pragma unroll
      for (int pl = 0; pl < ZB; ++pl) {
        const int zq = b * ZB + pl;
        a[pl] = fma(SG[zq * K1 + z], uz, a[pl]);
        c[pl] = fma(DG[zq * K1 + z], uz, c[pl]);
      }
    }
#pragma unroll
    for (int pl = 0; pl < ZB; ++pl) {
      AZ[(pl * 2 + 0) * 256 + sw16(lx, ly)] = a[pl];
      AZ[(pl * 2 + 1) * 256 + sw16(lx, ly)] = c[pl];
    }
  };
  auto backward_z = [&](int b) {
    if (!zline) return;
    double q1[ZB], q2[ZB];
#pragma unroll
    for (int pl = 0; pl < ZB; ++pl) {
      q1[pl] = QQ[(pl * 2 + 0) * SZ_Q + lx * XS_Q + ly];
      q2[pl] = QQ[(pl * 2 + 1) * SZ_Q + lx * XS_Q + ly];
    }
#pragma unroll 4
    for (int z = 0; z < K1; ++z) {   // two independent partial sums per z (short dependency chains)
      double ts = 0.0, td = 0.0;
#pragma unroll
      for (int pl = 0; pl < ZB; ++pl) {
        const int zq = b * ZB + pl;
        ts = fma(SG[zq * K1 + z], q1[pl], ts);
        td = fma(DG[zq * K1 + z], q2[pl], td);
      }
      OUT[z * 256 + swu(lx, ly)] += ts + td;
    }
  };

  const int wpl = w / 3, wmt = w % 3;   // this warp's (plane, yq tile)
  for (long long cell = blockIdx.x; cell < ncell; cell += gridDim.x) {
  cp_async_wait_all();
  __syncthreads();   // U, VX of this cell landed; OUT zeroed
  if (EO) {   // x coefficients to the even / odd basis: u'_E0 = (u_0 + u_p)/2, u'_O0 = (u_0 - u_p)/2, permuted
    if (t < 256) {   // this thread's (z, y) row: read every source first (smem addressing), then write
      const int z = t >> 4, y = t & 15;
      double v[16];
#pragma unroll
      for (int pos = 0; pos < 16; ++pos) {
        const int j = tp.xsig[pos];
        v[pos] = j >= 0 ? U[z * 256 + swu(j, y)] : 0.0;
      }
      const double u0 = v[0], up = v[8];   // xsig[0] = 0, xsig[8] = p
      v[0] = 0.5 * (u0 + up);
      v[8] = 0.5 * (u0 - up);
#pragma unroll
      for (int pos = 0; pos < 16; ++pos) U[z * 256 + swu(pos, y)] = v[pos];
    }
    __syncthreads();
  }
  if (t < 24) {
    // x(xi, eta, zeta) = sum_a X_a prod_d (1 + s_ad xi_d) / 2 = sum_m GC[m] mono_m,
    // monomials m: 1, xi, eta, zeta, xi eta, xi zeta, eta zeta, xi eta zeta
    const int m = t / 3, i = t % 3;
    const int ex = (m == 1 || m == 4 || m == 5 || m == 7), ey = (m == 2 || m == 4 || m == 6 || m == 7),
              ez = (m == 3 || m == 5 || m == 6 || m == 7);
    double s = 0.0;
    for (int a = 0; a < 8; ++a) {
      const int ax = a & 1, ay = (a >> 1) & 1, az = a >> 2;
      const double sg = ((ex && !ax) ? -1.0 : 1.0) * ((ey && !ay) ? -1.0 : 1.0) * ((ez && !az) ? -1.0 : 1.0);
      s += sg * VX[a * 3 + i];
    }
    GC[m * 3 + i] = 0.125 * s;
  }
  forward_z(0);
  __syncthreads();   // also publishes GC
  const double al = VX[24], be = VX[25];
  const long long next = cell + gridDim.x;
  for (int b = 0; b < nb; ++b) {
    const int zq = b * ZB + wpl;
    if (b == nb - 1 && next < ncell) prefetch(next);   // U's last reader was forward_z(nb - 1)
    // ===== per-warp chain on rows yq in tile wmt of plane wpl (only __syncwarp inside)
    {   // forward y: AS/AD/BS rows [r][x] (x tiles 0, 1), 24 DMMA
      double cS[2][2] = {}, cD[2][2] = {}, cB[2][2] = {};
      const double* az = AZ + (wpl * 2 + 0) * 256;
      const double* bz = AZ + (wpl * 2 + 1) * 256;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double aS = fa(0, wmt, k), aD = fa(1, wmt, k);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int o = sw16(8 * nt + l4, 4 * k + lm);
          const double ba = az[o], bb = bz[o];
          dmma(cS[nt], aS, ba);
          dmma(cD[nt], aD, ba);
          dmma(cB[nt], aS, bb);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int o = l4 * XS_AS + ((8 * nt + 2 * lm) ^ h_as(l4));
        *reinterpret_cast<double2*>(WRg + 0 * SZ_ASF + o) = make_double2(cS[nt][0], cS[nt][1]);
        *reinterpret_cast<double2*>(WRg + 1 * SZ_ASF + o) = make_double2(cD[nt][0], cD[nt][1]);
        *reinterpret_cast<double2*>(WRg + 2 * SZ_ASF + o) = make_double2(cB[nt][0], cB[nt][1]);
      }
    }
    __syncwarp();
    if constexpr (EO) {
    // ----- even / odd x (TriParams::eo): per product the even part P_E = T_E a_E and the odd part
    // P_O = T_O a_O (K = 8, N = 12 point pairs); left / right points: values P_E +- P_O,
    // x-derivatives +-P_E + P_O (E' odd, O' even)
    double vE[4][2][2] = {}, vO[4][2][2] = {};   // [u, d_xi, d_eta, d_zeta][n tile][e]
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {   // even coefficients: k steps 0, 1; odd: k steps 2, 3
      const double* ae = WRg + l4 * XS_AS + ((4 * kk + lm) ^ h_as(l4));
      const double* ao = WRg + l4 * XS_AS + ((4 * (kk + 2) + lm) ^ h_as(l4));
      const double eS = ae[0], eD = ae[SZ_ASF], eB = ae[2 * SZ_ASF];
      const double oS = ao[0], oD = ao[SZ_ASF], oB = ao[2 * SZ_ASF];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double bSe = fx(0, 0, nt, kk), bDe = fx(1, 0, nt, kk), bSo = fx(0, 1, nt, kk), bDo = fx(1, 1, nt, kk);
        dmma(vE[0][nt], eS, bSe);
        dmma(vE[1][nt], eS, bDe);
        dmma(vE[2][nt], eD, bSe);
        dmma(vE[3][nt], eB, bSe);
        dmma(vO[0][nt], oS, bSo);
        dmma(vO[1][nt], oS, bDo);
        dmma(vO[2][nt], oD, bSo);
        dmma(vO[3][nt], oB, bSo);
      }
    }
    __syncwarp();   // AS rows consumed: the region now takes the pointwise combinations
    {   // pointwise at (zq, yq, x_r) and (zq, yq, -x_r); stores T+-, HX+-, HY+-, HZ+- [combo][row][r]
      const int yq = 8 * wmt + l4;
      const double ze = XQ[zq], et = XQ[yq];
      const double wzy = WQ[zq] * WQ[yq];
      double Jx[3], Jya[3], Jyb[3], Jza[3], Jzb[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double g1 = GC[3 + i], g2 = GC[6 + i], g3 = GC[9 + i], g4 = GC[12 + i], g5 = GC[15 + i], g6 = GC[18 + i],
                     g7 = GC[21 + i];
        Jx[i] = fma(fma(g7, ze, g4), et, fma(g5, ze, g1));
        Jya[i] = fma(g6, ze, g2);
        Jyb[i] = fma(g7, ze, g4);
        Jza[i] = fma(g6, et, g3);
        Jzb[i] = fma(g7, et, g5);
      }
      // 12 point pairs x 8 rows per warp = 3 slots per lane: the fragment layout gives lanes
      // lm < 2 four valid slots (n tile 1 holds r = 8..11) and lanes lm >= 2 two, so the slot
      // (n tile 1, e = 1) of lane lm is handed to lane lm + 2 (shuffle) and every lane runs three
      double hv[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        hv[q] = __shfl_xor_sync(0xffffffffu, vE[q][1][1], 2);
        hv[4 + q] = __shfl_xor_sync(0xffffffffu, vO[q][1][1], 2);
      }
#pragma unroll
      for (int sl = 0; sl < 3; ++sl) {
        double ve[4], vo[4];
        int r;
        if (sl < 2) {
          r = 2 * lm + sl;
#pragma unroll
          for (int q = 0; q < 4; ++q) { ve[q] = vE[q][0][sl]; vo[q] = vO[q][0][sl]; }
        } else if (lm < 2) {
          r = 8 + 2 * lm;
#pragma unroll
          for (int q = 0; q < 4; ++q) { ve[q] = vE[q][1][0]; vo[q] = vO[q][1][0]; }
        } else {
          r = 8 + 2 * (lm - 2) + 1;
#pragma unroll
          for (int q = 0; q < 4; ++q) { ve[q] = hv[q]; vo[q] = hv[4 + q]; }
        }
        {
          double out8[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // T+, T-, HX+, HX-, HY+, HY-, HZ+, HZ-
          if (r < tp.ne) {
            double tvs[2], hxs[2], hys[2], hzs[2];
#pragma unroll
            for (int side = 0; side < 2; ++side) {   // 0: left point r, 1: its mirror NQ - 1 - r
              const int xq = side ? NQ - 1 - r : r;
              const double sg = side ? -1.0 : 1.0;
              const double cu = fma(sg, vo[0], ve[0]);
              const double g0 = fma(sg, ve[1], vo[1]);
              const double g1 = fma(sg, vo[2], ve[2]);
              const double g2 = fma(sg, vo[3], ve[3]);
              const double xi = XQ[xq];
              double J[3][3];
#pragma unroll
              for (int i = 0; i < 3; ++i) {
                J[i][0] = Jx[i];
                J[i][1] = fma(Jyb[i], xi, Jya[i]);
                J[i][2] = fma(Jzb[i], xi, Jza[i]);
              }
              const double a00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], a01 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                           a02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
              const double a10 = J[1][2] * J[2][0] - J[1][0] * J[2][2], a11 = J[0][0] * J[2][2] - J[0][2] * J[2][0],
                           a12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
              const double a20 = J[1][0] * J[2][1] - J[1][1] * J[2][0], a21 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                           a22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
              const double det = J[0][0] * a00 + J[0][1] * a10 + J[0][2] * a20;
              const double wgt = wzy * WQ[xq];
              const double ad = fabs(det);
              const double kk = al * wgt * __drcp_rn(ad);
              const double v0 = a00 * g0 + a10 * g1 + a20 * g2, v1 = a01 * g0 + a11 * g1 + a21 * g2,
                           v2 = a02 * g0 + a12 * g1 + a22 * g2;
              hxs[side] = kk * (a00 * v0 + a01 * v1 + a02 * v2);
              hys[side] = kk * (a10 * v0 + a11 * v1 + a12 * v2);
              hzs[side] = kk * (a20 * v0 + a21 * v1 + a22 * v2);
              tvs[side] = be * wgt * ad * cu;
            }
            out8[0] = tvs[0] + tvs[1]; out8[1] = tvs[0] - tvs[1];
            out8[2] = hxs[0] + hxs[1]; out8[3] = hxs[0] - hxs[1];
            out8[4] = hys[0] + hys[1]; out8[5] = hys[0] - hys[1];
            out8[6] = hzs[0] + hzs[1]; out8[7] = hzs[0] - hzs[1];
          }
#pragma unroll
          for (int cmb = 0; cmb < 8; ++cmb) WRg[(cmb * 8 + l4) * XE + r] = out8[cmb];
        }
      }
    }
    __syncwarp();
    {   // backward x: even outputs from (T+, HX-, HY+, HZ+), odd outputs from (T-, HX+, HY-, HZ-), 24 DMMA
      double pE[4][2] = {}, pO[4][2] = {};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double* a = WRg + l4 * XE + 4 * k + lm;
        const double Tp = a[0], Tm = a[8 * XE], Xp = a[16 * XE], Xm = a[24 * XE], Yp = a[32 * XE], Ym = a[40 * XE],
                     Zp = a[48 * XE], Zm = a[56 * XE];
        const double sE = fb(0, 0, k), dE = fb(1, 0, k), sO = fb(0, 1, k), dO = fb(1, 1, k);
        dmma(pE[0], Tp, sE);
        dmma(pE[1], Xm, dE);
        dmma(pE[2], Yp, sE);
        dmma(pE[3], Zp, sE);
        dmma(pO[0], Tm, sO);
        dmma(pO[1], Xp, dO);
        dmma(pO[2], Ym, sO);
        dmma(pO[3], Zm, sO);
      }
      const int yq = 8 * wmt + l4;
      double* P = PP + (wpl * 3) * SZ_P;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int xe = 2 * lm + e, xo = 8 + 2 * lm + e;   // even / odd positions
        const int oe = xe * XS_P + (yq ^ h_p(xe)), oo = xo * XS_P + (yq ^ h_p(xo));
        P[oe] = pE[0][e] + pE[1][e];
        P[SZ_P + oe] = pE[2][e];
        P[2 * SZ_P + oe] = pE[3][e];
        P[oo] = pO[0][e] + pO[1][e];
        P[SZ_P + oo] = pO[2][e];
        P[2 * SZ_P + oo] = pO[3][e];
      }
    }
    } else {
    // forward x: u_q and hat-gradient at the 8 x 24 points of the rows, 48 DMMA
    double cu[3][2] = {}, c0[3][2] = {}, c1[3][2] = {}, c2[3][2] = {};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double* as = WRg + l4 * XS_AS + ((4 * k + lm) ^ h_as(l4));
      const double aS = as[0], aD = as[SZ_ASF], aB = as[2 * SZ_ASF];
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) {
        const double bS = fa(0, nt, k), bD = fa(1, nt, k);
        dmma(cu[nt], aS, bS);
        dmma(c0[nt], aS, bD);
        dmma(c1[nt], aD, bS);
        dmma(c2[nt], aB, bS);
      }
    }
    __syncwarp();   // AS rows consumed: the region now takes T/H rows
    {   // pointwise at (zq, yq, xq)
      const int yq = 8 * wmt + l4;
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
#pragma unroll
      for (int nt = 0; nt < 3; ++nt) {
        double tv[2], hx[2], hy[2], hz[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int xq = 8 * nt + 2 * lm + e;
          const double xi = XQ[xq];
          double J[3][3];
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            J[i][0] = Jx[i];
            J[i][1] = fma(Jyb[i], xi, Jya[i]);
            J[i][2] = fma(Jzb[i], xi, Jza[i]);
          }
          // adj(J): J^{-1} = adj / det
          const double a00 = J[1][1] * J[2][2] - J[1][2] * J[2][1], a01 = J[0][2] * J[2][1] - J[0][1] * J[2][2],
                       a02 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
          const double a10 = J[1][2] * J[2][0] - J[1][0] * J[2][2], a11 = J[0][0] * J[2][2] - J[0][2] * J[2][0],
                       a12 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
          const double a20 = J[1][0] * J[2][1] - J[1][1] * J[2][0], a21 = J[0][1] * J[2][0] - J[0][0] * J[2][1],
                       a22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
          const double det = J[0][0] * a00 + J[0][1] * a10 + J[0][2] * a20;
          const double wgt = wzy * WQ[xq];
          const double ad = fabs(det);
          const double kk = al * wgt * __drcp_rn(ad);
          const double g0 = c0[nt][e], g1 = c1[nt][e], g2 = c2[nt][e];
          // h = k adj adj^T g: v = adj^T g, h = k adj v
          const double v0 = a00 * g0 + a10 * g1 + a20 * g2, v1 = a01 * g0 + a11 * g1 + a21 * g2,
                       v2 = a02 * g0 + a12 * g1 + a22 * g2;
          hx[e] = kk * (a00 * v0 + a01 * v1 + a02 * v2);
          hy[e] = kk * (a10 * v0 + a11 * v1 + a12 * v2);
          hz[e] = kk * (a20 * v0 + a21 * v1 + a22 * v2);
          tv[e] = be * wgt * ad * cu[nt][e];
        }
        const int o = l4 * XS_TH + ((8 * nt + 2 * lm) ^ h_th(l4));
        *reinterpret_cast<double2*>(WRg + 0 * SZ_THF + o) = make_double2(tv[0], tv[1]);
        *reinterpret_cast<double2*>(WRg + 1 * SZ_THF + o) = make_double2(hx[0], hx[1]);
        *reinterpret_cast<double2*>(WRg + 2 * SZ_THF + o) = make_double2(hy[0], hy[1]);
        *reinterpret_cast<double2*>(WRg + 3 * SZ_THF + o) = make_double2(hz[0], hz[1]);
      }
    }
    __syncwarp();
    {   // backward x: P rows (x tiles 0, 1), 48 DMMA; P stored [x][yq] for the block-wide y stage
      double pa[2][2] = {}, pb[2][2] = {}, p2[2][2] = {}, p3[2][2] = {};
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double* a = WRg + l4 * XS_TH + ((4 * k + lm) ^ h_th(l4));
        const double aT = a[0], aX = a[SZ_THF], aY = a[2 * SZ_THF], aZ = a[3 * SZ_THF];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const double bS = ft(0, k, nt), bD = ft(1, k, nt);
          dmma(pa[nt], aT, bS);
          dmma(pb[nt], aX, bD);
          dmma(p2[nt], aY, bS);
          dmma(p3[nt], aZ, bS);
        }
      }
      const int yq = 8 * wmt + l4;
      double* P = PP + (wpl * 3) * SZ_P;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int x = 8 * nt + 2 * lm + e;
          const int o = x * XS_P + (yq ^ h_p(x));
          P[o] = pa[nt][e] + pb[nt][e];
          P[SZ_P + o] = p2[nt][e];
          P[2 * SZ_P + o] = p3[nt][e];
        }
    }
    }
    __syncthreads();
    // ===== backward y: warps 0-7 two Q1 jobs (2 terms), warps 8-11 four Q2 jobs; Q stored [x][y]
    if (w < 8) {
      double qa[2][2] = {}, qb[2][2] = {};
      const int mt = (w >> 1) & 1;   // shared by both jobs
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double aS = ft(0, k, mt), aD = ft(1, k, mt);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int j = w + 8 * i, pl = j >> 2, nt = j & 1;
          const int x = 8 * nt + l4;
          const double* P = PP + (pl * 3) * SZ_P + x * XS_P + ((4 * k + lm) ^ h_p(x));
          dmma(qa[i], aS, P[0]);
          dmma(qb[i], aD, P[SZ_P]);
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int j = w + 8 * i, pl = j >> 2, nt = j & 1;
        const int y = 8 * mt + l4, x0 = 8 * nt + 2 * lm;
        double* Q = QQ + (pl * 2) * SZ_Q + y;
        Q[x0 * XS_Q] = qa[i][0] + qb[i][0];
        Q[(x0 + 1) * XS_Q] = qa[i][1] + qb[i][1];
      }
    } else {
      double qc[4][2] = {};
#pragma unroll
      for (int k = 0; k < 6; ++k) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = (w - 8) + 4 * i, pl = j >> 2, mt = (j >> 1) & 1, nt = j & 1;
          const int x = 8 * nt + l4;
          dmma(qc[i], ft(0, k, mt), PP[(pl * 3 + 2) * SZ_P + x * XS_P + ((4 * k + lm) ^ h_p(x))]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int j = (w - 8) + 4 * i, pl = j >> 2, mt = (j >> 1) & 1, nt = j & 1;
        const int y = 8 * mt + l4, x0 = 8 * nt + 2 * lm;
        double* Q = QQ + (pl * 2 + 1) * SZ_Q + y;
        Q[x0 * XS_Q] = qc[i][0];
        Q[(x0 + 1) * XS_Q] = qc[i][1];
      }
    }
    __syncthreads();
    // ===== backward z of this batch, forward z of the next
    backward_z(b);
    if (b + 1 < nb) forward_z(b + 1);
    __syncthreads();
  }
  // local result of the cell: interior DoFs (owned by this cell alone) straight to out =
  // sign * A_K u (stores only; the gather adds f); skeleton entries (a local index 0 or p) ->
  // cellbuf [z][y][x].  OUT is zeroed for the next cell by the thread that read it.
  {
    const int cx = (int)(cell % tp.n[0]), cy = (int)((cell / tp.n[0]) % tp.n[1]),
              cz = (int)(cell / ((long long)tp.n[0] * tp.n[1]));
    const int n3 = P1 * P1 * P1;
    double* ob = cellbuf + cell * n3;

    for (int i = t; i < n3; i += TRI_THREADS) {
      const int z = i / (P1 * P1), y = (i / P1) % P1, x = i % P1;
      double v;
      if (EO) {   // back from the even / odd basis: v_0 = (v'_E0 + v'_O0)/2, v_p = (v'_E0 - v'_O0)/2
        if (x == 0 || x == p) {
          const double e0 = OUT[z * 256 + swu(0, y)], o0 = OUT[z * 256 + swu(8, y)];
          v = 0.5 * (x == 0 ? e0 + o0 : e0 - o0);
        } else {
          v = OUT[z * 256 + swu(XPOS[x], y)];
        }
      } else {
        v = OUT[z * 256 + swu(x, y)];
        OUT[z * 256 + swu(x, y)] = 0.0;
      }
      if (x == 0 || x == p || y == 0 || y == p || z == 0 || z == p) {
        ob[i] = v;
      } else {
        const long long ldx = tp.ldx_out > 0 ? tp.ldx_out : tp.Lx;
        const long long g = (((long long)cz * p + z) * tp.Ly + (long long)cy * p + y) * ldx + (long long)cx * p + x;
        out[g] = sign * v;
      }
    }
    if (EO) {   // the pair (E_0, O_0) is read by two threads: zero OUT after everyone has read it
      __syncthreads();
      for (int i = t; i < 4096; i += TRI_THREADS) OUT[i] = 0.0;
    }
  }
  }
}

// out[g] = f[g] (or 0) + (cell interior DoF: the value the apply kernel stored | skeleton DoF,
// on a cell face, edge or vertex: sign * the sum over the cells containing g of their local
// result, cells ascending in z, y, x: deterministic); constrained entries 0.  One warp per grid
// row (gy, gz), grid-stride over rows; 32-bit index math.
// x decode of the gathers: the (<= 2) cells containing gx and the local indices, and the flags
// (bit0: on a cell boundary, bit1: constrained); tabulated in shared memory for gx < 1024 and
// computed on the fly beyond (meshes with more than 1024 x entries)
constexpr int kXTab = 1024;
__device__ __forceinline__ void tri_xdec(const TriParams& tp, int gx, int4& xe, int& fl) {
  const int p = tp.p;
  int cc = gx / p;
  if (cc >= tp.n[0]) cc = tp.n[0] - 1;
  const int aa = gx - cc * p;
  xe = (aa == 0 && cc > 0) ? make_int4(cc - 1, p, cc, 0) : make_int4(cc, aa, 0, -1);
  fl = (aa == 0 || aa == p ? 1 : 0) | (tri_cons(gx, (long long)tp.n[0] * p, tp.gamma_d, 0) ? 2 : 0);
}

__global__ void tri_gather_kernel(const __grid_constant__ TriParams tp, const double* __restrict__ cellbuf,
                                  const double* __restrict__ f, double* __restrict__ out, double sign) {
  // per-x table (once per block): the (<= 2) cells containing gx and the local indices, skeleton
  // and constraint flags; per row the (<= 2 x 2) (cell-row, local) bases; every loop has constant
  // bounds (registers, no local memory) and one table lookup replaces the per-DoF divisions
  __shared__ int4 xtab[kXTab];   // (cell0, local0, cell1, local1); local1 < 0: one cell
  __shared__ unsigned char xfl[kXTab];   // bit0: on a cell boundary, bit1: constrained
  const int Lx = (int)tp.Lx, Ly = (int)tp.Ly, Lz = (int)tp.Lz;
  const int p = tp.p, P1 = p + 1, n3 = P1 * P1 * P1;
  for (int gx = threadIdx.x; gx < Lx && gx < kXTab; gx += blockDim.x) {
    int4 xe;
    int fl;
    tri_xdec(tp, gx, xe, fl);
    xtab[gx] = xe;
    xfl[gx] = (unsigned char)fl;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nrow = Ly * Lz, wstride = gridDim.x * (blockDim.x >> 5);
  const long long ldx = tp.ldx_out > 0 ? tp.ldx_out : Lx;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < nrow; row += wstride) {
    const int gy = row % Ly, gz = row / Ly;
    const bool rcons = tri_cons(gy, (long long)tp.n[1] * p, tp.gamma_d, 1) || tri_cons(gz, (long long)tp.n[2] * p, tp.gamma_d, 2);
    int cy0, ay0, cy1 = 0, ay1 = -1, cz0, az0, cz1 = 0, az1 = -1;
    {
      int cc = gy / p; if (cc >= tp.n[1]) cc = tp.n[1] - 1;
      const int aa = gy - cc * p;
      if (aa == 0 && cc > 0) { cy0 = cc - 1; ay0 = p; cy1 = cc; ay1 = 0; } else { cy0 = cc; ay0 = aa; }
    }
    {
      int cc = gz / p; if (cc >= tp.n[2]) cc = tp.n[2] - 1;
      const int aa = gz - cc * p;
      if (aa == 0 && cc > 0) { cz0 = cc - 1; az0 = p; cz1 = cc; az1 = 0; } else { cz0 = cc; az0 = aa; }
    }
    const bool rskel = ay0 == 0 || ay0 == p || az0 == 0 || az0 == p;
    // (cell-row base, local-row offset) of the (kz, ky) combinations; valid flags
    const int rb00 = (cz0 * tp.n[1] + cy0) * tp.n[0], ro00 = (az0 * P1 + ay0) * P1;
    const int rb01 = (cz0 * tp.n[1] + cy1) * tp.n[0], ro01 = (az0 * P1 + ay1) * P1;
    const int rb10 = (cz1 * tp.n[1] + cy0) * tp.n[0], ro10 = (az1 * P1 + ay0) * P1;
    const int rb11 = (cz1 * tp.n[1] + cy1) * tp.n[0], ro11 = (az1 * P1 + ay1) * P1;
    const bool v01 = ay1 >= 0, v10 = az1 >= 0, v11 = v01 && v10;
    const long long fbase = (long long)row * Lx, obase = (long long)row * ldx;
    for (int gx = lane; gx < Lx; gx += 32) {
      const long long g = obase + gx;
      int4 xe;
      int fl;
      if (gx < kXTab) { xe = xtab[gx]; fl = xfl[gx]; } else tri_xdec(tp, gx, xe, fl);
      if (rcons || (fl & 2)) { out[g] = 0.0; continue; }
      const double fv = f ? f[fbase + gx] : 0.0;
      if (!rskel && !(fl & 1)) { out[g] = fv + out[g]; continue; }   // cell interior (stored by the apply)
      auto at = [&](int rb, int ro, int c, int a) { return cellbuf[(size_t)(rb + c) * n3 + ro + a]; };
      double s = at(rb00, ro00, xe.x, xe.y);
      if (xe.w >= 0) s += at(rb00, ro00, xe.z, xe.w);
      if (v01) { s += at(rb01, ro01, xe.x, xe.y); if (xe.w >= 0) s += at(rb01, ro01, xe.z, xe.w); }
      if (v10) { s += at(rb10, ro10, xe.x, xe.y); if (xe.w >= 0) s += at(rb10, ro10, xe.z, xe.w); }
      if (v11) { s += at(rb11, ro11, xe.x, xe.y); if (xe.w >= 0) s += at(rb11, ro11, xe.z, xe.w); }
      out[g] = fv + sign * s;
    }
  }
  (void)Lz;
}

// Skeleton-only gather: the cell-interior entries are final already (the Cartesian H(grad) apply
// writes f + sign A_K u there; on the SC-fused path (ICC-SC, one rank) the SC pre step completed
// them in place between the apply and this kernel); only SKELETON DoFs are written, out[g] = f[g] + sign * (sum of the <= 8 cell contributions)
// and, for face-interior DoFs, minus the condensation line sums e of the (<= 2) cells sharing the
// face (lower cell first; fb != null) -- the same operations, in the same order, as the gather
// followed by sc_face_kernel.  Rows with y and z off the cell boundaries only visit the x-boundary DoFs.
// resident CTAs per SM: measured best with the line sums (cfg5: 8 vs 6 -> -15 us) and without them
// (cfg2: 4 vs 6 -> -4 us; 8 -> +12 us)
template <int MINB>
__global__ void __launch_bounds__(256, MINB) tri_gather_sc_kernel(const __grid_constant__ TriParams tp, const double* __restrict__ cellbuf,
                                     const double* __restrict__ f, double* __restrict__ out, double sign,
                                     const double* __restrict__ fb) {
  __shared__ int4 xtab[kXTab];
  __shared__ unsigned char xfl[kXTab];
  const int Lx = (int)tp.Lx, Ly = (int)tp.Ly;
  const int p = tp.p, P1 = p + 1, n3 = P1 * P1 * P1, pm = p - 1, nf = pm * pm;
  for (int gx = threadIdx.x; gx < Lx && gx < kXTab; gx += blockDim.x) {
    int4 xe;
    int fl;
    tri_xdec(tp, gx, xe, fl);
    xtab[gx] = xe;
    xfl[gx] = (unsigned char)fl;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nrow = Ly * (int)tp.Lz, wstride = gridDim.x * (blockDim.x >> 5);
  const long long ldx = tp.ldx_out > 0 ? tp.ldx_out : Lx;
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < nrow; row += wstride) {
    const int gy = row % Ly, gz = row / Ly;
    const bool rcons = tri_cons(gy, (long long)tp.n[1] * p, tp.gamma_d, 1) || tri_cons(gz, (long long)tp.n[2] * p, tp.gamma_d, 2);
    int cy0, ay0, cy1 = 0, ay1 = -1, cz0, az0, cz1 = 0, az1 = -1;
    {
      int cc = gy / p; if (cc >= tp.n[1]) cc = tp.n[1] - 1;
      const int aa = gy - cc * p;
      if (aa == 0 && cc > 0) { cy0 = cc - 1; ay0 = p; cy1 = cc; ay1 = 0; } else { cy0 = cc; ay0 = aa; }
    }
    {
      int cc = gz / p; if (cc >= tp.n[2]) cc = tp.n[2] - 1;
      const int aa = gz - cc * p;
      if (aa == 0 && cc > 0) { cz0 = cc - 1; az0 = p; cz1 = cc; az1 = 0; } else { cz0 = cc; az0 = aa; }
    }
    const bool by = gy % p == 0, bz = gz % p == 0;
    const bool rskel = by || bz;
    const int rb00 = (cz0 * tp.n[1] + cy0) * tp.n[0], ro00 = (az0 * P1 + ay0) * P1;
    const int rb01 = (cz0 * tp.n[1] + cy1) * tp.n[0], ro01 = (az0 * P1 + ay1) * P1;
    const int rb10 = (cz1 * tp.n[1] + cy0) * tp.n[0], ro10 = (az1 * P1 + ay0) * P1;
    const int rb11 = (cz1 * tp.n[1] + cy1) * tp.n[0], ro11 = (az1 * P1 + ay1) * P1;
    const bool v01 = ay1 >= 0, v10 = az1 >= 0, v11 = v01 && v10;
    const long long fbase = (long long)row * Lx, obase = (long long)row * ldx;
    // skeleton rows: every x; other rows: the x-boundary DoFs (cell index t = gx / p)
    const int nx_ = rskel ? Lx : tp.n[0] + 1;
    for (int t = lane; t < nx_; t += 32) {
      const int gx = rskel ? t : t * p;
      const long long g = obase + gx;
      int4 xe;
      int fl;
      if (gx < kXTab) { xe = xtab[gx]; fl = xfl[gx]; } else tri_xdec(tp, gx, xe, fl);
      if (rcons || (fl & 2)) { out[g] = 0.0; continue; }
      if (!(fl & 1) && !rskel) continue;   // cell interior (completed by the SC pre step)
      const double fv = f ? f[fbase + gx] : 0.0;
      auto at = [&](int rb, int ro, int c, int a) { return cellbuf[(size_t)(rb + c) * n3 + ro + a]; };
      double s = at(rb00, ro00, xe.x, xe.y);
      if (xe.w >= 0) s += at(rb00, ro00, xe.z, xe.w);
      if (v01) { s += at(rb01, ro01, xe.x, xe.y); if (xe.w >= 0) s += at(rb01, ro01, xe.z, xe.w); }
      if (v10) { s += at(rb10, ro10, xe.x, xe.y); if (xe.w >= 0) s += at(rb10, ro10, xe.z, xe.w); }
      if (v11) { s += at(rb11, ro11, xe.x, xe.y); if (xe.w >= 0) s += at(rb11, ro11, xe.z, xe.w); }
      double r = fv + sign * s;
      const bool bx = (fl & 1) != 0;
      if (fb && (int)bx + (int)by + (int)bz == 1) {   // face-interior DoF: the condensation line sums
        const int dir = bx ? 0 : (by ? 1 : 2);
        const int gg[3] = {gx, gy, gz};
        const int d1 = dir == 0 ? 1 : 0, d2 = dir == 2 ? 1 : 2;
        const int a = gg[d1] % p - 1, b = gg[d2] % p - 1, P = gg[dir] / p;
        int cell[3];
        cell[d1] = gg[d1] / p; cell[d2] = gg[d2] / p;
        double e = 0.0;
        if (P > 0) {
          cell[dir] = P - 1;
          const int K = (cell[2] * tp.n[1] + cell[1]) * tp.n[0] + cell[0];
          e += fb[((size_t)K * 6 + 2 * dir + 1) * nf + b * pm + a];
        }
        if (P < tp.n[dir]) {
          cell[dir] = P;
          const int K = (cell[2] * tp.n[1] + cell[1]) * tp.n[0] + cell[0];
          e += fb[((size_t)K * 6 + 2 * dir) * nf + b * pm + a];
        }
        r -= e;
      }
      out[g] = r;
    }
  }
}

cudaError_t launch_skeleton_gather_sc(const TriParams& tp, const double* cellbuf, const double* f, double* out,
                                      double sign, const double* fb, cudaStream_t st) {
  if (fb && tp.p < 2) return cudaErrorInvalidValue;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  if (fb) tri_gather_sc_kernel<8><<<(unsigned)(nsm * 8), 256, 0, st>>>(tp, cellbuf, f, out, sign, fb);
  else tri_gather_sc_kernel<4><<<(unsigned)(nsm * 8), 256, 0, st>>>(tp, cellbuf, f, out, sign, fb);
  return cudaGetLastError();
}

cudaError_t launch_apply_trilinear(const TriParams& tp, const double* tabs, const double* X, const double* alpha,
                                   const double* beta, int coef_const, const double* u, const double* f, double* out,
                                   double sign, double* cellbuf, cudaStream_t st, int* nlaunch, const KTimer* kt) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(apply_tri_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRI_SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(apply_tri_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TRI_SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (tp.p + 1 > K1 || tp.nq > NQP) return cudaErrorInvalidValue;
  const long long ncell = (long long)tp.n[0] * tp.n[1] * tp.n[2];
  const long long nd = tp.Lx * tp.Ly * tp.Lz;
  if (ncell <= 0) return cudaSuccess;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const unsigned grid = (unsigned)std::min<long long>(ncell, nsm);   // persistent: one CTA per SM
  if (kt) kt->begin(kt->arg);
  if (tp.eo)
    apply_tri_kernel<true><<<grid, TRI_THREADS, TRI_SMEM, st>>>(tp, tabs, X, alpha, beta, coef_const, u, f, out, sign, cellbuf);
  else
    apply_tri_kernel<false><<<grid, TRI_THREADS, TRI_SMEM, st>>>(tp, tabs, X, alpha, beta, coef_const, u, f, out, sign, cellbuf);
  if (kt) kt->end(kt->arg);
  if (!tp.skip_gather) tri_gather_kernel<<<(unsigned)(nsm * 8), 256, 0, st>>>(tp, cellbuf, f, out, sign);
  (void)nd;
  if (nlaunch) *nlaunch += tp.skip_gather ? 1 : 2;
  return cudaGetLastError();
}

cudaError_t launch_skeleton_gather(const TriParams& tp, const double* cellbuf, const double* f, double* out, double sign,
                                   cudaStream_t st) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  tri_gather_kernel<<<(unsigned)(nsm * 8), 256, 0, st>>>(tp, cellbuf, f, out, sign);
  return cudaGetLastError();
}

size_t tri_cellbuf_doubles(const TriParams& tp) {
  return (size_t)tp.n[0] * tp.n[1] * tp.n[2] * (tp.p + 1) * (tp.p + 1) * (tp.p + 1);
}

}  // namespace rm
