// p = 1 coarse level: assembly of A_0 and its block-tridiagonal Cholesky (coarse.hpp).
#include "coarse.hpp"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <tuple>

#include "basis.hpp"

namespace rm {

namespace {

// True operator of a trilinear hexahedron at p = 1 (Q_1, k = 0) by GLL quadrature with
// ceil(3 (1 + 1) / 2) = 3 points per direction (reading G1): [A_K]_ab = sum_q w_q |J|
// (beta phi_a phi_b + alpha (J^-T grad phi_a) . (J^-T grad phi_b)), local order z, y, x.
void q1_trilinear_matrix(const double Xc[8][3], double alpha, double beta, double A[64]) {
  const double xq[3] = {-1.0, 0.0, 1.0}, wq[3] = {1.0 / 3.0, 4.0 / 3.0, 1.0 / 3.0};
  std::memset(A, 0, 64 * sizeof(double));
  for (int qz = 0; qz < 3; ++qz)
    for (int qy = 0; qy < 3; ++qy)
      for (int qx = 0; qx < 3; ++qx) {
        const double t[3] = {xq[qx], xq[qy], xq[qz]};
        double phi[3][2], dphi[2] = {-0.5, 0.5};
        for (int d = 0; d < 3; ++d) { phi[d][0] = 0.5 * (1 - t[d]); phi[d][1] = 0.5 * (1 + t[d]); }
        double val[8], gref[8][3];
        for (int az = 0; az < 2; ++az)
          for (int ay = 0; ay < 2; ++ay)
            for (int ax = 0; ax < 2; ++ax) {
              const int a = (az * 2 + ay) * 2 + ax;
              val[a] = phi[0][ax] * phi[1][ay] * phi[2][az];
              gref[a][0] = dphi[ax] * phi[1][ay] * phi[2][az];
              gref[a][1] = phi[0][ax] * dphi[ay] * phi[2][az];
              gref[a][2] = phi[0][ax] * phi[1][ay] * dphi[az];
            }
        double J[3][3] = {{0}};   // J[i][d] = d x_i / d xi_d
        for (int a = 0; a < 8; ++a)
          for (int i = 0; i < 3; ++i)
            for (int d = 0; d < 3; ++d) J[i][d] += Xc[a][i] * gref[a][d];
        const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        if (!(det > 0)) throw std::runtime_error("coarse level: non-positive Jacobian");
        double Ji[3][3];   // inverse of J
        Ji[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
        Ji[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
        Ji[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
        Ji[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
        Ji[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
        Ji[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
        Ji[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
        Ji[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
        Ji[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
        double g[8][3];   // physical gradients J^-T grad-hat
        for (int a = 0; a < 8; ++a)
          for (int i = 0; i < 3; ++i) g[a][i] = Ji[0][i] * gref[a][0] + Ji[1][i] * gref[a][1] + Ji[2][i] * gref[a][2];
        const double w = wq[qx] * wq[qy] * wq[qz] * det;
        for (int a = 0; a < 8; ++a)
          for (int b = 0; b < 8; ++b)
            A[a * 8 + b] += w * (beta * val[a] * val[b] + alpha * (g[a][0] * g[b][0] + g[a][1] * g[b][1] + g[a][2] * g[b][2]));
      }
}

// in-place dense Cholesky of the lower triangle of S (m x m, row-major); returns false on a
// non-positive pivot
bool dense_cholesky(int m, double* S) {
  for (int k = 0; k < m; ++k) {
    double d = S[(size_t)k * m + k];
    for (int t = 0; t < k; ++t) d -= S[(size_t)k * m + t] * S[(size_t)k * m + t];
    if (!(d > 0)) return false;
    d = std::sqrt(d);
    S[(size_t)k * m + k] = d;
#pragma omp parallel for schedule(static)
    for (int i = k + 1; i < m; ++i) {
      double s = S[(size_t)i * m + k];
      const double* Li = S + (size_t)i * m;
      const double* Lk = S + (size_t)k * m;
      for (int t = 0; t < k; ++t) s -= Li[t] * Lk[t];
      S[(size_t)i * m + k] = s / d;
    }
  }
  for (int i = 0; i < m; ++i)
    for (int j = i + 1; j < m; ++j) S[(size_t)i * m + j] = 0.0;
  return true;
}

}  // namespace

void build_coarse(const CoarseSetupInput& in, CoarseFactor& F) {
  const int p = in.p;
  if (p > 15) throw std::runtime_error("coarse level: p > 15");
  Space& s1 = F.sp1;
  s1.init(in.k, 1, in.n[0], in.n[1], in.n[2]);
  F.ndof1 = s1.ndof();
  const int nl = s1.nloc();
  // ---- block order (z index of every coarse DoF) and positions
  const int nb = in.n[2] + 1;
  std::vector<int> blk(F.ndof1), pos(F.ndof1);
  std::vector<std::vector<int64_t>> members(nb);
  for (int m = 0; m < s1.ncomp; ++m)
    for (int64_t z = 0; z < s1.len(m, 2); ++z)
      for (int64_t y = 0; y < s1.len(m, 1); ++y)
        for (int64_t x = 0; x < s1.len(m, 0); ++x) {
          const int64_t g = s1.gidx(m, z, y, x);
          blk[g] = (int)z;
          pos[g] = (int)members[z].size();
          members[z].push_back(g);
        }
  F.bstart.assign(nb + 1, 0);
  for (int j = 0; j < nb; ++j) F.bstart[j + 1] = F.bstart[j] + (int)members[j].size();
  F.perm.clear();
  for (int j = 0; j < nb; ++j) F.perm.insert(F.perm.end(), members[j].begin(), members[j].end());
  F.cmask.assign(F.ndof1, 0);
  std::vector<uint8_t> con(F.ndof1, 0);
  F.nfree1 = 0;
  for (int m = 0; m < s1.ncomp; ++m)
    for (int64_t z = 0; z < s1.len(m, 2); ++z)
      for (int64_t y = 0; y < s1.len(m, 1); ++y)
        for (int64_t x = 0; x < s1.len(m, 0); ++x) {
          const int64_t g = s1.gidx(m, z, y, x);
          con[g] = s1.constrained(m, x, y, z, in.gamma_d) ? 1 : 0;
          F.nfree1 += !con[g];
        }
  for (size_t t = 0; t < F.perm.size(); ++t) F.cmask[t] = con[F.perm[t]];
  // ---- dense blocks of A_0: diagonal A_jj and sub-diagonal A_{j+1,j}
  std::vector<std::vector<double>> Ad(nb), As(nb > 1 ? nb - 1 : 0);
  auto msz = [&](int j) { return F.bstart[j + 1] - F.bstart[j]; };
  for (int j = 0; j < nb; ++j) Ad[j].assign((size_t)msz(j) * msz(j), 0.0);
  for (int j = 0; j + 1 < nb; ++j) As[j].assign((size_t)msz(j + 1) * msz(j), 0.0);
  std::vector<int> lc, la[3];
  for (int m = 0; m < s1.ncomp; ++m)
    for (int c = 0; c < s1.lsize(m, 2); ++c)
      for (int b = 0; b < s1.lsize(m, 1); ++b)
        for (int a = 0; a < s1.lsize(m, 0); ++a) { lc.push_back(m); la[0].push_back(a); la[1].push_back(b); la[2].push_back(c); }
  CellOperator op1;
  if (in.cartesian) op1 = build_cell_operator(in.k, 1);
  std::map<std::tuple<double, double, double>, CellEntries> cache;
  std::vector<double> Aq(64);
  for (int cz = 0; cz < in.n[2]; ++cz)
    for (int cy = 0; cy < in.n[1]; ++cy)
      for (int cx = 0; cx < in.n[0]; ++cx) {
        const int64_t cell = ((int64_t)cz * in.n[1] + cy) * in.n[0] + cx;
        const double al = in.n_alpha == 1 ? in.alpha[0] : in.alpha[cell];
        const double be = in.n_beta == 1 ? in.beta[0] : in.beta[cell];
        std::vector<int64_t> gl(nl);
        for (int l = 0; l < nl; ++l) gl[l] = s1.gidx(lc[l], (int64_t)cz + la[2][l], (int64_t)cy + la[1][l], (int64_t)cx + la[0][l]);
        auto add = [&](int i, int j, double v) {
          const int64_t gi = gl[i], gj = gl[j];
          const int bi = blk[gi], bj = blk[gj];
          if (bi == bj) Ad[bi][(size_t)pos[gi] * msz(bi) + pos[gj]] += v;
          else if (bi == bj + 1) As[bj][(size_t)pos[gi] * msz(bj) + pos[gj]] += v;
        };
        if (in.cartesian) {
          auto key = std::make_tuple(in.hx[cx], in.hy[cy], in.hz[cz]);
          auto it = cache.find(key);
          if (it == cache.end()) it = cache.emplace(key, cartesian_cell_entries(op1, s1, in.hx[cx], in.hy[cy], in.hz[cz])).first;
          const CellEntries& E = it->second;
          for (size_t t = 0; t < E.row.size(); ++t) add(E.row[t], E.col[t], al * E.kval[t] + be * E.mval[t]);
        } else {
          if (in.k != 0) throw std::runtime_error("coarse level on trilinear cells: H(grad) only");
          double Xc[8][3];
          for (int az = 0; az < 2; ++az)
            for (int ay = 0; ay < 2; ++ay)
              for (int ax = 0; ax < 2; ++ax) {
                const int64_t vi = (((int64_t)(cz + az) * (in.n[1] + 1) + (cy + ay)) * (in.n[0] + 1) + (cx + ax)) * 3;
                for (int i = 0; i < 3; ++i) Xc[(az * 2 + ay) * 2 + ax][i] = in.coords[vi + i];
              }
          q1_trilinear_matrix(Xc, al, be, Aq.data());
          for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 8; ++j) add(i, j, Aq[i * 8 + j]);
        }
      }
  // constrained coarse DoFs: identity rows / columns (held at zero: their right-hand side is masked)
  for (int j = 0; j < nb; ++j) {
    const int m = msz(j);
    for (int i = 0; i < m; ++i) {
      if (!F.cmask[F.bstart[j] + i]) continue;
      for (int t = 0; t < m; ++t) { Ad[j][(size_t)i * m + t] = 0.0; Ad[j][(size_t)t * m + i] = 0.0; }
      Ad[j][(size_t)i * m + i] = 1.0;
      if (j + 1 < nb) for (int r = 0; r < msz(j + 1); ++r) As[j][(size_t)r * m + i] = 0.0;
      if (j > 0) for (int t = 0; t < msz(j - 1); ++t) As[j - 1][(size_t)i * msz(j - 1) + t] = 0.0;
    }
  }
  // ---- block Cholesky
  F.o_linv.assign(nb, 0); F.o_linvt.assign(nb, 0); F.o_lsub.assign(nb, 0); F.o_lsubt.assign(nb, 0);
  int64_t tot = 0;
  for (int j = 0; j < nb; ++j) {
    F.o_linv[j] = tot; tot += (int64_t)msz(j) * msz(j);
    F.o_linvt[j] = tot; tot += (int64_t)msz(j) * msz(j);
    if (j + 1 < nb) { F.o_lsub[j] = tot; tot += (int64_t)msz(j + 1) * msz(j); F.o_lsubt[j] = tot; tot += (int64_t)msz(j + 1) * msz(j); }
  }
  F.vals.assign(tot, 0.0);
  std::vector<double> Lprev;   // L_{j,j-1} (m_j x m_{j-1})
  for (int j = 0; j < nb; ++j) {
    const int m = msz(j);
    std::vector<double>& S = Ad[j];
    if (j > 0) {   // S_j = A_jj - L_{j,j-1} L_{j,j-1}^T
      const int mp = msz(j - 1);
#pragma omp parallel for schedule(dynamic, 8)
      for (int i = 0; i < m; ++i)
        for (int t = 0; t <= i; ++t) {
          const double* a = &Lprev[(size_t)i * mp];
          const double* b = &Lprev[(size_t)t * mp];
          double s = 0.0;
          for (int q = 0; q < mp; ++q) s += a[q] * b[q];
          S[(size_t)i * m + t] -= s;
        }
    }
    if (!dense_cholesky(m, S.data()))
      throw std::runtime_error("coarse level: non-positive pivot in block " + std::to_string(j));
    double* Linv = &F.vals[F.o_linv[j]];
    // Linv = L^{-1}: column c solves L x = e_c (forward substitution), columns independent
#pragma omp parallel for schedule(dynamic, 8)
    for (int c = 0; c < m; ++c) {
      for (int i = 0; i < c; ++i) Linv[(size_t)i * m + c] = 0.0;
      Linv[(size_t)c * m + c] = 1.0 / S[(size_t)c * m + c];
      for (int i = c + 1; i < m; ++i) {
        double s = 0.0;
        for (int t = c; t < i; ++t) s -= S[(size_t)i * m + t] * Linv[(size_t)t * m + c];
        Linv[(size_t)i * m + c] = s / S[(size_t)i * m + i];
      }
    }
    double* LinvT = &F.vals[F.o_linvt[j]];
    for (int i = 0; i < m; ++i)
      for (int c = 0; c < m; ++c) LinvT[(size_t)c * m + i] = Linv[(size_t)i * m + c];
    if (j + 1 < nb) {   // L_{j+1,j} = A_{j+1,j} L_jj^{-T}: row r = Linv applied to A row r
      const int mn = msz(j + 1);
      Lprev.assign((size_t)mn * m, 0.0);
      const std::vector<double>& A = As[j];
#pragma omp parallel for schedule(dynamic, 8)
      for (int r = 0; r < mn; ++r) {
        const double* ar = &A[(size_t)r * m];
        for (int i = 0; i < m; ++i) {
          double s = 0.0;
          const double* li = Linv + (size_t)i * m;
          for (int t = 0; t <= i; ++t) s += li[t] * ar[t];
          Lprev[(size_t)r * m + i] = s;
        }
      }
      double* Ls = &F.vals[F.o_lsub[j]];
      double* LsT = &F.vals[F.o_lsubt[j]];
      std::memcpy(Ls, Lprev.data(), Lprev.size() * sizeof(double));
      for (int r = 0; r < mn; ++r)
        for (int i = 0; i < m; ++i) LsT[(size_t)i * mn + r] = Lprev[(size_t)r * m + i];
    }
  }
  // ---- 1D embedding coefficients (s_a, phi_0 / phi_1) by GLL quadrature exact to degree 2p+1
  const Basis1D& b = basis(p);
  std::vector<double> xq, wq, sv, dsv;
  gll_rule(p + 2, xq, wq);
  b.tab_s(xq, sv, dsv);
  for (int a = 1; a < p; ++a) {
    double s0 = 0.0, s1v = 0.0;
    for (size_t q = 0; q < xq.size(); ++q) {
      const double sa = sv[q * (p + 1) + a];
      s0 += wq[q] * sa * 0.5 * (1.0 - xq[q]);
      s1v += wq[q] * sa * 0.5 * (1.0 + xq[q]);
    }
    F.e0[a] = s0;
    F.e1[a] = s1v;
  }
}

}  // namespace rm
