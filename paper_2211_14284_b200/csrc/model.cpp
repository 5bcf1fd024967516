#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <tuple>

namespace rm {

static const int FAMS[4][3][3] = {
    {{FAM_P, FAM_P, FAM_P}, {0, 0, 0}, {0, 0, 0}},
    {{FAM_D, FAM_P, FAM_P}, {FAM_P, FAM_D, FAM_P}, {FAM_P, FAM_P, FAM_D}},
    {{FAM_P, FAM_D, FAM_D}, {FAM_D, FAM_P, FAM_D}, {FAM_D, FAM_D, FAM_P}},
    {{FAM_D, FAM_D, FAM_D}, {0, 0, 0}, {0, 0, 0}},
};
static int ncomp_of(int k) { return (k == 0 || k == 3) ? 1 : 3; }

void Space::init(int k_, int p_, int nx, int ny, int nz) {
  k = k_; p = p_; n[0] = nx; n[1] = ny; n[2] = nz;
  ncomp = ncomp_of(k);
  for (int m = 0; m < 3; ++m)
    for (int d = 0; d < 3; ++d) fam[m][d] = FAMS[k][m][d];
}

bool Space::constrained(int m, int64_t ix, int64_t iy, int64_t iz, uint32_t gamma_d) const {
  const int64_t idx[3] = {ix, iy, iz};
  for (int d = 0; d < 3; ++d) {
    if (fam[m][d] != FAM_P) continue;
    if (idx[d] == 0 && (gamma_d & (1u << (2 * d)))) return true;
    if (idx[d] == (int64_t)n[d] * p && (gamma_d & (1u << (2 * d + 1)))) return true;
  }
  return false;
}

// ----------------------------------------------------------------------------- 1D algebra
static Mat1 mk(int r, int c) { Mat1 m; m.rows = r; m.cols = c; m.v.assign((size_t)r * c, 0.0); return m; }
static Mat1 eye(int n) { Mat1 m = mk(n, n); for (int i = 0; i < n; ++i) m.v[i * n + i] = 1.0; return m; }
static Mat1 mul(const Mat1& a, const Mat1& b) {
  if (a.cols != b.rows) throw std::runtime_error("mul: shape");
  Mat1 c = mk(a.rows, b.cols);
  for (int i = 0; i < a.rows; ++i)
    for (int k = 0; k < a.cols; ++k) {
      double x = a(i, k);
      if (x == 0.0) continue;
      for (int j = 0; j < b.cols; ++j) c.v[(size_t)i * c.cols + j] += x * b(k, j);
    }
  return c;
}
static Mat1 tr(const Mat1& a) {
  Mat1 t = mk(a.cols, a.rows);
  for (int i = 0; i < a.rows; ++i)
    for (int j = 0; j < a.cols; ++j) t.v[(size_t)j * t.cols + i] = a(i, j);
  return t;
}

struct MassScale { double c; int e[3]; };
static MassScale mass_scale(int j, int n) {
  // pullback constants on an axis-aligned box: detJ = hx hy hz / 8
  MassScale s;
  switch (j) {
    case 0: s = {1.0 / 8.0, {1, 1, 1}}; break;
    case 1: s = {0.5, {1, 1, 1}}; s.e[n] -= 2; break;
    case 2: s = {2.0, {-1, -1, -1}}; s.e[n] += 2; break;
    default: s = {8.0, {-1, -1, -1}}; break;
  }
  return s;
}

struct Contrib { int m, e; double sigma; };   // d^k u contribution to target comp: sigma * d_e u_m
static std::vector<std::vector<Contrib>> derivative(int k) {
  std::vector<std::vector<Contrib>> L;
  if (k == 0) L = {{{0, 0, 1}}, {{0, 1, 1}}, {{0, 2, 1}}};
  else if (k == 1)   // standard curl (reading G17)
    L = {{{2, 1, 1}, {1, 2, -1}}, {{0, 2, 1}, {2, 0, -1}}, {{1, 0, 1}, {0, 1, -1}}};
  else if (k == 2) L = {{{0, 0, 1}, {1, 1, 1}, {2, 2, 1}}};
  else throw std::runtime_error("derivative: k");
  return L;
}

CellOperator build_cell_operator(int k, int p) {
  const Basis1D& b = basis(p);
  const int n = p + 1;
  Mat1 Bh = mk(n, n), Dh = mk(p, n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      bool pat = (i == j) || ((i == 0 || i == p) && (j == 0 || j == p));
      Bh.v[i * n + j] = pat ? b.B[i * n + j] : 0.0;
    }
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < n; ++j) {
      bool pat = (j == 0 || j == p || j == i);
      Dh.v[i * n + j] = pat ? b.D[i * n + j] : 0.0;
    }
  Mat1 DhT = tr(Dh), IP = eye(n), ID = eye(p);
  auto mass1 = [&](int f) -> const Mat1& { return f == FAM_P ? Bh : ID; };
  auto ident = [&](int f) -> const Mat1& { return f == FAM_P ? IP : ID; };

  CellOperator op;
  op.k = k; op.p = p;
  auto add_mat = [&](const Mat1& m) -> int {
    for (size_t i = 0; i < op.mats.size(); ++i)
      if (op.mats[i].rows == m.rows && op.mats[i].cols == m.cols && op.mats[i].v == m.v) return (int)i;
    op.mats.push_back(m);
    return (int)op.mats.size() - 1;
  };
  const int nc = ncomp_of(k);
  // mass terms M^k_beta
  for (int m = 0; m < nc; ++m) {
    MassScale s = mass_scale(k, m);
    Term t{m, m, 1, s.c, {s.e[0], s.e[1], s.e[2]}, {0, 0, 0}};
    for (int d = 0; d < 3; ++d) t.mat[d] = add_mat(mass1(FAMS[k][m][d]));
    op.terms.push_back(t);
  }
  // stiffness terms D^T M^{k+1}_alpha D
  auto L = derivative(k);
  for (size_t tn = 0; tn < L.size(); ++tn) {
    MassScale s = mass_scale(k + 1, (int)tn);
    for (const Contrib& a : L[tn])
      for (const Contrib& c : L[tn]) {
        Term t{a.m, c.m, 0, a.sigma * c.sigma * s.c, {s.e[0], s.e[1], s.e[2]}, {0, 0, 0}};
        for (int d = 0; d < 3; ++d) {
          int ft = FAMS[k + 1][tn][d];
          Mat1 left = (d == a.e) ? DhT : ident(ft);
          Mat1 right = (d == c.e) ? Dh : ident(ft);
          t.mat[d] = add_mat(mul(mul(left, mass1(ft)), right));
        }
        op.terms.push_back(t);
      }
  }
  return op;
}

CellEntries cartesian_cell_entries(const CellOperator& op, const Space& sp, double hx, double hy, double hz) {
  const int nl = sp.nloc();
  std::vector<int> coff(sp.ncomp + 1, 0);
  for (int m = 0; m < sp.ncomp; ++m) coff[m + 1] = coff[m] + sp.nloc_comp(m);
  std::vector<double> K((size_t)nl * nl, 0.0), M((size_t)nl * nl, 0.0);
  std::vector<char> touched((size_t)nl * nl, 0);
  const double h[3] = {hx, hy, hz};
  for (const Term& t : op.terms) {
    double sc = t.c;
    for (int d = 0; d < 3; ++d) sc *= std::pow(h[d], t.hexp[d]);
    const Mat1 &X = op.mats[t.mat[0]], &Y = op.mats[t.mat[1]], &Z = op.mats[t.mat[2]];
    const int ox = sp.lsize(t.mout, 0), oy = sp.lsize(t.mout, 1), oz = sp.lsize(t.mout, 2);
    const int ix_ = sp.lsize(t.min, 0), iy_ = sp.lsize(t.min, 1), iz_ = sp.lsize(t.min, 2);
    std::vector<double>& T = (t.coef == 0) ? K : M;
    for (int c = 0; c < oz; ++c)
      for (int b2 = 0; b2 < oy; ++b2)
        for (int a = 0; a < ox; ++a) {
          int row = coff[t.mout] + (c * oy + b2) * ox + a;
          for (int c2 = 0; c2 < iz_; ++c2) {
            double z = Z(c, c2);
            if (z == 0.0) continue;
            for (int bb = 0; bb < iy_; ++bb) {
              double y = Y(b2, bb);
              if (y == 0.0) continue;
              for (int aa = 0; aa < ix_; ++aa) {
                double x = X(a, aa);
                if (x == 0.0) continue;
                int col = coff[t.min] + (c2 * iy_ + bb) * ix_ + aa;
                T[(size_t)row * nl + col] += sc * x * y * z;
                touched[(size_t)row * nl + col] = 1;
              }
            }
          }
        }
  }
  CellEntries e;
  for (int r = 0; r < nl; ++r)
    for (int c = 0; c < nl; ++c)
      if (touched[(size_t)r * nl + c]) {
        e.row.push_back(r); e.col.push_back(c);
        e.kval.push_back(K[(size_t)r * nl + c]); e.mval.push_back(M[(size_t)r * nl + c]);
      }
  return e;
}

// ------------------------------------------------------------------ auxiliary operator k=0
// P_K = G0^T diag0 G0 + sum_m (G1 D)_m^T diag1_m (G1 D)_m (eq:sum-factorization_approx P:732-739):
// every entry is a fixed linear combination of the four sum-factorised diagonals, so the
// geometry enters only through aux_cell_diagonals and the entry map is built once per p.
namespace {
std::mutex aux_mu;
std::map<int, std::unique_ptr<AuxTables>> aux_cache;

AuxTables* make_aux_tables(int p) {
  auto T = std::make_unique<AuxTables>();
  const Basis1D& b = basis(p);
  const int n = p + 1;
  T->p = p;
  T->nq = (3 * (p + 1) + 1) / 2;   // reading G1/G2
  const int nq = T->nq;
  gll_rule(nq, T->xq, T->wq);
  std::vector<double> s, ds, r;
  b.tab_s(T->xq, s, ds);
  b.tab_r(T->xq, r);
  // broken P basis s-bar = s G^{-1}: only columns 0, p change (2x2 inverse of G_GG)
  const double g00 = b.G[0], g0p = b.G[p], gp0 = b.G[p * n], gpp = b.G[p * n + p];
  const double det = g00 * gpp - g0p * gp0;
  const double i00 = gpp / det, i0p = -g0p / det, ip0 = -gp0 / det, ipp = g00 / det;
  std::vector<double> sb(s);
  for (int q = 0; q < nq; ++q) {
    double s0 = s[q * n + 0], sp_ = s[q * n + p];
    sb[q * n + 0] = s0 * i00 + sp_ * ip0;
    sb[q * n + p] = s0 * i0p + sp_ * ipp;
  }
  T->sb2.resize(sb.size());
  for (size_t i = 0; i < sb.size(); ++i) T->sb2[i] = sb[i] * sb[i];
  T->r2.resize(r.size());
  for (size_t i = 0; i < r.size(); ++i) T->r2[i] = r[i] * r[i];
  T->off[0] = 0;
  T->off[1] = n * n * n;
  T->off[2] = T->off[1] + n * n * p;
  T->off[3] = T->off[2] + n * n * p;
  T->ndiag = T->off[3] + n * n * p;
  // sparse rows of G (n x n) and D-hat (p x n), structural pattern only
  std::vector<std::vector<std::pair<int, double>>> Gr(n), Dr(p);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      bool pat = (i == j) || ((i == 0 || i == p) && (j == 0 || j == p));
      if (pat) Gr[i].push_back({j, b.G[i * n + j]});
    }
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < n; ++j)
      if (j == 0 || j == p || j == i) Dr[i].push_back({j, b.D[i * n + j]});
  struct Tm { int g; double a, c; };
  std::map<std::pair<int, int>, std::vector<Tm>> acc;
  auto idx3 = [&](int l, int j, int i) { return (l * n + j) * n + i; };
  // G0^T diag0 G0 : broken dof (l,j,i) row of G0 = G[l,:] x G[j,:] x G[i,:]
  for (int l = 0; l < n; ++l)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        const int g = idx3(l, j, i);
        std::vector<std::pair<int, double>> rowv;
        for (auto& zl : Gr[l]) for (auto& yj : Gr[j]) for (auto& xi : Gr[i])
          rowv.push_back({idx3(zl.first, yj.first, xi.first), zl.second * yj.second * xi.second});
        for (auto& a : rowv) for (auto& c : rowv) acc[{a.first, c.first}].push_back({g, a.second, c.second});
      }
  // (G1 D)^T diag1 (G1 D): comp x row = G[l,:] x G[j,:] x D[i,:], etc.
  for (int m = 0; m < 3; ++m) {
    const int nx_ = (m == 0) ? p : n, ny_ = (m == 1) ? p : n, nz_ = (m == 2) ? p : n;
    for (int l = 0; l < nz_; ++l)
      for (int j = 0; j < ny_; ++j)
        for (int i = 0; i < nx_; ++i) {
          const int g = T->off[1 + m] + (l * ny_ + j) * nx_ + i;
          const auto& Rz = (m == 2) ? Dr[l] : Gr[l];
          const auto& Ry = (m == 1) ? Dr[j] : Gr[j];
          const auto& Rx = (m == 0) ? Dr[i] : Gr[i];
          std::vector<std::pair<int, double>> rowv;
          for (auto& zl : Rz) for (auto& yj : Ry) for (auto& xi : Rx)
            rowv.push_back({idx3(zl.first, yj.first, xi.first), zl.second * yj.second * xi.second});
          for (auto& a : rowv) for (auto& c : rowv) acc[{a.first, c.first}].push_back({g, a.second, c.second});
        }
  }
  T->tptr.push_back(0);
  for (auto& kv : acc) {
    T->row.push_back(kv.first.first); T->col.push_back(kv.first.second);
    for (const Tm& t : kv.second) { T->tg.push_back(t.g); T->ta.push_back(t.a); T->tc.push_back(t.c); }
    T->tptr.push_back((int)T->tg.size());
  }
  return T.release();
}
}  // namespace

const AuxTables& aux_tables(int p) {
  std::lock_guard<std::mutex> lk(aux_mu);
  auto it = aux_cache.find(p);
  if (it == aux_cache.end()) it = aux_cache.emplace(p, std::unique_ptr<AuxTables>(make_aux_tables(p))).first;
  return *it->second;
}

void aux_cell_diagonals(const AuxTables& T, const double Xc[8][3], double alpha, double beta, double* diag) {
  const int p = T.p, n = p + 1, nq = T.nq;
  // geometry at the nq^3 points: W0 = w detJ beta, W1[m] = w detJ alpha (J^{-1}J^{-T})_mm
  const size_t NQ = (size_t)nq * nq * nq;
  std::vector<double> W0(NQ), W1[3];
  for (int m = 0; m < 3; ++m) W1[m].resize(NQ);
  for (int qz = 0; qz < nq; ++qz)
    for (int qy = 0; qy < nq; ++qy)
      for (int qx = 0; qx < nq; ++qx) {
        const double t[3] = {T.xq[qx], T.xq[qy], T.xq[qz]};
        double phi[3][2], dphi[3][2];
        for (int d = 0; d < 3; ++d) { phi[d][0] = 0.5 * (1 - t[d]); phi[d][1] = 0.5 * (1 + t[d]); dphi[d][0] = -0.5; dphi[d][1] = 0.5; }
        double J[3][3] = {{0}};
        for (int az = 0; az < 2; ++az)
          for (int ay = 0; ay < 2; ++ay)
            for (int ax = 0; ax < 2; ++ax) {
              const double* X = Xc[az * 4 + ay * 2 + ax];
              double f0 = dphi[0][ax] * phi[1][ay] * phi[2][az];
              double f1 = phi[0][ax] * dphi[1][ay] * phi[2][az];
              double f2 = phi[0][ax] * phi[1][ay] * dphi[2][az];
              for (int i = 0; i < 3; ++i) { J[i][0] += X[i] * f0; J[i][1] += X[i] * f1; J[i][2] += X[i] * f2; }
            }
        double dJ = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
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
        const size_t q = ((size_t)qz * nq + qy) * nq + qx;
        const double w = T.wq[qx] * T.wq[qy] * T.wq[qz] * dJ;
        W0[q] = w * beta;
        for (int m = 0; m < 3; ++m) {
          double jj = Ji[m][0] * Ji[m][0] + Ji[m][1] * Ji[m][1] + Ji[m][2] * Ji[m][2];   // (J^{-1}J^{-T})_mm
          W1[m][q] = w * alpha * jj;
        }
      }
  // sum-factorised diagonals: diag[l,j,i] = sum_q Tz^2[qz,l] Ty^2[qy,j] Tx^2[qx,i] W[q]
  auto contract = [&](const std::vector<double>& W, const std::vector<double>& Tx, int nx_,
                      const std::vector<double>& Ty, int ny_, const std::vector<double>& Tz, int nz_, double* c) {
    std::vector<double> a((size_t)nq * nq * nx_, 0.0), bb((size_t)nq * ny_ * nx_, 0.0);
    for (int qz = 0; qz < nq; ++qz)
      for (int qy = 0; qy < nq; ++qy)
        for (int i = 0; i < nx_; ++i) {
          double acc = 0;
          for (int qx = 0; qx < nq; ++qx) acc += Tx[qx * nx_ + i] * W[((size_t)qz * nq + qy) * nq + qx];
          a[((size_t)qz * nq + qy) * nx_ + i] = acc;
        }
    for (int qz = 0; qz < nq; ++qz)
      for (int j = 0; j < ny_; ++j)
        for (int i = 0; i < nx_; ++i) {
          double acc = 0;
          for (int qy = 0; qy < nq; ++qy) acc += Ty[qy * ny_ + j] * a[((size_t)qz * nq + qy) * nx_ + i];
          bb[((size_t)qz * ny_ + j) * nx_ + i] = acc;
        }
    for (int l = 0; l < nz_; ++l)
      for (int j = 0; j < ny_; ++j)
        for (int i = 0; i < nx_; ++i) {
          double acc = 0;
          for (int qz = 0; qz < nq; ++qz) acc += Tz[qz * nz_ + l] * bb[((size_t)qz * ny_ + j) * nx_ + i];
          c[((size_t)l * ny_ + j) * nx_ + i] = acc;
        }
  };
  contract(W0, T.sb2, n, T.sb2, n, T.sb2, n, diag + T.off[0]);
  contract(W1[0], T.r2, p, T.sb2, n, T.sb2, n, diag + T.off[1]);
  contract(W1[1], T.sb2, n, T.r2, p, T.sb2, n, diag + T.off[2]);
  contract(W1[2], T.sb2, n, T.sb2, n, T.r2, p, diag + T.off[3]);
}

void aux_entries_from_diagonals(const AuxTables& T, const double* diag, double* vals) {
  const int ne = (int)T.row.size();
  for (int t = 0; t < ne; ++t) {
    double acc = 0.0;
    for (int k = T.tptr[t]; k < T.tptr[t + 1]; ++k) acc += T.ta[k] * diag[T.tg[k]] * T.tc[k];
    vals[t] = acc;
  }
}

void aux_interior_weights(const AuxTables& T, const double* diag, double* w_int) {
  const int p = T.p, n = p + 1, pm = p - 1, ni = pm * pm * pm;
  const double* d1[3] = {diag + T.off[1], diag + T.off[2], diag + T.off[3]};
  for (int k = 1; k < p; ++k)
    for (int j = 1; j < p; ++j)
      for (int i = 1; i < p; ++i) {
        const int I = ((k - 1) * pm + (j - 1)) * pm + (i - 1);
        w_int[0 * ni + I] = d1[0][((size_t)k * n + j) * p + i];   // x: (z P, y P, x DP)
        w_int[1 * ni + I] = d1[1][((size_t)k * p + j) * n + i];   // y: (z P, y DP, x P)
        w_int[2 * ni + I] = d1[2][((size_t)k * n + j) * n + i];   // z: (z DP, y P, x P)
      }
}

void aux_cell_entries(int p, const double Xc[8][3], double alpha, double beta, CellEntries& out, double* w_int) {
  const AuxTables& T = aux_tables(p);
  std::vector<double> diag(T.ndiag);
  aux_cell_diagonals(T, Xc, alpha, beta, diag.data());
  if (w_int) aux_interior_weights(T, diag.data(), w_int);
  out.row = T.row; out.col = T.col;
  out.kval.resize(T.row.size());
  aux_entries_from_diagonals(T, diag.data(), out.kval.data());
  out.mval.assign(T.row.size(), 0.0);
}

}  // namespace rm
