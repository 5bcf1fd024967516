// 1D FDM basis (PAPER.md eq:fdmbasis P:356-366, eq:unisolvence P:387-400, eq:eigs P:419-425,
// S_IG = -S_II S_II^T B_IG P:441-443, DP basis P:464-469, D-hat P:485-487, G-bar P:705-723).
#include "basis.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>

namespace rm {

static void legendre(int n, double x, double& Ln, double& dLn, double& d2Ln) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { Ln = 1; dLn = 0; d2Ln = 0; return; }
  for (int k = 1; k < n; ++k) {
    double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1; p1 = p2;
  }
  Ln = p1;
  // Legendre ODE: (1-x^2) L'' - 2x L' + n(n+1) L = 0 ; (1-x^2) L' = n (L_{n-1} - x L_n)
  dLn = n * (p0 - x * p1) / (1.0 - x * x);
  d2Ln = (2.0 * x * dLn - n * (n + 1) * p1) / (1.0 - x * x);
}

void gauss_rule(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0); w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));   // Chebyshev-like initial guess
    for (int it = 0; it < 100; ++it) {
      double L, dL, d2;
      legendre(n, t, L, dL, d2);
      double dt = L / dL;
      t -= dt;
      if (std::fabs(dt) < 1e-17) break;
    }
    double L, dL, d2;
    legendre(n, t, L, dL, d2);
    x[n - 1 - i] = t;
    w[n - 1 - i] = 2.0 / ((1.0 - t * t) * dL * dL);
  }
}

void gll_rule(int n, std::vector<double>& x, std::vector<double>& w) {
  if (n < 2) throw std::runtime_error("gll_rule: n < 2");
  int m = n - 1;
  x.assign(n, 0.0); w.assign(n, 0.0);
  x[0] = -1.0; x[n - 1] = 1.0;
  for (int i = 1; i < n - 1; ++i) {
    double t = -std::cos(M_PI * i / m);   // Chebyshev-Gauss-Lobatto guess, roots of L_m'
    for (int it = 0; it < 100; ++it) {
      double L, dL, d2;
      legendre(m, t, L, dL, d2);
      double dt = dL / d2;
      t -= dt;
      if (std::fabs(dt) < 1e-17) break;
    }
    x[i] = t;
  }
  for (int i = 0; i < n; ++i) {
    double L, dL, d2;
    if (i == 0 || i == n - 1) L = (i == 0 && (m % 2)) ? -1.0 : 1.0;
    else legendre(m, x[i], L, dL, d2);
    w[i] = 2.0 / (n * (n - 1) * L * L);
  }
}

void lagrange_tab(const std::vector<double>& nodes, const std::vector<double>& x,
                  std::vector<double>& V, std::vector<double>& dV) {
  const int n = (int)nodes.size(), nq = (int)x.size();
  std::vector<double> bw(n, 1.0);  // barycentric weights
  for (int j = 0; j < n; ++j)
    for (int m = 0; m < n; ++m)
      if (m != j) bw[j] /= (nodes[j] - nodes[m]);
  V.assign((size_t)nq * n, 0.0); dV.assign((size_t)nq * n, 0.0);
  for (int q = 0; q < nq; ++q) {
    int hit = -1;
    for (int j = 0; j < n; ++j) if (x[q] == nodes[j]) hit = j;
    if (hit >= 0) {
      V[q * n + hit] = 1.0;
      // derivative at a node: l_j'(x_i) = (bw_j/bw_i)/(x_i-x_j), l_i'(x_i) = -sum_{j!=i}
      double diag = 0.0;
      for (int j = 0; j < n; ++j) if (j != hit) {
        double d = (bw[j] / bw[hit]) / (nodes[hit] - nodes[j]);
        dV[q * n + j] = d; diag -= d;
      }
      dV[q * n + hit] = diag;
      continue;
    }
    // l_j(x) = l(x) bw_j/(x-x_j), l(x) = prod (x-x_m); l_j'(x) = l_j(x) * (sum_{m!=j} 1/(x-x_m))
    double lx = 1.0, ssum = 0.0;
    for (int m = 0; m < n; ++m) { lx *= (x[q] - nodes[m]); ssum += 1.0 / (x[q] - nodes[m]); }
    for (int j = 0; j < n; ++j) {
      double lj = lx * bw[j] / (x[q] - nodes[j]);
      V[q * n + j] = lj;
      dV[q * n + j] = lj * (ssum - 1.0 / (x[q] - nodes[j]));
    }
  }
}

// Symmetric eigenproblem C v = mu v by cyclic Jacobi rotations (C row-major n x n, overwritten).
static void jacobi_eig(int n, std::vector<double>& C, std::vector<double>& mu, std::vector<double>& Vv) {
  Vv.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) Vv[i * n + i] = 1.0;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) { double c2 = C[i * n + j] * C[i * n + j]; tot += c2; if (i != j) off += c2; }
    if (off <= 1e-30 * tot) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double apq = C[p * n + q];
        if (std::fabs(apq) < 1e-300) continue;
        double theta = (C[q * n + q] - C[p * n + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {  // columns p,q
          double ckp = C[k * n + p], ckq = C[k * n + q];
          C[k * n + p] = c * ckp - s * ckq; C[k * n + q] = s * ckp + c * ckq;
        }
        for (int k = 0; k < n; ++k) {  // rows p,q
          double cpk = C[p * n + k], cqk = C[q * n + k];
          C[p * n + k] = c * cpk - s * cqk; C[q * n + k] = s * cpk + c * cqk;
        }
        for (int k = 0; k < n; ++k) {
          double vkp = Vv[k * n + p], vkq = Vv[k * n + q];
          Vv[k * n + p] = c * vkp - s * vkq; Vv[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
  mu.resize(n);
  for (int i = 0; i < n; ++i) mu[i] = C[i * n + i];
}

void Basis1D::tab_s(const std::vector<double>& x, std::vector<double>& s, std::vector<double>& ds) const {
  std::vector<double> V, dV;
  lagrange_tab(nodes, x, V, dV);
  const int n = p + 1, nq = (int)x.size();
  s.assign((size_t)nq * n, 0.0); ds.assign((size_t)nq * n, 0.0);
  for (int q = 0; q < nq; ++q)
    for (int j = 0; j < n; ++j) {
      double a = 0, b = 0;
      for (int i = 0; i < n; ++i) { a += V[q * n + i] * S[i * n + j]; b += dV[q * n + i] * S[i * n + j]; }
      s[q * n + j] = a; ds[q * n + j] = b;
    }
}

void Basis1D::tab_r(const std::vector<double>& x, std::vector<double>& r) const {
  std::vector<double> s, ds;
  tab_s(x, s, ds);
  const int nq = (int)x.size();
  r.assign((size_t)nq * p, 0.0);
  for (int q = 0; q < nq; ++q) {
    r[q * p + 0] = 1.0 / std::sqrt(2.0);
    for (int j = 1; j < p; ++j) r[q * p + j] = ds[q * (p + 1) + j] / std::sqrt(lam[j]);
  }
}

static Basis1D build(int p) {
  if (p < 1) throw std::runtime_error("basis: p < 1");
  Basis1D b;
  b.p = p;
  const int n = p + 1;
  std::vector<double> w;
  gll_rule(n, b.nodes, w);
  std::vector<double> xq, wq, V, dV;
  gauss_rule(p + 2, xq, wq);                 // exact for degree 2p+3
  lagrange_tab(b.nodes, xq, V, dV);
  std::vector<double> Bg(n * n, 0.0), Ag(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double sb = 0, sa = 0;
      for (size_t q = 0; q < xq.size(); ++q) {
        sb += wq[q] * V[q * n + i] * V[q * n + j];
        sa += wq[q] * dV[q * n + i] * dV[q * n + j];
      }
      Bg[i * n + j] = sb; Ag[i * n + j] = sa;
    }
  b.S.assign(n * n, 0.0);
  b.S[0] = 1.0; b.S[p * n + p] = 1.0;        // S_GG = I, S_GI = 0
  b.lam.assign(n, 0.0);
  b.lam[0] = 2.0;
  const int m = p - 1;
  if (m > 0) {
    // Cholesky of B_II = L L^T; C = L^{-1} A_II L^{-T}; S_II = L^{-T} V
    std::vector<double> L(m * m, 0.0);
    for (int j = 0; j < m; ++j) {
      double d = Bg[(j + 1) * n + (j + 1)];
      for (int k = 0; k < j; ++k) d -= L[j * m + k] * L[j * m + k];
      if (!(d > 0)) throw std::runtime_error("basis: B_II not SPD");
      L[j * m + j] = std::sqrt(d);
      for (int i = j + 1; i < m; ++i) {
        double s = Bg[(i + 1) * n + (j + 1)];
        for (int k = 0; k < j; ++k) s -= L[i * m + k] * L[j * m + k];
        L[i * m + j] = s / L[j * m + j];
      }
    }
    // X = L^{-1} A_II  (forward substitution on columns), C = X L^{-T}
    std::vector<double> X(m * m), C(m * m);
    for (int c = 0; c < m; ++c)
      for (int i = 0; i < m; ++i) {
        double s = Ag[(i + 1) * n + (c + 1)];
        for (int k = 0; k < i; ++k) s -= L[i * m + k] * X[k * m + c];
        X[i * m + c] = s / L[i * m + i];
      }
    for (int r = 0; r < m; ++r)
      for (int j = 0; j < m; ++j) {
        double s = X[r * m + j];
        for (int k = 0; k < j; ++k) s -= C[r * m + k] * L[j * m + k];
        C[r * m + j] = s / L[j * m + j];
      }
    for (int i = 0; i < m; ++i)   // symmetrise
      for (int j = 0; j < i; ++j) { double a = 0.5 * (C[i * m + j] + C[j * m + i]); C[i * m + j] = C[j * m + i] = a; }
    std::vector<double> mu, Vv;
    jacobi_eig(m, C, mu, Vv);
    std::vector<int> ord(m);
    for (int i = 0; i < m; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](int a, int c) { return mu[a] < mu[c]; });   // reading G3
    // S_II = L^{-T} V (backward substitution)
    std::vector<double> Sii(m * m);
    for (int cc = 0; cc < m; ++cc) {
      int c = ord[cc];
      for (int i = m - 1; i >= 0; --i) {
        double s = Vv[i * m + c];
        for (int k = i + 1; k < m; ++k) s -= L[k * m + i] * Sii[k * m + cc];
        Sii[i * m + cc] = s / L[i * m + i];
      }
      b.lam[cc + 1] = mu[c];
    }
    // sign: s_j'(-1) > 0   (reading G3)
    std::vector<double> Vm, dVm;
    lagrange_tab(b.nodes, std::vector<double>{-1.0}, Vm, dVm);
    for (int cc = 0; cc < m; ++cc) {
      double slope = 0;
      for (int i = 0; i < m; ++i) slope += dVm[i + 1] * Sii[i * m + cc];
      if (slope < 0) for (int i = 0; i < m; ++i) Sii[i * m + cc] = -Sii[i * m + cc];
    }
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) b.S[(i + 1) * n + (j + 1)] = Sii[i * m + j];
    // S_IG = -S_II S_II^T B_IG
    for (int g = 0; g < 2; ++g) {
      int gc = g ? p : 0;
      std::vector<double> t(m, 0.0);
      for (int k = 0; k < m; ++k)
        for (int i = 0; i < m; ++i) t[k] += Sii[i * m + k] * Bg[(i + 1) * n + gc];
      for (int i = 0; i < m; ++i) {
        double s = 0;
        for (int k = 0; k < m; ++k) s += Sii[i * m + k] * t[k];
        b.S[(i + 1) * n + gc] = -s;
      }
    }
  }
  b.B.assign(n * n, 0.0); b.A.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double sb = 0, sa = 0;
      for (int a = 0; a < n; ++a)
        for (int c = 0; c < n; ++c) {
          sb += b.S[a * n + i] * Bg[a * n + c] * b.S[c * n + j];
          sa += b.S[a * n + i] * Ag[a * n + c] * b.S[c * n + j];
        }
      b.B[i * n + j] = sb; b.A[i * n + j] = sa;
    }
  // D-hat by Gauss quadrature of (r_i, s_j')
  std::vector<double> s, ds, r;
  b.tab_s(xq, s, ds);
  b.tab_r(xq, r);
  b.D.assign((size_t)p * n, 0.0);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < n; ++j) {
      double acc = 0;
      for (size_t q = 0; q < xq.size(); ++q) acc += wq[q] * r[q * p + i] * ds[q * n + j];
      b.D[i * n + j] = acc;
    }
  // G-bar: symmetric square root of the 2x2 interface Gram [[a, c],[c, a]] (a = B00 = Bpp by symmetry)
  b.G.assign(n * n, 0.0);
  for (int i = 0; i < n; ++i) b.G[i * n + i] = 1.0;
  {
    double a = b.B[0], d = b.B[p * n + p], c = b.B[p];
    // eigen-decomposition of a symmetric 2x2
    double tr = a + d, det = a * d - c * c;
    double disc = std::sqrt(std::max(0.0, 0.25 * (a - d) * (a - d) + c * c));
    double l1 = 0.5 * tr + disc, l2 = 0.5 * tr - disc;
    (void)det;
    double v1x, v1y;
    if (std::fabs(c) > 0) { v1x = l1 - d; v1y = c; } else { v1x = (a >= d) ? 1 : 0; v1y = (a >= d) ? 0 : 1; }
    double nv = std::sqrt(v1x * v1x + v1y * v1y); v1x /= nv; v1y /= nv;
    double v2x = -v1y, v2y = v1x;
    double s1 = std::sqrt(l1), s2 = std::sqrt(l2);
    b.G[0] = s1 * v1x * v1x + s2 * v2x * v2x;
    b.G[p] = s1 * v1x * v1y + s2 * v2x * v2y;
    b.G[p * n] = b.G[p];
    b.G[p * n + p] = s1 * v1y * v1y + s2 * v2y * v2y;
  }
  return b;
}

const Basis1D& basis(int p) {
  static std::mutex mu;
  static std::map<int, Basis1D> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(p);
  if (it == cache.end()) it = cache.emplace(p, build(p)).first;
  return it->second;
}

}  // namespace rm
