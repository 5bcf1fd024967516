// 1D FDM element of arXiv 2211.14284 (§2.2-2.3), host side of the product path.
// Independent of oracle/: own GLL/Gauss rules (Newton on Legendre), own generalized symmetric
// eigensolver (Cholesky reduction + cyclic Jacobi), own quadrature of D-hat.
#pragma once
#include <vector>

namespace rm {

void gll_rule(int n, std::vector<double>& x, std::vector<double>& w);
void gauss_rule(int n, std::vector<double>& x, std::vector<double>& w);
// values V[q*n+j] = l_j(x_q), derivatives dV likewise, barycentric form
void lagrange_tab(const std::vector<double>& nodes, const std::vector<double>& x,
                  std::vector<double>& V, std::vector<double>& dV);

struct Basis1D {
  int p = 0;
  std::vector<double> nodes;  // GLL nodes xi_0..xi_p
  std::vector<double> S;      // (p+1)^2, S[i*(p+1)+j] = s_j(xi_i)
  std::vector<double> lam;    // lam[0] = 2, lam[j] = (s_j', s_j') j=1..p-1  (eq:fdmbasis)
  std::vector<double> B, A;   // FDM mass / stiffness (p+1)^2 row-major
  std::vector<double> D;      // p x (p+1), D_ij = (r_i, s_j')
  std::vector<double> G;      // (p+1)^2 broken transform, G_GG = B_GG^{1/2}  (reading G4)
  // tabulations at arbitrary points
  void tab_s(const std::vector<double>& x, std::vector<double>& s, std::vector<double>& ds) const;
  void tab_r(const std::vector<double>& x, std::vector<double>& r) const;
};

const Basis1D& basis(int p);  // cached per p; throws std::runtime_error on failure

}  // namespace rm
