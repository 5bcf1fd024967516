// Structured de Rham layouts and the Cartesian cell operator as a sum of Kronecker terms.
//
// Layout (reading G16): per component m, a C-order [Z][Y][X] array; per
// direction d the family is P (n_d p + 1 entries, shared at multiples of p) or DP (n_d p).
// Component families: Q_p (P,P,P); NCE_p x:(D,P,P) y:(P,D,P) z:(P,P,D);
// NCF_p x:(P,D,D) y:(D,P,D) z:(D,D,P).
//
// Cartesian cell operator (eq:sum-factorization P:690-692 with the pullbacks P:640-648):
//   A_K = M^k_beta + D^T M^{k+1}_alpha D,  every block a Kronecker product of 1D matrices
//   (B-hat on P directions, identity on DP directions, D-hat / D-hat^T for derivatives) scaled by
//   coef_c * c_t * hx^ex hy^ey hz^ez.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "basis.hpp"

namespace rm {

enum { FAM_P = 0, FAM_D = 1 };

struct Space {
  int k = 0, p = 1;
  int n[3] = {1, 1, 1};   // cells per direction (global)
  int ncomp = 1;
  int fam[3][3];           // [comp][dir]
  void init(int k_, int p_, int nx, int ny, int nz);
  int64_t len(int m, int d) const { return fam[m][d] == FAM_P ? (int64_t)n[d] * p + 1 : (int64_t)n[d] * p; }
  int64_t comp_size(int m) const { return len(m, 0) * len(m, 1) * len(m, 2); }
  int64_t offset(int m) const { int64_t o = 0; for (int c = 0; c < m; ++c) o += comp_size(c); return o; }
  int64_t ndof() const { return offset(ncomp); }
  int lsize(int m, int d) const { return fam[m][d] == FAM_P ? p + 1 : p; }
  int nloc_comp(int m) const { return lsize(m, 0) * lsize(m, 1) * lsize(m, 2); }
  int nloc() const { int s = 0; for (int m = 0; m < ncomp; ++m) s += nloc_comp(m); return s; }
  int64_t gidx(int m, int64_t iz, int64_t iy, int64_t ix) const {
    return offset(m) + (iz * len(m, 1) + iy) * len(m, 0) + ix;
  }
  // constrained: one of the P-family indices on a Gamma_D plane
  bool constrained(int m, int64_t ix, int64_t iy, int64_t iz, uint32_t gamma_d) const;
};

// dense small 1D matrix
struct Mat1 {
  int rows = 0, cols = 0;
  std::vector<double> v;
  double operator()(int i, int j) const { return v[(size_t)i * cols + j]; }
};

struct Term {
  int mout, min;        // output / input component
  int coef;             // 0: alpha, 1: beta
  double c;             // constant factor (sign * pullback constant)
  int hexp[3];          // exponents of hx, hy, hz
  int mat[3];           // indices into the 1D matrix table (x, y, z)
};

struct CellOperator {
  int k = 0, p = 1;
  std::vector<Mat1> mats;   // distinct 1D matrices
  std::vector<Term> terms;
};

// Builds the Kronecker term list for V^k (k = 0, 1, 2) with structurally-zero 1D entries
// (B-hat off diag+(0,p), A-hat interior off-diagonal, D-hat interior columns off-diagonal)
// set to exact zero (eq:fdmbasis, eq:gradbasis).
CellOperator build_cell_operator(int k, int p);

// Cell-local dense-free sparse cell matrix for one Cartesian cell: entries (row, col, valK, valM)
// with A_K = alpha * K + beta * M, local order component-major then z, y, x.
struct CellEntries {
  std::vector<int> row, col;
  std::vector<double> kval, mval;
};
CellEntries cartesian_cell_entries(const CellOperator& op, const Space& sp, double hx, double hy, double hz);

// Auxiliary operator P_K for k = 0 on a trilinear cell (eq:sum-factorization_approx P:732-739):
// returns entries on the structural pattern (row, col, val) with alpha, beta folded in.
// w_int (optional, 3 (p-1)^3 doubles): the interior values of the three stiffness diagonals,
// w_int[m][(k-1, j-1, i-1)] = diag(M-bar^1_alpha)_m at the DP index of direction m equal to the
// interior index: every interior-to-face coupling of P_K is (D_ii w) D_i{0,p} (one term).
void aux_cell_entries(int p, const double Xc[8][3], double alpha, double beta, CellEntries& out,
                      double* w_int = nullptr);

// The same operator split into its geometry-dependent and geometry-independent parts (cached per
// p): four sum-factorised diagonals per cell (d0: (l,j,i) n^3; d1_x: n*n*p, d1_y: n*p*n,
// d1_z: p*n*n, concatenated at off[0..3]) and the entry map: entry t (in (row, col) order) =
// sum over its terms k of (ta[k] * diag[tg[k]]) * tc[k].  aux_cell_entries = diagonals + map.
struct AuxTables {
  int p = 0, nq = 0;
  std::vector<double> xq, wq;      // GLL rule, nq points (reading G1/G2)
  std::vector<double> sb2, r2;     // squared broken P basis (nq x n) and DP basis (nq x p)
  int off[4] = {0, 0, 0, 0}, ndiag = 0;
  std::vector<int> row, col, tptr, tg;
  std::vector<double> ta, tc;
};
const AuxTables& aux_tables(int p);
void aux_cell_diagonals(const AuxTables& T, const double Xc[8][3], double alpha, double beta, double* diag);
void aux_entries_from_diagonals(const AuxTables& T, const double* diag, double* vals);
void aux_interior_weights(const AuxTables& T, const double* diag, double* w_int);

}  // namespace rm
