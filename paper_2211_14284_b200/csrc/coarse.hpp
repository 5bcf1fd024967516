// The p = 1 coarse level of eq:asm-afw / eq:asm-hiptmair: A_0 = a^k rediscretised
// with the lowest-order element, R_0 = the transpose of the embedding V^k_{h,1} -> V^k_{h,p} in
// the FDM reference values, and a direct solve of A_0 (host setup; device solve in coarse.cu).
//
// Direct solver: the coarse DoFs are grouped by their z index (block j = the P-family plane j and
// the DP-family layer j of every component), so a cell layer couples blocks j and j + 1 only and
// A_0 is block tridiagonal.  Block Cholesky (host, untimed setup):
//   S_j = A_jj - L_{j,j-1} L_{j,j-1}^T,  L_jj = chol(S_j),  L_{j+1,j} = A_{j+1,j} L_jj^{-T};
// the device solve streams Linv_j = L_jj^{-1}, its transpose and L_{j+1,j} (dense, row-major).
#pragma once
#include <cstdint>
#include <vector>

#include "model.hpp"

namespace rm {

struct CoarseSetupInput {
  int k, p, n[3];
  uint32_t gamma_d;
  const double* coords;   // (nz+1)(ny+1)(nx+1)*3 or null (uniform unit-cube grid)
  bool cartesian;
  const double *hx, *hy, *hz;
  const double *alpha, *beta;
  int64_t n_alpha, n_beta;
};

struct CoarseFactor {
  Space sp1;                              // V^k_{h,1}
  int64_t ndof1 = 0, nfree1 = 0;
  std::vector<long long> perm;            // block order -> coarse layout index
  std::vector<uint8_t> cmask;             // block order: 1 = constrained (held at zero)
  std::vector<int> bstart;                // nb + 1 offsets of the blocks in block order
  // per block j: Linv_j (m_j x m_j), LinvT_j, and for j < nb - 1: Lsub_j = L_{j+1,j} (m_{j+1} x m_j)
  // and LsubT_j (m_j x m_{j+1}); all row-major, concatenated in `vals` at the offsets below
  std::vector<long long> o_linv, o_linvt, o_lsub, o_lsubt;
  std::vector<double> vals;
  // 1D embedding of the P family: interior coefficients e0[a] = (s_a, (1-x)/2), e1[a] = (s_a, (1+x)/2)
  double e0[16] = {0}, e1[16] = {0};
};

// Builds A_0 and factors it (throws std::runtime_error on a non-positive pivot)
void build_coarse(const CoarseSetupInput& in, CoarseFactor& out);

}  // namespace rm
