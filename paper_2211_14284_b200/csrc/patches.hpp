// Star patches, their matrices A_i = R_i A R_i^T or
// R_i P R_i^T (auxiliary operator) and their exact / incomplete factorizations
// (P:1131-1166), packed for the batched patch-solve kernel.
//
// Every patch solve computes x = A_i^{-1} b through a block elimination
//   level 0: cell-interior DoFs (block diagonal with blocks <= 3x3 on Cartesian cells and for
//            the auxiliary operator),
//   levels 1..: independent sets of the current Schur complement (diagonal pivots),
//   final:  the remaining Schur complement, either inverted exactly (dense, packed lower
//           triangle of the symmetric inverse; exact Cholesky family cfg1-4) or factorised by
//           ICC(0) on its own pattern (= ICC on the static-condensation pattern, cfg5).
// With exact elimination this equals A_i^{-1} b up to rounding; with ICC it is the ICC-SC
// factorization of P:1142-1151 (interiors first, pinned interface order, reading G6).
#pragma once
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "model.hpp"

namespace rm {

struct Sliced {            // sliced-ELL block, slice height 32; rows are positions [r0, r0+nrows)
  int r0 = 0, nrows = 0;
  std::vector<int> slice_w, slice_off;   // per slice: width, element offset
  std::vector<uint16_t> cols;            // element -> column position (padding: column 0, value 0)
  int64_t nelem = 0;
  int64_t vofs = 0;                      // value offset inside a patch value block
  std::vector<std::vector<int>> rowcols; // host: structural columns per row
};

struct Blocks {             // pivot blocks of one level, thread-per-block layout
  int nblk = 0, bs = 1;                  // bs = largest block size (1..3); smaller blocks padded
  std::vector<uint16_t> mem;             // [slot][block] member positions, 0xFFFF = padding
  int64_t vofs = 0;                      // values: [bs(bs+1)/2][nblk] lower Cholesky factor, diag inverted
  int64_t nval() const { return (int64_t)nblk * bs * (bs + 1) / 2; }
};

// One elimination level in Cholesky form: with the pivot blocks P_EE = L L^T,
//   forward  y_E = L^{-1} v_E,  v_R -= M y_E           (M = P_RE L^{-T}, sliced by R rows: w)
//   backward x_E = L^{-T} (y_E - M^T x_R)              (M^T sliced by E rows: wt)
// i.e. exactly the Cholesky factorization of the patch matrix with E eliminated first.
struct Level {
  int e0 = 0, e1 = 0;                    // E = positions [e0, e1), R = [e1, n)
  std::vector<std::vector<int>> blocks;  // pivot blocks (positions), sizes 1..3
  Blocks blk;
  Sliced w, wt;
};

enum FinalKind { FINAL_DENSE_INV = 0, FINAL_ICC = 1 };

struct ClassProgram {
  int n = 0;
  std::vector<int> offs;                 // relative global offset per position
  std::vector<int> group;                // 0 interior, 1 face, 2 edge, 3 vertex (per position)
  std::vector<int> comp;                 // component per position
  std::vector<int> slot_dc[3];           // cell offset of each star cell slot relative to the anchor cell
  std::vector<std::vector<int>> slot_map;// [slot][cell-local dof] -> position or -1
  std::vector<Level> lev;
  int m = 0;                             // final block = positions [n-m, n)
  int final_kind = FINAL_DENSE_INV;
  int64_t vofs_final = 0;
  // ICC final block: CSR (rows = final positions, lower incl. diagonal), diagonal stored inverted
  std::vector<int> icc_rowptr, icc_col;              // forward: rows of L
  std::vector<int> icc_level_ptr, icc_level_rows;    // forward level schedule
  std::vector<int> icct_rowptr, icct_col, icct_src;  // backward: rows of L^T (src = index into L values)
  std::vector<int> icct_level_ptr, icct_level_rows;
  int64_t nvals = 0;                     // doubles per patch value block
  // structural pattern of the patch matrix (CSR over positions)
  std::vector<int> prow, pcol;
};

struct PatchFamily {
  Space sp;
  int dim = 0;                    // entity dimension of the stars
  uint32_t gamma_d = 0;
  int factorization = 0;          // 0 exact, 1 icc_sc
  std::vector<ClassProgram> classes;
  // patches
  std::vector<int> pclass;        // per patch
  std::vector<int64_t> pbase;     // per patch global base index
  std::vector<int64_t> pvals;     // per patch value block offset (doubles), dedup'd
  std::vector<int> pcolor;
  int ncolors = 0;
  std::vector<double> values;     // all value blocks
  double sigma_max = 0.0;         // largest ICC restart shift used (reading G7)
  int64_t nfactors = 0;           // distinct value blocks
  std::string err;
};

struct SetupInput {
  int k, p, n[3];
  uint32_t gamma_d;
  const double* coords;           // (nz+1)(ny+1)(nx+1)*3 or null
  const double* alpha;            // per cell (n_alpha == ncells) or constant
  const double* beta;
  int64_t n_alpha, n_beta;
  int dim;                        // star dimension
  int factorization;              // 0 exact, 1 icc_sc
  int interior_only;
  bool cartesian;                 // all cells axis-aligned
  const double* hx; const double* hy; const double* hz;   // per-direction cell sizes (cartesian)
};

// Builds the full patch family. Throws std::runtime_error with a message on failure.
std::unique_ptr<PatchFamily> build_patch_family(const SetupInput& in);

}  // namespace rm
