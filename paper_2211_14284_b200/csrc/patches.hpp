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

// One elimination level.  With the pivot blocks P_EE = L L^T (stored: L with inverted diagonal),
//   forward  y^_E = L^{-T} L^{-1} v_E = P_EE^{-1} v_E  (in place),   v_R -= P_RE y^_E     (w)
//   backward x_E  = y^_E - W^ x_R,   W^ = P_EE^{-1} P_ER  (prescaled on the host)        (wt)
// i.e. block Gaussian elimination of the patch matrix with E eliminated first; the backward pass
// needs no pivots.
struct Level {
  int e0 = 0, e1 = 0;                    // E = positions [e0, e1), R = [e1, n)
  std::vector<std::vector<int>> blocks;  // pivot blocks (positions), sizes 1..3
  Blocks blk;
  Sliced w, wt;
};

enum FinalKind { FINAL_DENSE_INV = 0, FINAL_ICC = 1 };

// Stream layout.  A patch is processed as a sequence of PIECES, each streamed HBM/L2 -> shared
// memory by one producer warp with bulk copies (TMA) while the consumer warps work on earlier
// pieces.  A piece = a metadata block (from the class's L2-resident meta stream: a 16-byte
// header {a0, a1, e0, mbytes} then indices) followed by its factor values (from the patch's
// value block, <= kPieceMax doubles, 16-byte aligned), so the consumers never chase a global
// pointer.  Order of the pieces (= order of the values in the patch value block):
//   forward:  for l = 0..L-1: PIV(l) pieces (block members + pivots), W(l) pieces
//   final:    TILE pieces (row-major over I, J <= I; diagonal tiles packed lower, 528 doubles)
//             or ICC forward-row pieces then ICC backward-row pieces (split at level boundaries)
//   backward: for l = L-1..0: WT(l) pieces  (pivots and members reused from a shared copy)
// (gather / scatter use the class's codes (offs << 2 | comp) from global memory; the dense-tile
// units form their own channel, consumed by the tile warps only)
enum PieceKind { PK_PIV = 0, PK_W = 1, PK_TILE = 2, PK_ICCF = 3, PK_ICCB = 4, PK_WT = 5, PK_FINAL = 6, PK_ZERO = 7 };
constexpr int kPieceMax = 2048;      // doubles (16 KB) of values per piece
constexpr int kIccRows = 32;      // rows per ICC chunk: one row per lane of the warp that takes it
// chunks per ICC piece: chunk c of the level's piece k -> warp c + kIccChunks (k % (8 / kIccChunks));
// measured on cfg5 (chunks / value cap -> patch kernel): 8 / 8192 -> 1.34 ms, 4 / 4096 -> 1.27 ms,
// 2 / 2048 -> 1.56 ms (ring prefetch depth vs. number of piece headers walked)
#ifndef RM_ICC_CHUNKS            // tuning knobs (-D): chunks per ICC piece, values per ICC piece
#define RM_ICC_CHUNKS 4
#endif
#ifndef RM_ICC_PIECE_VALS
#define RM_ICC_PIECE_VALS 8192   // measured (cfg5 patch kernel): 2048 1.75, 3072 1.42, 4096 1.28, 6144 1.32, 8192 1.266, 12288 1.266, 16384 1.269 ms
#endif
constexpr int kIccChunks = RM_ICC_CHUNKS;
constexpr int kIccPieceVals = RM_ICC_PIECE_VALS;   // values per ICC piece (several pieces in flight in the ring)
struct IccChunk { int r0, cnt, L, sofs; };   // level-ordered rows [r0, r0+cnt), longest off-diag row, slot offset
constexpr int kGatherMax = 2048;     // positions per GATHER/SCATTER piece
// Dense tiles (32x32 blocks of the final block's inverse) in LANE-BLOCK order: lane l = 4a + b
// owns rows 4a..4a+3 and columns 8b..8b+7; step k (0..15) holds its elements (row 4a + k/4,
// columns 8b + 2(k%4) + {0,1}); the stream stores step k of all lanes contiguously
// (16 bytes per lane: one conflict-free LDS.128).  Diagonal tiles keep only the 20 sub-blocks
// (b <= a/2) that touch the lower triangle, with the strictly upper part zero and the diagonal
// halved, so that the tile equals L' + L'^T and one row-sum + column-sum pass applies it.
constexpr int kTileDiag = 640;       // 16 steps x 20 lanes x 2
inline int tile_pos_full(int r, int c) {
  const int l = (r >> 2) * 4 + (c >> 3), k = (r & 3) * 4 + ((c & 7) >> 1);
  return (k * 32 + l) * 2 + (c & 1);
}
inline int tile_diag_slot(int a, int b) { return a + (a >> 1) * ((a - 1) >> 1) + b; }   // b <= a/2
inline int tile_pos_diag(int r, int c) {   // c <= r
  const int a = r >> 2, b = c >> 3, k = (r & 3) * 4 + ((c & 7) >> 1);
  return (k * 20 + tile_diag_slot(a, b)) * 2 + (c & 1);
}
struct Piece {
  int kind, lev;
  int a0, a1;     // PIV: blocks; W/WT: slices; TILE: I, J; ICC: level-ordered rows; GATHER: positions
  int e0;         // W/WT: first element of the sliced array; ICC: longest off-diagonal row (L)
  int sofs;       // stream offset (doubles) inside the patch value block
  int nd;         // doubles (even)
  int cofs;       // source offset inside the canonical block (host packing only)
  int mofs = 0, mbytes = 0;   // metadata block inside the class meta stream (bytes, 16-aligned)
};

// Transfer unit: consecutive pieces moved by one mbarrier round trip (<= kUnitVals doubles of
// values and <= kUnitMeta bytes of metadata; the ring holds [metas][values] of the unit).
#ifndef RM_UNIT_VALS               // tuning knobs (-D): values per transfer unit of each channel
#define RM_UNIT_VALS 2048
#endif
#ifndef RM_UNIT_VALS_TILE
#define RM_UNIT_VALS_TILE 4096
#endif
constexpr int kUnitVals = RM_UNIT_VALS;             // sparse-channel units (16 KB of values)
constexpr int kUnitValsTile = RM_UNIT_VALS_TILE;    // tile-channel units (32 KB)
constexpr int kUnitMeta = 16384;
struct Unit { int p0, np, mofs, mbytes, sofs, nd; };

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
  // ICC in level order (stream layout): q = level-ordered row index; rp over values in stream order
  std::vector<int> iccf_row, iccf_rp, iccf_col, iccf_src, iccf_lpiece;   // forward (diag last)
  std::vector<int> iccb_row, iccb_rp, iccb_col, iccb_src, iccb_lpiece;   // backward (diag first)
  std::vector<IccChunk> iccf_chunk, iccb_chunk;   // pieces hold chunk ranges [a0, a1)
  int64_t nnzL = 0;                      // SURVEY 8(d) algorithmic factor size: nnz of the exact Cholesky
                                         // factor in the pinned order (G6), or of the ICC-SC mask
  int64_t nvals_canon = 0;               // doubles per canonical (factorization-order) block
  int64_t nvals = 0;                     // doubles per patch value block (stream layout)
  // stream pieces and the piece ranges of each section
  std::vector<Piece> pieces;
  std::vector<int> piv_b, w_b, w_e, wt_b, wt_e;   // per level: piece ranges (PIV(l) = [piv_b, w_b))
  int tile_p0 = 0, tile_p1 = 0;
  std::vector<int> piv_per, piv_ofs, mem_ofs;   // per level: blocks per PIV piece, shared-memory offsets
  int piv_total = 0;                     // doubles of the shared-memory pivot copy
  int mem_total = 0;                     // uint16 of the shared-memory block-member copy
  int ngs = 0;                           // GATHER pieces (= SCATTER pieces)
  std::vector<uint8_t> meta;             // class meta stream (pieces' metadata blocks)
  std::vector<Unit> units;
  int tu0 = 0, tu1 = 0;                  // units of the dense-tile phase (tile channel)
  int uf0 = 0, uf1 = 0;                  // final segment units [uf0, uf1) (tiles or ICC)
  // window box: per component the window origin relative to the anchor and its extent; per
  // position its coordinates inside the window, its box index, and the box entries to zero
  int wlo[3][3] = {{0}}, wext[3][3] = {{0}};
  int xshift[3] = {0, 0, 0};             // x-parity twin: box x index shifted by one (odd origins)
  bool sc = false;                       // cell interiors condensed per cell (ICC-SC families)
  int sub_org[3][3] = {{0}}, sub_ext[3][3] = {{0}};   // sub-boxes: origin rel. anchor, extent
  std::vector<int> psub;                 // per position: sub-box (-1: condensed interior)
  std::vector<int> pcoord, bidx, zlist;
  // structural pattern of the patch matrix (CSR over positions)
  std::vector<int> prow, pcol;
  // exact programs: per final row, the [lo, hi) range (final indices) of its independent block
  std::vector<int> frange;
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
  std::vector<int> porig;         // per patch [comp][dir]: window box origin (global index)
  int nsub = 0;                   // sub-boxes: components, or the 3 anchor planes (sc)
  int sub_comp[3] = {0, 0, 0};    // component of each sub-box
  int box[3][3] = {{0}};          // per sub-box extents (x even)
  int boff[4] = {0, 0, 0, 0};     // sub-box offsets inside the box vector
  // static condensation of the cell interiors (sc): per cell, interior DoFs (i,j,k) in 1..p-1
  // (x fastest): inverse diagonal, couplings to the 6 face DoFs [x-, x+, y-, y+, z-, z+], and the
  // number of patches containing the cell
  std::vector<double> sc_dinv, sc_c;
  std::vector<int> sc_nk;
  // compressed couplings (trilinear auxiliary operator): per cell the three interior stiffness
  // weights w[K][m][I] (sc_c empty); coupling to face 2m (+1) = (D_ii w) D_i0 (D_ip), i the
  // interior index along m -- bitwise the assembled value (model.hpp aux_cell_entries)
  std::vector<double> sc_w;
  std::vector<double> sc_kd, sc_k0, sc_kp;   // D_ii, D_i0, D_ip (i = 0..p)
  double sc_coupling(int64_t K, int f, int I, int ni, int iline) const {
    if (sc_w.empty()) return sc_c[((size_t)K * 6 + f) * ni + I];
    const double w = sc_w[((size_t)K * 3 + f / 2) * ni + I];
    return (sc_kd[iline] * w) * ((f & 1) ? sc_kp[iline] : sc_k0[iline]);
  }
  bool sc_pre = false;            // the static-condensation PRE step runs outside the patch kernel (sc programs)
  int box_total = 0;
  double sigma_max = 0.0;         // largest ICC restart shift used (reading G7)
  int64_t nfactors = 0;           // distinct value blocks
  int64_t nnzL_total = 0;         // sum over patches of ClassProgram::nnzL (algorithmic factor entries)
  int64_t unique_value_bytes = 0; // bytes of the distinct value blocks (what HBM holds)
  std::string err;
  // ---- device-resident numeric setup (SetupInput::defer_numeric): the host
  // builds the symbolic programs only; values / sc_dinv / sc_c / sc_w are left empty and computed
  // on the GPU (dsetup.cu) from these inputs
  bool deferred = false;
  int64_t nvalues = 0;                    // doubles of all distinct value blocks (host offsets)
  std::vector<int> fclass;                // per distinct block: class of its representative patch
  std::vector<int64_t> foff;              // per distinct block: host value offset
  std::vector<int> fcells;                // per distinct block: kMaxSlots star cells in slot order (-1 unused)
  std::vector<int> cell_rows, cell_cols;  // cell-matrix pattern (entry order of CellEntries)
  bool cartesian = true;
  std::vector<double> cset_k, cset_m;     // Cartesian: per distinct (hx, hy, hz) the K / M entries
  std::vector<int> cell_set;              // Cartesian: per cell its entry set
  std::vector<double> cell_alpha, cell_beta;   // per cell
  std::vector<double> coords;             // trilinear: (nz+1)(ny+1)(nx+1)*3 vertex coordinates
};

constexpr int kMaxSlots = 8;   // star cells per patch (vertex stars)

// Device numeric program of one class (host arrays; dsetup.cu uploads them).  Every value of the
// class's canonical block is produced by the same block elimination as the host factorization
// (factor_patch): assembly of P on the class pattern, level-0 pivot blocks, the interface Schur
// complement S, then either a dense Cholesky S = L L^T in position order (levels >= 1 read off L:
// pivots 1/L_qq, W = L_rq L_qq, W^ = L_rq / L_qq; the final block's inverse from L_FF) or ICC(0) on
// the final pattern; finally the canonical -> stream permutation (stream_map).
struct NumProg {
  int n = 0, nI = 0, nG = 0, m = 0, nnzP = 0, final_kind = 0;
  int nb0 = 0, bs0 = 1;                   // level-0 blocks and their padded size
  int64_t blk0_vofs = 0, vofs_final = 0, ncanon = 0, nvals = 0;
  std::vector<int> asm_ptr, asm_src;      // per P entry: terms slot * ne + t (host summation order)
  std::vector<int> pdiag;                 // per position: CSR index of the diagonal
  std::vector<int> b0;                    // per block 12 ints: bs, mem[3], lcsr[6] (lower, row-major), nb0, nb1
  std::vector<int> nbr;                   // per neighbour record 7 ints: r - nI, csr P(r, b_j) [3], canon W^ (b_j, r) [3]
  std::vector<int> w0;                    // pairs: canon index, CSR index (level-0 W = P_RE)
  std::vector<int> st_idx, st_csr, st_ptr, st_src;   // S targets: index (dense a*nG+c | ICC entry), P entry, pairs of records
  std::vector<int> rec;                   // exact levels >= 1: (canon, op, a, b), op 0 = 1/L_bb, 1 = L_ab L_bb, 2 = L_ab / L_bb
  std::vector<int> icc_rowptr, icc_col, icc_lptr, icc_lrows, icct_src;
  std::vector<int> smap;                  // per stream slot: canon c (>= 0), -1 zero, -2 - c (0.5 * canon c)
};
// cell_rows / cell_cols: the cell-matrix pattern; ne = its size
void build_numeric_program(const ClassProgram& C, const std::vector<int>& cell_rows,
                           const std::vector<int>& cell_cols, NumProg& out);

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
  int zv_lo = 0, zv_hi = 1 << 30;   // vertex stars kept: z vertex layers [zv_lo, zv_hi) (z-slab ownership)
  int orient = -1;                  // edge / face stars: keep one orientation (edge direction / face normal), -1 = all
  bool defer_numeric = false;       // device-resident numeric setup (PatchFamily::deferred)
  bool interface_only = false;      // SC-PH: the patches' interior corrections are dropped (their interface
                                    // part is the interface Schur complement solve, eq:LDU)
  bool sc_decomposition = false;    // SC-PAFW (eq:sc-asm-afw, k = 0): interface corrections from the patches, cell
                                    // interiors once afterwards (c_I = A_II^-1 (r_I - A_IG c_G), n_K = 1)
};

// Builds the full patch family. Throws std::runtime_error with a message on failure.
std::unique_ptr<PatchFamily> build_patch_family(const SetupInput& in);

}  // namespace rm
