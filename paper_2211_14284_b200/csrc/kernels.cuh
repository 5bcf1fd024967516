// Device-side data structures shared by the kernels and the host launcher (abi.cpp).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#include "exp_env.hpp"

namespace rm {


#define RM_MAXLEV 8
#define RM_MAXTERMS 16
#define RM_MAXMATS 12
#define RM_MAXMATNZ 160
#define RM_MAXP1 16   // p + 1 <= 16  (p <= 15)

// ---------------------------------------------------------------- Cartesian operator params
struct OpTerm { int mout, min, coef; int hexp[3]; int mat[3]; double c; };
struct OpParams {
  int k, p, ncomp, nterms, nmats;
  int n[3];                       // cells per direction
  int fam[3][3];                  // [comp][dir]
  long long len[3][3];            // [comp][dir] index lengths
  long long off[4];               // component offsets
  long long ldx_out;              // k = 0: x-stride of the output (0 = len[0][0]; the padded TMA layout)
  unsigned gamma_d;
  OpTerm terms[RM_MAXTERMS];
  // k = 0: the two 1D matrices of the H(grad) operator, B-hat and A-hat = D-hat^T D-hat,
  // (p+1)^2 row-major with structural zeros exact (used by the specialised apply_q kernel)
  double Bh[RM_MAXP1 * RM_MAXP1], Ah[RM_MAXP1 * RM_MAXP1];
  // D-hat (p x (p+1), row-major, structural zeros exact): the H(curl) / H(div) kernels
  double Dh[RM_MAXP1 * RM_MAXP1];
  short rowptr[RM_MAXMATS][RM_MAXP1 + 1];
  unsigned char col[RM_MAXMATS][RM_MAXMATNZ];
  double val[RM_MAXMATS][RM_MAXMATNZ];
};

// ---------------------------------------------------------------- patch programs
// (host counterparts and the stream layout: patches.hpp)
// producer's view of a transfer unit: meta bytes [mofs, mofs + (mb_np & 0xFFFF)) of the class
// meta stream, values [sofs, sofs + nd) of the patch value block, np = (mb_np >> 16) & 0x7FFF
// pieces, channel = bit 31 (1 = dense-tile channel)
struct DUnit { int mofs, mb_np, sofs, nd; };
struct DSliced { int r0, nrows; };
struct DBlocks { int nblk, bs; };
struct DLevel {
  int e0, e1;
  DBlocks blk;
  DSliced w, wt;
  int piv_b, w_b, w_e, wt_b, wt_e, piv_per, piv_ofs, mem_ofs;
};
// Per class: the elimination program's shape (levels, piece ranges); every per-DoF / per-entry
// index travels in the pieces' metadata blocks (class meta stream), not here.
struct DClass {
  int n, nlev, m, final_kind;
  DLevel lev[RM_MAXLEV];
  const DUnit* units;
  const unsigned char* meta;     // class meta stream (L2-resident)
  int nunits, ngs, tile_p0, tile_p1, iccf_nlev, iccb_nlev;
  int uf0, uf1, fin_tiles, pad2;  // final segment units [uf0, uf1); fin_tiles: on the tile channel
  const int *iccf_lp, *iccb_lp;  // per ICC level: first piece (size nlev + 1)
  const int2* ptab;              // per piece {meta offset, value offset} (class-batched kernel)
  int npieces, pad3;
  const int2* frange;            // per final row: [lo, hi) of its independent block (null: the whole block)
};
constexpr int RM_MAXCOLORS = 12;
struct ColorStarts { int ncolors; int start[RM_MAXCOLORS + 1]; };

// trilinear H(grad) apply (apply_tri.cu): 1D tables (S, D at the n_q GLL points, nodes, weights)
// in a device buffer [S (nq x (p+1)) | D (nq x (p+1)) | x (nq) | w (nq)]
struct TriParams {
  int p, nq, n[3];
  long long Lx, Ly, Lz;
  unsigned gamma_d;
  long long ldx_out;   // x-stride of the output (0 = Lx; the padded TMA layout)
  // even / odd split of the x contractions (nq even): the FDM basis functions have definite
  // parity (E_0 = s_0 + s_p, O_0 = s_0 - s_p, interior s_j even or odd) and the GLL points come in
  // mirror pairs, so each 24 x 16 contraction splits into two 12 x 8 ones.  xsig[pos] = the
  // original x index at even/odd position pos (0: E_0, 8: O_0, -1: padding); the tables follow the
  // standard ones in `tabs` (S_E, S_O, D_E, D_O at the left points, 12 x 8 each, zero padded)
  int eo, ne;          // even/odd path on; number of point pairs
  int xsig[16];
  int skip_gather;     // launch_apply_trilinear stops after the apply (the SC-fused residual path)
};
// optional hooks around a launcher's main kernel (the ABI records CUDA events there for the
// per-kernel timing phases of rm_timing_read)
struct KTimer {
  void (*begin)(void*);
  void (*end)(void*);
  void* arg;
};

cudaError_t launch_apply_trilinear(const TriParams& tp, const double* tabs, const double* X, const double* alpha,
                                   const double* beta, int coef_const, const double* u, const double* f, double* out,
                                   double sign, double* cellbuf, cudaStream_t st, int* nlaunch,
                                   const KTimer* kt = nullptr);
// doubles of the per-cell result buffer the trilinear apply needs (apply_tri.cu)
size_t tri_cellbuf_doubles(const TriParams& tp);
// skeleton gather of the SC-fused residual (ICC-SC, one rank): skeleton DoFs only, minus the
// condensation line sums fb of the face-interior DoFs (apply_tri.cu tri_gather_sc_kernel)
cudaError_t launch_skeleton_gather_sc(const TriParams& tp, const double* cellbuf, const double* f, double* out,
                                      double sign, const double* fb, cudaStream_t st);
// H(curl) / H(div) Cartesian apply (apply_kform.cu): one launch over all cells, interior entries
// stored as f + sign A u, skeleton entries through `cellbuf` (kform_cellbuf_doubles) and a gather
cudaError_t launch_apply_kform(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                               const double* hpow, const double* u, const double* f, double* out, long long ndof,
                               double* cellbuf, cudaStream_t st, int* nlaunch, const KTimer* kt);
size_t kform_cellbuf_doubles(int k, int p, const int* n);
// p = 1 coarse level (coarse.cu, host data from coarse.hpp): z += R_0^T A_0^{-1} R_0 r
struct CoarseLaunch {
  int p, ncomp, n[3], fam[3][3];
  long long len[3][3], off[4];      // fine layout (x, y, z extents per component)
  long long len1[3][3], off1[4];    // coarse layout
  long long ndof1;
  int nb;                           // z blocks of A_0
  const int* bstart;                // HOST: nb + 1 block offsets (block order)
  const long long *o_linv, *o_linvt, *o_lsub, *o_lsubt;   // HOST: offsets into vals
  const long long* perm;            // device: block order -> coarse layout
  const unsigned char* cmask;       // device: block order constrained flags
  const double* vals;               // device: block factors
  double *xc, *b, *y, *t;           // device: coarse vectors (ndof1)
  double *tA, *tB;                  // device: transfer temporaries (fine size)
  double e0[16], e1[16];            // 1D embedding, interior rows
};
cudaError_t launch_coarse_correct(const CoarseLaunch& L, const double* r, double* z, cudaStream_t st);
// out = f (or 0) with constrained entries zeroed (apply.cu)
cudaError_t launch_apply_init(const OpParams& op, const double* f, double* out, long long ndof, cudaStream_t st);

// launchers (kernels.cu)
cudaError_t launch_apply_cartesian(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                                   const double* hpow, const double* u, const double* f, double* out,
                                   long long ndof, cudaStream_t st, int* nlaunch, const KTimer* kt = nullptr,
                                   double* cellbuf = nullptr);
// out = f + sign * (sum of the cell-buffer skeleton entries | the stored interior values), constrained 0
// (the gather of the cell-buffer applies, apply_tri.cu)
cudaError_t launch_skeleton_gather(const TriParams& tp, const double* cellbuf, const double* f, double* out, double sign,
                                   cudaStream_t st);
// Padded component layout of the patch kernel's input r and correction c: x rows padded to an
// even length so that TMA tensor maps (row strides multiple of 16 bytes) can address them.
struct PadLayout {
  int ncomp;
  long long len[3][3];      // [comp][dir] unpadded extents (x, y, z)
  long long off[4];         // unpadded component offsets
  long long poff[4];        // padded component offsets
  long long lxp[3];         // padded x extents
};
struct TMaps { CUtensorMap r[3], c[3]; };   // 3D maps of the padded r / c, one per window sub-box

// One transfer of the producer's per-CTA issue lists (host-built, in consumption order): copy
// mb metadata bytes from `meta` and vb value bytes from `vals` into the channel's ring as one
// unit of np pieces.
struct XferEntry {
  const unsigned char* meta;
  const double* vals;
  unsigned mb_np;   // meta bytes | pieces << 16
  unsigned vb;      // value bytes
  unsigned long long pad;
};

// Persistent streaming patch solve over one family: patches sorted by colour, CTA b takes
// patches b, b + grid, ...; every patch works on its window box (gathered from rpad and
// reduce-added into cpad with TMA tensor copies); reduce-adds follow the colour order through
// *done (zeroed per launch).
struct PatchLaunch {
  const DClass* classes;
  const int* pclass;
  const long long* pvals;
  const int* porig;      // per patch [comp][dir] box origins
  const double* vals;
  int npatch;
  ColorStarts cs;
  unsigned* done;
  int ncomp, box[3][3], boff[4], box_total;
  int nsub, sub_comp[3];  // window sub-boxes (components, or anchor planes for static condensation)
  // static condensation of the cell interiors (ICC-SC, k = 0): per cell inverse interior
  // diagonal [ncell][(p-1)^3], face couplings [ncell][6][(p-1)^3], patches per cell
  const double* sc_dinv;
  const double* sc_c;    // [ncell][6][(p-1)^3] couplings, or null with sc_w (compressed, trilinear)
  const double* sc_w;    // [ncell][3][(p-1)^3] interior stiffness weights: coupling = (kd w) k0|kp
  double sc_kd[16], sc_k0[16], sc_kp[16];
  const int* sc_nk;
  double* sc_fb;         // per-cell face line sums of the pre step [ncell][6][(p-1)^2]
  int icc_only;          // every class ends in ICC (no dense tiles): the tile warps join the sparse warps
  int sc_pre;            // run the static-condensation pre step (sc programs); SC-PAFW with the exact
                         // program has only the post step
  int sc_p, sc_n[3];
  int n_max, piv_max, mem_max, aux_max;   // largest class: DoFs, pivot doubles, member u16, scratch doubles
  size_t smem_fixed;     // barriers + 2 boxes + aux (bytes)
  int ring_bytes;        // sparse-channel ring
  int ring_b_bytes;      // tile-channel ring
  int nbox;              // window-box buffers (2 or 3)
  int grid;
  int unit_bytes_max;    // largest transfer unit (meta + values)
  int unit_bytes_max_a, unit_bytes_max_b;   // per channel (sparse, tile)
  PadLayout pad;
  long long npad;
  double *rpad, *cpad;
  TMaps tm;
  TMaps* tm_dev;         // device copy of tm (owned by the launch plan)
  const XferEntry* xfer;         // per-CTA issue lists (sparse channel, then tile channel)
  const long long* xbeg;         // [2 * grid + 2]: CTA b's sparse list = [xbeg[2b], xbeg[2b+1]),
                                 //                tile list = [xbeg[2b+1], xbeg[2b+2])
  unsigned long long* prof;   // RM_PROFILE=1 instrumentation counters (else null)
  // Class-batched mode (families whose patches share few value blocks -- uniform Cartesian meshes,
  // cfg1/3/4): each CTA solves `batch` patches of ONE value block at once (the block is read once
  // for all of them, every elimination step has `batch` independent right-hand sides), one launch
  // per colour (patch_batch_kernel).  batch = 0: the persistent stream kernel.
  int batch, batch_nt;        // patches per CTA, threads per CTA (512: one CTA per SM, 256: two)
  const int* bpatch;          // [nbatch][batch] patch index (colour-sorted order), -1 = empty slot
  const int* bclass;          // per batch: class
  const long long* bblock;    // per batch: value-block offset in vals
  const long long* bfin;      // per batch: offset of the block's full final-block inverse in fin
  const double* fin;          // full symmetric final-block inverses, mr x mr row-major (mr = m rounded to 32)
  int bstart[RM_MAXCOLORS + 1];   // first batch of each colour
  int mr_max;
  size_t bsmem;               // dynamic shared memory of the batched kernel (bytes)
};
// shared memory of the class-batched kernel for B right-hand sides (0 if it does not fit)
constexpr int kBatchMaxPieces = 1024;   // piece table of a class, staged in shared memory
size_t patch_batch_smem(int box_total, int mr_max, int B, int NT);
// u += omega * (patch corrections of one family applied to r); r, u in the vector layout
// r_padded: r is already in the padded layout L.rpad (the apply wrote it there): no pad pass
// zero_c / combine: zero the padded correction first / add omega * c to u at the end (families
// sharing their padded buffers run back to back)
cudaError_t launch_patch_solve(const PatchLaunch& L, const double* r, double* u, double omega, cudaStream_t st,
                               const KTimer* kt = nullptr, bool r_padded = false, bool zero_c = true,
                               bool combine = true, bool sc_pre_done = false, const double* u_in = nullptr);
// (u_in: the combine writes u = u_in + omega c instead of u += omega c)
// ICC-SC pre step, part 1, on the residual of the SC-fused path: the cell-interior entries of rpad
// hold sign * (A u)_I (trilinear apply with skip_gather); r_I = f_I + rpad_I is completed in place
// and the condensation line sums go to L.sc_fb (f: the vector layout, x-stride lx)
cudaError_t launch_sc_pre_fused(const PatchLaunch& L, const double* f, long long lx, cudaStream_t st);
// u += omega * unpad(cpad) (the combine step of launch_patch_solve, on its own)
cudaError_t launch_patch_combine(const PatchLaunch& L, double* u, double omega, cudaStream_t st);
// shared-memory plan, grid size and tensor maps (rpad / cpad must be allocated)
cudaError_t plan_patch_solve(PatchLaunch& L);
constexpr int RM_PATCH_CONSUMER_WARPS = 8;
constexpr int RM_PATCH_TILE_WARPS = 4;   // consumer warps sharing the dense tiles (5 measured: cfg2 patch kernel 3.665 vs 3.658 ms)
cudaError_t launch_hiptmair_DT(int k, int p, const int* n, unsigned gamma_d, const double* Dh,
                               const double* r, double* t, cudaStream_t st);
cudaError_t launch_hiptmair_D_add(int k, int p, const int* n, unsigned gamma_d, const double* Dh,
                                  const double* s, double* u, double omega, cudaStream_t st);
// SC-PH (sc_ph.cu): layout of V^k, and the cell-interior blocks (<= 3x3) of the Cartesian cell
// operator: members as codes comp << 24 | c << 16 | b << 8 | a (cell-local x, y, z indices), per
// cell-size set the lower K and M entries (6 per block, row-major lower)
struct ScPhParams {
  int p, ncomp, n[3], nblk;
  int fam[3][3];                  // [comp][dir], 0 = P family
  long long len[3][3], off[4];
};
cudaError_t launch_scph_interior_solve(const ScPhParams& P, const double* alpha, const double* beta, int coef_const,
                                       const int* cell_set, const int* bmem, const double* bK, const double* bM,
                                       const double* x, double* y, cudaStream_t st);
cudaError_t launch_scph_vec(const ScPhParams& P, int mode, const double* a, const double* b, const double* c,
                            double* out, double omega, cudaStream_t st);
// y = a*x + b*y ; dot products with deterministic two-stage reduction
cudaError_t launch_axpby(long long n, double a, const double* x, double b, double* y, cudaStream_t st);
cudaError_t launch_dot(long long n, const double* x, const double* y, double* partial, double* out, cudaStream_t st);
cudaError_t launch_pcg_update(long long n, const double* alpha_num, const double* alpha_den, const double* p,
                              const double* q, double* x, double* r, cudaStream_t st);
cudaError_t launch_pcg_pupdate(long long n, const double* rz_new, const double* rz_old, const double* z,
                               double* p, cudaStream_t st);

}  // namespace rm
