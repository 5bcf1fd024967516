// Device-side data structures shared by the kernels and the host launcher (abi.cpp).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

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
  unsigned gamma_d;
  OpTerm terms[RM_MAXTERMS];
  // k = 0: the two 1D matrices of the H(grad) operator, B-hat and A-hat = D-hat^T D-hat,
  // (p+1)^2 row-major with structural zeros exact (used by the specialised apply_q kernel)
  double Bh[RM_MAXP1 * RM_MAXP1], Ah[RM_MAXP1 * RM_MAXP1];
  short rowptr[RM_MAXMATS][RM_MAXP1 + 1];
  unsigned char col[RM_MAXMATS][RM_MAXMATNZ];
  double val[RM_MAXMATS][RM_MAXMATNZ];
};

// ---------------------------------------------------------------- patch programs
struct DSliced {
  int r0, nrows, nslices, pad;
  const int* sw;
  const int* soff;
  const uint16_t* cols;
  long long vofs;
};
struct DBlocks { int nblk, bs; const uint16_t* mem; long long vofs; };
struct DLevel { int e0, e1; DBlocks blk; DSliced w, wt; };
struct DClass {
  int n, nlev, m, final_kind;
  const int* offs;
  const unsigned char* comp;
  DLevel lev[RM_MAXLEV];
  long long vofs_final;
  int icc_nlev, icct_nlev, icc_nnz, pad;
  const int *icc_rowptr, *icc_col, *icc_lptr, *icc_lrows;
  const int *icct_rowptr, *icct_col, *icct_lptr, *icct_lrows;
};

// launchers (kernels.cu)
cudaError_t launch_apply_cartesian(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                                   const double* hpow, const double* u, const double* f, double* out,
                                   long long ndof, cudaStream_t st, int* nlaunch);
cudaError_t launch_patch_solve(const DClass* classes, const int* pclass, const long long* pbase,
                               const long long* pvals, const double* vals, const double* r, double* u,
                               double omega, int npatch, size_t smem_bytes, cudaStream_t st);
// dynamic shared memory of the patch kernel for a class with n DoFs and max_aux scratch doubles
size_t patch_solve_smem_bytes(int n, int max_aux);
constexpr int RM_PATCH_CONSUMER_WARPS = 8;
cudaError_t launch_hiptmair_DT(int k, int p, const int* n, unsigned gamma_d, const double* Dh,
                               const double* r, double* t, cudaStream_t st);
cudaError_t launch_hiptmair_D_add(int k, int p, const int* n, unsigned gamma_d, const double* Dh,
                                  const double* s, double* u, double omega, cudaStream_t st);
// y = a*x + b*y ; dot products with deterministic two-stage reduction
cudaError_t launch_axpby(long long n, double a, const double* x, double b, double* y, cudaStream_t st);
cudaError_t launch_dot(long long n, const double* x, const double* y, double* partial, double* out, cudaStream_t st);
cudaError_t launch_pcg_update(long long n, const double* alpha_num, const double* alpha_den, const double* p,
                              const double* q, double* x, double* r, cudaStream_t st);
cudaError_t launch_pcg_pupdate(long long n, const double* rz_new, const double* rz_old, const double* z,
                               double* p, cudaStream_t st);

}  // namespace rm
