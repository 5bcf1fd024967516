/* rm.h -- C ABI of the B200-native multigrid relaxation sweep of arXiv 2211.14284
 * ("Optimal-complexity and robust multigrid relaxation for the de Rham Riesz maps").
 *
 * The operation (§3-§4):
 *   problems  beta u - div(alpha grad u) = f            (k = 0, H(grad))   eq:hgrad
 *             beta u + curl(alpha curl u) = f           (k = 1, H(curl))   eq:hcurl
 *             beta u - grad(alpha div u) = f            (k = 2, H(div))    eq:hdiv
 *   weak form a^k(v,u) = (v, beta u) + (d^k v, alpha d^k u)   eq:common_weak_formulation
 *   spaces    Q_p / NCE_p / NCF_p with the FDM basis on a logically structured hex mesh;
 *             DoFs are reference values.
 *   sweep     r = f - A u  (true A, sum-factorised, eq:sum-factorization P:690-692)
 *             u_out = u_in + omega * sum_i R_i^T A_i^{-1} R_i r          eq:asm-afw
 *             [+ omega * D (sum_j R_j^T B_j^{-1} R_j) D^T r  for the PH decomposition, eq:asm-hiptmair]
 *             with star patches and exact Cholesky or, on non-Cartesian
 *             cells, the auxiliary operator (eq:sum-factorization_approx P:732-739) with ICC on the
 *             static-condensation pattern.  rm_relax has no coarse term (reading
 *             G10); with options.coarse = 1 rm_precondition / rm_pcg use the hybrid V(1,1) cycle with
 *             the p = 1 coarse level R_0^T A_0^{-1} R_0 of eq:asm-afw.
 *
 * VECTOR LAYOUT (reading G16): component-major; each component a C-order
 * [Z][Y][X] array (X fastest).  Per direction d a component uses a P family (n_d p + 1 entries,
 * shared at multiples of p) or a DP family (n_d p entries):
 *   Q_p (P,P,P);  NCE_p x:(DP,P,P) y:(P,DP,P) z:(P,P,DP);  NCF_p x:(P,DP,DP) y:(DP,P,DP) z:(DP,DP,P).
 * A DoF is CONSTRAINED iff one of its P-family indices lies on a Gamma_D plane.
 * Inputs may hold anything in constrained entries (they are read as zero); outputs hold zero
 * in constrained entries, except rm_relax, which leaves u_out = u_in there.
 *
 * MEMORY: every vector argument of rm_apply / rm_residual / rm_relax / rm_precondition / rm_pcg
 * is an fp64 CUDA DEVICE pointer of n_local = rm_layout().n_local elements, owned by the caller
 * (e.g. a torch tensor).  The context owns every device buffer it allocates; rm_destroy frees
 * them.  Host-side arguments (coordinates, coefficients, masks, the *_host calls) are plain host
 * pointers, copied during the call.  Work is enqueued on options.stream (cudaStream_t; NULL =
 * the legacy default stream); rm_apply, rm_residual, rm_relax and rm_precondition are
 * asynchronous; rm_pcg, rm_relax_host and the query calls synchronise.
 *
 * ERRORS: every call returns an rm_status; no C++ exception crosses the ABI.  rm_last_error()
 * returns a thread-local message for the last failing call.  RM_NOT_CONVERGED from rm_pcg is a
 * report (iters == maxit), not an error.  A handle must not be used from two host threads at once.
 */
#ifndef RM_H_
#define RM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rm_ctx rm_ctx;

typedef enum { RM_HGRAD = 0, RM_HCURL = 1, RM_HDIV = 2 } rm_space;   /* form degree k */

typedef enum {
  RM_OK = 0,
  RM_NOT_CONVERGED = 1,
  RM_EINVAL = -1,     /* bad sizes, p < 1 or p > 15, bad mask, unsupported combination */
  RM_ENOMEM = -2,     /* host or device allocation failed */
  RM_ENUMERIC = -3,   /* non-positive pivot in a patch factorization (message names the patch) */
  RM_ECUDA = -4,      /* CUDA runtime error (message carries cudaGetErrorString) */
  RM_ENCCL = -5       /* NCCL error (multi-GPU) */
} rm_status;

/* decomposition: vertex stars | k-stars + potential | statically condensed vertex stars (SC-PAFW,
 * eq:sc-pafw / eq:sc-asm-afw, H(grad) only: interface corrections from the vertex-star Schur
 * complements S_v, cell interiors once, c_I = A_II^-1 (r_I - A_IG c_G)) */
enum { RM_PAFW = 0, RM_PH = 1, RM_SC_PAFW = 2, RM_SC_PH = 3 };
/* RM_SC_PH (eq:sc-ph / eq:sc-asm-hiptmair, k = 1, 2, Cartesian cells, exact factors, single rank,
 * one level): c = R_I^T A_II^-1 R_I r + R_G^T S_PH^-1 R_G r with S_PH^-1 = sum over k-stars of
 * S_i^-1 on their interface DoFs + D~ (sum over (k-1)-stars of B~_j^-1) D~^T, D~ = D_GG; the star
 * solves are the PH patch programs run on interface-only input with their interior corrections
 * dropped (eq:LDU), A_II^-1 by the <= 3x3 cell-interior blocks (remark P:1061-1066). */
enum { RM_CHOL = 0, RM_ICC_SC = 1 };                   /* patch factorization */
enum { RM_ALL_ENTITIES = 0, RM_INTERIOR_ONLY = 1 };    /* patch_entities (interior-only = test mode) */

/* Gamma_D bitmask: bit0 x=0, bit1 x=1, bit2 y=0, bit3 y=1, bit4 z=0, bit5 z=1 */
typedef struct {
  int32_t nx, ny, nz;        /* global cells per direction                                        */
  const double *coords;      /* host, (nz+1)(ny+1)(nx+1)*3, C-order [z][y][x][xyz];                */
                             /* NULL = uniform grid of the unit cube. Axis-aligned grids use the    */
                             /* Cartesian Kronecker path; any other grid is treated as trilinear.  */
  int32_t z_begin, z_end;    /* cell layers owned by this rank; [0, nz) on one GPU                 */
} rm_mesh;

typedef struct {
  int32_t decomposition;     /* RM_PAFW | RM_PH (k = 0: identical)                                 */
  int32_t factorization;     /* RM_CHOL | RM_ICC_SC of the scalar (H(grad)) patch problems: the     */
                             /* primary stars for k = 0, the PH potential vertex stars for k = 1     */
                             /* (P:1158-1160); k-stars of k = 1, 2 are always exact  */
  int32_t patch_entities;    /* RM_ALL_ENTITIES | RM_INTERIOR_ONLY                                  */
  double potential_shift;    /* eps_s for k = 2 PH (reading G8), default 1e-3                        */
  int32_t coarse;            /* 0: one-level additive Schwarz in rm_precondition / rm_pcg; 1: the    */
                             /* p = 1 coarse level (A_0 rediscretised, R_0 the FDM embedding, direct */
                             /* block-Cholesky solve) in a hybrid V(1,1) cycle with the patch sweep  */
                             /* damped by 1/N_c (readings G10 / G20);        */
                             /* single rank only. rm_relax is always the one-level sweep.           */
  void *stream;              /* cudaStream_t                                                        */
  const void *nccl_id;       /* 128-byte ncclUniqueId or NULL (single GPU)                          */
  int32_t rank, nranks, device;
  int32_t setup;             /* RM_SETUP_DEVICE (default): the numeric setup -- cell matrices (incl.  */
                             /* the trilinear auxiliary operator), patch assembly, block elimination,*/
                             /* dense Cholesky / ICC-SC with the G7 restart, stream packing -- runs  */
                             /* on the GPU; RM_SETUP_HOST: the same factorization   */
                             /* on the host (OpenMP).  The symbolic setup is host C++ in both.       */
} rm_options;

enum { RM_SETUP_HOST = 0, RM_SETUP_DEVICE = 1 };

typedef struct {
  int64_t n_local;           /* DoFs in the local vectors (constrained included)                   */
  int64_t n_free;            /* unconstrained DoFs (global)                                         */
  int64_t n_patches, n_patches_potential;
  int64_t n_factor_blocks;   /* distinct patch factors (identical patches share one)               */
  int64_t factor_bytes;      /* bytes of patch-factor values read by one sweep (primary+potential) */
  int64_t sweep_bytes;       /* algorithmic bytes of one sweep: factor values (per patch) + f,u,u_out */
  int32_t n_colors, n_classes;
  double icc_sigma_max;      /* largest ICC restart shift used (reading G7), 0 if none             */
  double setup_seconds;
  int64_t factor_nnz;        /* SURVEY 8(d) algorithmic factor entries of one sweep: sum over the   */
                             /* patches of nnz(L) of the exact Cholesky factor in the pinned order  */
                             /* (reading G6), or of the ICC-SC mask (primary + potential)           */
  int64_t factor_nnz_primary;   /* the same, primary (k-star) patches only                         */
  int64_t factor_unique_bytes;  /* bytes of the distinct value blocks held in HBM (identical       */
                                /* patches share one block)                                       */
  int32_t comm_nranks;       /* ranks of the context's NCCL communicator (0 = none)                 */
  int32_t coarse;            /* 1 if the p = 1 coarse level is set up (options.coarse)             */
  int64_t coarse_ndof;       /* unconstrained DoFs of the coarse problem A_0 (0 without it)        */
  int32_t batched_families;  /* patch families solved by the class-batched kernel (RM_PATCH_STREAM) */
  int32_t batch_width;       /* patches per CTA of the widest batched family (0 if none)           */
  int32_t setup_on_device;   /* 1 if the numeric setup ran on the GPU (options.setup)              */
  double setup_host_family_seconds;     /* host patch-family builds (symbolic programs; with        */
                                        /* RM_SETUP_HOST also the numeric factorization)            */
  double setup_device_numeric_seconds;  /* GPU numeric setup (RM_SETUP_DEVICE), incl. its uploads  */
} rm_info;

void rm_default_options(rm_options *opt);

/* Z-SLAB PARTITION (multi-GPU; every space and decomposition except SC-PAFW).  Rank g of G owns
 * the cell layers [mesh.z_begin, mesh.z_end) (contiguous slabs, rank order = z order), the DoF
 * planes z_begin*p .. z_end*p - 1 (the last rank also the top plane nz*p) and the star patches
 * (primary and potential) whose entity's z anchor -- a vertex layer, or the cell layer of an
 * entity spanning a cell in z -- lies in z_begin .. z_end - 1 (+ the vertex layer nz on the last rank).  Its LOCAL problem
 * is its slab plus one ghost cell layer below (rank > 0) and the shared plane above, so local
 * vectors hold planes z_cell0*p .. (z_cell0 + nz_local)*p.  Per sweep the neighbours exchange,
 * forward: u (and f) on the p planes below the slab and the shared plane above; reverse: the
 * patch corrections on the p - 1 planes below the slab, ADDED by their owner.  All plane ranges
 * below are LOCAL plane indices [first, last + 1); a plane is plane_len contiguous doubles.
 * With a communicator (options.nccl_id) the library exchanges the forward halos IN PLACE: the
 * non-owned planes of the input vectors of rm_apply / rm_residual / rm_relax / rm_precondition /
 * rm_pcg are overwritten with the owners' values (their input content is ignored), and the
 * non-owned planes of output vectors are unspecified on return (only owned planes are results).
 * Pure host arithmetic (no device needed). */
typedef struct {
  int32_t z_cell0, nz_local, ghost_lo;   /* global layer of local cell 0; local cell layers; 0|1 */
  int32_t v_lo, v_hi;                    /* owned vertex layers (local) = owned patches          */
  int32_t own_lo, own_hi;                /* owned DoF planes                                      */
  int32_t fwd_recv_lo[2], fwd_send_lo[2];   /* forward exchange with rank - 1 (u, f)            */
  int32_t fwd_recv_hi[2], fwd_send_hi[2];   /* forward exchange with rank + 1                    */
  int32_t rev_send_lo[2], rev_recv_hi[2];   /* reverse-add: corrections to rank - 1 / from + 1  */
  uint32_t gamma_local;                  /* Gamma_D bits of the local problem (cut planes free)  */
  int64_t plane_len;                     /* doubles per DoF plane: (nx p + 1)(ny p + 1)          */
  /* H(curl) / H(div): the ranges above hold for the components with a P family in z (planes
   * z_cell0*p .. (z_cell0 + nz_local)*p); components with a DP family in z have nz_local*p local
   * planes (plane c*p + a inside cell layer c, no shared plane) and use these instead.  A
   * component's plane has len_x * len_y doubles (rm_layout shape). */
  int32_t dp_own_lo, dp_own_hi;
  int32_t dp_fwd_recv_lo[2], dp_fwd_send_hi[2];   /* ghost cell layer <- rank - 1; my top layer -> rank + 1 */
  int32_t dp_rev_send_lo[2], dp_rev_recv_hi[2];   /* corrections on the ghost layer -> rank - 1 (added)   */
} rm_partition_info;
rm_status rm_partition(const rm_mesh *mesh, int32_t p, rm_space space, uint32_t gamma_d, int32_t rank,
                       int32_t nranks, rm_partition_info *info);
/* 128-byte ncclUniqueId for options.nccl_id (rank 0 creates it, the caller broadcasts it). */
rm_status rm_nccl_unique_id(void *id128);
/* Diagnostic: loads NCCL, builds a one-rank communicator on `device`, runs a grouped send/recv to
 * itself and an allreduce on a stream and checks the data (RM_ENCCL on any failure). */
rm_status rm_nccl_check(int32_t device);

/* Builds the 1D FDM tables, the structured layout, all patch factors and uploads them.
 * alpha, beta: host arrays, n == 1 (constant) or one value per cell, C-order [z][y][x].
 * Environment read at setup (the only runtime knobs of the product build):
 *   RM_SETUP_THREADS=n  host threads of the setup (default: all cores);
 *   RM_NBOX1=1          the persistent patch kernel keeps one window box in flight (test switch);
 *   RM_PATCH_STREAM=1   families whose patches share few factor blocks (uniform Cartesian meshes)
 *                       use the persistent stream kernel instead of the class-batched kernel
 *                       (test switch: both paths are parity-tested). */
rm_status rm_setup(rm_ctx **ctx, const rm_mesh *mesh, int32_t p, rm_space space,
                   const double *alpha, int64_t n_alpha, const double *beta, int64_t n_beta,
                   uint32_t gamma_d, const rm_options *opt);

/* shape[m][0..2] = (Z, Y, X) extents of component m (zeros for absent components). */
rm_status rm_layout(const rm_ctx *ctx, int64_t *n_local, int64_t *n_free, int32_t shape[3][3]);
rm_status rm_info_get(const rm_ctx *ctx, rm_info *info);
/* host mask[n_local]: 1 = constrained DoF. */
rm_status rm_constrained_mask(const rm_ctx *ctx, uint8_t *mask);

rm_status rm_apply(rm_ctx *ctx, const double *u, double *v);                 /* v = A u              */
rm_status rm_residual(rm_ctx *ctx, const double *f, const double *u, double *r);   /* r = f - A u  */
/* u_out = u_in + omega * P^{-1}(f - A u_in); u_out may alias u_in. */
rm_status rm_relax(rm_ctx *ctx, const double *f, const double *u_in, double *u_out, double omega);
/* z = M r: the additive Schwarz preconditioner (one sweep from zero with omega = 1), or with
 * options.coarse = 1 the hybrid V(1,1) cycle with the p = 1 coarse level. */
rm_status rm_precondition(rm_ctx *ctx, const double *r, double *z);
/* Multi-rank sweep in two stages, for callers that move the halos themselves (and the
 * single-GPU partition tests): rm_relax_begin reads f and u_in on every local plane (the caller
 * filled the forward halos) and writes the local patch correction c (all local planes, nonzero
 * on the ghost planes too); the caller reverse-adds the rev_* planes of c between its ranks;
 * rm_relax_end writes u_out = u_in + omega c.  With options.nccl_id set, rm_relax does all of
 * this itself over NCCL on the context's stream. */
rm_status rm_relax_begin(rm_ctx *ctx, const double *f, const double *u_in, double *c);
rm_status rm_relax_end(rm_ctx *ctx, const double *u_in, const double *c, double *u_out, double omega);
/* Same as rm_relax with HOST buffers: copies f, u_in to the device, sweeps, copies u_out back,
 * synchronises. */
rm_status rm_relax_host(rm_ctx *ctx, const double *f, const double *u_in, double *u_out, double omega);
/* PCG on the true A with the sweep preconditioner from u = 0; stops at the first k with
 * sqrt(r_k^T z_k) <= rtol sqrt(r_0^T z_0). u: device, overwritten. */
rm_status rm_pcg(rm_ctx *ctx, const double *f, double *u, double rtol, int32_t maxit,
                 int32_t *iters, double *rel_natural_residual);

/* Phase timing (instrumentation used by bench.py).  While enabled, rm_relax / rm_precondition /
 * rm_pcg record CUDA events on their stream around each phase: [0] residual (apply kernels incl.
 * init / gather), [1] primary patch stage (pad, condensation, patch kernel, combine), [2] potential
 * stage (D^T, patch stage, D), [3] everything else (copies, PCG vector kernels); and around single
 * kernels (subsets of the phases above): [4] the persistent patch kernel launches (primary and
 * potential families), [5] the apply kernel launches (without init / gather).  rm_timing_read
 * synchronises and returns the accumulated milliseconds and launches per entry since the last
 * enable/read.  Arrays have RM_NPHASE entries. */
#define RM_NPHASE 8
rm_status rm_timing_enable(rm_ctx *ctx, int32_t on);
rm_status rm_timing_read(rm_ctx *ctx, double ms[RM_NPHASE], int64_t launches[RM_NPHASE]);

void rm_destroy(rm_ctx *ctx);
const char *rm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* RM_H_ */
