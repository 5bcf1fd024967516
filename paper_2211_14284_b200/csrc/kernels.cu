// sm_100a kernels of the relaxation sweep, part 1:
//
//  hiptmair_DT / _D_add    t = D^T r and u += omega D s for the Pavarino-Hiptmair potential stage
//                          (eq:asm-hiptmair P:961-975) with D the Kronecker-tabulated d^{k-1};
//                          output-stationary gathers, deterministic.
//  axpby / dot / pcg_*     PCG vector kernels, fp64, deterministic two-stage dots.
// The matrix-free apply is in apply.cu, the batched patch solve in patch_solve.cu.
#include "kernels.cuh"

namespace rm {

enum { FAM_P_ = 0, FAM_D_ = 1 };

__device__ __forceinline__ bool is_constrained_idx(int fam, long long idx, long long last, unsigned gamma_d, int d) {
  if (fam != FAM_P_) return false;
  if (idx == 0 && (gamma_d & (1u << (2 * d)))) return true;
  if (idx == last && (gamma_d & (1u << (2 * d + 1)))) return true;
  return false;
}

__device__ __forceinline__ int cells_of(long long I, int fam, int p, int ncell, int* c, int* a) {
  if (fam == FAM_D_) { c[0] = (int)(I / p); a[0] = (int)(I % p); return 1; }
  long long q = I / p;
  int r = (int)(I % p);
  if (r != 0) { c[0] = (int)q; a[0] = r; return 1; }
  int cnt = 0;
  if (q - 1 >= 0) { c[cnt] = (int)q - 1; a[cnt] = p; ++cnt; }
  if (q < ncell) { c[cnt] = (int)q; a[cnt] = 0; ++cnt; }
  return cnt;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ====================================================================== Hiptmair D, D^T
// contributions of d^{k-1} (standard curl, reading G17): target comp n <- sum sigma * d_e s_m
struct HipContrib { int n, m, e, sigma; };
__constant__ HipContrib c_grad[3] = {{0, 0, 0, 1}, {1, 0, 1, 1}, {2, 0, 2, 1}};
__constant__ HipContrib c_curl[6] = {{0, 2, 1, 1}, {0, 1, 2, -1}, {1, 0, 2, 1}, {1, 2, 0, -1}, {2, 1, 0, 1}, {2, 0, 1, -1}};

struct HipParams {
  int kpot;                 // form degree of the potential space (k - 1)
  int p, n[3];
  int fam_pot[3][3], fam_pri[3][3];
  long long len_pot[3][3], len_pri[3][3];
  long long off_pot[4], off_pri[4];
  int ncomp_pot, ncomp_pri;
  unsigned gamma_d;
  double D[RM_MAXP1 * RM_MAXP1];   // p x (p+1) row-major
};

__device__ __forceinline__ void decode(long long g, int ncomp, const long long* off, const long long (*len)[3],
                                       int& m, long long* idx) {
  m = 0;
  while (m + 1 < ncomp && g >= off[m + 1]) ++m;
  // 32-bit index math (component sizes < 2^31): the 64-bit divisions dominated these kernels
  const int rr = (int)(g - off[m]);
  const int l0 = (int)len[m][0], l1 = (int)len[m][1];
  const int q = rr / l0;
  idx[0] = rr - q * l0;
  idx[1] = q % l1;
  idx[2] = q / l1;
}

// t = D^T r on the potential space (zero on constrained potential DoFs).  D-hat's column
// structure (eq:gradbasis: an interior column j has the single entry (j, j); columns 0 and p are
// full) makes an interior index a one-term gather and a vertex index a p-term line sum.
__global__ void hiptmair_DT_kernel(const __grid_constant__ HipParams hp, const double* __restrict__ r,
                                   double* __restrict__ t, long long npot) {
  __shared__ double Ds[RM_MAXP1 * RM_MAXP1];   // lane-varying indices: shared memory, not the param bank
  for (int i = threadIdx.x; i < hp.p * (hp.p + 1); i += blockDim.x) Ds[i] = hp.D[i];
  __syncthreads();
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npot) return;
  int m;
  long long idx[3];
  decode(g, hp.ncomp_pot, hp.off_pot, hp.len_pot, m, idx);
  const int p = hp.p, P1 = p + 1;
  for (int d = 0; d < 3; ++d)
    if (is_constrained_idx(hp.fam_pot[m][d], idx[d], (long long)hp.n[d] * p, hp.gamma_d, d)) { t[g] = 0.0; return; }
  const HipContrib* L = hp.kpot == 0 ? c_grad : c_curl;
  const int nL = hp.kpot == 0 ? 3 : 6;
  double acc = 0.0;
  for (int q = 0; q < nL; ++q) {
    if (L[q].m != m) continue;
    const int n = L[q].n, e = L[q].e;
    // (D^T r)_I along e: I is a P index in direction e; r_n has a DP index c p + a along e
    const int lx = (int)hp.len_pri[n][0], ly = (int)hp.len_pri[n][1];
    const int stride = e == 0 ? 1 : (e == 1 ? lx : lx * ly);
    int j[3] = {(int)idx[0], (int)idx[1], (int)idx[2]};
    const int I = j[e], c = I / p, aa = I - c * p;
    j[e] = 0;
    const double* rb = r + hp.off_pri[n] + ((long long)j[2] * ly + j[1]) * lx + j[0];
    double s = 0.0;
    if (aa != 0) {                 // interior column: the single entry (aa, aa)
      s = Ds[aa * P1 + aa] * rb[(c * p + aa) * stride];
    } else {                       // vertex column: cells c - 1 (as column p) and c (as column 0)
      if (c >= 1)
        for (int a = 0; a < p; ++a) s += Ds[a * P1 + p] * rb[((c - 1) * p + a) * stride];
      if (c < hp.n[e])
        for (int a = 0; a < p; ++a) s += Ds[a * P1] * rb[(c * p + a) * stride];
    }
    acc += L[q].sigma * s;
  }
  t[g] = acc;
}

// u += omega * D s on the primal space (zero contribution on constrained primal DoFs).  D-hat
// row a has the entries (a, 0), (a, p) and, for a >= 1, (a, a): three gathers per term.
__global__ void hiptmair_D_add_kernel(const __grid_constant__ HipParams hp, const double* __restrict__ s,
                                      double* __restrict__ u, double omega, long long npri) {
  __shared__ double Ds[RM_MAXP1 * RM_MAXP1];
  for (int i = threadIdx.x; i < hp.p * (hp.p + 1); i += blockDim.x) Ds[i] = hp.D[i];
  __syncthreads();
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= npri) return;
  int n;
  long long idx[3];
  decode(g, hp.ncomp_pri, hp.off_pri, hp.len_pri, n, idx);
  const int p = hp.p, P1 = p + 1;
  for (int d = 0; d < 3; ++d)
    if (is_constrained_idx(hp.fam_pri[n][d], idx[d], (long long)hp.n[d] * p, hp.gamma_d, d)) return;
  const HipContrib* L = hp.kpot == 0 ? c_grad : c_curl;
  const int nL = hp.kpot == 0 ? 3 : 6;
  double acc = 0.0;
  for (int q = 0; q < nL; ++q) {
    if (L[q].n != n) continue;
    const int m = L[q].m, e = L[q].e;
    // (d_e s_m)_I : I is a DP index along e in cell c = I / p, a = I % p
    const int lx = (int)hp.len_pot[m][0], ly = (int)hp.len_pot[m][1];
    const int stride = e == 0 ? 1 : (e == 1 ? lx : lx * ly);
    int j[3] = {(int)idx[0], (int)idx[1], (int)idx[2]};
    const int c = j[e] / p, a = j[e] - (j[e] / p) * p;
    j[e] = c * p;
    const double* sb = s + hp.off_pot[m] + ((long long)j[2] * ly + j[1]) * lx + j[0];
    double sum = Ds[a * P1] * sb[0] + Ds[a * P1 + p] * sb[p * stride];
    if (a >= 1) sum += Ds[a * P1 + a] * sb[a * stride];
    acc += L[q].sigma * sum;
  }
  u[g] += omega * acc;
}

// Row-per-warp forms of the two kernels above (one (y, z) row of one component per warp, lanes
// along x; no per-DoF index decode).  D^T: for the terms along x (e = 0) the warp stages the
// source row of r_n in shared memory once, so the vertex columns' p-term sums read shared memory
// instead of diverging global loops.  Same addends in the same order: bitwise equal.
#ifndef RM_HIP_WARPS   // tuning knob (-D): warps per CTA of the Hiptmair row kernels (4: cfg4 potential +0.17 ms)
#define RM_HIP_WARPS 8
#endif
constexpr int HIP_ROWS_WARPS = RM_HIP_WARPS;
constexpr int HIP_ROW_MAX = 640;    // 2 staged rows of <= 320 doubles per warp; longer rows read global memory
__global__ void __launch_bounds__(32 * HIP_ROWS_WARPS) hiptmair_DT_rows_kernel(const __grid_constant__ HipParams hp,
                                                                               const double* __restrict__ r,
                                                                               double* __restrict__ t) {
  __shared__ double Ds[RM_MAXP1 * RM_MAXP1];
  __shared__ double rowbuf[HIP_ROWS_WARPS][2][HIP_ROW_MAX / 2];
  for (int i = threadIdx.x; i < hp.p * (hp.p + 1); i += blockDim.x) Ds[i] = hp.D[i];
  __syncthreads();
  const int p = hp.p, P1 = p + 1, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const HipContrib* L = hp.kpot == 0 ? c_grad : c_curl;
  const int nL = hp.kpot == 0 ? 3 : 6;
  int rows_before = 0;
  for (int m = 0; m < hp.ncomp_pot; ++m) {
    const int Lx = (int)hp.len_pot[m][0], Ly = (int)hp.len_pot[m][1], nrow = Ly * (int)hp.len_pot[m][2];
    for (int row = blockIdx.x * HIP_ROWS_WARPS + w - rows_before; row < nrow; row += gridDim.x * HIP_ROWS_WARPS) {
      if (row < 0) continue;
      const int iy = row % Ly, iz = row / Ly;
      const bool rcon = is_constrained_idx(hp.fam_pot[m][1], iy, (long long)hp.n[1] * p, hp.gamma_d, 1) ||
                        is_constrained_idx(hp.fam_pot[m][2], iz, (long long)hp.n[2] * p, hp.gamma_d, 2);
      double* trow = t + hp.off_pot[m] + (long long)row * Lx;
      if (rcon) {
        for (int x = lane; x < Lx; x += 32) trow[x] = 0.0;
        continue;
      }
      // stage the x-direction source rows (terms with e = 0; at most two per component)
      int ns = 0;
      const double* xsrc[2] = {nullptr, nullptr};
      for (int q = 0; q < nL; ++q) {
        if (L[q].m != m || L[q].e != 0) continue;
        const int n = L[q].n;
        const int lx = (int)hp.len_pri[n][0], ly = (int)hp.len_pri[n][1];
        const double* rb = r + hp.off_pri[n] + ((long long)iz * ly + iy) * lx;
        if (lx <= HIP_ROW_MAX / 2 && ns < 2) {
          for (int x = lane; x < lx; x += 32) rowbuf[w][ns][x] = rb[x];
          xsrc[ns] = rowbuf[w][ns];
        } else {
          xsrc[ns] = rb;
        }
        ++ns;
      }
      __syncwarp();
      for (int x = lane; x < Lx; x += 32) {
        if (is_constrained_idx(hp.fam_pot[m][0], x, (long long)hp.n[0] * p, hp.gamma_d, 0)) { trow[x] = 0.0; continue; }
        double acc = 0.0;
        int si = 0;
        for (int q = 0; q < nL; ++q) {
          if (L[q].m != m) continue;
          const int n = L[q].n, e = L[q].e;
          const int lx = (int)hp.len_pri[n][0], ly = (int)hp.len_pri[n][1];
          const int j[3] = {x, iy, iz};
          const int I = j[e], c = I / p, aa = I - c * p;
          const double* rb;
          int stride;
          if (e == 0) {
            rb = xsrc[si++];
            stride = 1;
          } else {
            int jj[3] = {x, iy, iz};
            jj[e] = 0;
            rb = r + hp.off_pri[n] + ((long long)jj[2] * ly + jj[1]) * lx + jj[0];
            stride = e == 1 ? lx : lx * ly;
          }
          double s = 0.0;
          if (aa != 0) {
            s = Ds[aa * P1 + aa] * rb[(c * p + aa) * stride];
          } else {
            if (c >= 1)
              for (int a = 0; a < p; ++a) s += Ds[a * P1 + p] * rb[((c - 1) * p + a) * stride];
            if (c < hp.n[e])
              for (int a = 0; a < p; ++a) s += Ds[a * P1] * rb[(c * p + a) * stride];
          }
          acc += L[q].sigma * s;
        }
        trow[x] = acc;
      }
      __syncwarp();
    }
    rows_before += nrow;
  }
}

__global__ void __launch_bounds__(32 * HIP_ROWS_WARPS) hiptmair_D_add_rows_kernel(const __grid_constant__ HipParams hp,
                                                                                  const double* __restrict__ s,
                                                                                  double* __restrict__ u, double omega) {
  __shared__ double Ds[RM_MAXP1 * RM_MAXP1];
  for (int i = threadIdx.x; i < hp.p * (hp.p + 1); i += blockDim.x) Ds[i] = hp.D[i];
  __syncthreads();
  const int p = hp.p, P1 = p + 1, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const HipContrib* L = hp.kpot == 0 ? c_grad : c_curl;
  const int nL = hp.kpot == 0 ? 3 : 6;
  int rows_before = 0;
  for (int n = 0; n < hp.ncomp_pri; ++n) {
    const int Lx = (int)hp.len_pri[n][0], Ly = (int)hp.len_pri[n][1], nrow = Ly * (int)hp.len_pri[n][2];
    for (int row = blockIdx.x * HIP_ROWS_WARPS + w - rows_before; row < nrow; row += gridDim.x * HIP_ROWS_WARPS) {
      if (row < 0) continue;
      const int iy = row % Ly, iz = row / Ly;
      if (is_constrained_idx(hp.fam_pri[n][1], iy, (long long)hp.n[1] * p, hp.gamma_d, 1) ||
          is_constrained_idx(hp.fam_pri[n][2], iz, (long long)hp.n[2] * p, hp.gamma_d, 2))
        continue;
      double* urow = u + hp.off_pri[n] + (long long)row * Lx;
      for (int x = lane; x < Lx; x += 32) {
        if (is_constrained_idx(hp.fam_pri[n][0], x, (long long)hp.n[0] * p, hp.gamma_d, 0)) continue;
        double acc = 0.0;
        for (int q = 0; q < nL; ++q) {
          if (L[q].n != n) continue;
          const int m = L[q].m, e = L[q].e;
          const int lx = (int)hp.len_pot[m][0], ly = (int)hp.len_pot[m][1];
          const int stride = e == 0 ? 1 : (e == 1 ? lx : lx * ly);
          int j[3] = {x, iy, iz};
          const int c = j[e] / p, a = j[e] - c * p;
          j[e] = c * p;
          const double* sb = s + hp.off_pot[m] + ((long long)j[2] * ly + j[1]) * lx + j[0];
          double sum = Ds[a * P1] * sb[0] + Ds[a * P1 + p] * sb[p * stride];
          if (a >= 1) sum += Ds[a * P1 + a] * sb[a * stride];
          acc += L[q].sigma * sum;
        }
        urow[x] += omega * acc;
      }
    }
    rows_before += nrow;
  }
}

static HipParams make_hip(int k, int p, const int* n, unsigned gamma_d, const double* Dh) {
  static const int FAMS[4][3][3] = {
      {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
      {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}},
      {{0, 1, 1}, {1, 0, 1}, {1, 1, 0}},
      {{1, 1, 1}, {0, 0, 0}, {0, 0, 0}},
  };
  HipParams hp{};
  hp.kpot = k - 1; hp.p = p;
  for (int d = 0; d < 3; ++d) hp.n[d] = n[d];
  hp.ncomp_pot = (k - 1 == 0) ? 1 : 3;
  hp.ncomp_pri = (k == 0 || k == 3) ? 1 : 3;
  hp.gamma_d = gamma_d;
  long long o1 = 0, o2 = 0;
  for (int m = 0; m < 3; ++m) {
    hp.off_pot[m] = o1; hp.off_pri[m] = o2;
    long long s1 = 1, s2 = 1;
    for (int d = 0; d < 3; ++d) {
      hp.fam_pot[m][d] = FAMS[k - 1][m][d];
      hp.fam_pri[m][d] = FAMS[k][m][d];
      hp.len_pot[m][d] = hp.fam_pot[m][d] == 0 ? (long long)n[d] * p + 1 : (long long)n[d] * p;
      hp.len_pri[m][d] = hp.fam_pri[m][d] == 0 ? (long long)n[d] * p + 1 : (long long)n[d] * p;
      s1 *= hp.len_pot[m][d]; s2 *= hp.len_pri[m][d];
    }
    if (m < hp.ncomp_pot) o1 += s1;
    if (m < hp.ncomp_pri) o2 += s2;
  }
  hp.off_pot[3] = o1; hp.off_pri[3] = o2;
  for (int i = 0; i < p * (p + 1); ++i) hp.D[i] = Dh[i];
  return hp;
}

cudaError_t launch_hiptmair_DT(int k, int p, const int* n, unsigned gamma_d, const double* Dh, const double* r,
                               double* t, cudaStream_t st) {
  HipParams hp = make_hip(k, p, n, gamma_d, Dh);
  const long long N = hp.off_pot[hp.ncomp_pot];
  if (exp_env("RM_HIP_PERDOF")) hiptmair_DT_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(hp, r, t, N);
  else hiptmair_DT_rows_kernel<<<148 * 8, 32 * HIP_ROWS_WARPS, 0, st>>>(hp, r, t);
  return cudaGetLastError();
}

cudaError_t launch_hiptmair_D_add(int k, int p, const int* n, unsigned gamma_d, const double* Dh, const double* s,
                                  double* u, double omega, cudaStream_t st) {
  HipParams hp = make_hip(k, p, n, gamma_d, Dh);
  const long long N = hp.off_pri[hp.ncomp_pri];
  if (exp_env("RM_HIP_PERDOF")) hiptmair_D_add_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(hp, s, u, omega, N);
  else hiptmair_D_add_rows_kernel<<<148 * 8, 32 * HIP_ROWS_WARPS, 0, st>>>(hp, s, u, omega);
  return cudaGetLastError();
}

// ====================================================================== vector kernels
__global__ void axpby_kernel(long long n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}
cudaError_t launch_axpby(long long n, double a, const double* x, double b, double* y, cudaStream_t st) {
  axpby_kernel<<<148 * 8, 256, 0, st>>>(n, a, x, b, y);
  return cudaGetLastError();
}

#define RM_DOT_BLOCKS 592
__global__ void dot_stage1(long long n, const double* __restrict__ x, const double* __restrict__ y, double* partial) {
  __shared__ double sh[8];
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += x[i] * y[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < 8 ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
  }
}
__global__ void dot_stage2(const double* partial, int nb, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) *out = t;
  }
}
cudaError_t launch_dot(long long n, const double* x, const double* y, double* partial, double* out, cudaStream_t st) {
  dot_stage1<<<RM_DOT_BLOCKS, 256, 0, st>>>(n, x, y, partial);
  dot_stage2<<<1, 256, 0, st>>>(partial, RM_DOT_BLOCKS, out);
  return cudaGetLastError();
}

// x += a p ; r -= a q  with a = num/den read on device
__global__ void pcg_update_kernel(long long n, const double* num, const double* den, const double* __restrict__ p,
                                  const double* __restrict__ q, double* __restrict__ x, double* __restrict__ r) {
  const double a = *num / *den;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    x[i] += a * p[i];
    r[i] -= a * q[i];
  }
}
cudaError_t launch_pcg_update(long long n, const double* num, const double* den, const double* p, const double* q,
                              double* x, double* r, cudaStream_t st) {
  pcg_update_kernel<<<148 * 8, 256, 0, st>>>(n, num, den, p, q, x, r);
  return cudaGetLastError();
}
// p = z + (rz_new/rz_old) p
__global__ void pcg_pupdate_kernel(long long n, const double* rzn, const double* rzo, const double* __restrict__ z,
                                   double* __restrict__ p) {
  const double b = *rzn / *rzo;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = z[i] + b * p[i];
}
cudaError_t launch_pcg_pupdate(long long n, const double* rz_new, const double* rz_old, const double* z, double* p,
                               cudaStream_t st) {
  pcg_pupdate_kernel<<<148 * 8, 256, 0, st>>>(n, rz_new, rz_old, z, p);
  return cudaGetLastError();
}

}  // namespace rm
