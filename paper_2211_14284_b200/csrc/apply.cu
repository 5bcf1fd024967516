// Matrix-free Cartesian operator: r = f - A u or v = A u.
//
// Sum factorization of eq:sum-factorization: on an axis-aligned cell every block of
// A_K is a sum of Kronecker products X (x) Y (x) Z of 1D FDM matrices (B-hat, A-hat, I, D-hat,
// D-hat^T; model.cpp), scaled by alpha_K or beta_K and powers of the cell sizes.  One warp owns
// one cell: it stages the cell's (p+1)^3-sized coefficient window in shared memory, applies each
// term as three 1D contractions over the sparse rows of X, Y, Z (B-hat is diagonal plus a corner,
// A-hat an arrow, D-hat has <= 3 entries per row, so a 1D sweep costs O(p^3) per cell), and adds
// the result into the output.  Cells are processed in 8 parity colours (cells of one colour
// share no DoF), so the accumulation is a plain read-modify-write: deterministic, no atomics.
#include "kernels.cuh"

namespace rm {

enum { FAMP = 0, FAMD = 1 };
// shared-memory table area (doubles): values, row pointers (short), columns (uchar), rounded up
constexpr int RM_APPLY_TABLE_DOUBLES =
    RM_MAXMATS * RM_MAXMATNZ + (RM_MAXMATS * (RM_MAXP1 + 1) * 2 + RM_MAXMATS * RM_MAXMATNZ + 7) / 8 + 1;

__device__ __forceinline__ bool cons_idx(int fam, long long idx, long long last, unsigned gamma_d, int d) {
  if (fam != FAMP) return false;
  if (idx == 0 && (gamma_d & (1u << (2 * d)))) return true;
  if (idx == last && (gamma_d & (1u << (2 * d + 1)))) return true;
  return false;
}

// one component (k = 0): one row (y, z) per warp, grid-stride, 32-bit index math; out may be padded
__global__ void apply_init_q_kernel(const __grid_constant__ OpParams op, const double* __restrict__ f,
                                    double* __restrict__ out) {
  const int Lx = (int)op.len[0][0], Ly = (int)op.len[0][1], Lz = (int)op.len[0][2];
  const long long ldx = op.ldx_out > 0 ? op.ldx_out : Lx;
  const int lane = threadIdx.x & 31;
  const int nrow = Ly * Lz, wstride = gridDim.x * (blockDim.x >> 5);
  for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); row < nrow; row += wstride) {
    const int y = row % Ly, z = row / Ly;
    const bool rc = cons_idx(op.fam[0][1], y, (long long)op.n[1] * op.p, op.gamma_d, 1) ||
                    cons_idx(op.fam[0][2], z, (long long)op.n[2] * op.p, op.gamma_d, 2);
    const long long fb = (long long)row * Lx, ob = (long long)row * ldx;
    for (int x = lane; x < Lx; x += 32) {
      const bool con = rc || cons_idx(op.fam[0][0], x, (long long)op.n[0] * op.p, op.gamma_d, 0);
      out[ob + x] = (con || !f) ? 0.0 : f[fb + x];
    }
  }
}

// out = f (or 0) with constrained entries zeroed
__global__ void apply_init_kernel(const __grid_constant__ OpParams op, const double* __restrict__ f,
                                  double* __restrict__ out, long long ndof) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ndof) return;
  int m = 0;
  while (m + 1 < op.ncomp && g >= op.off[m + 1]) ++m;
  const long long rr = g - op.off[m];
  const long long Lx = op.len[m][0], Ly = op.len[m][1];
  const long long idx[3] = {rr % Lx, (rr / Lx) % Ly, rr / (Lx * Ly)};
  bool con = false;
  for (int d = 0; d < 3; ++d) con |= cons_idx(op.fam[m][d], idx[d], (long long)op.n[d] * op.p, op.gamma_d, d);
  const long long og = (op.ldx_out > 0 && op.ncomp == 1) ? (idx[2] * Ly + idx[1]) * op.ldx_out + idx[0] : g;
  out[og] = (con || !f) ? 0.0 : f[g];
}

template <int WPB>
__global__ void __launch_bounds__(WPB * 32) apply_cells_kernel(const __grid_constant__ OpParams op,
                                                                const double* __restrict__ alpha,
                                                                const double* __restrict__ beta, int coef_const,
                                                                const double* __restrict__ hpow,
                                                                const double* __restrict__ u, double* __restrict__ out,
                                                                double sign, int px, int py, int pz) {
  extern __shared__ double smx[];
  // 1D matrix tables copied from the (constant-bank) kernel parameters to shared memory: lanes
  // read different rows, which the constant cache would serialise
  double* sval = smx;                                                       // [RM_MAXMATS][RM_MAXMATNZ]
  short* srow = reinterpret_cast<short*>(sval + RM_MAXMATS * RM_MAXMATNZ);   // [RM_MAXMATS][RM_MAXP1+1]
  unsigned char* scol = reinterpret_cast<unsigned char*>(srow + RM_MAXMATS * (RM_MAXP1 + 1));
  for (int i = threadIdx.x; i < op.nmats * RM_MAXMATNZ; i += blockDim.x) {
    sval[i] = op.val[i / RM_MAXMATNZ][i % RM_MAXMATNZ];
    scol[i] = op.col[i / RM_MAXMATNZ][i % RM_MAXMATNZ];
  }
  for (int i = threadIdx.x; i < op.nmats * (RM_MAXP1 + 1); i += blockDim.x)
    srow[i] = op.rowptr[i / (RM_MAXP1 + 1)][i % (RM_MAXP1 + 1)];
  __syncthreads();
  double* sm = smx + RM_APPLY_TABLE_DOUBLES;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p = op.p;
  const int P1 = p + 1;
  const int cap = P1 * P1 * P1;
#define ROWPTR(mm, i) srow[(mm) * (RM_MAXP1 + 1) + (i)]
#define COL(mm, e) scol[(mm) * RM_MAXMATNZ + (e)]
#define VAL(mm, e) sval[(mm) * RM_MAXMATNZ + (e)]
  // local layout
  int lsz[3][3], lo[4];
  lo[0] = 0;
  for (int m = 0; m < op.ncomp; ++m) {
    for (int d = 0; d < 3; ++d) lsz[m][d] = op.fam[m][d] == FAMP ? P1 : p;
    lo[m + 1] = lo[m] + lsz[m][0] * lsz[m][1] * lsz[m][2];
  }
  const int nloc = lo[op.ncomp];
  double* ul = sm + (size_t)warp * (2 * nloc + 2 * cap);
  double* vl = ul + nloc;
  double* t1 = vl + nloc;
  double* t2 = t1 + cap;
  // cell of this warp within the colour
  const int ncx = (op.n[0] - px + 1) / 2, ncy = (op.n[1] - py + 1) / 2, ncz = (op.n[2] - pz + 1) / 2;
  const long long cw = (long long)blockIdx.x * WPB + warp;
  if (cw >= (long long)ncx * ncy * ncz) return;
  const int cx = px + 2 * (int)(cw % ncx), cy = py + 2 * (int)((cw / ncx) % ncy), cz = pz + 2 * (int)(cw / ((long long)ncx * ncy));
  const long long cell = ((long long)cz * op.n[1] + cy) * op.n[0] + cx;
  // gather u (constrained entries read as zero)
  for (int m = 0; m < op.ncomp; ++m) {
    const int sx = lsz[m][0], sy = lsz[m][1], sz = lsz[m][2];
    const long long Lx = op.len[m][0], Ly = op.len[m][1];
    const double* ub = u + op.off[m];
    for (int l = lane; l < sx * sy * sz; l += 32) {
      const int a = l % sx, b = (l / sx) % sy, c = l / (sx * sy);
      const long long ix = (long long)cx * p + a, iy = (long long)cy * p + b, iz = (long long)cz * p + c;
      const bool con = cons_idx(op.fam[m][0], ix, (long long)op.n[0] * p, op.gamma_d, 0) ||
                       cons_idx(op.fam[m][1], iy, (long long)op.n[1] * p, op.gamma_d, 1) ||
                       cons_idx(op.fam[m][2], iz, (long long)op.n[2] * p, op.gamma_d, 2);
      ul[lo[m] + l] = con ? 0.0 : __ldg(ub + (iz * Ly + iy) * Lx + ix);
      vl[lo[m] + l] = 0.0;
    }
  }
  __syncwarp();
  const double al = coef_const ? alpha[0] : alpha[cell];
  const double be = coef_const ? beta[0] : beta[cell];
  const int hoff1 = 7 * op.n[0], hoff2 = 7 * (op.n[0] + op.n[1]);
  for (int t = 0; t < op.nterms; ++t) {
    const OpTerm& T = op.terms[t];
    const int mi = T.min, mo = T.mout;
    const int ix_ = lsz[mi][0], iy_ = lsz[mi][1], iz_ = lsz[mi][2];
    const int ox = lsz[mo][0], oy = lsz[mo][1], oz = lsz[mo][2];
    const double scale = T.c * (T.coef == 0 ? al : be) * hpow[(T.hexp[0] + 3) * op.n[0] + cx] *
                         hpow[hoff1 + (T.hexp[1] + 3) * op.n[1] + cy] * hpow[hoff2 + (T.hexp[2] + 3) * op.n[2] + cz];
    const int mx = T.mat[0], my = T.mat[1], mz = T.mat[2];
    const double* uin = ul + lo[mi];
    // x: t1[ci][bi][ao]
    for (int l = lane; l < iz_ * iy_ * ox; l += 32) {
      const int ao = l % ox, r = l / ox;   // r = ci*iy + bi
      double s = 0.0;
      for (int e = ROWPTR(mx, ao); e < ROWPTR(mx, ao + 1); ++e) s += VAL(mx, e) * uin[r * ix_ + COL(mx, e)];
      t1[l] = s;
    }
    __syncwarp();
    // y: t2[ci][bo][ao]
    for (int l = lane; l < iz_ * oy * ox; l += 32) {
      const int ao = l % ox, bo = (l / ox) % oy, ci = l / (ox * oy);
      double s = 0.0;
      for (int e = ROWPTR(my, bo); e < ROWPTR(my, bo + 1); ++e)
        s += VAL(my, e) * t1[(ci * iy_ + COL(my, e)) * ox + ao];
      t2[l] = s;
    }
    __syncwarp();
    // z: v[co][bo][ao] += scale * sum Z t2
    double* vo = vl + lo[mo];
    for (int l = lane; l < oz * oy * ox; l += 32) {
      const int plane = l % (oy * ox), co = l / (oy * ox);
      double s = 0.0;
      for (int e = ROWPTR(mz, co); e < ROWPTR(mz, co + 1); ++e) s += VAL(mz, e) * t2[COL(mz, e) * (oy * ox) + plane];
      vo[l] += scale * s;
    }
    __syncwarp();
  }
  // scatter (constrained rows stay zero)
  for (int m = 0; m < op.ncomp; ++m) {
    const int sx = lsz[m][0], sy = lsz[m][1], sz = lsz[m][2];
    const long long Lx = op.len[m][0], Ly = op.len[m][1];
    double* ob = out + op.off[m];
    for (int l = lane; l < sx * sy * sz; l += 32) {
      const int a = l % sx, b = (l / sx) % sy, c = l / (sx * sy);
      const long long ix = (long long)cx * p + a, iy = (long long)cy * p + b, iz = (long long)cz * p + c;
      const bool con = cons_idx(op.fam[m][0], ix, (long long)op.n[0] * p, op.gamma_d, 0) ||
                       cons_idx(op.fam[m][1], iy, (long long)op.n[1] * p, op.gamma_d, 1) ||
                       cons_idx(op.fam[m][2], iz, (long long)op.n[2] * p, op.gamma_d, 2);
      if (!con) ob[(iz * Ly + iy) * Lx + ix] += sign * vl[lo[m] + l];
    }
  }
}

// ----------------------------------------------------------------------------------------
// H(grad) specialisation (k = 0): A_K u = beta s_M (B x B x B) u + alpha sum_d s_d (.. A_d ..) u,
// factored as three line stages with every 1D line held in registers (p compile-time):
//   x-stage  bx = B_x u, ax = A_x u
//   y-stage  P = beta s_M B_y bx + alpha s_x B_y ax + alpha s_y A_y bx,   Q = B_y bx
//   z-stage  v = B_z P + alpha s_z A_z Q
// B-hat is diagonal plus the (0,p) corner and A-hat interior rows have 3 entries, so a line
// costs O(p).  One thread per line of one cell, several cells per block, 8 parity colours.
template <int P>
__device__ __forceinline__ void apply_B(const double* __restrict__ Bh, const double (&x)[P + 1], double (&y)[P + 1]) {
  constexpr int N = P + 1;
#pragma unroll
  for (int i = 1; i < P; ++i) y[i] = Bh[i * N + i] * x[i];
  y[0] = Bh[0] * x[0] + Bh[P] * x[P];
  y[P] = Bh[P * N] * x[0] + Bh[P * N + P] * x[P];
}
template <int P>
__device__ __forceinline__ void apply_A(const double* __restrict__ Ah, const double (&x)[P + 1], double (&y)[P + 1]) {
  constexpr int N = P + 1;
#pragma unroll
  for (int i = 1; i < P; ++i) y[i] = Ah[i * N] * x[0] + Ah[i * N + i] * x[i] + Ah[i * N + P] * x[P];
  double s0 = 0.0, sP = 0.0;
#pragma unroll
  for (int j = 0; j < N; ++j) { s0 += Ah[j] * x[j]; sP += Ah[P * N + j] * x[j]; }
  y[0] = s0;
  y[P] = sP;
}

#ifndef RM_Q_THREADS   // CTA size of the k = 0 apply (tuning knob: -DRM_Q_THREADS, -DRM_Q_MINB)
#define RM_Q_THREADS 256
#endif
#ifndef RM_Q_MINB
#define RM_Q_MINB 5
#endif
template <int P>
__global__ void __launch_bounds__(RM_Q_THREADS, RM_Q_MINB) apply_q_kernel(const __grid_constant__ OpParams op,
                                                       const double* __restrict__ alpha,
                                                       const double* __restrict__ beta, int coef_const,
                                                       const double* __restrict__ hpow,
                                                       const double* __restrict__ u, double* __restrict__ out,
                                                       double sign, int px, int py, int pz,
                                                       double* __restrict__ cellbuf, const double* __restrict__ f) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  // cell window in shared memory with x lines padded to N + 1 doubles: the x stage (thread per
  // x line) and the y stage read conflict-free (unpadded, stride-N lines were 16-way conflicts)
  constexpr int NP = N + 1, NW = N2 * NP;
  constexpr int CPB = (RM_Q_THREADS / N2) > 0 ? (RM_Q_THREADS / N2) : 1;
  extern __shared__ double sm[];
  const int tid = threadIdx.x;
  const int cs = tid / N2, q = tid % N2;
  double* A = sm + cs * 2 * NW;
  double* Bf = A + NW;
  // colour mode: the cells of parity (px, py, pz), out += sign A_K u; cell-buffer mode (cellbuf):
  // every cell, interior DoFs stored as sign A_K u, skeleton entries to cellbuf (summed by the gather)
  const int ncx = cellbuf ? op.n[0] : (op.n[0] - px + 1) / 2, ncy = cellbuf ? op.n[1] : (op.n[1] - py + 1) / 2,
            ncz = cellbuf ? op.n[2] : (op.n[2] - pz + 1) / 2;
  const int cstep = cellbuf ? 1 : 2, ox = cellbuf ? 0 : px, oy = cellbuf ? 0 : py, oz = cellbuf ? 0 : pz;
  const long long cw = (long long)blockIdx.x * CPB + cs;
  const bool valid = cw < (long long)ncx * ncy * ncz;
  int cx = 0, cy = 0, cz = 0;
  if (valid) {
    cx = ox + cstep * (int)(cw % ncx); cy = oy + cstep * (int)((cw / ncx) % ncy);
    cz = oz + cstep * (int)(cw / ((long long)ncx * ncy));
  }
  const long long Lx = op.len[0][0], Ly = op.len[0][1];
  const long long LDX = op.ldx_out > 0 ? op.ldx_out : Lx;   // output row stride (padded layout)
  const long long lastx = (long long)op.n[0] * P, lasty = (long long)op.n[1] * P, lastz = (long long)op.n[2] * P;
  if (valid) {
    for (int l = q; l < N3; l += N2) {
      const int a = l % N, b = (l / N) % N, c = l / N2;
      const long long ix = (long long)cx * P + a, iy = (long long)cy * P + b, iz = (long long)cz * P + c;
      const bool con = cons_idx(FAMP, ix, lastx, op.gamma_d, 0) || cons_idx(FAMP, iy, lasty, op.gamma_d, 1) ||
                       cons_idx(FAMP, iz, lastz, op.gamma_d, 2);
      A[(c * N + b) * NP + a] = con ? 0.0 : __ldg(u + (iz * Ly + iy) * Lx + ix);
    }
  }
  __syncthreads();
  double x[N], y1[N], y2[N];
  // x-stage: thread q = (b, c)
  if (valid) {
    const int base = q * NP;
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = A[base + i];
    apply_B<P>(op.Bh, x, y1);
    apply_A<P>(op.Ah, x, y2);
#pragma unroll
    for (int i = 0; i < N; ++i) { Bf[base + i] = y1[i]; A[base + i] = y2[i]; }
  }
  __syncthreads();
  const long long cell = ((long long)cz * op.n[1] + cy) * op.n[0] + cx;
  const double al = coef_const ? alpha[0] : alpha[valid ? cell : 0];
  const double be = coef_const ? beta[0] : beta[valid ? cell : 0];
  const double hx = hpow[4 * op.n[0] + cx], hy = hpow[7 * op.n[0] + 4 * op.n[1] + cy],
               hz = hpow[7 * (op.n[0] + op.n[1]) + 4 * op.n[2] + cz];
  const double sM = be * hx * hy * hz * 0.125, sx = al * hy * hz / (2.0 * hx), sy = al * hx * hz / (2.0 * hy),
               sz = al * hx * hy / (2.0 * hz);
  // y-stage: thread q = (a, c): lines A[c][.][a]
  if (valid) {
    const int a = q % N, c = q / N;
    double bx[N], Pv[N];
#pragma unroll
    for (int j = 0; j < N; ++j) { bx[j] = Bf[(c * N + j) * NP + a]; x[j] = A[(c * N + j) * NP + a]; }
    apply_B<P>(op.Bh, x, y1);    // B_y ax
    apply_A<P>(op.Ah, bx, y2);   // A_y bx
    apply_B<P>(op.Bh, bx, x);    // Q = B_y bx
#pragma unroll
    for (int j = 0; j < N; ++j) Pv[j] = sM * x[j] + sx * y1[j] + sy * y2[j];
#pragma unroll
    for (int j = 0; j < N; ++j) { A[(c * N + j) * NP + a] = Pv[j]; Bf[(c * N + j) * NP + a] = x[j]; }
  }
  __syncthreads();
  // z-stage: thread q = (a, b): lines [.][b][a]
  if (valid) {
    const int a = q % N, b = q / N;
    double Qv[N];
#pragma unroll
    for (int k = 0; k < N; ++k) { x[k] = A[(k * N + b) * NP + a]; Qv[k] = Bf[(k * N + b) * NP + a]; }
    apply_B<P>(op.Bh, x, y1);
    apply_A<P>(op.Ah, Qv, y2);
    const long long ix = (long long)cx * P + a, iy = (long long)cy * P + b;
    if (cellbuf) {
      double* cb = cellbuf + (long long)((cz * op.n[1] + cy) * op.n[0] + cx) * N3 + b * N + a;
      const bool skel_ab = a == 0 || a == P || b == 0 || b == P;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const double vv = y1[k] + sz * y2[k];
        if (skel_ab || k == 0 || k == P) cb[k * N2] = vv;
        else {   // cell interior (owned by this cell alone): final, out = f + sign A_K u
          const long long row = (long long)cz * P + k;
          out[(row * Ly + iy) * LDX + ix] = (f ? __ldg(f + (row * Ly + iy) * Lx + ix) : 0.0) + sign * vv;
        }
      }
      return;
    }
    const bool conxy = cons_idx(FAMP, ix, lastx, op.gamma_d, 0) || cons_idx(FAMP, iy, lasty, op.gamma_d, 1);
    if (!conxy) {
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const long long iz = (long long)cz * P + k;
        if (cons_idx(FAMP, iz, lastz, op.gamma_d, 2)) continue;
        out[(iz * Ly + iy) * LDX + ix] += sign * (y1[k] + sz * y2[k]);
      }
    }
  }
}

template <int P>
static cudaError_t launch_q(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                            const double* hpow, const double* u, double* out, double sign, cudaStream_t st, int& nl,
                            double* cellbuf, const double* f = nullptr) {
  constexpr int N = P + 1, N2 = N * N, N3 = N2 * N;
  constexpr int CPB = (RM_Q_THREADS / N2) > 0 ? (RM_Q_THREADS / N2) : 1;
  const size_t smem = (size_t)CPB * 2 * N2 * (N + 1) * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(apply_q_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (cellbuf) {   // one launch over every cell (the skeleton gather follows)
    const long long ncell = (long long)op.n[0] * op.n[1] * op.n[2];
    apply_q_kernel<P><<<(unsigned)((ncell + CPB - 1) / CPB), CPB * N2, smem, st>>>(op, alpha, beta, coef_const, hpow, u,
                                                                                  out, sign, 0, 0, 0, cellbuf, f);
    ++nl;
    return cudaGetLastError();
  }
  for (int pz = 0; pz < 2; ++pz)
    for (int py = 0; py < 2; ++py)
      for (int px = 0; px < 2; ++px) {
        const long long ncell = (long long)((op.n[0] - px + 1) / 2) * ((op.n[1] - py + 1) / 2) * ((op.n[2] - pz + 1) / 2);
        if (ncell <= 0) continue;
        const unsigned grid = (unsigned)((ncell + CPB - 1) / CPB);
        apply_q_kernel<P><<<grid, CPB * N2, smem, st>>>(op, alpha, beta, coef_const, hpow, u, out, sign, px, py, pz,
                                                        nullptr, nullptr);
        ++nl;
      }
  return cudaGetLastError();
}

cudaError_t launch_apply_init(const OpParams& op, const double* f, double* out, long long ndof, cudaStream_t st) {
  apply_init_kernel<<<(unsigned)((ndof + 255) / 256), 256, 0, st>>>(op, f, out, ndof);
  return cudaGetLastError();
}

cudaError_t launch_apply_cartesian(const OpParams& op, const double* alpha, const double* beta, int coef_const,
                                   const double* hpow, const double* u, const double* f, double* out,
                                   long long ndof, cudaStream_t st, int* nlaunch, const KTimer* kt,
                                   double* cellbuf) {
  if (cellbuf && op.k == 0 && op.ncomp == 1 && !exp_env("RM_APPLY_PW")) {
    // H(grad): ONE launch of the line-stage kernel over every cell (cell-interior DoFs final,
    // out = f + sign A_K u; skeleton entries to the cell buffer), then the skeleton-only gather
    const double sgn = f ? -1.0 : 1.0;
    int nl = 0;
    cudaError_t e;
    if (kt) kt->begin(kt->arg);
    switch (op.p) {
#define RM_QC(PP) case PP: e = launch_q<PP>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, cellbuf, f); break;
      RM_QC(1) RM_QC(2) RM_QC(3) RM_QC(4) RM_QC(5) RM_QC(6) RM_QC(7) RM_QC(8)
      RM_QC(9) RM_QC(10) RM_QC(11) RM_QC(12) RM_QC(13) RM_QC(14) RM_QC(15)
#undef RM_QC
      default: e = cudaErrorInvalidValue;
    }
    if (kt) kt->end(kt->arg);
    if (e != cudaSuccess) return e;
    TriParams tp{};
    tp.p = op.p;
    for (int d = 0; d < 3; ++d) tp.n[d] = op.n[d];
    tp.Lx = op.len[0][0]; tp.Ly = op.len[0][1]; tp.Lz = op.len[0][2];
    tp.gamma_d = op.gamma_d;
    tp.ldx_out = op.ldx_out;
    e = launch_skeleton_gather_sc(tp, cellbuf, f, out, sgn, nullptr, st);
    if (nlaunch) *nlaunch = nl + 1;
    return e;
  }
  if (cellbuf && (op.k != 0 || exp_env("RM_APPLY_PW")))   // pointwise-stage kernels (apply_kform.cu) + gather, k = 1, 2
    return launch_apply_kform(op, alpha, beta, coef_const, hpow, u, f, out, ndof, cellbuf, st, nlaunch, kt);
  int nl = 1;
  if (op.ncomp == 1) apply_init_q_kernel<<<148 * 8, 256, 0, st>>>(op, f, out);
  else apply_init_kernel<<<(unsigned)((ndof + 255) / 256), 256, 0, st>>>(op, f, out, ndof);
  if (kt) kt->begin(kt->arg);
  struct End {
    const KTimer* kt;
    ~End() { if (kt) kt->end(kt->arg); }
  } end_{kt};
  if (op.k == 0) {
    const double sgn = f ? -1.0 : 1.0;
    cudaError_t e;
    switch (op.p) {
      case 1: e = launch_q<1>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 2: e = launch_q<2>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 3: e = launch_q<3>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 4: e = launch_q<4>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 5: e = launch_q<5>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 6: e = launch_q<6>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 7: e = launch_q<7>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 8: e = launch_q<8>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 9: e = launch_q<9>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 10: e = launch_q<10>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 11: e = launch_q<11>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 12: e = launch_q<12>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 13: e = launch_q<13>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      case 14: e = launch_q<14>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
      default: e = launch_q<15>(op, alpha, beta, coef_const, hpow, u, out, sgn, st, nl, nullptr); break;
    }
    if (nlaunch) *nlaunch = nl;
    return e;
  }
  const int P1 = op.p + 1;
  int nloc = 0;
  for (int m = 0; m < op.ncomp; ++m) {
    int s = 1;
    for (int d = 0; d < 3; ++d) s *= (op.fam[m][d] == FAMP ? P1 : op.p);
    nloc += s;
  }
  const size_t per_warp = (size_t)(2 * nloc + 2 * P1 * P1 * P1) * sizeof(double);
  constexpr int WPB = 4;
  const size_t smem = per_warp * WPB + RM_APPLY_TABLE_DOUBLES * sizeof(double);
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(apply_cells_kernel<WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  const double sign = f ? -1.0 : 1.0;
  for (int pz = 0; pz < 2; ++pz)
    for (int py = 0; py < 2; ++py)
      for (int px = 0; px < 2; ++px) {
        const long long ncell = (long long)((op.n[0] - px + 1) / 2) * ((op.n[1] - py + 1) / 2) * ((op.n[2] - pz + 1) / 2);
        if (ncell <= 0) continue;
        const unsigned grid = (unsigned)((ncell + WPB - 1) / WPB);
        apply_cells_kernel<WPB><<<grid, WPB * 32, smem, st>>>(op, alpha, beta, coef_const, hpow, u, out, sign, px, py, pz);
        ++nl;
      }
  if (nlaunch) *nlaunch = nl;
  return cudaGetLastError();
}

}  // namespace rm
