// Device side of the p = 1 coarse level (coarse.hpp): C_0 r = R_0^T A_0^{-1} R_0 r.
//
// R_0 / R_0^T are Kronecker products of 1D embeddings (P family: vertex rows identity, interior
// rows (s_a, (1 -+ x)/2); DP family: index c p <-> c), applied one direction at a time
// (transfer_kernel: one thread per output entry, <= 2p - 1 reads).  A_0^{-1} is the block
// forward / backward substitution with the stored dense blocks (row-per-warp GEMVs; lower / upper
// triangles skipped).
#include "kernels.cuh"

namespace rm {

namespace {

struct TransferDir {
  int d;                 // axis (0 x, 1 y, 2 z)
  int fam;               // 0 P, 1 DP
  int p, ncell;          // degree, cells along d
  int restrict_;         // 1: fine -> coarse (R_0), 0: coarse -> fine (R_0^T)
  int accumulate;        // prolongation into the output: out += result
  long long idim[3], odim[3];   // (x, y, z) extents of input / output
  double e0[16], e1[16];
};

__global__ void transfer_kernel(const __grid_constant__ TransferDir t, const double* __restrict__ in,
                                double* __restrict__ out) {
  const long long nout = t.odim[0] * t.odim[1] * t.odim[2];
  const int p = t.p;
  for (long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += (long long)gridDim.x * blockDim.x) {
    long long ix[3] = {o % t.odim[0], (o / t.odim[0]) % t.odim[1], o / (t.odim[0] * t.odim[1])};
    const long long sd = t.d == 0 ? 1 : (t.d == 1 ? t.idim[0] : t.idim[0] * t.idim[1]);
    const long long io = ix[t.d];
    ix[t.d] = 0;
    const double* base = in + (ix[2] * t.idim[1] + ix[1]) * t.idim[0] + ix[0];
    double v = 0.0;
    if (t.restrict_) {
      const long long c = io;
      if (t.fam == 1) {
        v = base[c * p * sd];
      } else {
        v = base[c * p * sd];
        for (int a = 1; a < p; ++a) {
          if (c < t.ncell) v += t.e0[a] * base[(c * p + a) * sd];
          if (c >= 1) v += t.e1[a] * base[((c - 1) * p + a) * sd];
        }
      }
    } else {
      const long long i = io;
      long long c = i / p;
      const int a = (int)(i - c * p);
      if (t.fam == 1) {
        v = a == 0 ? base[c * sd] : 0.0;
      } else {
        v = a == 0 ? base[c * sd] : t.e0[a] * base[c * sd] + t.e1[a] * base[(c + 1) * sd];
      }
    }
    if (t.accumulate) out[o] += v;
    else out[o] = v;
  }
}

// b[t] = mask[t] ? 0 : x[perm[t]]  (to block order)  /  x[perm[t]] = b[t]  (back)
__global__ void permute_kernel(const long long* __restrict__ perm, const unsigned char* __restrict__ mask,
                               const double* __restrict__ src, double* __restrict__ dst, long long n, int to_block) {
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    if (to_block) dst[t] = mask[t] ? 0.0 : src[perm[t]];
    else dst[perm[t]] = mask[t] ? 0.0 : src[t];
  }
}

// y[i] = (b ? b[i] : 0) + sign * sum_j M[i][j] x[j]; tri: 0 full, 1 lower (j <= i), 2 upper (j >= i)
__global__ void gemv_rows_kernel(const double* __restrict__ M, const double* __restrict__ x, const double* __restrict__ b,
                                 double* __restrict__ y, int nrows, int ncols, double sign, int tri) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= nrows) return;
  const int j0 = tri == 2 ? row : 0, j1 = tri == 1 ? row + 1 : ncols;
  const double* mr = M + (size_t)row * ncols;
  double s = 0.0;
  for (int j = j0 + lane; j < j1; j += 32) s += mr[j] * x[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = (b ? b[row] : 0.0) + sign * s;
}

void gemv(const double* M, const double* x, const double* b, double* y, int nrows, int ncols, double sign, int tri,
          cudaStream_t st) {
  const int wpb = 8;
  gemv_rows_kernel<<<(nrows + wpb - 1) / wpb, wpb * 32, 0, st>>>(M, x, b, y, nrows, ncols, sign, tri);
}

unsigned grid_for(long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 148LL * 32); }

}  // namespace

cudaError_t launch_coarse_correct(const CoarseLaunch& L, const double* r, double* z, cudaStream_t st) {
  // ---- restriction R_0 r, component by component, x then y then z, into the coarse layout
  for (int m = 0; m < L.ncomp; ++m) {
    long long dims[3] = {L.len[m][0], L.len[m][1], L.len[m][2]};
    const double* src = r + L.off[m];
    for (int d = 0; d < 3; ++d) {
      TransferDir t{};
      t.d = d; t.fam = L.fam[m][d]; t.p = L.p; t.ncell = L.n[d]; t.restrict_ = 1; t.accumulate = 0;
      for (int q = 0; q < 3; ++q) { t.idim[q] = dims[q]; t.odim[q] = dims[q]; }
      t.odim[d] = L.len1[m][d];
      for (int a = 0; a < 16; ++a) { t.e0[a] = L.e0[a]; t.e1[a] = L.e1[a]; }
      double* dst = d == 2 ? L.xc + L.off1[m] : (d == 0 ? L.tA : L.tB);
      const long long no = t.odim[0] * t.odim[1] * t.odim[2];
      transfer_kernel<<<grid_for(no), 256, 0, st>>>(t, src, dst);
      src = dst;
      dims[d] = L.len1[m][d];
    }
  }
  // ---- A_0^{-1} in block order (constrained coarse DoFs held at zero)
  permute_kernel<<<grid_for(L.ndof1), 256, 0, st>>>(L.perm, L.cmask, L.xc, L.b, L.ndof1, 1);
  for (int j = 0; j < L.nb; ++j) {   // forward: y_j = Linv_j (b_j - L_{j,j-1} y_{j-1})
    const int m = L.bstart[j + 1] - L.bstart[j];
    const double* bj = L.b + L.bstart[j];
    if (j > 0) {
      const int mp = L.bstart[j] - L.bstart[j - 1];
      gemv(L.vals + L.o_lsub[j - 1], L.y + L.bstart[j - 1], bj, L.t, m, mp, -1.0, 0, st);
      bj = L.t;
    }
    gemv(L.vals + L.o_linv[j], bj, nullptr, L.y + L.bstart[j], m, m, 1.0, 1, st);
  }
  for (int j = L.nb - 1; j >= 0; --j) {   // backward: x_j = Linv_j^T (y_j - L_{j+1,j}^T x_{j+1})
    const int m = L.bstart[j + 1] - L.bstart[j];
    const double* yj = L.y + L.bstart[j];
    if (j + 1 < L.nb) {
      const int mn = L.bstart[j + 2] - L.bstart[j + 1];
      gemv(L.vals + L.o_lsubt[j], L.b + L.bstart[j + 1], yj, L.t, m, mn, -1.0, 0, st);
      yj = L.t;
    }
    gemv(L.vals + L.o_linvt[j], yj, nullptr, L.b + L.bstart[j], m, m, 1.0, 2, st);   // x overwrites b
  }
  permute_kernel<<<grid_for(L.ndof1), 256, 0, st>>>(L.perm, L.cmask, L.b, L.xc, L.ndof1, 0);
  // ---- prolongation z += R_0^T x, component by component, z then y then x (the last accumulates)
  for (int m = 0; m < L.ncomp; ++m) {
    long long dims[3] = {L.len1[m][0], L.len1[m][1], L.len1[m][2]};
    const double* src = L.xc + L.off1[m];
    for (int d = 2; d >= 0; --d) {
      TransferDir t{};
      t.d = d; t.fam = L.fam[m][d]; t.p = L.p; t.ncell = L.n[d]; t.restrict_ = 0; t.accumulate = d == 0;
      for (int q = 0; q < 3; ++q) { t.idim[q] = dims[q]; t.odim[q] = dims[q]; }
      t.odim[d] = L.len[m][d];
      for (int a = 0; a < 16; ++a) { t.e0[a] = L.e0[a]; t.e1[a] = L.e1[a]; }
      double* dst = d == 0 ? z + L.off[m] : (d == 2 ? L.tA : L.tB);
      const long long no = t.odim[0] * t.odim[1] * t.odim[2];
      transfer_kernel<<<grid_for(no), 256, 0, st>>>(t, src, dst);
      src = dst;
      dims[d] = L.len[m][d];
    }
  }
  return cudaGetLastError();
}

}  // namespace rm
