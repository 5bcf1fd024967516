// TEST INFRASTRUCTURE ONLY (never linked into librm.so): a host re-enactment of the packed
// patch programs built by paper_2211_14284_b200/csrc/patches.cpp, following the same steps as
// patch_solve_kernel (gather, forward eliminations, final block, back substitution, scatter),
// plus a host assembly of the Cartesian operator from the product's Kronecker term list.
// Lets the CPU test-suite check the product's setup (basis, term lists, classes, elimination
// schedules, ICC, packing) against the oracle without a GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "model.hpp"
#include "patches.hpp"

using namespace rm;

static void emulate_family(const PatchFamily& F, const double* r, double* z) {
  const size_t np = F.pclass.size();
  for (int color = 0; color < F.ncolors; ++color)
    for (size_t t = 0; t < np; ++t) {
      if (F.pcolor[t] != color) continue;
      const ClassProgram& C = F.classes[F.pclass[t]];
      const double* V = F.values.data() + F.pvals[t];
      const int n = C.n;
      std::vector<double> v(n);
      for (int q = 0; q < n; ++q) v[q] = r[F.pbase[3 * t + C.comp[q]] + C.offs[q]];
      auto sliced = [&](const Sliced& S, int row, const double* x) {
        double acc = 0;
        int sl = row / 32, l = row % 32;
        for (int kk = 0; kk < S.slice_w[sl]; ++kk) {
          int e = S.slice_off[sl] + kk * 32 + l;
          acc += V[S.vofs + e] * x[S.cols[e]];
        }
        return acc;
      };
      auto bval = [&](const Blocks& B, int slot, int i) { return V[B.vofs + (size_t)slot * B.nblk + i]; };
      for (const Level& L : C.lev) {
        const Blocks& B = L.blk;
        for (int i = 0; i < B.nblk; ++i) {   // y = L^{-1} v on the block
          int mm[3];
          for (int j = 0; j < 3; ++j) mm[j] = (j < B.bs) ? B.mem[(size_t)j * B.nblk + i] : 0xFFFF;
          double y[3];
          int slot = 0;
          for (int r = 0; r < B.bs; ++r) {
            double s = (mm[r] != 0xFFFF) ? v[mm[r]] : 0.0;
            for (int c = 0; c < r; ++c) s -= bval(B, slot + c, i) * y[c];
            y[r] = s * bval(B, slot + r, i);
            slot += r + 1;
            if (mm[r] != 0xFFFF) v[mm[r]] = y[r];
          }
        }
        for (int row = 0; row < L.w.nrows; ++row) v[L.w.r0 + row] -= sliced(L.w, row, v.data());
      }
      const int m = C.m, f0 = n - m;
      if (C.final_kind == FINAL_DENSE_INV) {
        const int T = (m + 31) / 32;
        std::vector<double> x(32 * T, 0.0), g(32 * T, 0.0);
        for (int i = 0; i < m; ++i) g[i] = v[f0 + i];
        for (int I = 0; I < T; ++I)
          for (int J = 0; J <= I; ++J) {
            const double* tb = V + C.vofs_final + (size_t)(I * (I + 1) / 2 + J) * 1024;
            for (int r = 0; r < 32; ++r)
              for (int c = 0; c < 32; ++c) {
                const double s = tb[r * 32 + ((c + r) & 31)];
                x[32 * I + r] += s * g[32 * J + c];
                if (I != J) x[32 * J + c] += s * g[32 * I + r];
              }
          }
        for (int i = 0; i < m; ++i) v[f0 + i] = x[i];
      } else {
        const double* Lv = V + C.vofs_final;
        const int nnz = C.icc_rowptr[m];
        const double* LTv = Lv + nnz;
        double* y = v.data() + f0;
        for (size_t l = 0; l + 1 < C.icc_level_ptr.size(); ++l)
          for (int q = C.icc_level_ptr[l]; q < C.icc_level_ptr[l + 1]; ++q) {
            int a = C.icc_level_rows[q];
            int t0 = C.icc_rowptr[a], t1 = C.icc_rowptr[a + 1] - 1;
            double s = y[a];
            for (int tt = t0; tt < t1; ++tt) s -= Lv[tt] * y[C.icc_col[tt]];
            y[a] = s * Lv[t1];
          }
        for (size_t l = 0; l + 1 < C.icct_level_ptr.size(); ++l)
          for (int q = C.icct_level_ptr[l]; q < C.icct_level_ptr[l + 1]; ++q) {
            int b = C.icct_level_rows[q];
            int t0 = C.icct_rowptr[b], t1 = C.icct_rowptr[b + 1];
            double s = y[b];
            for (int tt = t0 + 1; tt < t1; ++tt) s -= LTv[tt] * y[C.icct_col[tt]];
            y[b] = s * LTv[t0];
          }
      }
      for (int l = (int)C.lev.size() - 1; l >= 0; --l) {
        const Level& L = C.lev[l];
        std::vector<double> a(L.e1 - L.e0);
        for (int row = 0; row < L.wt.nrows; ++row) a[row] = v[L.e0 + row] - sliced(L.wt, row, v.data());
        const Blocks& B = L.blk;
        for (int i = 0; i < B.nblk; ++i) {   // x = L^{-T} a on the block
          int mm[3];
          for (int j = 0; j < 3; ++j) mm[j] = (j < B.bs) ? B.mem[(size_t)j * B.nblk + i] : 0xFFFF;
          double x[3] = {0, 0, 0};
          for (int r = B.bs - 1; r >= 0; --r) {
            if (mm[r] == 0xFFFF) continue;
            double s = a[mm[r] - L.e0];
            for (int c = r + 1; c < B.bs; ++c)
              if (mm[c] != 0xFFFF) s -= bval(B, c * (c + 1) / 2 + r, i) * x[c];
            x[r] = s * bval(B, r * (r + 1) / 2 + r, i);
            v[mm[r]] = x[r];
          }
        }
      }
      for (int q = 0; q < n; ++q) z[F.pbase[3 * t + C.comp[q]] + C.offs[q]] += v[q];
    }
}

extern "C" {

// z += P^{-1} r over one patch family on the uniform unit-cube grid (or the given coords).
int emu_precondition(int k, int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na,
                     const double* beta, long long nb, const double* coords, int dim, int fact, int interior_only,
                     const double* r, double* z, char* err, int errlen, long long* stats) {
  try {
    std::vector<double> h[3];
    const int n[3] = {nx, ny, nz};
    for (int d = 0; d < 3; ++d) h[d].assign(n[d], 1.0 / n[d]);
    SetupInput in{};
    in.k = k; in.p = p; in.n[0] = nx; in.n[1] = ny; in.n[2] = nz; in.gamma_d = gamma;
    in.coords = coords; in.alpha = alpha; in.beta = beta; in.n_alpha = na; in.n_beta = nb;
    in.dim = dim; in.factorization = fact; in.interior_only = interior_only;
    in.cartesian = (coords == nullptr);
    in.hx = h[0].data(); in.hy = h[1].data(); in.hz = h[2].data();
    auto F = build_patch_family(in);
    emulate_family(*F, r, z);
    if (stats) {
      stats[0] = (long long)F->pclass.size();
      stats[1] = (long long)F->classes.size();
      stats[2] = F->nfactors;
      long long nlev = 0, mfin = 0, nv = 0;
      for (auto& C : F->classes) { nlev = std::max<long long>(nlev, C.lev.size()); mfin = std::max<long long>(mfin, C.m); nv = std::max<long long>(nv, C.nvals); }
      stats[3] = nlev; stats[4] = mfin; stats[5] = nv;
    }
    return 0;
  } catch (const std::exception& e) {
    snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// Global Cartesian operator from the product's Kronecker term list (host assembly, COO out).
// Returns the number of entries written (or -needed if cap too small).
long long emu_assemble(int k, int p, int nx, int ny, int nz, const double* alpha, const double* beta,
                       long long* rows, long long* cols, double* vals, long long cap) {
  Space sp;
  sp.init(k, p, nx, ny, nz);
  CellOperator op = build_cell_operator(k, p);
  CellEntries e = cartesian_cell_entries(op, sp, 1.0 / nx, 1.0 / ny, 1.0 / nz);
  std::vector<int> lc, la[3];
  for (int m = 0; m < sp.ncomp; ++m)
    for (int c = 0; c < sp.lsize(m, 2); ++c)
      for (int b = 0; b < sp.lsize(m, 1); ++b)
        for (int a = 0; a < sp.lsize(m, 0); ++a) { lc.push_back(m); la[0].push_back(a); la[1].push_back(b); la[2].push_back(c); }
  long long cnt = 0;
  for (int cz = 0; cz < nz; ++cz)
    for (int cy = 0; cy < ny; ++cy)
      for (int cx = 0; cx < nx; ++cx) {
        const long long cell = ((long long)cz * ny + cy) * nx + cx;
        for (size_t t = 0; t < e.row.size(); ++t) {
          int i = e.row[t], j = e.col[t];
          if (cnt < cap) {
            rows[cnt] = sp.gidx(lc[i], (long long)cz * p + la[2][i], (long long)cy * p + la[1][i], (long long)cx * p + la[0][i]);
            cols[cnt] = sp.gidx(lc[j], (long long)cz * p + la[2][j], (long long)cy * p + la[1][j], (long long)cx * p + la[0][j]);
            vals[cnt] = alpha[cell] * e.kval[t] + beta[cell] * e.mval[t];
          }
          ++cnt;
        }
      }
  return cnt <= cap ? cnt : -cnt;
}

// 1D basis tables of the product (for cross-checks against the oracle's basis)
int emu_basis(int p, double* S, double* lam, double* B, double* A, double* D, double* G) {
  const Basis1D& b = basis(p);
  const int n = p + 1;
  std::memcpy(S, b.S.data(), sizeof(double) * n * n);
  std::memcpy(lam, b.lam.data(), sizeof(double) * n);
  std::memcpy(B, b.B.data(), sizeof(double) * n * n);
  std::memcpy(A, b.A.data(), sizeof(double) * n * n);
  std::memcpy(D, b.D.data(), sizeof(double) * p * n);
  std::memcpy(G, b.G.data(), sizeof(double) * n * n);
  return 0;
}

}  // extern "C"
