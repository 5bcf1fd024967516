// TEST INFRASTRUCTURE ONLY (never linked into librm.so): a host re-enactment of the packed
// patch programs built by paper_2211_14284_b200/csrc/patches.cpp, following the same steps as
// patch_solve_kernel (gather, forward eliminations, final block, back substitution, scatter),
// plus a host assembly of the Cartesian operator from the product's Kronecker term list.
// Lets the CPU test-suite check the product's setup (basis, term lists, classes, elimination
// schedules, ICC, packing) against the oracle without a GPU.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "model.hpp"
#include "patches.hpp"
#include "coarse.hpp"

using namespace rm;

// Re-enacts patch_stream_kernel on the STREAM layout (patches.hpp): every index comes from the
// pieces' metadata blocks (class meta stream) and every value from the pieces of the patch value
// block, in piece order, exactly as the kernel's shared-memory ring presents them.
struct PieceView {
  const uint8_t* pb;      // metadata block
  const double* val;      // values
  int a0, a1, e0, mbytes, nd;
};
// Builds every piece's view the way the kernel sees it: per transfer unit, one buffer holding
// [metas of the unit's pieces][values of the unit's pieces]; inside it the consumer walks the
// pieces with a meta cursor and a value cursor advanced by the header's (mbytes, nd).
static std::vector<PieceView> unit_views(const ClassProgram& C, const double* V, std::vector<std::vector<uint8_t>>& bufs) {
  std::vector<PieceView> out(C.pieces.size());
  bufs.assign(C.units.size(), {});
  for (size_t k = 0; k < C.units.size(); ++k) {
    const Unit& u = C.units[k];
    std::vector<uint8_t>& b = bufs[k];
    b.resize((size_t)u.mbytes + (size_t)u.nd * 8 + 16);
    std::memcpy(b.data(), C.meta.data() + u.mofs, u.mbytes);
    std::memcpy(b.data() + u.mbytes, V + u.sofs, (size_t)u.nd * 8);
    const uint8_t* mcur = b.data();
    const uint8_t* vcur = b.data() + u.mbytes;
    for (int i = u.p0; i < u.p0 + u.np; ++i) {
      PieceView w;
      int32_t h[4];
      std::memcpy(h, mcur, 16);
      w.pb = mcur; w.a0 = h[0]; w.a1 = h[1]; w.e0 = h[2];
      w.mbytes = (int)((uint32_t)h[3] & 0xFFFFu); w.nd = (int)((uint32_t)h[3] >> 16);
      if (w.mbytes != C.pieces[i].mbytes || w.nd != C.pieces[i].nd) throw std::runtime_error("meta header mismatch");
      w.val = reinterpret_cast<const double*>(vcur);
      out[i] = w;
      mcur += w.mbytes;
      vcur += (size_t)w.nd * 8;
    }
  }
  return out;
}
template <class T> static T rd(const uint8_t* b, size_t i) { T x; std::memcpy(&x, b + i * sizeof(T), sizeof(T)); return x; }

static void emulate_family(const PatchFamily& F, const double* r_in, double* z_out) {
  const size_t np = F.pclass.size();
  const Space& sp = F.sp;
  // static condensation (sc): r_sc = r - sum_K R_K^T P_GI P_II^{-1} r_I on face DoFs; the patches
  // solve on the interface only; post: c_I = n_K P_II^{-1} r_I - P_II^{-1} P_IG c_G per cell
  const bool sc = !F.sc_nk.empty();
  const int p = sp.p, pm = p - 1, ni = pm * pm * pm;
  auto cell_dof = [&](int cx, int cy, int cz, int a, int b, int c) {
    return sp.gidx(0, (int64_t)cz * p + c, (int64_t)cy * p + b, (int64_t)cx * p + a);
  };
  auto face_dof = [&](int cx, int cy, int cz, int face, int i, int j, int k) {
    const int a = face == 0 ? 0 : face == 1 ? p : i, b = face == 2 ? 0 : face == 3 ? p : j, c = face == 4 ? 0 : face == 5 ? p : k;
    return cell_dof(cx, cy, cz, a, b, c);
  };
  std::vector<double> rsc(r_in, r_in + sp.ndof()), cacc(sp.ndof(), 0.0);
  if (sc && F.sc_pre)   // (SC-PAFW with the exact program: the patch elimination does the pre step)
    for (int cz = 0; cz < sp.n[2]; ++cz)
      for (int cy = 0; cy < sp.n[1]; ++cy)
        for (int cx = 0; cx < sp.n[0]; ++cx) {
          const int64_t K = ((int64_t)cz * sp.n[1] + cy) * sp.n[0] + cx;
          for (int k = 1; k < p; ++k)
            for (int j = 1; j < p; ++j)
              for (int i = 1; i < p; ++i) {
                const int I = ((k - 1) * pm + (j - 1)) * pm + (i - 1);
                const double y = r_in[cell_dof(cx, cy, cz, i, j, k)] * F.sc_dinv[(size_t)K * ni + I];
                for (int f = 0; f < 6; ++f) rsc[face_dof(cx, cy, cz, f, i, j, k)] -= F.sc_coupling(K, f, I, ni, f < 2 ? i : (f < 4 ? j : k)) * y;
              }
        }
  const double* r = rsc.data();
  double* z = cacc.data();
  for (int color = 0; color < F.ncolors; ++color)
    for (size_t t = 0; t < np; ++t) {
      if (F.pcolor[t] != color) continue;
      const ClassProgram& C = F.classes[F.pclass[t]];
      const double* V = F.values.data() + F.pvals[t];
      std::vector<std::vector<uint8_t>> bufs;
      const std::vector<PieceView> views = unit_views(C, V, bufs);
      auto view = [&](int i) { return views[i]; };
      const int L = (int)C.lev.size();
      // ---- gather: TMA box load of every component window (out of bounds -> 0)
      std::vector<double> v(F.box_total, 0.0);
      auto box_walk = [&](auto&& fn) {
        for (int sb = 0; sb < F.nsub; ++sb) {
          const int m = F.sub_comp[sb];
          const int* o = &F.porig[t * 9 + sb * 3];
          for (int bz = 0; bz < F.box[sb][2]; ++bz)
            for (int by = 0; by < F.box[sb][1]; ++by)
              for (int bx = 0; bx < F.box[sb][0]; ++bx) {
                const int64_t gx = o[0] + bx, gy = o[1] + by, gz = o[2] + bz;
                const int b = F.boff[sb] + (bz * F.box[sb][1] + by) * F.box[sb][0] + bx;
                if (gx < sp.len(m, 0) && gy < sp.len(m, 1) && gz < sp.len(m, 2)) fn(b, sp.gidx(m, gz, gy, gx));
              }
        }
      };
      box_walk([&](int b, int64_t g) { v[b] = r[g]; });
      // sliced piece: per slice (start/32, count); per slice 32 row boxes; column boxes
      auto sliced_piece = [&](const PieceView& w, auto&& emit) {
        const int nsl = w.a1 - w.a0;
        const uint8_t* rows = w.pb + 16 + 4 * nsl;
        const uint8_t* cols = rows + 64 * nsl;
        for (int ls = 0; ls < nsl; ++ls) {
          const uint32_t info = rd<uint32_t>(w.pb + 16, ls);
          const int st = 32 * (int)(info & 0xFFFF), cnt = (int)(info >> 16);
          for (int lane = 0; lane < 32; ++lane) {
            double acc = 0;
            for (int kk = 0; kk < cnt; ++kk) {
              const int e = st + kk * 32 + lane;
              acc += w.val[e] * v[rd<uint16_t>(cols, e)];
            }
            emit(ls, lane, rd<uint16_t>(rows, ls * 32 + lane), acc);
          }
        }
      };
      for (int l = 0; l < L; ++l) {
        const Level& Lv = C.lev[l];
        const int bs = Lv.blk.bs;
        for (int pi = C.piv_b[l]; pi < C.w_b[l]; ++pi) {
          PieceView w = view(pi);
          const int cnt = w.a1 - w.a0;
          auto pc = [&](int slot, int li) { return w.val[slot * cnt + li]; };
          for (int li = 0; li < cnt; ++li) {
            int mm[3];
            for (int j = 0; j < 3; ++j) mm[j] = (j < bs) ? rd<uint16_t>(w.pb + 16, (size_t)j * cnt + li) : 0xFFFF;
            double y[3] = {0, 0, 0};
            for (int rr = 0; rr < bs; ++rr) {   // y = L^{-1} v
              if (mm[rr] == 0xFFFF) continue;
              double s = v[mm[rr]];
              for (int c = 0; c < rr; ++c) s -= pc(rr * (rr + 1) / 2 + c, li) * y[c];
              y[rr] = s * pc(rr * (rr + 1) / 2 + rr, li);
            }
            for (int rr = bs - 1; rr >= 0; --rr) {   // y^ = L^{-T} y
              if (mm[rr] == 0xFFFF) continue;
              double s = y[rr];
              for (int c = rr + 1; c < bs; ++c)
                if (mm[c] != 0xFFFF) s -= pc(c * (c + 1) / 2 + rr, li) * y[c];
              y[rr] = s * pc(rr * (rr + 1) / 2 + rr, li);
              v[mm[rr]] = y[rr];
            }
          }
        }
        for (int pi = C.w_b[l]; pi < C.w_e[l]; ++pi) {
          PieceView w = view(pi);
          sliced_piece(w, [&](int ls, int lane, int rb, double acc) {
            if ((w.a0 + ls) * 32 + lane < Lv.w.nrows) v[rb] -= acc;
          });
        }
      }
      const int m = C.m;
      if (C.final_kind == FINAL_DENSE_INV) {
        if (m > 0) {
          const int T = (m + 31) / 32;
          PieceView fw = view(C.tile_p0);
          std::vector<int> fb(m);
          for (int j = 0; j < m; ++j) fb[j] = rd<uint16_t>(fw.pb + 16, j);
          std::vector<double> x(32 * T, 0.0), g(32 * T, 0.0);
          for (int i = 0; i < m; ++i) g[i] = v[fb[i]];
          for (int pi = C.tile_p0 + 1; pi < C.tile_p1; ++pi) {
            PieceView w = view(pi);
            const int I = w.a0, J = w.a1;
            const double* tb = w.val;
            for (int rr = 0; rr < 32; ++rr)   // tile = S (off-diagonal) or L' with S = L' + L'^T (diagonal)
              for (int c = 0; c < 32; ++c) {
                if (I == J && c > rr) continue;
                const double s = (I == J) ? tb[tile_pos_diag(rr, c)] : tb[tile_pos_full(rr, c)];
                x[32 * I + rr] += s * g[32 * J + c];
                x[32 * J + c] += s * g[32 * I + rr];
              }
          }
          for (int i = 0; i < m; ++i) v[fb[i]] = x[i];
        }
      } else {
        for (int pi = C.tile_p0; pi < C.tile_p1; ++pi) {   // multi-chunk lane-interleaved ICC pieces
          PieceView w = view(pi);
          const int nch = w.a1 - w.a0;
          for (int c = 0; c < nch; ++c) {
            const int cnt = rd<int32_t>(w.pb + 16, 4 * c), Lm = rd<int32_t>(w.pb + 16, 4 * c + 1);
            const int mo = rd<int32_t>(w.pb + 16, 4 * c + 2), vo = rd<int32_t>(w.pb + 16, 4 * c + 3);
            const uint8_t* rows = w.pb + mo;
            const uint8_t* cols = rows + 64;
            const double* val = w.val + vo;
            for (int k = 0; k < cnt; ++k) {   // same arithmetic order as the kernel
              const int a = rd<uint16_t>(rows, k);
              double s0 = v[a], s1 = 0.0;
              for (int j = 0; j < Lm; ++j) {
                const double x = v[rd<uint16_t>(cols, 32 * j + k)], wv = val[32 + 32 * j + k];
                if (j & 1) s1 = std::fma(-wv, x, s1);
                else s0 = std::fma(-wv, x, s0);
              }
              v[a] = (s0 + s1) * val[k];
            }
          }
        }
      }
      for (int l = L - 1; l >= 0; --l) {   // x_E = y^_E - W^ x_R, in place
        const Level& Lv = C.lev[l];
        std::vector<std::pair<int, double>> upd;
        for (int pi = C.wt_b[l]; pi < C.wt_e[l]; ++pi) {
          PieceView w = view(pi);
          sliced_piece(w, [&](int ls, int lane, int rb, double acc) {
            if ((w.a0 + ls) * 32 + lane < Lv.wt.nrows) upd.push_back({rb, acc});
          });
        }
        for (auto& pr : upd) v[pr.first] -= pr.second;
      }
      // ---- scatter: zero the non-patch box entries, TMA reduce-add of the boxes
      PieceView zw = view((int)C.pieces.size() - 1);
      for (int k = 0; k < zw.a1 - zw.a0; ++k) v[rd<uint16_t>(zw.pb + 16, k)] = 0.0;
      box_walk([&](int b, int64_t g) { z[g] += v[b]; });
    }
  if (sc)
    for (int cz = 0; cz < sp.n[2]; ++cz)
      for (int cy = 0; cy < sp.n[1]; ++cy)
        for (int cx = 0; cx < sp.n[0]; ++cx) {
          const int64_t K = ((int64_t)cz * sp.n[1] + cy) * sp.n[0] + cx;
          for (int k = 1; k < p; ++k)
            for (int j = 1; j < p; ++j)
              for (int i = 1; i < p; ++i) {
                const int I = ((k - 1) * pm + (j - 1)) * pm + (i - 1);
                const double dinv = F.sc_dinv[(size_t)K * ni + I];
                double s = 0.0;
                for (int f = 0; f < 6; ++f) s += F.sc_coupling(K, f, I, ni, f < 2 ? i : (f < 4 ? j : k)) * cacc[face_dof(cx, cy, cz, f, i, j, k)];
                cacc[cell_dof(cx, cy, cz, i, j, k)] = F.sc_nk[K] * r_in[cell_dof(cx, cy, cz, i, j, k)] * dinv - dinv * s;
              }
        }
  for (int64_t g = 0; g < sp.ndof(); ++g) z_out[g] += cacc[g];
}

extern "C" {

// z += P^{-1} r over one patch family on the uniform unit-cube grid (or the given coords).
static int emu_precondition_impl(int k, int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na,
                                 const double* beta, long long nb, const double* coords, int dim, int fact,
                                 int interior_only, int zv_lo, int zv_hi, const double* hz, const double* r,
                                 double* z, char* err, int errlen, long long* stats);

int emu_precondition(int k, int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na,
                     const double* beta, long long nb, const double* coords, int dim, int fact, int interior_only,
                     const double* r, double* z, char* err, int errlen, long long* stats) {
  return emu_precondition_impl(k, p, nx, ny, nz, gamma, alpha, na, beta, nb, coords, dim, fact, interior_only, 0,
                               1 << 30, nullptr, r, z, err, errlen, stats);
}

// same, keeping only the vertex stars of the z vertex layers [zv_lo, zv_hi) (z-slab ownership);
// hz: z cell sizes of an axis-aligned slab (coords == NULL), NULL = 1/nz
int emu_precondition_zv(int k, int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na,
                        const double* beta, long long nb, const double* coords, int dim, int fact, int zv_lo,
                        int zv_hi, const double* hz, const double* r, double* z, char* err, int errlen) {
  return emu_precondition_impl(k, p, nx, ny, nz, gamma, alpha, na, beta, nb, coords, dim, fact, 0, zv_lo, zv_hi, hz, r,
                               z, err, errlen, nullptr);
}

static int emu_precondition_impl(int k, int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na,
                                 const double* beta, long long nb, const double* coords, int dim, int fact,
                                 int interior_only, int zv_lo, int zv_hi, const double* hz, const double* r,
                                 double* z, char* err, int errlen, long long* stats) {
  try {
    std::vector<double> h[3];
    const int n[3] = {nx, ny, nz};
    for (int d = 0; d < 3; ++d) h[d].assign(n[d], 1.0 / n[d]);
    if (hz) h[2].assign(hz, hz + nz);
    SetupInput in{};
    in.k = k; in.p = p; in.n[0] = nx; in.n[1] = ny; in.n[2] = nz; in.gamma_d = gamma;
    in.coords = coords; in.alpha = alpha; in.beta = beta; in.n_alpha = na; in.n_beta = nb;
    in.dim = dim; in.factorization = fact; in.interior_only = interior_only & 1;
    in.sc_decomposition = (interior_only & 2) != 0;   // bit 1: SC-PAFW
    in.cartesian = (coords == nullptr);
    in.hx = h[0].data(); in.hy = h[1].data(); in.hz = h[2].data();
    in.zv_lo = zv_lo; in.zv_hi = zv_hi;
    auto F = build_patch_family(in);
    emulate_family(*F, r, z);
    if (stats) {
      stats[0] = (long long)F->pclass.size();
      stats[1] = (long long)F->classes.size();
      stats[2] = F->nfactors;
      long long nlev = 0, mfin = 0, nv = 0;
      for (auto& C : F->classes) { nlev = std::max<long long>(nlev, C.lev.size()); mfin = std::max<long long>(mfin, C.m); nv = std::max<long long>(nv, C.nvals); }
      stats[3] = nlev; stats[4] = mfin; stats[5] = nv;
      if (stats[6] == -1) {   // extended stats requested: window box, largest units (bytes) per channel
        long long ua = 0, ub = 0;
        for (auto& C : F->classes)
          for (size_t u = 0; u < C.units.size(); ++u) {
            const bool tile = (int)u >= C.tu0 && (int)u < C.tu1;
            const long long by = C.units[u].mbytes + 8LL * C.units[u].nd;
            if (tile) ub = std::max(ub, by); else ua = std::max(ua, by);
          }
        stats[6] = F->box_total; stats[7] = ua; stats[8] = ub;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// r_sc = r - sum_K R_K^T P_GI P_II^{-1} r_I of an ICC-SC family (static condensation, pre step)
int emu_sc_pre(int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na, const double* beta,
               long long nb, const double* coords, const double* r, double* rsc) {
  std::vector<double> h[3];
  const int n[3] = {nx, ny, nz};
  for (int d = 0; d < 3; ++d) h[d].assign(n[d], 1.0 / n[d]);
  SetupInput in{};
  in.k = 0; in.p = p; in.n[0] = nx; in.n[1] = ny; in.n[2] = nz; in.gamma_d = gamma;
  in.coords = coords; in.alpha = alpha; in.beta = beta; in.n_alpha = na; in.n_beta = nb;
  in.dim = 0; in.factorization = 1; in.interior_only = 0;
  in.cartesian = (coords == nullptr);
  in.hx = h[0].data(); in.hy = h[1].data(); in.hz = h[2].data();
  auto F = build_patch_family(in);
  const Space& sp = F->sp;
  const int pm = p - 1, ni = pm * pm * pm;
  for (int64_t g = 0; g < sp.ndof(); ++g) rsc[g] = r[g];
  auto cd = [&](int cx, int cy, int cz, int a, int b, int c) { return sp.gidx(0, (int64_t)cz * p + c, (int64_t)cy * p + b, (int64_t)cx * p + a); };
  for (int cz = 0; cz < nz; ++cz)
    for (int cy = 0; cy < ny; ++cy)
      for (int cx = 0; cx < nx; ++cx) {
        const int64_t K = ((int64_t)cz * ny + cy) * nx + cx;
        for (int k = 1; k < p; ++k)
          for (int j = 1; j < p; ++j)
            for (int i = 1; i < p; ++i) {
              const int I = ((k - 1) * pm + (j - 1)) * pm + (i - 1);
              const double y = r[cd(cx, cy, cz, i, j, k)] * F->sc_dinv[(size_t)K * ni + I];
              const int fa[6][3] = {{0, j, k}, {p, j, k}, {i, 0, k}, {i, p, k}, {i, j, 0}, {i, j, p}};
              for (int f = 0; f < 6; ++f) rsc[cd(cx, cy, cz, fa[f][0], fa[f][1], fa[f][2])] -= F->sc_coupling(K, f, I, ni, f < 2 ? i : (f < 4 ? j : k)) * y;
            }
      }
  return 0;
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

// SURVEY 8(d) algorithmic factor entries of a family (alpha = beta = 1, uniform grid):
// out[0] = sum over patches of nnz(L), out[1] = patches, out[2] = largest class nnz(L)
int emu_family_nnz(int k, int p, int nx, int ny, int nz, unsigned gamma, int dim, int fact, int interior_only,
                   long long* out, char* err, int errlen) {
  try {
    std::vector<double> h[3];
    const int n[3] = {nx, ny, nz};
    for (int d = 0; d < 3; ++d) h[d].assign(n[d], 1.0 / n[d]);
    const double one = 1.0;
    SetupInput in{};
    in.k = k; in.p = p; in.n[0] = nx; in.n[1] = ny; in.n[2] = nz; in.gamma_d = gamma;
    in.coords = nullptr; in.alpha = &one; in.beta = &one; in.n_alpha = 1; in.n_beta = 1;
    in.dim = dim; in.factorization = fact; in.interior_only = interior_only & 1;
    in.sc_decomposition = (interior_only & 2) != 0;   // bit 1: SC-PAFW
    in.cartesian = true;
    in.hx = h[0].data(); in.hy = h[1].data(); in.hz = h[2].data();
    auto F = build_patch_family(in);
    out[0] = F->nnzL_total;
    out[1] = (long long)F->pclass.size();
    long long mx = 0;
    for (auto& C : F->classes) mx = std::max<long long>(mx, C.nnzL);
    out[2] = mx;
    return 0;
  } catch (const std::exception& e) {
    snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// z = R_0^T A_0^{-1} R_0 r with the product's host coarse factor (coarse.cpp), re-enacting
// launch_coarse_correct (coarse.cu) on the host: restriction by the 1D embedding tables, block
// forward / backward substitution with the stored Linv / Lsub blocks, prolongation.
int emu_coarse(int k, int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na,
               const double* beta, long long nb_, const double* coords, const double* r, double* z, char* err,
               int errlen) {
  try {
    std::vector<double> h[3];
    const int n[3] = {nx, ny, nz};
    for (int d = 0; d < 3; ++d) h[d].assign(n[d], 1.0 / n[d]);
    CoarseSetupInput in{};
    in.k = k; in.p = p; in.n[0] = nx; in.n[1] = ny; in.n[2] = nz; in.gamma_d = gamma; in.coords = coords;
    in.cartesian = coords == nullptr; in.hx = h[0].data(); in.hy = h[1].data(); in.hz = h[2].data();
    in.alpha = alpha; in.beta = beta; in.n_alpha = na; in.n_beta = nb_;
    CoarseFactor F;
    build_coarse(in, F);
    Space sp;
    sp.init(k, p, nx, ny, nz);
    const Space& s1 = F.sp1;
    // 1D embedding E[i][c] of one direction
    auto E = [&](int fam, int i, int c) -> double {
      if (fam == FAM_D) return (i == c * p) ? 1.0 : 0.0;
      const int cc = i / p, a = i - cc * p;
      if (a == 0) return cc == c ? 1.0 : 0.0;
      if (c == cc) return F.e0[a];
      if (c == cc + 1) return F.e1[a];
      return 0.0;
    };
    std::vector<double> xc(F.ndof1, 0.0);
    for (int m = 0; m < sp.ncomp; ++m)
      for (int64_t Z = 0; Z < s1.len(m, 2); ++Z)
        for (int64_t Y = 0; Y < s1.len(m, 1); ++Y)
          for (int64_t X = 0; X < s1.len(m, 0); ++X) {
            double acc = 0.0;
            for (int64_t iz = std::max<int64_t>(0, (Z - 1) * p); iz <= std::min<int64_t>(sp.len(m, 2) - 1, (Z + 1) * p); ++iz) {
              const double ez = E(sp.fam[m][2], (int)iz, (int)Z);
              if (ez == 0.0) continue;
              for (int64_t iy = std::max<int64_t>(0, (Y - 1) * p); iy <= std::min<int64_t>(sp.len(m, 1) - 1, (Y + 1) * p); ++iy) {
                const double ey = E(sp.fam[m][1], (int)iy, (int)Y);
                if (ey == 0.0) continue;
                for (int64_t ix = std::max<int64_t>(0, (X - 1) * p); ix <= std::min<int64_t>(sp.len(m, 0) - 1, (X + 1) * p); ++ix) {
                  const double ex = E(sp.fam[m][0], (int)ix, (int)X);
                  if (ex != 0.0) acc += ex * ey * ez * r[sp.gidx(m, iz, iy, ix)];
                }
              }
            }
            xc[s1.gidx(m, Z, Y, X)] = acc;
          }
    const int nb = (int)F.bstart.size() - 1;
    std::vector<double> b(F.ndof1), y(F.ndof1), x(F.ndof1), t;
    for (int64_t q = 0; q < F.ndof1; ++q) b[q] = F.cmask[q] ? 0.0 : xc[F.perm[q]];
    auto gemv = [&](const double* M, const double* v, int rows, int cols, double* out, const double* add, double sg) {
      for (int i = 0; i < rows; ++i) {
        double s = 0.0;
        for (int j = 0; j < cols; ++j) s += M[(size_t)i * cols + j] * v[j];
        out[i] = (add ? add[i] : 0.0) + sg * s;
      }
    };
    for (int j = 0; j < nb; ++j) {
      const int m = F.bstart[j + 1] - F.bstart[j];
      std::vector<double> rhs(b.begin() + F.bstart[j], b.begin() + F.bstart[j + 1]);
      if (j > 0) {
        const int mp = F.bstart[j] - F.bstart[j - 1];
        gemv(&F.vals[F.o_lsub[j - 1]], &y[F.bstart[j - 1]], m, mp, rhs.data(), rhs.data(), -1.0);
      }
      gemv(&F.vals[F.o_linv[j]], rhs.data(), m, m, &y[F.bstart[j]], nullptr, 1.0);
    }
    for (int j = nb - 1; j >= 0; --j) {
      const int m = F.bstart[j + 1] - F.bstart[j];
      std::vector<double> rhs(y.begin() + F.bstart[j], y.begin() + F.bstart[j + 1]);
      if (j + 1 < nb) {
        const int mn = F.bstart[j + 2] - F.bstart[j + 1];
        gemv(&F.vals[F.o_lsubt[j]], &x[F.bstart[j + 1]], m, mn, rhs.data(), rhs.data(), -1.0);
      }
      gemv(&F.vals[F.o_linvt[j]], rhs.data(), m, m, &x[F.bstart[j]], nullptr, 1.0);
    }
    std::fill(xc.begin(), xc.end(), 0.0);
    for (int64_t q = 0; q < F.ndof1; ++q) xc[F.perm[q]] = F.cmask[q] ? 0.0 : x[q];
    for (int m = 0; m < sp.ncomp; ++m)
      for (int64_t iz = 0; iz < sp.len(m, 2); ++iz)
        for (int64_t iy = 0; iy < sp.len(m, 1); ++iy)
          for (int64_t ix = 0; ix < sp.len(m, 0); ++ix) {
            double acc = 0.0;
            for (int64_t Z = iz / p; Z <= std::min<int64_t>(s1.len(m, 2) - 1, iz / p + 1); ++Z)
              for (int64_t Y = iy / p; Y <= std::min<int64_t>(s1.len(m, 1) - 1, iy / p + 1); ++Y)
                for (int64_t X = ix / p; X <= std::min<int64_t>(s1.len(m, 0) - 1, ix / p + 1); ++X)
                  acc += E(sp.fam[m][0], (int)ix, (int)X) * E(sp.fam[m][1], (int)iy, (int)Y) * E(sp.fam[m][2], (int)iz, (int)Z) *
                         xc[s1.gidx(m, Z, Y, X)];
            z[sp.gidx(m, iz, iy, ix)] = acc;
          }
    return 0;
  } catch (const std::exception& e) {
    snprintf(err, errlen, "%s", e.what());
    return 1;
  }
}

// values per piece kind (PIV, W, TILE, ICCF, ICCB, WT, FINAL, ZERO) of the largest class of a family
// (diagnostic of the stream layout), plus its n, m, levels
int emu_family_breakdown(int k, int p, int nx, int dim, int orient, long long* out) {
  std::vector<double> h(nx, 1.0 / nx);
  const double one = 1.0;
  SetupInput in{};
  in.k = k; in.p = p; in.n[0] = in.n[1] = in.n[2] = nx; in.gamma_d = 63;
  in.coords = nullptr; in.alpha = &one; in.beta = &one; in.n_alpha = 1; in.n_beta = 1;
  in.dim = dim; in.factorization = 0; in.interior_only = 1; in.cartesian = true;
  in.hx = h.data(); in.hy = h.data(); in.hz = h.data(); in.orient = orient;
  auto F = build_patch_family(in);
  const ClassProgram* best = nullptr;
  for (auto& C : F->classes) if (!best || C.nvals > best->nvals) best = &C;
  for (int q = 0; q < 12; ++q) out[q] = 0;
  if (!best) return 1;
  for (auto& pc : best->pieces) out[pc.kind] += pc.nd;
  out[8] = best->n; out[9] = best->m; out[10] = (long long)best->lev.size(); out[11] = best->nvals;
  return 0;
}

// Host re-enactment of the DEVICE numeric setup program (patches.hpp NumProg, executed by
// dsetup.cu factor_kernel): evaluates every value block from the program's assembly lists,
// level-0 records, Schur targets, a dense Cholesky of S, the level recipes, the final inverse /
// ICC(0) and the stream map, and compares with the host factorization (factor_patch) of the same
// family.  Returns the largest |difference| / max|value| over all blocks in *rel (-1 on error).
static void numprog_eval(const NumProg& g, const PatchFamily& F, int f, const std::vector<double>& cent_all,
                         int ne, double* out) {
  const int* cells = F.fcells.data() + (size_t)f * kMaxSlots;
  std::vector<double> Pv(g.nnzP), C(g.ncanon, 0.0), M(3 * (g.nbr.size() / 7), 0.0);
  for (int e = 0; e < g.nnzP; ++e) {
    double v = 0.0;
    for (int k = g.asm_ptr[e]; k < g.asm_ptr[e + 1]; ++k) {
      const int src = g.asm_src[k], sl = src / ne, t = src % ne, cell = cells[sl];
      if (F.cartesian) {
        const size_t so = (size_t)F.cell_set[cell] * ne + t;
        v += F.cell_alpha[cell] * F.cset_k[so] + F.cell_beta[cell] * F.cset_m[so];
      } else {
        v += cent_all[(size_t)cell * ne + t];
      }
    }
    Pv[e] = v;
  }
  auto pv = [&](int x) { return x < 0 ? 0.0 : Pv[x]; };
  for (int bi = 0; bi < g.nb0; ++bi) {
    const int* rc = &g.b0[12 * bi];
    const int bs = rc[0];
    double Lm[3][3] = {{0}};
    for (int j = 0; j < bs; ++j) {
      double d = pv(rc[4 + j * (j + 1) / 2 + j]);
      for (int k = 0; k < j; ++k) d -= Lm[j][k] * Lm[j][k];
      if (!(d > 0)) throw std::runtime_error("numprog: level-0 breakdown");
      Lm[j][j] = std::sqrt(d);
      for (int i = j + 1; i < bs; ++i) {
        double s = pv(rc[4 + i * (i + 1) / 2 + j]);
        for (int k = 0; k < j; ++k) s -= Lm[i][k] * Lm[j][k];
        Lm[i][j] = s / Lm[j][j];
      }
    }
    for (int r = 0, slot = 0; r < g.bs0; ++r)
      for (int c = 0; c <= r; ++c, ++slot) {
        double v = r < bs ? Lm[r][c] : 0.0;
        if (r == c) v = r < bs ? 1.0 / v : 0.0;
        C[g.blk0_vofs + (int64_t)slot * g.nb0 + bi] = v;
      }
    for (int k = rc[10]; k < rc[11]; ++k) {
      const int* nr = &g.nbr[7 * k];
      double y[3] = {0, 0, 0}, z[3] = {0, 0, 0};
      for (int j = 0; j < bs; ++j) {
        double s = pv(nr[1 + j]);
        for (int kk = 0; kk < j; ++kk) s -= Lm[j][kk] * y[kk];
        y[j] = s / Lm[j][j];
      }
      for (int j = 0; j < 3; ++j) M[3 * k + j] = y[j];
      for (int j = bs - 1; j >= 0; --j) {
        double s = y[j];
        for (int kk = j + 1; kk < bs; ++kk) s -= Lm[kk][j] * z[kk];
        z[j] = s / Lm[j][j];
        C[nr[4 + j]] = z[j];
      }
    }
  }
  for (size_t i = 0; i < g.w0.size() / 2; ++i) C[g.w0[2 * i]] = pv(g.w0[2 * i + 1]);
  const bool icc = g.final_kind == FINAL_ICC;
  const int nG = g.nG;
  std::vector<double> S(icc ? (g.icc_rowptr.empty() ? 0 : g.icc_rowptr.back()) : (size_t)nG * nG, 0.0);
  for (size_t q = 0; q < g.st_idx.size(); ++q) {
    double v = pv(g.st_csr[q]);
    for (int k = g.st_ptr[q]; k < g.st_ptr[q + 1]; ++k) {
      const double* a = &M[3 * g.st_src[2 * k]];
      const double* c = &M[3 * g.st_src[2 * k + 1]];
      v -= a[0] * c[0] + a[1] * c[1] + a[2] * c[2];
    }
    S[g.st_idx[q]] = v;
  }
  if (!icc) {
    for (int j = 0; j < nG; ++j) {   // dense Cholesky, lower, row-major
      double d = S[(size_t)j * nG + j];
      for (int k = 0; k < j; ++k) d -= S[(size_t)j * nG + k] * S[(size_t)j * nG + k];
      if (!(d > 0)) throw std::runtime_error("numprog: interface breakdown");
      d = std::sqrt(d);
      S[(size_t)j * nG + j] = d;
      for (int i = j + 1; i < nG; ++i) {
        double s = S[(size_t)i * nG + j];
        for (int k = 0; k < j; ++k) s -= S[(size_t)i * nG + k] * S[(size_t)j * nG + k];
        S[(size_t)i * nG + j] = s / d;
      }
    }
    for (size_t i = 0; i < g.rec.size() / 4; ++i) {
      const int* r = &g.rec[4 * i];
      const double lab = S[(size_t)r[2] * nG + r[3]], lbb = S[(size_t)r[3] * nG + r[3]];
      C[r[0]] = r[1] == 0 ? 1.0 / lbb : (r[1] == 1 ? lab * lbb : lab / lbb);
    }
    const int m = g.m, g0 = nG - m;
    if (m > 0) {
      std::vector<double> Y((size_t)m * m, 0.0), Fi((size_t)m * m, 0.0);
      auto L = [&](int i, int j) { return S[(size_t)(g0 + i) * nG + g0 + j]; };
      for (int c = 0; c < m; ++c)
        for (int i = c; i < m; ++i) {
          double s = (i == c) ? 1.0 : 0.0;
          for (int k = c; k < i; ++k) s -= L(i, k) * Y[(size_t)k * m + c];
          Y[(size_t)i * m + c] = s / L(i, i);
        }
      for (int i = 0; i < m; ++i)
        for (int j = 0; j <= i; ++j) {
          double s = 0.0;
          for (int k = i; k < m; ++k) s += Y[(size_t)k * m + i] * Y[(size_t)k * m + j];
          Fi[(size_t)i * m + j] = Fi[(size_t)j * m + i] = s;
        }
      const int T = (m + 31) / 32;
      for (int I = 0; I < T; ++I)
        for (int J = 0; J <= I; ++J)
          for (int r = 0; r < 32; ++r)
            for (int c = 0; c < 32; ++c) {
              const int i = 32 * I + r, j = 32 * J + c;
              C[g.vofs_final + (int64_t)(I * (I + 1) / 2 + J) * 1024 + r * 32 + ((c + r) & 31)] =
                  (i < m && j < m) ? Fi[(size_t)i * m + j] : 0.0;
            }
    }
  } else {
    const int nnz = (int)S.size();
    for (size_t lv = 0; lv + 1 < g.icc_lptr.size(); ++lv)
      for (int q = g.icc_lptr[lv]; q < g.icc_lptr[lv + 1]; ++q) {
        const int ra = g.icc_lrows[q], a0 = g.icc_rowptr[ra], a1 = g.icc_rowptr[ra + 1];
        for (int t = a0; t < a1; ++t) {
          const int b = g.icc_col[t];
          double s = S[t];
          int ia = a0, ib = g.icc_rowptr[b];
          const int eb = g.icc_rowptr[b + 1] - 1;
          while (ia < t && ib < eb) {
            const int ca = g.icc_col[ia], cb = g.icc_col[ib];
            if (ca == cb) { s -= S[ia] * S[ib]; ++ia; ++ib; }
            else if (ca < cb) ++ia; else ++ib;
          }
          if (b == ra) {
            if (!(s > 0)) throw std::runtime_error("numprog: icc breakdown");
            S[t] = std::sqrt(s);
          } else {
            S[t] = s / S[g.icc_rowptr[b + 1] - 1];
          }
        }
      }
    double* o = C.data() + g.vofs_final;
    for (int ra = 0; ra < g.m; ++ra)
      for (int t = g.icc_rowptr[ra]; t < g.icc_rowptr[ra + 1]; ++t) o[t] = (t == g.icc_rowptr[ra + 1] - 1) ? 1.0 / S[t] : S[t];
    for (int t = 0; t < nnz; ++t) o[nnz + t] = o[g.icct_src[t]];
  }
  for (int64_t k = 0; k < g.nvals; ++k) {
    const int c = g.smap[k];
    out[k] = c >= 0 ? C[c] : (c == -1 ? 0.0 : 0.5 * C[-2 - c]);
  }
}

int emu_numeric_program_check(int k, int p, int nx, int ny, int nz, unsigned gamma, const double* alpha, long long na,
                              const double* beta, long long nb, const double* coords, int dim, int fact, double* rel,
                              char* err, int errlen) {
  try {
    std::vector<double> h[3];
    const int n[3] = {nx, ny, nz};
    for (int d = 0; d < 3; ++d) h[d].assign(n[d], 1.0 / n[d]);
    SetupInput in{};
    in.k = k; in.p = p; in.n[0] = nx; in.n[1] = ny; in.n[2] = nz; in.gamma_d = gamma;
    in.coords = coords; in.alpha = alpha; in.beta = beta; in.n_alpha = na; in.n_beta = nb;
    in.dim = dim; in.factorization = fact; in.cartesian = (coords == nullptr);
    in.hx = h[0].data(); in.hy = h[1].data(); in.hz = h[2].data();
    auto Fh = build_patch_family(in);
    in.defer_numeric = true;
    auto Fd = build_patch_family(in);
    if (Fd->foff.size() != (size_t)Fh->nfactors) throw std::runtime_error("block count differs");
    const int ne = (int)Fd->cell_rows.size();
    std::vector<double> cent;
    if (!Fd->cartesian) {   // per-cell entries through the AuxTables split (what the device computes)
      const AuxTables& T = aux_tables(p);
      const int64_t ncell = (int64_t)nx * ny * nz;
      cent.resize((size_t)ncell * ne);
      std::vector<double> dg(T.ndiag);
      for (int64_t K = 0; K < ncell; ++K) {
        const int cx = (int)(K % nx), cy = (int)((K / nx) % ny), cz = (int)(K / ((int64_t)nx * ny));
        double Xc[8][3];
        for (int v = 0; v < 8; ++v)
          for (int i = 0; i < 3; ++i)
            Xc[v][i] = coords[(((int64_t)(cz + (v >> 2)) * (ny + 1) + (cy + ((v >> 1) & 1))) * (nx + 1) + (cx + (v & 1))) * 3 + i];
        aux_cell_diagonals(T, Xc, Fd->cell_alpha[K], Fd->cell_beta[K], dg.data());
        aux_entries_from_diagonals(T, dg.data(), &cent[(size_t)K * ne]);
      }
    }
    std::vector<NumProg> progs(Fd->classes.size());
    std::vector<char> built(Fd->classes.size(), 0);
    double md = 0.0, mv = 0.0;
    for (size_t f = 0; f < Fd->foff.size(); ++f) {
      const int c = Fd->fclass[f];
      if (!built[c]) { build_numeric_program(Fd->classes[c], Fd->cell_rows, Fd->cell_cols, progs[c]); built[c] = 1; }
      const NumProg& g = progs[c];
      std::vector<double> out(g.nvals);
      numprog_eval(g, *Fd, (int)f, cent, ne, out.data());
      const double* ref = Fh->values.data() + Fd->foff[f];
      for (int64_t q = 0; q < g.nvals; ++q) {
        md = std::max(md, std::fabs(out[q] - ref[q]));
        mv = std::max(mv, std::fabs(ref[q]));
      }
    }
    *rel = mv > 0 ? md / mv : md;
    return 0;
  } catch (const std::exception& e) {
    snprintf(err, errlen, "%s", e.what());
    *rel = -1;
    return 1;
  }
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
