#include "patches.hpp"
#include "exp_env.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <tuple>
#include <unordered_map>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace rm {

namespace {

struct DirSpec { int kind; int v; };   // kind 0 = node (vertex-type direction), 1 = cell
struct Entity { DirSpec s[3]; };

// per-direction window of a family (oracle reading G5 is the same rule)
void window(const DirSpec& s, int fam, int p, int ncell, int& lo, int& hi) {
  if (fam == FAM_P) {
    if (s.kind == 0) { lo = s.v * p - (p - 1); hi = s.v * p + (p - 1); }
    else { lo = s.v * p + 1; hi = s.v * p + p - 1; }
    lo = std::max(lo, 0); hi = std::min(hi, ncell * p);
  } else {
    if (s.kind == 0) { lo = s.v * p - p; hi = s.v * p + p - 1; }
    else { lo = s.v * p; hi = s.v * p + p - 1; }
    lo = std::max(lo, 0); hi = std::min(hi, ncell * p - 1);
  }
}

std::vector<Entity> entities(const Space& sp, int dim, bool interior_only) {
  std::vector<Entity> out;
  auto push = [&](Entity e) {
    if (interior_only)
      for (int d = 0; d < 3; ++d)
        if (e.s[d].kind == 0 && (e.s[d].v == 0 || e.s[d].v == sp.n[d])) return;
    out.push_back(e);
  };
  if (dim == 0) {
    for (int z = 0; z <= sp.n[2]; ++z)
      for (int y = 0; y <= sp.n[1]; ++y)
        for (int x = 0; x <= sp.n[0]; ++x) push(Entity{{{0, x}, {0, y}, {0, z}}});
  } else if (dim == 1 || dim == 2) {
    for (int e = 0; e < 3; ++e) {
      int lim[3];
      for (int d = 0; d < 3; ++d) {
        bool cellkind = (dim == 1) ? (d == e) : (d != e);
        lim[d] = cellkind ? sp.n[d] : sp.n[d] + 1;
      }
      for (int z = 0; z < lim[2]; ++z)
        for (int y = 0; y < lim[1]; ++y)
          for (int x = 0; x < lim[0]; ++x) {
            int idx[3] = {x, y, z};
            Entity en;
            for (int d = 0; d < 3; ++d) {
              bool cellkind = (dim == 1) ? (d == e) : (d != e);
              en.s[d] = {cellkind ? 1 : 0, idx[d]};
            }
            push(en);
          }
    }
  } else {
    throw std::runtime_error("entities: dim");
  }
  return out;
}

typedef std::array<int, 9> ClassKey;   // per direction: kind, low clip, high clip
ClassKey class_key(const Space& sp, const Entity& e) {
  ClassKey k;
  for (int d = 0; d < 3; ++d) {
    k[3 * d] = e.s[d].kind;
    k[3 * d + 1] = (e.s[d].kind == 0 && e.s[d].v == 0);
    k[3 * d + 2] = (e.s[d].kind == 0 && e.s[d].v == sp.n[d]);
  }
  return k;
}

int color_of(const Entity& e, int dim) {
  if (dim == 0) return (e.s[0].v & 1) | ((e.s[1].v & 1) << 1) | ((e.s[2].v & 1) << 2);
  int dir = 0;
  for (int d = 0; d < 3; ++d)
    if ((dim == 1 && e.s[d].kind == 1) || (dim == 2 && e.s[d].kind == 0)) dir = d;
  int bits = 0, nb = 0;
  for (int d = 0; d < 3; ++d)
    if (e.s[d].kind == 0) bits |= (e.s[d].v & 1) << (nb++);
  return dir * (1 << nb) + bits;
}

int64_t anchor_coord(const DirSpec& s, int p) { return (int64_t)s.v * p; }

struct NatDof { int comp, ix, iy, iz, group; int64_t g; };

// small dense SPD inverse (n <= 3) via Gauss-Jordan on the SPD block
bool small_inverse(int n, const double* a, double* inv) {
  double m[3][6];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 2 * n; ++j) m[i][j] = (j < n) ? a[i * n + j] : (j - n == i ? 1.0 : 0.0);
  for (int c = 0; c < n; ++c) {
    if (!(m[c][c] > 0)) return false;
    double piv = m[c][c];
    for (int j = 0; j < 2 * n; ++j) m[c][j] /= piv;
    for (int r = 0; r < n; ++r)
      if (r != c) {
        double f = m[r][c];
        for (int j = 0; j < 2 * n; ++j) m[r][j] -= f * m[c][j];
      }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) inv[i * n + j] = m[i][j + n];
  return true;
}

void build_sliced(Sliced& s, int r0, const std::vector<std::vector<int>>& rowcols) {
  s.r0 = r0; s.nrows = (int)rowcols.size();
  s.rowcols = rowcols;
  int nsl = (s.nrows + 31) / 32;
  s.slice_w.assign(nsl, 0); s.slice_off.assign(nsl, 0);
  int64_t off = 0;
  for (int sl = 0; sl < nsl; ++sl) {
    int w = 0;
    for (int l = 0; l < 32; ++l) {
      int r = sl * 32 + l;
      if (r < s.nrows) w = std::max(w, (int)rowcols[r].size());
    }
    s.slice_w[sl] = w; s.slice_off[sl] = (int)off;
    off += (int64_t)w * 32;
  }
  s.nelem = off;
  s.cols.assign(off, 0);
  for (int sl = 0; sl < nsl; ++sl)
    for (int l = 0; l < 32; ++l) {
      int r = sl * 32 + l;
      if (r >= s.nrows) continue;
      for (size_t kk = 0; kk < rowcols[r].size(); ++kk) s.cols[s.slice_off[sl] + kk * 32 + l] = (uint16_t)rowcols[r][kk];
    }
}

void build_blocks(Blocks& B, const std::vector<std::vector<int>>& blocks) {
  B.nblk = (int)blocks.size();
  B.bs = 1;
  for (auto& b : blocks) B.bs = std::max(B.bs, (int)b.size());
  B.mem.assign((size_t)B.bs * B.nblk, 0xFFFF);
  for (int i = 0; i < B.nblk; ++i)
    for (size_t j = 0; j < blocks[i].size(); ++j) B.mem[j * B.nblk + i] = (uint16_t)blocks[i][j];
}

// ---------------------------------------------------------------- stream layout (patches.hpp)
void add_piece(ClassProgram& C, int64_t& s, Piece p) {
  if (p.nd <= 0 && p.kind != PK_FINAL && p.kind != PK_ZERO) return;
  p.nd = (p.nd + 1) & ~1;
  // lane-interleaved ICC pieces are padded to 32 x (longest row): up to 4 x kPieceMax (the
  // header fields are 16-bit; units and rings are sized from the actual units)
  if (p.nd > ((p.kind == PK_ICCF || p.kind == PK_ICCB) ? 4 * kPieceMax : kPieceMax))
    throw std::runtime_error("stream piece larger than kPieceMax");
  p.sofs = (int)s;
  s += p.nd;
  C.pieces.push_back(p);
}

void sliced_pieces(ClassProgram& C, int64_t& s, int kind, int lev, const Sliced& S) {
  const int ns = (int)S.slice_w.size();
  int sl = 0;
  while (sl < ns) {
    const int sz = 32 * S.slice_w[sl];
    if (sz > kPieceMax) {   // one wide slice: split its columns
      const int per = kPieceMax / 32;
      for (int k0 = 0; k0 < S.slice_w[sl]; k0 += per) {
        const int nk = std::min(per, S.slice_w[sl] - k0);
        add_piece(C, s, Piece{kind, lev, sl, sl + 1, S.slice_off[sl] + 32 * k0, 0, 32 * nk, (int)S.vofs + S.slice_off[sl] + 32 * k0});
      }
      ++sl;
      continue;
    }
    const int a0 = sl;
    int tot = 0;
    while (sl < ns && tot + 32 * S.slice_w[sl] <= kPieceMax) tot += 32 * S.slice_w[sl++];
    add_piece(C, s, Piece{kind, lev, a0, sl, S.slice_off[a0], 0, tot, (int)S.vofs + S.slice_off[a0]});
  }
}

// class meta stream: one 16-byte-aligned block per piece, header {a0, a1, e0, mbytes | nd << 16};
// every DoF reference is a BOX index (C.bidx): the patch's working vector is its window box
void build_meta(ClassProgram& C) {
  std::vector<uint8_t>& M = C.meta;
  M.clear();
  auto put = [&](const void* p, size_t nb) { const uint8_t* b = (const uint8_t*)p; M.insert(M.end(), b, b + nb); };
  auto put16 = [&](int x) { uint16_t h = (uint16_t)x; if (x < 0 || x > 0xFFFF) throw std::runtime_error("meta u16 overflow"); put(&h, 2); };
  auto align16 = [&]() { while (M.size() & 15) M.push_back(0); };
  const int f0 = C.n - C.m;
  for (size_t i = 0; i < C.pieces.size(); ++i) {
    Piece& p = C.pieces[i];
    if (p.kind == PK_ZERO) p.a1 = (int)C.zlist.size();
    const size_t at = M.size();
    int32_t hdr[4] = {p.a0, p.a1, p.e0, 0};
    put(hdr, 16);
    switch (p.kind) {
      case PK_PIV: {   // uint16 block members [slot][block]
        const Blocks& B = C.lev[p.lev].blk;
        for (int sl = 0; sl < B.bs; ++sl)
          for (int b = p.a0; b < p.a1; ++b) {
            const int mpos = B.mem[(size_t)sl * B.nblk + b];
            put16(mpos == 0xFFFF ? 0xFFFF : C.bidx[mpos]);
          }
        break;
      }
      case PK_W:
      case PK_WT: {   // per slice (start/32 | count << 16); per slice 32 row boxes; column boxes
        const Sliced& S = (p.kind == PK_W) ? C.lev[p.lev].w : C.lev[p.lev].wt;
        for (int sl = p.a0; sl < p.a1; ++sl) {
          const int o = S.slice_off[sl];
          const int k0 = std::max(0, (p.e0 - o) / 32), k1 = std::min(S.slice_w[sl], (p.e0 + p.nd - o) / 32);
          const int start = o + 32 * k0 - p.e0;
          const uint32_t info = (uint32_t)(start / 32) | ((uint32_t)std::max(0, k1 - k0) << 16);
          put(&info, 4);
        }
        for (int sl = p.a0; sl < p.a1; ++sl)
          for (int l = 0; l < 32; ++l) {
            const int row = sl * 32 + l;
            put16(row < S.nrows ? C.bidx[S.r0 + row] : 0);
          }
        for (int e = p.e0; e < p.e0 + p.nd; ++e) put16(C.bidx[S.cols[e]]);
        break;
      }
      case PK_TILE:
        break;
      case PK_FINAL:   // uint16 boxes of the final block's positions
        for (int j = 0; j < C.m; ++j) put16(C.bidx[f0 + j]);
        break;
      case PK_ZERO:    // uint16 boxes that are not DoFs of the patch (zeroed before the reduce-add)
        for (int z : C.zlist) put16(z);
        break;
      case PK_ICCF:
      case PK_ICCB: {  // chunk table {cnt, L, meta offset, value offset} x nchunks, then per chunk
                       // 32 uint16 row boxes and the interleaved column boxes (pads: box 0)
        const bool f = p.kind == PK_ICCF;
        const std::vector<int>& row = f ? C.iccf_row : C.iccb_row;
        const std::vector<int>& col = f ? C.iccf_col : C.iccb_col;
        const std::vector<IccChunk>& ch = f ? C.iccf_chunk : C.iccb_chunk;
        const size_t tab = M.size();
        M.resize(M.size() + 16 * (p.a1 - p.a0), 0);
        for (int c = p.a0; c < p.a1; ++c) {
          const IccChunk& k = ch[c];
          const int32_t ent[4] = {k.cnt, k.L, (int)(M.size() - at), k.sofs - ch[p.a0].sofs};
          std::memcpy(&M[tab + 16 * (c - p.a0)], ent, 16);
          for (int q = 0; q < 32; ++q) put16(q < k.cnt ? C.bidx[f0 + row[k.r0 + q]] : 0);
          for (int q = 32; q < 32 + 32 * k.L; ++q) put16(col[k.sofs + q] < 0 ? 0 : C.bidx[f0 + col[k.sofs + q]]);
        }
        break;
      }
      default:
        throw std::runtime_error("build_meta: piece kind");
    }
    align16();
    p.mofs = (int)at;
    p.mbytes = (int)(M.size() - at);
    if (p.mbytes > 0xFFFF || p.nd > 0xFFFF) throw std::runtime_error("piece too large for its header");
    const uint32_t w3 = (uint32_t)p.mbytes | ((uint32_t)p.nd << 16);
    std::memcpy(&M[at + 12], &w3, 4);
  }
  // transfer units: consecutive pieces (metas and values both contiguous), split at the
  // dense-tile section (its own channel)
  static const int unit_vals = exp_env("RM_UNIT_VALS") ? atoi(exp_env("RM_UNIT_VALS")) : kUnitVals;
  static const int unit_vals_tile = exp_env("RM_UNIT_VALS_TILE") ? atoi(exp_env("RM_UNIT_VALS_TILE")) : kUnitValsTile;
  C.units.clear();
  for (int i = 0; i < (int)C.pieces.size();) {
    Unit u{i, 0, C.pieces[i].mofs, 0, C.pieces[i].sofs, 0};
    const bool tile_sec = C.final_kind == FINAL_DENSE_INV && i >= C.tile_p0 && i < C.tile_p1;
    const int cap_vals = tile_sec ? unit_vals_tile : unit_vals;
    while (i < (int)C.pieces.size()) {
      const Piece& p = C.pieces[i];
      const bool boundary = u.np > 0 && (i == C.tile_p0 || i == C.tile_p1);
      if (u.np > 0 && (boundary || u.nd + p.nd > cap_vals || u.mbytes + p.mbytes > kUnitMeta)) break;
      u.np++; u.mbytes += p.mbytes; u.nd += p.nd;
      ++i;
    }
    C.units.push_back(u);
  }
  // unit ranges of the three segments: forward [0, uf0), final [uf0, uf1), backward [uf1, end)
  C.uf0 = C.uf1 = (int)C.units.size();
  for (int k = (int)C.units.size() - 1; k >= 0; --k) {
    if (C.units[k].p0 >= C.tile_p0) C.uf0 = k;
    if (C.units[k].p0 >= C.tile_p1) C.uf1 = k;
  }
  C.tu0 = C.tu1 = 0;
  if (C.final_kind == FINAL_DENSE_INV && C.m > 0) { C.tu0 = C.uf0; C.tu1 = C.uf1; }
}

void build_stream(ClassProgram& C) {
  C.pieces.clear();
  const int L = (int)C.lev.size();
  C.ngs = 0;
  C.piv_b.assign(L, 0); C.w_b.assign(L, 0); C.w_e.assign(L, 0); C.wt_b.assign(L, 0); C.wt_e.assign(L, 0);
  C.piv_per.assign(L, 1); C.piv_ofs.assign(L, 0); C.mem_ofs.assign(L, 0);
  int64_t s = 0;
  int pivofs = 0, memofs = 0;
  for (int l = 0; l < L; ++l) {
    const Blocks& B = C.lev[l].blk;
    const int ns = B.bs * (B.bs + 1) / 2;
    const int per = std::max(1, (kPieceMax / ns) & ~1);
    if (C.sc) {   // cell interiors are condensed per cell, outside the patch kernel
      C.piv_per[l] = per; C.piv_b[l] = C.w_b[l] = C.w_e[l] = (int)C.pieces.size();
      continue;
    }
    C.piv_per[l] = per;
    C.piv_ofs[l] = pivofs;
    C.mem_ofs[l] = memofs;
    pivofs += ns * B.nblk;
    memofs += B.bs * B.nblk;
    C.piv_b[l] = (int)C.pieces.size();
    for (int a0 = 0; a0 < B.nblk; a0 += per) {
      const int a1 = std::min(B.nblk, a0 + per);
      add_piece(C, s, Piece{PK_PIV, l, a0, a1, 0, 0, ns * (a1 - a0), (int)B.vofs});
    }
    C.w_b[l] = (int)C.pieces.size();
    sliced_pieces(C, s, PK_W, l, C.lev[l].w);
    C.w_e[l] = (int)C.pieces.size();
  }
  C.piv_total = (pivofs + 1) & ~1;
  C.mem_total = (memofs + 7) & ~7;
  C.tile_p0 = (int)C.pieces.size();
  const int m = C.m;
  if (C.final_kind == FINAL_DENSE_INV) {
    const int T = (m + 31) / 32;
    if (m > 0) add_piece(C, s, Piece{PK_FINAL, 0, 0, m, 0, 0, 0, -1});
    for (int I = 0; I < T; ++I)
      for (int J = 0; J <= I; ++J)
        add_piece(C, s, Piece{PK_TILE, 0, I, J, 0, 0, I == J ? kTileDiag : 1024,
                              (int)C.vofs_final + (I * (I + 1) / 2 + J) * 1024});
  } else {
    // ICC pieces, LANE-INTERLEAVED: the rows of a level, sorted by length (longest first), in
    // chunks of <= 32 (one row per lane of the warp that takes the piece); values = the 32
    // inverted diagonals, then step j of every row at [32 + 32 j + lane] (zero padded to the
    // chunk's longest row); meta = 32 row boxes, then the column boxes in the same interleaved
    // order.  Forward: rows of L (diagonal last in the CSR); backward: rows of L^T (first).
    const int nnz = C.icc_rowptr.empty() ? 0 : C.icc_rowptr[m];
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<int>& rowv = pass == 0 ? C.iccf_row : C.iccb_row;
      std::vector<int>& slot = pass == 0 ? C.iccf_src : C.iccb_src;   // per piece value slot -> canonical (-1: 0)
      std::vector<int>& colv = pass == 0 ? C.iccf_col : C.iccb_col;   // per piece value slot -> column (-1: pad)
      std::vector<int>& lpiece = pass == 0 ? C.iccf_lpiece : C.iccb_lpiece;
      std::vector<IccChunk>& chunks = pass == 0 ? C.iccf_chunk : C.iccb_chunk;
      const std::vector<int>& lptr = pass == 0 ? C.icc_level_ptr : C.icct_level_ptr;
      const std::vector<int>& lrows = pass == 0 ? C.icc_level_rows : C.icct_level_rows;
      const std::vector<int>& rp = pass == 0 ? C.icc_rowptr : C.icct_rowptr;
      const std::vector<int>& cl = pass == 0 ? C.icc_col : C.icct_col;
      rowv.clear(); slot.clear(); colv.clear(); lpiece.clear(); chunks.clear();
      C.iccf_rp.clear(); C.iccb_rp.clear();
      const int nl = (int)lptr.size() - 1;
      for (int l = 0; l < nl; ++l) {
        lpiece.push_back((int)C.pieces.size());
        std::vector<int> lr(lrows.begin() + lptr[l], lrows.begin() + lptr[l + 1]);
        std::stable_sort(lr.begin(), lr.end(), [&](int x, int y) { return rp[x + 1] - rp[x] > rp[y + 1] - rp[y]; });
        const int ch0 = (int)chunks.size();
        for (size_t c0 = 0; c0 < lr.size(); c0 += kIccRows) {   // chunks of <= 32 rows
          const int cnt = (int)std::min<size_t>(kIccRows, lr.size() - c0);
          int Lmax = 0;
          for (int k = 0; k < cnt; ++k) Lmax = std::max(Lmax, rp[lr[c0 + k] + 1] - rp[lr[c0 + k]] - 1);
          const int nd = 32 + 32 * Lmax;
          if (nd > 4 * kPieceMax) throw std::runtime_error("ICC row too long for a piece");
          const int sofs = (int)slot.size();
          chunks.push_back(IccChunk{(int)rowv.size(), cnt, Lmax, sofs});
          slot.resize(sofs + nd, -1);
          colv.resize(sofs + nd, -1);
          for (int k = 0; k < cnt; ++k) {
            const int a = lr[c0 + k];
            rowv.push_back(a);
            const int d = pass == 0 ? rp[a + 1] - 1 : rp[a];         // diagonal entry (stored inverted)
            const int o0 = pass == 0 ? rp[a] : rp[a] + 1;            // off-diagonal entries, CSR order
            slot[sofs + k] = (pass == 0 ? 0 : nnz) + d;   // canonical: L values, then L^T values (CSR of L^T)
            for (int j = 0; o0 + j < (pass == 0 ? rp[a + 1] - 1 : rp[a + 1]); ++j) {
              const int t = o0 + j;
              slot[sofs + 32 + 32 * j + k] = (pass == 0 ? 0 : nnz) + t;
              colv[sofs + 32 + 32 * j + k] = cl[t];
            }
          }
        }
        // pieces of <= kIccChunks consecutive chunks and <= kIccPieceVals values (one chunk may exceed it)
        for (int c = ch0; c < (int)chunks.size();) {
          const int c0 = c;
          int nd = 0;
          while (c < (int)chunks.size() && c - c0 < kIccChunks) {
            const int cd = 32 + 32 * chunks[c].L;
            if (c > c0 && nd + cd > kIccPieceVals) break;
            nd += cd;
            ++c;
          }
          add_piece(C, s, Piece{pass == 0 ? PK_ICCF : PK_ICCB, l, c0, c, c - c0, 0, nd, chunks[c0].sofs});
        }
      }
      lpiece.push_back((int)C.pieces.size());
    }
  }
  C.tile_p1 = (int)C.pieces.size();
  for (int l = L - 1; l >= 0; --l) {
    C.wt_b[l] = (int)C.pieces.size();
    if (!C.sc) sliced_pieces(C, s, PK_WT, l, C.lev[l].wt);
    C.wt_e[l] = (int)C.pieces.size();
  }
  add_piece(C, s, Piece{PK_ZERO, 0, 0, 0, 0, 0, 0, -1});   // a1 = zero-list length, set by build_meta
  C.nvals = s;
}

// canonical (factorization-order) block -> stream block
void pack_stream(const ClassProgram& C, const double* canon, double* out) {
  for (const Piece& p : C.pieces) {
    double* o = out + p.sofs;
    std::fill(o, o + p.nd, 0.0);
    switch (p.kind) {
      case PK_PIV: {
        const Blocks& B = C.lev[p.lev].blk;
        const int ns = B.bs * (B.bs + 1) / 2, cnt = p.a1 - p.a0;
        for (int slot = 0; slot < ns; ++slot)
          for (int i = p.a0; i < p.a1; ++i) o[slot * cnt + (i - p.a0)] = canon[p.cofs + (size_t)slot * B.nblk + i];
        break;
      }
      case PK_W:
      case PK_WT:
        std::copy(canon + p.cofs, canon + p.cofs + p.nd, o);
        break;
      case PK_TILE:   // canonical tiles hold element (r, c) at r*32 + ((c + r) & 31)
        for (int r = 0; r < 32; ++r)
          for (int c = 0; c < 32; ++c) {
            const double x = canon[p.cofs + r * 32 + ((c + r) & 31)];
            if (p.a0 != p.a1) o[tile_pos_full(r, c)] = x;
            else if (c < r) o[tile_pos_diag(r, c)] = x;
            else if (c == r) o[tile_pos_diag(r, c)] = 0.5 * x;
          }
        break;
      case PK_ICCF:
      case PK_ICCB: {   // lane-interleaved slots (p.cofs = first slot of the piece)
        const std::vector<int>& slot = p.kind == PK_ICCF ? C.iccf_src : C.iccb_src;
        for (int k = 0; k < p.nd; ++k) {
          const int src = slot[p.cofs + k];
          o[k] = src < 0 ? 0.0 : canon[C.vofs_final + src];
        }
        break;
      }
      default:   // metadata-only pieces (FINAL, ZERO)
        break;
    }
  }
}

}  // namespace

// ===================================================================================== builder
struct Builder {
  const SetupInput& in;
  Space sp;
  PatchFamily* fam;
  CellOperator op;
  std::vector<int> cell_rows, cell_cols;   // structural pattern of the cell matrix
  int nloc = 0;
  std::vector<int> loc_comp, loc_a[3];     // local dof -> comp, local index per direction

  explicit Builder(const SetupInput& in_, PatchFamily* f) : in(in_), fam(f) {
    sp.init(in.k, in.p, in.n[0], in.n[1], in.n[2]);
    nloc = sp.nloc();
    for (int m = 0; m < sp.ncomp; ++m)
      for (int c = 0; c < sp.lsize(m, 2); ++c)
        for (int b = 0; b < sp.lsize(m, 1); ++b)
          for (int a = 0; a < sp.lsize(m, 0); ++a) {
            loc_comp.push_back(m); loc_a[0].push_back(a); loc_a[1].push_back(b); loc_a[2].push_back(c);
          }
    if (in.cartesian) {
      op = build_cell_operator(in.k, in.p);
      CellEntries e = cartesian_cell_entries(op, sp, 1.0, 1.0, 1.0);
      cell_rows = e.row; cell_cols = e.col;
    } else {
      if (in.k != 0) throw std::runtime_error("trilinear cells are supported for H(grad) only");
      double Xc[8][3];
      for (int a = 0; a < 8; ++a) { Xc[a][0] = a & 1; Xc[a][1] = (a >> 1) & 1; Xc[a][2] = (a >> 2) & 1; }
      CellEntries e;
      aux_cell_entries(in.p, Xc, 1.0, 1.0, e);
      cell_rows = e.row; cell_cols = e.col;
    }
  }

  double coef(const double* arr, int64_t n_arr, int cx, int cy, int cz) const {
    if (n_arr == 1) return arr[0];
    return arr[((int64_t)cz * sp.n[1] + cy) * sp.n[0] + cx];
  }

  // ---------------------------------------------------------------- class program (symbolic)
  void build_class(const Entity& e, ClassProgram& C) {
    const int p = sp.p;
    static const bool sc_off = exp_env("RM_NO_SC") != nullptr;   // experiments: ICC-SC inside the patch kernel
    const bool sc = in.factorization == 1 && in.k == 0 && !sc_off;   // ICC-SC: condense cell interiors per cell
    std::vector<NatDof> dofs;
    int wlo_abs[3][3] = {{0}};
    for (int m = 0; m < sp.ncomp; ++m) {
      int lo[3], hi[3];
      for (int d = 0; d < 3; ++d) {
        window(e.s[d], sp.fam[m][d], p, sp.n[d], lo[d], hi[d]);
        wlo_abs[m][d] = lo[d];
        C.wlo[m][d] = lo[d] - (int)anchor_coord(e.s[d], p);   // window origin relative to the anchor
        C.wext[m][d] = hi[d] - lo[d] + 1;
      }
      for (int iz = lo[2]; iz <= hi[2]; ++iz)
        for (int iy = lo[1]; iy <= hi[1]; ++iy)
          for (int ix = lo[0]; ix <= hi[0]; ++ix) {
            if (sp.constrained(m, ix, iy, iz, in.gamma_d)) continue;
            int grp = 0;
            const int idx[3] = {ix, iy, iz};
            for (int d = 0; d < 3; ++d) if (sp.fam[m][d] == FAM_P && idx[d] % p == 0) ++grp;
            dofs.push_back({m, ix, iy, iz, grp, sp.gidx(m, iz, iy, ix)});
          }
    }
    // natural (pinned) order: group, comp, z, y, x (reading G6)
    std::sort(dofs.begin(), dofs.end(), [](const NatDof& a, const NatDof& b) {
      return std::tie(a.group, a.comp, a.iz, a.iy, a.ix) < std::tie(b.group, b.comp, b.iz, b.iy, b.ix);
    });
    const int n = (int)dofs.size();
    std::unordered_map<int64_t, int> nat_of;
    for (int i = 0; i < n; ++i) nat_of[dofs[i].g] = i;
    // star cells
    std::vector<int> cr[3];
    for (int d = 0; d < 3; ++d) {
      const DirSpec& s = e.s[d];
      if (s.kind == 1) cr[d] = {s.v};
      else { if (s.v - 1 >= 0) cr[d].push_back(s.v - 1); if (s.v < sp.n[d]) cr[d].push_back(s.v); }
    }
    std::vector<std::vector<int>> slot_nat;
    for (int cz : cr[2]) for (int cy : cr[1]) for (int cx : cr[0]) {
      std::vector<int> mp(nloc, -1);
      for (int l = 0; l < nloc; ++l) {
        int m = loc_comp[l];
        int64_t g = sp.gidx(m, (int64_t)cz * p + loc_a[2][l], (int64_t)cy * p + loc_a[1][l], (int64_t)cx * p + loc_a[0][l]);
        auto it = nat_of.find(g);
        if (it != nat_of.end()) mp[l] = it->second;
      }
      slot_nat.push_back(mp);
      C.slot_dc[0].push_back(cx - (int)(anchor_coord(e.s[0], 1)));
      C.slot_dc[1].push_back(cy - (int)(anchor_coord(e.s[1], 1)));
      C.slot_dc[2].push_back(cz - (int)(anchor_coord(e.s[2], 1)));
    }
    // structural pattern (natural indices)
    std::vector<std::vector<int>> adj(n);
    for (auto& mp : slot_nat)
      for (size_t t = 0; t < cell_rows.size(); ++t) {
        int i = mp[cell_rows[t]], j = mp[cell_cols[t]];
        if (i >= 0 && j >= 0) adj[i].push_back(j);
      }
    for (auto& a : adj) { std::sort(a.begin(), a.end()); a.erase(std::unique(a.begin(), a.end()), a.end()); }
    // algorithmic factor size: exact Cholesky -> nnz(L) in the pinned order by the
    // elimination-tree row walk (every row of L = the etree paths from its A-row entries);
    // ICC-SC -> the mask tril(pattern(P_v)) U tril(pattern(P_GI P_IG)) (interiors first)
    {
      int64_t nnz = 0;
      if (in.factorization == 0) {
        std::vector<int> parent(n, -1), flag(n, -1);
        for (int i = 0; i < n; ++i) {
          flag[i] = i;
          ++nnz;
          for (int j : adj[i]) {
            if (j >= i) break;
            for (int k = j; flag[k] != i; k = parent[k]) {
              if (parent[k] == -1) parent[k] = i;
              ++nnz;
              flag[k] = i;
            }
          }
        }
      } else {
        std::vector<char> interior(n, 0);
        for (int i = 0; i < n; ++i) interior[i] = dofs[i].group == 0;
        std::vector<int> mark(n, -1);
        for (int i = 0; i < n; ++i) {
          std::vector<int> row;
          for (int j : adj[i]) if (j <= i) row.push_back(j);
          if (!interior[i])
            for (int k : adj[i])
              if (interior[k])
                for (int j : adj[k]) if (!interior[j] && j <= i) row.push_back(j);
          for (int j : row) if (mark[j] != i) { mark[j] = i; ++nnz; }
        }
      }
      C.nnzL = nnz;
    }

    // ---- symbolic elimination
    // face orientation of group-1 DoFs (direction of the P index on a cell boundary), 3 otherwise
    std::vector<int> orient(n, 3);
    for (int i = 0; i < n; ++i) {
      if (dofs[i].group != 1) continue;
      const int idx[3] = {dofs[i].ix, dofs[i].iy, dofs[i].iz};
      for (int d = 0; d < 3; ++d)
        if (sp.fam[dofs[i].comp][d] == FAM_P && idx[d] % p == 0) orient[i] = d;
    }
    std::vector<int> E0;
    for (int i = 0; i < n; ++i) if (dofs[i].group == 0) E0.push_back(i);
    std::vector<char> isE0(n, 0);
    for (int i : E0) isE0[i] = 1;
    // blocks of E0 = connected components inside E0
    std::vector<int> blk(n, -1);
    std::vector<std::vector<int>> blocks0;
    for (int i : E0) {
      if (blk[i] >= 0) continue;
      std::vector<int> st{i}, comp;
      blk[i] = (int)blocks0.size();
      while (!st.empty()) {
        int u = st.back(); st.pop_back(); comp.push_back(u);
        for (int v : adj[u]) if (isE0[v] && blk[v] < 0) { blk[v] = blk[i]; st.push_back(v); }
      }
      if (comp.size() > 3) throw std::runtime_error("interior block larger than 3x3: operator not in FDM-sparse form");
      std::sort(comp.begin(), comp.end());
      blocks0.push_back(comp);
    }
    std::vector<int> G;   // interface natural indices
    for (int i = 0; i < n; ++i) if (!isE0[i]) G.push_back(i);
    const int nG = (int)G.size();
    std::vector<int> gpos(n, -1);
    for (int t = 0; t < nG; ++t) gpos[G[t]] = t;
    std::vector<char> Sb((size_t)nG * nG, 0);   // Schur pattern over interface
    for (int t = 0; t < nG; ++t)
      for (int j : adj[G[t]]) if (gpos[j] >= 0) Sb[(size_t)t * nG + gpos[j]] = 1;
    for (auto& b : blocks0) {
      std::vector<int> nb;
      for (int u : b) for (int v : adj[u]) if (gpos[v] >= 0) nb.push_back(gpos[v]);
      std::sort(nb.begin(), nb.end()); nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
      for (int a : nb) for (int c : nb) Sb[(size_t)a * nG + c] = 1;
    }
    // exact: greedy independent-set levels on the Schur pattern; icc: none
    std::vector<std::vector<int>> Elev;   // interface local indices per level (after level 0)
    std::vector<char> alive(nG, 1);
    int nalive = nG;
    if (in.factorization == 0) {
      while (nalive > 16 && (int)Elev.size() < 5) {   // <= 6 levels incl. level 0 (kernel limit 8)
        std::vector<int> R, deg(nG, 0);
        for (int t = 0; t < nG; ++t) if (alive[t]) R.push_back(t);
        for (int t : R) {
          int d = 0;
          for (int u : R) if (u != t && Sb[(size_t)t * nG + u]) ++d;
          deg[t] = d;
        }
        // candidate independent sets: greedy by degree, and greedy preferring each face
        // orientation first (faces normal to one direction do not couple after the interior
        // elimination on Cartesian stars); keep the cheapest
        std::vector<int> ord;
        std::vector<int> pick;
        int64_t best = -1;
        const int64_t m = (int64_t)R.size();
        for (int pref = -1; pref < 3; ++pref) {
          ord = R;
          std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
            int oa = (pref >= 0 && orient[G[a]] == pref) ? 0 : 1, ob = (pref >= 0 && orient[G[b]] == pref) ? 0 : 1;
            if (oa != ob) return oa < ob;
            return deg[a] < deg[b];
          });
          std::vector<char> blocked(nG, 0);
          std::vector<int> cand;
          for (int t : ord) {
            if (blocked[t]) continue;
            cand.push_back(t); blocked[t] = 1;
            for (int u : R) if (Sb[(size_t)t * nG + u]) blocked[u] = 1;
          }
          int64_t nE = (int64_t)cand.size(), nnzW = 0;
          for (int t : cand) nnzW += deg[t];
          int64_t c = nE + 2 * nnzW + (m - nE) * (m - nE + 1) / 2;
          if (best < 0 || c < best) { best = c; pick = cand; }
        }
        int64_t nE = (int64_t)pick.size(), nnzW = 0;
        for (int t : pick) nnzW += deg[t];
        int64_t oldc = m * (m + 1) / 2;
        int64_t newc = nE + 2 * nnzW + (m - nE) * (m - nE + 1) / 2;
        if (exp_env("RM_DEBUG_LEVELS"))
          fprintf(stderr, "[levels] n=%d nG=%d m=%lld pick=%lld nnzW=%lld mindeg=%d maxdeg=%d old=%lld new=%lld\n", n, nG,
                  (long long)m, (long long)nE, (long long)nnzW, deg[ord.front()], deg[ord.back()], (long long)oldc,
                  (long long)newc);
        if (newc > (oldc * 97) / 100) break;
        std::sort(pick.begin(), pick.end());
        for (int t : pick) { alive[t] = 0; --nalive; }
        for (int t : pick) {
          std::vector<int> nb;
          for (int u : R) if (alive[u] && Sb[(size_t)t * nG + u]) nb.push_back(u);
          for (int a : nb) for (int c : nb) Sb[(size_t)a * nG + c] = 1;
        }
        Elev.push_back(pick);
      }
    }
    // ---- positions: E0 | E1 | ... | final (natural order inside each set)
    std::vector<int> order;
    for (int i : E0) order.push_back(i);
    for (auto& L : Elev) for (int t : L) order.push_back(G[t]);
    std::vector<int> finalset;
    for (int t = 0; t < nG; ++t) if (alive[t]) finalset.push_back(t);
    // exact programs: the final Schur block decouples into independent blocks (edge stars: ~p
    // blocks); order them contiguously (natural order inside each) so that its
    // inverse is block diagonal in position order and every final row records its block's range
    std::vector<int> fcomp_start;   // per final index: first index of its block; block end below
    if (in.factorization == 0 && !finalset.empty()) {
      const int nf = (int)finalset.size();
      std::vector<int> par(nf);
      for (int i = 0; i < nf; ++i) par[i] = i;
      std::function<int(int)> root = [&](int i) { return par[i] == i ? i : par[i] = root(par[i]); };
      for (int i = 0; i < nf; ++i)
        for (int j = 0; j < i; ++j)
          if (Sb[(size_t)finalset[i] * nG + finalset[j]] || Sb[(size_t)finalset[j] * nG + finalset[i]]) par[root(i)] = root(j);
      std::vector<int> first(nf, -1), ord;
      for (int i = 0; i < nf; ++i) if (first[root(i)] < 0) first[root(i)] = i;
      std::vector<std::pair<int, int>> key(nf);
      for (int i = 0; i < nf; ++i) key[i] = {first[root(i)], i};
      std::sort(key.begin(), key.end());
      std::vector<int> fs2(nf);
      fcomp_start.assign(nf, 0);
      for (int i = 0; i < nf; ++i) fs2[i] = finalset[key[i].second];
      for (int i = 0; i < nf; ++i) fcomp_start[i] = (i > 0 && key[i].first == key[i - 1].first) ? fcomp_start[i - 1] : i;
      finalset.swap(fs2);
      C.frange.assign(2 * (size_t)nf, 0);
      for (int i = 0; i < nf; ++i) {
        int e = i;
        while (e < nf && fcomp_start[e] == fcomp_start[i]) ++e;
        C.frange[2 * i] = fcomp_start[i];
        C.frange[2 * i + 1] = e;
      }
    } else {
      C.frange.clear();
    }
    for (int t : finalset) order.push_back(G[t]);
    std::vector<int> pos(n);
    for (int q = 0; q < n; ++q) pos[order[q]] = q;
    C.n = n;
    C.offs.resize(n); C.group.resize(n);
    std::vector<int> comp_of_pos(n);
    for (int q = 0; q < n; ++q) {
      const NatDof& d = dofs[order[q]];
      C.group[q] = d.group;
      comp_of_pos[q] = d.comp;
      int64_t base = sp.gidx(d.comp, anchor_coord(e.s[2], p), anchor_coord(e.s[1], p), anchor_coord(e.s[0], p));
      int64_t rel = d.g - base;
      if (rel > INT32_MAX || rel < INT32_MIN) throw std::runtime_error("patch offset overflow");
      C.offs[q] = (int)rel;
    }
    C.comp = comp_of_pos;
    // window sub-boxes: one per component, or -- static condensation of the cell interiors (sc,
    // ICC-SC families) -- the three anchor planes that carry the patch's interface DoFs
    const int an[3] = {(int)anchor_coord(e.s[0], p), (int)anchor_coord(e.s[1], p), (int)anchor_coord(e.s[2], p)};
    C.sc = sc;
    if (!sc) {
      for (int m = 0; m < sp.ncomp; ++m)
        for (int d = 0; d < 3; ++d) { C.sub_org[m][d] = C.wlo[m][d]; C.sub_ext[m][d] = C.wext[m][d]; }
    } else {
      for (int sb = 0; sb < 3; ++sb)
        for (int d = 0; d < 3; ++d) {
          C.sub_org[sb][d] = (d == sb) ? 0 : C.wlo[0][d];
          C.sub_ext[sb][d] = (d == sb) ? 1 : C.wext[0][d];
        }
    }
    C.psub.assign(n, -1);
    C.pcoord.assign(3 * (size_t)n, 0);
    for (int q = 0; q < n; ++q) {
      const NatDof& d = dofs[order[q]];
      const int rel[3] = {d.ix - an[0], d.iy - an[1], d.iz - an[2]};
      int sb = d.comp;
      if (sc) {
        if (d.group == 0) continue;              // cell interiors: condensed per cell (sc kernels)
        sb = (rel[0] == 0) ? 0 : (rel[1] == 0 ? 1 : 2);
        if (rel[sb] != 0) throw std::runtime_error("static condensation: interface DoF off the anchor planes");
      }
      C.psub[q] = sb;
      for (int k2 = 0; k2 < 3; ++k2) C.pcoord[3 * q + k2] = rel[k2] - C.sub_org[sb][k2];
    }
    C.slot_map.clear();
    for (auto& mp : slot_nat) {
      std::vector<int> m2(nloc, -1);
      for (int l = 0; l < nloc; ++l) if (mp[l] >= 0) m2[l] = pos[mp[l]];
      C.slot_map.push_back(m2);
    }
    // pattern CSR over positions
    C.prow.assign(n + 1, 0); C.pcol.clear();
    {
      std::vector<std::vector<int>> pa(n);
      for (int i = 0; i < n; ++i) for (int j : adj[i]) pa[pos[i]].push_back(pos[j]);
      for (int q = 0; q < n; ++q) {
        std::sort(pa[q].begin(), pa[q].end());
        C.prow[q + 1] = C.prow[q] + (int)pa[q].size();
        C.pcol.insert(C.pcol.end(), pa[q].begin(), pa[q].end());
      }
    }
    // ---- levels
    C.lev.clear();
    int64_t vofs = 0;
    auto place = [&](Sliced& s) { s.vofs = vofs; vofs += s.nelem; };
    auto placeb = [&](Blocks& b) { b.vofs = vofs; vofs += b.nval(); };
    {   // level 0
      Level L;
      L.e0 = 0; L.e1 = (int)E0.size();
      std::vector<std::vector<int>> wrows(n - L.e1), wtrows(L.e1);
      for (auto& b : blocks0) {
        std::vector<int> bp;
        for (int u : b) bp.push_back(pos[u]);
        L.blocks.push_back(bp);
        std::vector<int> nb;
        for (int u : b) for (int v : adj[u]) if (!isE0[v]) nb.push_back(pos[v]);
        std::sort(nb.begin(), nb.end()); nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
        for (int q : bp) wtrows[q] = nb;
        for (int r : nb) for (int q : bp) wrows[r - L.e1].push_back(q);
      }
      for (auto& w : wrows) std::sort(w.begin(), w.end());
      build_blocks(L.blk, L.blocks); placeb(L.blk);
      build_sliced(L.w, L.e1, wrows); place(L.w);
      build_sliced(L.wt, L.e0, wtrows); place(L.wt);
      C.lev.push_back(std::move(L));
    }
    {   // levels >= 1 (recompute the evolving Schur pattern to get W patterns)
      std::vector<char> Sb2((size_t)nG * nG, 0);
      for (int t = 0; t < nG; ++t)
        for (int j : adj[G[t]]) if (gpos[j] >= 0) Sb2[(size_t)t * nG + gpos[j]] = 1;
      for (auto& b : blocks0) {
        std::vector<int> nb;
        for (int u : b) for (int v : adj[u]) if (gpos[v] >= 0) nb.push_back(gpos[v]);
        std::sort(nb.begin(), nb.end()); nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
        for (int a : nb) for (int c : nb) Sb2[(size_t)a * nG + c] = 1;
      }
      std::vector<char> al(nG, 1);
      int start = (int)E0.size();
      for (auto& Lset : Elev) {
        Level L;
        L.e0 = start; L.e1 = start + (int)Lset.size();
        std::vector<std::vector<int>> wrows(n - L.e1), wtrows(Lset.size());
        for (size_t a = 0; a < Lset.size(); ++a) {
          int t = Lset[a];
          int q = pos[G[t]];
          L.blocks.push_back({q});
          std::vector<int> nb;
          for (int u = 0; u < nG; ++u)
            if (u != t && al[u] && Sb2[(size_t)t * nG + u]) {
              bool inE = std::binary_search(Lset.begin(), Lset.end(), u);
              if (!inE) nb.push_back(pos[G[u]]);
            }
          std::sort(nb.begin(), nb.end());
          wtrows[a] = nb;
          for (int r : nb) wrows[r - L.e1].push_back(q);
        }
        for (auto& w : wrows) std::sort(w.begin(), w.end());
        for (int t : Lset) al[t] = 0;
        for (int t : Lset) {
          std::vector<int> nb;
          for (int u = 0; u < nG; ++u) if (al[u] && Sb2[(size_t)t * nG + u]) nb.push_back(u);
          for (int a : nb) for (int c : nb) Sb2[(size_t)a * nG + c] = 1;
        }
        build_blocks(L.blk, L.blocks); placeb(L.blk);
        build_sliced(L.w, L.e1, wrows); place(L.w);
        build_sliced(L.wt, L.e0, wtrows); place(L.wt);
        C.lev.push_back(std::move(L));
        start = C.lev.back().e1;
      }
      // final block
      C.m = n - start;
      vofs = (vofs + 1) & ~int64_t(1);   // 16-byte alignment of the tile stream (TMA bulk copies)
      C.vofs_final = vofs;
      if (in.factorization == 0) {
        C.final_kind = FINAL_DENSE_INV;
        const int64_t T = (C.m + 31) / 32;
        vofs += T * (T + 1) / 2 * 1024;
      } else {
        C.final_kind = FINAL_ICC;
        // ICC(0) on the Schur pattern of the final block (positions start..n-1, pinned order)
        const int m = C.m;
        std::vector<std::vector<int>> rows(m);
        for (int a = 0; a < m; ++a) {
          int ta = finalset[a];
          for (int b = 0; b <= a; ++b) if (Sb2[(size_t)ta * nG + finalset[b]]) rows[a].push_back(b);
        }
        C.icc_rowptr.assign(m + 1, 0); C.icc_col.clear();
        for (int a = 0; a < m; ++a) {
          C.icc_rowptr[a + 1] = C.icc_rowptr[a] + (int)rows[a].size();
          C.icc_col.insert(C.icc_col.end(), rows[a].begin(), rows[a].end());
        }
        const int nnz = C.icc_rowptr[m];
        // forward levels
        std::vector<int> lv(m, 0);
        int maxl = 0;
        for (int a = 0; a < m; ++a) {
          int l = 0;
          for (int t = C.icc_rowptr[a]; t < C.icc_rowptr[a + 1]; ++t) { int b = C.icc_col[t]; if (b != a) l = std::max(l, lv[b] + 1); }
          lv[a] = l; maxl = std::max(maxl, l);
        }
        C.icc_level_ptr.assign(maxl + 2, 0); C.icc_level_rows.clear();
        for (int l = 0; l <= maxl; ++l) {
          for (int a = 0; a < m; ++a) if (lv[a] == l) C.icc_level_rows.push_back(a);
          C.icc_level_ptr[l + 1] = (int)C.icc_level_rows.size();
        }
        // transpose (rows of L^T), diag last -> first
        std::vector<std::vector<std::pair<int, int>>> trows(m);
        for (int a = 0; a < m; ++a)
          for (int t = C.icc_rowptr[a]; t < C.icc_rowptr[a + 1]; ++t) trows[C.icc_col[t]].push_back({a, t});
        C.icct_rowptr.assign(m + 1, 0); C.icct_col.clear(); C.icct_src.clear();
        for (int b = 0; b < m; ++b) {
          std::sort(trows[b].begin(), trows[b].end());
          C.icct_rowptr[b + 1] = C.icct_rowptr[b] + (int)trows[b].size();
          for (auto& pr : trows[b]) { C.icct_col.push_back(pr.first); C.icct_src.push_back(pr.second); }
        }
        std::vector<int> lt(m, 0);
        int maxt = 0;
        for (int b = m - 1; b >= 0; --b) {
          int l = 0;
          for (int t = C.icct_rowptr[b]; t < C.icct_rowptr[b + 1]; ++t) { int a = C.icct_col[t]; if (a != b) l = std::max(l, lt[a] + 1); }
          lt[b] = l; maxt = std::max(maxt, l);
        }
        C.icct_level_ptr.assign(maxt + 2, 0); C.icct_level_rows.clear();
        for (int l = 0; l <= maxt; ++l) {
          for (int b = 0; b < m; ++b) if (lt[b] == l) C.icct_level_rows.push_back(b);
          C.icct_level_ptr[l + 1] = (int)C.icct_level_rows.size();
        }
        vofs += 2 * (int64_t)nnz;   // L values (row order) then L^T values (transpose order)
      }
    }
    C.nvals_canon = (vofs + 1) & ~int64_t(1);
  }

  // ---------------------------------------------------------------- numeric factorization
  // Returns false on a non-positive pivot (message in err).
  bool factor_patch(const ClassProgram& C, const Entity& e, double* out, double shift, std::string& err) {
    const int n = C.n;
    const int p = sp.p;
    std::vector<double> P(C.pcol.size(), 0.0);
    // assemble from the star cells
    std::vector<int> cr[3];
    for (int d = 0; d < 3; ++d) {
      const DirSpec& s = e.s[d];
      if (s.kind == 1) cr[d] = {s.v};
      else { if (s.v - 1 >= 0) cr[d].push_back(s.v - 1); if (s.v < sp.n[d]) cr[d].push_back(s.v); }
    }
    int slot = 0;
    CellEntries ce;
    for (int cz : cr[2]) for (int cy : cr[1]) for (int cx : cr[0]) {
      const std::vector<int>& mp = C.slot_map[slot++];
      const double a = coef(in.alpha, in.n_alpha, cx, cy, cz), b = coef(in.beta, in.n_beta, cx, cy, cz);
      const CellEntries* E;
      if (in.cartesian) {
        E = &cart_entries(in.hx[cx], in.hy[cy], in.hz[cz]);
      } else {
        double Xc[8][3];
        for (int az = 0; az < 2; ++az)
          for (int ay = 0; ay < 2; ++ay)
            for (int ax = 0; ax < 2; ++ax) {
              int64_t vi = (((int64_t)(cz + az) * (sp.n[1] + 1) + (cy + ay)) * (sp.n[0] + 1) + (cx + ax)) * 3;
              for (int i = 0; i < 3; ++i) Xc[az * 4 + ay * 2 + ax][i] = in.coords[vi + i];
            }
        aux_cell_entries(p, Xc, a, b, ce);
        E = &ce;
      }
      const bool cart = in.cartesian;
      for (size_t t = 0; t < E->row.size(); ++t) {
        int i = mp[E->row[t]], j = mp[E->col[t]];
        if (i < 0 || j < 0) continue;
        const int* b0 = &C.pcol[C.prow[i]];
        const int* b1 = &C.pcol[C.prow[i + 1]];
        const int* it = std::lower_bound(b0, b1, j);
        double v = cart ? (a * E->kval[t] + b * E->mval[t]) : E->kval[t];
        P[it - C.pcol.data()] += v;
      }
    }
    if (shift != 0.0)
      for (int i = 0; i < n; ++i) {
        const int* b0 = &C.pcol[C.prow[i]];
        const int* it = std::lower_bound(b0, &C.pcol[C.prow[i + 1]], i);
        P[it - C.pcol.data()] *= (1.0 + shift);
      }
    auto Pij = [&](int i, int j) -> double {
      const int* b0 = &C.pcol[C.prow[i]];
      const int* b1 = &C.pcol[C.prow[i + 1]];
      const int* it = std::lower_bound(b0, b1, j);
      return (it != b1 && *it == j) ? P[it - C.pcol.data()] : 0.0;
    };
    const Level& L0 = C.lev[0];
    const int nI = L0.e1, nG = n - nI;
    // dense Schur complement over positions nI..n-1
    std::vector<double> S((size_t)nG * nG, 0.0);
    for (int r = nI; r < n; ++r)
      for (int t = C.prow[r]; t < C.prow[r + 1]; ++t) {
        int c = C.pcol[t];
        if (c >= nI) S[(size_t)(r - nI) * nG + (c - nI)] = P[t];
      }
    // level 0: block inverses, W = P_RE Dinv, S -= W P_ER
    auto put_sliced = [&](const Sliced& s, auto&& val) {
      double* o = out + s.vofs;
      const int nsl = (int)s.slice_w.size();
      for (int sl = 0; sl < nsl; ++sl)
        for (int l = 0; l < 32; ++l) {
          int r = sl * 32 + l;
          if (r >= s.nrows) continue;
          const auto& rc = s.rowcols[r];
          for (size_t kk = 0; kk < rc.size(); ++kk) o[s.slice_off[sl] + kk * 32 + l] = val(s.r0 + r, rc[kk]);
        }
    };
    auto put_blocks = [&](const Blocks& B, const std::vector<std::vector<double>>& Lb) {
      // Lb[i]: row-major lower factor of block i (bs_i x bs_i); stored slot-major, diag inverted
      double* o = out + B.vofs;
      for (int i = 0; i < B.nblk; ++i) {
        const int bs = (int)std::lround(std::sqrt((double)Lb[i].size()));
        int slot = 0;
        for (int r = 0; r < B.bs; ++r)
          for (int c = 0; c <= r; ++c, ++slot) {
            double v = 0.0;
            if (r < bs && c <= r) v = Lb[i][r * bs + c];
            if (r == c) v = (r < bs) ? 1.0 / v : 0.0;
            o[(size_t)slot * B.nblk + i] = v;
          }
      }
    };
    {
      // level 0: Cholesky of each interior block, M = P_RE L^{-T}, S -= M M^T
      const int nb0 = (int)L0.blocks.size();
      std::vector<std::vector<double>> Lb(nb0);
      std::vector<int> bid(n, -1), bidx(n, 0);
      for (int bi = 0; bi < nb0; ++bi) {
        const auto& b = L0.blocks[bi];
        const int bs = (int)b.size();
        std::vector<double> Lm(bs * bs, 0.0);
        for (int j = 0; j < bs; ++j) {
          double d = Pij(b[j], b[j]);
          for (int k = 0; k < j; ++k) d -= Lm[j * bs + k] * Lm[j * bs + k];
          if (!(d > 0)) { err = "non-positive pivot in an interior block"; return false; }
          Lm[j * bs + j] = std::sqrt(d);
          for (int i = j + 1; i < bs; ++i) {
            double t = Pij(b[i], b[j]);
            for (int k = 0; k < j; ++k) t -= Lm[i * bs + k] * Lm[j * bs + k];
            Lm[i * bs + j] = t / Lm[j * bs + j];
          }
        }
        for (int i = 0; i < bs; ++i) { bid[b[i]] = bi; bidx[b[i]] = i; }
        Lb[bi] = Lm;
      }
      put_blocks(L0.blk, Lb);
      // M rows per block: for r in nb(block): M[r][b] = solve L_b m = P[b][r]  (m = L^{-1} P_br)
      std::vector<std::map<int, double>> What(nG);   // interface row -> (E position -> (P_EE^{-1} P_ER)^T)
      for (int bi = 0; bi < nb0; ++bi) {
        const auto& b = L0.blocks[bi];
        const int bs = (int)b.size();
        std::vector<int> nb;
        for (int q : b)
          for (int t = C.prow[q]; t < C.prow[q + 1]; ++t) if (C.pcol[t] >= nI) nb.push_back(C.pcol[t]);
        std::sort(nb.begin(), nb.end()); nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
        const std::vector<double>& Lm = Lb[bi];
        std::vector<double> Mv(nb.size() * bs);
        for (size_t i = 0; i < nb.size(); ++i) {
          double y[3];
          for (int j = 0; j < bs; ++j) {
            double t = Pij(nb[i], b[j]);
            for (int k = 0; k < j; ++k) t -= Lm[j * bs + k] * y[k];
            y[j] = t / Lm[j * bs + j];
            Mv[i * bs + j] = y[j];
          }
        }
        for (size_t i = 0; i < nb.size(); ++i)
          for (size_t c = 0; c < nb.size(); ++c) {
            double s = 0;
            for (int j = 0; j < bs; ++j) s += Mv[i * bs + j] * Mv[c * bs + j];
            S[(size_t)(nb[i] - nI) * nG + (nb[c] - nI)] -= s;
          }
        // backward coupling W^ = P_EE^{-1} P_ER: z = L^{-T} y for every neighbour column
        for (size_t i = 0; i < nb.size(); ++i) {
          double z[3];
          for (int j = bs - 1; j >= 0; --j) {
            double t = Mv[i * bs + j];
            for (int k = j + 1; k < bs; ++k) t -= Lm[k * bs + j] * z[k];
            z[j] = t / Lm[j * bs + j];
            What[nb[i] - nI][b[j]] = z[j];
          }
        }
      }
      // forward: v_R -= P_RE y^_E with y^_E = P_EE^{-1} v_E (computed in place by the pivot step);
      // backward: x_E = y^_E - (P_EE^{-1} P_ER) x_R
      put_sliced(L0.w, [&](int r, int q) { return Pij(r, q); });
      put_sliced(L0.wt, [&](int q, int r) {
        const auto& mr = What[r - nI];
        auto it = mr.find(q);
        return it == mr.end() ? 0.0 : it->second;
      });
    }
    // levels >= 1 on the dense Schur complement, 1x1 pivots: L = sqrt(S_qq), M = S_Rq / L
    for (size_t l = 1; l < C.lev.size(); ++l) {
      const Level& L = C.lev[l];
      auto Sv = [&](int r, int c) -> double& { return S[(size_t)(r - nI) * nG + (c - nI)]; };
      std::vector<std::vector<double>> Lb;
      for (int q = L.e0; q < L.e1; ++q) {
        if (!(Sv(q, q) > 0)) { err = "non-positive pivot in an interface level"; return false; }
        Lb.push_back({std::sqrt(Sv(q, q))});
      }
      put_blocks(L.blk, Lb);
      put_sliced(L.w, [&](int r, int q) { return Sv(r, q); });
      put_sliced(L.wt, [&](int q, int r) { return Sv(q, r) / Sv(q, q); });
      for (int q = L.e0; q < L.e1; ++q) {
        const auto& nb = L.wt.rowcols[q - L.e0];
        double d = Sv(q, q);
        std::vector<double> w(nb.size()), sq(nb.size());
        for (size_t i = 0; i < nb.size(); ++i) { w[i] = Sv(nb[i], q) / d; sq[i] = Sv(q, nb[i]); }
        for (size_t i = 0; i < nb.size(); ++i)
          for (size_t c = 0; c < nb.size(); ++c) Sv(nb[i], nb[c]) -= w[i] * sq[c];
      }
    }
    // final block
    const int m = C.m, f0 = n - m;
    std::vector<double> F((size_t)m * m);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) F[(size_t)i * m + j] = S[(size_t)(f0 + i - nI) * nG + (f0 + j - nI)];
    if (C.final_kind == FINAL_DENSE_INV) {
      // Cholesky F = L L^T (lower, in place), Linv, then inverse lower = (Linv^T Linv) lower part
      for (int j = 0; j < m; ++j) {
        double d = F[(size_t)j * m + j];
        for (int k = 0; k < j; ++k) d -= F[(size_t)j * m + k] * F[(size_t)j * m + k];
        if (!(d > 0)) { err = "non-positive pivot in the final interface block"; return false; }
        d = std::sqrt(d);
        F[(size_t)j * m + j] = d;
        for (int i = j + 1; i < m; ++i) {
          double s = F[(size_t)i * m + j];
          const double* fi = &F[(size_t)i * m];
          const double* fj = &F[(size_t)j * m];
          for (int k = 0; k < j; ++k) s -= fi[k] * fj[k];
          F[(size_t)i * m + j] = s / d;
        }
      }
      // Linv lower (row-major): solve L X = I column by column
      std::vector<double> Li((size_t)m * m, 0.0);
      for (int c = 0; c < m; ++c) {
        Li[(size_t)c * m + c] = 1.0 / F[(size_t)c * m + c];
        for (int i = c + 1; i < m; ++i) {
          double s = 0;
          const double* fi = &F[(size_t)i * m];
          for (int k = c; k < i; ++k) s += fi[k] * Li[(size_t)k * m + c];
          Li[(size_t)i * m + c] = -s / F[(size_t)i * m + i];
        }
      }
      // inverse(i,j) = sum_{k >= max(i,j)} Li(k,i) Li(k,j)
      // transpose Li for contiguous access: LiT[i][k] = Li[k][i]
      std::vector<double> LiT((size_t)m * m), Sinv((size_t)m * m);
      for (int i = 0; i < m; ++i) for (int k = 0; k < m; ++k) LiT[(size_t)i * m + k] = Li[(size_t)k * m + i];
      for (int i = 0; i < m; ++i)
        for (int j = 0; j <= i; ++j) {
          const double* a = &LiT[(size_t)i * m];
          const double* b = &LiT[(size_t)j * m];
          double s = 0;
          for (int k = i; k < m; ++k) s += a[k] * b[k];
          Sinv[(size_t)i * m + j] = Sinv[(size_t)j * m + i] = s;
        }
      // 32x32 tiles of the lower block triangle, row-major over (I, J <= I), diagonal tiles full;
      // inside a tile element (r, c) sits at r*32 + ((c + r) & 31) (bank-conflict-free rows and
      // columns in shared memory after a TMA bulk copy)
      double* o = out + C.vofs_final;
      const int T = (m + 31) / 32;
      for (int I = 0; I < T; ++I)
        for (int J = 0; J <= I; ++J) {
          double* tb = o + (size_t)(I * (I + 1) / 2 + J) * 1024;
          for (int r = 0; r < 32; ++r)
            for (int c = 0; c < 32; ++c) {
              const int i = 32 * I + r, j = 32 * J + c;
              tb[r * 32 + ((c + r) & 31)] = (i < m && j < m) ? Sinv[(size_t)i * m + j] : 0.0;
            }
        }
    } else {
      // ICC(0) on the final pattern, up-looking rows (same definition as oracle/patches.py)
      const int nnz = C.icc_rowptr[m];
      std::vector<double> Lv(nnz, 0.0);
      for (int a = 0; a < m; ++a) {
        for (int t = C.icc_rowptr[a]; t < C.icc_rowptr[a + 1]; ++t) {
          int b = C.icc_col[t];
          double s = F[(size_t)a * m + b];
          // sum_{k<b} L_ak L_bk over the two sparse rows
          int ia = C.icc_rowptr[a], ib = C.icc_rowptr[b];
          const int ea = t, eb = C.icc_rowptr[b + 1] - 1;   // exclude column b itself in both rows
          while (ia < ea && ib < eb) {
            int ca = C.icc_col[ia], cb = C.icc_col[ib];
            if (ca == cb) { s -= Lv[ia] * Lv[ib]; ++ia; ++ib; }
            else if (ca < cb) ++ia; else ++ib;
          }
          if (b == a) {
            if (!(s > 0)) { err = "icc breakdown"; return false; }
            Lv[t] = std::sqrt(s);
          } else {
            Lv[t] = s / Lv[C.icc_rowptr[b + 1] - 1];
          }
        }
      }
      double* o = out + C.vofs_final;
      for (int t = 0; t < nnz; ++t) o[t] = Lv[t];
      for (int a = 0; a < m; ++a) { int t = C.icc_rowptr[a + 1] - 1; o[t] = 1.0 / Lv[t]; }
      for (int t = 0; t < nnz; ++t) {
        int src = C.icct_src[t];
        o[nnz + t] = o[src];
      }
    }
    return true;
  }

  std::map<std::tuple<double, double, double>, CellEntries> cart_cache;
  std::mutex cart_mu;
  const CellEntries& cart_entries(double hx, double hy, double hz) {
    std::lock_guard<std::mutex> lk(cart_mu);
    auto key = std::make_tuple(hx, hy, hz);
    auto it = cart_cache.find(key);
    if (it == cart_cache.end()) it = cart_cache.emplace(key, cartesian_cell_entries(op, sp, hx, hy, hz)).first;
    return it->second;
  }
};

// ------------------------------------------------------------------ device numeric program
// (patches.hpp NumProg; executed by dsetup.cu).  Mirrors factor_patch value by value.
void build_numeric_program(const ClassProgram& C, const std::vector<int>& cell_rows,
                           const std::vector<int>& cell_cols, NumProg& o) {
  o = NumProg();
  const int n = C.n;
  o.n = n;
  o.nnzP = (int)C.pcol.size();
  o.final_kind = C.final_kind;
  o.ncanon = C.nvals_canon;
  o.nvals = C.nvals;
  o.vofs_final = C.vofs_final;
  if (n == 0) return;
  const Level& L0 = C.lev[0];
  const int nI = L0.e1, nG = n - nI;
  o.nI = nI; o.nG = nG; o.m = C.m;
  auto csr = [&](int i, int j) -> int {
    const int* b0 = &C.pcol[C.prow[i]];
    const int* b1 = &C.pcol[C.prow[i + 1]];
    const int* it = std::lower_bound(b0, b1, j);
    return (it != b1 && *it == j) ? (int)(it - C.pcol.data()) : -1;
  };
  // canonical index of element (row r, column col) of a sliced block
  auto sliced_at = [&](const Sliced& S, int r, int col) -> int {
    const int rr = r - S.r0, sl = rr / 32, l = rr % 32;
    const auto& rc = S.rowcols[rr];
    const int kk = (int)(std::lower_bound(rc.begin(), rc.end(), col) - rc.begin());
    if (kk >= (int)rc.size() || rc[kk] != col) throw std::runtime_error("numeric program: sliced entry missing");
    return (int)(S.vofs + S.slice_off[sl] + (int64_t)kk * 32 + l);
  };
  // assembly terms in factor_patch's order: slot, then cell entry
  const int ne = (int)cell_rows.size();
  std::vector<std::vector<int>> terms(o.nnzP);
  for (size_t slot = 0; slot < C.slot_map.size(); ++slot) {
    const std::vector<int>& mp = C.slot_map[slot];
    for (int t = 0; t < ne; ++t) {
      const int i = mp[cell_rows[t]], j = mp[cell_cols[t]];
      if (i < 0 || j < 0) continue;
      const int e = csr(i, j);
      if (e < 0) throw std::runtime_error("numeric program: cell entry outside the patch pattern");
      terms[e].push_back((int)slot * ne + t);
    }
  }
  o.asm_ptr.assign(o.nnzP + 1, 0);
  for (int e = 0; e < o.nnzP; ++e) {
    o.asm_ptr[e + 1] = o.asm_ptr[e] + (int)terms[e].size();
    o.asm_src.insert(o.asm_src.end(), terms[e].begin(), terms[e].end());
  }
  o.pdiag.resize(n);
  for (int i = 0; i < n; ++i) o.pdiag[i] = csr(i, i);
  // level 0: blocks, neighbour records (r, P(r, b_j), canon W^(b_j, r)), W = P_RE copies
  o.nb0 = (int)L0.blocks.size();
  o.bs0 = L0.blk.bs;
  o.blk0_vofs = L0.blk.vofs;
  std::vector<std::vector<int>> nbs(o.nb0);
  for (int bi = 0; bi < o.nb0; ++bi) {
    const auto& b = L0.blocks[bi];
    const int bs = (int)b.size();
    int rec[12];
    std::fill(rec, rec + 12, -1);
    rec[0] = bs;
    for (int j = 0; j < bs; ++j) rec[1 + j] = b[j];
    for (int i = 0, k = 0; i < 3; ++i)
      for (int j = 0; j <= i; ++j, ++k) rec[4 + k] = (i < bs && j < bs) ? csr(b[i], b[j]) : -1;
    std::vector<int> nb;
    for (int q : b)
      for (int t = C.prow[q]; t < C.prow[q + 1]; ++t) if (C.pcol[t] >= nI) nb.push_back(C.pcol[t]);
    std::sort(nb.begin(), nb.end()); nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    rec[10] = (int)(o.nbr.size() / 7);
    for (int r : nb) {
      o.nbr.push_back(r - nI);
      for (int j = 0; j < 3; ++j) o.nbr.push_back(j < bs ? csr(r, b[j]) : -1);
      for (int j = 0; j < 3; ++j) o.nbr.push_back(j < bs ? sliced_at(L0.wt, b[j], r) : -1);
    }
    rec[11] = (int)(o.nbr.size() / 7);
    o.b0.insert(o.b0.end(), rec, rec + 12);
    nbs[bi] = nb;
  }
  for (int rr = 0; rr < L0.w.nrows; ++rr)
    for (int q : L0.w.rowcols[rr]) {
      const int r = L0.w.r0 + rr;
      o.w0.push_back(sliced_at(L0.w, r, q));
      o.w0.push_back(csr(r, q));
    }
  // S targets (lower): P_GG entries and the level-0 contributions M_a . M_c, in block order
  const bool icc = C.final_kind == FINAL_ICC;
  if (icc && C.m != nG) throw std::runtime_error("numeric program: ICC final block is not the whole interface");
  std::map<std::pair<int, int>, int> tid;
  std::vector<int> tcsr;
  std::vector<std::vector<int>> tsrc;
  auto target = [&](int a, int c) -> int {
    auto it = tid.find({a, c});
    if (it != tid.end()) return it->second;
    const int id = (int)tcsr.size();
    tid.emplace(std::make_pair(a, c), id);
    tcsr.push_back(csr(nI + a, nI + c));
    tsrc.emplace_back();
    return id;
  };
  for (int r = nI; r < n; ++r)
    for (int t = C.prow[r]; t < C.prow[r + 1]; ++t)
      if (C.pcol[t] >= nI && C.pcol[t] <= r) target(r - nI, C.pcol[t] - nI);
  for (int bi = 0; bi < o.nb0; ++bi) {
    const int r0 = o.b0[12 * bi + 10];
    const auto& nb = nbs[bi];
    for (size_t i = 0; i < nb.size(); ++i)
      for (size_t c = 0; c <= i; ++c) {
        const int id = target(nb[i] - nI, nb[c] - nI);
        tsrc[id].push_back(r0 + (int)i);
        tsrc[id].push_back(r0 + (int)c);
      }
  }
  std::vector<int> icc_at;
  if (icc) {   // ICC entry of (row a, column c) in the final pattern
    o.icc_rowptr = C.icc_rowptr; o.icc_col = C.icc_col;
    o.icc_lptr = C.icc_level_ptr; o.icc_lrows = C.icc_level_rows;
    o.icct_src = C.icct_src;
  }
  o.st_ptr.push_back(0);
  for (auto& kv : tid) {
    const int a = kv.first.first, c = kv.first.second, id = kv.second;
    int idx;
    if (icc) {
      const int* b0 = &C.icc_col[C.icc_rowptr[a]];
      const int* b1 = &C.icc_col[C.icc_rowptr[a + 1]];
      const int* it = std::lower_bound(b0, b1, c);
      if (it == b1 || *it != c) throw std::runtime_error("numeric program: Schur entry outside the ICC pattern");
      idx = (int)(it - C.icc_col.data());
    } else {
      idx = a * nG + c;
    }
    o.st_idx.push_back(idx);
    o.st_csr.push_back(tcsr[id]);
    o.st_src.insert(o.st_src.end(), tsrc[id].begin(), tsrc[id].end());
    o.st_ptr.push_back((int)o.st_src.size() / 2);
  }
  // exact levels >= 1 read off the dense Cholesky factor of S (position order)
  if (!icc)
    for (size_t l = 1; l < C.lev.size(); ++l) {
      const Level& L = C.lev[l];
      for (int i = 0; i < L.blk.nblk; ++i) {
        const int q = L.blocks[i][0] - nI;
        o.rec.insert(o.rec.end(), {(int)(L.blk.vofs + i), 0, q, q});
      }
      for (int rr = 0; rr < L.w.nrows; ++rr)
        for (int q : L.w.rowcols[rr]) {
          const int r = L.w.r0 + rr;
          o.rec.insert(o.rec.end(), {sliced_at(L.w, r, q), 1, r - nI, q - nI});
        }
      for (int qq = 0; qq < L.wt.nrows; ++qq)
        for (int r : L.wt.rowcols[qq]) {
          const int q = L.wt.r0 + qq;
          o.rec.insert(o.rec.end(), {sliced_at(L.wt, q, r), 2, r - nI, q - nI});
        }
    }
  // canonical -> stream map: pack canon[c] = 2c + 1 (odd integers; halved entries are not integers)
  std::vector<double> canon(C.nvals_canon), out(C.nvals);
  for (int64_t c = 0; c < C.nvals_canon; ++c) canon[c] = 2.0 * (double)c + 1.0;
  pack_stream(C, canon.data(), out.data());
  o.smap.resize(C.nvals);
  for (int64_t k = 0; k < C.nvals; ++k) {
    const double x = out[k];
    if (x == 0.0) o.smap[k] = -1;
    else if (x == std::floor(x)) o.smap[k] = (int)((x - 1.0) / 2.0);
    else o.smap[k] = -2 - (int)(x - 0.5);
  }
}

std::unique_ptr<PatchFamily> build_patch_family(const SetupInput& in) {
  auto fam = std::make_unique<PatchFamily>();
  Builder B(in, fam.get());
  fam->sp = B.sp; fam->dim = in.dim; fam->gamma_d = in.gamma_d; fam->factorization = in.factorization;
  std::vector<Entity> ents = entities(B.sp, in.dim, in.interior_only != 0);
  if (in.orient >= 0 && (in.dim == 1 || in.dim == 2)) {   // one orientation: tighter window boxes
    std::vector<Entity> kept;
    for (const Entity& e : ents) {
      int dir = -1;
      for (int d = 0; d < 3; ++d)
        if ((in.dim == 1 && e.s[d].kind == 1) || (in.dim == 2 && e.s[d].kind == 0)) dir = d;
      if (dir == in.orient) kept.push_back(e);
    }
    ents.swap(kept);
  }
  if (in.zv_lo > 0 || in.zv_hi <= B.sp.n[2]) {
    // z-slab ownership: the stars whose entity's z anchor (a vertex layer, or a cell layer for
    // entities spanning a cell in z) lies in the owned layers [zv_lo, zv_hi)
    std::vector<Entity> kept;
    for (const Entity& e : ents)
      if (e.s[2].v >= in.zv_lo && e.s[2].v < in.zv_hi) kept.push_back(e);
    ents.swap(kept);
  }
  std::map<ClassKey, int> cls_of;
  std::vector<int> ecls(ents.size());
  std::vector<Entity> rep;
  for (size_t i = 0; i < ents.size(); ++i) {
    ClassKey k = class_key(B.sp, ents[i]);
    auto it = cls_of.find(k);
    if (it == cls_of.end()) { it = cls_of.emplace(k, (int)rep.size()).first; rep.push_back(ents[i]); }
    ecls[i] = it->second;
  }
  fam->classes.resize(rep.size());
  for (size_t c = 0; c < rep.size(); ++c) B.build_class(rep[c], fam->classes[c]);
  // window boxes (the patches' working vectors): per sub-box (component, or anchor plane for
  // static condensation) the largest extent of any class plus one in x (box origins are rounded
  // down to even x: a TMA box row must start 16-byte aligned), x extent rounded up to even (TMA
  // rows are multiples of 16 bytes); sub-boxes at 128-byte aligned offsets
  const Space& spf = B.sp;
  const bool fam_sc = !fam->classes.empty() && fam->classes[0].sc;
  fam->nsub = fam_sc ? 3 : spf.ncomp;
  for (int sb = 0; sb < 3; ++sb) fam->sub_comp[sb] = fam_sc ? 0 : sb;
  {
    for (int m = 0; m < 3; ++m)
      for (int d = 0; d < 3; ++d) fam->box[m][d] = 0;
    for (auto& C : fam->classes)
      if (C.n > 0)
        for (int m = 0; m < fam->nsub; ++m)
          for (int d = 0; d < 3; ++d) fam->box[m][d] = std::max(fam->box[m][d], C.sub_ext[m][d] + (d == 0 ? 1 : 0));
    int off = 0;
    for (int m = 0; m < fam->nsub; ++m) {
      fam->box[m][0] = (fam->box[m][0] + 1) & ~1;
      fam->boff[m] = off;
      off += (fam->box[m][0] * fam->box[m][1] * fam->box[m][2] + 15) & ~15;
    }
    for (int m = fam->nsub; m <= 3; ++m) fam->boff[m] = off;
    fam->box_total = off;
    if (off > 0xFFFF) throw std::runtime_error("patch window box larger than 65535 entries");
    for (auto& C : fam->classes) build_stream(C);   // piece layout (metadata after the box indices)
  }
  // drop empty patches
  std::vector<size_t> keep;
  for (size_t i = 0; i < ents.size(); ++i) if (fam->classes[ecls[i]].n > 0) keep.push_back(i);
  const size_t np = keep.size();
  fam->pclass.resize(np); fam->pbase.resize(np * 3); fam->pvals.resize(np); fam->pcolor.resize(np);
  fam->porig.resize(np * 9);
  fam->ncolors = (in.dim == 0) ? 8 : (in.dim == 1 ? 12 : 6);
  // dedup key: class + per-slot coefficients (+ cell sizes); trilinear cells are never shared;
  // x-parity twins of a class share value blocks (same program, different box indices)
  std::map<std::vector<double>, int64_t> dedup;
  std::map<std::pair<int, int>, int> twins;
  std::vector<int64_t> fid(np);
  std::vector<int64_t> foff;
  std::vector<size_t> frep;
  int64_t total = 0;
  for (size_t t = 0; t < np; ++t) {
    const Entity& e = ents[keep[t]];
    const int c = ecls[keep[t]];
    fam->pcolor[t] = color_of(e, in.dim);
    int xmask = 0;
    for (int m = 0; m < 3; ++m)
      for (int d = 0; d < 3; ++d) {
        int o = (m < fam->nsub) ? (int)anchor_coord(e.s[d], B.sp.p) + fam->classes[c].sub_org[m][d] : 0;
        if (d == 0 && (o & 1)) { --o; xmask |= 1 << m; }   // even x origin: the class twin shifts by one
        fam->porig[t * 9 + m * 3 + d] = o;
      }
    {
      auto tw = twins.find({c, xmask});
      if (tw == twins.end()) {
        int idx = c;
        if (xmask != 0) {
          idx = (int)fam->classes.size();
          ClassProgram twin = fam->classes[c];
          for (int m = 0; m < 3; ++m) twin.xshift[m] = (xmask >> m) & 1;
          fam->classes.push_back(std::move(twin));
        }
        tw = twins.emplace(std::make_pair(c, xmask), idx).first;
      }
      fam->pclass[t] = tw->second;
    }
    for (int m = 0; m < 3; ++m)
      fam->pbase[t * 3 + m] = (m < B.sp.ncomp)
          ? B.sp.gidx(m, anchor_coord(e.s[2], B.sp.p), anchor_coord(e.s[1], B.sp.p), anchor_coord(e.s[0], B.sp.p)) : 0;
    std::vector<double> key{(double)c};
    if (in.cartesian) {
      std::vector<int> cr[3];
      for (int d = 0; d < 3; ++d) {
        const DirSpec& s = e.s[d];
        if (s.kind == 1) cr[d] = {s.v};
        else { if (s.v - 1 >= 0) cr[d].push_back(s.v - 1); if (s.v < B.sp.n[d]) cr[d].push_back(s.v); }
      }
      for (int cz : cr[2]) for (int cy : cr[1]) for (int cx : cr[0]) {
        key.push_back(B.coef(in.alpha, in.n_alpha, cx, cy, cz));
        key.push_back(B.coef(in.beta, in.n_beta, cx, cy, cz));
        key.push_back(in.hx[cx]); key.push_back(in.hy[cy]); key.push_back(in.hz[cz]);
      }
    } else {
      key.push_back(-1.0 - (double)t);
    }
    auto it = dedup.find(key);
    if (it == dedup.end()) {
      it = dedup.emplace(key, (int64_t)foff.size()).first;
      foff.push_back(total);
      frep.push_back(t);
      total += fam->classes[c].nvals;
    }
    fam->nnzL_total += fam->classes[c].nnzL;
    fid[t] = it->second;
    fam->pvals[t] = foff[fid[t]];
  }
  // box indices of every class (and twin), the zero lists, and the class meta streams
  for (auto& C : fam->classes) {
    C.bidx.assign(C.n, -1);
    std::vector<char> used(fam->box_total, 0);
    for (int t2 = 0; t2 < C.n; ++t2) {
      const int m = C.psub[t2];
      if (m < 0) continue;   // condensed cell interior (sc)
      const int b = fam->boff[m] + (C.pcoord[3 * t2 + 2] * fam->box[m][1] + C.pcoord[3 * t2 + 1]) * fam->box[m][0] +
                    C.pcoord[3 * t2 + 0] + C.xshift[m];
      C.bidx[t2] = b;
      used[b] = 1;
    }
    C.zlist.clear();
    for (int m = 0; m < fam->nsub; ++m)
      for (int b = fam->boff[m]; b < fam->boff[m] + fam->box[m][0] * fam->box[m][1] * fam->box[m][2]; ++b)
        if (!used[b]) C.zlist.push_back(b);
    // SC-PAFW with the exact elimination program: the patch-local interior corrections are not
    // scattered (the post step computes the cell interiors once from the interface corrections)
    if ((in.sc_decomposition || in.interface_only) && !C.sc)
      for (int t2 = 0; t2 < C.n; ++t2)
        if (C.group[t2] == 0 && C.bidx[t2] >= 0) C.zlist.push_back(C.bidx[t2]);
    build_meta(C);
  }
  fam->nfactors = (int64_t)foff.size();
  fam->unique_value_bytes = total * (int64_t)sizeof(double);
  if (!in.defer_numeric) fam->values.assign(total, 0.0);   // deferred: the blocks live on the device only
  std::string first_err;
  std::mutex emu;
  double smax = 0.0;
  const int64_t nf = (int64_t)foff.size();
  fam->nvalues = total;
  if (in.defer_numeric) {   // device-resident numeric setup: record the inputs, factor nothing here
    fam->deferred = true;
    fam->values.clear();
    fam->values.shrink_to_fit();
    fam->fclass.resize(nf);
    fam->foff = foff;
    fam->fcells.assign((size_t)nf * kMaxSlots, -1);
    for (int64_t f = 0; f < nf; ++f) {
      const size_t t = frep[f];
      const Entity& e = ents[keep[t]];
      fam->fclass[f] = fam->pclass[t];
      std::vector<int> cr[3];
      for (int d = 0; d < 3; ++d) {
        const DirSpec& ds = e.s[d];
        if (ds.kind == 1) cr[d] = {ds.v};
        else { if (ds.v - 1 >= 0) cr[d].push_back(ds.v - 1); if (ds.v < B.sp.n[d]) cr[d].push_back(ds.v); }
      }
      int slot = 0;
      for (int cz : cr[2]) for (int cy : cr[1]) for (int cx : cr[0])
        fam->fcells[(size_t)f * kMaxSlots + slot++] = (cz * B.sp.n[1] + cy) * B.sp.n[0] + cx;
    }
    fam->cell_rows = B.cell_rows; fam->cell_cols = B.cell_cols;
    fam->cartesian = in.cartesian;
    const int64_t ncell = (int64_t)B.sp.n[0] * B.sp.n[1] * B.sp.n[2];
    fam->cell_alpha.resize(ncell); fam->cell_beta.resize(ncell);
    std::map<std::tuple<double, double, double>, int> sets;
    if (in.cartesian) fam->cell_set.resize(ncell);
    for (int64_t K = 0; K < ncell; ++K) {
      const int cx = (int)(K % B.sp.n[0]), cy = (int)((K / B.sp.n[0]) % B.sp.n[1]), cz = (int)(K / ((int64_t)B.sp.n[0] * B.sp.n[1]));
      fam->cell_alpha[K] = B.coef(in.alpha, in.n_alpha, cx, cy, cz);
      fam->cell_beta[K] = B.coef(in.beta, in.n_beta, cx, cy, cz);
      if (in.cartesian) {
        auto key = std::make_tuple(in.hx[cx], in.hy[cy], in.hz[cz]);
        auto it = sets.find(key);
        if (it == sets.end()) {
          it = sets.emplace(key, (int)sets.size()).first;
          const CellEntries& E = B.cart_entries(in.hx[cx], in.hy[cy], in.hz[cz]);
          if (E.row != B.cell_rows || E.col != B.cell_cols) throw std::runtime_error("cell pattern depends on the cell size");
          fam->cset_k.insert(fam->cset_k.end(), E.kval.begin(), E.kval.end());
          fam->cset_m.insert(fam->cset_m.end(), E.mval.begin(), E.mval.end());
        }
        fam->cell_set[K] = it->second;
      }
    }
    if (!in.cartesian) fam->coords.assign(in.coords, in.coords + (B.sp.n[0] + 1) * (B.sp.n[1] + 1) * (B.sp.n[2] + 1) * 3);
  }
#pragma omp parallel for schedule(dynamic, 4) reduction(max : smax)
  for (int64_t f = 0; f < (in.defer_numeric ? 0 : nf); ++f) {
    size_t t = frep[f];
    const Entity& e = ents[keep[t]];
    const ClassProgram& C = fam->classes[fam->pclass[t]];
    std::string err;
    std::vector<double> canon(C.nvals_canon, 0.0);
    bool ok = B.factor_patch(C, e, canon.data(), 0.0, err);
    if (!ok && in.factorization == 1) {   // reading G7: P + sigma diag(P), sigma = 1e-10 doubling
      for (double shift = 1e-10; shift <= 1e-2 && !ok; shift *= 2.0) {
        std::fill(canon.begin(), canon.end(), 0.0);
        ok = B.factor_patch(C, e, canon.data(), shift, err);
        if (ok) smax = std::max(smax, shift);
      }
    }
    if (ok) pack_stream(C, canon.data(), fam->values.data() + foff[f]);
    if (!ok) {
      std::lock_guard<std::mutex> lk(emu);
      if (first_err.empty()) {
        char buf[256];
        snprintf(buf, sizeof buf, "patch %zu (entity %d,%d,%d): %s", t, e.s[0].v, e.s[1].v, e.s[2].v, err.c_str());
        first_err = buf;
      }
    }
  }
  fam->sigma_max = smax;
  fam->sc_pre = fam_sc;
  if (fam_sc || in.sc_decomposition) {
    // per-cell static-condensation data from the same cell entries the patch matrices use
    const Space& sp = B.sp;
    const int p = sp.p, P1 = p + 1, pm = p - 1, ni = pm * pm * pm;
    const int64_t ncell = (int64_t)sp.n[0] * sp.n[1] * sp.n[2];
    fam->sc_dinv.assign((size_t)ncell * ni, 0.0);
    const bool cmp = !in.cartesian;   // trilinear auxiliary operator: compressed couplings
    if (cmp) {
      fam->sc_w.assign((size_t)ncell * 3 * ni, 0.0);
      const Basis1D& b1 = basis(p);
      fam->sc_kd.assign(P1, 0.0); fam->sc_k0.assign(P1, 0.0); fam->sc_kp.assign(P1, 0.0);
      for (int i = 1; i < p; ++i) {
        fam->sc_kd[i] = b1.D[i * P1 + i]; fam->sc_k0[i] = b1.D[i * P1]; fam->sc_kp[i] = b1.D[i * P1 + p];
      }
    } else {
      fam->sc_c.assign((size_t)ncell * 6 * ni, 0.0);
    }
    fam->sc_nk.assign(ncell, 0);
    std::string sc_err;
    if (in.defer_numeric) {   // sc_dinv / sc_c / sc_w are computed on the device (sizes kept)
      fam->sc_dinv.clear(); fam->sc_c.clear(); fam->sc_w.clear();
    }
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t K = 0; K < (in.defer_numeric ? 0 : ncell); ++K) {
      const int cx = (int)(K % sp.n[0]), cy = (int)((K / sp.n[0]) % sp.n[1]), cz = (int)(K / ((int64_t)sp.n[0] * sp.n[1]));
      const double a = B.coef(in.alpha, in.n_alpha, cx, cy, cz), b = B.coef(in.beta, in.n_beta, cx, cy, cz);
      CellEntries ce;
      const CellEntries* E;
      if (in.cartesian) {
        E = &B.cart_entries(in.hx[cx], in.hy[cy], in.hz[cz]);
      } else {
        double Xc[8][3];
        for (int az = 0; az < 2; ++az)
          for (int ay = 0; ay < 2; ++ay)
            for (int ax = 0; ax < 2; ++ax) {
              const int64_t vi = (((int64_t)(cz + az) * (sp.n[1] + 1) + (cy + ay)) * (sp.n[0] + 1) + (cx + ax)) * 3;
              for (int i = 0; i < 3; ++i) Xc[az * 4 + ay * 2 + ax][i] = in.coords[vi + i];
            }
        aux_cell_entries(p, Xc, a, b, ce, cmp ? &fam->sc_w[(size_t)K * 3 * ni] : nullptr);
        E = &ce;
      }
      std::vector<int> nc(ni, 0);
      for (size_t t = 0; t < E->row.size(); ++t) {
        const int r = E->row[t], c = E->col[t];
        const int ra = r % P1, rb = (r / P1) % P1, rc = r / (P1 * P1);
        if (ra == 0 || ra == p || rb == 0 || rb == p || rc == 0 || rc == p) continue;   // row not interior
        const int I = ((rc - 1) * pm + (rb - 1)) * pm + (ra - 1);
        const double v = in.cartesian ? a * E->kval[t] + b * E->mval[t] : E->kval[t];
        const int ca = c % P1, cb = (c / P1) % P1, cc = c / (P1 * P1);
        int face = -1;
        if (c == r) { fam->sc_dinv[(size_t)K * ni + I] += v; continue; }
        if (cb == rb && cc == rc && (ca == 0 || ca == p)) face = ca == 0 ? 0 : 1;
        else if (ca == ra && cc == rc && (cb == 0 || cb == p)) face = cb == 0 ? 2 : 3;
        else if (ca == ra && cb == rb && (cc == 0 || cc == p)) face = cc == 0 ? 4 : 5;
        if (face < 0) {
          if (v != 0.0) {
#pragma omp critical
            sc_err = "static condensation: interior DoF coupled outside its 6 face lines";
          }
          continue;
        }
        if (cmp) {   // the compressed form must reproduce the assembled coupling exactly
          const int iline = face < 2 ? ra : (face < 4 ? rb : rc);
          const double w = fam->sc_w[((size_t)K * 3 + face / 2) * ni + I];
          const double rec = (fam->sc_kd[iline] * w) * ((face & 1) ? fam->sc_kp[iline] : fam->sc_k0[iline]);
          if (rec != v) {
#pragma omp critical
            sc_err = "static condensation: compressed coupling differs from the assembled one";
          }
        } else {
          fam->sc_c[((size_t)K * 6 + face) * ni + I] += v;
        }
        ++nc[I];
      }
      for (int I = 0; I < ni; ++I) {
        double& d = fam->sc_dinv[(size_t)K * ni + I];
        if (!(d > 0)) {
#pragma omp critical
          sc_err = "static condensation: non-positive interior diagonal";
        }
        d = 1.0 / d;
      }
    }
    if (!sc_err.empty()) throw std::runtime_error(sc_err);
    for (size_t t = 0; t < np; ++t) {   // patches containing each cell (its interiors in the window)
      const Entity& e = ents[keep[t]];
      std::vector<int> cr[3];
      for (int d = 0; d < 3; ++d) {
        const DirSpec& ds = e.s[d];
        if (ds.kind == 1) cr[d] = {ds.v};
        else { if (ds.v - 1 >= 0) cr[d].push_back(ds.v - 1); if (ds.v < sp.n[d]) cr[d].push_back(ds.v); }
      }
      for (int cz : cr[2]) for (int cy : cr[1]) for (int cx : cr[0]) ++fam->sc_nk[((int64_t)cz * sp.n[1] + cy) * sp.n[0] + cx];
    }
    // SC-PAFW: the cell interiors are solved once (eq:schur: R_I^T A_II^-1 R_I + R_G^T S^-1 R_G)
    if (in.sc_decomposition) std::fill(fam->sc_nk.begin(), fam->sc_nk.end(), 1);
  }
  if (!first_err.empty()) throw std::runtime_error(first_err);
  return fam;
}

}  // namespace rm
