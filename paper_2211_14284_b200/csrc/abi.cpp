// C ABI (include/rm.h): context, setup (host factorization + upload), sweep orchestration.
#include "../../include/rm.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <omp.h>
#include <nccl.h>   // types and prototypes only: the library is dlopen'ed (rank > 1 only)

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <tuple>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "basis.hpp"
#include "coarse.hpp"
#include "dsetup.hpp"
#include "kernels.cuh"
#include "model.hpp"
#include "patches.hpp"

namespace {

thread_local std::string g_err;

struct RmError : std::runtime_error {
  rm_status st;
  RmError(rm_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) throw RmError(RM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------ NCCL (loaded on demand)
// The process may already hold torch's libnccl.so.2; dlopen returns that one.  No link-time
// dependency: single-GPU use never touches NCCL.
struct NcclApi {
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGroupStart) gstart = nullptr;
  decltype(&ncclGroupEnd) gend = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};
const NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.get_id = reinterpret_cast<decltype(api.get_id)>(dlsym(h, "ncclGetUniqueId"));
      api.init = reinterpret_cast<decltype(api.init)>(dlsym(h, "ncclCommInitRank"));
      api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
      api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
      api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
      api.gstart = reinterpret_cast<decltype(api.gstart)>(dlsym(h, "ncclGroupStart"));
      api.gend = reinterpret_cast<decltype(api.gend)>(dlsym(h, "ncclGroupEnd"));
      api.allreduce = reinterpret_cast<decltype(api.allreduce)>(dlsym(h, "ncclAllReduce"));
      api.errstr = reinterpret_cast<decltype(api.errstr)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  if (!api.init || !api.send || !api.recv || !api.gstart || !api.gend || !api.allreduce || !api.get_id)
    throw RmError(RM_ENCCL, "libnccl.so.2 not loadable");
  return api;
}
#define NK(x)                                                                                       \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess)                                                                          \
      throw RmError(RM_ENCCL, std::string(#x) + ": " + (nccl().errstr ? nccl().errstr(r_) : "error")); \
  } while (0)

// ------------------------------------------------------------------ z-slab partition (rm.h)
void compute_partition(const rm_mesh& m, int p, int space, uint32_t gamma, int rank, int nranks,
                       rm_partition_info& P) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw RmError(RM_EINVAL, "bad rank / nranks");
  (void)space;
  const int zb = m.z_begin, ze = m.z_end;
  if (!(0 <= zb && zb < ze && ze <= m.nz)) throw RmError(RM_EINVAL, "bad z_begin / z_end");
  if (nranks == 1 && (zb != 0 || ze != m.nz)) throw RmError(RM_EINVAL, "one rank must own all layers");
  if (rank == 0 && zb != 0) throw RmError(RM_EINVAL, "rank 0 must start at layer 0");
  if (rank == nranks - 1 && ze != m.nz) throw RmError(RM_EINVAL, "the last rank must end at layer nz");
  std::memset(&P, 0, sizeof P);
  const bool lo = rank > 0, hi = rank < nranks - 1;
  P.ghost_lo = lo ? 1 : 0;
  P.z_cell0 = zb - P.ghost_lo;
  P.nz_local = ze - P.z_cell0;
  const int top = P.nz_local * p;   // local index of the upper plane
  P.v_lo = P.ghost_lo;
  P.v_hi = hi ? P.nz_local : P.nz_local + 1;
  P.own_lo = P.ghost_lo * p;
  P.own_hi = hi ? top : top + 1;
  if (lo) {
    P.fwd_recv_lo[0] = 0; P.fwd_recv_lo[1] = p;          // ghost layer planes, owned by rank - 1
    P.fwd_send_lo[0] = p; P.fwd_send_lo[1] = p + 1;      // my first plane = rank - 1's upper plane
    P.rev_send_lo[0] = 1; P.rev_send_lo[1] = p;          // corrections on the ghost layer's interior
  }
  if (hi) {
    P.fwd_recv_hi[0] = top; P.fwd_recv_hi[1] = top + 1;  // shared upper plane, owned by rank + 1
    P.fwd_send_hi[0] = top - p; P.fwd_send_hi[1] = top;  // rank + 1's ghost layer
    P.rev_recv_hi[0] = top - p + 1; P.rev_recv_hi[1] = top;
  }
  // DP-family components (z index c p + a inside cell layer c): no shared plane
  P.dp_own_lo = P.ghost_lo * p;
  P.dp_own_hi = P.nz_local * p;
  if (lo) {
    P.dp_fwd_recv_lo[0] = 0; P.dp_fwd_recv_lo[1] = p;   // the ghost cell layer, owned by rank - 1
    P.dp_rev_send_lo[0] = 0; P.dp_rev_send_lo[1] = p;   // corrections on the ghost layer
  }
  if (hi) {
    P.dp_fwd_send_hi[0] = top - p; P.dp_fwd_send_hi[1] = top;   // my top layer = rank + 1's ghost layer
    P.dp_rev_recv_hi[0] = top - p; P.dp_rev_recv_hi[1] = top;
  }
  P.gamma_local = gamma & 0x0Fu;
  if (!lo) P.gamma_local |= gamma & 0x10u;
  if (!hi) P.gamma_local |= gamma & 0x20u;
  P.plane_len = ((int64_t)m.nx * p + 1) * ((int64_t)m.ny * p + 1);
}

struct DevFamily {
  std::vector<void*> allocs;
  rm::PatchLaunch launch{};
  std::vector<int> color_start;
  int64_t npatch = 0, nfactors = 0, nclasses = 0;
  int64_t sweep_value_bytes = 0;   // sum over patches of value-block bytes
  int64_t nnzL = 0, unique_bytes = 0;   // algorithmic factor entries (sum over patches), distinct block bytes
  int ncolors = 0;
  double sigma_max = 0.0;
  double numeric_s = 0.0;          // seconds of the numeric setup (device or host) of this family
  bool present = false;

  template <class T>
  T* upload(const std::vector<T>& h) {
    if (h.empty()) return nullptr;
    void* d = nullptr;
    if (cudaMalloc(&d, h.size() * sizeof(T)) != cudaSuccess) throw RmError(RM_ENOMEM, "cudaMalloc failed");
    allocs.push_back(d);
    CK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    return static_cast<T*>(d);
  }
  template <class T>
  T* alloc(size_t n) {
    void* d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) throw RmError(RM_ENOMEM, "cudaMalloc failed");
    allocs.push_back(d);
    return static_cast<T*>(d);
  }
  void release() {
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
    if (launch.tm_dev) cudaFree(launch.tm_dev);
    launch.tm_dev = nullptr;
  }
};

// Class-batched mode (patch_solve.cu, patch_batch_kernel): families whose patches share few value
// blocks (on average >= 4 patches per block), with exact programs (dense final block or none) and
// no static condensation.  Batches = runs of <= B patches of one (class, value block) inside one
// colour; B = the largest of 8, 4, 2 whose working set fits in shared memory.  RM_PATCH_STREAM=1
// (documented test knob, rm.h) keeps the persistent stream kernel.
// pc / pv / pvn: per patch in colour-sorted order: class, host stream-block offset, device offset.
void plan_batches(DevFamily& F, const rm::PatchFamily& P, const std::vector<int>& pc, const std::vector<long long>& pv,
                  const std::vector<long long>& pvn, size_t nblocks, const double* hvals) {
  rm::PatchLaunch& Lh = F.launch;
  Lh.batch = 0;
  const size_t np = pc.size();
  if (np == 0 || std::getenv("RM_PATCH_STREAM") || !P.sc_nk.empty() || nblocks * 4 > np) return;
  int mr_max = 0, np_max = 0;
  for (const auto& C : P.classes) {
    if (C.n > 0 && (C.final_kind != rm::FINAL_DENSE_INV || C.sc)) return;
    mr_max = std::max(mr_max, (C.m + 31) & ~31);
    np_max = std::max(np_max, (int)C.pieces.size());
  }
  if (np_max > rm::kBatchMaxPieces) return;
  // configuration (measured on cfg3 / cfg4, scripts/gpu_batch_sweep.sh): 16 resident warps per SM
  // first (one CTA of 512 or two of 256 threads), then the most patches in flight, then two CTAs
  int B = 0, NT = 0;
  size_t smem = 0;
  long best = -1;
  for (int nt : {256, 384, 512})
    for (int b : {8, 4, 2}) {
      if (nt == 384 && b == 8) continue;   // no instantiation (B = 8 needs > 85 registers)
#ifndef RM_BATCH_384
      if (nt == 384) continue;
#endif
      const size_t sm = rm::patch_batch_smem(P.box_total, mr_max, b, nt);
      if (sm == 0) continue;
#ifdef RM_BATCH_512X2   // tuning build: the 512-thread kernels are capped at 64 registers (two CTAs per SM)
      const int ctas = (2 * (sm + 2048) <= 233472) ? 2 : 1;
#else
      // resident CTAs per SM (patch_solve.cu batch_minb): 256 threads: 3 (B <= 4) or 2 by shared
      // memory; 384 threads: 2 (24 warps where three 256-thread CTAs do not fit); 512: 1
      int ctas = 1;
#ifdef RM_BATCH_384
      if (nt == 256) ctas = (b <= 4 && 3 * (sm + 2048) <= 233472) ? 3 : (2 * (sm + 2048) <= 233472 ? 2 : 1);
#else
      if (nt == 256) ctas = 2 * (sm + 2048) <= 233472 ? 2 : 1;   // (a third CTA, where it fits, does not change the choice)
#endif
      if (nt == 384) {
        if (2 * (sm + 2048) > 233472) continue;
        ctas = 2;
      }
#endif
      const long score = (long)(ctas * nt / 32) * 10000 + (long)(b * ctas) * 10 + ctas;
      if (score > best) { best = score; B = b; NT = nt; smem = sm; }
    }
  if (const char* e = rm::exp_env("RM_BATCH_CFG")) {   // experiments: "B,NT"
    int b = 0, nt = 0;
    size_t sm = 0;
    if (sscanf(e, "%d,%d", &b, &nt) == 2 && (sm = rm::patch_batch_smem(P.box_total, mr_max, b, nt)) > 0) {
      B = b; NT = nt; smem = sm;
    }
  }
  if (B == 0) return;
  std::vector<int> bp;
  std::vector<int> bc;
  std::vector<long long> bb, bf;
  std::vector<double> fin;
  std::unordered_map<long long, long long> fin_of;   // host block offset -> offset in fin
  auto full_inverse = [&](int cls, long long hofs) -> long long {
    const rm::ClassProgram& C = P.classes[cls];
    if (C.m == 0) return 0;
    auto it = fin_of.find(hofs);
    if (it != fin_of.end()) return it->second;
    const int m = C.m, mr = (m + 31) & ~31;
    const long long at = (long long)fin.size();
    fin.resize(fin.size() + (size_t)mr * mr, 0.0);
    double* S = fin.data() + at;
    const double* blk = hvals + hofs;
    for (int pi = C.tile_p0; pi < C.tile_p1; ++pi) {   // half-stored lane-block tiles -> full matrix
      const rm::Piece& pcs = C.pieces[pi];
      if (pcs.kind != rm::PK_TILE) continue;
      const int I = pcs.a0, J = pcs.a1;
      for (int r = 0; r < 32; ++r)
        for (int c = 0; c < 32; ++c) {
          const int gr = 32 * I + r, gc = 32 * J + c;
          if (gr >= m || gc >= m) continue;
          double x;
          if (I != J) x = blk[pcs.sofs + rm::tile_pos_full(r, c)];
          else if (c < r) x = blk[pcs.sofs + rm::tile_pos_diag(r, c)];
          else if (c == r) x = 2.0 * blk[pcs.sofs + rm::tile_pos_diag(r, c)];
          else continue;
          S[(size_t)gr * mr + gc] = x;
          S[(size_t)gc * mr + gr] = x;
        }
    }
    fin_of.emplace(hofs, at);
    return at;
  };
  for (int c = 0; c < P.ncolors; ++c) {
    Lh.bstart[c] = (int)bc.size();
    // runs of one (class, block) in first-appearance order inside the colour
    std::vector<std::pair<long long, int>> keys;
    std::unordered_map<long long, std::vector<int>> runs;
    for (int i = F.color_start[c]; i < F.color_start[c + 1]; ++i) {
      const long long key = pvn[i] * 4096 + pc[i];
      auto it = runs.find(key);
      if (it == runs.end()) { keys.emplace_back(key, i); it = runs.emplace(key, std::vector<int>()).first; }
      it->second.push_back(i);
    }
    for (const auto& k : keys) {
      const std::vector<int>& r = runs[k.first];
      const int i0 = k.second;
      const long long fo = full_inverse(pc[i0], pv[i0]);
      for (size_t s = 0; s < r.size(); s += B) {
        for (int b = 0; b < B; ++b) bp.push_back(s + b < r.size() ? r[s + b] : -1);
        bc.push_back(pc[i0]);
        bb.push_back(pvn[i0]);
        bf.push_back(fo);
      }
    }
  }
  Lh.bstart[P.ncolors] = (int)bc.size();
  Lh.bpatch = F.upload(bp);
  Lh.bclass = F.upload(bc);
  Lh.bblock = F.upload(bb);
  Lh.bfin = F.upload(bf);
  Lh.fin = fin.empty() ? nullptr : F.upload(fin);
  Lh.mr_max = mr_max;
  Lh.bsmem = smem;
  Lh.batch = B;
  Lh.batch_nt = NT;
  if (rm::exp_env("RM_VERBOSE"))
    fprintf(stderr, "[rm] batched patch solve: %zu patches, %zu blocks, B=%d NT=%d, %zu batches, smem=%zu\n", np, nblocks,
            B, NT, bc.size(), smem);
}

// share: a family of the same space whose padded r / c buffers this one uses (orientation families)
void upload_family(DevFamily& F, const rm::PatchFamily& P, const DevFamily* share = nullptr) {
  const int NW = rm::RM_PATCH_TILE_WARPS;
  std::vector<rm::DClass> hc(P.classes.size());
  int n_max = 0, piv_max = 0, mem_max = 0, aux_max = 0, unit_max = 0, unit_max_a = 0, unit_max_b = 0;
  for (size_t c = 0; c < P.classes.size(); ++c) {
    const rm::ClassProgram& C = P.classes[c];
    rm::DClass& d = hc[c];
    std::memset(&d, 0, sizeof d);
    d.n = C.n; d.nlev = C.sc ? 0 : (int)C.lev.size(); d.m = C.m; d.final_kind = C.final_kind;
    if (d.nlev > RM_MAXLEV) throw RmError(RM_EINVAL, "too many elimination levels");
    int auxn = 0;
    for (int l = 0; l < d.nlev; ++l) {
      const rm::Level& L = C.lev[l];
      rm::DLevel& dl = d.lev[l];
      dl.e0 = L.e0; dl.e1 = L.e1;
      dl.blk.nblk = L.blk.nblk;
      dl.blk.bs = L.blk.bs;
      dl.w.r0 = L.w.r0; dl.w.nrows = L.w.nrows;
      dl.wt.r0 = L.wt.r0; dl.wt.nrows = L.wt.nrows;
      dl.piv_b = C.piv_b[l]; dl.w_b = C.w_b[l]; dl.w_e = C.w_e[l]; dl.wt_b = C.wt_b[l]; dl.wt_e = C.wt_e[l];
      dl.piv_per = C.piv_per[l]; dl.piv_ofs = C.piv_ofs[l]; dl.mem_ofs = C.mem_ofs[l];
    }
    std::vector<rm::DUnit> us(C.units.size());
    for (size_t i = 0; i < us.size(); ++i) {
      const rm::Unit& u = C.units[i];
      const bool tile = (int)i >= C.tu0 && (int)i < C.tu1;
      if (u.np > 0x7FFF || u.mbytes > 0xFFFF) throw RmError(RM_EINVAL, "transfer unit too large");
      us[i] = rm::DUnit{u.mofs, (int)((uint32_t)u.mbytes | ((uint32_t)u.np << 16) | (tile ? 0x80000000u : 0u)), u.sofs, u.nd};
      unit_max = std::max(unit_max, u.mbytes + 8 * u.nd);
      if (tile) unit_max_b = std::max(unit_max_b, u.mbytes + 8 * u.nd);
      else unit_max_a = std::max(unit_max_a, u.mbytes + 8 * u.nd);
    }
    d.units = F.upload(us);
    d.meta = F.upload(C.meta);
    {
      std::vector<int2> pt(C.pieces.size());
      for (size_t i = 0; i < pt.size(); ++i) pt[i] = make_int2(C.pieces[i].mofs, C.pieces[i].sofs);
      d.ptab = F.upload(pt);
      d.npieces = (int)pt.size();
    }
    if (!C.frange.empty()) {
      std::vector<int2> fr(C.frange.size() / 2);
      for (size_t i = 0; i < fr.size(); ++i) fr[i] = make_int2(C.frange[2 * i], C.frange[2 * i + 1]);
      d.frange = F.upload(fr);
    }
    d.nunits = (int)us.size();
    d.ngs = C.ngs;
    d.tile_p0 = C.tile_p0; d.tile_p1 = C.tile_p1;
    d.uf0 = C.uf0; d.uf1 = C.uf1;
    d.fin_tiles = (C.final_kind == rm::FINAL_DENSE_INV && C.m > 0) ? 1 : 0;
    if (C.final_kind == rm::FINAL_DENSE_INV) {
      if ((C.m + 31) / 32 > 32) throw RmError(RM_EINVAL, "final Schur block larger than 1024");
      // g + per-tile-warp partials + final-block box list (uint16)
      auxn = std::max(auxn, ((C.m + 31) / 32) * 32 * (NW + 1) + ((C.m + 31) / 32) * 8 + 2);
    } else {
      d.iccf_nlev = (int)C.iccf_lpiece.size() - 1;
      d.iccb_nlev = (int)C.iccb_lpiece.size() - 1;
      d.iccf_lp = F.upload(C.iccf_lpiece);
      d.iccb_lp = F.upload(C.iccb_lpiece);
    }
    n_max = std::max(n_max, C.n);
    piv_max = std::max(piv_max, C.piv_total);
    mem_max = std::max(mem_max, C.mem_total);
    aux_max = std::max(aux_max, (auxn + 1) & ~1);
  }
  if (P.ncolors > rm::RM_MAXCOLORS) throw RmError(RM_EINVAL, "too many colours");
  rm::PatchLaunch& Lh = F.launch;
  Lh.classes = F.upload(hc);
  // patches sorted by colour
  const size_t np = P.pclass.size();
  std::vector<size_t> order(np);
  F.color_start.assign(P.ncolors + 1, 0);
  for (size_t t = 0; t < np; ++t) F.color_start[P.pcolor[t] + 1]++;
  for (int c = 0; c < P.ncolors; ++c) F.color_start[c + 1] += F.color_start[c];
  std::vector<int> fill(F.color_start.begin(), F.color_start.end() - 1);
  for (size_t t = 0; t < np; ++t) order[fill[P.pcolor[t]]++] = t;
  std::vector<int> pc(np), po(9 * np);
  std::vector<long long> pv(np);
  int64_t bytes = 0;
  for (size_t i = 0; i < np; ++i) {
    size_t t = order[i];
    pc[i] = P.pclass[t];
    for (int k = 0; k < 9; ++k) po[9 * i + k] = P.porig[9 * t + k];
    pv[i] = P.pvals[t];
    bytes += P.classes[P.pclass[t]].nvals * 8;
  }
  Lh.pclass = F.upload(pc);
  Lh.porig = F.upload(po);
  // window boxes and the padded component layout of r / c (TMA row strides: multiples of 16 B)
  Lh.ncomp = P.sp.ncomp;
  for (int m = 0; m < 3; ++m) {
    for (int d = 0; d < 3; ++d) Lh.box[m][d] = P.box[m][d];
    Lh.boff[m] = P.boff[m];
  }
  Lh.boff[3] = P.boff[3];
  Lh.box_total = P.box_total;
  Lh.nsub = P.nsub;
  for (int sb = 0; sb < 3; ++sb) Lh.sub_comp[sb] = P.sub_comp[sb];
  if (!P.sc_nk.empty()) {
    if (P.deferred) {   // filled by the device numeric setup below
      const size_t ni = (size_t)(P.sp.p - 1) * (P.sp.p - 1) * (P.sp.p - 1), nc = P.sc_nk.size();
      Lh.sc_dinv = F.alloc<double>(nc * ni);
      Lh.sc_c = P.cartesian ? F.alloc<double>(nc * 6 * ni) : nullptr;
      Lh.sc_w = P.cartesian ? nullptr : F.alloc<double>(nc * 3 * ni);
    } else {
      Lh.sc_dinv = F.upload(P.sc_dinv);
      Lh.sc_c = P.sc_c.empty() ? nullptr : F.upload(P.sc_c);
      Lh.sc_w = P.sc_w.empty() ? nullptr : F.upload(P.sc_w);
    }
    for (size_t i = 0; i < 16 && i < P.sc_kd.size(); ++i) { Lh.sc_kd[i] = P.sc_kd[i]; Lh.sc_k0[i] = P.sc_k0[i]; Lh.sc_kp[i] = P.sc_kp[i]; }
    Lh.sc_nk = F.upload(P.sc_nk);
    Lh.sc_fb = F.upload(std::vector<double>(P.sc_nk.size() * 6 * (size_t)(P.sp.p - 1) * (P.sp.p - 1), 0.0));
    Lh.sc_p = P.sp.p;
    Lh.sc_pre = P.sc_pre ? 1 : 0;
    for (int d = 0; d < 3; ++d) Lh.sc_n[d] = P.sp.n[d];
  }
  {
    rm::PadLayout& pl = Lh.pad;
    std::memset(&pl, 0, sizeof pl);
    pl.ncomp = P.sp.ncomp;
    long long o = 0, po2 = 0;
    for (int m = 0; m < pl.ncomp; ++m) {
      for (int d = 0; d < 3; ++d) pl.len[m][d] = P.sp.len(m, d);
      pl.lxp[m] = pl.len[m][0] + (pl.len[m][0] & 1);
      pl.off[m] = o; pl.poff[m] = po2;
      o += pl.len[m][0] * pl.len[m][1] * pl.len[m][2];
      po2 += pl.lxp[m] * pl.len[m][1] * pl.len[m][2];
    }
    for (int m = pl.ncomp; m <= 3; ++m) { pl.off[m] = o; pl.poff[m] = po2; }
    Lh.npad = po2;
    if (share) {   // orientation families run back to back on ONE padded r / c pair (add_precond)
      if (share->launch.npad != po2) throw RmError(RM_EINVAL, "orientation families: padded layouts differ");
      if (!P.sc_nk.empty() || share->launch.sc_dinv)
        throw RmError(RM_EINVAL, "static-condensation families modify rpad and cannot share it");
      Lh.rpad = share->launch.rpad; Lh.cpad = share->launch.cpad;
    } else {
      void *a = nullptr, *b = nullptr;
      if (cudaMalloc(&a, po2 * sizeof(double)) != cudaSuccess || cudaMalloc(&b, po2 * sizeof(double)) != cudaSuccess)
        throw RmError(RM_ENOMEM, "cudaMalloc failed (padded r / c)");
      F.allocs.push_back(a); F.allocs.push_back(b);
      Lh.rpad = static_cast<double*>(a); Lh.cpad = static_cast<double*>(b);
      // the pad column of rpad stays zero when the apply writes the residual there directly
      CK(cudaMemset(Lh.rpad, 0, po2 * sizeof(double)));
    }
  }
  Lh.npatch = (int)np;
  // tile warps joining the ICC solve (measured slower: more ring walkers), opt-in experiment
  Lh.icc_only = rm::exp_env("RM_ICC_ONLY") ? 1 : 0;
  for (const auto& C : P.classes)
    if (C.final_kind != rm::FINAL_ICC || !C.sc) Lh.icc_only = 0;
  Lh.cs.ncolors = P.ncolors;
  for (int c = 0; c <= P.ncolors; ++c) Lh.cs.start[c] = F.color_start[c];
  Lh.done = F.upload(std::vector<unsigned>(1, 0u));
  Lh.n_max = n_max; Lh.piv_max = piv_max; Lh.mem_max = mem_max; Lh.aux_max = aux_max;
  Lh.unit_bytes_max = unit_max;
  Lh.unit_bytes_max_a = unit_max_a;
  Lh.unit_bytes_max_b = unit_max_b;
  if (np > 0) {
    cudaError_t e = rm::plan_patch_solve(Lh);
    if (e != cudaSuccess)
      throw RmError(RM_EINVAL, "patch too large for the shared-memory patch kernel (fixed " +
                                   std::to_string(Lh.smem_fixed) + " bytes): " + cudaGetErrorString(e));
  }
  // HBM layout of the value blocks: CTA b of the persistent grid takes patches b, b + grid, ...
  // (colour-sorted); distinct blocks are placed in that consumption order so that every CTA
  // streams one contiguous region (scattered blocks cost ~35% of the stream rate: TLB reach).
  {
    const int G = std::max(1, Lh.grid);
    std::unordered_map<long long, long long> remap;
    remap.reserve(2 * P.nfactors + 16);
    std::vector<long long> pvn(np);
    void* dv = nullptr;
    const int64_t nvalues = P.deferred ? P.nvalues : (int64_t)P.values.size();
    if (nvalues > 0) {
      if (cudaMalloc(&dv, nvalues * sizeof(double)) != cudaSuccess) throw RmError(RM_ENOMEM, "cudaMalloc failed (patch factors)");
      F.allocs.push_back(dv);
    }
    double* dvals = static_cast<double*>(dv);
    std::vector<std::pair<long long, long long>> blocks_nv;   // distinct blocks: host offset, doubles
    std::vector<double> stage;
    const size_t chunk = (size_t)32 << 20;   // doubles per staging flush (256 MB)
    long long cur = 0, flushed = 0;
    auto flush = [&]() {
      if (stage.empty()) return;
      CK(cudaMemcpy(dvals + flushed, stage.data(), stage.size() * sizeof(double), cudaMemcpyHostToDevice));
      flushed += (long long)stage.size();
      stage.clear();
    };
    for (int b = 0; b < G; ++b)
      for (size_t q = (size_t)b; q < np; q += (size_t)G) {
        // an empty block (fully condensed patch) shares its offset with the next block: never a key
        if (P.classes[pc[q]].nvals == 0) { pvn[q] = 0; continue; }
        auto it = remap.find(pv[q]);
        if (it == remap.end()) {
          const long long nv = P.classes[pc[q]].nvals;
          it = remap.emplace(pv[q], cur).first;
          blocks_nv.push_back({pv[q], nv});
          if (!P.deferred) stage.insert(stage.end(), P.values.begin() + pv[q], P.values.begin() + pv[q] + nv);
          cur += nv;
          if (stage.size() >= chunk) flush();
        }
        pvn[q] = it->second;
      }
    flush();
    Lh.pvals = F.upload(pvn);
    Lh.vals = dvals;
    std::vector<double> hcopy;   // host copy of device-computed blocks at host offsets (batch planning)
    const double* hvals = P.values.data();
    if (P.deferred) {
      // device-resident numeric setup: every distinct block computed on the GPU at its device offset
      std::vector<long long> fdst(P.foff.size(), 0);
      for (size_t f = 0; f < P.foff.size(); ++f) {
        auto it = remap.find(P.foff[f]);
        fdst[f] = it == remap.end() ? 0 : it->second;
      }
      double sg = 0.0;
      const auto t0 = std::chrono::steady_clock::now();
      try {
        rm::device_numeric_setup(P, fdst, dvals, const_cast<double*>(Lh.sc_dinv), const_cast<double*>(Lh.sc_c), const_cast<double*>(Lh.sc_w),
                                 nullptr, &sg);
      } catch (const rm::NumericError& e) {
        throw RmError(RM_ENUMERIC, e.what());
      } catch (const std::runtime_error& e) {
        throw RmError(RM_ECUDA, e.what());
      }
      F.sigma_max = sg;
      F.numeric_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (remap.size() * 4 <= np) {   // few shared blocks: the class-batched plan reads them on the host
        hcopy.assign(P.nvalues, 0.0);
        for (const auto& b : blocks_nv)
          CK(cudaMemcpy(hcopy.data() + b.first, dvals + remap[b.first], b.second * sizeof(double), cudaMemcpyDeviceToHost));
        hvals = hcopy.data();
      }
    }
    plan_batches(F, P, pc, pv, pvn, remap.size(), hvals);
    // per-CTA producer issue lists in consumption order (patch_solve.cu): sparse channel
    // fwd(0), then per i: fwd(i+1), final(i) unless dense tiles, bwd(i); tile channel tiles(i)
    std::vector<unsigned char*> dmeta(P.classes.size());
    for (size_t c = 0; c < P.classes.size(); ++c) dmeta[c] = const_cast<unsigned char*>(hc[c].meta);
    std::vector<rm::XferEntry> xl;
    std::vector<long long> xb;
    xl.reserve(np * 32);
    auto push = [&](size_t q, int u0, int u1) {
      const rm::ClassProgram& C = P.classes[pc[q]];
      for (int u = u0; u < u1; ++u) {
        const rm::Unit& U = C.units[u];
        rm::XferEntry e{};
        e.meta = dmeta[pc[q]] + U.mofs;
        e.vals = dvals + pvn[q] + U.sofs;
        e.mb_np = (unsigned)U.mbytes | ((unsigned)U.np << 16);
        e.vb = (unsigned)U.nd * 8u;
        xl.push_back(e);
      }
    };
    auto fin_tiles = [&](size_t q) { const rm::ClassProgram& C = P.classes[pc[q]]; return C.final_kind == rm::FINAL_DENSE_INV && C.m > 0; };
    for (int b = 0; b < G; ++b) {
      std::vector<size_t> qs;
      for (size_t q = (size_t)b; q < np; q += (size_t)G) qs.push_back(q);
      const int n = (int)qs.size();
      xb.push_back((long long)xl.size());
      if (Lh.nbox >= 2) {   // pipelined consumption order: fwd(0), then per i: fwd(i+1), [final(i)], bwd(i)
        if (n > 0) push(qs[0], 0, P.classes[pc[qs[0]]].uf0);
        for (int i = 0; i < n; ++i) {
          if (i + 1 < n) push(qs[i + 1], 0, P.classes[pc[qs[i + 1]]].uf0);
          const rm::ClassProgram& C = P.classes[pc[qs[i]]];
          if (!fin_tiles(qs[i])) push(qs[i], C.uf0, C.uf1);
          push(qs[i], C.uf1, (int)C.units.size());
        }
      } else {              // one box buffer: per i: fwd(i), [final(i)], bwd(i)
        for (int i = 0; i < n; ++i) {
          const rm::ClassProgram& C = P.classes[pc[qs[i]]];
          push(qs[i], 0, C.uf0);
          if (!fin_tiles(qs[i])) push(qs[i], C.uf0, C.uf1);
          push(qs[i], C.uf1, (int)C.units.size());
        }
      }
      xb.push_back((long long)xl.size());
      for (int i = 0; i < n; ++i)
        if (fin_tiles(qs[i])) push(qs[i], P.classes[pc[qs[i]]].uf0, P.classes[pc[qs[i]]].uf1);
    }
    xb.push_back((long long)xl.size());
    Lh.xfer = F.upload(xl);
    Lh.xbeg = F.upload(xb);
  }
  F.npatch = (int64_t)np;
  F.nfactors = P.nfactors;
  F.nclasses = (int64_t)P.classes.size();
  F.sweep_value_bytes = bytes;
  F.nnzL = P.nnzL_total;
  F.unique_bytes = P.unique_value_bytes;
  F.ncolors = P.ncolors;
  if (!P.deferred) F.sigma_max = P.sigma_max;
  F.present = true;
}

}  // namespace

struct rm_ctx {
  int k = 0, p = 1, n[3] = {1, 1, 1};
  uint32_t gamma = 0;
  int decomposition = RM_PAFW;
  bool cartesian = true;
  bool setup_device = false;   // numeric setup ran on the GPU (options.setup)
  double setup_family_s = 0.0;  // host build_patch_family (symbolic; + numeric with RM_SETUP_HOST)
  rm::Space sp, spot;
  int64_t ndof = 0, npot = 0, nfree = 0;
  cudaStream_t st = nullptr;
  int device = 0;
  rm::OpParams op{};
  std::vector<void*> allocs;
  double *d_alpha = nullptr, *d_beta = nullptr, *d_hpow = nullptr;
  double *d_X = nullptr, *d_tabs = nullptr;   // trilinear cells: vertices, 1D tables
  double* d_cellbuf = nullptr;                 // trilinear apply: per-cell local results
  rm::TriParams tri{};
  int coef_const = 0;
  // patch families: one per star orientation for edge / face stars (tighter window boxes), one
  // for vertex stars; prims[0] / pots[0] always exist (possibly empty)
  std::vector<DevFamily> prims = std::vector<DevFamily>(1), pots = std::vector<DevFamily>(1);
  std::vector<double> Dh;   // p x (p+1)
  double *d_r = nullptr, *d_t = nullptr, *d_s = nullptr;
  double *d_z = nullptr, *d_pp = nullptr, *d_q = nullptr, *d_pr = nullptr;
  double *d_sc = nullptr, *d_part = nullptr;
  double *d_hf = nullptr, *d_hu = nullptr;
  std::vector<uint8_t> mask;
  double setup_seconds = 0.0;
  // phase timing (rm_timing_enable / rm_timing_read)
  bool timing = false;
  struct Ev { int phase; cudaEvent_t a, b; };
  std::vector<Ev> events;
  int64_t launches[RM_NPHASE] = {};
  // z-slab partition (nranks > 1)
  int rank = 0, nranks = 1;
  rm_partition_info part{};
  ncclComm_t comm = nullptr;
  double *d_c = nullptr, *d_rtmp = nullptr;
  int64_t nfree_global = 0;
  // p = 1 coarse level + hybrid V(1,1) (options.coarse, reading G20)
  std::unique_ptr<rm::CoarseFactor> coarse;
  rm::CoarseLaunch cl{};
  double *d_vz = nullptr, *d_vt = nullptr;   // cycle temporaries (fine size)
  // SC-PH (sc_ph.cu): layout, cell-interior blocks, temporaries y = A_II^-1 r_I, w, R_G r, c_G, z
  rm::ScPhParams scph{};
  int* d_scph_set = nullptr;
  int* d_scph_mem = nullptr;
  double *d_scph_K = nullptr, *d_scph_M = nullptr;
  double *d_sy = nullptr, *d_sw = nullptr, *d_srg = nullptr, *d_scg = nullptr, *d_sz = nullptr;
  double smoother_omega = 1.0;

  double* dalloc(size_t n) {
    void* d = nullptr;
    if (cudaMalloc(&d, std::max<size_t>(n, 1) * sizeof(double)) != cudaSuccess) throw RmError(RM_ENOMEM, "cudaMalloc failed");
    allocs.push_back(d);
    return static_cast<double*>(d);
  }
  // rm_relax_host on the SC-fused path: f is copied on a second stream while the apply runs
  cudaStream_t st_copy = nullptr;
  cudaEvent_t ev_u = nullptr, ev_f = nullptr;
  ~rm_ctx() {
    if (ev_u) cudaEventDestroy(ev_u);
    if (ev_f) cudaEventDestroy(ev_f);
    if (st_copy) cudaStreamDestroy(st_copy);
    if (comm) { try { if (nccl().destroy) nccl().destroy(comm); } catch (...) {} }
    for (auto& e : events) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    for (void* p : allocs) cudaFree(p);
    for (auto& F : prims) F.release();
    for (auto& F : pots) F.release();
  }
};

namespace {

rm::OpParams make_op(const rm::Space& sp, uint32_t gamma) {
  rm::CellOperator co = rm::build_cell_operator(sp.k, sp.p);
  rm::OpParams op;
  std::memset(&op, 0, sizeof op);
  op.k = sp.k; op.p = sp.p; op.ncomp = sp.ncomp;
  for (int d = 0; d < 3; ++d) op.n[d] = sp.n[d];
  for (int m = 0; m < 3; ++m)
    for (int d = 0; d < 3; ++d) {
      op.fam[m][d] = sp.fam[m][d];
      op.len[m][d] = m < sp.ncomp ? sp.len(m, d) : 0;
    }
  for (int m = 0; m <= 3; ++m) op.off[m] = sp.offset(std::min(m, sp.ncomp));
  op.gamma_d = gamma;
  if ((int)co.terms.size() > RM_MAXTERMS || (int)co.mats.size() > RM_MAXMATS)
    throw RmError(RM_EINVAL, "operator term table overflow");
  op.nterms = (int)co.terms.size();
  op.nmats = (int)co.mats.size();
  for (int t = 0; t < op.nterms; ++t) {
    const rm::Term& T = co.terms[t];
    op.terms[t].mout = T.mout; op.terms[t].min = T.min; op.terms[t].coef = T.coef; op.terms[t].c = T.c;
    for (int d = 0; d < 3; ++d) { op.terms[t].hexp[d] = T.hexp[d]; op.terms[t].mat[d] = T.mat[d]; }
  }
  for (int m = 0; m < op.nmats; ++m) {
    const rm::Mat1& M = co.mats[m];
    if (M.rows > RM_MAXP1) throw RmError(RM_EINVAL, "p too large");
    int nz = 0;
    for (int i = 0; i < M.rows; ++i) {
      op.rowptr[m][i] = (short)nz;
      for (int j = 0; j < M.cols; ++j)
        if (M(i, j) != 0.0) {
          if (nz >= RM_MAXMATNZ) throw RmError(RM_EINVAL, "1D matrix too dense");
          op.col[m][nz] = (unsigned char)j; op.val[m][nz] = M(i, j); ++nz;
        }
    }
    op.rowptr[m][M.rows] = (short)nz;
  }
  {   // B-hat and D-hat with their structural zeros exact (reading G18), for the line kernels
    const rm::Basis1D& b = rm::basis(sp.p);
    const int n = sp.p + 1;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        const bool pat = (i == j) || ((i == 0 || i == sp.p) && (j == 0 || j == sp.p));
        op.Bh[i * n + j] = pat ? b.B[i * n + j] : 0.0;
      }
    for (int i = 0; i < sp.p; ++i)
      for (int j = 0; j < n; ++j) op.Dh[i * n + j] = (j == 0 || j == sp.p || j == i) ? b.D[i * n + j] : 0.0;
  }
  if (sp.k == 0) {   // x-stiffness term: X = A-hat, Y = Z = B-hat
    for (int t = 0; t < op.nterms; ++t) {
      const rm::Term& T = co.terms[t];
      if (T.coef == 0 && T.mat[0] != T.mat[1]) {
        const rm::Mat1 &A = co.mats[T.mat[0]], &B = co.mats[T.mat[1]];
        for (size_t i = 0; i < A.v.size(); ++i) { op.Ah[i] = A.v[i]; op.Bh[i] = B.v[i]; }
        break;
      }
    }
  }
  return op;
}

void check_cuda_status() { CK(cudaGetLastError()); }

rm_status fail(const RmError& e) { g_err = e.what(); return e.st; }

}  // namespace

// SC-PH cell-interior blocks (remark P:1061-1066: <= 3x3 on Cartesian cells): from the cell
// operator's entries, per distinct cell size (hx, hy, hz); members as cell-local codes
void setup_scph(rm_ctx* c, const std::vector<double>* h) {
  const rm::Space& sp = c->sp;
  const int p = c->p;
  rm::ScPhParams& P = c->scph;
  std::memset(&P, 0, sizeof P);
  P.p = p; P.ncomp = sp.ncomp;
  for (int d = 0; d < 3; ++d) P.n[d] = c->n[d];
  for (int m = 0; m < sp.ncomp; ++m) {
    for (int d = 0; d < 3; ++d) { P.fam[m][d] = sp.fam[m][d] == rm::FAM_P ? 0 : 1; P.len[m][d] = sp.len(m, d); }
    P.off[m] = sp.offset(m);
  }
  for (int m = sp.ncomp; m <= 3; ++m) P.off[m] = sp.ndof();
  // cell-local DoFs (component-major, z, y, x), interior flags and codes
  std::vector<int> code, interior;
  for (int m = 0; m < sp.ncomp; ++m)
    for (int cc = 0; cc < sp.lsize(m, 2); ++cc)
      for (int b = 0; b < sp.lsize(m, 1); ++b)
        for (int a = 0; a < sp.lsize(m, 0); ++a) {
          const int idx[3] = {a, b, cc};
          bool in = true;
          for (int d = 0; d < 3; ++d)
            if (sp.fam[m][d] == rm::FAM_P && (idx[d] == 0 || idx[d] == p)) in = false;
          code.push_back(m << 24 | cc << 16 | b << 8 | a);
          interior.push_back(in);
        }
  const rm::CellOperator op = rm::build_cell_operator(c->k, p);
  std::map<std::tuple<double, double, double>, int> sets;
  std::vector<int> cset((size_t)c->n[0] * c->n[1] * c->n[2]);
  std::vector<rm::CellEntries> ents;
  for (size_t K = 0; K < cset.size(); ++K) {
    const int cx = (int)(K % c->n[0]), cy = (int)((K / c->n[0]) % c->n[1]), cz = (int)(K / ((size_t)c->n[0] * c->n[1]));
    auto key = std::make_tuple(h[0][cx], h[1][cy], h[2][cz]);
    auto it = sets.find(key);
    if (it == sets.end()) {
      it = sets.emplace(key, (int)ents.size()).first;
      ents.push_back(rm::cartesian_cell_entries(op, sp, h[0][cx], h[1][cy], h[2][cz]));
    }
    cset[K] = it->second;
  }
  // blocks = connected components of the interior-interior pattern (the same for every set)
  const int nl = (int)code.size();
  std::vector<int> parent(nl);
  for (int i = 0; i < nl; ++i) parent[i] = i;
  std::function<int(int)> root = [&](int i) { return parent[i] == i ? i : parent[i] = root(parent[i]); };
  const rm::CellEntries& E0 = ents[0];
  for (size_t t = 0; t < E0.row.size(); ++t)
    if (interior[E0.row[t]] && interior[E0.col[t]]) parent[root(E0.row[t])] = root(E0.col[t]);
  std::map<int, std::vector<int>> comps;
  for (int i = 0; i < nl; ++i) if (interior[i]) comps[root(i)].push_back(i);
  std::vector<int> mem;
  std::vector<std::vector<int>> blocks;
  for (auto& kv : comps) {
    if (kv.second.size() > 3) throw RmError(RM_EINVAL, "SC-PH: cell-interior block larger than 3x3");
    blocks.push_back(kv.second);
    for (int j = 0; j < 3; ++j) mem.push_back(j < (int)kv.second.size() ? code[kv.second[j]] : -1);
  }
  P.nblk = (int)blocks.size();
  std::vector<double> bk((size_t)ents.size() * P.nblk * 6, 0.0), bm(bk.size(), 0.0);
  for (size_t s = 0; s < ents.size(); ++s) {
    std::map<std::pair<int, int>, std::pair<double, double>> at;
    for (size_t t = 0; t < ents[s].row.size(); ++t) at[{ents[s].row[t], ents[s].col[t]}] = {ents[s].kval[t], ents[s].mval[t]};
    for (int b = 0; b < P.nblk; ++b)
      for (int i = 0, q = 0; i < 3; ++i)
        for (int j = 0; j <= i; ++j, ++q) {
          if (i >= (int)blocks[b].size() || j >= (int)blocks[b].size()) continue;
          auto it = at.find({blocks[b][i], blocks[b][j]});
          if (it == at.end()) continue;
          bk[(s * P.nblk + b) * 6 + q] = it->second.first;
          bm[(s * P.nblk + b) * 6 + q] = it->second.second;
        }
  }
  auto upi = [&](const std::vector<int>& v) {
    int* d = nullptr;
    CK(cudaMalloc(&d, std::max<size_t>(v.size(), 1) * sizeof(int)));
    c->allocs.push_back(d);
    if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice));
    return d;
  };
  auto upd = [&](const std::vector<double>& v) {
    double* d = c->dalloc(std::max<size_t>(v.size(), 1));
    if (!v.empty()) CK(cudaMemcpy(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
    return d;
  };
  c->d_scph_set = upi(cset);
  c->d_scph_mem = upi(mem);
  c->d_scph_K = upd(bk);
  c->d_scph_M = upd(bm);
  c->d_sy = c->dalloc(c->ndof); c->d_sw = c->dalloc(c->ndof); c->d_srg = c->dalloc(c->ndof);
  c->d_scg = c->dalloc(c->ndof); c->d_sz = c->dalloc(c->ndof);
}

extern "C" {

void rm_default_options(rm_options* o) {
  std::memset(o, 0, sizeof *o);
  o->decomposition = RM_PAFW;
  o->factorization = RM_CHOL;
  o->patch_entities = RM_ALL_ENTITIES;
  o->potential_shift = 1e-3;   // reading G8: roundoff of the sweep grows like eps/eps_s
  o->nranks = 1;
  o->setup = RM_SETUP_DEVICE;
}

const char* rm_last_error(void) { return g_err.c_str(); }

rm_status rm_partition(const rm_mesh* mesh, int32_t p, rm_space space, uint32_t gamma_d, int32_t rank, int32_t nranks,
                       rm_partition_info* info) {
  try {
    if (!mesh || !info) throw RmError(RM_EINVAL, "null argument");
    if (p < 1 || p > 15) throw RmError(RM_EINVAL, "p must be in 1..15");
    compute_partition(*mesh, p, space, gamma_d, rank, nranks, *info);
    return RM_OK;
  } catch (const RmError& e) {
    return fail(e);
  }
}

rm_status rm_nccl_check(int32_t device) {
  // one-rank communicator on `device`: grouped send/recv to self and an in-place allreduce on a
  // stream, results checked on the host (the transport calls rm_relax uses with nranks > 1)
  try {
    CK(cudaSetDevice(device));
    const NcclApi& N = nccl();
    ncclUniqueId id;
    NK(N.get_id(&id));
    ncclComm_t comm = nullptr;
    NK(N.init(&comm, 1, id, 0));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    const int n = 4096;
    std::vector<double> h(n), back(n);
    for (int i = 0; i < n; ++i) h[i] = 0.5 * i - 7.0;
    double *a = nullptr, *b = nullptr;
    CK(cudaMalloc(&a, n * sizeof(double)));
    CK(cudaMalloc(&b, n * sizeof(double)));
    CK(cudaMemcpy(a, h.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemset(b, 0, n * sizeof(double)));
    NK(N.gstart());
    NK(N.send(a, n, ncclDouble, 0, comm, st));
    NK(N.recv(b, n, ncclDouble, 0, comm, st));
    NK(N.gend());
    NK(N.allreduce(b, b, n, ncclDouble, ncclSum, comm, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(back.data(), b, n * sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(a); cudaFree(b); cudaStreamDestroy(st);
    if (N.destroy) N.destroy(comm);
    for (int i = 0; i < n; ++i)
      if (back[i] != h[i]) throw RmError(RM_ENCCL, "NCCL self send/recv returned wrong data");
    return RM_OK;
  } catch (const RmError& e) {
    return fail(e);
  }
}

rm_status rm_nccl_unique_id(void* id128) {
  try {
    if (!id128) throw RmError(RM_EINVAL, "null argument");
    ncclUniqueId id;
    NK(nccl().get_id(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(id128, &id, sizeof id);
    return RM_OK;
  } catch (const RmError& e) {
    return fail(e);
  }
}

rm_status rm_setup(rm_ctx** out, const rm_mesh* mesh, int32_t p, rm_space space, const double* alpha,
                   int64_t n_alpha, const double* beta, int64_t n_beta, uint32_t gamma_d, const rm_options* opt) {
  auto t0 = std::chrono::steady_clock::now();
  try {
    if (!out || !mesh || !alpha || !beta) throw RmError(RM_EINVAL, "null argument");
    // host setup threads (OpenMP); launchers that pin OMP_NUM_THREADS=1 per rank can override
    if (const char* e = getenv("RM_SETUP_THREADS")) omp_set_num_threads(std::max(1, atoi(e)));
    *out = nullptr;
    rm_options o;
    if (opt) o = *opt; else rm_default_options(&o);
    if (p < 1 || p > 15) throw RmError(RM_EINVAL, "p must be in 1..15");
    if (space < 0 || space > 2) throw RmError(RM_EINVAL, "space must be 0, 1 or 2");
    if (mesh->nx < 1 || mesh->ny < 1 || mesh->nz < 1) throw RmError(RM_EINVAL, "mesh sizes must be >= 1");
    if (gamma_d > 0x3F) throw RmError(RM_EINVAL, "gamma_d has bits above bit 5");
    if (o.coarse != 0 && o.coarse != 1) throw RmError(RM_EINVAL, "coarse must be 0 or 1");
    if (o.coarse && o.nranks > 1) throw RmError(RM_EINVAL, "the coarse level is single-rank only");
    if (o.decomposition != RM_PAFW && o.decomposition != RM_PH && o.decomposition != RM_SC_PAFW &&
        o.decomposition != RM_SC_PH)
      throw RmError(RM_EINVAL, "bad decomposition");
    if (o.decomposition == RM_SC_PAFW && space != 0)
      throw RmError(RM_EINVAL, "SC-PAFW is the H(grad) decomposition (k = 1, 2: SC-PH)");
    if (o.decomposition == RM_SC_PH && (space == 0 || o.nranks > 1 || o.coarse))
      throw RmError(RM_EINVAL, "SC-PH: k = 1, 2, single rank, one level");
    if (o.decomposition == RM_SC_PAFW && o.nranks > 1)
      throw RmError(RM_EINVAL, "SC-PAFW is single-rank only");
    if (o.factorization != RM_CHOL && o.factorization != RM_ICC_SC) throw RmError(RM_EINVAL, "bad factorization");
    const int64_t ncell = (int64_t)mesh->nx * mesh->ny * mesh->nz;
    if (!(n_alpha == 1 || n_alpha == ncell) || !(n_beta == 1 || n_beta == ncell))
      throw RmError(RM_EINVAL, "alpha/beta must have 1 or ncells entries");
    for (int64_t i = 0; i < n_alpha; ++i) if (!(alpha[i] > 0)) throw RmError(RM_EINVAL, "alpha must be > 0");
    for (int64_t i = 0; i < n_beta; ++i) if (!(beta[i] >= 0)) throw RmError(RM_EINVAL, "beta must be >= 0");
    // z-slab partition: the rest of the setup runs on the LOCAL mesh (slab + ghost layer below
    // + shared plane above), with the patches of the owned vertex layers only
    rm_partition_info part;
    {
      rm_mesh gm = *mesh;
      if (o.nranks <= 1) { gm.z_begin = 0; gm.z_end = mesh->nz; }
      compute_partition(gm, p, space, gamma_d, o.nranks > 1 ? o.rank : 0, std::max(o.nranks, 1), part);
    }
    const uint32_t gamma_global = gamma_d;
    const int nz_global = mesh->nz;
    rm_mesh lm = *mesh;
    std::vector<double> lcoords;
    if (o.nranks > 1) {
      lm.nz = part.nz_local;
      const size_t vplane = (size_t)(mesh->nx + 1) * (mesh->ny + 1) * 3;
      if (mesh->coords) {
        lm.coords = mesh->coords + (size_t)part.z_cell0 * vplane;
      } else {   // the uniform unit-cube grid, sliced
        lcoords.resize(vplane * (part.nz_local + 1));
        for (int z = 0; z <= part.nz_local; ++z)
          for (int y = 0; y <= mesh->ny; ++y)
            for (int x = 0; x <= mesh->nx; ++x) {
              double* X = &lcoords[((size_t)z * (mesh->ny + 1) + y) * (mesh->nx + 1) * 3 + (size_t)x * 3];
              X[0] = (double)x / mesh->nx; X[1] = (double)y / mesh->ny; X[2] = (double)(part.z_cell0 + z) / nz_global;
            }
        lm.coords = lcoords.data();
      }
      const int64_t cplane = (int64_t)mesh->nx * mesh->ny;
      if (n_alpha > 1) { alpha += part.z_cell0 * cplane; n_alpha = cplane * part.nz_local; }
      if (n_beta > 1) { beta += part.z_cell0 * cplane; n_beta = cplane * part.nz_local; }
      gamma_d = part.gamma_local;
      mesh = &lm;
    }
    CK(cudaSetDevice(o.device));
    std::unique_ptr<rm_ctx> c(new rm_ctx);
    c->rank = o.nranks > 1 ? o.rank : 0;
    c->nranks = std::max(o.nranks, 1);
    c->part = part;
    c->k = space; c->p = p; c->n[0] = mesh->nx; c->n[1] = mesh->ny; c->n[2] = mesh->nz;
    c->gamma = gamma_d;
    c->decomposition = (space == 0) ? (o.decomposition == RM_SC_PAFW ? RM_SC_PAFW : RM_PAFW) : o.decomposition;
    c->st = static_cast<cudaStream_t>(o.stream);
    c->device = o.device;
    c->sp.init(space, p, mesh->nx, mesh->ny, mesh->nz);
    c->ndof = c->sp.ndof();
    // geometry: detect an axis-aligned grid
    std::vector<double> h[3];
    bool cart = true;
    for (int d = 0; d < 3; ++d) h[d].assign(c->n[d], 1.0 / c->n[d]);
    if (mesh->coords) {
      const double* X = mesh->coords;
      auto at = [&](int z, int y, int x, int i) { return X[(((int64_t)z * (c->n[1] + 1) + y) * (c->n[0] + 1) + x) * 3 + i]; };
      for (int z = 0; z <= c->n[2] && cart; ++z)
        for (int y = 0; y <= c->n[1] && cart; ++y)
          for (int x = 0; x <= c->n[0] && cart; ++x) {
            if (at(z, y, x, 0) != at(0, 0, x, 0) || at(z, y, x, 1) != at(0, y, 0, 1) || at(z, y, x, 2) != at(z, 0, 0, 2)) cart = false;
          }
      if (cart) {
        for (int x = 0; x < c->n[0]; ++x) h[0][x] = at(0, 0, x + 1, 0) - at(0, 0, x, 0);
        for (int y = 0; y < c->n[1]; ++y) h[1][y] = at(0, y + 1, 0, 1) - at(0, y, 0, 1);
        for (int z = 0; z < c->n[2]; ++z) h[2][z] = at(z + 1, 0, 0, 2) - at(z, 0, 0, 2);
        for (int d = 0; d < 3; ++d)
          for (double v : h[d]) if (!(v > 0)) throw RmError(RM_EINVAL, "non-positive cell size");
      }
    }
    c->cartesian = cart;
    if (!cart) {
      // trilinear cells (H(grad) only): vertex array and the 1D tables at the n_q GLL points
      if (space != 0) throw RmError(RM_EINVAL, "trilinear (non-axis-aligned) meshes are supported for H(grad) only");
      const int nq = (3 * (p + 1) + 1) / 2;   // reading G1
      if (nq > 24) throw RmError(RM_EINVAL, "trilinear apply: p too large");
      const rm::Basis1D& b1 = rm::basis(p);
      std::vector<double> xq, wq, sv, dsv;
      rm::gll_rule(nq, xq, wq);
      b1.tab_s(xq, sv, dsv);
      std::vector<double> tabs;
      tabs.insert(tabs.end(), sv.begin(), sv.end());
      tabs.insert(tabs.end(), dsv.begin(), dsv.end());
      tabs.insert(tabs.end(), xq.begin(), xq.end());
      tabs.insert(tabs.end(), wq.begin(), wq.end());
      // even / odd tables of the x contractions (TriParams): needs mirror point pairs (nq even)
      // and definite parity of every interior FDM basis function at the quadrature points
      c->tri.eo = 0;
      if (nq % 2 == 0) {
        const int P1 = p + 1, ne = nq / 2;
        std::vector<int> ev, od;
        bool ok = true;
        for (int j = 1; j < p && ok; ++j) {
          double se = 0, so = 0, mx = 0;
          for (int q = 0; q < nq; ++q) {
            const double a = sv[q * P1 + j], b = sv[(nq - 1 - q) * P1 + j];
            se = std::max(se, std::fabs(a - b)); so = std::max(so, std::fabs(a + b)); mx = std::max(mx, std::fabs(a));
          }
          if (se <= 1e-12 * mx) ev.push_back(j);
          else if (so <= 1e-12 * mx) od.push_back(j);
          else ok = false;
        }
        if (ok && ev.size() <= 7 && od.size() <= 7) {
          for (int k = 0; k < 16; ++k) c->tri.xsig[k] = -1;
          c->tri.xsig[0] = 0; c->tri.xsig[8] = p;   // E_0 / O_0 (the vertex pair, butterflied)
          for (size_t i = 0; i < ev.size(); ++i) c->tri.xsig[1 + i] = ev[i];
          for (size_t i = 0; i < od.size(); ++i) c->tri.xsig[9 + i] = od[i];
          std::vector<double> T(4 * 12 * 8, 0.0);   // S_E, S_O, D_E, D_O [r][e]
          for (int r = 0; r < ne; ++r)
            for (int e = 0; e < 8; ++e) {
              const int je = c->tri.xsig[e], jo = c->tri.xsig[8 + e];
              double sE = 0, sO = 0, dE = 0, dO = 0;
              if (e == 0) {
                sE = sv[r * P1] + sv[r * P1 + p]; dE = dsv[r * P1] + dsv[r * P1 + p];
                sO = sv[r * P1] - sv[r * P1 + p]; dO = dsv[r * P1] - dsv[r * P1 + p];
              } else {
                if (je >= 0) { sE = sv[r * P1 + je]; dE = dsv[r * P1 + je]; }
                if (jo >= 0) { sO = sv[r * P1 + jo]; dO = dsv[r * P1 + jo]; }
              }
              T[0 * 96 + r * 8 + e] = sE; T[1 * 96 + r * 8 + e] = sO;
              T[2 * 96 + r * 8 + e] = dE; T[3 * 96 + r * 8 + e] = dO;
            }
          tabs.insert(tabs.end(), T.begin(), T.end());
          c->tri.eo = 1;
          c->tri.ne = ne;
        }
      }
      c->d_tabs = c->dalloc(tabs.size());
      CK(cudaMemcpy(c->d_tabs, tabs.data(), tabs.size() * 8, cudaMemcpyHostToDevice));
      const size_t nv = (size_t)(c->n[0] + 1) * (c->n[1] + 1) * (c->n[2] + 1) * 3;
      c->d_X = c->dalloc(nv);
      CK(cudaMemcpy(c->d_X, mesh->coords, nv * 8, cudaMemcpyHostToDevice));
      c->tri.p = p; c->tri.nq = nq;
      for (int d = 0; d < 3; ++d) c->tri.n[d] = c->n[d];
      c->tri.Lx = c->sp.len(0, 0); c->tri.Ly = c->sp.len(0, 1); c->tri.Lz = c->sp.len(0, 2);
      c->tri.gamma_d = gamma_d;
      c->d_cellbuf = c->dalloc(rm::tri_cellbuf_doubles(c->tri));
    } else {
      // Cartesian: one apply launch over all cells + the skeleton gather.  H(curl) / H(div): the
      // pointwise-stage kernels (apply_kform.cu); H(grad): the line-stage kernel of apply.cu
      // (interior entries final) + the skeleton-only gather (round 2; the 8-colour launches
      // measured 0.34 ms at cfg2, the k = 0 pointwise kernel, experiment RM_APPLY_PW, 0.48 ms)
      c->d_cellbuf = c->dalloc(rm::kform_cellbuf_doubles(space, p, c->n));
    }
    // ---- device operator
    c->op = make_op(c->sp, gamma_d);
    c->coef_const = (n_alpha == 1 && n_beta == 1);
    {
      std::vector<double> hp;
      for (int d = 0; d < 3; ++d)
        for (int e = -3; e <= 3; ++e)
          for (int i = 0; i < c->n[d]; ++i) hp.push_back(std::pow(h[d][i], e));
      c->d_hpow = c->dalloc(hp.size());
      CK(cudaMemcpy(c->d_hpow, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice));
      std::vector<double> a(alpha, alpha + n_alpha), b(beta, beta + n_beta);
      if (!c->coef_const) {   // expand to per-cell
        if (n_alpha == 1) a.assign(ncell, alpha[0]);
        if (n_beta == 1) b.assign(ncell, beta[0]);
      }
      c->d_alpha = c->dalloc(a.size()); c->d_beta = c->dalloc(b.size());
      CK(cudaMemcpy(c->d_alpha, a.data(), a.size() * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->d_beta, b.data(), b.size() * 8, cudaMemcpyHostToDevice));
    }
    // constrained mask / free count
    c->mask.assign(c->ndof, 0);
    {
      int64_t nf = 0;
      for (int m = 0; m < c->sp.ncomp; ++m)
        for (int64_t z = 0; z < c->sp.len(m, 2); ++z)
          for (int64_t y = 0; y < c->sp.len(m, 1); ++y)
            for (int64_t x = 0; x < c->sp.len(m, 0); ++x) {
              bool con = c->sp.constrained(m, x, y, z, gamma_d);
              c->mask[c->sp.gidx(m, z, y, x)] = con;
              nf += !con;
            }
      c->nfree = nf;
    }
    // ---- patch families
    rm::SetupInput in{};
    in.k = space; in.p = p; in.n[0] = mesh->nx; in.n[1] = mesh->ny; in.n[2] = mesh->nz;
    in.gamma_d = gamma_d; in.coords = mesh->coords; in.alpha = alpha; in.beta = beta;
    in.n_alpha = n_alpha; in.n_beta = n_beta;
    const bool scph = c->decomposition == RM_SC_PH;
    in.dim = (c->decomposition == RM_PH || scph) ? space : 0;
    in.sc_decomposition = c->decomposition == RM_SC_PAFW;
    in.interface_only = scph;   // SC-PH: interface corrections S_i^{-1} only (eq:LDU)
    // options.factorization applies to the scalar (H(grad)) patch problems: the primary patches
    // for k = 0, the PH potential vertex stars for k = 1; k-star patches of k = 1, 2
    // are factored exactly (optimal fill)
    in.factorization = space == 0 ? o.factorization : RM_CHOL;
    in.interior_only = o.patch_entities == RM_INTERIOR_ONLY;
    in.cartesian = cart;
    in.hx = h[0].data(); in.hy = h[1].data(); in.hz = h[2].data();
    in.zv_lo = part.v_lo; in.zv_hi = part.v_hi;   // owned vertex layers (all of them on one rank)
    in.defer_numeric = o.setup == RM_SETUP_DEVICE;   // numeric factorization on the GPU (dsetup.cu)
    c->setup_device = in.defer_numeric;
    {
      // edge / face stars: one family per orientation (window boxes ~2-4x smaller than the hull)
      const int no = (in.dim == 1 || in.dim == 2) && !rm::exp_env("RM_ONE_FAMILY") ? 3 : 1;
      c->prims.assign(no, DevFamily{});
      for (int o = 0; o < no; ++o) {
        rm::SetupInput io = in;
        io.orient = no > 1 ? o : -1;
        const auto tb = std::chrono::steady_clock::now();
        auto fam = rm::build_patch_family(io);
        c->setup_family_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tb).count();
        upload_family(c->prims[o], *fam, o > 0 ? &c->prims[0] : nullptr);
      }
    }
    if ((c->decomposition == RM_PH || scph) && space >= 1) {
      // potential problem B = D^T A D (+ eps_s beta M^{k-1} for k = 2): the V^{k-1} operator with
      // (alpha', beta') = (beta, 0) for k = 1 and (beta, eps_s beta) for k = 2 (reading G8)
      std::vector<double> ap(beta, beta + n_beta), bp(n_beta);
      for (int64_t i = 0; i < n_beta; ++i) bp[i] = (space == 2) ? o.potential_shift * beta[i] : 0.0;
      for (double v : ap) if (!(v > 0)) throw RmError(RM_EINVAL, "PH potential needs beta > 0");
      rm::SetupInput ip = in;
      ip.k = space - 1; ip.alpha = ap.data(); ip.beta = bp.data(); ip.n_alpha = n_beta; ip.n_beta = n_beta;
      ip.dim = space - 1;
      ip.factorization = (space == 1 && !scph) ? o.factorization : RM_CHOL;
      ip.interface_only = scph;   // SC-PH: B~_j^{-1} on interface-only input, interface part kept
      const int no = (ip.dim == 1 || ip.dim == 2) && !rm::exp_env("RM_ONE_FAMILY") ? 3 : 1;
      c->pots.assign(no, DevFamily{});
      for (int o = 0; o < no; ++o) {
        rm::SetupInput io = ip;
        io.orient = no > 1 ? o : -1;
        const auto tb = std::chrono::steady_clock::now();
        auto fam = rm::build_patch_family(io);
        c->setup_family_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tb).count();
        upload_family(c->pots[o], *fam, o > 0 ? &c->pots[0] : nullptr);
      }
      c->spot.init(space - 1, p, mesh->nx, mesh->ny, mesh->nz);
      c->npot = c->spot.ndof();
      const rm::Basis1D& b = rm::basis(p);
      c->Dh.assign(p * (p + 1), 0.0);
      for (int i = 0; i < p; ++i)
        for (int j = 0; j <= p; ++j)
          if (j == 0 || j == p || j == i) c->Dh[i * (p + 1) + j] = b.D[i * (p + 1) + j];
      c->d_t = c->dalloc(c->npot); c->d_s = c->dalloc(c->npot);
    }
    if (scph) setup_scph(c.get(), h);
    c->d_r = c->dalloc(c->ndof);
    if (c->nranks > 1) {
      // global free count; buffers of the multi-rank sweep; the communicator (if an id is given)
      const uint32_t g = gamma_global;
      const int ng[3] = {c->n[0], c->n[1], nz_global};
      c->nfree = 0;
      for (int m = 0; m < c->sp.ncomp; ++m) {   // per direction: P family n p + 1 minus Dirichlet ends, DP n p
        int64_t fm = 1;
        for (int d = 0; d < 3; ++d)
          fm *= c->sp.fam[m][d] == rm::FAM_P ? (int64_t)ng[d] * p + 1 - ((g >> (2 * d)) & 1) - ((g >> (2 * d + 1)) & 1)
                                             : (int64_t)ng[d] * p;
        c->nfree += fm;
      }
      c->d_c = c->dalloc(c->ndof);
      // reverse-add receive buffer: p planes of the vector layout or of the padded (even-x) layout
      c->d_rtmp = c->dalloc((size_t)3 * p * ((int64_t)c->n[0] * p + 2) * ((int64_t)c->n[1] * p + 1));
      if (o.nccl_id) {
        ncclUniqueId id;
        std::memcpy(&id, o.nccl_id, sizeof id);
        NK(nccl().init(&c->comm, c->nranks, id, c->rank));
      }
    }
    if (o.coarse) {
      // p = 1 coarse level: A_0 rediscretised, block-tridiagonal Cholesky, R_0 tables
      rm::CoarseSetupInput ci{};
      ci.k = space; ci.p = p; ci.n[0] = c->n[0]; ci.n[1] = c->n[1]; ci.n[2] = c->n[2];
      ci.gamma_d = gamma_d; ci.coords = mesh->coords; ci.cartesian = cart;
      ci.hx = h[0].data(); ci.hy = h[1].data(); ci.hz = h[2].data();
      ci.alpha = alpha; ci.beta = beta; ci.n_alpha = n_alpha; ci.n_beta = n_beta;
      c->coarse.reset(new rm::CoarseFactor);
      rm::build_coarse(ci, *c->coarse);
      const rm::CoarseFactor& F = *c->coarse;
      rm::CoarseLaunch& L = c->cl;
      L.p = p; L.ncomp = c->sp.ncomp;
      for (int d = 0; d < 3; ++d) L.n[d] = c->n[d];
      for (int m = 0; m < 3; ++m)
        for (int d = 0; d < 3; ++d) {
          L.fam[m][d] = c->sp.fam[m][d];
          L.len[m][d] = m < c->sp.ncomp ? c->sp.len(m, d) : 0;
          L.len1[m][d] = m < c->sp.ncomp ? F.sp1.len(m, d) : 0;
        }
      for (int m = 0; m <= 3; ++m) { L.off[m] = c->sp.offset(std::min(m, c->sp.ncomp)); L.off1[m] = F.sp1.offset(std::min(m, c->sp.ncomp)); }
      L.ndof1 = F.ndof1;
      L.nb = (int)F.bstart.size() - 1;
      L.bstart = F.bstart.data();
      L.o_linv = F.o_linv.data(); L.o_linvt = F.o_linvt.data(); L.o_lsub = F.o_lsub.data(); L.o_lsubt = F.o_lsubt.data();
      auto up = [&](const void* h, size_t bytes) {
        void* d = nullptr;
        if (cudaMalloc(&d, std::max<size_t>(bytes, 8)) != cudaSuccess) throw RmError(RM_ENOMEM, "cudaMalloc failed (coarse level)");
        c->allocs.push_back(d);
        CK(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
        return d;
      };
      L.perm = static_cast<const long long*>(up(F.perm.data(), F.perm.size() * sizeof(long long)));
      L.cmask = static_cast<const unsigned char*>(up(F.cmask.data(), F.cmask.size()));
      L.vals = static_cast<const double*>(up(F.vals.data(), F.vals.size() * sizeof(double)));
      L.xc = c->dalloc(F.ndof1); L.b = c->dalloc(F.ndof1); L.y = c->dalloc(F.ndof1); L.t = c->dalloc(F.ndof1);
      L.tA = c->dalloc(c->ndof); L.tB = c->dalloc(c->ndof);
      for (int a = 0; a < 16; ++a) { L.e0[a] = F.e0[a]; L.e1[a] = F.e1[a]; }
      c->d_vz = c->dalloc(c->ndof); c->d_vt = c->dalloc(c->ndof);
      // reading G20: smoother damping 1 / N_c (N_c = patch colours of the level, potential included)
      int nc = c->prims[0].ncolors + (c->pots[0].present ? c->pots[0].ncolors : 0);
      c->smoother_omega = 1.0 / std::max(nc, 1);
    }
    c->d_sc = c->dalloc(8);
    c->d_part = c->dalloc(1024);
    CK(cudaDeviceSynchronize());
    c->setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = c.release();
    return RM_OK;
  } catch (const RmError& e) {
    return fail(e);
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return RM_ENOMEM;
  } catch (const std::exception& e) {
    std::string m = e.what();
    g_err = m;
    if (m.find("pivot") != std::string::npos || m.find("breakdown") != std::string::npos) return RM_ENUMERIC;
    return RM_EINVAL;
  }
}

rm_status rm_layout(const rm_ctx* c, int64_t* n_local, int64_t* n_free, int32_t shape[3][3]) {
  if (!c) { g_err = "null context"; return RM_EINVAL; }
  if (n_local) *n_local = c->ndof;
  if (n_free) *n_free = c->nfree;
  if (shape)
    for (int m = 0; m < 3; ++m)
      for (int d = 0; d < 3; ++d) shape[m][d] = (m < c->sp.ncomp) ? (int32_t)c->sp.len(m, 2 - d) : 0;
  return RM_OK;
}

rm_status rm_info_get(const rm_ctx* c, rm_info* info) {
  if (!c || !info) { g_err = "null argument"; return RM_EINVAL; }
  std::memset(info, 0, sizeof *info);
  info->n_local = c->ndof;
  info->n_free = c->nfree;
  for (const auto& F : c->prims) {
    info->n_patches += F.npatch;
    info->n_factor_blocks += F.nfactors;
    info->factor_bytes += F.sweep_value_bytes;
    info->n_classes += (int32_t)F.nclasses;
  }
  for (const auto& F : c->pots) {
    info->n_patches_potential += F.npatch;
    info->n_factor_blocks += F.nfactors;
    info->factor_bytes += F.sweep_value_bytes;
    info->n_classes += (int32_t)F.nclasses;
  }
  info->sweep_bytes = info->factor_bytes + 3 * 8 * c->ndof;
  for (const auto& F : c->prims) {
    info->n_colors += F.ncolors;
    info->factor_nnz_primary += F.nnzL;
    info->icc_sigma_max = std::max(info->icc_sigma_max, F.sigma_max);
  }
  info->factor_nnz = info->factor_nnz_primary;
  for (const auto& F : c->prims) info->factor_unique_bytes += F.unique_bytes;
  for (const auto& F : c->pots) {
    info->factor_nnz += F.nnzL;
    info->factor_unique_bytes += F.unique_bytes;
    info->icc_sigma_max = std::max(info->icc_sigma_max, F.sigma_max);
  }
  info->comm_nranks = c->comm ? c->nranks : 0;
  info->coarse = c->coarse ? 1 : 0;
  info->coarse_ndof = c->coarse ? c->coarse->nfree1 : 0;
  for (const auto* fams : {&c->prims, &c->pots})
    for (const auto& F : *fams)
      if (F.launch.batch) {
        ++info->batched_families;
        info->batch_width = std::max(info->batch_width, F.launch.batch);
      }
  info->setup_seconds = c->setup_seconds;
  info->setup_on_device = c->setup_device ? 1 : 0;
  info->setup_host_family_seconds = c->setup_family_s;
  for (const auto* fams : {&c->prims, &c->pots})
    for (const auto& F : *fams) info->setup_device_numeric_seconds += F.numeric_s;
  return RM_OK;
}

rm_status rm_constrained_mask(const rm_ctx* c, uint8_t* mask) {
  if (!c || !mask) { g_err = "null argument"; return RM_EINVAL; }
  std::memcpy(mask, c->mask.data(), c->mask.size());
  return RM_OK;
}

}  // extern "C"

namespace {

// records CUDA events around one kernel launch (phases 4, 5) when timing is enabled
struct KPhase {
  rm_ctx* c;
  int ph;
  cudaEvent_t a = nullptr;
  static void begin(void* p) {
    auto* k = static_cast<KPhase*>(p);
    if (!k->c->timing) return;
    if (cudaEventCreate(&k->a) != cudaSuccess || cudaEventRecord(k->a, k->c->st) != cudaSuccess) k->a = nullptr;
  }
  static void end(void* p) {
    auto* k = static_cast<KPhase*>(p);
    if (!k->a) return;
    cudaEvent_t b;
    if (cudaEventCreate(&b) == cudaSuccess && cudaEventRecord(b, k->c->st) == cudaSuccess) {
      k->c->events.push_back({k->ph, k->a, b});
      k->c->launches[k->ph] += 1;
    } else {
      cudaEventDestroy(k->a);
    }
    k->a = nullptr;
  }
  rm::KTimer timer() { return rm::KTimer{&KPhase::begin, &KPhase::end, this}; }
};

// records CUDA events around a phase when timing is enabled
struct Phase {
  rm_ctx* c;
  int ph;
  cudaEvent_t a = nullptr;
  Phase(rm_ctx* c_, int ph_) : c(c_), ph(ph_) {
    if (!c->timing) return;
    CK(cudaEventCreate(&a));
    CK(cudaEventRecord(a, c->st));
  }
  ~Phase() {
    if (!a) return;
    cudaEvent_t b;
    if (cudaEventCreate(&b) == cudaSuccess && cudaEventRecord(b, c->st) == cudaSuccess) c->events.push_back({ph, a, b});
    else cudaEventDestroy(a);
  }
};

// out = f - A u (or A u); ldx > 0 (k = 0): out in the padded layout with x-stride ldx
void do_apply(rm_ctx* c, const double* u, const double* f, double* out, long long ldx = 0) {
  Phase ph(c, 0);
  int nl = 0;
  KPhase kp{c, 5};
  const rm::KTimer kt = kp.timer();
  if (c->cartesian) {
    c->op.ldx_out = ldx;
    CK(rm::launch_apply_cartesian(c->op, c->d_alpha, c->d_beta, c->coef_const, c->d_hpow, u, f, out, c->ndof, c->st, &nl,
                                  &kt, c->d_cellbuf));
    c->op.ldx_out = 0;
  } else {
    c->tri.ldx_out = ldx;
    CK(rm::launch_apply_trilinear(c->tri, c->d_tabs, c->d_X, c->d_alpha, c->d_beta, c->coef_const, u, f, out,
                                  f ? -1.0 : 1.0, c->d_cellbuf, c->st, &nl, &kt));
    c->tri.ldx_out = 0;
  }
  c->launches[0] += nl;
}

// families of one space run back to back on shared padded buffers: the first pads r and zeroes c,
// the last adds omega c to u
int run_family(rm_ctx* c, DevFamily& F, const double* r, double* u, double omega, bool r_padded = false,
               bool zero_c = true, bool combine = true, bool sc_pre_done = false, const double* u_in = nullptr) {
  if (!F.present) {
    if (combine && u_in && u_in != u) CK(cudaMemcpyAsync(u, u_in, c->ndof * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    return 0;
  }
  KPhase kp{c, 4};
  const rm::KTimer kt = kp.timer();
  CK(rm::launch_patch_solve(F.launch, r, u, omega, c->st, &kt, r_padded, zero_c, combine, sc_pre_done,
                            u_in != u ? u_in : nullptr));
  return 3;   // pad(r), persistent patch kernel, u += omega * unpad(c)
}

// u += omega * P^{-1} r  (r zero on constrained DoFs)
// u_in (optional, != u): the primary combine writes u = u_in + omega c (no u_out = u_in copy)
void add_precond(rm_ctx* c, const double* r, double* u, double omega, bool r_padded = false,
                 const double* u_in = nullptr) {
  if (u_in && u_in != u && (c->decomposition == RM_SC_PH || c->prims.empty())) {
    CK(cudaMemcpyAsync(u, u_in, c->ndof * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    u_in = nullptr;
  }
  if (c->decomposition == RM_SC_PH) {
    // c = R_I^T A_II^{-1} R_I r + R_G^T S_PH^{-1} R_G r (eq:schur, eq:sc-asm-hiptmair)
    const rm::ScPhParams& P = c->scph;
    const double* al = c->d_alpha;
    const double* be = c->d_beta;
    const int cc = c->coef_const;
    {
      Phase ph(c, 1);
      CK(rm::launch_scph_interior_solve(P, al, be, cc, c->d_scph_set, c->d_scph_mem, c->d_scph_K, c->d_scph_M, r,
                                        c->d_sy, c->st));                       // y = A_II^-1 r_I
    }
    do_apply(c, c->d_sy, nullptr, c->d_sw);                                     // w = A y
    {
      Phase ph(c, 1);
      CK(rm::launch_scph_vec(P, 0, r, c->d_sw, nullptr, c->d_srg, 0.0, c->st));  // R_G r = (r - A y)_G
      CK(cudaMemsetAsync(c->d_scg, 0, c->ndof * sizeof(double), c->st));
      const int nf = (int)c->prims.size();
      for (int o = 0; o < nf; ++o)                                              // c_G = sum_i R~_i^T S_i^-1 R~_i R_G r
        c->launches[1] += run_family(c, c->prims[o], c->d_srg, c->d_scg, 1.0, o > 0, o == 0, o == nf - 1);
      c->launches[1] += 3;
    }
    {
      Phase ph(c, 2);                                                           // + D~ (sum_j B~_j^-1) D~^T R_G r
      CK(rm::launch_hiptmair_DT(c->k, c->p, c->n, c->gamma, c->Dh.data(), c->d_srg, c->d_t, c->st));
      CK(cudaMemsetAsync(c->d_s, 0, c->npot * sizeof(double), c->st));
      const int np = (int)c->pots.size();
      for (int o = 0; o < np; ++o)
        c->launches[2] += run_family(c, c->pots[o], c->d_t, c->d_s, 1.0, o > 0, o == 0, o == np - 1);
      CK(rm::launch_hiptmair_D_add(c->k, c->p, c->n, c->gamma, c->Dh.data(), c->d_s, c->d_scg, 1.0, c->st));
      CK(rm::launch_scph_vec(P, 1, nullptr, nullptr, nullptr, c->d_scg, 0.0, c->st));   // D~ = D_GG
      c->launches[2] += 3;
    }
    do_apply(c, c->d_scg, nullptr, c->d_sw);                                    // w = A c_G
    {
      Phase ph(c, 1);
      CK(rm::launch_scph_interior_solve(P, al, be, cc, c->d_scph_set, c->d_scph_mem, c->d_scph_K, c->d_scph_M,
                                        c->d_sw, c->d_sz, c->st));              // z = A_II^-1 (A c_G)_I
      CK(rm::launch_scph_vec(P, 2, c->d_sy, c->d_sz, c->d_scg, u, omega, c->st));   // u += omega (y_I - z_I ; c_G)
      c->launches[1] += 4;
    }
    return;
  }
  {
    Phase ph(c, 1);
    const int nf = (int)c->prims.size();
    for (int o = 0; o < nf; ++o)
      c->launches[1] += run_family(c, c->prims[o], r, u, omega, r_padded || o > 0, o == 0, o == nf - 1, false,
                                   o == nf - 1 ? u_in : nullptr);
  }
  if (c->pots[0].present) {
    Phase ph(c, 2);
    CK(rm::launch_hiptmair_DT(c->k, c->p, c->n, c->gamma, c->Dh.data(), r, c->d_t, c->st));
    CK(cudaMemsetAsync(c->d_s, 0, c->npot * sizeof(double), c->st));
    c->launches[2] += 2;
    const int np = (int)c->pots.size();
    for (int o = 0; o < np; ++o)
      c->launches[2] += run_family(c, c->pots[o], c->d_t, c->d_s, 1.0, o > 0, o == 0, o == np - 1);
    CK(rm::launch_hiptmair_D_add(c->k, c->p, c->n, c->gamma, c->Dh.data(), c->d_s, u, omega, c->st));
  }
}

// z = M r: the PCG preconditioner.  One level: the additive sweep from zero.  With the coarse
// level: the hybrid V(1,1) cycle (reading G20)
//   z1 = w S r,  z2 = z1 + R_0^T A_0^{-1} R_0 (r - A z1),  z = z2 + w S (r - A z2)
// (r zero on constrained DoFs; z overwritten)
void apply_cycle(rm_ctx* c, const double* r, double* z) {
  CK(cudaMemsetAsync(z, 0, c->ndof * sizeof(double), c->st));
  if (!c->coarse) {
    add_precond(c, r, z, 1.0);
    return;
  }
  const double w = c->smoother_omega;
  add_precond(c, r, z, w);
  do_apply(c, z, r, c->d_vt);                         // r - A z1
  {
    Phase ph(c, 3);
    CK(rm::launch_coarse_correct(c->cl, c->d_vt, z, c->st));
  }
  do_apply(c, z, r, c->d_vt);                         // r - A z2
  add_precond(c, c->d_vt, z, w);
}

// ------------------------------------------------------------------ multi-rank sweep pieces
// Per component: offset, doubles per z plane, and whether its z family is DP (H(curl) / H(div)
// components; rm.h: the dp_* ranges)
struct CompPlanes { long long off, L; bool dp; };
std::vector<CompPlanes> comp_planes(const rm_ctx* c) {
  std::vector<CompPlanes> v;
  for (int m = 0; m < c->sp.ncomp; ++m)
    v.push_back({(long long)c->sp.offset(m), (long long)(c->sp.len(m, 0) * c->sp.len(m, 1)), c->sp.fam[m][2] == rm::FAM_D});
  return v;
}

// Forward halo: the non-owned planes of each vector <- the owners' planes (NCCL send/recv in ONE
// group on the stream, in place: the non-owned planes of the caller's input vectors are
// overwritten, include/rm.h), component by component.
void halo_forward(rm_ctx* c, double* const* vs, int nv) {
  const rm_partition_info& P = c->part;
  const NcclApi& N = nccl();
  const std::vector<CompPlanes> cp = comp_planes(c);
  NK(N.gstart());
  for (int i = 0; i < nv; ++i)
    for (const CompPlanes& q : cp) {
      double* v = vs[i] + q.off;
      const size_t L = (size_t)q.L;
      const int* rlo = q.dp ? P.dp_fwd_recv_lo : P.fwd_recv_lo;
      const int* slo = q.dp ? nullptr : P.fwd_send_lo;
      const int* rhi = q.dp ? nullptr : P.fwd_recv_hi;
      const int* shi = q.dp ? P.dp_fwd_send_hi : P.fwd_send_hi;
      if (c->rank > 0) {
        if (slo && slo[1] > slo[0]) NK(N.send(v + slo[0] * L, (slo[1] - slo[0]) * L, ncclDouble, c->rank - 1, c->comm, c->st));
        if (rlo[1] > rlo[0]) NK(N.recv(v + rlo[0] * L, (rlo[1] - rlo[0]) * L, ncclDouble, c->rank - 1, c->comm, c->st));
      }
      if (c->rank < c->nranks - 1) {
        if (shi[1] > shi[0]) NK(N.send(v + shi[0] * L, (shi[1] - shi[0]) * L, ncclDouble, c->rank + 1, c->comm, c->st));
        if (rhi && rhi[1] > rhi[0]) NK(N.recv(v + rhi[0] * L, (rhi[1] - rhi[0]) * L, ncclDouble, c->rank + 1, c->comm, c->st));
      }
    }
  NK(N.gend());
}
void halo_forward(rm_ctx* c, double* v) { halo_forward(c, &v, 1); }
// Reverse-add: the corrections my patches put on rank - 1's planes go there and are added by it,
// component by component (Lpad > 0: one component in the patch kernel's padded layout, plane
// length Lpad).
void reverse_add(rm_ctx* c, double* cv, size_t Lpad = 0) {
  const rm_partition_info& P = c->part;
  const NcclApi& N = nccl();
  std::vector<CompPlanes> cp = comp_planes(c);
  if (Lpad) cp = {{0, (long long)Lpad, false}};
  std::vector<size_t> roff(cp.size() + 1, 0);
  for (size_t i = 0; i < cp.size(); ++i) {
    const int* r = cp[i].dp ? P.dp_rev_recv_hi : P.rev_recv_hi;
    roff[i + 1] = roff[i] + (size_t)(r[1] - r[0]) * cp[i].L;
  }
  NK(N.gstart());
  for (size_t i = 0; i < cp.size(); ++i) {
    const CompPlanes& q = cp[i];
    const int* sl = q.dp ? P.dp_rev_send_lo : P.rev_send_lo;
    if (c->rank > 0 && sl[1] > sl[0])
      NK(N.send(cv + q.off + sl[0] * q.L, (sl[1] - sl[0]) * q.L, ncclDouble, c->rank - 1, c->comm, c->st));
    if (c->rank < c->nranks - 1 && roff[i + 1] > roff[i])
      NK(N.recv(c->d_rtmp + roff[i], roff[i + 1] - roff[i], ncclDouble, c->rank + 1, c->comm, c->st));
  }
  NK(N.gend());
  if (c->rank < c->nranks - 1)
    for (size_t i = 0; i < cp.size(); ++i) {
      const int* r = cp[i].dp ? P.dp_rev_recv_hi : P.rev_recv_hi;
      if (roff[i + 1] > roff[i])
        CK(rm::launch_axpby((long long)(roff[i + 1] - roff[i]), 1.0, c->d_rtmp + roff[i], 1.0, cv + cp[i].off + r[0] * cp[i].L,
                            c->st));
    }
}
// In-place sum over ranks of device scalars.
void allreduce_sum(rm_ctx* c, double* x, size_t n) {
  if (c->nranks > 1) NK(nccl().allreduce(x, x, n, ncclDouble, ncclSum, c->comm, c->st));
}
// Local patch correction cv = P_local^{-1} (f - A u): f, u with their forward halos filled.
void local_correction(rm_ctx* c, const double* f, const double* u, double* cv) {
  do_apply(c, u, f, c->d_r);
  CK(cudaMemsetAsync(cv, 0, c->ndof * sizeof(double), c->st));
  add_precond(c, c->d_r, cv, 1.0);
}
void need_comm(const rm_ctx* c) {
  if (c->nranks > 1 && !c->comm)
    throw RmError(RM_EINVAL, "multi-rank call needs options.nccl_id (or the rm_relax_begin / rm_relax_end stages)");
}

template <class F>
rm_status guarded(rm_ctx* c, F&& f) {
  if (!c) { g_err = "null context"; return RM_EINVAL; }
  try {
    CK(cudaSetDevice(c->device));
    f();
    return RM_OK;
  } catch (const RmError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    g_err = e.what();
    return RM_EINVAL;
  }
}

// the forward halo of an input vector, exchanged in place (multi-rank with a communicator; the
// caller's non-owned planes are overwritten, include/rm.h); the vector itself otherwise
const double* with_halo(rm_ctx* c, const double* u) {
  if (c->nranks == 1 || !c->comm) return u;
  halo_forward(c, const_cast<double*>(u));
  return u;
}

bool fused_k0(const rm_ctx* c) {
  return c->k == 0 && !c->pots[0].present && c->prims.size() == 1 && c->prims[0].npatch > 0;
}

// trilinear ICC-SC family on one rank: the SC pre step joins the residual (apply -> condensation
// of the cell interiors -> skeleton gather minus the line sums)
bool sc_fused(const rm_ctx* c) {
  return fused_k0(c) && !c->cartesian && c->nranks == 1 && c->prims[0].launch.sc_dinv && c->prims[0].launch.sc_pre;
}

// f_ready (optional): f arrives on another stream; the apply (u only) runs before the wait
void residual_sc_fused(rm_ctx* c, const double* u, const double* f, const rm::PatchLaunch& L,
                       cudaEvent_t f_ready = nullptr) {
  Phase ph(c, 0);
  int nl = 0;
  KPhase kp{c, 5};
  const rm::KTimer kt = kp.timer();
  c->tri.ldx_out = L.pad.lxp[0];
  c->tri.skip_gather = 1;
  CK(rm::launch_apply_trilinear(c->tri, c->d_tabs, c->d_X, c->d_alpha, c->d_beta, c->coef_const, u, f, L.rpad, -1.0,
                                c->d_cellbuf, c->st, &nl, &kt));
  c->tri.skip_gather = 0;
  if (f_ready) CK(cudaStreamWaitEvent(c->st, f_ready, 0));
  CK(rm::launch_sc_pre_fused(L, f, c->tri.Lx, c->st));
  CK(rm::launch_skeleton_gather_sc(c->tri, c->d_cellbuf, f, L.rpad, -1.0, L.sc_fb, c->st));
  c->tri.ldx_out = 0;
  c->launches[0] += nl + 2;   // the apply (skip_gather: 1), sc_cell, the skeleton gather
}

// one sweep u_out = u_in + omega P^{-1} (f - A u_in) (z-slab: halos, local correction, reverse-add)
void relax_impl(rm_ctx* c, const double* f, const double* u_in, double* u_out, double omega) {
  if (c->nranks > 1) {
    need_comm(c);
    {
      double* vs[2] = {const_cast<double*>(f), const_cast<double*>(u_in)};
      halo_forward(c, vs, 2);   // f and u_in, in place, one NCCL group
    }
    if (fused_k0(c)) {
      // as on one rank: the residual straight into the padded TMA layout, corrections accumulated
      // in the padded c, reverse-added there (padded planes), then u_out = u_in + omega c
      const rm::PatchLaunch& L = c->prims[0].launch;
      do_apply(c, u_in, f, L.rpad, L.pad.lxp[0]);
      {
        Phase ph(c, 1);
        c->launches[1] += run_family(c, c->prims[0], L.rpad, u_out, omega, true, true, false);
      }
      reverse_add(c, L.cpad, (size_t)(L.pad.lxp[0] * L.pad.len[0][1]));
      if (u_out != u_in) CK(cudaMemcpyAsync(u_out, u_in, c->ndof * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
      CK(rm::launch_patch_combine(L, u_out, omega, c->st));
      return;
    }
    local_correction(c, f, u_in, c->d_c);
    reverse_add(c, c->d_c);
    if (u_out != u_in) CK(cudaMemcpyAsync(u_out, u_in, c->ndof * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    CK(rm::launch_axpby(c->ndof, omega, c->d_c, 1.0, u_out, c->st));
    return;
  }
  if (sc_fused(c)) {
    const rm::PatchLaunch& L = c->prims[0].launch;
    residual_sc_fused(c, u_in, f, L);
    Phase ph(c, 1);
    c->launches[1] += run_family(c, c->prims[0], L.rpad, u_out, omega, true, true, true, true, u_in);
    return;
  }
  if (fused_k0(c)) {
    // the residual goes straight into the primary family's padded (TMA) layout: no pad pass
    const rm::PatchLaunch& L = c->prims[0].launch;
    do_apply(c, u_in, f, L.rpad, L.pad.lxp[0]);
    add_precond(c, L.rpad, u_out, omega, true, u_in);
    return;
  }
  do_apply(c, u_in, f, c->d_r);
  add_precond(c, c->d_r, u_out, omega, false, u_in);
}

}  // namespace

extern "C" {

rm_status rm_apply(rm_ctx* c, const double* u, double* v) {
  return guarded(c, [&] {
    if (!u || !v) throw RmError(RM_EINVAL, "null vector");
    do_apply(c, with_halo(c, u), nullptr, v);
  });
}

rm_status rm_residual(rm_ctx* c, const double* f, const double* u, double* r) {
  return guarded(c, [&] {
    if (!f || !u || !r) throw RmError(RM_EINVAL, "null vector");
    do_apply(c, with_halo(c, u), f, r);
  });
}

rm_status rm_relax(rm_ctx* c, const double* f, const double* u_in, double* u_out, double omega) {
  return guarded(c, [&] {
    if (!f || !u_in || !u_out) throw RmError(RM_EINVAL, "null vector");
    relax_impl(c, f, u_in, u_out, omega);
  });
}

rm_status rm_relax_begin(rm_ctx* c, const double* f, const double* u_in, double* cv) {
  return guarded(c, [&] {
    if (!f || !u_in || !cv) throw RmError(RM_EINVAL, "null vector");
    local_correction(c, f, u_in, cv);
  });
}

rm_status rm_relax_end(rm_ctx* c, const double* u_in, const double* cv, double* u_out, double omega) {
  return guarded(c, [&] {
    if (!u_in || !cv || !u_out) throw RmError(RM_EINVAL, "null vector");
    if (u_out != u_in) CK(cudaMemcpyAsync(u_out, u_in, c->ndof * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
    CK(rm::launch_axpby(c->ndof, omega, cv, 1.0, u_out, c->st));
  });
}

rm_status rm_precondition(rm_ctx* c, const double* r, double* z) {
  return guarded(c, [&] {
    if (!r || !z) throw RmError(RM_EINVAL, "null vector");
    need_comm(c);
    // r with constrained entries read as zero: the residual kernel with u = 0
    const double* rh = with_halo(c, r);
    CK(cudaMemsetAsync(z, 0, c->ndof * sizeof(double), c->st));
    do_apply(c, z, rh, c->d_r);   // d_r = r - A*0 = r, constrained entries zeroed
    apply_cycle(c, c->d_r, z);
    if (c->nranks > 1) reverse_add(c, z);
  });
}

rm_status rm_relax_host(rm_ctx* c, const double* f, const double* u_in, double* u_out, double omega) {
  return guarded(c, [&] {
    if (!f || !u_in || !u_out) throw RmError(RM_EINVAL, "null vector");
    if (!c->d_hf) { c->d_hf = c->dalloc(c->ndof); c->d_hu = c->dalloc(c->ndof); }
    const size_t B = c->ndof * sizeof(double);
    if (sc_fused(c)) {
      // the trilinear apply needs u only: copy u first, then f on a second stream while the
      // apply runs (f is first read by the SC pre step); same kernels and results as relax_impl
      if (!c->st_copy) {
        CK(cudaStreamCreateWithFlags(&c->st_copy, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_u, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_f, cudaEventDisableTiming));
      }
      CK(cudaMemcpyAsync(c->d_hu, u_in, B, cudaMemcpyHostToDevice, c->st));
      CK(cudaEventRecord(c->ev_u, c->st));
      CK(cudaStreamWaitEvent(c->st_copy, c->ev_u, 0));   // u's copy first (one H2D engine at a time)
      CK(cudaMemcpyAsync(c->d_hf, f, B, cudaMemcpyHostToDevice, c->st_copy));
      CK(cudaEventRecord(c->ev_f, c->st_copy));
      const rm::PatchLaunch& L = c->prims[0].launch;
      residual_sc_fused(c, c->d_hu, c->d_hf, L, c->ev_f);
      Phase ph(c, 1);
      c->launches[1] += run_family(c, c->prims[0], L.rpad, c->d_hu, omega, true, true, true, true, nullptr);
      CK(cudaMemcpyAsync(u_out, c->d_hu, B, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      return;
    }
    CK(cudaMemcpyAsync(c->d_hf, f, B, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->d_hu, u_in, B, cudaMemcpyHostToDevice, c->st));
    relax_impl(c, c->d_hf, c->d_hu, c->d_hu, omega);
    CK(cudaMemcpyAsync(u_out, c->d_hu, B, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  });
}

rm_status rm_pcg(rm_ctx* c, const double* f, double* u, double rtol, int32_t maxit, int32_t* iters, double* rel) {
  rm_status conv = RM_OK;
  rm_status s = guarded(c, [&] {
    if (!f || !u) throw RmError(RM_EINVAL, "null vector");
    if (!c->d_z) { c->d_z = c->dalloc(c->ndof); c->d_pp = c->dalloc(c->ndof); c->d_q = c->dalloc(c->ndof); c->d_pr = c->dalloc(c->ndof); }
    const size_t B = c->ndof * sizeof(double);
    double* r = c->d_pr;
    double* rz = c->d_sc + 0;
    double* pq = c->d_sc + 1;
    double* rzn = c->d_sc + 2;
    need_comm(c);
    // multi-rank: dots over the owned planes (a contiguous range) + allreduce; halo of the
    // search direction before each apply; reverse-add after each preconditioner application
    // multi-rank: owned planes of every component (a contiguous range per component)
    const std::vector<CompPlanes> cpl = comp_planes(c);
    auto dot = [&](const double* x, const double* y, double* out) {
      if (c->nranks == 1) {
        CK(rm::launch_dot(c->ndof, x, y, c->d_part, out, c->st));
        return;
      }
      for (size_t m = 0; m < cpl.size(); ++m) {
        const CompPlanes& q = cpl[m];
        const int lo = q.dp ? c->part.dp_own_lo : c->part.own_lo, hi = q.dp ? c->part.dp_own_hi : c->part.own_hi;
        const long long o = q.off + (long long)lo * q.L, nn = (long long)(hi - lo) * q.L;
        CK(rm::launch_dot(nn, x + o, y + o, c->d_part, m == 0 ? out : c->d_sc + 4, c->st));
        if (m > 0) CK(rm::launch_axpby(1, 1.0, c->d_sc + 4, 1.0, out, c->st));
      }
      allreduce_sum(c, out, 1);
    };
    auto precond = [&](const double* rr, double* zz) {
      apply_cycle(c, rr, zz);
      if (c->nranks > 1) reverse_add(c, zz);
    };
    CK(cudaMemsetAsync(u, 0, B, c->st));
    do_apply(c, u, with_halo(c, f), r);   // r = f (masked)
    precond(r, c->d_z);
    dot(r, c->d_z, rz);
    double rz0 = 0.0;
    CK(cudaMemcpyAsync(&rz0, rz, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    int it = 0;
    double relv = 0.0;
    if (rz0 != 0.0) {
      relv = 1.0;
      CK(cudaMemcpyAsync(c->d_pp, c->d_z, B, cudaMemcpyDeviceToDevice, c->st));
      bool done = false;
      for (it = 1; it <= maxit; ++it) {
        if (c->nranks > 1) halo_forward(c, c->d_pp);
        do_apply(c, c->d_pp, nullptr, c->d_q);
        dot(c->d_pp, c->d_q, pq);
        CK(rm::launch_pcg_update(c->ndof, rz, pq, c->d_pp, c->d_q, u, r, c->st));
        precond(r, c->d_z);
        dot(r, c->d_z, rzn);
        double h = 0.0;
        CK(cudaMemcpyAsync(&h, rzn, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        relv = std::sqrt(std::max(h, 0.0) / rz0);
        if (relv <= rtol) { done = true; break; }
        CK(rm::launch_pcg_pupdate(c->ndof, rzn, rz, c->d_z, c->d_pp, c->st));
        CK(cudaMemcpyAsync(rz, rzn, 8, cudaMemcpyDeviceToDevice, c->st));
      }
      if (!done) { it = maxit; conv = RM_NOT_CONVERGED; }
    }
    CK(cudaStreamSynchronize(c->st));
    if (iters) *iters = it;
    if (rel) *rel = relv;
  });
  return s != RM_OK ? s : conv;
}

rm_status rm_timing_enable(rm_ctx* c, int32_t on) {
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->st));
    for (auto& e : c->events) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
    c->events.clear();
    for (auto& l : c->launches) l = 0;
    c->timing = on != 0;
  });
}

rm_status rm_timing_read(rm_ctx* c, double ms[RM_NPHASE], int64_t launches[RM_NPHASE]) {
  return guarded(c, [&] {
    CK(cudaStreamSynchronize(c->st));
    double acc[RM_NPHASE] = {};
    for (auto& e : c->events) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, e.a, e.b));
      acc[e.phase] += t;
      cudaEventDestroy(e.a); cudaEventDestroy(e.b);
    }
    c->events.clear();
    for (int i = 0; i < RM_NPHASE; ++i) {
      if (ms) ms[i] = acc[i];
      if (launches) launches[i] = c->launches[i];
      c->launches[i] = 0;
    }
  });
}

void rm_destroy(rm_ctx* c) { delete c; }

}  // extern "C"
