// Batched star-patch solve as ONE persistent streaming kernel
// per patch family and sweep.
//
// Per patch i:
//   gather   v = R_i r                                   (structured offsets per class)
//   forward  per elimination level: y^_E = P_EE^{-1} v_E (pivot blocks <= 3x3, Cholesky form),
//            v_R -= P_RE y^_E
//   final    x_F = S_F^{-1} v_F  (S_F^{-1} as 32x32 tiles of the lower block triangle, symmetric
//            tile GEMV) -- or, for ICC-SC, level-scheduled triangular solves
//   backward per level in reverse: x_E = y^_E - (P_EE^{-1} P_ER) x_R
//   scatter  u += omega R_i^T x
// This is block Gaussian elimination of the patch matrix with the eliminated sets first (exact
// for the Cholesky family), so x = A_i^{-1} R_i r up to rounding.
//
// B200 structure.  Every factor value is read exactly once per sweep, so the kernel is an HBM
// stream.  Each patch value block is laid out in consumption order (patches.hpp); consecutive
// pieces form transfer units (16 KB sparse, 32 KB dense-tile).  One persistent CTA per SM,
// warp-specialised and software-pipelined across the CTA's patches i = 0, 1, ...:
//   producer  streams the units HBM -> shared memory with cp.async.bulk (TMA, UBLKCP) into two
//             rings (sparse channel, tile channel) and loads each patch's window box of r with a
//             TMA tensor copy (UTMALDG) into one of three box buffers;
//   8 sparse warps   forward(i+1), then [final(i) if not dense], backward(i) -- the sparse
//             eliminations of two patches around the dense phase of one;
//   4 tile warps     the dense final-block GEMV of patch i (lane-block tiles, LDS.128 + DFMA);
//   store     reduce-adds the finished box into the correction c with a TMA tensor reduction
//             (UTMAREDG .add, fp64, atomic per element) once the colour order allows.
// The tile stream (~78% of the bytes) therefore runs while the latency-bound sparse phases of
// the neighbouring patches execute, and no global gather/scatter loop is left on compute warps.
//
// Colours.  Patches of one colour are disjoint, so their corrections commute; patches are
// sorted by colour and a colour-c box is reduce-added only after every box of colours < c has
// landed (a device counter, acquire/release).  Each c entry therefore receives its updates in
// colour order (boxes also add exact zeros outside their patch, which commute): the sweep is
// bitwise deterministic, with one launch instead of one per colour.  All CTAs are co-resident
// (grid = occupancy x SMs) and take patches in increasing order (CTA b: b, b + grid, ...); the
// wait cannot deadlock (the pending reduction of lowest colour never waits; induction on the
// colour).  The value blocks are laid out in HBM in that per-CTA order (abi.cpp), so every CTA
// streams one contiguous region.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace rm {

namespace {

constexpr int NC = RM_PATCH_CONSUMER_WARPS;   // sparse warps
constexpr int NT = NC * 32;
constexpr int NTW = RM_PATCH_TILE_WARPS;       // tile warps
#ifndef RM_ICC_CHUNKS
#define RM_ICC_CHUNKS 4
#endif
constexpr int kIccChunksDev = RM_ICC_CHUNKS;   // = kIccChunks (patches.hpp): chunks per ICC piece
constexpr int WT0 = NC, WPROD_A = NC + NTW, WPROD_B = NC + NTW + 1, WSTORE = NC + NTW + 2;
constexpr int NTHR = 32 * (NC + NTW + 3);
#ifndef RM_NDESC
#define RM_NDESC 16
#endif
constexpr int NDESC = RM_NDESC;                // in-flight transfer units per channel
constexpr int NBOX = 3;                        // window-box buffers (patches i-1, i, i+1)
// shared-memory header: per channel full/empty mbarriers and slot tables (offset, pieces, meta),
// then the box barriers vfull (TMA box landed), gready (forward done), xready (tiles done),
// vdone (backward done), vempty (reduction has read the box), NBOX each
constexpr int CH_BYTES = 2 * NDESC * 8 + 3 * NDESC * 4;   // 448
constexpr int VBAR_OFS = 2 * CH_BYTES;
constexpr int BAR_BYTES = (VBAR_OFS + 5 * NBOX * 8 + 127) & ~127;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}
// L2 eviction priorities (tuning knobs): the factor values are read once per sweep, the window
// boxes of r (and the reduce-added c boxes) are re-read by the patches of the other colours
#ifndef RM_L2_VALS   // 1: factor value stream with L2::evict_first (measured, pass AK: cfg5 patch kernel
#define RM_L2_VALS 1  // 1.273 -> 1.253 ms; cfg2 unchanged 3.647 / 3.644; the box / reduce hints add nothing)
#endif
#ifndef RM_L2_BOX    // 1: window-box loads of r with L2::evict_last
#define RM_L2_BOX 0
#endif
#ifndef RM_L2_RED    // 1: reduce-adds into c with L2::evict_last
#define RM_L2_RED 0
#endif
__device__ __forceinline__ uint64_t l2_policy(bool last) {
  uint64_t pol;
  if (last) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void bulk_vals(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
#if RM_L2_VALS
  bulk_g2s_hint(dst, src, bytes, b, l2_policy(false));
#else
  bulk_g2s(dst, src, bytes, b);
#endif
}
// named barriers: 1 = sparse warps, 2 = tile warps
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred P;\n mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tsync() { asm volatile("bar.sync 2, %0;" ::"n"(NTW * 32) : "memory"); }

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* tm, int x, int y, int z, uint64_t* bar) {
#if RM_L2_BOX
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(l2_policy(true))
      : "memory");
#else
  tma_load_3d(dst, tm, x, y, z, bar);
#endif
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* tm, int x, int y, int z, const void* src);
__device__ __forceinline__ void tma_reduce_box(const CUtensorMap* tm, int x, int y, int z, const void* src) {
#if RM_L2_RED
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;" ::"l"(tm),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src)), "l"(l2_policy(true))
               : "memory");
#else
  tma_reduce_add_3d(tm, x, y, z, src);
#endif
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* tm, int x, int y, int z, const void* src) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
               "r"(x), "r"(y), "r"(z), "r"(smem_u32(src))
               : "memory");
}

// one lane of a converged warp (PTX elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// shared-memory view of one channel
struct ChanSm {
  uint64_t* full;
  uint64_t* empty;
  int* ofs;
  int* np;
  int* mb;
};
__device__ __forceinline__ ChanSm chan_sm(unsigned char* smraw, int ch) {
  unsigned char* b = smraw + ch * CH_BYTES;
  ChanSm c;
  c.full = reinterpret_cast<uint64_t*>(b);
  c.empty = c.full + NDESC;
  c.ofs = reinterpret_cast<int*>(c.empty + NDESC);
  c.np = c.ofs + NDESC;
  c.mb = c.np + NDESC;
  return c;
}

// Ring placement (producer only): units at increasing virtual byte offsets, never straddling
// the end of the ring.
__device__ __forceinline__ uint32_t ring_place(uint32_t& H, uint32_t nbytes, uint32_t cap) {
  const uint32_t off = H % cap;
  if (off + nbytes > cap) H += cap - off;
  const uint32_t vs = H;
  H += nbytes;
  return vs;
}

struct Piece_ { const unsigned char* pb; const double* val; };

// Consumer side of one channel: unit j sits in slot j % NDESC; inside a unit the pieces are
// walked with a meta cursor and a value cursor (header word 3 = meta bytes | values << 16).
struct Consumer {
  ChanSm c;
  const unsigned char* ring;
  int j, left;
  const unsigned char* mcur;
  const unsigned char* vcur;
  __device__ __forceinline__ Piece_ acquire() {
    if (left == 0) {
      const int d = j % NDESC;
      mbar_wait(&c.full[d], (uint32_t)(j / NDESC) & 1u);
      mcur = ring + c.ofs[d];
      vcur = mcur + c.mb[d];
      left = c.np[d];
    }
    return Piece_{mcur, reinterpret_cast<const double*>(vcur)};
  }
  // done with the current piece; the unit is released after its last piece
  __device__ __forceinline__ void release(int lane) {
    const uint32_t w3 = reinterpret_cast<const uint32_t*>(mcur)[3];
    mcur += w3 & 0xFFFFu;
    vcur += (size_t)(w3 >> 16) * 8u;
    if (--left == 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&c.empty[j % NDESC]);
      ++j;
    }
  }
};

struct Hdr { int a0, a1, e0, mbytes; };
__device__ __forceinline__ Hdr hdr(const unsigned char* pb) {
  const int4 h = *reinterpret_cast<const int4*>(pb);
  return Hdr{h.x, h.y, h.z, h.w & 0xFFFF};
}

// one sliced-ELL piece: slice s is owned by warp s % NC (so split slices stay in one warp);
// meta = per slice (start/32 | count << 16), per slice 32 row boxes, column boxes (uint16)
template <class Emit>
__device__ __forceinline__ void sliced_piece(Piece_ pc, const double* v, int nrows, int warp, int lane, Emit&& emit) {
  const Hdr h = hdr(pc.pb);
  const int nsl = h.a1 - h.a0;
  const uint32_t* si = reinterpret_cast<const uint32_t*>(pc.pb + 16);
  const uint16_t* rows = reinterpret_cast<const uint16_t*>(si + nsl);
  const uint16_t* cols = rows + 32 * nsl;
  const double* val = pc.val;
  for (int ls = (warp - h.a0 % NC + NC) % NC; ls < nsl; ls += NC) {
    const uint32_t info = si[ls];
    const int st = 32 * (int)(info & 0xFFFFu) + lane, cnt = (int)(info >> 16);
    double acc = 0.0;
    int kk = 0;
    for (; kk + 4 <= cnt; kk += 4) {
      const int e = st + kk * 32;
      acc += val[e] * v[cols[e]] + val[e + 32] * v[cols[e + 32]] + val[e + 64] * v[cols[e + 64]] +
             val[e + 96] * v[cols[e + 96]];
    }
    for (; kk < cnt; ++kk) {
      const int e = st + kk * 32;
      acc += val[e] * v[cols[e]];
    }
    if ((h.a0 + ls) * 32 + lane < nrows) emit(rows[ls * 32 + lane], acc);
  }
}

// One 32x32 tile of the final block's inverse (lane-block layout, patches.hpp):
//   x_I += S g_J (row sums) and x_J += S^T g_I (column sums); for a diagonal tile (I == J) the
//   stored L' (strictly lower + half diagonal) gives S g = L' g + L'^T g with the same two sums.
// Lane (a, b) = (lane >> 2, lane & 3) accumulates 4 row partials and 8 column partials; two
// shuffle reduce-scatters leave row 4a + b and column 8b + a in lane (a, b).
__device__ __forceinline__ void tile_gemv(const double* __restrict__ tile, const double* __restrict__ g,
                                          double* __restrict__ part, int I, int J, int lane) {
  const unsigned FULL = 0xffffffffu;
  const int a = lane >> 2, b = lane & 3;
  const bool diag = (I == J);
  const bool active = !diag || b <= (a >> 1);
  const int slot = diag ? a + (a >> 1) * ((a - 1) >> 1) + b : lane;
  const int stride = diag ? 20 : 32;
  double ra0 = 0.0, ra1 = 0.0, ra2 = 0.0, ra3 = 0.0;
  double ca[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) ca[q] = 0.0;
  if (active) {
    const double2* T = reinterpret_cast<const double2*>(tile) + slot;
    const double2* gJ2 = reinterpret_cast<const double2*>(g + 32 * J + 8 * b);
    const double* gI = g + 32 * I + 4 * a;
#pragma unroll
    for (int i = 0; i < 4; ++i) {   // row 4a + i: four steps (8 columns), loads issued together
      double2 t[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = T[(4 * i + q) * stride];
      const double gi = gI[i];
      double& ra = (i == 0) ? ra0 : (i == 1) ? ra1 : (i == 2) ? ra2 : ra3;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 gj = gJ2[q];   // broadcast within the 8 lanes of equal b
        ra = fma(t[q].x, gj.x, ra);
        ra = fma(t[q].y, gj.y, ra);
        ca[2 * q] = fma(t[q].x, gi, ca[2 * q]);
        ca[2 * q + 1] = fma(t[q].y, gi, ca[2 * q + 1]);
      }
    }
  }
  // rows: reduce-scatter 4 values over the 4 lanes b = 0..3 (lane bits 0, 1)
  double rowsum;
  {
    const bool hi = (b & 2) != 0;
    double k0 = hi ? ra2 : ra0, k1 = hi ? ra3 : ra1;
    const double s0 = hi ? ra0 : ra2, s1 = hi ? ra1 : ra3;
    k0 += __shfl_xor_sync(FULL, s0, 2);
    k1 += __shfl_xor_sync(FULL, s1, 2);
    const bool h1 = (b & 1) != 0;
    rowsum = (h1 ? k1 : k0) + __shfl_xor_sync(FULL, h1 ? k0 : k1, 1);
  }
  // columns: reduce-scatter 8 values over the 8 lanes a = 0..7 (lane bits 2, 3, 4)
  double colsum;
  {
    const bool h4 = (a & 4) != 0;
    double k4[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double keep = h4 ? ca[4 + q] : ca[q], send = h4 ? ca[q] : ca[4 + q];
      k4[q] = keep + __shfl_xor_sync(FULL, send, 16);
    }
    const bool h2 = (a & 2) != 0;
    double k2[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double keep = h2 ? k4[2 + q] : k4[q], send = h2 ? k4[q] : k4[2 + q];
      k2[q] = keep + __shfl_xor_sync(FULL, send, 8);
    }
    const bool h1 = (a & 1) != 0;
    colsum = (h1 ? k2[1] : k2[0]) + __shfl_xor_sync(FULL, h1 ? k2[0] : k2[1], 4);
  }
  part[32 * I + 4 * a + b] += rowsum;
  part[32 * J + 8 * b + a] += colsum;
}

__device__ __forceinline__ int color_of(int q, const ColorStarts& cs) {
  int col = 0;
  while (col + 1 < cs.ncolors && cs.start[col + 1] <= q) ++col;
  return col;
}

}  // namespace

struct BoxGeom { int ncomp, box[3][3], boff[3], bytes; };   // ncomp = number of window sub-boxes

namespace {

// producer-side state of one channel ring (unused by the blocking per-channel producers)
struct ProdChan {
  ChanSm c;
  unsigned char* ring;
  uint32_t cap, H;
  int j, rel;
  uint32_t vs_of[NDESC];
  // try to place a unit of `tot` bytes; releases finished units without blocking
  __device__ __forceinline__ bool room(uint32_t tot, uint32_t& vs) {
    const uint32_t off = H % cap;
    const uint32_t start = (off + tot > cap) ? H + (cap - off) : H;
    const uint32_t end = start + tot;
    while (rel < j && (j - rel >= NDESC || end - vs_of[rel % NDESC] > cap)) {
      if (!mbar_test(&c.empty[rel % NDESC], (uint32_t)(rel / NDESC) & 1u)) return false;
      ++rel;
    }
    vs = start;
    H = end;
    return true;
  }
  __device__ __forceinline__ void issue(uint32_t vs, const unsigned char* meta, uint32_t mb, const double* vals,
                                        uint32_t vb, int np) {
    const int sl = j % NDESC;
    c.ofs[sl] = (int)(vs % cap);
    c.np[sl] = np;
    c.mb[sl] = (int)mb;
    vs_of[sl] = vs;
    mbar_arrive_expect_tx(&c.full[sl], mb + vb);
    bulk_g2s(ring + vs % cap, meta, mb, &c.full[sl]);
    if (vb) bulk_vals(ring + vs % cap + mb, vals, vb, &c.full[sl]);
    ++j;
  }
};

}  // namespace

__global__ void __launch_bounds__(NTHR, 1) patch_stream_kernel(const TMaps* __restrict__ tmg,
                                                               const DClass* __restrict__ classes,
                                                               const int* __restrict__ pclass,
                                                               const long long* __restrict__ pvals,
                                                               const int* __restrict__ porig,
                                                               const double* __restrict__ vals, int npatch,
                                                               ColorStarts cs, BoxGeom bg,
                                                               unsigned* __restrict__ done, uint32_t capA,
                                                               uint32_t capB, int box_total,
                                                               const XferEntry* __restrict__ xfer,
                                                               const long long* __restrict__ xbeg, int nbox,
                                                               unsigned long long* __restrict__ prof, int icc_only) {
  extern __shared__ __align__(128) unsigned char smraw[];
  unsigned char* ringA = smraw + BAR_BYTES;
  unsigned char* ringB = ringA + capA;
  uint64_t* vfull = reinterpret_cast<uint64_t*>(smraw + VBAR_OFS);
  uint64_t* gready = vfull + NBOX;
  uint64_t* xready = gready + NBOX;
  uint64_t* vdone = xready + NBOX;
  uint64_t* vempty = vdone + NBOX;
  const int boxd = (box_total + 15) & ~15;   // doubles per box buffer (128-byte multiple)
  double* box0 = reinterpret_cast<double*>(ringB + capB);
  double* aux = box0 + nbox * boxd;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int n = ((int)blockIdx.x < npatch) ? (npatch - (int)blockIdx.x + G - 1) / G : 0;   // patches of this CTA
  if (tid == 0) {
    for (int ch = 0; ch < 2; ++ch) {
      ChanSm c = chan_sm(smraw, ch);
      for (int s = 0; s < NDESC; ++s) {
        mbar_init(&c.full[s], 1);
        mbar_init(&c.empty[s], ch == 0 ? (icc_only ? NC + NTW : NC) : NTW);
      }
    }
    for (int b = 0; b < NBOX; ++b) {
      mbar_init(&vfull[b], 1); mbar_init(&gready[b], NC); mbar_init(&xready[b], NTW);
      mbar_init(&vdone[b], icc_only ? NC + NTW : NC); mbar_init(&vempty[b], 1);   // vempty unused
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // ================================================================== producer warps
  if (warp == WPROD_A || warp == WPROD_B) {
    // one producer per channel: a plain blocking loop over the CTA's host-built issue list
    // (abi.cpp: consumption order, absolute source pointers), the next entry prefetched
    if (lane != 0) return;
    const int ch = warp == WPROD_A ? 0 : 1;
    const ChanSm c = chan_sm(smraw, ch);
    unsigned char* ring = ch == 0 ? ringA : ringB;
    const uint32_t cap = ch == 0 ? capA : capB;
    const long long e0 = xbeg[2 * blockIdx.x + ch], e1 = xbeg[2 * blockIdx.x + ch + 1];
    uint32_t H = 0;
    int j = 0, rel = 0;
    uint32_t vs_of[NDESC];
    int4 nlo = make_int4(0, 0, 0, 0), nhi = nlo;
    if (e0 < e1) { const int4* pe = reinterpret_cast<const int4*>(xfer + e0); nlo = pe[0]; nhi = pe[1]; }
    unsigned long long t_wait = 0, t0 = prof ? clock64() : 0;
    for (long long e = e0; e < e1; ++e) {
      const int4 lo = nlo, hi = nhi;
      if (e + 1 < e1) { const int4* pe = reinterpret_cast<const int4*>(xfer + e + 1); nlo = pe[0]; nhi = pe[1]; }
      const uint32_t mb = (uint32_t)hi.x & 0xFFFFu, vb = (uint32_t)hi.y, tot = mb + vb;
      const uint32_t vs = ring_place(H, tot, cap);
      const unsigned long long ta = prof ? clock64() : 0;
      while (rel < j && (j - rel >= NDESC || H - vs_of[rel % NDESC] > cap)) {   // room: oldest released
        mbar_wait(&c.empty[rel % NDESC], (uint32_t)(rel / NDESC) & 1u);
        ++rel;
      }
      if (prof) t_wait += clock64() - ta;
      const int sl = j % NDESC;
      c.ofs[sl] = (int)(vs % cap);
      c.np[sl] = (int)(((uint32_t)hi.x >> 16) & 0x7FFFu);
      c.mb[sl] = (int)mb;
      vs_of[sl] = vs;
      const unsigned char* meta = reinterpret_cast<const unsigned char*>(((unsigned long long)(unsigned)lo.y << 32) | (unsigned)lo.x);
      const double* src = reinterpret_cast<const double*>(((unsigned long long)(unsigned)lo.w << 32) | (unsigned)lo.z);
      mbar_arrive_expect_tx(&c.full[sl], tot);
      bulk_g2s(ring + vs % cap, meta, mb, &c.full[sl]);
      if (vb) bulk_vals(ring + vs % cap + mb, src, vb, &c.full[sl]);
      ++j;
    }
    if (prof) { unsigned long long* o = prof + 24 * blockIdx.x + 12 + 2 * ch; o[0] = clock64() - t0; o[1] = t_wait; }
    return;
  }
  // ================================================================== store warp
  if (warp == WSTORE) {   // one lane: window-box loads (TMA tensor) and reductions (TMA reduce-add)
    if (lane != 0) return;
    auto load_box = [&](int i) {   // box of patch i into buffer i % nbox
      const int b = i % nbox;
      const int q = (int)blockIdx.x + i * G;
      const int* o = porig + 9 * q;
      double* vb = box0 + b * boxd;
      mbar_arrive_expect_tx(&vfull[b], (uint32_t)bg.bytes);
      tma_load_box(vb + bg.boff[0], &tmg->r[0], o[0], o[1], o[2], &vfull[b]);
      if (bg.ncomp > 1) tma_load_box(vb + bg.boff[1], &tmg->r[1], o[3], o[4], o[5], &vfull[b]);
      if (bg.ncomp > 2) tma_load_box(vb + bg.boff[2], &tmg->r[2], o[6], o[7], o[8], &vfull[b]);
    };
    for (int i = 0; i < n && i < nbox; ++i) load_box(i);
    unsigned long long st_done = 0, st_col = 0, st0 = prof ? clock64() : 0;
    for (int i = 0; i < n; ++i) {
      const int q = (int)blockIdx.x + i * G;
      const int b = i % nbox;
      unsigned long long ta = prof ? clock64() : 0;
      mbar_wait(&vdone[b], (uint32_t)(i / nbox) & 1u);
      if (prof) { const unsigned long long tb = clock64(); st_done += tb - ta; ta = tb; }
      const int col = color_of(q, cs);
      if (col > 0) {
        const unsigned need = (unsigned)cs.start[col];
        while (ld_acquire(done) < need) __nanosleep(64);
      }
      if (prof) st_col += clock64() - ta;
      const int* o = porig + 9 * q;
      const double* vb = box0 + b * boxd;
      tma_reduce_box(&tmg->c[0], o[0], o[1], o[2], vb + bg.boff[0]);
      if (bg.ncomp > 1) tma_reduce_box(&tmg->c[1], o[3], o[4], o[5], vb + bg.boff[1]);
      if (bg.ncomp > 2) tma_reduce_box(&tmg->c[2], o[6], o[7], o[8], vb + bg.boff[2]);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (i + nbox < n) load_box(i + nbox);   // the buffer has been read: reload it
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence();
      atomicAdd(done, 1u);
    }
    if (prof) {
      unsigned long long* o = prof + 24 * blockIdx.x;
      o[2] = clock64() - st0; o[3] = st_done; o[4] = st_col;
    }
    return;
  }
  // ================================================================== tile warps
  // (families whose classes all end in ICC (ICC-SC) have no tile work: the tile warps join the
  // sparse warps instead, icc_only)
  if (warp >= WT0 && !icc_only) {
    const int tw = warp - WT0;
    Consumer ct{chan_sm(smraw, 1), ringB, 0, 0, nullptr, nullptr};
    unsigned long long tt_wait = 0, tt0 = prof ? clock64() : 0;
    for (int i = 0; i < n; ++i) {
      const int q = (int)blockIdx.x + i * G;
      const DClass& C = classes[pclass[q]];
      const int b = i % nbox;
      double* v = box0 + b * boxd;
      unsigned long long ta = (prof && tw == 0 && lane == 0) ? clock64() : 0;
      mbar_wait(&gready[b], (uint32_t)(i / nbox) & 1u);   // forward(i) done
      if (prof && tw == 0 && lane == 0) tt_wait += clock64() - ta;
      if (C.fin_tiles) {
        const int m = C.m;
        const int T = (m + 31) >> 5, mpad = 32 * T;
        double* g = aux;                                                // padded copy of v_F
        double* parts = aux + mpad;                                     // per-tile-warp partials
        uint16_t* fb = reinterpret_cast<uint16_t*>(parts + NTW * mpad);   // final-block boxes
        const int tt = tid - 32 * WT0;   // 0 .. 32*NTW-1
        {
          const Piece_ pc = ct.acquire();   // FINAL piece: boxes of the final block
          const uint16_t* fbs = reinterpret_cast<const uint16_t*>(pc.pb + 16);
          for (int jj = tt; jj < mpad; jj += 32 * NTW) {
            const int bx = (jj < m) ? fbs[jj] : 0;
            fb[jj] = (uint16_t)bx;
            g[jj] = (jj < m) ? v[bx] : 0.0;
          }
          for (int jj = lane; jj < mpad; jj += 32) parts[tw * mpad + jj] = 0.0;
          ct.release(lane);
        }
        tsync();
        // whole tiles per warp (tile t of the patch -> tile warp t % NTW), lane-block layout
        // (patches.hpp): 16 conflict-free LDS.128 and 64 independent DFMA per lane and tile
        double* mypart = parts + tw * mpad;
        for (int pi = C.tile_p0 + 1; pi < C.tile_p1; ++pi) {
          const Piece_ pc = ct.acquire();
          if (((pi - C.tile_p0 - 1) % NTW) == tw) {
            const Hdr h = hdr(pc.pb);
            tile_gemv(pc.val, g, mypart, h.a0, h.a1, lane);
          }
          ct.release(lane);
        }
        tsync();
        for (int jj = tt; jj < m; jj += 32 * NTW) {
          double x = 0.0;
#pragma unroll
          for (int w = 0; w < NTW; ++w) x += parts[w * mpad + jj];
          v[fb[jj]] = x;
        }
        tsync();   // aux is reused by the next patch
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&xready[b]);
    }
    if (prof && tw == 0 && lane == 0) {
      unsigned long long* o = prof + 24 * blockIdx.x;
      o[5] = clock64() - tt0; o[6] = tt_wait;
    }
    return;
  }
  // ================================================================== sparse warps
  Consumer cn{chan_sm(smraw, 0), ringA, 0, 0, nullptr, nullptr};
  unsigned long long sp_box = 0, sp_x = 0, sp_fwd = 0, sp_bwd = 0, sp0 = prof ? clock64() : 0;
  const bool pf = prof != nullptr && tid == 0;
  unsigned long long sp_acq = 0, sp_piv = 0, sp_w = 0, sp_sync = 0;
  const int ncw = icc_only ? NC + NTW : NC, nct = 32 * ncw;   // consumer warps / threads
  auto csync_n = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(nct) : "memory"); };
  auto forward = [&](int i) {
    const int q = (int)blockIdx.x + i * G;
    const DClass& C = classes[pclass[q]];
    const int b = i % nbox;
    double* v = box0 + b * boxd;
    unsigned long long ta = pf ? clock64() : 0;
    mbar_wait(&vfull[b], (uint32_t)(i / nbox) & 1u);   // the window box of r has landed
    if (pf) { const unsigned long long tb = clock64(); sp_box += tb - ta; ta = tb; }
    const int nlev = C.nlev;
    for (int l = 0; l < nlev; ++l) {
      const DLevel& L = C.lev[l];
      const int bs = L.blk.bs;
      // y^_E = L^{-T} L^{-1} v_E in place (pivot blocks <= 3x3, diagonal stored inverted)
      for (int pi = L.piv_b; pi < L.w_b; ++pi) {
        unsigned long long tq = pf ? clock64() : 0;
        const Piece_ pc = cn.acquire();
        if (pf) { const unsigned long long t2 = clock64(); sp_acq += t2 - tq; tq = t2; }
        const Hdr h = hdr(pc.pb);
        const uint16_t* mem = reinterpret_cast<const uint16_t*>(pc.pb + 16);
        const double* pv = pc.val;
        const int cnt = h.a1 - h.a0;
        for (int li = tid; li < cnt; li += NT) {
          const int m0 = mem[li];
          if (bs == 1) {
            const double d = pv[li];
            v[m0] *= d * d;
            continue;
          }
          const int m1 = mem[cnt + li];
          const int m2 = (bs > 2) ? mem[2 * cnt + li] : 0xFFFF;
          const double l00 = pv[li], l10 = pv[cnt + li], l11 = pv[2 * cnt + li];
          double y0 = v[m0] * l00, y1 = 0.0, y2 = 0.0;
          if (m1 != 0xFFFF) y1 = (v[m1] - l10 * y0) * l11;
          if (m2 != 0xFFFF) {
            const double l20 = pv[3 * cnt + li], l21 = pv[4 * cnt + li], l22 = pv[5 * cnt + li];
            y2 = (v[m2] - l20 * y0 - l21 * y1) * l22;
            y2 *= l22;
            v[m2] = y2;
            if (m1 != 0xFFFF) y1 -= l21 * y2;
            y0 -= l20 * y2;
          }
          if (m1 != 0xFFFF) {
            y1 *= l11;
            v[m1] = y1;
            y0 -= l10 * y1;
          }
          v[m0] = y0 * l00;
        }
        cn.release(lane);
        if (pf) sp_piv += clock64() - tq;
      }
      { const unsigned long long tq = pf ? clock64() : 0; csync_n(); if (pf) sp_sync += clock64() - tq; }
      for (int pi = L.w_b; pi < L.w_e; ++pi) {
        unsigned long long tq = pf ? clock64() : 0;
        const Piece_ pc = cn.acquire();
        if (pf) { const unsigned long long t2 = clock64(); sp_acq += t2 - tq; tq = t2; }
        sliced_piece(pc, v, L.w.nrows, warp, lane, [&](int rb, double acc) { v[rb] -= acc; });
        cn.release(lane);
        if (pf) sp_w += clock64() - tq;
      }
      { const unsigned long long tq = pf ? clock64() : 0; csync_n(); if (pf) sp_sync += clock64() - tq; }
    }
    __syncwarp();
    if (lane == 0 && !icc_only) mbar_arrive(&gready[b]);   // the tile warps may read v_F
    if (pf) sp_fwd += clock64() - ta;
  };
  auto backward = [&](int i) {
    const int q = (int)blockIdx.x + i * G;
    const DClass& C = classes[pclass[q]];
    const int b = i % nbox;
    double* v = box0 + b * boxd;
    unsigned long long ta = pf ? clock64() : 0;
    if (!icc_only) mbar_wait(&xready[b], (uint32_t)(i / nbox) & 1u);   // tiles(i) done (or skipped)
    if (pf) { const unsigned long long tb = clock64(); sp_x += tb - ta; ta = tb; }
    if (C.final_kind != 0) {
      // ICC(0) on the final block: forward rows of L by levels (diag last, stored inverted),
      // then backward rows of L^T by levels (diag first); rows of one level are independent.
      // meta = uint16 row boxes, uint16 value starts (cnt + 1), uint16 column boxes
      for (int pass = 0; pass < 2; ++pass) {
        const int nl = pass == 0 ? C.iccf_nlev : C.iccb_nlev;
        const int* lp = pass == 0 ? C.iccf_lp : C.iccb_lp;
        for (int l = 0; l < nl; ++l) {
          const int pe = lp[l + 1];
          for (int pi = lp[l]; pi < pe; ++pi) {
            const Piece_ pc = cn.acquire();
            // multi-chunk ICC piece (patches.cpp): chunk c (<= 32 rows, lane-interleaved) is
            // taken by consumer warp c; one header and one table entry per warp and piece
            // chunk c of the level's piece k is taken by warp c + kIccChunks (k % groups): several
            // pieces in work at once (and in flight in the ring)
            const Hdr h = hdr(pc.pb);
            const int ch = warp - kIccChunksDev * ((pi - lp[l]) % (NC / kIccChunksDev));
            if (ch >= 0 && ch < h.a1 - h.a0) {
              const int4 ent = reinterpret_cast<const int4*>(pc.pb + 16)[ch];   // cnt, L, meta, values
              const int cnt = ent.x, Lm = ent.y;
              if (lane < cnt) {
                const uint16_t* rows = reinterpret_cast<const uint16_t*>(pc.pb + ent.z);
                const uint16_t* cols = rows + 32 + lane;
                const double* dgv = pc.val + ent.w;
                const double* off = dgv + 32 + lane;
                const int a = rows[lane];
                double s0 = v[a], s1 = 0.0;
                int j = 0;
                for (; j + 3 < Lm; j += 4) {   // step j of this row: conflict-free value / column loads
                  const int c0 = cols[32 * j], c1 = cols[32 * j + 32], c2 = cols[32 * j + 64], c3 = cols[32 * j + 96];
                  const double w0 = off[32 * j], w1 = off[32 * j + 32], w2 = off[32 * j + 64], w3 = off[32 * j + 96];
                  const double x0 = v[c0], x1 = v[c1], x2 = v[c2], x3 = v[c3];
                  s0 = fma(-w0, x0, s0);
                  s1 = fma(-w1, x1, s1);
                  s0 = fma(-w2, x2, s0);
                  s1 = fma(-w3, x3, s1);
                }
                for (; j < Lm; ++j) {
                  const double x = v[cols[32 * j]];
                  if (j & 1) s1 = fma(-off[32 * j], x, s1);
                  else s0 = fma(-off[32 * j], x, s0);
                }
                v[a] = (s0 + s1) * dgv[lane];
              }
            }
            cn.release(lane);
          }
          csync_n();
        }
      }
    }
    // x_E = y^_E - W^ x_R  (W^ = P_EE^{-1} P_ER, in place)
    for (int l = C.nlev - 1; l >= 0; --l) {
      const DLevel& L = C.lev[l];
      for (int pi = L.wt_b; pi < L.wt_e; ++pi) {
        const Piece_ pc = cn.acquire();
        sliced_piece(pc, v, L.wt.nrows, warp, lane, [&](int rb, double acc) { v[rb] -= acc; });
        cn.release(lane);
      }
      csync_n();
    }
    {   // zero the box entries outside the patch, hand the box to the store warp
      const Piece_ pc = cn.acquire();   // ZERO piece
      const Hdr h = hdr(pc.pb);
      const uint16_t* zl = reinterpret_cast<const uint16_t*>(pc.pb + 16);
      for (int k = tid; k < h.a1 - h.a0; k += nct) v[zl[k]] = 0.0;
      cn.release(lane);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> TMA reads
    __syncwarp();
    if (lane == 0) mbar_arrive(&vdone[b]);
    if (pf) sp_bwd += clock64() - ta;
  };
  if (nbox >= 2) {   // pipelined: forward(i+1) runs while the tiles of patch i are in flight
    if (n > 0) forward(0);
    for (int i = 0; i < n; ++i) {
      if (i + 1 < n) forward(i + 1);
      backward(i);
    }
  } else {           // one box buffer (very large windows): box i+1 arrives after patch i is reduced
    for (int i = 0; i < n; ++i) {
      forward(i);
      backward(i);
    }
  }
  if (pf) {
    unsigned long long* o = prof + 24 * blockIdx.x;
    o[7] = clock64() - sp0; o[8] = sp_box; o[9] = sp_x; o[10] = sp_fwd; o[11] = sp_bwd;
    o[16] = sp_acq; o[17] = sp_piv; o[18] = sp_w; o[19] = sp_sync;

  }
}

namespace {

// ===================================================================== class-batched patch solve
// Families whose patches share few value blocks (uniform Cartesian meshes: cfg1, cfg3, cfg4 have
// 27 to 54 distinct blocks for 10^4 .. 10^5 patches) keep their blocks in L2, and the stream kernel
// above is then latency-bound: one right-hand side per elimination level, the same block re-read
// per patch (cfg4 potential family, RM_PROFILE: ~36 us per patch and SM, producers waiting for
// ring room 75% of the time).  Here one CTA takes B patches of ONE value block and runs the same
// elimination program -- the class's stream pieces, read straight from global memory / L2 -- on
// all B at once: every value and index is loaded once per B patches, and every lane carries B
// independent FMA chains.  The B window boxes are interleaved in shared memory (box entry e of
// patch b at X[e B + b]); gather and scatter are plain coalesced loads and fp64 atomic adds of
// the NONZERO box entries: within a colour the patches are disjoint and the box entries outside a
// patch are zeroed first (ZERO piece), so every c entry receives at most one nonzero addend per
// launch -- deterministic.  One launch per colour (the stream kernel's colour order).  The dense
// final block is applied with the full symmetric inverse (row-major mr x mr, host-expanded from the
// half-stored tiles): one coalesced column read per row, B vectors per read.
// threads per CTA NT: 512 (one CTA per SM) or 256 (two CTAs per SM: one CTA's TMA / barrier phases
// overlap the other's elimination)

struct BatchArgs {
  const DClass* classes;
  const double* vals;
  const double* fin;
  const int* bpatch;
  const int* bclass;
  const long long* bblock;
  const long long* bfin;
  const int* porig;
  const TMaps* tm;                              // the family's r / c tensor maps (one per sub-box)
  int nsub, boxd, gofs, pofs, tofs;             // sub-boxes; box stride; G / partials / piece-table offsets (doubles)
  int boff[3];
  unsigned box_bytes;                           // bytes of one patch's window box (all sub-boxes)
};

// one sliced-ELL piece (W or WT) on the B boxes (stride boxd): slice s owned by warp s % BW.  The
// values and indices come from global memory (L2): steps of U entries per lane with every load
// of a step issued before its first use (predicated tail; the slice length is warp-uniform)
template <int B, int BW>
__device__ __forceinline__ void batch_sliced(const unsigned char* pb, const double* __restrict__ val, int nrows,
                                             int warp, int lane, double* __restrict__ X, int boxd) {
#ifndef RM_BATCH_U
#define RM_BATCH_U 4
#endif
  constexpr int U = RM_BATCH_U;   // entries per lane and step (measured at cfg4: U = 2 10.2 ms, 4 9.35 ms, 8 9.82 ms, 16 10.4 ms)
  const Hdr h = hdr(pb);
  const int nsl = h.a1 - h.a0;
  const uint32_t* si = reinterpret_cast<const uint32_t*>(pb + 16);
  const uint16_t* rows = reinterpret_cast<const uint16_t*>(si + nsl);
  const uint16_t* cols = rows + 32 * nsl;
#ifndef RM_BATCH_SLICES
#define RM_BATCH_SLICES 1   // slices a warp works on at once when B <= 2 (B = 4: 2; 1: the look-ahead loop).
                            // Measured (pass AP, cfg4): 1: 8.82 ms, 2: 10.0 ms, 4: 12.5 ms -- the look-ahead wins
#endif
#if RM_BATCH_SLICES > 1 && !defined(RM_BATCH_NOPIPE)
  // ncu (pass AO, cfg4 NCE8 edge-star potential family): a level has ~3.5 slices per warp of
  // ~1.4 steps each, every step one L2 round trip (header word -> values / columns), and the
  // FMAs of a step are far shorter than the trip -- long-scoreboard stalls dominate.  The warp
  // therefore takes S slices at once: S header words in one trip, the first steps of all S in
  // the next, further steps (the longest slice counts) again S at a time.  Each row still sums
  // its entries in order: bitwise the one-slice sums.
  constexpr int S = B <= 2 ? RM_BATCH_SLICES : (B <= 4 ? (RM_BATCH_SLICES > 2 ? 2 : RM_BATCH_SLICES) : 1);
  for (int l0 = (warp - h.a0 % BW + BW) % BW; l0 < nsl; l0 += S * BW) {
    int st[S], cnt[S], rb[S];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const int ls = l0 + q * BW;
      const uint32_t info = ls < nsl ? si[ls] : 0u;
      st[q] = 32 * (int)(info & 0xFFFFu) + lane;
      cnt[q] = (int)(info >> 16);
    }
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const int ls = l0 + q * BW;
      rb[q] = ls < nsl && (h.a0 + ls) * 32 + lane < nrows ? (int)rows[ls * 32 + lane] : -1;
    }
    double acc[S][B];
#pragma unroll
    for (int q = 0; q < S; ++q)
#pragma unroll
      for (int b = 0; b < B; ++b) acc[q][b] = 0.0;
    int cmax = 0;
#pragma unroll
    for (int q = 0; q < S; ++q) cmax = max(cmax, cnt[q]);
    for (int kk = 0; kk < cmax; kk += U) {
      double w[S][U];
      int c[S][U];
#pragma unroll
      for (int q = 0; q < S; ++q)
#pragma unroll
        for (int j = 0; j < U; ++j) {
          const bool on = kk + j < cnt[q];
          const int e = st[q] + (kk + j) * 32;
          w[q][j] = on ? __ldg(val + e) : 0.0;
          c[q][j] = on ? (int)cols[e] : 0;
        }
#pragma unroll
      for (int q = 0; q < S; ++q)
        if (kk < cnt[q]) {
#pragma unroll
          for (int j = 0; j < U; ++j)
#pragma unroll
            for (int b = 0; b < B; ++b) acc[q][b] = fma(w[q][j], X[b * boxd + c[q][j]], acc[q][b]);
        }
    }
#pragma unroll
    for (int q = 0; q < S; ++q)
      if (rb[q] >= 0) {
#pragma unroll
        for (int b = 0; b < B; ++b) X[b * boxd + rb[q]] -= acc[q][b];
      }
  }
#elif !defined(RM_BATCH_NOPIPE)
  // the warp's (slice, step) pairs form ONE stream with a one-step look-ahead: the values and
  // columns of the next step -- of this slice or of the warp's next one, whose header word was
  // fetched a slice earlier -- are requested before the FMAs of the current step, so the L2
  // latency of a step overlaps the arithmetic of the step before it instead of following it
  // (same addends in the same order: bitwise the unpipelined sums)
#ifdef RM_BATCH_SERP
  // serpentine slice -> warp map (round r of BW slices: warp i takes slice i in even rounds,
  // BW - 1 - i in odd ones): the slices of a sorted sliced-ELL piece shorten with their index,
  // and plain round-robin gives warp 0 the longest slice of every round
  auto at = [&](int r) { return r * BW + ((r & 1) ? BW - 1 - warp : warp) - h.a0; };
  auto nxt = [&](int l) { return at((h.a0 + l) / BW + 1); };
  int ls = at(h.a0 / BW);
  if (ls < 0) ls = at(h.a0 / BW + 1);
#else
  auto nxt = [&](int l) { return l + BW; };
  int ls = (warp - h.a0 % BW + BW) % BW;
#endif
  if (ls >= nsl) return;
  uint32_t info = si[ls];
  uint32_t info_n = nxt(ls) < nsl ? si[nxt(ls)] : 0u;
  int rb = rows[ls * 32 + lane];
  int kk = 0;
  double w[U];
  int c[U];
  {
    const int st = 32 * (int)(info & 0xFFFFu) + lane, cnt = (int)(info >> 16);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const bool on = j < cnt;
      const int e = st + j * 32;
      w[j] = on ? __ldg(val + e) : 0.0;
      c[j] = on ? (int)cols[e] : 0;
    }
  }
  double acc[B];
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.0;
  for (;;) {
    const int cnt = (int)(info >> 16);
    const bool last = kk + U >= cnt;   // the slice's last step
    const int ls2 = last ? nxt(ls) : ls, kk2 = last ? 0 : kk + U;
    const uint32_t info2 = last ? info_n : info;
    const bool more = ls2 < nsl;
    double w2[U];
    int c2[U];
    {
      const int st2 = 32 * (int)(info2 & 0xFFFFu) + lane, cnt2 = more ? (int)(info2 >> 16) : 0;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const bool on = kk2 + j < cnt2;
        const int e = st2 + (kk2 + j) * 32;
        w2[j] = on ? __ldg(val + e) : 0.0;
        c2[j] = on ? (int)cols[e] : 0;
      }
    }
    int rb2 = rb;
    uint32_t info_n2 = info_n;
    if (last && more) {
      rb2 = rows[ls2 * 32 + lane];
      info_n2 = nxt(ls2) < nsl ? si[nxt(ls2)] : 0u;
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = fma(w[j], X[b * boxd + c[j]], acc[b]);
    if (last) {
      if ((h.a0 + ls) * 32 + lane < nrows) {
#pragma unroll
        for (int b = 0; b < B; ++b) X[b * boxd + rb] -= acc[b];
      }
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = 0.0;
    }
    if (!more) break;
    ls = ls2; kk = kk2; info = info2; info_n = info_n2; rb = rb2;
#pragma unroll
    for (int j = 0; j < U; ++j) { w[j] = w2[j]; c[j] = c2[j]; }
  }
#else   // the unpipelined loop (tuning reference: -DRM_BATCH_NOPIPE)
  for (int ls = (warp - h.a0 % BW + BW) % BW; ls < nsl; ls += BW) {
    const uint32_t info = si[ls];
    const int st = 32 * (int)(info & 0xFFFFu) + lane, cnt = (int)(info >> 16);
    const int rb = rows[ls * 32 + lane];
    double acc[B];
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = 0.0;
    for (int kk = 0; kk < cnt; kk += U) {
      double w[U];
      int c[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const bool on = kk + j < cnt;
        const int e = st + (kk + j) * 32;
        w[j] = on ? __ldg(val + e) : 0.0;
        c[j] = on ? (int)cols[e] : 0;
      }
#pragma unroll
      for (int j = 0; j < U; ++j)
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = fma(w[j], X[b * boxd + c[j]], acc[b]);
    }
    if ((h.a0 + ls) * 32 + lane < nrows) {
#pragma unroll
      for (int b = 0; b < B; ++b) X[b * boxd + rb] -= acc[b];
    }
  }
#endif
}

#ifndef RM_BATCH_CHAINF
#define RM_BATCH_CHAINF 0   // 1: the colour chain continues across the orientation families of a space (measured without
                            // timing events, pass BA: cfg3 3.066 vs 3.033 ms, cfg4 8.364 vs 8.395 ms -- no gain, left off)
#endif
#ifndef RM_BATCH_PDL
#define RM_BATCH_PDL 1   // colours c >= 1 of a family as programmatic dependent launches (0: plain stream order)
#endif
// MINB: resident CTAs per SM the register allocation allows (512 threads: 1; 256 threads: 2, or 3
// for the families whose working set leaves room for a third CTA -- 24 warps per SM at <= 85 registers)
template <int B, int BT, int MINB>
#ifdef RM_BATCH_512X2   // tuning: two 512-thread CTAs per SM (32 warps, 64 registers per thread)
__global__ void __launch_bounds__(BT, MINB < 2 ? 2 : MINB) patch_batch_kernel(
#else
__global__ void __launch_bounds__(BT, MINB) patch_batch_kernel(
#endif
    const __grid_constant__ BatchArgs a, int batch0) {
  constexpr int BW = BT / 32;
  extern __shared__ __align__(128) double smb[];
  __shared__ int sq[B];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bt = batch0 + (int)blockIdx.x;
  const int boxd = a.boxd;
  double* X = smb;   // box of slot b at X + b * boxd (the TMA box layout)
#if RM_BATCH_PDL
  // let the next colour's CTAs take the SM slots this launch's last wave leaves idle (they block
  // at their reduce-add until this grid is complete)
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  if (tid < B) sq[tid] = a.bpatch[(long long)bt * B + tid];
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // ---- gather: the window boxes of r by TMA tensor copies (out-of-domain entries zero-filled)
  if (tid == 0) {
    int nv = 0;
    for (int b = 0; b < B; ++b) nv += sq[b] >= 0;
    mbar_arrive_expect_tx(&bar, (uint32_t)nv * a.box_bytes);
    for (int b = 0; b < B; ++b) {
      if (sq[b] < 0) continue;
      const int* o = a.porig + 9LL * sq[b];
      for (int sb = 0; sb < a.nsub; ++sb)
        tma_load_3d(X + b * boxd + a.boff[sb], &a.tm->r[sb], o[3 * sb], o[3 * sb + 1], o[3 * sb + 2], &bar);
    }
  }
  const DClass& C = a.classes[a.bclass[bt]];
  // the class program's piece table {meta offset, value offset} in shared memory
  int2* ptab = reinterpret_cast<int2*>(smb + a.tofs);
  for (int i = tid; i < C.npieces; i += BT) ptab[i] = C.ptab[i];
  const unsigned char* const meta = C.meta;
  const double* const vblk = a.vals + a.bblock[bt];
  __syncthreads();
  mbar_wait(&bar, 0u);
  const int nlev = C.nlev;
  for (int l = 0; l < nlev; ++l) {   // forward
    const DLevel& L = C.lev[l];
    const int bs = L.blk.bs;
    for (int pi = L.piv_b; pi < L.w_b; ++pi) {   // y^_E = L^{-T} L^{-1} v_E (pivot blocks <= 3x3)
      const int2 pt = ptab[pi];
      const unsigned char* mc = meta + pt.x;
      const Hdr h = hdr(mc);
      const uint16_t* mem = reinterpret_cast<const uint16_t*>(mc + 16);
      const double* pv = vblk + pt.y;
      const int cnt = h.a1 - h.a0;
      // PU iterations at a time, every index and factor load of all PU issued before the first
      // dependent shared-memory access (pass AO: ~3 iterations per thread and level, each one
      // L2 round trip when taken one after the other)
      constexpr int PU = 3;
      for (int t0 = tid; t0 < cnt * B; t0 += PU * BT) {
        int m0[PU], m1[PU], m2[PU];
        double f0[PU], f1[PU], f2[PU], f3[PU], f4[PU], f5[PU];
#pragma unroll
        for (int u = 0; u < PU; ++u) {
          const int t = t0 + u * BT;
          const bool on = t < cnt * B;
          const int li = on ? t / B : 0;
          m0[u] = on ? (int)mem[li] : -1;
          f0[u] = __ldg(pv + li);
          m1[u] = m2[u] = 0xFFFF;
          f1[u] = f2[u] = f3[u] = f4[u] = f5[u] = 0.0;
          if (bs > 1) {
            m1[u] = mem[cnt + li];
            f1[u] = __ldg(pv + cnt + li);
            f2[u] = __ldg(pv + 2 * cnt + li);
            if (bs > 2) {
              m2[u] = mem[2 * cnt + li];
              f3[u] = __ldg(pv + 3 * cnt + li);
              f4[u] = __ldg(pv + 4 * cnt + li);
              f5[u] = __ldg(pv + 5 * cnt + li);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < PU; ++u) {
          if (m0[u] < 0) continue;
          const int t = t0 + u * BT;
          double* Xb = X + (t % B) * boxd;
          if (bs == 1) {
            const double d = f0[u];
            Xb[m0[u]] *= d * d;
            continue;
          }
          const double l00 = f0[u], l10 = f1[u], l11 = f2[u];
          double y0 = Xb[m0[u]] * l00, y1 = 0.0, y2 = 0.0;
          if (m1[u] != 0xFFFF) y1 = (Xb[m1[u]] - l10 * y0) * l11;
          if (m2[u] != 0xFFFF) {
            const double l20 = f3[u], l21 = f4[u], l22 = f5[u];
            y2 = (Xb[m2[u]] - l20 * y0 - l21 * y1) * l22;
            y2 *= l22;
            Xb[m2[u]] = y2;
            if (m1[u] != 0xFFFF) y1 -= l21 * y2;
            y0 -= l20 * y2;
          }
          if (m1[u] != 0xFFFF) {
            y1 *= l11;
            Xb[m1[u]] = y1;
            y0 -= l10 * y1;
          }
          Xb[m0[u]] = y0 * l00;
        }
      }
    }
    __syncthreads();
    for (int pi = L.w_b; pi < L.w_e; ++pi) {   // v_R -= P_RE y^_E
      const int2 pt = ptab[pi];
      batch_sliced<B, BW>(meta + pt.x, vblk + pt.y, L.w.nrows, warp, lane, X, boxd);
    }
    __syncthreads();
  }
  const int m = C.m;
  if (m > 0) {   // x_F = S_F^{-1} v_F with the full inverse
    const uint16_t* fbs = reinterpret_cast<const uint16_t*>(meta + ptab[C.tile_p0].x + 16);   // FINAL piece: final-block boxes
    const int mr = (m + 31) & ~31;
    double* G = smb + a.gofs;
    double* PT = smb + a.pofs;
    for (int t = tid; t < m * B; t += BT) {
      const int j = t / B, b = t - j * B;
      G[t] = X[b * boxd + fbs[j]];
    }
    __syncthreads();
    const double* S = a.fin + a.bfin[bt];
    const int ns = mr < BT ? BT / mr : 1;   // column segments per row (partials summed below)
    const int seg = (m + ns - 1) / ns;
    for (int t = tid; t < ns * mr; t += BT) {
      const int hs = t / mr, r = t - hs * mr;
      double acc[B];
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = 0.0;
      if (r < m) {
        // columns of row r's independent block only (the inverse is block diagonal in the final
        // order, patches.cpp frange): the edge-star final blocks split into ~p blocks
        int c0 = hs * seg, c1 = min(m, c0 + seg);
        if (C.frange) {
          const int2 fr = C.frange[r];
          c0 = max(c0, fr.x);
          c1 = min(c1, fr.y);
        }
        const double* Sr = S + r;
        for (int c = c0; c < c1; c += 8) {   // 8 column loads in flight, predicated tail
          double s[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) s[j] = c + j < c1 ? __ldg(Sr + (long long)(c + j) * mr) : 0.0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const double2* g2 = reinterpret_cast<const double2*>(G + min(c + j, c1 - 1) * B);
#pragma unroll
            for (int b = 0; b < B / 2; ++b) {
              const double2 gv = g2[b];
              acc[2 * b] = fma(s[j], gv.x, acc[2 * b]);
              acc[2 * b + 1] = fma(s[j], gv.y, acc[2 * b + 1]);
            }
          }
        }
      }
#pragma unroll
      for (int b = 0; b < B; ++b) PT[t * B + b] = acc[b];
    }
    __syncthreads();
    for (int t = tid; t < m * B; t += BT) {
      const int r = t / B, b = t - r * B;
      double s = 0.0;
      for (int hs = 0; hs < ns; ++hs) s += PT[(hs * mr + r) * B + b];
      X[b * boxd + fbs[r]] = s;
    }
    __syncthreads();
  }
  for (int l = nlev - 1; l >= 0; --l) {   // backward: x_E = y^_E - (P_EE^{-1} P_ER) x_R
    const DLevel& L = C.lev[l];
    for (int pi = L.wt_b; pi < L.wt_e; ++pi) {
      const int2 pt = ptab[pi];
      batch_sliced<B, BW>(meta + pt.x, vblk + pt.y, L.wt.nrows, warp, lane, X, boxd);
    }
    __syncthreads();
  }
  {   // ZERO piece (the last): box entries that are not DoFs of the patch
    const unsigned char* mc = meta + ptab[C.npieces - 1].x;
    const Hdr h = hdr(mc);
    const uint16_t* zl = reinterpret_cast<const uint16_t*>(mc + 16);
    const int cnt = h.a1 - h.a0;
    constexpr int ZU = 4;   // index loads in flight per thread
    for (int t0 = tid; t0 < cnt * B; t0 += ZU * BT) {
      int z[ZU];
#pragma unroll
      for (int u = 0; u < ZU; ++u) {
        const int t = t0 + u * BT;
        z[u] = t < cnt * B ? (t % B) * boxd + (int)zl[t / B] : -1;
      }
#pragma unroll
      for (int u = 0; u < ZU; ++u)
        if (z[u] >= 0) X[z[u]] = 0.0;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> TMA reads
  __syncthreads();
  // ---- scatter: TMA tensor reduce-add of every box into c (fp64 add per element; within a
  // colour the patches are disjoint and the entries outside a patch are zero, so every c entry
  // receives at most one nonzero addend per launch: deterministic)
  if (tid == 0) {
#if RM_BATCH_PDL
    // the previous colour's launch (programmatic dependent launch, launch_batched) must be complete
    // and its reduce-adds visible before this colour adds into c: same order of addends as with
    // plain stream order.  Everything above reads only r and the class data, final before colour 0
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
    for (int b = 0; b < B; ++b) {
      if (sq[b] < 0) continue;
      const int* o = a.porig + 9LL * sq[b];
      for (int sb = 0; sb < a.nsub; ++sb)
        tma_reduce_add_3d(&a.tm->c[sb], o[3 * sb], o[3 * sb + 1], o[3 * sb + 2], X + b * boxd + a.boff[sb]);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // complete before the next colour's launch
  }
}

size_t batch_smem_t(int B, int NT, int box_total, int mr_max) {
  const size_t boxd = (size_t)((box_total + 15) & ~15);
  const size_t mr = (size_t)((mr_max + 31) & ~31);
  return sizeof(double) * (B * (boxd + mr + std::max<size_t>(NT, mr)) + kBatchMaxPieces);   // + piece table (int2)
}

// rp = pad(r): one (y, z) row of one component per warp, grid-stride (the per-element 64-bit
// divisions of a thread-per-entry pad dominated it); the pad column is written as zero
__global__ void pad_kernel(const __grid_constant__ PadLayout P, const double* __restrict__ r, double* __restrict__ rp,
                           long long npad) {
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * (blockDim.x >> 5);
  int rows_before = 0;
  for (int m = 0; m < P.ncomp; ++m) {
    const int Lx = (int)P.len[m][0], Lxp = (int)P.lxp[m], nrow = (int)(P.len[m][1] * P.len[m][2]);
    for (int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) - rows_before; row < nrow; row += wstride) {
      if (row < 0) continue;
      const double* src = r + P.off[m] + (long long)row * Lx;
      double* dst = rp + P.poff[m] + (long long)row * Lxp;
      for (int x = lane; x < Lxp; x += 32) dst[x] = x < Lx ? src[x] : 0.0;
    }
    rows_before += nrow;
  }
  (void)npad;
}

__global__ void unpad_axpy_kernel(const __grid_constant__ PadLayout P, const double* __restrict__ cp, double* u,
                                  double omega, long long n, int skip_p, const double* uin) {
  // u = (uin ? uin : u) + omega * unpad(cp): out of place the sweep needs no u_out = u_in copy
  // one (y, z) row of one component per warp, grid-stride: no per-element 64-bit division;
  // skip_p > 0 (one component, static condensation with the post step writing u): the cell
  // interiors are already done, only the skeleton entries (an index at a multiple of p) remain
  const int lane = threadIdx.x & 31;
  const int wstride = gridDim.x * (blockDim.x >> 5);
  int rows_before = 0;
  for (int m = 0; m < P.ncomp; ++m) {
    const int Lx = (int)P.len[m][0], Ly = (int)P.len[m][1], nrow = (int)(P.len[m][1] * P.len[m][2]);
    for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) - rows_before; r < nrow; r += wstride) {
      if (r < 0) continue;
      const long long ub = P.off[m] + (long long)r * Lx, cb = P.poff[m] + (long long)r * P.lxp[m];
      if (skip_p > 0 && (r % Ly) % skip_p != 0 && (r / Ly) % skip_p != 0) {   // interior row: x skeleton only
        for (int x = lane * skip_p; x < Lx; x += 32 * skip_p) u[ub + x] = (uin ? uin[ub + x] : u[ub + x]) + omega * cp[cb + x];
        continue;
      }
      for (int x = lane; x < Lx; x += 32) u[ub + x] = (uin ? uin[ub + x] : u[ub + x]) + omega * cp[cb + x];
    }
    rows_before += nrow;
  }
  (void)n;
}

// ---- static condensation of the cell interiors (ICC-SC families, k = 0), on the padded layout
#ifndef RM_SCC_THREADS   // CTA sizes of the SC pre / post steps (tuning knobs)
#define RM_SCC_THREADS 256
#endif
#ifndef RM_SCP_THREADS   // measured: 128 / 256 / 512 -> cfg5 patch stage 1.560 / 1.572 / 1.652 ms
#define RM_SCP_THREADS 128
#endif
// pre:  rp[f] -= sum over the 2 cells K at face DoF f, sum_i c_K(f, I) dinv_K(I) rp[I]   (one thread per face DoF)
// post: cp[I] = n_K dinv_K(I) rp[I] - dinv_K(I) sum_faces c_K(f, I) cp[f]               (one thread per interior DoF)
struct ScGeom {
  int p, n[3];
  long long lxp, ly;
  int cmp;                          // couplings from the interior stiffness weights (sc_w)
  double kd[16], k0[16], kp[16];    // D_ii, D_i0, D_ip
};


__device__ __forceinline__ long long sc_idx(const ScGeom& G, long long x, long long y, long long z) {
  return (z * G.ly + y) * G.lxp + x;
}

// ICC-SC pre step, part 1 (one CTA per cell K): y_I = P_II^{-1} r_I, then per face f of K the
// line sums e_f(j, k) = sum_i (P_GI)_{f, I(i, j, k)} y_I into the per-cell face buffer fb.
// Every global array is read contiguously (couplings per (K, f) are stored I-contiguous).
__global__ void sc_cell_kernel(const __grid_constant__ ScGeom G, const double* __restrict__ dinv,
                               const double* __restrict__ cc, const double* __restrict__ cw,
                               double* __restrict__ rp, double* __restrict__ fb, const double* __restrict__ f,
                               long long lxf) {
  extern __shared__ double scs[];
  const int p = G.p, pm = p - 1, ni = pm * pm * pm, nf = pm * pm;
  double* y = scs;          // [k][j][i]
  const int K = blockIdx.x;
  const int cx = K % G.n[0], cy = (K / G.n[0]) % G.n[1], cz = K / (G.n[0] * G.n[1]);
  const double* dk = dinv + (size_t)K * ni;
  for (int I = threadIdx.x; I < ni; I += blockDim.x) {
    const int i = I % pm + 1, j = (I / pm) % pm + 1, k = I / nf + 1;
    const long long gx = (long long)cx * p + i, gy = (long long)cy * p + j, gz = (long long)cz * p + k;
    const long long g = sc_idx(G, gx, gy, gz);
    double r = rp[g];
    if (f) {   // SC-fused residual: rp holds sign * (A u)_I; complete r_I = f_I + rp_I in place
      r = f[(gz * G.ly + gy) * lxf + gx] + r;
      rp[g] = r;
    }
    y[I] = dk[I] * r;
  }
  __syncthreads();
  // one thread per (direction, line): the line through face position (a, b) along the face
  // normal serves both faces of that direction (the - face with D_i0, the + face with D_ip): one
  // pass over the weights and y, two sums (each in the order of the one-face loop: bitwise equal)
  for (int q = threadIdx.x; q < 3 * nf; q += blockDim.x) {
    const int dir = q / nf, pos = q - dir * nf;
    const int a = pos % pm, b = pos / pm;
    const int I0 = dir == 0 ? (b * pm + a) * pm : (dir == 1 ? b * pm * pm + a : b * pm + a);
    const int st = dir == 0 ? 1 : (dir == 1 ? pm : nf);
    double e0 = 0.0, e1 = 0.0;
    if (G.cmp) {   // the line runs along the face normal: interior index l + 1 of the 1D tables
      const double* wf = cw + ((size_t)K * 3 + dir) * ni;
#pragma unroll 7
      for (int l = 0; l < pm; ++l) {
        const double kw = __dmul_rn(G.kd[l + 1], wf[I0 + l * st]), yv = y[I0 + l * st];
        e0 = fma(__dmul_rn(kw, G.k0[l + 1]), yv, e0);
        e1 = fma(__dmul_rn(kw, G.kp[l + 1]), yv, e1);
      }
    } else {
      const double* cf0 = cc + ((size_t)K * 6 + 2 * dir) * ni;
      const double* cf1 = cf0 + ni;
      for (int l = 0; l < pm; ++l) {
        const double yv = y[I0 + l * st];
        e0 = fma(cf0[I0 + l * st], yv, e0);
        e1 = fma(cf1[I0 + l * st], yv, e1);
      }
    }
    fb[((size_t)K * 6 + 2 * dir) * nf + pos] = e0;
    fb[((size_t)K * 6 + 2 * dir + 1) * nf + pos] = e1;
  }
}

// ICC-SC pre step, part 2 (one thread per face-interior DoF): r_G -= the line sums of the
// (<= 2) cells sharing the face, lower cell first (fixed order: deterministic)
__global__ void sc_face_kernel(const __grid_constant__ ScGeom G, const double* __restrict__ fb,
                               double* __restrict__ rp, int nface) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nface) return;
  const int p = G.p, pm = p - 1, nf = pm * pm;
  const int per_x = (G.n[0] + 1) * G.n[1] * G.n[2] * nf, per_y = (G.n[1] + 1) * G.n[0] * G.n[2] * nf;
  int dir, r = t;
  if (r < per_x) dir = 0;
  else if ((r -= per_x) < per_y) dir = 1;
  else { r -= per_y; dir = 2; }
  const int d1 = dir == 0 ? 1 : 0, d2 = dir == 2 ? 1 : 2;   // in-face directions (ascending)
  const int a = r % pm;  r /= pm;                           // along d1 (0-based)
  const int b = r % pm;  r /= pm;                           // along d2
  const int c1 = r % G.n[d1]; r /= G.n[d1];
  const int c2 = r % G.n[d2]; r /= G.n[d2];
  const int P = r;                                          // plane 0..n_dir
  int cell[3], g[3];
  cell[d1] = c1; cell[d2] = c2;
  g[dir] = P * p; g[d1] = c1 * p + a + 1; g[d2] = c2 * p + b + 1;
  double e = 0.0;
  if (P > 0) {          // cell below: its + face
    cell[dir] = P - 1;
    const int K = (cell[2] * G.n[1] + cell[1]) * G.n[0] + cell[0];
    e += fb[((size_t)K * 6 + 2 * dir + 1) * nf + b * pm + a];
  }
  if (P < G.n[dir]) {   // cell above: its - face
    cell[dir] = P;
    const int K = (cell[2] * G.n[1] + cell[1]) * G.n[0] + cell[0];
    e += fb[((size_t)K * 6 + 2 * dir) * nf + b * pm + a];
  }
  rp[sc_idx(G, g[0], g[1], g[2])] -= e;
}

#ifndef RM_SCP_DOFS   // interior DoFs per thread of the SC post step (all loads issued before the stores);
#define RM_SCP_DOFS 2   // measured 1 / 2 / 4: cfg5 patch stage 1.544 / 1.500 / 1.519 ms (pass AJ)
#endif
template <int D>
__global__ void sc_post_kernel(const __grid_constant__ ScGeom G, const double* __restrict__ dinv,
                               const double* __restrict__ cc, const double* __restrict__ cw, const int* __restrict__ nk,
                               const double* __restrict__ rp, double* __restrict__ cp, long long nint,
                               double* u, double omega, long long lx, const double* uin) {
  // one cell per blockIdx.y row of blocks, interior DoFs across x-blocks: 32-bit index math;
  // D DoFs per thread (I, I + blockDim, ...): every load of the D DoFs precedes the first store
  // (cp is read and written), the same operations per DoF as D = 1 (bitwise equal)
  __shared__ double kt[3][16];   // D_ii, D_i0, D_ip: lane-varying indices (shared, not the param bank)
  if (threadIdx.x < 48) kt[threadIdx.x >> 4][threadIdx.x & 15] =
      (threadIdx.x < 16 ? G.kd : (threadIdx.x < 32 ? G.k0 : G.kp))[threadIdx.x & 15];
  __syncthreads();
  const int p = G.p, pm = p - 1, ni = pm * pm * pm;
  const int K32 = (int)blockIdx.y;   // 32-bit decode (the 64-bit divisions were most of the instructions)
  const long long K = K32;
  const int cx = K32 % G.n[0], cy = (K32 / G.n[0]) % G.n[1], cz = K32 / (G.n[0] * G.n[1]);
  (void)nint;
  const long long x = (long long)cx * p, y = (long long)cy * p, z = (long long)cz * p;
  const double nkK = (double)nk[K];
  double cres[D];
  long long gout[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int I = (blockIdx.x * D + d) * blockDim.x + threadIdx.x;
    gout[d] = -1;
    if (I >= ni) continue;
    const int i = I % pm + 1, j = (I / pm) % pm + 1, k = I / (pm * pm) + 1;
    const double dv = dinv[K * ni + I];
    double c0, c1, c2, c3, c4, c5;
    if (G.cmp) {   // couplings (D_ii w) D_i{0,p} rebuilt from the three interior stiffness weights
      const double wx = cw[(K * 3 + 0) * ni + I], wy = cw[(K * 3 + 1) * ni + I], wz = cw[(K * 3 + 2) * ni + I];
      const double ax = __dmul_rn(kt[0][i], wx), ay = __dmul_rn(kt[0][j], wy), az = __dmul_rn(kt[0][k], wz);
      c0 = __dmul_rn(ax, kt[1][i]); c1 = __dmul_rn(ax, kt[2][i]);
      c2 = __dmul_rn(ay, kt[1][j]); c3 = __dmul_rn(ay, kt[2][j]);
      c4 = __dmul_rn(az, kt[1][k]); c5 = __dmul_rn(az, kt[2][k]);
    } else {
      c0 = cc[(K * 6 + 0) * ni + I]; c1 = cc[(K * 6 + 1) * ni + I]; c2 = cc[(K * 6 + 2) * ni + I];
      c3 = cc[(K * 6 + 3) * ni + I]; c4 = cc[(K * 6 + 4) * ni + I]; c5 = cc[(K * 6 + 5) * ni + I];
    }
    double s = c0 * cp[sc_idx(G, x, y + j, z + k)];
    s = fma(c1, cp[sc_idx(G, x + p, y + j, z + k)], s);
    s = fma(c2, cp[sc_idx(G, x + i, y, z + k)], s);
    s = fma(c3, cp[sc_idx(G, x + i, y + p, z + k)], s);
    s = fma(c4, cp[sc_idx(G, x + i, y + j, z)], s);
    s = fma(c5, cp[sc_idx(G, x + i, y + j, z + p)], s);
    const long long gi = sc_idx(G, x + i, y + j, z + k);
    cres[d] = dv * (nkK * rp[gi] - s);
    gout[d] = u ? ((z + k) * G.ly + y + j) * lx + x + i : gi;
  }
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (gout[d] < 0) continue;
    if (u) {   // fused combine: u = (uin ? uin : u) + omega c_I directly (the combine skips the interiors)
      const long long gu = gout[d];
      u[gu] = (uin ? uin[gu] : u[gu]) + omega * cres[d];
    }
    else cp[gout[d]] = cres[d];
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

cudaError_t encode_maps(PatchLaunch& L) {
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult qr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
    if (e != cudaSuccess || !enc) return cudaErrorNotSupported;
  }
  for (int sb = 0; sb < L.nsub; ++sb) {
    const int m = L.sub_comp[sb];
    cuuint64_t dims[3] = {(cuuint64_t)L.pad.lxp[m], (cuuint64_t)L.pad.len[m][1], (cuuint64_t)L.pad.len[m][2]};
    cuuint64_t strides[2] = {(cuuint64_t)L.pad.lxp[m] * 8, (cuuint64_t)L.pad.lxp[m] * L.pad.len[m][1] * 8};
    cuuint32_t box[3] = {(cuuint32_t)L.box[sb][0], (cuuint32_t)L.box[sb][1], (cuuint32_t)L.box[sb][2]}, es[3] = {1, 1, 1};
    for (int w = 0; w < 2; ++w) {
      double* base = (w == 0 ? L.rpad : L.cpad) + L.pad.poff[m];
      CUresult r = enc(w == 0 ? &L.tm.r[sb] : &L.tm.c[sb], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    }
  }
  return cudaSuccess;
}

}  // namespace

cudaError_t plan_patch_solve(PatchLaunch& L) {
  const size_t boxd = (size_t)((L.box_total + 15) & ~15);
  // three box buffers (patches i-1, i, i+1 in flight) when they fit, else two
  L.nbox = getenv("RM_NBOX1") ? 1 : (exp_env("RM_NBOX2") ? 2 : NBOX);   // RM_NBOX1: documented test switch (rm.h)
  L.smem_fixed = BAR_BYTES + (L.nbox * boxd + (size_t)L.aux_max) * sizeof(double);
  int dev = 0, nsm = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(patch_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin)) != cudaSuccess)
    return e;
  // one CTA per SM; the rings share what the boxes leave: about 1/3 sparse channel, 2/3 tile
  // channel, each holding at least two of its largest units (env RM_RING_A_KB overrides)
  const size_t ua = (size_t)((L.unit_bytes_max_a + 127) & ~127), ub = (size_t)((L.unit_bytes_max_b + 127) & ~127);
  // fewer box buffers when the windows are large (3 -> 2 -> 1; with one buffer the sparse warps
  // run the patches strictly in sequence and the host issue list follows that order)
  while ((size_t)optin < L.smem_fixed + 2 * ua + 2 * ub && L.nbox > 1) {
    --L.nbox;
    L.smem_fixed = BAR_BYTES + (L.nbox * boxd + (size_t)L.aux_max) * sizeof(double);
  }
  if ((size_t)optin < L.smem_fixed + 2 * ua + 2 * ub) return cudaErrorInvalidValue;
  const size_t rings = (optin - L.smem_fixed) & ~(size_t)127;
  size_t capA = (rings / 3) & ~(size_t)127;
  if (const char* s = exp_env("RM_RING_A_KB")) capA = ((size_t)atoi(s) * 1024) & ~(size_t)127;
  capA = std::min(std::max(capA, 2 * ua), rings - 2 * ub);
  if (ub == 0) capA = rings - 128;   // no dense tiles in this family: the sparse channel takes the rings
  capA = std::max(capA, (size_t)128);
  const size_t capB = (rings - capA) & ~(size_t)127;
  L.ring_bytes = (int)capA;
  L.ring_b_bytes = (int)capB;
  int occ = 0;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, patch_stream_kernel, NTHR, L.smem_fixed + capA + capB)) !=
      cudaSuccess)
    return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  L.grid = std::max(1, std::min(L.npatch, occ * nsm));
  if (const char* g = exp_env("RM_GRID")) L.grid = std::max(1, std::min(L.grid, atoi(g)));   // experiments
  if ((e = encode_maps(L)) != cudaSuccess) return e;
  if (exp_env("RM_PROFILE") && !L.prof && (e = cudaMalloc(&L.prof, (size_t)24 * 8 * L.grid)) != cudaSuccess) return e;
  // descriptors live in global memory (64-byte aligned allocation), read by the TMA unit
  if (!L.tm_dev && (e = cudaMalloc(&L.tm_dev, sizeof(TMaps))) != cudaSuccess) return e;
  if ((e = cudaMemcpy(L.tm_dev, &L.tm, sizeof(TMaps), cudaMemcpyHostToDevice)) != cudaSuccess) return e;
  if (exp_env("RM_VERBOSE"))
    fprintf(stderr, "[rm] patch plan: npatch=%d box=%d x%d aux_max=%d fixed=%zu ringA=%zu ringB=%zu occ=%d grid=%d\n",
            L.npatch, L.box_total, L.nbox, L.aux_max, L.smem_fixed, capA, capB, occ, L.grid);
  return cudaSuccess;
}

#ifndef RM_BATCH_CTA3
#define RM_BATCH_CTA3 1   // 1: a third 256-thread CTA per SM where shared memory allows (0: tuning reference)
#endif
#define RM_BATCH_CFGS(X) \
  X(8, 512, 1) X(4, 512, 1) X(2, 512, 1) X(8, 256, 2) X(4, 256, 2) X(2, 256, 2) X(4, 256, 3) X(2, 256, 3) X(4, 384, 2) X(2, 384, 2)

// resident 256-thread CTAs per SM by shared memory (the chooser in abi.cpp counts two the same way)
static int batch_minb(int B, int NT, size_t smem) {
  if (NT == 384) return 2;   // two 384-thread CTAs: 24 warps where three 256-thread CTAs do not fit
  if (NT != 256) return 1;
  return RM_BATCH_CTA3 && B <= 4 && 3 * (smem + 2048) <= 233472 ? 3 : 2;   // B = 8 needs > 85 registers
}

size_t patch_batch_smem(int box_total, int mr_max, int B, int NT) {
  const size_t s = batch_smem_t(B, NT, box_total, mr_max);
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) return 0;
  if (s + 1024 > (size_t)optin) return 0;   // + the static shared arrays
  // the attribute is per instantiation, shared by every family: always the full opt-in size
  const int lim = optin - 1024;
  cudaError_t e = cudaErrorInvalidValue;
#define RM_SET(BB, NN, MM) \
  if (B == BB && NT == NN && (e == cudaSuccess || e == cudaErrorInvalidValue)) \
    e = cudaFuncSetAttribute(patch_batch_kernel<BB, NN, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, lim);
  RM_BATCH_CFGS(RM_SET)
#undef RM_SET
  return e == cudaSuccess ? s : 0;
}

namespace {

cudaError_t launch_batched(const PatchLaunch& L, cudaStream_t st, bool chain_first) {
  BatchArgs a{};
  a.classes = L.classes; a.vals = L.vals; a.fin = L.fin;
  a.bpatch = L.bpatch; a.bclass = L.bclass; a.bblock = L.bblock; a.bfin = L.bfin;
  a.porig = L.porig; a.tm = L.tm_dev;
  a.nsub = L.nsub;
  a.boxd = (L.box_total + 15) & ~15;
  const int mr = (L.mr_max + 31) & ~31;
  a.gofs = a.boxd * L.batch;
  a.pofs = a.gofs + mr * L.batch;
  a.tofs = a.pofs + std::max(L.batch_nt, mr) * L.batch;
  a.box_bytes = 0;
  for (int sb = 0; sb < 3; ++sb) {
    a.boff[sb] = L.boff[sb];
    if (sb < L.nsub) a.box_bytes += 8u * (unsigned)(L.box[sb][0] * L.box[sb][1] * L.box[sb][2]);
  }
  const int minb = batch_minb(L.batch, L.batch_nt, L.bsmem);
  // colour 0 in plain stream order (r and c of the kernels before it complete and visible); colours
  // c >= 1 as programmatic dependent launches: their CTAs start while the previous colour's last
  // wave runs and wait (griddepcontrol.wait) before their reduce-adds
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.dynamicSmemBytes = L.bsmem;
  cfg.stream = st;
  cfg.attrs = pdl;
  // chain_first: this family follows another batched family of the same padded r / c pair with
  // nothing but timing events in between (orientation families): its colour 0 joins that chain
  bool chained = chain_first;
  for (int c = 0; c < L.cs.ncolors; ++c) {
    const int nb = L.bstart[c + 1] - L.bstart[c];
    if (nb <= 0) continue;
    bool launched = false;
#define RM_LAUNCH(BB, NN, MM) \
    if (L.batch == BB && L.batch_nt == NN && minb == MM) { \
      cfg.gridDim = dim3(nb); cfg.blockDim = dim3(NN); \
      cfg.numAttrs = (RM_BATCH_PDL && chained) ? 1 : 0; \
      const cudaError_t le = cudaLaunchKernelEx(&cfg, patch_batch_kernel<BB, NN, MM>, a, L.bstart[c]); \
      if (le != cudaSuccess) return le; \
      launched = true; \
    }
    RM_BATCH_CFGS(RM_LAUNCH)
#undef RM_LAUNCH
    if (!launched) return cudaErrorInvalidConfiguration;   // no instantiation for (B, threads, CTAs per SM)
    chained = true;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_patch_combine(const PatchLaunch& L, double* u, double omega, cudaStream_t st) {
  unpad_axpy_kernel<<<148 * 8, 256, 0, st>>>(L.pad, L.cpad, u, omega, L.pad.off[L.pad.ncomp], 0, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_sc_pre_fused(const PatchLaunch& L, const double* f, long long lx, cudaStream_t st) {
  if (!L.sc_dinv || !L.sc_pre) return cudaErrorInvalidValue;
  ScGeom sg{};
  sg.p = L.sc_p;
  for (int d = 0; d < 3; ++d) sg.n[d] = L.sc_n[d];
  sg.lxp = L.pad.lxp[0];
  sg.ly = L.pad.len[0][1];
  sg.cmp = L.sc_w ? 1 : 0;
  for (int a = 0; a < 16; ++a) { sg.kd[a] = L.sc_kd[a]; sg.k0[a] = L.sc_k0[a]; sg.kp[a] = L.sc_kp[a]; }
  const int pm = L.sc_p - 1;
  const int ncell = sg.n[0] * sg.n[1] * sg.n[2];
  if (ncell == 0 || pm <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * (size_t)(pm * pm * pm);
  static size_t smem_set = 0;
  cudaError_t e;
  if (smem > 48 * 1024 && smem > smem_set) {
    if ((e = cudaFuncSetAttribute(sc_cell_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return e;
    smem_set = smem;
  }
  sc_cell_kernel<<<(unsigned)ncell, RM_SCC_THREADS, smem, st>>>(sg, L.sc_dinv, L.sc_c, L.sc_w, L.rpad, L.sc_fb, f, lx);
  return cudaGetLastError();
}

cudaError_t launch_patch_solve(const PatchLaunch& L, const double* r, double* u, double omega, cudaStream_t st,
                               const KTimer* kt, bool r_padded, bool zero_c, bool combine, bool sc_pre_done,
                               const double* u_in) {
  if (L.npatch <= 0) {   // an empty family still does its part of a shared sequence
    if (!L.cpad) return cudaSuccess;
    if (!r_padded) pad_kernel<<<148 * 8, 256, 0, st>>>(L.pad, r, L.rpad, L.npad);
    if (zero_c) cudaMemsetAsync(L.cpad, 0, (size_t)L.npad * sizeof(double), st);
    if (combine) unpad_axpy_kernel<<<148 * 8, 256, 0, st>>>(L.pad, L.cpad, u, omega, L.pad.off[L.pad.ncomp], 0, u_in);
    return cudaGetLastError();
  }
  const long long n = L.pad.off[L.pad.ncomp];
  cudaError_t e;
  if (!r_padded) {
    pad_kernel<<<148 * 8, 256, 0, st>>>(L.pad, r, L.rpad, L.npad);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  ScGeom sg{};
  long long nface = 0, nint = 0;
  if (L.sc_dinv) {   // geometry for the pre / post steps
    sg.p = L.sc_p;
    for (int d = 0; d < 3; ++d) sg.n[d] = L.sc_n[d];
    sg.lxp = L.pad.lxp[0];
    sg.ly = L.pad.len[0][1];
    sg.cmp = L.sc_w ? 1 : 0;
    for (int a = 0; a < 16; ++a) { sg.kd[a] = L.sc_kd[a]; sg.k0[a] = L.sc_k0[a]; sg.kp[a] = L.sc_kp[a]; }
    const long long pm = L.sc_p - 1;
    nface = ((long long)(sg.n[0] + 1) * sg.n[1] * sg.n[2] + (long long)(sg.n[1] + 1) * sg.n[0] * sg.n[2] +
             (long long)(sg.n[2] + 1) * sg.n[0] * sg.n[1]) * pm * pm;
    nint = (long long)sg.n[0] * sg.n[1] * sg.n[2] * pm * pm * pm;
    if (nface > 0 && L.sc_pre && !sc_pre_done) {
      const int ncell = sg.n[0] * sg.n[1] * sg.n[2];
      const size_t smem = sizeof(double) * (size_t)(pm * pm * pm);
      static size_t smem_set = 0;
      if (smem > 48 * 1024 && smem > smem_set) {
        if ((e = cudaFuncSetAttribute(sc_cell_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
          return e;
        smem_set = smem;
      }
      sc_cell_kernel<<<(unsigned)ncell, RM_SCC_THREADS, smem, st>>>(sg, L.sc_dinv, L.sc_c, L.sc_w, L.rpad, L.sc_fb, nullptr, 0);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      sc_face_kernel<<<(unsigned)((nface + 255) / 256), 256, 0, st>>>(sg, L.sc_fb, L.rpad, (int)nface);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
  }
  if (zero_c && (e = cudaMemsetAsync(L.cpad, 0, (size_t)L.npad * sizeof(double), st)) != cudaSuccess) return e;
  if (!L.batch && (e = cudaMemsetAsync(L.done, 0, sizeof(unsigned), st)) != cudaSuccess) return e;   // the stream kernel's colour counter
  BoxGeom bg;
  bg.ncomp = L.nsub;
  bg.bytes = 0;
  for (int m = 0; m < 3; ++m) {
    for (int d = 0; d < 3; ++d) bg.box[m][d] = L.box[m][d];
    bg.boff[m] = L.boff[m];
    if (m < L.nsub) bg.bytes += 8 * L.box[m][0] * L.box[m][1] * L.box[m][2];
  }
  if (kt) kt->begin(kt->arg);
  if (L.batch) {
    e = launch_batched(L, st, RM_BATCH_CHAINF && r_padded && !zero_c);
  } else
  // cooperative launch: the colour wait of the store warps spins on a counter advanced by other
  // CTAs, so every CTA of the grid must be resident at once -- the runtime guarantees that (or
  // fails the launch with cudaErrorCooperativeLaunchTooLarge) instead of a possible hang under
  // MPS / green contexts / concurrent kernels holding SMs
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)L.grid);
    cfg.blockDim = dim3(NTHR);
    cfg.dynamicSmemBytes = L.smem_fixed + L.ring_bytes + L.ring_b_bytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, patch_stream_kernel, (const TMaps*)L.tm_dev, L.classes, L.pclass, L.pvals, L.porig,
                           L.vals, L.npatch, L.cs, bg, L.done, (uint32_t)L.ring_bytes, (uint32_t)L.ring_b_bytes,
                           L.box_total, L.xfer, L.xbeg, L.nbox, L.prof, L.icc_only);
  }
  if (kt) kt->end(kt->arg);
  if (e != cudaSuccess) return e;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (L.prof && !L.batch) {   // RM_PROFILE=1: per-CTA clock64 counters averaged over CTAs (instrumentation only)
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    std::vector<unsigned long long> h((size_t)24 * L.grid);
    if ((e = cudaMemcpy(h.data(), L.prof, h.size() * 8, cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
    double a[24] = {0};
    for (int b = 0; b < L.grid; ++b)
      for (int k = 0; k < 24; ++k) a[k] += (double)h[24 * b + k] / L.grid / 1e3;
    fprintf(stderr,
            "[rm prof kcyc] producer total %.0f idle %.0f | store total %.0f wait-done %.0f colour %.0f | tiles total %.0f "
            "wait-fwd %.0f | sparse total %.0f box-wait %.0f x-wait %.0f fwd %.0f bwd %.0f | prodA total %.0f room-wait %.0f "
            "| prodB total %.0f room-wait %.0f | fwd: acquire %.0f piv %.0f w %.0f sync %.0f\n",
            a[0], a[1], a[2], a[3], a[4], a[5], a[6], a[7], a[8], a[9], a[10], a[11], a[12], a[13], a[14], a[15],
            a[16], a[17], a[18], a[19]);
  }
  if (L.sc_dinv && nint > 0) {
    const int ni = (L.sc_p - 1) * (L.sc_p - 1) * (L.sc_p - 1);
    const dim3 gp((unsigned)((ni + RM_SCP_THREADS * RM_SCP_DOFS - 1) / (RM_SCP_THREADS * RM_SCP_DOFS)),
                  (unsigned)(sg.n[0] * sg.n[1] * sg.n[2]));
    // c_I to cpad; the combine below writes u for every DoF (measured twice: writing u_out = u_in +
    // omega c_I from the post step and a skeleton-only combine is slower -- cfg5 patch stage 1.562
    // -> 1.587 ms in round 2 -- the post step's scattered u traffic costs more than the streaming pass)
    const bool fuse = combine && L.pad.ncomp == 1 && exp_env("RM_POST_FUSED") != nullptr;
    sc_post_kernel<RM_SCP_DOFS><<<gp, RM_SCP_THREADS, 0, st>>>(sg, L.sc_dinv, L.sc_c, L.sc_w, L.sc_nk, L.rpad, L.cpad, nint,
                                       fuse ? u : nullptr, omega, L.pad.len[0][0], u_in);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (fuse) {
      unpad_axpy_kernel<<<148 * 8, 256, 0, st>>>(L.pad, L.cpad, u, omega, n, L.sc_p, u_in);
      return cudaGetLastError();
    }
  }
  if (combine) unpad_axpy_kernel<<<148 * 8, 256, 0, st>>>(L.pad, L.cpad, u, omega, n, 0, u_in);
  return cudaGetLastError();
}

}  // namespace rm
