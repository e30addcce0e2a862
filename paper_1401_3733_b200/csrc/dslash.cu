// Wilson hopping term on the even-odd tiled layout (sm_100a).
//
// Replaces the reference's scalar site loop dirac_site/dirac_interior
// (proj/include/latbench/kernel_ops.hpp:128-215) and, for decomposed runs,
// its full-spinor halo exchange (proj/src/transport.cpp:175-203).
//
// One thread owns one output site of one parity and accumulates the 8 hops
//   acc = sum_mu [(1-g_mu) U_mu(x) in(x+mu) + (1+g_mu) U_mu(x-mu)^dag in(x-mu)]
// with the spin projection done before the colour multiply (2 of 4 spin
// components), then applies a fused epilogue
//   out_upper = a x_upper + b acc_upper
//   out_lower = s5x a x_lower + s5acc b acc_lower        (gamma5 folds)
// optionally storing it, taking |out|^2 block partials, or instead applying
// the CG residual update r -= alpha out and reducing |r|^2 (out never stored).
//
// Memory layout: spinor components / link entries are tiled by 32
// checkerboard sites (device.cuh: element e of site i at tile(i)*nc*32 +
// e*32 + i%32), so a warp issues fully coalesced 512-byte (LDG.128) loads for
// each component with compile-time element offsets. Links are read in their
// storage format (links.cuh) and rebuilt in registers.
//
// Decomposed directions: boundary sites are handled by a second launch that
// reads half-spinor halos produced by pack_kernel on the neighbour rank:
//   face dir 0 (to -mu partner): h = (1 - g_mu) projection of in at x_mu = 0
//   face dir 1 (to +mu partner): g = U_mu(y)^dag (1 + g_mu) projection at
//                                x_mu = L_mu - 1 (no gauge halo needed).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "links.cuh"
#include "objects.hpp"

namespace lbcu {

namespace {

struct HopArgs {
  DevGeo g;
  const double2* in[2];  // input blocks indexed by input parity
  double2* out[2];       // output blocks by output parity
  const double2* x[2];   // diagonal-term blocks by output parity (nullable)
  double2* r[2];         // CG residual blocks by output parity
  const void* gauge;     // [2 parity][4 mu] blocks of entries x stride (tiled), storage format
  double a, b, s5x, s5acc;
  unsigned s5in;  // sign mask of the gamma5 on the input (sign_mask)
  const double* alpha;
  int par0;    // output parity of a single-parity launch
  int both;    // 1: parity = blockIdx.x & 1
  int nsites;  // sites per parity
  const int* list[2];
  const double2* hfwd[2][4];  // halos by output parity and mu (boundary launches)
  const double2* hbwd[2][4];
  int hcount[4];
  // antiperiodic time sign applied in-kernel (compact formats): the U_0 link
  // whose global time coordinate is bc_tlast carries a factor -1
  int bc_kernel, t_off, bc_tlast;
  // L2-blocked schedule (sched_len > 0): the lattice is cut into spatial
  // blocks of sched_bx x-planes (all y, z) and each block is swept along t;
  // within one time slice a block is one contiguous cb range of sched_len
  // sites, cut into sched_cpb chunks of blockDim.x. Both uses of every link
  // and all 8 uses of every spinor then fall within ~2 slices of one block,
  // a window sized to stay in L2 (hop_apply).
  int sched_len, sched_cpb, sched_bx;
  int ioff[2];  // cb offset of a list-free partial launch (contiguous interior)
  Reduce red;
};

// block index (per parity) + thread -> cb site under the L2-blocked schedule
__device__ __forceinline__ int sched_site(const HopArgs& A, int blk, int bsz, int tid, bool& ok) {
  const int Lt = A.g.L[0], Lx = A.g.L[1];
  const int per_sb = Lt * A.sched_cpb;
  const int sb = blk / per_sb, rem = blk - sb * per_sb;
  const int t = rem / A.sched_cpb, chunk = rem - t * A.sched_cpb;
  const int off = chunk * bsz + tid;
  ok = off < A.sched_len;
  const int row_sites = A.g.vh / (Lt * Lx);  // cb sites per x-plane of a slice
  return (t * Lx + sb * A.sched_bx) * row_sites + off;
}

template <int D, int R0, int R1, int Q0, int Q1>
__device__ __forceinline__ void reconstruct(double2 (&acc)[4][D], const double2 (&g)[2][D]) {
#pragma unroll
  for (int c = 0; c < D; ++c) {
    acc[0][c] = cadd(acc[0][c], g[0][c]);
    acc[1][c] = cadd(acc[1][c], g[1][c]);
    acc[2][c] = cadd(acc[2][c], phm<Q0>(g[R0][c]));
    acc[3][c] = cadd(acc[3][c], phm<Q1>(g[R1][c]));
  }
}

// element stride inside a 32-site tile (device.cuh); the block stride `st`
// only locates (parity, mu) blocks
__device__ __forceinline__ long long estride(long long) { return kTile; }

// h_a = psi_a + F_a * s5 * psi_{p_a}: spin projection of the spinor at cb site nb
template <int D, int P0, int P1, int F0, int F1>
__device__ __forceinline__ void project(double2 (&h)[2][D], const double2* __restrict__ in,
                                        long long st, int nb, unsigned s5) {
  const double2* __restrict__ q = site_ptr<4 * D>(in, nb);
  const long long es = estride(st);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double2 a0 = ldg(q + (long long)(0 * D + c) * es);
    const double2 a1 = ldg(q + (long long)(1 * D + c) * es);
    const double2 b0 = ldg(q + (long long)(P0 * D + c) * es);
    const double2 b1 = ldg(q + (long long)(P1 * D + c) * es);
    h[0][c] = cadd(a0, phm<F0>(cflip(s5, b0)));
    h[1][c] = cadd(a1, phm<F1>(cflip(s5, b1)));
  }
}

template <int D>
__device__ __forceinline__ void negate(double2 (&h)[2][D]) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) h[a][c] = make_double2(-h[a][c].x, -h[a][c].y);
}

template <int D, bool REAL, int FMT>
using ElemT = typename LinkFmt<D, REAL, FMT>::Elem;

// pointer to entry 0 of the (parity, mu) link block at cb site `site`
template <int D, bool REAL, int FMT>
__device__ __forceinline__ const ElemT<D, REAL, FMT>* link_ptr(const void* gauge, long long st,
                                                               int par, int mu, int site) {
  constexpr int E = LinkFmt<D, REAL, FMT>::entries;
  return site_ptr<E>(static_cast<const ElemT<D, REAL, FMT>*>(gauge) + (long long)(par * 4 + mu) * E * st, site);
}

// Multiply by the link and reconstruct into acc. Small dr: row-fused (no
// intermediate g); large dr: the two-phase form schedules better.
template <int D, bool REAL, int FMT, bool DAG, int R0, int R1, int Q0, int Q1, bool SM = false>
__device__ __forceinline__ void link_hop(double2 (&acc)[4][D], const ElemT<D, REAL, FMT>* p,
                                         long long st, const double2 (&h)[2][D]) {
  if constexpr (D <= 3 || FMT == GF_AS4 || FMT == GF_AS4R) {
    link_mul_acc<D, REAL, FMT, DAG, R0, R1, Q0, Q1, SM>(acc, p, estride(st), h);
  } else {
    double2 g[2][D];
    link_mul<D, REAL, FMT, DAG, SM>(g, p, estride(st), h);
    reconstruct<D, R0, R1, Q0, Q1>(acc, g);
  }
}

// ---- warp-private link staging ------------------------------------------------
// The hop is bound by the bytes its warps keep in flight, and every byte a
// thread loads with LDG holds a destination register from issue to use. The
// link tiles a warp needs at its own cb tile (the four forward links) and at
// the tile shifted by a whole number of tiles (backward t and x links) are
// contiguous entries x 512 B runs in the tiled layout, so lane 0 fetches them
// with one bulk async copy each (cp.async.bulk, completion counted on a
// warp-private mbarrier) into shared memory at the top of the kernel: up to 7
// link tiles per warp travel without holding a register, and the hops read
// them back with conflict-free LDS.128 at the same in-tile offsets.
// Slots: 0-3 forward mu = t, x, y, z (output parity, own tile); 4, 5 backward
// t, x (input parity, the neighbour's tile); 6 the input-parity z link at the
// own tile (hop_z_shared). A kernel stages slots [0, NL).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

template <int D, bool REAL, int FMT, int NL>
struct LinkStage {
  using Elem = ElemT<D, REAL, FMT>;
  static constexpr int TILE = LinkFmt<D, REAL, FMT>::entries * kTile;  // elements per tile
  static constexpr int slots = NL;
  const Elem* lane = nullptr;  // this lane's entry 0 of slot 0
  unsigned bar = 0;
  bool ready = false;
  __device__ __forceinline__ void wait() {
    if constexpr (NL > 0) {
      if (!ready) {
        unsigned done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done)
              : "r"(bar), "r"(0u)
              : "memory");
        ready = true;
      }
    }
  }
  template <int SLOT>
  __device__ __forceinline__ const Elem* slot() const {
    return lane + SLOT * TILE;
  }
};

template <int D, bool REAL, int FMT, int NL>
__device__ __forceinline__ LinkStage<D, REAL, FMT, NL> stage_links(const void* gauge, const DevGeo& g, int par,
                                                                   int i, int s, const int c[4]) {
  LinkStage<D, REAL, FMT, NL> ls;
  if constexpr (NL > 0) {
    using Elem = ElemT<D, REAL, FMT>;
    constexpr int TILE = LinkStage<D, REAL, FMT, NL>::TILE;
    constexpr int E = LinkFmt<D, REAL, FMT>::entries;
    extern __shared__ __align__(128) unsigned char ls_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    Elem* w = reinterpret_cast<Elem*>(ls_raw) + (size_t)warp * NL * TILE;
    unsigned long long* bar =
        reinterpret_cast<unsigned long long*>(ls_raw + (size_t)nw * NL * TILE * sizeof(Elem)) + warp;
    ls.lane = w + lane;
    ls.bar = smem_u32(bar);
    if (lane == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ls.bar), "r"(1));
      asm volatile("fence.mbarrier_init.release.cluster;");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ls.bar),
                   "r"((unsigned)(NL * TILE * sizeof(Elem)))
                   : "memory");
      const Elem* gb = static_cast<const Elem*>(gauge);
      auto copy = [&](int slot, int pp, int mu, int site) {
        const Elem* src = gb + (long long)(pp * 4 + mu) * E * g.stride + (long long)(site >> 5) * TILE;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(w + slot * TILE)),
            "l"(src), "r"((unsigned)(TILE * sizeof(Elem))), "r"(ls.bar)
            : "memory");
      };
#pragma unroll
      for (int mu = 0; mu < 4; ++mu)
        if (mu < NL) copy(mu, par, mu, i);
      if constexpr (NL > 4) copy(4, par ^ 1, 0, nb_bwd(g, s, c, 0) >> 1);
      if constexpr (NL > 5) copy(5, par ^ 1, 1, nb_bwd(g, s, c, 1) >> 1);
      if constexpr (NL > 6) copy(6, par ^ 1, 3, i);
    }
    __syncwarp();
  }
  return ls;
}

// Antiperiodic-t sign of a compact link (dense links carry it baked in):
// branch-free so the scheduler can still hoist the next direction's loads.
template <int D, int FMT>
__device__ __forceinline__ void bc_sign(double2 (&h)[2][D], bool neg) {
  if constexpr (FMT != GF_FULL) {
    const unsigned m = sign_mask(neg);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < D; ++c) h[a][c] = cflip(m, h[a][c]);
  }
}

template <int D, bool REAL, int FMT, bool BND, int MU, class LS>
__device__ __forceinline__ void hop_mu(double2 (&acc)[4][D], const HopArgs& A,
                                       const double2* __restrict__ in, int par, int i, int s,
                                       const int c[4], LS& ls) {
  using G = Gam<MU>;
  const long long st = A.g.stride;
  auto fwd = [&] {  // forward: (1 - g_mu) U_mu(x) in(x + mu)
    double2 h[2][D];
    if (BND && !A.g.wrap[MU] && c[MU] == A.g.L[MU] - 1) {
      const int j = face_pos(A.g, c, MU) >> 1;
      const int hc = A.hcount[MU];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int cc = 0; cc < D; ++cc) h[a][cc] = ldg(A.hfwd[par][MU] + (a * D + cc) * hc + j);
    } else {
      project<D, G::p0, G::p1, G::f0, G::f1>(h, in, st, nb_fwd(A.g, s, c, MU) >> 1, A.s5in);
    }
    if constexpr (MU == 0) bc_sign<D, FMT>(h, A.bc_kernel && A.t_off + c[0] == A.bc_tlast);
    if constexpr (MU < LS::slots) {
      ls.wait();
      link_hop<D, REAL, FMT, false, G::r0, G::r1, G::q0, G::q1, true>(acc, ls.template slot<MU>(), st, h);
    } else {
      link_hop<D, REAL, FMT, false, G::r0, G::r1, G::q0, G::q1>(
          acc, link_ptr<D, REAL, FMT>(A.gauge, st, par, MU, i), st, h);
    }
  };
  auto bwd = [&] {  // backward: (1 + g_mu) U_mu(x - mu)^dag in(x - mu)
    if (BND && !A.g.wrap[MU] && c[MU] == 0) {
      double2 g[2][D];
      const int j = face_pos(A.g, c, MU) >> 1;
      const int hc = A.hcount[MU];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int cc = 0; cc < D; ++cc) g[a][cc] = ldg(A.hbwd[par][MU] + (a * D + cc) * hc + j);
      if constexpr (FMT == GF_AS4R) {  // halo records are in the standard basis
        double2 t[2][D];
        as4r_in(t[0], g[0]);
        as4r_in(t[1], g[1]);
        reconstruct<D, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1>(acc, t);
      } else {
        reconstruct<D, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1>(acc, g);
      }
    } else {
      double2 h[2][D];
      const int nb = nb_bwd(A.g, s, c, MU) >> 1;
      project<D, G::p0, G::p1, G::f0 ^ 1, G::f1 ^ 1>(h, in, st, nb, A.s5in);
      if constexpr (MU == 0) {
        const int tl = c[0] > 0 ? c[0] - 1 : A.g.L[0] - 1;
        bc_sign<D, FMT>(h, A.bc_kernel && A.t_off + tl == A.bc_tlast);
      }
      if constexpr (MU < 2 && 4 + MU < LS::slots) {
        ls.wait();
        link_hop<D, REAL, FMT, true, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1, true>(acc, ls.template slot<4 + MU>(),
                                                                                st, h);
      } else {
        link_hop<D, REAL, FMT, true, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1>(
            acc, link_ptr<D, REAL, FMT>(A.gauge, st, par ^ 1, MU, nb), st, h);
      }
    }
  };
#ifndef LBCU_HOP_BWDFIRST
#define LBCU_HOP_BWDFIRST 0
#endif
  if constexpr (LBCU_HOP_BWDFIRST) {
    bwd();
    fwd();
  } else {
    fwd();
    bwd();
  }
}

// Both spin projections (1 -/+ g_mu) of the spinor at cb site nb from one load.
template <int D, int P0, int P1, int F0, int F1>
__device__ __forceinline__ void project2(double2 (&hm)[2][D], double2 (&hp)[2][D],
                                         const double2* __restrict__ in, int nb, unsigned s5) {
  const double2* __restrict__ q = site_ptr<4 * D>(in, nb);
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double2 a0 = ldg(q + (0 * D + c) * kTile);
    const double2 a1 = ldg(q + (1 * D + c) * kTile);
    const double2 b0 = phm<F0>(cflip(s5, ldg(q + (P0 * D + c) * kTile)));
    const double2 b1 = phm<F1>(cflip(s5, ldg(q + (P1 * D + c) * kTile)));
    hm[0][c] = cadd(a0, b0);
    hm[1][c] = cadd(a1, b1);
    hp[0][c] = csub(a0, b0);
    hp[1][c] = csub(a1, b1);
  }
}

// Colour frame of the accumulator: GF_AS4R works in the real basis Wt.
template <int D, int FMT>
__device__ __forceinline__ void to_frame(double2 (&h)[2][D]) {
  if constexpr (FMT == GF_AS4R) {
    double2 t[2][6];
    as4r_in(t[0], h[0]);
    as4r_in(t[1], h[1]);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < D; ++c) h[a][c] = t[a][c];
  }
}

// g = M h in the accumulator frame, M = U or U^dag
template <int D, bool REAL, int FMT, bool DAG, bool SM = false>
__device__ __forceinline__ void mul_frame(double2 (&g)[2][D], const ElemT<D, REAL, FMT>* p,
                                          const double2 (&h)[2][D]) {
  if constexpr (FMT == GF_AS4R) as4r_mul<DAG, SM>(g, p, kTile, h);
  else link_mul<D, REAL, FMT, DAG, SM>(g, p, kTile, h);
}

template <int D>
__device__ __forceinline__ double2 shfl_d2(unsigned mask, double2 v, int src) {
  return make_double2(__shfl_sync(mask, v.x, src), __shfl_sync(mask, v.y, src));
}

// z hops with the neighbour spinors shared inside the warp (ZS kernels).
// Needs every warp to cover whole z-rows of consecutive cb sites (Lz/2
// divides 32, no site list): then both z-neighbours of an output site are
// in[q] at its own cb index i (the "own" one: z+ when the site's z is even,
// dz = 0; z- when odd) and at cb i -/+ 1 (row wrap i +/- (Lz/2 - 1)), which
// is the own cb of another lane of the same row. Each lane loads only its
// own in[q] spinor w and the two links stored at cb i (U_z^q(i), U_z^p(i)),
// forms both projections and the backward product gb = U_z^q(i)^dag P+ w,
// and hands its row neighbour what that lane is missing: gb (dz = 0 rows:
// the consumer's backward hop) or P- w (dz = 1: the consumer's forward hop,
// multiplied by the consumer's own U_z^p). Same arithmetic as hop_mu<3>, one
// spinor load per site fewer.
template <int D, bool REAL, int FMT, class LS>
__device__ __forceinline__ void hop_z_shared(double2 (&acc)[4][D], const HopArgs& A,
                                             const double2* __restrict__ in, int par, int i, int s,
                                             unsigned mask, LS& ls) {
  using G = Gam<3>;
  const long long st = A.g.stride;
  const int dz = s & 1;
  const int hz = A.g.L[3] >> 1;  // cb sites per z-row
  const int z = s % A.g.L[3];
  int o;  // cb index of the other z-neighbour
  if (dz == 0) o = (z == 0) ? i + hz - 1 : i - 1;
  else o = (z == A.g.L[3] - 1) ? i - hz + 1 : i + 1;
  const int src = (threadIdx.x & 31) + (o - i);
  double2 hm[2][D], hp[2][D], gb[2][D];
  project2<D, G::p0, G::p1, G::f0, G::f1>(hm, hp, in, i, A.s5in);
  to_frame<D, FMT>(hm);
  to_frame<D, FMT>(hp);
  if constexpr (6 < LS::slots) {
    ls.wait();
    mul_frame<D, REAL, FMT, true, true>(gb, ls.template slot<6>(), hp);
  } else {
    mul_frame<D, REAL, FMT, true>(gb, link_ptr<D, REAL, FMT>(A.gauge, st, par ^ 1, 3, i), hp);
  }
  double2 r[2][D];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) r[a][c] = shfl_d2<D>(mask, dz ? hm[a][c] : gb[a][c], src);
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double2 f = dz ? r[a][c] : hm[a][c];
      const double2 b = dz ? gb[a][c] : r[a][c];
      hm[a][c] = f;
      gb[a][c] = b;
    }
  double2 gf[2][D];
  if constexpr (3 < LS::slots) {
    ls.wait();
    mul_frame<D, REAL, FMT, false, true>(gf, ls.template slot<3>(), hm);
  } else {
    mul_frame<D, REAL, FMT, false>(gf, link_ptr<D, REAL, FMT>(A.gauge, st, par, 3, i), hm);
  }
  reconstruct<D, G::r0, G::r1, G::q0, G::q1>(acc, gf);
  reconstruct<D, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1>(acc, gb);
}

template <int D, bool REAL, int FMT, bool BND, int EPI, bool ZS, int NL>
__device__ __forceinline__ void site_body(const HopArgs& A, int par, int idx, double (&nrm)[1], unsigned mask);
template <int D, int EPI>
__device__ __forceinline__ void epilogue(const HopArgs& A, int par, int i, const double2 (&acc)[4][D],
                                         double (&nrm)[1]);

template <int D, bool REAL, int FMT, bool BND, int EPI, int MINB, bool ZS, int NL = 0>
__global__ void __launch_bounds__(128, MINB) hop_kernel(const __grid_constant__ HopArgs A) {
  int par, blk, bsz = blockDim.x, tid = threadIdx.x;
  if (A.both == 2) {  // both parities of one cb range in a block: warps [0, n/2) parity 0, the rest parity 1
    bsz = blockDim.x >> 1;
    par = threadIdx.x >= bsz;
    tid = threadIdx.x - par * bsz;
    blk = blockIdx.x;
  } else if (A.both) {
    par = blockIdx.x & 1;
    blk = blockIdx.x >> 1;
  } else {
    par = A.par0;
    blk = blockIdx.x;
  }
  double nrm[1] = {0.0};
  int idx;
  bool ok;
  if (A.sched_len > 0) {
    idx = sched_site(A, blk, bsz, tid, ok);
  } else {
    idx = blk * bsz + tid;
    ok = idx < A.nsites;
  }
  if constexpr (ZS) {
    const unsigned mask = __ballot_sync(0xffffffffu, ok);
    if (ok) site_body<D, REAL, FMT, BND, EPI, ZS, NL>(A, par, idx, nrm, mask);
  } else {
    if (ok) site_body<D, REAL, FMT, BND, EPI, ZS, NL>(A, par, idx, nrm, 0u);
  }
  if constexpr (EPI != EPI_STORE) block_reduce_partial<1>(A.red, nrm);
}

template <int D, bool REAL, int FMT, bool BND, int EPI, bool ZS, int NL>
__device__ __forceinline__ void site_body(const HopArgs& A, int par, int idx, double (&nrm)[1], unsigned mask) {
  {
    const int i = (NL > 0 || !A.list[par]) ? idx + A.ioff[par] : A.list[par][idx];
    int c[4], s;
    cb_coords(A.g, i, par, c, s);
    // NL > 0: whole warps on one cb tile (host check), lane 0 stages the link tiles
    auto ls = stage_links<D, REAL, FMT, NL>(A.gauge, A.g, par, i, s, c);
    double2 acc[4][D];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) acc[k][cc] = make_double2(0.0, 0.0);
    const double2* in = A.in[par ^ 1];
    // Direction order as a 4-digit code of mu values, first hop first
    // (profiles/r03_tune_order*, r03_tune_perm*): the order changes how ptxas
    // batches the loads. z y x t (3210) is 6 % faster for the full Dphi and
    // 2-5 % for the eo hop with SU(2) links (fundamental and adjoint);
    // t x y z (0123) stays best for R12 and AS4R. -DLBCU_HOP_PERM=dddd forces
    // one order for A/B builds (tools/build_variant.sh).
#ifndef LBCU_HOP_PERM
#define LBCU_HOP_PERM -1
#endif
    constexpr int kPerm = LBCU_HOP_PERM >= 0 ? LBCU_HOP_PERM : (FMT == GF_SU2 || (D == 2 && !REAL)) ? 3210 : 123;
    auto dir = [&](auto Mc) {
      constexpr int MU = decltype(Mc)::value;
      if constexpr (MU == 3 && ZS) hop_z_shared<D, REAL, FMT>(acc, A, in, par, i, s, mask, ls);
      else hop_mu<D, REAL, FMT, BND, MU>(acc, A, in, par, i, s, c, ls);
    };
    dir(std::integral_constant<int, kPerm / 1000>{});
    dir(std::integral_constant<int, kPerm / 100 % 10>{});
    dir(std::integral_constant<int, kPerm / 10 % 10>{});
    dir(std::integral_constant<int, kPerm % 10>{});
    if constexpr (FMT == GF_AS4R) {  // back from the real-basis colour frame
#pragma unroll
      for (int sp = 0; sp < 4; ++sp) as4r_out(acc[sp], 0.5);
    }

    epilogue<D, EPI>(A, par, i, acc, nrm);
  }
}

// ---- experiment: TMA-staged row blocks (full Dphi, SU(2) links, Lz = 32) ----
// A block of 8 warps owns 8 consecutive y-rows of one (t, x) plane, both
// parities (warps 0-3 parity 0, 4-7 parity 1; a warp = one 32-site tile = 2
// rows). Thread 0 stages, with 12 bulk copies (cp.async.bulk, one 4 KB tile
// each, completion on an mbarrier), the input tiles of rows y0-2 .. y0+9 of
// both parities: every y, z and diagonal operand of the block. While they
// travel, each thread does its t and x hops from global memory; then the y
// and z hops and the diagonal term read shared memory.
constexpr int kRbRows = 8, kRbTiles = (kRbRows + 4) / 2;  // tiles per parity

template <int D, int P0, int P1, int F0, int F1>
__device__ __forceinline__ void project_sm(double2 (&h)[2][D], const double2* q, unsigned s5) {
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double2 a0 = q[(0 * D + c) * kTile], a1 = q[(1 * D + c) * kTile];
    const double2 b0 = q[(P0 * D + c) * kTile], b1 = q[(P1 * D + c) * kTile];
    h[0][c] = cadd(a0, phm<F0>(cflip(s5, b0)));
    h[1][c] = cadd(a1, phm<F1>(cflip(s5, b1)));
  }
}

template <int D, bool REAL, int FMT, int MINB>
__global__ void __launch_bounds__(256, MINB) hop_rowblock_kernel(const __grid_constant__ HopArgs A) {
  extern __shared__ __align__(128) unsigned char rb_raw[];
  constexpr int TILE = 4 * D * kTile;                 // double2 per tile
  constexpr int STAGE = 2 * kRbTiles * TILE;          // double2 per stage
  double2* sm0 = reinterpret_cast<double2*>(rb_raw);  // [stage][parity][kRbTiles][4D][32]
  __shared__ __align__(8) unsigned long long bar[2];
  const int Ly = A.g.L[2];
  const int nyb = Ly / kRbRows;
  const int nblk = A.g.L[0] * A.g.L[1] * nyb;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int par = w >> 2, pairk = w & 3;
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[k])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int blk, int stage) {
    const int yb = blk % nyb, tx = blk / nyb, y0 = yb * kRbRows;
    const unsigned bytes = STAGE * sizeof(double2);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[stage])), "r"(bytes)
                 : "memory");
    for (int pp = 0; pp < 2; ++pp)
      for (int k = 0; k < kRbTiles; ++k) {
        const int y = (y0 - 2 + 2 * k + Ly) % Ly;
        const double2* src = A.in[pp] + (long long)((tx * Ly + y) >> 1) * TILE;
        double2* dst = sm0 + stage * STAGE + (pp * kRbTiles + k) * TILE;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(dst)),
            "l"(src), "r"((unsigned)(TILE * sizeof(double2))), "r"(smem_u32(&bar[stage]))
            : "memory");
      }
  };
  if (threadIdx.x == 0 && blockIdx.x < nblk) issue(blockIdx.x, 0);
  int it = 0;
  for (int blk = blockIdx.x; blk < nblk; blk += gridDim.x, ++it) {
    const int stage = it & 1;
    // prefetch the next block into the other stage (its previous contents
    // were consumed before the __syncthreads at the end of the last iteration)
    if (threadIdx.x == 0 && blk + gridDim.x < nblk) issue(blk + gridDim.x, stage ^ 1);
    double2* sm = sm0 + stage * STAGE;
    const int yb = blk % nyb, tx = blk / nyb, y0 = yb * kRbRows;
    auto tile_of = [&](int y) { return (tx * Ly + y) >> 1; };
  // this thread's output site
  const int i = tile_of(y0 + 2 * pairk) * 32 + lane;  // cb index in parity `par`
  int c[4], s;
  cb_coords(A.g, i, par, c, s);
  double2 acc[4][D];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int cc = 0; cc < D; ++cc) acc[k][cc] = make_double2(0.0, 0.0);
  const double2* in = A.in[par ^ 1];
  LinkStage<D, REAL, FMT, 0> nols;
  hop_mu<D, REAL, FMT, false, 1>(acc, A, in, par, i, s, c, nols);
  hop_mu<D, REAL, FMT, false, 0>(acc, A, in, par, i, s, c, nols);
  // wait for the staged tiles of this stage (phase flips every second block)
  {
    unsigned done = 0;
    const unsigned phase = (it >> 1) & 1;
    while (!done)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&bar[stage])), "r"(phase)
          : "memory");
  }
  const long long st = A.g.stride;
  const int q = par ^ 1;
  // staged-tile address of the input site (row y, cb within row) of parity pp
  auto sm_site = [&](int pp, int y, int cbrow) -> const double2* {
    int k = ((y - (y0 - 2) + Ly) % Ly) >> 1;  // row pair slot
    const int r = y & 1;
    return sm + (pp * kRbTiles + k) * TILE + r * 16 + cbrow;
  };
  const int hz = A.g.L[3] >> 1;  // 16
  const int cbrow = i % hz;        // position of the output cb within its row
  const int dz = s & 1, yy = c[2];
#pragma unroll
  for (int dir = 0; dir < 2; ++dir) {
    using G = Gam<2>;
    // y hops: neighbour rows y +- 1, same cb position within the row
    double2 h[2][D];
    const int yn = dir == 0 ? (yy + 1) % Ly : (yy - 1 + Ly) % Ly;
    if (dir == 0) {
      project_sm<D, G::p0, G::p1, G::f0, G::f1>(h, sm_site(q, yn, cbrow), A.s5in);
      link_hop<D, REAL, FMT, false, G::r0, G::r1, G::q0, G::q1>(acc, link_ptr<D, REAL, FMT>(A.gauge, st, par, 2, i), st, h);
    } else {
      project_sm<D, G::p0, G::p1, G::f0 ^ 1, G::f1 ^ 1>(h, sm_site(q, yn, cbrow), A.s5in);
      const int nb = nb_bwd(A.g, s, c, 2) >> 1;
      link_hop<D, REAL, FMT, true, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1>(acc, link_ptr<D, REAL, FMT>(A.gauge, st, q, 2, nb), st, h);
    }
  }
  {
    using G = Gam<3>;
    // z hops: own row; z+ at cb position (dz == 0 ? same : +1), z- at (dz == 0 ? -1 : same), row-periodic
    const int cp = dz == 0 ? cbrow : (cbrow + 1) % hz;
    const int cm = dz == 0 ? (cbrow - 1 + hz) % hz : cbrow;
    double2 h[2][D];
    project_sm<D, G::p0, G::p1, G::f0, G::f1>(h, sm_site(q, yy, cp), A.s5in);
    link_hop<D, REAL, FMT, false, G::r0, G::r1, G::q0, G::q1>(acc, link_ptr<D, REAL, FMT>(A.gauge, st, par, 3, i), st, h);
    project_sm<D, G::p0, G::p1, G::f0 ^ 1, G::f1 ^ 1>(h, sm_site(q, yy, cm), A.s5in);
    const int nb = nb_bwd(A.g, s, c, 3) >> 1;
    link_hop<D, REAL, FMT, true, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1>(acc, link_ptr<D, REAL, FMT>(A.gauge, st, q, 3, nb), st, h);
  }
  // epilogue: out = a x + b acc with x = in (full Dphi), x from shared memory
  const double2* xs = sm_site(par, yy, cbrow);
  double2* __restrict__ out = site_ptr<4 * D>(A.out[par], i);
#pragma unroll
  for (int sp = 0; sp < 4; ++sp)
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      const double bs = sp < 2 ? A.b : A.b * A.s5acc;
      const double as = sp < 2 ? A.a : A.a * A.s5x;
      const double2 xv = xs[(sp * D + cc) * kTile];
      double2 v = cscale(bs, acc[sp][cc]);
      v.x = fma(as, xv.x, v.x);
      v.y = fma(as, xv.y, v.y);
      out[(sp * D + cc) * kTile] = v;
    }
  __syncthreads();  // every warp is done with this stage before it is refilled
  }
}

// out = a x + b acc (gamma5 signs folded), then store / store + |out|^2 /
// CG residual update. Two phases: every load (x, r) is issued before any
// store, and the pointers are restrict-qualified, so the 4 dr round trips
// overlap instead of serialising behind possible aliasing.
template <int D, int EPI>
__device__ __forceinline__ void epilogue(const HopArgs& A, int par, int i, const double2 (&acc)[4][D],
                                         double (&nrm)[1]) {
  const long long st = estride(A.g.stride);
  const double2* __restrict__ x = A.x[par] ? site_ptr<4 * D>(A.x[par], i) : nullptr;
  double2* __restrict__ out = A.out[par] ? site_ptr<4 * D>(A.out[par], i) : nullptr;
  double2* __restrict__ r = A.r[par] ? site_ptr<4 * D>(A.r[par], i) : nullptr;
  double2 xv[4][D], rv[4][D];
#pragma unroll
  for (int sp = 0; sp < 4; ++sp)
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      const long long o = (long long)(sp * D + cc) * st;
      xv[sp][cc] = x ? ldg(x + o) : make_double2(0.0, 0.0);
      if constexpr (EPI == EPI_CG) rv[sp][cc] = __ldcg(r + o);
    }
  const double alpha = (EPI == EPI_CG) ? *A.alpha : 0.0;
#pragma unroll
  for (int sp = 0; sp < 4; ++sp)
#pragma unroll
    for (int cc = 0; cc < D; ++cc) {
      const long long o = (long long)(sp * D + cc) * st;
      const double bs = sp < 2 ? A.b : A.b * A.s5acc;
      const double as = sp < 2 ? A.a : A.a * A.s5x;
      double2 v = cscale(bs, acc[sp][cc]);
      v.x = fma(as, xv[sp][cc].x, v.x);
      v.y = fma(as, xv[sp][cc].y, v.y);
      if constexpr (EPI == EPI_CG) {
        double2 w = rv[sp][cc];
        w.x = fma(-alpha, v.x, w.x);
        w.y = fma(-alpha, v.y, w.y);
        r[o] = w;
        nrm[0] = fma(w.x, w.x, fma(w.y, w.y, nrm[0]));
      } else {
        out[o] = v;
        if constexpr (EPI == EPI_STORE_NORM) nrm[0] = fma(v.x, v.x, fma(v.y, v.y, nrm[0]));
      }
    }
}

// Pack one face of the input field into half-spinor records (see header).
struct PackArgs {
  DevGeo g;
  const double2* in;  // input parity block
  const void* gauge;
  int in_par, mu, dir, count;
  unsigned s5in;  // sign mask (sign_mask)
  int bc_kernel, t_off, bc_tlast;
  double2* outbuf;  // [2D][count]
};

template <int D, bool REAL, int FMT, int MU>
__device__ __forceinline__ void pack_site(const PackArgs& P, int j) {
  using G = Gam<MU>;
  const long long st = P.g.stride;
  // record j -> site on the x_mu = edge slab with parity in_par (host: face_site)
  int c[4];
  const int edge = P.dir ? P.g.L[MU] - 1 : 0;
  {
    int fp = 2 * j;
    int last = -1;
#pragma unroll
    for (int d = 3; d >= 0; --d) {
      if (d == MU) continue;
      if (last < 0) last = d;
      c[d] = fp % P.g.L[d];
      fp /= P.g.L[d];
    }
    c[MU] = edge;
    c[last] += (c[0] + c[1] + c[2] + c[3] + P.in_par) & 1;
  }
  const int s = ((c[0] * P.g.L[1] + c[1]) * P.g.L[2] + c[2]) * P.g.L[3] + c[3];
  const int cb = s >> 1;
  double2 h[2][D];
  if (P.dir == 0) {
    project<D, G::p0, G::p1, G::f0, G::f1>(h, P.in, st, cb, P.s5in);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) P.outbuf[(a * D + cc) * P.count + j] = h[a][cc];
  } else {
    project<D, G::p0, G::p1, G::f0 ^ 1, G::f1 ^ 1>(h, P.in, st, cb, P.s5in);
    if (MU == 0 && P.bc_kernel && P.t_off + c[0] == P.bc_tlast) negate<D>(h);
    double2 g[2][D];
    link_mul<D, REAL, FMT, true>(g, link_ptr<D, REAL, FMT>(P.gauge, st, P.in_par, MU, cb), estride(st), h);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) P.outbuf[(a * D + cc) * P.count + j] = g[a][cc];
  }
}

// All faces of all requested parities in one launch: job k covers blocks
// [first[k], first[k + 1]) and packs one (parity, face) record set.
constexpr int kMaxPackJobs = 16;
struct PackAll {
  PackArgs job[kMaxPackJobs];
  int first[kMaxPackJobs + 1];
  int njobs;
};

template <int D, bool REAL, int FMT>
__global__ void __launch_bounds__(128) pack_kernel(const __grid_constant__ PackAll P) {
  int k = 0;
  while (k + 1 < P.njobs && (int)blockIdx.x >= P.first[k + 1]) ++k;
  const PackArgs& J = P.job[k];
  const int j = (blockIdx.x - P.first[k]) * blockDim.x + threadIdx.x;
  if (j >= J.count) return;
  switch (J.mu) {
    case 0: pack_site<D, REAL, FMT, 0>(J, j); break;
    case 1: pack_site<D, REAL, FMT, 1>(J, j); break;
    case 2: pack_site<D, REAL, FMT, 2>(J, j); break;
    default: pack_site<D, REAL, FMT, 3>(P.job[k], j); break;
  }
}

constexpr int kBlock = 128;  // launch-bounds block size (pack kernel, upper bound)

// Occupancy knob: LBCU_HOP_MINB = minimum resident 128-thread blocks per SM
// requested from ptxas (__launch_bounds__), i.e. a register cap.
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

template <int D, bool REAL, int FMT>
int default_minb() {
  // profiles/r01_tune_minb_*, r02 (tiled layout): 4 blocks/SM for the compact
  // SU(2) fundamental links (2-4 %), 3 for the other dr <= 3 formats (R12
  // 1 %, dense; SU(2) adjoint: eo hop 3-5 % and eo CG 6 % faster than at 4,
  // profiles/r2g_*minb_cfg4.log; R10 6 %, r2g_tune_minb_block_cfg3.log);
  // larger dr spill under any cap.
  if (FMT == GF_SU2 && !REAL) return 4;
  if (D <= 3) return 3;
  return 1;
}

// hop block size (<= kBlock); LBCU_HOP_BLOCK=64 halves it (finer scheduling)
int hop_block() {
  static const int b = [] {
    const char* e = std::getenv("LBCU_HOP_BLOCK");
    const int v = e ? std::atoi(e) : kBlock;
    return (v == 32 || v == 64) ? v : kBlock;
  }();
  return b;
}

int hop_blocks(int nsites, int npar, int /*dr*/) { return (nsites + hop_block() - 1) / hop_block() * npar; }

// Link tiles staged per warp (LinkStage) by the list-free, undecomposed kernels
// of each storage format; 0 = none. Measured (profiles/r2s_sweep_ls_mix.log,
// r2r_traffic_ls_mix.txt, r2x_ls_r12_balance.log): the four forward tiles help
// the SU(3) R10 hop (config 3: eo hop -3 to -4 %, eo CG -2 %, full Dphi -0.5 %;
// six tiles leave too little L1); R12's 3 KB tiles cost the full Dphi 8-11 %
// for 1-2 % on the eo hop, SU(2) links lose 2-7 % (their links shared L1 lines
// with the other parity) and AS4R's 9 KB tiles 13 %. -DLBCU_HOP_NL=n forces one
// value for A/B builds (tools/build_variant.sh).
#ifndef LBCU_HOP_NL
#define LBCU_HOP_NL -1
#endif
template <int D, bool REAL, int FMT, bool ZS>
constexpr int ls_slots() {
  if (LBCU_HOP_NL >= 0) return (LBCU_HOP_NL == 7 && !ZS) ? 6 : LBCU_HOP_NL;
  if (FMT == GF_R10) return 4;
  return 0;
}

template <int D, bool REAL, int FMT, int MINB>
void launch_hop_minb(const HopArgs& A, bool bnd, int epi, bool zs, bool ls, int blocks, cudaStream_t s) {
#define LBCU_HOP_CASE(B, E, Z)                                                      \
  if (bnd == B && epi == E && zs == Z) {                                            \
    constexpr int NL = B ? 0 : ls_slots<D, REAL, FMT, Z>();                         \
    if constexpr (NL > 0) {                                                         \
      if (ls) {                                                                     \
        auto* k = hop_kernel<D, REAL, FMT, B, E, MINB, Z, NL>;                      \
        const int nw = hop_block() / 32;                                            \
        const size_t smem = (size_t)nw * NL * LinkStage<D, REAL, FMT, NL>::TILE *   \
                                sizeof(ElemT<D, REAL, FMT>) + nw * 8;               \
        static bool attr = false;                                                   \
        if (!attr) {                                                                \
          LBCU_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
          attr = true;                                                              \
        }                                                                           \
        k<<<blocks, hop_block(), smem, s>>>(A);                                     \
        return;                                                                     \
      }                                                                             \
    }                                                                               \
    hop_kernel<D, REAL, FMT, B, E, MINB, Z><<<blocks, hop_block(), 0, s>>>(A);      \
    return;                                                                         \
  }
  if constexpr (D == 2 && !REAL) {
    LBCU_HOP_CASE(false, EPI_STORE, true)
    LBCU_HOP_CASE(false, EPI_STORE_NORM, true)
    LBCU_HOP_CASE(false, EPI_CG, true)
  }
  LBCU_HOP_CASE(false, EPI_STORE, false)
  LBCU_HOP_CASE(false, EPI_STORE_NORM, false)
  LBCU_HOP_CASE(false, EPI_CG, false)
  LBCU_HOP_CASE(true, EPI_STORE, false)
  LBCU_HOP_CASE(true, EPI_STORE_NORM, false)
  LBCU_HOP_CASE(true, EPI_CG, false)
#undef LBCU_HOP_CASE
  throw Error(LBCU_CONTRACT_VIOLATION, "hop: no kernel for this variant");
}

template <int D, bool REAL, int FMT>
void launch_hop(const HopArgs& A, bool bnd, int epi, int nsites, int npar, cudaStream_t s,
                int blocks_override = 0, bool zs = false, bool ls = false) {
  if (nsites <= 0) return;
  // measured (profiles/r03_tune_zs_*, r03_tune_xcol_zs_*): +2.5 % for SU(2)
  // fundamental; -1.5 % (SU(3) R12), -3 % (SU(2) adjoint), -15 % (AS4R) from
  // the extra live values, so only the dr = 2 complex kernels share z hops
  if constexpr (!(D == 2 && !REAL)) zs = false;
  const int blocks = blocks_override > 0 ? blocks_override : hop_blocks(nsites, npar, D);
  if constexpr (D <= 3) {
    const int minb = env_int("LBCU_HOP_MINB", default_minb<D, REAL, FMT>());
    if (minb == 4) {
      launch_hop_minb<D, REAL, FMT, 4>(A, bnd, epi, zs, ls, blocks, s);
      return;
    }
    if constexpr (D == 2 && FMT == GF_SU2) {
      if (minb == 5) {
        launch_hop_minb<D, REAL, FMT, 5>(A, bnd, epi, zs, ls, blocks, s);
        return;
      }
    }
    if (minb == 3) {
      launch_hop_minb<D, REAL, FMT, 3>(A, bnd, epi, zs, ls, blocks, s);
      return;
    }
  }
  launch_hop_minb<D, REAL, FMT, 1>(A, bnd, epi, zs, ls, blocks, s);
}

// Supported representation dimensions and storage formats (compile-time
// specialisations). complex: SU(2)F 2, SU(3)F/SU(3)AS 3, SU(4)F 4,
// SU(4)AS/SU(3)S/SU(6)F 6, SU(4)S 10; real: SU(2)A 3, SU(3)A 8.
template <class F>
void dispatch(int dr, bool real, int fmt, F&& f) {
  using std::integral_constant;
  if (!real) {
    switch (dr) {
      case 2:
        if (fmt == GF_SU2) return f(integral_constant<int, 2>{}, std::false_type{}, integral_constant<int, GF_SU2>{});
        return f(integral_constant<int, 2>{}, std::false_type{}, integral_constant<int, GF_FULL>{});
      case 3:
        if (fmt == GF_R12) return f(integral_constant<int, 3>{}, std::false_type{}, integral_constant<int, GF_R12>{});
        if (fmt == GF_R10) return f(integral_constant<int, 3>{}, std::false_type{}, integral_constant<int, GF_R10>{});
        return f(integral_constant<int, 3>{}, std::false_type{}, integral_constant<int, GF_FULL>{});
      case 4: return f(integral_constant<int, 4>{}, std::false_type{}, integral_constant<int, GF_FULL>{});
      case 6:
        if (fmt == GF_AS4) return f(integral_constant<int, 6>{}, std::false_type{}, integral_constant<int, GF_AS4>{});
        if (fmt == GF_AS4R) return f(integral_constant<int, 6>{}, std::false_type{}, integral_constant<int, GF_AS4R>{});
        return f(integral_constant<int, 6>{}, std::false_type{}, integral_constant<int, GF_FULL>{});
      case 10: return f(integral_constant<int, 10>{}, std::false_type{}, integral_constant<int, GF_FULL>{});
    }
  } else {
    switch (dr) {
      case 3:
        if (fmt == GF_SU2) return f(integral_constant<int, 3>{}, std::true_type{}, integral_constant<int, GF_SU2>{});
        return f(integral_constant<int, 3>{}, std::true_type{}, integral_constant<int, GF_FULL>{});
      case 8: return f(integral_constant<int, 8>{}, std::true_type{}, integral_constant<int, GF_FULL>{});
    }
  }
  throw Error(LBCU_CONFIG_ERROR, "no device specialisation for representation dimension " +
                                     std::to_string(dr) + (real ? " (real)" : " (complex)"));
}

#define LBCU_TPARAMS(Dc, Rc, Fc) decltype(Dc)::value, decltype(Rc)::value, decltype(Fc)::value

HaloBufs& halo_bufs(lbcu_ctx_s* ctx, int dr) {
  HaloBufs& hb = ctx->halo[dr];
  size_t need = 0;
  for (int f = 0; f < 8; ++f) need = std::max<size_t>(need, 2 * dr * ctx->plan.count[f]);
  Transport* T = ctx->world->t.get();
  if (T->direct()) {  // collective on first use per dr: every rank maps every arena
    if (!hb.arena) {
      hb.slot = (need + 31) / 32 * 32;
      const size_t bytes = 2 * 8 * 2 * hb.slot * sizeof(double2);
      LBCU_CUDA(cudaMalloc(&hb.arena, bytes));
      T->map_arena(ctx->rank, dr, hb.arena, bytes);
    }
    return hb;
  }
  if (hb.cap < need) {
    for (int p = 0; p < 2; ++p)
      for (int f = 0; f < 8; ++f) {
        if (hb.send[p][f]) cudaFree(hb.send[p][f]);
        if (hb.recv[p][f]) cudaFree(hb.recv[p][f]);
        hb.send[p][f] = hb.recv[p][f] = nullptr;
        if (ctx->plan.count[f] == 0) continue;
        LBCU_CUDA(cudaMalloc(&hb.send[p][f], need * sizeof(double2)));
        LBCU_CUDA(cudaMalloc(&hb.recv[p][f], need * sizeof(double2)));
      }
    hb.cap = need;
  }
  return hb;
}

}  // namespace

void hop_apply(lbcu_ctx_s* ctx, const HopCall& c) {
  const Geometry& geo = ctx->geo;
  const int dr = c.in->dr;
  const bool real = c.g->real;
  const int fmt = c.g->fmt;
  const int pars[2] = {c.out_parity == 2 ? 0 : c.out_parity, c.out_parity == 2 ? 1 : c.out_parity};
  const int npar = c.out_parity == 2 ? 2 : 1;
  for (int k = 0; k < npar; ++k) {
    const int p = pars[k];
    if (!c.out->has(p) || !c.in->has(p ^ 1) || (c.x && !c.x->has(p)) || (c.r && !c.r->has(p)))
      throw Error(LBCU_CONTRACT_VIOLATION, "hop: field subsets do not cover the requested parity");
  }

  HopArgs A{};
  A.g = ctx->dgeo;
  for (int p = 0; p < 2; ++p) {
    A.in[p] = c.in->par[p];
    A.out[p] = c.out->par[p];
    A.x[p] = c.x ? c.x->par[p] : nullptr;
    A.r[p] = c.r ? c.r->par[p] : nullptr;
  }
  A.gauge = c.g->base;
  A.a = c.a;
  A.b = c.b;
  A.s5in = sign_mask(c.s5in < 0.0);
  A.s5x = c.s5x;
  A.s5acc = c.s5acc;
  A.alpha = c.alpha;
  A.bc_kernel = (c.g->bc == LBCU_BC_ANTIPERIODIC_T && fmt != GF_FULL) ? 1 : 0;
  A.t_off = geo.coords[0] * geo.local[0];
  A.bc_tlast = geo.global[0] - 1;
  const bool reduce = c.epi != EPI_STORE;
  cudaStream_t s = ctx->stream;

  if (!geo.any_decomposed) {
    A.nsites = static_cast<int>(geo.vh);
    A.both = npar == 2;
    A.par0 = pars[0];
    int blocks = hop_blocks(A.nsites, npar, dr);
    // full Dphi: both parities of one cb range in a block (warps 0-1 parity 0,
    // warps 2-3 parity 1), so a block's diagonal, z and y operands and its y and
    // z links are the other half's neighbour operands and meet in L1: L2 -> SM
    // bytes -9 %, time -1.4 to -3 % on configs 2-5 (profiles/r2r_traffic_ls_mix.txt)
    const bool mix = npar == 2 && env_int("LBCU_HOP_MIX", 1) && hop_block() % 64 == 0;
    const int bsz = mix ? hop_block() / 2 : hop_block();
    if (mix) {
      A.both = 2;
      blocks = (A.nsites + bsz - 1) / bsz;
    }
    // L2-blocked schedule: spatial blocks of bx x-planes whose two-slice
    // working set (spinor in/out + links as stored) fits the L2 budget
    if (env_int("LBCU_HOP_SCHED", 1)) {
      const int lb = fmt == GF_SU2 ? 32 : fmt == GF_R12 ? 96 : fmt == GF_R10 ? 80 : fmt == GF_AS4 ? 256
                     : fmt == GF_AS4R ? 288 : dr * dr * (real ? 8 : 16);
      const double site_bytes = 128.0 * dr + (npar == 2 ? 4 : 8) * lb;
      const double plane_bytes = site_bytes * geo.local[2] * geo.local[3];
      const double budget = env_int("LBCU_HOP_L2MB", 32) * 1e6;
      int bx = 1;
      for (int d = 1; d <= geo.local[1]; ++d)
        if (geo.local[1] % d == 0 && d * plane_bytes <= budget) bx = d;
      if (bx < geo.local[1]) {  // a whole slice fits: the linear order is the same sweep
        A.sched_bx = bx;
        A.sched_len = bx * geo.local[2] * geo.local[3] / 2;
        A.sched_cpb = (A.sched_len + bsz - 1) / bsz;
        blocks = (geo.local[1] / bx) * geo.local[0] * A.sched_cpb * (mix ? 1 : npar);
      }
    }
    if (reduce) {
      if (blocks > ctx->max_partials) throw Error(LBCU_CUDA_ERROR, "reduction workspace too small");
      A.red = Reduce{ctx->partials, c.result, 0, blocks,
                     c.post, ctx->dcg, ctx->dhist, c.handle, c.use_graph};
    }
    // experiment (off by default, 8 % slower: profiles/r03_tune_rb*_cfg2.log):
    // TMA-staged row blocks for the full Dphi with SU(2) links
    if (env_int("LBCU_HOP_RB", 0) && npar == 2 && c.epi == EPI_STORE && c.x == c.in && fmt == GF_SU2 &&
        dr == 2 && !real && geo.local[3] == 32 && geo.local[2] % kRbRows == 0) {
      const int nb = std::min(geo.local[0] * geo.local[1] * (geo.local[2] / kRbRows), 148 * 2);
      const size_t smem = 2ull * 2ull * kRbTiles * 4 * dr * kTile * sizeof(double2);
      static bool attr = false;
      if (!attr) {
        LBCU_CUDA(cudaFuncSetAttribute(hop_rowblock_kernel<2, false, GF_SU2, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
      }
      hop_rowblock_kernel<2, false, GF_SU2, 2><<<nb, 256, smem, s>>>(A);
      ctx->launches += 1;
      LBCU_CUDA(cudaGetLastError());
      return;
    }
    // warp-shared z hops when every warp covers whole z-rows (hop_z_shared)
    const int hz = geo.local[3] / 2;
    const bool zs = env_int("LBCU_HOP_ZS", 1) && hz > 0 && 32 % hz == 0;
    // link staging (LinkStage): every warp must sit on one cb tile of one x-plane
    const bool ls = env_int("LBCU_HOP_LS", 1) && (geo.local[2] * geo.local[3] / 2) % kTile == 0 &&
                    hop_block() % kTile == 0;
    dispatch(dr, real, fmt, [&](auto Dc, auto Rc, auto Fc) {
      launch_hop<LBCU_TPARAMS(Dc, Rc, Fc)>(A, false, c.epi, A.nsites, npar, s, blocks, zs, ls);
    });
    ctx->launches += 1;
    if (reduce) {
      k_reduce_finish<1><<<1, kFinishThreads, 0, s>>>(A.red);
      ctx->launches += 1;
    }
    LBCU_CUDA(cudaGetLastError());
    return;
  }

  // ---- decomposed: pack -> exchange -> interior -> boundary -------------
  // One fused pack launch for every (output parity, face), one exchange, then
  // one interior and one boundary launch covering the requested parities
  // (per parity only if their site counts differ).
  HaloBufs& hb = halo_bufs(ctx, dr);
  if (c.post != POST_NONE)
    throw Error(LBCU_CONTRACT_VIOLATION, "fused CG scalar steps need a single rank");
  Transport* T = ctx->world->t.get();
  const bool direct = T->direct();
  const long long epoch = ctx->xepoch++;
  auto arena_off = [&](int p, int f) { return ((p * 8 + f) * 2 + (epoch & 1)) * hb.slot; };
  PackAll PA{};
  std::vector<Transport::Msg> msgs;
  int pack_blocks = 0;
  for (int k = 0; k < npar; ++k) {
    const int p = pars[k], q = p ^ 1;
    for (int f = 0; f < 8; ++f) {
      if (ctx->plan.count[f] == 0) continue;
      if (PA.njobs == kMaxPackJobs) throw Error(LBCU_CUDA_ERROR, "too many halo faces");
      PackArgs& P = PA.job[PA.njobs];
      P.g = ctx->dgeo;
      P.in = c.in->par[q];
      P.gauge = c.g->base;
      P.in_par = q;
      P.mu = f / 2;
      P.dir = f % 2;
      P.count = static_cast<int>(ctx->plan.count[f]);
      P.s5in = A.s5in;
      P.bc_kernel = A.bc_kernel;
      P.t_off = A.t_off;
      P.bc_tlast = A.bc_tlast;
      if (direct) {  // straight into the receiving rank's arena slot [p][f ^ 1][epoch]
        auto* peer = static_cast<double2*>(T->peer_arena(ctx->rank, dr, ctx->plan.partner[f]));
        if (!peer) throw Error(LBCU_TRANSPORT_ERROR, "direct halo: peer arena not mapped");
        P.outbuf = peer + arena_off(p, f ^ 1);
      } else {
        P.outbuf = hb.send[p][f];
      }
      PA.first[PA.njobs] = pack_blocks;
      pack_blocks += (P.count + kBlock - 1) / kBlock;
      PA.njobs++;
      // face f goes to partner[f]; the matching halo arrives from the opposite
      // partner into recv[f ^ 1] (dir 0 record -> receiver's forward halo)
      Transport::Msg m;
      m.send = hb.send[p][f];
      m.recv = hb.recv[p][f ^ 1];
      m.bytes = sizeof(double2) * 2 * dr * ctx->plan.count[f];
      m.peer_send = ctx->plan.partner[f];
      m.peer_recv = ctx->plan.partner[f ^ 1];
      msgs.push_back(m);
    }
  }
  PA.first[PA.njobs] = pack_blocks;
  // The pack (and, for message transports, the exchange) runs on the
  // high-priority comm stream, forked from the compute stream, so the
  // interior launch below runs concurrently with it: with a direct transport
  // the pack's NVLink stores into the peers' arenas overlap the interior
  // stencil; with NCCL the pack + send/recv do.
  const cudaStream_t cs = ctx->comm_stream;
  LBCU_CUDA(cudaEventRecord(ctx->ev_fork, s));
  LBCU_CUDA(cudaStreamWaitEvent(cs, ctx->ev_fork, 0));
  if (pack_blocks > 0) {
    dispatch(dr, real, fmt, [&](auto Dc, auto Rc, auto Fc) {
      pack_kernel<LBCU_TPARAMS(Dc, Rc, Fc)><<<pack_blocks, kBlock, 0, cs>>>(PA);
    });
    ctx->launches += 1;
    LBCU_CUDA(cudaGetLastError());
  }
  // launch groups: both parities in one launch when their site counts agree
  const bool joint = npar == 2 && ctx->nint[0] == ctx->nint[1] && ctx->nbnd[0] == ctx->nbnd[1];
  const int ngroups = joint ? 1 : npar;
  int int_blocks[2] = {0, 0}, bnd_blocks[2] = {0, 0}, total_blocks = 0;
  for (int gi = 0; gi < ngroups; ++gi) {
    const int p = pars[gi], np = joint ? 2 : 1;
    int_blocks[gi] = hop_blocks(ctx->nint[p], np, dr);
    bnd_blocks[gi] = hop_blocks(ctx->nbnd[p], np, dr);
    total_blocks += int_blocks[gi] + bnd_blocks[gi];
  }
  if (reduce && total_blocks > ctx->max_partials) throw Error(LBCU_CUDA_ERROR, "reduction workspace too small");
  auto group_args = [&](int gi, bool bnd) {
    HopArgs G = A;
    const int p = pars[gi];
    G.both = joint ? 1 : 0;
    G.par0 = p;
    G.nsites = bnd ? ctx->nbnd[p] : ctx->nint[p];
    for (int pp = 0; pp < 2; ++pp) {
      const bool run = !bnd && ctx->int_lo[pp] >= 0;
      G.list[pp] = run ? nullptr : bnd ? ctx->blist[pp] : ctx->ilist[pp];
      G.ioff[pp] = run ? ctx->int_lo[pp] : 0;
    }
    int off = 0;
    for (int g2 = 0; g2 < gi; ++g2) off += int_blocks[g2] + bnd_blocks[g2];
    if (bnd) off += int_blocks[gi];
    if (reduce) G.red = Reduce{ctx->partials, c.result, off, total_blocks};
    return G;
  };
  // interior sites (no halo dependency) run on the compute stream while the
  // halos travel; boundary sites wait for them. Direct transports: the pack
  // kernel stores into the peers, its completion is posted as an event that
  // the peers' compute streams wait on before their boundary launch.
  if (direct) T->post(ctx->rank, epoch, cs);
  LBCU_CUDA(cudaEventRecord(ctx->ev_pack, cs));
  // warp-shared z hops for a contiguous interior whose warps cover whole z-rows
  const int hz = geo.local[3] / 2;
  for (int gi = 0; gi < ngroups; ++gi) {
    HopArgs Ai = group_args(gi, false);
    const bool zs = env_int("LBCU_HOP_ZS", 1) && !geo.decomposed[3] && hz > 0 && 32 % hz == 0 &&
                    ctx->int_lo[0] >= 0 && ctx->int_lo[1] >= 0 && ctx->int_lo[0] % 32 == 0 &&
                    ctx->int_lo[1] % 32 == 0;
    dispatch(dr, real, fmt, [&](auto Dc, auto Rc, auto Fc) {
      launch_hop<LBCU_TPARAMS(Dc, Rc, Fc)>(Ai, false, c.epi, Ai.nsites, joint ? 2 : 1, s, 0, zs);
    });
    ctx->launches += 1;
  }
  if (direct) {
    // join the own pack (it reads `in`, which later work on s may overwrite;
    // the chain pack(k+2) after boundary(k+1) keeps the arena slots safe),
    // then every peer's pack of this exchange
    LBCU_CUDA(cudaStreamWaitEvent(s, ctx->ev_pack, 0));
    std::vector<int> peers;
    for (int f = 0; f < 8; ++f)
      if (ctx->plan.count[f] && std::find(peers.begin(), peers.end(), ctx->plan.partner[f]) == peers.end())
        peers.push_back(ctx->plan.partner[f]);
    T->await(ctx->rank, epoch, peers, s);
  } else {
    T->exchange(ctx->rank, msgs, cs);  // after the interior launch: may block the host
    LBCU_CUDA(cudaEventRecord(ctx->ev_comm, cs));
    LBCU_CUDA(cudaStreamWaitEvent(s, ctx->ev_comm, 0));
  }
  for (int gi = 0; gi < ngroups; ++gi) {
    HopArgs Ab = group_args(gi, true);
    for (int pp = 0; pp < 2; ++pp)
      for (int mu = 0; mu < 4; ++mu) {
        // recv[2 mu + 1] holds the +mu partner's dir-0 face (forward halo),
        // recv[2 mu] the -mu partner's dir-1 face (backward halo)
        Ab.hfwd[pp][mu] = direct ? hb.arena + arena_off(pp, 2 * mu + 1) : hb.recv[pp][2 * mu + 1];
        Ab.hbwd[pp][mu] = direct ? hb.arena + arena_off(pp, 2 * mu + 0) : hb.recv[pp][2 * mu + 0];
        Ab.hcount[mu] = static_cast<int>(ctx->plan.count[2 * mu]);
      }
    dispatch(dr, real, fmt, [&](auto Dc, auto Rc, auto Fc) {
      launch_hop<LBCU_TPARAMS(Dc, Rc, Fc)>(Ab, true, c.epi, Ab.nsites, joint ? 2 : 1, s);
    });
    ctx->launches += 1;
  }
  if (reduce) {  // all interior and boundary partials are in place
    Reduce R{ctx->partials, c.result, 0, total_blocks};
    k_reduce_finish<1><<<1, kFinishThreads, 0, s>>>(R);
    ctx->launches += 1;
  }
  LBCU_CUDA(cudaGetLastError());
}

}  // namespace lbcu
