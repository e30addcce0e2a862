// Wilson hopping term on the even-odd SoA layout (sm_100a).
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
// Memory layout: every spinor component / link entry is a contiguous
// double2 (or double for real links) array over checkerboard sites, so a warp
// issues fully coalesced 512-byte (LDG.128) loads for each component.
//
// Decomposed directions: boundary sites are handled by a second launch that
// reads half-spinor halos produced by pack_kernel on the neighbour rank:
//   face dir 0 (to -mu partner): h = (1 - g_mu) projection of in at x_mu = 0
//   face dir 1 (to +mu partner): g = U_mu(y)^dag (1 + g_mu) projection at
//                                x_mu = L_mu - 1 (no gauge halo needed).
#include <cstdlib>
#include <type_traits>

#include "objects.hpp"

namespace lbcu {

namespace {

struct HopArgs {
  DevGeo g;
  const double2* in[2];  // input blocks indexed by input parity
  double2* out[2];       // output blocks by output parity
  const double2* x[2];   // diagonal-term blocks by output parity (nullable)
  double2* r[2];         // CG residual blocks by output parity
  const void* gauge;     // [2][4][D*D][stride]
  double a, b, s5in, s5x, s5acc;
  const double* alpha;
  int par0;    // output parity of a single-parity launch
  int both;    // 1: parity = blockIdx.x & 1
  int nsites;  // sites per parity
  const int* list[2];
  const double2* hfwd[4];
  const double2* hbwd[4];
  int hcount[4];
  Reduce red;
};

template <bool REAL>
using LinkT = std::conditional_t<REAL, double, double2>;

template <int D, bool REAL>
__device__ __forceinline__ void umul(double2 (&g)[2][D], const LinkT<REAL>* __restrict__ U,
                                     long long st, int site, const double2 (&h)[2][D],
                                     bool dagger) {
#pragma unroll
  for (int r = 0; r < D; ++r) {
    g[0][r] = make_double2(0.0, 0.0);
    g[1][r] = make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int r = 0; r < D; ++r)
#pragma unroll
    for (int c = 0; c < D; ++c) {
      if constexpr (REAL) {
        const double u = ldg(U + (long long)(dagger ? c * D + r : r * D + c) * st + site);
        rmac(g[0][r], u, h[0][c]);
        rmac(g[1][r], u, h[1][c]);
      } else {
        const double2 u = ldg(U + (long long)(dagger ? c * D + r : r * D + c) * st + site);
        if (dagger) {
          cmac_conj(g[0][r], u, h[0][c]);
          cmac_conj(g[1][r], u, h[1][c]);
        } else {
          cmac(g[0][r], u, h[0][c]);
          cmac(g[1][r], u, h[1][c]);
        }
      }
    }
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

// h_a = psi_a + F_a * s5 * psi_{p_a}: spin projection of the spinor at cb site nb
template <int D, int P0, int P1, int F0, int F1>
__device__ __forceinline__ void project(double2 (&h)[2][D], const double2* __restrict__ in,
                                        long long st, int nb, double s5) {
#pragma unroll
  for (int c = 0; c < D; ++c) {
    const double2 a0 = ldg(in + (long long)(0 * D + c) * st + nb);
    const double2 a1 = ldg(in + (long long)(1 * D + c) * st + nb);
    const double2 b0 = ldg(in + (long long)(P0 * D + c) * st + nb);
    const double2 b1 = ldg(in + (long long)(P1 * D + c) * st + nb);
    h[0][c] = cadd(a0, phm<F0>(cscale(s5, b0)));
    h[1][c] = cadd(a1, phm<F1>(cscale(s5, b1)));
  }
}

template <int D, bool REAL, bool BND, int MU>
__device__ __forceinline__ void hop_mu(double2 (&acc)[4][D], const HopArgs& A,
                                       const double2* __restrict__ in,
                                       const LinkT<REAL>* __restrict__ Uown,
                                       const LinkT<REAL>* __restrict__ Uoth, int i, int s,
                                       const int c[4]) {
  using G = Gam<MU>;
  const long long st = A.g.stride;
  const LinkT<REAL>* Uo = Uown + (long long)MU * D * D * st;
  const LinkT<REAL>* Ub = Uoth + (long long)MU * D * D * st;
  {  // forward: (1 - g_mu) U_mu(x) in(x + mu)
    double2 h[2][D], g[2][D];
    if (BND && !A.g.wrap[MU] && c[MU] == A.g.L[MU] - 1) {
      const int j = face_pos(A.g, c, MU) >> 1;
      const int hc = A.hcount[MU];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int cc = 0; cc < D; ++cc) h[a][cc] = ldg(A.hfwd[MU] + (a * D + cc) * hc + j);
    } else {
      project<D, G::p0, G::p1, G::f0, G::f1>(h, in, st, nb_fwd(A.g, s, c, MU) >> 1, A.s5in);
    }
    umul<D, REAL>(g, Uo, st, i, h, false);
    reconstruct<D, G::r0, G::r1, G::q0, G::q1>(acc, g);
  }
  {  // backward: (1 + g_mu) U_mu(x - mu)^dag in(x - mu)
    double2 g[2][D];
    if (BND && !A.g.wrap[MU] && c[MU] == 0) {
      const int j = face_pos(A.g, c, MU) >> 1;
      const int hc = A.hcount[MU];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int cc = 0; cc < D; ++cc) g[a][cc] = ldg(A.hbwd[MU] + (a * D + cc) * hc + j);
    } else {
      double2 h[2][D];
      const int nb = nb_bwd(A.g, s, c, MU) >> 1;
      project<D, G::p0, G::p1, G::f0 ^ 1, G::f1 ^ 1>(h, in, st, nb, A.s5in);
      umul<D, REAL>(g, Ub, st, nb, h, true);
    }
    reconstruct<D, G::r0, G::r1, G::q0 ^ 1, G::q1 ^ 1>(acc, g);
  }
}

template <int D, bool REAL, bool BND, int EPI, int MINB>
__global__ void __launch_bounds__(128, MINB) hop_kernel(const __grid_constant__ HopArgs A) {
  int par, idx;
  if (A.both) {
    par = blockIdx.x & 1;
    idx = (blockIdx.x >> 1) * blockDim.x + threadIdx.x;
  } else {
    par = A.par0;
    idx = blockIdx.x * blockDim.x + threadIdx.x;
  }
  double nrm[1] = {0.0};
  if (idx < A.nsites) {
    const int i = A.list[par] ? A.list[par][idx] : idx;
    int c[4], s;
    cb_coords(A.g, i, par, c, s);
    double2 acc[4][D];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) acc[k][cc] = make_double2(0.0, 0.0);
    const long long st = A.g.stride;
    const LinkT<REAL>* Ug = static_cast<const LinkT<REAL>*>(A.gauge);
    const LinkT<REAL>* Uown = Ug + (long long)par * 4 * D * D * st;
    const LinkT<REAL>* Uoth = Ug + (long long)(par ^ 1) * 4 * D * D * st;
    const double2* in = A.in[par ^ 1];
    hop_mu<D, REAL, BND, 0>(acc, A, in, Uown, Uoth, i, s, c);
    hop_mu<D, REAL, BND, 1>(acc, A, in, Uown, Uoth, i, s, c);
    hop_mu<D, REAL, BND, 2>(acc, A, in, Uown, Uoth, i, s, c);
    hop_mu<D, REAL, BND, 3>(acc, A, in, Uown, Uoth, i, s, c);

    const double2* x = A.x[par];
    double2* out = A.out[par];
    double2* r = A.r[par];
    const double alpha = (EPI == EPI_CG) ? *A.alpha : 0.0;
#pragma unroll
    for (int sp = 0; sp < 4; ++sp)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) {
        const long long o = (long long)(sp * D + cc) * st + i;
        const double bs = sp < 2 ? A.b : A.b * A.s5acc;
        double2 v = cscale(bs, acc[sp][cc]);
        if (x) {
          const double as = sp < 2 ? A.a : A.a * A.s5x;
          const double2 xv = ldg(x + o);
          v.x = fma(as, xv.x, v.x);
          v.y = fma(as, xv.y, v.y);
        }
        if constexpr (EPI == EPI_CG) {
          double2 rv = r[o];
          rv.x = fma(-alpha, v.x, rv.x);
          rv.y = fma(-alpha, v.y, rv.y);
          r[o] = rv;
          nrm[0] = fma(rv.x, rv.x, fma(rv.y, rv.y, nrm[0]));
        } else {
          out[o] = v;
          if constexpr (EPI == EPI_STORE_NORM) nrm[0] = fma(v.x, v.x, fma(v.y, v.y, nrm[0]));
        }
      }
  }
  if constexpr (EPI != EPI_STORE) block_reduce_finalize<1>(A.red, nrm);
}

// Pack one face of the input field into half-spinor records (see header).
struct PackArgs {
  DevGeo g;
  const double2* in;  // input parity block
  const void* gauge;
  int in_par, mu, dir, count;
  double s5in;
  double2* outbuf;  // [2D][count]
};

template <int D, bool REAL, int MU>
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
    double2 g[2][D];
    const LinkT<REAL>* U =
        static_cast<const LinkT<REAL>*>(P.gauge) + (long long)(P.in_par * 4 + MU) * D * D * st;
    umul<D, REAL>(g, U, st, cb, h, true);
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int cc = 0; cc < D; ++cc) P.outbuf[(a * D + cc) * P.count + j] = g[a][cc];
  }
}

template <int D, bool REAL>
__global__ void __launch_bounds__(128) pack_kernel(const __grid_constant__ PackArgs P) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P.count) return;
  switch (P.mu) {
    case 0: pack_site<D, REAL, 0>(P, j); break;
    case 1: pack_site<D, REAL, 1>(P, j); break;
    case 2: pack_site<D, REAL, 2>(P, j); break;
    default: pack_site<D, REAL, 3>(P, j); break;
  }
}

constexpr int kBlock = 128;

// Occupancy knob: LBCU_HOP_MINB = minimum resident 128-thread blocks per SM
// requested from ptxas (__launch_bounds__), i.e. a register cap. Measured
// defaults per representation dimension; 1 = no cap.
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

template <int D, bool REAL>
int default_minb() {
  // profiles/r01_tune_minb_cfg*.log: a cap of 3 blocks/SM helps D = 2 and
  // D = 3 (2-4 %); larger D spill under any cap.
  return D <= 3 ? 3 : 1;
}

template <int D, bool REAL>
int hop_blocks(int nsites, int npar) {
  return (nsites + kBlock - 1) / kBlock * npar;
}

template <int D, bool REAL, int MINB>
void launch_hop_minb(const HopArgs& A, bool bnd, int epi, int blocks, cudaStream_t s) {
#define LBCU_HOP_CASE(B, E)                                                         \
  if (bnd == B && epi == E) {                                                       \
    hop_kernel<D, REAL, B, E, MINB><<<blocks, kBlock, 0, s>>>(A);                   \
    return;                                                                         \
  }
  LBCU_HOP_CASE(false, EPI_STORE)
  LBCU_HOP_CASE(false, EPI_STORE_NORM)
  LBCU_HOP_CASE(false, EPI_CG)
  LBCU_HOP_CASE(true, EPI_STORE)
  LBCU_HOP_CASE(true, EPI_STORE_NORM)
  LBCU_HOP_CASE(true, EPI_CG)
#undef LBCU_HOP_CASE
}

template <int D, bool REAL>
void launch_hop(const HopArgs& A, bool bnd, int epi, int nsites, int npar, cudaStream_t s) {
  if (nsites <= 0) return;
  const int blocks = hop_blocks<D, REAL>(nsites, npar);
  switch (env_int("LBCU_HOP_MINB", default_minb<D, REAL>())) {
    case 3: launch_hop_minb<D, REAL, 3>(A, bnd, epi, blocks, s); return;
    default: launch_hop_minb<D, REAL, 1>(A, bnd, epi, blocks, s); return;
  }
}

template <int D, bool REAL>
void launch_pack(const PackArgs& P, cudaStream_t s) {
  pack_kernel<D, REAL><<<(P.count + kBlock - 1) / kBlock, kBlock, 0, s>>>(P);
}

// Supported representation dimensions (compile-time specialisations).
// complex: SU(2)F 2, SU(3)F/SU(3)AS 3, SU(4)F 4, SU(4)AS/SU(3)S/SU(6)F 6,
//          SU(4)S 10; real: SU(2)A 3, SU(3)A 8.
template <class F>
void dispatch_rep(int dr, bool real, F&& f) {
  if (!real) {
    switch (dr) {
      case 2: f(std::integral_constant<int, 2>{}, std::false_type{}); return;
      case 3: f(std::integral_constant<int, 3>{}, std::false_type{}); return;
      case 4: f(std::integral_constant<int, 4>{}, std::false_type{}); return;
      case 6: f(std::integral_constant<int, 6>{}, std::false_type{}); return;
      case 10: f(std::integral_constant<int, 10>{}, std::false_type{}); return;
    }
  } else {
    switch (dr) {
      case 3: f(std::integral_constant<int, 3>{}, std::true_type{}); return;
      case 8: f(std::integral_constant<int, 8>{}, std::true_type{}); return;
    }
  }
  throw Error(LBCU_CONFIG_ERROR, "no device specialisation for representation dimension " +
                                     std::to_string(dr) + (real ? " (real)" : " (complex)"));
}

HaloBufs& halo_bufs(lbcu_ctx_s* ctx, int dr) {
  HaloBufs& hb = ctx->halo[dr];
  size_t need = 0;
  for (int f = 0; f < 8; ++f) need = std::max<size_t>(need, 2 * dr * ctx->plan.count[f]);
  if (hb.cap < need) {
    for (int f = 0; f < 8; ++f) {
      if (hb.send[f]) cudaFree(hb.send[f]);
      if (hb.recv[f]) cudaFree(hb.recv[f]);
      hb.send[f] = hb.recv[f] = nullptr;
      if (ctx->plan.count[f] == 0) continue;
      LBCU_CUDA(cudaMalloc(&hb.send[f], need * sizeof(double2)));
      LBCU_CUDA(cudaMalloc(&hb.recv[f], need * sizeof(double2)));
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
  A.s5in = c.s5in;
  A.s5x = c.s5x;
  A.s5acc = c.s5acc;
  A.alpha = c.alpha;
  const bool reduce = c.epi != EPI_STORE;
  cudaStream_t s = ctx->stream;

  if (!geo.any_decomposed) {
    A.nsites = static_cast<int>(geo.vh);
    A.both = npar == 2;
    A.par0 = pars[0];
    int blocks = 0;
    dispatch_rep(dr, real, [&](auto Dc, auto Rc) {
      blocks = hop_blocks<decltype(Dc)::value, decltype(Rc)::value>(A.nsites, npar);
    });
    if (reduce) {
      if (blocks > ctx->max_partials) throw Error(LBCU_CUDA_ERROR, "reduction workspace too small");
      A.red = Reduce{ctx->partials, ctx->ticket, c.result, 0, blocks};
    }
    dispatch_rep(dr, real, [&](auto Dc, auto Rc) {
      launch_hop<decltype(Dc)::value, decltype(Rc)::value>(A, false, c.epi, A.nsites, npar, s);
    });
    ctx->launches += 1;
    LBCU_CUDA(cudaGetLastError());
    return;
  }

  // ---- decomposed: pack -> exchange -> interior -> boundary -------------
  HaloBufs& hb = halo_bufs(ctx, dr);
  int total_blocks = 0, bnd_off[2] = {0, 0}, int_blocks[2] = {0, 0}, bnd_blocks[2] = {0, 0};
  for (int k = 0; k < npar; ++k) {
    const int p = pars[k];
    dispatch_rep(dr, real, [&](auto Dc, auto Rc) {
      int_blocks[k] = hop_blocks<decltype(Dc)::value, decltype(Rc)::value>(ctx->nint[p], 1);
      bnd_blocks[k] = hop_blocks<decltype(Dc)::value, decltype(Rc)::value>(ctx->nbnd[p], 1);
    });
    total_blocks += int_blocks[k] + bnd_blocks[k];
  }
  if (reduce && total_blocks > ctx->max_partials)
    throw Error(LBCU_CUDA_ERROR, "reduction workspace too small");
  // the exchange for one output parity at a time keeps message buffers simple
  for (int k = 0; k < npar; ++k) {
    const int p = pars[k], q = p ^ 1;
    std::vector<Transport::Msg> msgs;
    for (int f = 0; f < 8; ++f) {
      if (ctx->plan.count[f] == 0) continue;
      PackArgs P{};
      P.g = ctx->dgeo;
      P.in = c.in->par[q];
      P.gauge = c.g->base;
      P.in_par = q;
      P.mu = f / 2;
      P.dir = f % 2;
      P.count = static_cast<int>(ctx->plan.count[f]);
      P.s5in = c.s5in;
      P.outbuf = hb.send[f];
      dispatch_rep(dr, real, [&](auto Dc, auto Rc) {
        launch_pack<decltype(Dc)::value, decltype(Rc)::value>(P, s);
      });
      ctx->launches += 1;
      // face f goes to partner[f]; the matching halo arrives from the opposite
      // partner into recv[f ^ 1] (dir 0 record -> receiver's forward halo)
      Transport::Msg m;
      m.send = hb.send[f];
      m.recv = hb.recv[f ^ 1];
      m.bytes = sizeof(double2) * 2 * dr * ctx->plan.count[f];
      m.peer_send = ctx->plan.partner[f];
      m.peer_recv = ctx->plan.partner[f ^ 1];
      msgs.push_back(m);
    }
    LBCU_CUDA(cudaGetLastError());
    // interior sites (no halo dependency) run on the compute stream while the
    // halos travel on the comm stream; boundary sites wait for both.
    HopArgs Ai = A;
    Ai.both = 0;
    Ai.par0 = p;
    Ai.nsites = ctx->nint[p];
    Ai.list[p] = ctx->ilist[p];
    int off = 0;
    for (int kk = 0; kk < k; ++kk) off += int_blocks[kk] + bnd_blocks[kk];
    if (reduce) Ai.red = Reduce{ctx->partials, ctx->ticket, c.result, off, total_blocks};
    LBCU_CUDA(cudaEventRecord(ctx->ev_pack, s));
    dispatch_rep(dr, real, [&](auto Dc, auto Rc) {
      launch_hop<decltype(Dc)::value, decltype(Rc)::value>(Ai, false, c.epi, Ai.nsites, 1, s);
    });
    ctx->launches += 1;
    LBCU_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_pack, 0));
    ctx->world->t->exchange(ctx->rank, msgs, ctx->comm_stream);
    LBCU_CUDA(cudaEventRecord(ctx->ev_comm, ctx->comm_stream));
    LBCU_CUDA(cudaStreamWaitEvent(s, ctx->ev_comm, 0));
    HopArgs Ab = Ai;
    Ab.nsites = ctx->nbnd[p];
    Ab.list[p] = ctx->blist[p];
    for (int mu = 0; mu < 4; ++mu) {
      // recv[2 mu + 1] holds the +mu partner's dir-0 face (forward halo),
      // recv[2 mu] the -mu partner's dir-1 face (backward halo)
      Ab.hfwd[mu] = hb.recv[2 * mu + 1];
      Ab.hbwd[mu] = hb.recv[2 * mu + 0];
      Ab.hcount[mu] = static_cast<int>(ctx->plan.count[2 * mu]);
    }
    bnd_off[k] = off + int_blocks[k];
    if (reduce) Ab.red = Reduce{ctx->partials, ctx->ticket, c.result, bnd_off[k], total_blocks};
    dispatch_rep(dr, real, [&](auto Dc, auto Rc) {
      launch_hop<decltype(Dc)::value, decltype(Rc)::value>(Ab, true, c.epi, Ab.nsites, 1, s);
    });
    ctx->launches += 1;
    LBCU_CUDA(cudaGetLastError());
  }
}

}  // namespace lbcu
