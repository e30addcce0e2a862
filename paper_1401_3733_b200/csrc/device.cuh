// Device-side building blocks shared by the kernels: even-odd indexing,
// the gamma-basis spin tables, unit-phase arithmetic and deterministic
// block reductions.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lbcu {

// Per-site arrays (spinor components, link entries) of one parity block are
// tiled by 32 cb sites: element e of site i, with nc elements per site, sits at
//   (i / 32) * nc * 32 + e * 32 + i % 32.
// A warp over 32 consecutive sites still reads one 512-byte segment per
// element, and element offsets inside a tile are compile-time immediates
// (one 64-bit site address per neighbour instead of one per element).
constexpr int kTile = 32;
__host__ __device__ __forceinline__ long long eidx(int nc, int e, long long i) {
  return (i >> 5) * (32LL * nc) + 32LL * e + (i & 31);
}
template <int NC, class T>
__host__ __device__ __forceinline__ T* site_ptr(T* base, long long i) {
  return base + (i >> 5) * (32LL * NC) + (i & 31);
}

// Local lattice as seen by a kernel. Sites of one parity are stored in
// "checkerboard" order cb = s >> 1 of the local lexicographic index s
// (t,x,y,z; z fastest). Every local extent is even, so (z, z+1) pairs split
// across parities and each parity block is dense.
struct DevGeo {
  int L[4];       // local extents t, x, y, z
  int sx[4];      // lexicographic strides: Lx*Ly*Lz, Ly*Lz, Lz, 1
  int vh;         // sites per parity
  long long stride;  // component stride of one parity block (>= vh)
  int wrap[4];    // 1: direction not decomposed -> local periodic wrap
};

// cb index + parity -> local coordinates and lexicographic index
__device__ __forceinline__ void cb_coords(const DevGeo& g, int i, int par, int c[4], int& s) {
  const int s0 = 2 * i;
  const int z0 = s0 % g.L[3];
  int r = s0 / g.L[3];
  c[2] = r % g.L[2];
  r /= g.L[2];
  c[1] = r % g.L[1];
  c[0] = r / g.L[1];
  const int dz = (c[0] + c[1] + c[2] + z0 + par) & 1;
  c[3] = z0 + dz;
  s = s0 + dz;
}

// lexicographic neighbour of s in direction mu (periodic inside the rank)
__device__ __forceinline__ int nb_fwd(const DevGeo& g, int s, const int c[4], int mu) {
  return (c[mu] + 1 < g.L[mu]) ? s + g.sx[mu] : s - (g.L[mu] - 1) * g.sx[mu];
}
__device__ __forceinline__ int nb_bwd(const DevGeo& g, int s, const int c[4], int mu) {
  return (c[mu] > 0) ? s - g.sx[mu] : s + (g.L[mu] - 1) * g.sx[mu];
}

// in-face lexicographic position over the three coordinates other than mu
__device__ __forceinline__ int face_pos(const DevGeo& g, const int c[4], int mu) {
  int p = 0;
#pragma unroll
  for (int d = 0; d < 4; ++d)
    if (d != mu) p = p * g.L[d] + c[d];
  return p;
}

// ---- gamma basis (proj/src/gamma.cpp:46-61, chiral, gamma5 = diag(1,1,-1,-1)).
// Unit phases P1, M1, PI, MI as 0..3 (proj/include/latbench/gamma.hpp:18);
// negation flips the low bit. (1 - gamma_mu) psi projects to
//   h_a = psi_a + PROJ_PH[mu][a] psi_{PAIR[mu][a]}, a = 0, 1
// and reconstructs as (h0, h1, REC_PH[mu][0] h_{REC[mu][0]}, REC_PH[mu][1] h_{REC[mu][1]}).
// (1 + gamma_mu) uses the same pairs with negated phases.
template <int MU>
struct Gam;
template <>
struct Gam<0> {
  static constexpr int p0 = 2, p1 = 3, f0 = 0, f1 = 0, r0 = 0, r1 = 1, q0 = 0, q1 = 0;
};
template <>
struct Gam<1> {
  static constexpr int p0 = 3, p1 = 2, f0 = 2, f1 = 2, r0 = 1, r1 = 0, q0 = 3, q1 = 3;
};
template <>
struct Gam<2> {
  static constexpr int p0 = 3, p1 = 2, f0 = 0, f1 = 1, r0 = 1, r1 = 0, q0 = 1, q1 = 0;
};
template <>
struct Gam<3> {
  static constexpr int p0 = 2, p1 = 3, f0 = 2, f1 = 3, r0 = 0, r1 = 1, q0 = 3, q1 = 2;
};

template <int P>
__device__ __forceinline__ double2 phm(double2 z) {
  if constexpr (P == 0) return z;
  else if constexpr (P == 1) return make_double2(-z.x, -z.y);
  else if constexpr (P == 2) return make_double2(-z.y, z.x);
  else return make_double2(z.y, -z.x);
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
// a or -a by a sign mask (0 or 1 << 63 in the high word): the +-1 factors of
// the hop (gamma5 on the input, the antiperiodic time sign). As an fp64
// multiply by default; -DLBCU_SIGN_XOR=1 flips the sign bit with an integer
// XOR instead (moves the work off the fp64 pipe, but measured 2-4 % slower for
// the SU(2) hop and neutral for SU(3): profiles/r2e_ab_sign.log)
__host__ __device__ __forceinline__ unsigned sign_mask(bool neg) { return neg ? 0x80000000u : 0u; }
#if LBCU_SIGN_XOR
__device__ __forceinline__ double flip(double a, unsigned m) {
  return __hiloint2double(__double2hiint(a) ^ static_cast<int>(m), __double2loint(a));
}
__device__ __forceinline__ double2 cflip(unsigned m, double2 a) { return make_double2(flip(a.x, m), flip(a.y, m)); }
#else
__device__ __forceinline__ double2 cflip(unsigned m, double2 a) { return cscale(m ? -1.0 : 1.0, a); }
#endif

// acc += u * v
__device__ __forceinline__ void cmac(double2& acc, double2 u, double2 v) {
  acc.x = fma(u.x, v.x, fma(-u.y, v.y, acc.x));
  acc.y = fma(u.x, v.y, fma(u.y, v.x, acc.y));
}
// acc += conj(u) * v
__device__ __forceinline__ void cmac_conj(double2& acc, double2 u, double2 v) {
  acc.x = fma(u.x, v.x, fma(u.y, v.y, acc.x));
  acc.y = fma(u.x, v.y, fma(-u.y, v.x, acc.y));
}
// acc += r * v (real link)
__device__ __forceinline__ void rmac(double2& acc, double u, double2 v) {
  acc.x = fma(u, v.x, acc.x);
  acc.y = fma(u, v.y, acc.y);
}

template <class T>
__device__ __forceinline__ T ldg(const T* p) {
  return __ldg(p);
}

// ---- deterministic reductions ---------------------------------------------
// Each block reduces NR values (warp shuffles + shared memory) and writes its
// partials to part[(offset + blockIdx) * NR + k]; k_reduce_finish, launched
// after the last contributing kernel, sums all partials in a fixed order and
// writes result[k], so the value does not depend on block scheduling.
// Device CG state (one per context, solver.cpp).
struct CgState {
  double rr, rr_new, pap, alpha, beta, bnorm, tol, best, rel;
  long long k, maxit;
  int conv, done;
};

// CG scalar steps (solver.cpp:53-69), run by one thread: either a 1-thread
// kernel after a multi-rank allreduce, or fused into the last block of the
// reduction that produced the value (single rank).
// Every CG state step is a no-op once the solve is done: the multi-rank host
// loop enqueues iteration k + 1 before it has read iteration k's state, and
// that speculative iteration must leave x, p and the state untouched.
__device__ __forceinline__ void cg_post_alpha(CgState* st, double pap) {
  if (st->done) return;
  st->pap = pap;
  st->alpha = st->rr / pap;
}

__device__ __forceinline__ void cg_post_end(CgState* st, double rrn, double* hist,
                                            unsigned long long handle, int use_graph) {
  if (st->done) return;
  const double rel = sqrt(rrn) / st->bnorm;
  const long long k = st->k;
  hist[k] = rel;
  st->rel = rel;
  st->rr_new = rrn;
  if (rel < st->best) st->best = rel;
  st->k = k + 1;
  if (rel < st->tol) {
    st->conv = 1;
    st->done = 1;
  } else if (k + 1 >= st->maxit) {
    st->done = 1;
  }
  st->beta = rrn / st->rr;
  st->rr = rrn;
  if (use_graph) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(handle), st->done ? 0u : 1u);
}

enum RedPost { POST_NONE = 0, POST_ALPHA = 1, POST_END = 2 };

struct Reduce {
  double* part;        // partials, >= total_blocks * NR
  double* result;      // NR outputs
  int offset;          // this launch's first partial slot
  int total_blocks;    // partial slots over all launches that feed this result
  // optional CG scalar step on result[0] by k_reduce_finish
  int post;
  CgState* cg;
  double* hist;
  unsigned long long handle;
  int use_graph;
};

// Split form (measured: profiles/r03_cg_epilogue_breakdown.txt): each block
// only writes its partial (no fence, no atomic ticket, so it retires as soon
// as its warps are done), and k_reduce_finish sums the partials in a fixed
// order and runs the CG step. The earlier last-block form (fence + atomic +
// second barrier in every block) kept every block's registers idle for ~2 us
// and cost 20-29 us per 0.5 M-site eo hop.
template <int NR>
__device__ __forceinline__ void block_reduce_partial(const Reduce& R, double (&v)[NR]) {
  __shared__ double sh[32][NR];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int k = 0; k < NR; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NR; ++k) sh[warp][k] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += sh[w][k];
      R.part[(size_t)(R.offset + blockIdx.x) * NR + k] = s;
    }
  }
}

constexpr int kFinishThreads = 1024;

template <int NR>
__global__ void __launch_bounds__(kFinishThreads) k_reduce_finish(const Reduce R) {
  __shared__ double sh[kFinishThreads / 32][NR];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[NR];
#pragma unroll
  for (int k = 0; k < NR; ++k) acc[k] = 0.0;
  // 8 independent loads in flight per thread, then a fixed-order sum
  constexpr int U = 8;
  for (int base = 0; base < R.total_blocks; base += U * kFinishThreads) {
    double v[U][NR];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int b = base + j * kFinishThreads + threadIdx.x;
#pragma unroll
      for (int k = 0; k < NR; ++k) v[j][k] = b < R.total_blocks ? R.part[(size_t)b * NR + k] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < U; ++j)
#pragma unroll
      for (int k = 0; k < NR; ++k) acc[k] += v[j][k];
  }
#pragma unroll
  for (int k = 0; k < NR; ++k)
    for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_down_sync(0xffffffffu, acc[k], o);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NR; ++k) sh[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      double s = 0.0;
      for (int w = 0; w < kFinishThreads / 32; ++w) s += sh[w][k];
      R.result[k] = s;
    }
    if (R.post == POST_ALPHA) cg_post_alpha(R.cg, R.result[0]);
    else if (R.post == POST_END) cg_post_end(R.cg, R.result[0], R.hist, R.handle, R.use_graph);
  }
}

}  // namespace lbcu
