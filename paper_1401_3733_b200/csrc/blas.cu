// Streaming vector kernels, CG scalar kernels and host<->device layout
// transposes (sm_100a).
//
// Replaces the reference's BLAS-1 helpers (proj/src/kernels.cpp:36-104,
// proj/include/latbench/kernel_ops.hpp:105-121) and its global sums
// (proj/src/transport.cpp:83-100): a spinor's parity blocks are one dense
// double2 array (padding kept at zero), so every vector op is a flat,
// coalesced grid-stride loop with 128-bit accesses; reductions are
// deterministic (fixed-order block partials, see device.cuh).
#include <cstdlib>
#include <cstring>

#include <type_traits>

#include "links.cuh"

#include "objects.hpp"

namespace lbcu {

namespace {

constexpr int kThreads = 256;

int flat_blocks(lbcu_ctx_s* ctx, size_t n) {
  const size_t want = (n + kThreads * 4 - 1) / (kThreads * 4);
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(want, ctx->max_partials)));
}

__global__ void k_sqnorm(const double2* __restrict__ a, size_t n, Reduce R) {
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 z = __ldg(a + i);
    v[0] = fma(z.x, z.x, fma(z.y, z.y, v[0]));
  }
  block_reduce_partial<1>(R, v);
}

// sum conj(a) b
__global__ void k_dot(const double2* __restrict__ a, const double2* __restrict__ b, size_t n, Reduce R) {
  double v[2] = {0.0, 0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 x = __ldg(a + i), y = __ldg(b + i);
    v[0] = fma(x.x, y.x, fma(x.y, y.y, v[0]));
    v[1] = fma(x.x, y.y, fma(-x.y, y.x, v[1]));
  }
  block_reduce_partial<2>(R, v);
}

// y += a x
__global__ void k_axpy(double2* __restrict__ y, const double2* __restrict__ x, size_t n, double ar, double ai) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 xv = __ldg(x + i);
    double2 yv = y[i];
    yv.x = fma(ar, xv.x, fma(-ai, xv.y, yv.x));
    yv.y = fma(ar, xv.y, fma(ai, xv.x, yv.y));
    y[i] = yv;
  }
}

// y = x + a y
__global__ void k_xpay(double2* __restrict__ y, const double2* __restrict__ x, size_t n, double ar, double ai) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 xv = __ldg(x + i);
    const double2 yv = y[i];
    y[i] = make_double2(fma(ar, yv.x, fma(-ai, yv.y, xv.x)), fma(ar, yv.y, fma(ai, yv.x, xv.y)));
  }
}

// negate spin components 2,3: the upper half [2 dr 32, 4 dr 32) of every tile
__global__ void k_gamma5(double2* __restrict__ f, size_t block_elems, size_t half, int nblocks) {
  const size_t n = half * nblocks;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / half, j = i % half;
    double2* p = f + b * block_elems + half + j;
    const double2 v = *p;
    *p = make_double2(-v.x, -v.y);
  }
}

// ---- CG (device scalars in CgState) -------------------------------------
// x += alpha p_old ; p = r + beta p_old      (deferred x update)
__global__ void k_cg_p(double2* __restrict__ p, const double2* __restrict__ r, double2* __restrict__ x,
                       size_t n, const CgState* __restrict__ st) {
  if (st->done) return;  // speculative iteration after convergence (device.cuh)
  const double alpha = st->alpha, beta = st->beta;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 pv = p[i], rv = __ldg(r + i);
    double2 xv = x[i];
    xv.x = fma(alpha, pv.x, xv.x);
    xv.y = fma(alpha, pv.y, xv.y);
    x[i] = xv;
    p[i] = make_double2(fma(beta, pv.x, rv.x), fma(beta, pv.y, rv.y));
  }
}

// r -= alpha ap ; |r|^2
__global__ void k_cg_r(double2* __restrict__ r, const double2* __restrict__ ap, size_t n,
                       const CgState* __restrict__ st, Reduce R) {
  const double alpha = st->alpha;
  double v[1] = {0.0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 a = __ldg(ap + i);
    double2 rv = r[i];
    rv.x = fma(-alpha, a.x, rv.x);
    rv.y = fma(-alpha, a.y, rv.y);
    r[i] = rv;
    v[0] = fma(rv.x, rv.x, fma(rv.y, rv.y, v[0]));
  }
  block_reduce_partial<1>(R, v);
}

// Single-reduction CG (Chronopoulos & Gear), multi-rank runs (solver.cpp):
//   p = r + beta p ; s = w + beta s ; x += alpha p ; r -= alpha s ; |r|^2
// (s = A p and w = A r carried as vectors, so the iteration's two scalars,
// |r|^2 here and (r, A r) from the operator epilogue, meet in one allreduce).
// A no-op once the solve is done (speculative host-loop iteration).
__global__ void k_cg1_update(double2* __restrict__ p, double2* __restrict__ s, double2* __restrict__ x,
                             double2* __restrict__ r, const double2* __restrict__ w, size_t n,
                             const CgState* __restrict__ st, Reduce R) {
  double v[1] = {0.0};
  if (!st->done) {
    const double alpha = st->alpha, beta = st->beta;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const double2 rv = r[i], wv = __ldg(w + i);
      double2 pv = p[i], sv = s[i], xv = x[i];
      pv = make_double2(fma(beta, pv.x, rv.x), fma(beta, pv.y, rv.y));
      sv = make_double2(fma(beta, sv.x, wv.x), fma(beta, sv.y, wv.y));
      xv = make_double2(fma(alpha, pv.x, xv.x), fma(alpha, pv.y, xv.y));
      const double2 rn = make_double2(fma(-alpha, sv.x, rv.x), fma(-alpha, sv.y, rv.y));
      p[i] = pv;
      s[i] = sv;
      x[i] = xv;
      r[i] = rn;
      v[0] = fma(rn.x, rn.x, fma(rn.y, rn.y, v[0]));
    }
  }
  block_reduce_partial<1>(R, v);
}

// start: gd = (|b|^2, (b, A b)) -> alpha_0 = gamma_0 / delta_0, beta_0 = 0
__global__ void k_cg1_start(CgState* st, const double* gd) {
  st->rr = gd[0];
  st->alpha = gd[0] / gd[1];
  st->beta = 0.0;
}

// end of iteration k: gd = (gamma', delta') = (|r'|^2, (r', A r')); history,
// convergence as cg_post_end, then beta = gamma'/gamma,
// alpha' = gamma' / (delta' - beta gamma' / alpha)
__global__ void k_cg1_end(CgState* st, const double* gd, double* hist) {
  if (st->done) return;
  const double g = gd[0], d = gd[1];
  const double rel = sqrt(g) / st->bnorm;
  const long long k = st->k;
  hist[k] = rel;
  st->rel = rel;
  st->rr_new = g;
  if (rel < st->best) st->best = rel;
  st->k = k + 1;
  if (rel < st->tol) {
    st->conv = 1;
    st->done = 1;
  } else if (k + 1 >= st->maxit) {
    st->done = 1;
  }
  const double beta = g / st->rr;
  st->alpha = g / (d - beta * g / st->alpha);
  st->beta = beta;
  st->rr = g;
}

__global__ void k_cg_xfinal(double2* __restrict__ x, const double2* __restrict__ p, size_t n,
                            const CgState* __restrict__ st) {
  const double alpha = st->alpha;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double2 pv = __ldg(p + i);
    double2 xv = x[i];
    xv.x = fma(alpha, pv.x, xv.x);
    xv.y = fma(alpha, pv.y, xv.y);
    x[i] = xv;
  }
}

__global__ void k_cg_init(CgState* st, const double* b2, double tol, long long maxit) {
  st->rr = *b2;
  st->rr_new = *b2;
  st->bnorm = sqrt(*b2);
  st->tol = tol;
  st->best = 1.0;
  st->rel = 1.0;
  st->alpha = 0.0;
  st->beta = 0.0;
  st->pap = 0.0;
  st->k = 0;
  st->maxit = maxit;
  st->conv = 0;
  st->done = 0;
}

__global__ void k_cg_alpha(CgState* st, const double* pap) { cg_post_alpha(st, *pap); }

// end of iteration k (solver.cpp:58-69): relative residual, history,
// convergence, beta, rr <- rr_new; optionally drives a graph while-loop.
__global__ void k_cg_end(CgState* st, const double* rr_new, double* hist,
                         cudaGraphConditionalHandle handle, int use_graph) {
  cg_post_end(st, *rr_new, hist, static_cast<unsigned long long>(handle), use_graph);
}

// ---- layout transposes -----------------------------------------------------
__device__ __forceinline__ double neg(double a) { return -a; }
__device__ __forceinline__ double2 neg(double2 a) { return make_double2(-a.x, -a.y); }

// Host order: site-major local lexicographic records of nv entries.
// Device order: per parity block, nv / ng groups (link: one per mu) of ng
// elements per site, each group stride x ng elements in 32-site tiles (eidx).
// A block stages TS consecutive sites (TS even -> TS/2 cb sites per parity).
// Per (parity, cb) slot of the block's tile: the site's row in the staged
// tile (local lexicographic s - s0), with bit 30 set when the antiperiodic
// sign applies, or -1 past the end. Computed once per site, not per element.
__device__ __forceinline__ void tile_rows(int* rows, long long s0, int half, long long vol, const DevGeo& g,
                                          int sign_t, int t_off) {
  for (int pj = threadIdx.x; pj < 2 * half; pj += blockDim.x) {
    const int p = pj / half, jj = pj - p * half;
    const long long cb = s0 / 2 + jj;
    int row = -1;
    if (2 * cb < vol) {
      int c[4], s;
      cb_coords(g, (int)cb, p, c, s);
      row = static_cast<int>(s - s0) | ((c[0] + t_off == sign_t) ? (1 << 30) : 0);
    }
    rows[pj] = row;
  }
}

// Host AoS (site-major records of nv entries) -> device tiled parity blocks.
// The staged tile uses a row stride of nv + 1 entries, so the column reads of
// the scatter phase (consecutive cb sites = every other row) hit distinct
// shared-memory banks; stores are 32-site coalesced.
template <class T>
__global__ void k_aos_to_soa(const T* __restrict__ src, T* dst0, T* dst1, int nv, int ng, long long vol,
                             long long stride, int TS, DevGeo g, int sign_entries, int sign_t,
                             int t_off) {
  extern __shared__ unsigned char smraw[];
  const int ld = nv + 1;
  T* sm = reinterpret_cast<T*>(smraw);
  int* rows = reinterpret_cast<int*>(sm + (size_t)TS * ld);
  const long long s0 = (long long)blockIdx.x * TS;
  const int half = TS / 2;
  tile_rows(rows, s0, half, vol, g, sign_t, t_off);
  const int tile = TS * nv;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) {
    const int site = e / nv, k = e - site * nv;
    if (s0 + site < vol) sm[site * ld + k] = src[s0 * nv + e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * nv * half; e += blockDim.x) {
    const int jj = e % half, pk = e / half, p = pk & 1, k = pk >> 1;
    T* dst = p ? dst1 : dst0;
    const int row = rows[p * half + jj];
    if (!dst || row < 0) continue;
    T v = sm[(row & ((1 << 30) - 1)) * ld + k];
    if (k < sign_entries && (row >> 30)) v = neg(v);
    dst[(k / ng) * ng * stride + eidx(ng, k % ng, s0 / 2 + jj)] = v;
  }
}

template <class T>
__global__ void k_soa_to_aos(const T* src0, const T* src1, T* __restrict__ dst, int nv, int ng,
                             long long vol, long long stride, int TS, DevGeo g) {
  extern __shared__ unsigned char smraw[];
  const int ld = nv + 1;
  T* sm = reinterpret_cast<T*>(smraw);
  int* rows = reinterpret_cast<int*>(sm + (size_t)TS * ld);
  const long long s0 = (long long)blockIdx.x * TS;
  const int half = TS / 2;
  tile_rows(rows, s0, half, vol, g, -1, 0);
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * nv * half; e += blockDim.x) {
    const int jj = e % half, pk = e / half, p = pk & 1, k = pk >> 1;
    const int row = rows[p * half + jj];
    if (row < 0) continue;
    const T* src = p ? src1 : src0;
    sm[row * ld + k] = src ? src[(k / ng) * ng * stride + eidx(ng, k % ng, s0 / 2 + jj)] : T{};
  }
  __syncthreads();
  const int tile = TS * nv;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) {
    const int site = e / nv, k = e - site * nv;
    if (s0 + site < vol) dst[s0 * nv + e] = sm[site * ld + k];
  }
}

// Spinor fast path: NV = 4 dr entries per site known at compile time, one
// group (ng = nv), 128 sites (2 device tiles per parity) per block, so every
// index split is a shift or a constant division.
template <int NV>
constexpr int kSpTS = NV <= 16 ? 128 : 64;  // static shared memory <= 48 KB
template <int NV>
__global__ void __launch_bounds__(256) k_sp_to_soa(const double2* __restrict__ src, double2* dst0, double2* dst1,
                                                   long long vol, DevGeo g) {
  constexpr int TS = kSpTS<NV>, ld = NV + 1, half = TS / 2;
  __shared__ double2 sm[TS * ld];
  __shared__ int rows[TS];
  const long long s0 = (long long)blockIdx.x * TS;
  tile_rows(rows, s0, half, vol, g, -1, 0);
  for (int e = threadIdx.x; e < TS * NV; e += blockDim.x) {
    const int site = e / NV, k = e - site * NV;
    if (s0 + site < vol) sm[site * ld + k] = src[s0 * NV + e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * NV * half; e += blockDim.x) {
    const int jj = e & (half - 1), pk = e / half, p = pk & 1, k = pk >> 1;
    double2* dst = p ? dst1 : dst0;
    const int row = rows[p * half + jj];
    if (!dst || row < 0) continue;
    dst[eidx(NV, k, s0 / 2 + jj)] = sm[row * ld + k];
  }
}

template <int NV>
__global__ void __launch_bounds__(256) k_sp_to_aos(const double2* src0, const double2* src1,
                                                   double2* __restrict__ dst, long long vol, DevGeo g) {
  constexpr int TS = kSpTS<NV>, ld = NV + 1, half = TS / 2;
  __shared__ double2 sm[TS * ld];
  __shared__ int rows[TS];
  const long long s0 = (long long)blockIdx.x * TS;
  tile_rows(rows, s0, half, vol, g, -1, 0);
  __syncthreads();
  for (int e = threadIdx.x; e < 2 * NV * half; e += blockDim.x) {
    const int jj = e & (half - 1), pk = e / half, p = pk & 1, k = pk >> 1;
    const int row = rows[p * half + jj];
    if (row < 0) continue;
    const double2* src = p ? src1 : src0;
    sm[row * ld + k] = src ? src[eidx(NV, k, s0 / 2 + jj)] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < TS * NV; e += blockDim.x) {
    const int site = e / NV, k = e - site * NV;
    if (s0 + site < vol) dst[s0 * NV + e] = sm[site * ld + k];
  }
}

template <class T>
int tile_sites(int nv) {
  // up to 256 sites (4 device tiles per parity) within ~40 KB of staging
  int ts = static_cast<int>((40 * 1024) / ((nv + 1) * sizeof(T) + sizeof(int)));
  ts = ts >= 64 ? std::min(256, ts) & ~63 : ts & ~1;
  return std::max(2, ts);
}

void ensure_staging(lbcu_ctx_s* ctx, size_t bytes) {
  if (ctx->staging_bytes >= bytes) return;
  if (ctx->staging) LBCU_CUDA(cudaFree(ctx->staging));
  ctx->staging = nullptr;
  LBCU_CUDA(cudaMalloc(&ctx->staging, bytes));
  ctx->staging_bytes = bytes;
}

}  // namespace

static Reduce make_reduce(lbcu_ctx_s* ctx, double* res, int blocks) {
  return Reduce{ctx->partials, res, 0, blocks};
}

void blas_sqnorm(lbcu_ctx_s* ctx, const lbcu_spinor_s* f, double* dres) {
  const int nb = flat_blocks(ctx, f->elems);
  k_sqnorm<<<nb, kThreads, 0, ctx->stream>>>(f->base, f->elems, make_reduce(ctx, dres, nb));
  k_reduce_finish<1><<<1, kFinishThreads, 0, ctx->stream>>>(make_reduce(ctx, dres, nb));
  ctx->launches += 2;
  LBCU_CUDA(cudaGetLastError());
}

void blas_dot(lbcu_ctx_s* ctx, const lbcu_spinor_s* a, const lbcu_spinor_s* b, double* dres2) {
  const int nb = flat_blocks(ctx, a->elems);
  k_dot<<<nb, kThreads, 0, ctx->stream>>>(a->base, b->base, a->elems, make_reduce(ctx, dres2, nb));
  k_reduce_finish<2><<<1, kFinishThreads, 0, ctx->stream>>>(make_reduce(ctx, dres2, nb));
  ctx->launches += 2;
  LBCU_CUDA(cudaGetLastError());
}

void blas_axpy(lbcu_ctx_s* ctx, lbcu_spinor_s* y, double ar, double ai, const lbcu_spinor_s* x) {
  k_axpy<<<flat_blocks(ctx, y->elems), kThreads, 0, ctx->stream>>>(y->base, x->base, y->elems, ar, ai);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void blas_xpay(lbcu_ctx_s* ctx, lbcu_spinor_s* y, double ar, double ai, const lbcu_spinor_s* x) {
  k_xpay<<<flat_blocks(ctx, y->elems), kThreads, 0, ctx->stream>>>(y->base, x->base, y->elems, ar, ai);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void blas_copy(lbcu_ctx_s* ctx, lbcu_spinor_s* dst, const lbcu_spinor_s* src) {
  LBCU_CUDA(cudaMemcpyAsync(dst->base, src->base, dst->elems * sizeof(double2),
                            cudaMemcpyDeviceToDevice, ctx->stream));
}

void blas_zero(lbcu_ctx_s* ctx, lbcu_spinor_s* f) {
  LBCU_CUDA(cudaMemsetAsync(f->base, 0, f->elems * sizeof(double2), ctx->stream));
}

void blas_gamma5(lbcu_ctx_s* ctx, lbcu_spinor_s* f) {
  const size_t blk = static_cast<size_t>(4 * f->dr) * kTile;
  const int nblocks = static_cast<int>(f->elems / blk);
  const size_t half = blk / 2;
  k_gamma5<<<flat_blocks(ctx, half * nblocks), kThreads, 0, ctx->stream>>>(f->base, blk, half, nblocks);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void cg_p_update(lbcu_ctx_s* ctx, lbcu_spinor_s* p, const lbcu_spinor_s* r, lbcu_spinor_s* x) {
  k_cg_p<<<flat_blocks(ctx, p->elems), kThreads, 0, ctx->stream>>>(p->base, r->base, x->base, p->elems, ctx->dcg);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void cg_r_update(lbcu_ctx_s* ctx, lbcu_spinor_s* r, const lbcu_spinor_s* ap, double* dres) {
  const int nb = flat_blocks(ctx, r->elems);
  k_cg_r<<<nb, kThreads, 0, ctx->stream>>>(r->base, ap->base, r->elems, ctx->dcg, make_reduce(ctx, dres, nb));
  k_reduce_finish<1><<<1, kFinishThreads, 0, ctx->stream>>>(make_reduce(ctx, dres, nb));
  ctx->launches += 2;
  LBCU_CUDA(cudaGetLastError());
}

void cg1_update(lbcu_ctx_s* ctx, lbcu_spinor_s* p, lbcu_spinor_s* sv, lbcu_spinor_s* x, lbcu_spinor_s* r,
                const lbcu_spinor_s* w, double* dres) {
  const int nb = flat_blocks(ctx, r->elems);
  k_cg1_update<<<nb, kThreads, 0, ctx->stream>>>(p->base, sv->base, x->base, r->base, w->base, r->elems, ctx->dcg,
                                                 make_reduce(ctx, dres, nb));
  k_reduce_finish<1><<<1, kFinishThreads, 0, ctx->stream>>>(make_reduce(ctx, dres, nb));
  ctx->launches += 2;
  LBCU_CUDA(cudaGetLastError());
}

void cg1_scalar_start(lbcu_ctx_s* ctx, const double* gd) {
  k_cg1_start<<<1, 1, 0, ctx->stream>>>(ctx->dcg, gd);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void cg1_scalar_end(lbcu_ctx_s* ctx, const double* gd) {
  k_cg1_end<<<1, 1, 0, ctx->stream>>>(ctx->dcg, gd, ctx->dhist);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void cg_x_final(lbcu_ctx_s* ctx, lbcu_spinor_s* x, const lbcu_spinor_s* p) {
  k_cg_xfinal<<<flat_blocks(ctx, x->elems), kThreads, 0, ctx->stream>>>(x->base, p->base, x->elems, ctx->dcg);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void cg_scalar_init(lbcu_ctx_s* ctx, const double* b2, double tol, long long maxit) {
  k_cg_init<<<1, 1, 0, ctx->stream>>>(ctx->dcg, b2, tol, maxit);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void cg_scalar_alpha(lbcu_ctx_s* ctx, const double* pap) {
  k_cg_alpha<<<1, 1, 0, ctx->stream>>>(ctx->dcg, pap);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void cg_scalar_end(lbcu_ctx_s* ctx, const double* rr_new, unsigned long long handle, int use_graph) {
  k_cg_end<<<1, 1, 0, ctx->stream>>>(ctx->dcg, rr_new, ctx->dhist,
                                     static_cast<cudaGraphConditionalHandle>(handle), use_graph);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

template <class F>
static bool spinor_fast(int nv, F&& f) {
  switch (nv) {
    case 8: f(std::integral_constant<int, 8>{}); return true;
    case 12: f(std::integral_constant<int, 12>{}); return true;
    case 16: f(std::integral_constant<int, 16>{}); return true;
    case 24: f(std::integral_constant<int, 24>{}); return true;
    default: return false;
  }
}

template <class T>
static void launch_to_soa(lbcu_ctx_s* ctx, const T* src, T* d0, T* d1, int nv, int sign_entries,
                          int ng = 0) {
  const Geometry& geo = ctx->geo;
  if constexpr (std::is_same_v<T, double2>) {
    if (sign_entries == 0 && (ng == 0 || ng == nv) &&
        spinor_fast(nv, [&](auto Nc) {
          constexpr int TS = kSpTS<decltype(Nc)::value>;
          const int blocks = static_cast<int>((geo.volume + TS - 1) / TS);
          k_sp_to_soa<decltype(Nc)::value><<<blocks, 256, 0, ctx->stream>>>(src, d0, d1, geo.volume, ctx->dgeo);
        })) {
      ctx->launches++;
      LBCU_CUDA(cudaGetLastError());
      return;
    }
  }
  const int TS = tile_sites<T>(nv);
  const size_t smem = static_cast<size_t>(TS) * (nv + 1) * sizeof(T) + TS * sizeof(int);
  const int blocks = static_cast<int>((geo.volume + TS - 1) / TS);
  const int sign_t = sign_entries ? geo.global[0] - 1 : -1;
  const int t_off = geo.coords[0] * geo.local[0];
  k_aos_to_soa<T><<<blocks, 256, smem, ctx->stream>>>(src, d0, d1, nv, ng ? ng : nv, geo.volume, geo.stride, TS,
                                                      ctx->dgeo, sign_entries, sign_t, t_off);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

template <class T>
static void launch_to_aos(lbcu_ctx_s* ctx, const T* s0, const T* s1, T* dst, int nv, int ng = 0) {
  const Geometry& geo = ctx->geo;
  if constexpr (std::is_same_v<T, double2>) {
    if ((ng == 0 || ng == nv) && spinor_fast(nv, [&](auto Nc) {
          constexpr int TS = kSpTS<decltype(Nc)::value>;
          const int blocks = static_cast<int>((geo.volume + TS - 1) / TS);
          k_sp_to_aos<decltype(Nc)::value><<<blocks, 256, 0, ctx->stream>>>(s0, s1, dst, geo.volume, ctx->dgeo);
        })) {
      ctx->launches++;
      LBCU_CUDA(cudaGetLastError());
      return;
    }
  }
  const int TS = tile_sites<T>(nv);
  const size_t smem = static_cast<size_t>(TS) * (nv + 1) * sizeof(T) + TS * sizeof(int);
  const int blocks = static_cast<int>((geo.volume + TS - 1) / TS);
  k_soa_to_aos<T><<<blocks, 256, smem, ctx->stream>>>(s0, s1, dst, nv, ng ? ng : nv, geo.volume, geo.stride, TS,
                                                      ctx->dgeo);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
}

void spinor_upload(lbcu_ctx_s* ctx, lbcu_spinor_s* s, const double* host) {
  const int nv = 4 * s->dr;
  const size_t bytes = static_cast<size_t>(ctx->geo.volume) * nv * sizeof(double2);
  ensure_staging(ctx, bytes);
  LBCU_CUDA(cudaMemcpyAsync(ctx->staging, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  launch_to_soa<double2>(ctx, static_cast<const double2*>(ctx->staging), s->par[0], s->par[1], nv, 0);
  // value semantics: the caller may reuse its host buffer on return
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Host-field Dphi with copy/compute overlap: field k's host->device copy runs
// on pipe.h2d while field k-1 is transposed and multiplied on the compute
// stream and field k-2's result returns on pipe.d2h (two device slots, events
// order the reuse of each slot). Pinned host buffers give full PCIe duplex.
void dphi_host_batch(lbcu_ctx_s* ctx, const lbcu_gauge_s* g, double mass, int n,
                     const double* const* in, double* const* out) {
  auto& P = ctx->pipe;
  const int dr = g->dr, nv = 4 * dr;
  const size_t bytes = static_cast<size_t>(ctx->geo.volume) * nv * sizeof(double2);
  if (!P.h2d) {
    LBCU_CUDA(cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking));
    LBCU_CUDA(cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking));
    for (int s = 0; s < 2; ++s) {
      LBCU_CUDA(cudaEventCreateWithFlags(&P.ev_h2d[s], cudaEventDisableTiming));
      LBCU_CUDA(cudaEventCreateWithFlags(&P.ev_in_free[s], cudaEventDisableTiming));
      LBCU_CUDA(cudaEventCreateWithFlags(&P.ev_out[s], cudaEventDisableTiming));
      LBCU_CUDA(cudaEventCreateWithFlags(&P.ev_d2h[s], cudaEventDisableTiming));
    }
  }
  if (P.bytes < bytes) {
    for (int s = 0; s < 2; ++s) {
      if (P.stage_in[s]) LBCU_CUDA(cudaFree(P.stage_in[s]));
      if (P.stage_out[s]) LBCU_CUDA(cudaFree(P.stage_out[s]));
      LBCU_CUDA(cudaMalloc(&P.stage_in[s], bytes));
      LBCU_CUDA(cudaMalloc(&P.stage_out[s], bytes));
    }
    P.bytes = bytes;
  }
  lbcu_spinor_s* sin[2] = {scratch_spinor(ctx, dr, LBCU_FULL, 300), scratch_spinor(ctx, dr, LBCU_FULL, 301)};
  lbcu_spinor_s* sout[2] = {scratch_spinor(ctx, dr, LBCU_FULL, 302), scratch_spinor(ctx, dr, LBCU_FULL, 303)};
  // the slots start free
  for (int s = 0; s < 2; ++s) {
    LBCU_CUDA(cudaEventRecord(P.ev_in_free[s], ctx->stream));
    LBCU_CUDA(cudaEventRecord(P.ev_d2h[s], ctx->stream));
  }
  for (int k = 0; k < n; ++k) {
    const int s = k & 1;
    LBCU_CUDA(cudaStreamWaitEvent(P.h2d, P.ev_in_free[s], 0));
    LBCU_CUDA(cudaMemcpyAsync(P.stage_in[s], in[k], bytes, cudaMemcpyHostToDevice, P.h2d));
    LBCU_CUDA(cudaEventRecord(P.ev_h2d[s], P.h2d));
    LBCU_CUDA(cudaStreamWaitEvent(ctx->stream, P.ev_h2d[s], 0));
    launch_to_soa<double2>(ctx, static_cast<const double2*>(P.stage_in[s]), sin[s]->par[0], sin[s]->par[1], nv, 0);
    LBCU_CUDA(cudaEventRecord(P.ev_in_free[s], ctx->stream));
    HopCall hc;
    hc.in = sin[s];
    hc.out = sout[s];
    hc.x = sin[s];
    hc.g = g;
    hc.out_parity = 2;
    hc.a = 4.0 + mass;
    hc.b = -0.5;
    hop_apply(ctx, hc);
    LBCU_CUDA(cudaStreamWaitEvent(ctx->stream, P.ev_d2h[s], 0));
    launch_to_aos<double2>(ctx, sout[s]->par[0], sout[s]->par[1], static_cast<double2*>(P.stage_out[s]), nv);
    LBCU_CUDA(cudaEventRecord(P.ev_out[s], ctx->stream));
    LBCU_CUDA(cudaStreamWaitEvent(P.d2h, P.ev_out[s], 0));
    LBCU_CUDA(cudaMemcpyAsync(out[k], P.stage_out[s], bytes, cudaMemcpyDeviceToHost, P.d2h));
    LBCU_CUDA(cudaEventRecord(P.ev_d2h[s], P.d2h));
  }
  // the compute stream owns completion: later work and timing events see it
  for (int s = 0; s < 2; ++s) LBCU_CUDA(cudaStreamWaitEvent(ctx->stream, P.ev_d2h[s], 0));
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
}

void host_pipe_release(lbcu_ctx_s* ctx) {
  auto& P = ctx->pipe;
  for (int s = 0; s < 2; ++s) {
    if (P.stage_in[s]) cudaFree(P.stage_in[s]);
    if (P.stage_out[s]) cudaFree(P.stage_out[s]);
    if (P.ev_h2d[s]) cudaEventDestroy(P.ev_h2d[s]);
    if (P.ev_in_free[s]) cudaEventDestroy(P.ev_in_free[s]);
    if (P.ev_out[s]) cudaEventDestroy(P.ev_out[s]);
    if (P.ev_d2h[s]) cudaEventDestroy(P.ev_d2h[s]);
  }
  if (P.h2d) cudaStreamDestroy(P.h2d);
  if (P.d2h) cudaStreamDestroy(P.d2h);
  P = lbcu_ctx_s::HostPipe{};
}

void spinor_download(lbcu_ctx_s* ctx, const lbcu_spinor_s* s, double* host) {
  const int nv = 4 * s->dr;
  const size_t bytes = static_cast<size_t>(ctx->geo.volume) * nv * sizeof(double2);
  ensure_staging(ctx, bytes);
  launch_to_aos<double2>(ctx, s->par[0], s->par[1], static_cast<double2*>(ctx->staging), nv);
  LBCU_CUDA(cudaMemcpyAsync(host, ctx->staging, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ---- gauge storage: upload, compression to the compact formats, download --
namespace {

// compact format available for a representation (links.cuh)
// Compact formats to try, most compact first; the first whose every link
// rebuilds to 1e-12 is kept (gauge_adopt_dense). SU(3) fundamental: R10, then
// R12 (LBCU_SU3_STORAGE=r12 skips R10).
std::vector<int> compact_formats(const lbcu_gauge_s* g) {
  if (g->dr == 2 && !g->real) return {GF_SU2};  // SU(2) fundamental
  if (g->dr == 3 && g->real && g->n == 2) return {GF_SU2};  // SU(2) adjoint
  if (g->dr == 3 && !g->real && g->n == 3 && g->rep == LBCU_REP_FUNDAMENTAL) {
    const char* e = std::getenv("LBCU_SU3_STORAGE");
    if (e && std::string(e) == "r12") return {GF_R12};
    return {GF_R10, GF_R12};
  }
  if (g->dr == 6 && !g->real && g->n == 4 && g->rep == LBCU_REP_ANTISYMMETRIC) return {GF_AS4R};
  return {};
}

int fmt_entries(int fmt, int dr) {
  return fmt == GF_SU2 ? 2 : fmt == GF_R12 ? 6 : fmt == GF_R10 ? 5 : fmt == GF_AS4 ? 16 : fmt == GF_AS4R ? 18
                                                                                            : dr * dr;
}

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* p, double v) {
  atomicMax(p, __double_as_longlong(v));  // non-negative doubles order like their bit patterns
}

__device__ __forceinline__ double cabs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// full dense link -> compact storage, with the reconstruction error
template <int D, bool REAL, int FMT>
__global__ void k_compress(const LinkT<REAL>* __restrict__ full, double2* __restrict__ compact,
                           long long stride, int vh, unsigned long long* err) {
  constexpr int E = LinkFmt<D, REAL, FMT>::entries;
  const long long n = 8LL * vh;  // (parity, mu) blocks x sites
  double worst = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long blk = t / vh, cb = t % vh;
    const LinkT<REAL>* f = site_ptr<D * D>(full + blk * D * D * stride, cb);
    double2* cp = site_ptr<E>(compact + blk * E * stride, cb);
    LinkT<REAL> u[D * D];
#pragma unroll
    for (int e = 0; e < D * D; ++e) u[e] = f[(long long)e * kTile];
    double2 st[E];
    if constexpr (FMT == GF_SU2 && !REAL) {
      st[0] = u[0];
      st[1] = u[1];
    } else if constexpr (FMT == GF_SU2 && REAL) {
      // SO(3) -> unit quaternion (w, v) with R = (w^2-|v|^2) I + 2 v v^T + 2 w [v]x,
      // Shepperd's branch choice; then a0 = w, a = -v (links.cuh convention)
      const double tr = u[0] + u[4] + u[8];
      double w, vx, vy, vz;
      if (tr > 0) {
        w = 0.5 * sqrt(1.0 + tr);
        vx = (u[7] - u[5]) / (4 * w);
        vy = (u[2] - u[6]) / (4 * w);
        vz = (u[3] - u[1]) / (4 * w);
      } else if (u[0] >= u[4] && u[0] >= u[8]) {
        vx = 0.5 * sqrt(fmax(0.0, 1.0 + u[0] - u[4] - u[8]));
        w = (u[7] - u[5]) / (4 * vx);
        vy = (u[1] + u[3]) / (4 * vx);
        vz = (u[2] + u[6]) / (4 * vx);
      } else if (u[4] >= u[8]) {
        vy = 0.5 * sqrt(fmax(0.0, 1.0 + u[4] - u[0] - u[8]));
        w = (u[2] - u[6]) / (4 * vy);
        vx = (u[1] + u[3]) / (4 * vy);
        vz = (u[5] + u[7]) / (4 * vy);
      } else {
        vz = 0.5 * sqrt(fmax(0.0, 1.0 + u[8] - u[0] - u[4]));
        w = (u[3] - u[1]) / (4 * vz);
        vx = (u[2] + u[6]) / (4 * vz);
        vy = (u[5] + u[7]) / (4 * vz);
      }
      st[0] = make_double2(w, -vz);   // al = a0 + i a3
      st[1] = make_double2(-vy, -vx); // be = a2 + i a1
    } else if constexpr (FMT == GF_AS4R) {
      as4r_from_dense(u, st);  // imaginary residue caught by the rebuild check below
    } else if constexpr (FMT == GF_R10) {
      st[0] = u[0];
      st[1] = u[1];
      st[2] = u[2];
      st[3] = u[4];
      st[4] = u[5];
    } else {
#pragma unroll
      for (int e = 0; e < 6; ++e) st[e] = u[e];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) cp[(long long)e * kTile] = st[e];
    // validate: rebuild from the stored entries and compare with the dense link
    LinkT<REAL> r[D * D];
    build_link<D, REAL, FMT>(r, st);
#pragma unroll
    for (int e = 0; e < D * D; ++e) {
      double d;
      if constexpr (REAL) d = fabs(r[e] - u[e]);
      else d = sqrt(cabs2(make_double2(r[e].x - u[e].x, r[e].y - u[e].y)));
      worst = fmax(worst, d);
    }
  }
  if (worst > 0.0 || !isfinite(worst)) atomic_max_nonneg(err, isfinite(worst) ? worst : 1e300);
}

// SU(4) fundamental elements -> GF_AS4R (minors, then the real basis);
// err = max |Im R'| (non-zero only for non-SU(4) input)
__global__ void k_as4r_from_fund(const double2* __restrict__ fund, double2* __restrict__ compact,
                                 long long stride, int vh, unsigned long long* err) {
  const long long n = 8LL * vh;
  double worst = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long blk = t / vh, cb = t % vh;
    double2 s[16], u[36], st[18];
    const double2* f = site_ptr<16>(fund + blk * 16 * stride, cb);
#pragma unroll
    for (int e = 0; e < 16; ++e) s[e] = f[(long long)e * kTile];
    build_link<6, false, GF_AS4>(u, s);
    worst = fmax(worst, as4r_from_dense(u, st));
    double2* cp = site_ptr<18>(compact + blk * 18 * stride, cb);
#pragma unroll
    for (int e = 0; e < 18; ++e) cp[(long long)e * kTile] = st[e];
  }
  if (worst > 0.0 || !isfinite(worst)) atomic_max_nonneg(err, isfinite(worst) ? worst : 1e300);
}

// compact -> dense (downloads)
template <int D, bool REAL, int FMT>
__global__ void k_expand(const double2* __restrict__ compact, LinkT<REAL>* __restrict__ full,
                         long long stride, int vh) {
  constexpr int E = LinkFmt<D, REAL, FMT>::entries;
  const long long n = 8LL * vh;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const long long blk = t / vh, cb = t % vh;
    LinkT<REAL> u[D * D];
    load_link<D, REAL, FMT>(u, site_ptr<E>(compact + blk * E * stride, cb), kTile);
    LinkT<REAL>* f = site_ptr<D * D>(full + blk * D * D * stride, cb);
#pragma unroll
    for (int e = 0; e < D * D; ++e) f[(long long)e * kTile] = u[e];
  }
}

// antiperiodic time: negate U_0 on the last global time slice (dense storage)
template <class T>
__global__ void k_bake_sign(T* full, long long stride, int entries, DevGeo g, int t_off, int tlast) {
  const long long n = 2LL * g.vh;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int par = static_cast<int>(t / g.vh), cb = static_cast<int>(t % g.vh);
    int c[4], s;
    cb_coords(g, cb, par, c, s);
    if (c[0] + t_off != tlast) continue;
    T* base = full + (long long)par * 4 * entries * stride;  // mu = 0 block
    for (int e = 0; e < entries; ++e) {
      const long long o = eidx(entries, e, cb);
      base[o] = neg(base[o]);
    }
  }
}

template <class F>
void dispatch_compact(const lbcu_gauge_s* g, int fmt, F&& f) {
  using std::integral_constant;
  if (fmt == GF_SU2 && !g->real)
    return f(integral_constant<int, 2>{}, std::false_type{}, integral_constant<int, GF_SU2>{});
  if (fmt == GF_SU2 && g->real)
    return f(integral_constant<int, 3>{}, std::true_type{}, integral_constant<int, GF_SU2>{});
  if (fmt == GF_R12)
    return f(integral_constant<int, 3>{}, std::false_type{}, integral_constant<int, GF_R12>{});
  if (fmt == GF_R10)
    return f(integral_constant<int, 3>{}, std::false_type{}, integral_constant<int, GF_R10>{});
  if (fmt == GF_AS4R)
    return f(integral_constant<int, 6>{}, std::false_type{}, integral_constant<int, GF_AS4R>{});
  throw Error(LBCU_CONTRACT_VIOLATION, "no compact gauge format");
}

// formats that can only be expanded (they are uploaded in compact form)
template <class F>
void dispatch_expand(const lbcu_gauge_s* g, int fmt, F&& f) {
  using std::integral_constant;
  if (fmt == GF_AS4)
    return f(integral_constant<int, 6>{}, std::false_type{}, integral_constant<int, GF_AS4>{});
  dispatch_compact(g, fmt, f);
}

int grid_for(long long n) { return static_cast<int>(std::min<long long>((n + 255) / 256, 148 * 16)); }

bool compaction_enabled(const lbcu_gauge_s* g) {
  const char* e = std::getenv("LBCU_GAUGE_COMPACT");
  return g->compact_ok && !(e && e[0] == '0');
}

}  // namespace

void gauge_upload(lbcu_ctx_s* ctx, lbcu_gauge_s* g, const double* host) {
  const Geometry& geo = ctx->geo;
  const int dd = g->dr * g->dr;
  const int nv = 4 * dd;
  const size_t esz = g->real ? sizeof(double) : sizeof(double2);
  const size_t bytes = static_cast<size_t>(geo.volume) * nv * esz;
  const size_t full_bytes = 2 * static_cast<size_t>(nv) * geo.stride * esz;
  ensure_staging(ctx, bytes);
  void* full = nullptr;
  if (g->fmt == GF_FULL && g->base) {
    full = g->base;
  } else {
    LBCU_CUDA(cudaMalloc(&full, full_bytes));
    LBCU_CUDA(cudaMemsetAsync(full, 0, full_bytes, ctx->stream));
  }
  LBCU_CUDA(cudaMemcpyAsync(ctx->staging, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  const size_t pstride = static_cast<size_t>(nv) * geo.stride;
  if (g->real) {
    double* b = static_cast<double*>(full);
    launch_to_soa<double>(ctx, static_cast<const double*>(ctx->staging), b, b + pstride, nv, 0, dd);
  } else {
    double2* b = static_cast<double2*>(full);
    launch_to_soa<double2>(ctx, static_cast<const double2*>(ctx->staging), b, b + pstride, nv, 0, dd);
  }
  gauge_adopt_dense(ctx, g, full);
}

// Take ownership of dense device links [2][4][dr*dr][stride] (no BC sign):
// compress them when they reconstruct exactly, else bake the BC sign in.
void gauge_adopt_dense(lbcu_ctx_s* ctx, lbcu_gauge_s* g, void* full) {
  const Geometry& geo = ctx->geo;
  const int dd = g->dr * g->dr;
  auto adopt = [&](void* base, int fmt) {
    if (g->base && g->base != base) LBCU_CUDA(cudaFree(g->base));
    g->base = base;
    g->fmt = fmt;
  };
  double best_err = -1.0;
  for (const int cf : compaction_enabled(g) ? compact_formats(g) : std::vector<int>{}) {
    const size_t cbytes = 2 * 4 * static_cast<size_t>(fmt_entries(cf, g->dr)) * geo.stride * sizeof(double2);
    void* compact = nullptr;
    LBCU_CUDA(cudaMalloc(&compact, cbytes));
    LBCU_CUDA(cudaMemsetAsync(compact, 0, cbytes, ctx->stream));
    unsigned long long* derr = reinterpret_cast<unsigned long long*>(ctx->dscal + 60);
    LBCU_CUDA(cudaMemsetAsync(derr, 0, sizeof(unsigned long long), ctx->stream));
    dispatch_compact(g, cf, [&](auto Dc, auto Rc, auto Fc) {
      constexpr int D = decltype(Dc)::value;
      constexpr bool REAL = decltype(Rc)::value;
      k_compress<D, REAL, decltype(Fc)::value><<<grid_for(8LL * geo.vh), 256, 0, ctx->stream>>>(
          static_cast<const LinkT<REAL>*>(full), static_cast<double2*>(compact), geo.stride,
          static_cast<int>(geo.vh), derr);
    });
    ctx->launches++;
    LBCU_CUDA(cudaGetLastError());
    unsigned long long bits = 0;
    LBCU_CUDA(cudaMemcpyAsync(&bits, derr, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream));
    LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
    double err;
    std::memcpy(&err, &bits, sizeof(err));
    if (best_err < 0.0 || err < best_err) best_err = err;
    if (err <= 1e-12) {
      g->compact_err = err;
      if (full != g->base) LBCU_CUDA(cudaFree(full));
      adopt(compact, cf);  // frees the previous storage
      return;
    }
    LBCU_CUDA(cudaFree(compact));
  }
  g->compact_err = best_err;
  if (g->bc == LBCU_BC_ANTIPERIODIC_T) {
    const int t_off = geo.coords[0] * geo.local[0];
    if (g->real)
      k_bake_sign<double><<<grid_for(2 * geo.vh), 256, 0, ctx->stream>>>(
          static_cast<double*>(full), geo.stride, dd, ctx->dgeo, t_off, geo.global[0] - 1);
    else
      k_bake_sign<double2><<<grid_for(2 * geo.vh), 256, 0, ctx->stream>>>(
          static_cast<double2*>(full), geo.stride, dd, ctx->dgeo, t_off, geo.global[0] - 1);
    ctx->launches++;
    LBCU_CUDA(cudaGetLastError());
  }
  adopt(full, GF_FULL);
  // the staging buffer is reused by the next transfer: finish this one first
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Links given as fundamental SU(N) elements; the representation is formed in
// the kernels (GF_AS4: two-index antisymmetric of SU(4)).
void gauge_upload_fundamental(lbcu_ctx_s* ctx, lbcu_gauge_s* g, const double* host) {
  if (!(g->rep == LBCU_REP_ANTISYMMETRIC && g->n == 4))
    throw Error(LBCU_CONFIG_ERROR,
                "fundamental-link storage is implemented for the SU(4) antisymmetric representation");
  const Geometry& geo = ctx->geo;
  const int nv = 4 * 16;
  const size_t bytes = static_cast<size_t>(geo.volume) * nv * sizeof(double2);
  ensure_staging(ctx, bytes);
  const size_t cbytes = 2 * static_cast<size_t>(nv) * geo.stride * sizeof(double2);
  void* base = nullptr;
  LBCU_CUDA(cudaMalloc(&base, cbytes));
  LBCU_CUDA(cudaMemsetAsync(base, 0, cbytes, ctx->stream));
  LBCU_CUDA(cudaMemcpyAsync(ctx->staging, host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  double2* b = static_cast<double2*>(base);
  launch_to_soa<double2>(ctx, static_cast<const double2*>(ctx->staging), b,
                         b + static_cast<size_t>(nv) * geo.stride, nv, 0, 16);
  gauge_adopt_fundamental(ctx, g, base);
}

// Take ownership of tiled SU(4) fundamental links [2][4] x 16 entries:
// store them as real SO(6) matrices (GF_AS4R) when every link is SU(4) to
// 1e-12, else keep the fundamental elements (GF_AS4, exact for any input).
// LBCU_AS4_STORAGE=fund keeps GF_AS4.
void gauge_adopt_fundamental(lbcu_ctx_s* ctx, lbcu_gauge_s* g, void* fund) {
  const Geometry& geo = ctx->geo;
  const char* env = std::getenv("LBCU_AS4_STORAGE");
  const bool want_real = compaction_enabled(g) && !(env && std::string(env) == "fund");
  if (g->base && g->base != fund) LBCU_CUDA(cudaFree(g->base));
  g->base = fund;
  g->fmt = GF_AS4;
  g->compact_err = 0.0;
  if (want_real) {
    const size_t cbytes = 2 * 4 * 18 * static_cast<size_t>(geo.stride) * sizeof(double2);
    void* compact = nullptr;
    LBCU_CUDA(cudaMalloc(&compact, cbytes));
    LBCU_CUDA(cudaMemsetAsync(compact, 0, cbytes, ctx->stream));
    unsigned long long* derr = reinterpret_cast<unsigned long long*>(ctx->dscal + 60);
    LBCU_CUDA(cudaMemsetAsync(derr, 0, sizeof(unsigned long long), ctx->stream));
    k_as4r_from_fund<<<grid_for(8LL * geo.vh), 256, 0, ctx->stream>>>(
        static_cast<const double2*>(fund), static_cast<double2*>(compact), geo.stride,
        static_cast<int>(geo.vh), derr);
    ctx->launches++;
    LBCU_CUDA(cudaGetLastError());
    unsigned long long bits = 0;
    LBCU_CUDA(cudaMemcpyAsync(&bits, derr, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream));
    LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
    double err;
    std::memcpy(&err, &bits, sizeof(err));
    if (err <= 1e-12) {
      LBCU_CUDA(cudaFree(fund));
      g->base = compact;
      g->fmt = GF_AS4R;
      g->compact_err = err;
    } else {
      LBCU_CUDA(cudaFree(compact));
    }
  }
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
}

void gauge_download(lbcu_ctx_s* ctx, const lbcu_gauge_s* g, double* host) {
  const Geometry& geo = ctx->geo;
  const int nv = 4 * g->dr * g->dr;
  const size_t esz = g->real ? sizeof(double) : sizeof(double2);
  const size_t bytes = static_cast<size_t>(geo.volume) * nv * esz;
  ensure_staging(ctx, bytes);
  const size_t pstride = static_cast<size_t>(nv) * geo.stride;
  const void* full = g->base;
  void* tmp = nullptr;
  if (g->fmt != GF_FULL) {
    LBCU_CUDA(cudaMalloc(&tmp, 2 * pstride * esz));
    dispatch_expand(g, g->fmt, [&](auto Dc, auto Rc, auto Fc) {
      constexpr int D = decltype(Dc)::value;
      constexpr bool REAL = decltype(Rc)::value;
      k_expand<D, REAL, decltype(Fc)::value><<<grid_for(8LL * geo.vh), 256, 0, ctx->stream>>>(
          static_cast<const double2*>(g->base), static_cast<LinkT<REAL>*>(tmp), geo.stride,
          static_cast<int>(geo.vh));
    });
    ctx->launches++;
    full = tmp;
  }
  if (g->real) {
    const double* b = static_cast<const double*>(full);
    launch_to_aos<double>(ctx, b, b + pstride, static_cast<double*>(ctx->staging), nv, nv / 4);
  } else {
    const double2* b = static_cast<const double2*>(full);
    launch_to_aos<double2>(ctx, b, b + pstride, static_cast<double2*>(ctx->staging), nv, nv / 4);
  }
  LBCU_CUDA(cudaMemcpyAsync(host, ctx->staging, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
  if (tmp) LBCU_CUDA(cudaFree(tmp));
  if (g->fmt == GF_FULL && g->bc == LBCU_BC_ANTIPERIODIC_T) {  // report the links as uploaded
    const int per = nv * (g->real ? 1 : 2);
    const int64_t slab = geo.volume / geo.local[0];
    if (geo.coords[0] == geo.grid[0] - 1)
      for (int64_t s = (geo.local[0] - 1) * slab; s < geo.volume; ++s)
        for (int k = 0; k < g->dr * g->dr * (g->real ? 1 : 2); ++k) host[s * per + k] = -host[s * per + k];
  }
}

}  // namespace lbcu
