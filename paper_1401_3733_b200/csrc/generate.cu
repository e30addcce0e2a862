// On-device seeded field generation.
//
// The same keyed generators as csrc/host_fields.cpp / the reference
// (rng.hpp:16-72, fields.cpp:22-40 and 86-107, group.cpp:42-114), evaluated
// per site on the GPU and written straight into the device layout: no host
// generation and no PCIe upload of the links. Integer hashing is exact; the
// floating-point steps follow the host operation order, and this translation
// unit is compiled with --fmad=false so no FMA contraction reorders the
// rounding. Values then agree with the host generator to a few ulp (CUDA's
// log/sin/cos/atan2/hypot are not always correctly rounded like glibc's),
// far inside the 1e-12 Dphi tolerance; tests/test_gpu_generate.py checks it.
#include "links.cuh"
#include "objects.hpp"

namespace lbcu {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <int N>
__device__ __forceinline__ uint64_t key_hash(const uint64_t (&w)[N]) {
  uint64_t h = 0x243f6a8885a308d3ull;
#pragma unroll
  for (int i = 0; i < N; ++i) h = mix64(h ^ (w[i] + 0x9e3779b97f4a7c15ull));
  return h;
}

__device__ __forceinline__ double u01(uint64_t bits) {
  return (static_cast<double>(bits >> 11) + 1.0) * 0x1.0p-53;
}

__device__ __forceinline__ void gauss_pair(uint64_t key, double& g0, double& g1) {
  const double u1 = u01(mix64(key ^ 0x5555555555555555ull));
  const double u2 = u01(mix64(key ^ 0xaaaaaaaaaaaaaaaaull));
  const double r = sqrt(-2.0 * log(u1));
  const double th = 2.0 * 3.141592653589793 * u2;
  g0 = r * cos(th);
  g1 = r * sin(th);
}

struct Stream {  // RngStream, rng.hpp:45-70
  uint64_t key, counter = 0;
  double spare = 0.0;
  bool have = false;
  __device__ explicit Stream(uint64_t k) : key(k) {}
  __device__ double gauss() {
    if (have) {
      have = false;
      return spare;
    }
    double a, b;
    const uint64_t w[2] = {key, ++counter};
    gauss_pair(key_hash(w), a, b);
    spare = b;
    have = true;
    return a;
  }
  __device__ double2 gauss_cplx() {
    double a, b;
    const uint64_t w[2] = {key, ++counter};
    gauss_pair(key_hash(w), a, b);
    return make_double2(a, b);
  }
};

// complex helpers in the host operation order (std::complex, no FMA)
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cs(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 ca(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 cj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double cabs(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {  // textbook complex division
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

// random_group_element, group.cpp:82-114 (first attempt; degenerate draws
// are astronomically rare and fall back to the identity flagged by *bad)
template <int N>
__device__ void random_su_n(double2 (&u)[N * N], Stream& rng, int* bad) {
  for (int attempt = 0; attempt < 16; ++attempt) {
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) u[i * N + j] = rng.gauss_cplx();
    bool degenerate = false;
    for (int j = 0; j < N && !degenerate; ++j) {
      for (int k = 0; k < j; ++k) {
        double2 proj = make_double2(0.0, 0.0);
        for (int i = 0; i < N; ++i) proj = ca(proj, cm(cj(u[i * N + k]), u[i * N + j]));
        for (int i = 0; i < N; ++i) u[i * N + j] = cs(u[i * N + j], cm(proj, u[i * N + k]));
      }
      double nrm = 0.0;
      for (int i = 0; i < N; ++i) nrm += u[i * N + j].x * u[i * N + j].x + u[i * N + j].y * u[i * N + j].y;
      nrm = sqrt(nrm);
      if (nrm < 1e-8) {
        degenerate = true;
        break;
      }
      for (int i = 0; i < N; ++i) u[i * N + j] = make_double2(u[i * N + j].x / nrm, u[i * N + j].y / nrm);
    }
    if (degenerate) continue;
    // det by LU with partial pivoting (matrix.hpp:80-106)
    double2 a[N * N];
    for (int e = 0; e < N * N; ++e) a[e] = u[e];
    double2 d = make_double2(1.0, 0.0);
    bool zero = false;
    for (int k = 0; k < N && !zero; ++k) {
      int piv = k;
      double best = cabs(a[k * N + k]);
      for (int i = k + 1; i < N; ++i) {
        const double m = cabs(a[i * N + k]);
        if (m > best) {
          best = m;
          piv = i;
        }
      }
      if (best == 0.0) {
        zero = true;
        break;
      }
      if (piv != k) {
        for (int j = 0; j < N; ++j) {
          const double2 t = a[k * N + j];
          a[k * N + j] = a[piv * N + j];
          a[piv * N + j] = t;
        }
        d = make_double2(-d.x, -d.y);
      }
      d = cm(d, a[k * N + k]);
      for (int i = k + 1; i < N; ++i) {
        const double2 f = cdiv(a[i * N + k], a[k * N + k]);
        for (int j = k; j < N; ++j) a[i * N + j] = cs(a[i * N + j], cm(f, a[k * N + j]));
      }
    }
    const double phi = zero ? 0.0 : atan2(d.y, d.x);
    const double2 s = make_double2(cos(-phi / N), sin(-phi / N));
    for (int e = 0; e < N * N; ++e) u[e] = cm(u[e], s);
    return;
  }
  *bad = 1;
}

// su(N) generators (group.cpp:42-71): T_a entries for index a
template <int N>
__device__ double2 gen(int a, int i, int j) {
  constexpr int npair = N * (N - 1) / 2;
  if (a < 2 * npair) {
    const int sym = a < npair;
    int p = sym ? a : a - npair, r = 0;
    int ii = 0, jj = 0;
    for (int x = 0; x < N; ++x)
      for (int y = x + 1; y < N; ++y) {
        if (r == p) {
          ii = x;
          jj = y;
        }
        ++r;
      }
    if (sym) return (i == ii && j == jj) || (i == jj && j == ii) ? make_double2(0.5, 0.0) : make_double2(0.0, 0.0);
    if (i == ii && j == jj) return make_double2(0.0, -0.5);
    if (i == jj && j == ii) return make_double2(0.0, 0.5);
    return make_double2(0.0, 0.0);
  }
  const int k = a - 2 * npair + 1;
  if (i != j) return make_double2(0.0, 0.0);
  const double norm = 1.0 / sqrt(2.0 * k * (k + 1));
  if (i < k) return make_double2(norm, 0.0);
  if (i == k) return make_double2(-static_cast<double>(k) * norm, 0.0);
  return make_double2(0.0, 0.0);
}

// U = exp(i eps sum_a xi_a T_a) by scaling and squaring, degree-16 Taylor
template <int N>
__device__ void near_unit(double2 (&u)[N * N], Stream& rng, double eps) {
  double2 a[N * N];
  for (int e = 0; e < N * N; ++e) a[e] = make_double2(0.0, 0.0);
  for (int g = 0; g < N * N - 1; ++g) {
    const double xi = rng.gauss();
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) a[i * N + j] = ca(a[i * N + j], cm(make_double2(0.0, eps * xi), gen<N>(g, i, j)));
  }
  int sq = 0;
  double mx = 0.0;
  for (int e = 0; e < N * N; ++e) mx = fmax(mx, cabs(a[e]));
  double nrm = mx * N;
  while (nrm > 0.5) {
    nrm *= 0.5;
    ++sq;
  }
  const double sc = ldexp(1.0, -sq);
  for (int e = 0; e < N * N; ++e) a[e] = make_double2(a[e].x * sc, a[e].y * sc);
  double2 term[N * N], t2[N * N];
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) u[i * N + j] = term[i * N + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
  for (int k = 1; k <= 16; ++k) {
    for (int i = 0; i < N; ++i)  // term = term * a (matrix.hpp:30-38 loop order)
      for (int j = 0; j < N; ++j) t2[i * N + j] = make_double2(0.0, 0.0);
    for (int i = 0; i < N; ++i)
      for (int kk = 0; kk < N; ++kk) {
        const double2 v = term[i * N + kk];
        for (int j = 0; j < N; ++j) t2[i * N + j] = ca(t2[i * N + j], cm(v, a[kk * N + j]));
      }
    const double inv = 1.0 / k;
    for (int e = 0; e < N * N; ++e) {
      term[e] = make_double2(t2[e].x * inv, t2[e].y * inv);
      u[e] = ca(u[e], term[e]);
    }
  }
  for (int q = 0; q < sq; ++q) {
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) t2[i * N + j] = make_double2(0.0, 0.0);
    for (int i = 0; i < N; ++i)
      for (int kk = 0; kk < N; ++kk) {
        const double2 v = u[i * N + kk];
        for (int j = 0; j < N; ++j) t2[i * N + j] = ca(t2[i * N + j], cm(v, u[kk * N + j]));
      }
    for (int e = 0; e < N * N; ++e) u[e] = t2[e];
  }
}

// adjoint of SU(2) (group.cpp:126-143) via the closed form of links.cuh
__device__ void adjoint_su2(double (&r)[9], const double2 (&u)[4]) {
  const double a0 = u[0].x, a3 = u[0].y, a2 = u[1].x, a1 = u[1].y;
  const double d = a0 * a0 - (a1 * a1 + a2 * a2 + a3 * a3);
  r[0] = d + 2 * a1 * a1;
  r[1] = 2 * a1 * a2 + 2 * a0 * a3;
  r[2] = 2 * a1 * a3 - 2 * a0 * a2;
  r[3] = 2 * a2 * a1 - 2 * a0 * a3;
  r[4] = d + 2 * a2 * a2;
  r[5] = 2 * a2 * a3 + 2 * a0 * a1;
  r[6] = 2 * a3 * a1 + 2 * a0 * a2;
  r[7] = 2 * a3 * a2 - 2 * a0 * a1;
  r[8] = d + 2 * a3 * a3;
}

struct GenArgs {
  DevGeo g;
  int coords[4], local[4];
  uint64_t seed;
  double eps;
  int links;    // LBCU_LINKS_*
  int out_dr;   // entries written per link: N*N (fundamental) or 9 (adjoint)
  int adjoint;  // write the SU(2) adjoint as real links
  void* out;    // [2][4] blocks of out_dr^2 x stride (tiled) double2 or double
  int* bad;
};

template <int N>
__global__ void k_gauge_generate(const GenArgs A) {
  const long long n = 8LL * A.g.vh;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int par = static_cast<int>(t / (4LL * A.g.vh));
    const int rem = static_cast<int>(t % (4LL * A.g.vh));
    const int mu = rem / A.g.vh, cb = rem % A.g.vh;
    int c[4], s;
    cb_coords(A.g, cb, par, c, s);
    const uint64_t w[7] = {A.seed, 0x47u,
                           static_cast<uint64_t>(A.coords[0] * A.local[0] + c[0]),
                           static_cast<uint64_t>(A.coords[1] * A.local[1] + c[1]),
                           static_cast<uint64_t>(A.coords[2] * A.local[2] + c[2]),
                           static_cast<uint64_t>(A.coords[3] * A.local[3] + c[3]),
                           static_cast<uint64_t>(mu)};
    double2 u[N * N];
    if (A.links == LBCU_LINKS_UNIT) {
      for (int i = 0; i < N; ++i)
        for (int j = 0; j < N; ++j) u[i * N + j] = make_double2(i == j ? 1.0 : 0.0, 0.0);
    } else {
      Stream rng(key_hash(w));
      if (A.links == LBCU_LINKS_HAAR) random_su_n<N>(u, rng, A.bad);
      else near_unit<N>(u, rng, A.eps);
    }
    const long long st = A.g.stride;
    if (A.adjoint) {
      double r[9];
      if constexpr (N == 2) adjoint_su2(r, u);
      double* o = site_ptr<9>(static_cast<double*>(A.out) + ((long long)(par * 4 + mu) * 9) * st, cb);
      for (int e = 0; e < 9; ++e) o[(long long)e * kTile] = r[e];
    } else {
      double2* o = site_ptr<N * N>(static_cast<double2*>(A.out) + ((long long)(par * 4 + mu) * N * N) * st, cb);
      for (int e = 0; e < N * N; ++e) o[(long long)e * kTile] = u[e];
    }
  }
}

struct SpinArgs {
  DevGeo g;
  int coords[4], local[4];
  uint64_t seed, field;
  int dr;
  double2* par[2];
};

__global__ void k_spinor_generate(const SpinArgs A) {
  const int nv = 4 * A.dr;
  const long long n = 2LL * A.g.vh * nv;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int p = static_cast<int>(t / ((long long)A.g.vh * nv));
    const long long rem = t % ((long long)A.g.vh * nv);
    const int k = static_cast<int>(rem / A.g.vh), cb = static_cast<int>(rem % A.g.vh);
    if (!A.par[p]) continue;
    int c[4], s;
    cb_coords(A.g, cb, p, c, s);
    const int spin = k / A.dr, col = k % A.dr;
    const uint64_t w[9] = {A.seed, 0x53u, A.field,
                           static_cast<uint64_t>(A.coords[0] * A.local[0] + c[0]),
                           static_cast<uint64_t>(A.coords[1] * A.local[1] + c[1]),
                           static_cast<uint64_t>(A.coords[2] * A.local[2] + c[2]),
                           static_cast<uint64_t>(A.coords[3] * A.local[3] + c[3]),
                           static_cast<uint64_t>(spin), static_cast<uint64_t>(col)};
    double a, b;
    gauss_pair(key_hash(w), a, b);
    A.par[p][eidx(nv, k, cb)] = make_double2(a, b);
  }
}

int gen_grid(long long n) { return static_cast<int>(std::min<long long>((n + 127) / 128, 148 * 32)); }

}  // namespace

void spinor_generate(lbcu_ctx_s* ctx, lbcu_spinor_s* sp, uint64_t seed, uint64_t field) {
  SpinArgs A{};
  A.g = ctx->dgeo;
  for (int d = 0; d < 4; ++d) {
    A.coords[d] = ctx->geo.coords[d];
    A.local[d] = ctx->geo.local[d];
  }
  A.seed = seed;
  A.field = field;
  A.dr = sp->dr;
  A.par[0] = sp->par[0];
  A.par[1] = sp->par[1];
  k_spinor_generate<<<gen_grid(2LL * ctx->geo.vh * 4 * sp->dr), 128, 0, ctx->stream>>>(A);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
}

// Generate the fundamental SU(N) links (or the SU(2) adjoint) into a dense
// [2][4][entries][stride] buffer; returns it (caller owns).
void* gauge_generate_dense(lbcu_ctx_s* ctx, const lbcu_gauge_s* g, int links, uint64_t seed, double eps,
                           bool fundamental) {
  const int N = g->n;
  const bool adjoint = !fundamental && g->rep == LBCU_REP_ADJOINT;
  if (!fundamental && !(g->rep == LBCU_REP_FUNDAMENTAL || (adjoint && N == 2)))
    throw Error(LBCU_CONFIG_ERROR, "device generation supports fundamental links and the SU(2) adjoint");
  if (N < 2 || N > 4) throw Error(LBCU_CONFIG_ERROR, "device generation supports SU(2), SU(3), SU(4)");
  if (links == LBCU_LINKS_NEAR_UNIT && (adjoint || g->rep != LBCU_REP_FUNDAMENTAL && !fundamental))
    throw Error(LBCU_CONFIG_ERROR, "near-unit links are generated for the fundamental rep only");
  const int entries = adjoint ? 9 : N * N;
  const size_t esz = adjoint ? sizeof(double) : sizeof(double2);
  const size_t bytes = 2 * 4 * static_cast<size_t>(entries) * ctx->geo.stride * esz;
  void* out = nullptr;
  LBCU_CUDA(cudaMalloc(&out, bytes));
  LBCU_CUDA(cudaMemsetAsync(out, 0, bytes, ctx->stream));
  int* bad = reinterpret_cast<int*>(ctx->dscal + 62);
  LBCU_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
  GenArgs A{};
  A.g = ctx->dgeo;
  for (int d = 0; d < 4; ++d) {
    A.coords[d] = ctx->geo.coords[d];
    A.local[d] = ctx->geo.local[d];
  }
  A.seed = seed;
  A.eps = eps;
  A.links = links;
  A.adjoint = adjoint ? 1 : 0;
  A.out = out;
  A.bad = bad;
  const int grid = gen_grid(8LL * ctx->geo.vh);
  if (N == 2) k_gauge_generate<2><<<grid, 128, 0, ctx->stream>>>(A);
  else if (N == 3) k_gauge_generate<3><<<grid, 128, 0, ctx->stream>>>(A);
  else k_gauge_generate<4><<<grid, 128, 0, ctx->stream>>>(A);
  ctx->launches++;
  LBCU_CUDA(cudaGetLastError());
  int hbad = 0;
  LBCU_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  LBCU_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hbad) {
    cudaFree(out);
    throw Error(LBCU_CONFIG_ERROR, "random group element generation degenerated repeatedly");
  }
  return out;
}

}  // namespace lbcu
