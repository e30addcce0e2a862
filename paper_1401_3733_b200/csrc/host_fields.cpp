// Host-side seeded inputs, bit-compatible with the reference generators.
//
// Restates (does not include) the reference algorithms:
//   counter RNG          proj/include/latbench/rng.hpp:16-72
//   su(N) generators     proj/src/group.cpp:42-71
//   Haar-ish SU(N)       proj/src/group.cpp:82-114 (Gaussian, MGS, det phase)
//   represent()          proj/src/group.cpp:119-196 (adjoint / AS / S maps)
//   field keying         proj/src/fields.cpp:22-40 (spinor), :86-107 (gauge)
// plus the near-unit generator of BASELINE config 3 (U = exp(i eps H),
// SURVEY.md §8d). Work is split over std::threads by site; every value is a
// pure function of (seed, global coordinate), so any split is identical.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <thread>
#include <vector>

#include "lbcu_internal.hpp"

namespace lbcu {

using Cplx = std::complex<double>;

namespace {

uint64_t mix64(uint64_t x) {  // rng.hpp:16-22
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <size_t N>
uint64_t key_hash(const uint64_t (&w)[N]) {  // rng.hpp:25-29
  uint64_t h = 0x243f6a8885a308d3ull;
  for (size_t i = 0; i < N; ++i) h = mix64(h ^ (w[i] + 0x9e3779b97f4a7c15ull));
  return h;
}

double u01(uint64_t bits) { return (static_cast<double>(bits >> 11) + 1.0) * 0x1.0p-53; }

void gauss_pair(uint64_t key, double& g0, double& g1) {  // rng.hpp:35-42
  const double u1 = u01(mix64(key ^ 0x5555555555555555ull));
  const double u2 = u01(mix64(key ^ 0xaaaaaaaaaaaaaaaaull));
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double th = 2.0 * 3.141592653589793 * u2;
  g0 = r * std::cos(th);
  g1 = r * std::sin(th);
}

// RngStream, rng.hpp:45-70: gauss() keeps a spare, gauss_cplx() does not.
struct Stream {
  uint64_t key, counter = 0;
  double spare = 0.0;
  bool have_spare = false;
  explicit Stream(uint64_t k) : key(k) {}
  double gauss() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double a, b;
    const uint64_t w[2] = {key, ++counter};
    gauss_pair(key_hash(w), a, b);
    spare = b;
    have_spare = true;
    return a;
  }
  Cplx gauss_cplx() {
    double a, b;
    const uint64_t w[2] = {key, ++counter};
    gauss_pair(key_hash(w), a, b);
    return {a, b};
  }
};

// Small dense row-major complex matrix.
struct M {
  int n = 0;
  std::vector<Cplx> e;
  M() = default;
  explicit M(int k) : n(k), e(static_cast<size_t>(k) * k) {}
  Cplx& at(int i, int j) { return e[static_cast<size_t>(i) * n + j]; }
  const Cplx& at(int i, int j) const { return e[static_cast<size_t>(i) * n + j]; }
  static M eye(int k) {
    M m(k);
    for (int i = 0; i < k; ++i) m.at(i, i) = 1.0;
    return m;
  }
  M operator*(const M& o) const {  // matrix.hpp:30-38 loop order
    M r(n);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) {
        const Cplx a = at(i, k);
        for (int j = 0; j < n; ++j) r.at(i, j) += a * o.at(k, j);
      }
    return r;
  }
  M dagger() const {
    M r(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) r.at(j, i) = std::conj(at(i, j));
    return r;
  }
  double max_abs() const {
    double m = 0.0;
    for (const auto& v : e) m = std::max(m, std::abs(v));
    return m;
  }
  Cplx det() const {  // matrix.hpp:80-106: LU with partial pivoting
    M a = *this;
    Cplx d = 1.0;
    for (int k = 0; k < n; ++k) {
      int piv = k;
      double best = std::abs(a.at(k, k));
      for (int i = k + 1; i < n; ++i) {
        const double m = std::abs(a.at(i, k));
        if (m > best) {
          best = m;
          piv = i;
        }
      }
      if (best == 0.0) return 0.0;
      if (piv != k) {
        for (int j = 0; j < n; ++j) std::swap(a.at(k, j), a.at(piv, j));
        d = -d;
      }
      d *= a.at(k, k);
      for (int i = k + 1; i < n; ++i) {
        const Cplx f = a.at(i, k) / a.at(k, k);
        for (int j = k; j < n; ++j) a.at(i, j) -= f * a.at(k, j);
      }
    }
    return d;
  }
};

std::vector<M> make_generators(int n) {  // group.cpp:42-71
  std::vector<M> ts;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      M t(n);
      t.at(i, j) = 0.5;
      t.at(j, i) = 0.5;
      ts.push_back(t);
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      M t(n);
      t.at(i, j) = Cplx(0.0, -0.5);
      t.at(j, i) = Cplx(0.0, 0.5);
      ts.push_back(t);
    }
  for (int k = 1; k < n; ++k) {
    M t(n);
    const double norm = 1.0 / std::sqrt(2.0 * k * (k + 1));
    for (int i = 0; i < k; ++i) t.at(i, i) = norm;
    t.at(k, k) = -static_cast<double>(k) * norm;
    ts.push_back(t);
  }
  return ts;
}

M random_su_n(int n, Stream& rng) {  // group.cpp:82-114
  for (int attempt = 0; attempt < 16; ++attempt) {
    M u(n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) u.at(i, j) = rng.gauss_cplx();
    bool degenerate = false;
    for (int j = 0; j < n && !degenerate; ++j) {
      for (int k = 0; k < j; ++k) {
        Cplx proj = 0.0;
        for (int i = 0; i < n; ++i) proj += std::conj(u.at(i, k)) * u.at(i, j);
        for (int i = 0; i < n; ++i) u.at(i, j) -= proj * u.at(i, k);
      }
      double nrm = 0.0;
      for (int i = 0; i < n; ++i) nrm += std::norm(u.at(i, j));
      nrm = std::sqrt(nrm);
      if (nrm < 1e-8) {
        degenerate = true;
        break;
      }
      for (int i = 0; i < n; ++i) u.at(i, j) /= nrm;
    }
    if (degenerate) continue;
    const double phi = std::arg(u.det());
    const Cplx s = std::polar(1.0, -phi / n);
    for (auto& v : u.e) v *= s;
    return u;
  }
  throw Error(LBCU_CONFIG_ERROR, "random group element generation degenerated repeatedly");
}

std::vector<std::pair<int, int>> pairs(int n, bool diag) {
  std::vector<std::pair<int, int>> ps;
  for (int i = 0; i < n; ++i)
    for (int j = diag ? i : i + 1; j < n; ++j) ps.emplace_back(i, j);
  return ps;
}

M represent(const M& u, int rep, const std::vector<M>& ts) {  // group.cpp:119-196
  const int n = u.n;
  if (rep == LBCU_REP_FUNDAMENTAL) return u;
  if (rep == LBCU_REP_ADJOINT) {
    const int d = n * n - 1;
    const M udag = u.dagger();
    M r(d);
    std::vector<M> rot;
    rot.reserve(d);
    for (int b = 0; b < d; ++b) rot.push_back(u * ts[b] * udag);
    for (int a = 0; a < d; ++a)
      for (int b = 0; b < d; ++b) {
        Cplx t = 0.0;
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) t += ts[a].at(i, j) * rot[b].at(j, i);
        r.at(a, b) = 2.0 * t;
      }
    return r;
  }
  const bool sym = rep == LBCU_REP_SYMMETRIC;
  const auto ps = pairs(n, sym);
  const int d = static_cast<int>(ps.size());
  const double rt2 = std::sqrt(2.0);
  M r(d);
  for (int p = 0; p < d; ++p) {
    const auto [i, j] = ps[p];
    for (int q = 0; q < d; ++q) {
      const auto [k, l] = ps[q];
      Cplx v;
      if (!sym) {
        v = u.at(i, k) * u.at(j, l) - u.at(i, l) * u.at(j, k);
      } else if (i == j && k == l) {
        v = u.at(i, k) * u.at(i, k);
      } else if (i == j) {
        v = rt2 * u.at(i, k) * u.at(i, l);
      } else if (k == l) {
        v = rt2 * u.at(i, k) * u.at(j, k);
      } else {
        v = u.at(i, k) * u.at(j, l) + u.at(i, l) * u.at(j, k);
      }
      r.at(p, q) = v;
    }
  }
  return r;
}

// exp(A) by scaling and squaring with a degree-16 Taylor polynomial.
M expm(M a) {
  const int n = a.n;
  int sq = 0;
  double nrm = a.max_abs() * n;
  while (nrm > 0.5) {
    nrm *= 0.5;
    ++sq;
  }
  const double sc = std::ldexp(1.0, -sq);
  for (auto& v : a.e) v *= sc;
  M e = M::eye(n), term = M::eye(n);
  for (int k = 1; k <= 16; ++k) {
    term = term * a;
    for (auto& v : term.e) v *= 1.0 / k;
    for (size_t i = 0; i < e.e.size(); ++i) e.e[i] += term.e[i];
  }
  for (int k = 0; k < sq; ++k) e = e * e;
  return e;
}

template <class F>
void parallel_sites(int64_t n, int nthreads, F&& f) {
  if (nthreads <= 0) nthreads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  nthreads = static_cast<int>(std::min<int64_t>(nthreads, std::max<int64_t>(1, n / 256)));
  if (nthreads <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> errs(nthreads);
  for (int k = 0; k < nthreads; ++k)
    th.emplace_back([&, k] {
      try {
        f(n * k / nthreads, n * (k + 1) / nthreads);
      } catch (...) {
        errs[k] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

void host_spinor_random(const Geometry& geo, int dr, uint64_t seed, uint64_t field, double* out) {
  const int nv = 4 * dr;
  parallel_sites(geo.volume, 0, [&](int64_t lo, int64_t hi) {
    for (int64_t s = lo; s < hi; ++s) {
      int gc[4];
      geo.global_coords(s, gc);
      double* rec = out + s * nv * 2;
      for (int spin = 0; spin < 4; ++spin)
        for (int c = 0; c < dr; ++c) {
          const uint64_t w[9] = {seed,
                                 0x53u,
                                 field,
                                 static_cast<uint64_t>(gc[0]),
                                 static_cast<uint64_t>(gc[1]),
                                 static_cast<uint64_t>(gc[2]),
                                 static_cast<uint64_t>(gc[3]),
                                 static_cast<uint64_t>(spin),
                                 static_cast<uint64_t>(c)};
          gauss_pair(key_hash(w), rec[2 * (spin * dr + c)], rec[2 * (spin * dr + c) + 1]);
        }
    }
  });
}

void host_gauge_random(const Geometry& geo, int n, int rep, int links, uint64_t seed, double eps,
                       int nthreads, double* out) {
  const int dr = rep_dim(rep, n);
  const bool real = rep == LBCU_REP_ADJOINT;
  const int per_entry = real ? 1 : 2;
  const size_t per_link = static_cast<size_t>(dr) * dr * per_entry;
  if (links == LBCU_LINKS_NEAR_UNIT && rep != LBCU_REP_FUNDAMENTAL)
    throw Error(LBCU_CONFIG_ERROR, "near-unit links are generated for the fundamental rep only");
  const std::vector<M> ts = make_generators(n);
  parallel_sites(geo.volume, nthreads, [&](int64_t lo, int64_t hi) {
    for (int64_t s = lo; s < hi; ++s) {
      int gc[4];
      geo.global_coords(s, gc);
      for (int mu = 0; mu < 4; ++mu) {
        double* dst = out + (static_cast<size_t>(s) * 4 + mu) * per_link;
        if (links == LBCU_LINKS_UNIT) {  // fields.cpp:71-84
          std::memset(dst, 0, sizeof(double) * per_link);
          for (int i = 0; i < dr; ++i) dst[(static_cast<size_t>(i) * dr + i) * per_entry] = 1.0;
          continue;
        }
        const uint64_t w[7] = {seed,
                               0x47u,
                               static_cast<uint64_t>(gc[0]),
                               static_cast<uint64_t>(gc[1]),
                               static_cast<uint64_t>(gc[2]),
                               static_cast<uint64_t>(gc[3]),
                               static_cast<uint64_t>(mu)};
        Stream rng(key_hash(w));
        M u;
        if (links == LBCU_LINKS_HAAR) {
          u = random_su_n(n, rng);
        } else {  // near-unit: a = i eps sum_a xi_a T_a
          M a(n);
          for (size_t k = 0; k < ts.size(); ++k) {
            const double xi = rng.gauss();
            for (int i = 0; i < n; ++i)
              for (int j = 0; j < n; ++j) a.at(i, j) += Cplx(0.0, eps * xi) * ts[k].at(i, j);
          }
          u = expm(a);
        }
        const M r = represent(u, rep, ts);
        for (int i = 0; i < dr; ++i)
          for (int j = 0; j < dr; ++j) {
            const Cplx v = r.at(i, j);
            if (real) {
              dst[i * dr + j] = v.real();
            } else {
              dst[2 * (i * dr + j)] = v.real();
              dst[2 * (i * dr + j) + 1] = v.imag();
            }
          }
      }
    }
  });
}

}  // namespace lbcu
