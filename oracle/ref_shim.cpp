// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (latbench, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). The
// tests, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg load it through ctypes as the checker and the CPU baseline.
//
// All field arrays cross this boundary in GLOBAL lexicographic site order
// (t,x,y,z), z fastest — exactly the interior layout of a one-worker run
// (proj/include/latbench/geometry.hpp:40-42, proj/src/fields.cpp:14-40):
//   spinor: [site][spin 4][colour dr] complex<double>
//   gauge : [site][mu 4][row dr][col dr] complex<double> (real double for the
//           adjoint, proj/include/latbench/fields.hpp:37-57)
// Operators scatter those arrays over any worker grid (one std::thread per
// worker, the reference's own run_workers, proj/src/transport.cpp:114-140),
// run the reference kernel, and gather the result back.
//
// Pieces NOT in the reference, composed here on top of its public API and
// marked as such:
//   * antiperiodic time BC: U_0 negated on the last global time slice before
//     the gauge halo exchange;
//   * near-unit links U = exp(i eps H), H = sum_a xi_a T_a;
//   * the even-odd Schur operator Mhat and the eo CG, built from
//     apply_dirac (hop = (4+m) psi - D psi) and the reference cg_solve.

#include <latbench/bench.hpp>
#include <latbench/errors.hpp>
#include <latbench/fields.hpp>
#include <latbench/flops.hpp>
#include <latbench/gamma.hpp>
#include <latbench/geometry.hpp>
#include <latbench/group.hpp>
#include <latbench/kernels.hpp>
#include <latbench/rng.hpp>
#include <latbench/solver.hpp>
#include <latbench/transport.hpp>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

using namespace latbench;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const NonConvergence*>(&e)) return 4;
  if (dynamic_cast<const TransportError*>(&e)) return 3;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const ContractViolation*>(&e)) return 1;
  return 9;
}

#define SHIM_TRY try {
#define SHIM_CATCH                         \
  }                                        \
  catch (const std::exception& e) {        \
    return fail(e);                        \
  }                                        \
  return 0;

Coord4 c4(const int* a) { return {a[0], a[1], a[2], a[3]}; }

int64_t lex(const Coord4& g, const Coord4& L) {
  return ((static_cast<int64_t>(g[0]) * L[1] + g[1]) * L[2] + g[2]) * L[3] + g[3];
}

int vals_per_link_entry(bool real) { return real ? 1 : 2; }

// global array -> this worker's interior
void scatter_spinor(SpinorField& f, const double* glob) {
  const Geometry& geo = *f.geo;
  const int nv = f.vals_per_site();
  for (int s = 0; s < geo.interior; ++s) {
    const int64_t G = lex(geo.global_coords(s), geo.global);
    std::memcpy(f.site(s), glob + G * nv * 2, sizeof(double) * 2 * nv);
  }
}

void gather_spinor(const SpinorField& f, double* glob) {
  const Geometry& geo = *f.geo;
  const int nv = f.vals_per_site();
  for (int s = 0; s < geo.interior; ++s) {
    const int64_t G = lex(geo.global_coords(s), geo.global);
    std::memcpy(glob + G * nv * 2, f.site(s), sizeof(double) * 2 * nv);
  }
}

// global gauge array -> interior links; antiperiodic-in-time applied as the
// U_0 sign flip on the last global time slice.
void scatter_gauge(GaugeField& g, const double* glob, int bc_time) {
  const Geometry& geo = *g.geo;
  const size_t per_site = g.vals_per_site();
  for (int s = 0; s < geo.interior; ++s) {
    const Coord4 gc = geo.global_coords(s);
    const int64_t G = lex(gc, geo.global);
    const double flip0 = (bc_time && gc[0] == geo.global[0] - 1) ? -1.0 : 1.0;
    for (int mu = 0; mu < 4; ++mu) {
      const double sgn = mu == 0 ? flip0 : 1.0;
      const size_t n = static_cast<size_t>(g.dr) * g.dr;
      const size_t base = static_cast<size_t>(s) * per_site + mu * n;
      const size_t gbase = static_cast<size_t>(G) * per_site + mu * n;
      for (size_t k = 0; k < n; ++k) {
        if (g.real_links)
          g.rdata[base + k] = sgn * glob[gbase + k];
        else
          g.cdata[base + k] = Cplx(sgn * glob[2 * (gbase + k)], sgn * glob[2 * (gbase + k) + 1]);
      }
    }
  }
}

struct Problem {
  Coord4 global, grid;
  int n, dr;
  Representation rep;
  bool real;
};

Problem make_problem(const int* global, const int* grid, int n, int rep) {
  Problem p;
  p.global = c4(global);
  p.grid = c4(grid);
  p.n = n;
  p.rep = static_cast<Representation>(rep);
  p.dr = rep_dim(p.rep, n);
  p.real = rep_is_real(p.rep);
  return p;
}

// Zero the interior sites whose global parity differs from `keep`.
void mask_parity(SpinorField& f, int keep) {
  const Geometry& geo = *f.geo;
  for (int s = 0; s < geo.interior; ++s) {
    const Coord4 g = geo.global_coords(s);
    if (((g[0] + g[1] + g[2] + g[3]) & 1) != keep)
      for (int k = 0; k < f.vals_per_site(); ++k) f.site(s)[k] = Cplx(0.0, 0.0);
  }
}

// hop(psi) = (4+m) psi - D psi  (= 1/2 H psi), composed from apply_dirac.
void hop(SpinorField& out, const GaugeField& g, SpinorField& in, double mass, Worker& w,
         const ExchangePlan& plan) {
  apply_dirac(out, g, in, mass, w, plan);
  const double a = 4.0 + mass;
  const size_t n = static_cast<size_t>(out.geo->interior) * out.vals_per_site();
  for (size_t i = 0; i < n; ++i) out.data[i] = a * in.data[i] - out.data[i];
}

// Mhat x_e = (4+m) x_e - hop(hop(x_e))/(4+m) on even sites, zero on odd.
void mhat(SpinorField& out, const GaugeField& g, SpinorField& in, double mass, Worker& w,
          const ExchangePlan& plan, SpinorField& t1, SpinorField& t2) {
  copy_interior(t2, in);
  mask_parity(t2, 0);
  hop(t1, g, t2, mass, w, plan);
  mask_parity(t1, 1);
  hop(out, g, t1, mass, w, plan);
  const double a = 4.0 + mass;
  const size_t n = static_cast<size_t>(out.geo->interior) * out.vals_per_site();
  for (size_t i = 0; i < n; ++i) out.data[i] = a * t2.data[i] - out.data[i] / a;
  mask_parity(out, 0);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

long long ref_flops_per_site(int kernel, int dr, int real_rep) {
  return flops_per_site(static_cast<BenchKernel>(kernel), dr, real_rep != 0);
}

int ref_rep_dim(int rep, int n) {
  try {
    return rep_dim(static_cast<Representation>(rep), n);
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

void ref_hop_tables(int* out) {
  // [pair 4x2][proj_phase 4x2][rec_src 4x2][rec_phase 4x2], phases as Ph enum values
  const HopTables& t = hop_tables();
  for (int mu = 0; mu < 4; ++mu)
    for (int a = 0; a < 2; ++a) {
      out[0 + mu * 2 + a] = t.proj_pair[mu][a];
      out[8 + mu * 2 + a] = static_cast<int>(t.proj_phase[mu][a]);
      out[16 + mu * 2 + a] = t.rec_src[mu][a];
      out[24 + mu * 2 + a] = static_cast<int>(t.rec_phase[mu][a]);
    }
}

void ref_gamma_matrices(double* out) {  // 5 x 4 x 4 complex
  const auto& g = gamma_matrices();
  for (int k = 0; k < 5; ++k)
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        out[((k * 4 + i) * 4 + j) * 2] = g[k].at(i, j).real();
        out[((k * 4 + i) * 4 + j) * 2 + 1] = g[k].at(i, j).imag();
      }
}

int ref_generators(int n, double* out) {
  SHIM_TRY const auto ts = generators(n);
  size_t o = 0;
  for (const auto& t : ts)
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        out[o++] = t.at(i, j).real();
        out[o++] = t.at(i, j).imag();
      }
  SHIM_CATCH
}

int ref_random_group_element(int n, uint64_t key, double* out) {
  SHIM_TRY RngStream rng(key);
  const Mat u = random_group_element(n, rng);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      out[2 * (i * n + j)] = u.at(i, j).real();
      out[2 * (i * n + j) + 1] = u.at(i, j).imag();
    }
  SHIM_CATCH
}

int ref_represent(int n, int rep, const double* u_in, double* out) {
  SHIM_TRY Mat u(n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) u.at(i, j) = Cplx(u_in[2 * (i * n + j)], u_in[2 * (i * n + j) + 1]);
  const RepMatrix r = represent(u, static_cast<Representation>(rep));
  const int d = r.dim();
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      out[2 * (i * d + j)] = r.m.at(i, j).real();
      out[2 * (i * d + j) + 1] = r.m.at(i, j).imag();
    }
  SHIM_CATCH
}

void ref_mix(uint64_t key, double* g0, double* g1) { gauss_pair(key, *g0, *g1); }

uint64_t ref_key_hash(const uint64_t* words, int n) {
  // key_hash takes an initializer_list; expose the arities the fields use
  switch (n) {
    case 1: return key_hash({words[0]});
    case 2: return key_hash({words[0], words[1]});
    case 7: return key_hash({words[0], words[1], words[2], words[3], words[4], words[5], words[6]});
    case 9:
      return key_hash({words[0], words[1], words[2], words[3], words[4], words[5], words[6],
                       words[7], words[8]});
    default: return 0;
  }
}

// ---- seeded inputs (one worker, the whole lattice) ------------------------

int ref_spinor_random(const int* global, int dr, uint64_t seed, uint64_t field_index,
                      double* out) {
  SHIM_TRY const int grid[4] = {1, 1, 1, 1};
  const Geometry geo = build_geometry(c4(global), c4(grid), 0, false);
  const SpinorField f = init_spinor_random(geo, dr, seed, field_index);
  gather_spinor(f, out);
  SHIM_CATCH
}

// Per-worker interior (reference local lexicographic order) of a decomposed run.
int ref_spinor_random_local(const int* global, const int* grid, int rank, int dr, uint64_t seed,
                            uint64_t field_index, double* out) {
  SHIM_TRY const Geometry geo = build_geometry(c4(global), c4(grid), rank, false);
  const SpinorField f = init_spinor_random(geo, dr, seed, field_index);
  std::memcpy(out, f.data.data(), sizeof(double) * 2 * geo.interior * f.vals_per_site());
  SHIM_CATCH
}

int ref_gauge_random(const int* global, int n, int rep, uint64_t seed, int nthreads, double* out) {
  SHIM_TRY
  // Decomposition-invariant keyed generation (proj/src/fields.cpp:86-107):
  // run it over a T-split worker grid so large lattices generate in parallel,
  // then gather in global order.
  Coord4 grid{1, 1, 1, 1};
  const Coord4 G = c4(global);
  for (int k = nthreads; k > 1; --k)
    if (G[0] % k == 0) {
      grid[0] = k;
      break;
    }
  const Representation r = static_cast<Representation>(rep);
  const int dr = rep_dim(r, n);
  const bool real = rep_is_real(r);
  const size_t per_site = static_cast<size_t>(4) * dr * dr * vals_per_link_entry(real);
  run_workers(grid, [&](Worker& w) {
    const Geometry geo = build_geometry(G, grid, w.rank(), false);
    GaugeField g = make_gauge(geo, n, r);
    randomize_gauge_interior(g, seed);
    for (int s = 0; s < geo.interior; ++s) {
      const int64_t gi = lex(geo.global_coords(s), G);
      if (real)
        std::memcpy(out + gi * per_site, g.rdata.data() + s * per_site, sizeof(double) * per_site);
      else
        std::memcpy(out + gi * per_site, reinterpret_cast<const double*>(g.cdata.data()) + s * per_site,
                    sizeof(double) * per_site);
    }
  });
  SHIM_CATCH
}

int ref_gauge_unit(const int* global, int n, int rep, double* out) {
  SHIM_TRY const int grid[4] = {1, 1, 1, 1};
  const Geometry geo = build_geometry(c4(global), c4(grid), 0, false);
  const GaugeField g = make_unit_gauge(geo, n, static_cast<Representation>(rep));
  const size_t per_site = g.vals_per_site() * vals_per_link_entry(g.real_links);
  if (g.real_links)
    std::memcpy(out, g.rdata.data(), sizeof(double) * per_site * geo.interior);
  else
    std::memcpy(out, g.cdata.data(), sizeof(double) * per_site * geo.interior);
  SHIM_CATCH
}

// NOT IN THE REFERENCE (BASELINE config 3): near-unit fundamental links
// U = exp(i eps H), H = sum_a xi_a T_a, xi_a = RngStream::gauss() in
// generator order from RngStream(key_hash{seed,0x47,t,x,y,z,mu})
// (SURVEY.md §8d pins this normalisation). exp by scaling and squaring with a
// degree-16 Taylor polynomial on the reference's Mat type.
Mat near_unit_link(int n, double eps, uint64_t seed, const Coord4& gc, int mu) {
  const auto& ts = cached_generators(n);
  RngStream rng(key_hash({seed, 0x47u, static_cast<uint64_t>(gc[0]), static_cast<uint64_t>(gc[1]),
                          static_cast<uint64_t>(gc[2]), static_cast<uint64_t>(gc[3]),
                          static_cast<uint64_t>(mu)}));
  Mat a(n);  // a = i eps H
  for (size_t k = 0; k < ts.size(); ++k) {
    const double xi = rng.gauss();
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) a.at(i, j) += Cplx(0.0, eps * xi) * ts[k].at(i, j);
  }
  int sq = 0;
  double nrm = a.max_abs() * n;
  while (nrm > 0.5) {
    nrm *= 0.5;
    ++sq;
  }
  a.scale(std::ldexp(1.0, -sq));
  Mat e = Mat::identity(n), term = Mat::identity(n);
  for (int k = 1; k <= 16; ++k) {
    term = term * a;
    term.scale(1.0 / k);
    e = e + term;
  }
  for (int k = 0; k < sq; ++k) e = e * e;
  return e;
}

int ref_gauge_near_unit(const int* global, int n, double eps, uint64_t seed, double* out) {
  SHIM_TRY const Coord4 G = c4(global);
  (void)cached_generators(n);  // build the cache before the workers read it
  const int64_t V = static_cast<int64_t>(G[0]) * G[1] * G[2] * G[3];
  // T-split over the host threads (keyed per global site: order-independent)
  Coord4 grid{1, 1, 1, 1};
  const int nthreads = static_cast<int>(std::thread::hardware_concurrency());
  for (int k = nthreads; k > 1; --k)
    if (G[0] % k == 0) {
      grid[0] = k;
      break;
    }
  const int64_t per = V / grid[0];
  run_workers(grid, [&](Worker& w) {
    for (int64_t s = w.rank() * per; s < (w.rank() + 1) * per; ++s) {
      int64_t r = s;
      Coord4 gc;
      gc[3] = r % G[3];
      r /= G[3];
      gc[2] = r % G[2];
      r /= G[2];
      gc[1] = r % G[1];
      gc[0] = r / G[1];
      for (int mu = 0; mu < 4; ++mu) {
        const Mat e = near_unit_link(n, eps, seed, gc, mu);
        for (int i = 0; i < n; ++i)
          for (int j = 0; j < n; ++j) {
            const size_t o = ((static_cast<size_t>(s) * 4 + mu) * n * n + i * n + j) * 2;
            out[o] = e.at(i, j).real();
            out[o + 1] = e.at(i, j).imag();
          }
      }
    }
  });
  SHIM_CATCH
}

// ---- operators over a worker grid ------------------------------------------

int ref_apply_dirac(const int* global, const int* grid, int n, int rep, int bc_time, double mass,
                    const double* gauge, const double* in, double* out) {
  SHIM_TRY const Problem p = make_problem(global, grid, n, rep);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = make_gauge(geo, p.n, p.rep);
    scatter_gauge(g, gauge, bc_time);
    halo_exchange(w, plan, g);
    SpinorField a = make_spinor(geo, p.dr), b = make_spinor(geo, p.dr);
    scatter_spinor(a, in);
    apply_dirac(b, g, a, mass, w, plan);
    gather_spinor(b, out);
  });
  SHIM_CATCH
}

int ref_apply_h(const int* global, const int* grid, int n, int rep, int bc_time, double mass,
                const double* gauge, const double* in, double* out) {
  SHIM_TRY const Problem p = make_problem(global, grid, n, rep);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = make_gauge(geo, p.n, p.rep);
    scatter_gauge(g, gauge, bc_time);
    halo_exchange(w, plan, g);
    SpinorField a = make_spinor(geo, p.dr), b = make_spinor(geo, p.dr), t = make_spinor(geo, p.dr);
    scatter_spinor(a, in);
    apply_h(b, g, a, mass, w, plan, t);
    gather_spinor(b, out);
  });
  SHIM_CATCH
}

// Counted twin of apply_dirac on one worker: returns the FLOP tally per site
// (proj/src/kernels.cpp:62-65, proj/include/latbench/kernel_ops.hpp:19-28).
int ref_counted_dirac(const int* global, int n, int rep, long long* flops_per_site_out) {
  SHIM_TRY const int grid[4] = {1, 1, 1, 1};
  const Problem p = make_problem(global, grid, n, rep);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, 0, false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = init_gauge_random(w, plan, geo, p.n, p.rep, 1);
    SpinorField a = init_spinor_random(geo, p.dr, 1, 0), b = make_spinor(geo, p.dr);
    FlopTally t;
    apply_dirac_counted(b, g, a, 0.1, w, plan, t);
    *flops_per_site_out = t.flops() / geo.interior;
  });
  SHIM_CATCH
}

int ref_sqnorm(const int* global, const int* grid, int dr, const double* in, double* result) {
  SHIM_TRY const Coord4 G = c4(global), P = c4(grid);
  run_workers(P, [&](Worker& w) {
    const Geometry geo = build_geometry(G, P, w.rank(), false);
    SpinorField a = make_spinor(geo, dr);
    scatter_spinor(a, in);
    const double v = sqnorm(a, w);
    if (w.rank() == 0) *result = v;
  });
  SHIM_CATCH
}

int ref_mul_add(const int* global, const int* grid, int dr, double c_re, double c_im, double* psi2,
                const double* psi1) {
  SHIM_TRY const Coord4 G = c4(global), P = c4(grid);
  run_workers(P, [&](Worker& w) {
    const Geometry geo = build_geometry(G, P, w.rank(), false);
    SpinorField a = make_spinor(geo, dr), b = make_spinor(geo, dr);
    scatter_spinor(a, psi2);
    scatter_spinor(b, psi1);
    w.barrier();  // every worker has read psi2 before anyone writes it back
    mul_add(a, Cplx(c_re, c_im), b);
    gather_spinor(a, psi2);
  });
  SHIM_CATCH
}

int ref_dot(const int* global, const int* grid, int dr, const double* a_in, const double* b_in,
            double* re, double* im) {
  SHIM_TRY const Coord4 G = c4(global), P = c4(grid);
  run_workers(P, [&](Worker& w) {
    const Geometry geo = build_geometry(G, P, w.rank(), false);
    SpinorField a = make_spinor(geo, dr), b = make_spinor(geo, dr);
    scatter_spinor(a, a_in);
    scatter_spinor(b, b_in);
    const Cplx v = dot(a, b, w);
    if (w.rank() == 0) {
      *re = v.real();
      *im = v.imag();
    }
  });
  SHIM_CATCH
}

// Reference plain CG on H = gamma5 D gamma5 D (proj/src/solver.cpp:24-82).
// history must hold max_iterations doubles.
int ref_cg_h(const int* global, const int* grid, int n, int rep, int bc_time, double mass,
             const double* gauge, const double* rhs, double tol, int max_iterations, double* x,
             long* iterations, double* rel, double* true_rel, double* seconds, double* history) {
  SHIM_TRY const Problem p = make_problem(global, grid, n, rep);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = make_gauge(geo, p.n, p.rep);
    scatter_gauge(g, gauge, bc_time);
    halo_exchange(w, plan, g);
    SpinorField b = make_spinor(geo, p.dr), t = make_spinor(geo, p.dr);
    scatter_spinor(b, rhs);
    SteadyClock clock;
    CgSettings st;
    st.tolerance = tol;
    st.max_iterations = max_iterations;
    const CgOutcome o = cg_solve(make_h_operator(g, mass, w, plan, t), b, st, w, clock);
    gather_spinor(o.solution, x);
    if (w.rank() == 0) {
      *iterations = o.iterations;
      *rel = o.rel_residual;
      *true_rel = o.true_rel_residual;
      *seconds = o.seconds;
      for (size_t k = 0; k < o.residual_history.size(); ++k) history[k] = o.residual_history[k];
    }
  });
  SHIM_CATCH
}

// NOT IN THE REFERENCE: the even-odd Schur operator composed from the
// reference apply_dirac. in/out are full-lattice arrays; only
// even sites of `in` are read, odd sites of `out` are zero.
int ref_mhat(const int* global, const int* grid, int n, int rep, int bc_time, double mass,
             const double* gauge, const double* in, double* out) {
  SHIM_TRY const Problem p = make_problem(global, grid, n, rep);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = make_gauge(geo, p.n, p.rep);
    scatter_gauge(g, gauge, bc_time);
    halo_exchange(w, plan, g);
    SpinorField a = make_spinor(geo, p.dr), b = make_spinor(geo, p.dr);
    SpinorField t1 = make_spinor(geo, p.dr), t2 = make_spinor(geo, p.dr);
    scatter_spinor(a, in);
    mhat(b, g, a, mass, w, plan, t1, t2);
    gather_spinor(b, out);
  });
  SHIM_CATCH
}

// NOT IN THE REFERENCE: eo-preconditioned CG = the reference cg_solve driven
// by a LinearOp that applies gamma5 Mhat gamma5 Mhat (= Mhat^dag Mhat) on the
// even sublattice; rhs is the even part of `rhs`.
int ref_cg_eo(const int* global, const int* grid, int n, int rep, int bc_time, double mass,
              const double* gauge, const double* rhs, double tol, int max_iterations, double* x,
              long* iterations, double* rel, double* true_rel, double* seconds, double* history) {
  SHIM_TRY const Problem p = make_problem(global, grid, n, rep);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = make_gauge(geo, p.n, p.rep);
    scatter_gauge(g, gauge, bc_time);
    halo_exchange(w, plan, g);
    SpinorField b = make_spinor(geo, p.dr);
    scatter_spinor(b, rhs);
    mask_parity(b, 0);
    SpinorField t1 = make_spinor(geo, p.dr), t2 = make_spinor(geo, p.dr),
                t3 = make_spinor(geo, p.dr);
    LinearOp op = [&](SpinorField& out, SpinorField& in) {
      mhat(t3, g, in, mass, w, plan, t1, t2);
      apply_gamma5(t3);
      mhat(out, g, t3, mass, w, plan, t1, t2);
      apply_gamma5(out);
    };
    SteadyClock clock;
    CgSettings st;
    st.tolerance = tol;
    st.max_iterations = max_iterations;
    const CgOutcome o = cg_solve(op, b, st, w, clock);
    gather_spinor(o.solution, x);
    if (w.rank() == 0) {
      *iterations = o.iterations;
      *rel = o.rel_residual;
      *true_rel = o.true_rel_residual;
      *seconds = o.seconds;
      for (size_t k = 0; k < o.residual_history.size(); ++k) history[k] = o.residual_history[k];
    }
  });
  SHIM_CATCH
}

// ---- CPU baseline timing ----------------------------------------------------
// Per-worker inputs of the BASELINE workloads, generated in parallel on the
// worker's own interior (keyed per global site, so identical for any worker
// grid): Haar links via the reference's randomize_gauge_interior, or the
// near-unit links above (config 3); antiperiodic t as the U_0 sign flip on the
// last global time slice; then the reference gauge halo exchange
// (init_gauge_random, proj/src/transport.cpp:223-229, with the flip inserted).
GaugeField make_links(Worker& w, const ExchangePlan& plan, const Geometry& geo, const Problem& p,
                      int links, double eps, uint64_t seed, int bc_time) {
  GaugeField g = make_gauge(geo, p.n, p.rep);
  if (links == 1) {  // near-unit fundamental links
    if (p.rep != Representation::Fundamental) throw ConfigError("near-unit links are fundamental only");
    const size_t nn = static_cast<size_t>(p.n) * p.n;
    for (int s = 0; s < geo.interior; ++s) {
      const Coord4 gc = geo.global_coords(s);
      for (int mu = 0; mu < 4; ++mu) {
        const Mat e = near_unit_link(p.n, eps, seed, gc, mu);
        for (int i = 0; i < p.n; ++i)
          for (int j = 0; j < p.n; ++j) g.cdata[(static_cast<size_t>(s) * 4 + mu) * nn + i * p.n + j] = e.at(i, j);
      }
    }
  } else {
    randomize_gauge_interior(g, seed);
  }
  if (bc_time) {
    const size_t nn = static_cast<size_t>(g.dr) * g.dr;
    for (int s = 0; s < geo.interior; ++s) {
      if (geo.global_coords(s)[0] != geo.global[0] - 1) continue;
      const size_t base = static_cast<size_t>(s) * 4 * nn;  // mu = 0
      for (size_t k = 0; k < nn; ++k) {
        if (g.real_links)
          g.rdata[base + k] = -g.rdata[base + k];
        else
          g.cdata[base + k] = -g.cdata[base + k];
      }
    }
  }
  halo_exchange(w, plan, g);
  return g;
}

// The reference's own Dirac benchmark body (proj/src/bench.cpp:190-248) with a
// fixed application count on the BASELINE workload (links kind, antiperiodic
// t): fields generated per worker, `nwarm` warm-up applications, then
// `nsamples` samples of `napps` timed applications between barriers, rank-0
// clock, seconds[k] per sample.
int ref_bench_dirac(const int* global, const int* grid, int n, int rep, int links, double eps, int bc_time,
                    double mass, uint64_t seed, int nwarm, int napps, int nsamples, double* seconds) {
  SHIM_TRY const Problem p = make_problem(global, grid, n, rep);
  if (links == 1) (void)cached_generators(n);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = make_links(w, plan, geo, p, links, eps, seed, bc_time);
    SpinorField a = init_spinor_random(geo, p.dr, seed, 0), b = make_spinor(geo, p.dr);
    for (int i = 0; i < nwarm; ++i) apply_dirac(b, g, a, mass, w, plan);  // warm-up
    SteadyClock clock;
    for (int k = 0; k < nsamples; ++k) {
      w.barrier();
      const double t0 = w.rank() == 0 ? clock.seconds() : 0.0;
      for (int i = 0; i < napps; ++i) apply_dirac(b, g, a, mass, w, plan);
      w.barrier();
      const double dt = w.rank() == 0 ? clock.seconds() - t0 : 0.0;
      const double tot = w.global_sum(dt);
      if (w.rank() == 0) seconds[k] = tot;
    }
  });
  SHIM_CATCH
}

// The reference cg_solve (proj/src/solver.cpp:24-82) timed on the BASELINE
// workload, inputs generated per worker. eo = 0: the reference's own plain CG
// on H = g5 D g5 D (make_h_operator); eo = 1: the reference cg_solve driven by
// the composed g5 Mhat g5 Mhat LinearOp (as ref_cg_eo), rhs = even part of
// spinor field 0. tol > 0: a real solve to tol (at most max_iterations);
// tol <= 0: a bounded CPU sample of exactly max_iterations iterations with an
// unreachable tolerance, the NonConvergence at the cap caught. *seconds is
// the wall time of the whole cg_solve call on the rank-0 clock (setup and,
// for a solve, the exit true-residual check included), *iterations the
// iterations run, *true_rel the exit true residual (solve only, else -1),
// *seconds_per_iteration the solve time / iterations, or for a sample the
// time difference to a 1-iteration call / (max_iterations - 1), so that the
// per-solve setup (field allocation, |b|) is not counted per iteration.
int ref_cg_probe(const int* global, const int* grid, int n, int rep, int links, double eps, int bc_time,
                 double mass, uint64_t seed, int eo, double tol, int max_iterations, double* seconds,
                 long* iterations, double* true_rel, double* seconds_per_iteration) {
  SHIM_TRY const Problem p = make_problem(global, grid, n, rep);
  if (links == 1) (void)cached_generators(n);
  run_workers(p.grid, [&](Worker& w) {
    const Geometry geo = build_geometry(p.global, p.grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = make_links(w, plan, geo, p, links, eps, seed, bc_time);
    SpinorField b = init_spinor_random(geo, p.dr, seed, 0);
    if (eo) mask_parity(b, 0);
    SpinorField t1 = make_spinor(geo, p.dr), t2 = make_spinor(geo, p.dr), t3 = make_spinor(geo, p.dr);
    LinearOp op;
    if (eo) {
      op = [&](SpinorField& out, SpinorField& in) {
        mhat(t3, g, in, mass, w, plan, t1, t2);
        apply_gamma5(t3);
        mhat(out, g, t3, mass, w, plan, t1, t2);
        apply_gamma5(out);
      };
    } else {
      op = make_h_operator(g, mass, w, plan, t1);
    }
    SteadyClock clock;
    CgSettings st;
    st.tolerance = tol > 0.0 ? tol : 1e-300;
    st.max_iterations = max_iterations;
    long its = max_iterations;
    double trel = -1.0;
    auto timed = [&](int cap) {  // wall time of one cg_solve call, rank-0 clock
      st.max_iterations = cap;
      w.barrier();
      const double t0 = w.rank() == 0 ? clock.seconds() : 0.0;
      try {
        const CgOutcome o = cg_solve(op, b, st, w, clock);
        its = o.iterations;
        trel = o.true_rel_residual;
      } catch (const NonConvergence&) {
        if (tol > 0.0) throw;
        its = cap;
      }
      w.barrier();
      const double dt = w.rank() == 0 ? clock.seconds() - t0 : 0.0;
      return w.global_sum(dt);
    };
    double tot = 0.0, per_it = 0.0;
    if (tol > 0.0 || max_iterations < 2) {
      tot = timed(max_iterations);
      per_it = tot / std::max<long>(1, its);
    } else {  // sample: a 1-iteration call calibrates the setup cost away
      const double t1 = timed(1);
      tot = timed(max_iterations);
      per_it = (tot - t1) / (max_iterations - 1);
    }
    if (w.rank() == 0) {
      *seconds = tot;
      *iterations = its;
      *true_rel = trel;
      *seconds_per_iteration = per_it;
    }
  });
  SHIM_CATCH
}

#ifdef SHIM_HAVE_REPORT
// Report interop (proj/src/report.cpp:152-217): parse a format-1 JSON report
// with the reference's report_from_json and re-emit it with format_report
// (format 0 text, 1 json, 2 csv). rc 2 (ConfigError) for a report the
// reference rejects. *len is the full length; out gets at most cap-1 bytes.
int ref_report_reformat(const char* json_text, int format, char* out, size_t cap, size_t* len) {
  SHIM_TRY const BenchReport r = report_from_json(json_text);
  const ReportFormat f = format == 0 ? ReportFormat::Text : format == 1 ? ReportFormat::Json : ReportFormat::Csv;
  const std::string txt = format_report(r, f);
  *len = txt.size();
  if (cap > 0) {
    const size_t n = std::min(cap - 1, txt.size());
    std::memcpy(out, txt.data(), n);
    out[n] = 0;
  }
  SHIM_CATCH
}
#endif

}  // extern "C"
