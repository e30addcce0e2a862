// latbench_b200_dropin.hpp — source-level drop-in for the reference's hot-path
// calls, on the reference's OWN types.
//
// A latbench caller keeps its fields, geometry, workers and exchange plans
// (latbench::SpinorField / GaugeField / Worker / ExchangePlan / Clock from
// /root/reference/proj/include/latbench/*.hpp, host memory, run_workers
// threads) and swaps the namespace of the hot calls only:
//
//   latbench::apply_dirac(out, g, in, m, w, plan)        kernels.hpp:19-20
//   latbench::apply_h(out, g, in, m, w, plan, tmp)       solver.hpp:32-33
//   latbench::make_h_operator(g, m, w, plan, tmp)        solver.hpp:36-37
//   latbench::cg_solve(op, rhs, settings, w, clock)      solver.hpp:43-44
//   latbench::consistency_check(g, rhs, m, st, w, plan, clock)   solver.hpp:59-61
//
// become latbench::gpu::<same name>(<same arguments>) (or
// latbench_b200::dropin::...). Each worker (rank) is bound to one library
// context on GPU rank % device_count, shared by every call with the same
// global lattice and worker grid; a multi-worker group becomes an in-process
// thread world, so the calls stay collective exactly as in the reference.
// Links are uploaded once per GaugeField (again when its storage moves or a
// 256-value fingerprint of the links changes); after changing link values
// in place call invalidate(gauge). Worker contexts are keyed by (global
// lattice, grid, rank): two groups of the same shape must not run at once. The BC is
// whatever the links carry (an antiperiodic sign baked into U_0 by the caller
// is reproduced as given). Spinors cross PCIe in the reference's interior
// layout on every call; halo slots of `in` are not written (the reference
// fills them as a side effect of its exchange).
//
// cg_solve runs entirely on the device when `op` came from
// latbench::gpu::make_h_operator (fused D^dag D CG, lbcu_cg_solve_h); any
// other LinearOp is called back on the host every iteration on the
// reference's fields (lbcu_cg_solve with a callback). Errors are the
// reference's exception types (errors.hpp:9-63). Timing follows the
// reference: barrier, rank-0 Clock, global_sum.
//
// Needs the reference headers on the include path and its library at link
// time (for Worker, make_spinor, the exception types); tests/cpp/dropin_demo.cpp
// is the compile-and-run check.
#pragma once

#include <latbench/clock.hpp>
#include <latbench/errors.hpp>
#include <latbench/fields.hpp>
#include <latbench/kernels.hpp>
#include <latbench/solver.hpp>
#include <latbench/transport.hpp>

#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "lbcu.h"

namespace latbench_b200 {
namespace dropin {

namespace detail {

// status code -> the reference's exception classes
inline void check(int rc, long iters = 0, double best = 0.0) {
  if (rc == LBCU_OK) return;
  const std::string msg = lbcu_last_error();
  switch (rc) {
    case LBCU_CONTRACT_VIOLATION: throw latbench::ContractViolation(msg);
    case LBCU_CONFIG_ERROR:
      if (msg.find("divisible") != std::string::npos || msg.find("floor") != std::string::npos)
        throw latbench::DecompositionError(msg);
      throw latbench::ConfigError(msg);
    case LBCU_TRANSPORT_ERROR: throw latbench::TransportError(msg);
    case LBCU_NON_CONVERGENCE: throw latbench::NonConvergence(iters, best);
    default: throw latbench::Error("device: " + msg);
  }
}

struct DeviceGauge {
  lbcu_gauge h = nullptr;
  const void* data = nullptr;  // host storage the upload came from
  size_t size = 0;
  uint64_t sample = 0;         // fingerprint of 256 strided link values
};

// Fingerprint of the host links: 256 values spread over the whole array, so
// a GaugeField re-created at a recycled address (same vector storage, new
// links) is not mistaken for the uploaded one. In-place edits that miss the
// sampled entries still need invalidate().
inline uint64_t link_sample(const double* v, size_t n) {
  uint64_t h = 0x9e3779b97f4a7c15ULL ^ n;
  if (n == 0) return h;
  const size_t step = n / 256 + 1;
  for (size_t i = 0; i < n; i += step) {
    uint64_t bits;
    std::memcpy(&bits, v + i, sizeof(bits));
    h = (h ^ bits) * 0x100000001b3ULL;
  }
  return h;
}

struct RankState {
  lbcu_ctx ctx = nullptr;
  std::map<int, std::array<lbcu_spinor, 2>> work;  // by dr: in, out (FULL)
  std::map<const latbench::GaugeField*, DeviceGauge> gauges;
};

struct Registry {
  std::mutex m;
  std::map<std::array<int, 8>, lbcu_world> worlds;  // (global, grid)
  std::map<std::array<int, 9>, RankState> ranks;    // (global, grid, rank)
};

inline Registry& registry() {
  static Registry r;
  return r;
}

inline RankState& rank_state(latbench::Worker& w, const latbench::Geometry& geo) {
  Registry& R = registry();
  std::array<int, 8> wk{};
  std::array<int, 9> rk{};
  for (int d = 0; d < 4; ++d) {
    wk[d] = rk[d] = geo.global[d];
    wk[4 + d] = rk[4 + d] = geo.grid[d];
  }
  rk[8] = w.rank();
  lbcu_world world = nullptr;
  {
    std::lock_guard<std::mutex> lk(R.m);
    auto it = R.ranks.find(rk);
    if (it != R.ranks.end()) return it->second;
    if (w.size() > 1) {
      auto wi = R.worlds.find(wk);
      if (wi == R.worlds.end()) {
        check(lbcu_world_threads(w.size(), &world));
        R.worlds[wk] = world;
      } else {
        world = wi->second;
      }
    }
  }
  const int ndev = lbcu_device_count();
  if (ndev < 1) throw latbench::Error("latbench_b200: no CUDA device");
  RankState st;  // created outside the lock: other ranks may be doing the same
  check(lbcu_ctx_create(world, w.rank(), w.rank() % ndev, geo.global.data(), geo.grid.data(), 0, &st.ctx));
  std::lock_guard<std::mutex> lk(R.m);
  return R.ranks.emplace(rk, st).first->second;
}

inline lbcu_gauge device_gauge(RankState& rs, const latbench::GaugeField& g) {
  const void* data = g.real_links ? static_cast<const void*>(g.rdata.data()) : g.cdata.data();
  const size_t size = g.real_links ? g.rdata.size() : g.cdata.size();
  const uint64_t sample = link_sample(static_cast<const double*>(data), size * (g.real_links ? 1 : 2));
  std::lock_guard<std::mutex> lk(registry().m);  // invalidate() may scan the maps
  DeviceGauge& dg = rs.gauges[&g];
  if (dg.h && dg.data == data && dg.size == size && dg.sample == sample) return dg.h;
  if (dg.h) lbcu_gauge_destroy(dg.h);
  dg = DeviceGauge{};
  lbcu_gauge h = nullptr;
  // the reference's links carry any time BC themselves: periodic on the device
  check(lbcu_gauge_create(rs.ctx, g.group_rank, static_cast<int>(g.rep), LBCU_BC_PERIODIC, &h));
  const int rc = lbcu_gauge_upload(h, static_cast<const double*>(data));
  if (rc != LBCU_OK) {
    lbcu_gauge_destroy(h);
    check(rc);
  }
  dg.h = h;
  dg.data = data;
  dg.size = size;
  dg.sample = sample;
  return h;
}

inline std::array<lbcu_spinor, 2>& work(RankState& rs, int dr) {
  auto& wk = rs.work[dr];
  for (auto& s : wk)
    if (!s) check(lbcu_spinor_create(rs.ctx, dr, LBCU_FULL, &s));
  return wk;
}

inline void need(bool ok, const char* what) {
  if (!ok) throw latbench::ContractViolation(what);
}

inline const double* host(const latbench::SpinorField& f) {
  return reinterpret_cast<const double*>(f.data.data());
}
inline double* host(latbench::SpinorField& f) { return reinterpret_cast<double*>(f.data.data()); }

}  // namespace detail

// Forget the device copy of a GaugeField (after changing its links in place).
inline void invalidate(const latbench::GaugeField& g) {
  auto& R = detail::registry();
  std::lock_guard<std::mutex> lk(R.m);
  for (auto& kv : R.ranks) {
    auto it = kv.second.gauges.find(&g);
    if (it == kv.second.gauges.end()) continue;
    lbcu_gauge_destroy(it->second.h);
    kv.second.gauges.erase(it);
  }
}

// Free every context, world and device field the drop-in layer created (call
// after run_workers has returned).
inline void release() {
  auto& R = detail::registry();
  std::lock_guard<std::mutex> lk(R.m);
  for (auto& kv : R.ranks) {
    for (auto& g : kv.second.gauges) lbcu_gauge_destroy(g.second.h);
    for (auto& w : kv.second.work)
      for (auto s : w.second) lbcu_spinor_destroy(s);
    lbcu_ctx_destroy(kv.second.ctx);
  }
  R.ranks.clear();
  for (auto& kv : R.worlds) lbcu_world_destroy(kv.second);
  R.worlds.clear();
}

// kernels.hpp:19-20 — out = D in (interior), collective.
inline void apply_dirac(latbench::SpinorField& out, const latbench::GaugeField& gauge, latbench::SpinorField& in,
                        double mass, latbench::Worker& w, const latbench::ExchangePlan& plan) {
  detail::need(in.geo && out.geo && gauge.geo && plan.geo, "apply_dirac: field without geometry");
  detail::need(&out != &in, "apply_dirac: out aliases in");
  detail::need(out.dr == in.dr && gauge.dr == in.dr, "apply_dirac: representation dimensions differ");
  detail::RankState& rs = detail::rank_state(w, *in.geo);
  const lbcu_gauge g = detail::device_gauge(rs, gauge);
  auto& wk = detail::work(rs, in.dr);
  detail::check(lbcu_spinor_upload(wk[0], detail::host(in)));
  detail::check(lbcu_dphi(wk[1], g, wk[0], mass));
  detail::check(lbcu_spinor_download(wk[1], detail::host(out)));
}

// solver.hpp:32-33 — out = g5 D g5 D in; `tmp` is caller scratch (not written).
inline void apply_h(latbench::SpinorField& out, const latbench::GaugeField& gauge, latbench::SpinorField& in,
                    double mass, latbench::Worker& w, const latbench::ExchangePlan& plan,
                    latbench::SpinorField& /*tmp*/) {
  detail::need(in.geo && out.geo && gauge.geo && plan.geo, "apply_h: field without geometry");
  detail::need(&out != &in, "apply_h: out aliases in");
  detail::need(out.dr == in.dr && gauge.dr == in.dr, "apply_h: representation dimensions differ");
  detail::RankState& rs = detail::rank_state(w, *in.geo);
  const lbcu_gauge g = detail::device_gauge(rs, gauge);
  auto& wk = detail::work(rs, in.dr);
  detail::check(lbcu_spinor_upload(wk[0], detail::host(in)));
  detail::check(lbcu_h(wk[1], g, wk[0], mass));
  detail::check(lbcu_spinor_download(wk[1], detail::host(out)));
}

// The LinearOp make_h_operator returns: recognised by cg_solve, which then
// runs the fused D^dag D CG on the device instead of calling it back.
struct HOperator {
  const latbench::GaugeField* gauge;
  double mass;
  latbench::Worker* w;
  const latbench::ExchangePlan* plan;
  latbench::SpinorField* tmp;
  void operator()(latbench::SpinorField& out, latbench::SpinorField& in) const {
    latbench_b200::dropin::apply_h(out, *gauge, in, mass, *w, *plan, *tmp);  // qualified: no ADL
  }
};

// solver.hpp:36-37
inline latbench::LinearOp make_h_operator(const latbench::GaugeField& gauge, double mass, latbench::Worker& w,
                                          const latbench::ExchangePlan& plan, latbench::SpinorField& tmp) {
  return HOperator{&gauge, mass, &w, &plan, &tmp};
}

// solver.hpp:43-44 — the reference recurrence (x0 = 0, |r|/|b| < tol, true
// residual at exit, NonConvergence past max_iterations) on the device.
inline latbench::CgOutcome cg_solve(const latbench::LinearOp& op, const latbench::SpinorField& rhs,
                                    const latbench::CgSettings& settings, latbench::Worker& w,
                                    latbench::Clock& clock) {
  if (!(settings.tolerance > 0.0 && settings.tolerance < 1.0))
    throw latbench::ConfigError("cg tolerance must lie in (0, 1)");
  if (settings.max_iterations < 1) throw latbench::ConfigError("cg max iterations must be >= 1");
  detail::need(rhs.geo != nullptr, "cg_solve: rhs without geometry");
  const latbench::Geometry& geo = *rhs.geo;
  const int dr = rhs.dr;
  detail::RankState& rs = detail::rank_state(w, geo);
  latbench::CgOutcome out;
  out.solution = latbench::make_spinor(geo, dr);
  lbcu_spinor b = nullptr, x = nullptr;
  detail::check(lbcu_spinor_create(rs.ctx, dr, LBCU_FULL, &b));
  detail::check(lbcu_spinor_create(rs.ctx, dr, LBCU_FULL, &x));
  struct Fields {
    lbcu_spinor b, x;
    ~Fields() {
      lbcu_spinor_destroy(x);
      lbcu_spinor_destroy(b);
    }
  } own{b, x};
  std::vector<double> hist(static_cast<size_t>(settings.max_iterations) + 1);
  lbcu_cg_settings st{settings.tolerance, settings.max_iterations};
  lbcu_cg_outcome o{};

  w.barrier();
  const double t0 = w.rank() == 0 ? clock.seconds() : 0.0;
  detail::check(lbcu_spinor_upload(b, detail::host(rhs)));
  int rc;
  if (const HOperator* h = op.target<HOperator>()) {
    const lbcu_gauge g = detail::device_gauge(rs, *h->gauge);
    rc = lbcu_cg_solve_h(g, h->mass, b, x, &st, &o, hist.data());
  } else {
    // any other operator: called back on the host with the reference's fields
    struct Box {
      const latbench::LinearOp* op;
      latbench::SpinorField in, out;
    } box{&op, latbench::make_spinor(geo, dr), latbench::make_spinor(geo, dr)};
    auto tramp = [](void* user, lbcu_spinor dout, lbcu_spinor din) -> int {
      auto* bx = static_cast<Box*>(user);
      try {
        int r = lbcu_spinor_download(din, detail::host(bx->in));
        if (r != LBCU_OK) return r;
        (*bx->op)(bx->out, bx->in);
        return lbcu_spinor_upload(dout, detail::host(bx->out));
      } catch (const latbench::ContractViolation&) {
        return LBCU_CONTRACT_VIOLATION;
      } catch (const latbench::ConfigError&) {
        return LBCU_CONFIG_ERROR;
      } catch (const latbench::TransportError&) {
        return LBCU_TRANSPORT_ERROR;
      } catch (...) {
        return LBCU_CONTRACT_VIOLATION;
      }
    };
    rc = lbcu_cg_solve(rs.ctx, tramp, &box, b, x, &st, &o, hist.data());
  }
  if (rc == LBCU_NON_CONVERGENCE) throw latbench::NonConvergence(settings.max_iterations, o.best_residual);
  detail::check(rc);
  detail::check(lbcu_spinor_download(x, detail::host(out.solution)));
  out.iterations = o.iterations;
  out.rel_residual = o.rel_residual;
  out.true_rel_residual = o.true_rel_residual;
  out.residual_history.assign(hist.begin(), hist.begin() + o.iterations);
  w.barrier();
  const double dt = w.rank() == 0 ? clock.seconds() - t0 : 0.0;
  out.seconds = w.global_sum(dt);
  return out;
}

// solver.hpp:59-61 — invert H on rhs, pass iff the true residual < 2 tol.
inline latbench::ConsistencyResult consistency_check(const latbench::GaugeField& gauge,
                                                     const latbench::SpinorField& rhs, double mass,
                                                     const latbench::CgSettings& settings, latbench::Worker& w,
                                                     const latbench::ExchangePlan& plan, latbench::Clock& clock) {
  latbench::SpinorField tmp = latbench::make_spinor(*rhs.geo, rhs.dr);
  const latbench::CgOutcome cg = latbench_b200::dropin::cg_solve(
      latbench_b200::dropin::make_h_operator(gauge, mass, w, plan, tmp), rhs, settings, w, clock);
  latbench::ConsistencyResult res;
  res.iterations = cg.iterations;
  res.residual = cg.true_rel_residual;
  res.seconds = cg.seconds;
  res.status = cg.true_rel_residual < 2.0 * settings.tolerance ? latbench::ConsistencyResult::Status::Passed
                                                               : latbench::ConsistencyResult::Status::Failed;
  return res;
}

}  // namespace dropin
}  // namespace latbench_b200

// `latbench::gpu::apply_dirac(...)` etc.: the reference's namespace with the
// device versions of its hot calls beside the CPU ones.
namespace latbench {
namespace gpu {
using latbench_b200::dropin::apply_dirac;
using latbench_b200::dropin::apply_h;
using latbench_b200::dropin::cg_solve;
using latbench_b200::dropin::consistency_check;
using latbench_b200::dropin::invalidate;
using latbench_b200::dropin::make_h_operator;
using latbench_b200::dropin::release;
}  // namespace gpu
}  // namespace latbench
