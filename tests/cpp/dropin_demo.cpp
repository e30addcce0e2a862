// A reference (latbench) caller, written against the reference's own headers
// and types, that swaps its hot calls for the device ones
// (include/latbench_b200_dropin.hpp) and checks them against the CPU calls on
// the same fields, on a multi-worker grid run by the reference's run_workers.
// Prints one JSON line from rank 0; tests/test_cpp_api.py checks it.
//
//   usage: dropin_demo T X Y Z gT gX gY gZ N rep mass
#include <latbench/fields.hpp>
#include <latbench/geometry.hpp>
#include <latbench/kernels.hpp>
#include <latbench/solver.hpp>
#include <latbench/transport.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "latbench_b200_dropin.hpp"

using namespace latbench;

namespace {

// relative L2 distance of two fields over the interior, summed over workers
double rel_diff(const SpinorField& a, const SpinorField& b, Worker& w) {
  double d = 0.0, n = 0.0;
  const size_t nv = static_cast<size_t>(a.geo->interior) * a.vals_per_site();
  for (size_t i = 0; i < nv; ++i) {
    d += std::norm(a.data[i] - b.data[i]);
    n += std::norm(b.data[i]);
  }
  return std::sqrt(w.global_sum(d) / w.global_sum(n));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 12) {
    std::fprintf(stderr, "usage: dropin_demo T X Y Z gT gX gY gZ N rep mass\n");
    return 2;
  }
  const Coord4 global{std::atoi(argv[1]), std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4])};
  const Coord4 grid{std::atoi(argv[5]), std::atoi(argv[6]), std::atoi(argv[7]), std::atoi(argv[8])};
  const int n = std::atoi(argv[9]);
  const auto rep = static_cast<Representation>(std::atoi(argv[10]));
  const double mass = std::atof(argv[11]);
  std::string json;
  run_workers(grid, [&](Worker& w) {
    const Geometry geo = build_geometry(global, grid, w.rank(), false);
    const ExchangePlan plan = build_exchange_plan(geo);
    GaugeField g = init_gauge_random(w, plan, geo, n, rep, 1);
    const int dr = g.dr;
    SpinorField a = init_spinor_random(geo, dr, 1, 0);
    SpinorField cpu = make_spinor(geo, dr), dev = make_spinor(geo, dr), tmp = make_spinor(geo, dr);

    // kernels.hpp:19-20
    latbench::apply_dirac(cpu, g, a, mass, w, plan);
    latbench::gpu::apply_dirac(dev, g, a, mass, w, plan);
    const double e_dirac = rel_diff(dev, cpu, w);
    // solver.hpp:32-33
    latbench::apply_h(cpu, g, a, mass, w, plan, tmp);
    latbench::gpu::apply_h(dev, g, a, mass, w, plan, tmp);
    const double e_h = rel_diff(dev, cpu, w);

    // solver.hpp:43-44 with the reference's make_h_operator and the device one
    CgSettings st;
    st.tolerance = 1e-10;
    st.max_iterations = 2000;
    SteadyClock clock;
    const CgOutcome ref = latbench::cg_solve(latbench::make_h_operator(g, mass, w, plan, tmp), a, st, w, clock);
    const CgOutcome fused =
        latbench::gpu::cg_solve(latbench::gpu::make_h_operator(g, mass, w, plan, tmp), a, st, w, clock);
    // any other LinearOp (here the reference's own CPU H) is called back per iteration
    const CgOutcome cb = latbench::gpu::cg_solve(latbench::make_h_operator(g, mass, w, plan, tmp), a, st, w, clock);
    const double e_x = rel_diff(fused.solution, ref.solution, w);
    const double e_xcb = rel_diff(cb.solution, ref.solution, w);
    const ConsistencyResult cc = latbench::gpu::consistency_check(g, a, mass, st, w, plan, clock);

    // the reference's exception types
    int nonconv = 0, config = 0;
    try {
      CgSettings few = st;
      few.max_iterations = 3;
      (void)latbench::gpu::cg_solve(latbench::gpu::make_h_operator(g, mass, w, plan, tmp), a, few, w, clock);
    } catch (const NonConvergence& e) {
      nonconv = e.iterations() == 3 && e.best_residual() > 0.0;
    }
    try {
      CgSettings bad = st;
      bad.tolerance = 2.0;
      (void)latbench::gpu::cg_solve(latbench::gpu::make_h_operator(g, mass, w, plan, tmp), a, bad, w, clock);
    } catch (const ConfigError&) {
      config = 1;
    }
    // links changed in place: invalidate() re-uploads them
    for (auto& c : g.cdata) c *= 0.5;
    for (auto& r : g.rdata) r *= 0.5;
    latbench::gpu::invalidate(g);
    latbench::apply_dirac(cpu, g, a, mass, w, plan);
    latbench::gpu::apply_dirac(dev, g, a, mass, w, plan);
    const double e_inval = rel_diff(dev, cpu, w);
    if (w.rank() == 0) {
      char buf[1024];
      std::snprintf(buf, sizeof(buf),
                    "{\"workers\": %d, \"dirac_rel\": %.3e, \"h_rel\": %.3e, \"cg_ref_iters\": %ld, "
                    "\"cg_dev_iters\": %ld, \"cg_cb_iters\": %ld, \"cg_dev_true\": %.3e, \"cg_cb_true\": %.3e, "
                    "\"x_rel\": %.3e, \"x_cb_rel\": %.3e, \"history\": %zu, \"consistency\": %d, "
                    "\"consistency_iters\": %ld, \"nonconvergence\": %d, \"config_error\": %d, "
                    "\"invalidate_rel\": %.3e}",
                    w.size(), e_dirac, e_h, ref.iterations, fused.iterations, cb.iterations,
                    fused.true_rel_residual, cb.true_rel_residual, e_x, e_xcb, fused.residual_history.size(),
                    cc.status == ConsistencyResult::Status::Passed, cc.iterations, nonconv, config, e_inval);
      json = buf;
    }
  });
  latbench::gpu::release();
  std::printf("%s\n", json.c_str());
  return 0;
}
