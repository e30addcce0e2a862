// Exercises the C++ mirror of the reference API (include/latbench_b200.hpp)
// the way a latbench caller would: keyed fields, apply_dirac, apply_h,
// cg_solve with a LinearOp, the fused solvers and consistency_check.
// Prints one JSON line; tests/test_cpp_api.py checks it.
#include <cmath>
#include <cstdio>

#include "latbench_b200.hpp"

namespace lb = latbench_b200;

int main() {
  const lb::Coord4 L{8, 4, 4, 4}, grid{1, 1, 1, 1};
  lb::Worker w(L, grid);
  const double m = 0.1;
  lb::GaugeField U = lb::init_gauge_random(w, L, grid, 3, lb::Representation::Fundamental, 1);
  lb::SpinorField b = lb::init_spinor_random(w, L, grid, 3, 1, 0);
  lb::SpinorField Db(w, 3), Hb(w, 3), tmp(w, 3);

  lb::apply_dirac(Db, U, b, m);
  const double nD = lb::sqnorm(Db);
  lb::apply_h(Hb, U, b, m);
  // <b, H b> = |D b|^2 (H = D^dag D)
  const std::complex<double> bHb = lb::dot(b, Hb);

  lb::CgSettings st{1e-10, 1000};
  lb::LinearOp op = [&](lb::SpinorField& out, lb::SpinorField& in) {  // solver.cpp:9-15
    lb::apply_dirac(tmp, U, in, m);
    lb::apply_gamma5(tmp);
    lb::apply_dirac(out, U, tmp, m);
    lb::apply_gamma5(out);
  };
  const lb::CgOutcome o = lb::cg_solve(op, b, st);
  const lb::CgOutcome f = lb::cg_solve_h(U, m, b, st);
  lb::SpinorField be(w, 3, lb::Subset::Even);
  std::vector<double> host = b.download();
  be.upload(host.data());
  const lb::CgOutcome e = lb::cg_solve_eo(U, m, be, st);
  const lb::ConsistencyResult c = lb::consistency_check(U, b, m, st);

  bool nonconv = false;
  try {
    lb::cg_solve_h(U, m, b, lb::CgSettings{1e-12, 2});
  } catch (const lb::NonConvergence& ex) {
    nonconv = ex.iterations() == 2 && ex.best_residual() < 1.0;
  }
  bool contract = false;
  try {
    lb::apply_dirac(Db, U, Db, m);  // output aliases input
  } catch (const lb::ContractViolation&) {
    contract = true;
  }
  std::printf(
      "{\"sqnorm_Db\": %.17g, \"bHb_re\": %.17g, \"bHb_im\": %.17g, \"cg_iters\": %ld, "
      "\"cg_true\": %.3e, \"cg_h_iters\": %ld, \"cg_eo_iters\": %ld, \"cg_eo_true\": %.3e, "
      "\"consistency\": %d, \"nonconvergence\": %d, \"contract\": %d, \"history\": %zu}\n",
      nD, bHb.real(), bHb.imag(), o.iterations, o.true_rel_residual, f.iterations, e.iterations,
      e.true_rel_residual, c.status == lb::ConsistencyResult::Status::Passed ? 1 : 0, nonconv ? 1 : 0,
      contract ? 1 : 0, o.residual_history.size());
  return 0;
}
