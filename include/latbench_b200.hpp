// latbench_b200.hpp — header-only C++ mirror of the reference operator API
// (latbench, /root/reference/proj/include/latbench/{fields,kernels,solver}.hpp)
// over the C-ABI in lbcu.h. Callers of the reference keep their shape:
//
//   reference (latbench::)                      here (latbench_b200::)
//   GaugeField / init_gauge_random              GaugeField / init_gauge_random
//   SpinorField / init_spinor_random            SpinorField / init_spinor_random
//   apply_dirac(out, gauge, in, m, w, plan)     apply_dirac(out, gauge, in, m)
//   apply_h(out, gauge, in, m, w, plan, tmp)    apply_h(out, gauge, in, m)
//   LinearOp + cg_solve(op, rhs, settings, ..)  LinearOp + cg_solve(op, rhs, settings)
//   consistency_check(...)                      consistency_check(...)
//   errors.hpp exception classes                same names, thrown from status codes
//
// The Worker / ExchangePlan pair of the reference becomes a Worker holding a
// device context (geometry, exchange schedule, CUDA stream, transport).
// Fields live on the device; host data crosses only through upload/download
// in the reference's own interior layout.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbcu.h"

namespace latbench_b200 {

// ---- errors.hpp:9-63 --------------------------------------------------------
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class DecompositionError : public ConfigError {
 public:
  using ConfigError::ConfigError;
};
class ContractViolation : public Error {
 public:
  using Error::Error;
};
class TransportError : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};
class NonConvergence : public Error {
 public:
  NonConvergence(long iterations, double best, const std::string& what)
      : Error(what), iterations_(iterations), best_residual_(best) {}
  long iterations() const { return iterations_; }
  double best_residual() const { return best_residual_; }

 private:
  long iterations_;
  double best_residual_;
};

inline void check(int rc, long iters = 0, double best = 0.0) {
  if (rc == LBCU_OK) return;
  const std::string msg = lbcu_last_error();
  switch (rc) {
    case LBCU_CONTRACT_VIOLATION: throw ContractViolation(msg);
    case LBCU_CONFIG_ERROR:
      if (msg.find("divisible") != std::string::npos || msg.find("odd") != std::string::npos ||
          msg.find("floor") != std::string::npos || msg.find("even local") != std::string::npos)
        throw DecompositionError(msg);
      throw ConfigError(msg);
    case LBCU_TRANSPORT_ERROR: throw TransportError(msg);
    case LBCU_NON_CONVERGENCE: throw NonConvergence(iters, best, msg);
    default: throw CudaError(msg);
  }
}

using Coord4 = std::array<int, 4>;
enum class Representation { Fundamental = 0, Adjoint = 1, Symmetric = 2, Antisymmetric = 3 };
enum class Subset { Full = LBCU_FULL, Even = LBCU_EVEN, Odd = LBCU_ODD };
enum class TimeBc { Periodic = LBCU_BC_PERIODIC, Antiperiodic = LBCU_BC_ANTIPERIODIC_T };

inline int rep_dim(Representation rep, int n) {
  int dr = 0, real = 0;
  check(lbcu_rep_dim(static_cast<int>(rep), n, &dr, &real));
  return dr;
}
inline bool rep_is_real(Representation rep) { return rep == Representation::Adjoint; }

// ---- WorkerGroup (transport.hpp:24-67) ------------------------------------
class WorkerGroup {
 public:
  static std::shared_ptr<WorkerGroup> threads(int nranks) {
    lbcu_world w = nullptr;
    check(lbcu_world_threads(nranks, &w));
    return std::shared_ptr<WorkerGroup>(new WorkerGroup(w));
  }
  static std::shared_ptr<WorkerGroup> nccl(int nranks, int rank, const unsigned char id[128]) {
    lbcu_world w = nullptr;
    check(lbcu_world_nccl(nranks, rank, id, &w));
    return std::shared_ptr<WorkerGroup>(new WorkerGroup(w));
  }
  // one process per GPU on one node; halos stored by the pack kernel into the
  // neighbour's arena over NVLink (CUDA IPC). shm_name: "/..." unique per job;
  // nccl_id (nullable): NCCL for the CG sums.
  static std::shared_ptr<WorkerGroup> ipc(int nranks, int rank, const std::string& shm_name,
                                          const unsigned char* nccl_id = nullptr) {
    lbcu_world w = nullptr;
    check(lbcu_world_ipc(nranks, rank, shm_name.c_str(), nccl_id, &w));
    return std::shared_ptr<WorkerGroup>(new WorkerGroup(w));
  }
  // in-process ranks with the same direct halo protocol
  static std::shared_ptr<WorkerGroup> threads_direct(int nranks) {
    lbcu_world w = nullptr;
    check(lbcu_world_threads_direct(nranks, &w));
    return std::shared_ptr<WorkerGroup>(new WorkerGroup(w));
  }
  void set_direct(bool on) { check(lbcu_world_set_direct(w_, on ? 1 : 0)); }
  ~WorkerGroup() { lbcu_world_destroy(w_); }
  lbcu_world handle() const { return w_; }

 private:
  explicit WorkerGroup(lbcu_world w) : w_(w) {}
  lbcu_world w_;
};

// ---- Worker = rank + Geometry + ExchangePlan + stream ---------------------
class Worker {
 public:
  Worker(const Coord4& global, const Coord4& grid = {1, 1, 1, 1}, int rank = 0, int device = 0,
         std::shared_ptr<WorkerGroup> group = nullptr, bool enforce_floor = false)
      : group_(std::move(group)), rank_(rank) {
    check(lbcu_ctx_create(group_ ? group_->handle() : nullptr, rank, device, global.data(),
                          grid.data(), enforce_floor ? 1 : 0, &ctx_));
    check(lbcu_ctx_local(ctx_, local_.data()));
  }
  ~Worker() { lbcu_ctx_destroy(ctx_); }
  Worker(const Worker&) = delete;
  Worker& operator=(const Worker&) = delete;

  int rank() const { return rank_; }
  const Coord4& local() const { return local_; }
  long long interior() const {
    return static_cast<long long>(local_[0]) * local_[1] * local_[2] * local_[3];
  }
  void barrier() { check(lbcu_barrier(ctx_)); }
  void synchronize() { check(lbcu_ctx_synchronize(ctx_)); }
  lbcu_ctx handle() const { return ctx_; }

 private:
  std::shared_ptr<WorkerGroup> group_;
  int rank_;
  lbcu_ctx ctx_ = nullptr;
  Coord4 local_{};
};

// ---- fields (fields.hpp:15-57) ---------------------------------------------
class SpinorField {
 public:
  SpinorField() = default;
  SpinorField(Worker& w, int dr, Subset subset = Subset::Full) : w_(&w), dr_(dr), subset_(subset) {
    lbcu_spinor s = nullptr;
    check(lbcu_spinor_create(w.handle(), dr, static_cast<int>(subset), &s));
    h_ = std::shared_ptr<lbcu_spinor_s>(s, [](lbcu_spinor p) { lbcu_spinor_destroy(p); });
  }
  int dr() const { return dr_; }
  Subset subset() const { return subset_; }
  int vals_per_site() const { return 4 * dr_; }
  size_t host_doubles() const { return static_cast<size_t>(w_->interior()) * vals_per_site() * 2; }
  // reference interior layout: [site][spin][colour] complex<double>
  void upload(const double* host) { check(lbcu_spinor_upload(h_.get(), host)); }
  void download(double* host) const { check(lbcu_spinor_download(h_.get(), host)); }
  std::vector<double> download() const {
    std::vector<double> v(host_doubles());
    download(v.data());
    return v;
  }
  lbcu_spinor handle() const { return h_.get(); }
  Worker& worker() const { return *w_; }
  // non-owning view of a library-owned field (the work fields cg_solve hands
  // to a LinearOp)
  static SpinorField view(Worker& w, int dr, Subset subset, lbcu_spinor h) {
    SpinorField f;
    f.w_ = &w;
    f.dr_ = dr;
    f.subset_ = subset;
    f.h_ = std::shared_ptr<lbcu_spinor_s>(h, [](lbcu_spinor) {});
    return f;
  }

 private:
  Worker* w_ = nullptr;
  int dr_ = 0;
  Subset subset_ = Subset::Full;
  std::shared_ptr<lbcu_spinor_s> h_;
};

class GaugeField {
 public:
  GaugeField(Worker& w, int group_rank, Representation rep, TimeBc bc = TimeBc::Antiperiodic)
      : w_(&w), n_(group_rank), rep_(rep), dr_(rep_dim(rep, group_rank)) {
    lbcu_gauge g = nullptr;
    check(lbcu_gauge_create(w.handle(), group_rank, static_cast<int>(rep), static_cast<int>(bc), &g));
    h_ = std::shared_ptr<lbcu_gauge_s>(g, [](lbcu_gauge p) { lbcu_gauge_destroy(p); });
  }
  int dr() const { return dr_; }
  int group_rank() const { return n_; }
  Representation rep() const { return rep_; }
  bool real_links() const { return rep_is_real(rep_); }
  size_t host_doubles() const {
    return static_cast<size_t>(w_->interior()) * 4 * dr_ * dr_ * (real_links() ? 1 : 2);
  }
  void upload(const double* host) { check(lbcu_gauge_upload(h_.get(), host)); }
  void download(double* host) const { check(lbcu_gauge_download(h_.get(), host)); }
  lbcu_gauge handle() const { return h_.get(); }

 private:
  Worker* w_;
  int n_;
  Representation rep_;
  int dr_;
  std::shared_ptr<lbcu_gauge_s> h_;
};

// init_gauge_random (transport.cpp:223-229): keyed links on this worker's
// interior, uploaded; no halo exchange is needed on the device.
inline GaugeField init_gauge_random(Worker& w, const Coord4& global, const Coord4& grid,
                                    int group_rank, Representation rep, uint64_t seed,
                                    TimeBc bc = TimeBc::Antiperiodic, int links = LBCU_LINKS_HAAR,
                                    double eps = 0.3) {
  GaugeField g(w, group_rank, rep, bc);
  std::vector<double> host(g.host_doubles());
  check(lbcu_host_gauge_random(global.data(), grid.data(), w.rank(), group_rank,
                               static_cast<int>(rep), links, seed, eps, 0, host.data()));
  g.upload(host.data());
  return g;
}

// init_spinor_random (fields.cpp:22-40)
inline SpinorField init_spinor_random(Worker& w, const Coord4& global, const Coord4& grid, int dr,
                                      uint64_t seed, uint64_t field_index,
                                      Subset subset = Subset::Full) {
  SpinorField f(w, dr, subset);
  std::vector<double> host(static_cast<size_t>(w.interior()) * 4 * dr * 2);
  check(lbcu_host_spinor_random(global.data(), grid.data(), w.rank(), dr, seed, field_index,
                                host.data()));
  f.upload(host.data());
  return f;
}

// ---- kernels.hpp:11-44 -------------------------------------------------------
inline double sqnorm(const SpinorField& f) {
  double v = 0;
  check(lbcu_sqnorm(f.handle(), &v));
  return v;
}
inline void apply_dirac(SpinorField& out, const GaugeField& g, const SpinorField& in, double m) {
  check(lbcu_dphi(out.handle(), g.handle(), in.handle(), m));
}
inline void apply_g5dirac(SpinorField& out, const GaugeField& g, const SpinorField& in, double m) {
  check(lbcu_g5dphi(out.handle(), g.handle(), in.handle(), m));
}
inline void dphi_eo(SpinorField& out_e, const GaugeField& g, const SpinorField& in_o) {
  check(lbcu_dphi_eo(out_e.handle(), g.handle(), in_o.handle()));
}
inline void dphi_oe(SpinorField& out_o, const GaugeField& g, const SpinorField& in_e) {
  check(lbcu_dphi_oe(out_o.handle(), g.handle(), in_e.handle()));
}
inline void mhat(SpinorField& out_e, const GaugeField& g, const SpinorField& in_e, double m) {
  check(lbcu_mhat(out_e.handle(), g.handle(), in_e.handle(), m));
}
inline void apply_h(SpinorField& out, const GaugeField& g, const SpinorField& in, double m) {
  check(lbcu_h(out.handle(), g.handle(), in.handle(), m));
}
inline std::complex<double> dot(const SpinorField& a, const SpinorField& b) {
  double re = 0, im = 0;
  check(lbcu_dot(a.handle(), b.handle(), &re, &im));
  return {re, im};
}
inline void axpy(SpinorField& y, std::complex<double> a, const SpinorField& x) {
  check(lbcu_axpy(y.handle(), a.real(), a.imag(), x.handle()));
}
inline void mul_add(SpinorField& psi2, std::complex<double> c, const SpinorField& psi1) {
  check(lbcu_mul_add(psi2.handle(), c.real(), c.imag(), psi1.handle()));
}
inline void xpay(SpinorField& y, std::complex<double> a, const SpinorField& x) {
  check(lbcu_xpay(y.handle(), a.real(), a.imag(), x.handle()));
}
inline void copy_interior(SpinorField& dst, const SpinorField& src) {
  check(lbcu_copy(dst.handle(), src.handle()));
}
inline void zero_interior(SpinorField& f) { check(lbcu_zero(f.handle())); }
inline void apply_gamma5(SpinorField& f) { check(lbcu_gamma5(f.handle())); }

// ---- solver.hpp:13-61 ---------------------------------------------------------
struct CgSettings {
  double tolerance = 1e-7;
  int max_iterations = 10000;
};

struct CgOutcome {
  SpinorField solution;
  long iterations = 0;
  double rel_residual = 0.0;
  double true_rel_residual = 0.0;
  double seconds = 0.0;
  std::vector<double> residual_history;
};

// LinearOp, solver.hpp:28: out = A(in) on device fields.
using LinearOp = std::function<void(SpinorField& out, SpinorField& in)>;

inline CgOutcome finish_outcome(SpinorField x, const lbcu_cg_outcome& o, std::vector<double> hist) {
  CgOutcome r;
  r.solution = std::move(x);
  r.iterations = o.iterations;
  r.rel_residual = o.rel_residual;
  r.true_rel_residual = o.true_rel_residual;
  r.seconds = o.seconds;
  hist.resize(static_cast<size_t>(o.iterations));
  r.residual_history = std::move(hist);
  return r;
}

// cg_solve with the fused D^dag D operator (make_h_operator + cg_solve)
inline CgOutcome cg_solve_h(const GaugeField& g, double m, const SpinorField& rhs,
                            const CgSettings& st) {
  SpinorField x(rhs.worker(), rhs.dr(), rhs.subset());
  lbcu_cg_settings s{st.tolerance, st.max_iterations};
  lbcu_cg_outcome o{};
  std::vector<double> hist(static_cast<size_t>(st.max_iterations));
  const int rc = lbcu_cg_solve_h(g.handle(), m, rhs.handle(), x.handle(), &s, &o, hist.data());
  check(rc, o.iterations, o.best_residual);  // o is filled before the status is raised
  return finish_outcome(std::move(x), o, std::move(hist));
}

// even-odd preconditioned CG on Mhat^dag Mhat (EVEN fields)
inline CgOutcome cg_solve_eo(const GaugeField& g, double m, const SpinorField& rhs_even,
                             const CgSettings& st) {
  SpinorField x(rhs_even.worker(), rhs_even.dr(), rhs_even.subset());
  lbcu_cg_settings s{st.tolerance, st.max_iterations};
  lbcu_cg_outcome o{};
  std::vector<double> hist(static_cast<size_t>(st.max_iterations));
  const int rc = lbcu_cg_solve_eo(g.handle(), m, rhs_even.handle(), x.handle(), &s, &o, hist.data());
  check(rc, o.iterations, o.best_residual);
  return finish_outcome(std::move(x), o, std::move(hist));
}

// cg_solve(LinearOp, rhs, settings), solver.cpp:24-82. The operator receives
// views of library-owned work fields and must only call device operators.
inline CgOutcome cg_solve(const LinearOp& op, const SpinorField& rhs, const CgSettings& st) {
  SpinorField x(rhs.worker(), rhs.dr(), rhs.subset());
  lbcu_cg_settings s{st.tolerance, st.max_iterations};
  lbcu_cg_outcome o{};
  std::vector<double> hist(static_cast<size_t>(st.max_iterations));
  struct Box {
    const LinearOp* op;
    const SpinorField* rhs;
  } box{&op, &rhs};
  auto tramp = [](void* user, lbcu_spinor out, lbcu_spinor in) -> int {
    auto* b = static_cast<Box*>(user);
    try {
      Worker& w = b->rhs->worker();
      SpinorField vo = SpinorField::view(w, b->rhs->dr(), b->rhs->subset(), out);
      SpinorField vi = SpinorField::view(w, b->rhs->dr(), b->rhs->subset(), in);
      (*b->op)(vo, vi);
      return LBCU_OK;
    } catch (const CudaError&) {
      return LBCU_CUDA_ERROR;
    } catch (const Error&) {
      return LBCU_CONTRACT_VIOLATION;
    }
  };
  const int rc = lbcu_cg_solve(rhs.worker().handle(), tramp, &box, rhs.handle(), x.handle(), &s, &o,
                               hist.data());
  check(rc, o.iterations, o.best_residual);
  return finish_outcome(std::move(x), o, std::move(hist));
}

// make_h_operator (solver.cpp:17-22)
inline LinearOp make_h_operator(const GaugeField& g, double m) {
  return [&g, m](SpinorField& out, SpinorField& in) { apply_h(out, g, in, m); };
}

struct ConsistencyResult {
  enum class Status { NotRun, Passed, Failed } status = Status::NotRun;
  long iterations = 0;
  double residual = 0.0;
  double seconds = 0.0;
};

// consistency_check (solver.cpp:93-108): pass iff the true residual < 2 tol
inline ConsistencyResult consistency_check(const GaugeField& g, const SpinorField& rhs, double m,
                                           const CgSettings& st) {
  const CgOutcome cg = cg_solve_h(g, m, rhs, st);
  ConsistencyResult r;
  r.iterations = cg.iterations;
  r.residual = cg.true_rel_residual;
  r.seconds = cg.seconds;
  r.status = cg.true_rel_residual < 2.0 * st.tolerance ? ConsistencyResult::Status::Passed
                                                       : ConsistencyResult::Status::Failed;
  return r;
}

// flops_per_site (flops.hpp:44)
inline long long flops_per_site(int kernel, int dr, bool real_rep) {
  return lbcu_flops_per_site(kernel, dr, real_rep ? 1 : 0);
}

}  // namespace latbench_b200
