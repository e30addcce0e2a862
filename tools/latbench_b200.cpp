// latbench_b200 — the benchmark driver (C++), run_suite / run_benchmark on B200.
//
// Restates the reference harness (proj/src/bench.cpp:14-321; CLI surface of
// SPEC.md:463) on the device path through include/latbench_b200.hpp:
//
//   latbench_b200 run   <params> [--format text|json|csv]
//   latbench_b200 check <params>          consistency check only
//   latbench_b200 model <params>          static model table, no GPU needed
//
// Parameter files are `key = value` lines with the reference's keys
// (bench.cpp:94-130: test, group_rank, representation, lattice, grid,
// spinor_fields, mass, kernel_seconds, consistency_check, cg_tolerance,
// cg_max_iterations, seed, enforce_local_floor, reference_*_flops) plus
// bc_time = periodic|antiperiodic, links = haar|near_unit, eo = true|false.
// A `test` key rebases on the preset (comms SU(2)A, balance SU(3)F, compute
// SU(6)F); unknown keys and bad values fail with the line number.
//
// Workers: like the reference's run_workers (transport.cpp:114-140), one host
// thread per grid rank; ranks share the visible GPUs round-robin and exchange
// halos through the in-process transport. Exit codes: 0 ok,
// 1 consistency check failed, 2 configuration error, 3 runtime failure.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <ctime>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "latbench_b200.hpp"

namespace lb = latbench_b200;

namespace {

struct ParseError : lb::ConfigError {
  ParseError(int line, const std::string& what)
      : lb::ConfigError("line " + std::to_string(line) + ": " + what) {}
};

struct Config {  // RegimeConfig, bench.hpp:20-44 (+ device-path keys)
  std::string test = "balance";
  int group_rank = 3;
  lb::Representation rep = lb::Representation::Fundamental;
  int spinor_fields = 6;
  double mass = 0.1;
  lb::Coord4 lattice{64, 32, 32, 32};
  lb::Coord4 grid{1, 1, 1, 1};
  double kernel_seconds = 60.0;
  bool consistency = true;
  lb::CgSettings cg;
  uint64_t seed = 4096;
  bool enforce_floor = true;
  std::optional<double> ref_sqnorm, ref_muladd, ref_dirac;
  lb::TimeBc bc = lb::TimeBc::Periodic;
  int links = LBCU_LINKS_HAAR;
  bool eo = false;

  int dr() const { return lb::rep_dim(rep, group_rank); }
  void validate() const {  // bench.cpp:14-24
    dr();
    if (spinor_fields < 2) throw lb::ConfigError("spinor_fields must be >= 2 to cycle field pairs");
    if (kernel_seconds <= 0.0) throw lb::ConfigError("kernel_seconds must be positive");
    if (!(cg.tolerance > 0.0 && cg.tolerance < 1.0)) throw lb::ConfigError("cg_tolerance must lie in (0, 1)");
    if (cg.max_iterations < 1) throw lb::ConfigError("cg_max_iterations must be >= 1");
    for (int d = 0; d < 4; ++d)
      if (lattice[d] <= 0 || grid[d] <= 0)
        throw lb::ConfigError("lattice extents and grid entries must be positive");
  }
};

Config preset(const std::string& name) {  // bench.cpp:26-42
  Config c;
  c.test = name;
  if (name == "comms") {
    c.group_rank = 2;
    c.rep = lb::Representation::Adjoint;
  } else if (name == "balance") {
    c.group_rank = 3;
    c.rep = lb::Representation::Fundamental;
  } else if (name == "compute") {
    c.group_rank = 6;
    c.rep = lb::Representation::Fundamental;
  } else {
    throw lb::ConfigError("unknown test '" + name + "' (expected comms, balance or compute)");
  }
  return c;
}

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r") - b + 1);
}
double pdouble(const std::string& v) {
  char* e = nullptr;
  const double x = std::strtod(v.c_str(), &e);
  if (e == v.c_str() || *e) throw lb::ConfigError("expected a number, got '" + v + "'");
  return x;
}
long long pint(const std::string& v) {
  char* e = nullptr;
  const long long x = std::strtoll(v.c_str(), &e, 10);
  if (e == v.c_str() || *e) throw lb::ConfigError("expected an integer, got '" + v + "'");
  return x;
}
bool pbool(const std::string& v) {
  if (v == "true" || v == "1" || v == "yes" || v == "on") return true;
  if (v == "false" || v == "0" || v == "no" || v == "off") return false;
  throw lb::ConfigError("expected a boolean, got '" + v + "'");
}
lb::Coord4 pcoord(const std::string& v) {
  lb::Coord4 c{};
  std::stringstream ss(v);
  std::string part;
  int i = 0;
  while (std::getline(ss, part, 'x')) {
    if (i >= 4) throw lb::ConfigError("expected TxXxYxZ, got '" + v + "'");
    c[i++] = static_cast<int>(pint(part));
  }
  if (i != 4) throw lb::ConfigError("expected TxXxYxZ, got '" + v + "'");
  return c;
}
lb::Representation prep(const std::string& v) {
  if (v == "fundamental") return lb::Representation::Fundamental;
  if (v == "adjoint") return lb::Representation::Adjoint;
  if (v == "symmetric") return lb::Representation::Symmetric;
  if (v == "antisymmetric") return lb::Representation::Antisymmetric;
  throw lb::ConfigError("unknown representation '" + v + "'");
}
const char* rep_name(lb::Representation r) {
  switch (r) {
    case lb::Representation::Fundamental: return "fundamental";
    case lb::Representation::Adjoint: return "adjoint";
    case lb::Representation::Symmetric: return "symmetric";
    case lb::Representation::Antisymmetric: return "antisymmetric";
  }
  return "?";
}

void set_key(Config& c, const std::string& k, const std::string& v) {  // bench.cpp:94-131
  if (k == "test") { preset(v); c.test = v; }
  else if (k == "group_rank") c.group_rank = static_cast<int>(pint(v));
  else if (k == "representation") c.rep = prep(v);
  else if (k == "lattice") c.lattice = pcoord(v);
  else if (k == "grid") c.grid = pcoord(v);
  else if (k == "spinor_fields") c.spinor_fields = static_cast<int>(pint(v));
  else if (k == "mass") c.mass = pdouble(v);
  else if (k == "kernel_seconds") c.kernel_seconds = pdouble(v);
  else if (k == "consistency_check") c.consistency = pbool(v);
  else if (k == "cg_tolerance") c.cg.tolerance = pdouble(v);
  else if (k == "cg_max_iterations") c.cg.max_iterations = static_cast<int>(pint(v));
  else if (k == "seed") c.seed = static_cast<uint64_t>(pint(v));
  else if (k == "enforce_local_floor") c.enforce_floor = pbool(v);
  else if (k == "reference_sqnorm_flops") c.ref_sqnorm = pdouble(v);
  else if (k == "reference_muladd_flops") c.ref_muladd = pdouble(v);
  else if (k == "reference_dirac_flops") c.ref_dirac = pdouble(v);
  else if (k == "bc_time") {
    if (v == "periodic") c.bc = lb::TimeBc::Periodic;
    else if (v == "antiperiodic") c.bc = lb::TimeBc::Antiperiodic;
    else throw lb::ConfigError("bc_time must be periodic or antiperiodic, got '" + v + "'");
  } else if (k == "links") {
    if (v == "haar") c.links = LBCU_LINKS_HAAR;
    else if (v == "near_unit") c.links = LBCU_LINKS_NEAR_UNIT;
    else if (v == "unit") c.links = LBCU_LINKS_UNIT;
    else throw lb::ConfigError("links must be haar, near_unit or unit, got '" + v + "'");
  } else if (k == "eo") c.eo = pbool(v);
  else throw lb::ConfigError("unknown key '" + k + "'");
}

Config parse_file(const std::string& path) {  // parse_params + apply_overrides
  std::ifstream in(path);
  if (!in) throw lb::ConfigError("cannot open parameter file '" + path + "'");
  std::vector<std::tuple<int, std::string, std::string>> ov;
  std::string raw;
  int line = 0;
  Config scratch;
  while (std::getline(in, raw)) {
    ++line;
    const std::string s = trim(raw);
    if (s.empty() || s[0] == '#') continue;
    const auto eq = s.find('=');
    if (eq == std::string::npos) throw ParseError(line, "expected 'key = value' in '" + s + "'");
    const std::string k = trim(s.substr(0, eq)), v = trim(s.substr(eq + 1));
    if (k.empty()) throw ParseError(line, "missing key before '='");
    try {
      set_key(scratch, k, v);
    } catch (const ParseError&) {
      throw;
    } catch (const lb::ConfigError& e) {
      throw ParseError(line, e.what());
    }
    ov.emplace_back(line, k, v);
  }
  Config c;
  for (auto& [l, k, v] : ov)
    if (k == "test") c = preset(v);
  for (auto& [l, k, v] : ov)
    if (k != "test") set_key(c, k, v);
  c.validate();
  return c;
}

struct KernelResult {
  std::string kernel;
  unsigned long long iterations = 0, flops = 0;
  double seconds = 0, flops_per_sec = 0, flops_per_sec_per_worker = 0;
  bool short_run = false;
  std::optional<double> ratio;
};

struct Model {
  long long sq = 0, ma = 0, di = 0;
  unsigned long long halo = 0;
  double intensity = 0;
};

struct Report {
  Config cfg;
  lb::Coord4 local{};
  int workers = 1;
  std::string timestamp;
  std::vector<KernelResult> kernels;
  lb::ConsistencyResult cons;
  Model model;
  bool eo_consistency = false;
};

double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

Model model_summary(const Config& c) {  // bench.cpp:252-266
  Model m;
  const int dr = c.dr();
  const bool real = lb::rep_is_real(c.rep);
  m.sq = lb::flops_per_site(LBCU_KERNEL_SQNORM, dr, real);
  m.ma = lb::flops_per_site(LBCU_KERNEL_MULADD, dr, real);
  m.di = lb::flops_per_site(LBCU_KERNEL_DIRAC, dr, real);
  int local[4];
  lb::check(lbcu_check_geometry(c.lattice.data(), c.grid.data(), 0, c.enforce_floor ? 1 : 0, local));
  const long long interior = 1LL * local[0] * local[1] * local[2] * local[3];
  // reference halo bytes: every face, full spinors (transport.hpp:124)
  long long boundary = 0;
  for (int d = 0; d < 4; ++d) boundary += 2 * interior / local[d];
  m.halo = static_cast<unsigned long long>(boundary) * 4 * dr * 16;
  m.intensity = static_cast<double>(m.di) * interior / static_cast<double>(m.halo);
  return m;
}

// run_suite on one worker thread (bench.cpp:268-311)
void run_suite(const Config& cfg, int rank, std::shared_ptr<lb::WorkerGroup> group, int ndev,
               Report* out) {
  lb::Worker w(cfg.lattice, cfg.grid, rank, rank % std::max(1, ndev), group, cfg.enforce_floor);
  const int dr = cfg.dr();
  lb::GaugeField gauge = lb::init_gauge_random(w, cfg.lattice, cfg.grid, cfg.group_rank, cfg.rep,
                                               cfg.seed, cfg.bc, cfg.links, 0.3);
  std::vector<lb::SpinorField> fields;
  for (int i = 0; i < cfg.spinor_fields; ++i)
    fields.push_back(lb::init_spinor_random(w, cfg.lattice, cfg.grid, dr, cfg.seed, i));

  lb::ConsistencyResult cons;
  if (cfg.consistency) {
    if (cfg.eo) {
      lb::SpinorField even(w, dr, lb::Subset::Even);
      std::vector<double> host = fields[0].download();
      even.upload(host.data());
      const lb::CgOutcome o = lb::cg_solve_eo(gauge, cfg.mass, even, cfg.cg);
      cons.iterations = o.iterations;
      cons.residual = o.true_rel_residual;
      cons.seconds = o.seconds;
      cons.status = o.true_rel_residual < 2.0 * cfg.cg.tolerance ? lb::ConsistencyResult::Status::Passed
                                                                 : lb::ConsistencyResult::Status::Failed;
    } else {
      cons = lb::consistency_check(gauge, fields[0], cfg.mass, cfg.cg);
    }
    fields[0] = lb::init_spinor_random(w, cfg.lattice, cfg.grid, dr, cfg.seed, cfg.spinor_fields);
  }

  const size_t nf = fields.size();
  const std::complex<double> cmul(0.3, 0.7);
  const long long V = 1LL * cfg.lattice[0] * cfg.lattice[1] * cfg.lattice[2] * cfg.lattice[3];
  const int workers = cfg.grid[0] * cfg.grid[1] * cfg.grid[2] * cfg.grid[3];
  std::vector<KernelResult> res;
  for (int kind = 0; kind < 3; ++kind) {  // run_kernel_benchmark, bench.cpp:190-248
    unsigned long long total = 0, cursor = 0, batch = 1;
    w.barrier();
    const double t0 = now();
    double wall = 0;
    for (;;) {
      for (unsigned long long i = 0; i < batch; ++i, ++cursor) {
        lb::SpinorField& a = fields[cursor % nf];
        lb::SpinorField& b = fields[(cursor + 1) % nf];
        if (kind == 0) (void)lb::sqnorm(a);
        else if (kind == 1) lb::mul_add(b, cmul, a);
        else lb::apply_dirac(b, gauge, a, cfg.mass);
      }
      total += batch;
      w.barrier();  // synchronizes the device stream, then the ranks
      // only rank 0 reads the clock; its decision and time are summed over
      // ranks so every worker agrees on the batch count (bench.cpp:215-226)
      double shared[2] = {0.0, 0.0};
      if (rank == 0) {
        shared[0] = now() - t0;
        shared[1] = shared[0] >= cfg.kernel_seconds ? 1.0 : 0.0;
      }
      lb::check(lbcu_allreduce_sum(w.handle(), shared, 2));
      if (shared[1] > 0.5) {
        wall = shared[0];
        break;
      }
      batch *= 2;
    }
    KernelResult r;
    r.kernel = kind == 0 ? "sqnorm" : kind == 1 ? "muladd" : "dirac";
    r.iterations = total;
    r.seconds = wall;
    r.short_run = total == 1;
    const long long per_site = lb::flops_per_site(kind, dr, lb::rep_is_real(cfg.rep));
    r.flops = static_cast<unsigned long long>(per_site) * V * total;
    r.flops_per_sec = r.flops / std::max(wall, 1e-12);
    r.flops_per_sec_per_worker = r.flops_per_sec / workers;
    const std::optional<double> ref = kind == 0 ? cfg.ref_sqnorm : kind == 1 ? cfg.ref_muladd : cfg.ref_dirac;
    if (ref) r.ratio = r.flops_per_sec / *ref;
    res.push_back(r);
  }
  if (rank != 0) return;
  out->cfg = cfg;
  out->local = w.local();
  out->workers = workers;
  out->kernels = res;
  out->cons = cons;
  out->eo_consistency = cfg.eo;
  out->model = model_summary(cfg);
  const std::time_t t = std::time(nullptr);
  std::tm tm{};
  gmtime_r(&t, &tm);
  char buf[32];
  std::strftime(buf, sizeof(buf), "%Y-%m-%dT%H:%M:%SZ", &tm);
  out->timestamp = buf;
}

const char* status_name(lb::ConsistencyResult::Status s) {
  switch (s) {
    case lb::ConsistencyResult::Status::NotRun: return "not_run";
    case lb::ConsistencyResult::Status::Passed: return "passed";
    case lb::ConsistencyResult::Status::Failed: return "failed";
  }
  return "?";
}

std::string coord(const lb::Coord4& c) {
  char b[64];
  std::snprintf(b, sizeof(b), "%dx%dx%dx%d", c[0], c[1], c[2], c[3]);
  return b;
}

std::string jcoord(const lb::Coord4& c) {
  return "[" + std::to_string(c[0]) + ", " + std::to_string(c[1]) + ", " + std::to_string(c[2]) + ", " +
         std::to_string(c[3]) + "]";
}

std::string num(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

std::string format(const Report& r, const std::string& fmt) {  // report.cpp:95-180
  std::ostringstream os;
  char line[256];
  if (fmt == "csv") {
    os << "kernel,iterations,seconds,flops,flops_per_sec,flops_per_sec_per_worker\n";
    for (const auto& k : r.kernels) {
      std::snprintf(line, sizeof(line), "%s,%llu,%.9e,%llu,%.9e,%.9e\n", k.kernel.c_str(), k.iterations,
                    k.seconds, k.flops, k.flops_per_sec, k.flops_per_sec_per_worker);
      os << line;
    }
    return os.str();
  }
  if (fmt == "json") {
    os << "{\n  \"format_version\": 1,\n  \"regime\": \"" << r.cfg.test << "\",\n  \"timestamp\": \""
       << r.timestamp << "\",\n  \"geometry\": {\"lattice\": " << jcoord(r.cfg.lattice)
       << ", \"grid\": " << jcoord(r.cfg.grid) << ", \"local\": " << jcoord(r.local)
       << ", \"workers\": " << r.workers << "},\n  \"group_rank\": " << r.cfg.group_rank
       << ",\n  \"representation\": \"" << rep_name(r.cfg.rep) << "\",\n  \"mass\": " << num(r.cfg.mass)
       << ",\n  \"seed\": " << r.cfg.seed << ",\n  \"kernels\": [";
    for (size_t i = 0; i < r.kernels.size(); ++i) {
      const auto& k = r.kernels[i];
      os << (i ? ",\n" : "\n") << "    {\"kernel\": \"" << k.kernel << "\", \"iterations\": " << k.iterations
         << ", \"seconds\": " << num(k.seconds) << ", \"flops\": " << k.flops
         << ", \"flops_per_sec\": " << num(k.flops_per_sec)
         << ", \"flops_per_sec_per_worker\": " << num(k.flops_per_sec_per_worker)
         << ", \"short_run\": " << (k.short_run ? "true" : "false")
         << ", \"reference_ratio\": " << (k.ratio ? num(*k.ratio) : "null") << "}";
    }
    os << "\n  ],\n  \"consistency\": {\"status\": \"" << status_name(r.cons.status)
       << "\", \"iterations\": " << r.cons.iterations << ", \"residual\": " << num(r.cons.residual)
       << ", \"seconds\": " << num(r.cons.seconds) << ", \"solver\": \""
       << (r.eo_consistency ? "eo" : "plain") << "\"},\n  \"model\": {\"sqnorm_flops_per_site\": " << r.model.sq
       << ", \"muladd_flops_per_site\": " << r.model.ma << ", \"dirac_flops_per_site\": " << r.model.di
       << ", \"halo_bytes_per_exchange\": " << r.model.halo << ", \"dirac_intensity\": " << num(r.model.intensity)
       << "},\n  \"device\": \"B200 (sm_100a), latbench-b200\"\n}\n";
    return os.str();
  }
  os << "latbench-b200 report (format 1)\n";
  os << "  regime         " << r.cfg.test << "  [SU(" << r.cfg.group_rank << "), " << rep_name(r.cfg.rep) << "]\n";
  os << "  lattice        " << coord(r.cfg.lattice) << "  grid " << coord(r.cfg.grid) << "  local "
     << coord(r.local) << "  workers " << r.workers << "\n";
  os << "  mass           " << r.cfg.mass << "\n  seed           " << r.cfg.seed << "\n";
  os << "  timestamp      " << r.timestamp << "\n  consistency    " << status_name(r.cons.status);
  if (r.cons.status != lb::ConsistencyResult::Status::NotRun) {
    std::snprintf(line, sizeof(line), " (%s CG, %ld iterations, residual %.3e, %.3f s)",
                  r.eo_consistency ? "eo" : "plain", r.cons.iterations, r.cons.residual, r.cons.seconds);
    os << line;
  }
  os << "\n\n";
  std::snprintf(line, sizeof(line), "  %-8s %12s %12s %16s %14s %14s %10s\n", "kernel", "iterations", "seconds",
                "FLOP", "FLOP/s", "FLOP/s/worker", "vs ref");
  os << line;
  for (const auto& k : r.kernels) {
    std::string ref = "-";
    if (k.ratio) {
      std::snprintf(line, sizeof(line), "%.3f", *k.ratio);
      ref = line;
    }
    std::snprintf(line, sizeof(line), "  %-8s %12llu %12.4f %16llu %14.5e %14.5e %10s%s\n", k.kernel.c_str(),
                  k.iterations, k.seconds, k.flops, k.flops_per_sec, k.flops_per_sec_per_worker, ref.c_str(),
                  k.short_run ? "  (short run)" : "");
    os << line;
  }
  std::snprintf(line, sizeof(line),
                "\n  the dirac line is the headline figure for machine comparisons\n"
                "  model: dirac %lld flop/site, halo %llu B/exchange/worker, intensity %.3f flop/B\n",
                r.model.di, r.model.halo, r.model.intensity);
  os << line;
  return os.str();
}

int usage() {
  std::cerr << "usage: latbench_b200 run|check|model <params> [--format text|json|csv]\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) return usage();
  const std::string cmd = argv[1], path = argv[2];
  std::string fmt = "text", all_prefix;
  for (int i = 3; i + 1 < argc; ++i) {
    if (std::string(argv[i]) == "--format") fmt = argv[i + 1];
    if (std::string(argv[i]) == "--emit-all") all_prefix = argv[i + 1];  // <prefix>.{txt,json,csv}
  }
  try {
    Config cfg = parse_file(path);
    if (cmd == "model") {
      const Model m = model_summary(cfg);
      std::printf("regime %s SU(%d) %s dr=%d\n  sqnorm %lld flop/site\n  muladd %lld flop/site\n"
                  "  dirac  %lld flop/site\n  halo   %llu B/exchange/worker\n  intensity %.4f flop/B\n",
                  cfg.test.c_str(), cfg.group_rank, rep_name(cfg.rep), cfg.dr(), m.sq, m.ma, m.di, m.halo,
                  m.intensity);
      return 0;
    }
    if (cmd != "run" && cmd != "check") return usage();
    if (cmd == "check") cfg.consistency = true;
    const int ndev = lbcu_device_count();
    if (ndev < 1) throw lb::CudaError("no CUDA device visible");
    const int workers = cfg.grid[0] * cfg.grid[1] * cfg.grid[2] * cfg.grid[3];
    Report rep;
    if (cmd == "check") cfg.kernel_seconds = 1e-9;  // one batch each
    if (workers == 1) {
      run_suite(cfg, 0, nullptr, ndev, &rep);
    } else {  // run_workers: one thread per rank
      auto group = lb::WorkerGroup::threads(workers);
      std::vector<std::thread> th;
      std::vector<std::exception_ptr> errs(workers);
      for (int r = 0; r < workers; ++r)
        th.emplace_back([&, r] {
          try {
            run_suite(cfg, r, group, ndev, &rep);
          } catch (...) {
            errs[r] = std::current_exception();
          }
        });
      for (auto& t : th) t.join();
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    }
    if (cmd == "check") {
      std::printf("consistency %s: %s CG, %ld iterations, true residual %.3e\n", status_name(rep.cons.status),
                  cfg.eo ? "eo" : "plain", rep.cons.iterations, rep.cons.residual);
    } else {
      std::cout << format(rep, fmt);
      for (const char* f : {"text", "json", "csv"}) {  // one report, every format
        if (all_prefix.empty()) break;
        const std::string ext = std::string(f) == "text" ? "txt" : f;
        std::ofstream(all_prefix + "." + ext) << format(rep, f);
      }
    }
    return rep.cons.status == lb::ConsistencyResult::Status::Failed ? 1 : 0;
  } catch (const lb::ConfigError& e) {
    std::cerr << "configuration error: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  }
}
