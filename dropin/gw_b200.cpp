// gw_b200.cpp — the drop-in: the reference's solver entry points
// (proj/include/gw/solvers.hpp:12-70, types.hpp:177-178) implemented on
// libgwb.so (include/gwb.h) for the B200 path.
//
// A maintainer compiles this file into gwtk next to the reference sources
// and drops the path functions it replaces:
//   * from proj/src/solvers.cpp: gw_objective, lipschitz_bound, bapg_solve,
//     bpg_solve, ebpg_solve, hbpg_solve, solve (fw_solve, gw_gradient,
//     bilinear_value and penalty_value stay — FW is outside the B200 path
//     and solve() still dispatches Algorithm::Fw to it);
//   * from proj/src/types.cpp:204-207: product_coupling.
// and links libgwb.so.  The same file is built here (dropin/Makefile)
// against the reference headers as they lie under /root/reference, with
// oracle/eigen_lite standing in for Eigen3, and tested through
// tests/test_gpu_dropin.py.
//
// Semantics kept from the reference:
//   * validation order require_algorithm -> validate -> validate_inputs ->
//     initial shape -> positivity (solvers.cpp:141-151), with the
//     reference's own validate / validate_inputs (types.cpp:176-202);
//   * exceptions: every gwb_status code is rethrown as the reference class
//     with the reference's message (types.hpp:27-59);
//   * SolveOptions::observer is called after every outer iteration with
//     the current iterate(s) (solvers.hpp:42-44; the library switches to its
//     host-synchronous slow path when an observer is set);
//   * the report: BAPG final = ½(π + w) with pi_half / w_half, the trace,
//     converged and iterations_used (solvers.cpp:214-215).
#include <algorithm>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gw/solvers.hpp"
#include "gw/types.hpp"
#include "gwb.h"

namespace gw {
namespace {

gwb_config to_abi(const SolverConfig& c) {
  gwb_config a;
  gwb_config_default(&a);
  a.algorithm = static_cast<int32_t>(c.algorithm);
  a.geometry = static_cast<int32_t>(c.geometry);
  a.rho = c.rho;
  a.step = c.step;
  a.epsilon_reg = c.epsilon_reg;
  a.inner_iters = c.inner_iters;
  a.inner_tol = c.inner_tol;
  a.rel_tol = c.rel_tol;
  a.max_iters = c.max_iters;
  a.perturbation = c.perturbation;
  a.switch_iters = c.switch_iters;
  a.seed = c.seed;
  a.log_domain = c.log_domain ? 1 : 0;
  a.record_residual = c.record_residual ? 1 : 0;
  return a;  // precision AUTO, warnings on: what a drop-in caller gets
}

// gwb_status -> the reference exception (types.hpp:27-59).
[[noreturn]] void rethrow(const gwb_status& st) {
  switch (st.code) {
    case GWB_ERR_CONFIG:
      throw ConfigError(st.message);
    case GWB_ERR_DIMENSION:
      throw DimensionMismatchError(st.message);
    case GWB_ERR_NUMERICAL: {
      // The message is already "numerical instability in <solver> at
      // iteration <k>: <detail>" (types.cpp:60-66); rebuild it from detail.
      const std::string msg = st.message;
      const std::string pre = std::string("numerical instability in ") + st.solver +
                              " at iteration " + std::to_string(st.iteration) + ": ";
      const std::string detail = msg.rfind(pre, 0) == 0 ? msg.substr(pre.size()) : msg;
      throw NumericalInstabilityError(st.solver, st.iteration, detail);
    }
    case GWB_ERR_ZERO_SUM:
      throw ZeroSumLineError(st.axis == GWB_ROWS ? Axis::Rows : Axis::Cols,
                             static_cast<Eigen::Index>(st.index));
    case GWB_ERR_INVALID:
      throw std::invalid_argument(st.message);
    case GWB_ERR_DOMAIN:
      throw std::domain_error(st.message);
    default:
      throw std::runtime_error(st.message);
  }
}

void check(const gwb_status& st) {
  if (st.code != GWB_OK) rethrow(st);
}

// require_algorithm (solvers.cpp:52-58), same message.
void require_algorithm(const SolverConfig& config, Algorithm expected, const char* who) {
  if (config.algorithm != expected)
    throw ConfigError(std::string(who) + " called with algorithm '" +
                      to_string(config.algorithm) + "'");
}

Matrix from_buffer(const double* p, Eigen::Index rows, Eigen::Index cols) {
  Matrix out(rows, cols);
  std::copy(p, p + rows * cols, out.data());
  return out;
}

struct ObserverCall {
  const SolveOptions* opts;
  std::exception_ptr error;
};

// gwb_observer -> SolveOptions::observer.  An exception thrown by the
// observer aborts the solve and is rethrown to the caller unchanged.
int32_t trampoline(void* user, int32_t iter, const double* pi, const double* w, int64_t n,
                   int64_t m) {
  auto* call = static_cast<ObserverCall*>(user);
  try {
    const Matrix p = from_buffer(pi, n, m);
    if (w) {
      const Matrix ww = from_buffer(w, n, m);
      call->opts->observer(iter, p, &ww);
    } else {
      call->opts->observer(iter, p, nullptr);
    }
    return 0;
  } catch (...) {
    call->error = std::current_exception();
    return 1;
  }
}

SolveReport call_solver(gwb_solve_fn fn, Algorithm expected, const char* who,
                        const DistanceMatrix& d_x, const DistanceMatrix& d_y,
                        const ProbabilityVector& mu, const ProbabilityVector& nu,
                        const SolverConfig& config, const SolveOptions& opts) {
  if (who) require_algorithm(config, expected, who);
  validate(config);
  validate_inputs(d_x, d_y, mu, nu);
  const Eigen::Index n = d_x.size(), m = d_y.size();
  if (opts.initial && (opts.initial->rows() != n || opts.initial->cols() != m))
    throw DimensionMismatchError("initial coupling shape mismatch");
  const gwb_config a = to_abi(config);
  const bool bapg = config.algorithm == Algorithm::Bapg;
  Matrix fin(n, m), pi, w;
  if (bapg) {
    pi.resize(n, m);
    w.resize(n, m);
  }
  std::vector<gwb_record> tr(static_cast<size_t>(std::max(1, config.max_iters)));
  int32_t nrec = 0, conv = 0, used = 0;
  gwb_status st;
  std::memset(&st, 0, sizeof(st));
  ObserverCall obs{&opts, nullptr};
  fn(&a, d_x.entries().data(), n, d_y.entries().data(), m, mu.weights().data(),
     nu.weights().data(), opts.initial ? opts.initial->data() : nullptr,
     opts.observer ? trampoline : nullptr, opts.observer ? &obs : nullptr, fin.data(),
     bapg ? pi.data() : nullptr, bapg ? w.data() : nullptr, tr.data(),
     static_cast<int32_t>(tr.size()), &nrec, &conv, &used, &st);
  if (obs.error) std::rethrow_exception(obs.error);
  check(st);
  std::vector<IterationRecord> trace;
  trace.reserve(static_cast<size_t>(nrec));
  for (int32_t k = 0; k < nrec; ++k) {
    const gwb_record& t = tr[static_cast<size_t>(k)];
    IterationRecord r;
    r.iter = t.iter;
    r.objective = t.objective;
    r.marginal_infeasibility = t.marginal_infeasibility;
    r.split_gap = t.split_gap;
    if (t.has_residual) r.residual = t.residual;
    r.rel_change = t.rel_change;
    r.elapsed_seconds = t.elapsed_seconds;
    r.phase = t.phase;
    trace.push_back(r);
  }
  SolveReport rep{Coupling(std::move(fin)), std::nullopt, std::nullopt, std::move(trace),
                  conv != 0, used};
  if (bapg) {
    rep.pi_half = Coupling(std::move(pi));
    rep.w_half = Coupling(std::move(w));
  }
  return rep;
}

}  // namespace

// solvers.hpp:12-13 / solvers.cpp:64-69.
double gw_objective(const DistanceMatrix& d_x, const DistanceMatrix& d_y, const Matrix& pi) {
  double out = 0.0;
  gwb_status st;
  gwb_gw_objective(d_x.entries().data(), d_x.size(), d_y.entries().data(), d_y.size(), pi.data(),
                   pi.rows(), pi.cols(), &out, &st);
  check(st);
  return out;
}

// solvers.hpp:37 / solvers.cpp:113-136.
double lipschitz_bound(const DistanceMatrix& d_x, const DistanceMatrix& d_y) {
  double out = 0.0;
  gwb_status st;
  gwb_lipschitz_bound(d_x.entries().data(), d_x.size(), d_y.entries().data(), d_y.size(), &out,
                      &st);
  check(st);
  return out;
}

// types.hpp:177-178 / types.cpp:204-207.
Coupling product_coupling(const ProbabilityVector& mu, const ProbabilityVector& nu) {
  Matrix out(mu.size(), nu.size());
  gwb_status st;
  gwb_product_coupling(mu.weights().data(), mu.size(), nu.weights().data(), nu.size(), out.data(),
                       &st);
  check(st);
  return Coupling(std::move(out));
}

// solvers.hpp:47-66 / solvers.cpp:138-426.
SolveReport bapg_solve(const DistanceMatrix& d_x, const DistanceMatrix& d_y,
                       const ProbabilityVector& mu, const ProbabilityVector& nu,
                       const SolverConfig& config, const SolveOptions& opts) {
  return call_solver(gwb_bapg_solve, Algorithm::Bapg, "bapg_solve", d_x, d_y, mu, nu, config,
                     opts);
}

SolveReport bpg_solve(const DistanceMatrix& d_x, const DistanceMatrix& d_y,
                      const ProbabilityVector& mu, const ProbabilityVector& nu,
                      const SolverConfig& config, const SolveOptions& opts) {
  return call_solver(gwb_bpg_solve, Algorithm::Bpg, "bpg_solve", d_x, d_y, mu, nu, config, opts);
}

SolveReport ebpg_solve(const DistanceMatrix& d_x, const DistanceMatrix& d_y,
                       const ProbabilityVector& mu, const ProbabilityVector& nu,
                       const SolverConfig& config, const SolveOptions& opts) {
  return call_solver(gwb_ebpg_solve, Algorithm::Ebpg, "ebpg_solve", d_x, d_y, mu, nu, config,
                     opts);
}

SolveReport hbpg_solve(const DistanceMatrix& d_x, const DistanceMatrix& d_y,
                       const ProbabilityVector& mu, const ProbabilityVector& nu,
                       const SolverConfig& config, const SolveOptions& opts) {
  return call_solver(gwb_hbpg_solve, Algorithm::Hbpg, "hbpg_solve", d_x, d_y, mu, nu, config,
                     opts);
}

// solvers.hpp:68-70 / solvers.cpp:499-515: FW stays in the reference's
// solvers.cpp (fw_solve); every other algorithm runs on the device.
SolveReport solve(const DistanceMatrix& d_x, const DistanceMatrix& d_y,
                  const ProbabilityVector& mu, const ProbabilityVector& nu,
                  const SolverConfig& config, const SolveOptions& opts) {
  switch (config.algorithm) {
    case Algorithm::Bapg:
      return bapg_solve(d_x, d_y, mu, nu, config, opts);
    case Algorithm::Bpg:
      return bpg_solve(d_x, d_y, mu, nu, config, opts);
    case Algorithm::Ebpg:
      return ebpg_solve(d_x, d_y, mu, nu, config, opts);
    case Algorithm::Hbpg:
      return hbpg_solve(d_x, d_y, mu, nu, config, opts);
    case Algorithm::Fw:
      return fw_solve(d_x, d_y, mu, nu, config, opts);
  }
  throw ConfigError("unknown algorithm");
}

}  // namespace gw
