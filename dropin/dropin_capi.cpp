// dropin_capi.cpp — TEST ENTRY POINTS for the compiled drop-in.
//
// tests/test_gpu_dropin.py drives the drop-in (gw_b200.cpp) through the
// reference's own C++ types and exceptions: these extern "C" wrappers build
// gw::DistanceMatrix / ProbabilityVector / SolverConfig / SolveOptions from
// plain buffers (the reference's validating constructors, types.cpp), call
// the gw:: entry point exactly as a reference caller would, and report the
// SolveReport fields or the exception's class name and what().  Nothing here
// is part of the product.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "gw/solvers.hpp"
#include "gw/types.hpp"

namespace {

struct Outcome {
  char kind[48];       // exception class name, "" on success
  char message[512];   // what()
  char solver[16];     // NumericalInstabilityError::solver()
  int32_t iteration;   // NumericalInstabilityError::iteration()
  int32_t axis;        // ZeroSumLineError::axis() (0 rows, 1 cols)
  int64_t index;       // ZeroSumLineError::index()
};

void set(Outcome* o, const char* kind, const char* what) {
  std::snprintf(o->kind, sizeof(o->kind), "%s", kind);
  std::snprintf(o->message, sizeof(o->message), "%s", what);
}

template <class F>
int32_t guarded(Outcome* o, F&& f) {
  std::memset(o, 0, sizeof(*o));
  try {
    f();
    return 0;
  } catch (const gw::NumericalInstabilityError& e) {
    set(o, "NumericalInstabilityError", e.what());
    std::snprintf(o->solver, sizeof(o->solver), "%s", e.solver().c_str());
    o->iteration = e.iteration();
  } catch (const gw::ZeroSumLineError& e) {
    set(o, "ZeroSumLineError", e.what());
    o->axis = e.axis() == gw::Axis::Rows ? 0 : 1;
    o->index = e.index();
  } catch (const gw::ConfigError& e) {
    set(o, "ConfigError", e.what());
  } catch (const gw::DimensionMismatchError& e) {
    set(o, "DimensionMismatchError", e.what());
  } catch (const std::domain_error& e) {
    set(o, "domain_error", e.what());
  } catch (const std::invalid_argument& e) {
    set(o, "invalid_argument", e.what());
  } catch (const std::runtime_error& e) {
    set(o, "runtime_error", e.what());
  } catch (const std::exception& e) {
    set(o, "exception", e.what());
  }
  return 1;
}

gw::Matrix mat(const double* p, int64_t r, int64_t c) {
  gw::Matrix m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

gw::Vector vec(const double* p, int64_t n) {
  gw::Vector v(n);
  std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
  return v;
}

// SolverConfig from a flat array in field order (types.hpp:132-147).
gw::SolverConfig config(const double* f) {
  gw::SolverConfig c;
  c.algorithm = static_cast<gw::Algorithm>(static_cast<int>(f[0]));
  c.geometry = static_cast<gw::Geometry>(static_cast<int>(f[1]));
  c.rho = f[2];
  c.step = f[3];
  c.epsilon_reg = f[4];
  c.inner_iters = static_cast<int>(f[5]);
  c.inner_tol = f[6];
  c.rel_tol = f[7];
  c.max_iters = static_cast<int>(f[8]);
  c.perturbation = f[9];
  c.switch_iters = static_cast<int>(f[10]);
  c.seed = static_cast<int64_t>(f[11]);
  c.log_domain = f[12] != 0.0;
  c.record_residual = f[13] != 0.0;
  return c;
}

}  // namespace

extern "C" {

// entry: 0 solve, 1 bapg_solve, 2 bpg_solve, 3 ebpg_solve, 4 hbpg_solve.
// trace rows: iter, objective, infeasibility, split_gap, rel_change, phase,
// residual (NaN if absent).  obs_iters / obs_mass (cap obs_cap) record the
// observer calls: iteration number and Σπ (+ Σw·1e3 when w is passed).
__attribute__((visibility("default"))) int32_t gwdi_solve(
    int32_t entry, const double* cfg, const double* dx, int64_t n, const double* dy, int64_t m,
    const double* mu, int64_t mu_len, const double* nu, int64_t nu_len, const double* initial,
    int64_t init_rows, int64_t init_cols, int32_t use_observer, int32_t* obs_iters,
    double* obs_mass, int32_t obs_cap, int32_t* obs_count, double* out_final, double* out_pi,
    double* out_w, double* trace, int32_t trace_cap, int32_t* n_records, int32_t* converged,
    int32_t* iterations_used, Outcome* out) {
  *obs_count = 0;
  return guarded(out, [&] {
    const gw::DistanceMatrix d_x(mat(dx, n, n));
    const gw::DistanceMatrix d_y(mat(dy, m, m));
    const gw::ProbabilityVector p_mu(vec(mu, mu_len));
    const gw::ProbabilityVector p_nu(vec(nu, nu_len));
    gw::SolveOptions opts;
    if (initial) opts.initial = mat(initial, init_rows, init_cols);
    if (use_observer)
      opts.observer = [&](int it, const gw::Matrix& pi, const gw::Matrix* w) {
        if (*obs_count < obs_cap) {
          obs_iters[*obs_count] = it;
          obs_mass[*obs_count] = pi.sum() + (w ? 1e3 * w->sum() : 0.0);
        }
        ++*obs_count;
      };
    const gw::SolverConfig c = config(cfg);
    gw::SolveReport r = [&] {
      switch (entry) {
        case 1: return gw::bapg_solve(d_x, d_y, p_mu, p_nu, c, opts);
        case 2: return gw::bpg_solve(d_x, d_y, p_mu, p_nu, c, opts);
        case 3: return gw::ebpg_solve(d_x, d_y, p_mu, p_nu, c, opts);
        case 4: return gw::hbpg_solve(d_x, d_y, p_mu, p_nu, c, opts);
        default: return gw::solve(d_x, d_y, p_mu, p_nu, c, opts);
      }
    }();
    const gw::Matrix& f = r.final_coupling.entries();
    std::memcpy(out_final, f.data(), sizeof(double) * static_cast<size_t>(f.size()));
    if (out_pi && r.pi_half)
      std::memcpy(out_pi, r.pi_half->entries().data(), sizeof(double) * static_cast<size_t>(f.size()));
    if (out_w && r.w_half)
      std::memcpy(out_w, r.w_half->entries().data(), sizeof(double) * static_cast<size_t>(f.size()));
    const int32_t cnt = static_cast<int32_t>(r.trace.size());
    if (cnt > trace_cap) throw std::runtime_error("trace capacity exceeded");
    for (int32_t k = 0; k < cnt; ++k) {
      const gw::IterationRecord& t = r.trace[static_cast<size_t>(k)];
      double* row = trace + 7 * k;
      row[0] = t.iter;
      row[1] = t.objective;
      row[2] = t.marginal_infeasibility;
      row[3] = t.split_gap;
      row[4] = t.rel_change;
      row[5] = t.phase;
      row[6] = t.residual ? *t.residual : __builtin_nan("");
    }
    *n_records = cnt;
    *converged = r.converged ? 1 : 0;
    *iterations_used = r.iterations_used;
  });
}

__attribute__((visibility("default"))) int32_t gwdi_gw_objective(
    const double* dx, int64_t n, const double* dy, int64_t m, const double* pi, int64_t rows,
    int64_t cols, double* out_value, Outcome* out) {
  return guarded(out, [&] {
    *out_value = gw::gw_objective(gw::DistanceMatrix(mat(dx, n, n)),
                                  gw::DistanceMatrix(mat(dy, m, m)), mat(pi, rows, cols));
  });
}

__attribute__((visibility("default"))) int32_t gwdi_product_coupling(
    const double* mu, int64_t n, const double* nu, int64_t m, double* out_pi, Outcome* out) {
  return guarded(out, [&] {
    const gw::Coupling c =
        gw::product_coupling(gw::ProbabilityVector(vec(mu, n)), gw::ProbabilityVector(vec(nu, m)));
    std::memcpy(out_pi, c.entries().data(), sizeof(double) * static_cast<size_t>(n * m));
  });
}

__attribute__((visibility("default"))) int32_t gwdi_lipschitz_bound(
    const double* dx, int64_t n, const double* dy, int64_t m, double* out_value, Outcome* out) {
  return guarded(out, [&] {
    *out_value = gw::lipschitz_bound(gw::DistanceMatrix(mat(dx, n, n)),
                                     gw::DistanceMatrix(mat(dy, m, m)));
  });
}

}  // extern "C"
