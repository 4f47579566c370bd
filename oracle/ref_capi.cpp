// ref_capi.cpp — extern "C" access to the reference's OWN solver code.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference translation units exactly as they lie under
// /root/reference/proj/src (types.cpp, projections.cpp, solvers.cpp,
// diagnostics.cpp, tasks.cpp), against oracle/eigen_lite, into
// oracle/_ref/libgwref.so.  Used to pin the C restatement
// (oracle/gw_oracle.c) and as the "reference" CPU baseline in bench.py.
// Nothing here is shipped in the product library.
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>

#include "../include/gwb.h"
#include "gw/diagnostics.hpp"
#include "gw/io.hpp"
#include "gw/projections.hpp"
#include "gw/solvers.hpp"
#include "gw/tasks.hpp"
#include "gw/types.hpp"

namespace {

gw::Matrix from_col_major(const double* p, int64_t r, int64_t c) {
  gw::Matrix m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

gw::Vector vec(const double* p, int64_t n) {
  gw::Vector v(n);
  std::memcpy(v.data(), p, sizeof(double) * static_cast<size_t>(n));
  return v;
}

void to_col_major(const gw::Matrix& m, double* out) {
  std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(m.size()));
}

int32_t fill(gwb_status* st, int32_t code, const std::string& what) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->code = code;
    std::snprintf(st->message, sizeof(st->message), "%s", what.c_str());
  }
  return code;
}

// Maps the reference exception hierarchy (types.hpp:27-59) to codes.
template <class F>
int32_t guarded(gwb_status* st, F&& f) {
  try {
    f();
    return fill(st, GWB_OK, "");
  } catch (const gw::NumericalInstabilityError& e) {
    fill(st, GWB_ERR_NUMERICAL, e.what());
    if (st) {
      st->iteration = e.iteration();
      std::snprintf(st->solver, sizeof(st->solver), "%s", e.solver().c_str());
    }
    return GWB_ERR_NUMERICAL;
  } catch (const gw::ZeroSumLineError& e) {
    fill(st, GWB_ERR_ZERO_SUM, e.what());
    if (st) {
      st->axis = e.axis() == gw::Axis::Rows ? GWB_ROWS : GWB_COLS;
      st->index = e.index();
    }
    return GWB_ERR_ZERO_SUM;
  } catch (const gw::ConfigError& e) {
    return fill(st, GWB_ERR_CONFIG, e.what());
  } catch (const gw::DimensionMismatchError& e) {
    return fill(st, GWB_ERR_DIMENSION, e.what());
  } catch (const std::domain_error& e) {
    return fill(st, GWB_ERR_DOMAIN, e.what());
  } catch (const std::invalid_argument& e) {
    return fill(st, GWB_ERR_INVALID, e.what());
  } catch (const std::exception& e) {
    return fill(st, GWB_ERR_RUNTIME, e.what());
  }
}

gw::SolverConfig to_config(const gwb_config* c) {
  gw::SolverConfig s;
  s.algorithm = static_cast<gw::Algorithm>(c->algorithm);
  s.geometry = static_cast<gw::Geometry>(c->geometry);
  s.rho = c->rho;
  s.step = c->step;
  s.epsilon_reg = c->epsilon_reg;
  s.inner_iters = c->inner_iters;
  s.inner_tol = c->inner_tol;
  s.rel_tol = c->rel_tol;
  s.max_iters = c->max_iters;
  s.perturbation = c->perturbation;
  s.switch_iters = c->switch_iters;
  s.seed = c->seed;
  s.log_domain = c->log_domain != 0;
  s.record_residual = c->record_residual != 0;
  return s;
}

void write_edges(const gw::Graph& g, int32_t* edges, int64_t cap,
                 int64_t* count) {
  *count = static_cast<int64_t>(g.edges().size());
  int64_t k = 0;
  for (auto [a, b] : g.edges()) {
    if (k >= cap) break;
    edges[2 * k] = a;
    edges[2 * k + 1] = b;
    ++k;
  }
}

gw::Graph read_graph(int64_t n, const int32_t* edges, int64_t count) {
  std::vector<std::pair<int, int>> e;
  e.reserve(static_cast<size_t>(count));
  for (int64_t k = 0; k < count; ++k) e.emplace_back(edges[2 * k], edges[2 * k + 1]);
  return gw::Graph(n, std::move(e));
}

}  // namespace

extern "C" {

int32_t gwref_solve(const gwb_config* cfg, const double* dx, int64_t n,
                    const double* dy, int64_t m, const double* mu,
                    const double* nu, const double* initial, double* out_final,
                    double* out_pi, double* out_w, gwb_record* trace,
                    int32_t trace_cap, int32_t* n_records, int32_t* converged,
                    int32_t* iterations_used, gwb_status* st) {
  *n_records = 0;
  return guarded(st, [&] {
    const gw::DistanceMatrix d_x(from_col_major(dx, n, n));
    const gw::DistanceMatrix d_y(from_col_major(dy, m, m));
    const gw::ProbabilityVector p_mu(vec(mu, n));
    const gw::ProbabilityVector p_nu(vec(nu, m));
    gw::SolveOptions opts;
    if (initial) opts.initial = from_col_major(initial, n, m);
    const gw::SolveReport rep = gw::solve(d_x, d_y, p_mu, p_nu, to_config(cfg), opts);
    to_col_major(rep.final_coupling.entries(), out_final);
    if (out_pi && rep.pi_half) to_col_major(rep.pi_half->entries(), out_pi);
    if (out_w && rep.w_half) to_col_major(rep.w_half->entries(), out_w);
    const int32_t cnt = static_cast<int32_t>(rep.trace.size());
    if (cnt > trace_cap) throw std::runtime_error("trace capacity exceeded");
    for (int32_t k = 0; k < cnt; ++k) {
      const gw::IterationRecord& r = rep.trace[k];
      gwb_record& o = trace[k];
      std::memset(&o, 0, sizeof(o));
      o.iter = r.iter;
      o.objective = r.objective;
      o.marginal_infeasibility = r.marginal_infeasibility;
      o.split_gap = r.split_gap;
      o.has_residual = r.residual.has_value();
      o.residual = r.residual.value_or(0.0);
      o.rel_change = r.rel_change;
      o.elapsed_seconds = r.elapsed_seconds;
      o.phase = r.phase;
    }
    *n_records = cnt;
    *converged = rep.converged;
    *iterations_used = rep.iterations_used;
  });
}

int32_t gwref_gw_objective(const double* dx, int64_t n, const double* dy,
                           int64_t m, const double* pi, int64_t rows,
                           int64_t cols, double* out, gwb_status* st) {
  return guarded(st, [&] {
    *out = gw::gw_objective(gw::DistanceMatrix(from_col_major(dx, n, n)),
                            gw::DistanceMatrix(from_col_major(dy, m, m)),
                            from_col_major(pi, rows, cols));
  });
}

int32_t gwref_product_coupling(const double* mu, int64_t n, const double* nu,
                               int64_t m, double* out, gwb_status* st) {
  return guarded(st, [&] {
    to_col_major(gw::product_coupling(gw::ProbabilityVector(vec(mu, n)),
                                      gw::ProbabilityVector(vec(nu, m)))
                     .entries(),
                 out);
  });
}

int32_t gwref_kl_scale(const double* pi, int64_t n, int64_t m,
                       const double* target, int64_t target_len, int32_t axis,
                       double* out, gwb_status* st) {
  return guarded(st, [&] {
    to_col_major(gw::kl_scale(from_col_major(pi, n, m),
                              gw::ProbabilityVector(vec(target, target_len)),
                              axis == GWB_ROWS ? gw::Axis::Rows : gw::Axis::Cols),
                 out);
  });
}

int32_t gwref_sinkhorn_project(const double* kernel, int64_t n, int64_t m,
                               const double* mu, const double* nu, double tol,
                               int32_t max_iters, int32_t log_domain,
                               double* out, int32_t* iterations,
                               double* marginal_error, int32_t* converged,
                               gwb_status* st) {
  return guarded(st, [&] {
    const gw::ProbabilityVector p_mu(vec(mu, n)), p_nu(vec(nu, m));
    const gw::Matrix k = from_col_major(kernel, n, m);
    const gw::SinkhornResult r =
        log_domain ? gw::sinkhorn_project_log(k, p_mu, p_nu, tol, max_iters)
                   : gw::sinkhorn_project(k, p_mu, p_nu, tol, max_iters);
    to_col_major(r.coupling, out);
    *iterations = r.iterations;
    *marginal_error = r.marginal_error;
    *converged = r.converged;
  });
}

int32_t gwref_lipschitz_bound(const double* dx, int64_t n, const double* dy,
                              int64_t m, double* out, gwb_status* st) {
  return guarded(st, [&] {
    *out = gw::lipschitz_bound(gw::DistanceMatrix(from_col_major(dx, n, n)),
                               gw::DistanceMatrix(from_col_major(dy, m, m)));
  });
}

int32_t gwref_marginal_infeasibility(const double* pi, int64_t n, int64_t m,
                                     const double* mu, const double* nu,
                                     double* out, gwb_status* st) {
  return guarded(st, [&] {
    *out = gw::marginal_infeasibility(from_col_major(pi, n, m),
                                      gw::ProbabilityVector(vec(mu, n)),
                                      gw::ProbabilityVector(vec(nu, m)));
  });
}

int32_t gwref_split_gap(const double* pi, const double* w, int64_t n, int64_t m,
                        double* out, gwb_status* st) {
  return guarded(st, [&] {
    *out = gw::split_gap(from_col_major(pi, n, m), from_col_major(w, n, m));
  });
}

int32_t gwref_hard_assignment(const double* pi, int64_t n, int64_t m,
                              int32_t* out, gwb_status* st) {
  return guarded(st, [&] {
    const std::vector<int> a = gw::hard_assignment(from_col_major(pi, n, m));
    for (int64_t i = 0; i < n; ++i) out[i] = a[static_cast<size_t>(i)];
  });
}

int32_t gwref_coupling_entropy(const double* pi, int64_t n, int64_t m, double* out,
                               gwb_status* st) {
  return guarded(st, [&] { *out = gw::coupling_entropy(from_col_major(pi, n, m)); });
}

int32_t gwref_alignment_accuracy(const int32_t* pred, int64_t n_pred, const int32_t* gt,
                                 int64_t n_gt, double* out, gwb_status* st) {
  return guarded(st, [&] {
    *out = gw::alignment_accuracy(std::vector<int>(pred, pred + n_pred),
                                  std::vector<int>(gt, gt + n_gt));
  });
}

int32_t gwref_dykstra_project(const double* pi, int64_t n, int64_t m, const double* mu,
                              const double* nu, double tol, int32_t max_iters, double* out,
                              int32_t* sweeps, gwb_status* st) {
  *sweeps = 0;  // the reference does not report the sweep count
  return guarded(st, [&] {
    to_col_major(gw::dykstra_project(from_col_major(pi, n, m), gw::ProbabilityVector(vec(mu, n)),
                                     gw::ProbabilityVector(vec(nu, m)), tol, max_iters),
                 out);
  });
}

int32_t gwref_luo_tseng_residual(const double* dx, int64_t n, const double* dy, int64_t m,
                                 const double* pi, const double* mu, const double* nu,
                                 double dykstra_tol, double* out, gwb_status* st) {
  return guarded(st, [&] {
    *out = gw::luo_tseng_residual(gw::DistanceMatrix(from_col_major(dx, n, n)),
                                  gw::DistanceMatrix(from_col_major(dy, m, m)),
                                  from_col_major(pi, n, m), gw::ProbabilityVector(vec(mu, n)),
                                  gw::ProbabilityVector(vec(nu, m)), dykstra_tol);
  });
}

// write_coupling_csv (io.cpp:183-193) into a caller buffer; *len = bytes
// needed (the text is written only if it fits in cap).
int32_t gwref_format_coupling_csv(const double* pi, int64_t n, int64_t m, char* out, int64_t cap,
                                  int64_t* len, gwb_status* st) {
  return guarded(st, [&] {
    std::ostringstream os;
    gw::write_coupling_csv(os, from_col_major(pi, n, m));
    const std::string s = os.str();
    *len = static_cast<int64_t>(s.size());
    if (out && cap >= *len) std::memcpy(out, s.data(), s.size());
  });
}

// Generators (tasks.cpp) — used to pin the product's instance builders.
int32_t gwref_gen_barabasi_albert(int32_t n, int32_t m_attach, uint64_t seed,
                                  int32_t* edges, int64_t cap, int64_t* count,
                                  gwb_status* st) {
  return guarded(st, [&] {
    write_edges(gw::gen_barabasi_albert(n, m_attach, seed), edges, cap, count);
  });
}

int32_t gwref_gen_gaussian_partition(int32_t n, int32_t k, double p_in,
                                     double p_out, uint64_t seed,
                                     int32_t* edges, int64_t cap,
                                     int64_t* count, int32_t* labels,
                                     gwb_status* st) {
  return guarded(st, [&] {
    const gw::PartitionInstance p = gw::gen_gaussian_partition(n, k, p_in, p_out, seed);
    write_edges(p.graph, edges, cap, count);
    for (int32_t i = 0; i < n; ++i) labels[i] = p.ground_truth_labels[static_cast<size_t>(i)];
  });
}

int32_t gwref_permute_graph(int64_t n, const int32_t* edges, int64_t count,
                            uint64_t seed, int32_t* out_edges, int32_t* perm,
                            gwb_status* st) {
  return guarded(st, [&] {
    auto [g, p] = gw::permute_graph(read_graph(n, edges, count), seed);
    int64_t c = 0;
    write_edges(g, out_edges, count, &c);
    for (int64_t i = 0; i < n; ++i) perm[i] = p[static_cast<size_t>(i)];
  });
}

int32_t gwref_adjacency_distance(int64_t n, const int32_t* edges, int64_t count,
                                 double* out, gwb_status* st) {
  return guarded(st, [&] {
    to_col_major(gw::adjacency_distance(read_graph(n, edges, count)).entries(), out);
  });
}

}  // extern "C"
