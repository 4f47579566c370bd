// capi.cu — the extern "C" boundary (include/gwb.h).
//
// Host-side responsibilities only: argument validation in the reference's
// order (require_algorithm → validate → validate_inputs → initial shape →
// positivity, solvers.cpp:141-151), error mapping to the reference's
// exception classes and message formats (types.cpp:54-66), and driving the
// device engines.  All arithmetic on the solver path runs in the sm_100a
// kernels; when no device is present every compute entry point fails with
// GWB_ERR_RUNTIME (there is no CPU fallback).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gwb.h"
#include "../../include/gwb_ext.h"
#include "solver.cuh"
#include "standalone.cuh"

#define GWB_STR2(x) #x
#define GWB_STR(x) GWB_STR2(x)

namespace {

using gwb::BapgEngine;

struct ApiError {
  int32_t code;
  std::string msg;
  int32_t iteration = 0;
  std::string solver;
  int32_t axis = 0;
  int64_t index = 0;
};

int32_t fill(gwb_status* st, const ApiError& e) {
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->code = e.code;
    st->iteration = e.iteration;
    st->axis = e.axis;
    st->index = e.index;
    std::snprintf(st->solver, sizeof(st->solver), "%s", e.solver.c_str());
    std::snprintf(st->message, sizeof(st->message), "%s", e.msg.c_str());
  }
  return e.code;
}

int32_t ok(gwb_status* st) {
  if (st) std::memset(st, 0, sizeof(*st));
  return GWB_OK;
}

std::string fmt(const char* f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  std::vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

[[noreturn]] void fail(int32_t code, const std::string& msg) { throw ApiError{code, msg}; }

// NumericalInstabilityError(solver, iter, detail), types.cpp:60-66.
[[noreturn]] void numerical(const char* solver, int iter, const std::string& detail) {
  ApiError e{GWB_ERR_NUMERICAL,
             fmt("numerical instability in %s at iteration %d: %s", solver, iter, detail.c_str())};
  e.iteration = iter;
  e.solver = solver;
  throw e;
}

// ZeroSumLineError message, types.cpp:54-58.
std::string zero_sum_msg(int axis, int64_t index) {
  return fmt("%s %lld has nonpositive sum; cannot rescale", axis == GWB_ROWS ? "row" : "column",
             static_cast<long long>(index));
}

template <class F>
int32_t guarded(gwb_status* st, F&& f) {
  try {
    f();
    return ok(st);
  } catch (const ApiError& e) {
    return fill(st, e);
  } catch (const gwb::CudaError& e) {
    return fill(st, ApiError{GWB_ERR_RUNTIME, e.what()});
  } catch (const std::bad_alloc&) {
    return fill(st, ApiError{GWB_ERR_RUNTIME, "host allocation failed"});
  } catch (const std::exception& e) {
    return fill(st, ApiError{GWB_ERR_RUNTIME, e.what()});
  }
}

// ---- device selection (side channel; the reference API has none) ----------
std::mutex g_dev_mu;
std::vector<int> g_devices;

int primary_device() {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_devices.empty()) {
    if (const char* env = std::getenv("GWB_DEVICES")) {
      const char* p = env;
      while (*p) {
        char* end = nullptr;
        const long v = std::strtol(p, &end, 10);
        if (end == p) break;
        g_devices.push_back(static_cast<int>(v));
        p = *end == ',' ? end + 1 : end;
      }
    }
    if (g_devices.empty()) g_devices.push_back(0);
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(GWB_ERR_RUNTIME, "no CUDA device available: the GW solver path runs only on sm_100 GPUs");
  }
  if (g_devices[0] >= count) fail(GWB_ERR_RUNTIME, fmt("device %d not present", g_devices[0]));
  // Compute capability, once per device (cudaGetDeviceProperties is slow).
  static std::vector<int> checked;
  if (std::find(checked.begin(), checked.end(), g_devices[0]) == checked.end()) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, g_devices[0]);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, g_devices[0]);
    if (major != 10)
      fail(GWB_ERR_RUNTIME, fmt("device %d is sm_%d%d; this build targets sm_100a", g_devices[0],
                                major, minor));
    checked.push_back(g_devices[0]);
  }
  return g_devices[0];
}

// All selected devices (gwb_set_devices / GWB_DEVICES), validated: present and
// sm_100.  A device listed twice runs two ranks / slices on it (the sharded
// solve then emulates its collectives: a one-GPU test mode, shard.cu).
std::vector<int> solve_devices() {
  primary_device();
  std::vector<int> devs;
  {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    devs = g_devices;
  }
  int count = 0;
  cudaGetDeviceCount(&count);
  for (size_t k = 0; k < devs.size(); ++k) {
    if (devs[k] < 0 || devs[k] >= count) fail(GWB_ERR_RUNTIME, fmt("device %d not present", devs[k]));
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, devs[k]);
    if (major != 10) fail(GWB_ERR_RUNTIME, fmt("device %d is not sm_100", devs[k]));
  }
  return devs;
}

const char* algo_name(int32_t a) {
  switch (a) {
    case GWB_BAPG: return "bapg";
    case GWB_BPG: return "bpg";
    case GWB_EBPG: return "ebpg";
    case GWB_HBPG: return "hbpg";
    case GWB_FW: return "fw";
  }
  return "?";
}

// validate(SolverConfig), types.cpp:176-188.
void validate_config(const gwb_config* c) {
  if (!c) fail(GWB_ERR_CONFIG, "null config");
  if (c->rho <= 0.0) fail(GWB_ERR_CONFIG, "rho must be positive");
  if (c->step <= 0.0) fail(GWB_ERR_CONFIG, "step must be positive");
  if (c->epsilon_reg <= 0.0) fail(GWB_ERR_CONFIG, "eps must be positive");
  if (c->inner_iters < 1) fail(GWB_ERR_CONFIG, "inner-iters must be >= 1");
  if (c->inner_tol <= 0.0) fail(GWB_ERR_CONFIG, "inner-tol must be positive");
  if (c->rel_tol <= 0.0) fail(GWB_ERR_CONFIG, "rel-tol must be positive");
  if (c->max_iters < 1) fail(GWB_ERR_CONFIG, "max-iters must be >= 1");
  if (c->perturbation < 0.0 || c->perturbation >= 1.0)
    fail(GWB_ERR_CONFIG, "perturbation must lie in [0, 1)");
  if (c->switch_iters < 0) fail(GWB_ERR_CONFIG, "switch-iters must be >= 0");
  if (c->precision < GWB_PREC_AUTO || c->precision > GWB_PREC_F16X3)
    fail(GWB_ERR_CONFIG, "unknown precision");
}

void require_algorithm(const gwb_config* c, int32_t expected, const char* who) {
  if (c->algorithm != expected)
    fail(GWB_ERR_CONFIG, fmt("%s called with algorithm '%s'", who, algo_name(c->algorithm)));
}

struct SolveOut {
  double* out_final;
  double* out_pi;
  double* out_w;
  gwb_record* trace;
  int32_t trace_cap;
  int32_t* n_records;
  int32_t* converged;
  int32_t* iterations_used;
};

// Decodes DevStatus flags in the reference's precedence (solvers.cpp:164-189).
void raise_device_flags(const gwb::DevStatus& s, const char* solver) {
  using namespace gwb;
  if (s.flags == 0) return;
  const int it = s.err_iter;
  if (s.flags & kFlagOverflowA) numerical(solver, it, "exp overflow; increase rho");
  if (s.flags & kFlagZeroA) numerical(solver, it, zero_sum_msg(GWB_ROWS, s.zero_index));
  if (s.flags & kFlagOverflowB) numerical(solver, it, "exp overflow; increase rho");
  if (s.flags & kFlagZeroB) numerical(solver, it, zero_sum_msg(GWB_COLS, s.zero_index));
  numerical(solver, it, "non-finite iterate");
}

// BAPG trace records (IterationRecord, phase 0) from the engine's records.
void fill_trace(const SolveOut& o, const std::vector<gwb::HostRecord>& recs, int used,
                const std::vector<double>& residuals) {
  if (o.trace) {
    for (int k = 0; k < used; ++k) {
      gwb_record& r = o.trace[k];
      std::memset(&r, 0, sizeof(r));
      r.iter = k + 1;
      r.objective = recs[k].objective;
      r.marginal_infeasibility = recs[k].marginal_infeasibility;
      r.split_gap = recs[k].split_gap;
      r.rel_change = recs[k].rel_change;
      r.elapsed_seconds = recs[k].elapsed;
      r.phase = 0;
      if (k < static_cast<int>(residuals.size())) {
        r.residual = residuals[k];
        r.has_residual = 1;
      }
    }
  }
  if (o.n_records) *o.n_records = o.trace ? used : 0;
}

// bapg_solve (solvers.cpp:138-217) on the device engine.
void bapg(const gwb_config* cfg, const double* dx, int64_t n, const double* dy, int64_t m,
          const double* mu, const double* nu, const double* initial, gwb_observer observer,
          void* user, const SolveOut& o, const gwb::GraphInput* graphs) {
  const bool entropy = cfg->geometry == GWB_ENTROPY;
  const size_t len = static_cast<size_t>(n) * static_cast<size_t>(m);
  std::vector<double> w0;
  if (initial && entropy) {
    // initial_coupling + positivity (solvers.cpp:146-151), w0 = kl_scale(π0, ν, Cols)
    // (solvers.cpp:152; projections.cpp:23-31) — an O(nm) host pass, once.
    for (size_t k = 0; k < len; ++k)
      if (!(initial[k] > 0.0))
        fail(GWB_ERR_CONFIG,
             "bapg entropy geometry requires a strictly positive initialization (the product "
             "coupling qualifies)");
    w0.assign(initial, initial + len);
    for (int64_t j = 0; j < m; ++j) {
      double s = 0.0;
      for (int64_t i = 0; i < n; ++i) s += w0[j * n + i];
      if (!(s > 0.0) || !std::isfinite(s)) {
        ApiError e{GWB_ERR_ZERO_SUM, zero_sum_msg(GWB_COLS, j)};
        e.axis = GWB_COLS;
        e.index = j;
        throw e;
      }
      const double f = nu[j] / s;
      for (int64_t i = 0; i < n; ++i) w0[j * n + i] *= f;
    }
  }
  if (o.trace_cap < cfg->max_iters && o.trace)
    fail(GWB_ERR_CAPACITY, fmt("trace capacity %d < max_iters %d", o.trace_cap, cfg->max_iters));
  // Small problems (n, m ≤ 128, product-coupling start, no observer): the
  // whole solve runs on one SM in the on-chip batched kernel (batched.cu),
  // which falls back to this engine itself for non-fp16-exact D.
  if (!observer && !cfg->record_residual && !initial && !graphs && entropy && n <= 128 && m <= 128 &&
      (cfg->precision == GWB_PREC_AUTO || cfg->precision == GWB_PREC_F16X2)) {
    gwb::device_bapg_batched(cfg, 1, dx, n, dy, m, mu, nu, o.out_final, o.out_pi, o.out_w,
                             o.trace, o.trace_cap, o.n_records, o.converged, o.iterations_used,
                             /*name_problem=*/false);
    return;
  }
  // Several devices selected (gwb_set_devices / GWB_DEVICES): one problem
  // row-sharded across them in this process (shard.cu, NCCL over NVLink).
  // The observer / residual slow path, a caller's initial coupling and graph
  // inputs stay on the primary device.
  const std::vector<int> devs = solve_devices();
  if (devs.size() > 1 && !observer && !cfg->record_residual && !initial && !graphs && entropy) {
    std::vector<gwb::HostRecord> recs;
    int prec = 0;
    const gwb::DevStatus s = gwb::bapg_multi_device(*cfg, devs, dx, n, dy, m, mu, nu, o.out_final,
                                                    o.out_pi, o.out_w, &recs, &prec);
    raise_device_flags(s, "bapg");
    const int used = s.iter - 1;
    fill_trace(o, recs, used, {});
    if (o.converged) *o.converged = s.converged;
    if (o.iterations_used) *o.iterations_used = used;
    return;
  }
  const int device = devs[0];
  // GWB_PHASE_TIMES=1: wall time of each phase of the call on stderr.
  static const bool phase_times = std::getenv("GWB_PHASE_TIMES") != nullptr;
  auto tick = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!phase_times) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "gwb_solve phase %-9s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tick).count());
    tick = now;
  };
  BapgEngine eng(device, n, m, cfg->rho, cfg->precision, cfg->max_iters, nullptr);
  eng.set_geometry(cfg->geometry);
  lap("create");
  if (graphs)
    eng.load_graphs(*graphs, mu, nu);
  else
    eng.load_host(dx, dy, mu, nu);
  lap("load");
  // Quadratic: π⁰ itself goes to the device, which projects it (reset()).
  eng.reset(initial ? (entropy ? w0.data() : initial) : nullptr);
  lap("reset");
  gwb::DevStatus s;
  std::vector<double> residuals;
  if (!observer && !cfg->record_residual) {
    eng.run(cfg->max_iters, cfg->rel_tol);
    s = eng.status();
    raise_device_flags(s, "bapg");
  } else {
    // Slow path: host-synchronous iterations so the record's Luo-Tseng
    // residual (solvers.cpp:202-204) and then the observer (:206) see π, w.
    std::vector<double> hp(observer ? len : 0), hw(observer ? len : 0);
    s = eng.run_stepped(cfg->max_iters, cfg->rel_tol, [&](int k, const gwb::DevStatus&) {
      if (cfg->record_residual) residuals.push_back(eng.residual_of_average(1e-8));
      if (observer) {
        eng.outputs(nullptr, hp.data(), hw.data());
        if (observer(user, k, hp.data(), hw.data(), n, m) != 0)
          fail(GWB_ERR_RUNTIME, "observer requested abort");
      }
    });
    raise_device_flags(s, "bapg");
  }
  lap("run");
  const int used = s.iter - 1;
  eng.tail();
  fill_trace(o, eng.records(used), used, residuals);
  if (o.converged) *o.converged = s.converged;
  if (o.iterations_used) *o.iterations_used = used;
  lap("tail");
  eng.outputs(o.out_final, o.out_pi, o.out_w);
  lap("outputs");
}

int32_t solve_impl(int32_t expected, const gwb_config* cfg, const double* dx, int64_t n,
                   const double* dy, int64_t m, const double* mu, const double* nu,
                   const double* initial, gwb_observer observer, void* user, double* out_final,
                   double* out_pi, double* out_w, gwb_record* trace, int32_t trace_cap,
                   int32_t* n_records, int32_t* converged, int32_t* iterations_used,
                   gwb_status* st, const gwb::GraphInput* graphs = nullptr) {
  return guarded(st, [&] {
    if (!cfg) fail(GWB_ERR_CONFIG, "null config");
    const int32_t algo = expected >= 0 ? expected : cfg->algorithm;
    if (expected >= 0) {
      static const char* names[] = {"bapg_solve", "bpg_solve", "ebpg_solve", "hbpg_solve", "fw_solve"};
      require_algorithm(cfg, expected, names[expected]);
    }
    validate_config(cfg);
    if (n < 1 || m < 1) fail(GWB_ERR_DIMENSION, "distance matrix must be nonempty");
    if ((!graphs && (!dx || !dy)) || !mu || !nu || !out_final)
      fail(GWB_ERR_INVALID, "null input/output buffer");
    if (n_records) *n_records = 0;
    const SolveOut o{out_final, out_pi, out_w, trace, trace_cap, n_records, converged, iterations_used};
    switch (algo) {
      case GWB_BAPG:
        bapg(cfg, dx, n, dy, m, mu, nu, initial, observer, user, o, graphs);
        return;
      case GWB_EBPG:
      case GWB_BPG:
      case GWB_HBPG:
        gwb::bregman_solve(cfg, algo, dx, n, dy, m, mu, nu, initial, observer, user, out_final,
                           trace, trace_cap, n_records, converged, iterations_used, graphs);
        return;
      case GWB_FW:
        fail(GWB_ERR_UNSUPPORTED,
             "Frank-Wolfe (transportation-simplex LMO) is outside the B200 path (DESIGN.md)");
      default:
        fail(GWB_ERR_CONFIG, "unknown algorithm");
    }
  });
}

}  // namespace

// Exceptions from the standalone / Bregman modules surface as these.
namespace gwb {
[[noreturn]] void api_fail(int32_t code, const std::string& msg) { fail(code, msg); }
[[noreturn]] void api_numerical(const char* solver, int iter, const std::string& detail) {
  numerical(solver, iter, detail);
}
[[noreturn]] void api_zero_sum(int axis, int64_t index) {
  ApiError e{GWB_ERR_ZERO_SUM, zero_sum_msg(axis, index)};
  e.axis = axis;
  e.index = index;
  throw e;
}
int api_device() { return primary_device(); }
}  // namespace gwb

extern "C" {

void gwb_config_default(gwb_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->algorithm = GWB_BAPG;
  c->geometry = GWB_ENTROPY;
  c->rho = 0.1;
  c->step = 5.0;
  c->epsilon_reg = 0.1;
  c->inner_iters = 1000;
  c->inner_tol = 1e-9;
  c->rel_tol = 1e-6;
  c->max_iters = 2000;
  c->perturbation = 0.0;
  c->switch_iters = 200;
  c->seed = 0;
  c->log_domain = 0;
  c->record_residual = 0;
  c->precision = GWB_PREC_AUTO;
  c->quiet = 0;
}

int32_t gwb_validate_config(const gwb_config* cfg, gwb_status* st) {
  return guarded(st, [&] { validate_config(cfg); });
}

#define GWB_SOLVE_ARGS                                                                        \
  cfg, dx, n, dy, m, mu, nu, initial, observer, user, out_final, out_pi, out_w, trace,        \
      trace_cap, n_records, converged, iterations_used, st

int32_t gwb_solve GWB_SOLVE_SIGNATURE { return solve_impl(-1, GWB_SOLVE_ARGS); }
int32_t gwb_bapg_solve GWB_SOLVE_SIGNATURE { return solve_impl(GWB_BAPG, GWB_SOLVE_ARGS); }
int32_t gwb_bpg_solve GWB_SOLVE_SIGNATURE { return solve_impl(GWB_BPG, GWB_SOLVE_ARGS); }
int32_t gwb_ebpg_solve GWB_SOLVE_SIGNATURE { return solve_impl(GWB_EBPG, GWB_SOLVE_ARGS); }
int32_t gwb_hbpg_solve GWB_SOLVE_SIGNATURE { return solve_impl(GWB_HBPG, GWB_SOLVE_ARGS); }

namespace {
// Graph::Graph validation (types.cpp:155-174).
void validate_graph(int64_t nodes, const int32_t* edges, int64_t count) {
  if (nodes <= 0) fail(GWB_ERR_INVALID, "graph must have at least one node");
  if (count < 0 || (count > 0 && !edges)) fail(GWB_ERR_INVALID, "null edge list");
  for (int64_t k = 0; k < count; ++k) {
    const int32_t a = edges[2 * k], b = edges[2 * k + 1];
    if (a == b) fail(GWB_ERR_INVALID, fmt("self-loop at node %d", a));
    if (a < 0 || b < 0 || a >= nodes || b >= nodes)
      fail(GWB_ERR_INVALID, fmt("edge (%d,%d) out of range for %lld nodes", a, b,
                                static_cast<long long>(nodes)));
  }
}
}  // namespace

int32_t gwb_solve_graphs(const gwb_config* cfg, int64_t n, const int32_t* edges_x,
                         int64_t count_x, int64_t m, const int32_t* edges_y, int64_t count_y,
                         const double* mu, const double* nu, const double* initial,
                         gwb_observer observer, void* user, double* out_final, double* out_pi,
                         double* out_w, gwb_record* trace, int32_t trace_cap,
                         int32_t* n_records, int32_t* converged, int32_t* iterations_used,
                         gwb_status* st) {
  const int32_t rc = guarded(st, [&] {
    validate_graph(n, edges_x, count_x);
    validate_graph(m, edges_y, count_y);
  });
  if (rc != GWB_OK) return rc;
  const gwb::GraphInput g{edges_x, count_x, edges_y, count_y};
  return solve_impl(-1, cfg, nullptr, n, nullptr, m, mu, nu, initial, observer, user, out_final,
                    out_pi, out_w, trace, trace_cap, n_records, converged, iterations_used, st,
                    &g);
}

int32_t gwb_gw_objective(const double* dx, int64_t n, const double* dy, int64_t m,
                         const double* pi, int64_t pi_rows, int64_t pi_cols, double* out,
                         gwb_status* st) {
  return guarded(st, [&] {
    if (pi_rows != n || pi_cols != m)
      fail(GWB_ERR_DIMENSION, "gw_objective: coupling shape mismatch");
    *out = gwb::device_gw_objective(dx, n, dy, m, pi);
  });
}

int32_t gwb_product_coupling(const double* mu, int64_t n, const double* nu, int64_t m,
                             double* out, gwb_status* st) {
  return guarded(st, [&] { gwb::device_product_coupling(mu, n, nu, m, out); });
}

int32_t gwb_lipschitz_bound(const double* dx, int64_t n, const double* dy, int64_t m, double* out,
                            gwb_status* st) {
  return guarded(st, [&] { *out = gwb::device_lipschitz_bound(dx, n, dy, m); });
}

int32_t gwb_kl_scale(const double* pi, int64_t n, int64_t m, const double* target,
                     int64_t target_len, int32_t axis, double* out, gwb_status* st) {
  return guarded(st, [&] {
    if (axis == GWB_ROWS && n != target_len)
      fail(GWB_ERR_DIMENSION, "kl_scale: row count does not match target");
    if (axis != GWB_ROWS && m != target_len)
      fail(GWB_ERR_DIMENSION, "kl_scale: column count does not match target");
    gwb::device_kl_scale(pi, n, m, target, axis, out);
  });
}

int32_t gwb_sinkhorn_project(const double* kernel, int64_t n, int64_t m, const double* mu,
                             const double* nu, double tol, int32_t max_iters, int32_t log_domain,
                             double* out, int32_t* iterations, double* marginal_error,
                             int32_t* converged, gwb_status* st) {
  return guarded(st, [&] {
    gwb::device_sinkhorn(kernel, n, m, mu, nu, tol, max_iters, log_domain, out, iterations,
                         marginal_error, converged);
  });
}

int32_t gwb_marginal_infeasibility(const double* pi, int64_t n, int64_t m, const double* mu,
                                   int64_t mu_len, const double* nu, int64_t nu_len, double* out,
                                   gwb_status* st) {
  return guarded(st, [&] {
    if (mu_len != n || nu_len != m)
      fail(GWB_ERR_DIMENSION, "marginal_infeasibility: shape mismatch");
    *out = gwb::device_marginal_infeasibility(pi, n, m, mu, nu);
  });
}

int32_t gwb_split_gap(const double* pi, const double* w, int64_t n, int64_t m, double* out,
                      gwb_status* st) {
  return guarded(st, [&] { *out = gwb::device_split_gap(pi, w, n, m); });
}

int32_t gwb_hard_assignment(const double* pi, int64_t n, int64_t m, int32_t* out,
                            gwb_status* st) {
  return guarded(st, [&] { gwb::device_hard_assignment(pi, n, m, out); });
}

int32_t gwb_coupling_entropy(const double* pi, int64_t n, int64_t m, double* out,
                             gwb_status* st) {
  return guarded(st, [&] {
    if (!pi || !out) fail(GWB_ERR_INVALID, "null buffer");
    *out = n * m > 0 ? gwb::device_coupling_entropy(pi, n, m) : 0.0;
  });
}

int32_t gwb_format_coupling_csv(const double* pi, int64_t n, int64_t m, char* out, int64_t cap,
                                int64_t* len, gwb_status* st) {
  return guarded(st, [&] {
    if ((!pi && n * m > 0) || !len) fail(GWB_ERR_INVALID, "null buffer");
    if (n < 0 || m < 0) fail(GWB_ERR_DIMENSION, "negative shape");
    int64_t pos = 0;
    gwb::device_coupling_csv(pi, n, m, [&](const char* b, int64_t k) {
      if (out && pos + k <= cap) std::memcpy(out + pos, b, static_cast<size_t>(k));
      pos += k;
    }, len);
    if (out && cap < *len)
      fail(GWB_ERR_CAPACITY, fmt("buffer of %lld bytes < %lld needed", static_cast<long long>(cap),
                                 static_cast<long long>(*len)));
  });
}

int32_t gwb_write_coupling_csv_file(const char* path, const double* pi, int64_t n, int64_t m,
                                    gwb_status* st) {
  return guarded(st, [&] {
    if (!path || (!pi && n * m > 0)) fail(GWB_ERR_INVALID, "null buffer");
    if (n < 0 || m < 0) fail(GWB_ERR_DIMENSION, "negative shape");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) fail(GWB_ERR_RUNTIME, std::string("cannot write '") + path + "'");  // io.cpp:197
    int64_t total = 0;
    bool ok = true;
    try {
      gwb::device_coupling_csv(pi, n, m, [&](const char* b, int64_t k) {
        ok = ok && std::fwrite(b, 1, static_cast<size_t>(k), f) == static_cast<size_t>(k);
      }, &total);
    } catch (...) {
      std::fclose(f);
      throw;
    }
    ok = std::fclose(f) == 0 && ok;
    if (!ok) fail(GWB_ERR_RUNTIME, std::string("cannot write '") + path + "'");
  });
}

int32_t gwb_dykstra_project(const double* pi, int64_t n, int64_t m, const double* mu,
                            const double* nu, double tol, int32_t max_iters, double* out,
                            gwb_status* st) {
  return guarded(st, [&] {
    if (!pi || !mu || !nu || !out) fail(GWB_ERR_INVALID, "null buffer");
    if (n < 1 || m < 1) fail(GWB_ERR_DIMENSION, "dykstra_project: shape mismatch");
    gwb::device_dykstra_project(pi, n, m, mu, nu, tol, max_iters, out);
  });
}

int32_t gwb_luo_tseng_residual(const double* dx, int64_t n, const double* dy, int64_t m,
                               const double* pi, const double* mu, const double* nu,
                               double dykstra_tol, double* out, gwb_status* st) {
  return guarded(st, [&] {
    if (!dx || !dy || !pi || !mu || !nu || !out) fail(GWB_ERR_INVALID, "null buffer");
    if (n < 1 || m < 1) fail(GWB_ERR_DIMENSION, "luo_tseng_residual: shape mismatch");
    *out = gwb::device_luo_tseng_residual(dx, n, dy, m, pi, mu, nu, dykstra_tol);
  });
}

int32_t gwb_alignment_accuracy(const int32_t* pred, int64_t n_pred, const int32_t* gt,
                               int64_t n_gt, double* out, gwb_status* st) {
  return guarded(st, [&] {
    // O(n) integer work: host side, as the reference.
    if (n_pred < n_gt)
      fail(GWB_ERR_DIMENSION, "alignment_accuracy: prediction does not cover all ground-truth nodes");
    if (n_gt == 0) fail(GWB_ERR_INVALID, "empty ground truth");
    int64_t hits = 0;
    for (int64_t i = 0; i < n_gt; ++i) hits += pred[i] == gt[i];
    *out = 100.0 * static_cast<double>(hits) / static_cast<double>(n_gt);
  });
}

int32_t gwb_bapg_solve_batched(const gwb_config* cfg, int64_t batch, const double* dx, int64_t n,
                               const double* dy, int64_t m, const double* mu, const double* nu,
                               double* out_final, double* out_pi, double* out_w,
                               gwb_record* trace, int32_t trace_cap, int32_t* n_records,
                               int32_t* converged, int32_t* iterations_used, gwb_status* st) {
  return guarded(st, [&] {
    if (!cfg) fail(GWB_ERR_CONFIG, "null config");
    require_algorithm(cfg, GWB_BAPG, "bapg_solve");
    validate_config(cfg);
    if (batch < 1 || n < 1 || m < 1) fail(GWB_ERR_DIMENSION, "empty batch or problem");
    // Several devices: contiguous ranges of problems per GPU, no
    // communication (one host thread per device); the lowest-index failing
    // problem raises, as on one device.
    const std::vector<int> devs = solve_devices();
    const int P = static_cast<int>(std::min<int64_t>(static_cast<int64_t>(devs.size()), batch));
    std::vector<double> ms(P, 0.0);
    std::vector<std::exception_ptr> errs(P);
    auto slice = [&](int r) {
      const int64_t b0 = batch * r / P, b1 = batch * (r + 1) / P;
      const int64_t nn = n * n, mm = m * m, nm = n * m;
      gwb::device_bapg_batched(cfg, b1 - b0, dx + b0 * nn, n, dy + b0 * mm, m, mu + b0 * n,
                               nu + b0 * m, out_final + b0 * nm, out_pi ? out_pi + b0 * nm : nullptr,
                               out_w ? out_w + b0 * nm : nullptr,
                               trace ? trace + b0 * trace_cap : nullptr, trace_cap,
                               n_records ? n_records + b0 : nullptr,
                               converged ? converged + b0 : nullptr,
                               iterations_used ? iterations_used + b0 : nullptr, true, devs[r], b0,
                               &ms[r]);
    };
    if (P <= 1) {
      slice(0);
    } else {
      std::vector<std::thread> th;
      for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] {
          try {
            slice(r);
          } catch (...) {
            errs[r] = std::current_exception();
          }
        });
      for (auto& t : th) t.join();
      for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    }
    gwb::set_batched_last(*std::max_element(ms.begin(), ms.end()), batch);
  });
}

int32_t gwb_set_devices(int32_t count, const int32_t* ids, gwb_status* st) {
  return guarded(st, [&] {
    if (count < 1 || !ids) fail(GWB_ERR_CONFIG, "gwb_set_devices needs at least one id");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    g_devices.assign(ids, ids + count);
  });
}

// ---- device-resident session ---------------------------------------------
struct gwb_session {
  std::unique_ptr<BapgEngine> eng;
  gwb_config cfg;
};

int32_t gwb_session_create(const gwb_config* cfg, int64_t n, int64_t m, int32_t device,
                           gwb_session** out, gwb_status* st) {
  return guarded(st, [&] {
    if (!cfg) fail(GWB_ERR_CONFIG, "null config");
    require_algorithm(cfg, GWB_BAPG, "bapg_solve");
    validate_config(cfg);
    if (n < 1 || m < 1) fail(GWB_ERR_DIMENSION, "distance matrix must be nonempty");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device >= count) {
      cudaGetLastError();
      fail(GWB_ERR_RUNTIME, "no CUDA device available");
    }
    auto* s = new gwb_session();
    s->cfg = *cfg;
    s->eng.reset(new BapgEngine(device, n, m, cfg->rho, cfg->precision, cfg->max_iters, nullptr));
    s->eng->set_geometry(cfg->geometry);
    *out = s;
  });
}

int32_t gwb_session_load_device(gwb_session* s, const float* dx, int64_t ldx, const float* dy,
                                int64_t ldy, const float* mu, const float* nu, void* stream,
                                gwb_status* st) {
  return guarded(st, [&] {
    (void)stream;
    s->eng->load_device(dx, ldx, dy, ldy, mu, nu);
  });
}

int32_t gwb_session_reset(gwb_session* s, void* stream, gwb_status* st) {
  return guarded(st, [&] {
    (void)stream;
    s->eng->reset(nullptr);
  });
}

int32_t gwb_session_iterate(gwb_session* s, int32_t iters, void* stream, int64_t* launches,
                            gwb_status* st) {
  return guarded(st, [&] {
    (void)stream;
    const bool timing = launches != nullptr && *launches < 0;
    s->eng->set_timing(timing);
    const int64_t l = s->eng->iterate(iters, s->cfg.rel_tol, !timing);
    if (launches) *launches = l;
  });
}

int32_t gwb_session_stream(gwb_session* s, void** stream, gwb_status* st) {
  return guarded(st, [&] { *stream = static_cast<void*>(s->eng->stream()); });
}

int32_t gwb_session_info(gwb_session* s, int32_t* precision, double* gemm_flops_per_iter,
                         gwb_status* st) {
  return guarded(st, [&] {
    *precision = s->eng->precision();
    *gemm_flops_per_iter = s->eng->gemm_flops_per_iter();
  });
}

int32_t gwb_session_pi(gwb_session* s, float** pi, int64_t* ld, gwb_status* st) {
  return guarded(st, [&] {
    *pi = s->eng->pi_dev();
    *ld = s->eng->ld();
  });
}

int32_t gwb_session_kernel_ms(gwb_session* s, int32_t kind, double* avg_ms, int64_t* count,
                              gwb_status* st) {
  return guarded(st, [&] { s->eng->kernel_ms(kind, avg_ms, count); });
}

int32_t gwb_session_readout(gwb_session* s, const int32_t* ground_truth, int64_t n_gt,
                            int32_t* assignment, gwb_readout* out, gwb_status* st) {
  return guarded(st, [&] {
    if (!s || !out) fail(GWB_ERR_INVALID, "null session or output");
    if (ground_truth) {
      if (n_gt == 0) fail(GWB_ERR_INVALID, "empty ground truth");
      if (s->eng->n() < n_gt)
        fail(GWB_ERR_DIMENSION,
             "alignment_accuracy: prediction does not cover all ground-truth nodes");
    }
    gwb::Readout r;
    s->eng->readout(ground_truth, n_gt, assignment, &r);
    std::memset(out, 0, sizeof(*out));
    out->objective = r.objective;
    out->marginal_infeasibility = r.marginal_infeasibility;
    out->entropy = r.entropy;
    out->split_gap = r.split_gap;
    out->residual = r.residual;
    out->accuracy = r.accuracy;
    out->has_accuracy = ground_truth != nullptr;
  });
}

int32_t gwb_session_write_coupling_csv(gwb_session* s, const char* path, gwb_status* st) {
  return guarded(st, [&] {
    if (!s || !path) fail(GWB_ERR_INVALID, "null session or path");
    std::FILE* f = std::fopen(path, "wb");
    if (!f) fail(GWB_ERR_RUNTIME, std::string("cannot write '") + path + "'");
    bool ok = true;
    try {
      s->eng->final_csv([&](const char* b, int64_t k) {
        ok = ok && std::fwrite(b, 1, static_cast<size_t>(k), f) == static_cast<size_t>(k);
      });
    } catch (...) {
      std::fclose(f);
      throw;
    }
    ok = std::fclose(f) == 0 && ok;
    if (!ok) fail(GWB_ERR_RUNTIME, std::string("cannot write '") + path + "'");
  });
}

// ---- row-sharded eBPG / BPG / hBPG (bregman.cu) ----------------------------
struct gwb_bshard {
  gwb::BregShard* b = nullptr;
  int64_t n = 0, m = 0;
  ~gwb_bshard() { gwb::bshard_destroy(b); }
};

int32_t gwb_bshard_create(const gwb_config* cfg, int64_t n, int64_t m, int32_t rank, int32_t world,
                          int32_t device, void* stream, gwb_bshard** out, gwb_status* st) {
  return guarded(st, [&] {
    if (!cfg || !out) fail(GWB_ERR_INVALID, "null argument");
    validate_config(cfg);
    if (cfg->algorithm != GWB_EBPG && cfg->algorithm != GWB_BPG && cfg->algorithm != GWB_HBPG)
      fail(GWB_ERR_CONFIG, "gwb_bshard_create: algorithm must be ebpg, bpg or hbpg");
    if (n < 1 || m < 1 || world < 1 || rank < 0 || rank >= world)
      fail(GWB_ERR_DIMENSION, "gwb_bshard_create: bad shape or rank");
    if (cfg->precision != GWB_PREC_BF16X3 && cfg->precision != GWB_PREC_BF16X2 &&
        cfg->precision != GWB_PREC_3XTF32 && cfg->precision != GWB_PREC_F16X2)
      fail(GWB_ERR_CONFIG,
           "gwb_bshard_create: resolve the precision across ranks first (f16x2, bf16x3, bf16x2 or 3xtf32; dist.resolve_precision)");
    if (cfg->record_residual) fail(GWB_ERR_UNSUPPORTED, "record_residual is single-GPU only");
    auto* s = new gwb_bshard();
    s->n = n;
    s->m = m;
    try {
      s->b = gwb::bshard_create(*cfg, cfg->algorithm, n, m, world, rank, device,
                                static_cast<cudaStream_t>(stream));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

int32_t gwb_bshard_layout(gwb_bshard* s, int64_t* rows_per_shard, int64_t* row_begin,
                          int64_t* rows_valid, int64_t* padded_rows, int64_t* ld, int32_t* planes,
                          int32_t* elem_bytes, int64_t* vt_bytes, gwb_status* st) {
  return guarded(st, [&] {
    gwb::bshard_layout(s->b, rows_per_shard, row_begin, rows_valid, padded_rows, ld);
    gwb::bshard_comm_layout(s->b, planes, elem_bytes, vt_bytes);
  });
}

int32_t gwb_bshard_set_comm(gwb_bshard* s, void* vt, float* g, gwb_status* st) {
  return guarded(st, [&] { gwb::bshard_set_comm(s->b, vt, g); });
}

int32_t gwb_bshard_load_device(gwb_bshard* s, const float* dx_rows, int64_t ldx, const float* dy,
                               int64_t ldy, const double* mu, const double* nu, gwb_status* st) {
  return guarded(st, [&] {
    if (!dy || !mu || !nu) fail(GWB_ERR_INVALID, "null input");
    gwb::bshard_load(s->b, dx_rows, ldx, dy, ldy, mu, nu, s->m);
  });
}

int32_t gwb_bshard_phase(gwb_bshard* s, int32_t k, int32_t op, gwb_status* st) {
  return guarded(st, [&] { gwb::bshard_phase(s->b, k, op); });
}

int32_t gwb_bshard_status(gwb_bshard* s, int32_t* done, int32_t* iter, int32_t* flags,
                          int32_t* converged, gwb_status* st) {
  return guarded(st, [&] { gwb::bshard_status(s->b, done, iter, flags, converged); });
}

int32_t gwb_bshard_stream(gwb_bshard* s, void** stream, gwb_status* st) {
  return guarded(st, [&] { *stream = gwb::bshard_stream(s->b); });
}

int32_t gwb_bshard_finish(gwb_bshard* s, double* out_final, gwb_record* trace, int32_t trace_cap,
                          int32_t* n_records, int32_t* converged, int32_t* iterations_used,
                          gwb_status* st) {
  return guarded(st, [&] {
    gwb::bshard_finish(s->b, out_final, trace, trace_cap, n_records, converged, iterations_used);
  });
}

int32_t gwb_bshard_destroy(gwb_bshard* s) {
  delete s;
  return GWB_OK;
}

int32_t gwb_session_destroy(gwb_session* s) {
  delete s;
  return GWB_OK;
}

int32_t gwb_debug_gemm_stamps(uint64_t* out, int32_t max_ctas, int32_t* count) {
  *count = gwb::gemm_debug_stamps(reinterpret_cast<unsigned long long*>(out), max_ctas);
  return GWB_OK;
}

int32_t gwb_debug_gemm(const float* a, int64_t lda, const float* b, int64_t ldb, float* c,
                       int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t precision,
                       void* stream, gwb_status* st) {
  return guarded(st, [&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    gwb::GemmDesc d;
    d.M = M;
    d.N = N;
    d.K = K;
    d.a = a;
    d.lda = lda;
    d.b = b;
    d.ldb = ldb;
    d.c = c;
    d.ldc = ldc;
    float* alo = nullptr;
    float* blo = nullptr;
    if (precision == GWB_PREC_3XTF32) {
      GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&alo), sizeof(float) * M * lda + 256, s));
      GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&blo), sizeof(float) * N * ldb + 256, s));
      gwb::launch_tf32_aux(a, M, K, lda, alo, 2, s);
      gwb::launch_tf32_aux(b, N, K, ldb, blo, 2, s);
      d.a_lo = alo;
      d.b_lo = blo;
      d.three_pass = true;
    }
    void* a16 = nullptr;
    float* bpl = nullptr;
    if (precision == GWB_PREC_F16X2 || precision == GWB_PREC_BF16X3) {
      // Split-plane path: A (exact in fp16 / bf16) × planes of B (fp16 planes
      // at scale 1: B must lie inside fp16 range).
      const bool f16 = precision == GWB_PREC_F16X2;
      GWB_CUDA(cudaMallocAsync(&a16, sizeof(uint16_t) * M * lda + 256, s));
      GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bpl), 6 * N * ldb + 256, s));
      if (f16) gwb::launch_to_f16(a, M, K, lda, a16, s);
      else gwb::launch_to_bf16(a, M, K, lda, a16, s);
      gwb::launch_tf32_aux(b, N, K, ldb, bpl, f16 ? 5 : 3, s, 1.0f);
      d.a = nullptr;
      d.b = nullptr;
      d.f16 = f16;
      d.bf16_planes = f16 ? 2 : 3;
      d.a_bf16 = a16;
      for (int k = 0; k < d.bf16_planes; ++k)
        d.b_bf16[k] = reinterpret_cast<uint16_t*>(bpl) + static_cast<int64_t>(k) * N * ldb;
    }
    if (precision == GWB_PREC_F16X3) {
      // Both operands as scale-1 fp16 hi + lo planes (values inside fp16
      // range), 3 passes.
      GWB_CUDA(cudaMallocAsync(&a16, sizeof(uint16_t) * 2 * M * lda + 256, s));
      GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bpl), 4 * N * ldb + 256, s));
      gwb::launch_tf32_aux(a, M, K, lda, static_cast<float*>(a16), 5, s, 1.0f);
      gwb::launch_tf32_aux(b, N, K, ldb, bpl, 5, s, 1.0f);
      d.a = nullptr;
      d.b = nullptr;
      d.f16 = true;
      d.bf16_planes = 2;
      d.a_bf16 = a16;
      d.a_bf16_lo = static_cast<uint16_t*>(a16) + M * lda;
      for (int k = 0; k < 2; ++k)
        d.b_bf16[k] = reinterpret_cast<uint16_t*>(bpl) + static_cast<int64_t>(k) * N * ldb;
    }
    gwb::GemmPlan* p = gwb::gemm_plan_create(d);
    const cudaError_t e = gwb::gemm_launch(p, s);
    gwb::gemm_plan_destroy(p);
    if (a16) cudaFreeAsync(a16, s);
    if (bpl) cudaFreeAsync(bpl, s);
    if (alo) cudaFreeAsync(alo, s);
    if (blo) cudaFreeAsync(blo, s);
    GWB_CUDA(e);
  });
}

const char* gwb_version(void) {
  return "gwb 0.1 (sm_100a: tcgen05 kind::tf32 GEMM chain, CUDA " GWB_STR(__CUDACC_VER_MAJOR__) "."
      GWB_STR(__CUDACC_VER_MINOR__) ")";
}

}  // extern "C"
