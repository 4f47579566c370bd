/*
 * gw_oracle.c — fp64 CPU restatement of the reference BAPG / eBPG / BPG /
 * hBPG path.  TEST INFRASTRUCTURE ONLY: used by tests/, smoke() and
 * bench.py's cpu_baseline leg as the checker; never shipped or measured as
 * the product.
 *
 * Every function cites the reference file:line it follows
 * (/root/reference/proj/...).  Storage is column-major fp64 as in Eigen.
 * Association orders match the reference: (D_X·π)·D_Y (solvers.cpp:16-19),
 * ROWS→COLS sweep order (projections.cpp:101-103), division by rho rather
 * than multiplication by 1/rho (solvers.cpp:164).
 */
#include "gw_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define IDX(i, j, ld) ((size_t)(j) * (size_t)(ld) + (size_t)(i))

static gwo_cblas_dgemm_fn g_dgemm = NULL;

void gwo_set_dgemm(gwo_cblas_dgemm_fn fn) { g_dgemm = fn; }

/* ---- status helpers --------------------------------------------------- */

static int32_t set_status(gwb_status* st, int32_t code, const char* solver,
                          int32_t iter, const char* fmt, ...) {
  if (st) {
    memset(st, 0, sizeof(*st));
    st->code = code;
    st->iteration = iter;
    if (solver) snprintf(st->solver, sizeof(st->solver), "%s", solver);
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(st->message, sizeof(st->message), fmt, ap);
    va_end(ap);
  }
  return code;
}

/* NumericalInstabilityError message format: types.cpp:60-66. */
static int32_t numerical(gwb_status* st, const char* solver, int32_t iter,
                         const char* detail) {
  char buf[512];
  snprintf(buf, sizeof(buf), "%s", detail);
  return set_status(st, GWB_ERR_NUMERICAL, solver, iter,
                    "numerical instability in %s at iteration %d: %s", solver,
                    iter, buf);
}

/* ZeroSumLineError message: types.cpp:54-58. */
static int32_t zero_sum(gwb_status* st, int32_t axis, int64_t index) {
  set_status(st, GWB_ERR_ZERO_SUM, NULL, 0,
             "%s %lld has nonpositive sum; cannot rescale",
             axis == GWB_ROWS ? "row" : "column", (long long)index);
  if (st) {
    st->axis = axis;
    st->index = index;
  }
  return GWB_ERR_ZERO_SUM;
}

static double now_seconds(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* ---- dense kernels ----------------------------------------------------- */

/* C(r×c) = A(r×k)·B(k×c), column-major. */
static void matmul(const double* a, const double* b, double* c, int64_t r,
                   int64_t k, int64_t cc) {
  if (g_dgemm) {
    /* CblasColMajor=102, CblasNoTrans=111 */
    g_dgemm(102, 111, 111, r, cc, k, 1.0, a, r, b, k, 0.0, c, r);
    return;
  }
  for (int64_t j = 0; j < cc; ++j) {
    double* cj = c + (size_t)j * r;
    for (int64_t i = 0; i < r; ++i) cj[i] = 0.0;
    for (int64_t p = 0; p < k; ++p) {
      const double bpj = b[IDX(p, j, k)];
      if (bpj == 0.0) continue;
      const double* ap = a + (size_t)p * r;
      for (int64_t i = 0; i < r; ++i) cj[i] += ap[i] * bpj;
    }
  }
}

/* structure_product: (D_X·π)·D_Y, solvers.cpp:16-19. */
void gwo_structure_product(const double* dx, int64_t n, const double* dy,
                           int64_t m, const double* pi, double* out) {
  double* t = (double*)malloc(sizeof(double) * (size_t)n * (size_t)m);
  matmul(dx, pi, t, n, n, m);
  matmul(t, dy, out, n, m, m);
  free(t);
}

static double fro_norm(const double* a, size_t len) {
  double s = 0.0;
  for (size_t k = 0; k < len; ++k) s += a[k] * a[k];
  return sqrt(s);
}

static double fro_diff(const double* a, const double* b, size_t len) {
  double s = 0.0;
  for (size_t k = 0; k < len; ++k) {
    const double d = a[k] - b[k];
    s += d * d;
  }
  return sqrt(s);
}

static int all_finite(const double* a, size_t len) {
  for (size_t k = 0; k < len; ++k)
    if (!isfinite(a[k])) return 0;
  return 1;
}

/* gw_objective: -Σ (D_X π D_Y) ⊙ π, solvers.cpp:64-69 (check_shape :21-26). */
int32_t gwo_gw_objective(const double* dx, int64_t n, const double* dy,
                         int64_t m, const double* pi, int64_t rows,
                         int64_t cols, double* out, gwb_status* st) {
  if (rows != n || cols != m)
    return set_status(st, GWB_ERR_DIMENSION, NULL, 0,
                      "gw_objective: coupling shape mismatch");
  const size_t len = (size_t)n * (size_t)m;
  double* mm = (double*)malloc(sizeof(double) * len);
  gwo_structure_product(dx, n, dy, m, pi, mm);
  double s = 0.0;
  for (size_t k = 0; k < len; ++k) s += mm[k] * pi[k];
  free(mm);
  *out = -s;
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* product_coupling: μνᵀ, types.cpp:204-207. */
int32_t gwo_product_coupling(const double* mu, int64_t n, const double* nu,
                             int64_t m, double* out, gwb_status* st) {
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < n; ++i) out[IDX(i, j, n)] = mu[i] * nu[j];
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* kl_scale: projections.cpp:12-34. */
int32_t gwo_kl_scale(const double* pi, int64_t n, int64_t m,
                     const double* target, int64_t target_len, int32_t axis,
                     double* out, gwb_status* st) {
  if (out != pi) memcpy(out, pi, sizeof(double) * (size_t)n * (size_t)m);
  if (axis == GWB_ROWS) {
    if (n != target_len)
      return set_status(st, GWB_ERR_DIMENSION, NULL, 0,
                        "kl_scale: row count does not match target");
    for (int64_t i = 0; i < n; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < m; ++j) s += out[IDX(i, j, n)];
      if (!(s > 0.0) || !isfinite(s)) return zero_sum(st, GWB_ROWS, i);
      const double f = target[i] / s;
      for (int64_t j = 0; j < m; ++j) out[IDX(i, j, n)] *= f;
    }
  } else {
    if (m != target_len)
      return set_status(st, GWB_ERR_DIMENSION, NULL, 0,
                        "kl_scale: column count does not match target");
    for (int64_t j = 0; j < m; ++j) {
      double* col = out + (size_t)j * n;
      double s = 0.0;
      for (int64_t i = 0; i < n; ++i) s += col[i];
      if (!(s > 0.0) || !isfinite(s)) return zero_sum(st, GWB_COLS, j);
      const double f = target[j] / s;
      for (int64_t i = 0; i < n; ++i) col[i] *= f;
    }
  }
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* marginal_error_inf: projections.cpp:81-88. */
static double marginal_error_inf(const double* pi, int64_t n, int64_t m,
                                 const double* mu, const double* nu) {
  double row_err = 0.0, col_err = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < m; ++j) s += pi[IDX(i, j, n)];
    const double e = fabs(s - mu[i]);
    if (e > row_err) row_err = e;
  }
  for (int64_t j = 0; j < m; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += pi[IDX(i, j, n)];
    const double e = fabs(s - nu[j]);
    if (e > col_err) col_err = e;
  }
  return row_err > col_err ? row_err : col_err;
}

/* log_sum_exp over one line, max-shifted: projections.cpp:121-125. */
static double log_sum_exp(const double* x, int64_t len, int64_t stride,
                          const double* add) {
  double c = -INFINITY;
  for (int64_t k = 0; k < len; ++k) {
    const double v = x[(size_t)k * stride] + add[k];
    if (v > c || isnan(v)) c = v;
  }
  if (!isfinite(c)) return c;
  double s = 0.0;
  for (int64_t k = 0; k < len; ++k) s += exp(x[(size_t)k * stride] + add[k] - c);
  return c + log(s);
}

/* sinkhorn_project (projections.cpp:92-116) and sinkhorn_project_log
 * (projections.cpp:129-163). */
int32_t gwo_sinkhorn_project(const double* kernel, int64_t n, int64_t m,
                             const double* mu, const double* nu, double tol,
                             int32_t max_iters, int32_t log_domain,
                             double* out, int32_t* iterations,
                             double* marginal_error, int32_t* converged,
                             gwb_status* st) {
  const size_t len = (size_t)n * (size_t)m;
  *iterations = 0;
  *marginal_error = 0.0;
  *converged = 0;
  if (!log_domain) {
    memcpy(out, kernel, sizeof(double) * len);
    for (int32_t sweep = 1; sweep <= max_iters; ++sweep) {
      int32_t rc = gwo_kl_scale(out, n, m, mu, n, GWB_ROWS, out, st);
      if (rc) return rc;
      rc = gwo_kl_scale(out, n, m, nu, m, GWB_COLS, out, st);
      if (rc) return rc;
      if (!all_finite(out, len))
        return numerical(st, "sinkhorn", sweep,
                         "non-finite entries after scaling sweep");
      *iterations = sweep;
      *marginal_error = marginal_error_inf(out, n, m, mu, nu);
      if (*marginal_error <= tol) {
        *converged = 1;
        break;
      }
    }
    return set_status(st, GWB_OK, NULL, 0, "");
  }
  double* f = (double*)calloc((size_t)n, sizeof(double));
  double* g = (double*)calloc((size_t)m, sizeof(double));
  double* tmp = (double*)malloc(sizeof(double) * (size_t)(n > m ? n : m));
  int32_t rc = GWB_OK;
  for (int32_t sweep = 1; sweep <= max_iters; ++sweep) {
    for (int64_t i = 0; i < n; ++i)
      f[i] = log(mu[i]) - log_sum_exp(kernel + i, m, n, g);
    for (int64_t j = 0; j < m; ++j)
      g[j] = log(nu[j]) - log_sum_exp(kernel + (size_t)j * n, n, 1, f);
    for (int64_t j = 0; j < m; ++j)
      for (int64_t i = 0; i < n; ++i)
        out[IDX(i, j, n)] = exp(kernel[IDX(i, j, n)] + f[i] + g[j]);
    if (!all_finite(out, len)) {
      rc = numerical(st, "sinkhorn-log", sweep,
                     "non-finite entries after scaling sweep");
      break;
    }
    *iterations = sweep;
    *marginal_error = marginal_error_inf(out, n, m, mu, nu);
    if (*marginal_error <= tol) {
      *converged = 1;
      break;
    }
  }
  free(f);
  free(g);
  free(tmp);
  if (rc) return rc;
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* marginal_infeasibility: diagnostics.cpp:9-20. */
double gwo_marginal_infeasibility(const double* pi, int64_t n, int64_t m,
                                  const double* mu, const double* nu) {
  double col = 0.0, row = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += pi[IDX(i, j, n)];
    col += (s - nu[j]) * (s - nu[j]);
  }
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < m; ++j) s += pi[IDX(i, j, n)];
    row += (s - mu[i]) * (s - mu[i]);
  }
  return sqrt(col) / (double)m + sqrt(row) / (double)n;
}

/* split_gap: diagnostics.cpp:22-27. */
double gwo_split_gap(const double* pi, const double* w, int64_t n, int64_t m) {
  return fro_diff(pi, w, (size_t)n * (size_t)m);
}

/* spectral_norm by power iteration on D², solvers.cpp:113-129. */
static double spectral_norm(const double* d, int64_t n, double tol, int cap) {
  if (fro_norm(d, (size_t)n * (size_t)n) == 0.0) return 0.0;
  double* x = (double*)malloc(sizeof(double) * (size_t)n);
  double* t = (double*)malloc(sizeof(double) * (size_t)n);
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) x[i] = 1.0 / sqrt((double)n);
  double lambda = 0.0;
  for (int it = 0; it < cap; ++it) {
    matmul(d, x, t, n, n, 1);
    matmul(d, t, y, n, n, 1);
    const double est = fro_norm(y, (size_t)n);
    if (est == 0.0) {
      lambda = 0.0;
      break;
    }
    for (int64_t i = 0; i < n; ++i) x[i] = y[i] / est;
    const double conv = fabs(est - lambda);
    lambda = est;
    if (conv <= tol * (est > 1.0 ? est : 1.0)) break;
  }
  free(x);
  free(t);
  free(y);
  return sqrt(lambda);
}

/* lipschitz_bound: solvers.cpp:133-136. */
double gwo_lipschitz_bound(const double* dx, int64_t n, const double* dy,
                           int64_t m) {
  return spectral_norm(dx, n, 1e-10, 10000) * spectral_norm(dy, m, 1e-10, 10000);
}

/* hard_assignment: tasks.cpp:190-200 (strict '>' ⇒ lowest index on ties). */
void gwo_hard_assignment(const double* pi, int64_t n, int64_t m, int32_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t best = 0;
    for (int64_t j = 1; j < m; ++j)
      if (pi[IDX(i, j, n)] > pi[IDX(i, best, n)]) best = j;
    out[i] = (int32_t)best;
  }
}

/* coupling_entropy: diagnostics.cpp:44-53, column-major walk, 0 log 0 := 0. */
double gwo_coupling_entropy(const double* pi, int64_t n, int64_t m) {
  double h = 0.0;
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < n; ++i) {
      const double p = pi[IDX(i, j, n)];
      if (p > 0.0) h -= p * log(p);
    }
  return h;
}

/* alignment_accuracy: tasks.cpp:202-214. */
int32_t gwo_alignment_accuracy(const int32_t* pred, int64_t n_pred, const int32_t* gt,
                               int64_t n_gt, double* out, gwb_status* st) {
  if (n_pred < n_gt)
    return set_status(st, GWB_ERR_DIMENSION, NULL, 0,
                      "alignment_accuracy: prediction does not cover all ground-truth nodes");
  if (n_gt == 0) return set_status(st, GWB_ERR_INVALID, NULL, 0, "empty ground truth");
  int64_t hits = 0;
  for (int64_t i = 0; i < n_gt; ++i) hits += pred[i] == gt[i];
  *out = 100.0 * (double)hits / (double)n_gt;
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* write_coupling_csv: io.cpp:183-193 — "rows,cols\n", then every row as
 * "%.17g" values joined by ',' and ended by '\n'.  *len = bytes needed; the
 * text is written only if it fits in cap. */
int32_t gwo_format_coupling_csv(const double* pi, int64_t n, int64_t m, char* out, int64_t cap,
                                int64_t* len, gwb_status* st) {
  char buf[32];
  int64_t pos = 0;
  const int h = snprintf(buf, sizeof(buf), "%lld,%lld\n", (long long)n, (long long)m);
  if (out && pos + h <= cap) memcpy(out + pos, buf, (size_t)h);
  pos += h;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < m; ++j) {
      int k = 0;
      if (j) buf[k++] = ',';
      k += snprintf(buf + k, sizeof(buf) - (size_t)k, "%.17g", pi[IDX(i, j, n)]);
      if (j == m - 1) buf[k++] = '\n';
      if (out && pos + k <= cap) memcpy(out + pos, buf, (size_t)k);
      pos += k;
    }
  if (m == 0)
    for (int64_t i = 0; i < n; ++i) {
      if (out && pos + 1 <= cap) out[pos] = '\n';
      ++pos;
    }
  *len = pos;
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* validate(SolverConfig): types.cpp:176-188. */
int32_t gwo_validate_config(const gwb_config* c, gwb_status* st) {
  if (c->rho <= 0.0) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "rho must be positive");
  if (c->step <= 0.0) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "step must be positive");
  if (c->epsilon_reg <= 0.0) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "eps must be positive");
  if (c->inner_iters < 1) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "inner-iters must be >= 1");
  if (c->inner_tol <= 0.0) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "inner-tol must be positive");
  if (c->rel_tol <= 0.0) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "rel-tol must be positive");
  if (c->max_iters < 1) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "max-iters must be >= 1");
  if (c->perturbation < 0.0 || c->perturbation >= 1.0)
    return set_status(st, GWB_ERR_CONFIG, NULL, 0, "perturbation must lie in [0, 1)");
  if (c->switch_iters < 0) return set_status(st, GWB_ERR_CONFIG, NULL, 0, "switch-iters must be >= 0");
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* validate_inputs: types.cpp:190-202. */
static int32_t validate_inputs(int64_t n, int64_t m, int64_t mu_len,
                               int64_t nu_len, gwb_status* st) {
  if (n != mu_len)
    return set_status(st, GWB_ERR_DIMENSION, NULL, 0,
                      "D_X is %lldx%lld but mu has length %lld", (long long)n,
                      (long long)n, (long long)mu_len);
  if (m != nu_len)
    return set_status(st, GWB_ERR_DIMENSION, NULL, 0,
                      "D_Y is %lldx%lld but nu has length %lld", (long long)m,
                      (long long)m, (long long)nu_len);
  return GWB_OK;
}

static const char* algo_name(int32_t a) {
  switch (a) {
    case GWB_BAPG: return "bapg";
    case GWB_BPG: return "bpg";
    case GWB_EBPG: return "ebpg";
    case GWB_HBPG: return "hbpg";
    case GWB_FW: return "fw";
  }
  return "?";
}

typedef struct {
  gwb_record* trace;
  int32_t cap;
  int32_t count;
} trace_buf;

static int32_t push_record(trace_buf* tb, const gwb_record* r, gwb_status* st) {
  if (tb->count >= tb->cap)
    return set_status(st, GWB_ERR_CAPACITY, NULL, 0, "trace capacity %d exceeded",
                      tb->cap);
  tb->trace[tb->count++] = *r;
  return GWB_OK;
}

/* initial_coupling: solvers.cpp:41-50 (shape already fixed by the C-ABI). */
static void initial_coupling(const double* mu, int64_t n, const double* nu,
                             int64_t m, const double* initial, double* pi) {
  if (initial) {
    memcpy(pi, initial, sizeof(double) * (size_t)n * (size_t)m);
  } else {
    gwo_product_coupling(mu, n, nu, m, pi, NULL);
  }
}

/* simplex_project: projections.cpp:36-53 — Euclidean projection of v onto
 * {x ≥ 0, Σx = s} by a descending sort and the running threshold. */
static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}

static void simplex_project(const double* v, int64_t n, int64_t stride, double s, double* u,
                            double* out) {
  for (int64_t j = 0; j < n; ++j) u[j] = v[j * stride];
  qsort(u, (size_t)n, sizeof(double), cmp_desc);
  double cumsum = 0.0, theta = u[0] - s;
  for (int64_t j = 0; j < n; ++j) {
    cumsum += u[j];
    const double cand = (cumsum - s) / (double)(j + 1);
    if (u[j] - cand > 0.0) theta = cand;
  }
  for (int64_t j = 0; j < n; ++j) {
    const double x = v[j * stride] - theta;
    out[j * stride] = x > 0.0 ? x : 0.0;
  }
}

/* euclid_project: projections.cpp:55-77, column-major pi. */
static void euclid_project(const double* pi, int64_t n, int64_t m, const double* target,
                           int axis, double* out) {
  const int64_t len = axis == GWB_ROWS ? m : n;
  double* u = (double*)malloc(sizeof(double) * (size_t)(len > 0 ? len : 1));
  if (axis == GWB_ROWS) {
    for (int64_t i = 0; i < n; ++i) simplex_project(pi + i, m, n, target[i], u, out + i);
  } else {
    for (int64_t j = 0; j < m; ++j)
      simplex_project(pi + j * n, n, 1, target[j], u, out + j * n);
  }
  free(u);
}

/* dykstra_project: projections.cpp:165-187 — Dykstra's alternating Euclidean
 * projections onto C1 (rows) and C2 (columns) with correction terms p, q;
 * stops once marginal_error_inf(x) ≤ tol, else runtime_error. */
int32_t gwo_dykstra_project(const double* pi, int64_t n, int64_t m, const double* mu,
                            const double* nu, double tol, int32_t max_iters, double* out,
                            int32_t* sweeps, gwb_status* st) {
  const size_t len = (size_t)n * (size_t)m;
  double* p = (double*)calloc(len, sizeof(double));
  double* q = (double*)calloc(len, sizeof(double));
  double* v = (double*)malloc(sizeof(double) * len);
  double* y = (double*)malloc(sizeof(double) * len);
  memcpy(out, pi, sizeof(double) * len);
  double err = 0.0;
  int32_t rc = GWB_ERR_RUNTIME;
  *sweeps = 0;
  for (int32_t sweep = 1; sweep <= max_iters; ++sweep) {
    for (size_t k = 0; k < len; ++k) v[k] = out[k] + p[k];
    euclid_project(v, n, m, mu, GWB_ROWS, y);
    for (size_t k = 0; k < len; ++k) p[k] = v[k] - y[k];
    for (size_t k = 0; k < len; ++k) v[k] = y[k] + q[k];
    euclid_project(v, n, m, nu, GWB_COLS, out);
    for (size_t k = 0; k < len; ++k) q[k] = v[k] - out[k];
    *sweeps = sweep;
    err = marginal_error_inf(out, n, m, mu, nu);
    if (err <= tol) {
      rc = GWB_OK;
      break;
    }
  }
  free(p);
  free(q);
  free(v);
  free(y);
  if (rc != GWB_OK)
    return set_status(st, GWB_ERR_RUNTIME, NULL, 0,
                      "dykstra_project did not converge in %d sweeps; final constraint "
                      "violation %g", max_iters, err);
  return set_status(st, GWB_OK, NULL, 0, "");
}

/* luo_tseng_residual: diagnostics.cpp:33-42 — ‖π − Proj_Π(μ,ν)(π + D_X π D_Y)‖_F
 * with the Dykstra projection at dykstra_tol (default 1e-8, 10000 sweeps). */
int32_t gwo_luo_tseng_residual(const double* dx, int64_t n, const double* dy, int64_t m,
                               const double* pi, const double* mu, const double* nu,
                               double dykstra_tol, double* out, gwb_status* st) {
  const size_t len = (size_t)n * (size_t)m;
  double* shifted = (double*)malloc(sizeof(double) * len);
  double* proj = (double*)malloc(sizeof(double) * len);
  gwo_structure_product(dx, n, dy, m, pi, shifted);
  for (size_t k = 0; k < len; ++k) shifted[k] = pi[k] + shifted[k];
  int32_t sweeps = 0;
  const int32_t rc = gwo_dykstra_project(shifted, n, m, mu, nu, dykstra_tol, 10000, proj,
                                         &sweeps, st);
  if (rc == GWB_OK) *out = fro_diff(pi, proj, len);
  free(shifted);
  free(proj);
  return rc;
}

/* The optional per-record residual (solvers.cpp:202-204, 278-280, 348-350). */
static int32_t record_residual(const gwb_config* cfg, const double* dx, int64_t n,
                               const double* dy, int64_t m, const double* pi,
                               const double* mu, const double* nu, gwb_record* rec,
                               gwb_status* st) {
  if (!cfg->record_residual) return GWB_OK;
  rec->has_residual = 1;
  return gwo_luo_tseng_residual(dx, n, dy, m, pi, mu, nu, 1e-8, &rec->residual, st);
}

/* bapg_solve, entropy geometry: solvers.cpp:138-217. */
static int32_t bapg(const gwb_config* cfg, const double* dx, int64_t n,
                    const double* dy, int64_t m, const double* mu,
                    const double* nu, const double* initial, double* out_final,
                    double* out_pi, double* out_w, trace_buf* tb,
                    int32_t* converged, int32_t* iters_used, gwb_status* st) {
  const int entropy = cfg->geometry == GWB_ENTROPY;
  const size_t len = (size_t)n * (size_t)m;
  double* pi = (double*)malloc(sizeof(double) * len);
  double* w = (double*)malloc(sizeof(double) * len);
  double* w_next = (double*)malloc(sizeof(double) * len);
  double* e = (double*)malloc(sizeof(double) * len);
  double* avg = (double*)malloc(sizeof(double) * len);
  int32_t rc = GWB_OK;
  initial_coupling(mu, n, nu, m, initial, pi);
  for (size_t k = 0; entropy && k < len; ++k) {
    if (!(pi[k] > 0.0)) {
      rc = set_status(st, GWB_ERR_CONFIG, NULL, 0,
                      "bapg entropy geometry requires a strictly positive "
                      "initialization (the product coupling qualifies)");
      goto done;
    }
  }
  if (entropy) {
    rc = gwo_kl_scale(pi, n, m, nu, m, GWB_COLS, w, st); /* :152-153 */
    if (rc) goto done;
  } else {
    euclid_project(pi, n, m, nu, GWB_COLS, w);
  }
  {
    const double t0 = now_seconds();
    int32_t iter = 0;
    *converged = 0;
    while (iter < cfg->max_iters) {
      ++iter;
      if (!entropy) { /* quadratic geometry, :179-182 */
        gwo_structure_product(dx, n, dy, m, w, e);
        for (size_t k = 0; k < len; ++k) e[k] = w[k] + e[k] / cfg->rho;
        euclid_project(e, n, m, mu, GWB_ROWS, pi);
        gwo_structure_product(dx, n, dy, m, pi, e);
        for (size_t k = 0; k < len; ++k) e[k] = pi[k] + e[k] / cfg->rho;
        euclid_project(e, n, m, nu, GWB_COLS, w_next);
        goto checked;
      }
      /* half-step a, :164-170 */
      gwo_structure_product(dx, n, dy, m, w, e);
      double emax = -INFINITY;
      for (size_t k = 0; k < len; ++k) {
        e[k] = e[k] / cfg->rho;
        if (e[k] > emax) emax = e[k];
      }
      if (emax > 700.0) {
        rc = numerical(st, "bapg", iter, "exp overflow; increase rho");
        goto done;
      }
      for (size_t k = 0; k < len; ++k) e[k] = w[k] * exp(e[k]);
      rc = gwo_kl_scale(e, n, m, mu, n, GWB_ROWS, pi, st);
      if (rc == GWB_ERR_ZERO_SUM) { /* :184-186 */
        char what[512];
        snprintf(what, sizeof(what), "%s", st->message);
        rc = numerical(st, "bapg", iter, what);
      }
      if (rc) goto done;
      /* half-step b, :171-177 */
      gwo_structure_product(dx, n, dy, m, pi, e);
      emax = -INFINITY;
      for (size_t k = 0; k < len; ++k) {
        e[k] = e[k] / cfg->rho;
        if (e[k] > emax) emax = e[k];
      }
      if (emax > 700.0) {
        rc = numerical(st, "bapg", iter, "exp overflow; increase rho");
        goto done;
      }
      for (size_t k = 0; k < len; ++k) e[k] = pi[k] * exp(e[k]);
      rc = gwo_kl_scale(e, n, m, nu, m, GWB_COLS, w_next, st);
      if (rc == GWB_ERR_ZERO_SUM) {
        char what[512];
        snprintf(what, sizeof(what), "%s", st->message);
        rc = numerical(st, "bapg", iter, what);
      }
      if (rc) goto done;
    checked:
      if (!all_finite(pi, len) || !all_finite(w_next, len)) { /* :187-189 */
        rc = numerical(st, "bapg", iter, "non-finite iterate");
        goto done;
      }
      const double rel_change = fro_diff(w_next, w, len) / fro_norm(w, len);
      double* tmp = w;
      w = w_next;
      w_next = tmp;
      for (size_t k = 0; k < len; ++k) avg[k] = 0.5 * (pi[k] + w[k]);
      gwb_record rec;
      memset(&rec, 0, sizeof(rec));
      rec.iter = iter;
      gwo_gw_objective(dx, n, dy, m, avg, n, m, &rec.objective, NULL);
      rec.marginal_infeasibility = gwo_marginal_infeasibility(avg, n, m, mu, nu);
      rec.split_gap = gwo_split_gap(pi, w, n, m);
      rec.rel_change = rel_change;
      rec.elapsed_seconds = now_seconds() - t0;
      rc = record_residual(cfg, dx, n, dy, m, avg, mu, nu, &rec, st);
      if (rc) goto done;
      rc = push_record(tb, &rec, st);
      if (rc) goto done;
      if (rel_change <= cfg->rel_tol) {
        *converged = 1;
        break;
      }
    }
    *iters_used = iter;
  }
  for (size_t k = 0; k < len; ++k) out_final[k] = 0.5 * (pi[k] + w[k]);
  if (out_pi) memcpy(out_pi, pi, sizeof(double) * len);
  if (out_w) memcpy(out_w, w, sizeof(double) * len);
  rc = set_status(st, GWB_OK, NULL, 0, "");
done:
  free(pi);
  free(w);
  free(w_next);
  free(e);
  free(avg);
  return rc;
}

/* ebpg_solve: solvers.cpp:295-363. */
static int32_t ebpg(const gwb_config* cfg, const double* dx, int64_t n,
                    const double* dy, int64_t m, const double* mu,
                    const double* nu, const double* initial, double* out_final,
                    trace_buf* tb, int32_t* converged, int32_t* iters_used,
                    gwb_status* st) {
  const size_t len = (size_t)n * (size_t)m;
  double* pi = (double*)malloc(sizeof(double) * len);
  double* e = (double*)malloc(sizeof(double) * len);
  double* next = (double*)malloc(sizeof(double) * len);
  int32_t rc = GWB_OK;
  initial_coupling(mu, n, nu, m, initial, pi);
  const double t0 = now_seconds();
  int32_t iter = 0;
  *converged = 0;
  while (iter < cfg->max_iters) {
    ++iter;
    gwo_structure_product(dx, n, dy, m, pi, e);
    const double scale = 2.0 / cfg->epsilon_reg;
    double emax = -INFINITY;
    for (size_t k = 0; k < len; ++k) {
      e[k] = scale * e[k];
      if (e[k] > emax) emax = e[k];
    }
    for (size_t k = 0; k < len; ++k) e[k] -= emax;
    int32_t sweeps = 0, conv = 0;
    double merr = 0.0;
    if (cfg->log_domain) {
      rc = gwo_sinkhorn_project(e, n, m, mu, nu, cfg->inner_tol,
                                cfg->inner_iters, 1, next, &sweeps, &merr,
                                &conv, st);
    } else {
      for (size_t k = 0; k < len; ++k) e[k] = exp(e[k]);
      int row_dead = 0, col_dead = 0;
      for (int64_t i = 0; i < n && !row_dead; ++i) {
        double mx = -INFINITY;
        for (int64_t j = 0; j < m; ++j)
          if (e[IDX(i, j, n)] > mx) mx = e[IDX(i, j, n)];
        if (mx <= 0.0) row_dead = 1;
      }
      for (int64_t j = 0; j < m && !col_dead; ++j) {
        double mx = -INFINITY;
        for (int64_t i = 0; i < n; ++i)
          if (e[IDX(i, j, n)] > mx) mx = e[IDX(i, j, n)];
        if (mx <= 0.0) col_dead = 1;
      }
      if (row_dead || col_dead) {
        rc = numerical(st, "ebpg", iter,
                       "kernel line underflowed to zero; increase eps or "
                       "enable the log-domain solver");
        goto done;
      }
      for (size_t k = 0; k < len; ++k)
        if (e[k] < 1e-300) e[k] = 1e-300;
      rc = gwo_sinkhorn_project(e, n, m, mu, nu, cfg->inner_tol,
                                cfg->inner_iters, 0, next, &sweeps, &merr,
                                &conv, st);
    }
    if (rc == GWB_ERR_ZERO_SUM) {
      char what[512];
      snprintf(what, sizeof(what), "%s", st->message);
      rc = numerical(st, "ebpg", iter, what);
    }
    if (rc) goto done;
    const double rel_change = fro_diff(next, pi, len) / fro_norm(pi, len);
    double* tmp = pi;
    pi = next;
    next = tmp;
    gwb_record rec;
    memset(&rec, 0, sizeof(rec));
    rec.iter = iter;
    gwo_gw_objective(dx, n, dy, m, pi, n, m, &rec.objective, NULL);
    rec.marginal_infeasibility = gwo_marginal_infeasibility(pi, n, m, mu, nu);
    rec.rel_change = rel_change;
    rec.elapsed_seconds = now_seconds() - t0;
    rc = record_residual(cfg, dx, n, dy, m, pi, mu, nu, &rec, st);
    if (rc) goto done;
    rc = push_record(tb, &rec, st);
    if (rc) goto done;
    if (rel_change <= cfg->rel_tol) {
      *converged = 1;
      break;
    }
  }
  *iters_used = iter;
  memcpy(out_final, pi, sizeof(double) * len);
  rc = set_status(st, GWB_OK, NULL, 0, "");
done:
  free(pi);
  free(e);
  free(next);
  return rc;
}

/* bpg_solve: solvers.cpp:219-293. */
static int32_t bpg(const gwb_config* cfg, const double* dx, int64_t n,
                   const double* dy, int64_t m, const double* mu,
                   const double* nu, const double* initial, double* out_final,
                   trace_buf* tb, int32_t* converged, int32_t* iters_used,
                   gwb_status* st) {
  const size_t len = (size_t)n * (size_t)m;
  const double lipschitz = gwo_lipschitz_bound(dx, n, dy, m);
  if (lipschitz > 0.0 && cfg->step > 1.0 / lipschitz && !cfg->quiet) {
    fprintf(stderr,
            "bpg: step %g exceeds sigma/L_f = %g; descent is not "
            "guaranteed at this step size\n",
            cfg->step, 1.0 / lipschitz);
  }
  double* pi = (double*)malloc(sizeof(double) * len);
  double* e = (double*)malloc(sizeof(double) * len);
  double* next = (double*)malloc(sizeof(double) * len);
  int32_t rc = GWB_OK;
  initial_coupling(mu, n, nu, m, initial, pi);
  const double uniform_mass = 1.0 / (double)(n * m);
  const double t0 = now_seconds();
  int32_t iter = 0;
  *converged = 0;
  while (iter < cfg->max_iters) {
    ++iter;
    gwo_structure_product(dx, n, dy, m, pi, e);
    const double scale = 2.0 * cfg->step;
    double emax = -INFINITY;
    for (size_t k = 0; k < len; ++k) {
      e[k] = scale * e[k];
      if (e[k] > emax) emax = e[k];
    }
    if (emax > 700.0) {
      rc = numerical(st, "bpg", iter, "exp overflow; reduce step");
      goto done;
    }
    for (size_t k = 0; k < len; ++k) {
      const double v = pi[k] * exp(e[k]);
      e[k] = v < 1e-300 ? 1e-300 : v;
    }
    int32_t sweeps = 0, conv = 0;
    double merr = 0.0;
    rc = gwo_sinkhorn_project(e, n, m, mu, nu, cfg->inner_tol, cfg->inner_iters,
                              0, next, &sweeps, &merr, &conv, st);
    if (rc == GWB_ERR_ZERO_SUM || rc == GWB_ERR_NUMERICAL) {
      char what[512];
      snprintf(what, sizeof(what), "%s", st->message);
      rc = numerical(st, "bpg", iter, what);
    }
    if (rc) goto done;
    if (cfg->perturbation > 0.0) {
      for (size_t k = 0; k < len; ++k)
        next[k] = (1.0 - cfg->perturbation) * next[k] +
                  cfg->perturbation * uniform_mass;
    }
    const double rel_change = fro_diff(next, pi, len) / fro_norm(pi, len);
    double* tmp = pi;
    pi = next;
    next = tmp;
    gwb_record rec;
    memset(&rec, 0, sizeof(rec));
    rec.iter = iter;
    gwo_gw_objective(dx, n, dy, m, pi, n, m, &rec.objective, NULL);
    rec.marginal_infeasibility = gwo_marginal_infeasibility(pi, n, m, mu, nu);
    rec.rel_change = rel_change;
    rec.elapsed_seconds = now_seconds() - t0;
    rc = record_residual(cfg, dx, n, dy, m, pi, mu, nu, &rec, st);
    if (rc) goto done;
    rc = push_record(tb, &rec, st);
    if (rc) goto done;
    if (rel_change <= cfg->rel_tol) {
      *converged = 1;
      break;
    }
  }
  *iters_used = iter;
  memcpy(out_final, pi, sizeof(double) * len);
  rc = set_status(st, GWB_OK, NULL, 0, "");
done:
  free(pi);
  free(e);
  free(next);
  return rc;
}

/* hbpg_solve: solvers.cpp:365-426. */
static int32_t hbpg(const gwb_config* cfg, const double* dx, int64_t n,
                    const double* dy, int64_t m, const double* mu,
                    const double* nu, const double* initial, double* out_final,
                    trace_buf* tb, int32_t* converged, int32_t* iters_used,
                    gwb_status* st) {
  const size_t len = (size_t)n * (size_t)m;
  double* start = (double*)malloc(sizeof(double) * len);
  double* warm = (double*)malloc(sizeof(double) * len);
  initial_coupling(mu, n, nu, m, initial, start);
  int32_t rc = GWB_OK;
  const int32_t budget1 =
      cfg->switch_iters < cfg->max_iters ? cfg->switch_iters : cfg->max_iters;
  int32_t used1 = 0, conv1 = 0, have_warm = 0;
  double elapsed1 = 0.0;
  if (budget1 >= 1) {
    gwb_config c1 = *cfg;
    c1.algorithm = GWB_EBPG;
    c1.max_iters = budget1;
    const int32_t first = tb->count;
    rc = ebpg(&c1, dx, n, dy, m, mu, nu, start, warm, tb, &conv1, &used1, st);
    if (rc) goto done;
    have_warm = 1;
    for (int32_t k = first; k < tb->count; ++k) tb->trace[k].phase = 1;
    if (tb->count > 0) elapsed1 = tb->trace[tb->count - 1].elapsed_seconds;
  }
  {
    const int32_t budget2 = cfg->max_iters - used1;
    if (budget2 < 1) {
      memcpy(out_final, warm, sizeof(double) * len);
      *converged = conv1;
      *iters_used = used1;
      rc = set_status(st, GWB_OK, NULL, 0, "");
      goto done;
    }
    gwb_config c2 = *cfg;
    c2.algorithm = GWB_BPG;
    c2.max_iters = budget2;
    const int32_t first = tb->count;
    int32_t conv2 = 0, used2 = 0;
    rc = bpg(&c2, dx, n, dy, m, mu, nu, have_warm ? warm : start, out_final, tb,
             &conv2, &used2, st);
    if (rc) goto done;
    for (int32_t k = first; k < tb->count; ++k) {
      tb->trace[k].phase = 2;
      tb->trace[k].iter += used1;
      tb->trace[k].elapsed_seconds += elapsed1;
    }
    *converged = conv2;
    *iters_used = used1 + used2;
  }
done:
  free(start);
  free(warm);
  return rc;
}

/* solve dispatch: solvers.cpp:499-515, with the per-solver preamble
 * require_algorithm → validate → validate_inputs (solvers.cpp:141-143). */
int32_t gwo_solve(const gwb_config* cfg, const double* dx, int64_t n,
                  const double* dy, int64_t m, const double* mu,
                  const double* nu, const double* initial, double* out_final,
                  double* out_pi, double* out_w, gwb_record* trace,
                  int32_t trace_cap, int32_t* n_records, int32_t* converged,
                  int32_t* iterations_used, gwb_status* st) {
  int32_t rc = gwo_validate_config(cfg, st);
  if (rc) return rc;
  rc = validate_inputs(n, m, n, m, st);
  if (rc) return rc;
  trace_buf tb = {trace, trace_cap, 0};
  *n_records = 0;
  *converged = 0;
  *iterations_used = 0;
  switch (cfg->algorithm) {
    case GWB_BAPG:
      rc = bapg(cfg, dx, n, dy, m, mu, nu, initial, out_final, out_pi, out_w,
                &tb, converged, iterations_used, st);
      break;
    case GWB_EBPG:
      rc = ebpg(cfg, dx, n, dy, m, mu, nu, initial, out_final, &tb, converged,
                iterations_used, st);
      break;
    case GWB_BPG:
      rc = bpg(cfg, dx, n, dy, m, mu, nu, initial, out_final, &tb, converged,
               iterations_used, st);
      break;
    case GWB_HBPG:
      rc = hbpg(cfg, dx, n, dy, m, mu, nu, initial, out_final, &tb, converged,
                iterations_used, st);
      break;
    default:
      rc = set_status(st, GWB_ERR_UNSUPPORTED, NULL, 0,
                      "algorithm '%s' is outside the oracle scope",
                      algo_name(cfg->algorithm));
  }
  *n_records = tb.count;
  return rc;
}
