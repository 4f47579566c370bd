/*
 * gw_oracle.h — CPU restatement of the reference solver path, used ONLY as
 * a test checker (tests/, __graft_entry__.smoke(), bench.py cpu_baseline).
 * It is never linked into or called by the product library.
 *
 * Pinning: the restatement is checked against (1) the reference's own
 * known-answer tests (proj/tests/test_core.cpp:56-89, SPEC.md prose KATs
 * listed in SURVEY.md §8c) and (2) the reference's own translation units
 * compiled here against oracle/eigen_lite (oracle/_ref/libgwref.so) on
 * seeded instances — see tests/test_oracle_*.py.
 *
 * Layout: column-major fp64 everywhere (Eigen MatrixXd, types.hpp:13).
 * Status/config/record structs are the C-ABI's (include/gwb.h).
 */
#ifndef GW_ORACLE_H_
#define GW_ORACLE_H_

#include <stdint.h>

#include "../include/gwb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Optional BLAS: ILP64 cblas_dgemm (e.g. numpy's scipy_cblas_dgemm64_).
 * NULL restores the built-in loop GEMM. */
typedef void (*gwo_cblas_dgemm_fn)(int, int, int, int64_t, int64_t, int64_t,
                                   double, const double*, int64_t,
                                   const double*, int64_t, double, double*,
                                   int64_t);
void gwo_set_dgemm(gwo_cblas_dgemm_fn fn);

void gwo_structure_product(const double* dx, int64_t n, const double* dy,
                           int64_t m, const double* pi, double* out);
int32_t gwo_gw_objective(const double* dx, int64_t n, const double* dy,
                         int64_t m, const double* pi, int64_t rows,
                         int64_t cols, double* out, gwb_status* st);
int32_t gwo_product_coupling(const double* mu, int64_t n, const double* nu,
                             int64_t m, double* out, gwb_status* st);
int32_t gwo_kl_scale(const double* pi, int64_t n, int64_t m,
                     const double* target, int64_t target_len, int32_t axis,
                     double* out, gwb_status* st);
int32_t gwo_sinkhorn_project(const double* kernel, int64_t n, int64_t m,
                             const double* mu, const double* nu, double tol,
                             int32_t max_iters, int32_t log_domain,
                             double* out, int32_t* iterations,
                             double* marginal_error, int32_t* converged,
                             gwb_status* st);
double gwo_marginal_infeasibility(const double* pi, int64_t n, int64_t m,
                                  const double* mu, const double* nu);
double gwo_split_gap(const double* pi, const double* w, int64_t n, int64_t m);
double gwo_lipschitz_bound(const double* dx, int64_t n, const double* dy,
                           int64_t m);
void gwo_hard_assignment(const double* pi, int64_t n, int64_t m, int32_t* out);
/* coupling_entropy, diagnostics.cpp:44-53. */
double gwo_coupling_entropy(const double* pi, int64_t n, int64_t m);
/* alignment_accuracy, tasks.cpp:202-214 (returns a gwb_code; *out in %). */
int32_t gwo_alignment_accuracy(const int32_t* pred, int64_t n_pred, const int32_t* gt,
                               int64_t n_gt, double* out, gwb_status* st);
/* dykstra_project, projections.cpp:165-187; luo_tseng_residual,
 * diagnostics.cpp:33-42 (gwb codes; GWB_ERR_RUNTIME on non-convergence). */
int32_t gwo_dykstra_project(const double* pi, int64_t n, int64_t m, const double* mu,
                            const double* nu, double tol, int32_t max_iters, double* out,
                            int32_t* sweeps, gwb_status* st);
int32_t gwo_luo_tseng_residual(const double* dx, int64_t n, const double* dy, int64_t m,
                               const double* pi, const double* mu, const double* nu,
                               double dykstra_tol, double* out, gwb_status* st);
/* write_coupling_csv, io.cpp:183-193 (%.17g). */
int32_t gwo_format_coupling_csv(const double* pi, int64_t n, int64_t m, char* out, int64_t cap,
                                int64_t* len, gwb_status* st);
int32_t gwo_validate_config(const gwb_config* cfg, gwb_status* st);
int32_t gwo_solve(const gwb_config* cfg, const double* dx, int64_t n,
                  const double* dy, int64_t m, const double* mu,
                  const double* nu, const double* initial, double* out_final,
                  double* out_pi, double* out_w, gwb_record* trace,
                  int32_t trace_cap, int32_t* n_records, int32_t* converged,
                  int32_t* iterations_used, gwb_status* st);

#ifdef __cplusplus
}
#endif

#endif /* GW_ORACLE_H_ */
