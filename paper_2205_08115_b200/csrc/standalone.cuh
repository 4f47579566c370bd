// standalone.cuh — device implementations of the single-shot entry points
// on the path (gw_objective, product_coupling, lipschitz_bound, kl_scale,
// Sinkhorn, diagnostics, hard_assignment), the eBPG/BPG/hBPG solvers and the
// batched small-problem BAPG.  Errors are raised through api_* (capi.cu).
#pragma once

#include <cstdint>
#include <functional>
#include <string>

#include "../../include/gwb.h"
#include "kernels.cuh"

namespace gwb {

[[noreturn]] void api_fail(int32_t code, const std::string& msg);
[[noreturn]] void api_numerical(const char* solver, int iter, const std::string& detail);
[[noreturn]] void api_zero_sum(int axis, int64_t index);
int api_device();

double device_gw_objective(const double* dx, int64_t n, const double* dy, int64_t m,
                           const double* pi);
// Device-resident forms used by the session readout.
double gw_objective_dev(const float* Dx, int64_t ldn, const float* Dy, int64_t ldm,
                        const float* P, int64_t n, int64_t m, cudaStream_t s);
double coupling_entropy_dev(const double* pi_dev, int64_t len, cudaStream_t s);
// G (row-major fp32, ld = ldm) = D_X·P·D_Y, 3xTF32 tcgen05 chain; synchronous.
void structure_product_dev(const float* Dx, int64_t ldn, const float* Dy, int64_t ldm,
                           const float* P, int64_t n, int64_t m, float* G, cudaStream_t s);

// Dykstra projection onto Π(μ, ν) (projections.cpp:165-187) and the
// Luo-Tseng residual (diagnostics.cpp:33-42), residual.cu.  x: column-major
// fp64 n×m on the device, projected in place.
struct DykstraOutcome {
  bool converged = false;
  int sweeps = 0;
  double err = 0.0;
};
DykstraOutcome dykstra_dev(double* x, int64_t n, int64_t m, const double* mu64,
                           const double* nu64, double tol, int max_iters, cudaStream_t s);
// runtime_error "dykstra_project did not converge in <k> sweeps; …"
[[noreturn]] void dykstra_fail(int max_iters, double err);
// ‖π − Proj(π + D_X π D_Y)‖_F for a device column-major fp64 π; D_X, D_Y
// row-major fp32.  Raises via dykstra_fail on non-convergence (10000 sweeps).
double luo_tseng_residual_dev(const float* Dx, int64_t ldn, const float* Dy, int64_t ldm,
                              const double* pi, int64_t n, int64_t m, const double* mu64,
                              const double* nu64, double tol, cudaStream_t s);
// write_coupling_csv (io.cpp:183-193) of a device column-major fp64 n×m
// coupling, formatted on the device ("%.17g") and streamed to `sink` in
// row blocks; returns the total byte count (csv.cu).
int64_t coupling_csv_dev(const double* pi, int64_t n, int64_t m, cudaStream_t s,
                         const std::function<void(const char*, int64_t)>& sink);
void device_coupling_csv(const double* pi, int64_t n, int64_t m,
                         const std::function<void(const char*, int64_t)>& sink,
                         int64_t* total);
void device_dykstra_project(const double* pi, int64_t n, int64_t m, const double* mu,
                            const double* nu, double tol, int32_t max_iters, double* out);
double device_luo_tseng_residual(const double* dx, int64_t n, const double* dy, int64_t m,
                                 const double* pi, const double* mu, const double* nu,
                                 double tol);
double device_coupling_entropy(const double* pi, int64_t n, int64_t m);
void device_product_coupling(const double* mu, int64_t n, const double* nu, int64_t m,
                             double* out);
double device_lipschitz_bound(const double* dx, int64_t n, const double* dy, int64_t m);
double device_lipschitz_bound_graphs(const GraphInput& g, int64_t n, int64_t m);
void device_kl_scale(const double* pi, int64_t n, int64_t m, const double* target, int32_t axis,
                     double* out);
void device_sinkhorn(const double* kernel, int64_t n, int64_t m, const double* mu,
                     const double* nu, double tol, int32_t max_iters, int32_t log_domain,
                     double* out, int32_t* iterations, double* marginal_error,
                     int32_t* converged);
double device_marginal_infeasibility(const double* pi, int64_t n, int64_t m, const double* mu,
                                     const double* nu);
double device_split_gap(const double* pi, const double* w, int64_t n, int64_t m);
void device_hard_assignment(const double* pi, int64_t n, int64_t m, int32_t* out);

// eBPG / BPG / hBPG (solvers.cpp:219-426) on the device.
void bregman_solve(const gwb_config* cfg, int32_t algo, const double* dx, int64_t n,
                   const double* dy, int64_t m, const double* mu, const double* nu,
                   const double* initial, gwb_observer observer, void* user, double* out_final,
                   gwb_record* trace, int32_t trace_cap, int32_t* n_records, int32_t* converged,
                   int32_t* iterations_used, const GraphInput* graphs = nullptr);

// Row-sharded eBPG / BPG / hBPG (bregman.cu): the chain runs on this rank's
// rows of D_X with caller-issued all-gathers of Vᵀ and G between phases;
// the Sinkhorn state and π are replicated (dist.py orchestrates).
struct BregShard;
BregShard* bshard_create(const gwb_config& cfg, int algo, int64_t n, int64_t m, int world, int rank,
                         int device, cudaStream_t s);
void bshard_destroy(BregShard* b);
void bshard_layout(BregShard* b, int64_t* rows_per_shard, int64_t* row_begin, int64_t* rows_valid,
                   int64_t* padded_rows, int64_t* ld);
void bshard_comm_layout(BregShard* b, int32_t* planes, int32_t* esize, int64_t* vt_bytes);
void bshard_set_comm(BregShard* b, void* vt, float* g);
void bshard_load(BregShard* b, const float* dx_rows, int64_t ldx, const float* dy, int64_t ldy,
                 const double* mu, const double* nu, int64_t m);
void bshard_phase(BregShard* b, int k, int op);
void bshard_status(BregShard* b, int32_t* done, int32_t* iter, int32_t* flags, int32_t* converged);
void* bshard_stream(BregShard* b);
void bshard_finish(BregShard* b, double* out_final, gwb_record* trace, int32_t trace_cap,
                   int32_t* n_records, int32_t* converged, int32_t* iterations_used);

// Batched BAPG over independent small problems (config 5).
void device_bapg_batched(const gwb_config* cfg, int64_t batch, const double* dx, int64_t n,
                         const double* dy, int64_t m, const double* mu, const double* nu,
                         double* out_final, double* out_pi, double* out_w, gwb_record* trace,
                         int32_t trace_cap, int32_t* n_records, int32_t* converged,
                         int32_t* iterations_used, bool name_problem = true, int device = -1,
                         int64_t index_base = 0, double* kernel_ms = nullptr);
// gwb_batched_last_kernel_ms's record (device time of the last batched call).
void set_batched_last(double ms, int64_t problems);

}  // namespace gwb
