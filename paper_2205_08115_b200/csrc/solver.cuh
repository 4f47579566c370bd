// solver.cuh — device-side BAPG engine: workspace in HBM, the per-iteration
// launch sequence (2×2 GEMMs + row/column projection passes + finalize),
// CUDA-graph capture of iteration chunks, device-side stop rule, and the
// fp64 boundary conversions.  Reference loop: bapg_solve,
// proj/src/solvers.cpp:138-217.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <functional>
#include <vector>

#include "../../include/gwb.h"
#include "gemm.cuh"
#include "kernels.cuh"
#include "skinny.cuh"
#include "sparse.cuh"

namespace gwb {

struct CudaError : std::exception {
  std::string msg;
  explicit CudaError(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};

void check_cuda(cudaError_t e, const char* what);
// Keep stream-ordered allocations cached in the device's default pool.
void pool_keep(int device);
#define GWB_CUDA(x) ::gwb::check_cuda((x), #x)

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Host-side view of one finished trace record (IterationRecord fields).
struct HostRecord {
  double objective, marginal_infeasibility, split_gap, rel_change, elapsed;
};

// run_cell's readout of the final coupling (experiment.cpp:169-195).
struct Readout {
  double objective = 0, marginal_infeasibility = 0, entropy = 0, split_gap = 0, accuracy = 0;
  double residual = 0;  // NaN when Dykstra does not converge (experiment.cpp:177-182)
};

class BapgEngine {
 public:
  // n×n D_X, m×m D_Y; `precision` resolved to PREC_TF32 or PREC_3XTF32.
  BapgEngine(int device, int64_t n, int64_t m, double rho, int precision, int max_iters,
             cudaStream_t stream);
  ~BapgEngine();
  BapgEngine(const BapgEngine&) = delete;
  BapgEngine& operator=(const BapgEngine&) = delete;

  int64_t n() const { return n_; }
  int64_t m() const { return m_; }
  cudaStream_t stream() const { return stream_; }

  // Inputs from host fp64 column-major (symmetric D: layout-free) or from
  // device fp32 row-major.
  void load_host(const double* dx, const double* dy, const double* mu, const double* nu);
  // D_X, D_Y = adjacency_distance of host edge lists, built on the device.
  void load_graphs(const GraphInput& g, const double* mu, const double* nu);
  void load_device(const float* dx, int64_t ldx, const float* dy, int64_t ldy, const float* mu,
                   const float* nu);
  // π0 = μνᵀ or `initial` (host fp64 col-major); w0 = kl_scale(π0, ν, Cols)
  // computed by the caller in fp64 and passed as w0 (nullable ⇒ w0 = π0,
  // exact for the product coupling).
  void reset(const double* w0_host);
  // Enqueues `iters` iterations (no host sync); returns kernel launches.
  int64_t iterate(int iters, double rel_tol, bool use_graph);
  // Polls convergence between chunks; returns when done or all enqueued.
  void run(int max_iters, double rel_tol);
  // Host-stepped solve (observer / record_residual slow path): one
  // iteration per step, after(k, status) once iteration k has executed;
  // stops at convergence, max_iters or a device flag (returned status).
  DevStatus run_stepped(int max_iters, double rel_tol,
                        const std::function<void(int, const DevStatus&)>& after);
  // luo_tseng_residual (diagnostics.cpp:33-42) of the current average
  // ½(π + w) (solvers.cpp:202-204); raises if Dykstra does not converge.
  double residual_of_average(double dykstra_tol);
  // write_coupling_csv of the final coupling ½(π + w) (K8 fix-up first),
  // formatted on the device and streamed to `sink`; returns the byte count.
  int64_t final_csv(const std::function<void(const char*, int64_t)>& sink);
  // Objective / row-infeasibility of the last iteration (one more chain).
  void tail();
  DevStatus status();
  std::vector<HostRecord> records(int count);
  // Outputs as host fp64 column-major (nullable pointers are skipped).
  void outputs(double* out_final, double* out_pi, double* out_w);
  // Post-solve readout on the device: objective, marginal infeasibility,
  // entropy of the final coupling, split gap, hard assignment (copied to
  // `assign_host` if non-null) and its accuracy against `gt_host` (n_gt
  // entries; skipped if null).  Only the scalars / assignment leave the GPU.
  void readout(const int32_t* gt_host, int64_t n_gt, int32_t* assign_host, Readout* r);
  // Device pointers (session API): an fp32 copy of π refreshed on request.
  float* pi_dev();
  int64_t ld() const { return ldm_; }
  int precision() const { return precision_; }
  // gwb_geometry: GWB_ENTROPY (KL projections) or GWB_QUADRATIC (Euclidean
  // simplex projections, quadratic.cu).  Set before reset().
  void set_geometry(int g) { geometry_ = g; }
  bool quadratic() const { return geometry_ == GWB_QUADRATIC; }
  // CUDA-event timing of kernel classes inside iterate() (enabled on demand).
  void set_timing(bool on) { timing_ = on; }
  void kernel_ms(int kind, double* avg_ms, int64_t* count);
  double gemm_flops_per_iter() const;
  bool d_exact() const { return dx_exact_ && dy_exact_; }
  int parity() const { return parity_; }

 private:
  void alloc();
  void build_plans();
  void prepare_d();
  void load_marginals(const double* mu, const double* nu);  // + prepare_d()
  int64_t enqueue_iteration(int parity, double rel_tol);
  int64_t enqueue_half(int parity, bool half_b, double rel_tol);
  void destroy_graphs();
  // π and the w in W[par] as column-major fp64 with the K8 fix-up.
  void iterates_to_colmajor64(int par, double* pi64, double* w64, double* work);

  int device_;
  int64_t n_, m_, ldn_, ldm_;
  double rho_;
  int precision_;
  int max_iters_;
  cudaStream_t stream_;
  bool own_stream_ = false;
  int parity_ = 0;  // which W buffer holds the current w
  bool dx_exact_ = true, dy_exact_ = true;

  // device buffers
  float *Dx_ = nullptr, *Dx_aux_ = nullptr, *Dy_ = nullptr, *Dy_aux_ = nullptr;
  float *Dx_bf_ = nullptr, *Dy_bf_ = nullptr;  // bf16 copies (bf16 split modes)
  Csr cx_, cy_;                                // sparse chain (GWB_PREC_SPARSE)
  float *Vs_ = nullptr, *DyT_ = nullptr;       // skinny chain (GWB_PREC_FP32): V, D_Yᵀ
  // Split-plane chains on kind::f16 (bf16 planes, or fp16 planes for f16x2).
  bool bf16() const {
    return precision_ == GWB_PREC_BF16X3 || precision_ == GWB_PREC_BF16X2 ||
           precision_ == GWB_PREC_F16X2 || precision_ == GWB_PREC_F16X3;
  }
  // fp16 planes of the power-of-two-scaled iterate (f16x2, f16x3).
  bool f16() const { return precision_ == GWB_PREC_F16X2 || precision_ == GWB_PREC_F16X3; }
  // f16x3: the structure matrices are split too (hi + lo fp16 planes of
  // D·2^sd_), for weighted D.
  bool split_d() const { return precision_ == GWB_PREC_F16X3; }
  int sdx_ = 0, sdy_ = 0;
  // Centred chain for weighted D: the GEMMs run on
  // D − c·J (c = max D / 2), whose signed terms keep the tensor core's
  // truncating fp32 accumulation unbiased; the rank-1 parts return as
  // GEMM biases — GEMM1: c_Y·rowsum(X) per output column (cb1_pi_ for
  // X = π: c_Y·μ; cb1_w_[q] for X = w_q, written by the column write pass),
  // GEMM2: c_X·colsum(V) per output column (cb2_, from GEMM1's row sums).
  bool center_ = false;
  double ctr_x_ = 0.0, ctr_y_ = 0.0;
  float *cb1_pi_ = nullptr, *cb1_w_[2] = {nullptr, nullptr}, *cb2_ = nullptr;
  float *Dxc_ = nullptr, *Dyc_ = nullptr;  // fp32 centred copies (TF32 hi operands)
  double cb1_factor() const {  // GEMM1 accumulates 2^(s1 + sdy)·(D̃_Y Xᵀ) (f16), else D̃_Y Xᵀ
    return f16() ? std::ldexp(ctr_y_, f16_s1_ + sdy_) : ctr_y_;
  }
  double cb2_factor() const { return f16() ? std::ldexp(ctr_x_, sdx_) : ctr_x_; }
  bool sparse() const { return precision_ == GWB_PREC_SPARSE; }
  bool fp32() const { return precision_ == GWB_PREC_FP32; }
  // Skinny bf16x3 chain (m ≤ 32, exact-bf16 D_X): FP32-pipe GEMM1 writing
  // Vᵀ planes, tensor-core GEMM2 (skinny_tc.cu).
  bool skinny_tc_ = false;
  SkinnyTcPlan* stc_ = nullptr;       // skip on done
  SkinnyTcPlan* stc_tail_ = nullptr;  // skip on flags
  void* Dxp_ = nullptr;               // D_X packed in GEMM2 tile order
  void* Vtp_ = nullptr;               // Vᵀ bf16 planes packed in tile order
  void* Vtp2_ = nullptr;              // second plane buffer: half-step b's Vᵀ, written by the
                                      // fused half-step a while Vtp_ is still being streamed
  SkinnyTcPlan* stc_b_ = nullptr;     // GEMM2 of half-step b on Vtp2_ (fused schedule)
  int64_t vtp_plane_ = 0;             // bf16 elements per packed plane
  bool no_planes() const { return sparse() || fp32() || skinny_tc_; }  // chains read the fp32 iterates
  int aux_mode() const {
    return precision_ == GWB_PREC_TF32 ? 1
           : precision_ == GWB_PREC_BF16X3 ? 3
           : precision_ == GWB_PREC_BF16X2 ? 4
           : precision_ == GWB_PREC_F16X2  ? 5
           : precision_ == GWB_PREC_F16X3  ? 5
                                           : 2;
  }
  // f16x2 scaling: every iterate entry is ≤ x_max_ =
  // max(max μ, max ν) (π_kl ≤ μ_k after the row projection, w_kl ≤ ν_l after
  // the column one), so the B planes of GEMM1 carry x·2^f16_s1_ with
  // f16_s1_ = 14 − ⌈log2 x_max_⌉; per-row scales for Vᵀ (f16_g1_rs_ on
  // GEMM1's output, f16_g2_cs_ undoing them on GEMM2's).
  double x_max_ = 1.0;
  int f16_s1_ = 0;
  float* f16_g1_rs_ = nullptr;
  float* f16_g2_cs_ = nullptr;
  float aux_scale() const { return f16() ? std::ldexp(1.0f, f16_s1_) : 1.0f; }
  // Entropy geometry: π, w are fp64 (P64_, W64_) like the reference's; P_,
  // W_ hold fp32 copies where a chain reads raw iterates (needs_copy()),
  // and the quadratic geometry's fp32 iterates.
  double *P64_ = nullptr, *W64_[2] = {nullptr, nullptr};
  float *P_ = nullptr, *P_aux_ = nullptr, *W_[2] = {nullptr, nullptr},
        *W_aux_[2] = {nullptr, nullptr};
  bool needs_copy() const {
    return quadratic() || no_planes() || precision_ == GWB_PREC_3XTF32;
  }
  float *Vt_ = nullptr, *Vt_aux_ = nullptr, *G_ = nullptr;
  float *mu32_ = nullptr, *nu32_ = nullptr;
  double *mu64_ = nullptr, *nu64_ = nullptr;
  RowPart* row_part_ = nullptr;
  ColWritePart* cw_part_ = nullptr;
  double *col_pmax_ = nullptr, *col_psum_ = nullptr, *col_max_ = nullptr, *col_scale_ = nullptr;
  double *col_psump_ = nullptr, *col_dev_ = nullptr;
  DevStatus* st_ = nullptr;
  DevRecord* rec_ = nullptr;
  int chunks_ = 1;
  int* h_done_ = nullptr;  // pinned

  // GEMM plans: [parity][half] for GEMM1 (operand W[parity] or P), GEMM2;
  // tail plans skip only on errors.
  GemmPlan* g1_[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  GemmPlan* g2_ = nullptr;
  GemmPlan* g1_tail_[2] = {nullptr, nullptr};
  GemmPlan* g2_tail_ = nullptr;

  cudaGraphExec_t graph_[2] = {nullptr, nullptr};  // chunk graph per start parity
  int graph_iters_ = 0;
  int64_t graph_launches_ = 0;  // kernels in one captured chunk

  int geometry_ = GWB_ENTROPY;
  bool timing_ = false;
  double last_ms_[2] = {0.0, 0.0};
  int64_t last_cnt_[2] = {0, 0};
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_marks_;
  cudaEvent_t ev_get();

  BapgDev dev_view(int parity) const;
};

// Row-sharded BAPG over several devices of this process (shard.cu: the
// sharded engines + NCCL single-process communicator); host fp64 in / out as
// gwb_solve.  Returns the agreed status (flags decoded by the caller);
// `records` receives the trace.
DevStatus bapg_multi_device(const gwb_config& cfg, const std::vector<int>& devices,
                            const double* dx, int64_t n, const double* dy, int64_t m,
                            const double* mu, const double* nu, double* out_final,
                            double* out_pi, double* out_w, std::vector<HostRecord>* records,
                            int* resolved_precision);

// Resolves GWB_PREC_AUTO (see gwb.h).
int resolve_precision(int requested, bool bf16_exact, bool f16_exact, bool quadratic);

}  // namespace gwb
