/*
 * gwb.h — C-ABI of the B200-native BAPG / hBPG Gromov-Wasserstein solver.
 *
 * This is the drop-in boundary for the reference toolkit's solver path
 * (/root/reference/proj/include/gw/solvers.hpp, types.hpp, projections.hpp,
 * diagnostics.hpp).  Every entry point names the reference interface it
 * replaces.  Conventions:
 *
 *   - Host buffers are column-major fp64, byte-identical to Eigen's
 *     MatrixXd::data() / VectorXd::data() (types.hpp:13-14).  The caller
 *     allocates every output.
 *   - No exceptions cross this boundary.  Every call returns a gwb_status
 *     code and fills `gwb_status` (nullable); the C++/Python mirrors rethrow
 *     the reference's exception classes from it (types.hpp:27-59).
 *   - Calls are reentrant: concurrent solves on distinct inputs are safe
 *     (one CUDA stream and one device workspace per call).
 *   - There is no CPU fallback: compute entry points fail with
 *     GWB_ERR_RUNTIME when no sm_100 device is present.
 */
#ifndef GWB_H_
#define GWB_H_

#include <stdint.h>

#if defined(__GNUC__)
#define GWB_API __attribute__((visibility("default")))
#else
#define GWB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* gw::Algorithm (types.hpp:19) */
enum gwb_algorithm { GWB_BAPG = 0, GWB_BPG = 1, GWB_EBPG = 2, GWB_HBPG = 3, GWB_FW = 4 };
/* gw::Geometry (types.hpp:20) */
enum gwb_geometry { GWB_ENTROPY = 0, GWB_QUADRATIC = 1 };
/* gw::Axis (types.hpp:17) */
enum gwb_axis { GWB_ROWS = 0, GWB_COLS = 1 };

/* Tensor-core precision of the D_X·π·D_Y chain (B200 extension, not in
 * SolverConfig).  All modes accumulate in fp32; the entropy engines keep
 * fp64 iterates.
 * AUTO picks, by the exactness of the structure matrices:
 *   - both exact in fp16 (0/1 graphs, small integer weights): F16X2 — in the
 *     BAPG, eBPG / BPG / hBPG and row-sharded engines and the batched
 *     n, m ≤ 128 kernel;
 *   - exact in bf16 only: BF16X3 (also the skinny m ≤ 32 chain for 0/1 D_X);
 *   - otherwise: F16X3 in the single-GPU BAPG engine, on the centred
 *     structure matrices D − (max D / 2)·J with the rank-1 parts added back
 *     exactly (the tensor core's truncating accumulation then has no sign
 *     bias); 3XTF32 in the other engines (also centred in the single-GPU
 *     BAPG engine).
 * An explicit split-plane request (F16X2 / BF16X3 / BF16X2) on a D that is
 * not exact in that format falls back F16X2 -> BF16X3 -> 3XTF32, as AUTO
 * would; TF32 (1 pass) and BF16X2 are faster, reduced-precision opt-ins. */
enum gwb_precision {
  GWB_PREC_AUTO = 0,
  GWB_PREC_TF32 = 1,    /* 1 kind::tf32 pass, rna-rounded operands */
  GWB_PREC_3XTF32 = 2,  /* hi/lo TF32 split passes (2 when D is 0/1) */
  GWB_PREC_BF16X3 = 3,  /* exact-bf16 D × 3 bf16 planes of the iterate (24-bit) */
  GWB_PREC_BF16X2 = 4,  /* exact-bf16 D × 2 bf16 planes (16-bit) */
  GWB_PREC_SPARSE = 5,  /* CSR row-gather chain, fp32 exact-order sums (sparse D) */
  GWB_PREC_FP32 = 6,    /* FP32-pipe chain for skinny problems (m ≤ 32); AUTO picks it */
  GWB_PREC_F16X2 = 7,   /* exact-fp16 D × 2 fp16 planes of the power-of-two-scaled
                           iterate (22-bit operands); AUTO picks it for 0/1 graphs */
  GWB_PREC_F16X3 = 8    /* both operands as scaled fp16 hi + lo planes, 3 kind::f16
                           passes (hi·hi + hi·lo + lo·hi, 22-bit operands); AUTO picks
                           it for weighted D in the single-GPU BAPG engine */
};

/* Error codes; each maps to one reference exception class. */
enum gwb_code {
  GWB_OK = 0,
  GWB_ERR_CONFIG = 1,        /* gw::ConfigError            types.hpp:27-29 */
  GWB_ERR_DIMENSION = 2,     /* gw::DimensionMismatchError types.hpp:31-33 */
  GWB_ERR_NUMERICAL = 3,     /* gw::NumericalInstabilityError types.hpp:49-59 */
  GWB_ERR_ZERO_SUM = 4,      /* gw::ZeroSumLineError       types.hpp:36-45 */
  GWB_ERR_INVALID = 5,       /* std::invalid_argument (value-type checks) */
  GWB_ERR_DOMAIN = 6,        /* std::domain_error */
  GWB_ERR_UNSUPPORTED = 7,   /* outside the B200 path (FW) */
  GWB_ERR_RUNTIME = 8,       /* CUDA / NCCL / no device: std::runtime_error */
  GWB_ERR_CAPACITY = 9       /* caller-provided trace buffer too small */
};

/* gw::SolverConfig, field for field (types.hpp:132-147), then extensions. */
typedef struct gwb_config {
  int32_t algorithm;     /* gwb_algorithm, default GWB_BAPG */
  int32_t geometry;      /* gwb_geometry, default GWB_ENTROPY */
  double rho;            /* 0.1 */
  double step;           /* 5.0 */
  double epsilon_reg;    /* 0.1 */
  int32_t inner_iters;   /* 1000 */
  double inner_tol;      /* 1e-9 */
  double rel_tol;        /* 1e-6 */
  int32_t max_iters;     /* 2000 */
  double perturbation;   /* 0.0 */
  int32_t switch_iters;  /* 200 */
  int64_t seed;          /* 0 */
  int32_t log_domain;    /* 0 */
  int32_t record_residual; /* 0 */
  /* --- B200 extensions --- */
  int32_t precision;     /* gwb_precision, default GWB_PREC_AUTO */
  int32_t quiet;         /* suppress the bpg step-size warning on stderr */
} gwb_config;

/* gw::IterationRecord (types.hpp:152-161); `residual` is valid iff has_residual. */
typedef struct gwb_record {
  int32_t iter;
  double objective;
  double marginal_infeasibility;
  double split_gap;
  double residual;
  int32_t has_residual;
  double rel_change;
  double elapsed_seconds;
  int32_t phase;
} gwb_record;

typedef struct gwb_status {
  int32_t code;          /* gwb_code */
  int32_t iteration;     /* NumericalInstabilityError::iteration() */
  int32_t axis;          /* ZeroSumLineError::axis() */
  int64_t index;         /* ZeroSumLineError::index() */
  char solver[16];       /* NumericalInstabilityError::solver() */
  char message[512];     /* what() of the reference exception, verbatim format */
} gwb_status;

/* SolveOptions::observer (solvers.hpp:44).  Called after every outer
 * iteration with the current iterate(s) as column-major fp64; `w` is
 * non-null only for BAPG.  A nonzero return aborts the solve with
 * GWB_ERR_RUNTIME.  Setting an observer switches the solver to its
 * per-iteration host-synchronous slow path. */
typedef int32_t (*gwb_observer)(void* user, int32_t iter, const double* pi,
                                const double* w, int64_t n, int64_t m);

/* Fills `cfg` with the SolverConfig defaults (types.hpp:132-147). */
GWB_API void gwb_config_default(gwb_config* cfg);

/* gw::validate(SolverConfig) (types.hpp:129 / types.cpp:176-188). */
GWB_API int32_t gwb_validate_config(const gwb_config* cfg, gwb_status* st);

/* gw::solve / bapg_solve / bpg_solve / ebpg_solve / hbpg_solve
 * (solvers.hpp:47-70, solvers.cpp:138-426, 499-515).
 *   dx: n×n, dy: m×m (already symmetrized, as gw::DistanceMatrix holds them)
 *   mu: n, nu: m (gw::ProbabilityVector weights)
 *   initial: n×m or NULL (SolveOptions::initial)
 *   out_final: n×m, SolveReport::final_coupling (BAPG: ½(π+w))
 *   out_pi, out_w: n×m or NULL; BAPG's pi_half / w_half
 *   trace: capacity `trace_cap` records (max_iters suffices)
 * gwb_solve dispatches on cfg->algorithm; the named variants first check it
 * (require_algorithm, solvers.cpp:52-58). */
typedef int32_t (*gwb_solve_fn)(const gwb_config*, const double*, int64_t,
                                const double*, int64_t, const double*,
                                const double*, const double*, gwb_observer,
                                void*, double*, double*, double*, gwb_record*,
                                int32_t, int32_t*, int32_t*, int32_t*,
                                gwb_status*);
#define GWB_SOLVE_SIGNATURE                                                    \
  (const gwb_config* cfg, const double* dx, int64_t n, const double* dy,       \
   int64_t m, const double* mu, const double* nu, const double* initial,       \
   gwb_observer observer, void* user, double* out_final, double* out_pi,       \
   double* out_w, gwb_record* trace, int32_t trace_cap, int32_t* n_records,    \
   int32_t* converged, int32_t* iterations_used, gwb_status* st)
GWB_API int32_t gwb_solve GWB_SOLVE_SIGNATURE;
GWB_API int32_t gwb_bapg_solve GWB_SOLVE_SIGNATURE;
GWB_API int32_t gwb_bpg_solve GWB_SOLVE_SIGNATURE;
GWB_API int32_t gwb_ebpg_solve GWB_SOLVE_SIGNATURE;
GWB_API int32_t gwb_hbpg_solve GWB_SOLVE_SIGNATURE;

/* gw::solve(adjacency_distance(Graph(n, edges_x)), adjacency_distance(Graph(m,
 * edges_y)), mu, nu, cfg) — tasks.cpp:167-174 + types.cpp:155-174 + solvers.cpp
 * :499-515 in one call.  Edge lists are int32 pairs (a, b); they are
 * validated as the reference Graph constructor does (GWB_ERR_INVALID:
 * "graph must have at least one node", "self-loop at node a",
 * "edge (a,b) out of range for N nodes"; duplicates are harmless) and the
 * dense 0/1 structure matrices are built on the device from 8 B per edge
 * instead of uploading n² + m² fp64 entries.  Outputs and errors as
 * gwb_solve. */
GWB_API int32_t gwb_solve_graphs(const gwb_config* cfg, int64_t n,
                                 const int32_t* edges_x, int64_t count_x,
                                 int64_t m, const int32_t* edges_y,
                                 int64_t count_y, const double* mu,
                                 const double* nu, const double* initial,
                                 gwb_observer observer, void* user,
                                 double* out_final, double* out_pi,
                                 double* out_w, gwb_record* trace,
                                 int32_t trace_cap, int32_t* n_records,
                                 int32_t* converged, int32_t* iterations_used,
                                 gwb_status* st);

/* gw::gw_objective (solvers.hpp:12-13, solvers.cpp:64-69): -Σ (D_X π D_Y)⊙π.
 * pi is pi_rows×pi_cols (shape-checked against n, m). */
GWB_API int32_t gwb_gw_objective(const double* dx, int64_t n, const double* dy,
                         int64_t m, const double* pi, int64_t pi_rows,
                         int64_t pi_cols, double* out, gwb_status* st);

/* gw::product_coupling (types.hpp:177-178, types.cpp:204-207): μνᵀ. */
GWB_API int32_t gwb_product_coupling(const double* mu, int64_t n, const double* nu,
                             int64_t m, double* out, gwb_status* st);

/* gw::lipschitz_bound (solvers.hpp:37, solvers.cpp:113-136):
 * σmax(D_X)·σmax(D_Y) by fp64 power iteration on D², tol 1e-10, cap 10000. */
GWB_API int32_t gwb_lipschitz_bound(const double* dx, int64_t n, const double* dy,
                            int64_t m, double* out, gwb_status* st);

/* gw::kl_scale (projections.hpp:18, projections.cpp:12-34). */
GWB_API int32_t gwb_kl_scale(const double* pi, int64_t n, int64_t m,
                     const double* target, int64_t target_len, int32_t axis,
                     double* out, gwb_status* st);

/* gw::sinkhorn_project / sinkhorn_project_log (projections.hpp:35-47,
 * projections.cpp:92-163).  `log_domain` selects the log variant, in which
 * case `kernel` holds the exponent. */
GWB_API int32_t gwb_sinkhorn_project(const double* kernel, int64_t n, int64_t m,
                             const double* mu, const double* nu, double tol,
                             int32_t max_iters, int32_t log_domain,
                             double* out, int32_t* iterations,
                             double* marginal_error, int32_t* converged,
                             gwb_status* st);

/* gw::marginal_infeasibility / split_gap (diagnostics.hpp:18-23,
 * diagnostics.cpp:9-27). */
GWB_API int32_t gwb_marginal_infeasibility(const double* pi, int64_t n, int64_t m,
                                   const double* mu, int64_t mu_len,
                                   const double* nu, int64_t nu_len,
                                   double* out, gwb_status* st);
GWB_API int32_t gwb_split_gap(const double* pi, const double* w, int64_t n, int64_t m,
                      double* out, gwb_status* st);

/* gw::hard_assignment (tasks.hpp:58, tasks.cpp:190-200): per-row argmax,
 * strict '>' so ties resolve to the lowest column. */
GWB_API int32_t gwb_hard_assignment(const double* pi, int64_t n, int64_t m,
                            int32_t* out, gwb_status* st);

/* gw::coupling_entropy (diagnostics.hpp:37-38, diagnostics.cpp:44-53):
 * -Σ π log π over positive entries, nats (fp64 device reduction). */
GWB_API int32_t gwb_coupling_entropy(const double* pi, int64_t n, int64_t m,
                                     double* out, gwb_status* st);

/* gw::alignment_accuracy (tasks.hpp:64, tasks.cpp:202-214): percentage of
 * gt entries matched by pred.  GWB_ERR_DIMENSION if n_pred < n_gt
 * ("alignment_accuracy: prediction does not cover all ground-truth nodes"),
 * GWB_ERR_INVALID if n_gt == 0 ("empty ground truth"). */
GWB_API int32_t gwb_alignment_accuracy(const int32_t* pred, int64_t n_pred,
                                       const int32_t* gt, int64_t n_gt,
                                       double* out, gwb_status* st);

/* gw::write_coupling_csv / write_coupling_csv_file (io.hpp:36-37,
 * io.cpp:183-199): "rows,cols\n" then each row's entries as "%.17g" joined
 * by ',' and ended by '\n' — formatted on the device (exact decimal
 * conversion, round-half-even as glibc), only text crosses PCIe.
 * gwb_format_coupling_csv writes into `out` (cap bytes) and sets *len to the
 * bytes needed; out == NULL queries the size, a short buffer gives
 * GWB_ERR_CAPACITY.  The file form fails with GWB_ERR_RUNTIME
 * "cannot write '<path>'" as the reference. */
GWB_API int32_t gwb_format_coupling_csv(const double* pi, int64_t n, int64_t m, char* out,
                                        int64_t cap, int64_t* len, gwb_status* st);
GWB_API int32_t gwb_write_coupling_csv_file(const char* path, const double* pi, int64_t n,
                                            int64_t m, gwb_status* st);

/* gw::dykstra_project (projections.hpp:46-51, projections.cpp:165-187):
 * Euclidean projection of pi onto Π(μ, ν) by Dykstra's alternating
 * projections; stops once the inf-norm marginal error ≤ tol.
 * GWB_ERR_RUNTIME "dykstra_project did not converge in <max_iters> sweeps;
 * final constraint violation <err>" otherwise (fp64 on the device). */
GWB_API int32_t gwb_dykstra_project(const double* pi, int64_t n, int64_t m,
                                    const double* mu, const double* nu, double tol,
                                    int32_t max_iters, double* out, gwb_status* st);

/* gw::luo_tseng_residual (diagnostics.hpp:27-29, diagnostics.cpp:33-42):
 * ‖π − dykstra_project(π + D_X π D_Y, μ, ν, dykstra_tol)‖_F (10000 sweeps;
 * the reference default dykstra_tol is 1e-8).  Also filled into every
 * gwb_record when gwb_config.record_residual is set. */
GWB_API int32_t gwb_luo_tseng_residual(const double* dx, int64_t n, const double* dy,
                                       int64_t m, const double* pi, const double* mu,
                                       const double* nu, double dykstra_tol, double* out,
                                       gwb_status* st);

/* Batched BAPG over `batch` independent problems sharing n and m (config 5).
 * The reference has no batched API; its equivalent is `batch` calls of
 * gw::solve from the experiment worker pool (experiment.cpp:273-304).
 * Inputs are `batch` consecutive column-major blocks; records are per
 * problem, `trace_cap` each (may be 0 with trace NULL). */
GWB_API int32_t gwb_bapg_solve_batched(const gwb_config* cfg, int64_t batch,
                               const double* dx, int64_t n, const double* dy,
                               int64_t m, const double* mu, const double* nu,
                               double* out_final, double* out_pi, double* out_w,
                               gwb_record* trace, int32_t trace_cap,
                               int32_t* n_records, int32_t* converged,
                               int32_t* iterations_used, gwb_status* st);

/* Device selection side channel (the reference API has no device knob).
 * Also read from env GWB_DEVICES="0,1,..." on first use.  The first id runs
 * single-device work.  With several ids, BAPG solves without observer /
 * residual / initial coupling / graph inputs are row-sharded over all of them
 * in this process (NCCL single-process communicator, loaded at run time;
 * a device listed twice emulates the collectives — a one-GPU test mode), and
 * gwb_bapg_solve_batched splits its problems across them. */
GWB_API int32_t gwb_set_devices(int32_t count, const int32_t* ids, gwb_status* st);

/* ---------------------------------------------------------------------------
 * Device-resident session API (B200 extension).  Used to time the hot path
 * with inputs already in HBM.  Pointers are device pointers to fp32
 * row-major matrices with leading dimension `ld` (elements).
 * ------------------------------------------------------------------------- */
typedef struct gwb_session gwb_session;

GWB_API int32_t gwb_session_create(const gwb_config* cfg, int64_t n, int64_t m,
                           int32_t device, gwb_session** out, gwb_status* st);
/* Copies fp32 device inputs into the session workspace (async on `stream`). */
GWB_API int32_t gwb_session_load_device(gwb_session* s, const float* dx, int64_t ldx,
                                const float* dy, int64_t ldy, const float* mu,
                                const float* nu, void* stream, gwb_status* st);
/* Resets the iterate to the product coupling (solvers.cpp:41-50, 146-153). */
GWB_API int32_t gwb_session_reset(gwb_session* s, void* stream, gwb_status* st);
/* Enqueues `iters` BAPG iterations on the session stream without host
 * synchronisation (CUDA graphs).  Returns the number of kernel launches
 * enqueued in *launches; if *launches < 0 on entry, launches are issued
 * eagerly with CUDA events bracketing each kernel class (for
 * gwb_session_kernel_ms). */
GWB_API int32_t gwb_session_iterate(gwb_session* s, int32_t iters, void* stream,
                            int64_t* launches, gwb_status* st);
/* The CUDA stream (cudaStream_t) every session kernel is launched on. */
GWB_API int32_t gwb_session_stream(gwb_session* s, void** stream, gwb_status* st);
/* Resolved precision (gwb_precision) and algorithmic GEMM FLOPs per
 * iteration, 4·n·m·(n+m). */
GWB_API int32_t gwb_session_info(gwb_session* s, int32_t* precision,
                         double* gemm_flops_per_iter, gwb_status* st);
/* Device pointer to the π half (fp32 row-major, ld = *ld). */
GWB_API int32_t gwb_session_pi(gwb_session* s, float** pi, int64_t* ld, gwb_status* st);
/* Average duration (ms) of the dominant kernel class over the launches
 * recorded since the last call, timed with CUDA events on the launching
 * stream.  kind: 0 = GEMM chain, 1 = scaling/normalisation. */
GWB_API int32_t gwb_session_kernel_ms(gwb_session* s, int32_t kind, double* avg_ms,
                              int64_t* count, gwb_status* st);
GWB_API int32_t gwb_session_destroy(gwb_session* s);

/* run_cell's post-solve readout (experiment.cpp:169-195) of the session's
 * final coupling ½(π + w), computed on the device: gw_objective,
 * marginal_infeasibility, coupling_entropy, split_gap(π, w), and the
 * luo_tseng_residual (NaN when its Dykstra projection does not converge, as
 * run_cell's catch, experiment.cpp:177-182), the
 * hard_assignment (written to `assignment`, n entries, if non-null) with its
 * alignment_accuracy against `ground_truth` (n_gt entries, if non-null;
 * same errors as gwb_alignment_accuracy).  Nothing n×m crosses PCIe. */
typedef struct gwb_readout {
  double objective;
  double marginal_infeasibility;
  double entropy;
  double split_gap;
  double residual;      /* luo_tseng_residual; NaN if Dykstra did not converge */
  double accuracy;      /* valid iff has_accuracy */
  int32_t has_accuracy;
} gwb_readout;
GWB_API int32_t gwb_session_readout(gwb_session* s, const int32_t* ground_truth,
                                    int64_t n_gt, int32_t* assignment,
                                    gwb_readout* out, gwb_status* st);

/* write_coupling_csv_file of the session's final coupling ½(π + w)
 * (run_cell's `--coupling-out`, experiment.cpp; io.cpp:195-199), formatted
 * on the device. */
GWB_API int32_t gwb_session_write_coupling_csv(gwb_session* s, const char* path,
                                               gwb_status* st);

/* Library identity: build string including the compiled GPU arch. */
GWB_API const char* gwb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GWB_H_ */
