// kernels.cuh — HBM-bound kernels around the GEMM chain: the BAPG row/column
// KL projections (kl_scale of the multiplicative update, projections.cpp:12-34
// as used by solvers.cpp:164-177), the per-iteration diagnostics fused into
// those passes, the Sinkhorn sweeps for eBPG/BPG, and layout conversions at
// the C-ABI boundary.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace gwb {

// Error bits raised by device kernels (decoded on the host in reference
// precedence order, solvers.cpp:164-189).
enum DevFlag : int {
  kFlagOverflowA = 1,   // max(D_X w D_Y / rho) > 700 in half-step a
  kFlagZeroA = 2,       // a row of w ⊙ exp(E) has nonpositive / non-finite sum
  kFlagOverflowB = 4,   // same checks in half-step b
  kFlagZeroB = 8,
  kFlagNonFinite = 16,  // non-finite iterate
  kFlagDeadLine = 32,   // eBPG: kernel row/column underflowed to zero
  kFlagOverflowK = 64,  // BPG: max(2t·M(π)) > 700
  kFlagSinkNonFinite = 128,
};

// Device-resident solver status; every kernel returns immediately when
// `done` is set, so a converged or failed solve turns the remainder of an
// already-enqueued CUDA graph into no-ops.
struct DevStatus {
  int done;        // read by every kernel's prologue
  int flags;       // DevFlag bits
  int iter;        // current 1-based outer iteration
  int err_iter;    // iteration at which flags were first raised
  int converged;
  int zero_index;  // lowest offending line (atomicMin)
  int sink_sweeps; // last Sinkhorn sweep count
  int sink_err_sweep;
  int gdone;       // sharded solver: globally agreed done (set by the finalize)
  unsigned long long t0;  // %globaltimer at reset
};

// Per-iteration trace record kept on the device (fp64).
struct DevRecord {
  double mpi_pi;     // ⟨M(π), π⟩
  double mpi_w;      // ⟨M(π), w⟩
  double mw_w;       // ⟨M(w), w⟩   (filled one half-step later)
  double col_sq;     // Σ_j (colsum(π)_j − ν_j)²
  double row_sq;     // Σ_i (rowsum(w)_i − μ_i)²  (filled one half-step later)
  double split_sq;   // ‖π − w‖²
  double diff_sq;    // ‖w' − w‖²
  double wold_sq;    // ‖w‖²
  double elapsed;    // seconds since reset
};

struct RowPart {     // per-row fp64 partials of the half-step-a pass
  double gw;         // ⟨G_i, W_i⟩
  double rowdev;     // (Σ_j W_ij − μ_i)²
};

struct ColWritePart {  // per-row fp64 partials of the half-step-b write pass
  double gw;         // ⟨G_i, W'_i⟩
  double split;      // ‖P_i − W'_i‖²
  double diff;       // ‖W'_i − W_i‖²
  double wold;       // ‖W_i‖²
  double gp;         // ⟨G_i, P_i⟩
};

struct BapgDev {
  int64_t n, m, ld;         // P/W/G are n×m row-major, leading dim ld
  float inv_rho;
  double inv_rho64;
  const float* G;
  const float* mu;          // fp32 marginals
  const float* nu;
  const double* mu64;
  const double* nu64;
  // Entropy geometry: the iterates are fp64 (P64, W64 → W64_new), as the
  // reference's; the fp32 arrays are optional copies written alongside
  // (nullable): the hi operand of the TF32 chains and the input of the
  // raw-iterate chains (sparse, skinny).  Quadratic geometry (quadratic.cu)
  // keeps fp32 iterates in P / W / W_new.
  double* P64;
  double* W64;              // current w (read in both half-steps)
  double* W64_new;          // next w (written by half-step b)
  float* P;
  float* P_aux;             // GEMM copy of P, see aux_mode (nullable)
  float* W;                 // current w (quadratic)
  float* W_new;             // next w (fp32 copy / quadratic iterate)
  float* W_aux;             // GEMM copy of W_new, see aux_mode (nullable)
  int aux_mode;             // 1: aux = rna_tf32(x) (1xTF32 operand)
                            // 2: aux = rn_tf32(x − trunc_tf32(x)) (3xTF32 residual)
                            // 3/4: 3 / 2 bf16 split planes (bf16x3 / bf16x2)
                            // 5: 2 fp16 split planes of x·aux_scale (f16x2)
  float aux_scale;          // power of two (mode 5), else 1
  int64_t plane;            // elements per bf16 plane (n·ld)
  RowPart* row_part;        // n
  ColWritePart* cw_part;    // n
  double* col_pmax;         // chunks × m
  double* col_psum;         // chunks × m
  double* col_psump;        // chunks × m : Σ_i P_ij partials
  double* col_max;          // m
  double* col_scale;        // m
  double* col_dev;          // m : (colsum(P)_j − ν_j)²
  int chunks;
  DevStatus* st;
  DevRecord* rec;           // [max_rec + 2]
  int max_rec;              // records beyond this iteration are not kept
  // Centred chain (weighted D): the write pass of half-step b
  // also stores wsum_factor · Σ_j W'_ij (fp64 sum, fp32 result), the next
  // GEMM1's rank-1 bias (nullable).
  float* wsum_bias;
  double wsum_factor;
};

// Half-step a (solvers.cpp:164-170): E = G/ρ, P = diag(μ/rowsum)·(W ⊙ e^E),
// with per-row max shift; also ⟨G,W⟩ and rowsum(W) diagnostics for the
// previous iteration's record.  `write` = false computes diagnostics only.
void launch_row_update(const BapgDev& d, bool write, cudaStream_t s);
// Half-step b (solvers.cpp:171-177): column (max, Σ P e^{E−max}) partials,
// combine + checks, then W_new = P ⊙ e^E · diag(ν/colsum) with fused
// split-gap / rel-change / objective partials.
void launch_col_update(const BapgDev& d, cudaStream_t s);
// The two data passes of half-step b separately (sharded solver): chunk
// partials of (max, Σ π e^{E−max}, Σ π) per column, and — once col_max /
// col_scale / col_dev hold the global merge — the W' write pass.
void launch_col_partial(const BapgDev& d, cudaStream_t s);
void launch_col_write(const BapgDev& d, cudaStream_t s);
// Reduces the per-line partials in fixed order into rec[iter] / rec[iter-1],
// evaluates the stop rule (solvers.cpp:191,208) and advances st->iter.
void launch_finalize(const BapgDev& d, double rel_tol, bool tail, cudaStream_t s);
void launch_status_reset(DevStatus* st, cudaStream_t s);

// Layout conversions at the boundary.
// dst (rows×cols row-major fp32, ld) = src (rows×cols column-major fp64)
void launch_colmajor64_to_rowmajor32(const double* src, int64_t rows, int64_t cols, float* dst,
                                     int64_t ld, cudaStream_t s);
// dst (column-major fp64) = src (row-major fp32) with optional fp64 exact
// re-projection of rows (axis 0, target mu) or columns (axis 1, target nu):
// the K8 fix-up that restores the fp64 marginal invariants of the reference
// (types.cpp:120-152).  axis = -1: plain widening.
void launch_rowmajor32_to_colmajor64(const float* src, int64_t rows, int64_t cols, int64_t ld,
                                     double* dst, int axis, const double* target, double* work,
                                     cudaStream_t s);
// The same from a row-major fp64 iterate (entropy BAPG).
void launch_rowmajor64_to_colmajor64(const double* src, int64_t rows, int64_t cols, int64_t ld,
                                     double* dst, int axis, const double* target, double* work,
                                     cudaStream_t s);
// dst (row-major fp64, ld) = src (column-major fp64).
void launch_colmajor64_to_rowmajor64(const double* src, int64_t rows, int64_t cols, double* dst,
                                     int64_t ld, cudaStream_t s);
// fp32 copy (nullable) and GEMM operand planes (nullable; aux_mode / scale
// as BapgDev) of a row-major fp64 iterate.
void launch_iterate_copies(const double* x, int64_t rows, int64_t cols, int64_t ld, float* copy32,
                           float* aux, int mode, float scale, cudaStream_t s);
// Centred structure-matrix operands: from D − c (formed in
// fp64), an optional fp32 copy (the TF32 hi operand) and the operand planes
// of `mode` / `scale` as launch_iterate_copies.
void launch_center_copies(const float* D, int64_t rows, int64_t cols, int64_t ld, double c,
                          float* copy32, float* aux, int mode, float scale, cudaStream_t s);
// out[i] = factor · Σ_j x[i][j] (row-major fp64, fixed order) in fp32.
void launch_row_bias64(const double* x, int64_t rows, int64_t cols, int64_t ld, double factor,
                       float* out, cudaStream_t s);
// P = μ νᵀ in row-major fp64.
void launch_product_coupling64(const double* mu, const double* nu, int64_t n, int64_t m, int64_t ld,
                               double* P, cudaStream_t s);
// dst = 0.5 (a + b), column-major fp64 of len elements.
void launch_average64(const double* a, const double* b, double* dst, int64_t len, cudaStream_t s);
// GEMM operand copy of x (ld multiple of 4): mode 1: rna_tf32(x);
// 2: x − trunc_tf32(x); 3/4: 3 or 2 bf16 split planes (plane = rows·ld);
// 5: 2 fp16 split planes of x·scale.
void launch_tf32_aux(const float* x, int64_t rows, int64_t cols, int64_t ld, float* out, int mode,
                     cudaStream_t s, float scale = 1.0f);
// out (fp16, same ld) = fp16_rn(x).
void launch_to_f16(const float* x, int64_t rows, int64_t cols, int64_t ld, void* out,
                   cudaStream_t s);
// f16x2 power-of-two scales (kernels.cu: f16_scales_kernel): per row i of
// the m×m structure matrix D, σ_i = 14 − ⌈log2(x_max · Σ_l |D[i][l]|)⌉;
// g1_row_scale[i] = 2^(σ_i − s1 − sa1), g2_col_scale[i] = 2^(−σ_i − sa2);
// sa1 / sa2: power-of-two shifts of GEMM1's / GEMM2's A planes (f16x3: the
// split structure matrices D_Y·2^sa1, D_X·2^sa2), 0 for exact D.
void launch_f16_scales(const float* D, int64_t m, int64_t ld, float x_max, int s1,
                       float* g1_row_scale, float* g2_col_scale, cudaStream_t s, int sa1 = 0,
                       int sa2 = 0);
// out (bf16, same ld) = bf16_rn(x).
void launch_to_bf16(const float* x, int64_t rows, int64_t cols, int64_t ld, void* out,
                    cudaStream_t s);
// Scans a structure matrix: *out_max = max entry, *out_inexact bit 1 if any
// entry is not exactly representable in TF32, bit 2 in bf16, bit 4 in fp16
// (0/1 adjacency is exact in all three).
void launch_analyze(const float* D, int64_t rows, int64_t cols, int64_t ld, float* out_max,
                    int* out_inexact, cudaStream_t s);
// launch_analyze + readback: the inexact bits of a structure matrix (0 for
// an empty one).  Synchronises the stream.
int analyze_inexact(const float* D, int64_t rows, int64_t cols, int64_t ld, cudaStream_t s);
// True if a structure matrix with these inexact bits is represented exactly
// by the operand copy of a split-plane chain (f16x2: fp16; bf16x3 / bf16x2:
// bf16).  The TF32 chains split both operands and need no exact D.
bool split_exact(int precision, int inexact_bits);
// P = μ νᵀ (product coupling, types.cpp:204-207) in row-major fp32.
// Post-solve readout on a device fp64 column-major coupling (n × m):
// row/column sums, per-row argmax (hard_assignment, tasks.cpp:190-200:
// strict '>', lowest column wins ties), ‖a − b‖² and agreement counts.
void launch_rowsums_cm64(const double* pi, int64_t n, int64_t m, double* out, cudaStream_t s);
void launch_colsums_cm64(const double* pi, int64_t n, int64_t m, double* out, cudaStream_t s);
void launch_argmax_rows_cm64(const double* pi, int64_t n, int64_t m, int32_t* out, cudaStream_t s);
// Σ (a_k − b_k)² (b nullable ⇒ Σ a_k²), fp64, deterministic; host result.
double sum_sq_diff_dev(const double* a, const double* b, int64_t len, cudaStream_t s);
// #{i : a_i == b_i} over len entries; host result.
int64_t count_equal_dev(const int32_t* a, const int32_t* b, int64_t len, cudaStream_t s);

// Quadratic (Euclidean) geometry, quadratic.cu: half-step a (row simplex
// projections of w + G/ρ, + flag check), half-step b (column projections of
// π + G/ρ into W_new, record partials, flag check), and w⁰ = column
// projection of π⁰ (reset).
void launch_row_quad(const BapgDev& d, cudaStream_t s);
void launch_col_quad(const BapgDev& d, cudaStream_t s);
void launch_quad_reset(const BapgDev& d, const float* pi0, float* w0, cudaStream_t s);

// Graph inputs: host int32 edge lists (pairs a, b; validated by the caller)
// standing for D = adjacency_distance(g) (tasks.cpp:167-174).
struct GraphInput {
  const int32_t* ex;
  int64_t cx;
  const int32_t* ey;
  int64_t cy;
};
// D (rows × rows fp32 row-major, leading dim ld) ← 0/1 adjacency of the host
// edge list: zero fill, one H2D of 8 B per edge, scatter D[a][b] = D[b][a] = 1.
void build_adjacency(const int32_t* edges_host, int64_t count, int64_t rows, float* D, int64_t ld,
                     cudaStream_t s);
void launch_product_coupling(const float* mu, const float* nu, int64_t n, int64_t m, int64_t ld,
                             float* P, cudaStream_t s);

}  // namespace gwb
