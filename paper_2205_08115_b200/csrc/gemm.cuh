// gemm.cuh — host interface of the tcgen05 TF32 / 3xTF32 GEMM ("TN": both
// operands K-major, i.e. row-major M×K and N×K with K contiguous).
//
//   C[M×N] = Σ_pass A_pass · B_passᵀ   (fp32 accumulate in TMEM)
//   epilogue: C *= row_scale[i] · col_scale[j]; optionally rounds the
//             output to TF32 (rna) or emits the residual C − trunc_tf32(C)
//             for a following 1xTF32 / 3xTF32 GEMM.
//
// This is the K1 kernel of SURVEY.md §2.3: each BAPG half-step issues two of
// these for the D_X·π·D_Y chain (reference: structure_product,
// proj/src/solvers.cpp:16-19, where Eigen's dense GEMM does the work).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace gwb {

struct GemmDesc {
  int64_t M = 0, N = 0, K = 0;
  const float* a = nullptr;     // M×K row-major, leading dim lda
  const float* a_lo = nullptr;  // optional residual A − trunc_tf32(A)
  int64_t lda = 0;
  const float* b = nullptr;     // N×K row-major, leading dim ldb
  const float* b_lo = nullptr;
  int64_t ldb = 0;
  float* c = nullptr;           // M×N row-major, leading dim ldc
  float* c_aux = nullptr;       // optional second output, see aux_mode
  int64_t ldc = 0;
  int aux_mode = 0;             // 0: none; 1: c holds rna_tf32(C) (for a
                                // following 1xTF32 GEMM), c_aux unused;
                                // 2: c holds C, c_aux = C − trunc_tf32(C)
  const float* row_scale = nullptr;  // length M
  const float* col_scale = nullptr;  // length N
  const int* skip = nullptr;         // device flag: nonzero ⇒ kernel is a no-op
  bool three_pass = false;           // 3xTF32 (drops A_lo·B_lo); needs *_lo
  int promote_every = 2;             // k-blocks per TMEM chunk; 0 = never
  // bf16 split mode (kind::f16): A is an exact bf16 matrix (e.g. 0/1
  // adjacency), B is given as `bf16_planes` bf16 planes whose sum is the
  // fp32 operand; C = Σ_p A·B_pᵀ.  Replaces a/b/*_lo when bf16_planes > 0.
  int bf16_planes = 0;               // 0 (TF32 path), 2 or 3
  const void* a_bf16 = nullptr;      // M×K bf16, leading dim lda
  const void* a_bf16_lo = nullptr;   // optional second A plane (f16x3: A = hi + lo fp16
                                     // planes; passes lo·hi + hi·lo + hi·hi, B has 2 planes)
  const void* b_bf16[3] = {nullptr, nullptr, nullptr};  // N×K planes, ldb
  // Output as bf16 split planes (for a following bf16-split GEMM) instead
  // of fp32 `c`: c_planes ∈ {0, 2, 3}; planes are M×N with leading dim ldc.
  int c_planes = 0;
  void* c_bf16[3] = {nullptr, nullptr, nullptr};
  // fp16 instead of bf16 for A, the B planes and the output planes
  // (kind::f16 with fp16 operands): 11-bit planes, so two planes carry a
  // 22-bit operand.  The caller keeps every plane inside fp16 range with
  // power-of-two scales folded into row_scale / col_scale.
  bool f16 = false;
  // Split planes in one pipeline stage {A, B_0, …} per k-block, A loaded
  // once for every plane pass (default); false: one stage per (pass,
  // k-block), A re-loaded per pass (A/B testing; env GWB_GEMM_UNFUSED=1).
  bool fuse_planes = true;
  // Blocked-K B operand (multi-GPU all-gather layout): when b_block_k > 0,
  // every B plane is stored as [K / b_block_k][N][b_block_k] (leading dim of
  // a block row = b_block_k); b_block_k must be a multiple of the k-block
  // (32 fp32 / 64 bf16 elements).
  int64_t b_block_k = 0;
  int64_t b_block_stride = 0;        // elements between blocks (0 ⇒ N·b_block_k)
  // C += A·Bᵀ instead of C = A·Bᵀ (fp32 `c` output only): K-split partial
  // products accumulated across launches (multi-GPU chunked GEMM2).
  bool accumulate = false;
  // Split-K for grids smaller than one wave of CTA pairs (small problems):
  // 0 = automatic, 1 = never, S ≥ 2 = force S splits.  Partial products go
  // to a plan-owned fp32 workspace and a second kernel sums them in a fixed
  // order and applies the epilogue (scales, operand copies, planes).
  int split_k = 0;
  // Centred structure matrices (weighted D): the caller passes
  // A − c·J and adds the rank-1 part back through col_bias, a length-N vector
  // added to the accumulated sum before the row / column scales.  With
  // `rowsums` the plan also keeps fp64 partial sums of every output row
  // (after scaling, before the plane split) for gemm_rowsum_bias.
  const float* col_bias = nullptr;
  bool rowsums = false;
  // Split A (f16x3) in fused stages with 4-k-block promotion chunks.  Only
  // for centred operands: on all-positive terms the 48-MMA chunks measured a
  // 3× larger truncation bias than separate pass stages.
  bool fuse_split_a = false;
  // A is a constant operand (a structure matrix), not written by the kernel
  // launched before this GEMM: its first stages are requested before the
  // programmatic-dependent-launch wait (fused schedule).
  bool a_const = false;
};

// 2-D TMA descriptor of a row-major rows×cols matrix (leading dim ld
// elements; esize 4 = fp32, 2 = bf16), box = box_rows × 128 B, 128-B swizzle,
// zero fill out of bounds.
CUtensorMap gemm_tensor_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                            int esize);

// Opaque, pre-encoded launch (TMA descriptors built once, reusable in graphs).
struct GemmPlan;

GemmPlan* gemm_plan_create(const GemmDesc& d);
void gemm_plan_destroy(GemmPlan* p);
cudaError_t gemm_launch(const GemmPlan* p, cudaStream_t s);
// Algorithmic FLOPs of one launch (2·M·N·K, independent of the pass count).
double gemm_flops(const GemmPlan* p);
int gemm_passes(const GemmPlan* p);
// Kernel launches per gemm_launch (2 with split-K).
int gemm_launches(const GemmPlan* p);
// out[i] = factor · Σ_j C[i][j] over the last launch's output rows (fp64 sum
// of the plan's row partials in a fixed order, rounded to fp32).  Needs
// GemmDesc::rowsums; one launch, a no-op when the plan's skip flag is set.
cudaError_t gemm_rowsum_bias(const GemmPlan* p, double factor, float* out, cudaStream_t s);
// Debug (GWB_GEMM_TIMING=1): copies the last timed launch's per-CTA stamps
// ([ctas][8] %globaltimer ns) to `out`; returns the CTA count (0 if none).
int gemm_debug_stamps(unsigned long long* out, int max_ctas);

}  // namespace gwb
