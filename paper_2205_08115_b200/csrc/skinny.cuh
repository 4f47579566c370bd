// skinny.cuh — FP32 chain for skinny problems (m ≤ 32; see skinny.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace gwb {

constexpr int64_t kSkinnyMaxN = 32;

// C[M×N] = A[M×K] · B[K×N], all fp32 row-major (leading dimensions lda, ldb,
// ldc), 1 ≤ N ≤ 32.  Columns ≥ N of C are not written.  No-op when *skip.
void launch_skinny(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                   int64_t M, int N, int64_t K, const int* skip, cudaStream_t s);
// As launch_skinny, but C is written transposed as `planes` (2 or 3) bf16
// split planes (hi = rn(c), mid = rn(c − hi), …): plane p holds Cᵀ (N × M,
// leading dim ldp) at element offset p·pstride — the B operand of the
// tensor-core skinny GEMM2 (skinny_tc.cu).
void launch_skinny_planes(const float* A, int64_t lda, const float* B, int64_t ldb, void* planes,
                          int nplanes, int64_t ldp, int64_t pstride, int64_t M, int N, int64_t K,
                          const int* skip, cudaStream_t s);

// G[M×N] (fp32 row-major, ldc) = D · Σ_p V_pᵀ on the tensor cores, D an
// exact-bf16 M×K matrix (leading dim ldd) and V_p the bf16 planes (N × K,
// leading dim ldv), N ≤ 32 (skinny_tc.cu).  Plans own their split-K
// workspace; a launch is one kernel.
struct SkinnyTcPlan;
SkinnyTcPlan* skinny_tc_plan_create(const void* d_bf16, int64_t ldd, const void* const* vt_planes,
                                    int planes, int64_t ldv, float* c, int64_t ldc, int64_t M,
                                    int N, int64_t K, const int* skip, cudaStream_t s);
void skinny_tc_plan_destroy(SkinnyTcPlan* plan, cudaStream_t s);
void skinny_tc_launch(const SkinnyTcPlan* plan, cudaStream_t s);

// dst (cols × rows, ldd) = srcᵀ (src rows × cols, lds).
void launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst,
                      int64_t ldd, cudaStream_t s);

}  // namespace gwb
