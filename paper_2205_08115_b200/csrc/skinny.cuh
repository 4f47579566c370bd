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
// leading dim ldp) at element offset p·pstride.  ldp == 0 writes the packed
// B operand of the tensor-core skinny GEMM2 instead (skinny_tc.cu; needs
// K, N ≤ 32; pstride = skinny_tc_packed_b_elems(M) per plane).
void launch_skinny_planes(const float* A, int64_t lda, const float* B, int64_t ldb, void* planes,
                          int nplanes, int64_t ldp, int64_t pstride, int64_t M, int N, int64_t K,
                          const int* skip, cudaStream_t s);

// G[M×N] (fp32 row-major, ldc) = D · Σ_p V_pᵀ on the tensor cores, N ≤ 32
// (skinny_tc.cu).  D (M×K, exact in bf16) is packed once into the kernel's
// shared-memory tile order (128 rows × 64 k per 16-KB tile, 128-B swizzle)
// so every load is one contiguous bulk copy; the V planes arrive packed
// the same way (32 × 64 per 4-KB tile) from launch_skinny_planes(ldp = 0).
// Plans own their split-K workspace; a launch is one kernel.
int64_t skinny_tc_packed_a_bytes(int64_t M, int64_t K);
int64_t skinny_tc_packed_b_elems(int64_t K);  // bf16 elements per plane
void skinny_tc_pack_a(const float* D, int64_t ld, int64_t M, int64_t K, void* out, cudaStream_t s);
struct SkinnyTcPlan;
SkinnyTcPlan* skinny_tc_plan_create(const void* a_packed, const void* b_packed, int planes,
                                    float* c, int64_t ldc, int64_t M, int N, int64_t K,
                                    const int* skip, cudaStream_t s);
void skinny_tc_plan_destroy(SkinnyTcPlan* plan, cudaStream_t s);
void skinny_tc_launch(const SkinnyTcPlan* plan, cudaStream_t s);
// Half-step a in one launch (entropy BAPG, fp64 iterates; solvers.cpp:164-170
// behind the chain): GEMM2 as above, then each cluster rank runs the row
// update of the rows it summed (d: the engine's device view, G read from
// shared memory) and forms half-step b's GEMM1 — the packed Vᵀ planes of
// (new π)·D_Yᵀ — into `next_b`, a plane buffer other than the one being
// streamed.  Replaces skinny_tc_launch + launch_row_update +
// launch_skinny_planes; same arithmetic.  Needs skinny_tc_can_fuse(plan).
struct BapgDev;
bool skinny_tc_can_fuse(const SkinnyTcPlan* plan);
void skinny_tc_launch_fused_a(const SkinnyTcPlan* plan, const BapgDev& d, const float* dyt,
                              int64_t ld_dyt, void* next_b, int64_t next_pstride, cudaStream_t s);

// dst (cols × rows, ldd) = srcᵀ (src rows × cols, lds).
void launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst,
                      int64_t ldd, cudaStream_t s);

}  // namespace gwb
