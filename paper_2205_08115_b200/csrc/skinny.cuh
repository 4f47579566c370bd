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
// dst (cols × rows, ldd) = srcᵀ (src rows × cols, lds).
void launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst,
                      int64_t ldd, cudaStream_t s);

}  // namespace gwb
