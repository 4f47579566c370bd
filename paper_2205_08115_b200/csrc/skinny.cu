// skinny.cu — the chain for skinny problems (m ≤ 32, SURVEY §8(a) config 3:
// graph partition n × K with K = 20).  A 256×256 tensor-core tile would be
// 92% padding there and the chain is HBM/L2-bound, so both products run on
// the FP32 pipes:
//   V = X · D_Yᵀ   (n × m, K = m)      G = D_X · V   (n × m, K = n)
// as C[M×N] = A[M×K] · B[K×N] with N ≤ 32.  One CTA = 8 warps × 2 rows of
// C; lanes split K (4 loads per row in flight), B is staged through shared
// memory in 256-row chunks, and each warp ends with a 32-lane
// transpose-reduce so lane c writes column c.  The product is latency-bound
// at config-3 size (ncu: few loads in flight per SM); a TMA-pipelined A
// stream is the next step.
// Sums are fp32 in a fixed order (deterministic, no operand splitting).
#include "skinny.cuh"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace gwb {

void check_cuda(cudaError_t e, const char* what);  // solver.cu

namespace {

constexpr int kRowsPerWarp = 2;
constexpr int kUnroll = 4;                   // k values per lane in flight
constexpr int kWarps = 8;
constexpr int kRows = kRowsPerWarp * kWarps;  // rows of C per CTA
constexpr int kChunk = 256;                  // K rows of B staged per step

__device__ __forceinline__ uint16_t bf16_bits(float x) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

template <int NQ>
__global__ void __launch_bounds__(kWarps * 32) skinny_kernel(
    const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb,
    float* __restrict__ C, int64_t ldc, int64_t M, int N, int64_t K, const int* skip,
    uint16_t* __restrict__ planes, int nplanes, int64_t ldp, int64_t pstride) {
  if (skip && *skip) return;
  constexpr int NP = NQ * 4;
  __shared__ __align__(16) float bs[kChunk][NP];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRows + warp * kRowsPerWarp;
  float acc[kRowsPerWarp][NP];
#pragma unroll
  for (int r = 0; r < kRowsPerWarp; ++r)
#pragma unroll
    for (int c = 0; c < NP; ++c) acc[r][c] = 0.f;
  const float* arow[kRowsPerWarp];
  bool rok[kRowsPerWarp];
#pragma unroll
  for (int r = 0; r < kRowsPerWarp; ++r) {
    rok[r] = row0 + r < M;
    arow[r] = A + (rok[r] ? row0 + r : 0) * lda;
  }
  for (int64_t k0 = 0; k0 < K; k0 += kChunk) {
    __syncthreads();
    for (int e = threadIdx.x; e < kChunk * NP; e += kWarps * 32) {
      const int kk = e / NP, c = e % NP;
      const int64_t k = k0 + kk;
      bs[kk][c] = (k < K && c < N) ? B[k * ldb + c] : 0.f;
    }
    __syncthreads();
    const int kmax = static_cast<int>(K - k0 < kChunk ? K - k0 : kChunk);
    for (int kb = 0; kb < kmax; kb += 32 * kUnroll) {
      // kUnroll × kRowsPerWarp independent loads in flight per lane.
      float a[kUnroll][kRowsPerWarp];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int kk = kb + 32 * u + lane;
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r)
          a[u][r] = (rok[r] && kk < kmax) ? __ldg(arow[r] + k0 + kk) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int kk = kb + 32 * u + lane;
        if (kb + 32 * u >= kmax) break;  // warp-uniform
        const int ks = kk < kmax ? kk : 0;  // a == 0 past kmax; keep the smem read in bounds
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float4 b = *reinterpret_cast<const float4*>(&bs[ks][4 * q]);
#pragma unroll
          for (int r = 0; r < kRowsPerWarp; ++r) {
            acc[r][4 * q + 0] = fmaf(a[u][r], b.x, acc[r][4 * q + 0]);
            acc[r][4 * q + 1] = fmaf(a[u][r], b.y, acc[r][4 * q + 1]);
            acc[r][4 * q + 2] = fmaf(a[u][r], b.z, acc[r][4 * q + 2]);
            acc[r][4 * q + 3] = fmaf(a[u][r], b.w, acc[r][4 * q + 3]);
          }
        }
      }
    }
  }
  // Transpose-reduce each row's NP partial sums over the 32 lanes: after the
  // five stages lane c holds the total of column c (fixed order).
#pragma unroll
  for (int r = 0; r < kRowsPerWarp; ++r) {
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = c < NP ? acc[r][c] : 0.f;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const bool upper = (lane & s) != 0;
#pragma unroll
      for (int k = 0; k < s; ++k) {
        const float send = upper ? v[k] : v[k + s];
        const float keep = upper ? v[k + s] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
      }
    }
    if (rok[r] && lane < N) {
      if (planes) {  // transposed bf16 split planes of the result
        float x = v[0];
        for (int q = 0; q < nplanes; ++q) {
          const float h = __bfloat162float(__float2bfloat16_rn(x));
          planes[q * pstride + lane * ldp + row0 + r] = bf16_bits(h);
          x -= h;
        }
      } else {
        C[(row0 + r) * ldc + lane] = v[0];
      }
    }
  }
}

__global__ void transpose_kernel(const float* __restrict__ src, int64_t rows, int64_t cols,
                                 int64_t lds, float* __restrict__ dst, int64_t ldd) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t r = e / cols, c = e % cols;
  dst[c * ldd + r] = src[r * lds + c];
}

// Small-K product with transposed bf16-plane output (GEMM1 of the skinny
// bf16x3 chain, K = N = m ≤ 32): one CTA per 32 rows of C, lane = row, the 8
// warps splitting the N output columns (the per-column FMA chains are the
// latency; a single warp per row block ran 4k dependent instructions).  The
// 32×K block of A is read coalesced (lane = k) into a padded shared tile, B
// (K×N ≤ 4 KB) is staged alongside; each lane sums over k in order and
// writes the split planes of Cᵀ — at a fixed column, 32 consecutive rows.
constexpr int kSmallKWarps = 8;
__global__ void __launch_bounds__(32 * kSmallKWarps) small_k_planes_kernel(
    const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb, int64_t M,
    int N, int K, const int* skip, uint16_t* __restrict__ planes, int nplanes, int64_t ldp,
    int64_t pstride) {
  if (skip && *skip) return;
  __shared__ float bs[32][32];
  __shared__ float at[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x / 32;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
  // Warp w stages rows / k-rows w, w+8, w+16, w+24: 8 loads in flight per lane.
  float bv[4], av[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int k = warp + kSmallKWarps * t;
    bv[t] = (k < K && lane < N) ? B[static_cast<int64_t>(k) * ldb + lane] : 0.f;
    av[t] = (r0 + k < M && lane < K) ? A[(r0 + k) * lda + lane] : 0.f;
  }
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    bs[warp + kSmallKWarps * t][lane] = bv[t];
    at[warp + kSmallKWarps * t][lane] = av[t];
  }
  __syncthreads();
  const int64_t row = r0 + lane;
  float a[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) a[k] = at[lane][k];
  for (int c = warp; c < N; c += kSmallKWarps) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < K) acc = fmaf(a[k], bs[k][c], acc);
    if (row < M) {
      // ldp == 0: the skinny GEMM2's packed operand — per 64-row k-block, a
      // 32 × 128-B tile in the 128-B swizzle layout (skinny_tc.cu).
      const int64_t off = ldp ? static_cast<int64_t>(c) * ldp + row
                              : (row >> 6) * 2048 + c * 64 +
                                    ((((row >> 3) & 7) ^ (c & 7)) << 3) + (row & 7);
      float x = acc;
      for (int q = 0; q < nplanes; ++q) {
        const float h = __bfloat162float(__float2bfloat16_rn(x));
        planes[q * pstride + off] = bf16_bits(h);
        x -= h;
      }
    }
  }
}

}  // namespace

void launch_transpose(const float* src, int64_t rows, int64_t cols, int64_t lds, float* dst,
                      int64_t ldd, cudaStream_t s) {
  const int64_t total = rows * cols;
  if (total == 0) return;
  transpose_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(src, rows, cols, lds,
                                                                             dst, ldd);
  check_cuda(cudaGetLastError(), "transpose_kernel");
}

namespace {
void skinny_dispatch(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                     int64_t ldc, int64_t M, int N, int64_t K, const int* skip, uint16_t* planes,
                     int nplanes, int64_t ldp, int64_t pstride, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>((M + kRows - 1) / kRows);
  const int nq = (N + 3) / 4;
#define GWB_SKINNY(Q) \
  case Q:             \
    skinny_kernel<Q><<<grid, kWarps * 32, 0, s>>>(A, lda, B, ldb, C, ldc, M, N, K, skip, planes, \
                                                  nplanes, ldp, pstride);                     \
    break;
  switch (nq) {
    GWB_SKINNY(1)
    GWB_SKINNY(2)
    GWB_SKINNY(3)
    GWB_SKINNY(4)
    GWB_SKINNY(5)
    GWB_SKINNY(6)
    GWB_SKINNY(7)
    GWB_SKINNY(8)
    default:
      check_cuda(cudaErrorInvalidValue, "launch_skinny: N must be in [1, 32]");
  }
#undef GWB_SKINNY
  check_cuda(cudaGetLastError(), "skinny_kernel");
}
}  // namespace

void launch_skinny(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                   int64_t M, int N, int64_t K, const int* skip, cudaStream_t s) {
  skinny_dispatch(A, lda, B, ldb, C, ldc, M, N, K, skip, nullptr, 0, 0, 0, s);
}

void launch_skinny_planes(const float* A, int64_t lda, const float* B, int64_t ldb, void* planes,
                          int nplanes, int64_t ldp, int64_t pstride, int64_t M, int N, int64_t K,
                          const int* skip, cudaStream_t s) {
  if (ldp == 0 && (K > 32 || N > 32))
    check_cuda(cudaErrorInvalidValue, "launch_skinny_planes: packed output needs K, N <= 32");
  if (K <= 32 && N <= 32) {
    small_k_planes_kernel<<<static_cast<unsigned>((M + 31) / 32), 32 * kSmallKWarps, 0, s>>>(A, lda, B, ldb, M, N, static_cast<int>(K), skip,
                                    static_cast<uint16_t*>(planes), nplanes, ldp, pstride);
    check_cuda(cudaGetLastError(), "small_k_planes_kernel");
    return;
  }
  skinny_dispatch(A, lda, B, ldb, nullptr, 0, M, N, K, skip, static_cast<uint16_t*>(planes),
                  nplanes, ldp, pstride, s);
}

}  // namespace gwb
