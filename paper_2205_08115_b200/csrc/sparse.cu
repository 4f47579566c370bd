// sparse.cu — CSR construction and the column-blocked row-gather SpMM used
// by the sparse chain (see sparse.cuh).
//
// G = D_X · X · D_Yᵀ is evaluated as
//   Uᵀ = (D_X · X)ᵀ     row-gather over the rows of X, tile-transposed store
//   G  = (D_Y · Uᵀ)ᵀ    row-gather over the rows of Uᵀ, tile-transposed store
// so both products gather whole rows (coalesced float4) and both results land
// in the layouts the projection kernels already read (G row-major).
#include "sparse.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <vector>

namespace gwb {

void check_cuda(cudaError_t e, const char* what);  // solver.cu

#define GWB_CUDA_S(x) ::gwb::check_cuda((x), #x)

namespace {

constexpr int kTileRows = 32;   // output rows per CTA
constexpr int kVec = 2;         // float4 column groups per lane
constexpr int kTileCols = 128 * kVec;  // output columns per CTA
constexpr int kThreads = 256;   // 8 warps × 4 rows

__global__ void csr_count_kernel(const float* __restrict__ D, int64_t rows, int64_t ld,
                                 int32_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  if (i >= rows) return;
  const int lane = threadIdx.x & 31;
  int c = 0;
  for (int64_t j = lane; j < rows; j += 32) c += D[i * ld + j] != 0.0f;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[i] = c;
}

__global__ void csr_fill_kernel(const float* __restrict__ D, int64_t rows, int64_t ld,
                                const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                                float* __restrict__ val) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  if (i >= rows) return;
  const int lane = threadIdx.x & 31;
  int32_t off = row_ptr[i];
  for (int64_t j0 = 0; j0 < rows; j0 += 32) {
    const int64_t j = j0 + lane;
    const float v = j < rows ? D[i * ld + j] : 0.0f;
    const unsigned mask = __ballot_sync(0xffffffffu, v != 0.0f);
    if (v != 0.0f) {
      const int32_t p = off + __popc(mask & ((1u << lane) - 1u));
      col[p] = static_cast<int32_t>(j);
      val[p] = v;
    }
    off += __popc(mask);
  }
}

// One CTA: kTileRows output rows × kTileCols columns.  Warp w owns rows
// r0 + 4w … r0 + 4w + 3; lane l owns the float4 column groups
// c0 + 4l + 128v (v < kVec), so every gathered row segment is kVec coalesced
// 512-B loads.  Each row's (col, val) pairs are fetched 32 at a time with one
// coalesced load and broadcast by shuffles; four neighbours are gathered per
// step, i.e. 4·kVec independent loads in flight per lane (the kernel is
// L2-latency-bound).
template <bool kTranspose>
__global__ void __launch_bounds__(kThreads) rowgather_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
    const float* __restrict__ val, int64_t rows_out, const float* __restrict__ in,
    int64_t ld_in, int64_t cols, float* __restrict__ out, int64_t ld_out, const int* skip) {
  if (skip && *skip) return;
  // [v][column mod 4][column / 4 within the 128-block][row]: conflict-free on
  // the scatter (lanes vary column / 4) and the transposed read (lanes vary row).
  __shared__ float tile[kTranspose ? kVec : 1][kTranspose ? 4 : 1][kTranspose ? 32 : 1][kTileRows + 1];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kTileRows;
  int64_t c[kVec];
  bool col_ok[kVec];
  const float* in_c[kVec];
#pragma unroll
  for (int v = 0; v < kVec; ++v) {
    c[v] = static_cast<int64_t>(blockIdx.y) * kTileCols + 128 * v + lane * 4;
    col_ok[v] = c[v] < cols;  // ld_in, ld_out are multiples of 32: c..c+3 stay inside
    in_c[v] = in + (col_ok[v] ? c[v] : 0);
  }
#pragma unroll 1
  for (int rr = 0; rr < kTileRows / 8; ++rr) {
    const int lr = warp * (kTileRows / 8) + rr;
    const int64_t i = r0 + lr;
    float4 acc[kVec];
#pragma unroll
    for (int v = 0; v < kVec; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < rows_out) {
      const int32_t beg = row_ptr[i], end = row_ptr[i + 1];
      for (int32_t base = beg; base < end; base += 32) {
        const int cnt = min(32, end - base);
        const int32_t my_k = lane < cnt ? col[base + lane] : 0;
        const float my_a = lane < cnt ? val[base + lane] : 0.f;
        for (int t = 0; t < cnt; t += 4) {
          int32_t k[4];
          float a[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            k[u] = __shfl_sync(0xffffffffu, my_k, (t + u) & 31);
            a[u] = __shfl_sync(0xffffffffu, my_a, (t + u) & 31);
            if (t + u >= cnt) a[u] = 0.f;  // k[u] is a valid row (lane ≥ cnt loads row 0)
          }
          float4 x[4][kVec];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < kVec; ++v)
              x[u][v] = col_ok[v] ? __ldg(reinterpret_cast<const float4*>(
                                        in_c[v] + static_cast<int64_t>(k[u]) * ld_in))
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < kVec; ++v) {
              acc[v].x = fmaf(a[u], x[u][v].x, acc[v].x);
              acc[v].y = fmaf(a[u], x[u][v].y, acc[v].y);
              acc[v].z = fmaf(a[u], x[u][v].z, acc[v].z);
              acc[v].w = fmaf(a[u], x[u][v].w, acc[v].w);
            }
        }
      }
    }
#pragma unroll
    for (int v = 0; v < kVec; ++v) {
      if (!kTranspose) {
        if (i < rows_out && col_ok[v]) *reinterpret_cast<float4*>(out + i * ld_out + c[v]) = acc[v];
      } else {
        tile[v][0][lane][lr] = acc[v].x;
        tile[v][1][lane][lr] = acc[v].y;
        tile[v][2][lane][lr] = acc[v].z;
        tile[v][3][lane][lr] = acc[v].w;
      }
    }
  }
  if (kTranspose) {
    __syncthreads();
    // outᵀ rows = columns of the tile: kTileRows lanes per output row, so a
    // warp writes 32 / kTileRows rows of kTileRows floats per step.
    constexpr int kPer = 32 / kTileRows;
    const int sub = lane / kTileRows, li = lane % kTileRows;
    for (int c2 = warp * kPer; c2 < kTileCols; c2 += (kThreads / 32) * kPer) {
      const int cc = c2 + sub;
      const int64_t j = static_cast<int64_t>(blockIdx.y) * kTileCols + cc;
      const int64_t i = r0 + li;
      const int v = cc >> 7, w = cc & 127;
      if (j < cols && i < rows_out) out[j * ld_out + i] = tile[v][w & 3][w >> 2][li];
    }
  }
}

}  // namespace

Csr csr_from_dense(const float* D, int64_t rows, int64_t ld, cudaStream_t s) {
  Csr c;
  c.rows = rows;
  int32_t* cnt = nullptr;
  GWB_CUDA_S(cudaMalloc(&cnt, sizeof(int32_t) * (rows + 1)));
  const unsigned grid = static_cast<unsigned>((rows + 7) / 8);
  csr_count_kernel<<<grid, 256, 0, s>>>(D, rows, ld, cnt);
  GWB_CUDA_S(cudaGetLastError());
  std::vector<int32_t> h(static_cast<size_t>(rows) + 1, 0);
  GWB_CUDA_S(cudaMemcpyAsync(h.data() + 1, cnt, sizeof(int32_t) * rows, cudaMemcpyDeviceToHost, s));
  GWB_CUDA_S(cudaStreamSynchronize(s));
  int64_t total = 0;
  for (int64_t i = 1; i <= rows; ++i) {
    total += h[i];
    h[i] = static_cast<int32_t>(total);
  }
  if (total > 0x7fffffffLL) {
    cudaFree(cnt);
    throw std::invalid_argument("structure matrix too dense for the sparse chain (nnz > 2^31)");
  }
  c.nnz = total;
  c.row_ptr = cnt;  // reused as row_ptr (rows + 1 entries)
  GWB_CUDA_S(cudaMemcpyAsync(c.row_ptr, h.data(), sizeof(int32_t) * (rows + 1), cudaMemcpyHostToDevice, s));
  GWB_CUDA_S(cudaMalloc(&c.col, sizeof(int32_t) * std::max<int64_t>(total, 1)));
  GWB_CUDA_S(cudaMalloc(&c.val, sizeof(float) * std::max<int64_t>(total, 1)));
  csr_fill_kernel<<<grid, 256, 0, s>>>(D, rows, ld, c.row_ptr, c.col, c.val);
  GWB_CUDA_S(cudaGetLastError());
  GWB_CUDA_S(cudaStreamSynchronize(s));  // h goes out of scope
  return c;
}

void csr_free(Csr& c) {
  if (c.row_ptr) cudaFree(c.row_ptr);
  if (c.col) cudaFree(c.col);
  if (c.val) cudaFree(c.val);
  c = Csr{};
}

void launch_rowgather(const Csr& A, const float* in, int64_t ld_in, int64_t cols, float* out,
                      int64_t ld_out, bool transpose_out, const int* skip, cudaStream_t s) {
  // blockIdx.x (fastest) walks row tiles, so one column slab of `in`
  // (rows × 512 B) is shared by all CTAs in flight and stays in L2.
  const dim3 grid(static_cast<unsigned>((A.rows + kTileRows - 1) / kTileRows),
                  static_cast<unsigned>((cols + kTileCols - 1) / kTileCols));
  if (transpose_out)
    rowgather_kernel<true><<<grid, kThreads, 0, s>>>(A.row_ptr, A.col, A.val, A.rows, in, ld_in,
                                                     cols, out, ld_out, skip);
  else
    rowgather_kernel<false><<<grid, kThreads, 0, s>>>(A.row_ptr, A.col, A.val, A.rows, in, ld_in,
                                                      cols, out, ld_out, skip);
  GWB_CUDA_S(cudaGetLastError());
}

}  // namespace gwb
