// kernels.cu — HBM-bound BAPG half-step kernels, fused diagnostics and the
// boundary conversions (see kernels.cuh).  All row-major buffers have a
// leading dimension that is a multiple of 32 floats with zeroed padding, so
// float4 accesses never leave the allocation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "../../include/gwb.h"
#include "devutil.cuh"
#include "kernels.cuh"
#include "launch.cuh"
#include "narrow.cuh"

namespace gwb {
void check_cuda(cudaError_t e, const char* what);  // solver.cu: throws CudaError
}
#define GWB_CUDA_K(x) ::gwb::check_cuda((x), #x)

namespace gwb {

namespace {

using namespace dev;
constexpr int kRowThreads = 256;

// Half-step a: one CTA per row.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRowThreads) row_update_kernel(BapgDev d, int write, int tail) {
  pdl_enter();
  if (tail ? d.st->flags != 0 : d.st->done != 0) return;
  const int64_t i = blockIdx.x;
  const float* g = d.G + i * d.ld;
  const double* w = d.W64 + i * d.ld;
  const int64_t m = d.m;
  const double inv_rho = d.inv_rho64;

  Lse64 ms{-INFINITY, 0.0};
  double sums[2] = {0.0, 0.0};  // ⟨G,W⟩, ΣW
  for (int64_t j = threadIdx.x * 4; j < m; j += kRowThreads * 4) {
    const float4 g4 = *reinterpret_cast<const float4*>(g + j);
    double wv[4];
    load_d4(w + j, wv);
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (j + q < m) {
        lse64_add(ms, expo(gv[q], inv_rho), wv[q]);
        sums[0] = __fma_rn(static_cast<double>(gv[q]), wv[q], sums[0]);
        sums[1] += wv[q];
      }
    }
  }
  block_reduce64<kRowThreads, 2>(ms, sums);

  if (threadIdx.x == 0) {
    d.row_part[i].gw = sums[0];
    const double dev = sums[1] - d.mu64[i];
    d.row_part[i].rowdev = dev * dev;
  }
  if (!write) return;
  const double S = ms.s;
  const double r = ms.mx;
  if (threadIdx.x == 0) {
    if (r > 700.0) raise_flag(d.st, kFlagOverflowA);
    if (!(S > 0.0) || !isfinite(S) || isnan(r)) {
      raise_flag(d.st, kFlagZeroA);
      atomicMin(&d.st->zero_index, static_cast<int>(i));
    }
  }
  const double scale = d.mu64[i] / S;
  double* p = d.P64 + i * d.ld;
  for (int64_t j = threadIdx.x * 4; j < m; j += kRowThreads * 4) {
    const float4 g4 = *reinterpret_cast<const float4*>(g + j);
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
    double wv[4], o[4];
    load_d4(w + j, wv);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = (j + q < m) ? scale * wv[q] * exp(expo(gv[q], inv_rho) - r) : 0.0;
    store_d4(p + j, o);
    aux_store4_64(d.P_aux, d.P, d.aux_mode, d.plane, i * d.ld + j, o, d.aux_scale);
  }
}

// Half-step a for rows of m ≤ 1024·V (c1, c2): the row stays in registers,
// so it is read once, the max is found first and each exponential is
// evaluated once (the online (max, Σ) of row_update_kernel re-scales and
// evaluates two per element; on short rows that and the block merge, not
// HBM, bound the pass).  Same map, fp64 throughout.
template <int V>
__global__ void __launch_bounds__(kRowThreads) row_update_reg_kernel(BapgDev d, int write, int tail) {
  pdl_enter();
  if (tail ? d.st->flags != 0 : d.st->done != 0) return;
  const int64_t i = blockIdx.x;
  const float* g = d.G + i * d.ld;
  const double* w = d.W64 + i * d.ld;
  const int64_t m = d.m;
  const double inv_rho = d.inv_rho64;
  float gv[V][4];
  double wv[V][4];
  double mx = -INFINITY;
  bool nan = false;
  double sums[3] = {0.0, 0.0, 0.0};  // ⟨G,W⟩, ΣW, then Σ W e^{x − max}
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int64_t j = (threadIdx.x + static_cast<int64_t>(v) * kRowThreads) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      gv[v][q] = 0.f;
      wv[v][q] = 0.0;
    }
    if (j < m) {
      const float4 g4 = *reinterpret_cast<const float4*>(g + j);
      gv[v][0] = g4.x;
      gv[v][1] = g4.y;
      gv[v][2] = g4.z;
      gv[v][3] = g4.w;
      load_d4(w + j, wv[v]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (j + q < m) {
        const double x = expo(gv[v][q], inv_rho);
        nan = nan || isnan(x);
        mx = fmax(mx, x);
        sums[0] = __fma_rn(static_cast<double>(gv[v][q]), wv[v][q], sums[0]);
        sums[1] += wv[v][q];
      }
    }
  }
  // Block max (fixed-order butterfly + warp-0 merge) with the two sums.
  __shared__ double s_m[kRowThreads / 32];
  __shared__ int s_nan;
  if (threadIdx.x == 0) s_nan = 0;
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (nan) s_nan = 1;
  double r = s_m[0];
#pragma unroll
  for (int q = 1; q < kRowThreads / 32; ++q) r = fmax(r, s_m[q]);
  Lse64 dummy{-INFINITY, 0.0};
  double ds[2] = {sums[0], sums[1]};
  block_reduce64<kRowThreads, 2, false>(dummy, ds);  // its barriers also publish s_nan
  if (s_nan) r = NAN;
  if (threadIdx.x == 0) {
    d.row_part[i].gw = ds[0];
    const double dev = ds[1] - d.mu64[i];
    d.row_part[i].rowdev = dev * dev;
  }
  if (!write) return;
  double ev[V][4];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int64_t j = (threadIdx.x + static_cast<int64_t>(v) * kRowThreads) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ev[v][q] = (j + q < m) ? exp(expo(gv[v][q], inv_rho) - r) : 0.0;
      sums[2] = __fma_rn(wv[v][q], ev[v][q], sums[2]);
    }
  }
  double ss[1] = {sums[2]};
  block_reduce64<kRowThreads, 1, false>(dummy, ss);
  const double S = ss[0];
  if (threadIdx.x == 0) {
    if (r > 700.0) raise_flag(d.st, kFlagOverflowA);
    if (!(S > 0.0) || !isfinite(S) || isnan(r)) {
      raise_flag(d.st, kFlagZeroA);
      atomicMin(&d.st->zero_index, static_cast<int>(i));
    }
  }
  const double scale = d.mu64[i] / S;
  double* p = d.P64 + i * d.ld;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int64_t j = (threadIdx.x + static_cast<int64_t>(v) * kRowThreads) * 4;
    if (j >= m) break;
    double o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = (j + q < m) ? scale * wv[v][q] * ev[v][q] : 0.0;
    store_d4(p + j, o);
    aux_store4_64(d.P_aux, d.P, d.aux_mode, d.plane, i * d.ld + j, o, d.aux_scale);
  }
}

// Diagnostics-only row pass on fp32 iterates (quadratic geometry's tail
// record): ⟨G_i, W_i⟩ and (Σ_j W_ij − μ_i)².
__global__ void __launch_bounds__(kRowThreads) row_diag32_kernel(BapgDev d) {
  if (d.st->flags != 0) return;
  const int64_t i = blockIdx.x;
  double sums[2] = {0.0, 0.0};
  for (int64_t j = threadIdx.x; j < d.m; j += kRowThreads) {
    const double g = d.G[i * d.ld + j], w = d.W[i * d.ld + j];
    sums[0] = __fma_rn(g, w, sums[0]);
    sums[1] += w;
  }
  Lse64 dummy{-INFINITY, 0.0};
  block_reduce64<kRowThreads, 2, false>(dummy, sums);
  if (threadIdx.x == 0) {
    d.row_part[i].gw = sums[0];
    const double dev = sums[1] - d.mu64[i];
    d.row_part[i].rowdev = dev * dev;
  }
}

// Narrow rows (m ≤ kNarrowM, config 3): one warp per row, 8 rows per CTA
// (narrow.cuh: the row sits in registers between the (max, Σ) pass and the
// write, no block barriers).
constexpr int kWarpRows = kRowThreads / 32;

__global__ void __launch_bounds__(kRowThreads) row_update_warps_kernel(BapgDev d, int write, int tail) {
  pdl_enter();
  if (tail ? d.st->flags != 0 : d.st->done != 0) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kWarpRows + threadIdx.x / 32;
  if (i >= d.n) return;
  narrow_row_update<32>(d, i, d.G + i * d.ld, threadIdx.x & 31, true, write, nullptr);
}

// ---------------------------------------------------------------------------
// Half-step b, pass 1: per (row chunk, 128-column block) partials.
// ---------------------------------------------------------------------------
constexpr int kColThreads = 256;
constexpr int kColWidth = 128;  // columns per CTA (32 lanes × 4)

__global__ void __launch_bounds__(kColThreads) col_partial_kernel(BapgDev d, int rows_per_chunk) {
  pdl_enter();
  if (d.st->done || d.st->flags) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kColWidth + lane * 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = (r0 + rows_per_chunk < d.n) ? r0 + rows_per_chunk : d.n;
  const double inv_rho = d.inv_rho64;
  Lse64 ms[4] = {{-INFINITY, 0.0}, {-INFINITY, 0.0}, {-INFINITY, 0.0}, {-INFINITY, 0.0}};
  double ps[4] = {0.0, 0.0, 0.0, 0.0};
  if (c0 < d.m) {
    for (int64_t i = r0 + warp; i < r1; i += kColThreads / 32) {
      const float4 g4 = *reinterpret_cast<const float4*>(d.G + i * d.ld + c0);
      double pv[4];
      load_d4(d.P64 + i * d.ld + c0, pv);
      lse64_add(ms[0], expo(g4.x, inv_rho), pv[0]);
      lse64_add(ms[1], expo(g4.y, inv_rho), pv[1]);
      lse64_add(ms[2], expo(g4.z, inv_rho), pv[2]);
      lse64_add(ms[3], expo(g4.w, inv_rho), pv[3]);
#pragma unroll
      for (int q = 0; q < 4; ++q) ps[q] += pv[q];
    }
  }
  __shared__ double s_mx[kColThreads / 32][kColWidth];
  __shared__ double s_s[kColThreads / 32][kColWidth];
  __shared__ double s_p[kColThreads / 32][kColWidth];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    s_mx[warp][lane * 4 + q] = ms[q].mx;
    s_s[warp][lane * 4 + q] = ms[q].s;
    s_p[warp][lane * 4 + q] = ps[q];
  }
  __syncthreads();
  if (threadIdx.x < kColWidth) {
    const int c = threadIdx.x;
    const int64_t col = static_cast<int64_t>(blockIdx.x) * kColWidth + c;
    if (col < d.m) {
      Lse64 r{-INFINITY, 0.0};
      double p = 0.0;
      for (int q = 0; q < kColThreads / 32; ++q) {
        r = lse64_merge(r, Lse64{s_mx[q][c], s_s[q][c]});
        p += s_p[q][c];
      }
      const int64_t o = static_cast<int64_t>(blockIdx.y) * d.m + col;
      d.col_pmax[o] = r.mx;
      d.col_psum[o] = r.s;
      d.col_psump[o] = p;
    }
  }
}

// Pass 1 for narrow rows (m ≤ 32, config 3): lane = column, warp w takes the
// chunk's rows w, w+8, …; the 8 warps' partials merge in fixed order.  (The
// 128-column layout above leaves 27 of 32 lanes idle at m = 20.)
__global__ void __launch_bounds__(kColThreads) col_partial_narrow_kernel(BapgDev d, int rows_per_chunk) {
  pdl_enter();
  if (d.st->done || d.st->flags) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = (r0 + rows_per_chunk < d.n) ? r0 + rows_per_chunk : d.n;
  const double inv_rho = d.inv_rho64;
  const bool col = lane < d.m;
  Lse64 ms{-INFINITY, 0.0};
  double ps = 0.0;
  if (col) {
    int64_t i = r0 + warp;
    for (; i + 3 * (kColThreads / 32) < r1; i += 4 * (kColThreads / 32)) {
      float g[4];
      double p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t r = i + u * (kColThreads / 32);
        g[u] = d.G[r * d.ld + lane];
        p[u] = d.P64[r * d.ld + lane];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        lse64_add(ms, expo(g[u], inv_rho), p[u]);
        ps += p[u];
      }
    }
    for (; i < r1; i += kColThreads / 32) {
      const double p = d.P64[i * d.ld + lane];
      lse64_add(ms, expo(d.G[i * d.ld + lane], inv_rho), p);
      ps += p;
    }
  }
  __shared__ double s_mx[kColThreads / 32][32], s_s[kColThreads / 32][32], s_p[kColThreads / 32][32];
  s_mx[warp][lane] = ms.mx;
  s_s[warp][lane] = ms.s;
  s_p[warp][lane] = ps;
  __syncthreads();
  if (threadIdx.x < d.m) {
    const int c = threadIdx.x;
    Lse64 r{-INFINITY, 0.0};
    double p = 0.0;
    for (int q = 0; q < kColThreads / 32; ++q) {
      r = lse64_merge(r, Lse64{s_mx[q][c], s_s[q][c]});
      p += s_p[q][c];
    }
    const int64_t o = static_cast<int64_t>(blockIdx.y) * d.m + c;
    d.col_pmax[o] = r.mx;
    d.col_psum[o] = r.s;
    d.col_psump[o] = p;
  }
}

// Pass 1 for short chunks (≤ kShortRows rows per warp) in at most one wave
// of CTAs (c1, c3): the
// online (max, Σ) above runs one dependent fp64 exponential per row and two
// per warp merge, ~22 in sequence per lane, and that latency — not HBM — is
// the pass's time at these sizes.  Here the chunk's rows sit in registers:
// column maxima first (warp-local, then across the 8 warps through shared
// memory, no exponentials), then Σ π·e^{x − max} with independent
// exponentials and plain sums across warps.  Same partial (max, Σ, Σπ) per
// (chunk, column); NaN exponents give (NaN, NaN) as lse64 does.
constexpr int kShortRows = 8;

template <bool kNarrow>
__global__ void __launch_bounds__(kColThreads) col_partial_short_kernel(BapgDev d, int rows_per_chunk) {
  pdl_enter();
  if (d.st->done || d.st->flags) return;
  constexpr int C = kNarrow ? 1 : 4;           // columns per lane
  constexpr int kWarps = kColThreads / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t c0 = kNarrow ? lane : static_cast<int64_t>(blockIdx.x) * kColWidth + lane * 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = (r0 + rows_per_chunk < d.n) ? r0 + rows_per_chunk : d.n;
  const double inv_rho = d.inv_rho64;
  double x[kShortRows][C], pv[kShortRows][C];
  double mx[C], ps[C];
  bool nan[C];
#pragma unroll
  for (int q = 0; q < C; ++q) {
    mx[q] = -INFINITY;
    ps[q] = 0.0;
    nan[q] = false;
  }
  const bool live = c0 < d.m;
#pragma unroll
  for (int u = 0; u < kShortRows; ++u) {
    const int64_t i = r0 + warp + static_cast<int64_t>(u) * kWarps;
    const bool ok = live && i < r1;
#pragma unroll
    for (int q = 0; q < C; ++q) {
      x[u][q] = -INFINITY;
      pv[u][q] = 0.0;
    }
    if (ok) {
      if constexpr (kNarrow) {
        x[u][0] = expo(d.G[i * d.ld + c0], inv_rho);
        pv[u][0] = d.P64[i * d.ld + c0];
      } else {
        const float4 g4 = *reinterpret_cast<const float4*>(d.G + i * d.ld + c0);
        load_d4(d.P64 + i * d.ld + c0, pv[u]);
        x[u][0] = expo(g4.x, inv_rho);
        x[u][1] = expo(g4.y, inv_rho);
        x[u][2] = expo(g4.z, inv_rho);
        x[u][3] = expo(g4.w, inv_rho);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < kShortRows; ++u)
#pragma unroll
    for (int q = 0; q < C; ++q) {
      nan[q] = nan[q] || isnan(x[u][q]);
      mx[q] = fmax(mx[q], x[u][q]);
      ps[q] += pv[u][q];
    }
  __shared__ double s_mx[kWarps][kColWidth];
  __shared__ double s_s[kWarps][kColWidth];
  __shared__ double s_p[kWarps][kColWidth];
#pragma unroll
  for (int q = 0; q < C; ++q) s_mx[warp][lane * C + q] = nan[q] ? NAN : mx[q];
  __syncthreads();
  double M[C], sum[C];
#pragma unroll
  for (int q = 0; q < C; ++q) {
    double v = s_mx[0][lane * C + q];
    bool bad = isnan(v);
#pragma unroll
    for (int k = 1; k < kWarps; ++k) {
      const double t = s_mx[k][lane * C + q];
      bad = bad || isnan(t);
      v = fmax(v, t);
    }
    M[q] = bad ? NAN : v;
    sum[q] = 0.0;
  }
#pragma unroll
  for (int u = 0; u < kShortRows; ++u)
#pragma unroll
    for (int q = 0; q < C; ++q) {
      const double e = x[u][q] == -INFINITY ? 0.0 : exp(x[u][q] - M[q]);
      sum[q] = __fma_rn(pv[u][q], e, sum[q]);
    }
#pragma unroll
  for (int q = 0; q < C; ++q) {
    s_s[warp][lane * C + q] = sum[q];
    s_p[warp][lane * C + q] = ps[q];
  }
  __syncthreads();
  if (threadIdx.x < (kNarrow ? 32 : kColWidth)) {
    const int c = threadIdx.x;
    const int64_t col = kNarrow ? c : static_cast<int64_t>(blockIdx.x) * kColWidth + c;
    if (col < d.m) {
      double mc = s_mx[0][c];
      bool bad = isnan(mc);
      double sc = 0.0, p = 0.0;
      for (int k = 0; k < kWarps; ++k) {
        const double t = s_mx[k][c];
        bad = bad || isnan(t);
        mc = fmax(mc, t);
        sc += s_s[k][c];
        p += s_p[k][c];
      }
      const int64_t o = static_cast<int64_t>(blockIdx.y) * d.m + col;
      d.col_pmax[o] = bad ? NAN : mc;
      d.col_psum[o] = bad ? NAN : sc;
      d.col_psump[o] = p;
    }
  }
}

// Half-step b, pass 2: merge chunk partials per column, raise errors.  One
// warp per column: lanes take the row chunks, then a fixed-order warp merge.
__global__ void col_combine_kernel(BapgDev d) {
  pdl_enter();
  if (d.st->done || d.st->flags) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  if (j >= d.m) return;
  const int lane = threadIdx.x & 31;
  Lse64 r{-INFINITY, 0.0};
  double p = 0.0;
  for (int c = lane; c < d.chunks; c += 32) {
    const int64_t o = static_cast<int64_t>(c) * d.m + j;
    r = lse64_merge(r, Lse64{d.col_pmax[o], d.col_psum[o]});
    p += d.col_psump[o];
  }
  r = lse64_warp_merge(r);
  p = warp_sum(p);
  if (lane != 0) return;
  if (r.mx > 700.0) raise_flag(d.st, kFlagOverflowB);
  if (!(r.s > 0.0) || !isfinite(r.s) || isnan(r.mx)) {
    raise_flag(d.st, kFlagZeroB);
    atomicMin(&d.st->zero_index, static_cast<int>(j));
  }
  d.col_max[j] = r.mx;
  d.col_scale[j] = d.nu64[j] / r.s;
  const double dev = p - d.nu64[j];
  d.col_dev[j] = dev * dev;
}

// One element of the half-step-b write: w' = scale_j · π · e^{x − max_j},
// with the fused record partials (gw, split, diff, wold, gp).
template <int kN>
__device__ __forceinline__ double col_write_elem(float g, double p, double w, double mx,
                                                 double sc, double inv_rho, double (&sums)[kN],
                                                 bool& finite) {
  const double o = sc * p * exp(expo(g, inv_rho) - mx);
  finite = finite && isfinite(o);
  sums[0] = __fma_rn(static_cast<double>(g), o, sums[0]);
  const double sp = p - o;
  sums[1] = __fma_rn(sp, sp, sums[1]);
  const double df = o - w;
  sums[2] = __fma_rn(df, df, sums[2]);
  sums[3] = __fma_rn(w, w, sums[3]);
  sums[4] = __fma_rn(static_cast<double>(g), p, sums[4]);
  return o;
}

// Half-step b, pass 3: write W_new, fused diagnostics. One CTA per row.
__global__ void __launch_bounds__(kRowThreads) col_write_kernel(BapgDev d) {
  pdl_enter();
  if (d.st->done) return;
  if (d.st->flags != 0) return;
  const int64_t i = blockIdx.x;
  const float* g = d.G + i * d.ld;
  const double* p = d.P64 + i * d.ld;
  const double* wo = d.W64 + i * d.ld;
  double* wn = d.W64_new + i * d.ld;
  const double inv_rho = d.inv_rho64;
  const int64_t m = d.m;
  double sums[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // gw, split, diff, wold, gp, ΣW'
  bool finite = true;
  for (int64_t j = threadIdx.x * 4; j < m; j += kRowThreads * 4) {
    const float4 g4 = *reinterpret_cast<const float4*>(g + j);
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
    double pv[4], wv[4], mv[4], sv[4], o[4];
    load_d4(p + j, pv);
    load_d4(wo + j, wv);
    load_d4(d.col_max + j, mv);
    load_d4(d.col_scale + j, sv);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      o[q] = (j + q < m) ? col_write_elem(gv[q], pv[q], wv[q], mv[q], sv[q], inv_rho, sums, finite)
                         : 0.0;
      sums[5] += o[q];
    }
    store_d4(wn + j, o);
    aux_store4_64(d.W_aux, d.W_new, d.aux_mode, d.plane, i * d.ld + j, o, d.aux_scale);
  }
  Lse64 dummy{-INFINITY, 0.0};
  block_reduce64<kRowThreads, 6, false>(dummy, sums);
  if (!__syncthreads_and(finite ? 1 : 0) && threadIdx.x == 0)
    raise_flag(d.st, kFlagNonFinite);
  if (threadIdx.x == 0) {
    ColWritePart& c = d.cw_part[i];
    c.gw = sums[0];
    c.split = sums[1];
    c.diff = sums[2];
    c.wold = sums[3];
    c.gp = sums[4];
    if (d.wsum_bias) d.wsum_bias[i] = static_cast<float>(d.wsum_factor * sums[5]);
  }
}

// col_write for narrow rows (m ≤ 128): one warp per row, as row_update_warps.
__global__ void __launch_bounds__(kRowThreads) col_write_warps_kernel(BapgDev d) {
  pdl_enter();
  if (d.st->done) return;
  if (d.st->flags != 0) return;
  const int lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kWarpRows + threadIdx.x / 32;
  if (i >= d.n) return;
  const int64_t m = d.m;
  const double inv_rho = d.inv_rho64;
  double sums[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // gw, split, diff, wold, gp, ΣW'
  bool finite = true;
#pragma unroll 2
  for (int v = 0; v < kNarrowV; ++v) {
    const int64_t j = lane * 4 + 128 * v;
    if (j >= m) break;
    const float4 g4 = *reinterpret_cast<const float4*>(d.G + i * d.ld + j);
    const float gv[4] = {g4.x, g4.y, g4.z, g4.w};
    double pv[4], wv[4], mv[4], sv[4], o[4];
    load_d4(d.P64 + i * d.ld + j, pv);
    load_d4(d.W64 + i * d.ld + j, wv);
    load_d4(d.col_max + j, mv);
    load_d4(d.col_scale + j, sv);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      o[q] = (j + q < m) ? col_write_elem(gv[q], pv[q], wv[q], mv[q], sv[q], inv_rho, sums, finite)
                         : 0.0;
      sums[5] += o[q];
    }
    store_d4(d.W64_new + i * d.ld + j, o);
    aux_store4_64(d.W_aux, d.W_new, d.aux_mode, d.plane, i * d.ld + j, o, d.aux_scale);
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) sums[q] = warp_sum(sums[q]);
  if (!__all_sync(0xffffffffu, finite ? 1 : 0) && lane == 0) raise_flag(d.st, kFlagNonFinite);
  if (lane == 0) {
    ColWritePart& c = d.cw_part[i];
    c.gw = sums[0];
    c.split = sums[1];
    c.diff = sums[2];
    c.wold = sums[3];
    c.gp = sums[4];
    if (d.wsum_bias) d.wsum_bias[i] = static_cast<float>(d.wsum_factor * sums[5]);
  }
}

constexpr int kFinThreads = 512;

__global__ void __launch_bounds__(kFinThreads) finalize_kernel(BapgDev d, double rel_tol, int tail) {
  pdl_enter();
  DevStatus* st = d.st;
  if (tail ? st->flags != 0 : st->done != 0) return;
  if (!tail && st->flags != 0) {  // raised this iteration (raise_flag): stop here
    if (threadIdx.x == 0) st->done = 1;
    return;
  }
  const int k = tail ? st->iter - 1 : st->iter;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // acc: 0 gw_row, 1 rowdev, 2 cw.gw, 3 split, 4 diff, 5 wold, 6 gp, 7 coldev
  for (int64_t i = threadIdx.x; i < d.n; i += kFinThreads) {
    acc[0] += d.row_part[i].gw;
    acc[1] += d.row_part[i].rowdev;
    if (!tail) {
      const ColWritePart c = d.cw_part[i];
      acc[2] += c.gw;
      acc[3] += c.split;
      acc[4] += c.diff;
      acc[5] += c.wold;
      acc[6] += c.gp;
    }
  }
  if (!tail)
    for (int64_t j = threadIdx.x; j < d.m; j += kFinThreads) acc[7] += d.col_dev[j];
  __shared__ double s[8][kFinThreads / 32];
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double v = warp_sum(acc[q]);
    if (l == 0) s[q][w] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  double t[8];
  for (int q = 0; q < 8; ++q) {
    t[q] = 0.0;
    for (int r = 0; r < kFinThreads / 32; ++r) t[q] += s[q][r];
  }
  // Iterations past max_rec (session API) share a scratch slot.
  auto slot = [&](int it) { return it <= d.max_rec ? it : d.max_rec + 1; };
  if (tail) {
    d.rec[slot(k)].mw_w = t[0];
    d.rec[slot(k)].row_sq = t[1];
    return;
  }
  if (k >= 2) {  // the row pass of iteration k saw w^{k-1}
    d.rec[slot(k - 1)].mw_w = t[0];
    d.rec[slot(k - 1)].row_sq = t[1];
  }
  DevRecord& r = d.rec[slot(k)];
  r.mpi_w = t[2];
  r.split_sq = t[3];
  r.diff_sq = t[4];
  r.wold_sq = t[5];
  r.mpi_pi = t[6];
  r.col_sq = t[7];
  r.elapsed = 1e-9 * static_cast<double>(globaltimer() - st->t0);
  const double rel = sqrt(t[4]) / sqrt(t[5]);
  st->iter = k + 1;
  // fp64 iterates: the reference's rule as is (solvers.cpp:208), including
  // exact fp64 fixed points (rel_change == 0) under a pinned rel_tol; fp32
  // iterates (quadratic geometry): dev::stop_rule.
  if (d.P64 ? rel <= rel_tol : stop_rule(rel, rel_tol)) {
    st->converged = 1;
    st->done = 1;
  }
}

__global__ void status_reset_kernel(DevStatus* st) {
  st->done = 0;
  st->flags = 0;
  st->iter = 1;
  st->err_iter = 0;
  st->converged = 0;
  st->zero_index = 0x7fffffff;
  st->sink_sweeps = 0;
  st->sink_err_sweep = 0;
  st->gdone = 0;
  st->t0 = globaltimer();
}

// ---------------------------------------------------------------------------
// Conversions.
// ---------------------------------------------------------------------------
template <class T>
__global__ void c64_to_r32_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                  T* __restrict__ dst, int64_t ld) {
  __shared__ T tile[32][33];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;  // row block
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * 32;  // col block
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + y;
    if (i < rows && j < cols) tile[y][threadIdx.x] = static_cast<T>(src[j * rows + i]);
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t i = i0 + y, j = j0 + threadIdx.x;
    if (i < rows && j < cols) dst[i * ld + j] = tile[threadIdx.x][y];
  }
}

template <class T>
__global__ void row_sums64_kernel(const T* src, int64_t rows, int64_t cols, int64_t ld,
                                  double* out) {
  const int64_t i = blockIdx.x;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) s += src[i * ld + j];
  s = warp_sum(s);
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < static_cast<int>(blockDim.x / 32); ++q) t += sh[q];
    out[i] = t;
  }
}

template <class T>
__global__ void col_sums64_kernel(const T* src, int64_t rows, int64_t cols, int64_t ld,
                                  double* out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= cols) return;
  double s = 0.0;
  for (int64_t i = 0; i < rows; ++i) s += src[i * ld + j];
  out[j] = s;
}

template <class T>
__global__ void r32_to_c64_kernel(const T* __restrict__ src, int64_t rows, int64_t cols,
                                  int64_t ld, double* __restrict__ dst, int axis,
                                  const double* __restrict__ target,
                                  const double* __restrict__ sums) {
  __shared__ double tile[32][33];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t i = i0 + y, j = j0 + threadIdx.x;
    if (i < rows && j < cols) {
      double v = static_cast<double>(src[i * ld + j]);
      if (axis == 0) v *= target[i] / sums[i];
      if (axis == 1) v *= target[j] / sums[j];
      tile[y][threadIdx.x] = v;
    }
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t j = j0 + y, i = i0 + threadIdx.x;
    if (i < rows && j < cols) dst[j * rows + i] = tile[threadIdx.x][y];
  }
}

__global__ void average64_kernel(const double* a, const double* b, double* dst, int64_t len) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = 0.5 * (a[k] + b[k]);
}

__global__ void tf32_aux_kernel(const float* x, int64_t rows, int64_t cols, int64_t ld,
                                float* out, int mode, int64_t plane, float scale) {
  const int64_t i = blockIdx.x;
  // ld is a multiple of 32, so whole float4 groups stay inside the row pitch.
  for (int64_t j = threadIdx.x * 4; j < cols; j += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(x + i * ld + j);
    aux_store4(out, mode, plane, i * ld + j, v.x, v.y, v.z, v.w, scale);
  }
}

__global__ void to_bf16_kernel(const float* x, int64_t rows, int64_t cols, int64_t ld,
                               __nv_bfloat16* out) {
  const int64_t i = blockIdx.x;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
    out[i * ld + j] = __float2bfloat16_rn(x[i * ld + j]);
}

__global__ void to_f16_kernel(const float* x, int64_t rows, int64_t cols, int64_t ld, __half* out) {
  const int64_t i = blockIdx.x;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
    out[i * ld + j] = __float2half_rn(x[i * ld + j]);
}

// f16x2 row scales of the GEMM1 output Vᵀ = D_Y·Xᵀ (f16x2).
// Row i of Vᵀ is bounded a priori by x_max · Σ_l |D_Y[i][l]| (x_max bounds
// every iterate entry: π_kl ≤ μ_k, w_kl ≤ ν_l), so σ_i = 14 − ⌈log2 bound⌉
// keeps Vᵀ[i,:]·2^σ_i ≤ 2^14 inside fp16 range.  GEMM1 accumulates
// 2^s1·Vᵀ (its B planes carry 2^s1), so its row scale is 2^(σ_i − s1);
// GEMM2's column scale 2^−σ_j undoes σ.  All scales are powers of two.
__global__ void f16_scales_kernel(const float* D, int64_t m, int64_t ld, float x_max, int s1,
                                  int sa1, int sa2, float* g1_row_scale, float* g2_col_scale) {
  const int64_t i = blockIdx.x;
  double acc = 0.0;
  for (int64_t l = threadIdx.x; l < m; l += blockDim.x) acc += fabs(static_cast<double>(D[i * ld + l]));
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double part[32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) sum += part[w];
    const double bound = static_cast<double>(x_max) * sum;
    int sigma = 0;
    if (bound > 0.0) sigma = 14 - static_cast<int>(ceil(log2(bound)));
    sigma = max(-100, min(100, sigma));
    g1_row_scale[i] = ldexpf(1.0f, sigma - s1 - sa1);
    g2_col_scale[i] = ldexpf(1.0f, -sigma - sa2);
  }
}

template <class T>
__global__ void product_coupling_kernel(const T* mu, const T* nu, int64_t n, int64_t m,
                                        int64_t ld, T* P) {
  const int64_t i = blockIdx.x;
  const T a = mu[i];
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) P[i * ld + j] = a * nu[j];
}

// fp32 copy / GEMM operand planes of an fp64 iterate (ld multiple of 4).
__global__ void iterate_copies_kernel(const double* x, int64_t cols, int64_t ld, float* copy32,
                                      float* aux, int mode, int64_t plane, float scale) {
  const int64_t i = blockIdx.x;
  for (int64_t j = threadIdx.x * 4; j < cols; j += blockDim.x * 4) {
    double v[4];
    load_d4(x + i * ld + j, v);
    aux_store4_64(aux, copy32, mode, plane, i * ld + j, v, scale);
  }
}

// Centred operand copies of a structure matrix: x = D − c in fp64.
__global__ void center_copies_kernel(const float* D, int64_t cols, int64_t ld, double c,
                                     float* copy32, float* aux, int mode, int64_t plane,
                                     float scale) {
  const int64_t i = blockIdx.x;
  for (int64_t j = threadIdx.x * 4; j < cols; j += blockDim.x * 4) {
    const float4 f = *reinterpret_cast<const float4*>(D + i * ld + j);
    const float fv[4] = {f.x, f.y, f.z, f.w};
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = j + q < cols ? static_cast<double>(fv[q]) - c : 0.0;
    aux_store4_64(aux, copy32, mode, plane, i * ld + j, v, scale);
  }
}

// out[i] = factor · Σ_j x[i][j], one warp per row, fixed order.
__global__ void row_bias64_kernel(const double* x, int64_t rows, int64_t cols, int64_t ld,
                                  double factor, float* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
  if (i >= rows) return;
  double t = 0.0;
  for (int64_t j = threadIdx.x & 31; j < cols; j += 32) t += x[i * ld + j];
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) out[i] = static_cast<float>(factor * t);
}

__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  // valid for v >= 0 (structure matrices are nonnegative)
  atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}

__global__ void analyze_kernel(const float* D, int64_t rows, int64_t cols, int64_t ld,
                               float* out_max, int* out_inexact) {
  const int64_t i = blockIdx.x;
  float mx = 0.f;
  int inexact = 0;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
    const float v = D[i * ld + j];
    mx = fmaxf(mx, v);
    inexact |= (v != trunc_tf32(v)) ? 1 : 0;
    inexact |= (v != bf16_round(v)) ? 2 : 0;
    inexact |= (fabsf(v) > 65504.0f || v != __half2float(__float2half_rn(v))) ? 4 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    inexact |= __shfl_xor_sync(0xffffffffu, inexact, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(out_max, mx);
    if (inexact) atomicOr(out_inexact, inexact);
  }
}

inline unsigned grid1d(int64_t work, int threads) {
  return static_cast<unsigned>((work + threads - 1) / threads);
}

}  // namespace

namespace {
void launch_col_write_pass(const BapgDev& d, cudaStream_t s) {
  if (d.m <= kNarrowM)
    launch_pdl(col_write_warps_kernel, dim3(static_cast<unsigned>((d.n + kWarpRows - 1) / kWarpRows)),
               dim3(kRowThreads), 0, s, d);
  else
    launch_pdl(col_write_kernel, dim3(static_cast<unsigned>(d.n)), dim3(kRowThreads), 0, s, d);
}
}  // namespace

namespace {
void launch_col_partial_pass(const BapgDev& d, dim3 grid, int rows_per_chunk, cudaStream_t s) {
  // GWB_COL_ONLINE=1 keeps the online (max, Σ) pass at every size (A/B knob).
  static const bool online_env = [] {
    const char* e = std::getenv("GWB_COL_ONLINE");
    return e && e[0] == '1';
  }();
  // Short form only where the pass is at most one wave of CTAs, i.e. bound by
  // one CTA's latency (c1 +2.8%, c3 +1.2%); with several CTAs per SM the
  // online form's streaming loads win (c2: −2.9% with the short form).
  const int64_t ctas = static_cast<int64_t>(d.m <= 32 ? 1 : grid.x) * d.chunks;
  const bool is_short =
      !online_env && rows_per_chunk <= kShortRows * (kColThreads / 32) && ctas <= 148;
  const dim3 narrow_grid(1, static_cast<unsigned>(d.chunks));
  if (d.m <= 32 && is_short)
    launch_pdl(col_partial_short_kernel<true>, narrow_grid, dim3(kColThreads), 0, s, d, rows_per_chunk);
  else if (d.m <= 32)
    launch_pdl(col_partial_narrow_kernel, narrow_grid, dim3(kColThreads), 0, s, d, rows_per_chunk);
  else if (is_short)
    launch_pdl(col_partial_short_kernel<false>, grid, dim3(kColThreads), 0, s, d, rows_per_chunk);
  else
    launch_pdl(col_partial_kernel, grid, dim3(kColThreads), 0, s, d, rows_per_chunk);
}
}  // namespace

void launch_row_update(const BapgDev& d, bool write, cudaStream_t s) {
  if (!d.P64) {  // fp32 iterates (quadratic geometry): diagnostics only
    if (!write && d.n >= 1) row_diag32_kernel<<<static_cast<unsigned>(d.n), kRowThreads, 0, s>>>(d);
    return;
  }
  if (d.n >= 1 && d.m <= kNarrowM)
    launch_pdl(row_update_warps_kernel, dim3(static_cast<unsigned>((d.n + kWarpRows - 1) / kWarpRows)),
               dim3(kRowThreads), 0, s, d, write ? 1 : 0, write ? 0 : 1);
  else if (d.n >= 1 && d.m <= 1024)
    launch_pdl(row_update_reg_kernel<1>, dim3(static_cast<unsigned>(d.n)), dim3(kRowThreads), 0, s, d,
               write ? 1 : 0, write ? 0 : 1);
  else if (d.n >= 1 && d.m <= 2048)
    launch_pdl(row_update_reg_kernel<2>, dim3(static_cast<unsigned>(d.n)), dim3(kRowThreads), 0, s, d,
               write ? 1 : 0, write ? 0 : 1);
  else if (d.n >= 1 && d.m <= 4096)
    launch_pdl(row_update_reg_kernel<4>, dim3(static_cast<unsigned>(d.n)), dim3(kRowThreads), 0, s, d,
               write ? 1 : 0, write ? 0 : 1);
  else if (d.n >= 1)
    launch_pdl(row_update_kernel, dim3(static_cast<unsigned>(d.n)), dim3(kRowThreads), 0, s, d,
               write ? 1 : 0, write ? 0 : 1);
}

void launch_col_update(const BapgDev& d, cudaStream_t s) {
  const int rows_per_chunk = static_cast<int>((d.n + d.chunks - 1) / d.chunks);
  dim3 grid(static_cast<unsigned>((d.m + kColWidth - 1) / kColWidth),
            static_cast<unsigned>(d.chunks));
  launch_col_partial_pass(d, grid, rows_per_chunk, s);
  launch_pdl(col_combine_kernel, dim3(grid1d(d.m * 32, 256)), dim3(256), 0, s, d);
  launch_col_write_pass(d, s);
}

void launch_col_partial(const BapgDev& d, cudaStream_t s) {
  if (d.n < 1) return;
  const int rows_per_chunk = static_cast<int>((d.n + d.chunks - 1) / d.chunks);
  dim3 grid(static_cast<unsigned>((d.m + kColWidth - 1) / kColWidth),
            static_cast<unsigned>(d.chunks));
  launch_col_partial_pass(d, grid, rows_per_chunk, s);
}

void launch_col_write(const BapgDev& d, cudaStream_t s) {
  if (d.n >= 1) launch_col_write_pass(d, s);
}

void launch_finalize(const BapgDev& d, double rel_tol, bool tail, cudaStream_t s) {
  launch_pdl(finalize_kernel, dim3(1), dim3(kFinThreads), 0, s, d, rel_tol, tail ? 1 : 0);
}

void launch_status_reset(DevStatus* st, cudaStream_t s) { status_reset_kernel<<<1, 1, 0, s>>>(st); }

void launch_colmajor64_to_rowmajor32(const double* src, int64_t rows, int64_t cols, float* dst,
                                     int64_t ld, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
  c64_to_r32_kernel<float><<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, dst, ld);
}

void launch_colmajor64_to_rowmajor64(const double* src, int64_t rows, int64_t cols, double* dst,
                                     int64_t ld, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
  c64_to_r32_kernel<double><<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, dst, ld);
}

template <class T>
static void to_colmajor64(const T* src, int64_t rows, int64_t cols, int64_t ld, double* dst,
                          int axis, const double* target, double* work, cudaStream_t s) {
  if (axis == 0) row_sums64_kernel<T><<<static_cast<unsigned>(rows), 256, 0, s>>>(src, rows, cols, ld, work);
  if (axis == 1) col_sums64_kernel<T><<<grid1d(cols, 256), 256, 0, s>>>(src, rows, cols, ld, work);
  dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
  r32_to_c64_kernel<T><<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, ld, dst, axis, target, work);
}

void launch_rowmajor32_to_colmajor64(const float* src, int64_t rows, int64_t cols, int64_t ld,
                                     double* dst, int axis, const double* target, double* work,
                                     cudaStream_t s) {
  to_colmajor64(src, rows, cols, ld, dst, axis, target, work, s);
}

void launch_rowmajor64_to_colmajor64(const double* src, int64_t rows, int64_t cols, int64_t ld,
                                     double* dst, int axis, const double* target, double* work,
                                     cudaStream_t s) {
  to_colmajor64(src, rows, cols, ld, dst, axis, target, work, s);
}

void launch_iterate_copies(const double* x, int64_t rows, int64_t cols, int64_t ld, float* copy32,
                           float* aux, int mode, float scale, cudaStream_t s) {
  if (rows < 1 || (!copy32 && !aux)) return;
  iterate_copies_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(x, cols, ld, copy32, aux, mode,
                                                                    rows * ld, scale);
}

void launch_center_copies(const float* D, int64_t rows, int64_t cols, int64_t ld, double c,
                          float* copy32, float* aux, int mode, float scale, cudaStream_t s) {
  if (rows < 1 || (!copy32 && !aux)) return;
  center_copies_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(D, cols, ld, c, copy32, aux, mode,
                                                                   rows * ld, scale);
}

void launch_row_bias64(const double* x, int64_t rows, int64_t cols, int64_t ld, double factor,
                       float* out, cudaStream_t s) {
  if (rows < 1) return;
  row_bias64_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(x, rows, cols, ld, factor, out);
}

void launch_product_coupling64(const double* mu, const double* nu, int64_t n, int64_t m, int64_t ld,
                               double* P, cudaStream_t s) {
  product_coupling_kernel<double><<<static_cast<unsigned>(n), 256, 0, s>>>(mu, nu, n, m, ld, P);
}

void launch_average64(const double* a, const double* b, double* dst, int64_t len, cudaStream_t s) {
  average64_kernel<<<1184, 256, 0, s>>>(a, b, dst, len);
}

void launch_tf32_aux(const float* x, int64_t rows, int64_t cols, int64_t ld, float* out, int mode,
                     cudaStream_t s, float scale) {
  tf32_aux_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(x, rows, cols, ld, out, mode,
                                                               rows * ld, scale);
}

void launch_to_f16(const float* x, int64_t rows, int64_t cols, int64_t ld, void* out,
                   cudaStream_t s) {
  to_f16_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(x, rows, cols, ld,
                                                            static_cast<__half*>(out));
}

void launch_f16_scales(const float* D, int64_t m, int64_t ld, float x_max, int s1,
                       float* g1_row_scale, float* g2_col_scale, cudaStream_t s, int sa1,
                       int sa2) {
  f16_scales_kernel<<<static_cast<unsigned>(m), 256, 0, s>>>(D, m, ld, x_max, s1, sa1, sa2,
                                                             g1_row_scale, g2_col_scale);
}

void launch_to_bf16(const float* x, int64_t rows, int64_t cols, int64_t ld, void* out,
                    cudaStream_t s) {
  to_bf16_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(x, rows, cols, ld,
                                                             static_cast<__nv_bfloat16*>(out));
}

void launch_analyze(const float* D, int64_t rows, int64_t cols, int64_t ld, float* out_max,
                    int* out_inexact, cudaStream_t s) {
  analyze_kernel<<<static_cast<unsigned>(rows), 256, 0, s>>>(D, rows, cols, ld, out_max, out_inexact);
}

int analyze_inexact(const float* D, int64_t rows, int64_t cols, int64_t ld, cudaStream_t s) {
  if (rows < 1 || cols < 1) return 0;
  void* buf = nullptr;
  GWB_CUDA_K(cudaMallocAsync(&buf, 16, s));
  GWB_CUDA_K(cudaMemsetAsync(buf, 0, 16, s));
  float* d_max = static_cast<float*>(buf);
  int* d_inexact = reinterpret_cast<int*>(static_cast<char*>(buf) + 8);
  launch_analyze(D, rows, cols, ld, d_max, d_inexact, s);
  int h = 0;
  GWB_CUDA_K(cudaMemcpyAsync(&h, d_inexact, sizeof(h), cudaMemcpyDeviceToHost, s));
  GWB_CUDA_K(cudaFreeAsync(buf, s));
  GWB_CUDA_K(cudaStreamSynchronize(s));
  return h;
}

bool split_exact(int precision, int inexact_bits) {
  if (precision == GWB_PREC_F16X2) return (inexact_bits & 4) == 0;
  if (precision == GWB_PREC_BF16X3 || precision == GWB_PREC_BF16X2) return (inexact_bits & 2) == 0;
  return true;
}

void launch_product_coupling(const float* mu, const float* nu, int64_t n, int64_t m, int64_t ld,
                             float* P, cudaStream_t s) {
  product_coupling_kernel<float><<<static_cast<unsigned>(n), 256, 0, s>>>(mu, nu, n, m, ld, P);
}

namespace {
__global__ void adjacency_kernel(const int2* __restrict__ e, int64_t count, float* D, int64_t ld) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int2 p = e[k];
    D[static_cast<int64_t>(p.x) * ld + p.y] = 1.0f;
    D[static_cast<int64_t>(p.y) * ld + p.x] = 1.0f;
  }
}
}  // namespace

void build_adjacency(const int32_t* edges_host, int64_t count, int64_t rows, float* D, int64_t ld,
                     cudaStream_t s) {
  GWB_CUDA_K(cudaMemsetAsync(D, 0, sizeof(float) * static_cast<size_t>(rows) * ld, s));
  if (count <= 0) return;
  int2* e = nullptr;
  GWB_CUDA_K(cudaMallocAsync(reinterpret_cast<void**>(&e), sizeof(int2) * count, s));
  GWB_CUDA_K(cudaMemcpyAsync(e, edges_host, sizeof(int2) * count, cudaMemcpyHostToDevice, s));
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 148 * 8);
  adjacency_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(e, count, D, ld);
  GWB_CUDA_K(cudaGetLastError());
  GWB_CUDA_K(cudaFreeAsync(e, s));
}

// ---------------------------------------------------------------------------
// Post-solve readout (column-major fp64 couplings).
// ---------------------------------------------------------------------------
namespace {
__global__ void rowsums_cm64_kernel(const double* pi, int64_t n, int64_t m, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t j = 0; j < m; ++j) s += pi[j * n + i];  // coalesced across threads
  out[i] = s;
}

__global__ void colsums_cm64_kernel(const double* pi, int64_t n, int64_t m, double* out) {
  const int64_t j = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += pi[j * n + i];
  s = warp_sum(s);
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += sh[w];
    out[j] = t;
  }
}

__global__ void argmax_rows_cm64_kernel(const double* pi, int64_t n, int64_t m, int32_t* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t best = 0;
  double bv = pi[i];
  for (int64_t j = 1; j < m; ++j) {
    const double v = pi[j * n + i];
    if (v > bv) {
      bv = v;
      best = j;
    }
  }
  out[i] = static_cast<int32_t>(best);
}

__global__ void sqdiff_kernel(const double* a, const double* b, int64_t len, double* part) {
  double t = 0.0;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double d = b ? a[k] - b[k] : a[k];
    t += d * d;
  }
  t = warp_sum(t);
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) u += sh[w];
    part[blockIdx.x] = u;
  }
}

__global__ void count_equal_kernel(const int32_t* a, const int32_t* b, int64_t len,
                                   unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += a[k] == b[k];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);  // integer: order-free
}

template <class T>
T* dev_alloc(size_t count) {
  void* p = nullptr;
  GWB_CUDA_K(cudaMalloc(&p, sizeof(T) * (count ? count : 1)));
  return static_cast<T*>(p);
}
}  // namespace

void launch_rowsums_cm64(const double* pi, int64_t n, int64_t m, double* out, cudaStream_t s) {
  rowsums_cm64_kernel<<<grid1d(n, 256), 256, 0, s>>>(pi, n, m, out);
  GWB_CUDA_K(cudaGetLastError());
}

void launch_colsums_cm64(const double* pi, int64_t n, int64_t m, double* out, cudaStream_t s) {
  colsums_cm64_kernel<<<static_cast<unsigned>(m), 256, 0, s>>>(pi, n, m, out);
  GWB_CUDA_K(cudaGetLastError());
}

void launch_argmax_rows_cm64(const double* pi, int64_t n, int64_t m, int32_t* out, cudaStream_t s) {
  argmax_rows_cm64_kernel<<<grid1d(n, 256), 256, 0, s>>>(pi, n, m, out);
  GWB_CUDA_K(cudaGetLastError());
}

double sum_sq_diff_dev(const double* a, const double* b, int64_t len, cudaStream_t s) {
  constexpr int kBlocks = 592;
  double* part = dev_alloc<double>(kBlocks);
  sqdiff_kernel<<<kBlocks, 256, 0, s>>>(a, b, len, part);
  GWB_CUDA_K(cudaGetLastError());
  double h[kBlocks];
  GWB_CUDA_K(cudaMemcpyAsync(h, part, sizeof(h), cudaMemcpyDeviceToHost, s));
  GWB_CUDA_K(cudaStreamSynchronize(s));
  cudaFree(part);
  double t = 0.0;
  for (double v : h) t += v;
  return t;
}

int64_t count_equal_dev(const int32_t* a, const int32_t* b, int64_t len, cudaStream_t s) {
  auto* c = dev_alloc<unsigned long long>(1);
  GWB_CUDA_K(cudaMemsetAsync(c, 0, sizeof(unsigned long long), s));
  count_equal_kernel<<<std::min<unsigned>(grid1d(len, 256), 592u), 256, 0, s>>>(a, b, len, c);
  GWB_CUDA_K(cudaGetLastError());
  unsigned long long h = 0;
  GWB_CUDA_K(cudaMemcpyAsync(&h, c, sizeof(h), cudaMemcpyDeviceToHost, s));
  GWB_CUDA_K(cudaStreamSynchronize(s));
  cudaFree(c);
  return static_cast<int64_t>(h);
}

}  // namespace gwb
