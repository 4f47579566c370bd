// quadratic.cu — BAPG with the quadratic (Euclidean) geometry, SURVEY §8(f)
// row 4 (solvers.cpp:179-182):
//   π  = euclid_project(w + M(w)/ρ, μ, Rows)
//   w' = euclid_project(π + M(π)/ρ, ν, Cols)
// euclid_project projects every row (column) onto the scaled simplex
// {x ≥ 0, Σx = s} (projections.cpp:36-77).  The reference sorts each line;
// here the threshold θ comes from Michelot's active-set iteration
//   θ ← (Σ_{v > θ} v − s) / #{v > θ},  starting from θ = (Σ v − s)/len,
// which reaches the same θ (the sorted prefix of the support) in a handful
// of passes without a sort; v and θ are fp64, sums in a fixed order.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "devutil.cuh"
#include "kernels.cuh"

namespace gwb {

void check_cuda(cudaError_t e, const char* what);

namespace {

using namespace dev;
constexpr int kThreads = 256;
constexpr int kMaxPasses = 64;  // Michelot converges in far fewer; a hard stop

__device__ __forceinline__ double warp_sum_d(double v) { return warp_sum(v); }
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sums of (double, int); every thread gets the totals.
__device__ void block_sum2(double& a, int& c) {
  __shared__ double sa[kThreads / 32];
  __shared__ int sc[kThreads / 32];
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  a = warp_sum_d(a);
  c = warp_sum_i(c);
  __syncthreads();  // previous readers done
  if (l == 0) {
    sa[w] = a;
    sc[w] = c;
  }
  __syncthreads();
  double ta = 0.0;
  int tc = 0;
  for (int q = 0; q < kThreads / 32; ++q) {
    ta += sa[q];
    tc += sc[q];
  }
  a = ta;
  c = tc;
}

// Half-step a: one CTA per row.  v = w + G/ρ (fp64), P = max(v − θ, 0).
// Also the previous record's row diagnostics (⟨G,w⟩, (Σw − μ)²) as
// row_update_kernel does, the GEMM operand copy of P, and the flags.
__global__ void __launch_bounds__(kThreads) row_quad_kernel(BapgDev d) {
  if (d.st->done) return;
  const int64_t i = blockIdx.x;
  const float* g = d.G + i * d.ld;
  const float* w = d.W + i * d.ld;
  const int64_t m = d.m;
  const double ir = static_cast<double>(d.inv_rho);
  const double s = d.mu64[i];
  double gw = 0.0, rw = 0.0, vs = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += kThreads) {
    const double gj = g[j], wj = w[j];
    gw += gj * wj;
    rw += wj;
    vs += wj + gj * ir;
  }
  // diagnostics (fixed order)
  {
    double a = gw;
    int c = 0;
    block_sum2(a, c);
    gw = a;
    a = rw;
    block_sum2(a, c);
    rw = a;
  }
  int cnt = static_cast<int>(m);
  block_sum2(vs, cnt);
  double theta = (vs - s) / static_cast<double>(m);
  int support = static_cast<int>(m);
  for (int pass = 0; pass < kMaxPasses; ++pass) {
    double S = 0.0;
    int c = 0;
    for (int64_t j = threadIdx.x; j < m; j += kThreads) {
      const double v = static_cast<double>(w[j]) + static_cast<double>(g[j]) * ir;
      if (v > theta) {
        S += v;
        ++c;
      }
    }
    block_sum2(S, c);
    if (c == 0) break;  // cannot happen for s > 0; keeps θ finite
    const double nt = (S - s) / static_cast<double>(c);
    const bool stable = c == support;
    theta = nt;
    support = c;
    if (stable) break;
  }
  if (threadIdx.x == 0) {
    d.row_part[i].gw = gw;
    const double dv = rw - s;
    d.row_part[i].rowdev = dv * dv;
    if (!isfinite(theta)) atomicOr(&d.st->flags, kFlagNonFinite);
  }
  float* p = d.P + i * d.ld;
  bool finite = true;
  for (int64_t j0 = static_cast<int64_t>(threadIdx.x) * 4; j0 < m; j0 += kThreads * 4) {
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t j = j0 + q;
      if (j < m) {
        const double v = static_cast<double>(w[j]) + static_cast<double>(g[j]) * ir;
        const double x = v - theta;
        o[q] = x > 0.0 ? static_cast<float>(x) : 0.f;
        finite = finite && isfinite(o[q]);
      } else {
        o[q] = 0.f;
      }
    }
    *reinterpret_cast<float4*>(p + j0) = make_float4(o[0], o[1], o[2], o[3]);
    if (d.P_aux) aux_store4(d.P_aux, d.aux_mode, d.plane, i * d.ld + j0, o[0], o[1], o[2], o[3], d.aux_scale);
  }
  if (!__syncthreads_and(finite ? 1 : 0) && threadIdx.x == 0) atomicOr(&d.st->flags, kFlagNonFinite);
}

// Half-step b: one CTA per 32-column block; warp w walks rows w, w+8, …;
// lane l owns column c0 + l.  v = X + G/ρ (use_g) or X (reset: w⁰ from π⁰).
// Writes `out` (W_new) and, for the record, (Σ_i P_ij − ν_j)².
constexpr int kColW = 32;
__global__ void __launch_bounds__(kThreads) col_quad_kernel(BapgDev d, const float* X, float* out,
                                                           int use_g, int reset) {
  if (!reset && d.st->done) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kColW + lane;
  const bool ok = j < d.m;
  const double ir = use_g ? static_cast<double>(d.inv_rho) : 0.0;
  const int64_t n = d.n;
  const double s = ok ? d.nu64[j] : 1.0;
  __shared__ double sd[kThreads / 32][kColW];
  __shared__ int si[kThreads / 32][kColW];
  __shared__ double sx[kColW];   // per-column scalar exchange
  __shared__ int sdone;
  auto vval = [&](int64_t i) -> double {
    const double x = X[i * d.ld + j];
    return use_g ? x + static_cast<double>(d.G[i * d.ld + j]) * ir : x;
  };
  // column sums of v (θ start) and of X (record: colsum(π) − ν)
  double vs = 0.0, xs = 0.0;
  if (ok)
    for (int64_t i = warp; i < n; i += kThreads / 32) {
      vs += vval(i);
      xs += X[i * d.ld + j];
    }
  sd[warp][lane] = vs;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
    for (int q = 0; q < kThreads / 32; ++q) t += sd[q][lane];
    sx[lane] = t;
  }
  __syncthreads();
  double theta = (sx[lane] - s) / static_cast<double>(n);
  __syncthreads();
  sd[warp][lane] = xs;
  __syncthreads();
  if (warp == 0 && ok && !reset) {
    double t = 0.0;
    for (int q = 0; q < kThreads / 32; ++q) t += sd[q][lane];
    const double dv = t - s;
    d.col_dev[j] = dv * dv;
  }
  int support = static_cast<int>(n);
  bool col_done = !ok;
  for (int pass = 0; pass < kMaxPasses; ++pass) {
    double S = 0.0;
    int c = 0;
    if (!col_done)
      for (int64_t i = warp; i < n; i += kThreads / 32) {
        const double v = vval(i);
        if (v > theta) {
          S += v;
          ++c;
        }
      }
    __syncthreads();
    sd[warp][lane] = S;
    si[warp][lane] = c;
    if (threadIdx.x == 0) sdone = 1;
    __syncthreads();
    if (warp == 0) {
      double tS = 0.0;
      int tc = 0;
      for (int q = 0; q < kThreads / 32; ++q) {
        tS += sd[q][lane];
        tc += si[q][lane];
      }
      sd[0][lane] = tS;
      si[0][lane] = tc;
    }
    __syncthreads();
    if (!col_done) {
      const double tS = sd[0][lane];
      const int tc = si[0][lane];
      if (tc > 0) {
        const bool stable = tc == support;
        theta = (tS - s) / static_cast<double>(tc);
        support = tc;
        col_done = stable;
      } else {
        col_done = true;
      }
    }
    if (!col_done) sdone = 0;  // benign race: every writer stores 0
    __syncthreads();
    if (sdone) break;
  }
  if (!ok) return;
  for (int64_t i = warp; i < n; i += kThreads / 32) {
    const double x = vval(i) - theta;
    out[i * d.ld + j] = x > 0.0 ? static_cast<float>(x) : 0.f;
  }
}

// Half-step b, second pass (one CTA per row): the record's per-row
// partials (⟨G,w'⟩, ‖π−w'‖², ‖w'−w‖², ‖w‖², ⟨G,π⟩) as col_write_kernel,
// the GEMM operand copy of w', and the non-finite flag.
__global__ void __launch_bounds__(kThreads) quad_col_diag_kernel(BapgDev d) {
  if (d.st->done) return;
  const int64_t i = blockIdx.x;
  const float* g = d.G + i * d.ld;
  const float* p = d.P + i * d.ld;
  const float* wo = d.W + i * d.ld;
  const float* wn = d.W_new + i * d.ld;
  double sums[5] = {0, 0, 0, 0, 0};
  bool finite = true;
  for (int64_t j0 = static_cast<int64_t>(threadIdx.x) * 4; j0 < d.m; j0 += kThreads * 4) {
    const float4 n4 = *reinterpret_cast<const float4*>(wn + j0);
    const float nv[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t j = j0 + q;
      if (j < d.m) {
        const double gv = g[j], pv = p[j], wv = wo[j], o = nv[q];
        finite = finite && isfinite(nv[q]);
        sums[0] += gv * o;
        sums[1] += (pv - o) * (pv - o);
        sums[2] += (o - wv) * (o - wv);
        sums[3] += wv * wv;
        sums[4] += gv * pv;
      }
    }
    if (d.W_aux) aux_store4(d.W_aux, d.aux_mode, d.plane, i * d.ld + j0, n4.x, n4.y, n4.z, n4.w, d.aux_scale);
  }
  MaxSum dummy{-INFINITY, 0.f};
  block_reduce<kThreads, 5>(dummy, sums);
  if (!__syncthreads_and(finite ? 1 : 0) && threadIdx.x == 0) atomicOr(&d.st->flags, kFlagNonFinite);
  if (threadIdx.x == 0) {
    ColWritePart& c = d.cw_part[i];
    c.gw = sums[0];
    c.split = sums[1];
    c.diff = sums[2];
    c.wold = sums[3];
    c.gp = sums[4];
  }
}

__global__ void quad_flag_kernel(DevStatus* st) {
  if (st->done) return;
  if (st->flags != 0) {
    st->done = 1;
    st->err_iter = st->iter;
  }
}

}  // namespace

void launch_row_quad(const BapgDev& d, cudaStream_t s) {
  row_quad_kernel<<<static_cast<unsigned>(d.n), kThreads, 0, s>>>(d);
  quad_flag_kernel<<<1, 1, 0, s>>>(d.st);
  check_cuda(cudaGetLastError(), "row_quad_kernel");
}

void launch_col_quad(const BapgDev& d, cudaStream_t s) {
  col_quad_kernel<<<static_cast<unsigned>((d.m + kColW - 1) / kColW), kThreads, 0, s>>>(
      d, d.P, d.W_new, 1, 0);
  quad_col_diag_kernel<<<static_cast<unsigned>(d.n), kThreads, 0, s>>>(d);
  quad_flag_kernel<<<1, 1, 0, s>>>(d.st);
  check_cuda(cudaGetLastError(), "col_quad_kernel");
}

void launch_quad_reset(const BapgDev& d, const float* pi0, float* w0, cudaStream_t s) {
  col_quad_kernel<<<static_cast<unsigned>((d.m + kColW - 1) / kColW), kThreads, 0, s>>>(
      d, pi0, w0, 0, 1);
  check_cuda(cudaGetLastError(), "col_quad_kernel(reset)");
}

}  // namespace gwb
