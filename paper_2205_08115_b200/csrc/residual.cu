// residual.cu — the Luo-Tseng residual (diagnostics.cpp:33-42) and the
// Dykstra projection onto Π(μ, ν) it uses (projections.cpp:165-187), SURVEY
// §8(f) row 4.  fp64 throughout: the Dykstra stop test is an absolute 1e-8
// on marginal sums, below fp32 resolution for masses near 1.
//
// Layout: column-major fp64 (ld = n), the boundary's own layout, so the
// input coupling and the residual's ‖π − Proj(π + Mπ)‖ need no transpose.
// One Dykstra sweep is three launches:
//   rows : y = P_rows(x + p), p ← x + p − y   (cluster per 8 rows)
//          + max_i |Σ_j x_ij − μ_i| of the previous sweep's x
//   check: stop once marginal_error_inf(x) ≤ tol   (one thread)
//   cols : x = P_cols(y + q), q ← y + q − x   (cluster per column)
//          + max_j |Σ_i x_ij − ν_j|
// Algorithmic traffic: 64 B per element and sweep (each pass reads two fp64
// matrices and writes two).
// The row error of x_s is only known after the row pass of sweep s+1
// (which writes y and p, never x), so the check runs one pass late and x_s
// is returned intact.  Line maxima combine through atomicMax on the IEEE
// bits of non-negative doubles (order-independent, so deterministic; NaN
// dominates).  Per-line thresholds: warm-started Newton/Michelot steps on
// lines staged in shared memory across a thread-block cluster (below).
// Sweeps run in captured chunks; every kernel returns once `done`.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/gwb_ext.h"
#include "devutil.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "solver.cuh"
#include "standalone.cuh"

namespace gwb {

namespace {

using namespace dev;

constexpr int kThreads = 256;
constexpr int kMaxPasses = 64;
constexpr int kChunk = 32;                        // sweeps per captured graph
constexpr size_t kStageBytes = 80 * 1024;  // dynamic smem per CTA (a 20000-long row block stages over 16 CTAs)

struct DykState {
  int done;
  int started;   // a column pass has run: the row pass may score x
  int checked;   // sweeps whose x has been scored
  int sweeps;    // sweeps used when done
  double err;    // last scored marginal_error_inf
  unsigned long long row_bits, col_bits;
};

__device__ __forceinline__ void max_bits(unsigned long long* slot, double v) {
  atomicMax(slot, static_cast<unsigned long long>(__double_as_longlong(fabs(v))));
}

// Per-line Euclidean projection onto {x ≥ 0, Σx = s}: θ by Newton steps on
// f(θ) = Σ max(v − θ, 0) − s, i.e. θ ← (Σ_{v>θ} v − s) / #{v > θ}.  f is
// convex and decreasing, so from any start one step lands at or left of θ*
// and the steps then rise monotonically; equal supports on consecutive steps
// mean a fixed point.  From the cold start (Σv − s)/len this is Michelot's
// iteration; Dykstra warm-starts each line from its θ of the previous sweep
// (per-line state), which usually leaves one verification pass.  The result
// is the same (S − s)/c over the same support, summed in the same order.
//
// One kernel serves both passes.  A cluster of C CTAs owns R lines; CTA k
// of the cluster holds elements [k·chunk, (k+1)·chunk) of each, staged in
// shared memory (v = a + corr) so the Newton passes never return to HBM,
// and per-line totals combine across the cluster through distributed
// shared memory in rank order (deterministic).  Element e of line t lives
// at t·line_stride + e·elem_stride: rows of the column-major matrix are
// (line_stride 1, elem_stride n) with R = 8 lines per CTA, so a warp load
// covers 4 columns × 8 consecutive rows; columns are (n, 1) with R = 1.
// Lane l works on line l % R and element offset l / R.
namespace cg = cooperative_groups;

template <int R, bool kErrOfOut>
__global__ void __launch_bounds__(kThreads)
    dyk_lines_kernel(const double* __restrict__ a, double* __restrict__ corr,
                     double* __restrict__ out, int64_t nlines, int64_t len, int64_t line_stride,
                     int64_t elem_stride, int64_t chunk, const double* __restrict__ target,
                     double* __restrict__ theta_line, int staged, int mode,
                     unsigned long long* err_slot, int set_started, DykState* st) {
  if (st->done) return;  // uniform: written by the previous launch
  cg::cluster_group cluster = cg::this_cluster();
  const int C = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  constexpr int kW = kThreads / 32;
  constexpr int kPer = 32 / R;          // elements per warp step
  constexpr int kStep = kW * kPer;      // elements per CTA step
  extern __shared__ double sv[];        // [chunk][R] when staged
  __shared__ double wpart[kW][R][4];
  __shared__ double cpart[2][R][4];
  __shared__ double ctot[R][4];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int t = lane % R, eo = lane / R;
  const int64_t line = (static_cast<int64_t>(blockIdx.x) / C) * R + t;
  const bool ok = line < nlines;
  const int64_t e_begin = static_cast<int64_t>(rank) * chunk;
  const int64_t e_end = ok ? (e_begin + chunk < len ? e_begin + chunk : len) : e_begin;
  const int64_t e0 = e_begin + w * kPer + eo;
  const double s = ok ? target[line] : 1.0;
  const double* al = a + line * line_stride;
  double* cl = corr + line * line_stride;
  double* ol = out + line * line_stride;
  int slot = 0;
  // Per-line totals of v[0..3]: lanes sharing the line (xor over the
  // element bits), warps in order, then cluster ranks in order.
  auto totals = [&](double (&v)[4]) {
#pragma unroll
    for (int o = R; o < 32; o <<= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    __syncthreads();
    if (eo == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) wpart[w][t][q] = v[q];
    __syncthreads();
    if (threadIdx.x < R) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < kW; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += wpart[k][threadIdx.x][q];
#pragma unroll
      for (int q = 0; q < 4; ++q) cpart[slot][threadIdx.x][q] = acc[q];
    }
    cluster.sync();
    if (threadIdx.x < R) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int k = 0; k < C; ++k) {
        const double* rp = cluster.map_shared_rank(&cpart[slot][threadIdx.x][0], k);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += rp[q];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) ctot[threadIdx.x][q] = acc[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = ctot[t][q];
    slot ^= 1;
  };
  const bool score = kErrOfOut || mode == 1 || st->started;
  const double warm = ok && mode == 0 ? theta_line[line] : NAN;
  const bool has_warm = !isnan(warm);
  double sa = 0.0, vs = 0.0, S = 0.0, c = 0.0;
  constexpr int kU = 4;  // loads in flight per thread and array
  for (int64_t e = e0; e < e_end; e += kU * kStep) {
    double av[kU], cv[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int64_t ee = e + k * kStep;
      av[k] = ee < e_end ? al[ee * elem_stride] : 0.0;
      cv[k] = (mode == 0 && ee < e_end) ? cl[ee * elem_stride] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int64_t ee = e + k * kStep;
      if (ee >= e_end) break;
      sa += av[k];
      if (mode == 0) {
        const double v = av[k] + cv[k];
        if (staged) sv[(ee - e_begin) * R + t] = v;
        vs += v;
        if (has_warm && v > warm) {
          S += v;
          c += 1.0;
        }
      }
    }
  }
  double tv[4] = {sa, vs, S, c};
  totals(tv);
  const double tot_a = tv[0], tot_v = tv[1], tot_S = tv[2], tot_c = tv[3];
  if (!kErrOfOut && score && ok && rank == 0 && w == 0 && eo == 0) max_bits(err_slot, tot_a - s);
  if (mode == 1) {
    cluster.sync();  // peers may still read this CTA's partials
    return;
  }
  double theta;
  double support;
  if (tot_c > 0.0) {  // one Newton step from the warm start
    theta = (tot_S - s) / tot_c;
    support = tot_c;
  } else {
    theta = (tot_v - s) / static_cast<double>(len);
    support = static_cast<double>(len);
  }
  auto vget = [&](int64_t e) {
    return staged ? sv[(e - e_begin) * R + t] : al[e * elem_stride] + cl[e * elem_stride];
  };
  bool line_done = !ok;
  for (int pass = 0; pass < kMaxPasses; ++pass) {
    double ps = 0.0, pc = 0.0;
    if (!line_done)
      for (int64_t e = e0; e < e_end; e += kStep) {
        const double v = vget(e);
        if (v > theta) {
          ps += v;
          pc += 1.0;
        }
      }
    double pv[4] = {ps, pc, 0.0, 0.0};
    totals(pv);
    const double tS = pv[0], tc = pv[1];
    if (!line_done) {
      if (tc > 0.0) {
        line_done = tc == support;
        theta = (tS - s) / tc;
        support = tc;
      } else {
        line_done = true;
      }
    }
    // Same totals in every CTA of the cluster ⇒ the same decision.
    if (!__syncthreads_or(line_done ? 0 : 1)) break;
  }
  double so = 0.0;
  for (int64_t e = e0; e < e_end; e += kStep) {
    const double v = vget(e);
    const double o = v - theta > 0.0 ? v - theta : 0.0;
    ol[e * elem_stride] = o;
    cl[e * elem_stride] = v - o;
    so += o;
  }
  if (kErrOfOut) {
    double ov[4] = {so, 0.0, 0.0, 0.0};
    totals(ov);
    if (ok && rank == 0 && w == 0 && eo == 0) max_bits(err_slot, ov[0] - s);
  }
  if (ok && rank == 0 && w == 0 && eo == 0) theta_line[line] = theta;
  if (set_started && blockIdx.x == 0 && threadIdx.x == 0) st->started = 1;
  cluster.sync();  // peers may still read this CTA's partials
}

__global__ void dyk_check_kernel(DykState* st, double tol) {
  if (st->done || !st->started) return;
  const double rb = __longlong_as_double(static_cast<long long>(st->row_bits));
  const double cb = __longlong_as_double(static_cast<long long>(st->col_bits));
  const double e = (isnan(rb) || isnan(cb)) ? NAN : fmax(rb, cb);
  st->checked += 1;
  st->err = e;
  st->row_bits = 0;
  st->col_bits = 0;
  if (e <= tol) {
    st->done = 1;
    st->sweeps = st->checked;
  }
}

// x (column-major fp64) = π (column-major fp64) + G (row-major fp32, ld),
// through 32×32 shared-memory tiles so both sides are coalesced.
__global__ void shift_kernel(const double* __restrict__ pi, const float* __restrict__ G,
                             int64_t ld, int64_t n, int64_t m, double* __restrict__ x) {
  __shared__ float t[32][33];
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * 32, j0 = static_cast<int64_t>(blockIdx.x) * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    t[r][threadIdx.x] = (i < n && j < m) ? G[i * ld + j] : 0.f;
  }
  __syncthreads();
  for (int c = threadIdx.y; c < 32; c += blockDim.y) {
    const int64_t j = j0 + c, i = i0 + threadIdx.x;
    if (i < n && j < m) x[j * n + i] = pi[j * n + i] + static_cast<double>(t[threadIdx.x][c]);
  }
}

double g_last_ms = 0.0;  // gwb_dykstra_last_stats
int g_last_sweeps = 0;

}  // namespace

DykstraOutcome dykstra_dev(double* x, int64_t n, int64_t m, const double* mu64,
                           const double* nu64, double tol, int max_iters, cudaStream_t s) {
  const size_t len = static_cast<size_t>(n) * m;
  double *y = nullptr, *p = nullptr, *q = nullptr;
  DykState* st = nullptr;
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&y), len * sizeof(double), s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), len * sizeof(double), s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&q), len * sizeof(double), s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&st), sizeof(DykState), s));
  GWB_CUDA(cudaMemsetAsync(p, 0, len * sizeof(double), s));
  GWB_CUDA(cudaMemsetAsync(q, 0, len * sizeof(double), s));
  GWB_CUDA(cudaMemsetAsync(st, 0, sizeof(DykState), s));
  double* theta = nullptr;  // per-line warm starts: rows [0, n), columns [n, n+m)
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&theta), (n + m) * sizeof(double), s));
  GWB_CUDA(cudaMemsetAsync(theta, 0xff, (n + m) * sizeof(double), s));  // NaN: cold start
  int dev = 0;
  GWB_CUDA(cudaGetDevice(&dev));
  // Cluster size per pass: the smallest power of two that stages a line
  // block (R lines × chunk) in kStageBytes; beyond 16 CTAs, unstaged.
  auto plan = [](int R, int64_t len, int& C, int64_t& chunk, int& staged) {
    C = 1;
    while (C < 16 && static_cast<size_t>(R) * ((len + C - 1) / C) * sizeof(double) > kStageBytes) C *= 2;
    chunk = (len + C - 1) / C;
    staged = static_cast<size_t>(R) * chunk * sizeof(double) <= kStageBytes;
  };
  // Measured at n = m = 8192 (B200): R = 8 rows per CTA with 64–96 KB stages
  // beats R = 16 / 32 (1.18 vs 1.37 / 1.73 ms per sweep) and 24–40 KB or
  // 160 KB stages.
  constexpr int kRowR = 8;
  int row_C, col_C, row_staged, col_staged;
  int64_t row_chunk, col_chunk;
  plan(kRowR, m, row_C, row_chunk, row_staged);
  plan(1, n, col_C, col_chunk, col_staged);
  static thread_local int attr_device = -1;
  if (attr_device != dev) {  // per device context (as gemm.cu)
    const int b = static_cast<int>(kStageBytes);
    for (const void* f : {reinterpret_cast<const void*>(dyk_lines_kernel<kRowR, false>),
                          reinterpret_cast<const void*>(dyk_lines_kernel<1, true>)}) {
      GWB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, b));
      GWB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    attr_device = dev;
  }
  auto launch = [&](auto kern, int R, int C, int64_t chunk, int staged, int64_t nlines,
                    int64_t len, int64_t line_stride, int64_t elem_stride, const double* a,
                    double* corr, double* out, const double* target, double* th, int mode,
                    unsigned long long* slot, int set_started) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(((nlines + R - 1) / R) * C));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = staged ? static_cast<size_t>(R) * chunk * sizeof(double) : 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(C);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GWB_CUDA(cudaLaunchKernelEx(&cfg, kern, a, corr, out, nlines, len, line_stride, elem_stride,
                                chunk, target, th, staged, mode, slot, set_started, st));
  };
  auto sweep = [&](int mode) {
    // rows: y = P_rows(x + p), p ← x + p − y; scores Σ_j x_ij − μ_i
    launch(dyk_lines_kernel<kRowR, false>, kRowR, row_C, row_chunk, row_staged, n, m,
           int64_t{1}, n, x, p, y, mu64, theta, mode, &st->row_bits, 0);
    dyk_check_kernel<<<1, 1, 0, s>>>(st, tol);
    // columns: x = P_cols(y + q), q ← y + q − x; scores Σ_i x_ij − ν_j
    if (mode == 0)
      launch(dyk_lines_kernel<1, true>, 1, col_C, col_chunk, col_staged, m, n, n, int64_t{1}, y,
             q, x, nu64, theta + n, 0, &st->col_bits, 1);
  };
  int* h_done = nullptr;
  GWB_CUDA(cudaMallocHost(&h_done, sizeof(int)));
  cudaEvent_t e0, e1;
  GWB_CUDA(cudaEventCreate(&e0));
  GWB_CUDA(cudaEventCreate(&e1));
  GWB_CUDA(cudaEventRecord(e0, s));
  cudaGraphExec_t ge = nullptr;
  int ran = 0;
  bool stop = false;
  while (ran < max_iters && !stop) {
    const int k = std::min(kChunk, max_iters - ran);
    if (k == kChunk) {
      if (!ge) {
        cudaGraph_t g;
        GWB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        for (int t = 0; t < kChunk; ++t) sweep(0);
        GWB_CUDA(cudaStreamEndCapture(s, &g));
        GWB_CUDA(cudaGraphInstantiate(&ge, g, 0));
        GWB_CUDA(cudaGraphDestroy(g));
      }
      GWB_CUDA(cudaGraphLaunch(ge, s));
    } else {
      for (int t = 0; t < k; ++t) sweep(0);
    }
    GWB_CUDA(cudaGetLastError());
    ran += k;
    GWB_CUDA(cudaMemcpyAsync(h_done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, s));
    GWB_CUDA(cudaStreamSynchronize(s));
    stop = *h_done != 0;
  }
  if (!stop) sweep(1);  // score the last sweep's x
  GWB_CUDA(cudaGetLastError());
  GWB_CUDA(cudaEventRecord(e1, s));
  DykState h;
  GWB_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
  GWB_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  GWB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ge) cudaGraphExecDestroy(ge);
  cudaFreeHost(h_done);
  for (void* b : {static_cast<void*>(y), static_cast<void*>(p), static_cast<void*>(q),
                  static_cast<void*>(st), static_cast<void*>(theta)})
    cudaFreeAsync(b, s);
  DykstraOutcome out;
  out.converged = h.done != 0;
  out.sweeps = h.done ? h.sweeps : h.checked;
  out.err = h.err;
  g_last_ms = ms;
  g_last_sweeps = out.sweeps;
  return out;
}

[[noreturn]] void dykstra_fail(int max_iters, double err) {
  char buf[160];
  // std::ostream's default double format (6 significant digits) = %g.
  std::snprintf(buf, sizeof(buf),
                "dykstra_project did not converge in %d sweeps; final constraint violation %g",
                max_iters, err);
  api_fail(GWB_ERR_RUNTIME, buf);
}

double luo_tseng_residual_dev(const float* Dx, int64_t ldn, const float* Dy, int64_t ldm,
                              const double* pi, int64_t n, int64_t m, const double* mu64,
                              const double* nu64, double tol, cudaStream_t s) {
  const size_t len = static_cast<size_t>(n) * m;
  float *P = nullptr, *G = nullptr;
  double* x = nullptr;
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&P), static_cast<size_t>(n) * ldm * sizeof(float), s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&G), static_cast<size_t>(n) * ldm * sizeof(float), s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&x), len * sizeof(double), s));
  GWB_CUDA(cudaMemsetAsync(P, 0, static_cast<size_t>(n) * ldm * sizeof(float), s));
  // shifted = π + D_X π D_Y (diagnostics.cpp:39), chain on the fp32 copy.
  launch_colmajor64_to_rowmajor32(pi, n, m, P, ldm, s);
  structure_product_dev(Dx, ldn, Dy, ldm, P, n, m, G, s);
  dim3 grid(static_cast<unsigned>((m + 31) / 32), static_cast<unsigned>((n + 31) / 32));
  shift_kernel<<<grid, dim3(32, 8), 0, s>>>(pi, G, ldm, n, m, x);
  GWB_CUDA(cudaGetLastError());
  cudaFreeAsync(P, s);
  cudaFreeAsync(G, s);
  const DykstraOutcome o = dykstra_dev(x, n, m, mu64, nu64, tol, 10000, s);
  if (!o.converged) {
    cudaFreeAsync(x, s);
    dykstra_fail(10000, o.err);
  }
  const double r = std::sqrt(sum_sq_diff_dev(pi, x, static_cast<int64_t>(len), s));
  cudaFreeAsync(x, s);
  return r;
}

// Host-buffer leaves (gwb_dykstra_project / gwb_luo_tseng_residual), each
// on its own stream (the sweep chunks are graph-captured, which the legacy
// stream does not allow).
namespace {
struct OwnStream {
  cudaStream_t s = nullptr;
  OwnStream() { GWB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~OwnStream() {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
  }
};
}  // namespace

void device_dykstra_project(const double* pi, int64_t n, int64_t m, const double* mu,
                            const double* nu, double tol, int32_t max_iters, double* out) {
  GWB_CUDA(cudaSetDevice(api_device()));
  OwnStream own;
  cudaStream_t s = own.s;
  const size_t len = static_cast<size_t>(n) * m;
  double *x = nullptr, *dmu = nullptr, *dnu = nullptr;
  GWB_CUDA(cudaMalloc(&x, len * sizeof(double)));
  GWB_CUDA(cudaMalloc(&dmu, n * sizeof(double)));
  GWB_CUDA(cudaMalloc(&dnu, m * sizeof(double)));
  GWB_CUDA(cudaMemcpyAsync(x, pi, len * sizeof(double), cudaMemcpyHostToDevice, s));
  GWB_CUDA(cudaMemcpyAsync(dmu, mu, n * sizeof(double), cudaMemcpyHostToDevice, s));
  GWB_CUDA(cudaMemcpyAsync(dnu, nu, m * sizeof(double), cudaMemcpyHostToDevice, s));
  DykstraOutcome o;
  try {
    o = dykstra_dev(x, n, m, dmu, dnu, tol, max_iters, s);
  } catch (...) {
    cudaFree(x);
    cudaFree(dmu);
    cudaFree(dnu);
    throw;
  }
  if (o.converged) {
    GWB_CUDA(cudaMemcpyAsync(out, x, len * sizeof(double), cudaMemcpyDeviceToHost, s));
    GWB_CUDA(cudaStreamSynchronize(s));
  }
  cudaFree(x);
  cudaFree(dmu);
  cudaFree(dnu);
  if (!o.converged) dykstra_fail(max_iters, o.err);
}

double device_luo_tseng_residual(const double* dx, int64_t n, const double* dy, int64_t m,
                                 const double* pi, const double* mu, const double* nu,
                                 double tol) {
  GWB_CUDA(cudaSetDevice(api_device()));
  OwnStream own;
  cudaStream_t s = own.s;
  const int64_t ldn = round_up(n, 32), ldm = round_up(m, 32);
  const size_t len = static_cast<size_t>(n) * m;
  const size_t big = static_cast<size_t>(std::max(n * n, m * m));
  double *stage = nullptr, *dpi = nullptr, *dmu = nullptr, *dnu = nullptr;
  float *Dx = nullptr, *Dy = nullptr;
  GWB_CUDA(cudaMalloc(&stage, big * sizeof(double)));
  GWB_CUDA(cudaMalloc(&dpi, len * sizeof(double)));
  GWB_CUDA(cudaMalloc(&dmu, n * sizeof(double)));
  GWB_CUDA(cudaMalloc(&dnu, m * sizeof(double)));
  GWB_CUDA(cudaMalloc(&Dx, static_cast<size_t>(n) * ldn * sizeof(float)));
  GWB_CUDA(cudaMalloc(&Dy, static_cast<size_t>(m) * ldm * sizeof(float)));
  GWB_CUDA(cudaMemsetAsync(Dx, 0, static_cast<size_t>(n) * ldn * sizeof(float), s));
  GWB_CUDA(cudaMemsetAsync(Dy, 0, static_cast<size_t>(m) * ldm * sizeof(float), s));
  auto release = [&] {
    for (void* b : {static_cast<void*>(stage), static_cast<void*>(dpi), static_cast<void*>(dmu),
                    static_cast<void*>(dnu), static_cast<void*>(Dx), static_cast<void*>(Dy)})
      cudaFree(b);
  };
  double r = 0.0;
  try {
    GWB_CUDA(cudaMemcpyAsync(stage, dx, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
    launch_colmajor64_to_rowmajor32(stage, n, n, Dx, ldn, s);
    GWB_CUDA(cudaStreamSynchronize(s));  // stage is reused
    GWB_CUDA(cudaMemcpyAsync(stage, dy, sizeof(double) * m * m, cudaMemcpyHostToDevice, s));
    launch_colmajor64_to_rowmajor32(stage, m, m, Dy, ldm, s);
    GWB_CUDA(cudaMemcpyAsync(dpi, pi, len * sizeof(double), cudaMemcpyHostToDevice, s));
    GWB_CUDA(cudaMemcpyAsync(dmu, mu, n * sizeof(double), cudaMemcpyHostToDevice, s));
    GWB_CUDA(cudaMemcpyAsync(dnu, nu, m * sizeof(double), cudaMemcpyHostToDevice, s));
    r = luo_tseng_residual_dev(Dx, ldn, Dy, ldm, dpi, n, m, dmu, dnu, tol, s);
  } catch (...) {
    cudaStreamSynchronize(s);
    release();
    throw;
  }
  release();
  return r;
}

}  // namespace gwb

extern "C" int32_t gwb_dykstra_last_stats(int32_t* sweeps, double* ms) {
  if (sweeps) *sweeps = gwb::g_last_sweeps;
  if (ms) *ms = gwb::g_last_ms;
  return GWB_OK;
}
