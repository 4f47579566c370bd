// standalone.cu — fp64 device kernels for the single-shot entry points on
// the path.  These are not iteration-hot (each runs once per call) but they
// are part of the drop-in surface, so they run on the GPU like everything
// else; fp64 keeps them bit-close to the reference's Eigen arithmetic.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "devutil.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "solver.cuh"
#include "standalone.cuh"

namespace gwb {

namespace {

// The leaf entry points (device_*) each run on their own non-blocking
// stream: a LeafStream scope creates it and points t_leaf at it, so every
// buffer fill, copy and kernel of the call is ordered on that stream and
// nothing touches the legacy default stream (which would serialise with
// other work on the device).  Outside a scope (the engine-stream helpers
// structure_product_dev / gw_objective_dev / coupling_entropy_dev) t_leaf is
// null and buffers are filled synchronously.
thread_local cudaStream_t t_leaf = nullptr;

struct LeafStream {
  cudaStream_t prev;
  cudaStream_t s = nullptr;
  LeafStream() : prev(t_leaf) {
    GWB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    t_leaf = s;
  }
  ~LeafStream() {
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    t_leaf = prev;
  }
  LeafStream(const LeafStream&) = delete;
  LeafStream& operator=(const LeafStream&) = delete;
};

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  explicit DBuf(size_t count) : n(count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T) + 256;
    GWB_CUDA(cudaMalloc(&p, bytes));
    if (t_leaf) {
      GWB_CUDA(cudaMemsetAsync(p, 0, bytes, t_leaf));
    } else {
      // Not inside a leaf scope: fill synchronously, so the buffer is ready
      // for the caller's (non-blocking) stream.
      GWB_CUDA(cudaMemset(p, 0, bytes));
      GWB_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
    }
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void up(const T* h) {
    if (t_leaf)
      GWB_CUDA(cudaMemcpyAsync(p, h, n * sizeof(T), cudaMemcpyHostToDevice, t_leaf));
    else
      GWB_CUDA(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
  }
  void down(T* h) const {
    if (t_leaf) {
      GWB_CUDA(cudaMemcpyAsync(h, p, n * sizeof(T), cudaMemcpyDeviceToHost, t_leaf));
      GWB_CUDA(cudaStreamSynchronize(t_leaf));
    } else {
      GWB_CUDA(cudaMemcpy(h, p, n * sizeof(T), cudaMemcpyDeviceToHost));
    }
  }
};

unsigned blocks(int64_t work, int threads) {
  return static_cast<unsigned>(std::max<int64_t>(1, (work + threads - 1) / threads));
}

// ---- column-major fp64 kernels ---------------------------------------------
__global__ void outer_kernel(const double* mu, int64_t n, const double* nu, int64_t m,
                             double* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n * m) return;
  const int64_t i = k % n, j = k / n;
  out[k] = mu[i] * nu[j];
}

// Row sums of a column-major matrix (thread per row; coalesced over rows).
__global__ void rowsum_kernel(const double* a, int64_t n, int64_t m, double* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t j = 0; j < m; ++j) s += a[j * n + i];
  out[i] = s;
}

// Column sums (block per column, contiguous).
__global__ void colsum_kernel(const double* a, int64_t n, int64_t m, double* out) {
  const int64_t j = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += a[j * n + i];
  __shared__ double sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[j] = sh[0];
}

// Scale lines by target/sum; records the lowest bad line (kl_scale check,
// projections.cpp:19-21, 28-30).
__global__ void scale_lines_kernel(double* a, int64_t n, int64_t m, const double* target,
                                   const double* sums, int axis, int* bad) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n * m) return;
  const int64_t i = k % n, j = k / n;
  const int64_t line = axis == GWB_ROWS ? i : j;
  const double s = sums[line];
  if (!(s > 0.0) || !isfinite(s)) {
    atomicMin(bad, static_cast<int>(line));
    return;
  }
  a[k] *= target[line] / s;
}

__global__ void sq_diff_kernel(const double* a, const double* b, int64_t len, double* part) {
  double s = 0.0;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double d = a[k] - (b ? b[k] : 0.0);
    s += d * d;
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void all_finite_kernel(const double* a, int64_t len, int* bad) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (!isfinite(a[k])) atomicOr(bad, 1);
}

__global__ void argmax_kernel(const double* a, int64_t n, int64_t m, int32_t* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t best = 0;
  double bv = a[i];
  for (int64_t j = 1; j < m; ++j) {
    const double v = a[j * n + i];
    if (v > bv) {  // strict: ties keep the lowest column (tasks.cpp:195)
      bv = v;
      best = j;
    }
  }
  out[i] = static_cast<int32_t>(best);
}

// y = D x for symmetric column-major D (warp per output; contiguous column).
__global__ void symv64_kernel(const double* d, int64_t n, const double* x, double* y) {
  const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t j = lane; j < n; j += 32) s += d[i * n + j] * x[j];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[i] = s;
}

__global__ void div_kernel(double* y, int64_t n, double s) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] /= s;
}

// Log-domain Sinkhorn line updates (projections.cpp:143-148).
__global__ void lse_rows_kernel(const double* e, int64_t n, int64_t m, const double* g,
                                const double* mu, double* f) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double c = -INFINITY;
  for (int64_t j = 0; j < m; ++j) {
    const double v = e[j * n + i] + g[j];
    if (v > c || isnan(v)) c = v;
  }
  double lse = c;
  if (isfinite(c)) {
    double s = 0.0;
    for (int64_t j = 0; j < m; ++j) s += exp(e[j * n + i] + g[j] - c);
    lse = c + log(s);
  }
  f[i] = log(mu[i]) - lse;
}

__global__ void lse_cols_kernel(const double* e, int64_t n, int64_t m, const double* f,
                                const double* nu, double* g) {
  const int64_t j = blockIdx.x;
  __shared__ double sh[256];
  double c = -INFINITY;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = e[j * n + i] + f[i];
    if (v > c || isnan(v)) c = v;
  }
  sh[threadIdx.x] = c;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double a = sh[threadIdx.x], b = sh[threadIdx.x + o];
      sh[threadIdx.x] = (b > a || isnan(b)) ? b : a;
    }
    __syncthreads();
  }
  c = sh[0];
  __syncthreads();
  double s = 0.0;
  if (isfinite(c))
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += exp(e[j * n + i] + f[i] - c);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) g[j] = log(nu[j]) - (isfinite(c) ? c + log(sh[0]) : c);
}

__global__ void exp_fg_kernel(const double* e, int64_t n, int64_t m, const double* f,
                              const double* g, double* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n * m) return;
  out[k] = exp(e[k] + f[k % n] + g[k / n]);
}

// ⟨G, P⟩ per row in fp64 (row-major fp32 operands).
__global__ void dot_rows_kernel(const float* g, const float* p, int64_t n, int64_t m, int64_t ld,
                                double* part) {
  const int64_t i = blockIdx.x;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x)
    s += static_cast<double>(g[i * ld + j]) * p[i * ld + j];
  __shared__ double sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[i] = sh[0];
}

double reduce_host(const DBuf<double>& part) {
  std::vector<double> h(part.n);
  part.down(h.data());
  double s = 0.0;
  for (double v : h) s += v;
  return s;
}

double sum_sq_diff(const double* a, const double* b, int64_t len) {
  DBuf<double> part(592);
  sq_diff_kernel<<<592, 256, 0, t_leaf>>>(a, b, len, part.p);
  GWB_CUDA(cudaGetLastError());
  return reduce_host(part);
}

double marginal_err_inf(const DBuf<double>& c, int64_t n, int64_t m, const double* mu,
                        const double* nu, DBuf<double>& rs, DBuf<double>& cs) {
  rowsum_kernel<<<blocks(n, 256), 256, 0, t_leaf>>>(c.p, n, m, rs.p);
  colsum_kernel<<<static_cast<unsigned>(m), 256, 0, t_leaf>>>(c.p, n, m, cs.p);
  std::vector<double> hr(n), hc(m);
  rs.down(hr.data());
  cs.down(hc.data());
  double row = 0.0, col = 0.0;
  for (int64_t i = 0; i < n; ++i) row = std::max(row, std::fabs(hr[i] - mu[i]));
  for (int64_t j = 0; j < m; ++j) col = std::max(col, std::fabs(hc[j] - nu[j]));
  return std::max(row, col);
}

// kl_scale on device data; throws ZeroSumLineError for the lowest bad line.
void kl_scale_dev(DBuf<double>& a, int64_t n, int64_t m, const DBuf<double>& target, int axis,
                  DBuf<double>& sums) {
  if (axis == GWB_ROWS) rowsum_kernel<<<blocks(n, 256), 256, 0, t_leaf>>>(a.p, n, m, sums.p);
  else colsum_kernel<<<static_cast<unsigned>(m), 256, 0, t_leaf>>>(a.p, n, m, sums.p);
  DBuf<int> bad(1);
  const int init = 0x7fffffff;
  bad.up(&init);
  scale_lines_kernel<<<blocks(n * m, 256), 256, 0, t_leaf>>>(a.p, n, m, target.p, sums.p, axis, bad.p);
  int hb;
  bad.down(&hb);
  if (hb != 0x7fffffff) api_zero_sum(axis, hb);
}

}  // namespace

void device_product_coupling(const double* mu, int64_t n, const double* nu, int64_t m,
                             double* out) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  DBuf<double> dmu(n), dnu(m), o(static_cast<size_t>(n) * m);
  dmu.up(mu);
  dnu.up(nu);
  outer_kernel<<<blocks(n * m, 256), 256, 0, t_leaf>>>(dmu.p, n, dnu.p, m, o.p);
  GWB_CUDA(cudaGetLastError());
  o.down(out);
}

void device_kl_scale(const double* pi, int64_t n, int64_t m, const double* target, int32_t axis,
                     double* out) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  DBuf<double> a(static_cast<size_t>(n) * m), t(axis == GWB_ROWS ? n : m),
      sums(axis == GWB_ROWS ? n : m);
  a.up(pi);
  t.up(target);
  kl_scale_dev(a, n, m, t, axis, sums);
  a.down(out);
}

double device_marginal_infeasibility(const double* pi, int64_t n, int64_t m, const double* mu,
                                     const double* nu) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  DBuf<double> a(static_cast<size_t>(n) * m), rs(n), cs(m);
  a.up(pi);
  rowsum_kernel<<<blocks(n, 256), 256, 0, t_leaf>>>(a.p, n, m, rs.p);
  colsum_kernel<<<static_cast<unsigned>(m), 256, 0, t_leaf>>>(a.p, n, m, cs.p);
  std::vector<double> hr(n), hc(m);
  rs.down(hr.data());
  cs.down(hc.data());
  double col = 0.0, row = 0.0;  // diagnostics.cpp:14-19
  for (int64_t j = 0; j < m; ++j) col += (hc[j] - nu[j]) * (hc[j] - nu[j]);
  for (int64_t i = 0; i < n; ++i) row += (hr[i] - mu[i]) * (hr[i] - mu[i]);
  return std::sqrt(col) / static_cast<double>(m) + std::sqrt(row) / static_cast<double>(n);
}

double device_split_gap(const double* pi, const double* w, int64_t n, int64_t m) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  DBuf<double> a(static_cast<size_t>(n) * m), b(static_cast<size_t>(n) * m);
  a.up(pi);
  b.up(w);
  return std::sqrt(sum_sq_diff(a.p, b.p, n * m));
}

void device_hard_assignment(const double* pi, int64_t n, int64_t m, int32_t* out) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  DBuf<double> a(static_cast<size_t>(n) * m);
  DBuf<int32_t> o(n);
  a.up(pi);
  argmax_kernel<<<blocks(n, 128), 128, 0, t_leaf>>>(a.p, n, m, o.p);
  GWB_CUDA(cudaGetLastError());
  o.down(out);
}

// spectral_norm (solvers.cpp:113-129): power iteration on D² in fp64.
static double spectral_norm_on_device(const double* d, int64_t n) {
  DBuf<double> x(n), t(n), y(n);
  if (sum_sq_diff(d, nullptr, n * n) == 0.0) return 0.0;
  std::vector<double> hx(n, 1.0 / std::sqrt(static_cast<double>(n)));
  x.up(hx.data());
  double lambda = 0.0;
  for (int it = 0; it < 10000; ++it) {
    symv64_kernel<<<blocks(n * 32, 256), 256, 0, t_leaf>>>(d, n, x.p, t.p);
    symv64_kernel<<<blocks(n * 32, 256), 256, 0, t_leaf>>>(d, n, t.p, y.p);
    const double est = std::sqrt(sum_sq_diff(y.p, nullptr, n));
    if (est == 0.0) return 0.0;
    div_kernel<<<blocks(n, 256), 256, 0, t_leaf>>>(y.p, n, est);
    std::swap(x.p, y.p);
    const double conv = std::fabs(est - lambda);
    lambda = est;
    if (conv <= 1e-10 * std::max(1.0, est)) break;
  }
  return std::sqrt(lambda);
}

static double spectral_norm_dev(const double* d_host, int64_t n) {
  DBuf<double> d(static_cast<size_t>(n) * n);
  d.up(d_host);
  return spectral_norm_on_device(d.p, n);
}

__global__ void adjacency64_kernel(const int2* e, int64_t count, int64_t n, double* D) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int2 p = e[k];
    D[static_cast<int64_t>(p.x) * n + p.y] = 1.0;
    D[static_cast<int64_t>(p.y) * n + p.x] = 1.0;
  }
}

// ‖A‖₂ of adjacency_distance(g) (tasks.cpp:167-174) built on the device.
static double spectral_norm_graph(const int32_t* edges, int64_t count, int64_t n) {
  DBuf<double> d(static_cast<size_t>(n) * n);
  if (count > 0) {
    DBuf<int2> e(static_cast<size_t>(count));
    GWB_CUDA(cudaMemcpyAsync(e.p, edges, sizeof(int2) * count, cudaMemcpyHostToDevice, t_leaf));
    adjacency64_kernel<<<static_cast<unsigned>(std::min<int64_t>(blocks(count, 256), 1184)), 256, 0, t_leaf>>>(
        e.p, count, n, d.p);
    GWB_CUDA(cudaGetLastError());
  }
  return spectral_norm_on_device(d.p, n);
}

double device_lipschitz_bound(const double* dx, int64_t n, const double* dy, int64_t m) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  return spectral_norm_dev(dx, n) * spectral_norm_dev(dy, m);
}

double device_lipschitz_bound_graphs(const GraphInput& g, int64_t n, int64_t m) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  return spectral_norm_graph(g.ex, g.cx, n) * spectral_norm_graph(g.ey, g.cy, m);
}

void device_sinkhorn(const double* kernel, int64_t n, int64_t m, const double* mu,
                     const double* nu, double tol, int32_t max_iters, int32_t log_domain,
                     double* out, int32_t* iterations, double* marginal_error,
                     int32_t* converged) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  const int64_t len = n * m;
  DBuf<double> c(static_cast<size_t>(len)), dmu(n), dnu(m), rs(n), cs(m);
  dmu.up(mu);
  dnu.up(nu);
  *iterations = 0;
  *marginal_error = 0.0;
  *converged = 0;
  DBuf<int> bad(1);
  if (!log_domain) {  // projections.cpp:92-116
    c.up(kernel);
    for (int sweep = 1; sweep <= max_iters; ++sweep) {
      kl_scale_dev(c, n, m, dmu, GWB_ROWS, rs);
      kl_scale_dev(c, n, m, dnu, GWB_COLS, cs);
      const int zero = 0;
      bad.up(&zero);
      all_finite_kernel<<<592, 256, 0, t_leaf>>>(c.p, len, bad.p);
      int hb;
      bad.down(&hb);
      if (hb) api_numerical("sinkhorn", sweep, "non-finite entries after scaling sweep");
      *iterations = sweep;
      *marginal_error = marginal_err_inf(c, n, m, mu, nu, rs, cs);
      if (*marginal_error <= tol) {
        *converged = 1;
        break;
      }
    }
  } else {  // projections.cpp:129-163
    DBuf<double> e(static_cast<size_t>(len)), f(n), g(m);
    e.up(kernel);
    for (int sweep = 1; sweep <= max_iters; ++sweep) {
      lse_rows_kernel<<<blocks(n, 128), 128, 0, t_leaf>>>(e.p, n, m, g.p, dmu.p, f.p);
      lse_cols_kernel<<<static_cast<unsigned>(m), 256, 0, t_leaf>>>(e.p, n, m, f.p, dnu.p, g.p);
      exp_fg_kernel<<<blocks(len, 256), 256, 0, t_leaf>>>(e.p, n, m, f.p, g.p, c.p);
      const int zero = 0;
      bad.up(&zero);
      all_finite_kernel<<<592, 256, 0, t_leaf>>>(c.p, len, bad.p);
      int hb;
      bad.down(&hb);
      if (hb) api_numerical("sinkhorn-log", sweep, "non-finite entries after scaling sweep");
      *iterations = sweep;
      *marginal_error = marginal_err_inf(c, n, m, mu, nu, rs, cs);
      if (*marginal_error <= tol) {
        *converged = 1;
        break;
      }
    }
  }
  c.down(out);
}

// G = D_X π D_Y (solvers.cpp:16-19) on device fp32 row-major operands with
// the tcgen05 chain in 3xTF32 (splits computed here); G row-major, ld = ldm.
void structure_product_dev(const float* Dx_in, int64_t ldn, const float* Dy_in, int64_t ldm,
                           const float* P_in, int64_t n, int64_t m, float* G_out,
                           cudaStream_t s) {
  DBuf<float> Dx_lo(n * ldn), Dy_lo(m * ldm), P_lo(n * ldm), Vt(m * round_up(n, 32)),
      Vt_lo(m * round_up(n, 32));
  launch_tf32_aux(Dx_in, n, n, ldn, Dx_lo.p, 2, s);
  launch_tf32_aux(Dy_in, m, m, ldm, Dy_lo.p, 2, s);
  launch_tf32_aux(P_in, n, m, ldm, P_lo.p, 2, s);
  const int64_t ldv = round_up(n, 32);
  GemmDesc g1;
  g1.M = m; g1.N = n; g1.K = m;
  g1.a = Dy_in; g1.a_lo = Dy_lo.p; g1.lda = ldm;
  g1.b = P_in; g1.b_lo = P_lo.p; g1.ldb = ldm;
  g1.c = Vt.p; g1.c_aux = Vt_lo.p; g1.ldc = ldv; g1.aux_mode = 2;
  g1.three_pass = true;
  GemmDesc g2;
  g2.M = n; g2.N = m; g2.K = n;
  g2.a = Dx_in; g2.a_lo = Dx_lo.p; g2.lda = ldn;
  g2.b = Vt.p; g2.b_lo = Vt_lo.p; g2.ldb = ldv;
  g2.c = G_out; g2.ldc = ldm;
  g2.three_pass = true;
  GemmPlan* p1 = gemm_plan_create(g1);
  GemmPlan* p2 = gemm_plan_create(g2);
  GWB_CUDA(gemm_launch(p1, s));
  GWB_CUDA(gemm_launch(p2, s));
  GWB_CUDA(cudaStreamSynchronize(s));  // the DBuf temporaries are freed on return
  gemm_plan_destroy(p1);
  gemm_plan_destroy(p2);
}

// −⟨D_X π D_Y, π⟩ (solvers.cpp:64-69) on device fp32 row-major operands.
double gw_objective_dev(const float* Dx_in, int64_t ldn, const float* Dy_in, int64_t ldm,
                        const float* P_in, int64_t n, int64_t m, cudaStream_t s) {
  DBuf<float> G(n * ldm);
  structure_product_dev(Dx_in, ldn, Dy_in, ldm, P_in, n, m, G.p, s);
  DBuf<double> part(n);
  dot_rows_kernel<<<static_cast<unsigned>(n), 256, 0, s>>>(G.p, P_in, n, m, ldm, part.p);
  GWB_CUDA(cudaGetLastError());
  GWB_CUDA(cudaStreamSynchronize(s));
  return -reduce_host(part);
}

double device_gw_objective(const double* dx, int64_t n, const double* dy, int64_t m,
                           const double* pi) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  const int64_t ldn = round_up(n, 32), ldm = round_up(m, 32);
  const int64_t big = std::max(n * n, std::max(m * m, n * m));
  DBuf<double> stage(static_cast<size_t>(big));
  DBuf<float> Dx(n * ldn), Dy(m * ldm), P(n * ldm);
  cudaStream_t s = leaf.s;
  GWB_CUDA(cudaMemcpyAsync(stage.p, dx, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
  launch_colmajor64_to_rowmajor32(stage.p, n, n, Dx.p, ldn, s);
  GWB_CUDA(cudaMemcpyAsync(stage.p, dy, sizeof(double) * m * m, cudaMemcpyHostToDevice, s));
  launch_colmajor64_to_rowmajor32(stage.p, m, m, Dy.p, ldm, s);
  GWB_CUDA(cudaMemcpyAsync(stage.p, pi, sizeof(double) * n * m, cudaMemcpyHostToDevice, s));
  launch_colmajor64_to_rowmajor32(stage.p, n, m, P.p, ldm, s);
  return gw_objective_dev(Dx.p, ldn, Dy.p, ldm, P.p, n, m, s);
}

// coupling_entropy (diagnostics.cpp:44-53): −Σ π log π over positive entries.
__global__ void entropy_kernel(const double* __restrict__ pi, int64_t len, double* part) {
  double h = 0.0;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double p = pi[k];
    if (p > 0.0) h -= p * log(p);
  }
  h = dev::warp_sum(h);
  __shared__ double sh[32];
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

double coupling_entropy_dev(const double* pi_dev, int64_t len, cudaStream_t s) {
  constexpr int kBlocks = 592;
  DBuf<double> part(kBlocks);
  entropy_kernel<<<kBlocks, 256, 0, s>>>(pi_dev, len, part.p);
  GWB_CUDA(cudaGetLastError());
  GWB_CUDA(cudaStreamSynchronize(s));
  return reduce_host(part);
}

double device_coupling_entropy(const double* pi, int64_t n, int64_t m) {
  GWB_CUDA(cudaSetDevice(api_device()));
  LeafStream leaf;
  DBuf<double> d(static_cast<size_t>(n) * m);
  d.up(pi);
  return coupling_entropy_dev(d.p, n * m, leaf.s);
}

}  // namespace gwb
