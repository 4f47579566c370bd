// bregman.cu — eBPG / BPG / hBPG on the device (reference solvers.cpp:219-426).
//
// Per outer iteration k (π = current coupling, P[q]):
//   GEMM chain            G = D_X·π·D_Y                       (tcgen05, 3xTF32)
//   form   (row pass)     ⟨G,π⟩ for record k−1's objective;
//                         eBPG: E = (2/ε)G, BPG: E = 2t·G, log-kernel
//                         LK = E (eBPG) or log π + E (BPG), stored (fp64)
//                         in one pass; max_j LK per row for the dead-line test
//   check                 BPG overflow (max E > 700), eBPG dead lines,
//                         reset of the Sinkhorn potentials
//   sweeps s=1..inner     row LSE → f (fp64), column LSE (chunked partials +
//                         fixed-order merge) → g, then the write pass
//                         π' = exp(max(LK, clamp) + f + g) (+ perturbation)
//                         with row/column sums, ‖π'−π‖², ‖π‖², whose row sums
//                         give the early-exit test of sweep s (the reference's
//                         ∞-norm marginal test after a full ROWS→COLS sweep,
//                         projections.cpp:101-113); later sweeps are skipped
//   finalize              trace record, stop rule, hBPG phase switch.
// The Sinkhorn runs in the log domain with fp64 potentials over the fp64
// log-kernel (any row shift is absorbed by the row potential f): identical to the reference's plain-domain
// alternating scaling (rows first) whenever the latter is finite, with the
// reference's 1e-300 kernel clamp applied as a log-space floor and its error
// semantics (dead lines, zero-sum lines, overflow, non-finite) emulated.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "devutil.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "solver.cuh"
#include "standalone.cuh"

namespace gwb {

namespace {

using namespace dev;

constexpr double kLogClamp = -690.7755278982137;     // log(1e-300)
constexpr double kExpUnderflow = -745.1332191019412;  // fp64 exp(x) == 0 below
constexpr int kThreads = 256;
constexpr int kColWidth = 128;

enum BFlag : int {
  kBOverflow = 1,   // BPG: max(2t·D_X π D_Y) > 700
  kBDeadLine = 2,   // eBPG (plain): a kernel line underflowed to zero
  kBZeroRow = 4,    // Sinkhorn row with zero sum   (index: zero_index)
  kBZeroCol = 8,    // Sinkhorn column with zero sum
  kBNonFinite = 16, // Sinkhorn produced non-finite values (sweep: err_sweep)
};

struct BState {
  int done, flags, iter, err_iter, converged;
  int zero_index, err_sweep;
  int phase;      // 1 = eBPG, 2 = BPG
  int used1, conv1;
  int sink_done, sweeps;
  int gmax_bits;  // max of E over the matrix (E ≥ 0), float bits
  unsigned long long t0;
};

struct BRecord {
  double obj;      // ⟨M(π), π⟩, filled one iteration later
  double rel, infeas, elapsed;
  int phase, sweeps;
};

struct BDev {
  int64_t n, m, ld;
  const float* G;       // chain output (fp32)
  double* LK;           // row-shifted log-kernel LKs (fp64, n × ld)
  const double* P;      // π_k (fp64)
  double* P_new;
  float* P32_new;       // fp32 copy of π_{k+1}: the 3xTF32 hi operand (nullable)
  float* P_aux_new;
  int aux_mode;         // GEMM operand copy of P_new: 2 = 3xTF32 residual, 3/4 = bf16
                        // planes, 5 = fp16 planes of P_new·aux_scale (f16x2)
  float aux_scale;
  int64_t plane;        // elements per bf16 plane (n·ld)
  const double* mu64;
  const double* nu64;
  double* f;
  double* f_new;
  double* g;
  double* rowmax;
  double* row_sum_raw;  // colblocks × n: write-pass row sums before the BPG perturbation
  double* err_part;     // sweep marginal-error partials (max), as dev_part
  double* col_err;
  double* col_pm;       // chunks × m  (max, fp64)
  double* col_ps;       // chunks × m  (Σ exp, fp64)
  float* col_pemax;     // chunks × m  (max of unshifted E; sweep 1, eBPG plain)
  double* col_sum;      // chunks × m  (write-pass column sums)
  double* row_sum;      // colblocks × n
  double* obj_part;     // n
  double* wpart;        // (colblocks·chunks) × 2
  double* dev_part;     // marginal deviation partials: row blocks, then column blocks
  int chunks, colblocks;
  int dev_rb, dev_cb;   // blocks of 256 rows / columns in dev_part
  double eb_scale;      // 2/ε
  double bp_scale;      // 2t
  int log_domain;
  double perturb, uniform_mass;
  int budget1, max_iters, has_phase2;
  double rel_tol, inner_tol;
  BState* st;
  BRecord* rec;
  int max_rec;
};

__device__ __forceinline__ bool skip(const BDev& d) { return d.st->done != 0; }
__device__ __forceinline__ bool skip_sink(const BDev& d) {
  return d.st->done != 0 || d.st->sink_done != 0;
}

// Clamp floor of the log-kernel: the reference clamps the kernel at 1e-300
// (solvers.cpp:252, :331); eBPG's kernel is exp(E − max E), so its floor on
// LK = E sits at log(1e-300) + max E.
__device__ __forceinline__ double clamp_floor(const BDev& d) {
  if (d.st->phase == 1) {
    if (d.log_domain) return -INFINITY;
    return kLogClamp + static_cast<double>(__int_as_float(d.st->gmax_bits));
  }
  return kLogClamp;
}

__device__ double block_sum(double v) {
  __shared__ double sh[32];
  v = warp_sum(v);
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  for (int q = 0; q < static_cast<int>(blockDim.x / 32); ++q) t += sh[q];
  return t;
}

__device__ float block_max(float v) {
  __shared__ float sh[32];
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  float t = -INFINITY;
  for (int q = 0; q < static_cast<int>(blockDim.x / 32); ++q) t = fmaxf(t, sh[q]);
  return t;
}

__device__ double block_max_d(double v) {
  __shared__ double sh[32];
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = -INFINITY;
  for (int q = 0; q < static_cast<int>(blockDim.x / 32); ++q) t = fmax(t, sh[q]);
  return t;
}

// (max, Σ e^{x−max}) in fp64 state with fp32 exponentials of small
// arguments: the online LSE accumulator of the BAPG projections
// (devutil.cuh), instantiated for fp64 with unit weights.

// ---------------------------------------------------------------------------
// form: one warp per row (8 rows per CTA).  A CTA per row kept too few
// bytes in flight per SM: 78 elements per thread, a block-merge tail per row.
constexpr int kRowsPerCta = kThreads / 32;

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(kThreads) form_kernel(BDev d, int tail) {
  if (tail ? d.st->flags != 0 : skip(d)) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + warp;
  const bool ebpg = d.st->phase == 1;
  const double sc = ebpg ? d.eb_scale : d.bp_scale;
  float emax = 0.0f;
  if (i < d.n) {
    const float* g = d.G + i * d.ld;
    const double* p = d.P + i * d.ld;
    double* lkrow = d.LK + i * d.ld;
    double obj = 0.0;
    double rmax = -INFINITY;
    // One pass: G and π are read once and LK is written unshifted (a row
    // shift would need a second pass; the row potential f absorbs it).
    // 4 consecutive columns per lane (float4 of G, double2 pairs of π and
    // LK); ld is a multiple of 32, so a group that starts in the row stays
    // in it, and padding columns (G = π = 0) are masked.
#pragma unroll 2
    for (int64_t j = 4 * lane; j < d.m; j += 128) {
      const float4 g4 = *reinterpret_cast<const float4*>(g + j);
      const double2 p01 = *reinterpret_cast<const double2*>(p + j);
      const double2 p23 = *reinterpret_cast<const double2*>(p + j + 2);
      const double gv[4] = {g4.x, g4.y, g4.z, g4.w};
      const double pv[4] = {p01.x, p01.y, p23.x, p23.y};
      double lk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool in = j + q < d.m;
        obj = __fma_rn(gv[q], pv[q], obj);
        const double e = sc * gv[q];
        lk[q] = ebpg ? e : e + log(pv[q]);
        if (in) {
          emax = fmaxf(emax, static_cast<float>(e));
          rmax = fmax(rmax, lk[q]);
        }
      }
      if (tail) continue;
      *reinterpret_cast<double2*>(lkrow + j) = make_double2(lk[0], lk[1]);
      *reinterpret_cast<double2*>(lkrow + j + 2) = make_double2(lk[2], lk[3]);
    }
    obj = warp_sum(obj);
    rmax = warp_max_d(rmax);
    if (lane == 0) {
      d.obj_part[i] = obj;
      if (!tail) d.rowmax[i] = rmax;
    }
  }
  if (tail) return;
  emax = block_max(emax);
  if (threadIdx.x == 0) atomicMax(&d.st->gmax_bits, __float_as_int(emax));
}

// Checks after the form pass + Sinkhorn reset.  One block.
__global__ void form_check_kernel(BDev d) {
  BState* st = d.st;
  if (skip(d)) return;
  const float gmax = __int_as_float(st->gmax_bits);
  double rmin = INFINITY;
  for (int64_t i = threadIdx.x; i < d.n; i += blockDim.x) rmin = fmin(rmin, d.rowmax[i]);
  rmin = -block_max_d(-rmin);
  for (int64_t j = threadIdx.x; j < d.m; j += blockDim.x) d.g[j] = 0.0;
  if (threadIdx.x == 0) {
    st->sink_done = 0;
    st->sweeps = 0;
    if (st->phase == 2 && gmax > 700.0f) {
      atomicOr(&st->flags, kBOverflow);
    } else if (st->phase == 1 && !d.log_domain &&
               static_cast<double>(rmin) - gmax < kExpUnderflow) {
      atomicOr(&st->flags, kBDeadLine);
    }
    if (st->flags) {
      st->done = 1;
      st->err_iter = st->iter;
    }
  }
}

// Adds four terms to an online (max, Σ): at most one rescale per group, then
// four independent exponentials.  Per-term new-max branches diverge across
// a warp on most steps of a short per-lane chain, evaluating both sides.
// NaN in any term gives NaN.
__device__ __forceinline__ void lse64_add4(Lse64& a, const double (&x)[4]) {
  const bool bad = isnan(x[0]) || isnan(x[1]) || isnan(x[2]) || isnan(x[3]);
  const double m4 = fmax(fmax(x[0], x[1]), fmax(x[2], x[3]));
  if (m4 > a.mx) {
    a.s = a.mx == -INFINITY ? 0.0 : a.s * exp(a.mx - m4);
    a.mx = m4;
  }
  if (m4 > -INFINITY) {
    const double e0 = exp(x[0] - a.mx), e1 = exp(x[1] - a.mx);
    const double e2 = exp(x[2] - a.mx), e3 = exp(x[3] - a.mx);
    a.s += (e0 + e1) + (e2 + e3);
  }
  if (bad) a.mx = NAN;
}

// Sinkhorn row update for sweep s: f_new = log μ − LSE_j(max(LK, floor) + g),
// fp64 terms and exponentials (the reference's arithmetic, projections.cpp:92-163).
__global__ void __launch_bounds__(kThreads) row_lse_kernel(BDev d, int s) {
  if (skip_sink(d)) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kRowsPerCta + warp;
  if (i >= d.n) return;
  const double* lk = d.LK + i * d.ld;
  const double fl = clamp_floor(d);
  // One warp per row.  Each step loads 8 columns per lane (four coalesced
  // double2 loads of LK and g over a 256-column window) into two
  // independent accumulators.  ld is a multiple of 32, so a pair that
  // starts inside the row stays inside it.
  Lse64 a[2] = {{-INFINITY, 0.0}, {-INFINITY, 0.0}};
  for (int64_t b = 0; b < d.m; b += 256) {
    double2 v[4], gg[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int64_t j = b + 64 * h + 2 * lane;
      if (j < d.m) {
        v[h] = *reinterpret_cast<const double2*>(lk + j);
        gg[h] = *reinterpret_cast<const double2*>(d.g + j);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      double x[4];
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int h = 2 * u + h2;
        const int64_t j = b + 64 * h + 2 * lane;
        x[2 * h2] = j < d.m ? fmax(v[h].x, fl) + gg[h].x : -INFINITY;
        x[2 * h2 + 1] = j + 1 < d.m ? fmax(v[h].y, fl) + gg[h].y : -INFINITY;
      }
      lse64_add4(a[u], x);
    }
  }
  const Lse64 r = lse64_warp_merge(lse64_merge(a[0], a[1]));
  if (lane != 0) return;
  const double lse = r.mx + log(r.s);
  const double fn = log(d.mu64[i]) - lse;
  d.f_new[i] = fn;
  if (isnan(lse) || !(r.s > 0.0) || r.mx == -INFINITY) {
    const bool plain = !(d.st->phase == 1 && d.log_domain);
    if (plain && !isnan(lse)) {
      atomicOr(&d.st->flags, kBZeroRow);
      atomicMin(&d.st->zero_index, static_cast<int>(i));
    } else {
      atomicOr(&d.st->flags, kBNonFinite);
    }
  }
}

// Row-pass flags and f ← f_new.  One block.
__global__ void row_decide_kernel(BDev d, int s) {
  BState* st = d.st;
  if (skip_sink(d)) return;
  if (st->flags) {
    if (threadIdx.x == 0) {
      st->done = 1;
      st->err_iter = st->iter;
      st->err_sweep = s;
    }
    return;
  }
  for (int64_t i = threadIdx.x; i < d.n; i += blockDim.x) d.f[i] = d.f_new[i];
  if (threadIdx.x == 0) st->sweeps = s;
}

// Column LSE partials: (128-column block, row chunk) per CTA.
__global__ void __launch_bounds__(kThreads) col_lse_partial_kernel(BDev d, int rows_per_chunk,
                                                                   int first_sweep) {
  if (skip_sink(d)) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kColWidth + lane * 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = (r0 + rows_per_chunk < d.n) ? r0 + rows_per_chunk : d.n;
  const bool want_emax = first_sweep && d.st->phase == 1 && !d.log_domain;
  const double fl = clamp_floor(d);
  Lse64 a[4] = {{-INFINITY, 0.0}, {-INFINITY, 0.0}, {-INFINITY, 0.0}, {-INFINITY, 0.0}};
  float emax[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  if (c0 < d.m) {
    for (int64_t i = r0 + warp; i < r1; i += kThreads / 32) {
      const double* lk = d.LK + i * d.ld + c0;
      const double2 v01 = *reinterpret_cast<const double2*>(lk);
      const double2 v23 = *reinterpret_cast<const double2*>(lk + 2);
      const double fi = d.f[i];
      const double vv[4] = {v01.x, v01.y, v23.x, v23.y};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        lse64_add(a[q], fmax(vv[q], fl) + fi, 1.0);
        if (want_emax) emax[q] = fmaxf(emax[q], static_cast<float>(vv[q]));
      }
    }
  }
  __shared__ double s_mx[kThreads / 32][kColWidth];
  __shared__ double s_s[kThreads / 32][kColWidth];
  __shared__ float s_e[kThreads / 32][kColWidth];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    s_mx[warp][lane * 4 + q] = a[q].mx;
    s_s[warp][lane * 4 + q] = a[q].s;
    s_e[warp][lane * 4 + q] = emax[q];
  }
  __syncthreads();
  if (threadIdx.x < kColWidth) {
    const int c = threadIdx.x;
    const int64_t col = static_cast<int64_t>(blockIdx.x) * kColWidth + c;
    if (col < d.m) {
      Lse64 r{-INFINITY, 0.0};
      float e = -INFINITY;
      for (int q = 0; q < kThreads / 32; ++q) {
        r = lse64_merge(r, Lse64{s_mx[q][c], s_s[q][c]});
        e = fmaxf(e, s_e[q][c]);
      }
      const int64_t o = static_cast<int64_t>(blockIdx.y) * d.m + col;
      d.col_pm[o] = r.mx;
      d.col_ps[o] = r.s;
      d.col_pemax[o] = e;
    }
  }
}

__global__ void col_lse_combine_kernel(BDev d, int first_sweep) {
  if (skip_sink(d)) return;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= d.m) return;
  Lse64 r{-INFINITY, 0.0};
  float e = -INFINITY;
  for (int c = 0; c < d.chunks; ++c) {
    const int64_t o = static_cast<int64_t>(c) * d.m + j;
    r = lse64_merge(r, Lse64{d.col_pm[o], d.col_ps[o]});
    e = fmaxf(e, d.col_pemax[o]);
  }
  const double lse = r.mx + log(r.s);
  const double gn = log(d.nu64[j]) - lse;
  d.g[j] = gn;
  d.col_err[j] = fabs(exp(gn + lse) - d.nu64[j]);
  const bool plain = !(d.st->phase == 1 && d.log_domain);
  if (first_sweep && d.st->phase == 1 && !d.log_domain &&
      static_cast<double>(e) - __int_as_float(d.st->gmax_bits) < kExpUnderflow)
    atomicOr(&d.st->flags, kBDeadLine);
  if (isnan(lse) || !(r.s > 0.0) || r.mx == -INFINITY) {
    if (plain && !isnan(lse)) {
      atomicOr(&d.st->flags, kBZeroCol);
      atomicMin(&d.st->zero_index, static_cast<int>(j));
    } else {
      atomicOr(&d.st->flags, kBNonFinite);
    }
  }
}

__global__ void col_flag_kernel(BDev d, int s) {
  BState* st = d.st;
  if (skip_sink(d)) return;
  if (st->flags) {
    st->done = 1;
    st->err_iter = st->iter;
    st->err_sweep = s;
  }
}

// π' = exp(max(LKs, floor) + f + g) (+ perturbation), fused sums.
__global__ void __launch_bounds__(kThreads) write_kernel(BDev d, int rows_per_chunk) {
  if (skip_sink(d)) return;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kColWidth + lane * 4;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * rows_per_chunk;
  const int64_t r1 = (r0 + rows_per_chunk < d.n) ? r0 + rows_per_chunk : d.n;
  // Remark-1 perturbation applies to BPG iterations only (solvers.cpp:263-267).
  const bool perturb = d.perturb > 0.0 && d.st->phase == 2;
  const double keep = 1.0 - d.perturb;
  const double add = d.perturb * d.uniform_mass;
  double cs[4] = {0.0, 0.0, 0.0, 0.0};
  double diff = 0.0, old = 0.0;
  const bool ok = c0 < d.m;
  double gj[4] = {0.0, 0.0, 0.0, 0.0};
  if (ok)
#pragma unroll
    for (int q = 0; q < 4; ++q) gj[q] = (c0 + q < d.m) ? d.g[c0 + q] : 0.0;
  const double fl = clamp_floor(d);
#pragma unroll 2
  for (int64_t i = r0 + warp; i < r1; i += kThreads / 32) {
    double rs = 0.0, rr = 0.0;
    if (ok) {
      // c0 < m ≤ ld and ld is a multiple of 32: the 4 entries stay in the row.
      const double2 lk01 = *reinterpret_cast<const double2*>(d.LK + i * d.ld + c0);
      const double2 lk23 = *reinterpret_cast<const double2*>(d.LK + i * d.ld + c0 + 2);
      const double2 pp01 = *reinterpret_cast<const double2*>(d.P + i * d.ld + c0);
      const double2 pp23 = *reinterpret_cast<const double2*>(d.P + i * d.ld + c0 + 2);
      const double lk[4] = {lk01.x, lk01.y, lk23.x, lk23.y};
      const double pp[4] = {pp01.x, pp01.y, pp23.x, pp23.y};
      const double fi = d.f[i];
      double o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (c0 + q < d.m) {
          const double x = fmax(lk[q], fl) + fi + gj[q];
          double val = exp(x);
          rr += val;
          if (perturb) val = keep * val + add;
          o[q] = val;
          cs[q] += val;
          rs += val;
          const double df = val - pp[q];
          diff += df * df;
          old += pp[q] * pp[q];
        } else {
          o[q] = 0.0;
        }
      }
      double* pn = d.P_new + i * d.ld + c0;
      *reinterpret_cast<double2*>(pn) = make_double2(o[0], o[1]);
      *reinterpret_cast<double2*>(pn + 2) = make_double2(o[2], o[3]);
      aux_store4_64(d.P_aux_new, d.P32_new, d.aux_mode, d.plane, i * d.ld + c0, o, d.aux_scale);
    }
    rs = warp_sum(rs);
    if (lane == 0) d.row_sum[static_cast<int64_t>(blockIdx.x) * d.n + i] = rs;
    if (perturb) {
      rr = warp_sum(rr);
      if (lane == 0) d.row_sum_raw[static_cast<int64_t>(blockIdx.x) * d.n + i] = rr;
    }
  }
  __shared__ double s_c[kThreads / 32][kColWidth];
#pragma unroll
  for (int q = 0; q < 4; ++q) s_c[warp][lane * 4 + q] = cs[q];
  diff = block_sum(diff);
  old = block_sum(old);
  __syncthreads();
  if (threadIdx.x < kColWidth) {
    const int64_t col = static_cast<int64_t>(blockIdx.x) * kColWidth + threadIdx.x;
    if (col < d.m) {
      double t = 0.0;
      for (int q = 0; q < kThreads / 32; ++q) t += s_c[q][threadIdx.x];
      d.col_sum[static_cast<int64_t>(blockIdx.y) * d.m + col] = t;
    }
  }
  if (threadIdx.x == 0) {
    const int64_t cta = static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x;
    d.wpart[2 * cta] = diff;
    d.wpart[2 * cta + 1] = old;
  }
}

// After the write pass of a sweep, per block of 256 lines (fixed order):
// the record's marginal deviations Σ_i (row sum − μ_i)², Σ_j (column sum −
// ν_j)² of the written coupling, and the sweep's ∞-norm marginal error
// (|row sum − μ_i| of the coupling before the BPG perturbation, and the
// column errors of the column step).  (One block reading the colblocks × n
// row partials took 1.2 ms at c4.)
__global__ void __launch_bounds__(256) sink_partial_kernel(BDev d) {
  if (skip_sink(d)) return;
  const int b = blockIdx.x;
  const bool perturb = d.perturb > 0.0 && d.st->phase == 2;
  double v = 0.0, e = 0.0;
  if (b < d.dev_rb) {
    const int64_t i = static_cast<int64_t>(b) * 256 + threadIdx.x;
    if (i < d.n) {
      double s = 0.0;
      for (int c = 0; c < d.colblocks; ++c) s += d.row_sum[static_cast<int64_t>(c) * d.n + i];
      v = (s - d.mu64[i]) * (s - d.mu64[i]);
      if (perturb) {
        s = 0.0;
        for (int c = 0; c < d.colblocks; ++c) s += d.row_sum_raw[static_cast<int64_t>(c) * d.n + i];
      }
      e = fabs(s - d.mu64[i]);
    }
  } else {
    const int64_t j = static_cast<int64_t>(b - d.dev_rb) * 256 + threadIdx.x;
    if (j < d.m) {
      double s = 0.0;
      for (int c = 0; c < d.chunks; ++c) s += d.col_sum[static_cast<int64_t>(c) * d.m + j];
      v = (s - d.nu64[j]) * (s - d.nu64[j]);
      e = d.col_err[j];
    }
  }
  v = block_sum(v);
  e = block_max_d(e);
  if (threadIdx.x == 0) {
    d.dev_part[b] = v;
    d.err_part[b] = e;
  }
}

// Early exit after sweep s: ∞-norm marginal error ≤ inner_tol, or the last
// sweep.  One block.
__global__ void sink_decide_kernel(BDev d, int s, int last) {
  BState* st = d.st;
  if (skip_sink(d)) return;
  double e = 0.0;
  for (int b = threadIdx.x; b < d.dev_rb + d.dev_cb; b += blockDim.x) e = fmax(e, d.err_part[b]);
  e = block_max_d(e);
  if (threadIdx.x == 0) {
    st->sweeps = s;
    if (last || e <= d.inner_tol) st->sink_done = 1;
  }
}

// Record k, stop rule, phase logic.  One block.
__global__ void breg_finalize_kernel(BDev d, int tail) {
  BState* st = d.st;
  if (tail ? st->flags != 0 : skip(d)) return;
  const int k = tail ? st->iter - 1 : st->iter;
  auto slot = [&](int it) { return it <= d.max_rec ? it : d.max_rec + 1; };
  double obj = 0.0;
  for (int64_t i = threadIdx.x; i < d.n; i += blockDim.x) obj += d.obj_part[i];
  obj = block_sum(obj);
  if (tail) {
    if (threadIdx.x == 0) d.rec[slot(k)].obj = obj;
    return;
  }
  double rowdev = 0.0, coldev = 0.0, diff = 0.0, old = 0.0;
  for (int b = threadIdx.x; b < d.dev_rb; b += blockDim.x) rowdev += d.dev_part[b];
  for (int b = threadIdx.x; b < d.dev_cb; b += blockDim.x) coldev += d.dev_part[d.dev_rb + b];
  const int64_t ctas = static_cast<int64_t>(d.chunks) * d.colblocks;
  for (int64_t c = threadIdx.x; c < ctas; c += blockDim.x) {
    diff += d.wpart[2 * c];
    old += d.wpart[2 * c + 1];
  }
  rowdev = block_sum(rowdev);
  coldev = block_sum(coldev);
  diff = block_sum(diff);
  old = block_sum(old);
  if (threadIdx.x != 0) return;
  if (k >= 2) d.rec[slot(k - 1)].obj = obj;
  BRecord& r = d.rec[slot(k)];
  r.rel = sqrt(diff) / sqrt(old);
  r.infeas = sqrt(coldev) / static_cast<double>(d.m) + sqrt(rowdev) / static_cast<double>(d.n);
  r.elapsed = 1e-9 * static_cast<double>(globaltimer() - st->t0);
  r.phase = st->phase;
  r.sweeps = st->sweeps;
  const bool conv = dev::stop_rule(r.rel, d.rel_tol);
  st->iter = k + 1;
  st->gmax_bits = 0;
  if (st->phase == 1) {
    if (conv || k >= d.budget1) {
      st->used1 = k;
      st->conv1 = conv;
      if (!d.has_phase2 || d.max_iters - k < 1) {
        st->done = 1;
        st->converged = conv;
      } else {
        st->phase = 2;
      }
    }
  } else if (conv) {
    st->done = 1;
    st->converged = 1;
  }
  if (k >= d.max_iters) st->done = 1;
}

__global__ void breg_reset_kernel(BState* st, int phase) {
  st->done = 0;
  st->flags = 0;
  st->iter = 1;
  st->err_iter = 0;
  st->converged = 0;
  st->zero_index = 0x7fffffff;
  st->err_sweep = 0;
  st->phase = phase;
  st->used1 = 0;
  st->conv1 = 0;
  st->sink_done = 0;
  st->sweeps = 0;
  st->gmax_bits = 0;
  st->t0 = globaltimer();
}

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  GWB_CUDA(cudaMalloc(&p, count * sizeof(T) + 256));
  GWB_CUDA(cudaMemset(p, 0, count * sizeof(T) + 256));
  GWB_CUDA(cudaStreamSynchronize(cudaStreamLegacy));  // see solver.cu dalloc
  return static_cast<T*>(p);
}

struct DevFree {
  void operator()(void* p) const {
    if (p) cudaFree(p);
  }
};

// ---------------------------------------------------------------------------
class BregmanEngine {
 public:
  // world > 0: row-sharded chain (rank of world).  Rank r owns
  // rows [r·n_r, r·n_r + n_r) of D_X (n_r = ⌈n/world⌉ rounded up to 64) and
  // computes those rows of G; Vᵀ and G are completed by caller-issued
  // all-gathers between the phases (sphase), and π, the Sinkhorn state and
  // the records stay replicated — every rank runs the same deterministic
  // kernels on the same data, so stop and phase decisions agree.
  BregmanEngine(int device, int64_t n, int64_t m, const gwb_config& cfg, int algo,
                int world = 0, int rank = 0, cudaStream_t stream = nullptr)
      : dev_(device), n_(n), m_(m), ldn_(round_up(n, 32)), ldm_(round_up(m, 32)), cfg_(cfg),
        algo_(algo) {
    GWB_CUDA(cudaSetDevice(dev_));
    if (stream) {
      s_ = stream;
    } else {
      GWB_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
      own_stream_ = true;
    }
    pool_keep(dev_);
    {
      // Grow the pool once by (an upper bound of) the engine's workspace and
      // return it, so the ~36 buffers below are carved from it instead of
      // growing the pool one mapping at a time (cold solve at c4: 1.2 s).
      const size_t nm_b = static_cast<size_t>(round_up(n_, 64)) * static_cast<size_t>(ldm_);
      const size_t total = 60 * nm_b + 16 * static_cast<size_t>(ldn_) * ldn_ +
                           16 * static_cast<size_t>(ldm_) * ldm_;
      void* w = nullptr;
      if (cudaMallocAsync(&w, total, s_) == cudaSuccess) cudaFreeAsync(w, s_);
      cudaGetLastError();
    }
    sharded_ = world > 0;
    rows_alloc_ = n_;
    if (sharded_) {
      world_ = world;
      rank_ = rank;
      nr_ = round_up((n_ + world_ - 1) / world_, 64);
      npad_ = nr_ * world_;
      row0_ = static_cast<int64_t>(rank_) * nr_;
      rows_valid_ = std::max<int64_t>(0, std::min<int64_t>(nr_, n_ - row0_));
      ldk_ = round_up(npad_, 64);
      rows_alloc_ = npad_;
      // The chain precision is fixed up front (resolved by the orchestrator):
      // it sets the exchange-buffer layout the caller allocates.
      const int req = cfg_.precision;
      aux_mode_ = req == GWB_PREC_BF16X3 ? 3 : req == GWB_PREC_BF16X2 ? 4 : req == GWB_PREC_F16X2 ? 5 : 2;
      planes_ = aux_mode_ == 3 ? 3 : 2;
      esize_ = aux_mode_ >= 3 ? 2 : 4;
    }
    pstride_ = rows_alloc_ * ldm_;
    const size_t nm = static_cast<size_t>(rows_alloc_) * ldm_;
    const size_t dx_elems =
        sharded_ ? static_cast<size_t>(nr_) * ldk_ : static_cast<size_t>(n_) * ldn_;
    Dx_ = keep(salloc<float>(dx_elems));
    Dy_ = keep(salloc<float>(static_cast<size_t>(m_) * ldm_));
    Dx_lo_ = keep(salloc<float>(dx_elems));
    Dy_lo_ = keep(salloc<float>(static_cast<size_t>(m_) * ldm_));
    for (int q = 0; q < 2; ++q) {
      P_[q] = keep(salloc<float>(nm));            // fp32 hi operand (3xTF32)
      Pa_[q] = keep(salloc<float>(nm * 3 / 2));  // fp32 residual or up to 3 bf16 planes
      P64_[q] = keep(salloc<double>(nm));         // the iterate π (fp64)
    }
    LK_ = keep(salloc<double>(nm));               // row-shifted log-kernel (fp64)
    Vt_ = sharded_ ? nullptr : keep(salloc<float>(static_cast<size_t>(m_) * ldn_));
    Vta_ = sharded_ ? nullptr : keep(salloc<float>(static_cast<size_t>(m_) * ldn_ * 3 / 2));
    G_ = sharded_ ? nullptr : keep(salloc<float>(nm));  // sharded: caller-owned (set_comm)
    mu_ = keep(salloc<double>(n_));
    nu_ = keep(salloc<double>(m_));
    f_ = keep(salloc<double>(n_));
    fn_ = keep(salloc<double>(n_));
    g_ = keep(salloc<double>(m_));
    rowmax_ = keep(salloc<double>(n_));
    col_err_ = keep(salloc<double>(m_));
    colblocks_ = static_cast<int>((m_ + kColWidth - 1) / kColWidth);
    // Row chunks of the column passes: ~16 CTAs per SM — the fp64 online LSE
    // per element is latency-bound, so the column pass needs the parallelism
    // (4 per SM ran the c4 column partial at 1.96 TB/s).
    chunks_ = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((n_ + 63) / 64, (16 * 148 + colblocks_ - 1) / colblocks_)));
    col_pm_ = keep(salloc<double>(static_cast<size_t>(chunks_) * m_));
    col_ps_ = keep(salloc<double>(static_cast<size_t>(chunks_) * m_));
    col_pe_ = keep(salloc<float>(static_cast<size_t>(chunks_) * m_));
    col_sum_ = keep(salloc<double>(static_cast<size_t>(chunks_) * m_));
    row_sum_ = keep(salloc<double>(static_cast<size_t>(colblocks_) * n_));
    obj_part_ = keep(salloc<double>(n_));
    wpart_ = keep(salloc<double>(2 * static_cast<size_t>(chunks_) * colblocks_));
    dev_rb_ = static_cast<int>((n_ + 255) / 256);
    dev_cb_ = static_cast<int>((m_ + 255) / 256);
    dev_part_ = keep(salloc<double>(static_cast<size_t>(dev_rb_ + dev_cb_)));
    err_part_ = keep(salloc<double>(static_cast<size_t>(dev_rb_ + dev_cb_)));
    row_sum_raw_ = keep(salloc<double>(static_cast<size_t>(colblocks_) * n_));
    st_ = keep(salloc<BState>(1));
    rec_ = keep(salloc<BRecord>(static_cast<size_t>(cfg_.max_iters) + 2));
  }
  ~BregmanEngine() {
    cudaSetDevice(dev_);
    cudaStreamSynchronize(s_);
    for (auto* p : plans_) gemm_plan_destroy(p);
    for (void* p : bufs_) cudaFreeAsync(p, s_);
    cudaStreamSynchronize(s_);
    if (own_stream_) cudaStreamDestroy(s_);
  }

  // ---- sharded mode --------------------------------------------------------
  int64_t rows_per_shard() const { return nr_; }
  int64_t row_begin() const { return row0_; }
  int64_t rows_valid() const { return rows_valid_; }
  int64_t padded_rows() const { return npad_; }
  int64_t ld() const { return ldm_; }
  int planes() const { return planes_; }
  int esize() const { return esize_; }
  int64_t vt_bytes() const { return static_cast<int64_t>(planes_) * world_ * m_ * nr_ * esize_; }
  cudaStream_t stream() const { return s_; }
  // vt: [world][planes][m][n_r] gather buffer; g: npad × ld fp32 (G, all rows).
  void set_comm(void* vt, float* g) {
    vt_ = static_cast<uint8_t*>(vt);
    G_ = g;
  }

  // Sharded inputs: device fp32 rows of D_X (rows_valid × n, leading dim
  // ldx) and D_Y (m × m, ldy); host fp64 μ (n) and ν (m).  The precision
  // must be resolved (the ranks' exactness verdict, dist.resolve_precision).
  void load_sharded(const float* dx_rows, int64_t ldx, const float* dy, int64_t ldy,
                    const double* mu, const double* nu) {
    if (!vt_ || !G_) api_fail(GWB_ERR_INVALID, "bregman shard: set_comm before load");
    if (rows_valid_ > 0)
      GWB_CUDA(cudaMemcpy2DAsync(Dx_, ldk_ * 4, dx_rows, ldx * 4, n_ * 4, rows_valid_,
                                 cudaMemcpyDeviceToDevice, s_));
    GWB_CUDA(cudaMemcpy2DAsync(Dy_, ldm_ * 4, dy, ldy * 4, m_ * 4, m_, cudaMemcpyDeviceToDevice, s_));
    if (aux_mode_ >= 3) {
      // Split planes round D to fp16 / bf16: refuse an inexact D (the
      // orchestrator downgrades across ranks first, dist.resolve_precision).
      const int bits = analyze_inexact(Dx_, rows_valid_, n_, ldk_, s_) |
                       analyze_inexact(Dy_, m_, m_, ldm_, s_);
      if (!split_exact(cfg_.precision, bits))
        api_fail(GWB_ERR_CONFIG,
                 "bregman shard: the requested split-plane precision needs structure matrices "
                 "exact in fp16 (f16x2) / bf16 (bf16x3, bf16x2); resolve it across ranks first "
                 "(dist.resolve_precision)");
      Dx_bf_ = keep(salloc<float>(static_cast<size_t>(nr_) * ldk_ / 2 + 16));
      Dy_bf_ = keep(salloc<float>(static_cast<size_t>(m_) * ldm_ / 2 + 16));
      if (aux_mode_ == 5) {
        // f16x2: every rank holds the full μ, ν (host) and D_Y, so the
        // bound and the Vᵀ row scales agree across ranks.
        x_max_ = 0.0;
        for (int64_t i = 0; i < n_; ++i) x_max_ = std::max(x_max_, std::fabs(mu[i]));
        for (int64_t j = 0; j < m_; ++j) x_max_ = std::max(x_max_, std::fabs(nu[j]));
        launch_to_f16(Dx_, nr_, ldk_, ldk_, Dx_bf_, s_);
        launch_to_f16(Dy_, m_, m_, ldm_, Dy_bf_, s_);
        f16_s1_ = 14 - static_cast<int>(std::ceil(std::log2(std::max(x_max_, 1e-30))));
        f16_g1_rs_ = keep(salloc<float>(ldm_));
        f16_g2_cs_ = keep(salloc<float>(ldm_));
        launch_f16_scales(Dy_, m_, ldm_, static_cast<float>(x_max_), f16_s1_, f16_g1_rs_,
                          f16_g2_cs_, s_);
      } else {
        launch_to_bf16(Dx_, nr_, ldk_, ldk_, Dx_bf_, s_);
        launch_to_bf16(Dy_, m_, m_, ldm_, Dy_bf_, s_);
      }
    } else {
      launch_tf32_aux(Dx_, nr_, ldk_, ldk_, Dx_lo_, 2, s_);
      launch_tf32_aux(Dy_, m_, m_, ldm_, Dy_lo_, 2, s_);
    }
    GWB_CUDA(cudaMemcpyAsync(mu_, mu, sizeof(double) * n_, cudaMemcpyHostToDevice, s_));
    GWB_CUDA(cudaMemcpyAsync(nu_, nu, sizeof(double) * m_, cudaMemcpyHostToDevice, s_));
    launch_product_coupling64(mu_, nu_, n_, m_, ldm_, P64_[0], s_);
    init_copies();
    GWB_CUDA(cudaStreamSynchronize(s_));
    build_shard_plans();
    begin();
  }

  // One step of the sharded schedule for outer iteration k (ops 0–2) or the
  // tail record after `k` = iterations used (ops 3–5):
  //   0 / 3: local GEMM1 → this rank's Vᵀ slot     [caller: all-gather vt]
  //   1 / 4: local GEMM2 → this rank's rows of G   [caller: all-gather G]
  //   2: form, Sinkhorn sweeps, write, finalize (replicated); 5: tail record.
  void sphase(int k, int op) {
    GWB_CUDA(cudaSetDevice(dev_));
    switch (op) {
      case 0: GWB_CUDA(gemm_launch(s1_[(k - 1) & 1], s_)); break;
      case 1: GWB_CUDA(gemm_launch(s2_, s_)); break;
      case 2: iterate_rest(k); break;
      case 3: GWB_CUDA(gemm_launch(s1t_[k & 1], s_)); break;
      case 4: GWB_CUDA(gemm_launch(s2t_, s_)); break;
      case 5: tail_rest(k); break;
      default: api_fail(GWB_ERR_INVALID, "bregman shard: unknown phase");
    }
    GWB_CUDA(cudaGetLastError());
  }

  void load(const double* dx, const double* dy, const double* mu, const double* nu,
            const double* initial, const GraphInput* graphs) {
    const int64_t big = graphs ? n_ * m_ : std::max(std::max(n_ * n_, m_ * m_), n_ * m_);
    std::unique_ptr<void, DevFree> stage(dalloc<double>(static_cast<size_t>(big)));
    double* sp = static_cast<double*>(stage.get());
    if (graphs) {
      build_adjacency(graphs->ex, graphs->cx, n_, Dx_, ldn_, s_);
      build_adjacency(graphs->ey, graphs->cy, m_, Dy_, ldm_, s_);
    } else {
      GWB_CUDA(cudaMemcpyAsync(sp, dx, sizeof(double) * n_ * n_, cudaMemcpyHostToDevice, s_));
      launch_colmajor64_to_rowmajor32(sp, n_, n_, Dx_, ldn_, s_);
      GWB_CUDA(cudaMemcpyAsync(sp, dy, sizeof(double) * m_ * m_, cudaMemcpyHostToDevice, s_));
      launch_colmajor64_to_rowmajor32(sp, m_, m_, Dy_, ldm_, s_);
    }
    // f16x2 bound on every iterate entry: the written coupling has column
    // sums ν (the Sinkhorn scaling ends on a column update; BPG's
    // perturbation adds ≤ 1/(nm)), π₀ = μνᵀ or the caller's initial coupling.
    x_max_ = 0.0;
    for (int64_t i = 0; i < n_; ++i) x_max_ = std::max(x_max_, std::fabs(mu[i]));
    for (int64_t j = 0; j < m_; ++j) x_max_ = std::max(x_max_, std::fabs(nu[j]));
    if (initial)
      for (int64_t k = 0; k < n_ * m_; ++k) x_max_ = std::max(x_max_, std::fabs(initial[k]));
    choose_precision();
    GWB_CUDA(cudaMemcpyAsync(mu_, mu, sizeof(double) * n_, cudaMemcpyHostToDevice, s_));
    GWB_CUDA(cudaMemcpyAsync(nu_, nu, sizeof(double) * m_, cudaMemcpyHostToDevice, s_));
    if (initial) {
      GWB_CUDA(cudaMemcpyAsync(sp, initial, sizeof(double) * n_ * m_, cudaMemcpyHostToDevice, s_));
      launch_colmajor64_to_rowmajor64(sp, n_, m_, P64_[0], ldm_, s_);
    } else {
      launch_product_coupling64(mu_, nu_, n_, m_, ldm_, P64_[0], s_);
    }
    init_copies();
    GWB_CUDA(cudaStreamSynchronize(s_));
    build_plans();
  }

  // Device status reset and the hBPG phase budget (solvers.cpp:365-426).
  void begin() {
    const int budget1 = algo_ == GWB_EBPG ? cfg_.max_iters
                        : algo_ == GWB_BPG ? 0
                                           : std::min(cfg_.switch_iters, cfg_.max_iters);
    breg_reset_kernel<<<1, 1, 0, s_>>>(st_, budget1 >= 1 ? 1 : 2);
    GWB_CUDA(cudaGetLastError());
    BDev d = view(0);
    d.budget1 = budget1;
    d.has_phase2 = algo_ != GWB_EBPG;
    base_ = d;
  }

  unsigned row_ctas() const { return static_cast<unsigned>((n_ + kRowsPerCta - 1) / kRowsPerCta); }

  // Everything of outer iteration k after the chain: the form pass, ≤
  // inner_iters Sinkhorn sweeps, the write pass and the record; returns the
  // device status after the iteration.
  BState iterate_rest(int k) {
    const int q = (k - 1) & 1;
    BDev v = base_;
    rebind(v, q);
    const int rows_per_chunk = static_cast<int>((n_ + chunks_ - 1) / chunks_);
    {
      form_kernel<<<row_ctas(), kThreads, 0, s_>>>(v, 0);
      form_check_kernel<<<1, 1024, 0, s_>>>(v);
      // Large problems poll the early exit after every sweep (one host sync,
      // instead of enqueueing up to inner_iters sweeps of skipped launches).
      const bool poll = n_ * m_ >= (int64_t{1} << 23);
      for (int sw = 1; sw <= cfg_.inner_iters; ++sw) {
        row_lse_kernel<<<row_ctas(), kThreads, 0, s_>>>(v, sw);
        row_decide_kernel<<<1, 1024, 0, s_>>>(v, sw);
        dim3 grid(static_cast<unsigned>(colblocks_), static_cast<unsigned>(chunks_));
        col_lse_partial_kernel<<<grid, kThreads, 0, s_>>>(v, rows_per_chunk, sw == 1);
        col_lse_combine_kernel<<<static_cast<unsigned>((m_ + 255) / 256), 256, 0, s_>>>(v, sw == 1);
        col_flag_kernel<<<1, 1, 0, s_>>>(v, sw);
        write_kernel<<<grid, kThreads, 0, s_>>>(v, rows_per_chunk);
        sink_partial_kernel<<<static_cast<unsigned>(v.dev_rb + v.dev_cb), 256, 0, s_>>>(v);
        sink_decide_kernel<<<1, 256, 0, s_>>>(v, sw, sw == cfg_.inner_iters);
        if (poll ? sw < cfg_.inner_iters : cfg_.inner_iters > 64 && (sw % 32) == 0) {
          // Long inner loops: stop enqueueing once the device has converged.
          BState h;
          GWB_CUDA(cudaMemcpyAsync(&h, st_, sizeof(h), cudaMemcpyDeviceToHost, s_));
          GWB_CUDA(cudaStreamSynchronize(s_));
          if (h.done || h.sink_done) break;
        }
      }
      breg_finalize_kernel<<<1, 1024, 0, s_>>>(v, 0);
      GWB_CUDA(cudaGetLastError());
    }
    BState h;
    GWB_CUDA(cudaMemcpyAsync(&h, st_, sizeof(h), cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
    return h;
  }

  // Runs the whole solve (single GPU).
  void run(gwb_observer observer, void* user, std::vector<double>* host_pi) {
    begin();
    for (int k = 1; k <= cfg_.max_iters; ++k) {
      const int q = (k - 1) & 1;
      GWB_CUDA(gemm_launch(g1_[q], s_));
      GWB_CUDA(gemm_launch(g2_, s_));
      const BState h = iterate_rest(k);
      if (h.flags) break;
      // record_residual (solvers.cpp:278-280, 348-350), before the observer.
      if (cfg_.record_residual && h.iter - 1 == k) residuals_.push_back(residual_of(P64_[k & 1]));
      if (observer && h.iter - 1 == k) {
        to_host(P64_[k & 1], 1, host_pi);
        if (observer(user, k, host_pi->data(), nullptr, n_, m_) != 0)
          api_fail(GWB_ERR_RUNTIME, "observer requested abort");
      }
      if (h.done) break;
    }
  }

  const std::vector<double>& residuals() const { return residuals_; }

  BState status() {
    BState h;
    GWB_CUDA(cudaMemcpyAsync(&h, st_, sizeof(h), cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
    return h;
  }

  // Objective of the last record: one more chain on the final π.
  void tail(int used) {
    const int q = used & 1;
    GWB_CUDA(gemm_launch(g1t_[q], s_));
    GWB_CUDA(gemm_launch(g2t_, s_));
    tail_rest(used);
  }
  void tail_rest(int used) {
    BDev v = base_;
    rebind(v, used & 1);
    form_kernel<<<row_ctas(), kThreads, 0, s_>>>(v, 1);
    breg_finalize_kernel<<<1, 1024, 0, s_>>>(v, 1);
    GWB_CUDA(cudaGetLastError());
  }

  std::vector<BRecord> records(int count) {
    std::vector<BRecord> r(static_cast<size_t>(count) + 1);
    GWB_CUDA(cudaMemcpyAsync(r.data(), rec_, sizeof(BRecord) * (count + 1), cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
    return r;
  }

  // Final π to host fp64 column-major with exact fp64 column re-projection
  // onto `col_target` (the reference's last Sinkhorn step is a column scaling).
  void output(int used, double* out, const std::vector<double>& col_target) {
    std::unique_ptr<void, DevFree> o(dalloc<double>(static_cast<size_t>(n_) * m_)),
        w(dalloc<double>(std::max(n_, m_))), t(dalloc<double>(m_));
    GWB_CUDA(cudaMemcpyAsync(t.get(), col_target.data(), sizeof(double) * m_, cudaMemcpyHostToDevice, s_));
    launch_rowmajor64_to_colmajor64(P64_[used & 1], n_, m_, ldm_, static_cast<double*>(o.get()), 1,
                                    static_cast<double*>(t.get()), static_cast<double*>(w.get()), s_);
    GWB_CUDA(cudaMemcpyAsync(out, o.get(), sizeof(double) * n_ * m_, cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
  }

 private:
  template <class T>
  T* keep(T* p) {
    bufs_.push_back(p);
    return p;
  }
  // Engine buffers: stream-ordered, zero-filled, from the device pool
  // (pool_keep), so repeated solves reuse their workspace instead of paying
  // cudaMalloc of tens of GB (c4: 279 ms per solve before).
  template <class T>
  T* salloc(size_t count) {
    void* p = nullptr;
    GWB_CUDA(cudaMallocAsync(&p, count * sizeof(T) + 256, s_));
    GWB_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T) + 256, s_));
    return static_cast<T*>(p);
  }

  // fp32 hi operand (3xTF32 only) and GEMM planes of the initial iterate.
  void init_copies() {
    launch_iterate_copies(P64_[0], rows_alloc_, m_, ldm_, aux_mode_ == 2 ? P_[0] : nullptr, Pa_[0],
                          aux_mode_, aux_scale(), s_);
  }

  // luo_tseng_residual (diagnostics.cpp:33-42) of the fp64 iterate P.
  double residual_of(const double* P) {
    std::unique_ptr<void, DevFree> o(dalloc<double>(static_cast<size_t>(n_) * m_));
    double* pi64 = static_cast<double*>(o.get());
    launch_rowmajor64_to_colmajor64(P, n_, m_, ldm_, pi64, -1, nullptr, nullptr, s_);
    return luo_tseng_residual_dev(Dx_, ldn_, Dy_, ldm_, pi64, n_, m_, mu_, nu_, 1e-8, s_);
  }

  void to_host(const double* P, int, std::vector<double>* out) {
    out->resize(static_cast<size_t>(n_) * m_);
    std::unique_ptr<void, DevFree> o(dalloc<double>(static_cast<size_t>(n_) * m_));
    launch_rowmajor64_to_colmajor64(P, n_, m_, ldm_, static_cast<double*>(o.get()), -1, nullptr,
                                    nullptr, s_);
    GWB_CUDA(cudaMemcpyAsync(out->data(), o.get(), sizeof(double) * n_ * m_, cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
  }

  BDev view(int q) {
    BDev d;
    std::memset(&d, 0, sizeof(d));
    d.n = n_;
    d.m = m_;
    d.ld = ldm_;
    d.G = G_;
    d.aux_mode = aux_mode_;
    d.aux_scale = aux_scale();
    d.plane = pstride_;
    d.mu64 = mu_;
    d.nu64 = nu_;
    d.f = f_;
    d.f_new = fn_;
    d.g = g_;
    d.rowmax = rowmax_;
    d.row_sum_raw = row_sum_raw_;
    d.err_part = err_part_;
    d.col_err = col_err_;
    d.col_pm = col_pm_;
    d.col_ps = col_ps_;
    d.col_pemax = col_pe_;
    d.col_sum = col_sum_;
    d.row_sum = row_sum_;
    d.obj_part = obj_part_;
    d.wpart = wpart_;
    d.dev_part = dev_part_;
    d.dev_rb = dev_rb_;
    d.dev_cb = dev_cb_;
    d.chunks = chunks_;
    d.colblocks = colblocks_;
    d.eb_scale = 2.0 / cfg_.epsilon_reg;
    d.bp_scale = 2.0 * cfg_.step;
    d.log_domain = cfg_.log_domain;
    d.perturb = cfg_.perturbation;
    d.uniform_mass = 1.0 / (static_cast<double>(n_) * static_cast<double>(m_));
    d.max_iters = cfg_.max_iters;
    d.rel_tol = cfg_.rel_tol;
    d.inner_tol = cfg_.inner_tol;
    d.st = st_;
    d.rec = rec_;
    d.max_rec = cfg_.max_iters;
    rebind(d, q);
    return d;
  }

  void rebind(BDev& d, int q) {
    d.P = P64_[q];
    d.P_new = P64_[1 - q];
    d.P32_new = aux_mode_ == 2 ? P_[1 - q] : nullptr;
    d.P_aux_new = Pa_[1 - q];
    d.LK = LK_;
  }

  // Chain precision, as for BAPG: fp16 planes of the scaled
  // iterate against exact fp16 structure matrices (f16x2) when both are
  // 0/1-like, bf16x3 when exact in bf16 only, otherwise 3xTF32 (both
  // operands split).
  void choose_precision() {
    std::unique_ptr<void, DevFree> mx(dalloc<float>(2)), ix(dalloc<int>(2));
    float* d_max = static_cast<float*>(mx.get());
    int* d_inexact = static_cast<int*>(ix.get());
    launch_analyze(Dx_, n_, n_, ldn_, d_max, d_inexact, s_);
    launch_analyze(Dy_, m_, m_, ldm_, d_max + 1, d_inexact + 1, s_);
    int h[2];
    GWB_CUDA(cudaMemcpyAsync(h, d_inexact, sizeof(h), cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
    const bool bf16_exact = (h[0] & 2) == 0 && (h[1] & 2) == 0;
    const bool f16_exact = (h[0] & 4) == 0 && (h[1] & 4) == 0;
    const int req = cfg_.precision;
    if (f16_exact && (req == GWB_PREC_AUTO || req == GWB_PREC_F16X2))
      aux_mode_ = 5;
    else if (bf16_exact && (req == GWB_PREC_AUTO || req == GWB_PREC_BF16X3 || req == GWB_PREC_F16X2))
      aux_mode_ = 3;
    else if (bf16_exact && req == GWB_PREC_BF16X2) aux_mode_ = 4;
    else aux_mode_ = 2;
    if (aux_mode_ >= 3) {
      Dx_bf_ = keep(salloc<float>(static_cast<size_t>(n_) * ldn_ / 2 + 16));
      Dy_bf_ = keep(salloc<float>(static_cast<size_t>(m_) * ldm_ / 2 + 16));
      if (aux_mode_ == 5) {
        // f16x2 scales as in the BAPG engine.
        launch_to_f16(Dx_, n_, n_, ldn_, Dx_bf_, s_);
        launch_to_f16(Dy_, m_, m_, ldm_, Dy_bf_, s_);
        f16_s1_ = 14 - static_cast<int>(std::ceil(std::log2(std::max(x_max_, 1e-30))));
        f16_g1_rs_ = keep(salloc<float>(ldm_));
        f16_g2_cs_ = keep(salloc<float>(ldm_));
        launch_f16_scales(Dy_, m_, ldm_, static_cast<float>(x_max_), f16_s1_, f16_g1_rs_,
                          f16_g2_cs_, s_);
      } else {
        launch_to_bf16(Dx_, n_, n_, ldn_, Dx_bf_, s_);
        launch_to_bf16(Dy_, m_, m_, ldm_, Dy_bf_, s_);
      }
    } else {
      launch_tf32_aux(Dx_, n_, n_, ldn_, Dx_lo_, 2, s_);
      launch_tf32_aux(Dy_, m_, m_, ldm_, Dy_lo_, 2, s_);
    }
  }
  float aux_scale() const { return aux_mode_ == 5 ? std::ldexp(1.0f, f16_s1_) : 1.0f; }

  void build_plans() {
    if (aux_mode_ >= 3) {
      const int planes = aux_mode_ == 3 ? 3 : 2;
      auto plane_k = [](float* base, int64_t plane_elems, int k) {
        return static_cast<void*>(reinterpret_cast<uint16_t*>(base) + k * plane_elems);
      };
      auto b1 = [&](int q, const int* skip) {
        GemmDesc d;
        d.M = m_; d.N = n_; d.K = m_;
        d.bf16_planes = planes;
        d.a_bf16 = Dy_bf_; d.lda = ldm_;
        for (int k = 0; k < planes; ++k) d.b_bf16[k] = plane_k(Pa_[q], pstride_, k);
        d.ldb = ldm_;
        d.c_planes = planes;
        for (int k = 0; k < planes; ++k) d.c_bf16[k] = plane_k(Vta_, m_ * ldn_, k);
        d.ldc = ldn_;
        d.skip = skip;
        d.f16 = aux_mode_ == 5;
        if (d.f16) d.row_scale = f16_g1_rs_;
        GemmPlan* p = gemm_plan_create(d);
        plans_.push_back(p);
        return p;
      };
      auto b2 = [&](const int* skip) {
        GemmDesc d;
        d.M = n_; d.N = m_; d.K = n_;
        d.bf16_planes = planes;
        d.a_bf16 = Dx_bf_; d.lda = ldn_;
        for (int k = 0; k < planes; ++k) d.b_bf16[k] = plane_k(Vta_, m_ * ldn_, k);
        d.ldb = ldn_;
        d.c = G_; d.ldc = ldm_;
        d.skip = skip;
        d.f16 = aux_mode_ == 5;
        if (d.f16) d.col_scale = f16_g2_cs_;
        GemmPlan* p = gemm_plan_create(d);
        plans_.push_back(p);
        return p;
      };
      for (int q = 0; q < 2; ++q) {
        g1_[q] = b1(q, &st_->done);
        g1t_[q] = b1(q, &st_->flags);
      }
      g2_ = b2(&st_->done);
      g2t_ = b2(&st_->flags);
      return;
    }
    auto g1 = [&](int q, const int* skip) {
      GemmDesc d;
      d.M = m_; d.N = n_; d.K = m_;
      d.a = Dy_; d.a_lo = Dy_lo_; d.lda = ldm_;
      d.b = P_[q]; d.b_lo = Pa_[q]; d.ldb = ldm_;
      d.c = Vt_; d.c_aux = Vta_; d.ldc = ldn_; d.aux_mode = 2;
      d.skip = skip;
      d.three_pass = true;
      GemmPlan* p = gemm_plan_create(d);
      plans_.push_back(p);
      return p;
    };
    auto g2 = [&](const int* skip) {
      GemmDesc d;
      d.M = n_; d.N = m_; d.K = n_;
      d.a = Dx_; d.a_lo = Dx_lo_; d.lda = ldn_;
      d.b = Vt_; d.b_lo = Vta_; d.ldb = ldn_;
      d.c = G_; d.ldc = ldm_;
      d.skip = skip;
      d.three_pass = true;
      GemmPlan* p = gemm_plan_create(d);
      plans_.push_back(p);
      return p;
    };
    for (int q = 0; q < 2; ++q) {
      g1_[q] = g1(q, &st_->done);
      g1t_[q] = g1(q, &st_->flags);
    }
    g2_ = g2(&st_->done);
    g2t_ = g2(&st_->flags);
  }

  void* slot(int p, int r) const {
    return vt_ + ((static_cast<int64_t>(r) * planes_ + p) * m_ * nr_) * esize_;
  }

  // Local chain plans (as ShardEngine, csrc/shard.cu): GEMM1 on this rank's
  // rows of π into its Vᵀ slot, GEMM2 of its D_X rows against the gathered
  // blocked-K Vᵀ into its rows of G.
  void build_shard_plans() {
    const bool bf = aux_mode_ >= 3;
    auto make1 = [&](int q, const int* skip) {
      GemmDesc d;
      d.M = m_; d.N = nr_; d.K = m_;
      d.lda = ldm_; d.ldb = ldm_; d.ldc = nr_;
      d.skip = skip;
      if (bf) {
        d.bf16_planes = planes_;
        d.a_bf16 = Dy_bf_;
        for (int p = 0; p < planes_; ++p)
          d.b_bf16[p] = reinterpret_cast<uint16_t*>(Pa_[q]) + p * pstride_ + row0_ * ldm_;
        d.c_planes = planes_;
        for (int p = 0; p < planes_; ++p) d.c_bf16[p] = slot(p, rank_);
        d.f16 = aux_mode_ == 5;
        if (d.f16) d.row_scale = f16_g1_rs_;
      } else {
        d.a = Dy_; d.a_lo = Dy_lo_;
        d.b = P_[q] + row0_ * ldm_; d.b_lo = Pa_[q] + row0_ * ldm_;
        d.c = static_cast<float*>(slot(0, rank_));
        d.c_aux = static_cast<float*>(slot(1, rank_));
        d.aux_mode = 2;
        d.three_pass = true;
      }
      GemmPlan* p = gemm_plan_create(d);
      plans_.push_back(p);
      return p;
    };
    auto make2 = [&](const int* skip) {
      GemmDesc d;
      d.M = nr_; d.N = m_; d.K = npad_;
      d.lda = ldk_;
      d.b_block_k = nr_;
      d.b_block_stride = static_cast<int64_t>(planes_) * m_ * nr_;
      d.c = G_ + row0_ * ldm_; d.ldc = ldm_;
      d.skip = skip;
      if (bf) {
        d.bf16_planes = planes_;
        d.a_bf16 = Dx_bf_;
        for (int p = 0; p < planes_; ++p) d.b_bf16[p] = slot(p, 0);
        d.f16 = aux_mode_ == 5;
        if (d.f16) d.col_scale = f16_g2_cs_;
      } else {
        d.a = Dx_; d.a_lo = Dx_lo_;
        d.b = static_cast<const float*>(slot(0, 0));
        d.b_lo = static_cast<const float*>(slot(1, 0));
        d.three_pass = true;
      }
      GemmPlan* p = gemm_plan_create(d);
      plans_.push_back(p);
      return p;
    };
    for (int q = 0; q < 2; ++q) {
      s1_[q] = make1(q, &st_->done);
      s1t_[q] = make1(q, &st_->flags);
    }
    s2_ = make2(&st_->done);
    s2t_ = make2(&st_->flags);
  }

  int dev_;
  int64_t n_, m_, ldn_, ldm_;
  gwb_config cfg_;
  int algo_;
  bool own_stream_ = false;
  bool sharded_ = false;
  int world_ = 1, rank_ = 0, planes_ = 3, esize_ = 2;
  int64_t nr_ = 0, npad_ = 0, row0_ = 0, rows_valid_ = 0, ldk_ = 0, rows_alloc_ = 0, pstride_ = 0;
  uint8_t* vt_ = nullptr;
  GemmPlan *s1_[2] = {nullptr, nullptr}, *s1t_[2] = {nullptr, nullptr}, *s2_ = nullptr,
           *s2t_ = nullptr;
  cudaStream_t s_ = nullptr;
  std::vector<void*> bufs_;
  std::vector<GemmPlan*> plans_;
  float *Dx_, *Dy_, *Dx_lo_, *Dy_lo_, *P_[2], *Pa_[2], *Vt_, *Vta_, *G_;
  double *P64_[2] = {nullptr, nullptr}, *LK_ = nullptr, *rowmax_ = nullptr;
  float* Dx_bf_ = nullptr;
  float* Dy_bf_ = nullptr;
  int aux_mode_ = 2;
  double x_max_ = 1.0;  // f16x2: bound on every iterate entry
  int f16_s1_ = 0;
  float* f16_g1_rs_ = nullptr;
  float* f16_g2_cs_ = nullptr;
  double *mu_, *nu_, *f_, *fn_, *g_, *row_sum_raw_, *err_part_, *col_err_, *col_pm_, *col_ps_, *col_sum_,
      *row_sum_, *obj_part_, *wpart_, *dev_part_;
  float* col_pe_;
  int chunks_ = 1, colblocks_ = 1, dev_rb_ = 1, dev_cb_ = 1;
  BState* st_;
  BRecord* rec_;
  BDev base_;
  std::vector<double> residuals_;
  GemmPlan *g1_[2], *g1t_[2], *g2_, *g2t_;
};

// Error precedence and wrapping of ebpg_solve / bpg_solve (solvers.cpp:246-261,
// :312-336): eBPG rethrows only ZeroSumLineError; BPG wraps both.
void raise_breg(const BState& s, bool log_domain) {
  const int it = s.err_iter;
  const bool bpg_phase = s.phase == 2;
  const char* solver = bpg_phase ? "bpg" : "ebpg";
  char detail[400];
  if (s.flags & kBOverflow) api_numerical("bpg", it, "exp overflow; reduce step");
  if (s.flags & kBDeadLine)
    api_numerical("ebpg", it,
                  "kernel line underflowed to zero; increase eps or enable the log-domain solver");
  if (s.flags & (kBZeroRow | kBZeroCol)) {
    std::snprintf(detail, sizeof(detail), "%s %d has nonpositive sum; cannot rescale",
                  (s.flags & kBZeroRow) ? "row" : "column", s.zero_index);
    api_numerical(solver, it, detail);
  }
  // non-finite entries after a sweep (projections.cpp:104-107 / 151-154)
  const bool logd = !bpg_phase && log_domain;
  std::snprintf(detail, sizeof(detail),
                "numerical instability in %s at iteration %d: non-finite entries after scaling sweep",
                logd ? "sinkhorn-log" : "sinkhorn", s.err_sweep);
  if (bpg_phase) api_numerical("bpg", it, detail);
  api_numerical(logd ? "sinkhorn-log" : "sinkhorn", s.err_sweep,
                "non-finite entries after scaling sweep");
}

}  // namespace

void bregman_solve(const gwb_config* cfg, int32_t algo, const double* dx, int64_t n,
                   const double* dy, int64_t m, const double* mu, const double* nu,
                   const double* initial, gwb_observer observer, void* user, double* out_final,
                   gwb_record* trace, int32_t trace_cap, int32_t* n_records, int32_t* converged,
                   int32_t* iterations_used, const GraphInput* graphs) {
  if (trace && trace_cap < cfg->max_iters) api_fail(GWB_ERR_CAPACITY, "trace capacity < max_iters");
  if (initial) {
    const size_t len = static_cast<size_t>(n) * m;
    for (size_t k = 0; k < len; ++k)
      if (!(initial[k] >= 0.0) || !std::isfinite(initial[k]))
        api_fail(GWB_ERR_INVALID, "initial coupling must be finite and nonnegative");
  }
  const int device = api_device();
  // BPG step-size warning (solvers.cpp:226-234), only if a BPG phase can run.
  const bool bpg_may_run =
      algo == GWB_BPG || (algo == GWB_HBPG && cfg->max_iters >= 1);
  // GWB_PHASE_TIMES=1: wall time of each phase of the call on stderr.
  static const bool phase_times = std::getenv("GWB_PHASE_TIMES") != nullptr;
  auto tick = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!phase_times) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "bregman phase %-9s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - tick).count());
    tick = now;
  };
  BregmanEngine eng(device, n, m, *cfg, algo);
  lap("create");
  eng.load(dx, dy, mu, nu, initial, graphs);
  lap("load");
  std::vector<double> host_pi;
  eng.run(observer, user, &host_pi);
  lap("run");
  const BState s = eng.status();
  if (s.flags) raise_breg(s, cfg->log_domain != 0);
  const int used = s.iter - 1;
  if (bpg_may_run && (algo == GWB_BPG || s.used1 < used || s.phase == 2) && !cfg->quiet) {
    const double lip = graphs ? device_lipschitz_bound_graphs(*graphs, n, m)
                              : device_lipschitz_bound(dx, n, dy, m);
    if (lip > 0.0 && cfg->step > 1.0 / lip)
      std::fprintf(stderr,
                   "bpg: step %g exceeds sigma/L_f = %g; descent is not guaranteed at this step "
                   "size\n",
                   cfg->step, 1.0 / lip);
  }
  eng.tail(used);
  const std::vector<BRecord> r = eng.records(used);
  if (trace) {
    for (int k = 1; k <= used; ++k) {
      gwb_record& o = trace[k - 1];
      std::memset(&o, 0, sizeof(o));
      o.iter = k;
      o.objective = -r[k].obj;
      o.marginal_infeasibility = r[k].infeas;
      o.rel_change = r[k].rel;
      o.elapsed_seconds = r[k].elapsed;
      o.phase = algo == GWB_HBPG ? r[k].phase : 0;
      if (k <= static_cast<int>(eng.residuals().size())) {
        o.residual = eng.residuals()[k - 1];
        o.has_residual = 1;
      }
    }
  }
  if (n_records) *n_records = trace ? used : 0;
  if (converged) *converged = s.converged;
  if (iterations_used) *iterations_used = used;
  // Column sums of the returned coupling: ν after a Sinkhorn column step, or
  // (1−p)ν + p/m after a perturbed BPG step.
  const bool last_bpg = used >= 1 && r[used].phase == 2;
  const double p = last_bpg ? cfg->perturbation : 0.0;
  std::vector<double> target(m);
  for (int64_t j = 0; j < m; ++j) target[j] = (1.0 - p) * nu[j] + p / static_cast<double>(m);
  lap("tail");
  eng.output(used, out_final, target);
  lap("output");
}

// ---- row-sharded eBPG / BPG / hBPG (C-ABI in capi.cu) ---------
struct BregShard {
  std::unique_ptr<BregmanEngine> eng;
  gwb_config cfg;
  int algo;
  std::vector<double> nu;
};

BregShard* bshard_create(const gwb_config& cfg, int algo, int64_t n, int64_t m, int world, int rank,
                         int device, cudaStream_t s) {
  auto* b = new BregShard();
  b->cfg = cfg;
  b->algo = algo;
  b->eng.reset(new BregmanEngine(device, n, m, cfg, algo, world, rank, s));
  return b;
}
void bshard_destroy(BregShard* b) { delete b; }
void bshard_layout(BregShard* b, int64_t* rows_per_shard, int64_t* row_begin, int64_t* rows_valid,
                   int64_t* padded_rows, int64_t* ld) {
  *rows_per_shard = b->eng->rows_per_shard();
  *row_begin = b->eng->row_begin();
  *rows_valid = b->eng->rows_valid();
  *padded_rows = b->eng->padded_rows();
  *ld = b->eng->ld();
}
void bshard_comm_layout(BregShard* b, int32_t* planes, int32_t* esize, int64_t* vt_bytes) {
  *planes = b->eng->planes();
  *esize = b->eng->esize();
  *vt_bytes = b->eng->vt_bytes();
}
void bshard_set_comm(BregShard* b, void* vt, float* g) { b->eng->set_comm(vt, g); }
void bshard_load(BregShard* b, const float* dx_rows, int64_t ldx, const float* dy, int64_t ldy,
                 const double* mu, const double* nu, int64_t m) {
  b->nu.assign(nu, nu + m);
  b->eng->load_sharded(dx_rows, ldx, dy, ldy, mu, nu);
}
void bshard_phase(BregShard* b, int k, int op) { b->eng->sphase(k, op); }
void bshard_status(BregShard* b, int32_t* done, int32_t* iter, int32_t* flags, int32_t* converged) {
  const BState h = b->eng->status();
  *done = h.done;
  *iter = h.iter;
  *flags = h.flags;
  *converged = h.converged;
}
void* bshard_stream(BregShard* b) { return b->eng->stream(); }

// After the schedule (and, without flags, the tail ops 3–5): the reference
// errors, records, convergence and the final coupling, as bregman_solve.
void bshard_finish(BregShard* b, double* out_final, gwb_record* trace, int32_t trace_cap,
                   int32_t* n_records, int32_t* converged, int32_t* iterations_used) {
  BregmanEngine& eng = *b->eng;
  const BState s = eng.status();
  if (s.flags) raise_breg(s, b->cfg.log_domain != 0);
  const int used = s.iter - 1;
  if (trace && trace_cap < used) api_fail(GWB_ERR_CAPACITY, "trace capacity < iterations used");
  const std::vector<BRecord> r = eng.records(used);
  if (trace) {
    for (int k = 1; k <= used; ++k) {
      gwb_record& o = trace[k - 1];
      std::memset(&o, 0, sizeof(o));
      o.iter = k;
      o.objective = -r[k].obj;
      o.marginal_infeasibility = r[k].infeas;
      o.rel_change = r[k].rel;
      o.elapsed_seconds = r[k].elapsed;
      o.phase = b->algo == GWB_HBPG ? r[k].phase : 0;
    }
  }
  if (n_records) *n_records = trace ? used : 0;
  if (converged) *converged = s.converged;
  if (iterations_used) *iterations_used = used;
  if (out_final) {
    const int64_t m = static_cast<int64_t>(b->nu.size());
    const bool last_bpg = used >= 1 && r[used].phase == 2;
    const double p = last_bpg ? b->cfg.perturbation : 0.0;
    std::vector<double> target(m);
    for (int64_t j = 0; j < m; ++j) target[j] = (1.0 - p) * b->nu[j] + p / static_cast<double>(m);
    eng.output(used, out_final, target);
  }
}

}  // namespace gwb
