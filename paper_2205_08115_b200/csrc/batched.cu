// batched.cu — config 5: many independent small BAPG problems (n, m ≤ 128),
// one CTA per problem, every iteration on-chip.
//
// The reference runs such a batch as independent gw::solve calls from its
// experiment worker pool (experiment.cpp:273-304); each problem follows
// bapg_solve (solvers.cpp:138-217).  Here a persistent CTA owns one problem
// at a time.  The two half-steps run in opposite orientations, so every
// line reduction (row sums in a, column sums in b) is a per-thread loop and
// no shuffle transposes are needed:
//   half-step a (lane = row i):    G  = (D_X·X)·D_Y      X = w
//   half-step b (lane = column j): Gᵀ = D_Y·(D_X·X)ᵀ     X = π
// The operand planes are written by the lane that owns the line — w by
// column (K-major B operand), π by row (MN-major B operand) — and the
// iterates cross between the orientations through one fp32 buffer T[i][j]
// that every thread reads and overwrites along its own line.
//   SMEM  D_X, D_Y as fp16 (exact for 0/1 / small-integer D; 32 KB each,
//         128-B swizzled K-major; D symmetric, so the D_Y tile is both
//         GEMM2's B and GEMM2ᵀ's A); two fp16 planes (hi, lo) of the current
//         GEMM operand (X, then V = D_X·X) with power-of-two scales (f16x2,
//         DESIGN.md §4); T (fp32 128×132); reduction scratch, marginals.
//   TMEM  accumulator · wᵀ · πᵀ (the unnormalised kernel t stays in
//         registers: TMEM→register reads, 64 B/clk per SM, are the scarce
//         resource, so each half-step reads its accumulator once).
// The fp64 diagnostics, trace record and stop rule are evaluated by the
// CTA; nothing leaves the SM until the problem finishes.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "devutil.cuh"
#include "kernels.cuh"
#include "ptx.cuh"
#include "solver.cuh"
#include "standalone.cuh"
#include "../../include/gwb_ext.h"

namespace gwb {

namespace {

using namespace dev;

double g_last_ms = 0.0;       // gwb_batched_last_kernel_ms
int64_t g_last_problems = 0;

constexpr int kT = 128;                         // padded problem side
constexpr int kW = 64;                          // cross-line entries per thread
constexpr int kH = kT / kW;                     // threads per line (2)
constexpr int kThreads = 128 * kH;              // 8 warps: 4 lane quadrants × 2 column halves
// (16 warps with 32 entries each measured 9% slower: the FP32 pipes, not
// latency, bound the SIMT phases.)
constexpr uint32_t kTileBytes = kT * kT * 2;    // one fp16 operand plane (32 KB)
constexpr uint32_t kHalfTile = kTileBytes / 2;  // one 64-wide K chunk (16 KB)
constexpr int kTLd = kT + 4;                    // T row pitch (floats): conflict-free rows and columns
constexpr uint32_t kAcc = 0, kWT = 128, kPT = 256;  // TMEM columns (256 used of 512)
constexpr size_t kScratch = 12 * 1024;
constexpr size_t kSmem = 1024 + 4 * static_cast<size_t>(kTileBytes) +
                         static_cast<size_t>(kT) * kTLd * 4 + kScratch;

struct BatchStatus {
  int flags, err_iter, zero_index, used, converged, pad[3];
};

struct BatchArgs {
  const uint8_t* dpack;  // [batch][2][32 KB] pre-swizzled fp16: D_X, D_Y
  const double* mu;      // [batch][128], zero padded
  const double* nu;
  const int* scl;        // [batch] s: iterates, X and V planes are held ×2^s
  float* P;              // [batch][128][128] final π
  float* W;              // [batch][128][128] final w
  DevRecord* rec;        // [batch][max_iters + 2] or null
  BatchStatus* st;
  int* next;             // problem counter (zeroed per launch): dynamic scheduling
  int batch, n, m, max_iters;
  float inv_rho;
  double rel_tol;
};

// Byte offset of fp16 element (row, k) in a 128×128 K-major operand stored
// as two 64-wide K chunks, each the canonical 128-B swizzle layout.
__host__ __device__ __forceinline__ uint32_t sw_off(int row, int k) {
  return static_cast<uint32_t>(k >> 6) * kHalfTile + static_cast<uint32_t>(row) * 128u +
         ((static_cast<uint32_t>((k >> 3) & 7) ^ static_cast<uint32_t>(row & 7)) << 4) +
         (static_cast<uint32_t>(k & 7) << 1);
}

// Two fp32 values (already in fp16 range) → hi and lo fp16x2 planes,
// hi = rn(x), lo = rn(x − hi) (22-bit operand, DESIGN.md §4 f16x2).
__device__ __forceinline__ void split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hi) : "f"(b), "f"(a));
  const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hi));
  const float ra = a - hf.x, rb = b - hf.y;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(lo) : "f"(rb), "f"(ra));
}

// Operand packing: fp64 column-major inputs → fp16 swizzled tiles, the
// fp16-exactness check, zero-padded fp64 marginals and the power-of-two
// scale s = 14 − ⌈log2(x_max · max(1, max_i Σ_k |D_X[i][k]|))⌉: x_max =
// max(max μ, max ν) bounds every iterate entry (π_kl ≤ μ_k, w_kl ≤ ν_l) and
// x_max·Σ_k|D_X[i][k]| every entry of V = D_X·X, so X·2^s and V·2^s both
// stay inside fp16's range and GEMM1's accumulator is V's operand as is.
__global__ void batched_pack_kernel(const double* __restrict__ dx, const double* __restrict__ dy,
                                    const double* __restrict__ mu, const double* __restrict__ nu,
                                    int n, int m, uint8_t* __restrict__ dpack,
                                    double* __restrict__ mu_p, double* __restrict__ nu_p,
                                    int* __restrict__ scl, int* inexact) {
  const int64_t b = blockIdx.x;
  const int op = blockIdx.y;  // 0: D_X, 1: D_Y
  const int dim = op == 0 ? n : m;
  const double* src = (op == 0 ? dx : dy) + b * static_cast<int64_t>(dim) * dim;
  __half* dst = reinterpret_cast<__half*>(dpack + (b * 2 + op) * static_cast<int64_t>(kTileBytes));
  bool bad = false;
  for (int idx = threadIdx.x; idx < kT * kT; idx += blockDim.x) {
    // idx = c·128 + r walks the column-major source contiguously.
    const int c = idx / kT, r = idx % kT;
    double v = 0.0;
    if (r < dim && c < dim) v = src[static_cast<int64_t>(c) * dim + r];
    const __half hv = __double2half(v);
    if (static_cast<double>(__half2float(hv)) != v) bad = true;
    dst[sw_off(r, c) / 2] = hv;
  }
  if (bad) atomicOr(inexact, 1);
  if (op != 0) return;
  __shared__ double s_deg[kT], s_x[kT];
  const int t = threadIdx.x;
  if (t < kT) {
    double deg = 0.0;
    if (t < n)
      for (int c = 0; c < n; ++c) deg += fabs(src[static_cast<int64_t>(c) * n + t]);
    s_deg[t] = deg;
    const double a = t < n ? mu[b * n + t] : 0.0;
    const double w = t < m ? nu[b * m + t] : 0.0;
    mu_p[b * kT + t] = a;
    nu_p[b * kT + t] = w;
    s_x[t] = fmax(fabs(a), fabs(w));
  }
  __syncthreads();
  if (t == 0) {
    double deg = 1.0, x = 0.0;
    for (int k = 0; k < kT; ++k) {
      deg = fmax(deg, s_deg[k]);
      x = fmax(x, s_x[k]);
    }
    const double vb = x * deg;
    const int sv = vb > 0.0 ? 14 - static_cast<int>(ceil(log2(vb))) : 0;
    scl[b] = max(-100, min(100, sv));
  }
}

// UMMA descriptor of GEMM1's B operand π[k = i][n = j] stored row-major in
// the same swizzled tiles as sw_off(i, j): MN-major, 64-wide N blocks
// LBO = 16 KB apart, 8-row K groups SBO = 1024 B apart, 128-B swizzle.
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(kHalfTile >> 4) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Line sums of a thread's kW fp32 terms as 8-term fp32 partials added in
// fp64 (short independent chains; the normalisers and record sums keep
// ~1e-7 relative accuracy instead of a long fp32 chain's).  f(t) is the term.
template <class F>
__device__ __forceinline__ double sumw(F f) {
  constexpr int G = kW / 8;
  float p[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    p[g] = f(8 * g);
#pragma unroll
    for (int u = 1; u < 8; ++u) p[g] += f(8 * g + u);
  }
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < G; ++g) s += static_cast<double>(p[g]);
  return s;
}
// Σ a_t·b_t the same way, as fused multiply-adds.
template <class FA, class FB>
__device__ __forceinline__ double dotw(FA fa, FB fb) {
  constexpr int G = kW / 8;
  float p[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    p[g] = fa(8 * g) * fb(8 * g);
#pragma unroll
    for (int u = 1; u < 8; ++u) p[g] = fmaf(fa(8 * g + u), fb(8 * g + u), p[g]);
  }
  double s = 0.0;
#pragma unroll
  for (int g = 0; g < G; ++g) s += static_cast<double>(p[g]);
  return s;
}

__global__ void __launch_bounds__(kThreads, 1) bapg_batched_kernel(BatchArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sD = smem;                                                // D_X | D_Y
  uint8_t* sPl = smem + 2 * kTileBytes;                              // hi | lo planes
  float* T = reinterpret_cast<float*>(sPl + 2 * kTileBytes);         // [128][kTLd]
  float* red_m = T + kT * kTLd;                                      // [kH][128] line maxima
  double* red_d = reinterpret_cast<double*>(red_m + kH * kT);        // [3][kH][128] line sums
  double* diag = red_d + 3 * kH * kT;                                // [16][8]
  double* s_mu = diag + 8 * (kThreads / 32);                         // [128]
  double* s_nu = s_mu + kT;                                          // [128]
  int* ctl = reinterpret_cast<int*>(s_nu + kT);                      // flags, zero_index, stop
  uint64_t* bars = reinterpret_cast<uint64_t*>(ctl + 8);             // load, mma
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2;
  const int L = q * 32 + lane;  // line owned: row i (half-step a) or column j (b); TMEM lane
  const int c0 = h * kW;        // first of the kW cross-line entries owned
  const int n = a.n, m = a.m;
  const float inv_rho = a.inv_rho;

  if (warp == 0) ptx::tmem_alloc<256>(tmem_slot);
  if (tid == 0) {
    ptx::mbar_init(&bars[0], 1);
    ptx::mbar_init(&bars[1], 1);
    ptx::fence_barrier_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const uint32_t tl = tbase + (static_cast<uint32_t>(q * 32) << 16);  // this warp's lanes
  const uint32_t sD_a = ptx::smem_u32(sD), sPl_a = ptx::smem_u32(sPl);
  uint32_t load_ph = 0, mma_ph = 0;
  // Operand row L, k-chunks of this thread's entries: sw_off(L, c0 + 8c) =
  // (c0 / 64)·16 KB + 128·L + (((c0 / 8 + c) & 7) ^ (L & 7)) << 4.
  uint8_t* const pl_row = sPl + (c0 >> 6) * kHalfTile + L * 128;
  const int xg = ((c0 >> 3) & 7) ^ (L & 7);

  // kW columns of this warp's lanes from / to TMEM, 32 columns per access.
  auto ldw = [&](uint32_t col, float (&v)[kW]) {
    uint32_t r[kW];
#pragma unroll
    for (int c = 0; c < kW; c += 32) ptx::tmem_ld_32x32b_x32(tl + col + c, *reinterpret_cast<uint32_t(*)[32]>(r + c));
    ptx::tmem_wait_ld();
#pragma unroll
    for (int t = 0; t < kW; ++t) v[t] = __uint_as_float(r[t]);
  };
  auto st = [&](uint32_t col, const float (&v)[kW]) {
#pragma unroll
    for (int c = 0; c < kW; c += 32) {
      uint32_t r[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) r[t] = __float_as_uint(v[c + t]);
      ptx::tmem_st_32x32b_x32(tl + col + c, r);
    }
  };
  // This thread's entries [c0, c0 + kW) of line L (scaled units, inside fp16
  // range) as the two fp16 planes of operand row L.
  auto store_planes = [&](const float (&v)[kW]) {
#pragma unroll
    for (int c8 = 0; c8 < kW / 8; ++c8) {
      uint32_t hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) split_f16x2(v[c8 * 8 + 2 * e], v[c8 * 8 + 2 * e + 1], hi[e], lo[e]);
      uint8_t* p = pl_row + ((xg ^ c8) << 4);
      *reinterpret_cast<uint4*>(p) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<uint4*>(p + kTileBytes) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
  };
  // MMA issue (one thread).  GEMM1: V = D_X·X, B = X planes, K-major (X = w,
  // written by columns) or MN-major (X = π, written by rows).  GEMM2: G =
  // V·D_Y (A = V planes, B = D_Y) or Gᵀ = D_Y·Vᵀ (A = D_Y, B = V planes).
  // Smallest plane first into one accumulator: the accumulator's truncation
  // acts on the hi-plane terms only.
  auto issue = [&](int kind) {  // 0: GEMM1 K-major X, 1: GEMM1 MN-major X, 2: G, 3: Gᵀ
    ptx::tc_fence_after();
    const uint32_t idesc = ptx::idesc_f16(128, 128) | (kind == 1 ? (1u << 16) : 0u);
#pragma unroll 1
    for (int pi = 0; pi < 2; ++pi) {
      const uint32_t pl = sPl_a + (1 - pi) * kTileBytes;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // K = 128 in steps of 16
        const uint32_t koff = (kk >> 2) * kHalfTile + (kk & 3) * 32;
        uint64_t ad, bd;
        if (kind <= 1) {
          ad = ptx::umma_desc_sw128(sD_a + koff);
          bd = kind == 1 ? desc_mn(pl + kk * 2048) : ptx::umma_desc_sw128(pl + koff);
        } else if (kind == 2) {
          ad = ptx::umma_desc_sw128(pl + koff);
          bd = ptx::umma_desc_sw128(sD_a + kTileBytes + koff);
        } else {
          ad = ptx::umma_desc_sw128(sD_a + kTileBytes + koff);
          bd = ptx::umma_desc_sw128(pl + koff);
        }
        ptx::mma_bf16(tbase + kAcc, ad, bd, idesc, (pi || kk) ? 1u : 0u);
      }
    }
    ptx::mma_commit(&bars[1]);
  };
  auto mma_sync = [&]() {
    ptx::mbar_wait(&bars[1], mma_ph);
    mma_ph ^= 1;
    ptx::tc_fence_after();
  };
  // Block sum of up to 8 doubles per thread (fixed order); result on thread 0.
  auto block_sum8 = [&](double (&v)[8], int cnt) {
    for (int k = 0; k < cnt; ++k) {
      const double s = warp_sum(v[k]);
      if (lane == 0) diag[warp * 8 + k] = s;
    }
    __syncthreads();
    if (tid == 0)
      for (int k = 0; k < cnt; ++k) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += diag[w * 8 + k];
        v[k] = s;
      }
    __syncthreads();
  };
  // Line max over the kH threads of a line, in order.
  auto line_max = [&](float v) {
    red_m[h * kT + L] = v;
    __syncthreads();
    float r = red_m[L];
#pragma unroll
    for (int hh = 1; hh < kH; ++hh) r = fmaxf(r, red_m[hh * kT + L]);
    return r;
  };
  // Line sum of slot `k` of red_d over the kH threads, in order.
  auto line_sum = [&](int k) {
    double r = red_d[(k * kH) * kT + L];
#pragma unroll
    for (int hh = 1; hh < kH; ++hh) r += red_d[(k * kH + hh) * kT + L];
    return r;
  };

  // Zero padding (lines ≥ n / m, D beyond its side) keeps every padded entry
  // at 0 through the updates: G ≥ 0 there is never above a true maximum,
  // t = 0·e^{≤0} = 0, and the padded scales are forced to 0.
  // Dynamic scheduling: a CTA takes the next problem when it finishes one
  // (problems stop at the reference's rule after 149-500 iterations; a static
  // round-robin left the busiest SM ~15% above the mean).  Results do not
  // depend on which SM solves a problem.
  __shared__ int s_next;
  for (;;) {
    if (tid == 0) s_next = atomicAdd(a.next, 1);
    __syncthreads();
    const int b = s_next;
    if (b >= a.batch) break;
    DevRecord* rec = a.rec ? a.rec + static_cast<int64_t>(b) * (a.max_iters + 2) : nullptr;
    if (tid == 0) {
      ptx::mbar_arrive_expect_tx(&bars[0], 2 * kTileBytes);
      const uint8_t* src = a.dpack + static_cast<int64_t>(b) * 2 * kTileBytes;
      ptx::bulk_g2s(sD, src, kTileBytes, &bars[0]);
      ptx::bulk_g2s(sD + kTileBytes, src + kTileBytes, kTileBytes, &bars[0]);
      ctl[0] = 0;
      ctl[1] = 0x7fffffff;
      ctl[2] = 0;
    }
    if (tid < kT) {
      s_mu[tid] = a.mu[static_cast<int64_t>(b) * kT + tid];
      s_nu[tid] = a.nu[static_cast<int64_t>(b) * kT + tid];
    }
    // Scaled units: π̂ = π·2^s, ŵ = w·2^s (exact), so GEMM1's accumulator is
    // V̂ = V·2^s and GEMM2's 2^s·G; every record sum is rescaled in fp64.
    const int sc = a.scl[b];
    const float up = ldexpf(1.0f, sc);
    const double un64 = ldexp(1.0, -sc), un2_64 = ldexp(1.0, -2 * sc);
    const float g_true = ldexpf(1.0f, -sc) * inv_rho;  // raw accumulator → G/ρ
    // exp(G/ρ − r) = 2^(acc·k2 − r·k2), k2 = 2^−s/ρ·log2 e.
    const float k2 = g_true * 1.4426950408889634f;
    const unsigned long long t0 = globaltimer();
    __syncthreads();
    // TMEM reads are the scarce resource (64 B/clk per SM): each half-step
    // reads its accumulator once into registers (x = this thread's entries
    // [c0, c0 + kW) of its line) and keeps the kernel t there.
    float x[kW];
    // ŵ⁰ = (μνᵀ)·2^s in fp32 (product_coupling_kernel), held column-wise
    // (lane j = L): TMEM wᵀ, T[i][j] and the K-major planes of GEMM1's B.
    {
      const float nu_j = static_cast<float>(s_nu[L]);
#pragma unroll
      for (int t = 0; t < kW; ++t) {
        x[t] = (static_cast<float>(s_mu[c0 + t]) * up) * nu_j;
        T[(c0 + t) * kTLd + L] = x[t];
      }
      st(kWT + c0, x);
      store_planes(x);
      ptx::tmem_wait_st();
    }
    ptx::mbar_wait(&bars[0], load_ph);
    load_ph ^= 1;

    auto load_acc = [&]() { ldw(kAcc + c0, x); };
    auto acc_max = [&]() {
      float m4[4] = {0.f, 0.f, 0.f, 0.f};  // G ≥ 0
#pragma unroll
      for (int t = 0; t < kW; ++t) m4[t & 3] = fmaxf(m4[t & 3], x[t]);
      return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    };

    int k = 1, phase = 0, used = 0, converged = 0, err_iter = 0;
    // GEMM1 of the first chain (X̂ = ŵ⁰).  Every later chain's GEMM1 is
    // issued at the end of the preceding half-step, as soon as its operand
    // planes are written, so its MMAs run under that half-step's record sums.
    ptx::fence_proxy_async();
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) issue(0);
    for (;;) {
      // ---- chain: V̂ = D_X·X̂ → planes → G (a) or Gᵀ (b), ×2^s, in kAcc.
      mma_sync();
      load_acc();
      store_planes(x);
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      __syncthreads();
      if (tid == 0) issue(phase == 1 ? 3 : 2);
      // While GEMM2 runs: the current iterate's entries of line L from T
      // (ŵ by rows for a / the tail, π̂ by columns for b) and their sum.
      float xo[kW];
      if (phase != 1) {
        const float* Trow = T + L * kTLd + c0;
#pragma unroll
        for (int t = 0; t < kW; t += 4) {
          const float4 w4 = *reinterpret_cast<const float4*>(Trow + t);
          xo[t] = w4.x;
          xo[t + 1] = w4.y;
          xo[t + 2] = w4.z;
          xo[t + 3] = w4.w;
        }
      } else {
#pragma unroll
        for (int t = 0; t < kW; ++t) xo[t] = T[(c0 + t) * kTLd + L];
      }
      const double xo_sum = sumw([&](int t) { return xo[t]; });
      mma_sync();
      load_acc();  // x = 2^s·G (row L) or 2^s·Gᵀ (column L)

      if (phase != 1) {
        // ---- half-step a (phase 0) / tail (phase 2), lane = row i = L ----
        const bool row_ok = L < n;
        const float rmax = line_max(acc_max());
        const float rr = rmax * k2;
        // t̂ = ŵ ⊙ e^{G/ρ − r} (into x), Ŝ = Σ_j t̂; ⟨G, w⟩ and Σ_j w for the
        // previous record.  ŵ is row L of T.
        float* Trow = T + L * kTLd + c0;
        const float (&wv)[kW] = xo;
        const double gw = dotw([&](int t) { return x[t]; }, [&](int t) { return wv[t]; });
        const double rw = xo_sum;
#pragma unroll
        for (int t = 0; t < kW; ++t) x[t] = wv[t] * ex2(fmaf(x[t], k2, -rr));
        const double S = sumw([&](int t) { return x[t]; });
        red_d[(0 * kH + h) * kT + L] = S;
        red_d[(1 * kH + h) * kT + L] = gw;
        red_d[(2 * kH + h) * kT + L] = rw;
        __syncthreads();
        double ra[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (h == 0 && row_ok) {
          ra[0] = line_sum(1) * un2_64;
          const double dv = line_sum(2) * un64 - s_mu[L];
          ra[1] = dv * dv;
        }
        if (phase == 0) {
          const double St = line_sum(0);
          if (h == 0 && row_ok) {
            if (rmax * g_true > 700.0f) atomicOr(&ctl[0], kFlagOverflowA);
            if (!(St > 0.0) || !isfinite(St) || isnan(rmax)) {
              atomicOr(&ctl[0], kFlagZeroA);
              atomicMin(&ctl[1], L);
            }
          }
          // π̂ = t̂ · μ_i 2^s / Ŝ: row i of T and the MN-major planes of GEMM1's B.
          const float scale = row_ok ? static_cast<float>(s_mu[L] * static_cast<double>(up) / St) : 0.f;
#pragma unroll
          for (int t = 0; t < kW; ++t) x[t] *= scale;
#pragma unroll
          for (int t = 0; t < kW; t += 4)
            *reinterpret_cast<float4*>(Trow + t) = make_float4(x[t], x[t + 1], x[t + 2], x[t + 3]);
          store_planes(x);
          // Next GEMM1 (X̂ = π̂, MN-major) now.  The flags raised above are
          // visible after the barrier; a failing problem issues nothing.
          ptx::fence_proxy_async();
          ptx::tc_fence_before();
          __syncthreads();
          if (tid == 0 && ctl[0] == 0) issue(1);
        }
        block_sum8(ra, 2);
        if (phase == 2) {
          if (tid == 0 && rec) {
            rec[used].mw_w = ra[0];
            rec[used].row_sq = ra[1];
          }
          break;
        }
        if (tid == 0 && rec && k >= 2) {
          rec[k - 1].mw_w = ra[0];
          rec[k - 1].row_sq = ra[1];
        }
        if (ctl[0] != 0) {  // set before block_sum8's barriers
          err_iter = used = k;
          break;
        }
        phase = 1;
        continue;
      }
      // ---- half-step b, lane = column j = L: w' = (π ⊙ e^{G/ρ − c}) ν_j / C_j.
      const bool col_ok = L < m;
      const float cmax = line_max(acc_max());
      const float cr = cmax * k2;
      // t̂ = π̂ e^{G/ρ − c} (into x); Ĉ = Σ_i t̂, Σ_i π̂, ⟨G, π⟩ and Σ_i G t̂ (so
      // ⟨G, w'⟩ = s_j Σ_i G t̂ needs no second accumulator read).  π̂ is
      // column L of T; it also goes to TMEM for the final output.
      double gp, gt;
      {
        const float (&pv)[kW] = xo;
        const double P = xo_sum;
        gp = dotw([&](int t) { return x[t]; }, [&](int t) { return pv[t]; });
        float tv[kW];
#pragma unroll
        for (int t = 0; t < kW; ++t) tv[t] = pv[t] * ex2(fmaf(x[t], k2, -cr));
        gt = dotw([&](int t) { return x[t]; }, [&](int t) { return tv[t]; });
#pragma unroll
        for (int t = 0; t < kW; ++t) x[t] = tv[t];
        const double C = sumw([&](int t) { return x[t]; });
        st(kPT + c0, pv);
        red_d[(0 * kH + h) * kT + L] = C;
        red_d[(1 * kH + h) * kT + L] = P;
      }
      __syncthreads();
      double dsum[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // gw, split, diff, wold, gp, coldev
      const double Ct = line_sum(0);
      if (col_ok && h == 0) {
        if (cmax * g_true > 700.0f) atomicOr(&ctl[0], kFlagOverflowB);
        if (!(Ct > 0.0) || !isfinite(Ct) || isnan(cmax)) {
          atomicOr(&ctl[0], kFlagZeroB);
          atomicMin(&ctl[1], L);
        }
        const double dv = line_sum(1) * un64 - s_nu[L];
        dsum[5] = dv * dv;
      }
      const float sj = col_ok ? static_cast<float>(s_nu[L] * static_cast<double>(up) / Ct) : 0.f;
      ptx::tmem_wait_st();
      __syncthreads();
      if (ctl[0] != 0) {
        err_iter = used = k;
        break;
      }
      // ŵ' = sj t̂ (into x); fused diagnostics; ŵ'ᵀ → TMEM, column L of T,
      // K-major planes.  The old ŵ comes from TMEM, π̂ from T.
      double f1, f3, dd;
      {
        float wo[kW];
        ldw(kWT + c0, wo);
#pragma unroll
        for (int t = 0; t < kW; ++t) x[t] *= sj;
        st(kWT + c0, x);
        store_planes(x);
        ptx::tmem_wait_st();
        // Next GEMM1 (X̂ = ŵ', K-major: the next iteration or the tail) now;
        // the diagnostics below run under its MMAs.
        ptx::fence_proxy_async();
        ptx::tc_fence_before();
        __syncthreads();
        if (tid == 0) issue(0);
        f3 = dotw([&](int t) { return wo[t]; }, [&](int t) { return wo[t]; });
        // ‖w' − w‖² in fp64: near convergence the changes are off-support
        // entries of 1e-31 and below (the pinned rel_tol = 1e-30 is crossed
        // there, as in the reference, solvers.cpp:191,208), whose squares
        // underflow fp32.
        double d2[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int t = 0; t < kW; ++t) {
          const double df = static_cast<double>(x[t] - wo[t]);
          d2[t & 3] = __fma_rn(df, df, d2[t & 3]);
        }
        dd = (d2[0] + d2[1]) + (d2[2] + d2[3]);
#pragma unroll
        for (int t = 0; t < kW; ++t) {
          wo[t] = T[(c0 + t) * kTLd + L] - x[t];  // π̂ − ŵ'
          T[(c0 + t) * kTLd + L] = x[t];
        }
        f1 = dotw([&](int t) { return wo[t]; }, [&](int t) { return wo[t]; });
      }
      dsum[0] = gt * static_cast<double>(sj) * un2_64;
      dsum[1] = f1 * un2_64;
      dsum[2] = dd * un2_64;
      dsum[3] = f3 * un2_64;
      dsum[4] = gp * un2_64;
      block_sum8(dsum, 6);
      if (tid == 0) {
        if (rec) {
          DevRecord& r = rec[k];
          r.mpi_w = dsum[0];
          r.split_sq = dsum[1];
          r.diff_sq = dsum[2];
          r.wold_sq = dsum[3];
          r.mpi_pi = dsum[4];
          r.col_sq = dsum[5];
          r.elapsed = 1e-9 * static_cast<double>(globaltimer() - t0);
        }
        // The reference's rule as is: rel_change ≤ rel_tol (solvers.cpp:208).
        ctl[2] = sqrt(dsum[2]) / sqrt(dsum[3]) <= a.rel_tol ? 1 : 0;
      }
      __syncthreads();
      used = k;
      if (ctl[0] != 0) {  // (no flag is raised after the check above)
        mma_sync();
        err_iter = k;
        break;
      }
      if (ctl[2]) converged = 1;
      if (converged || k == a.max_iters) {
        phase = 2;  // tail: ⟨M(w), w⟩ and the row residual of the last w
      } else {
        ++k;
        phase = 0;
      }
    }
    // Final π (TMEM π̂ᵀ) and w (TMEM ŵᵀ) → HBM, fp32 padded 128×128 row-major;
    // a warp writes 32 consecutive columns of one row.
    {
      const float dn = ldexpf(1.0f, -sc);
      float* P = a.P + static_cast<int64_t>(b) * kT * kT + L;
      float* W = a.W + static_cast<int64_t>(b) * kT * kT + L;
      float pr[kW], wr[kW];
      ldw(kPT + c0, pr);
      ldw(kWT + c0, wr);
#pragma unroll
      for (int t = 0; t < kW; ++t) {
        const int i = c0 + t;
        P[i * kT] = pr[t] * dn;
        W[i * kT] = wr[t] * dn;
      }
    }
    if (tid == 0) {
      BatchStatus s{};
      s.flags = ctl[0];
      s.err_iter = err_iter;
      s.zero_index = ctl[1];
      s.used = used;
      s.converged = converged;
      a.st[b] = s;
    }
    ptx::tc_fence_before();
    __syncthreads();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<256>(tbase);
}

// K8 fix-up per problem: π rows rescaled to μ, w columns to ν in fp64,
// column-major outputs and the average ½(π + w).
__global__ void batched_fixup_kernel(const float* __restrict__ P, const float* __restrict__ W,
                                     const double* __restrict__ mu_p,
                                     const double* __restrict__ nu_p, int n, int m,
                                     double* out_pi, double* out_w, double* out_final) {
  const int64_t b = blockIdx.x;
  const float* p = P + b * kT * kT;
  const float* w = W + b * kT * kT;
  __shared__ double rs[kT], cs[kT];
  const int t = threadIdx.x;
  if (t < n) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s += p[t * kT + j];
    rs[t] = mu_p[b * kT + t] / s;
  }
  if (t < m) {
    double s = 0.0;
    for (int r = 0; r < n; ++r) s += w[r * kT + t];
    cs[t] = nu_p[b * kT + t] / s;
  }
  __syncthreads();
  const int64_t len = static_cast<int64_t>(n) * m;
  for (int64_t idx = t; idx < len; idx += blockDim.x) {
    const int j = static_cast<int>(idx / n), r = static_cast<int>(idx % n);
    const double vp = static_cast<double>(p[r * kT + j]) * rs[r];
    const double vw = static_cast<double>(w[r * kT + j]) * cs[j];
    if (out_pi) out_pi[b * len + idx] = vp;
    if (out_w) out_w[b * len + idx] = vw;
    out_final[b * len + idx] = 0.5 * (vp + vw);
  }
}

template <class T>
struct DevBuf {
  // Stream-ordered allocation: the default pool keeps the memory, so repeated
  // batched calls do not pay cudaMalloc/cudaFree of gigabytes each time.
  T* p = nullptr;
  cudaStream_t s = nullptr;
  DevBuf(size_t count, cudaStream_t stream) : s(stream) {
    if (count) GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

std::string fmtmsg(const char* f, long long a, const char* s) {
  char buf[512];
  std::snprintf(buf, sizeof(buf), f, a, s);
  return buf;
}

HostRecord to_host(const DevRecord& d, int64_t n, int64_t m) {
  HostRecord h;
  h.objective = -0.25 * (d.mpi_pi + 2.0 * d.mpi_w + d.mw_w);
  h.marginal_infeasibility = 0.5 * std::sqrt(d.col_sq) / static_cast<double>(m) +
                             0.5 * std::sqrt(d.row_sq) / static_cast<double>(n);
  h.split_gap = std::sqrt(d.split_sq);
  h.rel_change = std::sqrt(d.diff_sq) / std::sqrt(d.wold_sq);
  h.elapsed = d.elapsed;
  return h;
}

void fill_trace(gwb_record* out, const HostRecord* recs, int used) {
  for (int k = 0; k < used; ++k) {
    gwb_record& r = out[k];
    std::memset(&r, 0, sizeof(r));
    r.iter = k + 1;
    r.objective = recs[k].objective;
    r.marginal_infeasibility = recs[k].marginal_infeasibility;
    r.split_gap = recs[k].split_gap;
    r.rel_change = recs[k].rel_change;
    r.elapsed_seconds = recs[k].elapsed;
    r.phase = 0;
  }
}

struct BatchedOut {
  double* out_final;
  double* out_pi;
  double* out_w;
  gwb_record* trace;
  int32_t trace_cap;
  int32_t* n_records;
  int32_t* converged;
  int32_t* iterations_used;
};

// First failing problem (lowest index) raises, in bapg_solve's precedence.
struct Failure {
  int64_t problem = -1;
  int flags = 0, iter = 0, zero_index = 0;
};

// Same precedence as the single-problem path (capi.cu raise_device_flags,
// solvers.cpp:164-189); the detail names the problem.
[[noreturn]] void raise_failure(const Failure& f, bool name_problem = true) {
  std::string detail;
  if (f.flags & kFlagOverflowA)
    detail = "exp overflow; increase rho";
  else if (f.flags & kFlagZeroA)
    detail = fmtmsg("row %lld has nonpositive sum; cannot rescale", f.zero_index, "");
  else if (f.flags & kFlagOverflowB)
    detail = "exp overflow; increase rho";
  else if (f.flags & kFlagZeroB)
    detail = fmtmsg("column %lld has nonpositive sum; cannot rescale", f.zero_index, "");
  else
    detail = "non-finite iterate";
  if (!name_problem) api_numerical("bapg", f.iter, detail);
  api_numerical("bapg", f.iter, fmtmsg("problem %lld: %s", f.problem, detail.c_str()));
}

// Generic path: the full BapgEngine, one problem after another.  Problem
// indices in the returned failure are offset by `base`.
Failure batched_generic(const gwb_config* cfg, int device, int64_t batch, const double* dx,
                        int64_t n, const double* dy, int64_t m, const double* mu,
                        const double* nu, const BatchedOut& o, int64_t base) {
  BapgEngine eng(device, n, m, cfg->rho, cfg->precision, cfg->max_iters, nullptr);
  eng.set_geometry(cfg->geometry);
  const size_t len = static_cast<size_t>(n) * m;
  Failure first;
  for (int64_t b = 0; b < batch; ++b) {
    eng.load_host(dx + b * n * n, dy + b * m * m, mu + b * n, nu + b * m);
    eng.reset(nullptr);
    std::vector<double> residuals;
    DevStatus s;
    if (cfg->record_residual) {  // per-record Luo-Tseng residual (solvers.cpp:202-204)
      s = eng.run_stepped(cfg->max_iters, cfg->rel_tol, [&](int, const DevStatus&) {
        residuals.push_back(eng.residual_of_average(1e-8));
      });
    } else {
      eng.run(cfg->max_iters, cfg->rel_tol);
      s = eng.status();
    }
    if (s.flags) {
      if (first.problem < 0) first = Failure{base + b, s.flags, s.err_iter, s.zero_index};
      continue;
    }
    const int used = s.iter - 1;
    eng.tail();
    if (o.trace) {
      const std::vector<HostRecord> recs = eng.records(used);
      gwb_record* t = o.trace + b * o.trace_cap;
      fill_trace(t, recs.data(), used);
      for (size_t k = 0; k < residuals.size() && k < static_cast<size_t>(used); ++k) {
        t[k].residual = residuals[k];
        t[k].has_residual = 1;
      }
    }
    if (o.n_records) o.n_records[b] = o.trace ? used : 0;
    if (o.converged) o.converged[b] = s.converged;
    if (o.iterations_used) o.iterations_used[b] = used;
    eng.outputs(o.out_final + b * len, o.out_pi ? o.out_pi + b * len : nullptr,
                o.out_w ? o.out_w + b * len : nullptr);
  }
  return first;
}

}  // namespace

void device_bapg_batched(const gwb_config* cfg, int64_t batch, const double* dx, int64_t n,
                         const double* dy, int64_t m, const double* mu, const double* nu,
                         double* out_final, double* out_pi, double* out_w, gwb_record* trace,
                         int32_t trace_cap, int32_t* n_records, int32_t* converged,
                         int32_t* iterations_used, bool name_problem, int device,
                         int64_t index_base, double* kernel_ms) {
  if (!dx || !dy || !mu || !nu || !out_final) api_fail(GWB_ERR_INVALID, "null input/output buffer");
  if (trace && trace_cap < cfg->max_iters) api_fail(GWB_ERR_CAPACITY, "trace capacity < max_iters");
  if (device < 0) device = api_device();
  GWB_CUDA(cudaSetDevice(device));
  const BatchedOut o{out_final, out_pi, out_w, trace, trace_cap, n_records, converged, iterations_used};
  // The on-chip kernel runs the f16x2 chain (AUTO for 0/1 graphs, DESIGN.md
  // §4); other explicit precisions take the generic engine.
  const bool onchip_prec = cfg->precision == GWB_PREC_AUTO || cfg->precision == GWB_PREC_F16X2;
  double ms_total = 0.0;
  if (kernel_ms) *kernel_ms = 0.0;
  // The on-chip kernel implements the entropy geometry; the quadratic one
  // runs problem by problem on the generic engine.
  if (n > kT || m > kT || !onchip_prec || cfg->geometry != GWB_ENTROPY || cfg->record_residual) {
    const Failure f = batched_generic(cfg, device, batch, dx, n, dy, m, mu, nu, o, index_base);
    if (f.problem >= 0) raise_failure(f, name_problem);
    return;
  }
  pool_keep(device);
  // Streams: `s` stages the inputs (and owns the allocations), sc[0/1] run
  // alternate sub-chunks (pack, kernel, fix-up; a sub-chunk's kernel can start
  // while the previous one drains its last problems), `so` returns results.
  // H2D of sub-chunk c+1 and D2H of sub-chunk c-1 overlap sub-chunk c's kernel.
  cudaStream_t s, sc[2], so;
  GWB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  GWB_CUDA(cudaStreamCreateWithFlags(&sc[0], cudaStreamNonBlocking));
  GWB_CUDA(cudaStreamCreateWithFlags(&sc[1], cudaStreamNonBlocking));
  GWB_CUDA(cudaStreamCreateWithFlags(&so, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s[4];
    ~StreamGuard() {
      for (auto x : s) cudaStreamDestroy(x);
    }
  } sg{{s, sc[0], sc[1], so}};
  int sms = 148;
  GWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  // Bound the device working set: problems are processed in chunks.
  const int64_t chunk = std::min<int64_t>(batch, 16384);
  const size_t len = static_cast<size_t>(n) * m;
  constexpr int kSub = 8;  // max pipelined sub-chunks per chunk (each ≥ one wave)
  static const int sub_env = [] {
    const char* e = std::getenv("GWB_BATCHED_SUB");
    return e ? std::max(1, std::min(8, std::atoi(e))) : 0;
  }();
  const int sub_req = sub_env ? sub_env : 4;
  DevBuf<double> d_dx(chunk * n * n, s), d_dy(chunk * m * m, s), d_mu(chunk * n, s),
      d_nu(chunk * m, s);
  DevBuf<uint8_t> d_pack(chunk * 2 * kTileBytes, s);
  DevBuf<double> d_mup(chunk * kT, s), d_nup(chunk * kT, s);
  DevBuf<int> d_scl(chunk, s);
  DevBuf<float> d_P(chunk * kT * kT, s), d_W(chunk * kT * kT, s);
  DevBuf<DevRecord> d_rec(trace ? chunk * (cfg->max_iters + 2) : 0, s);
  DevBuf<BatchStatus> d_st(chunk, s);
  DevBuf<double> d_pi(out_pi ? chunk * len : 0, s), d_w(out_w ? chunk * len : 0, s),
      d_fin(chunk * len, s);
  DevBuf<int> d_inexact(1, s), d_next(kSub, s);
  GWB_CUDA(cudaFuncSetAttribute(bapg_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmem)));
  std::vector<cudaEvent_t> evs;
  auto event = [&](bool timing) {
    cudaEvent_t e;
    GWB_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    evs.push_back(e);
    return e;
  };
  struct EventGuard {
    std::vector<cudaEvent_t>* v;
    ~EventGuard() {
      for (auto e : *v) cudaEventDestroy(e);
    }
  } eg{&evs};
  std::vector<BatchStatus> hst(chunk);
  std::vector<DevRecord> hrec(trace ? chunk * (cfg->max_iters + 2) : 0);
  std::vector<HostRecord> hr(trace ? cfg->max_iters + 1 : 0);
  Failure first;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t cb = std::min(chunk, batch - b0);
    const int nsub = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sub_req, cb / sms)));
    GWB_CUDA(cudaMemsetAsync(d_inexact.p, 0, sizeof(int), s));
    GWB_CUDA(cudaMemsetAsync(d_next.p, 0, sizeof(int) * kSub, s));
    const cudaEvent_t ready = event(false);  // allocations and resets done
    GWB_CUDA(cudaEventRecord(ready, s));
    for (auto x : {sc[0], sc[1], so}) GWB_CUDA(cudaStreamWaitEvent(x, ready, 0));
    const cudaEvent_t k0 = event(true);
    std::vector<cudaEvent_t> kend(nsub);
    for (int c = 0; c < nsub; ++c) {
      const int64_t c0 = cb * c / nsub, c1 = cb * (c + 1) / nsub, cc = c1 - c0;
      const int64_t g0 = b0 + c0;  // problem index of the sub-chunk's first problem
      GWB_CUDA(cudaMemcpyAsync(d_dx.p + c0 * n * n, dx + g0 * n * n, sizeof(double) * cc * n * n, cudaMemcpyHostToDevice, s));
      GWB_CUDA(cudaMemcpyAsync(d_dy.p + c0 * m * m, dy + g0 * m * m, sizeof(double) * cc * m * m, cudaMemcpyHostToDevice, s));
      GWB_CUDA(cudaMemcpyAsync(d_mu.p + c0 * n, mu + g0 * n, sizeof(double) * cc * n, cudaMemcpyHostToDevice, s));
      GWB_CUDA(cudaMemcpyAsync(d_nu.p + c0 * m, nu + g0 * m, sizeof(double) * cc * m, cudaMemcpyHostToDevice, s));
      const cudaEvent_t in = event(false);
      GWB_CUDA(cudaEventRecord(in, s));
      const cudaStream_t cs = sc[c & 1];
      GWB_CUDA(cudaStreamWaitEvent(cs, in, 0));
      batched_pack_kernel<<<dim3(static_cast<unsigned>(cc), 2), 256, 0, cs>>>(
          d_dx.p + c0 * n * n, d_dy.p + c0 * m * m, d_mu.p + c0 * n, d_nu.p + c0 * m, static_cast<int>(n),
          static_cast<int>(m), d_pack.p + c0 * 2 * kTileBytes, d_mup.p + c0 * kT, d_nup.p + c0 * kT,
          d_scl.p + c0, d_inexact.p);
      GWB_CUDA(cudaGetLastError());
      BatchArgs a;
      a.dpack = d_pack.p + c0 * 2 * kTileBytes;
      a.mu = d_mup.p + c0 * kT;
      a.nu = d_nup.p + c0 * kT;
      a.scl = d_scl.p + c0;
      a.P = d_P.p + c0 * kT * kT;
      a.W = d_W.p + c0 * kT * kT;
      a.rec = trace ? d_rec.p + c0 * (cfg->max_iters + 2) : nullptr;
      a.st = d_st.p + c0;
      a.next = d_next.p + c;
      a.batch = static_cast<int>(cc);
      a.n = static_cast<int>(n);
      a.m = static_cast<int>(m);
      a.max_iters = cfg->max_iters;
      a.inv_rho = static_cast<float>(1.0 / cfg->rho);
      a.rel_tol = cfg->rel_tol;
      if (c == 0) GWB_CUDA(cudaEventRecord(k0, cs));
      bapg_batched_kernel<<<static_cast<unsigned>(std::min<int64_t>(cc, sms)), kThreads, kSmem, cs>>>(a);
      GWB_CUDA(cudaGetLastError());
      kend[c] = event(true);
      GWB_CUDA(cudaEventRecord(kend[c], cs));
      batched_fixup_kernel<<<static_cast<unsigned>(cc), kT, 0, cs>>>(
          a.P, a.W, a.mu, a.nu, static_cast<int>(n), static_cast<int>(m),
          out_pi ? d_pi.p + c0 * len : nullptr, out_w ? d_w.p + c0 * len : nullptr, d_fin.p + c0 * len);
      GWB_CUDA(cudaGetLastError());
      const cudaEvent_t done = event(false);
      GWB_CUDA(cudaEventRecord(done, cs));
      GWB_CUDA(cudaStreamWaitEvent(so, done, 0));
      GWB_CUDA(cudaMemcpyAsync(out_final + g0 * len, d_fin.p + c0 * len, sizeof(double) * cc * len, cudaMemcpyDeviceToHost, so));
      if (out_pi) GWB_CUDA(cudaMemcpyAsync(out_pi + g0 * len, d_pi.p + c0 * len, sizeof(double) * cc * len, cudaMemcpyDeviceToHost, so));
      if (out_w) GWB_CUDA(cudaMemcpyAsync(out_w + g0 * len, d_w.p + c0 * len, sizeof(double) * cc * len, cudaMemcpyDeviceToHost, so));
    }
    GWB_CUDA(cudaMemcpyAsync(hst.data(), d_st.p, sizeof(BatchStatus) * cb, cudaMemcpyDeviceToHost, so));
    if (trace)
      GWB_CUDA(cudaMemcpyAsync(hrec.data(), d_rec.p, sizeof(DevRecord) * cb * (cfg->max_iters + 2), cudaMemcpyDeviceToHost, so));
    int inexact = 0;
    GWB_CUDA(cudaMemcpyAsync(&inexact, d_inexact.p, sizeof(int), cudaMemcpyDeviceToHost, so));
    for (auto x : {s, sc[0], sc[1], so}) GWB_CUDA(cudaStreamSynchronize(x));
    // Device time of the chunk's solve: first kernel start → last kernel end.
    float kms = 0.f;
    for (int c = 0; c < nsub; ++c) {
      float t = 0.f;
      GWB_CUDA(cudaEventElapsedTime(&t, k0, kend[c]));
      kms = std::max(kms, t);
    }
    if (inexact) {
      // Structure matrices not exact in fp16: the on-chip kernel keeps D in
      // one fp16 plane, so these problems take the generic engine (its
      // results overwrite the on-chip ones).
      const BatchedOut sub{out_final + b0 * len, out_pi ? out_pi + b0 * len : nullptr,
                           out_w ? out_w + b0 * len : nullptr,
                           trace ? trace + b0 * trace_cap : nullptr, trace_cap,
                           n_records ? n_records + b0 : nullptr,
                           converged ? converged + b0 : nullptr,
                           iterations_used ? iterations_used + b0 : nullptr};
      const Failure f = batched_generic(cfg, device, cb, dx + b0 * n * n, n, dy + b0 * m * m, m,
                                        mu + b0 * n, nu + b0 * m, sub, b0);
      if (first.problem < 0 && f.problem >= 0) first = f;
      continue;
    }
    ms_total += kms;
    for (int64_t k = 0; k < cb; ++k) {
      const BatchStatus& st = hst[k];
      const int64_t b = b0 + k;
      if (st.flags) {
        if (first.problem < 0) first = Failure{b, st.flags, st.err_iter, st.zero_index};
        continue;
      }
      if (trace) {
        const DevRecord* r = hrec.data() + k * (cfg->max_iters + 2);
        for (int it = 1; it <= st.used; ++it) hr[it - 1] = to_host(r[it], n, m);
        fill_trace(trace + b * trace_cap, hr.data(), st.used);
      }
      if (n_records) n_records[b] = trace ? st.used : 0;
      if (converged) converged[b] = st.converged;
      if (iterations_used) iterations_used[b] = st.used;
    }
  }
  if (kernel_ms) *kernel_ms = ms_total;
  if (first.problem >= 0) {
    first.problem += index_base;
    raise_failure(first, name_problem);
  }
}

void set_batched_last(double ms, int64_t problems) {
  g_last_ms = ms;
  g_last_problems = problems;
}

}  // namespace gwb

int32_t gwb_batched_last_kernel_ms(double* ms, int64_t* problems) {
  if (ms) *ms = gwb::g_last_ms;
  if (problems) *problems = gwb::g_last_problems;
  return GWB_OK;
}
