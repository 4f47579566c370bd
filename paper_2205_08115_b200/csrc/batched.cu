// batched.cu — config 5: many independent small BAPG problems (n, m ≤ 128),
// one CTA per problem, every iteration on-chip.
//
// The reference runs such a batch as independent gw::solve calls from its
// experiment worker pool (experiment.cpp:273-304); each problem follows
// bapg_solve (solvers.cpp:138-217).  Here a persistent CTA owns one problem
// at a time:
//   SMEM  D_X (GEMM1 A operand) and D_Yᵀ (GEMM2 B operand) as bf16, exact
//         for 0/1 structure matrices (32 KB each, 128-B swizzled K-major);
//         one 96 KB buffer holding three bf16 planes of the current GEMM
//         operand — the iterate X (GEMM1's B, read MN-major) or V = D_X·X
//         (GEMM2's A), both written row by row by the owning thread; 15 KB
//         of reduction scratch and the marginals.
//   TMEM  512 columns: [0,128) accumulator of the hi plane, [128,256) π,
//         [256,384) w, [384,512) accumulator of the mid+lo planes (split
//         accumulation).
// One half-step = GEMM1 (3 planes × 8 MMAs of 128×128×16) → V planes →
// GEMM2 → row (a) or column (b) normalisation read straight from TMEM (G is
// folded into one TMEM block, the unnormalised kernel t cached in another),
// which also writes the next operand planes.  Column statistics use a
// 32-lane transpose-reduce plus a fixed-order merge of the 4 lane quadrants.  The fp64 diagnostics, trace record
// and the stop rule are evaluated by the CTA itself; nothing leaves the SM
// until the problem finishes.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
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
constexpr int kThreads = 256;                   // 8 warps: 4 lane quadrants × 2 column halves
constexpr uint32_t kTileBytes = kT * kT * 2;    // one bf16 operand plane (32 KB)
constexpr uint32_t kHalfTile = kTileBytes / 2;  // one 64-wide K chunk (16 KB)
constexpr uint32_t kAccHi = 0, kPi = 128, kW = 256, kAccLo = 384;  // TMEM columns
constexpr size_t kScratch = 16 * 1024;
constexpr size_t kSmem = 1024 + 5 * static_cast<size_t>(kTileBytes) + kScratch;

struct BatchStatus {
  int flags, err_iter, zero_index, used, converged, pad[3];
};

struct BatchArgs {
  const uint8_t* dpack;  // [batch][2][32 KB] pre-swizzled bf16: D_X (A), D_Yᵀ (B)
  const double* mu;      // [batch][128], zero padded
  const double* nu;
  float* P;              // [batch][128][128] final π
  float* W;              // [batch][128][128] final w
  DevRecord* rec;        // [batch][max_iters + 2] or null
  BatchStatus* st;
  int batch, n, m, max_iters;
  float inv_rho;
  double rel_tol;
};

// Byte offset of bf16 element (row, k) in a 128×128 K-major operand stored
// as two 64-wide K chunks, each the canonical 128-B swizzle layout.
__host__ __device__ __forceinline__ uint32_t sw_off(int row, int k) {
  return static_cast<uint32_t>(k >> 6) * kHalfTile + static_cast<uint32_t>(row) * 128u +
         ((static_cast<uint32_t>((k >> 3) & 7) ^ static_cast<uint32_t>(row & 7)) << 4) +
         (static_cast<uint32_t>(k & 7) << 1);
}

// Two fp32 values → three packed bf16x2 planes whose sum is exact
// (hi = rn(x), mid = rn(x − hi), lo = rn(x − hi − mid)).  One F2FP per plane
// pair; a bf16 is the upper half of the fp32 with the same value.
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo_elem, float hi_elem) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}
__device__ __forceinline__ void split3x2(float a, float b, uint32_t& p0, uint32_t& p1,
                                         uint32_t& p2) {
  p0 = cvt_bf16x2(a, b);
  a -= __uint_as_float(p0 << 16);
  b -= __uint_as_float(p0 & 0xFFFF0000u);
  p1 = cvt_bf16x2(a, b);
  a -= __uint_as_float(p1 << 16);
  b -= __uint_as_float(p1 & 0xFFFF0000u);
  p2 = cvt_bf16x2(a, b);
}

// Transpose-reduce: lane l holds v[0..31] (one row, 32 columns); afterwards
// v[0] of lane l is op over all 32 lanes of column l.  31 shuffles, fixed
// combination order (deterministic).
template <class T, class Op>
__device__ __forceinline__ T xreduce32(T (&v)[32], int lane, Op op) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const T send = upper ? v[k] : v[k + s];
      const T keep = upper ? v[k + s] : v[k];
      const T recv = __shfl_xor_sync(0xffffffffu, send, s);
      v[k] = op(keep, recv);
    }
  }
  return v[0];
}

struct FMax {
  __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};
struct FAdd {
  __device__ float operator()(float a, float b) const { return a + b; }
};
struct DAdd {
  __device__ double operator()(double a, double b) const { return a + b; }
};

// Operand packing: fp64 column-major inputs → bf16 swizzled tiles, the
// bf16-exactness check and zero-padded fp64 marginals.
__global__ void batched_pack_kernel(const double* __restrict__ dx, const double* __restrict__ dy,
                                    const double* __restrict__ mu, const double* __restrict__ nu,
                                    int n, int m, uint8_t* __restrict__ dpack,
                                    double* __restrict__ mu_p, double* __restrict__ nu_p,
                                    int* inexact) {
  const int64_t b = blockIdx.x;
  const int op = blockIdx.y;  // 0: D_X as A[i][k];  1: D_Yᵀ as B[j][k] = D_Y(k, j)
  const int dim = op == 0 ? n : m;
  const double* src = (op == 0 ? dx : dy) + b * static_cast<int64_t>(dim) * dim;
  __nv_bfloat16* dst =
      reinterpret_cast<__nv_bfloat16*>(dpack + (b * 2 + op) * static_cast<int64_t>(kTileBytes));
  bool bad = false;
  for (int idx = threadIdx.x; idx < kT * kT; idx += blockDim.x) {
    // idx = c·128 + r walks the column-major source contiguously.
    const int c = idx / kT, r = idx % kT;
    double v = 0.0;
    if (r < dim && c < dim) v = src[static_cast<int64_t>(c) * dim + r];
    const __nv_bfloat16 h = __float2bfloat16_rn(static_cast<float>(v));
    if (static_cast<double>(__bfloat162float(h)) != v) bad = true;
    // op 0: element (row r, col c) of D_X → A[r][c];  op 1: D_Y(r, c) → B[c][r].
    const uint32_t off = op == 0 ? sw_off(r, c) : sw_off(c, r);
    dst[off / 2] = h;
  }
  if (bad) atomicOr(inexact, 1);
  if (op == 0 && threadIdx.x < kT) {
    mu_p[b * kT + threadIdx.x] = threadIdx.x < n ? mu[b * n + threadIdx.x] : 0.0;
    nu_p[b * kT + threadIdx.x] = threadIdx.x < m ? nu[b * m + threadIdx.x] : 0.0;
  }
}

// UMMA descriptor of GEMM1's B operand, the iterate X[k = i][n = j] stored
// row-major in the same swizzled tiles as sw_off(i, j): MN-major, 64-wide N
// blocks LBO = 16 KB apart, 8-row K groups SBO = 1024 B apart, 128-B swizzle.
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(kHalfTile >> 4) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

__global__ void __launch_bounds__(kThreads, 1) bapg_batched_kernel(BatchArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sD = smem;                    // D_X | D_Yᵀ
  uint8_t* sPl = smem + 2 * kTileBytes;  // 3 operand planes
  float* red_f = reinterpret_cast<float*>(sPl + 3 * kTileBytes);  // [4][128]
  double* red_d = reinterpret_cast<double*>(red_f + 4 * kT);      // [4][128]
  float* col_c = reinterpret_cast<float*>(red_d + 4 * kT);        // [128]
  float* col_s = col_c + kT;                                      // [128]
  float* row_x = col_s + kT;                                      // [2][128]
  double* row_d = reinterpret_cast<double*>(row_x + 2 * kT);      // [2][128][2]
  double* diag = row_d + 4 * kT;                                  // [8][8]
  double* s_mu = diag + 64;                                       // [128]
  double* s_nu = s_mu + kT;                                       // [128]
  int* ctl = reinterpret_cast<int*>(s_nu + kT);                   // flags, zero_index, stop
  uint64_t* bars = reinterpret_cast<uint64_t*>(ctl + 8);          // load, mma
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, h = warp >> 2;
  const int i = q * 32 + lane;  // row owned (TMEM lane)
  const int c0 = h * 64;        // first of the 64 columns owned
  const int n = a.n, m = a.m;
  const bool row_ok = i < n;
  const float inv_rho = a.inv_rho;

  if (warp == 0) ptx::tmem_alloc<512>(tmem_slot);
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

  // TMEM loads are issued back to back and waited once per phase.
  auto ld = [&](uint32_t col, uint32_t (&r)[32]) { ptx::tmem_ld_32x32b_x32(tl + col, r); };
  auto load_cols = [&](uint32_t col, float (&v)[32]) {
    uint32_t r[32];
    ptx::tmem_ld_32x32b_x32(tl + col, r);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = __uint_as_float(r[t]);
  };
  // G chunk from the split accumulators (hi plane + mid/lo planes).
  auto load_acc = [&](int g, float (&v)[32]) {
    uint32_t hi[32];
    ptx::tmem_ld_32x32b_x32(tl + kAccHi + c0 + 32 * g, hi);
    ptx::tmem_wait_ld();
#pragma unroll
    for (int t = 0; t < 32; ++t) v[t] = __uint_as_float(hi[t]);
  };
  auto store_cols = [&](uint32_t col, const float (&v)[32]) {
    uint32_t r[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) r[t] = __float_as_uint(v[t]);
    ptx::tmem_st_32x32b_x32(tl + col, r);
  };
  // Row i, columns [col, col+32) of the next GEMM operand as bf16x3 planes.
  auto store_planes = [&](const float (&v)[32], int col) {
#pragma unroll
    for (int c8 = 0; c8 < 4; ++c8) {
      uint32_t pk[3][4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        split3x2(v[c8 * 8 + 2 * e], v[c8 * 8 + 2 * e + 1], pk[0][e], pk[1][e], pk[2][e]);
      const uint32_t off = sw_off(i, col + 8 * c8);
#pragma unroll
      for (int p = 0; p < 3; ++p)
        *reinterpret_cast<uint4*>(sPl + p * kTileBytes + off) =
            make_uint4(pk[p][0], pk[p][1], pk[p][2], pk[p][3]);
    }
  };
  // GEMM1: V = D_X · X (A = D_X K-major, B = X planes MN-major);
  // GEMM2: G = V · D_Y (A = V planes K-major, B = D_Yᵀ K-major).
  // Plane 0 accumulates into kAccHi, planes 1-2 into kAccLo.
  auto issue = [&](bool gemm1) {
    ptx::tc_fence_after();
    constexpr uint32_t id1 = ptx::idesc_bf16(128, 128) | (1u << 16);  // B MN-major
    constexpr uint32_t id2 = ptx::idesc_bf16(128, 128);
    // One accumulator, smallest plane first (lo, mid, hi): the small terms
    // are summed while the running sum is small, so the accumulator's
    // truncation acts on the 128 hi-plane terms only — the same bound as a
    // separate hi accumulator.
#pragma unroll 1
    for (int pi = 0; pi < 3; ++pi) {
      const int p = 2 - pi;
      const uint32_t d = tbase + kAccHi;
      const uint32_t pl = sPl_a + p * kTileBytes;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {  // K = 128 in steps of 16
        const uint32_t koff = (kk >> 2) * kHalfTile + (kk & 3) * 32;
        const uint64_t ad = ptx::umma_desc_sw128(gemm1 ? sD_a + koff : pl + koff);
        const uint64_t bd = gemm1 ? desc_mn(pl + kk * 2048) : ptx::umma_desc_sw128(sD_a + kTileBytes + koff);
        ptx::mma_bf16(d, ad, bd, gemm1 ? id1 : id2, (pi || kk) ? 1u : 0u);
      }
    }
    ptx::mma_commit(&bars[1]);
  };
  auto mma_sync = [&]() {
    ptx::mbar_wait(&bars[1], mma_ph);
    mma_ph ^= 1;
    ptx::tc_fence_after();
  };
  // G = D_X · X · D_Y for the X in the operand planes; V = D_X·X is re-split
  // into bf16x3 planes in between.  Result in the two accumulators.
  auto chain = [&]() {
    ptx::fence_proxy_async();
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) issue(true);
    mma_sync();
#pragma unroll 1
    for (int g = 0; g < 2; ++g) {
      float v[32];
      load_acc(g, v);
      store_planes(v, c0 + 32 * g);
    }
    ptx::fence_proxy_async();
    ptx::tc_fence_before();
    __syncthreads();
    if (tid == 0) issue(false);
    mma_sync();
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

  // Zero padding (rows ≥ n, columns ≥ m of D, π, w) keeps every padded
  // entry at 0 through the updates: G ≥ 0 there is never above a true
  // maximum, t = 0·e^{≤0} = 0, and the padded scales are forced to 0.
  for (int b = blockIdx.x; b < a.batch; b += gridDim.x) {
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
    const unsigned long long t0 = globaltimer();
    __syncthreads();
    // w⁰ = μνᵀ in fp32 (product_coupling_kernel, kernels.cu).
    {
      const float mu_i = static_cast<float>(s_mu[i]);
#pragma unroll 1
      for (int g = 0; g < 2; ++g) {
        float wv[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) wv[t] = mu_i * static_cast<float>(s_nu[c0 + 32 * g + t]);
        store_cols(kW + c0 + 32 * g, wv);
        store_planes(wv, c0 + 32 * g);
      }
      ptx::tmem_wait_st();
    }
    ptx::mbar_wait(&bars[0], load_ph);
    load_ph ^= 1;

    int k = 1, phase = 0, used = 0, converged = 0, err_iter = 0;
    for (;;) {
      chain();
      if (phase != 1) {
        // ---- half-step a (phase 0) / tail (phase 2): rows of G against w.
        float rmax = -INFINITY;
        double gw = 0.0, rw = 0.0;
#pragma unroll 1
        for (int g = 0; g < 2; ++g) {
          uint32_t ha[32], wr[32];
          ld(kAccHi + c0 + 32 * g, ha);
          ld(kW + c0 + 32 * g, wr);
          ptx::tmem_wait_ld();
          float gv[32], wv[32];
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            gv[t] = __uint_as_float(ha[t]);
            wv[t] = __uint_as_float(wr[t]);
          }
          float gwf = 0.f;
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            rmax = fmaxf(rmax, gv[t] * inv_rho);
            gwf = fmaf(gv[t], wv[t], gwf);
            rw += static_cast<double>(wv[t]);
          }
          gw += static_cast<double>(gwf);
        }
        row_x[h * kT + i] = rmax;
        row_d[(h * kT + i) * 2 + 0] = gw;
        row_d[(h * kT + i) * 2 + 1] = rw;
        __syncthreads();
        double ra[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (h == 0 && row_ok) {
          ra[0] = row_d[i * 2 + 0] + row_d[(kT + i) * 2 + 0];
          const double dv = row_d[i * 2 + 1] + row_d[(kT + i) * 2 + 1] - s_mu[i];
          ra[1] = dv * dv;
        }
        if (phase == 0) {
          // π = diag(μ / S) (w ⊙ e^{G/ρ − r}),  S = Σ_j w e^{G/ρ − r}
          ptx::tmem_wait_st();
          const float r = fmaxf(row_x[i], row_x[kT + i]);
          float S = 0.f;
#pragma unroll 1
          for (int g = 0; g < 2; ++g) {
            uint32_t gr[32], wr[32];
            ld(kAccHi + c0 + 32 * g, gr);
            ld(kW + c0 + 32 * g, wr);
            ptx::tmem_wait_ld();
            float gv[32];
#pragma unroll
            for (int t = 0; t < 32; ++t) {
              gv[t] = __uint_as_float(wr[t]) * __expf(__uint_as_float(gr[t]) * inv_rho - r);
              S += gv[t];
            }
            store_cols(kPi + c0 + 32 * g, gv);
          }
          __syncthreads();  // row_x (max) reads complete before reuse
          row_x[h * kT + i] = S;
          __syncthreads();
          const float St = row_x[i] + row_x[kT + i];
          if (h == 0 && row_ok) {
            if (r > 700.0f) atomicOr(&ctl[0], kFlagOverflowA);
            if (!(St > 0.0f) || !isfinite(St) || isnan(r)) {
              atomicOr(&ctl[0], kFlagZeroA);
              atomicMin(&ctl[1], i);
            }
          }
          const float scale = row_ok ? static_cast<float>(s_mu[i] / static_cast<double>(St)) : 0.f;
          ptx::tmem_wait_st();
#pragma unroll 1
          for (int g = 0; g < 2; ++g) {
            float pv[32];
            load_cols(kPi + c0 + 32 * g, pv);
#pragma unroll
            for (int t = 0; t < 32; ++t) pv[t] *= scale;
            store_cols(kPi + c0 + 32 * g, pv);
            store_planes(pv, c0 + 32 * g);
          }
          ptx::tmem_wait_st();
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
      // ---- half-step b: w' = (π ⊙ e^{G/ρ − c}) diag(ν / C) -----------------
      // B1: fold G, column max over rows.
#pragma unroll 1
      for (int g = 0; g < 2; ++g) {
        float gv[32];
        load_acc(g, gv);
#pragma unroll
        for (int t = 0; t < 32; ++t) gv[t] *= inv_rho;
        const float cm = xreduce32(gv, lane, FMax{});
        red_f[q * kT + c0 + 32 * g + lane] = cm;
      }
      __syncthreads();
      if (tid < kT) {
        float c = red_f[tid];
        for (int qq = 1; qq < 4; ++qq) c = fmaxf(c, red_f[qq * kT + tid]);
        col_c[tid] = c;
      }
      ptx::tmem_wait_st();
      __syncthreads();
      // B2: t = π e^{G/ρ − c} (kept in kAccLo); column sums of t (fp32) and π (fp64).
#pragma unroll 1
      for (int g = 0; g < 2; ++g) {
        uint32_t gr[32], pr[32];
        ld(kAccHi + c0 + 32 * g, gr);
        ld(kPi + c0 + 32 * g, pr);
        ptx::tmem_wait_ld();
        float gv[32];
        double pd[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const float pv = __uint_as_float(pr[t]);
          gv[t] = pv * __expf(__uint_as_float(gr[t]) * inv_rho - col_c[c0 + 32 * g + t]);
          pd[t] = static_cast<double>(pv);
        }
        store_cols(kAccLo + c0 + 32 * g, gv);
        const float cs = xreduce32(gv, lane, FAdd{});
        const double ps = xreduce32(pd, lane, DAdd{});
        red_f[q * kT + c0 + 32 * g + lane] = cs;
        red_d[q * kT + c0 + 32 * g + lane] = ps;
      }
      __syncthreads();
      double dsum[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // gw, split, diff, wold, gp, coldev
      if (tid < kT) {
        const int j = tid;
        float C = red_f[j];
        double P = red_d[j];
        for (int qq = 1; qq < 4; ++qq) {
          C += red_f[qq * kT + j];
          P += red_d[qq * kT + j];
        }
        if (j < m) {
          const float c = col_c[j];
          if (c > 700.0f) atomicOr(&ctl[0], kFlagOverflowB);
          if (!(C > 0.0f) || !isfinite(C) || isnan(c)) {
            atomicOr(&ctl[0], kFlagZeroB);
            atomicMin(&ctl[1], j);
          }
          col_s[j] = static_cast<float>(s_nu[j] / static_cast<double>(C));
          const double dv = P - s_nu[j];
          dsum[5] = dv * dv;
        } else {
          col_s[j] = 0.f;
        }
      }
      ptx::tmem_wait_st();
      __syncthreads();
      if (ctl[0] != 0) {
        err_iter = used = k;
        break;
      }
      // B3: w', fused diagnostics, next operand planes.
      bool finite = true;
#pragma unroll 1
      for (int g = 0; g < 2; ++g) {
        uint32_t gr[32], pr[32], wr[32], tr[32];
        ld(kAccHi + c0 + 32 * g, gr);
        ld(kPi + c0 + 32 * g, pr);
        ld(kW + c0 + 32 * g, wr);
        ld(kAccLo + c0 + 32 * g, tr);
        ptx::tmem_wait_ld();
        float tv[32];
#define gv(t) __uint_as_float(gr[t])
#define pv(t) __uint_as_float(pr[t])
#define wv(t) __uint_as_float(wr[t])
        float f[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
        // ‖w' − w‖² in fp64: near convergence the changes are off-support
        // entries of 1e-31 and below (the pinned rel_tol = 1e-30 is crossed
        // there, as in the reference, solvers.cpp:191,208), whose squares
        // underflow fp32.
        double dd = 0.0;
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const float o = col_s[c0 + 32 * g + t] * __uint_as_float(tr[t]);
          finite = finite && isfinite(o);
          f[0] = fmaf(gv(t), o, f[0]);
          const float sp = pv(t) - o;
          f[1] = fmaf(sp, sp, f[1]);
          const double df = static_cast<double>(o) - static_cast<double>(wv(t));
          dd = __fma_rn(df, df, dd);
          f[3] = fmaf(wv(t), wv(t), f[3]);
          f[4] = fmaf(gv(t), pv(t), f[4]);
          tv[t] = o;
        }
#undef gv
#undef pv
#undef wv
        f[2] = 0.f;
#pragma unroll
        for (int s = 0; s < 5; ++s) dsum[s] += static_cast<double>(f[s]);
        dsum[2] += dd;
        store_cols(kW + c0 + 32 * g, tv);
        store_planes(tv, c0 + 32 * g);
      }
      ptx::tmem_wait_st();
      if (!__syncthreads_and(finite ? 1 : 0) && tid == 0) ctl[0] |= kFlagNonFinite;
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
      if (ctl[0] != 0) {
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
    // Final π, w → HBM (fp32, padded 128×128).
    {
      float* P = a.P + static_cast<int64_t>(b) * kT * kT + static_cast<int64_t>(i) * kT + c0;
      float* W = a.W + static_cast<int64_t>(b) * kT * kT + static_cast<int64_t>(i) * kT + c0;
#pragma unroll 1
      for (int g = 0; g < 2; ++g) {
        uint32_t pr[32], wr[32];
        ld(kPi + c0 + 32 * g, pr);
        ld(kW + c0 + 32 * g, wr);
        ptx::tmem_wait_ld();
        float pv[32], wv[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          pv[t] = __uint_as_float(pr[t]);
          wv[t] = __uint_as_float(wr[t]);
        }
#pragma unroll
        for (int t = 0; t < 32; t += 4) {
          *reinterpret_cast<float4*>(P + 32 * g + t) = make_float4(pv[t], pv[t + 1], pv[t + 2], pv[t + 3]);
          *reinterpret_cast<float4*>(W + 32 * g + t) = make_float4(wv[t], wv[t + 1], wv[t + 2], wv[t + 3]);
        }
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
  if (warp == 0) ptx::tmem_dealloc<512>(tbase);
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
  const bool onchip_prec = cfg->precision == GWB_PREC_AUTO || cfg->precision == GWB_PREC_BF16X3;
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
  cudaStream_t s;
  GWB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};
  int sms = 148;
  GWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  // Bound the device working set: problems are processed in chunks.
  const int64_t chunk = std::min<int64_t>(batch, 16384);
  const size_t len = static_cast<size_t>(n) * m;
  DevBuf<double> d_dx(chunk * n * n, s), d_dy(chunk * m * m, s), d_mu(chunk * n, s),
      d_nu(chunk * m, s);
  DevBuf<uint8_t> d_pack(chunk * 2 * kTileBytes, s);
  DevBuf<double> d_mup(chunk * kT, s), d_nup(chunk * kT, s);
  DevBuf<float> d_P(chunk * kT * kT, s), d_W(chunk * kT * kT, s);
  DevBuf<DevRecord> d_rec(trace ? chunk * (cfg->max_iters + 2) : 0, s);
  DevBuf<BatchStatus> d_st(chunk, s);
  DevBuf<double> d_pi(out_pi ? chunk * len : 0, s), d_w(out_w ? chunk * len : 0, s),
      d_fin(chunk * len, s);
  DevBuf<int> d_inexact(1, s);
  GWB_CUDA(cudaFuncSetAttribute(bapg_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmem)));
  cudaEvent_t ev0, ev1;
  GWB_CUDA(cudaEventCreate(&ev0));
  GWB_CUDA(cudaEventCreate(&ev1));
  struct EventGuard {
    cudaEvent_t a, b;
    ~EventGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } eg{ev0, ev1};
  std::vector<BatchStatus> hst(chunk);
  std::vector<DevRecord> hrec(trace ? chunk * (cfg->max_iters + 2) : 0);
  std::vector<HostRecord> hr(trace ? cfg->max_iters + 1 : 0);
  Failure first;
  for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
    const int64_t cb = std::min(chunk, batch - b0);
    GWB_CUDA(cudaMemcpyAsync(d_dx.p, dx + b0 * n * n, sizeof(double) * cb * n * n, cudaMemcpyHostToDevice, s));
    GWB_CUDA(cudaMemcpyAsync(d_dy.p, dy + b0 * m * m, sizeof(double) * cb * m * m, cudaMemcpyHostToDevice, s));
    GWB_CUDA(cudaMemcpyAsync(d_mu.p, mu + b0 * n, sizeof(double) * cb * n, cudaMemcpyHostToDevice, s));
    GWB_CUDA(cudaMemcpyAsync(d_nu.p, nu + b0 * m, sizeof(double) * cb * m, cudaMemcpyHostToDevice, s));
    GWB_CUDA(cudaMemsetAsync(d_inexact.p, 0, sizeof(int), s));
    batched_pack_kernel<<<dim3(static_cast<unsigned>(cb), 2), 256, 0, s>>>(
        d_dx.p, d_dy.p, d_mu.p, d_nu.p, static_cast<int>(n), static_cast<int>(m), d_pack.p,
        d_mup.p, d_nup.p, d_inexact.p);
    GWB_CUDA(cudaGetLastError());
    int inexact = 0;
    GWB_CUDA(cudaMemcpyAsync(&inexact, d_inexact.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    GWB_CUDA(cudaStreamSynchronize(s));
    if (inexact) {
      // Structure matrices not exact in bf16: the on-chip kernel keeps D in
      // one bf16 plane, so these problems take the generic (3xTF32) engine.
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
    BatchArgs a;
    a.dpack = d_pack.p;
    a.mu = d_mup.p;
    a.nu = d_nup.p;
    a.P = d_P.p;
    a.W = d_W.p;
    a.rec = trace ? d_rec.p : nullptr;
    a.st = d_st.p;
    a.batch = static_cast<int>(cb);
    a.n = static_cast<int>(n);
    a.m = static_cast<int>(m);
    a.max_iters = cfg->max_iters;
    a.inv_rho = static_cast<float>(1.0 / cfg->rho);
    a.rel_tol = cfg->rel_tol;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(cb, sms));
    GWB_CUDA(cudaEventRecord(ev0, s));
    bapg_batched_kernel<<<grid, kThreads, kSmem, s>>>(a);
    GWB_CUDA(cudaGetLastError());
    GWB_CUDA(cudaEventRecord(ev1, s));
    batched_fixup_kernel<<<static_cast<unsigned>(cb), kT, 0, s>>>(
        d_P.p, d_W.p, d_mup.p, d_nup.p, static_cast<int>(n), static_cast<int>(m),
        out_pi ? d_pi.p : nullptr, out_w ? d_w.p : nullptr, d_fin.p);
    GWB_CUDA(cudaGetLastError());
    GWB_CUDA(cudaMemcpyAsync(out_final + b0 * len, d_fin.p, sizeof(double) * cb * len, cudaMemcpyDeviceToHost, s));
    if (out_pi) GWB_CUDA(cudaMemcpyAsync(out_pi + b0 * len, d_pi.p, sizeof(double) * cb * len, cudaMemcpyDeviceToHost, s));
    if (out_w) GWB_CUDA(cudaMemcpyAsync(out_w + b0 * len, d_w.p, sizeof(double) * cb * len, cudaMemcpyDeviceToHost, s));
    GWB_CUDA(cudaMemcpyAsync(hst.data(), d_st.p, sizeof(BatchStatus) * cb, cudaMemcpyDeviceToHost, s));
    if (trace)
      GWB_CUDA(cudaMemcpyAsync(hrec.data(), d_rec.p, sizeof(DevRecord) * cb * (cfg->max_iters + 2), cudaMemcpyDeviceToHost, s));
    GWB_CUDA(cudaStreamSynchronize(s));
    float kms = 0.f;
    GWB_CUDA(cudaEventElapsedTime(&kms, ev0, ev1));
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
