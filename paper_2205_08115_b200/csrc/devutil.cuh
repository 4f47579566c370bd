// devutil.cuh — device helpers shared by the projection / Sinkhorn kernels:
// TF32 operand splitting, %globaltimer, and the (max, Σ v·e^{x−max}) online
// accumulator with deterministic (fixed-order) warp and block reductions.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

namespace gwb {
namespace dev {

// Stop rule rel_change ≤ rel_tol (solvers.cpp:208, :284, :354) for the engines
// whose iterate still passes through fp32 (quadratic BAPG, eBPG / BPG /
// hBPG): their iterate stops moving once changes fall below fp32 resolution
// (rel_change exactly 0) where the reference's fp64 iterate still moves, so a
// tolerance below the fp64 noise floor is not compared against it.  The fp64
// entropy BAPG engines and the batched kernel (fp64 ‖Δw‖²) apply the
// reference's rule as is — pinned c5 problems do cross rel_tol = 1e-30
// (iteration 149-350) in the reference.
constexpr double kFp64Floor = 1e-15;
__host__ __device__ __forceinline__ bool stop_rule(double rel, double rel_tol) {
  return rel_tol >= kFp64Floor && rel <= rel_tol;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(a));
  const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(b));
  return lo | (hi << 16);
}

__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}

__device__ __forceinline__ float trunc_tf32(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Operand copy for the next GEMM: 1 → TF32 round-to-nearest-away (unbiased
// 1xTF32 input), 2 → residual x − trunc_tf32(x) (3xTF32 low part), itself
// rounded to nearest at TF32 precision: kind::tf32 truncates its fp32
// operands, and a truncated residual biases every product low (measured:
// 1e-6 relative on c2's weighted chain); a pre-rounded one is read exactly.
__device__ __forceinline__ float aux_of(float x, int mode) {
  return mode == 1 ? rna_tf32(x) : rna_tf32(x - trunc_tf32(x));
}

// GEMM operand copy of 4 consecutive values at element offset `off`:
//   mode 1/2: one fp32 plane (rna_tf32(x) or x − trunc_tf32(x));
//   mode 3/4: 3 or 2 bf16 planes, `plane` elements apart, whose sum is x
//             (round-to-nearest splits hi = rn(x), mid = rn(x − hi), …);
//   mode 5:   2 fp16 planes of x·scale (scale a power of two chosen by the
//             caller so that x·scale stays inside fp16 range; f16x2).
__device__ __forceinline__ void aux_store4(float* aux, int mode, int64_t plane, int64_t off,
                                           float a, float b, float c, float d,
                                           float scale = 1.0f) {
  if (mode <= 2) {
    *reinterpret_cast<float4*>(aux + off) =
        make_float4(aux_of(a, mode), aux_of(b, mode), aux_of(c, mode), aux_of(d, mode));
    return;
  }
  if (mode == 5) {
    __half* base = reinterpret_cast<__half*>(aux);
    float v[4] = {a * scale, b * scale, c * scale, d * scale};
    for (int pl = 0; pl < 2; ++pl) {
      __half h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        h[q] = __float2half_rn(v[q]);
        v[q] -= __half2float(h[q]);
      }
      *reinterpret_cast<uint2*>(base + pl * plane + off) =
          make_uint2(__half_as_ushort(h[0]) | (static_cast<uint32_t>(__half_as_ushort(h[1])) << 16),
                     __half_as_ushort(h[2]) | (static_cast<uint32_t>(__half_as_ushort(h[3])) << 16));
    }
    return;
  }
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(aux);
  float v[4] = {a, b, c, d};
  const int planes = mode == 3 ? 3 : 2;
  for (int pl = 0; pl < planes; ++pl) {
    float h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = bf16_round(v[q]);
      v[q] -= h[q];
    }
    *reinterpret_cast<uint2*>(base + pl * plane + off) =
        make_uint2(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3]));
  }
}

// GEMM operand copies of 4 consecutive fp64 iterate values (entropy BAPG
// keeps π, w in fp64).  `copy32` (nullable) receives the fp32
// value — the hi operand of the TF32 chains and the input of the raw-iterate
// chains (sparse, skinny).  Planes are split from the fp64 value, so the
// split keeps the bits below fp32:
//   mode 1: aux = rna_tf32(fp32(x));
//   mode 2: aux = rna_tf32(x − trunc_tf32(fp32(x)))  (hi is read from copy32);
//   mode 3/4: 3 / 2 bf16 planes, hi = rn(x), mid = rn(x − hi), …;
//   mode 5: 2 fp16 planes of x·scale.
__device__ __forceinline__ void aux_store4_64(float* aux, float* copy32, int mode, int64_t plane,
                                              int64_t off, const double (&x)[4], float scale) {
  if (copy32) {
    *reinterpret_cast<float4*>(copy32 + off) =
        make_float4(static_cast<float>(x[0]), static_cast<float>(x[1]), static_cast<float>(x[2]),
                    static_cast<float>(x[3]));
  }
  if (!aux) return;
  if (mode <= 2) {
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float f = static_cast<float>(x[q]);
      o[q] = mode == 1 ? rna_tf32(f)
                       : rna_tf32(static_cast<float>(x[q] - static_cast<double>(trunc_tf32(f))));
    }
    *reinterpret_cast<float4*>(aux + off) = make_float4(o[0], o[1], o[2], o[3]);
    return;
  }
  if (mode == 5) {
    __half* base = reinterpret_cast<__half*>(aux);
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = x[q] * static_cast<double>(scale);
    for (int pl = 0; pl < 2; ++pl) {
      __half h[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        h[q] = __double2half(v[q]);
        v[q] -= static_cast<double>(__half2float(h[q]));
      }
      *reinterpret_cast<uint2*>(base + pl * plane + off) =
          make_uint2(__half_as_ushort(h[0]) | (static_cast<uint32_t>(__half_as_ushort(h[1])) << 16),
                     __half_as_ushort(h[2]) | (static_cast<uint32_t>(__half_as_ushort(h[3])) << 16));
    }
    return;
  }
  __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(aux);
  double v[4] = {x[0], x[1], x[2], x[3]};
  const int planes = mode == 3 ? 3 : 2;
  for (int pl = 0; pl < planes; ++pl) {
    float h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      h[q] = __bfloat162float(__double2bfloat16(v[q]));
      v[q] -= static_cast<double>(h[q]);
    }
    *reinterpret_cast<uint2*>(base + pl * plane + off) =
        make_uint2(pack_bf16x2(h[0], h[1]), pack_bf16x2(h[2], h[3]));
  }
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Online log-sum-exp accumulator (max, Σ w·e^{x−max}) shared by the BAPG
// projections (kernels.cu: fp32 state, iterate weights) and the eBPG / BPG
// Sinkhorn scaling (bregman.cu: fp64 potentials, unit weights): the same
// add, merge and warp butterfly, in a fixed order.  Per-element
// exponentials are fp32 MUFU in both (arguments ≤ 0); the merge exp is fp32
// for the fp32 state and libdevice exp for the fp64 one.  FMAs are explicit
// so every kernel that inlines these computes bit-identical sums (no
// context-dependent contraction).
template <class T>
struct OnlineLse {
  T mx;
  T s;
};
__device__ __forceinline__ float lse_ex(float x) { return __expf(x); }
__device__ __forceinline__ double lse_ex(double x) {
  return static_cast<double>(__expf(static_cast<float>(x)));
}
__device__ __forceinline__ float lse_ex_merge(float x) { return __expf(x); }
__device__ __forceinline__ double lse_ex_merge(double x) { return exp(x); }
__device__ __forceinline__ float lse_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double lse_fma(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float lse_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double lse_mul(double a, double b) { return __dmul_rn(a, b); }

// a ⊕= (x, w): -inf contributes nothing, NaN poisons the max.
template <class T>
__device__ __forceinline__ void lse_add(OnlineLse<T>& a, T x, T w) {
  if (x > a.mx) {
    a.s = lse_fma(a.s, lse_ex(a.mx - x), w);
    a.mx = x;
  } else if (x > -INFINITY) {
    a.s = lse_fma(w, lse_ex(x - a.mx), a.s);
  } else if (isnan(x)) {
    a.mx = NAN;
  }
}

// a ⊕= K unit-weight terms at once: one max / rescale per block, the K
// exponentials in fp32, summed, then added in the accumulator's type — the
// bandwidth-bound form of K lse_add(a, x, 1) calls (equal up to rounding).
template <int K, class T>
__device__ __forceinline__ void lse_add_block(OnlineLse<T>& a, const T (&x)[K]) {
  T mb = -INFINITY;
  bool nan = false;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    nan = nan || isnan(x[q]);
    mb = x[q] > mb ? x[q] : mb;
  }
  if (nan) {
    a.mx = NAN;
    return;
  }
  if (mb == -INFINITY) return;
  if (mb > a.mx) {
    a.s = lse_mul(a.s, lse_ex(a.mx - mb));
    a.mx = mb;
  }
  float sum = 0.f;
#pragma unroll
  for (int q = 0; q < K; ++q) sum += __expf(static_cast<float>(x[q] - a.mx));
  a.s += static_cast<T>(sum);
}

template <class T>
__device__ __forceinline__ OnlineLse<T> lse_merge(OnlineLse<T> a, OnlineLse<T> b) {
  if (isnan(a.mx) || isnan(b.mx)) return OnlineLse<T>{static_cast<T>(NAN), static_cast<T>(NAN)};
  if (b.mx == -INFINITY) return a;
  if (a.mx == -INFINITY) return b;
  const T M = a.mx > b.mx ? a.mx : b.mx;
  return OnlineLse<T>{M, lse_fma(a.s, lse_ex_merge(a.mx - M), lse_mul(b.s, lse_ex_merge(b.mx - M)))};
}

// xor butterfly over the warp; lanes may differ by an ulp afterwards, so
// callers that need one value per warp take lane 0's.
template <class T>
__device__ __forceinline__ OnlineLse<T> lse_warp_merge(OnlineLse<T> a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    OnlineLse<T> b;
    b.mx = __shfl_xor_sync(0xffffffffu, a.mx, o);
    b.s = __shfl_xor_sync(0xffffffffu, a.s, o);
    a = lse_merge(a, b);
  }
  return a;
}

// The BAPG names (fp32 state, iterate-weighted terms).
using MaxSum = OnlineLse<float>;
__device__ __forceinline__ void ms_add(MaxSum& a, float e, float v) { lse_add(a, e, v); }
__device__ __forceinline__ MaxSum ms_merge(MaxSum a, MaxSum b) { return lse_merge(a, b); }
__device__ __forceinline__ MaxSum warp_merge(MaxSum a) { return lse_warp_merge(a); }

// fp64 online (max, Σ w·e^{x−max}) with correctly rounded-class fp64
// exponentials: the accumulator of the entropy BAPG projections, whose
// iterates are fp64 like the reference's (the fp32 MUFU form above injects
// ~1e-7 relative noise per element and half-step, which BAPG's saddle
// escapes amplify past the 1e-5 objective bound on c1).
struct Lse64 {
  double mx;
  double s;
};
__device__ __forceinline__ void lse64_add(Lse64& a, double x, double w) {
  if (x > a.mx) {
    a.s = __fma_rn(a.s, exp(a.mx - x), w);
    a.mx = x;
  } else if (x > -INFINITY) {
    a.s = __fma_rn(w, exp(x - a.mx), a.s);
  } else if (isnan(x)) {
    a.mx = NAN;
  }
}
__device__ __forceinline__ Lse64 lse64_merge(Lse64 a, Lse64 b) {
  if (isnan(a.mx) || isnan(b.mx)) return Lse64{NAN, NAN};
  if (b.mx == -INFINITY) return a;
  if (a.mx == -INFINITY) return b;
  const double M = a.mx > b.mx ? a.mx : b.mx;
  return Lse64{M, __fma_rn(a.s, exp(a.mx - M), __dmul_rn(b.s, exp(b.mx - M)))};
}
// Warp-wide merge of (max, Σ) pairs over the first `lanes` lanes (a power
// of two; the others must hold {−inf, 0}): the max by an xor butterfly, then
// each lane rescales its own sum once (one exp per lane instead of one per
// butterfly step) and the rescaled sums are added by a butterfly.  NaN in
// any max gives NaN.  The sum's butterfly rounds lane-dependently; every
// lane returns lane 0's value (deterministic).
template <int kLanes = 32>
__device__ __forceinline__ Lse64 lse64_warp_merge(Lse64 a) {
  const bool nan = __any_sync(0xffffffffu, isnan(a.mx));
  double M = a.mx;
#pragma unroll
  for (int o = kLanes / 2; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
  double s = (a.mx == -INFINITY || M == -INFINITY) ? 0.0 : a.s * exp(a.mx - M);
#pragma unroll
  for (int o = kLanes / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  s = __shfl_sync(0xffffffffu, s, 0);
  if (nan) return Lse64{NAN, NAN};
  return Lse64{M, s};
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide (max,sum) merge + up to 5 fp64 sums; result broadcast to all.
template <int kThreads, int kSums>
__device__ void block_reduce(MaxSum& ms, double (&sums)[kSums]) {
  constexpr int kWarps = kThreads / 32;
  __shared__ float s_mx[kWarps], s_s[kWarps];
  __shared__ double s_d[kSums][kWarps];
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  ms = warp_merge(ms);
#pragma unroll
  for (int k = 0; k < kSums; ++k) sums[k] = warp_sum(sums[k]);
  if (l == 0) {
    s_mx[w] = ms.mx;
    s_s[w] = ms.s;
#pragma unroll
    for (int k = 0; k < kSums; ++k) s_d[k][w] = sums[k];
  }
  __syncthreads();
  MaxSum r{-INFINITY, 0.f};
  double t[kSums];
#pragma unroll
  for (int k = 0; k < kSums; ++k) t[k] = 0.0;
  for (int q = 0; q < kWarps; ++q) {  // fixed order ⇒ deterministic
    r = ms_merge(r, MaxSum{s_mx[q], s_s[q]});
#pragma unroll
    for (int k = 0; k < kSums; ++k) t[k] += s_d[k][q];
  }
  ms = r;
#pragma unroll
  for (int k = 0; k < kSums; ++k) sums[k] = t[k];
  __syncthreads();
}

// block_reduce for the fp64 accumulator; lane 0 of each warp feeds a
// fixed-order merge, the result is broadcast to all threads.
// Warp 0 merges the kWarps per-warp results (lanes < kWarps, fixed order)
// and broadcasts them through shared memory: one exp per lane per level.
// `with_lse` = false skips the (max, Σ) merge (sums only).
template <int kThreads, int kSums, bool with_lse = true>
__device__ void block_reduce64(Lse64& ms, double (&sums)[kSums]) {
  constexpr int kWarps = kThreads / 32;
  static_assert(kWarps <= 32 && (kWarps & (kWarps - 1)) == 0, "warps: power of two ≤ 32");
  __shared__ double s_mx[kWarps], s_s[kWarps];
  __shared__ double s_d[kSums > 0 ? kSums : 1][kWarps];
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  if (with_lse) ms = lse64_warp_merge(ms);
#pragma unroll
  for (int k = 0; k < kSums; ++k) sums[k] = warp_sum(sums[k]);
  if (l == 0) {
    s_mx[w] = ms.mx;
    s_s[w] = ms.s;
#pragma unroll
    for (int k = 0; k < kSums; ++k) s_d[k][w] = sums[k];
  }
  __syncthreads();
  if (w == 0) {
    Lse64 r{-INFINITY, 0.0};
    if (with_lse && l < kWarps) r = Lse64{s_mx[l], s_s[l]};
    if (with_lse) r = lse64_warp_merge<kWarps>(r);
    double t[kSums > 0 ? kSums : 1];
#pragma unroll
    for (int k = 0; k < kSums; ++k) {
      t[k] = 0.0;
      if (l == 0)
        for (int q = 0; q < kWarps; ++q) t[k] += s_d[k][q];
    }
    __syncwarp();
    if (l == 0) {
      s_mx[0] = r.mx;
      s_s[0] = r.s;
#pragma unroll
      for (int k = 0; k < kSums; ++k) s_d[k][0] = t[k];
    }
  }
  __syncthreads();
  if (with_lse) ms = Lse64{s_mx[0], s_s[0]};
#pragma unroll
  for (int k = 0; k < kSums; ++k) sums[k] = s_d[k][0];
  __syncthreads();
}

}  // namespace dev
}  // namespace gwb
