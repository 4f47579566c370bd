// narrow.cuh — device-side pieces of the entropy BAPG projections that more
// than one translation unit runs: the fp64 exponent helpers and the
// warp-per-row half-step a for narrow rows (m ≤ 128; config 3), which
// kernels.cu launches on its own and skinny_tc.cu runs inside the skinny
// GEMM2's epilogue (solvers.cpp:164-170).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "devutil.cuh"
#include "kernels.cuh"

namespace gwb {
namespace dev {

// ---------------------------------------------------------------------------
// Entropy BAPG projections on fp64 iterates.  G arrives in
// fp32 from the chain; the exponent x = g·(1/ρ), the online (max, Σ), the
// exponentials and the iterates are fp64, as the reference computes them
// (solvers.cpp:164-177, projections.cpp:12-34).  The same helper forms x
// in the (max, Σ) pass and the write pass, so numerators and normaliser
// agree bitwise.
__device__ __forceinline__ double expo(float g, double inv_rho) {
  return __dmul_rn(static_cast<double>(g), inv_rho);
}

__device__ __forceinline__ void load_d4(const double* p, double (&v)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x;
  v[1] = a.y;
  v[2] = b.x;
  v[3] = b.y;
}

__device__ __forceinline__ void store_d4(double* p, const double (&v)[4]) {
  *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
}

// PDL (launch.cuh): wait for the predecessor kernel's results, then let the
// successor's CTAs be scheduled.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// A device error flag (DevFlag) raised at the current iteration: the first
// raise records err_iter; the iteration's remaining projection kernels skip
// on `flags`, and the finalize marks the solve done (no separate check
// launches).
__device__ __forceinline__ void raise_flag(DevStatus* st, int flag) {
  atomicOr(&st->flags, flag);
  atomicCAS(&st->err_iter, 0, st->iter);
}

// Narrow rows (m ≤ kNarrowM, config 3): one warp per row, 8 rows per CTA,
// lane l covering the 4-column groups at 4l + 128v — the row sits in
// registers between the (max, Σ) pass and the write, no block barriers.
constexpr int kNarrowM = 128;
constexpr int kNarrowV = kNarrowM / 128;  // 4-column groups per lane

// fp64 sum over aligned groups of GW lanes (a power of two).  Lanes holding
// 0 do not change a bit of the result, so a row that fits GW lanes gives the
// same value for every GW.
template <int GW>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = GW / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Half-step a of row i by an aligned group of GW lanes; all 32 lanes of the
// warp call it together (GW = 32: one row per warp, m ≤ 128; GW = 8: four
// rows per warp, m ≤ 32), `active` false for a group without a row.  `g` is
// row i of G (global or shared memory, 16-byte aligned, m values).  `keep32`
// (nullable) also receives the fp32 copy of the new row — the operand of the
// next GEMM1 when the caller forms it in the same kernel.
template <int GW>
__device__ __forceinline__ void narrow_row_update(const BapgDev& d, int64_t i, const float* g,
                                                  int lane, bool active, int write, float* keep32) {
  static_assert(GW == 32 || kNarrowV == 1, "sub-warp groups cover one 4-column group per lane");
  const int lig = lane & (GW - 1);
  const int64_t m = active ? d.m : 0;
  const double* w = d.W64 + (active ? i : 0) * d.ld;
  const double inv_rho = d.inv_rho64;
  double mx = -INFINITY;
  bool nan = false;
  double sums[3] = {0.0, 0.0, 0.0};  // ⟨G,W⟩, ΣW, then Σ W e^{x − max}
  float gv[kNarrowV][4];
  double wv[kNarrowV][4];
#pragma unroll
  for (int v = 0; v < kNarrowV; ++v) {
    const int64_t j = lig * 4 + 128 * v;
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
  // The row's max first (as row_update_reg_kernel), then every exponential
  // once: it serves the normaliser and the written value.
  const unsigned nans = __ballot_sync(0xffffffffu, nan);
  const unsigned group = GW == 32 ? 0xffffffffu : (((1u << (GW & 31)) - 1u) << (lane & ~(GW - 1)));
#pragma unroll
  for (int o = GW / 2; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const double r = (nans & group) ? NAN : mx;
  double ev[kNarrowV][4];
#pragma unroll
  for (int v = 0; v < kNarrowV; ++v) {
    const int64_t j = lig * 4 + 128 * v;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      ev[v][q] = (j + q < m) ? exp(expo(gv[v][q], inv_rho) - r) : 0.0;
      sums[2] = __fma_rn(wv[v][q], ev[v][q], sums[2]);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    sums[k] = group_sum<GW>(sums[k]);
    // The butterfly rounds lane-dependently; every lane takes its leader's.
    sums[k] = __shfl_sync(0xffffffffu, sums[k], lane & ~(GW - 1));
  }
  if (!active) return;
  if (lig == 0) {
    d.row_part[i].gw = sums[0];
    const double dev = sums[1] - d.mu64[i];
    d.row_part[i].rowdev = dev * dev;
  }
  if (!write) return;
  const double S = sums[2];
  if (lig == 0) {
    if (r > 700.0) raise_flag(d.st, kFlagOverflowA);
    if (!(S > 0.0) || !isfinite(S) || isnan(r)) {
      raise_flag(d.st, kFlagZeroA);
      atomicMin(&d.st->zero_index, static_cast<int>(i));
    }
  }
  const double scale = d.mu64[i] / S;
#pragma unroll
  for (int v = 0; v < kNarrowV; ++v) {
    const int64_t j = lig * 4 + 128 * v;
    if (j >= m) break;
    double o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = (j + q < m) ? scale * wv[v][q] * ev[v][q] : 0.0;
    store_d4(d.P64 + i * d.ld + j, o);
    aux_store4_64(d.P_aux, d.P, d.aux_mode, d.plane, i * d.ld + j, o, d.aux_scale);
    if (keep32 != nullptr) {
#pragma unroll
      for (int q = 0; q < 4; ++q) keep32[j + q] = static_cast<float>(o[q]);
    }
  }
}

}  // namespace dev
}  // namespace gwb
