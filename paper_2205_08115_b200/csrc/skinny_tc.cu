// skinny_tc.cu — GEMM2 of the skinny chain (m ≤ 32, config 3) on the tensor
// cores: G[M×N] = D · Σ_p V_pᵀ with D an exact-bf16 n×n structure matrix
// (0/1 graph) and V_p the three bf16 planes of Vᵀ (N×K, N ≤ 32), i.e. the
// bf16x3 chain with N padded to 32.  The product is a pure stream of D
// (K-major, TMA, 128-B swizzle): 16 KB of D per 64-wide k-block against
// 3 × 4 KB of V planes, 12 tcgen05.mma (M=128, N=32, K=16) per k-block.
//
// One CTA per (128-row tile, K split); the split count fills the SMs with
// one CTA each.  Warp 0: TMA producer over a 6-stage ring; warp 1: MMA
// issuer; warps 2–5: epilogue, one TMEM lane quadrant each.  As in gemm.cu,
// the tensor core's truncating fp32 accumulation is bounded by restarting it
// every 2 k-blocks in one of two TMEM buffers and promoting each chunk into
// fp32 registers with round-to-nearest adds.  K-split partials go to a
// workspace; in the last CTA of a row tile to finish (arrival counter) each
// epilogue thread sums its row's partials in split order and writes it —
// deterministic, no second launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>

#include "gemm.cuh"
#include "ptx.cuh"
#include "skinny.cuh"

namespace gwb {

void check_cuda(cudaError_t e, const char* what);  // solver.cu

namespace {

constexpr int kBM = 128, kBN = 32, kBK = 64;  // bf16: 64 K-elements per 128-B row
constexpr int kStages = 6;
constexpr int kPromote = 2;                    // k-blocks per TMEM chunk
constexpr uint32_t kATile = kBM * 128;         // 16 KB
constexpr uint32_t kBTile = kBN * 128;         // 4 KB
constexpr uint32_t kStageBytes = kATile + 3 * kBTile;
constexpr int kThreads = 192;
constexpr size_t kSmem = 1024 + static_cast<size_t>(kStages) * kStageBytes;

struct SkinnyTcParams {
  CUtensorMap a_map;
  CUtensorMap b_map[3];
  int planes;
  float* c;
  int64_t ldc;
  float* ws;            // [splits][M][kBN] partial sums (splits > 1)
  unsigned* counters;   // per row tile (splits > 1), left at 0 after each launch
  int64_t M;
  int N;
  int kblocks, splits, kb_per;
  const int* skip;
};

__global__ void __launch_bounds__(kThreads, 1)
    skinny_tc_kernel(const __grid_constant__ SkinnyTcParams p) {
  if (p.skip != nullptr && *p.skip != 0) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t full[kStages], empty[kStages], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int last_cta;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int tile = blockIdx.x / p.splits, split = blockIdx.x % p.splits;
  const int kb0 = split * p.kb_per;
  const int nkb = max(0, min(p.kblocks - kb0, p.kb_per));
  const int nchunks = (nkb + kPromote - 1) / kPromote;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&p.a_map);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], 1);
      ptx::mbar_init(&acc_empty[b], 4);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<2 * kBN>(&tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (ptx::elect_one()) {
      const uint32_t bytes = kATile + static_cast<uint32_t>(p.planes) * kBTile;
      for (int it = 0; it < nkb; ++it) {
        const int s = it % kStages;
        ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        uint8_t* st = smem + static_cast<size_t>(s) * kStageBytes;
        ptx::mbar_arrive_expect_tx(&full[s], bytes);
        const int kc = (kb0 + it) * kBK;
        ptx::tma_load_2d(st, &p.a_map, &full[s], kc, tile * kBM);
        for (int q = 0; q < p.planes; ++q)
          ptx::tma_load_2d(st + kATile + q * kBTile, &p.b_map[q], &full[s], kc, 0);
      }
    }
  } else if (warp == 1) {
    if (ptx::elect_one()) {
      constexpr uint32_t idesc = ptx::idesc_bf16(kBM, kBN);
      for (int it = 0; it < nkb; ++it) {
        const int c = it / kPromote, b = c & 1;
        const bool first = (it % kPromote) == 0;
        if (first) {
          ptx::mbar_wait(&acc_empty[b], ((c >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
        }
        const int s = it % kStages;
        ptx::mbar_wait(&full[s], (it / kStages) & 1);
        ptx::tc_fence_after();
        const uint32_t a_addr = ptx::smem_u32(smem + static_cast<size_t>(s) * kStageBytes);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          for (int q = p.planes - 1; q >= 0; --q) {  // smallest plane first
            const uint64_t ad = ptx::umma_desc_sw128(a_addr + kk * 32);
            const uint64_t bd = ptx::umma_desc_sw128(a_addr + kATile + q * kBTile + kk * 32);
            const uint32_t acc = (first && kk == 0 && q == p.planes - 1) ? 0u : 1u;
            ptx::mma_bf16(tmem + static_cast<uint32_t>(b * kBN), ad, bd, idesc, acc);
          }
        ptx::mma_commit(&empty[s]);
        if ((it % kPromote) == kPromote - 1 || it == nkb - 1) ptx::mma_commit(&acc_full[b]);
      }
    }
  } else {
    const uint32_t quad = static_cast<uint32_t>(warp & 3);
    float acc[kBN];
#pragma unroll
    for (int j = 0; j < kBN; ++j) acc[j] = 0.f;
    for (int c = 0; c < nchunks; ++c) {
      const int b = c & 1;
      ptx::mbar_wait(&acc_full[b], (c >> 1) & 1);
      ptx::tc_fence_after();
      uint32_t v[32];
      ptx::tmem_ld_32x32b_x32(tmem + ((quad * 32) << 16) + static_cast<uint32_t>(b * kBN), v);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < kBN; ++j) acc[j] = __fadd_rn(acc[j], __uint_as_float(v[j]));
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[b]);
    }
    const int64_t row = static_cast<int64_t>(tile) * kBM + quad * 32 + lane;
    const bool rok = row < p.M;
    if (p.splits > 1 && rok) {
      float4* w = reinterpret_cast<float4*>(p.ws + (static_cast<int64_t>(split) * p.M + row) * kBN);
#pragma unroll
      for (int j = 0; j < kBN / 4; ++j)
        w[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
    bool write = p.splits == 1;
    if (p.splits > 1) {
      // The last CTA of the row tile to arrive sums the partials in split
      // order (its own from registers: the same bits it stored).
      __threadfence();
      asm volatile("bar.sync 1, 128;" ::: "memory");  // the 4 epilogue warps
      if (warp == 2 && lane == 0)
        last_cta = atomicAdd(&p.counters[tile], 1u) == static_cast<unsigned>(p.splits - 1);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      write = last_cta != 0;
      if (write) {
        __threadfence();
        float tot[kBN];
#pragma unroll
        for (int j = 0; j < kBN; ++j) tot[j] = 0.f;
        for (int s2 = 0; s2 < p.splits; ++s2) {
          float part[kBN];
          if (s2 == split) {
#pragma unroll
            for (int j = 0; j < kBN; ++j) part[j] = acc[j];
          } else if (rok) {
            const float4* w = reinterpret_cast<const float4*>(
                p.ws + (static_cast<int64_t>(s2) * p.M + row) * kBN);
#pragma unroll
            for (int j = 0; j < kBN / 4; ++j) {
              const float4 v4 = __ldcg(w + j);
              part[4 * j] = v4.x;
              part[4 * j + 1] = v4.y;
              part[4 * j + 2] = v4.z;
              part[4 * j + 3] = v4.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < kBN; ++j) part[j] = 0.f;
          }
#pragma unroll
          for (int j = 0; j < kBN; ++j) tot[j] += part[j];
        }
#pragma unroll
        for (int j = 0; j < kBN; ++j) acc[j] = tot[j];
        if (warp == 2 && lane == 0) p.counters[tile] = 0u;  // ready for the next launch
      }
    }
    if (write && rok)
      for (int j = 0; j < p.N; ++j) p.c[row * p.ldc + j] = acc[j];
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2 * kBN>(tmem);
  }
}

}  // namespace

struct SkinnyTcPlan {
  SkinnyTcParams params;
  int grid = 0;
};

SkinnyTcPlan* skinny_tc_plan_create(const void* d_bf16, int64_t ldd, const void* const* vt_planes,
                                    int planes, int64_t ldv, float* c, int64_t ldc, int64_t M,
                                    int N, int64_t K, const int* skip, cudaStream_t s) {
  if (N < 1 || N > kBN) throw std::invalid_argument("skinny_tc: N must be in [1, 32]");
  if (planes < 1 || planes > 3) throw std::invalid_argument("skinny_tc: 1..3 planes");
  auto* plan = new SkinnyTcPlan();
  SkinnyTcParams& p = plan->params;
  p.a_map = gemm_tensor_map(d_bf16, M, K, ldd, kBM, 2);
  for (int q = 0; q < planes; ++q) p.b_map[q] = gemm_tensor_map(vt_planes[q], N, K, ldv, kBN, 2);
  p.planes = planes;
  p.c = c;
  p.ldc = ldc;
  p.M = M;
  p.N = N;
  p.kblocks = static_cast<int>((K + kBK - 1) / kBK);
  p.skip = skip;
  int dev = 0, sms = 148;
  check_cuda(cudaGetDevice(&dev), "skinny_tc: device");
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "skinny_tc: SMs");
  const int tiles = static_cast<int>((M + kBM - 1) / kBM);
  // One CTA per SM: split K so that tiles × splits ≤ #SMs, ≥ 2 k-blocks each.
  int splits = std::max(1, std::min(sms / std::max(tiles, 1), p.kblocks / 2));
  p.kb_per = (p.kblocks + splits - 1) / splits;
  splits = (p.kblocks + p.kb_per - 1) / p.kb_per;  // no empty splits
  p.splits = splits;
  p.ws = nullptr;
  p.counters = nullptr;
  if (splits > 1) {
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&p.ws),
                               static_cast<size_t>(splits) * M * kBN * sizeof(float), s),
               "skinny_tc: workspace");
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&p.counters), tiles * sizeof(unsigned), s),
               "skinny_tc: counters");
    check_cuda(cudaMemsetAsync(p.counters, 0, tiles * sizeof(unsigned), s), "skinny_tc: counters");
  }
  plan->grid = tiles * splits;
  static thread_local int attr_device = -1;
  if (attr_device != dev) {
    check_cuda(cudaFuncSetAttribute(skinny_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem)),
               "skinny_tc: smem attribute");
    attr_device = dev;
  }
  return plan;
}

void skinny_tc_plan_destroy(SkinnyTcPlan* plan, cudaStream_t s) {
  if (!plan) return;
  if (plan->params.ws) cudaFreeAsync(plan->params.ws, s);
  if (plan->params.counters) cudaFreeAsync(plan->params.counters, s);
  delete plan;
}

void skinny_tc_launch(const SkinnyTcPlan* plan, cudaStream_t s) {
  skinny_tc_kernel<<<plan->grid, kThreads, kSmem, s>>>(plan->params);
  check_cuda(cudaGetLastError(), "skinny_tc_kernel");
}

}  // namespace gwb
