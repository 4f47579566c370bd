// skinny_tc.cu — GEMM2 of the skinny chain (m ≤ 32, config 3) on the tensor
// cores: G[M×N] = D · Σ_p V_pᵀ with D an exact-bf16 n×n structure matrix
// (0/1 graph) and V_p the three bf16 planes of Vᵀ (N×K, N ≤ 32), i.e. the
// bf16x3 chain with N padded to 32.  The product is a pure stream of D:
// 16 KB of D per 64-wide k-block against 3 × 4 KB of V planes, 12
// tcgen05.mma (M=128, N=32, K=16) per k-block.  D is constant across the
// solve, so it is packed once into the exact shared-memory tile order
// (K-major, 128-B swizzle) and each k-block is one contiguous 16-KB bulk
// copy: with 2-D TMA boxes (128 rows × 128 B scattered at the row pitch) the
// same stream reached only 1.4 TB/s.
//
// One CTA per (128-row tile, K split); the split count fills the SMs with
// one CTA each.  Warp 0: TMA producer over a 6-stage ring; warp 1: MMA
// issuer; warps 2–5: epilogue, one TMEM lane quadrant each.  As in gemm.cu,
// the tensor core's truncating fp32 accumulation is bounded by restarting it
// every 2 k-blocks in one of two TMEM buffers and promoting each chunk into
// fp32 registers with round-to-nearest adds.  The K splits of a row tile run
// as one thread-block cluster: partials stay in shared memory and are summed
// in split order through distributed shared memory (deterministic; no
// workspace, fences or second launch — a global-memory arrival-counter
// version spent 2–7 µs of a ~20 µs launch in that tail).
#include <cooperative_groups.h>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>

#include "gemm.cuh"
#include "narrow.cuh"
#include "ptx.cuh"
#include "skinny.cuh"

namespace gwb {

namespace cg = cooperative_groups;

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
  const uint8_t* a;     // packed D: [tile][k-block] 16-KB swizzled tiles
  const uint8_t* b;     // packed planes: [plane][k-block] 4-KB swizzled tiles
  int planes;
  float* c;
  int64_t ldc;
  int64_t M;
  int N;
  int kblocks, splits, kb_per;
  const int* skip;
  // Fused half-step a (kEpi == 1): the cluster rank that sums rows
  // [rbeg, rend) of G then runs their row update (narrow.cuh) and forms the
  // next GEMM1, Vᵀ planes of (new π)·D_Yᵀ, into `next_b` — a second packed
  // plane buffer, since peers are still streaming `b`.
  BapgDev d;
  const float* dyt;  // D_Yᵀ, N×N fp32 row-major
  int64_t ld_dyt;
  uint16_t* next_b;
  int64_t next_pstride;
};

constexpr int kFuseRows = 32;  // rows per cluster rank in the fused epilogue (splits ≥ 4)

template <int kEpi>
__global__ void __launch_bounds__(kThreads, 1)
    skinny_tc_kernel(const __grid_constant__ SkinnyTcParams p) {
  if (p.skip != nullptr && *p.skip != 0) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t full[kStages], empty[kStages], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) float part[kBM][kBN + 4];  // split-K partial (padded rows)
  // Fused epilogue: this rank's summed rows of G, the fp32 copy of their new
  // π rows, D_Yᵀ.
  __shared__ __align__(16) float gsum[kEpi ? kFuseRows : 1][kBN + 4];
  __shared__ float xs[kEpi ? kFuseRows : 1][kBN + 1];
  __shared__ float bs[kEpi ? kBN : 1][kBN];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const int tile = blockIdx.x / p.splits, split = blockIdx.x % p.splits;
  const int kb0 = split * p.kb_per;
  const int nkb = max(0, min(p.kblocks - kb0, p.kb_per));
  const int nchunks = (nkb + kPromote - 1) / kPromote;

  if (warp == 0 && lane == 0) {
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
        const int64_t kb = kb0 + it;
        ptx::bulk_g2s(st, p.a + (static_cast<int64_t>(tile) * p.kblocks + kb) * kATile, kATile,
                      &full[s]);
        for (int q = 0; q < p.planes; ++q)
          ptx::bulk_g2s(st + kATile + q * kBTile,
                        p.b + (static_cast<int64_t>(q) * p.kblocks + kb) * kBTile, kBTile, &full[s]);
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
    if (p.splits == 1) {
      if (row < p.M)
        for (int j = 0; j < p.N; ++j) p.c[row * p.ldc + j] = acc[j];
    } else {
      float* pr = &part[quad * 32 + lane][0];
#pragma unroll
      for (int j = 0; j < kBN / 4; ++j)
        reinterpret_cast<float4*>(pr)[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
  }
  if (p.splits > 1) {
    // The splits of a row tile form a cluster: rank k sums rows
    // [k·128/S, (k+1)·128/S) of the S partials through distributed shared
    // memory, in split order (deterministic), and writes them coalesced.
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    const int S = p.splits;
    const int rows_per = (kBM + S - 1) / S;
    const int rbeg = split * rows_per, rend = min(kBM, rbeg + rows_per);
    for (int e = threadIdx.x; e < (rend - rbeg) * kBN; e += kThreads) {
      const int r = rbeg + e / kBN, j = e % kBN;
      const int64_t row = static_cast<int64_t>(tile) * kBM + r;
      if (row >= p.M || j >= p.N) continue;
      float sum = 0.f;
      for (int q = 0; q < S; ++q) sum += *cluster.map_shared_rank(&part[r][j], q);
      p.c[row * p.ldc + j] = sum;
      if constexpr (kEpi == 1) gsum[r - rbeg][j] = sum;
    }
    if constexpr (kEpi == 1) {
      for (int e = threadIdx.x; e < kBN * kBN; e += kThreads) {
        const int k = e / kBN, c = e % kBN;
        bs[k][c] = (k < p.N && c < p.N) ? p.dyt[static_cast<int64_t>(k) * p.ld_dyt + c] : 0.f;
      }
    }
    cluster.sync();  // peers may still read this CTA's partials
    if constexpr (kEpi == 1) {
      // Half-step a on this rank's rows (the standalone
      // row_update_warps_kernel's arithmetic, bit for bit), keeping the fp32 rows.
      // Eight lanes per row (N ≤ 32 = 8 lanes × 4 columns), four rows per warp.
      for (int r0 = rbeg; r0 < rend; r0 += kThreads / 8) {
        const int r = r0 + static_cast<int>(threadIdx.x) / 8;
        const int64_t row = static_cast<int64_t>(tile) * kBM + r;
        const bool active = r < rend && row < p.d.n;
        const int rl = active ? r - rbeg : 0;
        dev::narrow_row_update<8>(p.d, row, &gsum[rl][0], lane, active, 1, &xs[rl][0]);
      }
      __syncthreads();
      // GEMM1 of half-step b for the same rows: lane = row, warps over the
      // output columns; k in order with fmaf, the bf16 planes written in
      // GEMM2's packed order (small_k_planes_kernel's arithmetic, skinny.cu).
      const int64_t row = static_cast<int64_t>(tile) * kBM + rbeg + lane;
      if (rbeg + lane < rend && row < p.M) {
        float a[kBN];
#pragma unroll
        for (int k = 0; k < kBN; ++k) a[k] = xs[lane][k];
        for (int c = warp; c < p.N; c += kThreads / 32) {
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < kBN; ++k)
            if (k < p.N) acc = fmaf(a[k], bs[k][c], acc);
          const int64_t off =
              (row >> 6) * 2048 + c * 64 + ((((row >> 3) & 7) ^ (c & 7)) << 3) + (row & 7);
          float x = acc;
          for (int q = 0; q < p.planes; ++q) {
            const __nv_bfloat16 hb = __float2bfloat16_rn(x);
            p.next_b[q * p.next_pstride + off] = __bfloat16_as_ushort(hb);
            x -= __bfloat162float(hb);
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2 * kBN>(tmem);
  }
}

// D (fp32 row-major, exact in bf16) → packed tiles; zero beyond M × K.
__global__ void pack_a_kernel(const float* __restrict__ D, int64_t ld, int64_t M, int64_t K,
                              int kblocks, uint16_t* __restrict__ out) {
  const int64_t t = blockIdx.x;  // tile · kblocks + k-block
  const int64_t mt = t / kblocks, kb = t % kblocks;
  uint16_t* dst = out + t * (kATile / 2);
  for (int idx = threadIdx.x; idx < kBM * kBK; idx += blockDim.x) {
    const int r = idx / kBK, k = idx % kBK;  // k fastest: coalesced reads
    const int64_t gr = mt * kBM + r, gk = kb * kBK + k;
    const float v = (gr < M && gk < K) ? D[gr * ld + gk] : 0.f;
    const int off = r * 64 + ((((k >> 3) & 7) ^ (r & 7)) << 3) + (k & 7);
    dst[off] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
  }
}

}  // namespace

int64_t skinny_tc_packed_a_bytes(int64_t M, int64_t K) {
  return ((M + kBM - 1) / kBM) * ((K + kBK - 1) / kBK) * static_cast<int64_t>(kATile);
}

int64_t skinny_tc_packed_b_elems(int64_t K) { return ((K + kBK - 1) / kBK) * (kBTile / 2); }

void skinny_tc_pack_a(const float* D, int64_t ld, int64_t M, int64_t K, void* out, cudaStream_t s) {
  const int kblocks = static_cast<int>((K + kBK - 1) / kBK);
  const int64_t tiles = (M + kBM - 1) / kBM;
  pack_a_kernel<<<static_cast<unsigned>(tiles * kblocks), 256, 0, s>>>(D, ld, M, K, kblocks,
                                                                       static_cast<uint16_t*>(out));
  check_cuda(cudaGetLastError(), "pack_a_kernel");
}

struct SkinnyTcPlan {
  SkinnyTcParams params;
  int grid = 0;
};

SkinnyTcPlan* skinny_tc_plan_create(const void* a_packed, const void* b_packed, int planes,
                                    float* c, int64_t ldc, int64_t M, int N, int64_t K,
                                    const int* skip, cudaStream_t s) {
  if (N < 1 || N > kBN) throw std::invalid_argument("skinny_tc: N must be in [1, 32]");
  if (planes < 1 || planes > 3) throw std::invalid_argument("skinny_tc: 1..3 planes");
  auto* plan = new SkinnyTcPlan();
  SkinnyTcParams& p = plan->params;
  p.a = static_cast<const uint8_t*>(a_packed);
  p.b = static_cast<const uint8_t*>(b_packed);
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
  // One CTA per SM: split K so that tiles × splits ≤ #SMs, ≥ 2 k-blocks
  // each; the splits of a tile form one cluster (≤ 8, portable).
  int splits = std::max(1, std::min(std::min(sms / std::max(tiles, 1), p.kblocks / 2), 8));
  p.kb_per = (p.kblocks + splits - 1) / splits;
  splits = (p.kblocks + p.kb_per - 1) / p.kb_per;  // no empty splits
  p.splits = splits;
  plan->grid = tiles * splits;
  static thread_local int attr_device = -1;
  if (attr_device != dev) {
    check_cuda(cudaFuncSetAttribute(skinny_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem)),
               "skinny_tc: smem attribute");
    check_cuda(cudaFuncSetAttribute(skinny_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmem)),
               "skinny_tc: smem attribute (fused)");
    attr_device = dev;
  }
  return plan;
}

void skinny_tc_plan_destroy(SkinnyTcPlan* plan, cudaStream_t s) {
  (void)s;
  delete plan;
}

namespace {
template <int kEpi>
void launch_tc(const SkinnyTcPlan* plan, const SkinnyTcParams& params, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(plan->grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  // Not launched with PDL: measured 4% slower at c3 (the skinny chain's
  // kernels are a few µs each; launch.cuh).
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(plan->params.splits);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  check_cuda(cudaLaunchKernelEx(&cfg, skinny_tc_kernel<kEpi>, params), "skinny_tc_kernel");
}
}  // namespace

void skinny_tc_launch(const SkinnyTcPlan* plan, cudaStream_t s) { launch_tc<0>(plan, plan->params, s); }

bool skinny_tc_can_fuse(const SkinnyTcPlan* plan) {
  // Each cluster rank sums ⌈128 / splits⌉ rows; the fused epilogue holds 32.
  return plan->params.splits > 1 &&
         (kBM + plan->params.splits - 1) / plan->params.splits <= kFuseRows;
}

void skinny_tc_launch_fused_a(const SkinnyTcPlan* plan, const BapgDev& d, const float* dyt,
                              int64_t ld_dyt, void* next_b, int64_t next_pstride, cudaStream_t s) {
  if (!skinny_tc_can_fuse(plan)) throw std::logic_error("skinny_tc: fused epilogue needs ≥ 4 K splits");
  SkinnyTcParams params = plan->params;
  params.d = d;
  params.dyt = dyt;
  params.ld_dyt = ld_dyt;
  params.next_b = static_cast<uint16_t*>(next_b);
  params.next_pstride = next_pstride;
  launch_tc<1>(plan, params, s);
}

}  // namespace gwb
