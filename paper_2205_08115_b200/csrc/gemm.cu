// gemm.cu — tcgen05 / TMEM / TMA GEMM for sm_100a, kind::tf32 with optional
// 3xTF32 split-precision passes (see gemm.cuh).
//
// One CTA PAIR (cluster of 2, cta_group::2) per 256×256 output tile; each CTA
// owns 128 rows of the tile (its TMEM lanes) and loads its half of A (128
// rows) and its half of B (128 of the 256 N rows), so per CTA and k-block the
// TMA writes and the MMA reads 32 KB of shared memory instead of 48 KB.
//   warp 0    : TMA producer (both CTAs) — 6-stage ring of {A 128×32, B 128×32}
//               fp32 tiles, 128-B swizzle; completion counted on the LEADER's
//               full barrier (cp.async.bulk.tensor.cta_group::2)
//   warp 1    : TMEM allocation (cta_group::2, 512 columns) and, in the leader
//               only, the single-thread tcgen05.mma.cta_group::2.kind::tf32
//               issuer (M=256, N=256, K=8, 4 per stage); commits multicast to
//               both CTAs' empty / tmem-full barriers
//   warps 2-17: epilogue (both CTAs) — drain each finished K-chunk from TMEM
//               (tcgen05.ld 32x32b) into fp32 registers (RN adds), then scale
//               and store; drain completion is reported to the leader
// Tiles are rasterised in groups of kGroupM row-blocks so concurrently
// resident pairs share A and B panels in L2.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "gemm.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace gwb {

namespace {

constexpr int kBM = 128;                   // rows per CTA
constexpr int kPairM = 2 * kBM;            // rows per CTA pair (MMA M)
constexpr int kBN = 256;                   // columns per tile (MMA N)
constexpr int kBK = 32;                    // 32 fp32 = 128 B = one swizzle row
constexpr int kBK16 = 64;                  // 64 bf16 = 128 B
constexpr int kStages = 6;
constexpr int kGroupM = 8;
constexpr int kEpiWarps = 16;              // 4 lane quadrants × 4 column slices
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr uint32_t kABytes = kBM * kBK * 4;
constexpr size_t smem_bytes(int bn) {
  // stage ring + alignment slack + barriers / TMEM slot (256) + column staging (2·bn floats)
  return kStages * (kABytes + static_cast<size_t>(bn / 2) * kBK * 4) + 1024 + 256 + 8 * bn;
}

// Round-to-nearest split of 8 fp32 values into three planes whose sum is x
// (hi = rn(x), mid = rn(x − hi), lo = rn(x − hi − mid); each difference is
// exact in fp32), as raw bf16 or fp16 bits.  A 2-plane consumer reads hi and
// mid, i.e. rn(x − hi).
__device__ __forceinline__ void split_planes8(const float* x, bool f16, uint16_t (&h)[3][8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float r = x[q];
#pragma unroll
    for (int pl = 0; pl < 3; ++pl) {
      if (f16) {
        const __half v = __float2half_rn(r);
        h[pl][q] = __half_as_ushort(v);
        r -= __half2float(v);
      } else {
        const __nv_bfloat16 v = __float2bfloat16_rn(r);
        h[pl][q] = __bfloat16_as_ushort(v);
        r -= __bfloat162float(v);
      }
    }
  }
}

struct __align__(64) GemmParams {
  CUtensorMap a_map[2];
  CUtensorMap b_map[3];
  int32_t M, N, K;
  int32_t passes;
  int32_t a_sel[3];
  int32_t b_sel[3];
  int32_t tiles_m, tiles_n;  // tiles_m counts 256-row pair tiles
  int32_t chunk;  // k-blocks accumulated in TMEM before promotion to registers
  int32_t kind;   // 0: kind::tf32 (fp32 operands), 1: kind::f16 with bf16
                  // operands, 2: kind::f16 with fp16 operands
  int32_t b_block_k;  // > 0: B maps are 3-D [K/b_block_k][N][b_block_k]
  int32_t c_planes;
  int32_t c_f16;  // output planes are fp16 (else bf16)
  int32_t fused;  // split planes share one stage: {A_0 … A_{a_planes−1}, B_0 … B_{b_planes−1}}
  int32_t a_planes, b_planes;  // fused stage contents (pass p reads A_{a_sel[p]}, B_{b_sel[p]})
  int32_t group_m;  // row tiles per rasterisation group (kGroupM; env GWB_GEMM_GROUP_M)
  uint16_t* c_pl[3];
  float* c;
  float* c_aux;
  int64_t ldc;
  int32_t aux_mode;
  const float* row_scale;
  const float* col_scale;
  const int* skip;
  int32_t accumulate;
  int32_t splits;      // > 1: split-K; partials to ws[split][M][ldw]
  int32_t kb_per_split;
  float* ws;
  int64_t ldw;
  int* counters;       // split-K: per (tile, CTA) arrival counters, in-kernel reduction
  const float* col_bias;  // [N] added before scaling (centred operands)
  double* rs_part;        // [M][rs_stride] fp64 row partial sums of the output
  int32_t rs_stride;      // tiles_n · 4 (one per 64-column slice), 1 with the reduce kernel
  unsigned long long* stamps;  // GWB_GEMM_TIMING: [grid][8] %globaltimer stamps (debug)
  int32_t bulk_store;          // epilogue rows leave SMEM by bulk copies (else coalesced st.global)
  int32_t a_const;             // A tiles of the first ring fill requested before the PDL wait
};

__device__ __forceinline__ float trunc_tf32(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// 3xTF32 low operand x − trunc_tf32(x), pre-rounded to TF32 so the MMA's
// operand truncation reads it exactly (a truncated residual biases every
// product low).
__device__ __forceinline__ float tf32_lo(float x) { return rna_tf32(x - trunc_tf32(x)); }

// The tensor core's fp32 accumulation truncates (measured: relative bias
// ≈ −3.6e-8 per accumulated term, linear in K).  The MMA warp therefore
// restarts accumulation every `chunk` k-blocks in one of two TMEM buffers
// and the epilogue warps add each finished chunk into fp32 registers with
// round-to-nearest adds ("promotion"), bounding the bias by the chunk length.
template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tf32_kernel(const __grid_constant__ GemmParams p) {
  // Tile width BN (MMA N): 256, or 192 / 128 for grids of few tiles (small n).
  constexpr int kBN_ = BN;
  constexpr int kHalfN_ = BN / 2;                        // B rows loaded per CTA
  constexpr int kSlice_ = BN / 4;                        // accumulator columns per epilogue thread
  constexpr uint32_t kBB_ = kHalfN_ * kBK * 4;
  constexpr uint32_t kStageB_ = kABytes + kBB_;          // per CTA
  constexpr uint32_t kTmem_ = BN == 192 ? 512 : 2 * BN;  // double-buffered accumulator (power of 2)

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  float* sA = reinterpret_cast<float*>(smem);
  float* sB = reinterpret_cast<float*>(smem + kStages * kABytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageB_);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2] chunk accumulated (per CTA)
  uint64_t* tempty = tfull + 2;       // [2] chunk drained (leader's counts both CTAs)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = ptx::warp_idx();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;

  // Persistent CTA pairs: pair `pair` processes work items pair, pair +
  // npairs, …  (item = split · tiles + tile; tiles in grouped rasterisation,
  // split-K: one tile sweep per split).  The stage ring and the two TMEM
  // chunk buffers run on across items, so the epilogue's drain and store of
  // one tile overlap the MMAs of the next and the prologue is paid once.
  const int tiles_all = p.tiles_m * p.tiles_n;
  const int npairs = static_cast<int>(gridDim.x >> 1);
  const int pair = static_cast<int>(blockIdx.x >> 1);
  const int per_group = p.group_m * p.tiles_n;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&p.a_map[0]);
    ptx::tma_prefetch(&p.b_map[0]);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 2 * kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  unsigned long long* const stamp = p.stamps ? p.stamps + blockIdx.x * 8 : nullptr;
  auto mark = [&](int k) {
    if (stamp) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      stamp[k] = t;
    }
  };
  if (threadIdx.x == 0) mark(0);
  if (warp == 1) ptx::tmem_alloc_2sm<kTmem_>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) mark(1);

  const int kblk = p.kind ? kBK16 : kBK;  // elements per 128-B k-block
  const int kblocks_all = (p.K + kblk - 1) / kblk;
  const int chunk = p.chunk;
  const uint32_t f_a_bytes = static_cast<uint32_t>(p.a_planes) * kABytes;
  const uint32_t f_stage_bytes = f_a_bytes + static_cast<uint32_t>(p.b_planes) * kBB_;
  const int f_stages = static_cast<int>((kStages * kStageB_) / f_stage_bytes);

  // Coordinates and k-range of work item `item`.
  struct Item {
    int split, tm, tn, kb_begin, kblocks, total, nchunks, a_row, b_row;
  };
  auto item_of = [&](int item) {
    Item t;
    t.split = item / tiles_all;
    const int pid = item - t.split * tiles_all;
    const int group = pid / per_group;
    const int first_m = group * p.group_m;
    const int gsize = min(p.tiles_m - first_m, p.group_m);
    const int in_group = pid % per_group;
    t.tm = first_m + in_group % gsize;
    t.tn = in_group / gsize;
    t.kb_begin = p.splits > 1 ? t.split * p.kb_per_split : 0;
    t.kblocks = p.splits > 1 ? max(0, min(kblocks_all - t.kb_begin, p.kb_per_split)) : kblocks_all;
    // Fused planes: the work item is a k-block carrying every plane pass.
    t.total = p.fused ? t.kblocks : p.passes * t.kblocks;
    t.nchunks = (t.total + chunk - 1) / chunk;
    t.a_row = t.tm * kPairM + static_cast<int>(rank) * kBM;
    t.b_row = t.tn * kBN_ + static_cast<int>(rank) * kHalfN_;
    return t;
  };

  // A constant A operand (the structure matrix) does not depend on the
  // predecessor kernel: the producer requests the A tiles of its first ring
  // fill before the PDL wait (only the expected bytes, no arrival yet; the
  // B tiles and the arrival follow the wait), so the first stage is not a
  // full TMA round trip behind the predecessor's last store.
  const bool elected0 = warp == 0 && ptx::elect_one();
  int pre = 0;
  if (p.a_const && p.fused && elected0 && pair < tiles_all * p.splits) {
    const Item t0 = item_of(pair);
    pre = min(f_stages, t0.total);
    for (int it = 0; it < pre; ++it) {
      const int kb = t0.kb_begin + it;
      const uint32_t fbar = ptx::mapa(&full[it], 0);
      if (leader) ptx::mbar_expect_tx(&full[it], 2 * f_a_bytes);
      for (int pa = 0; pa < p.a_planes; ++pa)
        ptx::tma_load_2d_2sm(smem + it * f_stage_bytes + pa * kABytes, &p.a_map[pa], fbar, kb * kblk,
                             t0.a_row);
    }
  }
  // PDL: the prologue above overlapped the predecessor kernel; nothing it
  // wrote (B operands, the skip flag) is read before this point.
  ptx::griddep_wait();
  if (threadIdx.x == 0) mark(2);
  ptx::griddep_launch();
  const bool skip = p.skip != nullptr && *p.skip != 0;
  const int items = skip ? 0 : tiles_all * p.splits;
  if (skip && pre > 0) {
    // Skipped launch: arrive on the prefetched stages and let their A
    // tiles land before the CTA (and its peer) can exit.
    for (int it = 0; it < pre; ++it) {
      if (leader) {
        ptx::mbar_arrive(&full[it]);
        ptx::mbar_wait(&full[it], 0);
      }
    }
  }

  if (warp == 0) {
    if (elected0) {
      int g = 0;  // stage iterations issued so far (all items)
      for (int item = pair; item < items; item += npairs) {
        const Item t = item_of(item);
        if (p.fused) {
          // One stage per k-block: A once, then every B plane (A is shared by
          // the plane passes, so it crosses L2 → SMEM once instead of per pass).
          for (int it = 0; it < t.total; ++it, ++g) {
            const int s = g % f_stages;
            const uint32_t ph = (g / f_stages) & 1;
            const int kb = t.kb_begin + it;
            const uint32_t fbar = ptx::mapa(&full[s], 0);
            uint8_t* st = smem + s * f_stage_bytes;
            if (g < pre) {  // A already requested before the PDL wait
              if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * (f_stage_bytes - f_a_bytes));
            } else {
              ptx::mbar_wait(&empty[s], ph ^ 1);
              if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * f_stage_bytes);
              for (int pa = 0; pa < p.a_planes; ++pa)
                ptx::tma_load_2d_2sm(st + pa * kABytes, &p.a_map[pa], fbar, kb * kblk, t.a_row);
            }
            for (int pl = 0; pl < p.b_planes; ++pl) {
              void* dst = st + f_a_bytes + pl * kBB_;
              if (p.b_block_k > 0) {
                const int kk = kb * kblk;
                ptx::tma_load_3d_2sm(dst, &p.b_map[pl], fbar, kk % p.b_block_k, t.b_row,
                                     kk / p.b_block_k);
              } else {
                ptx::tma_load_2d_2sm(dst, &p.b_map[pl], fbar, kb * kblk, t.b_row);
              }
            }
          }
        } else {
          for (int it = 0; it < t.total; ++it, ++g) {
            const int s = g % kStages;
            const uint32_t ph = (g / kStages) & 1;
            ptx::mbar_wait(&empty[s], ph ^ 1);
            const int pass = it / t.kblocks;
            const int kb = t.kb_begin + it - pass * t.kblocks;
            const uint32_t fbar = ptx::mapa(&full[s], 0);
            if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * kStageB_);
            ptx::tma_load_2d_2sm(sA + s * (kBM * kBK), &p.a_map[p.a_sel[pass]], fbar, kb * kblk,
                                 t.a_row);
            if (p.b_block_k > 0) {
              const int kk = kb * kblk;
              ptx::tma_load_3d_2sm(sB + s * (kHalfN_ * kBK), &p.b_map[p.b_sel[pass]], fbar,
                                   kk % p.b_block_k, t.b_row, kk / p.b_block_k);
            } else {
              ptx::tma_load_2d_2sm(sB + s * (kHalfN_ * kBK), &p.b_map[p.b_sel[pass]], fbar,
                                   kb * kblk, t.b_row);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && ptx::elect_one()) {
      const uint32_t idesc = p.kind == 2   ? ptx::idesc_f16(kPairM, kBN_)
                             : p.kind == 1 ? ptx::idesc_bf16(kPairM, kBN_)
                                           : ptx::idesc_tf32(kPairM, kBN_);
      int g0 = 0;  // stage iterations of the previous items
      int c = 0;   // chunks of all items so far
      for (int item = pair; item < items; item += npairs) {
        const Item t = item_of(item);
        for (int cc = 0; cc < t.nchunks; ++cc, ++c) {
          const int b = c & 1;
          ptx::mbar_wait(&tempty[b], ((c >> 1) & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t acc = tmem + static_cast<uint32_t>(b * kBN_);
          const int it0 = cc * chunk;
          const int it1 = min(t.total, it0 + chunk);
          if (p.fused) {
            for (int it = it0; it < it1; ++it) {
              const int g = g0 + it;
              const int s = g % f_stages;
              const uint32_t ph = (g / f_stages) & 1;
              ptx::mbar_wait(&full[s], ph);
              if (g == 0) mark(3);
              ptx::tc_fence_after();
              const uint32_t st_base = ptx::smem_u32(smem + s * f_stage_bytes);
              // Smallest pass first (the last pass index is the smallest
              // product): the tensor core's truncating accumulation then acts
              // on the hi-plane terms only (as in batched.cu).
              for (int pl = p.passes - 1; pl >= 0; --pl) {
                const uint32_t a_base = st_base + p.a_sel[pl] * kABytes;
                const uint32_t b_base = st_base + f_a_bytes + p.b_sel[pl] * kBB_;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint64_t ad = ptx::umma_desc_sw128(a_base + k * 32);
                  const uint64_t bd = ptx::umma_desc_sw128(b_base + k * 32);
                  const uint32_t accum = (it != it0 || pl != p.passes - 1 || k != 0) ? 1u : 0u;
                  ptx::mma_bf16_2sm(acc, ad, bd, idesc, accum);
                }
              }
              ptx::mma_commit_2sm(&empty[s], 0x3);
            }
          } else {
            for (int it = it0; it < it1; ++it) {
              const int g = g0 + it;
              const int s = g % kStages;
              const uint32_t ph = (g / kStages) & 1;
              ptx::mbar_wait(&full[s], ph);
              ptx::tc_fence_after();
              const uint32_t a_base = ptx::smem_u32(sA + s * (kBM * kBK));
              const uint32_t b_base = ptx::smem_u32(sB + s * (kHalfN_ * kBK));
              // 4 MMAs per 128-B k-block: K = 8 (tf32) or 16 (bf16), +32 B each.
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const uint64_t ad = ptx::umma_desc_sw128(a_base + k * 32);
                const uint64_t bd = ptx::umma_desc_sw128(b_base + k * 32);
                const uint32_t accum = (it != it0 || k != 0) ? 1u : 0u;
                if (p.kind) ptx::mma_bf16_2sm(acc, ad, bd, idesc, accum);
                else ptx::mma_tf32_2sm(acc, ad, bd, idesc, accum);
              }
              ptx::mma_commit_2sm(&empty[s], 0x3);
            }
          }
          ptx::mma_commit_2sm(&tfull[b], 0x3);
        }
        g0 += t.total;
      }
      mark(4);
    }
  } else {
    // Epilogue: warp w (2..17) owns TMEM lanes 32·(w%4).. and columns
    // [64·slice, 64·slice + 64) of this CTA's 128×256 accumulator.
    const uint32_t quad = warp & 3;
    const uint32_t slice = (warp - 2) >> 2;
    const uint32_t lane_base = quad * 32;
    const uint32_t col_base = slice * kSlice_;
    const uint32_t tempty_leader[2] = {ptx::mapa(&tempty[0], 0), ptx::mapa(&tempty[1], 0)};
    // The tile's column bias / scale are staged in shared memory while the
    // MMAs run, so the final epilogue reads them at SMEM latency instead of
    // from L2 on the kernel's tail (named barrier 2: the 16 epilogue warps).
    float* s_cb = reinterpret_cast<float*>(tmem_slot + 4);  // [kBN_]
    float* s_cs = s_cb + kBN_;                              // [kBN_]
    const bool stage_cols = p.splits == 1 && (p.col_bias != nullptr || p.col_scale != nullptr);
    int c = 0;
    for (int item = pair; item < items; item += npairs) {
      const Item t = item_of(item);
      const int split = t.split, tn = t.tn, a_row = t.a_row;
      if (stage_cols) {
        ptx::named_barrier_sync(2, 32 * kEpiWarps);  // previous tile's epilogue done
        for (int j = static_cast<int>(threadIdx.x) - 64; j < kBN_; j += 32 * kEpiWarps) {
          const int col = tn * kBN_ + j;
          s_cb[j] = p.col_bias != nullptr && col < p.N ? __ldg(p.col_bias + col) : 0.0f;
          s_cs[j] = p.col_scale != nullptr ? (col < p.N ? __ldg(p.col_scale + col) : 0.0f) : 1.0f;
        }
        ptx::named_barrier_sync(2, 32 * kEpiWarps);
      }
      float acc[kSlice_];
#pragma unroll
      for (int j = 0; j < kSlice_; ++j) acc[j] = 0.0f;
      for (int cc = 0; cc < t.nchunks; ++cc, ++c) {
        const int b = c & 1;
        ptx::mbar_wait(&tfull[b], (c >> 1) & 1);
        ptx::tc_fence_after();
        const uint32_t taddr = tmem + (lane_base << 16) + static_cast<uint32_t>(b * kBN_) + col_base;
#pragma unroll
        for (int h = 0; h < kSlice_ / 32; ++h) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(taddr + h * 32, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 32; ++j) acc[h * 32 + j] = __fadd_rn(acc[h * 32 + j], __uint_as_float(v[j]));
        }
        if constexpr (kSlice_ % 32 != 0) {  // BN = 192: 48 columns = 32 + 16
          constexpr int h0 = kSlice_ / 32 * 32;
          uint32_t v[16];
          ptx::tmem_ld_32x32b_x16(taddr + h0, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[h0 + j] = __fadd_rn(acc[h0 + j], __uint_as_float(v[j]));
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader[b]);
      }
      if (warp == 2 && lane == 0) mark(5);
      const int row = a_row + static_cast<int>(lane_base + lane);
      // Coalesced stores (one pair per tile, i.e. the stage ring is idle once
      // the last chunk is drained): each warp transposes its 32 rows × kSlice_
      // columns through shared memory and writes whole row segments, instead
      // of one 16-B piece of 32 different rows per instruction.
      const bool staged = npairs >= items && p.counters == nullptr;
      float* const sw = reinterpret_cast<float*>(smem) + (warp - 2) * 32 * (kSlice_ + 4);
      auto stage_rows = [&]() {
        float* r = sw + lane * (kSlice_ + 4);
#pragma unroll
        for (int j = 0; j < kSlice_; j += 4) *reinterpret_cast<float4*>(r + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        __syncwarp();
      };
      if (staged && p.splits > 1) {
        // Split-K: raw partial sums to the workspace (reduced by the next kernel).
        stage_rows();
        const int col0w = tn * kBN_ + static_cast<int>(col_base);
        constexpr int cpr = kSlice_ / 4;
        for (int idx = lane; idx < 32 * cpr; idx += 32) {
          const int r = idx / cpr, ch = idx - r * cpr;
          const int grow = a_row + static_cast<int>(lane_base) + r;
          const int col = col0w + 4 * ch;
          if (grow < p.M && col < p.ldw)
            *reinterpret_cast<float4*>(p.ws + static_cast<int64_t>(split) * p.M * p.ldw +
                                       static_cast<int64_t>(grow) * p.ldw + col) =
                *reinterpret_cast<const float4*>(sw + r * (kSlice_ + 4) + 4 * ch);
        }
        __syncwarp();
        continue;
      }
      if (p.splits > 1) {
        // Split-K: raw partial sums to the workspace; the CTA that completes
        // the tile's last split (per-tile arrival counter) then sums the
        // partials in split order — the fixed order of the standalone reduce
        // kernel, so results are bitwise the same — and runs the epilogue.
        const int col0 = tn * kBN_ + static_cast<int>(col_base);
        if (row < p.M) {
          float* wrow = p.ws + static_cast<int64_t>(split) * p.M * p.ldw + static_cast<int64_t>(row) * p.ldw;
#pragma unroll
          for (int j = 0; j < kSlice_; j += 4)
            if (col0 + j < p.ldw)
              *reinterpret_cast<float4*>(wrow + col0 + j) =
                  make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        }
        if (p.counters == nullptr) continue;  // standalone reduce kernel follows
        __threadfence();
        ptx::named_barrier_sync(1, 32 * kEpiWarps);
        __shared__ int s_last;
        int* cnt = p.counters + (item - split * tiles_all) * 2 + static_cast<int>(rank);
        if (warp == 2 && lane == 0) s_last = atomicAdd(cnt, 1) == p.splits - 1;
        ptx::named_barrier_sync(1, 32 * kEpiWarps);
        if (!s_last) continue;
        __threadfence();
        if (warp == 2 && lane == 0) *cnt = 0;  // every split arrived: ready for the next launch
        if (row < p.M) {
#pragma unroll
          for (int j = 0; j < kSlice_; ++j) acc[j] = 0.0f;
          for (int sp = 0; sp < p.splits; ++sp) {
            const float* w = p.ws + static_cast<int64_t>(sp) * p.M * p.ldw +
                             static_cast<int64_t>(row) * p.ldw + col0;
#pragma unroll
            for (int j = 0; j < kSlice_; j += 4) {
              if (col0 + j < p.ldw) {
                const float4 v = __ldcg(reinterpret_cast<const float4*>(w + j));
                acc[j] = __fadd_rn(acc[j], v.x);
                acc[j + 1] = __fadd_rn(acc[j + 1], v.y);
                acc[j + 2] = __fadd_rn(acc[j + 2], v.z);
                acc[j + 3] = __fadd_rn(acc[j + 3], v.w);
              }
            }
          }
        }
      }
      if (row < p.M) {
        const float rs = p.row_scale != nullptr ? p.row_scale[row] : 1.0f;
        const bool round_out = p.aux_mode == 1;
        const int col0 = tn * kBN_ + static_cast<int>(col_base);
        if (stage_cols) {
  #pragma unroll
          for (int j = 0; j < kSlice_; ++j) {
            float a = acc[j];
            if (p.col_bias != nullptr) a = __fadd_rn(a, s_cb[col_base + j]);
            float x = a * rs;
            if (p.col_scale != nullptr) x *= s_cs[col_base + j];
            acc[j] = round_out ? rna_tf32(x) : x;
          }
        } else {
  #pragma unroll
          for (int j = 0; j < kSlice_; ++j) {
            float a = acc[j];
            if (p.col_bias != nullptr) a = __fadd_rn(a, (col0 + j < p.N) ? __ldg(p.col_bias + col0 + j) : 0.0f);
            float x = a * rs;
            if (p.col_scale != nullptr) x *= (col0 + j < p.N) ? __ldg(p.col_scale + col0 + j) : 0.0f;
            acc[j] = round_out ? rna_tf32(x) : x;
          }
        }
        if (p.rs_part != nullptr) {
          double s = 0.0;
  #pragma unroll
          for (int j = 0; j < kSlice_; ++j)
            if (col0 + j < p.N) s += static_cast<double>(acc[j]);
          p.rs_part[static_cast<int64_t>(row) * p.rs_stride + tn * 4 + static_cast<int>(slice)] = s;
        }
      }
      const int col0w_ = tn * kBN_ + static_cast<int>(col_base);
      if (staged && p.bulk_store && !p.accumulate && p.c_planes <= 2 && col0w_ + kSlice_ <= p.N) {
        // Whole row segments: each lane stages its own row (fp32, or the
        // split planes) and one bulk copy per row and output array streams it
        // to global memory asynchronously.
        const bool planes = p.c_planes > 0;
        const bool aligned = planes ? (p.ldc & 7) == 0 : (p.ldc & 3) == 0;
        if (aligned) {
          if (row < p.M) {
            uint8_t* my = reinterpret_cast<uint8_t*>(sw + lane * (kSlice_ + 4));
            if (planes) {
              // planes back to back in the row's slot: kSlice_ fp16 each
#pragma unroll
              for (int j0 = 0; j0 < kSlice_; j0 += 8) {
                __align__(16) uint16_t h[3][8];
                split_planes8(acc + j0, p.c_f16 != 0, h);
                for (int pl = 0; pl < p.c_planes; ++pl)
                  *reinterpret_cast<uint4*>(my + pl * kSlice_ * 2 + j0 * 2) = *reinterpret_cast<const uint4*>(h[pl]);
              }
            } else {
#pragma unroll
              for (int j = 0; j < kSlice_; j += 4)
                *reinterpret_cast<float4*>(my + j * 4) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            }
            ptx::fence_proxy_async();
            const int64_t off = static_cast<int64_t>(row) * p.ldc + col0w_;
            if (planes) {
              for (int pl = 0; pl < p.c_planes; ++pl)
                ptx::bulk_s2g(p.c_pl[pl] + off, my + pl * kSlice_ * 2, kSlice_ * 2);
            } else {
              ptx::bulk_s2g(p.c + off, my, kSlice_ * 4);
            }
            ptx::bulk_commit();
            if (!planes && p.aux_mode == 2) {
              // second array (3xTF32 residual operand) after the first left SMEM
              ptx::bulk_wait_all();
#pragma unroll
              for (int j = 0; j < kSlice_; j += 4)
                *reinterpret_cast<float4*>(my + j * 4) =
                    make_float4(tf32_lo(acc[j]), tf32_lo(acc[j + 1]), tf32_lo(acc[j + 2]), tf32_lo(acc[j + 3]));
              ptx::fence_proxy_async();
              ptx::bulk_s2g(p.c_aux + off, my, kSlice_ * 4);
              ptx::bulk_commit();
            }
            ptx::bulk_wait_all();
          }
          continue;
        }
      }
      if (staged) {
        stage_rows();
        const int col0w = tn * kBN_ + static_cast<int>(col_base);
        if (p.c_planes > 0) {
          constexpr int cpr = kSlice_ / 8;
          for (int idx = lane; idx < 32 * cpr; idx += 32) {
            const int r = idx / cpr, ch = idx - r * cpr;
            const int grow = a_row + static_cast<int>(lane_base) + r;
            const int col = col0w + 8 * ch;
            if (grow >= p.M || col >= p.N) continue;
            __align__(16) uint16_t h[3][8];
            split_planes8(sw + r * (kSlice_ + 4) + 8 * ch, p.c_f16 != 0, h);
            const int64_t off = static_cast<int64_t>(grow) * p.ldc + col;
            const bool vec = col + 8 <= p.N && (p.ldc & 7) == 0;
            for (int pl = 0; pl < p.c_planes; ++pl) {
              uint16_t* dst = p.c_pl[pl] + off;
              if (vec) {
                *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(h[pl]);
              } else {
                for (int q = 0; q < 8; ++q)
                  if (col + q < p.N) dst[q] = h[pl][q];
              }
            }
          }
        } else {
          constexpr int cpr = kSlice_ / 4;
          float* clo_base = p.aux_mode == 2 ? p.c_aux : nullptr;
          for (int idx = lane; idx < 32 * cpr; idx += 32) {
            const int r = idx / cpr, ch = idx - r * cpr;
            const int grow = a_row + static_cast<int>(lane_base) + r;
            const int col = col0w + 4 * ch;
            if (grow >= p.M || col >= p.N) continue;
            float4 v = *reinterpret_cast<const float4*>(sw + r * (kSlice_ + 4) + 4 * ch);
            float* crow = p.c + static_cast<int64_t>(grow) * p.ldc;
            float* clo = clo_base ? clo_base + static_cast<int64_t>(grow) * p.ldc : nullptr;
            if (col + 4 <= p.N && (p.ldc & 3) == 0) {
              if (p.accumulate) {
                const float4 o = *reinterpret_cast<const float4*>(crow + col);
                v = make_float4(__fadd_rn(o.x, v.x), __fadd_rn(o.y, v.y), __fadd_rn(o.z, v.z), __fadd_rn(o.w, v.w));
              }
              *reinterpret_cast<float4*>(crow + col) = v;
              if (clo)
                *reinterpret_cast<float4*>(clo + col) =
                    make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
            } else {
              const float f[4] = {v.x, v.y, v.z, v.w};
              for (int q = 0; q < 4; ++q) {
                if (col + q >= p.N) break;
                const float x = p.accumulate ? __fadd_rn(crow[col + q], f[q]) : f[q];
                crow[col + q] = x;
                if (clo) clo[col + q] = tf32_lo(x);
              }
            }
          }
        }
        __syncwarp();
        continue;
      }
      if (row < p.M) {
        const int col0 = tn * kBN_ + static_cast<int>(col_base);
        float* crow = p.c + static_cast<int64_t>(row) * p.ldc;
        float* clo = p.aux_mode == 2 ? p.c_aux + static_cast<int64_t>(row) * p.ldc : nullptr;
        if (p.c_planes > 0) {
          // Split planes (RN): x ≈ hi + mid (+ lo), bf16 or fp16, for a
          // split-operand GEMM.
          const int64_t off = static_cast<int64_t>(row) * p.ldc + col0;
          const bool vec = col0 + kSlice_ <= p.N && (p.ldc & 7) == 0;
  #pragma unroll
          for (int j0 = 0; j0 < kSlice_; j0 += 8) {
            __align__(16) uint16_t h[3][8];
            split_planes8(acc + j0, p.c_f16 != 0, h);
            for (int pl = 0; pl < p.c_planes; ++pl) {
              uint16_t* dst = p.c_pl[pl] + off + j0;
              if (vec) {
                *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(h[pl]);
              } else {
                for (int q = 0; q < 8; ++q)
                  if (col0 + j0 + q < p.N) dst[q] = h[pl][q];
              }
            }
          }
        } else if (col0 + kSlice_ <= p.N && (p.ldc & 3) == 0) {
  #pragma unroll
          for (int j = 0; j < kSlice_; j += 4) {
            if (p.accumulate) {
              const float4 o = *reinterpret_cast<const float4*>(crow + col0 + j);
              acc[j] = __fadd_rn(o.x, acc[j]);
              acc[j + 1] = __fadd_rn(o.y, acc[j + 1]);
              acc[j + 2] = __fadd_rn(o.z, acc[j + 2]);
              acc[j + 3] = __fadd_rn(o.w, acc[j + 3]);
            }
            *reinterpret_cast<float4*>(crow + col0 + j) =
                make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            if (clo)
              *reinterpret_cast<float4*>(clo + col0 + j) = make_float4(
                  tf32_lo(acc[j]), tf32_lo(acc[j + 1]), tf32_lo(acc[j + 2]), tf32_lo(acc[j + 3]));
          }
        } else {
  #pragma unroll
          for (int j = 0; j < kSlice_; ++j) {
            if (col0 + j < p.N) {
              if (p.accumulate) acc[j] = __fadd_rn(crow[col0 + j], acc[j]);
              crow[col0 + j] = acc[j];
              if (clo) clo[col0 + j] = tf32_lo(acc[j]);
            }
          }
        }
      }
    }
  }

  if (warp == 2 && lane == 0) mark(6);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_2sm<kTmem_>(tmem);
  }
  if (threadIdx.x == 0) mark(7);
}

// Split-K reduction + epilogue: one CTA per output row, fixed summation order
// over the splits, then the same output modes as the GEMM epilogue.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const __grid_constant__ GemmParams p) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  if (p.skip != nullptr && *p.skip != 0) return;
  const int row = blockIdx.x;
  const float rs = p.row_scale != nullptr ? p.row_scale[row] : 1.0f;
  double rsum = 0.0;  // row sum of the output (rs_part)
  // ldw (a multiple of 8) and ldc (of 32) and 256-B aligned buffers make
  // every 8-column group 16-B aligned (fp32 float4 pairs, bf16 uint4).
  for (int c0 = threadIdx.x * 8; c0 < p.N; c0 += blockDim.x * 8) {
    float x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = 0.0f;
    // Splits in order; 4 at a time with all their loads in flight.
    for (int s0 = 0; s0 < p.splits; s0 += 4) {
      float4 v[4][2];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (s0 + t < p.splits) {
          const float4* w = reinterpret_cast<const float4*>(
              p.ws + static_cast<int64_t>(s0 + t) * p.M * p.ldw + static_cast<int64_t>(row) * p.ldw + c0);
          v[t][0] = __ldcs(w);
          v[t][1] = __ldcs(w + 1);
        }
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (s0 + t >= p.splits) break;
        const float f[8] = {v[t][0].x, v[t][0].y, v[t][0].z, v[t][0].w,
                            v[t][1].x, v[t][1].y, v[t][1].z, v[t][1].w};
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = __fadd_rn(x[q], f[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float a = x[q];
      if (p.col_bias != nullptr) a = __fadd_rn(a, (c0 + q < p.N) ? p.col_bias[c0 + q] : 0.0f);
      float v = a * rs;
      if (p.col_scale != nullptr) v *= (c0 + q < p.N) ? p.col_scale[c0 + q] : 0.0f;
      x[q] = p.aux_mode == 1 ? rna_tf32(v) : v;
      if (c0 + q < p.N) rsum += static_cast<double>(x[q]);
    }
    const int64_t off = static_cast<int64_t>(row) * p.ldc + c0;
    const bool full = c0 + 8 <= p.N;
    if (p.c_planes > 0) {
      alignas(16) uint16_t h[3][8];
      split_planes8(x, p.c_f16 != 0, h);
      for (int pl = 0; pl < p.c_planes; ++pl) {
        if (full) {
          *reinterpret_cast<uint4*>(p.c_pl[pl] + off) = *reinterpret_cast<const uint4*>(h[pl]);
        } else {
          for (int q = 0; q < 8 && c0 + q < p.N; ++q) p.c_pl[pl][off + q] = h[pl][q];
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (c0 + q >= p.N) continue;
        float v = x[q];
        if (p.accumulate) v = __fadd_rn(p.c[off + q], v);
        p.c[off + q] = v;
        if (p.aux_mode == 2) p.c_aux[off + q] = tf32_lo(v);
      }
    }
  }
  if (p.rs_part != nullptr) {
    // Fixed-order block sum: warp butterflies, then warps in order.
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
      p.rs_part[static_cast<int64_t>(row) * p.rs_stride] = t;
    }
  }
}

// out[i] = factor · Σ_k rs_part[i][k] (fixed order), rounded to fp32.
__global__ void rowsum_bias_kernel(const __grid_constant__ GemmParams p, double factor, float* out) {
  ptx::griddep_wait();
  ptx::griddep_launch();
  if (p.skip != nullptr && *p.skip != 0) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p.M) return;
  const double* r = p.rs_part + static_cast<int64_t>(i) * p.rs_stride;
  double t = 0.0;
  for (int k = 0; k < p.rs_stride; ++k) t += r[k];
  out[i] = static_cast<float>(factor * t);
}

// ---- host side ---------------------------------------------------------------

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}

// Row-major rows×cols matrix (leading dim ld elements) of fp32 (esize 4) or
// bf16 (esize 2); box = box_rows × 128 B.
CUtensorMap make_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                     int esize = 4) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  if ((ld * esize) % 16 != 0 || (reinterpret_cast<uintptr_t>(ptr) & 15) != 0)
    throw std::runtime_error("gemm: TMA needs 16-B aligned base and row pitch");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esize};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esize), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                          : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(ptr), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld ld=%lld",
                  static_cast<int>(r), (long long)rows, (long long)cols, (long long)ld);
    throw std::runtime_error(buf);
  }
  return m;
}

// Blocked-K operand [blocks][rows][block_k] (contiguous), box = box_rows ×
// 128 B within one block.
CUtensorMap make_map_blocked(const void* ptr, int64_t rows, int64_t block_k, int64_t blocks,
                             int box_rows, int esize, int64_t block_stride = 0) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  if (block_stride == 0) block_stride = block_k * rows;
  if ((block_k * esize) % 16 != 0 || (block_stride * esize) % 16 != 0 ||
      (reinterpret_cast<uintptr_t>(ptr) & 15) != 0)
    throw std::runtime_error("gemm: blocked TMA needs 16-B aligned base and block pitch");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(block_k), static_cast<cuuint64_t>(rows),
                        static_cast<cuuint64_t>(blocks)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(block_k) * esize,
                           static_cast<cuuint64_t>(block_stride) * esize};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(128 / esize), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                          : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           3, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (3-D) failed");
  return m;
}

}  // namespace

CUtensorMap gemm_tensor_map(const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                            int esize) {
  return make_map(ptr, rows, cols, ld, box_rows, esize);
}

// GWB_GEMM_TIMING=1 (debug): every launch writes per-CTA %globaltimer
// stamps (entry, prologue done, PDL wait done, first stage, last MMA, last
// chunk drained, stores done, exit) to one device buffer that
// gwb_debug_gemm_stamps() copies out.
unsigned long long* g_stamps = nullptr;
int g_stamps_grid = 0;
unsigned long long* stamps_buffer() {
  static const bool on = std::getenv("GWB_GEMM_TIMING") != nullptr;
  if (!on) return nullptr;
  if (!g_stamps && cudaMalloc(&g_stamps, sizeof(unsigned long long) * 8 * 1024) != cudaSuccess)
    g_stamps = nullptr;
  return g_stamps;
}

struct GemmPlan {
  GemmParams params;
  int grid = 0;
  int bn = 256;  // tile width (MMA N): 256, or 128 for grids of few tiles
  double flops = 0.0;
  float* ws = nullptr;  // split-K workspace (owned)
  int* counters = nullptr;
  double* rs_part = nullptr;  // row partial sums (owned)
  ~GemmPlan() {
    if (ws) cudaFree(ws);
    if (counters) cudaFree(counters);
    if (rs_part) cudaFree(rs_part);
  }
};

GemmPlan* gemm_plan_create(const GemmDesc& d) {
  // Per current device (attributes are per device context); cheap, and plans
  // are created once per solve.
  cudaFuncSetAttribute(gemm_tf32_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem_bytes(256)));
  cudaFuncSetAttribute(gemm_tf32_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem_bytes(128)));
  cudaFuncSetAttribute(gemm_tf32_kernel<192>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem_bytes(192)));
  cudaFuncSetAttribute(gemm_tf32_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem_bytes(64)));
  auto* p = new GemmPlan();
  // Tile width for grids of a few waves (n ≲ 4000): the width among 256 /
  // 192 / 128 that minimises waves × width (the time of one pair's tiles)
  // over the 74 SM pairs, e.g. c2's 48 tiles of 256 (65% of the pairs) become
  // 64-66 tiles of 192 (c1: 32 tiles of 128).  Large grids keep 256 (best
  // operand reuse).  GWB_GEMM_BN=64/128/192/256 forces (A/B).
  {
    static const int bn_env = [] {
      const char* e = std::getenv("GWB_GEMM_BN");
      return e ? std::atoi(e) : 0;
    }();
    const int64_t tm = (d.M + kPairM - 1) / kPairM;
    auto cost = [&](int bn) { return (tm * ((d.N + bn - 1) / bn) + 73) / 74 * bn; };
    int bn = 256;
    if (tm * ((d.N + 255) / 256) <= 4 * 74) {
      if (cost(192) < cost(bn)) bn = 192;
      if (cost(128) < cost(bn)) bn = 128;
      // 64 wide where it fills more than half of the SM pairs in one wave
      // with no split-K (c1: 64 tiles): the K loop is twice as long as with
      // 128-wide tiles split in two, but the four reduce launches per
      // iteration go (c1 9.95K -> 10.45K it/s, alternating runs).
      const int64_t t64 = tm * ((d.N + 63) / 64);
      if (cost(64) < cost(bn) && t64 > 37 && t64 <= 74 && d.split_k == 0) bn = 64;
    }
    p->bn = bn_env == 64 || bn_env == 128 || bn_env == 192 || bn_env == 256 ? bn_env : bn;
  }
  const int halfn = p->bn / 2;
  GemmParams& g = p->params;
  std::memset(&g, 0, sizeof(g));
  g.M = static_cast<int32_t>(d.M);
  g.N = static_cast<int32_t>(d.N);
  g.K = static_cast<int32_t>(d.K);
  g.passes = 1;
  g.a_sel[0] = 0;
  g.b_sel[0] = 0;
  if (d.bf16_planes > 0) {
    // Σ_p A·B_p over bf16 (or fp16) planes (A exact in that format).
    g.kind = d.f16 ? 2 : 1;
    g.a_map[0] = make_map(d.a_bf16, d.M, d.K, d.lda, kBM, 2);
    g.a_map[1] = g.a_map[0];
    for (int pl = 0; pl < d.bf16_planes; ++pl) {
      g.b_map[pl] = d.b_block_k > 0
                        ? make_map_blocked(d.b_bf16[pl], d.N, d.b_block_k, d.K / d.b_block_k,
                                           halfn, 2, d.b_block_stride)
                        : make_map(d.b_bf16[pl], d.N, d.K, d.ldb, halfn, 2);
      g.a_sel[pl] = 0;
      g.b_sel[pl] = pl;
    }
    g.passes = d.bf16_planes;
    if (d.a_bf16_lo) {
      // f16x3: A and B both split in two planes; the lo·lo term is dropped.
      if (d.bf16_planes != 2) throw std::runtime_error("gemm: split A needs two B planes");
      g.a_map[1] = make_map(d.a_bf16_lo, d.M, d.K, d.lda, kBM, 2);
      g.a_sel[0] = 0;  // hi·hi
      g.b_sel[0] = 0;
      g.a_sel[1] = 0;  // hi·lo
      g.b_sel[1] = 1;
      g.a_sel[2] = 1;  // lo·hi (smallest: issued first in the fused schedule)
      g.b_sel[2] = 0;
      g.passes = 3;
    }
  } else {
  auto bmap = [&](const float* b) {
    return d.b_block_k > 0 ? make_map_blocked(b, d.N, d.b_block_k, d.K / d.b_block_k, halfn, 4,
                                              d.b_block_stride)
                           : make_map(b, d.N, d.K, d.ldb, halfn);
  };
  g.a_map[0] = make_map(d.a, d.M, d.K, d.lda, kBM);
  g.b_map[0] = bmap(d.b);
  g.a_map[1] = d.a_lo ? make_map(d.a_lo, d.M, d.K, d.lda, kBM) : g.a_map[0];
  g.b_map[1] = d.b_lo ? bmap(d.b_lo) : g.b_map[0];
  g.b_map[2] = g.b_map[0];
  if (d.three_pass) {
    // A·B + A·B_lo + A_lo·B; a missing residual means that operand is exact
    // in TF32 (e.g. 0/1 adjacency), so its pass is dropped.
    if (d.b_lo) {
      g.a_sel[g.passes] = 0;
      g.b_sel[g.passes] = 1;
      ++g.passes;
    }
    if (d.a_lo) {
      g.a_sel[g.passes] = 1;
      g.b_sel[g.passes] = 0;
      ++g.passes;
    }
  }
  }
  g.tiles_m = static_cast<int32_t>((d.M + kPairM - 1) / kPairM);
  g.tiles_n = static_cast<int32_t>((d.N + p->bn - 1) / p->bn);
  g.chunk = d.promote_every > 0 ? d.promote_every : 1 << 30;
  static const int group_env = [] {
    const char* e = std::getenv("GWB_GEMM_GROUP_M");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  g.group_m = group_env > 0 ? group_env : kGroupM;
  // Split planes share one pipeline stage (A loaded once per k-block).
  // Promotion chunk: 2·promote_every k-blocks of all planes (4: 256 K
  // elements, 32 MMAs for f16x2).  Short chunks leave the MMA warp waiting
  // on the epilogue drain: c4 8.86 / 10.45 / 11.21 / 11.56 it/s at 1 / 2 /
  // 3 / 4 k-blocks (one box).  Truncation bias of the chunk, measured with
  // all-positive terms at K = 20000 (tools/acc_probe.py): mean −2.0e-7,
  // max 6.7e-7 relative at 4 k-blocks (f16x2), vs −4.5e-8 / 5.7e-7 at 1.
  static const bool unfused_env = std::getenv("GWB_GEMM_UNFUSED") != nullptr;
  // Split A (f16x3) keeps separate pass stages: its fused 3-pass chunks
  // accumulate 48 MMAs per promotion and measured a 3× larger truncation
  // bias (−1.5e-6 vs −4.6e-7 relative at K = 2048, tests/test_gpu_gemm.py).
  if (d.bf16_planes >= 2 && d.fuse_planes && !unfused_env && (!d.a_bf16_lo || d.fuse_split_a)) {
    g.fused = 1;
    g.a_planes = d.a_bf16_lo ? 2 : 1;
    g.b_planes = d.bf16_planes;
    // Split A (centred f16x3): promotion every promote_every k-blocks (c2,
    // 2 vs 4: same speed, objective error 1.4e-7 vs 3.5e-7).
    if (d.promote_every > 0) g.chunk = (d.a_bf16_lo ? 1 : 2) * d.promote_every;
    // A/B knob: k-blocks per promotion chunk in the fused schedule.
    static const int chunk_env = [] {
      const char* e = std::getenv("GWB_GEMM_CHUNK_KB");
      return e ? std::max(1, std::atoi(e)) : 0;
    }();
    if (chunk_env > 0) g.chunk = chunk_env;
  }
  g.b_block_k = static_cast<int32_t>(d.b_block_k);
  if (d.b_block_k > 0 &&
      (d.K % d.b_block_k != 0 || d.b_block_k % (d.bf16_planes > 0 ? kBK16 : kBK) != 0))
    throw std::runtime_error("gemm: blocked K must tile K and be a multiple of the k-block");
  g.c = d.c;
  g.c_aux = d.c_aux;
  g.ldc = d.ldc;
  g.aux_mode = d.aux_mode;
  g.c_planes = d.c_planes;
  g.c_f16 = d.f16 ? 1 : 0;
  for (int pl = 0; pl < 3; ++pl) g.c_pl[pl] = static_cast<uint16_t*>(d.c_bf16[pl]);
  g.row_scale = d.row_scale;
  g.col_scale = d.col_scale;
  g.col_bias = d.col_bias;
  g.accumulate = d.accumulate ? 1 : 0;
  g.skip = d.skip;
  // Split-K when one sweep of pair tiles leaves most of the 74 SM pairs idle
  // (n ≲ 2000): each split keeps ≥ 4 k-blocks, the grid stays one wave.
  // (Splitting a grid that already fills a wave loses: measured at config 2,
  // 48 pair tiles, S = 3 — 2479 → 2113 it/s — the per-tile prologue and
  // epilogue do not shrink with K.)
  const int tiles = g.tiles_m * g.tiles_n;
  const int kblocks = (g.K + (g.kind ? kBK16 : kBK) - 1) / (g.kind ? kBK16 : kBK);
  int splits = 1;
  // A/B knob (recorded by bench.py): GWB_GEMM_SPLITK=1 disables split-K,
  // ≥ 2 forces that many splits.
  static const int splitk_env = [] {
    const char* e = std::getenv("GWB_GEMM_SPLITK");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int split_req = splitk_env > 0 ? splitk_env : d.split_k;
  if (split_req >= 2) {
    splits = split_req;
  } else if (split_req == 0 && tiles < 74) {
    splits = std::max(1, std::min(74 / tiles, kblocks / 4));
  }
  splits = std::max(1, std::min(splits, kblocks));
  g.splits = splits;
  if (splits > 1) {
    g.kb_per_split = (kblocks + splits - 1) / splits;
    g.splits = (kblocks + g.kb_per_split - 1) / g.kb_per_split;  // no empty splits
    g.ldw = (d.N + 7) / 8 * 8;
    if (cudaMalloc(&p->ws, sizeof(float) * static_cast<size_t>(g.splits) * d.M * g.ldw) != cudaSuccess)
      throw std::runtime_error("gemm: split-K workspace allocation failed");
    g.ws = p->ws;
    // Reduction: the separate fixed-order reduce kernel (one CTA per output
    // row, the whole chip) by default.  GWB_GEMM_SPLITK_INKERNEL=1 lets the
    // last-arriving split's CTAs reduce inside the GEMM instead (bitwise the
    // same sums) — measured 2× slower at c1 (285 vs 140 µs per iteration):
    // a quarter of the CTAs, one row per lane, do all the reduction reads.
    static const bool in_kernel = std::getenv("GWB_GEMM_SPLITK_INKERNEL") != nullptr;
    if (in_kernel) {
      const size_t bytes = sizeof(int) * 2 * static_cast<size_t>(g.tiles_m) * g.tiles_n;
      if (cudaMalloc(&p->counters, bytes) != cudaSuccess || cudaMemset(p->counters, 0, bytes) != cudaSuccess)
        throw std::runtime_error("gemm: split-K counter allocation failed");
      g.counters = p->counters;
    }
  }
  // One CTA pair per work item by default; GWB_GEMM_PERSISTENT=1 runs one
  // pair per SM pair looping over its items.  Measured at c4 (3 alternating
  // runs, one box): persistent 11.40-11.44 it/s at 1590-1612 MHz vs
  // 11.77-11.78 at 1665-1702 MHz — +2.7% per clock, but the chip is power-
  // capped (sw_power_cap) and the persistent grid's higher draw costs more
  // clock than it gains.
  if (d.rowsums) {
    // One partial per (row, 64-column slice of a tile) from the GEMM's
    // epilogue; the standalone split-K reduce kernel sums whole rows.
    g.rs_stride = (g.splits > 1 && g.counters == nullptr) ? 1 : g.tiles_n * 4;
    if (cudaMalloc(&p->rs_part, sizeof(double) * static_cast<size_t>(d.M) * g.rs_stride) != cudaSuccess)
      throw std::runtime_error("gemm: row-sum workspace allocation failed");
    g.rs_part = p->rs_part;
  }
  g.stamps = stamps_buffer();
  // Epilogue stores (measured A/B, one box, alternating runs): bulk copies of
  // whole row segments win on 256-wide tiles (c4 @ 8192: 158.5 vs 156.4
  // it/s), coalesced st.global on the smaller grids (c2, 192-wide: 4576 vs
  // 4411).  GWB_GEMM_BULK_STORE=0/1 forces.
  static const int bulk_env = [] {
    const char* e = std::getenv("GWB_GEMM_BULK_STORE");
    return e ? std::atoi(e) : -1;
  }();
  g.bulk_store = bulk_env >= 0 ? bulk_env : (p->bn == 256 ? 1 : 0);
  static const bool no_prefetch = std::getenv("GWB_GEMM_NO_A_PREFETCH") != nullptr;
  g.a_const = d.a_const && !no_prefetch ? 1 : 0;
  const int items = g.tiles_m * g.tiles_n * g.splits;
  static const bool persistent = [] {
    const char* e = std::getenv("GWB_GEMM_PERSISTENT");
    return e && e[0] == '1';
  }();
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  p->grid = 2 * (persistent ? std::min(items, std::max(1, sms / 2)) : items);
  p->flops = 2.0 * static_cast<double>(d.M) * static_cast<double>(d.N) * static_cast<double>(d.K);
  return p;
}

void gemm_plan_destroy(GemmPlan* p) { delete p; }

cudaError_t gemm_launch(const GemmPlan* p, cudaStream_t s) {
  if (p->params.stamps) g_stamps_grid = p->grid;
  cudaError_t e =
      p->bn == 64    ? launch_pdl(gemm_tf32_kernel<64>, dim3(p->grid), dim3(kThreads), smem_bytes(64), s, p->params)
      : p->bn == 128 ? launch_pdl(gemm_tf32_kernel<128>, dim3(p->grid), dim3(kThreads), smem_bytes(128), s, p->params)
      : p->bn == 192 ? launch_pdl(gemm_tf32_kernel<192>, dim3(p->grid), dim3(kThreads), smem_bytes(192), s, p->params)
                     : launch_pdl(gemm_tf32_kernel<256>, dim3(p->grid), dim3(kThreads), smem_bytes(256), s, p->params);
  if (e != cudaSuccess) return e;
  if (p->params.splits > 1 && p->params.counters == nullptr)
    e = launch_pdl(splitk_reduce_kernel, dim3(p->params.M), dim3(256), 0, s, p->params);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int gemm_debug_stamps(unsigned long long* out, int max_ctas) {
  if (!g_stamps) return 0;
  const int n = std::min(max_ctas, std::min(g_stamps_grid, 1024));
  if (cudaMemcpy(out, g_stamps, sizeof(unsigned long long) * 8 * n, cudaMemcpyDeviceToHost) != cudaSuccess)
    return 0;
  return n;
}

cudaError_t gemm_rowsum_bias(const GemmPlan* p, double factor, float* out, cudaStream_t s) {
  if (p->params.rs_part == nullptr) return cudaErrorInvalidValue;
  const cudaError_t e = launch_pdl(rowsum_bias_kernel, dim3((p->params.M + 255) / 256), dim3(256), 0, s,
                                   p->params, factor, out);
  return e != cudaSuccess ? e : cudaGetLastError();
}

int gemm_launches(const GemmPlan* p) {
  return p->params.splits > 1 && p->params.counters == nullptr ? 2 : 1;
}

double gemm_flops(const GemmPlan* p) { return p->flops; }
int gemm_passes(const GemmPlan* p) { return p->params.passes; }

}  // namespace gwb
