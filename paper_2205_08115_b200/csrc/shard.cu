// shard.cu — one rank of the row-sharded multi-GPU BAPG.
//
// Rank r owns rows [r·n_r, r·n_r + n_r) of π, w and D_X (n_r = ceil(n/P)
// rounded up to 64; rows ≥ n are zero padding).  D_Y is replicated.  Per
// half-step (reference solvers.cpp:164-177):
//   GEMM1   Vᵀ[:, rows_r] = D_Y · X_rᵀ       → slot r of the gather buffer
//   ── all-gather (NCCL, in place): the buffer is Vᵀ as [P][m][n_r] blocks ──
//   GEMM2   G_r = D_X[rows_r, :] · V          (B read through a blocked-K
//                                              3-D TMA map over the P blocks)
//   a: row projection, fully local
//   b: local column (max, Σ, Σπ) partials → slot r
//   ── all-gather of the column partials; merged in fixed rank order ──
//      column write pass, local fp64 diagnostic partial sums
//   ── all-reduce (sum) of 8 diagnostic scalars, all-reduce (max) of flags ──
//   finalize: identical record / stop rule / error decision on every rank.
// The collectives are issued by the caller (torch.distributed over NCCL, or
// the single-GPU emulation in tests) between gwb_shard_phase() calls on the
// shard's stream; every kernel is a no-op once the solve is done, while the
// collectives always run, so ranks never diverge in their collective calls.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <vector>

#include "../../include/gwb.h"
#include "../../include/gwb_ext.h"
#include "devutil.cuh"
#include "gemm.cuh"
#include "kernels.cuh"
#include "solver.cuh"
#include "standalone.cuh"

namespace gwb {

namespace {

using namespace dev;

constexpr int kDiag = 8;  // ⟨G,W⟩, rowdev, ⟨G,W'⟩, split, diff, ‖W‖², ⟨G,P⟩, coldev
constexpr int kErr = 8;   // ovfA, zeroA, ovfB, zeroB, nonfinite, −row idx, −col idx, unused

__global__ void shard_col_local_kernel(BapgDev d, double* slot, int64_t m) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double mx = -INFINITY, s = 0.0, p = 0.0;
  if (!d.st->done && d.n >= 1) {
    for (int c = 0; c < d.chunks; ++c) {
      const int64_t o = static_cast<int64_t>(c) * m + j;
      const double cm = d.col_pmax[o], cs = d.col_psum[o];
      if (cm > -INFINITY) {
        if (cm > mx) {
          s = s * exp(mx - cm) + cs;
          mx = cm;
        } else {
          s += cs * exp(cm - mx);
        }
      } else if (isnan(cm)) {
        mx = NAN;
      }
      p += d.col_psump[o];
    }
  }
  slot[j] = mx;
  slot[m + j] = s;
  slot[2 * m + j] = p;
}

// Merge the P rank slots in rank order (deterministic), raise column errors.
__global__ void shard_col_global_kernel(BapgDev d, const double* stats, int P) {
  if (d.st->done) return;
  const int64_t m = d.m;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double mx = -INFINITY, s = 0.0, p = 0.0;
  bool nan = false;
  for (int r = 0; r < P; ++r) {
    const double* sl = stats + static_cast<int64_t>(r) * 3 * m;
    const double cm = sl[j], cs = sl[m + j];
    if (isnan(cm)) nan = true;
    if (cm > -INFINITY) {
      if (cm > mx) {
        s = s * exp(mx - cm) + cs;
        mx = cm;
      } else {
        s += cs * exp(cm - mx);
      }
    }
    p += sl[2 * m + j];
  }
  if (mx > 700.0) atomicOr(&d.st->flags, kFlagOverflowB);
  if (nan || !(s > 0.0) || !isfinite(s)) {
    atomicOr(&d.st->flags, kFlagZeroB);
    atomicMin(&d.st->zero_index, static_cast<int>(j));
  }
  d.col_max[j] = mx;
  d.col_scale[j] = d.nu64[j] / s;
  const double dev = p - d.nu64[j];
  d.col_dev[j] = dev * dev;
}

__device__ double block_sum_d(double v) {
  __shared__ double sh[32];
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x / 32] = v;
  __syncthreads();
  double t = 0.0;
  for (int q = 0; q < static_cast<int>(blockDim.x / 32); ++q) t += sh[q];
  return t;
}

// Local fp64 partial sums + local error flags (always written: the
// all-reduce that follows runs on every rank unconditionally).
__global__ void shard_diag_kernel(BapgDev d, double* diag, double* err, int rank,
                                  int64_t row_begin, int tail) {
  const DevStatus* st = d.st;
  // The tail pass runs after convergence (gdone set) but not after errors.
  const bool active = tail ? st->flags == 0 : !st->gdone;
  double acc[kDiag] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (active) {
    for (int64_t i = threadIdx.x; i < d.n; i += blockDim.x) {
      acc[0] += d.row_part[i].gw;
      acc[1] += d.row_part[i].rowdev;
      if (!tail) {
        const ColWritePart c = d.cw_part[i];
        acc[2] += c.gw;
        acc[3] += c.split;
        acc[4] += c.diff;
        acc[5] += c.wold;
        acc[6] += c.gp;
      }
    }
    if (!tail && rank == 0)
      for (int64_t j = threadIdx.x; j < d.m; j += blockDim.x) acc[7] += d.col_dev[j];
  }
  for (int q = 0; q < kDiag; ++q) {
    const double t = block_sum_d(acc[q]);
    if (threadIdx.x == 0) diag[q] = t;
  }
  if (threadIdx.x == 0) {
    const int f = active ? st->flags : 0;
    err[0] = (f & kFlagOverflowA) ? 1.0 : 0.0;
    err[1] = (f & kFlagZeroA) ? 1.0 : 0.0;
    err[2] = (f & kFlagOverflowB) ? 1.0 : 0.0;
    err[3] = (f & kFlagZeroB) ? 1.0 : 0.0;
    err[4] = (f & kFlagNonFinite) ? 1.0 : 0.0;
    err[5] = (f & kFlagZeroA) ? -static_cast<double>(row_begin + st->zero_index) : -1e18;
    err[6] = (f & kFlagZeroB) ? -static_cast<double>(st->zero_index) : -1e18;
    err[7] = 0.0;
  }
}

// Global record / stop rule / error decision from the all-reduced vectors.
__global__ void shard_finalize_kernel(BapgDev d, const double* diag, const double* err,
                                      double rel_tol, int tail) {
  DevStatus* st = d.st;
  if (st->gdone) {
    st->done = 1;
    if (!tail || st->flags) return;
  }
  auto slot = [&](int it) { return it <= d.max_rec ? it : d.max_rec + 1; };
  if (tail) {
    const int k = st->iter - 1;
    d.rec[slot(k)].mw_w = diag[0];
    d.rec[slot(k)].row_sq = diag[1];
    return;
  }
  const int k = st->iter;
  int gflags = 0;
  if (err[0] > 0.5) gflags |= kFlagOverflowA;
  if (err[1] > 0.5) gflags |= kFlagZeroA;
  if (err[2] > 0.5) gflags |= kFlagOverflowB;
  if (err[3] > 0.5) gflags |= kFlagZeroB;
  if (err[4] > 0.5) gflags |= kFlagNonFinite;
  if (gflags) {
    st->flags = gflags;
    st->zero_index = static_cast<int>((gflags & kFlagZeroA) ? -err[5] : -err[6]);
    st->err_iter = k;
    st->done = st->gdone = 1;
    return;
  }
  if (k >= 2) {
    d.rec[slot(k - 1)].mw_w = diag[0];
    d.rec[slot(k - 1)].row_sq = diag[1];
  }
  DevRecord& r = d.rec[slot(k)];
  r.mpi_w = diag[2];
  r.split_sq = diag[3];
  r.diff_sq = diag[4];
  r.wold_sq = diag[5];
  r.mpi_pi = diag[6];
  r.col_sq = diag[7];
  r.elapsed = 1e-9 * static_cast<double>(globaltimer() - st->t0);
  st->iter = k + 1;
  // Local flags (if any) were all clean; keep the local done in sync.
  st->flags = 0;
  st->done = 0;
  // fp64 iterates: the reference's rule as is (solvers.cpp:208).
  if (sqrt(diag[4]) / sqrt(diag[5]) <= rel_tol) {
    st->converged = 1;
    st->done = st->gdone = 1;
  }
}

// A configuration the engine refuses (maps to GWB_ERR_CONFIG).
struct ShardConfigError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

template <class T>
T* dalloc(size_t count) {
  void* p = nullptr;
  GWB_CUDA(cudaMalloc(&p, count * sizeof(T) + 256));
  GWB_CUDA(cudaMemset(p, 0, count * sizeof(T) + 256));
  GWB_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  return static_cast<T*>(p);
}

}  // namespace

class ShardEngine {
 public:
  ShardEngine(const gwb_config& cfg, int64_t n, int64_t m, int rank, int world, int device,
              cudaStream_t stream)
      : cfg_(cfg), n_(n), m_(m), rank_(rank), world_(world), dev_(device), s_(stream) {
    GWB_CUDA(cudaSetDevice(dev_));
    if (!s_) {
      GWB_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
      own_stream_ = true;
    }
    // AUTO depends on the exactness of every rank's rows of D_X, which this
    // rank cannot see: the orchestrator resolves it (dist.resolve_precision).
    if (cfg.precision == GWB_PREC_AUTO)
      throw std::invalid_argument(
          "gwb_shard_create: resolve AUTO precision across ranks first (f16x2, bf16x3 or 3xtf32; dist.resolve_precision)");
    prec_ = cfg.precision;
    f16_ = prec_ == GWB_PREC_F16X2;
    bf16_ = prec_ == GWB_PREC_BF16X3 || prec_ == GWB_PREC_BF16X2 || f16_;  // split planes
    planes_ = prec_ == GWB_PREC_BF16X3 ? 3 : (prec_ == GWB_PREC_TF32 ? 1 : 2);
    esize_ = bf16_ ? 2 : 4;
    aux_mode_ = prec_ == GWB_PREC_TF32 ? 1 : prec_ == GWB_PREC_3XTF32 ? 2
                : prec_ == GWB_PREC_BF16X3 ? 3 : f16_ ? 5 : 4;
    nr_ = round_up((n_ + world_ - 1) / world_, 64);
    row_begin_ = static_cast<int64_t>(rank_) * nr_;
    rows_valid_ = std::max<int64_t>(0, std::min<int64_t>(nr_, n_ - row_begin_));
    ldk_ = round_up(nr_ * world_, 64);
    ldm_ = round_up(m_, 64);
    const size_t nm = static_cast<size_t>(nr_) * ldm_;
    Dx_ = keep(dalloc<float>(static_cast<size_t>(nr_) * ldk_));
    Dy_ = keep(dalloc<float>(static_cast<size_t>(m_) * ldm_));
    Dx_aux_ = keep(dalloc<float>(static_cast<size_t>(nr_) * ldk_));
    Dy_aux_ = keep(dalloc<float>(static_cast<size_t>(m_) * ldm_));
    P_ = keep(dalloc<float>(nm));
    P64_ = keep(dalloc<double>(nm));
    for (int q = 0; q < 2; ++q) W64_[q] = keep(dalloc<double>(nm));
    P_aux_ = keep(dalloc<float>(nm * 3 / 2));
    for (int q = 0; q < 2; ++q) {
      W_[q] = keep(dalloc<float>(nm));
      W_aux_[q] = keep(dalloc<float>(nm * 3 / 2));
    }
    G_ = keep(dalloc<float>(nm));
    mu32_ = keep(dalloc<float>(nr_));
    nu32_ = keep(dalloc<float>(ldm_));
    mu64_ = keep(dalloc<double>(nr_));
    nu64_ = keep(dalloc<double>(ldm_));
    row_part_ = keep(dalloc<RowPart>(nr_));
    cw_part_ = keep(dalloc<ColWritePart>(nr_));
    const int64_t col_blocks = (m_ + 127) / 128;
    chunks_ = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((std::max<int64_t>(rows_valid_, 1) + 63) / 64,
                             (4 * 148 + col_blocks - 1) / col_blocks)));
    col_pmax_ = keep(dalloc<double>(static_cast<size_t>(chunks_) * m_));
    col_psum_ = keep(dalloc<double>(static_cast<size_t>(chunks_) * m_));
    col_psump_ = keep(dalloc<double>(static_cast<size_t>(chunks_) * m_));
    col_max_ = keep(dalloc<double>(ldm_));
    col_scale_ = keep(dalloc<double>(ldm_));
    col_dev_ = keep(dalloc<double>(ldm_));
    st_ = keep(dalloc<DevStatus>(1));
    rec_ = keep(dalloc<DevRecord>(static_cast<size_t>(cfg_.max_iters) + 2));
  }
  ~ShardEngine() {
    cudaSetDevice(dev_);
    cudaStreamSynchronize(s_);
    for (auto* p : plans_) gemm_plan_destroy(p);
    for (void* p : bufs_) cudaFree(p);
    if (own_stream_) cudaStreamDestroy(s_);
  }

  int64_t rows_per_shard() const { return nr_; }
  int64_t row_begin() const { return row_begin_; }
  int64_t rows_valid() const { return rows_valid_; }
  int planes() const { return planes_; }
  int esize() const { return esize_; }
  int64_t vt_bytes() const {
    return static_cast<int64_t>(planes_) * world_ * m_ * nr_ * esize_;
  }
  int64_t stats_bytes() const { return static_cast<int64_t>(world_) * 3 * m_ * 8; }
  cudaStream_t stream() const { return s_; }

  void set_comm(void* vt, void* stats, double* diag, double* err) {
    vt_ = static_cast<uint8_t*>(vt);
    stats_ = static_cast<double*>(stats);
    diag_ = diag;
    err_ = err;
  }

  // dx_rows: rows_valid × n fp32 (leading dim ldx) = D_X[row_begin : …, :];
  // dy: m × m; mu_rows: rows_valid; nu: m.  Device pointers.
  void load(const float* dx_rows, int64_t ldx, const float* dy, int64_t ldy, const float* mu_rows,
            const float* nu) {
    GWB_CUDA(cudaSetDevice(dev_));
    if (!vt_) throw CudaError("gwb_shard: set_comm must precede load");
    if (rows_valid_ > 0)
      GWB_CUDA(cudaMemcpy2DAsync(Dx_, ldk_ * 4, dx_rows, ldx * 4, n_ * 4, rows_valid_,
                                 cudaMemcpyDeviceToDevice, s_));
    GWB_CUDA(cudaMemcpy2DAsync(Dy_, ldm_ * 4, dy, ldy * 4, m_ * 4, m_, cudaMemcpyDeviceToDevice, s_));
    if (rows_valid_ > 0)
      GWB_CUDA(cudaMemcpyAsync(mu32_, mu_rows, 4 * rows_valid_, cudaMemcpyDeviceToDevice, s_));
    GWB_CUDA(cudaMemcpyAsync(nu32_, nu, 4 * m_, cudaMemcpyDeviceToDevice, s_));
    std::vector<float> h_mu(std::max<int64_t>(rows_valid_, 1)), h_nu(m_);
    if (rows_valid_ > 0)
      GWB_CUDA(cudaMemcpyAsync(h_mu.data(), mu_rows, 4 * rows_valid_, cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaMemcpyAsync(h_nu.data(), nu, 4 * m_, cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
    std::vector<double> d_mu(h_mu.begin(), h_mu.end()), d_nu(h_nu.begin(), h_nu.end());
    GWB_CUDA(cudaMemcpyAsync(mu64_, d_mu.data(), 8 * std::max<int64_t>(rows_valid_, 1),
                             cudaMemcpyHostToDevice, s_));
    GWB_CUDA(cudaMemcpyAsync(nu64_, d_nu.data(), 8 * m_, cudaMemcpyHostToDevice, s_));
    // A split-plane chain rounds D_X / D_Y to fp16 or bf16: refuse a D that
    // is not exact there (the orchestrator agrees the precision across ranks
    // and downgrades first, dist.resolve_precision, as the single-GPU engine
    // does; reaching this is a caller error, never a silent rounding).
    if (bf16_) {
      const int bits = analyze_inexact(Dx_, rows_valid_, n_, ldk_, s_) |
                       analyze_inexact(Dy_, m_, m_, ldm_, s_);
      if (!split_exact(prec_, bits))
        throw ShardConfigError(
            "gwb_shard: the requested split-plane precision needs structure matrices exact in "
            "fp16 (f16x2) / bf16 (bf16x3, bf16x2); resolve it across ranks first "
            "(dist.resolve_precision)");
    }
    // Operand copies of the structure matrices.
    if (f16_) {
      // f16x2: the scales derive from the global iterate
      // bound and the replicated D_Y, so every rank writes its Vᵀ block with
      // the same per-row scales and GEMM2 undoes them with one column scale.
      if (!(x_max_ > 0.0))
        throw std::invalid_argument(
            "gwb_shard: f16x2 needs gwb_shard_set_iterate_bound (max of mu and nu over all "
            "ranks) before load");
      launch_to_f16(Dx_, nr_, ldk_, ldk_, Dx_aux_, s_);
      launch_to_f16(Dy_, m_, ldm_, ldm_, Dy_aux_, s_);
      f16_s1_ = 14 - static_cast<int>(std::ceil(std::log2(x_max_)));
      if (!f16_g1_rs_) f16_g1_rs_ = keep(dalloc<float>(ldm_));
      if (!f16_g2_cs_) f16_g2_cs_ = keep(dalloc<float>(ldm_));
      launch_f16_scales(Dy_, m_, ldm_, static_cast<float>(x_max_), f16_s1_, f16_g1_rs_,
                        f16_g2_cs_, s_);
    } else if (bf16_) {
      launch_to_bf16(Dx_, nr_, ldk_, ldk_, Dx_aux_, s_);
      launch_to_bf16(Dy_, m_, ldm_, ldm_, Dy_aux_, s_);
    } else {
      launch_tf32_aux(Dx_, nr_, ldk_, ldk_, Dx_aux_, aux_mode_, s_);
      launch_tf32_aux(Dy_, m_, ldm_, ldm_, Dy_aux_, aux_mode_, s_);
    }
    GWB_CUDA(cudaStreamSynchronize(s_));
    build_plans();
  }

  void reset() {
    GWB_CUDA(cudaSetDevice(dev_));
    launch_status_reset(st_, s_);
    if (rows_valid_ > 0) {
      launch_product_coupling64(mu64_, nu64_, rows_valid_, m_, ldm_, W64_[0], s_);
      launch_iterate_copies(W64_[0], nr_, m_, ldm_, needs_copy() ? W_[0] : nullptr, W_aux_[0],
                            aux_mode_, aux_scale(), s_);
    }
    parity_ = 0;
    GWB_CUDA(cudaGetLastError());
  }

  // Phases between collectives (see file comment).
  int64_t launches() const { return launches_; }

  // Chunked GEMM2 (compute/collective overlap): the partial product of the
  // Vᵀ block owned by rank `src`, G_r (+)= D_X[rows_r, cols_src]·V_src.  The
  // caller launches the local block first (it overwrites G_r) and the others
  // as their collective lands; phases 21/23/27 are then 1/3/7 without the
  // monolithic GEMM2.
  void gemm2_chunk(int src, bool tail) {
    GWB_CUDA(cudaSetDevice(dev_));
    if (src < 0 || src >= world_) throw CudaError("gwb_shard_gemm2_chunk: bad source rank");
    GWB_CUDA(gemm_launch(tail ? g2ct_[src] : g2c_[src], s_));
    if (!tail) launches_ += 1;
  }

  void phase(int ph) {
    GWB_CUDA(cudaSetDevice(dev_));
    const int q = parity_;
    BapgDev d = view(q);
    const bool chunked = ph >= 20;  // GEMM2 issued by gemm2_chunk
    if (chunked) {
      if (ph != 21 && ph != 23 && ph != 27) throw CudaError("gwb_shard_phase: unknown phase");
      ph -= 20;
    }
    switch (ph) {
      case 0:  // A1: Vᵀ slot ← D_Y · W_rᵀ
        GWB_CUDA(gemm_launch(g1_[q], s_));
        launches_ += 1;
        break;
      case 1:  // A2: G_r, row projection
        if (!chunked) GWB_CUDA(gemm_launch(g2_, s_));
        launch_row_update(d, true, s_);
        launches_ += chunked ? 1 : 2;
        break;
      case 2:  // B1
        GWB_CUDA(gemm_launch(g1p_, s_));
        launches_ += 1;
        break;
      case 3:  // B2: G_r, local column partials → stats slot
        if (!chunked) GWB_CUDA(gemm_launch(g2_, s_));
        launch_col_partial(d, s_);
        shard_col_local_kernel<<<static_cast<unsigned>((m_ + 255) / 256), 256, 0, s_>>>(
            d, stats_ + static_cast<int64_t>(rank_) * 3 * m_, m_);
        launches_ += chunked ? 2 : 3;
        break;
      case 4:  // B3: global column merge, write pass, local diagnostics
        shard_col_global_kernel<<<static_cast<unsigned>((m_ + 255) / 256), 256, 0, s_>>>(
            d, stats_, world_);
        launch_col_write(d, s_);
        shard_diag_kernel<<<1, 512, 0, s_>>>(d, diag_, err_, rank_, row_begin_, 0);
        launches_ += d.n >= 1 ? 3 : 2;
        break;
      case 5:  // F: global finalize; w' becomes w
        shard_finalize_kernel<<<1, 1, 0, s_>>>(d, diag_, err_, cfg_.rel_tol, 0);
        parity_ ^= 1;
        launches_ += 1;
        break;
      case 6:  // tail A1 (chain on the final w; runs after convergence)
        GWB_CUDA(gemm_launch(g1t_[q], s_));
        break;
      case 7:  // tail A2: diagnostics-only row pass
        if (!chunked) GWB_CUDA(gemm_launch(g2t_, s_));
        launch_row_update(d, false, s_);
        shard_diag_kernel<<<1, 512, 0, s_>>>(d, diag_, err_, rank_, row_begin_, 1);
        break;
      case 8:  // tail F
        shard_finalize_kernel<<<1, 1, 0, s_>>>(d, diag_, err_, 0.0, 1);
        break;
      default:
        throw CudaError("gwb_shard_phase: unknown phase");
    }
    GWB_CUDA(cudaGetLastError());
  }

  DevStatus status() {
    DevStatus h;
    GWB_CUDA(cudaMemcpyAsync(&h, st_, sizeof(h), cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
    return h;
  }

  // After the loop the current w is W[(iterations used) % 2].
  void sync_parity() {
    const DevStatus h = status();
    parity_ = (h.iter - 1) & 1;
  }

  std::vector<DevRecord> records(int count) {
    std::vector<DevRecord> r(static_cast<size_t>(count) + 1);
    GWB_CUDA(cudaMemcpyAsync(r.data(), rec_, sizeof(DevRecord) * (count + 1), cudaMemcpyDeviceToHost, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
    return r;
  }

  // Local rows of π and w as row-major fp64 (rows_valid × m).
  void rows(double* pi, double* w) {
    auto get = [&](const double* src, double* dst) {
      if (!dst || rows_valid_ == 0) return;
      GWB_CUDA(cudaMemcpy2DAsync(dst, 8 * m_, src, 8 * ldm_, 8 * m_, rows_valid_,
                                 cudaMemcpyDeviceToHost, s_));
      GWB_CUDA(cudaStreamSynchronize(s_));
    };
    get(P64_, pi);
    get(W64_[parity_], w);
  }

  // Exact fp64 marginals (the load path carries fp32 device copies).
  void set_marginals64(const double* mu_rows, const double* nu) {
    GWB_CUDA(cudaSetDevice(dev_));
    if (rows_valid_ > 0)
      GWB_CUDA(cudaMemcpyAsync(mu64_, mu_rows, 8 * rows_valid_, cudaMemcpyHostToDevice, s_));
    GWB_CUDA(cudaMemcpyAsync(nu64_, nu, 8 * m_, cudaMemcpyHostToDevice, s_));
    GWB_CUDA(cudaStreamSynchronize(s_));
  }

 private:
  template <class T>
  T* keep(T* p) {
    bufs_.push_back(p);
    return p;
  }

  BapgDev view(int q) const {
    BapgDev d;
    std::memset(&d, 0, sizeof(d));
    d.n = rows_valid_;
    d.m = m_;
    d.ld = ldm_;
    d.inv_rho = static_cast<float>(1.0 / cfg_.rho);
    d.inv_rho64 = 1.0 / cfg_.rho;
    d.G = G_;
    d.mu = mu32_;
    d.nu = nu32_;
    d.mu64 = mu64_;
    d.nu64 = nu64_;
    d.P64 = P64_;
    d.W64 = W64_[q];
    d.W64_new = W64_[1 - q];
    d.P = needs_copy() ? P_ : nullptr;
    d.P_aux = P_aux_;
    d.W = W_[q];
    d.W_new = needs_copy() ? W_[1 - q] : nullptr;
    d.W_aux = W_aux_[1 - q];
    d.aux_mode = aux_mode_;
    d.aux_scale = aux_scale();
    d.plane = nr_ * ldm_;
    d.row_part = row_part_;
    d.cw_part = cw_part_;
    d.col_pmax = col_pmax_;
    d.col_psum = col_psum_;
    d.col_psump = col_psump_;
    d.col_max = col_max_;
    d.col_scale = col_scale_;
    d.col_dev = col_dev_;
    d.chunks = chunks_;
    d.st = st_;
    d.rec = rec_;
    d.max_rec = cfg_.max_iters;
    return d;
  }

  // Gather buffer layout [world][planes][m][n_r]: rank r's planes are one
  // contiguous chunk, so a single in-place all-gather moves every plane.
  void* slot(int plane, int rank) const {
    return vt_ + ((static_cast<int64_t>(rank) * planes_ + plane) * m_ * nr_) * esize_;
  }
  void* plane_base(int plane) const {
    return vt_ + (static_cast<int64_t>(plane) * m_ * nr_) * esize_;
  }
  void* aux_plane(float* aux, int p) const {
    return reinterpret_cast<uint8_t*>(aux) + static_cast<int64_t>(p) * nr_ * ldm_ * 2;
  }

  GemmPlan* make1(float* X, float* X_aux, const int* skip) {
    GemmDesc d;
    d.a_const = true;  // A = a structure matrix (constant)
    d.M = m_;
    d.N = nr_;
    d.K = m_;
    d.ldb = ldm_;
    d.lda = ldm_;
    d.ldc = nr_;
    d.skip = skip;
    if (bf16_) {
      d.bf16_planes = planes_;
      d.a_bf16 = Dy_aux_;
      for (int p = 0; p < planes_; ++p) d.b_bf16[p] = aux_plane(X_aux, p);
      d.c_planes = planes_;
      for (int p = 0; p < planes_; ++p) d.c_bf16[p] = slot(p, rank_);
      d.f16 = f16_;
      if (f16_) d.row_scale = f16_g1_rs_;
    } else {
      const bool tf32 = prec_ == GWB_PREC_TF32;
      d.a = tf32 ? Dy_aux_ : Dy_;
      d.a_lo = tf32 ? nullptr : Dy_aux_;
      d.b = tf32 ? X_aux : X;
      d.b_lo = tf32 ? nullptr : X_aux;
      d.c = static_cast<float*>(slot(0, rank_));
      d.c_aux = tf32 ? nullptr : static_cast<float*>(slot(1, rank_));
      d.aux_mode = tf32 ? 1 : 2;
      d.three_pass = !tf32;
    }
    GemmPlan* p = gemm_plan_create(d);
    plans_.push_back(p);
    return p;
  }

  // Partial GEMM2 over the Vᵀ block of rank `src`: K = n_r columns of the
  // local D_X rows starting at src·n_r, B = that rank's slot (plain 2-D).
  GemmPlan* make2_chunk(int src, const int* skip) {
    GemmDesc d;
    d.a_const = true;  // A = a structure matrix (constant)
    d.M = nr_;
    d.N = m_;
    d.K = nr_;
    d.lda = ldk_;
    d.ldb = nr_;
    d.c = G_;
    d.ldc = ldm_;
    d.skip = skip;
    d.accumulate = src != rank_;  // the local block is launched first
    const int64_t koff = static_cast<int64_t>(src) * nr_;
    if (bf16_) {
      d.bf16_planes = planes_;
      d.a_bf16 = reinterpret_cast<const uint8_t*>(Dx_aux_) + koff * 2;
      for (int p = 0; p < planes_; ++p) d.b_bf16[p] = slot(p, src);
      d.f16 = f16_;
      if (f16_) d.col_scale = f16_g2_cs_;
    } else {
      const bool tf32 = prec_ == GWB_PREC_TF32;
      d.a = (tf32 ? Dx_aux_ : Dx_) + koff;
      d.a_lo = tf32 ? nullptr : Dx_aux_ + koff;
      d.b = static_cast<const float*>(slot(0, src));
      d.b_lo = tf32 ? nullptr : static_cast<const float*>(slot(1, src));
      d.three_pass = !tf32;
    }
    GemmPlan* p = gemm_plan_create(d);
    plans_.push_back(p);
    return p;
  }

  GemmPlan* make2(const int* skip) {
    GemmDesc d;
    d.a_const = true;  // A = a structure matrix (constant)
    d.M = nr_;
    d.N = m_;
    d.K = nr_ * world_;
    d.lda = ldk_;
    d.b_block_k = nr_;
    d.b_block_stride = static_cast<int64_t>(planes_) * m_ * nr_;
    d.c = G_;
    d.ldc = ldm_;
    d.skip = skip;
    if (bf16_) {
      d.bf16_planes = planes_;
      d.a_bf16 = Dx_aux_;
      for (int p = 0; p < planes_; ++p) d.b_bf16[p] = plane_base(p);
      d.f16 = f16_;
      if (f16_) d.col_scale = f16_g2_cs_;
    } else {
      const bool tf32 = prec_ == GWB_PREC_TF32;
      d.a = tf32 ? Dx_aux_ : Dx_;
      d.a_lo = tf32 ? nullptr : Dx_aux_;
      d.b = static_cast<const float*>(plane_base(0));
      d.b_lo = tf32 ? nullptr : static_cast<const float*>(plane_base(1));
      d.three_pass = !tf32;
    }
    GemmPlan* p = gemm_plan_create(d);
    plans_.push_back(p);
    return p;
  }

  void build_plans() {
    for (int q = 0; q < 2; ++q) {
      g1_[q] = make1(W_[q], W_aux_[q], &st_->done);
      g1t_[q] = make1(W_[q], W_aux_[q], &st_->flags);
    }
    g1p_ = make1(P_, P_aux_, &st_->done);
    g2_ = make2(&st_->done);
    g2t_ = make2(&st_->flags);
    g2c_.assign(world_, nullptr);
    g2ct_.assign(world_, nullptr);
    for (int s = 0; s < world_; ++s) {
      g2c_[s] = make2_chunk(s, &st_->done);
      g2ct_[s] = make2_chunk(s, &st_->flags);
    }
  }

  gwb_config cfg_;
  int64_t n_, m_;
  int rank_, world_, dev_;
  cudaStream_t s_;
  bool own_stream_ = false;
  int prec_, planes_, esize_, aux_mode_;
  bool bf16_, f16_ = false;
  // f16x2: global bound on every iterate entry (max μ, max ν over all
  // ranks, set by the orchestrator) and the scales derived from it.
  double x_max_ = 0.0;
  int f16_s1_ = 0;
  float* f16_g1_rs_ = nullptr;
  float* f16_g2_cs_ = nullptr;

 public:
  void set_iterate_bound(double x_max) { x_max_ = x_max; }
  float aux_scale() const { return f16_ ? std::ldexp(1.0f, f16_s1_) : 1.0f; }

 private:
  int64_t nr_, row_begin_, rows_valid_, ldk_, ldm_;
  int parity_ = 0;
  int64_t launches_ = 0;  // kernels launched by phases 0-5 (bench gpu_launches)
  std::vector<void*> bufs_;
  std::vector<GemmPlan*> plans_;
  std::vector<GemmPlan*> g2c_, g2ct_;  // chunked GEMM2 per source rank (owned by plans_)
  float *Dx_, *Dy_, *Dx_aux_, *Dy_aux_, *P_, *P_aux_, *W_[2], *W_aux_[2], *G_;
  float *mu32_, *nu32_;
  double *mu64_, *nu64_;
  RowPart* row_part_;
  ColWritePart* cw_part_;
  double *col_pmax_, *col_psum_, *col_max_, *col_scale_;
  double *col_psump_, *col_dev_;
  // fp64 iterates (as the single-GPU engine); P_ / W_ hold the
  // fp32 hi operand copies of the 3xTF32 chain only.
  double *P64_ = nullptr, *W64_[2] = {nullptr, nullptr};
  bool needs_copy() const { return prec_ == GWB_PREC_3XTF32; }
  int chunks_ = 1;
  DevStatus* st_;
  DevRecord* rec_;
  uint8_t* vt_ = nullptr;
  double* stats_ = nullptr;
  double* diag_ = nullptr;
  double* err_ = nullptr;
  GemmPlan *g1_[2] = {nullptr, nullptr}, *g1t_[2] = {nullptr, nullptr}, *g1p_ = nullptr,
           *g2_ = nullptr, *g2t_ = nullptr;
};


// ---------------------------------------------------------------------------
// In-library multi-device BAPG (one process, several GPUs): the row-sharded
// engines above driven by the phase / collective schedule of
// dist.iterate_sharded (all-gather form), with NCCL's single-process
// communicator (ncclCommInitAll) over NVLink / NVSwitch.  NCCL is loaded at
// run time (dlopen), so libgwb.so has no link dependency on it and a
// single-device caller never touches it.
namespace {

struct NcclApi {
  decltype(&ncclCommInitAll) comm_init_all = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;

  static const NcclApi& get() {
    static NcclApi api = [] {
      NcclApi a;
      void* h = nullptr;
      for (const char* name : {"libnccl.so.2", "libnccl.so"})
        if ((h = dlopen(name, RTLD_NOW | RTLD_LOCAL))) break;
      if (!h) return a;
      a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
      a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
      a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
      a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
      a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
      a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
      a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
      return a;
    }();
    if (!api.comm_init_all || !api.all_gather || !api.all_reduce || !api.group_start ||
        !api.group_end || !api.comm_destroy)
      throw CudaError("multi-device solve: libnccl.so.2 not found (GWB_DEVICES lists several GPUs)");
    return api;
  }
  void check(ncclResult_t r, const char* what) const {
    if (r != ncclSuccess)
      throw CudaError(std::string("NCCL ") + what + ": " + (error_string ? error_string(r) : "error"));
  }
};

__global__ void f64_to_f32_kernel(const double* __restrict__ src, float* __restrict__ dst,
                                  int64_t count) {
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[k] = static_cast<float>(src[k]);
}

// Device buffer freed on scope exit (current device set by the caller).
struct DevBuf {
  void* p = nullptr;
  int dev = 0;
  DevBuf() = default;
  DevBuf(int device, size_t bytes) : dev(device) {
    GWB_CUDA(cudaSetDevice(dev));
    GWB_CUDA(cudaMalloc(&p, bytes + 256));
    GWB_CUDA(cudaMemset(p, 0, bytes + 256));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), dev(o.dev) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      dev = o.dev;
      o.p = nullptr;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (p) {
      cudaSetDevice(dev);
      cudaFree(p);
      p = nullptr;
    }
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace

DevStatus bapg_multi_device(const gwb_config& cfg_in, const std::vector<int>& devices,
                            const double* dx, int64_t n, const double* dy, int64_t m,
                            const double* mu, const double* nu, double* out_final,
                            double* out_pi, double* out_w, std::vector<HostRecord>* records,
                            int* resolved_precision) {
  const int P = static_cast<int>(devices.size());
  gwb_config cfg = cfg_in;
  const int64_t nr = round_up((n + P - 1) / P, 64);
  // 1. Stage every rank's rows of D_X (a symmetric D's rows are its
  //    contiguous columns in the column-major input), D_Y and the marginals
  //    in fp32 on its device; agree on the chain precision from the
  //    exactness of all ranks' rows (dist.resolve_precision's rules).
  std::vector<DevBuf> rows(P), dys(P), mus(P), nus(P);
  int bits = 0;
  for (int r = 0; r < P; ++r) {
    const int dev = devices[r];
    const int64_t rb = static_cast<int64_t>(r) * nr;
    const int64_t rv = std::max<int64_t>(0, std::min<int64_t>(nr, n - rb));
    GWB_CUDA(cudaSetDevice(dev));
    const int64_t big = std::max(std::max<int64_t>(rv, 1) * n, m * m);
    DevBuf stage(dev, sizeof(double) * big);
    rows[r] = DevBuf(dev, sizeof(float) * std::max<int64_t>(rv, 1) * n);
    dys[r] = DevBuf(dev, sizeof(float) * m * m);
    mus[r] = DevBuf(dev, sizeof(float) * std::max<int64_t>(rv, 1));
    nus[r] = DevBuf(dev, sizeof(float) * m);
    if (rv > 0) {
      GWB_CUDA(cudaMemcpy(stage.p, dx + rb * n, sizeof(double) * rv * n, cudaMemcpyHostToDevice));
      f64_to_f32_kernel<<<1184, 256>>>(stage.as<double>(), rows[r].as<float>(), rv * n);
      GWB_CUDA(cudaMemcpy(stage.p, mu + rb, sizeof(double) * rv, cudaMemcpyHostToDevice));
      f64_to_f32_kernel<<<1, 256>>>(stage.as<double>(), mus[r].as<float>(), rv);
      bits |= analyze_inexact(rows[r].as<float>(), rv, n, n, nullptr);
    }
    GWB_CUDA(cudaMemcpy(stage.p, dy, sizeof(double) * m * m, cudaMemcpyHostToDevice));
    f64_to_f32_kernel<<<1184, 256>>>(stage.as<double>(), dys[r].as<float>(), m * m);
    GWB_CUDA(cudaMemcpy(stage.p, nu, sizeof(double) * m, cudaMemcpyHostToDevice));
    f64_to_f32_kernel<<<1, 256>>>(stage.as<double>(), nus[r].as<float>(), m);
    if (r == 0) bits |= analyze_inexact(dys[r].as<float>(), m, m, m, nullptr);
    GWB_CUDA(cudaDeviceSynchronize());
  }
  const bool f16 = (bits & 4) == 0, bf16 = (bits & 2) == 0;
  int prec = cfg.precision;
  if (prec == GWB_PREC_AUTO) prec = f16 ? GWB_PREC_F16X2 : bf16 ? GWB_PREC_BF16X3 : GWB_PREC_3XTF32;
  if (prec == GWB_PREC_F16X2 && !f16) prec = GWB_PREC_BF16X3;
  if ((prec == GWB_PREC_BF16X3 || prec == GWB_PREC_BF16X2) && !bf16) prec = GWB_PREC_3XTF32;
  if (prec == GWB_PREC_F16X3) prec = GWB_PREC_3XTF32;  // the sharded engine's weighted-D chain
  cfg.precision = prec;
  if (resolved_precision) *resolved_precision = prec;
  double x_max = 0.0;
  for (int64_t i = 0; i < n; ++i) x_max = std::max(x_max, std::fabs(mu[i]));
  for (int64_t j = 0; j < m; ++j) x_max = std::max(x_max, std::fabs(nu[j]));

  // 2. Engines, exchange buffers, communicators.
  std::vector<std::unique_ptr<ShardEngine>> eng;
  std::vector<DevBuf> vt(P), stats(P), diag(P), err(P);
  for (int r = 0; r < P; ++r) {
    eng.emplace_back(new ShardEngine(cfg, n, m, r, P, devices[r], nullptr));
    vt[r] = DevBuf(devices[r], static_cast<size_t>(eng[r]->vt_bytes()));
    stats[r] = DevBuf(devices[r], static_cast<size_t>(eng[r]->stats_bytes()));
    diag[r] = DevBuf(devices[r], sizeof(double) * kDiag);
    err[r] = DevBuf(devices[r], sizeof(double) * kErr);
    eng[r]->set_comm(vt[r].p, stats[r].p, diag[r].as<double>(), err[r].as<double>());
    if (prec == GWB_PREC_F16X2) eng[r]->set_iterate_bound(x_max);
    eng[r]->load(rows[r].as<float>(), n, dys[r].as<float>(), m, mus[r].as<float>(),
                 nus[r].as<float>());
    const int64_t rb = eng[r]->row_begin(), rv = eng[r]->rows_valid();
    eng[r]->set_marginals64(rv > 0 ? mu + rb : mu, nu);
    eng[r]->reset();
  }
  rows.clear();
  dys.clear();
  // A device listed twice (e.g. GWB_DEVICES=0,0 on a one-GPU box) runs the
  // same schedule with emulated collectives: host-synchronised device copies
  // in rank order and host reductions (dist.EmuComm's semantics) — a test
  // mode for the orchestration; distinct devices use NCCL.
  bool emulate = false;
  for (int r = 0; r < P; ++r)
    for (int q = 0; q < r; ++q) emulate = emulate || devices[q] == devices[r];
  const NcclApi* nccl = emulate ? nullptr : &NcclApi::get();
  std::vector<ncclComm_t> comms(emulate ? 0 : P);
  if (!emulate) nccl->check(nccl->comm_init_all(comms.data(), P, devices.data()), "ncclCommInitAll");
  struct CommGuard {
    const NcclApi* api;
    std::vector<ncclComm_t>& c;
    ~CommGuard() {
      for (auto x : c) api->comm_destroy(x);
    }
  } guard{nccl, comms};
  auto sync_all = [&]() {
    for (auto& e : eng) GWB_CUDA(cudaStreamSynchronize(e->stream()));
  };

  auto all_phase = [&](int ph) {
    for (auto& e : eng) e->phase(ph);
  };
  auto gather = [&](std::vector<DevBuf>& buf, size_t chunk_bytes) {
    if (emulate) {
      sync_all();
      for (int r = 0; r < P; ++r)
        for (int q = 0; q < P; ++q)
          if (q != r)
            GWB_CUDA(cudaMemcpyPeer(buf[q].as<uint8_t>() + r * chunk_bytes, devices[q],
                                    buf[r].as<uint8_t>() + r * chunk_bytes, devices[r], chunk_bytes));
      return;
    }
    nccl->check(nccl->group_start(), "group start");
    for (int r = 0; r < P; ++r) {
      GWB_CUDA(cudaSetDevice(devices[r]));
      uint8_t* base = buf[r].as<uint8_t>();
      nccl->check(nccl->all_gather(base + r * chunk_bytes, base, chunk_bytes, ncclUint8, comms[r],
                                 eng[r]->stream()),
                 "all-gather");
    }
    nccl->check(nccl->group_end(), "group end");
  };
  auto reduce_diag = [&]() {
    if (emulate) {
      sync_all();
      double dsum[kDiag] = {0}, emax[kErr];
      for (int q = 0; q < kErr; ++q) emax[q] = -INFINITY;
      for (int r = 0; r < P; ++r) {
        double d[kDiag], e[kErr];
        GWB_CUDA(cudaMemcpy(d, diag[r].p, sizeof(d), cudaMemcpyDeviceToHost));
        GWB_CUDA(cudaMemcpy(e, err[r].p, sizeof(e), cudaMemcpyDeviceToHost));
        for (int q = 0; q < kDiag; ++q) dsum[q] += d[q];
        for (int q = 0; q < kErr; ++q) emax[q] = std::max(emax[q], e[q]);
      }
      for (int r = 0; r < P; ++r) {
        GWB_CUDA(cudaMemcpy(diag[r].p, dsum, sizeof(dsum), cudaMemcpyHostToDevice));
        GWB_CUDA(cudaMemcpy(err[r].p, emax, sizeof(emax), cudaMemcpyHostToDevice));
      }
      return;
    }
    nccl->check(nccl->group_start(), "group start");
    for (int r = 0; r < P; ++r) {
      GWB_CUDA(cudaSetDevice(devices[r]));
      nccl->check(nccl->all_reduce(diag[r].p, diag[r].p, kDiag, ncclFloat64, ncclSum, comms[r],
                                 eng[r]->stream()),
                 "all-reduce");
      nccl->check(nccl->all_reduce(err[r].p, err[r].p, kErr, ncclFloat64, ncclMax, comms[r],
                                 eng[r]->stream()),
                 "all-reduce");
    }
    nccl->check(nccl->group_end(), "group end");
  };
  const size_t vt_chunk = static_cast<size_t>(eng[0]->vt_bytes() / P);
  const size_t stats_chunk = static_cast<size_t>(eng[0]->stats_bytes() / P);

  // 3. Iterations (dist.iterate_sharded, all-gather schedule), the agreed
  //    done flag polled every 16 iterations, then the tail record.
  for (int it = 1; it <= cfg.max_iters; ++it) {
    all_phase(0);
    gather(vt, vt_chunk);
    all_phase(1);
    all_phase(2);
    gather(vt, vt_chunk);
    all_phase(3);
    gather(stats, stats_chunk);
    all_phase(4);
    reduce_diag();
    all_phase(5);
    if (it % 16 == 0 || it == cfg.max_iters) {
      if (eng[0]->status().done) break;
    }
  }
  DevStatus st = eng[0]->status();
  if (!st.flags) {
    all_phase(6);
    gather(vt, vt_chunk);
    all_phase(7);
    reduce_diag();
    all_phase(8);
  }
  for (auto& e : eng) e->sync_parity();
  st = eng[0]->status();
  if (st.flags) return st;

  // 4. Outputs: rows of π, w (fp64) into the column-major host layout.
  const int used = st.iter - 1;
  if (records) {
    const std::vector<DevRecord> r = eng[0]->records(used);
    records->assign(static_cast<size_t>(used), HostRecord{});
    for (int k = 1; k <= used; ++k) {
      const DevRecord& d = r[k];
      HostRecord& h = (*records)[k - 1];
      h.objective = -0.25 * (d.mpi_pi + 2.0 * d.mpi_w + d.mw_w);
      h.marginal_infeasibility = 0.5 * std::sqrt(d.col_sq) / static_cast<double>(m) +
                                 0.5 * std::sqrt(d.row_sq) / static_cast<double>(n);
      h.split_gap = std::sqrt(d.split_sq);
      h.rel_change = std::sqrt(d.diff_sq) / std::sqrt(d.wold_sq);
      h.elapsed = d.elapsed;
    }
  }
  std::vector<double> pr, wr;
  for (int r = 0; r < P; ++r) {
    const int64_t rb = eng[r]->row_begin(), rv = eng[r]->rows_valid();
    if (rv <= 0) continue;
    pr.assign(static_cast<size_t>(rv * m), 0.0);
    wr.assign(static_cast<size_t>(rv * m), 0.0);
    eng[r]->rows(pr.data(), wr.data());
    for (int64_t i = 0; i < rv; ++i)
      for (int64_t j = 0; j < m; ++j) {
        const double p = pr[i * m + j], w = wr[i * m + j];
        const int64_t o = j * n + rb + i;
        if (out_pi) out_pi[o] = p;
        if (out_w) out_w[o] = w;
        if (out_final) out_final[o] = 0.5 * (p + w);
      }
  }
  return st;
}

}  // namespace gwb

// ---------------------------------------------------------------------------
// C-ABI (include/gwb_ext.h)
// ---------------------------------------------------------------------------
struct gwb_shard {
  std::unique_ptr<gwb::ShardEngine> eng;
  int64_t n, m;
};

namespace {
template <class F>
int32_t shard_guard(gwb_status* st, F&& f) {
  try {
    f();
    if (st) std::memset(st, 0, sizeof(*st));
    return GWB_OK;
  } catch (const gwb::ShardConfigError& e) {
    if (st) {
      std::memset(st, 0, sizeof(*st));
      st->code = GWB_ERR_CONFIG;
      std::snprintf(st->message, sizeof(st->message), "%s", e.what());
    }
    return GWB_ERR_CONFIG;
  } catch (const std::exception& e) {
    if (st) {
      std::memset(st, 0, sizeof(*st));
      st->code = GWB_ERR_RUNTIME;
      std::snprintf(st->message, sizeof(st->message), "%s", e.what());
    }
    return GWB_ERR_RUNTIME;
  }
}
}  // namespace

extern "C" {

int32_t gwb_shard_create(const gwb_config* cfg, int64_t n, int64_t m, int32_t rank, int32_t world,
                         int32_t device, void* stream, gwb_shard** out, gwb_status* st) {
  return shard_guard(st, [&] {
    if (!cfg || n < 1 || m < 1 || world < 1 || rank < 0 || rank >= world)
      throw std::invalid_argument("gwb_shard_create: bad arguments");
    if (cfg->precision == GWB_PREC_SPARSE || cfg->precision == GWB_PREC_FP32 ||
        cfg->precision == GWB_PREC_F16X3)
      throw std::invalid_argument(
          "gwb_shard_create: the sparse, fp32 and f16x3 chains are single-GPU only");
    if (cfg->geometry != GWB_ENTROPY)
      throw std::invalid_argument("gwb_shard_create: the quadratic geometry is single-GPU only");
    if (cfg->record_residual)  // Dykstra on a row shard would need per-sweep column exchanges
      throw std::invalid_argument("gwb_shard_create: record_residual is single-GPU only");
    auto* s = new gwb_shard();
    s->n = n;
    s->m = m;
    s->eng.reset(new gwb::ShardEngine(*cfg, n, m, rank, world, device,
                                      static_cast<cudaStream_t>(stream)));
    *out = s;
  });
}

int32_t gwb_shard_layout(gwb_shard* s, int64_t* rows_per_shard, int64_t* row_begin,
                         int64_t* rows_valid, int32_t* planes, int32_t* elem_bytes,
                         int64_t* vt_bytes, int64_t* stats_bytes, gwb_status* st) {
  return shard_guard(st, [&] {
    *rows_per_shard = s->eng->rows_per_shard();
    *row_begin = s->eng->row_begin();
    *rows_valid = s->eng->rows_valid();
    *planes = s->eng->planes();
    *elem_bytes = s->eng->esize();
    *vt_bytes = s->eng->vt_bytes();
    *stats_bytes = s->eng->stats_bytes();
  });
}

int32_t gwb_shard_set_comm(gwb_shard* s, void* vt_gather, void* col_stats, double* diag,
                           double* err, gwb_status* st) {
  return shard_guard(st, [&] { s->eng->set_comm(vt_gather, col_stats, diag, err); });
}

int32_t gwb_shard_load_device(gwb_shard* s, const float* dx_rows, int64_t ldx, const float* dy,
                              int64_t ldy, const float* mu_rows, const float* nu, gwb_status* st) {
  return shard_guard(st, [&] { s->eng->load(dx_rows, ldx, dy, ldy, mu_rows, nu); });
}

int32_t gwb_shard_set_marginals64(gwb_shard* s, const double* mu_rows, const double* nu,
                                  gwb_status* st) {
  return shard_guard(st, [&] {
    if (!s || !nu) throw std::invalid_argument("gwb_shard_set_marginals64: null argument");
    s->eng->set_marginals64(mu_rows, nu);
  });
}

int32_t gwb_shard_set_iterate_bound(gwb_shard* s, double x_max, gwb_status* st) {
  return shard_guard(st, [&] {
    if (!(x_max > 0.0) || !std::isfinite(x_max))
      throw std::invalid_argument("gwb_shard_set_iterate_bound: bound must be positive and finite");
    s->eng->set_iterate_bound(x_max);
  });
}

int32_t gwb_shard_reset(gwb_shard* s, gwb_status* st) {
  return shard_guard(st, [&] { s->eng->reset(); });
}

int32_t gwb_shard_phase(gwb_shard* s, int32_t phase, gwb_status* st) {
  return shard_guard(st, [&] { s->eng->phase(phase); });
}

int32_t gwb_shard_gemm2_chunk(gwb_shard* s, int32_t src, int32_t tail, gwb_status* st) {
  return shard_guard(st, [&] { s->eng->gemm2_chunk(src, tail != 0); });
}

int32_t gwb_shard_launches(gwb_shard* s, int64_t* launches) {
  if (!s || !launches) return GWB_ERR_INVALID;
  *launches = s->eng->launches();
  return GWB_OK;
}

int32_t gwb_shard_stream(gwb_shard* s, void** stream, gwb_status* st) {
  return shard_guard(st, [&] { *stream = static_cast<void*>(s->eng->stream()); });
}

int32_t gwb_shard_status(gwb_shard* s, int32_t* done, int32_t* iter, int32_t* flags,
                         int32_t* converged, int32_t* err_iter, int32_t* zero_index,
                         gwb_status* st) {
  return shard_guard(st, [&] {
    const gwb::DevStatus h = s->eng->status();
    *done = h.done;
    *iter = h.iter;
    *flags = h.flags;
    *converged = h.converged;
    *err_iter = h.err_iter;
    *zero_index = h.zero_index;
  });
}

int32_t gwb_shard_finish(gwb_shard* s, gwb_status* st) {
  return shard_guard(st, [&] { s->eng->sync_parity(); });
}

int32_t gwb_shard_records(gwb_shard* s, int32_t count, gwb_record* out, gwb_status* st) {
  return shard_guard(st, [&] {
    const std::vector<gwb::DevRecord> r = s->eng->records(count);
    for (int k = 1; k <= count; ++k) {
      const gwb::DevRecord& d = r[k];
      gwb_record& o = out[k - 1];
      std::memset(&o, 0, sizeof(o));
      o.iter = k;
      o.objective = -0.25 * (d.mpi_pi + 2.0 * d.mpi_w + d.mw_w);
      o.marginal_infeasibility = 0.5 * std::sqrt(d.col_sq) / static_cast<double>(s->m) +
                                 0.5 * std::sqrt(d.row_sq) / static_cast<double>(s->n);
      o.split_gap = std::sqrt(d.split_sq);
      o.rel_change = std::sqrt(d.diff_sq) / std::sqrt(d.wold_sq);
      o.elapsed_seconds = d.elapsed;
    }
  });
}

int32_t gwb_shard_rows(gwb_shard* s, double* pi_rows, double* w_rows, gwb_status* st) {
  return shard_guard(st, [&] { s->eng->rows(pi_rows, w_rows); });
}

int32_t gwb_shard_destroy(gwb_shard* s) {
  delete s;
  return GWB_OK;
}

}  // extern "C"
