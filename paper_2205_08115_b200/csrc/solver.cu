// solver.cu — BAPG device engine (see solver.cuh).
//
// One iteration (reference solvers.cpp:159-212) is 12 launches:
//   half a: GEMM1 Vᵀ = D_Y·Wᵀ, GEMM2 G = D_X·V, row_update (+flag check)
//   half b: GEMM1 Vᵀ = D_Y·Pᵀ, GEMM2 G = D_X·V, col partial/combine/write
//           (+2 flag checks), finalize (trace record + stop rule)
// Every kernel returns immediately once DevStatus::done is set, so chunks of
// iterations are captured once as CUDA graphs and replayed without host
// synchronisation; the host polls `done` two chunks behind.
#include "solver.cuh"

#include "standalone.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>

namespace gwb {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s at %s", cudaGetErrorString(e), what);
    throw CudaError(buf);
  }
}

namespace {

constexpr int kChunkIters = 16;  // iterations per captured graph (even)

template <class T>
T* dalloc(cudaStream_t s, size_t count) {
  // Stream-ordered allocation + zero fill on the engine's own stream: ordered
  // with every later kernel, and served from the device's memory pool on
  // repeated solves (pool_keep) instead of fresh cudaMalloc/cudaFree.
  void* p = nullptr;
  GWB_CUDA(cudaMallocAsync(&p, count * sizeof(T) + 256, s));
  GWB_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T) + 256, s));
  return static_cast<T*>(p);
}

void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

}  // namespace

// Keep freed stream-ordered memory cached in the device's default pool (the
// default release threshold of 0 would return it to the driver at every
// synchronisation), so repeated solves — the experiment worker pool — reuse
// their workspace.  Once per device.
void pool_keep(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done.push_back(device);
}

namespace {

}  // namespace

int resolve_precision(int requested, bool bf16_exact, bool f16_exact, bool quadratic) {
  if (requested != GWB_PREC_AUTO) return requested;
  // Quadratic geometry: the simplex projection changes its support
  // discontinuously, so the BAPG map amplifies fp32-level differences near
  // convergence (measured: ×2.4 per iteration on uniform-marginal 0/1
  // graphs, where projection inputs tie exactly).  It keeps the 24-bit
  // bf16x3 chain with separate plane passes (tests/test_gpu_quadratic.py,
  // tools/quad_probe.py).
  if (quadratic) return bf16_exact ? GWB_PREC_BF16X3 : GWB_PREC_3XTF32;
  // AUTO (measured on B200): a split-operand chain with fp32
  // accumulate, at least as precise as 3xTF32.  When both structure
  // matrices are exact in fp16 (0/1 graphs) it runs as f16x2 — D × (hi +
  // lo) fp16 planes of the power-of-two-scaled iterate, 22-bit operands in
  // 2 kind::f16 passes; exact in bf16 only: bf16x3 (24-bit, 3 passes);
  // otherwise 3xTF32.  1xTF32 misses the 1e-5 objective bound and bf16x2
  // (16-bit operands) is reduced precision; both stay explicit opt-ins.
  if (f16_exact) return GWB_PREC_F16X2;
  // Weighted D: both operands split into scaled fp16 hi/lo planes, 3
  // kind::f16 passes.  The kind::tf32 MMA's truncating accumulation biased
  // 3xTF32's chain by ~1e-6 relative, which c2 (ρ = 0.05, 1000 iterations)
  // amplified to 3e-4 of the coupling's scale; kind::f16 accumulates with
  // ~30× less bias, at half the passes' cost.
  return bf16_exact ? GWB_PREC_BF16X3 : GWB_PREC_F16X3;
}

BapgEngine::BapgEngine(int device, int64_t n, int64_t m, double rho, int precision,
                       int max_iters, cudaStream_t stream)
    : device_(device),
      n_(n),
      m_(m),
      ldn_(round_up(n, 32)),
      ldm_(round_up(m, 32)),
      rho_(rho),
      precision_(precision),
      max_iters_(max_iters),
      stream_(stream) {
  GWB_CUDA(cudaSetDevice(device_));
  if (!stream_) {
    GWB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    own_stream_ = true;
  }
  pool_keep(device_);
  alloc();
}

BapgEngine::~BapgEngine() {
  cudaSetDevice(device_);
  cudaStreamSynchronize(stream_);
  destroy_graphs();
  for (int q = 0; q < 2; ++q) {
    gemm_plan_destroy(g1_[q][0]);
    if (q == 0) gemm_plan_destroy(g1_[q][1]);
    gemm_plan_destroy(g1_tail_[q]);
  }
  gemm_plan_destroy(g2_);
  gemm_plan_destroy(g2_tail_);
  csr_free(cx_);
  csr_free(cy_);
  skinny_tc_plan_destroy(stc_, stream_);
  skinny_tc_plan_destroy(stc_tail_, stream_);
  skinny_tc_plan_destroy(stc_b_, stream_);
  dfree(Vs_, stream_);
  dfree(DyT_, stream_);
  dfree(Dxp_, stream_);
  dfree(Vtp_, stream_);
  dfree(Vtp2_, stream_);
  for (void* p : std::initializer_list<void*>{
           Dx_, Dx_aux_, Dy_, Dy_aux_, Dx_bf_, Dy_bf_, P_, P_aux_, W_[0], W_[1], W_aux_[0],
           W_aux_[1], P64_, W64_[0], W64_[1], Vt_,
           Vt_aux_, G_, mu32_, nu32_, mu64_, nu64_, row_part_, cw_part_, col_pmax_, col_psum_,
           col_max_, col_scale_, col_psump_, col_dev_, st_, rec_, f16_g1_rs_, f16_g2_cs_,
           cb1_pi_, cb1_w_[0], cb1_w_[1], cb2_, Dxc_, Dyc_})
    dfree(p, stream_);
  if (h_done_) cudaFreeHost(h_done_);
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto& mk : ev_marks_) {
    cudaEventDestroy(mk.second.first);
    cudaEventDestroy(mk.second.second);
  }
  if (own_stream_) cudaStreamDestroy(stream_);
}

void BapgEngine::alloc() {
  const size_t nm = static_cast<size_t>(n_) * ldm_;
  Dx_ = dalloc<float>(stream_, static_cast<size_t>(n_) * ldn_);
  Dy_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldm_);
  P_ = dalloc<float>(stream_, nm);
  // Operand copies hold one fp32 plane (TF32 modes) or up to three bf16
  // planes (bf16x3): size them for 6 B/element.
  P_aux_ = dalloc<float>(stream_, nm * 3 / 2);
  for (int q = 0; q < 2; ++q) {
    W_[q] = dalloc<float>(stream_, nm);
    W_aux_[q] = dalloc<float>(stream_, nm * 3 / 2);
  }
  P64_ = dalloc<double>(stream_, nm);
  for (int q = 0; q < 2; ++q) W64_[q] = dalloc<double>(stream_, nm);
  Vt_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldn_);
  if (precision_ != GWB_PREC_TF32)
    Vt_aux_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldn_ * 3 / 2);
  G_ = dalloc<float>(stream_, nm);
  mu32_ = dalloc<float>(stream_, ldn_);
  nu32_ = dalloc<float>(stream_, ldm_);
  mu64_ = dalloc<double>(stream_, ldn_);
  nu64_ = dalloc<double>(stream_, ldm_);
  row_part_ = dalloc<RowPart>(stream_, n_);
  cw_part_ = dalloc<ColWritePart>(stream_, n_);
  // Column-pass chunking: ~16 CTAs per SM (large n), so the column-partial
  // grid balances across the 148 SMs (4 per SM left 628 CTAs at c4: 4.24
  // waves, the busiest SMs 18% above the mean).  GWB_COL_CTAS_PER_SM (A/B).
  const int64_t col_blocks = (m_ + 127) / 128;
  static const int64_t col_per_sm = [] {
    const char* e = std::getenv("GWB_COL_CTAS_PER_SM");
    return static_cast<int64_t>(e && std::atoi(e) > 0 ? std::atoi(e) : 16);
  }();
  chunks_ = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>((n_ + 63) / 64, (col_per_sm * 148 + col_blocks - 1) / col_blocks)));
  col_pmax_ = dalloc<double>(stream_, static_cast<size_t>(chunks_) * m_);
  col_psum_ = dalloc<double>(stream_, static_cast<size_t>(chunks_) * m_);
  col_psump_ = dalloc<double>(stream_, static_cast<size_t>(chunks_) * m_);
  col_max_ = dalloc<double>(stream_, ldm_);
  col_scale_ = dalloc<double>(stream_, ldm_);
  col_dev_ = dalloc<double>(stream_, ldm_);
  st_ = dalloc<DevStatus>(stream_, 1);
  rec_ = dalloc<DevRecord>(stream_, static_cast<size_t>(max_iters_) + 2);
  GWB_CUDA(cudaMallocHost(&h_done_, 4 * sizeof(int)));
}

BapgDev BapgEngine::dev_view(int q) const {
  BapgDev d;
  std::memset(&d, 0, sizeof(d));
  d.n = n_;
  d.m = m_;
  d.ld = ldm_;
  d.inv_rho = static_cast<float>(1.0 / rho_);
  d.inv_rho64 = 1.0 / rho_;
  d.G = G_;
  d.mu = mu32_;
  d.nu = nu32_;
  d.mu64 = mu64_;
  d.nu64 = nu64_;
  d.P64 = quadratic() ? nullptr : P64_;  // null selects fp32 semantics (quadratic.cu)
  d.W64 = W64_[q];
  d.W64_new = W64_[1 - q];
  // fp32 copies only where a consumer reads them; the raw-iterate chains
  // (sparse, skinny) take no operand planes.
  d.P = needs_copy() ? P_ : nullptr;
  d.P_aux = no_planes() ? nullptr : P_aux_;
  d.W = W_[q];
  d.W_new = needs_copy() ? W_[1 - q] : nullptr;
  d.W_aux = no_planes() ? nullptr : W_aux_[1 - q];
  d.aux_mode = aux_mode();
  d.aux_scale = aux_scale();
  d.plane = n_ * ldm_;
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
  d.max_rec = max_iters_;
  d.wsum_bias = center_ ? cb1_w_[1 - q] : nullptr;
  d.wsum_factor = cb1_factor();
  return d;
}

void BapgEngine::prepare_d() {
  // Exactness / max of each structure matrix decides the operand copies.
  float* d_max = dalloc<float>(stream_, 2);
  int* d_inexact = dalloc<int>(stream_, 2);
  launch_analyze(Dx_, n_, n_, ldn_, d_max, d_inexact, stream_);
  launch_analyze(Dy_, m_, m_, ldm_, d_max + 1, d_inexact + 1, stream_);
  float h_max[2];
  int h_inexact[2];
  GWB_CUDA(cudaMemcpyAsync(h_max, d_max, sizeof(h_max), cudaMemcpyDeviceToHost, stream_));
  GWB_CUDA(cudaMemcpyAsync(h_inexact, d_inexact, sizeof(h_inexact), cudaMemcpyDeviceToHost, stream_));
  GWB_CUDA(cudaStreamSynchronize(stream_));
  dfree(d_max, stream_);
  dfree(d_inexact, stream_);
  dx_exact_ = (h_inexact[0] & 1) == 0;
  dy_exact_ = (h_inexact[1] & 1) == 0;
  // Skinny problems (m ≤ 32, config 3).  With an exact-bf16 D_X (0/1
  // graphs) AUTO / BF16X3 run the bf16x3 chain as FP32-pipe GEMM1 (K = m)
  // writing Vᵀ planes + tensor-core GEMM2 streaming D_X (skinny_tc.cu);
  // otherwise AUTO takes the FP32-pipe chain (skinny.cu).  An explicit
  // GWB_PREC_FP32 with larger m resolves like AUTO.
  if (precision_ == GWB_PREC_FP32 && m_ > kSkinnyMaxN) precision_ = GWB_PREC_AUTO;
  skinny_tc_plan_destroy(stc_, stream_);
  skinny_tc_plan_destroy(stc_tail_, stream_);
  skinny_tc_plan_destroy(stc_b_, stream_);
  stc_ = stc_tail_ = stc_b_ = nullptr;
  skinny_tc_ = false;
  if (m_ <= kSkinnyMaxN && (h_inexact[0] & 2) == 0 &&
      (precision_ == GWB_PREC_AUTO || precision_ == GWB_PREC_BF16X3)) {
    destroy_graphs();
    precision_ = GWB_PREC_BF16X3;
    skinny_tc_ = true;
    if (!DyT_) DyT_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldm_);
    launch_transpose(Dy_, m_, m_, ldm_, DyT_, ldm_, stream_);
    if (!Dxp_) Dxp_ = dalloc<uint8_t>(stream_, static_cast<size_t>(skinny_tc_packed_a_bytes(n_, n_)));
    skinny_tc_pack_a(Dx_, ldn_, n_, n_, Dxp_, stream_);
    vtp_plane_ = skinny_tc_packed_b_elems(n_);
    if (!Vtp_) Vtp_ = dalloc<uint16_t>(stream_, static_cast<size_t>(3 * vtp_plane_));  // zero tails
    stc_ = skinny_tc_plan_create(Dxp_, Vtp_, 3, G_, ldm_, n_, static_cast<int>(m_), n_, &st_->done,
                                 stream_);
    stc_tail_ = skinny_tc_plan_create(Dxp_, Vtp_, 3, G_, ldm_, n_, static_cast<int>(m_), n_,
                                      &st_->flags, stream_);
    // Fused schedule (entropy geometry): half-step a's GEMM2 also runs the
    // row update and half-step b's GEMM1 (skinny_tc_launch_fused_a), writing
    // the second plane buffer, which half-step b's GEMM2 streams.
    // GWB_SKINNY_UNFUSED=1 keeps one launch per stage (A/B knob).
    static const bool unfused_env = [] {
      const char* e = std::getenv("GWB_SKINNY_UNFUSED");
      return e && e[0] == '1';
    }();
    if (!unfused_env && skinny_tc_can_fuse(stc_)) {
      if (!Vtp2_) Vtp2_ = dalloc<uint16_t>(stream_, static_cast<size_t>(3 * vtp_plane_));
      stc_b_ = skinny_tc_plan_create(Dxp_, Vtp2_, 3, G_, ldm_, n_, static_cast<int>(m_), n_,
                                     &st_->done, stream_);
    }
    GWB_CUDA(cudaStreamSynchronize(stream_));
    return;
  }
  if (precision_ == GWB_PREC_AUTO && m_ <= kSkinnyMaxN) precision_ = GWB_PREC_FP32;
  if (precision_ == GWB_PREC_FP32) {
    destroy_graphs();
    if (!Vs_) Vs_ = dalloc<float>(stream_, static_cast<size_t>(n_) * ldm_);
    if (!DyT_) DyT_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldm_);
    launch_transpose(Dy_, m_, m_, ldm_, DyT_, ldm_, stream_);
    GWB_CUDA(cudaStreamSynchronize(stream_));
    return;
  }
  if (precision_ == GWB_PREC_SPARSE) {
    destroy_graphs();
    csr_free(cx_);
    csr_free(cy_);
    cx_ = csr_from_dense(Dx_, n_, ldn_, stream_);
    cy_ = csr_from_dense(Dy_, m_, ldm_, stream_);
    return;
  }
  const bool bf16_exact = (h_inexact[0] & 2) == 0 && (h_inexact[1] & 2) == 0;
  const bool f16_exact = (h_inexact[0] & 4) == 0 && (h_inexact[1] & 4) == 0;
  if (precision_ == GWB_PREC_AUTO)
    precision_ = resolve_precision(GWB_PREC_AUTO, bf16_exact, f16_exact, quadratic());
  // Split-plane chains need exactly representable structure matrices (0/1
  // graphs); otherwise fall back to bf16x3 (f16x2 only) or 3xTF32, which
  // splits both operands.
  if (precision_ == GWB_PREC_F16X2 && !f16_exact) precision_ = GWB_PREC_BF16X3;
  if ((precision_ == GWB_PREC_BF16X3 || precision_ == GWB_PREC_BF16X2) && !bf16_exact)
    precision_ = GWB_PREC_3XTF32;
  if (precision_ != GWB_PREC_TF32 && !Vt_aux_)
    Vt_aux_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldn_ * 3 / 2);
  // Weighted D (f16x3, or a TF32 chain on inexact D) runs centred, entropy
  // geometry only (the column write pass provides rowsum(w)).
  center_ = !quadratic() &&
            (split_d() || ((precision_ == GWB_PREC_3XTF32 || precision_ == GWB_PREC_TF32) &&
                           !(dx_exact_ && dy_exact_)));
  ctr_x_ = center_ ? 0.5 * static_cast<double>(h_max[0]) : 0.0;
  ctr_y_ = center_ ? 0.5 * static_cast<double>(h_max[1]) : 0.0;
  if (center_) {
    if (!cb1_pi_) cb1_pi_ = dalloc<float>(stream_, ldn_);
    for (int q = 0; q < 2; ++q)
      if (!cb1_w_[q]) cb1_w_[q] = dalloc<float>(stream_, ldn_);
    if (!cb2_) cb2_ = dalloc<float>(stream_, ldm_);
  }
  if (bf16()) {
    // One bf16 / fp16 plane per structure matrix (2 B/element), two for f16x3.
    const size_t per = split_d() ? 1 : 2;  // elements per float
    dfree(Dx_bf_, stream_);
    dfree(Dy_bf_, stream_);
    Dx_bf_ = dalloc<float>(stream_, static_cast<size_t>(n_) * ldn_ / per + 16);
    Dy_bf_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldm_ / per + 16);
    if (f16()) {
      if (split_d()) {
        // D·2^s ≤ 2^14 keeps both fp16 planes inside the normal range.
        auto shift = [](float mx) {
          return mx > 0.f ? 14 - static_cast<int>(std::ceil(std::log2(static_cast<double>(mx)))) : 0;
        };
        // Centred: planes of (D − c)·2^s from fp64, |D − c| ≤ c.
        sdx_ = shift(static_cast<float>(ctr_x_));
        sdy_ = shift(static_cast<float>(ctr_y_));
        launch_center_copies(Dx_, n_, n_, ldn_, ctr_x_, nullptr, Dx_bf_, 5, std::ldexp(1.0f, sdx_),
                             stream_);
        launch_center_copies(Dy_, m_, m_, ldm_, ctr_y_, nullptr, Dy_bf_, 5, std::ldexp(1.0f, sdy_),
                             stream_);
      } else {
        sdx_ = sdy_ = 0;
        launch_to_f16(Dx_, n_, n_, ldn_, Dx_bf_, stream_);
        launch_to_f16(Dy_, m_, m_, ldm_, Dy_bf_, stream_);
      }
      f16_s1_ = 14 - static_cast<int>(std::ceil(std::log2(std::max(x_max_, 1e-30))));
      if (!f16_g1_rs_) f16_g1_rs_ = dalloc<float>(stream_, ldm_);
      if (!f16_g2_cs_) f16_g2_cs_ = dalloc<float>(stream_, ldm_);
      launch_f16_scales(Dy_, m_, ldm_, static_cast<float>(x_max_), f16_s1_, f16_g1_rs_, f16_g2_cs_,
                        stream_, sdy_, sdx_);
    } else {
      launch_to_bf16(Dx_, n_, n_, ldn_, Dx_bf_, stream_);
      launch_to_bf16(Dy_, m_, m_, ldm_, Dy_bf_, stream_);
    }
    if (center_) launch_row_bias64(mu64_, n_, 1, 1, cb1_factor(), cb1_pi_, stream_);
    build_plans();
    return;
  }
  const int mode = precision_ == GWB_PREC_TF32 ? 1 : 2;
  if (center_) {
    // TF32 chains on centred D: hi = fp32(D − c) (3xTF32) and the residual
    // or the rna copy (1xTF32), both from fp64 D − c.
    if (!Dx_aux_) Dx_aux_ = dalloc<float>(stream_, static_cast<size_t>(n_) * ldn_);
    if (!Dy_aux_) Dy_aux_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldm_);
    if (mode == 2) {
      if (!Dxc_) Dxc_ = dalloc<float>(stream_, static_cast<size_t>(n_) * ldn_);
      if (!Dyc_) Dyc_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldm_);
    }
    launch_center_copies(Dx_, n_, n_, ldn_, ctr_x_, mode == 2 ? Dxc_ : nullptr, Dx_aux_, mode, 1.0f,
                         stream_);
    launch_center_copies(Dy_, m_, m_, ldm_, ctr_y_, mode == 2 ? Dyc_ : nullptr, Dy_aux_, mode, 1.0f,
                         stream_);
    launch_row_bias64(mu64_, n_, 1, 1, cb1_factor(), cb1_pi_, stream_);
    build_plans();
    return;
  }
  if (!dx_exact_) {
    if (!Dx_aux_) Dx_aux_ = dalloc<float>(stream_, static_cast<size_t>(n_) * ldn_);
    launch_tf32_aux(Dx_, n_, n_, ldn_, Dx_aux_, mode, stream_);
  }
  if (!dy_exact_) {
    if (!Dy_aux_) Dy_aux_ = dalloc<float>(stream_, static_cast<size_t>(m_) * ldm_);
    launch_tf32_aux(Dy_, m_, m_, ldm_, Dy_aux_, mode, stream_);
  }
  build_plans();
}

void BapgEngine::build_plans() {
  destroy_graphs();
  for (int q = 0; q < 2; ++q) {
    gemm_plan_destroy(g1_[q][0]);
    if (q == 0) gemm_plan_destroy(g1_[q][1]);
    g1_[q][1] = nullptr;
    gemm_plan_destroy(g1_tail_[q]);
  }
  gemm_plan_destroy(g2_);
  gemm_plan_destroy(g2_tail_);

  const int* done = &st_->done;
  const int* flags = &st_->flags;
  if (bf16()) {
    // Split-plane chain: A = D (exact bf16 / fp16), B = planes of W / P / V.
    // f16x2 carries power-of-two scales: GEMM1's B planes hold X·2^s1, its
    // row scale maps row i of the accumulator to Vᵀ·2^σ_i, GEMM2's column
    // scale 2^−σ_j returns G unscaled.
    const int planes = precision_ == GWB_PREC_BF16X3 ? 3 : 2;
    const bool f16 = this->f16();
    auto planes_of = [](float* base, int64_t plane_elems, int k) {
      return static_cast<void*>(reinterpret_cast<uint16_t*>(base) + k * plane_elems);
    };
    auto gemm1 = [&](float* X_aux, const float* bias, const int* skip) {
      GemmDesc d;
      d.a_const = true;  // A = a structure matrix (constant)
      d.M = m_;
      d.N = n_;
      d.K = m_;
      d.col_bias = center_ ? bias : nullptr;
      d.rowsums = center_;
      d.bf16_planes = planes;
      d.a_bf16 = Dy_bf_;
      if (split_d()) {
        // Separate pass stages, promotion every 2 k-blocks (DESIGN.md §4a:
        // the measured-best c2 schedule; every 1 k-block halves the bias but
        // drains TMEM every 4 MMAs).
        d.a_bf16_lo = reinterpret_cast<uint16_t*>(Dy_bf_) + m_ * ldm_;
      }
      d.lda = ldm_;
      for (int k = 0; k < planes; ++k) d.b_bf16[k] = planes_of(X_aux, n_ * ldm_, k);
      d.ldb = ldm_;
      d.c_planes = planes;
      for (int k = 0; k < planes; ++k) d.c_bf16[k] = planes_of(Vt_aux_, m_ * ldn_, k);
      d.ldc = ldn_;
      d.skip = skip;
      d.f16 = f16;
      if (f16) d.row_scale = f16_g1_rs_;
      d.fuse_planes = !quadratic();  // separate plane passes keep exact ties (see resolve_precision)
      d.fuse_split_a = center_;
      return gemm_plan_create(d);
    };
    auto gemm2 = [&](const int* skip) {
      GemmDesc d;
      d.a_const = true;  // A = a structure matrix (constant)
      d.M = n_;
      d.N = m_;
      d.K = n_;
      d.bf16_planes = planes;
      d.a_bf16 = Dx_bf_;
      if (split_d()) {
        d.a_bf16_lo = reinterpret_cast<uint16_t*>(Dx_bf_) + n_ * ldn_;
      }
      d.lda = ldn_;
      for (int k = 0; k < planes; ++k) d.b_bf16[k] = planes_of(Vt_aux_, m_ * ldn_, k);
      d.ldb = ldn_;
      d.c = G_;
      d.ldc = ldm_;
      d.skip = skip;
      d.f16 = f16;
      d.col_bias = center_ ? cb2_ : nullptr;
      if (f16) d.col_scale = f16_g2_cs_;
      d.fuse_planes = !quadratic();
      d.fuse_split_a = center_;
      return gemm_plan_create(d);
    };
    for (int q = 0; q < 2; ++q) {
      g1_[q][0] = gemm1(W_aux_[q], cb1_w_[q], done);
      g1_tail_[q] = gemm1(W_aux_[q], cb1_w_[q], flags);
    }
    g1_[0][1] = gemm1(P_aux_, cb1_pi_, done);
    g1_[1][1] = g1_[0][1];
    g2_ = gemm2(done);
    g2_tail_ = gemm2(flags);
    return;
  }
  const bool tf32 = precision_ == GWB_PREC_TF32;
  // A operands (structure matrices).
  const float* ax = Dx_;
  const float* ax_lo = nullptr;
  const float* ay = Dy_;
  const float* ay_lo = nullptr;
  if (center_) {
    ax = tf32 ? Dx_aux_ : Dxc_;
    ax_lo = tf32 ? nullptr : Dx_aux_;
    ay = tf32 ? Dy_aux_ : Dyc_;
    ay_lo = tf32 ? nullptr : Dy_aux_;
  } else {
    if (!dx_exact_) {
      if (tf32) ax = Dx_aux_;
      else ax_lo = Dx_aux_;
    }
    if (!dy_exact_) {
      if (tf32) ay = Dy_aux_;
      else ay_lo = Dy_aux_;
    }
  }
  auto gemm1 = [&](float* X, float* X_aux, const float* bias, const int* skip) {
    GemmDesc d;
    d.a_const = true;  // A = a structure matrix (constant)
    d.M = m_;
    d.N = n_;
    d.K = m_;
    d.col_bias = center_ ? bias : nullptr;
    d.rowsums = center_;
    d.a = ay;
    d.a_lo = ay_lo;
    d.lda = ldm_;
    d.b = tf32 ? X_aux : X;
    d.b_lo = tf32 ? nullptr : X_aux;
    d.ldb = ldm_;
    d.c = Vt_;
    d.c_aux = Vt_aux_;
    d.ldc = ldn_;
    d.aux_mode = tf32 ? 1 : 2;
    d.skip = skip;
    d.three_pass = !tf32;
    return gemm_plan_create(d);
  };
  auto gemm2 = [&](const int* skip) {
    GemmDesc d;
    d.a_const = true;  // A = a structure matrix (constant)
    d.M = n_;
    d.N = m_;
    d.K = n_;
    d.a = ax;
    d.a_lo = ax_lo;
    d.lda = ldn_;
    d.b = Vt_;
    d.b_lo = tf32 ? nullptr : Vt_aux_;
    d.ldb = ldn_;
    d.c = G_;
    d.ldc = ldm_;
    d.aux_mode = 0;
    d.skip = skip;
    d.three_pass = !tf32;
    d.col_bias = center_ ? cb2_ : nullptr;
    return gemm_plan_create(d);
  };
  for (int q = 0; q < 2; ++q) {
    g1_[q][0] = gemm1(W_[q], W_aux_[q], cb1_w_[q], done);
    g1_tail_[q] = gemm1(W_[q], W_aux_[q], cb1_w_[q], flags);
  }
  g1_[0][1] = gemm1(P_, P_aux_, cb1_pi_, done);
  g1_[1][1] = g1_[0][1];
  g2_ = gemm2(done);
  g2_tail_ = gemm2(flags);
}

void BapgEngine::load_host(const double* dx, const double* dy, const double* mu,
                           const double* nu) {
  GWB_CUDA(cudaSetDevice(device_));
  const int64_t big = std::max(n_ * n_, m_ * m_);
  double* stage = nullptr;
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&stage), static_cast<size_t>(big) * sizeof(double), stream_));
  GWB_CUDA(cudaMemcpyAsync(stage, dx, sizeof(double) * n_ * n_, cudaMemcpyHostToDevice, stream_));
  launch_colmajor64_to_rowmajor32(stage, n_, n_, Dx_, ldn_, stream_);
  GWB_CUDA(cudaMemcpyAsync(stage, dy, sizeof(double) * m_ * m_, cudaMemcpyHostToDevice, stream_));
  launch_colmajor64_to_rowmajor32(stage, m_, m_, Dy_, ldm_, stream_);
  GWB_CUDA(cudaStreamSynchronize(stream_));
  GWB_CUDA(cudaFreeAsync(stage, stream_));
  load_marginals(mu, nu);
}

void BapgEngine::load_graphs(const GraphInput& g, const double* mu, const double* nu) {
  GWB_CUDA(cudaSetDevice(device_));
  build_adjacency(g.ex, g.cx, n_, Dx_, ldn_, stream_);
  build_adjacency(g.ey, g.cy, m_, Dy_, ldm_, stream_);
  load_marginals(mu, nu);
}

void BapgEngine::load_marginals(const double* mu, const double* nu) {
  std::vector<float> mu32(n_), nu32(m_);
  for (int64_t i = 0; i < n_; ++i) mu32[i] = static_cast<float>(mu[i]);
  for (int64_t j = 0; j < m_; ++j) nu32[j] = static_cast<float>(nu[j]);
  x_max_ = 0.0;
  for (int64_t i = 0; i < n_; ++i) x_max_ = std::max(x_max_, std::fabs(mu[i]));
  for (int64_t j = 0; j < m_; ++j) x_max_ = std::max(x_max_, std::fabs(nu[j]));
  GWB_CUDA(cudaMemcpyAsync(mu64_, mu, sizeof(double) * n_, cudaMemcpyHostToDevice, stream_));
  GWB_CUDA(cudaMemcpyAsync(nu64_, nu, sizeof(double) * m_, cudaMemcpyHostToDevice, stream_));
  GWB_CUDA(cudaMemcpyAsync(mu32_, mu32.data(), sizeof(float) * n_, cudaMemcpyHostToDevice, stream_));
  GWB_CUDA(cudaMemcpyAsync(nu32_, nu32.data(), sizeof(float) * m_, cudaMemcpyHostToDevice, stream_));
  prepare_d();
}

void BapgEngine::load_device(const float* dx, int64_t ldx, const float* dy, int64_t ldy,
                             const float* mu, const float* nu) {
  GWB_CUDA(cudaSetDevice(device_));
  GWB_CUDA(cudaMemcpy2DAsync(Dx_, ldn_ * 4, dx, ldx * 4, n_ * 4, n_, cudaMemcpyDeviceToDevice, stream_));
  GWB_CUDA(cudaMemcpy2DAsync(Dy_, ldm_ * 4, dy, ldy * 4, m_ * 4, m_, cudaMemcpyDeviceToDevice, stream_));
  GWB_CUDA(cudaMemcpyAsync(mu32_, mu, sizeof(float) * n_, cudaMemcpyDeviceToDevice, stream_));
  GWB_CUDA(cudaMemcpyAsync(nu32_, nu, sizeof(float) * m_, cudaMemcpyDeviceToDevice, stream_));
  std::vector<float> mu32(n_), nu32(m_);
  GWB_CUDA(cudaMemcpyAsync(mu32.data(), mu, sizeof(float) * n_, cudaMemcpyDeviceToHost, stream_));
  GWB_CUDA(cudaMemcpyAsync(nu32.data(), nu, sizeof(float) * m_, cudaMemcpyDeviceToHost, stream_));
  GWB_CUDA(cudaStreamSynchronize(stream_));
  std::vector<double> mu64(mu32.begin(), mu32.end()), nu64(nu32.begin(), nu32.end());
  x_max_ = 0.0;
  for (double v : mu64) x_max_ = std::max(x_max_, std::fabs(v));
  for (double v : nu64) x_max_ = std::max(x_max_, std::fabs(v));
  GWB_CUDA(cudaMemcpyAsync(mu64_, mu64.data(), sizeof(double) * n_, cudaMemcpyHostToDevice, stream_));
  GWB_CUDA(cudaMemcpyAsync(nu64_, nu64.data(), sizeof(double) * m_, cudaMemcpyHostToDevice, stream_));
  GWB_CUDA(cudaStreamSynchronize(stream_));
  prepare_d();
}

void BapgEngine::reset(const double* w0_host) {
  GWB_CUDA(cudaSetDevice(device_));
  launch_status_reset(st_, stream_);
  // Entropy: w0_host is w⁰ (the caller applied kl_scale).  Quadratic: it is
  // π⁰ (or null for μνᵀ) and w⁰ = euclid_project(π⁰, ν, Cols) on the device
  // (solvers.cpp:152-153), staged through P (overwritten by half-step a).
  if (!quadratic()) {
    // fp64 w⁰ (the caller's kl_scale of π⁰, or μνᵀ), then its copies.
    if (w0_host) {
      double* stage = nullptr;
      GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&stage), sizeof(double) * n_ * m_, stream_));
      GWB_CUDA(cudaMemcpyAsync(stage, w0_host, sizeof(double) * n_ * m_, cudaMemcpyHostToDevice, stream_));
      launch_colmajor64_to_rowmajor64(stage, n_, m_, W64_[0], ldm_, stream_);
      GWB_CUDA(cudaStreamSynchronize(stream_));
      GWB_CUDA(cudaFreeAsync(stage, stream_));
    } else {
      launch_product_coupling64(mu64_, nu64_, n_, m_, ldm_, W64_[0], stream_);
    }
    launch_iterate_copies(W64_[0], n_, m_, ldm_, needs_copy() ? W_[0] : nullptr,
                          no_planes() ? nullptr : W_aux_[0], aux_mode(), aux_scale(), stream_);
    if (center_) launch_row_bias64(W64_[0], n_, m_, ldm_, cb1_factor(), cb1_w_[0], stream_);
    parity_ = 0;
    GWB_CUDA(cudaGetLastError());
    return;
  }
  float* dst = P_;
  if (w0_host) {
    double* stage = nullptr;
    GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&stage), sizeof(double) * n_ * m_, stream_));
    GWB_CUDA(cudaMemcpyAsync(stage, w0_host, sizeof(double) * n_ * m_, cudaMemcpyHostToDevice, stream_));
    launch_colmajor64_to_rowmajor32(stage, n_, m_, dst, ldm_, stream_);
    GWB_CUDA(cudaStreamSynchronize(stream_));
    GWB_CUDA(cudaFreeAsync(stage, stream_));
  } else {
    launch_product_coupling(mu32_, nu32_, n_, m_, ldm_, dst, stream_);
  }
  launch_quad_reset(dev_view(0), P_, W_[0], stream_);
  launch_tf32_aux(W_[0], n_, m_, ldm_, W_aux_[0], aux_mode(), stream_, aux_scale());
  parity_ = 0;
  GWB_CUDA(cudaGetLastError());
}

cudaEvent_t BapgEngine::ev_get() {
  if (!ev_pool_.empty()) {
    cudaEvent_t e = ev_pool_.back();
    ev_pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  GWB_CUDA(cudaEventCreate(&e));
  return e;
}

int64_t BapgEngine::enqueue_half(int q, bool half_b, double rel_tol) {
  const BapgDev d = dev_view(q);
  int64_t launches = 0;
  bool row_fused = false;  // half-step a's row update ran inside the chain's last kernel
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  if (timing_) {
    e0 = ev_get();
    e1 = ev_get();
    e2 = ev_get();
    GWB_CUDA(cudaEventRecord(e0, stream_));
  }
  if (sparse()) {
    // Uᵀ = (D_X·X)ᵀ, then G = (D_Y·Uᵀ)ᵀ: two CSR row-gathers (sparse.cu).
    launch_rowgather(cx_, half_b ? P_ : W_[q], ldm_, m_, Vt_, ldn_, true, &st_->done, stream_);
    launch_rowgather(cy_, Vt_, ldn_, n_, G_, ldm_, true, &st_->done, stream_);
  } else if (skinny_tc_ && stc_b_ && !quadratic()) {
    // Fused schedule: a = {GEMM1 on w, GEMM2 + row update + GEMM1 on the new
    // π}, b = {GEMM2 on the planes half-step a left in Vtp2_}.
    if (!half_b) {
      launch_skinny_planes(W_[q], ldm_, DyT_, ldm_, Vtp_, 3, 0, vtp_plane_, n_,
                           static_cast<int>(m_), m_, &st_->done, stream_);
      skinny_tc_launch_fused_a(stc_, d, DyT_, ldm_, Vtp2_, vtp_plane_, stream_);
      row_fused = true;
    } else {
      skinny_tc_launch(stc_b_, stream_);
      launches -= 1;
    }
  } else if (skinny_tc_) {
    // Vᵀ planes = (X·D_Yᵀ)ᵀ on the FP32 pipes, then G = D_X·V on the tensor cores.
    launch_skinny_planes(half_b ? P_ : W_[q], ldm_, DyT_, ldm_, Vtp_, 3, 0, vtp_plane_, n_,
                         static_cast<int>(m_), m_, &st_->done, stream_);
    skinny_tc_launch(stc_, stream_);
  } else if (fp32()) {
    // V = X·D_Yᵀ, then G = D_X·V on the FP32 pipes (skinny.cu).
    launch_skinny(half_b ? P_ : W_[q], ldm_, DyT_, ldm_, Vs_, ldm_, n_, static_cast<int>(m_), m_,
                  &st_->done, stream_);
    launch_skinny(Dx_, ldn_, Vs_, ldm_, G_, ldm_, n_, static_cast<int>(m_), n_, &st_->done,
                  stream_);
  } else {
    GWB_CUDA(gemm_launch(g1_[q][half_b ? 1 : 0], stream_));
    if (center_) {
      GWB_CUDA(gemm_rowsum_bias(g1_[q][half_b ? 1 : 0], cb2_factor(), cb2_, stream_));
      ++launches;
    }
    GWB_CUDA(gemm_launch(g2_, stream_));
    launches += gemm_launches(g1_[q][half_b ? 1 : 0]) + gemm_launches(g2_) - 2;
  }
  launches += 2;
  if (timing_) GWB_CUDA(cudaEventRecord(e1, stream_));
  if (!half_b) {
    if (quadratic())
      launch_row_quad(d, stream_);
    else if (!row_fused)
      launch_row_update(d, true, stream_);
    launches += quadratic() ? 2 : (row_fused ? 0 : 1);  // quadratic: + its flag check
  } else {
    if (quadratic())
      launch_col_quad(d, stream_);
    else
      launch_col_update(d, stream_);
    launch_finalize(d, rel_tol, false, stream_);
    launches += 4;  // column passes (partial, combine, write / quadratic's) + finalize
  }
  if (timing_) {
    GWB_CUDA(cudaEventRecord(e2, stream_));
    ev_marks_.push_back({0, {e0, e1}});
    ev_marks_.push_back({1, {e1, e2}});
  }
  GWB_CUDA(cudaGetLastError());
  return launches;
}

int64_t BapgEngine::enqueue_iteration(int q, double rel_tol) {
  return enqueue_half(q, false, rel_tol) + enqueue_half(q, true, rel_tol);
}

void BapgEngine::destroy_graphs() {
  for (auto& g : graph_) {
    if (g) cudaGraphExecDestroy(g);
    g = nullptr;
  }
}

int64_t BapgEngine::iterate(int iters, double rel_tol, bool use_graph) {
  GWB_CUDA(cudaSetDevice(device_));
  int64_t launches = 0;
  int done = 0;
  if (use_graph && !timing_) {
    while (iters - done >= kChunkIters) {
      cudaGraphExec_t& ge = graph_[parity_];
      if (!ge) {
        cudaGraph_t g;
        GWB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        int q = parity_;
        graph_launches_ = 0;
        for (int k = 0; k < kChunkIters; ++k) {
          graph_launches_ += enqueue_iteration(q, rel_tol);
          q ^= 1;
        }
        GWB_CUDA(cudaStreamEndCapture(stream_, &g));
        GWB_CUDA(cudaGraphInstantiate(&ge, g, 0));
        GWB_CUDA(cudaGraphDestroy(g));
        graph_iters_ = kChunkIters;
      }
      GWB_CUDA(cudaGraphLaunch(ge, stream_));
      launches += graph_launches_;
      done += kChunkIters;  // even ⇒ parity unchanged
    }
  }
  for (; done < iters; ++done) {
    launches += enqueue_iteration(parity_, rel_tol);
    parity_ ^= 1;
  }
  return launches;
}

void BapgEngine::run(int max_iters, double rel_tol) {
  GWB_CUDA(cudaSetDevice(device_));
  int remaining = max_iters;
  int c = 0;
  cudaEvent_t ev[4];
  for (auto& e : ev) GWB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  bool stop = false;
  while (remaining > 0 && !stop) {
    const int chunk = std::min(remaining, kChunkIters);
    iterate(chunk, rel_tol, true);
    remaining -= chunk;
    GWB_CUDA(cudaMemcpyAsync(&h_done_[c % 4], &st_->done, sizeof(int), cudaMemcpyDeviceToHost, stream_));
    GWB_CUDA(cudaEventRecord(ev[c % 4], stream_));
    if (c >= 2) {
      GWB_CUDA(cudaEventSynchronize(ev[(c - 2) % 4]));
      if (h_done_[(c - 2) % 4]) stop = true;
    }
    ++c;
  }
  GWB_CUDA(cudaStreamSynchronize(stream_));
  for (auto& e : ev) cudaEventDestroy(e);
  // The current w lives in W_[iterations_used % 2] (iteration k writes it).
  const DevStatus s = status();
  parity_ = (s.iter - 1) & 1;
}

DevStatus BapgEngine::run_stepped(int max_iters, double rel_tol,
                                  const std::function<void(int, const DevStatus&)>& after) {
  DevStatus s = status();
  for (int k = 0; k < max_iters; ++k) {
    iterate(1, rel_tol, false);
    s = status();
    if (s.flags) return s;
    after(s.iter - 1, s);
    if (s.converged) break;
  }
  return s;
}

double BapgEngine::residual_of_average(double dykstra_tol) {
  GWB_CUDA(cudaSetDevice(device_));
  const size_t len = static_cast<size_t>(n_) * m_;
  double* pi64 = dalloc<double>(stream_, len);
  double* w64 = dalloc<double>(stream_, len);
  double* work = dalloc<double>(stream_, static_cast<size_t>(std::max(n_, m_)));
  // The reference's fp64 halves: K8 fix-up, then ½(π + w) (solvers.cpp:193).
  iterates_to_colmajor64(parity_, pi64, w64, work);
  launch_average64(pi64, w64, pi64, static_cast<int64_t>(len), stream_);
  auto release = [&] {
    for (void* p : std::initializer_list<void*>{pi64, w64, work}) dfree(p, stream_);
  };
  double r = 0.0;
  try {
    r = luo_tseng_residual_dev(Dx_, ldn_, Dy_, ldm_, pi64, n_, m_, mu64_, nu64_, dykstra_tol,
                               stream_);
  } catch (...) {
    release();
    throw;
  }
  release();
  return r;
}

int64_t BapgEngine::final_csv(const std::function<void(const char*, int64_t)>& sink) {
  GWB_CUDA(cudaSetDevice(device_));
  const DevStatus s = status();
  const int par = s.iter >= 1 ? (s.iter - 1) & 1 : parity_;  // buffer holding the current w
  const size_t len = static_cast<size_t>(n_) * m_;
  double* pi64 = dalloc<double>(stream_, len);
  double* w64 = dalloc<double>(stream_, len);
  double* work = dalloc<double>(stream_, static_cast<size_t>(std::max(n_, m_)));
  iterates_to_colmajor64(par, pi64, w64, work);
  launch_average64(pi64, w64, pi64, static_cast<int64_t>(len), stream_);
  int64_t total = 0;
  try {
    total = coupling_csv_dev(pi64, n_, m_, stream_, sink);
  } catch (...) {
    for (void* p : std::initializer_list<void*>{pi64, w64, work}) dfree(p, stream_);
    throw;
  }
  for (void* p : std::initializer_list<void*>{pi64, w64, work}) dfree(p, stream_);
  return total;
}

void BapgEngine::tail() {
  GWB_CUDA(cudaSetDevice(device_));
  const BapgDev d = dev_view(parity_);
  if (sparse()) {
    launch_rowgather(cx_, W_[parity_], ldm_, m_, Vt_, ldn_, true, &st_->flags, stream_);
    launch_rowgather(cy_, Vt_, ldn_, n_, G_, ldm_, true, &st_->flags, stream_);
  } else if (skinny_tc_) {
    launch_skinny_planes(W_[parity_], ldm_, DyT_, ldm_, Vtp_, 3, 0, vtp_plane_, n_,
                         static_cast<int>(m_), m_, &st_->flags, stream_);
    skinny_tc_launch(stc_tail_, stream_);
  } else if (fp32()) {
    launch_skinny(W_[parity_], ldm_, DyT_, ldm_, Vs_, ldm_, n_, static_cast<int>(m_), m_,
                  &st_->flags, stream_);
    launch_skinny(Dx_, ldn_, Vs_, ldm_, G_, ldm_, n_, static_cast<int>(m_), n_, &st_->flags,
                  stream_);
  } else {
    GWB_CUDA(gemm_launch(g1_tail_[parity_], stream_));
    if (center_) GWB_CUDA(gemm_rowsum_bias(g1_tail_[parity_], cb2_factor(), cb2_, stream_));
    GWB_CUDA(gemm_launch(g2_tail_, stream_));
  }
  launch_row_update(d, false, stream_);
  launch_finalize(d, 0.0, true, stream_);
  GWB_CUDA(cudaGetLastError());
}

DevStatus BapgEngine::status() {
  DevStatus s;
  GWB_CUDA(cudaMemcpyAsync(&s, st_, sizeof(s), cudaMemcpyDeviceToHost, stream_));
  GWB_CUDA(cudaStreamSynchronize(stream_));
  return s;
}

std::vector<HostRecord> BapgEngine::records(int count) {
  std::vector<DevRecord> r(static_cast<size_t>(count) + 1);
  GWB_CUDA(cudaMemcpyAsync(r.data(), rec_, sizeof(DevRecord) * (count + 1), cudaMemcpyDeviceToHost, stream_));
  GWB_CUDA(cudaStreamSynchronize(stream_));
  std::vector<HostRecord> out(static_cast<size_t>(count));
  for (int k = 1; k <= count; ++k) {
    const DevRecord& d = r[k];
    HostRecord& h = out[k - 1];
    // f(½(π+w)) = −¼[⟨Mπ,π⟩ + 2⟨Mπ,w⟩ + ⟨Mw,w⟩]  (D_X, D_Y symmetric)
    h.objective = -0.25 * (d.mpi_pi + 2.0 * d.mpi_w + d.mw_w);
    h.marginal_infeasibility = 0.5 * std::sqrt(d.col_sq) / static_cast<double>(m_) +
                               0.5 * std::sqrt(d.row_sq) / static_cast<double>(n_);
    h.split_gap = std::sqrt(d.split_sq);
    h.rel_change = std::sqrt(d.diff_sq) / std::sqrt(d.wold_sq);
    h.elapsed = d.elapsed;
  }
  return out;
}

void BapgEngine::outputs(double* out_final, double* out_pi, double* out_w) {
  GWB_CUDA(cudaSetDevice(device_));
  const size_t len = static_cast<size_t>(n_) * m_;
  double* pi64 = nullptr;
  double* w64 = nullptr;
  double* work = nullptr;
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&pi64), len * sizeof(double), stream_));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&w64), len * sizeof(double), stream_));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&work), sizeof(double) * std::max(n_, m_), stream_));
  // K8 fix-up: exact fp64 row (π) / column (w) re-projection.
  iterates_to_colmajor64(parity_, pi64, w64, work);
  if (out_pi) GWB_CUDA(cudaMemcpyAsync(out_pi, pi64, len * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  if (out_w) GWB_CUDA(cudaMemcpyAsync(out_w, w64, len * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  if (out_final) {
    launch_average64(pi64, w64, pi64, static_cast<int64_t>(len), stream_);
    GWB_CUDA(cudaMemcpyAsync(out_final, pi64, len * sizeof(double), cudaMemcpyDeviceToHost, stream_));
  }
  GWB_CUDA(cudaStreamSynchronize(stream_));
  cudaFreeAsync(pi64, stream_);
  cudaFreeAsync(w64, stream_);
  cudaFreeAsync(work, stream_);
}

void BapgEngine::iterates_to_colmajor64(int par, double* pi64, double* w64, double* work) {
  // K8 fix-up: exact fp64 row (π) / column (w) re-projection at the
  // boundary (a no-op up to rounding for the fp64 entropy iterates).
  if (quadratic()) {
    launch_rowmajor32_to_colmajor64(P_, n_, m_, ldm_, pi64, 0, mu64_, work, stream_);
    launch_rowmajor32_to_colmajor64(W_[par], n_, m_, ldm_, w64, 1, nu64_, work, stream_);
  } else {
    launch_rowmajor64_to_colmajor64(P64_, n_, m_, ldm_, pi64, 0, mu64_, work, stream_);
    launch_rowmajor64_to_colmajor64(W64_[par], n_, m_, ldm_, w64, 1, nu64_, work, stream_);
  }
}

float* BapgEngine::pi_dev() {
  if (!quadratic()) {
    launch_iterate_copies(P64_, n_, m_, ldm_, P_, nullptr, aux_mode(), aux_scale(), stream_);
    GWB_CUDA(cudaStreamSynchronize(stream_));
  }
  return P_;
}

void BapgEngine::kernel_ms(int kind, double* avg_ms, int64_t* count) {
  GWB_CUDA(cudaStreamSynchronize(stream_));
  if (ev_marks_.empty()) {  // already harvested: report the cached class
    *avg_ms = kind >= 0 && kind < 2 ? last_ms_[kind] : 0.0;
    *count = kind >= 0 && kind < 2 ? last_cnt_[kind] : 0;
    return;
  }
  double tot[2] = {0.0, 0.0};
  int64_t cnts[2] = {0, 0};
  for (auto& mk : ev_marks_) {
    float ms = 0.f;
    GWB_CUDA(cudaEventElapsedTime(&ms, mk.second.first, mk.second.second));
    tot[mk.first] += ms;
    ++cnts[mk.first];
  }
  for (int k = 0; k < 2; ++k) {
    last_ms_[k] = cnts[k] ? tot[k] / static_cast<double>(cnts[k]) : 0.0;
    last_cnt_[k] = cnts[k];
  }
  const double total = kind >= 0 && kind < 2 ? tot[kind] : 0.0;
  const int64_t cnt = kind >= 0 && kind < 2 ? cnts[kind] : 0;
  // Return all events to the pool (events are shared between marks).
  std::vector<cudaEvent_t> evs;
  for (auto& mk : ev_marks_) {
    evs.push_back(mk.second.first);
    evs.push_back(mk.second.second);
  }
  std::sort(evs.begin(), evs.end());
  evs.erase(std::unique(evs.begin(), evs.end()), evs.end());
  for (auto e : evs) ev_pool_.push_back(e);
  ev_marks_.clear();
  // One mark per half-step of each kind; GEMM marks cover two launches.
  *avg_ms = cnt ? total / static_cast<double>(cnt) : 0.0;
  *count = cnt;
}

void BapgEngine::readout(const int32_t* gt_host, int64_t n_gt, int32_t* assign_host,
                         Readout* r) {
  GWB_CUDA(cudaSetDevice(device_));
  const DevStatus s = status();
  const int par = s.iter >= 1 ? (s.iter - 1) & 1 : parity_;  // buffer holding the current w
  const size_t len = static_cast<size_t>(n_) * m_;
  double* pi64 = dalloc<double>(stream_, len);
  double* w64 = dalloc<double>(stream_, len);
  double* fin64 = dalloc<double>(stream_, len);
  double* work = dalloc<double>(stream_, static_cast<size_t>(std::max(n_, m_)));
  double* rs = dalloc<double>(stream_, n_);
  double* cs = dalloc<double>(stream_, m_);
  float* fin32 = dalloc<float>(stream_, static_cast<size_t>(n_) * ldm_);
  int32_t* assign = dalloc<int32_t>(stream_, n_);
  // K8 fix-up, then the final coupling ½(π + w) (solvers.cpp:214-216).
  iterates_to_colmajor64(par, pi64, w64, work);
  launch_average64(pi64, w64, fin64, static_cast<int64_t>(len), stream_);
  r->split_gap = std::sqrt(sum_sq_diff_dev(pi64, w64, static_cast<int64_t>(len), stream_));
  // marginal_infeasibility (diagnostics.cpp:9-19): ‖πᵀ1 − ν‖/m + ‖π1 − μ‖/n.
  launch_rowsums_cm64(fin64, n_, m_, rs, stream_);
  launch_colsums_cm64(fin64, n_, m_, cs, stream_);
  r->marginal_infeasibility = std::sqrt(sum_sq_diff_dev(cs, nu64_, m_, stream_)) / m_ +
                              std::sqrt(sum_sq_diff_dev(rs, mu64_, n_, stream_)) / n_;
  r->entropy = coupling_entropy_dev(fin64, static_cast<int64_t>(len), stream_);
  // luo_tseng_residual of the final coupling; run_cell records NaN when the
  // Dykstra projection throws (experiment.cpp:177-182).
  try {
    r->residual = luo_tseng_residual_dev(Dx_, ldn_, Dy_, ldm_, fin64, n_, m_, mu64_, nu64_, 1e-8,
                                         stream_);
  } catch (const CudaError&) {
    throw;
  } catch (...) {
    r->residual = std::nan("");
  }
  // gw_objective of the final coupling (3xTF32 chain on its fp32 copy).
  launch_colmajor64_to_rowmajor32(fin64, n_, m_, fin32, ldm_, stream_);
  r->objective = gw_objective_dev(Dx_, ldn_, Dy_, ldm_, fin32, n_, m_, stream_);
  // hard_assignment (tasks.cpp:190-200) and alignment_accuracy (:202-214).
  launch_argmax_rows_cm64(fin64, n_, m_, assign, stream_);
  if (assign_host)
    GWB_CUDA(cudaMemcpyAsync(assign_host, assign, sizeof(int32_t) * n_, cudaMemcpyDeviceToHost, stream_));
  if (gt_host) {
    int32_t* gt = dalloc<int32_t>(stream_, static_cast<size_t>(n_gt));
    GWB_CUDA(cudaMemcpyAsync(gt, gt_host, sizeof(int32_t) * n_gt, cudaMemcpyHostToDevice, stream_));
    const int64_t hits = count_equal_dev(assign, gt, n_gt, stream_);
    r->accuracy = 100.0 * static_cast<double>(hits) / static_cast<double>(n_gt);
    dfree(gt, stream_);
  }
  GWB_CUDA(cudaStreamSynchronize(stream_));
  for (void* p : std::initializer_list<void*>{pi64, w64, fin64, work, rs, cs, fin32, assign}) dfree(p, stream_);
}

double BapgEngine::gemm_flops_per_iter() const {
  if (sparse())  // two half-steps × two row-gathers, 2 flops per stored entry touched
    return 2.0 * 2.0 * (static_cast<double>(cx_.nnz) * m_ + static_cast<double>(cy_.nnz) * n_);
  // Two half-steps × (m·n·m + n·m·n) MACs × 2.
  return 2.0 * 2.0 * static_cast<double>(n_) * m_ * static_cast<double>(n_ + m_);
}

}  // namespace gwb
