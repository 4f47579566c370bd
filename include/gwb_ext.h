/*
 * gwb_ext.h — B200-side extensions of the C-ABI that have no reference
 * counterpart: kernel-level test hooks and the synthetic-instance
 * generators used by tests and bench.py.
 */
#ifndef GWB_EXT_H_
#define GWB_EXT_H_

#include "gwb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* C[M×N] = A[M×K]·B[N×K]ᵀ on device fp32 row-major buffers through the
 * tcgen05 GEMM (precision: GWB_PREC_TF32 = 1 pass on the given operands,
 * GWB_PREC_3XTF32 = hi/lo split passes computed internally).  `stream` is a
 * cudaStream_t (NULL = legacy default).  Test hook for the K1 kernel. */
/* Debug (GWB_GEMM_TIMING=1): per-CTA %globaltimer stamps of the last chain
 * GEMM launch, [ctas][8] ns: entry, prologue done, PDL wait done, first
 * stage ready, last MMA issued (leader CTA), last chunk drained, stores
 * done, exit.  *count = CTAs written (0 when timing is off). */
GWB_API int32_t gwb_debug_gemm_stamps(uint64_t* out, int32_t max_ctas, int32_t* count);
GWB_API int32_t gwb_debug_gemm(const float* a, int64_t lda, const float* b,
                               int64_t ldb, float* c, int64_t ldc, int64_t M,
                               int64_t N, int64_t K, int32_t precision,
                               void* stream, gwb_status* st);

/* Device time (CUDA events on its stream) of the last on-chip batched BAPG
 * kernel launched by gwb_bapg_solve_batched in this process, summed over its
 * batch chunks, and the number of problems it covered; 0 / 0 if the last
 * batched call took the generic engine.  Measurement hook for bench.py. */
GWB_API int32_t gwb_batched_last_kernel_ms(double* ms, int64_t* problems);

/* Sweeps used and device time (CUDA events around the sweep loop on its
 * stream) of the last Dykstra projection run in this process (the
 * gwb_dykstra_project leaf, a Luo-Tseng residual or a readout).
 * Measurement hook for tools/bench_residual.py. */
GWB_API int32_t gwb_dykstra_last_stats(int32_t* sweeps, double* ms);

/* ---------------------------------------------------------------------------
 * Row-sharded multi-GPU BAPG, one shard per rank (csrc/shard.cu).  The
 * caller owns the communication buffers (e.g. torch tensors used with
 * torch.distributed/NCCL) and issues the collectives between phases on the
 * shard's stream:
 *   per iteration: phase 0, all-gather(vt), phase 1, phase 2,
 *                  all-gather(vt), phase 3, all-gather(col_stats), phase 4,
 *                  all-reduce-sum(diag[8]), all-reduce-max(err[8]), phase 5
 *   after the loop: phase 6, all-gather(vt), phase 7, all-reduce-sum(diag),
 *                   all-reduce-max(err), phase 8, then gwb_shard_finish.
 * vt is world × planes × m × rows_per_shard elements, rank r's chunk being
 * its block of Vᵀ (the all-gather is in place, one collective for all
 * planes); col_stats is world × 3 × m fp64; diag and err are 8 fp64 each.
 * ------------------------------------------------------------------------- */
typedef struct gwb_shard gwb_shard;

GWB_API int32_t gwb_shard_create(const gwb_config* cfg, int64_t n, int64_t m,
                                 int32_t rank, int32_t world, int32_t device,
                                 void* stream, gwb_shard** out,
                                 gwb_status* st);
GWB_API int32_t gwb_shard_layout(gwb_shard* s, int64_t* rows_per_shard,
                                 int64_t* row_begin, int64_t* rows_valid,
                                 int32_t* planes, int32_t* elem_bytes,
                                 int64_t* vt_bytes, int64_t* stats_bytes,
                                 gwb_status* st);
GWB_API int32_t gwb_shard_set_comm(gwb_shard* s, void* vt_gather,
                                   void* col_stats, double* diag, double* err,
                                   gwb_status* st);
/* dx_rows: rows_valid × n fp32 rows of D_X owned by this rank (device). */
GWB_API int32_t gwb_shard_load_device(gwb_shard* s, const float* dx_rows,
                                      int64_t ldx, const float* dy,
                                      int64_t ldy, const float* mu_rows,
                                      const float* nu, gwb_status* st);
/* f16x2 chains (GWB_PREC_F16X2) only, before load: the bound on every
 * iterate entry, max(max μ, max ν) over ALL ranks (the row projection
 * keeps π_kl ≤ μ_k, the column projection w_kl ≤ ν_l).  Every rank must
 * pass the same value: it sets the power-of-two plane scales of the
 * gathered Vᵀ blocks. */
GWB_API int32_t gwb_shard_set_iterate_bound(gwb_shard* s, double x_max, gwb_status* st);
GWB_API int32_t gwb_shard_reset(gwb_shard* s, gwb_status* st);
GWB_API int32_t gwb_shard_phase(gwb_shard* s, int32_t phase, gwb_status* st);
/* Compute/collective overlap: instead of all-gather(vt) + phase 1 (3, 7),
 * issue one collective per source rank (e.g. a broadcast of that rank's vt
 * chunk) and, as each lands, gwb_shard_gemm2_chunk(src) — the partial
 * G_r (+)= D_X[rows_r, cols_src]·V_src, own rank first (it overwrites G_r),
 * tail = 1 for the tail pass — then phase 21 (23, 27): phase 1 (3, 7)
 * without its GEMM2. */
GWB_API int32_t gwb_shard_gemm2_chunk(gwb_shard* s, int32_t src, int32_t tail,
                                      gwb_status* st);
/* Kernels launched so far by phases 0-5 of this shard (measurement hook). */
GWB_API int32_t gwb_shard_launches(gwb_shard* s, int64_t* launches);
/* Exact fp64 marginals for this shard (host: its rows_valid entries of μ,
 * all m of ν), after gwb_shard_load_device and before reset: the iterates
 * are fp64 and the projections scale to these (projections.cpp:12-34). */
GWB_API int32_t gwb_shard_set_marginals64(gwb_shard* s, const double* mu_rows, const double* nu,
                                          gwb_status* st);
GWB_API int32_t gwb_shard_stream(gwb_shard* s, void** stream, gwb_status* st);
GWB_API int32_t gwb_shard_status(gwb_shard* s, int32_t* done, int32_t* iter,
                                 int32_t* flags, int32_t* converged,
                                 int32_t* err_iter, int32_t* zero_index,
                                 gwb_status* st);
GWB_API int32_t gwb_shard_finish(gwb_shard* s, gwb_status* st);
GWB_API int32_t gwb_shard_records(gwb_shard* s, int32_t count,
                                  gwb_record* out, gwb_status* st);
/* Local rows of π and w, row-major fp64 rows_valid × m (nullable). */
GWB_API int32_t gwb_shard_rows(gwb_shard* s, double* pi_rows, double* w_rows,
                               gwb_status* st);
GWB_API int32_t gwb_shard_destroy(gwb_shard* s);

/* ---------------------------------------------------------------------------
 * Row-sharded eBPG / BPG / hBPG (csrc/bregman.cu, orchestrated by dist.py).
 * Rank r owns rows [r·n_r, r·n_r + n_r) of D_X (n_r = ⌈n/world⌉ rounded up
 * to 64, padded_rows = world·n_r) and computes those rows of the chain;
 * π, the Sinkhorn potentials and the records are replicated.  The caller
 * owns two buffers and issues the collectives on the shard's stream:
 *   vt: vt_bytes, [world][planes][m][n_r] (rank r's slot = its Vᵀ block),
 *   g:  padded_rows × ld fp32 (G; rank r's rows are one contiguous block).
 * Per outer iteration k = 1, 2, …:  phase(k, 0) · all-gather(vt) ·
 * phase(k, 1) · all-gather(g) · phase(k, 2) [form, Sinkhorn sweeps, write,
 * record; identical on every rank] · status.  After the loop, unless flags
 * are set: phase(used, 3) · all-gather(vt) · phase(used, 4) · all-gather(g)
 * · phase(used, 5) (the last record's objective), then finish.
 * cfg->precision must be resolved (GWB_PREC_BF16X3 / BF16X2 / 3XTF32);
 * the observer and record_residual are single-GPU only.
 * ------------------------------------------------------------------------- */
typedef struct gwb_bshard gwb_bshard;

GWB_API int32_t gwb_bshard_create(const gwb_config* cfg, int64_t n, int64_t m, int32_t rank,
                                  int32_t world, int32_t device, void* stream,
                                  gwb_bshard** out, gwb_status* st);
GWB_API int32_t gwb_bshard_layout(gwb_bshard* s, int64_t* rows_per_shard, int64_t* row_begin,
                                  int64_t* rows_valid, int64_t* padded_rows, int64_t* ld,
                                  int32_t* planes, int32_t* elem_bytes, int64_t* vt_bytes,
                                  gwb_status* st);
GWB_API int32_t gwb_bshard_set_comm(gwb_bshard* s, void* vt, float* g, gwb_status* st);
/* dx_rows: rows_valid × n fp32 on the device (leading dim ldx), dy: m × m
 * fp32 device (ldy); mu (n) and nu (m) host fp64. */
GWB_API int32_t gwb_bshard_load_device(gwb_bshard* s, const float* dx_rows, int64_t ldx,
                                       const float* dy, int64_t ldy, const double* mu,
                                       const double* nu, gwb_status* st);
GWB_API int32_t gwb_bshard_phase(gwb_bshard* s, int32_t k, int32_t op, gwb_status* st);
GWB_API int32_t gwb_bshard_status(gwb_bshard* s, int32_t* done, int32_t* iter, int32_t* flags,
                                  int32_t* converged, gwb_status* st);
GWB_API int32_t gwb_bshard_stream(gwb_bshard* s, void** stream, gwb_status* st);
/* The reference error (if flags are set), the trace, convergence and the
 * final coupling (host fp64 column-major n × m, nullable). */
GWB_API int32_t gwb_bshard_finish(gwb_bshard* s, double* out_final, gwb_record* trace,
                                  int32_t trace_cap, int32_t* n_records, int32_t* converged,
                                  int32_t* iterations_used, gwb_status* st);
GWB_API int32_t gwb_bshard_destroy(gwb_bshard* s);

#ifdef __cplusplus
}
#endif

#endif /* GWB_EXT_H_ */
