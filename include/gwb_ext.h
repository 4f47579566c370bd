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
GWB_API int32_t gwb_debug_gemm(const float* a, int64_t lda, const float* b,
                               int64_t ldb, float* c, int64_t ldc, int64_t M,
                               int64_t N, int64_t K, int32_t precision,
                               void* stream, gwb_status* st);

/* Instance generators (paper_2205_08115_b200/csrc/instances.cpp).  Edge
 * lists are int32 pairs (a < b), canonical order; return the edge count
 * (the buffer holds min(count, cap) edges) or -1 on invalid arguments. */
GWB_API int64_t gwb_gen_barabasi_albert(int32_t n, int32_t m_attach,
                                        uint64_t seed, int32_t* out,
                                        int64_t cap);
GWB_API int64_t gwb_gen_erdos_renyi(int32_t n, double p, uint64_t seed,
                                    int32_t* out, int64_t cap);
GWB_API int64_t gwb_gen_sbm_equal(int32_t n, int32_t k, double p_in,
                                  double p_out, uint64_t seed, int32_t* out,
                                  int64_t cap, int32_t* labels);
GWB_API int64_t gwb_edge_noise(int32_t n, const int32_t* edges, int64_t count,
                               double q_remove, double q_add, uint64_t seed,
                               int32_t* out, int64_t cap);
GWB_API int64_t gwb_permute_graph(int32_t n, const int32_t* edges,
                                  int64_t count, uint64_t seed, int32_t* out,
                                  int32_t* perm);
GWB_API void gwb_gen_gmm3d(int32_t n, int32_t k, double sigma, uint64_t seed,
                           double* xyz);
GWB_API void gwb_distance_maxnorm_f32(int32_t n, const double* xyz,
                                      float* out);

#ifdef __cplusplus
}
#endif

#endif /* GWB_EXT_H_ */
