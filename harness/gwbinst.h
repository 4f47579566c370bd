/* gwbinst.h — seeded synthetic-instance generators (bench / test harness).
 *
 * NOT part of the product library: built into harness/libgwbinst.so, which
 * bench.py and tests/ use to make BASELINE.json's workloads.
 * Generators that exist in the reference follow its algorithm and RNG
 * contract draw for draw (proj/include/gw/rng.hpp:13-53, proj/src/tasks.cpp);
 * the others are new and documented in DESIGN.md §10.
 *
 * Edge lists are int32 pairs (a < b) in canonical order; the edge functions
 * return the edge count (the buffer holds min(count, cap) edges) or -1 on
 * invalid arguments. */
#ifndef GWBINST_H
#define GWBINST_H

#include <stdint.h>

#ifdef __cplusplus
#define GWBINST_API extern "C" __attribute__((visibility("default")))
#else
#define GWBINST_API __attribute__((visibility("default")))
#endif

/* gen_barabasi_albert (tasks.cpp:22-65). */
GWBINST_API int64_t gwbinst_gen_barabasi_albert(int32_t n, int32_t m_attach, uint64_t seed,
                                                int32_t* out, int64_t cap);
/* G(n, p) = gen_gaussian_partition(n, 1, p, 0, seed) (tasks.cpp:67-112). */
GWBINST_API int64_t gwbinst_gen_erdos_renyi(int32_t n, double p, uint64_t seed, int32_t* out,
                                            int64_t cap);
/* Equal-block SBM (new: the reference draws Gaussian block sizes). */
GWBINST_API int64_t gwbinst_gen_sbm_equal(int32_t n, int32_t k, double p_in, double p_out,
                                          uint64_t seed, int32_t* out, int64_t cap,
                                          int32_t* labels);
/* Remove q_remove·|E| edges, add q_add·|E| absent pairs (new; rejection
 * sampling for additions). */
GWBINST_API int64_t gwbinst_edge_noise(int32_t n, const int32_t* edges, int64_t count,
                                       double q_remove, double q_add, uint64_t seed,
                                       int32_t* out, int64_t cap);
/* permute_graph (tasks.cpp:141-154); perm[old] = new. */
GWBINST_API int64_t gwbinst_permute_graph(int32_t n, const int32_t* edges, int64_t count,
                                          uint64_t seed, int32_t* out, int32_t* perm);
/* 3-D isotropic Gaussian mixture, means U[0,1]^3 (new). xyz: n×3 row-major. */
GWBINST_API void gwbinst_gen_gmm3d(int32_t n, int32_t k, double sigma, uint64_t seed,
                                   double* xyz);
/* Euclidean distances ÷ max, rounded to fp32.  out: n×n. */
GWBINST_API void gwbinst_distance_maxnorm_f32(int32_t n, const double* xyz, float* out);
/* jittered_product (experiment.cpp:41-58): μνᵀ with entry (i,j) scaled by
 * 1 + jitter·U(−1,1), drawn in column-major order, then divided by its sum.
 * out: n×m column-major fp64. */
GWBINST_API void gwbinst_jittered_product(const double* mu, int64_t n, const double* nu,
                                          int64_t m, double jitter, uint64_t seed,
                                          double* out);

#endif /* GWBINST_H */
