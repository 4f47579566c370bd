// sparse.cuh — the D_X·π·D_Y chain for sparse structure matrices (SURVEY
// §8(f) row 2): graph adjacencies have density ~1e-4–1e-2, so the chain
// becomes two CSR row-gathers (fp32 exact-order sums, HBM/L2-bound) instead
// of two dense tensor-core GEMMs.  Selected with precision GWB_PREC_SPARSE;
// same results as the reference within the fp32 iterate tolerance (the sums
// are exact-order fp32, more accurate than the split tensor-core chains).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace gwb {

struct Csr {
  int64_t rows = 0;
  int64_t nnz = 0;
  int32_t* row_ptr = nullptr;  // rows + 1
  int32_t* col = nullptr;      // nnz, ascending within a row
  float* val = nullptr;        // nnz
};

// CSR of a dense fp32 row-major matrix already on the device (rows × rows,
// leading dimension ld).  Synchronises `s` once (to size the arrays).
Csr csr_from_dense(const float* D, int64_t rows, int64_t ld, cudaStream_t s);
void csr_free(Csr& c);

// out = A · in, A in CSR (rows_out × k), in row-major (k × cols, ld_in):
// out[i, :] = Σ_p val[p] · in[col[p], :].  transpose_out writes outᵀ
// (cols × rows_out, leading dimension ld_out) instead.  Column-blocked so
// the gathered slab of `in` stays L2-resident.  No-op when *skip != 0.
void launch_rowgather(const Csr& A, const float* in, int64_t ld_in, int64_t cols, float* out,
                      int64_t ld_out, bool transpose_out, const int* skip, cudaStream_t s);

}  // namespace gwb
