// Tall-skinny FP64 kernels for the P x k blocks (k = 32, 64 or 128); see tallskinny.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace wssr {

// k handled by the tall-skinny kernels
bool ts_supported(int64_t k);
// the 16-byte fragment loads / stores of the row-block products need aligned rows
bool ts_mul_supported(int64_t k, const double* A, int64_t lda, const double* Y, int64_t ldy);

// out[j] = alpha sum_i A[i][j] x[i], A rows x n (lda), any n (device GEMV for the k-vectors)
cudaError_t ts_gemv_t(Context& ctx, int64_t rows, int64_t n, const double* A, int64_t lda,
                      const double* x, double alpha, double* out);
// G (k x k, dense) = A^T A, A rows x k (lda)
cudaError_t ts_gram(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                    double* G);
// C (k x k, dense) = A^T B
cudaError_t ts_cross(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C);
// Y = A (alpha M), M k x k dense (upper: M upper triangular, the zero tiles are skipped)
cudaError_t ts_mul(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                   const double* M, bool upper, double alpha, double* Y, int64_t ldy);
// Y = Cin + A (alpha M)
cudaError_t ts_mul_add(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                       const double* M, double alpha, const double* Cin, int64_t ldcin, double* Y,
                       int64_t ldy);
// *out (device) = ||Cin + A (alpha M)||_F^2, nothing else written
cudaError_t ts_mul_add_sumsq(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                             const double* M, double alpha, const double* Cin, int64_t ldcin,
                             double* out);

}  // namespace wssr
