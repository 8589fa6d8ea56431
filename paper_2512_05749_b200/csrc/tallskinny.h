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
// The k x k operands G, C and M are dense with leading dimension ldg / ldc / ldm (0 = k), so a
// 128-column block of a wider matrix can be addressed in place (k = 256 runs as 2 x 2 blocks of
// the k = 128 kernels, engine.cu).
// G (k x k) = A^T A, A rows x k (lda)
cudaError_t ts_gram(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                    double* G, int64_t ldg = 0);
// C (k x k) = A^T B
cudaError_t ts_cross(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc = 0);
// Y = A (alpha M), M k x k (upper: M upper triangular, the zero tiles are skipped)
cudaError_t ts_mul(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                   const double* M, bool upper, double alpha, double* Y, int64_t ldy,
                   int64_t ldm = 0);
// Y = Cin + A (alpha M)
cudaError_t ts_mul_add(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                       const double* M, double alpha, const double* Cin, int64_t ldcin, double* Y,
                       int64_t ldy, int64_t ldm = 0);
// *out (device) = ||Cin + A (alpha M)||_F^2, nothing else written
cudaError_t ts_mul_add_sumsq(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                             const double* M, double alpha, const double* Cin, int64_t ldcin,
                             double* out);

}  // namespace wssr
