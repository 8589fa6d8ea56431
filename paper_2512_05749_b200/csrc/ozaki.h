// FP64 O-pass GEMMs on the int8 tensor cores (exact digit products; see ozaki.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace wssr {

// Length (in {mu, scale} pairs) of the per-parameter scale table for `cols` parameters.
int64_t ozaki_scale_len(int64_t cols);

// Per-parameter table mu_inv[p] = {mu_p, 2^(54 - e_p)}, e_p the exponent bound of
// max_n |O_np - mu_p| over the (rows x cols, ld lda) sample block; pads to ozaki_scale_len.
cudaError_t ozaki_scales(Context& ctx, const void* A, bool f32, int64_t lda, int64_t rows,
                         int64_t cols, const double* mu, double* mu_inv, cudaStream_t st);

// Same GemmArgs contract as gemm() for the two sample-block layouts (shift = mu is taken from
// mu_inv); false when the operands do not suit the TMA/tensor-core path.
bool ozaki_supported(Layout L, const GemmArgs& a, bool f32);
cudaError_t ozaki_gemm(Context& ctx, Layout L, const GemmArgs& a, bool f32, const double* mu_inv,
                       cudaStream_t st);

}  // namespace wssr
