// FP64 O-pass GEMMs on the int8 tensor cores (exact digit products; see ozaki.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.h"

namespace wssr {

// Slots of the per-parameter scale table for `cols` parameters (cols rounded up to 32).
int64_t ozaki_scale_len(int64_t cols);
// Doubles of that table (4 per slot).
int64_t ozaki_table_doubles(int64_t cols);

// Per-parameter table, slot {cw_p, 2^(54 - e_p), mu_p, 0} (stored in a block-transposed slot
// order, see tab_slot in ozaki.cu; cw_p the integer centring word, see biased_digits), e_p the
// exponent bound of max_n |O_np - mu_p| over the (rows x cols, ld lda) sample block; pads to
// ozaki_scale_len slots.
cudaError_t ozaki_scales(Context& ctx, const void* A, bool f32, int64_t lda, int64_t rows,
                         int64_t cols, const double* mu, double* mu_inv, cudaStream_t st);

// A table of padding slots only (a rank without samples).
cudaError_t ozaki_table_clear(Context& ctx, double* mu_inv, int64_t cols, cudaStream_t st);

// The same table from per-column extrema of the sample block (fused into assemble's pass).
cudaError_t ozaki_scales_minmax(Context& ctx, const double* cmin, const double* cmax,
                                const double* mu, int64_t cols, double* mu_inv, cudaStream_t st);

// Same GemmArgs contract as gemm() for the two sample-block layouts (shift = mu is taken from
// mu_inv); false when the operands do not suit the TMA/tensor-core path.
// profiling only: CTA 0's per-K-block timestamps of the last debug-9 launch
cudaError_t ozaki_trace(long long* host, size_t bytes);

bool ozaki_supported(Layout L, const GemmArgs& a, bool f32);
// planes: the step's pre-digitised sample block (ozaki_digitize) or nullptr (digitise on the
// fly); store: with planes == nullptr and the row-major (v) layout, also write the digit planes
// the on-the-fly pass produces (same layout as ozaki_digitize), so later passes can stream them.
// rowcnt (on-the-fly v pass only): per sample row, the precision guard's packed digit-integer
// counts (see ozaki_row_guard)
// nds: sample digits the pass uses - 7 (FP64-grade, 28 digit pairs) or 5 (float32 samples: the
// top 5 of the same digits, X to 2^-38 of its column's scale, 20 pairs; see ozaki.cu issue_pairs)
cudaError_t ozaki_gemm(Context& ctx, Layout L, const GemmArgs& a, bool f32, const double* mu_inv,
                       cudaStream_t st, const int8_t* planes = nullptr, int8_t* store = nullptr,
                       unsigned long long* rowcnt = nullptr, int nds = 7);

// Precision guard: the row counts from the sample block directly (one read; for a first O-pass
// that is not the digitising v pass), and the verdict: *flag |= 1 when fewer than 1/64 of a
// sample row's nonzero elements lie within 12 bits of their columns' digit scales.
cudaError_t ozaki_row_headroom(Context& ctx, const void* A, bool f32, int64_t lda, int64_t rows,
                               int64_t cols, const double* mu_inv, unsigned long long* rowcnt,
                               cudaStream_t st);
cudaError_t ozaki_row_guard(Context& ctx, const unsigned long long* rowcnt, int64_t rows, int* flag,
                            cudaStream_t st);

// Digit planes [nds][rows][ozaki_plane_pitch(cols)] int8 of the centred, scaled sample block
// (rows = samples, cols = parameters, row-major with pitch lda; the nds most significant of the 7
// digits); written once per step and streamed by both O-passes.
// digit pairs kept per product by the FP64-grade scheme of this build (28, or 34 with
// -DWSSR_OZ_LEVELS=8)
int ozaki_digit_pairs();
int64_t ozaki_plane_pitch(int64_t cols);
size_t ozaki_planes_bytes(int64_t rows, int64_t cols, int nds = 7);
cudaError_t ozaki_digitize(Context& ctx, const void* A, bool f32, int64_t lda, int64_t rows,
                           int64_t cols, const double* mu_inv, int8_t* planes, cudaStream_t st,
                           int nds = 7);

}  // namespace wssr
