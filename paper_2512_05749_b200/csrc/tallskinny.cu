// Tall-skinny FP64 kernels for the P x k blocks of the SSI loop (k = 32, 64 or 128, rows = P up to
// 10^6): the Grams and triangular products of CholeskyQR2 (qr_orthonormalize, linalg.py:29-61),
// the Rayleigh quotient q^T w and the residual ||w - q (q^T w)||_F (svdengine.py:137-139), and the
// drift block u2 - u1 (u1^T u2) (svdengine.py:217-221).
//
// These operands are 67 MB at c1 (10 us of HBM) and the products are 2 P k^2 FLOP (29 us of
// DMMA at the measured 37 TF/s), so the generic TMA tile GEMM - built for the N x P sample block -
// wastes most of its time on split-K slabs, a 64 x 64 output tile per CTA and full (not
// triangular / symmetric) products.  Here every warp streams its own rows straight into DMMA
// fragments (no shared-memory staging of the tall operand: each fragment load is a full 32-byte
// sector per row), and:
//   * Grams compute only the upper 8 x 8 tiles (36 of 64 at k = 64): the A and B fragments of
//     A^T A are the same register, so one load per column block feeds every tile of a k-step;
//   * products with the triangular CholeskyQR2 factors R^-1 skip the zero tiles (72 of 128 DMMAs
//     per 8 rows);
//   * the residual ||W - A M||_F^2 is reduced in registers and never written;
//   * per-CTA partials are summed in a fixed order (bitwise repeatable, like every reduction in
//     this library);
//   * occupancy over work per thread: the k x k products run 8-row blocks per warp at two CTAs
//     per SM, the cross-Grams 16 warps per CTA (measured faster than fewer, fatter warps; the
//     symmetric Gram is the exception - one load feeding 36 DMMAs wins there).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "common.cuh"
#include "engine.h"
#include "tallskinny.h"

namespace wssr {
namespace ts {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kRowStep = 16;  // rows per warp iteration (4 DMMA k-steps of the Grams)

__device__ __forceinline__ double2 ld2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}

// ---- Gram / cross-Gram: slabs[cta] (KC x KC, upper tiles only when SYM) ------------------------
// SYM: C = A^T A, every warp owns all NB(NB+1)/2 upper tiles and a contiguous row range.
// !SYM: C = A^T B, warps pair up: warp w owns the column blocks [h NB/2, (h+1) NB/2), h = w & 1,
// of the row range of pair w >> 1.
// Fragments (mma.m8n8k4.f64, lane = 4 g + t): a = A^T[8bi + g][r0 + t] = A[r0 + t][8bi + g],
// b = B[r0 + t][8bj + g]; c[e] = C[8bi + g][8bj + 2t + e].
template <int KC, bool SYM>
__global__ void __launch_bounds__(kThreads, 1)
    gram_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                int64_t ldb, int64_t rows, int64_t rows_per_cta, double* __restrict__ slabs) {
  pdl_wait();
  constexpr int NB = KC / 8;
  constexpr int NJ = SYM ? NB : NB / 2;  // column blocks per warp
  constexpr int U = kRowStep / 4;
  constexpr int GROUPS = SYM ? kWarps : kWarps / 2;  // row groups per CTA
  __shared__ __align__(16) double red[NB * NB * 64];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  const int grp = SYM ? warp : warp >> 1;
  const int jb0 = SYM ? 0 : (warp & 1) * NJ;

  const int64_t cta_r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t cta_r1 = min(rows, cta_r0 + rows_per_cta);
  const int64_t per_grp = (rows_per_cta / GROUPS + kRowStep - 1) / kRowStep * kRowStep;
  const int64_t r_begin = cta_r0 + grp * per_grp;
  const int64_t r_end = min(cta_r1, r_begin + per_grp);

  double acc[NB][NJ][2];
#pragma unroll
  for (int i = 0; i < NB; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // two-stage register pipeline: the fragments of the next 8 rows are in flight while the DMMAs
  // of the current 8 run (a load stall would otherwise open every iteration)
  constexpr int H = U / 2;  // k-steps per stage
  auto load = [&](int64_t r0, double (&fa)[H][NB], double (&fb)[H][NJ]) {
#pragma unroll
    for (int u = 0; u < H; ++u) {
      const int64_t r = r0 + 4 * u + t;
      const bool ok = r < r_end;
      const double* pa = A + (ok ? r : 0) * lda + g;
      const double* pb = B + (ok ? r : 0) * ldb + g + 8 * jb0;
#pragma unroll
      for (int b = 0; b < NB; ++b) fa[u][b] = ok ? pa[8 * b] : 0.0;
      if (!SYM) {
#pragma unroll
        for (int b = 0; b < NJ; ++b) fb[u][b] = ok ? pb[8 * b] : 0.0;
      }
    }
  };
  auto compute = [&](const double (&fa)[H][NB], const double (&fb)[H][NJ]) {
#pragma unroll
    for (int u = 0; u < H; ++u)
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          if (SYM && j < i) continue;
          dmma884(acc[i][j], fa[u][i], SYM ? fa[u][j] : fb[u][j]);
        }
  };
  double fa0[H][NB], fb0[H][NJ], fa1[H][NB], fb1[H][NJ];
  load(r_begin, fa0, fb0);
  for (int64_t r0 = r_begin; r0 < r_end; r0 += kRowStep) {
    load(r0 + 4 * H, fa1, fb1);
    compute(fa0, fb0);
    load(r0 + kRowStep, fa0, fb0);
    compute(fa1, fb1);
  }

  // CTA reduction over the row groups, in group order (deterministic)
  for (int gi = 0; gi < GROUPS; ++gi) {
    if (grp == gi) {
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          if (SYM && j < i) continue;
          double2* slot = reinterpret_cast<double2*>(red + ((i * NB + jb0 + j) * 64 + 2 * lane));
          if (gi == 0) {
            *slot = make_double2(acc[i][j][0], acc[i][j][1]);
          } else {
            double2 v = *slot;
            v.x += acc[i][j][0];
            v.y += acc[i][j][1];
            *slot = v;
          }
        }
    }
    __syncthreads();
  }
  // slab in matrix layout: C[8bi + g][8bj + 2t + e] (lower tiles left unwritten when SYM)
  double* slab = slabs + (size_t)blockIdx.x * KC * KC;
  for (int idx = threadIdx.x; idx < NB * NB * 32; idx += kThreads) {
    const int tile = idx >> 5, l = idx & 31;
    const int bi = tile / NB, bj = tile % NB;
    if (SYM && bj < bi) continue;
    const double2 v = *reinterpret_cast<const double2*>(red + tile * 64 + 2 * l);
    *reinterpret_cast<double2*>(slab + (8 * bi + (l >> 2)) * KC + 8 * bj + 2 * (l & 3)) = v;
  }
}

// ---- grouped Gram / cross-Gram.  Warp w = (group G = w % NG, row quarter w / NG), NG = NB/2
// groups.  SYM: group G "folds" row blocks G and NB-1-G, i.e. the tiles (G, j >= G) and
// (NB-1-G, j >= NB-1-G) - NB + 1 tiles, equal for every group; its fragments are the column
// blocks G..NB-1.  !SYM: group G owns the column blocks [2G, 2G+2) against all NB row blocks.
// The group index is a template parameter (warp-uniform switch), so every fragment and
// accumulator index stays static.  k = 32/64: 16 warps (~120 registers: 16 warps per SM hide the
// DMMA and load latencies); k = 128: 8 warps, one per group, each writing its tiles straight to
// the CTA's slab.
template <int KC>
struct GramCfg {
  static constexpr int NB = KC / 8;
  static constexpr int NG = NB / 2;
  static constexpr int WARPS = KC == 128 ? 8 : 16;
  static constexpr int RQ = WARPS / NG;  // row quarters
};

template <int KC, bool SYM, int G>
__device__ __forceinline__ void gram16_group(const double* __restrict__ A, int64_t lda,
                                             const double* __restrict__ B, int64_t ldb,
                                             int64_t r_begin, int64_t r_end, int rq, int lane,
                                             double* red, double* slab) {
  using Cfg = GramCfg<KC>;
  constexpr int NB = Cfg::NB;
  constexpr int RQ = Cfg::RQ;
  constexpr int CW = 2;  // !SYM: column blocks per group
  constexpr int I0 = G, I1 = NB - 1 - G;
  // tile (i, j) -> accumulator slot; -1: not this group's
  auto slot = [](int i, int j) constexpr -> int {
    if (SYM) {
      if (i == I0 && j >= I0) return j - I0;
      if (i == I1 && j >= I1) return (NB - I0) + (j - I1);
      return -1;
    }
    return (j >= G * CW && j < (G + 1) * CW) ? i * CW + (j - G * CW) : -1;
  };
  constexpr int NT = SYM ? (NB - I0) + (NB - I1) : NB * CW;
  constexpr int FB0 = SYM ? I0 : 0;  // first A fragment block needed
  const int g = lane >> 2, t = lane & 3;
  double acc[NT][2];
#pragma unroll
  for (int q = 0; q < NT; ++q) acc[q][0] = acc[q][1] = 0.0;
  constexpr int H = (SYM && KC <= 64) ? 2 : 1;  // k-steps (4 rows each) per pipeline stage
  auto load = [&](int64_t r0, double (&fa)[H][NB], double (&fb)[H][CW]) {
#pragma unroll
    for (int u = 0; u < H; ++u) {
      const int64_t r = r0 + 4 * u + t;
      const bool ok = r < r_end;
      const double* pa = A + (ok ? r : 0) * lda + g;
#pragma unroll
      for (int b = FB0; b < NB; ++b) fa[u][b] = ok ? pa[8 * b] : 0.0;
      if (!SYM) {
        const double* pb = B + (ok ? r : 0) * ldb + g + 8 * G * CW;
#pragma unroll
        for (int b = 0; b < CW; ++b) fb[u][b] = ok ? pb[8 * b] : 0.0;
      }
    }
  };
  auto compute = [&](const double (&fa)[H][NB], const double (&fb)[H][CW]) {
#pragma unroll
    for (int u = 0; u < H; ++u)
#pragma unroll
      for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const int q = slot(i, j);
          if (q < 0) continue;
          dmma884(acc[q], fa[u][i], SYM ? fa[u][j] : fb[u][j - G * CW]);
        }
  };
  double fa0[H][NB], fb0[H][CW], fa1[H][NB], fb1[H][CW];
  const int64_t step = 4 * H;
  // this warp's rows: 2*step-row slices interleaved over the RQ quarters
  load(r_begin + 2 * step * rq, fa0, fb0);
  for (int64_t r0 = r_begin + 2 * step * rq; r0 < r_end; r0 += 2 * step * RQ) {
    load(r0 + step, fa1, fb1);
    compute(fa0, fb0);
    load(r0 + 2 * step * RQ, fa0, fb0);
    compute(fa1, fb1);
  }
  if constexpr (RQ == 1) {
    // sole owner of its tiles: straight to the slab, C[8i + g][8j + 2t + e]
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int q = slot(i, j);
        if (q < 0) continue;
        *reinterpret_cast<double2*>(slab + (8 * i + g) * KC + 8 * j + 2 * t) =
            make_double2(acc[q][0], acc[q][1]);
      }
  } else {
    // deterministic CTA reduction: row quarters in order, groups in parallel (disjoint tiles)
    for (int qi = 0; qi < RQ; ++qi) {
      if (rq == qi) {
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            const int q = slot(i, j);
            if (q < 0) continue;
            double2* dst = reinterpret_cast<double2*>(red + ((i * NB + j) * 64 + 2 * lane));
            if (qi == 0) {
              *dst = make_double2(acc[q][0], acc[q][1]);
            } else {
              double2 v = *dst;
              v.x += acc[q][0];
              v.y += acc[q][1];
              *dst = v;
            }
          }
      }
      __syncthreads();
    }
  }
}

template <int KC, bool SYM>
__global__ void __launch_bounds__(32 * GramCfg<KC>::WARPS, 1)
    gram16_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                  int64_t ldb, int64_t rows, int64_t rows_per_cta, double* __restrict__ slabs) {
  pdl_wait();
  using Cfg = GramCfg<KC>;
  constexpr int NB = Cfg::NB;
  constexpr int NG = Cfg::NG;
  constexpr int NRED = Cfg::RQ > 1 ? NB * NB * 64 : 2;
  __shared__ __align__(16) double red[NRED];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = warp % NG, rq = warp / NG;
  const int64_t r_begin = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r_end = min(rows, r_begin + rows_per_cta);
  double* slab = slabs + (size_t)blockIdx.x * KC * KC;
#define WSSR_GRAM_CASE(c)                                                                     \
  case c:                                                                                      \
    if constexpr (NG > c)                                                                      \
      gram16_group<KC, SYM, (NG > c ? c : 0)>(A, lda, B, ldb, r_begin, r_end, rq, lane, red,   \
                                              slab);                                            \
    break;
  switch (grp) {  // warp-uniform
    WSSR_GRAM_CASE(0)
    WSSR_GRAM_CASE(1)
    WSSR_GRAM_CASE(2)
    WSSR_GRAM_CASE(3)
    WSSR_GRAM_CASE(4)
    WSSR_GRAM_CASE(5)
    WSSR_GRAM_CASE(6)
    WSSR_GRAM_CASE(7)
    default: break;
  }
#undef WSSR_GRAM_CASE
  if constexpr (Cfg::RQ > 1) {
    for (int idx = threadIdx.x; idx < NB * NB * 32; idx += 32 * Cfg::WARPS) {
      const int tile = idx >> 5, l = idx & 31;
      const int bi = tile / NB, bj = tile % NB;
      if (SYM && bj < bi) continue;
      const double2 v = *reinterpret_cast<const double2*>(red + tile * 64 + 2 * l);
      *reinterpret_cast<double2*>(slab + (8 * bi + (l >> 2)) * KC + 8 * bj + 2 * (l & 3)) = v;
    }
  }
}

// C[i][j] = sum over slabs in slab order; SYM mirrors the upper tiles.  Block: 32 consecutive
// entries x 8 slab groups.
template <int KC, bool SYM>
__global__ void __launch_bounds__(512)
    gram_finish_kernel(const double* __restrict__ slabs, int nslab, double* __restrict__ C,
                       int64_t ldc) {
  pdl_wait();
  __shared__ double part[16][33];
  const int jj = threadIdx.x & 31, sg = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + jj;  // entry (row-major KC x KC)
  const int i = e / KC, j = e % KC;
  const int src = (SYM && (j >> 3) < (i >> 3)) ? j * KC + i : e;
  double s0 = 0.0, s1 = 0.0;
  int c = sg;
  for (; c + 16 < nslab; c += 32) {
    s0 += slabs[(size_t)c * KC * KC + src];
    s1 += slabs[(size_t)(c + 16) * KC * KC + src];
  }
  if (c < nslab) s0 += slabs[(size_t)c * KC * KC + src];
  part[sg][jj] = s0 + s1;
  __syncthreads();
  if (sg == 0) {
    double tot = part[0][jj];
#pragma unroll
    for (int q = 1; q < 16; ++q) tot += part[q][jj];
    C[(int64_t)i * ldc + j] = tot;
  }
}

// ---- row-block products: Y = A M, Y = Cin + A M, or ||Cin + A M||_F^2 -------------------------
// M (KC x KC) is staged once per CTA in fragment order: Ms[jp][bn][lane] = {M[8jp + 2t][8bn + g],
// M[8jp + 2t + 1][8bn + g]}; the k-slots of DMMA step 2jp (2jp + 1) are the columns 8jp + 2t
// (8jp + 2t + 1), so each lane fetches its A pair with one 16-byte load.  TRI: M upper
// triangular, the tiles (jp > bn) are skipped.  Every warp takes 16-row blocks.
enum Mode : int { kStore = 0, kAddStore = 1, kAddSumsq = 2 };

// MBR 8-row blocks per warp iteration: 1 keeps the kernel near 110 registers, so two CTAs (16
// warps) share an SM and hide the DMMA / load latencies.
constexpr int MBR = 1;

template <int KC, bool TRI, int MODE>
__global__ void __launch_bounds__(kThreads, KC == 128 ? 1 : 2)
    mul_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ M,
               int64_t ldm, double alpha, const double* __restrict__ Cin, int64_t ldcin,
               double* __restrict__ Y, int64_t ldy, int64_t rows, double* __restrict__ partial) {
  pdl_wait();
  constexpr int NB = KC / 8;
  extern __shared__ __align__(16) double2 Ms[];  // NB * NB * 32 (KC^2 doubles)
  __shared__ double scratch[32];
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  for (int idx = threadIdx.x; idx < NB * NB * 32; idx += kThreads) {
    const int l = idx & 31, bn = (idx >> 5) % NB, jp = (idx >> 5) / NB;
    const int gg = l >> 2, tt = l & 3;
    const int r = 8 * jp + 2 * tt, c = 8 * bn + gg;
    Ms[idx] = make_double2(alpha * M[r * ldm + c], alpha * M[(r + 1) * ldm + c]);
  }
  __syncthreads();

  double ss = 0.0;
  const int64_t nblk = (rows + 8 * MBR - 1) / (8 * MBR);
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp, nw = (int64_t)gridDim.x * kWarps;
  // the next block's A fragments are loaded while this block's DMMAs run
  auto load = [&](int64_t blk, double2 (&a)[MBR][NB]) {
#pragma unroll
    for (int mb = 0; mb < MBR; ++mb) {
      const int64_t r = blk * 8 * MBR + 8 * mb + g;
      const bool ok = blk < nblk && r < rows;
      const double* pa = A + (ok ? r : 0) * lda + 2 * t;
#pragma unroll
      for (int jp = 0; jp < NB; ++jp) a[mb][jp] = ok ? ld2(pa + 8 * jp) : make_double2(0.0, 0.0);
    }
  };
  double2 a[MBR][NB], an[MBR][NB];
  load(gw, an);
  for (int64_t blk = gw; blk < nblk; blk += nw) {
    const int64_t r0 = blk * 8 * MBR;
#pragma unroll
    for (int mb = 0; mb < MBR; ++mb)
#pragma unroll
      for (int jp = 0; jp < NB; ++jp) a[mb][jp] = an[mb][jp];
    load(blk + nw, an);
    double acc[MBR][NB][2];
#pragma unroll
    for (int mb = 0; mb < MBR; ++mb)
#pragma unroll
      for (int bn = 0; bn < NB; ++bn) acc[mb][bn][0] = acc[mb][bn][1] = 0.0;
#pragma unroll
    for (int bn = 0; bn < NB; ++bn)
#pragma unroll
      for (int jp = 0; jp < NB; ++jp) {
        if (TRI && jp > bn) continue;
        const double2 m = Ms[(jp * NB + bn) * 32 + lane];
#pragma unroll
        for (int mb = 0; mb < MBR; ++mb) {
          dmma884(acc[mb][bn], a[mb][jp].x, m.x);
          dmma884(acc[mb][bn], a[mb][jp].y, m.y);
        }
      }
#pragma unroll
    for (int mb = 0; mb < MBR; ++mb) {
      const int64_t r = r0 + 8 * mb + g;
      if (r >= rows) continue;
#pragma unroll
      for (int bn = 0; bn < NB; ++bn) {
        double2 y = make_double2(acc[mb][bn][0], acc[mb][bn][1]);
        if (MODE != kStore) {
          const double2 c = ld2(Cin + r * ldcin + 8 * bn + 2 * t);
          y.x = c.x + y.x;
          y.y = c.y + y.y;
        }
        if (MODE == kAddSumsq) {
          ss = fma(y.x, y.x, ss);
          ss = fma(y.y, y.y, ss);
        } else {
          *reinterpret_cast<double2*>(Y + r * ldy + 8 * bn + 2 * t) = y;
        }
      }
    }
  }
  if (MODE == kAddSumsq) {
    ss = block_sum(ss, scratch);
    if (threadIdx.x == 0) partial[blockIdx.x] = ss;
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ partials, int n,
                                    double* __restrict__ out) {
  pdl_wait();
  __shared__ double scratch[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) *out = s;
}

// ---- transposed GEMV: out[j] = alpha sum_i A[i][j] x[i] (the k-vectors U^T gbar and V^T lhat,
// optimizers.py:361, 380).  Block: columns [blockIdx.y * CW, + CW) x (256 / CW) row lanes over a
// contiguous row range; partials[blockIdx.x][j] summed in block order by the finish kernel.
__global__ void __launch_bounds__(256)
    gemv_t_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ x,
                  int64_t rows, int n, int cw, int64_t rows_per_block,
                  double* __restrict__ partial) {
  pdl_wait();
  __shared__ double red[256];
  const int c = threadIdx.x % cw, rl = threadIdx.x / cw, lanes = 256 / cw;
  const int j = blockIdx.y * cw + c;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (j < n) {
    int64_t r = r0 + rl;
    for (; r + 7 * lanes < r1; r += 8 * lanes) {  // 8 independent loads in flight per thread
#pragma unroll
      for (int q = 0; q < 8; ++q) s[q] = fma(A[(r + q * lanes) * lda + j], x[r + q * lanes], s[q]);
    }
    for (; r < r1; r += lanes) s[0] = fma(A[r * lda + j], x[r], s[0]);
  }
  red[threadIdx.x] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  __syncthreads();
  if (rl == 0 && j < n) {
    double t = red[c];
    for (int q = 1; q < lanes; ++q) t += red[q * cw + c];
    partial[(size_t)blockIdx.x * n + j] = t;
  }
}

// out[j] = alpha sum_b partial[b][j]: one block per output, fixed-order block reduction
__global__ void __launch_bounds__(128)
    gemv_t_finish_kernel(const double* __restrict__ partial, int nblk, int n, double alpha,
                         double* __restrict__ out) {
  pdl_wait();
  __shared__ double scratch[32];
  const int j = blockIdx.x;
  double t = 0.0;
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) t += partial[(size_t)b * n + j];
  t = block_sum(t, scratch);
  if (threadIdx.x == 0) out[j] = alpha * t;
}

template <int KC, bool SYM>
cudaError_t gram_launch(Context& ctx, int64_t rows, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double* C, int64_t ldc) {
  const int64_t min_rows = 64;  // keep every CTA's share at least a few row steps
  int grid = (int)std::min<int64_t>(ctx.num_sms, std::max<int64_t>(1, rows / min_rows));
  int64_t rpc = (rows + grid - 1) / grid;
  rpc = (rpc + kRowStep - 1) / kRowStep * kRowStep;
  grid = (int)((rows + rpc - 1) / rpc);
  if (grid < 1) grid = 1;
  double* slabs = ctx.splitk_buffer((size_t)grid * KC * KC);
  if (!slabs) return cudaErrorMemoryAllocation;
  // symmetric Grams: the 8-warp kernel (one load per column block feeds 36 DMMAs; measured
  // 29 us at c1 against 35.5 for the 16-warp fold split); cross-Grams: the 16-warp kernel (44 us
  // against 51)
  if constexpr (SYM && KC <= 64)
    launch_pdl(gram_kernel<KC, SYM>, grid, kThreads, 0, ctx.stream, A, lda, B, ldb, rows, rpc,
               slabs);
  else
    launch_pdl(gram16_kernel<KC, SYM>, grid, 32 * GramCfg<KC>::WARPS, 0, ctx.stream, A, lda, B,
               ldb, rows, rpc, slabs);
  launch_pdl(gram_finish_kernel<KC, SYM>, KC * KC / 32, 512, 0, ctx.stream, slabs, grid, C, ldc);
  ctx.kernel_launches += 2;
  return cudaGetLastError();
}

template <int KC, bool TRI, int MODE>
cudaError_t mul_launch(Context& ctx, int64_t rows, const double* A, int64_t lda, const double* M,
                       int64_t ldm, double alpha, const double* Cin, int64_t ldcin, double* Y,
                       int64_t ldy, double* out) {
  const int64_t nblk = (rows + 8 * MBR - 1) / (8 * MBR);
  int grid = (int)std::min<int64_t>(2 * ctx.num_sms, std::max<int64_t>(1, (nblk + 7) / 8));
  double* partial = nullptr;
  if (MODE == kAddSumsq) {
    partial = ctx.splitk_buffer((size_t)grid);
    if (!partial) return cudaErrorMemoryAllocation;
  }
  constexpr int smem = KC * KC * 8;  // R^-1 / M in fragment order
  static std::atomic<uint64_t> attr{0};  // one per instantiation, one bit per device
  cudaError_t e = smem_attr_once(attr, mul_kernel<KC, TRI, MODE>, smem);
  if (e != cudaSuccess) return e;
  launch_pdl(mul_kernel<KC, TRI, MODE>, grid, kThreads, smem, ctx.stream, A, lda, M, ldm, alpha,
             Cin, ldcin, Y, ldy, rows, partial);
  ctx.kernel_launches += 1;
  if (MODE == kAddSumsq) {
    launch_pdl(sum_partials_kernel, 1, 256, 0, ctx.stream, partial, grid, out);
    ctx.kernel_launches += 1;
  }
  return cudaGetLastError();
}

bool aligned16(const void* p, int64_t ld) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && (ld & 1) == 0;
}

}  // namespace ts

bool ts_supported(int64_t k) { return k == 32 || k == 64 || k == 128; }

cudaError_t ts_gemv_t(Context& ctx, int64_t rows, int64_t n, const double* A, int64_t lda,
                      const double* x, double alpha, double* out) {
  if (n <= 0) return cudaSuccess;
  if (rows <= 0) return cudaMemsetAsync(out, 0, sizeof(double) * n, ctx.stream);
  const int cw = n >= 256 ? 256 : (n > 128 ? 256 : (n > 64 ? 128 : (n > 32 ? 64 : 32)));
  const int ycols = (int)((n + cw - 1) / cw);
  const int64_t lanes = 256 / cw;
  int nblk = (int)std::min<int64_t>(4 * ctx.num_sms, std::max<int64_t>(1, rows / (16 * lanes)));
  const int64_t rpb = (rows + nblk - 1) / nblk;
  nblk = (int)((rows + rpb - 1) / rpb);
  double* partial = ctx.splitk_buffer((size_t)nblk * n);
  if (!partial) return cudaErrorMemoryAllocation;
  launch_pdl(ts::gemv_t_kernel, dim3(nblk, ycols), 256, 0, ctx.stream, A, lda, x, rows, (int)n, cw, rpb,
                                                              partial);
  launch_pdl(ts::gemv_t_finish_kernel, (unsigned)n, 128, 0, ctx.stream, 
      partial, nblk, (int)n, alpha, out);
  ctx.kernel_launches += 2;
  return cudaGetLastError();
}

cudaError_t ts_gram(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                    double* G, int64_t ldg) {
  if (ldg <= 0) ldg = k;
  if (rows <= 0)
    return cudaMemset2DAsync(G, sizeof(double) * ldg, 0, sizeof(double) * k, k, ctx.stream);
  if (k == 128) return ts::gram_launch<128, true>(ctx, rows, A, lda, A, lda, G, ldg);
  if (k == 64) return ts::gram_launch<64, true>(ctx, rows, A, lda, A, lda, G, ldg);
  return ts::gram_launch<32, true>(ctx, rows, A, lda, A, lda, G, ldg);
}

cudaError_t ts_cross(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc) {
  if (ldc <= 0) ldc = k;
  if (rows <= 0)
    return cudaMemset2DAsync(C, sizeof(double) * ldc, 0, sizeof(double) * k, k, ctx.stream);
  if (k == 128) return ts::gram_launch<128, false>(ctx, rows, A, lda, B, ldb, C, ldc);
  if (k == 64) return ts::gram_launch<64, false>(ctx, rows, A, lda, B, ldb, C, ldc);
  return ts::gram_launch<32, false>(ctx, rows, A, lda, B, ldb, C, ldc);
}

bool ts_mul_supported(int64_t k, const double* A, int64_t lda, const double* Y, int64_t ldy) {
  return ts_supported(k) && ts::aligned16(A, lda) && ts::aligned16(Y, ldy);
}

namespace {
// k (32 / 64 / 128) and triangularity as template arguments
template <int MODE>
cudaError_t mul_dispatch(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                         const double* M, bool upper, double alpha, const double* Cin,
                         int64_t ldcin, double* Y, int64_t ldy, double* out, int64_t ldm = 0) {
  auto go = [&](auto kc, auto tri) {
    return ts::mul_launch<decltype(kc)::value, decltype(tri)::value, MODE>(
        ctx, rows, A, lda, M, ldm > 0 ? ldm : k, alpha, Cin, ldcin, Y, ldy, out);
  };
  using T = std::true_type;
  using F = std::false_type;
  using K32 = std::integral_constant<int, 32>;
  using K64 = std::integral_constant<int, 64>;
  using K128 = std::integral_constant<int, 128>;
  if (k == 128) return upper ? go(K128{}, T{}) : go(K128{}, F{});
  if (k == 64) return upper ? go(K64{}, T{}) : go(K64{}, F{});
  return upper ? go(K32{}, T{}) : go(K32{}, F{});
}
}  // namespace

cudaError_t ts_mul(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                   const double* M, bool upper, double alpha, double* Y, int64_t ldy,
                   int64_t ldm) {
  if (rows <= 0) return cudaSuccess;
  return mul_dispatch<ts::kStore>(ctx, rows, k, A, lda, M, upper, alpha, nullptr, 0, Y, ldy,
                                  nullptr, ldm);
}

cudaError_t ts_mul_add(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                       const double* M, double alpha, const double* Cin, int64_t ldcin, double* Y,
                       int64_t ldy, int64_t ldm) {
  if (rows <= 0) return cudaSuccess;
  return mul_dispatch<ts::kAddStore>(ctx, rows, k, A, lda, M, false, alpha, Cin, ldcin, Y, ldy,
                                     nullptr, ldm);
}

cudaError_t ts_mul_add_sumsq(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                             const double* M, double alpha, const double* Cin, int64_t ldcin,
                             double* out) {
  if (rows <= 0) return cudaMemsetAsync(out, 0, sizeof(double), ctx.stream);
  return mul_dispatch<ts::kAddSumsq>(ctx, rows, k, A, lda, M, false, alpha, Cin, ldcin, nullptr,
                                     0, out);
}

}  // namespace wssr
