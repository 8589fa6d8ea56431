// FP64 O-pass GEMMs as exact integer digit products on the 5th-generation tensor cores.
//
// FP64 tensor math on sm_100a is DMMA (mma.sync m8n8k4, ~37 TF/s measured), which puts the two
// O-passes of every SSI iteration (svdengine.py:133-134) 3x above the HBM time of streaming O.
// This path computes the same FP64 products exactly in integer arithmetic on tcgen05.mma
// kind::i8 (the Ozaki splitting):
//
//   * every element of the centred sample block  x = O - mu  is scaled by a power of two per
//     parameter column p (2^(54-e_p), e_p = exponent bound of max_n |O_np - mu_p|) and rounded to
//     an integer |X| <= 2^54 + 1 (integer centring rint(O s) - rint(mu s), or rint((O - mu) s)
//     when O - mu is exact; see biased_digits), split into 7 signed base-256 digits
//     X = sum_i d_i 256^i, d_i in [-128, 127] (bytes of X + 0x0080808080808080, each XOR 0x80);
//   * the thin operand (q or v, P x k / N x k) is split the same way per output column;
//   * digit products are exact int8 x int8 -> int32 tensor-core MMAs; the 28 digit pairs (a, b)
//     with a + b <= 6 (most-significant-first) are kept - the dropped ones sum below 2^-51.4 of
//     the product of the column scales (6 pairs of level 7 at <= 2^14 2^40 each against 2^108),
//     the size of one FP64 rounding of a full-scale product, and unlike FP64 the kept sums are
//     exact over K - and pairs of equal significance a + b = s share one int32 TMEM accumulator
//     D_s, 7 x 64 of the 512 columns (no overflow: 7 pairs x 2^14 x K-chunk <= 16384 < 2^31).
//     WSSR_OZ_LEVELS=8 at build time keeps level 7 as well (34 pairs, dropped below 2^-59):
//     +9% smem-pipe time per pass for a closed-loop update error that measures the same
//     (DESIGN.md section 4);
//   * the epilogue combines sum_s D_s 2^(96 - 8 s) in FP64 and applies the power-of-two scales.
//
// Each element is thus represented to 2^-54 of its column's magnitude and every product and sum
// of digits is exact, so the result is FP64-grade (tests/test_gpu_ozaki.py compares the error
// with DMMA's against an exact reference).  O is read once per pass in its storage type (FP64
// or FP32) and digitised in shared memory on the fly: the pass is HBM-bound instead of
// FP64-tensor-bound.
//
// Kernel structure (one CTA per SM, persistent over work units = (row tile, 64-column block,
// K chunk)):
//   warp 0      TMA producer of the raw ring: O tile (+ mu/scale slice), 4 stages, freed by the
//               converters as soon as they have digitised it;
//   warp 2      TMA producer of the thin-operand digit tiles (4-stage ring);
//   warps 1, 3  MMA issuers taking alternate K-blocks (tcgen05.mma kind::i8, D in TMEM,
//               tcgen05.commit frees the stages); warp 1 also owns the TMEM allocation;
//   warps 4-19  converters in two groups taking alternate K-blocks: raw tile -> 7 int8 digit
//               planes (K-major, 32-byte swizzle) in shared memory; then all 16 run the epilogue (tcgen05.ld of the 8 accumulators, FP64 combine, store).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "engine.h"
#include "gemm.cuh"
#include "gemm_tma.cuh"
#include "ozaki.h"

namespace wssr {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();
bool make_map_2d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t pitch,
                 int box_outer, int esize);
bool make_map_1d(CUtensorMap* map, const double* ptr, int64_t n, int box);

namespace oz {

constexpr int BM = 128;            // rows of the output tile (TMEM lanes)
constexpr int BK = 32;             // K per stage (one kind::i8 MMA-K)
constexpr int ND = 7;              // digits per operand
#ifndef WSSR_OZ_LEVELS
#define WSSR_OZ_LEVELS 7
#endif
constexpr int NL = WSSR_OZ_LEVELS; // significance levels kept (s = a + b < NL), one TMEM block each
constexpr int NB = 64;             // output columns per unit
constexpr int BROWS = ND * NB;     // thin-operand digit rows per stage (448)
constexpr int RSTAGES = 3;         // raw tile ring (TMA -> converters)
constexpr int DSTAGES = 2;         // sample-digit ring (converters -> MMA)
constexpr int BSTAGES = 4;         // thin-operand digit ring (TMA -> MMA)
constexpr int KCHUNK = 16384;      // int32 accumulator bound (see header)
constexpr int kConvWarps = 16;
constexpr int kThreads = 32 * (4 + kConvWarps);
constexpr uint64_t kBias = 0x0080808080808080ull;

constexpr int A_RAW = BM * BK * 8;            // 32 KB (FP64 tile; FP32 uses half)
constexpr int A_DIG = ND * BM * BK;           // 28 KB
constexpr int B_DIG = BROWS * BK;             // 14 KB
constexpr int TABW = 4;                       // doubles per scale-table slot (see tab_slot)
constexpr int MI_BYTES = TABW * BK * 8;       // scale-table slice (row-major mode only)
constexpr int RSTAGE = A_RAW;                 // raw tile, 1 KB aligned
constexpr int DSTAGE = A_DIG;                 // 28 KB, 1 KB aligned
constexpr int BSTAGE = B_DIG;                 // 14 KB, 1 KB aligned
constexpr size_t kSmem = (size_t)RSTAGE * RSTAGES + (size_t)DSTAGE * DSTAGES +
                         (size_t)BSTAGE * BSTAGES + (size_t)MI_BYTES * RSTAGES + 256 + 1024;
static_assert(kSmem <= 232448, "shared memory budget");

// ---- tcgen05 / TMEM wrappers ------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ uint64_t smem_desc_sw32(uint32_t addr) {
  // K-major, SWIZZLE_32B: rows of 32 B, 8-row groups 256 B apart (SBO); LBO unused (1);
  // version 1 (sm_100); layout type 6.
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (16ull << 32) | (1ull << 46) |
         (6ull << 61);
}
__device__ __forceinline__ uint32_t idesc_i8(int n) {
  // D s32 (bits 4-5 = 2), A/B signed 8-bit (bits 7-9, 10-12 = 1), both K-major,
  // N >> 3 at bits 17-22, M >> 4 at bits 24-28 (M = 128).
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ uint64_t smem_desc_mn_sw32(uint32_t addr) {
  // MN-major, SWIZZLE_32B: 32 int8 along M per 32-byte row, 8-row K atoms of 256 B (SBO), the
  // four 32-wide M blocks 1 KB apart (LBO); layout type 6
  return (uint64_t)((addr >> 4) & 0x3FFF) | (64ull << 16) | (16ull << 32) | (1ull << 46) |
         (6ull << 61);
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// plain bulk copy global -> shared (contiguous bytes, no tensor map; the data are stored
// pre-swizzled so they land in the MMA's canonical layout)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}


// Biased integers Y = X + kBias -> digit planes: plane a holds byte (6 - a) of every Y (most
// significant digit first), XOR 0x80 = the signed digit.
// 8 biased integers -> 7 digit planes x 8 bytes (2 words each)
__device__ __forceinline__ void pack_digits8(const uint64_t (&y)[8], uint32_t (&w)[ND][2]) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint32_t l0 = (uint32_t)y[4 * q], l1 = (uint32_t)y[4 * q + 1];
    const uint32_t l2 = (uint32_t)y[4 * q + 2], l3 = (uint32_t)y[4 * q + 3];
    const uint32_t h0 = (uint32_t)(y[4 * q] >> 32), h1 = (uint32_t)(y[4 * q + 1] >> 32);
    const uint32_t h2 = (uint32_t)(y[4 * q + 2] >> 32), h3 = (uint32_t)(y[4 * q + 3] >> 32);
    uint32_t u0 = __byte_perm(l0, l1, 0x5140), u1 = __byte_perm(l0, l1, 0x7362);
    uint32_t v0 = __byte_perm(l2, l3, 0x5140), v1 = __byte_perm(l2, l3, 0x7362);
    w[6][q] = __byte_perm(u0, v0, 0x5410) ^ 0x80808080u;
    w[5][q] = __byte_perm(u0, v0, 0x7632) ^ 0x80808080u;
    w[4][q] = __byte_perm(u1, v1, 0x5410) ^ 0x80808080u;
    w[3][q] = __byte_perm(u1, v1, 0x7632) ^ 0x80808080u;
    u0 = __byte_perm(h0, h1, 0x5140);
    u1 = __byte_perm(h0, h1, 0x7362);
    v0 = __byte_perm(h2, h3, 0x5140);
    v1 = __byte_perm(h2, h3, 0x7362);
    w[2][q] = __byte_perm(u0, v0, 0x5410) ^ 0x80808080u;
    w[1][q] = __byte_perm(u0, v0, 0x7632) ^ 0x80808080u;
    w[0][q] = __byte_perm(u1, v1, 0x5410) ^ 0x80808080u;
  }
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

// mbarrier wait that suspends the thread in hardware until the phase flips (single-thread
// producer / MMA roles: no issue slots burnt spinning)
#ifdef WSSR_OZ_WATCHDOG
// debugging build: a wait that has not completed after ~2^28 polls reports where and traps
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __noinline__ void mbar_watch(uint64_t* bar, uint32_t parity) {
  for (long long i = 0; !mbar_try(bar, parity); ++i) {
    if (i == (1ll << 20)) {
      printf("WATCHDOG block %d warp %d lane %d bar smem+%u parity %u\n", blockIdx.x,
             threadIdx.x >> 5, threadIdx.x & 31, smem_u32(bar) & 0xFFFFF, parity);
      __trap();
    }
  }
}
__device__ __forceinline__ void mbar_sleep_wait(uint64_t* bar, uint32_t parity) {
  mbar_watch(bar, parity);
}
#define mbar_wait mbar_watch
#else
__device__ __forceinline__ void mbar_sleep_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif

// Slot of parameter p in the scale table: inside each block of 32 parameters the order is
// transposed (p % 8, p / 8 % 4) so that a converter warp's K-quarter groups read the 4
// parameters they need at one step from 64 contiguous bytes (one shared-memory wavefront).
__host__ __device__ __forceinline__ int64_t tab_slot(int64_t p) {
  return (p & ~int64_t(31)) | ((p & 7) << 2) | ((p >> 3) & 3);
}

__device__ __forceinline__ uint64_t to_biased(double x) {
  return (uint64_t)__double2ll_rn(x) + kBias;
}

// ---- digit integers ---------------------------------------------------------------------------
// X_np, the integer the 7 digits of element (n, p) represent, with s_p = 2^(54 - e_p):
//   |mu_p| <  2^(e_p + 1):  X = rint(O_np s_p) - rint(mu_p s_p)   (integer centring: |O s| < 2^56,
//                                                                  both conversions exact)
//   |mu_p| >= 2^(e_p + 1):  X = rint((O_np - mu_p) s_p)          (O - mu is exact by Sterbenz:
//                                                                  every O_np lies within 2^e_p
//                                                                  of mu_p, i.e. within a factor 2)
// Either way X is (O - mu) s to within one unit and |X| <= 2^54 + 1.  The scaling by s is an
// integer add to the exponent field, then one conversion (F2I): no FP64 arithmetic on the common
// path (FP64 SIMT shares the SM datapath with the int8 MMAs and stalls beside them; ncu of the
// earlier DADD/DMUL converters: "math" stalls on the DADDs dominated the converter warps).
// Scale-table slot p (tab_slot order, TABW doubles): {cw_p, s_p, mu_p, f} with
// cw_p = kBias - rint(mu_p s_p) as a 64-bit pattern, or kCwExact for the Sterbenz form, and f
// (a 64-bit pattern) nonzero in every slot of a 32-parameter block that holds a Sterbenz-form
// column: the converters branch on it once per K-block.  Padding slots: {kBias, 0, 0, f}.
constexpr uint64_t kCwExact = 0x8000000000000000ull;

// rint(v s) for s = 2^d, given as its high word hs = (d + 1023) << 20 (0 for padding columns):
// an integer add to the exponent field, then one conversion.  Branch-free; zero, subnormal,
// underflowing (|v s| < 2^-1022: rint 0) and non-finite inputs give 0.  The callers guarantee
// |v s| < 2^57, so the shifted exponent cannot overflow.
__device__ __forceinline__ long long rint_pow2(double v, uint32_t hs) {
  const uint32_t hi = (uint32_t)__double2hiint(v);
  const uint32_t ef = hi & 0x7ff00000u;
  const bool ok = ef - 0x00100000u < 0x7fe00000u && ef + hs > 0x3ff00000u;
  const long long r =
      __double2ll_rn(__hiloint2double((int)(hi + hs - 0x3ff00000u), __double2loint(v)));
  return ok ? r : 0;
}
__device__ __forceinline__ long long rint_pow2(float v, uint32_t hs) {
  const uint32_t b = (uint32_t)__float_as_int(v);
  const uint32_t ef = b & 0x7f800000u;
  const int d = (int)(hs >> 20) - 1023;
  const bool ok = ef - 0x00800000u < 0x7f000000u && (int)(ef >> 23) + d > 0;
  const long long r = __float2ll_rn(__int_as_float((int)(b + ((uint32_t)d << 23))));
  return ok ? r : 0;
}
__device__ __forceinline__ uint32_t hi_word(double s) { return (uint32_t)__double2hiint(s); }
// biased digit integer Y = X + kBias of sample value v: integer-form column {cw, s} ...
template <typename T>
__device__ __forceinline__ uint64_t biased_int(T v, uint64_t cw, uint32_t hs) {
  return (uint64_t)rint_pow2(v, hs) + cw;
}
// ... or a column of either form {cw, s, mu}
template <typename T>
__device__ __forceinline__ uint64_t biased_digits(T v, uint64_t cw, double s, double mu) {
  if (cw != kCwExact) return biased_int(v, cw, hi_word(s));
  return (uint64_t)rint_pow2((double)v - mu, hi_word(s)) + kBias;
}
__device__ __forceinline__ uint64_t as_u64(double x) { return (uint64_t)__double_as_longlong(x); }
// Precision guard counts of one biased digit integer y = X + kBias, packed for one 64-bit sum:
// low word +1 when X != 0, high word +1 when |X| >= 2^(54 - kGuardBits) (the element keeps at
// least 54 - kGuardBits bits of its own magnitude).
constexpr int kGuardBits = 12;
__device__ __forceinline__ uint64_t guard_count(uint64_t y) {
  const int64_t x = (int64_t)(y - kBias);
  const uint64_t a = (uint64_t)(x ^ (x >> 63));  // |X| (ones' complement: |X| - 1 for X < 0)
  return (uint64_t)(x != 0) | ((uint64_t)((a >> (54 - kGuardBits)) != 0) << 32);
}

// ---- digit pairs of one K-block -------------------------------------------------------------
// Sample digit a (most significant first) against the thin digits b, into the int32 level
// accumulators D_s, s = a + b < nl (TMEM columns 64 s ...), thin digits concatenated along N (up
// to 256 per MMA).  nds = 7, nl = NL = 7: the FP64 scheme (28 pairs, dropped levels below 2^-51.4 of
// the product of the column scales; NL = 8: 34 pairs, 2^-59).  nds = 5, nl = 6 for float32 samples: the top 5 of the same 7
// digit planes (X to 2^-38 of its column's scale - every float32 element within 14 binades of
// its column's maximum exactly) and levels to 2^-48: 20 pairs, 5 planes in HBM.  Digit 1 goes
// first and digit 0's range is split at column 64, so on a unit's first K-block (first = 0)
// every TMEM column is first written by an MMA with accumulate = 0.
// levels kept for NDS sample digits: NL (FP64 scheme) or NDS + 1
template <int NDS>
__host__ __device__ constexpr int levels() { return NDS == ND ? NL : NDS + 1; }

// One MMA per <= 256 thin-digit rows: sample digit a against thin digits b0 .. b0 + nb - 1,
// written to the levels a + b0 ... (all compile-time: descriptors and TMEM columns fold into
// immediates, so the issuing thread does no address arithmetic between MMAs).
template <int A, int B0, int NB, typename ADesc, typename BDesc>
__device__ __forceinline__ void issue_range(uint32_t tmem, ADesc adesc, BDesc bdesc,
                                            uint32_t amajor, uint32_t acc) {
  constexpr int left = 64 * NB, n0 = left > 256 ? 256 : left;
  if constexpr (left > 0) {
    mma_i8(tmem + 64 * (A + B0), adesc(A), bdesc(64 * B0), idesc_i8(n0) | amajor, acc);
    if constexpr (left > 256)
      issue_range<A, B0 + 4, NB - 4>(tmem, adesc, bdesc, amajor, acc);
  }
}
template <int A, int NDS, typename ADesc, typename BDesc>
__device__ __forceinline__ void issue_rest(uint32_t tmem, ADesc adesc, BDesc bdesc,
                                           uint32_t amajor) {
  if constexpr (A < NDS) {
    constexpr int L = levels<NDS>(), nb = (L - A) < ND ? (L - A) : ND;
    issue_range<A, 0, nb>(tmem, adesc, bdesc, amajor, 1u);
    issue_rest<A + 1, NDS>(tmem, adesc, bdesc, amajor);
  }
}
template <int NDS, typename ADesc, typename BDesc>
__device__ __forceinline__ void issue_pairs(uint32_t tmem, ADesc adesc, BDesc bdesc,
                                            uint32_t amajor, uint32_t first) {
  constexpr int L = levels<NDS>();
  constexpr int nb1 = (L - 1) < ND ? (L - 1) : ND, nb0 = (L < ND ? L : ND) - 1;
  issue_range<1, 0, nb1>(tmem, adesc, bdesc, amajor, first);
  issue_range<0, 0, 1>(tmem, adesc, bdesc, amajor, first);
  issue_range<0, 1, nb0>(tmem, adesc, bdesc, amajor, 1u);
  issue_rest<2, NDS>(tmem, adesc, bdesc, amajor);
}
// thin-digit rows of a K-block that the pairs read (64 per thin digit b < min(7, nl))
__host__ __device__ constexpr int thin_rows(int nl) { return NB * (nl < ND ? nl : ND); }

// profiling only (debug 9): per-K-block timestamps of CTA 0, see tools/ozaki_timeline.py
constexpr int kTraceBlocks = 96;
__device__ long long g_oz_trace[8][kTraceBlocks];

struct Params {
  // A: the sample block.  RM: A is (M x K) row-major (rows = samples, K = parameters, the
  // v = Ohat^T q pass); CM: A is stored (K x M) row-major (K = samples, M = parameters, the
  // u = Ohat v pass).
  int64_t M, K, N;
  int nblk, nch, mtiles;
  int64_t kblocks;
  const double* mu_inv;    // [Kpad or M][2] = {mu_p, 2^(54 - e_p)} per parameter column
  const double* colfac;    // [nblk * 64] thin-operand column factors
  double alpha;
  double* C;
  int64_t ldc;
  int accumulate;
  double* slab;            // nch > 1: [nch][M][N] partial results
  const int8_t* planes;    // pre-digitised: blocked, pre-swizzled planes [7][pblocks][prows][32]
  int64_t prows, pblocks;
  const int8_t* bd;        // blocked, pre-swizzled thin digits [nblk * kblocks][448][32]
  int8_t* store;           // on-the-fly v pass: also write the digit planes (layout as `planes`)
  unsigned long long* rowcnt;  // on-the-fly v pass: per sample row, packed digit-integer counts
                               // of the precision guard (see row_guard_kernel)
  int nds, nl;             // sample digits used (7; 5 for float32 samples) and levels kept
                           // (8; 6), see issue_pairs
  int debug;               // profiling only, low bits: 1 = skip digitising, 2 = skip MMAs,
                           // 3 = both, 4 = skip the sample-block loads too; +8 = trace CTA 0
};

template <bool RM, typename TA, int NDS>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmS, const Params p) {
  constexpr bool F32 = sizeof(TA) == 4;
  constexpr int A_BYTES = BM * BK * (int)sizeof(TA);
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1 KB-aligned base, derived from smem_raw without an integer round trip so every access
  // stays an explicit shared-memory instruction
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* dring = smem + (size_t)RSTAGE * RSTAGES;
  unsigned char* bring = dring + (size_t)DSTAGE * DSTAGES;
  unsigned char* miring = bring + (size_t)BSTAGE * BSTAGES;
  uint64_t* rfull = reinterpret_cast<uint64_t*>(miring + (size_t)MI_BYTES * RSTAGES);
  uint64_t* rempty = rfull + RSTAGES;
  uint64_t* bfull = rempty + RSTAGES;
  uint64_t* bempty = bfull + BSTAGES;
  uint64_t* conv = bempty + BSTAGES;
  uint64_t* dempty = conv + DSTAGES;
  uint64_t* tfull = dempty + DSTAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto a_raw = [&](int s) { return smem + (size_t)s * RSTAGE; };
  auto s_mi = [&](int s) { return reinterpret_cast<const double*>(miring + (size_t)s * MI_BYTES); };
  auto a_dig = [&](int d) { return dring + (size_t)d * DSTAGE; };
  auto b_dig = [&](int b) { return bring + (size_t)b * BSTAGE; };

  if (tid == 0) {
    for (int s = 0; s < RSTAGES; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], kConvWarps / 2);  // one converter group per K-block
    }
    for (int d = 0; d < DSTAGES; ++d) {
      mbar_init(&conv[d], kConvWarps / 2);
      mbar_init(&dempty[d], 1);
    }
    for (int b = 0; b < BSTAGES; ++b) {
      mbar_init(&bfull[b], 1);
      mbar_init(&bempty[b], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kConvWarps);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: barrier init and TMEM allocation above overlap the previous
  // kernel's tail; nothing before this point reads memory it writes
  pdl_wait();

  const int64_t units = (int64_t)p.mtiles * p.nblk * p.nch;
  // unit -> (64-column block fastest, then row tile, then K chunk): the column blocks of one row
  // tile run on neighbouring CTAs at the same time, so the second reads the tile from L2
  auto decode = [&](int64_t u, int64_t& m0, int& nb, int& kc, int64_t& kb0, int64_t& kb1) {
    nb = (int)(u % p.nblk);
    const int64_t rest = u / p.nblk;
    m0 = (rest % p.mtiles) * BM;
    kc = (int)(rest / p.mtiles);
    kb0 = p.kblocks * kc / p.nch;
    kb1 = p.kblocks * (kc + 1) / p.nch;
  };

  if (warp == 0) {
    // ===== TMA producer: raw ring =====
    if (lane == 0) {
      prefetch_tmap(&tmA);
      if (RM) prefetch_tmap(&tmS);
      uint32_t g = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t m0, kb0, kb1;
        int nb, kc;
        decode(u, m0, nb, kc, kb0, kb1);
        for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % RSTAGES;
          mbar_sleep_wait(&rempty[s], ((g / RSTAGES) & 1) ^ 1);
          if (p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks) g_oz_trace[0][g] = clock64();
          const int k0 = (int)(kb * BK);
          if ((p.debug & 7) == 4) {  // profiling: no sample-block traffic at all
            mbar_arrive(&rfull[s]);
            continue;
          }
          mbar_arrive_expect_tx(&rfull[s], A_BYTES + (RM ? MI_BYTES : 0));
          if (RM) {
            tma_load_2d(a_raw(s), &tmA, k0, (int)m0, &rfull[s]);
            if (!F32) tma_load_2d(a_raw(s) + 16384, &tmA, k0 + 16, (int)m0, &rfull[s]);
            tma_load_1d((void*)s_mi(s), &tmS, TABW * k0, &rfull[s]);
          } else {
            tma_load_2d(a_raw(s), &tmA, (int)m0, k0, &rfull[s]);
          }
        }
      }
    }
  } else if (warp == 2) {
    // ===== TMA producer: thin-operand digit tiles =====
    if (lane == 0) {
      uint32_t g = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t m0, kb0, kb1;
        int nb, kc;
        decode(u, m0, nb, kc, kb0, kb1);
        for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
          const int b = g % BSTAGES;
          mbar_sleep_wait(&bempty[b], ((g / BSTAGES) & 1) ^ 1);
          constexpr uint32_t bbytes = thin_rows(levels<NDS>()) * BK;
          mbar_arrive_expect_tx(&bfull[b], bbytes);
          bulk_load(b_dig(b), p.bd + (nb * p.kblocks + kb) * (int64_t)B_DIG, bbytes, &bfull[b]);
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ===== MMA issuers: warps 1 and 3 take alternate K-blocks =====
    // tcgen05.mma issue blocks while the tensor pipe is busy, so a single issuing thread would
    // expose its barrier waits between K-blocks.  Two warps alternate: one waits for its
    // K-block's operands while the other issues; a token passed through named barriers 1/2
    // keeps the issue order (a unit's accumulate = 0 MMAs come first).  Integer accumulation
    // is exact, so which warp issued a K-block does not affect the result.
    const int me = warp == 1 ? 0 : 1;
    int64_t total = 0;  // K-blocks of this CTA over all its units
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int64_t m0, kb0, kb1;
      int nb, kc;
      decode(u, m0, nb, kc, kb0, kb1);
      total += kb1 - kb0;
    }
    uint32_t g = 0, t = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++t) {
      int64_t m0, kb0, kb1;
      int nb, kc;
      decode(u, m0, nb, kc, kb0, kb1);
      // both issuers observe every tempty phase in order (a warp that skipped a unit would
      // otherwise see a stale parity two phases ahead): the epilogue of unit t-1 has drained
      // the TMEM before any K-block of unit t is issued
      mbar_sleep_wait(tempty, (t & 1) ^ 1);
      for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
        if ((int)(g & 1) != me) continue;
        const int d = g % DSTAGES, bs = g % BSTAGES;
        mbar_sleep_wait(&bfull[bs], (g / BSTAGES) & 1);
        mbar_sleep_wait(&conv[d], (g / DSTAGES) & 1);
        if (p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks && lane == 0)
          g_oz_trace[1][g] = clock64();
        if (g > 0) asm volatile("bar.sync %0, 64;\n" ::"r"(1 + me) : "memory");  // token in
        if (p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks && lane == 0)
          g_oz_trace[2][g] = clock64();
        tc_fence_after();
        const bool stored = RM && p.store && nb == 0;
        if (lane == 0 && stored) {
          // the digit tile in shared memory already has the planes' pre-swizzled layout:
          // one 4 KB bulk store per plane (async; its shared-memory reads are awaited before
          // this stage's slot is released below)
          const int64_t pstride = p.pblocks * p.prows * 32;
#pragma unroll
          for (int a = 0; a < NDS; ++a)
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;\n" ::"l"(
                    p.store + a * pstride + (kb * p.prows + m0) * 32),
                "r"(smem_u32(a_dig(d) + a * BM * BK))
                : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        if (lane == 0) {
          if ((p.debug & 7) != 2 && (p.debug & 7) != 3) {
            const uint32_t abase = smem_u32(a_dig(d)), bbase = smem_u32(b_dig(bs));
            const uint32_t first = kb == kb0 ? 0u : 1u;
            issue_pairs<NDS>(
                tmem, [&](int a) { return smem_desc_sw32(abase + a * BM * BK); },
                [&](int row) { return smem_desc_sw32(bbase + row * BK); }, 0u, first);
          }
          // commits track this thread's MMAs; the tensor pipe executes in issue order, so the
          // other warp's earlier K-blocks are complete as well
          if (stored) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          mma_commit(&dempty[d]);
          mma_commit(&bempty[bs]);
          if (kb + 1 == kb1) mma_commit(tfull);
          if (p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks) g_oz_trace[3][g] = clock64();
        }
        __syncwarp();
        if ((int64_t)g + 1 < total) asm volatile("bar.arrive %0, 64;\n" ::"r"(2 - me) : "memory");
      }
    }
  } else if (warp >= 4) {
    // ===== converters + epilogue =====
    // Two groups of 8 warps take alternate K-blocks (each has two K-blocks of time per block).
    // Group warp wi owns tile rows 16 wi + r8 and 16 wi + 8 + r8, lane = r8 + 8 q: K quarter q
    // (8 consecutive K values) - quarter-warps read 8 rows of one K range (conflict-free under
    // the 128-byte swizzle) and a warp's digit stores cover 8 full 32-byte rows.
    const int cw = warp - 4;
    const int cg = cw >> 3, wi = cw & 7;
    const int q = lane >> 3;
    const int rowA = 16 * wi + (lane & 7), rowB = rowA + 8;
    const int quad = warp & 3;                // TMEM lane quadrant of this warp (epilogue)
    const int ecol = 16 * (cw >> 2);          // epilogue column group
    const int erow = quad * 32 + lane;
    auto convert8 = [&](int s, int row, uint64_t cw_r, double inv_r, double mu_r, bool exact,
                        uint64_t (&y)[8]) {
      if (RM) {
        // the table slot of K index 8 q + i is 4 i + q: {cw, s} at double2 8 i + 2 q, mu next;
        // `exact`: this K-block has Sterbenz-form columns (uniform over the CTA)
        const double2* mi = reinterpret_cast<const double2*>(s_mi(s)) + 2 * q;
        if (F32) {
          const unsigned char* base = a_raw(s) + row * 128;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const float4 f = *reinterpret_cast<const float4*>(
                base + (((2 * q + c) ^ (row & 7)) << 4));
            const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const double2 m = mi[8 * (4 * c + e)];
              y[4 * c + e] = exact ? biased_digits(fv[e], as_u64(m.x), m.y, mi[8 * (4 * c + e) + 1].x)
                                   : biased_int(fv[e], as_u64(m.x), hi_word(m.y));
            }
          }
        } else {
          const unsigned char* base = a_raw(s) + (q >> 1) * 16384 + row * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double2 v =
                *reinterpret_cast<const double2*>(base + (((4 * (q & 1) + c) ^ (row & 7)) << 4));
            const double2 m0v = mi[8 * (2 * c)], m1v = mi[8 * (2 * c + 1)];
            if (exact) {
              y[2 * c] = biased_digits(v.x, as_u64(m0v.x), m0v.y, mi[8 * (2 * c) + 1].x);
              y[2 * c + 1] = biased_digits(v.y, as_u64(m1v.x), m1v.y, mi[8 * (2 * c + 1) + 1].x);
            } else {
              y[2 * c] = biased_int(v.x, as_u64(m0v.x), hi_word(m0v.y));
              y[2 * c + 1] = biased_int(v.y, as_u64(m1v.x), hi_word(m1v.y));
            }
          }
        }
      } else {
        const TA* base = reinterpret_cast<const TA*>(a_raw(s)) + (8 * q) * BM + row;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          y[i] = exact ? biased_digits(base[i * BM], cw_r, inv_r, mu_r)
                       : biased_int(base[i * BM], cw_r, hi_word(inv_r));
      }
    };
    // row-major fast path (no Sterbenz-form column in the K-block): the table entries of this
    // thread's 8 K values are read once and serve both of its rows
    auto load_tab = [&](int s, uint64_t (&cw)[8], uint32_t (&hs)[8]) {
      const double2* mi = reinterpret_cast<const double2*>(s_mi(s)) + 2 * q;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double2 m = mi[8 * j];
        cw[j] = as_u64(m.x);
        hs[j] = hi_word(m.y);
      }
    };
    auto convert8_tab = [&](int s, int row, const uint64_t (&cw)[8], const uint32_t (&hs)[8],
                            uint64_t (&y)[8]) {
      if (F32) {
        const unsigned char* base = a_raw(s) + row * 128;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float4 f =
              *reinterpret_cast<const float4*>(base + (((2 * q + c) ^ (row & 7)) << 4));
          const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) y[4 * c + e] = biased_int(fv[e], cw[4 * c + e], hs[4 * c + e]);
        }
      } else {
        const unsigned char* base = a_raw(s) + (q >> 1) * 16384 + row * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 v =
              *reinterpret_cast<const double2*>(base + (((4 * (q & 1) + c) ^ (row & 7)) << 4));
          y[2 * c] = biased_int(v.x, cw[2 * c], hs[2 * c]);
          y[2 * c + 1] = biased_int(v.y, cw[2 * c + 1], hs[2 * c + 1]);
        }
      }
    };
    // column-major fast path: the K rows of the raw tile are 1 KB apart, so the four K-quarter
    // lane groups of a row would hit the same banks (4-way).  Odd quarters read row B while even
    // ones read row A (64 bytes apart: the other 16 banks), then the other row: 2-way at most,
    // i.e. the ideal two wavefronts per 256-byte load.
    auto convert16_cm = [&](int s, uint64_t cw_a, uint32_t hs_a, uint64_t cw_b, uint32_t hs_b,
                            uint64_t (&ya)[8], uint64_t (&yb)[8]) {
      const TA* base = reinterpret_cast<const TA*>(a_raw(s)) + (8 * q) * BM;
      const bool odd = q & 1;
      const TA* p0 = base + (odd ? rowB : rowA);
      const TA* p1 = base + (odd ? rowA : rowB);
      TA x0[8], x1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x0[i] = p0[i * BM];
#pragma unroll
      for (int i = 0; i < 8; ++i) x1[i] = p1[i * BM];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        ya[i] = biased_int(odd ? x1[i] : x0[i], cw_a, hs_a);
        yb[i] = biased_int(odd ? x0[i] : x1[i], cw_b, hs_b);
      }
    };
    auto store8 = [&](int d, int row, const uint32_t (&w)[ND][2]) {
      unsigned char* dst =
          a_dig(d) + row * BK + ((((q >> 1) ^ ((row >> 2) & 1))) << 4) + ((q & 1) << 3);
#pragma unroll
      for (int a = 0; a < ND; ++a)
        *reinterpret_cast<uint2*>(dst + a * BM * BK) = make_uint2(w[a][0], w[a][1]);
    };
    uint32_t g = 0, t = 0;
    const bool guard = RM && p.rowcnt != nullptr;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++t) {
      int64_t m0, kb0, kb1;
      int nb, kc;
      decode(u, m0, nb, kc, kb0, kb1);
      uint64_t cntA = 0, cntB = 0;  // precision guard counts over this unit's K range
      double muA = 0.0, invA = 0.0, muB = 0.0, invB = 0.0;
      uint64_t cwA = kBias, cwB = kBias;
      if (!RM) {
        if (m0 + rowA < p.M) {
          const double* t = p.mu_inv + TABW * tab_slot(m0 + rowA);
          cwA = as_u64(t[0]);
          invA = t[1];
          muA = t[2];
        }
        if (m0 + rowB < p.M) {
          const double* t = p.mu_inv + TABW * tab_slot(m0 + rowB);
          cwB = as_u64(t[0]);
          invB = t[1];
          muB = t[2];
        }
      }
      // CM: a row's column form is fixed over the unit; one vote makes the branch warp-uniform
      const bool exactCM = !RM && __any_sync(0xffffffffu, cwA == kCwExact || cwB == kCwExact);
      for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
        if ((int)(g & 1) != cg) continue;
        const int s = g % RSTAGES, d = g % DSTAGES;
        mbar_wait(&rfull[s], (g / RSTAGES) & 1);
        const bool tr = p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks && lane == 0 && wi == 0;
        if (tr) g_oz_trace[4][g] = clock64();
        if ((p.debug & 7) == 1 || (p.debug & 7) == 3 || (p.debug & 7) == 4) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&rempty[s]);
          mbar_wait(&dempty[d], ((g / DSTAGES) & 1) ^ 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[d]);
          continue;
        }
        // one row at a time (digits packed before the next row converts: fewer live registers)
        uint32_t wA[ND][2], wB[ND][2];
        const bool exact =
            RM ? __double_as_longlong(s_mi(s)[3]) != 0 : exactCM;  // uniform per K-block
        if (!RM && !exact) {
          uint64_t ya[8], yb[8];
          convert16_cm(s, cwA, hi_word(invA), cwB, hi_word(invB), ya, yb);
          pack_digits8(ya, wA);
          pack_digits8(yb, wB);
        } else if (RM && !exact) {
          uint64_t tcw[8];
          uint32_t ths[8];
          load_tab(s, tcw, ths);
          {
            uint64_t y[8];
            convert8_tab(s, rowA, tcw, ths, y);
            if (guard) {
#pragma unroll
              for (int i = 0; i < 8; ++i) cntA += guard_count(y[i]);
            }
            pack_digits8(y, wA);
          }
          {
            uint64_t y[8];
            convert8_tab(s, rowB, tcw, ths, y);
            if (guard) {
#pragma unroll
              for (int i = 0; i < 8; ++i) cntB += guard_count(y[i]);
            }
            pack_digits8(y, wB);
          }
        } else {
          {
            uint64_t y[8];
            convert8(s, rowA, cwA, invA, muA, exact, y);
            if (guard) {
#pragma unroll
              for (int i = 0; i < 8; ++i) cntA += guard_count(y[i]);
            }
            pack_digits8(y, wA);
          }
          {
            uint64_t y[8];
            convert8(s, rowB, cwB, invB, muB, exact, y);
            if (guard) {
#pragma unroll
              for (int i = 0; i < 8; ++i) cntB += guard_count(y[i]);
            }
            pack_digits8(y, wB);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[s]);  // raw tile consumed (values are in registers)
        if (tr) g_oz_trace[5][g] = clock64();
        mbar_wait(&dempty[d], ((g / DSTAGES) & 1) ^ 1);  // MMA done with this digit slot
        if (tr) g_oz_trace[6][g] = clock64();
        store8(d, rowA, wA);
        store8(d, rowB, wB);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[d]);
        if (tr) g_oz_trace[7][g] = clock64();
      }
      if (guard) {
        // the 4 K-quarter lanes of a row, then one atomic per row (integer sums: exact and
        // order-independent)
        cntA += __shfl_xor_sync(0xffffffffu, cntA, 8);
        cntA += __shfl_xor_sync(0xffffffffu, cntA, 16);
        cntB += __shfl_xor_sync(0xffffffffu, cntB, 8);
        cntB += __shfl_xor_sync(0xffffffffu, cntB, 16);
        if (q == 0) {
          if (cntA && m0 + rowA < p.M) atomicAdd(p.rowcnt + m0 + rowA, (unsigned long long)cntA);
          if (cntB && m0 + rowB < p.M) atomicAdd(p.rowcnt + m0 + rowB, (unsigned long long)cntB);
        }
      }
      // ---- epilogue: D_s (s = 0..7) -> FP64 ----
      mbar_sleep_wait(tfull, t & 1);
      tc_fence_after();
      const int64_t gm = m0 + erow;
      double rowfac = 1.0;
      if (!RM && gm < p.M) rowfac = 1.0 / p.mu_inv[TABW * tab_slot(gm) + 1];
      double acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
      for (int sd = 0; sd < levels<NDS>(); ++sd) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + NB * sd + ecol, r);
        tmem_ld_wait();
        const double wgt = __longlong_as_double((long long)(1023 + 96 - 8 * sd) << 52);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = fma((double)(int)r[j], wgt, acc[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);  // TMEM may be overwritten by the next unit
      if (gm < p.M) {
        const int64_t gj0 = (int64_t)nb * NB + ecol;
        const double rf = p.alpha * rowfac;
        if (p.nch > 1) {
          double* dst = p.slab + ((int64_t)kc * p.M + gm) * p.N;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (gj0 + j < p.N) dst[gj0 + j] = rf * p.colfac[gj0 + j] * acc[j];
        } else {
          double* dst = p.C + gm * p.ldc;
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (gj0 + j < p.N) {
              const double v = rf * p.colfac[gj0 + j] * acc[j];
              dst[gj0 + j] = p.accumulate ? dst[gj0 + j] + v : v;
            }
        }
      }
    }
  }
  if ((warp == 1 || warp == 3) && lane == 0 && RM && p.store)
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // digit planes written
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem)
                 : "memory");
  }
}

// ---- transposed on-the-fly variant (row-major pass, 65-128 thin columns) --------------------
// With 128 thin columns (k = 128: c2/c3) the kernel above runs each 128-row tile twice, once per
// 64-column block, because one block's 8 int32 level accumulators fill the 512 TMEM columns -
// and so converts every sample twice.  This variant swaps the operand roles: the thin digits are
// the MMA's A operand (M = 128 thin columns) and the sample digits its B operand (N = 64 samples
// per digit, digits stacked along N), so D_s holds 128 thin columns x 64 samples per level
// (8 x 64 TMEM columns again) and every sample is converted once for all 128 columns.  The
// tensor-core operand traffic per product is unchanged; the conversion traffic through the
// shared-memory pipe (raw-tile TMA writes and reads, digit stores, scale table) halves.
constexpr int TBM = 64;                         // sample rows per unit
constexpr int T_RSTAGES = 4;                    // raw ring
constexpr int T_DSTAGES = 3;                    // sample-digit ring (converters -> MMA)
constexpr int T_BSTAGES = 3;                    // thin-digit ring (bulk copies -> MMA)
constexpr int T_RSTAGE = TBM * BK * 8;          // 16 KB (FP64 tile; FP32 uses half)
constexpr int T_DSTAGE = ND * TBM * BK;         // 14 KB
constexpr int T_BSTAGE = ND * 128 * BK;         // 28 KB
constexpr size_t kTSmem = (size_t)T_RSTAGE * T_RSTAGES + (size_t)T_DSTAGE * T_DSTAGES +
                          (size_t)T_BSTAGE * T_BSTAGES + (size_t)MI_BYTES * T_RSTAGES + 256 + 1024;
static_assert(kTSmem <= 232448, "shared memory budget");

// Digit pairs with the roles swapped: A digit x (thin, 7 digits) against B digits y (samples,
// NB digits), levels x + y < L.  First writers as in issue_pairs: x = 1 covers levels 1..L-1
// (NB >= L - 1), then x = 0 splits at level 0.
template <int X, int Y0, int NY, typename ADesc, typename BDesc>
__device__ __forceinline__ void issue_range_t(uint32_t tmem, ADesc adesc, BDesc bdesc,
                                              uint32_t acc) {
  constexpr int left = 64 * NY, n0 = left > 256 ? 256 : left;
  if constexpr (left > 0) {
    mma_i8(tmem + 64 * (X + Y0), adesc(X), bdesc(64 * Y0), idesc_i8(n0), acc);
    if constexpr (left > 256) issue_range_t<X, Y0 + 4, NY - 4>(tmem, adesc, bdesc, acc);
  }
}
template <int X, int NB, int L, typename ADesc, typename BDesc>
__device__ __forceinline__ void issue_rest_t(uint32_t tmem, ADesc adesc, BDesc bdesc) {
  if constexpr (X < ND && X < L) {
    constexpr int ny = (L - X) < NB ? (L - X) : NB;
    issue_range_t<X, 0, ny>(tmem, adesc, bdesc, 1u);
    issue_rest_t<X + 1, NB, L>(tmem, adesc, bdesc);
  }
}
template <int NB, typename ADesc, typename BDesc>
__device__ __forceinline__ void issue_pairs_t(uint32_t tmem, ADesc adesc, BDesc bdesc,
                                              uint32_t first) {
  constexpr int L = levels<NB>();
  static_assert(NB >= L - 1, "x = 1 must cover levels 1..L-1");
  issue_range_t<1, 0, L - 1>(tmem, adesc, bdesc, first);
  issue_range_t<0, 0, 1>(tmem, adesc, bdesc, first);
  issue_range_t<0, 1, (L < NB ? L : NB) - 1>(tmem, adesc, bdesc, 1u);
  issue_rest_t<2, NB, L>(tmem, adesc, bdesc);
}

template <bool RM, typename TA, int NDS>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_gemm_t_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmS, const Params p) {
  constexpr bool F32 = sizeof(TA) == 4;
  constexpr int A_BYTES = TBM * BK * (int)sizeof(TA);
  constexpr int L = levels<NDS>();
  constexpr int THIN = L < ND ? L : ND;  // thin digits the pairs read
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* dring = smem + (size_t)T_RSTAGE * T_RSTAGES;
  unsigned char* bring = dring + (size_t)T_DSTAGE * T_DSTAGES;
  unsigned char* miring = bring + (size_t)T_BSTAGE * T_BSTAGES;
  uint64_t* rfull = reinterpret_cast<uint64_t*>(miring + (size_t)MI_BYTES * T_RSTAGES);
  uint64_t* rempty = rfull + T_RSTAGES;
  uint64_t* bfull = rempty + T_RSTAGES;
  uint64_t* bempty = bfull + T_BSTAGES;
  uint64_t* conv = bempty + T_BSTAGES;
  uint64_t* dempty = conv + T_DSTAGES;
  uint64_t* tfull = dempty + T_DSTAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto a_raw = [&](int s) { return smem + (size_t)s * T_RSTAGE; };
  auto s_mi = [&](int s) { return reinterpret_cast<const double*>(miring + (size_t)s * MI_BYTES); };
  auto s_dig = [&](int d) { return dring + (size_t)d * T_DSTAGE; };
  auto t_dig = [&](int b) { return bring + (size_t)b * T_BSTAGE; };

  if (tid == 0) {
    for (int s = 0; s < T_RSTAGES; ++s) {
      mbar_init(&rfull[s], 1);
      mbar_init(&rempty[s], kConvWarps / 2);
    }
    for (int d = 0; d < T_DSTAGES; ++d) {
      mbar_init(&conv[d], kConvWarps / 2);
      mbar_init(&dempty[d], 1);
    }
    for (int b = 0; b < T_BSTAGES; ++b) {
      mbar_init(&bfull[b], 1);
      mbar_init(&bempty[b], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, kConvWarps);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  const int64_t units = (int64_t)p.mtiles * p.nch;  // mtiles: 64-row tiles here
  auto decode = [&](int64_t u, int64_t& m0, int& kc, int64_t& kb0, int64_t& kb1) {
    m0 = (u % p.mtiles) * TBM;
    kc = (int)(u / p.mtiles);
    kb0 = p.kblocks * kc / p.nch;
    kb1 = p.kblocks * (kc + 1) / p.nch;
  };

  if (warp == 0) {
    // ===== TMA producer: raw ring (RM: 64 sample rows x 32 parameters + the scale-table slice;
    // CM: 32 sample rows x 64 parameters) =====
    if (lane == 0) {
      prefetch_tmap(&tmA);
      if (RM) prefetch_tmap(&tmS);
      uint32_t g = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t m0, kb0, kb1;
        int kc;
        decode(u, m0, kc, kb0, kb1);
        for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
          const int s = g % T_RSTAGES;
          mbar_sleep_wait(&rempty[s], ((g / T_RSTAGES) & 1) ^ 1);
          const int k0 = (int)(kb * BK);
          if (RM) {
            mbar_arrive_expect_tx(&rfull[s], A_BYTES + MI_BYTES);
            tma_load_2d(a_raw(s), &tmA, k0, (int)m0, &rfull[s]);
            if (!F32) tma_load_2d(a_raw(s) + TBM * 128, &tmA, k0 + 16, (int)m0, &rfull[s]);
            tma_load_1d((void*)s_mi(s), &tmS, TABW * k0, &rfull[s]);
          } else {
            mbar_arrive_expect_tx(&rfull[s], A_BYTES);
            tma_load_2d(a_raw(s), &tmA, (int)m0, k0, &rfull[s]);
          }
        }
      }
    }
  } else if (warp == 2) {
    // ===== bulk producer: thin digits of a K-block, [digit][128 columns][32 K] =====
    if (lane == 0) {
      uint32_t g = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t m0, kb0, kb1;
        int kc;
        decode(u, m0, kc, kb0, kb1);
        for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
          const int b = g % T_BSTAGES;
          mbar_sleep_wait(&bempty[b], ((g / T_BSTAGES) & 1) ^ 1);
          constexpr uint32_t bbytes = THIN * 128 * BK;
          mbar_arrive_expect_tx(&bfull[b], bbytes);
          bulk_load(t_dig(b), p.bd + kb * (int64_t)T_BSTAGE, bbytes, &bfull[b]);
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ===== MMA issuers, alternate K-blocks (see ozaki_gemm_kernel) =====
    const int me = warp == 1 ? 0 : 1;
    int64_t total = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int64_t m0, kb0, kb1;
      int kc;
      decode(u, m0, kc, kb0, kb1);
      total += kb1 - kb0;
    }
    uint32_t g = 0, t = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++t) {
      int64_t m0, kb0, kb1;
      int kc;
      decode(u, m0, kc, kb0, kb1);
      mbar_sleep_wait(tempty, (t & 1) ^ 1);
      for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
        if ((int)(g & 1) != me) continue;
        const int d = g % T_DSTAGES, bs = g % T_BSTAGES;
        mbar_sleep_wait(&bfull[bs], (g / T_BSTAGES) & 1);
        mbar_sleep_wait(&conv[d], (g / T_DSTAGES) & 1);
        if (g > 0) asm volatile("bar.sync %0, 64;\n" ::"r"(1 + me) : "memory");  // token in
        tc_fence_after();
        const bool stored = RM && p.store != nullptr && m0 < p.prows;
        if (lane == 0 && stored) {
          // one 2 KB bulk store per plane: the 64-row digit tile is already in the planes'
          // pre-swizzled layout
          const int64_t pstride = p.pblocks * p.prows * 32;
#pragma unroll
          for (int a = 0; a < NDS; ++a)
            asm volatile(
                "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 2048;\n" ::"l"(
                    p.store + a * pstride + (kb * p.prows + m0) * 32),
                "r"(smem_u32(s_dig(d) + a * TBM * BK))
                : "memory");
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        if (lane == 0) {
          const uint32_t abase = smem_u32(t_dig(bs)), bbase = smem_u32(s_dig(d));
          const uint32_t first = kb == kb0 ? 0u : 1u;
          issue_pairs_t<NDS>(
              tmem, [&](int x) { return smem_desc_sw32(abase + x * 128 * BK); },
              [&](int row) { return smem_desc_sw32(bbase + row * BK); }, first);
          if (stored) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
          mma_commit(&dempty[d]);
          mma_commit(&bempty[bs]);
          if (kb + 1 == kb1) mma_commit(tfull);
        }
        __syncwarp();
        if ((int64_t)g + 1 < total) asm volatile("bar.arrive %0, 64;\n" ::"r"(2 - me) : "memory");
      }
    }
  } else if (warp >= 4) {
    // ===== converters + epilogue =====
    // Two groups of 8 warps take alternate K-blocks; one tile row and one K quarter q (8
    // consecutive K values) per thread.
    //   RM: group warp wi owns tile rows 8 wi + r8, lane = r8 + 8 q (the raw rows are 128-byte
    //       swizzled, so the quarter-warps of one row range read distinct banks).
    //   CM: the raw tile is [32 samples][64 parameters] unswizzled, K rows 512 bytes apart, so
    //       the lanes of a warp cover 16 consecutive parameters (128 bytes, all 32 banks) x 2
    //       quarters: row = 16 (wi & 3) + r16, q = 2 (wi >> 2) + lane / 16.  Loads are then two
    //       wavefronts per 256 bytes, and the digit stores of 16 rows x 16 bytes (one 16-byte
    //       half of each row, flipped with bit 2 of the row) hit every bank once per 8 rows.
    const int cw = warp - 4;
    const int cg = cw >> 3, wi = cw & 7;
    const int q = RM ? lane >> 3 : 2 * (wi >> 2) + (lane >> 4);
    const int row = RM ? 8 * wi + (lane & 7) : 16 * (wi & 3) + (lane & 15);
    const int quad = warp & 3;          // TMEM lane quadrant of this warp (epilogue)
    const int ecol = 16 * (cw >> 2);    // epilogue: 16 sample (RM) / parameter (CM) columns
    const bool guard = RM && p.rowcnt != nullptr;
    uint32_t g = 0, t = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++t) {
      int64_t m0, kb0, kb1;
      int kc;
      decode(u, m0, kc, kb0, kb1);
      uint64_t cnt = 0;
      // CM: this thread's parameter column is fixed over the unit
      uint64_t cwr = kBias;
      double invr = 0.0, mur = 0.0;
      if (!RM && m0 + row < p.M) {
        const double* tb = p.mu_inv + TABW * tab_slot(m0 + row);
        cwr = as_u64(tb[0]);
        invr = tb[1];
        mur = tb[2];
      }
      const bool exactCM = !RM && __any_sync(0xffffffffu, cwr == kCwExact);
      for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
        if ((int)(g & 1) != cg) continue;
        const int s = g % T_RSTAGES, d = g % T_DSTAGES;
        mbar_wait(&rfull[s], (g / T_RSTAGES) & 1);
        const double2* mi = reinterpret_cast<const double2*>(s_mi(s)) + 2 * q;
        uint64_t y[8];
        if (!RM) {
          const TA* base = reinterpret_cast<const TA*>(a_raw(s)) + (8 * q) * TBM + row;
          TA x[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = base[i * TBM];
          if (exactCM) {
#pragma unroll
            for (int i = 0; i < 8; ++i) y[i] = biased_digits(x[i], cwr, invr, mur);
          } else {
            const uint32_t hs = hi_word(invr);
#pragma unroll
            for (int i = 0; i < 8; ++i) y[i] = biased_int(x[i], cwr, hs);
          }
        } else if (F32) {
          const bool exact = __double_as_longlong(s_mi(s)[3]) != 0;  // uniform per K-block
          const unsigned char* base = a_raw(s) + row * 128;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const float4 f =
                *reinterpret_cast<const float4*>(base + (((2 * q + c) ^ (row & 7)) << 4));
            const float fv[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const double2 m = mi[8 * (4 * c + e)];
              y[4 * c + e] = exact ? biased_digits(fv[e], as_u64(m.x), m.y, mi[8 * (4 * c + e) + 1].x)
                                   : biased_int(fv[e], as_u64(m.x), hi_word(m.y));
            }
          }
        } else {
          const bool exact = __double_as_longlong(s_mi(s)[3]) != 0;  // uniform per K-block
          const unsigned char* base = a_raw(s) + (q >> 1) * (TBM * 128) + row * 128;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double2 v =
                *reinterpret_cast<const double2*>(base + (((4 * (q & 1) + c) ^ (row & 7)) << 4));
            const double2 m0v = mi[8 * (2 * c)], m1v = mi[8 * (2 * c + 1)];
            if (exact) {
              y[2 * c] = biased_digits(v.x, as_u64(m0v.x), m0v.y, mi[8 * (2 * c) + 1].x);
              y[2 * c + 1] = biased_digits(v.y, as_u64(m1v.x), m1v.y, mi[8 * (2 * c + 1) + 1].x);
            } else {
              y[2 * c] = biased_int(v.x, as_u64(m0v.x), hi_word(m0v.y));
              y[2 * c + 1] = biased_int(v.y, as_u64(m1v.x), hi_word(m1v.y));
            }
          }
        }
        if (guard) {
#pragma unroll
          for (int i = 0; i < 8; ++i) cnt += guard_count(y[i]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&rempty[s]);  // raw tile consumed
        uint32_t w[ND][2];
        pack_digits8(y, w);
        mbar_wait(&dempty[d], ((g / T_DSTAGES) & 1) ^ 1);
        unsigned char* dst = s_dig(d) + row * BK + ((((q >> 1) ^ ((row >> 2) & 1))) << 4) +
                             ((q & 1) << 3);
#pragma unroll
        for (int a = 0; a < ND; ++a)
          *reinterpret_cast<uint2*>(dst + a * TBM * BK) = make_uint2(w[a][0], w[a][1]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[d]);
      }
      if (guard) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, 8);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, 16);
        if (q == 0 && cnt && m0 + row < p.M) atomicAdd(p.rowcnt + m0 + row, (unsigned long long)cnt);
      }
      // ---- epilogue: D_s (128 thin columns x 64 samples per level) -> FP64 ----
      mbar_sleep_wait(tfull, t & 1);
      tc_fence_after();
      double acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
      for (int sd = 0; sd < L; ++sd) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + NB * sd + ecol, r);
        tmem_ld_wait();
        const double wgt = __longlong_as_double((long long)(1023 + 96 - 8 * sd) << 52);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = fma((double)(int)r[j], wgt, acc[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      const int64_t jcol = quad * 32 + lane;  // thin column = TMEM lane
      if (jcol < p.N) {
        const double cf = p.alpha * p.colfac[jcol];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int64_t gm = m0 + ecol + c;
          if (gm < p.M) {
            // CM: output row = parameter column gm, whose digits carry the scale s_gm
            const double v =
                RM ? cf * acc[c] : cf * acc[c] / p.mu_inv[TABW * tab_slot(gm) + 1];
            if (p.nch > 1) {
              p.slab[((int64_t)kc * p.M + gm) * p.N + jcol] = v;
            } else {
              double* dst = p.C + gm * p.ldc + jcol;
              *dst = p.accumulate ? *dst + v : v;
            }
          }
        }
      }
    }
  }
  if ((warp == 1 || warp == 3) && lane == 0 && RM && p.store)
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem)
                 : "memory");
  }
}

// ---- pre-digitised variant ---------------------------------------------------------------------
// When the step's digit planes fit in HBM they are written once per step (digitize_kernel, with
// no tensor-core work running: FP64 SIMT arithmetic shares the SM's math datapath with the
// int8 MMAs and runs ~2.5x slower beside them), and every O-pass streams them with TMA straight
// into the MMA operands: planes [7][N][Ppad] int8, parameter-contiguous.  The u = Ohat v pass
// reads the same planes as an MN-major operand (parameters along M), so one layout serves both.
constexpr int PBK = 32;                // K per stage (kind::i8 MMA-K steps of 32 bytes)
constexpr int PA_DIG = ND * BM * PBK;  // 28 KB
constexpr int PB_DIG = BROWS * PBK;    // 14 KB
constexpr int PSTAGES = 5;             // sample-digit ring (deep: the tiles stream from HBM)
constexpr int PBSTAGES = 5;            // thin-operand digit ring
constexpr int kPreThreads = 256;       // warps 0,2 producers; 1,3 MMA issuers; 4-7 epilogue
constexpr size_t kPreSmem = (size_t)PA_DIG * PSTAGES + (size_t)PB_DIG * PBSTAGES + 256 + 1024;

__device__ __forceinline__ uint64_t smem_desc_sw64(uint32_t addr) {
  // K-major, SWIZZLE_64B: rows of 64 B, 8-row groups 512 B apart (SBO); layout type 4
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (32ull << 32) | (1ull << 46) |
         (4ull << 61);
}

__device__ __forceinline__ uint64_t smem_desc_mn_sw128(uint32_t addr) {
  // MN-major, SWIZZLE_128B: 128 int8 along M per 128-byte row, 8-row atoms of 1 KB along K (SBO)
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

template <bool RM, int NDS>
__global__ void __launch_bounds__(kPreThreads, 1)
    ozaki_pre_kernel(const __grid_constant__ CUtensorMap tmA, const Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* bring = smem + (size_t)PA_DIG * PSTAGES;
  uint64_t* afull = reinterpret_cast<uint64_t*>(bring + (size_t)PB_DIG * PBSTAGES);
  uint64_t* aempty = afull + PSTAGES;
  uint64_t* bfull = aempty + PSTAGES;
  uint64_t* bempty = bfull + PBSTAGES;
  uint64_t* tfull = bempty + PBSTAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto a_dig = [&](int s) { return smem + (size_t)s * PA_DIG; };
  auto b_dig = [&](int s) { return bring + (size_t)s * PB_DIG; };

  if (tid == 0) {
    for (int s = 0; s < PSTAGES; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < PBSTAGES; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
                     smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: barrier init and TMEM allocation above overlap the previous
  // kernel's tail; nothing before this point reads memory it writes
  pdl_wait();

  const int64_t units = (int64_t)p.mtiles * p.nblk * p.nch;
  // unit -> (64-column block fastest, then row tile, then K chunk): the column blocks of one row
  // tile run on neighbouring CTAs at the same time, so the second reads the tile from L2
  auto decode = [&](int64_t u, int64_t& m0, int& nb, int& kc, int64_t& kb0, int64_t& kb1) {
    nb = (int)(u % p.nblk);
    const int64_t rest = u / p.nblk;
    m0 = (rest % p.mtiles) * BM;
    kc = (int)(rest / p.mtiles);
    kb0 = p.kblocks * kc / p.nch;
    kb1 = p.kblocks * (kc + 1) / p.nch;
  };

  if (warp == 0 || warp == 2) {
    // ===== TMA producers: warp 0 the sample digits, warp 2 the thin-operand digits =====
    if (lane == 0) {
      const bool A = warp == 0;
      if (A) prefetch_tmap(&tmA);
      uint32_t g = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t m0, kb0, kb1;
        int nb, kc;
        decode(u, m0, nb, kc, kb0, kb1);
        for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
          const int k0 = (int)(kb * PBK);
          if (A) {
            const int s = g % PSTAGES;
            mbar_sleep_wait(&aempty[s], ((g / PSTAGES) & 1) ^ 1);
            if (p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks) g_oz_trace[5][g] = clock64();
            if ((p.debug & 7) == 5) {  // profiling: no sample-digit traffic
              mbar_arrive(&afull[s]);
              continue;
            }
            mbar_arrive_expect_tx(&afull[s], NDS * BM * PBK);
            // 128-byte rows over the pre-swizzled planes, no TMA swizzle
            if (RM)  // [7][128 n][32 p]: one 4 KB run per plane
              tma_load_4d(a_dig(s), &tmA, 0, (int)(m0 / 4), (int)kb, 0, &afull[s]);
            else     // [7][4 p-blocks][32 n][32 p]: four 1 KB runs per plane
              tma_load_4d(a_dig(s), &tmA, 0, k0 / 4, (int)(m0 / 32), 0, &afull[s]);
          } else {
            const int b = g % PBSTAGES;
            mbar_sleep_wait(&bempty[b], ((g / PBSTAGES) & 1) ^ 1);
            if (p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks) g_oz_trace[6][g] = clock64();
            if ((p.debug & 7) == 6) {  // profiling: no thin-digit traffic
              mbar_arrive(&bfull[b]);
              continue;
            }
            constexpr uint32_t bbytes = thin_rows(levels<NDS>()) * PBK;
            mbar_arrive_expect_tx(&bfull[b], bbytes);
            bulk_load(b_dig(b), p.bd + (nb * p.kblocks + kb) * (int64_t)PB_DIG, bbytes, &bfull[b]);
          }
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ===== MMA issuers taking alternate K-blocks (see ozaki_gemm_kernel) =====
    const int me = warp == 1 ? 0 : 1;
    int64_t total = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int64_t m0, kb0, kb1;
      int nb, kc;
      decode(u, m0, nb, kc, kb0, kb1);
      total += kb1 - kb0;
    }
    const uint32_t amajor = RM ? 0u : (1u << 15);
    auto adesc_of = [&](uint32_t addr) {
      return RM ? smem_desc_sw32(addr) : smem_desc_mn_sw32(addr);
    };
    uint32_t g = 0, t = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++t) {
      int64_t m0, kb0, kb1;
      int nb, kc;
      decode(u, m0, nb, kc, kb0, kb1);
      mbar_sleep_wait(tempty, (t & 1) ^ 1);  // every phase, in order (see ozaki_gemm_kernel)
      for (int64_t kb = kb0; kb < kb1; ++kb, ++g) {
        if ((int)(g & 1) != me) continue;
        const int s = g % PSTAGES, bs = g % PBSTAGES;
        const bool tr = p.debug >= 8 && blockIdx.x == 0 && g < kTraceBlocks && lane == 0;
        if (tr) g_oz_trace[0][g] = clock64();
        mbar_sleep_wait(&bfull[bs], (g / PBSTAGES) & 1);
        if (tr) g_oz_trace[1][g] = clock64();
        mbar_sleep_wait(&afull[s], (g / PSTAGES) & 1);
        if (tr) g_oz_trace[2][g] = clock64();
        if (g > 0) asm volatile("bar.sync %0, 64;\n" ::"r"(1 + me) : "memory");  // token in
        if (tr) g_oz_trace[3][g] = clock64();
        tc_fence_after();
        if (lane == 0 && (p.debug & 7) == 7) {  // profiling: no MMAs
          mma_commit(&aempty[s]);
          mma_commit(&bempty[bs]);
          if (kb + 1 == kb1) mma_commit(tfull);
        } else if (lane == 0) {
          // two MMA-K steps per stage: K-major operands advance 32 bytes inside the 64-byte
          // swizzled rows; the MN-major sample digits advance 32 rows (4 KB)
#pragma unroll
          for (int kk = 0; kk < PBK / 32; ++kk) {
            const uint32_t abase = smem_u32(a_dig(s));
            const uint32_t bbase = smem_u32(b_dig(bs)) + 32u * kk;
            const uint32_t first = (kb == kb0 && kk == 0) ? 0u : 1u;
            auto bdesc = [&](int row) {
              return PBK == 64 ? smem_desc_sw64(bbase + row * PBK) : smem_desc_sw32(bbase + row * PBK);
            };
            issue_pairs<NDS>(tmem, [&](int a) { return adesc_of(abase + a * BM * PBK); }, bdesc,
                             amajor, first);
          }
          mma_commit(&aempty[s]);
          mma_commit(&bempty[bs]);
          if (kb + 1 == kb1) mma_commit(tfull);
        } else if (lane == 0) {
          // two MMA-K steps per stage: K-major operands advance 32 bytes inside the 64-byte
          // swizzled rows; the MN-major sample digits advance 32 rows (4 KB)
#pragma unroll
          for (int kk = 0; kk < PBK / 32; ++kk) {
            const uint32_t abase = smem_u32(a_dig(s));
            const uint32_t bbase = smem_u32(b_dig(bs)) + 32u * kk;
            const uint32_t first = (kb == kb0 && kk == 0) ? 0u : 1u;
            auto bdesc = [&](int row) {
              return PBK == 64 ? smem_desc_sw64(bbase + row * PBK) : smem_desc_sw32(bbase + row * PBK);
            };
            const uint64_t ad1 = adesc_of(abase + 1 * BM * PBK);
            const uint64_t ad0 = adesc_of(abase);
            mma_i8(tmem + 64, ad1, bdesc(0), idesc_i8(256) | amajor, first);
            mma_i8(tmem + 320, ad1, bdesc(256), idesc_i8(192) | amajor, first);
            mma_i8(tmem + 0, ad0, bdesc(0), idesc_i8(64) | amajor, first);
            mma_i8(tmem + 64, ad0, bdesc(64), idesc_i8(256) | amajor, 1u);
            mma_i8(tmem + 320, ad0, bdesc(320), idesc_i8(128) | amajor, 1u);
#pragma unroll
            for (int a = 2; a < ND; ++a) {
              const uint64_t adesc = adesc_of(abase + a * BM * PBK);
              int col = NB * a, brow = 0, left = NB * (NL - a);
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                if (left > 0) {
                  const int n = left > 256 ? 256 : left;
                  mma_i8(tmem + col, adesc, bdesc(brow), idesc_i8(n) | amajor, 1u);
                  col += n;
                  brow += n;
                  left -= n;
                }
              }
            }
          }
          mma_commit(&aempty[s]);
          mma_commit(&bempty[bs]);
          if (kb + 1 == kb1) mma_commit(tfull);
          if (tr) g_oz_trace[4][g] = clock64();
        }
        __syncwarp();
        if ((int64_t)g + 1 < total) asm volatile("bar.arrive %0, 64;\n" ::"r"(2 - me) : "memory");
      }
    }
  } else {
    // ===== epilogue: warps 4-7, TMEM lane quadrant = warp % 4, all 64 columns =====
    const int quad = warp & 3;
    const int erow = quad * 32 + lane;
    uint32_t t = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x, ++t) {
      int64_t m0, kb0, kb1;
      int nb, kc;
      decode(u, m0, nb, kc, kb0, kb1);
      mbar_sleep_wait(tfull, t & 1);
      tc_fence_after();
      const int64_t gm = m0 + erow;
      double rowfac = 1.0;
      if (!RM && gm < p.M) rowfac = 1.0 / p.mu_inv[TABW * tab_slot(gm) + 1];
      double out[NB];
#pragma unroll
      for (int jc = 0; jc < NB / 16; ++jc) {
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
        for (int sd = 0; sd < levels<NDS>(); ++sd) {
          uint32_t r[16];
          tmem_ld16(tmem + ((uint32_t)(quad * 32) << 16) + NB * sd + 16 * jc, r);
          tmem_ld_wait();
          const double wgt = __longlong_as_double((long long)(1023 + 96 - 8 * sd) << 52);
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[j] = fma((double)(int)r[j], wgt, acc[j]);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[16 * jc + j] = acc[j];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
      if (gm < p.M) {
        const int64_t gj0 = (int64_t)nb * NB;
        const double rf = p.alpha * rowfac;
        if (p.nch > 1) {
          double* dst = p.slab + ((int64_t)kc * p.M + gm) * p.N;
#pragma unroll
          for (int j = 0; j < NB; ++j)
            if (gj0 + j < p.N) dst[gj0 + j] = rf * p.colfac[gj0 + j] * out[j];
        } else {
          double* dst = p.C + gm * p.ldc;
#pragma unroll
          for (int j = 0; j < NB; ++j)
            if (gj0 + j < p.N) {
              const double v = rf * p.colfac[gj0 + j] * out[j];
              dst[gj0 + j] = p.accumulate ? dst[gj0 + j] + v : v;
            }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem)
                 : "memory");
  }
}

// Blocked digit planes: digit a (most significant first) of X_np = rint((O_np - mu_p) 2^(54 - e_p))
// at planes[((a * ppad / 32 + p / 32) * prows + n) * 32 + (p % 32 ^ 16 [bit 2 of n])] - a K-block
// of either O-pass is then one (v pass) or four (u pass) contiguous runs per plane, stored
// pre-swizzled (32-byte swizzle) so bulk copies land in the MMA operand layout.  Parameters past
// `cols` get zero digits; rows past `rows` (up to prows) are left untouched (never used).
template <typename TA>
__global__ void __launch_bounds__(256)
    digitize_kernel(const TA* __restrict__ A, int64_t lda, int64_t rows, int64_t prows,
                    int64_t cols, int64_t ppad, const double* __restrict__ mu_inv,
                    int8_t* __restrict__ planes, int nds) {
  pdl_wait();
  const int64_t pblocks = ppad / 32;
  const int64_t plane = prows * ppad;
  const int64_t total = pblocks * rows * 8;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    // thread = (p block, row n, quad of 4 parameters): a warp writes 4 rows x 32 bytes contiguous
    const int q8 = (int)(idx & 7);
    const int64_t n = (idx >> 3) % rows, pb = (idx >> 3) / rows;
    const int64_t p0 = pb * 32 + 4 * q8;
    uint64_t y[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t pp = p0 + i;
      y[i] = kBias;
      if (pp < cols) {
        const double* t = mu_inv + TABW * tab_slot(pp);
        y[i] = biased_digits(A[n * lda + pp], as_u64(t[0]), t[1], t[2]);
      }
    }
    const uint32_t l0 = (uint32_t)y[0], l1 = (uint32_t)y[1], l2 = (uint32_t)y[2], l3 = (uint32_t)y[3];
    const uint32_t h0 = (uint32_t)(y[0] >> 32), h1 = (uint32_t)(y[1] >> 32);
    const uint32_t h2 = (uint32_t)(y[2] >> 32), h3 = (uint32_t)(y[3] >> 32);
    uint32_t u0 = __byte_perm(l0, l1, 0x5140), u1 = __byte_perm(l0, l1, 0x7362);
    uint32_t v0 = __byte_perm(l2, l3, 0x5140), v1 = __byte_perm(l2, l3, 0x7362);
    uint32_t w[ND];
    w[6] = __byte_perm(u0, v0, 0x5410) ^ 0x80808080u;
    w[5] = __byte_perm(u0, v0, 0x7632) ^ 0x80808080u;
    w[4] = __byte_perm(u1, v1, 0x5410) ^ 0x80808080u;
    w[3] = __byte_perm(u1, v1, 0x7632) ^ 0x80808080u;
    u0 = __byte_perm(h0, h1, 0x5140);
    u1 = __byte_perm(h0, h1, 0x7362);
    v0 = __byte_perm(h2, h3, 0x5140);
    v1 = __byte_perm(h2, h3, 0x7362);
    w[2] = __byte_perm(u0, v0, 0x5410) ^ 0x80808080u;
    w[1] = __byte_perm(u0, v0, 0x7632) ^ 0x80808080u;
    w[0] = __byte_perm(u1, v1, 0x5410) ^ 0x80808080u;
    int8_t* dst = planes + (pb * prows + n) * 32 + ((4 * q8) ^ (((n >> 2) & 1) << 4));
#pragma unroll
    for (int a = 0; a < ND; ++a)
      if (a < nds) *reinterpret_cast<uint32_t*>(dst + a * plane) = w[a];
  }
}

// ---- precision guard ------------------------------------------------------------------------
// The digits represent every element to 2^-54 of its parameter column's scale.  A sample row whose
// elements sit far below their columns' scales (heavy-tailed rows: a few samples dominate the
// column maxima) keeps fewer bits, so its v = Ohat^T q entries lose precision relative to
// themselves (normwise they stay FP64-grade).  rowcnt[n] packs, over the row's parameters, the
// number of nonzero digit integers (low word) and of those within kGuardBits bits of full scale
// (high word).  A row with fewer than 1/64 of its nonzero elements within kGuardBits bits of
// their columns' scales sets *flag, and the engine re-runs the step's SSI on the FP64 DMMA path
// (engine.cu with_fallback).  Gaussian samples keep > 99.9% of their elements within 12 bits;
// all-zero rows carry no information and are exempt.
__global__ void row_guard_kernel(const unsigned long long* __restrict__ rowcnt, int64_t rows,
                                 int* __restrict__ flag) {
  pdl_wait();
  bool bad = false;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < rows;
       n += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = rowcnt[n];
    const uint64_t nonzero = v & 0xffffffffull, big = v >> 32;
    bad |= nonzero != 0 && 64 * big < nonzero;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// rowcnt from the sample block itself (one read of O): used when the step's first O-pass is not
// a digitising v pass.  CTAs over rows, threads over parameters.
template <typename TA>
__global__ void __launch_bounds__(256)
    row_headroom_kernel(const TA* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                        const double* __restrict__ mu_inv, unsigned long long* __restrict__ rowcnt) {
  pdl_wait();
  for (int64_t n = blockIdx.x; n < rows; n += gridDim.x) {
    uint64_t acc = 0;
    for (int64_t pp = threadIdx.x; pp < cols; pp += blockDim.x) {
      const double* t = mu_inv + TABW * tab_slot(pp);
      acc += guard_count(biased_digits(A[n * lda + pp], as_u64(t[0]), t[1], t[2]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(rowcnt + n, (unsigned long long)acc);
  }
}

// ---- column scales of the centred sample block -------------------------------------------------
// max_n |fl(O_np - mu_p)| per parameter column p, as the bit pattern of a nonnegative double
// (order-preserving as an unsigned integer, so atomicMax is exact and order-independent).
template <typename TA, bool RM>
__global__ void __launch_bounds__(256)
    colmax_kernel(const TA* __restrict__ A, int64_t lda, int64_t rows, int64_t cols,
                  const double* __restrict__ mu, unsigned long long* __restrict__ out) {
  pdl_wait();
  // element (sample n, parameter p) at A[n * lda + p] in both layouts (row-major sample block)
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= cols) return;
  const double m = mu ? mu[p] : 0.0;
  const int64_t r0 = rows * blockIdx.y / gridDim.y, r1 = rows * (blockIdx.y + 1) / gridDim.y;
  double best = 0.0;
  int64_t n = r0;
  for (; n + 4 <= r1; n += 4) {
    const double a0 = fabs((double)A[n * lda + p] - m);
    const double a1 = fabs((double)A[(n + 1) * lda + p] - m);
    const double a2 = fabs((double)A[(n + 2) * lda + p] - m);
    const double a3 = fabs((double)A[(n + 3) * lda + p] - m);
    best = fmax(best, fmax(fmax(a0, a1), fmax(a2, a3)));
  }
  for (; n < r1; ++n) best = fmax(best, fabs((double)A[n * lda + p] - m));
  if (best > 0.0) atomicMax(out + p, (unsigned long long)__double_as_longlong(best));
}

// Columns below 2^-968 keep the scale 2^1022 (the largest finite power of two): their digits then
// resolve 2^-1022 absolutely, the FP64 normal range, instead of the factor overflowing.
constexpr int kMinScaleExp = -968;

// centring word of a slot (see biased_digits)
__device__ __forceinline__ uint64_t centre_word(double m, double s, int e) {
  if (fabs(m) < ldexp(1.0, e + 1)) return kBias - (uint64_t)__double2ll_rn(m * s);
  return kCwExact;
}
// Called by every lane of a warp for 32 consecutive parameters (one slot block): the block's
// Sterbenz flag is a warp vote.
__device__ __forceinline__ void write_slot(double* tab, int64_t p, uint64_t cw, double s, double m) {
  const bool blk = __any_sync(0xffffffffu, cw == kCwExact);
  double* t = tab + TABW * tab_slot(p);
  t[0] = __longlong_as_double((long long)cw);
  t[1] = s;
  t[2] = m;
  t[3] = __longlong_as_double(blk ? 1ll : 0ll);
}

// mu_inv[p] = {cw_p, 2^(54 - e_p), mu_p, 0} with max_p < 2^e_p; padding columns {kBias, 0, 0, 0}.
__global__ void mu_inv_kernel(const unsigned long long* __restrict__ cmax,
                              const double* __restrict__ mu, int64_t cols, int64_t cols_pad,
                              double* __restrict__ mu_inv) {
  pdl_wait();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < cols_pad;
       p += (int64_t)gridDim.x * blockDim.x) {
    double m = 0.0, inv = 0.0;
    uint64_t cw = kBias;
    if (p < cols) {
      m = mu ? mu[p] : 0.0;
      int e = 0;
      frexp(__longlong_as_double((long long)cmax[p]), &e);  // max < 2^e (0 -> e = 0)
      e = max(e, kMinScaleExp);
      inv = ldexp(1.0, 54 - e);
      cw = centre_word(m, inv, e);
    }
    write_slot(mu_inv, p, cw, inv, m);
  }
}

// Same table from column extrema: max_n |fl(O_np - mu_p)| = max(|fl(max_p - mu_p)|,
// |fl(min_p - mu_p)|) exactly, since rounding is monotone.
__global__ void mu_inv_minmax_kernel(const double* __restrict__ cmin,
                                     const double* __restrict__ cmax,
                                     const double* __restrict__ mu, int64_t cols, int64_t cols_pad,
                                     double* __restrict__ mu_inv) {
  pdl_wait();
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < cols_pad;
       p += (int64_t)gridDim.x * blockDim.x) {
    double m = 0.0, inv = 0.0;
    uint64_t cw = kBias;
    if (p < cols) {
      m = mu ? mu[p] : 0.0;
      const double big = fmax(fabs(cmax[p] - m), fabs(cmin[p] - m));
      int e = 0;
      frexp(isfinite(big) ? big : 0.0, &e);
      e = max(e, kMinScaleExp);
      inv = ldexp(1.0, 54 - e);
      cw = centre_word(m, inv, e);
    }
    write_slot(mu_inv, p, cw, inv, m);
  }
}

// ---- thin operand: column maxima and digits ---------------------------------------------------
// w_kj = B_kj * rowmul_k (rowmul_k = 2^e_k = 2^54 / inv_k of the K-side parameter column, or 1)
__device__ __forceinline__ double thin_value(const double* B, int64_t ldb, int64_t k, int64_t j,
                                             const double* mu_inv) {
  const double b = B[k * ldb + j];
  if (!mu_inv) return b;
  // 2^54 / inv exactly, from the exponent field of the power of two inv (no division)
  const long long ebits = __double_as_longlong(mu_inv[TABW * tab_slot(k) + 1]) >> 52;
  return b * __longlong_as_double((long long)(2046 + 54 - ebits) << 52);
}

// Thread layout of both thin-operand kernels: block = 64 columns x 4 groups of 4 consecutive K
// rows (16 rows per pass), lane-fast over the K groups so each warp reads 8 rows x 4 columns
// (full 32-byte sectors) and writes 4 rows x 8 K-groups of 4-byte digit words (full sectors).
__global__ void __launch_bounds__(256)
    thin_colmax_kernel(const double* __restrict__ B, int64_t ldb, int64_t K, int64_t N,
                       const double* __restrict__ mu_inv, unsigned long long* __restrict__ out) {
  pdl_wait();
  // block: 64 columns of one 64-column block x 4 row lanes, 128 rows; 8 independent rows in
  // flight per thread
  const int j = threadIdx.x & 63, kl = threadIdx.x >> 6;
  const int64_t jj = (int64_t)blockIdx.y * 64 + j;
  double best = 0.0;
  if (jj < N) {
    const int64_t k0 = (int64_t)blockIdx.x * 128 + kl;
#pragma unroll
    for (int u = 0; u < 32; u += 8) {
      double v[8], mul[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t k = k0 + 4 * (u + i);
        v[i] = 0.0;
        mul[i] = 1.0;
        if (k < K) {
          v[i] = __ldg(B + k * ldb + jj);
          if (mu_inv) {
            const double inv = __ldg(mu_inv + TABW * tab_slot(k) + 1);
            // 2^54 / inv from the exponent field (0 for padding columns: inv == 0)
            mul[i] = inv == 0.0 ? 0.0
                                : __longlong_as_double(
                                      (long long)(2046 + 54 - (__double_as_longlong(inv) >> 52))
                                      << 52);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) best = fmax(best, fabs(v[i] * mul[i]));
    }
  }
  __shared__ double red[4][64];
  red[kl][j] = best;
  __syncthreads();
  if (kl == 0 && jj < N) {
    best = fmax(fmax(red[0][j], red[1][j]), fmax(red[2][j], red[3][j]));
    if (best > 0.0) atomicMax(out + jj, (unsigned long long)__double_as_longlong(best));
  }
}

// digits, blocked by 32 K: Bd[nb][k / 32][a * 64 + j][k % 32] (every K-block's 448 x 32-byte
// tile is one contiguous 14 KB run), stored pre-swizzled (32-byte swizzle: the 16-byte half of
// row r is flipped when bit 2 of r is set) so a plain bulk copy lands in the MMA layout;
// colfac[nb*64 + jj]
__global__ void __launch_bounds__(256)
    thin_digits_kernel(const double* __restrict__ B, int64_t ldb, int64_t K, int64_t N,
                       int64_t kpad, const double* __restrict__ mu_inv,
                       const unsigned long long* __restrict__ cmax, int extra_exp,
                       int8_t* __restrict__ Bd, double* __restrict__ colfac, int tlay) {
  pdl_wait();
  // thread: column jl (of 32) and K group kg (of 8, 4 rows each); block covers 32 K x 32 columns
  const int kg = threadIdx.x & 7, jl = threadIdx.x >> 3;
  const int nb = blockIdx.y >> 1;
  const int j = (blockIdx.y & 1) * 32 + jl;
  const int64_t jj = (int64_t)nb * 64 + j;
  const int64_t k0 = (int64_t)blockIdx.x * 32 + 4 * kg;
  double inv = 0.0;
  if (jj < N) {
    int e = 0;
    frexp(__longlong_as_double((long long)cmax[jj]), &e);
    e = max(e, kMinScaleExp);
    inv = ldexp(1.0, 54 - e);
    if (blockIdx.x == 0 && kg == 0) colfac[jj] = ldexp(1.0, e - 54 - extra_exp);
  } else if (blockIdx.x == 0 && kg == 0) {
    colfac[jj] = 0.0;
  }
  uint64_t y[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t k = k0 + i;
    double x = 0.0;
    if (jj < N && k < K && !(mu_inv && mu_inv[TABW * tab_slot(k) + 1] == 0.0))
      x = thin_value(B, ldb, k, jj, mu_inv) * inv;
    y[i] = to_biased(x);
  }
  uint32_t w[ND];
  {
    const uint32_t l0 = (uint32_t)y[0], l1 = (uint32_t)y[1], l2 = (uint32_t)y[2], l3 = (uint32_t)y[3];
    const uint32_t h0 = (uint32_t)(y[0] >> 32), h1 = (uint32_t)(y[1] >> 32);
    const uint32_t h2 = (uint32_t)(y[2] >> 32), h3 = (uint32_t)(y[3] >> 32);
    uint32_t u0 = __byte_perm(l0, l1, 0x5140), u1 = __byte_perm(l0, l1, 0x7362);
    uint32_t v0 = __byte_perm(l2, l3, 0x5140), v1 = __byte_perm(l2, l3, 0x7362);
    w[6] = __byte_perm(u0, v0, 0x5410) ^ 0x80808080u;
    w[5] = __byte_perm(u0, v0, 0x7632) ^ 0x80808080u;
    w[4] = __byte_perm(u1, v1, 0x5410) ^ 0x80808080u;
    w[3] = __byte_perm(u1, v1, 0x7632) ^ 0x80808080u;
    u0 = __byte_perm(h0, h1, 0x5140);
    u1 = __byte_perm(h0, h1, 0x7362);
    v0 = __byte_perm(h2, h3, 0x5140);
    v1 = __byte_perm(h2, h3, 0x7362);
    w[2] = __byte_perm(u0, v0, 0x5410) ^ 0x80808080u;
    w[1] = __byte_perm(u0, v0, 0x7632) ^ 0x80808080u;
    w[0] = __byte_perm(u1, v1, 0x5410) ^ 0x80808080u;
  }
  if (tlay) {  // [K-block][digit][128 columns][32]: the A operand of ozaki_gemm_t_kernel
#pragma unroll
    for (int a = 0; a < ND; ++a)
      *reinterpret_cast<uint32_t*>(
          Bd + (((int64_t)blockIdx.x * ND + a) * 128 + nb * 64 + j) * 32 +
          ((4 * kg) ^ (((j >> 2) & 1) << 4))) = w[a];
    return;
  }
#pragma unroll
  for (int a = 0; a < ND; ++a)
    *reinterpret_cast<uint32_t*>(
        Bd + (((int64_t)nb * (kpad / 32) + blockIdx.x) * BROWS + a * 64 + j) * 32 +
        ((4 * kg) ^ ((((a * 64 + j) >> 2) & 1) << 4))) = w[a];
}

// (K x M) row-major sample block, box = 128 parameters x 32 samples, no swizzle
bool make_map_cm(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t pitch,
                 int esize, int box_inner = BM) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)(pitch * esize)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)BK};
  cuuint32_t es[2] = {1u, 1u};
  return fn(map, esize == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
            const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool RM, typename TA, int NDS>
cudaError_t launch_nds(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tS,
                       const Params& p, int grid, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  cudaError_t e = smem_attr_once(attr, ozaki_gemm_kernel<RM, TA, NDS>, (int)kSmem);
  if (e != cudaSuccess) return e;
  launch_pdl(ozaki_gemm_kernel<RM, TA, NDS>, grid, kThreads, kSmem, st, tA, tB, tS, p);
  return cudaGetLastError();
}
template <bool RM, typename TA>
cudaError_t launch(const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tS,
                   const Params& p, int grid, cudaStream_t st) {
  if (sizeof(TA) == 4 && p.nds == 5) return launch_nds<RM, TA, 5>(tA, tB, tS, p, grid, st);
  return launch_nds<RM, TA, ND>(tA, tB, tS, p, grid, st);
}

template <bool RM, int NDS>
cudaError_t launch_pre_nds(const CUtensorMap& tA, const Params& p, int grid, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  cudaError_t e = smem_attr_once(attr, ozaki_pre_kernel<RM, NDS>, (int)kPreSmem);
  if (e != cudaSuccess) return e;
  launch_pdl(ozaki_pre_kernel<RM, NDS>, grid, kPreThreads, kPreSmem, st, tA, p);
  return cudaGetLastError();
}
template <bool RM, typename TA, int NDS>
cudaError_t launch_t_nds(const CUtensorMap& tA, const CUtensorMap& tS, const Params& p, int grid,
                         cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  cudaError_t e = smem_attr_once(attr, ozaki_gemm_t_kernel<RM, TA, NDS>, (int)kTSmem);
  if (e != cudaSuccess) return e;
  launch_pdl(ozaki_gemm_t_kernel<RM, TA, NDS>, grid, kThreads, kTSmem, st, tA, tS, p);
  return cudaGetLastError();
}
template <bool RM, typename TA>
cudaError_t launch_t(const CUtensorMap& tA, const CUtensorMap& tS, const Params& p, int grid,
                     cudaStream_t st) {
  if (sizeof(TA) == 4 && p.nds == 5) return launch_t_nds<RM, TA, 5>(tA, tS, p, grid, st);
  return launch_t_nds<RM, TA, ND>(tA, tS, p, grid, st);
}

template <bool RM>
cudaError_t launch_pre(const CUtensorMap& tA, const Params& p, int grid, cudaStream_t st) {
  return p.nds == 5 ? launch_pre_nds<RM, 5>(tA, p, grid, st)
                    : launch_pre_nds<RM, ND>(tA, p, grid, st);
}

// 4-D map over the blocked, pre-swizzled digit planes viewed as 128-byte rows:
// {128 B (4 sample rows), prows / 4, ppad / 32 parameter blocks, 7 planes}, no TMA swizzle
bool make_map_planes(CUtensorMap* map, const int8_t* planes, int64_t prows, int64_t pblocks,
                     bool rm, int nds) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)(prows / 4), (cuuint64_t)pblocks, (cuuint64_t)nds};
  cuuint64_t strides[3] = {128, (cuuint64_t)(32 * prows), (cuuint64_t)(32 * prows * pblocks)};
  cuuint32_t box[4] = {128, rm ? 32u : 8u, rm ? 1u : 4u, (cuuint32_t)nds};
  cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(planes), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace oz

int ozaki_digit_pairs() {
  int pairs = 0;
  for (int a = 0; a < oz::ND; ++a)
    for (int b = 0; b < oz::ND; ++b) pairs += a + b < oz::NL ? 1 : 0;
  return pairs;
}

// ---- host side ---------------------------------------------------------------------------------
cudaError_t ozaki_trace(long long* host, size_t n) {
  return cudaMemcpyFromSymbol(host, oz::g_oz_trace, std::min(n, sizeof(oz::g_oz_trace)));
}

int64_t ozaki_scale_len(int64_t cols) { return ((cols + oz::BK - 1) / oz::BK) * oz::BK; }
int64_t ozaki_table_doubles(int64_t cols) { return oz::TABW * ozaki_scale_len(cols); }

cudaError_t ozaki_table_clear(Context& ctx, double* mu_inv, int64_t cols, cudaStream_t st) {
  const int64_t cpad = ozaki_scale_len(cols);
  launch_pdl(oz::mu_inv_kernel, (int)std::max<int64_t>(1, std::min<int64_t>((cpad + 255) / 256, 4 * ctx.num_sms)), 256, 0, st,
             (const unsigned long long*)nullptr, (const double*)nullptr, (int64_t)0, cpad, mu_inv);
  ctx.kernel_launches += 1;
  return cudaGetLastError();
}

cudaError_t ozaki_scales(Context& ctx, const void* A, bool f32, int64_t lda, int64_t rows,
                         int64_t cols, const double* mu, double* mu_inv, cudaStream_t st) {
  const int64_t cpad = ozaki_scale_len(cols);
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(ctx.splitk_buffer(cols));
  if (!cmax) return cudaErrorMemoryAllocation;
  cudaError_t e = cudaMemsetAsync(cmax, 0, sizeof(double) * cols, st);
  if (e != cudaSuccess) return e;
  const int gx = (int)((cols + 255) / 256);
  const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(rows / 64, (8 * ctx.num_sms + gx - 1) / gx));
  if (f32)
    launch_pdl(oz::colmax_kernel<float, true>, dim3(gx, gy), 256, 0, st, 
        static_cast<const float*>(A), lda, rows, cols, mu, cmax);
  else
    launch_pdl(oz::colmax_kernel<double, true>, dim3(gx, gy), 256, 0, st, 
        static_cast<const double*>(A), lda, rows, cols, mu, cmax);
  launch_pdl(oz::mu_inv_kernel, (int)std::min<int64_t>((cpad + 255) / 256, 4 * ctx.num_sms), 256, 0, st, 
      cmax, mu, cols, cpad, mu_inv);
  ctx.kernel_launches += 2;
  return cudaGetLastError();
}

cudaError_t ozaki_scales_minmax(Context& ctx, const double* cmin, const double* cmax,
                                const double* mu, int64_t cols, double* mu_inv, cudaStream_t st) {
  const int64_t cpad = ozaki_scale_len(cols);
  launch_pdl(oz::mu_inv_minmax_kernel, (int)std::min<int64_t>((cpad + 255) / 256, 4 * ctx.num_sms), 256, 0, st, cmin, cmax, mu, cols, cpad, mu_inv);
  ctx.kernel_launches += 1;
  return cudaGetLastError();
}

bool ozaki_supported(Layout L, const GemmArgs& a, bool f32) {
  const size_t es = f32 ? 4 : 8;
  return tma_encode_fn() != nullptr && (reinterpret_cast<uintptr_t>(a.A) % 16 == 0) &&
         ((a.lda * es) % 16 == 0) && a.M < (1LL << 31) && a.K < (1LL << 31) &&
         a.N <= 4096 && !a.partial && !a.Cin && (L == Layout::RM || L == Layout::CM);
}

int64_t ozaki_plane_pitch(int64_t cols) { return ((cols + 127) / 128) * 128; }
int64_t ozaki_plane_rows(int64_t rows) { return ((rows + 127) / 128) * 128; }
size_t ozaki_planes_bytes(int64_t rows, int64_t cols, int nds) {
  return (size_t)nds * ozaki_plane_rows(rows) * ozaki_plane_pitch(cols);
}

cudaError_t ozaki_digitize(Context& ctx, const void* A, bool f32, int64_t lda, int64_t rows,
                           int64_t cols, const double* mu_inv, int8_t* planes, cudaStream_t st,
                           int nds) {
  const int64_t ppad = ozaki_plane_pitch(cols), prows = ozaki_plane_rows(rows);
  const int64_t work = rows * (ppad / 4);  // threads: one per 4 parameters of a row
  const int grid = (int)std::min<int64_t>((work + 255) / 256, 16 * ctx.num_sms);
  if (f32)
    launch_pdl(oz::digitize_kernel<float>, grid, 256, 0, st, static_cast<const float*>(A), lda, rows,
                                                     prows, cols, ppad, mu_inv, planes, nds);
  else
    launch_pdl(oz::digitize_kernel<double>, grid, 256, 0, st, static_cast<const double*>(A), lda, rows,
                                                      prows, cols, ppad, mu_inv, planes, nds);
  ctx.kernel_launches += 1;
  return cudaGetLastError();
}

cudaError_t ozaki_row_headroom(Context& ctx, const void* A, bool f32, int64_t lda, int64_t rows,
                               int64_t cols, const double* mu_inv, unsigned long long* rowcnt,
                               cudaStream_t st) {
  const int grid = (int)std::min<int64_t>(std::max<int64_t>(rows, 1), 8 * ctx.num_sms);
  if (f32)
    launch_pdl(oz::row_headroom_kernel<float>, grid, 256, 0, st, static_cast<const float*>(A), lda,
               rows, cols, mu_inv, rowcnt);
  else
    launch_pdl(oz::row_headroom_kernel<double>, grid, 256, 0, st, static_cast<const double*>(A),
               lda, rows, cols, mu_inv, rowcnt);
  ctx.kernel_launches += 1;
  return cudaGetLastError();
}

cudaError_t ozaki_row_guard(Context& ctx, const unsigned long long* rowcnt, int64_t rows,
                            int* flag, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((rows + 255) / 256, ctx.num_sms);
  launch_pdl(oz::row_guard_kernel, std::max(grid, 1), 256, 0, st, rowcnt, rows, flag);
  ctx.kernel_launches += 1;
  return cudaGetLastError();
}

cudaError_t ozaki_gemm(Context& ctx, Layout L, const GemmArgs& a, bool f32, const double* mu_inv,
                       cudaStream_t st, const int8_t* planes, int8_t* store,
                       unsigned long long* rowcnt, int nds) {
  if (nds != 5 && nds != oz::ND) return cudaErrorInvalidValue;
  using namespace oz;
  const bool RMm = L == Layout::RM;
  const int64_t M = a.M, N = a.N, K = a.K;
  if (M == 0 || N == 0) return cudaSuccess;
  const int nblk = (int)((N + NB - 1) / NB);
  const int kstep = planes ? PBK : BK;  // K per pipeline stage
  const int64_t kpad = ((K + kstep - 1) / kstep) * kstep;
  const int64_t kblocks = kpad / kstep;
  // the transposed on-the-fly kernel: 65-128 thin columns, digits not yet in HBM
  // (WSSR_OZ_TKERNEL=0 falls back to one 64-column block per unit for both passes, =1 keeps it
  // for the row-major pass only)
  static const int t_mode = [] {
    const char* e = std::getenv("WSSR_OZ_TKERNEL");
    return e ? std::atoi(e) : 2;
  }();
  const bool tkern = !planes && nblk == 2 && (RMm ? t_mode >= 1 : t_mode >= 2);
  const int mtiles = tkern ? (int)((M + TBM - 1) / TBM) : (int)((M + BM - 1) / BM);
  // thin-operand digits + factors (workspace owned by the context)
  const size_t dig_bytes = (size_t)nblk * BROWS * kpad;
  const size_t ws_doubles = (dig_bytes + 7) / 8 + (size_t)nblk * NB + N + 64;
  if (ctx.oz_ws_cap < ws_doubles) {
    if (ctx.oz_ws) cudaFreeAsync(ctx.oz_ws, st);
    ctx.oz_ws = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ctx.oz_ws), ws_doubles * 8, st);
    if (e != cudaSuccess) return e;
    ctx.oz_ws_cap = ws_doubles;
  }
  int8_t* Bd = reinterpret_cast<int8_t*>(ctx.oz_ws);
  double* colfac = ctx.oz_ws + (dig_bytes + 7) / 8;
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(colfac + (size_t)nblk * NB);
  cudaError_t e = cudaMemsetAsync(cmax, 0, sizeof(double) * N, st);
  if (e != cudaSuccess) return e;
  // RM (v = Ohat^T q): the thin operand's rows are parameters -> carries the column scales
  const double* bmu = RMm ? mu_inv : nullptr;
  {
    launch_pdl(thin_colmax_kernel, dim3((unsigned)((K + 127) / 128), nblk), 256, 0, st, a.B, a.ldb, K, N,
                                                                               bmu, cmax);
    launch_pdl(thin_digits_kernel, dim3((unsigned)(kpad / 32), 2 * nblk), 256, 0, st, 
        a.B, a.ldb, K, N, kpad, bmu, cmax, RMm ? 54 : 0, Bd, colfac, tkern ? 1 : 0);
    ctx.kernel_launches += 2;
  }
  // K chunks: int32 bound, then enough units to fill the machine evenly
  int nch = (int)((kpad + KCHUNK - 1) / KCHUNK);
  {
    const int64_t base = (int64_t)mtiles * (tkern ? 1 : nblk);
    int best = nch;
    double best_eff = 0.0;
    for (int c = nch; c <= std::max(nch, 64); ++c) {
      if ((int64_t)c > kblocks) break;
      const int64_t units = base * c;
      const int64_t waves = (units + ctx.num_sms - 1) / ctx.num_sms;
      const double eff = (double)units / ((double)waves * ctx.num_sms);
      if (eff > best_eff + 0.02) {
        best_eff = eff;
        best = c;
      }
      if (eff >= 0.92 && units >= ctx.num_sms) break;
    }
    nch = best;
    static const int force_nch = [] {
      const char* e = std::getenv("WSSR_OZ_NCH");  // profiling / debugging only
      return e ? std::atoi(e) : 0;
    }();
    if (force_nch > 0) nch = (int)std::min<int64_t>(std::max<int64_t>(force_nch, nch), kblocks);
  }
  Params p{};
  p.M = M;
  p.K = K;
  p.N = N;
  p.nblk = nblk;
  p.nch = nch;
  p.mtiles = mtiles;
  p.kblocks = kblocks;
  p.mu_inv = mu_inv;
  p.colfac = colfac;
  p.alpha = a.alpha;
  p.C = a.C;
  p.ldc = a.ldc;
  p.accumulate = a.accumulate;
  p.slab = nullptr;
  p.bd = Bd;
  if (nds == 5 && !f32) nds = oz::ND;  // the 5-digit scheme is for float32 samples only
  p.nds = nds;
  p.nl = nds == oz::ND ? oz::NL : nds + 1;
  p.planes = planes;
  p.store = (!planes && RMm) ? store : nullptr;
  p.rowcnt = (!planes && RMm) ? rowcnt : nullptr;
  if (planes || p.store) {
    p.prows = ozaki_plane_rows(RMm ? M : K);
    p.pblocks = ozaki_plane_pitch(RMm ? K : M) / 32;
  }
  {
    static const int dbg = [] {
      const char* e = std::getenv("WSSR_OZ_DEBUG");
      return e ? std::atoi(e) : 0;
    }();
    p.debug = dbg;
  }
  if (nch > 1) {
    p.slab = ctx.splitk_buffer((size_t)nch * M * N);
    if (!p.slab) return cudaErrorMemoryAllocation;
  }
  CUtensorMap tA, tB, tS;
  std::memset(&tS, 0, sizeof(tS));
  const int es = f32 ? 4 : 8;
  bool ok;
  if (planes) {
    if (!make_map_planes(&tA, planes, p.prows, p.pblocks, RMm, nds)) return cudaErrorInvalidValue;
    const int64_t units = (int64_t)mtiles * nblk * nch;
    const int grid = (int)std::min<int64_t>(units, ctx.num_sms);
    e = RMm ? launch_pre<true>(tA, p, grid, st) : launch_pre<false>(tA, p, grid, st);
    ctx.kernel_launches += 1;
    ctx.gemm_launches += 1;
  } else if (RMm) {
    ok = make_map_2d(&tA, a.A, K, M, a.lda, tkern ? TBM : BM, es) &&
         make_map_1d(&tS, mu_inv, TABW * kpad, TABW * BK);
  } else {
    ok = make_map_cm(&tA, a.A, M, K, a.lda, es, tkern ? TBM : BM);
  }
  if (!planes && tkern) {
    if (!ok) return cudaErrorInvalidValue;
    const int64_t units = (int64_t)mtiles * nch;
    const int grid = (int)std::min<int64_t>(units, ctx.num_sms);
    if (RMm)
      e = f32 ? launch_t<true, float>(tA, tS, p, grid, st) : launch_t<true, double>(tA, tS, p, grid, st);
    else
      e = f32 ? launch_t<false, float>(tA, tS, p, grid, st)
              : launch_t<false, double>(tA, tS, p, grid, st);
    ctx.kernel_launches += 1;
    ctx.gemm_launches += 1;
  } else if (!planes) {
    std::memset(&tB, 0, sizeof(tB));  // thin digits arrive by plain bulk copies
    if (!ok) return cudaErrorInvalidValue;
    const int64_t units = (int64_t)mtiles * nblk * nch;
    const int grid = (int)std::min<int64_t>(units, ctx.num_sms);
    if (RMm)
      e = f32 ? launch<true, float>(tA, tB, tS, p, grid, st)
              : launch<true, double>(tA, tB, tS, p, grid, st);
    else
      e = f32 ? launch<false, float>(tA, tB, tS, p, grid, st)
              : launch<false, double>(tA, tB, tS, p, grid, st);
    ctx.kernel_launches += 1;
    ctx.gemm_launches += 1;
  }
  if (e != cudaSuccess || nch == 1) return e;
  const int64_t total = M * N;
  const int rb = (int)std::min<int64_t>((total + 255) / 256, 16 * ctx.num_sms);
  if (nch <= 8)
    launch_pdl(splitk_reduce_few_kernel, rb, 256, 0, st, p.slab, nch, M, N, a.C, a.ldc, 1.0, a.accumulate,
                                                nullptr, 0);
  else
    launch_pdl(splitk_reduce_kernel, (int)std::min<int64_t>((total + 31) / 32, 16 * ctx.num_sms), 256, 0, st, p.slab, nch, M, N, a.C, a.ldc, 1.0, a.accumulate, nullptr, 0);
  ctx.kernel_launches += 1;
  return cudaGetLastError();
}

}  // namespace wssr
