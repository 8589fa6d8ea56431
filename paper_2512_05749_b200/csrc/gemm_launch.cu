// Host-side dispatch for the DMMA GEMM family: tile-config choice by output width, operand
// vector width (16-byte cp.async when rows are 16-byte aligned) and split-K sizing.
#include <cudaTypedefs.h>

#include <cstring>

#include "engine.h"
#include "gemm.cuh"
#include "gemm_tma.cuh"

namespace wssr {

// ---- TMA + mbarrier warp-specialised tiles (gemm_tma.cuh) ----------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D map over a row-major (outer x inner) FP64 array with row pitch `pitch` elements;
// box = 16 doubles (128 B, SWIZZLE_128B) x box_outer rows.
bool make_map_2d(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t pitch,
                 int box_outer, int esize = 8) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)std::max<int64_t>(pitch * esize, 16)};
  cuuint32_t box[2] = {(cuuint32_t)(128 / esize), (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1u, 1u};
  return fn(map, esize == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
            const_cast<void*>(ptr), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool make_map_1d(CUtensorMap* map, const double* ptr, int64_t n, int box) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[1] = {(cuuint64_t)n};
  cuuint64_t strides[1] = {0};
  cuuint32_t bx[1] = {(cuuint32_t)box};
  cuuint32_t es[1] = {1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, const_cast<double*>(ptr), dims, strides, bx,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

thread_local int64_t g_launches = 0;

template <Layout L, int BM, int BN, int BK, int WMW, int WNW, int ST, int VA, int VB>
cudaError_t launch_one(const GemmArgs& a, int splits, cudaStream_t st) {
  using Cfg = GemmCfg<L, BM, BN, BK, WMW, WNW, ST>;
  auto kern = gemm_dmma_kernel<L, BM, BN, BK, WMW, WNW, ST, VA, VB>;
  static std::atomic<uint64_t> attr_set{0};  // per instantiation, one bit per device
  cudaError_t e = smem_attr_once(attr_set, kern, (int)Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)((a.M + BM - 1) / BM), (unsigned)((a.N + BN - 1) / BN), (unsigned)splits);
  launch_pdl(kern, grid, Cfg::kThreads, Cfg::kSmemBytes, st, a);
  ++g_launches;
  return cudaGetLastError();
}

template <Layout L, int BM, int BN, int BK, int WMW, int WNW, int ST>
struct Tile {
  static constexpr int kBM = BM, kBN = BN, kBK = BK;
  using Cfg = GemmCfg<L, BM, BN, BK, WMW, WNW, ST>;
  static cudaError_t launch(const GemmArgs& a, int splits, bool va2, bool vb2, cudaStream_t st) {
    if (va2 && vb2) return launch_one<L, BM, BN, BK, WMW, WNW, ST, 2, 2>(a, splits, st);
    if (va2) return launch_one<L, BM, BN, BK, WMW, WNW, ST, 2, 1>(a, splits, st);
    if (vb2) return launch_one<L, BM, BN, BK, WMW, WNW, ST, 1, 2>(a, splits, st);
    return launch_one<L, BM, BN, BK, WMW, WNW, ST, 1, 1>(a, splits, st);
  }
  static int ctas_per_sm() {
    static int occ = -1;
    if (occ < 0) {
      auto kern = gemm_dmma_kernel<L, BM, BN, BK, WMW, WNW, ST, 2, 2>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)Cfg::kSmemBytes);
      int o = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Cfg::kThreads,
                                                        Cfg::kSmemBytes) != cudaSuccess)
        o = 1;
      occ = o < 1 ? 1 : o;
    }
    return occ;
  }
};

template <Layout L, int BM, int BN, int BK, int WMW, int WNW, int ST, typename TA = double,
          bool PERSIST = false>
struct TmaTile {
  static constexpr int kBM = BM, kBN = BN, kBK = BK;
  using Cfg = TmaCfg<L, BM, BN, BK, WMW, WNW, ST, TA>;
  static int num_sms() {
    static int n = 0;
    if (!n) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
      if (n < 1) n = 148;
    }
    return n;
  }
  static cudaError_t launch(const GemmArgs& a, int splits, bool, bool, cudaStream_t st) {
    auto kern = gemm_tma_kernel<L, BM, BN, BK, WMW, WNW, ST, TA, PERSIST>;
    static std::atomic<uint64_t> attr_set{0};
    cudaError_t e = smem_attr_once(attr_set, kern, (int)Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    CUtensorMap tA, tB, tS;
    std::memset(&tS, 0, sizeof(tS));
    bool ok;
    if (L == Layout::CM)
      ok = make_map_2d(&tA, a.A, a.M, a.K, a.lda, BK, (int)sizeof(TA));
    else
      ok = make_map_2d(&tA, a.A, a.K, a.M, a.lda, BM, (int)sizeof(TA));
    ok = ok && make_map_2d(&tB, a.B, a.N, a.K, a.ldb, BK);
    if (L == Layout::RM && a.shift) ok = ok && make_map_1d(&tS, a.shift, a.K, BK);
    if (!ok) return cudaErrorInvalidValue;
    if (PERSIST) {
      const int64_t units = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN) * splits;
      const int64_t cap = (int64_t)num_sms() * ctas_per_sm();
      launch_pdl(kern, (unsigned)std::min(units, cap), Cfg::kThreads, Cfg::kSmemBytes, st, tA, tB, tS, a);
    } else {
      dim3 grid((unsigned)((a.M + BM - 1) / BM), (unsigned)((a.N + BN - 1) / BN),
                (unsigned)splits);
      launch_pdl(kern, grid, Cfg::kThreads, Cfg::kSmemBytes, st, tA, tB, tS, a);
    }
    ++g_launches;
    return cudaGetLastError();
  }
  static int ctas_per_sm() {
    static int occ = -1;
    if (occ < 0) {
      auto kern = gemm_tma_kernel<L, BM, BN, BK, WMW, WNW, ST, TA, PERSIST>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)Cfg::kSmemBytes);
      int o = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Cfg::kThreads,
                                                        Cfg::kSmemBytes) != cudaSuccess)
        o = 1;
      occ = o < 1 ? 1 : o;
    }
    return occ;
  }
};

// (BM, BN, BK, warps M x N, stages) from tools/microbench/gemm_sweep on B200
using TCM32 = TmaTile<Layout::CM, 256, 32, 32, 8, 1, 2, double, true>;
using TCM64 = TmaTile<Layout::CM, 128, 64, 64, 4, 2, 2, double, true>;
using TCM128 = TmaTile<Layout::CM, 64, 128, 32, 2, 4, 3, double, true>;
using TCM256 = TmaTile<Layout::CM, 32, 256, 32, 1, 8, 2, double, true>;
using TCMsq32 = TmaTile<Layout::CM, 32, 32, 32, 1, 1, 4>;
using TCMsq64 = TmaTile<Layout::CM, 64, 64, 32, 2, 2, 4>;
using TRM32 = TmaTile<Layout::RM, 256, 32, 32, 8, 1, 2, double, true>;
using TRM64 = TmaTile<Layout::RM, 128, 64, 64, 4, 2, 2, double, true>;
using TRM128 = TmaTile<Layout::RM, 64, 128, 32, 2, 4, 3, double, true>;
using TRM256 = TmaTile<Layout::RM, 32, 256, 32, 1, 8, 2, double, true>;
// FP32 A operand (O stored as float32, BASELINE configs[3]); widened to FP64 in registers
using FCM32 = TmaTile<Layout::CM, 256, 32, 32, 8, 1, 2, float, true>;
using FCM64 = TmaTile<Layout::CM, 128, 64, 64, 4, 2, 2, float, true>;
using FCM128 = TmaTile<Layout::CM, 64, 128, 32, 2, 4, 3, float, true>;
using FCM256 = TmaTile<Layout::CM, 32, 256, 32, 1, 8, 2, float, true>;
using FRM32 = TmaTile<Layout::RM, 256, 32, 32, 8, 1, 2, float, true>;
using FRM64 = TmaTile<Layout::RM, 128, 64, 64, 4, 2, 2, float, true>;
using FRM128 = TmaTile<Layout::RM, 64, 128, 32, 2, 4, 3, float, true>;
using FRM256 = TmaTile<Layout::RM, 32, 256, 32, 1, 8, 2, float, true>;

// short contractions (K <= 256: X * R^-1, X * C, w - q * quotient): small CTAs, 3-4 resident
using TRMs64 = TmaTile<Layout::RM, 64, 64, 16, 2, 2, 4>;
using TRMs128 = TmaTile<Layout::RM, 64, 128, 32, 2, 4, 2>;

// Config table.
using CM32 = Tile<Layout::CM, 256, 32, 16, 8, 1, 4>;
using CM64 = Tile<Layout::CM, 128, 64, 16, 4, 2, 4>;
using CM128 = Tile<Layout::CM, 64, 128, 16, 2, 4, 4>;
using CM256 = Tile<Layout::CM, 32, 256, 8, 1, 8, 4>;
using CMsq32 = Tile<Layout::CM, 32, 32, 16, 1, 1, 4>;
using CMsq64 = Tile<Layout::CM, 64, 64, 16, 2, 2, 4>;
using RM32 = Tile<Layout::RM, 256, 32, 16, 8, 1, 3>;
using RM64 = Tile<Layout::RM, 128, 64, 8, 4, 2, 4>;
using RM128 = Tile<Layout::RM, 64, 128, 8, 2, 4, 4>;
using RM256 = Tile<Layout::RM, 32, 256, 16, 1, 8, 3>;

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Split-K only pays when the contraction is long and there are too few output tiles to fill
// the machine: every split adds an M x N slab of partial traffic plus a reduction.
int choose_splits(int64_t tiles, int64_t M, int64_t N, int64_t K, int BK, int capacity,
                  int max_splits) {
  if (max_splits <= 1) return 1;
  constexpr int64_t kMinChunk = 512;  // minimum K per split
  int64_t kmax = K / kMinChunk;
  int smax = (int)std::min<int64_t>(max_splits, std::max<int64_t>(1, kmax));
  if (smax <= 1 || tiles >= 8LL * capacity) return 1;
  // partial slabs must stay small next to the streamed operand
  const double slab = (double)M * N, stream = (double)M * K + (double)K * N;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= smax; ++s) {
    if (s > 1 && s * slab > 0.25 * stream) break;
    double waves = (double)(tiles * s) / capacity;
    double eff = waves / std::ceil(waves);
    if (eff >= 0.94) return s;
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
  }
  return best;
}

template <class T>
cudaError_t run_tile(Context& ctx, GemmArgs a, bool va2, bool vb2, int max_splits,
                     cudaStream_t st) {
  const int64_t tiles = ((a.M + T::kBM - 1) / T::kBM) * ((a.N + T::kBN - 1) / T::kBN);
  const int cap = ctx.num_sms * T::ctas_per_sm();
  int s = choose_splits(tiles, a.M, a.N, a.K, T::kBK, cap, max_splits);
  int64_t kc = (a.K + s - 1) / s;
  kc = ((kc + T::kBK - 1) / T::kBK) * T::kBK;
  if (kc <= 0) kc = T::kBK;
  s = (int)std::max<int64_t>(1, (a.K + kc - 1) / kc);
  a.k_chunk = kc;
  if (s == 1) {
    a.partial = nullptr;
    return T::launch(a, 1, va2, vb2, st);
  }
  const size_t need = (size_t)s * a.M * a.N;
  double* part = ctx.splitk_buffer(need);
  if (!part) return cudaErrorMemoryAllocation;
  double* C = a.C;
  const int64_t ldc = a.ldc;
  const double alpha = a.alpha;
  const int acc = a.accumulate;
  a.partial = part;
  a.alpha = 1.0;
  cudaError_t e = T::launch(a, s, va2, vb2, st);
  if (e != cudaSuccess) return e;
  const int64_t total = a.M * a.N;
  if (s <= 8) {
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 16LL * ctx.num_sms);
    launch_pdl(splitk_reduce_few_kernel, std::max(blocks, 1), 256, 0, st, part, s, a.M, a.N, C, ldc, alpha,
                                                                  acc, a.Cin, a.ldcin);
  } else {
    int blocks = (int)std::min<int64_t>((total + 31) / 32, 8LL * ctx.num_sms);
    launch_pdl(splitk_reduce_kernel, std::max(blocks, 1), 256, 0, st, part, s, a.M, a.N, C, ldc, alpha,
                                                              acc, a.Cin, a.ldcin);
  }
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_dispatch(Context& ctx, Layout layout, const GemmArgs& args, int max_splits,
                          cudaStream_t st);

bool gemm_f32_supported(Layout layout, const GemmArgs& a) {
  (void)layout;
  return tma_encode_fn() != nullptr && (a.lda % 4 == 0) && aligned16(a.A) && (a.ldb % 2 == 0) &&
         aligned16(a.B) && (!a.shift || aligned16(a.shift)) && a.M < (1LL << 31) &&
         a.N < (1LL << 31) && a.K < (1LL << 31);
}

// A operand stored as float32 (args.A reinterpreted); TMA path only - callers check
// gemm_f32_supported() and otherwise widen the operand to FP64 first.
cudaError_t gemm_f32a(Context& ctx, Layout layout, const GemmArgs& args, int max_splits,
                      cudaStream_t st) {
  g_launches = 0;
  cudaError_t e = cudaSuccess;
  GemmArgs a = args;
  if (a.M > 0 && a.N > 0 && a.K > 0) {
    if (layout == Layout::CM) {
      if (a.N <= 32) e = run_tile<FCM32>(ctx, a, true, true, max_splits, st);
      else if (a.N <= 64) e = run_tile<FCM64>(ctx, a, true, true, max_splits, st);
      else if (a.N <= 128) e = run_tile<FCM128>(ctx, a, true, true, max_splits, st);
      else e = run_tile<FCM256>(ctx, a, true, true, max_splits, st);
    } else {
      if (a.N <= 32) e = run_tile<FRM32>(ctx, a, true, true, max_splits, st);
      else if (a.N <= 64) e = run_tile<FRM64>(ctx, a, true, true, max_splits, st);
      else if (a.N <= 128) e = run_tile<FRM128>(ctx, a, true, true, max_splits, st);
      else e = run_tile<FRM256>(ctx, a, true, true, max_splits, st);
    }
  }
  ctx.kernel_launches += g_launches;
  ctx.gemm_launches += g_launches;
  return e;
}

cudaError_t gemm(Context& ctx, Layout layout, const GemmArgs& args, int max_splits,
                 cudaStream_t st) {
  g_launches = 0;
  cudaError_t e = gemm_dispatch(ctx, layout, args, max_splits, st);
  ctx.kernel_launches += g_launches;
  ctx.gemm_launches += g_launches;
  return e;
}

cudaError_t gemm_dispatch(Context& ctx, Layout layout, const GemmArgs& args, int max_splits,
                          cudaStream_t st) {
  if (args.M <= 0 || args.N <= 0) return cudaSuccess;
  GemmArgs a = args;
  if (a.K <= 0) {
    // empty contraction: C = 0 (or unchanged when accumulating)
    if (a.Cin)
      return cudaMemcpy2DAsync(a.C, sizeof(double) * a.ldc, a.Cin, sizeof(double) * a.ldcin,
                               sizeof(double) * a.N, a.M, cudaMemcpyDeviceToDevice, st);
    if (!a.accumulate)
      return cudaMemset2DAsync(a.C, sizeof(double) * a.ldc, 0, sizeof(double) * a.N, a.M, st);
    return cudaSuccess;
  }
  const bool va2 = (a.lda % 2 == 0) && aligned16(a.A);
  const bool vb2 = (a.ldb % 2 == 0) && aligned16(a.B);
  const bool small = a.M * a.N * a.K < (int64_t)1 << 22;  // tiny problems: plain cp.async path
  const bool tma = va2 && vb2 && !small && !ctx.disable_tma && tma_encode_fn() != nullptr &&
                   (layout == Layout::CM || !a.shift || aligned16(a.shift)) &&
                   a.M < (1LL << 31) && a.N < (1LL << 31) && a.K < (1LL << 31);
  if (tma) {
    if (layout == Layout::CM) {
      if (a.M <= 32 && a.N <= 32) return run_tile<TCMsq32>(ctx, a, va2, vb2, max_splits, st);
      if (a.M <= 64 && a.N <= 64) return run_tile<TCMsq64>(ctx, a, va2, vb2, max_splits, st);
      if (a.N <= 32) return run_tile<TCM32>(ctx, a, va2, vb2, max_splits, st);
      if (a.N <= 64) return run_tile<TCM64>(ctx, a, va2, vb2, max_splits, st);
      if (a.N <= 128) return run_tile<TCM128>(ctx, a, va2, vb2, max_splits, st);
      return run_tile<TCM256>(ctx, a, va2, vb2, max_splits, st);
    }
    if (a.K <= 256 && a.N <= 64) return run_tile<TRMs64>(ctx, a, va2, vb2, max_splits, st);
    if (a.K <= 256 && a.N <= 128) return run_tile<TRMs128>(ctx, a, va2, vb2, max_splits, st);
    if (a.N <= 32) return run_tile<TRM32>(ctx, a, va2, vb2, max_splits, st);
    if (a.N <= 64) return run_tile<TRM64>(ctx, a, va2, vb2, max_splits, st);
    if (a.N <= 128) return run_tile<TRM128>(ctx, a, va2, vb2, max_splits, st);
    return run_tile<TRM256>(ctx, a, va2, vb2, max_splits, st);
  }
  if (layout == Layout::CM) {
    if (a.M <= 32 && a.N <= 32) return run_tile<CMsq32>(ctx, a, va2, vb2, max_splits, st);
    if (a.M <= 64 && a.N <= 64) return run_tile<CMsq64>(ctx, a, va2, vb2, max_splits, st);
    if (a.N <= 32) return run_tile<CM32>(ctx, a, va2, vb2, max_splits, st);
    if (a.N <= 64) return run_tile<CM64>(ctx, a, va2, vb2, max_splits, st);
    if (a.N <= 128) return run_tile<CM128>(ctx, a, va2, vb2, max_splits, st);
    return run_tile<CM256>(ctx, a, va2, vb2, max_splits, st);
  }
  if (a.N <= 32) return run_tile<RM32>(ctx, a, va2, vb2, max_splits, st);
  if (a.N <= 64) return run_tile<RM64>(ctx, a, va2, vb2, max_splits, st);
  if (a.N <= 128) return run_tile<RM128>(ctx, a, va2, vb2, max_splits, st);
  return run_tile<RM256>(ctx, a, va2, vb2, max_splits, st);
}

}  // namespace wssr
