// Host-side dispatch for the DMMA GEMM family: tile-config choice by output width, operand
// vector width (16-byte cp.async when rows are 16-byte aligned) and split-K sizing.
#include "engine.h"
#include "gemm.cuh"

namespace wssr {

namespace {

thread_local int64_t g_launches = 0;

template <Layout L, int BM, int BN, int BK, int WMW, int WNW, int ST, int VA, int VB>
cudaError_t launch_one(const GemmArgs& a, int splits, cudaStream_t st) {
  using Cfg = GemmCfg<L, BM, BN, BK, WMW, WNW, ST>;
  auto kern = gemm_dmma_kernel<L, BM, BN, BK, WMW, WNW, ST, VA, VB>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((unsigned)((a.M + BM - 1) / BM), (unsigned)((a.N + BN - 1) / BN), (unsigned)splits);
  kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes, st>>>(a);
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

int choose_splits(int64_t tiles, int64_t K, int BK, int capacity, int max_splits) {
  if (max_splits <= 1) return 1;
  int64_t kmax = (K + 4 * BK - 1) / (4 * BK);  // keep >= 4 k-tiles per split
  int smax = (int)std::min<int64_t>(max_splits, std::max<int64_t>(1, kmax));
  if (tiles >= 6LL * capacity) return 1;
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= smax; ++s) {
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
  int s = choose_splits(tiles, a.K, T::kBK, cap, max_splits);
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
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 4LL * ctx.num_sms);
  if (blocks < 1) blocks = 1;
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(part, s, a.M, a.N, C, ldc, alpha, acc);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t gemm_dispatch(Context& ctx, Layout layout, const GemmArgs& args, int max_splits,
                          cudaStream_t st);

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
    if (!a.accumulate)
      return cudaMemset2DAsync(a.C, sizeof(double) * a.ldc, 0, sizeof(double) * a.N, a.M, st);
    return cudaSuccess;
  }
  const bool va2 = (a.lda % 2 == 0) && aligned16(a.A);
  const bool vb2 = (a.ldb % 2 == 0) && aligned16(a.B);
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
