// Tile-config sweep for the DMMA GEMM family on the WSSR phase shapes (dev tool).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <algorithm>
#include "../../paper_2512_05749_b200/csrc/gemm_tma.cuh"
#include <cudaTypedefs.h>
#include <cstring>

using namespace wssr;

static double* dalloc(size_t n) { double* p; cudaMalloc(&p, n * 8); return p; }
__global__ void fill(double* p, size_t n, double s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = sin(s * (double)(i % 1000003) + 0.1);
}

template <Layout L, int BM, int BN, int BK, int WMW, int WNW, int ST>
void run(const char* tag, int64_t M, int64_t N, int64_t K, double* A, double* B, double* sh, double* C, double* part) {
  using Cfg = GemmCfg<L, BM, BN, BK, WMW, WNW, ST>;
  auto kern = gemm_dmma_kernel<L, BM, BN, BK, WMW, WNW, ST, 2, 2>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmemBytes) != cudaSuccess) {
    printf("%s: smem too large\n", tag); cudaGetLastError(); return;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::kThreads, Cfg::kSmemBytes);
  int cap = 148 * std::max(occ, 1);
  int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  double best_ms = 1e30; int best_s = 1;
  std::vector<int> cands;
  for (int s = 1; s <= 64; ++s) {
    double w = (double)(tiles * s) / cap; double eff = w / std::ceil(w);
    if (eff > 0.9 || s == 1) cands.push_back(s);
    if (cands.size() > 6) break;
  }
  for (int s : cands) {
    int64_t kc = (K + s - 1) / s; kc = (kc + BK - 1) / BK * BK; int ss = (int)((K + kc - 1) / kc);
    GemmArgs a{A, L == Layout::CM ? M : K, B, N, sh, C, N, M, N, K, kc, 1.0, 0, ss > 1 ? part : nullptr, nullptr, 0};
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)ss);
    for (int w = 0; w < 2; ++w) kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(a);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(a);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    if (cudaGetLastError() != cudaSuccess) { printf("%s: launch error\n", tag); return; }
    if (ms < best_ms) { best_ms = ms; best_s = ss; }
  }
  printf("%-34s M=%-7lld N=%-4lld K=%-7lld occ=%d smem=%6zu  best_s=%-3d %.3f ms  %.2f TF/s\n", tag,
         (long long)M, (long long)N, (long long)K, occ, Cfg::kSmemBytes, best_s, best_ms,
         2.0 * M * N * K / best_ms / 1e9);
}

PFN_cuTensorMapEncodeTiled_v12000 enc() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) { void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q); fn = (PFN_cuTensorMapEncodeTiled_v12000)p; }
  return fn;
}
void map2(CUtensorMap* m, const double* p, int64_t inner, int64_t outer, int64_t pitch, int bo) {
  cuuint64_t d[2] = {(cuuint64_t)inner, (cuuint64_t)outer}; cuuint64_t st[1] = {(cuuint64_t)pitch * 8};
  cuuint32_t b[2] = {16u, (cuuint32_t)bo}; cuuint32_t es[2] = {1, 1};
  if (enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)p, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) printf("map fail\n");
}
void map1(CUtensorMap* m, const double* p, int64_t n, int bo) {
  cuuint64_t d[1] = {(cuuint64_t)n}; cuuint64_t st[1] = {0}; cuuint32_t b[1] = {(cuuint32_t)bo}; cuuint32_t es[1] = {1};
  if (enc()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, (void*)p, d, st, b, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) printf("map1 fail\n");
}
template <Layout L, int BM, int BN, int BK, int WMW, int WNW, int ST>
void runt(const char* tag, int64_t M, int64_t N, int64_t K, double* A, double* B, double* sh, double* C, double* part) {
  using Cfg = TmaCfg<L, BM, BN, BK, WMW, WNW, ST>;
  auto kern = gemm_tma_kernel<L, BM, BN, BK, WMW, WNW, ST>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmemBytes) != cudaSuccess) {
    printf("%s: smem too large\n", tag); cudaGetLastError(); return;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cfg::kThreads, Cfg::kSmemBytes);
  int cap = 148 * std::max(occ, 1);
  int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  CUtensorMap tA, tB, tS; memset(&tS, 0, sizeof(tS));
  if (L == Layout::CM) map2(&tA, A, M, K, M, BK); else map2(&tA, A, K, M, K, BM);
  map2(&tB, B, N, K, N, BK);
  if (L == Layout::RM && sh) map1(&tS, sh, K, BK);
  double best_ms = 1e30; int best_s = 1;
  std::vector<int> cands;
  for (int s = 1; s <= 256; ++s) {
    double w = (double)(tiles * s) / cap; double eff = w / std::ceil(w);
    if (K / s < 256 && s > 1) break;
    if (eff > 0.9 || s == 1) cands.push_back(s);
    if (cands.size() > 5) break;
  }
  for (int s : cands) {
    int64_t kc = (K + s - 1) / s; kc = (kc + BK - 1) / BK * BK; int ss = (int)((K + kc - 1) / kc);
    GemmArgs a{A, L == Layout::CM ? M : K, B, N, sh, C, N, M, N, K, kc, 1.0, 0, ss > 1 ? part : nullptr, nullptr, 0};
    dim3 grid((unsigned)((M + BM - 1) / BM), (unsigned)((N + BN - 1) / BN), (unsigned)ss);
    for (int w = 0; w < 2; ++w) kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(tA, tB, tS, a);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) kern<<<grid, Cfg::kThreads, Cfg::kSmemBytes>>>(tA, tB, tS, a);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
    cudaError_t er = cudaGetLastError();
    if (er != cudaSuccess) { printf("%s: launch error %s\n", tag, cudaGetErrorString(er)); return; }
    if (ms < best_ms) { best_ms = ms; best_s = ss; }
  }
  printf("%-36s M=%-7lld N=%-4lld K=%-7lld occ=%d smem=%6zu  best_s=%-3d %.4f ms  %.2f TF/s\n", tag,
         (long long)M, (long long)N, (long long)K, occ, Cfg::kSmemBytes, best_s, best_ms,
         2.0 * M * N * K / best_ms / 1e9);
}
#define RUNTRM(BM, BN, BK, WM, WN, ST) runt<Layout::RM, BM, BN, BK, WM, WN, ST>("TRM<" #BM "," #BN "," #BK "," #WM "x" #WN ",s" #ST ">", M, N, K, A, B, sh, C, part)
#define RUNTCM(BM, BN, BK, WM, WN, ST) runt<Layout::CM, BM, BN, BK, WM, WN, ST>("TCM<" #BM "," #BN "," #BK "," #WM "x" #WN ",s" #ST ">", M, N, K, A, B, sh, C, part)
#define RUNRM(BM, BN, BK, WM, WN, ST) run<Layout::RM, BM, BN, BK, WM, WN, ST>("RM<" #BM "," #BN "," #BK "," #WM "x" #WN ",s" #ST ">", M, N, K, A, B, sh, C, part)
#define RUNCM(BM, BN, BK, WM, WN, ST) run<Layout::CM, BM, BN, BK, WM, WN, ST>("CM<" #BM "," #BN "," #BK "," #WM "x" #WN ",s" #ST ">", M, N, K, A, B, sh, C, part)

int main() {
  const size_t big = (size_t)16384 * 65536;
  double* A = dalloc(big); double* B = dalloc(1 << 24); double* sh0 = dalloc(1 << 22); double* C = dalloc(1 << 24);
  double* part = dalloc((size_t)1 << 27);
  fill<<<1024, 256>>>(A, big, 1.1); fill<<<1024, 256>>>(B, 1 << 24, 0.7); fill<<<1024, 256>>>(sh0, 1 << 22, 0.3);
  cudaDeviceSynchronize();
  {
    int64_t M = 131072, N = 64, K = 64; double* sh = nullptr;  // TRMM
    RUNTRM(128, 64, 64, 4, 2, 1); RUNTRM(64, 64, 64, 2, 2, 1); RUNTRM(64, 64, 32, 2, 2, 2);
    RUNTRM(32, 64, 64, 1, 2, 1); RUNTRM(64, 64, 16, 2, 2, 4); RUNTRM(128, 64, 32, 4, 2, 2);
  }
  {
    int64_t M = 1048576, N = 128, K = 128; double* sh = nullptr;  // TRMM c2
    RUNTRM(64, 128, 32, 2, 4, 2); RUNTRM(64, 128, 64, 2, 4, 2); RUNTRM(32, 128, 64, 1, 4, 2);
    RUNTRM(64, 128, 128, 2, 4, 1);
  }
  {
    int64_t M = 64, N = 64, K = 131072; double* sh = nullptr;  // Gram
    RUNTCM(64, 64, 32, 2, 2, 4); RUNTCM(64, 64, 64, 2, 2, 2); RUNTCM(64, 64, 32, 2, 2, 2);
    RUNTCM(64, 64, 64, 2, 2, 3); RUNTCM(64, 64, 16, 2, 2, 6);
  }
  {
    int64_t M = 128, N = 128, K = 1048576; double* sh = nullptr;  // Gram c2
    RUNTCM(64, 128, 32, 2, 4, 3); RUNTCM(128, 128, 32, 4, 4, 2); RUNTCM(64, 128, 64, 2, 4, 2);
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
