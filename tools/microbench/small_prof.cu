// Cycle profile of the k x k latency kernels (maxeig64: tridiagonalisation vs Sturm rounds).
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -I../../paper_2512_05749_b200/csrc small_prof.cu
#include <cstdio>
#include <vector>
#include <random>
#include "kernels.cuh"
using namespace wssr;
int main() {
  const int k = 64;
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::vector<double> x(3 * k * k), g(k * k, 0.0);
  for (auto& v : x) v = nd(rng) * 1e-3;
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j)
      for (int r = 0; r < 3 * k; ++r) g[i * k + j] += x[r * k + i] * x[r * k + j];
  double *dG, *dout;
  long long* dprof;
  cudaMalloc(&dG, sizeof(double) * k * k);
  cudaMalloc(&dout, 8);
  cudaMalloc(&dprof, 8 * 32);
  cudaMemcpy(dG, g.data(), sizeof(double) * k * k, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(dprof, 0, 8 * 32);
    cudaEventRecord(a);
    maxeig64_kernel<<<1, 1024>>>(dG, k, dout, rep == 2 ? dprof : nullptr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long p[32];
    cudaMemcpy(p, dprof, sizeof(p), cudaMemcpyDeviceToHost);
    double ev;
    cudaMemcpy(&ev, dout, 8, cudaMemcpyDeviceToHost);
    printf("lambda_max %.17g\n", ev);
    printf("maxeig64: %.1f us  tridiag %lld cyc; rounds:", ms * 1e3, p[0] - p[1]);
    long long prev = p[0];
    for (int r = 0; r < 12 && p[2 + r]; ++r) { printf(" %lld", p[2 + r] - prev); prev = p[2 + r]; }
    printf("\n  step 10:");
    for (int q = 21; q <= 26; ++q) printf(" %lld", p[q] - p[q - 1]);
    printf("\n");
  }
  // CholeskyQR2 core: a generic SPD Gram (first pass) and a near-identity one (series path)
  {
    double *dR, *dRi; int* dst;
    cudaMemset(dprof, 0, 8 * 32);
    cudaMalloc(&dR, 8 * k * k); cudaMalloc(&dRi, 8 * k * k); cudaMalloc(&dst, 8);
    cudaFuncSetAttribute(chol_inv_reg64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * 64 * 65 * 8);
    std::vector<double> gi(k * k);
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) gi[i * k + j] = (i == j ? 1.0 : 0.0) + 1e-7 * (g[i * k + j] / g[0]);
    for (int which = 0; which < 2; ++which) {
      cudaMemcpy(dG, which ? gi.data() : g.data(), 8 * k * k, cudaMemcpyHostToDevice);
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(dst, 0, 8);
        cudaEventRecord(a);
        chol_inv_reg64_kernel<<<1, 256, 2 * 64 * 65 * 8>>>(dG, k, dR, dRi, dst, 1e-13, 1,
                                                            rep == 2 ? dprof : nullptr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        int st[2];
        cudaMemcpy(st, dst, 8, cudaMemcpyDeviceToHost);
        printf("chol_inv_reg64 %s: %.1f us (status %d)\n", which ? "series" : "sweep", ms * 1e3, st[0]);
        long long pp[32];
        cudaMemcpy(pp, dprof, sizeof(pp), cudaMemcpyDeviceToHost);
        if (!which) printf("   loop %lld cyc; step 10: %lld %lld %lld %lld %lld\n", pp[1] - pp[0],
                           pp[11] - pp[10], pp[12] - pp[11], pp[13] - pp[12], pp[14] - pp[13], pp[15] - pp[14]);
      }
    }
  }
  return 0;
}
