// Does DFMA (fp64 pipe) run concurrently with DMMA (tensor pipe) on B200?  Warps w < split do
// DMMA.8x8x4 chains, warps >= split do DFMA chains; report the combined FP64 TFLOP/s.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mixed(double* out, int iters, int split, int dfma_chains_per_iter) {
  const int w = threadIdx.x >> 5;
  double s = 0;
  if (w < split) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    const int n = iters * dfma_chains_per_iter;
    for (int it = 0; it < n; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 1.0000001, 1e-9);
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  double* d; cudaMalloc(&d, 1 << 20);
  const int blocks = 148 * 2, threads = 512, iters = 4000;
  for (int split : {16, 0, 8, 12, 10}) {
    for (int ratio : {8, 16, 32}) {  // DFMA iterations per DMMA iteration
      mixed<<<blocks, threads>>>(d, 100, split, ratio);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      mixed<<<blocks, threads>>>(d, iters, split, ratio);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const int nw = threads / 32;
      double fl_mma = 2.0 * 8 * 256 * (double)iters * blocks * split;
      double fl_fma = 2.0 * 8 * 32 * (double)iters * ratio * blocks * (nw - split);
      printf("split=%2d/16 ratio=%2d  %.3f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF/s\n", split, ratio, ms,
             fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
      if (split == 16 || split == 0) break;
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
