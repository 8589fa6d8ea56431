// Dependent-chain latency (cycles) of FP64 / FP32 ops and shuffles on one warp.
#include <cstdio>
#include <cuda_runtime.h>
#define N 256
__global__ void k(double* out, long long* t, double a, float af) {
  double x = a, y = a * 0.5;
  float f = af;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fma(x, 0.999, 1e-3);
  t1 = clock64(); t[0] = t1 - t0;
  // DADD chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) y = y + 1e-3;
  t1 = clock64(); t[1] = t1 - t0;
  // FFMA chain
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) f = fmaf(f, 0.999f, 1e-3f);
  t1 = clock64(); t[2] = t1 - t0;
  // double shuffle chain (data-dependent so it cannot fold)
  double z = x + y + threadIdx.x;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) z = __shfl_xor_sync(0xffffffffu, z, 1 + (i & 3)) + 1.0;
  t1 = clock64(); t[3] = t1 - t0;
  // sqrt chain
  double s = z + 2.0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) s = sqrt(s) + 1.0;
  t1 = clock64(); t[4] = t1 - t0;
  // rcp chain (IEEE)
  double r = s;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) r = 1.0 / r + 1.0;
  t1 = clock64(); t[5] = t1 - t0;
  // DMUL chain
  double m = r;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) m = m * 1.0000001;
  t1 = clock64(); t[6] = t1 - t0;
  // shared-memory load chain (pointer chasing through smem)
  __shared__ int sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7 + 1) & 1023;
  __syncwarp();
  int idx = threadIdx.x;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) idx = sm[idx];
  t1 = clock64(); t[7] = t1 - t0;
  out[threadIdx.x] = x + y + f + z + s + r + m + idx;
}
int main() {
  double* o; long long* t;
  cudaMalloc(&o, 8 * 32); cudaMalloc(&t, 8 * 8);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(o, t, 1.0, 1.0f);
    long long h[8] = {0};
    cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost);
    const char* nm[] = {"DFMA", "DADD", "FFMA", "SHFL.f64+DADD", "sqrt+add", "1/x+add", "DMUL", "LDS chase"};
    for (int i = 0; i < 8; ++i) printf("%-10s %.1f cyc/op\n", nm[i], (double)h[i] / N);
  }
  return 0;
}
