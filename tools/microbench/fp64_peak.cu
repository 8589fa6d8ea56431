// FP64 peak microbenchmark for B200 (sm_100a): DFMA (SIMT) vs DMMA (mma.sync f64).
// Establishes the measured FP64 roofline denominator used by bench.py / DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma884_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 * i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void ffma_loop(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.678f) out[threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"device\": \"%s\", \"sms\": %d", p.name, p.multiProcessorCount);
  double* d; CK(cudaMalloc(&d, 1 << 20));
  int sms = p.multiProcessorCount;
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 4, threads = 32 * wpb, iters = 20000;
    float ms = time_it([&] { dfma_loop<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9); });
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_w%d_tflops\": %.2f", wpb, fl / ms / 1e9);
    ms = time_it([&] { dmma884_loop<<<blocks, threads>>>(d, iters); });
    fl = 2.0 * 8 * 256 * iters * (double)blocks * wpb;
    printf(", \"dmma884_w%d_tflops\": %.2f", wpb, fl / ms / 1e9);
    ms = time_it([&] { dmma16816_loop<<<blocks, threads>>>(d, iters / 4); });
    fl = 2.0 * 4 * 16 * 8 * 16 * (iters / 4) * (double)blocks * wpb;
    printf(", \"dmma16816_w%d_tflops\": %.2f", wpb, fl / ms / 1e9);
    ms = time_it([&] { ffma_loop<<<blocks, threads>>>((float*)d, iters, 1.0000001f, 1e-9f); });
    fl = 2.0 * 16 * iters * (double)blocks * threads;
    printf(", \"ffma_w%d_tflops\": %.2f", wpb, fl / ms / 1e9);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
