// DMMA.8x8x4 throughput vs resident warps per SM and independent accumulator chains per warp
// (sizing the tall-skinny kernels of csrc/tallskinny.cu).  nvcc -O3 -arch=sm_100a dmma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) dmma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}
template <int C>
void run(int warps_per_cta, int ctas_per_sm) {
  int sms = 148;
  double* o;
  cudaMalloc(&o, 8192);
  int iters = 4096 * 8 / C;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<C><<<sms * ctas_per_sm, 32 * warps_per_cta>>>(o, iters);
  cudaEventRecord(a);
  k<C><<<sms * ctas_per_sm, 32 * warps_per_cta>>>(o, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double dmmas = (double)sms * ctas_per_sm * warps_per_cta * iters * C;
  printf("warps/SM %3d chains %3d : %.1f TF/s  (%.3f DMMA/ns/SM)\n", warps_per_cta * ctas_per_sm,
         C, dmmas * 512 / (ms * 1e-3) / 1e12, dmmas / (ms * 1e6) / sms);
  cudaFree(o);
}
int main() {
  run<8>(4, 1); run<8>(8, 1); run<8>(16, 1); run<8>(32, 1);
  run<16>(8, 1); run<16>(16, 1);
  run<36>(8, 1); run<18>(16, 1); run<32>(8, 1); run<32>(16, 1);
  run<4>(8, 1); run<4>(16, 1); run<2>(16, 1); run<1>(32, 1);
  return 0;
}
