// Cost of a dependent "publish -> __syncthreads -> read -> __syncthreads" step on one CTA.
#include <cstdio>
__global__ void steps(double* out, int n, int variant) {
  __shared__ double buf[64];
  __shared__ double s_val;
  double acc = threadIdx.x;
  if (threadIdx.x == 0) s_val = 1.0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double v = s_val;
    if (variant >= 1 && threadIdx.x < 64) buf[threadIdx.x] = acc * v;
    __syncthreads();
    if (variant >= 1) acc += buf[(threadIdx.x + j) & 63];
    if (variant >= 2 && threadIdx.x == (j & 255)) s_val = sqrt(acc) + 1.0 / (acc + 1.0);
    __syncthreads();
  }
  if (acc == 12345.0) out[0] = acc;
}
int main() {
  double* d; cudaMalloc(&d, 64);
  for (int variant = 0; variant < 3; ++variant) {
    for (int threads : {32, 256, 1024}) {
      steps<<<1, threads>>>(d, 64, variant);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      for (int r = 0; r < 20; ++r) steps<<<1, threads>>>(d, 640, variant);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("variant %d threads %4d: %.1f ns per step\n", variant, threads, ms * 1e6 / (20 * 640));
    }
  }
}
