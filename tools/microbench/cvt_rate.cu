// Throughput of the converter's per-element ops on sm_100a: F2I.S64.F64 (__double2ll_rn),
// DADD/DMUL, and an integer-only alternative (exponent/mantissa bit extraction).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_f2i(double* in, long long* out, int iters) {
  double x[8]; long long acc = 0;
  for (int i = 0; i < 8; ++i) x[i] = in[threadIdx.x + i] * (1 << 20);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc += __double2ll_rn(x[i]); x[i] += 1.0; }
  }
  if (acc == 42) out[0] = acc;
}
__global__ void k_dadd(double* in, long long* out, int iters) {
  double x[8]; double acc = 0;
  for (int i = 0; i < 8; ++i) x[i] = in[threadIdx.x + i];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { x[i] = (x[i] - 0.5) * 1.0000001; }
  }
  for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 42) out[0] = (long long)acc;
}
// integer path: X = mantissa shifted by (e - E0): exact for |x| < 2^54 scaled values with rounding
__device__ __forceinline__ long long int_round(double x) {
  // x already scaled so that |x| < 2^54; use the 2^52 magic for the low part
  const double big = 6755399441055744.0;  // 1.5 * 2^52
  const double hi = rint(x * (1.0 / 4096.0));       // top part (integer multiple of 4096 in x units)
  const double lo = x - hi * 4096.0;                 // |lo| <= 2048, exact
  const long long H = __double_as_longlong(hi + big) - __double_as_longlong(big);
  const long long L = __double_as_longlong(lo + big) - __double_as_longlong(big);
  return H * 4096 + L;
}
__global__ void k_magic(double* in, long long* out, int iters) {
  double x[8]; long long acc = 0;
  for (int i = 0; i < 8; ++i) x[i] = in[threadIdx.x + i] * (1 << 20);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { acc += int_round(x[i]); x[i] += 1.0; }
  }
  if (acc == 42) out[0] = acc;
}
// converter-like: 16 independent elements per thread, DADD -> DMUL -> F2I -> +bias
__global__ void k_conv16(double* in, long long* out, int iters, int use_f2i) {
  double x[16]; unsigned long long acc = 0;
  for (int i = 0; i < 16; ++i) x[i] = in[(threadIdx.x + i) & 4095] + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double t = (x[i] - 0.25) * 1024.0;
      unsigned long long y;
      if (use_f2i) y = (unsigned long long)__double2ll_rn(t) + 0x0080808080808080ull;
      else y = (unsigned long long)(__double_as_longlong(t + 6755399441055744.0) - 0x4338000000000000ll) + 0x0080808080808080ull;
      acc ^= y;
      x[i] += 1.0;
    }
  }
  if (acc == 42) out[0] = acc;
}

int main() {
  double* in; long long* out; cudaMalloc(&in, 4096 * 8); cudaMalloc(&out, 8); cudaMemset(in, 0, 4096 * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int kind = 0; kind < 3; ++kind) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (kind == 0) k_f2i<<<sms * 4, 512>>>(in, out, iters);
      if (kind == 1) k_dadd<<<sms * 4, 512>>>(in, out, iters);
      if (kind == 2) k_magic<<<sms * 4, 512>>>(in, out, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)sms * 4 * 512 * iters * 8;
    printf("%s: %.1f Gop/s  = %.1f per clk per SM @1.9GHz\n", kind == 0 ? "F2I.S64.F64 (+DADD)" : kind == 1 ? "DADD+DMUL" : "magic int round",
           ops / (ms * 1e6), ops / (ms * 1e-3) / sms / 1.9e9);
  }
  for (int use = 0; use < 2; ++use)
    for (int warps : {8, 16, 32}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        k_conv16<<<sms, 32 * warps>>>(in, out, 1024, use);
        cudaEventRecord(b); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double el = (double)sms * 32 * warps * 1024 * 16;
      printf("conv16 %s warps/SM=%d: %.1f elements/clk/SM\n", use ? "F2I  " : "magic", warps, el / (ms * 1e-3) / sms / 1.9e9);
    }
  return 0;
}
