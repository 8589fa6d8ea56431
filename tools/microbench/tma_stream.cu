// HBM streaming rate of TMA loads by tile shape (one CTA per SM, 5-stage ring, no compute):
//   mode 0: 4-D tiled box {32 B, 128 rows, 1, 7} (the blocked digit planes: 7 runs of 4 KB)
//   mode 1: 2-D tiled box {128 B, 32 rows} x 7 (128-byte rows, 4 KB each)
//   mode 2: 1-D bulk copies, 7 x 4 KB contiguous runs
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__global__ void __launch_bounds__(128, 1) stream(const __grid_constant__ CUtensorMap t4, const __grid_constant__ CUtensorMap t2,
                                                 const int8_t* base, int64_t plane, int64_t tiles, int mode, int64_t rows) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[5];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 5; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int64_t per = (tiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = blockIdx.x * per, t1 = min(tiles, t0 + per);
  int64_t g = 0;
  for (int64_t t = t0; t < t1 + 5; ++t, ++g) {
    if (t >= t0 + 5) wait(&full[(g - 5) % 5], ((g - 5) / 5) & 1);
    if (t >= t1) continue;
    const int s = g % 5;
    unsigned char* dst = sm + s * 28672;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&full[s])), "r"(28672) : "memory");
    // tile t -> (kb, mtile) with 32 rows of tiles per 128-row block
    const int64_t mt = t % (rows / 128), kb = t / (rows / 128);
    if (mode == 0) {
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n"
                   ::"r"(su32(dst)), "l"((uint64_t)&t4), "r"(0), "r"((int)(mt * 128)), "r"((int)kb), "r"(0), "r"(su32(&full[s])) : "memory");
    } else if (mode == 1) {
      for (int a = 0; a < 7; ++a)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
                     ::"r"(su32(dst + a * 4096)), "l"((uint64_t)&t2), "r"(0), "r"((int)((a * (plane / 128)) + (kb * rows + mt * 128) / 4)), "r"(su32(&full[s])) : "memory");
    } else {
      for (int a = 0; a < 7; ++a) {
        const int8_t* src = base + a * plane + (kb * rows + mt * 128) * 32;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(su32(dst + a * 4096)), "l"(src), "r"(4096), "r"(su32(&full[s])) : "memory");
      }
    }
  }
}
int main() {
  const int64_t rows = 4096, P = 131072, plane = rows * P;  // 7 planes of 512 MiB
  int8_t* buf; if (cudaMalloc(&buf, 7 * plane) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(buf, 1, 7 * plane);
  void* fp; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  CUtensorMap t4, t2;
  cuuint64_t d4[4] = {32, (cuuint64_t)rows, (cuuint64_t)(P / 32), 7}; cuuint64_t s4[3] = {32, 32 * rows, (cuuint64_t)plane};
  cuuint32_t b4[4] = {32, 128, 1, 7}; cuuint32_t e4[4] = {1, 1, 1, 1};
  enc(&t4, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, buf, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d2[2] = {128, (cuuint64_t)(7 * plane / 128)}; cuuint64_t s2[1] = {128};
  cuuint32_t b2[2] = {128, 32}; cuuint32_t e2[2] = {1, 1};
  enc(&t2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 28672);
  const int64_t tiles = (rows / 128) * (P / 32);
  for (int mode = 0; mode < 3; ++mode) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      stream<<<sms, 128, 5 * 28672>>>(t4, t2, buf, plane, tiles, mode, rows);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    cudaError_t e = cudaGetLastError();
    printf("mode %d: %.3f ms  %.2f TB/s  (%s)\n", mode, ms, 7.0 * plane / (ms * 1e9), cudaGetErrorString(e));
  }
  return 0;
}
