// Does FP64 SIMT arithmetic (the converter's DADD/DMUL/F2I) slow down concurrently running
// tcgen05 kind::i8 MMAs (and vice versa)?  Warp 1 issues the Ozaki 11-MMA stage back to back;
// warps 4.. run converter-like FP64 arithmetic (mode 1), integer-only work (mode 2), or nothing.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw32(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (16ull << 32) | (1ull << 46) | (6ull << 61);
}
__device__ unsigned long long g_sink;
__global__ void __launch_bounds__(640, 1) ov(int stages, int mode, int conv_iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t fin;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * 43008 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&fin)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (warp == 1 && lane == 0 && stages > 0) {
    auto mma = [&](uint32_t col, uint32_t a, uint32_t b, int n) {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem + col), "l"(desc_sw32(a)), "l"(desc_sw32(b)), "r"(idesc), "r"(1) : "memory");
    };
    unsigned long long t0 = clock64();
    for (int it = 0; it < stages; ++it) {
      const uint32_t abase = su32(sm) + (it % 3) * 43008, bbase = abase + 28672;
      mma(64, abase + 4096, bbase, 256); mma(320, abase + 4096, bbase + 256 * 32, 192);
      mma(0, abase, bbase, 64); mma(64, abase, bbase + 64 * 32, 256); mma(320, abase, bbase + 320 * 32, 128);
      for (int a = 2; a < 7; ++a) {
        int col = 64 * a, brow = 0, left = 64 * (8 - a);
        while (left > 0) { const int n = left > 256 ? 256 : left; mma(col, abase + a * 4096, bbase + brow * 32, n); col += n; brow += n; left -= n; }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&fin)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&fin)) : "memory");
    if (blockIdx.x == 0) cyc[0] = clock64() - t0;
  } else if (warp >= 4 && mode > 0) {
    double x[16]; unsigned long long acc = 0; uint32_t u[16];
    for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * 1e-3 + i; u[i] = threadIdx.x * 7 + i; }
    unsigned long long t0 = clock64();
    for (int it = 0; it < conv_iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (mode == 1) {
          const double t = (x[i] - 0.25) * 1024.0;
          acc ^= (unsigned long long)__double2ll_rn(t) + 0x0080808080808080ull;
          x[i] += 1.0;
        } else {
          u[i] = __byte_perm(u[i], u[(i + 1) & 15], 0x5140) ^ 0x80808080u;
          acc += u[i];
        }
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 128) cyc[1] = clock64() - t0;
    if (acc == 42) g_sink = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(ov, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 43008);
  const int stages = 400, conv_iters = 256;
  for (int mma_on = 0; mma_on < 2; ++mma_on)
    for (int mode = 0; mode < 3; ++mode) {
      if (!mma_on && !mode) continue;
      unsigned long long h[2] = {0, 0};
      for (int rep = 0; rep < 2; ++rep) {
        cudaMemset(d, 0, 16);
        ov<<<sms, 640, 3 * 43008>>>(mma_on ? stages : 0, mode, conv_iters, d);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      }
      printf("mma=%d conv_mode=%d: MMA %.0f clk/stage, converter work %.0f clk (16 warps x 16 x %d elements)\n",
             mma_on, mode, mma_on ? (double)h[0] / stages : 0.0, (double)h[1], conv_iters);
    }
  return 0;
}
