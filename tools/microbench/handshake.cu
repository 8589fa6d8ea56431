// Handshake cost of the Ozaki pipeline shape: one MMA thread issues the 11-MMA stage and commits
// to dempty[d]; 16 "converter" warps wait dempty[d] (stage g - D) and arrive on conv[d]; the MMA
// thread waits conv[d] before issuing stage g.  Reports cycles per stage for D = 2, 3, 4 and
// spin vs suspend-hint waits.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_sw32(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (16ull << 32) | (1ull << 46) | (6ull << 61);
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par, int sleep) {
  if (sleep)
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n@!p bra W;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}
__global__ void __launch_bounds__(640, 1) hs(int iters, int D, int sleep, int do_fence, unsigned long long* cycles, int nconv, int dual) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t conv[4], dempty[4], fin;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 4 * 43008 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    for (int d = 0; d < 4; ++d) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(&conv[d])), "r"(nconv));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&dempty[d])));
    }
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
  unsigned long long t0 = clock64();
  const bool issuer = dual ? (warp == 1 || warp == 3) : (warp == 1);
  if (issuer) {
    auto mma = [&](uint32_t col, uint32_t a, uint32_t b, int n) {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem + col), "l"(desc_sw32(a)), "l"(desc_sw32(b)), "r"(idesc), "r"(1) : "memory");
    };
    const int me = dual ? (warp == 1 ? 0 : 1) : 0;
    const int step = dual ? 2 : 1;
    for (int g = me; g < iters; g += step) {
      const int d = g % D;
      if (D > 1) wait(&conv[d], (g / D) & 1, sleep);
      if (dual && g > 0) asm volatile("bar.sync %0, 64;\n" ::"r"(1 + me) : "memory");  // token in
      if (lane == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t abase = su32(sm) + d * 43008, bbase = abase + 28672;
        mma(64, abase + 4096, bbase, 256); mma(320, abase + 4096, bbase + 256 * 32, 192);
        mma(0, abase, bbase, 64); mma(64, abase, bbase + 64 * 32, 256); mma(320, abase, bbase + 320 * 32, 128);
        for (int a = 2; a < 7; ++a) {
          int col = 64 * a, brow = 0, left = 64 * (8 - a);
          while (left > 0) { const int n = left > 256 ? 256 : left; mma(col, abase + a * 4096, bbase + brow * 32, n); col += n; brow += n; left -= n; }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&dempty[d])) : "memory");
      }
      __syncwarp();
      if (dual && g + 1 < iters) asm volatile("bar.arrive %0, 64;\n" ::"r"(1 + (1 - me)) : "memory");  // token out
    }
    if (lane == 0 && me == ((iters - 1) % step)) {
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&fin)) : "memory");
      wait(&fin, 0, 0);
      if (blockIdx.x == 0) *cycles = clock64() - t0;
    }
  } else if (warp >= 4 && warp < 4 + nconv && D > 1) {
    for (int g = 0; g < iters; ++g) {
      const int d = g % D;
      wait(&dempty[d], ((g / D) & 1) ^ 1, sleep);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(&conv[d])) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}
int main() {
  unsigned long long* dd; CK(cudaMalloc(&dd, 8));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(hs, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 43008));
  for (int threads : {128, 640}) {
    hs<<<sms, threads, 4 * 43008>>>(2000, 1, 0, 1, dd, 16, 0);
    CK(cudaDeviceSynchronize());
    unsigned long long c; CK(cudaMemcpy(&c, dd, 8, cudaMemcpyDeviceToHost));
    printf("no handshake, %d threads: %.0f cycles/stage\n", threads, c / 2000.0);
  }
  for (int dual = 0; dual < 2; ++dual)
  for (int nconv : {1, 16})
  for (int D = 2; D <= 4; D += 2)
    for (int sleep = 0; sleep < 1; ++sleep)
      for (int f = 1; f < 2; ++f) {
        hs<<<sms, 640, 4 * 43008>>>(2000, D, sleep, f, dd, nconv, dual);
        CK(cudaDeviceSynchronize());
        unsigned long long c; CK(cudaMemcpy(&c, dd, 8, cudaMemcpyDeviceToHost));
        printf("dual=%d nconv=%d D=%d: %.0f cycles/stage\n", dual, nconv, D, c / 2000.0);
      }
  return 0;
}
