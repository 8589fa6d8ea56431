// tcgen05.mma issue-rate microbenchmark (sm_100a): one CTA per SM issues back-to-back MMAs on
// static shared-memory operands (no TMA, no epilogue) and reports the per-SM MAC rate for
// kind::i8 and kind::f16 with M = 128 (cta_group::1) at several N.  Establishes whether the
// single-SM int8 tensor-core path runs at the chip's dense peak.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc_sw32(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | (16ull << 32) | (1ull << 46) |
         (6ull << 61);
}

template <int KIND>  // 0 = i8 (K=32 bytes), 1 = f16 (K=16 elements = 32 bytes)
__global__ void __launch_bounds__(128, 1) umma_loop(int n, int iters, unsigned long long* cycles,
                                                    int rotate) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    uint32_t idesc;
    if (KIND == 0)
      idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    else  // f16 x f16 -> f32
      idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t a0 = su32(sm), b0 = su32(sm + 16384);
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = rotate ? (j & 3) : 0;
        const uint64_t ad = desc_sw32(a0 + r * 4096), bd = desc_sw32(b0 + r * 8192);
        if (KIND == 0)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1) : "memory");
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

// the Ozaki stage: 11 MMAs (see csrc/ozaki.cu) over 3 rotating 42 KB stage buffers
__global__ void __launch_bounds__(128, 1) ozaki_seq(int iters, unsigned long long* cycles,
                                                    int commit_each) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 3 * 43008 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    auto mma = [&](uint32_t col, uint32_t a, uint32_t b, int n, uint32_t acc) {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(tmem + col), "l"(desc_sw32(a)), "l"(desc_sw32(b)), "r"(idesc), "r"(acc) : "memory");
    };
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t abase = su32(sm) + (it % 3) * 43008, bbase = abase + 28672;
      mma(64, abase + 4096, bbase, 256, 1);
      mma(320, abase + 4096, bbase + 256 * 32, 192, 1);
      mma(0, abase, bbase, 64, 1);
      mma(64, abase, bbase + 64 * 32, 256, 1);
      mma(320, abase, bbase + 320 * 32, 128, 1);
      for (int a = 2; a < 7; ++a) {
        int col = 64 * a, brow = 0, left = 64 * (8 - a);
        while (left > 0) {
          const int n = left > 256 ? 256 : left;
          mma(col, abase + a * 4096, bbase + brow * 32, n, 1);
          col += n; brow += n; left -= n;
        }
      }
      if (commit_each == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar2)) : "memory");
      if (commit_each == 2) {  // commit and wait for the stage two back (a 2-deep ring)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar2)) : "memory");
        if (it >= 1) {
          const uint32_t par = (it - 1) & 1;
          asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(su32(&bar2)), "r"(par) : "memory");
        }
      }
    }
    unsigned long long tissue = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) { *cycles = t1 - t0; cycles[1] = tissue - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

int main() {
  unsigned long long* d;
  CK(cudaMalloc(&d, 16));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(umma_loop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
  CK(cudaFuncSetAttribute(umma_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024));
  const int iters = 2000;
  for (int rotate = 0; rotate < 2; ++rotate)
  for (int kind = 0; kind < 2; ++kind) {
    for (int n : {64, 128, 256}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        if (kind == 0) umma_loop<0><<<sms, 128, 48 * 1024>>>(n, iters, d, rotate);
        else umma_loop<1><<<sms, 128, 48 * 1024>>>(n, iters, d, rotate);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long cyc;
        CK(cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost));
        const double macs_per_mma = 128.0 * n * (kind == 0 ? 32 : 16);
        const double total = macs_per_mma * 8 * iters;
        if (rep == 1)
          printf("rotate=%d %s M=128 N=%3d: %.0f MAC/clk/SM (%.0f cycles/MMA), chip %.2f POPS (%.3f ms)\n",
                 rotate, kind == 0 ? "i8 " : "f16", n, total / cyc, (double)cyc / (8.0 * iters),
                 2.0 * total * sms / (ms * 1e-3) / 1e15, ms);
      }
    }
  }
  CK(cudaFuncSetAttribute(ozaki_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 43008));
  for (int ce = 0; ce < 3; ++ce)
  for (int rep = 0; rep < 2; ++rep) {
    ozaki_seq<<<sms, 128, 3 * 43008>>>(1000, d, ce);
    CK(cudaDeviceSynchronize());
    unsigned long long cyc;
    CK(cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost));
    unsigned long long iss; CK(cudaMemcpy(&iss, d + 1, 8, cudaMemcpyDeviceToHost));
    if (rep) printf("ozaki 11-MMA stage (commit mode %d): %.0f cycles/stage (ideal 1104), issue done after %.0f cycles/stage\n", ce, cyc / 1000.0, iss / 1000.0);
  }
  return 0;
}
