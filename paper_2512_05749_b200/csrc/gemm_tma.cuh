// Warp-specialised TMA + mbarrier pipeline for the FP64 DMMA tall-skinny GEMMs (same contract as
// gemm_dmma_kernel in gemm.cuh: Layout::CM / Layout::RM, centring shift, alpha, split-K slabs).
//
//   warp W (the last one)  : producer - one elected lane issues cp.async.bulk.tensor (TMA) loads of
//                            the A/B tiles (and the shift slice) into a STAGES-deep ring, arming the
//                            stage's "full" mbarrier with the transaction byte count;
//   warps 0..W-1           : consumers - wait on "full", run mma.sync.m8n8k4.f64 (DMMA.8x8x4) from
//                            swizzled shared memory, then arrive on the stage's "empty" mbarrier.
// No CTA-wide barrier sits in the k-loop, so DMMA issue never waits for the slowest warp.
//
// Tiles land in shared memory through 2-D tensor maps with 16-double (128 B) inner boxes and
// SWIZZLE_128B: inside every 1 KB atom the 16-byte unit index is XORed with the line index mod 8.
// Each lane fetches pairs of doubles with LDS.128; which pair a lane owns is permuted
// (f(g) = (g>>1) | ((g&1)<<2) on the swizzled axes) so that every quarter-warp touches 8 distinct
// 16-byte bank groups - conflict-free - and the permutation is undone in the epilogue.
#pragma once
#include <cuda.h>

#include "gemm.cuh"

namespace wssr {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const CUtensorMap* map, int c0,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2}], [%3];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__host__ __device__ constexpr int fperm(int g) { return (g >> 1) | ((g & 1) << 2); }

// TA = element type of the streamed A operand (O): double, or float for the FP32 variant
// (BASELINE configs[3]).  FP32 tiles are widened to FP64 in registers, so products and sums are
// exact FP64 arithmetic on the FP32 inputs.
template <Layout L, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES,
          typename TA = double>
struct TmaCfg {
  static constexpr bool kF32 = sizeof(TA) == 4;
  static constexpr int EA = 128 / (int)sizeof(TA);  // A elements per 128-byte box line
  static constexpr int kConsumerWarps = WARPS_M * WARPS_N;
  static constexpr int kThreads = 32 * (kConsumerWarps + 1);
  static constexpr int WM = BM / WARPS_M;
  static constexpr int WN = BN / WARPS_N;
  static constexpr int MS = WM / 8;
  static constexpr int NS = WN / 8;
  static constexpr bool kCM = (L == Layout::CM);
  static constexpr int A_BYTES = BM * BK * (int)sizeof(TA);
  static constexpr int B_BYTES = BK * BN * 8;
  static constexpr int S_BYTES = kCM ? 0 : 1024;  // shift slice (BK doubles), padded
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + S_BYTES;
  static constexpr size_t kSmemBytes = (size_t)STAGE_BYTES * STAGES + 1024 /*align*/ + 256;
  static_assert(BK % 16 == 0 && BM % 16 == 0 && BN % 16 == 0, "16-double boxes");
  static_assert(WM % 16 == 0 || (!kCM && WM % 8 == 0), "warp M tile");
  static_assert(WN % 16 == 0, "warp N tile");
  static_assert(STAGE_BYTES % 1024 == 0, "swizzle atoms");
  static_assert(!kF32 || (kCM ? (WM % 32 == 0 && BM % 32 == 0) : BK % 32 == 0), "fp32 tiling");
};

// PERSIST: grid.x CTAs loop over work units u = blockIdx.x + i * gridDim.x (unit -> m-tile,
// n-tile, K split); the producer streams the next unit's tiles while the consumers finish the
// previous one, hiding pipeline fill and epilogue.  Non-persistent: one unit per CTA taken from
// (blockIdx.x, blockIdx.y, blockIdx.z), C staged through shared memory for coalesced stores.
template <Layout L, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES,
          typename TA = double, bool PERSIST = false>
__global__ void __launch_bounds__(32 * (WARPS_M * WARPS_N + 1))
    gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmS, const GemmArgs args) {
  pdl_wait();
  using Cfg = TmaCfg<L, BM, BN, BK, WARPS_M, WARPS_N, STAGES, TA>;
  constexpr bool CM = Cfg::kCM;
  constexpr bool F32 = Cfg::kF32;
  constexpr int EA = Cfg::EA;
  constexpr int MS = Cfg::MS, NS = Cfg::NS;
  constexpr int NCW = Cfg::kConsumerWarps;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)Cfg::STAGE_BYTES * STAGES);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const bool has_shift = args.shift != nullptr;
  const int64_t M = args.M, N = args.N;
  const int64_t mt = (M + BM - 1) / BM, ntl = (N + BN - 1) / BN;
  const int64_t nsplit = PERSIST ? (args.K + args.k_chunk - 1) / args.k_chunk : 1;
  const int64_t units = PERSIST ? mt * ntl * (nsplit > 0 ? nsplit : 1) : 1;
  // unit -> (m0, n0, kbeg, kend, ntiles, z)
  struct Unit {
    int64_t m0, n0, kbeg, kend;
    int ntiles;
    int64_t z;
  };
  auto unit_of = [&](int64_t u) {
    Unit w;
    if (PERSIST) {
      const int64_t mi = u % mt, rest = u / mt;
      w.m0 = mi * BM;
      w.n0 = (rest % ntl) * BN;
      w.z = rest / ntl;
    } else {
      w.m0 = (int64_t)blockIdx.x * BM;
      w.n0 = (int64_t)blockIdx.y * BN;
      w.z = blockIdx.z;
    }
    w.kbeg = w.z * args.k_chunk;
    w.kend = min(args.K, w.kbeg + args.k_chunk);
    w.ntiles = w.kend > w.kbeg ? (int)((w.kend - w.kbeg + BK - 1) / BK) : 0;
    return w;
  };
  const int64_t u_first = PERSIST ? blockIdx.x : 0;
  const int64_t u_step = PERSIST ? gridDim.x : 1;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == NCW) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      if (!CM && has_shift) prefetch_tmap(&tmS);
      const uint32_t bytes = Cfg::A_BYTES + Cfg::B_BYTES + ((!CM && has_shift) ? BK * 8 : 0);
      int64_t gi = 0;  // global stage counter across units
      for (int64_t u = u_first; u < units; u += u_step) {
        const Unit w = unit_of(u);
        const int m0 = (int)w.m0, n0 = (int)w.n0;
        for (int it = 0; it < w.ntiles; ++it, ++gi) {
          const int s = (int)(gi % STAGES);
          if (gi >= STAGES) mbar_wait(empty + s, (uint32_t)(((gi / STAGES) - 1) & 1));
          unsigned char* st = smem + (size_t)s * Cfg::STAGE_BYTES;
          const int k0 = (int)(w.kbeg + (int64_t)it * BK);
          mbar_arrive_expect_tx(full + s, bytes);
          if (CM) {
#pragma unroll
            for (int c = 0; c < BM / EA; ++c)
              tma_load_2d(st + c * (BK * 128), &tmA, m0 + EA * c, k0, full + s);
          } else {
#pragma unroll
            for (int c = 0; c < BK / EA; ++c)
              tma_load_2d(st + c * (BM * 128), &tmA, k0 + EA * c, m0, full + s);
            if (has_shift) tma_load_1d(st + Cfg::A_BYTES + Cfg::B_BYTES, &tmS, k0, full + s);
          }
#pragma unroll
          for (int c = 0; c < BN / 16; ++c)
            tma_load_2d(st + Cfg::A_BYTES + c * (BK * 128), &tmB, n0 + 16 * c, k0, full + s);
        }
      }
    }
    return;
  }

  // ------------------------------ consumers ------------------------------
  const int g = lane >> 2, t = lane & 3;
  const int fg = fperm(g);
  const int wm0 = (warp % WARPS_M) * Cfg::WM;
  const int wn0 = (warp / WARPS_M) * Cfg::WN;

  int64_t gi = 0;  // global stage counter across units (matches the producer's)
  for (int64_t u = u_first; u < units; u += u_step) {
    const Unit w = unit_of(u);
    const int64_t m0 = w.m0, n0 = w.n0, zslab = w.z;
    const int ntiles = w.ntiles;
    double acc[MS][NS][2];
  #pragma unroll
    for (int i = 0; i < MS; ++i)
  #pragma unroll
      for (int j = 0; j < NS; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    double mu[MS];
  #pragma unroll
    for (int i = 0; i < MS; ++i) {
      mu[i] = 0.0;
      if (CM && has_shift) {
        const int64_t m = F32 ? m0 + wm0 + 32 * (i >> 2) + 4 * fg + (i & 3)
                              : m0 + wm0 + 16 * (i >> 1) + 2 * fg + (i & 1);
        if (m < M) mu[i] = args.shift[m];
      }
    }

    for (int it = 0; it < ntiles; ++it, ++gi) {
      const int s = (int)(gi % STAGES);
      mbar_wait(full + s, (uint32_t)((gi / STAGES) & 1));
      const unsigned char* sA = smem + (size_t)s * Cfg::STAGE_BYTES;
      const unsigned char* sB = sA + Cfg::A_BYTES;
      if (CM) {
  #pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
          const int k = kk + t;  // row inside the box (BK rows of 128 B)
          const int sw = k & 7;
          double a[MS], b[NS];
          if constexpr (F32) {
            // one LDS.128 = 4 consecutive m of one 8-row sub-tile quartet
  #pragma unroll
            for (int i = 0; i < MS / 4; ++i) {
              const int c = (wm0 >> 5) + i;
              const float4 x = *reinterpret_cast<const float4*>(
                  sA + c * (BK * 128) + k * 128 + ((fg ^ sw) << 4));
              a[4 * i] = (double)x.x - mu[4 * i];
              a[4 * i + 1] = (double)x.y - mu[4 * i + 1];
              a[4 * i + 2] = (double)x.z - mu[4 * i + 2];
              a[4 * i + 3] = (double)x.w - mu[4 * i + 3];
            }
          } else {
  #pragma unroll
            for (int i = 0; i < MS / 2; ++i) {
              const int c = (wm0 >> 4) + i;
              const double2 x = *reinterpret_cast<const double2*>(
                  sA + c * (BK * 128) + k * 128 + ((fg ^ sw) << 4));
              a[2 * i] = x.x - mu[2 * i];
              a[2 * i + 1] = x.y - mu[2 * i + 1];
            }
          }
  #pragma unroll
          for (int j = 0; j < NS / 2; ++j) {
            const int c = (wn0 >> 4) + j;
            const double2 y = *reinterpret_cast<const double2*>(
                sB + c * (BK * 128) + k * 128 + ((fg ^ sw) << 4));
            b[2 * j] = y.x;
            b[2 * j + 1] = y.y;
          }
  #pragma unroll
          for (int i = 0; i < MS; ++i)
  #pragma unroll
            for (int j = 0; j < NS; ++j) dmma884(acc[i][j], a[i], b[j]);
        }
      } else if constexpr (F32) {
        // K-quads: lane t holds k = kk + 4t + s for MMA step s (same permutation on A and B)
        const double* sS = reinterpret_cast<const double*>(sB + Cfg::B_BYTES);
  #pragma unroll
        for (int kk = 0; kk < BK; kk += 16) {
          double sh[4] = {0.0, 0.0, 0.0, 0.0};
          if (has_shift) {
            const double2 s0 = *reinterpret_cast<const double2*>(sS + kk + 4 * t);
            const double2 s1 = *reinterpret_cast<const double2*>(sS + kk + 4 * t + 2);
            sh[0] = s0.x;
            sh[1] = s0.y;
            sh[2] = s1.x;
            sh[3] = s1.y;
          }
          const int ca = kk >> 5;
          const int unit = 4 * ((kk >> 4) & 1) + t;
          double aq[4][MS];
  #pragma unroll
          for (int i = 0; i < MS; ++i) {
            const int m = wm0 + 8 * i + fg;
            const float4 x = *reinterpret_cast<const float4*>(
                sA + ca * (BM * 128) + m * 128 + ((unit ^ fg) << 4));
            aq[0][i] = (double)x.x - sh[0];
            aq[1][i] = (double)x.y - sh[1];
            aq[2][i] = (double)x.z - sh[2];
            aq[3][i] = (double)x.w - sh[3];
          }
  #pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int kr = kk + 4 * t + q;
            double bq[NS];
  #pragma unroll
            for (int j = 0; j < NS / 2; ++j) {
              const int c = (wn0 >> 4) + j;
              const double2 y = *reinterpret_cast<const double2*>(
                  sB + c * (BK * 128) + kr * 128 + ((g ^ (kr & 7)) << 4));
              bq[2 * j] = y.x;
              bq[2 * j + 1] = y.y;
            }
  #pragma unroll
            for (int i = 0; i < MS; ++i)
  #pragma unroll
              for (int j = 0; j < NS; ++j) dmma884(acc[i][j], aq[q][i], bq[j]);
          }
        }
      } else {
        const double* sS = reinterpret_cast<const double*>(sB + Cfg::B_BYTES);
  #pragma unroll
        for (int kk = 0; kk < BK; kk += 8) {
          double2 sh = make_double2(0.0, 0.0);
          if (has_shift) sh = *reinterpret_cast<const double2*>(sS + kk + 2 * t);
          const int ca = kk >> 4;
          const int unit = 4 * ((kk >> 3) & 1) + t;
          double a0[MS], a1[MS], b0[NS], b1[NS];
  #pragma unroll
          for (int i = 0; i < MS; ++i) {
            const int m = wm0 + 8 * i + fg;  // m & 7 == fg
            const double2 x = *reinterpret_cast<const double2*>(
                sA + ca * (BM * 128) + m * 128 + ((unit ^ fg) << 4));
            a0[i] = x.x - sh.x;
            a1[i] = x.y - sh.y;
          }
          const int k0r = kk + 2 * t, k1r = k0r + 1;
  #pragma unroll
          for (int j = 0; j < NS / 2; ++j) {
            const int c = (wn0 >> 4) + j;
            const double2 y0 = *reinterpret_cast<const double2*>(
                sB + c * (BK * 128) + k0r * 128 + ((g ^ (k0r & 7)) << 4));
            const double2 y1 = *reinterpret_cast<const double2*>(
                sB + c * (BK * 128) + k1r * 128 + ((g ^ (k1r & 7)) << 4));
            b0[2 * j] = y0.x;
            b0[2 * j + 1] = y0.y;
            b1[2 * j] = y1.x;
            b1[2 * j + 1] = y1.y;
          }
  #pragma unroll
          for (int i = 0; i < MS; ++i)
  #pragma unroll
            for (int j = 0; j < NS; ++j) dmma884(acc[i][j], a0[i], b0[j]);
  #pragma unroll
          for (int i = 0; i < MS; ++i)
  #pragma unroll
            for (int j = 0; j < NS; ++j) dmma884(acc[i][j], a1[i], b1[j]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
    }

    // epilogue: undo the lane permutations into a shared-memory C tile (the operand ring is idle -
    // every TMA write has been consumed), then write rows out coalesced.  Tiles whose C block does
    // not fit the ring store straight from registers.
    constexpr int SC = BN + 1;  // odd stride
    const double alpha = args.alpha;
    auto store = [&](int64_t m, int64_t n, double val) {
      if (args.partial) {
        args.partial[(zslab * M + m) * N + n] = val;
      } else {
        double* dst = args.C + m * args.ldc + n;
        if (args.Cin)
          *dst = args.Cin[m * args.ldcin + n] + val;
        else
          *dst = args.accumulate ? *dst + val : val;
      }
    };
    if constexpr (!PERSIST && (size_t)BM * SC * 8 <= (size_t)Cfg::STAGE_BYTES * STAGES) {
      double* sC = reinterpret_cast<double*>(smem);
      asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");  // all consumers left the ring
  #pragma unroll
      for (int i = 0; i < MS; ++i) {
        const int ml = CM ? (F32 ? wm0 + 32 * (i >> 2) + 4 * fg + (i & 3)
                                 : wm0 + 16 * (i >> 1) + 2 * fg + (i & 1))
                          : wm0 + 8 * i + fg;
  #pragma unroll
        for (int j = 0; j < NS; ++j) {
  #pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int nl = CM ? wn0 + 16 * (j >> 1) + 2 * fperm(2 * t + e) + (j & 1)
                              : wn0 + 16 * (j >> 1) + 2 * (2 * t + e) + (j & 1);
            sC[ml * SC + nl] = alpha * acc[i][j][e];
          }
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"r"(NCW * 32) : "memory");
      const int rows = (int)min((int64_t)BM, M - m0), cols = (int)min((int64_t)BN, N - n0);
      for (int e = tid; e < BM * BN; e += NCW * 32) {
        const int ml = e / BN, nl = e % BN;  // BN is a power of two
        if (ml >= rows || nl >= cols) continue;
        store(m0 + ml, n0 + nl, sC[ml * SC + nl]);
      }
    } else {
  #pragma unroll
      for (int i = 0; i < MS; ++i) {
        const int64_t m = CM ? (F32 ? m0 + wm0 + 32 * (i >> 2) + 4 * fg + (i & 3)
                                    : m0 + wm0 + 16 * (i >> 1) + 2 * fg + (i & 1))
                             : m0 + wm0 + 8 * i + fg;
        if (m >= M) continue;
  #pragma unroll
        for (int j = 0; j < NS; ++j) {
  #pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int64_t n = CM ? n0 + wn0 + 16 * (j >> 1) + 2 * fperm(2 * t + e) + (j & 1)
                                 : n0 + wn0 + 16 * (j >> 1) + 2 * (2 * t + e) + (j & 1);
            if (n < N) store(m, n, alpha * acc[i][j][e]);
          }
        }
      }
    }

  }
}

}  // namespace wssr
