// FP64 tensor-core (DMMA) tall-skinny GEMMs for the WSSR subspace iteration.
//
// Two operand layouts cover every contraction on the hot path:
//
//   Layout::CM  C(M x N) = alpha * sum_k (A(k,m) - shift[m]) * B(k,n),  A stored [K][M] (row k
//               contiguous in m).  Used for u = Ohat v  (svdengine.py:134; A = O rows, K = samples,
//               M = params, shift = column mean mu) and for every Gram / cross-product X^T Y over
//               the parameter axis (svdengine.py:137-138, linalg.py:56 via CholeskyQR2,
//               optimizers.py:361, svdengine.py:220).
//   Layout::RM  C(M x N) = alpha * sum_k (A(m,k) - shift[k]) * B(k,n),  A stored [M][K] (row m
//               contiguous in k).  Used for v = Ohat^T q (svdengine.py:133; A = O, M = samples,
//               K = params, shift = mu) and for the small right-multiplications X * R^-1 / X * C.
//
// Centring (estimators.py:91) is applied in registers on the A fragment, and the 1/sqrt(N) and
// sqrt(1-delta) scales (estimators.py:90, optimizers.py:322) are folded into alpha, so the
// reference's centred/transposed/concatenated copies of O are never materialised.
//
// Tiles are staged global->shared with cp.async (LDGSTS, zero-filled at the edges) through a
// STAGES-deep ring, then fed to mma.sync.m8n8k4.f64 (DMMA.8x8x4; tcgen05 has no f64 kind on
// sm_100a).  Shared rows are padded so that every fragment load is a conflict-free LDS.128:
// each lane loads a pair of doubles and the pair's two halves feed two different 8-wide
// sub-tiles (an M/N permutation inside the warp tile, undone in the epilogue), or - for the
// RM A operand - two consecutive k-steps (a K permutation applied identically to A and B).
//
// Split-K: blockIdx.z owns k in [z*k_chunk, min(K,(z+1)*k_chunk)); with `partial` set every
// split writes its own slab and splitk_reduce() sums the slabs in a fixed order, so results are
// bitwise reproducible run to run (reference determinism contract, test_svdengine.py:124-132).
#pragma once
#include "common.cuh"

namespace wssr {

enum class Layout : int { CM = 0, RM = 1 };

struct GemmArgs {
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  const double* shift;
  double* C;
  int64_t ldc;
  int64_t M, N, K;
  int64_t k_chunk;
  double alpha;
  int accumulate;
  double* partial;
  const double* Cin;  // optional: result = Cin + alpha*acc (ld = ldcin); used when !partial
  int64_t ldcin;
};

__host__ __device__ constexpr int pad_doubles(int base, int mod_bytes, int target_bytes) {
  int p = 0;
  while (((base + p) * 8) % mod_bytes != target_bytes) ++p;
  return p;
}

template <Layout L, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
struct GemmCfg {
  static constexpr int kThreads = 32 * WARPS_M * WARPS_N;
  static constexpr int WM = BM / WARPS_M;
  static constexpr int WN = BN / WARPS_N;
  static constexpr int MS = WM / 8;  // 8-row sub-tiles per warp
  static constexpr int NS = WN / 8;  // 8-col sub-tiles per warp
  static constexpr bool kCM = (L == Layout::CM);
  // shared strides (doubles); see the bank analysis in the file header
  static constexpr int SA = kCM ? BM + pad_doubles(BM, 128, 32) : BK + pad_doubles(BK, 128, 64);
  static constexpr int SB = kCM ? BN + pad_doubles(BN, 128, 32) : BN + pad_doubles(BN, 64, 16);
  static constexpr int A_STAGE = kCM ? BK * SA : BM * SA;
  static constexpr int B_STAGE = BK * SB;
  static constexpr int S_STAGE = kCM ? 0 : BK;
  static constexpr int STAGE = A_STAGE + B_STAGE + S_STAGE;
  static constexpr size_t kSmemBytes = sizeof(double) * (size_t)STAGE * STAGES;
  static_assert(WM % 16 == 0 || (!kCM && WM % 8 == 0), "warp M tile");
  static_assert(WN % 16 == 0, "warp N tile must hold sub-tile pairs");
  static_assert(BK % 8 == 0, "BK multiple of 8");
};

template <int VEC>
__device__ __forceinline__ void load_chunk(double* dst, const double* base, const double* src,
                                           int nvalid) {
  if (VEC == 2) {
    cp_async16(dst, nvalid > 0 ? src : base, nvalid * 8);
  } else {
    cp_async8(dst, nvalid > 0 ? src : base, nvalid * 8);
  }
}

template <Layout L, int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int VA, int VB>
__global__ void __launch_bounds__(32 * WARPS_M * WARPS_N)
    gemm_dmma_kernel(const GemmArgs args) {
  pdl_wait();
  using Cfg = GemmCfg<L, BM, BN, BK, WARPS_M, WARPS_N, STAGES>;
  constexpr bool CM = Cfg::kCM;
  constexpr int NT = Cfg::kThreads;
  constexpr int MS = Cfg::MS, NS = Cfg::NS;
  extern __shared__ __align__(16) double smem[];

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % WARPS_M) * Cfg::WM;
  const int wn0 = (warp / WARPS_M) * Cfg::WN;

  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = (int64_t)blockIdx.y * BN;
  const int64_t kbeg = (int64_t)blockIdx.z * args.k_chunk;
  const int64_t kend = min(args.K, kbeg + args.k_chunk);
  const int ntiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

  const double* __restrict__ A = args.A;
  const double* __restrict__ B = args.B;
  const double* __restrict__ shift = args.shift;
  const bool has_shift = shift != nullptr;
  const int64_t M = args.M, N = args.N;

  auto load_stage = [&](int slot, int64_t k0) {
    double* sA = smem + (size_t)slot * Cfg::STAGE;
    double* sB = sA + Cfg::A_STAGE;
    if (CM) {
      constexpr int CPR = BM / VA;  // chunks per row
      for (int c = tid; c < BK * CPR; c += NT) {
        const int r = c / CPR, cc = c % CPR;
        const int64_t k = k0 + r, m = m0 + (int64_t)cc * VA;
        int nv = (k < kend) ? (int)max((int64_t)0, min((int64_t)VA, M - m)) : 0;
        load_chunk<VA>(sA + r * Cfg::SA + cc * VA, A, A + k * args.lda + m, nv);
      }
    } else {
      constexpr int CPR = BK / VA;
      for (int c = tid; c < BM * CPR; c += NT) {
        const int r = c / CPR, cc = c % CPR;
        const int64_t m = m0 + r, k = k0 + (int64_t)cc * VA;
        int nv = (m < M) ? (int)max((int64_t)0, min((int64_t)VA, kend - k)) : 0;
        load_chunk<VA>(sA + r * Cfg::SA + cc * VA, A, A + m * args.lda + k, nv);
      }
      if (has_shift) {
        double* sS = sB + Cfg::B_STAGE;
        for (int c = tid; c < BK; c += NT) {
          const int64_t k = k0 + c;
          cp_async8(sS + c, k < kend ? shift + k : shift, k < kend ? 8 : 0);
        }
      }
    }
    {
      constexpr int CPR = BN / VB;
      for (int c = tid; c < BK * CPR; c += NT) {
        const int r = c / CPR, cc = c % CPR;
        const int64_t k = k0 + r, n = n0 + (int64_t)cc * VB;
        int nv = (k < kend) ? (int)max((int64_t)0, min((int64_t)VB, N - n)) : 0;
        load_chunk<VB>(sB + r * Cfg::SB + cc * VB, B, B + k * args.ldb + n, nv);
      }
    }
  };

  double acc[MS][NS][2];
#pragma unroll
  for (int i = 0; i < MS; ++i)
#pragma unroll
    for (int j = 0; j < NS; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // CM: the centring shift is indexed by m, which is fixed per lane -> registers.
  double mu[MS];
#pragma unroll
  for (int i = 0; i < MS; ++i) {
    mu[i] = 0.0;
    if (CM && has_shift) {
      const int64_t m = m0 + wm0 + 16 * (i >> 1) + 2 * g + (i & 1);
      if (m < M) mu[i] = shift[m];
    }
  }

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) load_stage(s, kbeg + (int64_t)s * BK);
    cp_async_commit();
  }

  for (int it = 0; it < ntiles; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nx = it + STAGES - 1;
      if (nx < ntiles) load_stage(nx % STAGES, kbeg + (int64_t)nx * BK);
      cp_async_commit();
    }
    const double* sA = smem + (size_t)(it % STAGES) * Cfg::STAGE;
    const double* sB = sA + Cfg::A_STAGE;
    if (CM) {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        double a[MS], b[NS];
        const double* ra = sA + (kk + t) * Cfg::SA + wm0 + 2 * g;
        const double* rb = sB + (kk + t) * Cfg::SB + wn0 + 2 * g;
#pragma unroll
        for (int i = 0; i < MS / 2; ++i) {
          const double2 x = *reinterpret_cast<const double2*>(ra + 16 * i);
          a[2 * i] = x.x - mu[2 * i];
          a[2 * i + 1] = x.y - mu[2 * i + 1];
        }
#pragma unroll
        for (int j = 0; j < NS / 2; ++j) {
          const double2 y = *reinterpret_cast<const double2*>(rb + 16 * j);
          b[2 * j] = y.x;
          b[2 * j + 1] = y.y;
        }
#pragma unroll
        for (int i = 0; i < MS; ++i)
#pragma unroll
          for (int j = 0; j < NS; ++j) dmma884(acc[i][j], a[i], b[j]);
      }
    } else {
      const double* sS = sB + Cfg::B_STAGE;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 8) {
        double2 sh = make_double2(0.0, 0.0);
        if (has_shift) sh = *reinterpret_cast<const double2*>(sS + kk + 2 * t);
        double a0[MS], a1[MS], b0[NS], b1[NS];
#pragma unroll
        for (int i = 0; i < MS; ++i) {
          const double2 x =
              *reinterpret_cast<const double2*>(sA + (wm0 + 8 * i + g) * Cfg::SA + kk + 2 * t);
          a0[i] = x.x - sh.x;
          a1[i] = x.y - sh.y;
        }
        const double* rb0 = sB + (kk + 2 * t) * Cfg::SB + wn0 + 2 * g;
        const double* rb1 = rb0 + Cfg::SB;
#pragma unroll
        for (int j = 0; j < NS / 2; ++j) {
          const double2 y0 = *reinterpret_cast<const double2*>(rb0 + 16 * j);
          const double2 y1 = *reinterpret_cast<const double2*>(rb1 + 16 * j);
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
  }
  cp_async_wait<0>();

  // epilogue: undo the intra-warp M/N permutations and store
  const double alpha = args.alpha;
#pragma unroll
  for (int i = 0; i < MS; ++i) {
    const int64_t m = CM ? m0 + wm0 + 16 * (i >> 1) + 2 * g + (i & 1) : m0 + wm0 + 8 * i + g;
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t n = n0 + wn0 + 16 * (j >> 1) + 4 * t + 2 * e + (j & 1);
        if (n >= N) continue;
        const double val = alpha * acc[i][j][e];
        if (args.partial) {
          args.partial[((int64_t)blockIdx.z * M + m) * N + n] = val;
        } else {
          double* dst = args.C + m * args.ldc + n;
          if (args.Cin)
            *dst = args.Cin[m * args.ldcin + n] + val;
          else
            *dst = args.accumulate ? *dst + val : val;
        }
      }
    }
  }
}

// Few slabs (S <= 8): one thread per output, slabs summed in order; bandwidth-bound.
static __global__ void __launch_bounds__(256)
    splitk_reduce_few_kernel(const double* __restrict__ partial, int S, int64_t M, int64_t N,
                             double* __restrict__ C, int64_t ldc, double alpha, int accumulate,
                             const double* __restrict__ Cin, int64_t ldcin) {
  pdl_wait();
  const int64_t total = M * N;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double s = partial[idx];
    for (int z = 1; z < S; ++z) s += partial[(int64_t)z * total + idx];
    const int64_t m = idx / N, n = idx % N;
    double* dst = C + m * ldc + n;
    const double val = alpha * s;
    *dst = Cin ? Cin[m * ldcin + n] + val : (accumulate ? *dst + val : val);
  }
}

// C(m,n) = alpha * sum_{z<S} partial[z][m][n]  (+ C if accumulate).
// Block = 8 warps x 32 lanes: lane <-> 32 consecutive outputs (coalesced), warp w sums the slabs
// z = w, w+8, ... in order, then warp partials are added in warp order - a fixed order, so the
// result is bitwise reproducible while S up to a few hundred slabs stays latency-cheap.
static __global__ void __launch_bounds__(256)
    splitk_reduce_kernel(const double* __restrict__ partial, int S, int64_t M, int64_t N,
                         double* __restrict__ C, int64_t ldc, double alpha, int accumulate,
                         const double* __restrict__ Cin, int64_t ldcin) {
  pdl_wait();
  __shared__ double red[8][33];
  const int64_t total = M * N;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = (int64_t)blockIdx.x * 32; base < total; base += (int64_t)gridDim.x * 32) {
    const int64_t idx = base + lane;
    double s = 0.0;
    if (idx < total) {
      int z = w;
      for (; z + 24 < S; z += 32) {
        const double a0 = partial[(int64_t)z * total + idx];
        const double a1 = partial[(int64_t)(z + 8) * total + idx];
        const double a2 = partial[(int64_t)(z + 16) * total + idx];
        const double a3 = partial[(int64_t)(z + 24) * total + idx];
        s += a0;
        s += a1;
        s += a2;
        s += a3;
      }
      for (; z < S; z += 8) s += partial[(int64_t)z * total + idx];
    }
    red[w][lane] = s;
    __syncthreads();
    if (w == 0 && idx < total) {
      double t = red[0][lane];
#pragma unroll
      for (int q = 1; q < 8; ++q) t += red[q][lane];
      const int64_t m = idx / N, n = idx % N;
      double* dst = C + m * ldc + n;
      const double val = alpha * t;
      *dst = Cin ? Cin[m * ldcin + n] + val : (accumulate ? *dst + val : val);
    }
    __syncthreads();
  }
}

}  // namespace wssr
