// Device producer of O: the parameter log-derivatives of the pooled-feature determinant ansatz,
// AceWavefunction.grad_theta_batch (wavefunction.py:307-321), for a batch of walkers - so a VMC
// loop uploads the walker positions (W x N x 3) instead of O (W x N T, 4.3 GB per step at c1).
//
// Per walker w (one CTA):
//   phi[i][o]    = exp(-zeta_o r) r^n_o [x_axis(o)] gate_o(spin_i),  r = |x_i - R_center(o)|
//                  (orbital_values, wavefunction.py:143-178)
//   pooled[i][o] = sum_j phi[j][o] - phi[i][o]                     (wavefunction.py:265)
//   F[i][t]      = phi[i][head_t] prod_{p in tail_t} pooled[i][p]   (wavefunction.py:266-272)
//   M[i][k]      = sum_t F[i][t] C[k][t]                            (wavefunction.py:280-282)
//   slogdet(M): sign 0 or log|det| < -700 -> node flag (NodeProximity, wavefunction.py:317-318)
//   O[w][k T + t] = sum_i inv(M)[k][i] F[i][t]                      (wavefunction.py:319-321)
// F is staged in the walker's output row itself (N T doubles, exactly O's row) and transformed in
// place column by column.  M is inverted by Gauss-Jordan with partial pivoting in shared memory.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "engine.h"
#include "producer.h"

namespace wssr {
namespace prod {

constexpr int kThreads = 256;
constexpr int kTile = 128;  // feature columns per tile of the F C^T contraction (at most)
constexpr int kMaxPairs = 16;  // (i, k) pairs of M per thread: n_electrons <= 64
constexpr double kLogAbsUnderflow = -700.0;  // system.py:16

__global__ void __launch_bounds__(kThreads)
    grad_theta_kernel(const wssr_ace_spec s, const double* __restrict__ pos, int64_t W,
                      double* __restrict__ out, int64_t ldo, int* __restrict__ node_flag,
                      int tile) {
  pdl_wait();
  const int64_t w = blockIdx.x;
  if (w >= W) return;
  const int N = (int)s.n_electrons, NO = (int)s.n_orbitals, T = (int)s.n_features;
  const int MT = (int)s.max_tail;
  extern __shared__ __align__(16) double sm[];
  double* phi = sm;                      // N x NO
  double* pooled = phi + N * NO;         // N x NO
  double* Mx = pooled + N * NO;          // N x (2N): [M | I] -> [I | M^-1]
  double* Fs = Mx + 2 * N * N;           // N x (tile + 1): a tile of F (padded rows)
  double* Cs = Fs + N * (tile + 1);      // N x (tile + 1): the same tile of C
  __shared__ double s_logabs;
  __shared__ int s_sing;
  const int tid = threadIdx.x;
  const double* xw = pos + w * (int64_t)N * 3;
  double* ow = out + w * ldo;

  // phi
  for (int e = tid; e < N * NO; e += kThreads) {
    const int i = e / NO, o = e % NO;
    const int c = s.orb_center[o];
    const double dx = xw[3 * i] - s.nuclei[3 * c], dy = xw[3 * i + 1] - s.nuclei[3 * c + 1],
                 dz = xw[3 * i + 2] - s.nuclei[3 * c + 2];
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    double v = exp(-s.orb_zeta[o] * r);
    for (int q = 0; q < s.orb_n[o]; ++q) v *= r;
    const int ax = s.orb_axis[o];
    if (ax >= 0) v *= (ax == 0 ? dx : (ax == 1 ? dy : dz));
    const int gate = s.orb_gate[o];  // 0 up, 1 down, 2 either
    const int up = s.spins[i] == 0;
    const double gv = gate == 2 ? 1.0 : (gate == 0 ? (up ? 1.0 : 0.0) : (up ? 0.0 : 1.0));
    phi[e] = v * gv;
  }
  __syncthreads();
  // pooled: column sums minus own row
  for (int e = tid; e < N * NO; e += kThreads) {
    const int i = e / NO, o = e % NO;
    double tot = 0.0;
    for (int j = 0; j < N; ++j) tot += phi[j * NO + o];
    pooled[e] = tot - phi[i * NO + o];
  }
  __syncthreads();
  // Features into the output row (F[i][t] at ow[i T + t]) and M = F C^T, tile by tile: each
  // tile of F is computed into shared memory (and written out once for the O pass below), the
  // matching tile of C (L2-resident: every walker reads it) is staged beside it, and every
  // thread accumulates its (i, k) entries of M from the two tiles (rows padded: conflict-free).
  const int npairs = N * N;
  double acc[kMaxPairs];
#pragma unroll
  for (int j = 0; j < kMaxPairs; ++j) acc[j] = 0.0;
  for (int t0 = 0; t0 < T; t0 += tile) {
    for (int e = tid; e < N * tile; e += kThreads) {
      const int i = e / tile, tt = e % tile, t = t0 + tt;
      double f = 0.0, c = 0.0;
      if (t < T) {
        f = phi[i * NO + s.heads[t]];
        for (int q = 0; q < MT; ++q) {
          const int p = s.tails[(int64_t)t * MT + q];
          if (p < 0) break;
          f *= pooled[i * NO + p];
        }
        ow[(int64_t)i * T + t] = f;
        c = s.coef[(int64_t)i * T + t];  // C has the same N x T shape
      }
      Fs[i * (tile + 1) + tt] = f;
      Cs[i * (tile + 1) + tt] = c;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kMaxPairs; ++j) {
      const int pr = tid + j * kThreads;
      if (pr < npairs) {
        const double* fr = Fs + (pr / N) * (tile + 1);
        const double* cr = Cs + (pr % N) * (tile + 1);
        double a = acc[j];
        for (int tt = 0; tt < tile; ++tt) a = fma(fr[tt], cr[tt], a);
        acc[j] = a;
      }
    }
    __syncthreads();
  }
  // M augmented with I
#pragma unroll
  for (int j = 0; j < kMaxPairs; ++j) {
    const int pr = tid + j * kThreads;
    if (pr < npairs) {
      const int i = pr / N, k = pr % N;
      Mx[i * 2 * N + k] = acc[j];
      Mx[i * 2 * N + N + k] = (i == k) ? 1.0 : 0.0;
    }
  }
  if (tid == 0) {
    s_logabs = 0.0;
    s_sing = 0;
  }
  __syncthreads();
  // Gauss-Jordan with partial pivoting (row swaps), log|det| = sum log|pivot|
  __shared__ int s_piv;
  for (int col = 0; col < N; ++col) {
    if (tid == 0) {
      int best = col;
      double bv = fabs(Mx[col * 2 * N + col]);
      for (int r = col + 1; r < N; ++r) {
        const double a = fabs(Mx[r * 2 * N + col]);
        if (a > bv) {
          bv = a;
          best = r;
        }
      }
      s_piv = best;
      if (bv == 0.0) s_sing = 1;
      else s_logabs += log(bv);
    }
    __syncthreads();
    if (s_sing) break;
    const int pr = s_piv;
    if (pr != col) {
      for (int c = tid; c < 2 * N; c += kThreads) {
        const double a = Mx[col * 2 * N + c];
        Mx[col * 2 * N + c] = Mx[pr * 2 * N + c];
        Mx[pr * 2 * N + c] = a;
      }
      __syncthreads();
    }
    // eliminate with the unscaled pivot row (multiplier m_r = a_r,col / pivot, as LU does: two
    // identical rows cancel exactly and give an exact zero pivot, the reference's sign 0), then
    // scale the pivot row
    const double pv = Mx[col * 2 * N + col];
    for (int e = tid; e < N * 2 * N; e += kThreads) {
      const int r = e / (2 * N), c = e % (2 * N);
      if (r == col || c == col) continue;
      const double f = Mx[r * 2 * N + col] / pv;
      Mx[e] = fma(-f, Mx[col * 2 * N + c], Mx[e]);
    }
    __syncthreads();
    for (int r = tid; r < N; r += kThreads)
      if (r != col) Mx[r * 2 * N + col] = 0.0;
    const double inv = 1.0 / pv;
    for (int c = tid; c < 2 * N; c += kThreads) Mx[col * 2 * N + c] *= inv;
    __syncthreads();
  }
  if (s_sing || s_logabs < kLogAbsUnderflow) {
    if (tid == 0) atomicExch(node_flag, 1);
    return;
  }
  // O[k][t] = sum_i inv[k][i] F[i][t], column by column in place
  double fcol[64];
  for (int t = tid; t < T; t += kThreads) {
    for (int i = 0; i < N; ++i) fcol[i] = ow[(int64_t)i * T + t];
    for (int k = 0; k < N; ++k) {
      double a = 0.0;
      for (int i = 0; i < N; ++i) a = fma(Mx[k * 2 * N + N + i], fcol[i], a);
      ow[(int64_t)k * T + t] = a;
    }
  }
}

}  // namespace prod

size_t grad_theta_smem(const wssr_ace_spec& s, int tile) {
  return sizeof(double) *
         (2 * (size_t)s.n_electrons * s.n_orbitals + 2 * (size_t)s.n_electrons * s.n_electrons +
          2 * (size_t)s.n_electrons * (tile + 1));
}

// the widest feature tile (<= 128) whose staging fits beside the per-walker tables
int grad_theta_tile(const wssr_ace_spec& s) {
  int tile = prod::kTile;
  while (tile > 8 && grad_theta_smem(s, tile) > (size_t)200 * 1024) tile /= 2;
  return tile;
}

cudaError_t grad_theta(Context& ctx, const wssr_ace_spec& s, const double* positions, int64_t W,
                       double* out, int64_t ldo, int* node_flag) {
  if (W <= 0) return cudaSuccess;
  const int tile = grad_theta_tile(s);
  const size_t smem = grad_theta_smem(s, tile);
  cudaError_t e = cudaFuncSetAttribute(prod::grad_theta_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(prod::grad_theta_kernel, (unsigned)W, prod::kThreads, smem, ctx.stream, s,
                 positions, W, out, ldo, node_flag, tile);
  ctx.kernel_launches += 1;
  return e;
}

}  // namespace wssr
