// Non-GEMM kernels of the WSSR step: batch statistics (estimators.py), k x k factorisations
// (CholeskyQR2 core, Jacobi eigen-solver), sorting/rank logic (svdengine.py, optimizers.py) and
// the fused low-rank-plus-floor preconditioner (optimizers.py:361-364).
#pragma once
#include "common.cuh"

namespace wssr {

// ---------------------------------------------------------------------------------------------
// Local-energy statistics and clipping: estimators.py:53-71 (clip_local_energies) and :87-92.
// One CTA. scal_out = [loss, raw_loss, mean, std].  l_scaled = (clip(E)-loss)*scale,
// l_raw = clip(E)-loss (unscaled, used by the column-statistics pass for the gradient).
// ---------------------------------------------------------------------------------------------
__global__ void energy_stats_kernel(const double* __restrict__ E, int64_t n, double n_std,
                                    int clip_enabled, double scale, double* __restrict__ l_scaled,
                                    double* __restrict__ l_raw, double* __restrict__ scal_out) {
  __shared__ double scratch[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += E[i];
  const double mean = block_sum(s, scratch) / (double)n;
  double q = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = E[i] - mean;
    q += d * d;
  }
  const double sd = sqrt(block_sum(q, scratch) / (double)n);
  const bool do_clip = clip_enabled && sd != 0.0;
  const double lo = mean - n_std * sd, hi = mean + n_std * sd;
  double c = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double e = E[i];
    if (do_clip) e = fmin(fmax(e, lo), hi);
    c += e;
  }
  const double loss = block_sum(c, scratch) / (double)n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double e = E[i];
    if (do_clip) e = fmin(fmax(e, lo), hi);
    const double r = e - loss;
    l_raw[i] = r;
    l_scaled[i] = r * scale;
  }
  if (threadIdx.x == 0) {
    scal_out[0] = loss;
    scal_out[1] = mean;
    scal_out[2] = mean;
    scal_out[3] = sd;
  }
}

// ---------------------------------------------------------------------------------------------
// Column statistics of the raw derivative block (estimators.py:91,93) in ONE pass over O:
//   mu[p]   = mean_n O[n,p]
//   m2[p]   = sum_n (O[n,p]-mu[p])^2          (-> ||o_matrix||_F^2 = sum_p m2 / N)
//   gsum[p] = sum_n (O[n,p]-mu[p]) * lraw[n]  (-> gradient = 2*gsum/N)
// CTA = 8 warps over 32 columns (lane = column); each warp owns a contiguous row chunk and
// accumulates shifted sums (shift = the chunk's first row, so the sums stay well conditioned);
// chunks are merged with Chan's pairwise update in a fixed order.
// ---------------------------------------------------------------------------------------------
constexpr int kColStatsWarps = 8;

__global__ void __launch_bounds__(32 * kColStatsWarps)
    colstats_kernel(const double* __restrict__ O, int64_t n, int64_t p, int64_t ld,
                    const double* __restrict__ lraw, double* __restrict__ mu,
                    double* __restrict__ m2, double* __restrict__ gsum) {
  __shared__ double sh[kColStatsWarps][5][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t col = (int64_t)blockIdx.x * 32 + lane;
  const bool active = col < p;
  const int64_t rows_per = (n + kColStatsWarps - 1) / kColStatsWarps;
  const int64_t r0 = min(n, (int64_t)w * rows_per), r1 = min(n, r0 + rows_per);
  double K = 0.0, s1 = 0.0, s2 = 0.0, sl = 0.0, lsum = 0.0;
  if (r1 > r0) {
    if (active) K = O[r0 * ld + col];
    const double* src = O + col;
    int64_t r = r0;
    for (; r + 4 <= r1; r += 4) {
      double x[4], l[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        x[u] = active ? __ldg(src + (r + u) * ld) : 0.0;
        l[u] = __ldg(lraw + r + u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double d = active ? x[u] - K : 0.0;
        s1 += d;
        s2 = fma(d, d, s2);
        sl = fma(d, l[u], sl);
        lsum += l[u];
      }
    }
    for (; r < r1; ++r) {
      const double x = active ? __ldg(src + r * ld) : 0.0;
      const double l = __ldg(lraw + r);
      const double d = active ? x - K : 0.0;
      s1 += d;
      s2 = fma(d, d, s2);
      sl = fma(d, l, sl);
      lsum += l;
    }
  }
  const double cnt = (double)(r1 - r0);
  double mean = 0.0, M2 = 0.0, G = 0.0;
  if (cnt > 0) {
    const double dm = s1 / cnt;
    mean = K + dm;
    M2 = fmax(s2 - s1 * dm, 0.0);
    G = sl - dm * lsum;
  }
  sh[w][0][lane] = cnt;
  sh[w][1][lane] = mean;
  sh[w][2][lane] = M2;
  sh[w][3][lane] = G;
  sh[w][4][lane] = lsum;
  __syncthreads();
  if (w == 0) {
    double na = sh[0][0][lane], ma = sh[0][1][lane], Ma = sh[0][2][lane], Ga = sh[0][3][lane],
           La = sh[0][4][lane];
    for (int c = 1; c < kColStatsWarps; ++c) {
      const double nb = sh[c][0][lane];
      if (nb == 0) continue;
      const double mb = sh[c][1][lane], Mb = sh[c][2][lane], Gb = sh[c][3][lane],
                   Lb = sh[c][4][lane];
      if (na == 0) {
        na = nb; ma = mb; Ma = Mb; Ga = Gb; La = Lb;
        continue;
      }
      const double nn = na + nb;
      const double delta = mb - ma;
      const double mnew = ma + delta * (nb / nn);
      Ma = Ma + Mb + delta * delta * (na * nb / nn);
      Ga = Ga + (ma - mnew) * La + Gb + (mb - mnew) * Lb;
      La += Lb;
      ma = mnew;
      na = nn;
    }
    if (active) {
      mu[col] = ma;
      m2[col] = Ma;
      gsum[col] = Ga;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Deterministic reductions.  reduce_partials: block b sums x[b*chunk : (b+1)*chunk] (op 0 = sum,
// 1 = sum of squares) in a fixed order; reduce_final: one block sums the block partials.
// ---------------------------------------------------------------------------------------------
__global__ void reduce_partials_kernel(const double* __restrict__ x, int64_t n, int64_t chunk,
                                       int op, double* __restrict__ partials) {
  __shared__ double scratch[32];
  const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double s = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const double v = x[i];
    s += op == 1 ? v * v : v;
  }
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}
__global__ void reduce_final_kernel(const double* __restrict__ partials, int nparts, double scale,
                                    double* __restrict__ out) {
  __shared__ double scratch[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) *out = s * scale;
}

// Row sums of squares of an (rows x cols, ld) matrix: out[r] = sqrt(sum_c x[r,c]^2) if sqrt_out.
// One block per row, fixed order.  Used for ||obar[:, j]|| (optimizers.py:370).
__global__ void row_norms_kernel(const double* __restrict__ x, int64_t cols, int64_t ld,
                                 double* __restrict__ out, int sqrt_out) {
  __shared__ double scratch[32];
  const double* row = x + (int64_t)blockIdx.x * ld;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) s = fma(row[c], row[c], s);
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt_out ? sqrt(s) : s;
}

// Sum of squares of a strided (rows x cols, ld) matrix into per-block partials (row chunks).
__global__ void matrix_sumsq_partials_kernel(const double* __restrict__ x, int64_t rows,
                                             int64_t cols, int64_t ld, int64_t rows_per_block,
                                             double* __restrict__ partials) {
  __shared__ double scratch[32];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  double s = 0.0;
  const int64_t total = (r1 - r0) * cols;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t r = r0 + e / cols, c = e % cols;
    const double v = x[r * ld + c];
    s = fma(v, v, s);
  }
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// ---------------------------------------------------------------------------------------------
// k x k Cholesky + triangular inverse for CholeskyQR2 (replaces LAPACK dgeqrf/dorgqr behind
// linalg.py:56).  G = L L^T; outputs R = L^T and Rinv = L^-T (upper, zero below diagonal).
// W is k x k scratch (shared memory when it fits, global otherwise).  status[0] is set to the
// 1-based index of the first pivot that is not safely positive (CholeskyQR2 would lose
// orthogonality there) - the host then takes the two-pass Gram-Schmidt path of
// linalg.py:64-105.  A zero matrix (trace 0) sets status[1] (ZeroMatrix, linalg.py:53-54).
// ---------------------------------------------------------------------------------------------
__device__ void chol_inv_body(const double* __restrict__ G, int k, double* W, double* dX,
                              double* __restrict__ R, double* __restrict__ Rinv,
                              int* __restrict__ status, double pivot_rel) {
  __shared__ double s_gmax, s_trace;
  __shared__ int s_fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int e = tid; e < k * k; e += nt) W[e] = G[e];
  for (int j = tid; j < k; j += nt) dX[j] = G[j * k + j];  // original diagonal
  if (tid == 0) {
    double gm = 0.0, tr = 0.0;
    for (int j = 0; j < k; ++j) {
      gm = fmax(gm, G[j * k + j]);
      tr += G[j * k + j];
    }
    s_gmax = gm;
    s_trace = tr;
    s_fail = 0;
  }
  __syncthreads();
  // |R_jj| <= 1e-12 ||A||_F is the reference's switch to the patch path (linalg.py:58-61)
  const double deficient_sq = 1.0000001e-24 * s_trace;
  if (s_gmax == 0.0 || !(s_gmax < 1.0 / 0.0)) {
    if (tid == 0) {
      if (s_gmax == 0.0) atomicExch(status + 1, 1);
      atomicCAS(status, 0, 1);
    }
    return;
  }
  // right-looking Cholesky, lower triangle in place
  for (int j = 0; j < k; ++j) {
    if (tid == 0) {
      const double d = W[j * k + j];
      // scale-invariant pivot test (Schur complement vs the column's own norm) + the
      // reference's deficiency rule; either sends the block to the careful path
      if (!(d > pivot_rel * dX[j]) || !(d > deficient_sq)) {
        s_fail = j + 1;
      } else {
        W[j * k + j] = sqrt(d);
      }
    }
    __syncthreads();
    if (s_fail) break;
    const double piv = W[j * k + j];
    for (int i = j + 1 + tid; i < k; i += nt) W[i * k + j] /= piv;
    __syncthreads();
    const int m = k - j - 1;
    for (int e = tid; e < m * m; e += nt) {
      const int i = j + 1 + e / m, l = j + 1 + e % m;
      if (l <= i) W[i * k + l] -= W[i * k + j] * W[l * k + j];
    }
    __syncthreads();
  }
  if (s_fail) {
    if (tid == 0) atomicCAS(status, 0, s_fail);
    return;
  }
  // X = L^-1 (lower): row i of X from rows < i.  X[i][j] (i>j) is stored at W[j][i].
  for (int i = 0; i < k; ++i) {
    const double lii = W[i * k + i];
    for (int j = tid; j <= i; j += nt) {
      if (j == i) {
        dX[i] = 1.0 / lii;
      } else {
        double s = 0.0;
        // sum_{l=j}^{i-1} L[i][l] * X[l][j]
        s = fma(W[i * k + j], dX[j], s);
        for (int l = j + 1; l < i; ++l) s = fma(W[i * k + l], W[j * k + l], s);
        W[j * k + i] = -s / lii;
      }
    }
    __syncthreads();
  }
  for (int e = tid; e < k * k; e += nt) {
    const int r = e / k, c = e % k;
    if (c < r) {
      R[e] = 0.0;
      Rinv[e] = 0.0;
    } else if (c == r) {
      R[e] = W[r * k + r];
      Rinv[e] = dX[r];
    } else {
      R[e] = W[c * k + r];   // L[c][r]
      Rinv[e] = W[r * k + c];  // X[c][r]
    }
  }
}

__global__ void chol_inv_smem_kernel(const double* G, int k, double* R, double* Rinv, int* status,
                                     double pivot_rel) {
  extern __shared__ __align__(16) double smem[];
  chol_inv_body(G, k, smem, smem + k * k, R, Rinv, status, pivot_rel);
}
__global__ void chol_inv_gmem_kernel(const double* G, int k, double* W, double* R, double* Rinv,
                                     int* status, double pivot_rel) {
  chol_inv_body(G, k, W, W + (size_t)k * k, R, Rinv, status, pivot_rel);
}

// C = A * B for k x k upper-triangular A, B (row-major, ld k).
__global__ void triu_mul_kernel(const double* __restrict__ A, const double* __restrict__ B, int k,
                                double* __restrict__ C) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const int r = e / k, c = e % k;
  double s = 0.0;
  for (int l = r; l <= c; ++l) s = fma(A[r * k + l], B[l * k + c], s);
  C[e] = (c < r) ? 0.0 : s;
}

// ---------------------------------------------------------------------------------------------
// sigma = |diag R_v| sorted descending with a stable argsort, positive prefix, rank cut:
// svdengine.py:144-150 and optimizers.py:348-349.  One CTA.
// ints_out = [k_pos, r_eff]; order_out[k]; sigma_out[k] (sorted).
// ---------------------------------------------------------------------------------------------
__global__ void sort_sigma_kernel(const double* __restrict__ Rv, int k, double r_reg,
                                  int64_t* __restrict__ order_out, double* __restrict__ sigma_out,
                                  int* __restrict__ ints_out) {
  extern __shared__ double sd[];
  for (int i = threadIdx.x; i < k; i += blockDim.x) sd[i] = Rv[i * k + i];
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double si = sd[i];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double sj = sd[j];
      rank += (sj > si) || (sj == si && j < i);
    }
    order_out[rank] = i;
    sigma_out[rank] = si;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int kp = 0;
    double top = 0.0;
    for (int r = 0; r < k; ++r) {
      const double s = sigma_out[r];
      if (s > 0.0) ++kp;
    }
    int reff = 0;
    if (kp > 0) {
      top = sigma_out[0] * sigma_out[0];
      for (int r = 0; r < kp; ++r) {
        const double s = sigma_out[r];
        if (s * s >= r_reg * top) ++reff;
      }
    }
    ints_out[0] = kp;
    ints_out[1] = reff;
  }
}

// out[r, j] = in[r, order[j]] for j < kk  (column gather; svdengine.py:151-152)
__global__ void gather_cols_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows,
                                   const int64_t* __restrict__ order, int kk,
                                   double* __restrict__ out, int64_t ldo) {
  const int64_t total = rows * kk;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / kk;
    const int j = (int)(e % kk);
    out[r * ldo + j] = in[r * ldi + order[j]];
  }
}

// strided 2-D copy (rows x cols), optional scale
__global__ void copy2d_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows,
                              int64_t cols, double scale, double* __restrict__ out, int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    out[r * ldo + c] = scale * in[r * ldi + c];
  }
}

// out (cols x rows, ld_out) = (in (rows x cols) * diag(colscale))^T.  obar = u * sigma
// (optimizers.py:378) written parameter-contiguous so it is the next step's history block.
__global__ void transpose_scale_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows,
                                       int cols, const double* __restrict__ colscale,
                                       double* __restrict__ out, int64_t ldo) {
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i;
    const int c = c0 + tx;
    tile[i][tx] = (r < rows && c < cols) ? in[r * ldi + c] * colscale[c] : 0.0;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i;
    const int64_t r = r0 + tx;
    if (c < cols && r < rows) out[(int64_t)c * ldo + r] = tile[tx][i];
  }
}

// y[i] = a*x[i] + b*y[i]
__global__ void axpby_kernel(int64_t n, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i] + (b == 0.0 ? 0.0 : b * y[i]);
}

// ---------------------------------------------------------------------------------------------
// Fused preconditioner apply + parameter update (optimizers.py:361-364):
//   update = U (c / sigma^2) + (gbar - U c) / floor ;  theta' = theta - eta * update
// c = U^T gbar is computed beforehand by a split-K DMMA GEMM.  One warp per parameter row.
// ---------------------------------------------------------------------------------------------
__global__ void precond_update_kernel(const double* __restrict__ U, int64_t ldu, int64_t P, int r,
                                      const double* __restrict__ c,
                                      const double* __restrict__ sigma,
                                      const double* __restrict__ gbar, double inv_floor,
                                      const double* __restrict__ theta, double eta,
                                      double* __restrict__ theta_out,
                                      double* __restrict__ update_out) {
  extern __shared__ double sc[];  // [2r]: c/sigma^2, c
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    const double s = sigma[j];
    sc[j] = c[j] / (s * s);
    sc[r + j] = c[j];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < P; p += warps) {
    const double* row = U + p * ldu;
    double a = 0.0, b = 0.0;
    for (int j = lane; j < r; j += 32) {
      const double x = row[j];
      a = fma(x, sc[j], a);
      b = fma(x, sc[r + j], b);
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      const double upd = a + (gbar[p] - b) * inv_floor;
      if (update_out) update_out[p] = upd;
      theta_out[p] = theta[p] - eta * upd;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Largest eigenvalue of a symmetric k x k matrix by parallel cyclic Jacobi (one CTA; round-robin
// pairing so k/2 rotations run concurrently).  Gives ||U2 - U1 (U1^T U2)||_2^2 for the projector
// drift (svdengine.py:217-221) from the k x k Gram of the out-of-span block.
// ---------------------------------------------------------------------------------------------
__device__ void jacobi_maxeig_body(const double* __restrict__ Ain, int k, double* A, int* perm,
                                   double* out) {
  __shared__ double s_off, s_tot;
  __shared__ double scratch[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int kk = k + (k & 1);  // pad to even with a dummy index
  for (int e = tid; e < kk * kk; e += nt) {
    const int r = e / kk, c = e % kk;
    A[e] = (r < k && c < k) ? 0.5 * (Ain[r * k + c] + Ain[c * k + r]) : 0.0;
  }
  for (int i = tid; i < kk; i += nt) perm[i] = i;
  __syncthreads();
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int e = tid; e < kk * kk; e += nt) {
      const int r = e / kk, c = e % kk;
      const double v = A[e] * A[e];
      tot += v;
      if (r != c) off += v;
    }
    off = block_sum(off, scratch);
    tot = block_sum(tot, scratch);
    if (tid == 0) {
      s_off = off;
      s_tot = tot;
    }
    __syncthreads();
    if (!(s_off > 1e-30 * s_tot) || s_tot == 0.0) break;
    for (int round = 0; round < kk - 1; ++round) {
      // pairs (perm[i], perm[kk-1-i]) for i < kk/2: compute rotation per pair then apply to rows
      // and columns in two phases.
      __shared__ double cs[2 * 256 + 2];
      for (int i = tid; i < kk / 2; i += nt) {
        int p = perm[i], q = perm[kk - 1 - i];
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        const double apq = A[p * kk + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double app = A[p * kk + p], aqq = A[q * kk + q];
          const double tau = (aqq - app) / (2.0 * apq);
          const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + tt * tt);
          s = tt * c;
        }
        cs[2 * i] = c;
        cs[2 * i + 1] = s;
      }
      __syncthreads();
      // rows: for each pair, rotate rows p,q across all columns
      for (int e = tid; e < (kk / 2) * kk; e += nt) {
        const int i = e / kk, col = e % kk;
        int p = perm[i], q = perm[kk - 1 - i];
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        const double c = cs[2 * i], s = cs[2 * i + 1];
        const double ap = A[p * kk + col], aq = A[q * kk + col];
        A[p * kk + col] = c * ap - s * aq;
        A[q * kk + col] = s * ap + c * aq;
      }
      __syncthreads();
      for (int e = tid; e < (kk / 2) * kk; e += nt) {
        const int i = e / kk, row = e % kk;
        int p = perm[i], q = perm[kk - 1 - i];
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        const double c = cs[2 * i], s = cs[2 * i + 1];
        const double ap = A[row * kk + p], aq = A[row * kk + q];
        A[row * kk + p] = c * ap - s * aq;
        A[row * kk + q] = s * ap + c * aq;
      }
      __syncthreads();
      // round-robin: keep perm[0], rotate the rest
      if (tid == 0) {
        const int last = perm[kk - 1];
        for (int i = kk - 1; i > 1; --i) perm[i] = perm[i - 1];
        perm[1] = last;
      }
      __syncthreads();
    }
  }
  double mx = -1.0 / 0.0;
  for (int i = tid; i < k; i += nt) mx = fmax(mx, A[i * kk + i]);
  mx = block_max(mx, scratch);
  if (tid == 0) *out = mx;
}

__global__ void jacobi_maxeig_smem_kernel(const double* Ain, int k, double* out) {
  extern __shared__ __align__(16) double smem[];
  const int kk = k + (k & 1);
  jacobi_maxeig_body(Ain, k, smem, reinterpret_cast<int*>(smem + kk * kk), out);
}
__global__ void jacobi_maxeig_gmem_kernel(const double* Ain, int k, double* W, double* out) {
  extern __shared__ int perm_sm[];
  jacobi_maxeig_body(Ain, k, W, perm_sm, out);
}

// ||a[:r] - b[:r]||_2 and the off-diagonal Frobenius norm of a k x k matrix (svdengine.py:216,
// svdengine.py:140).  One CTA.
__global__ void small_norms_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                   int r, const double* __restrict__ Q, int k,
                                   double* __restrict__ out) {
  __shared__ double scratch[32];
  double s = 0.0;
  if (a) {
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
      const double d = a[i] - b[i];
      s = fma(d, d, s);
    }
  }
  s = block_sum(s, scratch);
  double o = 0.0;
  if (Q) {
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
      if (e / k != e % k) o = fma(Q[e], Q[e], o);
    }
  }
  o = block_sum(o, scratch);
  if (threadIdx.x == 0) {
    out[0] = sqrt(s);
    out[1] = sqrt(o);
  }
}

}  // namespace wssr
