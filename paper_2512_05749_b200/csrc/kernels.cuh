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
  pdl_wait();
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

// VEC columns per lane (VEC = 2: 16-byte loads, a warp streams 512 contiguous bytes per row);
// UNROLL rows in flight per lane so each SM keeps >= 64 KB of loads outstanding.
template <typename T, int VEC, int UNROLL>
__global__ void __launch_bounds__(32 * kColStatsWarps, 2)
    colstats_kernel(const T* __restrict__ O, int64_t n, int64_t p, int64_t ld,
                    const double* __restrict__ lraw, double* __restrict__ mu,
                    double* __restrict__ m2, double* __restrict__ gsum,
                    double* __restrict__ cmin, double* __restrict__ cmax) {
  pdl_wait();
  __shared__ double sh[kColStatsWarps][5][32 * VEC];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t col0 = (int64_t)blockIdx.x * (32 * VEC) + (int64_t)lane * VEC;
  bool act[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) act[v] = col0 + v < p;
  const int64_t rows_per = (n + kColStatsWarps - 1) / kColStatsWarps;
  const int64_t r0 = min(n, (int64_t)w * rows_per), r1 = min(n, r0 + rows_per);
  // samples stay in their storage type until used (FP32: half the registers, so twice the rows
  // in flight); extrema are exact in that type
  double K[VEC], s1[VEC], s2[VEC], sl[VEC];
  T mn[VEC], mx[VEC];
  double lsum = 0.0;
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    K[v] = s1[v] = s2[v] = sl[v] = 0.0;
    mn[v] = (T)(1.0 / 0.0);
    mx[v] = (T)(-1.0 / 0.0);
  }
  auto load = [&](int64_t r, T (&x)[VEC]) {
    if constexpr (sizeof(T) == 8 && VEC == 2) {
      if (act[VEC - 1]) {
        const double2 y = __ldg(reinterpret_cast<const double2*>(O + r * ld + col0));
        x[0] = y.x;
        x[VEC - 1] = y.y;
        return;
      }
    } else if constexpr (sizeof(T) == 4 && VEC == 4) {
      if (act[VEC - 1]) {
        const float4 y = __ldg(reinterpret_cast<const float4*>(O + r * ld + col0));
        x[0] = y.x;
        x[1 % VEC] = y.y;
        x[2 % VEC] = y.z;
        x[3 % VEC] = y.w;
        return;
      }
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) x[v] = act[v] ? __ldg(O + r * ld + col0 + v) : (T)0;
  };
  if (r1 > r0) {
    T x0[VEC];
    load(r0, x0);
#pragma unroll
    for (int v = 0; v < VEC; ++v) K[v] = act[v] ? (double)x0[v] : 0.0;
    int64_t r = r0;
    for (; r + UNROLL <= r1; r += UNROLL) {
      T x[UNROLL][VEC];
      double l[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        load(r + u, x[u]);
        l[u] = __ldg(lraw + r + u);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        lsum += l[u];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const double d = act[v] ? (double)x[u][v] - K[v] : 0.0;
          s1[v] += d;
          s2[v] = fma(d, d, s2[v]);
          sl[v] = fma(d, l[u], sl[v]);
          mn[v] = x[u][v] < mn[v] ? x[u][v] : mn[v];  // (no NaN propagation)
          mx[v] = x[u][v] > mx[v] ? x[u][v] : mx[v];
        }
      }
    }
    for (; r < r1; ++r) {
      T x[VEC];
      load(r, x);
      const double l = __ldg(lraw + r);
      lsum += l;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const double d = act[v] ? (double)x[v] - K[v] : 0.0;
        s1[v] += d;
        s2[v] = fma(d, d, s2[v]);
        sl[v] = fma(d, l, sl[v]);
        mn[v] = x[v] < mn[v] ? x[v] : mn[v];
        mx[v] = x[v] > mx[v] ? x[v] : mx[v];
      }
    }
  }
  const double cnt = (double)(r1 - r0);
#pragma unroll
  for (int v = 0; v < VEC; ++v) {
    double mean = 0.0, M2 = 0.0, G = 0.0;
    if (cnt > 0) {
      const double dm = s1[v] / cnt;
      mean = K[v] + dm;
      M2 = fmax(s2[v] - s1[v] * dm, 0.0);
      G = sl[v] - dm * lsum;
    }
    const int c = lane * VEC + v;
    sh[w][0][c] = cnt;
    sh[w][1][c] = mean;
    sh[w][2][c] = M2;
    sh[w][3][c] = G;
    sh[w][4][c] = lsum;
  }
  __syncthreads();
  // Chan merge of the row chunks, fixed order, one thread per column
  for (int c = threadIdx.x; c < 32 * VEC; c += blockDim.x) {
    const int64_t col = (int64_t)blockIdx.x * (32 * VEC) + c;
    if (col >= p) continue;
    double na = sh[0][0][c], ma = sh[0][1][c], Ma = sh[0][2][c], Ga = sh[0][3][c],
           La = sh[0][4][c];
    for (int q = 1; q < kColStatsWarps; ++q) {
      const double nb = sh[q][0][c];
      if (nb == 0) continue;
      const double mb = sh[q][1][c], Mb = sh[q][2][c], Gb = sh[q][3][c], Lb = sh[q][4][c];
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
    mu[col] = ma;
    m2[col] = Ma;
    gsum[col] = Ga;
  }
  if (cmin) {  // column extrema (scale table of the int8 tensor-core O-passes), order-free
    __syncthreads();
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      sh[w][0][lane * VEC + v] = (double)mn[v];
      sh[w][1][lane * VEC + v] = (double)mx[v];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 32 * VEC; c += blockDim.x) {
      const int64_t col = (int64_t)blockIdx.x * (32 * VEC) + c;
      if (col >= p) continue;
      double a = sh[0][0][c], b = sh[0][1][c];
      for (int q = 1; q < kColStatsWarps; ++q) {
        a = fmin(a, sh[q][0][c]);
        b = fmax(b, sh[q][1][c]);
      }
      cmin[col] = a;
      cmax[col] = b;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Deterministic reductions.  reduce_partials: block b sums x[b*chunk : (b+1)*chunk] (op 0 = sum,
// 1 = sum of squares) in a fixed order; reduce_final: one block sums the block partials.
// ---------------------------------------------------------------------------------------------
__global__ void reduce_partials_kernel(const double* __restrict__ x, int64_t n, int64_t chunk,
                                       int op, double* __restrict__ partials) {
  pdl_wait();
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
  pdl_wait();
  __shared__ double scratch[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += partials[i];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) *out = s * scale;
}

// Row norms of an (rows x cols, ld) matrix, two levels: block (r, b) sums the b-th chunk of row r
// into partial[r * nb + b]; row_norms_final sums the nb chunks in order.  Used for ||obar[:, j]||
// (optimizers.py:370), where rows are P = 10^5..10^6 long.
__global__ void row_sumsq_partials_kernel(const double* __restrict__ x, int64_t cols, int64_t ld,
                                          int64_t chunk, double* __restrict__ partial) {
  pdl_wait();
  __shared__ double scratch[32];
  const int64_t r = blockIdx.y, b = blockIdx.x;
  const double* row = x + r * ld;
  const int64_t c0 = b * chunk, c1 = min(cols, c0 + chunk);
  double s0 = 0.0, s1 = 0.0;
  int64_t c = c0 + threadIdx.x;
  for (; c + blockDim.x < c1; c += 2 * blockDim.x) {
    const double a0 = row[c], a1 = row[c + blockDim.x];
    s0 = fma(a0, a0, s0);
    s1 = fma(a1, a1, s1);
  }
  if (c < c1) s0 = fma(row[c], row[c], s0);
  const double s = block_sum(s0 + s1, scratch);
  if (threadIdx.x == 0) partial[r * gridDim.x + b] = s;
}
__global__ void row_norms_final_kernel(const double* __restrict__ partial, int nb, int rows,
                                       double* __restrict__ out, int sqrt_out) {
  pdl_wait();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += partial[(int64_t)r * nb + b];
  out[r] = sqrt_out ? sqrt(s) : s;
}

// Sum of squares of a strided (rows x cols, ld) matrix into per-block partials (row chunks).
// Dense rows (ld == cols) are streamed as one flat vector.
__global__ void matrix_sumsq_partials_kernel(const double* __restrict__ x, int64_t rows,
                                             int64_t cols, int64_t ld, int64_t rows_per_block,
                                             double* __restrict__ partials) {
  pdl_wait();
  __shared__ double scratch[32];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  double s0 = 0.0, s1 = 0.0;
  if (ld == cols) {
    const double* base = x + r0 * cols;
    const int64_t n = (r1 - r0) * cols;
    int64_t e = threadIdx.x;
    for (; e + blockDim.x < n; e += 2 * blockDim.x) {
      const double a0 = base[e], a1 = base[e + blockDim.x];
      s0 = fma(a0, a0, s0);
      s1 = fma(a1, a1, s1);
    }
    if (e < n) s0 = fma(base[e], base[e], s0);
  } else {
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const double v = x[r * ld + c];
        s0 = fma(v, v, s0);
      }
  }
  const double s = block_sum(s0 + s1, scratch);
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
// k x k Cholesky + triangular inverse for CholeskyQR2 (replaces LAPACK dgeqrf/dorgqr behind
// linalg.py:56).  One CTA of 256 threads laid out as a 16 x 16 grid; right-looking sweeps with two
// block barriers per column and no integer division in the inner loops (the k^3 work is spread
// over the grid, the k-long dependency chain costs ~2k cheap barriers).
//   G = L L^T  ->  R = L^T, Rinv = L^-T (upper, zero below the diagonal).
// W is k x (k+1) scratch (odd stride).  status[0] = 1-based index of the first pivot that is not
// safely positive (CholeskyQR2 would lose orthogonality there: the host re-runs the block on the
// Gram-Schmidt path of linalg.py:64-105); status[1] = zero matrix (linalg.py:53-54).
// PACKED: X = L^-1 (lower triangular, like L) lives transposed in the unused upper part of W,
// X[i][c] at W[c][i + 1] (the odd stride k + 1 leaves column k free), so one k x (k + 1) array
// holds both and k = 128 fits in shared memory (133 KB) instead of falling to global scratch.
template <bool PACKED>
__device__ void chol_inv_body(const double* __restrict__ G, int k, double* W, double* X,
                              double* dorig, double* __restrict__ R, double* __restrict__ Rinv,
                              int* __restrict__ status, double pivot_rel,
                              const double* __restrict__ dref = nullptr,
                              const double* __restrict__ tref = nullptr, int pivot_base = 0) {
  __shared__ double s_gmax, s_trace;
  __shared__ int s_fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 grid (blockDim.x == 256)
  const int ld = k + 1;
  auto XA = [&](int i, int c) -> double& { return PACKED ? W[c * ld + i + 1] : X[i * ld + c]; };
  for (int r = ty; r < k; r += 16)
    for (int c = tx; c < k; c += 16) {
      if (!PACKED || c <= r) W[r * ld + c] = G[r * k + c];
      if (!PACKED || c <= r) XA(r, c) = (r == c) ? 1.0 : 0.0;
    }
  // dref / tref (a diagonal block of a larger Gram, see chol_inv_blocked2 in engine.cu): the
  // pivot tests refer to the ORIGINAL diagonal entries of these rows and to the whole trace
  for (int j = tid; j < k; j += nt) dorig[j] = dref ? dref[j] : G[j * k + j];
  __syncthreads();
  if (tid == 0) {  // from shared memory: a serial loop over global loads would cost ~k x 600 cycles
    double gm = 0.0, tr = 0.0;
    for (int j = 0; j < k; ++j) {
      gm = fmax(gm, dorig[j]);
      tr += dorig[j];
    }
    s_gmax = gm;
    s_trace = tref ? *tref : tr;
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
  // Fused sweep, two barriers per column j:
  //   A: scale column j of L by 1/sqrt(pivot) and row j of X = L^-1 by the same factor;
  //   B: rank-1 trailing update of W (columns j < c <= i) and elimination of X (columns c <= j).
  // The thread that produces W[j+1][j+1] in phase B checks the next pivot and precomputes its
  // square root and inverse, so no thread waits on sqrt/div at the top of a step.
  __shared__ double s_sq, s_inv;
  auto pivot = [&](int j, double d) {
    if (!(d > pivot_rel * dorig[j]) || !(d > deficient_sq)) {
      s_fail = j + 1;
    } else {
      const double y = fast_rsqrt(d);
      s_sq = d * y;
      s_inv = y;
    }
  };
  if (tid == 0) pivot(0, W[0]);
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (s_fail) break;
    const double inv = s_inv;
    for (int i = j + 1 + tid; i < k; i += nt) W[i * ld + j] *= inv;
    for (int c = tid; c <= j; c += nt) XA(j, c) *= inv;
    if (tid == 0) W[j * ld + j] = s_sq;
    __syncthreads();
    for (int i = j + 1 + ty; i < k; i += 16) {
      const double lij = W[i * ld + j];
      double* wi = W + i * ld;
      for (int c = tx; c <= i; c += 16) {
        if (c <= j) {
          XA(i, c) = fma(-lij, XA(j, c), XA(i, c));
        } else {
          const double nv = fma(-lij, W[c * ld + j], wi[c]);
          wi[c] = nv;
          if (c == j + 1 && i == j + 1) pivot(j + 1, nv);
        }
      }
    }
    __syncthreads();
  }
  if (s_fail) {
    if (tid == 0) atomicCAS(status, 0, s_fail + pivot_base);
    return;
  }
  for (int r = ty; r < k; r += 16)
    for (int c = tx; c < k; c += 16) {
      const int e = r * k + c;
      if (c < r) {
        R[e] = 0.0;
        Rinv[e] = 0.0;
      } else {
        R[e] = W[c * ld + r];     // L[c][r]
        Rinv[e] = XA(c, r);       // X[c][r]
      }
    }
}

constexpr double kCholSeriesMax = 1e-5;  // ||G - I||_max below which the series path is taken

// Series Cholesky + inverse of a near-identity k x k Gram (k <= 64), one CTA of 256 threads.
// w holds the thread's 4 x 4 slice of G (rows ty + 16 a, columns tx + 16 b, identity-padded).
// buf: 2 x 64 x 65 doubles of shared memory.
__device__ __forceinline__ void chol_series(const double (&w)[4][4], double em, int k,
                                         double* __restrict__ R, double* __restrict__ Rinv,
                                         double* buf) {
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  constexpr int LD = 65;
  double* X = buf;
  double* Y = buf + 64 * LD;
  // With e = k em >= ||E||_2: X0 = U(E) is off by O(e^2) and each correction gains a factor e,
  // so n corrections leave e^(n+2); the Neumann sum to (-X)^J leaves e^(J+1).  Both are taken
  // below 1e-20 (FP64 resolves 1e-16 of the unit diagonal): em = 1e-12 (a typical second
  // CholeskyQR2 pass) needs no correction and one Horner product.
  const double lg = log10(fmax(em * (double)k, 1e-300));
  const int corr = em == 0.0 ? 0 : max(0, (int)ceil(-20.0 / lg) - 2);
  const int horner = em == 0.0 ? 0 : max(1, (int)ceil(-20.0 / lg) - 1);
  double e[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      e[a][b] = w[a][b] - (i == c ? 1.0 : 0.0);
      X[i * LD + c] = i < c ? e[a][b] : (i == c ? 0.5 * e[a][b] : 0.0);
    }
  __syncthreads();
  for (int it = 0; it < corr; ++it) {  // X <- U(E - X^T X)
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int m = 0; m < 64; ++m) {
      double xa[4], xb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xa[a] = X[m * LD + ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) xb[b] = X[m * LD + tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(xa[a], xb[b], acc[a][b]);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * a, c = tx + 16 * b;
        const double v = e[a][b] - acc[a][b];
        X[i * LD + c] = i < c ? v : (i == c ? 0.5 * v : 0.0);
      }
    __syncthreads();
  }
  // Y = sum_{j <= horner} (-X)^j by Horner: Y <- I - X Y, `horner` times
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      // the first Horner step from Y = I is Y = I - X (X I is exact): no product
      Y[i * LD + c] = (i == c ? 1.0 : 0.0) - (horner > 0 ? X[i * LD + c] : 0.0);
    }
  __syncthreads();
  for (int it = 1; it < horner; ++it) {
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int m = 0; m < 64; ++m) {
      double xa[4], yb[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) xa[a] = X[(ty + 16 * a) * LD + m];
#pragma unroll
      for (int b = 0; b < 4; ++b) yb[b] = Y[m * LD + tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(xa[a], yb[b], acc[a][b]);
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * a, c = tx + 16 * b;
        Y[i * LD + c] = (i == c ? 1.0 : 0.0) - acc[a][b];
      }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      if (i < k && c < k) {
        R[i * k + c] = i <= c ? (i == c ? 1.0 : 0.0) + X[i * LD + c] : 0.0;
        Rinv[i * k + c] = i <= c ? Y[i * LD + c] : 0.0;
      }
    }
}

// k <= 64: the matrix is padded to 64 x 64 with an identity tail and loaded in a 16 x 16 thread
// grid (thread (ty, tx) holds rows {ty + 16 a} x columns {tx + 16 b}); a near-identity Gram
// takes the series path, any other the blocked sweep below (same pivot tests and status codes as
// the generic chol_inv_body).
__global__ void __launch_bounds__(256) chol_inv_reg64_kernel(const double* __restrict__ G, int k,
                                                             double* __restrict__ R,
                                                             double* __restrict__ Rinv,
                                                             int* __restrict__ status,
                                                             double pivot_rel, int use_series,
                                                             long long* prof = nullptr) {
  pdl_wait();
  extern __shared__ double series_buf[];  // 2 x 64 x 65 doubles when use_series
  __shared__ double dg[64];
  __shared__ double s_tr, s_gmax;
  __shared__ int s_fail;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double w[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, c = tx + 16 * b;
      w[a][b] = (i < k && c < k) ? G[i * k + c] : (i == c ? 1.0 : 0.0);
    }
  if (tid < 64) dg[tid] = tid < k ? G[tid * k + tid] : 1.0;
  __syncthreads();
  {
    // Near-identity Gram (the second pass of CholeskyQR2): R = I + X with X upper triangular,
    // X + X^T + X^T X = E = G - I, solved by X <- U(E - X^T X) (U: strict upper part plus half
    // the diagonal), and R^-1 = sum_j (-X)^j.  Each iteration gains one order of ||E||, so a
    // handful of 64 x 64 products replace the 64-step dependent Cholesky sweep.
    double em = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = ty + 16 * a, c = tx + 16 * b;
        // NaN/Inf entries force em = +inf (fmax would drop a NaN): such a Gram takes the
        // blocked sweep, whose pivot test reports it
        const double d = fabs(w[a][b] - (i == c ? 1.0 : 0.0));
        em = d <= 1.79769313486231570e308 ? fmax(em, d) : __longlong_as_double(0x7ff0000000000000ll);
      }
    __shared__ double red_em[8];
    em = warp_max(em);
    if ((tid & 31) == 0) red_em[tid >> 5] = em;
    __syncthreads();
    if (tid < 32) {
      double v = tid < 8 ? red_em[tid] : 0.0;
      v = warp_max(v);
      if (tid == 0) red_em[0] = v;
    }
    __syncthreads();
    em = red_em[0];
    if (use_series && em < kCholSeriesMax) {
      chol_series(w, em, k, R, Rinv, series_buf);
      return;
    }
  }
  // ---- blocked right-looking Cholesky (8-column panels) + blocked triangular inverse ----------
  // Warp 0 factorises each 64 x 8 panel in registers (pivot by shuffle, one rsqrt per column);
  // all 256 threads then apply the panel's rank-8 update to the trailing block.  The inverse
  // X = L^-1 is formed by 8x8 blocks: the 8 diagonal blocks in parallel (one warp each), then
  // block rows i = 1..7 with X_ij = -X_ii sum_{m=j}^{i-1} L_im X_mj.  Shared memory: L and X,
  // 64 x 65 doubles each (the series path's buffer).
  constexpr int LD = 65;
  double* Ls = series_buf;
  double* Xs = series_buf + 64 * LD;
  __shared__ double s_invd[64];
  __shared__ double T[64 * 8];  // block-row scratch: T_ij rows (8 per block) x 8
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) Ls[(ty + 16 * a) * LD + tx + 16 * b] = w[a][b];
  if (tid == 0) {
    double gm = 0.0, tr = 0.0;
    for (int jj = 0; jj < k; ++jj) {
      gm = fmax(gm, dg[jj]);
      tr += dg[jj];
    }
    s_gmax = gm;
    s_tr = tr;
    s_fail = (!(gm > 0.0) || !(gm < 1.0 / 0.0)) ? -1 : 0;
  }
  __syncthreads();
  if (s_fail < 0) {
    if (tid == 0) {
      if (s_gmax == 0.0) atomicExch(status + 1, 1);
      atomicCAS(status, 0, 1);
    }
    return;
  }
  const double defic = 1.0000001e-24 * s_tr;
  for (int p = 0; p < 8; ++p) {
    const int c0 = 8 * p;
    if (warp == 0) {
      double pv[2][8];
      const int r0 = c0 + lane, r1 = c0 + lane + 32;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        pv[0][jj] = r0 < 64 ? Ls[r0 * LD + c0 + jj] : 0.0;
        pv[1][jj] = r1 < 64 ? Ls[r1 * LD + c0 + jj] : 0.0;
      }
      int fail = 0;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int cj = c0 + jj;
        const double d = __shfl_sync(0xffffffffu, pv[0][jj], jj);
        if (cj < k && (!(d > pivot_rel * dg[cj]) || !(d > defic))) {
          fail = cj + 1;
          break;
        }
        const double y = fast_rsqrt(d), sq = d * y;
        // column jj of L (rows above the pivot are not part of L)
        pv[0][jj] = lane > jj ? pv[0][jj] * y : (lane == jj ? sq : 0.0);
        pv[1][jj] = pv[1][jj] * y;
        if (lane == 0) s_invd[cj] = y;
        // rank-1 update of the panel's remaining columns: L[r][jj] L[c0 + jn][jj]
#pragma unroll
        for (int jn = jj + 1; jn < 8; ++jn) {
          const double lc = __shfl_sync(0xffffffffu, pv[0][jj], jn);
          pv[0][jn] = fma(-pv[0][jj], lc, pv[0][jn]);
          pv[1][jn] = fma(-pv[1][jj], lc, pv[1][jn]);
        }
      }
      if (fail) {
        if (lane == 0) s_fail = fail;
      } else {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          if (r0 < 64) Ls[r0 * LD + c0 + jj] = pv[0][jj];
          if (r1 < 64) Ls[r1 * LD + c0 + jj] = pv[1][jj];
        }
      }
    }
    __syncthreads();
    if (s_fail) {
      if (tid == 0) atomicCAS(status, 0, s_fail);
      return;
    }
    // trailing update W[r][c] -= sum_jj L[r][c0+jj] L[c][c0+jj], r, c >= c0 + 8 (full square)
    const int t0 = c0 + 8, m = 64 - t0;
    if (m > 0) {
      const int rl = tid >> 2, cg = tid & 3;
      if (rl < m) {
        const int r = t0 + rl;
        double lr[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) lr[jj] = Ls[r * LD + c0 + jj];
        for (int cl = cg; cl < m; cl += 8) {  // two columns per pass: independent chains
          const int c = t0 + cl, c2 = c + 4;
          const bool two = cl + 4 < m;
          double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll
          for (int jj = 0; jj < 8; jj += 2) {
            a0 = fma(lr[jj], Ls[c * LD + c0 + jj], a0);
            a1 = fma(lr[jj + 1], Ls[c * LD + c0 + jj + 1], a1);
            if (two) {
              b0 = fma(lr[jj], Ls[c2 * LD + c0 + jj], b0);
              b1 = fma(lr[jj + 1], Ls[c2 * LD + c0 + jj + 1], b1);
            }
          }
          Ls[r * LD + c] -= a0 + a1;
          if (two) Ls[r * LD + c2] -= b0 + b1;
        }
      }
    }
    __syncthreads();
  }
  // ---- X = L^-1: diagonal blocks (warp w inverts block w; lane c < 8 owns column c) ---------
  {
    const int b0 = 8 * warp;
    if (lane < 8) {
      const int c = lane;
      double xc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double acc = (i == c) ? 1.0 : 0.0;
#pragma unroll
        for (int mm = 0; mm < i; ++mm) acc = fma(-Ls[(b0 + i) * LD + b0 + mm], xc[mm], acc);
        xc[i] = i < c ? 0.0 : acc * s_invd[b0 + i];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) Xs[(b0 + i) * LD + b0 + c] = xc[i];
    }
  }
  __syncthreads();
  // block rows i = 1..7: T_ij = sum_{m=j}^{i-1} L_im X_mj, then X_ij = -X_ii T_ij (j < i)
  for (int bi = 1; bi < 8; ++bi) {
    const int r0 = 8 * bi, ncol = 8 * bi;  // columns 0 .. 8 bi - 1 of block row bi
    // T (8 rows x ncol columns): thread per entry
    for (int e = tid; e < 8 * ncol; e += 256) {
      const int rr = e / ncol, cc = e % ncol;  // cc in block bj = cc / 8
      const int mstart = cc & ~7;  // a multiple of 8, as is r0: whole 8-blocks of the sum
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const double* lrow = Ls + (r0 + rr) * LD;
      for (int mm = mstart; mm < r0; mm += 4) {  // 4 independent chains
        a0 = fma(lrow[mm], Xs[mm * LD + cc], a0);
        a1 = fma(lrow[mm + 1], Xs[(mm + 1) * LD + cc], a1);
        a2 = fma(lrow[mm + 2], Xs[(mm + 2) * LD + cc], a2);
        a3 = fma(lrow[mm + 3], Xs[(mm + 3) * LD + cc], a3);
      }
      T[rr * 64 + cc] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();
    for (int e = tid; e < 8 * ncol; e += 256) {
      const int rr = e / ncol, cc = e % ncol;
      double acc = 0.0;
#pragma unroll
      for (int mm = 0; mm < 8; ++mm) acc = fma(Xs[(r0 + rr) * LD + r0 + mm], T[mm * 64 + cc], acc);
      Xs[(r0 + rr) * LD + cc] = -acc;
    }
    __syncthreads();
  }
  // R = L^T, Rinv = X^T (upper triangular), k x k
  for (int e = tid; e < k * k; e += 256) {
    const int r = e / k, c = e % k;  // output row r, column c
    R[e] = (c >= r) ? Ls[c * LD + r] : 0.0;
    Rinv[e] = (c >= r) ? Xs[c * LD + r] : 0.0;
  }
}

__host__ __device__ inline size_t chol_scratch_doubles(int k) {
  return 2 * (size_t)k * (k + 1) + (size_t)k;
}
__host__ __device__ inline size_t chol_packed_doubles(int k) {
  return (size_t)k * (k + 1) + (size_t)k;
}

__global__ void __launch_bounds__(256) chol_inv_smem_kernel(const double* G, int k, double* R,
                                                            double* Rinv, int* status,
                                                            double pivot_rel) {
  pdl_wait();
  extern __shared__ __align__(16) double smem[];
  double* W = smem;
  double* X = W + (size_t)k * (k + 1);
  chol_inv_body<false>(G, k, W, X, X + (size_t)k * (k + 1), R, Rinv, status, pivot_rel);
}
// L and L^-1 packed into one k x (k + 1) shared array (k <= ~160)
// Near-identity Grams (the second pass of CholeskyQR2, G = I + E with k max|E| <= 1e-9) skip the
// sweep: with X = U(E) (strict upper part plus half the diagonal), R = I + X satisfies
// R^T R = I + E + X^T X and R^-1 = I - X + X^2 - ..., so R = I + X and R^-1 = I - X hold to
// k max|E|^2 <= 1e-18 (the first-order case of chol_series for k <= 64).
constexpr double kCholFirstOrderMax = 1e-9;
__global__ void __launch_bounds__(256) chol_inv_packed_kernel(const double* G, int k, double* R,
                                                              double* Rinv, int* status,
                                                              double pivot_rel, int use_series,
                                                              const double* dref,
                                                              const double* tref,
                                                              int pivot_base) {
  pdl_wait();
  extern __shared__ __align__(16) double smem[];
  double* W = smem;
  if (use_series) {
    double em = 0.0;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
      const double d = fabs(G[e] - (e / k == e % k ? 1.0 : 0.0));
      // NaN/Inf entries force em = +inf (fmax would drop a NaN): the sweep's pivot test reports
      em = d <= 1.79769313486231570e308 ? fmax(em, d) : __longlong_as_double(0x7ff0000000000000ll);
    }
    em = block_max(em, W);
    if (em * k <= kCholFirstOrderMax) {
      for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int r = e / k, c = e % k;
        const double x = c > r ? G[e] : 0.5 * (G[e] - 1.0);
        R[e] = c > r ? x : (c == r ? 1.0 + x : 0.0);
        Rinv[e] = c > r ? -x : (c == r ? 1.0 - x : 0.0);
      }
      return;
    }
  }
  chol_inv_body<true>(G, k, W, nullptr, W + (size_t)k * (k + 1), R, Rinv, status, pivot_rel, dref,
                      tref, pivot_base);
}

// ---- pieces of the two-block Cholesky for 160 < k <= 256 (engine.cu chol_inv_blocked2) ----------
// diag[j] = G_jj, diag[k] = trace(G)
__global__ void chol_diag_trace_kernel(const double* __restrict__ G, int k,
                                       double* __restrict__ diag) {
  pdl_wait();
  __shared__ double scratch[32];
  double t = 0.0;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const double d = G[(size_t)j * k + j];
    diag[j] = d;
    t += d;
  }
  t = block_sum(t, scratch);
  if (threadIdx.x == 0) diag[k] = t;
}
// C (m x n, ldc) = C0 + alpha A B for small operands given by element strides (a transpose is a
// stride swap): A(i, q) = A[i a_rs + q a_cs], B(q, j) = B[q b_rs + j b_cs]; C0 may be null.
// 16 x 16 tiles, fixed summation order.
__global__ void __launch_bounds__(256)
    small_gemm_kernel(int m, int n, int kk, const double* __restrict__ A, int64_t a_rs,
                      int64_t a_cs, const double* __restrict__ B, int64_t b_rs, int64_t b_cs,
                      const double* __restrict__ C0, int64_t c0_ld, double alpha,
                      double* __restrict__ C, int64_t ldc) {
  pdl_wait();
  __shared__ double sa[16][17], sb[16][17];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i = blockIdx.y * 16 + ty, j = blockIdx.x * 16 + tx;
  double acc = 0.0;
  for (int q0 = 0; q0 < kk; q0 += 16) {
    sa[ty][tx] = (i < m && q0 + tx < kk) ? A[i * a_rs + (q0 + tx) * a_cs] : 0.0;
    sb[ty][tx] = (q0 + ty < kk && j < n) ? B[(q0 + ty) * b_rs + j * b_cs] : 0.0;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = fma(sa[ty][q], sb[q][tx], acc);
    __syncthreads();
  }
  if (i < m && j < n) C[i * ldc + j] = (C0 ? C0[i * c0_ld + j] : 0.0) + alpha * acc;
}
// R = [[R11, R12], [0, R22]], R^-1 = [[R11i, T], [0, R22i]] (k x k, row-major) from the blocks
__global__ void chol_assemble2_kernel(int k, int h, const double* __restrict__ R11,
                                      const double* __restrict__ R11i,
                                      const double* __restrict__ R12, const double* __restrict__ T,
                                      const double* __restrict__ R22,
                                      const double* __restrict__ R22i, double* __restrict__ R,
                                      double* __restrict__ Rinv) {
  pdl_wait();
  const int k2 = k - h;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < k * k; e += gridDim.x * blockDim.x) {
    const int r = e / k, c = e % k;
    double a, b;
    if (r < h && c < h) {
      a = R11[r * h + c];
      b = R11i[r * h + c];
    } else if (r < h) {
      a = R12[r * k2 + (c - h)];
      b = T[r * k2 + (c - h)];
    } else if (c < h) {
      a = b = 0.0;
    } else {
      a = R22[(r - h) * k2 + (c - h)];
      b = R22i[(r - h) * k2 + (c - h)];
    }
    R[e] = a;
    Rinv[e] = b;
  }
}
__global__ void __launch_bounds__(256) chol_inv_gmem_kernel(const double* G, int k, double* ws,
                                                            double* R, double* Rinv, int* status,
                                                            double pivot_rel) {
  pdl_wait();
  double* W = ws;
  double* X = W + (size_t)k * (k + 1);
  chol_inv_body<false>(G, k, W, X, X + (size_t)k * (k + 1), R, Rinv, status, pivot_rel);
}

// C = A * B for k x k upper-triangular A, B (row-major, ld k).
__global__ void triu_mul_kernel(const double* __restrict__ A, const double* __restrict__ B, int k,
                                double* __restrict__ C) {
  pdl_wait();
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
  pdl_wait();
  extern __shared__ double sd[];
  // NaN keys (a failed factorisation upstream, the with-fallback pass) sort last: the order is a
  // permutation whatever the values, so the column gathers below never index out of range
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double v = Rv[i * k + i];
    sd[i] = isnan(v) ? -INFINITY : v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const double si = sd[i];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double sj = sd[j];
      rank += (sj > si) || (sj == si && j < i);
    }
    order_out[rank] = i;
    sigma_out[rank] = Rv[i * k + i];
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
  pdl_wait();
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
  pdl_wait();
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
  pdl_wait();
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
  pdl_wait();
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
  pdl_wait();
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
// Largest eigenvalue of a symmetric k x k matrix (one CTA): Householder reduction to
// tridiagonal form, then Sturm-count multisection on the tridiagonal (every thread evaluates the
// inertia at its own shift, 256-way per round).  Gives ||U2 - U1 (U1^T U2)||_2^2 for the
// projector drift (svdengine.py:217-221) from the k x k Gram of the out-of-span block.
__device__ void maxeig_body(const double* __restrict__ Ain, int k, double* A, double* vbuf,
                            double* out) {
  __shared__ double scratch[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ld = k + 1;      // odd stride: conflict-free row-parallel matvec
  double* v = vbuf;          // [k] Householder vector
  double* p = vbuf + k;      // [k]
  double* dg = vbuf + 2 * k; // [k] diagonal
  double* od = vbuf + 3 * k; // [k] off-diagonal (od[j] couples j and j+1)
  for (int r = tid >> 4; r < k; r += 16)
    for (int c = tid & 15; c < k; c += 16) A[r * ld + c] = 0.5 * (Ain[r * k + c] + Ain[c * k + r]);
  __syncthreads();
  for (int j = 0; j + 2 < k; ++j) {
    const int n = k - j - 1;  // length of x = A[j+1:, j]
    double s = 0.0;
    for (int i = tid; i < n; i += nt) {
      const double x = A[(j + 1 + i) * ld + j];
      s = fma(x, x, s);
    }
    const double xnorm2 = block_sum(s, scratch);
    const double x0 = A[(j + 1) * ld + j];
    const double xn = sqrt(xnorm2);
    const double alpha = x0 >= 0.0 ? -xn : xn;
    // v = x - alpha e1, beta = 2 / v^T v  (v^T v = 2 xn (xn + |x0|))
    const double vtv = 2.0 * xn * (xn + fabs(x0));
    for (int i = tid; i < n; i += nt) v[i] = A[(j + 1 + i) * ld + j] - (i == 0 ? alpha : 0.0);
    if (tid == 0) {
      dg[j] = A[j * ld + j];
      od[j] = (vtv > 0.0) ? alpha : x0;
    }
    __syncthreads();
    if (!(vtv > 0.0)) continue;  // column already reduced
    const double beta = 2.0 * fast_rcp(vtv);
    // p = beta * A' v  (A' = trailing n x n block)
    for (int i = tid; i < n; i += nt) {
      const double* row = A + (j + 1 + i) * ld + (j + 1);
      double q = 0.0;
      for (int l = 0; l < n; ++l) q = fma(row[l], v[l], q);
      p[i] = beta * q;
    }
    __syncthreads();
    double t = 0.0;
    for (int i = tid; i < n; i += nt) t = fma(v[i], p[i], t);
    const double Kc = 0.5 * beta * block_sum(t, scratch);
    // A' -= v w^T + w v^T,  w = p - K v   (16 x 16 thread grid, no integer division)
    {
      const int tx = tid & 15, ty = tid >> 4;
      for (int r = ty; r < n; r += 16) {
        const double vr = v[r], wr = p[r] - Kc * v[r];
        double* Arow = A + (j + 1 + r) * ld + (j + 1);
        for (int c = tx; c < n; c += 16) Arow[c] -= vr * (p[c] - Kc * v[c]) + wr * v[c];
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (k >= 2) {
      dg[k - 2] = A[(k - 2) * ld + (k - 2)];
      od[k - 2] = A[(k - 1) * ld + (k - 2)];
    }
    dg[k - 1] = A[(k - 1) * ld + (k - 1)];
  }
  __syncthreads();
  // Gershgorin bracket, then multisection on the largest eigenvalue:
  // count(x) = #eigenvalues < x from the signs of the LDL^T pivots of T - x I.
  __shared__ double s_lo, s_hi;
  __shared__ int s_best;
  if (tid == 0) {
    double lo = 1.0 / 0.0, hi = -1.0 / 0.0;
    for (int i = 0; i < k; ++i) {
      const double r = (i > 0 ? fabs(od[i - 1]) : 0.0) + (i + 1 < k ? fabs(od[i]) : 0.0);
      lo = fmin(lo, dg[i] - r);
      hi = fmax(hi, dg[i] + r);
    }
    s_lo = lo;
    s_hi = hi;
  }
  __syncthreads();
  for (int round = 0; round < 12; ++round) {
    const double lo = s_lo, hi = s_hi;
    if (!(hi - lo > 2e-16 * fmax(fabs(hi), fabs(lo)))) break;
    // thread t tests x_t = lo + (t+1) (hi-lo)/(nt+1): all k eigenvalues < x_t  <=>  x_t > lambda_max
    const double x = lo + (hi - lo) * (double)(tid + 1) / (double)(nt + 1);
    int cnt = 0;
    double d = 1.0;
    for (int i = 0; i < k; ++i) {
      const double e2 = i > 0 ? od[i - 1] * od[i - 1] : 0.0;
      d = (dg[i] - x) - (i > 0 ? e2 * fast_rcp(d) : 0.0);
      if (d == 0.0) d = -1e-300;
      cnt += d < 0.0;
    }
    const int above = cnt == k;  // x > lambda_max
    if (tid == 0) s_best = nt;
    __syncthreads();
    if (above) atomicMin(&s_best, tid);
    __syncthreads();
    if (tid == 0) {
      const int b = s_best;  // first shift above lambda_max
      const double step = (hi - lo) / (double)(nt + 1);
      s_lo = lo + step * (double)b;
      s_hi = (b < nt) ? lo + step * (double)(b + 1) : hi;
    }
    __syncthreads();
  }
  if (tid == 0) *out = 0.5 * (s_lo + s_hi);
}

// k <= 64: the same Householder tridiagonalisation + Sturm multisection, laid out for latency.
// Warp 0 forms each reflector (v, beta) from the column in shared memory; the matvec and the
// rank-2 update give every thread 4 x 16 entries (row t / 4, columns t % 4 + 4 i) so no step needs
// more than a 2-level shuffle; barriers are cheap (~30 cycles), long shuffle chains are not.
// The Sturm counts use the three-term recurrence of det(T_i - x I) (one dependent FMA per row,
// power-of-two rescaling every 8 rows) on T scaled to unit Gershgorin radius, instead of the
// pivot recurrence with a reciprocal per row.
__global__ void __launch_bounds__(1024) maxeig64_kernel(const double* __restrict__ Ain, int k,
                                                        double* __restrict__ out,
                                                        long long* prof = nullptr) {
  pdl_wait();
  constexpr int LD = 65;
  __shared__ double A[64 * LD];
  __shared__ double p[64], dg[64], od[64], e2[64];
  __shared__ double s_lo, s_hi, s_scale;
  __shared__ int s_best;
  const int tid = threadIdx.x, lane = tid & 31;
  const int row = tid >> 4, qq = tid & 15;  // 64 rows x 16 column lanes
  if (prof && tid == 0) prof[1] = clock64();
  for (int e = tid; e < k * k; e += 1024) {
    const int r = e / k, c = e % k;
    A[r * LD + c] = 0.5 * (Ain[r * k + c] + Ain[c * k + r]);
  }
  __syncthreads();
  // Two barriers per reflector: every warp forms (v, beta) itself from the column (v stays in
  // registers, lane l holding v[l] and v[l + 32]; bitwise the same in every warp), the matvec
  // takes v by shuffle, and every warp reduces K = beta v^T p / 2 itself after the p barrier.
  for (int j = 0; j + 2 < k; ++j) {
    const int n = k - j - 1;
    const int i0 = lane, i1 = lane + 32;
    const double x0v = i0 < n ? A[(j + 1 + i0) * LD + j] : 0.0;
    const double x1v = i1 < n ? A[(j + 1 + i1) * LD + j] : 0.0;
    const double xnorm2 = warp_sum(fma(x0v, x0v, x1v * x1v));
    const double x0 = __shfl_sync(0xffffffffu, x0v, 0);
    const double xn = sqrt(xnorm2);
    const double alpha = x0 >= 0.0 ? -xn : xn;
    const double vtv = 2.0 * xn * (xn + fabs(x0));
    if (tid == 0) {
      dg[j] = A[j * LD + j];
      od[j] = (vtv > 0.0) ? alpha : x0;
    }
    if (!(vtv > 0.0)) {  // column already reduced (uniform in every warp)
      __syncthreads();
      continue;
    }
    const double v0 = x0v - (i0 == 0 ? alpha : 0.0), v1 = x1v;  // v[lane], v[lane + 32]
    const double beta = 2.0 * fast_rcp(vtv);
    // v at the columns qq + 16 i of this thread: lanes qq / qq + 16, slots 0 / 1
    double vc[4];
    vc[0] = __shfl_sync(0xffffffffu, v0, qq);
    vc[1] = __shfl_sync(0xffffffffu, v0, qq + 16);
    vc[2] = __shfl_sync(0xffffffffu, v1, qq);
    vc[3] = __shfl_sync(0xffffffffu, v1, qq + 16);
    // p = beta A' v: row `row`, columns qq + 16 i
    double* ar = A + (j + 1 + row) * LD + (j + 1);
    double q = 0.0;
    if (row < n) {
      double qa = 0.0, qb = 0.0;
#pragma unroll
      for (int i = 0; i < 4; i += 2) {
        const int c0 = qq + 16 * i, c1 = c0 + 16;
        if (c0 < n) qa = fma(ar[c0], vc[i], qa);
        if (c1 < n) qb = fma(ar[c1], vc[i + 1], qb);
      }
      q = qa + qb;
    }
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (qq == 0 && row < n) p[row] = beta * q;
    __syncthreads();
    const double p0 = i0 < n ? p[i0] : 0.0, p1 = i1 < n ? p[i1] : 0.0;
    const double kc = 0.5 * beta * warp_sum(fma(v0, p0, v1 * p1));
    // A' -= v w^T + w v^T,  w = p - Kc v; v_row by shuffle (rows 2w, 2w+1 of warp w sit on the
    // same side of 32, so the slot choice is warp-uniform)
    const double vr = __shfl_sync(0xffffffffu, row < 32 ? v0 : v1, row & 31);
    if (row < n) {
      const double wr = p[row] - kc * vr;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = qq + 16 * i;
        if (c < n) {
          const double wc = p[c] - kc * vc[i];
          ar[c] -= vr * wc + wr * vc[i];
        }
      }
    }
    __syncthreads();
  }
  if (prof && tid == 0) prof[0] = clock64();
  if (tid == 0) {
    if (k >= 2) {
      dg[k - 2] = A[(k - 2) * LD + (k - 2)];
      od[k - 2] = A[(k - 1) * LD + (k - 2)];
    }
    dg[k - 1] = A[(k - 1) * LD + (k - 1)];
    double lo = 1.0 / 0.0, hi = -1.0 / 0.0;
    for (int i = 0; i < k; ++i) {
      const double r = (i > 0 ? fabs(od[i - 1]) : 0.0) + (i + 1 < k ? fabs(od[i]) : 0.0);
      lo = fmin(lo, dg[i] - r);
      hi = fmax(hi, dg[i] + r);
    }
    const double m = fmax(fabs(lo), fabs(hi));
    // power-of-two scale to unit Gershgorin radius (exact)
    int ex = 0;
    frexp(m, &ex);
    s_scale = (m > 0.0 && isfinite(m)) ? ldexp(1.0, -ex) : 1.0;
    s_lo = lo * s_scale;
    s_hi = hi * s_scale;
  }
  __syncthreads();
  const double sc = s_scale;
  if (tid < k) {
    dg[tid] *= sc;
    e2[tid] = tid > 0 ? (od[tid - 1] * sc) * (od[tid - 1] * sc) : 0.0;
  }
  __syncthreads();
  for (int round = 0; round < 12; ++round) {
    const double lo = s_lo, hi = s_hi;
    if (!(hi - lo > 2e-16 * fmax(fabs(hi), fabs(lo)))) break;
    const double x = lo + (hi - lo) * (double)(tid + 1) / 1025.0;
    // q_i = (a_i - x) q_{i-1} - e_i^2 q_{i-2}; eigenvalues below x = sign changes (a zero takes
    // the sign opposite to its predecessor, i.e. the pivot q_i / q_{i-1} counts as negative)
    double q1 = 1.0, q2 = 0.0;
    int sprev = 1, cnt = 0;
    for (int i = 0; i < k; ++i) {
      const double qn = fma(dg[i] - x, q1, -e2[i] * q2);
      const int sn = qn > 0.0 ? 1 : (qn < 0.0 ? -1 : -sprev);
      cnt += sn != sprev;
      sprev = sn;
      q2 = q1;
      q1 = qn;
      if ((i & 7) == 7) {  // rescale by a power of two (exact) to stay in range
        const int e = (__double2hiint(q1) >> 20) & 0x7ff;
        if (e > 0 && e < 0x7ff) {
          const double f = __hiloint2double((2046 - e) << 20, 0);  // 2^(1023 - e)
          q1 *= f;
          q2 *= f;
        }
      }
    }
    const int above = cnt == k;  // x > lambda_max
    if (tid == 0) s_best = 1024;
    __syncthreads();
    if (above) atomicMin(&s_best, tid);
    __syncthreads();
    if (tid == 0) {
      const int b = s_best;
      const double step = (hi - lo) / 1025.0;
      s_lo = lo + step * (double)b;
      s_hi = (b < 1024) ? lo + step * (double)(b + 1) : hi;
    }
    __syncthreads();
    if (prof && tid == 0) prof[2 + round] = clock64();
  }
  if (tid == 0) *out = 0.5 * (s_lo + s_hi) / sc;
}

__global__ void maxeig_smem_kernel(const double* Ain, int k, double* out) {
  pdl_wait();
  extern __shared__ __align__(16) double smem[];
  maxeig_body(Ain, k, smem, smem + (size_t)k * (k + 1), out);
}
__global__ void maxeig_gmem_kernel(const double* Ain, int k, double* W, double* out) {
  pdl_wait();
  maxeig_body(Ain, k, W, W + (size_t)k * (k + 1), out);
}

// ---------------------------------------------------------------------------------------------
// Dense SVD core for the step-0 / 'exact' / 'randomized' backends (svdengine.py:75-85, 161-196;
// linalg.py:108-121): one-sided (Hestenes) Jacobi on a small square factor W (n x n, n <= 512,
// the R of a QR pre-reduction).  Columns of W are orthogonalised by plane rotations that are
// accumulated into V; round-robin pairing lets every warp rotate a disjoint pair concurrently.
// One CTA; W and V live in global memory (L2-resident at these sizes).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int rr_index(int pos, int round, int kk) {
  // circle-method round-robin: position 0 fixed, the others rotate by one each round
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (kk - 1);
}

__global__ void jacobi_svd_kernel(double* __restrict__ W, double* __restrict__ V, int n, int ld,
                                  int max_sweeps, int* __restrict__ sweeps_out) {
  pdl_wait();
  __shared__ int s_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int nn = n + (n & 1);
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e % n;
    V[r * ld + c] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < nn - 1; ++round) {
      for (int i = warp; i < nn / 2; i += nw) {
        int p = rr_index(i, round, nn), q = rr_index(nn - 1 - i, round, nn);
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        if (q >= n) continue;  // dummy partner for odd n
        double a = 0.0, b = 0.0, c = 0.0;
        for (int r = lane; r < n; r += 32) {
          const double wp = W[r * ld + p], wq = W[r * ld + q];
          a = fma(wp, wp, a);
          b = fma(wq, wq, b);
          c = fma(wp, wq, c);
        }
        a = warp_sum(a);
        b = warp_sum(b);
        c = warp_sum(c);
        if (c == 0.0 || !(fabs(c) > 1e-15 * sqrt(a * b))) continue;
        const double zeta = (b - a) / (2.0 * c);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int r = lane; r < n; r += 32) {
          const double wp = W[r * ld + p], wq = W[r * ld + q];
          W[r * ld + p] = cs * wp - sn * wq;
          W[r * ld + q] = sn * wp + cs * wq;
          const double vp = V[r * ld + p], vq = V[r * ld + q];
          V[r * ld + p] = cs * vp - sn * vq;
          V[r * ld + q] = sn * vp + cs * vq;
        }
        if (lane == 0) atomicAdd(&s_rot, 1);
      }
      __syncthreads();
    }
    if (s_rot == 0) break;
    __syncthreads();
  }
  if (tid == 0) *sweeps_out = sweep;
}

// sigma_j = ||W[:, j]||, sorted descending (stable); Us[:, j] = W[:, order_j] / sigma_j (0 when
// sigma_j = 0), Vs[:, j] = V[:, order_j].  One CTA.
__global__ void svd_finalize_kernel(const double* __restrict__ W, const double* __restrict__ V,
                                    int n, int ld, double* __restrict__ sigma,
                                    double* __restrict__ Us, double* __restrict__ Vs, int lds) {
  pdl_wait();
  extern __shared__ double sn[];  // [n] norms, then [n] order (as double)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < n; j += nw) {
    double a = 0.0;
    for (int r = lane; r < n; r += 32) a = fma(W[r * ld + j], W[r * ld + j], a);
    a = warp_sum(a);
    if (lane == 0) sn[j] = sqrt(a);
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    const double si = sn[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += (sn[j] > si) || (sn[j] == si && j < i);
    sn[n + rank] = (double)i;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int r = e / n, j = e % n;
    const int src = (int)sn[n + j];
    const double sg = sn[src];
    Us[r * lds + j] = sg > 0.0 ? W[r * ld + src] / sg : 0.0;
    Vs[r * lds + j] = V[r * ld + src];
  }
  for (int j = tid; j < n; j += blockDim.x) sigma[j] = sn[(int)sn[n + j]];
}

// out (cols x rows) = scale * (in (rows x cols, ldi) - shift[col])^T, shift optional
__global__ void transpose_shift_kernel(const double* __restrict__ in, int64_t ldi, int64_t rows,
                                       int64_t cols, const double* __restrict__ shift,
                                       double scale, double* __restrict__ out, int64_t ldo) {
  pdl_wait();
  __shared__ double tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    tile[i][tx] = (r < rows && c < cols) ? scale * (in[r * ldi + c] - (shift ? shift[c] : 0.0))
                                         : 0.0;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + tx;
    if (c < cols && r < rows) out[c * ldo + r] = tile[tx][i];
  }
}

// ||a[:r] - b[:r]||_2 and the off-diagonal Frobenius norm of a k x k matrix (svdengine.py:216,
// svdengine.py:140).  One CTA.
__global__ void small_norms_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                   int r, const double* __restrict__ Q, int k,
                                   double* __restrict__ out) {
  pdl_wait();
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
