// Blocked one-sided (Hestenes) Jacobi SVD for the dense backends beyond the single-CTA size
// (min(m, n) > 512): step 0, svd_backend="exact" and the randomized sketch's small factor
// (optimizers.py:327-338 -> svdengine.py:75-85 -> linalg.py:108-121, numpy's dgesdd there).
//
// The nv vectors to orthogonalise are the rows of X (nv x L, row-major, ld ldx), padded with
// zero rows to nvp = 16 nb (nb even).  Rows are grouped in blocks of 16; a sweep pairs every two
// blocks once (circle-method round robin, nb - 1 rounds of nb/2 disjoint pairs, one CTA per
// pair).  For a pair (I, J) the CTA
//   1. forms the 32 x 32 Gram G = Y Y^T of its rows Y = X[I u J] on the FP64 tensor cores
//      (DMMA m8n8k4: the A and B fragments of Y Y^T are the same registers; 10 upper tiles;
//      fixed-order sum of the 8 warps' partials, so results are bitwise repeatable);
//   2. diagonalises G in shared memory by cyclic two-sided Jacobi (16 disjoint rotations per
//      round), accumulating the rotation Q (G_final = Q^T G Q);
//   3. applies Y <- Q^T Y and W[I u J] <- Q^T W[I u J] on DMMA (Q^T fragments held in
//      registers, Y streamed once, updated in place).
// W (nvp x nvp) accumulates the row operations: X_final = W X_initial.  A pair rotates only
// where |G_ab| > tol sqrt(G_aa G_bb); a sweep in which no pair rotated ends the iteration.
// High relative accuracy of one-sided Jacobi (no Gram of the whole matrix is ever formed).
#pragma once
#include "common.cuh"

namespace wssr {
namespace bj {

constexpr int kRows = 32;                // rows per pair (two blocks of 16)
constexpr int kThreads = 256;
constexpr int kLd = 33;                  // padded row stride of the 32 x 32 smem matrices
constexpr int kInnerSweeps = 16;
constexpr size_t kSmem = sizeof(double) * (8 * 10 * 64 + 2 * kRows * kLd + 2 * 16) +
                         sizeof(int) * (2 * 16 + 4);

__device__ __forceinline__ int rr(int pos, int round, int kk) {
  // circle-method round robin: position 0 fixed, the others rotate by one each round
  return pos == 0 ? 0 : 1 + (pos - 1 + round) % (kk - 1);
}

// the pair's local row i (0..31) of a matrix with leading dimension ld: block I, then block J
__device__ __forceinline__ double* pair_row(double* base, int64_t ld, int64_t rI, int64_t rJ,
                                            int i) {
  return base + (i < 16 ? rI + i : rJ + i - 16) * ld;
}

// Y (the pair's 32 rows of `base`, len columns) <- Q^T Y in place, Q^T fragments in qa.
__device__ __forceinline__ void apply_qt(double* base, int64_t ld, int64_t rI, int64_t rJ,
                                         int64_t len, const double (&qa)[4][8], int warp,
                                         int lane) {
  const int g = lane >> 2, t = lane & 3;
  for (int64_t c0 = 8 * (int64_t)warp; c0 < len; c0 += 64) {
    double b[8];
    const int64_t c = c0 + g;
#pragma unroll
    for (int s = 0; s < 8; ++s) b[s] = c < len ? pair_row(base, ld, rI, rJ, 4 * s + t)[c] : 0.0;
    double acc[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
      for (int s = 0; s < 8; ++s) dmma884(acc[j], qa[j][s], b[s]);
    }
    __syncwarp();  // every lane has read this chunk before any lane overwrites it
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double* dst = pair_row(base, ld, rI, rJ, 8 * j + g);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t cc = c0 + 2 * t + e;
        if (cc < len) dst[cc] = acc[j][e];
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads)
    round_kernel(double* __restrict__ X, int64_t ldx, int64_t L, double* __restrict__ W,
                 int64_t ldw, int nb, int round, double tol, int* __restrict__ rotated) {
  pdl_wait();
  extern __shared__ __align__(16) double sm[];
  double* part = sm;                        // [8 warps][10 tiles][64]
  double* G = part + 8 * 10 * 64;           // [32][33]
  double* Q = G + kRows * kLd;              // [32][33]
  double* cs = Q + kRows * kLd;             // [16][2]
  int* pq = reinterpret_cast<int*>(cs + 2 * 16);  // [16][2]
  int* flags = pq + 2 * 16;                 // any rotation (this round of the inner sweep), any at all

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  int I = rr(blockIdx.x, round, nb), J = rr(nb - 1 - blockIdx.x, round, nb);
  if (I > J) { const int tmp = I; I = J; J = tmp; }
  const int64_t rI = 16 * (int64_t)I, rJ = 16 * (int64_t)J;

  // ---- 1. Gram on DMMA: lane (g, t) holds Y[8 j + g][c0 + 2 t + s], s = 0, 1 (k permuted
  // identically for both operands) ----
  {
    const int tiles[10][2] = {{0, 0}, {0, 1}, {0, 2}, {0, 3}, {1, 1},
                              {1, 2}, {1, 3}, {2, 2}, {2, 3}, {3, 3}};
    double acc[10][2];
#pragma unroll
    for (int i = 0; i < 10; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int64_t c0 = 8 * (int64_t)warp; c0 < L; c0 += 64) {
      double v[4][2];
      const int64_t c = c0 + 2 * t;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double* src = pair_row(X, ldx, rI, rJ, 8 * j + g);
        if (c + 1 < L) {
          const double2 d = *reinterpret_cast<const double2*>(src + c);
          v[j][0] = d.x;
          v[j][1] = d.y;
        } else {
          v[j][0] = c < L ? src[c] : 0.0;
          v[j][1] = 0.0;
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int i = 0; i < 10; ++i) dmma884(acc[i], v[tiles[i][0]][s], v[tiles[i][1]][s]);
    }
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      part[(warp * 10 + i) * 64 + 2 * lane] = acc[i][0];
      part[(warp * 10 + i) * 64 + 2 * lane + 1] = acc[i][1];
    }
    __syncthreads();
    for (int e = tid; e < 10 * 64; e += kThreads) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += part[w * 640 + e];  // fixed order
      const int i = e / 64, l = (e % 64) / 2, el = e % 2;
      const int row = 8 * tiles[i][0] + (l >> 2), col = 8 * tiles[i][1] + 2 * (l & 3) + el;
      G[row * kLd + col] = s;
      G[col * kLd + row] = s;
    }
    for (int e = tid; e < kRows * kRows; e += kThreads)
      Q[(e / kRows) * kLd + e % kRows] = (e / kRows == e % kRows) ? 1.0 : 0.0;
    if (tid == 0) flags[1] = 0;
    __syncthreads();
  }

  // ---- 2. cyclic two-sided Jacobi on G (32 x 32), Q accumulated ----
  for (int sweep = 0; sweep < kInnerSweeps; ++sweep) {
    if (tid == 0) flags[0] = 0;
    __syncthreads();
    for (int rd = 0; rd < kRows - 1; ++rd) {
      if (tid < 16) {
        int p = rr(tid, rd, kRows), q = rr(kRows - 1 - tid, rd, kRows);
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        const double app = G[p * kLd + p], aqq = G[q * kLd + q], apq = G[p * kLd + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0 && fabs(apq) > tol * sqrt(app * aqq)) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + tt * tt);
          s = tt * c;
          flags[0] = 1;
        }
        cs[2 * tid] = c;
        cs[2 * tid + 1] = s;
        pq[2 * tid] = p;
        pq[2 * tid + 1] = q;
      }
      __syncthreads();
      // columns p, q of G and Q (G <- G J, Q <- Q J)
      for (int e = tid; e < 16 * kRows; e += kThreads) {
        const int i = e / kRows, r = e % kRows;
        const double c = cs[2 * i], s = cs[2 * i + 1];
        if (s == 0.0) continue;
        const int p = pq[2 * i], q = pq[2 * i + 1];
        const double gp = G[r * kLd + p], gq = G[r * kLd + q];
        G[r * kLd + p] = c * gp - s * gq;
        G[r * kLd + q] = s * gp + c * gq;
        const double qp = Q[r * kLd + p], qq = Q[r * kLd + q];
        Q[r * kLd + p] = c * qp - s * qq;
        Q[r * kLd + q] = s * qp + c * qq;
      }
      __syncthreads();
      // rows p, q of G (G <- J^T G)
      for (int e = tid; e < 16 * kRows; e += kThreads) {
        const int i = e / kRows, col = e % kRows;
        const double c = cs[2 * i], s = cs[2 * i + 1];
        if (s == 0.0) continue;
        const int p = pq[2 * i], q = pq[2 * i + 1];
        const double gp = G[p * kLd + col], gq = G[q * kLd + col];
        G[p * kLd + col] = c * gp - s * gq;
        G[q * kLd + col] = s * gp + c * gq;
      }
      __syncthreads();
    }
    const int any = flags[0];
    if (tid == 0 && any) flags[1] = 1;
    __syncthreads();
    if (!any) break;
  }
  if (!flags[1]) return;  // already orthogonal to tol: nothing to rotate
  if (tid == 0) atomicOr(rotated, 1);

  // ---- 3. Y <- Q^T Y, W[I u J] <- Q^T W[I u J] on DMMA ----
  double qa[4][8];  // (Q^T)[8 j + g][4 s + t] = Q[4 s + t][8 j + g]
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int s = 0; s < 8; ++s) qa[j][s] = Q[(4 * s + t) * kLd + 8 * j + g];
  apply_qt(X, ldx, rI, rJ, L, qa, warp, lane);
  apply_qt(W, ldw, rI, rJ, ldw, qa, warp, lane);
}

// W = I (nvp x nvp)
__global__ void identity_kernel(double* __restrict__ W, int64_t n) {
  pdl_wait();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * n;
       e += (int64_t)gridDim.x * blockDim.x)
    W[e] = (e / n == e % n) ? 1.0 : 0.0;
}

// norms[i] = ||X[i, :L]|| (one warp per row, fixed-order sums)
__global__ void row_norms_kernel(const double* __restrict__ X, int64_t ldx, int64_t L, int nv,
                                 double* __restrict__ norms) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nv;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double s = 0.0;
    for (int64_t c = lane; c < L; c += 32) s = fma(X[i * ldx + c], X[i * ldx + c], s);
    s = warp_sum(s);
    if (lane == 0) norms[i] = sqrt(s);
  }
}

// stable descending order: order[rank(i)] = i, sigma[rank] = norms[i]
__global__ void rank_kernel(const double* __restrict__ norms, int nv, int* __restrict__ order,
                            double* __restrict__ sigma) {
  pdl_wait();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
    const double si = norms[i];
    int r = 0;
    for (int j = 0; j < nv; ++j) {
      const double sj = norms[j];
      r += (sj > si) || (sj == si && j < i);
    }
    order[r] = i;
    sigma[r] = si;
  }
}

// dst[j, :len] = src[order_j, :len] * (inv ? 1 / sigma_j (0 if sigma_j == 0) : 1), j < q
__global__ void gather_rows_kernel(const double* __restrict__ src, int64_t lds, int64_t len,
                                   const int* __restrict__ order, const double* __restrict__ sigma,
                                   int q, int inv, double* __restrict__ dst, int64_t ldd) {
  pdl_wait();
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)q * len;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / len);
    const int64_t c = e % len;
    double f = 1.0;
    if (inv) f = sigma[j] > 0.0 ? 1.0 / sigma[j] : 0.0;
    dst[j * ldd + c] = src[(int64_t)order[j] * lds + c] * f;
  }
}

// dst[c, j] = src[order_j, c] * (inv ? 1 / sigma_j : 1)  (dst len x q, ld ldd): 32 x 32 tiles
__global__ void gather_transpose_kernel(const double* __restrict__ src, int64_t lds, int64_t len,
                                        const int* __restrict__ order,
                                        const double* __restrict__ sigma, int q, int inv,
                                        double* __restrict__ dst, int64_t ldd) {
  pdl_wait();
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int i = ty; i < 32; i += 8) {
    const int j = j0 + i;
    const int64_t c = c0 + tx;
    double v = 0.0;
    if (j < q && c < len) {
      double f = 1.0;
      if (inv) f = sigma[j] > 0.0 ? 1.0 / sigma[j] : 0.0;
      v = src[(int64_t)order[j] * lds + c] * f;
    }
    tile[i][tx] = v;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i;
    const int j = j0 + tx;
    if (c < len && j < q) dst[c * ldd + j] = tile[tx][i];
  }
}

}  // namespace bj
}  // namespace wssr
