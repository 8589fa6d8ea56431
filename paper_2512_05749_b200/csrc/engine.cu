// WSSR engine: the reference control flow of assemble / qr_orthonormalize / ssi_svd /
// subspace_drift / wssr_step, re-expressed as stream-ordered launches of the sm_100a kernels.
// Every function cites the reference lines it follows.  Host synchronisation happens only where
// the reference returns a Python scalar that decides control flow (the SSI exit test,
// svdengine.py:139-141, and the rank cut, optimizers.py:348-355).
#include <dlfcn.h>

#include <condition_variable>
#include <mutex>

#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <utility>
#include <chrono>
#include <map>
#include <tuple>
#include <vector>
#include <cstdlib>

#include "engine.h"
#include "ozaki.h"
#include "gemm.cuh"
#include "kernels.cuh"
#include "tallskinny.h"
#include "producer.h"
#include "jacobi.cuh"

struct wssr_ctx {
  wssr::Context c;
};

namespace wssr {

struct Fail {
  int code;
  std::string msg;
};

#define WSSR_CUDA(expr)                                                                      \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      throw Fail{WSSR_ERR_CUDA, std::string(#expr) + " -> " + cudaGetErrorString(e_)};       \
  } while (0)

constexpr double kDeficientColumnRel = 1e-12;  // linalg.py:16 DEFICIENT_COLUMN_REL
constexpr double kZeroMatrixNorm = 1e-300;     // linalg.py:15 ZERO_MATRIX_NORM
constexpr double kCholPivotRel = 1e-13;        // CholeskyQR2 safety margin (see kernels.cuh)

double* Context::splitk_buffer(size_t n) {
  if (n > splitk_cap) {
    if (splitk) {
      cudaStreamSynchronize(stream);
      cudaFree(splitk);
      splitk = nullptr;
    }
    size_t cap = std::max(n, splitk_cap * 2);
    if (cudaMalloc(&splitk, cap * sizeof(double)) != cudaSuccess) {
      splitk = nullptr;
      splitk_cap = 0;
      return nullptr;
    }
    splitk_cap = cap;
  }
  return splitk;
}

namespace {

// Stream-ordered scratch allocation from the device's default memory pool.
// profiling only (WSSR_HOST_PROF=1): host seconds spent in allocation / synchronisation calls
struct HostProf {
  bool on = std::getenv("WSSR_HOST_PROF") != nullptr;
  double alloc_s = 0, sync_s = 0, free_s = 0;
  int64_t allocs = 0, syncs = 0;
  static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
  }
};
HostProf g_hprof;

// Step scratch: blocks released by a Buf are kept per (device, stream, size) and handed to the
// next Buf of that size on the same stream.  Same-stream reuse is exactly the ordering
// cudaFreeAsync / cudaMallocAsync give, without a pool call per buffer: at c2 (137 GB of O
// resident) a cudaMallocAsync of a 1 GB P x k block blocked the host for up to 130 ms while the
// pool searched for space.  On allocation failure the cached blocks are returned to the pool
// and the allocation is retried.
struct ScratchCache {
  std::mutex mu;
  struct Key {
    int dev;
    cudaStream_t st;
    size_t bytes;
    bool operator<(const Key& o) const {
      return std::tie(dev, st, bytes) < std::tie(o.dev, o.st, o.bytes);
    }
  };
  std::map<Key, std::vector<void*>> free_blocks;
  std::map<void*, size_t> sizes;
  size_t cached_bytes = 0;
  void* take(size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free_blocks.find(Key{dev, st, bytes});
      if (it != free_blocks.end() && !it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        cached_bytes -= bytes;
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      trim(dev);
      e = cudaMallocAsync(&p, bytes, st);
      if (e != cudaSuccess) throw Fail{WSSR_ERR_CUDA, cudaGetErrorString(e)};
    }
    std::lock_guard<std::mutex> lk(mu);
    sizes[p] = bytes;
    return p;
  }
  void give(void* p, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu);
      const size_t bytes = sizes[p];
      if (cached_bytes + bytes <= kCap) {
        free_blocks[Key{dev, st, bytes}].push_back(p);
        cached_bytes += bytes;
        return;
      }
      sizes.erase(p);
    }
    cudaFreeAsync(p, st);
  }
  // return this device's cached blocks to the pool (after a device synchronisation, so streams
  // that no longer exist do not matter)
  void trim(int dev) {
    std::vector<void*> out;
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto it = free_blocks.begin(); it != free_blocks.end();) {
        if (it->first.dev != dev) {
          ++it;
          continue;
        }
        for (void* p : it->second) {
          out.push_back(p);
          sizes.erase(p);
          cached_bytes -= it->first.bytes;
        }
        it = free_blocks.erase(it);
      }
    }
    if (out.empty()) return;
    cudaDeviceSynchronize();
    for (void* p : out) cudaFree(p);
  }
  static constexpr size_t kCap = (size_t)16 << 30;  // bytes kept cached over all devices
};
ScratchCache g_scratch;

struct Buf {
  double* p = nullptr;
  cudaStream_t st = nullptr;
  Buf() = default;
  Buf(size_t n, cudaStream_t s) : st(s) {
    if (!n) return;
    const double t0 = g_hprof.on ? HostProf::now() : 0.0;
    p = static_cast<double*>(g_scratch.take(n * sizeof(double), s));
    if (g_hprof.on) g_hprof.alloc_s += HostProf::now() - t0, ++g_hprof.allocs;
  }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
  Buf(Buf&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
  Buf& operator=(Buf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      st = o.st;
      o.p = nullptr;
    }
    return *this;
  }
  ~Buf() { release(); }
  void release() {
    if (!p) return;
    const double t0 = g_hprof.on ? HostProf::now() : 0.0;
    g_scratch.give(p, st);
    if (g_hprof.on) g_hprof.free_s += HostProf::now() - t0;
    p = nullptr;
  }
  operator double*() const { return p; }
  int64_t* i64() const { return reinterpret_cast<int64_t*>(p); }
  int* i32() const { return reinterpret_cast<int*>(p); }
};

inline int blocks_for(int64_t n, int threads, int cap) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (int)b;
}

void post_launch(Context& ctx) {
  ++ctx.kernel_launches;
  WSSR_CUDA(cudaGetLastError());
}

void collect_timing(Context& ctx);
void sync(Context& ctx) {
  const double t0 = g_hprof.on ? HostProf::now() : 0.0;
  WSSR_CUDA(cudaStreamSynchronize(ctx.stream));
  if (g_hprof.on) g_hprof.sync_s += HostProf::now() - t0, ++g_hprof.syncs;
  if (!ctx.pending.empty()) collect_timing(ctx);
}

void d2h(Context& ctx, void* dst, const void* src, size_t bytes) {
  WSSR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx.stream));
}

void allreduce(Context& ctx, double* buf, size_t n) {
  cudaError_t e = ctx.allreduce(buf, n);
  if (e != cudaSuccess) throw Fail{WSSR_ERR_NCCL, "allreduce failed"};
}

// ---- phase timing (bench.py roofline) ------------------------------------------------------
cudaEvent_t take_event(Context& ctx) {
  if (!ctx.event_pool.empty()) {
    cudaEvent_t e = ctx.event_pool.back();
    ctx.event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  WSSR_CUDA(cudaEventCreate(&e));
  return e;
}
struct PhaseTimer {
  Context& ctx;
  int phase;
  double flops, bytes;
  cudaEvent_t a = nullptr;
  PhaseTimer(Context& c, int ph, double f, double b) : ctx(c), phase(ph), flops(f), bytes(b) {
    if (ctx.timing && ph >= 0) {
      a = take_event(ctx);
      WSSR_CUDA(cudaEventRecord(a, ctx.stream));
    }
  }
  ~PhaseTimer() {
    if (!a) return;
    cudaEvent_t b = take_event(ctx);
    cudaEventRecord(b, ctx.stream);
    ctx.pending.push_back({phase, a, b, flops, bytes});
  }
};
// fold finished event pairs into the per-phase totals (call after a stream sync)
void collect_timing(Context& ctx) {
  std::vector<Context::PendingEvent> later;  // pairs on the aux stream that have not finished
  for (auto& pe : ctx.pending) {
    if (cudaEventQuery(pe.b) == cudaErrorNotReady) {
      later.push_back(pe);
      continue;
    }
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pe.a, pe.b) == cudaSuccess) {
      ctx.phase_ms[pe.phase] += ms;
      ctx.phase_flops[pe.phase] += pe.flops;
      ctx.phase_bytes[pe.phase] += pe.bytes;
      ctx.phase_count[pe.phase] += 1;
    }
    ctx.event_pool.push_back(pe.a);
    ctx.event_pool.push_back(pe.b);
  }
  cudaGetLastError();  // clear cudaErrorNotReady
  ctx.pending.swap(later);
}

// ---- GEMM wrappers ------------------------------------------------------------------------
// CM: C(MxN) = alpha * sum_k (A[k*lda+m] - shift[m]) B[k*ldb+n]
void gemm_cm(Context& ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
             const double* shift, const double* B, int64_t ldb, double* C, int64_t ldc,
             double alpha, bool accumulate, int max_splits = 1024) {
  GemmArgs a{A, lda, B, ldb, shift, C, ldc, M, N, K, 0, alpha, accumulate ? 1 : 0, nullptr,
             nullptr, 0};
  WSSR_CUDA(gemm(ctx, Layout::CM, a, max_splits, ctx.stream));
}
// RM: C(MxN) = alpha * sum_k (A[m*lda+k] - shift[k]) B[k*ldb+n]
void gemm_rm(Context& ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
             const double* shift, const double* B, int64_t ldb, double* C, int64_t ldc,
             double alpha, bool accumulate, int max_splits = 1024) {
  GemmArgs a{A, lda, B, ldb, shift, C, ldc, M, N, K, 0, alpha, accumulate ? 1 : 0, nullptr,
             nullptr, 0};
  WSSR_CUDA(gemm(ctx, Layout::RM, a, max_splits, ctx.stream));
}
// C = Cin + alpha * A(MxK, row-major) B   (the "w - q * quotient" / "u2 - u1 C" shape)
void gemm_rm_add(Context& ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                 const double* B, int64_t ldb, const double* Cin, int64_t ldcin, double* C,
                 int64_t ldc, double alpha) {
  GemmArgs a{A, lda, B, ldb, nullptr, C, ldc, M, N, K, 0, alpha, 0, nullptr, Cin, ldcin};
  WSSR_CUDA(gemm(ctx, Layout::RM, a, 1024, ctx.stream));
}

// k = 256 (BASELINE configs[4]) runs on the k = 128 tall-skinny kernels as 2 x 2 blocks: the two
// 128-column halves of a rows x 256 block and the four 128 x 128 blocks of a 256 x 256 operand are
// addressed in place through their leading dimensions.
constexpr int64_t kTsHalf = 128;
bool ts_blocked(const Context& ctx, int64_t k) { return ctx.tallskinny && k == 2 * kTsHalf; }
bool ts_blocked_rows(const double* A, int64_t lda, const double* Y, int64_t ldy) {
  return ts_mul_supported(kTsHalf, A, lda, Y, ldy) &&
         ts_mul_supported(kTsHalf, A + kTsHalf, lda, Y + kTsHalf, ldy);
}
void transpose(Context& ctx, const double* in, int64_t ldi, int64_t rows, int64_t cols,
               const double* shift, double scale, double* out, int64_t ldo);

// Gram G (k x k) = A^T A, A rows x k (lda); allreduced over ranks when rows are sharded.
void gram(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda, double* G,
          bool distributed) {
  if (ts_blocked(ctx, k)) {
    const int64_t h = kTsHalf;
    WSSR_CUDA(ts_gram(ctx, rows, h, A, lda, G, k));
    WSSR_CUDA(ts_gram(ctx, rows, h, A + h, lda, G + h * k + h, k));
    WSSR_CUDA(ts_cross(ctx, rows, h, A, lda, A + h, lda, G + h, k));
    transpose(ctx, G + h, k, h, h, nullptr, 1.0, G + h * k, k);  // G21 = G12^T
  } else if (ctx.tallskinny && ts_supported(k)) {
    WSSR_CUDA(ts_gram(ctx, rows, k, A, lda, G));
  } else {
    gemm_cm(ctx, k, k, rows, A, lda, nullptr, A, lda, G, k, 1.0, false);
  }
  if (distributed) allreduce(ctx, G, (size_t)(k * k));
}

// C (k x k) = A^T B for rows x k blocks
void cross(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda, const double* B,
           int64_t ldb, double* C) {
  if (ts_blocked(ctx, k)) {
    const int64_t h = kTsHalf;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j)
        WSSR_CUDA(ts_cross(ctx, rows, h, A + i * h, lda, B + j * h, ldb, C + i * h * k + j * h, k));
  } else if (ctx.tallskinny && ts_supported(k)) {
    WSSR_CUDA(ts_cross(ctx, rows, k, A, lda, B, ldb, C));
  } else {
    gemm_cm(ctx, k, k, rows, A, lda, nullptr, B, ldb, C, k, 1.0, false);
  }
}

// out[j] = sum_i A[i][j] x[i] (A rows x n): the k-vectors of the preconditioner / state refresh
void gemv_t(Context& ctx, int64_t rows, int64_t n, const double* A, int64_t lda, const double* x,
            double* out) {
  if (ctx.tallskinny) {
    WSSR_CUDA(ts_gemv_t(ctx, rows, n, A, lda, x, 1.0, out));
  } else {
    gemm_cm(ctx, n, 1, rows, A, lda, nullptr, x, 1, out, 1, 1.0, false);
  }
}

// Y = A M for a rows x k block A and a k x k M (upper: M upper triangular, e.g. R^-1)
void mul_small(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
               const double* M, bool upper, double* Y, int64_t ldy) {
  if (ts_blocked(ctx, k) && ts_blocked_rows(A, lda, Y, ldy) && A != Y) {
    // [Y1 Y2] = [A1 A2] [[M11, M12], [M21, M22]]  (M21 = 0 when upper)
    const int64_t h = kTsHalf;
    WSSR_CUDA(ts_mul(ctx, rows, h, A, lda, M, upper, 1.0, Y, ldy, k));
    if (!upper) WSSR_CUDA(ts_mul_add(ctx, rows, h, A + h, lda, M + h * k, 1.0, Y, ldy, Y, ldy, k));
    WSSR_CUDA(ts_mul(ctx, rows, h, A, lda, M + h, false, 1.0, Y + h, ldy, k));
    WSSR_CUDA(ts_mul_add(ctx, rows, h, A + h, lda, M + h * k + h, 1.0, Y + h, ldy, Y + h, ldy, k));
  } else if (ctx.tallskinny && ts_mul_supported(k, A, lda, Y, ldy)) {
    WSSR_CUDA(ts_mul(ctx, rows, k, A, lda, M, upper, 1.0, Y, ldy));
  } else {
    gemm_rm(ctx, rows, k, k, A, lda, nullptr, M, k, Y, ldy, 1.0, false);
  }
}

// Y = Cin - A M
void sub_mul_small(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda,
                   const double* M, const double* Cin, int64_t ldcin, double* Y, int64_t ldy) {
  if (ts_blocked(ctx, k) && ts_blocked_rows(A, lda, Y, ldy) && ts_blocked_rows(Cin, ldcin, Y, ldy) &&
      A != Y) {
    const int64_t h = kTsHalf;
    for (int j = 0; j < 2; ++j) {  // Y_j = Cin_j - A1 M_1j - A2 M_2j
      WSSR_CUDA(ts_mul_add(ctx, rows, h, A, lda, M + j * h, -1.0, Cin + j * h, ldcin, Y + j * h,
                           ldy, k));
      WSSR_CUDA(ts_mul_add(ctx, rows, h, A + h, lda, M + h * k + j * h, -1.0, Y + j * h, ldy,
                           Y + j * h, ldy, k));
    }
  } else if (ctx.tallskinny && ts_mul_supported(k, A, lda, Y, ldy) &&
      ts_mul_supported(k, Cin, ldcin, Y, ldy)) {
    WSSR_CUDA(ts_mul_add(ctx, rows, k, A, lda, M, -1.0, Cin, ldcin, Y, ldy));
  } else {
    gemm_rm_add(ctx, rows, k, k, A, lda, M, k, Cin, ldcin, Y, ldy, -1.0);
  }
}

// ---- small helpers -------------------------------------------------------------------------
void copy2d(Context& ctx, const double* in, int64_t ldi, int64_t rows, int64_t cols, double scale,
            double* out, int64_t ldo) {
  if (rows <= 0 || cols <= 0) return;
  launch_pdl(copy2d_kernel, blocks_for(rows * cols, 256, 8 * ctx.num_sms), 256, 0, ctx.stream, 
      in, ldi, rows, cols, scale, out, ldo);
  post_launch(ctx);
}

// sum of squares of a strided matrix -> device scalar (deterministic)
void sumsq_matrix(Context& ctx, const double* x, int64_t rows, int64_t cols, int64_t ld,
                  double* out_dev, double scale = 1.0) {
  if (rows <= 0 || cols <= 0) {
    WSSR_CUDA(cudaMemsetAsync(out_dev, 0, sizeof(double), ctx.stream));
    return;
  }
  const int nblk = std::min<int64_t>(2 * ctx.num_sms, rows);
  const int64_t rpb = (rows + nblk - 1) / nblk;
  const int nb = (int)((rows + rpb - 1) / rpb);
  Buf part(nb, ctx.stream);
  launch_pdl(matrix_sumsq_partials_kernel, nb, 256, 0, ctx.stream, x, rows, cols, ld, rpb, part);
  post_launch(ctx);
  launch_pdl(reduce_final_kernel, 1, 256, 0, ctx.stream, part, nb, scale, out_dev);
  post_launch(ctx);
}

// out[r] = ||x[r, :]|| for an (rows x cols, ld) matrix
void row_norms(Context& ctx, const double* x, int64_t rows, int64_t cols, int64_t ld,
               double* out) {
  const int64_t chunk = 8192;
  const int nb = (int)std::max<int64_t>(1, (cols + chunk - 1) / chunk);
  Buf part((size_t)rows * nb, ctx.stream);
  launch_pdl(row_sumsq_partials_kernel, dim3(nb, (unsigned)rows), 256, 0, ctx.stream, x, cols, ld, chunk,
                                                                               part);
  post_launch(ctx);
  launch_pdl(row_norms_final_kernel, (unsigned)((rows + 127) / 128), 128, 0, ctx.stream, part, nb,
                                                                                (int)rows, out, 1);
  post_launch(ctx);
}

double read_scalar(Context& ctx, const double* dev) {
  double h = 0.0;
  d2h(ctx, &h, dev, sizeof(double));
  sync(ctx);
  return h;
}

// ---- k x k Cholesky + inverse ---------------------------------------------------------------
void launch_chol_packed(Context& ctx, const double* G, int k, double* R, double* Rinv, int* status,
                        const double* dref, const double* tref, int pivot_base) {
  static std::atomic<uint64_t> attr{0};
  WSSR_CUDA(smem_attr_once(attr, chol_inv_packed_kernel, 200 * 1024));
  launch_pdl(chol_inv_packed_kernel, 1, 256, sizeof(double) * chol_packed_doubles(k), ctx.stream,
             G, k, R, Rinv, status, kCholPivotRel, ctx.chol_series ? 1 : 0, dref, tref,
             pivot_base);
  post_launch(ctx);
}

// 160 < k <= 256 (BASELINE configs[4], k = 256): two diagonal blocks through the shared-memory
// kernel instead of one sweep over global scratch (7 ms per call at k = 256).  With
// G = [[G11, G12], [G12^T, G22]] and R upper: R11 = chol(G11), R12 = R11^-T G12,
// R22 = chol(G22 - R12^T R12), R^-1 = [[R11^-1, -R11^-1 R12 R22^-1], [0, R22^-1]].  The pivot
// tests of both blocks refer to the original diagonal and trace of G, as the one-sweep kernel's.
void chol_inv_blocked2(Context& ctx, const double* G, int k, double* R, double* Rinv,
                       int* status) {
  cudaStream_t st = ctx.stream;
  const int h = (k + 1) / 2, k2 = k - h;
  Buf dt((size_t)k + 1, st), G11((size_t)h * h, st), R11((size_t)h * h, st),
      R11i((size_t)h * h, st), R12((size_t)h * k2, st), S((size_t)k2 * k2, st),
      R22((size_t)k2 * k2, st), R22i((size_t)k2 * k2, st), W((size_t)h * k2, st),
      T((size_t)h * k2, st);
  auto sgemm = [&](int m, int n, int kk, const double* A, int64_t a_rs, int64_t a_cs,
                   const double* B, int64_t b_rs, int64_t b_cs, const double* C0, int64_t c0_ld,
                   double alpha, double* C, int64_t ldc) {
    launch_pdl(small_gemm_kernel, dim3((unsigned)((n + 15) / 16), (unsigned)((m + 15) / 16)), 256,
               0, st, m, n, kk, A, a_rs, a_cs, B, b_rs, b_cs, C0, c0_ld, alpha, C, ldc);
    post_launch(ctx);
  };
  launch_pdl(chol_diag_trace_kernel, 1, 256, 0, st, G, k, dt.p);
  post_launch(ctx);
  copy2d(ctx, G, k, h, h, 1.0, G11, h);
  launch_chol_packed(ctx, G11, h, R11, R11i, status, nullptr, dt + k, 0);
  sgemm(h, k2, h, R11i, 1, h, G + h, k, 1, nullptr, 0, 1.0, R12, k2);        // R11^-T G12
  sgemm(k2, k2, h, R12, 1, k2, R12, k2, 1, G + (size_t)h * k + h, k, -1.0, S, k2);
  launch_chol_packed(ctx, S, k2, R22, R22i, status, dt + h, dt + k, h);
  sgemm(h, k2, k2, R12, k2, 1, R22i, k2, 1, nullptr, 0, 1.0, W, k2);          // R12 R22^-1
  sgemm(h, k2, h, R11i, h, 1, W, k2, 1, nullptr, 0, -1.0, T, k2);             // -R11^-1 (...)
  launch_pdl(chol_assemble2_kernel, blocks_for((int64_t)k * k, 256, 256), 256, 0, st, k, h,
             (const double*)R11, (const double*)R11i, (const double*)R12, (const double*)T,
             (const double*)R22, (const double*)R22i, R, Rinv);
  post_launch(ctx);
}

void chol_inv(Context& ctx, const double* G, int k, double* R, double* Rinv, int* status) {
  const size_t smem = sizeof(double) * chol_scratch_doubles(k);
  if (k <= 64) {
    // dynamic shared memory enables the near-identity series path (second CholeskyQR2 pass)
    const int series_smem = (int)(2 * 64 * 65 * sizeof(double));  // series path / blocked sweep
    static std::atomic<uint64_t> attr{0};
    WSSR_CUDA(smem_attr_once(attr, chol_inv_reg64_kernel, series_smem));
    launch_pdl(chol_inv_reg64_kernel, 1, 256, series_smem, ctx.stream, G, k, R, Rinv, status,
                                                                 kCholPivotRel,
                                                                 ctx.chol_series ? 1 : 0, nullptr);
  } else if (smem <= 200 * 1024) {
    static std::atomic<uint64_t> attr{0};
    WSSR_CUDA(smem_attr_once(attr, chol_inv_smem_kernel, 200 * 1024));
    launch_pdl(chol_inv_smem_kernel, 1, 256, smem, ctx.stream, G, k, R, Rinv, status, kCholPivotRel);
  } else if (sizeof(double) * chol_packed_doubles(k) <= 200 * 1024) {
    // k = 128 (BASELINE configs[2], [3]): L and L^-1 share one shared-memory array
    launch_chol_packed(ctx, G, k, R, Rinv, status, nullptr, nullptr, 0);
    return;
  } else if (sizeof(double) * chol_packed_doubles((k + 1) / 2) <= 200 * 1024) {
    chol_inv_blocked2(ctx, G, k, R, Rinv, status);
    return;
  } else {
    Buf W(chol_scratch_doubles(k), ctx.stream);
    launch_pdl(chol_inv_gmem_kernel, 1, 256, 0, ctx.stream, G, k, W, R, Rinv, status, kCholPivotRel);
  }
  post_launch(ctx);
}

// ---- QR: CholeskyQR2 fast path, two-pass Gram-Schmidt with canonical fill as the exact
// re-statement of linalg.py:64-105 when CholeskyQR2 cannot resolve the block. -------------------

// Fast CholeskyQR2.  Q (rows x k, ldq), R (k x k).  Failure is recorded in status[] (device)
// and checked by the caller; no host synchronisation.
void cholqr2(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda, double* Q,
             int64_t ldq, double* R, int* status, bool distributed) {
  PhaseTimer tm(ctx, rows >= 65536 ? 3 : 7, 8.0 * rows * k * k, 4.0 * 8.0 * rows * k);
  Buf G((size_t)k * k, ctx.stream), R1((size_t)k * k, ctx.stream), R1i((size_t)k * k, ctx.stream),
      R2((size_t)k * k, ctx.stream), R2i((size_t)k * k, ctx.stream),
      T((size_t)rows * k, ctx.stream);
  const bool fine = ctx.fine_phases && ctx.timing;
  auto sub = [&](int ph) { return std::make_unique<PhaseTimer>(ctx, fine ? ph : -1, 0.0, 0.0); };
  { auto t = sub(8); gram(ctx, rows, k, A, lda, G, distributed); }
  { auto t = sub(9); chol_inv(ctx, G, (int)k, R1, R1i, status); }
  { auto t = sub(10); mul_small(ctx, rows, k, A, lda, R1i, true, T, k); }
  { auto t = sub(11); gram(ctx, rows, k, T, k, G, distributed); }
  { auto t = sub(12); chol_inv(ctx, G, (int)k, R2, R2i, status); }
  { auto t = sub(13); mul_small(ctx, rows, k, T, k, R2i, true, Q, ldq); }
  if (R) {  // R = R2 R1 (only the callers that read R ask for it)
    launch_pdl(triu_mul_kernel, blocks_for(k * k, 256, 1 << 20), 256, 0, ctx.stream, R2, R1, (int)k, R);
    post_launch(ctx);
  }
}

__global__ void set_entry_kernel(double* p, double v) {
  pdl_wait(); *p = v; }
__global__ void add_col_kernel(double* R, int64_t ldr, int64_t col, const double* c, int64_t n) {
  pdl_wait();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) R[i * ldr + col] += c[i];
}

// linalg.py:64-84 (_gram_schmidt_with_patch) + 87-105 (_canonical_fill), on the device with a
// host loop over columns.  Single-rank only.
void cgs2_patch(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda, double* Q,
                int64_t ldq, double* R, double fro) {
  const double tol = kDeficientColumnRel * fro;
  WSSR_CUDA(cudaMemsetAsync(R, 0, sizeof(double) * k * k, ctx.stream));
  Buf coeff(std::max<int64_t>(k, 1), ctx.stream), scal(1, ctx.stream);
  auto project_out = [&](int64_t j, double* v, int64_t ldv, bool into_r) {
    // v -= Q[:, :j] (Q[:, :j]^T v), twice
    for (int pass = 0; pass < 2; ++pass) {
      if (j == 0) break;
      gemm_cm(ctx, j, 1, rows, Q, ldq, nullptr, v, ldv, coeff, 1, 1.0, false);
      if (into_r) {
        launch_pdl(add_col_kernel, 1, 256, 0, ctx.stream, R, k, j, coeff, j);
        post_launch(ctx);
      }
      gemm_rm(ctx, rows, 1, j, Q, ldq, nullptr, coeff, 1, v, ldv, -1.0, true);
    }
  };
  for (int64_t j = 0; j < k; ++j) {
    double* qj = Q + j;
    copy2d(ctx, A + j, lda, rows, 1, 1.0, qj, ldq);
    project_out(j, qj, ldq, true);
    sumsq_matrix(ctx, qj, rows, 1, ldq, scal);
    const double norm = std::sqrt(read_scalar(ctx, scal));
    if (norm > tol) {
      copy2d(ctx, qj, ldq, rows, 1, 1.0 / norm, qj, ldq);
      launch_pdl(set_entry_kernel, 1, 1, 0, ctx.stream, R + j * k + j, norm);
      post_launch(ctx);
      continue;
    }
    // canonical fill: first e_i whose projected remainder has norm > 0.5, else the best one
    int64_t best = -1;
    double best_norm = -1.0;
    bool done = false;
    for (int64_t i = 0; i < rows && !done; ++i) {
      WSSR_CUDA(cudaMemset2DAsync(qj, sizeof(double) * ldq, 0, sizeof(double), rows, ctx.stream));
      launch_pdl(set_entry_kernel, 1, 1, 0, ctx.stream, qj + i * ldq, 1.0);
      post_launch(ctx);
      project_out(j, qj, ldq, false);
      sumsq_matrix(ctx, qj, rows, 1, ldq, scal);
      const double nw = std::sqrt(read_scalar(ctx, scal));
      if (nw > 0.5) {
        copy2d(ctx, qj, ldq, rows, 1, 1.0 / nw, qj, ldq);
        done = true;
      } else if (nw > best_norm) {
        best_norm = nw;
        best = i;
      }
    }
    if (!done) {
      if (best < 0 || best_norm <= 0.0)
        throw Fail{WSSR_ERR_ZERO_MATRIX, "no canonical direction available for deficiency patch"};
      WSSR_CUDA(cudaMemset2DAsync(qj, sizeof(double) * ldq, 0, sizeof(double), rows, ctx.stream));
      launch_pdl(set_entry_kernel, 1, 1, 0, ctx.stream, qj + best * ldq, 1.0);
      post_launch(ctx);
      project_out(j, qj, ldq, false);
      copy2d(ctx, qj, ldq, rows, 1, 1.0 / best_norm, qj, ldq);
    }
    // R[j][j] stays 0 (linalg.py:193)
  }
}

// qr_orthonormalize (linalg.py:29-61).  careful=false: CholeskyQR2 only, failures flagged in
// status (device) for the caller's end-of-step check.  careful=true: host-checked; falls back
// to the Gram-Schmidt patch path exactly where the reference leaves its LAPACK fast path.
void qr(Context& ctx, int64_t rows, int64_t k, const double* A, int64_t lda, double* Q,
        int64_t ldq, double* R, int* status, bool careful, bool distributed) {
  if (!careful) {
    cholqr2(ctx, rows, k, A, lda, Q, ldq, R, status, distributed);
    return;
  }
  Buf s(1, ctx.stream);
  sumsq_matrix(ctx, A, rows, k, lda, s);
  if (distributed) allreduce(ctx, s, 1);
  const double fro = std::sqrt(read_scalar(ctx, s));
  if (fro < kZeroMatrixNorm) {
    char msg[128];
    std::snprintf(msg, sizeof msg, "cannot orthonormalize a numerically zero matrix (norm %.3e)",
                  fro);
    throw Fail{WSSR_ERR_ZERO_MATRIX, msg};
  }
  Buf st(1, ctx.stream);
  WSSR_CUDA(cudaMemsetAsync(st, 0, sizeof(double), ctx.stream));
  cholqr2(ctx, rows, k, A, lda, Q, ldq, R, st.i32(), distributed);
  int hst[2] = {0, 0};
  d2h(ctx, hst, st, sizeof(hst));
  sync(ctx);
  if (hst[0] == 0) return;
  if (distributed)
    throw Fail{WSSR_ERR_UNSUPPORTED, "rank-deficient block under row sharding"};
  Buf Rscratch(R ? 0 : (size_t)k * k, ctx.stream);
  cgs2_patch(ctx, rows, k, A, lda, Q, ldq, R ? R : (double*)Rscratch, fro);
}

// ---- the stacked matrix Ohat (optimizers.py:321-324) as a virtual two-block operator ----------
struct Ohat {
  int64_t P = 0;
  const double* hist = nullptr;
  int64_t r = 0, ldh = 0;
  double sh = 0.0;
  const double* samp = nullptr;
  int64_t n = 0, lds = 0;
  const double* mu = nullptr;
  double ss = 1.0;
  bool f32 = false;  // samples stored as float32 (BASELINE configs[3])
  // per-parameter scale table of the int8 tensor-core path: from assemble, or built on first use
  // (shared by copies)
  const double* scale_tab = nullptr;
  mutable std::shared_ptr<Buf> oz_scale;
  // the pre-digitised sample block (in the context's plane buffer), built on first use
  struct Planes {
    const int8_t* ptr = nullptr;
    int64_t rows = 0;  // planes cover samples [0, rows); the rest is digitised on the fly
  };
  mutable std::shared_ptr<Planes> oz_planes;
  // precision guard (ozaki.cu row_guard_kernel): status word the verdict goes to (status[2] of
  // the step's device status, see with_fallback), and whether this operand was checked already
  mutable int* status = nullptr;
  mutable bool guard_done = false;
  int64_t cols() const { return r + n; }
};

// The context's digit-plane buffer, grown on demand while HBM allows (keeps 2 GiB free);
// false: digitise on the fly instead.
bool ensure_planes(Context& ctx, size_t bytes) {
  if (bytes <= ctx.oz_planes_cap) return true;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  const size_t margin = (size_t)2 << 30;
  if (free_b + ctx.oz_planes_cap < bytes + margin) return false;
  WSSR_CUDA(cudaStreamSynchronize(ctx.stream));
  if (ctx.oz_planes) cudaFree(ctx.oz_planes);
  ctx.oz_planes = nullptr;
  ctx.oz_planes_cap = 0;
  if (cudaMalloc(reinterpret_cast<void**>(&ctx.oz_planes), bytes) != cudaSuccess) {
    cudaGetLastError();
    ctx.oz_planes = nullptr;
    return false;
  }
  ctx.oz_planes_cap = bytes;
  return true;
}

// Samples whose digit planes the step keeps (a multiple of 128, or all of them): every sample
// when the planes fit next to the step's workspace, else as many as HBM allows (c2/c3: the
// 7-byte planes of 16384 x 2^20 samples are 120 GB), 0 below 1024.  The first step plans with a
// cold margin (2 GiB + 16 P x k blocks: its scratch is not allocated yet); a partial plan is
// revisited once at the next step, when the step's scratch sits in the context's pool and
// cudaMemGetInfo already counts it, with a warm margin of 2 GiB + 6 P x k blocks (room for the
// caller's own per-step tensors).
int sample_digits(const Context& ctx, const Ohat& o) {
  return (o.f32 && ctx.f32_digits == 5) ? 5 : 7;
}

int64_t plan_plane_rows(Context& ctx, const Ohat& o, int64_t k) {
  const int nds = sample_digits(ctx, o);
  const size_t full = ozaki_planes_bytes(o.n, o.P, nds);
  const char* cap_env0 = std::getenv("WSSR_OZ_PLANE_ROWS");
  const bool same = ctx.plan_n == o.n && ctx.plan_p == o.P && ctx.plan_k == k &&
                    ctx.plan_nds == nds;
  const bool warm = ctx.steps_done > 0;
  // no memory query when the decision is already known: cudaMemGetInfo can stall the host for
  // milliseconds (it contends with NVML clients), and the stream drains meanwhile
  if (!cap_env0) {
    if (full <= ctx.oz_planes_cap) return o.n;
    if (same && !(ctx.plan_provisional && warm)) return ctx.plan_rows;
  }
  const size_t blocks = warm && same ? 6 : 16;
  const size_t margin = ((size_t)2 << 30) + blocks * o.P * std::max<int64_t>(k, 1) * 8;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  const size_t have = free_b + ctx.oz_planes_cap;
  const size_t avail = have > margin ? have - margin : 0;
  // testing only: cap the planes at WSSR_OZ_PLANE_ROWS samples (exercises the split passes)
  const char* cap_env = std::getenv("WSSR_OZ_PLANE_ROWS");
  const int64_t cap = cap_env ? std::max<int64_t>(0, std::atoll(cap_env)) / 128 * 128 : -1;
  if (full <= avail && (cap < 0 || cap >= o.n)) {
    const bool ok = ensure_planes(ctx, full);
    if (std::getenv("WSSR_VERBOSE"))
      std::fprintf(stderr, "[wssr] digit planes (%d digits) for all %lld samples (%s; free %.1f GB)\n",
                   nds, (long long)o.n, ok ? "ok" : "alloc failed", free_b / 1e9);
    return ok ? o.n : 0;
  }
  const int64_t prev = same ? ctx.plan_rows : 0;
  ctx.plan_n = o.n, ctx.plan_p = o.P, ctx.plan_k = k, ctx.plan_rows = 0, ctx.plan_nds = nds;
  ctx.plan_provisional = !(warm && same);
  int64_t rows = (int64_t)(avail / ozaki_planes_bytes(128, o.P, nds)) * 128;
  rows = std::max(rows, prev);  // never shrink an existing plan
  if (cap >= 0) rows = std::min(rows, cap);
  else if (rows < 1024) return 0;
  if (rows <= 0) return 0;
  const bool ok = ensure_planes(ctx, ozaki_planes_bytes(rows, o.P, nds));
  if (!cap_env) ctx.plan_rows = ok ? rows : 0;
  if (std::getenv("WSSR_VERBOSE"))
    std::fprintf(stderr, "[wssr] digit planes (%d digits) for %lld of %lld samples (%s; free %.1f GB, "
                 "avail %.1f GB)\n", nds, (long long)rows, (long long)o.n, ok ? "ok" : "alloc failed",
                 free_b / 1e9, avail / 1e9);
  return ok ? rows : 0;
}

// O-pass GEMMs over the sample block in its storage type
void gemm_samples(Context& ctx, Layout layout, const Ohat& o, int64_t M, int64_t N, int64_t K,
                  const double* B, int64_t ldb, double* C, int64_t ldc, double alpha) {
  GemmArgs a{o.samp, o.lds, B, ldb, o.mu, C, ldc, M, N, K, 0, alpha, 0, nullptr, nullptr, 0};
  if (ctx.ozaki && !ctx.disable_tma && (double)M * (double)K >= ctx.oz_min_elems &&
      ozaki_supported(layout, a, o.f32)) {
    const double* tab = o.scale_tab;
    if (!tab) {
      if (!o.oz_scale) {
        o.oz_scale = std::make_shared<Buf>(ozaki_table_doubles(o.P), ctx.stream);
        WSSR_CUDA(ozaki_scales(ctx, o.samp, o.f32, o.lds, o.n, o.P, o.mu, *o.oz_scale, ctx.stream));
      }
      tab = *o.oz_scale;
    }
    const int8_t* planes = nullptr;
    int8_t* store = nullptr;
    const int nds = sample_digits(ctx, o);
    int64_t n_pl = 0;  // samples covered by planes (or by the store of this first pass)
    if (ctx.oz_pre == 0) {
      if (!o.oz_planes) {
        o.oz_planes = std::make_shared<Ohat::Planes>();
        n_pl = plan_plane_rows(ctx, o, N);
        if (n_pl > 0) {
          if (layout == Layout::RM) {
            // the first pass (v = Ohat^T q) digitises on the fly and writes the planes
            store = ctx.oz_planes;
          } else {
            WSSR_CUDA(ozaki_digitize(ctx, o.samp, o.f32, o.lds, n_pl, o.P, tab, ctx.oz_planes,
                                     ctx.stream, nds));
            planes = ctx.oz_planes;
          }
          o.oz_planes->ptr = ctx.oz_planes;
          o.oz_planes->rows = n_pl;
        }
      } else if (o.oz_planes->ptr) {
        planes = o.oz_planes->ptr;
        n_pl = o.oz_planes->rows;
      }
    }
    // precision guard on the first pass over this operand: the digitising v pass collects the
    // row headroom as it goes; any other first pass reads the block once for it
    std::unique_ptr<Buf> guard_rows;
    unsigned long long* rowcnt = nullptr;
    if (o.status && !o.guard_done && ctx.oz_guard) {
      o.guard_done = true;
      guard_rows = std::make_unique<Buf>((size_t)o.n, ctx.stream);
      rowcnt = reinterpret_cast<unsigned long long*>(guard_rows->p);
      WSSR_CUDA(cudaMemsetAsync(rowcnt, 0, sizeof(double) * o.n, ctx.stream));
      if (layout != Layout::RM || planes) {
        WSSR_CUDA(ozaki_row_headroom(ctx, o.samp, o.f32, o.lds, o.n, o.P, tab, rowcnt, ctx.stream));
        WSSR_CUDA(ozaki_row_guard(ctx, rowcnt, o.n, o.status + 2, ctx.stream));
        rowcnt = nullptr;
      }
    }
    // On-the-fly passes with more than 128 thin columns (k = 256, BASELINE configs[4]) run per
    // 128-column group, each on the transposed kernel (one conversion of a sample tile serves
    // 128 columns; the 64-column kernel would convert it once per 64).  The plane store and the
    // guard's row counts ride on the first group only.
    auto ozaki_fly = [&](const GemmArgs& g, int8_t* st_planes, unsigned long long* rc) {
      constexpr int64_t kGroup = 128;
      if (g.N <= kGroup)
        return ozaki_gemm(ctx, layout, g, o.f32, tab, ctx.stream, nullptr, st_planes, rc, nds);
      for (int64_t c0 = 0; c0 < g.N; c0 += kGroup) {
        GemmArgs sub = g;
        sub.N = std::min<int64_t>(kGroup, g.N - c0);
        sub.B = g.B + c0;
        sub.C = g.C + c0;
        const cudaError_t e = ozaki_gemm(ctx, layout, sub, o.f32, tab, ctx.stream, nullptr,
                                         c0 == 0 ? st_planes : nullptr, c0 == 0 ? rc : nullptr,
                                         nds);
        if (e != cudaSuccess) return e;
      }
      return cudaSuccess;
    };
    if (n_pl == 0 || n_pl >= o.n) {
      // profiling (WSSR_FINE_PHASES): 14 = the step's digitising first pass, 15 = the other
      // row-major (v) passes
      const int fp = (ctx.fine_phases && layout == Layout::RM) ? (store ? 14 : 15) : -1;
      PhaseTimer tm(ctx, fp, 0.0, 0.0);
      if (planes) {
        WSSR_CUDA(ozaki_gemm(ctx, layout, a, o.f32, tab, ctx.stream, planes, store, rowcnt, nds));
      } else {
        WSSR_CUDA(ozaki_fly(a, store, rowcnt));
      }
      if (rowcnt) WSSR_CUDA(ozaki_row_guard(ctx, rowcnt, o.n, o.status + 2, ctx.stream));
      return;
    }
    // planes for samples [0, n_pl), on-the-fly digits for the rest
    const size_t es = o.f32 ? 4 : 8;
    const double* tail = reinterpret_cast<const double*>(
        reinterpret_cast<const char*>(o.samp) + (size_t)n_pl * o.lds * es);
    GemmArgs a1 = a, a2 = a;
    a2.A = tail;
    if (layout == Layout::RM) {  // M = samples: disjoint rows of C
      a1.M = n_pl;
      a2.M = o.n - n_pl;
      a2.C = C + n_pl * ldc;
    } else {                     // K = samples: the second part accumulates
      a1.K = n_pl;
      a2.K = o.n - n_pl;
      a2.B = B + n_pl * ldb;
      a2.accumulate = 1;
    }
    if (planes) {
      WSSR_CUDA(ozaki_gemm(ctx, layout, a1, o.f32, tab, ctx.stream, planes, store, rowcnt, nds));
    } else {
      WSSR_CUDA(ozaki_fly(a1, store, rowcnt));
    }
    WSSR_CUDA(ozaki_fly(a2, nullptr, rowcnt ? rowcnt + n_pl : nullptr));
    if (rowcnt) WSSR_CUDA(ozaki_row_guard(ctx, rowcnt, o.n, o.status + 2, ctx.stream));
    return;
  }
  if (o.f32) {
    if (!gemm_f32_supported(layout, a))
      throw Fail{WSSR_ERR_UNSUPPORTED, "fp32 samples need 16-byte aligned rows (ld % 4 == 0)"};
    WSSR_CUDA(gemm_f32a(ctx, layout, a, 1024, ctx.stream));
  } else {
    WSSR_CUDA(gemm(ctx, layout, a, 1024, ctx.stream));
  }
}

// v (cols x k, ldv) = Ohat^T q   (svdengine.py:133)
void apply_OT(Context& ctx, const Ohat& o, const double* q, int64_t ldq, int64_t k, double* v,
              int64_t ldv) {
  if (o.r > 0) {
    if (o.sh == 0.0) {
      WSSR_CUDA(cudaMemset2DAsync(v, sizeof(double) * ldv, 0, sizeof(double) * k, o.r,
                                  ctx.stream));
    } else {
      gemm_rm(ctx, o.r, k, o.P, o.hist, o.ldh, nullptr, q, ldq, v, ldv, o.sh, false);
    }
  }
  if (o.n > 0) {
    PhaseTimer tm(ctx, 0, 2.0 * o.n * o.P * k, (o.f32 ? 4.0 : 8.0) * o.n * o.P);
    gemm_samples(ctx, Layout::RM, o, o.n, k, o.P, q, ldq, v + o.r * ldv, ldv, o.ss);
  }
}

// u (P x k, ldu) = Ohat v   (svdengine.py:134), summed over ranks: all of it (allreduce), or
// with slice > 0 only this rank's slice of `slice` rows (reduce-scatter; u then has world * slice
// rows of storage)
void apply_O(Context& ctx, const Ohat& o, const double* v, int64_t ldv, int64_t k, double* u,
             int64_t ldu, int64_t slice = 0) {
  if (o.n > 0) {
    PhaseTimer tm(ctx, 1, 2.0 * o.n * o.P * k, (o.f32 ? 4.0 : 8.0) * o.n * o.P);
    gemm_samples(ctx, Layout::CM, o, o.P, k, o.n, v + o.r * ldv, ldv, u, ldu, o.ss);
  } else {
    WSSR_CUDA(cudaMemset2DAsync(u, sizeof(double) * ldu, 0, sizeof(double) * k, o.P, ctx.stream));
  }
  if (o.r > 0 && o.sh != 0.0)
    gemm_cm(ctx, o.P, k, o.r, o.hist, o.ldh, nullptr, v, ldv, u, ldu, o.sh, true);
  if (ctx.world() > 1) {
    if (ldu != k) throw Fail{WSSR_ERR_VALUE, "sharded apply_O needs a dense output"};
    if (slice > 0) {
      if (ctx.comm->reduce_scatter_sum(u, (size_t)(slice * k), ctx.stream) != cudaSuccess)
        throw Fail{WSSR_ERR_NCCL, "reduce-scatter failed"};
    } else {
      allreduce(ctx, u, (size_t)(o.P * k));
    }
  }
}

// Tail sharding of a row-sharded run: the P x k blocks of the SSI (q, u, w) are worked on in
// P-slices, one per rank - u and w arrive by reduce-scatter instead of allreduce, the
// CholeskyQR2 of each block runs on the slice (k x k Grams allreduced) and q is all-gathered
// for the next O-pass - so the P x k work of a step divides by the number of ranks and the u
// exchange costs what the allreduce did.  Slices are S = ceil(P / world) rows; storage is padded
// to world * S rows (the pad rows of the last slice are never read).  The careful (reference
// Gram-Schmidt) re-run stays replicated.
struct PSlice {
  bool on = false;
  int64_t S = 0, p0 = 0, rows = 0, padded = 0;
};
PSlice p_slice(const Context& ctx, int64_t P, bool careful) {
  PSlice sl;
  sl.rows = sl.padded = sl.S = P;
  const int G = ctx.world();
  if (G <= 1 || !ctx.tail_shard || careful) return sl;
  const int64_t S = (P + G - 1) / G;
  if (S * (G - 1) >= P) return sl;  // the last rank would have no rows
  sl.on = true;
  sl.S = S;
  sl.p0 = (int64_t)ctx.comm->rank * S;
  sl.rows = std::min(S, P - sl.p0);
  sl.padded = S * G;
  return sl;
}

// ||Ohat||_F^2 (svdengine.py:118,129): history block plus the sample block (known from
// assemble, or computed).  Returns the host value (global over ranks).
double ohat_fro2(Context& ctx, const Ohat& o, double samples_fro2, bool hist_owned) {
  double total = 0.0;
  Buf s(1, ctx.stream);
  if (o.r > 0 && o.sh != 0.0 && hist_owned) {
    sumsq_matrix(ctx, o.hist, o.r, o.P, o.ldh, s, o.sh * o.sh);
    total += read_scalar(ctx, s);
  }
  if (o.n > 0 || ctx.world() > 1) {
    if (samples_fro2 >= 0.0) {
      total += samples_fro2;
    } else {
      if (o.mu || o.f32)
        throw Fail{WSSR_ERR_VALUE, "samples_fro2 required for a centred or fp32 block"};
      sumsq_matrix(ctx, o.samp, o.n, o.P, o.lds, s, o.ss * o.ss);
      allreduce(ctx, s, 1);
      total += read_scalar(ctx, s);
    }
  }
  return total;
}

// ||Ohat||_F^2: a host part plus, when assemble deferred its scalars, a device part read back at
// the first host synchronisation of the SSI (so the step never waits on assemble).
struct Fro2 {
  double host = 0.0;
  const double* dev = nullptr;
  double dev_scale = 1.0;
  double dev_val = 0.0;
  bool enqueued = false;
  double* stage = nullptr;  // pinned slot the device value is copied into
  void enqueue(Context& ctx) {
    if (dev && !enqueued) {
      stage = ctx.hbuf + 3;
      d2h(ctx, stage, dev, sizeof(double));
      enqueued = true;
    }
  }
  // valid after a stream sync that follows enqueue()
  double value() {
    if (dev && stage) {
      dev_val = *stage;
      stage = nullptr;
    }
    return dev ? host + dev_scale * dev_val : host;
  }
};

// ---- ssi_svd (svdengine.py:88-158) ------------------------------------------------------------
struct SsiResult {
  int64_t k_pos = 0, r_eff = 0, iterations = 0;
  double residual = std::numeric_limits<double>::quiet_NaN();
  double sigma0 = 0.0;
  Buf qv;          // (cols x k) right vectors, columns already in sorted order
  Buf order;       // int64 [k]
};

// U_out (P x k, ldU) gets the re-orthonormalised left vectors (first k_pos columns), sigma_out
// the sorted values.  fro2 is the global ||Ohat||_F^2.
SsiResult ssi_core(Context& ctx, const Ohat& o, int64_t k, int64_t max_iters,
                   const double* u_init, int64_t ld_init, double tol, Fro2& fro2_in, bool final_res,
                   bool careful, double* U_out, int64_t ldU, double* sigma_out, double r_reg,
                   int* status) {
  const int64_t P = o.P, cols = o.cols();
  const bool dist = ctx.world() > 1;
  cudaStream_t st = ctx.stream;
  o.status = status;  // the O-passes' precision guard reports into status[2]
  const PSlice sl = p_slice(ctx, P, careful);
  Buf qbuf((size_t)sl.padded * k, st), ua((size_t)sl.padded * k, st),
      ub((size_t)sl.padded * k, st);
  double* q = qbuf;
  const int64_t r0 = sl.on ? sl.p0 : 0, nr = sl.on ? sl.rows : P;  // rows this rank works on
  // q = QR(in) on this rank's slice (k x k Grams allreduced), then all-gathered; or replicated
  auto qr_block = [&](const double* in, int64_t ldin, double* out) {
    qr(ctx, nr, k, in + r0 * ldin, ldin, out + r0 * k, k, nullptr, status, careful, sl.on);
    if (sl.on && ctx.comm->all_gather(out, (size_t)(sl.S * k), st) != cudaSuccess)
      throw Fail{WSSR_ERR_NCCL, "all-gather failed"};
  };
  const int64_t scatter = sl.on ? sl.S : 0;
  Buf va((size_t)std::max<int64_t>(cols, 1) * k, st), vb((size_t)std::max<int64_t>(cols, 1) * k, st);
  Buf quot((size_t)k * k, st), scal(4, st);
  double* u = ua;
  double* w = ub;
  double* v = va;
  double* v2 = vb;

  qr_block(u_init, ld_init, q);  // svdengine.py:130
  apply_OT(ctx, o, q, k, k, v, k);
  apply_O(ctx, o, v, k, k, u, k, scatter);
  SsiResult res;
  int64_t it = 0;
  bool deferred_residual = false;
  while (true) {  // svdengine.py:132-142
    // the last iteration's q is the returned U when the order comes out sorted
    // (svdengine.py:151): write it there directly
    if (it + 1 == max_iters && ldU == k && U_out && !sl.on) q = U_out;
    qr_block(u, k, q);
    ++it;
    if (it >= max_iters && !final_res) {
      res.residual = std::numeric_limits<double>::quiet_NaN();  // look-ahead skipped
      break;
    }
    // look-ahead pass: w = Ohat Ohat^T q is also the next iteration's u (svdengine.py:137)
    apply_OT(ctx, o, q, k, k, v2, k);
    apply_O(ctx, o, v2, k, k, w, k, scatter);
    {
      PhaseTimer tm(ctx, 4, 0.0, 0.0);
      const double* qs = q + r0 * k;
      const double* ws = w + r0 * k;
      cross(ctx, nr, k, qs, k, ws, k, quot);  // quotient = q^T w
      if (sl.on) allreduce(ctx, quot, (size_t)(k * k));
      if (ctx.tallskinny && ts_mul_supported(k, qs, k, ws, k)) {
        // ||w - q quotient||_F^2 straight from registers (nothing written)
        WSSR_CUDA(ts_mul_add_sumsq(ctx, nr, k, qs, k, quot, -1.0, ws, k, scal));
      } else {
        Buf tmp((size_t)nr * k, st);
        sub_mul_small(ctx, nr, k, qs, k, quot, ws, k, tmp, k);  // w - q quotient
        sumsq_matrix(ctx, tmp, nr, k, k, scal);
      }
      if (sl.on) allreduce(ctx, scal, 1);
      launch_pdl(small_norms_kernel, 1, 256, 0, st, nullptr, nullptr, 0, quot, (int)k, scal + 1);
      post_launch(ctx);
    }
    double* h = ctx.hbuf;  // pinned: the copies are asynchronous
    d2h(ctx, h, scal, 3 * sizeof(double));
    fro2_in.enqueue(ctx);
    if (it >= max_iters) {
      // the loop ends whatever the residual is: read it at the next synchronisation (the rank
      // cut) instead of waiting here
      deferred_residual = true;
      break;
    }
    sync(ctx);
    const double fro2 = fro2_in.value();
    if (fro2 == 0.0) throw Fail{WSSR_ERR_DEGENERATE_INPUT, "cannot factorize an all-zero matrix"};
    const double residual = std::sqrt(h[0]) / fro2;
    const double mixing = h[2] / fro2;
    res.residual = residual;
    if (std::max(residual, mixing) < tol) break;
    std::swap(v, v2);
    std::swap(u, w);
  }
  res.iterations = it;

  // sigma from the QR of the final v block, sorted (svdengine.py:144-150)
  Buf qv_raw((size_t)std::max<int64_t>(cols, 1) * k, st), Rv((size_t)k * k, st);
  qr(ctx, cols, k, v, k, qv_raw, k, Rv, status, careful, dist);
  res.order = Buf(k, st);
  Buf ints(1, st);
  launch_pdl(sort_sigma_kernel, 1, 256, sizeof(double) * k, st, Rv, (int)k, r_reg, res.order.i64(),
                                                       sigma_out, ints.i32());
  post_launch(ctx);
  // one synchronisation for the counts, the top value, the order (and a deferred residual);
  // staged through pinned memory so the copies do not each block the host
  const bool big_k = 16 + k > 4096;
  std::vector<int64_t> hord_big(big_k ? k : 0);
  int* hi = reinterpret_cast<int*>(ctx.hbuf + 8);
  double* hsig0 = ctx.hbuf + 9;
  int64_t* hord = big_k ? hord_big.data() : reinterpret_cast<int64_t*>(ctx.hbuf + 16);
  d2h(ctx, hi, ints, 2 * sizeof(int));
  d2h(ctx, hsig0, sigma_out, sizeof(double));
  d2h(ctx, hord, res.order, sizeof(int64_t) * k);
  sync(ctx);
  if (deferred_residual) {
    const double fro2 = fro2_in.value();
    if (fro2 == 0.0) throw Fail{WSSR_ERR_DEGENERATE_INPUT, "cannot factorize an all-zero matrix"};
    res.residual = std::sqrt(ctx.hbuf[0]) / fro2;
  }
  res.sigma0 = *hsig0;
  res.k_pos = hi[0];
  res.r_eff = hi[1];
  if (res.k_pos == 0)
    throw Fail{WSSR_ERR_DEGENERATE_INPUT, "iteration produced no positive singular values"};
  const int64_t kp = res.k_pos;
  // U = QR(u[:, order[:k]]) and V = q_v[:, order] (svdengine.py:151-152).  When the order is
  // the identity the QR is exactly the one already computed at the top of the last iteration
  // (q = QR(u), same inputs, same deterministic kernels), so it is reused.
  bool identity = kp == k;
  for (int64_t j = 0; j < kp && identity; ++j) identity = hord[j] == j;
  if (identity) {
    if (q != U_out) copy2d(ctx, q, k, P, k, 1.0, U_out, ldU);
  } else if (sl.on) {
    // this rank's slice of u, permuted, QR'd on the slices and all-gathered
    Buf uperm((size_t)sl.padded * kp, st), ufull((size_t)sl.padded * kp, st);
    launch_pdl(gather_cols_kernel, blocks_for(nr * kp, 256, 16 * ctx.num_sms), 256, 0, st,
               (const double*)(u + r0 * k), k, nr, res.order.i64(), (int)kp,
               uperm.p + r0 * kp, kp);
    post_launch(ctx);
    qr(ctx, nr, kp, uperm.p + r0 * kp, kp, ufull.p + r0 * kp, kp, nullptr, status, careful,
       true);
    if (ctx.comm->all_gather(ufull, (size_t)(sl.S * kp), st) != cudaSuccess)
      throw Fail{WSSR_ERR_NCCL, "all-gather failed"};
    copy2d(ctx, ufull, kp, P, kp, 1.0, U_out, ldU);
  } else {
    Buf uperm((size_t)P * kp, st);
    launch_pdl(gather_cols_kernel, blocks_for(P * kp, 256, 16 * ctx.num_sms), 256, 0, st, 
        u, k, P, res.order.i64(), (int)kp, uperm, kp);
    post_launch(ctx);
    qr(ctx, P, kp, uperm, kp, U_out, ldU, nullptr, status, careful, false);
  }
  res.qv = Buf((size_t)std::max<int64_t>(cols, 1) * k, st);
  if (cols > 0) {
    launch_pdl(gather_cols_kernel, blocks_for(cols * kp, 256, 16 * ctx.num_sms), 256, 0, st, 
        qv_raw, k, cols, res.order.i64(), (int)kp, res.qv, k);
    post_launch(ctx);
  }
  return res;
}

// Runs the SSI optimistically (no per-QR host checks); if any CholeskyQR2 flagged a block it
// could not resolve, re-runs in careful mode, which reproduces the reference's QR branches.  If
// the int8 O-passes' precision guard fired (status[2]: a sample row far below its columns' digit
// scales, ozaki.cu row_guard_kernel), the SSI is re-run with the O-passes on FP64 DMMA.
// Device status words: [0] CholeskyQR2 could not resolve a block, [1] zero matrix, [2] guard.
__global__ void flag_to_double_kernel(const int* f, double* d) {
  pdl_wait();
  if (threadIdx.x == 0) d[0] = f[0] ? 1.0 : 0.0;
}
__global__ void double_to_flag_kernel(const double* d, int* f) {
  pdl_wait();
  if (threadIdx.x == 0) f[0] = d[0] > 0.0 ? 1 : 0;
}
// OR of a device int flag over the ranks (row-sharded runs take the same fallback branch)
void allreduce_flag(Context& ctx, int* flag) {
  if (ctx.world() <= 1) return;
  Buf d(1, ctx.stream);
  launch_pdl(flag_to_double_kernel, 1, 32, 0, ctx.stream, (const int*)flag, d.p);
  post_launch(ctx);
  allreduce(ctx, d, 1);
  launch_pdl(double_to_flag_kernel, 1, 32, 0, ctx.stream, (const double*)d.p, flag);
  post_launch(ctx);
}

template <class F>
auto with_fallback(Context& ctx, int64_t flags, F&& body) -> decltype(body(false, (int*)nullptr)) {
  struct OzakiRestore {
    Context& c;
    bool saved;
    ~OzakiRestore() { c.ozaki = saved; }
  } restore{ctx, ctx.ozaki};
  bool careful = (flags & WSSR_FLAG_CAREFUL) != 0;
  int* hs = reinterpret_cast<int*>(ctx.hbuf + 4);
  while (true) {
    Buf status(2, ctx.stream);
    WSSR_CUDA(cudaMemsetAsync(status, 0, 2 * sizeof(double), ctx.stream));
    if (careful && !ctx.ozaki) return body(true, status.i32());
    try {
      auto r = body(careful, status.i32());
      if (ctx.ozaki) allreduce_flag(ctx, status.i32() + 2);
      d2h(ctx, hs, status, 3 * sizeof(int));
      sync(ctx);
      if (hs[2] == 0 && (careful || hs[0] == 0)) return r;
    } catch (const Fail& f) {
      // a host-side verdict (no positive singular values, ...) reached on the values of a block
      // the optimistic pass could not factorise is not the reference's verdict: re-run carefully
      if (f.code == WSSR_ERR_CUDA || f.code == WSSR_ERR_NCCL) throw;
      d2h(ctx, hs, status, 3 * sizeof(int));
      sync(ctx);
      if (hs[2] == 0 && (careful || hs[0] == 0)) throw;
    }
    if (hs[2] != 0) {
      if (std::getenv("WSSR_VERBOSE"))
        std::fprintf(stderr, "[wssr] precision guard: heavy-tailed sample rows, O-passes on DMMA\n");
      ctx.ozaki = false;
      ++ctx.precision_fallbacks;
    }
    if (hs[0] != 0) careful = true;
  }
}

// ---- largest eigenvalue of a small symmetric matrix ---------------------------------------
void maxeig(Context& ctx, const double* A, int k, double* out_dev) {
  if (k <= 64) {
    launch_pdl(maxeig64_kernel, 1, 1024, 0, ctx.stream, A, k, out_dev, nullptr);
    return;
  }
  const size_t smem = sizeof(double) * ((size_t)k * (k + 1) + 4 * (size_t)k);
  if (smem <= 200 * 1024) {
    static std::atomic<uint64_t> attr{0};
    WSSR_CUDA(smem_attr_once(attr, maxeig_smem_kernel, 200 * 1024));
    launch_pdl(maxeig_smem_kernel, 1, 256, smem, ctx.stream, A, k, out_dev);
  } else {
    Buf W((size_t)k * (k + 1) + 4 * (size_t)k, ctx.stream);
    launch_pdl(maxeig_gmem_kernel, 1, 256, 0, ctx.stream, A, k, W, out_dev);
  }
}

// ---- subspace_drift (svdengine.py:199-226) ----------------------------------------------------
// {sigma_drift, projector_drift} from {||s1 - s2||, -, lambda_max}: sqrt and the 1e-12 -> 0 rule
// (svdengine.py:222-225)
__global__ void drift_finalize_kernel(const double* __restrict__ in, double* __restrict__ out) {
  pdl_wait();
  if (threadIdx.x == 0) {
    double sd = in[0];
    double pd = sqrt(fmax(in[2], 0.0));
    out[0] = sd < 1e-12 ? 0.0 : sd;
    out[1] = pd < 1e-12 ? 0.0 : pd;
  }
}

// Enqueue the drift on ctx.stream; out2 (device, 2 doubles) = {sigma_drift, projector_drift}.
// sliced (row-sharded runs with the P-sliced tail): u1 and u2 are replicated, so each rank works
// its own P-slice of the two P x r passes and the r x r cross product and Gram are allreduced.
void drift_enqueue(Context& ctx, int64_t rows, const double* u1, int64_t ld1, const double* s1,
                   int64_t r, const double* u2, int64_t ld2, const double* s2, double* out2,
                   bool sliced = false) {
  cudaStream_t st = ctx.stream;
  if (sliced) {
    const PSlice sl = p_slice(ctx, rows, false);
    sliced = sl.on;
    if (sl.on) {
      u1 += sl.p0 * ld1;
      u2 += sl.p0 * ld2;
      rows = sl.rows;
    }
  }
  Buf C((size_t)r * r, st), X((size_t)rows * r, st), GX((size_t)r * r, st), out(3, st);
  launch_pdl(small_norms_kernel, 1, 256, 0, st, s1, s2, (int)r, nullptr, 0, out);
  post_launch(ctx);
  cross(ctx, rows, r, u1, ld1, u2, ld2, C);                  // u1^T u2
  if (sliced) allreduce(ctx, C, (size_t)(r * r));
  sub_mul_small(ctx, rows, r, u1, ld1, C, u2, ld2, X, r);    // u2 - u1 (u1^T u2)
  gram(ctx, rows, r, X, r, GX, sliced);
  maxeig(ctx, GX, (int)r, out + 2);
  post_launch(ctx);
  launch_pdl(drift_finalize_kernel, 1, 32, 0, st, (const double*)out, out2);
  post_launch(ctx);
}

std::pair<double, double> drift(Context& ctx, int64_t rows, const double* u1, int64_t ld1,
                                const double* s1, int64_t r1, const double* u2, int64_t ld2,
                                const double* s2, int64_t r2, bool sliced = false) {
  const int64_t r = std::min(r1, r2);
  if (r == 0) return {0.0, 0.0};
  Buf out2(2, ctx.stream);
  {
    PhaseTimer tm(ctx, 5, 0.0, 0.0);
    drift_enqueue(ctx, rows, u1, ld1, s1, r, u2, ld2, s2, out2, sliced);
  }
  double h[2];
  d2h(ctx, h, out2, sizeof(h));
  sync(ctx);
  return {h[0], h[1]};
}

// ---- estimators.assemble (estimators.py:74-100) --------------------------------------------
__global__ void merge_rank_stats_kernel(int64_t p, double n_local, double n_global,
                                        const double* mu_loc, const double* m2_loc,
                                        const double* g_loc, double lsum_loc, const double* mu,
                                        double* m2_out, double* g_out) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = mu_loc[i] - mu[i];
    m2_out[i] = n_local > 0 ? m2_loc[i] + n_local * d * d : 0.0;
    g_out[i] = n_local > 0 ? g_loc[i] + d * lsum_loc : 0.0;
  }
}
__global__ void scale_kernel(int64_t n, double a, const double* x, double* y) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a * x[i];
}

template <typename T>
void assemble(Context& ctx, const T* derivs, int64_t n, int64_t p, int64_t ld,
              const double* energies, double n_std, wssr_assemble_out* out) {
  cudaStream_t st = ctx.stream;
  const bool dist = ctx.world() > 1;
  int64_t n_global = n;
  int64_t offset = 0;
  if (dist) {
    // global sample count and this rank's offset (exact in doubles for n < 2^53)
    Buf cnt(ctx.world(), st);
    WSSR_CUDA(cudaMemsetAsync(cnt, 0, sizeof(double) * ctx.world(), st));
    const double nd = (double)n;
    WSSR_CUDA(cudaMemcpyAsync(cnt + ctx.comm->rank, &nd, sizeof(double), cudaMemcpyHostToDevice, st));
    allreduce(ctx, cnt, ctx.world());
    std::vector<double> h(ctx.world());
    d2h(ctx, h.data(), cnt, sizeof(double) * h.size());
    sync(ctx);
    n_global = 0;
    for (int r = 0; r < ctx.world(); ++r) {
      if (r < ctx.comm->rank) offset += (int64_t)h[r];
      n_global += (int64_t)h[r];
    }
  }
  out->n_global = n_global;
  if (n_global < 2) throw Fail{WSSR_ERR_DEGENERATE_BATCH, "need at least two samples to center the batch"};
  if (std::isfinite(n_std) && n_std < 0.0)
    throw Fail{WSSR_ERR_VALUE, "clipping width must be nonnegative"};
  const double scale = 1.0 / std::sqrt((double)n_global);
  const int clip = std::isfinite(n_std) ? 1 : 0;

  // energy statistics on the full (gathered) energy vector; each rank keeps its slice of L
  Buf e_all, l_all((size_t)n_global, st), lraw_all((size_t)n_global, st), scal(4, st);
  const double* E = energies;
  if (dist) {
    e_all = Buf((size_t)n_global, st);
    WSSR_CUDA(cudaMemsetAsync(e_all, 0, sizeof(double) * n_global, st));
    WSSR_CUDA(cudaMemcpyAsync(e_all + offset, energies, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    allreduce(ctx, e_all, (size_t)n_global);
    E = e_all;
  }
  launch_pdl(energy_stats_kernel, 1, 1024, 0, st, E, n_global, n_std, clip, scale, l_all, lraw_all, scal);
  post_launch(ctx);
  WSSR_CUDA(cudaMemcpyAsync(out->l_vector, l_all + offset, sizeof(double) * n,
                            cudaMemcpyDeviceToDevice, st));
  const double* lraw = lraw_all + offset;

  // one pass over O: column means, centred second moments, centred gradient sums
  Buf m2(p, st), gsum(p, st), cext;
  double* cmin = nullptr;
  double* cmax = nullptr;
  if (out->scale_table && n > 0) {
    cext = Buf((size_t)2 * p, st);
    cmin = cext;
    cmax = cext + p;
  }
  if (n > 0) {
    PhaseTimer tm(ctx, 2, 4.0 * n * p, (double)sizeof(T) * n * p);
    const bool al16 = (reinterpret_cast<uintptr_t>(derivs) & 15) == 0;
    if (sizeof(T) == 8 && ld % 2 == 0 && al16) {
      launch_pdl(colstats_kernel<T, 2, 8>, (unsigned)((p + 63) / 64), 32 * kColStatsWarps, 0, st, 
          derivs, n, p, ld, lraw, out->mu, m2, gsum, cmin, cmax);
    } else if (sizeof(T) == 4 && ld % 4 == 0 && al16) {
      launch_pdl(colstats_kernel<T, 4, 8>, (unsigned)((p + 127) / 128), 32 * kColStatsWarps, 0, st, 
          derivs, n, p, ld, lraw, out->mu, m2, gsum, cmin, cmax);
    } else {
      launch_pdl(colstats_kernel<T, 1, 8>, (unsigned)((p + 31) / 32), 32 * kColStatsWarps, 0, st, 
          derivs, n, p, ld, lraw, out->mu, m2, gsum, cmin, cmax);
    }
    post_launch(ctx);
  } else {
    WSSR_CUDA(cudaMemsetAsync(out->mu, 0, sizeof(double) * p, st));
    WSSR_CUDA(cudaMemsetAsync(m2, 0, sizeof(double) * p, st));
    WSSR_CUDA(cudaMemsetAsync(gsum, 0, sizeof(double) * p, st));
  }
  if (dist) {
    // mu = sum_r n_r mu_r / N ; M2 = sum_r [M2_r + n_r (mu_r - mu)^2] ; G likewise
    Buf mu_loc(p, st), mu(p, st), lsum(1, st);
    WSSR_CUDA(cudaMemcpyAsync(mu_loc, out->mu, sizeof(double) * p, cudaMemcpyDeviceToDevice, st));
    launch_pdl(scale_kernel, blocks_for(p, 256, 8 * ctx.num_sms), 256, 0, st, p, (double)n, mu_loc, mu);
    post_launch(ctx);
    allreduce(ctx, mu, p);
    launch_pdl(scale_kernel, blocks_for(p, 256, 8 * ctx.num_sms), 256, 0, st, p, 1.0 / n_global, mu, mu);
    post_launch(ctx);
    Buf parts(1, st);
    launch_pdl(reduce_final_kernel, 1, 256, 0, st, lraw, (int)n, 1.0, lsum);
    post_launch(ctx);
    const double lsum_h = read_scalar(ctx, lsum);
    launch_pdl(merge_rank_stats_kernel, blocks_for(p, 256, 8 * ctx.num_sms), 256, 0, st, 
        p, (double)n, (double)n_global, mu_loc, m2, gsum, lsum_h, mu, m2, gsum);
    post_launch(ctx);
    allreduce(ctx, m2, p);
    allreduce(ctx, gsum, p);
    WSSR_CUDA(cudaMemcpyAsync(out->mu, mu, sizeof(double) * p, cudaMemcpyDeviceToDevice, st));
  }
  if (out->scale_table) {
    if (n > 0) {
      WSSR_CUDA(ozaki_scales_minmax(ctx, cmin, cmax, out->mu, p, out->scale_table, st));
    } else {
      WSSR_CUDA(ozaki_table_clear(ctx, out->scale_table, p, st));  // padding slots only
    }
  }
  // gradient = 2 * o_matrix @ l_vector = 2 * gsum / N   (estimators.py:93)
  launch_pdl(scale_kernel, blocks_for(p, 256, 8 * ctx.num_sms), 256, 0, st, p, 2.0 / n_global, gsum,
                                                                     out->gradient);
  post_launch(ctx);
  Buf fro(1, st);
  {
    const int nb = (int)std::min<int64_t>(2 * ctx.num_sms, (p + 255) / 256);
    const int64_t chunk = (p + nb - 1) / nb;
    const int nbb = (int)((p + chunk - 1) / chunk);
    Buf part(nbb, st);
    launch_pdl(reduce_partials_kernel, nbb, 256, 0, st, m2, p, chunk, 0, part);
    post_launch(ctx);
    launch_pdl(reduce_final_kernel, 1, 256, 0, st, part, nbb, 1.0 / n_global, fro);
    post_launch(ctx);
  }
  if (out->deferred && !dist) {
    // stream-ordered host scalars; the caller synchronises before reading them
    if (out->fro2_dev)
      WSSR_CUDA(cudaMemcpyAsync(out->fro2_dev, fro, sizeof(double), cudaMemcpyDeviceToDevice, st));
    d2h(ctx, out->deferred, scal, 4 * sizeof(double));
    d2h(ctx, out->deferred + 4, fro, sizeof(double));
    out->loss = out->raw_loss = out->e_mean = out->e_std = out->fro2 =
        std::numeric_limits<double>::quiet_NaN();
    return;
  }
  double hs[4];
  d2h(ctx, hs, scal, sizeof(hs));
  d2h(ctx, &out->fro2, fro, sizeof(double));
  sync(ctx);
  out->loss = hs[0];
  out->raw_loss = hs[1];
  out->e_mean = hs[2];
  out->e_std = hs[3];
}

// ---- dense SVD (linalg.py:108-121) for min(m, n) <= 512 ---------------------------------------
// QR pre-reduction of the tall orientation (the reference's QR with its deficiency patch), then
// one-sided Jacobi on the small square R.  Singular vectors carry an arbitrary joint sign, like
// LAPACK's; everything the WSSR step derives from them (update, obar obar^T, obar lbar) is
// sign-invariant.
constexpr int64_t kDenseSvdMax = 512;

void transpose(Context& ctx, const double* in, int64_t ldi, int64_t rows, int64_t cols,
               const double* shift, double scale, double* out, int64_t ldo) {
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
  launch_pdl(transpose_shift_kernel, grid, dim3(32, 8), 0, ctx.stream, in, ldi, rows, cols, shift, scale,
                                                               out, ldo);
  post_launch(ctx);
}

// Dense SVD for min(m, n) > kDenseSvdMax: blocked one-sided Jacobi (jacobi.cuh) directly on the
// min(m, n) vectors of A (no QR pre-reduction: the step-0 Ohat is exactly rank-deficient - its
// sample columns sum to zero - which CholeskyQR cannot factor; one-sided Jacobi needs no full
// rank and keeps high relative accuracy).
void dense_svd_blocked(Context& ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                       double* U, int64_t ldu, double* S, double* VT, int64_t ldvt) {
  cudaStream_t st = ctx.stream;
  const bool by_cols = m >= n;  // vectors: the columns of A (X = A^T) or its rows (X = A)
  const int64_t nv = by_cols ? n : m, L = by_cols ? m : n;
  int nb = (int)((nv + 15) / 16);
  nb += nb & 1;
  const int64_t nvp = 16 * (int64_t)nb, ldx = L + (L & 1);  // even ld: 16-byte aligned rows
  Buf X((size_t)(nvp * ldx), st), Wm((size_t)(nvp * nvp), st), sig((size_t)(2 * nv + 2), st);
  WSSR_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * nvp * ldx, st));
  if (by_cols)
    transpose(ctx, A, lda, m, n, nullptr, 1.0, X, ldx);  // X (n x m) = A^T
  else
    copy2d(ctx, A, lda, m, n, 1.0, X, ldx);
  launch_pdl(bj::identity_kernel, blocks_for(nvp * nvp, 256, 16 * ctx.num_sms), 256, 0, st,
             Wm.p, nvp);
  post_launch(ctx);
  static std::atomic<uint64_t> attr{0};
  WSSR_CUDA(smem_attr_once(attr, bj::round_kernel, (int)bj::kSmem));
  // rounding of a length-L Gram entry grows like sqrt(L) eps (LAPACK dgesvj uses sqrt(m) eps)
  const double tol = std::max(1e-15, 4.0 * std::numeric_limits<double>::epsilon() *
                                          std::sqrt((double)L));
  int* rotated = reinterpret_cast<int*>(sig.p + 2 * nv);
  int* h_rot = reinterpret_cast<int*>(ctx.hbuf + 4000);
  auto sweep = [&](double t) {
    WSSR_CUDA(cudaMemsetAsync(rotated, 0, sizeof(int), st));
    for (int round = 0; round < nb - 1; ++round) {
      launch_pdl(bj::round_kernel, nb / 2, bj::kThreads, bj::kSmem, st, X.p, ldx, L, Wm.p, nvp,
                 nb, round, t, rotated);
      post_launch(ctx);
    }
  };
  int sweeps = 0;
  for (; sweeps < 60; ++sweeps) {
    sweep(tol);
    d2h(ctx, h_rot, rotated, sizeof(int));
    sync(ctx);
    if (*h_rot == 0) break;
  }
  if (sweeps >= 60) throw Fail{WSSR_ERR_DEGENERATE_INPUT, "dense SVD: Jacobi did not converge"};
  // polish: two sweeps that rotate every pair measurably off orthogonal (tol = eps) take the
  // remaining cosines from the convergence threshold down to the noise of the Gram itself
  for (int i = 0; i < 2; ++i) sweep(std::numeric_limits<double>::epsilon());
  sweeps += 2;
  double* norms = sig.p;
  double* sorted = sig.p + nv;
  Buf order((size_t)(nv + 1) / 2 + 1, st);
  int* ord = order.i32();
  launch_pdl(bj::row_norms_kernel, blocks_for(nv * 32, 256, 16 * ctx.num_sms), 256, 0, st, X.p,
             ldx, L, (int)nv, norms);
  post_launch(ctx);
  launch_pdl(bj::rank_kernel, blocks_for(nv, 128, 16 * ctx.num_sms), 128, 0, st, norms, (int)nv,
             ord, sorted);
  post_launch(ctx);
  WSSR_CUDA(cudaMemcpyAsync(S, sorted, sizeof(double) * nv, cudaMemcpyDeviceToDevice, st));
  const int q = (int)nv;
  if (by_cols) {
    // A W^T = X_final^T = U Sigma: U[:, j] = X[order_j]^T / sigma_j, V^T[j] = W[order_j]
    dim3 grid((unsigned)((m + 31) / 32), (unsigned)((q + 31) / 32));
    launch_pdl(bj::gather_transpose_kernel, grid, dim3(32, 8), 0, st, X.p, ldx, m, ord, sorted,
               q, 1, U, ldu);
    post_launch(ctx);
    launch_pdl(bj::gather_rows_kernel, blocks_for((int64_t)q * n, 256, 16 * ctx.num_sms), 256, 0,
               st, Wm.p, nvp, n, ord, sorted, q, 0, VT, ldvt);
    post_launch(ctx);
  } else {
    // A = W^T X_final: U[:, j] = W[order_j]^T, V^T[j] = X[order_j] / sigma_j
    dim3 grid((unsigned)((m + 31) / 32), (unsigned)((q + 31) / 32));
    launch_pdl(bj::gather_transpose_kernel, grid, dim3(32, 8), 0, st, Wm.p, nvp, m, ord, sorted,
               q, 0, U, ldu);
    post_launch(ctx);
    launch_pdl(bj::gather_rows_kernel, blocks_for((int64_t)q * n, 256, 16 * ctx.num_sms), 256, 0,
               st, X.p, ldx, n, ord, sorted, q, 1, VT, ldvt);
    post_launch(ctx);
  }
  ctx.dense_svd_sweeps = sweeps + 1;
}

void dense_svd(Context& ctx, int64_t m, int64_t n, const double* A, int64_t lda, double* U,
               int64_t ldu, double* S, double* VT, int64_t ldvt) {
  cudaStream_t st = ctx.stream;
  const int64_t q = std::min(m, n), rows = std::max(m, n);
  if (q > kDenseSvdMax || ctx.force_blocked_svd) {
    dense_svd_blocked(ctx, m, n, A, lda, U, ldu, S, VT, ldvt);
    return;
  }
  Buf T;
  const double* Tp = A;
  int64_t ldt = lda;
  if (m < n) {
    T = Buf((size_t)n * m, st);
    transpose(ctx, A, lda, m, n, nullptr, 1.0, T, m);
    Tp = T;
    ldt = m;
  }
  Buf Q((size_t)rows * q, st), R((size_t)q * q, st);
  qr(ctx, rows, q, Tp, ldt, Q, q, R, nullptr, true, false);
  Buf W((size_t)q * q, st), V((size_t)q * q, st), Us((size_t)q * q, st), Vs((size_t)q * q, st),
      sw(1, st);
  copy2d(ctx, R, q, q, q, 1.0, W, q);
  launch_pdl(jacobi_svd_kernel, 1, 1024, 0, st, W, V, (int)q, (int)q, 60, sw.i32());
  post_launch(ctx);
  launch_pdl(svd_finalize_kernel, 1, 1024, 2 * sizeof(double) * q, st, W, V, (int)q, (int)q, S, Us, Vs,
                                                              (int)q);
  post_launch(ctx);
  if (m >= n) {
    gemm_rm(ctx, m, q, q, Q, q, nullptr, Us, q, U, ldu, 1.0, false);  // u = Q U_R
    transpose(ctx, Vs, q, q, q, nullptr, 1.0, VT, ldvt);              // vt = V_R^T
  } else {
    copy2d(ctx, Vs, q, q, q, 1.0, U, ldu);                            // u = V_R
    Buf QU((size_t)n * q, st);
    gemm_rm(ctx, n, q, q, Q, q, nullptr, Us, q, QU, q, 1.0, false);
    transpose(ctx, QU, q, n, q, nullptr, 1.0, VT, ldvt);             // vt = (Q U_R)^T
  }
}

// Ohat (P x cols, parameter-major like optimizers.py:323) written out explicitly - only the
// dense backends need it.
void materialize_ohat(Context& ctx, const wssr_ohat_f64& oh, double delta, double* out,
                      int64_t ldo) {
  if (oh.samples_f32)
    throw Fail{WSSR_ERR_UNSUPPORTED, "dense backends need float64 samples"};
  const double sh = std::sqrt(delta) * oh.hist_scale, ss = std::sqrt(1.0 - delta) * oh.samples_scale;
  const int64_t P = oh.n_params, r = oh.hist_rank;
  if (r > 0) transpose(ctx, oh.hist, oh.hist_ld, r, P, nullptr, sh, out, ldo);
  if (oh.n_samples > 0)
    transpose(ctx, oh.samples, oh.samples_ld, oh.n_samples, P, oh.mu, ss, out + r, ldo);
}

// ---- exact truncated SVD without forming Ohat (svdengine.py:75-85 -> linalg.py:108-121) --------
// The dense first step factorises the P x (r + N) Ohat.  Written out it is as large as the sample
// block itself (137 GB at BASELINE configs[2], on every rank under row sharding), so this path
// never forms it: a block power iteration with oversampling on the implicit operator (the O-pass
// kernels of the SSI, rows sharded with the same collectives) run until the leading `rank` Ritz
// triplets have converged, then Rayleigh-Ritz on the small global block Y = Ohat^T Q:
//   Q = orth(Z),  Y = Ohat^T Q  (cols x b),  Z = Ohat Y = Ohat Ohat^T Q,
//   Y = V_y S W_y^T (device dense SVD)  =>  Ohat ~= (Q W_y) S V_y^T,
// and since Ohat V_y = Z W_y S^-1, the Ritz residual of triplet i is
//   ||Ohat v_i - s_i u_i|| = ||Z w_i / s_i - s_i Q w_i||   (no extra O-pass).
// The top singular triplets are unique (up to sign) wherever the reference's are well defined,
// so the result agrees with LAPACK's to the accuracy the residual certifies.
__global__ void fill_normal_kernel(double* x, int64_t n, uint64_t seed) {
  pdl_wait();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    // splitmix64 of (seed, i) -> two uniforms -> Box-Muller
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    const double u1 = ((double)(z >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    uint64_t y = z * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
    y = (y ^ (y >> 29)) * 0xBF58476D1CE4E5B9ull;
    y ^= y >> 32;
    const double u2 = ((double)(y >> 11)) * (1.0 / 9007199254740992.0);
    x[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

// partial[b][j] = sum over this block's rows of (T_pj / s_j - s_j U_pj)^2, j < k (fixed order)
__global__ void ritz_residual_kernel(const double* __restrict__ T, const double* __restrict__ U,
                                     int64_t ld, int64_t rows, int k, const double* __restrict__ S,
                                     double* __restrict__ partial) {
  pdl_wait();
  const int64_t chunk = (rows + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    const double s = S[j], inv = s > 0.0 ? 1.0 / s : 0.0;
    double acc = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      const double d = T[r * ld + j] * inv - s * U[r * ld + j];
      acc = fma(d, d, acc);
    }
    partial[(int64_t)blockIdx.x * k + j] = acc;
  }
}
__global__ void sum_partials_kernel(const double* __restrict__ partial, int nb, int k,
                                    double* __restrict__ out) {
  pdl_wait();
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += partial[(int64_t)b * k + j];
    out[j] = acc;
  }
}

struct ImplicitSvdResult {
  int64_t k_pos = 0;
  int64_t iterations = 0;
  double residual = 0.0;  // max_i ||Ohat v_i - s_i u_i|| / s_i over the returned triplets
};

// U (P x rank, ldu), sigma (rank), V_local (this rank's cols x rank, ldv: rows c0 .. c0 + cols of
// the global right vectors).  cols_global = r + N over all ranks; c0 = this rank's first column.
ImplicitSvdResult implicit_svd(Context& ctx, const Ohat& o, int64_t rank, int64_t cols_global,
                               int64_t c0, uint64_t seed, int64_t max_iters, double tol, double* U,
                               int64_t ldu, double* sigma, double* V, int64_t ldv, int* status,
                               bool careful) {
  cudaStream_t st = ctx.stream;
  const int64_t P = o.P, cols = o.cols(), mn = std::min(P, cols_global);
  if (rank < 1 || rank > mn)
    throw Fail{WSSR_ERR_RANK_TOO_LARGE, "rank outside [1, min(m, n)]"};
  o.status = status;
  // block width: 2x oversampling (at least 16 extra columns), within the single-CTA dense SVD
  int64_t b = std::max<int64_t>(2 * rank, rank + 16);
  if (b > kDenseSvdMax) b = std::max<int64_t>(rank + 16, kDenseSvdMax);
  b = std::min(b, mn);
  const bool dist = ctx.world() > 1;
  Buf Q((size_t)P * b, st), Z((size_t)P * b, st), Yl((size_t)std::max<int64_t>(cols, 1) * b, st),
      Yg(dist ? (size_t)cols_global * b : 0, st), Vy((size_t)cols_global * b, st), S(b, st),
      WyT((size_t)b * b, st), Wy((size_t)b * b, st), T((size_t)P * rank, st),
      Uk((size_t)P * rank, st), res(rank, st);
  const int nbp = (int)std::min<int64_t>(4 * ctx.num_sms, std::max<int64_t>(1, P / 64));
  Buf partial((size_t)nbp * rank, st);
  launch_pdl(fill_normal_kernel, blocks_for(P * b, 256, 16 * ctx.num_sms), 256, 0, st, Z.p,
             P * b, seed);
  post_launch(ctx);
  std::vector<double> hs(b), hres(rank);
  ImplicitSvdResult out;
  double best = std::numeric_limits<double>::infinity();
  int stalls = 0;
  for (int64_t it = 1; it <= max_iters; ++it) {
    qr(ctx, P, b, Z, b, Q, b, nullptr, status, careful, false);  // replicated: Z is global
    apply_OT(ctx, o, Q, b, b, Yl, b);                          // this rank's rows of Y
    if (it == 1) {  // Y = Ohat^T Q vanishes (Q random) only for Ohat = 0
      Buf y2(1, st);
      sumsq_matrix(ctx, Yl, cols, b, b, y2);
      if (dist) allreduce(ctx, y2, 1);
      if (!(read_scalar(ctx, y2) > 0.0))
        throw Fail{WSSR_ERR_DEGENERATE_INPUT, "cannot factorize an all-zero matrix"};
    }
    apply_O(ctx, o, Yl, b, b, Z, b);                           // Z = Ohat Y (summed over ranks)
    if (dist) {
      WSSR_CUDA(cudaMemsetAsync(Yg, 0, sizeof(double) * cols_global * b, st));
      if (cols > 0) copy2d(ctx, Yl, b, cols, b, 1.0, Yg.p + c0 * b, b);
      allreduce(ctx, Yg, (size_t)(cols_global * b));  // disjoint rows: the sum is exact
    }
    dense_svd(ctx, cols_global, b, dist ? Yg.p : Yl.p, b, Vy, b, S, WyT, b);  // Y = V_y S W_y^T
    transpose(ctx, WyT, b, b, b, nullptr, 1.0, Wy, b);
    gemm_rm(ctx, P, rank, b, Z, b, nullptr, Wy, b, T, rank, 1.0, false);   // Z w_i
    gemm_rm(ctx, P, rank, b, Q, b, nullptr, Wy, b, Uk, rank, 1.0, false);  // u_i = Q w_i
    launch_pdl(ritz_residual_kernel, nbp, 128, 0, st, (const double*)T.p, (const double*)Uk.p,
               rank, P, (int)rank, (const double*)S.p, partial.p);
    post_launch(ctx);
    launch_pdl(sum_partials_kernel, 1, 128, 0, st, (const double*)partial.p, nbp, (int)rank, res.p);
    post_launch(ctx);
    d2h(ctx, hs.data(), S, sizeof(double) * b);
    d2h(ctx, hres.data(), res, sizeof(double) * rank);
    sync(ctx);
    if (!(hs[0] > 0.0)) throw Fail{WSSR_ERR_DEGENERATE_INPUT, "cannot factorize an all-zero matrix"};
    // residual of the triplets that count (exact zeros are dropped, svdengine.py:70-72),
    // relative to each singular value
    double worst = 0.0;
    for (int64_t i = 0; i < rank; ++i)
      if (hs[i] > 0.0) worst = std::max(worst, std::sqrt(hres[i]) / hs[i]);
      else if (hs[i] != 0.0 || !(hres[i] >= 0.0)) worst = std::numeric_limits<double>::infinity();
    out.iterations = it;
    out.residual = worst;
    // the block spans the whole space: exact after one pass
    if (worst <= tol || b == mn) break;
    // stagnation at the rounding floor: no halving over two iterations
    if (worst < 0.5 * best) {
      best = worst;
      stalls = 0;
    } else if (++stalls >= 2) {
      break;
    }
  }
  int64_t kp = 0;
  while (kp < rank && hs[kp] > 0.0) ++kp;
  out.k_pos = kp;
  if (kp == 0) throw Fail{WSSR_ERR_DEGENERATE_INPUT, "cannot factorize an all-zero matrix"};
  copy2d(ctx, Uk, rank, P, kp, 1.0, U, ldu);
  copy2d(ctx, S, 1, 1, kp, 1.0, sigma, kp);
  if (cols > 0) copy2d(ctx, Vy.p + c0 * b, b, cols, kp, 1.0, V, ldv);
  return out;
}

Ohat ohat_from(const Context& ctx, const wssr_ohat_f64& oh, double delta) {
  const bool owner = ctx.world() <= 1 || ctx.comm->rank == 0;  // history block lives on rank 0
  Ohat o;
  o.P = oh.n_params;
  o.hist = oh.hist;
  o.r = owner ? oh.hist_rank : 0;
  o.ldh = oh.hist_ld;
  o.sh = std::sqrt(delta) * oh.hist_scale;
  o.samp = oh.samples;
  o.n = oh.n_samples;
  o.lds = oh.samples_ld;
  o.mu = oh.mu;
  o.ss = std::sqrt(1.0 - delta) * oh.samples_scale;
  o.f32 = oh.samples_f32 != 0;
  o.scale_tab = oh.samples_scale_table;
  return o;
}

// ---- wssr_step (optimizers.py:292-391), ssi branch -------------------------------------------
void step_impl(Context& ctx, const wssr_step_in* in, wssr_step_out* out) {
  const wssr_ohat_f64& oh = *in->ohat;
  cudaStream_t st = ctx.stream;
  const int64_t P = oh.n_params, k = in->requested;
  const bool dist = ctx.world() > 1;
  const bool owner = !dist || ctx.comm->rank == 0;  // history block lives on rank 0
  const double sq_old = std::sqrt(in->delta), sq_new = std::sqrt(1.0 - in->delta);
  Ohat o;
  o.P = P;
  o.hist = oh.hist;
  o.r = owner ? oh.hist_rank : 0;
  o.ldh = oh.hist_ld;
  o.sh = sq_old * oh.hist_scale;
  o.samp = oh.samples;
  o.n = oh.n_samples;
  o.lds = oh.samples_ld;
  o.mu = oh.mu;
  o.ss = sq_new * oh.samples_scale;
  o.f32 = oh.samples_f32 != 0;
  o.scale_tab = oh.samples_scale_table;
  const int64_t cols = o.cols();
  if (k < 1) throw Fail{WSSR_ERR_RANK_TOO_LARGE, "rank must be at least 1"};

  double samples_fro2 = oh.samples_fro2 >= 0.0 ? oh.samples_fro2 * (sq_new * sq_new) : -1.0;
  Ohat ofull = o;  // the history block is replicated: every rank adds its norm
  ofull.r = oh.hist_rank;
  Fro2 fro2;
  if (samples_fro2 < 0.0 && oh.samples_fro2_dev && !dist) {
    fro2.host = ohat_fro2(ctx, ofull, 0.0, true);  // history part; samples part still on device
    fro2.dev = oh.samples_fro2_dev;
    fro2.dev_scale = sq_new * sq_new;
  } else {
    fro2.host = ohat_fro2(ctx, ofull, samples_fro2, true);
    if (fro2.host == 0.0)
      throw Fail{WSSR_ERR_DEGENERATE_INPUT, "cannot factorize an all-zero matrix"};
  }

  // lhat = [sqrt(delta) lbar, sqrt(1-delta) L]  (optimizers.py:324)
  Buf lhat((size_t)std::max<int64_t>(cols, 1), st);
  if (o.r > 0) copy2d(ctx, in->lbar, 1, o.r, 1, sq_old, lhat, 1);
  if (o.n > 0) copy2d(ctx, in->l_vector, 1, o.n, 1, sq_new, lhat + o.r, 1);

  SsiResult sr;
  if (in->ext_u) {
    // factors from a dense backend (optimizers.py:327-338): U (P x k_pos), sigma, V as columns
    const int64_t kp = in->ext_k_pos;
    if (kp < 1 || kp > k) throw Fail{WSSR_ERR_VALUE, "bad external factor rank"};
    copy2d(ctx, in->ext_u, in->ext_ld_u, P, kp, 1.0, out->u_next, out->ld_u);
    copy2d(ctx, in->ext_sigma, 1, kp, 1, 1.0, out->sigma, 1);
    sr.qv = Buf((size_t)std::max<int64_t>(cols, 1) * k, st);
    if (cols > 0) copy2d(ctx, in->ext_v, in->ext_ld_v, cols, kp, 1.0, sr.qv, k);
    std::vector<double> hs(kp);
    d2h(ctx, hs.data(), in->ext_sigma, sizeof(double) * kp);
    sync(ctx);
    sr.k_pos = kp;
    sr.sigma0 = hs[0];
    const double top = hs[0] * hs[0];
    sr.r_eff = 0;
    for (int64_t j = 0; j < kp; ++j) sr.r_eff += (hs[j] * hs[j] >= in->r_reg * top) ? 1 : 0;
    sr.iterations = 0;
    sr.residual = 0.0;
  } else {
    sr = with_fallback(ctx, in->flags, [&](bool careful, int* status) {
      return ssi_core(ctx, o, k, in->max_iters, in->u_init, in->ld_init, in->residual_tol, fro2,
                      (in->flags & WSSR_FLAG_FINAL_RESIDUAL) != 0, careful, out->u_next,
                      out->ld_u, out->sigma, in->r_reg, status);
    });
  }
  const int64_t r_eff = sr.r_eff;
  if (r_eff < 1) throw Fail{WSSR_ERR_RANK_COLLAPSE, "no singular value passed the relative cutoff"};

  // drift telemetry against the previous factors (optimizers.py:366-374)
  double sd = 0.0, pd = 0.0;
  const int64_t r_hist = oh.hist_rank;
  const int64_t r_drift = in->r_prev > 0 ? std::min(std::min(r_hist, in->r_prev), r_eff) : 0;
  if (r_drift > 0 && out->drift_host && ctx.aux && !dist) {
    // asynchronous: the drift runs on the auxiliary stream as soon as U and sigma are final,
    // beside the preconditioner and the state refresh, and while the caller moves on;
    // {sigma_drift, projector_drift} land in out->drift_host in aux-stream order
    if (!ctx.aux_event) WSSR_CUDA(cudaEventCreateWithFlags(&ctx.aux_event, cudaEventDisableTiming));
    WSSR_CUDA(cudaEventRecord(ctx.aux_event, st));
    WSSR_CUDA(cudaStreamWaitEvent(ctx.aux, ctx.aux_event, 0));
    // the aux stream gets its own slab buffer (the main stream's is reused by the next step)
    cudaStream_t main_stream = ctx.stream;
    std::swap(ctx.splitk, ctx.aux_splitk);
    std::swap(ctx.splitk_cap, ctx.aux_splitk_cap);
    ctx.stream = ctx.aux;
    auto restore = [&] {
      ctx.stream = main_stream;
      std::swap(ctx.splitk, ctx.aux_splitk);
      std::swap(ctx.splitk_cap, ctx.aux_splitk_cap);
    };
    try {
      Buf sprev(r_hist, ctx.aux), out2(2, ctx.aux);
      PhaseTimer tm(ctx, 5, 0.0, 0.0);  // events on the aux stream
      row_norms(ctx, oh.hist, r_hist, P, oh.hist_ld, sprev);
      drift_enqueue(ctx, P, in->u_prev, in->ld_prev, sprev, r_drift, out->u_next, out->ld_u,
                    out->sigma, out2);
      d2h(ctx, out->drift_host, out2, 2 * sizeof(double));
    } catch (...) {
      restore();
      throw;
    }
    restore();
    sd = pd = std::numeric_limits<double>::quiet_NaN();
  } else if (in->r_prev > 0) {
    Buf sprev(std::max<int64_t>(r_hist, 1), st);
    if (r_hist > 0) row_norms(ctx, oh.hist, r_hist, P, oh.hist_ld, sprev);
    const int64_t r1 = std::min(r_hist, in->r_prev);
    auto d = drift(ctx, P, in->u_prev, in->ld_prev, sprev, r1, out->u_next, out->ld_u, out->sigma,
                   r_eff, dist);
    sd = d.first;
    pd = d.second;
  }
  if (out->drift_host && !std::isnan(sd)) {
    out->drift_host[0] = sd;
    out->drift_host[1] = pd;
  }
  const bool binding = sr.k_pos == k && k == in->r_max && r_eff == in->r_max;
  int64_t next_r_max = in->r_max;
  if (binding) {
    next_r_max = (int64_t)std::ceil((1.0 + in->eps_grow) * (double)in->r_max);
    next_r_max = std::min(next_r_max, P);
  }
  const double top_sq = sr.sigma0 * sr.sigma0;

  // gbar = Ohat lhat  (optimizers.py:359)
  Buf gbar(P, st);
  if (in->gradient) {
    // bundle.gradient = 2 o_matrix l_vector, exact for bundles assembled by this library
    launch_pdl(scale_kernel, blocks_for(P, 256, 8 * ctx.num_sms), 256, 0, st, 
        P, 0.5 * sq_new * sq_new, in->gradient, gbar);
    post_launch(ctx);
  } else {
    if (o.f32) throw Fail{WSSR_ERR_UNSUPPORTED, "fp32 samples need the assembled gradient"};
    if (o.n > 0) {
      gemm_cm(ctx, P, 1, o.n, o.samp, o.lds, o.mu, in->l_vector, 1, gbar, 1, o.ss * sq_new, false);
    } else {
      WSSR_CUDA(cudaMemsetAsync(gbar, 0, sizeof(double) * P, st));
    }
    if (dist) allreduce(ctx, gbar, P);
  }
  if (oh.hist_rank > 0 && o.sh != 0.0)
    gemm_cm(ctx, P, 1, oh.hist_rank, oh.hist, oh.hist_ld, nullptr, in->lbar, 1, gbar, 1,
            o.sh * sq_old, true);

  // preconditioned update (optimizers.py:361-364)
  Buf c(r_eff, st);
  {
  PhaseTimer tm(ctx, 6, 0.0, 0.0);
  gemv_t(ctx, P, r_eff, out->u_next, out->ld_u, gbar, c);
  const double floor = in->sigma_floor * (in->sigma_floor_relative ? top_sq : 1.0);
  {
    const int threads = 256;
    const int blocks = blocks_for(P * 32, threads, 16 * ctx.num_sms);
    launch_pdl(precond_update_kernel, blocks, threads, sizeof(double) * 2 * r_eff, st, 
        out->u_next, out->ld_u, P, (int)r_eff, c, out->sigma, gbar, 1.0 / floor, in->theta,
        in->eta, out->theta_next, out->update);
    post_launch(ctx);
  }

  // state refresh (optimizers.py:376-383): obar = U sigma, lbar = V[:r] lhat
  {
    dim3 grid((unsigned)((P + 31) / 32), (unsigned)((r_eff + 31) / 32));
    launch_pdl(transpose_scale_kernel, grid, dim3(32, 8), 0, st, out->u_next, out->ld_u, P, (int)r_eff,
                                                         out->sigma, out->obar_next_t,
                                                         out->ld_obar);
    post_launch(ctx);
  }
  if (cols > 0) {
    gemv_t(ctx, cols, r_eff, sr.qv, k, lhat, out->lbar_next);
  } else {
    WSSR_CUDA(cudaMemsetAsync(out->lbar_next, 0, sizeof(double) * r_eff, st));
  }
  }
  if (dist) allreduce(ctx, out->lbar_next, r_eff);

  // No final wait: every host output is known by now (the rank cut synchronised); the
  // preconditioner / state-refresh kernels finish in stream order while the caller builds the
  // next state (a kernel fault would surface at the next synchronising call).  The phase timer
  // events still need collecting at some point: do it when they are done.
  if (!ctx.pending.empty() && cudaStreamQuery(ctx.stream) == cudaSuccess) collect_timing(ctx);
  cudaGetLastError();

  out->r_eff = r_eff;
  out->k_pos = sr.k_pos;
  out->iterations = sr.iterations;
  out->next_r_max = next_r_max;
  out->binding = binding ? 1 : 0;
  out->residual = sr.residual;
  out->sigma_drift = sd;
  out->projector_drift = pd;
}

void step(Context& ctx, const wssr_step_in* in, wssr_step_out* out) {
  if (!g_hprof.on) return step_impl(ctx, in, out);
  g_hprof = HostProf();
  const double t0 = HostProf::now();
  step_impl(ctx, in, out);
  std::fprintf(stderr,
               "[wssr host] step %.2f ms: alloc %.2f ms (%lld), free %.2f ms, sync waits %.2f ms "
               "(%lld)\n",
               1e3 * (HostProf::now() - t0), 1e3 * g_hprof.alloc_s, (long long)g_hprof.allocs,
               1e3 * g_hprof.free_s, 1e3 * g_hprof.sync_s, (long long)g_hprof.syncs);
}

// ---- NCCL (dlopen'd so the library has no link-time NCCL dependency) ------------------------
// ncclUniqueId is a 128-byte struct that ncclCommInitRank takes BY VALUE (nccl.h):
//   ncclResult_t ncclCommInitRank(ncclComm_t*, int nranks, ncclUniqueId commId, int rank);
struct NcclUniqueId {
  char internal[128];
};
typedef int (*nccl_get_id_fn)(NcclUniqueId*);
typedef int (*nccl_init_rank_fn)(void**, int, NcclUniqueId, int);
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_reduce_scatter_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_all_gather_fn)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*nccl_destroy_fn)(void*);

struct NcclLib {
  void* h = nullptr;
  nccl_get_id_fn get_id = nullptr;
  nccl_init_rank_fn init_rank = nullptr;
  nccl_allreduce_fn allreduce = nullptr;
  nccl_reduce_scatter_fn reduce_scatter = nullptr;
  nccl_all_gather_fn all_gather = nullptr;
  nccl_destroy_fn destroy = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    get_id = (nccl_get_id_fn)dlsym(h, "ncclGetUniqueId");
    init_rank = (nccl_init_rank_fn)dlsym(h, "ncclCommInitRank");
    allreduce = (nccl_allreduce_fn)dlsym(h, "ncclAllReduce");
    reduce_scatter = (nccl_reduce_scatter_fn)dlsym(h, "ncclReduceScatter");
    all_gather = (nccl_all_gather_fn)dlsym(h, "ncclAllGather");
    destroy = (nccl_destroy_fn)dlsym(h, "ncclCommDestroy");
    return get_id && init_rank && allreduce && reduce_scatter && all_gather && destroy;
  }
};
NcclLib g_nccl;

struct NcclComm : Comm {
  void* comm = nullptr;
  cudaError_t allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    // ncclFloat64 = 8, ncclSum = 0
    int r = g_nccl.allreduce(buf, buf, n, 8, 0, comm, st);
    return r == 0 ? cudaSuccess : cudaErrorUnknown;
  }
  // in place: recvbuff = sendbuff + rank * count (nccl.h "in-place operations")
  cudaError_t reduce_scatter_sum(double* buf, size_t count, cudaStream_t st) override {
    int r = g_nccl.reduce_scatter(buf, buf + (size_t)rank * count, count, 8, 0, comm, st);
    return r == 0 ? cudaSuccess : cudaErrorUnknown;
  }
  // in place: sendbuff = recvbuff + rank * count
  cudaError_t all_gather(double* buf, size_t count, cudaStream_t st) override {
    int r = g_nccl.all_gather(buf + (size_t)rank * count, buf, count, 8, comm, st);
    return r == 0 ? cudaSuccess : cudaErrorUnknown;
  }
  ~NcclComm() override {
    if (comm) g_nccl.destroy(comm);
  }
};

// ---- thread-emulated communicator (tests the sharded engine on ONE GPU) ------------------------
// Each emulated rank is a host thread with its own context and stream.  allreduce: every rank
// publishes its buffer after a stream sync, rank 0 sums the buffers in rank order into a scratch
// buffer, everyone copies it back.  All waiting happens on the host; no kernel waits on another.
struct EmuSumArgs {
  const double* src[8];
};
__global__ void emu_sum_kernel(EmuSumArgs a, int world, size_t n, double* out) {
  pdl_wait();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    double s = a.src[0][i];
    for (int r = 1; r < world; ++r) s += a.src[r][i];
    out[i] = s;
  }
}

struct EmuGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  bool aborted = false;
  std::vector<double*> bufs;
  double* scratch = nullptr;
  size_t cap = 0;
  // false when a rank aborted the group (its peers then fail instead of waiting forever)
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const int64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen || aborted; });
    }
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

struct EmuComm : Comm {
  EmuGroup* g = nullptr;
  cudaError_t allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      g->abort();
      return e;
    }
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->bufs[rank] = buf;
    }
    if (!g->barrier()) return cudaErrorUnknown;
    if (rank == 0) {
      if (n > g->cap) {
        if (g->scratch) cudaFree(g->scratch);
        if ((e = cudaMalloc(&g->scratch, n * sizeof(double))) != cudaSuccess) {
          g->abort();
          return e;
        }
        g->cap = n;
      }
      EmuSumArgs a{};
      for (int r = 0; r < world; ++r) a.src[r] = g->bufs[r];
      launch_pdl(emu_sum_kernel, 256, 256, 0, st, a, world, n, g->scratch);
      e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) g->abort();
    }
    if (!g->barrier()) return cudaErrorUnknown;
    e = cudaMemcpyAsync(buf, g->scratch, n * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (!g->barrier()) return cudaErrorUnknown;
    return e;
  }
  // every rank copies the other ranks' slices straight from their buffers (same device)
  cudaError_t all_gather(double* buf, size_t count, cudaStream_t st) override {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      g->abort();
      return e;
    }
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->bufs[rank] = buf;
    }
    if (!g->barrier()) return cudaErrorUnknown;
    for (int r = 0; r < world && e == cudaSuccess; ++r)
      if (r != rank)
        e = cudaMemcpyAsync(buf + (size_t)r * count, g->bufs[r] + (size_t)r * count,
                            count * sizeof(double), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (!g->barrier()) return cudaErrorUnknown;
    return e;
  }
};

}  // namespace
}  // namespace wssr

namespace wssr {
__global__ void dmma_peak_kernel(double* out, int iters) {
  pdl_wait();
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma884(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}
}  // namespace wssr

// ================================ C ABI =====================================================
using namespace wssr;

namespace {
int fail(wssr_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->c.last_error = msg;
  return code;
}
template <class F>
int guarded(wssr_ctx* ctx, F&& f) {
  if (!ctx) return WSSR_ERR_VALUE;
  try {
    WSSR_CUDA(cudaSetDevice(ctx->c.device));
    f();
    return WSSR_OK;
  } catch (const Fail& e) {
    return fail(ctx, e.code, e.msg);
  } catch (const std::exception& e) {
    return fail(ctx, WSSR_ERR_VALUE, e.what());
  }
}
}  // namespace

extern "C" {

int wssr_version(void) { return 1; }

int wssr_ctx_create(int device, wssr_ctx** out) {
  if (!out) return WSSR_ERR_VALUE;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return WSSR_ERR_CUDA;
  if (device < 0 || device >= n) return WSSR_ERR_VALUE;
  if (cudaSetDevice(device) != cudaSuccess) return WSSR_ERR_CUDA;
  auto* c = new wssr_ctx();
  c->c.device = device;
  cudaDeviceGetAttribute(&c->c.num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  if (cudaMallocHost(reinterpret_cast<void**>(&c->c.hbuf), 4096 * sizeof(double)) != cudaSuccess) {
    delete c;
    return WSSR_ERR_CUDA;
  }
  *out = c;
  return WSSR_OK;
}

void wssr_ctx_destroy(wssr_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  if (ctx->c.splitk || ctx->c.oz_ws || ctx->c.oz_planes) cudaDeviceSynchronize();
  if (ctx->c.aux) cudaStreamSynchronize(ctx->c.aux);
  if (ctx->c.hbuf) {
    cudaDeviceSynchronize();
    cudaFreeHost(ctx->c.hbuf);
  }
  g_scratch.trim(ctx->c.device);
  if (ctx->c.aux_event) cudaEventDestroy(ctx->c.aux_event);
  if (ctx->c.aux_splitk) cudaFree(ctx->c.aux_splitk);
  if (ctx->c.splitk) cudaFree(ctx->c.splitk);
  if (ctx->c.oz_ws) cudaFree(ctx->c.oz_ws);
  if (ctx->c.oz_planes) cudaFree(ctx->c.oz_planes);
  delete ctx->c.comm;
  delete ctx;
}

const char* wssr_last_error(const wssr_ctx* ctx) { return ctx ? ctx->c.last_error.c_str() : ""; }

int wssr_release_memory(wssr_ctx* ctx) {
  if (!ctx) return WSSR_ERR_VALUE;
  Context& c = ctx->c;
  cudaSetDevice(c.device);
  cudaDeviceSynchronize();
  if (c.oz_planes) cudaFree(c.oz_planes);
  c.oz_planes = nullptr;
  c.oz_planes_cap = 0;
  c.plan_n = c.plan_p = c.plan_k = -1;
  c.plan_rows = 0;
  c.plan_provisional = false;
  if (c.oz_ws) cudaFree(c.oz_ws);
  c.oz_ws = nullptr;
  c.oz_ws_cap = 0;
  g_scratch.trim(c.device);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, c.device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  return cudaGetLastError() == cudaSuccess ? WSSR_OK : WSSR_ERR_CUDA;
}

int wssr_set_stream(wssr_ctx* ctx, void* stream) {
  if (!ctx) return WSSR_ERR_VALUE;
  ctx->c.stream = reinterpret_cast<cudaStream_t>(stream);
  return WSSR_OK;
}

int64_t wssr_kernel_launches(const wssr_ctx* ctx) { return ctx ? ctx->c.kernel_launches : 0; }

int wssr_set_precision_guard(wssr_ctx* ctx, int enabled) {
  if (!ctx) return WSSR_ERR_VALUE;
  ctx->c.oz_guard = enabled != 0;
  return WSSR_OK;
}

int64_t wssr_precision_fallbacks(const wssr_ctx* ctx) {
  return ctx ? ctx->c.precision_fallbacks : 0;
}

int wssr_set_gemm_path(wssr_ctx* ctx, int path) {
  if (!ctx || path < 0 || path > 4) return WSSR_ERR_VALUE;
  ctx->c.disable_tma = path == 1;
  ctx->c.ozaki = path == 0 || path >= 3;
  ctx->c.oz_min_elems = path >= 3 ? 0.0 : 4194304.0;
  ctx->c.oz_pre = path == 4 ? 1 : 0;
  return WSSR_OK;
}

int wssr_set_tail_shard(wssr_ctx* ctx, int enabled) {
  if (!ctx) return WSSR_ERR_VALUE;
  ctx->c.tail_shard = enabled != 0;
  return WSSR_OK;
}

int wssr_ozaki_digit_pairs(void) { return ozaki_digit_pairs(); }

int wssr_set_fp32_digits(wssr_ctx* ctx, int digits) {
  if (!ctx || (digits != 5 && digits != 7)) return WSSR_ERR_VALUE;
  ctx->c.f32_digits = digits;
  return WSSR_OK;
}

int wssr_set_dense_svd_mode(wssr_ctx* ctx, int mode) {
  if (!ctx || mode < 0 || mode > 1) return WSSR_ERR_VALUE;
  ctx->c.force_blocked_svd = mode == 1;
  return WSSR_OK;
}

int wssr_dense_svd_sweeps(const wssr_ctx* ctx) { return ctx ? ctx->c.dense_svd_sweeps : -1; }

int wssr_set_tallskinny(wssr_ctx* ctx, int enabled) {
  if (!ctx) return WSSR_ERR_VALUE;
  ctx->c.tallskinny = enabled != 0;
  return WSSR_OK;
}

int wssr_debug_tallskinny(wssr_ctx* ctx, int op, int64_t rows, int64_t k, const double* a,
                          const double* b, const double* m, const double* cin, double alpha,
                          double* out) {
  return guarded(ctx, [&] {
    Context& c = ctx->c;
    if (k == 2 * kTsHalf && rows >= 0 && c.tallskinny) {
      // k = 256: the engine's 2 x 2 block composition of the k = 128 kernels (alpha = 1 for the
      // products, alpha = -1 for op 4, as the engine uses them)
      switch (op) {
        case 0: gram(c, rows, k, a, k, out, false); break;
        case 1: cross(c, rows, k, a, k, b, k, out); break;
        case 2:
        case 3:
          if (alpha != 1.0) throw Fail{WSSR_ERR_VALUE, "tall-skinny k = 256: alpha must be 1"};
          mul_small(c, rows, k, a, k, m, op == 2, out, k);
          break;
        case 4:
          if (alpha != -1.0) throw Fail{WSSR_ERR_VALUE, "tall-skinny k = 256: alpha must be -1"};
          sub_mul_small(c, rows, k, a, k, m, cin, k, out, k);
          break;
        default: throw Fail{WSSR_ERR_VALUE, "tall-skinny k = 256: ops 0-4"};
      }
      sync(c);
      return;
    }
    if (!ts_supported(k) || rows < 0) throw Fail{WSSR_ERR_VALUE, "tall-skinny: k must be 32, 64 or 128"};
    static const int reps = [] {
      const char* e = std::getenv("WSSR_DEBUG_REPS");  // profiling: back-to-back launches
      return e ? std::max(1, std::atoi(e)) : 1;
    }();
    for (int rep = 0; rep < reps; ++rep)
    switch (op) {
      case 0: WSSR_CUDA(ts_gram(c, rows, k, a, k, out)); break;
      case 1: WSSR_CUDA(ts_cross(c, rows, k, a, k, b, k, out)); break;
      case 2:
      case 3: WSSR_CUDA(ts_mul(c, rows, k, a, k, m, op == 2, alpha, out, k)); break;
      case 4: WSSR_CUDA(ts_mul_add(c, rows, k, a, k, m, alpha, cin, k, out, k)); break;
      case 5: WSSR_CUDA(ts_mul_add_sumsq(c, rows, k, a, k, m, alpha, cin, k, out)); break;
      case 6: WSSR_CUDA(ts_gemv_t(c, rows, k, a, k, cin, alpha, out)); break;
      default: throw Fail{WSSR_ERR_VALUE, "tall-skinny: unknown op"};
    }
    sync(c);
  });
}

int wssr_grad_theta_f64(wssr_ctx* ctx, const wssr_ace_spec* spec, const double* positions,
                        int64_t n_walkers, double* out, int64_t ld_out) {
  return guarded(ctx, [&] {
    Context& c = ctx->c;
    if (!spec || n_walkers < 0 || (n_walkers > 0 && (!positions || !out)))
      throw Fail{WSSR_ERR_VALUE, "bad arguments"};
    const wssr_ace_spec& s = *spec;
    if (s.n_electrons < 1 || s.n_electrons > 64 || s.n_orbitals < 1 || s.n_features < 1 ||
        s.max_tail < 0 || ld_out < s.n_electrons * s.n_features)
      throw Fail{WSSR_ERR_VALUE, "bad ansatz dimensions (n_electrons must be 1..64)"};
    if (grad_theta_smem(s, grad_theta_tile(s)) > 200 * 1024)
      throw Fail{WSSR_ERR_UNSUPPORTED, "orbital table too large for one CTA"};
    Buf flag(1, c.stream);
    WSSR_CUDA(cudaMemsetAsync(flag, 0, sizeof(double), c.stream));
    WSSR_CUDA(grad_theta(c, s, positions, n_walkers, out, ld_out, flag.i32()));
    int* hf = reinterpret_cast<int*>(c.hbuf + 6);
    d2h(c, hf, flag, sizeof(int));
    sync(c);
    if (*hf) throw Fail{WSSR_ERR_NODE_PROXIMITY, "parameter gradient requested on top of a node"};
  });
}

int wssr_set_aux_stream(wssr_ctx* ctx, void* stream) {
  if (!ctx) return WSSR_ERR_VALUE;
  ctx->c.aux = static_cast<cudaStream_t>(stream);
  return WSSR_OK;
}

int wssr_set_timing(wssr_ctx* ctx, int enabled) {
  if (!ctx) return WSSR_ERR_VALUE;
  ctx->c.timing = enabled != 0;
  {
    const char* e = std::getenv("WSSR_FINE_PHASES");  // profiling only
    ctx->c.fine_phases = e && e[0] == '1';
  }
  for (int i = 0; i < Context::kPhases; ++i) {
    ctx->c.phase_ms[i] = ctx->c.phase_flops[i] = ctx->c.phase_bytes[i] = 0.0;
    ctx->c.phase_count[i] = 0;
  }
  return WSSR_OK;
}

int wssr_phase_stats(wssr_ctx* ctx, int phase, double* ms, int64_t* launches, double* flops,
                     double* bytes) {
  if (!ctx || phase < 0 || phase >= Context::kPhases) return WSSR_ERR_VALUE;
  if (!ctx->c.pending.empty()) {
    cudaDeviceSynchronize();
    collect_timing(ctx->c);
  }
  *ms = ctx->c.phase_ms[phase];
  *launches = ctx->c.phase_count[phase];
  *flops = ctx->c.phase_flops[phase];
  *bytes = ctx->c.phase_bytes[phase];
  return WSSR_OK;
}

// FP64 tensor-core peak probe: DMMA.8x8x4 with independent accumulators, 4 CTAs of 8 warps per
// SM, timed with CUDA events.  Gives the measured roofline denominator (TFLOP/s).
int wssr_dmma_peak_probe(wssr_ctx* ctx, double* tflops) {
  return guarded(ctx, [&] {
    const int iters = 4096;
    const int blocks = ctx->c.num_sms * 4, threads = 256;
    Buf sink(threads, ctx->c.stream);
    cudaEvent_t a, b;
    WSSR_CUDA(cudaEventCreate(&a));
    WSSR_CUDA(cudaEventCreate(&b));
    launch_pdl(dmma_peak_kernel, blocks, threads, 0, ctx->c.stream, sink, iters);
    WSSR_CUDA(cudaEventRecord(a, ctx->c.stream));
    launch_pdl(dmma_peak_kernel, blocks, threads, 0, ctx->c.stream, sink, iters);
    WSSR_CUDA(cudaEventRecord(b, ctx->c.stream));
    WSSR_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *tflops = 2.0 * 8 * 256 * (double)iters * blocks * (threads / 32) / (ms * 1e-3) / 1e12;
  });
}

int wssr_nccl_unique_id(wssr_ctx* ctx, unsigned char out_id[128]) {
  return guarded(ctx, [&] {
    if (!g_nccl.load()) throw Fail{WSSR_ERR_NCCL, "libnccl.so.2 not loadable"};
    NcclUniqueId uid;
    if (g_nccl.get_id(&uid) != 0) throw Fail{WSSR_ERR_NCCL, "ncclGetUniqueId failed"};
    std::memcpy(out_id, uid.internal, sizeof(uid.internal));
  });
}

int wssr_nccl_attach(wssr_ctx* ctx, const unsigned char id[128], int rank, int world) {
  return guarded(ctx, [&] {
    if (world < 1 || rank < 0 || rank >= world) throw Fail{WSSR_ERR_VALUE, "bad rank/world"};
    delete ctx->c.comm;
    ctx->c.comm = nullptr;
    // world == 1 builds a 1-rank communicator: the engine treats it as unsharded (world() == 1)
    // and wssr_allreduce_f64 exercises the transport
    if (!g_nccl.load()) throw Fail{WSSR_ERR_NCCL, "libnccl.so.2 not loadable"};
    auto* cm = new NcclComm();
    cm->rank = rank;
    cm->world = world;
    NcclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    if (g_nccl.init_rank(&cm->comm, world, uid, rank) != 0) {
      delete cm;
      throw Fail{WSSR_ERR_NCCL, "ncclCommInitRank failed"};
    }
    ctx->c.comm = cm;
  });
}

int wssr_emu_group_create(int world, void** group) {
  if (!group || world < 1 || world > 8) return WSSR_ERR_VALUE;
  auto* g = new EmuGroup();
  g->world = world;
  g->bufs.assign(world, nullptr);
  *group = g;
  return WSSR_OK;
}

void wssr_emu_group_abort(void* group) {
  if (group) static_cast<EmuGroup*>(group)->abort();
}

void wssr_emu_group_destroy(void* group) {
  auto* g = static_cast<EmuGroup*>(group);
  if (!g) return;
  if (g->scratch) cudaFree(g->scratch);
  delete g;
}

int wssr_emu_attach(wssr_ctx* ctx, void* group, int rank) {
  return guarded(ctx, [&] {
    auto* g = static_cast<EmuGroup*>(group);
    if (!g || rank < 0 || rank >= g->world) throw Fail{WSSR_ERR_VALUE, "bad emulated rank"};
    delete ctx->c.comm;
    ctx->c.comm = nullptr;
    if (g->world == 1) return;
    auto* cm = new EmuComm();
    cm->g = g;
    cm->rank = rank;
    cm->world = g->world;
    ctx->c.comm = cm;
  });
}

int wssr_allreduce_f64(wssr_ctx* ctx, double* buf, int64_t n) {
  return guarded(ctx, [&] {
    if (n < 0 || (n > 0 && !buf)) throw Fail{WSSR_ERR_VALUE, "bad buffer"};
    if (n == 0 || !ctx->c.comm) return;
    // also with a 1-rank communicator (a self-test of the transport)
    if (ctx->c.comm->allreduce_sum(buf, (size_t)n, ctx->c.stream) != cudaSuccess)
      throw Fail{WSSR_ERR_NCCL, "allreduce failed"};
    sync(ctx->c);
  });
}

int wssr_assemble_f64(wssr_ctx* ctx, const double* derivs, int64_t n, int64_t p, int64_t ld,
                      const double* energies, double clip_n_std, wssr_assemble_out* out) {
  return guarded(ctx, [&] {
    if (!out || p < 1 || n < 0 || ld < p) throw Fail{WSSR_ERR_VALUE, "bad assemble arguments"};
    assemble(ctx->c, derivs, n, p, ld, energies, clip_n_std, out);
  });
}

int wssr_assemble_f32(wssr_ctx* ctx, const float* derivs, int64_t n, int64_t p, int64_t ld,
                      const double* energies, double clip_n_std, wssr_assemble_out* out) {
  return guarded(ctx, [&] {
    if (!out || p < 1 || n < 0 || ld < p) throw Fail{WSSR_ERR_VALUE, "bad assemble arguments"};
    assemble(ctx->c, derivs, n, p, ld, energies, clip_n_std, out);
  });
}

int wssr_qr_f64(wssr_ctx* ctx, int64_t rows, int64_t cols, const double* a, int64_t lda,
                double* q, int64_t ldq, double* r, int64_t flags) {
  return guarded(ctx, [&] {
    if (rows < cols) throw Fail{WSSR_ERR_VALUE, "need at least as many rows as columns"};
    if (cols < 1 || lda < cols || ldq < cols) throw Fail{WSSR_ERR_VALUE, "bad qr arguments"};
    Context& c = ctx->c;
    with_fallback(c, flags | WSSR_FLAG_CAREFUL, [&](bool careful, int* status) {
      qr(c, rows, cols, a, lda, q, ldq, r, status, careful, false);
      return 0;
    });
    sync(c);
  });
}

int wssr_ssi_svd_f64(wssr_ctx* ctx, const wssr_ohat_f64* ohat, int64_t rank, int64_t max_iters,
                     const double* u_init, int64_t ld_init, double residual_tol, int64_t flags,
                     wssr_ssi_out* out) {
  return guarded(ctx, [&] {
    Context& c = ctx->c;
    if (!ohat || !out || !u_init) throw Fail{WSSR_ERR_VALUE, "null argument"};
    Ohat o;
    o.P = ohat->n_params;
    o.hist = ohat->hist;
    o.r = (c.world() > 1 && c.comm->rank != 0) ? 0 : ohat->hist_rank;
    o.ldh = ohat->hist_ld;
    o.sh = ohat->hist_scale;
    o.samp = ohat->samples;
    o.n = ohat->n_samples;
    o.lds = ohat->samples_ld;
    o.mu = ohat->mu;
    o.ss = ohat->samples_scale;
    o.f32 = ohat->samples_f32 != 0;
    o.scale_tab = ohat->samples_scale_table;
    if (max_iters < 1) throw Fail{WSSR_ERR_VALUE, "max_iters must be at least 1"};
    Fro2 fro2;
    fro2.host = ohat_fro2(c, o, ohat->samples_fro2, true);
    if (fro2.host == 0.0)
      throw Fail{WSSR_ERR_DEGENERATE_INPUT, "cannot factorize an all-zero matrix"};
    SsiResult sr = with_fallback(c, flags, [&](bool careful, int* status) {
      return ssi_core(c, o, rank, max_iters, u_init, ld_init, residual_tol, fro2,
                      (flags & WSSR_FLAG_FINAL_RESIDUAL) != 0, careful, out->u, out->ld_u,
                      out->sigma, 0.5, status);
    });
    if (out->v && o.cols() > 0) copy2d(c, sr.qv, rank, o.cols(), sr.k_pos, 1.0, out->v, out->ld_v);
    sync(c);
    out->k_pos = sr.k_pos;
    out->iterations = sr.iterations;
    out->residual = sr.residual;
  });
}

int wssr_subspace_drift_f64(wssr_ctx* ctx, int64_t n_rows, const double* u1, int64_t ld1,
                            const double* s1, int64_t r1, const double* u2, int64_t ld2,
                            const double* s2, int64_t r2, double* sigma_drift,
                            double* projector_drift) {
  return guarded(ctx, [&] {
    auto d = drift(ctx->c, n_rows, u1, ld1, s1, r1, u2, ld2, s2, r2);
    *sigma_drift = d.first;
    *projector_drift = d.second;
  });
}

int wssr_step_f64(wssr_ctx* ctx, const wssr_step_in* in, wssr_step_out* out) {
  return guarded(ctx, [&] {
    if (!in || !out || !in->ohat) throw Fail{WSSR_ERR_VALUE, "null argument"};
    if (in->max_iters < 1) throw Fail{WSSR_ERR_VALUE, "max_iters must be at least 1"};
    step(ctx->c, in, out);
    ++ctx->c.steps_done;
  });
}

int wssr_exact_svd_f64(wssr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                       double* u, int64_t ldu, double* sigma, double* vt, int64_t ldvt) {
  return guarded(ctx, [&] {
    if (m < 1 || n < 1) throw Fail{WSSR_ERR_VALUE, "empty matrix"};
    dense_svd(ctx->c, m, n, a, lda, u, ldu, sigma, vt, ldvt);
    sync(ctx->c);
  });
}

int wssr_materialize_ohat_f64(wssr_ctx* ctx, const wssr_ohat_f64* ohat, double delta, double* out,
                              int64_t ldo) {
  return guarded(ctx, [&] {
    if (!ohat || !out) throw Fail{WSSR_ERR_VALUE, "null argument"};
    materialize_ohat(ctx->c, *ohat, delta, out, ldo);
  });
}

int wssr_implicit_svd_f64(wssr_ctx* ctx, const wssr_ohat_f64* ohat, double delta, int64_t rank,
                          int64_t cols_global, int64_t col0, uint64_t seed, int64_t max_iters,
                          double tol, double* u, int64_t ldu, double* sigma, double* v_local,
                          int64_t ldv, int64_t* k_pos, int64_t* iterations, double* residual) {
  return guarded(ctx, [&] {
    if (!ohat || !u || !sigma || !k_pos) throw Fail{WSSR_ERR_VALUE, "null argument"};
    if (max_iters < 1) throw Fail{WSSR_ERR_VALUE, "max_iters must be at least 1"};
    Context& c = ctx->c;
    const ImplicitSvdResult r = with_fallback(c, 0, [&](bool careful, int* status) {
      const Ohat o = ohat_from(c, *ohat, delta);  // fresh per attempt (precision guard)
      if (col0 < 0 || col0 + o.cols() > cols_global)
        throw Fail{WSSR_ERR_VALUE, "column range outside the global Ohat"};
      return implicit_svd(c, o, rank, cols_global, col0, seed, max_iters, tol, u, ldu, sigma,
                          v_local, ldv, status, careful);
    });
    sync(c);
    *k_pos = r.k_pos;
    if (iterations) *iterations = r.iterations;
    if (residual) *residual = r.residual;
  });
}

int wssr_debug_small_f64(wssr_ctx* ctx, int op, int k, const double* in, double* out1,
                         double* out2, int* status) {
  return guarded(ctx, [&] {
    Context& c = ctx->c;
    if (op == 0) {
      Buf st(1, c.stream);
      WSSR_CUDA(cudaMemsetAsync(st, 0, sizeof(double), c.stream));
      chol_inv(c, in, k, out1, out2, st.i32());
      WSSR_CUDA(cudaMemcpyAsync(status, st, 2 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    } else if (op == 1) {
      maxeig(c, in, k, out1);
    } else {
      throw Fail{WSSR_ERR_VALUE, "unknown op"};
    }
    sync(c);
  });
}

int wssr_debug_gemm_f32a(wssr_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k,
                         const float* a, int64_t lda, const double* shift, const double* b,
                         int64_t ldb, double* c, int64_t ldc, double alpha) {
  return guarded(ctx, [&] {
    GemmArgs g{reinterpret_cast<const double*>(a), lda, b, ldb, shift, c, ldc, m, n, k, 0, alpha,
               0, nullptr, nullptr, 0};
    const Layout L = layout == 0 ? Layout::CM : Layout::RM;
    if (!gemm_f32_supported(L, g)) throw Fail{WSSR_ERR_UNSUPPORTED, "operands not TMA-aligned"};
    WSSR_CUDA(gemm_f32a(ctx->c, L, g, 1024, ctx->c.stream));
  });
}

int wssr_debug_ozaki_gemm(wssr_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k,
                          const void* a, int64_t lda, int a_f32, const double* shift,
                          const double* b, int64_t ldb, double* c, int64_t ldc, double alpha) {
  return guarded(ctx, [&] {
    Context& cx = ctx->c;
    const Layout L = layout == 0 ? Layout::CM : Layout::RM;
    GemmArgs g{reinterpret_cast<const double*>(a), lda, b, ldb, shift, c, ldc, m, n, k, 0, alpha,
               0, nullptr, nullptr, 0};
    if (!ozaki_supported(L, g, a_f32 != 0)) throw Fail{WSSR_ERR_UNSUPPORTED, "operands not TMA-aligned"};
    // parameters run along K (RM) or M (CM); samples along the other
    const int64_t params = L == Layout::RM ? k : m, samples = L == Layout::RM ? m : k;
    Buf scale((size_t)ozaki_table_doubles(params), cx.stream);
    WSSR_CUDA(ozaki_scales(cx, a, a_f32 != 0, lda, samples, params, shift, scale, cx.stream));
    Buf planes;
    const int nds = (a_f32 && cx.f32_digits == 5) ? 5 : 7;
    if (cx.oz_pre == 0) {
      planes = Buf((ozaki_planes_bytes(samples, params, nds) + 7) / 8, cx.stream);
      WSSR_CUDA(ozaki_digitize(cx, a, a_f32 != 0, lda, samples, params, scale,
                               reinterpret_cast<int8_t*>(planes.p), cx.stream, nds));
    }
    WSSR_CUDA(ozaki_gemm(cx, L, g, a_f32 != 0, scale, cx.stream,
                         reinterpret_cast<const int8_t*>(planes.p), nullptr, nullptr, nds));
    sync(cx);
  });
}

int wssr_debug_ozaki_trace(wssr_ctx* ctx, long long* out, int64_t n) {
  return guarded(ctx, [&] {
    sync(ctx->c);
    WSSR_CUDA(ozaki_trace(out, (size_t)n * sizeof(long long)));
  });
}

int wssr_gemm_f64(wssr_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k, const double* a,
                  int64_t lda, const double* shift, const double* b, int64_t ldb, double* c,
                  int64_t ldc, double alpha, int accumulate, int max_splits) {
  return guarded(ctx, [&] {
    if (layout == 0)
      gemm_cm(ctx->c, m, n, k, a, lda, shift, b, ldb, c, ldc, alpha, accumulate != 0, max_splits);
    else
      gemm_rm(ctx->c, m, n, k, a, lda, shift, b, ldb, c, ldc, alpha, accumulate != 0, max_splits);
  });
}

}  // extern "C"
