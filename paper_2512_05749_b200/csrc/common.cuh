// Shared device helpers for the WSSR sm_100a kernels.
//
// Conventions used by every kernel in this directory:
//   * "O" is the per-sample log-derivative matrix stored sample-major, i.e. row-major N x P
//     (rows = samples/walkers, columns = parameters).  This is the same memory as the
//     reference's parameter-major o_matrix (P x N, estimators.py:40) read column-major, so
//     no transpose copy is ever made (reference copies it at estimators.py:91,97).
//   * P x k blocks (q, u, w, U, u_prev) are row-major P x ld (ld >= k).
//   * All reductions run in a fixed order (no floating-point atomics) so repeated calls are
//     bitwise identical, matching the reference's determinism contract
//     (tests/test_svdengine.py:124-132 of the reference).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <utility>

namespace wssr {

constexpr int kWarp = 32;

// Programmatic dependent launch.  Every kernel of this library is launched with
// programmaticStreamSerialization, so its CTAs may be scheduled while the previous kernel in the
// stream drains; each kernel therefore starts with pdl_wait() (griddepcontrol.wait), which
// returns once the previous grid has completed and its memory is visible.  What overlaps is the
// launch latency and CTA rasterisation of kernel i+1 with the tail of kernel i (~2-3 us per
// boundary, over ~120 launches per WSSR step).  WSSR_NO_PDL=1 launches plainly.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("WSSR_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: `done` (one per kernel
// instantiation, at the call site) keeps one bit per device id, so a context on a second GPU of
// the same process sets it again.  Two threads racing here both set it, which is harmless.
template <typename K>
inline cudaError_t smem_attr_once(std::atomic<uint64_t>& done, K kern, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// D(8x8) += A(8x4,row) * B(4x8,col), FP64 tensor core (SASS: DMMA.8x8x4).
// Fragment ownership (PTX ISA, mma.m8n8k4 .f64): lane = 4*g + t,
//   a = A[g][t], b = B[t][g], c[e] = C[g][2t+e].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// cp.async (LDGSTS) with zero-fill of the bytes past src_bytes.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// FP64 reciprocal / reciprocal square root on a latency-critical path: float SFU seed + two
// Newton steps (relative error ~1e-16; IEEE div/sqrt sequences cost ~250 cycles each, which
// dominated the k-step dependency chains of the k x k solvers).  Inputs outside the float range
// take the exact library path.
__device__ __forceinline__ double fast_rcp(double x) {
  const double ax = fabs(x);
  if (!(ax > 1e-36 && ax < 1e36)) return 1.0 / x;
  double y = (double)__frcp_rn((float)x);
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  if (!(x > 1e-36 && x < 1e36)) return 1.0 / sqrt(x);
  double y = (double)rsqrtf((float)x);
  double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum in a fixed order (warp butterflies, then warp 0 over the warp partials).
// `scratch` needs blockDim.x/32 doubles. Result is broadcast to every thread.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane_id() == 0) scratch[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane_id() < nw ? scratch[lane_id()] : 0.0;
    t = warp_sum(t);
    if (lane_id() == 0) scratch[0] = t;
  }
  __syncthreads();
  t = scratch[0];
  __syncthreads();
  return t;
}

__device__ __forceinline__ double block_max(double v, double* scratch) {
  v = warp_max(v);
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane_id() == 0) scratch[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane_id() < nw ? scratch[lane_id()] : -1.0 / 0.0;
    t = warp_max(t);
    if (lane_id() == 0) scratch[0] = t;
  }
  __syncthreads();
  t = scratch[0];
  __syncthreads();
  return t;
}

}  // namespace wssr
