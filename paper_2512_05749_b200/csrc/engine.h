// Native WSSR engine: owns the device workspace, launches the sm_100a kernels in stream order
// and implements the reference's control flow (assemble, ssi_svd, wssr_step) in C++.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/wssr.h"

namespace wssr {

enum class Layout : int;
struct GemmArgs;

// Collective interface for row (sample) sharding.  world == 1 -> no-op.
struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  virtual cudaError_t allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;
  // In place over buf[world * count]: afterwards this rank's slice [rank * count, +count) holds
  // the sum over ranks (the other slices are unspecified).
  virtual cudaError_t reduce_scatter_sum(double* buf, size_t count, cudaStream_t st) {
    return allreduce_sum(buf, (size_t)world * count, st);
  }
  // In place over buf[world * count]: every rank's slice is copied to all ranks.
  virtual cudaError_t all_gather(double* buf, size_t count, cudaStream_t st) = 0;
};

struct Context {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  std::string last_error;
  double* splitk = nullptr;
  size_t splitk_cap = 0;  // doubles
  int* flags = nullptr;   // device status words (see engine.cu)
  Comm* comm = nullptr;
  int64_t gemm_launches = 0;  // statistics for bench.py
  int64_t kernel_launches = 0;
  bool disable_tma = false;  // force the cp.async GEMM path (tests / A-B comparisons)
  bool ozaki = true;         // O-passes on the int8 tensor cores (exact digit products)
  double oz_min_elems = 4194304.0;  // smallest sample block (elements) sent to that path
  bool oz_guard = true;      // precision guard of the int8 path (ozaki.cu row_guard_kernel)
  int64_t precision_fallbacks = 0;  // SSI re-runs on DMMA after the guard fired
  bool chol_series = true;   // near-identity Grams: series Cholesky (kernels.cuh chol_series)
  bool tallskinny = true;    // k = 32/64 Grams and products of P x k blocks: tallskinny.cu
  bool force_blocked_svd = false;  // dense SVD: blocked Jacobi at every size (tests)
  bool tail_shard = true;          // row-sharded runs: the P x k tail of the SSI on P-slices
  int dense_svd_sweeps = 0;        // outer sweeps of the last blocked dense SVD
  double* hbuf = nullptr;          // pinned host staging for the step's small readbacks (4096)
  cudaStream_t aux = nullptr;      // optional: asynchronous drift telemetry (wssr_set_aux_stream)
  cudaEvent_t aux_event = nullptr;
  double* aux_splitk = nullptr;    // the aux stream's own split-K / slab buffer
  size_t aux_splitk_cap = 0;
  int oz_pre = 0;            // digit planes: 0 = pre-digitise when they fit, 1 = on the fly only
  int8_t* oz_planes = nullptr;  // the step's pre-digitised sample block (reused across steps)
  size_t oz_planes_cap = 0;     // bytes
  int64_t plan_n = -1, plan_p = -1, plan_k = -1, plan_rows = 0;  // last partial-planes decision
  int plan_nds = 7;
  bool plan_provisional = false;  // that decision used the cold (first-step) memory margin
  int f32_digits = 5;             // sample digits of the int8 O-passes for float32 samples (5|7)
  int64_t steps_done = 0;         // completed wssr_step calls (the scratch pool is warm after one)
  double* oz_ws = nullptr;   // Ozaki thin-operand digits + factors
  size_t oz_ws_cap = 0;      // doubles

  // optional per-phase timing of the O-passes (CUDA events on the launching stream)
  // 0: v = Ohat^T q, 1: u = Ohat v, 2: assemble column pass, 3: CholeskyQR2 of P x k blocks,
  // 4: SSI quotient + residual, 5: drift, 6: preconditioner + state refresh, 7: QR(v) + sort
  // 8-15 (WSSR_FINE_PHASES=1, profiling): CholeskyQR2 pieces - Gram 1, chol 1, TRMM 1, Gram 2,
  // chol 2, TRMM 2, triu product, other
  static constexpr int kPhases = 16;
  bool fine_phases = false;
  bool timing = false;
  struct PendingEvent {
    int phase;
    cudaEvent_t a, b;
    double flops, bytes;
  };
  std::vector<PendingEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  double phase_ms[kPhases] = {};
  double phase_flops[kPhases] = {};
  double phase_bytes[kPhases] = {};
  int64_t phase_count[kPhases] = {};

  double* splitk_buffer(size_t n);
  int world() const { return comm ? comm->world : 1; }
  cudaError_t allreduce(double* buf, size_t n) {
    if (!comm || comm->world == 1 || n == 0) return cudaSuccess;
    return comm->allreduce_sum(buf, n, stream);
  }
};

cudaError_t gemm(Context& ctx, Layout layout, const GemmArgs& args, int max_splits,
                 cudaStream_t st);
// A operand stored as float32 (O of the FP32 variant)
bool gemm_f32_supported(Layout layout, const GemmArgs& args);
cudaError_t gemm_f32a(Context& ctx, Layout layout, const GemmArgs& args, int max_splits,
                      cudaStream_t st);

// Status codes mirror include/wssr.h.
struct Error {
  int code;
  std::string msg;
};

}  // namespace wssr
