/*
 * wssr.h - C ABI of the B200-native warm-started stochastic-reconfiguration (WSSR) step.
 *
 * Drop-in boundary for the reference package `vmcsr` (arXiv 2512.05749).  Every entry point
 * replaces one reference function; the Python shim in paper_2512_05749_b200/ binds them with
 * ctypes and keeps the reference's names, argument meaning and exception classes.
 *
 *   wssr_assemble_f64    <- vmcsr.estimators.assemble          estimators.py:74-100
 *                           (+ clip_local_energies              estimators.py:53-71)
 *   wssr_qr_f64          <- vmcsr.linalg.qr_orthonormalize      linalg.py:29-105
 *   wssr_ssi_svd_f64     <- vmcsr.svdengine.ssi_svd             svdengine.py:88-158
 *   wssr_subspace_drift_f64 <- vmcsr.svdengine.subspace_drift   svdengine.py:199-226
 *   wssr_step_f64        <- vmcsr.optimizers.wssr_step          optimizers.py:292-391
 *                           (svd_backend="ssi", state.step >= 1)
 *   wssr_gemm_f64        test/diagnostic export of the DMMA GEMM family (no reference twin)
 *
 * All array arguments are DEVICE pointers (CUDA global memory) of IEEE float64, row-major with
 * an explicit leading dimension.  The per-sample log-derivative matrix is passed sample-major
 * (N x P row-major, the reference's SampleBatch.theta_logderivs, estimators.py:22); the
 * reference's parameter-major o_matrix (P x N) is the same memory read column-major, so the
 * library never makes the transposed/centred copy the reference makes (estimators.py:91,97).
 *
 * No C++ exceptions cross this boundary.  Every function returns a WSSR_* status; the message
 * of the last failure is available from wssr_last_error().  Calls are stream-ordered on the
 * stream set with wssr_set_stream (default: the legacy default stream) and a context must not
 * be shared between host threads (reference: single control thread).
 */
#ifndef WSSR_H_
#define WSSR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  The shim raises the reference exception class named beside each code. */
enum {
  WSSR_OK = 0,
  WSSR_ERR_VALUE = 1,             /* ValueError (shapes/arguments, svdengine.py:124-125)     */
  WSSR_ERR_RANK_TOO_LARGE = 2,    /* errors.RankTooLarge   (svdengine.py:116-117)            */
  WSSR_ERR_DEGENERATE_INPUT = 3,  /* errors.DegenerateInput (svdengine.py:118-119, 149-150)  */
  WSSR_ERR_ZERO_MATRIX = 4,       /* errors.ZeroMatrix      (linalg.py:53-54, 103-104)       */
  WSSR_ERR_RANK_COLLAPSE = 5,     /* errors.RankCollapse    (optimizers.py:350-351)          */
  WSSR_ERR_DEGENERATE_BATCH = 6,  /* errors.DegenerateBatch (estimators.py:61-62, 84-85)     */
  WSSR_ERR_CUDA = 7,              /* CUDA runtime failure                                     */
  WSSR_ERR_NCCL = 8,              /* collective failure                                       */
  WSSR_ERR_UNSUPPORTED = 9,       /* configuration not implemented on the device path         */
  WSSR_ERR_NODE_PROXIMITY = 10    /* errors.NodeProximity   (wavefunction.py:317-318)        */
};

/* ssi / step flags */
#define WSSR_FLAG_FINAL_RESIDUAL 0x1 /* also run the look-ahead after the last iteration so   */
                                     /* SsiReport.subspace_residual is filled (svdengine.py:137) */
#define WSSR_FLAG_CAREFUL 0x2        /* host-checked QR with the Gram-Schmidt patch path        */

typedef struct wssr_ctx wssr_ctx;

/*
 * The stacked matrix Ohat of optimizers.py:323, in the sample-major view:
 *   Ohat^T = [ hist_scale    * hist                       ]   (hist_rank rows)
 *            [ samples_scale * (samples - 1 * mu^T)       ]   (n_samples rows)
 * hist = state.obar^T (hist_rank x P), samples = raw log-derivatives (n_samples x P),
 * mu = column means (P, or NULL for no centring).  samples_fro2 = ||samples_scale*(samples-mu)||_F^2
 * when known (from wssr_assemble_f64), or < 0 to have the library compute it.
 * Under row sharding `samples` is this rank's row shard and the history block lives on rank 0.
 */
typedef struct wssr_ohat_f64 {
  int64_t n_params;
  const double* hist;
  int64_t hist_rank;
  int64_t hist_ld;
  double hist_scale;
  const double* samples;
  int64_t n_samples;
  int64_t samples_ld;
  const double* mu;
  double samples_scale;
  double samples_fro2;
  int64_t samples_f32; /* 1: `samples` points to float32 data (FP32 variant, BASELINE configs[3]);
                          the library widens it to FP64 in registers. Requires ld % 4 == 0,
                          16-byte alignment, mu and samples_fro2 (i.e. an assembled bundle). */
  const double* samples_scale_table; /* optional [4 * roundup(n_params, 32)]: the per-parameter
                          {cw_p, 2^(54 - e_p), mu_p, 0} table of the int8 tensor-core O-passes
                          (cw_p: integer centring word, csrc/ozaki.cu biased_digits), as written
                          by assemble (wssr_assemble_out.scale_table); NULL: computed on demand
                          with one extra read of the sample block. */
  const double* samples_fro2_dev; /* optional: when samples_fro2 < 0, the device value of the
                          sample block's ||.||_F^2 (wssr_assemble_out.fro2_dev); read at the first
                          host synchronisation of the step instead of up front. */
} wssr_ohat_f64;

/* --- context ------------------------------------------------------------------------------ */
int wssr_ctx_create(int device, wssr_ctx** out);
void wssr_ctx_destroy(wssr_ctx* ctx);
const char* wssr_last_error(const wssr_ctx* ctx);
int wssr_set_stream(wssr_ctx* ctx, void* cuda_stream);
int wssr_version(void);
/* number of kernels this context launched so far (bench.py's gpu_launches) */
int64_t wssr_kernel_launches(const wssr_ctx* ctx);

/* GEMM path of the O-passes:
 *   0 = auto: large sample blocks on the int8 tensor cores (exact digit products, ozaki.cu),
 *       digitised once per step into HBM when the planes fit, else on the fly; the rest on
 *       FP64 DMMA with the TMA + mbarrier pipeline;
 *   1 = FP64 DMMA with the cp.async pipeline only;
 *   2 = FP64 DMMA only (TMA where operands allow it);
 *   3 = int8 tensor-core path for every sample block it supports (tests);
 *   4 = as 3 with on-the-fly digitising only (tests). */
int wssr_set_gemm_path(wssr_ctx* ctx, int path);

/* Precision guard of the int8 O-passes (on by default).  The digits keep every element to 2^-54
 * of its parameter column's scale; when fewer than 1/64 of a sample row's nonzero elements keep
 * 42 bits of their own magnitude (heavy-tailed rows: a few samples dominate the column maxima)
 * the step's SSI is re-run with the O-passes on FP64 DMMA.  wssr_precision_fallbacks counts
 * those re-runs. */
int wssr_set_precision_guard(wssr_ctx* ctx, int enabled);
int64_t wssr_precision_fallbacks(const wssr_ctx* ctx);

/* bench instrumentation: per-phase CUDA-event timing of the O-passes.
 * phase 0 = v = Ohat^T q (svdengine.py:133), 1 = u = Ohat v (svdengine.py:134),
 * 2 = assemble's column-statistics pass (estimators.py:91,93).  Enabling resets the totals. */
int wssr_set_timing(wssr_ctx* ctx, int enabled);
int wssr_phase_stats(wssr_ctx* ctx, int phase, double* ms, int64_t* launches, double* flops,
                     double* bytes);
/* measured FP64 tensor-core (DMMA) peak of this device, TFLOP/s (roofline denominator) */
int wssr_dmma_peak_probe(wssr_ctx* ctx, double* tflops);

/* --- row sharding over NCCL (one process per GPU) ----------------------------------------- */
/* 128-byte ncclUniqueId produced on rank 0 and broadcast by the caller (torch.distributed). */
int wssr_nccl_unique_id(wssr_ctx* ctx, unsigned char out_id[128]);
int wssr_nccl_attach(wssr_ctx* ctx, const unsigned char id[128], int rank, int world);
/* (world == 1 builds a 1-rank communicator: the engine stays unsharded and wssr_allreduce_f64
 * then exercises the NCCL transport itself.) */

/* Thread-emulated communicator for testing the sharded engine on one GPU: `world` host threads,
 * each with its own context and stream, attach to one group; collectives synchronise on the host
 * and sum in rank order.  Not for production use (no GPU-side waits, no overlap). */
int wssr_emu_group_create(int world, void** group);
void wssr_emu_group_abort(void* group); /* a failed rank releases its waiting peers */
void wssr_emu_group_destroy(void* group);
int wssr_emu_attach(wssr_ctx* ctx, void* group, int rank);

/* In-place sum over the attached communicator's ranks (no-op when none is attached).  Used by
 * the host mirror to gather the dense first-step matrix of a row-sharded run
 * (optimizers.py:327-331 factorises the whole Ohat). */
int wssr_allreduce_f64(wssr_ctx* ctx, double* buf, int64_t n);

/* --- estimators.assemble (estimators.py:74-100) ------------------------------------------- */
typedef struct wssr_assemble_out {
  double* mu;       /* [P]  column means of theta_logderivs (global over ranks)               */
  double* l_vector; /* [N]  (clip(E) - loss) / sqrt(N_global)                                 */
  double* gradient; /* [P]  2 * o_matrix @ l_vector                                           */
  /* host outputs */
  double loss, raw_loss, e_mean, e_std;
  double fro2;      /* ||o_matrix||_F^2                                                      */
  int64_t n_global;
  double* scale_table; /* optional [4 * roundup(P, 32)]: per-parameter scales of the int8
                          tensor-core O-passes, from the same column pass (this rank's rows) */
  /* optional deferred host outputs (single rank): when `deferred` (pinned host memory, 5
     doubles) is non-NULL the call returns without waiting for the device; {loss, raw_loss,
     e_mean, e_std, fro2} land there in stream order (valid once the stream reaches this point)
     and the host fields above are left unset.  fro2_dev (device, 1 double) then receives fro2
     for wssr_ohat_f64.samples_fro2_dev, so a following wssr_step never waits on assemble. */
  double* deferred;
  double* fro2_dev;
} wssr_assemble_out;
int wssr_assemble_f64(wssr_ctx* ctx, const double* derivs, int64_t n, int64_t p, int64_t ld,
                      const double* energies, double clip_n_std, wssr_assemble_out* out);

/* FP32 variant of wssr_assemble_f64: float32 derivs, FP64 statistics and outputs */
int wssr_assemble_f32(wssr_ctx* ctx, const float* derivs, int64_t n, int64_t p, int64_t ld,
                      const double* energies, double clip_n_std, wssr_assemble_out* out);

/* --- linalg.qr_orthonormalize (linalg.py:29-61) ------------------------------------------- */
int wssr_qr_f64(wssr_ctx* ctx, int64_t rows, int64_t cols, const double* a, int64_t lda,
                double* q, int64_t ldq, double* r /* cols x cols */, int64_t flags);

/* --- svdengine.ssi_svd (svdengine.py:88-158) ---------------------------------------------- */
typedef struct wssr_ssi_out {
  double* u;       /* [P x rank], ld_u: left vectors; first k_pos columns valid              */
  int64_t ld_u;
  double* sigma;   /* [rank] sorted singular values (first k_pos valid)                     */
  double* v;       /* [(hist_rank+n_samples) x rank], ld_v: right vectors as columns, or NULL */
  int64_t ld_v;
  /* host outputs */
  int64_t k_pos;
  int64_t iterations;
  double residual; /* NaN when the final look-ahead was skipped (no WSSR_FLAG_FINAL_RESIDUAL) */
} wssr_ssi_out;
int wssr_ssi_svd_f64(wssr_ctx* ctx, const wssr_ohat_f64* ohat, int64_t rank, int64_t max_iters,
                     const double* u_init, int64_t ld_init, double residual_tol, int64_t flags,
                     wssr_ssi_out* out);

/* --- svdengine.subspace_drift (svdengine.py:199-226) -------------------------------------- */
int wssr_subspace_drift_f64(wssr_ctx* ctx, int64_t n_rows, const double* u1, int64_t ld1,
                            const double* s1, int64_t r1, const double* u2, int64_t ld2,
                            const double* s2, int64_t r2, double* sigma_drift,
                            double* projector_drift);

/* --- optimizers.wssr_step (optimizers.py:292-391), warm-started SSI branch ----------------- */
typedef struct wssr_step_in {
  const wssr_ohat_f64* ohat; /* hist = state.obar^T, hist_scale = 1 (library applies sqrt(delta));
                                samples_scale = bundle scale (library applies sqrt(1-delta))  */
  const double* lbar;        /* [hist_rank] state.lbar                                        */
  const double* l_vector;    /* [n_samples] bundle.l_vector                                    */
  const double* gradient;    /* [P] bundle.gradient when it is exactly 2*o_matrix@l_vector
                                (as produced by wssr_assemble_f64), else NULL -> recomputed   */
  const double* theta;       /* [P] */
  double eta;
  const double* u_init;      /* [P x requested] warm start (optimizers.py:277-289, prepared by
                                the caller: it owns the host-side PCG64 draws)               */
  int64_t ld_init;
  int64_t requested;         /* min(r_max, P, r + N)  (optimizers.py:326)                      */
  const double* u_prev;      /* state.u_prev [P x r_prev] (drift telemetry)                    */
  int64_t ld_prev;
  int64_t r_prev;
  double delta, sigma_floor, r_reg, eps_grow;
  int64_t sigma_floor_relative;
  int64_t r_max;
  int64_t max_iters;
  double residual_tol;
  int64_t flags;
  /* optional externally computed factors (dense 'exact' / 'randomized' backends and the first
     step, optimizers.py:327-338): when ext_u != NULL the SSI is skipped and the rank cut, gbar,
     preconditioner, drift and state refresh run on U [P x ext_k_pos], sigma (sorted, positive)
     and V [(hist_rank+n_samples) x ext_k_pos] (right vectors as columns). */
  const double* ext_u;
  int64_t ext_ld_u;
  const double* ext_sigma;
  const double* ext_v;
  int64_t ext_ld_v;
  int64_t ext_k_pos;
} wssr_step_in;

typedef struct wssr_step_out {
  double* theta_next;   /* [P] */
  double* update;       /* [P] preconditioned direction, or NULL */
  double* u_next;       /* [P x requested], ld_u: state'.u_prev (first r_eff columns)          */
  int64_t ld_u;
  double* obar_next_t;  /* [requested x P], ld_obar: state'.obar^T = (U sigma)^T              */
  int64_t ld_obar;
  double* lbar_next;    /* [requested] state'.lbar (first r_eff entries)                     */
  double* sigma;        /* [requested] sorted singular values                                */
  /* host outputs */
  int64_t r_eff, k_pos, iterations, next_r_max, binding;
  double residual, sigma_drift, projector_drift;
  /* optional: pinned host memory for {sigma_drift, projector_drift}.  With an auxiliary stream set
     (wssr_set_aux_stream) and a single rank, the drift telemetry (optimizers.py:366-374) runs on
     that stream after the step's own work and its two values land here in aux-stream order;
     the host fields above then read NaN and the call does not wait for them.  Without an aux
     stream the values are written here too (synchronously). */
  double* drift_host;
} wssr_step_out;
int wssr_step_f64(wssr_ctx* ctx, const wssr_step_in* in, wssr_step_out* out);

/* --- linalg.exact_svd (linalg.py:108-121; numpy's dgesdd there): u [m x q], sigma [q] sorted
 * descending, vt [q x n], q = min(m, n).  min(m, n) <= 512: QR pre-reduction + single-CTA
 * one-sided Jacobi; larger: blocked one-sided Jacobi on the min(m, n) vectors of a (csrc/jacobi.cuh,
 * DMMA Grams and updates, any rank). */
int wssr_exact_svd_f64(wssr_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                       double* u, int64_t ldu, double* sigma, double* vt, int64_t ldvt);
/* exact_truncated_svd (svdengine.py:75-85) of the implicit Ohat of optimizers.py:323 (history
 * scaled by sqrt(delta), samples by sqrt(1 - delta)) without forming it: oversampled block power
 * iteration on the O-pass kernels until the leading `rank` Ritz triplets have residual
 * ||Ohat v_i - s_i u_i|| <= tol * s_i (or stagnate at the rounding floor), then Rayleigh-Ritz.
 * Row-sharded: every rank passes its own samples (history on rank 0), cols_global = r + N over
 * all ranks and col0 = this rank's first global column; u and sigma come out replicated and
 * v_local holds this rank's rows of the right vectors (cols x rank).  k_pos = leading positive
 * singular values kept (svdengine.py:70-72). */
int wssr_implicit_svd_f64(wssr_ctx* ctx, const wssr_ohat_f64* ohat, double delta, int64_t rank,
                          int64_t cols_global, int64_t col0, uint64_t seed, int64_t max_iters,
                          double tol, double* u, int64_t ldu, double* sigma, double* v_local,
                          int64_t ldv, int64_t* k_pos, int64_t* iterations, double* residual);
/* Ohat of optimizers.py:323 written out parameter-major: out [P x (hist_rank + n_samples)]. */
int wssr_materialize_ohat_f64(wssr_ctx* ctx, const wssr_ohat_f64* ohat, double delta, double* out,
                              int64_t ldo);

/* --- diagnostics: small k x k device routines (tests).  op 0: CholeskyQR core, in = G (k x k),
 * out1 = R, out2 = R^-1, status[2] = {failed pivot (1-based) or 0, zero-matrix flag};
 * op 1: largest eigenvalue of symmetric `in`, out1[0] = lambda_max. */
int wssr_debug_small_f64(wssr_ctx* ctx, int op, int k, const double* in, double* out1,
                         double* out2, int* status);

/* diagnostics: the FP32-operand GEMM (A float32, widened to FP64; layouts as wssr_gemm_f64) */
int wssr_debug_gemm_f32a(wssr_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k,
                         const float* a, int64_t lda, const double* shift, const double* b,
                         int64_t ldb, double* c, int64_t ldc, double alpha);

/* test hook: one O-pass GEMM on the int8 tensor-core path (scales computed from `a`).
 * layout 0: C (m x n) = alpha (A - 1 shift^T)^T B with A stored (k x m) row-major;
 * layout 1: C (m x n) = alpha (A - 1 shift^T) B with A (m x k) row-major.  a_f32: A is float. */
int wssr_debug_ozaki_gemm(wssr_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k,
                          const void* a, int64_t lda, int a_f32, const double* shift,
                          const double* b, int64_t ldb, double* c, int64_t ldc, double alpha);

/* profiling hook: per-K-block timestamps (SM clock) of CTA 0 of the last int8 O-pass launched
 * with WSSR_OZ_DEBUG=9, 8 rows x 96 K-blocks (producer, MMA issuers, converter group leaders). */
int wssr_debug_ozaki_trace(wssr_ctx* ctx, long long* out, int64_t n);

/* engine option: 1 (default) runs the Grams and k x k products of P x k blocks with k = 32, 64, 128
 * (CholeskyQR2, Rayleigh quotient and residual, drift) on the tall-skinny kernels
 * (csrc/tallskinny.cu); 0 on the generic tile GEMMs. */
int wssr_set_tallskinny(wssr_ctx* ctx, int enabled);

/* returns the context's cached device memory (digit planes, scratch blocks, the stream-ordered
 * pool's reserve) to the driver; everything regrows on demand.  Synchronises the device. */
int wssr_release_memory(wssr_ctx* ctx);

/* engine option (row-sharded runs): 1 (default) works the P x k tail of the SSI in P-slices, one
 * per rank (reduce-scatter of u and w, slice CholeskyQR2 with allreduced k x k Grams, all-gather
 * of q); 0 keeps it replicated on every rank (allreduce of u). */
int wssr_set_tail_shard(wssr_ctx* ctx, int enabled);

/* engine option: sample digits of the int8 O-passes for float32 samples (BASELINE configs[3]):
 * 5 (default) = the 5 most significant of the 7 digits (each element to 2^-38 of its column's
 * scale, exact for float32 values within 14 binades of the column maximum; 20 digit pairs and 5
 * planes in HBM), 7 = the FP64-grade scheme of float64 samples (28 pairs, 7 planes). */
int wssr_set_fp32_digits(wssr_ctx* ctx, int digits);

/* digit pairs per product that the FP64-grade int8 O-passes of this build keep: 28 (pairs of
 * significance a + b <= 6, truncation below 2^-51.4 of the column-scale product; the default)
 * or 34 (a + b <= 7, below 2^-59; built with -DWSSR_OZ_LEVELS=8). */
int wssr_ozaki_digit_pairs(void);

/* engine option: dense SVD mode, 0 (default) = single-CTA Jacobi up to min(m, n) = 512 and the
 * blocked Jacobi above; 1 = the blocked Jacobi at every size (tests). */
int wssr_set_dense_svd_mode(wssr_ctx* ctx, int mode);
/* outer sweeps of the last blocked dense SVD (diagnostics) */
int wssr_dense_svd_sweeps(const wssr_ctx* ctx);

/* auxiliary CUDA stream for the asynchronous drift telemetry of wssr_step_f64 (NULL: none).  The
 * caller keeps the step's inputs/outputs alive until that stream passes the step (e.g. torch's
 * record_stream). */
int wssr_set_aux_stream(wssr_ctx* ctx, void* cuda_stream);

/* test hook: one tall-skinny kernel, row-major operands with ld = k (k = 32, 64 or 128).
 * op 0: out = A^T A (k x k); op 1: out = A^T B; op 2: out (rows x k) = A (alpha M) with M upper
 * triangular; op 3: out = A (alpha M); op 4: out = Cin + A (alpha M);
 * op 5: out[0] = ||Cin + A (alpha M)||_F^2; op 6: out (k) = alpha A^T x, x = cin (rows). */
int wssr_debug_tallskinny(wssr_ctx* ctx, int op, int64_t rows, int64_t k, const double* a,
                          const double* b, const double* m, const double* cin, double alpha,
                          double* out);

/* --- producer of O: AceWavefunction.grad_theta_batch (wavefunction.py:307-321) on the device.
 * Every pointer is device memory.  Orbitals follow the reference's canonical basis order; axis is
 * the Cartesian component of a p orbital (x 0, y 1, z 2; -1 for s), gate 0 up / 1 down /
 * 2 either; tails are n_features x max_tail orbital indices padded with -1 (the pooled factors of
 * each feature, build_tuple_index); coef is theta as (n_electrons x n_features). */
typedef struct wssr_ace_spec {
  int64_t n_electrons, n_orbitals, n_features, n_nuclei, max_tail;
  const double* nuclei;      /* [n_nuclei x 3] */
  const int32_t* spins;      /* [n_electrons]: 0 up, 1 down */
  const int32_t* orb_center; /* [n_orbitals] */
  const int32_t* orb_n;
  const int32_t* orb_axis;
  const int32_t* orb_gate;
  const double* orb_zeta;
  const int32_t* heads;      /* [n_features] */
  const int32_t* tails;      /* [n_features x max_tail] */
  const double* coef;        /* [n_electrons x n_features] */
} wssr_ace_spec;
/* out [W x ld_out]: row w = d log|psi| / d theta at positions[w] ([W x N x 3]); n_electrons <= 64.
 * Returns WSSR_ERR_NODE_PROXIMITY when a walker's determinant vanishes or underflows. */
int wssr_grad_theta_f64(wssr_ctx* ctx, const wssr_ace_spec* spec, const double* positions,
                        int64_t n_walkers, double* out, int64_t ld_out);

/* --- diagnostics: C(MxN) = alpha * op(A) B (+C); layout 0: A stored [K][M], 1: A stored [M][K] */
int wssr_gemm_f64(wssr_ctx* ctx, int layout, int64_t m, int64_t n, int64_t k, const double* a,
                  int64_t lda, const double* shift, const double* b, int64_t ldb, double* c,
                  int64_t ldc, double alpha, int accumulate, int max_splits);

#ifdef __cplusplus
}
#endif

#endif /* WSSR_H_ */
