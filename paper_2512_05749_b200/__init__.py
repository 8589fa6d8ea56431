"""B200-native drop-in for the WSSR step of arXiv 2512.05749 (reference package `vmcsr`).

Public surface mirrors the reference modules used on the hot path:
  estimators   SampleBatch, EstimatorBundle, clip_local_energies, assemble
  linalg       qr_orthonormalize
  svdengine    TruncatedSvd, SsiReport, ssi_svd, subspace_drift, subspace_residual
  optimizers   WssrState, WssrDiagnostics, wssr_step, rssr_step
  errors       the reference exception classes
Compute runs in libwssr.so (hand-written sm_100a kernels behind the C ABI in include/wssr.h).
"""

__version__ = "0.1.0"

from . import errors  # noqa: F401
