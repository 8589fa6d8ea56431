"""Dense kernels on the device: drop-in for vmcsr.linalg.qr_orthonormalize (linalg.py:29-105).

The thin QR is CholeskyQR2 on FP64 tensor cores (Gram by DMMA GEMM, k x k Cholesky + inverse in
shared memory, Q = A R^-1 by DMMA GEMM, twice).  Where CholeskyQR2 cannot resolve a column
(pivot below its safety margin, or |R_jj| near the reference's 1e-12 ||A||_F deficiency rule)
the library runs the reference's own two-pass Gram-Schmidt with canonical-vector fill on the
device, so Q, R and the patched R_jj == 0 follow linalg.py:64-105.
"""

from __future__ import annotations

import torch

from . import _arrays, _lib

ZERO_MATRIX_NORM = 1e-300      # linalg.py:15
DEFICIENT_COLUMN_REL = 1e-12   # linalg.py:16


def _as_matrix(a):
    t = _arrays.to_tensor(a)
    if t.dim() == 1:
        t = t[:, None]
    if t.dim() != 2:
        raise ValueError(f"expected a matrix, got ndim={t.dim()}")
    return t


def exact_svd(a):
    """Economy SVD a = u @ diag(sigma) @ vt with sigma nonincreasing (linalg.py:108-121).

    On the device, in libwssr: min(m, n) <= 512 by a QR pre-reduction + single-CTA one-sided
    Jacobi; larger problems (the dense first step / 'exact' backend at BASELINE sizes,
    optimizers.py:327-330) by the blocked one-sided Jacobi of csrc/jacobi.cuh, which needs no
    full rank (the step-0 Ohat is rank-deficient by construction).  Singular vectors carry an
    arbitrary joint sign, as LAPACK's do.
    """
    a = _as_matrix(a)
    if not bool(torch.isfinite(a).all()):
        raise ValueError("matrix has non-finite entries")
    m, n = a.shape
    q = min(m, n)
    dev = a.device
    u = torch.zeros(m, q, dtype=torch.float64, device=dev)
    sig = torch.zeros(q, dtype=torch.float64, device=dev)
    vt = torch.zeros(q, n, dtype=torch.float64, device=dev)
    if not bool((a != 0).any()):
        u[:q, :q] = torch.eye(q, dtype=torch.float64, device=dev)
        vt[:q, :q] = torch.eye(q, dtype=torch.float64, device=dev)
        return u, sig, vt
    a = _arrays.rows_view(a)
    _lib.context().call("wssr_exact_svd_f64", m, n, _lib.ptr(a), _arrays.ld(a), _lib.ptr(u), q,
                        _lib.ptr(sig), _lib.ptr(vt), n)
    return u, sig, vt


def qr_orthonormalize(a):
    """Thin QR with orthonormal Q and a nonnegative diagonal of R (linalg.py:29-61).

    Returns:
      (q, r): q (m, n) with orthonormal columns, r (n, n) upper triangular, diag(r) >= 0.
    Raises:
      ZeroMatrix: if ||a||_F < 1e-300.  ValueError: if m < n.
    """
    a = _as_matrix(a)
    m, n = a.shape
    if m < n:
        raise ValueError(f"need at least as many rows as columns, got {tuple(a.shape)}")
    a = _arrays.rows_view(a)
    q = torch.empty(m, n, dtype=torch.float64, device=a.device)
    r = torch.empty(n, n, dtype=torch.float64, device=a.device)
    _lib.context().call("wssr_qr_f64", m, n, _lib.ptr(a), _arrays.ld(a), _lib.ptr(q), n,
                        _lib.ptr(r), 0)
    return _arrays.device_array(q), _arrays.device_array(r)
