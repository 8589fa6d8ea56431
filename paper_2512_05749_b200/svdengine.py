"""Truncated-SVD engine on the device: drop-in for vmcsr.svdengine (svdengine.py:1-226).

``ssi_svd`` is the warm-startable block subspace iteration of svdengine.py:88-158 with every
O-pass on FP64 tensor cores and every QR by CholeskyQR2; sigma is |diag R| of the QR of the
final v block, sorted with a stable argsort, exactly as the reference defines it
(svdengine.py:144-152).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays, _lib
from .errors import DegenerateInput, RankTooLarge, Unsupported

DEFAULT_RESIDUAL_EXIT = 1e-10   # svdengine.py:16
_COLD_START_SEED = 0x5EED       # svdengine.py:17


@dataclass(frozen=True)
class TruncatedSvd:
    """Rank-r factors: a ~= u @ diag(sigma) @ v (svdengine.py:20-44)."""

    u: object      # (m, r)
    sigma: object  # (r,)
    v: object      # (r, n)

    def __post_init__(self):
        for name in ("u", "sigma", "v"):  # numpy-readable device arrays (_arrays.DeviceArray)
            object.__setattr__(self, name, _arrays.device_array(getattr(self, name)))
        r = self.sigma.shape[0]
        if self.u.dim() != 2 if isinstance(self.u, torch.Tensor) else np.ndim(self.u) != 2:
            raise ValueError("malformed factor shapes")
        if tuple(self.u.shape)[1] != r or tuple(self.v.shape)[0] != r or len(self.sigma.shape) != 1:
            raise ValueError(
                f"inconsistent ranks: u {tuple(self.u.shape)}, sigma {r}, v {tuple(self.v.shape)}"
            )
        if r:
            s = _arrays.host(self.sigma)
            if np.any(s <= 0.0) or np.any(np.diff(s) > 0.0):
                raise ValueError("sigma must be strictly positive and nonincreasing")

    @property
    def rank(self):
        return self.sigma.shape[0]

    def reconstruct(self):
        return (self.u * self.sigma) @ self.v


@dataclass(frozen=True)
class SsiReport:
    """Telemetry from one factorization call (svdengine.py:47-53)."""

    iterations_used: int
    subspace_residual: float
    warm_started: bool


def _ohat_struct(samples, mu=None, scale=1.0, fro2=-1.0, hist=None, hist_scale=0.0,
                 scale_table=None, fro2_dev=None):
    """wssr_ohat_f64 for Ohat^T = [hist_scale*hist ; scale*(samples - mu)] (sample-major).

    scale_table: the bundle's per-parameter table from assemble (same mu), or None.
    """
    p = int(samples.shape[1])
    o = _lib.OhatF64()
    o.n_params = p
    if hist is not None and hist.shape[0] > 0:
        o.hist = hist.data_ptr()
        o.hist_rank = int(hist.shape[0])
        o.hist_ld = _arrays.ld(hist)
        o.hist_scale = float(hist_scale)
    else:
        o.hist, o.hist_rank, o.hist_ld, o.hist_scale = None, 0, p, 0.0
    o.samples = samples.data_ptr() if samples.shape[0] > 0 else None
    o.n_samples = int(samples.shape[0])
    o.samples_ld = _arrays.ld(samples) if samples.shape[0] > 0 else p
    o.mu = mu.data_ptr() if mu is not None else None
    o.samples_scale = float(scale)
    o.samples_fro2 = float(fro2)
    o.samples_f32 = int(samples.dtype == torch.float32)
    o.samples_scale_table = scale_table.data_ptr() if scale_table is not None else None
    # fro2 < 0 with fro2_dev: the value is still on its way from assemble (read by the engine at
    # its first host synchronisation)
    o.samples_fro2_dev = fro2_dev.data_ptr() if (fro2 < 0 and fro2_dev is not None) else None
    return o


def _sample_major(ohat):
    """(m, n) parameter-major matrix -> its (n, m) sample-major row view (no copy if possible)."""
    t = _arrays.to_tensor(ohat)
    if t.dim() != 2:
        raise ValueError("ohat must be a matrix")
    return _arrays.rows_view(t.t())


def subspace_residual(ohat, u_orthonormal):
    """||G U - U (U^T G U)||_F / ||ohat||_F^2 with G = ohat ohat^T (svdengine.py:56-67)."""
    ctx = _lib.context()
    s = _sample_major(ohat)                       # n x m
    u = _arrays.rows_view(_arrays.to_tensor(u_orthonormal))
    m, k = u.shape
    n = s.shape[0]
    fro2 = float(torch.linalg.vector_norm(s)) ** 2 if s.numel() else 0.0
    if fro2 == 0.0:
        raise DegenerateInput("residual undefined for a zero matrix")
    dev = u.device
    y = torch.empty(n, k, dtype=torch.float64, device=dev)
    w = torch.empty(m, k, dtype=torch.float64, device=dev)
    quo = torch.empty(k, k, dtype=torch.float64, device=dev)
    # y = ohat^T u (RM), w = ohat y (CM), quo = u^T w (CM), w -= u quo (RM)
    ctx.call("wssr_gemm_f64", 1, n, k, m, _lib.ptr(s), _arrays.ld(s), None, _lib.ptr(u),
             _arrays.ld(u), _lib.ptr(y), k, 1.0, 0, 1024)
    ctx.call("wssr_gemm_f64", 0, m, k, n, _lib.ptr(s), _arrays.ld(s), None, _lib.ptr(y), k,
             _lib.ptr(w), k, 1.0, 0, 1024)
    ctx.call("wssr_gemm_f64", 0, k, k, m, _lib.ptr(u), _arrays.ld(u), None, _lib.ptr(w), k,
             _lib.ptr(quo), k, 1.0, 0, 1024)
    ctx.call("wssr_gemm_f64", 1, m, k, k, _lib.ptr(u), _arrays.ld(u), None, _lib.ptr(quo), k,
             _lib.ptr(w), k, -1.0, 1, 1024)
    return float(torch.linalg.vector_norm(w)) / fro2


def _positive_prefix(sigma, limit):
    """svdengine.py:70-72."""
    return int((sigma[:limit] > 0.0).sum().item())


def exact_truncated_svd(ohat, rank):
    """Dense SVD truncated to the leading triplets, exact zeros dropped (svdengine.py:75-85).

    Device path: libwssr's one-sided Jacobi SVD (single-CTA up to min(m, n) = 512, blocked above).
    """
    from .linalg import exact_svd

    a = _arrays.to_tensor(ohat)
    m, n = a.shape
    if rank < 1 or rank > min(m, n):
        raise RankTooLarge(f"rank {rank} outside [1, {min(m, n)}] for shape {(m, n)}")
    if not bool((a != 0).any()):
        raise DegenerateInput("cannot factorize an all-zero matrix")
    u, sigma, vt = exact_svd(a)
    k = _positive_prefix(sigma, rank)
    return TruncatedSvd(u=u[:, :k], sigma=sigma[:k], v=vt[:k, :])


def randomized_svd(ohat, rank, oversample=10, rng_seed=0):
    """Rank-r factors from a Gaussian range sketch (svdengine.py:161-196).

    The sketch omega is drawn on the host with the reference's PCG64 stream (bit-identical),
    y = ohat (ohat^T omega) and b = q^T ohat run as DMMA GEMMs, q by the device QR, and the small
    b is factorised by the device dense SVD.
    """
    from .linalg import exact_svd, qr_orthonormalize

    s = _sample_major(ohat)  # n x m (= ohat^T, row-major)
    n, m = s.shape
    width = rank + oversample
    if rank < 1 or oversample < 0 or width > min(m, n):
        raise RankTooLarge(
            f"rank+oversample {width} outside [1, {min(m, n)}] for shape {(m, n)}")
    if not bool((s != 0).any()):
        raise DegenerateInput("cannot factorize an all-zero matrix")
    ctx = _lib.context()
    dev = s.device
    omega = _arrays.rows_view(_arrays.to_tensor(
        np.random.default_rng(rng_seed).standard_normal((m, width))))
    t = torch.empty(n, width, dtype=torch.float64, device=dev)
    y = torch.empty(m, width, dtype=torch.float64, device=dev)
    ctx.call("wssr_gemm_f64", 1, n, width, m, _lib.ptr(s), _arrays.ld(s), None, _lib.ptr(omega),
             width, _lib.ptr(t), width, 1.0, 0, 1024)                       # ohat^T omega
    ctx.call("wssr_gemm_f64", 0, m, width, n, _lib.ptr(s), _arrays.ld(s), None, _lib.ptr(t),
             width, _lib.ptr(y), width, 1.0, 0, 1024)                       # ohat (ohat^T omega)
    q, _ = qr_orthonormalize(y)
    bt = torch.empty(n, width, dtype=torch.float64, device=dev)
    ctx.call("wssr_gemm_f64", 1, n, width, m, _lib.ptr(s), _arrays.ld(s), None, _lib.ptr(q),
             width, _lib.ptr(bt), width, 1.0, 0, 1024)                      # b^T = ohat^T q
    ub_t, sigma, vt_t = exact_svd(bt)                                      # b = vt_t^T S ub_t^T
    k = _positive_prefix(sigma, rank)
    if k == 0:
        raise DegenerateInput("sketch captured no positive singular values")
    u_b = vt_t.t()[:, :k].contiguous()
    uu = torch.empty(m, k, dtype=torch.float64, device=dev)
    ctx.call("wssr_gemm_f64", 1, m, k, width, _lib.ptr(q), width, None, _lib.ptr(u_b), k,
             _lib.ptr(uu), k, 1.0, 0, 1024)                                 # q @ u_b
    return TruncatedSvd(u=uu, sigma=sigma[:k], v=ub_t[:, :k].t())


def ssi_svd(ohat, rank, max_iters=3, u_init=None, residual_tol=DEFAULT_RESIDUAL_EXIT,
            *, report_final_residual=True, _careful=False):
    """Dominant singular triplets by warm-startable block subspace iteration
    (svdengine.py:88-158).

    ``ohat`` is the (m, n) parameter-major matrix of the reference.  Passing the transpose view of
    a sample-major (n, m) tensor avoids any copy.  ``report_final_residual=False`` skips the
    look-ahead after the last iteration, whose only output is SsiReport.subspace_residual
    (returned as NaN then).
    """
    s = _sample_major(ohat)
    n, m = s.shape
    if rank < 1 or rank > min(m, n):
        raise RankTooLarge(f"rank {rank} outside [1, {min(m, n)}] for shape {(m, n)}")
    warm = u_init is not None
    if warm:
        block = _arrays.to_tensor(u_init)
        if tuple(block.shape) != (m, rank):
            raise ValueError(f"u_init must have shape {(m, rank)}, got {tuple(block.shape)}")
    else:
        block = _arrays.to_tensor(
            np.random.default_rng(_COLD_START_SEED).standard_normal((m, rank)))
    block = _arrays.rows_view(block)
    dev = block.device
    u = torch.empty(m, rank, dtype=torch.float64, device=dev)
    sig = torch.empty(rank, dtype=torch.float64, device=dev)
    v = torch.empty(n, rank, dtype=torch.float64, device=dev)
    o = _ohat_struct(s)
    out = _lib.SsiOut(u=u.data_ptr(), ld_u=rank, sigma=sig.data_ptr(), v=v.data_ptr(), ld_v=rank)
    flags = _lib.WSSR_FLAG_FINAL_RESIDUAL if report_final_residual else 0
    if _careful:  # testing: every QR host-checked, the Gram-Schmidt patch path where it applies
        flags |= _lib.WSSR_FLAG_CAREFUL
    _lib.context().call("wssr_ssi_svd_f64", ctypes.byref(o), int(rank), int(max_iters),
                        _lib.ptr(block), _arrays.ld(block), float(residual_tol), flags,
                        ctypes.byref(out))
    k = int(out.k_pos)
    factors = TruncatedSvd(u=u[:, :k], sigma=sig[:k], v=v[:, :k].t())
    report = SsiReport(iterations_used=int(out.iterations),
                       subspace_residual=float(out.residual), warm_started=warm)
    return factors, report


def subspace_drift(prev, curr):
    """Change in singular values and in the left-subspace projector (svdengine.py:199-226)."""
    r = min(prev.rank, curr.rank)
    if tuple(prev.u.shape)[0] != tuple(curr.u.shape)[0]:
        raise ValueError("factor sets live in different row spaces")
    if r == 0:
        return 0.0, 0.0
    u1 = _arrays.rows_view(_arrays.to_tensor(prev.u))
    u2 = _arrays.rows_view(_arrays.to_tensor(curr.u))
    s1 = _arrays.to_tensor(prev.sigma).contiguous()
    s2 = _arrays.to_tensor(curr.sigma).contiguous()
    sd, pd = ctypes.c_double(), ctypes.c_double()
    _lib.context().call("wssr_subspace_drift_f64", int(u1.shape[0]), _lib.ptr(u1),
                        _arrays.ld(u1), _lib.ptr(s1), int(prev.rank), _lib.ptr(u2),
                        _arrays.ld(u2), _lib.ptr(s2), int(curr.rank), ctypes.byref(sd),
                        ctypes.byref(pd))
    return float(sd.value), float(pd.value)


def _is_nan(x):
    return isinstance(x, float) and math.isnan(x)
