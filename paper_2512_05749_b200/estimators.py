"""Batch estimators on the device: drop-in for vmcsr.estimators (estimators.py:1-110).

``assemble`` runs two kernels - a one-CTA energy-statistics/clipping kernel and ONE pass over
the raw log-derivative matrix that yields the column means, the centred second moments
(||o_matrix||_F^2) and the gradient - instead of the reference's centre/scale/transpose copies
(estimators.py:90-97).  The returned bundle keeps the raw sample-major matrix plus its column
means and scale; ``o_matrix`` is materialised only if a caller asks for it.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays, _lib
from .errors import DegenerateBatch


@dataclass(frozen=True)
class SampleBatch:
    """Decorrelated draws with their local energies and log-derivatives (estimators.py:16-31)."""

    configs: tuple
    local_energies: object   # (batch,)
    theta_logderivs: object  # (batch, n_params), sample-major

    def __post_init__(self):
        n = len(self.configs)
        e_shape = tuple(self.local_energies.shape)
        d_shape = tuple(self.theta_logderivs.shape)
        if e_shape != (n,) or d_shape[0] != n:
            raise ValueError("batch fields disagree on the sample count")

    @property
    def size(self):
        return len(self.configs)


@dataclass(frozen=True, eq=False, repr=False)
class EstimatorBundle:
    """Everything one optimizer step consumes (estimators.py:34-50): a frozen dataclass with the
    reference's fields (``dataclasses.fields/replace/asdict`` work).

    Constructed either by ``assemble`` (then it holds the raw sample-major derivative block,
    its column means and scale 1/sqrt(N); ``o_matrix`` is the lazy view ((derivs - mu) *
    scale).T, materialised on first access, and ``loss``/``raw_loss`` of a single-rank assemble
    resolve when first read) or directly with an explicit (n_params, batch) ``o_matrix`` as in
    the reference's test helpers (test_optimizers.py:27-34).
    """

    loss: float                # mean clipped energy
    raw_loss: float            # mean energy before clipping
    o_matrix: object           # (n_params, batch), centered, 1/sqrt(batch)
    l_vector: object           # (batch,), clipped residuals, 1/sqrt(batch)
    gradient: object           # (n_params,) = 2 * O @ L

    @classmethod
    def _assembled(cls, loss, raw_loss, samples, mu, scale, fro2, l_vector, gradient, n_global,
                   scale_table=None, deferred=None):
        """deferred: (event, pinned host [loss, raw_loss, e_mean, e_std, fro2], device fro2) -
        the scalars of an assemble that returned without waiting for the device; they resolve on
        first access (the optimizer step takes fro2 from the device copy and never waits)."""
        self = cls.__new__(cls)
        self._init(loss, raw_loss, samples, mu, scale, fro2, _arrays.device_array(l_vector),
                   _arrays.device_array(gradient), True, n_global)
        object.__setattr__(self, "_scale_table", scale_table)
        object.__setattr__(self, "_deferred", deferred)
        return self

    def _init(self, loss, raw_loss, samples, mu, scale, fro2, l_vector, gradient, exact,
              n_global):
        set_ = object.__setattr__
        set_(self, "_loss", loss)
        set_(self, "_raw_loss", raw_loss)
        set_(self, "_l_vector", l_vector)
        set_(self, "_gradient", gradient)
        set_(self, "_samples", samples)
        set_(self, "_mu", mu)
        set_(self, "_scale", scale)
        set_(self, "_fro2_val", fro2)
        set_(self, "_deferred", None)
        set_(self, "_gradient_exact", exact)
        set_(self, "_o_cache", None)
        set_(self, "_n_global", n_global)
        set_(self, "_scale_table", None)

    def _resolve(self):
        d = self._deferred
        if d is not None:
            event, host, _ = d
            event.synchronize()
            vals = host.tolist()
            set_ = object.__setattr__
            set_(self, "_loss", float(vals[0]))
            set_(self, "_raw_loss", float(vals[1]))
            set_(self, "_fro2_val", float(vals[4]))
            set_(self, "_deferred", None)

    @property
    def _fro2(self) -> float:
        """||o_matrix||_F^2 (host value; waits for a deferred assemble)"""
        self._resolve()
        return self._fro2_val

    def _fro2_args(self):
        """(host fro2 or -1, device fro2 or None) for the engine, without waiting"""
        d = self._deferred
        if d is not None:
            if d[0].query():
                self._resolve()
            else:
                return -1.0, d[2]
        return self._fro2_val, None

    def __repr__(self):
        # the lazy o_matrix stays unmaterialised (at BASELINE sizes it is the whole batch)
        return (f"EstimatorBundle(loss={self.loss!r}, raw_loss={self.raw_loss!r}, "
                f"o_matrix=<({self.n_params}, {self.batch_size}) lazy>, "
                f"l_vector=<({self.batch_size},)>, gradient=<({self.n_params},)>)")

    @property
    def n_params(self):
        return int(self._samples.shape[1])

    @property
    def batch_size(self):
        return int(self._samples.shape[0])


def _bundle_init(self, loss, raw_loss, o_matrix, l_vector, gradient):
    """EstimatorBundle(loss, raw_loss, o_matrix, l_vector, gradient) (the reference constructor)"""
    o = _arrays.to_tensor(o_matrix)
    if o.dim() == 1:
        o = o[:, None]
    samples = o.t()
    if not (samples.stride(1) == 1 and samples.stride(0) >= samples.shape[1]):
        samples = samples.contiguous()
    self._init(float(loss), float(raw_loss), samples, None, 1.0, -1.0,
               _arrays.device_array(_arrays.to_tensor(l_vector)),
               _arrays.device_array(_arrays.to_tensor(gradient)), False, samples.shape[0])


def _get_loss(self):
    """mean of the clipped local energies (estimators.py:92)"""
    self._resolve()
    return self._loss


def _get_raw_loss(self):
    """mean of the raw local energies (estimators.py:89)"""
    self._resolve()
    return self._raw_loss


def _get_o_matrix(self):
    """(n_params, batch) centred and scaled matrix (materialised on first access)"""
    if self._o_cache is None:
        x = self._samples.to(torch.float64)
        if self._mu is None and self._scale == 1.0:
            o = x.t()
        else:
            o = ((x - self._mu[None, :]) * self._scale).t()
        object.__setattr__(self, "_o_cache", _arrays.device_array(o))
    return self._o_cache


def _readonly(name):
    def _set(self, value):
        raise AttributeError(f"EstimatorBundle.{name} is read-only")
    return _set


# the dataclass fields are served lazily (deferred scalars, lazy o_matrix); the generated
# __init__ is replaced by the reference constructor above, so fields/replace/asdict all work
EstimatorBundle.__init__ = _bundle_init
EstimatorBundle.loss = property(_get_loss, _readonly("loss"))
EstimatorBundle.raw_loss = property(_get_raw_loss, _readonly("raw_loss"))
EstimatorBundle.o_matrix = property(_get_o_matrix, _readonly("o_matrix"))
EstimatorBundle.l_vector = property(lambda self: self._l_vector, _readonly("l_vector"))
EstimatorBundle.gradient = property(lambda self: self._gradient, _readonly("gradient"))


def clip_local_energies(energies, n_std=5.0):
    """Clamp outliers to mean +- n_std * population std (estimators.py:53-71), on the device."""
    e = _arrays.to_tensor(energies).reshape(-1).contiguous()
    if e.numel() < 2:
        raise DegenerateBatch("clipping window needs at least two samples")
    if not math.isfinite(n_std):
        return e.clone()
    if n_std < 0:
        raise ValueError("clipping width must be nonnegative")
    n = e.numel()
    bundle = assemble(_Batch(e, torch.zeros(n, 1, dtype=torch.float64, device=e.device)),
                      clip_n_std=n_std)
    # l_raw = clip(E) - loss ;  clip(E) = l_vector * sqrt(N) + loss
    return bundle.l_vector * math.sqrt(n) + bundle.loss


class _Batch:
    """Minimal batch duck type used internally."""

    def __init__(self, energies, derivs):
        self.local_energies = energies
        self.theta_logderivs = derivs

    @property
    def size(self):
        return int(self.local_energies.shape[0])


def assemble(batch, clip_n_std=5.0):
    """Build the centred estimator bundle from one sample batch (estimators.py:74-100).

    Raises:
      DegenerateBatch: fewer than two samples (nothing to center).
    """
    if batch.size < 2:
        raise DegenerateBatch("need at least two samples to center the batch")
    ctx = _lib.context()
    derivs = _arrays.rows_view(_arrays.to_tensor_f64_or_f32(batch.theta_logderivs))
    energies = _arrays.to_tensor(batch.local_energies).reshape(-1).contiguous()
    n, p = derivs.shape
    dev = derivs.device
    mu = torch.empty(p, dtype=torch.float64, device=dev)
    lvec = torch.empty(n, dtype=torch.float64, device=dev)
    grad = torch.empty(p, dtype=torch.float64, device=dev)
    # per-parameter scales of the int8 tensor-core O-passes, from the same column pass
    table = torch.empty(_lib.scale_table_len(p), dtype=torch.float64, device=dev)
    # single rank: the host scalars arrive asynchronously (no wait on the column pass, so the
    # optimizer step that follows is enqueued while the device is still busy)
    defer = int(getattr(ctx, "world", 1)) == 1
    host = ctx.pinned_slot(5) if defer else None
    fro2_dev = torch.empty(1, dtype=torch.float64, device=dev) if defer else None
    out = _lib.AssembleOut(mu=mu.data_ptr(), l_vector=lvec.data_ptr(), gradient=grad.data_ptr(),
                           scale_table=table.data_ptr(),
                           deferred=host.data_ptr() if defer else None,
                           fro2_dev=fro2_dev.data_ptr() if defer else None)
    entry = "wssr_assemble_f32" if derivs.dtype == torch.float32 else "wssr_assemble_f64"
    if derivs.dtype == torch.float32 and (derivs.stride(0) % 4 or derivs.data_ptr() % 16):
        derivs = _pad_rows_f32(derivs)
    ctx.call(entry, _lib.ptr(derivs), n, p, _arrays.ld(derivs),
             _lib.ptr(energies), float(clip_n_std), ctypes.byref(out))
    scale = 1.0 / np.sqrt(out.n_global)
    deferred = None
    if defer:
        event = torch.cuda.Event()
        event.record(torch.cuda.current_stream(dev))
        deferred = (event, host, fro2_dev)
    return EstimatorBundle._assembled(out.loss, out.raw_loss, derivs, mu, scale, out.fro2, lvec,
                                      grad, int(out.n_global), table, deferred)


def _pad_rows_f32(x):
    """float32 rows padded to a multiple of 4 elements (16-byte TMA pitch)."""
    n, p = x.shape
    ldp = (p + 3) // 4 * 4
    buf = torch.zeros(n, ldp, dtype=torch.float32, device=x.device)
    buf[:, :p] = x
    return buf[:, :p]


def s_matrix(bundle):
    """Parameter-space covariance O @ O^T (estimators.py:103-105); small-P diagnostics only."""
    o = bundle.o_matrix
    return o @ o.t()


def t_matrix(bundle):
    """Sample-space companion O^T @ O (estimators.py:108-110); small-N diagnostics only."""
    o = bundle.o_matrix
    return o.t() @ o
