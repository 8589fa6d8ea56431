"""Warm-started low-rank preconditioned update on the device: drop-in for the WSSR part of
vmcsr.optimizers (optimizers.py:188-401).

``wssr_step`` keeps the reference signature and returns (theta', state', WssrDiagnostics) - theta'
as numpy when theta came in as a host array (the reference runner's convention), else as a CUDA
tensor; the
whole step after the host-side warm-start preparation is ONE call into libwssr
(wssr_step_f64): SSI factorisation, rank cut/growth, gbar, the fused preconditioner apply,
drift telemetry and the state refresh.  State arrays are float64 CUDA tensors; ``obar`` is kept
parameter-contiguous (a (P, r) view of an (r, P) buffer) because the next step streams it as
the history block of Ohat.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _arrays, _lib
from .linalg import qr_orthonormalize
from .svdengine import SsiReport

DEFAULT_LEARNING_RATE = 0.015      # optimizers.py:28
DEFAULT_RATE_DECAY = 1000.0
DEFAULT_TIKHONOV_EPS = 1e-3
DEFAULT_MOMENTUM = 0.99
DEFAULT_AVERAGING_WEIGHT = 0.95    # optimizers.py:32
DEFAULT_SIGMA_FLOOR = 1e-3
DEFAULT_RANK_CUTOFF = 1e-6
DEFAULT_RANK_GROWTH = 0.1
DEFAULT_RANK_INIT = 400
DEFAULT_SSI_MAX_ITERS = 3          # optimizers.py:37
SVD_BACKENDS = ("ssi", "randomized", "exact")


def _shape(x):
    return tuple(x.shape)


@dataclass(frozen=True)
class WssrState:
    """Carry-over for the warm-started low-rank scheme (optimizers.py:188-247)."""

    obar: object
    lbar: object
    u_prev: object
    r_max: int
    delta: float = DEFAULT_AVERAGING_WEIGHT
    sigma_floor: float = DEFAULT_SIGMA_FLOOR
    sigma_floor_relative: bool = False
    r_reg: float = DEFAULT_RANK_CUTOFF
    eps_grow: float = DEFAULT_RANK_GROWTH
    step: int = 0

    def __post_init__(self):
        if len(_shape(self.obar)) != 2 or len(_shape(self.u_prev)) != 2 or len(_shape(self.lbar)) != 1:
            raise ValueError("malformed history shapes")
        if _shape(self.obar)[1] != _shape(self.lbar)[0]:
            raise ValueError("history rank mismatch between obar and lbar")
        if self.r_max < 1:
            raise ValueError("r_max must be at least 1")
        if not 0.0 <= self.delta < 1.0:
            raise ValueError("averaging weight must lie in [0, 1)")
        if self.sigma_floor <= 0.0:
            raise ValueError("sigma_floor must be positive")
        if not 0.0 < self.r_reg < 1.0:
            raise ValueError("rank cutoff must lie in (0, 1)")
        if self.eps_grow < 0.0:
            raise ValueError("rank growth factor must be nonnegative")

    @property
    def history_rank(self):
        return _shape(self.obar)[1]

    @classmethod
    def initial(cls, n_params, rank_init=DEFAULT_RANK_INIT, delta=DEFAULT_AVERAGING_WEIGHT,
                sigma_floor=DEFAULT_SIGMA_FLOOR, sigma_floor_relative=False,
                r_reg=DEFAULT_RANK_CUTOFF, eps_grow=DEFAULT_RANK_GROWTH):
        dev = _arrays.default_device()
        z = torch.zeros(0, n_params, dtype=torch.float64, device=dev)
        return cls(obar=z.t(), lbar=torch.zeros(0, dtype=torch.float64, device=dev),
                   u_prev=torch.zeros(n_params, 0, dtype=torch.float64, device=dev),
                   r_max=int(rank_init), delta=delta, sigma_floor=sigma_floor,
                   sigma_floor_relative=sigma_floor_relative, r_reg=r_reg, eps_grow=eps_grow)


@dataclass(frozen=True)
class WssrDiagnostics:
    """Per-step telemetry mirrored into the trace file (optimizers.py:250-258): a frozen
    dataclass with the reference's fields.

    The two drift values of a single-rank step are computed on a side stream after the step's
    own work; they resolve (waiting for that stream) on first access, so a caller that never
    reads them never waits.
    """

    ssi: SsiReport
    effective_rank: int
    r_max: int
    sigma_drift: float
    projector_drift: float

    @classmethod
    def _deferred(cls, ssi, effective_rank, r_max, event, host):
        self = cls(ssi, effective_rank, r_max, float("nan"), float("nan"))
        object.__setattr__(self, "_pending", (event, host))
        return self

    def _resolve(self):
        pending = self.__dict__.get("_pending")
        if pending is not None:
            event, host = pending
            event.synchronize()
            sd, pd = (float(x) for x in host.tolist())
            self.__dict__["_sigma_drift"] = sd
            self.__dict__["_projector_drift"] = pd
            self.__dict__["_pending"] = None
        return self.__dict__["_sigma_drift"], self.__dict__["_projector_drift"]


def _drift_setter(name):
    def _set(self, value):
        if "_" + name in self.__dict__:
            raise AttributeError(f"WssrDiagnostics.{name} is read-only")
        self.__dict__["_" + name] = float(value)  # the dataclass __init__ (object.__setattr__)
    return _set


WssrDiagnostics.sigma_drift = property(lambda self: self._resolve()[0],
                                       _drift_setter("sigma_drift"))
WssrDiagnostics.projector_drift = property(lambda self: self._resolve()[1],
                                           _drift_setter("projector_drift"))


def _per_step_seed(rng_seed, step):
    """optimizers.py:273-274."""
    return int(np.random.SeedSequence((int(rng_seed), int(step))).generate_state(1)[0])


def _prepare_warm_start(u_prev, requested, n_rows, seed):
    """Previous left vectors widened (or cut) to the requested block size (optimizers.py:277-289).

    The widening draws its Gaussian columns on the host with the reference's PCG64 stream so the
    warm start is bit-identical; the QR runs on the device.
    """
    u_prev = _arrays.to_tensor(u_prev)
    if u_prev.shape[1] >= requested:
        return u_prev[:, :requested]
    extra = np.random.default_rng(seed).standard_normal((n_rows, requested - u_prev.shape[1]))
    block = torch.cat([u_prev, _arrays.to_tensor(extra)], dim=1)
    q, _ = qr_orthonormalize(block)
    return q


# Dense first step / 'exact' backend without forming Ohat (engine.cu implicit_svd): taken when
# Ohat would not fit beside the sample block, for float32 samples, and under row sharding (each
# rank would otherwise hold the whole P x (r + N) matrix).  WSSR_DENSE_STEP=implicit|materialize
# forces either path.
IMPLICIT_MAX_ITERS = 100
IMPLICIT_TOL = 1e-12       # ||Ohat v_i - s_i u_i|| / s_i of every kept triplet (or stagnation)
_IMPLICIT_SEED = 0x5EED
# telemetry of the last implicit solve: power iterations and max_i ||Ohat v_i - s_i u_i|| / s_i
last_implicit_svd: dict = {}


def _implicit_dense_step(ctx, samples, m, n_cols):
    mode = os.environ.get("WSSR_DENSE_STEP", "auto")
    if mode == "implicit":
        return True
    if mode == "materialize":
        return False
    if int(getattr(ctx, "world", 1)) > 1 or samples.dtype == torch.float32:
        return True
    # Ohat plus the dense SVD's working copies
    free, _ = torch.cuda.mem_get_info(samples.device)
    return 3 * 8 * m * n_cols > free


def wssr_step(theta, bundle, eta, state, svd_backend="ssi",
              ssi_max_iters=DEFAULT_SSI_MAX_ITERS, ssi_residual_tol=1e-10, rng_seed=0,
              *, report_final_residual=True, return_update=False):
    """One step of the warm-started low-rank preconditioned descent (optimizers.py:292-391).

        theta' = theta - eta * (U sigma^-2 U^T + floor^-1 (I - U U^T)) gbar

    Returns:
      (theta', state', WssrDiagnostics)  [+ the update vector when return_update=True]
    """
    if svd_backend not in SVD_BACKENDS:
        raise ValueError(f"svd_backend must be one of {SVD_BACKENDS}, got {svd_backend!r}")
    dense = state.step == 0 or svd_backend in ("exact", "randomized")
    ctx = _lib.context()
    host_theta = _arrays.is_host_array(theta)
    theta = _arrays.to_tensor(theta).reshape(-1).contiguous()
    samples = bundle._samples
    m = bundle.n_params
    n = bundle.batch_size
    obar = _arrays.to_tensor(state.obar)
    r = obar.shape[1]
    hist = obar.t()
    if r > 0 and not (hist.stride(1) == 1 and hist.stride(0) >= m):
        hist = hist.contiguous()
    lbar = _arrays.to_tensor(state.lbar).contiguous()
    n_global = int(getattr(bundle, "_n_global", n))
    requested = min(state.r_max, m, r + n_global)
    if dense:
        u_init = None
    else:
        u_init = _prepare_warm_start(state.u_prev, requested, m,
                                     _per_step_seed(rng_seed, state.step))
        u_init = _arrays.rows_view(u_init)
    u_prev = _arrays.to_tensor(state.u_prev)
    if u_prev.shape[1] > 0:
        u_prev = _arrays.rows_view(u_prev)
    dev = theta.device
    k = requested
    theta_next = torch.empty(m, dtype=torch.float64, device=dev)
    update = torch.empty(m, dtype=torch.float64, device=dev) if return_update else None
    u_next = torch.empty(m, k, dtype=torch.float64, device=dev)
    obar_t = torch.empty(k, m, dtype=torch.float64, device=dev)
    lbar_next = torch.empty(k, dtype=torch.float64, device=dev)
    sigma = torch.empty(k, dtype=torch.float64, device=dev)

    from .svdengine import _ohat_struct
    fro2_host, fro2_dev = bundle._fro2_args()
    if fro2_dev is not None:  # assemble's outputs may still be in flight on another stream
        torch.cuda.current_stream(dev).wait_event(bundle._deferred[0])
    o = _ohat_struct(samples, bundle._mu, bundle._scale, fro2_host, hist, 1.0,
                     bundle._scale_table, fro2_dev)
    lvec = bundle.l_vector.contiguous()
    grad = bundle.gradient if bundle._gradient_exact else None
    ext = None
    if dense and svd_backend != "randomized" and _implicit_dense_step(
            ctx, samples, m, r + n_global):
        # optimizers.py:327-338 without forming Ohat: exact_truncated_svd of the implicit
        # operator on the O-pass kernels (svdengine.py:75-85; engine.cu implicit_svd), rows
        # sharded like the SSI; every rank gets U and sigma, and its own rows of V
        world = int(getattr(ctx, "world", 1))
        if world > 1:
            counts = torch.zeros(world, dtype=torch.float64, device=dev)
            counts[ctx.rank] = n
            ctx.call("wssr_allreduce_f64", _lib.ptr(counts), world)
            counts = [int(c) for c in counts.tolist()]
            c0 = 0 if ctx.rank == 0 else r + sum(counts[:ctx.rank])
            n_local = (r if ctx.rank == 0 else 0) + n
            o_imp = _ohat_struct(samples, bundle._mu, bundle._scale, bundle._fro2,
                                 hist if ctx.rank == 0 else hist[:0], 1.0, bundle._scale_table)
            n_cols = r + sum(counts)
        else:
            c0, n_local, o_imp, n_cols = 0, r + n, o, r + n
        fu = torch.empty(m, k, dtype=torch.float64, device=dev)
        fs = torch.empty(k, dtype=torch.float64, device=dev)
        fv = torch.empty(max(n_local, 1), k, dtype=torch.float64, device=dev)
        k_pos, iters, resid = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        ctx.call("wssr_implicit_svd_f64", ctypes.byref(o_imp), float(state.delta), k, n_cols, c0,
                 ctypes.c_uint64(_IMPLICIT_SEED + int(state.step)), IMPLICIT_MAX_ITERS,
                 IMPLICIT_TOL, _lib.ptr(fu), k, _lib.ptr(fs), _lib.ptr(fv), k,
                 ctypes.byref(k_pos), ctypes.byref(iters), ctypes.byref(resid))
        ext = (fu, fs, fv, int(k_pos.value))
        # the reference reports iterations_used=0 / residual 0.0 for the dense step
        # (optimizers.py:328-331); the implicit solve's own certificate is kept here
        last_implicit_svd.update(iterations=int(iters.value), residual=float(resid.value),
                                 block=min(max(2 * k, k + 16), m, n_cols))
    elif dense:
        # optimizers.py:327-338: dense first step / 'exact' backend, or the randomized sketch
        from .svdengine import exact_truncated_svd, randomized_svd
        world = int(getattr(ctx, "world", 1))
        if world > 1:
            # row-sharded: every rank writes its own columns of the global Ohat
            # [hist | samples of rank 0 | rank 1 | ...] and one sum gathers them (disjoint, so
            # the sum is exact); every rank then factorises the same matrix.
            counts = torch.zeros(world, dtype=torch.float64, device=dev)
            counts[ctx.rank] = n
            ctx.call("wssr_allreduce_f64", _lib.ptr(counts), world)
            counts = [int(c) for c in counts.tolist()]
            c0 = 0 if ctx.rank == 0 else r + sum(counts[:ctx.rank])
            n_local = (r if ctx.rank == 0 else 0) + n
            ohat = torch.zeros(m, r + sum(counts), dtype=torch.float64, device=dev)
            o_local = _ohat_struct(samples, bundle._mu, bundle._scale, bundle._fro2,
                                   hist if ctx.rank == 0 else hist[:0], 1.0)
            ctx.call("wssr_materialize_ohat_f64", ctypes.byref(o_local), float(state.delta),
                     _lib._vp(ohat.data_ptr() + 8 * c0), ohat.shape[1])
            ctx.call("wssr_allreduce_f64", _lib.ptr(ohat), ohat.numel())
        else:
            c0, n_local = 0, r + n
            ohat = torch.empty(m, r + n, dtype=torch.float64, device=dev)
            ctx.call("wssr_materialize_ohat_f64", ctypes.byref(o), float(state.delta),
                     _lib.ptr(ohat), r + n)
        if state.step == 0 or svd_backend == "exact":
            factors = exact_truncated_svd(ohat, requested)
        else:
            room = min(ohat.shape) - requested
            factors = randomized_svd(ohat, requested, oversample=min(10, max(0, room)),
                                     rng_seed=_per_step_seed(rng_seed, state.step))
        del ohat
        fu = _arrays.rows_view(factors.u)
        fs = factors.sigma.contiguous()
        fv = factors.v[:, c0:c0 + n_local].t().contiguous()
        ext = (fu, fs, fv, int(factors.rank))
    sin = _lib.StepIn(
        ohat=ctypes.pointer(o), lbar=lbar.data_ptr() if r > 0 else None,
        l_vector=lvec.data_ptr(), gradient=grad.data_ptr() if grad is not None else None,
        theta=theta.data_ptr(), eta=float(eta),
        u_init=u_init.data_ptr() if u_init is not None else None,
        ld_init=_arrays.ld(u_init) if u_init is not None else 1, requested=k,
        u_prev=u_prev.data_ptr() if u_prev.shape[1] > 0 else None,
        ld_prev=_arrays.ld(u_prev) if u_prev.shape[1] > 0 else 1, r_prev=int(u_prev.shape[1]),
        delta=float(state.delta), sigma_floor=float(state.sigma_floor), r_reg=float(state.r_reg),
        eps_grow=float(state.eps_grow), sigma_floor_relative=int(bool(state.sigma_floor_relative)),
        r_max=int(state.r_max), max_iters=int(ssi_max_iters),
        residual_tol=float(ssi_residual_tol),
        flags=_lib.WSSR_FLAG_FINAL_RESIDUAL if report_final_residual else 0,
    )
    if ext is not None:
        sin.ext_u, sin.ext_ld_u = ext[0].data_ptr(), _arrays.ld(ext[0])
        sin.ext_sigma, sin.ext_v = ext[1].data_ptr(), ext[2].data_ptr()
        sin.ext_ld_v, sin.ext_k_pos = _arrays.ld(ext[2]) if ext[2].shape[0] > 1 else ext[3], ext[3]
    sout = _lib.StepOut(
        theta_next=theta_next.data_ptr(), update=update.data_ptr() if update is not None else None,
        u_next=u_next.data_ptr(), ld_u=k, obar_next_t=obar_t.data_ptr(), ld_obar=m,
        lbar_next=lbar_next.data_ptr(), sigma=sigma.data_ptr(),
    )
    aux = ctx.aux_stream() if int(getattr(ctx, "world", 1)) == 1 and hasattr(ctx, "aux_stream") \
        else None
    drift_host = ctx.pinned_slot(2) if hasattr(ctx, "pinned_slot") else \
        torch.empty(2, dtype=torch.float64, pin_memory=True)
    sout.drift_host = drift_host.data_ptr()
    ctx.call("wssr_step_f64", ctypes.byref(sin), ctypes.byref(sout))
    bundle._fro2_args()  # resolves the bundle's deferred scalars if they have landed (no wait)
    r_eff = int(sout.r_eff)
    deferred = aux is not None and math.isnan(sout.projector_drift)
    if deferred:
        # the drift kernels still read these on the side stream
        event = torch.cuda.Event()
        event.record(aux)
        for t in (u_prev, hist, u_next, sigma):
            if t is not None and t.numel() > 0 and t.is_cuda:
                t.record_stream(aux)
    state_next = replace(
        state,
        obar=_arrays.device_array(obar_t[:r_eff].t()),
        lbar=_arrays.device_array(lbar_next[:r_eff]),
        u_prev=_arrays.device_array(u_next[:, :r_eff]),
        r_max=int(sout.next_r_max),
        step=state.step + 1,
    )
    report = SsiReport(iterations_used=int(sout.iterations),
                       subspace_residual=float(sout.residual), warm_started=not dense)
    if deferred:
        diag = WssrDiagnostics._deferred(report, r_eff, int(state.r_max), event, drift_host)
    else:
        diag = WssrDiagnostics(ssi=report, effective_rank=r_eff, r_max=int(state.r_max),
                               sigma_drift=float(sout.sigma_drift),
                               projector_drift=float(sout.projector_drift))
    if host_theta:
        # the reference runner's convention (runner.py:299, 314): numpy theta in, numpy theta'
        # out (one P-double copy); the state stays on the device (numpy-readable DeviceArrays)
        theta_next = theta_next.cpu().numpy()
    if return_update:
        return theta_next, state_next, diag, update
    return theta_next, state_next, diag


def rssr_step(theta, bundle, eta, state, ssi_max_iters=DEFAULT_SSI_MAX_ITERS, rng_seed=0):
    """Low-rank step with a fresh random sketch each step (optimizers.py:394-401)."""
    return wssr_step(theta, bundle, eta, state, svd_backend="randomized",
                     ssi_max_iters=ssi_max_iters, rng_seed=rng_seed)


def sigma_of(state) -> torch.Tensor:
    """Singular values carried by a state: column norms of obar (optimizers.py:370)."""
    return torch.linalg.vector_norm(_arrays.to_tensor(state.obar), dim=0)


__all__ = [
    "WssrState", "WssrDiagnostics", "wssr_step", "rssr_step", "_prepare_warm_start",
    "_per_step_seed", "SVD_BACKENDS", "sigma_of", "math",
]
