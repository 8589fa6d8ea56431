"""Device producer of O for the pooled-feature determinant ansatz.

`grad_theta_batch(wavefunction, positions)` is AceWavefunction.grad_theta_batch
(wavefunction.py:307-321) on the device: d log|psi| / d theta for a batch of walkers, written
straight into a (W, n_params) float64 CUDA tensor that `estimators.SampleBatch` takes as
`theta_logderivs` - a VMC loop then moves the walker positions (W x N x 3) to the GPU instead of
O (W x n_params).  The feature pipeline (orbital values, pooled tuple products, the orbital
matrix, its inverse and the contraction) runs in one libwssr kernel per call (csrc/producer.cu).

`AceSpec.from_wavefunction(wf)` reads a reference AceWavefunction by duck typing (basis
orbitals, system geometry and spins, feature index, theta) - no import of the reference.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _arrays, _lib

_M_TO_AXIS = {-1: 1, 0: 2, 1: 0}   # real solid harmonics m = -1, 0, 1 -> y, z, x (wavefunction.py:25)
_GATES = {"up": 0, "down": 1, "either": 2}


class AceSpec:
    """Device tables of one ansatz (orbitals, feature index, coefficients)."""

    def __init__(self, nuclei, spins, orbitals, feature_index, theta, device=None):
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        orbs = list(orbitals)
        n_el = len(spins)
        n_feat = len(feature_index)
        max_tail = max((len(tail) for _, tail in feature_index), default=0)
        tails = np.full((n_feat, max(max_tail, 1)), -1, dtype=np.int32)
        for t, (_, tail) in enumerate(feature_index):
            tails[t, :len(tail)] = tail

        # the producer indexes its tables with these values on the device: check them here
        n_orb, n_nuc = len(orbs), int(np.asarray(nuclei, dtype=np.float64).reshape(-1, 3).shape[0])
        heads = np.asarray([h for h, _ in feature_index], dtype=np.int64)
        if heads.size and (heads.min() < 0 or heads.max() >= n_orb):
            raise ValueError("feature heads must index the orbital list")
        if tails.size and (tails.min() < -1 or tails.max() >= n_orb):
            raise ValueError("feature tails must index the orbital list")
        if any(not 0 <= o.center < n_nuc for o in orbs):
            raise ValueError("orbital centres must index the nuclei")
        if any(o.n < 0 or (o.ell == 1 and o.m not in _M_TO_AXIS) for o in orbs):
            raise ValueError("unsupported orbital (n < 0 or p-type m outside -1..1)")
        if any(o.spin not in _GATES for o in orbs):
            raise ValueError("orbital spin gate must be 'up', 'down' or 'either'")

        def i32(a):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev)

        def f64(a):
            return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)

        self.device = dev
        self.n_electrons, self.n_features = n_el, n_feat
        self.n_params = n_el * n_feat
        self._t = dict(
            nuclei=f64(np.asarray(nuclei, dtype=np.float64).reshape(-1, 3)),
            spins=i32([0 if int(s) == 0 else 1 for s in spins]),
            orb_center=i32([o.center for o in orbs]),
            orb_n=i32([o.n for o in orbs]),
            orb_axis=i32([_M_TO_AXIS[o.m] if o.ell == 1 else -1 for o in orbs]),
            orb_gate=i32([_GATES[o.spin] for o in orbs]),
            orb_zeta=f64([o.zeta for o in orbs]),
            heads=i32([h for h, _ in feature_index]),
            tails=i32(tails),
        )
        self.set_theta(theta)
        self._spec = _lib.AceSpec(
            n_electrons=n_el, n_orbitals=len(orbs), n_features=n_feat,
            n_nuclei=int(self._t["nuclei"].shape[0]), max_tail=max_tail,
            **{k: v.data_ptr() for k, v in self._t.items()}, coef=self._coef.data_ptr())

    @classmethod
    def from_wavefunction(cls, wf, device=None):
        return cls(wf.system.nuclear_positions, wf.system.spins, wf.basis.orbitals,
                   wf.feature_index, wf.theta, device)

    def set_theta(self, theta):
        t = _arrays.to_tensor(theta, dev=self.device).reshape(self.n_electrons, self.n_features)
        self._coef = t.contiguous()
        if hasattr(self, "_spec"):
            self._spec.coef = self._coef.data_ptr()


def grad_theta_batch(spec, positions, out=None):
    """(W, n_params) float64 CUDA tensor of d log|psi| / d theta (wavefunction.py:307-321).

    `spec` is an AceSpec or a reference AceWavefunction (tables built per call then).
    `out` (not in the reference): a preallocated (W, n_params) float64 CUDA tensor to write
    into, for runs whose sample block fills the GPU and is reused from step to step.
    Raises NodeProximity when a walker's determinant vanishes or underflows, as the reference.
    """
    if not isinstance(spec, AceSpec):
        spec = AceSpec.from_wavefunction(spec)
    x = _arrays.to_tensor(positions).to(spec.device).contiguous()
    if x.dim() != 3 or x.shape[1] != spec.n_electrons or x.shape[2] != 3:
        raise ValueError(f"positions must be (W, {spec.n_electrons}, 3), got {tuple(x.shape)}")
    w = int(x.shape[0])
    if out is None:
        out = torch.empty(w, spec.n_params, dtype=torch.float64, device=spec.device)
    elif (tuple(out.shape) != (w, spec.n_params) or out.dtype != torch.float64
          or out.device != x.device or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous ({w}, {spec.n_params}) float64 tensor on "
                         f"{x.device}")
    _lib.context().call("wssr_grad_theta_f64", ctypes.byref(spec._spec), _lib.ptr(x), w,
                        _lib.ptr(out), spec.n_params)
    return out


__all__ = ["AceSpec", "grad_theta_batch"]
