"""CPU oracle for the device producer of O (TEST INFRASTRUCTURE ONLY: imported by tests/ as the
checker, never by the product path).

A numpy restatement of the reference's AceWavefunction.grad_theta_batch
(pkg/src/vmcsr/wavefunction.py:307-321) on the flat tables the device producer takes
(csrc/producer.cu, include/wssr.h wssr_ace_spec):

* orbital values   (wavefunction.py:143-178)  phi[w,i,o] = exp(-zeta_o r) r^n_o [axis] gate_o(s_i)
* pooled features  (wavefunction.py:261-272)  F[w,i,t] = phi[w,i,head_t] prod_p pooled[w,i,p]
* orbital matrix   (wavefunction.py:280-282)  M[w,i,k] = sum_t F[w,i,t] theta[k,t]
* node check       (wavefunction.py:316-318)  sign 0 or log|det| < -700 -> NodeProximity
* derivative       (wavefunction.py:319-321)  O[w, k T + t] = sum_i inv(M)[w,k,i] F[w,i,t]

Pinned by tests/test_oracle_wavefunction.py against tests/golden/ace_grad.npz, which the
reference itself wrote (tests/golden/make_wavefunction_golden.py).
"""

from __future__ import annotations

import numpy as np

LOG_ABS_UNDERFLOW = -700.0          # vmcsr/system.py:16
SPIN_UP = 0                         # vmcsr/system.py:18
_M_TO_AXIS = {-1: 1, 0: 2, 1: 0}    # wavefunction.py:25 (real solid harmonics -> y, z, x)


class NodeProximity(RuntimeError):
    """A walker sits on (or numerically at) a node of the determinant."""


def orbital_values(nuclei, spins, orb, zeta, positions):
    """(W, N, n_orb); orb rows are (center, n, ell, m, gate) with gate 0 up / 1 down / 2 either."""
    pos = np.asarray(positions, dtype=np.float64)
    w, n, _ = pos.shape
    up = (np.asarray(spins) == SPIN_UP).astype(np.float64)
    gates = {0: up, 1: 1.0 - up, 2: np.ones(n)}
    out = np.empty((w, n, len(orb)))
    for o, ((c, nn, ell, m, gate), z) in enumerate(zip(orb, zeta)):
        d = pos - np.asarray(nuclei, dtype=np.float64)[int(c)][None, None, :]
        r = np.sqrt(np.sum(d * d, axis=-1))
        v = np.exp(-float(z) * r)
        if nn:
            v = v * r ** int(nn)
        if int(ell) == 1:
            v = v * d[..., _M_TO_AXIS[int(m)]]
        out[:, :, o] = v * gates[int(gate)][None, :]
    return out


def pooled_features(phi, heads, tails):
    """(W, N, T); tails is (T, max_tail) padded with -1."""
    pooled = phi.sum(axis=1, keepdims=True) - phi
    feats = phi[:, :, np.asarray(heads)].copy()
    tails = np.asarray(tails)
    for t in range(tails.shape[0]):
        for p in tails[t]:
            if p < 0:
                break
            feats[:, :, t] *= pooled[:, :, int(p)]
    return feats


def grad_theta(nuclei, spins, orb, zeta, heads, tails, theta, positions):
    """(W, N T) float64, d log|psi| / d theta of every walker."""
    pos = np.asarray(positions, dtype=np.float64)
    n = pos.shape[1]
    feats = pooled_features(orbital_values(nuclei, spins, orb, zeta, pos), heads, tails)
    coef = np.asarray(theta, dtype=np.float64).reshape(n, -1)
    m = np.einsum("wit,kt->wik", feats, coef)
    sign, logdet = np.linalg.slogdet(m)
    if np.any(sign == 0.0) or np.any(logdet < LOG_ABS_UNDERFLOW):
        raise NodeProximity("parameter gradient requested on top of a node")
    return np.einsum("wki,wit->wkt", np.linalg.inv(m), feats).reshape(pos.shape[0], -1)
