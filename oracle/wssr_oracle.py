"""CPU oracle of the WSSR step - TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import this module,
and only as the checker / the timed reference arm.  The product path (paper_2512_05749_b200/)
never imports it.

It restates, in plain numpy/LAPACK, the reference algorithm of the package `vmcsr`
(arXiv 2512.05749, /root/reference/pkg/src/vmcsr):

  clip_energies    estimators.py:53-71    assemble         estimators.py:74-100
  qr_pos           linalg.py:29-105       ssi              svdengine.py:88-158
  subspace_drift   svdengine.py:199-226   residual         svdengine.py:56-67
  warm_start       optimizers.py:277-289  wssr_step        optimizers.py:292-391 (ssi branch)

Parity pinned: tests/golden/*.npz were produced by tests/golden/make_golden.py, which runs the
reference package itself; tests/test_oracle_golden.py checks this restatement against them and
against the reference's own known-answer tests.  The arithmetic dependency is numpy/LAPACK
(reference pins numpy>=1.24, scipy>=1.10; pyproject.toml:10-13).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DEFICIENT_REL = 1e-12   # linalg.py:16
ZERO_NORM = 1e-300      # linalg.py:15
COLD_SEED = 0x5EED      # svdengine.py:17


class OracleError(Exception):
    def __init__(self, kind, msg=""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ---- estimators ---------------------------------------------------------------------------
def clip_energies(e, n_std=5.0):
    """Population-std clamp (estimators.py:53-71)."""
    e = np.asarray(e, dtype=np.float64)
    if e.size < 2:
        raise OracleError("DegenerateBatch", "clipping window needs at least two samples")
    if not np.isfinite(n_std):
        return e.copy()
    if n_std < 0:
        raise ValueError("clipping width must be nonnegative")
    mid, sd = float(e.mean()), float(e.std())
    if sd == 0.0:
        return e.copy()
    return np.minimum(np.maximum(e, mid - n_std * sd), mid + n_std * sd)


def assemble(derivs, energies, n_std=5.0):
    """Centred bundle (estimators.py:74-100).  Returns a dict with the reference field names."""
    d = np.asarray(derivs, dtype=np.float64)
    n = d.shape[0]
    if n < 2:
        raise OracleError("DegenerateBatch", "need at least two samples")
    c = clip_energies(energies, n_std)
    loss = float(c.mean())
    s = 1.0 / math.sqrt(n)
    o = np.ascontiguousarray(((d - d.mean(axis=0)) * s).T)
    lv = (c - loss) * s
    return dict(loss=loss, raw_loss=float(np.mean(energies)), o_matrix=o, l_vector=lv,
                gradient=2.0 * (o @ lv))


# ---- QR -------------------------------------------------------------------------------------
def _fill_direction(qb, m):
    """First canonical vector with a large remainder against qb (linalg.py:87-105)."""
    best, best_norm = None, -1.0
    for i in range(m):
        w = np.zeros(m)
        w[i] = 1.0
        for _ in range(2):
            if qb.shape[1]:
                w = w - qb @ (qb.T @ w)
        nw = float(np.linalg.norm(w))
        if nw > 0.5:
            return w / nw
        if nw > best_norm:
            best, best_norm = w, nw
    if best is None or best_norm <= 0.0:
        raise OracleError("ZeroMatrix", "no canonical direction")
    return best / best_norm


def qr_pos(a):
    """Thin QR with diag(R) >= 0 and the rank-deficiency patch (linalg.py:29-84)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    m, n = a.shape
    if m < n:
        raise ValueError("need at least as many rows as columns")
    fro = float(np.linalg.norm(a))
    if fro < ZERO_NORM:
        raise OracleError("ZeroMatrix", "numerically zero matrix")
    q, r = np.linalg.qr(a, mode="reduced")
    dg = np.diagonal(r)
    if np.min(np.abs(dg)) > DEFICIENT_REL * fro:
        sg = np.where(dg < 0.0, -1.0, 1.0)
        return q * sg, r * sg[:, None]
    # two-pass classical Gram-Schmidt, canonical fill for deficient columns
    q = np.zeros((m, n))
    r = np.zeros((n, n))
    tol = DEFICIENT_REL * fro
    for j in range(n):
        v = a[:, j].copy()
        for _ in range(2):
            if j:
                cf = q[:, :j].T @ v
                r[:j, j] += cf
                v = v - q[:, :j] @ cf
        nv = float(np.linalg.norm(v))
        if nv > tol:
            q[:, j] = v / nv
            r[j, j] = nv
        else:
            q[:, j] = _fill_direction(q[:, :j], m)
    return q, r


# ---- truncated SVD ----------------------------------------------------------------------------
def residual(ohat, u):
    """||G U - U(U^T G U)||_F / ||ohat||_F^2 (svdengine.py:56-67)."""
    fro2 = float(np.linalg.norm(ohat)) ** 2
    w = ohat @ (ohat.T @ u)
    return float(np.linalg.norm(w - u @ (u.T @ w)) / fro2)


def ssi(ohat, rank, max_iters=3, u_init=None, tol=1e-10):
    """Block subspace iteration with QR-diagonal sigma (svdengine.py:88-158)."""
    ohat = np.asarray(ohat, dtype=np.float64)
    m, n = ohat.shape
    if rank < 1 or rank > min(m, n):
        raise OracleError("RankTooLarge", f"rank {rank}")
    fro = float(np.linalg.norm(ohat))
    if fro == 0.0:
        raise OracleError("DegenerateInput", "zero matrix")
    warm = u_init is not None
    blk = (np.asarray(u_init, dtype=np.float64) if warm
           else np.random.default_rng(COLD_SEED).standard_normal((m, rank)))
    fro2 = fro * fro
    q = qr_pos(blk)[0]
    it = 0
    while True:
        v = ohat.T @ q
        u = ohat @ v
        q = qr_pos(u)[0]
        it += 1
        w = ohat @ (ohat.T @ q)
        quo = q.T @ w
        res = float(np.linalg.norm(w - q @ quo)) / fro2
        mix = float(np.linalg.norm(quo - np.diag(np.diagonal(quo)))) / fro2
        if max(res, mix) < tol or it >= max_iters:
            break
    qv, rv = qr_pos(v)
    raw = np.diagonal(rv).copy()
    order = np.argsort(-raw, kind="stable")
    sig = raw[order]
    k = int(np.sum(sig[:rank] > 0.0))
    if k == 0:
        raise OracleError("DegenerateInput", "no positive singular values")
    uf = qr_pos(u[:, order[:k]])[0]
    return dict(u=uf, sigma=sig[:k], v=qv[:, order[:k]].T, iterations=it, residual=res,
                warm=warm)


def subspace_drift(u1, s1, u2, s2):
    """sigma drift and projector drift (svdengine.py:199-226)."""
    r = min(len(s1), len(s2))
    if r == 0:
        return 0.0, 0.0
    sd = float(np.linalg.norm(np.asarray(s1)[:r] - np.asarray(s2)[:r]))
    a, b = u1[:, :r], u2[:, :r]
    pd = float(np.linalg.norm(b - a @ (a.T @ b), ord=2))
    return (0.0 if sd < 1e-12 else sd), (0.0 if pd < 1e-12 else pd)


# ---- WSSR step ------------------------------------------------------------------------------
@dataclass
class State:
    """Mirror of WssrState (optimizers.py:188-247)."""

    obar: np.ndarray
    lbar: np.ndarray
    u_prev: np.ndarray
    r_max: int
    delta: float = 0.95
    sigma_floor: float = 1e-3
    sigma_floor_relative: bool = False
    r_reg: float = 1e-6
    eps_grow: float = 0.1
    step: int = 0
    extra: dict = field(default_factory=dict)


def step_seed(rng_seed, step):
    """optimizers.py:273-274."""
    return int(np.random.SeedSequence((int(rng_seed), int(step))).generate_state(1)[0])


def warm_start(u_prev, requested, m, seed):
    """optimizers.py:277-289."""
    if u_prev.shape[1] >= requested:
        return np.ascontiguousarray(u_prev[:, :requested])
    extra = np.random.default_rng(seed).standard_normal((m, requested - u_prev.shape[1]))
    return qr_pos(np.concatenate([u_prev, extra], axis=1))[0]


def wssr_step(theta, o_matrix, l_vector, eta, st: State, max_iters=3, tol=1e-10, rng_seed=0):
    """One WSSR step, ssi branch with state.step >= 1 (optimizers.py:292-391).

    Returns (theta_next, state_next, info) with info = dict(update, sigma, r_eff, iterations,
    residual, sigma_drift, projector_drift, next_r_max).
    """
    if st.step == 0:
        raise ValueError("oracle covers the warm-started branch (step >= 1)")
    theta = np.asarray(theta, dtype=np.float64)
    m = o_matrix.shape[0]
    a, b = math.sqrt(st.delta), math.sqrt(1.0 - st.delta)
    ohat = np.concatenate([a * st.obar, b * o_matrix], axis=1)
    lhat = np.concatenate([a * st.lbar, b * l_vector])
    req = min(st.r_max, m, ohat.shape[1])
    u0 = warm_start(st.u_prev, req, m, step_seed(rng_seed, st.step))
    f = ssi(ohat, req, max_iters=max_iters, u_init=u0, tol=tol)
    top = f["sigma"][0] ** 2
    r_eff = int(np.count_nonzero(f["sigma"] ** 2 >= st.r_reg * top))
    if r_eff < 1:
        raise OracleError("RankCollapse", "")
    binding = len(f["sigma"]) == req == st.r_max and r_eff == st.r_max
    nxt = min(math.ceil((1.0 + st.eps_grow) * st.r_max), m) if binding else st.r_max
    u = f["u"][:, :r_eff]
    sig = f["sigma"][:r_eff]
    g = ohat @ lhat
    c = u.T @ g
    fl = st.sigma_floor * (top if st.sigma_floor_relative else 1.0)
    upd = u @ (c / sig ** 2) + (g - u @ c) / fl
    if st.u_prev.shape[1] == 0:
        sd = pd = 0.0
    else:
        sd, pd = subspace_drift(st.u_prev, np.linalg.norm(st.obar, axis=0), u, sig)
    nst = State(obar=u * sig, lbar=f["v"][:r_eff, :] @ lhat, u_prev=u, r_max=nxt,
                delta=st.delta, sigma_floor=st.sigma_floor,
                sigma_floor_relative=st.sigma_floor_relative, r_reg=st.r_reg,
                eps_grow=st.eps_grow, step=st.step + 1)
    info = dict(update=upd, sigma=sig, r_eff=r_eff, iterations=f["iterations"],
                residual=f["residual"], sigma_drift=sd, projector_drift=pd, next_r_max=nxt,
                v=f["v"][:r_eff])
    return theta - eta * upd, nst, info


def baseline_state(P, k, v0_raw, delta, lam, r_reg=1e-6):
    """BASELINE recipe: WssrState(obar=0 cols, u_prev=V0, r_max=k, eps_grow=0, step=1)
    (SURVEY.md 8(d))."""
    v0 = qr_pos(v0_raw)[0]
    return State(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=v0, r_max=k, delta=delta,
                 sigma_floor=lam, r_reg=r_reg, eps_grow=0.0, step=1)
