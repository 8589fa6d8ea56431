"""Row-sharded restatement of the WSSR step - TEST INFRASTRUCTURE ONLY.

Mirrors, in numpy, the decomposition the CUDA engine uses under row (walker) sharding
(csrc/engine.cu: assemble(), apply_O(), ssi_core(), step()), with the collective passed in as
`allreduce(np.ndarray) -> np.ndarray` (sum over ranks).  tests/test_sharding_gloo.py runs it on
world_size 2 with torch.distributed/gloo and checks it against the unsharded oracle, which is
itself pinned to the reference (oracle/wssr_oracle.py).
"""

from __future__ import annotations

import math

import numpy as np

from . import wssr_oracle as orc


def assemble_sharded(derivs_local, energies_local, offset, n_global, allreduce, n_std=5.0):
    """estimators.assemble over row shards: energies gathered by a zero-padded sum, column
    statistics merged with Chan's update expressed as sums (engine.cu assemble())."""
    n = derivs_local.shape[0]
    e_all = np.zeros(n_global)
    e_all[offset:offset + n] = energies_local
    e_all = allreduce(e_all)
    c = orc.clip_energies(e_all, n_std)
    loss = float(c.mean())
    lraw = (c - loss)[offset:offset + n]
    s = 1.0 / math.sqrt(n_global)
    mu_loc = derivs_local.mean(axis=0)
    d = derivs_local - mu_loc
    m2_loc = (d * d).sum(axis=0)
    g_loc = d.T @ lraw
    mu = allreduce(n * mu_loc) / n_global
    delta = mu_loc - mu
    m2 = allreduce(m2_loc + n * delta * delta)
    g = allreduce(g_loc + delta * lraw.sum())
    return dict(loss=loss, raw_loss=float(e_all.mean()), mu=mu, l_local=lraw * s,
                gradient=2.0 * g / n_global, fro2=float(m2.sum()) / n_global)


def _cholqr2_rows(v, allreduce):
    """CholeskyQR2 of a row-sharded block with allreduced Grams."""
    g1 = allreduce(v.T @ v)
    r1 = np.linalg.cholesky(g1).T
    q1 = v @ np.linalg.inv(r1)
    g2 = allreduce(q1.T @ q1)
    r2 = np.linalg.cholesky(g2).T
    return q1 @ np.linalg.inv(r2), r2 @ r1


def wssr_step_sharded(derivs_local, bundle, st, allreduce, max_iters=3, tol=1e-10, rng_seed=0):
    """warm-started ssi branch of wssr_step (delta = 0) on a row shard; returns
    (update, sigma, U, iterations, r_eff)."""
    P = derivs_local.shape[1]
    s = 1.0 / math.sqrt(bundle["n_global"])
    oc = (derivs_local - bundle["mu"]) * s            # this rank's rows of Ohat^T
    req = min(st.r_max, P, bundle["n_global"])
    u0 = orc.warm_start(st.u_prev, req, P, orc.step_seed(rng_seed, st.step))
    fro2 = bundle["fro2"]
    q = orc.qr_pos(u0)[0]
    v = oc @ q
    u = allreduce(oc.T @ v)
    it = 0
    while True:
        q = orc.qr_pos(u)[0]
        it += 1
        v2 = oc @ q
        w = allreduce(oc.T @ v2)
        quo = q.T @ w
        res = float(np.linalg.norm(w - q @ quo)) / fro2
        mix = float(np.linalg.norm(quo - np.diag(np.diagonal(quo)))) / fro2
        if max(res, mix) < tol or it >= max_iters:
            break
        v, u = v2, w
    qv, rv = _cholqr2_rows(v, allreduce)
    raw = np.diagonal(rv).copy()
    order = np.argsort(-raw, kind="stable")
    sig = raw[order]
    k = int(np.sum(sig > 0))
    U = orc.qr_pos(u[:, order[:k]])[0]
    r_eff = int(np.count_nonzero(sig[:k] ** 2 >= st.r_reg * sig[0] ** 2))
    U = U[:, :r_eff]
    sig = sig[:r_eff]
    gbar = 0.5 * bundle["gradient"]
    c = U.T @ gbar
    upd = U @ (c / sig ** 2) + (gbar - U @ c) / st.sigma_floor
    lbar = allreduce(qv[:, order[:r_eff]].T @ bundle["l_local"])
    return dict(update=upd, sigma=sig, U=U, iterations=it, r_eff=r_eff, lbar=lbar)
