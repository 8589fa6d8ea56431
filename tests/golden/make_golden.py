"""Generate the golden fixtures by running the REFERENCE package itself (vmcsr, read-only at
/root/reference/pkg/src).  Run in the build container (the reference does not travel to the GPU
box); the resulting .npz files are committed.

    python tests/golden/make_golden.py

Fixtures (inputs are re-generated from seeds by paper_2512_05749_b200.synthetic; each fixture
stores input checksums so generator drift is caught):
  c0_T20.npz     BASELINE config 0 (N=1024, P=4096, k=32, lambda=1e-3), T=20 warm-started steps
  hist_T4.npz    small config with history averaging (delta=0.9), 4 steps
  growth_T4.npz  small config with rank growth (eps_grow=0.5) and widened warm starts
  kat.npz        known-answer vectors: QR patch, SSI closed forms, assemble closed form
  heavy_*.npz    heavy-tailed sample rows (pairs at 1e4/1e6/1e8, Student-t row scales df 1.5 and
                 1.0, Student-t elements df 1.5) with the reference's own reordering floor
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from vmcsr.estimators import SampleBatch, assemble  # noqa: E402
from vmcsr.linalg import qr_orthonormalize  # noqa: E402
from vmcsr.optimizers import WssrState, wssr_step  # noqa: E402
from vmcsr.svdengine import ssi_svd, subspace_drift  # noqa: E402

from paper_2512_05749_b200 import synthetic  # noqa: E402


def batch(o, e):
    b = SampleBatch.__new__(SampleBatch)
    object.__setattr__(b, "configs", (None,) * o.shape[0])
    object.__setattr__(b, "local_energies", e)
    object.__setattr__(b, "theta_logderivs", o)
    return b


def run(cfg, index, T, path, eps_grow=0.0, r_reg=1e-6, k_init=None, save_v_every=False):
    wl = synthetic.HostWorkload.from_config(cfg, index)
    v0, _ = qr_orthonormalize(wl.v0_raw())
    if k_init is not None:
        v0 = v0[:, :k_init]
    state = WssrState(obar=np.zeros((cfg["P"], 0)), lbar=np.zeros(0), u_prev=v0,
                      r_max=cfg["k"], delta=cfg["delta"], sigma_floor=cfg["lam"], r_reg=r_reg,
                      eps_grow=eps_grow, step=1)
    out = {"T": T, "N": cfg["N"], "P": cfg["P"], "k": cfg["k"], "delta": cfg["delta"],
           "lam": cfg["lam"], "eps_grow": eps_grow, "r_reg": r_reg,
           "k_init": cfg["k"] if k_init is None else k_init}
    for t in range(T):
        o, e = wl.next()
        out[f"in_sum_{t}"] = np.array([o.sum(), (o * o).sum(), e.sum()])
        bundle = assemble(batch(o, e))
        theta1, state_next, diag = wssr_step(np.zeros(cfg["P"]), bundle, 1.0, state)
        out[f"loss_{t}"] = np.array([bundle.loss, bundle.raw_loss])
        if t == 0:
            out["gradient_0"] = bundle.gradient
            out["l_vector_0"] = bundle.l_vector
        out[f"update_{t}"] = -theta1
        out[f"sigma_{t}"] = np.linalg.norm(state_next.obar, axis=0)
        out[f"lbar_{t}"] = state_next.lbar
        out[f"ints_{t}"] = np.array([diag.effective_rank, diag.ssi.iterations_used, diag.r_max,
                                     state_next.r_max])
        out[f"diag_{t}"] = np.array([diag.ssi.subspace_residual, diag.sigma_drift,
                                     diag.projector_drift])
        if save_v_every or t in (0, T - 1):
            out[f"V_{t}"] = state_next.u_prev
        state = state_next
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


def heavy(kind, mag, path, T=2, N=1024, P=4096, k=8):
    """Heavy-tailed sample rows (synthetic.HeavyRowWorkload), run by the reference twice: on the
    batch as generated and with the samples permuted.  The permuted run only reorders the
    reference's own FP64 sums; its distance to the first run is the conditioning floor of the
    outputs on this input, stored beside them (floor_update / floor_sigma / floor_angle)."""
    cfg = synthetic.config("c0", N=N, P=P, k=k, L=24, delta=0.0, lam=1e-3)
    out = {"T": T, "N": N, "P": P, "k": k, "kind": kind, "mag": mag, "lam": cfg["lam"]}
    perm = np.random.default_rng(99).permutation(N)
    runs = []
    for permuted in (False, True):
        wl = synthetic.HeavyRowWorkload(N, P, k, cfg["L"], cfg["alpha"], cfg["drift"], 300, 400,
                                        kind, mag)
        v0, _ = qr_orthonormalize(wl.v0_raw())
        state = WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=v0, r_max=k,
                          delta=0.0, sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
        res = []
        for t in range(T):
            o, e = wl.next()
            if not permuted:
                out[f"in_sum_{t}"] = np.array([o.sum(), (o * o).sum(), e.sum()])
            else:
                o, e = o[perm], e[perm]
            theta1, state, diag = wssr_step(np.zeros(P), assemble(batch(o, e)), 1.0, state)
            res.append((-theta1, np.linalg.norm(state.obar, axis=0), state.u_prev,
                        np.array([diag.effective_rank, diag.ssi.iterations_used])))
        runs.append(res)
    for t in range(T):
        (u1, s1, v1, i1), (u2, s2, v2, i2) = runs[0][t], runs[1][t]
        out[f"update_{t}"] = u1
        out[f"sigma_{t}"] = s1
        out[f"ints_{t}"] = i1
        if t == T - 1:
            out[f"V_{t}"] = v1
        r = min(v1.shape[1], v2.shape[1])
        out[f"floor_{t}"] = np.array([
            np.linalg.norm(u2 - u1) / np.linalg.norm(u1),
            np.linalg.norm(s2[:r] - s1[:r]) / np.linalg.norm(s1[:r]),
            np.linalg.norm(v2[:, :r] - v1[:, :r] @ (v1[:, :r].T @ v2[:, :r]), 2),
            float(np.array_equal(i1, i2))])
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes", [out[f"floor_{t}"] for t in range(T)])


def kat(path):
    out = {}
    # QR patch (test_linalg.py:45-51 shape): duplicated column -> r[1,1] == 0
    rng = np.random.default_rng(7)
    a = rng.standard_normal((6, 2))
    dfc = np.column_stack([a[:, 0], a[:, 0], a[:, 1]])
    q, r = qr_orthonormalize(dfc)
    out.update(qr_patch_a=dfc, qr_patch_q=q, qr_patch_r=r)
    # QR of a tall random block (fast path)
    a2 = np.random.default_rng(42).standard_normal((200, 16))
    q2, r2 = qr_orthonormalize(a2)
    out.update(qr_a=a2, qr_q=q2, qr_r=r2)
    # SSI cold start on diag(5,4,3,2,1) (test_svdengine.py:30-36)
    f, rep = ssi_svd(np.diag([5.0, 4.0, 3.0, 2.0, 1.0]), rank=2, max_iters=60)
    out.update(ssi_diag_sigma=f.sigma, ssi_diag_u=f.u, ssi_diag_iters=np.array([rep.iterations_used]))
    # SSI warm start on a mid-size random low-rank-plus-noise matrix
    rng = np.random.default_rng(123)
    m, n, k = 300, 120, 10
    uu = np.linalg.qr(rng.standard_normal((m, 30)))[0]
    vv = np.linalg.qr(rng.standard_normal((n, 30)))[0]
    mat = (uu * (0.8 ** np.arange(30))) @ vv.T + 1e-3 * rng.standard_normal((m, n))
    u0 = np.linalg.qr(rng.standard_normal((m, k)))[0]
    f, rep = ssi_svd(mat, rank=k, max_iters=4, u_init=u0)
    out.update(ssi_mat=mat, ssi_u0=u0, ssi_u=f.u, ssi_sigma=f.sigma, ssi_v=f.v,
               ssi_rep=np.array([rep.iterations_used, rep.subspace_residual]))
    sd, pd = subspace_drift(f, type(f)(u=u0, sigma=np.linspace(2, 1, k), v=f.v))
    out.update(drift=np.array([sd, pd]))
    # assemble two-sample closed form (test_estimators.py:79-91)
    aa = np.array([1.0, -2.0, 0.5])
    bb = np.array([0.2, 0.7, -1.1])
    ee = np.array([3.0, 1.0])
    bd = assemble(batch(np.stack([aa, bb]), ee), clip_n_std=np.inf)
    out.update(asm_o=bd.o_matrix, asm_l=bd.l_vector, asm_g=bd.gradient)
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


def main(which):
    if "base" in which:
        c0 = synthetic.config("c0")
        run(c0, 0, 20, os.path.join(HERE, "c0_T20.npz"))
        small = synthetic.config("c0", N=96, P=300, k=12, L=20, delta=0.9, lam=1e-3)
        run(small, 7, 4, os.path.join(HERE, "hist_T4.npz"), save_v_every=True)
        grow = synthetic.config("c0", N=64, P=160, k=6, L=12, delta=0.5, lam=1e-2)
        run(grow, 8, 4, os.path.join(HERE, "growth_T4.npz"), eps_grow=0.5, k_init=4,
            save_v_every=True)
        kat(os.path.join(HERE, "kat.npz"))
    if "heavy" in which:
        for kind, mag in (("pair", 1e4), ("pair", 1e6), ("pair", 1e8), ("tscale", 1.5),
                          ("tscale", 1.0), ("telem", 1.5)):
            heavy(kind, mag, os.path.join(HERE, f"heavy_{kind}_{mag:g}.npz"))


if __name__ == "__main__":
    # python tests/golden/make_golden.py [base] [heavy]   (default: all)
    main(sys.argv[1:] or ["base", "heavy"])
