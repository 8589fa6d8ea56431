"""Dense first step (state.step == 0, optimizers.py:327-330) and exact_truncated_svd
(svdengine.py:75-85) beyond the 512-column limit of the hand-written device Jacobi: cuSOLVER's
SVD on the device (linalg.exact_svd), checked against numpy's LAPACK SVD."""

import numpy as np
import pytest

from conftest import rel, subspace_sine

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_exact_truncated_svd_large():
    from paper_2512_05749_b200.svdengine import exact_truncated_svd

    rng = np.random.default_rng(3)
    m, n, L = 3000, 700, 60
    a = rng.standard_normal((m, L)) @ np.diag(np.arange(1, L + 1) ** -1.0) @ \
        rng.standard_normal((L, n)) + 1e-3 * rng.standard_normal((m, n))
    f = exact_truncated_svd(a, 20)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    assert rel(f.sigma.cpu().numpy(), s[:20]) < 1e-12
    assert subspace_sine(f.u.cpu().numpy(), u[:, :20]) < 1e-9
    assert subspace_sine(f.v.cpu().numpy().T, vt[:20].T) < 1e-9


def test_dense_first_step_large():
    from paper_2512_05749_b200 import estimators, optimizers

    rng = np.random.default_rng(4)
    N, P, k, lam = 600, 2048, 16, 1e-3
    o = rng.standard_normal((N, 40)) @ rng.standard_normal((40, P)) * 0.1 + \
        0.01 * rng.standard_normal((N, P))
    e = -1.0 + 0.1 * rng.standard_normal(N)
    st = optimizers.WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=np.zeros((P, 0)),
                              r_max=k, delta=0.0, sigma_floor=lam, eps_grow=0.0, step=0)
    b = estimators.assemble(estimators.SampleBatch((None,) * N, e, o))
    _, st1, diag, upd = optimizers.wssr_step(np.zeros(P), b, 1.0, st, return_update=True)
    # reference step 0: exact SVD of ohat = o_matrix, top-k, rank cut, preconditioner
    om = ((o - o.mean(0)) / np.sqrt(N)).T
    ec = np.clip(e, e.mean() - 5 * e.std(), e.mean() + 5 * e.std())
    lv = (ec - ec.mean()) / np.sqrt(N)
    u, s, _ = np.linalg.svd(om, full_matrices=False)
    u, s = u[:, :k], s[:k]
    r = int(np.count_nonzero(s ** 2 >= 1e-6 * s[0] ** 2))
    u, s = u[:, :r], s[:r]
    g = om @ lv
    c = u.T @ g
    ref = u @ (c / s ** 2) + (g - u @ c) / lam
    assert diag.effective_rank == r
    assert rel(upd.cpu().numpy(), ref) < 1e-10
    assert rel(torch.linalg.vector_norm(st1.obar, dim=0).cpu().numpy(), s) < 1e-9
