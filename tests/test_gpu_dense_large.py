"""Dense first step (state.step == 0, optimizers.py:327-330) and exact_truncated_svd
(svdengine.py:75-85 -> linalg.py:108-121, numpy's dgesdd in the reference) beyond the
512-column limit of the single-CTA device Jacobi: the blocked one-sided Jacobi of
csrc/jacobi.cuh (DMMA Grams and updates, no cuSOLVER), checked against numpy's LAPACK SVD -
including BASELINE configs[1] (c1) at full size from WssrState.initial-style step 0."""

import numpy as np
import pytest

from conftest import rel, subspace_sine

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture
def blocked_mode():
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    ctx.lib.wssr_set_dense_svd_mode(ctx.handle, 1)
    yield ctx
    ctx.lib.wssr_set_dense_svd_mode(ctx.handle, 0)


def _check_full_svd(a, tol_s=1e-11, tol_v=1e-9):
    from paper_2512_05749_b200 import linalg

    u, s, vt = (x.cpu().numpy() for x in linalg.exact_svd(a))
    ur, sr, vtr = np.linalg.svd(a, full_matrices=False)
    q = min(a.shape)
    assert u.shape == (a.shape[0], q) and vt.shape == (q, a.shape[1])
    assert np.all(np.diff(s) <= 0.0)
    np.testing.assert_allclose(s, sr, rtol=0, atol=tol_s * sr[0])
    keep = sr > 1e-8 * sr[0]   # the numerically nonzero part
    nk = int(keep.sum())
    assert np.abs(u[:, :nk].T @ u[:, :nk] - np.eye(nk)).max() < 1e-11
    assert np.abs(vt @ vt.T - np.eye(q)).max() < 1e-11
    assert np.abs((u * s) @ vt - a).max() < 1e-11 * sr[0]
    # well-separated leading subspaces agree with LAPACK's
    for k in (1, 5, 20):
        if k < nk and sr[k - 1] > 1.01 * sr[k]:
            assert subspace_sine(u[:, :k], ur[:, :k]) < tol_v
            assert subspace_sine(vt[:k].T, vtr[:k].T) < tol_v


@pytest.mark.parametrize("m,n", [(600, 550), (550, 600), (2000, 700), (700, 2000), (1500, 1500)])
def test_blocked_jacobi_matches_lapack(m, n):
    rng = np.random.default_rng(m + 7 * n)
    L = min(m, n)
    a = rng.standard_normal((m, L)) @ np.diag(np.linspace(1.0, 1e-3, L)) @ \
        rng.standard_normal((L, n))
    _check_full_svd(a)


def test_blocked_jacobi_rank_deficient_centred():
    """The step-0 shape: centred sample columns (sum to zero, so rank <= N - 1) plus exact
    duplicate columns."""
    rng = np.random.default_rng(11)
    P, N = 3000, 800
    o = rng.standard_normal((N, 50)) @ rng.standard_normal((50, P)) + 0.01 * rng.standard_normal(
        (N, P))
    o[5] = o[9]
    a = ((o - o.mean(0)) / np.sqrt(N)).T
    _check_full_svd(a)


@pytest.mark.parametrize("m,n", [(300, 200), (77, 130), (129, 129)])
def test_blocked_mode_small_matches_single_cta_path(m, n, blocked_mode):
    """The blocked Jacobi forced on sizes the single-CTA path also handles (odd sizes, padding
    rows and an odd block count)."""
    rng = np.random.default_rng(m * n)
    a = rng.standard_normal((m, n)) @ np.diag(0.97 ** np.arange(n))
    _check_full_svd(a)


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


def _step0_reference(o, e, k, lam):
    """optimizers.py:292-391 at step 0: exact SVD of ohat = o_matrix (LAPACK), top-k, rank cut,
    preconditioner."""
    N = o.shape[0]
    om = ((o - o.mean(0)) / np.sqrt(N)).T
    ec = np.clip(e, e.mean() - 5 * e.std(), e.mean() + 5 * e.std())
    lv = (ec - ec.mean()) / np.sqrt(N)
    u, s, _ = np.linalg.svd(om, full_matrices=False)
    u, s = u[:, :k], s[:k]
    r = int(np.count_nonzero(s ** 2 >= 1e-6 * s[0] ** 2))
    u, s = u[:, :r], s[:r]
    g = om @ lv
    c = u.T @ g
    return u @ (c / s ** 2) + (g - u @ c) / lam, u, s, r


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
    ref, _, s, r = _step0_reference(o, e, k, lam)
    assert diag.effective_rank == r
    assert rel(upd.cpu().numpy(), ref) < 1e-10
    assert rel(torch.linalg.vector_norm(st1.obar, dim=0).cpu().numpy(), s) < 1e-9


def test_c1_step0_against_lapack():
    """BASELINE configs[1] (N=4096, P=131072, k=64) from step 0: the 131072 x 4096 Ohat is
    factorised by the blocked Jacobi on the device and the resulting WSSR step compared with
    LAPACK's SVD of the same matrix at the north_star tolerances."""
    import time

    from paper_2512_05749_b200 import _lib, estimators, optimizers, synthetic

    cfg = synthetic.config("c1")
    N, P, k, lam = cfg["N"], cfg["P"], cfg["k"], cfg["lam"]
    wl = synthetic.HostWorkload.from_config(cfg, 1)
    o, e = wl.next()
    st = optimizers.WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=np.zeros((P, 0)),
                              r_max=k, delta=0.0, sigma_floor=lam, eps_grow=0.0, step=0)
    b = estimators.assemble(estimators.SampleBatch((None,) * N, e, o))
    t0 = time.perf_counter()
    _, st1, diag, upd = optimizers.wssr_step(np.zeros(P), b, 1.0, st, return_update=True)
    torch.cuda.synchronize()
    t_dev = time.perf_counter() - t0
    ctx = _lib.context()
    sweeps = ctx.lib.wssr_dense_svd_sweeps(ctx.handle)
    del b
    t0 = time.perf_counter()
    ref, u, s, r = _step0_reference(o, e, k, lam)
    t_cpu = time.perf_counter() - t0
    print(f"c1 step 0: device {t_dev:.1f} s ({sweeps} Jacobi sweeps), LAPACK reference "
          f"{t_cpu:.1f} s")
    assert diag.effective_rank == r
    assert rel(upd.cpu().numpy(), ref) < 1e-10
    assert rel(torch.linalg.vector_norm(st1.obar, dim=0).cpu().numpy(), s) < 1e-9
    assert subspace_sine(st1.u_prev.cpu().numpy(), u) < 1e-8
