"""The reference's own WSSR / SVD-engine / linalg test bodies, restated against the drop-in API on
the GPU (reference: pkg/tests/test_optimizers.py:256-425, test_svdengine.py:135-170,
test_linalg.py:302-336, test_acceptance.py:282-413).  These exercise the first (dense) step,
the 'exact' and 'randomized' backends, rank growth/truncation and the history recursion."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def H(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def raw_bundle(o, l):
    from paper_2512_05749_b200.estimators import EstimatorBundle

    o = np.asarray(o, dtype=np.float64)
    l = np.asarray(l, dtype=np.float64)
    return EstimatorBundle(loss=0.0, raw_loss=0.0, o_matrix=o, l_vector=l, gradient=2.0 * (o @ l))


def pinv_sr(theta, o, l, eta, rel_tol=1e-12):
    """Full SR with pseudo-inverse on S = o o^T and gradient o l (optimizers.py:68-115)."""
    s = o @ o.T
    g = o @ l
    w, v = np.linalg.eigh(s)
    lam = np.max(np.abs(w))
    keep = np.abs(w) >= rel_tol * lam
    inv = np.where(keep, 1.0 / np.where(keep, w, 1.0), 0.0)
    return theta - eta * (v @ (inv * (v.T @ g)))


# ------------------------------------------------------------------- optimizers.wssr_step
def test_first_step_averages_current_batch_only():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    rng = np.random.default_rng(14)
    o = rng.standard_normal((5, 12))
    l = rng.standard_normal(12)
    state = WssrState.initial(5, rank_init=5, delta=0.95)
    _, state1, diag = wssr_step(np.zeros(5), raw_bundle(o, l), 0.01, state)
    ob = H(state1.obar)
    np.testing.assert_allclose(ob @ ob.T, 0.05 * (o @ o.T), atol=1e-10)
    np.testing.assert_allclose(ob @ H(state1.lbar), 0.05 * (o @ l), atol=1e-10)
    assert not diag.ssi.warm_started
    assert diag.sigma_drift == 0.0 and diag.projector_drift == 0.0


def test_three_step_recursion_matches_reference_averaging():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    delta = 0.7
    state = WssrState.initial(5, rank_init=5, delta=delta, r_reg=1e-30)
    theta = np.zeros(5)
    s_ref = np.zeros((5, 5))
    g_ref = np.zeros(5)
    for seed in (20, 21, 22):
        step_rng = np.random.default_rng(seed)
        o = step_rng.standard_normal((5, 12))
        l = step_rng.standard_normal(12)
        theta, state, _ = wssr_step(theta, raw_bundle(o, l), 0.01, state, svd_backend="exact")
        s_ref = delta * s_ref + (1.0 - delta) * (o @ o.T)
        g_ref = delta * g_ref + (1.0 - delta) * (o @ l)
    ob = H(state.obar)
    np.testing.assert_allclose(ob @ ob.T, s_ref, atol=1e-10)
    np.testing.assert_allclose(ob @ H(state.lbar), g_ref, atol=1e-10)


def test_full_rank_update_matches_pseudo_inverse_oracle():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    rng = np.random.default_rng(16)
    o = rng.standard_normal((5, 12))
    l = rng.standard_normal(12)
    theta = rng.standard_normal(5)
    state = WssrState.initial(5, rank_init=5, delta=0.0)
    got, _, diag = wssr_step(theta, raw_bundle(o, l), 0.2, state)
    assert diag.effective_rank == 5
    np.testing.assert_allclose(H(got), pinv_sr(theta, o, l, 0.2), atol=1e-10)


def test_complement_branch_and_relative_floor_first_step():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    o = np.array([[5.0, -5.0, 0.0, 0.0], [0.0, 0.0, 1.0, -1.0]])
    l = np.array([0.0, 0.0, 0.5, -0.5])
    state = WssrState.initial(2, rank_init=2, delta=0.0, r_reg=0.1, sigma_floor=1e-3)
    got, _, diag = wssr_step(np.zeros(2), raw_bundle(o, l), 0.01, state)
    assert diag.effective_rank == 1
    np.testing.assert_allclose(H(got), -0.01 * np.array([0.0, 1.0]) / 1e-3, atol=1e-10)
    state = WssrState.initial(2, rank_init=2, delta=0.0, r_reg=0.1, sigma_floor=1e-3,
                              sigma_floor_relative=True)
    got, _, _ = wssr_step(np.zeros(2), raw_bundle(o, l), 0.01, state)
    np.testing.assert_allclose(H(got), -0.01 * np.array([0.0, 1.0]) / (1e-3 * 50.0), atol=1e-10)


def test_preconditioner_spectrum_and_descent():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    rng = np.random.default_rng(17)
    for trial in range(10):
        m = 6
        o = rng.standard_normal((m, 14))
        l = rng.standard_normal(14)
        state = WssrState.initial(m, rank_init=4, r_reg=1e-3)
        theta1, state1, diag = wssr_step(np.zeros(m), raw_bundle(o, l), 1.0, state)
        u = H(state1.u_prev)
        sig = np.linalg.norm(H(state1.obar), axis=0)
        floor = state.sigma_floor
        p = u @ np.diag(sig ** -2) @ u.T + (np.eye(m) - u @ u.T) / floor
        eigs = np.linalg.eigvalsh(p)
        lo = min(1.0 / floor, sig[0] ** -2)
        hi = max(1.0 / floor, sig[-1] ** -2)
        assert eigs.min() >= lo * (1 - 1e-9)
        assert eigs.max() <= hi * (1 + 1e-9)
        g_bar = 0.05 * (o @ l)
        assert (-H(theta1)) @ g_bar > 0.0


def test_rank_grows_only_when_binding_and_caps_at_params():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    rng = np.random.default_rng(18)
    state = WssrState.initial(8, rank_init=2, r_reg=1e-6, eps_grow=0.5)
    theta = np.zeros(8)
    seen = [state.r_max]
    for _ in range(6):
        bundle = raw_bundle(rng.standard_normal((8, 12)), rng.standard_normal(12))
        theta, state, diag = wssr_step(theta, bundle, 0.01, state)
        assert diag.effective_rank >= 1
        assert state.r_max >= seen[-1]
        if state.r_max > seen[-1]:
            assert diag.effective_rank == diag.r_max == seen[-1]
        seen.append(state.r_max)
    assert seen == [2, 3, 5, 8, 8, 8, 8]


def test_truncation_blocks_growth():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    rng = np.random.default_rng(19)
    u = rng.standard_normal(6)
    state = WssrState.initial(6, rank_init=2, r_reg=1e-6)
    theta = np.zeros(6)
    for _ in range(3):
        o = np.outer(u, rng.standard_normal(9))
        o += 1e-9 * rng.standard_normal(o.shape)
        theta, state, diag = wssr_step(theta, raw_bundle(o, rng.standard_normal(9)), 0.01, state)
        assert diag.effective_rank == 1
    assert state.r_max == 2


def test_warm_start_engages_after_first_step_and_rssr():
    from paper_2512_05749_b200.optimizers import WssrState, rssr_step, wssr_step

    rng = np.random.default_rng(20)
    state = WssrState.initial(6, rank_init=3)
    theta = np.zeros(6)
    bundle = raw_bundle(rng.standard_normal((6, 10)), rng.standard_normal(10))
    theta, state, diag0 = wssr_step(theta, bundle, 0.01, state)
    assert not diag0.ssi.warm_started
    bundle2 = raw_bundle(rng.standard_normal((6, 10)), rng.standard_normal(10))
    _, _, diag1 = wssr_step(theta, bundle2, 0.01, state)
    assert diag1.ssi.warm_started and diag1.ssi.iterations_used >= 1
    _, st2, diag2 = rssr_step(theta, bundle2, 0.01, state)
    assert not diag2.ssi.warm_started and diag2.ssi.iterations_used == 0
    assert st2.step == state.step + 1


def test_criterion_07_full_rank_wssr_equals_pseudo_inverse():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    rng = np.random.default_rng(707)
    rng.standard_normal(7)
    o3 = rng.standard_normal((5, 12))
    l3 = rng.standard_normal(12)
    theta3 = rng.standard_normal(5)
    via, _, diag = wssr_step(theta3, raw_bundle(o3, l3), 0.2, WssrState.initial(5, rank_init=5,
                                                                                 delta=0.0))
    assert diag.effective_rank == 5
    np.testing.assert_allclose(H(via), pinv_sr(theta3, o3, l3, 0.2), atol=1e-10)


# ------------------------------------------------------------------- svdengine / linalg
def _haar(m, n, rng):
    return np.linalg.qr(rng.standard_normal((m, n)))[0]


def test_criterion_04_backends_match_exact_truncation():
    from paper_2512_05749_b200.svdengine import exact_truncated_svd, randomized_svd, ssi_svd

    rng = np.random.default_rng(404)
    worst_it = worst_sk = 0.0
    for trial in range(20):
        rank = int(rng.integers(4, 9))
        u = _haar(60, 12, rng)
        v = _haar(40, 12, rng)
        spectrum = (0.9 + 0.2 * rng.random(12)) * 0.5 ** np.arange(12)
        matrix = u @ np.diag(spectrum) @ v.T
        exact = exact_truncated_svd(matrix, rank)
        cold, _ = ssi_svd(matrix, rank, max_iters=30, residual_tol=0.0)
        worst_it = max(worst_it, np.linalg.norm(H(cold.reconstruct()) - H(exact.reconstruct())))
        low = u[:, :rank] @ np.diag(spectrum[:rank]) @ v[:, :rank].T
        sk = randomized_svd(low, rank, rng_seed=trial)
        worst_sk = max(worst_sk, np.linalg.norm(H(sk.reconstruct()) - low))
    assert worst_it < 1e-8 and worst_sk < 1e-10


def test_randomized_svd_reference_contract():
    from paper_2512_05749_b200.errors import DegenerateInput, RankTooLarge
    from paper_2512_05749_b200.svdengine import randomized_svd

    rng = np.random.default_rng(70)
    u = _haar(50, 3, rng)
    v = _haar(30, 3, rng)
    a = (u * np.array([3.0, 2.0, 1.0])) @ v.T
    for seed in (0, 1, 7, 123, 99999):
        f = randomized_svd(a, rank=3, oversample=5, rng_seed=seed)
        np.testing.assert_allclose(H(f.sigma), [3.0, 2.0, 1.0], atol=1e-10)
        np.testing.assert_allclose(H(f.reconstruct()), a, atol=1e-9)
    with pytest.raises(DegenerateInput):
        randomized_svd(np.zeros((30, 20)), rank=2, oversample=5)
    with pytest.raises(RankTooLarge):
        randomized_svd(np.eye(8), rank=4, oversample=5)
    b = rng.standard_normal((40, 30))
    f1 = randomized_svd(b, rank=5, oversample=5, rng_seed=3)
    f2 = randomized_svd(b, rank=5, oversample=5, rng_seed=3)
    np.testing.assert_array_equal(H(f1.u), H(f2.u))


def test_exact_svd_reference_contract():
    from paper_2512_05749_b200.linalg import exact_svd

    u, s, vt = exact_svd(np.diag([3.0, 2.0, 1.0]))
    np.testing.assert_allclose(H(s), [3.0, 2.0, 1.0], atol=1e-15)
    np.testing.assert_allclose(H((u * s) @ vt), np.diag([3.0, 2.0, 1.0]), atol=1e-14)
    a = np.zeros((4, 4))
    a[0, 0] = 2.0
    _, s, _ = exact_svd(a)
    np.testing.assert_allclose(H(s), [2.0, 0.0, 0.0, 0.0], atol=1e-15)
    rng = np.random.default_rng(3)
    for shape in ((6, 4), (4, 6), (300, 40), (30, 200), (257, 257)):
        a = rng.standard_normal(shape)
        u, s, vt = exact_svd(a)
        u, s, vt = H(u), H(s), H(vt)
        q = min(shape)
        assert u.shape == (shape[0], q) and vt.shape == (q, shape[1])
        assert np.all(np.diff(s) <= 0.0)
        np.testing.assert_allclose(u.T @ u, np.eye(q), atol=1e-12)
        np.testing.assert_allclose(vt @ vt.T, np.eye(q), atol=1e-12)
        np.testing.assert_allclose(s, np.linalg.svd(a, compute_uv=False), rtol=1e-12)
        assert np.linalg.norm((u * s) @ vt - a) / np.linalg.norm(a) < 1e-13
    with pytest.raises(ValueError):
        exact_svd(np.array([[1.0, np.nan], [0.0, 1.0]]))
