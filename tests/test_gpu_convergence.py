"""The reference's convergence and early-exit contract, restated on the device.

Restates, against the drop-in ssi_svd / subspace_drift / subspace_residual:
* test_svdengine.py:64-78   residual monotone in the iteration budget;
* test_svdengine.py:80-103  warm start beats cold start (at most half the iterations);
* test_svdengine.py:116-122 column permutation leaves sigma unchanged;
* test_svdengine.py:172-212 subspace_drift properties;
* test_svdengine.py:215-224 subspace_residual diagnostic;
* test_acceptance.py:311-340 criterion 5a (warm restarts halve the iteration count at 1e-8).

On top of the reference's own assertions, every trial checks the device against the CPU oracle
(oracle/wssr_oracle.py) on the same input: the same iterations_used (the early-exit branch of
svdengine.py:139-141, SURVEY trap 9), the same sigma, and the same reported residual.
"""

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def H(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


def _orthonormal(rng, m, r):
    return np.linalg.qr(rng.standard_normal((m, r)))[0]


def _with_spectrum(rng, m, n, sigma):
    u = _orthonormal(rng, m, len(sigma))
    v = _orthonormal(rng, n, len(sigma))
    return (u * np.asarray(sigma)) @ v.T, u, v


def _ssi_both(a, rank, max_iters, u_init=None, tol=1e-10):
    """Device and oracle on the same input; asserts the branch structure agrees."""
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import ssi_svd

    f, rep = ssi_svd(a, rank=rank, max_iters=max_iters, u_init=u_init, residual_tol=tol)
    ref = orc.ssi(a, rank, max_iters=max_iters, u_init=u_init, tol=tol)
    assert rep.iterations_used == ref["iterations"], (rep.iterations_used, ref["iterations"])
    assert rep.warm_started == ref["warm"]
    np.testing.assert_allclose(H(f.sigma), ref["sigma"], rtol=1e-9)
    # residuals are compared where they carry signal (they bottom out at rounding level)
    if ref["residual"] > 1e-13:
        assert abs(rep.subspace_residual - ref["residual"]) <= 1e-6 * ref["residual"] + 1e-15
    return f, rep, ref


def test_residual_monotone_in_iteration_budget():
    """test_svdengine.py:64-78."""
    rng = np.random.default_rng(33)
    worse = 0
    for _ in range(20):
        a, _, _ = _with_spectrum(rng, 25, 18, [5.0, 4.0, 2.0, 0.5, 0.2, 0.1])
        residuals = []
        for m in (1, 2, 4, 8, 16):
            _, rep, _ = _ssi_both(a, 3, m, tol=0.0)
            assert rep.iterations_used == m
            residuals.append(rep.subspace_residual)
        worse += sum(residuals[i + 1] > residuals[i] + 1e-12 for i in range(len(residuals) - 1))
    assert worse == 0


def test_warm_start_beats_cold_start():
    """test_svdengine.py:80-103: warm iterations <= max(1, cold // 2) in all 20 trials."""
    rng = np.random.default_rng(44)
    wins = 0
    for _ in range(20):
        sigma = np.array([8.0, 6.0, 5.0, 1.0, 0.5, 0.25])
        a, _, _ = _with_spectrum(rng, 60, 40, sigma)
        perturbed = a + 1e-4 * np.linalg.norm(a) / np.sqrt(a.size) * rng.standard_normal(a.shape)
        u_warm = np.linalg.svd(a)[0]
        warm_iters = cold_iters = None
        for m in range(1, 41):
            _, rep, _ = _ssi_both(perturbed, 3, m, u_init=u_warm[:, :3], tol=1e-8)
            if rep.subspace_residual < 1e-8:
                warm_iters = rep.iterations_used
                break
        for m in range(1, 41):
            _, rep, _ = _ssi_both(perturbed, 3, m, tol=1e-8)
            if rep.subspace_residual < 1e-8:
                cold_iters = rep.iterations_used
                break
        assert warm_iters is not None and cold_iters is not None
        if warm_iters <= max(1, cold_iters // 2):
            wins += 1
    assert wins == 20


def test_column_permutation_leaves_sigma_unchanged():
    """test_svdengine.py:116-122."""
    from paper_2512_05749_b200.svdengine import ssi_svd

    rng = np.random.default_rng(55)
    a, _, _ = _with_spectrum(rng, 30, 12, [4.0, 3.0, 2.0, 1.0])
    perm = rng.permutation(12)
    f1, _ = ssi_svd(a, rank=4, max_iters=40)
    f2, _ = ssi_svd(np.ascontiguousarray(a[:, perm]), rank=4, max_iters=40)
    np.testing.assert_allclose(H(f1.sigma), H(f2.sigma), atol=1e-10)


def test_criterion_05a_warm_start_halves_iterations():
    """test_acceptance.py:311-340: 20 drifting matrices, warm restarts at most half the cold
    iterations at residual_tol 1e-8, with the iteration counts equal to the oracle's."""
    from paper_2512_05749_b200.svdengine import ssi_svd

    counts = []
    for trial in range(20):
        rng = np.random.default_rng(100 + trial)
        u = np.linalg.qr(rng.standard_normal((80, 14)))[0]
        v = np.linalg.qr(rng.standard_normal((60, 14)))[0]
        spectrum = np.array([8, 6.5, 5, 4, 3, 2.4, 1.2, 0.9, 0.7, 0.5, 0.4, 0.3, 0.2, 0.1],
                            dtype=np.float64)
        base = u @ np.diag(spectrum) @ v.T
        settled, _ = ssi_svd(base, 6, max_iters=300, residual_tol=1e-8)
        noise = rng.standard_normal((80, 60))
        noise *= 1e-4 * np.linalg.norm(base) / np.linalg.norm(noise)
        drifted = base + noise
        _, cold, _ = _ssi_both(drifted, 6, 300, tol=1e-8)
        _, warm, _ = _ssi_both(drifted, 6, 300, u_init=H(settled.u), tol=1e-8)
        assert warm.warm_started and not cold.warm_started
        assert warm.iterations_used * 2 <= cold.iterations_used
        counts.append((warm.iterations_used, cold.iterations_used))
    assert np.mean([w for w, _ in counts]) * 2 <= np.mean([c for _, c in counts])


def test_early_exit_branch_on_generic_spectra():
    """The exit test (svdengine.py:139-141) fires at the oracle's iteration on matrices that are
    not exactly low rank, across tolerances (SURVEY trap 9)."""
    rng = np.random.default_rng(7)
    exits = 0
    for trial in range(12):
        m, n = 90 + 7 * trial, 50 + 3 * trial
        sig = np.concatenate([[10.0, 7.0, 5.0, 3.0], 0.5 * 0.7 ** np.arange(30)])
        a, u, _ = _with_spectrum(rng, m, n, sig)
        warm = u[:, :4] + 1e-3 * rng.standard_normal((m, 4))
        for tol in (1e-6, 1e-8, 1e-10):
            _, rep, ref = _ssi_both(a, 4, 60, u_init=warm, tol=tol)
            exits += ref["iterations"] < 60
    assert exits >= 30


# ---------------------------------------------------------------- subspace_drift (172-212)
def test_drift_identical_factors():
    from paper_2512_05749_b200.svdengine import exact_truncated_svd, subspace_drift

    rng = np.random.default_rng(80)
    a, _, _ = _with_spectrum(rng, 20, 10, [2.0, 1.0, 0.5])
    fact = exact_truncated_svd(a, 3)
    assert subspace_drift(fact, fact) == (0.0, 0.0)


def test_drift_in_span_rotation_keeps_projector():
    from paper_2512_05749_b200.svdengine import TruncatedSvd, subspace_drift

    rng = np.random.default_rng(81)
    u = _orthonormal(rng, 20, 3)
    sigma = np.array([2.0, 1.5, 1.0])
    v = _orthonormal(rng, 12, 3).T
    rot, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    f1 = TruncatedSvd(u=u, sigma=sigma, v=v)
    f2 = TruncatedSvd(u=u @ rot, sigma=sigma, v=v)
    sdrift, pdrift = subspace_drift(f1, f2)
    assert sdrift == 0.0
    assert pdrift < 1e-7


def test_drift_matches_brute_force_projector_norm():
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import TruncatedSvd, subspace_drift

    rng = np.random.default_rng(82)
    u1 = _orthonormal(rng, 20, 3)
    u2 = _orthonormal(rng, 20, 3)
    sigma = np.array([3.0, 2.0, 1.0])
    v = _orthonormal(rng, 15, 3).T
    f1 = TruncatedSvd(u=u1, sigma=sigma, v=v)
    f2 = TruncatedSvd(u=u2, sigma=sigma + 0.25, v=v)
    sdrift, pdrift = subspace_drift(f1, f2)
    brute = np.linalg.norm(u1 @ u1.T - u2 @ u2.T, ord=2)
    np.testing.assert_allclose(pdrift, brute, atol=1e-10)
    np.testing.assert_allclose(sdrift, np.linalg.norm(np.full(3, 0.25)), atol=1e-12)
    osd, opd = orc.subspace_drift(u1, sigma, u2, sigma + 0.25)
    assert abs(sdrift - osd) <= 1e-14 and abs(pdrift - opd) <= 1e-12


def test_drift_rank_mismatch_truncates():
    from paper_2512_05749_b200.svdengine import TruncatedSvd, subspace_drift

    rng = np.random.default_rng(83)
    u = _orthonormal(rng, 10, 4)
    f_big = TruncatedSvd(u=u, sigma=np.array([4.0, 3.0, 2.0, 1.0]), v=_orthonormal(rng, 8, 4).T)
    f_small = TruncatedSvd(u=u[:, :2], sigma=np.array([4.0, 3.0]), v=_orthonormal(rng, 8, 2).T)
    assert subspace_drift(f_big, f_small) == (0.0, 0.0)


@pytest.mark.parametrize("seed", range(6))
def test_drift_matches_oracle_on_random_pairs(seed):
    """Random factor pairs of mixed ranks and sizes against the oracle's dgesdd norm."""
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import TruncatedSvd, subspace_drift

    rng = np.random.default_rng(900 + seed)
    m = [40, 200, 1000, 3000, 64, 130][seed]
    r1, r2 = [(3, 3), (8, 5), (16, 16), (32, 20), (64, 64), (7, 12)][seed]
    u1 = _orthonormal(rng, m, r1)
    base = np.hstack([u1, rng.standard_normal((m, max(0, r2 - r1)))])[:, :r2]
    u2 = np.linalg.qr(base + 1e-3 * rng.standard_normal(base.shape))[0]
    s1 = np.sort(rng.uniform(0.5, 5.0, r1))[::-1]
    s2 = np.sort(rng.uniform(0.5, 5.0, r2))[::-1]
    f1 = TruncatedSvd(u=u1, sigma=s1, v=_orthonormal(rng, 9 + r1, r1).T)
    f2 = TruncatedSvd(u=u2, sigma=s2, v=_orthonormal(rng, 9 + r2, r2).T)
    sd, pd = subspace_drift(f1, f2)
    osd, opd = orc.subspace_drift(u1, s1, u2, s2)
    assert abs(sd - osd) <= 1e-12 * max(1.0, osd)
    assert abs(pd - opd) <= 1e-9 * max(1.0, opd)


# ---------------------------------------------------------------- subspace_residual (215-224)
def test_residual_invariant_subspace_gives_zero():
    from paper_2512_05749_b200.svdengine import subspace_residual

    rng = np.random.default_rng(90)
    a, u_true, _ = _with_spectrum(rng, 25, 15, [3.0, 1.0])
    assert subspace_residual(a, u_true) < 1e-14


def test_residual_generic_subspace_gives_positive():
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import subspace_residual

    rng = np.random.default_rng(91)
    a = rng.standard_normal((25, 15))
    q = _orthonormal(rng, 25, 3)
    got = subspace_residual(a, q)
    assert got > 1e-4
    assert rel(got, orc.residual(a, q)) < 1e-12


@pytest.mark.parametrize("m,n,k", [(300, 120, 8), (2000, 700, 32), (5000, 1500, 64)])
def test_residual_matches_oracle(m, n, k):
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import subspace_residual

    rng = np.random.default_rng(m + n + k)
    a = rng.standard_normal((m, n)) @ np.diag(0.9 ** np.arange(n))
    q = _orthonormal(rng, m, k)
    assert rel(subspace_residual(a, q), orc.residual(a, q)) < 1e-12
