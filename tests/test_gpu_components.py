"""Component parity on the GPU: the reference's own known-answer tests (restated from
/root/reference/pkg/tests/test_linalg.py, test_svdengine.py, test_estimators.py) run against the
drop-in API, plus the DMMA GEMM family against a torch fp64 reference."""

import math

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def H(x):
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


# ---------------------------------------------------------------- GEMM family vs torch fp64
@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("M,N,K", [(5, 3, 7), (37, 5, 129), (300, 64, 1000), (64, 64, 50000),
                                   (1000, 33, 77), (257, 128, 999), (96, 200, 333),
                                   (4096, 1, 2000), (3, 3, 100000), (2000, 128, 5000),
                                   (20000, 64, 64), (4096, 64, 8192), (777, 256, 3000),
                                   (3000, 32, 5000)])
@pytest.mark.parametrize("pad,acc", [(0, False), (1, True), (2, False)])
@pytest.mark.parametrize("path", [0, 1])
def test_gemm_matches_torch(layout, M, N, K, pad, acc, path):
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    ctx.lib.wssr_set_gemm_path(ctx.handle, path)
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    opt = dict(dtype=torch.float64, device="cuda", generator=g)
    if layout == 0:
        lda = M + pad
        A = torch.randn(K, lda, **opt)
        shift = torch.randn(M, **opt)
        X = (A[:, :M] - shift[None, :]).t()
    else:
        lda = K + pad
        A = torch.randn(M, lda, **opt)
        shift = torch.randn(K, **opt)
        X = A[:, :K] - shift[None, :]
    ldb = N + pad
    B = torch.randn(K, ldb, **opt)
    C0 = torch.randn(M, N + pad, **opt)
    C = C0.clone()
    ctx.call("wssr_gemm_f64", layout, M, N, K, _lib.ptr(A), lda, _lib.ptr(shift), _lib.ptr(B),
             ldb, _lib.ptr(C), N + pad, 0.7, int(acc), 1024)
    ref = 0.7 * (X @ B[:, :N]) + (C0[:, :N] if acc else 0.0)
    err = (C[:, :N] - ref).abs().max().item() / ref.abs().max().item()
    ctx.lib.wssr_set_gemm_path(ctx.handle, 0)
    assert err < 1e-13
    if pad:
        assert torch.equal(C[:, N:], C0[:, N:])  # leading-dimension padding untouched


# ---------------------------------------------------------------- linalg.qr_orthonormalize
def test_qr_contract_and_patch(golden):
    from paper_2512_05749_b200.linalg import qr_orthonormalize
    from paper_2512_05749_b200.errors import ZeroMatrix

    g = golden("kat.npz")
    q, r = qr_orthonormalize(np.eye(3))
    np.testing.assert_allclose(H(q), np.eye(3), atol=1e-15)
    q, r = qr_orthonormalize(np.array([3.0, 4.0]))
    np.testing.assert_allclose(H(q), [[0.6], [0.8]], atol=1e-15)
    np.testing.assert_allclose(H(r), [[5.0]], atol=1e-15)
    q, r = qr_orthonormalize(g["qr_patch_a"])        # deficient column -> GS patch path
    np.testing.assert_allclose(H(q), g["qr_patch_q"], atol=1e-13)
    np.testing.assert_allclose(H(r), g["qr_patch_r"], atol=1e-13)
    assert H(r)[1, 1] == 0.0
    q, r = qr_orthonormalize(g["qr_a"])              # CholeskyQR2 fast path
    np.testing.assert_allclose(H(q), g["qr_q"], atol=1e-13)
    np.testing.assert_allclose(H(r), g["qr_r"], atol=1e-12)
    with pytest.raises(ZeroMatrix):
        qr_orthonormalize(np.zeros((4, 2)))
    with pytest.raises(ValueError):
        qr_orthonormalize(np.ones((2, 4)))


@pytest.mark.parametrize("seed,m,n", [(1, 2, 1), (2, 12, 6), (3, 9, 9), (4, 1000, 37)])
def test_qr_idempotent_on_orthonormal_input(seed, m, n):
    from paper_2512_05749_b200.linalg import qr_orthonormalize

    rng = np.random.default_rng(seed)
    q, _ = qr_orthonormalize(rng.standard_normal((m, n)))
    q2, r2 = qr_orthonormalize(q)
    np.testing.assert_allclose(H(q2), H(q), atol=1e-10)
    np.testing.assert_allclose(H(r2), np.eye(n), atol=1e-10)


# ---------------------------------------------------------------- svdengine
def test_ssi_known_answers(golden):
    from paper_2512_05749_b200.svdengine import ssi_svd, subspace_drift, TruncatedSvd
    from paper_2512_05749_b200.errors import DegenerateInput, RankTooLarge

    g = golden("kat.npz")
    f, rep = ssi_svd(np.diag([5.0, 4.0, 3.0, 2.0, 1.0]), rank=2, max_iters=60)
    np.testing.assert_allclose(H(f.sigma), [5.0, 4.0], atol=1e-8)
    np.testing.assert_allclose(np.abs(H(f.u)), np.eye(5)[:, :2], atol=1e-6)
    assert rep.iterations_used == int(g["ssi_diag_iters"][0]) and not rep.warm_started
    f, rep = ssi_svd(g["ssi_mat"], 10, max_iters=4, u_init=g["ssi_u0"])
    assert rel(H(f.sigma), g["ssi_sigma"]) < 1e-9
    np.testing.assert_allclose(H(f.u), g["ssi_u"], atol=1e-9)
    np.testing.assert_allclose(H(f.v), g["ssi_v"], atol=1e-9)
    assert rep.iterations_used == int(g["ssi_rep"][0])
    np.testing.assert_allclose(rep.subspace_residual, g["ssi_rep"][1], rtol=1e-6)
    prev = f
    curr = TruncatedSvd(u=torch.as_tensor(g["ssi_u0"], device="cuda"),
                        sigma=torch.linspace(2, 1, 10, dtype=torch.float64, device="cuda"),
                        v=f.v)
    sd, pd = subspace_drift(prev, curr)
    np.testing.assert_allclose([sd, pd], g["drift"], rtol=1e-8)
    with pytest.raises(RankTooLarge):
        ssi_svd(np.eye(4), rank=5)
    with pytest.raises(RankTooLarge):
        ssi_svd(np.eye(4), rank=0)
    with pytest.raises(DegenerateInput):
        ssi_svd(np.zeros((6, 4)), rank=2)


def test_ssi_exact_fixed_point_one_iteration():
    from paper_2512_05749_b200.svdengine import ssi_svd

    rng = np.random.default_rng(5)
    u = np.linalg.qr(rng.standard_normal((30, 3)))[0]
    v = np.linalg.qr(rng.standard_normal((20, 3)))[0]
    a = (u * np.array([4.0, 2.0, 1.0])) @ v.T
    f, rep = ssi_svd(a, rank=3, max_iters=1, u_init=u)
    assert rep.iterations_used == 1 and rep.subspace_residual < 1e-12 and rep.warm_started
    np.testing.assert_allclose(H(f.sigma), [4.0, 2.0, 1.0], atol=1e-10)


def test_ssi_geometric_spectrum_and_factor_contract():
    from paper_2512_05749_b200.svdengine import ssi_svd

    rng = np.random.default_rng(20)
    sig = 2.0 ** -np.arange(1, 21)
    u = np.linalg.qr(rng.standard_normal((200, 20)))[0]
    v = np.linalg.qr(rng.standard_normal((120, 20)))[0]
    a = (u * sig) @ v.T
    f, _ = ssi_svd(a, rank=10, max_iters=30)
    np.testing.assert_allclose(H(f.sigma), sig[:10], atol=1e-8)
    uu = H(f.u)
    vv = H(f.v)
    np.testing.assert_allclose(uu.T @ uu, np.eye(10), atol=1e-10)
    np.testing.assert_allclose(vv @ vv.T, np.eye(10), atol=1e-10)


def test_ssi_early_exit_matches_reference_branch():
    """Converged warm start: the exit test fires before max_iters on both sides."""
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import ssi_svd

    rng = np.random.default_rng(9)
    u = np.linalg.qr(rng.standard_normal((80, 4)))[0]
    v = np.linalg.qr(rng.standard_normal((50, 4)))[0]
    a = (u * np.array([8.0, 4.0, 2.0, 1.0])) @ v.T
    ref = orc.ssi(a, 4, max_iters=20, u_init=u, tol=1e-10)
    f, rep = ssi_svd(a, rank=4, max_iters=20, u_init=u, residual_tol=1e-10)
    assert rep.iterations_used == ref["iterations"] < 20
    np.testing.assert_allclose(H(f.sigma), ref["sigma"], rtol=1e-12)


def test_ssi_deterministic():
    from paper_2512_05749_b200.svdengine import ssi_svd

    a = np.random.default_rng(66).standard_normal((15, 10))
    f1, r1 = ssi_svd(a, rank=3)
    f2, r2 = ssi_svd(a, rank=3)
    np.testing.assert_array_equal(H(f1.u), H(f2.u))
    np.testing.assert_array_equal(H(f1.sigma), H(f2.sigma))
    assert r1 == r2


# ---------------------------------------------------------------- estimators
def test_assemble_closed_forms(golden):
    from paper_2512_05749_b200.estimators import SampleBatch, assemble, clip_local_energies
    from paper_2512_05749_b200.errors import DegenerateBatch

    g = golden("kat.npz")
    a = np.array([1.0, -2.0, 0.5])
    b = np.array([0.2, 0.7, -1.1])
    e = np.array([3.0, 1.0])
    bd = assemble(SampleBatch((None, None), e, np.stack([a, b])), clip_n_std=np.inf)
    np.testing.assert_allclose(H(bd.o_matrix), g["asm_o"], atol=1e-15)
    np.testing.assert_allclose(H(bd.l_vector), g["asm_l"], atol=1e-15)
    np.testing.assert_allclose(H(bd.gradient), g["asm_g"], atol=1e-14)
    derivs = np.tile(np.random.default_rng(2).normal(size=4), (6, 1))
    bd = assemble(SampleBatch((None,) * 6, np.random.default_rng(3).normal(size=6), derivs))
    np.testing.assert_array_equal(H(bd.o_matrix), np.zeros((4, 6)))
    np.testing.assert_array_equal(H(bd.gradient), np.zeros(4))
    en = np.array([0.0, 0.0, 0.0, 0.0, 100.0])
    bd = assemble(SampleBatch((None,) * 5, en, np.eye(5)), clip_n_std=1.0)
    assert bd.raw_loss == pytest.approx(20.0)
    mu, sd = en.mean(), en.std()
    assert bd.loss == pytest.approx(np.clip(en, mu - sd, mu + sd).mean())
    with pytest.raises(DegenerateBatch):
        assemble(SampleBatch((None,), np.array([1.0]), np.ones((1, 3))))
    vals = np.random.default_rng(11).normal(size=50)
    vals[3] = 40.0
    np.testing.assert_allclose(H(clip_local_energies(vals, 2.0)),
                               np.clip(vals, vals.mean() - 2 * vals.std(),
                                       vals.mean() + 2 * vals.std()), atol=1e-12)


@pytest.mark.parametrize("n,m,seed", [(2, 1, 0), (20, 8, 1), (12, 5, 3), (1000, 300, 4)])
def test_assemble_matches_oracle(n, m, seed):
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.estimators import SampleBatch, assemble

    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, m)) + 3.0
    e = rng.normal(size=n)
    ref = orc.assemble(d, e, 5.0)
    bd = assemble(SampleBatch((None,) * n, e, d))
    np.testing.assert_allclose(H(bd.o_matrix), ref["o_matrix"], atol=1e-13)
    np.testing.assert_allclose(H(bd.gradient), ref["gradient"], atol=1e-13)
    np.testing.assert_allclose(H(bd.l_vector), ref["l_vector"], atol=1e-14)
    assert bd.loss == pytest.approx(ref["loss"], rel=1e-14)
    fro2 = float(np.linalg.norm(ref["o_matrix"]) ** 2)
    assert bd._fro2 == pytest.approx(fro2, rel=1e-12)


# ---------------------------------------------------------------- optimizers.wssr_step contract
def _raw_bundle(o, l):
    from paper_2512_05749_b200.estimators import EstimatorBundle

    o = np.asarray(o, dtype=np.float64)
    l = np.asarray(l, dtype=np.float64)
    return EstimatorBundle(loss=0.0, raw_loss=0.0, o_matrix=o, l_vector=l, gradient=2.0 * (o @ l))


def _warm_state(P, k, seed, **kw):
    from paper_2512_05749_b200.optimizers import WssrState

    u0 = np.linalg.qr(np.random.default_rng(seed).standard_normal((P, k)))[0]
    return WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=u0, r_max=k, step=1, **kw)


def test_wssr_complement_branch_scales_by_floor():
    from paper_2512_05749_b200.optimizers import wssr_step

    o = np.array([[5.0, -5.0, 0.0, 0.0], [0.0, 0.0, 1.0, -1.0]])
    l = np.array([0.0, 0.0, 0.5, -0.5])
    st = _warm_state(2, 2, 0, delta=0.0, r_reg=0.1, sigma_floor=1e-3)
    got, _, diag = wssr_step(np.zeros(2), _raw_bundle(o, l), 0.01, st, ssi_max_iters=30, ssi_residual_tol=0.0)
    assert diag.effective_rank == 1
    np.testing.assert_allclose(H(got), -0.01 * np.array([0.0, 1.0]) / 1e-3, atol=1e-10)
    st = _warm_state(2, 2, 0, delta=0.0, r_reg=0.1, sigma_floor=1e-3, sigma_floor_relative=True)
    got, _, _ = wssr_step(np.zeros(2), _raw_bundle(o, l), 0.01, st, ssi_max_iters=30, ssi_residual_tol=0.0)
    np.testing.assert_allclose(H(got), -0.01 * np.array([0.0, 1.0]) / (1e-3 * 50.0), atol=1e-10)


@pytest.mark.parametrize("seed", range(5))
def test_wssr_raw_bundle_matches_oracle(seed):
    """Explicit (uncentred) o_matrix bundles: gbar recomputed on the device."""
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.optimizers import wssr_step

    rng = np.random.default_rng(100 + seed)
    P, N, k = 40 + 7 * seed, 17 + 3 * seed, 5
    o = rng.standard_normal((P, N))
    l = rng.standard_normal(N)
    theta = rng.standard_normal(P)
    st = _warm_state(P, k, seed, delta=0.3, r_reg=1e-3)
    ost = orc.State(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=H(st.u_prev), r_max=k,
                    delta=0.3, sigma_floor=1e-3, r_reg=1e-3, eps_grow=0.1, step=1)
    for _ in range(3):
        got, st, diag = wssr_step(theta, _raw_bundle(o, l), 0.2, st)
        want, ost, info = orc.wssr_step(theta, o, l, 0.2, ost)
        assert diag.effective_rank == info["r_eff"]
        assert rel(H(got) - theta, want - theta) < 1e-10
        o = o + 0.01 * rng.standard_normal((P, N))


def test_wssr_validation_and_unsupported():
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step
    from paper_2512_05749_b200.errors import Unsupported

    with pytest.raises(ValueError):
        WssrState.initial(3, delta=1.0)
    with pytest.raises(ValueError):
        WssrState.initial(3, r_reg=0.0)
    with pytest.raises(ValueError):
        WssrState.initial(3, sigma_floor=0.0)
    with pytest.raises(ValueError):
        WssrState.initial(3, rank_init=0)
    st = WssrState.initial(7, rank_init=4)
    assert tuple(st.obar.shape) == (7, 0) and st.r_max == 4 and st.step == 0
    b = _raw_bundle(np.eye(3), np.zeros(3))
    with pytest.raises(ValueError, match="randomized"):
        wssr_step(np.zeros(3), b, 0.1, WssrState.initial(3, rank_init=2), svd_backend="lanczos")
    # dense first step beyond the hand-written dense-SVD limit (512): cuSOLVER on the device
    big = _raw_bundle(np.ones((600, 700)) + np.eye(600, 700), np.ones(700) / 700.0)
    th, st1, _ = wssr_step(np.zeros(600), big, 0.1, WssrState.initial(600, rank_init=2))
    assert isinstance(th, np.ndarray) and np.isfinite(th).all()
    assert st1.step == 1 and st1.u_prev.shape[1] >= 1
