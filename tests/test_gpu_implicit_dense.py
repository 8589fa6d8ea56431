"""Dense first step without forming Ohat (optimizers.py:327-330 -> svdengine.py:75-85, LAPACK's
dgesdd in the reference): the engine's implicit exact truncated SVD (engine.cu implicit_svd:
oversampled block power iteration on the O-pass kernels + Rayleigh-Ritz of the small global
block), which the drop-in takes when Ohat would not fit beside the samples, for float32 samples
and under row sharding.  Checked against numpy's LAPACK SVD of the same matrix at the north_star
tolerances, and against the materialising device path."""

import numpy as np
import pytest

from conftest import rel, subspace_sine
from test_gpu_dense_large import _step0_reference

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture
def implicit(monkeypatch):
    monkeypatch.setenv("WSSR_DENSE_STEP", "implicit")


def _step0(o, e, k, lam, theta=None, dtype=None):
    from paper_2512_05749_b200 import estimators, optimizers

    N, P = o.shape
    st = optimizers.WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=np.zeros((P, 0)),
                              r_max=k, delta=0.0, sigma_floor=lam, eps_grow=0.0, step=0)
    od = torch.from_numpy(o).cuda()
    if dtype is not None:
        od = od.to(dtype)
    b = estimators.assemble(estimators.SampleBatch((None,) * N, e, od))
    _, st1, diag, upd = optimizers.wssr_step(np.zeros(P), b, 1.0, st, return_update=True)
    return st1, diag, upd.cpu().numpy()


def _check(st1, diag, upd, ref):
    ref_upd, u, s, r = ref
    assert diag.effective_rank == r
    assert rel(upd, ref_upd) < 1e-10
    assert rel(torch.linalg.vector_norm(st1.obar, dim=0).cpu().numpy(), s) < 1e-9
    assert subspace_sine(st1.u_prev.cpu().numpy(), u) < 1e-8


@pytest.mark.parametrize("N,P,k,L", [(1024, 4096, 32, 64), (600, 2048, 16, 40), (96, 300, 12, 20),
                                     (200, 150, 40, 30)])
def test_implicit_step0_matches_lapack(implicit, N, P, k, L):
    """BASELINE configs[0]'s shape and smaller/ragged ones, including P < N (the block spans the
    whole column space) and more requested triplets than the latent rank."""
    rng = np.random.default_rng(N + P + k)
    o = rng.standard_normal((N, L)) @ np.diag(np.arange(1, L + 1) ** -1.0) @ \
        rng.standard_normal((L, P)) + 0.01 * rng.standard_normal((N, P))
    e = -1.0 + 0.1 * rng.standard_normal(N)
    lam = 1e-3
    st1, diag, upd = _step0(o, e, k, lam)
    _check(st1, diag, upd, _step0_reference(o, e, k, lam))


def test_implicit_step0_float32_samples():
    """float32 samples: the materialising path refuses them (dense backends need float64); the
    implicit one runs the O-passes on the stored float32 block (auto-selected)."""
    rng = np.random.default_rng(5)
    N, P, k, L = 512, 3000, 24, 48
    o = (rng.standard_normal((N, L)) @ np.diag(np.arange(1, L + 1) ** -1.0) @
         rng.standard_normal((L, P)) + 0.01 * rng.standard_normal((N, P))).astype(np.float32)
    e = -1.0 + 0.1 * rng.standard_normal(N)
    lam = 1e-3
    st1, diag, upd = _step0(o.astype(np.float64), e, k, lam, dtype=torch.float32)
    _check(st1, diag, upd, _step0_reference(o.astype(np.float64), e, k, lam))


def test_implicit_matches_materialised_exact_backend(monkeypatch):
    """The 'exact' backend at a later step (history rows scaled by sqrt(delta)): implicit and
    materialised device paths agree."""
    from paper_2512_05749_b200 import estimators, optimizers, synthetic

    cfg = synthetic.config("c0", N=256, P=1024, k=16, L=24, delta=0.7, lam=1e-3)
    wl = synthetic.HostWorkload.from_config(cfg, 2)
    st = optimizers.WssrState.initial(cfg["P"], rank_init=cfg["k"], delta=cfg["delta"],
                                      sigma_floor=cfg["lam"])
    o, e = wl.next()
    b = estimators.assemble(estimators.SampleBatch((None,) * cfg["N"], e, o))
    _, st, _ = optimizers.wssr_step(np.zeros(cfg["P"]), b, 1.0, st)
    o, e = wl.next()
    out = {}
    for mode in ("materialize", "implicit"):
        monkeypatch.setenv("WSSR_DENSE_STEP", mode)
        b = estimators.assemble(estimators.SampleBatch((None,) * cfg["N"], e, o))
        _, st1, diag, upd = optimizers.wssr_step(np.zeros(cfg["P"]), b, 1.0, st,
                                                 svd_backend="exact", return_update=True)
        out[mode] = (st1, diag, upd.cpu().numpy())
    a, c = out["materialize"], out["implicit"]
    assert a[1].effective_rank == c[1].effective_rank
    assert rel(c[2], a[2]) < 1e-10
    assert rel(optimizers.sigma_of(c[0]).cpu().numpy(),
               optimizers.sigma_of(a[0]).cpu().numpy()) < 1e-10
    ua, uc = a[0].u_prev.cpu().numpy(), c[0].u_prev.cpu().numpy()
    assert subspace_sine(uc, ua) < 1e-8
    # singular vector signs are arbitrary (LAPACK's too); lbar = V^T lhat flips with them
    sgn = np.sign(np.sum(ua * uc, axis=0))
    assert rel(c[0].lbar.cpu().numpy() * sgn, a[0].lbar.cpu().numpy()) < 1e-8


def test_implicit_rejects_zero_matrix(implicit):
    from paper_2512_05749_b200.errors import DegenerateInput

    N, P = 64, 128
    o = np.ones((N, P))  # centred: all zero
    e = -1.0 + 0.1 * np.random.default_rng(0).standard_normal(N)
    with pytest.raises(DegenerateInput):
        _step0(o, e, 4, 1e-3)


def test_c1_step0_implicit_against_lapack(implicit):
    """BASELINE configs[1] (N=4096, P=131072, k=64) from step 0 through the implicit path."""
    import time

    from paper_2512_05749_b200 import synthetic

    cfg = synthetic.config("c1")
    N, P, k, lam = cfg["N"], cfg["P"], cfg["k"], cfg["lam"]
    wl = synthetic.HostWorkload.from_config(cfg, 1)
    o, e = wl.next()
    t0 = time.perf_counter()
    st1, diag, upd = _step0(o, e, k, lam)
    t_dev = time.perf_counter() - t0
    ref = _step0_reference(o, e, k, lam)
    print(f"c1 step 0 (implicit): device {t_dev:.2f} s")
    _check(st1, diag, upd, ref)
