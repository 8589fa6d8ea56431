"""The host-checked ("careful") SSI: every QR checked on the host and the reference's
Gram-Schmidt-with-patch branch (linalg.py:64-105) taken where CholeskyQR2 cannot resolve the
block - the path with_fallback re-runs after a flagged CholeskyQR2.  Checked against the CPU
oracle on a generic input (the same answers as the optimistic path) and on an exactly
rank-deficient one (the patch columns of the reference)."""

import numpy as np
import pytest

from conftest import rel, subspace_sine

pytestmark = pytest.mark.gpu


def _ohat(rng, m, n, rank, noise):
    a = rng.standard_normal((m, rank)) @ np.diag(np.arange(1, rank + 1) ** -1.0) @ \
        rng.standard_normal((rank, n))
    return a + noise * rng.standard_normal((m, n))


@pytest.mark.parametrize("careful", [False, True])
def test_careful_ssi_matches_oracle_generic(careful):
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import ssi_svd

    rng = np.random.default_rng(31)
    oh = _ohat(rng, 3000, 400, 40, 1e-3)
    u0 = orc.qr_pos(rng.standard_normal((3000, 16)))[0]
    ref = orc.ssi(oh, 16, max_iters=3, u_init=u0)
    f, rep = ssi_svd(oh, 16, max_iters=3, u_init=u0, _careful=careful)
    assert rep.iterations_used == ref["iterations"]
    assert rel(f.sigma.cpu().numpy(), ref["sigma"]) < 1e-9
    assert subspace_sine(f.u.cpu().numpy(), ref["u"]) < 1e-8


def test_careful_ssi_rank_deficient_matches_oracle():
    """Exact rank 5 < k = 8: the QRs of u meet the reference's deficiency rule, and the
    careful path fills the missing columns canonically like the reference does."""
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import ssi_svd

    rng = np.random.default_rng(32)
    oh = _ohat(rng, 600, 120, 5, 0.0)
    u0 = orc.qr_pos(rng.standard_normal((600, 8)))[0]
    ref = orc.ssi(oh, 8, max_iters=3, u_init=u0)
    f, rep = ssi_svd(oh, 8, max_iters=3, u_init=u0, _careful=True)
    k = len(ref["sigma"])
    assert f.sigma.shape[0] == k
    assert rel(f.sigma.cpu().numpy(), ref["sigma"]) < 1e-9
    top = int(np.sum(ref["sigma"] > 1e-8 * ref["sigma"][0]))
    assert subspace_sine(f.u.cpu().numpy()[:, :top], ref["u"][:, :top]) < 1e-8


def test_optimistic_path_falls_back_on_rank_deficiency():
    """Without the flag the step runs CholeskyQR2 optimistically; the flagged block makes it
    re-run in careful mode (with_fallback), so the answer equals the careful one bit for bit."""
    import torch

    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200.svdengine import ssi_svd

    rng = np.random.default_rng(32)
    oh = _ohat(rng, 600, 120, 5, 0.0)
    u0 = orc.qr_pos(rng.standard_normal((600, 8)))[0]
    fa, _ = ssi_svd(oh, 8, max_iters=3, u_init=u0)
    fb, _ = ssi_svd(oh, 8, max_iters=3, u_init=u0, _careful=True)
    assert torch.equal(fa.sigma, fb.sigma) and torch.equal(fa.u, fb.u)


@pytest.mark.parametrize("careful_rank,k", [(5, 8), (3, 16)])
def test_step_on_rank_deficient_batch_matches_oracle(careful_rank, k):
    """A whole WSSR step (assemble + wssr_step) on a batch whose centred O has exact rank
    below k: the step's optimistic SSI flags the QR of the iterate, re-runs carefully, and the
    update, sigma and r_eff match the oracle replaying the reference's patch path."""
    import torch

    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import estimators, optimizers

    rng = np.random.default_rng(40 + careful_rank)
    n, p = 48, 320
    o = rng.standard_normal((n, careful_rank)) @ rng.standard_normal((careful_rank, p)) + \
        rng.standard_normal(p)[None, :]
    e = -1.0 + 0.1 * rng.standard_normal(n)
    u0 = orc.qr_pos(rng.standard_normal((p, k)))[0]
    b = orc.assemble(o, e)
    # g lies in the span of O exactly, so the floor term (g - U U^T g) / lambda is pure rounding;
    # lambda = 1 keeps it from dominating the comparison (with 1e-3 it is ~1e-10 of the update)
    st = orc.State(obar=np.zeros((p, 0)), lbar=np.zeros(0), u_prev=u0, r_max=k, delta=0.0,
                   sigma_floor=1.0, r_reg=1e-6, eps_grow=0.0, step=1)
    _, ost, info = orc.wssr_step(np.zeros(p), b["o_matrix"], b["l_vector"], 1.0, st)

    dev = torch.device("cuda")
    dst = optimizers.WssrState(obar=torch.zeros(0, p, dtype=torch.float64, device=dev).t(),
                               lbar=torch.zeros(0, dtype=torch.float64, device=dev),
                               u_prev=torch.as_tensor(u0, device=dev), r_max=k, delta=0.0,
                               sigma_floor=1.0, r_reg=1e-6, eps_grow=0.0, step=1)
    bundle = estimators.assemble(estimators.SampleBatch((None,) * n, e, o))
    _, nst, diag, upd = optimizers.wssr_step(torch.zeros(p, dtype=torch.float64, device=dev),
                                             bundle, 1.0, dst, return_update=True)
    assert diag.effective_rank == info["r_eff"] == careful_rank
    assert diag.ssi.iterations_used == info["iterations"]
    err = rel(upd.cpu().numpy(), info["update"])
    print(f"update rel err {err:.2e}")
    assert err < 1e-10
    sig = torch.linalg.vector_norm(nst.obar, dim=0).cpu().numpy()
    assert rel(sig, info["sigma"]) < 1e-9
    assert subspace_sine(nst.u_prev.cpu().numpy(), ost.u_prev) < 1e-8
