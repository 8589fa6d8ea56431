"""BASELINE configs[4] semantics at reduced size on one GPU: exponential averaging of the low-rank
history (delta = 0.95, the k history rows are streamed next to the new samples) with k = 256
(the largest rank: k x k kernels leave shared memory), closed loop vs the CPU oracle."""

import numpy as np
import pytest

from conftest import rel, subspace_sine

pytestmark = pytest.mark.gpu


def test_history_delta095_k256_matches_oracle():
    import torch

    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import estimators, optimizers, synthetic

    cfg = synthetic.config("c4", N=1024, P=16384, k=256, L=512)
    P, N, k = cfg["P"], cfg["N"], cfg["k"]
    wl = synthetic.HostWorkload.from_config(cfg, 4)
    ost = orc.baseline_state(P, k, wl.v0_raw(), cfg["delta"], cfg["lam"])
    st = optimizers.WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=ost.u_prev,
                              r_max=k, delta=cfg["delta"], sigma_floor=cfg["lam"], eps_grow=0.0,
                              step=1)
    for t in range(3):
        o, e = wl.next()
        b = orc.assemble(o, e)
        _, ost, info = orc.wssr_step(np.zeros(P), b["o_matrix"], b["l_vector"], 1.0, ost)
        bundle = estimators.assemble(estimators.SampleBatch((None,) * N, e, o))
        _, st, diag, upd = optimizers.wssr_step(np.zeros(P), bundle, 1.0, st, return_update=True)
        assert diag.effective_rank == info["r_eff"]
        assert diag.ssi.iterations_used == info["iterations"]
        assert rel(upd.cpu().numpy(), info["update"]) < 1e-10, t
        sig = torch.linalg.vector_norm(st.obar, dim=0).cpu().numpy()
        assert rel(sig, info["sigma"]) < 1e-9, t
        assert subspace_sine(st.u_prev.cpu().numpy(), ost.u_prev) < 1e-8, t
        assert rel(st.lbar.cpu().numpy(), ost.lbar) < 1e-8, t
        np.testing.assert_allclose(diag.projector_drift, info["projector_drift"], rtol=1e-6,
                                   atol=1e-13)
