"""Parity at the benchmark configuration (BASELINE configs[1], c1: N=4096, P=131072, k=64):
two closed-loop WSSR steps through the C ABI vs the CPU oracle on the same seeded host inputs.
Slow (~1-2 min on the GPU box: 4.3 GB of host data and two 16-core oracle steps)."""

import numpy as np
import pytest

from conftest import rel, subspace_sine

pytestmark = pytest.mark.gpu


def test_c1_two_steps_match_oracle():
    import torch

    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import estimators, optimizers, synthetic

    cfg = synthetic.config("c1")
    P, N, k = cfg["P"], cfg["N"], cfg["k"]
    wl = synthetic.HostWorkload.from_config(cfg, 1)
    v0_raw = wl.v0_raw()
    ost = orc.baseline_state(P, k, v0_raw, cfg["delta"], cfg["lam"])
    dev = torch.device("cuda")
    st = optimizers.WssrState(obar=torch.zeros(0, P, dtype=torch.float64, device=dev).t(),
                              lbar=torch.zeros(0, dtype=torch.float64, device=dev),
                              u_prev=torch.as_tensor(ost.u_prev, device=dev), r_max=k,
                              delta=cfg["delta"], sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
    for t in range(2):
        o, e = wl.next()
        b = orc.assemble(o, e)
        _, ost, info = orc.wssr_step(np.zeros(P), b["o_matrix"], b["l_vector"], 1.0, ost)
        del b
        bundle = estimators.assemble(estimators.SampleBatch((None,) * N, e, o))
        _, st, diag, upd = optimizers.wssr_step(torch.zeros(P, dtype=torch.float64, device=dev),
                                                bundle, 1.0, st, return_update=True)
        assert diag.effective_rank == info["r_eff"] == k
        assert diag.ssi.iterations_used == info["iterations"]
        assert rel(upd.cpu().numpy(), info["update"]) < 1e-10, t
        sig = torch.linalg.vector_norm(st.obar, dim=0).cpu().numpy()
        assert rel(sig, info["sigma"]) < 1e-9, t
        assert subspace_sine(st.u_prev.cpu().numpy(), ost.u_prev) < 1e-8, t
        np.testing.assert_allclose(diag.ssi.subspace_residual, info["residual"], rtol=1e-6)
        np.testing.assert_allclose(diag.projector_drift, info["projector_drift"], rtol=1e-6,
                                   atol=1e-13)
        del bundle
