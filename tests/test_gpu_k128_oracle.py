"""k = 128 (the BASELINE c2/c3 rank) through the whole step against the CPU oracle: two
closed-loop steps at P = 65536 (so the P x k QRs, residuals and drift take the k = 128
tall-skinny kernels and the O-passes the int8 tensor-core path), with history averaging
(delta = 0.5) and FP64 and FP32 sample storage."""

import numpy as np
import pytest

from conftest import F32_DIGIT_TOL, rel, subspace_sine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("f32", [False, True])
def test_k128_two_steps_match_oracle(f32, fp32_digits):
    import torch

    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import _lib, estimators, optimizers, synthetic

    if not f32 and fp32_digits == 5:
        pytest.skip("the float32 digit mode does not apply to float64 samples")
    tol = F32_DIGIT_TOL[fp32_digits] if f32 else F32_DIGIT_TOL[7]
    cfg = synthetic.config("c2", N=1024, P=65536, k=128, L=192, delta=0.5, lam=1e-4)
    P, N, k = cfg["P"], cfg["N"], cfg["k"]
    wl = synthetic.HostWorkload.from_config(cfg, 12)
    v0_raw = wl.v0_raw()
    ost = orc.baseline_state(P, k, v0_raw, cfg["delta"], cfg["lam"])
    dev = torch.device("cuda")
    st = optimizers.WssrState(obar=torch.zeros(0, P, dtype=torch.float64, device=dev).t(),
                              lbar=torch.zeros(0, dtype=torch.float64, device=dev),
                              u_prev=torch.as_tensor(ost.u_prev, device=dev), r_max=k,
                              delta=cfg["delta"], sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
    ctx = _lib.context()
    ctx.lib.wssr_set_gemm_path(ctx.handle, 3)  # int8 O-passes at this size too
    try:
        for t in range(2):
            o, e = wl.next()
            if f32:
                o = o.astype(np.float32)
            b = orc.assemble(o.astype(np.float64), e)
            _, ost, info = orc.wssr_step(np.zeros(P), b["o_matrix"], b["l_vector"], 1.0, ost)
            bundle = estimators.assemble(estimators.SampleBatch((None,) * N, e, o))
            _, st, diag, upd = optimizers.wssr_step(
                torch.zeros(P, dtype=torch.float64, device=dev), bundle, 1.0, st,
                return_update=True)
            assert diag.effective_rank == info["r_eff"]
            assert diag.ssi.iterations_used == info["iterations"]
            e_upd = rel(upd.cpu().numpy(), info["update"])
            sig = torch.linalg.vector_norm(st.obar, dim=0).cpu().numpy()
            e_sig = rel(sig, info["sigma"])
            e_sin = subspace_sine(st.u_prev.cpu().numpy(), ost.u_prev)
            print(f"k128 f32={f32} digits={fp32_digits} step {t}: update {e_upd:.2e} "
                  f"sigma {e_sig:.2e} sine {e_sin:.2e}")
            assert e_upd < tol["update"] and e_sig < tol["sigma"] and e_sin < tol["sine"], t
            np.testing.assert_allclose(diag.projector_drift, info["projector_drift"], rtol=1e-6,
                                       atol=1e-13)
    finally:
        ctx.lib.wssr_set_gemm_path(ctx.handle, 0)
