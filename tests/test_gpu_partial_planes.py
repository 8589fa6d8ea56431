"""Digit planes for only part of the sample block (c2/c3, where the 7-byte planes of all samples
do not fit next to O): the first rows stream pre-digitised planes, the rest is digitised on the
fly in every pass (v pass: disjoint output rows; u pass: the second part accumulates).  Forced
here with WSSR_OZ_PLANE_ROWS on small shapes and checked against the CPU oracle and the
all-planes run."""

import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _step(cfg, o, e, v0):
    from paper_2512_05749_b200 import estimators, optimizers

    st = optimizers.WssrState(obar=np.zeros((cfg["P"], 0)), lbar=np.zeros(0), u_prev=v0,
                              r_max=cfg["k"], delta=0.0, sigma_floor=cfg["lam"], eps_grow=0.0,
                              step=1)
    b = estimators.assemble(estimators.SampleBatch((None,) * cfg["N"], e, o))
    _, st1, diag, upd = optimizers.wssr_step(np.zeros(cfg["P"]), b, 1.0, st, return_update=True)
    return (upd.cpu().numpy(), torch.linalg.vector_norm(st1.obar, dim=0).cpu().numpy(), diag)


@pytest.mark.parametrize("rows_cap", [0, 128, 384])
@pytest.mark.parametrize("f32", [False, True])
def test_partial_planes_match_oracle(rows_cap, f32):
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import _lib, synthetic

    cfg = synthetic.config("c0", N=640, P=4096, k=32, L=64, delta=0.0, lam=1e-3)
    wl = synthetic.HostWorkload.from_config(cfg, 5)
    o, e = wl.next()
    if f32:
        o = o.astype(np.float32)
    v0 = orc.qr_pos(wl.v0_raw())[0]
    ref_b = orc.assemble(o.astype(np.float64), e)
    ost = orc.baseline_state(cfg["P"], cfg["k"], wl.v0_raw(), 0.0, cfg["lam"])
    _, _, info = orc.wssr_step(np.zeros(cfg["P"]), ref_b["o_matrix"], ref_b["l_vector"], 1.0,
                               ost)
    ctx = _lib.context()
    ctx.lib.wssr_set_gemm_path(ctx.handle, 3)  # int8 tensor-core O-passes at this size
    old = os.environ.get("WSSR_OZ_PLANE_ROWS")
    try:
        os.environ["WSSR_OZ_PLANE_ROWS"] = str(rows_cap)
        upd, sig, diag = _step(cfg, o, e, v0)
        del os.environ["WSSR_OZ_PLANE_ROWS"]
        upd_full, sig_full, _ = _step(cfg, o, e, v0)
    finally:
        if old is not None:
            os.environ["WSSR_OZ_PLANE_ROWS"] = old
        ctx.lib.wssr_set_gemm_path(ctx.handle, 0)
    tol = 1e-4 if f32 else 1e-10
    assert rel(upd, info["update"]) < tol
    assert rel(sig, info["sigma"]) < (1e-6 if f32 else 1e-9)
    assert diag.effective_rank == info["r_eff"]
    assert rel(upd, upd_full) < 1e-12 and rel(sig, sig_full) < 1e-13
