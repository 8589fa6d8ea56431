"""Parity at scale and over the full horizons (VERDICT r1 "next" item 2).

* The torch-FP64 transliteration (tests/fp64_transliteration.py: cuBLAS DGEMM + cuSOLVER QR, no
  libwssr code) is first pinned to the CPU oracle: c0 for 5 closed-loop steps and one full c1
  step, to ~1e-12.
* It then stands in for the oracle where the CPU cannot go:
  - c1 (N=4096, P=131072, k=64) closed loop over BASELINE's full horizon T=50;
  - c2 (N=16384, P=2^20, k=128, 137 GB of FP64 samples) and c3 (the same in float32) at full
    size, 3 closed-loop steps each, on the production path (int8 tensor-core O-passes with digit
    planes where they fit, on-the-fly digits for the rest).
Every step asserts the north_star tolerances: update <= 1e-10 relative L2, sigma <= 1e-9
relative, subspace sine <= 1e-8, and identical iterations_used and effective rank.
"""

import numpy as np
import pytest

from conftest import rel, subspace_sine

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

UPD_TOL, SIG_TOL, SINE_TOL = 1e-10, 1e-9, 1e-8


def _t_sine(a, b):
    """largest principal-angle sine between two orthonormal column blocks (on the device)."""
    m = b - a @ (a.t() @ b)
    ev = torch.linalg.eigvalsh(m.t() @ m)
    return float(ev[-1].clamp_min(0.0).sqrt())


def _t_rel(a, b):
    return float(torch.linalg.vector_norm(a - b) / torch.linalg.vector_norm(b))


def _ours_state(v0, cfg):
    from paper_2512_05749_b200 import optimizers

    P = v0.shape[0]
    return optimizers.WssrState(obar=torch.zeros(0, P, dtype=torch.float64,
                                                 device=v0.device).t(),
                                lbar=torch.zeros(0, dtype=torch.float64, device=v0.device),
                                u_prev=v0, r_max=cfg["k"], delta=cfg["delta"],
                                sigma_floor=cfg["lam"], eps_grow=0.0, step=1)


def _ours_step(O, E, st):
    from paper_2512_05749_b200 import estimators, optimizers

    P = O.shape[1]
    bundle = estimators.assemble(estimators.SampleBatch((None,) * O.shape[0], E, O))
    _, st1, diag, upd = optimizers.wssr_step(torch.zeros(P, dtype=torch.float64,
                                                         device=O.device),
                                             bundle, 1.0, st, return_update=True)
    sig = torch.linalg.vector_norm(st1.obar, dim=0)
    return st1, diag, upd, sig


def test_transliteration_pinned_to_oracle_c0():
    import fp64_transliteration as t64
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import synthetic

    cfg = synthetic.config("c0")
    P, k = cfg["P"], cfg["k"]
    wl = synthetic.HostWorkload.from_config(cfg, 0)
    v0_raw = wl.v0_raw()
    ost = orc.baseline_state(P, k, v0_raw, cfg["delta"], cfg["lam"])
    tst = t64.baseline_state(torch.as_tensor(ost.u_prev, device="cuda"), k, cfg["delta"],
                             cfg["lam"])
    for t in range(5):
        o, e = wl.next()
        b = orc.assemble(o, e)
        _, ost, info = orc.wssr_step(np.zeros(P), b["o_matrix"], b["l_vector"], 1.0, ost)
        S, lv, _ = t64.assemble(torch.as_tensor(o, device="cuda"), torch.as_tensor(e,
                                                                                device="cuda"))
        _, tst, tinfo = t64.wssr_step(torch.zeros(P, dtype=torch.float64, device="cuda"), S, lv,
                                      1.0, tst)
        assert tinfo["iterations"] == info["iterations"] and tinfo["r_eff"] == info["r_eff"]
        assert rel(tinfo["update"].cpu().numpy(), info["update"]) < 1e-12, t
        assert rel(tinfo["sigma"].cpu().numpy(), info["sigma"]) < 1e-12, t
        assert subspace_sine(tst.u_prev.cpu().numpy(), ost.u_prev) < 1e-10, t
        np.testing.assert_allclose(tinfo["projector_drift"], info["projector_drift"],
                                   rtol=1e-8, atol=1e-14)


def test_transliteration_pinned_to_oracle_c1():
    import fp64_transliteration as t64
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import synthetic

    cfg = synthetic.config("c1")
    P, k = cfg["P"], cfg["k"]
    wl = synthetic.HostWorkload.from_config(cfg, 1)
    ost = orc.baseline_state(P, k, wl.v0_raw(), cfg["delta"], cfg["lam"])
    tst = t64.baseline_state(torch.as_tensor(ost.u_prev, device="cuda"), k, cfg["delta"],
                             cfg["lam"])
    o, e = wl.next()
    b = orc.assemble(o, e)
    _, ost, info = orc.wssr_step(np.zeros(P), b["o_matrix"], b["l_vector"], 1.0, ost)
    del b
    S, lv, _ = t64.assemble(torch.as_tensor(o, device="cuda"), torch.as_tensor(e, device="cuda"))
    _, tst, tinfo = t64.wssr_step(torch.zeros(P, dtype=torch.float64, device="cuda"), S, lv, 1.0,
                                  tst)
    assert tinfo["iterations"] == info["iterations"] and tinfo["r_eff"] == info["r_eff"]
    assert rel(tinfo["update"].cpu().numpy(), info["update"]) < 1e-12
    assert rel(tinfo["sigma"].cpu().numpy(), info["sigma"]) < 1e-12
    assert subspace_sine(tst.u_prev.cpu().numpy(), ost.u_prev) < 1e-10


def _closed_loop(cfg, steps, seed, dtype=torch.float64, tag="", tol=None):
    import fp64_transliteration as t64
    from paper_2512_05749_b200 import linalg, synthetic

    N, P, k = cfg["N"], cfg["P"], cfg["k"]
    wl = synthetic.DeviceWorkload(N, P, k, cfg["L"], cfg["alpha"], cfg["drift"], seed=seed,
                                  device=torch.device("cuda"), dtype=dtype)
    v0 = linalg.qr_orthonormalize(wl.v0_raw())[0].as_subclass(torch.Tensor)
    st = _ours_state(v0, cfg)
    tst = t64.baseline_state(v0.clone(), k, cfg["delta"], cfg["lam"])
    worst = [0.0, 0.0, 0.0]
    for t in range(steps):
        O, E = wl.next()
        st, diag, upd, sig = _ours_step(O, E, st)
        S, lv, _ = t64.assemble(O, E)
        _, tst, tinfo = t64.wssr_step(torch.zeros(P, dtype=torch.float64, device="cuda"), S, lv,
                                      1.0, tst)
        del S
        assert diag.ssi.iterations_used == tinfo["iterations"], (tag, t)
        assert diag.effective_rank == tinfo["r_eff"], (tag, t)
        e_upd = _t_rel(upd, tinfo["update"])
        e_sig = _t_rel(sig, tinfo["sigma"])
        e_sin = _t_sine(tst.u_prev, st.u_prev)
        worst = [max(worst[0], e_upd), max(worst[1], e_sig), max(worst[2], e_sin)]
        tu, ts, tn = (UPD_TOL, SIG_TOL, SINE_TOL) if tol is None else (
            tol["update"], tol["sigma"], tol["sine"])
        assert e_upd < tu and e_sig < ts and e_sin < tn, (tag, t, e_upd, e_sig, e_sin)
        np.testing.assert_allclose(diag.ssi.subspace_residual, tinfo["residual"], rtol=1e-6)
        np.testing.assert_allclose(diag.projector_drift, tinfo["projector_drift"], rtol=1e-6,
                                   atol=1e-12)
    print(f"{tag}: {steps} closed-loop steps vs torch FP64: worst update {worst[0]:.2e}, "
          f"sigma {worst[1]:.2e}, sine {worst[2]:.2e}")
    return worst


def test_c1_full_horizon_T50_vs_transliteration():
    from paper_2512_05749_b200 import synthetic

    cfg = synthetic.config("c1")
    _closed_loop(cfg, cfg["T"], seed=101, tag="c1 T=50")


def _need_big_gpu():
    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a 180 GB B200")


def _release():
    import gc

    from paper_2512_05749_b200 import _lib

    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # return the 69-137 GB sample block to the driver
    _lib.context().call("wssr_release_memory")  # and the engine's planes / scratch reserve


@pytest.fixture
def release_memory():
    _release()  # earlier tests may have left the engine's digit planes at their largest
    yield
    _release()


def test_c2_full_size_three_steps_vs_transliteration(release_memory, monkeypatch):
    from paper_2512_05749_b200 import synthetic

    _need_big_gpu()
    # the transliteration's own P x k temporaries need room next to the 137 GB block: cap the
    # engine's digit planes at 4096 samples (the rest is digitised on the fly, as at full c2)
    monkeypatch.setenv("WSSR_OZ_PLANE_ROWS", "4096")
    _closed_loop(synthetic.config("c2"), 3, seed=202, tag="c2")


def test_c3_full_size_three_steps_vs_transliteration(release_memory, monkeypatch, fp32_digits):
    from conftest import F32_DIGIT_TOL
    from paper_2512_05749_b200 import synthetic

    _need_big_gpu()
    if fp32_digits == 7:  # the 7-byte planes of all samples do not fit beside O and the test's
        monkeypatch.setenv("WSSR_OZ_PLANE_ROWS", "8192")  # own temporaries: half of them
    _closed_loop(synthetic.config("c3"), 3, seed=303, dtype=torch.float32,
                 tag=f"c3 ({fp32_digits} digits)", tol=F32_DIGIT_TOL[fp32_digits])


def test_c4_semantics_slice_T10_vs_transliteration(release_memory):
    """BASELINE configs[4] semantics (k=256, history averaging delta=0.95, latent rank 512,
    alpha=0.8, drift 5e-4) over its full horizon T=10, on a one-GPU slice of its shape: all
    N=32768 samples with P reduced to 2^18 (68.7 GB; the full 550 GB block is an 8-GPU
    configuration)."""
    from paper_2512_05749_b200 import synthetic

    _need_big_gpu()
    cfg = synthetic.config("c4", P=262144)
    _closed_loop(cfg, cfg["T"], seed=404, tag="c4 slice T=10")


def test_c4_full_width_rank_shard_vs_transliteration(release_memory):
    """BASELINE configs[4] at its full width and rank (P = 2^21 parameters, k = 256, history
    averaging delta = 0.95) on the sample rows one GPU can hold next to the independent FP64
    transliteration's own copy: N = 2048 of c4's 32768 walkers (34 GB; an 8-way rank holds
    4096), three closed-loop steps so the P x 256 history block is live from the second one."""
    from paper_2512_05749_b200 import synthetic

    _need_big_gpu()
    cfg = synthetic.config("c4", N=2048)
    _closed_loop(cfg, 3, seed=405, tag="c4 full width, N=2048")
