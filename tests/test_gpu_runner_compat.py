"""The reference runner's use of the step, replayed with the drop-in (runner.py:284-351): numpy
batches in, the NaN guards on bundle.raw_loss and theta' (runner.py:293-300), set_theta on a
numpy theta (runner.py:314), the trace fields from WssrDiagnostics (runner.py:322-347), the
snapshot through np.asarray of the state arrays (runner.py:145-157 + checkpoint.py:45) and the
resume (runner.py:203-216).  Outputs are checked against the CPU oracle on the same inputs, and
the resumed run against the uninterrupted one bit for bit (test_runner.py:109-126)."""

import dataclasses

import numpy as np
import pytest

from conftest import rel, subspace_sine
from oracle import wssr_oracle as orc
from paper_2512_05749_b200 import synthetic

pytestmark = pytest.mark.gpu


class FakeWavefunction:
    """set_theta / log_abs_batch as the runner calls them (runner.py:314-317)."""

    def __init__(self, P):
        self.theta = np.zeros(P)

    def set_theta(self, theta):
        assert isinstance(theta, np.ndarray) and theta.dtype == np.float64
        self.theta = theta.copy()

    def log_abs_batch(self, positions):
        return np.zeros(len(positions))


def _state_arrays(opt_state):
    # what the reference's write_checkpoint does with them (checkpoint.py:45, 49)
    return {name: np.ascontiguousarray(np.asarray(getattr(opt_state, key)))
            for name, key in (("wssr_obar", "obar"), ("wssr_lbar", "lbar"),
                              ("wssr_u_prev", "u_prev"))}


def _replay(cfg, batches, v0, start=None):
    from paper_2512_05749_b200.estimators import SampleBatch, assemble
    from paper_2512_05749_b200.optimizers import WssrState, wssr_step

    P = cfg["P"]
    if start is None:
        theta = np.zeros(P)
        opt_state = WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=v0, r_max=cfg["k"],
                              delta=cfg["delta"], sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
    else:
        theta, opt_state = start
    wf = FakeWavefunction(P)
    records, snaps = [], []
    for o, e in batches:
        batch = SampleBatch((None,) * o.shape[0], e, o)
        bundle = assemble(batch, clip_n_std=5.0)
        assert np.isfinite(bundle.raw_loss)                                  # runner.py:293
        theta_next, opt_state_next, diag = wssr_step(theta, bundle, 0.5, opt_state,
                                                     svd_backend="ssi", ssi_max_iters=3,
                                                     ssi_residual_tol=1e-10, rng_seed=7)
        assert np.all(np.isfinite(theta_next))                               # runner.py:299
        theta, opt_state = theta_next, opt_state_next
        wf.set_theta(theta)                                                  # runner.py:314
        records.append(dict(raw_energy=bundle.raw_loss, clipped_energy=bundle.loss,
                            energy_variance=float(np.var(batch.local_energies)),
                            effective_rank=diag.effective_rank, r_max=diag.r_max,
                            ssi_iterations=diag.ssi.iterations_used,
                            sigma_drift=diag.sigma_drift, projector_drift=diag.projector_drift))
        snaps.append((theta.copy(), _state_arrays(opt_state), dict(
            delta=opt_state.delta, sigma_floor=opt_state.sigma_floor,
            sigma_floor_relative=opt_state.sigma_floor_relative, r_reg=opt_state.r_reg,
            eps_grow=opt_state.eps_grow, r_max=opt_state.r_max, step=opt_state.step)))
    return theta, opt_state, records, snaps


def test_runner_loop_replay_matches_oracle_and_resumes_bitwise(tmp_path):
    from paper_2512_05749_b200 import checkpoint
    from paper_2512_05749_b200.optimizers import WssrState

    cfg = synthetic.config("c0", N=256, P=2048, k=12, L=24, delta=0.9, lam=1e-3)
    wl = synthetic.HostWorkload.from_config(cfg, 11)
    v0 = orc.qr_pos(wl.v0_raw())[0]
    batches = [tuple(np.array(x) for x in wl.next()) for _ in range(4)]
    theta, st, records, snaps = _replay(cfg, batches, v0)

    # oracle on the same inputs
    ost = orc.State(obar=np.zeros((cfg["P"], 0)), lbar=np.zeros(0), u_prev=v0, r_max=cfg["k"],
                    delta=cfg["delta"], sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
    oth = np.zeros(cfg["P"])
    for (o, e), rec in zip(batches, records):
        b = orc.assemble(o, e)
        oth, ost, info = orc.wssr_step(oth, b["o_matrix"], b["l_vector"], 0.5, ost, rng_seed=7)
        assert rec["effective_rank"] == info["r_eff"]
        assert rec["ssi_iterations"] == info["iterations"]
        np.testing.assert_allclose([rec["raw_energy"], rec["clipped_energy"]],
                                   [b["raw_loss"], b["loss"]], rtol=1e-13)
        np.testing.assert_allclose([rec["sigma_drift"], rec["projector_drift"]],
                                   [info["sigma_drift"], info["projector_drift"]], rtol=1e-6,
                                   atol=1e-13)
    assert rel(theta, oth) < 1e-10
    assert subspace_sine(np.asarray(st.u_prev), ost.u_prev) < 1e-8

    # snapshot after step 2 in the reference format from numpy arrays, restore, continue
    th2, arrays2, scal2 = snaps[1]
    path = tmp_path / "run.wssr"
    checkpoint.write_checkpoint(path, {"wssr": scal2}, {"theta": th2, **arrays2}, [])
    s, a, _ = checkpoint.read_checkpoint(path)
    w = s["wssr"]
    restored = WssrState(obar=a["wssr_obar"], lbar=a["wssr_lbar"], u_prev=a["wssr_u_prev"],
                         r_max=int(w["r_max"]), delta=float(w["delta"]),
                         sigma_floor=float(w["sigma_floor"]),
                         sigma_floor_relative=bool(w["sigma_floor_relative"]),
                         r_reg=float(w["r_reg"]), eps_grow=float(w["eps_grow"]),
                         step=int(w["step"]))
    theta_r, st_r, _, _ = _replay(cfg, batches[2:], v0, start=(a["theta"], restored))
    np.testing.assert_array_equal(theta_r, theta)
    np.testing.assert_array_equal(np.asarray(st_r.u_prev), np.asarray(st.u_prev))


def test_dataclass_contract_of_the_step_outputs():
    """Frozen dataclasses with the reference's field names (estimators.py:34-50,
    optimizers.py:188-258, svdengine.py:20-53)."""
    from paper_2512_05749_b200.estimators import EstimatorBundle, SampleBatch, assemble
    from paper_2512_05749_b200.optimizers import WssrDiagnostics, WssrState, wssr_step
    from paper_2512_05749_b200.svdengine import SsiReport, TruncatedSvd

    names = lambda c: [f.name for f in dataclasses.fields(c)]  # noqa: E731
    assert names(EstimatorBundle) == ["loss", "raw_loss", "o_matrix", "l_vector", "gradient"]
    assert names(WssrDiagnostics) == ["ssi", "effective_rank", "r_max", "sigma_drift",
                                      "projector_drift"]
    assert names(SsiReport) == ["iterations_used", "subspace_residual", "warm_started"]
    assert names(TruncatedSvd) == ["u", "sigma", "v"]
    cfg = synthetic.config("c0", N=64, P=256, k=6, L=8)
    wl = synthetic.HostWorkload.from_config(cfg, 3)
    o, e = wl.next()
    b = assemble(SampleBatch((None,) * 64, e, o))
    st = WssrState(obar=np.zeros((256, 0)), lbar=np.zeros(0),
                   u_prev=orc.qr_pos(wl.v0_raw())[0], r_max=6, step=1)
    th, st1, diag = wssr_step(np.zeros(256), b, 1.0, st)
    with pytest.raises(dataclasses.FrozenInstanceError):
        diag.r_max = 3
    with pytest.raises(dataclasses.FrozenInstanceError):
        b.loss = 0.0
    d = dataclasses.asdict(diag)
    assert d["ssi"]["warm_started"] is True and d["sigma_drift"] == diag.sigma_drift
    assert dataclasses.replace(diag, r_max=99).r_max == 99
    b2 = dataclasses.replace(b, loss=1.5)
    assert b2.loss == 1.5 and b2.raw_loss == b.raw_loss
    np.testing.assert_allclose(np.asarray(b2.o_matrix), np.asarray(b.o_matrix))
    ref = orc.assemble(o, e)
    np.testing.assert_allclose(np.asarray(b.o_matrix), ref["o_matrix"], atol=1e-15)
    assert isinstance(np.asarray(st1.obar), np.ndarray)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_large_host_arrays_upload_through_the_pinned_pipeline(dtype, monkeypatch):
    """numpy blocks above 256 MB (the runner's per-step sample block) go up in pinned chunks
    (_arrays._upload_pipelined): same bytes as the direct copy, for sizes that are not a multiple
    of the staging buffer, read-only arrays, and back-to-back calls reusing the buffers."""
    import torch

    from paper_2512_05749_b200 import _arrays

    monkeypatch.setattr(_arrays, "_STAGE_BYTES", 8 << 20)
    monkeypatch.setattr(_arrays, "_PIPELINE_MIN_BYTES", 16 << 20)
    monkeypatch.setattr(_arrays, "_stage_local", __import__("threading").local())
    rng = np.random.default_rng(3)
    for rows, cols in ((1031, 4099), (2048, 4096)):
        a = rng.standard_normal((rows, cols)).astype(dtype)
        a.setflags(write=False)
        t = _arrays.to_tensor_f64_or_f32(a)
        b = _arrays.to_tensor_f64_or_f32(a[::-1])  # a second upload right behind the first
        assert t.dtype == (torch.float64 if dtype == np.float64 else torch.float32)
        assert t.shape == a.shape and t.is_cuda
        assert np.array_equal(t.cpu().numpy(), a)
        assert np.array_equal(b.cpu().numpy(), a[::-1])
    small = rng.standard_normal((8, 8))
    assert np.array_equal(_arrays.to_tensor(small).cpu().numpy(), small)
