"""Host-side logic that needs no GPU: WssrState construction and validation (the reference's
TestWssrState, test_optimizers.py:254-270), the WSSR snapshot round trip of a state
(runner.py:145-157, 203-216), the ctypes table against include/wssr.h, and the status-code to
exception mapping (the reference's error classes).  CPU-only."""

import os
import re

import numpy as np
import pytest
import torch


def test_initial_state_shape():
    from paper_2512_05749_b200.optimizers import WssrState

    st = WssrState.initial(7, rank_init=4)
    assert tuple(st.obar.shape) == (7, 0) and tuple(st.lbar.shape) == (0,)
    assert tuple(st.u_prev.shape) == (7, 0)
    assert st.r_max == 4 and st.step == 0


@pytest.mark.parametrize("kw", [dict(delta=1.0), dict(delta=-0.1), dict(r_reg=0.0),
                                dict(r_reg=1.0), dict(sigma_floor=0.0), dict(rank_init=0),
                                dict(eps_grow=-1.0)])
def test_initial_state_validation(kw):
    from paper_2512_05749_b200.optimizers import WssrState

    with pytest.raises(ValueError):
        WssrState.initial(3, **kw)


def test_state_shape_validation():
    from paper_2512_05749_b200.optimizers import WssrState

    z = np.zeros
    with pytest.raises(ValueError):
        WssrState(obar=z((5, 2)), lbar=z(3), u_prev=z((5, 2)), r_max=2)
    with pytest.raises(ValueError):
        WssrState(obar=z(5), lbar=z(2), u_prev=z((5, 2)), r_max=2)


def test_state_snapshot_round_trip(tmp_path):
    from paper_2512_05749_b200 import checkpoint
    from paper_2512_05749_b200.optimizers import WssrState

    rng = np.random.default_rng(3)
    f64 = dict(dtype=torch.float64)
    st = WssrState(obar=torch.tensor(rng.standard_normal((9, 3)), **f64),
                   lbar=torch.tensor(rng.standard_normal(3), **f64),
                   u_prev=torch.tensor(np.linalg.qr(rng.standard_normal((9, 3)))[0], **f64),
                   r_max=5, delta=0.9, sigma_floor=2e-3, sigma_floor_relative=True, r_reg=1e-7,
                   eps_grow=0.2, step=11)
    scalars, arrays = checkpoint.wssr_state_snapshot(st)
    assert set(arrays) == {"wssr_obar", "wssr_lbar", "wssr_u_prev"}
    path = tmp_path / "s.wssr"
    checkpoint.write_checkpoint(path, {"wssr": scalars}, arrays, [])
    s2, a2, _ = checkpoint.read_checkpoint(path)
    back = checkpoint.wssr_state_restore(s2["wssr"], a2, device=torch.device("cpu"))
    for name in ("delta", "sigma_floor", "sigma_floor_relative", "r_reg", "eps_grow", "r_max",
                 "step"):
        assert getattr(back, name) == getattr(st, name)
    for name in ("obar", "lbar", "u_prev"):
        assert torch.equal(getattr(back, name), getattr(st, name))


def test_ctypes_table_matches_header():
    """Every entry point the Python side binds is declared in include/wssr.h with the same
    number of parameters."""
    from paper_2512_05749_b200 import _lib

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "include", "wssr.h")) as fh:
        text = re.sub(r"/\*.*?\*/", "", fh.read(), flags=re.S)
    decls = {}
    for m in re.finditer(r"\b(wssr_\w+)\s*\(([^;{]*?)\)\s*;", text):
        args = m.group(2).strip()
        decls[m.group(1)] = 0 if args in ("", "void") else args.count(",") + 1
    for name, sig in _lib.SIGNATURES.items():
        assert name in decls, name
        argtypes = sig[1] if isinstance(sig, tuple) else sig
        assert len(argtypes) == decls[name], name


def test_status_codes_map_to_reference_errors():
    from paper_2512_05749_b200 import _lib, errors

    want = {1: ValueError, 2: errors.RankTooLarge, 3: errors.DegenerateInput,
            4: errors.ZeroMatrix, 5: errors.RankCollapse, 6: errors.DegenerateBatch,
            10: errors.NodeProximity}
    for code, exc in want.items():
        assert issubclass(_lib._STATUS[code], exc), code



def test_ace_spec_rejects_out_of_range_tables():
    """The producer indexes its tables on the device; AceSpec checks them on the host."""
    from collections import namedtuple

    from paper_2512_05749_b200.wavefunction import AceSpec

    Orb = namedtuple("Orb", "center n ell m spin zeta")
    orbs = [Orb(0, 0, 0, 0, "either", 1.0), Orb(0, 1, 1, 1, "up", 0.5)]
    nuc = np.zeros((1, 3))
    theta = np.zeros(2 * 2)
    cpu = torch.device("cpu")
    AceSpec(nuc, [0, 1], orbs, [(0, ()), (1, (0,))], theta, device=cpu)
    with pytest.raises(ValueError):
        AceSpec(nuc, [0, 1], orbs, [(0, ()), (2, (0,))], theta, device=cpu)
    with pytest.raises(ValueError):
        AceSpec(nuc, [0, 1], orbs, [(0, ()), (1, (5,))], theta, device=cpu)
    with pytest.raises(ValueError):
        AceSpec(nuc, [0, 1], [Orb(1, 0, 0, 0, "up", 1.0)] + orbs[1:], [(0, ()), (1, ())],
                theta, device=cpu)


def test_bundle_and_diagnostics_are_reference_dataclasses():
    """estimators.py:34-50 / optimizers.py:250-258: frozen dataclasses with the reference
    fields; the bundle's deferred scalars and lazy o_matrix behave as fields (CPU tensors)."""
    import dataclasses

    import torch

    from paper_2512_05749_b200.estimators import EstimatorBundle
    from paper_2512_05749_b200.optimizers import WssrDiagnostics
    from paper_2512_05749_b200.svdengine import SsiReport

    s = torch.tensor([[1.0, 2.0, 3.0], [3.0, 2.0, 1.0]], dtype=torch.float64)
    mu = s.mean(0)
    b = EstimatorBundle._assembled(1.0, 2.0, s, mu, 2 ** -0.5, 4.0, torch.zeros(2),
                                   torch.zeros(3), 2)
    assert [f.name for f in dataclasses.fields(b)] == ["loss", "raw_loss", "o_matrix",
                                                       "l_vector", "gradient"]
    np.testing.assert_allclose(np.asarray(b.o_matrix),
                               ((s - mu) * 2 ** -0.5).t().numpy())
    assert sorted(dataclasses.asdict(b)) == ["gradient", "l_vector", "loss", "o_matrix",
                                             "raw_loss"]
    with pytest.raises(dataclasses.FrozenInstanceError):
        b.raw_loss = 0.0
    assert "lazy" in repr(b)
    d = WssrDiagnostics(SsiReport(3, 1e-6, True), 4, 5, 0.25, 0.5)
    assert dataclasses.replace(d, effective_rank=2).effective_rank == 2
    assert dataclasses.asdict(d)["projector_drift"] == 0.5
    with pytest.raises(dataclasses.FrozenInstanceError):
        d.sigma_drift = 1.0

    class _Done:
        def synchronize(self):
            pass

    lazy = WssrDiagnostics._deferred(SsiReport(3, 1e-6, True), 4, 5, _Done(),
                                     torch.tensor([0.125, 0.75], dtype=torch.float64))
    assert (lazy.sigma_drift, lazy.projector_drift) == (0.125, 0.75)
    assert lazy == WssrDiagnostics(SsiReport(3, 1e-6, True), 4, 5, 0.125, 0.75)
