"""Pin the CPU oracle (oracle/wssr_oracle.py) to the golden fixtures produced by the reference
package itself (tests/golden/make_golden.py) and to the reference's own known answers.
CPU-only."""

import numpy as np
import pytest

from conftest import rel, subspace_sine
from oracle import wssr_oracle as orc

from _runs import FIXTURES, HEAVY, heavy_oracle_run, oracle_run

TOL = 1e-12


@pytest.mark.parametrize("name", list(FIXTURES))
def test_oracle_matches_reference_fixture(golden, name):
    g = golden(name)
    runs = oracle_run(name, g)
    for t, r in enumerate(runs):
        np.testing.assert_allclose(r["in_sum"], g[f"in_sum_{t}"], rtol=1e-13)  # generator pin
        np.testing.assert_allclose([r["loss"], r["raw_loss"]], g[f"loss_{t}"], rtol=1e-13)
        ints = g[f"ints_{t}"]
        assert r["r_eff"] == ints[0] and r["iterations"] == ints[1]
        assert r["r_max_next"] == ints[3]
        assert rel(r["update"], g[f"update_{t}"]) < TOL
        assert rel(r["sigma"], g[f"sigma_{t}"]) < TOL
        assert rel(r["lbar"], g[f"lbar_{t}"]) < 1e-10
        d = g[f"diag_{t}"]
        np.testing.assert_allclose(r["residual"], d[0], rtol=1e-8)
        np.testing.assert_allclose([r["sigma_drift"], r["projector_drift"]], d[1:], rtol=1e-9,
                                   atol=1e-14)
        if f"V_{t}" in g:
            assert subspace_sine(r["V"], g[f"V_{t}"]) < 1e-12
            np.testing.assert_allclose(r["V"], g[f"V_{t}"], atol=1e-11)
        if t == 0 and "gradient_0" in g:
            assert rel(r["gradient"], g["gradient_0"]) < TOL
            assert rel(r["l_vector"], g["l_vector_0"]) < TOL


def test_oracle_known_answers(golden):
    g = golden("kat.npz")
    q, r = orc.qr_pos(g["qr_patch_a"])
    np.testing.assert_allclose(q, g["qr_patch_q"], atol=1e-14)
    np.testing.assert_allclose(r, g["qr_patch_r"], atol=1e-14)
    assert r[1, 1] == 0.0
    q, r = orc.qr_pos(g["qr_a"])
    np.testing.assert_allclose(q, g["qr_q"], atol=1e-13)
    f = orc.ssi(np.diag([5.0, 4.0, 3.0, 2.0, 1.0]), 2, max_iters=60)
    np.testing.assert_allclose(f["sigma"], g["ssi_diag_sigma"], rtol=1e-14)
    assert f["iterations"] == g["ssi_diag_iters"][0]
    f = orc.ssi(g["ssi_mat"], 10, max_iters=4, u_init=g["ssi_u0"])
    np.testing.assert_allclose(f["sigma"], g["ssi_sigma"], rtol=1e-13)
    np.testing.assert_allclose(f["u"], g["ssi_u"], atol=1e-12)
    np.testing.assert_allclose([f["iterations"], f["residual"]], g["ssi_rep"], rtol=1e-9)
    sd, pd = orc.subspace_drift(f["u"], f["sigma"], g["ssi_u0"], np.linspace(2, 1, 10))
    np.testing.assert_allclose([sd, pd], g["drift"], rtol=1e-9)
    b = orc.assemble(np.stack([[1.0, -2.0, 0.5], [0.2, 0.7, -1.1]]), np.array([3.0, 1.0]),
                     np.inf)
    np.testing.assert_allclose(b["o_matrix"], g["asm_o"], atol=1e-15)
    np.testing.assert_allclose(b["gradient"], g["asm_g"], atol=1e-15)


def test_oracle_reference_contract_closed_forms():
    """Known answers restated from the reference's tests (test_svdengine.py, test_linalg.py,
    test_estimators.py)."""
    q, r = orc.qr_pos(np.array([[3.0], [4.0]]))
    np.testing.assert_allclose(q, [[0.6], [0.8]], atol=1e-15)
    np.testing.assert_allclose(r, [[5.0]], atol=1e-15)
    with pytest.raises(orc.OracleError):
        orc.qr_pos(np.zeros((4, 2)))
    rng = np.random.default_rng(5)
    u = np.linalg.qr(rng.standard_normal((30, 3)))[0]
    v = np.linalg.qr(rng.standard_normal((20, 3)))[0]
    a = (u * np.array([4.0, 2.0, 1.0])) @ v.T
    f = orc.ssi(a, 3, max_iters=1, u_init=u)
    assert f["iterations"] == 1 and f["residual"] < 1e-12
    np.testing.assert_allclose(f["sigma"], [4.0, 2.0, 1.0], atol=1e-10)
    e = np.array([0.0, 0.0, 0.0, 0.0, 100.0])
    b = orc.assemble(np.eye(5), e, 1.0)
    assert b["raw_loss"] == pytest.approx(20.0)


@pytest.mark.parametrize("name", HEAVY)
def test_oracle_matches_heavy_row_fixtures(golden, name):
    """Heavy-tailed sample rows (written by the reference): the oracle lands inside the
    reference's own reordering floor (the distance between the reference's run and its run on
    the same samples permuted), which is 3e-9 on the update at 1e8 outlier pairs."""
    g = golden(name)
    for t, r in enumerate(heavy_oracle_run(g)):
        np.testing.assert_allclose(r["in_sum"], g[f"in_sum_{t}"], rtol=1e-13)
        fl = g[f"floor_{t}"]
        assert fl[3] == 1.0  # the reordered reference takes the same branches
        assert [r["r_eff"], r["iterations"]] == list(g[f"ints_{t}"])
        assert rel(r["update"], g[f"update_{t}"]) <= max(1e-12, 4 * fl[0])
        assert rel(r["sigma"], g[f"sigma_{t}"]) <= max(1e-12, 4 * fl[1])
        if f"V_{t}" in g:
            assert subspace_sine(r["V"], g[f"V_{t}"]) <= max(1e-12, 4 * fl[2])
