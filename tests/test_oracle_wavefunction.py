"""Pin the producer oracle (oracle/wavefunction_oracle.py) to tests/golden/ace_grad.npz, which
the reference's AceWavefunction.grad_theta_batch (wavefunction.py:307-321) wrote; and its node
rule (wavefunction.py:316-318) on a walker with two electrons at the same point.  CPU-only."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import wavefunction_oracle as wfo


def _tables(g, tag):
    return (g[f"{tag}_nuclei"], g[f"{tag}_spins"], g[f"{tag}_orb"], g[f"{tag}_zeta"],
            g[f"{tag}_heads"], g[f"{tag}_tails"], g[f"{tag}_theta"])


@pytest.mark.parametrize("tag", ["be2", "o2", "lih3"])
def test_oracle_matches_reference_gradients(tag):
    g = load_golden("ace_grad.npz")
    got = wfo.grad_theta(*_tables(g, tag), g[f"{tag}_positions"])
    assert got.shape == g[f"{tag}_grad"].shape
    assert rel(got, g[f"{tag}_grad"]) < 1e-12


def test_oracle_node_proximity():
    g = load_golden("ace_grad.npz")
    pos = g["be2_positions"][:2].copy()
    pos[1, 1] = pos[1, 0]           # electrons 0 and 1 share spin and position: equal rows of M
    spins = g["be2_spins"]
    assert spins[0] == spins[1]
    with pytest.raises(wfo.NodeProximity):
        wfo.grad_theta(*_tables(g, "be2"), pos)
