"""Writes tests/golden/ace_grad.npz: AceWavefunction.grad_theta_batch of the REFERENCE
(vmcsr/wavefunction.py:307-321, imported read-only from /root/reference) on seeded walkers of a
few preset systems, with the ansatz tables the device producer needs (orbitals, feature index,
theta) so the GPU test runs without the reference.  Run in the build container:
    python tests/golden/make_wavefunction_golden.py"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from vmcsr import system as vsys  # noqa: E402
from vmcsr import wavefunction as vwf  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
GATES = {"up": 0, "down": 1, "either": 2}
out = {}
for tag, name, order, cap, walkers in (("be2", "be", 2, None, 16), ("lih3", "lih", 3, 2, 2),
                                       ("o2", "o", 2, None, 8)):
    sysm = vsys.preset_system(name)
    basis = vwf.default_basis(sysm)
    wf = vwf.AceWavefunction(sysm, basis, correlation_order=order, degree_cap=cap)
    rng = np.random.default_rng(len(tag) * 7 + order)
    centers = sysm.nuclear_positions[rng.integers(0, len(sysm.nuclear_positions),
                                                  size=(walkers, sysm.n_electrons))]
    pos = centers + rng.standard_normal((walkers, sysm.n_electrons, 3))
    grad = wf.grad_theta_batch(pos)
    orbs = basis.orbitals
    max_tail = max(len(t) for _, t in wf.feature_index)
    tails = np.full((len(wf.feature_index), max(max_tail, 1)), -1, dtype=np.int64)
    for i, (_, t) in enumerate(wf.feature_index):
        tails[i, :len(t)] = t
    out.update({
        f"{tag}_positions": pos, f"{tag}_grad": grad, f"{tag}_theta": wf.theta,
        f"{tag}_nuclei": sysm.nuclear_positions, f"{tag}_spins": np.asarray(sysm.spins),
        f"{tag}_orb": np.array([[o.center, o.n, o.ell, o.m, GATES[o.spin]] for o in orbs]),
        f"{tag}_zeta": np.array([o.zeta for o in orbs]),
        f"{tag}_heads": np.array([h for h, _ in wf.feature_index]), f"{tag}_tails": tails,
    })
    print(tag, sysm.n_electrons, "electrons,", len(orbs), "orbitals,", len(wf.feature_index),
          "features, n_params", wf.n_params)
np.savez_compressed(os.path.join(HERE, "ace_grad.npz"), **out)
