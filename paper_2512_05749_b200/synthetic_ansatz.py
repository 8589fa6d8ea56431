"""A seeded synthetic instance of the pooled-feature determinant ansatz (wavefunction.py:143-321)
sized to a BASELINE configuration, for measuring the device producer of O
(wavefunction.grad_theta_batch) at benchmark scale: n_electrons x n_features = P parameters,
walkers = N samples.  The reference's own systems (Be, LiH, O) are far smaller than c1; this
instance keeps their structure (s and p Slater-type orbitals on a few nuclei, spin-gated, features
of one head orbital times pooled tail orbitals) at c1's P.
"""

from __future__ import annotations

from collections import namedtuple

import numpy as np

Orbital = namedtuple("Orbital", "center n ell m zeta spin")


def ansatz(n_electrons=16, n_features=8192, n_nuclei=4, orbitals_per_nucleus=16, tail=2,
           seed=0):
    """(AceSpec arguments, walker sampler) for a synthetic ansatz with P = n_electrons x
    n_features parameters."""
    rng = np.random.default_rng(seed)
    nuclei = rng.uniform(-2.0, 2.0, (n_nuclei, 3))
    spins = [0] * (n_electrons // 2) + [1] * (n_electrons - n_electrons // 2)
    orbs = []
    for c in range(n_nuclei):
        for j in range(orbitals_per_nucleus):
            kind = j % 4
            gate = ("up", "down", "either")[j % 3]
            zeta = 0.6 + 0.15 * (j // 4)
            if kind == 0:
                orbs.append(Orbital(c, j // 8, 0, 0, zeta, gate))
            else:
                orbs.append(Orbital(c, 0, 1, (-1, 0, 1)[kind - 1], zeta, gate))
    n_orb = len(orbs)
    feats = [(int(rng.integers(n_orb)), tuple(int(x) for x in rng.integers(n_orb, size=tail)))
             for _ in range(n_features)]
    theta = 0.01 * rng.standard_normal(n_electrons * n_features)

    def walkers(w, step_seed):
        r = np.random.default_rng((seed, step_seed))
        centre = nuclei[r.integers(n_nuclei, size=(w, n_electrons))]
        return centre + 0.8 * r.standard_normal((w, n_electrons, 3))

    return dict(nuclei=nuclei, spins=spins, orbitals=orbs, feature_index=feats,
                theta=theta), walkers
