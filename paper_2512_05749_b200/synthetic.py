"""Seeded synthetic WSSR workloads of BASELINE.json.

    O_0 = A diag(s) B^T + 0.01 G,   s_i = i^-alpha,   A (N x L), B (P x L), G (N x P) ~ N(0,1)
    O_t = O_{t-1} + drift * G_t,    E_t ~ N(-1, 0.1^2),   V_0 = QR(N(0,1) P x k)

Two generators with the same distribution:
  * ``HostWorkload`` (numpy PCG64, seeds 100+c / 200+c, draw order A, B, G_0, then per step
    G_t (t>0), E_t) - bit-reproducible inputs for the CPU oracle and the golden fixtures;
  * ``DeviceWorkload`` (torch Philox on the GPU) - the same shapes and value distributions for
    the large configurations, never materialised on the host (the benchmark uses it).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CONFIGS = {
    # name: N, P, k, latent L, alpha, delta, lambda, drift, T, dtype
    "c0": dict(N=1024, P=4096, k=32, L=64, alpha=1.0, delta=0.0, lam=1e-3, drift=1e-3, T=20,
               dtype="f64"),
    "c1": dict(N=4096, P=131072, k=64, L=128, alpha=1.5, delta=0.0, lam=1e-4, drift=1e-3, T=50,
               dtype="f64"),
    "c2": dict(N=16384, P=1048576, k=128, L=256, alpha=1.0, delta=0.0, lam=1e-4, drift=1e-3,
               T=20, dtype="f64"),
    "c3": dict(N=16384, P=1048576, k=128, L=256, alpha=1.0, delta=0.0, lam=1e-4, drift=1e-3,
               T=20, dtype="f32"),
    "c4": dict(N=32768, P=2097152, k=256, L=512, alpha=0.8, delta=0.95, lam=1e-4, drift=5e-4,
               T=10, dtype="f64"),
    # one 8-way rank's share of c4's sample rows at c4's full width and rank: what a single
    # B200 can hold of the 550 GB block (bench.py --config c4s; not a BASELINE entry of its own)
    "c4s": dict(N=4096, P=2097152, k=256, L=512, alpha=0.8, delta=0.95, lam=1e-4, drift=5e-4,
                T=10, dtype="f64",
                label="c4s: 4096 of BASELINE configs[4]'s 32768 sample rows (one 8-way rank's "
                      "share) at its full P=2097152 params, k=256, delta=0.95, f64"),
}


def config(name, **overrides):
    cfg = dict(CONFIGS[name])
    cfg.update(overrides)
    cfg["name"] = name
    return cfg


@dataclass
class HostWorkload:
    """numpy generator; ``step(t)`` returns (O_t (N x P), E_t (N,))."""

    N: int
    P: int
    k: int
    L: int
    alpha: float
    drift: float
    data_seed: int
    v0_seed: int

    def __post_init__(self):
        self.rng = np.random.default_rng(self.data_seed)
        a = self.rng.standard_normal((self.N, self.L))
        b = self.rng.standard_normal((self.P, self.L))
        s = np.arange(1, self.L + 1, dtype=np.float64) ** (-self.alpha)
        self.O = (a * s) @ b.T + 0.01 * self.rng.standard_normal((self.N, self.P))
        self.t = -1

    @classmethod
    def from_config(cls, cfg, index):
        return cls(N=cfg["N"], P=cfg["P"], k=cfg["k"], L=cfg["L"], alpha=cfg["alpha"],
                   drift=cfg["drift"], data_seed=100 + index, v0_seed=200 + index)

    def v0_raw(self):
        return np.random.default_rng(self.v0_seed).standard_normal((self.P, self.k))

    def next(self):
        """Advance to the next step; returns (O_t, E_t)."""
        self.t += 1
        if self.t > 0:
            self.O = self.O + self.drift * self.rng.standard_normal((self.N, self.P))
        e = -1.0 + 0.1 * self.rng.standard_normal(self.N)
        return self.O, e


class DeviceWorkload:
    """torch/Philox generator on the GPU with the same shapes and distributions.

    Rows can be restricted to a shard [row0, row0+rows) so that under row sharding each rank
    generates exactly its own rows; the latent factor B is replicated from one seed and the
    row-dependent draws come from per-(block, step) seeds so the global O does not depend on the
    number of ranks.
    """

    BLOCK = 256

    def __init__(self, N, P, k, L, alpha, drift, seed, row0=0, rows=None, device="cuda",
                 dtype=None):
        import torch

        self.torch = torch
        self.N, self.P, self.k, self.L = N, P, k, L
        self.alpha, self.drift, self.seed = alpha, drift, seed
        self.row0 = row0
        self.rows = N - row0 if rows is None else rows
        self.device = device
        self.dtype = torch.float64 if dtype is None else dtype
        g = torch.Generator(device=device).manual_seed(seed * 1000003 + 17)
        s = torch.arange(1, L + 1, device=device, dtype=torch.float64) ** (-alpha)
        B = torch.randn(P, L, generator=g, device=device, dtype=torch.float64)
        self.Bs = (B * s).t().contiguous()  # L x P
        del B
        self.O = torch.empty(self.rows, P, device=device, dtype=self.dtype)
        for r0 in range(0, self.rows, self.BLOCK):
            r1 = min(self.rows, r0 + self.BLOCK)
            gb = self._gen(r0, 0)
            a = torch.randn(r1 - r0, L, generator=gb, device=device, dtype=torch.float64)
            blk = a @ self.Bs
            blk += 0.01 * torch.randn(r1 - r0, P, generator=gb, device=device,
                                      dtype=torch.float64)
            self.O[r0:r1] = blk.to(self.dtype)
        self.t = -1

    def _gen(self, local_r0, t):
        blk = (self.row0 + local_r0) // self.BLOCK
        return self.torch.Generator(device=self.device).manual_seed(
            (self.seed * 7919 + blk) * 104729 + t)

    def v0_raw(self):
        g = self.torch.Generator(device=self.device).manual_seed(self.seed * 31 + 5)
        return self.torch.randn(self.P, self.k, generator=g, device=self.device,
                                dtype=self.torch.float64)

    def next(self):
        """Advance one step in place: O += drift * G_t (t > 0); returns (O, E_t)."""
        torch = self.torch
        self.t += 1
        if self.t > 0:
            for r0 in range(0, self.rows, self.BLOCK):
                r1 = min(self.rows, r0 + self.BLOCK)
                g = self._gen(r0, self.t)
                self.O[r0:r1].add_(torch.randn(r1 - r0, self.P, generator=g, device=self.device,
                                               dtype=self.dtype), alpha=self.drift)
        ge = torch.Generator(device=self.device).manual_seed(self.seed * 13 + 1000 * self.t + 7)
        e_all = -1.0 + 0.1 * torch.randn(self.N, generator=ge, device=self.device,
                                         dtype=torch.float64)
        return self.O, e_all[self.row0:self.row0 + self.rows].contiguous()


class HeavyRowWorkload(HostWorkload):
    """The BASELINE generator with heavy-tailed sample rows (precision tests of the int8 O-pass
    digits, which scale per parameter column):

      * ``kind="pair"``: two rows get +mag z and -mag z for one shared N(0,1) P-vector z (a
        near-node walker pair: the column means do not move, the column maxima do);
      * ``kind="tscale"``: every row is multiplied by |t_df| with df = mag (Student-t row scales);
      * ``kind="telem"``: every element is multiplied by an independent |t_df| draw.

    The heavy part is drawn once (seeded) and kept fixed while the O_t drift as in
    ``HostWorkload``."""

    def __init__(self, N, P, k, L, alpha, drift, data_seed, v0_seed, kind, mag):
        super().__init__(N, P, k, L, alpha, drift, data_seed, v0_seed)
        hr = np.random.default_rng(data_seed + 7777)
        self.kind, self.mag = kind, mag
        if kind == "pair":
            z = hr.standard_normal(P)
            self.rows = (3 % N, (N // 2 + 5) % N)
            self.add = np.zeros((N, P))
            self.add[self.rows[0]] += mag * z
            self.add[self.rows[1]] -= mag * z
            self.mul = None
        elif kind == "tscale":
            self.add = None
            self.mul = np.abs(hr.standard_t(mag, size=N))[:, None]
        elif kind == "telem":
            self.add = None
            self.mul = np.abs(hr.standard_t(mag, size=(N, P)))
        else:
            raise ValueError(kind)

    def next(self):
        o, e = super().next()
        if self.add is not None:
            return o + self.add, e
        return o * self.mul, e
