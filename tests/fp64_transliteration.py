"""Torch-FP64 transliteration of the WSSR step - TEST INFRASTRUCTURE ONLY (secondary oracle).

SURVEY.md 8(c)/7.2: the CPU oracle (oracle/wssr_oracle.py) cannot hold configs c2-c4 (the
reference needs ~4|O| of host RAM and hours per step), so parity at scale is checked against this
independent restatement of the same algorithm in plain torch FP64 on the GPU: cuBLAS DGEMM for
the O-passes, cuSOLVER Householder QR with the reference's sign convention, eigvalsh for the
2-norm.  It shares no code with the product (no libwssr call, no int8 digits, no CholeskyQR2, no
DMMA kernels of ours) and is itself pinned to the CPU oracle at c0/c1
(tests/test_gpu_fp64_transliteration.py).

Restated reference (/root/reference/pkg/src/vmcsr):
  clip_energies / assemble   estimators.py:53-100
  qr_orthonormalize          linalg.py:29-61 (full-rank blocks; a deficient block raises here)
  ssi_svd                    svdengine.py:88-158
  subspace_drift             svdengine.py:199-226
  _prepare_warm_start        optimizers.py:277-289
  wssr_step (ssi, step >= 1) optimizers.py:292-391

The sample block is never centred or copied: Ohat^T q = s (O q - 1 (mu^T q)) and
Ohat v = s (O^T v - mu (1^T v)) with s = 1/sqrt(N), over row chunks for float32 samples.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

DEFICIENT_REL = 1e-12   # linalg.py:16
F64 = torch.float64


def qr_pos(a):
    """linalg.py:29-61: reduced QR with diag(R) >= 0 (full-rank blocks only)."""
    q, r = torch.linalg.qr(a, mode="reduced")
    dg = r.diagonal()
    fro = torch.linalg.vector_norm(a)
    if bool((dg.abs().min() <= DEFICIENT_REL * fro).item()):
        raise AssertionError("rank-deficient block: outside the transliteration's scope")
    sg = torch.where(dg < 0, -1.0, 1.0).to(F64)
    return q * sg, r * sg[:, None]


class Samples:
    """o_matrix = ((O - mu) s)^T applied implicitly; O is (N x P) sample-major, f64 or f32."""

    CHUNK = 256  # rows per FP64 widening chunk of float32 samples (2 GB at P = 2^20)

    def __init__(self, O, mu, s):
        self.O, self.mu, self.s = O, mu, s

    def _chunks(self):
        if self.O.dtype == F64:
            yield 0, self.O
        else:
            for r0 in range(0, self.O.shape[0], self.CHUNK):
                yield r0, self.O[r0:r0 + self.CHUNK].double()

    def ot(self, q):
        """o_matrix^T q (N x k)."""
        out = torch.empty(self.O.shape[0], q.shape[1], dtype=F64, device=q.device)
        for r0, blk in self._chunks():
            torch.matmul(blk, q, out=out[r0:r0 + blk.shape[0]])
        return (out - (self.mu @ q)[None, :]) * self.s

    def o(self, v):
        """o_matrix v (P x k)."""
        acc = None
        for r0, blk in self._chunks():
            part = blk.t() @ v[r0:r0 + blk.shape[0]]
            acc = part if acc is None else acc + part
        return (acc - self.mu[:, None] * v.sum(0)[None, :]) * self.s

    def fro2(self):
        tot = torch.zeros((), dtype=F64, device=self.mu.device)
        for _, blk in self._chunks():
            for r0 in range(0, blk.shape[0], 128):
                d = blk[r0:r0 + 128] - self.mu[None, :]
                tot += (d * d).sum()
        return float(tot) * self.s * self.s


def assemble(O, E, n_std=5.0):
    """estimators.py:74-100 (the bundle of the ssi path): mu, l_vector, loss, sample operator."""
    n = O.shape[0]
    if O.dtype == F64:
        mu = O.mean(0)
    else:
        mu = torch.zeros(O.shape[1], dtype=F64, device=O.device)
        for r0 in range(0, n, Samples.CHUNK):
            mu += O[r0:r0 + Samples.CHUNK].double().sum(0)
        mu /= n
    mid, sd = E.mean(), E.std(unbiased=False)
    c = E if float(sd) == 0.0 else torch.clamp(E, mid - n_std * sd, mid + n_std * sd)
    loss = float(c.mean())
    s = 1.0 / math.sqrt(n)
    return Samples(O, mu, s), (c - loss) * s, loss


@dataclass
class State:
    """Mirror of WssrState (optimizers.py:188-247) with torch tensors."""

    obar: torch.Tensor
    lbar: torch.Tensor
    u_prev: torch.Tensor
    r_max: int
    delta: float
    sigma_floor: float
    sigma_floor_relative: bool = False
    r_reg: float = 1e-6
    eps_grow: float = 0.0
    step: int = 1


class Ohat:
    """[sqrt(delta) obar | sqrt(1 - delta) o_matrix] (optimizers.py:323)."""

    def __init__(self, st: State, S: Samples):
        self.a, self.b = math.sqrt(st.delta), math.sqrt(1.0 - st.delta)
        self.obar, self.S, self.r = st.obar, S, st.obar.shape[1]
        self._fro2 = self.a ** 2 * float((st.obar * st.obar).sum()) + self.b ** 2 * S.fro2()

    def t(self, q):
        top = self.a * (self.obar.t() @ q)
        return torch.cat([top, self.b * self.S.ot(q)], 0)

    def __call__(self, v):
        out = self.b * self.S.o(v[self.r:])
        if self.r:
            out = out + self.a * (self.obar @ v[:self.r])
        return out


def ssi(oh: Ohat, rank, max_iters, u_init, tol):
    """svdengine.py:88-158 (warm-started; sigma = |diag R| of QR(v), no Rayleigh-Ritz)."""
    fro2 = oh._fro2
    q = qr_pos(u_init)[0]
    it = 0
    while True:
        v = oh.t(q)
        u = oh(v)
        q = qr_pos(u)[0]
        it += 1
        w = oh(oh.t(q))
        quo = q.t() @ w
        res = float(torch.linalg.matrix_norm(w - q @ quo)) / fro2
        mix = float(torch.linalg.matrix_norm(quo - torch.diag(quo.diagonal()))) / fro2
        if max(res, mix) < tol or it >= max_iters:
            break
    qv, rv = qr_pos(v)
    raw = rv.diagonal().cpu().numpy()
    order = np.argsort(-raw, kind="stable")
    sig = raw[order]
    k = int(np.sum(sig[:rank] > 0.0))
    idx = torch.as_tensor(order[:k], device=u.device)
    uf = qr_pos(u[:, idx])[0]
    return dict(u=uf, sigma=torch.as_tensor(sig[:k], device=u.device), v=qv[:, idx].t(),
                iterations=it, residual=res)


def _two_norm(m):
    """||m||_2 from the largest eigenvalue of the small Gram m^T m."""
    ev = torch.linalg.eigvalsh(m.t() @ m)
    return math.sqrt(max(float(ev[-1]), 0.0))


def subspace_drift(u1, s1, u2, s2):
    """svdengine.py:199-226."""
    r = min(s1.shape[0], s2.shape[0])
    if r == 0:
        return 0.0, 0.0
    sd = float(torch.linalg.vector_norm(s1[:r] - s2[:r]))
    a, b = u1[:, :r], u2[:, :r]
    pd = _two_norm(b - a @ (a.t() @ b))
    return (0.0 if sd < 1e-12 else sd), (0.0 if pd < 1e-12 else pd)


def step_seed(rng_seed, step):
    """optimizers.py:273-274."""
    return int(np.random.SeedSequence((int(rng_seed), int(step))).generate_state(1)[0])


def wssr_step(theta, S: Samples, l_vector, eta, st: State, max_iters=3, tol=1e-10, rng_seed=0):
    """optimizers.py:292-391, ssi branch with st.step >= 1.  Returns (theta', state', info)."""
    assert st.step >= 1
    m = S.mu.shape[0]
    oh = Ohat(st, S)
    lhat = torch.cat([oh.a * st.lbar, oh.b * l_vector])
    req = min(st.r_max, m, oh.r + S.O.shape[0])
    if st.u_prev.shape[1] >= req:
        u0 = st.u_prev[:, :req]
    else:  # widening with host PCG64 columns (optimizers.py:284-289)
        extra = np.random.default_rng(step_seed(rng_seed, st.step)).standard_normal(
            (m, req - st.u_prev.shape[1]))
        u0 = qr_pos(torch.cat([st.u_prev, torch.as_tensor(extra, device=S.mu.device)], 1))[0]
    f = ssi(oh, req, max_iters, u0, tol)
    sigma = f["sigma"]
    top = float(sigma[0]) ** 2
    r_eff = int((sigma ** 2 >= st.r_reg * top).sum())
    assert r_eff >= 1
    binding = sigma.shape[0] == req == st.r_max and r_eff == st.r_max
    nxt = min(math.ceil((1.0 + st.eps_grow) * st.r_max), m) if binding else st.r_max
    u = f["u"][:, :r_eff]
    sig = sigma[:r_eff]
    g = oh(lhat[:, None])[:, 0]
    c = u.t() @ g
    fl = st.sigma_floor * (top if st.sigma_floor_relative else 1.0)
    upd = u @ (c / sig ** 2) + (g - u @ c) / fl
    if st.u_prev.shape[1] == 0:
        sd = pd = 0.0
    else:
        sd, pd = subspace_drift(st.u_prev, torch.linalg.vector_norm(st.obar, dim=0), u, sig)
    nst = State(obar=u * sig, lbar=f["v"][:r_eff] @ lhat, u_prev=u, r_max=nxt, delta=st.delta,
                sigma_floor=st.sigma_floor, sigma_floor_relative=st.sigma_floor_relative,
                r_reg=st.r_reg, eps_grow=st.eps_grow, step=st.step + 1)
    info = dict(update=upd, sigma=sig, r_eff=r_eff, iterations=f["iterations"],
                residual=f["residual"], sigma_drift=sd, projector_drift=pd, next_r_max=nxt)
    return theta - eta * upd, nst, info


def baseline_state(v0, k, delta, lam):
    """WssrState(obar=0 cols, u_prev=V0, r_max=k, eps_grow=0, step=1)."""
    P = v0.shape[0]
    return State(obar=torch.zeros(P, 0, dtype=F64, device=v0.device),
                 lbar=torch.zeros(0, dtype=F64, device=v0.device), u_prev=v0, r_max=k,
                 delta=delta, sigma_floor=lam)
