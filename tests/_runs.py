"""Shared drivers: replay a golden fixture's workload through the oracle or the device path."""

import numpy as np

from oracle import wssr_oracle as orc
from paper_2512_05749_b200 import synthetic

FIXTURES = {
    "c0_T20.npz": dict(cfg=("c0", {}), index=0),
    "hist_T4.npz": dict(cfg=("c0", dict(N=96, P=300, k=12, L=20, delta=0.9, lam=1e-3)), index=7),
    "growth_T4.npz": dict(cfg=("c0", dict(N=64, P=160, k=6, L=12, delta=0.5, lam=1e-2)), index=8),
}


def fixture_config(name, g):
    spec = FIXTURES[name]
    cfg = synthetic.config(spec["cfg"][0], **spec["cfg"][1])
    return cfg, spec["index"], int(g["T"]), float(g["eps_grow"]), float(g["r_reg"]), int(g["k_init"])


def oracle_run(name, g):
    """Closed-loop oracle replay of a fixture.  Yields per-step dicts."""
    cfg, index, T, eps_grow, r_reg, k_init = fixture_config(name, g)
    wl = synthetic.HostWorkload.from_config(cfg, index)
    v0 = orc.qr_pos(wl.v0_raw())[0][:, :k_init]
    st = orc.State(obar=np.zeros((cfg["P"], 0)), lbar=np.zeros(0), u_prev=v0, r_max=cfg["k"],
                   delta=cfg["delta"], sigma_floor=cfg["lam"], r_reg=r_reg, eps_grow=eps_grow,
                   step=1)
    out = []
    for t in range(T):
        o, e = wl.next()
        b = orc.assemble(o, e)
        th, st, info = orc.wssr_step(np.zeros(cfg["P"]), b["o_matrix"], b["l_vector"], 1.0, st)
        info.update(loss=b["loss"], raw_loss=b["raw_loss"], gradient=b["gradient"],
                    l_vector=b["l_vector"], V=st.u_prev, lbar=st.lbar, r_max_next=st.r_max,
                    in_sum=np.array([o.sum(), (o * o).sum(), e.sum()]))
        out.append(info)
    return out


def device_run(name, g, report_final_residual=True, rows=None, dtype=None):
    """Closed-loop replay through the drop-in API on the GPU.

    rows=(row0, n): this rank's shard of the samples (row-sharded runs); dtype: cast O to it.
    """
    import torch

    from paper_2512_05749_b200 import estimators, optimizers, linalg

    cfg, index, T, eps_grow, r_reg, k_init = fixture_config(name, g)
    wl = synthetic.HostWorkload.from_config(cfg, index)
    v0 = linalg.qr_orthonormalize(wl.v0_raw())[0][:, :k_init]
    P = cfg["P"]
    dev = torch.device("cuda")
    st = optimizers.WssrState(obar=torch.zeros(0, P, dtype=torch.float64, device=dev).t(),
                              lbar=torch.zeros(0, dtype=torch.float64, device=dev), u_prev=v0,
                              r_max=cfg["k"], delta=cfg["delta"], sigma_floor=cfg["lam"],
                              r_reg=r_reg, eps_grow=eps_grow, step=1)
    out = []
    for t in range(T):
        o, e = wl.next()
        if rows is not None:
            o, e = o[rows[0]:rows[0] + rows[1]], e[rows[0]:rows[0] + rows[1]]
        if dtype is not None:
            o = o.astype(dtype)
        batch = estimators.SampleBatch((None,) * o.shape[0], e, o)
        b = estimators.assemble(batch)
        th, st, diag, upd = optimizers.wssr_step(torch.zeros(P, dtype=torch.float64, device=dev), b,
                                                 1.0, st, return_update=True,
                                                 report_final_residual=report_final_residual)
        out.append(dict(update=upd.cpu().numpy(), theta=th.cpu().numpy(),
                        sigma=torch.linalg.vector_norm(st.obar, dim=0).cpu().numpy(),
                        V=st.u_prev.cpu().numpy(), lbar=st.lbar.cpu().numpy(),
                        r_eff=diag.effective_rank, iterations=diag.ssi.iterations_used,
                        residual=diag.ssi.subspace_residual, sigma_drift=diag.sigma_drift,
                        projector_drift=diag.projector_drift, r_max=diag.r_max,
                        r_max_next=st.r_max, loss=b.loss, raw_loss=b.raw_loss,
                        gradient=b.gradient.cpu().numpy(), l_vector=b.l_vector.cpu().numpy()))
    return out


HEAVY = ["heavy_pair_10000.npz", "heavy_pair_1e+06.npz", "heavy_pair_1e+08.npz",
         "heavy_tscale_1.5.npz", "heavy_tscale_1.npz", "heavy_telem_1.5.npz"]


def heavy_workload(g):
    """The seeded heavy-tailed-row workload of a heavy_*.npz fixture (make_golden.py heavy())."""
    N, P, k = int(g["N"]), int(g["P"]), int(g["k"])
    cfg = synthetic.config("c0", N=N, P=P, k=k, L=24, delta=0.0, lam=float(g["lam"]))
    wl = synthetic.HeavyRowWorkload(N, P, k, cfg["L"], cfg["alpha"], cfg["drift"], 300, 400,
                                    str(g["kind"]), float(g["mag"]))
    return cfg, wl


def heavy_oracle_run(g):
    cfg, wl = heavy_workload(g)
    P, k = cfg["P"], cfg["k"]
    st = orc.State(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=orc.qr_pos(wl.v0_raw())[0],
                   r_max=k, delta=0.0, sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
    out = []
    for t in range(int(g["T"])):
        o, e = wl.next()
        b = orc.assemble(o, e)
        _, st, info = orc.wssr_step(np.zeros(P), b["o_matrix"], b["l_vector"], 1.0, st)
        info.update(V=st.u_prev, in_sum=np.array([o.sum(), (o * o).sum(), e.sum()]))
        out.append(info)
    return out


def heavy_device_run(g):
    import torch

    from paper_2512_05749_b200 import estimators, linalg, optimizers

    cfg, wl = heavy_workload(g)
    P, k = cfg["P"], cfg["k"]
    dev = torch.device("cuda")
    st = optimizers.WssrState(obar=torch.zeros(0, P, dtype=torch.float64, device=dev).t(),
                              lbar=torch.zeros(0, dtype=torch.float64, device=dev),
                              u_prev=linalg.qr_orthonormalize(wl.v0_raw())[0], r_max=k,
                              delta=0.0, sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
    out = []
    for t in range(int(g["T"])):
        o, e = wl.next()
        b = estimators.assemble(estimators.SampleBatch((None,) * o.shape[0], e, o))
        _, st, diag, upd = optimizers.wssr_step(torch.zeros(P, dtype=torch.float64, device=dev),
                                                b, 1.0, st, return_update=True)
        out.append(dict(update=upd.cpu().numpy(),
                        sigma=torch.linalg.vector_norm(st.obar, dim=0).cpu().numpy(),
                        V=st.u_prev.cpu().numpy(), r_eff=diag.effective_rank,
                        iterations=diag.ssi.iterations_used))
    return out
