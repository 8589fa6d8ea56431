"""Row-sharded WSSR steps over real NCCL: one process per GPU (torch.multiprocessing, gloo for
the rendezvous, the library's own NCCL communicator for the engine's collectives - allreduce,
reduce-scatter and all-gather of the P-sliced SSI tail).  Needs two visible GPUs; skipped on a
one-GPU box (there the same sharded code paths run through the thread-emulated communicator,
tests/test_gpu_sharded_emulated.py)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _steps(rows, T=3):
    from paper_2512_05749_b200 import estimators, linalg, optimizers, synthetic

    cfg = synthetic.config("c0", N=2048, P=32768, k=64, L=96, delta=0.5, lam=1e-4)
    N, P, k = cfg["N"], cfg["P"], cfg["k"]
    wl = synthetic.HostWorkload.from_config(cfg, 31)
    v0 = linalg.qr_orthonormalize(wl.v0_raw())[0]
    dev = torch.device("cuda")
    st = optimizers.WssrState(obar=torch.zeros(0, P, dtype=torch.float64, device=dev).t(),
                              lbar=torch.zeros(0, dtype=torch.float64, device=dev), u_prev=v0,
                              r_max=k, delta=cfg["delta"], sigma_floor=cfg["lam"], eps_grow=0.0,
                              step=1)
    out = []
    for _ in range(T):
        o, e = wl.next()
        if rows is not None:
            o, e = o[rows[0]:rows[0] + rows[1]], e[rows[0]:rows[0] + rows[1]]
        b = estimators.assemble(estimators.SampleBatch((None,) * o.shape[0], e, o))
        _, st, diag, upd = optimizers.wssr_step(torch.zeros(P, dtype=torch.float64, device=dev),
                                                b, 1.0, st, return_update=True)
        out.append(dict(update=upd.cpu().numpy(), V=st.u_prev.cpu().numpy(),
                        it=diag.ssi.iterations_used))
    return N, out


def _rank_main(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_05749_b200 import _lib, distributed

        ctx = _lib.context()
        distributed.attach_nccl(ctx)
        n = 2048
        _, out = _steps(distributed.row_shard(n, rank, world))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_process_nccl_matches_single_rank():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (one process per GPU)")
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, single = _steps(None)
    for r in range(2):
        for a, b in zip(single, res[r]):
            assert a["it"] == b["it"]
            d = np.linalg.norm(b["update"] - a["update"]) / np.linalg.norm(a["update"])
            assert d < 1e-10
