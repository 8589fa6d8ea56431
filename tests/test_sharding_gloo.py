"""Row sharding of the WSSR step on CPU: world_size 2 over torch.distributed/gloo.

The sharded decomposition the engine uses (oracle/sharded.py mirrors csrc/engine.cu) must give
the unsharded oracle's results; plus the host-side shard arithmetic of
paper_2512_05749_b200/distributed.py."""

import os
import socket

import numpy as np
import pytest

from paper_2512_05749_b200.distributed import row_shard


def test_row_shard_partitions_rows():
    for n in (1, 7, 1024, 4097):
        for world in (1, 2, 3, 8):
            spans = [row_shard(n, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (a0, a1), (b0, _) in zip(spans, spans[1:]):
                assert a0 + a1 == b0
            assert sum(r for _, r in spans) == n
            assert max(r for _, r in spans) - min(r for _, r in spans) <= 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_q, n_samples=96):
    import torch
    import torch.distributed as dist

    from oracle import sharded, wssr_oracle as orc
    from paper_2512_05749_b200 import synthetic

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(x):
        t = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy().copy()

    cfg = synthetic.config("c0", N=n_samples, P=256, k=8, L=16, delta=0.0, lam=1e-3)
    wl = synthetic.HostWorkload.from_config(cfg, 5)
    st = orc.baseline_state(cfg["P"], cfg["k"], wl.v0_raw(), 0.0, cfg["lam"])
    row0, rows = row_shard(cfg["N"], rank, world)
    results = []
    for _ in range(3):
        o, e = wl.next()
        b = sharded.assemble_sharded(o[row0:row0 + rows], e[row0:row0 + rows], row0, cfg["N"],
                                     allreduce)
        b["n_global"] = cfg["N"]
        r = sharded.wssr_step_sharded(o[row0:row0 + rows], b, st, allreduce)
        ref_b = orc.assemble(o, e)
        _, st, info = orc.wssr_step(np.zeros(cfg["P"]), ref_b["o_matrix"], ref_b["l_vector"], 1.0,
                                    st)
        results.append((
            float(np.linalg.norm(r["update"] - info["update"]) / np.linalg.norm(info["update"])),
            float(np.linalg.norm(r["sigma"] - info["sigma"]) / np.linalg.norm(info["sigma"])),
            float(np.linalg.norm(b["gradient"] - ref_b["gradient"]) /
                  np.linalg.norm(ref_b["gradient"])),
            r["iterations"] == info["iterations"] and r["r_eff"] == info["r_eff"],
            float(np.linalg.norm(r["lbar"] - st.lbar) / max(np.linalg.norm(st.lbar), 1e-300)),
        ))
    out_q.put((rank, results))
    dist.destroy_process_group()


def _run_world(world, n_samples):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, n_samples))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in range(world):
        for upd, sig, grad, same_ints, lbar in outs[rank]:
            assert upd < 1e-10 and sig < 1e-12 and grad < 1e-12 and same_ints and lbar < 1e-9


def test_sharded_step_matches_unsharded_oracle_world2():
    _run_world(2, 96)


def test_sharded_step_ragged_shards_world3():
    """97 samples over 3 ranks: shards of 33, 32 and 32 rows."""
    _run_world(3, 97)
