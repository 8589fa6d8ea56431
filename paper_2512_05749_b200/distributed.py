"""Row (sample/walker) sharding of the WSSR step over one process per GPU.

Each rank owns a contiguous block of rows of O; the library combines the
partial products with NCCL allreduces (u = Ohat v per SSI pass, the k x k Grams of the final
QR(v), the column statistics of assemble, gbar and lbar).  The communicator is created inside
libwssr from an ncclUniqueId that rank 0 produces and torch.distributed broadcasts.
"""

from __future__ import annotations

import ctypes
import os

from . import _lib


def env_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def row_shard(n_rows: int, rank: int, world: int):
    """Balanced contiguous split: (row0, rows) of this rank."""
    base, extra = divmod(n_rows, world)
    rows = base + (1 if rank < extra else 0)
    row0 = rank * base + min(rank, extra)
    return row0, rows


def attach_nccl(ctx, group=None):
    """Create the library's NCCL communicator over the torch.distributed world."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if world == 1:
        return
    buf = ctypes.create_string_buffer(128)
    if rank == 0:
        ctx.call("wssr_nccl_unique_id", buf)
    obj = [bytes(buf.raw) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ident = ctypes.create_string_buffer(obj[0], 128)
    ctx.call("wssr_nccl_attach", ident, rank, world)
    ctx.rank, ctx.world = rank, world


class EmulatedGroup:
    """`world` ranks on ONE GPU, one host thread each, joined by libwssr's thread-emulated
    communicator (wssr_emu_*): exercises every sharded code path of the engine (row-split
    assemble, per-pass allreduces, history ownership, sharded dense first step) where only one
    GPU is available.  Collectives synchronise on the host, so no kernel ever waits on another.
    Test infrastructure, not a production transport.
    """

    def __init__(self, world: int, device: int = 0):
        lib = _lib.load_library()
        h = _lib._vp()
        if lib.wssr_emu_group_create(int(world), ctypes.byref(h)) != _lib.WSSR_OK:
            raise ValueError(f"bad emulated world size {world}")
        self._lib, self._group, self.world = lib, h, int(world)
        self.contexts = []
        for r in range(self.world):
            c = _lib.Context(device)
            c.call("wssr_emu_attach", h, r)
            c.rank, c.world = r, self.world
            self.contexts.append(c)

    def run(self, fn, timeout: float = 300.0):
        """fn(rank, world) on every rank concurrently, each on its own CUDA stream; returns the
        per-rank results (re-raises the first rank failure)."""
        import threading

        import torch

        results, failures = [None] * self.world, []

        def body(r):
            ctx = self.contexts[r]
            _lib.set_thread_context(ctx)
            try:
                with torch.cuda.device(ctx.device), torch.cuda.stream(torch.cuda.Stream(ctx.device)):
                    results[r] = fn(r, self.world)
                    torch.cuda.current_stream().synchronize()
            except BaseException as e:  # noqa: BLE001 - surfaced below
                failures.append((r, e))
                self._lib.wssr_emu_group_abort(self._group)
            finally:
                _lib.set_thread_context(None)

        threads = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(self.world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout)
        if any(t.is_alive() for t in threads):
            raise TimeoutError("an emulated rank did not finish (collective mismatch?)")
        if failures:
            raise failures[0][1]
        return results

    def close(self):
        for c in self.contexts:
            c.__del__()
        self.contexts = []
        if self._group:
            self._lib.wssr_emu_group_destroy(self._group)
            self._group = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
