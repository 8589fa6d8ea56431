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
