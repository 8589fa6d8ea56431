"""The NCCL transport of the row-sharded engine on one GPU: a 1-rank communicator built through
the library's own dlopen'd ncclGetUniqueId / ncclCommInitRank (the 128-byte unique id passed by
value) and an allreduce through it.  Multi-rank runs need one GPU per rank; the sharded engine
arithmetic itself is covered by tests/test_gpu_sharded_emulated.py and the gloo tests."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_one_rank_nccl_communicator_allreduce():
    from paper_2512_05749_b200 import _lib

    ctx = _lib.Context(0)  # a private context: the default one stays communicator-free
    uid = ctypes.create_string_buffer(128)
    ctx.call("wssr_nccl_unique_id", uid)
    assert any(uid.raw)
    ctx.call("wssr_nccl_attach", uid, 0, 1)
    x = torch.arange(1000, dtype=torch.float64, device="cuda") * 0.5
    y = x.clone()
    ctx.call("wssr_allreduce_f64", _lib.ptr(y), y.numel())
    torch.cuda.synchronize()
    assert torch.equal(x, y)  # the sum over one rank
