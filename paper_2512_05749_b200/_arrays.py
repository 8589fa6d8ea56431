"""Host-array <-> device-tensor plumbing for the drop-in API.

Inputs may be numpy arrays, Python sequences or torch tensors (any device); the device path
works on float64 CUDA tensors.  Array outputs are float64 CUDA tensors of the ``DeviceArray``
subclass, which numpy reads (``np.asarray`` copies to the host), so reference-side code that hands
them to numpy (the runner's snapshot, checkpoint.write_checkpoint) keeps working.
"""

from __future__ import annotations

import os
import threading
import warnings

import numpy as np
import torch


class DeviceArray(torch.Tensor):
    """A (CUDA) tensor numpy can read: ``np.asarray(x)`` returns a host copy.  Everything else is
    torch.Tensor."""

    def __array__(self, dtype=None, copy=None):
        a = torch.Tensor.detach(self).cpu().numpy()
        return a if dtype is None else a.astype(dtype, copy=False)

    def __deepcopy__(self, memo):
        return device_array(torch.Tensor.clone(self.as_subclass(torch.Tensor)))


def device_array(t):
    """View a tensor as a DeviceArray (no copy)."""
    if t is None or not isinstance(t, torch.Tensor) or isinstance(t, DeviceArray):
        return t
    return t.as_subclass(DeviceArray)


def is_host_array(x) -> bool:
    """numpy arrays and Python sequences: the reference's calling convention (host in, host out)."""
    return not isinstance(x, torch.Tensor)


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def default_device() -> torch.device:
    """CUDA when present (the compute path), else CPU (state construction/validation only)."""
    return device() if torch.cuda.is_available() else torch.device("cpu")


# Large host arrays (the reference runner hands assemble a numpy sample block every step,
# runner.py:284-292) go up through two pinned staging buffers: the host copy of chunk i + 1 (torch's
# multi-threaded CPU copy) overlaps the asynchronous H2D of chunk i, instead of one synchronous
# pageable cudaMemcpy.  WSSR_UPLOAD_STAGE_MB sizes a buffer (0 turns the pipeline off).
_STAGE_BYTES = int(os.environ.get("WSSR_UPLOAD_STAGE_MB", "64")) << 20
_PIPELINE_MIN_BYTES = 256 << 20
_stage_local = threading.local()  # one pair of buffers per host thread and device


def _stages(dev):
    per_dev = getattr(_stage_local, "per_dev", None)
    if per_dev is None:
        per_dev = _stage_local.per_dev = {}
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    st = per_dev.get(idx)
    if st is None:
        st = per_dev[idx] = [
            (torch.empty(_STAGE_BYTES, dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
            for _ in range(2)]
    return st


def _upload_pipelined(a: np.ndarray, dev) -> torch.Tensor:
    """C-contiguous float64/float32 host array -> device tensor of the same dtype, stream-ordered
    on the current stream; `a` may be reused as soon as this returns."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # read-only arrays: only read here
        src = torch.from_numpy(a.reshape(-1))
    out = torch.empty(a.shape, dtype=src.dtype, device=dev)
    dst = out.view(-1)
    n, step = src.numel(), _STAGE_BYTES // src.element_size()
    stream = torch.cuda.current_stream(dev)
    stages = _stages(dev)
    for i, off in enumerate(range(0, n, step)):
        buf8, ev = stages[i & 1]
        ev.synchronize()  # the H2D that last read this buffer has finished
        m = min(step, n - off)
        buf = buf8.view(src.dtype)[:m]
        buf.copy_(src[off:off + m])
        dst[off:off + m].copy_(buf, non_blocking=True)
        ev.record(stream)
    return out


def to_tensor(x, dtype=torch.float64, dev=None) -> torch.Tensor:
    """Any array-like -> float64 tensor on `dev` (default: current CUDA device)."""
    dev = device() if dev is None else dev
    if isinstance(x, torch.Tensor):
        if x.dtype != dtype or x.device != dev:
            x = x.to(device=dev, dtype=dtype)
        return x
    a = np.asarray(x, dtype=np.float32 if dtype == torch.float32 else np.float64)
    if any(st < 0 for st in a.strides):  # reversed views (a[::-1]): torch rejects them
        a = np.ascontiguousarray(a)
    if (_STAGE_BYTES > 0 and a.nbytes >= _PIPELINE_MIN_BYTES and a.flags.c_contiguous
            and dev.type == "cuda"):
        return _upload_pipelined(a, dev)
    return torch.as_tensor(a, dtype=dtype).to(dev)


def to_tensor_f64_or_f32(x, dev=None) -> torch.Tensor:
    """Like to_tensor, but float32 data stays float32 (the FP32 variant streams O as float32)."""
    is_f32 = (isinstance(x, torch.Tensor) and x.dtype == torch.float32) or \
        (isinstance(x, np.ndarray) and x.dtype == np.float32)
    return to_tensor(x, dtype=torch.float32 if is_f32 else torch.float64, dev=dev)


def rows_view(x: torch.Tensor) -> torch.Tensor:
    """2-D tensor with unit column stride (row-major with a leading dimension)."""
    if x.dim() != 2:
        raise ValueError(f"expected a matrix, got ndim={x.dim()}")
    if x.stride(1) != 1 or x.stride(0) < max(1, x.shape[1]):
        x = x.contiguous()
    return x


def ld(x: torch.Tensor) -> int:
    return int(x.stride(0)) if x.shape[0] > 1 else max(int(x.shape[1]), 1)


def host(x) -> np.ndarray:
    """Tensor/array -> numpy float64 (test and reporting convenience)."""
    if isinstance(x, torch.Tensor):
        return x.detach().to("cpu", torch.float64).numpy()
    return np.asarray(x, dtype=np.float64)
