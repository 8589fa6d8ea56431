"""Host-array <-> device-tensor plumbing for the drop-in API.

Inputs may be numpy arrays, Python sequences or torch tensors (any device); the device path
works on float64 CUDA tensors.  Array outputs are float64 CUDA tensors of the ``DeviceArray``
subclass, which numpy reads (``np.asarray`` copies to the host), so reference-side code that hands
them to numpy (the runner's snapshot, checkpoint.write_checkpoint) keeps working.
"""

from __future__ import annotations

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


def to_tensor(x, dtype=torch.float64, dev=None) -> torch.Tensor:
    """Any array-like -> float64 tensor on `dev` (default: current CUDA device)."""
    dev = device() if dev is None else dev
    if isinstance(x, torch.Tensor):
        if x.dtype != dtype or x.device != dev:
            x = x.to(device=dev, dtype=dtype)
        return x
    a = np.asarray(x, dtype=np.float64)
    if any(st < 0 for st in a.strides):  # reversed views (a[::-1]): torch rejects them
        a = np.ascontiguousarray(a)
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
