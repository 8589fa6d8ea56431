"""Host-array <-> device-tensor plumbing for the drop-in API.

Inputs may be numpy arrays, Python sequences or torch tensors (any device); the device path
works on float64 CUDA tensors.  Outputs are float64 CUDA tensors.
"""

from __future__ import annotations

import numpy as np
import torch


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
    return torch.as_tensor(np.asarray(x, dtype=np.float64), dtype=dtype).to(dev)


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
