"""WSSR state persistence for runs whose optimizer state lives on the device.

The reference snapshots a run into its "WSSR" binary format (vmcsr/checkpoint.py:3-19):

    magic b"WSSR" | u32 format version 1 | u64 header length | UTF-8 JSON header (sorted keys,
    compact separators) | float64 / int64 array payloads in manifest order | u32 CRC32 of all
    preceding bytes                                                   (all little-endian)

and `runner._snapshot` / `runner._restore` (runner.py:145-157, 203-216) store the WSSR state as
the scalars {"delta", "sigma_floor", "sigma_floor_relative", "r_reg", "eps_grow", "r_max",
"step"} plus the arrays "wssr_obar", "wssr_lbar", "wssr_u_prev".  The drop-in's state holds
CUDA tensors, which `np.asarray` (the reference writer) cannot take; this module reads and
writes the same bytes with device arrays on either side:

* `write_checkpoint` / `read_checkpoint`: the format itself, accepting numpy arrays or torch
  tensors (copied to the host) and returning numpy arrays, byte-compatible with the reference
  (tests/test_checkpoint.py checks a file written by the reference's own writer);
* `wssr_state_snapshot(state)` -> (scalars, arrays) in the runner's naming;
* `wssr_state_restore(scalars, arrays, device)` -> a `WssrState` on the device.

A runner switched to the drop-in calls `wssr_state_snapshot` where `_snapshot` reads
`opt_state.*` and `wssr_state_restore` where `_restore` rebuilds it.
"""

from __future__ import annotations

import json
import os
import struct
import zlib

import numpy as np

from .errors import CorruptChecksum, VersionMismatch

MAGIC = b"WSSR"
FORMAT_VERSION = 1
_PREFIX = struct.Struct("<4sIQ")     # magic, version, header length
_TRAILER = struct.Struct("<I")       # CRC32
_CODES = {"float64": "<f8", "int64": "<i8"}


def _host_array(name, value):
    """numpy view/copy of `value` (numpy array, scalar or torch tensor on any device)."""
    if hasattr(value, "detach") and hasattr(value, "cpu"):
        value = value.detach().cpu().numpy()
    arr = np.asarray(value)
    code = _CODES.get(arr.dtype.name)
    if code is None:
        raise ValueError(f"checkpoint arrays must be float64 or int64: {name!r} is {arr.dtype}")
    return arr, code


def encode(scalars, arrays, rng_states) -> bytes:
    """The complete snapshot bytes (see the module docstring)."""
    manifest, payload = [], []
    for name, value in arrays.items():
        arr, code = _host_array(name, value)
        manifest.append({"name": name, "dtype": code, "shape": list(arr.shape)})
        payload.append(np.ascontiguousarray(arr, dtype=np.dtype(code)).tobytes())
    header = json.dumps({"scalars": scalars, "arrays": manifest, "rng_states": rng_states},
                        sort_keys=True, separators=(",", ":")).encode("utf-8")
    head = _PREFIX.pack(MAGIC, FORMAT_VERSION, len(header)) + header
    crc = zlib.crc32(b"".join(payload), zlib.crc32(head)) & 0xFFFFFFFF
    return b"".join([head, *payload, _TRAILER.pack(crc)])


def write_checkpoint(path, scalars, arrays, rng_states) -> None:
    """Write the snapshot next to `path` and rename it into place (a crash never leaves a torn
    file where the previous snapshot was)."""
    blob = encode(scalars, arrays, rng_states)
    path = os.fspath(path)
    tmp = f"{path}.tmp"
    with open(tmp, "wb") as fh:
        fh.write(blob)
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, path)


def decode(data: bytes):
    """(scalars, arrays, rng_states) from snapshot bytes.

    Raises CorruptChecksum for structural damage (short file, bad magic, CRC mismatch, header or
    payload out of bounds, trailing bytes) and VersionMismatch for an intact file of another
    format version - the reference's split (checkpoint.py:74-125).
    """
    data = bytes(data)
    if len(data) < _PREFIX.size + _TRAILER.size:
        raise CorruptChecksum(f"snapshot too short ({len(data)} bytes)")
    magic, version, hlen = _PREFIX.unpack_from(data, 0)
    if magic != MAGIC:
        raise CorruptChecksum(f"not a WSSR snapshot (magic {magic!r})")
    if version != FORMAT_VERSION:
        raise VersionMismatch(f"snapshot format version {version}; this reader knows "
                              f"{FORMAT_VERSION}")
    end = len(data) - _TRAILER.size
    (crc,) = _TRAILER.unpack_from(data, end)
    if crc != zlib.crc32(memoryview(data)[:end]) & 0xFFFFFFFF:
        raise CorruptChecksum("snapshot CRC32 does not match its contents")
    pos = _PREFIX.size + hlen
    if pos > end:
        raise CorruptChecksum("snapshot header runs past the payload")
    try:
        header = json.loads(data[_PREFIX.size:pos].decode("utf-8"))
        scalars, manifest, rng_states = (header["scalars"], header["arrays"],
                                         header["rng_states"])
    except (ValueError, KeyError, TypeError, UnicodeDecodeError) as exc:
        raise CorruptChecksum(f"unreadable snapshot header: {exc}") from exc
    arrays = {}
    for item in manifest:
        try:
            name, dtype = item["name"], np.dtype(item["dtype"])
            shape = tuple(int(d) for d in item["shape"])
        except (KeyError, TypeError, ValueError) as exc:
            raise CorruptChecksum(f"unreadable array entry: {exc}") from exc
        count = int(np.prod(shape, dtype=np.int64))
        nbytes = count * dtype.itemsize
        if pos + nbytes > end:
            raise CorruptChecksum(f"payload of {name!r} runs past the end of the snapshot")
        arrays[name] = np.frombuffer(data, dtype=dtype, count=count, offset=pos).reshape(
            shape).copy()
        pos += nbytes
    if pos != end:
        raise CorruptChecksum("unexpected bytes between the payload and the CRC")
    return scalars, arrays, rng_states


def read_checkpoint(path):
    """Inverse of write_checkpoint: (scalars, arrays as numpy, rng_states)."""
    with open(path, "rb") as fh:
        return decode(fh.read())


_WSSR_SCALARS = ("delta", "sigma_floor", "sigma_floor_relative", "r_reg", "eps_grow", "r_max",
                 "step")


def wssr_state_snapshot(state):
    """(scalars, arrays) of a WssrState in the runner's naming (runner.py:145-157); the device
    arrays are copied to the host."""
    scalars = {name: getattr(state, name) for name in _WSSR_SCALARS}
    scalars["sigma_floor_relative"] = bool(scalars["sigma_floor_relative"])
    scalars["r_max"] = int(scalars["r_max"])
    scalars["step"] = int(scalars["step"])
    arrays = {
        "wssr_obar": _host_array("wssr_obar", state.obar)[0].astype(np.float64, copy=False),
        "wssr_lbar": _host_array("wssr_lbar", state.lbar)[0].astype(np.float64, copy=False),
        "wssr_u_prev": _host_array("wssr_u_prev", state.u_prev)[0].astype(np.float64,
                                                                          copy=False),
    }
    return scalars, arrays


def wssr_state_restore(scalars, arrays, device=None):
    """WssrState rebuilt from a snapshot (runner.py:203-216) with its arrays on `device`
    (default: the current CUDA device)."""
    import torch

    from .optimizers import WssrState

    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device

    def dev_array(name):
        return torch.as_tensor(np.ascontiguousarray(arrays[name], dtype=np.float64), device=dev)

    return WssrState(obar=dev_array("wssr_obar"), lbar=dev_array("wssr_lbar"),
                     u_prev=dev_array("wssr_u_prev"), r_max=int(scalars["r_max"]),
                     delta=float(scalars["delta"]), sigma_floor=float(scalars["sigma_floor"]),
                     sigma_floor_relative=bool(scalars["sigma_floor_relative"]),
                     r_reg=float(scalars["r_reg"]), eps_grow=float(scalars["eps_grow"]),
                     step=int(scalars["step"]))


__all__ = ["MAGIC", "FORMAT_VERSION", "encode", "decode", "write_checkpoint",
           "read_checkpoint", "wssr_state_snapshot", "wssr_state_restore"]
