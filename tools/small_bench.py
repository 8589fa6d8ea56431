"""Time the k x k device routines (debug ABI) with CUDA events."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_05749_b200 import _lib  # noqa: E402

ctx = _lib.context()
for k in (32, 64, 128, 256):
    rng = np.random.default_rng(k)
    x = rng.standard_normal((3 * k, k))
    A = torch.as_tensor(x.T @ x, device="cuda")
    o1 = torch.zeros(k, k, dtype=torch.float64, device="cuda")
    o2 = torch.zeros(k, k, dtype=torch.float64, device="cuda")
    st = (ctypes.c_int * 2)()
    res = {}
    for op, name in ((0, "chol_inv"), (1, "maxeig")):
        for _ in range(2):
            ctx.call("wssr_debug_small_f64", op, k, _lib.ptr(A), _lib.ptr(o1), _lib.ptr(o2), st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ctx.call("wssr_debug_small_f64", op, k, _lib.ptr(A), _lib.ptr(o1), _lib.ptr(o2), st)
        e1.record()
        torch.cuda.synchronize()
        res[name] = round(e0.elapsed_time(e1) / 10 * 1e3, 1)
    print(k, res, "us (incl. host sync per call)")
