"""Per-K-block timeline of CTA 0 of one int8 O-pass (WSSR_OZ_DEBUG=9): who waits for whom."""
import ctypes
import os
import sys

os.environ["WSSR_OZ_DEBUG"] = os.environ.get("OZ_TRACE_MODE", "8")
import numpy as np
import torch

from paper_2512_05749_b200 import _lib

layout = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = _lib.context()
if os.environ.get("OZ_PRE", "0") == "1":
    ctx.lib.wssr_set_gemm_path(ctx.handle, 3)
else:
    ctx.lib.wssr_set_gemm_path(ctx.handle, 4)
if layout == 1:
    M, N, K = 4096, 64, 131072
else:
    M, N, K = 131072, 64, 4096
samples, params = (K, M) if layout == 0 else (M, K)
A = torch.randn(samples, params, dtype=torch.float64, device="cuda")
mu = A.mean(0)
B = torch.randn(K, N, dtype=torch.float64, device="cuda")
C = torch.empty(M, N, dtype=torch.float64, device="cuda")
for _ in range(2):
    ctx.call("wssr_debug_ozaki_gemm", layout, M, N, K, _lib.ptr(A), params, 0, _lib.ptr(mu),
             _lib.ptr(B), N, _lib.ptr(C), N, 1.0)
tr = np.zeros((8, 96), dtype=np.int64)
ctx.call("wssr_debug_ozaki_trace", ctypes.c_void_p(tr.ctypes.data), tr.size)
PRE = os.environ.get("OZ_PRE", "0") == "1"
names = (["raw TMA issue", "mma waits done", "mma token", "mma issued", "conv rfull ok",
          "conv computed", "conv dempty ok", "conv arrived"] if not PRE else
         ["mma start", "bfull ok", "afull ok", "token ok", "issued", "A TMA issue", "B TMA issue",
          "-"])
t0 = tr[0][0]
print("g   " + " ".join(f"{n[:13]:>13s}" for n in names))
for g in range(10, 40):
    print(f"{g:3d} " + " ".join(f"{(tr[i][g] - t0) if tr[i][g] else -1:13d}" for i in range(8)))
d = np.diff(tr[4 if PRE else 3][10:90])
print("MMA issued-to-issued per K-block: mean", d.mean(), "median", np.median(d))
