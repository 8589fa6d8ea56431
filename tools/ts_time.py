"""CUDA-event time per launch of the tall-skinny kernels at c1 shape (P=131072, k=64), launched
back to back (WSSR_DEBUG_REPS) so launch gaps and event overhead amortise away."""
import os
import sys

os.environ.setdefault("WSSR_DEBUG_REPS", "50")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2512_05749_b200 import _lib  # noqa: E402

reps = int(os.environ["WSSR_DEBUG_REPS"])
ctx = _lib.context()
P, k = 131072, 64
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(P, k, dtype=torch.float64, device="cuda", generator=g)
B = torch.randn(P, k, dtype=torch.float64, device="cuda", generator=g)
M = torch.triu(torch.randn(k, k, dtype=torch.float64, device="cuda", generator=g))
C = torch.randn(P, k, dtype=torch.float64, device="cuda", generator=g)
Y = torch.empty(P, k, dtype=torch.float64, device="cuda")
G = torch.empty(k, k, dtype=torch.float64, device="cuda")
s = torch.empty(k, dtype=torch.float64, device="cuda")
x = C[:, 0].contiguous()
ops = {0: ("gram", None, G), 1: ("cross", None, G), 2: ("trmm", None, Y), 3: ("mul", None, Y),
       4: ("mul_add", C, Y), 5: ("resid", C, s), 6: ("gemv_t", x, s)}
for op, (name, cin, out) in ops.items():
    args = (op, P, k, _lib.ptr(A), _lib.ptr(B), _lib.ptr(M),
            _lib.ptr(cin) if cin is not None else None, 1.0, _lib.ptr(out))
    ctx.call("wssr_debug_tallskinny", *args)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.call("wssr_debug_tallskinny", *args)
    b.record()
    torch.cuda.synchronize()
    print(f"{name:8s} {a.elapsed_time(b) / reps * 1e3:7.1f} us per launch")
