"""Where the host time of one step (c1, or the config named on the command line) goes: Python around the C calls vs the C calls themselves
(each wssr_* call is timed with perf_counter; the step ends with a device sync, so the wall time
of a step ~ its device time)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_05749_b200 import _lib, estimators, optimizers, synthetic  # noqa: E402

cfg = synthetic.config(sys.argv[1] if len(sys.argv) > 1 else "c1")
ctx = _lib.context()
calls = []
orig = ctx.call


def timed(name, *a):
    t0 = time.perf_counter()
    r = orig(name, *a)
    calls.append((name, time.perf_counter() - t0))
    return r


ctx.call = timed
N, P, k = cfg["N"], cfg["P"], cfg["k"]
g = torch.Generator(device="cuda").manual_seed(0)
O = torch.randn(N, P, dtype=torch.float64, device="cuda", generator=g) * 1e-2
E = -1.0 + 0.1 * torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
V0 = torch.linalg.qr(torch.randn(P, k, dtype=torch.float64, device="cuda", generator=g))[0]
st = optimizers.WssrState(obar=torch.zeros(P, 0, dtype=torch.float64, device="cuda"),
                          lbar=torch.zeros(0, dtype=torch.float64, device="cuda"), u_prev=V0,
                          r_max=k, delta=0.0, sigma_floor=1e-4, eps_grow=0.0, step=1)
th = torch.zeros(P, dtype=torch.float64, device="cuda")
cfgs = (None,) * N
for it in range(6):
    calls.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b = estimators.assemble(estimators.SampleBatch(cfgs, E, O))
    t1 = time.perf_counter()
    th, st, d = optimizers.wssr_step(th, b, 1.0, st)
    t2 = time.perf_counter()
    c = sum(x for _, x in calls)
    print(f"step {it}: total {1e3 * (t2 - t0):.2f} ms  assemble py {1e3 * (t1 - t0):.3f} ms  "
          f"wssr_step py+C {1e3 * (t2 - t1):.2f} ms  C calls {1e3 * c:.2f} ms  "
          f"python {1e3 * (t2 - t0 - c):.3f} ms  " + " ".join(f"{n}={1e3 * x:.2f}" for n, x in calls))
