"""Time the on-the-fly int8 O-pass kernel at a c2-like shape (N=16384 samples, k=128; P reduced
to 131072 to keep the sample block at 17 GB) under the kernel's profiling modes
(WSSR_OZ_DEBUG: 0 full, 1 no digitising, 2 no MMAs, 3 neither, 4 no sample loads either).
Each mode runs in its own process (the mode is read once per process)."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(layout, N, P, k, f32, reps=5):
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(N, P, dtype=torch.float64, device="cuda", generator=g)
    if f32:
        A = A.float()
    mu = A.double().mean(0)
    M, K = (P, N) if layout == 0 else (N, P)
    B = torch.randn(K, k, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(M, k, dtype=torch.float64, device="cuda")
    ctx.lib.wssr_set_gemm_path(ctx.handle, 4)

    def run():
        ctx.call("wssr_debug_ozaki_gemm", layout, M, k, K, _lib.ptr(A), P, int(f32),
                 _lib.ptr(mu), _lib.ptr(B), k, _lib.ptr(C), k, 1.0)

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        layout, N, P, k, f32 = (int(x) for x in sys.argv[2:7])
        print(f"{one(layout, N, P, k, bool(f32)):.3f}")
        sys.exit(0)
    N, P = 16384, 131072
    quick = len(sys.argv) > 1 and sys.argv[1] == "--quick"  # FP64, k = 128 only
    for f32 in ((0,) if quick else (0, 1)):
        for layout in (1, 0):
            for k in ((128,) if quick else (64, 128)):
                row = []
                for mode in (0, 1, 2, 3, 4):
                    env = dict(os.environ, WSSR_OZ_DEBUG=str(mode))
                    out = subprocess.run([sys.executable, __file__, "--child", str(layout), str(N),
                                          str(P), str(k), str(f32)], env=env,
                                         capture_output=True, text=True)
                    row.append(out.stdout.strip() or out.stderr.strip()[-200:])
                name = "v" if layout == 1 else "u"
                print(f"{name}-pass f32={f32} k={k}: full {row[0]} | no-digitise {row[1]} | "
                      f"no-MMA {row[2]} | loads only {row[3]} | nothing {row[4]} ms", flush=True)
