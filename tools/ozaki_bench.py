"""Time the two c1 O-pass GEMMs on the int8 tensor-core path vs FP64 DMMA (CUDA events)."""
import sys

import torch

from paper_2512_05749_b200 import _lib


def bench(layout, M, N, K, f32=False, reps=10):
    ctx = _lib.context()
    g = torch.Generator(device="cuda").manual_seed(1)
    samples, params = (K, M) if layout == 0 else (M, K)
    A = torch.randn(samples, params, dtype=torch.float64, device="cuda", generator=g)
    if f32:
        A = A.float()
    mu = A.double().mean(0)
    B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(M, N, dtype=torch.float64, device="cuda")
    res = {}
    for name in ("ozaki", "ozaki_fly", "dmma"):
        def run():
            if name.startswith("ozaki"):
                ctx.call("wssr_debug_ozaki_gemm", layout, M, N, K, _lib.ptr(A), params, int(f32),
                         _lib.ptr(mu), _lib.ptr(B), N, _lib.ptr(C), N, 1.0)
            elif f32:
                ctx.call("wssr_debug_gemm_f32a", layout, M, N, K, _lib.ptr(A), params,
                         _lib.ptr(mu), _lib.ptr(B), N, _lib.ptr(C), N, 1.0)
            else:
                ctx.call("wssr_gemm_f64", layout, M, N, K, _lib.ptr(A), params, _lib.ptr(mu),
                         _lib.ptr(B), N, _lib.ptr(C), N, 1.0, 0, 1024)
        ctx.lib.wssr_set_gemm_path(ctx.handle, {"ozaki": 0, "ozaki_fly": 4, "dmma": 2}[name])
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[name] = ms
    ctx.lib.wssr_set_gemm_path(ctx.handle, 0)
    gb = samples * params * A.element_size() / 1e9
    print(f"layout={layout} M={M} N={N} K={K} f32={f32}: ozaki {res['ozaki']:.3f} ms "
          f"(pre-digitised, incl. scales + digitise) on-the-fly {res['ozaki_fly']:.3f} ms  dmma {res['dmma']:.3f} ms "
          f"({2 * M * N * K / res['dmma'] / 1e9:.1f} TF/s)", flush=True)


if __name__ == "__main__":
    if "--one" in sys.argv:
        if sys.argv[-1] == "0":
            bench(0, 131072, 64, 4096, reps=3)
        else:
            bench(1, 4096, 64, 131072, reps=3)
        sys.exit(0)
    bench(1, 4096, 64, 131072)
    bench(0, 131072, 64, 4096)
    bench(1, 4096, 64, 131072, f32=True)
    bench(0, 131072, 64, 4096, f32=True)
    if "--big" in sys.argv:
        bench(1, 16384, 128, 262144)
        bench(0, 262144, 128, 16384)
