"""GPU check of the DMMA GEMM family against torch fp64, plus timing of the WSSR phase shapes.

usage: python tools/gemm_check.py [--time]
"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_05749_b200 import _lib  # noqa: E402


def gemm(ctx, layout, A, shift, B, C, M, N, K, lda, ldb, ldc, alpha=1.0, acc=0, max_splits=1024):
    ctx.call("wssr_gemm_f64", layout, M, N, K, _lib.ptr(A), lda, _lib.ptr(shift), _lib.ptr(B), ldb,
             _lib.ptr(C), ldc, alpha, acc, max_splits)


def ref(layout, A, shift, B, M, N, K, lda, ldb, alpha):
    if layout == 0:  # A stored [K][M]
        Am = A.view(-1)[: (K - 1) * lda + M].as_strided((K, M), (lda, 1))
        if shift is not None:
            Am = Am - shift[None, :M]
        X = Am.t()
    else:
        Am = A.view(-1)[: (M - 1) * lda + K].as_strided((M, K), (lda, 1))
        if shift is not None:
            Am = Am - shift[None, :K]
        X = Am
    Bm = B.view(-1)[: (K - 1) * ldb + N].as_strided((K, N), (ldb, 1))
    return alpha * (X @ Bm)


def check(ctx, layout, M, N, K, pad=0, use_shift=True, alpha=0.7, acc=False, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if layout == 0:
        lda = M + pad
        A = torch.randn(K * lda, dtype=torch.float64, device="cuda", generator=g)
        shift = torch.randn(M, dtype=torch.float64, device="cuda", generator=g) if use_shift else None
    else:
        lda = K + pad
        A = torch.randn(M * lda, dtype=torch.float64, device="cuda", generator=g)
        shift = torch.randn(K, dtype=torch.float64, device="cuda", generator=g) if use_shift else None
    ldb = N + pad
    B = torch.randn(K * ldb, dtype=torch.float64, device="cuda", generator=g)
    ldc = N + pad
    C0 = torch.randn(M * ldc, dtype=torch.float64, device="cuda", generator=g)
    C = C0.clone()
    gemm(ctx, layout, A, shift, B, C, M, N, K, lda, ldb, ldc, alpha, int(acc))
    torch.cuda.synchronize()
    R = ref(layout, A, shift, B, M, N, K, lda, ldb, alpha)
    Cm = C.view(-1)[: (M - 1) * ldc + N].as_strided((M, N), (ldc, 1))
    if acc:
        R = R + C0.view(-1)[: (M - 1) * ldc + N].as_strided((M, N), (ldc, 1))
    err = (Cm - R).abs().max().item() / max(R.abs().max().item(), 1e-300)
    return err


def bench(ctx, layout, M, N, K, reps=10):
    if layout == 0:
        A = torch.randn(K, M, dtype=torch.float64, device="cuda")
        shift = torch.randn(M, dtype=torch.float64, device="cuda")
        lda = M
    else:
        A = torch.randn(M, K, dtype=torch.float64, device="cuda")
        shift = torch.randn(K, dtype=torch.float64, device="cuda")
        lda = K
    B = torch.randn(K, N, dtype=torch.float64, device="cuda")
    C = torch.empty(M, N, dtype=torch.float64, device="cuda")
    for _ in range(2):
        gemm(ctx, layout, A, shift, B, C, M, N, K, lda, N, N)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gemm(ctx, layout, A, shift, B, C, M, N, K, lda, N, N)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, 2.0 * M * N * K / ms / 1e9, M * K * 8 / ms / 1e6


def main():
    ctx = _lib.context(0)
    if "--one" in sys.argv:
        which = sys.argv[sys.argv.index("--one") + 1]
        shapes = {"cm": (0, 131072, 64, 4096), "rm": (1, 4096, 64, 131072)}
        print(bench(ctx, *shapes[which], reps=3))
        return
    worst = {}
    cases = []
    path = int(sys.argv[sys.argv.index("--path") + 1]) if "--path" in sys.argv else 0
    ctx.lib.wssr_set_gemm_path(ctx.handle, path)
    for layout in (0, 1):
        for (M, N, K) in [(5, 3, 7), (37, 5, 129), (128, 64, 4096), (300, 64, 1000), (64, 64, 50000),
                          (1000, 33, 77), (257, 128, 999), (96, 200, 333), (31, 256, 2048),
                          (4096, 1, 2000), (3, 3, 100000), (2000, 128, 5000),
                          (131072, 64, 64), (64, 64, 131072), (4096, 64, 8192), (8192, 64, 4096),
                          (1000, 256, 3000), (3000, 32, 5000)]:
            for pad in (0, 1):
                for acc in (False, True):
                    e = check(ctx, layout, M, N, K, pad=pad, acc=acc, seed=M + N + K)
                    cases.append((layout, M, N, K, pad, acc, e))
    bad = [c for c in cases if not c[-1] < 1e-12]
    print(json.dumps({"cases": len(cases), "bad": bad, "worst": max(c[-1] for c in cases)}))
    if "--time" in sys.argv:
        out = {}
        for name, (layout, M, N, K) in {
            "c1_K4_OTq": (1, 4096, 64, 131072),
            "c1_K5_Ov": (0, 131072, 64, 4096),
            "c2s_K4_OTq": (1, 16384, 128, 65536),
            "c2s_K5_Ov": (0, 65536, 128, 16384),
            "c1_gram": (0, 64, 64, 131072),
            "c1_trmm": (1, 131072, 64, 64),
        }.items():
            ms, tf, gbs = bench(ctx, layout, M, N, K)
            out[name] = {"ms": round(ms, 4), "tflops": round(tf, 2), "A_GBps": round(gbs, 1)}
        print(json.dumps(out))


if __name__ == "__main__":
    main()
