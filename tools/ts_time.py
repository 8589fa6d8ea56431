"""CUDA-event time of the CholeskyQR2 tall-skinny GEMMs at c1 shape (P=131072, k=64)."""
import torch
from paper_2512_05749_b200 import _lib

ctx = _lib.context()
P, k = 131072, 64
A = torch.randn(P, k, dtype=torch.float64, device="cuda")
B = torch.triu(torch.randn(k, k, dtype=torch.float64, device="cuda"))
C = torch.empty(P, k, dtype=torch.float64, device="cuda")
G = torch.empty(k, k, dtype=torch.float64, device="cuda")


def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


trmm = lambda: ctx.call("wssr_gemm_f64", 1, P, k, k, _lib.ptr(A), k, None, _lib.ptr(B), k, _lib.ptr(C), k, 1.0, 0, 1024)
gram = lambda: ctx.call("wssr_gemm_f64", 0, k, k, P, _lib.ptr(A), k, None, _lib.ptr(A), k, _lib.ptr(G), k, 1.0, 0, 1024)
print(f"TRMM {t(trmm):.1f} us   Gram {t(gram):.1f} us")
