"""Time the pre-digitised int8 O-pass (wssr_debug_ozaki_gemm, path 3: scales + digitize + pass)
on float32 samples with 5 and 7 sample digits at a c3-like slice (N=16384, k=128, P reduced)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(layout, N, P, k, digits, reps=5):
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    ctx.lib.wssr_set_gemm_path(ctx.handle, 3)
    ctx.lib.wssr_set_fp32_digits(ctx.handle, digits)
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(N, P, dtype=torch.float32, device="cuda", generator=g)
    mu = A.double().mean(0)
    M, K = (P, N) if layout == 0 else (N, P)
    B = torch.randn(K, k, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(M, k, dtype=torch.float64, device="cuda")

    def call():
        ctx.call("wssr_debug_ozaki_gemm", layout, M, k, K, _lib.ptr(A), P, 1, _lib.ptr(mu),
                 _lib.ptr(B), k, _lib.ptr(C), k, 1.0)

    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    N, P = 16384, int(sys.argv[1]) if len(sys.argv) > 1 else 131072
    for layout in (1, 0):
        for k in (64, 128):
            t = {d: run(layout, N, P, k, d) for d in (5, 7)}
            print(f"{'v' if layout else 'u'}-pass k={k} N={N} P={P}: 5 digits {t[5]:.2f} ms, "
                  f"7 digits {t[7]:.2f} ms (scales + digitize + pass)", flush=True)


def modes():
    """WSSR_OZ_DEBUG profiling modes of the pre-digitised kernel (read once per process):
    0 full, 5 no sample-digit traffic, 6 no thin-digit traffic, 7 no MMAs."""
    import subprocess
    for digits in (5, 7):
        row = []
        for mode in (0, 5, 6, 7):
            env = dict(os.environ, WSSR_OZ_DEBUG=str(mode))
            out = subprocess.run([sys.executable, __file__, "--child", str(digits)], env=env,
                                 capture_output=True, text=True)
            row.append(out.stdout.strip() or out.stderr.strip()[-120:])
        print(f"v-pass k=128 digits={digits}: full {row[0]} | no A {row[1]} | no B {row[2]} | "
              f"no MMA {row[3]} ms", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        print(f"{run(1, 16384, 131072, 128, int(sys.argv[2])):.2f}")
    elif len(sys.argv) > 1 and sys.argv[1] == "--modes":
        modes()
    else:
        main()
