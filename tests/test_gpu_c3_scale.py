"""BASELINE configs[3] at full size (N=16384, P=2^20, k=128, float32 O = 68.7 GB): the CPU oracle
cannot hold it, so one WSSR step on the production path (int8 tensor-core O-passes with digit
planes for the samples that fit and on-the-fly digits for the rest) is checked against the same
step with every O-pass on FP64 DMMA (independent arithmetic on the same float32 inputs), plus
size-independent properties: orthonormal U, sorted positive sigma, and the preconditioner
identity update = U (c / sigma^2) + (g - U c) / lambda."""

import pytest

from conftest import F32_DIGIT_TOL

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_c3_step_int8_vs_dmma(fp32_digits, big_memory):
    from paper_2512_05749_b200 import _lib, estimators, linalg, optimizers, synthetic

    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a 180 GB B200")
    cfg = synthetic.config("c3")
    N, P, k = cfg["N"], cfg["P"], cfg["k"]
    dev = torch.device("cuda")
    wl = synthetic.DeviceWorkload(N, P, k, cfg["L"], cfg["alpha"], cfg["drift"], seed=303,
                                  device=dev, dtype=torch.float32)
    v0 = linalg.qr_orthonormalize(wl.v0_raw())[0]
    O, E = wl.next()
    ctx = _lib.context()
    out = {}
    for path in (0, 2):  # 0: int8 tensor cores (production), 2: FP64 DMMA
        ctx.lib.wssr_set_gemm_path(ctx.handle, path)
        st = optimizers.WssrState(obar=torch.zeros(0, P, dtype=torch.float64, device=dev).t(),
                                  lbar=torch.zeros(0, dtype=torch.float64, device=dev),
                                  u_prev=v0, r_max=k, delta=0.0, sigma_floor=cfg["lam"],
                                  eps_grow=0.0, step=1)
        b = estimators.assemble(estimators.SampleBatch((None,) * N, E, O))
        _, st1, diag, upd = optimizers.wssr_step(torch.zeros(P, dtype=torch.float64,
                                                             device=dev), b, 1.0, st,
                                                 return_update=True)
        sig = torch.linalg.vector_norm(st1.obar, dim=0)
        out[path] = (upd, sig, st1.u_prev, diag, b)
        torch.cuda.synchronize()
    ctx.lib.wssr_set_gemm_path(ctx.handle, 0)
    (u8, s8, U8, d8, b8), (u2, s2, U2, d2, _) = out[0], out[2]
    assert d8.effective_rank == d2.effective_rank
    assert d8.ssi.iterations_used == d2.ssi.iterations_used
    e_upd = (torch.linalg.vector_norm(u8 - u2) / torch.linalg.vector_norm(u2)).item()
    e_sig = (torch.linalg.vector_norm(s8 - s2) / torch.linalg.vector_norm(s2)).item()
    print(f"c3 int8 ({fp32_digits} digits) vs DMMA: update {e_upd:.2e}, sigma {e_sig:.2e}")
    tol = F32_DIGIT_TOL[fp32_digits]
    assert e_upd < tol["update"] and e_sig < tol["sigma"]
    # size-independent properties of the production step
    r = U8.shape[1]
    gram = U8.t() @ U8
    assert (gram - torch.eye(r, dtype=gram.dtype, device=dev)).abs().max().item() < 1e-12
    assert bool((s8[:-1] >= s8[1:]).all()) and bool((s8 > 0).all())
    g = 0.5 * b8.gradient  # gbar = Ohat lhat = gradient / 2 at delta = 0
    c = U8.t() @ g
    ref = U8 @ (c / s8 ** 2) + (g - U8 @ c) / cfg["lam"]
    assert (torch.linalg.vector_norm(u8 - ref) / torch.linalg.vector_norm(ref)).item() < 1e-10
