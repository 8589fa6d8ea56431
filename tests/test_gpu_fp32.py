"""FP32 variant (BASELINE configs[3]: float32 O, FP64 k x k Gram/Cholesky): FP32 storage is
widened to FP64 in registers, so the step equals the FP64 oracle run on the FP32-rounded inputs
(to FP64 tolerances) and the FP64 oracle on the unrounded inputs to the 1e-4 FP32 tolerance."""

import numpy as np
import pytest

from conftest import F32_DIGIT_TOL, rel, subspace_sine

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout", [0, 1])
@pytest.mark.parametrize("M,N,K", [(4096, 64, 8192), (8192, 64, 4096), (1024, 128, 5000),
                                   (3000, 32, 4096), (512, 256, 2048)])
def test_fp32_operand_gemm(layout, M, N, K):
    import torch

    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    if layout == 0:
        A = torch.randn(K, M, dtype=torch.float32, device="cuda", generator=g)
        shift = torch.randn(M, dtype=torch.float64, device="cuda", generator=g)
        X = (A.double() - shift[None, :]).t()
        lda = M
    else:
        A = torch.randn(M, K, dtype=torch.float32, device="cuda", generator=g)
        shift = torch.randn(K, dtype=torch.float64, device="cuda", generator=g)
        X = A.double() - shift[None, :]
        lda = K
    B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty(M, N, dtype=torch.float64, device="cuda")
    ref = 0.5 * (X @ B)
    ctx.call("wssr_debug_gemm_f32a", layout, M, N, K, _lib.ptr(A), lda, _lib.ptr(shift),
             _lib.ptr(B), N, _lib.ptr(C), N, 0.5)
    err = (C - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-13


def test_fp32_steps_match_fp64_oracle(fp32_digits):
    import torch

    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import estimators, optimizers, synthetic

    cfg = synthetic.config("c0", N=512, P=8192, k=32, L=48)
    P, N, k = cfg["P"], cfg["N"], cfg["k"]
    wl = synthetic.HostWorkload.from_config(cfg, 3)
    ost32 = orc.baseline_state(P, k, wl.v0_raw(), 0.0, cfg["lam"])
    ost64 = orc.baseline_state(P, k, wl.v0_raw(), 0.0, cfg["lam"])
    dev = torch.device("cuda")
    st = optimizers.WssrState(obar=np.zeros((P, 0)), lbar=np.zeros(0), u_prev=ost32.u_prev,
                              r_max=k, delta=0.0, sigma_floor=cfg["lam"], eps_grow=0.0, step=1)
    for t in range(3):
        o, e = wl.next()
        o32 = o.astype(np.float32)
        b = orc.assemble(o32.astype(np.float64), e)
        _, ost32, info32 = orc.wssr_step(np.zeros(P), b["o_matrix"], b["l_vector"], 1.0, ost32)
        b64 = orc.assemble(o, e)
        _, ost64, info64 = orc.wssr_step(np.zeros(P), b64["o_matrix"], b64["l_vector"], 1.0,
                                         ost64)
        bundle = estimators.assemble(estimators.SampleBatch((None,) * N, e, o32))
        assert bundle._samples.dtype == torch.float32
        _, st, diag, upd = optimizers.wssr_step(np.zeros(P), bundle, 1.0, st, return_update=True)
        upd = upd.cpu().numpy()
        assert diag.effective_rank == info32["r_eff"]
        tol = F32_DIGIT_TOL[fp32_digits]
        assert rel(upd, info32["update"]) < tol["update"]          # same inputs, FP64 oracle
        assert rel(upd, info64["update"]) < 1e-4                   # BASELINE FP32 tolerance
        sig = torch.linalg.vector_norm(st.obar, dim=0).cpu().numpy()
        assert rel(sig, info32["sigma"]) < tol["sigma"]
        assert subspace_sine(st.u_prev.cpu().numpy(), ost32.u_prev) < tol["sine"]
