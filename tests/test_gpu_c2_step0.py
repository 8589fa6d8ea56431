"""BASELINE configs[2] (N=16384, P=2^20, k=128, 137 GB of FP64 O) from WssrState.initial: the
dense first step (optimizers.py:327-330) cannot form the 137 GB Ohat beside O, so the drop-in
takes the implicit exact truncated SVD (engine.cu implicit_svd).  LAPACK cannot run at this size;
the result is certified independently with plain torch FP64 (cuBLAS) on the device: the
reference's subspace_residual (svdengine.py:56-67) of the returned U, and the singular values as
the Rayleigh quotients of U, then two warm-started SSI steps follow."""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_c2_from_initial_state():
    from paper_2512_05749_b200 import estimators, optimizers, synthetic

    if torch.cuda.get_device_properties(0).total_memory < 170e9:
        pytest.skip("needs a 180 GB B200")
    cfg = synthetic.config("c2")
    N, P, k = cfg["N"], cfg["P"], cfg["k"]
    wl = synthetic.DeviceWorkload(N, P, k, cfg["L"], cfg["alpha"], cfg["drift"], seed=101)
    st = optimizers.WssrState.initial(P, rank_init=k, delta=cfg["delta"], sigma_floor=cfg["lam"])
    O, E = wl.next()
    b = estimators.assemble(estimators.SampleBatch((None,) * N, E, O))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    th, st1, diag = optimizers.wssr_step(torch.zeros(P, dtype=torch.float64, device="cuda"), b,
                                         1.0, st)
    torch.cuda.synchronize()
    t_step0 = time.perf_counter() - t0
    info = dict(optimizers.last_implicit_svd)
    print(f"c2 step 0: {t_step0:.2f} s, implicit SVD {info}")
    assert info["residual"] < 1e-10
    assert diag.ssi.iterations_used == 0 and diag.ssi.subspace_residual == 0.0
    r = diag.effective_rank
    U = st1.u_prev.as_subclass(torch.Tensor).contiguous()
    sig = optimizers.sigma_of(st1).as_subclass(torch.Tensor)
    # certificate in plain torch FP64: Oc = (O - mu) / sqrt(N), W = Oc^T Oc U
    mu = O.mean(0)
    Y = (O @ U - (mu @ U)[None, :]) / np.sqrt(N)          # N x r
    W = (O.t() @ Y - mu[:, None] * Y.sum(0)[None, :]) / np.sqrt(N)  # P x r
    sq = sum(float(O[i:i + 512].pow(2).sum()) for i in range(0, N, 512))
    fro2 = (sq - N * float(mu.pow(2).sum())) / N
    quot = U.t() @ W
    res = float(torch.linalg.matrix_norm(W - U @ quot)) / fro2
    rq = torch.sqrt(torch.diagonal(quot))
    print(f"  subspace_residual {res:.2e}, rank {r}, sigma rel err "
          f"{float(torch.linalg.vector_norm(rq - sig) / torch.linalg.vector_norm(sig)):.2e}")
    assert res < 1e-12
    assert float(torch.linalg.vector_norm(rq - sig) / torch.linalg.vector_norm(sig)) < 1e-12
    off = quot - torch.diag(torch.diagonal(quot))
    assert float(torch.linalg.matrix_norm(off)) < 1e-10 * float(quot[0, 0])
    del Y, W, quot
    # two warm-started SSI steps from there
    for _ in range(2):
        O, E = wl.next()
        b = estimators.assemble(estimators.SampleBatch((None,) * N, E, O))
        th, st1, diag = optimizers.wssr_step(th, b, 1.0, st1)
        assert diag.effective_rank > 0 and np.isfinite(diag.ssi.subspace_residual)
    torch.cuda.synchronize()
