"""The tall-skinny P x k kernels (csrc/tallskinny.cu: Grams, triangular and dense k x k products,
the fused residual norm) against torch fp64, on ragged row counts; and the engine with them
switched off (generic tile GEMMs) against the engine with them on."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROWS = [1, 3, 15, 16, 17, 63, 1000, 4099, 131072 + 5]


def _ops(rows, k, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    opt = dict(dtype=torch.float64, device="cuda", generator=g)
    A = torch.randn(rows, k, **opt)
    B = torch.randn(rows, k, **opt)
    M = torch.randn(k, k, **opt)
    C = torch.randn(rows, k, **opt)
    return A, B, M, C


@pytest.mark.parametrize("k", [32, 64, 128])
@pytest.mark.parametrize("rows", ROWS)
def test_grams(k, rows):
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    A, B, _, _ = _ops(rows, k, rows * 3 + k)
    out = torch.full((k, k), float("nan"), dtype=torch.float64, device="cuda")
    ctx.call("wssr_debug_tallskinny", 0, rows, k, _lib.ptr(A), None, None, None, 1.0,
             _lib.ptr(out))
    ref = A.t() @ A
    assert torch.equal(out, out.t())  # mirrored exactly
    assert ((out - ref).abs().max() / ref.abs().max()).item() < 1e-14
    ctx.call("wssr_debug_tallskinny", 1, rows, k, _lib.ptr(A), _lib.ptr(B), None, None, 1.0,
             _lib.ptr(out))
    ref = A.t() @ B
    assert ((out - ref).abs().max() / ref.abs().max()).item() < 1e-14


@pytest.mark.parametrize("k", [32, 64, 128])
@pytest.mark.parametrize("rows", ROWS)
@pytest.mark.parametrize("alpha", [1.0, -1.0])
def test_products(k, rows, alpha):
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    A, _, M, C = _ops(rows, k, rows * 5 + k)
    U = torch.triu(M)
    Y = torch.full((rows, k), float("nan"), dtype=torch.float64, device="cuda")

    def check(op, ref, m, cin=None):
        ctx.call("wssr_debug_tallskinny", op, rows, k, _lib.ptr(A), None, _lib.ptr(m),
                 _lib.ptr(cin) if cin is not None else None, alpha, _lib.ptr(Y))
        assert ((Y - ref).abs().max() / ref.abs().max()).item() < 1e-14

    check(2, alpha * (A @ U), U)
    check(3, alpha * (A @ M), M)
    check(4, C + alpha * (A @ M), M, C)
    s = torch.zeros(1, dtype=torch.float64, device="cuda")
    ctx.call("wssr_debug_tallskinny", 5, rows, k, _lib.ptr(A), None, _lib.ptr(M), _lib.ptr(C),
             alpha, _lib.ptr(s))
    ref = ((C + alpha * (A @ M)) ** 2).sum()
    assert abs(s.item() - ref.item()) / ref.item() < 1e-13
    x = C[:, 0].contiguous()
    g = torch.empty(k, dtype=torch.float64, device="cuda")
    ctx.call("wssr_debug_tallskinny", 6, rows, k, _lib.ptr(A), None, None, _lib.ptr(x), alpha,
             _lib.ptr(g))
    ref = alpha * (A.t() @ x)
    assert ((g - ref).abs().max() / ref.abs().max()).item() < 1e-13


@pytest.mark.parametrize("rows", [1, 17, 1000, 4099, 65536 + 3])
def test_k256_as_blocks_of_the_k128_kernels(rows):
    """k = 256 (BASELINE configs[4]): Grams, cross products and the row-block products composed
    from the k = 128 kernels on the two 128-column halves (engine.cu ts_blocked)."""
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    k = 256
    A, B, M, C = _ops(rows, k, rows * 7 + k)
    U = torch.triu(M)
    out = torch.full((k, k), float("nan"), dtype=torch.float64, device="cuda")
    Y = torch.full((rows, k), float("nan"), dtype=torch.float64, device="cuda")

    def call(op, b=None, m=None, cin=None, alpha=1.0, dst=out):
        ctx.call("wssr_debug_tallskinny", op, rows, k, _lib.ptr(A),
                 _lib.ptr(b) if b is not None else None, _lib.ptr(m) if m is not None else None,
                 _lib.ptr(cin) if cin is not None else None, alpha, _lib.ptr(dst))

    def close(x, ref):
        return ((x - ref).abs().max() / ref.abs().max()).item() < 1e-14

    call(0)
    assert torch.equal(out, out.t()) and close(out, A.t() @ A)
    call(1, b=B)
    assert close(out, A.t() @ B)
    call(2, m=U, dst=Y)
    assert close(Y, A @ U)
    call(3, m=M, dst=Y)
    assert close(Y, A @ M)
    call(4, m=M, cin=C, alpha=-1.0, dst=Y)
    assert close(Y, C - A @ M)


def test_bitwise_repeatable():
    from paper_2512_05749_b200 import _lib

    ctx = _lib.context()
    A, B, M, C = _ops(50000, 64, 7)
    outs = []
    for _ in range(2):
        G = torch.empty(64, 64, dtype=torch.float64, device="cuda")
        s = torch.empty(1, dtype=torch.float64, device="cuda")
        ctx.call("wssr_debug_tallskinny", 0, 50000, 64, _lib.ptr(A), None, None, None, 1.0,
                 _lib.ptr(G))
        ctx.call("wssr_debug_tallskinny", 5, 50000, 64, _lib.ptr(A), None, _lib.ptr(M),
                 _lib.ptr(C), -1.0, _lib.ptr(s))
        outs.append((G, s))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("k", [32, 64])
def test_step_with_and_without_tallskinny(k):
    """A full warm-started WSSR step: tall-skinny kernels on vs the generic GEMMs."""
    from oracle import wssr_oracle as orc
    from paper_2512_05749_b200 import _lib, estimators, optimizers, synthetic

    cfg = synthetic.config("c0", N=512, P=8192, k=k, L=96, delta=0.0, lam=1e-3)
    wl = synthetic.HostWorkload.from_config(cfg, 11)
    o, e = wl.next()
    v0 = orc.qr_pos(wl.v0_raw())[0]
    ctx = _lib.context()
    res = []
    for on in (1, 0):
        ctx.lib.wssr_set_tallskinny(ctx.handle, on)
        st = optimizers.WssrState(obar=np.zeros((cfg["P"], 0)), lbar=np.zeros(0), u_prev=v0,
                                  r_max=k, delta=0.0, sigma_floor=cfg["lam"], eps_grow=0.0,
                                  step=1)
        bundle = estimators.assemble(estimators.SampleBatch((None,) * cfg["N"], e, o))
        _, st1, diag, upd = optimizers.wssr_step(np.zeros(cfg["P"]), bundle, 1.0, st,
                                                 return_update=True)
        res.append((upd.cpu().numpy(), torch.linalg.vector_norm(st1.obar, dim=0).cpu().numpy(),
                    diag))
    ctx.lib.wssr_set_tallskinny(ctx.handle, 1)
    (u1, s1, d1), (u0, s0, d0) = res
    assert np.linalg.norm(u1 - u0) / np.linalg.norm(u0) < 1e-11
    assert np.linalg.norm(s1 - s0) / np.linalg.norm(s0) < 1e-12
    assert d1.effective_rank == d0.effective_rank
    assert d1.ssi.iterations_used == d0.ssi.iterations_used
    assert abs(d1.projector_drift - d0.projector_drift) <= 1e-9 * max(d0.projector_drift, 1e-12)
