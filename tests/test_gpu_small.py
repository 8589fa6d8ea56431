"""k x k device routines (CholeskyQR core, largest-eigenvalue solver) against numpy."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _small(op, a):
    from paper_2512_05749_b200 import _lib

    k = a.shape[0]
    A = torch.as_tensor(np.ascontiguousarray(a), device="cuda")
    o1 = torch.zeros(k, k, dtype=torch.float64, device="cuda")
    o2 = torch.zeros(k, k, dtype=torch.float64, device="cuda")
    st = (ctypes.c_int * 2)()
    _lib.context().call("wssr_debug_small_f64", op, k, _lib.ptr(A), _lib.ptr(o1), _lib.ptr(o2), st)
    return o1.cpu().numpy(), o2.cpu().numpy(), (st[0], st[1])


@pytest.mark.parametrize("k", [1, 2, 7, 32, 64, 100, 128, 150, 161, 200, 255, 256, 300])
def test_cholesky_inverse(k):
    rng = np.random.default_rng(k)
    x = rng.standard_normal((3 * k + 5, k)) * np.exp(rng.uniform(-3, 3, k))
    g = x.T @ x
    r, rinv, st = _small(0, g)
    assert st == (0, 0)
    ref = np.linalg.cholesky(g).T
    np.testing.assert_allclose(r, ref, rtol=1e-11, atol=1e-12 * np.abs(ref).max())
    np.testing.assert_allclose(rinv @ r, np.eye(k), atol=1e-10)
    assert np.all(np.tril(rinv, -1) == 0.0) and np.all(np.tril(r, -1) == 0.0)


@pytest.mark.parametrize("dup", [(5, 40), (10, 200), (130, 250)])
def test_cholesky_two_block_flags_deficient_column(dup):
    """k = 256 runs as two diagonal blocks (engine.cu chol_inv_blocked2): a duplicated column is
    flagged at its own index whichever block it falls in, against the original diagonal."""
    rng = np.random.default_rng(8)
    x = rng.standard_normal((800, 256))
    x[:, dup[1]] = x[:, dup[0]]
    _, _, st = _small(0, x.T @ x)
    assert st[0] == dup[1] + 1, st


def test_cholesky_flags_deficient_and_zero():
    rng = np.random.default_rng(3)
    x = rng.standard_normal((20, 4))
    x[:, 2] = x[:, 0]
    _, _, st = _small(0, x.T @ x)
    assert st[0] == 3
    _, _, st = _small(0, np.zeros((3, 3)))
    assert st == (1, 1)


@pytest.mark.parametrize("k", [64, 128])
@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_cholesky_near_identity_nonfinite_is_flagged(bad, k):
    # a near-identity Gram (the series path's domain) with one non-finite off-diagonal pair must
    # not come back as a finite-looking factor with status 0 (fmax dropped NaN)
    g = np.eye(k) + 1e-14 * np.random.default_rng(5).standard_normal((k, k))
    g = 0.5 * (g + g.T)
    g[3, 40] = g[40, 3] = bad
    r, rinv, st = _small(0, g)
    assert st[0] != 0 or not (np.isfinite(r).all() and np.isfinite(rinv).all())


@pytest.mark.parametrize("k", [1, 2, 3, 17, 64, 128, 255])
def test_maxeig(k):
    rng = np.random.default_rng(100 + k)
    x = rng.standard_normal((k + 3, k)) * 1e-3
    a = x.T @ x
    lam, _, _ = _small(1, a)
    ref = np.linalg.eigvalsh(a)[-1]
    assert abs(lam[0, 0] - ref) <= 1e-12 * abs(ref)


def test_maxeig_clustered_top():
    rng = np.random.default_rng(7)
    q = np.linalg.qr(rng.standard_normal((64, 64)))[0]
    ev = np.concatenate([[1.0, 1.0 - 1e-12, 1.0 - 2e-12], np.linspace(0.5, 1e-8, 61)])
    a = (q * ev) @ q.T
    lam, _, _ = _small(1, a)
    assert abs(lam[0, 0] - 1.0) < 1e-13


@pytest.mark.parametrize("k", [1, 5, 32, 64, 100, 128, 150, 256])
@pytest.mark.parametrize("eps", [0.0, 1e-15, 1e-12, 1e-10, 3e-6])
def test_cholesky_near_identity_series(k, eps):
    """Near-identity Grams (the second CholeskyQR2 pass) take the series path: R and R^-1 agree
    with the Cholesky factor to rounding level and R^T R reproduces G."""
    rng = np.random.default_rng(int(k * 1000 + eps * 1e15) % 2**32)
    e = rng.standard_normal((k, k)) * eps
    g = np.eye(k) + (e + e.T) / 2
    r, rinv, st = _small(0, g)
    assert st == (0, 0)
    ref = np.linalg.cholesky(g).T
    # k > 64: first-order path (k max|E| <= 1e-9) or the general sweep, whose k-long sums round
    atol = 4e-16 if k <= 64 else 2e-15
    np.testing.assert_allclose(r, ref, rtol=0, atol=atol)
    np.testing.assert_allclose(r.T @ r, g, rtol=0, atol=atol)
    np.testing.assert_allclose(rinv @ r, np.eye(k), rtol=0, atol=atol)
    assert np.all(np.tril(rinv, -1) == 0.0) and np.all(np.tril(r, -1) == 0.0)


@pytest.mark.parametrize("rows,k", [(20000, 64), (9001, 37), (50000, 8)])
def test_tall_skinny_qr(rows, k):
    """CholeskyQR2 on the tall-skinny kernels (symmetric Gram, triangular products) reproduces
    the Householder QR: orthonormal Q, R with a nonnegative diagonal, A = Q R."""
    from paper_2512_05749_b200 import linalg

    g = torch.Generator(device="cuda").manual_seed(rows + k)
    a = torch.randn(rows, k, dtype=torch.float64, device="cuda", generator=g)
    a = a * torch.logspace(-3, 3, k, dtype=torch.float64, device="cuda")
    q, r = linalg.qr_orthonormalize(a)
    eye = torch.eye(k, dtype=torch.float64, device="cuda")
    assert (q.t() @ q - eye).abs().max().item() < 1e-13
    assert ((q @ r - a).norm() / a.norm()).item() < 1e-14
    q2, r2 = torch.linalg.qr(a)
    s = torch.sign(torch.diagonal(r2))
    r2 = r2 * s[:, None]
    assert ((r - r2).norm() / r2.norm()).item() < 1e-12
    assert torch.all(torch.tril(r, -1) == 0)
