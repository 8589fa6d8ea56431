"""The int8 digit scheme of the O-passes (csrc/ozaki.cu), restated in numpy: the arithmetic the
kernels rely on, checked on the CPU.

* digitising (ozaki.cu biased_digits), s = 2^(54 - e) with |x - mu| < 2^e:
  X = rint(x s) - rint(mu s) when |mu| < 2^(e + 1) (integer centring), else
  X = rint((x - mu) s) (x - mu exact by Sterbenz), biased by 0x80 in each of the low 7 bytes
  (kBias); plane a holds byte 6 - a XOR 0x80, a signed digit (pack_digits8).  The 7 signed digits
  reconstruct X exactly, and X is (x - mu) to one unit of 2^-54 of the column scale;
* products: level s = a + b collects the digit pairs of one significance; the kernels keep
  s <= 6 (28 pairs, NL = 7 TMEM levels; s <= 7, 34 pairs, with -DWSSR_OZ_LEVELS=8) and combine
  the int32 level sums in FP64.  The dropped pairs weigh at most 2^-56 of the top level (2^-64
  for NL = 8), so every product is exact to 2^-51.4 (2^-59) of the column-scale product and the
  sum over K adds no rounding - the size of the FP64 rounding of the same dot product.
CPU-only."""

import numpy as np

import pytest

ND = 7
BIAS = np.uint64(0x0080808080808080)


def digit_ints(x, mu, e):
    """X of ozaki.cu biased_digits (np.rint is round-half-even, like the device conversion)."""
    e = max(e, -968)  # ozaki.cu kMinScaleExp: the scale factor stays finite
    s = np.ldexp(1.0, 54 - e)
    if abs(mu) < np.ldexp(1.0, e + 1):
        return np.rint(x * s).astype(np.int64) - np.int64(np.rint(mu * s))
    d = x - mu  # exact (Sterbenz): every x lies within 2^e of mu, and |mu| >= 2^(e+1)
    assert np.all(d + mu == x)
    return np.rint(d * s).astype(np.int64)


def digits(x, mu, e):
    X = digit_ints(x, mu, e)
    y = X.astype(np.uint64) + BIAS
    planes = [(((y >> np.uint64(8 * (6 - a))) & np.uint64(0xFF)) ^ np.uint64(0x80))
              .astype(np.uint8).view(np.int8) for a in range(ND)]
    return X, np.stack(planes)


def test_digits_reconstruct_exactly():
    rng = np.random.default_rng(0)
    for scale in (1e-300, 1e-8, 1.0, 3e7, 1e300):
        x = rng.standard_normal(4096) * scale
        mu = x.mean()
        e = int(np.frexp(np.abs(x - mu).max())[1])
        X, planes = digits(x, mu, e)
        assert planes.min() >= -128 and planes[0].min() >= -64 and planes[0].max() <= 64
        rec = sum(planes[a].astype(object) * (256 ** (6 - a)) for a in range(ND))
        assert all(int(r) == int(v) for r, v in zip(rec, X))
        ec = max(e, -968)
        err = np.abs(np.ldexp(X.astype(np.float64), ec - 54) - (x - mu)).max()
        # one unit against the exact x - mu (two half-unit roundings), plus the half-ulp rounding
        # of the reference fl(x - mu) itself (one unit in the top binade)
        assert err <= np.ldexp(1.0, ec - 53) * (1 + 1e-12)


def test_both_centring_forms_stay_in_digit_range():
    """A column whose mean dwarfs its spread takes the exact-difference form; one whose mean is
    below 2^(e+1) the integer form.  Both keep |X| <= 2^54 + 1 and one unit of accuracy."""
    rng = np.random.default_rng(7)
    for mu_scale in (0.0, 0.7, 1.9, 2.1, 1e3, 1e12):
        x = 1.0 + 0.5 * rng.standard_normal(2048)
        x = x - x.mean() + mu_scale
        mu = x.mean()
        e = int(np.frexp(np.abs(x - mu).max())[1])
        X, planes = digits(x, mu, e)
        assert np.abs(X).max() <= 2 ** 54 + 1
        rec = sum(planes[a].astype(object) * (256 ** (6 - a)) for a in range(ND))
        assert all(int(r) == int(v) for r, v in zip(rec, X))
        err = np.abs(np.ldexp(X.astype(np.float64), e - 54) - (x - mu)).max()
        assert err <= np.ldexp(1.0, e - 53) * (1 + 1e-12)


@pytest.mark.parametrize("NL,npairs,acc", [(7, 28, 2.0 ** -43), (8, 34, 2.0 ** -48)])
def test_truncated_pair_product_is_fp64_grade(NL, npairs, acc):
    rng = np.random.default_rng(1)
    K = 4096
    a = rng.standard_normal(K) * np.exp(rng.uniform(-4, 4, K))
    b = rng.standard_normal(K)
    ea = int(np.frexp(np.abs(a).max())[1])
    eb = int(np.frexp(np.abs(b).max())[1])
    XA, pa = digits(a, 0.0, ea)
    XB, pb = digits(b, 0.0, eb)
    levels = np.zeros(NL, dtype=np.int64)   # int32 per K-chunk on the device; exact here
    pairs = 0
    for i in range(ND):
        for j in range(ND):
            if i + j < NL:
                levels[i + j] += int(np.dot(pa[i].astype(np.int64), pb[j].astype(np.int64)))
                pairs += 1
    assert pairs == npairs
    got = sum(np.ldexp(float(levels[s]), 8 * (12 - s) + ea + eb - 108) for s in range(NL))
    exact = sum(int(u) * int(v) for u, v in zip(XA, XB))             # the digitised operands
    exact_f = np.ldexp(float(exact), ea + eb - 108)
    # dropped levels s >= NL: at most 13 - s pairs of 128 x 128 at weight 2^(8 (12 - s))
    bound = K * 128 * 128 * 2.0 ** (8 * (12 - NL) + ea + eb - 108) * (13 - NL) * (1 + 2.0 ** -7)
    assert abs(got - exact_f) <= bound + 4 * np.finfo(float).eps * abs(exact_f)
    ref = float(np.dot(a.astype(np.longdouble), b.astype(np.longdouble)))
    scale = np.abs(a) @ np.abs(b)
    assert abs(got - ref) <= acc * scale
