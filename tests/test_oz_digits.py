"""The staging kernels' Ozaki digit extraction (stage.cu oz_digits): one scaled truncation and
integer fields must give exactly the digits of the iterated exact form v = 128 u, q = trunc(v),
u = v - q (the form the INT8 Gram's error bound is derived for, ozaki.cu).  numpy restatement of
both on adversarial values: exact binary fractions, values next to digit boundaries, tiny and
subnormal values, signed zeros, values just below 1."""

import numpy as np

DIGITS = 4


def iterated(u):
    out = []
    for _ in range(DIGITS):
        v = u * 128.0
        q = np.trunc(v)
        u = v - q
        out.append(q.astype(np.int64))
    return np.stack(out)


def scaled(u):
    t = u * 2.0 ** (7 * DIGITS)  # z * 2^(28 - e) with u = z * 2^-e
    q = np.trunc(t).astype(np.int64)
    au, neg = np.abs(q), q < 0
    out = []
    for a in range(DIGITS):
        d = (au >> (7 * (DIGITS - 1 - a))) & 127
        out.append(np.where(neg, -d, d))
    return np.stack(out)


def test_digits_match_the_iterated_form():
    rng = np.random.default_rng(0)
    u = np.concatenate([
        rng.uniform(-1, 1, 200000),
        rng.uniform(-1, 1, 1000) * 2.0 ** -rng.integers(1, 60, 1000),
        np.nextafter(1.0, 0.0) * np.array([1, -1]),
        np.array([0.0, -0.0, 5e-324, -5e-324, 2.0 ** -28, -(2.0 ** -28), 2.0 ** -29]),
        (rng.integers(-2 ** 27, 2 ** 27, 5000) / 2.0 ** 27),
        np.nextafter(rng.integers(-2 ** 20, 2 ** 20, 5000) / 2.0 ** 21, 0.0),
    ])
    assert np.array_equal(iterated(u), scaled(u))
    assert np.abs(scaled(u)).max() <= 127
