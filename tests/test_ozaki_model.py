"""Host model of K4z's arithmetic (leaf_ozaki.cu): the signed 8-bit digit
split (k_oz_split) and the digit-pair schedule of the MMAs, checked on the CPU
-- digits in int8 range, reconstruction exact to 2^-63 of the row scale,
each kept digit pair formed exactly once, and the product of the model within
FP64 rounding of an extended-precision product."""

from fractions import Fraction

import numpy as np

# the 10 MMAs: A slices (p, p+1) x B slices (q, q+1) into tile (p + q) / 2
COMBOS = [(0, 0), (0, 2), (2, 0), (0, 4), (2, 2), (4, 0), (0, 6), (2, 4), (4, 2), (6, 0)]


def exponents(x, axis):
    m = np.abs(x).max(axis)
    f, e = np.frexp(m)
    return np.where(m > 0, e + (f >= 0.994140625), 0)


def digits(x, e, rows=True):
    """x 2^-E = s_0 2^-7 + sum_p s_p 2^-(7+8p): floor digits of |x|, a carry
    pass (threshold 129 for x < 0), negation for x < 0 (leaf_ozaki.cu)."""
    sc = np.ldexp(1.0, -e)
    neg = x < 0
    t = np.abs(x) * (sc[:, None] if rows else sc[None, :]) * 128.0
    d0 = np.floor(t)
    r = t - d0
    u = []
    for _ in range(7):
        t = r * 256.0
        f = np.floor(t)
        r = t - f
        u.append(f)
    s = [None] * 8
    c = np.zeros_like(x)
    thr = np.where(neg, 129, 128)
    for p in range(7, 0, -1):
        v = u[p - 1] + c
        c = (v >= thr).astype(np.float64)
        s[p] = v - 256 * c
    s[0] = d0 + c
    return [np.where(neg, -v, v).astype(np.int64) for v in s]


def model_product(a, b):
    ea, eb = exponents(a, 1), exponents(b, 0)
    da, db = digits(a, ea, True), digits(b, eb, False)
    s = {}
    for p, q in COMBOS:
        for i in (0, 1):
            for j in (0, 1):
                s[p + q + i + j] = s.get(p + q + i + j, 0) + da[p + i] @ db[q + j]
    v = np.zeros(a.shape[0:1] + b.shape[1:2])
    for d in range(10, -1, -1):
        v = v * 2.0 ** -8 + s.get(d, 0)
    return np.ldexp(v, ea[:, None] + eb[None, :] - 14), da


def test_digit_range_and_exact_reconstruction():
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (64, 64)) * np.exp(rng.uniform(-40, 40, (64, 64)))
    x[3] = 0.0
    x[5, 7] = np.nextafter(1.0, 0) * 2.0 ** 5   # mantissa just below 1: exponent bump
    e = exponents(x, 1)
    ds = digits(x, e)
    for d in ds:
        assert d.min() >= -128 and d.max() <= 127
    # exact (rational) remainder of the 8-digit expansion: the digits of |x|
    # leave |x 2^-E - sum_p s_p 2^-(7+8p)| < 2^-63
    for r in range(64):
        for c in range(0, 64, 3):
            xr = Fraction(float(x[r, c])) / Fraction(2) ** int(e[r])
            rec = sum(Fraction(int(ds[p][r, c])) / Fraction(2) ** (7 + 8 * p) for p in range(8))
            assert abs(xr - rec) < Fraction(1, 2 ** 63)
    assert not any(d[3].any() for d in ds)


def test_pair_schedule_covers_low_digit_sums_once():
    seen = {}
    for p, q in COMBOS:
        for i in (0, 1):
            for j in (0, 1):
                seen[(p + i, q + j)] = seen.get((p + i, q + j), 0) + 1
    assert max(seen.values()) == 1
    assert all((p, q) in seen for p in range(8) for q in range(8) if p + q <= 7)
    assert len({(p + q) // 2 for p, q in COMBOS}) == 4      # 4 TMEM tiles of 128 columns
    # exact int32 headroom: 128-task chunks, <= 4 pairs per quadrant, K = 64
    assert 128 * 4 * 64 * 128 * 128 * 2 < 2 ** 31


def test_model_product_beats_fp64_rounding():
    rng = np.random.default_rng(1)
    n = 256
    i = np.arange(n)
    a = rng.uniform(-1, 1, (n, n)) * np.exp(-0.05 * np.abs(i[:, None] - i[None, :]))
    a = np.triu(a) + np.triu(a, 1).T
    c, _ = model_product(a, a)
    ex = a.astype(np.longdouble) @ a.astype(np.longdouble)
    e_model = float(np.linalg.norm((c - ex).astype(np.float64)) / np.linalg.norm(ex.astype(np.float64)))
    e_fp64 = float(np.linalg.norm((a @ a - ex).astype(np.float64)) / np.linalg.norm(ex.astype(np.float64)))
    assert e_model < 1e-16 and e_model < e_fp64
    assert np.array_equal(c, c.T)   # exact digit sums: symmetric operands give symmetric C
