"""The GPU's general float_to_decimal (f2d_general in csrc/kernels_f64.cuh,
SURVEY 8f row 2): the reference's shortest round-trip fixed numeral
(std::to_chars, key_model.cpp:135-158) found by an exact integer search —
the fewest fractional digits k such that an integer N with N / 10^k lies in
x's rounding interval, N the nearest such integer (ties to even) — then the
reference's rescale / half-up / overflow rules.

This restates the kernel's arithmetic step for step with Python integers
(the kernel holds the same numbers in 64-bit limbs; the asserted bounds are
the ones its limb counts rely on) and checks it against the reference
library itself (oracle/_ref) on random bit patterns over the whole double
range, integers past 2^53 and 2^64, subnormals, powers of two and ten, and
half-way ties."""
import math
import struct

import numpy as np
import pytest

OK, NON_FINITE, NEGATIVE, DIGITS, POW = "ok", "non_finite", "negative", "digits", "pow"
MAX_SCALE = 40  # the kernel's 5^k table reaches k = MAX_SCALE + 19


def _bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _finish(M: int, F: int, s: int):
    """DecimalValue{M, F} at scale s (key_model.cpp:150-157)."""
    if F <= s:
        if s - F > 19:
            return POW, s - F
        return OK, (M * 10 ** (s - F)) % (1 << 64)  # unchecked product: wraps like the reference
    d = F - s
    if d > 19:
        return POW, d
    p = 10 ** d
    return OK, M // p + (1 if M % p >= p // 2 else 0)


def _k_est(x: float) -> int:
    """Lower bound on the shortest numeral's fractional digits (the kernel's
    double log10, one digit of margin)."""
    return max(0, int(math.floor(-math.log10(x))) - 1)


def f2d_general(x: float, s: int):
    """Mirror of f2d_general: (status, key or error exponent)."""
    if math.isnan(x) or math.isinf(x):
        return NON_FINITE, 0
    if x < 0.0:
        return NEGATIVE, 0
    if x == 0.0:
        return _finish(0, 0, s)
    if x >= 9007199254740992.0:  # >= 2^53: integer valued, printed exactly
        if x >= 18446744073709551616.0:
            return DIGITS, 0
        return _finish(int(x), 0, s)
    b = _bits(x)
    be, f = (b >> 52) & 0x7FF, b & ((1 << 52) - 1)
    m, q = (f, -1074) if be == 0 else (f | (1 << 52), be - 1075)
    sh = 2 - q  # x = 4m * 2^-sh; the rounding interval is [L4, U4] * 2^-sh
    X4, U4 = 4 * m, 4 * m + 2
    L4 = 4 * m - (1 if (f == 0 and be > 1) else 2)
    incl = m % 2 == 0  # round-half-even parse: even significands own their boundaries

    def quo(V: int, k: int):
        """floor(V * 10^k / 2^sh) and whether the division is exact."""
        A = V * 5 ** k
        assert A < 1 << 192  # three 64-bit limbs
        t = sh - k
        if t <= 0:
            return A << -t, True
        return A >> t, (A & ((1 << t) - 1)) == 0

    def bounds(k: int):
        qa, ea = quo(L4, k)
        lo = qa if ea else qa + 1
        if ea and not incl:
            lo += 1
        qb, eb = quo(U4, k)
        hi = qb - 1 if (eb and not incl) else qb
        return lo, hi

    k0 = _k_est(x)
    if s >= 20 and s - 20 >= k0:
        lo, hi = bounds(s - 20)
        if lo <= hi:  # a numeral with <= s-20 fractional digits: 10^(s-F) overflows
            return POW, -1
    start = max(k0, s - 19 if s >= 19 else 0)
    for k in range(start, min(s + 19, k0 + 20) + 1):
        lo, hi = bounds(k)
        if lo <= hi:
            break
    else:
        return POW, -1  # shortest numeral has > s+19 fractional digits
    assert hi < 1 << 70
    if lo == hi:
        N = lo
    else:  # the integer nearest x * 10^k, ties to even
        A = X4 * 5 ** k
        t = sh - k
        if t <= 0:
            N = A << -t
        else:
            qn, r, half = A >> t, A & ((1 << t) - 1), 1 << (t - 1)
            N = qn + (1 if (r > half or (r == half and qn & 1)) else 0)
        assert lo <= N <= hi
    assert N < 10 ** 17
    return _finish(N, k, s)


STATUS = {0: OK, 4: "cell_budget", 6: NEGATIVE, 7: NON_FINITE}


def _ref_status(ref, x, s):
    st, v = ref.float_to_decimal_status(x, s)
    return st, v


def _check(ref, x: float, s: int):
    got = f2d_general(x, s)
    st, v = ref.float_to_decimal_status(x, s)
    if st == 0:
        assert got == (OK, v), (x, s, got, v)
    else:
        assert got[0] != OK, (x, s, got, st)


def _random_doubles(seed: int, n: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 1 << 63, n, dtype=np.uint64)  # non-negative, every exponent
    return bits.view(np.float64)


@pytest.mark.parametrize("seed", range(4))
def test_general_random_bit_patterns(ref, seed):
    xs = _random_doubles(seed, 3000)
    rng = np.random.default_rng(100 + seed)
    for x, s in zip(xs.tolist(), rng.integers(0, MAX_SCALE + 1, xs.size).tolist()):
        if math.isfinite(x):
            _check(ref, x, s)


def test_general_moderate_magnitudes(ref):
    """Where outputs are not errors: x in [1e-25, 1e20), scales 0..25."""
    rng = np.random.default_rng(7)
    xs = 10.0 ** rng.uniform(-25, 20, 20000)
    for x, s in zip(xs.tolist(), rng.integers(0, 26, xs.size).tolist()):
        _check(ref, x, s)


def test_general_special_values(ref):
    vals = [0.0, -0.0, 5e-324, 2.2250738585072014e-308, 2.225073858507201e-308, 1e-30, 1e-20, 0.1, 0.5,
            1.0, 2.5, 123.456, 2.0 ** 50 + 0.25, 2.0 ** 50 + 0.75, 2.0 ** 51 + 0.5, 2.0 ** 52 + 0.5,
            2.0 ** 53 - 1, 2.0 ** 53, 2.0 ** 53 + 2, 1e16, 1e17, 2.0 ** 60, 1e19, 1.8e19,
            18446744073709549568.0, 2.0 ** 64, 1e300, 1.7976931348623157e308]
    vals += [2.0 ** e for e in range(-1074, 64, 7)] + [10.0 ** e for e in range(-30, 20)]
    vals += [math.nextafter(v, math.inf) for v in vals if v > 0] + [math.nextafter(v, 0.0) for v in vals if v > 0]
    for x in vals:
        for s in (0, 1, 2, 3, 6, 12, 15, 16, 19, 20, 25, 33, MAX_SCALE):
            _check(ref, x, s)


def test_general_half_way_ties(ref):
    """x = N + 1/4 (and 3/4) above 2^50: two 1-digit numerals tie; the
    reference's to_chars picks the even one (2^50 + 0.25 -> ...4.2)."""
    base = 2.0 ** 50
    for i in range(0, 4000, 7):
        for frac in (0.25, 0.75):
            x = base + i + frac
            for s in (0, 1, 2, 3):
                _check(ref, x, s)


def test_errors_agree(ref):
    for x, s in [(float("nan"), 3), (float("inf"), 3), (-1.0, 3), (1e-30, 3), (5e-324, 3), (1.9e19, 0),
                 (1e300, 2), (0.0, 25), (1.5, 30)]:
        st, _ = ref.float_to_decimal_status(x, s)
        got = f2d_general(x, s)
        assert st != 0 and got[0] != OK, (x, s, st, got)
