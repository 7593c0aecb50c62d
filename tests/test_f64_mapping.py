"""The GPU's float_to_decimal (MapF64 in csrc/kernels_grid.cuh) replaces the
reference's string round trip (key_model.cpp:135-158) with exact IEEE tests.
This restates the kernel's arithmetic step for step in Python (Python floats
are IEEE doubles; fma is emulated exactly with Fraction) and checks it
against the oracle / reference float_to_decimal on the kernel's domain
x * 10^(scale+2) < 2^53, including the half-way and nudged cases."""
import math
from fractions import Fraction

import numpy as np
import pytest

LIMIT = 9007199254740992.0 / 100.0


def kernel_f64(x: float, scale: int):
    """Line-by-line mirror of MapF64::operator()."""
    P = float(10 ** scale)
    P2 = 2.0 * P
    if math.isnan(x) or math.isinf(x):
        return "non_finite"
    if x < 0.0:
        return "negative"
    p = x * P
    if not (p < LIMIT) or (x > 0.0 and x < 1.0000001 * 10.0 ** -(scale + 3)):
        return "domain"
    err = float(Fraction(x) * Fraction(P) - Fraction(p))  # fma(x, P, -p)
    f = float(math.floor(p))
    if p == f and err < 0.0:
        f -= 1.0
    m = int(f)
    fr = p - f
    if fr < 0.02 or fr > 0.98:
        c = m if fr < 0.5 else m + 1
        if float(c) / P == x:
            return c
    elif 0.48 < fr < 0.52:
        if float(2 * m + 1) / P2 == x:
            return m + 1
    up = fr > 0.5 or (fr == 0.5 and err > 0.0)
    return m + 1 if up else m


def _fma(a: float, b: float, c: float) -> float:
    """Exactly rounded a*b + c (IEEE fma)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def quotient_is(x: float, c: float, d: float):
    """Mirror of quotient_is (kernels_grid.cuh): is x == RN(c / d)?  1 yes,
    0 no, -1 undecided (the kernel then takes the exact path)."""
    xb = np.float64(x).view(np.uint64).item()
    ulp = np.uint64((xb & 0x7FF0000000000000) - (52 << 52)).view(np.float64).item()
    h = d * ulp * 0.5
    r = abs(_fma(-x, d, c))
    if (xb & ((1 << 52) - 1)) == 0 or r == h:
        return -1
    return 1 if r < h else 0


def kernel_f64_fast(x: float, scale: int):
    """Mirror of MapF64::fast; None = undecided (the kernel falls back to
    MapF64::operator(), mirrored by kernel_f64)."""
    P = float(10 ** scale)
    p = x * P
    if not (x >= 0.0) or not (p < LIMIT) or (x > 0.0 and x < 1.0000001 * 10.0 ** -(scale + 3)):
        return None
    err = _fma(x, P, -p)
    f = float(math.floor(p))
    if p == f and err < 0.0:
        f -= 1.0
    m = int(f)
    fr = p - f
    near_int = fr < 0.02 or fr > 0.98
    near_half = 0.48 < fr < 0.52
    c = m if fr < 0.5 else m + 1
    cv, dv = (float(c), P) if near_int else (float(2 * m + 1), 2.0 * P)
    q = 1 if x == 0.0 else (quotient_is(x, cv, dv) if (near_int or near_half) else 0)
    if q == -1:
        return None
    if q == 1:
        return c if near_int else m + 1
    return m + 1 if (fr > 0.5 or (fr == 0.5 and err > 0.0)) else m


def test_fast_path_matches_exact_path(oracle):
    rng = np.random.default_rng(5)
    undecided = decided = 0
    for scale in (0, 1, 2, 3, 6, 9, 12, 15):
        xs = [float(v) / 10.0 ** scale for v in rng.integers(0, 10 ** 7, 2000)]
        xs += [(2 * float(v) + 1) / (2 * 10.0 ** scale) for v in rng.integers(0, 10 ** 7, 1000)]
        xs += [float(np.nextafter((2 * float(v) + 1) / (2 * 10.0 ** scale), np.inf if v % 2 else 0.0))
               for v in rng.integers(0, 10 ** 7, 500)]
        xs += list(rng.random(1000) * 1e3) + [2.0 ** e for e in range(-40, 30)] + [0.0]
        for x in xs:
            if not in_domain(x, scale):
                continue
            got = kernel_f64_fast(x, scale)
            if got is None:
                undecided += 1
            else:
                decided += 1
                assert got == kernel_f64(x, scale) == oracle.float_to_decimal(x, scale), (x, scale)
    assert undecided < decided / 20


def test_quotient_test_agrees_with_division():
    """Whenever the division-free test decides, it agrees with IEEE division."""
    rng = np.random.default_rng(7)
    decided = 0
    for _ in range(20000):
        scale = int(rng.integers(0, 16))
        d = float(10 ** scale) * (2.0 if rng.random() < 0.3 else 1.0)
        c = float(int(rng.integers(0, 2 ** 40)))
        q = c / d
        for x in (q, float(np.nextafter(q, np.inf)), float(np.nextafter(q, 0.0))):
            t = quotient_is(x, c, d)
            if t != -1:
                decided += 1
                assert (t == 1) == (c / d == x), (x, c, d)
    assert decided > 50000


def in_domain(x: float, scale: int) -> bool:
    return x * 10.0 ** scale < LIMIT and (x == 0.0 or x >= 1.0000001 * 10.0 ** -(scale + 3))


def test_known_answers():
    # test_key_model.cpp:80-93
    assert kernel_f64(4.5, 1) == 45
    assert kernel_f64(0.0, 3) == 0
    assert kernel_f64(-0.0, 3) == 0
    assert kernel_f64(2.345, 2) == 235
    assert kernel_f64(0.285, 2) == 29
    assert kernel_f64(2.344, 2) == 234
    assert kernel_f64(7.0, 0) == 7
    assert kernel_f64(-1.0, 2) == "negative"
    assert kernel_f64(float("nan"), 1) == "non_finite"
    assert kernel_f64(float("inf"), 1) == "non_finite"


def test_matches_reference_golden(golden):
    xs = golden["f2d_x"]
    for scale in (0, 1, 2, 3, 4, 6):
        want = golden[f"f2d_scale{scale}"]
        for x, w in zip(xs.tolist(), want.tolist()):
            if in_domain(x, scale):
                assert kernel_f64(x, scale) == w, (x, scale)


@pytest.mark.parametrize("scale", [0, 1, 2, 3, 5, 8])
def test_matches_oracle_random(oracle, scale):
    rng = np.random.default_rng(1000 + scale)
    top = LIMIT / 10.0 ** scale
    k = rng.integers(0, 10 ** 7, 4000)
    xs = list(rng.random(4000) * min(top, 1e4))
    xs += [float(v) / 10.0 ** scale for v in k[:1000]]                       # exact decimals
    xs += [(2 * float(v) + 1) / (2 * 10.0 ** scale) for v in k[1000:2000]]   # half-way numerals
    xs += [float(np.nextafter((2 * float(v) + 1) / (2 * 10.0 ** scale), np.inf if v % 2 else 0.0))
           for v in k[2000:3000]]                                            # one ulp off half-way
    xs += list(np.exp(rng.uniform(-30, math.log(min(top, 1e12)), 1000)))    # wide magnitudes
    for x in xs:
        if not in_domain(x, scale):
            continue
        assert kernel_f64(x, scale) == oracle.float_to_decimal(x, scale), (x, scale)


def test_cfg3_values(oracle):
    # every cfg3 value k/1000 for a strided sweep of k in [0, 10^6)
    for k in range(0, 10 ** 6, 97):
        x = k / 1000.0
        assert kernel_f64(x, 3) == oracle.float_to_decimal(x, 3) == k
