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
