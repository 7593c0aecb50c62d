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
    """Line-by-line mirror of MapF64::exact (what operator() falls back to)."""
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


def _bits(x: float) -> int:
    return np.float64(x).view(np.uint64).item()


def _xlim_bits(scale: int) -> int:
    """make_map_f64 (capi.cu): bits of the least x with x * 10^scale >= LIMIT."""
    P = float(10 ** scale)
    xl = LIMIT / P
    while xl * P >= LIMIT:
        xl = float(np.nextafter(xl, 0.0))
    while xl * P < LIMIT:
        xl = float(np.nextafter(xl, np.inf))
    return _bits(xl)


def _fma(a: float, b: float, c: float) -> float:
    """Exactly rounded a*b + c (IEEE fma)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _sbits(x: float) -> int:
    return np.float64(x).view(np.int64).item()


def kernel_f64_fast(x: float, scale: int):
    """Line-by-line mirror of MapF64::fast; None = undecided (the kernel
    falls back to MapF64::exact, mirrored by kernel_f64)."""
    fast = scale <= 15
    P = float(10 ** scale) if fast else 1.0
    u = _bits(x)
    zero_bits = 0 if fast else 2 ** 64 - 1
    tiny_bits = _bits(1.0000001 * 10.0 ** -(scale + 3)) if fast else 0
    xlim_bits = _xlim_bits(scale) if fast else 0
    undecided = ((u - tiny_bits) & (2 ** 64 - 1)) >= ((xlim_bits - tiny_bits) & (2 ** 64 - 1)) and u != zero_bits
    if undecided:
        return None  # (the kernel computes on; its value is not used)
    p = x * P
    c = float(round(p))  # rint: ties to even
    d = p - c
    if (_sbits(d) >> 32) & 0x7FFFFFFF < 0x3FDEB851:
        return int(c)
    m = c if d >= 0.0 else c - 1.0
    dv = 2.0 * P
    hb = _sbits(dv) + (((u >> 52) - 1076) << 52)
    rb = _sbits(_fma(-x, dv, _fma(m, 2.0, 1.0))) & 0x7FFFFFFFFFFFFFFF
    if (u & ((1 << 52) - 1)) == 0 or rb == hb:
        return None
    if rb < hb:
        return int(m) + 1
    fr = p - m
    up = fr > 0.5 or (fr == 0.5 and _fma(x, P, -p) > 0.0)
    return int(m) + 1 if up else int(m)


def test_fast_path_matches_exact_path(oracle):
    rng = np.random.default_rng(5)
    decided = undecided = 0
    for scale in (0, 1, 2, 3, 6, 9, 12, 15):
        xs = [float(v) / 10.0 ** scale for v in rng.integers(0, 10 ** 7, 2000)]
        xs += [(2 * float(v) + 1) / (2 * 10.0 ** scale) for v in rng.integers(0, 10 ** 7, 1000)]
        xs += [float(np.nextafter((2 * float(v) + 1) / (2 * 10.0 ** scale), np.inf if v % 2 else 0.0))
               for v in rng.integers(0, 10 ** 7, 500)]
        xs += list(rng.random(1000) * 1e3) + [2.0 ** e for e in range(-40, 30)] + [0.0]
        # powers of two and their neighbours, and values at the fast domain's edges
        xs += [float(np.nextafter(2.0 ** e, t)) for e in range(-50, 40) for t in (0.0, np.inf)]
        top = LIMIT / 10.0 ** scale
        xs += [float(np.nextafter(top, 0.0)), top, 1.0000001 * 10.0 ** -(scale + 3)]
        for x in xs:
            got = kernel_f64_fast(x, scale)
            if not in_domain(x, scale):
                assert got is None or x == 0.0, (x, scale)
                continue
            if got is None:
                undecided += 1
                continue
            decided += 1
            assert got == kernel_f64(x, scale) == oracle.float_to_decimal(x, scale), (x, scale)
    assert decided > 30000 and undecided < decided / 20


def test_fast_path_neighbours():
    """Decimals scaled by 1, 1/2 and 1/4 and the doubles either side of them,
    against the division of exact()."""
    rng = np.random.default_rng(11)
    checked = 0
    for _ in range(4000):
        scale = int(rng.integers(1, 16))
        P = 10 ** scale
        x = float(rng.integers(1, 2 ** 40)) / float(P) * float(rng.choice([1.0, 0.5, 0.25]))
        if not in_domain(x, scale) or x == 0.0:
            continue
        for y in (x, float(np.nextafter(x, np.inf)), float(np.nextafter(x, 0.0))):
            got = kernel_f64_fast(y, scale)
            if in_domain(y, scale) and y > 0.0 and got is not None:
                assert got == kernel_f64(y, scale), (y, scale)
                checked += 1
    assert checked > 5000


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


def test_fast_path_product_rounded_onto_integer():
    """x = v / 10^scale whose product x * 10^scale rounds up onto the integer
    v (fr == 0, err < 0): the fast path takes no fix-up there (both
    candidates and the half-up rule give floor(p) = v)."""
    rng = np.random.default_rng(3)
    seen = 0
    for scale in (1, 2, 3, 6, 9):
        P = 10.0 ** scale
        for v in rng.integers(0, 10 ** 7, 3000).tolist():
            x = float(v) / P
            p = x * P
            if p == math.floor(p) and _fma(x, P, -p) < 0.0:
                seen += 1
                assert kernel_f64_fast(x, scale) == kernel_f64(x, scale) == v, (x, scale)
    assert seen > 1000
