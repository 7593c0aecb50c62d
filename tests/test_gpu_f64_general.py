"""GPU float_to_decimal for every double: rs_float_to_decimal
and rs_sort_f64 against the reference library itself (oracle/_ref,
key_model.cpp:135-158) — random bit patterns over the whole exponent range,
magnitudes where outputs are not errors, integers past 2^53 (and the
wrapping upscale past 2^64), subnormals, powers of two and ten, half-way
ties, scales 0..40, and the first failing element's status and message."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCALES = [0, 1, 2, 3, 6, 9, 12, 15, 16, 17, 19, 20, 25, 33, 40]


def _bitpatterns(seed, n):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 0x7FF0000000000000, n, dtype=np.uint64).view(np.float64)  # finite, >= 0
    return x


def _moderate(seed, n, lo=-25.0, hi=20.0):
    rng = np.random.default_rng(seed)
    return 10.0 ** rng.uniform(lo, hi, n)


def _specials():
    v = [0.0, 5e-324, 2.2250738585072014e-308, 1e-30, 1e-20, 0.1, 0.5, 1.0, 2.5, 123.456, 2.0 ** 50 + 0.25,
         2.0 ** 50 + 0.75, 2.0 ** 51 + 0.5, 2.0 ** 52 + 0.5, 2.0 ** 53 - 1, 2.0 ** 53, 2.0 ** 53 + 2, 1e16, 1e17,
         2.0 ** 60, 1e19, 1.8e19, 18446744073709549568.0]
    v += [2.0 ** e for e in range(-1074, 64, 3)] + [10.0 ** e for e in range(-40, 20)]
    v += [math.nextafter(a, math.inf) for a in list(v) if a > 0] + [math.nextafter(a, 0.0) for a in list(v) if a > 0]
    base = 2.0 ** 50
    v += [base + i + f for i in range(0, 3000, 7) for f in (0.25, 0.75)]
    return np.array(v, dtype=np.float64)


def _compare_valid(rs, ref, x, scale):
    """Elements the reference maps: bit-identical mantissas."""
    import torch

    want, st = ref.float_to_decimal_many(x, scale)
    ok = st == 0
    if not ok.any():
        return 0
    got = rs.float_to_decimal_column(torch.from_numpy(x[ok]).cuda(), scale)
    g = got.cpu().numpy().view(np.uint64)
    bad = np.nonzero(g != want[ok])[0]
    assert bad.size == 0, [(x[ok][i], scale, int(g[i]), int(want[ok][i])) for i in bad[:5]]
    return int(ok.sum())


@pytest.mark.parametrize("scale", SCALES)
def test_float_to_decimal_bit_patterns(rs, ref, scale):
    assert _compare_valid(rs, ref, _bitpatterns(scale, 200_000), scale) >= 0


@pytest.mark.parametrize("scale", SCALES)
def test_float_to_decimal_moderate(rs, ref, scale):
    n = _compare_valid(rs, ref, _moderate(50 + scale, 200_000, -scale - 21, 20.0), scale)
    assert n > 10_000  # this band is mostly mappable


@pytest.mark.parametrize("scale", SCALES)
def test_float_to_decimal_specials(rs, ref, scale):
    _compare_valid(rs, ref, _specials(), scale)


def test_float_to_decimal_every_status(rs, ref):
    """An element that fails stops the column at the first failure in input
    order, with the reference's status and message."""
    import torch

    from oracle import OracleError

    cases = [([1.5, 2.5, 1e-30, float("nan")], 3), ([1.0, float("inf"), -1.0], 3), ([1.0, -2.0, float("nan")], 3),
             ([3.0, 1.9e19], 0), ([0.25, 1e300], 2), ([7.0], 20), ([1.5], 30), ([2.0, 5e-324], 3)]
    for vals, scale in cases:
        first = None
        for v in vals:
            try:
                ref.float_to_decimal(v, scale)
            except OracleError as e:
                first = e
                break
        assert first is not None
        with pytest.raises(rs.Error) as got:
            rs.float_to_decimal_column(torch.tensor(vals, dtype=torch.float64, device="cuda"), scale)
        assert got.value.code == rs._lib.load().rs_status_name(first.status).decode(), (vals, scale)
        assert str(got.value) == first.message, (vals, scale)


@pytest.mark.parametrize("scale", [0, 1, 3, 6])
def test_sort_f64_general_vs_reference(rs, ref, scale):
    """rs_sort_f64 over values outside the fast mapper's domain (tiny values
    that map to 0 or 1 — the lean sort hands over to the general mapper):
    same keys and report as the reference's float_to_decimal + grid."""
    import torch

    rng = np.random.default_rng(scale)
    x = 10.0 ** rng.uniform(-(scale + 12), 8.5 - scale, 100_000)  # keys < 10^9 cells
    want_m, st = ref.float_to_decimal_many(x, scale)
    x = x[st == 0]
    want, wrep = ref.sort_f64(x, scale, max_cells=10**12)
    got, rep = rs.sort_f64(torch.from_numpy(x).cuda(), scale, max_cells=10**12)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), want)
    assert (rep.written, rep.cells_traversed, (rep.spec.radix, rep.spec.total_digits,
                                                rep.spec.integer_digits)) == wrep


def test_sort_f64_first_error_in_order(rs, ref):
    import torch

    from oracle import OracleError

    x = np.full(100_000, 1.25)
    x[70_000] = -3.0
    x[90_000] = float("nan")
    x[20_000] = 1e-40  # first: its numeral has 40 fractional digits -> 10^37 at scale 3
    with pytest.raises(OracleError) as want:
        ref.sort_f64(x, 3)
    with pytest.raises(rs.Error) as got:
        rs.sort_f64(torch.from_numpy(x).cuda(), 3)
    assert got.value.code == rs._lib.load().rs_status_name(want.value.status).decode()
    assert str(got.value) == want.value.message


@pytest.mark.parametrize("scale", [16, 19, 20, 33])
def test_sort_f64_high_scales_fail_like_reference(rs, ref, scale):
    """scale >= 16: every grid has >= 10^17 cells (scale > 19: 10^scale itself
    overflows) — the reference's error, after the element checks."""
    import torch

    from oracle import OracleError

    x = np.array([0.5, 1e-9, 3.25e-12, 0.0])
    with pytest.raises(OracleError) as want:
        ref.sort_f64(x, scale, max_cells=10**12)
    with pytest.raises(rs.Error) as got:
        rs.sort_f64(torch.from_numpy(x).cuda(), scale, max_cells=10**12)
    assert got.value.code == rs._lib.load().rs_status_name(want.value.status).decode()
    assert str(got.value) == want.value.message
