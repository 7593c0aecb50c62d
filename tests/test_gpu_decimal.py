"""GPU decimal text: parse_decimal / normalize_dataset /
format_scaled_decimal on the device (rs_sort_decimal_strings,
rs_format_decimals) against the reference library itself (oracle/_ref:
sort_decimals, sort.cpp:16-27) — values, reports, and the status and message
of the first failing numeral."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rep(r):
    return (r.written, r.cells_traversed, (r.spec.radix, r.spec.total_digits, r.spec.integer_digits))


def _numerals(seed, n, max_int_digits=4, max_frac=3):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        ip = str(int(rng.integers(0, 10 ** int(rng.integers(0, max_int_digits + 1)))))
        form = rng.integers(0, 5)
        if form == 0:
            out.append(ip)                                   # integer numeral
        elif form == 1:
            out.append("0" * int(rng.integers(1, 3)) + ip)  # leading zeros
        else:
            fd = int(rng.integers(1, max_frac + 1))
            fp = str(int(rng.integers(0, 10 ** fd))).rjust(fd, "0")
            out.append(("" if form == 2 and rng.random() < 0.3 else ip) + "." + fp)  # '.5' style too
    return out


@pytest.mark.parametrize("seed,n,digits,frac", [(1, 1000, 4, 3), (2, 20000, 2, 5), (3, 5000, 6, 0), (4, 777, 1, 1)])
def test_sort_decimals_vs_reference(rs, ref, seed, n, digits, frac):
    values = _numerals(seed, n, digits, max(frac, 1) if frac else 1) if frac else \
        [str(v) for v in np.random.default_rng(seed).integers(0, 10 ** digits, n)]
    want, wrep = ref.sort_decimals(values)
    got, rep = rs.sort_decimals(values)
    assert got == want
    assert _rep(rep) == wrep


def test_sort_decimal_keys_vs_reference(rs, ref):
    values = _numerals(9, 3000)
    want, wrep = ref.sort_decimals(values)
    keys, rep = rs.sort_decimal_keys(values)
    scale = rep.spec.scale
    assert [rs._format_scaled(k, scale) for k in keys] == want
    assert _rep(rep) == wrep


@pytest.mark.parametrize("bad", [
    ["1.5", ""],                      # empty numeral
    ["2", "-3", "x"],                 # negative before the later parse error
    ["1.2.3"],                        # multiple decimal points
    ["7", "5."],                      # no digits after the point
    ["."],                            # point only
    ["1e5"], ["12a"], ["+1"],         # invalid characters
    ["99999999999999999999"],         # mantissa overflows 64 bits
    ["0.000000000000000000001"],      # 10^21: integer_part's power overflows
    ["1.0", "123456789.123"],         # key space above the default budget
])
def test_errors_match_reference(rs, ref, bad):
    from oracle import OracleError

    with pytest.raises(OracleError) as want:
        ref.sort_decimals(bad)
    with pytest.raises(rs.Error) as got:
        rs.sort_decimals(bad)
    status_name = rs._lib.load().rs_status_name(want.value.status).decode()
    assert got.value.code == status_name
    assert str(got.value) == want.value.message


def test_first_failing_numeral_wins(rs):
    values = ["1"] * 5000 + ["-2"] + ["1"] * 5000 + ["x"]
    with pytest.raises(rs.Error) as e:
        rs.sort_decimals(values)
    assert e.value.code == "negative_value" and "'-2'" in str(e.value)


def test_empty_input(rs, ref):
    assert rs.sort_decimals([])[0] == ref.sort_decimals([])[0] == []


def test_large_column_on_device(rs):
    """2^22 numerals (1 to 6 integer digits, 0 to 3 fractional digits) parsed,
    sorted and rendered on the device; checked against numpy."""
    import torch

    rng = np.random.default_rng(21)
    n = 1 << 22
    ip = rng.integers(0, 10 ** 6, n)
    fd = rng.integers(0, 4, n)
    fp = rng.integers(0, 1000, n) % (10 ** fd)
    values = [f"{a}.{str(b).rjust(d, '0')}" if d else str(a) for a, b, d in zip(ip.tolist(), fp.tolist(), fd.tolist())]
    chars, offsets = rs._string_column(values)
    keys, rep = rs.sort_decimal_column(torch.from_numpy(chars.copy()).cuda(),
                                       torch.from_numpy(offsets.view(np.int64)).cuda(), max_cells=10**9)
    scaled = ip.astype(np.uint64) * np.uint64(1000) + fp.astype(np.uint64) * (10 ** (3 - fd)).astype(np.uint64)
    assert rep.spec.scale == 3 and rep.spec.integer_digits == len(str(int(ip.max())))
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), np.sort(scaled))
    out_chars, out_off = rs.format_decimal_column(keys, 3)
    text = bytes(out_chars.cpu().numpy())
    off = out_off.cpu().numpy()
    for i in (0, 1, n // 2, n - 1):
        k = int(np.sort(scaled)[i])
        assert text[off[i]:off[i + 1]].decode() == f"{k // 1000}.{str(k % 1000).rjust(3, '0')}"


@pytest.mark.parametrize("misalign", [0, 1, 3, 7])
def test_parse_every_shape_and_alignment(rs, misalign):
    """rs_parse_decimals over numerals of every length 1-19 with the point at
    every position (the SWAR fast path takes <= 16 bytes with at most one
    point that is not the last byte; longer numerals take the byte loop), each
    starting at every byte alignment, in a column whose first byte sits at
    `misalign` bytes past an 8-byte boundary, the last numerals ending at the
    column's last byte (where the fast path's third word would run past it)."""
    import ctypes

    import torch

    rng = np.random.default_rng(100 + misalign)
    vals = []
    for length in range(1, 20):
        for dot in [None] + list(range(0, length - 1)):
            for _ in range(3):
                nd = length - (dot is not None)
                digits = "".join(str(d) for d in rng.integers(0, 10, nd))
                vals.append(digits if dot is None else digits[:dot] + "." + digits[dot:])
    rng.shuffle(vals)
    vals += ["0", "7.5", "12.34"]  # short numerals at the very end
    data = "".join(vals).encode()
    offsets = np.zeros(len(vals) + 1, dtype=np.uint64)
    offsets[1:] = np.cumsum([len(v) for v in vals])
    buf = torch.zeros(len(data) + misalign, dtype=torch.uint8, device="cuda")
    buf[misalign:] = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    chars = buf[misalign:]
    off = torch.from_numpy(offsets.view(np.int64)).cuda()
    mant = torch.empty(len(vals), dtype=torch.int64, device="cuda")
    scales = torch.empty(len(vals), dtype=torch.int32, device="cuda")
    lib = rs._lib.load()
    rs._check(lib.rs_parse_decimals(ctypes.c_void_p(chars.data_ptr()), rs._ptr(off), len(vals), rs._ptr(mant),
                                    rs._ptr(scales), rs._stream()))
    want_m = [int(v.replace(".", "")) for v in vals]
    want_s = [len(v) - v.index(".") - 1 if "." in v else 0 for v in vals]
    assert [int(x) for x in mant.cpu().numpy().view(np.uint64)] == want_m
    assert scales.cpu().tolist() == want_s
