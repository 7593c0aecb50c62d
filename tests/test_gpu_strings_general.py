"""Strings beyond cfg4: records wider than 12 bytes,
alphabets from 2 to 255 symbols, variable lengths (NUL-terminated within the
record), the reference's check order (key spec before symbols) and its
symbol message — the facade against the reference library (oracle/_ref),
and the MSD extension (keys packed b = bit_length(|alphabet|) bits per
ordinal, width * b <= 64) against an ordinal-order restatement."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALNUM = "0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz"   # byte order == ordinal order
BYTES255 = bytes(range(1, 256))  # every non-NUL byte (radix 256)


def _b(alphabet):
    return alphabet if isinstance(alphabet, bytes) else alphabet.encode()


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _records(seed, n, width, alphabet, short_every=5):
    rng = np.random.default_rng(seed)
    sym = np.frombuffer(_b(alphabet), dtype=np.uint8)
    recs = sym[rng.integers(0, len(sym), (n, width))]
    lens = rng.integers(1, width + 1, n)
    lens[::short_every] = width
    recs[np.arange(width)[None, :] >= lens[:, None]] = 0
    return np.ascontiguousarray(recs)


def _ordinal_order(recs, alphabet):
    ords = np.zeros(256, dtype=np.int64)
    sym = np.frombuffer(_b(alphabet), dtype=np.uint8)
    ords[sym] = np.arange(1, len(sym) + 1)
    o = ords[recs]
    return np.lexsort([o[:, j] for j in reversed(range(recs.shape[1]))]), o


def _report(sorted_ords, radix, w):
    """cells_traversed of the single grid for these keys (extraction.cpp:16-30):
    per leading ordinal, max suffix - min suffix + 1 (Python integers)."""
    first = sorted_ords[:, 0]
    span = 0
    for r in np.unique(first):
        rows = sorted_ords[first == r]
        def suf(row):
            v = 0
            for j in range(1, w):
                v = v * radix + int(row[j])
            return v
        span += suf(rows[-1]) - suf(rows[0]) + 1
    return span


def _rep(r):
    return (r.written, r.cells_traversed, (r.spec.radix, r.spec.total_digits, r.spec.integer_digits))


@pytest.mark.parametrize("alphabet,width,max_cells", [("ab", 16, 10**8), ("ab", 18, 10**9), ("xy", 14, 10**8),
                                                      (ALNUM, 4, 10**8), (BYTES255, 3, 10**8),
                                                      ("zyxwvutsrqponmlkjihgfedcba", 5, 10**8)])
def test_facade_wide_and_large_alphabets_vs_reference(rs, ref, alphabet, width, max_cells):
    """The grid path (no MSD) at widths above 12 and alphabets above 31 symbols."""
    recs = _records(width * 31 + len(alphabet), 50_000, width, alphabet)
    want, wrep = ref.sort_strings(recs, alphabet, max_cells)
    out, rep = rs.sort_fixed_str(_t(recs), alphabet=alphabet, max_cells=max_cells)
    assert np.array_equal(out.cpu().numpy(), want)
    assert _rep(rep) == wrep


def test_python_facade_long_strings(rs, ref):
    values = ["ab" * 8, "b", "a" * 15, "ba", "abba" * 4, ""]
    want = sorted(values, key=lambda s: [1 + "ab".index(c) for c in s] + [0] * (16 - len(s)))
    got, rep = rs.sort_strings(values, alphabet="ab", max_cells=10**8)
    assert got == want
    assert rep.spec.radix == 3 and rep.spec.total_digits == 16


@pytest.mark.parametrize("recs_list,alphabet,max_cells", [
    ([b"ab", b"a?", b"c"], "abc", 10**8),          # symbol error (first bad: '?')
    ([b"abcabcabcabcab", b"?"], "abc", 10**8),    # both: the key spec is checked first
    ([b"ab", b"x" + b"a" * 13], "abc", 10**4),     # budget before the symbol
    ([b"a" * 41], "ab", 2**64 - 1),                # 3^41 overflows 64 bits
])
def test_string_errors_in_reference_order(rs, ref, recs_list, alphabet, max_cells):
    from oracle import OracleError

    width = max(len(r) for r in recs_list)
    recs = np.zeros((len(recs_list), width), dtype=np.uint8)
    for i, r in enumerate(recs_list):
        recs[i, :len(r)] = np.frombuffer(r, dtype=np.uint8)
    with pytest.raises(OracleError) as want:
        ref.sort_strings(recs, alphabet, max_cells)
    with pytest.raises(rs.Error) as got:
        rs.sort_fixed_str(_t(recs), alphabet=alphabet, max_cells=max_cells)
    assert got.value.code == rs._lib.load().rs_status_name(want.value.status).decode()
    assert str(got.value) == want.value.message


@pytest.mark.parametrize("alphabet,width", [("ab", 32),              # 2 bits per ordinal
                                            ("abcdefghijklmno", 16),  # 4 bits (15 symbols)
                                            (ALNUM, 10),              # 6 bits
                                            (BYTES255, 8),            # 8 bits, 64-bit records
                                            (BYTES255, 7),
                                            ("fedcba", 21)])          # 3 bits, table ordinals
def test_msd_packed_widths(rs, alphabet, width):
    n = 120_000
    recs = _records(width + 7 * len(alphabet), n, width, alphabet, short_every=3)
    recs[:2000] = recs[2000:4000]  # duplicates
    order, o = _ordinal_order(recs, alphabet)
    out, rep = rs.sort_fixed_str(_t(recs), alphabet=alphabet, msd=True)
    assert np.array_equal(out.cpu().numpy(), recs[order])
    w = int((recs != 0).sum(axis=1).max())
    assert rep.spec.radix == len(alphabet) + 1 and rep.spec.total_digits == w
    assert rep.cells_traversed == _report(o[order][:, :w], len(alphabet) + 1, w)


def test_msd_too_wide_keeps_reference_error(rs, ref):
    """width * b > 64: no packed key, the reference's budget error."""
    from oracle import OracleError

    recs = _records(3, 1000, 13, "abcdefghijklmnopqrstuvwxyz", short_every=1)
    with pytest.raises(OracleError) as want:
        ref.sort_strings(recs, "abcdefghijklmnopqrstuvwxyz", 10**8)
    with pytest.raises(rs.Error) as got:
        rs.sort_fixed_str(_t(recs), msd=True)
    assert str(got.value) == want.value.message


@pytest.mark.parametrize("bad_byte", [ord("`"), ord("{"), ord("A"), 0xFF, 1])
def test_w8_contiguous_alphabet_symbol_check(rs, ref, bad_byte):
    """8-byte records over a-z take the SWAR scan: a byte just below or above
    the alphabet, anywhere before the first NUL, is reported like the
    reference (after the key spec); bytes after a NUL are ignored."""
    from oracle import OracleError

    recs = _records(11, 5000, 8, "abcdefghijklmnopqrstuvwxyz", short_every=2)
    ok = recs.copy()
    ok[7, 3] = 0
    ok[7, 4:] = 0
    order, _ = _ordinal_order(ok, "abcdefghijklmnopqrstuvwxyz")
    ok[7, 5] = bad_byte  # after the NUL: not part of the string (the output record is NUL-padded)
    got, _ = rs.sort_fixed_str(_t(ok), msd=True)
    want = ok[order].copy()
    want[want[:, 3] == 0, 4:] = 0
    assert np.array_equal(got.cpu().numpy(), want)
    recs[4000, 0] = ord("a")
    recs[4000, 1] = bad_byte
    recs[4000, 2:] = ord("b")
    with pytest.raises(OracleError) as w:  # fails at the symbol, before any count space exists
        ref.sort_strings(recs, "abcdefghijklmnopqrstuvwxyz", 10**12)
    with pytest.raises(rs.Error) as g:
        rs.sort_fixed_str(_t(recs), msd=True)
    assert str(g.value) == w.value.message
