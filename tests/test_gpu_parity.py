"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the
reference-generated golden vectors on the same seeded inputs.  Integer,
byte and index work must be bit-exact, reports included."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _t(a, dtype=None):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda") if dtype is None else \
        torch.from_numpy(np.ascontiguousarray(a)).to("cuda").view(dtype)


def _np_u32(t):
    return t.cpu().numpy().view(np.uint32)


def _rep(r):
    return (r.written, r.cells_traversed, (r.spec.radix, r.spec.total_digits, r.spec.integer_digits))


def gen_u32_device(rs, seed, n, bound):
    import torch

    out = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(rs._lib.load().rs_gen_u32(seed, 0, n, bound, rs._ptr(out), rs._stream()))
    return out


# ------------------------------------------------ reference Python API mirror
GOLDEN_INPUT = ["4.5", "0.3", "2.3", "8.8", "7", "9.2", "4.5", "4.3", "8", "3.2"]
GOLDEN_SORTED = ["0.3", "2.3", "3.2", "4.3", "4.5", "4.5", "7.0", "8.0", "8.8", "9.2"]


def test_python_smoke_mirror(rs):
    # proj/tests/python/test_smoke.py, through the GPU path
    values, report = rs.sort_decimals(GOLDEN_INPUT)
    assert values == GOLDEN_SORTED
    assert report.written == 10 and report.cells_traversed == 17
    values, report = rs.sort_integers([3, 1, 2, 2])
    assert values == [1, 2, 2, 3] and report.written == 4
    values, _ = rs.sort_strings(["ba", "ab", "aa", "b"])
    assert values == ["aa", "ab", "b", "ba"]
    with pytest.raises(rs.Error, match="negative"):
        rs.sort_decimals(["-3"])
    with pytest.raises(rs.Error, match="budget"):
        rs.sort_decimals(["123456789012"])
    with pytest.raises(ValueError):
        rs.sort_integers([-1])


def test_worked_example_integers(rs):
    values, rep = rs.sort_integers([45, 3, 23, 88, 70, 92, 45, 43, 80, 32])
    assert values == [3, 23, 32, 43, 45, 45, 70, 80, 88, 92]
    assert (rep.written, rep.cells_traversed) == (10, 17)
    assert (rep.spec.radix, rep.spec.total_digits, rep.spec.integer_digits) == (10, 2, 2)


def test_facade_matches_reference_on_small_cases(rs, oracle):
    # test_extraction.cpp:42-63 and differential multisets (81-90)
    cases = [[57], [66] * 23, [3, 23, 32, 43, 45, 45, 70, 80, 88, 92], [0], [0, 0, 9], list(range(100))[::-1]]
    for inst in range(50):
        cases.append(oracle.gen_u32(0x3317 + inst, 0, inst * 4, 10 ** (1 + inst % 3)).tolist())
    for c in cases:
        got, rep = rs.sort_integers(c)
        want, wrep = oracle.sort_integers_i64(np.array(c, dtype=np.int64))
        assert got == want.tolist()
        assert _rep(rep) == wrep, c


# ---------------------------------------------------------- golden vectors
def test_golden_cfg1_cfg2(rs, golden):
    for cfg in ("cfg1", "cfg2"):
        out, rep = rs.sort_u32(_t(golden[f"{cfg}_keys"].view(np.int32)))
        assert np.array_equal(_np_u32(out), golden[f"{cfg}_sorted"])
        assert [rep.written, rep.cells_traversed, *_rep(rep)[2]] == golden[f"{cfg}_report"].tolist()


def test_golden_kv(rs, golden):
    ko, vo, _ = rs.sort_u32_kv(_t(golden["kv_keys"].view(np.int32)), _t(golden["kv_vals"].view(np.int32)))
    assert np.array_equal(_np_u32(ko), golden["kv_sorted_keys"])
    assert np.array_equal(_np_u32(vo), golden["kv_sorted_vals"])


def test_golden_f64(rs, golden):
    out, rep = rs.sort_f64(_t(golden["cfg3_x"]), 3)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), golden["cfg3_sorted"])
    assert [rep.written, rep.cells_traversed, *_rep(rep)[2]] == golden["cfg3_report"].tolist()


def test_golden_strings(rs, golden):
    out, rep = rs.sort_fixed_str(_t(golden["str_recs"]), alphabet="abc")
    assert np.array_equal(out.cpu().numpy(), golden["str_sorted"])
    assert [rep.written, rep.cells_traversed, *_rep(rep)[2]] == golden["str_report"].tolist()


# ------------------------------------------------- oracle at test sizes
@pytest.mark.parametrize("cfg,n,bound", [(1, 1 << 20, 1000), (2, 1 << 22, 10**6), (2, 999_999, 10**6),
                                         (5, 1 << 20, 10**5), (6, 12345, 10**8), (7, 1 << 21, 10**7)])
def test_u32_vs_oracle(rs, oracle, cfg, n, bound):
    keys = oracle.gen_u32(oracle.config_seed(cfg), 0, n, bound)
    want, wrep = oracle.sort_integers_u32(keys, max_cells=10**9)
    out, rep = rs.sort_u32(_t(keys.view(np.int32)), max_cells=10**9)
    assert np.array_equal(_np_u32(out), want)
    assert _rep(rep) == wrep


@pytest.mark.parametrize("hint", [0, 3, 6, 7, 9])
def test_declared_width_never_changes_result(rs, oracle, hint):
    keys = oracle.gen_u32(77, 0, 300_000, 10**6)
    want, wrep = oracle.sort_integers_u32(keys)
    out, rep = rs.sort_u32(_t(keys.view(np.int32)), key_digits=hint, max_cells=10**9)
    assert np.array_equal(_np_u32(out), want) and _rep(rep) == wrep


def test_kv_vs_oracle(rs, oracle):
    n = 1 << 22
    keys = oracle.gen_u32(oracle.config_seed(2), 0, n, 10**6)
    vals = np.arange(n, dtype=np.uint32)
    wk, wv = oracle.radix_sort_lsd_kv(keys, vals)
    ko, vo, rep = rs.sort_u32_kv(_t(keys.view(np.int32)), _t(vals.view(np.int32)), key_digits=6)
    assert np.array_equal(_np_u32(ko), wk) and np.array_equal(_np_u32(vo), wv)
    _, wrep = oracle.sort_integers_u32(keys)
    assert _rep(rep) == wrep


@pytest.mark.parametrize("bound", [10, 1000, 10**7, 0])
def test_kv_widths(rs, oracle, bound):
    n = 50_001
    keys = oracle.gen_u32(31 + bound, 0, n, bound)
    vals = oracle.gen_u32(32, 0, n, 0)
    wk, wv = oracle.radix_sort_lsd_kv(keys, vals)
    ko, vo, _ = rs.sort_u32_kv(_t(keys.view(np.int32)), _t(vals.view(np.int32)), max_cells=10**10)
    assert np.array_equal(_np_u32(ko), wk) and np.array_equal(_np_u32(vo), wv)


def test_f64_vs_oracle(rs, oracle):
    n = 1 << 21
    cdf = oracle.zipf_cdf()
    x = oracle.gen_f64_cfg3(oracle.config_seed(3), 0, n, cdf)
    want, wrep = oracle.sort_f64(x, 3)
    out, rep = rs.sort_f64(_t(x), 3)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want)
    assert _rep(rep) == wrep


def test_f64_device_generator_matches_host(rs, oracle):
    import torch

    n = 1 << 18
    cdf = oracle.zipf_cdf()
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    d_cdf = _t(cdf)
    rs._check(rs._lib.load().rs_gen_f64_cfg3(oracle.config_seed(3), 5, n, rs._ptr(d_cdf), cdf.size,
                                             rs._ptr(x), rs._stream()))
    assert np.array_equal(x.cpu().numpy(), oracle.gen_f64_cfg3(oracle.config_seed(3), 5, n, cdf))
    keys = gen_u32_device(rs, 99, 1 << 18, 10**6)
    assert np.array_equal(_np_u32(keys), oracle.gen_u32(99, 0, 1 << 18, 10**6))


@pytest.mark.parametrize("scale", [0, 1, 2, 3, 4, 6])
def test_f64_golden_table(rs, golden, scale):
    # every reference float_to_decimal value of the golden table that lies in
    # the documented domain, one key per call so each is checked exactly
    xs = golden["f2d_x"]
    want = golden[f"f2d_scale{scale}"]
    lim = 9007199254740992.0 / 100.0
    keep = [(x, w) for x, w in zip(xs.tolist(), want.tolist())
            if x * 10.0 ** scale < min(lim, 1e8) and (x == 0.0 or x >= 1.0000001 * 10.0 ** -(scale + 3))]
    x = np.array([k for k, _ in keep])
    w = np.sort(np.array([v for _, v in keep], dtype=np.uint64))
    out, _ = rs.sort_f64(_t(x), scale, max_cells=10**12)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), w)


def test_strings_vs_oracle(rs, oracle):
    recs = oracle.gen_str_cfg4(oracle.config_seed(4), 0, 200_000)[:, :5].copy()
    recs[::7, 4] = 0
    recs[::11, 3:] = 0
    want, wrep = oracle.sort_fixed_strings(recs)
    out, rep = rs.sort_fixed_str(_t(recs))
    assert np.array_equal(out.cpu().numpy(), want)
    assert _rep(rep) == wrep


# ------------------------------------------------------------ edge cases
def test_empty_and_tiny(rs):
    import torch

    for n in (0, 1, 2, 3, 5, 17):
        keys = torch.arange(n, 0, -1, dtype=torch.int32, device="cuda")
        out, rep = rs.sort_u32(keys)
        assert out.cpu().tolist() == sorted(keys.cpu().tolist())
        assert rep.written == n
    out, rep = rs.sort_u32(torch.empty(0, dtype=torch.int32, device="cuda"))
    assert _rep(rep) == (0, 0, (10, 1, 1))


def test_unaligned_pointers(rs, oracle):
    import torch

    keys = oracle.gen_u32(5, 0, 100_003, 10**6)
    big = _t(np.concatenate([[7], keys]).astype(np.uint32).view(np.int32))
    dst = torch.empty(100_005, dtype=torch.int32, device="cuda")
    out, rep = rs.sort_u32(big[1:], out=dst[1:100_004])
    want, wrep = oracle.sort_integers_u32(keys)
    assert np.array_equal(_np_u32(out), want) and _rep(rep) == wrep


def test_hot_cell_and_skew(rs, oracle):
    keys = np.concatenate([np.full(3_000_000, 424242, dtype=np.uint32), oracle.gen_u32(1, 0, 100_000, 10**6)])
    want, wrep = oracle.sort_integers_u32(keys)
    out, rep = rs.sort_u32(_t(keys.view(np.int32)), key_digits=6)
    assert np.array_equal(_np_u32(out), want) and _rep(rep) == wrep


def test_full_range_u32_budget(rs, oracle):
    keys = oracle.gen_u32(3, 0, 1000, 0)
    with pytest.raises(rs.Error) as e:
        rs.sort_u32(_t(keys.view(np.int32)))
    assert e.value.code == "cell_budget_exceeded"


def test_errors_match_reference_codes(rs):
    import torch

    with pytest.raises(rs.Error) as e:
        rs.sort_i64(torch.tensor([5, -2, 7], device="cuda"))
    assert e.value.code == "negative_value"
    with pytest.raises(rs.Error) as e:
        rs.sort_f64(torch.tensor([1.0, float("nan")], dtype=torch.float64, device="cuda"), 2)
    assert e.value.code == "non_finite"
    with pytest.raises(rs.Error) as e:
        rs.sort_f64(torch.tensor([1.0, -3.0], dtype=torch.float64, device="cuda"), 2)
    assert e.value.code == "negative_value"
    with pytest.raises(rs.Error) as e:
        rs.sort_u32(torch.arange(10, dtype=torch.int32, device="cuda"),
                    out=torch.empty(5, dtype=torch.int32, device="cuda"))
    assert e.value.code == "buffer_too_small"
    with pytest.raises(rs.Error) as e:
        rs.sort_keys(torch.tensor([5, 100], device="cuda"), rs.KeySpec(10, 2, 1))
    assert e.value.code == "spec_mismatch"
    with pytest.raises(rs.Error) as e:
        rs.sort_strings(["aZ"])
    assert e.value.code == "symbol_out_of_alphabet"
    with pytest.raises(rs.Error) as e:
        rs.sort_strings(["zzzzzz"])
    assert e.value.code == "cell_budget_exceeded"


# ----------------------------------- full BASELINE sizes: size-free properties
def _sorted_and_same_multiset(inp, out, bins):
    import torch

    assert bool((out[1:] >= out[:-1]).all())
    assert torch.equal(torch.bincount(inp, minlength=bins), torch.bincount(out, minlength=bins))


def test_cfg2_full_size_properties(rs):
    import torch

    n = 1 << 28
    keys = gen_u32_device(rs, rs_seed(2), n, 10**6)
    out, rep = rs.sort_u32(keys, key_digits=6)
    assert rep.written == n and rep.spec.total_digits == 6
    _sorted_and_same_multiset(keys.long(), out.long(), 10**6)
    # all 10^6 cells occupied -> each of the 10 rows spans 10^5 cells
    assert rep.cells_traversed == 10**6
    del out
    torch.cuda.empty_cache()


def test_cfg2_kv_full_size_stability(rs):
    import torch

    n = 1 << 28
    keys = gen_u32_device(rs, rs_seed(2), n, 10**6)
    vals = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(rs._lib.load().rs_gen_iota_u32(0, n, rs._ptr(vals), rs._stream()))
    ko, vo, rep = rs.sort_u32_kv(keys, vals, key_digits=6)
    assert bool((ko[1:] >= ko[:-1]).all())
    same = ko[1:] == ko[:-1]
    assert bool((vo[1:][same] > vo[:-1][same]).all())  # payload = index: stable
    assert torch.equal(keys[vo.long()], ko)              # payload points at its key
    del ko, vo
    torch.cuda.empty_cache()


def test_cfg3_full_size_properties(rs, oracle):
    """2^28 float64 k/1000 (half Zipf) at BASELINE size: sorted, and the same
    multiset of mantissas as round(x * 1000) (exact for these decimals)."""
    import torch

    n = 1 << 28
    cdf = torch.from_numpy(oracle.zipf_cdf()).cuda()
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    rs._check(rs._lib.load().rs_gen_f64_cfg3(rs_seed(3), 0, n, rs._ptr(cdf), cdf.numel(), rs._ptr(x), rs._stream()))
    out, rep = rs.sort_f64(x, 3, key_digits=6)
    assert rep.written == n and (rep.spec.total_digits, rep.spec.integer_digits) == (6, 3)
    want = torch.round(x * 1000.0).long()
    del x
    _sorted_and_same_multiset(want, out.view(torch.int64), 10**6)
    del out, want
    torch.cuda.empty_cache()


def test_cfg4_full_size_exact(rs):
    """2^26 eight-letter strings at BASELINE size through the MSD path,
    element for element against an independent checker (torch.sort of the
    records as big-endian integers: for a contiguous alphabet and NUL pad the
    reference's ordinal order is byte order; equal strings are equal rows, so
    the sorted output is unique)."""
    import torch

    n = 1 << 26
    recs = torch.empty((n, 8), dtype=torch.uint8, device="cuda")
    rs._check(rs._lib.load().rs_gen_str_cfg4(rs_seed(4), 0, n, rs._ptr(recs), rs._stream()))
    out, rep = rs.sort_fixed_str(recs, msd=True)
    assert rep.written == n and rep.spec.radix == 27 and rep.spec.total_digits == 8

    def as_key(r):  # big-endian: lexicographic byte order == integer order (ASCII < 128)
        k = torch.zeros(r.shape[0], dtype=torch.int64, device=r.device)
        for i in range(8):
            k = (k << 8) | r[:, i].long()
        return k

    want = torch.sort(as_key(recs)).values
    got = as_key(out)
    assert torch.equal(got, want)
    # the report: per leading-symbol row, the span of its base-27 suffixes (F4)
    ords = (out.long() - ord("a") + 1).clamp(min=0)
    k27 = torch.zeros(n, dtype=torch.int64, device="cuda")
    for i in range(8):
        k27 = k27 * 27 + ords[:, i]
    assert _cells_traversed(k27, 27 ** 7) == rep.cells_traversed
    del recs, out, want, got, ords, k27
    torch.cuda.empty_cache()


def _cells_traversed(sorted_keys, mod):
    """cells_traversed of a sorted int64 key tensor (extraction.cpp:16-30):
    sum over occupied rows (key // mod) of max - min + 1."""
    import torch

    rows = int(sorted_keys[-1]) // mod + 1
    lo = torch.arange(rows, device=sorted_keys.device, dtype=torch.int64) * mod
    a = torch.searchsorted(sorted_keys, lo)
    b = torch.searchsorted(sorted_keys, lo + mod)
    occ = b > a
    first = sorted_keys[a[occ]]
    last = sorted_keys[b[occ] - 1]
    return int((last - first + 1).sum())


def rs_seed(cfg):
    from oracle import Oracle

    return Oracle().config_seed(cfg)


# ------------------------------------------------- MSD (wide keys, A17)
@pytest.mark.parametrize("n,bound", [(1 << 22, 0), (300_001, 0), (1 << 20, 10**9), (5000, 0)])
def test_msd_u32_vs_oracle(rs, oracle, n, bound):
    keys = oracle.gen_u32(oracle.config_seed(5), 0, n, bound)
    want = np.sort(keys)
    out, rep = rs.sort_u32(_t(keys.view(np.int32)), msd=True)
    assert np.array_equal(_np_u32(out), want)
    d = len(str(int(want[-1])))
    assert _rep(rep) == oracle.report_from_sorted(want.astype(np.uint64), 10, d)


def test_msd_u32_skew_and_duplicates(rs, oracle):
    keys = np.concatenate([np.full(200_000, 4_000_000_000, dtype=np.uint32),
                           oracle.gen_u32(8, 0, 100_000, 0), np.arange(70_000, dtype=np.uint32) * 7,
                           np.full(70_000, 123, dtype=np.uint32)])
    out, _ = rs.sort_u32(_t(keys.view(np.int32)), msd=True)
    assert np.array_equal(_np_u32(out), np.sort(keys))


@pytest.mark.parametrize("n,bits", [(1 << 22, 63), (300_001, 40), (1 << 20, 33), (4097, 63), (1, 63)])
def test_msd_i64_vs_oracle(rs, oracle, n, bits):
    """int64 values past any grid budget: MSD digits over the max's bit width
    (A17 for the integer facade); report as the reference would compute it
    with an unlimited budget."""
    import torch

    rng = np.random.default_rng(bits * 7 + n)
    vals = rng.integers(0, 1 << bits, n, dtype=np.int64)
    if n > 100:
        vals[rng.random(n) < 0.3] = vals[0]  # one heavy value
    want = np.sort(vals)
    out, rep = rs.sort_i64(torch.from_numpy(vals).cuda(), msd=True)
    assert np.array_equal(out.cpu().numpy(), want)
    d = len(str(int(want[-1])))
    assert _rep(rep) == oracle.report_from_sorted(want.astype(np.uint64), 10, d)


def test_msd_i64_rejects_negative(rs):
    import torch

    vals = torch.tensor([5, 10**15, -1, 3], dtype=torch.int64, device="cuda")
    with pytest.raises(rs.Error) as e:
        rs.sort_i64(vals, msd=True)
    assert e.value.code == "negative_value"


@pytest.mark.parametrize("bound", [1 << 21, 12_000_000, (1 << 27) + 5])
def test_msd_u32_narrow_keys(rs, oracle, bound):
    """Keys above the budget but well below 2^32: the MSD levels start at the
    max's bit width (21, 24 and 28 bits here)."""
    keys = oracle.gen_u32(oracle.config_seed(5), 1, 1 << 21, bound)
    out, rep = rs.sort_u32(_t(keys.view(np.int32)), msd=True)
    want = np.sort(keys)
    assert np.array_equal(_np_u32(out), want)
    assert _rep(rep) == oracle.report_from_sorted(want.astype(np.uint64), 10, len(str(int(want[-1]))))


def test_msd_radix_leaf_fast_and_skewed(rs, oracle):
    """Leaves of ~3000 keys with 24 remaining bits: uniform ones take the
    split + insertion fast path, skewed ones (a handful of low values, so a
    sub-bucket holds hundreds of keys) the LSD passes; both with duplicates."""
    rng = np.random.default_rng(77)
    n = 256 * 3000
    hi = rng.integers(0, 256, n, dtype=np.uint64)
    low = rng.integers(0, 1 << 24, n, dtype=np.uint64)
    skew = (hi % 3) == 0
    low[skew] = rng.choice(np.array([5, 6, 1 << 20, (1 << 24) - 1], dtype=np.uint64), int(skew.sum()))
    low[::97] = low[::89][: low[::97].size]  # duplicates inside uniform leaves
    keys = ((hi << np.uint64(24)) | low).astype(np.uint32)
    out, _ = rs.sort_u32(_t(keys.view(np.int32)), msd=True)
    assert np.array_equal(_np_u32(out), np.sort(keys))
    wide = (keys.astype(np.uint64) << np.uint64(16)) | np.uint64(3)  # the same leaves as 64-bit keys
    import torch

    got, _ = rs.sort_i64(torch.from_numpy(wide.view(np.int64)).cuda(), msd=True)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), np.sort(wide))


def test_msd_count_grid_leaf_modes(rs, oracle):
    """16-bit count-grid leaves on both sides of the shared-memory staging
    capacity (~50K keys: scatter below, run-length emit above), a segment at
    the 65535-key limit, and one cell holding a whole segment."""
    parts = []
    for hi, size in [(3, 30_000), (9, 49_000), (11, 52_000), (12, 60_000), (200, 65_535), (201, 40_000)]:
        low = oracle.gen_u32(1000 + hi, 0, size, 1 << 16)
        parts.append((np.uint32(hi) << np.uint32(16)) | low)
    parts.append(np.full(45_000, (77 << 16) | 5, dtype=np.uint32))   # one cell, scatter mode
    parts.append(np.full(61_000, (78 << 16) | 65535, dtype=np.uint32))  # one cell, emit mode
    keys = np.concatenate(parts)
    keys = keys[np.argsort(oracle.gen_u32(99, 0, keys.size, 0), kind="stable")]
    out, _ = rs.sort_u32(_t(keys.view(np.int32)), msd=True)
    assert np.array_equal(_np_u32(out), np.sort(keys))


def test_msd_strings_vs_oracle(rs, oracle, golden):
    recs = oracle.gen_str_cfg4(oracle.config_seed(4), 0, 1 << 20)
    want, wrep = oracle.sort_fixed_strings(recs)
    out, rep = rs.sort_fixed_str(_t(recs), msd=True)
    assert np.array_equal(out.cpu().numpy(), want)
    assert _rep(rep) == wrep
    out, _ = rs.sort_fixed_str(_t(golden["cfg4_recs"]), msd=True)
    assert np.array_equal(out.cpu().numpy(), golden["cfg4_sorted"])


@pytest.mark.parametrize("alphabet,width", [("zyxwvutsrqponmlkjihgfedcba", 8),   # table path (not contiguous)
                                            ("abcdefghijklmnopqrstuvwxyz", 7),   # contiguous, unpacked stores
                                            ("0123456789", 8)])                  # contiguous, other base
def test_msd_strings_alphabets(rs, oracle, alphabet, width):
    n = 150_000
    pick = oracle.gen_u32(31 + width, 0, n * width, len(alphabet)).reshape(n, width)
    recs = np.frombuffer(alphabet.encode(), dtype=np.uint8)[pick]
    recs[::7, width - 2:] = 0  # some shorter strings
    # reference order = alphabet ordinals (strings_to_keys, key_model.cpp:190-247),
    # not byte order: key = sum ord_i * radix^(w-1-i), pad ordinal 0
    ords = np.zeros(256, dtype=np.uint64)
    ords[np.frombuffer(alphabet.encode(), dtype=np.uint8)] = np.arange(1, len(alphabet) + 1, dtype=np.uint64)
    radix = len(alphabet) + 1
    keys = np.zeros(n, dtype=np.uint64)
    for i in range(width):
        keys = keys * np.uint64(radix) + ords[recs[:, i]]
    order = np.argsort(keys, kind="stable")
    out, rep = rs.sort_fixed_str(_t(np.ascontiguousarray(recs)), alphabet=alphabet, msd=True)
    assert np.array_equal(out.cpu().numpy(), recs[order])
    assert _rep(rep) == oracle.report_from_sorted(keys[order], radix, width)


def test_msd_strings_variable_length(rs, oracle):
    recs = oracle.gen_str_cfg4(17, 0, 200_000)
    lens = oracle.gen_u32(18, 0, 200_000, 9)
    for i, l in enumerate(lens):
        recs[i, l:] = 0
    want, wrep = oracle.sort_fixed_strings(recs)
    out, rep = rs.sort_fixed_str(_t(recs), msd=True)
    assert np.array_equal(out.cpu().numpy(), want)
    assert _rep(rep) == wrep


def test_cfg5_full_size_exact(rs):
    """2^31 full-range uint32 keys (BASELINE cfg5 on one GPU), element for
    element: the input split by its top three bits (within one split int32
    order is uint32 order) and each split sorted by torch.sort, compared with
    the matching slice of the output; the report against the spans of the
    sorted keys (KeySpec{10,10,10}, rows = key / 10^9)."""
    import torch

    n = 1 << 31
    keys = gen_u32_device(rs, rs_seed(5), n, 0)
    out, rep = rs.sort_u32(keys, msd=True)
    assert rep.written == n and rep.spec.total_digits == 10
    pos = 0
    for j in range(8):
        sel = keys[((keys >> 29) & 7) == j]
        want = torch.sort(sel).values
        assert torch.equal(out[pos:pos + sel.numel()], want), j
        pos += sel.numel()
        del sel, want
    assert pos == n
    del keys
    wide = out.to(torch.int64) & 0xFFFFFFFF
    del out
    assert _cells_traversed(wide, 10**9) == rep.cells_traversed
    del wide
    torch.cuda.empty_cache()


def test_hot_cell_beyond_2_pow_32(rs):
    """One cell receiving 2^32 + 5 keys (the reference counts in uint64,
    hashing.hpp:86): nothing wraps, every key is written."""
    import torch

    n = (1 << 32) + 8
    k = torch.full((n,), 777, dtype=torch.int32, device="cuda")
    k[100], k[200], k[n - 1] = 3, 999_999, 5
    out, rep = rs.sort_u32(k)
    del k
    assert rep.written == n
    assert (rep.spec.total_digits, rep.cells_traversed) == (6, (777 - 3 + 1) + 1)
    assert int(out[0]) == 3 and int(out[1]) == 5 and int(out[n - 1]) == 999_999
    assert bool((out[2:n - 1] == 777).all())
    del out
    torch.cuda.empty_cache()


# ------------------------------------- multi-GPU device phases (1-rank NCCL)
def test_dist_paths_on_device_nccl(rs, oracle):
    """The sharded-grid, stable key/value and range-partition orchestration of
    dist.py with the real device phases (rs_count_u32 / rs_emit_u32 /
    rs_sort_u32_kv / rs_bucket_hist_u32 / rs_partition_u32) over a one-rank
    NCCL group."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_2107_01391_b200.dist import range_partition_sort, sharded_grid_sort, sharded_kv_sort

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        keys = oracle.gen_u32(21, 0, 1 << 22, 10**6)
        out = sharded_grid_sort(_t(keys.view(np.int32)), 10**6)
        assert np.array_equal(_np_u32(out), np.sort(keys))
        wide = oracle.gen_u32(22, 0, 1 << 21, 0)
        for exchange in ("p2p", "p2p", "nccl"):  # the fused peer-store exchange (twice: buffer reuse), then NCCL
            out = range_partition_sort(_t(wide.view(np.int32)), 10**7, 430, exchange=exchange)
            assert np.array_equal(_np_u32(out), np.sort(wide)), exchange
        vals = np.arange(keys.size, dtype=np.uint32)
        wk, wv = oracle.radix_sort_lsd_kv(keys, vals)
        for exchange in ("p2p", "p2p", "nccl"):  # fused placement over peer memory (twice), then NCCL
            ko, vo = sharded_kv_sort(_t(keys.view(np.int32)), _t(vals.view(np.int32)), 10**6, exchange=exchange)
            assert np.array_equal(_np_u32(ko), wk) and np.array_equal(_np_u32(vo), wv), exchange
    finally:
        dist.destroy_process_group()


def test_emit_phase_any_cell_range(rs, oracle):
    """rs_emit_u32 over cell ranges starting anywhere (the per-rank ranges of
    the multi-GPU paths): unaligned sub-grids take the scalar scan."""
    import torch

    lib = rs._lib.load()
    keys = oracle.gen_u32(31, 0, 1 << 20, 10**5)
    d = _t(keys.view(np.int32))
    counts = torch.empty(10**5, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_count_u32(rs._ptr(d), d.numel(), rs._ptr(counts), 10**5, None, rs._stream()))
    for lo, hi in [(0, 10**5), (1, 77_777), (3, 5), (12_345, 10**5), (99_999, 10**5), (50_001, 50_001)]:
        out = torch.empty(keys.size, dtype=torch.int32, device="cuda")
        w = ctypes.c_uint64()
        rs._check(lib.rs_emit_u32(rs._ptr(counts), 10**5, lo, hi, 0, rs._ptr(out), out.numel(), ctypes.byref(w),
                                  rs._stream()))
        want = np.sort(keys[(keys >= lo) & (keys < hi)])
        assert np.array_equal(_np_u32(out[: w.value]), want), (lo, hi)


def test_partition_phase_api(rs, oracle):
    import torch

    lib = rs._lib.load()
    keys = oracle.gen_u32(23, 0, 300_001, 0)
    d = _t(keys.view(np.int32))
    hist = torch.zeros(430, dtype=torch.int64, device="cuda")
    rs._check(lib.rs_bucket_hist_u32(rs._ptr(d), d.numel(), 10**7, rs._ptr(hist), 430, rs._stream()))
    assert np.array_equal(hist.cpu().numpy(), np.bincount(keys.astype(np.int64) // 10**7, minlength=430))
    bounds = [0, 100, 250, 430]
    out = torch.empty_like(d)
    hb = (ctypes.c_uint32 * 4)(*bounds)
    hc = (ctypes.c_uint64 * 3)()
    rs._check(lib.rs_partition_u32(rs._ptr(d), d.numel(), 10**7, hb, 3, rs._ptr(out), hc, rs._stream()))
    got = _np_u32(out)
    part = np.searchsorted(np.array(bounds[1:-1]), keys.astype(np.int64) // 10**7, side="right")
    assert list(hc) == np.bincount(part, minlength=3).tolist()
    start = 0
    for p in range(3):
        seg = got[start:start + hc[p]]
        assert np.array_equal(np.sort(seg), np.sort(keys[part == p]))
        start += hc[p]


@pytest.mark.parametrize("parts", [1, 3])
def test_sort_u32_multi_shards(rs, oracle, parts):
    """rs_sort_u32_multi with `parts` shards (on the one device here): the
    outputs concatenate to the sorted whole, the report is the single-grid
    one, and the slices are balanced cell ranges."""
    keys = oracle.gen_u32(77, 0, 3_000_001, 10**6)
    keys[:200_000] = 123_456  # a hot cell
    cuts = np.linspace(0, keys.size, parts + 1).astype(np.int64)
    shards = [_t(keys[a:b].view(np.int32)) for a, b in zip(cuts[:-1], cuts[1:])]
    outs, rep = rs.sort_u32_multi(shards)
    got = np.concatenate([_np_u32(o) for o in outs])
    want, wrep = oracle.sort_integers_u32(keys)
    assert np.array_equal(got, want)
    assert (rep.written, rep.cells_traversed) == wrep[:2]
    if parts > 1:
        assert all(_np_u32(a)[-1] < _np_u32(b)[0] for a, b in zip(outs, outs[1:]) if a.numel() and b.numel())


def test_two_rank_exchanges_emulated_on_one_gpu(rs, oracle):
    """The multi-GPU device phases with two "ranks" whose shards and receive
    buffers all live on this GPU (no collective needed): kv_placement tables
    + rs_kv_place_u32 into two buffers, and rs_part_counts_u32 +
    rs_partition_u32_to into two buffers — the exact writes two GPUs would
    make over NVLink; the rank slices must concatenate to the reference's
    stable order / the sorted keys."""
    import torch

    from paper_2107_01391_b200.dist import GpuOps, bucket_splitters, kv_placement

    ops = GpuOps()
    keys = oracle.gen_u32(41, 0, 2_000_003, 10**6)
    keys[::7] = 424_242  # a hot cell straddling both shards
    vals = np.arange(keys.size, dtype=np.uint32)
    half = keys.size // 2 + 5
    sk = [_t(keys[:half].view(np.int32)), _t(keys[half:].view(np.int32))]
    sv = [_t(vals[:half].view(np.int32)), _t(vals[half:].view(np.int32))]
    grids = torch.cat([ops.count(k, 10**6) for k in sk])
    bufk = [torch.zeros(keys.size, dtype=torch.int32, device="cuda") for _ in range(2)]
    bufv = [torch.zeros(keys.size, dtype=torch.int32, device="cuda") for _ in range(2)]
    sizes = None
    for r in range(2):
        off, owner, sizes = kv_placement(grids, r, 2)
        ks, vs = ops.sort_kv(sk[r], sv[r], 10**6)
        ops.kv_place(ks, vs, off, owner, [b.data_ptr() for b in bufk], [b.data_ptr() for b in bufv])
    torch.cuda.synchronize()
    n0, n1 = (int(s) for s in sizes.tolist())
    got_k = np.concatenate([_np_u32(bufk[0][:n0]), _np_u32(bufk[1][:n1])])
    got_v = np.concatenate([_np_u32(bufv[0][:n0]), _np_u32(bufv[1][:n1])])
    wk, wv = oracle.radix_sort_lsd_kv(keys, vals)
    assert n0 > 0 and n1 > 0
    assert np.array_equal(got_k, wk) and np.array_equal(got_v, wv)
    # wide keys: counts -> the 2 x 2 table -> offsets -> parts stored into both buffers
    wide = oracle.gen_u32(43, 0, 1_000_001, 0)
    sw = [_t(wide[:400_000].view(np.int32)), _t(wide[400_000:].view(np.int32))]
    hist = sum(ops.bucket_hist(k, 10**7, 430) for k in sw)
    bounds = bucket_splitters(hist.cpu(), 2)
    table = np.array([ops.part_counts(k, 10**7, bounds) for k in sw])  # [src][dst]
    recv = [torch.zeros(wide.size, dtype=torch.int32, device="cuda") for _ in range(2)]
    for g in range(2):
        ops.partition_to(sw[g], 10**7, bounds, [b.data_ptr() for b in recv], table[:g].sum(0).tolist())
    torch.cuda.synchronize()
    parts = [np.sort(_np_u32(recv[r][: int(table[:, r].sum())])) for r in range(2)]
    assert np.array_equal(np.concatenate(parts), np.sort(wide))


def test_more_than_2_pow_32_keys(rs, oracle):
    """2^32 + 4096 keys in one call (64-bit positions throughout): sorted,
    every key written, the report of a fully occupied 10^6-cell grid."""
    import torch

    lib = rs._lib.load()
    n = (1 << 32) + 4096
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_gen_u32(oracle.config_seed(2), 0, n, 10**6, rs._ptr(k), rs._stream()))
    out, rep = rs.sort_u32(k, key_digits=6)
    assert rep.written == n and rep.cells_traversed == 10**6
    assert bool((out[1:] >= out[:-1]).all())
    assert int(out[0]) == 0 and int(out[-1]) == 10**6 - 1
    del k, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("seed", range(10))
def test_sort_keys_any_radix_vs_reference(rs, ref, seed):
    """sort_keys (extraction.cpp:34-45) for radices 2..36 and widths whose
    grids span the shared, two-level and global count paths: keys and the
    report against the reference library's build_count_space + extract."""
    import torch

    rng = np.random.default_rng(700 + seed)
    radix = int(rng.integers(2, 37))
    d = 1
    while radix ** (d + 1) <= 3 * 10**6 and rng.random() < 0.85:
        d += 1
    ip = int(rng.integers(0, d + 1))
    cells = radix ** d
    n = int(rng.choice([1, 999, 100_000, 1_000_003]))
    keys = rng.integers(0, cells, n, dtype=np.uint64)
    if seed % 3 == 0:
        keys[: n // 2] = keys[0]  # a hot cell
    want, wrep = ref.sort_keys_core(keys, (radix, d, ip), max_cells=10**8)
    out, rep = rs.sort_keys(torch.from_numpy(keys.view(np.int64)).cuda(), rs.KeySpec(radix, d, ip), max_cells=10**8)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (radix, d)
    assert _rep(rep) == wrep, (radix, d)
