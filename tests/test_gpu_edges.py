"""GPU edge cases of the C-ABI beyond the sort kernels themselves: the
host-buffer entry points (their device staging must not alias any buffer a
sort pass uses), decoding of wide string keys, and the multi-GPU phase API's
checks on keys outside the grid."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _host_sort(rs, keys: np.ndarray, stream=None, **opt):
    lib = rs._lib.load()
    out = np.zeros_like(keys)
    rep = rs.RsReport()
    st = lib.rs_sort_u32_host(keys.ctypes.data_as(ctypes.c_void_p), keys.size, out.ctypes.data_as(ctypes.c_void_p),
                              ctypes.byref(rs._opts(opt.get("max_cells", rs.DEFAULT_CELL_BUDGET),
                                                    opt.get("key_digits", 0), opt.get("msd", False))),
                              ctypes.byref(rep), stream if stream is not None else rs._stream())
    rs._check(st)
    return out, rep


@pytest.mark.parametrize("n", [1, 7, 5000, 300_000, 3_000_001])
def test_host_entry_fresh_stream(rs, oracle, n):
    """rs_sort_u32_host on a stream that has never run a sort (a fresh
    workspace: every internal slot is allocated inside the call)."""
    import torch

    keys = oracle.gen_u32(900 + n, 0, n, 10**6)
    s = torch.cuda.Stream()
    out, rep = _host_sort(rs, keys, ctypes.c_void_p(s.cuda_stream))
    want, wrep = oracle.sort_integers_u32(keys)
    assert np.array_equal(out, want)
    assert (rep.written, rep.cells_traversed) == wrep[:2]


def test_host_entry_msd(rs, oracle):
    """msd=1 on host buffers: the MSD levels' segment lists are larger than
    the keys and must not land in the staging buffers."""
    import torch

    n = 2_000_003
    keys = oracle.gen_u32(77, 0, n, 0)
    s = torch.cuda.Stream()
    out, rep = _host_sort(rs, keys, ctypes.c_void_p(s.cuda_stream), msd=True)
    assert np.array_equal(out, np.sort(keys))
    assert rep.written == n and rep.spec.total_digits == 10
    out2, _ = _host_sort(rs, keys, ctypes.c_void_p(s.cuda_stream), msd=True)  # reused workspace
    assert np.array_equal(out2, out)


def test_host_entry_too_small_hint(rs, oracle):
    """A declared width below the data's redoes the sort with the derived
    width, reading the input a second time: the input must be intact."""
    n = 1_500_000
    keys = oracle.gen_u32(78, 0, n, 10**7)
    out, rep = _host_sort(rs, keys, key_digits=5)
    want, wrep = oracle.sort_integers_u32(keys)
    assert np.array_equal(out, want)
    assert (rep.written, rep.cells_traversed) == wrep[:2]
    assert rep.spec.total_digits == 7


def test_host_kv_entry(rs, oracle):
    lib = rs._lib.load()
    n = 1_000_003
    keys = oracle.gen_u32(79, 0, n, 10**6)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo = np.zeros_like(keys), np.zeros_like(vals)
    rep = rs.RsReport()
    rs._check(lib.rs_sort_u32_kv_host(keys.ctypes.data_as(ctypes.c_void_p), vals.ctypes.data_as(ctypes.c_void_p), n,
                                      ko.ctypes.data_as(ctypes.c_void_p), vo.ctypes.data_as(ctypes.c_void_p),
                                      ctypes.byref(rs._opts(rs.DEFAULT_CELL_BUDGET)), ctypes.byref(rep), rs._stream()))
    wk, wv = oracle.radix_sort_lsd_kv(keys, vals)
    assert np.array_equal(ko, wk) and np.array_equal(vo, wv)


@pytest.mark.parametrize("alphabet,width,budget", [("a", 20, 10**8), ("ab", 18, 10**9), ("z", 26, 10**8)])
def test_wide_string_keys_decode(rs, oracle, alphabet, width, budget):
    """Keys of more than 16 symbols (a 1- or 2-symbol alphabet: radix 2 or 3
    admits widths up to 26 / 18 within the budget) decoded back to records."""
    import torch

    n = 20_000
    rng = np.random.default_rng(width)
    sym = np.frombuffer(alphabet.encode(), dtype=np.uint8)
    recs = sym[rng.integers(0, len(sym), (n, width))]
    lens = rng.integers(0, width + 1, n)
    for i, l in enumerate(lens):
        recs[i, l:] = 0
    want, wrep = oracle.sort_fixed_strings(np.ascontiguousarray(recs), alphabet)
    out, rep = rs.sort_fixed_str(torch.from_numpy(np.ascontiguousarray(recs)).cuda(), alphabet=alphabet,
                                 max_cells=budget)
    assert np.array_equal(out.cpu().numpy(), want)
    assert (rep.written, rep.cells_traversed) == wrep[:2]


def test_count_phase_rejects_keys_outside_the_grid(rs):
    """rs_count_u32 (the multi-GPU count phase) fails on a key >= cells
    instead of silently dropping it from the grid."""
    import torch

    lib = rs._lib.load()
    k = torch.arange(1000, dtype=torch.int32, device="cuda")
    counts = torch.empty(1000, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_count_u32(rs._ptr(k), 1000, rs._ptr(counts), 1000, None, rs._stream()))
    assert bool((counts == 1).all())
    k[500] = 1000
    st = lib.rs_count_u32(rs._ptr(k), 1000, rs._ptr(counts), 1000, None, rs._stream())
    assert lib.rs_status_name(st).decode() == "out_of_range"


@pytest.mark.parametrize("cells", [823543, 123457, 1000000])
def test_direct_partition_cells_past_a_partial_last_bucket(rs, cells):
    """A grid whose last outer bucket is partial (cells not a multiple of the
    inner size): cells between the grid's end and that bucket's end share its
    bucket index in the direct partition.  In-grid keys count exactly; a key
    in that gap, or far outside, fails with out_of_range and nothing is
    written past the grid."""
    import torch

    lib = rs._lib.load()
    n = 1 << 22
    g = torch.Generator(device="cuda").manual_seed(cells)
    k = torch.randint(0, cells, (n,), dtype=torch.int32, device="cuda", generator=g)
    k[:64] = cells - 1  # the last cell is occupied
    guard = 4096
    buf = torch.full((cells + guard,), -7, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_count_u32(rs._ptr(k), n, rs._ptr(buf), cells, None, rs._stream()))
    assert torch.equal(buf[:cells].long(), torch.bincount(k.long(), minlength=cells))
    assert bool((buf[cells:] == -7).all())
    for bad in (cells, cells + 3, cells + 60000, 0x7fffffff):
        kb = k.clone()
        kb[12345] = bad
        kb[n - 1] = bad
        buf.fill_(-7)
        st = lib.rs_count_u32(rs._ptr(kb), n, rs._ptr(buf), cells, None, rs._stream())
        assert lib.rs_status_name(st).decode() == "out_of_range"
        assert bool((buf[cells:] == -7).all())


def test_kv_place_rejects_keys_outside_the_grid(rs):
    """rs_kv_place_u32 never stores a record whose key lies outside the
    placement tables (it would index past them and write into a peer's
    memory); the call fails instead."""
    import torch

    lib = rs._lib.load()
    n, cells = 1000, 100
    k = torch.arange(n, dtype=torch.int32, device="cuda") % cells
    v = torch.arange(n, dtype=torch.int32, device="cuda")
    off = torch.zeros(cells, dtype=torch.int64, device="cuda")
    owner = torch.zeros(cells, dtype=torch.uint8, device="cuda")
    dk = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    dv = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    hk = (ctypes.c_uint64 * 1)(dk.data_ptr())
    hv = (ctypes.c_uint64 * 1)(dv.data_ptr())
    k[7] = cells + 5
    st = lib.rs_kv_place_u32(rs._ptr(k), rs._ptr(v), n, rs._ptr(off), rs._ptr(owner), cells, hk, hv, 1, rs._stream())
    assert lib.rs_status_name(st).decode() == "out_of_range"
    owner[3] = 9  # an owner that is not a rank
    k[7] = 3
    st = lib.rs_kv_place_u32(rs._ptr(k), rs._ptr(v), n, rs._ptr(off), rs._ptr(owner), cells, hk, hv, 1, rs._stream())
    assert lib.rs_status_name(st).decode() == "out_of_range"


def test_sampled_width_too_small_redoes(rs, oracle):
    """Without a declared width, large inputs plan the grid from a strided
    sample's max; a larger key the sample missed makes the counting pass
    redo the sort at the data's true width (same keys, same report as the
    reference)."""
    import torch

    n = (1 << 22) + 5
    keys = oracle.gen_u32(80, 0, n, 1000)
    keys[1] = 9_999_999  # between sample points (every ~64th element)
    out, rep = rs.sort_u32(torch.from_numpy(keys.view(np.int32)).cuda())
    want, wrep = oracle.sort_integers_u32(keys)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)
    assert (rep.written, rep.cells_traversed) == wrep[:2] and rep.spec.total_digits == 7
    # int64 facade input, a negative value the sample misses: negative_value, as the reference
    vals = keys.astype(np.int64)
    vals[3] = -4
    with pytest.raises(rs.Error) as e:
        rs.sort_i64(torch.from_numpy(vals).cuda())
    assert e.value.code == "negative_value"


@pytest.mark.parametrize("pattern", ["switch", "sparse", "outside"])
def test_partition_ranges_under_shifting_buckets(rs, oracle, pattern):
    """The warp-specialised partition sizes each bucket's staging range from
    its count two tiles earlier; keys that find their range full are counted
    straight into the grid.  Inputs whose bucket mix changes from tile to
    tile (4096-key tiles): whole tiles of one bucket after uniform tiles
    ("switch"), buckets that appear only every few tiles ("sparse"), and
    keys outside a declared width mixed in (the dummy range, then the redo)."""
    import torch

    rng = np.random.default_rng(7)
    tiles = 2048
    keys = oracle.gen_u32(81, 0, tiles * 4096, 10**6).reshape(tiles, 4096)
    if pattern == "switch":
        for t in range(0, tiles, 5):
            keys[t] = 10**4 * (t % 100) + rng.integers(0, 10**4, 4096)  # one bucket per tile
    elif pattern == "sparse":
        for t in range(tiles):
            if t % 7 == 3:
                keys[t, :3000] = 990_000 + rng.integers(0, 10**4, 3000)  # bucket 99, 3000 keys, every 7th tile
    else:
        keys[::3, ::97] = 10**6 + rng.integers(0, 10**5, keys[::3, ::97].shape)
    keys = keys.reshape(-1).astype(np.uint32)
    digits = 6
    out, rep = rs.sort_u32(torch.from_numpy(keys.view(np.int32)).cuda(), key_digits=digits)
    want, wrep = oracle.sort_integers_u32(keys)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)
    assert (rep.written, rep.cells_traversed) == wrep[:2]


@pytest.mark.parametrize("pattern", ["hot-bucket", "one-value", "two-values"])
def test_direct_partition_overflowing_rings(rs, oracle, pattern):
    """The direct partition (4-byte keys) gives each bucket a 512-slot shared
    ring per tile window; a bucket taking more keys than its writable chunks
    hold counts the rest straight into the grid (warp-aggregated global
    atomics).  Inputs that overflow the rings on every tile: 60% of the keys
    spread over bucket 0's 10^4 cells, every key one value, half the keys on
    each of two cells of one bucket."""
    import torch

    rng = np.random.default_rng(11)
    n = (1 << 22) + 1234
    keys = oracle.gen_u32(82, 0, n, 10**6)
    if pattern == "hot-bucket":
        hot = rng.random(n) < 0.6
        keys[hot] = rng.integers(0, 10**4, int(hot.sum()))
    elif pattern == "one-value":
        keys[:] = 777_777
    else:
        keys[:] = np.where(rng.random(n) < 0.5, 500_001, 509_999)
    keys[-1] = 999_999  # the grid stays 10^6 cells (two-level split)
    keys = keys.astype(np.uint32)
    out, rep = rs.sort_u32(torch.from_numpy(keys.view(np.int32)).cuda(), key_digits=6)
    want, wrep = oracle.sort_integers_u32(keys)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)
    assert (rep.written, rep.cells_traversed) == wrep[:2]


@pytest.mark.parametrize("n", [(1 << 22) + 1, 3072 * 1000 + 7, 1536 * 999 + 5, 5_000_003])
@pytest.mark.parametrize("bound", [10**5, 10**6])
@pytest.mark.parametrize("width", [4, 8])
def test_direct_partition_tiles_and_tails(rs, oracle, n, bound, width):
    """The direct partition's tile geometry (3072 4-byte or 1536 8-byte keys
    per tile, two ring sets, partial last tile) and its tails (each bucket's
    last ring chunks padded into the page) on 10- and 100-bucket grids,
    through the reference semantics (no declared width) for uint32 and int64
    input."""
    import torch

    keys = oracle.gen_u32(83 + n % 7, 0, n, bound)
    keys[n // 3] = bound - 1  # the grid is 10^digits(bound - 1)
    if width == 4:
        want, wrep = oracle.sort_integers_u32(keys)
        out, rep = rs.sort_u32(torch.from_numpy(keys.view(np.int32)).cuda())
        got = out.cpu().numpy().view(np.uint32)
    else:
        vals = keys.astype(np.int64)
        want, wrep = oracle.sort_integers_i64(vals)
        out, rep = rs.sort_i64(torch.from_numpy(vals).cuda())
        got = out.cpu().numpy()
    assert np.array_equal(got, want)
    assert (rep.written, rep.cells_traversed) == wrep[:2]


@pytest.mark.parametrize("n,outlier", [(100, None), (4097, None), (1 << 20, None), (1 << 20, 999_999),
                                       (1 << 20, 1_234_567), ((1 << 22) - 3, 54_321), (1 << 20, 1000)])
def test_small_sort_sampled_grid(rs, oracle, n, outlier):
    """The one-launch small sort sizes an undeclared grid from a strided
    sample's max; a key past the sampled grid (an outlier off the sample's
    stride) makes the host redo the sort with the exact max, on the small
    path or the multi-pass one."""
    import torch

    keys = oracle.gen_u32(84, 0, n, 1000)
    if outlier is not None:
        keys[n // 2 + 1] = outlier  # off the sample's stride
    want, wrep = oracle.sort_integers_u32(keys)
    out, rep = rs.sort_u32(torch.from_numpy(keys.view(np.int32)).cuda())
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)
    assert (rep.written, rep.cells_traversed, (rep.spec.radix, rep.spec.total_digits, rep.spec.integer_digits)) == wrep


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_emit_part_cuts_match_cell_ranges(rs, oracle, parts):
    """rs_emit_part_u32 (the sharded grid's emit): the device cuts equal
    dist.cell_ranges' rule on a skewed grid, and the parts concatenate to
    the whole sorted sequence."""
    import torch

    from paper_2107_01391_b200.dist import GpuOps, cell_ranges

    lib = rs._lib.load()
    keys = oracle.gen_u32(82, 0, 3_000_017, 10**6)
    keys[::5] = 123_456  # a hot cell
    k = torch.from_numpy(keys.view(np.int32)).cuda()
    ops = GpuOps()
    counts = ops.count(k, 10**6)
    prefix = torch.cumsum(counts.to(torch.int64), 0).cpu()
    want_ranges = cell_ranges(prefix, parts)
    outs = []
    for p in range(parts):
        out = torch.empty(keys.size, dtype=torch.int32, device="cuda")
        written = ctypes.c_uint64()
        cells = (ctypes.c_uint64 * 2)()
        rs._check(lib.rs_emit_part_u32(rs._ptr(counts), 10**6, p, parts, rs._ptr(out), out.numel(),
                                       ctypes.byref(written), cells, rs._stream()))
        assert (cells[0], cells[1]) == want_ranges[p]
        outs.append(out[: written.value].cpu().numpy().view(np.uint32))
    assert np.array_equal(np.concatenate(outs), np.sort(keys))


@pytest.mark.parametrize("cells", [2_000_000, 2_560_000, 1_280_001])
def test_count_grids_with_two_buckets_per_store_thread(rs, oracle, cells):
    """Grids of 129-256 outer buckets: the warp-specialised partition's store
    threads keep two buckets each (rs_count_u32, the multi-GPU count phase,
    takes any grid size).  Counts against a bincount."""
    import torch

    lib = rs._lib.load()
    n = 5_000_011
    keys = oracle.gen_u32(83, 0, n, cells)
    keys[::11] = cells - 1
    k = torch.from_numpy(keys.view(np.int32)).cuda()
    counts = torch.empty(cells, dtype=torch.int32, device="cuda")
    mx = ctypes.c_uint32()
    rs._check(lib.rs_count_u32(rs._ptr(k), n, rs._ptr(counts), cells, ctypes.byref(mx), rs._stream()))
    assert mx.value == cells - 1
    assert np.array_equal(counts.cpu().numpy().astype(np.int64), np.bincount(keys.astype(np.int64), minlength=cells))


def test_kv_above_2_pow_31_records(rs, oracle):
    """Stable key/value over 2^31 + 3 records (uint32 positions and
    offsets throughout): sorted, stable (payload = index), every payload
    pointing at its key."""
    import torch

    lib = rs._lib.load()
    n = (1 << 31) + 3
    k = torch.empty(n, dtype=torch.int32, device="cuda")
    rs._check(lib.rs_gen_u32(oracle.config_seed(2), 0, n, 10**6, rs._ptr(k), rs._stream()))
    v = torch.empty_like(k)
    rs._check(lib.rs_gen_iota_u32(0, n, rs._ptr(v), rs._stream()))
    ko, vo, rep = rs.sort_u32_kv(k, v, key_digits=6)
    assert rep.written == n and rep.cells_traversed == 10**6
    assert bool((ko[1:] >= ko[:-1]).all())
    same = ko[1:] == ko[:-1]
    idx = vo.to(torch.int64) & 0xFFFFFFFF  # payloads past 2^31 are negative as int32
    assert bool((idx[1:][same] > idx[:-1][same]).all())
    del same
    assert torch.equal(k[idx], ko)
    del k, v, ko, vo
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [(1 << 22) + 77, 4096 * 700 + 1])
def test_int64_partition_matches_reference(rs, oracle, n):
    """int64 input (sort_integers' span<const int64_t>) through the two-level
    count: the warp-specialised partition maps 8-byte keys out of TMA-filled
    shared-memory tiles into saturated 32-bit cells (the bounds-checked
    global path for the partial last tile)."""
    import torch

    keys = oracle.gen_u32(82, 0, n, 10**6).astype(np.int64)
    keys[-3:] = [999_999, 0, 500_000]  # the partial tile's keys
    out, rep = rs.sort_i64(torch.from_numpy(keys).cuda())
    want, wrep = oracle.sort_integers_i64(keys)
    assert np.array_equal(out.cpu().numpy(), want)
    assert (rep.written, rep.cells_traversed) == wrep[:2] and rep.spec.total_digits == 6


def test_int64_partition_key_beyond_32_bits(rs, oracle):
    """With a declared 6-digit width, a key of 11 digits (> 2^33) saturates
    to an out-of-grid cell in the partition; the sort is redone at the true
    width from the exact 64-bit max, whose 10^11 cells exceed the budget —
    the reference's error for the same keys."""
    import torch

    keys = oracle.gen_u32(83, 0, (1 << 21) + 9, 10**6).astype(np.int64)
    keys[12345] = 10**10 + 3
    with pytest.raises(oracle_error_type()):
        oracle.sort_integers_i64(keys)
    with pytest.raises(rs.Error) as e:
        rs.sort_i64(torch.from_numpy(keys).cuda(), key_digits=6)
    assert e.value.code == "cell_budget_exceeded"
    assert "needs 100000000000 cells" in str(e.value)
    # in budget: the same keys below 10^7 after the redo (7 digits), as the reference
    keys[12345] = 9_999_999
    out, rep = rs.sort_i64(torch.from_numpy(keys).cuda(), key_digits=6)
    want, wrep = oracle.sort_integers_i64(keys)
    assert np.array_equal(out.cpu().numpy(), want)
    assert (rep.written, rep.cells_traversed) == wrep[:2] and rep.spec.total_digits == 7


def oracle_error_type():
    from oracle import OracleError

    return OracleError
