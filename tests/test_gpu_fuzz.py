"""Seeded fuzz of the integer paths against the oracle: sizes that end inside
tiles and pages, domains on both sides of every grid-plan switch (shared
grid, two-level split, L2 grid), hot values that turn on the partition's
lane replicas, and the MSD path over full 32-bit keys.  Bit-exact outputs
and reports."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.choice([1, 2, 7, 4095, 4097, 8191, 65537, 300_001, 1_048_583]))
    bound = int(rng.choice([10, 1000, 12288, 12289, 10**5, 10**6, 5 * 10**6, 10**7]))
    keys = rng.integers(0, bound, n, dtype=np.uint64).astype(np.uint32)
    mode = rng.integers(0, 3)
    if mode == 1 and n > 10:  # hot values: a few keys carry most of the mass
        hot = rng.integers(0, bound, 3)
        pick = rng.random(n) < 0.7
        keys[pick] = hot[rng.integers(0, 3, int(pick.sum()))].astype(np.uint32)
    elif mode == 2:  # sorted / reversed runs
        keys = np.sort(keys)
        if rng.random() < 0.5:
            keys = keys[::-1].copy()
    return keys, bound


@pytest.mark.parametrize("seed", range(24))
def test_sort_u32_fuzz(rs, oracle, seed):
    keys, bound = _case(seed)
    want, wrep = oracle.sort_integers_u32(keys, max_cells=10**9)
    digits = len(str(bound - 1))
    for hint in (0, digits):
        out, rep = rs.sort_u32(_t(keys), key_digits=hint, max_cells=10**9)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want), (seed, hint)
        assert (rep.written, rep.cells_traversed) == wrep[:2], (seed, hint)


@pytest.mark.parametrize("seed", range(8))
def test_sort_u32_msd_fuzz(rs, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.choice([33, 4097, 65536 + 13, 500_000, 2_000_003]))
    keys = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    if seed % 2:
        keys[rng.random(n) < 0.5] = np.uint32(rng.integers(0, 2**32))
    out, _ = rs.sort_u32(_t(keys), msd=True)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), np.sort(keys))


@pytest.mark.parametrize("seed", range(6))
def test_sort_u32_kv_fuzz(rs, oracle, seed):
    rng = np.random.default_rng(200 + seed)
    n = int(rng.choice([5, 4096, 4097, 70_001, 1 << 20]))
    bound = int(rng.choice([7, 100, 10**6, 10**9]))
    keys = rng.integers(0, bound, n, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    wk, wv = oracle.radix_sort_lsd_kv(keys, vals)
    ko, vo, _ = rs.sort_u32_kv(_t(keys), _t(vals), max_cells=10**10)
    assert np.array_equal(ko.cpu().numpy().view(np.uint32), wk)
    assert np.array_equal(vo.cpu().numpy().view(np.uint32), wv)


def _t(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32)).to("cuda")


@pytest.mark.parametrize("n", [(1 << 22) - 1, 1 << 22, (1 << 22) + 1])
@pytest.mark.parametrize("bound", [7, 10**4, 10**4 + 1])
def test_small_path_switch(rs, oracle, n, bound):
    """Around the one-launch small path's limits (2^22 keys; grids up to 10^4
    cells — 10^4 + 1 needs 5 digits, the multi-pass path): same keys and
    report either way, with and without a declared width."""
    rng = np.random.default_rng(n + bound)
    keys = rng.integers(0, bound, n, dtype=np.uint64).astype(np.uint32)
    want, wrep = oracle.sort_integers_u32(keys, max_cells=10**9)
    for hint in (0, len(str(bound - 1))):
        out, rep = rs.sort_u32(_t(keys), key_digits=hint, max_cells=10**9)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), want), hint
        assert (rep.written, rep.cells_traversed) == wrep[:2], hint


def _skewed(rng, n, bound):
    """Keys in [0, bound): uniform, a few hot values, one hot outer bucket
    (a tenth of the range), or sorted runs."""
    keys = rng.integers(0, bound, n, dtype=np.uint64)
    mode = rng.integers(0, 4)
    if mode == 1 and n > 10:
        hot = rng.integers(0, bound, 3, dtype=np.uint64)
        pick = rng.random(n) < 0.6
        keys[pick] = hot[rng.integers(0, 3, int(pick.sum()))]
    elif mode == 2 and n > 10:
        pick = rng.random(n) < 0.5
        keys[pick] = rng.integers(0, max(bound // 10, 1), int(pick.sum()), dtype=np.uint64)
    elif mode == 3:
        keys = np.sort(keys)
    return keys


@pytest.mark.parametrize("seed", range(12))
def test_sort_i64_direct_partition_fuzz(rs, oracle, seed):
    """int64 keys through the direct partition (grids of <= 104 outer
    buckets) and the warp-specialised one (more), across tile tails and
    skew, against the reference semantics (sort_integers)."""
    import torch

    rng = np.random.default_rng(300 + seed)
    n = int(rng.choice([4_194_305, 1536 * 997 + 3, 3_000_001, 5_500_007]))
    bound = int(rng.choice([10**5, 10**6, 2 * 10**6]))
    vals = _skewed(rng, n, bound).astype(np.int64)
    want, wrep = oracle.sort_integers_i64(vals, max_cells=10**9)
    out, rep = rs.sort_i64(torch.from_numpy(vals).cuda(), max_cells=10**9)
    assert np.array_equal(out.cpu().numpy(), want), seed
    assert (rep.written, rep.cells_traversed) == wrep[:2], seed


@pytest.mark.parametrize("seed", range(8))
def test_sort_f64_hot_bucket_fuzz(rs, oracle, seed):
    """float64 values k/1000 whose mapped cells skew one outer bucket (the
    direct partition's hot variant counts it in place), against the oracle."""
    import torch

    rng = np.random.default_rng(400 + seed)
    n = int(rng.choice([4_194_305, 3_000_001, 2_500_003]))
    k = _skewed(rng, n, 10**6)
    if seed % 2:  # a geometric head on top: the shape of cfg3's Zipf half
        head = rng.random(n) < 0.45
        k[head] = np.minimum(rng.geometric(0.002, int(head.sum())), 10**6 - 1).astype(np.uint64)
    x = k.astype(np.float64) / 1000.0
    want, wrep = oracle.sort_f64(x, 3)
    out, rep = rs.sort_f64(torch.from_numpy(x).cuda(), 3)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want), seed
    assert (rep.written, rep.cells_traversed, (rep.spec.radix, rep.spec.total_digits, rep.spec.integer_digits)) == wrep, seed
