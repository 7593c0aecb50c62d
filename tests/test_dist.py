"""Multi-GPU host logic (paper_2107_01391_b200/dist.py) on CPU:
world-size-2 gloo process groups with the device phases replaced by
test-only numpy stand-ins.  What is exercised is exactly the product's
collective / splitter / range logic: the grid all-reduce, the contiguous cell
ranges per rank, the MSD bucket splitters, the all-to-all exchange and the
concatenation property (rank outputs in rank order == the sorted input)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_01391_b200.dist import (bucket_splitters, cell_ranges, range_partition_sort, sharded_grid_sort,
                                        sharded_kv_sort)


class NumpyOps:
    """Test-only stand-ins for GpuOps (the product always uses the CUDA library)."""

    def count(self, keys, cells):
        return torch.from_numpy(np.bincount(keys.numpy().astype(np.int64), minlength=cells).astype(np.int32))

    def emit_part(self, counts, part, parts, cap):
        prefix = torch.cumsum(counts.to(torch.int64), 0)
        lo, hi = cell_ranges(prefix, parts)[part]
        c = counts.numpy()[lo:hi].astype(np.int64)
        out = np.repeat(np.arange(lo, hi, dtype=np.int64), c).astype(np.int32)
        assert out.size <= cap
        return torch.from_numpy(out)

    def bucket_hist(self, keys, divisor, buckets):
        b = (keys.numpy().view(np.uint32).astype(np.int64) // divisor)
        return torch.from_numpy(np.bincount(b, minlength=buckets).astype(np.int64))

    def partition(self, keys, divisor, bounds):
        k = keys.numpy().view(np.uint32).astype(np.int64)
        part = np.searchsorted(np.asarray(bounds[1:-1]), k // divisor, side="right")
        order = np.argsort(part, kind="stable")
        return torch.from_numpy(keys.numpy()[order].copy()), np.bincount(part, minlength=len(bounds) - 1).tolist()

    def sort_kv(self, keys, vals, cells):
        k = keys.numpy().view(np.uint32)
        assert k.size == 0 or int(k.max()) < cells
        order = np.argsort(k, kind="stable")
        return torch.from_numpy(keys.numpy()[order].copy()), torch.from_numpy(vals.numpy()[order].copy())

    # the fused exchange: "peer memory" = tensors shared by the test's processes
    def __init__(self, bufs=None, rank=0):
        self.bufs, self.rank = bufs, rank

    def part_counts(self, keys, divisor, bounds):
        k = keys.numpy().view(np.uint32).astype(np.int64)
        part = np.searchsorted(np.asarray(bounds[1:-1]), k // divisor, side="right")
        return np.bincount(part, minlength=len(bounds) - 1).tolist()

    def partition_to(self, keys, divisor, bounds, dsts, offsets):
        k = keys.numpy().view(np.uint32).astype(np.int64)
        part = np.searchsorted(np.asarray(bounds[1:-1]), k // divisor, side="right")
        for r, off in enumerate(offsets):
            mine = keys.numpy()[part == r]
            dsts[r][off:off + mine.size] = torch.from_numpy(mine.copy())

    def peer_buffer(self, cap, group=None, name="keys"):
        bufs = self.bufs[name] if isinstance(self.bufs, dict) else self.bufs
        assert cap <= bufs[self.rank].numel()
        return bufs[self.rank], bufs

    def kv_place(self, ks, vs, cell_off, owner, dst_k, dst_v):
        k = ks.numpy().view(np.uint32).astype(np.int64)
        pos = cell_off.numpy()[k] + np.arange(k.size)
        own = owner.numpy()[k]
        for r in range(len(dst_k)):
            sel = own == r
            dst_k[r][torch.from_numpy(pos[sel])] = torch.from_numpy(ks.numpy()[sel].copy())
            dst_v[r][torch.from_numpy(pos[sel])] = torch.from_numpy(vs.numpy()[sel].copy())

    def exchange_barrier(self, group=None):
        dist.barrier(group)

    def peer_exchange_ok(self, group=None):
        return self.bufs is not None

    def sort(self, keys, key_digits=0):
        return torch.from_numpy(np.sort(keys.numpy().view(np.uint32)).view(np.int32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, shared):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = shared["keys"]
        n = keys.numel()
        mine = keys[rank * n // world:(rank + 1) * n // world].clone()
        if mode == "grid":
            out = sharded_grid_sort(mine, shared["cells"], ops=NumpyOps())
        elif mode in ("kv", "kvp2p"):
            vals = torch.arange(rank * n // world, (rank + 1) * n // world, dtype=torch.int32)
            if mode == "kv":
                out = torch.stack(sharded_kv_sort(mine, vals, shared["cells"], ops=NumpyOps(), exchange="nccl"))
            else:
                out = torch.stack(sharded_kv_sort(mine, vals, shared["cells"], ops=NumpyOps(shared["bufs"], rank),
                                                  exchange="p2p"))
        elif mode == "p2p":
            out = range_partition_sort(mine, shared["divisor"], shared["buckets"],
                                       ops=NumpyOps(shared["bufs"], rank), exchange="p2p")
        else:
            out = range_partition_sort(mine, shared["divisor"], shared["buckets"], ops=NumpyOps(), exchange="nccl")
        torch.save(out, shared["dir"] + f"/out{rank}.pt")
    finally:
        dist.destroy_process_group()


def _run(mode, keys, tmp_path, **kw):
    world = 2
    shared = {"keys": keys, "dir": str(tmp_path), **kw}
    mp.spawn(_worker, args=(world, _free_port(), mode, shared), nprocs=world, join=True)
    return [torch.load(str(tmp_path) + f"/out{r}.pt") for r in range(world)]


def test_cell_ranges_balance_and_cover():
    counts = torch.tensor([5, 0, 0, 7, 1, 1, 0, 9, 2, 3])
    prefix = torch.cumsum(counts, 0)
    for world in (1, 2, 3, 4, 8):
        r = cell_ranges(prefix, world)
        assert r[0][0] == 0 and r[-1][1] == counts.numel()
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))  # contiguous, cuts on cell boundaries
    r = cell_ranges(prefix, 2)
    left = int(counts[r[0][0]:r[0][1]].sum())
    assert abs(left - (28 - left)) <= 9  # never splits a cell; within one cell of balance


def test_device_cell_bounds_match_host_ranges():
    from paper_2107_01391_b200.dist import cell_bounds_device

    g = torch.Generator().manual_seed(5)
    for trial in range(40):
        cells = int(torch.randint(1, 300, (1,), generator=g))
        counts = torch.randint(0, 4, (cells,), generator=g) * (torch.rand(cells, generator=g) < 0.5)
        if trial % 5 == 0:
            counts[int(torch.randint(0, cells, (1,), generator=g))] += 500  # one hot cell
        prefix = torch.cumsum(counts, 0, dtype=torch.int64)
        for world in (1, 2, 3, 5, 8):
            want = [lo for lo, _ in cell_ranges(prefix, world)] + [cells]
            assert cell_bounds_device(prefix, world).tolist() == want


def test_bucket_splitters_cover_all_buckets():
    hist = torch.tensor([0, 100, 3, 3, 3, 200, 0, 50])
    b = bucket_splitters(hist, 4)
    assert b[0] == 0 and b[-1] == hist.numel() and len(b) == 5
    assert all(x <= y for x, y in zip(b, b[1:]))


def test_sharded_grid_sort_gloo(tmp_path):
    rng = np.random.default_rng(3)
    keys = torch.from_numpy(rng.integers(0, 10**5, 200_001).astype(np.int32))
    outs = _run("grid", keys, tmp_path, cells=10**5)
    got = np.concatenate([o.numpy() for o in outs])
    assert np.array_equal(got, np.sort(keys.numpy()))
    # the rank slices are contiguous cell ranges and roughly balanced
    assert abs(outs[0].numel() - outs[1].numel()) < 200_001 // 10


def test_range_partition_sort_gloo(tmp_path):
    rng = np.random.default_rng(4)
    keys = torch.from_numpy(rng.integers(0, 2**32, 100_003, dtype=np.uint64).astype(np.uint32).view(np.int32))
    outs = _run("range", keys, tmp_path, divisor=10**7, buckets=430)
    got = np.concatenate([o.numpy().view(np.uint32) for o in outs])
    assert np.array_equal(got, np.sort(keys.numpy().view(np.uint32)))


@pytest.mark.parametrize("bound", [1000, 10**5])
def test_sharded_kv_sort_gloo_is_globally_stable(tmp_path, bound):
    """Values are global input indices: the rank slices, concatenated, must be
    the unique stable order (equal keys of rank 0's shard before rank 1's)."""
    rng = np.random.default_rng(bound)
    keys = rng.integers(0, bound, 150_001).astype(np.int32)
    keys[rng.random(keys.size) < 0.2] = 7  # a hot cell spread over both shards
    outs = _run("kv", torch.from_numpy(keys), tmp_path, cells=bound)
    got = np.concatenate([o.numpy() for o in outs], axis=1)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(got[0], keys[order])
    assert np.array_equal(got[1], order.astype(np.int32))


def test_range_partition_fused_exchange_gloo(tmp_path):
    """The fused exchange's bookkeeping (per-destination counts all-gathered,
    write offsets per source rank, parts stored straight into the peers'
    buffers, barrier, local sort) with two processes writing into each
    other's shared buffers; twice in a row, so the reused buffers are
    overwritten in order."""
    rng = np.random.default_rng(9)
    keys = torch.from_numpy(rng.integers(0, 2**32, 100_003, dtype=np.uint64).astype(np.uint32).view(np.int32))
    keys[:30_000] = keys[0]  # a hot bucket on rank 0's side
    bufs = [torch.zeros(keys.numel(), dtype=torch.int32).share_memory_() for _ in range(2)]
    for _ in range(2):
        outs = _run("p2p", keys, tmp_path, divisor=10**7, buckets=430, bufs=bufs)
        got = np.concatenate([o.numpy().view(np.uint32) for o in outs])
        assert np.array_equal(got, np.sort(keys.numpy().view(np.uint32)))


@pytest.mark.parametrize("bound", [1000, 10**5])
def test_sharded_kv_fused_placement_gloo(tmp_path, bound):
    """The fused key/value placement (all-gathered grids -> every record's
    final position -> stores into the owners' shared buffers): the rank
    slices concatenate to the unique stable order, hot cell included."""
    rng = np.random.default_rng(bound + 1)
    keys = rng.integers(0, bound, 150_001).astype(np.int32)
    keys[rng.random(keys.size) < 0.2] = 7
    bufs = {name: [torch.zeros(keys.size, dtype=torch.int32).share_memory_() for _ in range(2)]
            for name in ("kv_keys", "kv_vals")}
    outs = _run("kvp2p", torch.from_numpy(keys), tmp_path, cells=bound, bufs=bufs)
    got = np.concatenate([o.numpy() for o in outs], axis=1)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(got[0], keys[order])
    assert np.array_equal(got[1], order.astype(np.int32))


def test_kv_placement_tables():
    """kv_placement on a hand-checked 2-rank, 4-cell case."""
    from paper_2107_01391_b200.dist import kv_placement

    grids = torch.tensor([2, 0, 1, 3,   # rank 0's counts per cell
                          1, 2, 0, 1])  # rank 1's
    off0, owner, sizes = kv_placement(grids, 0, 2)
    off1, _, _ = kv_placement(grids, 1, 2)
    # totals [3, 2, 1, 4] -> starts [0, 3, 5, 6]; cuts at ceil(10/2) = 5 -> rank 0 owns cells 0-1
    assert owner.tolist() == [0, 0, 1, 1] and sizes.tolist() == [5, 5]
    # rank 0's sorted records: cell 0 (i = 0, 1), cell 2 (i = 2), cell 3 (i = 3, 4, 5)
    #   -> slice 0 positions 0, 1; slice 1 positions 0 (global 5) and 1, 2, 3 (global 6-8)
    assert [int(off0[k]) + i for k, i in [(0, 0), (0, 1), (2, 2), (3, 3), (3, 5)]] == [0, 1, 0, 1, 3]
    # rank 1's: cell 0 (i = 0) after rank 0's two -> 2; cell 1 (i = 1, 2) -> 3, 4; cell 3 (i = 3)
    #   after rank 0's three -> global 9 -> slice 1 position 4
    assert [int(off1[k]) + i for k, i in [(0, 0), (1, 1), (1, 2), (3, 3)]] == [2, 3, 4, 4]
