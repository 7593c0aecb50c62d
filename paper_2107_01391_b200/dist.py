"""Multi-GPU orchestration of the count-grid sort, one process per
GPU over torch.distributed (NCCL on the GPU box).

Small grids (cfg1-3): every rank counts its contiguous key shard into the full
grid (rs_count_u32), the grids are summed with one all-reduce over NVLink,
and each rank then emits a contiguous range of cells holding about total/G
keys (rs_emit_part_u32: global prefix, cuts and the range emit in one call).  No
key moves between GPUs: rank r's output is slice r
of the globally sorted sequence.

Stable key/value (cfg2 KV): the per-rank grids are all-gathered (a G x cells
table), which fixes the cell cuts and, for every record, its final global
position: global start of its cell + the earlier ranks' counts of that cell
+ its rank among this rank's equal keys.  Every rank sorts its
shard stably (rs_sort_u32_kv) and a placement kernel (rs_kv_place_u32)
writes each record straight to that position in the owning rank's output
slice through NVLink peer pointers — the exchange and the merge in one pass,
no receive-side sort.  The reference's stable order (radix_sort_lsd_by,
baselines.hpp:24-46) is unique, so the rank slices concatenate to it.  The
NCCL variant (all-to-all by cell range, then a stable sort of the received
runs) remains for groups without peer memory.

Wide keys (cfg5): the leading-digit bucket histogram (rs_bucket_hist_u32) is
all-reduced, G-1 splitters are cut on bucket boundaries and every rank sorts
the key range it owns.  The exchange is fused into the partition kernel:
per-destination counts are all-gathered (a G x G table, G^2 integers), each
rank's write offset in every destination follows from it, and the scatter
(rs_partition_u32_to) stores each part straight into its destination rank's
receive buffer through NVLink peer pointers (torch symmetric memory) — no
separate all-to-all pass over the keys.  A device-side barrier of the
symmetric buffer orders the writes before the local sorts.  The NCCL
all-to-all path (rs_partition_u32 + all_to_all_single) remains for process
groups without peer memory.

The device phases are injected (``ops``) so the collective and splitter logic
can be exercised on CPU with the gloo backend in tests; the product path
always uses ``GpuOps`` (the CUDA library) and there is no CPU fallback.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist


def cell_ranges(prefix: torch.Tensor, world: int) -> list[tuple[int, int]]:
    """Contiguous cell ranges with about total/world keys each.

    ``prefix`` is the inclusive prefix sum of the global grid (int64).  Range r
    ends at the first cell whose prefix reaches ceil((r+1)*total/world); cuts
    fall on cell boundaries, so a hot cell is never split."""
    cells = prefix.numel()
    total = int(prefix[-1]) if cells else 0
    bounds = [0]
    for r in range(1, world):
        target = (r * total + world - 1) // world
        cut = int(torch.searchsorted(prefix, torch.tensor([target], dtype=prefix.dtype), right=False)[0]) + 1
        cut = min(max(cut, bounds[-1]), cells)
        bounds.append(cut)
    bounds.append(cells)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def cell_bounds_device(prefix: torch.Tensor, world: int) -> torch.Tensor:
    """cell_ranges on the prefix's own device: the world+1 range bounds as a
    tensor (same cuts: first cell whose prefix reaches ceil(r*total/world),
    plus one, clamped to be monotone and <= cells)."""
    cells = prefix.numel()
    total = prefix[-1]
    r = torch.arange(1, world, device=prefix.device, dtype=torch.int64)
    targets = (r * total + world - 1) // world
    cuts = torch.searchsorted(prefix, targets, right=False) + 1
    cuts = torch.cummax(cuts.clamp(min=0, max=cells), 0).values
    zero = torch.zeros(1, dtype=torch.int64, device=prefix.device)
    return torch.cat([zero, cuts, torch.full((1,), cells, dtype=torch.int64, device=prefix.device)])


def bucket_splitters(hist: torch.Tensor, world: int) -> list[int]:
    """Part bounds over buckets (len world+1, bounds[0]=0, bounds[-1]=buckets)
    with about total/world keys per part, cut on bucket boundaries."""
    prefix = torch.cumsum(hist.to(torch.int64), 0)
    return [lo for lo, _ in cell_ranges(prefix, world)] + [hist.numel()]


class GpuOps:
    """Device phases through the C-ABI (include/recsort_b200.h)."""

    def __init__(self):
        self._symm = {}  # name -> (local tensor, symmetric-memory handle, capacity)

    def _lib(self):
        from . import _lib

        return _lib.load()

    def _check(self, st):
        from . import _check

        _check(st)

    @staticmethod
    def _stream():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def count(self, keys: torch.Tensor, cells: int) -> torch.Tensor:
        counts = torch.empty(cells, dtype=torch.int32, device=keys.device)  # rs_count_u32 overwrites it
        self._check(self._lib().rs_count_u32(ctypes.c_void_p(keys.data_ptr()), keys.numel(),
                                             ctypes.c_void_p(counts.data_ptr()), cells, None, self._stream()))
        return counts

    def emit_part(self, counts: torch.Tensor, part: int, parts: int, cap: int) -> torch.Tensor:
        """Range `part` of `parts` of the global grid (cuts as cell_ranges),
        emitted in one library call (rs_emit_part_u32)."""
        out = torch.empty(max(cap, 1), dtype=torch.int32, device=counts.device)
        written = ctypes.c_uint64()
        self._check(self._lib().rs_emit_part_u32(ctypes.c_void_p(counts.data_ptr()), counts.numel(), part, parts,
                                                 ctypes.c_void_p(out.data_ptr()), out.numel(), ctypes.byref(written),
                                                 None, self._stream()))
        return out[: written.value]

    def bucket_hist(self, keys: torch.Tensor, divisor: int, buckets: int) -> torch.Tensor:
        hist = torch.zeros(buckets, dtype=torch.int64, device=keys.device)
        self._check(self._lib().rs_bucket_hist_u32(ctypes.c_void_p(keys.data_ptr()), keys.numel(), divisor,
                                                   ctypes.c_void_p(hist.data_ptr()), buckets, self._stream()))
        return hist

    def partition(self, keys: torch.Tensor, divisor: int, bounds: list[int]) -> tuple[torch.Tensor, list[int]]:
        parts = len(bounds) - 1
        out = torch.empty_like(keys)
        hb = (ctypes.c_uint32 * (parts + 1))(*bounds)
        hc = (ctypes.c_uint64 * parts)()
        self._check(self._lib().rs_partition_u32(ctypes.c_void_p(keys.data_ptr()), keys.numel(), divisor, hb,
                                                 parts, ctypes.c_void_p(out.data_ptr()), hc, self._stream()))
        return out, [int(c) for c in hc]

    def sort_kv(self, keys: torch.Tensor, vals: torch.Tensor, cells: int) -> tuple[torch.Tensor, torch.Tensor]:
        from . import DEFAULT_CELL_BUDGET, sort_u32_kv

        # the grid's width bounds every key (keys >= cells were rejected by the count)
        digits = len(str(max(cells - 1, 0)))
        k, v, _ = sort_u32_kv(keys, vals, max_cells=max(cells, DEFAULT_CELL_BUDGET), key_digits=digits)
        return k, v

    def part_counts(self, keys: torch.Tensor, divisor: int, bounds: list[int]) -> list[int]:
        parts = len(bounds) - 1
        hb = (ctypes.c_uint32 * (parts + 1))(*bounds)
        hc = (ctypes.c_uint64 * parts)()
        self._check(self._lib().rs_part_counts_u32(ctypes.c_void_p(keys.data_ptr()), keys.numel(), divisor, hb, parts,
                                                   hc, self._stream()))
        return [int(x) for x in hc]

    def partition_to(self, keys: torch.Tensor, divisor: int, bounds: list[int], dsts: list[int],
                     offsets: list[int]) -> None:
        """Part p of `keys` written at device address dsts[p] + 4 * offsets[p]."""
        parts = len(bounds) - 1
        hb = (ctypes.c_uint32 * (parts + 1))(*bounds)
        hd = (ctypes.c_uint64 * parts)(*dsts)
        ho = (ctypes.c_uint64 * parts)(*offsets)
        self._check(self._lib().rs_partition_u32_to(ctypes.c_void_p(keys.data_ptr()), keys.numel(), divisor, hb,
                                                    parts, hd, ho, self._stream()))

    def peer_buffer(self, cap: int, group=None, name: str = "keys") -> tuple[torch.Tensor, list[int]]:
        """This rank's receive buffer `name` (>= cap int32) and every rank's
        address of it (symmetric memory over NVLink); grown identically on
        every rank (cap is a global quantity)."""
        import torch.distributed._symmetric_memory as symm

        t, h, have = self._symm.get(name, (None, None, 0))
        if have < cap:
            size = max(cap, 2 * have, 1 << 20)
            grp = group or dist.group.WORLD
            try:  # older releases need the group registered first; newer ones do it themselves
                if not symm.is_symm_mem_enabled_for_group(grp.group_name):
                    symm.enable_symm_mem_for_group(grp.group_name)
            except Exception:  # noqa: BLE001
                pass
            t = symm.empty(size, dtype=torch.int32, device=torch.device("cuda", torch.cuda.current_device()))
            h = symm.rendezvous(t, grp)
            self._symm[name] = (t, h, size)
        return t, [int(p) for p in h.buffer_ptrs]

    def exchange_barrier(self, group=None) -> None:
        """Device-side barrier over the symmetric buffers: every rank's writes
        before it are visible to every rank after it (stream-ordered)."""
        next(iter(self._symm.values()))[1].barrier()

    def kv_place(self, ks, vs, cell_off, owner, dst_k: list[int], dst_v: list[int]) -> None:
        ranks = len(dst_k)
        hk = (ctypes.c_uint64 * ranks)(*dst_k)
        hv = (ctypes.c_uint64 * ranks)(*dst_v)
        self._check(self._lib().rs_kv_place_u32(ctypes.c_void_p(ks.data_ptr()), ctypes.c_void_p(vs.data_ptr()),
                                                ks.numel(), ctypes.c_void_p(cell_off.data_ptr()),
                                                ctypes.c_void_p(owner.data_ptr()), cell_off.numel(), hk, hv, ranks,
                                                self._stream()))

    def peer_exchange_ok(self, group=None) -> bool:
        """NCCL groups whose symmetric-memory rendezvous works (tried once;
        a failure falls back to the NCCL exchanges)."""
        if dist.get_backend(group) != "nccl":
            return False
        if getattr(self, "_p2p_ok", None) is None:
            try:
                self.peer_buffer(1, group, "probe")
                self._p2p_ok = True
            except Exception:  # noqa: BLE001 — no peer memory here: the NCCL path
                self._p2p_ok = False
        return self._p2p_ok

    def sort(self, keys: torch.Tensor, key_digits: int = 0) -> torch.Tensor:
        from . import sort_u32

        return sort_u32(keys, key_digits=key_digits, msd=True)[0]


def sharded_grid_sort(keys: torch.Tensor, cells: int, ops=None, group=None) -> torch.Tensor:
    """Small-grid sharding: local count -> all-reduce(sum) -> own cell range.
    Returns this rank's contiguous slice of the global sorted sequence."""
    ops = ops or GpuOps()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # the grid travels as 32-bit counters: below 2^32 keys in all, no cell can
    # wrap (bounded here from the local shard, no extra collective)
    if keys.numel() * world >= 1 << 32:
        raise ValueError("sharded_grid_sort: fewer than 2^32 keys in total (world x shard) per call")
    counts = ops.count(keys, cells)
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)  # C1: the grid over NVLink
    # this rank's contiguous cell range (cut_rank .. cut_rank+1, cell_ranges'
    # rule) emitted in one library call; a slice can exceed the even share
    # by at most one cell's keys, so the output is sized for the whole input
    return ops.emit_part(counts, rank, world, keys.numel() * world)


def kv_placement(grids: torch.Tensor, rank: int, world: int):
    """From the all-gathered grids C[g][k]: every cell's owner rank, this
    rank's per-cell placement offset (final global position of its record i
    with key k = offset[k] + i, relative to the owner's slice) and every
    rank's slice size.  Cuts as sharded_grid_sort (cell_bounds_device)."""
    C = grids.view(world, -1).to(torch.int64)
    cells = C.shape[1]
    total = C.sum(0)
    prefix = torch.cumsum(total, 0)
    gstart = prefix - total
    bounds = cell_bounds_device(prefix, world)
    cell_idx = torch.arange(cells, device=grids.device, dtype=torch.int64)
    owner = torch.searchsorted(bounds[1:-1].contiguous(), cell_idx, right=True)
    zero = torch.zeros(1, dtype=torch.int64, device=grids.device)
    ends = torch.cat([zero, prefix])[bounds]  # position where each rank's slice starts (world + 1 entries)
    before = C[:rank].sum(0)
    mine = C[rank]
    local_start = torch.cumsum(mine, 0) - mine
    offset = gstart + before - local_start - ends[owner]
    return offset, owner.to(torch.uint8), (ends[1:] - ends[:-1])


def sharded_kv_sort(keys: torch.Tensor, vals: torch.Tensor, cells: int, ops=None,
                    group=None, exchange: str = "auto") -> tuple[torch.Tensor, torch.Tensor]:
    """Stable key/value across ranks.  p2p: local count ->
    all-gather of the grids -> per-record final positions -> local stable
    sort -> placement straight into the owners' slices over NVLink.  nccl:
    local count -> all-reduce -> cell cuts; local stable sort -> all-to-all by
    cell range -> stable sort of the received runs.  Rank g's shard must be
    slice g of the global input; returns slice r of the global stable order
    (cut on cell boundaries, as sharded_grid_sort)."""
    ops = ops or _gpu_ops()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    counts = ops.count(keys, cells)
    if exchange == "auto":
        exchange = "p2p" if getattr(ops, "peer_exchange_ok", lambda g: False)(group) else "nccl"
    if exchange == "p2p":
        grids = torch.empty(world * cells, dtype=counts.dtype, device=counts.device)
        dist.all_gather_into_tensor(grids, counts, group=group)  # C4: the per-rank grids
        offset, owner, sizes = kv_placement(grids, rank, world)
        ks, vs = ops.sort_kv(keys, vals, cells)
        sizes = sizes.tolist()
        bk, dk = ops.peer_buffer(int(max(sizes)), group, "kv_keys")
        bv, dv = ops.peer_buffer(int(max(sizes)), group, "kv_vals")
        ops.exchange_barrier(group)  # every rank is done with the buffers' previous contents
        ops.kv_place(ks, vs, offset, owner, dk, dv)
        ops.exchange_barrier(group)  # every record has landed
        n = int(sizes[rank])
        return bk[:n].clone(), bv[:n].clone()
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)  # C1
    bounds = cell_bounds_device(torch.cumsum(counts, 0, dtype=torch.int64), world)
    ks, vs = ops.sort_kv(keys, vals, cells)
    # records of cell range r are the run [cut[r], cut[r+1]) of the sorted shard
    cut = torch.searchsorted(ks.to(torch.int64), bounds)
    send = cut[1:] - cut[:-1]
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    both = torch.stack([send, recv]).cpu()
    send_counts, recv_counts = both[0].tolist(), both[1].tolist()
    rk = torch.empty(sum(recv_counts), dtype=keys.dtype, device=keys.device)
    rv = torch.empty(sum(recv_counts), dtype=vals.dtype, device=vals.device)
    dist.all_to_all_single(rk, ks, output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
    dist.all_to_all_single(rv, vs, output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
    return ops.sort_kv(rk, rv, cells)


_GPU_OPS = None


def _gpu_ops() -> "GpuOps":
    global _GPU_OPS
    if _GPU_OPS is None:  # one receive buffer per process, reused across calls
        _GPU_OPS = GpuOps()
    return _GPU_OPS


def range_partition_sort(keys: torch.Tensor, divisor: int, buckets: int, ops=None, group=None,
                         key_digits: int = 0, exchange: str = "auto") -> torch.Tensor:
    """Wide keys: MSD histogram -> all-reduce -> splitters -> partition fused
    with the exchange (peer stores) -> local sort.  Returns this rank's slice
    of the global order.  exchange: "p2p" (partition kernel writes into the
    peers' receive buffers), "nccl" (partition + all_to_all_single), "auto"."""
    ops = ops or _gpu_ops()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    hist = ops.bucket_hist(keys, divisor, buckets)
    dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)  # C2
    bounds = bucket_splitters(hist.cpu(), world)
    if exchange == "auto":
        exchange = "p2p" if getattr(ops, "peer_exchange_ok", lambda g: False)(group) else "nccl"
    if exchange == "p2p":
        send = torch.tensor(ops.part_counts(keys, divisor, bounds), dtype=torch.int64, device=keys.device)
        table = torch.empty(world * world, dtype=torch.int64, device=keys.device)
        dist.all_gather_into_tensor(table, send, group=group)  # C[g][r]: keys rank g sends to rank r
        table = table.view(world, world).cpu()
        offsets = table[:rank].sum(0).tolist()  # where this rank's part r starts in rank r's buffer
        n_recv = int(table[:, rank].sum())
        buf, dsts = ops.peer_buffer(int(table.sum(0).max()), group)
        ops.exchange_barrier(group)  # every rank is done with the buffer's previous contents
        ops.partition_to(keys, divisor, bounds, dsts, offsets)
        ops.exchange_barrier(group)  # every part has landed
        return ops.sort(buf[:n_recv], key_digits)
    parted, send_counts = ops.partition(keys, divisor, bounds)
    send = torch.tensor(send_counts, dtype=torch.int64, device=keys.device)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    recv_counts = [int(c) for c in recv.cpu()]
    received = torch.empty(sum(recv_counts), dtype=keys.dtype, device=keys.device)
    dist.all_to_all_single(received, parted, output_split_sizes=recv_counts, input_split_sizes=send_counts,
                           group=group)  # C3
    return ops.sort(received, key_digits)
