"""Multi-GPU execution of the hot path: one process per GPU, NCCL plumbing.

SURVEY.md §8(e): the stream index space shards naturally.  Rank g of G owns a
contiguous block of stream ordinals:
  * uniform-kind fills (ordinal i + g0*j): a block of grid columns j, aligned
    to column quads / pairs so the wide-store kernels apply;
  * normal fills (ordinal i*g1 + j): a block of grid rows i;
  * fisher_sim: a block of work items (= streams).

Fills need no data-path collective and each rank allocates only its own
cells.  A rank's block of grid columns [j_lo, j_hi) owns the matrix columns
c = j + g1 q; stored compactly as (nrow, q, j) it is exactly the fill of a
(nrow, Q w + rem) matrix on the sub-grid (g0, w = j_hi - j_lo) whose item
(i, j') is stream i + g0 (j' + j_lo): the same kernel on the state array
offset by g0 j_lo, the same draws in the same order (_kernels.py:50-80: an
item visits its cells row-major).  Normal fills shard grid rows the same way
(sub-grid (h, g1), stream offset i_lo g1, _kernels.py:108-166).  So per-rank
memory is ~1/G of the matrix and the output can exceed one GPU's HBM;
`gather_fill` assembles the full matrix on request.

fisher_sim does ONE all-reduce of the int64 hit count.  Stream states: each
rank advances only its block; with sync_states=True (default) the blocks are
all-gathered so every rank holds exactly the StreamSet a single-GPU run would
have produced (`sync_streams` does it later for callers that defer it).

The per-shard work goes through an executor.  `DeviceExecutor` is the product
(sm_100a kernels via the C ABI, NCCL over NVLink).  Tests substitute a CPU
executor to exercise this host logic with the `gloo` backend on machines without
GPUs; that executor lives in tests/ and is never used by the product path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidArgumentError
from .fisher import FisherResult, launch_fisher, plan_fisher
from .grid import MatrixBuffer, check_fill, launch_fill


def shard_range(n_units: int, rank: int, world: int, align: int = 1):
    """Contiguous block [lo, hi) of range(n_units) for `rank`; interior
    boundaries are multiples of `align` (the last block takes the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidArgumentError("bad rank/world")
    blocks = n_units // align
    lo = blocks * rank // world * align
    hi = n_units if rank == world - 1 else blocks * (rank + 1) // world * align
    return lo, hi


def fill_shard(kind: str, g0: int, g1: int, rank: int, world: int):
    """Stream-ordinal block of `rank` for a fill of this kind on a (g0, g1) grid."""
    if kind == "normal":
        return shard_range(g0 * g1, rank, world, align=g1)  # whole grid rows
    # whole column quads (the 256-bit store kernel) or pairs when possible
    align = 4 * g0 if g1 % 4 == 0 else 2 * g0 if g1 % 2 == 0 else g0
    return shard_range(g0 * g1, rank, world, align=align)


@dataclass(frozen=True)
class FillShard:
    """One rank's block of a sharded fill and its compact layout.

    Global problem: (nrow, ncol) on grid (g0, g1), stream ordinals [lo, hi).
    Compact problem: (sub_nrow, sub_ncol) on grid (sub_g0, sub_g1), stream
    ordinals [0, hi - lo) of the state array offset by `lo`."""

    kind: str
    nrow: int
    ncol: int
    g0: int
    g1: int
    lo: int
    hi: int
    sub_nrow: int
    sub_ncol: int
    sub_g0: int
    sub_g1: int

    @property
    def cells(self) -> int:
        return self.sub_nrow * self.sub_ncol

    def global_index(self):
        """Where the compact shard's rows (normal) or columns (uniform kinds)
        sit in the global matrix: an int64 array over the sharded axis."""
        if self.kind == "normal":
            h, i_lo = max(self.sub_g0, 1), self.lo // self.g1
            r = np.arange(self.sub_nrow, dtype=np.int64)
            return i_lo + r % h + self.g0 * (r // h)
        w, j_lo = max(self.sub_g1, 1), self.lo // self.g0
        c = np.arange(self.sub_ncol, dtype=np.int64)
        return j_lo + c % w + self.g1 * (c // w)


def fill_shard_layout(kind: str, nrow: int, ncol: int, g0: int, g1: int, rank: int,
                      world: int) -> FillShard:
    """The compact layout of `rank`'s block (see the module docstring)."""
    lo, hi = fill_shard(kind, g0, g1, rank, world)
    if kind == "normal":
        i_lo, i_hi = lo // g1, hi // g1
        h = i_hi - i_lo
        p, r0 = divmod(nrow, g0)
        rows = p * h + min(max(r0 - i_lo, 0), h)
        return FillShard(kind, nrow, ncol, g0, g1, lo, hi, rows, ncol if rows else 0, h, g1)
    j_lo, j_hi = lo // g0, hi // g0
    w = j_hi - j_lo
    q, r0 = divmod(ncol, g1)
    cols = q * w + min(max(r0 - j_lo, 0), w)
    return FillShard(kind, nrow, ncol, g0, g1, lo, hi, nrow if cols else 0, cols, g0, w)


def _dist():
    import torch.distributed as dist

    return dist


def _world(group):
    dist = _dist()
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


class DeviceExecutor:
    """Runs shards on this rank's GPU through libsfb.so (the product path)."""

    def __init__(self):
        import torch

        _lib.require_device()
        self.device = torch.device("cuda", torch.cuda.current_device())

    def states(self, streams):
        return streams.device_current(self.device)

    def commit_states(self, streams):
        streams._mark_device_ahead()

    def fisher(self, plan, streams, lo, hi, want_stats):
        import torch

        cur = self.states(streams)
        count = torch.zeros(1, dtype=torch.int64, device=self.device)
        stats = torch.empty(max(hi - lo, 0) * plan.reps, dtype=torch.float64,
                            device=self.device) if want_stats else None
        launch_fisher(plan, cur, streams.count, count, item_lo=lo, item_hi=hi, stats_dev=stats)
        self.commit_states(streams)
        return count, stats

    def fill(self, shard: FillShard, streams, rate, dtype):
        """The rank's compact shard: the sub-grid fill on the offset states."""
        import torch

        from .grid import _torch_dtype

        cur = self.states(streams)
        if shard.cells == 0:  # this rank's streams own no cell (and do not advance)
            t = torch.empty((shard.sub_nrow, shard.sub_ncol), dtype=_torch_dtype(dtype),
                            device=self.device)
            return MatrixBuffer.wrap(t, dtype)
        buf = MatrixBuffer.on_device(shard.sub_nrow, shard.sub_ncol, dtype=dtype)
        launch_fill(shard.kind, cur[shard.lo:], streams.count - shard.lo, buf.tensor,
                    shard.sub_nrow, shard.sub_ncol, shard.sub_ncol, shard.sub_g0, shard.sub_g1,
                    rate=rate)
        self.commit_states(streams)
        return buf


def _allgather_rows(executor, streams, lo, hi, group):
    """Every rank contributes its rows [lo, hi) of the state array; every rank
    installs all of them (padding to the largest block for the collective)."""
    import torch

    dist = _dist()
    _, world = _world(group)
    cur = executor.states(streams)
    bounds = torch.tensor([lo, hi], dtype=torch.int64, device=cur.device)
    allb = [torch.empty_like(bounds) for _ in range(world)]
    dist.all_gather(allb, bounds, group=group)
    allb = [tuple(int(x) for x in b.tolist()) for b in allb]
    width = max(h - l for l, h in allb)
    mine = torch.zeros((width, 6), dtype=torch.int64, device=cur.device)
    mine[: hi - lo] = cur[lo:hi]
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    for (l, h), part in zip(allb, parts):
        cur[l:h] = part[: h - l]
    executor.commit_states(streams)


def sync_streams(streams, lo, hi, group=None, executor=None):
    """Collective: after sharded calls made with sync_states=False, every rank
    contributes its block [lo, hi) and ends with the full single-GPU state."""
    _, world = _world(group)
    if world > 1:
        _allgather_rows(executor or DeviceExecutor(), streams, lo, hi, group)


def fisher_sim_sharded(table, n, streams, grid, return_stats=False, group=None,
                       executor=None, sync_states=True) -> FisherResult:
    """fisher_sim (fisher.py:118-164) over all ranks of `group`: identical
    counts, p-value, statistics and final states to a single-device run."""
    import torch

    dist = _dist()
    plan = plan_fisher(table, n, streams, grid)
    executor = executor or DeviceExecutor()
    rank, world = _world(group)
    lo, hi = shard_range(plan.nitems, rank, world)
    count, stats = executor.fisher(plan, streams, lo, hi, return_stats)
    if world > 1:
        dist.all_reduce(count, op=dist.ReduceOp.SUM, group=group)  # the one collective
    counts = int(count.item())
    full_stats = None
    if return_stats:
        if world > 1:
            width = max(b - a for a, b in (shard_range(plan.nitems, r, world)
                                           for r in range(world))) * plan.reps
            pad = torch.zeros(width, dtype=stats.dtype, device=stats.device)
            pad[: stats.numel()] = stats
            parts = [torch.empty_like(pad) for _ in range(world)]
            dist.all_gather(parts, pad, group=group)
            pieces = []
            for r, part in enumerate(parts):
                a, b = shard_range(plan.nitems, r, world)
                pieces.append(part[: (b - a) * plan.reps])
            stats = torch.cat(pieces)
        full_stats = _lib.to_host(stats)
    if world > 1 and sync_states:
        _allgather_rows(executor, streams, lo, hi, group)
    return FisherResult(threshold=plan.threshold, sim_num=plan.sim_num, counts=counts,
                        p_value=(1 + counts) / (plan.sim_num + 1), statistics=full_stats)


def gather_fill(buf: MatrixBuffer, group=None, npad=None) -> MatrixBuffer:
    """Collective: every rank's compact shard of one sharded fill, assembled
    into the full (nrow, npad) matrix on every rank (an all-gather of the
    shards padded to the largest; padding columns zero)."""
    import torch

    dist = _dist()
    shard = buf.shard
    _, world = _world(group)
    npad = shard.ncol if npad is None else npad
    full = torch.zeros((shard.nrow, npad), dtype=buf.tensor.dtype, device=buf.tensor.device)
    layouts = [fill_shard_layout(shard.kind, shard.nrow, shard.ncol, shard.g0, shard.g1, r,
                                 world) for r in range(world)]
    if world > 1:
        width = max(max(s.cells for s in layouts), 1)
        mine = torch.zeros(width, dtype=buf.tensor.dtype, device=buf.tensor.device)
        mine[: shard.cells] = buf.tensor.reshape(-1)
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
    else:
        parts = [buf.tensor.reshape(-1)]
    for s, part in zip(layouts, parts):
        if s.cells == 0:
            continue
        piece = part[: s.cells].reshape(s.sub_nrow, s.sub_ncol)
        idx = torch.from_numpy(s.global_index()).to(full.device)
        if s.kind == "normal":
            full.index_copy_(0, idx, piece)
        else:
            full.index_copy_(1, idx, piece)
    return MatrixBuffer.wrap(full, buf.dtype, ncol=shard.ncol)


def run_grid_sharded(streams, grid, nrow, ncol, kind, rate=1.0, npad=None, dtype=None,
                     group=None, executor=None, gather=False, sync_states=True):
    """run_grid (grid.py:112-144) over all ranks: each rank fills the cells of
    its stream block into a compact shard (`.shard` describes it; ~1/G of the
    matrix per rank).  gather=True returns the full (nrow, npad) matrix on
    every rank instead (gather_fill).  sync_states=True all-gathers the
    advanced stream blocks so every rank ends with the single-GPU StreamSet."""
    out_dtype = check_fill(streams, grid, kind, dtype)
    executor = executor or DeviceExecutor()
    rank, world = _world(group)
    shard = fill_shard_layout(kind, nrow, ncol, grid.nglobal0, grid.nglobal1, rank, world)
    buf = executor.fill(shard, streams, rate, out_dtype)
    buf.shard = shard
    if world > 1 and sync_states:
        _allgather_rows(executor, streams, shard.lo, shard.hi, group)
    if gather:
        full = gather_fill(buf, group, npad=ncol if npad is None else npad)
        full.shard = shard
        return full
    return buf
