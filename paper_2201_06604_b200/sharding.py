"""Multi-GPU execution of the hot path: one process per GPU, NCCL plumbing.

SURVEY.md §8(e): the stream index space shards naturally.  Rank g of G owns a
contiguous block of stream ordinals:
  * uniform-kind fills (ordinal i + g0*j): a block of grid columns j, aligned
    to column pairs so the 16-byte-store kernel applies;
  * normal fills (ordinal i*g1 + j): a block of grid rows i;
  * fisher_sim: a block of work items (= streams).
Fills need no data-path collective (each rank writes its cells; outputs stay
sharded unless `gather=True`).  fisher_sim does ONE all-reduce of the int64 hit
count.  Afterwards the updated stream states are all-gathered so every rank
holds exactly the StreamSet a single-GPU run would have produced.

The per-shard work goes through an executor.  `DeviceExecutor` is the product
(sm_100a kernels via the C ABI, NCCL over NVLink).  Tests substitute a CPU
executor to exercise this host logic with the `gloo` backend on machines without
GPUs; that executor lives in tests/ and is never used by the product path.
"""

from __future__ import annotations

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

    def fill(self, kind, streams, nrow, ncol, npad, g0, g1, lo, hi, rate, dtype, zero):
        cur = self.states(streams)
        buf = MatrixBuffer.on_device(nrow, ncol, npad, dtype=dtype, zero=zero)
        launch_fill(kind, cur, streams.count, buf.tensor, nrow, ncol, buf.npad, g0, g1,
                    rate=rate, item_lo=lo, item_hi=hi)
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


def fisher_sim_sharded(table, n, streams, grid, return_stats=False, group=None,
                       executor=None) -> FisherResult:
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
    if world > 1:
        _allgather_rows(executor, streams, lo, hi, group)
    return FisherResult(threshold=plan.threshold, sim_num=plan.sim_num, counts=counts,
                        p_value=(1 + counts) / (plan.sim_num + 1), statistics=full_stats)


def run_grid_sharded(streams, grid, nrow, ncol, kind, rate=1.0, npad=None, dtype=None,
                     group=None, executor=None, gather=False):
    """run_grid (grid.py:112-144) over all ranks: each rank fills the cells of
    its stream block; states are all-gathered.  With gather=True the buffers
    start zeroed and are summed across ranks (disjoint cells), so every rank
    returns the full matrix; otherwise only the rank's own cells are valid."""
    dist = _dist()
    out_dtype = check_fill(streams, grid, kind, dtype)
    executor = executor or DeviceExecutor()
    rank, world = _world(group)
    lo, hi = fill_shard(kind, grid.nglobal0, grid.nglobal1, rank, world)
    buf = executor.fill(kind, streams, nrow, ncol, ncol if npad is None else npad,
                        grid.nglobal0, grid.nglobal1, lo, hi, rate, out_dtype,
                        zero=gather and world > 1)
    if world > 1:
        if gather:
            dist.all_reduce(buf.tensor, op=dist.ReduceOp.SUM, group=group)
        _allgather_rows(executor, streams, lo, hi, group)
    buf.shard = (lo, hi)
    return buf
