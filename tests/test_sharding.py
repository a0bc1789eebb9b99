"""Multi-process tests of the sharded (multi-GPU) host logic on CPU.

world_size 2 with the `gloo` backend; the per-shard work runs through a CPU
executor built on the oracle (test infrastructure standing in for the GPU; the
product path is paper_2201_06604_b200.sharding.DeviceExecutor).  Asserts the
reference's invariance property (tests/test_grid.py:91-103,
test_fisher.py:166-178) across ranks: results identical to one device.
"""

import os
import pickle
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_2201_06604_b200 as sf
from paper_2201_06604_b200 import sharding
from paper_2201_06604_b200.grid import MatrixBuffer

import oracle_api as oa
from oracle import oracle as orc


# ------------------------------------------------------------------ unit
@pytest.mark.parametrize("n,world,align", [(16384, 2, 1), (16384, 8, 1), (10, 3, 1),
                                           (2048 * 1024, 8, 2048), (7, 8, 1), (512, 3, 4)])
def test_shard_range_partitions(n, world, align):
    seen = []
    for r in range(world):
        lo, hi = sharding.shard_range(n, r, world, align)
        assert lo <= hi
        if r < world - 1:
            assert lo % align == 0 and hi % align == 0
        seen.extend(range(lo, hi))
    assert seen == list(range(n))


def test_fill_shard_alignment():
    # uniform: column pairs (2*g0 ordinals); normal: whole grid rows (g1 ordinals)
    for r in range(4):
        lo, hi = sharding.fill_shard("uniform", 1024, 1024, r, 4)
        assert lo % 2048 == 0 and hi % 2048 == 0
        lo, hi = sharding.fill_shard("normal", 512, 512, r, 4)
        assert lo % 512 == 0 and hi % 512 == 0


# ------------------------------------------------------- oracle executor
class OracleExecutor:
    """CPU stand-in for DeviceExecutor (tests only)."""

    device = torch.device("cpu")

    def states(self, streams):
        streams._pull()
        return torch.from_numpy(streams._current)  # shares memory with the host array

    def commit_states(self, streams):
        pass

    def fisher(self, plan, streams, lo, hi, want_stats):
        cur = streams._current
        stats = np.empty(plan.nitems * plan.reps) if want_stats else None
        cnt = orc.fisher_replicates(cur, plan.row_margins, plan.col_margins, plan.lf,
                                    plan.kernel_threshold, plan.reps, hi, stats, item_lo=lo)
        st = torch.from_numpy(stats[lo * plan.reps:hi * plan.reps].copy()) if want_stats else None
        return torch.tensor([cnt], dtype=torch.int64), st

    def fill(self, shard, streams, rate, dtype):
        """The rank's compact shard, cut from a full oracle fill through the
        shard's own index map (an independent check of the sub-grid claim)."""
        cur = streams._current
        work = cur.copy()
        full = oa.fill(shard.kind, work, (shard.nrow, shard.ncol), (shard.g0, shard.g1),
                       rate=rate, out_dtype=dtype)
        idx = shard.global_index()
        if shard.kind == "normal":
            piece = full[idx, :][:, : shard.sub_ncol] if shard.cells else full[:0, :0]
        else:
            piece = full[:, idx][: shard.sub_nrow] if shard.cells else full[:0, :0]
        cur[shard.lo:shard.hi] = work[shard.lo:shard.hi]
        return MatrixBuffer.wrap(torch.from_numpy(np.ascontiguousarray(piece)), dtype)


# -------------------------------------------------------------- workers
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, job, outdir):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        ex = OracleExecutor()
        res = {}
        if job == "fisher":
            table = np.array([[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]])
            st = sf.create_streams(sf.set_base_creator(), 64)[0]
            r = sharding.fisher_sim_sharded(table, 5000, st, sf.WorkGrid(8, 8),
                                            return_stats=True, executor=ex)
            res = dict(counts=r.counts, sim_num=r.sim_num, p=r.p_value, stats=r.statistics,
                       states=st.current.copy())
        else:
            kind, shape, g = job
            st = sf.create_streams(sf.set_base_creator(), g[0] * g[1])[0]
            buf = sharding.run_grid_sharded(st, sf.WorkGrid(*g), shape[0], shape[1], kind,
                                            executor=ex, gather=True)
            st2 = sf.create_streams(sf.set_base_creator(), g[0] * g[1])[0]
            part = sharding.run_grid_sharded(st2, sf.WorkGrid(*g), shape[0], shape[1], kind,
                                             executor=ex)
            res = dict(data=buf.data.copy(), states=st.current.copy(), shard=buf.shard,
                       part=part.tensor.numpy().copy(), part_shard=part.shard,
                       states2=st2.current.copy())
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as fh:
            pickle.dump(res, fh)
    finally:
        dist.destroy_process_group()


def _run(job, world=2):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), job, d), nprocs=world, join=True)
        out = []
        for r in range(world):
            with open(os.path.join(d, f"r{r}.pkl"), "rb") as fh:
                out.append(pickle.load(fh))
    return out


def test_fisher_sharded_equals_single_device():
    out = _run("fisher")
    table = np.array([[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]])
    ref_st = oa.fresh_states(64)
    ref = oa.fisher(table, 5000, ref_st, (8, 8), return_stats=True)
    for r in out:
        assert r["counts"] == ref["counts"]
        assert r["sim_num"] == ref["sim_num"]
        assert r["p"] == ref["p_value"]
        assert np.array_equal(r["stats"], ref["statistics"])
        assert np.array_equal(r["states"], ref_st)


@pytest.mark.parametrize("job", [("uniform", (40, 48), (4, 6)),
                                 ("uniform-integer", (33, 20), (3, 4)),
                                 ("normal", (37, 45), (6, 4))])
def test_fill_sharded_equals_single_device(job):
    kind, shape, g = job
    out = _run(job)
    ref_st = oa.fresh_states(g[0] * g[1])
    ref = oa.fill(kind, ref_st, shape, g)
    assert out[0]["shard"] != out[1]["shard"]
    cells = 0
    for r in out:
        assert np.array_equal(r["data"], ref)
        assert np.array_equal(r["states"], ref_st)
        assert np.array_equal(r["states2"], ref_st)
        # the compact shard: exactly the rank's cells, nothing else allocated
        sh = r["part_shard"]
        idx = sh.global_index()
        assert r["part"].shape == (sh.sub_nrow, sh.sub_ncol)
        if sh.cells:  # a rank whose block owns no cell holds an empty shard
            want = ref[idx, :] if kind == "normal" else ref[:, idx]
            assert np.array_equal(r["part"], want)
        cells += r["part"].size
    assert cells == shape[0] * shape[1]


@pytest.mark.parametrize("kind", ["uniform", "normal"])
def test_fill_shard_layout_tiles_the_matrix(kind):
    """Every (shape, grid, world): the compact shards' index maps partition
    the sharded axis, and each shard is the sub-grid fill on offset states
    (checked on the oracle: sub-problem == the rank's cells of the whole)."""
    rng = np.random.default_rng(3)
    for _ in range(40):
        g0, g1 = int(rng.integers(1, 7)), 2 * int(rng.integers(1, 5))
        nrow, ncol = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        world = int(rng.integers(1, 5))
        ref_st = oa.fresh_states(g0 * g1)
        ref = oa.fill(kind, ref_st.copy(), (nrow, ncol), (g0, g1))
        seen = []
        for r in range(world):
            sh = sharding.fill_shard_layout(kind, nrow, ncol, g0, g1, r, world)
            seen.extend(sh.global_index().tolist() if sh.cells else [])
            if not sh.cells:
                continue
            st = oa.fresh_states(g0 * g1)[sh.lo:].copy()
            sub = oa.fill(kind, st, (sh.sub_nrow, sh.sub_ncol), (sh.sub_g0, sh.sub_g1))
            idx = sh.global_index()
            want = ref[idx, :] if kind == "normal" else ref[:, idx]
            assert np.array_equal(sub, want), (g0, g1, nrow, ncol, world, r)
        assert sorted(seen) == list(range(nrow if kind == "normal" else ncol))
