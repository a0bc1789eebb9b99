"""The multi-GPU path on one B200: world sizes 2 and 4, every rank a separate
process on cuda:0 with the `gloo` backend (NCCL refuses two ranks on one
device), running the PRODUCT executor (sharding.DeviceExecutor -> libsfb.so).
Mirrors the reference's scheduling-invariance tests (tests/test_grid.py:91-103,
tests/test_fisher.py:166-178) with ranks in place of threads: counts,
statistics, matrices and final stream states identical to one device.
"""

import os
import pickle
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T4 = np.array([[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]])
FILL_JOBS = [("uniform", (96, 200), (8, 12)), ("normal", (75, 90), (6, 10)),
             ("exponential", (33, 41), (3, 5))]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        import paper_2201_06604_b200 as sf
        from paper_2201_06604_b200 import sharding

        res = {}
        st = sf.create_streams(sf.set_base_creator(), 512)[0]
        r = sharding.fisher_sim_sharded(T4, 20000, st, sf.WorkGrid(16, 32), return_stats=True)
        res["fisher"] = dict(counts=r.counts, p=r.p_value, stats=r.statistics,
                             states=st.current.copy())
        for kind, shape, g in FILL_JOBS:
            st = sf.create_streams(sf.set_base_creator(), g[0] * g[1])[0]
            buf = sharding.run_grid_sharded(st, sf.WorkGrid(*g), shape[0], shape[1], kind,
                                            gather=True)
            # the compact shard alone (what a rank keeps): its cells only
            st2 = sf.create_streams(sf.set_base_creator(), g[0] * g[1])[0]
            part = sharding.run_grid_sharded(st2, sf.WorkGrid(*g), shape[0], shape[1], kind)
            res[kind] = dict(data=buf.tensor.cpu().numpy().copy(), states=st.current.copy(),
                             shard=buf.shard, part=part.tensor.cpu().numpy().copy(),
                             part_bytes=part.tensor.numel() * part.tensor.element_size(),
                             states2=st2.current.copy())
        # capacity: a C5-layout fill (2^14 streams, 2048 x 8192 f64 = 128 MiB)
        # allocates ~1/world of it per rank
        st = sf.create_streams(sf.set_base_creator(), 1 << 14)[0]
        torch.cuda.synchronize()
        before = torch.cuda.memory_allocated()
        part = sharding.run_grid_sharded(st, sf.WorkGrid(128, 128), 2048, 8192, "uniform",
                                         sync_states=False)
        res["capacity"] = dict(bytes=torch.cuda.memory_allocated() - before,
                               cells=part.shard.cells)
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as fh:
            pickle.dump(res, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_ranks_equal_single_device(world):
    import torch.multiprocessing as mp

    import paper_2201_06604_b200 as sf

    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), d), nprocs=world, join=True,
                           start_method="spawn")
        out = []
        for r in range(world):
            with open(os.path.join(d, f"r{r}.pkl"), "rb") as fh:
                out.append(pickle.load(fh))

    st = sf.create_streams(sf.set_base_creator(), 512)[0]
    ref = sf.fisher_sim(T4, 20000, st, grid=sf.WorkGrid(16, 32), return_stats=True)
    for r in out:
        f = r["fisher"]
        assert f["counts"] == ref.counts and f["p"] == ref.p_value
        assert np.array_equal(f["stats"], ref.statistics)
        assert np.array_equal(f["states"], st.current)
    for kind, shape, g in FILL_JOBS:
        st = sf.create_streams(sf.set_base_creator(), g[0] * g[1])[0]
        req = sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g))
        fill = {"uniform": sf.fill_uniform, "normal": sf.fill_normal,
                "exponential": sf.fill_exponential}[kind]
        want = fill(st, req).data
        shards = {r[kind]["shard"] for r in out}
        assert len(shards) == world, kind  # every rank owned a distinct block
        cells = 0
        for r in out:
            assert np.array_equal(r[kind]["data"][:, :shape[1]], want), kind
            assert np.array_equal(r[kind]["states"], st.current), kind
            assert np.array_equal(r[kind]["states2"], st.current), kind
            sh = r[kind]["shard"]
            idx = sh.global_index()
            assert r[kind]["part"].shape == (sh.sub_nrow, sh.sub_ncol)
            if sh.cells:
                ref = want[idx, :] if kind == "normal" else want[:, idx]
                assert np.array_equal(r[kind]["part"], ref), kind
            cells += sh.cells
        assert cells == shape[0] * shape[1], kind  # the shards tile the matrix
    for r in out:
        cap = r["capacity"]
        assert cap["cells"] * 8 == 2048 * 8192 * 8 // world
        assert cap["bytes"] <= 2048 * 8192 * 8 // world + (2 << 20)  # + allocator rounding
