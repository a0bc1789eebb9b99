"""Per-rank kernel time of the C5 uniform fill and the C4-shaped Fisher when
the work is split over N ranks (rank 0's shard timed alone on one GPU): the
strong-scaling efficiency bench.py's N-GPU runs can reach at best."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2201_06604_b200 as sf  # noqa: E402
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher  # noqa: E402
from paper_2201_06604_b200.grid import launch_fill  # noqa: E402
from paper_2201_06604_b200.sharding import fill_shard, shard_range  # noqa: E402


def timeit(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


st = sf.create_streams(sf.set_base_creator(), 1 << 20)[0]
cur = st.device_current()
out = torch.empty((65536, 65536), dtype=torch.float64, device="cuda")
base = None
for world in (1, 2, 4, 8):
    lo, hi = fill_shard("uniform", 1024, 1024, 0, world)
    ms = timeit(lambda: launch_fill("uniform", cur, st.count, out, 65536, 65536, 65536, 1024,
                                    1024, item_lo=lo, item_hi=hi))
    base = base or ms
    print(json.dumps({"w": "uniform_C5", "world": world, "rank0_ms": ms,
                      "efficiency": base / (world * ms)}), flush=True)
del out
torch.cuda.empty_cache()
with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
    t10 = np.array(json.load(fh)["T10"])
grid = sf.WorkGrid(2048, 1024)
st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
plan = plan_fisher(t10, 8 * grid.size, st, grid)
cur = st.device_current()
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
base = None
for world in (1, 2, 4, 8):
    lo, hi = shard_range(grid.size, 0, world)
    ms = timeit(lambda: launch_fisher(plan, cur, st.count, cnt, item_lo=lo, item_hi=hi), reps=3)
    base = base or ms
    print(json.dumps({"w": "fisher_T10_8reps", "world": world, "rank0_ms": ms,
                      "efficiency": base / (world * ms)}), flush=True)

if len(sys.argv) > 1 and sys.argv[1] == "sweep":
    st = sf.create_streams(sf.set_base_creator(), 1 << 20)[0]
    cur = st.device_current()
    out = torch.empty((65536, 65536), dtype=torch.float64, device="cuda")
    for world in (1, 8):
        lo, hi = fill_shard("uniform", 1024, 1024, 0, world)
        for v in (1, 2, 3, 4, 6, 8, 12):
            os.environ["SFB_UNIFORM_VARIANT"] = str(v)
            ms = timeit(lambda: launch_fill("uniform", cur, st.count, out, 65536, 65536, 65536,
                                            1024, 1024, item_lo=lo, item_hi=hi))
            print(json.dumps({"w": "uniform_C5", "world": world, "target_q": v,
                              "rank0_ms": ms}), flush=True)
    os.environ.pop("SFB_UNIFORM_VARIANT")
