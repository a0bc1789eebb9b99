"""Small driver for ncu captures: each hot kernel launched a few times at a
size whose working set ncu can save/restore for kernel replay.

    python tools/prof_driver.py [uniform|exponential|normal|fisher4|fisher10|all]
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2201_06604_b200 as sf  # noqa: E402
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher  # noqa: E402
from paper_2201_06604_b200.grid import launch_fill  # noqa: E402

T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]


def t10():
    import json

    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
        return np.array(json.load(fh)["T10"])


def uniform(reps=3, kind="uniform"):
    # C5 rows [0, 4096): 4096 x 65536 f64 = 2.1 GB, grid (1024, 1024), 2^20 streams
    st = sf.create_streams(sf.set_base_creator(), 1 << 20)[0]
    cur = st.device_current()
    out = torch.empty((4096, 65536), dtype=torch.float64, device="cuda")
    for _ in range(reps):
        launch_fill(kind, cur, st.count, out, 4096, 65536, 65536, 1024, 1024)
    torch.cuda.synchronize()


def normal(reps=3, rows=31250 // 4):
    st = sf.create_streams(sf.set_base_creator(), 1 << 18)[0]
    cur = st.device_current()
    out = torch.empty((rows, 32000), dtype=torch.float32, device="cuda")
    for _ in range(reps):
        launch_fill("normal", cur, st.count, out, rows, 32000, 32000, 512, 512)
    torch.cuda.synchronize()


def fisher(table, n, g, reps=3):
    grid = sf.WorkGrid(*g)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    plan = plan_fisher(np.asarray(table), n, st, grid)
    cur = st.device_current()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(reps):
        launch_fisher(plan, cur, st.count, cnt)
    torch.cuda.synchronize()


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("uniform", "all"):
        uniform()
    if what in ("exponential", "all"):
        uniform(kind="exponential")
    if what in ("normal", "all"):
        normal()
    if what in ("fisher4", "all"):
        fisher(T4, 10 ** 6, (256, 64))
    if what in ("fisher10", "all"):
        fisher(t10(), 1 << 22, (2048, 1024))


if __name__ == "__main__":
    main()
