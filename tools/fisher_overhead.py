"""Diagnose per-call overhead of the Fisher launch (T4, 1e6 tables)."""

import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2201_06604_b200 as sf  # noqa: E402
from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher  # noqa: E402

T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]


def main():
    grid = sf.WorkGrid(256, 64)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    plan = plan_fisher(np.asarray(T4), 10 ** 6, st, grid)
    cur = st.device_current()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        launch_fisher(plan, cur, st.count, cnt)
    torch.cuda.synchronize()
    # (a) back to back
    s.record()
    for _ in range(10):
        launch_fisher(plan, cur, st.count, cnt)
    e.record()
    e.synchronize()
    print("back-to-back ms/launch", s.elapsed_time(e) / 10)
    # (b) one at a time, synced, with and without flush
    for flush in (False, True):
        ts = []
        for _ in range(10):
            if flush:
                scratch.zero_()
            s.record()
            t0 = time.perf_counter()
            launch_fisher(plan, cur, st.count, cnt)
            t1 = time.perf_counter()
            e.record()
            e.synchronize()
            ts.append((s.elapsed_time(e), (t1 - t0) * 1e3))
        print("flush" if flush else "noflush", "event ms / host launch ms:",
              [f"{a:.3f}/{b:.3f}" for a, b in ts])


if __name__ == "__main__":
    main()


def e2e_breakdown(reps=20):
    """Where the fisher_sim end-to-end time goes (host-authoritative states)."""
    from paper_2201_06604_b200 import _lib

    grid = sf.WorkGrid(256, 64)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    sf.fisher_sim(T4, 10 ** 6, st, grid=grid)
    acc = {}

    def tick(k, t0):
        acc[k] = acc.get(k, 0.0) + time.perf_counter() - t0
        return time.perf_counter()

    for _ in range(reps):
        t = time.perf_counter()
        _ = st.current
        t = tick("pull states (D2H 786 KB)", t)
        plan = plan_fisher(np.asarray(T4), 10 ** 6, st, grid)
        t = tick("plan_fisher (host prep)", t)
        _lib.require_device()
        cur = st.device_current()
        t = tick("push states (H2D 786 KB)", t)
        cnt = torch.zeros(1, dtype=torch.int64, device=cur.device)
        t = tick("count alloc+zero", t)
        launch_fisher(plan, cur, st.count, cnt)
        t = tick("launch (C ABI)", t)
        st._mark_device_ahead()
        int(cnt.item())
        t = tick("kernel + count.item()", t)
    for k, v in acc.items():
        print(f"{k:32s} {1e3 * v / reps:8.3f} ms")


if __name__ == "__main__":
    e2e_breakdown()


def e2e_loop(reps=200):
    """Mean wall time of the bench's Fisher e2e step (host-authoritative states)."""
    grid = sf.WorkGrid(256, 64)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    for _ in range(5):
        _ = st.current
        sf.fisher_sim(T4, 10 ** 6, st, grid=grid)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        _ = st.current
        sf.fisher_sim(T4, 10 ** 6, st, grid=grid)
    ms = (time.perf_counter() - t0) * 1e3 / reps
    print(f"e2e step {ms:.3f} ms = {1015808 / ms * 1e3:.3e} tables/s")
    t0 = time.perf_counter()
    for _ in range(reps):
        plan_fisher(T4, 10 ** 6, st, grid)
    print(f"plan_fisher {1e3 * (time.perf_counter() - t0) / reps:.4f} ms")
