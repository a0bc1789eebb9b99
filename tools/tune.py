"""Kernel-variant sweep (tuning knobs SFB_NORMAL_VARIANT, SFB_FISHER_WALK/MINB).

    python tools/tune.py [normal] [fisher]

Prints one line per (workload, variant) with the CUDA-event time per launch.
"""

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

T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps


def normal_case(dtype):
    st = sf.create_streams(sf.set_base_creator(), 1 << 18)[0]
    cur = st.device_current()
    out = torch.empty((31250, 32000), dtype=dtype, device="cuda")
    return lambda: launch_fill("normal", cur, st.count, out, 31250, 32000, 32000, 512, 512)


def fisher_case(table, n, g):
    grid = sf.WorkGrid(*g)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    plan = plan_fisher(np.asarray(table), n, st, grid)
    cur = st.device_current()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    cur0 = cur.clone()

    def run():
        cur.copy_(cur0)  # same input states every launch (counts comparable)
        launch_fisher(plan, cur, st.count, cnt)

    return plan.sim_num, run, cnt


def main():
    what = sys.argv[1:] or ["normal", "fisher"]
    res = []
    if "uniform" in what:
        st = sf.create_streams(sf.set_base_creator(), 1 << 20)[0]
        cur = st.device_current()
        out = torch.empty((65536, 65536), dtype=torch.float64, device="cuda")

        def fn():
            launch_fill("uniform", cur, st.count, out, 65536, 65536, 65536, 1024, 1024)

        for v in (0, 0x4000, 0, 0x4000, 0):
            os.environ["SFB_UNIFORM_VARIANT"] = str(v)
            ms = timeit(fn)
            res.append({"w": "uniform_C5", "variant": hex(v), "ms": ms,
                        "gbs": out.numel() * 8 / (ms / 1e3) / 1e9})
            print(json.dumps(res[-1]), flush=True)
        os.environ.pop("SFB_UNIFORM_VARIANT")
        for kind, v in (("exponential", 0), ("exponential", 0x10), ("exponential", 0x30),
                        ("exponential", 0xa0), ("exponential", 0x4000), ("uniform-integer", 0)):
            os.environ["SFB_UNIFORM_VARIANT"] = str(v)
            out2 = out.view(torch.int64) if kind == "uniform-integer" else out

            def fn2(kind=kind, out2=out2):
                launch_fill(kind, cur, st.count, out2, 65536, 65536, 65536, 1024, 1024)

            ms = timeit(fn2)
            res.append({"w": f"{kind}_C5", "variant": hex(v), "ms": ms,
                        "gbs": out.numel() * 8 / (ms / 1e3) / 1e9})
            print(json.dumps(res[-1]), flush=True)
        os.environ.pop("SFB_UNIFORM_VARIANT", None)

        def fn3():
            launch_fill("exponential", cur, st.count, out, 65536, 65536, 65536, 1024, 1024,
                        rate=0.37)

        ms = timeit(fn3)
        res.append({"w": "exponential_rate0.37_C5", "ms": ms,
                    "gbs": out.numel() * 8 / (ms / 1e3) / 1e9})
        print(json.dumps(res[-1]), flush=True)
        del out
        torch.cuda.empty_cache()
    if "vector" in what:  # the API's default use: a 1 x n vector on the default 64 x 8 grid
        st = sf.create_streams(sf.set_base_creator(), 512)[0]
        cur = st.device_current()
        n = 10 ** 8
        for kind, dt in (("uniform", torch.float64), ("normal", torch.float64),
                         ("normal", torch.float32), ("exponential", torch.float64)):
            out = torch.empty((1, n), dtype=dt, device="cuda")

            def fnv(kind=kind, out=out):
                launch_fill(kind, cur, st.count, out, 1, n, n, 64, 8)

            ms = timeit(fnv)
            res.append({"w": f"vector_{kind}_{str(dt)[6:]}", "ms": ms, "per_s": n / (ms / 1e3),
                        "gbs": n * out.element_size() / (ms / 1e3) / 1e9})
            print(json.dumps(res[-1]), flush=True)
    if "normal" in what:
        for dt in (torch.float32, torch.float64):
            fn = normal_case(dt)
            for v in (10, 0, 3, 8, 2, 1, 4):
                os.environ["SFB_NORMAL_VARIANT"] = str(v)
                ms = timeit(fn)
                res.append({"w": f"normal_{str(dt)[6:]}", "variant": v, "ms": ms,
                            "per_s": 1e9 / (ms / 1e3)})
                print(json.dumps(res[-1]), flush=True)
        os.environ.pop("SFB_NORMAL_VARIANT")
    if "fisher" in what:
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
            t10 = np.array(json.load(fh)["T10"])
        month = np.asarray(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))["month"])
        only = os.environ.get("TUNE_FISHER_TABLES", "T4,T4x16,T10").split(",")
        for name, table, n, g in (("T4", T4, 10 ** 6, (256, 64)),
                                  ("T4x16", T4, 16 * 10 ** 6, (2048, 1024)),
                                  ("T10", t10, 1 << 23, (2048, 1024)),
                                  ("month", month, 1 << 22, (2048, 1024)),
                                  ("T4_default_grid", T4, 10 ** 6, (64, 16)),
                                  ("month_default_grid", month, 10 ** 6, (64, 16))):
            if name not in only:
                continue
            sim, fn, cnt = fisher_case(table, n, g)
            variants = [(f"walk{w}_minb{mb}", {"SFB_FISHER_WALK": str(w),
                                               "SFB_FISHER_MINB": str(mb)})
                        for w in (1, 3) for mb in (3, 4)]
            for vname, env in variants:
                os.environ.update(env)
                ms = timeit(fn, reps=3, warm=1)
                fn()
                res.append({"w": f"fisher_{name}", "variant": vname,
                            "ms": ms, "per_s": sim / (ms / 1e3),
                            "count_one_launch": int(cnt.item())})
                print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
