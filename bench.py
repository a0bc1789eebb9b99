"""Benchmark of the B200 hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

Primary line (BASELINE.json metric "MRG31k3p uniforms/s (HBM GB/s)"): the C5
workload -- 2^20 MRG31k3p streams x 4096 float64 uniforms each, a 65536 x 65536
matrix on WorkGrid(1024, 1024) (34.4 GB per step, far larger than the 126 MB
L2), sharded over ranks by contiguous stream-ordinal blocks (strong scaling:
the total is fixed).  `value` is uniforms/s over all ranks with states and
output resident in HBM; `e2e` is the same metric through the public API with
host stream states uploaded and the matrix downloaded into pinned host memory
every step.  The line also carries the other BASELINE workloads under
"workloads": configs[1] rnormGpu (1e9 float32 normals, 2^18 streams) and the
fisher.sim tables/s for C3 (T4, 1e6 tables) and C4 (T10 sparse 10x10).

`--impl reference` times the reference's CPU path (the oracle port of
_kernels.py, OpenMP over all host cores; the reference is pure Python + numba,
so there is nothing to compile into oracle/_ref) on a bounded sample of the
same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MRG31k3p uniforms/s (HBM GB/s); fisher.sim tables/s at 1/2/4/8 B200"

# C5 (BASELINE configs[4]): 2^20 streams x 4096 uniforms, grid (1024, 1024)
C5 = dict(n_streams=1 << 20, nrow=65536, ncol=65536, g0=1024, g1=1024)
# configs[1]: 1e9 float32 normals from 2^18 streams, grid (512, 512)
C2 = dict(n_streams=1 << 18, nrow=31250, ncol=32000, g0=512, g1=512)
T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]
T10_ROWS = [20000, 8000, 3000, 1000, 400, 150, 60, 25, 10, 5]
T10_COLS = [13000, 9000, 5000, 2500, 1200, 1000, 600, 250, 75, 25]
# FP64 ops per table at source level: F + 23E + 7S + IJ
FOPS = {"T4": 374.0, "T10": 5955.0}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons sampled (NVML, every 2 ms) during the timed
    region -- the same counters `nvidia-smi --query-gpu=clocks.sm,
    clocks_event_reasons.*` reads; a background thread so even a ~50 ms
    region gets many samples."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.sm, self.mx, self.bits = [], [], 0
        self._stop = None

    def _run(self):
        import pynvml as nv

        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.mx.append(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.bits |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            self._stop.wait(0.002)

    def __enter__(self):
        import threading

        try:
            import pynvml as nv

            nv.nvmlInit()
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
            t0 = time.time()
            while not self.sm and time.time() - t0 < 2:
                time.sleep(0.001)  # first sample before the timed region starts
        except Exception:
            self._stop = None
        return self

    def __exit__(self, *a):
        if self._stop is not None:
            self._stop.set()
            self._t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(k for k, b in self.REASONS.items() if self.bits & b),
                "samples": len(self.sm), "source": "NVML (2 ms)"}


def shard(n, rank, world, align=1):
    """contiguous block [lo, hi) of n units for `rank` (paper_2201_06604_b200.sharding)"""
    from paper_2201_06604_b200.sharding import shard_range

    return shard_range(n, rank, world, align)


class Timer:
    """CUDA events on the launching (current) stream."""

    def __init__(self, torch):
        self.torch = torch
        self.s = torch.cuda.Event(enable_timing=True)
        self.e = torch.cuda.Event(enable_timing=True)

    def start(self):
        self.s.record()

    def stop(self):
        self.e.record()
        # poll instead of a blocking synchronize: the sleeps release the GIL so
        # the NVML clock sampler keeps sampling during the timed region
        while not self.e.query():
            time.sleep(0.0002)
        self.e.synchronize()
        return self.s.elapsed_time(self.e)  # ms


def barrier(torch, world):
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()


def max_over_ranks(torch, world, v):
    if world == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def flush_l2(torch, scratch):
    scratch.zero_()


# ------------------------------------------------------------------ workloads
def run_uniform(torch, sf, rank, world, steps, warmup, cfg, kind="uniform"):
    """C5: one fill of the full matrix per step, items sharded by grid columns;
    each rank fills its compact shard (sharding.fill_shard_layout: ~1/N of
    the matrix, the sub-grid fill on its offset stream block)."""
    from paper_2201_06604_b200.grid import launch_fill
    from paper_2201_06604_b200.sharding import fill_shard_layout

    g0, g1 = cfg["g0"], cfg["g1"]
    st = sf.create_streams(sf.set_base_creator(), cfg["n_streams"])[0]
    sh = fill_shard_layout(kind, cfg["nrow"], cfg["ncol"], g0, g1, rank, world)
    lo, hi = sh.lo, sh.hi
    cur = st.device_current()[lo:]
    dt = torch.int64 if kind == "uniform-integer" else torch.float64
    out = torch.empty((sh.sub_nrow, sh.sub_ncol), dtype=dt, device="cuda")
    tm = Timer(torch)

    def step():
        launch_fill(kind, cur, st.count - lo, out, sh.sub_nrow, sh.sub_ncol, sh.sub_ncol,
                    sh.sub_g0, sh.sub_g1)

    for _ in range(warmup):
        step()
    barrier(torch, world)
    with ClockSampler(torch.cuda.current_device()) as clk:
        tm.start()
        for _ in range(steps):
            step()
        ms = tm.stop()
        barrier(torch, world)
    ms = max_over_ranks(torch, world, ms)
    values = cfg["nrow"] * cfg["ncol"]
    per_launch_ms = ms / steps
    # algorithmic bytes of this rank's launch: its output cells + state r/w
    alg_bytes = sh.cells * 8 + (hi - lo) * 48 * 2
    return dict(ms_per_step=ms / steps, value=values * steps / (ms / 1e3),
                launch_ms=per_launch_ms, alg_bytes=alg_bytes, clocks=clk.summary(),
                launches=steps, shard=[lo, hi])


def run_uniform_e2e(torch, sf, rank, world, steps, cfg):
    """Public API with host buffers, every step: host states uploaded, the fill,
    the result downloaded into pinned host memory.  N = 1: fill_uniform and the
    whole matrix.  N > 1: run_grid_sharded (the multi-GPU API: each rank fills
    its stream block, states all-gathered) and each rank downloads its own
    cells (MatrixBuffer.download_shard) -- the output stays sharded."""
    g = sf.WorkGrid(cfg["g0"], cfg["g1"])
    st = sf.create_streams(sf.set_base_creator(), cfg["n_streams"])[0]
    values = cfg["nrow"] * cfg["ncol"]
    if world == 1:
        req = sf.FillRequest(shape=(cfg["nrow"], cfg["ncol"]), grid=g)
        host = torch.empty((cfg["nrow"], cfg["ncol"]), dtype=torch.float64, pin_memory=True)

        def step():
            _ = st.current  # host-authoritative states: the next call uploads them
            buf = sf.fill_uniform(st, req)
            buf.download(host)
    else:
        from paper_2201_06604_b200.sharding import fill_shard_layout, run_grid_sharded

        sh = fill_shard_layout("uniform", cfg["nrow"], cfg["ncol"], cfg["g0"], cfg["g1"], rank,
                               world)
        host = torch.empty((sh.sub_nrow, sh.sub_ncol), dtype=torch.float64, pin_memory=True)

        def step():
            _ = st.current
            buf = run_grid_sharded(st, g, cfg["nrow"], cfg["ncol"], "uniform")
            buf.download(host)  # the rank's compact shard: its cells only
    tm = Timer(torch)
    step()  # warm-up
    torch.cuda.synchronize()
    barrier(torch, world)
    t0 = time.perf_counter()
    tm.start()
    for _ in range(steps):
        step()
    ms = tm.stop()
    barrier(torch, world)
    ms = max_over_ranks(torch, world, ms)
    wall = time.perf_counter() - t0
    return dict(value=values * steps / (ms / 1e3), unit="uniforms/s",
                h2d_bytes_per_step=cfg["n_streams"] * 48 * world,
                d2h_bytes_per_step=values * 8,
                wall_s=wall, steps=steps)


def run_normal(torch, sf, rank, world, steps, warmup, cfg, dtype):
    from paper_2201_06604_b200.grid import launch_fill
    from paper_2201_06604_b200.sharding import fill_shard_layout

    g0, g1 = cfg["g0"], cfg["g1"]
    st = sf.create_streams(sf.set_base_creator(), cfg["n_streams"])[0]
    sh = fill_shard_layout("normal", cfg["nrow"], cfg["ncol"], g0, g1, rank, world)
    cur = st.device_current()[sh.lo:]
    out = torch.empty((sh.sub_nrow, sh.sub_ncol), dtype=dtype, device="cuda")
    tm = Timer(torch)

    def step():
        launch_fill("normal", cur, st.count - sh.lo, out, sh.sub_nrow, sh.sub_ncol,
                    sh.sub_ncol, sh.sub_g0, sh.sub_g1)

    for _ in range(warmup):
        step()
    barrier(torch, world)
    tm.start()
    for _ in range(steps):
        step()
    ms = tm.stop()
    barrier(torch, world)
    ms = max_over_ranks(torch, world, ms)
    values = cfg["nrow"] * cfg["ncol"]
    es = 4 if dtype == torch.float32 else 8
    return dict(ms_per_step=ms / steps, value=values * steps / (ms / 1e3),
                unit="normals/s", gbs=values * es * steps / (ms / 1e3) / 1e9, launches=steps)


FISHER_WARM_S = 2.0  # steady-state warm-up of the Fisher workloads (seconds)
FISHER_WARM_MAX_S = 120.0  # ... waiting at most this long for background memo builds

def run_fisher(torch, sf, rank, world, steps, warmup, table, n, g, scratch):
    """One fisher_sim per step over this rank's item block + NCCL all-reduce."""
    from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher

    grid = sf.WorkGrid(*g)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    plan = plan_fisher(np.asarray(table), n, st, grid)
    lo, hi = shard(grid.size, rank, world)
    cur = st.device_current()
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    tm = Timer(torch)
    counts = []

    def step():
        launch_fisher(plan, cur, st.count, count, item_lo=lo, item_hi=hi)
        if world > 1:
            torch.distributed.all_reduce(count)

    for _ in range(warmup):
        step()
    # then steady state: repeated calls on one table get the larger memo sets,
    # built on host threads from the second call on (fisher.cu get_memo); keep
    # stepping for FISHER_WARM_S and until no build is pending, so the final
    # set has landed (and been uploaded) before the timed steps
    from paper_2201_06604_b200 import _lib

    t0 = time.perf_counter()
    while True:
        step()
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if el >= FISHER_WARM_MAX_S or (el >= FISHER_WARM_S and
                                       _lib.lib().sfb_fisher_memo_pending() == 0):
            break
    step()  # the first call on a newly installed set uploads it
    torch.cuda.synchronize()
    barrier(torch, world)
    total_ms = 0.0
    for _ in range(steps):
        flush_l2(torch, scratch)
        tm.start()
        step()
        total_ms += tm.stop()
        counts.append(int(count.item()))
    barrier(torch, world)
    ms = max_over_ranks(torch, world, total_ms)
    return dict(ms_per_step=ms / steps, value=plan.sim_num * steps / (ms / 1e3),
                unit="tables/s", sim_num=plan.sim_num, counts_last=counts[-1],
                launches=steps)


def run_fisher_e2e(torch, sf, steps, table, n, g):
    grid = sf.WorkGrid(*g)
    st = sf.create_streams(sf.set_base_creator(), grid.size)[0]
    r = sf.fisher_sim(table, n, st, grid=grid)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        _ = st.current  # states live on the host between calls
        r = sf.fisher_sim(table, n, st, grid=grid)
    wall = time.perf_counter() - t0
    return dict(value=r.sim_num * steps / wall, unit="tables/s",
                h2d_bytes_per_step=grid.size * 48 + 8 * (sum(map(sum, table)) + 1),
                d2h_bytes_per_step=8 + grid.size * 48)


# --------------------------------------------------------------- CPU baselines
def stream_io(api, n=1 << 20):
    """configs[4] host side: create 2^20 streams, checkpoint them to a stream
    file (atomic rewrite) and load them back -- the save/restore of the C5
    checkpoint (core.py:222-305).  `api` is this package or the reference."""
    import tempfile

    d = "/dev/shm" if os.path.isdir("/dev/shm") else None
    with tempfile.TemporaryDirectory(dir=d) as tmp:
        path = os.path.join(tmp, "streams.txt")
        t0 = time.perf_counter()
        streams, _ = api.create_streams(api.set_base_creator(), n)
        t1 = time.perf_counter()
        save = getattr(api, "save_streams_atomic", None)
        if save is None:  # the reference keeps it in streamforge.core
            import importlib

            save = importlib.import_module(api.__name__ + ".core").save_streams_atomic
        save(streams, path)
        t2 = time.perf_counter()
        back = api.load_streams(path)
        t3 = time.perf_counter()
        size = os.path.getsize(path)
    assert np.array_equal(back.current, streams.current)
    return {"streams": n, "create_s": t1 - t0, "save_s": t2 - t1, "load_s": t3 - t2,
            "file_bytes": size, "dir": d or "tmp"}


GRF_BATCH = [(1.0, 8.0, 1.0, 1.0, 0.0), (1.5, 12.0, 2.0, 2.0, 0.5), (0.5, 6.0, 1.5, 1.0, 0.0),
             (2.0, 10.0, 1.0, 1.5, 1.0)]


def time_chol(torch, sf):
    """Device time (ms, best of 3, CUDA events) of one sfb_chol_batch call on
    the GRF acceptance batch (4 x 5130^2)."""
    try:
        cov = sf.matern_cov([sf.MaternParams(*p) for p in GRF_BATCH], sf.GridSpec(90, 57, 1.0))
        sf.chol_batch(cov)  # warm-up
        best = None
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            sf.chol_batch(cov)
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e)
            best = ms if best is None else min(best, ms)
        return best
    except Exception:  # noqa: BLE001
        return None


def run_grf(api, steps):
    """simulate_grf on the reference's acceptance-11 batch
    (four Matern parameter sets on a 90 x 57 grid -> four 5130 x 5130
    covariance blocks, LDL^T, 2 realisations), through `api` (this package or
    the reference).  Seconds per call, best of `steps`."""
    best = None
    for _ in range(steps):
        st = api.create_streams(api.set_base_creator(), 64)[0]
        t0 = time.perf_counter()
        f = api.simulate_grf([api.MaternParams(*p) for p in GRF_BATCH], api.GridSpec(90, 57, 1.0),
                             2, st, api.WorkGrid(8, 8))
        dt = time.perf_counter() - t0
        assert f.shape == (4, 2, 57, 90)
        best = dt if best is None else min(best, dt)
    return best


def cpu_uniform_sample(orc, rows, threads=0):
    """C5 rows [0, rows) -- every item, rows/g0 owned rows each -- on the oracle."""
    c = C5
    states, _ = orc.create_streams((12345,) * 6, c["n_streams"])
    out = np.empty((rows, c["ncol"]), np.float64)
    t0 = time.perf_counter()
    orc.fill_real(states, out.ravel(), rows, c["ncol"], c["ncol"], c["g0"], c["g1"], 0, 1.0,
                  threads)
    dt = time.perf_counter() - t0
    return rows * c["ncol"] / dt, dt


def cpu_baseline(reps=3, rows=2048):
    """The reference's CPU path on a bounded C5 sample: the unmodified numba
    reference from baseline/_ref when installed, else the oracle C port."""
    from oracle import oracle as orc

    orc.lib()
    n = rows * C5["ncol"]
    sampler = numba_fill_sampler(rows)
    if sampler is not None:
        best = n / min(sampler() for _ in range(reps))
        return {"value": best, "unit": "uniforms/s",
                "cores": int(os.environ.get("NUMBA_NUM_THREADS", os.cpu_count())),
                "kind": "reference",
                "sample": f"C5 rows [0,{rows}) = {n} float64 uniforms from all 2^20 streams "
                          f"(unmodified streamforge numba _kernels.fill_real, baseline/_ref), "
                          f"best of {reps}"}
    cpu_uniform_sample(orc, 64)  # warm
    best = max(cpu_uniform_sample(orc, rows)[0] for _ in range(reps))
    return {"value": best, "unit": "uniforms/s", "cores": orc.max_threads(), "kind": "port",
            "sample": f"C5 rows [0,{rows}) = {n} float64 uniforms from all "
                      f"2^20 streams (oracle C port of _kernels.fill_real, OpenMP), best of {reps}"}


def cpu_fisher(table, n_items, reps, g=(256, 64)):
    from oracle import oracle as orc
    from scipy.special import gammaln

    t = np.asarray(table)
    lf = gammaln(np.arange(t.sum() + 1, dtype=np.float64) + 1.0)
    thr = float(-gammaln(t + 1.0).sum())
    states, _ = orc.create_streams((12345,) * 6, g[0] * g[1])
    t0 = time.perf_counter()
    orc.fisher_replicates(states, t.sum(1), t.sum(0), lf, thr + 1e-7 * abs(thr), reps, n_items)
    dt = time.perf_counter() - t0
    return n_items * reps / dt


def c5_sample_rows(steps, warmup):
    """the reference's generation timed at full size
    when 34 GB of RAM is free (65536 rows), else at 1/16 (rows [0, 4096)).
    Full size also needs the run to stay within a few minutes (~10 s per full
    step on 16 cores): at most 24 steps + warm-ups."""
    import psutil

    free = psutil.virtual_memory().available
    need = C5["nrow"] * C5["ncol"] * 8 + (4 << 30)  # output + states / headroom
    full = free >= need and steps + warmup <= 24
    return (C5["nrow"] if full else C5["nrow"] // 16), free


def reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle import oracle as orc

    orc.lib()
    rows, free = c5_sample_rows(args.steps, args.warmup)
    frac = rows / C5["nrow"]
    n = rows * C5["ncol"]
    numba_fill = numba_fill_sampler(rows)
    kind = "reference" if numba_fill else "port"
    sample = numba_fill or (lambda: cpu_uniform_sample(orc, rows)[1])
    for _ in range(args.warmup):
        sample()
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(sample())
    total = time.perf_counter() - t0
    v = n * args.steps / sum(vals)
    if rows == C5["nrow"]:
        config = {"workload": "C5 runifGpu: 2^20 MRG31k3p streams x 4096 float64 uniforms "
                              "(65536x65536 on WorkGrid(1024,1024)), one fill per step",
                  "streams": C5["n_streams"], "uniforms_per_step": n}
    else:
        config = {"workload": f"C5 runifGpu at 1/16 (BASELINE.md 3: less than 34 GB of RAM "
                              f"free): rows [0,{rows}) of the 65536x65536 matrix on "
                              "WorkGrid(1024,1024), every stream",
                  "streams": C5["n_streams"], "uniforms_per_step": n}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "uniforms/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config,
            "sample_fraction": frac, "host_ram_free_gb": free / 1e9,
            "best_of_steps": n / min(vals),
            "cpu_baseline": {"value": v, "unit": "uniforms/s",
                             "cores": int(os.environ.get("NUMBA_NUM_THREADS", os.cpu_count()))
                             if kind == "reference" else orc.max_threads(),
                             "kind": kind,
                             "sample": f"{n} uniforms per step (rows [0,{rows}) of C5, "
                                       f"fraction {frac:g}; {free / 1e9:.0f} GB RAM free), "
                                       + ("the unmodified reference's numba _kernels.fill_real "
                                          "from baseline/_ref" if kind == "reference" else
                                          "oracle C port of _kernels.fill_real (OpenMP)")
                                       + ", all host cores, mean over the timed steps"},
            "e2e": {"value": v, "unit": "uniforms/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    # the unmodified reference's own numbers where it is installed, the
    # oracle port's otherwise (both recorded)
    nr = numba_reference(2048)
    line["numba_reference"] = nr
    try:
        port = {"fisher_T4_tables_per_s": cpu_fisher(T4, 16384, 4),
                "fisher_T10_tables_per_s": cpu_fisher(np.array(_t10()), 16384, 1)}
    except Exception as e:  # noqa: BLE001
        port = {"error": str(e)}
    line["workloads"] = {k: nr.get(k, port.get(k)) for k in
                         ("fisher_T4_tables_per_s", "fisher_T10_tables_per_s")}
    if "fill_normal_per_s" in nr:
        line["workloads"]["rnormGpu_f64_sample_per_s"] = nr["fill_normal_per_s"]
    line["workloads"]["source"] = ("unmodified reference (baseline/_ref numba _kernels)"
                                   if "fisher_T4_tables_per_s" in nr else "oracle port")
    line["oracle_port"] = port
    try:
        if _import_reference() is None:
            raise RuntimeError("baseline/_ref not installed")
        import streamforge as ref_api

        line["workloads"]["stream_io_2p20"] = stream_io(ref_api)
        s_grf = run_grf(ref_api, 1)
        line["workloads"]["grf_4x5130"] = {"value": 1.0 / s_grf, "unit": "GRF batches/s",
                                           "seconds": s_grf}
    except Exception as e:  # noqa: BLE001
        line["workloads"]["stream_io_2p20"] = {"unavailable": f"{type(e).__name__}: {e}"}
    print(json.dumps(line), flush=True)


def _import_reference():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "streamforge")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sfb_numba_cache")
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from streamforge import _kernels as K

        return K
    except Exception:
        return None


def numba_fill_sampler(rows):
    """Callable timing one C5 sample (rows [0, rows), all streams) through the
    reference's own numba kernel (baseline/_ref), or None when the reference
    is not installed."""
    K = _import_reference()
    if K is None:
        return None
    from oracle import oracle as orc

    states, _ = orc.create_streams((12345,) * 6, C5["n_streams"])
    out = np.empty((rows, C5["ncol"]))
    out.fill(0.0)  # first touch outside the timed region (34 GB at full size)
    K.fill_real(states.copy(), out.ravel(), 64, C5["ncol"], C5["ncol"], C5["g0"], C5["g1"],
                0, 1.0)  # JIT warm-up

    def sample():
        cur = states.copy()
        t0 = time.perf_counter()
        K.fill_real(cur, out.ravel(), rows, C5["ncol"], C5["ncol"], C5["g0"], C5["g1"], 0, 1.0)
        return time.perf_counter() - t0

    return sample


def numba_reference(rows):
    """The UNMODIFIED reference (streamforge, numba) from baseline/_ref, timed
    through its own `_kernels` seam on the same bounded samples (informational
    beside the oracle port; NUMBA_NUM_THREADS = all host cores)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "streamforge")):
        return {"unavailable": "baseline/_ref not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sfb_numba_cache")
    os.environ.setdefault("NUMBA_NUM_THREADS", str(os.cpu_count()))
    sys.path.insert(0, ref)
    try:
        from scipy.special import gammaln
        from streamforge import _kernels as K

        from oracle import oracle as orc

        states, _ = orc.create_streams((12345,) * 6, C5["n_streams"])
        out = np.zeros((rows, C5["ncol"]))
        K.fill_real(states.copy(), out.ravel(), 64, C5["ncol"], C5["ncol"], C5["g0"], C5["g1"],
                    0, 1.0)  # JIT warm-up
        best = None
        for _ in range(3):
            cur = states.copy()
            t0 = time.perf_counter()
            K.fill_real(cur, out.ravel(), rows, C5["ncol"], C5["ncol"], C5["g0"], C5["g1"], 0, 1.0)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        res = {"fill_uniform_per_s": rows * C5["ncol"] / best,
               "threads": K.max_threads(), "sample": f"C5 rows [0,{rows}) via _kernels.fill_real"}
        t = np.asarray(T4)
        lf = gammaln(np.arange(t.sum() + 1, dtype=np.float64) + 1.0)
        thr = float(-gammaln(t + 1.0).sum())
        thr += 1e-7 * abs(thr)
        st16, _ = orc.create_streams((12345,) * 6, 16384)
        stats = np.empty(0)
        K.fisher_replicates(st16.copy(), t.sum(1), t.sum(0), lf, thr, 1, 64, stats, False)
        t0 = time.perf_counter()
        K.fisher_replicates(st16.copy(), t.sum(1), t.sum(0), lf, thr, 62, 16384, stats, False)
        res["fisher_T4_tables_per_s"] = 62 * 16384 / (time.perf_counter() - t0)
        t = np.array(_t10())
        lf = gammaln(np.arange(t.sum() + 1, dtype=np.float64) + 1.0)
        thr = float(-gammaln(t + 1.0).sum())
        thr += 1e-7 * abs(thr)
        t0 = time.perf_counter()
        K.fisher_replicates(st16.copy(), t.sum(1), t.sum(0), lf, thr, 32, 16384, stats, False)
        res["fisher_T10_tables_per_s"] = 32 * 16384 / (time.perf_counter() - t0)
        # configs[1] layout (2^18 streams on grid (512,512), 32000 columns),
        # rows [0, 1024): 3.3e7 float64 normals (the reference has no float32)
        st18, _ = orc.create_streams((12345,) * 6, 1 << 18)
        nout = np.zeros((1024, 32000))
        K.fill_normal(st18.copy(), nout.ravel(), 16, 32000, 32000, 512, 512)  # JIT warm-up
        best = None
        for _ in range(3):
            cur = st18.copy()
            t0 = time.perf_counter()
            K.fill_normal(cur, nout.ravel(), 1024, 32000, 32000, 512, 512)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        res["fill_normal_per_s"] = 1024 * 32000 / best
        res["fill_normal_sample"] = ("configs[1] layout rows [0,1024) via _kernels.fill_normal "
                                     "(float64), best of 3")
        return res
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {e}"}


def _t10():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as fh:
        return json.load(fh)["T10"]


def run_probes(torch, _lib):
    """Roofline denominators MEASURED_PEAKS.json lacks: write-only HBM
    bandwidth (sfb_probe_write: 16-byte streaming stores over 16 GiB, best of a
    grid-stride sweep and per-CTA contiguous segments) and the FP64 pipe (sfb_probe_fp64:
    8 independent DFMA chains per thread, 8 CTAs of 256 per SM)."""
    out = {}
    buf = torch.empty(16 << 30, dtype=torch.uint8, device="cuda")
    tm = Timer(torch)
    best = None
    st = _lib.stream_handle()
    per_variant = {}
    for variant in (0, 1, 2):
        vbest = None
        for _ in range(4):
            tm.start()
            _lib.check(_lib.lib().sfb_probe_write(_lib.dptr(buf), buf.numel(), variant, st))
            ms = tm.stop()
            vbest = ms if vbest is None else min(vbest, ms)
        per_variant[variant] = buf.numel() / (vbest / 1e3) / 1e9
        best = vbest if best is None else min(best, vbest)
    out["hbm_write_gbs"] = buf.numel() / (best / 1e3) / 1e9
    out["hbm_write_gbs_by_shape"] = {"grid_stride": per_variant[0],
                                     "cta_segments": per_variant[1],
                                     "cta_segments_256b": per_variant[2]}
    del buf
    d = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, iters = 148 * 8, 4096
    _lib.check(_lib.lib().sfb_probe_fp64(_lib.dptr(d), blocks, iters, st))
    best = None
    for _ in range(3):
        tm.start()
        _lib.check(_lib.lib().sfb_probe_fp64(_lib.dptr(d), blocks, iters, st))
        ms = tm.stop()
        best = ms if best is None else min(best, ms)
    out["fp64_ops_per_s"] = blocks * 256 * iters * 8 / (best / 1e3)  # DFMA/s (1 op each)
    # FP64 tensor cores: 4 warps x 4 CTAs per SM, 16 independent DMMA chains each
    blocks, iters = 148 * 4, 2048
    _lib.check(_lib.lib().sfb_probe_dmma(_lib.dptr(d), blocks, iters, st))
    best = None
    for _ in range(3):
        tm.start()
        _lib.check(_lib.lib().sfb_probe_dmma(_lib.dptr(d), blocks, iters, st))
        ms = tm.stop()
        best = ms if best is None else min(best, ms)
    out["dmma_flops_per_s"] = blocks * 4 * iters * 16 * 512 / (best / 1e3)
    return out


def ncu_pipes(key):
    """Pipe utilisation of a compute-bound kernel from the committed ncu capture
    (profiles/traffic.json, written by tools/summarize_ncu.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)[key]
    except Exception:
        return None


def ncu_traffic(kernel):
    """dram read+write bytes per algorithmic byte from the committed ncu capture
    (profiles/traffic.json, written by tools/summarize_ncu.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)[kernel]
        return t["dram_bytes"] / t["alg_bytes"], t["source"]
    except Exception:
        return None, None


# ---------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--only", default=None, help="primary|normal|fisher (debug)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    import torch

    # SFB_BENCH_SHARE_GPU=1: every rank on cuda:0 with gloo -- a smoke test of
    # the multi-rank path on a one-GPU box (numbers meaningless); default NCCL
    share = os.environ.get("SFB_BENCH_SHARE_GPU") == "1"
    torch.cuda.set_device(0 if share else local)
    if world > 1:
        if share:
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2201_06604_b200 as sf
    from paper_2201_06604_b200 import _lib

    _lib.require_device()
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > L2, for flushes
    peak, peak_kind = peaks()
    probe = run_probes(torch, _lib)

    prim = run_uniform(torch, sf, rank, world, args.steps, args.warmup, C5)
    workloads = {}
    if args.only in (None, "normal"):
        n32 = run_normal(torch, sf, rank, world, args.steps, args.warmup, C2, torch.float32)
        workloads["rnormGpu_f32_1e9"] = {k: n32[k] for k in ("value", "unit", "ms_per_step",
                                                              "gbs")}
        workloads["rnormGpu_f32_1e9"]["config"] = "configs[1]: 1e9 float32 normals, 2^18 " \
                                                  "streams, shape (31250,32000), grid (512,512)"
    if args.only in (None, "fisher"):
        f4 = run_fisher(torch, sf, rank, world, max(3, args.steps // 2), args.warmup, T4,
                        10 ** 6, (256, 64), scratch)
        workloads["fisher_T4_1e6"] = dict(value=f4["value"], unit="tables/s",
                                          ms_per_step=f4["ms_per_step"],
                                          counts=f4["counts_last"], sim_num=f4["sim_num"],
                                          fp64_ops_per_table=FOPS["T4"],
                                          config="configs[2]/C3: T4, 1e6 -> 1015808 tables, "
                                                 "grid (256,64)")
        t10 = np.array(_t10())
        # C4 per-GPU share: 2^21 items on grid (2048,1024); reps bounded for the
        # default run (1e10 tables would take ~a minute per GPU)
        n10 = (1 << 21) * 8 * world
        f10 = run_fisher(torch, sf, rank, world, 3, 1, t10, n10, (2048, 1024), scratch)
        workloads["fisher_T10"] = dict(value=f10["value"], unit="tables/s",
                                       ms_per_step=f10["ms_per_step"], sim_num=f10["sim_num"],
                                       fp64_ops_per_table=FOPS["T10"],
                                       config=f"configs[3]/C4 shape: T10 sparse 10x10 on grid "
                                              f"(2048,1024), {f10['sim_num']} tables per step")
    if args.only is None:
        ex = run_uniform(torch, sf, rank, world, max(3, args.steps // 2), args.warmup, C5,
                         kind="exponential")
        workloads["rexpGpu_C5"] = dict(value=ex["value"], unit="exponentials/s",
                                       ms_per_step=ex["ms_per_step"],
                                       gbs=ex["alg_bytes"] / (ex["launch_ms"] / 1e3) / 1e9,
                                       config="SURVEY 8(f) item 1: fill_exponential (rate 1) on "
                                              "the C5 layout, bit-exact glibc log1p port",
                                       ncu_pipes=ncu_pipes("pipes_exponential"))
    if args.only is None and rank == 0:
        # the API's default use (configs[0]/C1 pattern at GPU scale): a 1 x n
        # vector on the default 64 x 8 grid, i.e. 8 active streams of 512
        from paper_2201_06604_b200.grid import launch_fill

        st = sf.create_streams(sf.set_base_creator(), 512)[0]
        vcur = st.device_current()
        vout = torch.empty((1, 10 ** 8), dtype=torch.float64, device="cuda")
        tm = Timer(torch)
        for _ in range(args.warmup):
            launch_fill("uniform", vcur, st.count, vout, 1, 10 ** 8, 10 ** 8, 64, 8)
        tm.start()
        for _ in range(args.steps):
            launch_fill("uniform", vcur, st.count, vout, 1, 10 ** 8, 10 ** 8, 64, 8)
        vms = tm.stop() / args.steps
        workloads["runifGpu_vector_1e8"] = dict(
            value=1e8 / (vms / 1e3), unit="uniforms/s", ms_per_step=vms,
            gbs=8e8 / (vms / 1e3) / 1e9,
            config="configs[0] pattern at GPU scale: FillRequest(shape=1e8) on the default "
                   "WorkGrid(64,8) -> 8 active streams, generic kernel")
        del vout
        workloads["stream_io_2p20"] = dict(stream_io(sf), config="configs[4] host side: "
                                           "create / save_streams_atomic / load_streams of "
                                           "2^20 streams (C++ creation chain and stream files)")
    if args.only in (None, "fisher") and (world >= 8 or os.environ.get("SFB_BENCH_C4") == "1"):
        # configs[3]/C4 in full: T10, 1e10 tables on grid (2048,1024), 2^21
        # streams, sharded by items + one all-reduce (~2 s per step on 8 B200)
        t10 = np.array(_t10())
        c4 = run_fisher(torch, sf, rank, world, 1, 1, t10, 10 ** 10, (2048, 1024), scratch)
        workloads["fisher_C4_1e10"] = dict(value=c4["value"], unit="tables/s",
                                           ms_per_step=c4["ms_per_step"], sim_num=c4["sim_num"],
                                           counts=c4["counts_last"],
                                           config="configs[3]/C4: T10, 1e10 -> 10001317888 "
                                                  "tables on grid (2048,1024), 2^21 streams")
    if args.only is None and rank == 0:
        run_grf(sf, 1)  # warm-up (scratch buffers, look-ahead streams, kernels)
        s_grf = run_grf(sf, 3)
        workloads["grf_4x5130"] = dict(value=1.0 / s_grf, unit="GRF batches/s",
                                       ms_per_step=1e3 * s_grf,
                                       config="SURVEY 8(f) item 4: simulate_grf, 4 Matern sets "
                                              "on a 90x57 grid (4 x 5130^2 LDL^T), 2 "
                                              "realisations, host fields out (best of 3)")
        chol_ms = time_chol(torch, sf)
        if probe and chol_ms:
            ach = 4 * 5130 ** 3 / 3 / (chol_ms / 1e3)
            workloads["grf_4x5130"]["roofline"] = {
                "bound": "tensor", "kernel": "sfb_chol_batch (chol_update / chol_panel DMMA "
                "tile products, chol_diag chain)", "achieved": ach / 1e12,
                "peak": probe["dmma_flops_per_s"] / 1e12, "unit": "TFLOP/s",
                "frac": ach / probe["dmma_flops_per_s"], "chol_ms": chol_ms,
                "note": "n^3/3 flops per 5130^2 block x 4 over the device time of one "
                        "sfb_chol_batch call (CUDA events, best of 3); peak = sfb_probe_dmma "
                        "(mma.sync.m8n8k4.f64 issue rate; tcgen05 has no FP64 kind)"}
    e2e = run_uniform_e2e(torch, sf, rank, world, min(args.steps, 3), C5)
    if args.only in (None, "fisher") and world == 1:
        fe = run_fisher_e2e(torch, sf, 3, T4, 10 ** 6, (256, 64))
        workloads["fisher_T4_1e6"]["e2e"] = fe

    if rank != 0:
        return
    # per-workload rooflines against the probes measured above
    wpeak = probe["hbm_write_gbs"]
    if "rnormGpu_f32_1e9" in workloads:
        w = workloads["rnormGpu_f32_1e9"]
        w["roofline"] = {"bound": "hbm", "achieved": w["gbs"], "unit": "GB/s",
                         "peak_copy": peak, "frac_copy": w["gbs"] / peak,
                         "peak_write": wpeak, "frac_write": w["gbs"] / wpeak,
                         "note": "compute/issue bound: float32 form box_muller_pair_f32, ~88 SASS (30 FP64, 6 XU) per normal pair incl. 2 MRG31k3p steps"}
    for key, fops, pk in (("fisher_T4_1e6", FOPS["T4"], "pipes_fisher4"),
                          ("fisher_T10", FOPS["T10"], "pipes_fisher10")):
        if key in workloads:
            w = workloads[key]
            ach = w["value"] * fops
            w["roofline"] = {"bound": "fp64", "achieved": ach / 1e12, "unit": "Tops/s",
                             "peak": probe["fp64_ops_per_s"] / 1e12,
                             "frac": ach / probe["fp64_ops_per_s"],
                             "note": "source-level FP64 ops per table (SURVEY 8(d), a division "
                                     "counted as 1 op although it issues ~8 FP64 "
                                     "instructions) vs the measured DFMA issue rate "
                                     "(sfb_probe_fp64)",
                             "ncu_pipes": ncu_pipes(pk)}
    if "rnormGpu_f32_1e9" in workloads:
        workloads["rnormGpu_f32_1e9"]["roofline"]["ncu_pipes"] = ncu_pipes("pipes_normal")
    achieved = prim["alg_bytes"] / (prim["launch_ms"] / 1e3) / 1e9
    tr_ratio, tr_src = ncu_traffic("fill_uniform")
    line = {
        "metric": METRIC, "value": prim["value"], "unit": "uniforms/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": prim["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "C5 runifGpu: 2^20 MRG31k3p streams x 4096 float64 uniforms "
                               "(65536x65536 on WorkGrid(1024,1024)), one fill per step",
                   "streams": C5["n_streams"], "uniforms_per_step": C5["nrow"] * C5["ncol"],
                   "l2": "output 34.4 GB per step >> 126 MB L2 (no flush needed)",
                   "parallelism": f"stream-ordinal blocks x{world}"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": None if tr_ratio is None else tr_ratio * prim["alg_bytes"],
                     "traffic_source": tr_src,
                     "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs, "
                                  "read+write bytes of a device copy); this kernel only "
                                  "writes, and a write-only stream can exceed it slightly -- "
                                  "frac_write against the write-only probe is the tighter bound",
                     "peak_write_measured": wpeak, "frac_write": achieved / wpeak,
                     "kernel": "fill_uniform_quad<0> (256-bit stores)",
                     "algorithmic_bytes_per_launch": prim["alg_bytes"]},
        "probes": probe,
        "clocks": prim["clocks"],
        "gpu_launches": prim["launches"],
        "workloads": workloads,
    }
    if e2e:
        line["e2e"] = {k: e2e[k] for k in ("value", "unit", "h2d_bytes_per_step",
                                           "d2h_bytes_per_step")}
    if not args.no_cpu and world == 1:
        try:
            line["cpu_baseline"] = cpu_baseline()
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
