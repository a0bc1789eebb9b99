"""Generate the golden parity fixtures by running the REAL reference.

Usage (in the build container, where /root/reference exists):

    python tests/golden/gen_golden.py

It copies /root/reference/pkg/src/streamforge to a temp dir (numba's
cache=True and hypothesis would otherwise write into the read-only tree),
imports it, runs the reference's own public API on the BASELINE-derived
configurations and writes

    tests/golden/golden.json   scalars, digests, small vectors
    tests/golden/golden.npz    small full arrays (bit patterns)

These fixtures pin the CPU oracle (oracle/) and are the parity anchors for the
GPU tests; nothing at test/bench time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src/streamforge"
REF_DATA = "/root/reference/pkg/tests/data"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def import_reference():
    tmp = tempfile.mkdtemp(prefix="sfref_")
    shutil.copytree(REF_SRC, os.path.join(tmp, "streamforge"))
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "numba_cache"))
    sys.path.insert(0, tmp)
    import streamforge as sf  # noqa: E402

    return sf


T4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]
T10_ROWS = [20000, 8000, 3000, 1000, 400, 150, 60, 25, 10, 5]
T10_COLS = [13000, 9000, 5000, 2500, 1200, 1000, 600, 250, 75, 25]


def main():
    sf = import_reference()
    from streamforge import fisher as sff  # noqa: E402
    from streamforge.grid import run_grid  # noqa: E402

    G = {"meta": {
        "generator": "tests/golden/gen_golden.py",
        "reference": "streamforge 0.1.0 at /root/reference/pkg (pure Python + numba)",
        "python": platform.python_version(),
        "numpy": np.__version__,
        "machine": platform.machine(),
    }}
    import numba
    import scipy

    G["meta"]["numba"] = numba.__version__
    G["meta"]["scipy"] = scipy.__version__
    A = {}

    def fresh(n):
        return sf.create_streams(sf.set_base_creator(), n)[0]

    # ---- streams (core.py) -------------------------------------------------
    s4 = fresh(4)
    G["printed_matrix"] = s4.matrix().tolist()
    for e in (0, 1, 10, 134):
        j1, j2 = sf.core._jump_matrices(e)
        G[f"jump_{e}"] = {"j1": [list(r) for r in j1], "j2": [list(r) for r in j2]}
    st, c = sf.create_streams(sf.set_base_creator((11, 22, 33, 44, 55, 66)), 300)
    G["create_toy_300"] = {"sha": sha(st.current), "next_seed": list(c.next_seed),
                           "last": st.current[-1].tolist()}
    st, c = sf.create_streams(sf.set_base_creator(), 1 << 14)
    G["create_2p14"] = {"sha": sha(st.current), "next_seed": list(c.next_seed)}
    st, c = sf.create_streams(sf.set_base_creator(), 1 << 20)
    G["create_2p20"] = {"sha": sha(st.current), "next_seed": list(c.next_seed),
                        "row_12345": st.current[12345].tolist()}
    # single-step outputs from a few states
    s = sf.StreamState.from_seed(sf.DEFAULT_SEED)
    outs = []
    for _ in range(2000):
        s, z = sf.next_state(s)
        outs.append(z)
    G["next_state_2000"] = {"outs_sha": sha(np.array(outs, np.int64)),
                            "first": outs[:8], "final": list(s.g1 + s.g2)}

    # stream file format
    import io

    buf = io.StringIO()
    sf.save_streams(fresh(3), buf)
    G["save_3"] = buf.getvalue()

    # ---- uniform fills (grid.py, _kernels.fill_real/fill_integer) ----------
    st = fresh(4)
    v = sf.fill_uniform(st, sf.FillRequest(shape=8, grid=sf.WorkGrid(2, 2))).vector()
    G["sim_1"] = {"values": v.tolist(), "states": st.current.tolist()}

    def uni(name, n_streams, shape, grid, kind="uniform", npad=None, keep=False):
        st = fresh(n_streams)
        buf = sf.fill_uniform(st, sf.FillRequest(shape=shape, kind=kind, grid=grid,
                                                 npad=npad))
        d = {"shape": list(shape) if not isinstance(shape, int) else shape,
             "grid": [grid.nglobal0, grid.nglobal1], "n_streams": n_streams,
             "kind": kind, "npad": buf.npad, "data_sha": sha(buf.data),
             "values_sha": sha(buf.values), "states_sha": sha(st.current),
             "first": buf.data.ravel()[:4].tolist()}
        if keep:
            A[name + "_data"] = buf.data.copy()
        if n_streams <= 4096:
            A[name + "_states"] = st.current.copy()
        G[name] = d

    uni("U1a", 512, 10 ** 6, sf.WorkGrid(64, 8))
    uni("U1b", 512, 10 ** 6, sf.WorkGrid(1, 512))
    uni("U1c", 512, (1000, 1000), sf.WorkGrid(64, 8))
    uni("U1d", 512, (1000, 1000), sf.WorkGrid(64, 8), kind="uniform-integer")
    uni("Upad", 4, (3, 3), sf.WorkGrid(2, 2), npad=5, keep=True)
    uni("Uodd", 15, (37, 41), sf.WorkGrid(3, 5), keep=True)
    uni("Uodd_int", 15, (37, 41), sf.WorkGrid(3, 5), kind="uniform-integer", keep=True)
    uni("Uragged", 64, (130, 250), sf.WorkGrid(8, 8), npad=256, keep=True)
    uni("Uvec_odd", 21, 1001, sf.WorkGrid(3, 7), keep=True)
    uni("Uwide", 1024, (64, 4096), sf.WorkGrid(16, 64))
    uni("Ubig", 1 << 14, (8192, 8192), sf.WorkGrid(128, 128))

    # ---- normal fills (_kernels.fill_normal) -------------------------------
    def nrm(name, n_streams, shape, grid, npad=None, keep=False):
        st = fresh(n_streams)
        buf = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=grid, npad=npad))
        d = {"shape": list(shape) if not isinstance(shape, int) else shape,
             "grid": [grid.nglobal0, grid.nglobal1], "n_streams": n_streams,
             "npad": buf.npad, "data_sha": sha(buf.data),
             "f32_sha": sha(buf.data.astype(np.float32)),
             "states_sha": sha(st.current), "first": buf.data.ravel()[:4].tolist()}
        if keep:
            A[name + "_data"] = buf.data.copy()
        if n_streams <= 4096:
            A[name + "_states"] = st.current.copy()
        G[name] = d

    nrm("N1", 1 << 14, (2048, 2048), sf.WorkGrid(128, 128))
    nrm("N64", 16, (64, 64), sf.WorkGrid(4, 4), keep=True)
    nrm("N34", 4, (3, 4), sf.WorkGrid(2, 2), keep=True)
    nrm("Nodd", 2, (2, 3), sf.WorkGrid(1, 2), keep=True)
    nrm("Nodd2", 18, (37, 45), sf.WorkGrid(3, 6), npad=48, keep=True)
    nrm("Nvec", 8, 999, sf.WorkGrid(2, 4), keep=True)
    nrm("Nwide", 4096, (128, 2048), sf.WorkGrid(8, 512))

    # ---- exponential (_kernels.fill_real mode 1) ---------------------------
    for rate in (0.5, 1.0, 2.0):
        st = fresh(4)
        buf = sf.fill_exponential(st, sf.FillRequest(shape=(2, 4), kind="exponential",
                                                     rate=rate, grid=sf.WorkGrid(2, 2)))
        G[f"E24_{rate}"] = {"values": buf.values.tolist(), "states": st.current.tolist()}
    st = fresh(16)
    buf = sf.fill_exponential(st, sf.FillRequest(shape=(100, 100), kind="exponential",
                                                 rate=1.5, grid=sf.WorkGrid(4, 4)))
    A["E100_data"] = buf.data.copy()
    A["E100_states"] = st.current.copy()

    # ---- Fisher (fisher.py, _kernels.fisher_replicates) --------------------
    month = np.loadtxt(os.path.join(REF_DATA, "month.csv"), delimiter=",", dtype=np.int64)
    week = np.loadtxt(os.path.join(REF_DATA, "week.csv"), delimiter=",", dtype=np.int64)
    A["month"] = month
    A["week"] = week
    lf = sff.log_factorial_table(int(sum(T10_ROWS)))
    t10 = sf.rcont2(T10_ROWS, T10_COLS, np.array([12345] * 6, np.int64), lf)
    G["T10"] = t10.tolist()
    G["T4"] = T4
    tables = {"month": month, "week": week, "T4": np.array(T4), "T10": t10}
    for name in ("T4", "T10", "month", "week"):
        t = sff.ContingencyTable(tables[name])
        G[f"threshold_{name}"] = sff.logfact_sum(t)
        G[f"relaxed_{name}"] = sff.relaxed_threshold(sff.logfact_sum(t))
        lfn = sff.log_factorial_table(t.total)
        A[f"lf_{name}"] = lfn

    def fis(key, name, n, grid, n_streams, stats=False):
        st = fresh(n_streams)
        r = sf.fisher_sim(tables[name], n, st, grid=grid, return_stats=stats)
        d = {"table": name, "n": n, "grid": [grid.nglobal0, grid.nglobal1],
             "n_streams": n_streams, "sim_num": r.sim_num, "counts": r.counts,
             "p_value": r.p_value, "threshold": r.threshold,
             "states_sha": sha(st.current), "state0": st.current[0].tolist()}
        if stats:
            A[key + "_stats"] = r.statistics.copy()
            A[key + "_states"] = st.current.copy()
        G[key] = d
        print(key, r.counts, r.sim_num, flush=True)

    g = sf.WorkGrid(256, 64)
    fis("F_T4_1e6", "T4", 10 ** 6, g, 16384)
    fis("F_T10_1e6", "T10", 10 ** 6, g, 16384)
    fis("F_month_1e6", "month", 10 ** 6, g, 16384)
    fis("F_week_1e6", "week", 10 ** 6, g, 16384)
    fis("F_week_1e7", "week", 10 ** 7, g, 16384)
    fis("F_month_2e5", "month", 2 * 10 ** 5, g, 16384)
    fis("F_month_s", "month", 2000, sf.WorkGrid(4, 4), 16, stats=True)
    fis("F_T4_s", "T4", 4096, sf.WorkGrid(8, 8), 64, stats=True)
    fis("F_T10_s", "T10", 256, sf.WorkGrid(4, 8), 32, stats=True)
    fis("F_week_s", "week", 1000, sf.WorkGrid(2, 5), 12, stats=True)
    fis("F_2x2_s", "T4", 10, sf.WorkGrid(1, 1), 1, stats=True)
    # edge tables: 2x2, single-row-ish, zeros
    edge = {
        "E2x2": np.array([[3, 7], [6, 2]]),
        "E2x5": np.array([[0, 1, 0, 2, 5], [3, 0, 0, 1, 0]]),
        "E5x2": np.array([[0, 4], [1, 1], [9, 0], [0, 0], [2, 2]]),
        "Ezero_col": np.array([[3, 0, 2], [1, 0, 5], [2, 0, 2]]),
        "Eones": np.array([[1, 0], [0, 1]]),
        "Ebig": np.array([[500, 20, 3000], [10, 900, 40], [7000, 3, 1]]),
    }
    for name, tb in edge.items():
        tables[name] = tb
        A[f"tab_{name}"] = tb
        fis(f"F_{name}", name, 3000, sf.WorkGrid(4, 4), 16, stats=True)

    # rcont2 single tables (_kernels.rcont2_table)
    t = sff.ContingencyTable(month)
    state = np.array([12345] * 6, np.int64)
    lfm = sff.log_factorial_table(t.total)
    rc = [sf.rcont2(t.row_margins, t.col_margins, state, lfm) for _ in range(5)]
    A["rcont2_month5"] = np.array(rc)
    G["rcont2_month5_state"] = state.tolist()
    state = np.array([12345] * 6, np.int64)
    G["rcont2_1row"] = sf.rcont2([7], [2, 2, 3], state).tolist()
    G["rcont2_1row_state"] = state.tolist()

    # ---- checkpoint / resume (C5 at 1/64 scale) ----------------------------
    grid = sf.WorkGrid(128, 128)
    st = fresh(1 << 14)
    full = run_grid(st, grid, 8192, 8192, "uniform")
    G["C5_64"] = {"full_sha": sha(full.data), "states_sha": sha(st.current)}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **A)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(G, fh, indent=1, sort_keys=True)
    print("wrote", len(G), "json keys,", len(A), "arrays")


if __name__ == "__main__":
    main()
