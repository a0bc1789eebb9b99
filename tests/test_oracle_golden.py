"""Pin the CPU oracle against the golden fixtures produced by the real
reference (tests/golden/gen_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import PRINTED_STREAM_MATRIX, SIM_1, sha
from oracle import oracle as orc
import oracle_api as oa


def test_printed_matrix(G):
    rows = oa.fresh_states(4)
    m = np.vstack([rows.T, rows.T])
    assert np.array_equal(m, PRINTED_STREAM_MATRIX)
    assert np.array_equal(m, np.array(G["printed_matrix"]))


@pytest.mark.parametrize("e", [0, 1, 10, 134])
def test_jump_matrices(G, e):
    j1, j2 = orc.jump_matrices(e)
    assert j1.tolist() == G[f"jump_{e}"]["j1"]
    assert j2.tolist() == G[f"jump_{e}"]["j2"]


def test_create_chain(G):
    rows, nxt = orc.create_streams((11, 22, 33, 44, 55, 66), 300)
    assert sha(rows) == G["create_toy_300"]["sha"]
    assert list(nxt) == G["create_toy_300"]["next_seed"]
    rows, nxt = orc.create_streams(oa.DEFAULT_SEED, 1 << 14)
    assert sha(rows) == G["create_2p14"]["sha"]
    rows, nxt = orc.create_streams(oa.DEFAULT_SEED, 1 << 20)
    assert sha(rows) == G["create_2p20"]["sha"]
    assert list(nxt) == G["create_2p20"]["next_seed"]


def test_step_sequence(G):
    s = np.array(oa.DEFAULT_SEED, np.int64)
    outs = np.array([orc.step(s) for _ in range(2000)], np.int64)
    assert sha(outs) == G["next_state_2000"]["outs_sha"]
    assert s.tolist() == G["next_state_2000"]["final"]


@pytest.mark.parametrize("n", [0, 1, 2, 7, 1024, 12345])
def test_skip_equals_stepping(n):
    s = np.array([11, 22, 33, 44, 55, 66], np.int64)
    t = orc.skip(s, n)
    for _ in range(n):
        orc.step(s)
    assert np.array_equal(s, t)


def test_sim1(G):
    st = oa.fresh_states(4)
    v = oa.fill("uniform", st, 8, (2, 2)).ravel()
    assert tuple(np.round(v, 3)) == SIM_1
    assert v.tolist() == G["sim_1"]["values"]
    assert st.tolist() == G["sim_1"]["states"]


UNI = ["U1a", "U1b", "U1c", "U1d", "Upad", "Uodd", "Uodd_int", "Uragged",
       "Uvec_odd", "Uwide", "Ubig"]


@pytest.mark.parametrize("name", UNI)
def test_uniform_fixtures(G, A, name):
    g = G[name]
    st = oa.fresh_states(g["n_streams"])
    data = oa.fill(g["kind"], st, g["shape"], tuple(g["grid"]), npad=g["npad"])
    assert sha(data) == g["data_sha"]
    assert sha(st) == g["states_sha"]
    if name + "_data" in A:
        assert np.array_equal(data, A[name + "_data"])


NRM = ["N1", "N64", "N34", "Nodd", "Nodd2", "Nvec", "Nwide"]


@pytest.mark.parametrize("name", NRM)
def test_normal_fixtures_bit_exact(G, name):
    # the oracle calls host libm log/cos/sqrt like numba: bit-exact f64
    g = G[name]
    st = oa.fresh_states(g["n_streams"])
    data = oa.fill("normal", st, g["shape"], tuple(g["grid"]), npad=g["npad"])
    assert sha(data) == g["data_sha"]
    assert sha(data.astype(np.float32)) == g["f32_sha"]
    assert sha(st) == g["states_sha"]
    st = oa.fresh_states(g["n_streams"])
    d32 = oa.fill("normal", st, g["shape"], tuple(g["grid"]), npad=g["npad"],
                  out_dtype=np.float32)
    assert sha(d32) == g["f32_sha"]


@pytest.mark.parametrize("rate", [0.5, 1.0, 2.0])
def test_exponential_fixture(G, rate):
    st = oa.fresh_states(4)
    data = oa.fill("exponential", st, (2, 4), (2, 2), rate=rate)
    assert data.tolist() == G[f"E24_{rate}"]["values"]
    assert st.tolist() == G[f"E24_{rate}"]["states"]


def test_exponential_big(A):
    st = oa.fresh_states(16)
    data = oa.fill("exponential", st, (100, 100), (4, 4), rate=1.5)
    assert np.array_equal(data, A["E100_data"])
    assert np.array_equal(st, A["E100_states"])


def _tables(G, A):
    t = {"T4": np.array(G["T4"]), "T10": np.array(G["T10"]), "month": A["month"],
         "week": A["week"]}
    for k in list(A):
        if k.startswith("tab_"):
            t[k[4:]] = A[k]
    return t


def test_thresholds(G, A):
    tabs = _tables(G, A)
    for name in ("T4", "T10", "month", "week"):
        assert oa.logfact_sum(tabs[name]) == G[f"threshold_{name}"]
        assert oa.relaxed(G[f"threshold_{name}"]) == G[f"relaxed_{name}"]
        assert np.array_equal(oa.lf_table(int(tabs[name].sum())), A[f"lf_{name}"])


FIS = ["F_T4_1e6", "F_T10_1e6", "F_month_1e6", "F_week_1e6", "F_month_2e5",
       "F_month_s", "F_T4_s", "F_T10_s", "F_week_s", "F_2x2_s", "F_E2x2", "F_E2x5",
       "F_E5x2", "F_Ezero_col", "F_Eones", "F_Ebig"]


@pytest.mark.parametrize("key", FIS)
def test_fisher_fixtures(G, A, key):
    g = G[key]
    tabs = _tables(G, A)
    st = oa.fresh_states(g["n_streams"])
    want_stats = key + "_stats" in A
    r = oa.fisher(tabs[g["table"]], g["n"], st, tuple(g["grid"]), return_stats=want_stats)
    assert r["sim_num"] == g["sim_num"]
    assert r["counts"] == g["counts"]
    assert r["p_value"] == g["p_value"]
    assert r["threshold"] == g["threshold"]
    assert sha(st) == g["states_sha"]
    if want_stats:
        assert np.array_equal(r["statistics"], A[key + "_stats"])


def test_fisher_week_1e7_state0(G, A):
    g = G["F_week_1e7"]
    st = oa.fresh_states(g["n_streams"])
    r = oa.fisher(A["week"], g["n"], st, tuple(g["grid"]))
    assert r["counts"] == g["counts"] == 1281
    assert st[0].tolist() == g["state0"]


def test_rcont2(G, A):
    month = A["month"]
    lf = oa.lf_table(int(month.sum()))
    state = np.array([12345] * 6, np.int64)
    tabs = [orc.rcont2_table(month.sum(1), month.sum(0), lf, state) for _ in range(5)]
    assert np.array_equal(np.array(tabs), A["rcont2_month5"])
    assert state.tolist() == G["rcont2_month5_state"]
    state = np.array([12345] * 6, np.int64)
    t = orc.rcont2_table([7], [2, 2, 3], oa.lf_table(7), state)
    assert t.tolist() == G["rcont2_1row"]
    assert state.tolist() == [12345] * 6


T10_ROWS = [20000, 8000, 3000, 1000, 400, 150, 60, 25, 10, 5]
T10_COLS = [13000, 9000, 5000, 2500, 1200, 1000, 600, 250, 75, 25]


def test_t10_table_from_rcont2(G):
    # T10 is rcont2(rows, cols, state=[12345]*6)
    state = np.array([12345] * 6, np.int64)
    t = orc.rcont2_table(T10_ROWS, T10_COLS, oa.lf_table(sum(T10_ROWS)), state)
    assert t.tolist() == G["T10"]


def test_checkpoint_continuation(G):
    # C5 at 1/64 scale: rows [0,4096) then [4096,8192) == one run
    st = oa.fresh_states(1 << 14)
    a = oa.fill("uniform", st, (4096, 8192), (128, 128))
    b = oa.fill("uniform", st, (4096, 8192), (128, 128))
    assert sha(np.vstack([a, b])) == G["C5_64"]["full_sha"]
    assert sha(st) == G["C5_64"]["states_sha"]


def test_thread_invariance():
    ref = None
    for threads in (1, 2, 4, 8):
        st = oa.fresh_states(16)
        d = oa.fill("normal", st, (20, 20), (4, 4), threads=threads)
        st2 = oa.fresh_states(16)
        r = oa.fisher(np.array([[5, 9, 5], [9, 5, 9]]), 2000, st2, (4, 4), True, threads)
        key = (d.tobytes(), st.tobytes(), r["counts"], r["statistics"].tobytes())
        if ref is None:
            ref = key
        assert key == ref
