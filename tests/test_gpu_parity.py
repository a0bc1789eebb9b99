"""GPU parity: the sm_100a kernels (through the package API / C ABI) against
the reference-generated goldens and the CPU oracle.

Bars:
  * uniforms, integers, stream states, Fisher counts / statistics / states:
    bit-exact;
  * Box-Muller float64: |gpu - ref| <= 4 ulp(ref), or <= 2^-60 absolute (the
    four draws z2 = k 2^29 where theta is pi/2-multiple-adjacent);
  * Box-Muller float32: |gpu - float32(ref)| <= 1 ulp_f32 everywhere, and
    identical on >= 99.999 % of cells;
  * exponential: bit-exact (glibc log1p FMA-variant port, log1p_glibc.cuh).
"""

import math
import os

import numpy as np
import pytest

import paper_2201_06604_b200 as sf
from paper_2201_06604_b200 import _lib
from conftest import SIM_1, sha
from oracle import oracle as orc
import oracle_api as oa

pytestmark = pytest.mark.gpu


def fresh(n):
    return sf.create_streams(sf.set_base_creator(), n)[0]


def grid(g):
    return sf.WorkGrid(*g)


def ulp64(x):
    return np.spacing(np.abs(x).astype(np.float64))


def assert_normal_f64_close(got, ref):
    err = np.abs(got - ref)
    tol = np.maximum(4 * ulp64(ref), 2.0 ** -60)
    bad = err > tol
    assert not bad.any(), (got[bad][:5], ref[bad][:5], err.max())


def assert_normal_f32_close(got, ref64):
    ref = ref64.astype(np.float32)
    same = got == ref
    ulp = np.spacing(np.abs(ref))
    assert (np.abs(got.astype(np.float64) - ref.astype(np.float64)) <= ulp).all()
    assert same.mean() >= 0.99999, same.mean()


# ---------------------------------------------------------------- uniforms
def test_sim1_published_vector(G):
    st = fresh(4)
    v = sf.fill_uniform(st, sf.FillRequest(shape=8, grid=sf.WorkGrid(2, 2))).vector()
    assert tuple(np.round(v, 3)) == SIM_1
    assert v.tolist() == G["sim_1"]["values"]
    assert st.current.tolist() == G["sim_1"]["states"]


UNI = ["U1a", "U1b", "U1c", "U1d", "Upad", "Uodd", "Uodd_int", "Uragged", "Uvec_odd",
       "Uwide", "Ubig"]


@pytest.mark.parametrize("name", UNI)
def test_uniform_goldens_bit_exact(G, A, name):
    g = G[name]
    st = fresh(g["n_streams"])
    shape = g["shape"] if isinstance(g["shape"], int) else tuple(g["shape"])
    buf = sf.fill_uniform(st, sf.FillRequest(shape=shape, kind=g["kind"], grid=grid(g["grid"]),
                                             npad=g["npad"] if g["npad"] != (
                                                 shape if isinstance(shape, int)
                                                 else shape[1]) else None))
    assert sha(buf.data) == g["data_sha"]
    assert sha(st.current) == g["states_sha"]
    if name + "_data" in A:
        assert np.array_equal(buf.data, A[name + "_data"])


def test_single_item_grid_matches_sequential_stepping():
    st = fresh(4)
    buf = sf.fill_uniform(st, sf.FillRequest(shape=12, grid=sf.WorkGrid(1, 1)))
    s = sf.create_streams(sf.set_base_creator(), 1)[0][0]
    outs = []
    for _ in range(12):
        s, z = sf.next_state(s)
        outs.append(z)
    assert np.array_equal(buf.vector(), np.array(outs) * sf.NORM)


def test_unused_streams_unchanged_and_padding_zero():
    st = fresh(10)
    before = st.current.copy()
    buf = sf.run_grid(st, sf.WorkGrid(2, 2), 3, 3, "uniform", npad=5)
    assert np.array_equal(buf.data[:, 3:], np.zeros((3, 2)))
    assert (buf.values != 0).all()
    assert np.array_equal(st.current[4:], before[4:])
    assert not np.array_equal(st.current[:4], before[:4])


@pytest.mark.parametrize("shape,g,n", [
    ((1, 1), (1, 1), 1), ((5, 7), (2, 3), 6), ((129, 257), (4, 6), 24),
    ((64, 64), (64, 64), 4096), ((3, 1000), (2, 512), 1024), (100001, (1, 512), 512),
    ((250, 250), (16, 2), 32), ((17, 4096), (3, 64), 192), ((2048, 2048), (32, 32), 1024),
])
@pytest.mark.parametrize("kind", ["uniform", "uniform-integer"])
def test_uniform_layouts_vs_oracle(shape, g, n, kind):
    st = fresh(n)
    buf = sf.fill_uniform(st, sf.FillRequest(shape=shape, kind=kind, grid=sf.WorkGrid(*g)))
    ref_st = oa.fresh_states(n)
    ref = oa.fill(kind, ref_st, shape, g)
    assert np.array_equal(buf.data, ref)
    assert np.array_equal(st.current, ref_st)


def test_repeated_calls_chain_on_device():
    # device mirror: two fills without touching .current == one longer fill
    st = fresh(64)
    a = sf.fill_uniform(st, sf.FillRequest(shape=(64, 64), grid=sf.WorkGrid(8, 8)))
    b = sf.fill_uniform(st, sf.FillRequest(shape=(64, 64), grid=sf.WorkGrid(8, 8)))
    st2 = fresh(64)
    c = sf.fill_uniform(st2, sf.FillRequest(shape=(128, 64), grid=sf.WorkGrid(8, 8)))
    assert np.array_equal(np.vstack([a.data, b.data]), c.data)
    assert st == st2


def test_host_edits_between_calls_are_honoured():
    st = fresh(4)
    sf.fill_uniform(st, sf.FillRequest(shape=8, grid=sf.WorkGrid(2, 2)))
    st.current[0] = [12345] * 6  # in-place edit by the caller
    v = sf.fill_uniform(st, sf.FillRequest(shape=2, grid=sf.WorkGrid(1, 1))).vector()
    assert v[0] == G_first()


def G_first():
    return 0.7353244530968368


def test_ks_uniform():
    from scipy import stats

    st = fresh(64)
    v = sf.fill_uniform(st, sf.FillRequest(shape=100_000, grid=sf.WorkGrid(8, 8))).vector()
    d = stats.kstest(v, "uniform").statistic
    assert d < math.sqrt(-math.log(0.0005) / 2) / math.sqrt(100_000)
    assert v.min() > 0 and v.max() < 1


# ----------------------------------------------------------------- normals
NRM = ["N64", "N34", "Nodd", "Nodd2", "Nvec"]


@pytest.mark.parametrize("name", NRM)
def test_normal_goldens_within_tolerance(G, A, name):
    g = G[name]
    shape = g["shape"] if isinstance(g["shape"], int) else tuple(g["shape"])
    ncol = shape if isinstance(shape, int) else shape[1]
    npad = g["npad"] if g["npad"] != ncol else None
    st = fresh(g["n_streams"])
    buf = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=grid(g["grid"]), npad=npad))
    ref = A[name + "_data"]
    assert_normal_f64_close(buf.data, ref)
    assert sha(st.current) == g["states_sha"]
    st = fresh(g["n_streams"])
    b32 = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=grid(g["grid"]), npad=npad,
                                            dtype=np.float32))
    assert b32.data.dtype == np.float32
    assert_normal_f32_close(b32.data, ref)
    assert sha(st.current) == g["states_sha"]


@pytest.mark.parametrize("name", ["N1", "Nwide"])
def test_normal_large_vs_oracle(G, name):
    g = G[name]
    shape = tuple(g["shape"])
    st = fresh(g["n_streams"])
    buf = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=grid(g["grid"])))
    ref_st = oa.fresh_states(g["n_streams"])
    ref = oa.fill("normal", ref_st, shape, tuple(g["grid"]))
    assert sha(ref) == g["data_sha"]
    assert_normal_f64_close(buf.data, ref)
    assert np.array_equal(st.current, ref_st)
    st = fresh(g["n_streams"])
    b32 = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=grid(g["grid"]),
                                            dtype=np.float32))
    assert_normal_f32_close(b32.data, ref)


@pytest.mark.parametrize("shape,g,n", [
    ((3, 3), (1, 2), 2), ((7, 9), (2, 4), 8), ((100, 101), (4, 10), 40),
    ((64, 1000), (8, 512), 4096), ((31250 // 50, 32000 // 50), (16, 16), 256),
])
def test_normal_layouts_vs_oracle(shape, g, n):
    st = fresh(n)
    buf = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g)))
    ref_st = oa.fresh_states(n)
    ref = oa.fill("normal", ref_st, shape, g)
    assert_normal_f64_close(buf.data, ref)
    assert np.array_equal(st.current, ref_st)
    # float32 form through the same layouts (fast and generic kernels)
    st = fresh(n)
    b32 = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g), dtype=np.float32))
    assert_normal_f32_close(b32.data, ref)
    assert np.array_equal(st.current, ref_st)


@pytest.mark.parametrize("shape,g,n,npad", [((7, 9), (2, 4), 8, 12), ((33, 64), (4, 8), 32, 70),
                                            ((5, 3), (1, 2), 2, 4)])
def test_normal_f32_padded_vs_oracle(shape, g, n, npad):
    st = fresh(n)
    b32 = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g), npad=npad,
                                            dtype=np.float32))
    ref_st = oa.fresh_states(n)
    ref = oa.fill("normal", ref_st, shape, g, npad=npad)
    assert_normal_f32_close(b32.data, ref)
    assert np.array_equal(st.current, ref_st)


def test_rsqrt_seed_accuracy():
    """The rsqrt.approx.f64 seed of the float32 Box-Muller form is within
    the 2^-19 relative error the CPU tests model (tests/test_host_lib.py::
    RSQRT_SEED_BOUND), over the whole range of -2 ln u1 (measured 2^-20.06)."""
    import torch

    rng = np.random.default_rng(3)
    z = np.concatenate([rng.integers(1, sf.M1 + 1, 4_000_000),
                        np.arange(1, 4097), sf.M1 - np.arange(0, 4096)])
    x = -2.0 * np.log(z * sf.NORM)
    x = x[x > 0]
    dx = torch.from_numpy(x).cuda()
    dy = torch.empty_like(dx)
    _lib.check(_lib.lib().sfb_probe_rsqrt(_lib.dptr(dx), _lib.dptr(dy), len(x),
                                          _lib.stream_handle()))
    y = dy.cpu().numpy()
    rel = np.abs(y * np.sqrt(x) - 1.0)
    print(f"rsqrt.approx.f64 max relative error {rel.max():.3e} (2^{np.log2(rel.max()):.2f})")
    assert rel.max() <= 2.0 ** -19


def test_normal_f32_large_vs_oracle():
    """float32 normals (box_muller_pair_f32) on 33.5 M cells of the configs[1]
    layout family vs float32(oracle): <= 1 ulp_f32 everywhere, identical on
    >= 99.999 %; the float64-rounded variant (SFB_NORMAL_VARIANT=4) identical
    on every cell seen so far (same contract asserted)."""
    import os

    shape, g, n = (4096, 8192), (512, 512), 1 << 18
    ref_st = oa.fresh_states(n)
    ref = oa.fill("normal", ref_st, shape, g)
    for variant in (None, "0", "4"):
        if variant is not None:
            os.environ["SFB_NORMAL_VARIANT"] = variant
        try:
            st = fresh(n)
            b32 = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g),
                                                    dtype=np.float32))
            got = b32.data
        finally:
            os.environ.pop("SFB_NORMAL_VARIANT", None)
        assert_normal_f32_close(got, ref)
        assert np.array_equal(st.current, ref_st)
        print(f"variant {variant}: {(got != ref.astype(np.float32)).sum()} of {got.size} "
              "cells differ from float32(reference) by 1 ulp")


def test_box_muller_pair_identity():
    # reference tests/test_distributions.py:83-99: x^2 + y^2 == -2 log(u1)
    import math

    g = sf.WorkGrid(4, 4)
    st = fresh(16)
    before = st.copy()
    v = sf.fill_normal(st, sf.FillRequest(shape=(64, 64), grid=g)).values
    for i in range(4):
        for j0 in (0, 2):
            s0 = sf.stream_index("normal", g, i, j0)
            s = before[s0]
            for r in range(i, 64, 4):
                for c in range(j0, 64, 4):
                    s, z1 = sf.next_state(s)
                    target = -2.0 * math.log(z1 * sf.NORM)
                    x, y = v[r, c], v[r, c + 1]
                    assert abs(x * x + y * y - target) <= 1e-12 * abs(target)


def test_normal_moments():
    st = fresh(64)
    v = sf.fill_normal(st, sf.FillRequest(shape=(1000, 1000), grid=sf.WorkGrid(8, 8))).values
    v = v.ravel()
    assert -0.004 < v.mean() < 0.004
    assert 0.994 < v.var() < 1.006


def test_odd_width_discards_partner_but_advances_both():
    st = fresh(2)
    before = st.copy()
    sf.fill_normal(st, sf.FillRequest(shape=(2, 3), grid=sf.WorkGrid(1, 2)))
    for w in range(2):
        s = before[w]
        for _ in range(4):
            s, _ = sf.next_state(s)
        assert st[w].g1 == s.g1


# ------------------------------------------------------------- exponential
@pytest.mark.parametrize("rate", [0.5, 1.0, 2.0])
def test_exponential_small(G, rate):
    st = fresh(4)
    buf = sf.fill_exponential(st, sf.FillRequest(shape=(2, 4), kind="exponential", rate=rate,
                                                 grid=sf.WorkGrid(2, 2)))
    ref = np.array(G[f"E24_{rate}"]["values"])
    assert np.array_equal(buf.values, ref)
    assert st.current.tolist() == G[f"E24_{rate}"]["states"]


def test_exponential_big(A):
    st = fresh(16)
    buf = sf.fill_exponential(st, sf.FillRequest(shape=(100, 100), kind="exponential",
                                                 rate=1.5, grid=sf.WorkGrid(4, 4)))
    ref = A["E100_data"]
    assert np.array_equal(buf.data, ref)
    assert np.array_equal(st.current, A["E100_states"])


# ------------------------------------------------------------------ Fisher
def _tables(G, A):
    t = {"T4": np.array(G["T4"]), "T10": np.array(G["T10"]), "month": A["month"],
         "week": A["week"]}
    for k in list(A):
        if k.startswith("tab_"):
            t[k[4:]] = A[k]
    return t


FIS = ["F_T4_1e6", "F_T10_1e6", "F_month_1e6", "F_week_1e6", "F_month_2e5", "F_month_s",
       "F_T4_s", "F_T10_s", "F_week_s", "F_2x2_s", "F_E2x2", "F_E2x5", "F_E5x2",
       "F_Ezero_col", "F_Eones", "F_Ebig", "F_week_1e7"]


@pytest.mark.parametrize("key", FIS)
def test_fisher_goldens_bit_exact(G, A, key):
    g = G[key]
    tabs = _tables(G, A)
    st = fresh(g["n_streams"])
    want = key + "_stats" in A
    r = sf.fisher_sim(tabs[g["table"]], g["n"], st, grid=grid(g["grid"]), return_stats=want)
    assert r.sim_num == g["sim_num"]
    assert r.counts == g["counts"]
    assert r.p_value == g["p_value"]
    assert r.threshold == g["threshold"]
    assert sha(st.current) == g["states_sha"]
    if want:
        assert np.array_equal(r.statistics, A[key + "_stats"])


def test_fisher_rerun_and_chunk_invariance(A):
    # replicate chunking depends on the item count; results must not
    month = A["month"]
    base = None
    for g in [(1, 1), (2, 2), (4, 4), (16, 16)]:
        n_items = g[0] * g[1]
        st = fresh(n_items)
        r = sf.fisher_sim(month, 4096, st, grid=sf.WorkGrid(*g), return_stats=True)
        ref_st = oa.fresh_states(n_items)
        ref = oa.fisher(month, 4096, ref_st, g, return_stats=True)
        assert r.counts == ref["counts"]
        assert np.array_equal(r.statistics, ref["statistics"])
        assert np.array_equal(st.current, ref_st)
        if base is None:
            base = r.counts


def test_fisher_stream_advancement_audit(A):
    st = fresh(4)
    before = st.copy()
    r = sf.fisher_sim(A["month"], 8, st, grid=sf.WorkGrid(2, 2))
    reps = r.sim_num // 4
    for w in range(4):
        s = sf.skip_ahead(before[w], reps * 121)
        assert st[w].g1 == s.g1 and st[w].g2 == s.g2


def test_fisher_item_shards_compose(G, A):
    # the multi-GPU decomposition on one device: disjoint item ranges
    import torch

    from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher

    t10 = np.array(G["T10"])
    st = fresh(16384)
    plan = plan_fisher(t10, 10 ** 6, st, sf.WorkGrid(256, 64))
    cur = st.device_current()
    total = 0
    for lo, hi in [(0, 5000), (5000, 5001), (5001, 16384)]:
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        launch_fisher(plan, cur, st.count, cnt, item_lo=lo, item_hi=hi)
        total += int(cnt.item())
    st._mark_device_ahead()
    assert total == G["F_T10_1e6"]["counts"]
    assert sha(st.current) == G["F_T10_1e6"]["states_sha"]


def test_fisher_t10_sampled_items_many_reps(G):
    # C4 shape: per-item counts/final states for sampled items at 4769 reps
    import torch

    from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher

    t10 = np.array(G["T10"])
    n_items = 1 << 14
    st = fresh(n_items)
    plan = plan_fisher(t10, 4769 * n_items, st, sf.WorkGrid(128, 128))
    assert plan.reps == 4769
    rng = np.random.default_rng(5)
    items = np.sort(rng.choice(n_items, 12, replace=False))
    cur = st.device_current()
    ic = torch.zeros(n_items, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    launch_fisher(plan, cur, st.count, cnt, item_counts_dev=ic)
    st._mark_device_ahead()
    ic = ic.cpu().numpy()
    assert ic.sum() == int(cnt.item())
    ref_st = oa.fresh_states(n_items)
    for w in items:
        item_counts = np.zeros(1, np.int64)
        orc.fisher_replicates(ref_st, t10.sum(1), t10.sum(0), plan.lf, plan.kernel_threshold,
                              plan.reps, int(w) + 1, item_lo=int(w), item_counts=item_counts)
        assert ic[w] == item_counts[0]
        assert np.array_equal(st.current[w], ref_st[w])


def test_rcont2_goldens(G, A):
    month = A["month"]
    t = sf.ContingencyTable(month)
    lf = sf.fisher.log_factorial_table(t.total)
    state = np.array([12345] * 6, np.int64)
    tabs = [sf.rcont2(t.row_margins, t.col_margins, state, lf) for _ in range(5)]
    assert np.array_equal(np.array(tabs), A["rcont2_month5"])
    assert state.tolist() == G["rcont2_month5_state"]
    state = np.array([12345] * 6, np.int64)
    assert sf.rcont2([7], [2, 2, 3], state).tolist() == [[2, 2, 3]]
    assert state.tolist() == [12345] * 6
    state = np.array([12345] * 6, np.int64)
    t10 = sf.rcont2([20000, 8000, 3000, 1000, 400, 150, 60, 25, 10, 5],
                    [13000, 9000, 5000, 2500, 1200, 1000, 600, 250, 75, 25], state)
    assert t10.tolist() == G["T10"]


def test_2x2_converges_to_exact_fisher_p():
    from scipy.special import gammaln

    def pmf(k, ia, idv, ie):
        return math.exp(gammaln(ia + 1) + gammaln(ie - ia + 1) + gammaln(idv + 1)
                        + gammaln(ie - idv + 1) - gammaln(ie + 1) - gammaln(k + 1)
                        - gammaln(idv - k + 1) - gammaln(ia - k + 1)
                        - gammaln(ie - ia - idv + k + 1))

    table = np.array([[3, 7], [6, 2]])
    obs = sf.logfact_sum(table)
    total, ia, idv = 18, 10, 9
    exact = 0.0
    for k in range(max(0, ia + idv - total), min(ia, idv) + 1):
        cand = np.array([[k, ia - k], [idv - k, total - ia - idv + k]])
        if sf.logfact_sum(cand) <= sf.fisher.relaxed_threshold(obs):
            exact += pmf(k, ia, idv, total)
    res = sf.fisher_sim(table, 10 ** 6, fresh(64), grid=sf.WorkGrid(8, 8))
    se = math.sqrt(exact * (1 - exact) / res.sim_num)
    assert abs(res.p_value - exact) < 3 * se


# -------------------------------------------------------------- checkpoint
def test_checkpoint_continuation_c5_64(G, tmp_path):
    import torch

    g = sf.WorkGrid(128, 128)
    st = fresh(1 << 14)
    a = sf.run_grid(st, g, 4096, 8192, "uniform")
    p = tmp_path / "ckpt.txt"
    sf.save_streams_atomic(st, p)
    st2 = sf.load_streams(p)
    b = sf.run_grid(st2, g, 4096, 8192, "uniform")
    full = torch.cat([a.tensor, b.tensor]).cpu().numpy()
    assert sha(full) == G["C5_64"]["full_sha"]
    assert sha(st2.current) == G["C5_64"]["states_sha"]


@pytest.mark.slow
def test_checkpoint_continuation_c5_full(tmp_path):
    # C5 at full size on the device: 2^20 streams x 4096 uniforms (34.4 GB),
    # checkpoint after rows [0, 32768), resume -> identical bytes and states
    import torch

    g = sf.WorkGrid(1024, 1024)
    st_full = fresh(1 << 20)
    full = sf.run_grid(st_full, g, 65536, 65536, "uniform")
    st = fresh(1 << 20)
    a = sf.run_grid(st, g, 32768, 65536, "uniform")
    assert torch.equal(a.tensor, full.tensor[:32768])
    del a
    p = tmp_path / "c5.txt"
    sf.save_streams_atomic(st, p)
    st2 = sf.load_streams(p)
    b = sf.run_grid(st2, g, 32768, 65536, "uniform")
    assert torch.equal(b.tensor, full.tensor[32768:])
    assert st2 == st_full
    # against the oracle, not only self-consistency: every final state is
    # A^4096 s_w (4096 draws per stream), and sampled cells equal the oracle's
    # skip-ahead draws (_kernels.py:50-80: item (i, j) = stream i + g0 j owns
    # cells r = i mod g0, c = j mod g1, row-major)
    seeds = oa.fresh_states(1 << 20)
    assert np.array_equal(st_full.current, skip_all(seeds, 12))
    rng = np.random.default_rng(2026)
    rows = np.concatenate([rng.integers(0, 65536, 8192), [0, 0, 65535, 65535]])
    cols = np.concatenate([rng.integers(0, 65536, 8192), [0, 65535, 0, 65535]])
    got = full.tensor[torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()].cpu().numpy()
    for r, c, v in zip(rows, cols, got):
        w = (r % 1024) + 1024 * (c % 1024)
        s = orc.skip(seeds[w], (r // 1024) * 64 + c // 1024)
        assert v == orc.step(s) * 2.0 ** -31, (r, c)


def skip_all(states, e):
    """Every row of an (n, 6) state array advanced by 2^e steps (the oracle's
    jump matrices T^(2^e), core.py:55-62, applied with exact uint64 sums)."""
    j1, j2 = orc.jump_matrices(e)
    out = np.empty_like(states)
    for half, j, m in ((slice(0, 3), j1, sf.core.M1), (slice(3, 6), j2, sf.core.M2)):
        v = states[:, half].astype(np.uint64)
        acc = np.zeros_like(v)
        for k in range(3):  # three products < 2^62 each: the sum fits uint64
            acc += v[:, k:k + 1] * j.astype(np.uint64)[:, k][None, :]
        out[:, half] = (acc % np.uint64(m)).astype(np.int64)
    return out


@pytest.mark.slow
def test_normal_configs1_full_shape_vs_oracle():
    """configs[1] at its real shape: 31250 x 32000 float32 normals from 2^18
    streams on WorkGrid(512, 512) (ragged ownership: 31250 = 512*61 + 18 rows,
    62.5 columns per lane) vs float32(oracle): <= 1 ulp_f32 everywhere,
    identical on >= 99.999 % of the 1e9 cells, final states bit-exact."""
    shape, g, n = (31250, 32000), (512, 512), 1 << 18
    st = fresh(n)
    got = sf.fill_normal(st, sf.FillRequest(shape=shape, grid=sf.WorkGrid(*g),
                                            dtype=np.float32)).values
    ref_st = oa.fresh_states(n)
    ref = np.zeros(shape, np.float32)
    orc.fill_normal(ref_st, ref.ravel(), shape[0], shape[1], shape[1], g[0], g[1])
    assert np.array_equal(st.current, ref_st)
    diff = got != ref
    nd = int(diff.sum())
    print(f"configs[1]: {nd} of {got.size} cells differ from float32(reference)")
    assert nd <= got.size * 1e-5
    if nd:
        a = got[diff].astype(np.float64)
        b = ref[diff].astype(np.float64)
        assert (np.abs(a - b) <= np.spacing(np.abs(ref[diff])).astype(np.float64)).all()


def test_sharded_api_single_rank(A):
    # the multi-GPU entry points on one device (world size 1, no collective)
    from paper_2201_06604_b200 import sharding

    st = fresh(64)
    r = sharding.fisher_sim_sharded(A["month"], 3000, st, sf.WorkGrid(8, 8), return_stats=True)
    ref_st = oa.fresh_states(64)
    ref = oa.fisher(A["month"], 3000, ref_st, (8, 8), return_stats=True)
    assert r.counts == ref["counts"]
    assert np.array_equal(r.statistics, ref["statistics"])
    assert np.array_equal(st.current, ref_st)
    st = fresh(64)
    buf = sharding.run_grid_sharded(st, sf.WorkGrid(8, 8), 100, 120, "uniform")
    ref_st = oa.fresh_states(64)
    assert np.array_equal(buf.data, oa.fill("uniform", ref_st, (100, 120), (8, 8)))
    assert np.array_equal(st.current, ref_st)


@pytest.mark.parametrize("shape,g,n,rate", [((257, 300), (16, 16), 256, 0.7),
                                            ((64, 4096), (8, 512), 4096, 3.0),
                                            (5001, (1, 64), 64, 1.0)])
def test_exponential_layouts_bit_exact(shape, g, n, rate):
    st = fresh(n)
    buf = sf.fill_exponential(st, sf.FillRequest(shape=shape, kind="exponential", rate=rate,
                                                 grid=sf.WorkGrid(*g)))
    ref_st = oa.fresh_states(n)
    ref = oa.fill("exponential", ref_st, shape, g, rate=rate)
    assert np.array_equal(buf.data, ref)
    assert np.array_equal(st.current, ref_st)


@pytest.mark.parametrize("walk", [0, 1, 2, 3])
def test_fisher_walk_forms_bit_exact(G, A, walk, monkeypatch):
    monkeypatch.setenv("SFB_FISHER_WALK", str(walk))
    for key in ("F_T10_1e6", "F_month_s", "F_Ebig", "F_E5x2"):
        g = G[key]
        tabs = _tables(G, A)
        st = fresh(g["n_streams"])
        want = key + "_stats" in A
        r = sf.fisher_sim(tabs[g["table"]], g["n"], st, grid=grid(g["grid"]), return_stats=want)
        assert r.counts == g["counts"]
        assert sha(st.current) == g["states_sha"]
        if want:
            assert np.array_equal(r.statistics, A[key + "_stats"])


@pytest.mark.slow
def test_fisher_c4_full_scale_sampled_items(G):
    # C4 (BASELINE configs[3]): T10, 1e10 tables on grid (2048, 1024), 2^21
    # streams (4769 reps per item).  The total count is checked for
    # consistency with the per-item counts; 256 random items are re-run on the
    # oracle (1.2e6 tables) and must match counts and final states bit for bit.
    import torch

    from paper_2201_06604_b200.fisher import launch_fisher, plan_fisher

    t10 = np.array(G["T10"])
    grid = sf.WorkGrid(2048, 1024)
    st = fresh(grid.size)
    plan = plan_fisher(t10, 10 ** 10, st, grid)
    assert plan.reps == 4769 and plan.sim_num == 10001317888
    cur = st.device_current()
    ic = torch.zeros(grid.size, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    launch_fisher(plan, cur, st.count, cnt, item_counts_dev=ic)
    st._mark_device_ahead()
    ic = ic.cpu().numpy()
    assert ic.sum() == int(cnt.item())
    rng = np.random.default_rng(2201)
    items = rng.choice(grid.size, 256, replace=False)
    ref_st = oa.fresh_states(grid.size)
    final = st.current
    for w in items:
        one = np.zeros(1, np.int64)
        orc.fisher_replicates(ref_st, t10.sum(1), t10.sum(0), plan.lf, plan.kernel_threshold,
                              plan.reps, int(w) + 1, item_lo=int(w), item_counts=one)
        assert ic[w] == one[0], w
        assert np.array_equal(final[w], ref_st[w]), w


def test_chunked_pinned_download_matches_tensor():
    # MatrixBuffer.download splits large pinned copies over two copy streams
    import torch

    st = fresh(1 << 14)
    buf = sf.fill_uniform(st, sf.FillRequest(shape=(4099, 16384), grid=sf.WorkGrid(128, 128)))
    host = torch.empty((4099, 16384), dtype=torch.float64, pin_memory=True)
    buf.download(host)
    assert torch.equal(host, buf.tensor.cpu())


@pytest.mark.parametrize("shape,g1,jr", [((64, 4096), 1024, (128, 256)), ((33, 1000), 64, (4, 12)),
                                         ((5, 70), 32, (0, 32))])
def test_download_shard_matches_column_selection(shape, g1, jr):
    # MatrixBuffer.download_shard: a rank's grid columns, packed (row, q, j)
    import torch

    g0 = 4
    st = fresh(g0 * g1)
    buf = sf.fill_uniform(st, sf.FillRequest(shape=shape, grid=sf.WorkGrid(g0, g1)))
    got = buf.download_shard(g1, *jr).numpy()
    full = buf.values
    want = np.concatenate([full[r, [c for c in range(shape[1]) if jr[0] <= c % g1 < jr[1]]]
                           for r in range(shape[0])])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("kind", ["uniform", "uniform-integer", "exponential"])
def test_generic_kernel_beyond_2p31_cells(kind):
    """The generic kernel (odd g1) on a 46341 x 46347 matrix (2.15e9 cells >
    2^31: 64-bit offsets everywhere): 4096 sampled cells, the four corners and
    the final states of all 15 items against the oracle's skip-ahead."""
    import torch

    from paper_2201_06604_b200.grid import launch_fill

    nrow, ncol, g0, g1 = 46341, 46347, 3, 5
    assert nrow * ncol > 2 ** 31
    st = fresh(g0 * g1)
    cur = st.device_current()
    dt = torch.int64 if kind == "uniform-integer" else torch.float64
    out = torch.empty((nrow, ncol), dtype=dt, device="cuda")
    launch_fill(kind, cur, st.count, out, nrow, ncol, ncol, g0, g1, rate=0.37)
    torch.cuda.synchronize()
    rng = np.random.default_rng(31)
    rows = np.concatenate([rng.integers(0, nrow, 4096), [0, 0, nrow - 1, nrow - 1]])
    cols = np.concatenate([rng.integers(0, ncol, 4096), [0, ncol - 1, 0, ncol - 1]])
    got = out[torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()].cpu().numpy()
    seeds = oa.fresh_states(g0 * g1)
    for r, c, v in zip(rows, cols, got):
        i, j = r % g0, c % g1
        w = i + g0 * j
        ncols_item = (ncol - j + g1 - 1) // g1
        s = orc.skip(seeds[w], (r // g0) * ncols_item + c // g1)
        z = orc.step(s)
        if kind == "uniform-integer":
            want = z
        elif kind == "uniform":
            want = z * 2.0 ** -31
        else:
            want = -math.log1p(-(z * 2.0 ** -31)) / 0.37
        assert v == want, (kind, r, c, v, want)
    final = cur.cpu().numpy()
    for w in rng.choice(g0 * g1, 15, replace=False):
        i, j = w % g0, w // g0
        nr_item = (nrow - i + g0 - 1) // g0
        nc_item = (ncol - j + g1 - 1) // g1
        assert np.array_equal(final[w], orc.skip(seeds[w], nr_item * nc_item)), w


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_normal_beyond_2p31_cells(dtype):
    """Box-Muller fill of a 46341 x 46345 matrix (> 2^31 cells; odd ncol, so
    the last column's partner lane is discarded) on grid (3, 6): 4096 sampled
    cells and the corners against the oracle's transform of skip-ahead draws
    (float32: <= 1 ulp of float32(ref); float64: the 4-ulp contract)."""
    import torch

    from paper_2201_06604_b200.grid import launch_fill

    nrow, ncol, g0, g1 = 46341, 46345, 3, 6
    assert nrow * ncol > 2 ** 31
    st = fresh(g0 * g1)
    cur = st.device_current()
    out = torch.empty((nrow, ncol), dtype=getattr(torch, dtype), device="cuda")
    launch_fill("normal", cur, st.count, out, nrow, ncol, ncol, g0, g1)
    torch.cuda.synchronize()
    rng = np.random.default_rng(32)
    rows = np.concatenate([rng.integers(0, nrow, 4096), [0, 0, nrow - 1, nrow - 1]])
    cols = np.concatenate([rng.integers(0, ncol, 4096), [0, ncol - 1, 0, ncol - 1]])
    got = out[torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()].cpu().numpy()
    seeds = oa.fresh_states(g0 * g1)
    z1s, z2s = [], []
    for r, c in zip(rows, cols):
        i, j = r % g0, c % g1
        j0 = j - (j & 1)
        s0 = i * g1 + j0
        idx = (r // g0) * ((ncol - j0 + g1 - 1) // g1) + c // g1
        z1s.append(orc.step(orc.skip(seeds[s0], idx)))
        z2s.append(orc.step(orc.skip(seeds[s0 + 1], idx)))
    a, b = orc.box_muller(np.array(z1s), np.array(z2s))
    want = np.where(cols % 2 == 0, a, b)
    if dtype == "float32":
        ref = want.astype(np.float32)
        assert (np.abs(got.astype(np.float64) - ref) <= np.spacing(np.abs(ref))).all()
    else:
        assert_normal_f64_close(got, want)
    final = cur.cpu().numpy()
    for w in range(g0 * g1):
        i, j = w // g1, w % g1
        j0 = j - (j & 1)
        n = ((nrow - i + g0 - 1) // g0) * ((ncol - j0 + g1 - 1) // g1)
        assert np.array_equal(final[w], orc.skip(seeds[w], n)), w


@pytest.mark.parametrize("table", [[[500000, 500000], [400000, 600000]],
                                   [[300000, 2, 250000], [1, 310000, 5], [120000, 7, 20000]]])
def test_fisher_large_totals(table):
    """Totals in the millions (lf tables of ~8 MB in global memory, walks of
    hundreds to thousands of steps, memo sets over +-7 sigma windows of
    thousands of configurations): counts, statistics and states bit-exact."""
    t = np.array(table)
    st = fresh(64)
    r = sf.fisher_sim(t, 3000, st, grid=grid((8, 8)), return_stats=True)
    ref_st = oa.fresh_states(64)
    ref = oa.fisher(t, 3000, ref_st, (8, 8), return_stats=True)
    assert r.counts == ref["counts"] and r.sim_num == ref["sim_num"]
    assert np.array_equal(r.statistics, ref["statistics"])
    assert np.array_equal(st.current, ref_st)


def test_concurrent_host_threads_match_serial(G):
    """Four host threads calling fisher_sim (different tables: the per-device
    input cache switches under its lock), fills and rcont2 concurrently give
    the serial results."""
    import threading

    tables = [np.array(G["T4"]), np.array(G["T10"]), np.array([[3, 7], [6, 2]]),
              np.array([[5, 0, 4], [2, 6, 1]])]

    def work(t):
        st = fresh(256)
        r = sf.fisher_sim(t, 5000, st, grid=grid((16, 16)), return_stats=True)
        st2 = fresh(64)
        u = sf.fill_uniform(st2, sf.FillRequest(shape=(300, 200), grid=grid((8, 8)))).data
        s6 = fresh(1).current[0].copy()
        tab = sf.rcont2(t.sum(1), t.sum(0), s6)
        return (r.counts, r.statistics.tobytes(), st.current.tobytes(), u.tobytes(),
                st2.current.tobytes(), tab.tobytes(), s6.tobytes())

    serial = [work(t) for t in tables]
    for _ in range(3):
        out = [None] * len(tables)

        def run(i):
            out[i] = work(tables[i])

        th = [threading.Thread(target=run, args=(i,)) for i in range(len(tables))]
        for x in th:
            x.start()
        for x in th:
            x.join()
        assert out == serial


# ------------------------------------------- Fisher drop-in edge cases (r2)
def _random_table(rows, cols, lam, seed):
    t = np.random.default_rng(seed).poisson(lam, (rows, cols)).astype(np.int64)
    t[0, 0] += 1  # total >= 1
    return t


@pytest.mark.parametrize("shape,lam", [((2, 300), 3.0), ((3, 500), 2.0), ((300, 2), 3.0)])
def test_fisher_wide_tables_vs_oracle(shape, lam):
    """Tables wider than the shared-memory column work (>~198 columns) run
    with the column work in global memory (the reference allocates jwork for
    any nc, _kernels.py:193-194): counts, statistics, states bit-exact."""
    t = _random_table(*shape, lam, seed=shape[1])
    st = fresh(64)
    r = sf.fisher_sim(t, 640, st, grid=grid((8, 8)), return_stats=True)
    ref_st = oa.fresh_states(64)
    ref = oa.fisher(t, 640, ref_st, (8, 8), return_stats=True)
    assert r.counts == ref["counts"] and r.sim_num == ref["sim_num"]
    assert np.array_equal(r.statistics, ref["statistics"])
    assert np.array_equal(st.current, ref_st)


def test_fisher_wide_table_many_chunks():
    """A wide table on a small grid: many replicate chunks visited grid-stride
    by a capped grid; per-item counts and states bit-exact."""
    t = _random_table(3, 500, 2.0, seed=7)
    st = fresh(4)
    r = sf.fisher_sim(t, 4 * 700, st, grid=grid((2, 2)), return_stats=True)
    ref_st = oa.fresh_states(4)
    ref = oa.fisher(t, 4 * 700, ref_st, (2, 2), return_stats=True)
    assert r.counts == ref["counts"]
    assert np.array_equal(r.statistics, ref["statistics"])
    assert np.array_equal(st.current, ref_st)


def test_rcont2_very_wide_table_uses_global_column_work():
    """rcont2 on 2 x 20000 (80 KB of column work, beyond 48 KB of shared
    memory): table and state equal the oracle's rcont2_table."""
    rows = np.array([15000, 14000], np.int64)
    cols = np.full(20000, 1, np.int64)
    cols[:9000] += 1
    lf = oa.lf_table(int(rows.sum()))
    s_gpu = np.array([12345] * 6, np.int64)
    s_ref = s_gpu.copy()
    tab = sf.rcont2(rows, cols, s_gpu, lf)
    ref = orc.rcont2_table(rows, cols, lf, s_ref)
    assert np.array_equal(tab, ref)
    assert np.array_equal(s_gpu, s_ref)


def test_fisher_count_beyond_int32_per_cta():
    """2^32 replicates on a one-item grid: one CTA counts ~2.9e9 hits, which
    must not wrap (the reference counts in int64, _kernels.py:185,195,279).
    Both possible 2x2 tables of these margins score 0 <= threshold, so every
    replicate is a hit."""
    st = fresh(1)
    before = st.copy()
    r = sf.fisher_sim([[1, 0], [0, 1]], 2 ** 32, st, grid=grid((1, 1)))
    assert r.sim_num == 2 ** 32
    assert r.counts == r.sim_num
    s = sf.skip_ahead(before[0], 2 ** 32)  # one draw per replicate
    assert st[0].g1 == s.g1 and st[0].g2 == s.g2


# ------------------------------------------- host-path semantics
def test_held_current_reference_after_fisher_sim():
    """A reference to `.current` held across fisher_sim calls behaves like the
    reference's plain attribute: it shows the final states, and in-place edits
    made through it are honoured by the next call."""
    t4 = [[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]
    st = fresh(2048)  # 96 KiB: the page-locked path
    held = st.current
    sf.fisher_sim(t4, 2048 * 3, st, grid=grid((32, 64)))
    ref = oa.fresh_states(2048)
    ref_ct = oa.fisher(t4, 2048 * 3, ref, (32, 64))
    assert np.array_equal(held, ref)
    held[:] = oa.fresh_states(2048)  # rewind in place through the held array
    r = sf.fisher_sim(t4, 2048 * 3, st, grid=grid((32, 64)))
    assert r.counts == ref_ct["counts"]
    assert np.array_equal(held, ref)


def test_held_current_reference_after_fill_refreshes_on_read():
    """Fills leave the new states on the device (lazy host sync); the held
    array is the same object and is refreshed in place at the next `.current`
    read (documented contract)."""
    st = fresh(2048)
    held = st.current
    sf.fill_uniform(st, sf.FillRequest(shape=(64, 128), grid=grid((32, 64))))
    ref = oa.fresh_states(2048)
    oa.fill("uniform", ref, (64, 128), (32, 64))
    cur = st.current
    assert cur is held
    assert np.array_equal(held, ref)


def test_shared_pinned_array_leaves_no_cuda_error():
    """A StreamSet built on another one's (page-locked) array does not
    register it twice, and no CUDA error is left behind for the next launch."""
    import torch

    a = fresh(4096)
    a.device_current()  # page-locks a's array
    b = sf.StreamSet(a.current, a.initial)
    b.device_current()
    x = torch.ones(1024, device="cuda") * 2  # a plain torch launch after the registrations
    torch.cuda.synchronize()
    assert float(x.sum()) == 2048.0
    sf.fill_uniform(b, sf.FillRequest(shape=(8, 4096), grid=grid((1, 4096))))
    ref = oa.fresh_states(4096)
    oa.fill("uniform", ref, (8, 4096), (1, 4096))
    assert np.array_equal(b.current, ref)


def test_fisher_cache_on_two_streams_alternating_tables():
    """Alternating tables on two CUDA streams: every call reuses or refills an
    entry of the per-device input LRU; a reuse waits for the upload issued on
    the other stream, an overwrite waits for readers on every stream."""
    import torch

    tabs = [np.array([[5, 9, 5, 7], [9, 5, 9, 7], [8, 6, 2, 6], [10, 8, 8, 8]]),
            np.array([[3, 7], [6, 2]]), np.array([[5, 0, 4], [2, 6, 1]]),
            np.array([[1, 2, 3, 4, 5], [5, 4, 3, 2, 1]]), np.array([[9, 1], [1, 9], [4, 4]]),
            np.array([[2, 2, 2], [3, 3, 3], [1, 0, 7]])]
    want = []
    for t in tabs:
        ref = oa.fresh_states(256)
        want.append(oa.fisher(t, 256 * 40, ref, (16, 16))["counts"])
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for rnd in range(3):
        for k, t in enumerate(tabs):
            with torch.cuda.stream(s1 if (k + rnd) % 2 else s2):
                r = sf.fisher_sim(t, 256 * 40, fresh(256), grid=grid((16, 16)))
            assert r.counts == want[k], (rnd, k)


@pytest.mark.parametrize("shape", [(2, 2), (2, 3), (3, 2), (3, 3), (3, 4), (4, 3), (4, 4)])
@pytest.mark.parametrize("mode", ["fixed", "generic"])
def test_fisher_fixed_shapes_vs_oracle(shape, mode, monkeypatch):
    """The compile-time-shape samplers (sample_table_fixed: unrolled cells,
    column work in registers) and the generic one both equal the oracle:
    counts, statistics and final states, on many chunks (small grid), odd
    and even replicate counts, with tabulated, truncated and walked
    configurations (lambda = 6 and 40)."""
    monkeypatch.setenv("SFB_FISHER_FIXED", "0" if mode == "generic" else "1")
    for lam, n in ((6.0, 16 * 300), (40.0, 16 * 301), (6.0, 16 * 7)):
        t = _random_table(*shape, lam, seed=shape[0] * 10 + shape[1])
        st = fresh(16)
        r = sf.fisher_sim(t, n, st, grid=grid((4, 4)), return_stats=True)
        ref_st = oa.fresh_states(16)
        ref = oa.fisher(t, n, ref_st, (4, 4), return_stats=True)
        assert r.counts == ref["counts"]
        assert np.array_equal(r.statistics, ref["statistics"])
        assert np.array_equal(st.current, ref_st)


@pytest.mark.parametrize("table_key,n,g", [("T4", 10**6, (256, 64)), ("T10", 200000, (64, 16)),
                                           ("T4", 3000, (16, 16))])
def test_fisher_host_and_device_states_agree(G, table_key, n, g):
    """fisher_sim on host-authoritative states (one synchronous C-ABI call; for
    chunked launches the final states are computed on a side stream and
    downloaded while the sampling kernel runs) and on device-resident states
    (in-stream advance) give the same counts and final states, and both match
    the oracle's final states A^(reps F) s (fisher.py:118-164)."""
    import torch

    table = np.array(G[table_key])
    a, b = fresh(g[0] * g[1]), fresh(g[0] * g[1])
    _ = b.device_current()  # b starts device-resident
    ra = sf.fisher_sim(table, n, a, grid=grid(g))
    rb = sf.fisher_sim(table, n, b, grid=grid(g))
    torch.cuda.synchronize()
    assert ra.counts == rb.counts and ra.sim_num == rb.sim_num
    assert np.array_equal(a.current, b.current)
    f = (table.shape[0] - 1) * (table.shape[1] - 1)
    reps = ra.sim_num // (g[0] * g[1])
    seeds = oa.fresh_states(g[0] * g[1])
    for w in (0, 1, g[0] * g[1] // 2, g[0] * g[1] - 1):
        assert np.array_equal(a.current[w], orc.skip(seeds[w], reps * f)), w


@pytest.mark.parametrize("level", [2, 3])
def test_fisher_large_memo_level_bit_exact(G, A, monkeypatch, level):
    """The large memo sets (SFB_FISHER_MEMO_UPGRADE=2 / 3: level 1 / 2 built
    synchronously at the first use, with the budgets the background upgrade
    uses) give the golden counts, statistics and states bit for bit."""
    monkeypatch.setenv("SFB_FISHER_MEMO_UPGRADE", str(level))
    tabs = _tables(G, A)
    for key in ("F_T10_1e6", "F_month_s", "F_Ebig"):
        g = G[key]
        st = fresh(g["n_streams"])
        want = key + "_stats" in A
        r = sf.fisher_sim(tabs[g["table"]], g["n"], st, grid=grid(g["grid"]), return_stats=want)
        assert r.counts == g["counts"]
        assert sha(st.current) == g["states_sha"]
        if want:
            assert np.array_equal(r.statistics, A[key + "_stats"])


def test_fisher_background_memo_upgrades_land_and_agree(G):
    """Repeated calls on a capped table start the background builds (level 1,
    then 2); sfb_fisher_memo_pending() drops to 0 once both are installed, and
    the results before, during and after the upgrades equal the first call's
    (every memo level is bit-exact).  A T10 variant keeps the table's memo
    fresh in this process."""
    import time

    from paper_2201_06604_b200 import _lib

    t10 = np.array(G["T10"])
    t10[0, 0] += 1
    g = sf.WorkGrid(64, 32)
    ref = None
    t0 = time.perf_counter()
    seen_pending = False
    calls = 0
    while time.perf_counter() - t0 < 600:  # queued builds of earlier tests run first
        st = fresh(g.size)
        r = sf.fisher_sim(t10, 20000, st, grid=g, return_stats=True)
        calls += 1
        if ref is None:
            ref = (r.counts, r.statistics.copy(), st.current.copy())
        else:
            assert r.counts == ref[0]
            assert np.array_equal(r.statistics, ref[1])
            assert np.array_equal(st.current, ref[2])
        pend = _lib.lib().sfb_fisher_memo_pending()
        seen_pending |= pend > 0
        if calls > 2 and pend == 0 and seen_pending:
            break
        time.sleep(0.05)
    assert seen_pending, "no background memo build started"
    assert _lib.lib().sfb_fisher_memo_pending() == 0


def test_process_exits_cleanly_with_a_memo_build_in_flight(G, tmp_path):
    """A process that leaves a background memo build running (detached host
    thread) still exits with status 0: the memo cache is never destroyed, so
    the thread cannot touch freed state during static destruction."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "exit_check.py"
    script.write_text(
        "import json, sys\n"
        "import numpy as np\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_2201_06604_b200 as sf\n"
        "from paper_2201_06604_b200 import _lib\n"
        f"t10 = np.array(json.load(open({os.path.join(root, 'tests', 'golden', 'golden.json')!r}))['T10'])\n"
        "t10[1, 1] += 2\n"
        "g = sf.WorkGrid(64, 32)\n"
        "for i in range(3):\n"
        "    st = sf.create_streams(sf.set_base_creator(), g.size)[0]\n"
        "    sf.fisher_sim(t10, 20000, st, grid=g)\n"
        "print('pending', _lib.lib().sfb_fisher_memo_pending())\n")
    r = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "pending" in r.stdout
