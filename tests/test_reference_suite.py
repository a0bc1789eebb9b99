"""The reference's own behavioural tests, re-run against the B200 path.

Each test restates one case of /root/reference/pkg/tests/ (file:line in the
docstring) through this package's public API, so the drop-in is held to the
reference's acceptance criteria as well as to the oracle (test_gpu_parity.py).
"""

import math

import numpy as np
import pytest
from scipy import stats as scipy_stats
from scipy.special import gammaln

import paper_2201_06604_b200 as sf
from paper_2201_06604_b200.errors import (InvalidArgumentError, InsufficientStreamsError,
                                          InvalidMarginsError)
from paper_2201_06604_b200.fisher import log_factorial_table

pytestmark = pytest.mark.gpu


def fresh(n):
    return sf.create_streams(sf.set_base_creator(), n)[0]


def ks_bound(n):
    # the reference's 0.1 % two-sided KS acceptance bound
    return math.sqrt(-math.log(0.0005) / 2) / math.sqrt(n)


@pytest.fixture(scope="module")
def month_table():
    from conftest import golden_arrays

    return np.asarray(golden_arrays()["month"], np.int64)


@pytest.fixture(scope="module")
def week_table():
    from conftest import golden_arrays

    return np.asarray(golden_arrays()["week"], np.int64)


# ------------------------------------------------------------ distributions
def test_doubles_strictly_inside_unit_interval():
    """tests/test_distributions.py:27-33 (at 2.6e8 draws instead of 1e5)."""
    v = sf.fill_uniform(fresh(1 << 18), sf.FillRequest(shape=(16384, 16384),
                                                      grid=sf.WorkGrid(512, 512))).tensor
    assert float(v.min()) > 0.0 and float(v.max()) < 1.0
    assert float(v.min()) >= 2.0 ** -31 and float(v.max()) <= 1.0 - 2.0 ** -31


def test_integer_kind_range():
    """tests/test_distributions.py:35-44."""
    v = sf.fill_uniform(fresh(64), sf.FillRequest(shape=(1000, 1000), kind="uniform-integer",
                                                  grid=sf.WorkGrid(8, 8))).values
    assert v.dtype == np.int64
    assert v.min() >= 1 and v.max() <= sf.M1


def test_repeated_fill_from_copied_states_is_identical():
    """tests/test_distributions.py:46-51."""
    base = fresh(16)
    a = sf.fill_uniform(base.copy(), sf.FillRequest(shape=(40, 40), grid=sf.WorkGrid(4, 4)))
    b = sf.fill_uniform(base.copy(), sf.FillRequest(shape=(40, 40), grid=sf.WorkGrid(4, 4)))
    assert np.array_equal(a.values, b.values)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_acceptance_08_distribution_correctness(dtype):
    """tests/test_acceptance.py:139-168: uniform KS, normal moments and radial
    chi2(2) law (float64 and the float32 extension), exponential means."""
    grid = sf.WorkGrid(8, 8)
    uni = sf.fill_uniform(fresh(64), sf.FillRequest(shape=100_000, grid=grid))
    assert scipy_stats.kstest(uni.vector(), "uniform").statistic < ks_bound(100_000)
    nbuf = sf.fill_normal(fresh(64), sf.FillRequest(shape=(1000, 1000), grid=grid, dtype=dtype))
    vals = nbuf.values.astype(np.float64)
    assert abs(vals.mean()) < 0.004
    assert 0.994 < vals.var() < 1.006
    radii = (vals[:, 0::2] ** 2 + vals[:, 1::2] ** 2).ravel()
    assert scipy_stats.kstest(radii, "chi2", args=(2,)).statistic < ks_bound(radii.size)
    for rate in (0.5, 1.0, 2.0):
        e = sf.fill_exponential(fresh(64), sf.FillRequest(shape=(1000, 1000), kind="exponential",
                                                          rate=rate, grid=grid)).values
        assert abs(e.mean() - 1 / rate) < 4 / (rate * 1000.0)


def test_exponential_is_inverse_cdf_of_the_uniform_fill():
    """tests/test_distributions.py:145-157: same states, -log1p(-u)/rate."""
    g = sf.WorkGrid(4, 4)
    base = fresh(16)
    u = sf.fill_uniform(base.copy(), sf.FillRequest(shape=(33, 47), grid=g)).values
    e = sf.fill_exponential(base.copy(), sf.FillRequest(shape=(33, 47), kind="exponential",
                                                        rate=2.5, grid=g)).values
    want = np.array([-math.log1p(-x) / 2.5 for x in u.ravel()]).reshape(u.shape)
    assert np.array_equal(e, want)  # libm log1p == the device port, bit for bit


# ------------------------------------------------------------------ rcont2
def test_rcont2_single_row_forced_without_uniforms():
    """tests/test_fisher.py:69-74."""
    state = np.array([12345] * 6, dtype=np.int64)
    before = state.copy()
    table = sf.rcont2([7], [2, 2, 3], state)
    assert np.array_equal(table, [[2, 2, 3]])
    assert np.array_equal(state, before)


def test_rcont2_margin_mismatch_rejected():
    """tests/test_fisher.py:76-78."""
    with pytest.raises(InvalidMarginsError):
        sf.rcont2([3, 3], [2, 2], np.array([12345] * 6, dtype=np.int64))


def test_rcont2_consumes_one_uniform_per_free_cell():
    """tests/test_fisher.py:89-95: a 3x3 table advances the state 4 steps."""
    s = fresh(1)
    state = s.current[0].copy()
    sf.rcont2([5, 7, 3], [6, 4, 5], state)
    want = s[0]
    for _ in range(4):
        want, _ = sf.next_state(want)
    assert tuple(state[:3]) == want.g1 and tuple(state[3:]) == want.g2


def test_acceptance_07_table_sampler_distribution(month_table):
    """tests/test_acceptance.py:111-136: margins preserved over 100 month
    tables; the 2x2 [5,5]x[5,5] law matches the hypergeometric pmf (chi2)."""
    rm, cm = month_table.sum(1), month_table.sum(0)
    state = np.array([12345] * 6, dtype=np.int64)
    lf = log_factorial_table(int(month_table.sum()))
    for _ in range(100):
        t = sf.rcont2(rm, cm, state, lf)
        assert np.array_equal(t.sum(1), rm) and np.array_equal(t.sum(0), cm)

    def pmf(k):
        return math.exp(2 * gammaln(6) + 2 * gammaln(6) - gammaln(11)
                        - 2 * gammaln(k + 1) - 2 * gammaln(6 - k))

    counts = np.zeros(6, dtype=np.int64)
    lf10 = log_factorial_table(10)
    for _ in range(100_000):
        counts[sf.rcont2([5, 5], [5, 5], state, lf10)[0, 0]] += 1
    expected = np.array([pmf(k) for k in range(6)]) * counts.sum()
    chi2 = ((counts - expected) ** 2 / expected).sum()
    assert scipy_stats.chi2.sf(chi2, df=5) > 0.001


# ------------------------------------------------------------------ fisher
def test_fisher_thresholds(month_table, week_table):
    """tests/test_acceptance.py:105-108 / test_fisher.py:37-41."""
    assert round(sf.logfact_sum(month_table)) == -47955
    assert round(sf.logfact_sum(week_table)) == -54990


def test_fisher_sim_num_rounding_and_p_value(month_table):
    """tests/test_fisher.py:114-134."""
    r = sf.fisher_sim(month_table, 2000, fresh(16), grid=sf.WorkGrid(4, 4))
    assert r.sim_num == 2000
    r = sf.fisher_sim(month_table, 2001, fresh(16), grid=sf.WorkGrid(4, 4))
    assert r.sim_num == 2016
    assert r.p_value == (1 + r.counts) / (r.sim_num + 1)


def test_fisher_invalid_replicates_and_streams(month_table):
    """tests/test_fisher.py:136-142."""
    with pytest.raises(InvalidArgumentError):
        sf.fisher_sim(month_table, 0, fresh(16), grid=sf.WorkGrid(4, 4))
    with pytest.raises(InsufficientStreamsError):
        sf.fisher_sim(month_table, 100, fresh(4), grid=sf.WorkGrid(4, 4))


def test_fisher_thread_count_invariance(month_table):
    """tests/test_fisher.py:166-178: `threads=` never changes results."""
    a = sf.fisher_sim(month_table, 512, fresh(16), grid=sf.WorkGrid(4, 4), threads=1,
                      return_stats=True)
    b = sf.fisher_sim(month_table, 512, fresh(16), grid=sf.WorkGrid(4, 4), threads=8,
                      return_stats=True)
    assert a.counts == b.counts and np.array_equal(a.statistics, b.statistics)


def test_acceptance_04_05_month_and_week_benchmarks(month_table, week_table):
    """tests/test_acceptance.py:87-102: the paper's Fisher benchmarks."""
    m = sf.fisher_sim(month_table, 10 ** 6, fresh(16384), grid=sf.WorkGrid(256, 64))
    assert m.sim_num == 1015808
    assert 0.400 <= m.p_value <= 0.407
    w = sf.fisher_sim(week_table, 10 ** 7, fresh(16384), grid=sf.WorkGrid(256, 64))
    assert w.sim_num == 10010624
    assert 1.0e-4 <= w.p_value <= 1.7e-4
